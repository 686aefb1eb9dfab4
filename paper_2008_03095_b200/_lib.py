"""ctypes binding of libinfuser_b200.so (declared in include/infuser_b200.h).

The library is the only compute path of this package: there is no CPU
fallback.  Importing the package works without a GPU (so host-side logic can
be tested), but every call that needs the device raises ``RuntimeError``
when the library is missing or no sm_100 device is visible.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

LIB_NAME = "libinfuser_b200.so"
LIB_PATH = Path(__file__).resolve().parent / "lib" / LIB_NAME

IMX_OK = 0
IMX_EINVAL = -1
IMX_ENOMEM = -2
IMX_ECUDA = -3
IMX_ENODEV = -4
IMX_ECONSTRAINT = -5
IMX_EFORMAT = -6
IMX_EINTERNAL = -7
IMX_ENCCL = -8
COMM_ID_BYTES = 128

MODE_NAMES = {0: "init", 1: "hook", 2: "compress", 3: "verify"}

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_f64 = ctypes.c_double
c_f32 = ctypes.c_float
c_void_p = ctypes.c_void_p
P = ctypes.POINTER


class PropStats(ctypes.Structure):
    _fields_ = [("sweeps", c_i32), ("cap", c_i32),
                ("changed_pairs", P(c_i64)), ("label_sums", P(c_i64)),
                ("modes", P(c_i32))]


class Timings(ctypes.Structure):
    _fields_ = [("propagate_ms", c_f32), ("memoize_ms", c_f32), ("select_ms", c_f32),
                ("init_ms", c_f32), ("hook_ms", c_f32), ("compress_ms", c_f32),
                ("kernel_launches", c_i64), ("hook_launches", c_i64),
                ("celf_evaluations", c_i64)]


# name -> (restype, argtypes)
_SIGNATURES = {
    "imx_last_error": (ctypes.c_char_p, []),
    "imx_version": (c_i32, []),
    "imx_device_count": (c_i32, []),
    "imx_launch_count": (c_i64, []),
    "imx_graph_from_edges": (c_i32, [c_i32, c_i64, c_void_p, c_i64, c_void_p, c_f64, P(c_void_p)]),
    "imx_graph_from_csr": (c_i32, [c_i32, c_i64, c_i64, c_void_p, c_void_p, c_void_p, P(c_void_p)]),
    "imx_graph_generate": (c_i32, [c_i32, c_i32, c_i64, c_i64, c_i64, ctypes.c_uint64, c_void_p, c_void_p,
                                   P(c_void_p)]),
    "imx_graph_destroy": (None, [c_void_p]),
    "imx_graph_dims": (c_i32, [c_void_p, P(c_i64), P(c_i64)]),
    "imx_graph_get_csr": (c_i32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "imx_graph_reciprocal": (c_i32, [c_void_p, c_void_p]),
    "imx_graph_set_weights": (c_i32, [c_void_p, c_void_p]),
    "imx_graph_hashes": (c_i32, [c_void_p, c_void_p]),
    "imx_graph_set_hashes": (c_i32, [c_void_p, c_void_p]),
    "imx_graph_thresholds": (c_i32, [c_void_p, c_i32, c_void_p, P(c_i32)]),
    "imx_murmur3_pairs": (c_i32, [c_i32, c_void_p, c_void_p, c_i64, c_void_p]),
    "imx_create": (c_i32, [c_void_p, c_void_p, c_i32, c_i32, P(c_void_p)]),
    "imx_destroy": (None, [c_void_p]),
    "imx_propagate": (c_i32, [c_void_p, c_i32, P(PropStats)]),
    "imx_memoize": (c_i32, [c_void_p, c_void_p]),
    "imx_set_fuse_memo": (c_i32, [c_void_p, c_i32]),
    "imx_spec_defer": (c_i32, [c_void_p, c_i32]),
    "imx_spec_settle": (c_i32, [c_void_p, P(c_i32)]),
    "imx_load_labels": (c_i32, [c_void_p, c_void_p, c_void_p, c_i64]),
    "imx_copy_labels": (c_i32, [c_void_p, c_i32, c_i32, c_void_p]),
    "imx_copy_sizes": (c_i32, [c_void_p, c_i32, c_i32, c_void_p]),
    "imx_celf_reset": (c_i32, [c_void_p, c_void_p]),
    "imx_celf_top": (c_i32, [c_void_p, P(c_i64), P(c_i32)]),
    "imx_celf_prefix": (c_i32, [c_void_p, c_i64, c_i64, c_void_p, c_void_p, c_void_p, P(c_i64)]),
    "imx_celf_advance": (c_i32, [c_void_p, c_i64, c_i32, c_void_p, c_void_p, c_i64, P(c_i64)]),
    "imx_eval_gains": (c_i32, [c_void_p, c_void_p, c_i64, c_void_p]),
    "imx_commit": (c_i32, [c_void_p, c_i32, P(c_i64)]),
    "imx_celf_select": (c_i32, [c_void_p, c_i32, c_void_p, c_void_p, P(c_i64)]),
    "imx_celf_select_sharded": (c_i32, [c_void_p, c_i32, c_void_p, c_void_p, c_void_p, c_void_p, P(c_i64)]),
    "imx_celf_trace": (c_i32, [c_void_p, c_void_p, c_i64]),
    "imx_celf_trace_take": (c_i32, [c_void_p, P(c_void_p), P(c_i64)]),
    "imx_host_free": (None, [c_void_p]),
    "imx_per_sim": (c_i32, [c_void_p, c_void_p]),
    "imx_copy_owned": (c_i32, [c_void_p, c_void_p]),
    "imx_evaluate_seeds": (c_i32, [c_void_p, c_void_p, c_i32, c_i64, c_void_p, c_i64, c_void_p]),
    "imx_sampling_cdf": (c_i32, [c_void_p, c_void_p, c_i32, c_i64, c_i32, c_void_p, c_void_p, P(c_f64),
                                 P(c_i64)]),
    "imx_edge_list_parse": (c_i32, [ctypes.c_char_p, P(c_void_p), P(c_i64), P(c_i32), P(c_i64), c_void_p, c_i64]),
    "imx_edge_list_dims": (c_i32, [c_void_p, P(c_i64), P(c_i64)]),
    "imx_edge_list_copy": (c_i32, [c_void_p, c_void_p, c_void_p, c_void_p]),
    "imx_edge_list_free": (None, [c_void_p]),
    "imx_get_timings": (c_i32, [c_void_p, P(Timings)]),
    "imx_comm_unique_id": (c_i32, [c_void_p]),
    "imx_comm_create": (c_i32, [c_i32, c_i32, c_i32, c_void_p, P(c_void_p)]),
    "imx_local_group_create": (c_i32, [c_i32, P(c_void_p)]),
    "imx_local_group_destroy": (None, [c_void_p]),
    "imx_comm_create_local": (c_i32, [c_void_p, c_i32, c_i32, P(c_void_p)]),
    "imx_comm_destroy": (None, [c_void_p]),
    "imx_comm_allreduce": (c_i32, [c_void_p, c_void_p, c_i64]),
    "imx_ctx_attach_comm": (c_i32, [c_void_p, c_void_p]),
    "imx_celf_select_comm": (c_i32, [c_void_p, c_i32, c_void_p, c_void_p, P(c_i64)]),
    "imx_bench_propagate": (c_i32, [c_void_p, c_i32, c_i32, P(c_f32), P(c_f32), P(c_f32), P(c_f32)]),
}

EXPORTED = tuple(_SIGNATURES)

_lib = None


def library_path() -> Path:
    return Path(os.environ.get("INFUSER_B200_LIB", LIB_PATH))


def load(path=None):
    """Load (once) and return the ctypes library; raises if it is not built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path is not None else library_path()
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); "
            "this package has no CPU fallback")
    lib = ctypes.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path is None:
        _lib = lib
    return lib


class ConstraintError(ValueError):
    """A structurally valid request that violates a documented limit
    (graph.py:33-34 of the reference)."""


class GraphFormatError(ValueError):
    """Unreadable or malformed graph input (graph.py:29-30)."""


def check(rc: int) -> None:
    """Map an IMX_E* return code to the exception the reference raises."""
    if rc == IMX_OK:
        return
    msg = (load().imx_last_error() or b"").decode("utf-8", "replace")
    if rc == IMX_EINVAL:
        raise ValueError(msg)
    if rc == IMX_ECONSTRAINT:
        raise ConstraintError(msg)
    if rc == IMX_EFORMAT:
        raise GraphFormatError(msg)
    if rc == IMX_ENOMEM:
        raise MemoryError(msg)
    if rc == IMX_EINTERNAL:
        raise AssertionError(msg)
    if rc == IMX_ENCCL:
        raise RuntimeError(msg)
    raise RuntimeError(msg or f"libinfuser_b200 error {rc}")


def ptr(a: np.ndarray | None):
    """Raw data pointer of a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return ctypes.c_void_p(a.ctypes.data)


_device = None


def current_device() -> int:
    """CUDA device used by new graphs/contexts: set_device(), else LOCAL_RANK."""
    if _device is not None:
        return _device
    return int(os.environ.get("INFUSER_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def set_device(device: int) -> None:
    global _device
    _device = int(device)


_have_device = None


def require_device() -> None:
    global _have_device
    if _have_device is None:
        _have_device = load().imx_device_count() > 0
    if not _have_device:
        raise RuntimeError("no sm_100 CUDA device visible: libinfuser_b200 has no "
                           "CPU fallback")
