"""CELF over an attached NCCL communicator (one rank) vs the single-rank
persistent kernel: wall time of the selection on a config (host loop cost
of the sharded path)."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2008_03095_b200 as imx
from paper_2008_03095_b200 import _lib, configs
from paper_2008_03095_b200._lib import check
from paper_2008_03095_b200.celf import NativeComm
from paper_2008_03095_b200.context import DeviceContext

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
c = configs.CONFIGS[cfg]
g = configs.build(cfg)
X = imx.SimulationRandoms(c.R, 0).values
imx.build_hash_table(g).bind(g)
lib = _lib.load()
idbuf = (ctypes.c_uint8 * _lib.COMM_ID_BYTES)()
check(lib.imx_comm_unique_id(idbuf))
h = ctypes.c_void_p()
check(lib.imx_comm_create(_lib.current_device(), 1, 0, idbuf, ctypes.byref(h)))
comm = NativeComm(h, 0, 1)
for mode in ("single", "comm", "single", "comm"):
    ctx = DeviceContext(g, X, c.R)
    ctx.propagate()
    if mode == "comm":
        ctx.attach_comm(comm)
    ctx.memoize(want_gains=False)
    ctx.celf_reset(None)
    t0 = time.perf_counter()
    s, gg, tr = ctx.celf_select_comm(c.K) if mode == "comm" else ctx.celf_select(c.K)
    dt = time.perf_counter() - t0
    print(f"{cfg} {mode:6s} select {dt * 1e3:8.2f} ms  trace {len(tr)}  evals {ctx.timings()['celf_evaluations']}  seeds {s[:4].tolist()}")
    ctx.close()
