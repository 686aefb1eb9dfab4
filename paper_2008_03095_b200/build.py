"""Build libinfuser_b200.so in-tree for sm_100a (nvcc, static cudart)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
SOURCES = [PKG / "csrc" / f for f in ("graph.cu", "gen.cu", "ctx.cu", "propagate.cu", "scan.cu", "memo.cu", "celf.cu", "comm.cu", "evaluation.cu", "upload.cu", "io.cpp")]
HEADERS = list((PKG / "csrc").glob("*.cuh")) + [PKG.parent / "include" / "infuser_b200.h"]
OUT = PKG / "lib" / "libinfuser_b200.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "-diag-suppress", "1444",
    "-ldl",
]


def _code_only(text: str) -> str:
    """C/C++ source without comments and with whitespace runs collapsed, so
    that documentation edits do not change the stamp (string literals are kept
    as they are)."""
    import re
    pat = re.compile(r'"(?:\\.|[^"\\])*"|\'(?:\\.|[^\'\\])*\'|//[^\n]*|/\*.*?\*/', re.S)
    text = pat.sub(lambda m: m.group(0) if m.group(0)[0] in "\"'" else " ", text)
    return " ".join(text.split())


def source_hash() -> str:
    """sha256 (16 hex) over the library's sources and headers (code only:
    comments and layout do not count) and the compiler flags: stamps the ncu
    summaries under profiles/ so bench.py can refuse a stale one (the GPU box
    has no git history)."""
    import hashlib
    h = hashlib.sha256(" ".join(NVCC_FLAGS).encode())
    for p in sorted(SOURCES + HEADERS, key=lambda q: q.name):
        h.update(p.name.encode())
        h.update(_code_only(p.read_text()).encode())
    return h.hexdigest()[:16]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not OUT.exists():
        return False
    t = OUT.stat().st_mtime
    return all(p.stat().st_mtime <= t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> Path:
    """One object per source, compiled in parallel (no device code crosses
    translation units), then one shared link."""
    if not force and up_to_date():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    objdir = OUT.parent / "obj"
    objdir.mkdir(exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f not in ("-shared", "-cudart", "static", "-ldl")]
    hdr_t = max(p.stat().st_mtime for p in HEADERS)
    jobs = []
    for src in SOURCES:
        obj = objdir / (src.name + ".o")
        if force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, hdr_t):
            cmd = [nvcc(), *compile_flags, "-c", "-o", str(obj), str(src)]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            jobs.append(subprocess.Popen(cmd))
    if any(j.wait() != 0 for j in jobs):
        raise subprocess.CalledProcessError(1, "nvcc")
    tmp = OUT.with_suffix(".so.tmp")
    link = [nvcc(), *NVCC_FLAGS, "-o", str(tmp), *(str(objdir / (s.name + ".o")) for s in SOURCES)]
    if verbose:
        print(" ".join(link), file=sys.stderr)
    subprocess.run(link, check=True)
    os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
