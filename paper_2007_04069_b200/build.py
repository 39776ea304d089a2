"""Build the native engine in-tree: `libautoplan_b200.so` (sm_100a).

Every `.cu` / `.cpp` under `csrc/` is compiled by nvcc with
`-gencode arch=compute_100a,code=sm_100a -lineinfo` and linked into one
shared library exporting the C-ABI of `include/autoplan_b200.h`.  The `.so`
lands next to this file so it travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
CSRC = PKG_DIR / "csrc"
BUILD_DIR = PKG_DIR / "_build"
LIB_NAME = "libautoplan_b200.so"
LIB_PATH = PKG_DIR / LIB_NAME
INCLUDE_DIR = PKG_DIR.parent / "include"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", f"-I{INCLUDE_DIR}"]
# fp64 cost kernels must round every add / mul separately (bit parity with CPython)
PER_FILE = {"pipecost.cu": ["-fmad=false"], "dqn.cu": ["--expt-relaxed-constexpr"],
            # numpy's samplers round every product / sum separately (no FMA in its baseline build)
            "dataplane.cu": ["-fmad=false"], "parity.cu": ["-fmad=false"]}


def _nvcc() -> str:
    found = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(found):
        raise RuntimeError("nvcc not found; the CUDA toolkit is required to build the engine")
    return found


def _sources() -> list[Path]:
    return sorted(list(CSRC.glob("*.cu")) + list(CSRC.glob("*.cpp")))


def _headers() -> list[Path]:
    return sorted(list(CSRC.glob("*.h")) + list(CSRC.glob("*.cuh")) + list(INCLUDE_DIR.glob("*.h")))


def build(force: bool = False, verbose: bool = False) -> Path:
    """Compile changed sources and relink; returns the library path."""
    nvcc = _nvcc()
    BUILD_DIR.mkdir(exist_ok=True)
    newest_header = max((h.stat().st_mtime for h in _headers()), default=0.0)
    objects = []
    relink = force or not LIB_PATH.exists()
    for src in _sources():
        obj = BUILD_DIR / (src.name + ".o")
        objects.append(obj)
        stale = force or not obj.exists() or obj.stat().st_mtime < max(src.stat().st_mtime, newest_header)
        if not stale:
            continue
        cmd = [nvcc, *ARCH, *COMMON, *PER_FILE.get(src.name, []), "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        relink = True
    if not relink and LIB_PATH.stat().st_mtime < max(o.stat().st_mtime for o in objects):
        relink = True
    if relink:
        tmp = LIB_PATH.with_suffix(".so.tmp")
        cmd = [nvcc, *ARCH, "-shared", "-o", str(tmp), *map(str, objects)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB_PATH)
