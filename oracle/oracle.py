"""CPU ORACLE — test infrastructure only.

ctypes front-end of `liboracle.so` (ap_oracle.c, the C restatement of the
reference propagation, sharding.py:155-302) plus pure-Python restatements
of small reference pieces.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s cpu_baseline leg may import this module; the product package
never does.  Pinned against the reference's own outputs in `tests/golden/`.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

ORACLE_DIR = Path(__file__).resolve().parent
LIB = ORACLE_DIR / "liboracle.so"
_lib = None


def build() -> Path:
    srcs = list(ORACLE_DIR.glob("*.c"))
    if not LIB.exists() or LIB.stat().st_mtime < max(s.stat().st_mtime for s in srcs):
        subprocess.run(["make", "-s", "-C", str(ORACLE_DIR)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(str(LIB))
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def propagate_batch(flat, seed_slots, seeds, cand_slots, init_state=None):
    """Reference-order propagation of every row of `seeds` ([B, len(seed_slots)] int8).

    Returns (state [B, S] int8, outcome [B] int32, site [B] int32 position or -1).
    """
    seeds = np.ascontiguousarray(seeds, dtype=np.int8)
    if seeds.ndim == 1:
        seeds = seeds[None, :]
    b = seeds.shape[0]
    s = flat.num_slots
    seed_slots = np.ascontiguousarray(seed_slots, dtype=np.int64)
    cand_slots = np.ascontiguousarray(cand_slots, dtype=np.int64)
    state = np.empty((b, max(s, 1)), dtype=np.int8)
    outcome = np.empty(b, dtype=np.int32)
    site = np.empty(b, dtype=np.int32)
    init = None if init_state is None else np.ascontiguousarray(init_state, dtype=np.int8)
    rc = lib().orc_propagate(
        ctypes.c_int(flat.num_instructions), _p(flat.opcode), _p(flat.rank), _p(flat.dims_offset),
        _p(flat.dims if flat.dims.size else np.zeros(1, np.int64)), _p(flat.operand_offset),
        _p(flat.operands if flat.operands.size else np.zeros(1, np.int32)), _p(flat.gte_element),
        ctypes.c_int(len(seed_slots)), _p(seed_slots), _p(seeds), ctypes.c_int64(b), ctypes.c_int(len(cand_slots)),
        _p(cand_slots), None if init is None else _p(init), _p(state), _p(outcome), _p(site),
    )
    if rc != 0:
        raise RuntimeError(f"oracle propagate failed rc={rc}")
    return state[:, :s], outcome, site


# -- pure-Python restatements --------------------------------------------------


def cpython_sum(xs) -> float:
    """CPython >= 3.12 builtin sum() over floats (compensated, Neumaier).

    Restates Python/bltinmodule.c builtin_sum_impl: the int start value 0 is
    folded into the first float, then Neumaier compensation, and the
    compensation is added at the end only when non-zero and finite.  Used by
    reference pipecost.py:173-174,225.
    """
    it = iter(xs)
    try:
        first = next(it)
    except StopIteration:
        return 0
    total = 0 + first
    comp = 0.0
    for x in it:
        t = total + x
        if abs(total) >= abs(x):
            comp += (total - t) + x
        else:
            comp += (x - t) + total
        total = t
    if comp and comp not in (float("inf"), float("-inf")) and comp == comp:
        total += comp
    return total
