"""Profile arrays for PP-infer: prefix sums, right-endpoint coarsening, joint scaling.

Reference `autoplan.dataproc` (`pkg/src/autoplan/dataproc.py:52-145`).  This is
one-shot host preprocessing of 3 x 128 arrays (SURVEY §2 marks it out of the
hot path); it is kept so PipeInferEnv can be driven without the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GRANULARITY = 128


class ProfileError(Exception):
    """Malformed profile inputs."""


@dataclass(frozen=True)
class CoarsenedArrays:
    c: np.ndarray
    a: np.ndarray
    w: np.ndarray
    source_length: int

    @property
    def granularity(self) -> int:
        return len(self.c)


def coarsen(xs, target: int = GRANULARITY) -> np.ndarray:
    """Right-endpoint sampling: point i takes source index floor((i+1)*N/target)-1 (dataproc.py:79-96)."""
    arr = np.asarray(xs, dtype=np.float64)
    if target < 1 or arr.ndim != 1 or arr.size == 0:
        raise ProfileError("coarsen expects a non-empty 1-d array and target >= 1")
    if arr.size < target:
        arr = np.concatenate([arr, np.full(target - arr.size, arr[-1])])
    n = arr.size
    return arr[(np.arange(1, target + 1) * n) // target - 1]


def build_environment_arrays(c, a, w, granularity: int = GRANULARITY) -> CoarsenedArrays:
    """Prefix-sum C and W, coarsen all three, scale by the shared maximum (dataproc.py:99-120)."""
    cs = coarsen(np.cumsum(np.asarray(c, dtype=np.float64)), granularity)
    as_ = coarsen(np.asarray(a, dtype=np.float64), granularity)
    ws = coarsen(np.cumsum(np.asarray(w, dtype=np.float64)), granularity)
    peak = max(cs.max(initial=0.0), as_.max(initial=0.0), ws.max(initial=0.0))
    if peak > 0:
        cs, as_, ws = cs / peak, as_ / peak, ws / peak
    return CoarsenedArrays(cs, as_, ws, len(c))


def generate_environment(distribution: str, n: int, seed: int, granularity: int = GRANULARITY) -> CoarsenedArrays:
    """Synthetic U / N / B profile through the array pipeline (dataproc.py:123-145)."""
    if n < 1:
        raise ProfileError("environment length must be >= 1")
    rng = np.random.default_rng(seed)

    def draw():
        if distribution == "uniform":
            return rng.uniform(0.0, 1.0, n)
        if distribution == "normal":
            return np.clip(rng.normal(0.5, 0.15, n), 0.0, 1.0)
        if distribution == "binomial":
            return rng.binomial(100, 0.5, n) / 100
        raise ProfileError(f"unknown distribution {distribution!r}")

    c, a, w = draw(), draw(), draw()
    return build_environment_arrays(c, a, w, granularity)


def pcg64_states(seeds) -> np.ndarray:
    """[E, 4] uint64: numpy default_rng(seed)'s PCG64 (state hi, state lo, inc hi, inc lo) per seed."""
    seeds = list(seeds)
    out = np.empty((len(seeds), 4), dtype=np.uint64)
    mask = (1 << 64) - 1
    for i, s in enumerate(seeds):
        st = np.random.PCG64(s).state["state"]
        out[i] = (st["state"] >> 64, st["state"] & mask, st["inc"] >> 64, st["inc"] & mask)
    return out


def generate_environments_device(distribution: str, n: int, seeds, granularity: int = GRANULARITY, states=None):
    """generate_environment(distribution, n, s) for every seed s at once on the GPU
    (ap_generate_envs): a CUDA fp64 tensor [E, 3, G] of the scaled C, A, W arrays,
    bit-identical to the host path for all three distributions.  Uniform: one CTA per
    environment, PCG64 jump-ahead per thread; normal / binomial: numpy's ziggurat / BTPE
    samplers (data-dependent draw counts), one thread walking each environment's stream.
    `states` may pass precomputed pcg64_states(seeds)."""
    import torch

    from . import _native

    kinds = {"uniform": 0, "normal": 1, "binomial": 2}
    if distribution not in kinds:
        raise ProfileError(f"unknown distribution {distribution!r}")
    if n < 1:
        raise ProfileError("environment length must be >= 1")
    st = pcg64_states(seeds) if states is None else np.asarray(states, dtype=np.uint64)
    lib = _native.require_device()
    d_st = torch.from_numpy(st.view(np.int64)).cuda()
    out = torch.empty((st.shape[0], 3, granularity), dtype=torch.float64, device="cuda")
    _native.check(lib.ap_generate_envs(kinds[distribution], _native.ptr(d_st), st.shape[0], n, granularity,
                                       _native.ptr(out), _native.stream_handle()))
    return out
