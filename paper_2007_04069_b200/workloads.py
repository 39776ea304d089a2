"""Deterministic synthetic plan batches (SURVEY §8(d) "plan batches").

A plan-batch row is a seed vector over the candidate dims: a prefix of the
decision order (length k ~ U[1, |D|]) is seeded with iid fair P/R coins,
the rest stays unseeded — the shape of an OPP episode's state after k
decisions.  Rows come from a counter-based 32-bit hash evaluated with exact
int64 torch ops, so the same (seed, row index) gives the same row on the
GPU (bench arm) and on the CPU (reference arm), with no host RNG pass over
gigabytes of seeds.
"""

from __future__ import annotations

import numpy as np

BATCH_SEED = 20201007
_M32 = 0xFFFFFFFF


def _mulmod32(x, c: int):
    """(x * c) mod 2^32 for int64 x in [0, 2^32) without int64 overflow."""
    lo = x * (c & 0xFFFF)
    hi = ((x * (c >> 16)) & 0xFFFF) << 16
    return (lo + hi) & _M32


def mix32(x):
    """A 32-bit avalanche mixer (xorshift-multiply), exact in int64 arithmetic."""
    x = x ^ (x >> 16)
    x = _mulmod32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mulmod32(x, 0x846CA68B)
    return x ^ (x >> 16)


def prefix_seed_batch(order, start: int, count: int, seed: int = BATCH_SEED, device="cpu", chunk: int = 1 << 16,
                      kmax: int | None = None):
    """Rows [start, start+count) of the synthetic prefix batch as int8 [count, |D|].

    `order` is the decision order as flat candidate indices (e.g.
    `sorted_decision_order`); column `order[j]` belongs to prefix position j.
    Prefix lengths are k ~ U[1, min(|D|, kmax)] (kmax=None: the whole order).
    """
    import torch

    order_t = torch.as_tensor(np.asarray(order, dtype=np.int64), device=device)
    n = int(order_t.numel())
    # rows padded to a 16-byte stride (the fast kernel's vector loads); the view hides the pad
    out = torch.full((count, max(16, (n + 15) // 16 * 16)), -1, dtype=torch.int8, device=device)[:, :n]
    pos = torch.arange(n, dtype=torch.int64, device=device)
    s0 = mix32(torch.tensor(seed & _M32, dtype=torch.int64))
    s1 = mix32(s0 ^ 0x5BD1E995)
    for lo in range(0, count, chunk):
        hi = min(count, lo + chunk)
        rows = torch.arange(start + lo, start + hi, dtype=torch.int64, device=device)
        k = 1 + mix32(mix32((rows & _M32) ^ s0.to(device)) ^ (rows >> 32)) % min(n, kmax or n)
        e = rows[:, None] * n + pos[None, :]
        bits = mix32(mix32((e & _M32) ^ s1.to(device)) ^ (e >> 32)) & 1
        ordered = torch.where(pos[None, :] < k[:, None], bits, torch.full_like(bits, -1)).to(torch.int8)
        out[lo:hi, order_t] = ordered
    return out


def trigger_seed_batch(num_dims: int, start: int, count: int, device="cpu"):
    """Rows [start, start+count) of the 2*|D| linkage triggers tiled over the batch (row r is
    trigger r mod 2|D|: dim (r mod 2|D|) // 2 seeded P for even, R for odd), int8 [count, |D|]."""
    import torch

    n = num_dims
    out = torch.full((count, max(16, (n + 15) // 16 * 16)), -1, dtype=torch.int8, device=device)[:, :n]
    t = torch.arange(start, start + count, dtype=torch.int64, device=device) % (2 * n)
    rows = torch.arange(count, dtype=torch.int64, device=device)
    out[rows, t // 2] = (1 - (t % 2)).to(torch.int8)
    return out


def trigger_batch(num_dims: int):
    """The 2*|D| linkage triggers (row 2k: dim k P, row 2k+1: dim k R)."""
    from .linkage import trigger_matrix

    return trigger_matrix(num_dims)
