"""Thin wrapper of the tcgen05 GEMM (`ap_gemm_tf32`, csrc/gemm_tc.cu)."""

from __future__ import annotations

from . import _native


def gemm(a, b, *, trans_a: bool = False, trans_b: bool = False, bias=None, relu: bool = False,
         precision: int = 3, out=None, stream=None):
    """op(a) @ op(b) (+ bias) (ReLU) on the tensor cores; fp32 CUDA tensors, row-major.

    op(a) is [M, K] (a is [K, M] when trans_a), op(b) is [K, N] (b is [N, K]
    when trans_b).  precision 3 = 3xTF32 (fp32-accurate), 1 = TF32.
    """
    import torch

    if a.dtype != torch.float32 or b.dtype != torch.float32:
        raise TypeError("gemm expects fp32 tensors")
    if a.stride(1) != 1 or b.stride(1) != 1:
        raise ValueError("gemm expects unit stride along the last dim")
    m, k = (a.shape[1], a.shape[0]) if trans_a else (a.shape[0], a.shape[1])
    kb, n = (b.shape[1], b.shape[0]) if trans_b else (b.shape[0], b.shape[1])
    if k != kb:
        raise ValueError(f"inner dims differ: {k} vs {kb}")
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device=a.device)
    lib = _native.require_device()
    _native.check(lib.ap_gemm_tf32(_native.ptr(a), a.stride(0), int(trans_a), _native.ptr(b), b.stride(0),
                                   int(trans_b), _native.ptr(out), out.stride(0), m, n, k,
                                   _native.ptr(bias) if bias is not None else None, int(relu), int(precision),
                                   _native.stream_handle(stream)))
    return out
