"""The vector trainer's act GEMM alone: [4096, 1060] x [1060, 256] TF32 (tcgen05, TMA A-multicast).

    python profiles/probes/act_gemm.py [LAUNCHES]

CUDA-event time per launch over back-to-back launches (operands L2-resident after the first),
achieved TF32 TFLOP/s and operand bytes per CTA.  AP_GEMM_MC_STAGES=8 selects the 8-stage ring.
"""

import os
import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2007_04069_b200 import tc  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    M, K, N = 4096, 1060, 256
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randn((M, K), device="cuda", generator=g)
    w = torch.randn((N, K), device="cuda", generator=g) * 0.03
    out = torch.empty((M, N), device="cuda")
    for _ in range(10):
        tc.gemm(a, w, trans_b=True, precision=1, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        tc.gemm(a, w, trans_b=True, precision=1, out=out)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    ref = a @ w.T
    err = ((out - ref).abs().max() / ref.abs().max()).item()
    per_cta = (128 + 64) * K * 4
    print(f"stages={os.environ.get('AP_GEMM_MC_STAGES', '6')}: {us:.2f} us/launch, "
          f"{2 * M * N * K / us / 1e6:.1f} TFLOP/s TF32, operand bytes per CTA {per_cta / 1e3:.0f} KB "
          f"({per_cta / us / 1e3:.1f} GB/s per SM), max rel err vs fp32 {err:.2e}")


if __name__ == "__main__":
    main()
