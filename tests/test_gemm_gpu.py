"""tcgen05 GEMM numerics against a plain PyTorch fp64 reference of the same op."""

import pytest
import torch

from paper_2007_04069_b200.tc import gemm

pytestmark = pytest.mark.gpu

SHAPES = [
    (64, 256, 1060),   # Q-net layer 0 forward, batch 64, BERT-48 OPP state
    (64, 256, 256),    # layer 1
    (64, 3, 256),      # dueling heads (V + 2 advantages)
    (1060, 256, 64),   # dW0 = x^T dz
    (300, 40, 77),     # ragged everything
    (4096, 256, 1060), # batched act over 4096 envs
    (128, 2193, 256),  # PP-train advantage head (2192 actions + value)
]


def ref(a, b, ta, tb, bias, relu):
    x = (a.t() if ta else a).double() @ (b.t() if tb else b).double()
    if bias is not None:
        x = x + bias.double()
    if relu:
        x = x.clamp_min(0.0)
    return x


@pytest.mark.parametrize("m,n,k", SHAPES)
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True)])
def test_gemm_3xtf32_matches_fp64(cuda, m, n, k, ta, tb):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    a = torch.randn((k, m) if ta else (m, k), device="cuda", generator=g)
    b = torch.randn((n, k) if tb else (k, n), device="cuda", generator=g)
    bias = torch.randn(n, device="cuda", generator=g)
    out = gemm(a, b, trans_a=ta, trans_b=tb, bias=bias, relu=True, precision=3)
    r = ref(a, b, ta, tb, bias, True)
    err = (out.double() - r).abs().max().item()
    scale = (a.abs().double().t() if not ta else a.abs().double()).shape  # noqa: F841
    # fp32-level tolerance: |err| <= 1e-5 * sqrt(k) * |a||b| typical magnitude
    tol = 2e-5 * (k ** 0.5) * 4.0
    assert err < tol, (err, tol)


@pytest.mark.parametrize("m,n,k", SHAPES + [(64, 1060, 256), (257, 33, 1060)])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_pipelined_kernel_matches_simple_kernel(cuda, m, n, k, ta, tb, monkeypatch):
    """cp.async / split-K kernel (gemm_tc2.cu) vs the simple kernel (gemm_tc.cu), both vs fp64."""
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    a = torch.randn((k, m) if ta else (m, k), device="cuda", generator=g)
    b = torch.randn((n, k) if tb else (k, n), device="cuda", generator=g)
    for prec in (1, 3):
        fast = gemm(a, b, trans_a=ta, trans_b=tb, precision=prec)
        monkeypatch.setenv("AP_GEMM_V1", "1")
        slow = gemm(a, b, trans_a=ta, trans_b=tb, precision=prec)
        monkeypatch.delenv("AP_GEMM_V1")
        r = ref(a, b, ta, tb, None, False)
        scale = r.abs().max().item()
        tol = (2e-5 if prec == 3 else 5e-3) * scale
        assert (fast.double() - r).abs().max().item() < tol
        assert (slow.double() - r).abs().max().item() < tol


@pytest.mark.parametrize("m,n,k", SHAPES + [(128, 256, 1060), (1061, 256, 64), (257, 3, 64), (5, 7, 9),
                                            (4096, 3, 256)])
def test_tma_kernel_matches_cp_async_kernel(cuda, m, n, k, monkeypatch):
    """TMA-fed SW128 kernel (gemm_tc3.cu, TF32, K-major) vs the cp.async kernel and fp64."""
    g = torch.Generator(device="cuda").manual_seed(3 * m + n + 7 * k)
    a = torch.randn((m, k), device="cuda", generator=g)
    b = torch.randn((n, k), device="cuda", generator=g)
    bias = torch.randn(n, device="cuda", generator=g)
    tma = gemm(a, b, trans_b=True, bias=bias, relu=True, precision=1)
    monkeypatch.setenv("AP_GEMM_NO_TMA", "1")
    cpa = gemm(a, b, trans_b=True, bias=bias, relu=True, precision=1)
    monkeypatch.delenv("AP_GEMM_NO_TMA")
    r = ref(a, b, False, True, bias, True)
    scale = r.abs().max().item()
    assert (tma.double() - r).abs().max().item() < 5e-3 * scale
    assert (tma - cpa).abs().max().item() <= 1e-5 * scale


@pytest.mark.parametrize("m,n,k", [(64, 256, 1060), (128, 256, 1060), (64, 256, 256), (200, 40, 777)])
def test_cluster_splitk_matches_workspace_splitk(cuda, m, n, k, monkeypatch):
    """Split-K reduced through DSMEM inside a thread-block cluster == split-K through a
    global workspace + reduce kernel (same splits, same fixed order: bit-identical)."""
    g = torch.Generator(device="cuda").manual_seed(m * n + k)
    a = torch.randn((m, k), device="cuda", generator=g)
    b = torch.randn((n, k), device="cuda", generator=g)
    bias = torch.randn(n, device="cuda", generator=g)
    clu = gemm(a, b, trans_b=True, bias=bias, relu=True, precision=1)
    monkeypatch.setenv("AP_GEMM_NO_CLUSTER", "1")
    monkeypatch.setenv("AP_GEMM_MAX_SPLIT", "16")
    ws = gemm(a, b, trans_b=True, bias=bias, relu=True, precision=1)
    r = ref(a, b, False, True, bias, True)
    assert (clu.double() - r).abs().max().item() < 5e-3 * r.abs().max().item()
    assert torch.equal(clu, ws)


@pytest.mark.parametrize("m,n,k", SHAPES[:4])
def test_gemm_tf32_is_tf32_accurate(cuda, m, n, k):
    g = torch.Generator(device="cuda").manual_seed(1)
    a = torch.randn((m, k), device="cuda", generator=g)
    b = torch.randn((k, n), device="cuda", generator=g)
    out = gemm(a, b, precision=1)
    r = ref(a, b, False, False, None, False)
    rel = ((out.double() - r).abs().max() / r.abs().max()).item()
    assert rel < 5e-3
    out3 = gemm(a, b, precision=3)
    rel3 = ((out3.double() - r).abs().max() / r.abs().max()).item()
    assert rel3 < 1e-5 and rel3 < rel


@pytest.mark.parametrize("m,n,k", [(12681, 256, 64), (1024, 3171, 256), (257, 3171, 64), (300, 130, 1060),
                                   (64, 256, 1060)])
def test_bn128_tiles_match_bn64(cuda, m, n, k, monkeypatch):
    """BN = 128 tiles (picked automatically when they need fewer waves) vs BN = 64 tiles and fp64:
    the same k order per output element, so bit-identical without split-K."""
    g = torch.Generator(device="cuda").manual_seed(m + 3 * n + k)
    a = torch.randn((m, k), device="cuda", generator=g)
    b = torch.randn((n, k), device="cuda", generator=g)
    bias = torch.randn(n, device="cuda", generator=g)
    outs = []
    for bn in ("64", "128"):
        monkeypatch.setenv("AP_GEMM_V3_BN", bn)
        outs.append(gemm(a, b, trans_b=True, bias=bias, relu=True, precision=1))
    r = ref(a, b, False, True, bias, True)
    assert (outs[1].double() - r).abs().max().item() < 5e-3 * r.abs().max().item()
    assert (outs[1] - outs[0]).abs().max().item() <= 1e-5 * r.abs().max().item()


@pytest.mark.parametrize("m,n,k", [(4096, 256, 1060), (4096, 256, 256), (257, 256, 64), (1000, 512, 96),
                                   (300, 256, 1060)])
def test_a_multicast_matches_plain(cuda, m, n, k, monkeypatch):
    """A-tile multicast across a 4-CTA cluster (each CTA loads a quarter of the A tile for all four)
    == the one-CTA kernel, bit for bit (same MMAs in the same k order)."""
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    a = torch.randn((m, k), device="cuda", generator=g)
    b = torch.randn((n, k), device="cuda", generator=g)
    bias = torch.randn(n, device="cuda", generator=g)
    monkeypatch.setenv("AP_GEMM_MC", "1")
    mc = gemm(a, b, trans_b=True, bias=bias, relu=True, precision=1)
    monkeypatch.delenv("AP_GEMM_MC")
    monkeypatch.setenv("AP_GEMM_NO_MC", "1")
    plain = gemm(a, b, trans_b=True, bias=bias, relu=True, precision=1)
    assert torch.equal(mc, plain)
    r = ref(a, b, False, True, bias, True)
    assert (mc.double() - r).abs().max().item() < 5e-3 * r.abs().max().item()
