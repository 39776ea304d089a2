"""Fused small-batch Q-network kernels (csrc/fused_mlp.cu) against the fp64 reference and the
tensor-core GEMM learner.

* forward_fused: Q within 1e-5 of max|Q| of the reference's fp64 QNetwork.forward on the same
  weights and inputs (tests/golden/agent_qnet.npz, agent.py:93-109);
* one fused learn step == the GEMM learner step (3xTF32 tcgen05, agent.update_on_indices) on
  the same ring / sample: TD errors, loss, priorities and every gradient within fp32
  tolerance; Adam moments identical in sign pattern, parameters within lr-scaled tolerance;
* deterministic: two runs give identical bits.
"""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2007_04069_b200.agent import AgentConfig, DqnAgent, QNetwork, Transition

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(1e-30, np.abs(b).max()))


@pytest.mark.parametrize("tag", ["small", "opp_bert48"])
def test_forward_fused_matches_fp64_reference(cuda, tag):
    z = np.load(GOLDEN / "agent_qnet.npz")
    s, a, seed = z[f"{tag}_meta"]
    net = QNetwork(int(s), int(a), (256, 256), np.random.default_rng(int(seed)))
    x = torch.from_numpy(z[f"{tag}_x"]).float().cuda()
    q = net.forward_fused(x).double().cpu().numpy()
    assert rel(q, z[f"{tag}_q"]) < 1e-5
    q1 = net.forward_fused(x[:1]).double().cpu().numpy()
    assert rel(q1, z[f"{tag}_q"][:1]) < 1e-5


def _filled_agents(S, A, n, hidden=(256, 256), seed=4):
    cfg = AgentConfig(batch_size=64, buffer_capacity=256, lr=0.001, hidden=hidden)
    agents = [DqnAgent(cfg, S, A, seed) for _ in range(2)]
    rng = np.random.default_rng(seed + 1)
    for _ in range(n):
        mask = rng.random(A) < 0.7
        mask[rng.integers(A)] = True
        t = Transition(rng.uniform(-1, 1, S), int(rng.integers(A)), float(rng.normal()), rng.uniform(-1, 1, S),
                       bool(rng.random() < 0.1), mask)
        for ag in agents:
            ag.observe(t)
    agents[1].learner = "gemm"
    agents[1].net.fused_act = False
    return agents


@pytest.mark.parametrize("S,A,hidden", [(1060, 2, (256, 256)), (37, 5, (64, 48)), (300, 9, (128, 128, 96))])
def test_fused_learn_step_matches_gemm_learner(cuda, S, A, hidden):
    fused, gemm = _filled_agents(S, A, 200, hidden)
    for ag in (fused, gemm):
        ag.learn()
    torch.cuda.synchronize()
    assert fused.rng.bit_generator.state == gemm.rng.bit_generator.state
    assert rel(fused._fused.td.cpu(), gemm._batch.td.cpu()) < 1e-4
    assert rel(fused.net.grad.cpu(), gemm.net.grad.cpu()) < 1e-4
    pf, pg = fused.buffer.priorities, gemm.buffer.priorities
    assert rel(pf, pg) < 1e-4
    # the transposed copies the tensor-core path reads were refreshed by the fused Adam
    for k, w in fused.net.wt.items():
        assert torch.equal(w, fused.net.views[k].t()), k
    assert rel(fused.net.flat.cpu(), gemm.net.flat.cpu()) < 1e-2  # Adam's first step moves every weight by ~lr


def test_fused_learn_is_deterministic(cuda):
    a, b = _filled_agents(1060, 2, 150)
    b.learner = "fused"
    b.net.fused_act = True
    for _ in range(5):
        a.learn()
        b.learn()
    torch.cuda.synchronize()
    assert torch.equal(a.net.flat, b.net.flat) and torch.equal(a.optimizer.v, b.optimizer.v)
    assert np.array_equal(a.buffer.priorities, b.buffer.priorities)
