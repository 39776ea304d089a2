"""Vectorised device episode driver vs the reference-exact single environments."""

import numpy as np
import pytest
import torch

from paper_2007_04069_b200 import graphs
from paper_2007_04069_b200.agent import AgentConfig
from paper_2007_04069_b200.envs import OppEnv
from paper_2007_04069_b200.vec import VecDqnTrainer, VecPartitionEnv

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["bert_base", "vgg19"])
def test_vec_env_matches_single_envs(cuda, name):
    g = graphs.generate(name)
    E = 24
    venv = VecPartitionEnv(g, E)
    singles = [OppEnv(g) for _ in range(E)]
    states = [s.reset() for s in singles]
    rng = np.random.default_rng(3)
    ep_ret = np.zeros(E, dtype=np.float32)  # the driver accumulates returns in fp32
    best = None  # (partitions, return, global episode id, statuses), cli.py:237-240 rule
    for step in range(60):
        np.testing.assert_array_equal(venv.cur_state.cpu().numpy(), np.array(states, dtype=np.float32))
        actions = rng.integers(0, 2, size=E).astype(np.int32)
        venv.step(torch.from_numpy(actions).cuda(), step_base=step * E)
        rewards = venv.rewards.cpu().numpy()
        done = venv.done.cpu().numpy()
        nxt = venv.next_state.cpu().numpy()
        for e, env in enumerate(singles):
            res = env.step(int(actions[e]))
            assert abs(rewards[e] - res.reward) < 1e-5
            assert bool(done[e]) == res.done
            np.testing.assert_array_equal(nxt[e], res.next_state.astype(np.float32))
            ep_ret[e] += rewards[e]
            if res.done:
                if not res.info.get("conflict", False):
                    strat = env.strategy()
                    row = [int(strat[d]) for d in env.dims]
                    cand = (env.partition_count, float(ep_ret[e]), step * E + e, row)
                    if best is None or cand[:2] > best[:2] or (cand[:2] == best[:2] and cand[2] < best[2]):
                        best = cand
                ep_ret[e] = 0.0
            states[e] = env.reset() if res.done else res.next_state
    from paper_2007_04069_b200.distributed import select_first_wins

    k = select_first_wins(venv.best_partitions, venv.best_return, venv.best_episode)
    assert best is not None and k is not None
    assert int(venv.best_partitions[k]) == best[0]
    assert float(venv.best_return[k]) == best[1]
    assert int(venv.best_episode[k]) == best[2]
    assert venv.best_status[k, : venv.n].cpu().tolist() == best[3]


def test_vec_trainer_runs_and_learns(cuda):
    g = graphs.generate("bert_base")
    venv = VecPartitionEnv(g, 256)
    cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=200)
    tr = VecDqnTrainer(venv, cfg, capacity=8192, seed=1, learn_steps=2)
    for _ in range(120):
        tr.step()
    torch.cuda.synchronize()
    assert tr.train_steps > 0
    assert int(venv.episodes_done.sum().item()) > 256
    assert torch.isfinite(tr.net.flat).all()
    bp = tr.best_plan()
    assert bp is not None and bp.partitions >= 0 and bp.episode >= 0
    assert set(np.unique(bp.statuses)) <= {0, 1}  # a completed strategy decides every candidate
    g_bp = tr.best_plan_global()  # single process: identity reduction
    assert (g_bp.partitions, g_bp.episode) == (bp.partitions, bp.episode)


def _train(use_graph, steps, E=64, learn_steps=2):
    g = graphs.generate("bert_base")
    venv = VecPartitionEnv(g, E)
    cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=50, target_sync_every=4)
    tr = VecDqnTrainer(venv, cfg, capacity=512, seed=7, learn_steps=learn_steps, use_graph=use_graph)
    for _ in range(steps):
        tr.step()
    torch.cuda.synchronize()
    return tr


def test_cuda_graph_step_matches_eager(cuda):
    """One captured vector step replayed N times == N eager steps, bit for bit
    (counters in the device control block, counter-hash RNG, deterministic kernels)."""
    a = _train(False, 12)
    b = _train(True, 12)
    assert b.graph is not None
    for name in ("flat", "grad"):
        assert torch.equal(getattr(a.net, name), getattr(b.net, name)), name
    assert torch.equal(a.target.flat, b.target.flat)
    assert torch.equal(a.ctl, b.ctl)
    assert a.ctl.tolist() == [12, (12 * 64) % 512, 512, 12 * 2]  # step, slot, size, train
    for k in a.ring:
        assert torch.equal(a.ring[k], b.ring[k]), k
    for k in ("cur_state", "episodes_done", "ep_return", "best_partitions", "best_episode"):
        assert torch.equal(getattr(a.env, k), getattr(b.env, k)), k
    assert (a.train_steps, a.vector_steps, a.size, a.slot) == (b.train_steps, b.vector_steps, b.size, b.slot)


@pytest.mark.parametrize("K", [2, 3, 4])
def test_vec_pipe_env_matches_single_envs(cuda, K):
    """VecPipeTrainEnv (E envs on the device) vs E reference-exact PipeTrainEnv instances:
    states (fp32 of the fp64 state), masks, rewards, done flags and the incumbent."""
    from paper_2007_04069_b200.envs import PipeTrainEnv
    from paper_2007_04069_b200.topology import DeviceTopology
    from paper_2007_04069_b200.vec import VecPipeTrainEnv

    g = graphs.generate("bert_base")
    topo = DeviceTopology(2, 4)
    E = 16
    venv = VecPipeTrainEnv(g, topo, K, E)
    singles = [PipeTrainEnv(g, topo, K) for _ in range(E)]
    states = [s.reset() for s in singles]
    rng = np.random.default_rng(K)
    best = {}
    for step in range(3 * K):
        np.testing.assert_array_equal(venv.cur_state.cpu().numpy(), np.array(states, dtype=np.float32))
        masks = [s.action_mask() for s in singles]
        np.testing.assert_array_equal(venv.mask.cpu().numpy().astype(bool), np.array(masks))
        actions = np.array([rng.choice(np.flatnonzero(m)) for m in masks], dtype=np.int32)
        venv.step(torch.from_numpy(actions).cuda())
        rewards, done = venv.rewards.cpu().numpy(), venv.done.cpu().numpy()
        for e, env in enumerate(singles):
            res = env.step(int(actions[e]))
            assert bool(done[e]) == res.done
            assert rewards[e] == np.float32(res.reward)
            if res.done:
                L = res.info["pipeline_length"]
                if e not in best or L < best[e][0]:
                    best[e] = (L, tuple(res.info["plan"].pivot_ids))
                states[e] = env.reset()
            else:
                np.testing.assert_array_equal(venv.next_state[e].cpu().numpy(), res.next_state.astype(np.float32))
                states[e] = res.next_state
    got = venv.best_plan()
    want = min(best.values(), key=lambda t: t[0])
    assert got[0] == want[0]
    assert got[1] in {v[1] for v in best.values() if v[0] == want[0]}


def test_vec_pipe_trainer_graph_matches_eager(cuda):
    """The PP-train driver inside the CUDA-graph DQN trainer: replay == eager, bit for bit."""
    from paper_2007_04069_b200.topology import DeviceTopology
    from paper_2007_04069_b200.vec import VecPipeTrainEnv

    def run(use_graph):
        env = VecPipeTrainEnv(graphs.generate("bert_base"), DeviceTopology(2, 4), 3, 32)
        cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=50, target_sync_every=4)
        tr = VecDqnTrainer(env, cfg, capacity=256, seed=3, learn_steps=2, use_graph=use_graph)
        for _ in range(8):
            tr.step()
        torch.cuda.synchronize()
        return tr

    a, b = run(False), run(True)
    assert b.graph is not None
    assert torch.equal(a.net.flat, b.net.flat)
    assert torch.equal(a.env.cur_state, b.env.cur_state)
    assert torch.equal(a.env.best_len, b.env.best_len)
    assert int(a.env.episodes_done.sum()) > 0


@pytest.mark.parametrize("K,banded", [(2, False), (4, True), (4, False)])
def test_vec_infer_env_matches_single_envs(cuda, K, banded):
    """VecPipeInferEnv vs E reference-exact PipeInferEnv instances: states, phased masks,
    rewards, done flags and the incumbent."""
    from paper_2007_04069_b200.dataproc import generate_environment
    from paper_2007_04069_b200.envs import PipeInferEnv, infer_search_bands
    from paper_2007_04069_b200.topology import PRESETS
    from paper_2007_04069_b200.vec import VecPipeInferEnv

    arrays = generate_environment("uniform", 1280, K)
    topo = PRESETS["configc"]
    kw = {}
    if banded:
        bb, cc = infer_search_bands(arrays, topo, K, 3)
        kw = {"allowed_boundaries": bb, "allowed_cuts": cc}
    E = 12
    venv = VecPipeInferEnv(arrays, topo, K, E, **kw)
    singles = [PipeInferEnv(arrays, topo, K, **kw) for _ in range(E)]
    states = [s.reset() for s in singles]
    rng = np.random.default_rng(K + banded)
    best = []
    for step in range(5 * (K - 1)):
        np.testing.assert_array_equal(venv.cur_state.cpu().numpy(), np.array(states, dtype=np.float32))
        masks = [s.action_mask() for s in singles]
        np.testing.assert_array_equal(venv.mask.cpu().numpy().astype(bool), np.array(masks))
        actions = np.array([rng.choice(np.flatnonzero(m)) for m in masks], dtype=np.int32)
        venv.step(torch.from_numpy(actions).cuda())
        rewards, done = venv.rewards.cpu().numpy(), venv.done.cpu().numpy()
        for e, env in enumerate(singles):
            res = env.step(int(actions[e]))
            assert bool(done[e]) == res.done
            assert rewards[e] == np.float32(res.reward)
            if res.done:
                best.append((res.info["pipeline_length"], env.boundaries, env.device_cuts))
                states[e] = env.reset()
            else:
                states[e] = res.next_state
    got = venv.best_plan()
    want = min(b[0] for b in best)
    assert got[0] == want
    assert (got[1], got[2]) in {(b[1], b[2]) for b in best if b[0] == want}


@pytest.mark.parametrize("n", [1, 37, 4096, 16384, 24576, 30000])
def test_throughput_per_sampler(cuda, monkeypatch, n):
    """ap_per_sample_fast: the padded-CDF kernel (rings up to 24,576) and the warp-row kernel
    (AP_PER_ROWSCAN=1; larger rings use it with a global CDF) pick the same indices (the
    searchsorted(side='right') of u * total in the fp64 CDF, checked against numpy), and IS
    weights (n p)^-beta / max within fp32 rounding."""
    import numpy as np

    from paper_2007_04069_b200 import _native

    rng = np.random.default_rng(n)
    prio = rng.random(n) ** 0.6 + 1e-6
    u = rng.random(256).astype(np.float32)
    d_p = torch.from_numpy(prio).cuda()
    d_u = torch.from_numpy(u).cuda()
    cdf = torch.empty(n, dtype=torch.float64, device="cuda")
    lib = _native.require_device()
    res = []
    for rowscan in (False, True):
        if rowscan:
            monkeypatch.setenv("AP_PER_ROWSCAN", "1")
        idx = torch.empty(256, dtype=torch.int32, device="cuda")
        w = torch.empty(256, dtype=torch.float32, device="cuda")
        mx = torch.empty(1, dtype=torch.float64, device="cuda")
        _native.check(lib.ap_per_sample_fast(_native.ptr(d_p), n, 0.6, 0.4, _native.ptr(d_u), 256, _native.ptr(cdf),
                                             _native.ptr(idx), _native.ptr(w), _native.ptr(mx),
                                             _native.stream_handle()))
        res.append((idx.cpu().numpy(), w.cpu().numpy(), float(mx.item())))
    c = np.cumsum(prio)
    expect = np.minimum(np.searchsorted(c, u.astype(np.float64) * c[-1], side="right"), n - 1)
    for idx, w, mx in res:
        assert mx == prio.max()
        assert (idx == expect).mean() >= 0.99  # fp64 CDF rounding differs from numpy's only at exact ties
        p = prio[idx] / c[-1]
        ref = (n * p) ** -0.4
        np.testing.assert_allclose(w, ref / ref.max(), rtol=2e-6)
    np.testing.assert_array_equal(res[0][0], res[1][0])


@pytest.mark.parametrize("use_graph", [False, True])
def test_pipelined_learner_matches_serial(cuda, monkeypatch, use_graph):
    """Learner pipelining (priority scatter + next PER sample / gather on a branch beside the
    backward, Adam reading the advanced step counter) == the serial learn order, bit for bit."""
    monkeypatch.setenv("AP_DQN_NO_PIPELINE", "1")
    a = _train(use_graph, 10, learn_steps=3)
    monkeypatch.delenv("AP_DQN_NO_PIPELINE")
    b = _train(use_graph, 10, learn_steps=3)
    assert a.side2 is None and b.side2 is not None
    for name in ("flat", "grad"):
        assert torch.equal(getattr(a.net, name), getattr(b.net, name)), name
    assert torch.equal(a.opt.m, b.opt.m) and torch.equal(a.opt.v, b.opt.v)
    assert torch.equal(a.ctl, b.ctl)
    for k in a.ring:
        assert torch.equal(a.ring[k], b.ring[k]), k
    assert torch.equal(a.idx, b.idx) and torch.equal(a.weights, b.weights)


@pytest.mark.parametrize("use_graph", [False, True])
def test_fused_first_layer_adam_matches_unfused(cuda, monkeypatch, use_graph):
    """Adam for w0 / b0 fused into their weight-gradient GEMM epilogue (+ the transposed w0
    copy; opt-in AP_FUSED_ADAM=1) == the separate Adam kernel, bit for bit."""
    a = _train(use_graph, 8, learn_steps=3)
    monkeypatch.setenv("AP_FUSED_ADAM", "1")
    b = _train(use_graph, 8, learn_steps=3)
    for name in ("flat", "grad"):
        assert torch.equal(getattr(a.net, name), getattr(b.net, name)), name
    assert torch.equal(a.opt.m, b.opt.m) and torch.equal(a.opt.v, b.opt.v)
    for k in a.net.wt:
        assert torch.equal(a.net.wt[k], b.net.wt[k]), k
    assert torch.equal(a.ctl, b.ctl)


@pytest.mark.parametrize("cols,pad", [(1060, 12), (1414, 2), (37, 3)])
def test_gather_rows_pair_exact_and_in_bounds(cuda, cols, pad):
    """ap_gather_rows_pair: both destinations get exactly src[idx[b], :cols] (16-byte vector path when
    aligned, scalar otherwise); padding columns and rows past B keep their sentinel."""
    from paper_2007_04069_b200 import _native

    gen = torch.Generator(device="cuda").manual_seed(cols)
    R, B = 300, 64
    s0 = torch.randn(R, cols + pad, generator=gen, device="cuda")
    s1 = torch.randn(R, cols + pad, generator=gen, device="cuda")
    idx = torch.randint(0, R, (B,), generator=gen, device="cuda", dtype=torch.int32)
    d = torch.full((2 * B + 3, cols + pad), float("nan"), device="cuda")
    P = _native.ptr
    _native.check(_native.require_device().ap_gather_rows_pair(
        P(s0), s0.stride(0), P(d), d.stride(0), P(s1), s1.stride(0), P(d[B:]), d.stride(0), P(idx), B, cols,
        _native.stream_handle()))
    il = idx.long()
    assert torch.equal(d[:B, :cols], s0[il, :cols])
    assert torch.equal(d[B:2 * B, :cols], s1[il, :cols])
    assert torch.isnan(d[:, cols:]).all() and torch.isnan(d[2 * B:]).all()
