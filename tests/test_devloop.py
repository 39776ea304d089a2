"""The device search loop (paper_2007_04069_b200/devloop.py, csrc/parity.cu).

CPU: the numpy PCG64 emulation the loop draws through (csrc/pcg64.cuh, run on the host
via ap_pcg64_host_draws) reproduces numpy's Generator.random() / integers(n) streams and
leaves the bit generator in numpy's state, including the buffered 32-bit half that
integers() keeps between calls (agent.py:166-168, 220).

GPU: train_partition_device == search.train_partition on the same agent seed: every
step's state digest / action / reward, the best plan of both stages (with finetune), the
agent's RNG state, train steps, Adam step, ring and network parameters bit for bit; and
== the reference's free-running goldens.  Chunked launches equal one launch.
"""

import json

import numpy as np
import pytest

from goldens import GOLDEN
from paper_2007_04069_b200 import _native, graphs
from paper_2007_04069_b200.devloop import _adam_table, _rng_state, _rng_words


@pytest.mark.parametrize("seed", [0, 7, 123, 2**40 + 3])
def test_pcg64_emulation_matches_numpy(seed):
    lib = _native.load_library()
    rng = np.random.default_rng(seed)
    rng.random()
    rng.integers(3)  # leave a buffered 32-bit half behind
    words = _rng_words(rng.bit_generator.state).view(np.uint64).copy()
    draws = np.random.default_rng(seed + 1)
    ops = np.where(draws.random(4000) < 0.4, 0, draws.integers(1, 40, size=4000)).astype(np.int64)
    ops[::97] = 2 ** 32
    ops[::89] = 1000003
    ops[::83] = 1
    out = np.zeros(len(ops))
    _native.check(lib.ap_pcg64_host_draws(_native.ptr(words), _native.ptr(ops), len(ops), _native.ptr(out)))
    ref = np.array([rng.random() if o == 0 else rng.integers(o) for o in ops], dtype=np.float64)
    np.testing.assert_array_equal(out, ref)
    assert _rng_state(words.view(np.int64)) == rng.bit_generator.state


def test_adam_table_matches_host_bias_corrections():
    """fp32(1 - beta ** t) as the host AdamOptimizer passes it through ctypes (agent.py:241-242)."""
    import ctypes

    tab = _adam_table(1, 5000, 0.9, 0.999).reshape(-1, 2)
    for t in list(range(1, 200)) + [777, 4999, 5000]:
        assert tab[t - 1, 0] == ctypes.c_float(1.0 - 0.9 ** t).value
        assert tab[t - 1, 1] == ctypes.c_float(1.0 - 0.999 ** t).value


# -- GPU -------------------------------------------------------------------------------


def _agent_pair(env_factory, seed, lr, decay):
    from paper_2007_04069_b200.agent import AgentConfig, DqnAgent

    envs = [env_factory(), env_factory()]
    agents = [DqnAgent(AgentConfig(lr=lr, epsilon_decay_iters=decay), envs[0].state_dim, envs[0].num_actions, seed)
              for _ in range(2)]
    return envs, agents


def _env_factory(gname, task):
    from paper_2007_04069_b200.envs import AdpEnv, OppEnv

    g = graphs.generate(gname)
    return (lambda: OppEnv(g)) if task == "opp" else (lambda: AdpEnv(g))


def _assert_agents_equal(a, b):
    import torch

    assert a.rng.bit_generator.state == b.rng.bit_generator.state
    assert a.train_steps == b.train_steps and a.optimizer.t == b.optimizer.t
    assert len(a.buffer) == len(b.buffer) and a.buffer._next == b.buffer._next
    assert torch.equal(a.net.flat, b.net.flat) and torch.equal(a.target.flat, b.target.flat)
    assert torch.equal(a.optimizer.m, b.optimizer.m) and torch.equal(a.optimizer.v, b.optimizer.v)
    n = len(a.buffer)
    for k in ("states", "next_states", "actions", "rewards", "done", "next_mask", "priorities"):
        assert torch.equal(a.buffer.store[k][:n], b.buffer.store[k][:n]), k


def _plan(o):
    return None if o is None else (o.partitions, o.reward, o.episode, tuple(sorted((d.flat_index, int(s))
                                                                                     for d, s in o.strategy.items())))


@pytest.mark.gpu
@pytest.mark.parametrize("gname,task,seed,episodes,finetune", [("mlp2", "opp", 0, 150, 20), ("vgg19", "opp", 3, 40, 10),
                                                               ("vgg19", "adp", 0, 60, 0),
                                                               ("bert_base", "opp", 7, 10, 3)])
def test_device_loop_equals_host_loop(cuda, gname, task, seed, episodes, finetune):
    from paper_2007_04069_b200.devloop import train_partition_device
    from paper_2007_04069_b200.search import ListTrace, train_partition

    (e_h, e_d), (a_h, a_d) = _agent_pair(_env_factory(gname, task), seed, 0.0005, 500 if task == "adp" else 2000)
    tr_h, tr_d = ListTrace(), ListTrace()
    b_h = train_partition(e_h, a_h, episodes, None, tr_h)
    b_d = train_partition_device(e_d, a_d, episodes, None, tr_d, episodes_per_launch=7)
    assert tr_d.records == tr_h.records
    assert _plan(b_d) == _plan(b_h)
    _assert_agents_equal(a_h, a_d)
    if finetune and b_h is not None:
        f_h = train_partition(e_h, a_h, finetune, None, tr_h, finetune_base=b_h.strategy, episode_offset=episodes)
        f_d = train_partition_device(e_d, a_d, finetune, None, tr_d, finetune_base=b_d.strategy,
                                     episode_offset=episodes)
        assert tr_d.records == tr_h.records
        assert _plan(f_d) == _plan(f_h)
        _assert_agents_equal(a_h, a_d)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["opp_mlp2", "opp_vgg19", "adp_vgg19", "opp_bert_base", "adp_bert_base"])
def test_device_loop_matches_reference_goldens(cuda, name):
    """Free-running on the device == the reference's own run (tests/golden/search_*.json)."""
    from paper_2007_04069_b200.agent import AgentConfig, DqnAgent
    from paper_2007_04069_b200.devloop import train_partition_device
    from paper_2007_04069_b200.envs import AdpEnv, OppEnv
    from paper_2007_04069_b200.search import ListTrace, strategy_payload

    rec = json.loads((GOLDEN / f"search_{name}.json").read_text())
    g = graphs.generate(rec["graph_generator"])
    env = OppEnv(g) if rec["task"] == "opp" else AdpEnv(g)
    agent = DqnAgent(AgentConfig(lr=rec["lr"], epsilon_decay_iters=rec["epsilon_decay"]), env.state_dim,
                     env.num_actions, rec["seed"])
    trace = ListTrace()
    best = s1 = train_partition_device(env, agent, rec["episodes"], None, trace)
    s2 = None
    if best is not None and rec["finetune_episodes"]:
        s2 = train_partition_device(env, agent, rec["finetune_episodes"], None, trace, finetune_base=best.strategy,
                                    episode_offset=rec["episodes"])
        if s2 is not None and (s2.partitions, s2.reward) > (best.partitions, best.reward):
            best = s2

    def plan(o):
        return None if o is None else {"strategy": strategy_payload(g, o.strategy), "partitions": o.partitions,
                                       "reward": o.reward, "episode": o.episode}

    steps = lambda recs: [(r["episode"], s["state_digest"], s["action"], s["reward"], r["outcome"])  # noqa: E731
                          for r in recs for s in r["steps"]]
    assert steps(trace.records) == steps(rec["trace"])
    assert (plan(s1), plan(s2), plan(best)) == (rec["best_stage1"], rec["best_stage2"], rec["best"])
    assert agent.train_steps == rec["train_steps"]
    assert agent.rng.bit_generator.state == rec["rng_state"]


@pytest.mark.gpu
def test_device_loop_curve_and_chunking(cuda):
    """Curve rows (mean loss, return, epsilon) equal the host loop's; one launch == many."""
    from paper_2007_04069_b200.devloop import train_partition_device
    from paper_2007_04069_b200.search import train_partition

    class Curve:
        def __init__(self):
            self.rows = []

        def write(self, ep, loss, total, eps):
            self.rows.append((ep, loss, total, eps))

    (e_h, e_d), (a_h, a_d) = _agent_pair(_env_factory("vgg19", "opp"), 5, 0.0005, 2000)
    c_h, c_d = Curve(), Curve()
    train_partition(e_h, a_h, 30, c_h, None)
    train_partition_device(e_d, a_d, 30, c_d, None)
    assert c_d.rows == c_h.rows
    e3, a3 = _agent_pair(_env_factory("vgg19", "opp"), 5, 0.0005, 2000)
    b1 = train_partition_device(e3[0], a3[0], 30, None, None, episodes_per_launch=1)
    b2 = train_partition_device(e3[1], a3[1], 30, None, None)
    assert _plan(b1) == _plan(b2)
    _assert_agents_equal(a3[0], a3[1])


@pytest.mark.gpu
@pytest.mark.parametrize("per_iter", [1, 3])
def test_device_loop_steps_per_iteration(cuda, monkeypatch, per_iter):
    """A WHILE iteration of 1 or 3 steps (the act closes the steps past the budget, the later
    kernels of the body skip) gives the default body's results."""
    from paper_2007_04069_b200 import devloop

    (e1, e2), (a1, a2) = _agent_pair(_env_factory("mlp2", "opp"), 3, 0.0005, 300)
    b_default = devloop.train_partition_device(e1, a1, 60, None, None)
    monkeypatch.setattr(devloop, "_STEPS_PER_ITER", per_iter)
    b_other = devloop.train_partition_device(e2, a2, 60, None, None)
    assert _plan(b_default) == _plan(b_other)
    _assert_agents_equal(a1, a2)


def _sample_desc(t, cap, A, eps_decay):
    d = _native.ParityLoopDesc()
    d.ctl, d.rng, d.r_prio, d.cap, d.num_actions = t["ctl"].data_ptr(), t["rng"].data_ptr(), t["prio"].data_ptr(), cap, A
    d.eps_start, d.eps_final, d.eps_decay = 1.0, 0.05, eps_decay
    d.r_scaled, d.pstat, d.per_alpha = t["scaled"].data_ptr(), t["pstat"].data_ptr(), 0.6
    return d


@pytest.mark.gpu
@pytest.mark.parametrize("size,train", [(64, 0), (700, 150), (1999, 1999), (2000, 400), (2000, 5000)])
def test_early_per_sample_equals_sampling_after_the_push(cuda, size, train):
    """ap_parity_sample in early mode (launched beside the step's act / env.step: the ring and the
    random stream as the step starts, the act's draws replayed, the pending push counted) gives
    the indices, weights and final stream of numpy sampling after the act's draws and the push
    (agent.py:155-170, 197-223), and acknowledges its read; late mode (after the push) agrees."""
    import ctypes

    import torch

    cap, A, B, alpha, beta = 2000, 2, 64, 0.6, 0.4
    rng = np.random.default_rng(size + train)
    prio = np.zeros(cap)
    prio[:size] = rng.random(size) * 3 + 1e-6
    slot = size % cap
    gen = 41
    lib = _native.require_device()
    np_rng = np.random.default_rng(train + 1)
    np_rng.random(3)
    words = _rng_words(np_rng.bit_generator.state)
    W = _native.PL

    def run(early):
        ctl = np.zeros(W["WORDS"], dtype=np.int64)
        ctl[W["SLOT"]], ctl[W["TRAIN"]], ctl[W["GEN"]] = slot, train, gen
        ctl[W["BUDGET"]], ctl[W["MAX_STEPS"]], ctl[W["ACTIVE"]] = 1, 10, 1
        p = prio.copy()
        if early:
            ctl[W["SIZE"]] = size
            r = words.copy()
        else:  # the act's draws and the push already happened
            ctl[W["SIZE"]] = min(size + 1, cap)
            p[slot] = prio[:size].max() if size else 1.0
            g = np.random.default_rng()
            g.bit_generator.state = _rng_state(words.copy())
            eps = 1.0 + (0.05 - 1.0) * min(1.0, max(0.0, train / 2000))
            if g.random() < eps:
                g.integers(A)
            r = _rng_words(g.bit_generator.state)
        t = {"ctl": torch.from_numpy(ctl).cuda(), "rng": torch.from_numpy(r).cuda(),
             "prio": torch.from_numpy(p).cuda(), "scaled": torch.zeros(cap, dtype=torch.float64, device="cuda"),
             "pstat": torch.zeros(2, dtype=torch.float64, device="cuda")}
        _native.check(lib.ap_per_scaled(_native.ptr(t["prio"]), size, alpha, _native.ptr(t["scaled"]),
                                        _native.ptr(t["pstat"]), None))
        d = _sample_desc(t, cap, A, 2000)
        d.early_sample = int(early)
        scratch = torch.zeros(2 * cap + 1024, dtype=torch.float64, device="cuda")
        idx = torch.zeros(B, dtype=torch.int32, device="cuda")
        w = torch.zeros(B, dtype=torch.float32, device="cuda")
        u = torch.zeros(B, dtype=torch.float64, device="cuda")
        rng_next = torch.zeros(6, dtype=torch.int64, device="cuda")
        _native.check(lib.ap_parity_sample(ctypes.byref(d), B, alpha, beta, _native.ptr(scratch), _native.ptr(idx),
                                           _native.ptr(w), _native.ptr(u), _native.ptr(rng_next), int(early), None))
        torch.cuda.synchronize()
        final = rng_next if early else t["rng"]
        return (idx.cpu().numpy(), w.cpu().numpy(), u.cpu().numpy(), final.cpu().numpy(),
                t["ctl"].cpu().numpy(), p)

    n = min(size + 1, cap)
    early, late = run(True), run(False)
    p = late[5]
    # numpy: the act's draws, the push, then rng.choice's uniforms and searchsorted
    g = np.random.default_rng()
    g.bit_generator.state = _rng_state(words.copy())
    eps = 1.0 + (0.05 - 1.0) * min(1.0, max(0.0, train / 2000))
    if g.random() < eps:
        g.integers(A)
    uu = g.random(B)
    scaled = p[:n] ** alpha
    probs = scaled / scaled.sum()
    cdf = probs.cumsum()
    cdf /= cdf[-1]
    ref_idx = cdf.searchsorted(uu, side="right")
    ref_w = (n * probs[ref_idx]) ** (-beta)
    ref_w /= ref_w.max()
    for idx, w, u, final, ctl, _ in (early, late):
        np.testing.assert_array_equal(u, uu)
        np.testing.assert_array_equal(idx, ref_idx)
        assert np.max(np.abs(w - ref_w) / ref_w) < 1e-6
        assert _rng_state(final.view(np.int64)) == g.bit_generator.state
    np.testing.assert_array_equal(early[0], late[0])
    np.testing.assert_array_equal(early[1], late[1])
    assert early[4][W["ACK"]] == gen + 1 and late[4][W["ACK"]] == 0


@pytest.mark.gpu
def test_act_forward_any_grid_on_one_barrier(cuda):
    """The few-row forward's grid barrier allows a different grid from launch to launch on the
    same buffer: the full-grid host forward, then the loop's act (one SM left to the sampler),
    then the host forward again give the same Q."""
    import ctypes

    import torch

    from paper_2007_04069_b200.agent import QNetwork

    net = QNetwork(9, 2, (32, 32), np.random.default_rng(0))
    x = torch.randn((1, 9), dtype=torch.float32, device="cuda")
    q0 = net.forward_fused(x).clone()  # full grid on the network's forward barrier
    ws, bar = net._fused_scratch(256, True)
    Lh, dims, w_off, b_off = net.fused_layout()[:4]
    t = {"ctl": torch.zeros(_native.PL["WORDS"], dtype=torch.int64, device="cuda"),
         "rng": torch.zeros(6, dtype=torch.int64, device="cuda")}
    t["ctl"][_native.PL["BUDGET"]] = 1
    t["ctl"][_native.PL["MAX_STEPS"]] = 1
    t["ctl"][_native.PL["TRAIN"]] = 10 ** 6  # past the decay: epsilon 0.05, a greedy draw below
    t["ctl"][_native.PL["ACK"]] = 1  # as if the step's sampler had read the stream (GEN 0)
    g = np.random.default_rng(5)
    t["rng"].copy_(torch.from_numpy(_rng_words(g.bit_generator.state)))
    seeds = torch.full((16,), -1, dtype=torch.int8, device="cuda")
    seeds_try = seeds.clone()
    log = torch.zeros(4, dtype=torch.int32, device="cuda")
    d = _native.ParityLoopDesc()
    d.ctl, d.rng, d.state, d.num_actions, d.ld = t["ctl"].data_ptr(), t["rng"].data_ptr(), x.data_ptr(), 2, 16
    d.seeds, d.seeds_try, d.decided = seeds.data_ptr(), seeds_try.data_ptr(), seeds.data_ptr()
    d.log_action, d.log_pos = log.data_ptr(), log.data_ptr()
    d.eps_start, d.eps_final, d.eps_decay = 1.0, 0.05, 100
    d.early_sample = 1  # the loop's act: one SM left free, a smaller grid
    q = torch.zeros((1, 2), dtype=torch.float32, device="cuda")
    a = torch.zeros(1, dtype=torch.int32, device="cuda")
    lib = _native.require_device()
    _native.check(lib.ap_parity_act_fused(ctypes.byref(d), Lh, dims, w_off, b_off, _native.ptr(net.flat),
                                          _native.ptr(q), _native.ptr(ws), _native.ptr(bar), _native.ptr(a), None))
    q2 = net.forward_fused(x)
    torch.cuda.synchronize()
    if g.random() >= 0.05:  # the act exploited: it computed Q on the smaller grid
        assert torch.equal(q, q0)
    assert torch.equal(q2, q0)
