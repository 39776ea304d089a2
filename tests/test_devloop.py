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
