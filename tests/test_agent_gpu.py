"""DQN agent and search loops on the GPU vs the reference (tests/golden/agent_*, search_*).

Parity contract (SURVEY §7 hard part 2):
* Q-values / gradients: within fp32 tolerance of the fp64 reference on
  identical weights and inputs (rtol stated per test);
* PER sampling: identical indices for identical priorities and uniforms;
* RNG draw order: after the same stream of observe/learn calls the agent's
  numpy Generator is in exactly the reference's state;
* OPP / ADP free-running search: identical per-step state digests, actions,
  rewards and best plan;
* PP train / infer: replaying the reference's action trace gives
  bit-identical digests and rewards.
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2007_04069_b200.agent import AgentConfig, DqnAgent, QNetwork, Transition
from paper_2007_04069_b200.envs import AdpEnv, OppEnv, PipeInferEnv, PipeTrainEnv, infer_search_bands
from paper_2007_04069_b200.ir import graph_from_dict
from paper_2007_04069_b200.search import ListTrace, state_digest, strategy_payload, train_partition
from paper_2007_04069_b200.topology import PRESETS

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"

Q_RTOL = 1e-5      # Q-values relative to max |Q| (3xTF32 GEMMs, fp32 elementwise)
GRAD_RTOL = 1e-4   # gradients relative to max |grad|


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(1e-30, np.abs(np.asarray(b)).max()))


@pytest.mark.parametrize("tag", ["small", "opp_bert48"])
def test_qnetwork_forward_backward_within_fp32_tolerance(cuda, tag):
    z = np.load(GOLDEN / "agent_qnet.npz")
    s, a, seed = z[f"{tag}_meta"]
    net = QNetwork(int(s), int(a), (256, 256), np.random.default_rng(int(seed)))
    q, cache = net.forward_cached(z[f"{tag}_x"])
    assert rel(q, z[f"{tag}_q"]) < Q_RTOL
    grads = net.backward(cache, z[f"{tag}_dq"])
    for k, v in grads.items():
        assert rel(v, z[f"{tag}_grad_{k}"]) < GRAD_RTOL, k


def test_per_sampler_exact(cuda):
    from paper_2007_04069_b200.agent import PrioritizedReplayBuffer

    rng = np.random.default_rng(4)
    for n in (64, 100, 129, 1000, 2000):
        buf = PrioritizedReplayBuffer(2000, 3, 2)
        buf._alloc(3, 2)
        pr = rng.random(n) * 3 + 1e-6
        buf._store["priorities"][:n] = torch.from_numpy(pr)
        buf._size = n
        u = rng.random(64)
        idx, w = buf.sample_device(64, 0.2, 0.6, u)
        scaled = pr ** 0.2
        probs = scaled / scaled.sum()
        cdf = probs.cumsum()
        cdf /= cdf[-1]
        ref_idx = cdf.searchsorted(u, side="right")
        np.testing.assert_array_equal(idx.cpu().numpy(), ref_idx)
        ref_w = (n * probs[ref_idx]) ** (-0.6)
        ref_w /= ref_w.max()
        assert rel(w.cpu().numpy(), ref_w) < 1e-6


def test_agent_training_stream(cuda):
    z = np.load(GOLDEN / "agent_train.npz")
    meta = json.loads(bytes(z["cfg"]).decode())
    cfg = AgentConfig(batch_size=meta["batch_size"], buffer_capacity=meta["buffer_capacity"],
                      target_sync_every=meta["target_sync_every"], lr=meta["lr"])
    agent = DqnAgent(cfg, meta["state_dim"], meta["num_actions"], seed=meta["seed"])
    losses = []
    for k in range(len(z["actions"])):
        agent.observe(Transition(z["states"][k], int(z["actions"][k]), float(z["rewards"][k]), z["next_states"][k],
                                 bool(z["done"][k]), z["masks"][k]))
        loss = agent.learn()
        losses.append(np.nan if loss is None else loss)
    losses = np.array(losses)
    ref = z["losses"]
    np.testing.assert_array_equal(np.isnan(losses), np.isnan(ref))
    ok = ~np.isnan(ref)
    assert rel(losses[ok], ref[ok]) < 1e-3
    assert rel(agent.net.forward(z["probe"]), z["probe_q"]) < 1e-3
    assert rel(agent.buffer.priorities, z["priorities"]) < 1e-3
    # identical draw order: the generator ends in the reference's exact state
    assert agent.rng.bit_generator.state == json.loads(bytes(z["rng_state"]).decode())


def trace_of(records):
    return [(s["state_digest"], s["action"], s["reward"]) for r in records for s in r["steps"]]


@pytest.mark.parametrize("name", ["opp_attention_block", "opp_t5_block", "adp_vgg_classifier"])
def test_partition_search_free_running(cuda, name):
    rec = json.loads((GOLDEN / f"search_{name}.json").read_text())
    g = graph_from_dict(rec["graph"])
    env = OppEnv(g) if rec["task"] == "opp" else AdpEnv(g)
    agent = DqnAgent(AgentConfig(lr=rec["lr"], epsilon_decay_iters=rec["epsilon_decay"]), env.state_dim,
                     env.num_actions, rec["seed"])
    trace = ListTrace()
    best = train_partition(env, agent, rec["episodes"], None, trace)
    assert trace_of(trace.records) == trace_of(rec["trace"])
    assert strategy_payload(g, best.strategy) == rec["best"]["strategy"]
    assert (best.partitions, best.reward, best.episode) == (rec["best"]["partitions"], rec["best"]["reward"],
                                                            rec["best"]["episode"])


def replay(env, records):
    got = []
    for r in records:
        state = env.reset()
        for s in r["steps"]:
            res = env.step(s["action"])
            got.append((state_digest(state), s["action"], res.reward))
            state = res.next_state
    return got


def test_pp_train_trace_replay(cuda):
    rec = json.loads((GOLDEN / "search_pp_train_chain.json").read_text())
    g = graph_from_dict(rec["graph"])
    env = PipeTrainEnv(g, PRESETS[rec["topology"]], rec["stages"], radius=rec["radius"],
                       micro_batches=rec["micro_batches"])
    assert replay(env, rec["trace"]) == trace_of(rec["trace"])


def test_pp_infer_trace_replay(cuda):
    rec = json.loads((GOLDEN / "search_pp_infer_bert48.json").read_text())
    arr = np.asarray(rec["arrays"])

    class Arrays:
        c, a, w = arr[:128], arr[128:256], arr[256:]

    topo = PRESETS[rec["topology"]]
    bb, cc = infer_search_bands(Arrays, topo, rec["stages"], rec["radius"])
    env = PipeInferEnv(Arrays, topo, rec["stages"], micro_batches=rec["micro_batches"], allowed_boundaries=bb,
                       allowed_cuts=cc)
    assert replay(env, rec["trace"]) == trace_of(rec["trace"])


@pytest.mark.parametrize("shape", [(37, 5, (45, 33)), (1414, 9, (256, 256))])
def test_adam_tiled_transposed_matches_flat(cuda, monkeypatch, shape):
    """ap_dqn_adam_ctl_t: the tiled kernel (32x32 tiles, transposed copies through shared memory,
    flat blocks for the biases) equals the flat per-element kernel bit for bit."""
    from paper_2007_04069_b200 import _native

    s, a, hidden = shape
    lib = _native.require_device()
    P = _native.ptr

    def run():
        net = QNetwork(s, a, hidden, np.random.default_rng(3))
        gen = torch.Generator(device="cuda").manual_seed(5)
        net.grad.copy_(torch.randn(net.grad.shape, generator=gen, device="cuda"))
        m = torch.randn(net.flat.shape, generator=gen, device="cuda") * 0.1
        v = torch.rand(net.flat.shape, generator=gen, device="cuda") * 0.1
        ctl = torch.tensor([0, 0, 0, 7], dtype=torch.int64, device="cuda")
        for t in net.wt.values():
            t.fill_(float("nan"))
        _native.check(lib.ap_dqn_adam_ctl_t(P(net.flat), P(net.grad), P(m), P(v), net.flat.numel(), 1e-3, 0.9, 0.999,
                                            1e-8, P(ctl), *net.adam_segments(), _native.stream_handle()))
        return [net.flat.clone(), m, v] + [t.clone() for t in net.wt.values()]

    tiled = run()
    monkeypatch.setenv("AP_ADAM_FLAT", "1")
    flat = run()
    for x, y in zip(tiled, flat):
        assert torch.equal(x.nan_to_num(7.0), y.nan_to_num(7.0))


@pytest.mark.parametrize("A", [158, 3170])
def test_head_backward_dueling_closed_form(cuda, A):
    """ap_dqn_head_backward_dueling (O(B H) closed form for the TD kernels' dueling gradient)
    matches the O(B H A) product of ap_dqn_head_backward within fp32 rounding (1e-5 of max |dh|)."""
    from paper_2007_04069_b200 import _native

    B, H, A1 = 64, 256, A + 1
    gen = torch.Generator(device="cuda").manual_seed(A)
    g = torch.randn(B, generator=gen, device="cuda")
    g[::9] = 0.0
    a = torch.randint(0, A, (B,), generator=gen, device="cuda")
    q = g / torch.full_like(g, float(A))  # elementwise IEEE quotient, as the TD kernels compute it
    dz = torch.empty(B, A1, device="cuda")
    dz[:, 0] = g
    dz[:, 1:] = (0.0 - q)[:, None]
    dz[torch.arange(B), 1 + a] = g - q
    dz[5, 7] += 1.0  # one row not of the TD shape: the full-product fallback
    wh = torch.randn(H, A1, generator=gen, device="cuda")
    h = torch.randn(B, H, generator=gen, device="cuda")
    lib, P = _native.require_device(), _native.ptr
    outs = []
    for closed in (False, True):
        dh = torch.full((B, H), float("nan"), device="cuda")
        dh_t = torch.full((H, B), float("nan"), device="cuda")
        if closed:
            rs = torch.empty(H, device="cuda")
            _native.check(lib.ap_dqn_head_backward_dueling(P(dz), A1, P(wh), A1, P(h), H, B, H, A1, P(rs), P(dh), H,
                                                           P(dh_t), B, _native.stream_handle()))
        else:
            _native.check(lib.ap_dqn_head_backward(P(dz), A1, P(wh), A1, P(h), H, B, H, A1, P(dh), H, P(dh_t), B,
                                                   _native.stream_handle()))
        assert torch.equal(dh.t(), dh_t)
        outs.append(dh)
    ref = (dz.double() @ wh.double().t()) * (h > 0)
    scale = ref.abs().max().item()
    for o in outs:
        assert (o.double() - ref).abs().max().item() <= 1e-5 * scale
    assert torch.all(outs[1][::9] == 0)
