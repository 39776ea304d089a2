"""Golden fixtures for the DQN agent and the search loops, from the REFERENCE.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_goldens_agent.py

agent_qnet.npz   QNetwork(seed) forward on fixed states and backward for a
                 fixed dQ (agent.py:58-136).
agent_train.npz  DqnAgent fed a fixed synthetic transition stream: loss of
                 every learn step and Q on probe states at the end.
search_*.json    train_partition / train_pipe runs (cli.py:193-329): every
                 step's state digest, action and reward plus the best plan.
Generated with OPENBLAS_NUM_THREADS=1 (recorded): the reference itself is not
thread-count invariant on long PP runs (SURVEY §7 hard part 2).
"""

from __future__ import annotations

import json
import os
import platform
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))

from autoplan import zoo  # noqa: E402
from autoplan.agent import AgentConfig, DqnAgent, QNetwork, Transition  # noqa: E402
from autoplan.cli import _digest, _strategy_payload, train_partition, train_pipe  # noqa: E402
from autoplan.dataproc import build_environment_arrays  # noqa: E402
from autoplan.envs import AdpEnv, OppEnv, PipeInferEnv, PipeTrainEnv, infer_search_bands  # noqa: E402
from autoplan.topology import PRESETS  # noqa: E402

OUT = Path(__file__).resolve().parent
META = {"python": platform.python_version(), "numpy": np.__version__,
        "OPENBLAS_NUM_THREADS": os.environ.get("OPENBLAS_NUM_THREADS")}


class Trace:
    def __init__(self):
        self.records = []

    def write(self, episode, steps, outcome):
        self.records.append({"episode": episode, "steps": steps, "outcome": outcome})


def dump_qnet():
    out = {}
    for tag, (s, a, seed) in {"small": (40, 5, 3), "opp_bert48": (1060, 2, 7)}.items():
        net = QNetwork(s, a, (256, 256), np.random.default_rng(seed))
        rng = np.random.default_rng(seed + 1)
        x = rng.uniform(-1, 1, size=(16, s))
        q, cache = net.forward_cached(x)
        dq = rng.normal(size=q.shape) / 16
        g = net.backward(cache, dq)
        out[f"{tag}_meta"] = np.array([s, a, seed])
        out[f"{tag}_x"] = x
        out[f"{tag}_q"] = q
        out[f"{tag}_dq"] = dq
        for k, v in g.items():
            out[f"{tag}_grad_{k}"] = v
    np.savez_compressed(OUT / "agent_qnet.npz", **out)
    print("agent_qnet")


def synthetic_stream(rng, n, s, a):
    for _ in range(n):
        mask = rng.random(a) < 0.8
        mask[rng.integers(a)] = True
        yield Transition(rng.uniform(-1, 1, s), int(rng.integers(a)), float(rng.normal()), rng.uniform(-1, 1, s),
                         bool(rng.random() < 0.1), mask)


def dump_train():
    cfg = AgentConfig(batch_size=16, buffer_capacity=50, target_sync_every=10, lr=0.001)
    s, a = 12, 3
    agent = DqnAgent(cfg, s, a, seed=5)
    rng = np.random.default_rng(99)
    losses = []
    stream = list(synthetic_stream(rng, 90, s, a))
    for t in stream:
        agent.observe(t)
        loss = agent.learn()
        losses.append(np.nan if loss is None else loss)
    probe = np.random.default_rng(123).uniform(-1, 1, size=(8, s))
    np.savez_compressed(
        OUT / "agent_train.npz",
        cfg=np.frombuffer(json.dumps({"batch_size": 16, "buffer_capacity": 50, "target_sync_every": 10,
                                      "lr": 0.001, "state_dim": s, "num_actions": a, "seed": 5}).encode(), np.uint8),
        states=np.array([t.state for t in stream]), actions=np.array([t.action for t in stream]),
        rewards=np.array([t.reward for t in stream]), next_states=np.array([t.next_state for t in stream]),
        done=np.array([t.done for t in stream]), masks=np.array([t.next_mask for t in stream]),
        losses=np.array(losses), probe=probe, probe_q=agent.net.forward(probe),
        priorities=agent.buffer._priorities[: len(agent.buffer)].copy(),
        rng_state=np.frombuffer(json.dumps(agent.rng.bit_generator.state).encode(), np.uint8),
    )
    print("agent_train")


def run_partition(name, graph, task, seed, episodes, lr, decay):
    env = OppEnv(graph) if task == "opp" else AdpEnv(graph)
    cfg = AgentConfig(lr=lr, epsilon_decay_iters=decay)
    agent = DqnAgent(cfg, env.state_dim, env.num_actions, seed)
    trace = Trace()
    best = train_partition(env, agent, episodes, None, trace)
    rec = {"meta": META, "task": task, "seed": seed, "episodes": episodes, "lr": lr, "epsilon_decay": decay,
           "graph": graph.to_dict(), "trace": trace.records,
           "best": None if best is None else {"strategy": _strategy_payload(graph, best.strategy),
                                              "partitions": best.partitions, "reward": best.reward,
                                              "episode": best.episode},
           "final_probe_q": agent.net.forward(np.zeros((1, env.state_dim))).tolist()}
    (OUT / f"search_{name}.json").write_text(json.dumps(rec))
    print(name, rec["best"])


def run_pipe(name, env, seed, episodes, lr, decay, extra):
    cfg = AgentConfig(lr=lr, epsilon_decay_iters=decay)
    agent = DqnAgent(cfg, env.state_dim, env.num_actions, seed)
    trace = Trace()
    best = train_pipe([env], agent, episodes, None, trace)[0]
    rec = {"meta": META, "seed": seed, "episodes": episodes, "lr": lr, "epsilon_decay": decay, "trace": trace.records,
           "best": None if best is None else {"pivots": list(best.plan.pivot_ids),
                                              "device_cuts": list(best.plan.device_cuts),
                                              "length": best.pipeline_length, "episode": best.episode},
           **extra}
    (OUT / f"search_{name}.json").write_text(json.dumps(rec))
    print(name, rec["best"])


def main():
    dump_qnet()
    dump_train()
    run_partition("opp_attention_block", zoo.attention_block(), "opp", 7, 120, 0.0005, 2000)
    run_partition("opp_t5_block", zoo.t5_block(), "opp", 7, 80, 0.0005, 2000)
    run_partition("adp_vgg_classifier", zoo.vgg_classifier(), "adp", 0, 150, 0.0005, 500)
    chain = zoo.uniform_chain()
    run_pipe("pp_train_chain", PipeTrainEnv(chain, PRESETS["configa"], 2, radius=3, micro_batches=4), 0, 60, 0.001,
             10000, {"graph": chain.to_dict(), "topology": "configa", "stages": 2, "radius": 3, "micro_batches": 4})
    arrays = build_environment_arrays(zoo.bert48_profile())
    topo = PRESETS["configc"]
    bb, cc = infer_search_bands(arrays, topo, 4, 3)
    env = PipeInferEnv(arrays, topo, 4, micro_batches=1, allowed_boundaries=bb, allowed_cuts=cc)
    run_pipe("pp_infer_bert48", env, 0, 40, 0.001, 10000,
             {"arrays": np.concatenate([arrays.c, arrays.a, arrays.w]).tolist(), "topology": "configc", "stages": 4,
              "radius": 3, "micro_batches": 1})


if __name__ == "__main__":
    main()
