"""Small runs of every hot kernel family for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck  python profiles/probes/sanitize.py
    compute-sanitizer --tool racecheck python profiles/probes/sanitize.py

K1 fast (int8 slots, packed codes, TMA bulk rows) and generic kernels, the PP-train
table kernel (K2), the PP-infer search (K3), the TMA/tcgen05 GEMMs (v2 split-K, v3 with
cluster split-K and A-tile multicast), one vectorised DQN step (eager and captured) and
the device search loop (conditional-node graph).  Sizes are small: the tools serialise
and instrument every access.
"""

import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from paper_2007_04069_b200 import graphs  # noqa: E402
from paper_2007_04069_b200.ir import decision_dims  # noqa: E402
from paper_2007_04069_b200.sharding import PropagationEngine  # noqa: E402
from paper_2007_04069_b200.workloads import prefix_seed_batch, trigger_seed_batch  # noqa: E402


def k1():
    for name in ("bert48", "t5_large", "vgg19"):
        g = graphs.generate(name)
        dims = decision_dims(g, g.trainable_variables)
        eng = PropagationEngine(g, dims)
        n = len(dims)
        seeds = torch.cat([prefix_seed_batch(np.arange(n), 0, 500, device="cuda"),
                           trigger_seed_batch(n, 0, 100, device="cuda")])
        s = torch.full((seeds.shape[0], (n + 15) // 16 * 16), -1, dtype=torch.int8, device="cuda")[:, :n]
        s.copy_(seeds)
        B = s.shape[0]
        oc = torch.empty(B, dtype=torch.uint8, device="cuda")
        cnt = torch.empty((B, 4), dtype=torch.int32, device="cuda")
        st = torch.empty((B, (n + 15) // 16 * 16), dtype=torch.int8, device="cuda")
        slots = torch.empty((B, eng.slots_stride), dtype=torch.int8, device="cuda")
        pk = torch.empty((B, eng.packed_slots_stride), dtype=torch.uint8, device="cuda")
        eng.launch(s, oc, cnt, slots, st)
        eng.launch(s, oc, cnt, None, st, packed=pk)
        os.environ["AP_K1_BULK"] = "1"
        eng.launch(s, oc, cnt, slots, st)
        os.environ["AP_K1_BULK"] = "0"
        os.environ["AP_PROPAGATE_GENERIC"] = "1"
        eng.launch(s, oc, cnt, slots, st)
        eng.launch(s, oc, cnt, None, st, packed=pk)
        os.environ["AP_PROPAGATE_GENERIC"] = "0"
    torch.cuda.synchronize()
    print("k1 ok", flush=True)


def k2_k3():
    from paper_2007_04069_b200.dataproc import generate_environment
    from paper_2007_04069_b200.envs import PipeInferEnv, PipeTrainEnv, brute_force_plan
    from paper_2007_04069_b200.topology import PRESETS, DeviceTopology

    env = PipeTrainEnv(graphs.generate("bert_base"), DeviceTopology(2, 4), 4, radius=3)
    rng = np.random.default_rng(0)
    for _ in range(2):
        env.reset()
        while not env.done:
            allowed = np.flatnonzero(env.action_mask())
            env.step(int(allowed[rng.integers(len(allowed))]))
    ienv = PipeInferEnv(generate_environment("uniform", 256, 0), PRESETS["configa"], 3)
    brute_force_plan(ienv)
    torch.cuda.synchronize()
    print("k2/k3 ok", flush=True)


def gemms():
    from paper_2007_04069_b200.tc import gemm

    for m, n, k, prec in ((64, 256, 1060, 3), (64, 256, 1060, 1), (4096, 256, 1060, 1), (257, 33, 700, 3)):
        a = torch.randn(m, k, device="cuda")
        b = torch.randn(n, k, device="cuda")
        gemm(a, b, trans_b=True, precision=prec)
    torch.cuda.synchronize()
    print("gemm ok", flush=True)


def dqn():
    from paper_2007_04069_b200.agent import AgentConfig, DqnAgent
    from paper_2007_04069_b200.devloop import train_partition_device
    from paper_2007_04069_b200.envs import OppEnv
    from paper_2007_04069_b200.vec import VecDqnTrainer, VecPartitionEnv

    g = graphs.generate("vgg19")
    env = VecPartitionEnv(g, 256)
    tr = VecDqnTrainer(env, AgentConfig(lr=0.0005), capacity=1024, seed=0, learn_steps=2,
                       use_graph=os.environ.get("SANITIZE_GRAPH", "1") == "1")
    for _ in range(4):
        tr.step()
    oenv = OppEnv(graphs.generate("mlp2"))
    agent = DqnAgent(AgentConfig(lr=0.0005), oenv.state_dim, oenv.num_actions, 0)
    train_partition_device(oenv, agent, 30)
    torch.cuda.synchronize()
    print("dqn ok", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["k1", "k2_k3", "gemms", "dqn"]
    for w in which:
        globals()[w]()
