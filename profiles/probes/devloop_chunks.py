"""The device loop one episode per call (and optionally one long call): catches hangs and
per-call costs.  python profiles/probes/devloop_chunks.py GRAPH CALLS [EPISODES_IN_ONE_CALL]"""
import sys, time, json
sys.path.insert(0, ".")
import numpy as np, torch
import bench
from paper_2007_04069_b200 import devloop
from paper_2007_04069_b200.agent import AgentConfig, DqnAgent
from paper_2007_04069_b200.envs import OppEnv
from paper_2007_04069_b200.linkage import extract_linkage_groups
name = sys.argv[1]; eps = int(sys.argv[2])
g, dims = bench.workload_setup(name, "opp")
env = OppEnv(g, groups=extract_linkage_groups(g, dims))
agent = DqnAgent(AgentConfig(lr=0.0005, epsilon_decay_iters=2000), env.state_dim, env.num_actions, 0)
for k in range(eps):
    t0 = time.time()
    devloop.train_partition_device(env, agent, 1)
    print(k, "ok", round(time.time() - t0, 3), devloop.last_stats, flush=True)
if len(sys.argv) > 3:
    t0 = time.time()
    devloop.train_partition_device(env, agent, int(sys.argv[3]))
    print("big ok", round(time.time() - t0, 3), devloop.last_stats, flush=True)
