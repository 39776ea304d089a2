"""Per-phase timeline of the fused learn kernel (csrc/fused_mlp.cu) on the bench's BERT-48 agent.

    python profiles/probes/learn_phases.py [REPS]

The kernel's trace mode stamps %globaltimer on CTA 0 after every grid barrier (tr[k]) and
each CTA's arrival at the end of phase k (tr[64 + k * grid + cta]).  Prints, per phase, the
median over REPS warm launches of: CTA 0's phase time, the earliest / latest CTA arrival
(work done) and the barrier release after the latest arrival.
"""

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2007_04069_b200 import devloop  # noqa: E402
from paper_2007_04069_b200.agent import AgentConfig, DqnAgent  # noqa: E402
from paper_2007_04069_b200.envs import OppEnv  # noqa: E402
from paper_2007_04069_b200.linkage import extract_linkage_groups  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    g, dims = bench.workload_setup("bert48", "opp")
    env = OppEnv(g, groups=extract_linkage_groups(g, dims))
    agent = DqnAgent(AgentConfig(lr=0.0005, epsilon_decay_iters=2000), env.state_dim, env.num_actions, 0)
    devloop.train_partition_device(env, agent, 2)
    fused = agent._fused
    B = agent.config.batch_size
    gen = torch.Generator().manual_seed(0)
    idx = torch.randint(0, len(agent.buffer), (B,), generator=gen, dtype=torch.int32).cuda()
    w = torch.ones(B, dtype=torch.float32, device="cuda")
    grid = torch.cuda.get_device_properties(0).multi_processor_count
    tr = torch.zeros(max(64 + 16 * grid, 4096 + 8 * 64), dtype=torch.int64, device="cuda")
    fused.desc.trace = tr.data_ptr()
    rows = []
    for r in range(reps + 3):
        tr.zero_()
        fused.run(idx, w, correct1=0.5, correct2=0.5)
        torch.cuda.synchronize()
        t = tr.cpu().numpy()
        k = int(np.count_nonzero(t[:64]))
        marks = t[:k].astype(np.float64)
        arr = t[64:64 + 16 * grid].reshape(16, grid).astype(np.float64)
        ph = []
        for p in range(k - 1):
            a = arr[p + 1]  # arrivals are stamped with the index of the phase's end mark
            a = a[a > 0]
            ph.append((marks[p + 1] - marks[p], a.min() - marks[p] if a.size else 0, a.max() - marks[p] if a.size else 0))
        rows.append((marks[-1] - marks[0], ph))
    rows = rows[3:]
    print(f"total us (CTA 0, first mark -> last): {np.median([r[0] for r in rows]) / 1e3:.2f}")
    for p in range(len(rows[0][1])):
        v = np.median([[x for x in r[1][p]] for r in rows], axis=0) / 1e3
        print(f"phase {p}: {v[0]:7.2f} us   first CTA done {v[1]:6.2f}   last CTA done {v[2]:6.2f}   "
              f"barrier {v[0] - v[2]:5.2f}")
    # AP_FUSED_TILE_TRACE builds (build_trace_lib.sh): CTA 0's tiles of the last launch, stage
    # stamps relative to the tile start (loads issued, landed, k-loop done, k-groups added, stored)
    t = tr.cpu().numpy()
    tiles = t[4096:4096 + 8 * 64].reshape(64, 8)
    marks0 = t[0]
    for i, row in enumerate(tiles):
        if row[0] == 0:
            break
        print(f"tile {i}: start +{(row[0] - marks0) / 1e3:7.2f} us, stages " +
              " ".join(f"{(row[k] - row[0]) / 1e3:6.2f}" for k in range(1, 6)))
    fused.desc.trace = None


if __name__ == "__main__":
    main()
