"""One K1 configuration launched a few times (for ncu captures of a single kernel).

    python profiles/probes/k1_one.py GRAPH TASK MODE BATCH [LAUNCHES]

GRAPH in graphs.GENERATORS, TASK opp | adp, MODE full | env | packed.  The plan batch is the
bench's decision-order prefixes on the reference's order (bench.golden_order).
"""

import sys
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2007_04069_b200.sharding import PropagationEngine  # noqa: E402
from paper_2007_04069_b200.workloads import prefix_seed_batch  # noqa: E402


def main():
    name, task, mode, B = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
    launches = int(sys.argv[5]) if len(sys.argv) > 5 else 5
    g, dims = bench.workload_setup(name, task)
    order, _ = bench.golden_order(name, task, len(dims))
    eng = PropagationEngine(g, dims)
    seeds = prefix_seed_batch(order, 0, B, device="cuda", chunk=1 << 18)
    ms, conflict, _ = bench.k1_measure(eng, seeds, mode, launches=launches, warmup=2)
    print(f"{name} {task} {mode} B={B}: {ms:.4f} ms/launch, {B / ms / 1e6:.3f} G plans/s, conflict {conflict:.3f}")


if __name__ == "__main__":
    main()
