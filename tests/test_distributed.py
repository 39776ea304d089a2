"""Multi-process host logic of the N>1 path on CPU: world_size-2 gloo groups.

Covers the plan sharding (rank slices concatenate to the global batch), the
max-over-ranks timing reduction, the Q-gradient mean all-reduce and the
first-wins best-plan all-gather (cli.py:237-240) — the same functions
bench.py and vec.py call under NCCL on the GPU box.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2007_04069_b200 import distributed as D
from paper_2007_04069_b200.workloads import prefix_seed_batch

WORLD = 2


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surface worker failures in the parent
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def run_ranks(fn, world=WORLD):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(world)]


# ---- workers (module level: spawn pickles them by name) ---------------------------

ORDER = list(np.random.default_rng(5).permutation(37))


def _shard(rank, world):
    start, count = D.plan_shard(rank, 50)
    mine = prefix_seed_batch(ORDER, start, count)
    got = [torch.empty_like(mine.contiguous()) for _ in range(world)]
    dist.all_gather(got, mine.contiguous())
    return torch.cat(got).numpy()


def _max(rank, world):
    return D.max_over_ranks(1.5 + rank)


def _mean(rank, world):
    g = torch.arange(6, dtype=torch.float32) * (rank + 1)
    return D.allreduce_mean_(g).numpy()


def _best_tie(rank, world):
    # equal (partitions, return): the lower global episode id wins, whatever the rank
    ep = {0: 10, 1: 3}[rank]
    row = torch.full((5,), rank, dtype=torch.int8)
    b = D.reduce_best((7, 2.5, ep), row)
    return (b.partitions, b.reward, b.episode, b.statuses.tolist())


def _best_key(rank, world):
    # a strictly larger key wins over a lower episode id; a rank with nothing completed is ignored
    key = {0: (8, 1.0, 40), 1: (7, 9.0, 1)}[rank]
    row = torch.full((3,), 10 + rank, dtype=torch.int8)
    b = D.reduce_best(key, row)
    return (b.partitions, b.episode, b.statuses.tolist())


def _best_empty(rank, world):
    key = (-1, float("-inf"), -1) if rank == 0 else (2, 0.5, 17)
    b = D.reduce_best(key, torch.zeros(4, dtype=torch.int8))
    return (b.partitions, b.episode)


def _best_none(rank, world):
    return D.reduce_best((-1, float("-inf"), -1), torch.zeros(4, dtype=torch.int8))


# ---- tests -------------------------------------------------------------------------


def test_plan_shards_concatenate_to_global_batch():
    outs = run_ranks(_shard)
    full = prefix_seed_batch(ORDER, 0, 100).numpy()
    for o in outs:
        np.testing.assert_array_equal(o, full)


def test_max_over_ranks():
    assert run_ranks(_max) == [2.5, 2.5]


def test_gradient_mean_allreduce():
    for o in run_ranks(_mean):
        np.testing.assert_allclose(o, np.arange(6) * 1.5)


def test_best_plan_first_wins_by_global_episode():
    outs = run_ranks(_best_tie)
    assert outs[0] == outs[1] == (7, 2.5, 3, [1] * 5)


def test_best_plan_larger_key_wins():
    outs = run_ranks(_best_key)
    assert outs[0] == outs[1] == (8, 40, [10] * 3)


def test_best_plan_skips_ranks_without_completions():
    outs = run_ranks(_best_empty)
    assert outs[0] == outs[1] == (2, 17)
    assert run_ranks(_best_none) == [None, None]


def test_select_first_wins_single_process():
    p = torch.tensor([3, 5, 5, 5, -1], dtype=torch.int32)
    r = torch.tensor([9.0, 1.0, 2.0, 2.0, 99.0])
    e = torch.tensor([0, 4, 9, 6, -1])
    assert D.select_first_wins(p, r, e) == 3
    assert D.select_first_wins(p[-1:], r[-1:], e[-1:]) is None
