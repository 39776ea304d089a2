"""Multi-GPU plumbing for the plan-evaluation and DQN paths.

One process per GPU over `torch.distributed` (NCCL on the GPU box, gloo in the
CPU tests).  The data path has exactly two collectives:

* the Q-gradient all-reduce (mean) before every Adam step of the data-parallel
  learners (`vec.VecDqnTrainer.learn`);
* one all-gather of every rank's best completed plan, reduced with the
  reference's first-wins rule (`cli.py:237-240`: the incumbent is replaced only
  by a strictly greater (partitions, return), so among equal keys the earliest
  episode wins).  Episode ids are global, step·E·world + rank·E + env, so the
  winner never depends on rank order.

Plan evaluation itself needs no collective: rank r evaluates global plan rows
[r·B, (r+1)·B) (`plan_shard`); the timing uses the max over ranks.
"""

from __future__ import annotations


def rank_world(group=None) -> tuple[int, int]:
    import torch.distributed as dist

    if group is None and not (dist.is_available() and dist.is_initialized()):
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def plan_shard(rank: int, per_rank: int) -> tuple[int, int]:
    """(first global row, row count) of this rank's slice of the plan batch."""
    return rank * per_rank, per_rank


def _device_for(group):
    import torch
    import torch.distributed as dist

    return torch.device("cuda") if dist.get_backend(group) == "nccl" else torch.device("cpu")


def max_over_ranks(x: float, group=None) -> float:
    """Max of a per-rank scalar (device-timed milliseconds); identity on one process."""
    import torch
    import torch.distributed as dist

    if rank_world(group)[1] == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_device_for(group))
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def allreduce_mean_(t, group=None):
    """In-place mean over ranks (the data-parallel Q-gradient step)."""
    import torch.distributed as dist

    if group is not None or (dist.is_available() and dist.is_initialized()):
        if dist.get_world_size(group) > 1:
            if dist.get_backend(group) == "nccl":
                dist.all_reduce(t, op=dist.ReduceOp.AVG, group=group)
            else:  # gloo has no AVG
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
                t.div_(dist.get_world_size(group))
    return t


class PeerExchange:
    """Symmetric NVLink buffers for the fused gradient all-reduce + Adam kernel
    (`ap_dp_allreduce_adam`): per rank a [2, n] fp32 exchange buffer and a [W] flag
    row, mapped into every peer (torch symmetric memory).  `None` from `create`
    when symmetric memory is unavailable (the caller then uses NCCL)."""

    def __init__(self, n: int, group):
        import ctypes

        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm_mem

        self.rank, self.world = rank_world(group)
        dev = torch.device("cuda", torch.cuda.current_device())
        name = group.group_name if group is not None else dist.group.WORLD.group_name
        self.xbuf = symm_mem.empty(2 * n, dtype=torch.float32, device=dev)
        self.xbuf.zero_()
        hx = symm_mem.rendezvous(self.xbuf, name)
        self.pad = symm_mem.empty(self.world, dtype=torch.int32, device=dev)
        self.pad.zero_()
        hp = symm_mem.rendezvous(self.pad, name)
        self.counter = torch.zeros(1, dtype=torch.int32, device=dev)
        torch.cuda.synchronize()
        dist.barrier(group=group)  # every pad is zero before anyone signals
        W = self.world
        self.xbuf_ptrs = (ctypes.c_void_p * W)(*[hx.get_buffer(p, (2 * n,), torch.float32).data_ptr()
                                                 for p in range(W)])
        self.pad_ptrs = (ctypes.c_void_p * W)(*[hp.get_buffer(p, (W,), torch.int32).data_ptr() for p in range(W)])
        self._handles = (hx, hp)  # keep the mappings alive
        self.n = n

    @classmethod
    def create(cls, n: int, group):
        """Opt-in (AP_DP_FUSED=1).  Measured on 2 x B200 (BERT-48 OPP, E=4096, 4 learn
        steps per vector step, CUDA graph): 0.70 ms per vector step fused vs 0.63 ms
        with NCCL's all-reduce + the Adam kernel, so NCCL stays the default."""
        import os

        if os.environ.get("AP_DP_FUSED") != "1" or rank_world(group)[1] > 8:
            return None
        try:
            return cls(n, group)
        except Exception:  # no symmetric memory / peer access on this system
            return None


class BestPlan:
    """A completed partition plan: #partitioned candidates, return, global episode id,
    per-candidate statuses (int8, decision-dim order)."""

    __slots__ = ("partitions", "reward", "episode", "statuses")

    def __init__(self, partitions: int, reward: float, episode: int, statuses):
        self.partitions, self.reward, self.episode, self.statuses = partitions, reward, episode, statuses

    def key(self):
        return (self.partitions, self.reward)

    def __repr__(self) -> str:
        return f"BestPlan(partitions={self.partitions}, reward={self.reward}, episode={self.episode})"


def select_first_wins(partitions, returns, episodes):
    """Index of the max (partitions, return), lowest episode id among equal keys;
    entries with episode < 0 never completed.  None if nothing completed."""
    import torch

    valid = episodes >= 0
    if not bool(valid.any()):
        return None
    p = partitions.long()
    p = torch.where(valid, p, torch.full_like(p, -(1 << 40)))
    cand = valid & (p == p.max())
    r = torch.where(cand, returns.double(), torch.full_like(returns.double(), float("-inf")))
    cand &= r == r.max()
    e = torch.where(cand, episodes.long(), torch.full_like(episodes.long(), torch.iinfo(torch.int64).max))
    return int(torch.argmin(e))


def reduce_best(key, row, group=None) -> BestPlan | None:
    """All-gather every rank's (partitions, return, episode) and status row, pick the
    first-wins maximum.  Returns the same plan on every rank; None if no rank completed
    an episode.  `key` = (-1, -inf, -1) for a rank without a completed episode."""
    import torch
    import torch.distributed as dist

    k = torch.tensor([float(key[0]), float(key[1]), float(key[2])], dtype=torch.float64, device=row.device)
    world = rank_world(group)[1]
    if world == 1:
        keys, rows = k[None], row.reshape(1, -1)
    else:
        keys = torch.empty((world, 3), dtype=torch.float64, device=row.device)
        rows = torch.empty((world, row.numel()), dtype=row.dtype, device=row.device)
        dist.all_gather(list(keys.unbind(0)), k, group=group)
        dist.all_gather(list(rows.unbind(0)), row.contiguous().reshape(-1), group=group)
    j = select_first_wins(keys[:, 0].long(), keys[:, 1], keys[:, 2].long())
    if j is None:
        return None
    return BestPlan(int(keys[j, 0]), float(keys[j, 1]), int(keys[j, 2]), rows[j].cpu().numpy().copy())
