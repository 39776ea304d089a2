"""Device-resident vectorised search: E partition envs + a DQN learner, no host sync.

Throughput mode of the reference episode loop (`cli.py:193-248`): every
vector step does, for all E environments at once,

    act     Q over the E current states (tcgen05 GEMMs, M = E) + epsilon-greedy
    step    seed the chosen dims, batched propagation (K1), rewards / done /
            next positions / auto-reset (ap_vec_post)
    observe E transitions into the device replay ring
    learn   `learn_steps` double-DQN updates of batch `batch_size`

so the learn : env-step ratio is learn_steps : E (stated in every report).
Under torch.distributed each rank runs its own envs and learner replica;
the Q-gradient is all-reduced over NCCL before every Adam step, so replicas
stay identical (data-parallel DQN).  Parity with the reference's single
learner is a 1-GPU, E = 1 property of `search.train_partition`; this driver
is for throughput.
"""

from __future__ import annotations

import os

import numpy as np

from . import _native
from .distributed import BestPlan, PeerExchange, allreduce_mean_, rank_world, reduce_best, select_first_wins
from .agent import AdamOptimizer, AgentConfig, QNetwork, _Batch, fork_to, join_from, stream_or_current, sync_target
from .ir import decision_dims
from .linkage import extract_linkage_groups, sorted_decision_order
from .sharding import PropagationEngine, pad16


def _s():
    return _native.stream_handle()


class VecPartitionEnv:
    """E OPP (or ADP) environments stepping in lockstep on the device."""

    def __init__(self, graph, E: int, task: str = "opp"):
        import torch

        if task == "opp":
            dims = decision_dims(graph, graph.trainable_variables)
            order = sorted_decision_order(extract_linkage_groups(graph, dims))
        else:
            from .envs import adp_candidates

            dims = decision_dims(graph, [graph.instruction(i).name for i in adp_candidates(graph)])
            order = list(dims)
        self.dims = dims
        self.E = E
        self.n = n = len(dims)
        self.state_dim = n + 1
        self.num_actions = 2
        self.engine = PropagationEngine(graph, dims)
        self.engine.prepare()
        idx = {d: k for k, d in enumerate(dims)}
        self.order = torch.tensor([idx[d] for d in order], dtype=torch.int32, device="cuda")
        self.order_index = torch.empty_like(self.order)  # inverse permutation: dim -> rank in the order
        self.order_index[self.order.long()] = torch.arange(len(order), dtype=torch.int32, device="cuda")
        ld = pad16(n)
        dev = "cuda"
        self.seeds_full = torch.full((E, ld), -1, dtype=torch.int8, device=dev)
        self.seeds = self.seeds_full[:, :n]
        self.status = torch.empty((E, ld), dtype=torch.int8, device=dev)
        self.outcome = torch.empty(E, dtype=torch.uint8, device=dev)
        self.counts = torch.empty((E, 4), dtype=torch.int32, device=dev)
        self.prev_counts = torch.zeros((E, 2), dtype=torch.int32, device=dev)
        first = int(self.order[0].item())
        self.position = torch.full((E,), first, dtype=torch.int32, device=dev)
        self.cur_state = torch.full((E, self.state_dim), -1.0, dtype=torch.float32, device=dev)
        self.cur_state[:, n] = first / n
        self.next_state = torch.empty_like(self.cur_state)
        self.obs = torch.empty_like(self.cur_state)
        self.rewards = torch.empty(E, dtype=torch.float32, device=dev)
        self.done = torch.empty(E, dtype=torch.uint8, device=dev)
        self.next_mask = torch.empty((E, 2), dtype=torch.uint8, device=dev)
        self.mask = torch.ones((E, 2), dtype=torch.uint8, device=dev)
        self.ep_return = torch.zeros(E, dtype=torch.float32, device=dev)
        self.finished_return = torch.zeros(E, dtype=torch.float32, device=dev)
        self.finished_partitions = torch.full((E,), -1, dtype=torch.int32, device=dev)
        self.episodes_done = torch.zeros(E, dtype=torch.int32, device=dev)
        # per-env incumbent of completed episodes (cli.py:237-240), global episode ids
        self.best_partitions = torch.full((E,), -1, dtype=torch.int32, device=dev)
        self.best_return = torch.full((E,), float("-inf"), dtype=torch.float32, device=dev)
        self.best_episode = torch.full((E,), -1, dtype=torch.int64, device=dev)
        self.best_status = torch.full((E, ld), -1, dtype=torch.int8, device=dev)

    def step(self, actions, step_base: int = 0, ctl=None, world: int = 1, rank: int = 0) -> None:
        """Apply actions [E] int32 (device); fills rewards / done / next_state / next_mask.

        `step_base` + e is the global id of an episode finishing at this step
        (the best-plan tie-break: lowest id wins, cli.py:239).  With a device
        control block `ctl` the base is (ctl[0]·world + rank)·E instead."""
        lib = _native.require_device()
        P = _native.ptr
        self.obs.copy_(self.cur_state)
        _native.check(lib.ap_vec_apply(P(self.seeds_full), self.seeds_full.stride(0), P(self.position), P(actions),
                                       self.E, _s()))
        self.engine.launch(self.seeds, self.outcome, self.counts, None, self.status)
        _native.check(lib.ap_vec_post(self.E, self.n, self.seeds_full.stride(0), P(self.seeds_full), P(self.status),
                                      P(self.outcome), P(self.counts), P(self.prev_counts), P(self.position),
                                      P(self.order), P(self.order_index), P(self.cur_state), self.cur_state.stride(0),
                                      P(self.next_state),
                                      P(self.rewards), P(self.done), P(self.next_mask), 2, P(self.ep_return),
                                      P(self.finished_return), P(self.finished_partitions), P(self.episodes_done),
                                      _s()))
        _native.check(lib.ap_vec_track_best(self.E, self.n, self.seeds_full.stride(0), P(self.status), P(self.outcome),
                                            P(self.done), P(self.finished_partitions), P(self.finished_return),
                                            int(step_base), P(ctl) if ctl is not None else None, int(world),
                                            int(rank), P(self.best_partitions), P(self.best_return),
                                            P(self.best_episode), P(self.best_status), _s()))


class VecPipeTrainEnv:
    """E PipeTrainEnv episodes (envs.py:276-404) stepping in lockstep on the device.

    Each vector step appends one pivot per env (ap_vec_pipe_apply), evaluates the
    finished tuples (ap_pipe_metrics + ap_pipe_length over every env), pays the
    terminal rewards, records per-env incumbents and resets finished envs
    (ap_vec_pipe_post), then evaluates the next state of every env with K2
    (ap_pipe_train_state: all allowed candidates' features, [E, 4C]).  Finished
    transitions carry done = 1 and an empty next mask, so their next state (the
    reset state) never bootstraps.  Same device interface as VecPartitionEnv, so
    VecDqnTrainer drives it (and captures it in a CUDA graph) unchanged.
    """

    def __init__(self, graph, topo, num_stages: int, E: int, radius: int = 3, micro_batches: int = 4,
                 mem_per_device: float | None = None, reward_shape: str = "inv", backward_multiplier: float = 2.0):
        import torch

        from .envs import PipeTrainEnv

        host = PipeTrainEnv(graph, topo, num_stages, radius, micro_batches, mem_per_device=mem_per_device,
                            reward_shape=reward_shape, backward_multiplier=backward_multiplier)
        self.host = host
        self.E = E
        self.K = num_stages
        self.P = P = num_stages - 1
        self.C = C = host.num_actions
        self.a_max = max(1, num_stages - 2)
        self.num_actions = C
        self.state_dim = 4 * C
        self.topo_c = _native.Topology.of(topo)
        self.micro_batches = micro_batches
        self.mem = -1.0 if mem_per_device is None else float(mem_per_device)
        self.reward_shape = 0 if reward_shape == "inv" else 1
        self.bwm = float(backward_multiplier)
        dev = "cuda"
        i32, u8, f64, f32 = torch.int32, torch.uint8, torch.float64, torch.float32
        self.cand_pos = torch.from_numpy(host._cand_pos).to(dev)
        host._model.bind_candidates(self.cand_pos)  # stage-sum table: K2 by lookups
        self.dummy_pos = self.cand_pos[C - P:].clone()  # a legal increasing pivot tuple
        self.picks = torch.full((E, P), -1, dtype=i32, device=dev)
        self.positions = self.dummy_pos.repeat(E, 1).contiguous()
        self.n_applied = torch.zeros(E, dtype=i32, device=dev)
        self.done = torch.zeros(E, dtype=u8, device=dev)
        self.applied_state = torch.full((E, self.a_max), -1, dtype=i32, device=dev)
        self.mask = torch.zeros((E, C), dtype=u8, device=dev)
        self.next_mask = torch.zeros((E, C), dtype=u8, device=dev)
        self.state64 = torch.zeros((E, 4 * C), dtype=f64, device=dev)
        self.cur_state = torch.zeros((E, 4 * C), dtype=f32, device=dev)
        self.obs = torch.empty_like(self.cur_state)
        self.next_state = torch.empty_like(self.cur_state)
        self.rewards = torch.zeros(E, dtype=f32, device=dev)
        K = num_stages
        self.comp = torch.empty((E, K), dtype=f64, device=dev)
        self.act = torch.empty((E, K), dtype=f64, device=dev)
        self.param = torch.empty((E, K), dtype=f64, device=dev)
        self.nvars = torch.empty((E, K), dtype=i32, device=dev)
        self.cuts = torch.empty((E, K - 1), dtype=i32, device=dev)
        self.length = torch.zeros(E, dtype=f64, device=dev)
        self.feasible = torch.zeros(E, dtype=u8, device=dev)
        self.best_len = torch.full((E,), float("inf"), dtype=f64, device=dev)
        self.best_picks = torch.full((E, P), -1, dtype=i32, device=dev)
        self.best_episode = torch.full((E,), -1, dtype=torch.int64, device=dev)
        self.ep_return = torch.zeros(E, dtype=f32, device=dev)
        self.finished_return = torch.zeros(E, dtype=f32, device=dev)
        self.episodes_done = torch.zeros(E, dtype=i32, device=dev)
        self._ctl0 = torch.zeros(4, dtype=torch.int64, device=dev)
        self._post(self._ctl0, 1, 0)  # initial masks / applied rows (nothing is done yet)
        self._state_eval()

    def _post(self, ctl, world, rank) -> None:
        lib = _native.require_device()
        P_ = _native.ptr
        _native.check(lib.ap_vec_pipe_post(self.E, self.C, self.P, self.a_max, P_(self.length), P_(self.feasible),
                                           P_(self.done), self.reward_shape, P_(self.dummy_pos), P_(self.rewards),
                                           P_(self.picks), P_(self.positions), P_(self.n_applied),
                                           P_(self.applied_state), P_(self.mask), P_(self.next_mask),
                                           P_(self.best_len), P_(self.best_picks), P_(self.best_episode),
                                           P_(self.ep_return), P_(self.finished_return), P_(self.episodes_done),
                                           P_(ctl), int(world), int(rank), _s()))

    def _state_eval(self, next_too: bool = False) -> None:
        """K2 into state64 and the fp32 cur_state (and next_state) rows in one call."""
        import ctypes

        lib = _native.require_device()
        P_ = _native.ptr
        nxt = self.next_state if next_too else None
        _native.check(lib.ap_pipe_train_state_ex(self.host._model.handle, ctypes.byref(self.topo_c), P_(self.cand_pos),
                                                 self.C, P_(self.applied_state), self.a_max, P_(self.mask), self.E,
                                                 self.bwm, P_(self.state64), P_(self.cur_state),
                                                 self.cur_state.stride(0), P_(nxt) if nxt is not None else None,
                                                 nxt.stride(0) if nxt is not None else 0, _s()))

    def step(self, actions, step_base: int = 0, ctl=None, world: int = 1, rank: int = 0) -> None:
        """Apply one pick per env (actions [E] int32, device); fills rewards / done /
        next_state / next_mask and the post-reset cur_state / mask."""
        import ctypes

        lib = _native.require_device()
        P_ = _native.ptr
        self.obs.copy_(self.cur_state)
        _native.check(lib.ap_vec_pipe_apply(self.E, self.P, P_(actions), P_(self.cand_pos), P_(self.picks),
                                            P_(self.positions), P_(self.n_applied), P_(self.done), _s()))
        _native.check(lib.ap_pipe_metrics_bound(self.host._model.handle, P_(self.cand_pos), self.C, P_(self.positions),
                                                self.E, self.P, self.bwm, P_(self.comp), P_(self.act), P_(self.param),
                                                P_(self.nvars), _s()))
        _native.check(lib.ap_pipe_length(ctypes.byref(self.topo_c), self.K, self.micro_batches, self.E, P_(self.comp),
                                         P_(self.act), P_(self.param), P_(self.cuts), 0, self.mem, 4.0, 1,
                                         P_(self.length), P_(self.feasible), _s()))
        self._post(ctl if ctl is not None else self._ctl0, world, rank)
        self._state_eval(next_too=True)  # cur_state and next_state written by the K2 kernel

    def best_plan(self):
        """(pipeline length, pivot names, global episode id) of the best feasible finished
        episode on this rank (min length, lowest episode id among ties), or None."""
        import torch

        valid = self.best_episode >= 0
        if not bool(valid.any()):
            return None
        L = torch.where(valid, self.best_len, torch.full_like(self.best_len, float("inf")))
        cand = valid & (L == L.min())
        k = int(torch.argmin(torch.where(cand, self.best_episode, torch.full_like(self.best_episode, 1 << 62))))
        picks = self.best_picks[k].tolist()
        return float(self.best_len[k]), tuple(self.host.candidates[i] for i in picks), int(self.best_episode[k])


class VecPipeInferEnv:
    """E PipeInferEnv episodes (envs.py:407-626) stepping in lockstep on the device.

    Boundaries first, then device cuts (ap_vec_infer_apply); every row's point is
    evaluated by the batched PP-infer length kernel (ap_infer_length, dummy tails
    keep unfinished rows legal); ap_vec_infer_post pays 1 / L on the last cut,
    keeps per-env incumbents, resets, and rebuilds the phased masks and the pick
    slots of the fp32 state (static part: C*, A*, W*, normalised bandwidths).
    """

    def __init__(self, arrays, topo, num_stages: int, E: int, micro_batches: int = 1,
                 allowed_boundaries=None, allowed_cuts=None):
        import ctypes  # noqa: F401

        import torch

        from .envs import GRANULARITY, PipeInferEnv

        host = PipeInferEnv(arrays, topo, num_stages, micro_batches=micro_batches,
                            allowed_boundaries=allowed_boundaries, allowed_cuts=allowed_cuts)
        self.host = host
        self.E, self.K, self.P = E, num_stages, num_stages - 1
        self.G, self.D = GRANULARITY, topo.num_devices
        self.num_actions = host.num_actions
        self.state_dim = S = host.state_dim
        self.micro_batches = micro_batches
        self.topo_c = _native.Topology.of(host.topo_norm)
        dev = "cuda"
        i32, u8, f64, f32 = torch.int32, torch.uint8, torch.float64, torch.float32
        P, G, D = self.P, self.G, self.D
        self.arrays_dev = host._arrays_dev()
        self.dummy_b = torch.arange(G - P, G, dtype=i32, device=dev)
        self.dummy_c = torch.arange(D - P, D, dtype=i32, device=dev)
        band_b = np.ones((P, G), np.uint8)
        band_c = np.ones((P, D), np.uint8)
        for k in range(P):
            if allowed_boundaries is not None:
                band_b[k] = 0
                band_b[k, sorted(allowed_boundaries[k])] = 1
            if allowed_cuts is not None:
                band_c[k] = 0
                band_c[k, sorted(allowed_cuts[k])] = 1
        self.band_b = torch.from_numpy(band_b).to(dev)
        self.band_c = torch.from_numpy(band_c).to(dev)
        self.bnd = self.dummy_b.repeat(E, 1).contiguous()
        self.cut = self.dummy_c.repeat(E, 1).contiguous()
        self.nb = torch.zeros(E, dtype=i32, device=dev)
        self.nc = torch.zeros(E, dtype=i32, device=dev)
        self.done = torch.zeros(E, dtype=u8, device=dev)
        A = self.num_actions
        self.mask = torch.zeros((E, A), dtype=u8, device=dev)
        self.next_mask = torch.zeros((E, A), dtype=u8, device=dev)
        static = torch.from_numpy(host._static.astype(np.float32)).to(dev)
        # state rows padded to a 16-byte stride (TMA-fed GEMMs need it), width S
        ld = (S + 3) // 4 * 4
        self.cur_state = torch.zeros((E, ld), dtype=f32, device=dev)[:, :S]
        self.cur_state[:, : S - 2 * P] = static
        self.obs = torch.zeros((E, ld), dtype=f32, device=dev)[:, :S]
        self.next_state = torch.zeros((E, ld), dtype=f32, device=dev)[:, :S]
        self.rewards = torch.zeros(E, dtype=f32, device=dev)
        self.length = torch.zeros(E, dtype=f64, device=dev)
        self.best_len = torch.full((E,), float("inf"), dtype=f64, device=dev)
        self.best_b = torch.full((E, P), -1, dtype=i32, device=dev)
        self.best_c = torch.full((E, P), -1, dtype=i32, device=dev)
        self.best_episode = torch.full((E,), -1, dtype=torch.int64, device=dev)
        self.ep_return = torch.zeros(E, dtype=f32, device=dev)
        self.finished_return = torch.zeros(E, dtype=f32, device=dev)
        self.episodes_done = torch.zeros(E, dtype=i32, device=dev)
        self._ctl0 = torch.zeros(4, dtype=torch.int64, device=dev)
        self._post(self._ctl0, 1, 0)

    def _post(self, ctl, world, rank) -> None:
        lib = _native.require_device()
        P_ = _native.ptr
        _native.check(lib.ap_vec_infer_post(self.E, self.P, self.G, self.D, self.state_dim,
                                            self.cur_state.stride(0), P_(self.length),
                                            P_(self.done), P_(self.dummy_b), P_(self.dummy_c), P_(self.band_b),
                                            P_(self.band_c), P_(self.rewards), P_(self.bnd), P_(self.cut),
                                            P_(self.nb), P_(self.nc), P_(self.mask), P_(self.next_mask),
                                            P_(self.cur_state), P_(self.best_len), P_(self.best_b), P_(self.best_c),
                                            P_(self.best_episode), P_(self.ep_return), P_(self.finished_return),
                                            P_(self.episodes_done), P_(ctl), int(world), int(rank), _s()))

    def step(self, actions, step_base: int = 0, ctl=None, world: int = 1, rank: int = 0) -> None:
        import ctypes

        lib = _native.require_device()
        P_ = _native.ptr
        self.obs.copy_(self.cur_state)
        _native.check(lib.ap_vec_infer_apply(self.E, self.P, self.G, P_(actions), P_(self.bnd), P_(self.cut),
                                             P_(self.nb), P_(self.nc), P_(self.done), _s()))
        _native.check(lib.ap_infer_length(P_(self.arrays_dev), self.G, ctypes.byref(self.topo_c), self.K,
                                          self.micro_batches, P_(self.bnd), P_(self.cut), self.E, P_(self.length),
                                          _s()))
        self._post(ctl if ctl is not None else self._ctl0, world, rank)
        self.next_state.copy_(self.cur_state)

    def best_plan(self):
        """(pipeline length, boundaries, device cuts, global episode id) of the best finished
        episode on this rank (min length, lowest episode id among ties), or None."""
        import torch

        valid = self.best_episode >= 0
        if not bool(valid.any()):
            return None
        L = torch.where(valid, self.best_len, torch.full_like(self.best_len, float("inf")))
        cand = valid & (L == L.min())
        k = int(torch.argmin(torch.where(cand, self.best_episode, torch.full_like(self.best_episode, 1 << 62))))
        return (float(self.best_len[k]), tuple(self.best_b[k].tolist()), tuple(self.best_c[k].tolist()),
                int(self.best_episode[k]))


class VecDqnTrainer:
    """Batched acting + device replay + (data-parallel) DQN learner over a VecPartitionEnv.

    Every step counter the kernels need (vector step, ring slot / size, train
    steps) lives in a device control block `ctl` (`AP_CTL_*`), so one vector
    step has no host-baked arguments.  With `use_graph=True` the whole step —
    act, K1 propagation, post, best-plan tracking, replay push and the L learn
    steps (including the NCCL gradient all-reduce) — is captured once into a
    CUDA graph and replayed; the host keeps mirrors of the counters and does
    the target sync (a device copy) between replays every `target_sync_every`
    train steps.
    """

    CTL_STEP, CTL_SLOT, CTL_SIZE, CTL_TRAIN = 0, 1, 2, 3

    def __init__(self, env: VecPartitionEnv, config: AgentConfig, capacity: int, seed: int = 0,
                 learn_steps: int = 1, process_group=None, precision: int = 1, use_graph: bool = False):
        import torch

        self.env = env
        self.config = config
        self.capacity = capacity
        self.learn_steps = learn_steps
        self.pg = process_group
        self.seed = seed
        rng = np.random.default_rng(seed)
        self.net = QNetwork(env.state_dim, env.num_actions, config.hidden, rng)
        self.net.precision = precision  # TF32 tensor cores by default in throughput mode
        if process_group is not None:  # identical replicas: broadcast rank 0's init
            import torch.distributed as dist

            dist.broadcast(self.net.flat, src=0, group=process_group)
            self.net.refresh_transposed()
        self.target = self.net.clone()
        self.opt = AdamOptimizer(self.net, config)
        S, A, dev = env.state_dim, env.num_actions, "cuda"
        self.ring = {
            "states": torch.zeros((capacity, S), dtype=torch.float32, device=dev),
            "next_states": torch.zeros((capacity, S), dtype=torch.float32, device=dev),
            "actions": torch.zeros(capacity, dtype=torch.int32, device=dev),
            "rewards": torch.zeros(capacity, dtype=torch.float32, device=dev),
            "done": torch.zeros(capacity, dtype=torch.uint8, device=dev),
            "next_mask": torch.zeros((capacity, A), dtype=torch.uint8, device=dev),
            "priorities": torch.zeros(capacity, dtype=torch.float64, device=dev),
            "cdf": torch.zeros(capacity, dtype=torch.float64, device=dev),
        }
        self.max_prio = torch.ones(1, dtype=torch.float64, device=dev)
        self.ctl = torch.zeros(4, dtype=torch.int64, device=dev)
        self.size = 0  # host mirrors of ctl
        self.slot = 0
        self.actions = torch.empty(env.E, dtype=torch.int32, device=dev)
        self.batch = _Batch(config.batch_size, S, A)
        # [2B, S] with rows padded to a 16-byte stride (TMA operand rule)
        # double-buffered: the pipelined learner gathers step k + 1's batch while step k's backward reads its own
        self.sn_bufs = [torch.empty((2 * config.batch_size, (S + 3) // 4 * 4), dtype=torch.float32, device=dev)[:, :S]
                        for _ in range(2)]
        self.dz_t = torch.empty((1 + A, config.batch_size), dtype=torch.float32, device=dev)
        self.idx = torch.empty(config.batch_size, dtype=torch.int32, device=dev)
        self.weights = torch.empty(config.batch_size, dtype=torch.float32, device=dev)
        self.train_steps = 0
        self.vector_steps = 0
        self.launches = 0
        self.rank, self.world = rank_world(process_group) if process_group is not None else (0, 1)
        # fused NVLink all-reduce + Adam when the ranks can map each other's memory
        self.peer = PeerExchange.create(self.net.flat.numel(), process_group) if self.world > 1 else None
        self.use_graph = use_graph
        self.graph = None
        self._graph_launches = 0
        # side stream for the learner's parallel branches (target forward, weight gradients);
        # AP_DQN_NO_FORK=1 keeps one serial chain
        self.side = None if os.environ.get("AP_DQN_NO_FORK") else torch.cuda.Stream()
        # second branch: priority scatter + next sample / gather beside the backward (AP_DQN_NO_PIPELINE=1: serial)
        self.side2 = None if (os.environ.get("AP_DQN_NO_FORK") or os.environ.get("AP_DQN_NO_PIPELINE")) \
            else torch.cuda.Stream()

    # -- one vector step -------------------------------------------------------------

    def act(self) -> None:
        lib = _native.require_device()
        env, cfg = self.env, self.config
        q = self.net.forward_device(env.cur_state)
        _native.check(lib.ap_dqn_act_ctl(_native.ptr(q), q.stride(0), _native.ptr(env.mask), env.mask.stride(0), env.E,
                                         env.num_actions, float(cfg.epsilon_start), float(cfg.epsilon_final),
                                         int(cfg.epsilon_decay_iters), _native.ptr(self.ctl),
                                         _native.ptr(self.actions), _s()))
        self.launches += 4  # 3 GEMMs + act

    def observe(self) -> None:
        lib = _native.require_device()
        env, r = self.env, self.ring
        P = _native.ptr
        _native.check(lib.ap_per_push_ctl(env.E, env.state_dim, env.num_actions, self.capacity, P(env.obs),
                                          P(env.next_state), env.obs.stride(0), P(self.actions), P(env.rewards),
                                          P(env.done), P(env.next_mask), P(r["states"]), P(r["next_states"]),
                                          P(r["actions"]), P(r["rewards"]), P(r["done"]), P(r["next_mask"]),
                                          P(r["priorities"]), P(self.max_prio), P(self.ctl), _s()))
        self.launches += 1

    def _sample_gather(self, k: int) -> None:
        """PER sample of learn step k and its [2B, S] state / next-state block (buffer k % 2)."""
        cfg, r = self.config, self.ring
        B = cfg.batch_size
        lib = _native.require_device()
        P = _native.ptr
        _native.check(lib.ap_per_sample_ctl(P(r["priorities"]), self.capacity, cfg.per_beta, B,
                                            self.seed * 1000003 + self.rank,
                                            P(r["cdf"]), P(self.idx), P(self.weights), P(self.max_prio), P(self.ctl),
                                            _s()))
        # states and next states gathered into one [2B, S] block: the online
        # network runs once over both (M = 2B), the target net over the second half
        sn = self.sn_bufs[k % 2]
        s0, s1 = r["states"], r["next_states"]
        _native.check(lib.ap_gather_rows_pair(P(s0), s0.stride(0), P(sn[:B]), sn.stride(0), P(s1), s1.stride(0),
                                              P(sn[B:]), sn.stride(0), P(self.idx), B, s0.shape[1], _s()))

    def learn(self, k: int = 0, prefetched: bool = False, prefetch_next: bool = False) -> None:
        """One learner update.  Pipelined (self.side2): the priority scatter of this
        step, then the sample + gather of step k + 1, run on a parallel branch beside
        the backward pass; the branch joins before Adam, which then reads the already
        advanced step counter.  Every value equals the serial order's."""
        import torch

        cfg, r, b = self.config, self.ring, self.batch
        B = cfg.batch_size
        lib = _native.require_device()
        P = _native.ptr
        pipe = self.side2 is not None and self.peer is None
        if not prefetched:
            self._sample_gather(k)
        sn = self.sn_bufs[k % 2]
        side = self.side
        if side is not None:  # the target forward is a parallel branch beside the online forward
            fork_to(side)
        with stream_or_current(side):
            target_next = self.target.forward_device(sn[B:])
        q2, acts2 = self.net.forward_device(sn, cache=True)
        if side is not None:
            join_from(side)
        q_all, online_next = q2[:B], q2[B:]
        acts = [a[:B] for a in acts2]
        _native.check(lib.ap_dqn_td_ring(P(q_all), P(online_next), P(target_next), q2.stride(0), P(self.idx),
                                         P(r["actions"]), P(r["rewards"]), P(r["done"]), P(r["next_mask"]),
                                         r["next_mask"].stride(0), P(self.weights), B, self.env.num_actions,
                                         float(cfg.gamma), float(cfg.huber_delta), P(b.dz), b.dz.stride(0),
                                         P(self.dz_t), self.dz_t.stride(0), P(b.td), P(b.loss_rows), _s()))
        opt = self.opt
        fused_adam = None
        if pipe:  # priority scatter (+ step counter) and the next step's sample / gather, beside the backward
            fork_to(self.side2)
            with stream_or_current(self.side2):
                _native.check(lib.ap_per_update_scaled_ctl(P(r["priorities"]), P(self.idx), P(b.td), B,
                                                           float(cfg.per_alpha), P(self.ctl), _s()))
                if self.pg is None and side is not None and os.environ.get("AP_FUSED_ADAM"):
                    # opt-in (measured slower on B200: the gradient GEMM has too few CTAs to carry the
                    # Adam traffic): the first layer's Adam in its weight-gradient GEMM epilogue, after
                    # the step counter has advanced (the event), like the Adam below
                    counted = torch.cuda.Event()
                    counted.record(torch.cuda.current_stream())
                    fused_adam = dict(m=opt.m, v=opt.v, ctl=self.ctl, counter_advanced=1, lr=opt.lr,
                                      beta1=opt.beta1, beta2=opt.beta2, eps=opt.eps, wait=counted)
                if prefetch_next:
                    self._sample_gather(k + 1)
        fused = self.net.backward_device(acts, b.dz, self.dz_t, side=side, dueling_td=True,
                                         fused_w0_adam=fused_adam)
        if pipe:
            join_from(self.side2)
        if self.peer is not None:  # data-parallel: gradient all-reduce over NVLink peer memory fused with Adam
            x = self.peer
            _native.check(lib.ap_dp_allreduce_adam(x.world, x.rank, P(self.net.grad), x.xbuf_ptrs, x.pad_ptrs,
                                                   self.net.flat.numel(), P(self.net.flat), P(opt.m), P(opt.v),
                                                   opt.lr, opt.beta1, opt.beta2, opt.eps, P(self.ctl),
                                                   P(x.counter), _s()))
        else:
            if self.pg is not None:  # data-parallel learners without peer memory: NCCL mean all-reduce
                allreduce_mean_(self.net.grad, self.pg)
            # Adam also rewrites the transposed weight copies (no separate transpose launch;
            # measured faster than Adam + a tiled transpose even for the 4 M-parameter PP-train net)
            o = self.net.w0_block() if fused else 0  # fused: w0 / b0 were updated by their gradient GEMM
            sg = self.net.adam_segments(skip_w0=fused)
            _native.check(lib.ap_dqn_adam_ctl_t_adv(P(self.net.flat[o:]), P(self.net.grad[o:]), P(opt.m[o:]),
                                                    P(opt.v[o:]), self.net.flat.numel() - o, opt.lr, opt.beta1,
                                                    opt.beta2, opt.eps, P(self.ctl), *sg, 1 if pipe else 0, _s()))
        if self.peer is not None:
            self.net.refresh_transposed()
        if not pipe:  # the priority scatter also counts the learn step (ctl[AP_CTL_TRAIN] += 1)
            _native.check(lib.ap_per_update_scaled_ctl(P(r["priorities"]), P(self.idx), P(b.td), B,
                                                       float(cfg.per_alpha), P(self.ctl), _s()))
        Lh = len(self.net.hidden)
        head = 1 if 1 + self.env.num_actions <= 8 else 2  # narrow fused head | GEMM + dueling (row-sum + closed form)
        fwd = 2 * (Lh + head)  # online and target forwards
        bwd = 1 + 1 + head + Lh + 2 * (Lh - 1)  # transpose, head wgrad, head dgrad, wgrads, dgrad + ReLU per layer
        self.launches += 1 + 1 + fwd + 1 + bwd + 1 + 1  # sample, pair gather, .., td, .., adam, priority scatter

    def _step_body(self, learn: bool) -> None:
        self.act()
        E = self.env.E
        self.env.step(self.actions, ctl=self.ctl, world=self.world, rank=self.rank)
        self.launches += 4
        self.observe()
        # step counter, ring slot and size advance right after the push: every
        # reader of the step counter (act, track-best) has run, and the learner
        # must sample over the ring including this step's transitions
        lib = _native.require_device()
        _native.check(lib.ap_vec_ctl_advance(_native.ptr(self.ctl), 1, E, self.capacity, _s()))
        self.launches += 1
        if learn:
            pipe = self.side2 is not None and self.peer is None
            L = self.learn_steps
            for k in range(L):
                self.learn(k, prefetched=pipe and k > 0, prefetch_next=pipe and k + 1 < L)

    def _advance_host(self, learned: bool) -> None:
        E = self.env.E
        if learned:
            for _ in range(self.learn_steps):
                self.train_steps += 1
                if self.train_steps % self.config.target_sync_every == 0:
                    sync_target(self.net, self.target)
        self.slot = (self.slot + E) % self.capacity
        self.size = min(self.size + E, self.capacity)
        self.vector_steps += 1

    def step(self) -> None:
        import torch

        # learn once the ring holds a batch after this step's push (agent.py:318-337)
        learn = min(self.size + self.env.E, self.capacity) >= self.config.batch_size
        if not (self.use_graph and learn):
            self._step_body(learn)
            self._advance_host(learn)
            return
        if self.graph is None:
            # one eager step first, on the stream the capture will use: allocates every
            # lazily-sized buffer (split-K workspaces are per (device, stream), torch
            # temporaries) outside the capture
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                self._step_body(learn)
            torch.cuda.current_stream().wait_stream(s)
            self._advance_host(learn)
            launches0 = self.launches
            s.wait_stream(torch.cuda.current_stream())
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                with torch.cuda.graph(self.graph, stream=s):
                    self._step_body(learn)
            torch.cuda.current_stream().wait_stream(s)
            # capture records the work without running it: device state is unchanged
            self._graph_launches = self.launches - launches0
            self.launches = launches0
            return  # this call's vector step was the eager warm-up
        self.graph.replay()
        self.launches += self._graph_launches
        self._advance_host(learn)

    # -- reporting ---------------------------------------------------------------------

    def best_plan(self) -> BestPlan | None:
        """Best completed plan on this rank (max (partitions, return), lowest episode id);
        for the PP envs the env's own (length, picks..., episode) incumbent."""
        env = self.env
        if isinstance(env, (VecPipeTrainEnv, VecPipeInferEnv)):
            return env.best_plan()
        k = select_first_wins(env.best_partitions, env.best_return, env.best_episode)
        if k is None:
            return None
        return BestPlan(int(env.best_partitions[k]), float(env.best_return[k]), int(env.best_episode[k]),
                        env.best_status[k, : env.n].cpu().numpy().copy())

    def best_plan_global(self) -> BestPlan | None:
        """Best completed plan over all ranks: one all-gather of (key, episode id, statuses).
        PP envs: key (0, -length) so the shortest pipeline wins; the row holds the picks
        (PP-train pivots, or PP-infer boundaries followed by cuts)."""
        env = self.env
        if isinstance(env, (VecPipeTrainEnv, VecPipeInferEnv)):
            import torch

            best = env.best_plan()
            picks = env.best_picks if isinstance(env, VecPipeTrainEnv) else torch.cat([env.best_b, env.best_c], 1)
            if best is None:
                key, row = (-1, float("-inf"), -1), picks.new_full((picks.shape[1],), -1)
            else:
                k = int(torch_argmax_episode(env, best[-1]))
                key, row = (0, -best[0], best[-1]), picks[k]
            return reduce_best(key, row, self.pg)
        k = select_first_wins(env.best_partitions, env.best_return, env.best_episode)
        if k is None:
            key = (-1, float("-inf"), -1)
            row = env.best_status.new_full((env.n,), -1)
        else:
            key = (int(env.best_partitions[k]), float(env.best_return[k]), int(env.best_episode[k]))
            row = env.best_status[k, : env.n]
        return reduce_best(key, row, self.pg)


def torch_argmax_episode(env, episode: int) -> int:
    """Env index holding the incumbent with global episode id `episode`."""
    import torch

    return int(torch.nonzero(env.best_episode == episode)[0, 0])
