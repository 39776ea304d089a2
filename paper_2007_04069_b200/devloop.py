"""The reference episode loop on the device: `train_partition_device`.

Same signature, draws and results as `search.train_partition` (reference
`cli.py:193-248`) for one `OppEnv` / `AdpEnv` and a `DqnAgent`, but every step
runs on the GPU without returning to the host:

* agent.act (agent.py:155-170) -- `ap_parity_act`: numpy's PCG64 stream on the
  device (random(), then integers(#allowed) when exploring), masked argmax of the
  Q-network output otherwise;
* env.step (envs.py:133-175) -- K1 on one seed row + `ap_parity_post`: reward in
  fp64 exactly as the reference adds it, next decision position, CONFLICT /
  COMPLETE, the episode's return and the incumbent (strictly greater
  (partitions, return), first wins, cli.py:237-240), reset to the episode
  template (reset or finetune_reset);
* agent.observe (agent.py:197-205) -- the ring push at the current max priority;
* agent.learn (agent.py:207-337) -- 64 random() draws, the numpy-ordered PER
  sampler, the update shared with the host agent (`agent.update_on_indices`),
  Adam with the host's bias corrections, target sync every 100 train steps.

The step and learn sequences are captured once as CUDA graphs and wrapped by
`ap_loop_graph_create` in a graph with device-side control flow: WHILE
(episodes < budget) { step; learn }, where the learn kernels (fused learner)
skip themselves while the ring holds fewer than a batch (`learn_gate`), so the
body is one graph with programmatic-dependent-launch edges; the GEMM learner
keeps an IF (ring holds a batch) node around its learn graph instead.  One graph
launch runs a whole block of episodes.  Afterwards the agent (RNG state, train
steps, Adam step, ring) and the env are left exactly as the host loop leaves
them, so host and device loops can be mixed (the finetune stage continues the
same agent).  Per-step logs (actions, rewards, optionally the state rows for
trace digests) come back once per launch.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from . import _native
from .agent import DqnAgent, DivergenceError, epsilon_at, update_on_indices
from .envs import PartitionSearchEnv
from .ir import DimIndex
from .search import PartitionOutcome, state_digest
from .sharding import DimStatus, pad16

_LOG_BYTES = 256 << 20  # state-row log budget per launch (trace digests)
# steps per WHILE iteration of the self-gated loop graph (a WHILE iteration costs ~30 us)
_STEPS_PER_ITER = int(os.environ.get("AP_LOOP_STEPS_PER_ITER", "8"))
# device time / env steps / launches of the last train_partition_device call (bench.py reads it)
last_stats: dict = {}


def _stream():
    return _native.stream_handle()


class DeviceSearch:
    """Device buffers, captured graphs and the loop graph for one (env, agent) pair."""

    def __init__(self, env: PartitionSearchEnv, agent: DqnAgent, steps_per_launch: int, log_rows: bool):
        import torch

        self.env, self.agent = env, agent
        n = len(env.dims)
        A = env.num_actions
        cfg = agent.config
        self.n, self.A, self.ld = n, A, pad16(n)
        self.steps_cap = steps_per_launch
        self.log_rows = log_rows
        dev = "cuda"
        i8, i32, i64, f32, f64 = torch.int8, torch.int32, torch.int64, torch.float32, torch.float64
        buf = agent.buffer
        if buf.store is None:
            buf._alloc(env.state_dim, A)
        st = buf.store
        self.t = {
            "ctl": torch.zeros(_native.PL["WORDS"], dtype=i64, device=dev),
            "dctl": torch.zeros(2, dtype=f64, device=dev),
            "rng": torch.zeros(6, dtype=i64, device=dev),
            "rng_next": torch.zeros(6, dtype=i64, device=dev),
            "scaled": torch.zeros(buf.capacity, dtype=f64, device=dev),
            "pstat": torch.ones(2, dtype=f64, device=dev),
            "seeds": torch.full((self.ld,), -1, dtype=i8, device=dev),
            "seeds_try": torch.full((1, self.ld), -1, dtype=i8, device=dev),
            "decided": torch.full((self.ld,), -1, dtype=i8, device=dev),
            "status": torch.full((1, self.ld), -1, dtype=i8, device=dev),
            "outcome": torch.zeros(1, dtype=torch.uint8, device=dev),
            "order": torch.as_tensor(np.asarray(env._order_idx, dtype=np.int32), device=dev),
            "t_seeds": torch.full((self.ld,), -1, dtype=i8, device=dev),
            "t_decided": torch.full((self.ld,), -1, dtype=i8, device=dev),
            # contiguous [1, S], the shape the host agent's act feeds the Q-network (same GEMM path)
            "state": torch.zeros((1, env.state_dim), dtype=f32, device=dev),
            "action": torch.zeros(1, dtype=i32, device=dev),
            "q": torch.zeros((1, A), dtype=f32, device=dev),
            "act_bar": torch.zeros(4, dtype=i32, device=dev),
            "best_row": torch.full((self.ld,), -1, dtype=i8, device=dev),
            "log_action": torch.zeros(steps_per_launch, dtype=i32, device=dev),
            "log_reward": torch.zeros(steps_per_launch, dtype=f64, device=dev),
            "log_pos": torch.zeros(steps_per_launch, dtype=i32, device=dev),
            "log_decided": torch.zeros((steps_per_launch if log_rows else 1, self.ld), dtype=i8, device=dev),
            "ep_conflict": torch.zeros(steps_per_launch, dtype=torch.uint8, device=dev),
            "ep_len": torch.zeros(steps_per_launch, dtype=i32, device=dev),
            "ep_return": torch.zeros(steps_per_launch, dtype=f64, device=dev),
            "loss_log": torch.zeros(steps_per_launch, dtype=f32, device=dev),
            "ctab": torch.zeros(2 * steps_per_launch, dtype=f32, device=dev),
            "idx": torch.zeros(cfg.batch_size, dtype=i32, device=dev),
            "weights": torch.zeros(cfg.batch_size, dtype=f32, device=dev),
        }
        t = self.t
        P = lambda x: x.data_ptr()  # noqa: E731
        self.desc = _native.ParityLoopDesc(
            ctl=P(t["ctl"]), dctl=P(t["dctl"]), rng=P(t["rng"]), n=n, ld=self.ld, num_actions=A,
            seeds=P(t["seeds"]), seeds_try=P(t["seeds_try"]), decided=P(t["decided"]), status=P(t["status"]),
            outcome=P(t["outcome"]), order=P(t["order"]), t_seeds=P(t["t_seeds"]), t_decided=P(t["t_decided"]),
            state=P(t["state"]), r_states=P(st["states"]), r_next=P(st["next_states"]),
            r_ld=st["states"].stride(0), cap=buf.capacity, r_actions=P(st["actions"]), r_rewards=P(st["rewards"]),
            r_done=P(st["done"]), r_mask=P(st["next_mask"]), r_prio=P(st["priorities"]),
            eps_start=float(cfg.epsilon_start), eps_final=float(cfg.epsilon_final),
            eps_decay=int(cfg.epsilon_decay_iters), best_row=P(t["best_row"]), log_action=P(t["log_action"]),
            log_reward=P(t["log_reward"]), log_pos=P(t["log_pos"]),
            log_decided=P(t["log_decided"]) if log_rows else None, ep_conflict=P(t["ep_conflict"]),
            ep_len=P(t["ep_len"]), ep_return=P(t["ep_return"]), loss_log=P(t["loss_log"]),
            loss_cap=steps_per_launch)
        self.adam_offset = agent.optimizer.t - agent.train_steps  # invariant: both advance per learn step
        # the fused learner and the parity kernels gate themselves on the ring size; the GEMM
        # learner runs under the loop graph's IF node
        self.gated = agent.learner == "fused" and getattr(agent.net, "fused_act", False) and A + 1 <= 8
        self.desc.learn_gate = cfg.batch_size if self.gated else 0
        self.desc.early_sample = 1 if self.gated else 0
        if self.gated:  # the early sampler reads priorities ** alpha from a cache env.step / learn keep current
            self.desc.r_scaled = t["scaled"].data_ptr()
            self.desc.pstat = t["pstat"].data_ptr()
            self.desc.per_alpha = float(cfg.per_alpha)
        self._capture()

    # -- capture ---------------------------------------------------------------------------

    def _act(self):
        lib = _native.require_device()
        t, L = self.t, ctypes.byref(self.desc)
        net = self.agent.net
        if self.gated:
            # forward + epsilon-greedy decision in one launch (the host act's forward arithmetic);
            # it also closes the step once the budget is spent (the body runs several steps)
            Lh, dims, w_off, b_off = net.fused_layout()[:4]
            ws = net._fused_scratch(256, True)[0]
            # (its grid leaves an SM to the sampler; the few-row forward's barrier allows any grid)
            _native.check(lib.ap_parity_act_fused(L, Lh, dims, w_off, b_off, _native.ptr(net.flat),
                                                  _native.ptr(t["q"]), _native.ptr(ws), _native.ptr(t["act_bar"]),
                                                  _native.ptr(t["action"]), _stream()))
        else:
            q = net.forward_fused(t["state"]) if getattr(net, "fused_act", False) else net.forward_device(t["state"])
            _native.check(lib.ap_parity_act(L, _native.ptr(q), _native.ptr(t["action"]), _stream()))
            self._keep_q = q

    def _env_step(self):
        lib = _native.require_device()
        t, L = self.t, ctypes.byref(self.desc)
        self.env._engine.launch(t["seeds_try"][:, : self.n], t["outcome"], None, None, t["status"])
        _native.check(lib.ap_parity_post(L, _native.ptr(t["action"]), _stream()))

    def _sample(self, early: bool = False):
        lib = _native.require_device()
        cfg, t = self.agent.config, self.t
        st = self.agent.buffer.store
        _native.check(lib.ap_parity_sample(ctypes.byref(self.desc), cfg.batch_size, float(cfg.per_alpha),
                                           float(cfg.per_beta), _native.ptr(st["scratch"]), _native.ptr(t["idx"]),
                                           _native.ptr(t["weights"]), None,
                                           _native.ptr(t["rng_next"]) if early else None, int(early), _stream()))

    def _step_body(self):
        self._act()
        self._env_step()

    def _gated_body(self):
        """One step of the self-gated loop body: the PER sample of the step (early mode: the ring
        and random stream as the step starts, the act's draws replayed, the pending push counted)
        on a side branch beside act -> K1 -> env.step, then the learn step, which commits the
        sampler's stream state."""
        import torch

        cur = torch.cuda.current_stream()
        self.side.wait_stream(cur)
        with torch.cuda.stream(self.side):
            self._sample(early=True)
        self._act()
        self._env_step()
        cur.wait_stream(self.side)
        self._learn_body(sample=False)

    def _learn_body(self, sample: bool = True):
        lib = _native.require_device()
        agent, cfg, t = self.agent, self.agent.config, self.t
        L = ctypes.byref(self.desc)
        B = cfg.batch_size
        if sample:
            self._sample()
        opt, net = agent.optimizer, agent.net
        if agent.learner == "fused":
            # the learn tail (loss log, train counter) and the target sync run inside the kernel
            agent._fused.run(t["idx"], t["weights"], ctab=t["ctab"], ctl=t["ctl"], t_offset=self.adam_offset,
                             gate=B if self.gated else 0,
                             tail=(t["loss_log"], self.steps_cap, int(cfg.target_sync_every), self._sync_segments(),
                                   (t["rng_next"], t["rng"]) if self.gated else None),
                             scaled=t["scaled"] if self.gated else None, pstat=t["pstat"] if self.gated else None,
                             alpha=cfg.per_alpha, lazy_wt0=self.gated)
            return

        def adam_step():
            _native.check(lib.ap_dqn_adam_tab(_native.ptr(net.flat), _native.ptr(net.grad), _native.ptr(opt.m),
                                              _native.ptr(opt.v), net.flat.numel(), opt.lr, opt.beta1, opt.beta2,
                                              opt.eps, _native.ptr(t["ctab"]), _native.ptr(t["ctl"]),
                                              int(self.adam_offset), _stream()))
            net.refresh_transposed()

        loss = update_on_indices(net, agent.target, agent.buffer, cfg, t["idx"], t["weights"], agent._batch, adam_step)
        _native.check(lib.ap_parity_learn_tail(L, _native.ptr(loss), int(cfg.target_sync_every), _stream()))
        self._sync(lib)

    def _sync(self, lib):
        t = self.t
        segs = self._sync_segments()
        _native.check(lib.ap_parity_target_sync(_native.ptr(t["ctl"]), len(segs),
                                                (ctypes.c_void_p * len(segs))(*[s for s, _, _ in segs]),
                                                (ctypes.c_void_p * len(segs))(*[d for _, d, _ in segs]),
                                                (ctypes.c_int64 * len(segs))(*[c for _, _, c in segs]), _stream()))

    def _sync_segments(self):
        """(src, dst, count) of the online -> target copy: the flat parameters and every
        transposed copy (whole padded buffers), sync_target's result (agent.py:142-144).
        The self-gated loop's kernels read no transposed copy of the target (nor the online
        first layer's): those are refreshed once after each launch instead."""
        net, tgt = self.agent.net, self.agent.target
        segs = [(net.flat.data_ptr(), tgt.flat.data_ptr(), net.flat.numel())]
        if self.gated:
            return segs
        for k, w in net.wt.items():
            segs.append((w.data_ptr(), tgt.wt[k].data_ptr(), w.shape[0] * w.stride(0)))
        assert len(segs) <= 8
        return segs

    def _warm(self):
        """Lazily sized buffers (activation transposes, split-K workspaces, the learn batch)
        exist before the capture; touches only outputs and gradients, no search state."""
        import torch

        from .agent import FusedLearnState, _Batch

        agent, cfg = self.agent, self.agent.config
        if agent.learner == "fused" and agent._fused is None:
            agent._fused = FusedLearnState(agent.net, agent.target, agent.buffer, cfg, agent.optimizer)
        agent.net._fused_scratch(256, True)
        if agent._batch is None:
            agent._batch = _Batch(cfg.batch_size, agent.net.state_dim, agent.net.num_actions)
        b = agent._batch
        # K1's decision tables upload on first use (allocation + copy): not inside a capture
        t = self.t
        self.env._engine.launch(t["seeds_try"][:, : self.n], t["outcome"], None, None, t["status"])
        agent.net.forward_device(t["state"])
        agent.net.forward_device(b.next_states)
        agent.target.forward_device(b.next_states)
        _, acts = agent.net.forward_device(b.states, cache=True)
        agent.net.backward_device(acts, torch.zeros_like(b.dz))

    def _capture(self):
        import torch

        self.stream = torch.cuda.Stream()
        self.stream.wait_stream(torch.cuda.current_stream())
        import os

        pdl = os.environ.get("AP_NO_PDL")
        if not self.gated:
            os.environ["AP_NO_PDL"] = "1"  # plain edges inside the IF node's body
        import gc

        # no garbage collection inside the captures: a collected DeviceSearch of an earlier call
        # would destroy its CUDA graphs in the middle of this stream capture
        gc.collect()
        gc_was = gc.isenabled()
        gc.disable()
        try:
            with torch.cuda.stream(self.stream):
                self._warm()
                torch.cuda.current_stream().synchronize()
                self.g_step = torch.cuda.CUDAGraph(keep_graph=True)
                if self.gated:
                    # one body of _STEPS_PER_ITER steps; the learn kernels skip themselves while the
                    # ring holds fewer than a batch and every kernel after the act skips once the
                    # act found the budget spent (no IF node, one condition kernel per iteration)
                    self.side = torch.cuda.Stream()
                    with torch.cuda.graph(self.g_step, stream=self.stream):
                        for _ in range(_STEPS_PER_ITER):
                            self._gated_body()
                    self.g_learn = None
                else:
                    with torch.cuda.graph(self.g_step, stream=self.stream):
                        self._step_body()
                    self.g_learn = torch.cuda.CUDAGraph(keep_graph=True)
                    with torch.cuda.graph(self.g_learn, stream=self.stream):
                        self._learn_body()
        finally:
            if gc_was:
                gc.enable()
            if pdl is None:
                os.environ.pop("AP_NO_PDL", None)
            else:
                os.environ["AP_NO_PDL"] = pdl
        torch.cuda.current_stream().wait_stream(self.stream)
        h = ctypes.c_void_p()
        _native.check(_native.require_device().ap_loop_graph_create(
            ctypes.c_void_p(self.g_step.raw_cuda_graph()),
            ctypes.c_void_p(None if self.g_learn is None else self.g_learn.raw_cuda_graph()),
            _native.ptr(self.t["ctl"]), int(self.agent.config.batch_size), ctypes.byref(h)))
        self.loop = h

    def __del__(self):
        h = getattr(self, "loop", None)
        lib = getattr(_native, "_lib", None) if _native is not None else None
        if h is not None and lib is not None:
            try:
                lib.ap_loop_graph_destroy(h)
            except Exception:  # interpreter shutdown: the library may be half torn down
                pass

    # -- one launch -------------------------------------------------------------------------

    def launch(self, ctl_host: np.ndarray, ctab: np.ndarray) -> float:
        """One loop-graph launch (a block of episodes); returns its device time in ms."""
        import torch

        self.t["ctl"].copy_(torch.from_numpy(ctl_host))
        self.t["ctab"][: ctab.size].copy_(torch.from_numpy(ctab))
        if self.gated:  # the PER cache from the priorities as the host left them
            _native.check(_native.require_device().ap_per_scaled(
                _native.ptr(self.agent.buffer.store["priorities"]), int(ctl_host[_native.PL["SIZE"]]),
                float(self.agent.config.per_alpha), _native.ptr(self.t["scaled"]), _native.ptr(self.t["pstat"]),
                _native.stream_handle()))
        self.stream.wait_stream(torch.cuda.current_stream())
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(self.stream)
        _native.check(_native.require_device().ap_loop_graph_launch(self.loop, _native.stream_handle(self.stream)))
        e.record(self.stream)
        if self.gated:  # the transposed copies the loop left stale (outside the timed region)
            with torch.cuda.stream(self.stream):
                self.agent.net.refresh_transposed()
                self.agent.target.refresh_transposed()
        self.stream.synchronize()
        return s.elapsed_time(e)


def _rng_words(state: dict) -> np.ndarray:
    s = state["state"]["state"]
    inc = state["state"]["inc"]
    m = (1 << 64) - 1
    w = [(s >> 64) & m, s & m, (inc >> 64) & m, inc & m, int(state["has_uint32"]), int(state["uinteger"])]
    return np.array(w, dtype=np.uint64).view(np.int64)


def _rng_state(words: np.ndarray) -> dict:
    w = [int(x) for x in words.view(np.uint64)]
    return {"bit_generator": "PCG64", "state": {"state": (w[0] << 64) | w[1], "inc": (w[2] << 64) | w[3]},
            "has_uint32": int(w[4]), "uinteger": int(w[5])}


def _adam_table(t_first: int, count: int, beta1: float, beta2: float) -> np.ndarray:
    """fp32(1 - beta ** t) for t = t_first .. t_first + count - 1, the host agent's values
    (AdamOptimizer.step computes `1.0 - self.beta1 ** self.t` in fp64; ctypes rounds to fp32)."""
    t = np.arange(t_first, t_first + count, dtype=np.float64)
    out = np.empty((count, 2), dtype=np.float32)
    out[:, 0] = (1.0 - np.power(beta1, t)).astype(np.float32)
    out[:, 1] = (1.0 - np.power(beta2, t)).astype(np.float32)
    return out.reshape(-1)


def train_partition_device(env: PartitionSearchEnv, agent: DqnAgent, episodes: int, curve=None, trace=None,
                           finetune_base=None, episode_offset: int = 0, stop_when=None,
                           episodes_per_launch: int | None = None) -> PartitionOutcome | None:
    """`search.train_partition` with the whole loop on the device (see the module docstring)."""
    import torch

    if stop_when is not None:
        raise ValueError("train_partition_device: stop_when is a host callback; use search.train_partition")
    if episodes <= 0:
        return None
    if finetune_base is not None:
        env.finetune_reset(finetune_base)
        if env.done:  # nothing left to decide (cli.py:210-212)
            return None
    else:
        env.reset()
    n = len(env.dims)
    cfg = agent.config
    log_rows = trace is not None
    per_launch = episodes_per_launch or episodes
    if log_rows:
        per_launch = max(1, min(per_launch, _LOG_BYTES // max(1, n * pad16(n))))
    per_launch = min(per_launch, episodes)
    steps_cap = per_launch * n  # every non-conflicting step decides >= 1 dim; a conflict ends the episode
    ds = DeviceSearch(env, agent, steps_cap, log_rows)
    t = ds.t
    # device state from the host objects
    t["rng"].copy_(torch.from_numpy(_rng_words(agent.rng.bit_generator.state)))
    for key, vec in (("seeds", env._seed_vec), ("t_seeds", env._seed_vec), ("decided", env._status),
                     ("t_decided", env._status)):
        t[key][:n].copy_(torch.from_numpy(np.asarray(vec, dtype=np.int8)))
    state0 = env._state()
    t["state"][0].copy_(torch.from_numpy(state0.astype(np.float32)))
    pos0 = -1 if env._position is None else int(env._position)
    W = _native.PL
    ctl = np.zeros(W["WORDS"], dtype=np.int64)
    ctl[W["SLOT"]], ctl[W["SIZE"]], ctl[W["TRAIN"]] = agent.buffer._next, len(agent.buffer), agent.train_steps
    ctl[W["POS"]] = ctl[W["T_POS"]] = pos0
    ctl[W["BEST_PART"]] = ctl[W["BEST_EP"]] = ctl[W["LOSS_BAD"]] = -1
    ctl[W["MAX_STEPS"]] = steps_cap
    B = cfg.batch_size
    done_eps = 0
    losses_all: list[float] = []
    last_stats.clear()
    last_stats.update(device_ms=0.0, steps=0, launches=0, train_steps=0)
    while done_eps < episodes:
        budget = min(per_launch, episodes - done_eps)
        ctl[W["STEP"]] = 0
        ctl[W["EPISODES"]] = 0
        ctl[W["BUDGET"]] = budget
        ctl[W["EP_STEPS"]] = 0
        ctl[W["EP_BASE"]] = done_eps
        ctl[W["TRAIN0"]] = ctl[W["TRAIN"]]
        ctl[W["TAB_BASE"]] = ctl[W["TRAIN"]] + ds.adam_offset  # table entry 0 = Adam step TAB_BASE + 1
        size0, train0 = int(ctl[W["SIZE"]]), int(ctl[W["TRAIN"]])
        ms = ds.launch(ctl, _adam_table(int(ctl[W["TAB_BASE"]]) + 1, steps_cap, agent.optimizer.beta1,
                                        agent.optimizer.beta2))
        ctl = t["ctl"].cpu().numpy().copy()
        last_stats["device_ms"] += ms
        last_stats["steps"] += int(ctl[W["STEP"]])
        last_stats["launches"] += 1
        last_stats["train_steps"] += int(ctl[W["TRAIN"]]) - train0
        if ctl[W["FAULT"]]:
            raise RuntimeError("device loop: the act gave up waiting for the step's PER sample")
        if ctl[W["LOSS_BAD"]] >= 0:
            raise DivergenceError("training loss diverged on the device loop")
        steps = int(ctl[W["STEP"]])
        eps_n = int(ctl[W["EPISODES"]])
        if eps_n != budget:
            raise RuntimeError(f"device loop stopped after {eps_n} of {budget} episodes ({steps} steps)")
        acts = t["log_action"][:steps].cpu().numpy()
        rews = t["log_reward"][:steps].cpu().numpy()
        lens = t["ep_len"][:eps_n].cpu().numpy()
        confl = t["ep_conflict"][:eps_n].cpu().numpy()
        rets = t["ep_return"][:eps_n].cpu().numpy()
        n_train = int(ctl[W["TRAIN"]]) - train0
        loss_log = t["loss_log"][:n_train].double().cpu().numpy() / B
        rows = t["log_decided"][:steps, :n].cpu().numpy() if log_rows else None
        pos = t["log_pos"][:steps].cpu().numpy() if log_rows else None
        # per-step learn flags: step i learns once the ring holds a batch after its push
        learned = np.minimum(size0 + np.arange(1, steps + 1), agent.buffer.capacity) >= B
        k = 0
        li = 0
        for e in range(eps_n):
            L_e = int(lens[e])
            ep_losses = []
            steps_rec = []
            for i in range(k, k + L_e):
                if learned[i]:
                    ep_losses.append(float(loss_log[li]))
                    li += 1
                if log_rows:
                    vec = np.empty(n + 1, dtype=np.float64)
                    vec[:n] = rows[i]
                    vec[n] = pos[i] / n
                    steps_rec.append({"state_digest": state_digest(vec), "action": int(acts[i]),
                                      "reward": float(rews[i])})
            k += L_e
            ep_id = episode_offset + done_eps + e
            if curve is not None:
                mean_loss = sum(ep_losses) / len(ep_losses) if ep_losses else None
                # epsilon after the episode's last learn step (cli.py:241-243)
                train_after = train0 + sum(int(x) for x in learned[:k])
                curve.write(ep_id, mean_loss, float(rets[e]), epsilon_at(train_after, cfg))
            if trace is not None:
                trace.write(ep_id, steps_rec, "conflict" if confl[e] else "complete")
            losses_all += ep_losses
        done_eps += eps_n
    # leave the host objects as the host loop would
    agent.rng.bit_generator.state = _rng_state(t["rng"].cpu().numpy())
    agent.train_steps = int(ctl[W["TRAIN"]])
    agent.optimizer.t = agent.train_steps + ds.adam_offset
    agent.buffer._size = int(ctl[W["SIZE"]])
    agent.buffer._next = int(ctl[W["SLOT"]])
    env._done = True
    if ctl[W["BEST_PART"]] < 0:
        return None
    row = t["best_row"][:n].cpu().numpy()
    strategy = {env.dims[j]: DimStatus(int(row[j])) for j in range(n)}
    return PartitionOutcome(strategy, int(ctl[W["BEST_PART"]]), float(t["dctl"][1].item()),
                            episode_offset + int(ctl[W["BEST_EP"]]))
