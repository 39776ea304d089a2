"""The reference-semantics device search loop on BERT-48 OPP (bench's dqn single-env config).

    python profiles/probes/devloop_one.py [EPISODES] [--trace]

Prints device env-steps/s of one loop-graph launch over EPISODES episodes (after a
2-episode fill).  Under ncu (`--graph-profiling node`, the default) each kernel node of
the loop graph appears in the launch list, which gives the per-step kernel breakdown.
"""

import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_2007_04069_b200 import devloop  # noqa: E402
from paper_2007_04069_b200.agent import AgentConfig, DqnAgent  # noqa: E402
from paper_2007_04069_b200.envs import OppEnv  # noqa: E402
from paper_2007_04069_b200.linkage import extract_linkage_groups  # noqa: E402


def main():
    episodes = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 20
    g, dims = bench.workload_setup("bert48", "opp")
    groups = extract_linkage_groups(g, dims)
    env = OppEnv(g, groups=groups)
    cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=2000)
    agent = DqnAgent(cfg, env.state_dim, env.num_actions, 0)
    devloop.train_partition_device(env, agent, 2)
    t0 = time.perf_counter()
    best = devloop.train_partition_device(env, agent, episodes)
    wall = time.perf_counter() - t0
    st = dict(devloop.last_stats)
    st["steps_per_s_device"] = st["steps"] / (st["device_ms"] / 1e3)
    st["wall_s"] = wall
    st["best"] = None if best is None else best.partitions
    print(json.dumps(st))


if __name__ == "__main__" and "--eager" not in sys.argv and "--pieces" not in sys.argv:
    main()


def eager(steps: int):
    """The loop body's kernels launched eagerly for `steps` steps (per-kernel durations under ncu:
    conditional graph nodes are not profiled individually)."""
    import torch

    g, dims = bench.workload_setup("bert48", "opp")
    groups = extract_linkage_groups(g, dims)
    env = OppEnv(g, groups=groups)
    cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=2000)
    agent = DqnAgent(cfg, env.state_dim, env.num_actions, 0)
    devloop.train_partition_device(env, agent, 2)

    def fake_launch(self, ctl_host, ctab):
        self.t["ctl"].copy_(torch.from_numpy(ctl_host))
        self.t["ctab"][: ctab.size].copy_(torch.from_numpy(ctab))
        with torch.cuda.stream(self.stream):
            for _ in range(steps):
                self._step_body()
                self._learn_body()
        self.stream.synchronize()
        return 1.0

    devloop.DeviceSearch.launch = fake_launch
    try:
        devloop.train_partition_device(env, agent, 1)
    except RuntimeError as exc:
        print("eager stop:", exc)


if __name__ == "__main__" and "--eager" in sys.argv:
    eager(int(sys.argv[sys.argv.index("--eager") + 1]))


def pieces(reps: int = 20, fill: int = 15):
    """Warm in-graph time of each loop-body kernel: a CUDA graph of `reps` back-to-back launches
    of one piece (act, K1, post, sample, learn) or of the whole body, replayed; the control block
    is restored before each replay."""
    import ctypes

    import torch

    from paper_2007_04069_b200 import _native

    g, dims = bench.workload_setup("bert48", "opp")
    env = OppEnv(g, groups=extract_linkage_groups(g, dims))
    cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=2000)
    agent = DqnAgent(cfg, env.state_dim, env.num_actions, 0)
    devloop.train_partition_device(env, agent, fill)  # 15 episodes: a full ring (2,000 rows)
    out = {"ring_rows": len(agent.buffer)}

    def fake_launch(self, ctl_host, ctab):
        lib = _native.require_device()
        t, L = self.t, ctypes.byref(self.desc)
        net = self.agent.net
        Lh, dmz, w_off, b_off = net.fused_layout()[:4]
        ws, bar = net._fused_scratch(256, True)
        st = self.agent.buffer.store
        B = cfg.batch_size
        S = lambda: _native.stream_handle(self.stream)  # noqa: E731

        def act():  # (without the early sampler: the act would wait for its acknowledgement)
            self.desc.early_sample = 0  # full grid: the forward's own barrier
            _native.check(lib.ap_parity_act_fused(L, Lh, dmz, w_off, b_off, _native.ptr(net.flat), _native.ptr(t["q"]),
                                                  _native.ptr(ws), _native.ptr(bar), _native.ptr(t["action"]), S()))
            self.desc.early_sample = 1

        def k1():
            self.env._engine.launch(t["seeds_try"][:, : self.n], t["outcome"], None, None, t["status"],
                                    stream=self.stream)

        def post():
            _native.check(lib.ap_parity_post(L, _native.ptr(t["action"]), S()))

        def sample():
            with torch.cuda.stream(self.stream):
                self._sample(early=True)

        def learn():
            self.agent._fused.run(t["idx"], t["weights"], ctab=t["ctab"], ctl=t["ctl"], t_offset=self.adam_offset,
                                  gate=B, tail=(t["loss_log"], self.steps_cap, int(cfg.target_sync_every),
                                                self._sync_segments()))

        def body():
            self._gated_body()

        ctl0 = torch.from_numpy(ctl_host.copy())
        self.t["ctab"][: ctab.size].copy_(torch.from_numpy(ctab))
        def body_nopdl():
            os.environ["AP_NO_PDL"] = "1"
            try:
                self._gated_body()
            finally:
                os.environ.pop("AP_NO_PDL")

        for name, fn in (("act_fused", act), ("k1_one_row", k1), ("post", post), ("sample", sample),
                         ("learn", learn), ("body", body), ("body_nopdl", body_nopdl)):
            self.t["ctl"].copy_(ctl0)
            torch.cuda.synchronize()
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=self.stream):
                for _ in range(reps):
                    fn()
            ms = []
            for _ in range(6):
                self.t["ctl"].copy_(ctl0)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(self.stream):
                    e0.record(self.stream)
                    gr.replay()
                    e1.record(self.stream)
                self.stream.synchronize()
                ms.append(e0.elapsed_time(e1))
            out[name] = round(sorted(ms[1:])[len(ms[1:]) // 2] * 1e3 / reps, 2)
        lib = _native.load_library()
        if hasattr(lib, "ap_debug_sample_trace"):  # AP_LIB_PATH build with -DAP_SAMPLE_TRACE
            tr = (ctypes.c_ulonglong * 16)()
            lib.ap_debug_sample_trace(tr)
            seq = [0, 1, 4, 2, 6, 7, 3]  # start, staged, blocks, total, probs, cumsum, draws+weights
            out["sample_stage_cycles"] = [int(tr[seq[k + 1]] - tr[seq[k]]) for k in range(len(seq) - 1)]
        print(json.dumps({"us_per_launch_in_graph": out}))
        raise SystemExit(0)

    devloop.DeviceSearch.launch = fake_launch
    devloop.train_partition_device(env, agent, 1)


if __name__ == "__main__" and "--pieces" in sys.argv:
    pieces()
