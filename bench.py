#!/usr/bin/env python
"""Benchmark: candidate plans evaluated / s on the Auto-MAP plan-exploration hot path.

One step = one pass of the batched propagation kernel (K1) over one batch of
synthetic plans (random decision-order prefixes, `workloads.py`) on the
BERT-48 HLO graph: for every plan the full fixed point (all |S| slot
statuses), outcome and decided / newly counts (SURVEY §8(d) "full
contract").  Per-GPU work is fixed as N grows (weak scaling); plans are
sharded by global index, no collective on the data path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank runs its shard; the device time is the max over
ranks.  `--impl reference` times the reference planner's own CPU
implementation (baseline/_ref, all host cores) on a bounded sample of the
same workload; rank 0 alone runs it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "candidate plans evaluated/sec and DQN env-steps/sec at 1/2/4/8 B200"
UNIT = "plans/s"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=300)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default="bert48")
    p.add_argument("--batch", type=int, default=1 << 22, help="plans per GPU per step")
    p.add_argument("--e2e-batch", type=int, default=1 << 18)
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--cpu-seconds", type=float, default=15.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-secondary", action="store_true", help="skip the DQN / PP-train / PP-infer figures")
    p.add_argument("--dqn-envs", type=int, default=4096)
    p.add_argument("--dqn-learn-steps", type=int, default=4)
    p.add_argument("--dqn-steps", type=int, default=30)
    p.add_argument("--dqn-eager", action="store_true", help="launch the vector step eagerly (no CUDA graph)")
    p.add_argument("--pp-envs", type=int, default=512, help="PP-train env states evaluated per launch")
    p.add_argument("--pp-dqn-envs", type=int, default=1024, help="vectorised PP-train DQN envs per GPU")
    p.add_argument("--single-steps", type=int, default=300)
    return p.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def workload_setup(name: str):
    from paper_2007_04069_b200 import graphs
    from paper_2007_04069_b200.ir import decision_dims

    g = graphs.generate(name)
    dims = decision_dims(g, g.trainable_variables)
    return g, dims


def workload_config(name, g, dims, batch, extra=None):
    cfg = {
        "workload": f"{name} OPP propagation, full contract (all slot statuses + outcome + counts)",
        "graph": name,
        "instructions": len(g),
        "slots": int(g.flat().num_slots),
        "candidate_dims": len(dims),
        "plans_per_gpu_per_step": batch,
        "plan_batch": "decision-order prefixes k~U[1,|D|], fair P/R coins (workloads.prefix_seed_batch, seed 20201007)",
        "l2": "inputs larger than L2 (seeds + slot outputs per step >> 126 MB)",
    }
    if extra:
        cfg.update(extra)
    return cfg


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except OSError:
            self.proc = None
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sms, maxes, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sms.append(float(parts[0]))
                maxes.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {
            "sm_mhz": statistics.median(sms) if sms else None,
            "sm_max_mhz": max(maxes) if maxes else None,
            "reasons": sorted(reasons),
            "samples": len(sms),
        }


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel: str):
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    data = json.loads(p.read_text())
    k = data.get("kernels", {}).get(kernel)
    return None if k is None else k.get("dram_bytes_per_plan")


# -- CPU baselines (reference planner) ----------------------------------------------


def _ref_import():
    ref = ROOT / "baseline" / "_ref"
    if ref.exists() and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import autoplan  # noqa: F401
    from autoplan import ir as rir
    from autoplan import sharding as rsh

    return rir, rsh


_W = {}


def _ref_worker_init(graph_json, dims_raw):
    rir, rsh = _ref_import()
    g = rir.graph_from_dict(json.loads(graph_json))
    dims = [rir.DimIndex(*d) for d in dims_raw]
    _W["eng"] = rsh.PropagationEngine(g, dims)
    _W["dims"] = dims
    _W["vals"] = {0: rsh.DimStatus.REPLICATED, 1: rsh.DimStatus.PARTITIONED}


def _ref_eval_rows(rows):
    eng, dims, vals = _W["eng"], _W["dims"], _W["vals"]
    for row in rows:
        eng.run({dims[j]: vals[int(v)] for j, v in enumerate(row) if v != -1})
    return len(rows)


def cpu_baseline_single(g, dims, order, seconds: float):
    """The reference engine (reused, one core) on the first rows of the same batch."""
    from paper_2007_04069_b200.distributed import plan_shard
    from paper_2007_04069_b200.workloads import prefix_seed_batch

    dims_raw = [(d.flat_index, d.instruction_id, d.dim) for d in dims]
    sample = prefix_seed_batch(order, 0, 4096).numpy()
    try:
        _ref_worker_init(json.dumps(g.to_dict()), dims_raw)
        kind = "reference"
        done, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < seconds and done < len(sample):
            _ref_eval_rows(sample[done:done + 1])
            done += 1
        dt = time.perf_counter() - t0
    except ImportError:
        from oracle import oracle  # the port, only if the reference is not installed

        kind = "port"
        flat = g.flat()
        cand = [int(flat.slot_offset[d.instruction_id] + d.dim) for d in dims]
        done, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < seconds and done < len(sample):
            oracle.propagate_batch(flat, cand, sample[done:done + 64], cand)
            done += 64
        dt = time.perf_counter() - t0
    return {
        "value": done / dt,
        "unit": UNIT,
        "cores": 1,
        "kind": kind,
        "sample": f"first {done} plans of the same batch, "
                  + ("PropagationEngine(graph, dims).run per plan, engine reused, " if kind == "reference"
                     else "C oracle port (baseline/_ref not installed), 64-plan batches, ")
                  + f"{dt:.2f} s on 1 host core",
    }


def run_reference_arm(args):
    import multiprocessing as mp

    rank, world, _ = env_rank()
    if rank != 0:
        return
    g, dims = workload_setup(args.workload)
    from paper_2007_04069_b200.distributed import plan_shard
    from paper_2007_04069_b200.workloads import prefix_seed_batch

    # decision order from the reference's own linkage would take minutes at this
    # size; the batch only needs a fixed column order, so use the same one as
    # our arm (written next to the graph by a previous run) or the flat order
    order = _cached_order(args.workload, len(dims))
    cores = os.cpu_count() or 1
    per_worker = 1
    total_rows = (args.steps + args.warmup) * cores * per_worker
    sample = prefix_seed_batch(order, 0, total_rows).numpy()
    dims_raw = [(d.flat_index, d.instruction_id, d.dim) for d in dims]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_ref_worker_init, initargs=(json.dumps(g.to_dict()), dims_raw)) as pool:
        step_t = []
        cursor = 0
        for step in range(args.warmup + args.steps):
            chunks = [sample[cursor + w * per_worker: cursor + (w + 1) * per_worker] for w in range(cores)]
            cursor += cores * per_worker
            t0 = time.perf_counter()
            pool.map(_ref_eval_rows, chunks, chunksize=1)
            if step >= args.warmup:
                step_t.append(time.perf_counter() - t0)
    total = sum(step_t)
    value = args.steps * cores * per_worker / total
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int8",
        "data": "synthetic",
        "config": workload_config(args.workload, g, dims, cores * per_worker),
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": cores,
            "kind": "reference",
            "sample": f"{cores * per_worker} plans per step (one per worker process), reference "
                      f"PropagationEngine.run, engine reused, multiprocessing pool of {cores}",
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _cached_order(workload, n):
    import numpy as np

    p = ROOT / "profiles" / f"order_{workload}.json"
    if p.exists():
        order = json.loads(p.read_text())
        if len(order) == n:
            return np.asarray(order, dtype=np.int64)
    return np.arange(n, dtype=np.int64)


# -- our arm -------------------------------------------------------------------------


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2007_04069_b200.linkage import extract_linkage_groups, sorted_decision_order
    from paper_2007_04069_b200.sharding import PropagationEngine
    from paper_2007_04069_b200.distributed import plan_shard
    from paper_2007_04069_b200.workloads import prefix_seed_batch

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    g, dims = workload_setup(args.workload)
    n = len(dims)
    S = g.flat().num_slots
    eng = PropagationEngine(g, dims)

    # decision order from the linkage groups (one batched launch of 2|D| triggers)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    groups = extract_linkage_groups(g, dims)
    order = np.asarray([d.flat_index for d in sorted_decision_order(groups)], dtype=np.int64)
    linkage_s = time.perf_counter() - t0
    if rank == 0:
        (ROOT / "profiles").mkdir(exist_ok=True)
        (ROOT / "profiles" / f"order_{args.workload}.json").write_text(json.dumps(order.tolist()))

    B = args.batch
    seeds = prefix_seed_batch(order, *plan_shard(rank, B), device="cuda", chunk=1 << 18)
    stride = eng.slots_stride
    slots = torch.empty((B, stride), dtype=torch.int8, device="cuda")
    outcome = torch.empty(B, dtype=torch.uint8, device="cuda")
    counts = torch.empty((B, 4), dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        eng.launch(seeds, outcome, counts, slots, stream=stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for _ in range(args.steps):
        eng.launch(seeds, outcome, counts, slots, stream=stream)
    end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clock_info = clocks.stop()
    elapsed_ms = start.elapsed_time(end)
    max_ms = _max_over_ranks(elapsed_ms, world)
    conflict_rate = float((outcome == 2).float().mean().item())

    # e2e through the host-buffer API: pinned H2D + kernel + D2H every step
    Be = args.e2e_batch
    seeds_host = prefix_seed_batch(order, *plan_shard(rank, Be), device="cuda").cpu().pin_memory()
    out_host = None
    for _ in range(2):
        out_host = eng.run_batch_host(seeds_host, out=out_host)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        out_host = eng.run_batch_host(seeds_host, out=out_host)
    e2e_s = time.perf_counter() - t0
    e2e_s = _max_over_ranks(e2e_s, world)
    # the same host API with 2-bit packed slot rows (ap_pack_slots2): a quarter of the slot D2H
    out_pk = None
    for _ in range(2):
        out_pk = eng.run_batch_host(seeds_host, want_slots="packed", out=out_pk)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        out_pk = eng.run_batch_host(seeds_host, want_slots="packed", out=out_pk)
    e2e_pk_s = _max_over_ranks(time.perf_counter() - t0, world)
    e2e_packed = {
        "value": world * Be * args.e2e_steps / e2e_pk_s,
        "unit": UNIT,
        "h2d_bytes_per_step": Be * n,
        "d2h_bytes_per_step": Be * (eng.packed_slots_stride + 1 + 16),
        "api": 'PropagationEngine.run_batch_host(want_slots="packed") (K1 + ap_pack_slots2, 2-bit slot rows to host)',
    }
    del out_pk

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_single(g, dims, order, args.cpu_seconds)

    secondary = {"e2e_packed_slots": e2e_packed}
    if not args.no_secondary:
        want_cpu = rank == 0 and world == 1 and not args.no_cpu_baseline
        secondary["dqn_env_steps_per_s"] = bench_dqn_vec(args, g, world, rank)
        secondary["dqn_env_steps_per_s_pp_train"] = bench_dqn_pipe(args, g, world, rank)
        secondary["dqn_env_steps_per_s_pp_infer"] = bench_dqn_infer(args, world, rank)
        secondary["pp_train_candidates_per_s"] = bench_pp_train(args, world, want_cpu)
        secondary["pp_infer_points_per_s"] = bench_pp_infer(args, world, want_cpu)
        secondary["pp_infer_envs_generated_per_s"] = bench_env_gen(args, world, rank, want_cpu)
        if rank == 0 and world == 1:
            secondary["dqn_env_steps_per_s_single_env"] = bench_dqn_single(args, g, dims, groups, want_cpu)

    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return
    per_launch_s = max_ms / 1e3 / args.steps
    bytes_per_plan = n + S + 1 + 16
    achieved = B * bytes_per_plan / per_launch_s / 1e9
    peak, peak_src = measured_peak_hbm()
    traffic_per_plan = ncu_traffic("propagate_kernel")
    traffic = None if traffic_per_plan is None else traffic_per_plan * B
    value = world * B * args.steps / (max_ms / 1e3)
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": max_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int8",
        "data": "synthetic",
        "config": workload_config(args.workload, g, dims, B, {
            "parallelism": f"plan-sharded x{world} (no data-path collective)",
            "conflict_rate": round(conflict_rate, 4),
            "linkage_s": round(linkage_s, 4),
        }),
        "roofline": {
            "bound": "hbm",
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": traffic,
            "bytes_per_plan": bytes_per_plan,
            "peak_source": peak_src,
            "kernel": "apb::propagate_fast_kernel (K1)",
            "traffic_source": "profiles/ncu_summary.json dram bytes/plan x plans per launch (ncu --set full)",
        },
        "cpu_baseline": cpu,
        "e2e": {
            "value": world * Be * args.e2e_steps / e2e_s,
            "unit": UNIT,
            "h2d_bytes_per_step": Be * n,
            "d2h_bytes_per_step": Be * (stride + 1 + 16),
            "api": "PropagationEngine.run_batch_host (pinned host seeds -> host outcome/counts/slots)",
        },
        "gpu_launches": args.steps,
        "clocks": clock_info,
        "secondary": secondary,
    }
    print(json.dumps(line), flush=True)


# -- secondary metrics (DQN env-steps/s, PP-train and PP-infer plan evaluation) ----------


def _max_over_ranks(x: float, world: int) -> float:
    from paper_2007_04069_b200.distributed import max_over_ranks

    return max_over_ranks(x) if world > 1 else float(x)


def bench_dqn_pipe(args, g, world, rank):
    """Throughput-mode DQN on PP-train (BERT-48, 2x4, K=4): E VecPipeTrainEnv episodes per GPU, each vector
    step = act (state 4C wide) + pick + terminal metrics / length + K2 next states + L learn steps."""
    import torch
    import torch.distributed as dist

    from paper_2007_04069_b200.agent import AgentConfig
    from paper_2007_04069_b200.topology import DeviceTopology
    from paper_2007_04069_b200.vec import VecDqnTrainer, VecPipeTrainEnv

    E, L = args.pp_dqn_envs, args.dqn_learn_steps
    env = VecPipeTrainEnv(g, DeviceTopology(2, 4), 4, E)
    cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=2000)
    pg = dist.group.WORLD if world > 1 else None
    tr = VecDqnTrainer(env, cfg, capacity=4 * E, seed=rank, learn_steps=L, process_group=pg, use_graph=True)
    for _ in range(5):
        tr.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.dqn_steps):
        tr.step()
    e.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), world)
    best = tr.best_plan_global()
    return {
        "value": world * E * args.dqn_steps / (ms / 1e3),
        "unit": "env-steps/s",
        "config": {"graph": "bert48", "task": "pp-train", "topology": "2x4", "stages": 4, "radius": 3,
                   "candidates": env.C, "state_dim": env.state_dim, "envs_per_gpu": E,
                   "learn_steps_per_vector_step": L, "learn_batch": cfg.batch_size,
                   "learn_to_env_step_ratio": f"{L}:{E}", "hidden": list(cfg.hidden), "replay_capacity": tr.capacity,
                   "vector_steps": args.dqn_steps, "cuda_graph": tr.graph is not None},
        "ms_per_vector_step": ms / args.dqn_steps,
        "episodes_finished_rank0": int(env.episodes_done.sum().item()),
        "best_plan": None if best is None else {"pipeline_length": -best.reward, "global_episode": best.episode},
        "reference_note": "reference PipeTrainEnv._state takes seconds per state on the host (pp_train_candidates_per_s "
                          "cpu_baseline), i.e. < 1 env-step/s",
    }


def bench_dqn_infer(args, world, rank):
    """Throughput-mode DQN on PP-infer (configC, K=4, banded as in the paper's search): E VecPipeInferEnv
    episodes per GPU, each vector step = act + pick + batched terminal lengths + L learn steps."""
    import torch
    import torch.distributed as dist

    from paper_2007_04069_b200.agent import AgentConfig
    from paper_2007_04069_b200.dataproc import generate_environment
    from paper_2007_04069_b200.envs import infer_search_bands
    from paper_2007_04069_b200.topology import PRESETS
    from paper_2007_04069_b200.vec import VecDqnTrainer, VecPipeInferEnv

    E, L = args.dqn_envs, args.dqn_learn_steps
    arrays = generate_environment("uniform", 1280, 0)
    topo = PRESETS["configc"]
    bb, cc = infer_search_bands(arrays, topo, 4, 3)
    env = VecPipeInferEnv(arrays, topo, 4, E, allowed_boundaries=bb, allowed_cuts=cc)
    cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=2000)
    pg = dist.group.WORLD if world > 1 else None
    tr = VecDqnTrainer(env, cfg, capacity=max(4 * E, 4096), seed=rank, learn_steps=L, process_group=pg,
                       use_graph=True)
    for _ in range(5):
        tr.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(args.dqn_steps):
        tr.step()
    e.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), world)
    best = tr.best_plan_global()
    return {
        "value": world * E * args.dqn_steps / (ms / 1e3),
        "unit": "env-steps/s",
        "config": {"profile": "generate_environment(uniform, 1280, 0)", "topology": "configc", "stages": 4,
                   "bands": "infer_search_bands(radius 3)", "state_dim": env.state_dim, "actions": env.num_actions,
                   "envs_per_gpu": E, "learn_steps_per_vector_step": L, "learn_batch": cfg.batch_size,
                   "learn_to_env_step_ratio": f"{L}:{E}", "hidden": list(cfg.hidden), "vector_steps": args.dqn_steps,
                   "cuda_graph": tr.graph is not None},
        "ms_per_vector_step": ms / args.dqn_steps,
        "episodes_finished_rank0": int(env.episodes_done.sum().item()),
        "best_plan": None if best is None else {"pipeline_length": -best.reward, "global_episode": best.episode},
    }


def bench_dqn_vec(args, g, world, rank):
    """Throughput-mode DQN: E envs per GPU, batched act / step / observe, L learn steps (batch 64) per vector step."""
    import torch
    import torch.distributed as dist

    from paper_2007_04069_b200.agent import AgentConfig
    from paper_2007_04069_b200.vec import VecDqnTrainer, VecPartitionEnv

    E, L = args.dqn_envs, args.dqn_learn_steps
    env = VecPartitionEnv(g, E)
    cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=2000)
    pg = dist.group.WORLD if world > 1 else None
    tr = VecDqnTrainer(env, cfg, capacity=max(4 * E, 4096), seed=rank, learn_steps=L, process_group=pg,
                       use_graph=not args.dqn_eager)
    for _ in range(5):
        tr.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = tr.launches
    s.record()
    for _ in range(args.dqn_steps):
        tr.step()
    e.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), world)
    # tensor-pipe figure for the batched act forward (the dominant GEMMs)
    # (10 forwards captured in a CUDA graph: the kernels, not the Python launch path)
    x = env.cur_state
    for _ in range(3):
        tr.net.forward_device(x)
    torch.cuda.synchronize()
    fwd_graph = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        with torch.cuda.graph(fwd_graph, stream=side):
            for _ in range(10):
                tr.net.forward_device(x)
    torch.cuda.current_stream().wait_stream(side)
    fwd_graph.replay()
    torch.cuda.synchronize()
    s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2.record()
    fwd_graph.replay()
    e2.record()
    torch.cuda.synchronize()
    fwd_s = s2.elapsed_time(e2) / 1e3 / 10
    S, H = env.state_dim, cfg.hidden[0]
    flops = 2.0 * E * (S * H + H * H + H * 3)  # algorithmic (one pass; precision 3 would run three)
    best = tr.best_plan_global()  # all-gather of every rank's incumbent, first-wins by global episode id
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    tf32_peak = peaks.get("bf16_tflops", 1590.0) / 2.0
    return {
        "value": world * E * args.dqn_steps / (ms / 1e3),
        "unit": "env-steps/s",
        "config": {"graph": "bert48", "task": "opp", "envs_per_gpu": E, "learn_steps_per_vector_step": L,
                   "learn_batch": cfg.batch_size, "learn_to_env_step_ratio": f"{L}:{E}",
                   "hidden": list(cfg.hidden), "state_dim": S, "replay_capacity": tr.capacity,
                   "parallelism": (f"data-parallel DQN x{world}, " + ("Q-gradient all-reduce over NVLink peer memory fused "
                                   "with Adam (ap_dp_allreduce_adam)" if tr.peer is not None else
                                   "NCCL all-reduce of Q-gradients")) if world > 1 else "1 GPU",
                   "vector_steps": args.dqn_steps},
        "ms_per_vector_step": ms / args.dqn_steps,
        "cuda_graph": tr.graph is not None,
        "episodes_finished_rank0": int(env.episodes_done.sum().item()),
        "envs_with_completed_episode_rank0": int((env.best_episode >= 0).sum().item()),
        "best_plan": None if best is None else {"partitions": best.partitions, "return": best.reward,
                                                "global_episode": best.episode},
        "gpu_launches_per_vector_step": (tr.launches - launches0) / args.dqn_steps,
        "act_forward_tensor": {"bound": "tensor", "achieved": flops / fwd_s / 1e12, "unit": "TFLOP/s",
                               "peak": tf32_peak, "peak_source": "half of measured bf16 (dense TF32 = bf16/2)",
                               "frac": flops / fwd_s / 1e12 / tf32_peak, "gemm_m": E,
                               "note": f"3 GEMMs M=E K=state_dim/256 N=256/3, tcgen05 kind::tf32, "
                                       f"precision={tr.net.precision} (1 = TF32, 3 = 3xTF32)"},
    }




def bench_pp_train(args, world, want_cpu):
    """PP-train candidate plans/s: PipeTrainEnv._state over all allowed pivots of E random partial plans."""
    import ctypes

    import numpy as np
    import torch

    from paper_2007_04069_b200 import _native
    from paper_2007_04069_b200.envs import PipeTrainEnv
    from paper_2007_04069_b200.topology import DeviceTopology

    g, _ = workload_setup(args.workload)
    topo = DeviceTopology(2, 4)
    K = 4
    env = PipeTrainEnv(g, topo, K, radius=3)
    C = env.num_actions
    E = args.pp_envs
    rng = np.random.default_rng(7)
    applied = np.full((E, K - 2), -1, dtype=np.int32)
    mask = np.zeros((E, C), dtype=np.uint8)
    for e in range(E):
        k = int(rng.integers(0, K - 1))  # 0..K-2 picks so far
        picks = np.sort(rng.choice(C - (K - 1), size=k, replace=False)) if k else np.zeros(0, int)
        applied[e, :k] = picks
        last = picks[-1] if k else -1
        remaining = (K - 1) - k
        mask[e, last + 1: C - remaining + 1] = 1
    d_cand = torch.from_numpy(env._cand_pos).cuda()
    env._model.bind_candidates(d_cand)  # the table build is per env, outside the timed region
    d_app = torch.from_numpy(applied).cuda()
    d_mask = torch.from_numpy(mask).cuda()
    state = torch.empty((E, 4 * C), dtype=torch.float64, device="cuda")
    lib = _native.require_device()
    topo_c = _native.Topology.of(topo)

    def run():
        _native.check(lib.ap_pipe_train_state(env._model.handle, ctypes.byref(topo_c), _native.ptr(d_cand), C,
                                              _native.ptr(d_app), K - 2, _native.ptr(d_mask), E, 2.0,
                                              _native.ptr(state), _native.stream_handle()))

    for _ in range(2):
        run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 5
    s.record()
    for _ in range(iters):
        run()
    e.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), world)
    evaluated = int(mask.sum())
    F = env._model.num_forward
    cand_per_s = evaluated * iters / (ms / 1e3)  # per GPU
    out = {"value": world * cand_per_s, "unit": "candidate plans/s",
           "config": {"graph": args.workload, "topology": "2x4", "stages": K, "radius": 3, "candidates": C,
                      "env_states_per_launch": E, "allowed_candidates_per_launch": evaluated,
                      "forward_instructions": F, "stage_sums": "bound stage-sum table (ap_pipe_train_table)"},
           "ms_per_launch": ms / iters,
           # the reference re-sums N_f costs per candidate (SURVEY §8(d)'s fp64-add bound); the bound table
           # pays those sums once per candidate list, so this is the add rate the same answers would need
           "effective_fp64_adds_per_s": cand_per_s * F}
    # one fused kernel (train_state_tab_kernel): O(K) lookups + the feature math per candidate, bounded by
    # instruction issue; per-candidate thread instructions from the committed ncu capture
    ncu = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text()).get("kernels", {}).get("pp_train_state_tab")
    if ncu:
        props = torch.cuda.get_device_properties(0)
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        issue_peak = 4 * 32 * props.multi_processor_count * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        achieved = cand_per_s * ncu["thread_instructions_per_candidate"]
        out["roofline"] = {"bound": "issue", "achieved": achieved / 1e12, "peak": issue_peak / 1e12,
                           "unit": "T thread-instr/s", "frac": achieved / issue_peak,
                           "note": "CUDA-event launch time over the ncu per-allowed-candidate instruction count "
                                   "of train_state_tab_kernel (E=512 envs, BERT-48 2x4 K=4)"}
    if want_cpu:
        out["cpu_baseline"] = cpu_pp_train(g, topo, K, env, applied, mask)
    return out


def cpu_pp_train(g, topo, K, env, applied, mask):
    """The reference PipeTrainEnv._state (one core) on the first partial plan of the same batch."""
    try:
        rir, _ = _ref_import()
        from autoplan.envs import PipeTrainEnv as RefEnv
        from autoplan.topology import DeviceTopology as RefTopo
    except ImportError:
        return None
    rg = rir.graph_from_dict(g.to_dict())
    renv = RefEnv(rg, RefTopo(topo.num_servers, topo.gpus_per_server), K, radius=3)
    renv.reset()
    k = int((applied[0] >= 0).sum())
    renv._applied = [int(x) for x in applied[0, :k]]
    t0 = time.perf_counter()
    renv._state()
    dt = time.perf_counter() - t0
    n = int(renv.action_mask().sum())
    return {"value": n / dt, "unit": "candidate plans/s", "cores": 1, "kind": "reference",
            "sample": f"one PipeTrainEnv._state call ({n} allowed candidates, {dt:.1f} s)"}


def bench_env_gen(args, world, rank, want_cpu):
    """PP-infer data plane: synthetic uniform profiles (generate_environment('uniform', 1280, seed) ->
    3 x 128 scaled arrays) generated per second on the device, bit-identical to the host path.
    Each rank generates its own contiguous seed range (weak scaling, no collective)."""
    import torch

    from paper_2007_04069_b200.dataproc import pcg64_states
    from paper_2007_04069_b200 import _native

    E, n, G = 65536, 1280, 128
    st = pcg64_states(range(rank * E, (rank + 1) * E))  # PCG64 seeding stays numpy's (host, untimed)
    d_st = torch.from_numpy(st.view("int64")).cuda()
    out = torch.empty((E, 3, G), dtype=torch.float64, device="cuda")
    lib = _native.require_device()

    def run():
        _native.check(lib.ap_generate_uniform_envs(_native.ptr(d_st), E, n, G, _native.ptr(out),
                                                   _native.stream_handle()))

    for _ in range(3):
        run()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 10
    s.record()
    for _ in range(iters):
        run()
    e.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), world) / iters
    draws_per_s = E * 3 * n / (ms / 1e3)
    res = {"value": world * E / (ms / 1e3), "unit": "environments/s",
           "config": {"distribution": "uniform", "source_length": n, "granularity": G, "envs_per_launch": E,
                      "seeds": "rank * 65536 + [0, 65536)"},
           "ms_per_launch": ms, "pcg64_draws_per_s": draws_per_s}
    if want_cpu:
        try:
            _ref_import()
            from autoplan.dataproc import generate_environment as ref_gen

            k, t0 = 0, time.perf_counter()
            while time.perf_counter() - t0 < 2.0:
                ref_gen("uniform", n, k)
                k += 1
            res["cpu_baseline"] = {"value": k / (time.perf_counter() - t0), "unit": "environments/s", "cores": 1,
                                   "kind": "reference", "sample": f"{k} reference generate_environment calls (2 s)"}
        except ImportError:
            pass
    return res


def bench_pp_infer(args, world, want_cpu):
    """PP-infer (boundaries, cuts) points/s: the exhaustive search over the full configC K=4 space."""
    import torch

    from paper_2007_04069_b200.dataproc import generate_environment
    from paper_2007_04069_b200.envs import PipeInferEnv, brute_force_plan
    from paper_2007_04069_b200.topology import PRESETS

    arrays = generate_environment("uniform", 1280, 0)
    env = PipeInferEnv(arrays, PRESETS["configc"], 4)
    brute_force_plan(env)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    bb, cc, length, points = brute_force_plan(env)
    dt = _max_over_ranks(time.perf_counter() - t0, world)
    out = {"value": world * points / dt, "unit": "points/s",
           "config": {"profile": "generate_environment(uniform, 1280, 0)", "topology": "configc", "stages": 4,
                      "points_per_search": points, "best": {"boundaries": bb, "cuts": cc, "length": length}},
           "seconds_per_search": dt}
    # compute-only search (64 KB of DRAM traffic per 1.5 G points): bounded by instruction issue.  Per-point
    # instruction count from the committed ncu capture; peak = 4 schedulers x 32 lanes x SMs x max SM clock.
    ncu = json.loads((ROOT / "profiles" / "ncu_summary.json").read_text()).get("kernels", {}).get("pp_infer_search")
    if ncu:
        props = torch.cuda.get_device_properties(0)
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        issue_peak = 4 * 32 * props.multi_processor_count * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        achieved = points / dt * ncu["thread_instructions_per_point"]  # per GPU
        out["roofline"] = {"bound": "issue", "achieved": achieved / 1e12, "peak": issue_peak / 1e12,
                           "unit": "T thread-instr/s", "frac": achieved / issue_peak,
                           "note": "API call time (host combo words + launch + sync) over the ncu per-point "
                                   "instruction count of infer_search_tab_kernel"}
    if want_cpu:
        try:
            _ref_import()
            from autoplan.envs import PipeInferEnv as RefEnv
            from autoplan.pipecost import PipelinePlan, pipeline_length
            from autoplan.topology import PRESETS as RP

            renv = RefEnv(arrays, RP["configc"], 4)
            import itertools

            combos = itertools.product(itertools.combinations(range(1, 128), 3), itertools.combinations(range(1, 32), 3))
            n, t0 = 0, time.perf_counter()
            for b, c in combos:
                pipeline_length(PipelinePlan(b, c, 1), renv.decode_metrics(b), renv.topo_norm)
                n += 1
                if n % 256 == 0 and time.perf_counter() - t0 > 3.0:
                    break
            out["cpu_baseline"] = {"value": n / (time.perf_counter() - t0), "unit": "points/s", "cores": 1,
                                   "kind": "reference", "sample": f"first {n} points of the same space"}
        except ImportError:
            pass
    return out


def bench_dqn_single(args, g, dims, groups, want_cpu):
    """Reference-semantics loop (one env, act / step / observe / learn per step, batch 64) on BERT-48 OPP."""
    import torch

    from paper_2007_04069_b200.agent import AgentConfig, DqnAgent, Transition
    from paper_2007_04069_b200.envs import OppEnv

    env = OppEnv(g, groups=groups)
    cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=2000)
    agent = DqnAgent(cfg, env.state_dim, env.num_actions, 0)

    def run(steps):
        done = 0
        state = env.reset()
        while done < steps:
            if env.done:
                state = env.reset()
            a = agent.act(state, env.action_mask())
            r = env.step(a)
            agent.observe(Transition(state, a, r.reward, r.next_state, r.done, env.action_mask()))
            agent.learn()
            state = r.next_state
            done += 1

    run(80)  # fill past the first batch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run(args.single_steps)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out = {"value": args.single_steps / dt, "unit": "env-steps/s",
           "config": {"graph": args.workload, "task": "opp", "envs": 1, "learn_batch": 64,
                      "learn_to_env_step_ratio": "1:1", "semantics": "reference train_partition loop"}}
    if want_cpu:
        out["cpu_baseline"] = cpu_dqn_single(g, dims, groups, args.cpu_seconds)
    return out


def cpu_dqn_single(g, dims, groups, seconds):
    try:
        rir, rsh = _ref_import()
        from autoplan.agent import AgentConfig as RA
        from autoplan.agent import DqnAgent as RD
        from autoplan.agent import Transition as RT
        from autoplan.envs import OppEnv as RO
        from autoplan.linkage import LinkageGroup as RL
    except ImportError:
        return None
    rg = rir.graph_from_dict(g.to_dict())
    rdims = {(d.instruction_id, d.dim): rir.DimIndex(d.flat_index, d.instruction_id, d.dim) for d in dims}
    rgroups = {}
    for (d, st), grp in groups.items():  # same groups, as reference objects (skips its 18 s extraction)
        key = (rdims[(d.instruction_id, d.dim)], rsh.DimStatus(int(st)))
        rgroups[key] = RL(key, tuple((rdims[(x.instruction_id, x.dim)], rsh.DimStatus(int(s))) for x, s in grp.implied),
                          grp.infeasible)
    env = RO(rg, groups=rgroups)
    agent = RD(RA(lr=0.0005, epsilon_decay_iters=2000), env.state_dim, env.num_actions, 0)
    n, t0 = 0, time.perf_counter()
    state = env.reset()
    while time.perf_counter() - t0 < seconds:
        if env.done:
            state = env.reset()
        a = agent.act(state, env.action_mask())
        r = env.step(a)
        agent.observe(RT(state, a, r.reward, r.next_state, r.done, env.action_mask()))
        agent.learn()
        state = r.next_state
        n += 1
    dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "env-steps/s", "cores": 1, "kind": "reference",
            "sample": f"{n} reference train_partition steps on BERT-48 OPP ({dt:.1f} s; includes the first, "
                      f"learn-free steps)"}


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
