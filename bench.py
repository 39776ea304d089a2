#!/usr/bin/env python
"""Benchmark: candidate plans evaluated / s on the Auto-MAP plan-exploration hot path.

Headline step = one pass of the batched propagation kernel (K1) over one batch of
synthetic plans on the BERT-48 HLO graph (BASELINE config 3): for every plan the
full fixed point (all |S| slot statuses), outcome and decided / newly counts
(SURVEY §8(d) "full contract").  Plans are prefixes of the REFERENCE's decision
order (`sorted_decision_order`, pinned in tests/golden/linkage_bert48.npz) with
k ~ U[1, |D|] and fair P/R coins (`workloads.prefix_seed_batch`, seed 20201007).
Per-GPU work is fixed as N grows (weak scaling); plans are sharded by global
index, no collective on the data path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Under torchrun each rank runs its shard; the device time is the max over ranks.
`--impl reference` times the reference planner's own CPU implementation
(baseline/_ref, `PropagationEngine.run`, engine reused) on all host cores over the
same plan rows; rank 0 alone runs it.  The bench never writes into the repo.

`secondary` carries the other figures of the metric: K1 in its other output
modes and on conflict-light batches, every BASELINE config (MLP2, BERT-base,
BERT-48, VGG-19, T5-large) with its own CPU baseline, roofline, ingest costs and
the goldens that pin it, the vectorised DQN env-steps/s at both GEMM precisions,
PP-train / PP-infer evaluation and the reference-semantics single-env loop.
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
GOLDEN = ROOT / "tests" / "golden"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default="bert48")
    p.add_argument("--batch", type=int, default=1 << 22, help="plans per GPU per step")
    p.add_argument("--e2e-batch", type=int, default=1 << 18)
    p.add_argument("--e2e-steps", type=int, default=5)
    p.add_argument("--cpu-seconds", type=float, default=10.0)
    p.add_argument("--cpu-seconds-config", type=float, default=2.0, help="per-config reference CPU samples")
    p.add_argument("--ref-rows-per-worker", type=int, default=0,
                   help="reference arm: plan rows per worker process per step (0: ~1 s of work, 64..256)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-secondary", action="store_true", help="headline + e2e only")
    p.add_argument("--no-configs", action="store_true", help="skip the per-BASELINE-config block")
    p.add_argument("--dqn-envs", type=int, default=4096)
    p.add_argument("--dqn-learn-steps", type=int, default=4)
    p.add_argument("--dqn-steps", type=int, default=300)
    p.add_argument("--dqn-eager", action="store_true", help="launch the vector step eagerly (no CUDA graph)")
    p.add_argument("--pp-envs", type=int, default=512, help="PP-train env states evaluated per launch")
    p.add_argument("--pp-dqn-envs", type=int, default=1024, help="vectorised PP-train DQN envs per GPU")
    p.add_argument("--single-steps", type=int, default=300)
    p.add_argument("--single-episodes", type=int, default=30, help="episodes of the device-resident single-env loop")
    return p.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# -- workloads (identical in both arms) ------------------------------------------------


def workload_setup(name: str, task: str = "opp"):
    from paper_2007_04069_b200 import graphs
    from paper_2007_04069_b200.envs import adp_candidates
    from paper_2007_04069_b200.ir import decision_dims

    g = graphs.generate(name)
    names = g.trainable_variables if task == "opp" else [g.instruction(i).name for i in adp_candidates(g)]
    return g, decision_dims(g, names)


def golden_order(name: str, task: str, n: int):
    """The reference's decision order: `sorted_decision_order` from the committed linkage golden
    (OPP; linkage.py:71-83) or the identity (ADP, envs.py:264-273)."""
    import numpy as np

    if task == "adp":
        return np.arange(n, dtype=np.int64), "identity (AdpEnv, envs.py:264-273)"
    z = np.load(GOLDEN / f"linkage_{name}.npz")
    order = np.asarray(z["order"], dtype=np.int64)
    assert len(order) == n, (name, len(order), n)
    return order, f"reference sorted_decision_order (tests/golden/linkage_{name}.npz)"


def bench_config(name, g, dims, order_src, plan_batch="prefix"):
    desc = {
        "prefix": "decision-order prefixes k~U[1,|D|], fair P/R coins (workloads.prefix_seed_batch, seed 20201007)",
        "short": "decision-order prefixes k~U[1,16], fair P/R coins (workloads.prefix_seed_batch kmax=16)",
        "triggers": "the 2|D| linkage triggers tiled over the batch (workloads.trigger_seed_batch)",
    }[plan_batch]
    return {
        "workload": f"{name} OPP propagation, full contract (all slot statuses + outcome + counts)",
        "graph": name,
        "instructions": len(g),
        "slots": int(g.flat().num_slots),
        "candidate_dims": len(dims),
        "plan_batch": desc,
        "decision_order": order_src,
        "conflict_rows": "outcome + counts as the reference; slot rows hold the closure with P winning "
                         "(the reference's mid-sweep snapshot of a CONFLICT comes from ap_propagate_trace)",
        "l2": "inputs larger than L2 (seeds + slot outputs per step >> 126 MB)",
    }


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


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    return json.loads(p.read_text()) if p.exists() else {}


def measured_peak_hbm():
    pk = peaks()
    if "hbm_gbs" in pk:
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json, copy burst)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_kernel(key: str):
    p = ROOT / "profiles" / "ncu_summary.json"
    if not p.exists():
        return None
    return json.loads(p.read_text()).get("kernels", {}).get(key)


def issue_peak():
    import torch

    props = torch.cuda.get_device_properties(0)
    return 4 * 32 * props.multi_processor_count * float(peaks().get("sm_max_mhz", 1965.0)) * 1e6


# -- CPU baselines (reference planner, baseline/_ref) ------------------------------------


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
    """Reference PropagationEngine.run per row (engine reused); returns (rows, busy seconds)."""
    eng, dims, vals = _W["eng"], _W["dims"], _W["vals"]
    t0 = time.perf_counter()
    for row in rows:
        eng.run({dims[j]: vals[int(v)] for j, v in enumerate(row) if v != -1})
    return len(rows), time.perf_counter() - t0


def cpu_ref_propagation(g, dims, rows, seconds: float, what: str):
    """The reference engine (reused, one core) on the first rows of the same batch."""
    try:
        _ref_worker_init(json.dumps(g.to_dict()), [(d.flat_index, d.instruction_id, d.dim) for d in dims])
    except ImportError as exc:
        return {"unavailable": f"baseline/_ref not importable: {exc}"}
    done, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds and done < len(rows):
        _ref_eval_rows(rows[done:done + 1])
        done += 1
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"first {done} plans of {what}, reference PropagationEngine(graph, dims).run per plan, "
                      f"engine reused, {dt:.2f} s on 1 host core"}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def run_reference_arm(args):
    """The reference's own CPU implementation on all host cores (one process per core; its
    AUTOPLAN_THREADS thread pool is GIL-bound).  Each step = one pool.map of `per_worker`
    contiguous plan rows per worker over the SAME rows, order and graph as our arm."""
    import multiprocessing as mp

    from paper_2007_04069_b200.workloads import prefix_seed_batch

    rank, world, _ = env_rank()
    if rank != 0:
        return
    g, dims = workload_setup(args.workload)
    order, order_src = golden_order(args.workload, "opp", len(dims))
    cores = host_cores()
    per_worker = args.ref_rows_per_worker or max(64, min(256, int(150 * 190 / max(1, args.steps + args.warmup))))
    total_rows = (args.steps + args.warmup) * cores * per_worker
    sample = prefix_seed_batch(order, 0, total_rows).numpy()
    dims_raw = [(d.flat_index, d.instruction_id, d.dim) for d in dims]
    ctx = mp.get_context("fork")
    with ctx.Pool(cores, initializer=_ref_worker_init, initargs=(json.dumps(g.to_dict()), dims_raw)) as pool:
        step_t, busy = [], []
        cursor = 0
        for step in range(args.warmup + args.steps):
            chunks = [sample[cursor + w * per_worker: cursor + (w + 1) * per_worker] for w in range(cores)]
            cursor += cores * per_worker
            t0 = time.perf_counter()
            res = pool.map(_ref_eval_rows, chunks, chunksize=1)
            if step >= args.warmup:
                step_t.append(time.perf_counter() - t0)
                busy += [b for _, b in res]
    total = sum(step_t)
    value = args.steps * cores * per_worker / total
    per_core = len(busy) * per_worker / sum(busy)  # plans/s of one busy worker
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
        "config": bench_config(args.workload, g, dims, order_src),
        "run_info": {"plans_per_step": cores * per_worker, "rows_per_worker_per_step": per_worker,
                     "first_row": 0, "pool": f"multiprocessing fork pool of {cores} (sched_getaffinity)"},
        "cpu_baseline": {
            "value": value,
            "unit": UNIT,
            "cores": cores,
            "kind": "reference",
            "sample": f"{cores * per_worker} plans per step ({per_worker} contiguous rows per worker process, "
                      f"rows [0, {total_rows}) of the same batch), reference PropagationEngine.run, engine reused, "
                      f"multiprocessing pool of {cores}",
            "per_core_busy_plans_per_s": per_core,
            "ideal_plans_per_s": cores * per_core,
            "parallel_efficiency": value / (cores * per_core),
        },
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -- K1 measurement helpers ---------------------------------------------------------------


def _max_over_ranks(x: float, world: int) -> float:
    from paper_2007_04069_b200.distributed import max_over_ranks

    return max_over_ranks(x) if world > 1 else float(x)


def k1_bytes(n, S, mode):
    """Algorithmic HBM bytes per plan: seed row read + outputs written."""
    out = {"full": S, "env": n, "packed": (S + 15) // 16 * 4}[mode]
    return n + out + 1 + 16


def k1_outputs(eng, B, mode):
    import torch

    o = {"outcome": torch.empty(B, dtype=torch.uint8, device="cuda"),
         "counts": torch.empty((B, 4), dtype=torch.int32, device="cuda")}
    if mode == "full":
        o["slots"] = torch.empty((B, eng.slots_stride), dtype=torch.int8, device="cuda")
    elif mode == "env":
        o["statuses"] = torch.empty((B, max(16, (len(eng.candidates) + 15) // 16 * 16)), dtype=torch.int8,
                                    device="cuda")
    else:
        o["packed"] = torch.empty((B, eng.packed_slots_stride), dtype=torch.uint8, device="cuda")
    return o


def k1_launch(eng, seeds, o, stream):
    eng.launch(seeds, o["outcome"], o["counts"], o.get("slots"), o.get("statuses"), stream=stream,
               packed=o.get("packed"))


def k1_measure(eng, seeds, mode, launches=10, warmup=3, world=1):
    """Average device time per K1 launch (CUDA events on the launching stream)."""
    import torch

    B = seeds.shape[0]
    o = k1_outputs(eng, B, mode)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        k1_launch(eng, seeds, o, stream)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(launches):
        k1_launch(eng, seeds, o, stream)
    e.record(stream)
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), world) / launches
    conflict = float((o["outcome"] == 2).float().mean().item())
    return ms, conflict, o


def k1_entry(name, eng, seeds, mode, world, what, launches=10):
    n, S = len(eng.candidates), int(eng._eng.num_slots)
    B = seeds.shape[0]
    ms, conflict, _ = k1_measure(eng, seeds, mode, launches=launches, world=world)
    bpp = k1_bytes(n, S, mode)
    peak, peak_src = measured_peak_hbm()
    achieved = B * bpp / (ms / 1e3) / 1e9
    return {"value": world * B / (ms / 1e3), "unit": UNIT, "mode": mode, "plans_per_launch": B,
            "ms_per_launch": ms, "conflict_rate": round(conflict, 4), "batch": what,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "bytes_per_plan": bpp, "peak_source": peak_src,
                         "traffic": None}}


def auto_batch(n, S, target_bytes=2 << 30, lo=1 << 16, hi=1 << 24):
    per = (n + 15) // 16 * 16 + (S + 15) // 16 * 16 + 17
    b = lo
    while b < hi and b * per < target_bytes:
        b *= 2
    return b


# -- our arm -------------------------------------------------------------------------------


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2007_04069_b200.distributed import plan_shard
    from paper_2007_04069_b200.linkage import extract_linkage_groups, sorted_decision_order
    from paper_2007_04069_b200.sharding import PropagationEngine
    from paper_2007_04069_b200.workloads import prefix_seed_batch

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    g, dims = workload_setup(args.workload)
    n = len(dims)
    S = g.flat().num_slots
    order, order_src = golden_order(args.workload, "opp", n)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = PropagationEngine(g, dims)
    eng.prepare()  # ap_graph_create + decision tables (host C++ rule compile, device upload)
    torch.cuda.synchronize()
    ingest_s = time.perf_counter() - t0
    # our own linkage extraction (one batched launch of 2|D| triggers) must reproduce the golden order
    t0 = time.perf_counter()
    groups = extract_linkage_groups(g, dims)
    ours_order = np.asarray([d.flat_index for d in sorted_decision_order(groups)], dtype=np.int64)
    linkage_s = time.perf_counter() - t0

    B = args.batch
    seeds = prefix_seed_batch(order, *plan_shard(rank, B), device="cuda", chunk=1 << 18)
    o = k1_outputs(eng, B, "full")
    stream = torch.cuda.current_stream()

    for _ in range(args.warmup):
        k1_launch(eng, seeds, o, stream)
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
        k1_launch(eng, seeds, o, stream)
    end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clock_info = clocks.stop()
    elapsed_ms = start.elapsed_time(end)
    max_ms = _max_over_ranks(elapsed_ms, world)
    conflict_rate = float((o["outcome"] == 2).float().mean().item())
    del o

    # e2e through the host-buffer API: pinned H2D + kernel + D2H every step
    Be = args.e2e_batch
    seeds_host = prefix_seed_batch(order, *plan_shard(rank, Be), device="cuda").cpu().pin_memory()

    def e2e_run(want_slots):
        out_host = None
        for _ in range(2):
            out_host = eng.run_batch_host(seeds_host, want_slots=want_slots, out=out_host)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            out_host = eng.run_batch_host(seeds_host, want_slots=want_slots, out=out_host)
        return _max_over_ranks(time.perf_counter() - t0, world)

    e2e_s = e2e_run(True)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_ref_propagation(g, dims, prefix_seed_batch(order, 0, 4096).numpy(), args.cpu_seconds,
                                  "the same batch (rows 0..)")

    secondary = {}
    if not args.no_secondary:
        want_cpu = rank == 0 and world == 1 and not args.no_cpu_baseline
        e2e_pk_s = e2e_run("packed")
        secondary["e2e_packed_slots"] = {
            "value": world * Be * args.e2e_steps / e2e_pk_s,
            "unit": UNIT,
            "h2d_bytes_per_step": Be * n,
            "d2h_bytes_per_step": Be * (eng.packed_slots_stride + 1 + 16),
            "api": 'PropagationEngine.run_batch_host(want_slots="packed") (K1 emits 2-bit slot rows, '
                   'lossless: code = status + 1, decoded by sharding.unpack_slots2)',
        }
        secondary["k1_modes"] = bench_k1_modes(args, eng, g, order, world, rank)
        if not args.no_configs:
            secondary["configs"] = bench_configs(args, world, rank, want_cpu)
        secondary["dqn_env_steps_per_s"] = bench_dqn_vec(args, g, world, rank, precision=1)
        secondary["dqn_env_steps_per_s_precision3"] = bench_dqn_vec(args, g, world, rank, precision=3)
        secondary["dqn_env_steps_per_s_pp_train"] = bench_dqn_pipe(args, "bert48", world, rank)
        secondary["dqn_env_steps_per_s_pp_infer"] = bench_dqn_infer(args, world, rank)
        secondary["pp_train_candidates_per_s"] = bench_pp_train(args, "bert48", world, want_cpu)
        secondary["pp_infer_points_per_s"] = bench_pp_infer(args, world, want_cpu)
        secondary["pp_infer_envs_generated_per_s"] = bench_env_gen(args, world, rank, want_cpu)
        if rank == 0 and world == 1:
            secondary["dqn_env_steps_per_s_single_env"] = bench_dqn_single(args, g, dims, groups, want_cpu)

    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return
    per_launch_s = max_ms / 1e3 / args.steps
    bytes_per_plan = k1_bytes(n, S, "full")
    achieved = B * bytes_per_plan / per_launch_s / 1e9
    peak, peak_src = measured_peak_hbm()
    ncu = ncu_kernel("propagate_kernel")
    traffic = None if ncu is None else ncu["dram_bytes_per_plan"] * B
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
        "config": bench_config(args.workload, g, dims, order_src),
        "run_info": {
            "plans_per_gpu_per_step": B,
            "parallelism": f"plan-sharded x{world} (no data-path collective)",
            "conflict_rate": round(conflict_rate, 4),
            "order_matches_reference_golden": bool(np.array_equal(ours_order, order)),
            "ingest_s": {"graph_create_and_decision_tables": round(ingest_s, 4),
                         "linkage_2D_triggers_on_gpu": round(linkage_s, 4)},
        },
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
            "traffic_source": "profiles/ncu_summary.json propagate_kernel dram bytes/plan x plans per launch "
                              "(ncu --set full)",
        },
        "cpu_baseline": cpu,
        "e2e": {
            "value": world * Be * args.e2e_steps / e2e_s,
            "unit": UNIT,
            "h2d_bytes_per_step": Be * n,
            "d2h_bytes_per_step": Be * (eng.slots_stride + 1 + 16),
            "api": "PropagationEngine.run_batch_host (pinned host seeds -> host outcome/counts/int8 slots)",
        },
        "gpu_launches": args.steps,
        "clocks": clock_info,
        "secondary": secondary,
    }
    print(json.dumps(line), flush=True)


# -- secondary: K1 modes and conflict-light batches (BERT-48) -----------------------------


def bench_k1_modes(args, eng, g, order, world, rank):
    """K1 beside the headline: env-only output (candidate statuses instead of all slots), 2-bit packed
    slot rows emitted by K1 itself, and two conflict-light batches in the full contract."""
    import torch

    from paper_2007_04069_b200.distributed import plan_shard
    from paper_2007_04069_b200.workloads import prefix_seed_batch, trigger_seed_batch

    n = len(eng.candidates)
    B = args.batch
    out = {}
    seeds = prefix_seed_batch(order, *plan_shard(rank, B), device="cuda", chunk=1 << 18)
    out["env_only"] = k1_entry("bert48", eng, seeds, "env", world, "headline batch")
    out["packed_slots"] = k1_entry("bert48", eng, seeds, "packed", world, "headline batch")
    del seeds
    torch.cuda.empty_cache()
    seeds = trigger_seed_batch(n, *plan_shard(rank, B), device="cuda")
    out["full_linkage_triggers"] = k1_entry("bert48", eng, seeds, "full", world,
                                            "the 2|D| linkage triggers tiled to the batch")
    del seeds
    seeds = prefix_seed_batch(order, *plan_shard(rank, B), device="cuda", chunk=1 << 18, kmax=16)
    out["full_short_prefix"] = k1_entry("bert48", eng, seeds, "full", world, "decision-order prefixes k~U[1,16]")
    del seeds
    torch.cuda.empty_cache()
    out["parity"] = ("tests/test_bench_batches_gpu.py: >= 1,000 conflict-free rows of each batch (headline, "
                     "triggers, short prefixes) slot-checked against the C oracle, plus outcome/counts of sampled "
                     "rows; packed rows decode to the int8 rows")
    return out


# -- secondary: the five BASELINE configs ---------------------------------------------------


PARITY = {
    "mlp2": ["prop_mlp2", "linkage_mlp2", "search_opp_mlp2 (free-running + finetune)", "linkage_cache_mlp2"],
    "bert_base": ["prop_bert_base", "linkage_bert_base", "search_opp_bert_base (free-running + finetune)",
                  "search_adp_bert_base", "pipe_bert_base_2x4"],
    "bert48": ["prop_bert48", "linkage_bert48", "pipe_bert48_2x4 (PP-train trajectories K=4)"],
    "vgg19": ["prop_vgg19", "linkage_vgg19", "search_opp_vgg19 (free-running + finetune)", "search_adp_vgg19",
              "pipe_vgg19_configb", "linkage_cache_vgg19"],
    "t5_large": ["prop_t5_large", "linkage_t5_large", "pipe_t5_large_2x4 (PP-train trajectories K=4)"],
}


def bench_propagation_config(args, name, task, world, rank, want_cpu, dqn=True):
    """K1 plans/s (full contract) on one graph / task, its reference CPU sample, ingest costs and the
    vectorised DQN env-steps/s of the same task."""
    import torch

    from paper_2007_04069_b200.distributed import plan_shard
    from paper_2007_04069_b200.sharding import PropagationEngine
    from paper_2007_04069_b200.workloads import prefix_seed_batch

    g, dims = workload_setup(name, task)
    n, S = len(dims), int(g.flat().num_slots)
    order, order_src = golden_order(name, task, n)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = PropagationEngine(g, dims)
    eng.prepare()
    torch.cuda.synchronize()
    ingest = time.perf_counter() - t0
    B = auto_batch(n, S)
    seeds = prefix_seed_batch(order, *plan_shard(rank, B), device="cuda", chunk=1 << 18)
    res = k1_entry(name, eng, seeds, "full", world, "decision-order prefixes k~U[1,|D|]")
    del seeds
    torch.cuda.empty_cache()
    res.update({"task": task, "candidate_dims": n, "slots": S, "instructions": len(g), "decision_order": order_src,
                "ingest_s": {"graph_create_and_decision_tables": round(ingest, 4)}})
    if task == "opp":
        from paper_2007_04069_b200.linkage import extract_linkage_groups

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        extract_linkage_groups(g, dims)
        res["ingest_s"]["linkage_2D_triggers_on_gpu"] = round(time.perf_counter() - t0, 4)
    if want_cpu:
        res["cpu_baseline"] = cpu_ref_propagation(g, dims, prefix_seed_batch(order, 0, 2048).numpy(),
                                                  args.cpu_seconds_config, "the same batch")
    if dqn:
        res["dqn"] = bench_dqn_vec(args, g, world, rank, precision=1, task=task, name=name, light=True)
        if want_cpu:
            res["dqn"]["cpu_baseline"] = cpu_dqn_single(g, name, task, args.cpu_seconds_config)
    return res


def bench_configs(args, world, rank, want_cpu):
    cfg = {}
    cfg["1_mlp2_opp_2dev"] = {"opp": bench_propagation_config(args, "mlp2", "opp", world, rank, want_cpu),
                              "parity": PARITY["mlp2"],
                              "note": "the '2 devices' has no effect on OPP in the reference (sharding.py:6-9)"}
    cfg["2_bert_base_opp_dp_8dev"] = {
        "opp": bench_propagation_config(args, "bert_base", "opp", world, rank, want_cpu),
        "adp": bench_propagation_config(args, "bert_base", "adp", world, rank, want_cpu),
        "parity": PARITY["bert_base"]}
    cfg["3_bert48_opp_pp_dp_8dev"] = {
        "opp": "headline (value / roofline / cpu_baseline / e2e of this line; DQN in dqn_env_steps_per_s)",
        "adp": bench_propagation_config(args, "bert48", "adp", world, rank, want_cpu),
        "pp_train": "pp_train_candidates_per_s / dqn_env_steps_per_s_pp_train of this line (2x4 planned mesh, K=4)",
        "parity": PARITY["bert48"]}
    cfg["4_vgg19_adp_vs_opp_8dev"] = {
        "opp": bench_propagation_config(args, "vgg19", "opp", world, rank, want_cpu),
        "adp": bench_propagation_config(args, "vgg19", "adp", world, rank, want_cpu),
        "parity": PARITY["vgg19"]}
    cfg["5_t5_large_pp_8dev"] = {
        "pp_train": bench_pp_train(args, "t5_large", world, want_cpu),
        "dqn_pp_train": bench_dqn_pipe(args, "t5_large", world, rank),
        "opp": bench_propagation_config(args, "t5_large", "opp", world, rank, want_cpu, dqn=False),
        "parity": PARITY["t5_large"],
        "note": "8 devices planned as a 2x4 mesh: a single 8-GPU server leaves PP-train no legal pivot "
                "(pipecost.py:265, SURVEY §7 hard part 6)"}
    return cfg


# -- secondary: DQN, PP-train, PP-infer ------------------------------------------------------


def bench_dqn_pipe(args, name, world, rank):
    """Throughput-mode DQN on PP-train (2x4, K=4): E VecPipeTrainEnv episodes per GPU, each vector
    step = act (state 4C wide) + pick + terminal metrics / length + K2 next states + L learn steps."""
    import torch
    import torch.distributed as dist

    from paper_2007_04069_b200 import graphs
    from paper_2007_04069_b200.agent import AgentConfig
    from paper_2007_04069_b200.topology import DeviceTopology
    from paper_2007_04069_b200.vec import VecDqnTrainer, VecPipeTrainEnv

    g = graphs.generate(name)
    E, L = args.pp_dqn_envs, args.dqn_learn_steps
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    env = VecPipeTrainEnv(g, DeviceTopology(2, 4), 4, E)
    torch.cuda.synchronize()
    ingest = time.perf_counter() - t0
    cfg = AgentConfig(lr=0.001, epsilon_decay_iters=10000)
    pg = dist.group.WORLD if world > 1 else None
    tr = VecDqnTrainer(env, cfg, capacity=4 * E, seed=rank, learn_steps=L, process_group=pg, use_graph=True)
    for _ in range(5):
        tr.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    steps = max(30, args.dqn_steps // 4)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        tr.step()
    e.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), world)
    best = tr.best_plan_global()
    C = env.C
    return {
        "value": world * E * steps / (ms / 1e3),
        "unit": "env-steps/s",
        "config": {"graph": name, "task": "pp-train", "topology": "2x4", "stages": 4, "radius": 3,
                   "candidates": C, "state_dim": env.state_dim, "envs_per_gpu": E,
                   "learn_steps_per_vector_step": L, "learn_batch": cfg.batch_size,
                   "learn_to_env_step_ratio": f"{L}:{E}", "hidden": list(cfg.hidden), "replay_capacity": tr.capacity,
                   "vector_steps": steps, "cuda_graph": tr.graph is not None, "precision": tr.net.precision},
        "ms_per_vector_step": ms / steps,
        "episodes_finished_rank0": int(env.episodes_done.sum().item()),
        "best_plan": None if best is None else {"pipeline_length": -best.reward, "global_episode": best.episode},
        "ingest_s": {"env_ctor_incl_candidate_pivots_and_stage_sum_table": round(ingest, 4)},
        "stage_sum_table_bytes": 8 * ((C + 1) ** 2 + (C + 1)),
        "reference_note": "reference PipeTrainEnv._state takes seconds per state on the host (pp_train cpu_baseline),"
                          " i.e. < 1 env-step/s",
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
    cfg = AgentConfig(lr=0.001, epsilon_decay_iters=10000)
    pg = dist.group.WORLD if world > 1 else None
    tr = VecDqnTrainer(env, cfg, capacity=max(4 * E, 4096), seed=rank, learn_steps=L, process_group=pg,
                       use_graph=True)
    for _ in range(5):
        tr.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    steps = args.dqn_steps
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(steps):
        tr.step()
    e.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), world)
    best = tr.best_plan_global()
    return {
        "value": world * E * steps / (ms / 1e3),
        "unit": "env-steps/s",
        "config": {"profile": "generate_environment(uniform, 1280, 0)", "topology": "configc", "stages": 4,
                   "bands": "infer_search_bands(radius 3)", "state_dim": env.state_dim, "actions": env.num_actions,
                   "envs_per_gpu": E, "learn_steps_per_vector_step": L, "learn_batch": cfg.batch_size,
                   "learn_to_env_step_ratio": f"{L}:{E}", "hidden": list(cfg.hidden), "vector_steps": steps,
                   "cuda_graph": tr.graph is not None, "precision": tr.net.precision},
        "ms_per_vector_step": ms / steps,
        "episodes_finished_rank0": int(env.episodes_done.sum().item()),
        "best_plan": None if best is None else {"pipeline_length": -best.reward, "global_episode": best.episode},
    }


def bench_dqn_vec(args, g, world, rank, precision=1, task="opp", name="bert48", light=False):
    """Throughput-mode DQN: E envs per GPU, batched act / step / observe, L learn steps (batch 64) per
    vector step, the whole vector step captured in one CUDA graph."""
    import torch
    import torch.distributed as dist

    from paper_2007_04069_b200.agent import AgentConfig
    from paper_2007_04069_b200.vec import VecDqnTrainer, VecPartitionEnv

    E, L = args.dqn_envs, args.dqn_learn_steps
    env = VecPartitionEnv(g, E, task=task)
    cfg = AgentConfig(lr=0.0005, epsilon_decay_iters=500 if task == "adp" else 2000)
    pg = dist.group.WORLD if world > 1 else None
    tr = VecDqnTrainer(env, cfg, capacity=max(4 * E, 4096), seed=rank, learn_steps=L, process_group=pg,
                       precision=precision, use_graph=not args.dqn_eager)
    for _ in range(5):
        tr.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    steps = args.dqn_steps
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = tr.launches
    s.record()
    for _ in range(steps):
        tr.step()
    e.record()
    torch.cuda.synchronize()
    ms = _max_over_ranks(s.elapsed_time(e), world)
    best = tr.best_plan_global()  # all-gather of every rank's incumbent, first-wins by global episode id
    out = {
        "value": world * E * steps / (ms / 1e3),
        "unit": "env-steps/s",
        "config": {"graph": name, "task": task, "envs_per_gpu": E, "learn_steps_per_vector_step": L,
                   "learn_batch": cfg.batch_size, "learn_to_env_step_ratio": f"{L}:{E}",
                   "hidden": list(cfg.hidden), "state_dim": env.state_dim, "replay_capacity": tr.capacity,
                   "parallelism": (f"data-parallel DQN x{world}, " + ("Q-gradient all-reduce over NVLink peer memory "
                                   "fused with Adam (ap_dp_allreduce_adam)" if tr.peer is not None else
                                   "NCCL all-reduce of Q-gradients")) if world > 1 else "1 GPU",
                   "vector_steps": steps, "precision": precision,
                   "precision_note": "3 = 3xTF32 (Q within 1e-5 of the fp64 reference, tests/test_agent_gpu.py); "
                                     "1 = one TF32 pass (within 5e-3, test_gemm_tf32_is_tf32_accurate)"},
        "ms_per_vector_step": ms / steps,
        "cuda_graph": tr.graph is not None,
        "episodes_finished_rank0": int(env.episodes_done.sum().item()),
        "envs_with_completed_episode_rank0": int((env.best_episode >= 0).sum().item()),
        "best_plan": None if best is None else {"partitions": best.partitions, "return": best.reward,
                                                "global_episode": best.episode},
        "gpu_launches_per_vector_step": (tr.launches - launches0) / steps,
    }
    if light:
        return out
    # tensor-pipe figure for the batched act forward (the dominant GEMMs): 10 forwards in a CUDA graph
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
    flops = 2.0 * E * (S * H + H * H + H * 3)  # algorithmic, one pass
    passes = 3 if precision == 3 else 1  # 3xTF32 issues three TF32 MMAs per product
    tf32_peak = float(peaks().get("bf16_tflops", 1590.0)) / 2.0
    out["act_forward_tensor"] = {
        "bound": "tensor", "achieved": passes * flops / fwd_s / 1e12, "unit": "TFLOP/s (TF32 MMA issued)",
        "peak": tf32_peak, "peak_source": "half of measured bf16 (dense TF32 = bf16/2)",
        "frac": passes * flops / fwd_s / 1e12 / tf32_peak, "gemm_m": E, "us_per_forward": fwd_s * 1e6,
        "note": f"3 GEMMs M=E K=state_dim/256 N=256/3, tcgen05 kind::tf32, precision={precision}"}
    return out


def bench_pp_train(args, name, world, want_cpu):
    """PP-train candidate plans/s: PipeTrainEnv._state over all allowed pivots of E random partial plans."""
    import ctypes

    import numpy as np
    import torch

    from paper_2007_04069_b200 import _native, graphs
    from paper_2007_04069_b200.envs import PipeTrainEnv
    from paper_2007_04069_b200.topology import DeviceTopology

    g = graphs.generate(name)
    topo = DeviceTopology(2, 4)
    K = 4
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    env = PipeTrainEnv(g, topo, K, radius=3)
    torch.cuda.synchronize()
    ctor_s = time.perf_counter() - t0
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
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    env._model.bind_candidates(d_cand)  # the stage-sum table build (ingest, once per candidate list)
    torch.cuda.synchronize()
    table_s = time.perf_counter() - t0
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
           "config": {"graph": name, "topology": "2x4", "stages": K, "radius": 3, "candidates": C,
                      "env_states_per_launch": E, "allowed_candidates_per_launch": evaluated,
                      "forward_instructions": F, "stage_sums": "bound stage-sum table (ap_pipe_train_table)"},
           "ms_per_launch": ms / iters,
           "ingest_s": {"env_ctor_incl_candidate_pivots": round(ctor_s, 4), "stage_sum_table_build": round(table_s, 4)},
           "stage_sum_table_bytes": 8 * ((C + 1) ** 2 + (C + 1)),
           # the reference re-sums N_f costs per candidate (SURVEY §8(d)'s fp64-add bound); the bound table
           # pays those sums once per candidate list, so this is the add rate the same answers would need
           "effective_fp64_adds_per_s": cand_per_s * F}
    # one fused kernel (train_state_tab_kernel): O(K) lookups + the feature math per candidate, bounded by
    # instruction issue; per-candidate thread instructions from the committed ncu capture of the same shape
    ncu = ncu_kernel("pp_train_state_tab" if name == "bert48" else f"pp_train_state_tab_{name}")
    if ncu:
        pk = issue_peak()
        achieved = cand_per_s * ncu["thread_instructions_per_candidate"]
        out["roofline"] = {"bound": "issue", "achieved": achieved / 1e12, "peak": pk / 1e12,
                           "unit": "T thread-instr/s", "frac": achieved / pk,
                           "note": "CUDA-event launch time over the ncu per-allowed-candidate instruction count "
                                   f"of train_state_tab_kernel (E=512 envs, {name} 2x4 K=4)"}
    if want_cpu:
        out["cpu_baseline"] = cpu_pp_train(g, topo, K, applied)
    return out


def cpu_pp_train(g, topo, K, applied):
    """The reference PipeTrainEnv._state (one core) on the first partial plan of the same batch."""
    try:
        rir, _ = _ref_import()
        from autoplan.envs import PipeTrainEnv as RefEnv
        from autoplan.topology import DeviceTopology as RefTopo
    except ImportError as exc:
        return {"unavailable": f"baseline/_ref not importable: {exc}"}
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
    """PP-infer data plane: synthetic profiles (generate_environment(dist, 1280, seed) -> 3 x 128 scaled
    arrays) generated per second on the device, bit-identical to the host path, for the reference's three
    distributions.  Each rank generates its own contiguous seed range (weak scaling, no collective)."""
    import torch

    from paper_2007_04069_b200 import _native
    from paper_2007_04069_b200.dataproc import pcg64_states

    n, G = 1280, 128
    out_all = {}
    for kind, dist, E in ((0, "uniform", 65536), (1, "normal", 65536), (2, "binomial", 16384)):
        st = pcg64_states(range(rank * E, (rank + 1) * E))  # PCG64 seeding stays numpy's (host, untimed)
        d_st = torch.from_numpy(st.view("int64")).cuda()
        out = torch.empty((E, 3, G), dtype=torch.float64, device="cuda")
        lib = _native.require_device()

        def run():
            _native.check(lib.ap_generate_envs(kind, _native.ptr(d_st), E, n, G, _native.ptr(out),
                                               _native.stream_handle()))

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
        ms = _max_over_ranks(s.elapsed_time(e), world) / iters
        res = {"value": world * E / (ms / 1e3), "unit": "environments/s",
               "config": {"distribution": dist, "source_length": n, "granularity": G, "envs_per_launch": E,
                          "seeds": f"rank * {E} + [0, {E})",
                          "sampler": {"uniform": "PCG64 jump-ahead, one CTA per env",
                                      "normal": "numpy ziggurat, one thread per env",
                                      "binomial": "numpy BTPE, one thread per env"}[dist]},
               "ms_per_launch": ms}
        if want_cpu:
            try:
                _ref_import()
                from autoplan.dataproc import generate_environment as ref_gen

                k, t0 = 0, time.perf_counter()
                while time.perf_counter() - t0 < 1.5:
                    ref_gen(dist, n, k)
                    k += 1
                res["cpu_baseline"] = {"value": k / (time.perf_counter() - t0), "unit": "environments/s",
                                       "cores": 1, "kind": "reference",
                                       "sample": f"{k} reference generate_environment({dist!r}) calls (1.5 s)"}
            except ImportError as exc:
                res["cpu_baseline"] = {"unavailable": f"baseline/_ref not importable: {exc}"}
        out_all[dist] = res
        del out, d_st
    head = dict(out_all["uniform"])
    head["by_distribution"] = out_all
    return head


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
    ncu = ncu_kernel("pp_infer_search")
    if ncu:
        pk = issue_peak()
        achieved = points / dt * ncu["thread_instructions_per_point"]  # per GPU
        out["roofline"] = {"bound": "issue", "achieved": achieved / 1e12, "peak": pk / 1e12,
                           "unit": "T thread-instr/s", "frac": achieved / pk,
                           "note": "API call time (host combo words + launch + sync) over the ncu per-point "
                                   "instruction count of infer_search_tab_kernel"}
    if want_cpu:
        try:
            _ref_import()
            import itertools

            from autoplan.envs import PipeInferEnv as RefEnv
            from autoplan.pipecost import PipelinePlan, pipeline_length
            from autoplan.topology import PRESETS as RP

            renv = RefEnv(arrays, RP["configc"], 4)
            combos = itertools.product(itertools.combinations(range(1, 128), 3), itertools.combinations(range(1, 32), 3))
            n, t0 = 0, time.perf_counter()
            for b, c in combos:
                pipeline_length(PipelinePlan(b, c, 1), renv.decode_metrics(b), renv.topo_norm)
                n += 1
                if n % 256 == 0 and time.perf_counter() - t0 > 3.0:
                    break
            out["cpu_baseline"] = {"value": n / (time.perf_counter() - t0), "unit": "points/s", "cores": 1,
                                   "kind": "reference", "sample": f"first {n} points of the same space"}
        except ImportError as exc:
            out["cpu_baseline"] = {"unavailable": f"baseline/_ref not importable: {exc}"}
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
                      "learn_to_env_step_ratio": "1:1", "semantics": "reference train_partition loop",
                      "driver": "host loop (search.train_partition): Python per step, kernels per call",
                      "precision": agent.net.precision}}
    # the same loop entirely on the device (devloop.train_partition_device): numpy's PCG64 stream on the
    # GPU, one CUDA graph with WHILE / IF nodes over whole episodes; bit-identical to the host loop
    from paper_2007_04069_b200 import devloop

    env_d = OppEnv(g, groups=groups)
    agent_d = DqnAgent(cfg, env_d.state_dim, env_d.num_actions, 0)
    devloop.train_partition_device(env_d, agent_d, 2)  # fills the ring past the first batch
    t0 = time.perf_counter()
    devloop.train_partition_device(env_d, agent_d, args.single_episodes)
    wall = time.perf_counter() - t0
    st = dict(devloop.last_stats)
    out["device_loop"] = {"value": st["steps"] / (st["device_ms"] / 1e3), "unit": "env-steps/s",
                          "steps": st["steps"], "episodes": args.single_episodes, "train_steps": st["train_steps"],
                          "graph_launches": st["launches"], "device_ms": st["device_ms"],
                          "wall_incl_capture_and_log_readback": st["steps"] / wall,
                          "driver": "devloop.train_partition_device (CUDA graph, conditional nodes)"}
    if want_cpu:
        out["cpu_baseline"] = cpu_dqn_single(g, args.workload, "opp", args.cpu_seconds)
    return out


def cpu_dqn_single(g, name, task, seconds):
    """The reference train_partition loop body (act / step / observe / learn) on one host core; the OPP
    env gets the reference linkage groups from the committed golden (skips its extraction)."""
    try:
        rir, rsh = _ref_import()
        from autoplan.agent import AgentConfig as RA
        from autoplan.agent import DqnAgent as RD
        from autoplan.agent import Transition as RT
        from autoplan.envs import AdpEnv as RAE
        from autoplan.envs import OppEnv as RO
        from autoplan.ir import decision_dims as rdd
        from autoplan.linkage import LinkageGroup as RL
    except ImportError as exc:
        return {"unavailable": f"baseline/_ref not importable: {exc}"}
    import numpy as np

    rg = rir.graph_from_dict(g.to_dict())
    if task == "opp":
        rdims = rdd(rg, rg.trainable_variables)
        z = np.load(GOLDEN / f"linkage_{name}.npz")
        rgroups = {}
        for k, d in enumerate(rdims):
            for s_i, st in enumerate((rsh.DimStatus.PARTITIONED, rsh.DimStatus.REPLICATED)):
                row = z["implied"][2 * k + s_i]
                implied = tuple((rdims[j], rsh.DimStatus(int(row[j]))) for j in np.flatnonzero(row != -1))
                rgroups[(d, st)] = RL((d, st), implied, bool(z["infeasible"][2 * k + s_i]))
        env = RO(rg, groups=rgroups)
    else:
        env = RAE(rg)
    agent = RD(RA(lr=0.0005, epsilon_decay_iters=500 if task == "adp" else 2000), env.state_dim, env.num_actions, 0)
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
            "sample": f"{n} reference train_partition steps on {name} {task.upper()} ({dt:.1f} s; includes the "
                      f"first, learn-free steps)"}


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
