"""Digest an `ncu --set full` report into a small JSON record (run on the GPU box, where the
.ncu-rep files are too large to bring back).

    python profiles/probes/ncu_digest.py REPORT.ncu-rep NAME [--units N] > out.json

Keeps: duration, DRAM bytes, throughput / occupancy / IPC, registers, executed instructions,
the per-pipe utilisations and the warp-stall mix; `--units N` adds per-unit figures (bytes and
warp instructions per plan / candidate / step).
"""

import csv
import io
import json
import subprocess
import sys

WANT = {
    "duration_s": "gpu__time_duration.sum",
    "dram_bytes_read": "dram__bytes_read.sum",
    "dram_bytes_write": "dram__bytes_write.sum",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "ipc": "sm__inst_executed.avg.per_cycle_active",
    "warp_instructions": "smsp__inst_executed.sum",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "smem_per_block_bytes": "launch__shared_mem_per_block_dynamic",
}


def main():
    rep, name = sys.argv[1], sys.argv[2]
    units = None
    if "--units" in sys.argv:
        units = float(sys.argv[sys.argv.index("--units") + 1])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, unit_row, vals = rows[0], rows[1], rows[2]
    col = {h: i for i, h in enumerate(hdr)}

    scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Kbyte/block": 1e3, "byte/block": 1.0}

    def num(h):
        v = vals[col[h]].replace(",", "")
        try:
            x = float(v)
        except ValueError:
            return v
        return x * scale.get(unit_row[col[h]], 1.0)

    out = {"name": name, "kernel": vals[col.get("Kernel Name", 0)]}
    for k, h in WANT.items():
        if h in col:
            out[k] = num(h)
    pipes = {}
    for h in hdr:
        if h.startswith("sm__pipe_") and h.endswith("cycles_active.avg.pct_of_peak_sustained_active"):
            v = num(h)
            if isinstance(v, float) and v > 1.0:
                pipes[h[len("sm__pipe_"):-len("_cycles_active.avg.pct_of_peak_sustained_active")]] = v
        if h.startswith("sm__inst_executed_pipe_") and h.endswith("avg.pct_of_peak_sustained_active"):
            v = num(h)
            if isinstance(v, float) and v > 1.0:
                pipes["inst_" + h[len("sm__inst_executed_pipe_"):-len(".avg.pct_of_peak_sustained_active")]] = v
    out["pipes_pct"] = dict(sorted(pipes.items(), key=lambda kv: -kv[1])[:10])
    stalls = {}
    for h in hdr:
        pre = "smsp__pcsamp_warps_issue_stalled_"
        if h.startswith(pre) and "not_issued" not in h:
            v = num(h)
            if isinstance(v, float):
                stalls[h[len(pre):]] = v
    tot = sum(stalls.values()) or 1.0
    out["stall_pct"] = {k: round(100 * v / tot, 1) for k, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:8]}
    if units:
        out["units"] = units
        for k in ("dram_bytes_read", "dram_bytes_write", "warp_instructions"):
            if isinstance(out.get(k), float):
                out[k + "_per_unit"] = out[k] / units
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
