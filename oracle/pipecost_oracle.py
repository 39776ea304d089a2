"""CPU ORACLE for the pipeline cost model — test infrastructure only.

Pure-Python restatement of the reference's fp64 cost arithmetic, each
function following the cited reference lines (pkg/src/autoplan/...):
Python floats are IEEE binary64 and builtin `sum` is the CPython 3.12
compensated sum, so the restatement is bit-exact by construction when it
keeps the reference's evaluation order.  Pinned by tests/test_pipe_oracle.py
against tests/golden/pipe_*.npz and infer_*.npz.  Only tests/ may import it.
"""

from __future__ import annotations

import bisect
import math


def forward_tables(graph):
    """Forward order, positions, costs, sizes, forward consumers (pipecost.py:91-93, ir.py:464-470)."""
    order = [i for i in graph.topological_order if graph.instruction(i).is_forward]
    pos = {iid: p for p, iid in enumerate(order)}
    return order, pos


def stage_metrics(graph, pivots, backward_multiplier=2.0):
    """pipecost.py:72-141."""
    order, pos = forward_tables(graph)
    cuts = [pos[p] for p in pivots]
    k = len(cuts) + 1
    compute = [0.0] * k
    for i, iid in enumerate(order):
        compute[bisect.bisect_left(cuts, i)] += graph.instruction(iid).compute_cost_ms or 0.0
    activation = [0.0] * k
    for s, cut in enumerate(cuts):
        total = 0.0
        for i in range(cut + 1):
            iid = order[i]
            if any(pos.get(c, -1) > cut for c in graph.consumers(iid) if graph.instruction(c).is_forward):
                total += graph.instruction(iid).shape.byte_size
        activation[s] = total
    params = [0.0] * k
    nvars = [0] * k
    for vid in graph.trainable_ids():
        firsts = [pos[c] for c in graph.consumers(vid) if graph.instruction(c).is_forward and c in pos]
        if firsts:
            stage = bisect.bisect_left(cuts, min(firsts))
        else:
            stage = bisect.bisect_left(cuts, pos[vid]) if vid in pos else 0
        params[stage] += graph.instruction(vid).shape.byte_size
        nvars[stage] += 1
    scale = 1.0 + backward_multiplier
    return [(compute[s] * scale, activation[s], params[s], nvars[s]) for s in range(k)]


def proportional_counts(compute, d):
    """pipecost.py:207-237."""
    k = len(compute)
    total = sum(compute)
    quotas = [d / k] * k if total <= 0 else [d * c / total for c in compute]
    counts = [int(q) for q in quotas]
    rem = d - sum(counts)
    for i in sorted(range(k), key=lambda i: (-(quotas[i] - counts[i]), i))[:rem]:
        counts[i] += 1
    while 0 in counts:
        poor = counts.index(0)
        rich = max(range(k), key=lambda i: (counts[i], -i))
        counts[rich] -= 1
        counts[poor] = 1
    return counts


def bandwidth(topo, a, b):
    """topology.py:49-54 (a != b here)."""
    ga = a // topo["g"]
    gb = b // topo["g"]
    return topo["intra"] if ga == gb else topo["inter"]


def allreduce(topo, nbytes, start, end):
    """topology.py:131-148."""
    n = end - start
    if n <= 1 or nbytes == 0:
        return 0.0
    slow = min(bandwidth(topo, start + i, start + (i + 1) % n) for i in range(n))
    return 2.0 * (n - 1) / n * nbytes / slow


def groups_of(cuts, d):
    edges = [0, *cuts, d]
    return list(zip(edges[:-1], edges[1:]))


def pipeline_length(metrics, cuts, m, topo):
    """pipecost.py:144-176 (metrics = [(compute_ms, act, param, nvars)])."""
    groups = groups_of(cuts, topo["d"])
    times = [c[0] / 1000.0 / (e - s) for c, (s, e) in zip(metrics, groups)]
    transfers = [metrics[i][1] / bandwidth(topo, groups[i][1] - 1, groups[i + 1][0]) for i in range(len(groups) - 1)]
    reduces = [allreduce(topo, c[2], s, e) for c, (s, e) in zip(metrics, groups)]
    return (m - 1) * max(times) + sum(times) + sum(transfers) + max(reduces)


def memory_feasible(metrics, cuts, m, topo, mem, opt=4.0):
    """pipecost.py:179-204."""
    for s, (a, b) in enumerate(groups_of(cuts, topo["d"])):
        n = b - a
        act_in = metrics[s - 1][1] if s > 0 else 0.0
        if metrics[s][2] / n * opt + m * (act_in + metrics[s][1]) / n > mem:
            return False
    return True


def topo_dict(num_servers, gpus, intra, inter):
    return {"g": int(gpus), "d": int(num_servers) * int(gpus), "intra": float(intra), "inter": float(inter)}


def decode_length(arrays_c, arrays_a, arrays_w, boundaries, cuts, m, topo_norm, granularity=128):
    """envs.py:593-616 decode + pipecost.pipeline_length on the normalised topology."""
    edges = [0, *boundaries, granularity]
    metrics = []
    for lo, hi in zip(edges[:-1], edges[1:]):
        comp = arrays_c[hi - 1] - (arrays_c[lo - 1] if lo > 0 else 0.0)
        par = arrays_w[hi - 1] - (arrays_w[lo - 1] if lo > 0 else 0.0)
        act = arrays_a[hi - 1] if hi < granularity else 0.0
        metrics.append((comp * 1000.0, act, par, 0))
    return pipeline_length(metrics, list(cuts), m, topo_norm)


def sqrt_reward(length):
    return 1.0 / math.sqrt(length)
