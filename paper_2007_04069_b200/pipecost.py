"""Pipeline stage construction and the GPipe length model, evaluated on the GPU.

Public names follow reference `autoplan.pipecost` (`pipecost.py:21-336`).
Per-graph tables (forward order, crossing activations, parameter
ownership) are compiled once into an `ap_pipe` handle; every evaluation —
stage metrics, proportional device allocation, pipeline length, memory
check, pivot pruning — runs in `csrc/pipecost.cu`, bit-exact with the
reference's fp64 arithmetic (CPython 3.12 `sum()`, naive stage sums,
left-to-right association).  Small calls (one plan) pay
one launch + sync; batch through the `*_batch` functions or the
environments.
"""

from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass
from typing import Sequence

import numpy as np

from . import _native
from .ir import forward_subgraph


class InfeasiblePlanError(Exception):
    """A plan or configuration cannot be realized on the topology."""


@dataclass(frozen=True)
class StageMetrics:
    compute_ms: float
    activation_bytes: float
    param_bytes: float
    num_variables: int = 0


@dataclass(frozen=True)
class PipelinePlan:
    pivot_ids: tuple[int, ...]
    device_cuts: tuple[int, ...]
    micro_batches: int = 1
    micro_batch_size: int = 16

    def __post_init__(self) -> None:
        if len(self.pivot_ids) != len(self.device_cuts):
            raise InfeasiblePlanError("plan needs one device cut per pivot")
        if self.micro_batches < 1:
            raise InfeasiblePlanError("micro_batches must be >= 1")

    @property
    def num_stages(self) -> int:
        return len(self.pivot_ids) + 1


def device_groups(device_cuts: Sequence[int], num_devices: int) -> list[tuple[int, int]]:
    """Contiguous half-open device groups split at the cuts (pipecost.py:61-69)."""
    cuts = list(device_cuts)
    if any(b <= a for a, b in zip(cuts, cuts[1:])):
        raise InfeasiblePlanError("device cuts must be strictly increasing")
    if cuts and (cuts[0] < 1 or cuts[-1] > num_devices - 1):
        raise InfeasiblePlanError("device cuts must lie strictly inside (0, D)")
    edges = [0, *cuts, num_devices]
    return list(zip(edges[:-1], edges[1:]))


# -- per-graph device model -------------------------------------------------------


class PipeModel:
    """Forward-order tables of one graph as an `ap_pipe` handle."""

    def __init__(self, graph):
        self.graph = graph
        order = forward_subgraph(graph)
        if not order:
            raise InfeasiblePlanError("graph has no forward instructions")
        self.order = order
        self.pos = {iid: p for p, iid in enumerate(order)}
        F = len(order)
        cost = np.zeros(F, dtype=np.float64)
        nbytes = np.zeros(F, dtype=np.int64)
        last_use = np.full(F, -1, dtype=np.int32)
        for p, iid in enumerate(order):
            ins = graph.instruction(iid)
            cost[p] = ins.compute_cost_ms or 0.0
            nbytes[p] = ins.shape.byte_size
            uses = [self.pos[c] for c in graph.consumers(iid) if graph.instruction(c).is_forward]
            if uses:
                last_use[p] = max(uses)
        anchors, vbytes = [], []
        for vid in graph.trainable_ids():
            firsts = [self.pos[c] for c in graph.consumers(vid) if graph.instruction(c).is_forward and c in self.pos]
            if firsts:
                anchors.append(min(firsts))
            else:
                anchors.append(self.pos.get(vid, -1))
            vbytes.append(graph.instruction(vid).shape.byte_size)
        self.cost = cost
        self._keep = [cost, nbytes, last_use, np.asarray(anchors or [0], dtype=np.int32),
                      np.asarray(vbytes or [0], dtype=np.int64)]
        desc = _native.PipeDesc(F, cost.ctypes.data, nbytes.ctypes.data, last_use.ctypes.data, len(anchors),
                                self._keep[3].ctypes.data, self._keep[4].ctypes.data)
        lib = _native.load_library()
        handle = ctypes.c_void_p()
        _native.check(lib.ap_pipe_create(ctypes.byref(desc), ctypes.byref(handle)))
        self.handle = handle
        self.num_forward = F
        self._bound = {}

    def bind_candidates(self, cand_pos_dev) -> bool:
        """Stage-sum table for a device candidate list (ap_pipe_train_table).

        The tensor is kept alive with the handle, so its address (the table's
        key) cannot be reused by another list.  False when the table would be
        too large; ap_pipe_train_state then sweeps the cost array per candidate.
        """
        key = (cand_pos_dev.data_ptr(), cand_pos_dev.numel())
        if key in self._bound:
            return True
        rc = _native.load_library().ap_pipe_train_table(self.handle, _native.ptr(cand_pos_dev),
                                                         cand_pos_dev.numel(), _native.stream_handle())
        if rc == _native.AP_ERR_UNSUPPORTED:
            return False
        _native.check(rc)
        self._bound[key] = cand_pos_dev
        return True

    def positions(self, pivots: Sequence[int]) -> list[int]:
        out = []
        for p in pivots:
            if p not in self.pos:
                raise InfeasiblePlanError(f"pivot {p} is not a forward instruction")
            out.append(self.pos[p])
        if any(b <= a for a, b in zip(out, out[1:])):
            raise InfeasiblePlanError("pivots must be strictly increasing in forward order")
        return out

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _native._lib is not None:
            _native._lib.ap_pipe_destroy(h)
            self.handle = None


_MODELS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def pipe_model(graph) -> PipeModel:
    m = _MODELS.get(graph)
    if m is None:
        m = PipeModel(graph)
        _MODELS[graph] = m
    return m


# -- batched device entry points ----------------------------------------------------


def stage_metrics_batch(graph, pivot_positions, backward_multiplier: float = 2.0):
    """Device tensors (compute, act, param [B, P+1] fp64, nvars int32) for forward-position pivots [B, P]."""
    import torch

    model = pipe_model(graph)
    piv = torch.as_tensor(pivot_positions, dtype=torch.int32).cuda()
    if piv.dim() == 1:
        piv = piv.view(1, -1)
    piv = piv.contiguous()
    b, p = piv.shape
    out = [torch.empty((b, p + 1), dtype=torch.float64, device="cuda") for _ in range(3)]
    nvars = torch.empty((b, p + 1), dtype=torch.int32, device="cuda")
    lib = _native.require_device()
    _native.check(lib.ap_pipe_metrics(model.handle, _native.ptr(piv) if p else None, b, p, float(backward_multiplier),
                                      *[_native.ptr(t) for t in out], _native.ptr(nvars), _native.stream_handle()))
    return out[0], out[1], out[2], nvars


def pipeline_length_batch(topo, compute, act, param, micro_batches: int, cuts=None,
                          mem_per_device: float | None = None, optimizer_multiplier: float = 4.0,
                          python_floats: bool = True):
    """Device (length [B] fp64, feasible [B] uint8, cuts [B, K-1] int32) from per-stage metrics [B, K].

    With `cuts=None` the proportional allocation (pipecost.py:218-252) is
    computed and returned.  `python_floats` mirrors the reference's builtin
    sum() behaviour: compensated for Python floats, naive for numpy scalars.
    """
    import torch

    # keep every contiguous temporary alive until the launch is enqueued
    compute, act, param = compute.contiguous(), act.contiguous(), param.contiguous()
    b, k = compute.shape
    given = cuts is not None
    if given:
        cuts_t = torch.as_tensor(cuts, dtype=torch.int32).cuda().view(b, k - 1).contiguous()
    else:
        cuts_t = torch.empty((b, max(k - 1, 1)), dtype=torch.int32, device="cuda")
    length = torch.empty(b, dtype=torch.float64, device="cuda")
    feas = torch.empty(b, dtype=torch.uint8, device="cuda")
    lib = _native.require_device()
    topo_c = _native.Topology.of(topo)
    _native.check(lib.ap_pipe_length(ctypes.byref(topo_c), k, int(micro_batches), b, _native.ptr(compute),
                                     _native.ptr(act), _native.ptr(param), _native.ptr(cuts_t), int(given),
                                     -1.0 if mem_per_device is None else float(mem_per_device),
                                     float(optimizer_multiplier), int(bool(python_floats)), _native.ptr(length),
                                     _native.ptr(feas), _native.stream_handle()))
    return length, feas, cuts_t[:, : k - 1]


def _metrics_tensors(metrics: Sequence[StageMetrics]):
    import torch

    arr = np.array([[m.compute_ms, m.activation_bytes, m.param_bytes] for m in metrics], dtype=np.float64)
    t = torch.from_numpy(arr).cuda()
    return t[:, 0].reshape(1, -1), t[:, 1].reshape(1, -1), t[:, 2].reshape(1, -1)


def _python_floats(metrics: Sequence[StageMetrics]) -> bool:
    """True when CPython's sum() would take its float fast path (exact `float` values)."""
    return type(metrics[0].compute_ms) is float


# -- reference API --------------------------------------------------------------------


def stage_metrics(graph, pivots: Sequence[int], backward_multiplier: float = 2.0) -> list[StageMetrics]:
    """Per-stage compute / activation / parameter costs (pipecost.py:72-141)."""
    model = pipe_model(graph)
    positions = model.positions(pivots)
    comp, act, param, nvars = stage_metrics_batch(graph, [positions], backward_multiplier)
    comp, act, param, nvars = (t[0].cpu().numpy() for t in (comp, act, param, nvars))
    return [StageMetrics(float(c), float(a), float(w), int(v)) for c, a, w, v in zip(comp, act, param, nvars)]


def pipeline_length(plan: PipelinePlan, metrics: Sequence[StageMetrics], topo) -> float:
    """GPipe length (M-1)*max(t) + sum(t) + sum(transfers) + max(allreduce) (pipecost.py:144-176)."""
    if len(metrics) != plan.num_stages:
        raise InfeasiblePlanError("metrics do not match the plan's stage count")
    device_groups(plan.device_cuts, topo.num_devices)
    c, a, w = _metrics_tensors(metrics)
    length, _, _ = pipeline_length_batch(topo, c, a, w, plan.micro_batches, cuts=[list(plan.device_cuts)],
                                         python_floats=_python_floats(metrics))
    return float(length[0].item())


def memory_feasible(plan: PipelinePlan, metrics: Sequence[StageMetrics], topo, mem_per_device: float,
                    optimizer_multiplier: float = 4.0) -> bool:
    """Every device fits params x optimizer multiplier plus its activation working set (pipecost.py:179-204)."""
    device_groups(plan.device_cuts, topo.num_devices)
    if len(metrics) != plan.num_stages:
        raise InfeasiblePlanError("metrics do not match the plan's stage count")
    c, a, w = _metrics_tensors(metrics)
    _, feas, _ = pipeline_length_batch(topo, c, a, w, plan.micro_batches, cuts=[list(plan.device_cuts)],
                                       mem_per_device=mem_per_device, optimizer_multiplier=optimizer_multiplier)
    return bool(feas[0].item())


def proportional_device_counts(compute_ms: Sequence[float], num_devices: int) -> list[int]:
    """Devices per stage proportional to compute, largest remainder, min 1 (pipecost.py:218-237)."""
    import torch

    k = len(compute_ms)
    if k > num_devices:
        raise InfeasiblePlanError(f"{k} stages need more than {num_devices} devices")
    from .topology import DeviceTopology

    topo = DeviceTopology(1, num_devices)
    c = torch.tensor([list(map(float, compute_ms))], dtype=torch.float64, device="cuda")
    z = torch.zeros_like(c)
    _, _, cuts = pipeline_length_batch(topo, c, z, z, 1)
    edges = [0, *cuts[0].tolist(), num_devices]
    return [b - a for a, b in zip(edges[:-1], edges[1:])]


def proportional_device_cuts(metrics: Sequence[StageMetrics], topo) -> tuple[int, ...]:
    counts = proportional_device_counts([m.compute_ms for m in metrics], topo.num_devices)
    return tuple(int(x) for x in np.cumsum(counts)[:-1])


def allowed_device_cuts(topo, radius: int) -> list[int]:
    """Device cuts within `radius` of a server boundary (pipecost.py:255-268)."""
    if radius < 0:
        raise ValueError("radius must be >= 0")
    d, g = topo.num_devices, topo.gpus_per_server
    keep: set[int] = set()
    for m in range(g, d, g):
        keep.update(range(max(1, m - radius), min(d - 1, m + radius) + 1))
    return sorted(keep)


def two_stage_device_cut(prefix_compute: float, suffix_compute: float, topo) -> int:
    return proportional_device_counts([prefix_compute, suffix_compute], topo.num_devices)[0]


def candidate_pivots(graph, topo, num_stages: int, radius: int) -> list[int]:
    """Pruned pivot candidates (pipecost.py:279-336), evaluated by the device pruning kernel."""
    import torch

    if num_stages < 2:
        raise InfeasiblePlanError("pipeline planning needs at least two stages")
    if num_stages > topo.num_devices:
        raise InfeasiblePlanError("more stages than devices")
    if len(forward_subgraph(graph)) < 2:
        raise InfeasiblePlanError("graph is too small to cut")
    if radius < 0:
        raise ValueError("radius must be >= 0")
    model = pipe_model(graph)
    allowed = torch.empty(model.num_forward - 1, dtype=torch.uint8, device="cuda")
    lib = _native.require_device()
    topo_c = _native.Topology.of(topo)
    _native.check(lib.ap_pipe_candidates(model.handle, ctypes.byref(topo_c), int(num_stages), int(radius),
                                         _native.ptr(allowed), _native.stream_handle()))
    keep = np.flatnonzero(allowed.cpu().numpy())
    kept = [model.order[int(i)] for i in keep]
    if len(kept) < num_stages - 1:
        raise InfeasiblePlanError(
            f"only {len(kept)} candidate pivots for {num_stages} stages; the configuration is infeasible at this radius"
        )
    return kept
