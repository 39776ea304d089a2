"""Reference-side binding: the module a maintainer would add to the reference planner
(`autoplan/_b200.py`) to route `PropagationEngine.run` (reference sharding.py:210-248)
through the B200 engine's C-ABI (include/autoplan_b200.h) -- ctypes + numpy only, device
buffers from torch.  It does not import `paper_2007_04069_b200`: it is the FFI a non-B200
codebase writes against `libautoplan_b200.so`.

    from integration.autoplan_b200_binding import B200PropagationEngine
    engine = B200PropagationEngine(graph, candidates)      # graph: autoplan.ir.HloGraph
    result = engine.run({dim_index: DimStatus.PARTITIONED})  # autoplan.sharding.PropagationResult

Seeds are validated by the reference's own rules before the call (sharding.py:219-229);
the batched entry `run_batch(seed_rows)` returns (outcome, statuses) arrays.  CONFLICT
results carry the reference's exact partial snapshot and conflict site through
`ap_propagate_trace`, as the reference computes them.

Running this file checks the binding against the reference engine on the reference's own
zoo graphs (needs a GPU and the reference importable, e.g. from baseline/_ref):

    python integration/autoplan_b200_binding.py
"""

from __future__ import annotations

import ctypes
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
LIB_PATH = os.environ.get("AUTOPLAN_B200_LIB", str(ROOT / "paper_2007_04069_b200" / "libautoplan_b200.so"))

# enum ap_opcode (include/autoplan_b200.h), the reference vocabulary ir.py:33-68
OPCODES = {"parameter": 0, "constant": 1, "add": 2, "subtract": 3, "multiply": 4, "divide": 5, "exp": 6,
           "tanh": 7, "dot": 8, "reshape": 9, "transpose": 10, "broadcast": 11, "reduce": 12, "tuple": 13,
           "get-tuple-element": 14}
AP_OUTCOME_COMPLETE, AP_OUTCOME_INCOMPLETE, AP_OUTCOME_CONFLICT = 0, 1, 2
SEED_NONE, SEED_UNDECIDED = -1, 2


class GraphDesc(ctypes.Structure):
    _fields_ = [("num_instructions", ctypes.c_int32), ("opcode", ctypes.c_void_p), ("rank", ctypes.c_void_p),
                ("dims_offset", ctypes.c_void_p), ("dims", ctypes.c_void_p), ("operand_offset", ctypes.c_void_p),
                ("operands", ctypes.c_void_p), ("gte_element", ctypes.c_void_p)]


_VP, _I64, _I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(LIB_PATH)
        L.ap_graph_create.argtypes = [ctypes.POINTER(GraphDesc), ctypes.POINTER(_VP)]
        L.ap_graph_destroy.argtypes = [_VP]
        L.ap_decision_create.argtypes = [_VP, _VP, _VP, _I32, ctypes.POINTER(_VP)]
        L.ap_decision_destroy.argtypes = [_VP]
        L.ap_propagate_batch.argtypes = [_VP, _VP, _VP, _I64, _I64, _VP, _I64, _VP, _I64, _VP, _VP, _VP]
        L.ap_propagate_trace.argtypes = [_VP, _VP, _VP, _VP, _VP, _VP, _VP, _VP]
        L.ap_last_error.restype = ctypes.c_char_p
        _lib = L
    return _lib


def _check(rc: int, exc=RuntimeError):
    if rc != 0:
        raise exc(f"autoplan_b200 [{rc}]: {lib().ap_last_error().decode()}")


def compile_graph(graph):
    """ap_graph_create over a reference HloGraph: instructions in ascending id ("positions"),
    operands and get-tuple-element sources as positions (ir.py:199-384 semantics)."""
    from autoplan.ir import GraphValidationError

    instrs = sorted(graph.instructions, key=lambda i: i.id)
    pos = {ins.id: p for p, ins in enumerate(instrs)}
    rank = np.array([ins.shape.rank for ins in instrs], dtype=np.int32)
    dims_offset = np.zeros(len(instrs) + 1, dtype=np.int64)
    np.cumsum(rank, out=dims_offset[1:])
    dims = np.array([d for ins in instrs for d in ins.shape.dims] or [0], dtype=np.int64)
    nops = np.array([len(ins.operand_ids) for ins in instrs], dtype=np.int32)
    operand_offset = np.zeros(len(instrs) + 1, dtype=np.int32)
    np.cumsum(nops, out=operand_offset[1:])
    operands = np.array([pos[o] for ins in instrs for o in ins.operand_ids] or [0], dtype=np.int32)
    gte = np.full(len(instrs), -1, dtype=np.int32)
    for p, ins in enumerate(instrs):
        if ins.opcode == "get-tuple-element":
            tup = graph.instruction(ins.operand_ids[0])
            gte[p] = pos[tup.operand_ids[graph.tuple_element_index(ins)]]
    opcode = np.array([OPCODES[ins.opcode] for ins in instrs], dtype=np.int32)
    keep = (opcode, rank, dims_offset, dims, operand_offset, operands, gte)
    desc = GraphDesc(len(instrs), *[a.ctypes.data for a in keep])
    handle = ctypes.c_void_p()
    _check(lib().ap_graph_create(ctypes.byref(desc), ctypes.byref(handle)), GraphValidationError)
    return handle, instrs, dims_offset


class B200PropagationEngine:
    """`PropagationEngine(graph, candidates)` with `run` on the GPU (reference sharding.py:145-248)."""

    def __init__(self, graph, candidates=None):
        import torch

        self.graph = graph
        self.candidates = list(candidates) if candidates is not None else None
        self.handle, self.instrs, self.slot_offset = compile_graph(graph)
        self.pos = {ins.id: p for p, ins in enumerate(self.instrs)}
        self.num_slots = int(self.slot_offset[-1])
        self._dec = {}
        self.torch = torch

    def _slot(self, d) -> int:
        return int(self.slot_offset[self.pos[d.instruction_id]] + d.dim)

    def _decision(self, slots: tuple, is_cand: tuple):
        key = (slots, is_cand)
        if key not in self._dec:
            s = np.asarray(slots, dtype=np.int64)
            c = np.asarray(is_cand, dtype=np.uint8)
            h = ctypes.c_void_p()
            _check(lib().ap_decision_create(self.handle, s.ctypes.data, c.ctypes.data, len(s), ctypes.byref(h)))
            self._dec[key] = h
        return self._dec[key]

    def run(self, seeds):
        """One plan, the reference's return type (PropagationResult)."""
        from autoplan.ir import decision_dims
        from autoplan.sharding import (DimStatus, GraphValidationError, Outcome, PropagationResult,
                                       ShardingSpec)

        torch = self.torch
        cand = self.candidates
        if cand is None:
            cand = decision_dims(self.graph, {self.graph.instruction(d.instruction_id).name for d in seeds})
        # the reference validates seeds while applying them in (id, dim) order (sharding.py:219-229)
        for d in sorted(seeds, key=lambda x: (x.instruction_id, x.dim)):
            if d.instruction_id not in self.pos:
                raise GraphValidationError(f"seed references unknown instruction {d.instruction_id}")
            if d.dim >= self.graph.instruction(d.instruction_id).shape.rank:
                raise GraphValidationError(f"seed dim {d.dim} out of range for instruction {d.instruction_id}")
        cand_slots = [self._slot(d) for d in cand]
        seed_slots = {self._slot(d): int(v) for d, v in seeds.items()}
        slots = sorted(set(cand_slots) | set(seed_slots))
        where = {s: i for i, s in enumerate(slots)}
        cset = set(cand_slots)
        dec = self._decision(tuple(slots), tuple(1 if s in cset else 0 for s in slots))
        row = np.full(max(16, (len(slots) + 15) // 16 * 16), SEED_NONE, dtype=np.int8)
        for s, v in seed_slots.items():
            row[where[s]] = SEED_UNDECIDED if v == int(DimStatus.UNDECIDED) else v
        seeds_d = torch.from_numpy(row).cuda().view(1, -1)
        stride = max(16, (self.num_slots + 15) // 16 * 16)
        slots_d = torch.empty((1, stride), dtype=torch.int8, device="cuda")
        oc_d = torch.empty(1, dtype=torch.uint8, device="cuda")
        stream = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        _check(lib().ap_propagate_batch(self.handle, dec, seeds_d.data_ptr(), 1, row.size, slots_d.data_ptr(), stride,
                                        None, 0, oc_d.data_ptr(), None, stream))
        code = int(oc_d.item())
        site = None
        if code == AP_OUTCOME_CONFLICT:  # the reference's sweep-order snapshot and site
            st = np.empty(max(self.num_slots, 1), dtype=np.int8)
            out_code = np.zeros(1, dtype=np.int32)
            site_pos = np.zeros(1, dtype=np.int32)
            _check(lib().ap_propagate_trace(self.handle, dec, row.ctypes.data, None, st.ctypes.data,
                                            out_code.ctypes.data, site_pos.ctypes.data, stream))
            statuses = st[: self.num_slots]
            site = self.instrs[int(site_pos[0])].id if site_pos[0] >= 0 else None
        else:
            statuses = slots_d[0, : self.num_slots].cpu().numpy()
        assignments = {ins.id: ShardingSpec(tuple(int(statuses[self.slot_offset[p] + k])
                                                  for k in range(ins.shape.rank)), ins.shape.dims)
                       for p, ins in enumerate(self.instrs)}
        outcome = {AP_OUTCOME_COMPLETE: Outcome.COMPLETE, AP_OUTCOME_INCOMPLETE: Outcome.INCOMPLETE,
                   AP_OUTCOME_CONFLICT: Outcome.CONFLICT}[code]
        if outcome is Outcome.CONFLICT:
            return PropagationResult(outcome=outcome, assignments=assignments, conflict_site=site,
                                     newly_decided=())
        newly = tuple((d, DimStatus(int(statuses[s]))) for d, s in zip(cand, cand_slots)
                      if s not in seed_slots and statuses[s] != -1)
        return PropagationResult(outcome=outcome, assignments=assignments, conflict_site=None, newly_decided=newly)

    def close(self):
        for h in self._dec.values():
            lib().ap_decision_destroy(h)
        self._dec.clear()
        if self.handle:
            lib().ap_graph_destroy(self.handle)
            self.handle = None


def _selfcheck() -> int:
    """Reference engine vs the binding on the reference's zoo graphs, random seed sets."""
    ref = ROOT / "baseline" / "_ref"
    if ref.exists():
        sys.path.insert(0, str(ref))
    from autoplan import zoo
    from autoplan.ir import decision_dims
    from autoplan.sharding import DimStatus, PropagationEngine

    rng = np.random.default_rng(0)
    checked = 0
    for g in (zoo.attention_block(), zoo.t5_block(), zoo.vgg_classifier(), zoo.uniform_chain(length=12)):
        names = g.trainable_variables or [i.name for i in g.instructions if i.opcode == "parameter"]
        dims = decision_dims(g, names)
        ours, theirs = B200PropagationEngine(g, dims), PropagationEngine(g, dims)
        for _ in range(64):
            k = int(rng.integers(1, len(dims) + 1))
            pick = rng.permutation(len(dims))[:k]
            seeds = {dims[j]: (DimStatus.PARTITIONED if rng.random() < 0.5 else DimStatus.REPLICATED) for j in pick}
            a, b = ours.run(seeds), theirs.run(seeds)
            assert a.outcome == b.outcome and a.conflict_site == b.conflict_site, (a.outcome, b.outcome)
            assert a.newly_decided == b.newly_decided
            assert {i: s.statuses for i, s in a.assignments.items()} == \
                   {i: s.statuses for i, s in b.assignments.items()}
            checked += 1
        ours.close()
    print(f"binding == reference PropagationEngine.run on {checked} plans")
    return 0


if __name__ == "__main__":
    sys.exit(_selfcheck())
