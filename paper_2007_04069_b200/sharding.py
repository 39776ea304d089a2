"""Sharding propagation: the reference API, evaluated by the CUDA engine.

Public names and semantics follow reference `autoplan.sharding`
(`pkg/src/autoplan/sharding.py:36-392`): the three-valued `DimStatus`
lattice, `Outcome`, `ShardingSpec`, `PropagationResult`,
`PropagationEngine(graph, candidates).run(seeds)`, `propagate` and
`rule_for`.  The work is done on the GPU:

* `PropagationEngine` compiles the graph once per (graph, device) into the
  engine's link-class tables (`ap_graph_create`) — the reference rebuilds
  its rule table on every `propagate` call (`sharding.py:305-311`);
* `run` / `run_batch` launch the batched closure kernel
  (`ap_propagate_batch`, one warp per plan);
* for CONFLICT results of the single-plan API the reference's partial
  `assignments` snapshot and `conflict_site` depend on its sweep order;
  they are reproduced exactly by the engine's ordered replay
  (`ap_propagate_trace`).
"""

from __future__ import annotations

import weakref
from collections.abc import Mapping as _MappingABC
from dataclasses import dataclass
from enum import Enum, IntEnum
from typing import Iterable, Iterator, Mapping, Sequence

import numpy as np

from . import _native
from .ir import (
    ELEMENTWISE_BINARY,
    ELEMENTWISE_UNARY,
    DimIndex,
    GraphValidationError,
    HloGraph,
    Instruction,
    TensorShape,
    decision_dims,
    pair_broadcast,
    pair_reduce,
    pair_reshape,
)


class DimStatus(IntEnum):
    PARTITIONED = 1
    REPLICATED = 0
    UNDECIDED = -1


class Outcome(Enum):
    COMPLETE = "complete"
    INCOMPLETE = "incomplete"
    CONFLICT = "conflict"


_OUTCOME_OF_CODE = {
    _native.OUTCOME_COMPLETE: Outcome.COMPLETE,
    _native.OUTCOME_INCOMPLETE: Outcome.INCOMPLETE,
    _native.OUTCOME_CONFLICT: Outcome.CONFLICT,
}
_P, _R, _U = 1, 0, -1
SEED_NONE = -1
SEED_UNDECIDED = 2


def unpack_slots2(packed, num_slots: int) -> np.ndarray:
    """Decode ap_pack_slots2 rows ([B, >= ceil(n/4)] uint8) to int8 statuses [B, n] (-1 / 0 / 1)."""
    p = np.asarray(packed, dtype=np.uint8)
    codes = (p[:, :, None] >> np.array([0, 2, 4, 6], dtype=np.uint8)) & 3
    return codes.reshape(p.shape[0], -1)[:, :num_slots].astype(np.int8) - 1


def pad16(n: int) -> int:
    """Row stride (bytes) of seed / status rows: 16-byte multiple for vector loads and stores."""
    return max(16, (n + 15) // 16 * 16)


@dataclass(frozen=True)
class ShardingSpec:
    """Per-dim statuses of one tensor, optionally with its extents."""

    statuses: tuple[int, ...]
    dims: tuple[int, ...] | None = None

    def __post_init__(self) -> None:
        if self.dims is not None and len(self.dims) != len(self.statuses):
            raise ValueError("statuses and dims must have equal length")
        if list(self.statuses).count(_P) > 1:
            raise ValueError("at most one dim of a tensor can be partitioned")

    @classmethod
    def undecided(cls, rank: int, dims: tuple[int, ...] | None = None) -> "ShardingSpec":
        return cls(statuses=(_U,) * rank, dims=dims)

    @property
    def rank(self) -> int:
        return len(self.statuses)

    @property
    def partition_dim(self) -> int | None:
        return self.statuses.index(_P) if _P in self.statuses else None

    @property
    def is_fully_decided(self) -> bool:
        return _U not in self.statuses


@dataclass(frozen=True)
class PropagationResult:
    outcome: Outcome
    assignments: Mapping[int, ShardingSpec]
    conflict_site: int | None
    newly_decided: tuple[tuple[DimIndex, DimStatus], ...]


class SlotAssignments(_MappingABC):
    """`assignments` view over a flat slot-status vector.

    Behaves like the reference's `{instruction_id: ShardingSpec}` dict but
    builds a spec only when one is looked up.
    """

    __slots__ = ("_statuses", "_engine")

    def __init__(self, statuses: np.ndarray, engine: "_GraphEngine"):
        self._statuses = statuses
        self._engine = engine

    def __getitem__(self, instruction_id: int) -> ShardingSpec:
        pos = self._engine.pos_of_id.get(instruction_id)
        if pos is None:
            raise KeyError(instruction_id)
        lo, hi = self._engine.slot_offset[pos], self._engine.slot_offset[pos + 1]
        return ShardingSpec(tuple(int(v) for v in self._statuses[lo:hi]), self._engine.dims_of[pos])

    def __iter__(self) -> Iterator[int]:
        return iter(self._engine.ids)

    def __len__(self) -> int:
        return len(self._engine.ids)

    def status(self, instruction_id: int, dim: int) -> int:
        return int(self._statuses[self._engine.slot_offset[self._engine.pos_of_id[instruction_id]] + dim])

    @property
    def flat(self) -> np.ndarray:
        return self._statuses


# -- per-graph device engine cache ---------------------------------------------


class _GraphEngine:
    """Host metadata plus per-device tables of one graph."""

    def __init__(self, graph):
        self.graph = graph
        self.flat = graph.flat() if hasattr(graph, "flat") else _flatten(graph)
        self.ids = [int(i) for i in self.flat.ids]
        self.pos_of_id = {i: p for p, i in enumerate(self.ids)}
        self.slot_offset = self.flat.slot_offset
        instrs = sorted(graph.instructions, key=lambda ins: ins.id)
        self.dims_of = [tuple(ins.shape.dims) for ins in instrs]
        self.num_slots = self.flat.num_slots
        self._device: dict[int, _native.DeviceGraph] = {}

    def device(self, index: int | None = None) -> _native.DeviceGraph:
        import torch

        _native.require_device()
        idx = torch.cuda.current_device() if index is None else index
        dev = self._device.get(idx)
        if dev is None:
            dev = _native.DeviceGraph(self.flat, idx)
            self._device[idx] = dev
        return dev

    def slot(self, instruction_id: int, dim: int) -> int:
        return int(self.slot_offset[self.pos_of_id[instruction_id]] + dim)


def _flatten(graph):
    from .ir import flatten

    return flatten(graph)


_ENGINES: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def graph_engine(graph) -> _GraphEngine:
    eng = _ENGINES.get(graph)
    if eng is None:
        eng = _GraphEngine(graph)
        _ENGINES[graph] = eng
    return eng


# -- the engine ----------------------------------------------------------------


class PropagationEngine:
    """Reusable propagation over a fixed graph and candidate set.

    Same constructor and `run` contract as reference `PropagationEngine`
    (`sharding.py:145-248`).  `run_batch` is the batched device entry point.
    """

    def __init__(self, graph, candidates: Sequence[DimIndex] | None = None):
        self.graph = graph
        self.candidates = list(candidates) if candidates is not None else None
        self._eng = graph_engine(graph)

    # seeds -> decision set -------------------------------------------------------

    def _candidate_dims(self, seeds: Mapping[DimIndex, DimStatus]) -> list[DimIndex]:
        if self.candidates is not None:
            return self.candidates
        names = {self.graph.instruction(d.instruction_id).name for d in seeds}
        return decision_dims(self.graph, names)

    def _validate_seeds(self, seeds: Mapping[DimIndex, DimStatus]) -> list[tuple[int, int, int]]:
        """(instruction_id, dim, value) in application order, validated like the reference.

        The reference checks seeds while applying them in (id, dim) order and
        stops at the first seeding conflict, so a bad seed after a conflicting
        one is never inspected (`sharding.py:219-231`).  Seeding conflicts
        are decidable here: a slot is decided at seeding time only if it is
        forced replicated or pinned by an earlier partitioned seed of the
        same tensor.
        """
        eng = self._eng
        out: list[tuple[int, int, int]] = []
        pinned: dict[int, int] = {}
        forced = self._forced_slots()
        for d in sorted(seeds, key=lambda x: (x.instruction_id, x.dim)):
            tid, dim = d.instruction_id, d.dim
            pos = eng.pos_of_id.get(tid)
            if pos is None:
                raise GraphValidationError(f"seed references unknown instruction {tid}")
            rank = int(eng.slot_offset[pos + 1] - eng.slot_offset[pos])
            if dim >= rank:
                raise GraphValidationError(f"seed dim {dim} out of range for instruction {tid}")
            value = int(seeds[d])
            out.append((tid, dim, value))
            slot = eng.slot(tid, dim)
            decided = forced[slot] or (tid in pinned and pinned[tid] != dim)
            if decided and value != _R:
                break  # CONFLICT while seeding: later seeds are never looked at
            if value == _P:
                if tid in pinned:
                    break
                pinned[tid] = dim
        return out

    def _forced_slots(self) -> np.ndarray:
        eng = self._eng
        if not hasattr(eng, "_forced"):
            forced = np.zeros(eng.num_slots, dtype=bool)
            for s in _forced_slot_list(eng):
                forced[s] = True
            eng._forced = forced
        return eng._forced

    def _decision_for(self, cand: Sequence[DimIndex], extra: Iterable[tuple[int, int]] = ()):
        eng = self._eng
        cand_slots = [eng.slot(d.instruction_id, d.dim) for d in cand]
        slots = sorted(set(cand_slots) | {eng.slot(t, dd) for t, dd in extra})
        pos = {s: i for i, s in enumerate(slots)}
        is_cand = np.zeros(len(slots), dtype=np.uint8)
        for s in cand_slots:
            is_cand[pos[s]] = 1
        dev = eng.device()
        return dev, dev.decision(np.asarray(slots, dtype=np.int64), is_cand), pos, cand_slots

    # single plan ------------------------------------------------------------------

    def run(self, seeds: Mapping[DimIndex, DimStatus]) -> PropagationResult:
        import torch

        applied = self._validate_seeds(seeds)
        cand = self._candidate_dims(seeds)
        eng = self._eng
        dev, dec, pos, cand_slots = self._decision_for(cand, ((t, d) for t, d, _ in applied))
        # seeds after a seeding conflict are never applied (nor validated) by
        # the reference; the conflicting seed itself is the last applied one
        row = np.full(pad16(dec.n), SEED_NONE, dtype=np.int8)
        for t, d, v in applied:
            row[pos[eng.slot(t, d)]] = SEED_UNDECIDED if v == _U else v
        seeded_slots = {eng.slot(t, d) for t, d, _ in applied}
        with torch.cuda.device(dev.device_index):
            seeds_d = torch.from_numpy(row).cuda().view(1, -1)
            slots_d = torch.empty((1, self.slots_stride), dtype=torch.int8, device="cuda")
            outcome_d = torch.empty(1, dtype=torch.uint8, device="cuda")
            lib = _native.require_device()
            _native.check(
                lib.ap_propagate_batch(dev.handle, dec.handle, _native.ptr(seeds_d), 1, len(row),
                                       _native.ptr(slots_d), slots_d.shape[1], None, 0, _native.ptr(outcome_d),
                                       None, _native.stream_handle())
            )
            code = int(outcome_d.item())
            statuses = slots_d[0, : eng.num_slots].cpu().numpy()
            site = None
            if code == _native.OUTCOME_CONFLICT:
                statuses = np.empty(max(eng.num_slots, 1), dtype=np.int8)
                out_code = np.zeros(1, dtype=np.int32)
                site_pos = np.zeros(1, dtype=np.int32)
                _native.check(
                    lib.ap_propagate_trace(dev.handle, dec.handle, _native.ptr(row), None, _native.ptr(statuses),
                                           _native.ptr(out_code), _native.ptr(site_pos), _native.stream_handle())
                )
                statuses = statuses[: eng.num_slots]
                site = eng.ids[int(site_pos[0])] if site_pos[0] >= 0 else None
        assignments = SlotAssignments(statuses, eng)
        outcome = _OUTCOME_OF_CODE[code]
        if outcome is Outcome.CONFLICT:
            return PropagationResult(outcome, assignments, site, ())
        newly = tuple(
            (d, DimStatus(int(statuses[s])))
            for d, s in zip(cand, cand_slots)
            if s not in seeded_slots and statuses[s] != _U
        )
        return PropagationResult(outcome, assignments, None, newly)

    # batched --------------------------------------------------------------------

    def prepare(self):
        """Device graph + decision set for the candidate list (identity column order required)."""
        if self.candidates is None:
            raise ValueError("batched propagation needs an explicit candidate list")
        cached = self.__dict__.get("_prepared")
        if cached is not None and cached[0] is self.candidates:  # validated once per candidate list
            return cached[1], cached[2]
        dev, dec, pos, cand_slots = self._decision_for(self.candidates)
        if any(pos[s] != k for k, s in enumerate(cand_slots)):
            raise ValueError("launch() needs candidates in ascending (instruction id, dim) order")
        self.__dict__["_prepared"] = (self.candidates, dev, dec)
        return dev, dec

    @property
    def slots_stride(self) -> int:
        """Row stride of slot outputs: |S| rounded up to 16 bytes (vectorised stores)."""
        return max(16, (self._eng.num_slots + 15) // 16 * 16)

    @property
    def packed_slots_stride(self) -> int:
        """Row stride of 2-bit packed slot outputs: 4 bytes per 16 slots (ap_pack_slots2)."""
        return max(4, (self._eng.num_slots + 15) // 16 * 4)

    def launch(self, seeds, outcome, counts=None, slots=None, statuses=None, stream=None, packed=None) -> None:
        """Raw stream-ordered launch on preallocated device tensors (no allocation, no sync).

        seeds int8 [B, |D|] (candidate order, which must be ascending), outcome
        uint8 [B], counts int32 [B, 4] | None, slots int8 [B, >=|S|] | None,
        statuses int8 [B, >=|D|] | None, packed uint8 [B, >=packed_slots_stride]
        | None: the slot statuses as 2-bit codes written by K1 itself
        (exclusive with `slots`; decode with `unpack_slots2`).
        """
        dev, dec = self.prepare()
        lib = _native.require_device()
        b = seeds.shape[0]
        if seeds.dim() != 2 or seeds.shape[1] != dec.n:
            raise ValueError(f"seeds must be [B, {dec.n}] over the candidate list, got {tuple(seeds.shape)}")
        if packed is not None:
            if slots is not None:
                raise ValueError("launch: `slots` and `packed` are exclusive")
            _native.check(
                lib.ap_propagate_batch_packed(
                    dev.handle, dec.handle, _native.ptr(seeds), b, seeds.stride(0) if b else pad16(dec.n),
                    _native.ptr(packed), packed.stride(0),
                    _native.ptr(statuses), 0 if statuses is None else statuses.stride(0),
                    _native.ptr(outcome), _native.ptr(counts), _native.stream_handle(stream),
                )
            )
            return
        _native.check(
            lib.ap_propagate_batch(
                dev.handle, dec.handle, _native.ptr(seeds), b, seeds.stride(0) if b else pad16(dec.n),
                _native.ptr(slots), 0 if slots is None else slots.stride(0),
                _native.ptr(statuses), 0 if statuses is None else statuses.stride(0),
                _native.ptr(outcome), _native.ptr(counts), _native.stream_handle(stream),
            )
        )

    def run_batch_host(self, seeds_host, *, want_slots: bool = True, chunk: int = 1 << 16, out=None):
        """End-to-end batch from host memory: H2D, kernel, D2H, overlapped over two streams.

        `seeds_host` is a (preferably pinned) CPU int8 tensor [B, |D|].
        Returns pinned CPU tensors `outcome`, `counts` and optionally
        `slots` [B, slots_stride] after synchronising.  want_slots="packed"
        returns `slots_packed` [B, packed_slots_stride] uint8 instead: the same
        statuses at 2 bits per slot, emitted by K1 itself
        (ap_propagate_batch_packed, decoded by `unpack_slots2`), a quarter of
        the D2H bytes.
        """
        import torch

        self.prepare()
        packed = want_slots == "packed"
        if not (packed or isinstance(want_slots, bool)):
            raise ValueError("want_slots must be True, False or 'packed'")
        want_slots = bool(want_slots)
        b, n = seeds_host.shape
        if n != len(self.candidates):
            raise ValueError(f"seeds must be [B, {len(self.candidates)}] over the candidate list, got {tuple(seeds_host.shape)}")
        if out is None:
            out = {
                "outcome": torch.empty(b, dtype=torch.uint8, pin_memory=True),
                "counts": torch.empty((b, 4), dtype=torch.int32, pin_memory=True),
            }
            if packed:
                out["slots_packed"] = torch.empty((b, self.packed_slots_stride), dtype=torch.uint8, pin_memory=True)
            elif want_slots:
                out["slots"] = torch.empty((b, self.slots_stride), dtype=torch.int8, pin_memory=True)
        key = (chunk, n, want_slots, packed)
        bufs = getattr(self, "_host_bufs", None)
        if bufs is None or bufs[0] != key:
            streams = [torch.cuda.Stream(), torch.cuda.Stream()]
            dev_bufs = []
            for _ in range(2):
                d = {
                    "seeds": torch.empty((chunk, pad16(n)), dtype=torch.int8, device="cuda")[:, :n],
                    "outcome": torch.empty(chunk, dtype=torch.uint8, device="cuda"),
                    "counts": torch.empty((chunk, 4), dtype=torch.int32, device="cuda"),
                }
                if want_slots and not packed:
                    d["slots"] = torch.empty((chunk, self.slots_stride), dtype=torch.int8, device="cuda")
                if packed:
                    d["packed"] = torch.empty((chunk, self.packed_slots_stride), dtype=torch.uint8, device="cuda")
                dev_bufs.append(d)
            self._host_bufs = bufs = (key, streams, dev_bufs)
        _, streams, dev_bufs = bufs
        cur = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(cur)
        for i, lo in enumerate(range(0, b, chunk)):
            hi = min(b, lo + chunk)
            s, d = streams[i % 2], dev_bufs[i % 2]
            with torch.cuda.stream(s):
                d["seeds"][: hi - lo].copy_(seeds_host[lo:hi], non_blocking=True)
                self.launch(d["seeds"][: hi - lo], d["outcome"], d["counts"], d.get("slots"), stream=s,
                            packed=d["packed"][: hi - lo] if packed else None)
                out["outcome"][lo:hi].copy_(d["outcome"][: hi - lo], non_blocking=True)
                out["counts"][lo:hi].copy_(d["counts"][: hi - lo], non_blocking=True)
                if packed:
                    out["slots_packed"][lo:hi].copy_(d["packed"][: hi - lo], non_blocking=True)
                elif want_slots:
                    out["slots"][lo:hi].copy_(d["slots"][: hi - lo], non_blocking=True)
        for s in streams:
            s.synchronize()
        return out

    def run_batch(self, seeds, *, want_slots: bool = False, want_statuses: bool = True, stream=None):
        """Propagate a batch of seed vectors on the GPU.

        `seeds` is an int8 tensor or array [B, len(candidates)] over the
        candidate list (-1 unseeded, 0 R, 1 P, 2 UNDECIDED seed).  Returns a
        dict of device tensors: `outcome` [B] uint8 (0 complete, 1
        incomplete, 2 conflict), `counts` [B, 4] int32 (decided P, decided R,
        newly P, newly R over candidates), optional `statuses` [B, |D|]
        (candidate order) and `slots` [B, |S|].
        """
        import torch

        if self.candidates is None:
            raise ValueError("run_batch needs an explicit candidate list")
        eng = self._eng
        dev, dec, pos, cand_slots = self._decision_for(self.candidates)
        order = np.array([pos[s] for s in cand_slots], dtype=np.int64)
        identity = bool(np.array_equal(order, np.arange(len(order))))
        with torch.cuda.device(dev.device_index):
            s = torch.as_tensor(seeds, dtype=torch.int8).to("cuda", non_blocking=True)
            if s.dim() == 1:
                s = s.view(1, -1)
            if not identity:
                perm = torch.empty(dec.n, dtype=torch.long)
                perm[torch.from_numpy(order)] = torch.arange(len(order))
                s = s[:, perm.cuda()]
            b = s.shape[0]
            row = pad16(dec.n)
            if s.stride(0) != row or s.stride(1) != 1 or s.data_ptr() % 16:
                padded = torch.empty((b, row), dtype=torch.int8, device="cuda")
                padded[:, : dec.n].copy_(s)
                s = padded[:, : dec.n]
            out = {
                "outcome": torch.empty(b, dtype=torch.uint8, device="cuda"),
                "counts": torch.empty((b, 4), dtype=torch.int32, device="cuda"),
            }
            cand_t = torch.empty((b, row), dtype=torch.int8, device="cuda") if want_statuses else None
            slots_t = None
            if want_slots:
                stride = (eng.num_slots + 15) // 16 * 16 or 16
                slots_t = torch.empty((b, stride), dtype=torch.int8, device="cuda")
            lib = _native.require_device()
            _native.check(
                lib.ap_propagate_batch(dev.handle, dec.handle, _native.ptr(s), b, row,
                                       _native.ptr(slots_t), 0 if slots_t is None else slots_t.shape[1],
                                       _native.ptr(cand_t), 0 if cand_t is None else cand_t.shape[1],
                                       _native.ptr(out["outcome"]), _native.ptr(out["counts"]),
                                       _native.stream_handle(stream))
            )
            if cand_t is not None:
                out["statuses"] = cand_t[:, : dec.n] if identity else cand_t[:, torch.from_numpy(order).cuda()]
            if slots_t is not None:
                out["slots"] = slots_t[:, : eng.num_slots]
        return out


def _forced_slot_list(eng: _GraphEngine) -> list[int]:
    """Slots the rule table pins to REPLICATED before seeding (sharding.py:178-188)."""
    graph = eng.graph
    out: list[int] = []
    for ins in sorted(graph.instructions, key=lambda i: i.id):
        if ins.opcode == "reshape":
            src = graph.instruction(ins.operand_ids[0])
            _, lone_a, lone_b = pair_reshape(src.shape.dims, ins.shape.dims)
            out += [eng.slot(src.id, i) for i in lone_a] + [eng.slot(ins.id, j) for j in lone_b]
        elif ins.opcode == "broadcast":
            src = graph.instruction(ins.operand_ids[0])
            paired = {j for _, j in pair_broadcast(src.shape.dims, ins.shape.dims)}
            out += [eng.slot(ins.id, j) for j in range(ins.shape.rank) if j not in paired]
    return out


def propagate(graph, seeds: Mapping[DimIndex, DimStatus], candidates: Sequence[DimIndex] | None = None
              ) -> PropagationResult:
    """One-shot propagation (reference `sharding.py:305-311`); the compiled graph is cached."""
    return PropagationEngine(graph, candidates).run(seeds)


# -- rule_for: one opcode's rule applied to standalone specs -------------------


def rule_for(
    opcode: str,
    operand_specs: Sequence[ShardingSpec],
    output_spec: ShardingSpec,
) -> tuple[tuple[ShardingSpec, ...], ShardingSpec] | None:
    """Apply one opcode's rule to standalone specs (reference `sharding.py:314-392`).

    The specs become a one-rule graph whose start state is the given
    statuses; the engine's ordered replay runs the rule to its fixed point.
    Returns None on conflict.
    """

    def need_dims(spec: ShardingSpec) -> tuple[int, ...]:
        if spec.dims is None:
            raise ValueError(f"rule for {opcode} needs specs with dims attached")
        return spec.dims

    operands = list(operand_specs)
    if opcode in ELEMENTWISE_BINARY or opcode in ELEMENTWISE_UNARY or opcode == "get-tuple-element":
        if any(s.rank != output_spec.rank for s in operands):
            raise ValueError(f"rule for {opcode} needs operand ranks equal to the output rank")
    elif opcode == "transpose":
        if operands[0].rank != output_spec.rank:
            raise ValueError("rule for transpose needs operand rank equal to the output rank")
    elif opcode == "reshape":
        pair_reshape(need_dims(operands[0]), need_dims(output_spec))
    elif opcode == "broadcast":
        pair_broadcast(need_dims(operands[0]), need_dims(output_spec))
    elif opcode == "reduce":
        pair_reduce(need_dims(operands[0]), need_dims(output_spec))
    elif opcode not in ("parameter", "constant", "tuple", "dot"):
        raise ValueError(f"unknown opcode {opcode!r}")

    def extents(spec: ShardingSpec) -> tuple[int, ...]:
        return spec.dims if spec.dims is not None else (1,) * spec.rank

    instrs: list[Instruction] = []
    for k, spec in enumerate(operands):
        instrs.append(Instruction(k, f"operand{k}", "parameter", (), TensorShape(extents(spec))))
    out_id = len(operands)
    specs = operands + [output_spec]
    if opcode == "get-tuple-element":
        # the caller passes the selected tuple element as the single operand
        tup = Instruction(out_id + 1, "tuple", "tuple", (0,), TensorShape(extents(operands[0])))
        instrs.append(Instruction(out_id, "output", opcode, (out_id + 1,), TensorShape(extents(output_spec))))
        instrs.append(tup)
    elif opcode in ("parameter", "constant"):
        instrs.append(Instruction(out_id, "output", opcode, (), TensorShape(extents(output_spec))))
    else:
        instrs.append(
            Instruction(out_id, "output", opcode, tuple(range(len(operands))), TensorShape(extents(output_spec)))
        )
    graph = _UncheckedGraph(instrs)
    eng = graph_engine(graph)
    init = np.full(max(eng.num_slots, 1), _U, dtype=np.int8)
    for k, spec in enumerate(specs):
        lo = eng.slot_offset[eng.pos_of_id[k]]
        init[lo: lo + spec.rank] = spec.statuses
    dev = eng.device()
    dec = dev.decision(np.zeros(0, dtype=np.int64), np.zeros(0, dtype=np.uint8))
    lib = _native.require_device()
    state = np.empty_like(init)
    code = np.zeros(1, dtype=np.int32)
    site = np.zeros(1, dtype=np.int32)
    _native.check(lib.ap_propagate_trace(dev.handle, dec.handle, None, _native.ptr(init), _native.ptr(state),
                                         _native.ptr(code), _native.ptr(site), _native.stream_handle()))
    if code[0] == _native.OUTCOME_CONFLICT:
        return None
    new = []
    for k, spec in enumerate(specs):
        lo = eng.slot_offset[eng.pos_of_id[k]]
        new.append(ShardingSpec(tuple(int(v) for v in state[lo: lo + spec.rank]), spec.dims))
    return tuple(new[:-1]), new[-1]


class _UncheckedGraph:
    """Minimal graph for rule_for: shapes are only as real as the specs allow."""

    def __init__(self, instrs: Sequence[Instruction]):
        self._by_id = {i.id: i for i in instrs}
        self.trainable_variables: tuple[str, ...] = ()

    @property
    def instructions(self):
        return tuple(self._by_id[k] for k in sorted(self._by_id))

    def instruction(self, iid: int) -> Instruction:
        return self._by_id[iid]

    def tuple_element_index(self, ins: Instruction) -> int | None:
        return 0 if ins.opcode == "get-tuple-element" else None
