"""Linkage groups: every single-dim trigger propagated as one device batch.

Reference `autoplan.linkage` (`pkg/src/autoplan/linkage.py:26-128`) runs
the 2*|D| triggers one engine call at a time (18 s at BERT-48 scale).  Here
all triggers form one seed batch for the propagation kernel; the groups'
`implied` tuples are materialised lazily from the returned status matrix.
"""

from __future__ import annotations

import json
import logging
from typing import Mapping, Sequence

import numpy as np

from .ir import DimIndex
from .sharding import DimStatus, PropagationEngine

logger = logging.getLogger(__name__)

Trigger = tuple[DimIndex, DimStatus]
_TRIGGER_STATUSES = (DimStatus.PARTITIONED, DimStatus.REPLICATED)


class LinkageGroup:
    """Candidate dims decided by one trigger alone (the trigger excluded).

    Same fields as the reference dataclass (`linkage.py:26-40`).  Groups made
    by `extract_linkage_groups` keep the device status row and build the
    `implied` tuple on first access.
    """

    __slots__ = ("trigger", "infeasible", "_implied", "_row", "_dims", "_size")

    def __init__(self, trigger: Trigger, implied=(), infeasible: bool = False):
        self.trigger = trigger
        self.infeasible = bool(infeasible)
        self._implied = tuple(implied)
        self._row = None
        self._dims = None
        self._size = len(self._implied)

    @classmethod
    def from_row(cls, trigger: Trigger, row: np.ndarray, dims: Sequence[DimIndex], infeasible: bool) -> "LinkageGroup":
        g = cls(trigger, (), infeasible)
        g._implied = None
        g._row = row
        g._dims = dims
        g._size = int((row != -1).sum())
        return g

    @property
    def implied(self) -> tuple[tuple[DimIndex, DimStatus], ...]:
        if self._implied is None:
            self._implied = tuple((self._dims[j], DimStatus(int(self._row[j]))) for j in np.flatnonzero(self._row != -1))
        return self._implied

    @property
    def size(self) -> int:
        return self._size

    def __eq__(self, other) -> bool:
        if not isinstance(other, LinkageGroup):
            return NotImplemented
        return (self.trigger, self.infeasible, self.implied) == (other.trigger, other.infeasible, other.implied)

    def __hash__(self) -> int:
        return hash((self.trigger, self.infeasible, self.implied))

    def __repr__(self) -> str:
        return f"LinkageGroup(trigger={self.trigger!r}, size={self.size}, infeasible={self.infeasible})"


def trigger_matrix(num_dims: int) -> np.ndarray:
    """Seed rows of the 2*|D| triggers: row 2k seeds dim k P, row 2k+1 seeds it R."""
    seeds = np.full((2 * num_dims, num_dims), -1, dtype=np.int8)
    k = np.arange(num_dims)
    seeds[2 * k, k] = int(DimStatus.PARTITIONED)
    seeds[2 * k + 1, k] = int(DimStatus.REPLICATED)
    return seeds


def linkage_tables(graph, dims: Sequence[DimIndex]):
    """(implied [2D, D] int8: trigger and undecided dims -1; infeasible [2D] bool; sizes [2D])."""
    import torch

    dims = list(dims)
    n = len(dims)
    engine = PropagationEngine(graph, candidates=dims)
    seeds = torch.from_numpy(trigger_matrix(n))
    out = engine.run_batch(seeds, want_statuses=True)
    statuses = out["statuses"].clone()
    idx = torch.arange(n, device=statuses.device)
    statuses[2 * idx, idx] = -1
    statuses[2 * idx + 1, idx] = -1
    infeasible = out["outcome"] == 2
    statuses[infeasible] = -1
    sizes = (statuses != -1).sum(dim=1)
    return statuses.cpu().numpy(), infeasible.cpu().numpy(), sizes.cpu().numpy()


def extract_linkage_groups(graph, dims: Sequence[DimIndex], max_workers: int = 1) -> dict[Trigger, LinkageGroup]:
    """All (dim, status) triggers in one batched propagation (reference linkage.py:43-68).

    `max_workers` is accepted for signature compatibility; the batch is one
    kernel launch.
    """
    dims = list(dims)
    implied, infeasible, sizes = linkage_tables(graph, dims)
    groups: dict[Trigger, LinkageGroup] = {}
    for k, d in enumerate(dims):
        for s_i, st in enumerate(_TRIGGER_STATUSES):
            row = 2 * k + s_i
            trig = (d, st)
            groups[trig] = LinkageGroup.from_row(trig, implied[row], dims, bool(infeasible[row]))
    return groups


def sorted_decision_order(groups: Mapping[Trigger, LinkageGroup]) -> list[DimIndex]:
    """Dims by descending larger-group size, ties by flat index (linkage.py:71-83)."""
    best: dict[DimIndex, int] = {}
    for (d, _st), g in groups.items():
        best[d] = max(best.get(d, 0), g.size)
    return sorted(best, key=lambda d: (-best[d], d.flat_index))


def _dim_row(d: DimIndex) -> list[int]:
    return [d.flat_index, d.instruction_id, d.dim]


def save_cache(path: str, graph, groups: Mapping[Trigger, LinkageGroup]) -> None:
    """JSON cache keyed by the graph content hash (reference linkage.py:94-109 layout)."""
    payload = {
        "graph_hash": graph.content_hash(),
        "groups": [
            {
                "trigger": _dim_row(g.trigger[0]) + [int(g.trigger[1])],
                "implied": [_dim_row(d) + [int(s)] for d, s in g.implied],
                "infeasible": g.infeasible,
            }
            for g in groups.values()
        ],
    }
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(payload, sort_keys=True) + "\n")


def load_cache(path: str, graph) -> dict[Trigger, LinkageGroup] | None:
    try:
        with open(path, "r", encoding="utf-8") as fh:
            payload = json.load(fh)
    except (OSError, json.JSONDecodeError):
        return None
    if payload.get("graph_hash") != graph.content_hash():
        logger.info("linkage cache at %s does not match the graph, ignoring", path)
        return None
    out: dict[Trigger, LinkageGroup] = {}
    for raw in payload.get("groups", []):
        t = raw["trigger"]
        trig = (DimIndex(t[0], t[1], t[2]), DimStatus(t[3]))
        implied = tuple((DimIndex(e[0], e[1], e[2]), DimStatus(e[3])) for e in raw["implied"])
        out[trig] = LinkageGroup(trig, implied, raw["infeasible"])
    return out
