"""Loading helpers for the reference-generated fixtures in tests/golden/."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from paper_2007_04069_b200.ir import graph_from_dict

GOLDEN = Path(__file__).resolve().parent / "golden"


def prop_names() -> list[str]:
    return sorted(p.stem[len("prop_"):] for p in GOLDEN.glob("prop_*.npz"))


def linkage_names() -> list[str]:
    return sorted(p.stem[len("linkage_"):] for p in GOLDEN.glob("linkage_*.npz"))


class Fixture:
    def __init__(self, path: Path):
        z = np.load(path)
        self.data = {k: z[k] for k in z.files}
        self.graph = graph_from_dict(json.loads(bytes(self.data["graph_json"]).decode()))
        self.flat = self.graph.flat()
        self.cand = [(int(a), int(b)) for a, b in self.data["cand"]]
        pos = {int(i): p for p, i in enumerate(self.flat.ids)}
        self.cand_slots = np.array([self.flat.slot_offset[pos[i]] + d for i, d in self.cand], dtype=np.int64)

    def __getitem__(self, key):
        return self.data[key]


def load_prop(name: str) -> Fixture:
    return Fixture(GOLDEN / f"prop_{name}.npz")


def load_linkage(name: str) -> Fixture:
    return Fixture(GOLDEN / f"linkage_{name}.npz")


def rule_for_cases() -> list[dict]:
    return json.loads((GOLDEN / "rule_for.json").read_text())["cases"]
