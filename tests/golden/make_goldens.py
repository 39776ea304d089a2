"""Generate golden propagation fixtures by running the REFERENCE planner.

Run in the build container (the reference lives at /root/reference and does
not travel to the GPU box):

    python tests/golden/make_goldens.py

Each `prop_<name>.npz` holds one graph (reference JSON), its candidate dims,
a batch of seed rows over those candidates and the reference's outputs of
`PropagationEngine(graph, dims).run(seeds)` (sharding.py:210-248): outcome,
every slot status (conflict rows hold the reference snapshot), conflict site
(instruction id or -1) and the newly-decided mask.  `linkage_<name>.npz`
holds `extract_linkage_groups` + `sorted_decision_order` (linkage.py:43-83).
`rule_for.json` holds `rule_for` cases (sharding.py:314-392).
Seed encoding: -1 none, 0 R, 1 P, 2 UNDECIDED.  Versions are recorded.
"""

from __future__ import annotations

import itertools
import json
import platform
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))

import autoplan  # noqa: E402
import helpers  # noqa: E402
from autoplan import zoo  # noqa: E402
from autoplan.ir import decision_dims, graph_from_dict  # noqa: E402
from autoplan.linkage import extract_linkage_groups, sorted_decision_order  # noqa: E402
from autoplan.sharding import DimStatus, Outcome, PropagationEngine, ShardingSpec, rule_for  # noqa: E402

from paper_2007_04069_b200 import graphs as gens  # noqa: E402

OUT = Path(__file__).resolve().parent
OUTCODE = {Outcome.COMPLETE: 0, Outcome.INCOMPLETE: 1, Outcome.CONFLICT: 2}
VALUE = {-1: None, 0: DimStatus.REPLICATED, 1: DimStatus.PARTITIONED, 2: DimStatus.UNDECIDED}


def _versions() -> str:
    return json.dumps({"python": platform.python_version(), "numpy": np.__version__, "autoplan": autoplan.__version__})


def run_reference(graph, dims, seeds: np.ndarray):
    engine = PropagationEngine(graph, candidates=dims)
    ids = sorted(i.id for i in graph.instructions)
    S = sum(graph.instruction(i).shape.rank for i in ids)
    B = seeds.shape[0]
    outcome = np.zeros(B, np.int8)
    slots = np.zeros((B, S), np.int8)
    site = np.full(B, -1, np.int32)
    newly = np.zeros((B, len(dims)), np.int8)
    flat_pos = {d: k for k, d in enumerate(dims)}
    for b in range(B):
        sd = {dims[j]: VALUE[int(v)] for j, v in enumerate(seeds[b]) if v != -1}
        r = engine.run(sd)
        outcome[b] = OUTCODE[r.outcome]
        slots[b] = [s for i in ids for s in r.assignments[i].statuses]
        site[b] = -1 if r.conflict_site is None else r.conflict_site
        for d, st in r.newly_decided:
            newly[b, flat_pos[d]] = 1
    return outcome, slots, site, newly


def seed_rows(rng, n: int, exhaustive_limit: int = 10, random_full: int = 256, random_partial: int = 128,
              undecided: int = 16) -> np.ndarray:
    rows = []
    if n <= exhaustive_limit:
        rows += [list(v) for v in itertools.product((1, 0), repeat=n)]
    else:
        rows += rng.integers(0, 2, size=(random_full, n)).tolist()
    for _ in range(random_partial):  # prefix-style partial seeds, as in the bench batch
        k = int(rng.integers(1, n + 1))
        row = [-1] * n
        for j in rng.permutation(n)[:k]:
            row[j] = int(rng.integers(0, 2))
        rows.append(row)
    for _ in range(undecided):  # UNDECIDED seeds (legal in the reference run)
        row = rng.integers(-1, 3, size=n).tolist()
        rows.append(row)
    rows.append([-1] * n)
    return np.asarray(rows, dtype=np.int8)


def dump(name: str, graph, dims, seeds: np.ndarray) -> None:
    outcome, slots, site, newly = run_reference(graph, dims, seeds)
    np.savez_compressed(
        OUT / f"prop_{name}.npz",
        graph_json=np.frombuffer(json.dumps(graph.to_dict(), sort_keys=True).encode(), dtype=np.uint8),
        cand=np.asarray([[d.instruction_id, d.dim] for d in dims], dtype=np.int64).reshape(-1, 2),
        seeds=seeds,
        outcome=outcome,
        slots=slots,
        site=site,
        newly=newly,
        versions=np.frombuffer(_versions().encode(), dtype=np.uint8),
    )
    print(f"prop_{name}: B={len(seeds)} S={slots.shape[1]} D={len(dims)} conflicts={(outcome == 2).mean():.2f}")


def dump_linkage(name: str, graph, dims) -> None:
    groups = extract_linkage_groups(graph, dims)
    order = sorted_decision_order(groups)
    D = len(dims)
    implied = np.full((2 * D, D), -1, np.int8)
    infeasible = np.zeros(2 * D, np.uint8)
    pos = {d: k for k, d in enumerate(dims)}
    for k, d in enumerate(dims):
        for s_i, st in enumerate((DimStatus.PARTITIONED, DimStatus.REPLICATED)):
            g = groups[(d, st)]
            row = 2 * k + s_i
            infeasible[row] = g.infeasible
            for dd, v in g.implied:
                implied[row, pos[dd]] = int(v)
    np.savez_compressed(
        OUT / f"linkage_{name}.npz",
        graph_json=np.frombuffer(json.dumps(graph.to_dict(), sort_keys=True).encode(), dtype=np.uint8),
        cand=np.asarray([[d.instruction_id, d.dim] for d in dims], dtype=np.int64).reshape(-1, 2),
        implied=implied,
        infeasible=infeasible,
        order=np.asarray([d.flat_index for d in order], dtype=np.int64),
    )
    print(f"linkage_{name}: D={D} infeasible={int(infeasible.sum())}")


def dump_rule_for(rng) -> None:
    cases = []
    shapes = {"tanh": ((3, 4),), "add": ((3, 4), (3, 4)), "transpose": ((3, 4),), "dot": ((3, 5), (5, 4))}
    out_shape = {"tanh": (3, 4), "add": (3, 4), "transpose": (4, 3), "dot": (3, 4)}
    shaped = {"broadcast": ((4,), (3, 4)), "reduce": ((3, 4), (3,)), "reshape": ((6, 4), (2, 3, 4))}

    def rand_spec(dims_):
        r = len(dims_)
        st = [int(v) for v in rng.integers(-1, 2, size=r)]
        if st.count(1) > 1:
            keep = st.index(1)
            st = [(-1 if (v == 1 and i != keep) else v) for i, v in enumerate(st)]
        return st

    for opcode, ins in list(shapes.items()):
        for _ in range(40):
            ops = [rand_spec(s) for s in ins]
            out = rand_spec(out_shape[opcode])
            res = rule_for(opcode, [ShardingSpec(tuple(o)) for o in ops], ShardingSpec(tuple(out)))
            cases.append({"opcode": opcode, "operands": ops, "operand_dims": None, "output": out,
                          "output_dims": None,
                          "result": None if res is None else [[list(s.statuses) for s in res[0]],
                                                              list(res[1].statuses)]})
    for opcode, (src, dst) in shaped.items():
        for _ in range(40):
            op = rand_spec(src)
            out = rand_spec(dst)
            res = rule_for(opcode, [ShardingSpec(tuple(op), src)], ShardingSpec(tuple(out), dst))
            cases.append({"opcode": opcode, "operands": [op], "operand_dims": [list(src)], "output": out,
                          "output_dims": list(dst),
                          "result": None if res is None else [[list(s.statuses) for s in res[0]],
                                                              list(res[1].statuses)]})
    (OUT / "rule_for.json").write_text(json.dumps({"versions": json.loads(_versions()), "cases": cases}, indent=0))
    print(f"rule_for: {len(cases)} cases")


def main() -> None:
    rng = np.random.default_rng(20201007)
    small = {
        "linkage_chain": helpers.linkage_chain_graph(),
        "two_layer": helpers.two_layer_graph(),
        "attention_block": zoo.attention_block(),
        "t5_block": zoo.t5_block(),
    }
    for name, g in small.items():
        dims = decision_dims(g, g.trainable_variables)
        dump(name, g, dims, seed_rows(rng, len(dims)))
        dump_linkage(name, g, dims)
    # dot-rule graph with every tensor a candidate (test_sharding.py:59-68)
    vgg = zoo.vgg_classifier()
    adp_names = [i.name for i in vgg.instructions if i.opcode == "parameter" and i.name not in vgg.trainable_variables]
    adp_dims = decision_dims(vgg, adp_names)
    dump("vgg_classifier_adp", vgg, adp_dims, seed_rows(rng, len(adp_dims)))
    chain = zoo.uniform_chain(length=12)
    dump("uniform_chain_all", chain, decision_dims(chain, [i.name for i in chain.instructions]),
         seed_rows(rng, 28, random_full=64, random_partial=64))
    # the hypothesis graphs of test_sharding.py:279-327 (seeds 0..200), exhaustive over P/R
    for gs in range(0, 201):
        g = helpers.random_decision_graph(np.random.default_rng(gs))
        dims = decision_dims(g, g.trainable_variables)
        dump(f"random_{gs:03d}", g, dims, seed_rows(rng, len(dims), random_partial=16, undecided=4))
    # synthetic BASELINE models: a bounded sample (the reference runs ~10 ms per plan at BERT-48)
    for name, B in (("mlp2", 0), ("bert_base", 48), ("vgg19", 64), ("t5_large", 16), ("bert48", 16)):
        g = graph_from_dict(gens.generate(name).to_dict())
        dims = decision_dims(g, g.trainable_variables)
        if name == "mlp2":
            seeds = seed_rows(rng, len(dims))
        else:
            seeds = seed_rows(rng, len(dims), exhaustive_limit=0, random_full=B // 4, random_partial=B // 2,
                              undecided=B // 4)
        dump(name, g, dims, seeds)
        if name in ("mlp2", "bert_base", "vgg19"):
            dump_linkage(name, g, dims)
    dump_rule_for(rng)


if __name__ == "__main__":
    main()
