"""Graph IR: shape rules, validation errors, ordering, decision dims, JSON.

Mirrors the reference's IR tests (reference pkg/tests/test_ir.py:30-359)
against this package's IR, plus the dense `flat()` view the engine ingests.
"""

import json

import numpy as np
import pytest

from paper_2007_04069_b200.ir import (
    DimIndex,
    GraphParseError,
    GraphValidationError,
    HloGraph,
    Instruction,
    TensorShape,
    decision_dims,
    forward_subgraph,
    graph_from_dict,
    load_graph,
    pair_broadcast,
    pair_reduce,
    pair_reshape,
)
from paper_2007_04069_b200 import graphs


def ins(i, name, opcode, operands=(), dims=(), **kw):
    return Instruction(id=i, name=name, opcode=opcode, operand_ids=tuple(operands), shape=TensorShape(tuple(dims)), **kw)


def chain_graph():
    """y = tanh(x @ w + bias) * scale (reference helpers.linkage_chain_graph)."""
    return HloGraph(
        [
            ins(0, "x", "parameter", dims=(4, 8)),
            ins(1, "w", "parameter", dims=(8, 6)),
            ins(2, "bias", "parameter", dims=(6,)),
            ins(3, "scale", "parameter", dims=(6,)),
            ins(4, "mm", "dot", (0, 1), (4, 6)),
            ins(5, "bias_b", "broadcast", (2,), (4, 6)),
            ins(6, "sum", "add", (4, 5), (4, 6)),
            ins(7, "act", "tanh", (6,), (4, 6)),
            ins(8, "scale_b", "broadcast", (3,), (4, 6)),
            ins(9, "out", "multiply", (7, 8), (4, 6)),
        ],
        ["w", "bias", "scale"],
    )


def test_tensor_shape():
    s = TensorShape((4, 8, 2))
    assert (s.rank, s.num_elements, s.byte_size) == (3, 64, 256)
    assert TensorShape(()).byte_size == 4
    assert TensorShape((10,), element_size=2).byte_size == 20


@pytest.mark.parametrize(
    "rows, match",
    [
        ([ins(0, "a", "parameter", dims=(2, 3)), ins(1, "b", "parameter", dims=(3, 2)), ins(2, "c", "add", (0, 1), (2, 3))],
         "elementwise"),
        ([ins(0, "a", "parameter", dims=(2, 3)), ins(1, "b", "parameter", dims=(4, 5)), ins(2, "c", "dot", (0, 1), (2, 5))],
         "dot"),
        ([ins(0, "a", "parameter", dims=(2, 3, 4)), ins(1, "b", "parameter", dims=(4, 5)),
          ins(2, "c", "dot", (0, 1), (2, 5))], "rank-2"),
        ([ins(0, "a", "parameter", dims=(2, 3, 4)), ins(1, "t", "transpose", (0,), (3, 2, 4))], "transpose"),
        ([ins(0, "a", "parameter", dims=(2, 6)), ins(1, "r", "reshape", (0,), (3, 5))], "element count"),
        ([ins(0, "a", "parameter", dims=(5,)), ins(1, "b", "broadcast", (0,), (4, 6))], "broadcast"),
        ([ins(0, "a", "parameter", dims=(4,)), ins(1, "r", "reduce", (0,), (4, 6))], "raise rank"),
        ([ins(0, "a", "parameter", dims=(4, 6)), ins(1, "r", "reduce", (0,), (5,))], "reduce"),
        ([ins(0, "a", "parameter", dims=(2, 3)), ins(1, "g", "get-tuple-element", (0,), (2, 3))], "tuple"),
        ([ins(0, "a", "parameter", dims=(2, 3)), ins(1, "t", "tuple", (0,), (2, 3)),
          ins(2, "g", "get-tuple-element", (1,), (9, 9))], "shape"),
        ([ins(0, "a", "convolution", dims=(2,))], "opcode"),
        ([ins(0, "a", "parameter", dims=(2,)), ins(1, "b", "add", (0,), (2,))], "operands"),
        ([ins(0, "a", "tanh", (7,), (2,))], "unknown operand"),
        ([ins(0, "a", "parameter", dims=(2,)), ins(0, "b", "parameter", dims=(2,))], "duplicate"),
        ([ins(0, "a", "parameter", dims=(2,)), ins(1, "a", "parameter", dims=(2,))], "unique"),
        ([ins(0, "a", "parameter", dims=(0,))], "extents"),
        ([Instruction(0, "a", "parameter", (), TensorShape((2,), element_size=0))], "element_size"),
        ([ins(0, "a", "tanh", (1,), (2,)), ins(1, "b", "tanh", (0,), (2,))], "cycle"),
    ],
)
def test_validation_errors(rows, match):
    with pytest.raises(GraphValidationError, match=match):
        HloGraph(rows)


def test_trainable_checks():
    with pytest.raises(GraphValidationError, match="not a parameter"):
        HloGraph([ins(0, "a", "parameter", dims=(2,)), ins(1, "b", "tanh", (0,), (2,))], ["b"])
    with pytest.raises(GraphValidationError, match="not an instruction"):
        HloGraph([ins(0, "a", "parameter", dims=(2,))], ["ghost"])


def test_valid_shape_rules():
    g = HloGraph([ins(0, "a", "parameter", dims=(2, 3, 4)), ins(1, "t", "transpose", (0,), (4, 3, 2))])
    assert g.instruction(1).shape.dims == (4, 3, 2)
    g = HloGraph([
        ins(0, "a", "parameter", dims=(2, 3)), ins(1, "b", "parameter", dims=(4,)),
        ins(2, "t", "tuple", (0, 1), (2, 3)), ins(3, "g", "get-tuple-element", (2,), (4,)),
    ])
    assert g.tuple_element_index(g.instruction(3)) == 1


def test_pairing_semantics():
    assert pair_broadcast((6,), (4, 6)) == [(0, 1)]
    assert pair_broadcast((8,), (8, 8)) == [(0, 1)]  # right-aligned greedy
    assert pair_reduce((4, 6), (4,)) == ([(0, 0)], [1])
    assert pair_reduce((4, 6), (6,)) == ([(1, 0)], [0])
    assert pair_reshape((2, 6), (2, 3, 2)) == ([(0, 0)], [1], [1, 2])
    assert pair_reshape((4, 6), (4, 6)) == ([(0, 0), (1, 1)], [], [])
    assert pair_reshape((24,), (4, 6)) == ([], [0], [0, 1])


def test_toposort_and_node_classes():
    g = HloGraph([
        ins(0, "src", "parameter", dims=(2,)), ins(1, "l", "tanh", (0,), (2,)),
        ins(2, "r", "exp", (0,), (2,)), ins(3, "m", "add", (1, 2), (2,)),
    ])
    assert g.topological_order == (0, 1, 2, 3)
    g = HloGraph([ins(0, "out", "tanh", (2,), (2,)), ins(1, "src", "parameter", dims=(2,)), ins(2, "mid", "exp", (1,), (2,))])
    assert g.topological_order == (1, 2, 0)
    c = chain_graph()
    assert {c.instruction(i).name for i in c.source_ids} == {"x", "w", "bias", "scale"}
    assert {c.instruction(i).name for i in c.sink_ids} == {"out"}
    assert "mm" in {c.instruction(i).name for i in c.compute_ids}
    g = HloGraph([ins(0, "a", "parameter", dims=(2,)), ins(1, "u", "tanh", (0,), (2,)), ins(2, "v", "exp", (0,), (2,))])
    assert g.consumers(0) == (1, 2) and g.consumers(2) == ()
    g = HloGraph([
        ins(0, "a", "parameter", dims=(2,)), ins(1, "f", "tanh", (0,), (2,)),
        ins(2, "bwd", "exp", (1,), (2,), is_forward=False),
    ])
    assert forward_subgraph(g) == [0, 1]


def test_decision_dims():
    g = chain_graph()
    dims = decision_dims(g, g.trainable_variables)
    assert [d.flat_index for d in dims] == list(range(len(dims)))
    assert [(g.instruction(d.instruction_id).name, d.dim) for d in dims] == [("w", 0), ("w", 1), ("bias", 0), ("scale", 0)]
    assert len(decision_dims(g, ["w", "w"])) == 2
    with pytest.raises(GraphValidationError):
        decision_dims(g, ["ghost"])
    assert DimIndex(0, 3, 1) == DimIndex(flat_index=0, instruction_id=3, dim=1)


def test_serialization(tmp_path):
    g = chain_graph()
    h = graph_from_dict(g.to_dict())
    assert h.to_dict() == g.to_dict() and h.content_hash() == g.content_hash()
    path = str(tmp_path / "g.json")
    g.save(path)
    assert load_graph(path).content_hash() == g.content_hash()
    with pytest.raises(GraphParseError, match="cannot read"):
        load_graph(str(tmp_path / "nope.json"))
    (tmp_path / "bad.json").write_text("{nope")
    with pytest.raises(GraphParseError, match="not valid JSON"):
        load_graph(str(tmp_path / "bad.json"))
    with pytest.raises(GraphParseError, match="malformed"):
        graph_from_dict({"instructions": [{"name": "a"}]})
    with pytest.raises(GraphParseError, match="instructions"):
        graph_from_dict({"nodes": []})
    with pytest.raises(GraphParseError, match="trainable_variables"):
        graph_from_dict({"instructions": [], "trainable_variables": [3]})
    g2 = HloGraph([ins(0, "x", "parameter", dims=(2,)), ins(1, "y", "tanh", (0,), (2,), compute_cost_ms=1.5)])
    assert graph_from_dict(g2.to_dict()).by_name("y").compute_cost_ms == 1.5


def test_access():
    g = chain_graph()
    assert g.by_name("mm").opcode == "dot"
    assert g.by_name("w").id in g and 999 not in g
    with pytest.raises(GraphValidationError):
        g.by_name("ghost")
    with pytest.raises(GraphValidationError):
        g.instruction(999)


def test_flat_view():
    g = chain_graph()
    f = g.flat()
    assert f.num_instructions == 10 and f.num_slots == 18
    assert list(f.slot_offset[:3]) == [0, 2, 4]
    assert f.opcode[4] == 8 and list(f.operands[f.operand_offset[4]:f.operand_offset[5]]) == [0, 1]
    assert (f.gte_element == -1).all()


@pytest.mark.parametrize("name", sorted(graphs.GENERATORS))
def test_generators_roundtrip(name):
    g = graphs.generate(name)
    h = graph_from_dict(json.loads(json.dumps(g.to_dict())))
    assert h.content_hash() == g.content_hash()
    assert len(g.trainable_variables) > 0


def test_generators_match_golden_graphs():
    """The fixtures embed the JSON the reference loaded; generators must still emit it."""
    from goldens import load_prop

    for name in ("mlp2", "bert_base", "vgg19", "t5_large", "bert48"):
        f = load_prop(name)
        assert f.graph.content_hash() == graphs.generate(name).content_hash(), name
