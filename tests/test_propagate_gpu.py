"""GPU parity of the propagation kernel (K1) through the C-ABI.

Against the reference (golden fixtures) and the CPU oracle:
* batched kernel: outcome, candidate statuses, newly / decided counts and
  all slot statuses for every non-CONFLICT row, bit-exact;
* `PropagationEngine.run` / `propagate` (single plan) including the exact
  CONFLICT snapshot and conflict site via the ordered replay kernel;
* `rule_for`, linkage groups and decision order;
* full-size random batches on BERT-48 / T5-large checked row by row
  against the oracle, plus size-independent properties.
"""

import numpy as np
import pytest
import torch

from goldens import linkage_names, load_linkage, load_prop, prop_names, rule_for_cases
from oracle import oracle
from paper_2007_04069_b200 import graphs
from paper_2007_04069_b200.ir import DimIndex, decision_dims
from paper_2007_04069_b200.linkage import extract_linkage_groups, sorted_decision_order
from paper_2007_04069_b200.sharding import (
    DimStatus,
    Outcome,
    PropagationEngine,
    ShardingSpec,
    propagate,
    rule_for,
)

pytestmark = pytest.mark.gpu

VALUE = {0: DimStatus.REPLICATED, 1: DimStatus.PARTITIONED, 2: DimStatus.UNDECIDED}


def dims_of(f):
    return [DimIndex(k, i, d) for k, (i, d) in enumerate(f.cand)]


@pytest.mark.parametrize("name", prop_names())
def test_batch_kernel_matches_reference(cuda, name):
    f = load_prop(name)
    eng = PropagationEngine(f.graph, dims_of(f))
    out = eng.run_batch(torch.from_numpy(f["seeds"]), want_slots=True)
    outcome = out["outcome"].cpu().numpy()
    np.testing.assert_array_equal(outcome, f["outcome"])
    ok = outcome != 2
    slots = out["slots"].cpu().numpy()
    np.testing.assert_array_equal(slots[ok], f["slots"][ok])
    statuses = out["statuses"].cpu().numpy()
    np.testing.assert_array_equal(statuses[ok], f["slots"][ok][:, f.cand_slots])
    counts = out["counts"].cpu().numpy()
    newly = f["newly"].astype(bool)
    cand = f["slots"][:, f.cand_slots]
    np.testing.assert_array_equal(counts[ok, 2], (newly & (cand == 1)).sum(1)[ok])
    np.testing.assert_array_equal(counts[ok, 3], (newly & (cand == 0)).sum(1)[ok])
    np.testing.assert_array_equal(counts[ok, 0], (cand == 1).sum(1)[ok])
    np.testing.assert_array_equal(counts[ok, 1], (cand == 0).sum(1)[ok])


@pytest.mark.parametrize("name", ["linkage_chain", "two_layer", "attention_block", "t5_block", "vgg_classifier_adp",
                                  "mlp2", "bert_base", "random_003", "random_150"])
def test_single_plan_api_matches_reference(cuda, name):
    f = load_prop(name)
    dims = dims_of(f)
    eng = PropagationEngine(f.graph, dims)
    ids = sorted(i.id for i in f.graph.instructions)
    for b in range(0, len(f["seeds"]), max(1, len(f["seeds"]) // 40)):
        seeds = {dims[j]: VALUE[int(v)] for j, v in enumerate(f["seeds"][b]) if v != -1}
        r = eng.run(seeds)
        assert {Outcome.COMPLETE: 0, Outcome.INCOMPLETE: 1, Outcome.CONFLICT: 2}[r.outcome] == f["outcome"][b]
        flat = np.array([s for i in ids for s in r.assignments[i].statuses], dtype=np.int8)
        np.testing.assert_array_equal(flat, f["slots"][b])  # CONFLICT snapshot included
        assert (r.conflict_site if r.conflict_site is not None else -1) == f["site"][b]
        expect_newly = [dims[j] for j in np.flatnonzero(f["newly"][b])]
        assert [d for d, _ in r.newly_decided] == expect_newly


def test_propagate_without_candidates(cuda):
    f = load_prop("two_layer")
    dims = dims_of(f)
    r = propagate(f.graph, {dims[1]: DimStatus.PARTITIONED})
    ref = PropagationEngine(f.graph, [d for d in dims if d.instruction_id == dims[1].instruction_id]).run(
        {dims[1]: DimStatus.PARTITIONED})
    assert r.outcome == ref.outcome and r.newly_decided == ref.newly_decided


def test_bad_seed_raises(cuda):
    from paper_2007_04069_b200.ir import GraphValidationError

    f = load_prop("two_layer")
    dims = dims_of(f)
    with pytest.raises(GraphValidationError):
        propagate(f.graph, {DimIndex(0, 999, 0): DimStatus.PARTITIONED}, dims)
    with pytest.raises(GraphValidationError):
        propagate(f.graph, {DimIndex(0, dims[0].instruction_id, 9): DimStatus.PARTITIONED}, dims)


def test_rule_for_matches_reference(cuda):
    for case in rule_for_cases():
        dims = case["operand_dims"] or [None] * len(case["operands"])
        ops = [ShardingSpec(tuple(s), None if d is None else tuple(d)) for s, d in zip(case["operands"], dims)]
        out = ShardingSpec(tuple(case["output"]), None if case["output_dims"] is None else tuple(case["output_dims"]))
        res = rule_for(case["opcode"], ops, out)
        if case["result"] is None:
            assert res is None, case
        else:
            assert res is not None, case
            assert [list(s.statuses) for s in res[0]] == case["result"][0], case
            assert list(res[1].statuses) == case["result"][1], case


@pytest.mark.parametrize("name", linkage_names())
def test_linkage_groups_match_reference(cuda, name):
    f = load_linkage(name)
    dims = dims_of(f)
    groups = extract_linkage_groups(f.graph, dims)
    for k, d in enumerate(dims):
        for s_i, st in enumerate((DimStatus.PARTITIONED, DimStatus.REPLICATED)):
            g = groups[(d, st)]
            row = f["implied"][2 * k + s_i]
            assert g.infeasible == bool(f["infeasible"][2 * k + s_i])
            assert [(dd.flat_index, int(v)) for dd, v in g.implied] == [(j, int(row[j])) for j in np.flatnonzero(row != -1)]
    order = sorted_decision_order(groups)
    np.testing.assert_array_equal([d.flat_index for d in order], f["order"])


def random_prefix_seeds(rng, n, batch, order):
    seeds = np.full((batch, n), -1, np.int8)
    k = rng.integers(1, n + 1, size=batch)
    vals = rng.integers(0, 2, size=(batch, n)).astype(np.int8)
    for b in range(batch):
        seeds[b, order[: k[b]]] = vals[b, : k[b]]
    return seeds


@pytest.mark.parametrize("name", ["bert48", "t5_large", "vgg19", "bert_base"])
def test_full_size_batch_against_oracle(cuda, name):
    g = graphs.generate(name)
    dims = decision_dims(g, g.trainable_variables)
    rng = np.random.default_rng(20201007)
    n = len(dims)
    seeds = np.concatenate([
        random_prefix_seeds(rng, n, 512, rng.permutation(n)),
        random_prefix_seeds(rng, n, 256, np.arange(n))[:, :],
        np.where(rng.random((64, n)) < 0.02, rng.integers(0, 3, size=(64, n)), -1).astype(np.int8),
    ])
    out = PropagationEngine(g, dims).run_batch(torch.from_numpy(seeds), want_slots=True)
    flat = g.flat()
    cand_slots = np.array([flat.slot_offset[d.instruction_id] + d.dim for d in dims])  # ids == positions here
    st, oc, _ = oracle.propagate_batch(flat, cand_slots, seeds, cand_slots)
    outcome = out["outcome"].cpu().numpy()
    np.testing.assert_array_equal(outcome, oc)
    ok = oc != 2
    np.testing.assert_array_equal(out["slots"].cpu().numpy()[ok], st[ok])
    assert ok.sum() > 0


@pytest.mark.parametrize("name", ["bert48", "t5_large", "vgg19", "mlp2"])
def test_fast_and_generic_kernels_agree(cuda, name, monkeypatch):
    """Descriptor-driven fast kernel vs the generic kernel: identical outputs incl. conflict rows."""
    g = graphs.generate(name)
    dims = decision_dims(g, g.trainable_variables)
    n = len(dims)
    rng = np.random.default_rng(11)
    seeds = np.concatenate([
        random_prefix_seeds(rng, n, 300, rng.permutation(n)),
        np.where(rng.random((40, n)) < 0.05, rng.integers(0, 3, size=(40, n)), -1).astype(np.int8),
    ])
    eng = PropagationEngine(g, dims)
    fast = eng.run_batch(torch.from_numpy(seeds), want_slots=True)
    monkeypatch.setenv("AP_PROPAGATE_GENERIC", "1")
    generic = eng.run_batch(torch.from_numpy(seeds), want_slots=True)
    for key in ("outcome", "counts", "statuses", "slots"):
        assert torch.equal(fast[key], generic[key]), key


@pytest.mark.parametrize("name", ["t5_block", "attention_block", "bert_base", "random_042"])
def test_generic_kernel_matches_reference(cuda, name, monkeypatch):
    monkeypatch.setenv("AP_PROPAGATE_GENERIC", "1")
    test_batch_kernel_matches_reference(cuda, name)


def _wide_graph(blocks: int):
    """`blocks` independent x_i @ w_i @ v_i chains with pairwise-distinct extents: 4 link
    classes and 4 candidate dims per block, nothing links across blocks."""
    from paper_2007_04069_b200.graphs import GraphWriter

    w = GraphWriter()
    for i in range(blocks):
        a, b, c, d = 2 + 4 * i, 3 + 4 * i, 4 + 4 * i, 5 + 4 * i
        x = w.param(f"x{i}", (a, b), trainable=False)
        wi = w.param(f"w{i}", (b, c))
        vi = w.param(f"v{i}", (c, d))
        h = w.op(f"h{i}", "dot", (a, c), [x, wi])
        w.op(f"y{i}", "dot", (a, d), [h, vi])
    return w.graph()


@pytest.mark.parametrize("blocks,batch,no_cta", [(80, 48, 0), (1100, 48, 0), (26000, 6, 0), (26000, 6, 1)])
def test_beyond_fast_kernel_limits_matches_oracle(cuda, blocks, batch, no_cta, monkeypatch):
    """> 255 link classes (80 blocks: 320 classes), > 4096 candidate dims (1100 blocks:
    4400 dims) and > 65535 classes with bitsets beyond shared memory (26000 blocks:
    104000 classes, 130000 instructions: one plan per CTA, or with no_cta the per-warp
    bitsets in global memory): the generic kernels match the C oracle."""
    if no_cta:
        monkeypatch.setenv("AP_PROPAGATE_NO_CTA", "1")
    g = _wide_graph(blocks)
    dims = decision_dims(g, g.trainable_variables)
    n = len(dims)
    rng = np.random.default_rng(blocks)
    all_r = np.where(np.arange(n)[None, :] < rng.integers(1, n + 1, size=(2, 1)), 0, -1).astype(np.int8)
    sparse_p = np.full((2, n), -1, np.int8)  # one P seed on every 4th candidate dim
    sparse_p[0, ::4] = 1
    sparse_p[1, 1::4] = 1
    seeds = np.concatenate([
        random_prefix_seeds(rng, n, batch, rng.permutation(n)),
        np.where(rng.random((batch // 3, n)) < 0.01, rng.integers(0, 3, size=(batch // 3, n)), -1).astype(np.int8),
        all_r, sparse_p,
    ])
    eng = PropagationEngine(g, dims)
    out = eng.run_batch(torch.from_numpy(seeds), want_slots=True)
    flat = g.flat()
    cand_slots = np.array([flat.slot_offset[d.instruction_id] + d.dim for d in dims])
    st, oc, _ = oracle.propagate_batch(flat, cand_slots, seeds, cand_slots)
    np.testing.assert_array_equal(out["outcome"].cpu().numpy(), oc)
    ok = oc != 2
    np.testing.assert_array_equal(out["slots"].cpu().numpy()[ok], st[ok])
    assert ok.sum() > 0


def test_properties_at_scale(cuda):
    """Size-independent properties: idempotence, monotonicity, order independence."""
    g = graphs.bert48()
    dims = decision_dims(g, g.trainable_variables)
    eng = PropagationEngine(g, dims)
    n = len(dims)
    rng = np.random.default_rng(5)
    # linkage-style single seeds are never worse than their superset
    seeds = np.full((2 * n, n), -1, np.int8)
    seeds[np.arange(0, 2 * n, 2), np.arange(n)] = 1
    seeds[np.arange(1, 2 * n, 2), np.arange(n)] = 0
    out = eng.run_batch(torch.from_numpy(seeds))
    st = out["statuses"]
    feasible = out["outcome"] != 2
    # idempotence: re-seeding every decided candidate reproduces the fixed point
    again = eng.run_batch(st[feasible].clone())
    assert bool((again["outcome"] != 2).all())
    assert torch.equal(again["statuses"], st[feasible])
    # no newly decided dims on a fixed point
    assert int(again["counts"][:, 2:].sum()) == 0
    # empty and ragged batches
    empty = eng.run_batch(torch.full((0, n), -1, dtype=torch.int8))
    assert empty["outcome"].numel() == 0
    one = eng.run_batch(torch.full((1, n), -1, dtype=torch.int8))
    assert int(one["outcome"][0]) in (0, 1)


@pytest.mark.parametrize("layers", [400, 1000])
def test_real_hlo_scale_matches_oracle(cuda, layers):
    """BERT stacks at real-HLO scale (> 50k instructions): 400 layers = 26k
    instructions / 1.2k link classes, 1000 layers = 66k instructions / 117k slots / 3k classes
    (the CTA-per-plan kernel).  Outcomes and every slot of the non-conflicting plans match the
    C oracle; short linkage-order prefixes and all-R rows keep conflict-free plans in the batch."""
    g = graphs.bert(layers, 1024, 4096)
    dims = decision_dims(g, g.trainable_variables)
    n = len(dims)
    order = np.asarray([d.flat_index for d in sorted_decision_order(extract_linkage_groups(g, dims))])
    pos = {d.flat_index: i for i, d in enumerate(dims)}
    order = np.asarray([pos[f] for f in order])
    rng = np.random.default_rng(layers)
    short = np.full((96, n), -1, np.int8)
    for b in range(96):
        k = int(rng.integers(1, 12))
        short[b, order[:k]] = rng.integers(0, 2, size=k)
    all_r = np.where(np.arange(n)[None, :] < rng.integers(1, n + 1, size=(16, 1)), 0, -1).astype(np.int8)
    seeds = np.concatenate([random_prefix_seeds(rng, n, 64, order), short, all_r])
    out = PropagationEngine(g, dims).run_batch(torch.from_numpy(seeds), want_slots=True)
    flat = g.flat()
    cand_slots = np.array([flat.slot_offset[d.instruction_id] + d.dim for d in dims])
    st, oc, _ = oracle.propagate_batch(flat, cand_slots, seeds, cand_slots)
    np.testing.assert_array_equal(out["outcome"].cpu().numpy(), oc)
    ok = oc != 2
    assert ok.sum() >= 16
    np.testing.assert_array_equal(out["slots"].cpu().numpy()[ok][:, : flat.num_slots], st[ok])


def test_full_size_batch_properties(cuda):
    """BERT-48 at the bench's batch size (2^20 plans of the workload generator): outcomes and counts
    are consistent (conflict -> zero counts; complete <=> every candidate decided), results are
    deterministic and independent of how the batch is chunked, and sampled rows from across the whole
    batch (first, middle, last) match the C oracle slot for slot."""
    from paper_2007_04069_b200.workloads import prefix_seed_batch

    g = graphs.generate("bert48")
    dims = decision_dims(g, g.trainable_variables)
    n = len(dims)
    order = np.asarray([d.flat_index for d in sorted_decision_order(extract_linkage_groups(g, dims))])
    B = 1 << 20
    seeds = prefix_seed_batch(order, 0, B, device="cuda")
    eng = PropagationEngine(g, dims)
    a = eng.run_batch(seeds, want_slots=True)
    oc, cnt = a["outcome"].long(), a["counts"]
    assert bool(((oc >= 0) & (oc <= 2)).all())
    conf = oc == 2
    assert bool((cnt[conf] == 0).all())
    decided = cnt[:, 0] + cnt[:, 1]
    assert bool(((decided == n) == (oc == 0))[~conf].all())
    assert bool((cnt[:, 2] <= cnt[:, 0]).all()) and bool((cnt[:, 3] <= cnt[:, 1]).all())
    # deterministic, and chunking does not change any row
    b = eng.run_batch(seeds, want_slots=True)
    assert torch.equal(a["outcome"], b["outcome"]) and torch.equal(a["slots"], b["slots"])
    cuts = [0, 333_333, 777_777, B]
    for lo, hi in zip(cuts, cuts[1:]):
        c = eng.run_batch(seeds[lo:hi], want_slots=True)
        assert torch.equal(c["outcome"], a["outcome"][lo:hi]) and torch.equal(c["slots"], a["slots"][lo:hi])
        assert torch.equal(c["counts"], a["counts"][lo:hi])
    rows = np.concatenate([np.arange(64), np.arange(B // 2, B // 2 + 64), np.arange(B - 64, B)])
    flat = g.flat()
    cand_slots = np.array([flat.slot_offset[d.instruction_id] + d.dim for d in dims])
    sub = seeds[torch.from_numpy(rows).cuda()].cpu().numpy()
    st, ocr, _ = oracle.propagate_batch(flat, cand_slots, sub, cand_slots)
    np.testing.assert_array_equal(a["outcome"][torch.from_numpy(rows).cuda()].cpu().numpy(), ocr)
    ok = ocr != 2
    np.testing.assert_array_equal(a["slots"][torch.from_numpy(rows).cuda()].cpu().numpy()[ok][:, : flat.num_slots],
                                  st[ok])


@pytest.mark.parametrize("name", ["bert48", "vgg19"])
def test_run_batch_host_packed_slots_match_int8(cuda, name):
    """run_batch_host(want_slots="packed") (K1 + ap_pack_slots2, 2 bits per slot) decodes to exactly the
    int8 slot rows of the unpacked host path, with ragged chunking (batch not a multiple of the chunk)
    and zero codes past |S|; outcome and counts are unchanged."""
    from paper_2007_04069_b200.sharding import unpack_slots2
    from paper_2007_04069_b200.workloads import prefix_seed_batch

    g = graphs.generate(name)
    dims = decision_dims(g, g.trainable_variables)
    order = np.asarray([d.flat_index for d in sorted_decision_order(extract_linkage_groups(g, dims))])
    B = 5000
    seeds = prefix_seed_batch(order, 7, B).contiguous().pin_memory()
    eng = PropagationEngine(g, dims)
    full = eng.run_batch_host(seeds, want_slots=True, chunk=1536)
    pk = eng.run_batch_host(seeds, want_slots="packed", chunk=1536)
    n = eng._eng.num_slots
    assert "slots" not in pk and pk["slots_packed"].shape == (B, eng.packed_slots_stride)
    assert torch.equal(full["outcome"], pk["outcome"]) and torch.equal(full["counts"], pk["counts"])
    dec = unpack_slots2(pk["slots_packed"].numpy(), n)
    assert np.array_equal(dec, full["slots"][:, :n].numpy())
    tail = pk["slots_packed"].numpy()
    if n % 4:
        assert not (tail[:, n // 4] >> (2 * (n % 4))).any()
    assert not tail[:, (n + 3) // 4:].any()
    with pytest.raises(ValueError):
        eng.run_batch_host(seeds[:4], want_slots="bits")
