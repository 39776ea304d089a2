"""Parity at the bench's own plan distributions, and K1's other output modes (GPU).

* Every batch bench.py times on BERT-48 (the headline decision-order prefixes, the 2|D| linkage
  triggers tiled, prefixes k~U[1,16]) built from the reference's decision order
  (tests/golden/linkage_bert48.npz): >= 1,000 conflict-free rows of each are slot-checked against
  the C oracle (every slot, outcome, decided/newly counts), plus the outcome of sampled conflict
  rows.  The headline batch is 99.8% CONFLICT, so its conflict-free rows are collected from the
  first 2^21 rows.
* K1's packed output (ap_propagate_batch_packed: 2-bit codes emitted by K1 itself) decodes to the
  int8 rows bit for bit on every BASELINE graph, through the fast kernel (k <= 4 and k <= 8 chunk
  paths) and the generic kernel + pack fallback; outcome / counts / candidate statuses unchanged.
* AP_K1_BULK=1 (slot rows staged in shared memory, TMA bulk stores) is bit-identical to the
  per-lane stores.
"""

import numpy as np
import pytest
import torch

from oracle import oracle
from paper_2007_04069_b200 import graphs
from paper_2007_04069_b200.ir import decision_dims
from paper_2007_04069_b200.sharding import PropagationEngine, unpack_slots2
from paper_2007_04069_b200.workloads import prefix_seed_batch, trigger_seed_batch

pytestmark = pytest.mark.gpu
GOLDEN_ORDER = {}


def bert48():
    g = graphs.generate("bert48")
    dims = decision_dims(g, g.trainable_variables)
    if "bert48" not in GOLDEN_ORDER:
        from goldens import GOLDEN

        GOLDEN_ORDER["bert48"] = np.load(GOLDEN / "linkage_bert48.npz")["order"]
    return g, dims, GOLDEN_ORDER["bert48"]


def padded(rows):
    """Copy int8 seed rows into a 16-byte row stride (the fast kernel's seed loads)."""
    B, n = rows.shape
    out = torch.full((B, max(16, (n + 15) // 16 * 16)), -1, dtype=torch.int8, device=rows.device)[:, :n]
    out.copy_(rows)
    return out


def oracle_check(g, dims, seeds_np, outcome, counts, slots):
    flat = g.flat()
    cand = np.array([flat.slot_offset[d.instruction_id] + d.dim for d in dims])
    st, oc, _ = oracle.propagate_batch(flat, cand, seeds_np, cand)
    np.testing.assert_array_equal(outcome, oc)
    ok = oc != 2
    np.testing.assert_array_equal(slots[ok][:, : flat.num_slots], st[ok])
    # counts: decided P / R over candidates, newly = decided and not seeded (sharding.py:240-245)
    cs = st[:, cand]
    seeded = seeds_np != -1
    want = np.stack([(cs == 1).sum(1), (cs == 0).sum(1), ((cs == 1) & ~seeded).sum(1),
                     ((cs == 0) & ~seeded).sum(1)], 1)
    np.testing.assert_array_equal(counts[ok], want[ok])
    assert not counts[~ok].any()
    return int(ok.sum())


@pytest.mark.parametrize("batch", ["headline", "triggers", "short_prefix"])
def test_bench_batch_conflict_free_rows_match_oracle(cuda, batch):
    g, dims, order = bert48()
    n = len(dims)
    eng = PropagationEngine(g, dims)
    B = 1 << 21 if batch == "headline" else 1 << 16
    if batch == "headline":
        seeds = prefix_seed_batch(order, 0, B, device="cuda", chunk=1 << 18)
    elif batch == "triggers":
        seeds = trigger_seed_batch(n, 0, B, device="cuda")
    else:
        seeds = prefix_seed_batch(order, 0, B, device="cuda", chunk=1 << 18, kmax=16)
    out = {"outcome": torch.empty(B, dtype=torch.uint8, device="cuda"),
           "counts": torch.empty((B, 4), dtype=torch.int32, device="cuda")}
    eng.launch(seeds, out["outcome"], out["counts"])  # outcome pass over the whole batch
    free = torch.nonzero(out["outcome"] != 2).flatten()
    assert free.numel() >= 1000, f"only {free.numel()} conflict-free rows"
    rng = np.random.default_rng(5)
    pick_free = free[torch.from_numpy(rng.choice(free.numel(), 1000, replace=False)).cuda()]
    conf = torch.nonzero(out["outcome"] == 2).flatten()
    pick_conf = conf[torch.from_numpy(rng.choice(conf.numel(), min(200, conf.numel()), replace=False)).cuda()] \
        if conf.numel() else conf
    rows = torch.cat([pick_free, pick_conf]).sort().values
    sub = padded(seeds[rows])
    slots = torch.empty((rows.numel(), eng.slots_stride), dtype=torch.int8, device="cuda")
    oc = torch.empty(rows.numel(), dtype=torch.uint8, device="cuda")
    cnt = torch.empty((rows.numel(), 4), dtype=torch.int32, device="cuda")
    eng.launch(sub, oc, cnt, slots)
    assert torch.equal(oc, out["outcome"][rows]) and torch.equal(cnt, out["counts"][rows])
    checked = oracle_check(g, dims, sub.cpu().numpy(), oc.cpu().numpy(), cnt.cpu().numpy(), slots.cpu().numpy())
    assert checked >= 1000


@pytest.mark.parametrize("name", ["mlp2", "bert_base", "bert48", "vgg19", "t5_large"])
@pytest.mark.parametrize("generic", [False, True])
def test_packed_k1_matches_int8_rows(cuda, monkeypatch, name, generic):
    if generic:
        monkeypatch.setenv("AP_PROPAGATE_GENERIC", "1")
    g = graphs.generate(name)
    dims = decision_dims(g, g.trainable_variables)
    n = len(dims)
    eng = PropagationEngine(g, dims)
    rows = torch.cat([prefix_seed_batch(np.arange(n), 3, 3001, device="cuda"),
                      trigger_seed_batch(n, 0, 2 * n, device="cuda"),
                      torch.full((1, n), -1, dtype=torch.int8, device="cuda")])
    B = rows.shape[0]
    seeds = padded(rows)

    def run(packed):
        o = {"outcome": torch.empty(B, dtype=torch.uint8, device="cuda"),
             "counts": torch.empty((B, 4), dtype=torch.int32, device="cuda"),
             "statuses": torch.empty((B, max(16, (n + 15) // 16 * 16)), dtype=torch.int8, device="cuda")}
        if packed:
            o["packed"] = torch.full((B, eng.packed_slots_stride + 8), 0xAB, dtype=torch.uint8, device="cuda")
            eng.launch(seeds, o["outcome"], o["counts"], None, o["statuses"], packed=o["packed"][:, :eng.packed_slots_stride])
        else:
            o["slots"] = torch.empty((B, eng.slots_stride), dtype=torch.int8, device="cuda")
            eng.launch(seeds, o["outcome"], o["counts"], o["slots"], o["statuses"])
        return o

    a, p = run(False), run(True)
    for k in ("outcome", "counts", "statuses"):
        assert torch.equal(a[k][:, : n] if k == "statuses" else a[k], p[k][:, : n] if k == "statuses" else p[k]), k
    S = eng._eng.num_slots
    pk = p["packed"].cpu().numpy()
    np.testing.assert_array_equal(unpack_slots2(pk[:, : eng.packed_slots_stride], S), a["slots"][:, :S].cpu().numpy())
    # zero codes past |S| inside the row, untouched bytes past the row stride
    codes = (pk[:, : eng.packed_slots_stride, None] >> np.array([0, 2, 4, 6], np.uint8)) & 3
    assert not codes.reshape(B, -1)[:, S:].any()
    assert (pk[:, eng.packed_slots_stride:] == 0xAB).all()


def test_bulk_store_rows_match_plain(cuda, monkeypatch):
    g, dims, order = bert48()
    eng = PropagationEngine(g, dims)
    B = 40000
    seeds = prefix_seed_batch(order, 11, B, device="cuda")
    outs = []
    for bulk in ("0", "1"):
        monkeypatch.setenv("AP_K1_BULK", bulk)
        o = torch.empty(B, dtype=torch.uint8, device="cuda")
        c = torch.empty((B, 4), dtype=torch.int32, device="cuda")
        s = torch.full((B, eng.slots_stride), 7, dtype=torch.int8, device="cuda")
        eng.launch(seeds, o, c, s)
        outs.append((o, c, s))
    for x, y in zip(*outs):
        assert torch.equal(x, y)


def test_launch_rejects_wrong_seed_width(cuda):
    g, dims, order = bert48()
    eng = PropagationEngine(g, dims)
    bad = torch.full((4, len(dims) - 1), -1, dtype=torch.int8, device="cuda")
    with pytest.raises(ValueError):
        eng.launch(bad, torch.empty(4, dtype=torch.uint8, device="cuda"))
    with pytest.raises(ValueError):
        eng.run_batch_host(torch.full((4, len(dims) + 1), -1, dtype=torch.int8))


@pytest.mark.parametrize("name", ["mlp2", "vgg19", "attention_block", "t5_block"])
@pytest.mark.parametrize("mode", ["full", "packed"])
def test_lane_kernel_matches_warp_kernel(cuda, monkeypatch, name, mode):
    """K1-lane (one thread per plan, small graphs) == the warp-per-plan kernel, every output,
    including UNDECIDED seeds, all-unseeded rows and conflict rows."""
    from goldens import load_prop

    g = graphs.generate(name) if name in ("mlp2", "vgg19") else load_prop(name).graph
    dims = decision_dims(g, g.trainable_variables)
    n = len(dims)
    eng = PropagationEngine(g, dims)
    rng = np.random.default_rng(9)
    rows = np.concatenate([
        rng.integers(-1, 2, size=(3000, n)),                 # P / R / unseeded
        rng.integers(-1, 3, size=(500, n)),                  # with UNDECIDED seeds
        np.full((1, n), -1), np.zeros((1, n)),
    ]).astype(np.int8)
    seeds = padded(torch.from_numpy(rows).cuda())
    B = seeds.shape[0]

    def run():
        o = {"outcome": torch.empty(B, dtype=torch.uint8, device="cuda"),
             "counts": torch.empty((B, 4), dtype=torch.int32, device="cuda"),
             "statuses": torch.empty((B, max(16, (n + 15) // 16 * 16)), dtype=torch.int8, device="cuda")}
        if mode == "packed":
            o["packed"] = torch.zeros((B, eng.packed_slots_stride), dtype=torch.uint8, device="cuda")
            eng.launch(seeds, o["outcome"], o["counts"], None, o["statuses"], packed=o["packed"])
        else:
            o["slots"] = torch.zeros((B, eng.slots_stride), dtype=torch.int8, device="cuda")
            eng.launch(seeds, o["outcome"], o["counts"], o["slots"], o["statuses"])
        o["statuses"] = o["statuses"][:, :n]
        return o

    monkeypatch.setenv("AP_K1_LANE", "0")
    warp = run()
    monkeypatch.setenv("AP_K1_LANE", "1")
    lane = run()
    for k in warp:
        assert torch.equal(warp[k], lane[k]), k
