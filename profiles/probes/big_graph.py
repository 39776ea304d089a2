# K1 at real-HLO scale (> 50k instructions): BERT stacks of 400 / 1000 layers
import sys, time; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from oracle import oracle
from paper_2007_04069_b200 import graphs
from paper_2007_04069_b200.ir import decision_dims
from paper_2007_04069_b200.linkage import sorted_decision_order, extract_linkage_groups
from paper_2007_04069_b200.sharding import PropagationEngine
from paper_2007_04069_b200.workloads import prefix_seed_batch
for L in [int(x) for x in sys.argv[1:]] or [48, 400, 1000]:
    g = graphs.bert(L, 1024, 4096)
    dims = decision_dims(g, g.trainable_variables)
    t0 = time.perf_counter()
    eng = PropagationEngine(g, dims)
    dev = eng._eng.device()
    torch.cuda.synchronize(); t1 = time.perf_counter()
    groups = extract_linkage_groups(g, dims)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    order_i = np.asarray([d.flat_index for d in sorted_decision_order(groups)], dtype=np.int64)
    B = 1 << 16
    seeds = prefix_seed_batch(order_i, 0, B, device="cuda")
    out = eng.run_batch(seeds, want_slots=True)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): out = eng.run_batch(seeds, want_slots=True)
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 5
    flat = g.flat()
    cand = np.array([flat.slot_offset[d.instruction_id] + d.dim for d in dims])
    sub = seeds[:256].cpu().numpy()
    t3 = time.perf_counter()
    st, oc, _ = oracle.propagate_batch(flat, cand, sub, cand)
    t4 = time.perf_counter()
    ok = oc != 2
    same = np.array_equal(out["outcome"][:256].cpu().numpy(), oc) and np.array_equal(out["slots"][:256].cpu().numpy()[ok], st[ok])
    print(f"L={L} instrs={len(g.instructions)} slots={flat.num_slots} dims={len(dims)} classes={getattr(dev, 'num_classes', '?')} "
          f"ingest {t1-t0:.3f}s linkage {t2-t1:.2f}s  K1 {B / (ms / 1e3) / 1e6:.1f} M plans/s ({ms:.2f} ms / {B})  "
          f"oracle {256 / (t4 - t3):.0f} plans/s  parity(256)={same} conflict={float((out['outcome'] == 2).float().mean()):.3f}", flush=True)
