# one full-chunk run_batch_host(want_slots="packed") on BERT-48 (65,536 plans), for ncu of pack_slots2_kernel
import sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2007_04069_b200 import graphs
from paper_2007_04069_b200.ir import decision_dims
from paper_2007_04069_b200.linkage import extract_linkage_groups, sorted_decision_order
from paper_2007_04069_b200.sharding import PropagationEngine
from paper_2007_04069_b200.workloads import prefix_seed_batch
g = graphs.generate("bert48"); dims = decision_dims(g, g.trainable_variables)
order = np.asarray([d.flat_index for d in sorted_decision_order(extract_linkage_groups(g, dims))])
seeds = prefix_seed_batch(order, 0, 1 << 16).contiguous().pin_memory()
eng = PropagationEngine(g, dims)
for _ in range(3): eng.run_batch_host(seeds, want_slots="packed")
torch.cuda.synchronize(); print("ok")
