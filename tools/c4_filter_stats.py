"""C4 steps: the filter side per step (probe misses, scan words) from ct_batch_work."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18413_b200 import Table
from workloads import random_table
from workloads.policies import batch_coin_removals

p = random_table(6, 50, 1_000_000, seed=5)
tab = Table(p.lo, p.d, p.tuples)
S = 4096
b = tab.batch(S)
pats = batch_coin_removals(p.n, p.d, S, 16, seed=6)
rows = []
for k in range(40):
    b.propagate(pats[k % 16])
    w = b.work(reset=True)
    if k >= 10:
        rows.append((w["probe_misses"], w["filter_support_words"], w["update_sparse_states"]))
    b.restore_dead(tab.root)
r = np.array(rows)
print(json.dumps({"probe_misses_per_step": float(r[:, 0].mean()), "scan_words_per_step": float(r[:, 1].mean()),
                  "sparse_states": float(r[:, 2].mean())}))
