"""k_fast per-call phase stamps (ct_stats.phase_ns) for C3-family workloads:
python tools/fast_phases.py [t] [bulk|fix]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18413_b200 import Table
from workloads import random_table, banded_table, member_to_bitmap, bitmap_to_member, Rng, fix_one_value_removal
from workloads.policies import bulk_removal

t = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
kind = sys.argv[2] if len(sys.argv) > 2 else "bulk"
p = random_table(8, 100, t, seed=3) if kind == "bulk" else banded_table(8, 100, t, seed=4)
tab = Table(p.lo, p.d, p.tuples)
root = bitmap_to_member(tab.root_dom, p.d)
rng = Rng(11)
st = tab.root.clone()
ph = []
for k in range(60):
    rem = bulk_removal(rng, root, p.d) if kind == "bulk" else fix_one_value_removal(rng, root, p.d, var=0)
    st.copy_from(tab.root)
    st.propagate(member_to_bitmap(rem, p.d))
    if k >= 10:
        ph.append(list(st.stats().phase_ns))
ph = np.array(ph)
names = ["ingest", "update+barrier", "compact/probe", "p3", "scan/barrier2", "p5", "finalize"]
print(json.dumps({"t": t, "kind": kind, "grid": tab.info.grid, "phase_median_us": dict(zip(names, (np.median(ph, 0) / 1e3).round(2).tolist())),
                  "total_us": float(np.median(ph.sum(1)) / 1e3)}))
