"""C4 batched workload counters: per-step totals of the work the batch kernels do
(ct_batch_stats) next to the per-kernel event times.  python tools/exp_c4.py"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2507_18413_b200 import Table
from paper_2507_18413_b200 import ct as C

p = bench.c4_problem()
S = 4096
tab = Table(p.lo, p.d, p.tuples)
b = tab.batch(S)
K = 16
pats = bench.c4_patterns(p, S, K, seed=6)
rem = [torch.from_numpy(x.view(np.int64)).cuda() for x in pats]
out = torch.zeros((S, tab.Wd), dtype=torch.int64, device="cuda")
st = torch.zeros(S, dtype=torch.int32, device="cuda")
tot = {}
for k in range(40):
    if k == 20:
        C.ct_table_profile(tab.handle, True); C.ct_table_profile_read(tab.handle, reset=True)
    b.propagate_async(rem[k % K], out, st)
    if k >= 20:
        ss = b.stats()
        for f in ("words_in", "words_out", "n_update_rows", "update_support_words", "update_table_writes",
                  "filter_support_words", "n_filter_items", "n_residue_miss", "noop"):
            tot[f] = tot.get(f, 0) + sum(getattr(s, f) for s in ss)
        tot["fail"] = tot.get("fail", 0) + int((st.cpu().numpy() == 1).sum())
        tot["dead_in"] = tot.get("dead_in", 0) + sum(1 for s in ss if s.last_status == -5)
        for kk, vv in b.work(reset=True).items():
            tot["work_" + kk] = tot.get("work_" + kk, 0) + vv
    b.restore_dead(tab.root)
prof = C.ct_table_profile_read(tab.handle, reset=True)
steps = 20
print(json.dumps({k: v / steps for k, v in tot.items()}))
print(json.dumps({k: round(v[1] / max(v[0], 1), 4) for k, v in prof.items() if v[0]}))
sw = tot["work_update_support_words"]
print("update support words/step %.1f MB" % (8 * sw / steps / 1e6))
tab.close()
