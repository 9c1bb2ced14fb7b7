"""Kernel-only time of the single-state C3 bulk call (ct_table_profile events).
python tools/exp_fast.py [iters]   (CT_LIB_PATH selects a variant build)"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_18413_b200 import Table
from paper_2507_18413_b200 import ct as C
from workloads import random_table, member_to_bitmap, bitmap_to_member, Rng, bulk_removal

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
p = random_table(8, 100, 10_000_000, seed=3)
tab = Table(p.lo, p.d, p.tuples)
root_m = bitmap_to_member(tab.root_dom, p.d)
rng = Rng(11)
pats = [member_to_bitmap(bulk_removal(rng, root_m, p.d), p.d) for _ in range(8)]
remd = torch.from_numpy(np.stack(pats).view(np.int64)).cuda()
st = tab.root.clone()
out = torch.zeros(tab.Wd, dtype=torch.int64, device="cuda")
sd = torch.zeros(1, dtype=torch.int32, device="cuda")
for k in range(10):
    st.copy_from(tab.root); st.propagate_async(remd[k % 8], out, None, sd)
st.synchronize()
C.ct_table_profile(tab.handle, True); C.ct_table_profile_read(tab.handle, reset=True)
for k in range(iters):
    st.copy_from(tab.root); st.propagate_async(remd[k % 8], out, None, sd)
st.synchronize()
prof = C.ct_table_profile_read(tab.handle, reset=True)
s = st.stats()
print(os.environ.get("CT_TAG", "default"), json.dumps({k: round(v[1] / v[0] * 1e3, 2) for k, v in prof.items() if v[0]}),
      "phases", [round(x / 1e3, 2) for x in s.phase_ns], "grid", tab.info.grid)
tab.close()
