"""Drive k_small (C2) or k_fused (C3 bulk) for ncu captures: python tools/prof_kernels.py c2|c3 [iters]."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_18413_b200 import Table
from workloads import random_table, member_to_bitmap, bitmap_to_member, Rng, bulk_removal

which = sys.argv[1]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
p = random_table(5, 20, 100_000, seed=1) if which == "c2" else random_table(8, 100, 10_000_000, seed=3)
tab = Table(p.lo, p.d, p.tuples)
root_m = bitmap_to_member(tab.root_dom, p.d)
rng = Rng(11)
pats = [member_to_bitmap(bulk_removal(rng, root_m, p.d), p.d) for _ in range(8)]
remd = torch.from_numpy(np.stack(pats).view(np.int64)).cuda()
st = tab.root.clone()
out = torch.zeros(tab.Wd, dtype=torch.int64, device="cuda")
sd = torch.zeros(1, dtype=torch.int32, device="cuda")
for k in range(iters):
    st.copy_from(tab.root)
    st.propagate_async(remd[k % 8], out, None, sd)
st.synchronize()
s = st.stats()
print(which, "phase_us", [x / 1e3 for x in s.phase_ns])
tab.close()
