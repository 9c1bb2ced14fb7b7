"""Per-item probe timing of one C3 bulk call (needs a -DCT_PROBE_DEBUG build in CT_LIB_PATH)."""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_18413_b200 import Table
from paper_2507_18413_b200 import ct as C
from workloads import random_table, member_to_bitmap, bitmap_to_member, Rng, bulk_removal
p = random_table(8, 100, 10_000_000, seed=3)
tab = Table(p.lo, p.d, p.tuples)
root_m = bitmap_to_member(tab.root_dom, p.d)
rng = Rng(11)
pats = [member_to_bitmap(bulk_removal(rng, root_m, p.d), p.d) for _ in range(8)]
remd = torch.from_numpy(np.stack(pats).view(np.int64)).cuda()
st = tab.root.clone()
out = torch.zeros(tab.Wd, dtype=torch.int64, device="cuda")
sd = torch.zeros(1, dtype=torch.int32, device="cuda")
for k in range(20):
    st.copy_from(tab.root); st.propagate_async(remd[k % 8], out, None, sd)
st.synchronize()
buf = np.zeros((8192, 4), np.uint64)
C.lib().ct_debug_probe_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
s = st.stats()
n = s.n_filter_items
b = buf[:n].astype(np.int64)
t0 = b[:, 0]; t1 = b[:, 1]
dur = (t1 - t0) / 1e3
sm = (buf[:n, 2] >> 32).astype(int); cta = (buf[:n, 2] & 0xffffffff).astype(int)
nl = (buf[:n, 3] >> 32).astype(int); hit = (buf[:n, 3] & 0xffffffff).astype(int) - 1
print("items", n, "probe dur us: min %.2f p50 %.2f p90 %.2f max %.2f" % (dur.min(), np.median(dur), np.percentile(dur, 90), dur.max()))
print("start spread (us, per-SM clocks!)", (t0.max() - t0.min()) / 1e3)
order = np.argsort(-dur)[:12]
for i in order:
    print(f"item {i} cta {cta[i]} sm {sm[i]} dur {dur[i]:.2f} nl {nl[i]} hit {hit[i]}")
# same-SM comparisons: for each SM with >=2 items, spread of end times
from collections import defaultdict
g = defaultdict(list)
for i in range(n): g[sm[i]].append(i)
print("SMs with items:", len(g), "max items per SM:", max(len(v) for v in g.values()))
tab.close()
