"""Per-CTA phase timestamps of one k_fast call (needs a -DCT_FAST_TRACE build in
CT_LIB_PATH).  python tools/exp_trace.py [c3bulk|c3b]"""
import os, sys, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2507_18413_b200 import Table
from paper_2507_18413_b200 import ct as C
from workloads import member_to_bitmap, bitmap_to_member
wl = sys.argv[1] if len(sys.argv) > 1 else "c3bulk"
p = bench.c3_problem() if wl == "c3bulk" else bench.c3b_problem()
tab = Table(p.lo, p.d, p.tuples)
root_m = bitmap_to_member(tab.root_dom, p.d)
pats = bench.bulk_patterns(root_m, p.d, 8) if wl == "c3bulk" else bench.fix_patterns(root_m, p.d, 8)
remd = torch.from_numpy(np.stack([member_to_bitmap(m, p.d) for m in pats]).view(np.int64)).cuda()
st = tab.root.clone()
out = torch.zeros(tab.Wd, dtype=torch.int64, device="cuda")
sd = torch.zeros(1, dtype=torch.int32, device="cuda")
G = tab.info.grid
names = ["start", "ingest", "update", "barrier1", "compact", "probe", "barrier2", "scan", "done"]
acc = []
for k in range(30):
    st.copy_from(tab.root); st.propagate_async(remd[k % 8], out, None, sd)
    st.synchronize()
    if k >= 10:
        buf = np.zeros((4096, 10), np.uint64)
        C.lib().ct_debug_trace_read(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(buf.nbytes))
        t = buf[:G, :9].astype(np.int64)
        t0 = t[:, 0].min()
        acc.append((t - t0) / 1e3)
a = np.stack(acc)          # [calls][G][9] us from the first CTA start
print(wl, "grid", G, "phase stats over", a.shape[0], "calls (us since first CTA start): min / median / max over CTAs")
for i, nm in enumerate(names):
    col = a[:, :, i]
    if (col == 0).all() or (col < -1e6).any():
        continue
    print(f"{nm:9s} {np.median(col.min(1)):8.2f} {np.median(np.median(col, 1)):8.2f} {np.median(col.max(1)):8.2f}")
tab.close()
