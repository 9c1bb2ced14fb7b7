"""LIN-shaped (knapsack) table: per-call latency of ct_propagate on a P(2,0.5)
walk, device phase times, and the kernel path.  python tools/exp_lin.py [preset]"""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18413_b200 import CT_OK, Table
from paper_2507_18413_b200 import ct as C
from workloads import Rng, knapsack_table, LIN_PRESETS, member_to_bitmap, bitmap_to_member
from workloads.policies import walk_removal
preset = sys.argv[1] if len(sys.argv) > 1 else "lin_b"
p = knapsack_table(seed=21, **LIN_PRESETS[preset])
t0 = time.time()
tab = Table(p.lo, p.d, p.tuples)
print(preset, "n", p.n, "t", p.t, "R", p.R, "W", tab.info.words, "path", C.KERNEL_PATHS.get(tab.info.kernel_path),
      "build_s %.3f" % (time.time() - t0))
root_m = bitmap_to_member(tab.root_dom, p.d)
st = tab.root.clone()
rng = Rng(2, lanes=1)
cur = root_m.copy()
lat, dev, items = [], [], []
rem = np.zeros(tab.Wd, np.uint64); out = np.zeros(tab.Wd, np.uint64); pr = np.zeros(tab.Wd, np.uint64)
fn = C.lib().ct_propagate
args = (st.handle, rem.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p), pr.ctypes.data_as(ctypes.c_void_p))
fails = 0
for k in range(400):
    r = walk_removal(rng, cur, p.d)
    if r is None:
        st.copy_from(tab.root); cur = root_m.copy(); continue
    rem[:] = member_to_bitmap(r, p.d)
    a = time.perf_counter_ns(); s = fn(*args); b = time.perf_counter_ns()
    if k >= 50:
        lat.append((b - a) / 1e3)
        ss = st.stats()
        dev.append([x / 1e3 for x in ss.phase_ns[:5]])
        items.append(ss.n_filter_items)
    if s == CT_OK:
        cur = bitmap_to_member(out, p.d)
    else:
        fails += 1
        st.copy_from(tab.root); cur = root_m.copy()
dev = np.array(dev)
print("calls", len(lat), "fails", fails, "lat p50 %.1f p90 %.1f us" % (np.median(lat), np.percentile(lat, 90)),
      "items p50", int(np.median(items)), "phases p50 (ingest,update,probe,scan,fin)", np.round(np.median(dev, 0), 2))
tab.close()
