"""C2 (latency config) per-call device phases of k_small, and the same calls
forced through k_wide.  python tools/exp_c2.py"""
import os, sys, time, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2507_18413_b200 import CT_OK, Table
from paper_2507_18413_b200 import ct as C
from workloads import Rng, member_to_bitmap, bitmap_to_member
from workloads.policies import walk_removal
p = bench.c2_problem()
for mode in ("default", "wide"):
    if mode == "wide":
        os.environ["CT_WIDE"] = "1"
    tab = Table(p.lo, p.d, p.tuples)
    os.environ.pop("CT_WIDE", None)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    st = tab.root.clone()
    rem = np.zeros(tab.Wd, np.uint64); out = np.zeros(tab.Wd, np.uint64); pr = np.zeros(tab.Wd, np.uint64)
    fn = C.lib().ct_propagate
    args = (st.handle, rem.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p), pr.ctypes.data_as(ctypes.c_void_p))
    rng = Rng(2, lanes=1)
    cur = root_m.copy()
    lat, ph = [], []
    for k in range(600):
        r = walk_removal(rng, cur, p.d)
        if r is None:
            st.copy_from(tab.root); cur = root_m.copy(); continue
        rem[:] = member_to_bitmap(r, p.d)
        a = time.perf_counter_ns(); s = fn(*args); b = time.perf_counter_ns()
        if k >= 100:
            lat.append((b - a) / 1e3)
            ph.append([x / 1e3 for x in st.stats().phase_ns])
        if s == CT_OK:
            cur = bitmap_to_member(out, p.d)
        else:
            st.copy_from(tab.root); cur = root_m.copy()
    ph = np.array(ph)
    print(mode, C.KERNEL_PATHS[tab.info.kernel_path], "lat p50 %.1f p90 %.1f" % (np.median(lat), np.percentile(lat, 90)),
          "phases p50", np.round(np.median(ph, 0), 2), "sum p50 %.1f" % np.median(ph.sum(1)))
    tab.close()
