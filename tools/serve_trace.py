"""Served C2 calls with the -DCT_SERVE_TRACE variant library: median time
between the stamps of k_small_serve / small_call / warp_ingest (ns)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2507_18413_b200 import CT_OK, Table
from paper_2507_18413_b200 import ct as C
from workloads import Rng, random_table, member_to_bitmap, bitmap_to_member
from workloads.policies import walk_removal

p = random_table(5, 20, 100_000, seed=1)
tab = Table(p.lo, p.d, p.tuples)
root_m = bitmap_to_member(tab.root_dom, p.d)
st = tab.root.clone()
st.serve(True)
rng = Rng(2, lanes=1)
cur = root_m.copy()
tr = np.zeros(16, np.int64)
rows = []
for k in range(800):
    r = walk_removal(rng, cur, p.d)
    if r is None:
        st.copy_from(tab.root); cur = root_m.copy(); continue
    s, dom, _ = st.propagate(member_to_bitmap(r, p.d))
    C.lib().ct_debug_serve_trace(st.handle, tr.ctypes.data_as(ctypes.c_void_p))
    if k >= 100:
        rows.append(tr.copy())
    if s == CT_OK:
        cur = bitmap_to_member(dom, p.d)
    else:
        st.copy_from(tab.root); cur = root_m.copy()
R = np.array(rows)
order = [0, 1, 2, 3, 4, 5, 6, 7, 8, 15]
names = ["detect", "call", "ingest:dom+dead", "ingest:phase1", "ingest:rows", "ingest:ctl", "ingest sync",
         "update", "probe", "finalize"]
out = {}
for a, b, nm in zip(order[:-1], order[1:], names[1:]):
    d = R[:, b] - R[:, a]
    out[nm] = float(np.median(d))
out["total"] = float(np.median(R[:, 15] - R[:, 0]))
print(json.dumps(out))
