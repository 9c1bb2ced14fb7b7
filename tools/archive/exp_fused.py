"""Experiment: fused vs per-phase kernels, cooperative vs plain launch (GPU)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2507_18413_b200 import Table
from paper_2507_18413_b200 import ct as C
from workloads import random_table, member_to_bitmap, bitmap_to_member, Rng, bulk_removal

def run(p, fused, steps=200):
    tab = Table(p.lo, p.d, p.tuples, use_fused=fused)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    rng = Rng(11)
    pats = [member_to_bitmap(bulk_removal(rng, root_m, p.d), p.d) for _ in range(8)]
    remd = torch.from_numpy(np.stack(pats).view(np.int64)).cuda()
    st = tab.root.clone()
    out = torch.zeros(tab.Wd, dtype=torch.int64, device='cuda'); sd = torch.zeros(1, dtype=torch.int32, device='cuda')
    for k in range(20):
        st.copy_from(tab.root); st.propagate_async(remd[k % 8], out, None, sd)
    st.synchronize()
    s = st.stats()
    C.ct_table_profile(tab.handle, True); C.ct_table_profile_read(tab.handle)
    t0 = time.perf_counter()
    for k in range(steps):
        st.copy_from(tab.root); st.propagate_async(remd[k % 8], out, None, sd)
    st.synchronize()
    wall = (time.perf_counter() - t0) / steps * 1e6
    prof = C.ct_table_profile_read(tab.handle)
    tab.close()
    return dict(fused=fused, wall_us=wall, prof={k: (v[1] / v[0] * 1e3 if v[0] else None) for k, v in prof.items()},
                phase_us=[x / 1e3 for x in s.phase_ns])

for name, p in [("C2", random_table(5, 20, 100_000, seed=1)), ("C3", random_table(8, 100, 10_000_000, seed=3))]:
    for fused in (False, True):
        print(name, json.dumps(run(p, fused)), flush=True)
