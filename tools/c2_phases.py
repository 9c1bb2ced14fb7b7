"""Per-phase device time of the C2 latency walk (k_small): median of
ct_stats.phase_ns over 1000 P(2, 0.5) calls, plus the C-call latency."""
import ctypes, json, sys, time, os
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
if "--serve" in sys.argv:
    st.serve(True)       # ct_state_serve: the persistent kernel answers the calls
wd = tab.Wd
rem = np.zeros(wd, np.uint64); out = np.zeros(wd, np.uint64); pr = np.zeros(wd, np.uint64)
fn = C.lib().ct_propagate
args = (st.handle, rem.ctypes.data_as(ctypes.c_void_p), out.ctypes.data_as(ctypes.c_void_p), pr.ctypes.data_as(ctypes.c_void_p))
rng = Rng(2, lanes=1)
cur = root_m.copy()
lat, ph, cnt = [], [], []
for k in range(1100):
    r = walk_removal(rng, cur, p.d)
    if r is None:
        st.copy_from(tab.root); cur = root_m.copy(); continue
    rem[:] = member_to_bitmap(r, p.d)
    t0 = time.perf_counter_ns(); s = fn(*args); t1 = time.perf_counter_ns()
    if k >= 100:
        lat.append((t1 - t0) / 1e3)
        x = st.stats()
        ph.append([v / 1e3 for v in x.phase_ns])
        cnt.append([x.words_in, x.words_out, x.n_update_rows, x.n_filter_items, x.n_residue_miss])
    if s == CT_OK:
        cur = bitmap_to_member(out, p.d)
    else:
        st.copy_from(tab.root); cur = root_m.copy()
ph = np.array(ph); cnt = np.array(cnt)
print(json.dumps({"kernel_path": C.KERNEL_PATHS[tab.info.kernel_path],
                  "call_p50_us": float(np.median(lat)), "device_total_p50_us": float(np.median(ph.sum(1))),
                  "phase_p50_us": dict(zip(["ingest", "update", "probe", "scan", "finalize", "p5", "p6"], np.median(ph, 0).tolist())),
                  "phase_mean_us": dict(zip(["ingest", "update", "probe", "scan", "finalize", "p5", "p6"], ph.mean(0).tolist())),
                  "counters_mean": dict(zip(["L_in", "L_out", "rows", "items", "miss"], cnt.mean(0).tolist()))}))

# the same walk with device-resident buffers (ct_propagate_async): the phase
# times without the mapped host-memory read of the removals and the
# system-scope fence of the synchronous path
import torch
rem_d = torch.zeros(wd, dtype=torch.int64, device="cuda")
out_d = torch.zeros(wd, dtype=torch.int64, device="cuda")
st_d = torch.zeros(1, dtype=torch.int32, device="cuda")
st2 = tab.root.clone()
rng = Rng(2, lanes=1)
cur = root_m.copy()
ph2 = []
for k in range(600):
    r = walk_removal(rng, cur, p.d)
    if r is None:
        st2.copy_from(tab.root); cur = root_m.copy(); continue
    rem_d.copy_(torch.from_numpy(member_to_bitmap(r, p.d).view(np.int64)))
    torch.cuda.synchronize()
    st2.propagate_async(rem_d, out_d, None, st_d)
    st2.synchronize()
    if k >= 100:
        ph2.append([v / 1e3 for v in st2.stats().phase_ns])
    if int(st_d.cpu()[0]) == CT_OK:
        cur = bitmap_to_member(out_d.cpu().numpy().view(np.uint64), p.d)
    else:
        st2.copy_from(tab.root); cur = root_m.copy()
ph2 = np.array(ph2)
print(json.dumps({"async_device_buffers": {"device_total_p50_us": float(np.median(ph2.sum(1))),
                  "phase_p50_us": dict(zip(["ingest", "update", "probe", "scan", "finalize", "p5", "p6"], np.median(ph2, 0).tolist()))}}))
