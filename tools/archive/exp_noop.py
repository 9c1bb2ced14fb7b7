"""Launch overhead of k_fast: event time of no-op calls (nothing removed) vs bulk calls on C3."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2507_18413_b200 import Table
from paper_2507_18413_b200 import ct as C
from workloads import member_to_bitmap, bitmap_to_member
p = bench.c3_problem()
tab = Table(p.lo, p.d, p.tuples)
st = tab.root.clone()
zero = torch.zeros(tab.Wd, dtype=torch.int64, device="cuda")
out = torch.zeros(tab.Wd, dtype=torch.int64, device="cuda")
sd = torch.zeros(1, dtype=torch.int32, device="cuda")
stream = torch.cuda.ExternalStream(tab.stream_ptr)
for k in range(20):
    st.propagate_async(zero, out, None, sd)
st.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for k in range(500):
    st.propagate_async(zero, out, None, sd)
e1.record(stream)
e1.synchronize()
print("noop k_fast call: %.2f us per call (back to back)" % (e0.elapsed_time(e1) * 1e3 / 500))
s = st.stats()
print("phases of the last noop call (us):", [round(x / 1e3, 2) for x in s.phase_ns])
# copy_from alone
e0.record(stream)
for k in range(500):
    st.copy_from(tab.root)
e1.record(stream)
e1.synchronize()
print("ct_state_copy: %.2f us per copy" % (e0.elapsed_time(e1) * 1e3 / 500))
tab.close()
