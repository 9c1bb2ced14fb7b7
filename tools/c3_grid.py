"""C3 bulk device time per call vs k_fast's grid (ct_config.grid_override)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2507_18413_b200 import Table
from workloads import random_table, member_to_bitmap, bitmap_to_member, Rng
from workloads.policies import bulk_removal

p = random_table(8, 100, 10_000_000, seed=3)
out = {}
for g in [int(x) for x in (sys.argv[1:] or ["0", "296", "148", "370"])]:
    tab = Table(p.lo, p.d, p.tuples, grid_override=g)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    rng = Rng(11)
    rems = [torch.from_numpy(member_to_bitmap(bulk_removal(rng, root_m, p.d), p.d).view(np.int64)).cuda() for _ in range(16)]
    od = torch.zeros(tab.Wd, dtype=torch.int64, device="cuda"); sd = torch.zeros(1, dtype=torch.int32, device="cuda")
    w = tab.root.clone()
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(tab.stream_ptr)
    for k in range(20):
        w.propagate_from_async(tab.root, rems[k % 16], od, None, sd)
    w.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(300):
        w.propagate_from_async(tab.root, rems[k % 16], od, None, sd)
    e1.record(stream)
    e1.synchronize()
    out[g] = {"us_per_call": e0.elapsed_time(e1) / 300 * 1e3, "grid": tab.info.grid}
    w.close()
    tab.close()
print(json.dumps(out))
