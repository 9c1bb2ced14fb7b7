import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
from paper_2507_18413_b200 import CT_OK, CT_FAIL, Table
from workloads import Rng, random_table, member_to_bitmap, bitmap_to_member
from workloads.policies import walk_removal
from workloads.layout import bits_to_bool
n, d, t, lo = 10, 140, 60_005, -2
p = random_table(n, d, t, seed=5, lo=lo)
tab = Table(p.lo, p.d, p.tuples)
print("batch_tile", tab.info.batch_tile, "W", tab.info.words)
S = 67
b = tab.batch(S)
root_m = bitmap_to_member(tab.root_dom, p.d)
cur = [root_m.copy() for _ in range(S)]
rngs = [Rng(1000 + s, lanes=1) for s in range(S)]
for step in range(10):
    rem = np.zeros((S, tab.Wd), np.uint64)
    exp = []
    for s in range(S):
        r = walk_removal(rngs[s], cur[s], p.d)
        if r is None:
            r = np.zeros(p.R, np.uint8)
        rem[s] = member_to_bitmap(r, p.d)
        exp.append(oracle.gac(p.lo, p.d, p.tuples, cur[s] & (1 - r), want_valid=True))
    status, doms = b.propagate(rem)
    bad = 0
    for s in range(S):
        ok, dout, valid = exp[s]
        g_ok = status[s] == CT_OK
        if g_ok != ok:
            bad += 1
            T = bits_to_bool(b.read_table(s), p.t)
            print(f"step {step} state {s}: status gpu={status[s]} oracle_ok={ok} valid={valid.sum()} gpuT={T.sum()}")
        elif ok and not np.array_equal(bitmap_to_member(doms[s], p.d), dout):
            bad += 1
            T = bits_to_bool(b.read_table(s), p.t)
            g = bitmap_to_member(doms[s], p.d)
            print(f"step {step} state {s}: domains differ: gpu-only {np.nonzero(g & (1-dout))[0][:10]} oracle-only {np.nonzero(dout & (1-g))[0][:10]} valid={valid.sum()} gpuT={T.sum()} Tdiff={(T != valid).sum()}")
        if ok:
            cur[s] = dout
        else:
            cur[s] = root_m.copy()
    b.restore_dead(tab.root)
    if bad:
        print("step", step, "bad", bad)
        break
print("done")
