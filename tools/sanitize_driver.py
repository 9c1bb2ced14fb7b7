"""Small end-to-end exercise of every launch shape, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): tools/gpu_sanitize.sh runs it
under each tool.  Every call is also checked against the oracle, so a tool
that perturbs timing cannot hide a wrong answer.

Shapes: k_small (C2-like), k_fast with scans and with the gather filter
(banded, 300k tuples), k_fused (grid barrier per phase), per-phase kernels,
k_wide (LIN-like), the tile-major batch path, the negative-table kernels, the
short-table build, and the device-resident DFS (k_model_search)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2507_18413_b200 import CT_OK, CT_FAIL, Table, Model  # noqa: E402
from workloads import (Rng, random_table, banded_table, knapsack_table, short_table, negative_table,  # noqa: E402
                       member_to_bitmap, bitmap_to_member, fix_one_value_removal)
from workloads.csp import csp_model  # noqa: E402
from workloads.policies import walk_removal  # noqa: E402


def walk(tab, p, calls, seed, gac=None):
    gac = gac or (lambda din: oracle.gac(p.lo, p.d, p.tuples, din)[:2])
    ok, root = gac(np.ones(p.R, np.uint8))
    assert (tab.root_status == CT_OK) == ok
    rng = Rng(seed, lanes=1)
    st = tab.root.clone()
    cur = root.copy()
    for _ in range(calls):
        rem = walk_removal(rng, cur, p.d)
        if rem is None:
            st.copy_from(tab.root)
            cur = root.copy()
            continue
        din = cur & (1 - rem)
        ok, dout = gac(din)
        s, dom, _ = st.propagate(member_to_bitmap(rem, p.d))
        assert s == (CT_OK if ok else CT_FAIL)
        if ok:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout)
            cur = dout
        else:
            st.copy_from(tab.root)
            cur = root.copy()
    st.close()


def main():
    from paper_2507_18413_b200 import ct as C
    C.ct_debug_spin_limit(0, 600.0)   # instrumented CTAs are slow: no watchdog trap
    which = sys.argv[1:] or ["small", "fast", "fused", "phases", "wide", "batch", "batchwalk", "serve", "peer", "neg",
                             "short", "model"]
    if "small" in which:
        p = random_table(5, 20, 20_000, seed=1)
        t = Table(p.lo, p.d, p.tuples)
        walk(t, p, 40, 2)
        t.close()
        print("small ok", flush=True)
    if "fast" in which:
        p = banded_table(6, 60, 300_000, seed=4)
        for g in (True, False):
            t = Table(p.lo, p.d, p.tuples, use_gather=g, launch_shape="fast")
            root = bitmap_to_member(t.root_dom, p.d)
            st = t.root.clone()
            rng = Rng(3)
            for _ in range(3):
                rem = fix_one_value_removal(rng, root, p.d, var=0)
                ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, root & (1 - rem))
                st.copy_from(t.root)
                s, dom, _ = st.propagate(member_to_bitmap(rem, p.d))
                assert s == (CT_OK if ok else CT_FAIL)
                if ok:
                    assert np.array_equal(bitmap_to_member(dom, p.d), dout)
            walk(t, p, 10, 5)
            st.close()
            t.close()
        print("fast ok", flush=True)
    if "fused" in which:
        p = random_table(4, 30, 200_000, seed=6)
        t = Table(p.lo, p.d, p.tuples, launch_shape="fused")
        walk(t, p, 10, 7)
        t.close()
        print("fused ok", flush=True)
    if "phases" in which:
        p = random_table(4, 30, 100_000, seed=8)
        t = Table(p.lo, p.d, p.tuples, use_fused=False)
        walk(t, p, 10, 9)
        t.close()
        print("phases ok", flush=True)
    if "wide" in which:
        p = knapsack_table(60, 200, 3000, seed=21)
        t = Table(p.lo, p.d, p.tuples)
        walk(t, p, 10, 10)
        t.close()
        print("wide ok", flush=True)
    if "batch" in which:
        p = random_table(6, 20, 50_000, seed=5)
        t = Table(p.lo, p.d, p.tuples)
        ok, root, _ = oracle.gac(p.lo, p.d, p.tuples, np.ones(p.R, np.uint8))
        b = t.batch(64)
        rng = Rng(11)
        rems = [walk_removal(rng, root, p.d) for _ in range(64)]
        st, doms = b.propagate(np.stack([member_to_bitmap(r, p.d) for r in rems]))
        for s in range(64):
            ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, root & (1 - rems[s]))
            assert st[s] == (CT_OK if ok else CT_FAIL)
            if ok:
                assert np.array_equal(bitmap_to_member(doms[s], p.d), dout)
        b.close()
        t.close()
        print("batch ok", flush=True)
    if "batchwalk" in which:
        # several batch steps, so states thin out: the cell route inside
        # k_bupdate and the sparse-state route (k_bsparse) both run
        p = random_table(6, 50, 60_000, seed=15)
        t = Table(p.lo, p.d, p.tuples)
        ok, root, _ = oracle.gac(p.lo, p.d, p.tuples, np.ones(p.R, np.uint8))
        S = 32
        b = t.batch(S)
        rngs = [Rng(700 + s, lanes=1) for s in range(S)]
        cur = [root.copy() for _ in range(S)]
        for step in range(8):
            rems = []
            for s in range(S):
                r = walk_removal(rngs[s], cur[s], p.d)
                rems.append(r if r is not None else np.zeros(p.R, np.uint8))
            st, doms = b.propagate(np.stack([member_to_bitmap(r, p.d) for r in rems]))
            for s in range(S):
                ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, cur[s] & (1 - rems[s]))
                assert st[s] == (CT_OK if ok else CT_FAIL), (step, s)
                if ok:
                    assert np.array_equal(bitmap_to_member(doms[s], p.d), dout), (step, s)
                    cur[s] = dout
                else:
                    cur[s] = root.copy()
            b.restore_dead(t.root)
        w = b.work()
        assert w["update_sparse_states"] > 0 and w["update_cells_checked"] > 0, w
        b.close()
        t.close()
        print("batchwalk ok", flush=True)
    if "serve" in which:
        p = random_table(5, 20, 20_000, seed=1)
        t = Table(p.lo, p.d, p.tuples)
        ok, root, _ = oracle.gac(p.lo, p.d, p.tuples, np.ones(p.R, np.uint8))
        st = t.root.clone()
        st.serve(True)
        rng = Rng(4, lanes=1)
        cur = root.copy()
        for _ in range(40):
            rem = walk_removal(rng, cur, p.d)
            if rem is None:
                st.copy_from(t.root)
                cur = root.copy()
                continue
            ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, cur & (1 - rem))
            s, dom, _ = st.propagate(member_to_bitmap(rem, p.d))
            assert s == (CT_OK if ok else CT_FAIL)
            if ok:
                assert np.array_equal(bitmap_to_member(dom, p.d), dout)
                cur = dout
            else:
                st.copy_from(t.root)
                cur = root.copy()
        st.close()
        t.close()
        print("serve ok", flush=True)
    if "peer" in which:
        p = random_table(6, 40, 150_000, seed=12)
        t = Table(p.lo, p.d, p.tuples, launch_shape="fast")
        C.ct_peer_attach(t.handle, [C.ct_peer_export(t.handle)])
        walk(t, p, 20, 6)
        t.close()
        print("peer ok", flush=True)
    if "neg" in which:
        p = negative_table(3, 12, 1400, seed=31, lo=1)
        t = Table(p.lo, p.d, p.tuples, kind="negative")
        walk(t, p, 30, 8, gac=lambda din: oracle.gac_negative(p.lo, p.d, p.tuples, din)[:2])
        t.close()
        print("neg ok", flush=True)
    if "short" in which:
        p = short_table(4, 12, 300, seed=7, p_star=0.05)
        t = Table(p.lo, p.d, p.tuples, kind="short")
        walk(t, p, 30, 3, gac=lambda din: oracle.gac_short(p.lo, p.d, p.tuples, din)[:2])
        t.close()
        print("short ok", flush=True)
    if "model" in which:
        m = csp_model(8, 6, 5, 200, seed=81, arities=[3, 4, 2, 5, 3])
        M = Model(m["vlo"], m["vd"], m["scopes"], m["tables"])
        if M.root_status == CT_OK:
            a = M.search(value_order=0, max_solutions=0, max_nodes=300, driver="device")
            b = M.search(value_order=0, max_solutions=0, max_nodes=300, driver="host")
            assert a[2].trace_hash == b[2].trace_hash
        M.close()
        print("model ok", flush=True)


if __name__ == "__main__":
    main()
