"""GPU parity at the BASELINE configs' OWN sizes, in the launch configuration
bench.py times (SURVEY §8(d) "Oracle timing" / parity rows):

  C3 walk   1e7 tuples, 1000 policy-P(2, 0.5) calls (seed 11), every call vs
            the oracle (status, domains, pruned; currTable every 100 calls)
  C3b       banded 1e7 tuples, 3 calls fixing x0 (bench.py's seeded patterns)
  C4        4096 states x 100 batch steps of the 1e6-tuple table: all 4096
            states for the first 3 steps, then 128 seeded states for all 100
  C5        12 tables x 1e6 tuples: the first 1000 DFS nodes' trace vs oracle.dfs
  C3 / C3b at t = 1e6 (the HBM target's second size): a 300-call
            walk, and 3 calls fixing x0 (gather filter and Alg. 3 scans)

The oracle runs its tuple scan over every host core (oracle_gac_split, pinned
to the single-thread oracle in tests/test_oracle.py); every oracle input comes
from the oracle's previous output, never from the CUDA path.
"""
import numpy as np
import pytest

import oracle
from ctharness import check_root, oracle_call, run_walk
from paper_2507_18413_b200 import CT_OK, CT_FAIL, Table, Model
from workloads import (Rng, random_table, banded_table, member_to_bitmap, bitmap_to_member,
                       fix_one_value_removal)
from workloads.layout import bits_to_bool

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.mark.timeout(1800)
def test_c3_walk_1000_calls_full_size():
    p = random_table(8, 100, 10_000_000, seed=3)
    tab = Table(p.lo, p.d, p.tuples)
    nfail, nsolved = run_walk(tab, p, calls=1000, seed=11, check_table_every=100)
    assert nfail > 0
    tab.close()


@pytest.mark.timeout(900)
def test_c3b_banded_full_size():
    p = banded_table(8, 100, 10_000_000, seed=4)
    tab = Table(p.lo, p.d, p.tuples)
    ok, root_m = check_root(tab, p)
    assert ok
    rng = Rng(12)                                     # bench.py fix_patterns
    st = tab.root.clone()
    for k in range(3):
        rem = fix_one_value_removal(rng, root_m, p.d, var=0)
        din = root_m & (1 - rem)
        ok, dout, valid = oracle_call(p, din, want_valid=True)
        st.copy_from(tab.root)
        status, dom, pr = st.propagate(member_to_bitmap(rem, p.d))
        assert status == (CT_OK if ok else CT_FAIL), k
        if ok:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout), k
            assert np.array_equal(bitmap_to_member(pr, p.d), din & (1 - dout)), k
            assert np.array_equal(bits_to_bool(st.read_table(), p.t), valid), k
        assert st.stats().n_residue_miss > 0          # the full-scan filter ran
    st.close()
    tab.close()


@pytest.mark.timeout(2400)
def test_c4_batch_full_size():
    """bench.py --workload c4's step: ct_propagate_many of seeded per-state
    removals, then ct_batch_restore_dead(root) on the device."""
    from workloads.policies import batch_coin_removals
    p = random_table(6, 50, 1_000_000, seed=5)
    tab = Table(p.lo, p.d, p.tuples)
    assert tab.info.batch_tile == 32                  # the tile-major path bench.py times
    S, steps, K = 4096, 100, 16
    b = tab.batch(S)
    pats = batch_coin_removals(p.n, p.d, S, K, seed=6)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    watched = set(range(0, S, S // 128))              # 128 seeded states for all steps
    cur = {s: root_m.copy() for s in range(S)}
    th = oracle.host_threads()
    n_checked = n_fail = 0
    for step in range(steps):
        rem = pats[step % K]
        status, doms = b.propagate(rem)
        check = range(S) if step < 3 else sorted(watched)
        for s in check:
            r = bitmap_to_member(rem[s], p.d)
            ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, cur[s] & (1 - r), threads=th)
            assert status[s] == (CT_OK if ok else CT_FAIL), (step, s)
            if ok:
                assert np.array_equal(bitmap_to_member(doms[s], p.d), dout), (step, s)
                cur[s] = dout
            else:
                cur[s] = root_m.copy()                # restored by ct_batch_restore_dead below
                n_fail += 1
            n_checked += 1
        if step == 2:
            cur = {s: cur[s] for s in watched}
        b.restore_dead(tab.root)
    assert n_checked == 3 * S + 97 * 128 and n_fail > 0
    b.close()
    tab.close()


@pytest.mark.timeout(2400)
def test_c5_first_1000_nodes_full_size():
    from oracle.dfs import dfs as oracle_dfs
    from workloads.csp import csp_model
    m = csp_model(30, 40, 12, 1_000_000, seed=7)
    M = Model(m["vlo"], m["vd"], m["scopes"], m["tables"])
    st, sol, stats = M.search(value_order=0, max_nodes=1000, max_solutions=0, driver="device")
    ref = oracle_dfs(m["vlo"], m["vd"], m["scopes"], m["tables"], value_order=0, max_nodes=1000,
                     max_solutions=0, threads=oracle.host_threads())
    assert stats.nodes == ref["nodes"] == 1000
    assert (stats.failures, stats.solutions) == (ref["failures"], len(ref["solutions"]))
    assert stats.trace_hash == ref["trace_hash"]
    M.close()


@pytest.mark.timeout(900)
def test_c3_walk_1e6():
    p = random_table(8, 100, 1_000_000, seed=3)
    tab = Table(p.lo, p.d, p.tuples)
    nfail, nsolved = run_walk(tab, p, calls=300, seed=11, check_table_every=50)
    tab.close()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("gather", [True, False])
def test_c3b_banded_1e6(gather):
    p = banded_table(8, 100, 1_000_000, seed=4)
    tab = Table(p.lo, p.d, p.tuples, use_gather=gather)
    ok, root_m = check_root(tab, p)
    assert ok
    rng = Rng(12)
    st = tab.root.clone()
    for k in range(3):
        rem = fix_one_value_removal(rng, root_m, p.d, var=0)
        din = root_m & (1 - rem)
        ok, dout, valid = oracle_call(p, din, want_valid=True)
        st.copy_from(tab.root)
        status, dom, pr = st.propagate(member_to_bitmap(rem, p.d))
        assert status == (CT_OK if ok else CT_FAIL), k
        if ok:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout), k
            assert np.array_equal(bitmap_to_member(pr, p.d), din & (1 - dout)), k
            assert np.array_equal(bits_to_bool(st.read_table(), p.t), valid), k
    st.close()
    tab.close()
