"""Pins for the CPU oracle (oracle/ct_oracle.c) -- runs without a GPU.

Each test ties the oracle to something other than itself: the paper's printed
Table 1, brute-force Cartesian enumeration (oracle/cartesian.py), closed forms,
textbook special cases, and invariants of the GAC closure.
"""
import itertools
import math

import numpy as np
import pytest

import oracle
from oracle.cartesian import gac_cartesian, fixpoint_cartesian
from golden_io import load_table1, load_traces, load_counts, member_from_lists
from workloads import Rng, random_table, table1

T1 = load_table1()


# --------------------------------------------------------------------------- Table 1
def test_table1_fixture_matches_generator():
    p = table1()
    assert np.array_equal(p.tuples, T1["tuples"])
    assert np.array_equal(p.lo, T1["lo"]) and np.array_equal(p.d, T1["d"])


@pytest.mark.parametrize("key", sorted(T1["supports"].keys()))
def test_supports_rows_printed_in_paper(key):
    """printed supports rows, bit-exact."""
    i, v = key
    assert np.array_equal(oracle.supports_row(T1["tuples"], i, v), T1["supports"][key])


def test_currtable_printed_in_paper():
    """currTable 01010 (tau2, tau4 valid) <=> dom(x1) in {{1},{1,4}}."""
    for x1 in ([1], [1, 4]):
        din = member_from_lists(T1["lo"], T1["d"], [x1, [1, 2, 3, 4], [1, 2, 3, 4]])
        ok, _, valid = oracle.gac(T1["lo"], T1["d"], T1["tuples"], din, want_valid=True)
        assert ok and np.array_equal(valid, T1["currtable"])


@pytest.mark.parametrize("idx", range(len(load_traces())))
def test_table1_traces(idx):
    din_l, dout_l = load_traces()[idx]
    lo, d, tup = T1["lo"], T1["d"], T1["tuples"]
    din = member_from_lists(lo, d, din_l)
    ok, dout, _ = oracle.gac(lo, d, tup, din)
    ok2, dout2 = gac_cartesian(lo, d, tup, din)
    assert ok == ok2 == (dout_l is not None)
    if ok:
        exp = member_from_lists(lo, d, dout_l)
        assert np.array_equal(dout, exp) and np.array_equal(dout2, exp)


def test_table1_exhaustive_4096_states():
    """All 16^3 domain states of Table 1: C oracle == Cartesian, and the counts."""
    fx, _ = load_counts()
    lo, d, tup = T1["lo"], T1["d"], T1["tuples"]
    fails = empties = gac_already = 0
    for bits in itertools.product(range(16), repeat=3):
        din = np.array([(b >> k) & 1 for b in bits for k in range(4)], np.uint8)
        ok, dout, _ = oracle.gac(lo, d, tup, din)
        ok2, dout2 = gac_cartesian(lo, d, tup, din)
        assert ok == ok2
        if ok:
            assert np.array_equal(dout, dout2)
            assert np.all(dout <= din)                 # monotone: D' subset of D
            gac_already += int(np.array_equal(dout, din))
        else:
            fails += 1
        empties += int(any(b == 0 for b in bits))
    assert (16 ** 3, fails, empties, gac_already) == (fx["cases"], fx["fail"], fx["empty_input"], fx["already_gac"])


# --------------------------------------------------------------------------- exhaustive tiny tables
@pytest.mark.parametrize("case", load_counts()[1], ids=lambda c: f"n{c['n']}d{c['d']}")
def test_exhaustive_tiny_tables(case):
    n, dd = case["n"], case["d"]
    lo = np.full(n, 2, np.int32)             # lo != 0 on purpose
    d = np.full(n, dd, np.int32)
    all_tuples = np.array(list(itertools.product(*[range(2, 2 + dd)] * n)), np.int32)
    cases = fails = sum_out = 0
    for tmask in range(1 << len(all_tuples)):
        tup = all_tuples[[k for k in range(len(all_tuples)) if (tmask >> k) & 1]].reshape(-1, n)
        for dmask in range(1 << (n * dd)):
            din = np.array([(dmask >> k) & 1 for k in range(n * dd)], np.uint8)
            ok, dout, _ = oracle.gac(lo, d, tup, din)
            cases += 1
            if ok:
                sum_out += int(dout.sum())
            else:
                fails += 1
            if n * dd <= 4 or (tmask * 131 + dmask) % 97 == 0:      # Cartesian on a subset (speed)
                ok2, dout2 = gac_cartesian(lo, d, tup, din)
                assert ok == ok2 and (not ok or np.array_equal(dout, dout2))
    assert (cases, fails, sum_out) == (case["cases"], case["fail"], case["sum_out"])


@pytest.mark.parametrize("dd", [1, 2, 3, 4, 5])
def test_arity1_closed_form(dd):
    """Arity 1: over all 2^d tables x 2^d domains, #FAIL = 3^d, sum|D'| = d*4^(d-1)."""
    lo, d = np.array([0], np.int32), np.array([dd], np.int32)
    fails = total = 0
    for tmask in range(1 << dd):
        tup = np.array([[v] for v in range(dd) if (tmask >> v) & 1], np.int32).reshape(-1, 1)
        for dmask in range(1 << dd):
            din = np.array([(dmask >> v) & 1 for v in range(dd)], np.uint8)
            ok, dout, _ = oracle.gac(lo, d, tup, din)
            if ok:
                total += int(dout.sum())
                # arity 1: D' = D intersect values(T)
                assert all(dout[v] == (din[v] and (tmask >> v) & 1) for v in range(dd))
            else:
                fails += 1
    assert fails == 3 ** dd and total == dd * 4 ** (dd - 1)


def test_arity2_is_arc_consistency():
    """Arity 2: GAC = arc consistency of a binary relation (textbook AC): with the
    boolean matrix M[a][b] = (a,b) in T and a in D1 and b in D2, D1' = non-empty
    rows, D2' = non-empty columns, FAIL iff M is all-zero."""
    rng = Rng(77, lanes=16)
    for trial in range(300):
        d1, d2 = 1 + rng.below(7), 1 + rng.below(7)
        t = rng.below(12)
        tup = np.stack([rng.uniform(t, d1 + 2) - 1, rng.uniform(t, d2 + 2) - 1], axis=1).astype(np.int32).reshape(-1, 2)
        din = (rng.uniform(d1 + d2, 4) > 0).astype(np.uint8)
        M = np.zeros((d1, d2), bool)
        for a, b in tup:
            if 0 <= a < d1 and 0 <= b < d2:
                M[a, b] = True
        M &= din[:d1, None].astype(bool) & din[None, d1:].astype(bool)
        ok, dout, _ = oracle.gac([0, 0], [d1, d2], tup, din)
        assert ok == bool(M.any())
        if ok:
            assert np.array_equal(dout[:d1], M.any(axis=1).astype(np.uint8))
            assert np.array_equal(dout[d1:], M.any(axis=0).astype(np.uint8))


# --------------------------------------------------------------------------- special cases
def test_special_cases():
    lo, d = np.array([5, -3], np.int32), np.array([3, 4], np.int32)
    full = np.ones(7, np.uint8)
    # full Cartesian table -> no pruning
    cart = np.array(list(itertools.product(range(5, 8), range(-3, 1))), np.int32)
    ok, dout, _ = oracle.gac(lo, d, cart, full)
    assert ok and np.array_equal(dout, full)
    # single tuple -> that assignment
    ok, dout, _ = oracle.gac(lo, d, np.array([[6, -1]], np.int32), full)
    assert ok and dout.tolist() == [0, 1, 0, 0, 0, 1, 0]
    # single tuple outside the domains -> FAIL
    ok, _, valid = oracle.gac(lo, d, np.array([[8, -1]], np.int32), full, want_valid=True)
    assert not ok and valid.tolist() == [0]
    # empty table -> FAIL
    ok, _, _ = oracle.gac(lo, d, np.zeros((0, 2), np.int32), full)
    assert not ok
    # empty input domain -> FAIL
    din = full.copy(); din[3:] = 0
    ok, _, _ = oracle.gac(lo, d, cart, din)
    assert not ok


# --------------------------------------------------------------------------- invariants
def _random_instance(rng, max_n=6, max_d=10, max_t=50):
    n = 1 + rng.below(max_n)
    d = 1 + rng.uniform(n, max_d)
    lo = rng.uniform(n, 7) - 3
    t = rng.below(max_t + 1)
    # values drawn from [lo-1, lo+d] so some tuples fall outside the domain
    vals = rng.uniform(t * n, np.tile((d + 2).astype(np.uint64), t)).reshape(t, n) + lo[None, :] - 1
    din = (rng.uniform(int(d.sum()), 5) > 0).astype(np.uint8)
    return lo.astype(np.int32), d.astype(np.int32), vals.astype(np.int32).reshape(t, n), din


def test_random_vs_cartesian_and_invariants():
    """500 seeded random instances (n<=6, |dom|<=10, t<=50): oracle ==
    Cartesian; idempotence; monotone shrinkage; currTable
    exactness; confluence; tuple permutation/duplication invariance."""
    rng = Rng(2024, lanes=64)
    for case in range(500):
        lo, d, tup, din = _random_instance(rng)
        ok, dout, valid = oracle.gac(lo, d, tup, din, want_valid=True)
        ok2, dout2 = gac_cartesian(lo, d, tup, din) if np.prod(d.astype(float)) <= 2e4 else (ok, dout)
        assert ok == ok2
        # currTable exactness: valid[j] iff every tau_j[i] is in D_in(x_i)
        rb = np.concatenate([[0], np.cumsum(d)])
        for j in range(tup.shape[0]):
            inn = all(0 <= tup[j, i] - lo[i] < d[i] and din[rb[i] + tup[j, i] - lo[i]] for i in range(len(d)))
            assert valid[j] == inn
        assert ok == bool(valid.any())
        if not ok:
            continue
        assert np.array_equal(dout, dout2)
        assert np.all(dout <= din)
        ok3, dout3, _ = oracle.gac(lo, d, tup, dout)                  # idempotence
        assert ok3 and np.array_equal(dout3, dout)
        perm = rng.sample_without_replacement(np.arange(tup.shape[0]), tup.shape[0])
        dup = np.concatenate([tup[perm], tup[: tup.shape[0] // 2]])
        ok4, dout4, _ = oracle.gac(lo, d, dup, din)                   # permutation/duplication
        assert ok4 and np.array_equal(dout4, dout)
        # confluence: removing r1 then r2 (each followed by GAC) == removing r1|r2 at once
        r1 = (rng.uniform(dout.size, 4) == 0).astype(np.uint8)
        r2 = (rng.uniform(dout.size, 4) == 0).astype(np.uint8)
        okA, dA, _ = oracle.gac(lo, d, tup, dout & (1 - r1))
        if okA:
            okA, dA, _ = oracle.gac(lo, d, tup, dA & (1 - r2))
        okB, dB, _ = oracle.gac(lo, d, tup, dout & (1 - (r1 | r2)))
        assert okA == okB and (not okA or np.array_equal(dA, dB))


def test_larger_random_table_sampled_vs_cartesian():
    """Larger tables from the product generator (lo != 0, d = 6, n = 4, t = 600)."""
    p = random_table(4, 6, 600, seed=9, lo=3)
    rng = Rng(5)
    for _ in range(20):
        din = (rng.uniform(p.R, 3) > 0).astype(np.uint8)
        ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, din)
        ok2, dout2 = gac_cartesian(p.lo, p.d, p.tuples, din)
        assert ok == ok2 and (not ok or np.array_equal(dout, dout2))


# --------------------------------------------------------------------------- multi-table fixpoint
def test_fixpoint_vs_iterated_cartesian():
    rng = Rng(31, lanes=16)
    for trial in range(60):
        nv = 2 + rng.below(4)
        vd = (1 + rng.uniform(nv, 4)).astype(np.int32)
        vlo = np.zeros(nv, np.int32)
        ntab = 1 + rng.below(3)
        scopes, tables = [], []
        for _ in range(ntab):
            ar = 1 + rng.below(min(3, nv))
            sc = rng.sample_without_replacement(np.arange(nv), ar).astype(np.int32)
            t = rng.below(10)
            tb = np.stack([rng.uniform(t, vd[v]) for v in sc], axis=1).astype(np.int32).reshape(t, ar)
            scopes.append(sc)
            tables.append(tb)
        dom = (rng.uniform(int(vd.sum()), 5) > 0).astype(np.uint8)
        ok, out = oracle.fixpoint(vlo, vd, scopes, tables, dom)
        ok2, out2 = fixpoint_cartesian(vlo, vd, scopes, tables, dom)
        assert ok == ok2 and (not ok or np.array_equal(out, out2))


# --------------------------------------------------------------------------- DFS oracle (f1)
def _tiny_model(rng, nv=4, d=3, ntab=3):
    from workloads.csp import csp_model
    return csp_model(nv, d, ntab, 6, seed=int(rng.below(10**6)), arities=[min(nv, 2 + k % 2) for k in range(ntab)])


def test_dfs_all_solutions_equal_cartesian():
    from oracle.cartesian import all_solutions
    from oracle.dfs import dfs
    rng = Rng(404, lanes=4)
    for trial in range(25):
        m = _tiny_model(rng, nv=3 + trial % 3, d=2 + trial % 3, ntab=2 + trial % 3)
        res = dfs(m["vlo"], m["vd"], m["scopes"], m["tables"], value_order=trial % 2, max_solutions=0)
        exp = all_solutions(m["vlo"], m["vd"], m["scopes"], m["tables"])
        assert sorted(res["solutions"]) == sorted(exp)
        assert len(set(res["solutions"])) == len(res["solutions"])      # each solution once
        assert tuple(int(v) for v in m["sigma"]) in exp                   # planted solution


def test_dfs_table1_first_solution_and_all():
    """SPEC S:L394-395 (derived): Table 1 alone, input_order + indomain_max ->
    (3,4,3) = tau5 first; all solutions = exactly the 5 tuples."""
    from oracle.dfs import dfs
    p = table1()
    res = dfs(p.lo, p.d, [np.arange(3)], [p.tuples], value_order=0, max_solutions=1)
    assert res["last_solution"] == (3, 4, 3)
    res = dfs(p.lo, p.d, [np.arange(3)], [p.tuples], value_order=0, max_solutions=0)
    assert sorted(res["solutions"]) == sorted(tuple(int(v) for v in r) for r in p.tuples)


def test_dfs_lexicographic_order_and_node_identity():
    """input_order + indomain_max with sound propagation emits solutions in
    descending lexicographic order (ascending for indomain_min), PAPER.md
    L469-477; and with all solutions enumerated every OK non-solution node
    has two children, so nodes = 2 (failures + solutions) - 1."""
    from oracle.cartesian import all_solutions
    from oracle.dfs import dfs
    rng = Rng(405, lanes=4)
    n_nonempty = 0
    for trial in range(30):
        m = _tiny_model(rng, nv=3 + trial % 3, d=2 + trial % 3, ntab=2 + trial % 3)
        exp = all_solutions(m["vlo"], m["vd"], m["scopes"], m["tables"])
        for vo in (0, 1):
            res = dfs(m["vlo"], m["vd"], m["scopes"], m["tables"], value_order=vo, max_solutions=0)
            assert res["solutions"] == sorted(exp, reverse=(vo == 0)), (trial, vo)
            assert res["nodes"] == 2 * (res["failures"] + len(res["solutions"])) - 1, (trial, vo)
        n_nonempty += len(exp) > 1
    assert n_nonempty >= 10


def test_dfs_table1_hand_trace():
    """Table 1 alone (tau1..tau5 = (3,1,1), (1,2,3), (2,3,3), (1,4,1), (3,4,3),
    read off Table 1(a)/(b)), all solutions, input_order +
    indomain_max; every record (depth, var, value, branch 0: x = v / 1: x != v /
    2: root, status) derived by hand: a single GAC table never fails after a
    branch, so the search only splits."""
    from oracle.dfs import dfs, _Hash
    p = table1()
    res = dfs(p.lo, p.d, [np.arange(3)], [p.tuples], value_order=0, max_solutions=0, keep_trace=True)
    assert res["trace"] == [
        (0, -1, 0, 2, 0),     # root: x1 = {1,2,3}, x2 = {1..4}, x3 = {1,3}
        (1, 0, 3, 0, 0),      # x1 = 3: tau1, tau5
        (2, 1, 4, 0, 0),      # x2 = 4: tau5 -> solution (3,4,3)
        (2, 1, 4, 1, 0),      # x2 != 4: tau1 -> solution (3,1,1)
        (1, 0, 3, 1, 0),      # x1 != 3: tau2, tau3, tau4
        (2, 0, 2, 0, 0),      # x1 = 2: tau3 -> solution (2,3,3)
        (2, 0, 2, 1, 0),      # x1 != 2 -> x1 = 1: tau2, tau4
        (3, 1, 4, 0, 0),      # x2 = 4: tau4 -> solution (1,4,1)
        (3, 1, 4, 1, 0),      # x2 != 4: tau2 -> solution (1,2,3)
    ]
    assert res["solutions"] == [(3, 4, 3), (3, 1, 1), (2, 3, 3), (1, 4, 1), (1, 2, 3)]
    assert res["nodes"] == 9 and res["failures"] == 0
    h = _Hash()
    for rec in res["trace"]:
        for w in rec:
            h.word(w)
    assert h.h == res["trace_hash"]


def test_fnv1a_64_test_vector():
    """FNV-1a 64 (offset 0xcbf29ce484222325, prime 0x100000001b3) of b"foobar"
    is 0x85944171f73967e8 (the published FNV test vector)."""
    from oracle.dfs import _Hash, FNV_OFF, FNV_PRIME
    assert FNV_OFF == 0xcbf29ce484222325 and FNV_PRIME == 0x100000001b3
    h = _Hash()
    for b in b"foobar":
        h.byte(b)
    assert h.h == 0x85944171f73967e8


def test_split_oracle_equals_single_thread():
    """oracle_gac_split (tuple slices over host threads, results OR-ed) ==
    oracle_gac, and the split fixpoint == the plain one."""
    rng = Rng(406, lanes=4)
    for trial in range(40):
        n = 1 + trial % 6
        d = 2 + trial % 9
        t = int(rng.below(3000)) + (0 if trial % 7 else 0)
        p = random_table(n, d, t, seed=trial + 900, lo=trial % 3 - 1)
        din = (rng.uniform(p.R, 4) > 0).astype(np.uint8)
        a = oracle.gac(p.lo, p.d, p.tuples, din, want_valid=True)
        for th in (2, 3, 8):
            b = oracle.gac(p.lo, p.d, p.tuples, din, want_valid=True, threads=th)
            assert a[0] == b[0]
            assert np.array_equal(a[2], b[2])
            if a[0]:
                assert np.array_equal(a[1], b[1])
    from workloads.csp import csp_model
    for trial in range(10):
        m = csp_model(6, 5, 4, 400, seed=trial + 77)
        dom = np.ones(int(np.sum(m["vd"])), np.uint8)
        r1 = oracle.fixpoint(m["vlo"], m["vd"], m["scopes"], m["tables"], dom)
        r2 = oracle.fixpoint(m["vlo"], m["vd"], m["scopes"], m["tables"], dom, threads=4)
        assert r1[0] == r2[0] and (not r1[0] or np.array_equal(r1[1], r2[1]))
