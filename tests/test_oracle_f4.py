"""Pins for the f4 oracle functions (short and negative tables, SURVEY §8(f)
f4; PAPER.md L66-68 and footnote) -- runs without a GPU.

Both tables denote a plain relation (the footnote's definitions), so each
oracle is pinned by turning the table into the positive table it denotes
(oracle/cartesian.py: short_to_positive / negative_to_positive, written by
enumeration, not by the oracle's scan or count) and checking against the
already-pinned positive oracle `gac` and Cartesian enumeration of D_in, plus
closed forms a dropped term or wrong index would break.
"""
import itertools

import numpy as np
import pytest

import oracle
from oracle.cartesian import gac_cartesian, short_to_positive, negative_to_positive
from golden_io import load_table1

STAR = oracle.STAR
T1 = load_table1()


class Rng:
    """Seeded scalar draws for the tiny pin instances (numpy PCG64)."""

    def __init__(self, seed):
        self.g = np.random.default_rng(seed)

    def uniform(self, d):
        return int(self.g.integers(0, d)) if d > 0 else 0

    def permutation(self, n):
        return self.g.permutation(n)


def _rand_dom(rng, d):
    return np.array([1 if rng.uniform(3) else 0 for _ in range(int(np.sum(d)))], dtype=np.uint8)


def _rand_short(rng, n, dmax, t, p_star):
    lo = np.array([rng.uniform(5) - 2 for _ in range(n)], dtype=np.int32)
    d = np.array([1 + rng.uniform(dmax) for _ in range(n)], dtype=np.int32)
    tup = np.zeros((t, n), dtype=np.int32)
    for j in range(t):
        for i in range(n):
            if rng.uniform(1000) < int(p_star * 1000):
                tup[j, i] = STAR
            else:
                # mostly in range, sometimes one past either end (never valid, Q15)
                tup[j, i] = lo[i] - 1 + rng.uniform(int(d[i]) + 2)
    return lo, d, tup


# --------------------------------------------------------------------------- short tables
def test_short_star_free_equals_positive():
    """A short table without stars is a positive table (footnote: short = cells
    may hold more than one value; here every cell holds one)."""
    rng = Rng(101)
    for _ in range(200):
        lo, d, tup = _rand_short(rng, 1 + rng.uniform(4), 5, rng.uniform(12), 0.0)
        din = _rand_dom(rng, d)
        a = oracle.gac_short(lo, d, tup, din, want_valid=True)
        b = oracle.gac(lo, d, tup, din, want_valid=True)
        assert a[0] == b[0]
        if a[0]:
            assert np.array_equal(a[1], b[1])
        assert np.array_equal(a[2], b[2])


def test_short_vs_expansion_and_cartesian():
    """500 random short tables: oracle_gac_short == gac on the expanded table ==
    Cartesian enumeration of D_in against the expanded relation."""
    rng = Rng(102)
    for k in range(500):
        n = 1 + rng.uniform(4)
        lo, d, tup = _rand_short(rng, n, 4, rng.uniform(10), 0.3)
        din = _rand_dom(rng, d)
        ok, dout, _ = oracle.gac_short(lo, d, tup, din)
        pos = short_to_positive(lo, d, tup, STAR)
        ok2, dout2, _ = oracle.gac(lo, d, pos, din)
        ok3, dout3 = gac_cartesian(lo, d, pos, din)
        assert ok == ok2 == ok3, k
        if ok:
            assert np.array_equal(dout, dout2) and np.array_equal(dout, dout3), k


def test_short_valid_vector_is_product_meets_domain():
    """valid_out[j] = 1 iff the product of tau_j's cells meets D_in, i.e. iff the
    expansion of tau_j alone has a valid row."""
    rng = Rng(103)
    for _ in range(300):
        lo, d, tup = _rand_short(rng, 1 + rng.uniform(3), 4, 1 + rng.uniform(6), 0.4)
        din = _rand_dom(rng, d)
        _, _, valid = oracle.gac_short(lo, d, tup, din, want_valid=True)
        for j in range(tup.shape[0]):
            one = short_to_positive(lo, d, tup[j:j + 1], STAR)
            okj, _, _ = oracle.gac(lo, d, one, din)
            assert bool(valid[j]) == okj


def test_short_closed_forms():
    """All-star tuple: nothing is pruned while every domain is non-empty, FAIL as
    soon as one is empty.  Table 1 with x2 starred in tau5 (3,*,3): x2 keeps
    every value whenever tau5 is valid."""
    lo, d = np.array([1, 1, 1], np.int32), np.array([4, 4, 4], np.int32)
    allstar = np.full((1, 3), STAR, np.int32)
    for bits in itertools.product([0, 1], repeat=12):
        din = np.array(bits, np.uint8)
        ok, dout, _ = oracle.gac_short(lo, d, allstar, din)
        nonempty = all(din[4 * i:4 * i + 4].any() for i in range(3))
        assert ok == nonempty
        if ok:
            assert np.array_equal(dout, din)
    tup = T1["tuples"].copy()
    tup[4, 1] = STAR   # tau5 = (3, *, 3)
    din = np.ones(12, np.uint8)
    din[[0, 1, 3]] = 0          # x1 = {3}: tau1 (3,1,1) and tau5 (3,*,3) are valid
    ok, dout, _ = oracle.gac_short(T1["lo"], T1["d"], tup, din)
    # x1 = {3}; x2 = {1} u {1,2,3,4}; x3 = {1} u {3}
    assert ok and list(dout) == [0, 0, 1, 0, 1, 1, 1, 1, 1, 0, 1, 0]
    din[8] = 0                  # and x3 = {2,3,4}: only tau5, so x2 keeps all four values
    ok, dout, _ = oracle.gac_short(T1["lo"], T1["d"], tup, din)
    assert ok and list(dout) == [0, 0, 1, 0, 1, 1, 1, 1, 0, 0, 1, 0]


def test_short_single_pass_is_fixpoint():
    """One pass of GAC on one short table reaches the fixpoint (the valid
    products keep meeting the pruned domains): re-applying changes nothing."""
    rng = Rng(104)
    for _ in range(300):
        lo, d, tup = _rand_short(rng, 1 + rng.uniform(4), 5, rng.uniform(15), 0.3)
        din = _rand_dom(rng, d)
        ok, dout, _ = oracle.gac_short(lo, d, tup, din)
        if ok:
            ok2, dout2, _ = oracle.gac_short(lo, d, tup, dout)
            assert ok2 and np.array_equal(dout, dout2)


# --------------------------------------------------------------------------- negative tables
def _rand_neg(rng, n, dmax, t):
    lo = np.array([rng.uniform(5) - 2 for _ in range(n)], dtype=np.int32)
    d = np.array([1 + rng.uniform(dmax) for _ in range(n)], dtype=np.int32)
    tup = np.array([[lo[i] - 1 + rng.uniform(int(d[i]) + 2) for i in range(n)] for _ in range(t)],
                   dtype=np.int32).reshape(t, n)
    return lo, d, tup


def test_negative_vs_complement_and_cartesian():
    """500 random negative tables (dense lists so that pruning and FAIL occur):
    oracle_gac_negative == gac on the complement relation == Cartesian."""
    rng = Rng(111)
    seen = {"fail": 0, "prune": 0}
    for k in range(500):
        n = 1 + rng.uniform(3)
        lo, d, _ = _rand_neg(rng, n, 3, 0)
        total = int(np.prod(d))
        t = rng.uniform(2 * total + 2)
        tup = np.array([[lo[i] - (1 if rng.uniform(8) == 0 else 0) + rng.uniform(int(d[i]))
                         for i in range(n)] for _ in range(t)], dtype=np.int32).reshape(t, n)
        din = _rand_dom(rng, d)
        ok, dout, nv = oracle.gac_negative(lo, d, tup, din)
        pos = negative_to_positive(lo, d, tup)
        ok2, dout2, _ = oracle.gac(lo, d, pos, din)
        ok3, dout3 = gac_cartesian(lo, d, pos, din)
        assert ok == ok2 == ok3, k
        if ok:
            assert np.array_equal(dout, dout2) and np.array_equal(dout, dout3), k
            seen["prune"] += int(np.any(dout != din))
        else:
            seen["fail"] += 1
        # n_valid = distinct listed tuples inside D_in
        inside = {tuple(r) for r in tup.tolist()
                  if all(lo[i] <= r[i] < lo[i] + d[i] and din[int(np.sum(d[:i])) + r[i] - lo[i]]
                         for i in range(n))}
        assert nv == len(inside)
    assert seen["fail"] > 20 and seen["prune"] > 20


def test_negative_closed_forms():
    """Empty list: nothing pruned (FAIL iff a domain is empty).  The full product
    listed: FAIL.  Every assignment with x_0 = a listed: exactly (x_0, a) pruned."""
    lo, d = np.array([0, 0, 0], np.int32), np.array([3, 2, 4], np.int32)
    din = np.ones(9, np.uint8)
    ok, dout, nv = oracle.gac_negative(lo, d, np.zeros((0, 3), np.int32), din)
    assert ok and np.array_equal(dout, din) and nv == 0
    full = np.array(list(itertools.product(range(3), range(2), range(4))), np.int32)
    ok, _, nv = oracle.gac_negative(lo, d, full, din)
    assert not ok and nv == 24
    for a in range(3):
        slab = full[full[:, 0] == a]
        ok, dout, nv = oracle.gac_negative(lo, d, slab, din)
        exp = din.copy()
        exp[a] = 0
        assert ok and np.array_equal(dout, exp) and nv == 8
    # the slab minus one assignment: nothing pruned
    ok, dout, _ = oracle.gac_negative(lo, d, full[full[:, 0] == 1][1:], din)
    assert ok and np.array_equal(dout, din)


def test_negative_duplicates_and_out_of_range_invariance():
    rng = Rng(112)
    for _ in range(200):
        n = 1 + rng.uniform(3)
        lo, d, _ = _rand_neg(rng, n, 3, 0)
        t = rng.uniform(int(np.prod(d)) + 3)
        tup = np.array([[lo[i] + rng.uniform(int(d[i])) for i in range(n)] for _ in range(t)],
                       dtype=np.int32).reshape(t, n)
        din = _rand_dom(rng, d)
        ref = oracle.gac_negative(lo, d, tup, din)
        junk = np.array([[lo[i] + int(d[i]) + 3 for i in range(n)]], np.int32)
        noisy = np.concatenate([tup, tup[: t // 2], junk]).astype(np.int32)
        perm = rng.permutation(noisy.shape[0])
        got = oracle.gac_negative(lo, d, noisy[perm], din)
        assert ref[0] == got[0] and ref[2] == got[2]
        if ref[0]:
            assert np.array_equal(ref[1], got[1])


def test_negative_single_pass_is_fixpoint():
    rng = Rng(113)
    for _ in range(300):
        n = 1 + rng.uniform(3)
        lo, d, _ = _rand_neg(rng, n, 3, 0)
        t = rng.uniform(2 * int(np.prod(d)) + 1)
        tup = np.array([[lo[i] + rng.uniform(int(d[i])) for i in range(n)] for _ in range(t)],
                       dtype=np.int32).reshape(t, n)
        din = _rand_dom(rng, d)
        ok, dout, _ = oracle.gac_negative(lo, d, tup, din)
        if ok:
            ok2, dout2, _ = oracle.gac_negative(lo, d, tup, dout)
            assert ok2 and np.array_equal(dout, dout2)
