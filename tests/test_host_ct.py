"""The paper's serial CT propagator (placement CT_PLACE_HOST of the f3 ablation,
include/ct.h ct_host_*; Alg. 1-3 with RSparseBitSet and residues,
P:L276-306) vs the oracle, bit-exact.  Host-only: runs without a GPU.  The
GPU-offloaded placements (CT^u, CT^f, CT^uf) run the same checks in
tests/test_gpu_placement.py."""
import itertools

import numpy as np
import pytest

import oracle
from paper_2507_18413_b200 import CT_OK, CT_FAIL, CT_ESTATE, CT_POLICY_DOM, CT_POLICY_DELTA, CTError, HostTable
from workloads import Rng, random_table, banded_table, table1, member_to_bitmap, bitmap_to_member
from workloads.policies import walk_removal


def host_walk(tab, p, calls, seed, m=2, q=0.5):
    ok, root_o, _ = oracle.gac(p.lo, p.d, p.tuples, np.ones(p.R, np.uint8))
    assert (tab.root_status == CT_OK) == ok
    if not ok:
        return 0
    assert np.array_equal(bitmap_to_member(tab.root_dom, p.d), root_o)
    rng = Rng(seed, lanes=1)
    st = tab.root.clone()
    cur = root_o.copy()
    nfail = 0
    for k in range(calls):
        r = walk_removal(rng, cur, p.d, m=m, q=q)
        if r is None:
            st.copy_from(tab.root)
            cur = root_o.copy()
            continue
        din = cur & (1 - r)
        ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, din)
        status, dom, pr = st.propagate(member_to_bitmap(r, p.d))
        assert status == (CT_OK if ok else CT_FAIL), k
        if ok:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout), k
            assert np.array_equal(bitmap_to_member(pr, p.d), din & (1 - dout)), k
            cur = dout
        else:
            nfail += 1
            with pytest.raises(CTError) as e:
                st.propagate(None)
            assert e.value.status == CT_ESTATE
            st.copy_from(tab.root)
            cur = root_o.copy()
    return nfail


def table1_exhaustive(tab, p):
    st = tab.root.clone()
    root_m = bitmap_to_member(tab.root_dom, p.d)
    for bits in itertools.product(range(16), repeat=3):
        D = np.array([(b >> k) & 1 for b in bits for k in range(4)], np.uint8)
        ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, D)
        status, dom, pr = st.propagate(member_to_bitmap((1 - D).astype(np.uint8), p.d))
        assert status == (CT_OK if ok else CT_FAIL), bits
        if ok:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout), bits
            assert np.array_equal(bitmap_to_member(pr, p.d), (D & root_m) & (1 - dout)), bits
        st.copy_from(tab.root)


POLICIES = {"auto": {}, "dom": dict(update_policy=CT_POLICY_DOM), "delta": dict(update_policy=CT_POLICY_DELTA)}


@pytest.mark.parametrize("pol", list(POLICIES))
def test_host_ct_table1_exhaustive(pol):
    p = table1()
    tab = HostTable(p.lo, p.d, p.tuples, **POLICIES[pol])
    assert bitmap_to_member(tab.root_dom, p.d).tolist() == [1, 1, 1, 0, 1, 1, 1, 1, 1, 0, 1, 0]
    table1_exhaustive(tab, p)
    tab.close()


@pytest.mark.parametrize("pol", list(POLICIES))
@pytest.mark.parametrize("shape", [(5, 12, 3000, -4), (1, 9, 40, 0), (2, 70, 700, 3), (3, 130, 5000, 0),
                                   (8, 3, 64, 0), (4, 20, 4096 * 5 + 17, 1)])
def test_host_ct_walks(shape, pol):
    n, d, t, lo = shape
    p = random_table(n, d, t, seed=n * 1000 + d, lo=lo)
    tab = HostTable(p.lo, p.d, p.tuples, **POLICIES[pol])
    host_walk(tab, p, calls=150, seed=3)
    tab.close()


def test_host_ct_config2_walk():
    p = random_table(5, 20, 100_000, seed=1)
    tab = HostTable(p.lo, p.d, p.tuples)
    assert host_walk(tab, p, calls=300, seed=2) > 0
    tab.close()


def test_host_ct_banded_and_knapsack():
    from workloads import knapsack_table
    p = banded_table(5, 30, 20000, seed=4)
    tab = HostTable(p.lo, p.d, p.tuples)
    host_walk(tab, p, calls=120, seed=8, m=1, q=0.8)
    tab.close()
    p = knapsack_table(seed=22, n=60, max_dom=200, t=3000)
    tab = HostTable(p.lo, p.d, p.tuples)
    host_walk(tab, p, calls=80, seed=9)
    tab.close()


def test_host_ct_edge_cases():
    tab = HostTable([0, 0], [3, 3], np.zeros((0, 2), np.int32))
    assert tab.root_status == CT_FAIL and tab.root_dom is None
    tab.close()
    tab = HostTable([0], [4], np.array([[7], [-1], [4]], np.int32))
    assert tab.root_status == CT_FAIL
    tab.close()
    p = random_table(3, 10, 500, seed=9, lo=100)
    D = (Rng(4).uniform(p.R, 3) > 0).astype(np.uint8)
    tab = HostTable(p.lo, p.d, p.tuples, init_dom=member_to_bitmap(D, p.d))
    ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, D)
    assert (tab.root_status == CT_OK) == ok
    if ok:
        assert np.array_equal(bitmap_to_member(tab.root_dom, p.d), dout)
    tab.close()
    with pytest.raises(ValueError):
        HostTable([0, 0], [2, 2], np.zeros((3, 3), np.int32))
