"""Parity harness (test infrastructure): drives the CUDA library through the C ABI
and the CPU oracle on the same seeded inputs and compares element by element.

The oracle's output of call k drives the input of call k+1 (never the GPU's),
so no oracle input derives from the CUDA path.
"""
from __future__ import annotations

import numpy as np

import oracle
from paper_2507_18413_b200 import CT_OK, CT_FAIL, Table
from workloads import member_to_bitmap, bitmap_to_member, Rng
from workloads.layout import bits_to_bool
from workloads.policies import walk_removal


def oracle_call(p, member_in, want_valid=False, threads=None):
    """threads: host threads of the oracle's tuple scan (default: 1 for small
    tables, every core this process may use from 1e6 tuples on)."""
    if threads is None:
        threads = oracle.host_threads() if p.t >= 1_000_000 else 1
    return oracle.gac(p.lo, p.d, p.tuples, member_in, want_valid=want_valid, threads=threads)


def check_root(tab: Table, p):
    ok, dout, valid = oracle_call(p, np.ones(p.R, np.uint8), want_valid=True)
    assert (tab.root_status == CT_OK) == ok
    if ok:
        assert np.array_equal(bitmap_to_member(tab.root_dom, p.d), dout)
        assert np.array_equal(bits_to_bool(tab.root.read_table(), p.t), valid)
    return ok, dout


def run_walk(tab: Table, p, calls: int, seed: int, check_table_every: int = 0, m: int = 2, q: float = 0.5,
             serve: bool = False):
    """Policy P(m, q) walk from the root; restore the root after FAIL or when solved.
    Compares status, domains, pruned set (and currTable every k calls).
    serve: the walk's state answers through a persistent kernel (ct_state_serve)."""
    ok, root_member = check_root(tab, p)
    assert ok, "walk needs a satisfiable root"
    rng = Rng(seed, lanes=1)
    st = tab.root.clone()
    if serve:
        st.serve(True)
    cur = root_member.copy()
    nfail = nsolved = 0
    for k in range(calls):
        rem_m = walk_removal(rng, cur, p.d, m=m, q=q)
        if rem_m is None:                                   # solved: restore root
            st.copy_from(tab.root)
            cur = root_member.copy()
            nsolved += 1
            continue
        din = cur & (1 - rem_m)
        ok, dout, valid = oracle_call(p, din, want_valid=bool(check_table_every))
        status, gdom, gpr = st.propagate(member_to_bitmap(rem_m, p.d))
        assert status == (CT_OK if ok else CT_FAIL), f"call {k}: status {status} vs oracle ok={ok}"
        if ok:
            assert np.array_equal(bitmap_to_member(gdom, p.d), dout), f"call {k}: domains differ"
            assert np.array_equal(bitmap_to_member(gpr, p.d), din & (1 - dout)), f"call {k}: pruned differs"
            if check_table_every and k % check_table_every == 0:
                assert np.array_equal(bits_to_bool(st.read_table(), p.t), valid), f"call {k}: currTable differs"
            cur = dout
        else:
            nfail += 1
            st.copy_from(tab.root)
            cur = root_member.copy()
    st.close()
    return nfail, nsolved
