"""Second, independent formulation of GAC used ONLY to pin the C oracle on tiny
inputs (TEST INFRASTRUCTURE; never imported by the product path).

PAPER.md L48: rel(c) is a subset of dom(x_1) x ... x dom(x_n); L52-53: c is GAC
iff for every x_i and every a in dom(x_i) there is a tuple
(a_1..a_{i-1}, a, a_{i+1}..a_n) in rel(c).  Written literally: enumerate the
Cartesian product of the current domains, keep the assignments that are rows
of the table, and project.  No tuple scan, no bitsets -- a different route to
the same set, so a dropped term or wrong index in ct_oracle.c shows up as a
mismatch.
"""
from __future__ import annotations

import itertools

import numpy as np


def _doms(lo, d, dom_in):
    doms, base = [], 0
    for i in range(len(d)):
        doms.append([int(lo[i]) + a for a in range(int(d[i])) if dom_in[base + a]])
        base += int(d[i])
    return doms


def gac_cartesian(lo, d, tuples, dom_in):
    """Returns (ok, dom_out uint8[R] or None)."""
    rel = {tuple(int(v) for v in row) for row in np.asarray(tuples).reshape(-1, len(d))}
    doms = _doms(lo, d, dom_in)
    R = int(np.sum(d))
    out = np.zeros(R, dtype=np.uint8)
    found = False
    for assignment in itertools.product(*doms):
        if assignment in rel:
            found = True
            base = 0
            for i, v in enumerate(assignment):
                out[base + v - int(lo[i])] = 1
                base += int(d[i])
    return (True, out) if found else (False, None)


def fixpoint_cartesian(vlo, vd, scopes, tables, dom):
    """Iterate gac_cartesian over the tables (fixed order) until nothing changes."""
    vbase = np.concatenate([[0], np.cumsum(vd)]).astype(int)
    dom = np.array(dom, dtype=np.uint8, copy=True)
    changed = True
    while changed:
        changed = False
        for sc, tb in zip(scopes, tables):
            lo = [vlo[v] for v in sc]
            d = [vd[v] for v in sc]
            din = np.concatenate([dom[vbase[v]:vbase[v + 1]] for v in sc])
            ok, dout = gac_cartesian(lo, d, tb, din)
            if not ok:
                return False, None
            off = 0
            for v, dv in zip(sc, d):
                if not np.array_equal(dom[vbase[v]:vbase[v + 1]], dout[off:off + dv]):
                    dom[vbase[v]:vbase[v + 1]] = dout[off:off + dv]
                    changed = True
                off += dv
    return True, dom


def all_solutions(vlo, vd, scopes, tables):
    """All assignments of the model (Cartesian product of the initial domains)
    satisfying every table -- pins the DFS driver's all-solutions output."""
    rels = [{tuple(int(v) for v in row) for row in np.asarray(tb).reshape(-1, len(sc))}
            for sc, tb in zip(scopes, tables)]
    ranges = [range(int(vlo[v]), int(vlo[v]) + int(vd[v])) for v in range(len(vd))]
    sols = []
    for a in itertools.product(*ranges):
        if all(tuple(a[v] for v in sc) in rel for sc, rel in zip(scopes, rels)):
            sols.append(a)
    return sols
