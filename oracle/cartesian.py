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


def short_to_positive(lo, d, tuples, star):
    """Expand every short tuple into the Cartesian product of its cells (a star
    cell = the variable's whole initial domain): the positive table that the
    short table denotes (PAPER.md L66-68 footnote)."""
    rows = set()
    for row in np.asarray(tuples).reshape(-1, len(d)):
        cells = [range(int(lo[i]), int(lo[i]) + int(d[i])) if int(v) == star else [int(v)]
                 for i, v in enumerate(row)]
        rows.update(itertools.product(*cells))
    out = np.array(sorted(rows), dtype=np.int32)
    return out.reshape(-1, len(d))


def negative_to_positive(lo, d, tuples):
    """The positive table of a negative one: every assignment of the initial
    domains that the list does not forbid (PAPER.md L66-68 footnote)."""
    forbidden = {tuple(int(v) for v in row) for row in np.asarray(tuples).reshape(-1, len(d))}
    ranges = [range(int(lo[i]), int(lo[i]) + int(d[i])) for i in range(len(d))]
    rows = [a for a in itertools.product(*ranges) if a not in forbidden]
    return np.array(rows, dtype=np.int32).reshape(-1, len(d))
