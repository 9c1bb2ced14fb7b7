"""Oracle depth-first search over a model of several tables (TEST
INFRASTRUCTURE).  Plain Python driving oracle.fixpoint (the C
brute-force GAC iterated over the tables) at every node.

Search (PAPER.md L469-477 `int_search(input_order, indomain_max, complete)`;
binary branching x = v then x != v): at a node whose domains are
at the common fixpoint, pick the lowest-index variable with more than one
value, v = its largest (indomain_max) or smallest (indomain_min) value; branch
left x = v, right x != v, each followed by a fixpoint; a node with every
variable bound is a solution.  nodes counts the root and every branch, failures
the fixpoints that failed.  trace_hash is FNV-1a 64 over the 8-byte
little-endian words (depth, var, value, branch, status) of every node, root
first (var = -1, branch = 2).

Pinned (tests/test_oracle.py): all-solutions == Cartesian enumeration of the
whole model on tiny models; solutions appear in descending (indomain_max) or
ascending (indomain_min) lexicographic order -- with input_order the variables
before the branching one are bound, the left branch takes the largest
(smallest) value and sound propagation keeps every solution, so this order
pins both the variable and the value order; the node trace of Table 1 alone
(all solutions, indomain_max) derived by hand from Table 1(a);
nodes = 2 (failures + solutions) - 1 (every OK non-solution node has exactly
two children when all solutions are enumerated); the FNV-1a 64 test vector.
"""
from __future__ import annotations

import numpy as np

from . import fixpoint

FNV_OFF = 14695981039346656037   # 0xcbf29ce484222325, the FNV-1a 64 offset basis
FNV_PRIME = 1099511628211
M64 = (1 << 64) - 1


class _Hash:
    def __init__(self):
        self.h = FNV_OFF

    def byte(self, b: int):
        self.h ^= b & 0xFF
        self.h = (self.h * FNV_PRIME) & M64

    def word(self, x: int):
        x &= M64
        for i in range(8):
            self.byte(x >> (8 * i))


def dfs(vlo, vd, scopes, tables, value_order: int = 0, max_nodes: int = 0, max_solutions: int = 1,
        threads: int = 1, keep_trace: bool = False):
    """Returns dict(status, solutions=[...], nodes, failures, trace_hash, last_solution[, trace]).
    threads: host threads of each table's GAC scan (oracle.fixpoint); keep_trace:
    also return the node records (depth, var, value, branch, status)."""
    vlo = np.asarray(vlo, np.int32)
    vd = np.asarray(vd, np.int32)
    base = np.concatenate([[0], np.cumsum(vd)]).astype(int)
    H = _Hash()
    st = dict(nodes=0, failures=0, solutions=[], stop=False, trace=[])

    def account(depth, var, val, branch, ok):
        st["nodes"] += 1
        status = 0 if ok else 1
        if not ok:
            st["failures"] += 1
        for w in (depth, var, val, branch, status):
            H.word(w)
        if keep_trace:
            st["trace"].append((depth, var, val, branch, status))

    def node(dom, depth):
        if st["stop"]:
            return
        x = -1
        for v in range(len(vd)):
            if dom[base[v]:base[v + 1]].sum() > 1:
                x = v
                break
        if x < 0:
            st["solutions"].append(tuple(int(vlo[v]) + int(np.argmax(dom[base[v]:base[v + 1]])) for v in range(len(vd))))
            if max_solutions > 0 and len(st["solutions"]) >= max_solutions:
                st["stop"] = True
            return
        present = np.nonzero(dom[base[x]:base[x + 1]])[0]
        a = int(present[-1] if value_order == 0 else present[0])
        val = int(vlo[x]) + a
        for branch in (0, 1):
            if st["stop"]:
                return
            if max_nodes > 0 and st["nodes"] >= max_nodes:
                st["stop"] = True
                return
            din = dom.copy()
            if branch == 0:
                din[base[x]:base[x + 1]] = 0
                din[base[x] + a] = 1
            else:
                din[base[x] + a] = 0
            ok, dout = fixpoint(vlo, vd, scopes, tables, din, threads=threads)
            account(depth + 1, x, val, branch, ok)
            if ok:
                node(dout, depth + 1)

    dom0 = np.ones(int(vd.sum()), np.uint8)
    ok, root = fixpoint(vlo, vd, scopes, tables, dom0, threads=threads)
    account(0, -1, 0, 2, ok)
    if ok:
        node(root, 0)
    sols = st["solutions"]
    out = dict(status=0 if sols else 1, solutions=sols, nodes=st["nodes"], failures=st["failures"],
               trace_hash=H.h, last_solution=(sols[-1] if sols else None))
    if keep_trace:
        out["trace"] = st["trace"]
    return out
