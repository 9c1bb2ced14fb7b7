"""Parsers for tests/golden/*.txt fixtures (test helper)."""
from __future__ import annotations

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _lines(name):
    with open(os.path.join(GOLDEN, name)) as f:
        for raw in f:
            s = raw.split("#", 1)[0].strip()
            if s:
                yield s


def load_table1():
    tuples, supports, currtable, dom = [], {}, None, None
    for s in _lines("table1.txt"):
        kind, *rest = s.split()
        if kind == "tuple":
            tuples.append([int(v) for v in rest])
        elif kind == "domain":
            dom = (int(rest[0]), int(rest[1]))
        elif kind == "support":
            var, val, bits = rest
            supports[(int(var[1:]) - 1, int(val))] = np.array([int(c) for c in bits], np.uint8)
        elif kind == "currtable":
            currtable = np.array([int(c) for c in rest[0]], np.uint8)
    lo, hi = dom
    n = len(tuples[0])
    return dict(tuples=np.array(tuples, np.int32), lo=np.full(n, lo, np.int32),
                d=np.full(n, hi - lo + 1, np.int32), supports=supports, currtable=currtable)


def load_traces():
    out = []
    for s in _lines("table1_traces.txt"):
        assert s.startswith("trace ")
        lhs, rhs = s[len("trace "):].split("->")
        din = [[int(v) for v in part.split(",")] for part in lhs.split("|")]
        rhs = rhs.strip()
        dout = None if rhs == "FAIL" else [[int(v) for v in part.split(",")] for part in rhs.split("|")]
        out.append((din, dout))
    return out


def load_counts():
    fixture, tiny = None, []
    for s in _lines("exhaustive_counts.txt"):
        kind, *rest = s.split()
        vals = [int(v) for v in rest]
        if kind == "fixture":
            fixture = dict(zip(["cases", "fail", "empty_input", "already_gac"], vals))
        elif kind == "tiny":
            tiny.append(dict(zip(["n", "d", "cases", "fail", "sum_out"], vals)))
    return fixture, tiny


def member_from_lists(lo, d, lists):
    parts = []
    for i, vals in enumerate(lists):
        m = np.zeros(int(d[i]), np.uint8)
        for v in vals:
            m[v - int(lo[i])] = 1
        parts.append(m)
    return np.concatenate(parts)
