"""CPU oracle for Compact-Table propagation -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  The product path
(paper_2507_18413_b200/) never imports it and shares no code with it.

* ct_oracle.c  -- the oracle proper (plain C, brute-force tuple scan; see its
  header for the PAPER.md passages it follows).  Built here with gcc into
  oracle/liboracle.so on first use (or by __graft_entry__.build()).
* cartesian.py -- an independent second formulation (Cartesian-product
  enumeration of D_in, pure Python) used only to PIN the C oracle on tiny
  inputs.

Parity status per function:
  gac            pinned: Table 1, exhaustive 4096-state
                 fixture vs Cartesian enumeration, exhaustive tiny tables,
                 closed forms (arity 1), binary arc consistency (arity 2),
                 invariants (idempotence, monotonicity, confluence, tuple
                 permutation/duplication invariance).
  supports_row   pinned: Table 1(b) rows printed in PAPER.md L97-104.
  fixpoint       pinned: all-solutions of tiny multi-table models vs Cartesian
                 enumeration of the whole model.
  gac / fixpoint with threads > 1 (oracle_gac_split): the same scan over
                 contiguous tuple slices, results OR-ed; pinned equal to the
                 single-thread functions on random instances.
  gac_short      pinned: expansion of every short tuple into the product of its
                 cells, then `gac` (positive) and Cartesian enumeration; a
                 star-free table equals `gac`; all-star closed form.
  gac_negative   pinned: Cartesian enumeration of the complement relation
                 (product of the initial domains minus the list), then `gac`;
                 empty list / full list / one-value-slab closed forms;
                 duplicate and out-of-range invariance.
  dfs (dfs.py)   pinned: all-solutions == Cartesian enumeration; solutions in
                 descending (indomain_max) / ascending (indomain_min)
                 lexicographic order (input_order, sound propagation); the
                 hand-derived Table 1 node trace; full-binary-tree node count
                 nodes = 2 (failures + solutions) - 1; FNV-1a test vector.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ct_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile ct_oracle.c with gcc (plain -O2, single-threaded)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-shared", "-fPIC", "-pthread", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            L.oracle_gac.argtypes = [ctypes.c_int32, P, P, ctypes.c_int64, P, P, P, P]
            L.oracle_gac.restype = ctypes.c_int
            L.oracle_supports_row.argtypes = [ctypes.c_int32, ctypes.c_int64, P, ctypes.c_int32, ctypes.c_int32, P]
            L.oracle_supports_row.restype = None
            L.oracle_fixpoint.argtypes = [ctypes.c_int32, P, P, ctypes.c_int32, P, P, P, P, P]
            L.oracle_fixpoint.restype = ctypes.c_int
            L.oracle_gac_split.argtypes = [ctypes.c_int32, P, P, ctypes.c_int64, P, P, P, P, ctypes.c_int32]
            L.oracle_gac_split.restype = ctypes.c_int
            L.oracle_fixpoint_split.argtypes = [ctypes.c_int32, P, P, ctypes.c_int32, P, P, P, P, P, ctypes.c_int32]
            L.oracle_fixpoint_split.restype = ctypes.c_int
            L.oracle_gac_short.argtypes = [ctypes.c_int32, P, P, ctypes.c_int64, P, P, P, P]
            L.oracle_gac_short.restype = ctypes.c_int
            L.oracle_gac_negative.argtypes = [ctypes.c_int32, P, P, ctypes.c_int64, P, P, P, P]
            L.oracle_gac_negative.restype = ctypes.c_int
            _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def host_threads() -> int:
    """Host cores this process may use (sched_getaffinity)."""
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return max(1, os.cpu_count() or 1)


def gac(lo, d, tuples, dom_in, want_valid: bool = False, threads: int = 1):
    """Oracle GAC.  dom_in: uint8[R] (byte per value, see ct_oracle.c).
    threads > 1: the tuple scan split over that many host threads
    (oracle_gac_split: union of per-slice results, pinned to threads = 1).
    Returns (ok: bool, dom_out: uint8[R] or None on FAIL, valid: uint8[t] or None)."""
    lo = np.ascontiguousarray(lo, dtype=np.int32)
    d = np.ascontiguousarray(d, dtype=np.int32)
    tuples = np.ascontiguousarray(tuples, dtype=np.int32)
    dom_in = np.ascontiguousarray(dom_in, dtype=np.uint8)
    n = int(d.size)
    t = int(tuples.shape[0]) if tuples.ndim == 2 else 0
    assert dom_in.size == int(d.sum())
    dom_out = np.zeros(int(d.sum()), dtype=np.uint8)
    valid = np.zeros(max(t, 1), dtype=np.uint8) if want_valid else None
    r = lib().oracle_gac_split(n, _p(lo), _p(d), t, _p(tuples) if t else None, _p(dom_in), _p(dom_out),
                               _p(valid) if want_valid else None, int(threads)) if threads > 1 else \
        lib().oracle_gac(n, _p(lo), _p(d), t, _p(tuples) if t else None, _p(dom_in), _p(dom_out),
                         _p(valid) if want_valid else None)
    if r < 0:
        raise ValueError("oracle_gac: bad arguments")
    return bool(r), (dom_out if r else None), (valid[:t] if want_valid else None)


def supports_row(tuples, i: int, value: int):
    tuples = np.ascontiguousarray(tuples, dtype=np.int32)
    t, n = tuples.shape
    out = np.zeros(max(t, 1), dtype=np.uint8)
    lib().oracle_supports_row(n, t, _p(tuples), i, value, _p(out))
    return out[:t]


def fixpoint(vlo, vd, scopes, tables, dom, threads: int = 1):
    """Multi-table fixpoint.  scopes: list of int arrays (global var ids);
    tables: list of int32[t_k][ar_k]; dom: uint8[sum vd] (modified copy returned).
    Returns (ok, dom_out or None)."""
    vlo = np.ascontiguousarray(vlo, dtype=np.int32)
    vd = np.ascontiguousarray(vd, dtype=np.int32)
    ntab = len(tables)
    ar = np.array([len(s) for s in scopes], dtype=np.int32)
    sc = [np.ascontiguousarray(s, dtype=np.int32) for s in scopes]
    tb = [np.ascontiguousarray(x, dtype=np.int32) for x in tables]
    tt = np.array([x.shape[0] for x in tb], dtype=np.int64)
    sc_ptrs = (ctypes.c_void_p * ntab)(*[x.ctypes.data for x in sc])
    tb_ptrs = (ctypes.c_void_p * ntab)(*[x.ctypes.data if x.size else 0 for x in tb])
    out = np.ascontiguousarray(dom, dtype=np.uint8).copy()
    if threads > 1:
        r = lib().oracle_fixpoint_split(int(vd.size), _p(vlo), _p(vd), ntab, _p(ar),
                                        ctypes.cast(sc_ptrs, ctypes.c_void_p), _p(tt),
                                        ctypes.cast(tb_ptrs, ctypes.c_void_p), _p(out), int(threads))
    else:
        r = lib().oracle_fixpoint(int(vd.size), _p(vlo), _p(vd), ntab, _p(ar),
                                  ctypes.cast(sc_ptrs, ctypes.c_void_p), _p(tt),
                                  ctypes.cast(tb_ptrs, ctypes.c_void_p), _p(out))
    if r < 0:
        raise ValueError("oracle_fixpoint: bad arguments")
    return bool(r), (out if r else None)


STAR = -2147483648   # a short-table cell standing for every value (ct_oracle.c ORACLE_STAR)


def gac_short(lo, d, tuples, dom_in, want_valid: bool = False):
    """Oracle GAC on a short table (cells == STAR match any value; ct_oracle.c
    oracle_gac_short).  Returns (ok, dom_out uint8[R] or None, valid uint8[t] or None)."""
    lo = np.ascontiguousarray(lo, dtype=np.int32)
    d = np.ascontiguousarray(d, dtype=np.int32)
    tuples = np.ascontiguousarray(tuples, dtype=np.int32)
    dom_in = np.ascontiguousarray(dom_in, dtype=np.uint8)
    n = int(d.size)
    t = int(tuples.shape[0]) if tuples.ndim == 2 else 0
    dom_out = np.zeros(int(d.sum()), dtype=np.uint8)
    valid = np.zeros(max(t, 1), dtype=np.uint8) if want_valid else None
    r = lib().oracle_gac_short(n, _p(lo), _p(d), t, _p(tuples) if t else None, _p(dom_in), _p(dom_out),
                               _p(valid) if want_valid else None)
    if r < 0:
        raise ValueError("oracle_gac_short: bad arguments")
    return bool(r), (dom_out if r else None), (valid[:t] if want_valid else None)


_neg_lock = threading.Lock()   # oracle_gac_negative's qsort comparator reads one global


def gac_negative(lo, d, tuples, dom_in):
    """Oracle GAC on a negative table (the tuples are the forbidden assignments;
    ct_oracle.c oracle_gac_negative).  Returns (ok, dom_out or None, n_valid),
    n_valid = distinct forbidden tuples inside dom_in."""
    lo = np.ascontiguousarray(lo, dtype=np.int32)
    d = np.ascontiguousarray(d, dtype=np.int32)
    tuples = np.ascontiguousarray(tuples, dtype=np.int32)
    dom_in = np.ascontiguousarray(dom_in, dtype=np.uint8)
    n = int(d.size)
    t = int(tuples.shape[0]) if tuples.ndim == 2 else 0
    dom_out = np.zeros(int(d.sum()), dtype=np.uint8)
    nv = np.zeros(1, dtype=np.int64)
    with _neg_lock:
        r = lib().oracle_gac_negative(n, _p(lo), _p(d), t, _p(tuples) if t else None, _p(dom_in),
                                      _p(dom_out), _p(nv))
    if r < 0:
        raise ValueError("oracle_gac_negative: bad arguments")
    return bool(r), (dom_out if r else None), int(nv[0])
