"""Seeded multi-table CSP models (BASELINE config 5 shape).

csp_model(nv, d, ntab, t, seed): nv variables with domains [0, d); table k has
arity 4 + (k mod 5) (capped at nv), a seeded scope of distinct variables (the
first tables cover every variable at least once), t rows: a planted solution
sigma (one row per table, at a seeded position) and t-1 i.i.d. uniform rows.
Config 5 = csp_model(30, 40, 12, 1_000_000, seed=7).  No method arithmetic.
"""
from __future__ import annotations

import numpy as np

from .rng import Rng


def csp_model(nv: int, d: int, ntab: int, t: int, seed: int, arities=None):
    rng = Rng(seed)
    sigma = rng.uniform(nv, d).astype(np.int32)
    ar = [min(nv, 4 + (k % 5)) for k in range(ntab)] if arities is None else list(arities)
    order = rng.sample_without_replacement(np.arange(nv), nv)
    scopes, pos = [], 0
    for k in range(ntab):
        sc = []
        while pos < nv and len(sc) < ar[k]:          # cover every variable first
            sc.append(int(order[pos]))
            pos += 1
        rest = [v for v in rng.sample_without_replacement(np.arange(nv), nv) if v not in sc]
        sc += [int(v) for v in rest[: ar[k] - len(sc)]]
        scopes.append(np.array(sc, np.int32))
    tables = []
    for k in range(ntab):
        n = len(scopes[k])
        vals = rng.uniform(int(t) * n, d).reshape(int(t), n).astype(np.int32)
        j = rng.below(int(t))
        vals[j] = sigma[scopes[k]]
        tables.append(vals)
    return dict(vlo=np.zeros(nv, np.int32), vd=np.full(nv, d, np.int32), scopes=scopes, tables=tables,
                sigma=sigma)
