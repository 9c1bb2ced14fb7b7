"""Seeded call policies: which values each ct_propagate call removes.

All functions take the CURRENT domains in "member" form (uint8[R], see layout.py)
and return the removal set in the same form.  In parity tests the current
domains come from the oracle's previous output (never from the CUDA path); in
bench.py (no oracle) they come from the library's own output.

* bulk_removal (C3 bulk): from the root, remove a seeded random
  fraction q of every variable's present values.
* walk_removal, policy P(m, q): pick m distinct non-singleton
  variables; remove min(|dom|-1, ceil(q*|dom|)) random present values from each.
  Returns None when every variable is a singleton (walk solved -> restore root).
* fix_one_value_removal (C3b banded): remove all but one seeded present value of
  one variable.
* batch_coin_removals (C4 batched steps): per state, 2 random variables, each
  value removed with probability 1/2; state-independent bitmaps (values already
  absent are ignored by the library), [count][S][Wd] uint64.
"""
from __future__ import annotations

import math

import numpy as np

from .layout import row_bases
from .rng import Rng


def _present(member, rb, i):
    return np.nonzero(member[rb[i]:rb[i + 1]])[0]


def bulk_removal(rng: Rng, member: np.ndarray, d, q: float = 0.5) -> np.ndarray:
    rb = row_bases(d)
    rem = np.zeros_like(member)
    for i in range(len(d)):
        pres = _present(member, rb, i)
        k = int(round(q * pres.size))
        pick = rng.sample_without_replacement(pres, k)
        rem[rb[i] + pick] = 1
    return rem


def walk_removal(rng: Rng, member: np.ndarray, d, m: int = 2, q: float = 0.5):
    rb = row_bases(d)
    sizes = np.array([int(member[rb[i]:rb[i + 1]].sum()) for i in range(len(d))])
    cand = np.nonzero(sizes > 1)[0]
    if cand.size == 0:
        return None
    vars_ = rng.sample_without_replacement(cand, min(m, cand.size))
    rem = np.zeros_like(member)
    for i in vars_:
        pres = _present(member, rb, int(i))
        k = min(pres.size - 1, int(math.ceil(q * pres.size)))
        pick = rng.sample_without_replacement(pres, k)
        rem[rb[int(i)] + pick] = 1
    return rem


def fix_one_value_removal(rng: Rng, member: np.ndarray, d, var: int = 0) -> np.ndarray:
    rb = row_bases(d)
    pres = _present(member, rb, var)
    keep = pres[rng.below(pres.size)] if pres.size else None
    rem = np.zeros_like(member)
    for v in pres:
        if v != keep:
            rem[rb[var] + v] = 1
    return rem


def batch_coin_removals(n: int, d, S: int, count: int, seed: int = 6):
    """[count] arrays of [S][Wd] uint64 removal bitmaps (C4)."""
    from .layout import member_to_bitmap
    d = np.asarray(d)
    rng = Rng(seed)
    rb = row_bases(d)
    R = int(d.sum())
    pats = []
    for _ in range(count):
        vars_ = rng.uniform(S * 2, n).reshape(S, 2)
        coin = rng.uniform(S * 2 * int(d.max()), 2).reshape(S, 2, int(d.max()))
        rem = np.zeros((S, R), np.uint8)
        for j in range(2):
            for x in range(n):
                sel = vars_[:, j] == x
                rem[sel, rb[x]:rb[x + 1]] |= coin[sel, j, :d[x]].astype(np.uint8)
        pats.append(np.stack([member_to_bitmap(r, d) for r in rem]))
    return pats
