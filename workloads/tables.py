"""Seeded table-constraint instances shaped like the configs in BASELINE.json.

Shapes:
  C1  the paper's Table 1 example, lo = 1, d = 4, 5 tuples;
  C2  random positive table n=5, d=20, t=1e5, i.i.d. rows (seed 1);
  C3  random positive table n=8, d=100, t=1e7, i.i.d. rows (seed 3);
  C3b banded table n=8, d=100, t=1e7: x0 uniform, x_i = (x0*c_i + u_i) mod d,
      u_i in [0, 10) (seed 4) -- the correlated extreme that forces full scans;
  C4  random positive table n=6, d=50, t=1e6 (seed 5);
  LIN knapsack-configuration tables shaped like the paper's LIN_B / LIN_EB
      sets (Table tbl:instances L476-486): 80-200 variables,
      max domain size 600-800, 5e3-1.5e4 tuples.
Rows are i.i.d. (duplicates allowed).  The paper's own instances
(bounded-knapsack tables) are not published; these generators
bracket that regime (SURVEY §8(d) "Workload structure vs the paper").
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .rng import Rng


@dataclass
class Problem:
    name: str
    lo: np.ndarray          # int32[n]   first value of each initial domain
    d: np.ndarray           # int32[n]   initial domain sizes
    tuples: np.ndarray      # int32[t][n] row-major
    seed: int = 0
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.d.size)

    @property
    def t(self) -> int:
        return int(self.tuples.shape[0])

    @property
    def R(self) -> int:
        return int(self.d.sum())


def table1() -> Problem:
    """PAPER.md L78-86 (Table 1(a)): tau1..tau5 over x1,x2,x3 in {1..4} (L61)."""
    tuples = np.array([[3, 1, 1],
                       [1, 2, 3],
                       [2, 3, 3],
                       [1, 4, 1],
                       [3, 4, 3]], dtype=np.int32)
    return Problem("table1", np.array([1, 1, 1], np.int32), np.array([4, 4, 4], np.int32), tuples)


def random_table(n: int, d, t: int, seed: int, lo=0, name: str | None = None) -> Problem:
    """t i.i.d. rows; column i uniform over [lo_i, lo_i + d_i).  Generation order:
    one stream, value (j, i) at stream position j*n + i."""
    d = np.broadcast_to(np.asarray(d, dtype=np.int32), (n,)).copy()
    lo = np.broadcast_to(np.asarray(lo, dtype=np.int32), (n,)).copy()
    rng = Rng(seed)
    t = int(t)
    tuples = np.empty((t, n), dtype=np.int32)
    chunk = max(1, (1 << 22) // n)                      # rows per chunk (bounded memory)
    dd = d[0] if np.all(d == d[0]) else None
    for j0 in range(0, t, chunk):
        j1 = min(t, j0 + chunk)
        dv = dd if dd is not None else np.tile(d.astype(np.uint64), j1 - j0)
        vals = rng.uniform((j1 - j0) * n, dv)
        tuples[j0:j1] = vals.reshape(j1 - j0, n) + lo[None, :]
    return Problem(name or f"random_n{n}_t{t}_s{seed}", lo, d, tuples, seed)


BANDED_C = (37, 11, 53, 29, 71, 13, 89)


def banded_table(n: int, d: int, t: int, seed: int, band: int = 10, coeffs=BANDED_C,
                 name: str | None = None) -> Problem:
    """C3b: x0 uniform in [0,d); x_i = (x0*c_i + u_i) mod d, u_i uniform in [0,band).
    Stream order per row j: x0, then u_1..u_{n-1}."""
    assert n - 1 <= len(coeffs)
    rng = Rng(seed)
    t = int(t)
    tuples = np.empty((t, n), dtype=np.int32)
    chunk = max(1, (1 << 22) // n)
    for j0 in range(0, t, chunk):
        j1 = min(t, j0 + chunk)
        r = rng.uniform((j1 - j0) * n, np.tile(np.array([d] + [band] * (n - 1), np.uint64), j1 - j0))
        r = r.reshape(j1 - j0, n)
        x0 = r[:, 0]
        tuples[j0:j1, 0] = x0
        for i in range(1, n):
            tuples[j0:j1, i] = (x0 * coeffs[i - 1] + r[:, i]) % d
    return Problem(name or f"banded_n{n}_t{t}_s{seed}", np.zeros(n, np.int32),
                   np.full(n, d, np.int32), tuples, seed)


# PAPER.md Table tbl:instances (L476-486): variables, max domain size, tuples
LIN_PRESETS = {"lin_b": dict(n=120, max_dom=600, t=10_000), "lin_eb": dict(n=160, max_dom=800, t=15_000)}


def knapsack_table(n: int, max_dom: int, t: int, seed: int, kmax: int = 8, name: str | None = None) -> Problem:
    """Bounded-knapsack configurations: item i has weight w_i
    and bound b_i (domain of x_i = {0..b_i}, d_i = b_i + 1 <= max_dom, item 0 at
    the maximum); a row is one configuration x with sum w_i x_i <= capacity.
    Reading (the paper does not publish its generator or seeds):
    each row packs k ~ U[1, kmax] random items in order, item i gets a count
    uniform in [1, min(b_i, remaining // w_i)] (skipped if none fits), every
    other item 0.  Stream order: w (n draws), b (n draws), then per row: k, and
    per pick: item, count.  Rows are sparse, so value 0 is supported almost
    everywhere and most other values by only a few rows -- the filter-heavy,
    many-rows / few-words regime of the paper's instances."""
    rng = Rng(seed)
    w = rng.uniform(n, 50).astype(np.int64) + 1
    b = rng.uniform(n, max_dom - 1).astype(np.int64) + 1
    b[0] = max_dom - 1
    cap = int(np.sort(w * b)[n // 2])            # the median item at its bound fits
    tuples = np.zeros((int(t), n), dtype=np.int32)
    for j in range(int(t)):
        k = int(rng.below(kmax)) + 1
        rem = cap
        for _ in range(k):
            i = int(rng.below(n))
            hi = min(int(b[i]) - int(tuples[j, i]), rem // int(w[i]))
            if hi < 1:
                continue
            c = int(rng.below(hi)) + 1
            tuples[j, i] += c
            rem -= c * int(w[i])
    return Problem(name or f"knapsack_n{n}_d{max_dom}_t{t}_s{seed}", np.zeros(n, np.int32),
                   (b + 1).astype(np.int32), tuples, seed, meta=dict(weights=w, capacity=cap))


STAR = -2147483648   # short-table wildcard cell (include/ct.h CT_STAR = INT32_MIN)


def short_table(n: int, d, t: int, seed: int, p_star: float = 0.1, lo=0, name: str | None = None) -> Problem:
    """f4 short table (PAPER.md L66-68 footnote): random_table(n, d, t, seed, lo),
    then each cell independently becomes STAR with probability p_star (a second
    stream, Rng(seed + 1), one draw per cell in row-major order:
    u < p_star * 2^20 of uniform [0, 2^20))."""
    p = random_table(n, d, t, seed, lo=lo)
    rng = Rng(seed + 1)
    tuples = p.tuples
    chunk = max(1, (1 << 22) // n)
    thr = int(p_star * (1 << 20))
    for j0 in range(0, p.t, chunk):
        j1 = min(p.t, j0 + chunk)
        u = rng.uniform((j1 - j0) * n, 1 << 20).reshape(j1 - j0, n)
        tuples[j0:j1][u < thr] = STAR
    return Problem(name or f"short_n{n}_t{t}_p{p_star}_s{seed}", p.lo, p.d, tuples, seed,
                   meta=dict(p_star=p_star))


def negative_table(n: int, d, t: int, seed: int, lo=0, name: str | None = None) -> Problem:
    """f4 negative table: t forbidden assignments drawn i.i.d. over the product of
    [lo_i, lo_i + d_i) (random_table's stream; duplicates kept -- the library and
    the oracle merge them).  Dense lists (t comparable to prod d_i) make values
    lose all their allowed assignments once the domains shrink."""
    p = random_table(n, d, t, seed, lo=lo)
    return Problem(name or f"negative_n{n}_t{t}_s{seed}", p.lo, p.d, p.tuples, seed)
