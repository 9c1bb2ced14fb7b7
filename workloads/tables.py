"""Seeded table-constraint instances shaped like the configs in BASELINE.json.

Shapes:
  C1  the paper's Table 1 example, lo = 1, d = 4, 5 tuples;
  C2  random positive table n=5, d=20, t=1e5, i.i.d. rows (seed 1);
  C3  random positive table n=8, d=100, t=1e7, i.i.d. rows (seed 3);
  C3b banded table n=8, d=100, t=1e7: x0 uniform, x_i = (x0*c_i + u_i) mod d,
      u_i in [0, 10) (seed 4) -- the correlated extreme that forces full scans;
  C4  random positive table n=6, d=50, t=1e6 (seed 5).
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
