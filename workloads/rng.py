"""Portable counter-free PRNG: splitmix64 seeding -> xoshiro256** lanes.

Recipe:
  * lane l's four state words are outputs 4l..4l+3 of splitmix64(seed);
  * the stream is drawn in rounds; round r produces one xoshiro256** output per
    lane, and stream position p = r*lanes + l;
  * uniform integer in [0, d) = (u64 * d) >> 64 (Lemire's multiply-shift).

Anything that needs the same numbers (C oracle, CUDA path, numpy tests) gets
them from this module, as arrays.  No method arithmetic lives here.
"""
from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1
_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """First `count` outputs of splitmix64 started at state `seed`."""
    with np.errstate(over="ignore"):
        x = (np.uint64(seed & _M64) + _GOLDEN * np.arange(1, count + 1, dtype=np.uint64))
        z = x
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        return z ^ (z >> np.uint64(31))


def _rotl(x: np.ndarray, k: int) -> np.ndarray:
    return (x << np.uint64(k)) | (x >> np.uint64(64 - k))


class Rng:
    """xoshiro256** with `lanes` independent streams interleaved into one stream."""

    def __init__(self, seed: int, lanes: int = 4096):
        self.seed = int(seed)
        self.lanes = int(lanes)
        sm = splitmix64(self.seed, 4 * self.lanes).reshape(self.lanes, 4)
        self.s = [sm[:, i].copy() for i in range(4)]
        self._buf = np.empty(0, dtype=np.uint64)

    def _round(self) -> np.ndarray:
        s0, s1, s2, s3 = self.s
        with np.errstate(over="ignore"):
            out = _rotl(s1 * np.uint64(5), 7) * np.uint64(9)
            t = s1 << np.uint64(17)
            s2 ^= s0
            s3 ^= s1
            s1 ^= s2
            s0 ^= s3
            s2 ^= t
            s3 = _rotl(s3, 45)
        self.s = [s0, s1, s2, s3]
        return out

    def u64(self, count: int) -> np.ndarray:
        count = int(count)
        parts = [self._buf]
        have = self._buf.size
        if have < count:
            rounds = -(-(count - have) // self.lanes)
            parts.extend(self._round() for _ in range(rounds))
        allv = np.concatenate(parts) if len(parts) > 1 else parts[0]
        self._buf = allv[count:]
        return allv[:count]

    def uniform(self, count: int, d) -> np.ndarray:
        """Integers in [0, d) as int64; d may be a scalar or an array (broadcast)."""
        u = self.u64(count)
        d = np.asarray(d, dtype=np.uint64)
        hi = u >> np.uint64(32)
        lo = u & np.uint64(0xFFFFFFFF)
        with np.errstate(over="ignore"):
            r = (hi * d + ((lo * d) >> np.uint64(32))) >> np.uint64(32)
        return r.astype(np.int64)

    def below(self, d: int) -> int:
        return int(self.uniform(1, d)[0])

    def sample_without_replacement(self, population: np.ndarray, k: int) -> np.ndarray:
        """First k items of a partial Fisher-Yates shuffle of `population`."""
        pop = np.array(population, copy=True)
        n = pop.size
        k = min(int(k), n)
        if k == 0:
            return pop[:0]
        r = self.uniform(k, np.arange(n, n - k, -1, dtype=np.uint64))
        for i in range(k):
            j = i + int(r[i])
            pop[i], pop[j] = pop[j], pop[i]
        return pop[:k]
