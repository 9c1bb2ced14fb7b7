"""Generator module checks (CPU): the seeded recipe is what DESIGN.md states."""
import numpy as np

from workloads import Rng, splitmix64, random_table, banded_table, member_to_bitmap, bitmap_to_member
from workloads.layout import dom_word_offsets
from workloads.policies import walk_removal, bulk_removal

M = (1 << 64) - 1


def _sm_scalar(seed, k):
    out, x = [], seed
    for _ in range(k):
        x = (x + 0x9E3779B97F4A7C15) & M
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        out.append(z ^ (z >> 31))
    return out


def _xo_scalar(s, k):
    s = list(s)
    out = []
    rotl = lambda x, r: ((x << r) | (x >> (64 - r))) & M
    for _ in range(k):
        out.append((rotl((s[1] * 5) & M, 7) * 9) & M)
        t = (s[1] << 17) & M
        s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3]; s[2] ^= t; s[3] = rotl(s[3], 45)
    return out


def test_splitmix64_known_value():
    assert int(splitmix64(0, 1)[0]) == 0xE220A8397B1DCDAF       # published test vector
    assert [int(v) for v in splitmix64(12345, 9)] == _sm_scalar(12345, 9)


def test_xoshiro_lanes_interleave():
    r = Rng(7, lanes=3)
    got = [int(v) for v in r.u64(12)]
    sm = _sm_scalar(7, 12)
    lanes = [_xo_scalar(sm[4 * l:4 * l + 4], 4) for l in range(3)]
    exp = [lanes[p % 3][p // 3] for p in range(12)]
    assert got == exp


def test_uniform_range_and_split_draws():
    a = Rng(3, lanes=8).uniform(1000, 37)
    assert a.min() >= 0 and a.max() < 37
    r = Rng(3, lanes=8)
    b = np.concatenate([r.uniform(300, 37), r.uniform(700, 37)])
    assert np.array_equal(a, b)
    u = Rng(3, lanes=8).u64(1000)
    assert np.array_equal(a, ((u.astype(object) * 37) >> 64).astype(np.int64))


def test_tables_shapes():
    p = random_table(5, 20, 1000, seed=1)
    assert p.tuples.shape == (1000, 5) and p.tuples.min() >= 0 and p.tuples.max() < 20
    q = random_table(3, [4, 5, 6], 500, seed=2, lo=[1, -2, 10])
    assert np.all(q.tuples >= q.lo) and np.all(q.tuples < q.lo + q.d)
    b = banded_table(8, 100, 1000, seed=4)
    diff = (b.tuples[:, 1] - 37 * b.tuples[:, 0]) % 100
    assert diff.max() < 10


def test_bitmap_roundtrip():
    d = np.array([3, 64, 65, 130, 1])
    rng = Rng(1)
    m = (rng.uniform(int(d.sum()), 2)).astype(np.uint8)
    bm = member_to_bitmap(m, d)
    assert bm.size == dom_word_offsets(d)[-1] == 1 + 1 + 2 + 3 + 1
    assert np.array_equal(bitmap_to_member(bm, d), m)
    # value 64 of var 2 lives in bit 0 of var 2's second word
    m2 = np.zeros(int(d.sum()), np.uint8); m2[3 + 64 + 64] = 1
    assert member_to_bitmap(m2, d)[dom_word_offsets(d)[2] + 1] == 1


def test_policies():
    d = np.array([20] * 5)
    rng = Rng(2)
    m = np.ones(100, np.uint8)
    rem = walk_removal(rng, m, d)
    per = rem.reshape(5, 20).sum(axis=1)
    assert sorted(per.tolist()) == [0, 0, 0, 10, 10]
    rem = bulk_removal(Rng(3), m, d)
    assert rem.reshape(5, 20).sum(axis=1).tolist() == [10] * 5
    single = np.zeros(100, np.uint8); single[::20] = 1
    assert walk_removal(rng, single, d) is None


def test_knapsack_table_shape_and_invariants():
    """f2 generator: every row is a feasible bounded-knapsack
    configuration, values inside the declared domains, deterministic per seed,
    preset sizes as in Table tbl:instances (L476-486)."""
    import numpy as np
    from workloads import knapsack_table, LIN_PRESETS
    p = knapsack_table(seed=3, n=40, max_dom=100, t=500)
    w, cap = p.meta["weights"], p.meta["capacity"]
    assert p.tuples.shape == (500, 40) and p.d.max() == 100
    assert (p.tuples >= 0).all() and (p.tuples < p.d[None, :]).all()
    assert ((p.tuples.astype(np.int64) * w[None, :]).sum(1) <= cap).all()
    assert (p.tuples.sum(1) > 0).mean() > 0.9
    q = knapsack_table(seed=3, n=40, max_dom=100, t=500)
    assert np.array_equal(p.tuples, q.tuples) and np.array_equal(p.d, q.d)
    assert LIN_PRESETS["lin_b"]["max_dom"] == 600 and 80 <= LIN_PRESETS["lin_b"]["n"] <= 150
    assert LIN_PRESETS["lin_eb"]["max_dom"] == 800 and 100 <= LIN_PRESETS["lin_eb"]["n"] <= 200
