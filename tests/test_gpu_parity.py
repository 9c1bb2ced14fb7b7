"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact.

Run on a B200 with `python -m pytest tests -m gpu`.
"""
import itertools

import numpy as np
import pytest

import oracle
from ctharness import check_root, oracle_call, run_walk
from golden_io import load_table1, member_from_lists
from paper_2507_18413_b200 import (CT_OK, CT_FAIL, CT_ESTATE, CT_POLICY_AUTO, CT_POLICY_DOM,
                                   CT_POLICY_DELTA, CTError, Table)
from paper_2507_18413_b200 import ct as C
from workloads import (Rng, random_table, banded_table, table1, member_to_bitmap, bitmap_to_member,
                       bulk_removal, fix_one_value_removal)
from workloads.layout import bits_to_bool, dom_word_offsets
from workloads.policies import walk_removal

pytestmark = pytest.mark.gpu

KNOBS = [
    dict(),
    dict(update_policy=CT_POLICY_DOM),
    dict(update_policy=CT_POLICY_DELTA),
    dict(use_residues=False),
    dict(use_index=False),
    dict(use_graph=False),
    dict(use_fused=False),
    dict(_grid_fused=True),
    dict(_grid_fused=True, _fast=False),
    dict(_grid_fused=True, use_index=False),
    dict(_grid_fused=True, use_residues=False),
]
KNOB_IDS = ["auto", "dom", "delta", "nores", "noindex", "nograph", "nofused", "gridfused", "gridfused_v1",
            "gridfused_noindex", "gridfused_nores"]


@pytest.fixture(scope="module", autouse=True)
def _built():
    from paper_2507_18413_b200 import build
    build.build()
    import torch
    assert torch.cuda.is_available()


def make(p, _grid_fused=False, _fast=True, _grid=0, _wide=None, **kw):
    """_grid_fused: force a cooperative multi-CTA kernel even for tables small
    enough for the single-CTA one (ct_config.launch_shape); _fast=False: the
    barrier-per-phase k_fused instead of k_fast; _grid: fewer CTAs than tiles
    (grid_override); _wide=True/False: force / forbid the k_wide shape."""
    if _grid_fused:
        kw.setdefault("launch_shape", "fast" if _fast else "fused")
    elif not _fast:
        kw.setdefault("launch_shape", "fused")
    if _wide is True:
        kw.setdefault("launch_shape", "wide")
    elif _wide is False:
        kw.setdefault("launch_shape", "small")
    if _grid:
        kw["grid_override"] = _grid   # several tiles per CTA
    return Table(p.lo, p.d, p.tuples, **kw)


# --------------------------------------------------------------------------- a1 supports builder
def test_supports_table1_printed_rows():
    T1 = load_table1()
    p = table1()
    tab = make(p)
    rb = np.concatenate([[0], np.cumsum(p.d)])
    for (i, v), bits in T1["supports"].items():
        row = rb[i] + v - p.lo[i]
        got = bits_to_bool(C.ct_table_read_supports(tab.handle, int(row), 1), p.t)
        assert np.array_equal(got, bits), (i, v)
    tab.close()


@pytest.mark.parametrize("shape", [(3, 5, 1, 200), (4, 70, -3, 1000), (2, 130, 7, 4097), (6, 1, 0, 64)])
def test_supports_random_vs_definition(shape):
    n, d, lo, t = shape
    p = random_table(n, d + 2, t, seed=11, lo=lo - 1)        # values in [lo-1, lo+d]: some out of range
    p.lo[:] = lo
    p.d[:] = d
    tab = make(p)
    W = (t + 63) // 64
    for i in range(n):
        for a in range(d):
            row = i * d + a
            got = C.ct_table_read_supports(tab.handle, row, W)
            exp = oracle.supports_row(p.tuples, i, lo + a)
            assert np.array_equal(bits_to_bool(got, t), exp)
            if t % 64:
                assert int(got[-1]) >> (t % 64) == 0          # padding bits stay 0
    tab.close()


# --------------------------------------------------------------------------- Table 1
def test_table1_root_and_currtable():
    T1 = load_table1()
    p = table1()
    tab = make(p)
    check_root(tab, p)
    assert bitmap_to_member(tab.root_dom, p.d).tolist() == [1, 1, 1, 0, 1, 1, 1, 1, 1, 0, 1, 0]
    st = tab.root.clone()
    rem = member_from_lists(p.lo, p.d, [[2, 3], [], []])     # dom(x1) -> {1}
    status, dom, pr = st.propagate(member_to_bitmap(rem, p.d))
    assert status == CT_OK
    assert np.array_equal(bits_to_bool(st.read_table(), 5), T1["currtable"])
    assert bitmap_to_member(dom, p.d).tolist() == [1, 0, 0, 0, 0, 1, 0, 1, 1, 0, 1, 0]
    tab.close()


@pytest.mark.parametrize("knobs", KNOBS, ids=KNOB_IDS)
def test_table1_exhaustive_4096(knobs):
    """Every domain state of Table 1 (16^3), from the root, vs the oracle."""
    p = table1()
    tab = make(p, **knobs)
    st = tab.root.clone()
    root_m = bitmap_to_member(tab.root_dom, p.d)
    for bits in itertools.product(range(16), repeat=3):
        D = np.array([(b >> k) & 1 for b in bits for k in range(4)], np.uint8)
        ok, dout, valid = oracle_call(p, D, want_valid=True)
        rem = (1 - D).astype(np.uint8)
        status, dom, pr = st.propagate(member_to_bitmap(rem, p.d))
        assert status == (CT_OK if ok else CT_FAIL), bits
        if ok:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout), bits
            assert np.array_equal(bitmap_to_member(pr, p.d), (D & root_m) & (1 - dout)), bits
            assert np.array_equal(bits_to_bool(st.read_table(), 5), valid), bits
        st.copy_from(tab.root)
    tab.close()


# --------------------------------------------------------------------------- random walks
@pytest.mark.parametrize("knobs", KNOBS, ids=KNOB_IDS)
def test_walk_small_random(knobs):
    p = random_table(5, 12, 3000, seed=21, lo=-4)
    tab = make(p, **knobs)
    nfail, nsolved = run_walk(tab, p, calls=250, seed=5, check_table_every=7)
    assert nfail + nsolved > 0
    tab.close()


@pytest.mark.parametrize("shape", [(1, 9, 40), (2, 70, 700), (3, 130, 5000), (8, 3, 64), (4, 20, 4096 * 5 + 17)])
def test_walk_shapes(shape):
    """Edge shapes: arity 1 and 2, domains > 64 values (multi-word), t = 64, ragged t."""
    n, d, t = shape
    p = random_table(n, d, t, seed=n * 1000 + d)
    tab = make(p)
    run_walk(tab, p, calls=120, seed=3, check_table_every=5)
    tab.close()


@pytest.mark.parametrize("path", [dict(_grid_fused=True), dict(_grid_fused=True, _grid=3),
                                  dict(_grid_fused=True, _grid=3, _fast=False), dict(_grid_fused=True, _grid=5,
                                                                                     use_index=False)],
                         ids=["fast", "fast_g3", "v1_g3", "fast_g5_noindex"])
def test_walk_multitile(path):
    """Several update tiles per CTA (chained-scan look-back across rounds) and
    filter scans beyond the probe's first round."""
    p = random_table(6, 16, 300_000 + 77, seed=31)
    tab = make(p, **path)
    run_walk(tab, p, calls=120, seed=6, check_table_every=6)
    tab.close()


def test_walk_config2_full():
    """BASELINE config 2: arity 5, domain 20, 1e5 tuples, 1000 random-removal calls."""
    p = random_table(5, 20, 100_000, seed=1)
    tab = make(p)
    nfail, nsolved = run_walk(tab, p, calls=1000, seed=2, check_table_every=50)
    assert nfail > 0 and nsolved > 0
    tab.close()


def test_banded_walk():
    p = banded_table(5, 30, 20000, seed=4)
    tab = make(p)
    run_walk(tab, p, calls=200, seed=8, check_table_every=10, m=1, q=0.8)
    tab.close()


# --------------------------------------------------------------------------- C3 at full size (sampled)
@pytest.fixture(scope="module")
def c3():
    return random_table(8, 100, 10_000_000, seed=3)


@pytest.mark.parametrize("fast", [True, False], ids=["fast", "v1"])
def test_config3_bulk_full_size(c3, fast):
    """BASELINE config 3 (1e7 tuples, ~1 GB supports) in the bench's launch
    configuration: root, then bulk calls from the root, each vs the oracle
    (domains, pruned set and the full currTable)."""
    p = c3
    tab = make(p, _fast=fast)
    check_root(tab, p)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    rng = Rng(11)
    st = tab.root.clone()
    out_dev_checked = False
    for k in range(3):
        rem = bulk_removal(rng, root_m, p.d, q=0.5)
        din = root_m & (1 - rem)
        ok, dout, valid = oracle_call(p, din, want_valid=True)
        st.copy_from(tab.root)
        status, dom, pr = st.propagate(member_to_bitmap(rem, p.d))
        assert status == (CT_OK if ok else CT_FAIL)
        if ok:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout)
            assert np.array_equal(bits_to_bool(st.read_table(), p.t), valid)
        if not out_dev_checked:
            # the device-buffer entry point gives the same answer
            import torch
            wd = tab.Wd
            st.copy_from(tab.root)
            remd = torch.from_numpy(member_to_bitmap(rem, p.d).view(np.int64)).cuda()
            outd = torch.zeros(wd, dtype=torch.int64, device="cuda")
            sd = torch.zeros(1, dtype=torch.int32, device="cuda")
            torch.cuda.synchronize()   # torch's copies / memsets run on its own stream, the call on the state's
            st.propagate_async(remd, outd, None, sd)
            st.synchronize()
            assert int(sd.item()) == (CT_OK if ok else CT_FAIL)
            if ok:
                assert np.array_equal(bitmap_to_member(outd.cpu().numpy().view(np.uint64), p.d), dout)
            # and on pinned host buffers (zero-copy; bench.py's e2e calls)
            st.copy_from(tab.root)
            remh = torch.from_numpy(member_to_bitmap(rem, p.d).view(np.int64)).pin_memory()
            outh = torch.zeros(wd, dtype=torch.int64).pin_memory()
            prh = torch.zeros(wd, dtype=torch.int64).pin_memory()
            sh = torch.full((1,), -1, dtype=torch.int32).pin_memory()
            st.propagate_async(remh, outh, prh, sh)
            st.synchronize()
            assert int(sh.item()) == (CT_OK if ok else CT_FAIL)
            if ok:
                assert np.array_equal(bitmap_to_member(outh.numpy().view(np.uint64), p.d), dout)
                assert np.array_equal(bitmap_to_member(prh.numpy().view(np.uint64), p.d), din & (1 - dout))
            out_dev_checked = True
    # a few walk calls continuing from the last bulk state
    st.close()
    tab.close()


@pytest.mark.parametrize("path", [dict(), dict(_grid_fused=True), dict(_grid_fused=True, _fast=False),
                                  dict(_wide=True)], ids=["small", "fast", "fused", "wide"])
def test_pipelined_pinned_host_calls(path):
    """Many ct_propagate_async calls in flight on pinned host buffers (the
    kernels read the removals from and write status/domains/pruned to host
    memory), each from the root, checked against the oracle after one sync."""
    import torch
    p = random_table(4, 40, 30_000, seed=17)
    tab = make(p, **path)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    rng = Rng(5)
    st = tab.root.clone()
    n, wd = 24, tab.Wd
    rems = [bulk_removal(rng, root_m, p.d, q=0.3) for _ in range(n)]
    h_rem = torch.from_numpy(np.stack([member_to_bitmap(r, p.d) for r in rems]).view(np.int64)).pin_memory()
    h_dom = torch.zeros((n, wd), dtype=torch.int64).pin_memory()
    h_pr = torch.zeros((n, wd), dtype=torch.int64).pin_memory()
    h_st = torch.full((n,), -1, dtype=torch.int32).pin_memory()
    for k in range(n):
        st.copy_from(tab.root)
        st.propagate_async(h_rem[k], h_dom[k], h_pr[k], h_st[k])
    st.synchronize()
    for k in range(n):
        din = root_m & (1 - rems[k])
        ok, dout, _ = oracle_call(p, din)
        assert int(h_st[k]) == (CT_OK if ok else CT_FAIL), k
        if ok:
            assert np.array_equal(bitmap_to_member(h_dom[k].numpy().view(np.uint64), p.d), dout), k
            assert np.array_equal(bitmap_to_member(h_pr[k].numpy().view(np.uint64), p.d), din & (1 - dout)), k
    st.close()
    tab.close()


@pytest.mark.parametrize("fast,gather", [(True, True), (True, False), (False, True)], ids=["fast", "fast_scan", "v1"])
def test_config3b_banded_filter_heavy(fast, gather):
    """Fixing x0 on the banded table leaves ~1 % of the tuples valid and ~630
    unsupported values: k_fast resolves the residue misses by gathering the
    valid tuples' values (use_gather) or by Alg. 3's full scans; both vs the
    oracle, with currTable checked on the first call."""
    p = banded_table(8, 100, 2_000_000, seed=4)
    tab = make(p, _fast=fast, use_gather=gather)
    info = tab.info
    assert (info.gather_cell_bits == 8) == (fast and gather)
    check_root(tab, p)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    rng = Rng(12)
    st = tab.root.clone()
    for k in range(3):
        rem = fix_one_value_removal(rng, root_m, p.d, var=0)
        ok, dout, _ = oracle_call(p, root_m & (1 - rem))
        st.copy_from(tab.root)
        status, dom, _ = st.propagate(member_to_bitmap(rem, p.d))
        assert status == (CT_OK if ok else CT_FAIL)
        if ok:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout)
        s = st.stats()
        assert s.n_residue_miss > 0          # this workload exercises the full scans
        assert (s.filter_gathered_tuples > 0) == (fast and gather)
        if k == 0 and ok:
            _, _, valid = oracle_call(p, root_m & (1 - rem), want_valid=True)
            assert np.array_equal(bits_to_bool(st.read_table(), p.t), valid)
    st.close()
    tab.close()


@pytest.mark.parametrize("gather", [True, False], ids=["gather", "scan"])
@pytest.mark.parametrize("shape", [(3, 40, 200_000), (6, 100, 300_001), (5, 300, 400_003)])
def test_gather_filter_walks(shape, gather):
    """Banded tables (8-bit and 16-bit cells: d = 300) walked with P(2, 0.5)
    and with x0 fixed: the gather filter and the scan filter both equal the
    oracle on every call (domains, pruned sets, currTable every 7 calls)."""
    n, d, t = shape
    p = banded_table(n, d, t, seed=40 + n, band=max(3, d // 10))
    tab = make(p, _grid_fused=True, use_gather=gather)
    run_walk(tab, p, 60, seed=5, check_table_every=7)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    rng = Rng(13)
    st = tab.root.clone()
    for k in range(4):
        rem = fix_one_value_removal(rng, root_m, p.d, var=0)
        ok, dout, valid = oracle_call(p, root_m & (1 - rem), want_valid=True)
        st.copy_from(tab.root)
        status, dom, pr = st.propagate(member_to_bitmap(rem, p.d))
        assert status == (CT_OK if ok else CT_FAIL), k
        if ok:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout), k
            assert np.array_equal(bits_to_bool(st.read_table(), p.t), valid), k
    st.close()
    tab.close()


# --------------------------------------------------------------------------- f2: paper-shaped (LIN) tables, k_wide
@pytest.mark.parametrize("preset", ["lin_b", "lin_eb"])
def test_lin_knapsack_walk(preset):
    """Knapsack-configuration tables shaped like the paper's LIN_B / LIN_EB sets
    (Table tbl:instances): many support rows, few words,
    filter-heavy -> the k_wide shape.  Policy P(2, 0.5) walk, every call vs the
    oracle (status, domains, pruned, currTable every 10 calls)."""
    from workloads import knapsack_table, LIN_PRESETS
    p = knapsack_table(seed=21, **LIN_PRESETS[preset])
    tab = make(p)
    assert C.KERNEL_PATHS[tab.info.kernel_path] == "k_wide"
    nfail, _ = run_walk(tab, p, calls=120, seed=31, check_table_every=10)
    assert nfail > 0
    tab.close()


def test_lin_knapsack_assignments():
    """Search-like calls on a LIN table: fix one variable to one of its values
    (the x = v branch of the paper's DFS), from the root."""
    from workloads import knapsack_table, LIN_PRESETS
    p = knapsack_table(seed=22, n=90, max_dom=400, t=6000)
    tab = make(p)
    root_ok, root_m = check_root(tab, p)
    rng = Rng(41, lanes=1)
    st = tab.root.clone()
    for k in range(40):
        rem = fix_one_value_removal(rng, root_m, p.d, var=k % p.n)
        ok, dout, valid = oracle_call(p, root_m & (1 - rem), want_valid=True)
        st.copy_from(tab.root)
        status, dom, _ = st.propagate(member_to_bitmap(rem, p.d))
        assert status == (CT_OK if ok else CT_FAIL), k
        if ok:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout), k
            assert np.array_equal(bits_to_bool(st.read_table(), p.t), valid), k
    st.close()
    tab.close()


@pytest.mark.parametrize("knob", ["auto", "dom", "delta", "nores", "noindex", "nograph"])
def test_wide_forced_random(knob):
    """k_wide forced on an i.i.d. table (few rows) under every knob."""
    kw = {"auto": {}, "dom": dict(update_policy=CT_POLICY_DOM), "delta": dict(update_policy=CT_POLICY_DELTA),
          "nores": dict(use_residues=False), "noindex": dict(use_index=False), "nograph": dict(use_graph=False)}[knob]
    p = random_table(5, 20, 60_000 + 7, seed=13, lo=-4)
    tab = make(p, _wide=True, **kw)
    assert C.KERNEL_PATHS[tab.info.kernel_path] == "k_wide"
    run_walk(tab, p, calls=80, seed=17, check_table_every=8)
    tab.close()


# --------------------------------------------------------------------------- launch-shape boundaries
@pytest.mark.parametrize("t,expect", [(8192 * 128, "k_small"), (8192 * 128 + 1, "k_fast")])
def test_boundary_small_vs_fast(t, expect):
    """W2 = 8192 blocks is the last table of the one-CTA shape; one tuple more
    takes the cooperative grid."""
    p = random_table(3, 6, t, seed=61)
    tab = make(p)
    assert C.KERNEL_PATHS[tab.info.kernel_path] == expect
    run_walk(tab, p, calls=25, seed=62, check_table_every=6)
    tab.close()


@pytest.mark.parametrize("d,expect", [(2048, "k_fast"), (2049, "k_fused")])
def test_boundary_fast_rows(d, expect):
    """k_fast keeps the per-CTA lists in shared memory up to R = 4096 rows."""
    p = random_table(2, d, 1_200_000 + 3, seed=63)
    tab = make(p)
    assert C.KERNEL_PATHS[tab.info.kernel_path] == expect
    run_walk(tab, p, calls=25, seed=64, check_table_every=6)
    tab.close()


@pytest.mark.parametrize("d,expect", [(1023, "k_small"), (1024, "k_wide")])
def test_boundary_wide_rows(d, expect):
    """k_wide takes over from k_small at R = 2048 support rows."""
    p = random_table(2, d, 30_000 + 9, seed=65)   # W2 x R under k_small's work limit
    tab = make(p)
    assert C.KERNEL_PATHS[tab.info.kernel_path] == expect
    run_walk(tab, p, calls=40, seed=66, check_table_every=8)
    tab.close()


def test_fast_ranges_beyond_one_pass():
    """A table whose index exceeds 148 SMs x 6 CTAs x 128 entries: every k_fast
    CTA walks its range in several passes (W2 = 125 000 blocks)."""
    p = random_table(2, 8, 16_000_000, seed=67)
    tab = make(p)
    assert C.KERNEL_PATHS[tab.info.kernel_path] == "k_fast"
    assert (p.t + 127) // 128 > tab.info.grid * 128
    run_walk(tab, p, calls=8, seed=68, check_table_every=4)
    tab.close()


def test_batch_single_state():
    p = random_table(4, 12, 30_000, seed=69)
    tab = make(p)
    batch_walk(tab, p, S=1, steps=6, seed=70, check_table=True)
    tab.close()


# --------------------------------------------------------------------------- edge cases
def test_empty_table_root_fail():
    tab = Table([0, 0], [3, 3], np.zeros((0, 2), np.int32))
    assert tab.root_status == CT_FAIL and tab.root_dom is None
    with pytest.raises(CTError) as e:
        tab.root.propagate(None)
    assert e.value.status == CT_ESTATE
    tab.close()


def test_all_tuples_out_of_range_root_fail():
    tab = Table([0], [4], np.array([[7], [-1], [4]], np.int32))
    assert tab.root_status == CT_FAIL
    tab.close()


def test_init_dom_holes_and_single_tuple():
    p = random_table(3, 10, 500, seed=9, lo=100)
    D = (Rng(4).uniform(p.R, 3) > 0).astype(np.uint8)
    tab = Table(p.lo, p.d, p.tuples, init_dom=member_to_bitmap(D, p.d))
    ok, dout, _ = oracle_call(p, D)
    assert (tab.root_status == CT_OK) == ok
    if ok:
        assert np.array_equal(bitmap_to_member(tab.root_dom, p.d), dout)
    tab.close()
    one = np.array([[5, 6]], np.int32)
    tab = Table([5, 5], [3, 3], one)
    assert bitmap_to_member(tab.root_dom, [3, 3]).tolist() == [1, 0, 0, 0, 1, 0]
    tab.close()


def test_noop_idempotence_absent_values_and_garbage_bits():
    p = random_table(4, 70, 5000, seed=13)
    tab = make(p)
    st = tab.root.clone()
    root = tab.root_dom.copy()
    status, dom, pr = st.propagate(None)                  # nothing removed -> unchanged
    assert status == CT_OK and np.array_equal(dom, root) and not pr.any()
    assert st.stats().noop == 1
    # bits >= d and already-absent values are ignored (include/ct.h)
    garbage = np.zeros(tab.Wd, np.uint64)
    offs = dom_word_offsets(p.d)
    for i in range(p.n):
        garbage[offs[i + 1] - 1] = np.uint64(0xFFFFFFFFFFFFFFFF) << np.uint64(70 - 64)
    status, dom, _ = st.propagate(garbage)
    assert status == CT_OK and np.array_equal(dom, root)
    # idempotence after a real removal
    rem = np.zeros(p.R, np.uint8)
    rem[3:40] = 1
    status, d1, _ = st.propagate(member_to_bitmap(rem, p.d))
    status2, d2, pr2 = st.propagate(member_to_bitmap(rem, p.d))
    assert status == status2 == CT_OK and np.array_equal(d1, d2) and not pr2.any()
    tab.close()


def test_dead_state_and_restore():
    p = table1()
    tab = make(p)
    st = tab.root.clone()
    rem = member_from_lists(p.lo, p.d, [[2, 3], [2, 3, 4], []])   # x1={1}, x2={1} -> FAIL
    status, _, _ = st.propagate(member_to_bitmap(rem, p.d))
    assert status == CT_FAIL
    with pytest.raises(CTError) as e:
        st.propagate(None)
    assert e.value.status == CT_ESTATE
    st.copy_from(tab.root)
    status, dom, _ = st.propagate(None)
    assert status == CT_OK and np.array_equal(dom, tab.root_dom)
    tab.close()


def test_confluence_two_calls_vs_one():
    p = random_table(5, 20, 20000, seed=17)
    tab = make(p)
    rng = Rng(9)
    a, b = tab.root.clone(), tab.root.clone()
    for trial in range(30):
        r1 = (rng.uniform(p.R, 6) == 0).astype(np.uint8)
        r2 = (rng.uniform(p.R, 6) == 0).astype(np.uint8)
        a.copy_from(tab.root)
        b.copy_from(tab.root)
        s1, _, _ = a.propagate(member_to_bitmap(r1, p.d))
        if s1 == CT_OK:
            s1, da, _ = a.propagate(member_to_bitmap(r2, p.d))
        s2, db, _ = b.propagate(member_to_bitmap(r1 | r2, p.d))
        assert s1 == s2
        if s1 == CT_OK:
            assert np.array_equal(da, db)
    tab.close()


# --------------------------------------------------------------------------- batched (a9)
# (arity, domain, tuples, lo): tile widths 32 (R <= 400), 16 (R <= 800), 8
# (R <= 1600) and the per-state kernels beyond; R < 32; blocks not a multiple
# of the tile width; a single 16-byte block.
BATCH_SHAPES = {
    "c4like": (6, 50, 200_000, 0),
    "tw16": (8, 90, 120_000 + 77, 3),
    "tw8": (10, 140, 60_000 + 5, -2),
    "perstate": (12, 150, 30_000 + 1, 0),
    "tinyR": (3, 7, 5_000 + 13, 1),
    "oneblock": (4, 6, 100, 0),
}
BATCH_PATHS = {"tiled": {}, "legacy": {"batch_per_state": True}}


def make_env(p, cfg, **kw):
    return make(p, **cfg, **kw)


def batch_walk(tab, p, S, steps, seed, check_table=False, from_states=None, work_out=None):
    """S independent policy-P(2, 0.5) walks through ct_propagate_many, each state
    checked against the oracle (status, domains; currTable if asked); FAILed
    slots are restored by ct_batch_copy (odd steps) or ct_batch_restore_dead."""
    b = tab.batch(S)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    cur = [root_m.copy() for _ in range(S)]
    if from_states is not None:                   # slots initialised from single states
        for s, (st, m) in from_states.items():
            b.copy(s, st)
            cur[s] = m.copy()
    rngs = [Rng(seed + s, lanes=1) for s in range(S)]
    from workloads.policies import walk_removal
    nfail = 0
    for step in range(steps):
        rem = np.zeros((S, tab.Wd), np.uint64)
        exp = []
        for s in range(S):
            r = walk_removal(rngs[s], cur[s], p.d)
            if r is None:
                r = np.zeros(p.R, np.uint8)
            rem[s] = member_to_bitmap(r, p.d)
            exp.append(oracle_call(p, cur[s] & (1 - r), want_valid=check_table))
        status, doms = b.propagate(rem)
        for s in range(S):
            ok, dout, valid = exp[s]
            assert status[s] == (CT_OK if ok else CT_FAIL), (step, s)
            if ok:
                assert np.array_equal(bitmap_to_member(doms[s], p.d), dout), (step, s)
                if check_table:
                    assert np.array_equal(bits_to_bool(b.read_table(s), p.t), valid), (step, s)
                cur[s] = dout
            else:
                nfail += 1
                if step % 2:
                    b.copy(s, tab.root)             # host-driven restore of one slot
                cur[s] = root_m.copy()              # (even steps: restored by the device kernel)
        b.restore_dead(tab.root)
    if work_out is not None:
        work_out.update(b.work())
    b.close()
    return nfail


@pytest.mark.parametrize("path", list(BATCH_PATHS))
@pytest.mark.parametrize("shape", list(BATCH_SHAPES))
def test_batch_matches_oracle(shape, path):
    n, d, t, lo = BATCH_SHAPES[shape]
    p = random_table(n, d, t, seed=5, lo=lo)
    tab = make_env(p, BATCH_PATHS[path])
    tw = {"c4like": 32, "tw16": 16, "tw8": 8, "perstate": 0, "tinyR": 32, "oneblock": 32}[shape]
    assert tab.info.batch_tile == (tw if path == "tiled" else 0)
    batch_walk(tab, p, S=67, steps=10, seed=1000, check_table=(shape in ("c4like", "tinyR", "oneblock")))
    tab.close()


@pytest.mark.parametrize("cells", [True, False])
def test_batch_cell_and_sparse_routes(cells):
    """The tile-major update's cell route (few valid tuples in a (state, tile):
    each is checked against the new domains instead of OR-ing support rows) and
    the sparse-state route (k_bsparse: states with few active blocks updated
    through their index) reach the oracle's results; batch_cells = 0 turns
    both off.  Long walks so that states become sparse."""
    p = random_table(6, 50, 200_000, seed=15)
    tab = make(p, batch_cells=cells)
    assert tab.info.batch_tile == 32 and tab.info.batch_cells == int(cells)
    work = {}
    batch_walk(tab, p, S=48, steps=14, seed=4000, check_table=True, work_out=work)
    assert (work["update_cells_checked"] > 0) == cells
    assert (work["update_sparse_states"] > 0) == cells
    tab.close()


@pytest.mark.parametrize("knob", ["dom", "delta", "nores", "noindex"])
def test_batch_knobs(knob):
    kw = {"dom": dict(update_policy=CT_POLICY_DOM), "delta": dict(update_policy=CT_POLICY_DELTA),
          "nores": dict(use_residues=False), "noindex": dict(use_index=False)}[knob]
    p = random_table(6, 30, 40_000, seed=9)
    tab = make(p, **kw)
    batch_walk(tab, p, S=40, steps=8, seed=2000, check_table=True)
    tab.close()


def test_batch_banded_filter_scans():
    """Correlated (banded) table: fixing x0 leaves most values of the other
    variables unsupported, so the batch filter runs full scans."""
    p = banded_table(5, 40, 50_000, seed=4)
    tab = make(p)
    S = 40
    b = tab.batch(S)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    rem = np.zeros((S, tab.Wd), np.uint64)
    exp = []
    for s in range(S):
        r = fix_one_value_removal(Rng(300 + s, lanes=1), root_m, p.d, var=s % p.n)
        rem[s] = member_to_bitmap(r, p.d)
        exp.append(oracle_call(p, root_m & (1 - r), want_valid=True))
    status, doms = b.propagate(rem)
    for s in range(S):
        ok, dout, valid = exp[s]
        assert status[s] == (CT_OK if ok else CT_FAIL)
        if ok:
            assert np.array_equal(bitmap_to_member(doms[s], p.d), dout), s
            assert np.array_equal(bits_to_bool(b.read_table(s), p.t), valid), s
    st = b.stats()
    assert sum(x.n_residue_miss for x in st) > 0
    b.close()
    tab.close()


def test_batch_slots_from_compacted_states():
    """Slots copied from single states that carry a compacted index (k_fast /
    k_small history) continue correctly in the dense batch path, and a batch
    state equals the same state propagated alone."""
    p = random_table(6, 50, 200_000, seed=5)
    tab = make(p)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    rng = Rng(55, lanes=1)
    from workloads.policies import walk_removal
    singles = {}
    for s in (0, 3, 7):
        st = tab.root.clone()
        cur = root_m.copy()
        for _ in range(2):
            r = walk_removal(rng, cur, p.d, q=0.3)
            ok, dout, _ = oracle_call(p, cur & (1 - r))
            status, dom, _ = st.propagate(member_to_bitmap(r, p.d))
            assert status == (CT_OK if ok else CT_FAIL)
            if not ok:
                st.copy_from(tab.root)
                cur = root_m.copy()
            else:
                cur = dout
        singles[s] = (st, cur)
    batch_walk(tab, p, S=9, steps=6, seed=3000, check_table=True, from_states=singles)
    for st, _ in singles.values():
        st.close()
    tab.close()


# --------------------------------------------------------------------------- sharded (a10)
PATHS = {"small": dict(), "fast": dict(_grid_fused=True), "v1": dict(_grid_fused=True, _fast=False),
         "wide": dict(_wide=True)}


def _skewed_table(kind):
    """Shard-hostile tables: rows sorted by x0 (values of x0 live in one shard
    only), a two-block table whose halves support disjoint values, and a table
    so small that shard 0 owns no tuple word at G = 2 (ct_shard_range)."""
    from workloads.tables import Problem
    if kind == "iid":
        return random_table(5, 20, 50_000 + 33, seed=23)
    if kind == "sorted":
        p = random_table(5, 20, 50_000 + 33, seed=24)
        order = np.argsort(p.tuples[:, 0], kind="stable")
        return Problem("sorted_by_x0", p.lo, p.d, np.ascontiguousarray(p.tuples[order]), 24)
    if kind == "halves":
        t = np.zeros((2048, 2), np.int32)
        t[1024:] = 1
        return Problem("halves", np.zeros(2, np.int32), np.array([2, 2], np.int32), t, 0)
    if kind == "tiny":
        p = random_table(3, 6, 1000, seed=25)
        return p
    raise KeyError(kind)


def _combine_virtual(states):
    """Caller-side OR of the shard flags (all-reduce MAX over uint8), on one GPU."""
    import torch
    from paper_2507_18413_b200.sharded import flags_tensor
    for st in states:
        st.synchronize()
    fl = [flags_tensor(st.handle) for st in states]
    comb = torch.stack(fl).amax(dim=0)
    for f in fl:
        f.copy_(comb)
    torch.cuda.synchronize()


def _apply_virtual(states, wd):
    import torch
    outs = []
    for st in states:
        od = torch.zeros(max(wd, 1), dtype=torch.int64, device="cuda")
        pd = torch.zeros(max(wd, 1), dtype=torch.int64, device="cuda")
        sd = torch.zeros(1, dtype=torch.int32, device="cuda")
        torch.cuda.synchronize()
        C.ct_propagate_apply_async(st.handle, od, pd, sd)
        st.synchronize()
        outs.append((int(sd.item()), od.cpu().numpy().view(np.uint64)[:wd], pd.cpu().numpy().view(np.uint64)[:wd]))
    return outs


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("G", [2, 3, 5])
@pytest.mark.parametrize("kind", ["iid", "sorted", "halves", "tiny"])
def test_virtual_shards_one_gpu(G, path, kind):
    """G tuple-range shards on one device, flags OR-combined by the caller --
    the root included: ct_create returns CT_PENDING after the root's local phase
    and the root verdict comes from the combine + apply (include/ct.h).  Tables
    whose values are supported in one shard only, and shards with no tuple."""
    from paper_2507_18413_b200 import CT_PENDING
    p = _skewed_table(kind)
    full = make(p)
    shards = [make(p, n_shards=G, shard_rank=g, **PATHS[path]) for g in range(G)]
    ok0, root_o = oracle_call(p, np.ones(p.R, np.uint8))[:2]
    assert (full.root_status == CT_OK) == ok0
    for s in shards:
        assert s.root_status == CT_PENDING and s.root_dom is None
        with pytest.raises(CTError) as e:        # unusable until applied
            s.root.clone()
        assert e.value.status == CT_ESTATE
    wd = full.Wd
    roots = [s.root for s in shards]
    _combine_virtual(roots)
    for sd, od, _ in _apply_virtual(roots, wd):
        assert sd == (CT_OK if ok0 else CT_FAIL)
        if ok0:
            assert np.array_equal(bitmap_to_member(od, p.d), root_o)
    # the shards tile the table
    rngs = [C.ct_shard_range(p.t, G, g) for g in range(G)]
    assert rngs[0][0] == 0 and sum(w for _, w in rngs) == (p.t + 63) // 64
    if not ok0:
        return
    states = [s.root.clone() for s in shards]
    rng = Rng(77)
    cur = root_o.copy()
    from workloads.policies import walk_removal
    import torch
    for k in range(60):
        r = walk_removal(rng, cur, p.d)
        if r is None:
            for st, s in zip(states, shards):
                st.copy_from(s.root)
            cur = root_o.copy()
            continue
        din = cur & (1 - r)
        ok, dout, _ = oracle_call(p, din)
        remd = torch.from_numpy(member_to_bitmap(r, p.d).view(np.int64)).cuda()
        torch.cuda.synchronize()   # the H2D copy runs on torch's stream, the calls on the states' streams
        for st in states:
            C.ct_propagate_local_async(st.handle, remd)
        _combine_virtual(states)
        for sd, od, pd in _apply_virtual(states, wd):
            assert sd == (CT_OK if ok else CT_FAIL), k
            if ok:
                assert np.array_equal(bitmap_to_member(od, p.d), dout), k
                assert np.array_equal(bitmap_to_member(pd, p.d), din & (1 - dout)), k
        if ok:
            cur = dout
        else:
            for st, s in zip(states, shards):
                st.copy_from(s.root)
            cur = root_o.copy()
    for s in shards:
        s.close()
    full.close()


@pytest.mark.parametrize("path", list(PATHS))
def test_nccl_single_rank_path(path):
    """The in-library NCCL combine (all-reduce inside the call) on a 1-rank communicator."""
    p = random_table(5, 20, 30_000, seed=29)
    nid = C.ct_nccl_unique_id()
    tab = make(p, n_shards=1, shard_rank=0, nccl_unique_id=nid, **PATHS[path])
    run_walk(tab, p, calls=150, seed=4, check_table_every=10)
    tab.close()


@pytest.mark.parametrize("kind", ["iid", "banded"])
def test_peer_combine_single_rank(kind):
    """a10 over NVLink peer memory (ct_peer_attach) with one rank: k_fast's
    finalizer stores its shard flags into the inbox, releases them at system
    scope, acquires them back and ORs them before finalizing -- the protocol
    each of G ranks runs -- and every call of a walk (synchronous calls: the
    captured graph is re-captured after the attach) matches the oracle.  The
    banded table drives the filter through misses (gather / scans)."""
    p = random_table(8, 60, 400_000 + 77, seed=31) if kind == "iid" else banded_table(6, 40, 300_000, seed=8)
    tab = make(p, _grid_fused=True)
    assert tab.info.kernel_path == 2
    st0 = tab.root.clone()
    st0.propagate(np.zeros(tab.Wd, np.uint64))      # a graph captured before the attach goes stale
    h = C.ct_peer_export(tab.handle)
    assert len(h) == C.CT_PEER_HANDLE_BYTES
    C.ct_peer_attach(tab.handle, [h])
    with pytest.raises(CTError) as e:                # attach is once per table
        C.ct_peer_attach(tab.handle, [h])
    assert e.value.status == C.CT_EINVAL
    nfail, _ = run_walk(tab, p, calls=150, seed=9, check_table_every=10)
    st0.close()
    tab.close()


def test_peer_attach_needs_k_fast():
    p = random_table(5, 20, 30_000, seed=29)          # a k_small table
    tab = make(p)
    assert tab.info.kernel_path != 2
    h = C.ct_peer_export(tab.handle)
    with pytest.raises(CTError) as e:
        C.ct_peer_attach(tab.handle, [h])
    assert e.value.status == C.CT_EINVAL
    with pytest.raises(CTError):                     # wrong handle count
        C.ct_peer_attach(tab.handle, [h, h])
    tab.close()


@pytest.mark.parametrize("shape", ["c2", "tiny"])
def test_served_walk(shape):
    """ct_state_serve: a persistent k_small answers the synchronous calls
    through a doorbell in mapped host memory; every call of a walk (restores
    after FAIL / solved stop and restart the server) matches the oracle,
    currTable included."""
    p = random_table(5, 20, 100_000, seed=1) if shape == "c2" else random_table(3, 5, 300, seed=2)
    tab = make(p)
    assert tab.info.kernel_path == 3
    nfail, nsolved = run_walk(tab, p, calls=300, seed=12, check_table_every=25, serve=True)
    assert nfail + nsolved > 0
    tab.close()


def test_served_idle_restart():
    """The server stops on its idle limit; the next call finds it stopped and
    restarts it (the request is served exactly once)."""
    import time
    p = random_table(5, 20, 50_000, seed=3)
    tab = make(p)
    root_m = bitmap_to_member(tab.root_dom, p.d)
    st = tab.root.clone()
    st.serve(True)
    C.ct_debug_serve_idle(2_000_000)                  # 2 ms
    try:
        rng = Rng(5, lanes=1)
        cur = root_m.copy()
        for k in range(12):
            r = walk_removal(rng, cur, p.d, q=0.2)
            if r is None:
                break
            ok, dout = oracle_call(p, cur & (1 - r))[:2]
            status, dom, _ = st.propagate(member_to_bitmap(r, p.d))
            assert status == (CT_OK if ok else CT_FAIL), k
            if not ok:
                break
            assert np.array_equal(bitmap_to_member(dom, p.d), dout), k
            cur = dout
            time.sleep(0.01 if k % 2 else 0.0)        # every other call: the server has stopped
    finally:
        C.ct_debug_serve_idle(200_000_000)
    st.close()
    tab.close()


def test_serve_needs_single_cta_shape():
    p = random_table(5, 20, 30_000, seed=29)
    tab = make(p, _grid_fused=True)                   # k_fast
    with pytest.raises(CTError) as e:
        tab.root.clone().serve(True)
    assert e.value.status == C.CT_EINVAL
    tab.close()


# --------------------------------------------------------------------------- ct_propagate_from_async
FROM_SHAPES = {"fast": dict(_grid_fused=True), "fast_scan": dict(_grid_fused=True, use_gather=False),
               "fast_noindex": dict(_grid_fused=True, use_index=False), "v1": dict(_grid_fused=True, _fast=False),
               "small": dict()}


def test_pipelined_host_buffer_calls():
    """Calls kept in flight with pinned host-memory inputs and outputs
    (bench.py's e2e pattern): every call's removal is DMA'd into one of the
    state's two device slots on its copy stream while the previous call runs;
    each call propagates from the root into the work state and writes its
    outputs to its own host buffers, all checked against the oracle after one
    sync."""
    import torch
    from workloads.policies import bulk_removal
    p = random_table(6, 30, 300_000 + 5, seed=17)
    tab = make(p, _grid_fused=True)
    ok, root_m, _ = oracle_call(p, np.ones(p.R, np.uint8))
    wd = tab.Wd
    K = 12
    rng = Rng(33)
    rems = [bulk_removal(rng, root_m, p.d, q=0.3 + 0.04 * k) for k in range(K)]
    pin = lambda n, dt: torch.zeros(n, dtype=dt, pin_memory=True)
    rbuf = [pin(wd, torch.int64) for _ in range(K)]
    obuf = [pin(wd, torch.int64) for _ in range(K)]
    pbuf = [pin(wd, torch.int64) for _ in range(K)]
    sbuf = [pin(1, torch.int32) for _ in range(K)]
    for k in range(K):
        rbuf[k].numpy()[:] = member_to_bitmap(rems[k], p.d).view(np.int64)
    work = tab.root.clone()
    for k in range(K):
        work.propagate_from_async(tab.root, rbuf[k], obuf[k], pbuf[k], sbuf[k])
    work.synchronize()
    for k in range(K):
        din = root_m & (1 - rems[k])
        okk, dout, _ = oracle_call(p, din)
        assert int(sbuf[k][0]) == (CT_OK if okk else CT_FAIL), k
        if okk:
            assert np.array_equal(bitmap_to_member(obuf[k].numpy().view(np.uint64), p.d), dout), k
            assert np.array_equal(bitmap_to_member(pbuf[k].numpy().view(np.uint64), p.d), din & (1 - dout)), k
    work.close()
    tab.close()


@pytest.mark.parametrize("shape", list(FROM_SHAPES))
def test_propagate_from_walk(shape):
    """dst := src propagated (one pass on k_fast, copy + call elsewhere): a
    search-like walk where every call starts from a saved state and the result
    becomes the next source (so sources carry stale blocks outside their index
    only if the gap zeroing is wrong); domains, pruned sets and the whole
    currTable vs the oracle, the source unchanged, a no-op call from a source,
    and a batch seeded from a propagated state."""
    import torch
    p = banded_table(5, 30, 150_001, seed=9, band=6)
    tab = make(p, **FROM_SHAPES[shape])
    ok, root_m, _ = oracle_call(p, np.ones(p.R, np.uint8))
    assert ok
    wd = tab.Wd
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a).view(np.int64)).cuda()
    out = torch.zeros(wd, dtype=torch.int64, device="cuda")
    pr = torch.zeros(wd, dtype=torch.int64, device="cuda")
    sd = torch.zeros(1, dtype=torch.int32, device="cuda")
    states = [tab.root.clone(), tab.root.clone()]
    src, cur = tab.root, root_m.copy()
    rng = Rng(21, lanes=1)
    nfrom = 0
    for k in range(40):
        r = walk_removal(rng, cur, p.d)
        if r is None:
            src, cur = tab.root, root_m.copy()
            continue
        dst = states[k % 2] if states[k % 2] is not src else states[(k + 1) % 2]
        before = src.read_table().copy()
        din = cur & (1 - r)
        okk, dout, valid = oracle_call(p, din, want_valid=True)
        remd = dev(member_to_bitmap(r, p.d))
        torch.cuda.synchronize()
        dst.propagate_from_async(src, remd, out, pr, sd)
        dst.synchronize()
        src.synchronize()
        assert int(sd.item()) == (CT_OK if okk else CT_FAIL), k
        assert np.array_equal(src.read_table(), before), k          # the source is only read
        if okk:
            assert np.array_equal(bitmap_to_member(out.cpu().numpy().view(np.uint64), p.d), dout), k
            assert np.array_equal(bitmap_to_member(pr.cpu().numpy().view(np.uint64), p.d), din & (1 - dout)), k
            assert np.array_equal(bits_to_bool(dst.read_table(), p.t), valid), k
            src, cur = dst, dout
            nfrom += 1
        else:
            src, cur = tab.root, root_m.copy()
    assert nfrom > 10
    # a no-op call from a propagated source is a copy of it
    if src is not tab.root:
        dst = states[0] if states[0] is not src else states[1]
        torch.cuda.synchronize()
        dst.propagate_from_async(src, dev(np.zeros(wd, np.uint64)), out, pr, sd)
        dst.synchronize()
        assert int(sd.item()) == CT_OK
        assert np.array_equal(dst.read_table(), src.read_table())
        assert np.array_equal(out.cpu().numpy().view(np.uint64), src.read_dom())
        # batches read every block: a batch seeded from a propagated state
        b = tab.batch(4, init=dst)
        rems = [walk_removal(rng, cur, p.d) for _ in range(4)]
        rems = [x if x is not None else np.zeros(p.R, np.uint8) for x in rems]
        st_b, doms = b.propagate(np.stack([member_to_bitmap(x, p.d) for x in rems]))
        for s in range(4):
            okk, dout, _ = oracle_call(p, cur & (1 - rems[s]))
            assert st_b[s] == (CT_OK if okk else CT_FAIL), s
            if okk:
                assert np.array_equal(bitmap_to_member(doms[s], p.d), dout), s
        b.close()
    tab.close()
