"""GPU parity of f4 (PAPER.md L66-68 footnote): short tables
(star cells) and negative tables through the C ABI vs the oracle's
oracle_gac_short / oracle_gac_negative, bit-exact on every call of seeded
P(2, 0.5) walks, with the currTable checked against the oracle's valid set
(short) and its popcount against the oracle's count of valid forbidden tuples
(negative)."""
import numpy as np
import pytest

import oracle
from paper_2507_18413_b200 import (CT_OK, CT_FAIL, CT_POLICY_DOM, CT_POLICY_DELTA, CT_STAR, CTError, Table)
from paper_2507_18413_b200 import ct as C
from workloads import Rng, member_to_bitmap, bitmap_to_member, short_table, negative_table, bulk_removal
from workloads.layout import bits_to_bool
from workloads.policies import walk_removal

pytestmark = pytest.mark.gpu


def _make(p, kind, _grid_fused=False, **kw):
    if _grid_fused:
        kw["launch_shape"] = "fast"
    return Table(p.lo, p.d, p.tuples, kind=kind, **kw)


def _oracle(kind, p, member):
    if kind == "short":
        ok, dout, valid = oracle.gac_short(p.lo, p.d, p.tuples, member, want_valid=True)
        return ok, dout, valid
    ok, dout, nv = oracle.gac_negative(p.lo, p.d, p.tuples, member)
    return ok, dout, nv


def _walk(tab, p, kind, calls, seed, m=2, q=0.5):
    """P(m, q) walk; restore the root after FAIL or when solved.  Returns
    (fails, prunes) so callers can assert the regime was exercised."""
    root_in = np.ones(p.R, np.uint8)
    ok, root_m, aux = _oracle(kind, p, root_in)
    assert (tab.root_status == CT_OK) == ok
    if not ok:
        return 0, 0
    assert np.array_equal(bitmap_to_member(tab.root_dom, p.d), root_m)
    rng = Rng(seed, lanes=1)
    st = tab.root.clone()
    cur = root_m.copy()
    fails = prunes = 0
    for k in range(calls):
        rem = walk_removal(rng, cur, p.d, m=m, q=q)
        if rem is None:
            st.copy_from(tab.root)
            cur = root_m.copy()
            continue
        din = cur & (1 - rem)
        ok, dout, aux = _oracle(kind, p, din)
        status, gdom, gpr = st.propagate(member_to_bitmap(rem, p.d))
        assert status == (CT_OK if ok else CT_FAIL), f"call {k}"
        if ok:
            assert np.array_equal(bitmap_to_member(gdom, p.d), dout), f"call {k}: domains"
            assert np.array_equal(bitmap_to_member(gpr, p.d), din & (1 - dout)), f"call {k}: pruned"
            bits = st.read_table()
            if kind == "short":
                assert np.array_equal(bits_to_bool(bits, p.t), aux), f"call {k}: currTable"
            else:   # valid forbidden tuples w.r.t. the domains after the removal
                assert int(sum(bin(int(w)).count("1") for w in bits)) == aux, f"call {k}: |V|"
            prunes += int(np.any(dout != din))
            cur = dout
        else:
            fails += 1
            st.copy_from(tab.root)
            cur = root_m.copy()
    st.close()
    return fails, prunes


SHORT_KNOBS = [dict(), dict(update_policy=CT_POLICY_DOM), dict(update_policy=CT_POLICY_DELTA),
               dict(use_residues=False), dict(use_index=False), dict(use_fused=False), dict(_grid_fused=True)]
SHORT_IDS = ["auto", "dom", "delta", "nores", "noindex", "nofused", "gridfused"]


@pytest.mark.parametrize("knobs", SHORT_KNOBS, ids=SHORT_IDS)
@pytest.mark.parametrize("shape", [(3, 10, 40, 0.05), (4, 12, 300, 0.05), (5, 16, 3000, 0.02), (4, 30, 70_001, 0.01)])
def test_short_walk_vs_oracle(shape, knobs):
    n, d, t, ps = shape
    p = short_table(n, d, t, seed=7 + t, p_star=ps, lo=-2)
    tab = _make(p, "short", **knobs)
    fails, prunes = _walk(tab, p, "short", 120, seed=3)
    assert prunes > 0 and fails > 0
    tab.close()


def test_short_supports_rows_and_star_columns_take_dom_branch():
    """Star cells are in every row of their variable (supports vs definition),
    and a Δ-only policy still matches the oracle (the starred columns fall back
    to the dom-branch)."""
    p = short_table(3, 5, 300, seed=2, p_star=0.4)
    tab = _make(p, "short", update_policy=CT_POLICY_DELTA)
    W = (p.t + 63) // 64
    for i in range(p.n):
        for a in range(int(p.d[i])):
            got = bits_to_bool(C.ct_table_read_supports(tab.handle, i * int(p.d[i]) + a, W), p.t)
            exp = (p.tuples[:, i] == a) | (p.tuples[:, i] == CT_STAR)
            assert np.array_equal(got, exp), (i, a)
    _walk(tab, p, "short", 80, seed=5)
    tab.close()


def test_short_bulk_and_batch():
    """C3-bulk-shaped removal from the root on a multi-tile short table, and the
    batched path (ct_propagate_many) on the same table, vs the oracle."""
    p = short_table(6, 40, 200_003, seed=9, p_star=0.05)
    tab = _make(p, "short")
    rng = Rng(4)
    b = tab.batch(16)
    rems = []
    for s in range(16):
        rems.append(bulk_removal(rng, np.ones(p.R, np.uint8), p.d, q=0.5) if s % 2 == 0
                    else np.zeros(p.R, np.uint8))
    st, doms = b.propagate(np.stack([member_to_bitmap(r, p.d) for r in rems]))
    for s in range(16):
        ok, dout, _ = oracle.gac_short(p.lo, p.d, p.tuples, 1 - rems[s])
        assert st[s] == (CT_OK if ok else CT_FAIL), s
        if ok:
            assert np.array_equal(bitmap_to_member(doms[s], p.d), dout), s
    one = tab.root.clone()
    status, dom, _ = one.propagate(member_to_bitmap(rems[0], p.d))
    ok, dout, valid = oracle.gac_short(p.lo, p.d, p.tuples, 1 - rems[0], want_valid=True)
    assert status == (CT_OK if ok else CT_FAIL)
    if ok:
        assert np.array_equal(bitmap_to_member(dom, p.d), dout)
        assert np.array_equal(bits_to_bool(one.read_table(), p.t), valid)
    tab.close()


NEG_KNOBS = [dict(), dict(update_policy=CT_POLICY_DOM), dict(update_policy=CT_POLICY_DELTA),
             dict(use_index=False), dict(use_graph=False), dict(launch_shape="phases"),
             dict(launch_shape="phases", use_index=False), dict(launch_shape="fast", grid_override=3)]
NEG_IDS = ["auto", "dom", "delta", "noindex", "nograph", "kernels", "kernels_noindex", "fast_grid3"]


@pytest.mark.parametrize("knobs", NEG_KNOBS, ids=NEG_IDS)
@pytest.mark.parametrize("shape", [(2, 9, 70), (3, 12, 1400), (4, 10, 8000), (3, 60, 170_000)])
def test_negative_walk_vs_oracle(shape, knobs):
    """Dense forbidden lists (t ~ 0.8 x the product) so the walk prunes (FAIL is
    covered by test_negative_edge_cases)."""
    n, d, t = shape
    p = negative_table(n, d, t, seed=31 + t, lo=1)
    tab = _make(p, "negative", **knobs)
    expect = "negative" if knobs.get("launch_shape") == "phases" else "k_fast"
    assert C.KERNEL_PATHS[tab.info.kernel_path] == expect
    fails, prunes = _walk(tab, p, "negative", 150, seed=8, m=1, q=0.3)
    assert prunes > 0
    tab.close()


def test_negative_edge_cases():
    """Empty list: nothing pruned; the whole product listed: root FAIL;
    duplicates merged; slab x0 = a listed: exactly (x0, a) pruned; batches and
    shards rejected."""
    lo, d = np.array([0, 0, 0], np.int32), np.array([3, 2, 4], np.int32)
    empty = Table(lo, d, np.zeros((0, 3), np.int32), kind="negative")
    assert empty.root_status == CT_OK
    assert bitmap_to_member(empty.root_dom, d).tolist() == [1] * 9
    with pytest.raises(CTError):
        empty.batch(4)
    empty.close()
    full = np.array([[a, b, c] for a in range(3) for b in range(2) for c in range(4)], np.int32)
    t_full = Table(lo, d, np.concatenate([full, full[:5]]), kind="negative")
    assert t_full.root_status == CT_FAIL
    t_full.close()
    for a in range(3):
        slab = full[full[:, 0] == a]
        tab = Table(lo, d, np.concatenate([slab, slab]), kind="negative")
        exp = [1] * 9
        exp[a] = 0
        assert tab.root_status == CT_OK and bitmap_to_member(tab.root_dom, d).tolist() == exp
        # the pruned value's tuples leave currTable on the next call
        st = tab.root.clone()
        status, dom, _ = st.propagate(member_to_bitmap(np.array([0] * 9, np.uint8), d))
        assert status == CT_OK and bitmap_to_member(dom, d).tolist() == exp
        assert int(sum(bin(int(w)).count("1") for w in st.read_table())) == 0
        tab.close()
    with pytest.raises(CTError):
        Table(lo, d, full, kind="negative", n_shards=2, shard_rank=0)


def test_negative_bulk_large():
    """A 1e6-tuple negative table (n = 4, d = 40: 2.56e6 assignments) from the
    root: bulk removals that leave few enough assignments that rows get counted."""
    p = negative_table(4, 40, 1_000_000, seed=12)
    tab = _make(p, "negative")
    ok, root_m, _ = oracle.gac_negative(p.lo, p.d, p.tuples, np.ones(p.R, np.uint8))
    assert (tab.root_status == CT_OK) == ok
    rng = Rng(6)
    st = tab.root.clone()
    for k in range(6):
        rem = bulk_removal(rng, root_m, p.d, q=0.85)
        din = root_m & (1 - rem)
        okk, dout, nv = oracle.gac_negative(p.lo, p.d, p.tuples, din)
        st.copy_from(tab.root)
        status, dom, _ = st.propagate(member_to_bitmap(rem, p.d))
        assert status == (CT_OK if okk else CT_FAIL), k
        if okk:
            assert np.array_equal(bitmap_to_member(dom, p.d), dout), k
            assert int(np.unpackbits(st.read_table().view(np.uint8)).sum()) == nv, k
    tab.close()


@pytest.mark.parametrize("kind", ["short", "negative"])
def test_propagate_from_f4(kind):
    """ct_propagate_from_async on short and negative tables (k_fast reads the
    source, writes the output; the negative table's pending prunes travel with
    the source): a chain of calls, each from the previous output, vs the oracle."""
    import torch
    if kind == "short":
        p = short_table(4, 30, 70_001, seed=11, p_star=0.01)
    else:
        p = negative_table(3, 60, 170_000, seed=12, lo=1)
    tab = _make(p, kind, _grid_fused=True)
    assert C.KERNEL_PATHS[tab.info.kernel_path] == "k_fast"
    ok, root_m, _ = _oracle(kind, p, np.ones(p.R, np.uint8))
    assert ok
    wd = tab.Wd
    out = torch.zeros(wd, dtype=torch.int64, device="cuda")
    sd = torch.zeros(1, dtype=torch.int32, device="cuda")
    a, b = tab.root.clone(), tab.root.clone()
    src, cur = tab.root, root_m.copy()
    rng = Rng(31, lanes=1)
    done = 0
    for k in range(40):
        rem = walk_removal(rng, cur, p.d, m=1, q=0.3)
        if rem is None:
            src, cur = tab.root, root_m.copy()
            continue
        dst = a if src is not a else b
        din = cur & (1 - rem)
        okk, dout, _ = _oracle(kind, p, din)
        remd = torch.from_numpy(member_to_bitmap(rem, p.d).view(np.int64)).cuda()
        torch.cuda.synchronize()
        dst.propagate_from_async(src, remd, out, None, sd)
        dst.synchronize()
        assert int(sd.item()) == (CT_OK if okk else CT_FAIL), k
        if okk:
            assert np.array_equal(bitmap_to_member(out.cpu().numpy().view(np.uint64), p.d), dout), k
            src, cur = dst, dout
            done += 1
        else:
            src, cur = tab.root, root_m.copy()
    assert done > 10
    tab.close()
