"""GPU parity of the multi-table model: the on-device Jacobi
fixpoint and the library's DFS vs the oracle (oracle.fixpoint / oracle.dfs),
bit-exact: same fixpoint domains, same FAIL verdicts, same node trace."""
import numpy as np
import pytest

import oracle
from oracle.dfs import dfs as oracle_dfs
from paper_2507_18413_b200 import CT_OK, CT_FAIL, CT_ESTATE, CTError, Model
from workloads import Rng, member_to_bitmap, bitmap_to_member, table1
from workloads.csp import csp_model

pytestmark = pytest.mark.gpu


def _model(m, **cfg):
    return Model(m["vlo"], m["vd"], m["scopes"], m["tables"], **cfg)


def test_table1_model_first_solution():
    p = table1()
    M = Model(p.lo, p.d, [np.arange(3)], [p.tuples])
    st, sol, stats = M.search(value_order=0, max_solutions=1)   # device-resident driver
    assert st == CT_OK and sol.tolist() == [3, 4, 3]          # SPEC S:L394 (derived)
    ref = oracle_dfs(p.lo, p.d, [np.arange(3)], [p.tuples], value_order=0, max_solutions=1)
    assert (stats.nodes, stats.failures, stats.trace_hash) == (ref["nodes"], ref["failures"], ref["trace_hash"])
    st, sol, stats = M.search(value_order=0, max_solutions=0)
    assert stats.solutions == 5
    M.close()


@pytest.mark.parametrize("seed", range(8))
def test_random_model_fixpoints(seed):
    """Root fixpoint and random restrictions vs oracle.fixpoint."""
    m = csp_model(8, 12, 5, 3000, seed=seed, arities=[3, 4, 2, 5, 3])
    M = _model(m)
    ok, root = oracle.fixpoint(m["vlo"], m["vd"], m["scopes"], m["tables"], np.ones(int(m["vd"].sum()), np.uint8))
    assert (M.root_status == CT_OK) == ok
    if not ok:
        M.close()
        return
    assert np.array_equal(bitmap_to_member(M.root_dom, m["vd"]), root)
    rng = Rng(100 + seed)
    for trial in range(30):
        keep = (rng.uniform(root.size, 4) > 0).astype(np.uint8)
        din = root & keep
        ok, dout = oracle.fixpoint(m["vlo"], m["vd"], m["scopes"], m["tables"], din)
        M.push()
        st, gd = M.fixpoint(member_to_bitmap(din, m["vd"]))
        assert st == (CT_OK if ok else CT_FAIL), trial
        if ok:
            assert np.array_equal(bitmap_to_member(gd, m["vd"]), dout), trial
        else:
            with pytest.raises(CTError) as e:
                M.fixpoint(None)
            assert e.value.status == CT_ESTATE
        M.pop()
    M.close()


@pytest.mark.parametrize("driver", ["device", "host"])
@pytest.mark.parametrize("seed", range(6))
def test_search_all_solutions_matches_oracle(seed, driver):
    m = csp_model(6, 5, 4, 40, seed=50 + seed, arities=[3, 3, 2, 4])
    M = _model(m)
    for vo in (0, 1):
        st, sol, stats = M.search(value_order=vo, max_solutions=0, driver=driver)
        ref = oracle_dfs(m["vlo"], m["vd"], m["scopes"], m["tables"], value_order=vo, max_solutions=0)
        assert stats.solutions == len(ref["solutions"])
        assert (stats.nodes, stats.failures) == (ref["nodes"], ref["failures"])
        assert stats.trace_hash == ref["trace_hash"]
        if ref["solutions"]:
            assert tuple(sol.tolist()) == ref["solutions"][-1]
    M.close()


def test_search_first_solution_config5_shape():
    """Config 5 shape (30 vars, d = 40, 12 tables, arity 4-8) at 2e4 tuples per
    table: the first 300 nodes' trace equals the oracle's."""
    m = csp_model(30, 40, 12, 20_000, seed=7)
    M = _model(m)
    for driver in ("device", "host"):
        st, sol, stats = M.search(value_order=0, max_nodes=300, max_solutions=1, driver=driver)
        ref = oracle_dfs(m["vlo"], m["vd"], m["scopes"], m["tables"], value_order=0, max_nodes=300, max_solutions=1)
        assert (stats.nodes, stats.failures, stats.solutions) == (ref["nodes"], ref["failures"], len(ref["solutions"]))
        assert stats.trace_hash == ref["trace_hash"]
    M.close()


@pytest.mark.parametrize("seed", range(4))
def test_device_and_host_drivers_agree(seed):
    """The device-resident DFS and the host-driven one walk the same tree:
    every counter, the trace hash and the solution agree, and the model is
    left as it was (a fixpoint after the search equals one before it)."""
    m = csp_model(10, 8, 6, 400, seed=80 + seed, arities=[3, 4, 2, 5, 3, 4])
    M = _model(m)
    if M.root_status != CT_OK:
        M.close()
        return
    root = M.root_dom.copy()
    for vo, mx_sol, mx_nodes in ((0, 0, 0), (1, 1, 0), (0, 0, 57)):
        a = M.search(value_order=vo, max_solutions=mx_sol, max_nodes=mx_nodes, driver="device")
        b = M.search(value_order=vo, max_solutions=mx_sol, max_nodes=mx_nodes, driver="host")
        assert a[0] == b[0]
        for f in ("nodes", "failures", "solutions", "table_calls", "iterations", "max_depth", "trace_hash"):
            assert getattr(a[2], f) == getattr(b[2], f), f
        if a[1] is not None:
            assert np.array_equal(a[1], b[1])
        M.push()
        st, gd = M.fixpoint(None)
        assert st == CT_OK and np.array_equal(gd, root)
        M.pop()
    M.close()


def test_device_search_falls_back_when_the_trail_is_short():
    """A trail shorter than the search depth (ct_config.search_levels) makes
    the device driver stop and the host driver rerun the search: same results
    as a plain host-driven search."""
    m = csp_model(6, 5, 4, 40, seed=51, arities=[3, 3, 2, 4])
    M = _model(m, search_levels=3)
    a = M.search(value_order=0, max_solutions=0, driver="device")
    b = M.search(value_order=0, max_solutions=0, driver="host")
    ref = oracle_dfs(m["vlo"], m["vd"], m["scopes"], m["tables"], value_order=0, max_solutions=0)
    assert b[2].max_depth > 2                      # the trail was too short for this tree
    for f in ("nodes", "failures", "solutions", "trace_hash"):
        assert getattr(a[2], f) == getattr(b[2], f), f
    assert a[2].trace_hash == ref["trace_hash"]
    M.close()


@pytest.mark.parametrize("grid", [1, 3])
def test_model_grid_smaller_than_table_count(grid):
    """Model kernels on fewer CTAs than tables (ct_config.grid_override): one
    CTA ingests / finalizes several tables, so its barrier arrival carries
    several tables' verdicts.  Fixpoints and the DFS trace vs the oracle."""
    m = csp_model(10, 8, 6, 400, seed=91, arities=[3, 4, 2, 5, 3, 4])
    M = _model(m, grid_override=grid)
    ok, root = oracle.fixpoint(m["vlo"], m["vd"], m["scopes"], m["tables"], np.ones(int(m["vd"].sum()), np.uint8))
    assert (M.root_status == CT_OK) == ok
    if ok:
        rng = Rng(7)
        for trial in range(10):
            din = root & (rng.uniform(root.size, 3) > 0).astype(np.uint8)
            ok2, dout = oracle.fixpoint(m["vlo"], m["vd"], m["scopes"], m["tables"], din)
            M.push()
            st, gd = M.fixpoint(member_to_bitmap(din, m["vd"]))
            assert st == (CT_OK if ok2 else CT_FAIL), trial
            if ok2:
                assert np.array_equal(bitmap_to_member(gd, m["vd"]), dout), trial
            M.pop()
        for driver in ("device", "host"):
            st, sol, stats = M.search(value_order=0, max_solutions=0, driver=driver)
            ref = oracle_dfs(m["vlo"], m["vd"], m["scopes"], m["tables"], value_order=0, max_solutions=0)
            assert (stats.nodes, stats.failures, stats.solutions) == (ref["nodes"], ref["failures"],
                                                                      len(ref["solutions"]))
            assert stats.trace_hash == ref["trace_hash"]
    M.close()


@pytest.mark.parametrize("seed", range(3))
def test_private_variables_fixpoint_and_search(seed):
    """Most variables constrained by one table only (8 variables, scopes of
    3 + 3 + 2, i.e. independent tables): removals on such a variable do not
    count as a shared-domain change (the fixpoint may stop a round earlier);
    domains and the first 1500 DFS nodes' trace still equal the oracle's (the
    full tree has ~1e5 solutions)."""
    m = csp_model(8, 6, 3, 120, seed=300 + seed, arities=[3, 3, 2])
    M = _model(m)
    ok, root = oracle.fixpoint(m["vlo"], m["vd"], m["scopes"], m["tables"], np.ones(int(m["vd"].sum()), np.uint8))
    assert (M.root_status == CT_OK) == ok
    if ok:
        assert np.array_equal(bitmap_to_member(M.root_dom, m["vd"]), root)
        for vo in (0, 1):
            st, sol, stats = M.search(value_order=vo, max_solutions=0, max_nodes=1500, driver="device")
            ref = oracle_dfs(m["vlo"], m["vd"], m["scopes"], m["tables"], value_order=vo, max_solutions=0,
                             max_nodes=1500)
            assert (stats.nodes, stats.failures, stats.solutions) == (ref["nodes"], ref["failures"],
                                                                      len(ref["solutions"]))
            assert stats.trace_hash == ref["trace_hash"]
    M.close()


def test_device_search_repeated_same_trace():
    """Regression: the device-resident DFS once let a CTA restore the state pool
    (after a solution) while slower CTAs were still reading the shared domains,
    splitting the grid's control flow (a hang about once per ~300 searches;
    tools/hang_probe.py runs thousands).  12 all-solution searches: every trace
    equals the host driver's (a split now trips the spin watchdog: CT_ECUDA,
    not a hang)."""
    m = csp_model(10, 8, 6, 400, seed=81, arities=[3, 4, 2, 5, 3, 4])
    M = _model(m)
    if M.root_status != CT_OK:
        M.close()
        return
    ref = M.search(value_order=0, max_solutions=0, driver="host")[2]
    for i in range(12):
        s = M.search(value_order=i % 2, max_solutions=0, driver="device")[2]
        if i % 2 == 0:
            assert (s.nodes, s.failures, s.solutions, s.trace_hash) == \
                (ref.nodes, ref.failures, ref.solutions, ref.trace_hash), i
    M.close()
