"""Tuple-range sharding driven by the LIBRARY's own flags across processes
(SURVEY §8(a) a10, §8(e)): world_size 2, one process per shard, both on cuda:0
(the lease has one GPU; NCCL refuses two ranks on one device, so the combine is
a gloo all-reduce MAX of the flags the library wrote -- ShardedTable
mode="torch", ct_propagate_local_async / ct_state_flags / ct_propagate_apply_async).
Tables are chosen so that shards disagree: rows sorted by x0 (a value of x0 is
supported in one shard only), and a table so small that shard 0 owns no tuple.
Every call of a policy-P(2, 0.5) walk is compared with the oracle on both ranks.
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem(kind):
    from workloads import random_table
    from workloads.tables import Problem
    if kind == "sorted":
        p = random_table(5, 16, 40_000 + 5, seed=31)
        order = np.argsort(p.tuples[:, 0], kind="stable")
        return Problem("sorted_by_x0", p.lo, p.d, np.ascontiguousarray(p.tuples[order]), 31)
    if kind == "tiny":        # ct_shard_range(1000, 2, 0) owns 0 words
        return random_table(3, 6, 1000, seed=32)
    if kind == "fast":        # > 8192 blocks per shard: the cooperative k_fast shape on each rank
        p = random_table(4, 12, 2_600_000 + 3, seed=33)
        order = np.argsort(p.tuples[:, 1], kind="stable")
        return Problem("fast_sorted_by_x1", p.lo, p.d, np.ascontiguousarray(p.tuples[order]), 33)
    raise KeyError(kind)


def _worker(rank, world, port, kind, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2507_18413_b200 import CT_OK, CT_FAIL
        from paper_2507_18413_b200.sharded import ShardedTable
        from workloads import Rng, member_to_bitmap, bitmap_to_member
        from workloads.policies import walk_removal

        p = _problem(kind)
        sh = ShardedTable(p.lo, p.d, p.tuples, mode="torch", device=0)
        ok0, root_o, _ = oracle.gac(p.lo, p.d, p.tuples, np.ones(p.R, np.uint8))
        assert (sh.root_status == CT_OK) == ok0, (rank, sh.root_status)
        if ok0:
            assert np.array_equal(bitmap_to_member(sh.root_dom, p.d), root_o), rank
        st = sh.root.clone()
        rng = Rng(9, lanes=1)
        cur = root_o.copy()
        checked = fails = 0
        for k in range(80):
            r = walk_removal(rng, cur, p.d)
            if r is None:
                st.copy_from(sh.root)
                cur = root_o.copy()
                continue
            din = cur & (1 - r)
            ok, dout, _ = oracle.gac(p.lo, p.d, p.tuples, din)
            status, dom, pr = sh.propagate(st, member_to_bitmap(r, p.d))
            assert status == (CT_OK if ok else CT_FAIL), (rank, k)
            if ok:
                assert np.array_equal(bitmap_to_member(dom, p.d), dout), (rank, k)
                assert np.array_equal(bitmap_to_member(pr, p.d), din & (1 - dout)), (rank, k)
                cur = dout
            else:
                fails += 1
                st.copy_from(sh.root)
                cur = root_o.copy()
            checked += 1
        info = sh.table.info
        st.close()
        sh.close()
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", dict(checked=checked, fails=fails, words=int(info.words))))
    except Exception:
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.timeout(600)
@pytest.mark.parametrize("kind", ["sorted", "tiny", "fast"])
def test_two_process_library_flags(kind):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, kind, q)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=540) for _ in range(WORLD)]
    for pr in procs:
        pr.join(timeout=60)
    words = {}
    for rank, status, payload in res:
        assert status == "ok", payload
        assert payload["checked"] >= 40
        words[rank] = payload["words"]
    if kind == "tiny":
        assert words[0] == 0 and words[1] == 16
