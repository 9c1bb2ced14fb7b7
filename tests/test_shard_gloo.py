"""Multi-process (world_size 2, gloo, CPU) tests of the tuple-range sharding host
protocol: the partition the library uses (ct_shard_range), the
flag combine (all-reduce MAX over uint8 = OR on {0,1}) and the NCCL-id
bootstrap.  The per-shard flags here come from a test-side emulation of "row r
is supported by a valid tuple of my slice" on the oracle's valid-tuple vector,
so the check is: OR over shards == the oracle's global answer.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_18413_b200 import ct as C
from paper_2507_18413_b200.sharded import combine_flags_, shard_ranges, broadcast_nccl_id, exchange_handles

WORLD = 2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from workloads import random_table, Rng
        from workloads.policies import walk_removal

        results = {}
        # 1) partition: every rank computes its own range; gathered ranges tile the table
        for t in (0, 1, 63, 64, 1000, 10_000_000 + 17):
            b, w = C.ct_shard_range(t, world, rank)
            got = [None] * world
            dist.all_gather_object(got, (b, w))
            results.setdefault("ranges", []).append((t, got))
        # 2) flag combine == oracle support, over a short walk
        p = random_table(4, 9, 3000, seed=5)
        words = (p.t + 63) // 64
        b, w = C.ct_shard_range(p.t, world, rank)
        j0, j1 = min(64 * b, p.t), min(64 * (b + w), p.t)
        rb = np.concatenate([[0], np.cumsum(p.d)])
        rng = Rng(3, lanes=1)
        ok, root, _ = oracle.gac(p.lo, p.d, p.tuples, np.ones(p.R, np.uint8))
        cur = root
        checks = 0
        for k in range(60):
            rem = walk_removal(rng, cur, p.d)
            if rem is None:                       # solved: restore the root
                cur = root
                continue
            din = cur & (1 - rem)
            okg, dout, valid = oracle.gac(p.lo, p.d, p.tuples, din, want_valid=True)
            flags = torch.zeros(p.R + 1, dtype=torch.uint8)
            for j in range(j0, j1):
                if valid[j]:
                    for i in range(p.n):
                        flags[rb[i] + p.tuples[j, i] - p.lo[i]] = 1
            flags[p.R] = int(valid[j0:j1].any())
            combine_flags_(flags)
            assert bool(flags[p.R]) == okg, (rank, k)
            if okg:
                # kept values of non-singleton vars are exactly the supported ones
                exp = dout.astype(np.uint8)
                got = flags[:p.R].numpy() & din
                assert np.array_equal(got, exp), (rank, k)
                cur = dout
                checks += 1
            else:
                cur = root
        results["checks"] = checks
        # 3) NCCL unique-id bootstrap through torch.distributed
        try:
            nid = broadcast_nccl_id()
            got = [None] * world
            dist.all_gather_object(got, nid)
            results["nccl_id_same"] = all(g == got[0] for g in got) and len(got[0]) == 128
        except C.CTError as e:          # no NCCL bootstrap possible on this host
            results["nccl_id_same"] = f"skipped: {e}"
        # 4) peer-handle exchange (ct_peer_attach's input): rank order, bytes intact
        fake = bytes([rank + 1]) * C.CT_PEER_HANDLE_BYTES
        results["handles"] = exchange_handles(fake)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok", results))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, "error", traceback.format_exc()))


@pytest.mark.timeout(300)
def test_gloo_world2_shard_protocol():
    C.lib()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for pr in procs:
        pr.join(timeout=60)
    for rank, status, payload in res:
        assert status == "ok", payload
        for t, got in payload["ranges"]:
            wtot = (t + 63) // 64
            assert got[0][0] == 0
            assert sum(w for _, w in got) == wtot
            for g in range(WORLD - 1):
                assert got[g][0] + got[g][1] == got[g + 1][0]
                assert got[g + 1][0] % 16 == 0
            assert got == shard_ranges(t, WORLD)
        assert payload["checks"] > 5
        assert payload["handles"] == [bytes([g + 1]) * C.CT_PEER_HANDLE_BYTES for g in range(WORLD)]
        assert payload["nccl_id_same"] is True or str(payload["nccl_id_same"]).startswith("skipped")
