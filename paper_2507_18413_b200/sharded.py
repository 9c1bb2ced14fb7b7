"""Tuple-range sharding across GPUs: one process per
GPU, torch.distributed for the plumbing.

Every rank holds words [b_g, b_{g+1}) of currTable and of every support row
(ct_shard_range).  Per call each rank runs ingest/update/filter on its slice,
producing R+1 flag bytes (per support row "supported by a valid tuple in my
slice", plus "my slice is non-empty"); the flags are OR-combined across ranks
(all-reduce MAX over uint8 -- NCCL has no bitwise-or op, and MAX is OR on {0,1})
and every rank then applies the same domain update, so the states stay
bit-identical with no further traffic.  FAIL <=> the combined non-empty byte is 0.

Three combine modes:
  * "peer": the k_fast finalizer of every rank exchanges the flags with the
    others through NVLink peer memory and ORs them itself (ct_peer_export /
    ct_peer_attach; the IPC handles travel through torch.distributed), so a
    sharded call is ONE kernel; the root propagation (at create) uses NCCL;
  * "nccl" (default): the library owns an NCCL communicator (unique id broadcast
    through torch.distributed) and issues the all-reduce itself, on the table's
    stream, between the filter and finalize kernels -- one graph-capturable call;
  * "torch": the library stops after the local phase and the all-reduce is a
    torch.distributed collective on a zero-copy tensor view of the flags
    (works with any backend; used by the gloo/CPU tests of the host protocol).
"""
from __future__ import annotations

import numpy as np

from . import ct as C
from .api import Table


class _DevBytes:
    """Zero-copy __cuda_array_interface__ view of library-owned device bytes."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False), "version": 2}


def flags_tensor(state_handle):
    """torch.uint8 CUDA tensor aliasing the state's R+1 shard-flag bytes."""
    import torch
    ptr, n = C.ct_state_flags(state_handle)
    return torch.as_tensor(_DevBytes(ptr, n), device="cuda")


def shard_ranges(n_tuples: int, n_shards: int):
    return [C.ct_shard_range(n_tuples, n_shards, g) for g in range(n_shards)]


def broadcast_nccl_id(group=None) -> bytes:
    import torch.distributed as dist
    obj = [C.ct_nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def exchange_handles(handle: bytes, group=None) -> list:
    """Every rank's peer handle, in rank order (all_gather_object: any backend)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, bytes(handle), group=group)
    return out


def attach_peers(table_handle, group=None) -> None:
    """Collective: export this rank's inbox, gather every rank's, attach."""
    C.ct_peer_attach(table_handle, exchange_handles(C.ct_peer_export(table_handle), group))


def combine_flags_(flags, group=None):
    """In-place OR of shard flags across ranks (all-reduce MAX on uint8)."""
    import torch.distributed as dist
    if flags.device.type == "cuda" and dist.get_backend(group) != "nccl":
        # host-side collectives (gloo): stage through host memory
        h = flags.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        flags.copy_(h)
    else:
        dist.all_reduce(flags, op=dist.ReduceOp.MAX, group=group)
    return flags


def apply_async(state_handle, wd: int, device: int):
    """ct_propagate_apply_async into fresh device buffers; returns (status, dom, pruned) tensors."""
    import torch
    dev = torch.device("cuda", device)
    out = torch.zeros(max(wd, 1), dtype=torch.int64, device=dev)
    pr = torch.zeros(max(wd, 1), dtype=torch.int64, device=dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    C.ct_propagate_apply_async(state_handle, out, pr, status)
    return status, out, pr


def finish_pending_root(table: Table, combine) -> None:
    """Caller-combined shards: ct_create returned CT_PENDING after the root's
    local phase (include/ct.h).  `combine(flags_tensor)` ORs the root's flags
    across the shards in place; the apply then gives the root verdict/domains."""
    import torch
    if table.root_status != C.CT_PENDING:
        return
    h = table.root.handle
    stream = torch.cuda.ExternalStream(C.ct_state_stream(h), device=torch.device("cuda", table.device))
    stream.synchronize()
    combine(flags_tensor(h))
    torch.cuda.synchronize(table.device)
    status, out, _ = apply_async(h, table.Wd, table.device)
    stream.synchronize()
    st = int(status.item())
    if st < 0:
        raise C.CTError(st, "sharded root apply")
    table.root_status = st
    table.root_dom = out[:table.Wd].cpu().numpy().view(np.uint64).copy() if st == C.CT_OK else None


class ShardedTable:
    def __init__(self, lo, d, tuples, group=None, device: int | None = None, mode: str = "nccl", **kw):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.mode = mode
        dev = torch.cuda.current_device() if device is None else int(device)
        if mode not in ("nccl", "torch", "peer"):
            raise ValueError(f"unknown combine mode {mode!r}")
        nid = broadcast_nccl_id(group) if mode in ("nccl", "peer") else None
        self.table = Table(lo, d, tuples, device=dev, n_shards=self.world, shard_rank=self.rank,
                           nccl_unique_id=nid, **kw)
        if mode == "torch":
            finish_pending_root(self.table, lambda f: combine_flags_(f, self.group))
        if mode == "peer":
            attach_peers(self.table.handle, self.group)
        self.root = self.table.root
        self.root_status = self.table.root_status
        self.root_dom = self.table.root_dom
        self.Wd = self.table.Wd

    def propagate(self, state, removed=None):
        """Synchronous host call on every rank with identical `removed`."""
        if self.mode in ("nccl", "peer"):
            return state.propagate(removed)
        import torch
        wd = self.Wd
        dev = torch.device("cuda", self.table.device)
        rem = torch.zeros(max(wd, 1), dtype=torch.int64, device=dev)
        if removed is not None and wd:
            rem[:wd] = torch.from_numpy(np.ascontiguousarray(removed, np.uint64).view(np.int64))
        stream = torch.cuda.ExternalStream(C.ct_state_stream(state.handle), device=dev)
        torch.cuda.current_stream(dev).synchronize()
        C.ct_propagate_local_async(state.handle, rem)
        with torch.cuda.stream(stream):
            combine_flags_(flags_tensor(state.handle), self.group)
            status, out, pr = apply_async(state.handle, wd, self.table.device)
        stream.synchronize()
        st = int(status.item())
        if st < 0:
            raise C.CTError(st, "sharded propagate")
        if st != C.CT_OK:
            return st, None, None
        return st, out[:wd].cpu().numpy().view(np.uint64), pr[:wd].cpu().numpy().view(np.uint64)

    def close(self):
        self.table.close()
