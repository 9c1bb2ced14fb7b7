"""Object wrappers over the C names in ct.py (lifetime management only).

    tab = Table(lo, d, tuples)                  # ct_create: supports + root GAC on cuda:device
    st = tab.root.clone()                       # ct_state_clone
    status, dom, pruned = st.propagate(removed) # ct_propagate (host numpy uint64[Wd])
    st.copy_from(tab.root)                      # ct_state_copy (backtrack / restore)
    b = tab.batch(4096)                         # ct_batch_create
    status, doms = b.propagate(removed_SxWd)    # ct_propagate_many

Device memory comes from PyTorch's caching allocator and work is ordered on a
torch.cuda.Stream owned by the table (pass `stream=` to share one).
"""
from __future__ import annotations

import ctypes
import weakref

import numpy as np

from . import ct as C


class Table:
    def __init__(self, lo, d, tuples, init_dom=None, scope=None, device: int = 0, stream=None,
                 torch_alloc: bool = True, n_shards: int = 1, shard_rank: int = 0, nccl_unique_id=None,
                 update_policy: int = C.CT_POLICY_AUTO, use_residues: bool = True, use_index: bool = True,
                 use_graph: bool = True, use_fused: bool = True, kind: str | int = "positive",
                 use_gather: bool = True, launch_shape: int | str = 0, grid_override: int = 0,
                 batch_per_state: bool = False, batch_cells: bool = True):
        """kind: "positive" (ct_create), "short" (cells == CT_STAR match any value)
        or "negative" (the tuples are the forbidden assignments) -- include/ct.h f4."""
        import torch
        self.device = int(device)
        if stream is None:
            self.torch_stream = torch.cuda.Stream(device=self.device)
            stream_ptr = self.torch_stream.cuda_stream
        else:
            self.torch_stream = stream if hasattr(stream, "cuda_stream") else None
            stream_ptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        self.allocator = C.TorchAllocator(self.device) if torch_alloc else None
        cfg, self._keep = C.make_config(self.device, stream_ptr, self.allocator, n_shards, shard_rank,
                                        nccl_unique_id, update_policy, use_residues, use_index, use_graph,
                                        use_fused, use_gather, launch_shape, grid_override, batch_per_state,
                                        batch_cells=batch_cells)
        self.lo = np.ascontiguousarray(lo, np.int32)
        self.d = np.ascontiguousarray(d, np.int32)
        self.kind = C.TABLE_KINDS[kind] if isinstance(kind, str) else int(kind)
        status, handle, root, dom = C.ct_create(self.lo, self.d, tuples, init_dom, scope, cfg, kind=self.kind)
        self.handle = handle
        self._states = weakref.WeakSet()
        self._batches = weakref.WeakSet()
        self.info = C.ct_table_info_get(handle)
        self.Wd = int(self.info.dom_words)
        self.root_status = status
        self.root_dom = dom
        self.root = State(self, root)

    @property
    def stream_ptr(self) -> int:
        return C.ct_state_stream(self.root.handle)

    def batch(self, n_states: int, init: "State | None" = None) -> "Batch":
        return Batch(self, n_states, init or self.root)

    def close(self):
        if getattr(self, "handle", None):
            for b in list(self._batches):
                b.close()
            for s in list(self._states):
                s.close()
            C.ct_table_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class State:
    def __init__(self, table: Table, handle):
        self.table = table
        self.handle = handle
        table._states.add(self)

    def clone(self) -> "State":
        return State(self.table, C.ct_state_clone(self.handle))

    def copy_from(self, src: "State") -> None:
        C.ct_state_copy(self.handle, src.handle)

    def serve(self, on: bool = True) -> None:
        """Synchronous calls served by a persistent kernel (ct_state_serve)."""
        C.ct_state_serve(self.handle, on)

    def propagate(self, removed=None, out=None, pruned=None):
        """Synchronous host call.  Returns (status, dom, pruned); dom/pruned are
        None unless status == CT_OK.  out / pruned: optional preallocated
        uint64[Wd] host arrays (reused across calls by latency-sensitive callers)."""
        wd = self.table.Wd
        if out is None:
            out = np.zeros(max(wd, 1), np.uint64)
        if pruned is None:
            pruned = np.zeros(max(wd, 1), np.uint64)
        rem = None if removed is None else np.ascontiguousarray(removed, np.uint64).reshape(-1)
        st = C.ct_propagate(self.handle, rem, out, pruned, wd=wd)
        return (st, out[:wd], pruned[:wd]) if st == C.CT_OK else (st, None, None)

    def propagate_from_async(self, src: "State", removed, out_dom=None, out_pruned=None, out_status=None):
        """This state := `src` propagated with `removed` (ct_propagate_from_async)."""
        C.ct_propagate_from_async(self.handle, src.handle, removed, out_dom, out_pruned, out_status,
                                  wd=self.table.Wd)

    def propagate_async(self, removed, out_dom=None, out_pruned=None, out_status=None):
        C.ct_propagate_async(self.handle, removed, out_dom, out_pruned, out_status, wd=self.table.Wd)

    def read_table(self) -> np.ndarray:
        return C.ct_state_read_table(self.handle, int(self.table.info.words))

    def read_dom(self) -> np.ndarray:
        return C.ct_state_read_dom(self.handle, self.table.Wd)

    def stats(self):
        return C.ct_state_stats(self.handle)

    def synchronize(self):
        C.ct_synchronize(self.handle)

    def close(self):
        if getattr(self, "handle", None) and self.table.handle:
            C.ct_state_destroy(self.handle)
        self.handle = None


class Batch:
    def __init__(self, table: Table, n_states: int, init: State):
        self.table = table
        self.S = int(n_states)
        self.handle = C.ct_batch_create(table.handle, self.S, init.handle)
        table._batches.add(self)

    def copy(self, index: int, src: State):
        C.ct_batch_copy(self.handle, index, src.handle)

    def copy_all(self, src: State):
        C.ct_batch_copy_all(self.handle, src.handle)

    def restore_dead(self, src: State):
        C.ct_batch_restore_dead(self.handle, src.handle)

    def stats(self):
        return C.ct_batch_stats(self.handle, self.S)

    def work(self, reset: bool = False) -> dict:
        return C.ct_batch_work(self.handle, reset)

    def read_table(self, index: int) -> np.ndarray:
        return C.ct_batch_read_table(self.handle, index, int(self.table.info.words))

    def propagate(self, removed=None):
        wd = self.table.Wd
        out = np.zeros((self.S, max(wd, 1)), np.uint64)
        status = np.zeros(self.S, np.int32)
        rem = None if removed is None else np.ascontiguousarray(removed, np.uint64).reshape(self.S, wd)
        C.ct_propagate_many(self.handle, rem, out, status)
        return status, out[:, :wd]

    def propagate_async(self, removed, out_dom=None, out_status=None):
        C.ct_propagate_many_async(self.handle, removed, out_dom, out_status)

    def close(self):
        if getattr(self, "handle", None) and self.table.handle:
            C.ct_batch_destroy(self.handle)
        self.handle = None


class Model:
    """Several table constraints over shared variables (ct_model_*): on-device
    Jacobi fixpoint per call, DFS search in the library."""

    def __init__(self, var_lo, var_size, scopes, tables, device: int = 0, **cfg_kw):
        self.var_lo = np.ascontiguousarray(var_lo, np.int32)
        self.var_size = np.ascontiguousarray(var_size, np.int32)
        cfg, self._keep = C.make_config(device, None, None, **cfg_kw)
        self.root_status, self.handle, self.root_dom = C.ct_model_create(self.var_lo, self.var_size, scopes,
                                                                         tables, cfg)
        self.Wg = C.ct_model_dom_words(self.handle)

    def fixpoint(self, dom_in=None):
        out = np.zeros(max(self.Wg, 1), np.uint64)
        din = None if dom_in is None else np.ascontiguousarray(dom_in, np.uint64)
        st = C.ct_model_fixpoint(self.handle, din, out)
        return st, (out[:self.Wg] if st == C.CT_OK else None)

    def push(self):
        C.ct_model_push(self.handle)

    def pop(self):
        C.ct_model_pop(self.handle)

    def search(self, value_order: int = 0, max_nodes: int = 0, max_solutions: int = 1, driver=None):
        """driver: None (library default: device-resident DFS), "device" or "host"."""
        d = {None: None, "device": 0, "host": 1}[driver]
        return C.ct_model_search(self.handle, int(self.var_size.size), value_order, max_nodes, max_solutions, d)

    def close(self):
        if getattr(self, "handle", None):
            C.ct_model_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostTable:
    """The paper's serial CT and its GPU-offloaded derivatives (placement
    ablation; include/ct.h ct_host_*): placement "host" (serial CT),
    "u" (CT^u), "f" (CT^f) or "uf" (CT^uf).  Same call semantics as Table."""

    def __init__(self, lo, d, tuples, placement: str = "host", init_dom=None, device: int = 0,
                 update_policy: int = C.CT_POLICY_AUTO):
        self.placement = placement
        cfg = None
        if placement != "host":
            cfg, _ = C.make_config(device, None, None, update_policy=update_policy)
        else:
            cfg = C.ct_config()
            C.lib().ct_config_init(ctypes.byref(cfg))
            cfg.update_policy = update_policy
        self.root_status, self.handle, self._root, self.root_dom = C.ct_host_create(
            lo, d, tuples, C.PLACEMENTS[placement], init_dom=init_dom, cfg=cfg)
        self.Wd = int(C.lib().ct_host_dom_words(self.handle))
        self._states = [self._root]
        self.root = HostState(self, self._root)

    def stats(self, reset: bool = False) -> dict:
        return C.ct_host_stats(self.handle, reset)

    def close(self):
        if getattr(self, "handle", None):
            for h in self._states:
                C.ct_host_state_destroy(h)
            self._states = []
            C.ct_host_table_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class HostState:
    def __init__(self, table: HostTable, handle):
        self.table = table
        self.handle = handle

    def clone(self) -> "HostState":
        h = C.ct_host_clone(self.handle)
        self.table._states.append(h)
        return HostState(self.table, h)

    def copy_from(self, src: "HostState") -> None:
        C.ct_host_copy(self.handle, src.handle)

    def propagate(self, removed=None, out=None, pruned=None):
        wd = self.table.Wd
        if out is None:
            out = np.zeros(max(wd, 1), np.uint64)
        if pruned is None:
            pruned = np.zeros(max(wd, 1), np.uint64)
        rem = None if removed is None else np.ascontiguousarray(removed, np.uint64).reshape(-1)
        if rem is not None and rem.size < wd:
            raise ValueError(f"removed needs {wd} words")
        st = C.ct_host_propagate(self.handle, rem, out, pruned)
        return (st, out[:wd], pruned[:wd]) if st == C.CT_OK else (st, None, None)
