"""Thin ctypes binding of include/ct.h (libct_b200.so).

Same names as the C ABI; argument marshalling only -- every step of the
propagation runs in the library's CUDA kernels.  Host buffers are numpy arrays,
device buffers are torch CUDA tensors (their data_ptr()).  PyTorch supplies the
device memory (caching-allocator hooks passed as ct_allocator), the CUDA
stream, and -- for tuple-range sharding -- torch.distributed for broadcasting
the NCCL unique id.

There is no fallback: if the CUDA library is missing or fails to load, every
entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CT_LIB_PATH") or os.path.join(_PKG, "libct_b200.so")   # override: experiment builds

CT_OK, CT_FAIL, CT_EINVAL, CT_ENOMEM, CT_ECUDA, CT_ENCCL, CT_ESTATE = 0, 1, -1, -2, -3, -4, -5
CT_PENDING = 2   # ct_create of a caller-combined shard: combine the root's flags, then apply
CT_POLICY_AUTO, CT_POLICY_DOM, CT_POLICY_DELTA = 0, 1, 2
CT_TABLE_POSITIVE, CT_TABLE_SHORT, CT_TABLE_NEGATIVE = 0, 1, 2   # f4 (include/ct.h)
TABLE_KINDS = {"positive": CT_TABLE_POSITIVE, "short": CT_TABLE_SHORT, "negative": CT_TABLE_NEGATIVE}
CT_STAR = -2147483648   # short-table wildcard cell (INT32_MIN)
STATUS_NAMES = {0: "OK", 1: "FAIL", 2: "PENDING", -1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ENCCL", -5: "ESTATE"}


class CTError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)


class ct_allocator(ctypes.Structure):
    _fields_ = [("alloc", _ALLOC_FN), ("free", _FREE_FN), ("ctx", ctypes.c_void_p)]


class ct_config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("stream", ctypes.c_void_p),
                ("alloc", ctypes.POINTER(ct_allocator)),
                ("n_shards", ctypes.c_int32), ("shard_rank", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p),
                ("update_policy", ctypes.c_int32), ("use_residues", ctypes.c_int32),
                ("use_index", ctypes.c_int32), ("use_graph", ctypes.c_int32),
                ("use_fused", ctypes.c_int32), ("use_gather", ctypes.c_int32),
                ("launch_shape", ctypes.c_int32), ("grid_override", ctypes.c_int32),
                ("batch_per_state", ctypes.c_int32), ("search_levels", ctypes.c_int32),
                ("batch_cells", ctypes.c_int32)]

CT_SHAPE_AUTO, CT_SHAPE_PHASES, CT_SHAPE_FUSED, CT_SHAPE_FAST, CT_SHAPE_SMALL, CT_SHAPE_WIDE = 0, 1, 2, 3, 4, 5
SHAPES = {"auto": 0, "phases": 1, "fused": 2, "fast": 3, "small": 4, "wide": 5}


class ct_table_info(ctypes.Structure):
    _fields_ = [("n_vars", ctypes.c_int32), ("n_rows", ctypes.c_int32), ("dom_words", ctypes.c_int32),
                ("n_shards", ctypes.c_int32), ("shard_rank", ctypes.c_int32),
                ("n_tuples", ctypes.c_int64), ("words_total", ctypes.c_int64),
                ("word_begin", ctypes.c_int64), ("words", ctypes.c_int64),
                ("row_stride_words", ctypes.c_int64), ("device_bytes", ctypes.c_int64),
                ("state_bytes", ctypes.c_int64), ("kernel_path", ctypes.c_int32), ("grid", ctypes.c_int32),
                ("batch_tile", ctypes.c_int32), ("gather_cell_bits", ctypes.c_int32), ("kind", ctypes.c_int32),
                ("batch_cells", ctypes.c_int32)]

KERNEL_PATHS = {0: "per-phase", 1: "k_fused", 2: "k_fast", 3: "k_small", 4: "k_wide", 5: "negative"}


class ct_stats(ctypes.Structure):
    _fields_ = [("calls", ctypes.c_int64), ("last_status", ctypes.c_int32), ("noop", ctypes.c_int32),
                ("n_changed", ctypes.c_int32), ("n_update_rows", ctypes.c_int32),
                ("n_filter_items", ctypes.c_int32), ("n_residue_miss", ctypes.c_int32),
                ("words_in", ctypes.c_int64), ("words_out", ctypes.c_int64),
                ("update_support_words", ctypes.c_int64), ("update_table_writes", ctypes.c_int64),
                ("filter_support_words", ctypes.c_int64), ("phase_ns", ctypes.c_int64 * 7),
                ("filter_gathered_tuples", ctypes.c_int64)]


class ct_search_stats(ctypes.Structure):
    _fields_ = [("nodes", ctypes.c_int64), ("failures", ctypes.c_int64), ("solutions", ctypes.c_int64),
                ("table_calls", ctypes.c_int64), ("iterations", ctypes.c_int64), ("max_depth", ctypes.c_int64),
                ("device_ms", ctypes.c_double), ("trace_hash", ctypes.c_uint64)]


class ct_kernel_times(ctypes.Structure):
    _fields_ = [("launches", ctypes.c_int64 * 8), ("ms", ctypes.c_double * 8)]


class ct_place_stats(ctypes.Structure):
    _fields_ = [("calls", ctypes.c_int64), ("noops", ctypes.c_int64), ("kernel_launches", ctypes.c_int64),
                ("h2d_bytes", ctypes.c_int64), ("d2h_bytes", ctypes.c_int64),
                ("host_ms", ctypes.c_double), ("h2d_ms", ctypes.c_double), ("kernel_ms", ctypes.c_double),
                ("d2h_ms", ctypes.c_double)]


CT_PLACE_HOST, CT_PLACE_U, CT_PLACE_F, CT_PLACE_UF = 0, 1, 2, 3
PLACEMENTS = {"host": CT_PLACE_HOST, "u": CT_PLACE_U, "f": CT_PLACE_F, "uf": CT_PLACE_UF}

KERNEL_SLOTS = ("ingest", "update", "probe", "scan", "combine", "finalize", "fused", "small")


# exported symbol -> (restype, argtypes); the CPU test checks the .so exports all of them
P = ctypes.c_void_p
I32, I64 = ctypes.c_int32, ctypes.c_int64
SIGNATURES = {
    "ct_config_init": (None, [P]),
    "ct_create": (I32, [I32, P, P, P, P, I64, P, P, P, P, P]),
    "ct_create_table": (I32, [I32, I32, P, P, P, P, I64, P, P, P, P, P]),
    "ct_debug_diag_attach": (I32, [I32]),
    "ct_debug_diag_read": (I64, [P, I64]),
    "ct_debug_spin_limit": (I32, [I32, ctypes.c_double]),
    "ct_table_info_get": (I32, [P, P]),
    "ct_dom_words": (I32, [P]),
    "ct_dom_word_offset": (I32, [P, I32]),
    "ct_propagate": (I32, [P, P, P, P]),
    "ct_propagate_async": (I32, [P, P, P, P, P]),
    "ct_propagate_local_async": (I32, [P, P]),
    "ct_propagate_from_async": (I32, [P, P, P, P, P, P]),
    "ct_state_flags": (I32, [P, P, P]),
    "ct_propagate_apply_async": (I32, [P, P, P, P]),
    "ct_state_clone": (I32, [P, P]),
    "ct_state_copy": (I32, [P, P]),
    "ct_state_set_stream": (I32, [P, P]),
    "ct_state_stream": (P, [P]),
    "ct_synchronize": (I32, [P]),
    "ct_state_destroy": (None, [P]),
    "ct_table_destroy": (None, [P]),
    "ct_batch_create": (I32, [P, I32, P, P]),
    "ct_batch_size": (I32, [P]),
    "ct_batch_copy": (I32, [P, I32, P]),
    "ct_batch_copy_all": (I32, [P, P]),
    "ct_batch_restore_dead": (I32, [P, P]),
    "ct_propagate_many": (I32, [P, P, P, P]),
    "ct_propagate_many_async": (I32, [P, P, P, P]),
    "ct_batch_destroy": (None, [P]),
    "ct_state_read_table": (I32, [P, P]),
    "ct_table_read_supports": (I32, [P, I32, P]),
    "ct_state_read_dom": (I32, [P, P]),
    "ct_state_stats": (I32, [P, P]),
    "ct_batch_stats": (I32, [P, P]),
    "ct_batch_read_table": (I32, [P, I32, P]),
    "ct_batch_work": (I32, [P, P, I32]),
    "ct_nccl_unique_id": (I32, [P]),
    "ct_peer_export": (I32, [P, P]),
    "ct_state_serve": (I32, [P, I32]),
    "ct_debug_serve_idle": (I32, [I64]),
    "ct_debug_serve_trace": (I32, [P, P]),
    "ct_peer_attach": (I32, [P, I32, P]),
    "ct_shard_range": (I32, [I64, I32, I32, P, P]),
    "ct_table_profile": (I32, [P, I32]),
    "ct_table_profile_read": (I32, [P, P, I32]),
    "ct_model_create": (I32, [I32, P, P, I32, P, P, P, P, P, P, P]),
    "ct_model_dom_words": (I32, [P]),
    "ct_model_dom_word_offset": (I32, [P, I32]),
    "ct_model_fixpoint": (I32, [P, P, P]),
    "ct_model_push": (I32, [P]),
    "ct_model_pop": (I32, [P]),
    "ct_model_search": (I32, [P, I32, I64, I64, P, P]),
    "ct_model_search_ex": (I32, [P, I32, I64, I64, I32, P, P]),
    "ct_model_search_phases": (I32, [P, P]),
    "ct_model_destroy": (None, [P]),
    "ct_host_create": (I32, [I32, P, P, P, I64, P, I32, P, P, P, P]),
    "ct_host_propagate": (I32, [P, P, P, P]),
    "ct_host_clone": (I32, [P, P]),
    "ct_host_copy": (I32, [P, P]),
    "ct_host_dom_words": (I32, [P]),
    "ct_host_stats": (I32, [P, P, I32]),
    "ct_host_state_destroy": (None, [P]),
    "ct_host_table_destroy": (None, [P]),
    "ct_last_error": (ctypes.c_char_p, []),
    "ct_version": (ctypes.c_char_p, []),
}

_lib = None
_lock = threading.Lock()


def lib():
    """Load libct_b200.so (raises if it is missing -- build it with
    `python -m paper_2507_18413_b200.build` or __graft_entry__.build())."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"CUDA library {LIB_PATH} not built; run `python -m paper_2507_18413_b200.build`")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib


def ct_last_error() -> str:
    return lib().ct_last_error().decode(errors="replace")


def ct_version() -> str:
    return lib().ct_version().decode()


def _check(status: int, allow_fail: bool = True) -> int:
    if status < 0 or (status == CT_FAIL and not allow_fail):
        raise CTError(status, ct_last_error())
    return status


def _np_ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _dev_ptr(t):
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        # device memory, or pinned host memory (device-accessible under unified
        # addressing: the kernels read / write it in place, zero-copy)
        if not (t.is_cuda or t.is_pinned()) or not t.is_contiguous():
            raise ValueError("device buffers must be contiguous CUDA tensors or pinned host tensors")
        return ctypes.c_void_p(t.data_ptr())
    return ctypes.c_void_p(int(t))


# ---------------------------------------------------------------- torch plumbing
class TorchAllocator:
    """ct_allocator backed by PyTorch's CUDA caching allocator."""

    def __init__(self, device: int):
        import torch
        self.device = device
        self._live = {}

        def _alloc(nbytes, stream, ctx):
            try:
                p = torch.cuda.caching_allocator_alloc(int(nbytes), device=self.device, stream=int(stream or 0))
                self._live[p] = nbytes
                return p
            except Exception:
                return None

        def _free(ptr, nbytes, stream, ctx):
            if ptr in self._live:
                del self._live[ptr]
                torch.cuda.caching_allocator_delete(ptr)

        self._alloc_fn = _ALLOC_FN(_alloc)
        self._free_fn = _FREE_FN(_free)
        self.struct = ct_allocator(self._alloc_fn, self._free_fn, None)


def make_config(device: int = 0, stream=None, allocator=None, n_shards: int = 1, shard_rank: int = 0,
                nccl_unique_id: bytes | None = None, update_policy: int = CT_POLICY_AUTO,
                use_residues: bool = True, use_index: bool = True, use_graph: bool = True,
                use_fused: bool = True, use_gather: bool = True, launch_shape: int | str = 0,
                grid_override: int = 0, batch_per_state: bool = False, search_levels: int = 0,
                batch_cells: bool = True):
    cfg = ct_config()
    lib().ct_config_init(ctypes.byref(cfg))
    cfg.device = device
    cfg.stream = stream
    cfg.alloc = ctypes.pointer(allocator.struct) if allocator is not None else None
    cfg.n_shards = n_shards
    cfg.shard_rank = shard_rank
    keep = None
    if nccl_unique_id is not None:
        keep = ctypes.create_string_buffer(bytes(nccl_unique_id), 128)
        cfg.nccl_unique_id = ctypes.cast(keep, ctypes.c_void_p)
    cfg.update_policy = update_policy
    cfg.use_residues = int(bool(use_residues))
    cfg.use_index = int(bool(use_index))
    cfg.use_graph = int(bool(use_graph))
    cfg.use_fused = int(bool(use_fused))
    cfg.use_gather = int(bool(use_gather))
    cfg.launch_shape = SHAPES[launch_shape] if isinstance(launch_shape, str) else int(launch_shape)
    cfg.grid_override = int(grid_override)
    cfg.batch_per_state = int(bool(batch_per_state))
    cfg.search_levels = int(search_levels)
    cfg.batch_cells = int(bool(batch_cells))
    return cfg, keep


# ---------------------------------------------------------------- C names
def ct_create(lo, d, tuples, init_dom=None, scope=None, cfg=None, kind: int = CT_TABLE_POSITIVE):
    """Returns (status, table, root, root_dom).  root_dom: uint64[Wd] or None on FAIL.
    kind != CT_TABLE_POSITIVE calls ct_create_table (f4: short / negative tables)."""
    lo = np.ascontiguousarray(lo, dtype=np.int32)
    d = np.ascontiguousarray(d, dtype=np.int32)
    tuples = np.ascontiguousarray(tuples, dtype=np.int32)
    n = int(d.size)
    if lo.ndim != 1 or d.ndim != 1 or lo.size != n:
        raise ValueError(f"lo and d must be 1-D of the same length (got {lo.shape}, {d.shape})")
    if tuples.ndim != 2 or (tuples.shape[0] > 0 and tuples.shape[1] != n):
        raise ValueError(f"tuples must be int32[t][{n}] (got shape {tuples.shape})")
    t = int(tuples.shape[0])
    wd = int(((d.astype(np.int64) + 63) // 64).sum())
    if init_dom is not None and np.asarray(init_dom).size < wd:
        raise ValueError(f"init_dom needs {wd} words")
    if scope is not None and np.asarray(scope).size != n:
        raise ValueError(f"scope needs {n} entries")
    out_dom = np.zeros(max(wd, 1), dtype=np.uint64)
    sc = None if scope is None else np.ascontiguousarray(scope, dtype=np.int32)
    idom = None if init_dom is None else np.ascontiguousarray(init_dom, dtype=np.uint64)
    tab, root = ctypes.c_void_p(), ctypes.c_void_p()
    args = (n, _np_ptr(sc), _np_ptr(lo), _np_ptr(d), _np_ptr(idom), t, _np_ptr(tuples) if t else None,
            ctypes.byref(cfg) if cfg is not None else None, ctypes.byref(tab), ctypes.byref(root), _np_ptr(out_dom))
    st = lib().ct_create(*args) if kind == CT_TABLE_POSITIVE else lib().ct_create_table(int(kind), *args)
    _check(st)
    return st, tab, root, (out_dom[:wd] if st == CT_OK else None)


def _need_words(name, a, n):
    if a is not None and (a.ndim != 1 or a.size < n):
        raise ValueError(f"{name} must be a 1-D host array of >= {n} uint64 words (got {a.shape})")


def _need_dev_words(name, t, n):
    if t is not None and hasattr(t, "numel") and t.numel() * t.element_size() < 8 * n:
        raise ValueError(f"{name} must hold >= {n} 64-bit words")


def ct_table_info_get(table) -> ct_table_info:
    info = ct_table_info()
    _check(lib().ct_table_info_get(table, ctypes.byref(info)))
    return info


def ct_dom_words(table) -> int:
    return int(lib().ct_dom_words(table))


def ct_dom_word_offset(table, i: int) -> int:
    return int(lib().ct_dom_word_offset(table, i))


def ct_propagate(state, removed, out_dom, out_pruned=None, wd: int | None = None) -> int:
    """Host numpy buffers (uint64[Wd]); returns CT_OK / CT_FAIL (raises on errors,
    including CT_ESTATE).  wd: the table's Wd, if given the buffers are length-checked."""
    if wd is not None:
        for nm, a in (("removed", removed), ("out_dom", out_dom), ("out_pruned", out_pruned)):
            _need_words(nm, a, wd)
    return _check(lib().ct_propagate(state, _np_ptr(removed), _np_ptr(out_dom), _np_ptr(out_pruned)))


def ct_propagate_async(state, removed, out_dom=None, out_pruned=None, out_status=None,
                       wd: int | None = None) -> int:
    """Device tensors; enqueue only.  wd: if given, tensor buffers are length-checked."""
    if wd is not None:
        for nm, a in (("removed", removed), ("out_dom", out_dom), ("out_pruned", out_pruned)):
            _need_dev_words(nm, a, wd)
    return _check(lib().ct_propagate_async(state, _dev_ptr(removed), _dev_ptr(out_dom), _dev_ptr(out_pruned),
                                           _dev_ptr(out_status)), allow_fail=False)


def ct_propagate_from_async(dst, src, removed, out_dom=None, out_pruned=None, out_status=None,
                            wd: int | None = None) -> int:
    """dst := src propagated with `removed` (include/ct.h); device or pinned buffers, enqueue only."""
    if wd is not None:
        for nm, a in (("removed", removed), ("out_dom", out_dom), ("out_pruned", out_pruned)):
            _need_dev_words(nm, a, wd)
    return _check(lib().ct_propagate_from_async(dst, src, _dev_ptr(removed), _dev_ptr(out_dom), _dev_ptr(out_pruned),
                                                _dev_ptr(out_status)), allow_fail=False)


def ct_propagate_local_async(state, removed) -> int:
    return _check(lib().ct_propagate_local_async(state, _dev_ptr(removed)), allow_fail=False)


def ct_state_flags(state):
    """Returns (device pointer int, n_bytes) of the state's R+1 shard flag bytes."""
    p = ctypes.c_void_p()
    n = ctypes.c_int32()
    _check(lib().ct_state_flags(state, ctypes.byref(p), ctypes.byref(n)), allow_fail=False)
    return int(p.value or 0), int(n.value)


def ct_propagate_apply_async(state, out_dom=None, out_pruned=None, out_status=None) -> int:
    return _check(lib().ct_propagate_apply_async(state, _dev_ptr(out_dom), _dev_ptr(out_pruned),
                                                 _dev_ptr(out_status)), allow_fail=False)


def ct_state_clone(state):
    out = ctypes.c_void_p()
    _check(lib().ct_state_clone(state, ctypes.byref(out)), allow_fail=False)
    return out


def ct_state_copy(dst, src) -> None:
    _check(lib().ct_state_copy(dst, src), allow_fail=False)


def ct_state_set_stream(state, stream) -> None:
    _check(lib().ct_state_set_stream(state, ctypes.c_void_p(int(stream))), allow_fail=False)


def ct_state_stream(state) -> int:
    return int(lib().ct_state_stream(state) or 0)


def ct_synchronize(state) -> None:
    _check(lib().ct_synchronize(state), allow_fail=False)


def ct_state_destroy(state) -> None:
    lib().ct_state_destroy(state)


def ct_table_destroy(table) -> None:
    lib().ct_table_destroy(table)


def ct_batch_create(table, n_states: int, init_state):
    out = ctypes.c_void_p()
    _check(lib().ct_batch_create(table, n_states, init_state, ctypes.byref(out)), allow_fail=False)
    return out


def ct_batch_size(batch) -> int:
    return int(lib().ct_batch_size(batch))


def ct_batch_copy(batch, index: int, state) -> None:
    _check(lib().ct_batch_copy(batch, index, state), allow_fail=False)


def ct_batch_copy_all(batch, state) -> None:
    _check(lib().ct_batch_copy_all(batch, state), allow_fail=False)


def ct_batch_restore_dead(batch, state) -> None:
    _check(lib().ct_batch_restore_dead(batch, state), allow_fail=False)


def ct_propagate_many(batch, removed, out_dom, out_status) -> None:
    _check(lib().ct_propagate_many(batch, _np_ptr(removed), _np_ptr(out_dom), _np_ptr(out_status)),
           allow_fail=False)


def ct_propagate_many_async(batch, removed, out_dom=None, out_status=None) -> None:
    _check(lib().ct_propagate_many_async(batch, _dev_ptr(removed), _dev_ptr(out_dom), _dev_ptr(out_status)),
           allow_fail=False)


def ct_batch_destroy(batch) -> None:
    lib().ct_batch_destroy(batch)


def ct_state_read_table(state, n_words: int) -> np.ndarray:
    out = np.zeros(max(n_words, 1), dtype=np.uint64)
    _check(lib().ct_state_read_table(state, _np_ptr(out)), allow_fail=False)
    return out[:n_words]


def ct_batch_work(batch, reset: bool = False) -> dict:
    """Work counters of the tile-major batch path (include/ct.h)."""
    out = np.zeros(10, dtype=np.int64)
    _check(lib().ct_batch_work(batch, _np_ptr(out), int(bool(reset))), allow_fail=False)
    keys = ("update_support_words", "table_blocks_read", "table_blocks_written", "support_bytes_staged",
            "filter_support_words", "probe_misses", "update_cells_checked", "update_sparse_states",
            "update_active_blocks_in")
    return {k: int(v) for k, v in zip(keys, out)}


def ct_batch_read_table(batch, index: int, n_words: int) -> np.ndarray:
    out = np.zeros(max(n_words, 1), dtype=np.uint64)
    _check(lib().ct_batch_read_table(batch, int(index), _np_ptr(out)), allow_fail=False)
    return out[:n_words]


def ct_table_read_supports(table, row: int, n_words: int) -> np.ndarray:
    out = np.zeros(max(n_words, 1), dtype=np.uint64)
    _check(lib().ct_table_read_supports(table, row, _np_ptr(out)), allow_fail=False)
    return out[:n_words]


def ct_state_read_dom(state, wd: int) -> np.ndarray:
    out = np.zeros(max(wd, 1), dtype=np.uint64)
    _check(lib().ct_state_read_dom(state, _np_ptr(out)), allow_fail=False)
    return out[:wd]


def ct_state_stats(state) -> ct_stats:
    s = ct_stats()
    _check(lib().ct_state_stats(state, ctypes.byref(s)), allow_fail=False)
    return s


def ct_batch_stats(batch, n_states: int):
    """Per-state counters of a batch's last ct_propagate_many (list of ct_stats)."""
    arr = (ct_stats * max(int(n_states), 1))()
    _check(lib().ct_batch_stats(batch, arr), allow_fail=False)
    return list(arr)[:n_states]


def ct_table_profile(table, enable: bool) -> None:
    _check(lib().ct_table_profile(table, int(bool(enable))), allow_fail=False)


def ct_table_profile_read(table, reset: bool = True) -> dict:
    """{kernel: (launches, total_ms)} since the last reset."""
    kt = ct_kernel_times()
    _check(lib().ct_table_profile_read(table, ctypes.byref(kt), int(bool(reset))), allow_fail=False)
    return {name: (int(kt.launches[i]), float(kt.ms[i])) for i, name in enumerate(KERNEL_SLOTS)}


def ct_shard_range(n_tuples: int, n_shards: int, rank: int):
    """(word_begin, words) of shard `rank` (host-only; include/ct.h)."""
    b, w = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().ct_shard_range(n_tuples, n_shards, rank, ctypes.byref(b), ctypes.byref(w)), allow_fail=False)
    return int(b.value), int(w.value)


CT_PEER_HANDLE_BYTES = 64


def ct_state_serve(state, on: bool = True) -> None:
    """Serve the state's synchronous calls with a persistent kernel (include/ct.h)."""
    _check(lib().ct_state_serve(state, int(bool(on))), allow_fail=False)


def ct_debug_serve_idle(ns: int) -> None:
    _check(lib().ct_debug_serve_idle(int(ns)), allow_fail=False)


def ct_peer_export(table) -> bytes:
    """This rank's exchange inbox as a CUDA IPC handle (include/ct.h a10 over NVLink)."""
    buf = ctypes.create_string_buffer(CT_PEER_HANDLE_BYTES)
    _check(lib().ct_peer_export(table, buf), allow_fail=False)
    return buf.raw


def ct_peer_attach(table, handles) -> None:
    """handles: every rank's ct_peer_export bytes, in rank order."""
    blob = b"".join(bytes(h) for h in handles)
    if len(blob) != CT_PEER_HANDLE_BYTES * len(handles):
        raise ValueError("each handle must be CT_PEER_HANDLE_BYTES bytes")
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(lib().ct_peer_attach(table, len(handles), buf), allow_fail=False)


def ct_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().ct_nccl_unique_id(buf), allow_fail=False)
    return buf.raw


# ---------------------------------------------------------------- models (several tables)
def ct_model_create(var_lo, var_size, scopes, tables, cfg=None):
    """scopes: list of int arrays; tables: list of int32[t_k][arity_k].
    Returns (status, model, shared_dom uint64[Wg] or None)."""
    vlo = np.ascontiguousarray(var_lo, np.int32)
    vd = np.ascontiguousarray(var_size, np.int32)
    ar = np.array([len(s) for s in scopes], np.int32)
    sc = np.ascontiguousarray(np.concatenate([np.asarray(s, np.int32) for s in scopes]), np.int32)
    tb = [np.ascontiguousarray(t, np.int32) for t in tables]
    nt = np.array([t.shape[0] for t in tb], np.int64)
    ptrs = (ctypes.c_void_p * len(tb))(*[t.ctypes.data if t.size else 0 for t in tb])
    wg = int(((vd.astype(np.int64) + 63) // 64).sum())
    out_dom = np.zeros(max(wg, 1), np.uint64)
    m = ctypes.c_void_p()
    st = lib().ct_model_create(int(vd.size), _np_ptr(vlo), _np_ptr(vd), len(tb), _np_ptr(ar), _np_ptr(sc),
                               _np_ptr(nt), ctypes.cast(ptrs, ctypes.c_void_p),
                               ctypes.byref(cfg) if cfg is not None else None, ctypes.byref(m), _np_ptr(out_dom))
    _check(st)
    return st, m, (out_dom[:wg] if st == CT_OK else None)


def ct_model_dom_words(model) -> int:
    return int(lib().ct_model_dom_words(model))


def ct_model_fixpoint(model, dom_in, out_dom) -> int:
    return _check(lib().ct_model_fixpoint(model, _np_ptr(dom_in), _np_ptr(out_dom)))


def ct_model_push(model) -> None:
    _check(lib().ct_model_push(model), allow_fail=False)


def ct_model_pop(model) -> None:
    _check(lib().ct_model_pop(model), allow_fail=False)


def ct_model_search(model, n_vars: int, value_order: int = 0, max_nodes: int = 0, max_solutions: int = 1,
                    driver: int | None = None):
    """Returns (status, solution int32[n_vars] or None, ct_search_stats).
    driver: None = library default (device-resident), 0 = device, 1 = host."""
    sol = np.zeros(n_vars, np.int32)
    stats = ct_search_stats()
    if driver is None:
        st = _check(lib().ct_model_search(model, value_order, max_nodes, max_solutions, _np_ptr(sol),
                                          ctypes.byref(stats)))
    else:
        st = _check(lib().ct_model_search_ex(model, value_order, max_nodes, max_solutions, int(driver),
                                             _np_ptr(sol), ctypes.byref(stats)))
    return st, (sol if st == CT_OK else None), stats


def ct_model_search_phases(model) -> dict:
    out = np.zeros(6, np.int64)
    _check(lib().ct_model_search_phases(model, _np_ptr(out)), allow_fail=False)
    return dict(zip(("ingest", "update", "probe", "scan", "finalize", "trail"), (int(x) for x in out)))


def ct_model_destroy(model) -> None:
    lib().ct_model_destroy(model)


# ---------------------------------------------------------------- placement ablation
def ct_host_create(lo, d, tuples, placement: int, init_dom=None, cfg=None):
    """Returns (status, table, root, root_dom or None)."""
    lo = np.ascontiguousarray(lo, dtype=np.int32)
    d = np.ascontiguousarray(d, dtype=np.int32)
    tuples = np.ascontiguousarray(tuples, dtype=np.int32)
    n = int(d.size)
    if lo.ndim != 1 or d.ndim != 1 or lo.size != n:
        raise ValueError("lo and d must be 1-D of the same length")
    if tuples.ndim != 2 or (tuples.shape[0] > 0 and tuples.shape[1] != n):
        raise ValueError(f"tuples must be int32[t][{n}] (got shape {tuples.shape})")
    t = int(tuples.shape[0])
    wd = int(((d.astype(np.int64) + 63) // 64).sum())
    out_dom = np.zeros(max(wd, 1), dtype=np.uint64)
    idom = None if init_dom is None else np.ascontiguousarray(init_dom, dtype=np.uint64)
    tab, root = ctypes.c_void_p(), ctypes.c_void_p()
    st = lib().ct_host_create(n, _np_ptr(lo), _np_ptr(d), _np_ptr(idom), t, _np_ptr(tuples) if t else None,
                              int(placement), ctypes.byref(cfg) if cfg is not None else None,
                              ctypes.byref(tab), ctypes.byref(root), _np_ptr(out_dom))
    _check(st)
    return st, tab, root, (out_dom[:wd] if st == CT_OK else None)


def ct_host_propagate(state, removed, out_dom, out_pruned=None) -> int:
    return _check(lib().ct_host_propagate(state, _np_ptr(removed), _np_ptr(out_dom), _np_ptr(out_pruned)))


def ct_host_clone(state):
    out = ctypes.c_void_p()
    _check(lib().ct_host_clone(state, ctypes.byref(out)), allow_fail=False)
    return out


def ct_host_copy(dst, src) -> None:
    _check(lib().ct_host_copy(dst, src), allow_fail=False)


def ct_host_stats(table, reset: bool = False) -> dict:
    s = ct_place_stats()
    _check(lib().ct_host_stats(table, ctypes.byref(s), int(bool(reset))), allow_fail=False)
    return {k: getattr(s, k) for k, _ in ct_place_stats._fields_}


def ct_host_state_destroy(state) -> None:
    lib().ct_host_state_destroy(state)


def ct_host_table_destroy(table) -> None:
    lib().ct_host_table_destroy(table)


def ct_debug_diag_attach(device: int = 0) -> None:
    """Spin-watchdog diagnostics buffer for `device` (include/ct.h)."""
    _check(lib().ct_debug_diag_attach(int(device)), allow_fail=False)


def ct_debug_spin_limit(device: int, seconds: float) -> None:
    _check(lib().ct_debug_spin_limit(int(device), float(seconds)), allow_fail=False)


def ct_debug_diag_read(n_words: int = 64 + 128 + 2 * 4096) -> np.ndarray:
    out = np.zeros(n_words, np.uint64)
    n = int(lib().ct_debug_diag_read(_np_ptr(out), n_words))
    return out[:n]


def ct_debug_diag_summary() -> str:
    """Human-readable watchdog report ('' if none)."""
    d = ct_debug_diag_read()
    if d.size == 0 or int(d[0]) != 0xD1A6D1A6:
        return ""
    lines = []
    for k in range(16):
        r = d[64 + 8 * k: 64 + 8 * k + 8]
        if int(r[0]) == 0:
            continue
        lines.append(f"report {k}: kind={int(r[0])} cta={int(r[1])} a={int(r[2])} b={int(r[3])} c={int(r[4])} "
                     f"loc={int(r[5]):#x} bseq={int(r[6])} grid={int(r[7])}")
    G = int(d[64 + 7])
    loc = d[64 + 128: 64 + 128 + G]
    bseq = d[64 + 128 + 4096: 64 + 128 + 4096 + G]
    from collections import Counter
    lines.append("loc histogram: " + ", ".join(f"{int(k):#x} x{v}" for k, v in Counter(loc.tolist()).items()))
    lines.append("bseq histogram: " + ", ".join(f"{int(k)} x{v}" for k, v in Counter(bseq.tolist()).items()))
    odd = [i for i in range(G) if bseq[i] != np.bincount(bseq.astype(np.int64)).argmax()]
    lines.append(f"CTAs off the majority barrier count: {odd[:32]}")
    return "\n".join(lines)
