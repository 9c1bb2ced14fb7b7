// ct_runtime.cu -- host runtime and C ABI (include/ct.h) of the B200 Compact-Table
// propagation library.  Owns device memory (through the caller's allocator hook),
// streams, per-state CUDA graphs and the optional NCCL communicator for
// tuple-range sharding.  All propagation arithmetic is in ct_kernels.cuh.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <vector>

#include "ct.h"
#include "ct_kernels.cuh"
#include "ct_model.cuh"
#include "ct_fast.cuh"
#include "ct_batch.cuh"
#include "ct_wide.cuh"
#include "ct_neg.cuh"

// Support-row pitch padding in 64-bit words (a multiple of 16; experiment builds
// only, tools/gpu_pitch.sh: does the row pitch alias HBM channels in the scans?)
#ifndef CT_SUP_PITCH_PAD
#define CT_SUP_PITCH_PAD 0
#endif

using namespace ctk;

constexpr int32_t kPendingStatus = 0x7FFFFFFF;   // mapped status word before the kernel writes it

// ------------------------------------------------------------------ errors
static thread_local char g_err[1024] = "";

static ct_status fail(ct_status s, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return s;
}

#define CUDA_TRY(expr)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess) return fail(CT_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #expr, \
                                       cudaGetErrorString(e_));                              \
  } while (0)

#define NCCL_TRY(expr)                                                                       \
  do {                                                                                       \
    ncclResult_t r_ = (expr);                                                                \
    if (r_ != ncclSuccess) return fail(CT_ENCCL, "%s:%d %s: %s", __FILE__, __LINE__, #expr, \
                                       ncclGetErrorString(r_));                              \
  } while (0)

#define CT_TRY(expr)              \
  do {                            \
    ct_status s_ = (expr);        \
    if (s_ < 0) return s_;        \
  } while (0)

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

inline int plist_po(int) { return 16; }   // header: P, the cell-route descriptor (ct_batch.cuh k_bingest)

// Byte layout of one state's device block.  The persistent prefix [0, persist)
// is what ct_state_copy moves; the rest is per-call scratch.
struct StateLayout {
  size_t ctl, T, idx0, idx1, res, dom, persist;
  size_t din, ulist, items, scanlist, sup, varcnt, tilestat, out, slot, bar, bmask, plist, cnt, prod, desc, total;
};

}  // namespace

struct ct_table {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ct_allocator alloc{};
  bool has_alloc = false;
  int n = 0, R = 0, Wd = 0;
  int kind = CT_TABLE_POSITIVE;      // CT_TABLE_* (f4: short / negative tables)
  int64_t t = 0, Wtot = 0, wbeg = 0, W = 0, Wp = 0, t_local = 0;
  int policy = 0, use_res = 1, use_index = 1, use_graph = 1;
  int n_shards = 1, rank = 0;
  ncclComm_t comm = nullptr;
  // a10 over NVLink peer memory (ct_peer_export / ct_peer_attach)
  uint32_t *peer_inbox = nullptr;    // this rank's inbox (cudaMalloc: exportable through CUDA IPC)
  size_t peer_bytes = 0;
  std::vector<void *> peer_opened;   // other ranks' inboxes opened here
  uint32_t **d_peers = nullptr;      // device [n] inbox pointers
  bool peer_on = false;
  int graph_gen = 0;                 // bumped when the kernels' parameters change (captured graphs go stale)
  std::vector<int32_t> lo, d, rowBase, domOff, scope;
  std::vector<uint64_t> full_dom;    // full-interval domain bitmap
  void *meta = nullptr;
  size_t meta_bytes = 0;
  uint64_t *S = nullptr;
  size_t S_bytes = 0;
  uint32_t *cells = nullptr;         // gather filter (k_fast): packed value offsets per local tuple
  size_t cells_bytes = 0;
  TableDev dev{};
  StateLayout lay{};
  int sm_count = 148;
  // per-kernel event timing (ct_table_profile)
  bool prof_on = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Mark { int kid, e0, e1; };
  std::vector<Mark> marks;
  int upd_occ = 1, scan_occ = 1;
  int use_fused = 1, fused_grid = 1, fused_occ = 1, coop = 1, fused_grid_override = 0, use_small = 0;
  size_t fused_smem = 0, small_smem = 0;
  int use_fast = 0, fast_grid = 1;   // k_fast (ct_fast.cuh): tables with R <= kLocalRowsMax
  size_t fast_smem = 0;
  int use_wide = 0;                  // k_wide + k_wide_filter (ct_wide.cuh): many rows, few words
  size_t wide_smem = 0;
  int bt_tw = 0, bt_grid = 0;        // tile-major batch update (ct_batch.cuh): tile width, 0 = per-state kernels
  int bt_cells = 0;                  // 1: its cell route is on (tuple cells staged next to the support tile)
  size_t bt_smem = 0;
  int neg_occ = 1;                   // k_neg_count CTAs per SM (negative tables)
  int live = 0;   // states + batches alive

  void *dalloc(size_t bytes) {
    if (bytes == 0) bytes = 256;
    if (has_alloc) return alloc.alloc(bytes, (void *)stream, alloc.ctx);
    void *p = nullptr;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    return p;
  }
  void dfree(void *p, size_t bytes) {
    if (!p) return;
    if (bytes == 0) bytes = 256;
    if (has_alloc) alloc.free(p, bytes, (void *)stream, alloc.ctx);
    else cudaFree(p);
  }
};

struct ct_state {
  ct_table *tb = nullptr;
  cudaStream_t stream = nullptr;
  char *mem = nullptr;
  StateDev h{};              // host copy of the descriptor
  StateDev *d_desc = nullptr;
  uint64_t *h_in = nullptr;  // pinned [Wd]
  uint64_t *h_out = nullptr; // pinned [1 + 2 Wd]
  uint64_t *d_in_map = nullptr, *d_out_map = nullptr;   // device aliases of h_in / h_out
  cudaGraphExec_t gexec = nullptr;
  int gexec_gen = 0;         // tb->graph_gen when gexec was captured
  // async calls with host-memory removals: the removal is DMA'd into one of
  // two device slots on a side stream, so the copy of call i + 1 overlaps
  // call i (events: copy done, slot free again)
  cudaStream_t cp_stream = nullptr;
  cudaEvent_t cp_done[2] = {nullptr, nullptr}, slot_free[2] = {nullptr, nullptr};
  uint32_t cp_i = 0;
  // served calls (ct_state_serve): a persistent k_small_serve polls a doorbell
  bool serve = false, serving = false;
  uint32_t *h_door = nullptr, *d_door = nullptr;   // mapped pinned: [0, 256) tagged request words, then
                                                   // ctl[0] stop, ctl[1] server state (k_small_serve)
  uint32_t srv_seq = 0;      // requests issued
  cudaStream_t srv_stream = nullptr;
  bool pending = false;      // root of a caller-combined shard before its first apply
};

struct ct_batch {
  ct_table *tb = nullptr;
  int S = 0;
  char *mem = nullptr;
  size_t bytes = 0;
  StateDev *d_desc = nullptr;
  std::vector<StateDev> h;
  size_t desc_bytes = 0;
  uint64_t *h_in = nullptr, *h_dom = nullptr;   // pinned [S][Wd]
  int32_t *h_status = nullptr;                  // pinned [S]
  uint64_t *d_in = nullptr, *d_dom = nullptr;   // device [S][Wd]
  int32_t *d_status = nullptr;
  int32_t *d_bgo = nullptr;                     // device [S] (tile-major path)
  int2 *d_miss = nullptr;                       // device [2][S·R] miss lists + 2 counters
  size_t miss_bytes = 0;
  BatchDev bd{};
};

// ------------------------------------------------------------------ layout / descriptors
static StateLayout make_layout(const ct_table *tb) {
  StateLayout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t at = o;
    o = (size_t)round_up((int64_t)(o + bytes), 256);
    return at;
  };
  const int ntiles = tb->dev.ntiles_max;
  L.ctl = take(256);
  L.T = take(tb->Wp * 8);
  L.idx0 = take(tb->Wp / 2 * 4);   // index over 16-byte blocks
  L.idx1 = take(tb->Wp / 2 * 4);
  L.res = take((size_t)tb->R * 4);
  // negative tables: dom is followed by pend[Wd] (values pruned by the last
  // filter whose tuples are still in currTable; part of the state)
  L.dom = take((size_t)tb->Wd * 8 * (tb->kind == CT_TABLE_NEGATIVE ? 2 : 1));
  L.persist = o;
  L.din = take((size_t)tb->Wd * 8);
  L.ulist = take((size_t)tb->R * 4);
  L.items = take((size_t)tb->R * 4);
  L.scanlist = take((size_t)tb->R * 4);
  L.sup = take((size_t)tb->R + 1);
  L.varcnt = take((size_t)tb->n * 8);
  // chained-scan tile statuses (k_fused) / per-CTA survivor counts (k_fast, <= 16 CTAs per SM)
  L.tilestat = take(std::max((size_t)std::max(ntiles, 1) * 8, (size_t)tb->sm_count * 32 * 4));   // k_fast: 2 counts per CTA
  L.out = take((size_t)(1 + 2 * tb->Wd) * 8);
  L.slot = take((size_t)tb->Wd * 8 * 3);   // removal slots: two for async calls (the next call's copy
                                           // overlaps this call), one for the k_fast sync call's copy
  L.bar = take((size_t)kBarWords * 4);
  L.bmask = take((size_t)(tb->dev.W2 + 31) / 32 * 4);   // batch path: survivor bit per 16-byte block
  L.plist = take((size_t)(plist_po(tb->n) + tb->R + 3 * tb->n + 36) * 4);   // batch path: padded update list
  L.cnt = take(tb->kind == CT_TABLE_NEGATIVE ? (size_t)tb->R * 8 : 0);   // negative tables: row counts
  L.prod = take(tb->kind == CT_TABLE_NEGATIVE ? (size_t)tb->n * 8 : 0);  //   and P_x
  L.desc = take(sizeof(StateDev));
  L.total = o;
  return L;
}

static StateDev make_desc(const ct_table *tb, char *mem) {
  const StateLayout &L = tb->lay;
  StateDev s{};
  s.ctl = reinterpret_cast<Ctl *>(mem + L.ctl);
  s.T = reinterpret_cast<uint64_t *>(mem + L.T);
  s.idx0 = reinterpret_cast<int32_t *>(mem + L.idx0);
  s.idx1 = reinterpret_cast<int32_t *>(mem + L.idx1);
  s.res = reinterpret_cast<int32_t *>(mem + L.res);
  s.dom = reinterpret_cast<uint64_t *>(mem + L.dom);
  s.din = reinterpret_cast<uint64_t *>(mem + L.din);
  s.ulist = reinterpret_cast<int32_t *>(mem + L.ulist);
  s.items = reinterpret_cast<int32_t *>(mem + L.items);
  s.scanlist = reinterpret_cast<int32_t *>(mem + L.scanlist);
  s.sup = reinterpret_cast<uint8_t *>(mem + L.sup);
  s.varcnt = reinterpret_cast<int32_t *>(mem + L.varcnt);
  s.tilestat = reinterpret_cast<unsigned long long *>(mem + L.tilestat);
  s.out = reinterpret_cast<uint64_t *>(mem + L.out);
  s.slot = reinterpret_cast<uint64_t *>(mem + L.slot);
  s.bar = reinterpret_cast<uint32_t *>(mem + L.bar);
  if (tb->kind == CT_TABLE_NEGATIVE) {
    s.pend = s.dom + tb->Wd;
    s.cnt = reinterpret_cast<unsigned long long *>(mem + L.cnt);
    s.prod = reinterpret_cast<unsigned long long *>(mem + L.prod);
  }
  return s;
}

static CopyLayout copy_layout(const ct_table *tb) {
  const StateLayout &L = tb->lay;
  CopyLayout cl{};
  cl.T_bytes = (int64_t)tb->dev.W2 * 16;
  cl.o_T = (int64_t)L.T;
  cl.o_idx0 = (int64_t)L.idx0;
  cl.o_idx1 = (int64_t)L.idx1;
  cl.o_res = (int64_t)L.res;
  cl.o_dom = (int64_t)L.dom;
  cl.res_bytes = (int64_t)tb->R * 4;
  cl.dom_bytes = (int64_t)tb->Wd * 8 * (tb->kind == CT_TABLE_NEGATIVE ? 2 : 1);   // + pend
  return cl;
}

// A state copy on the device (ct_state_copy / ct_state_clone): an SM copy of
// the fields the state needs, sized to the bytes (a DMA-engine memcpy of the
// whole persistent block was ~10 us for the 2.2 MB C3 state).
static ct_status launch_state_copy(const ct_table *tb, char *dst, const char *src, cudaStream_t st) {
  const int64_t bytes = (int64_t)tb->dev.W2 * 16 + 2 * (int64_t)tb->dev.W2 * 4 + (int64_t)tb->R * 4 + 4096;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)tb->sm_count * 4, bytes / 4096));
  k_state_copy<<<grid, 256, 0, st>>>(dst, src, copy_layout(tb));
  CUDA_TRY(cudaGetLastError());
  return CT_OK;
}

// `waiter` waits for the work enqueued so far on `producer` (no-op if equal).
static ct_status order_after(cudaStream_t waiter, cudaStream_t producer) {
  if (waiter == producer) return CT_OK;
  cudaEvent_t ev;
  CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  cudaError_t e = cudaEventRecord(ev, producer);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(waiter, ev, 0);
  cudaEventDestroy(ev);
  if (e != cudaSuccess) return fail(CT_ECUDA, "stream ordering failed: %s", cudaGetErrorString(e));
  return CT_OK;
}

// ------------------------------------------------------------------ profiling
static int prof_event(ct_table *tb, cudaStream_t st) {
  if (!tb->prof_on) return -1;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return -1;
  if (tb->ev_used == tb->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    tb->ev_pool.push_back(e);
  }
  const int i = (int)tb->ev_used++;
  cudaEventRecord(tb->ev_pool[i], st);
  return i;
}
static void prof_mark(ct_table *tb, int kid, int e0, cudaStream_t st) {
  static_assert(sizeof(((ct_kernel_times *)nullptr)->ms) / sizeof(double) >= 7, "kernel slots");
  if (e0 < 0) return;
  const int e1 = prof_event(tb, st);
  if (e1 >= 0) tb->marks.push_back({kid, e0, e1});
}

// ------------------------------------------------------------------ launch helpers
static int update_blocks(const ct_table *tb, int S) {
  const int resident = tb->sm_count * tb->upd_occ;
  const int ntiles = std::max(tb->dev.ntiles_max, 1);
  int per_state = (resident + S - 1) / S;
  return std::max(1, std::min(per_state, ntiles));
}
static int scan_blocks(const ct_table *tb, int S) {
  const int resident = tb->sm_count * tb->scan_occ;
  return std::max(1, (resident + S - 1) / S);
}

// a2-a6 on S states (everything before the cross-shard combine).
static ct_status enqueue_local(ct_table *tb, const StateDev *d_desc, int S, const uint64_t *removed,
                               int root_mode, cudaStream_t st) {
  int e = prof_event(tb, st);
  k_ingest<<<dim3(1, S), kIngestTPB, ingest_smem_bytes(tb->n, tb->Wd), st>>>(tb->dev, d_desc, removed, tb->Wd,
                                                                             root_mode);
  prof_mark(tb, 0, e, st);
  e = prof_event(tb, st);
  k_update<<<dim3(update_blocks(tb, S), S), kUpdTPB, 0, st>>>(tb->dev, d_desc);
  prof_mark(tb, 1, e, st);
  e = prof_event(tb, st);
  constexpr int kProbeWarps = kProbeTPB / 32;
  k_probe<<<dim3((unsigned)std::max(1, (tb->R + kProbeWarps - 1) / kProbeWarps), S), kProbeTPB, 0, st>>>(
      tb->dev, d_desc);
  prof_mark(tb, 2, e, st);
  e = prof_event(tb, st);
  k_scan<<<dim3(scan_blocks(tb, S), S), kScanTPB, 0, st>>>(tb->dev, d_desc);
  prof_mark(tb, 3, e, st);
  CUDA_TRY(cudaGetLastError());
  return CT_OK;
}

static ct_status enqueue_combine(ct_table *tb, const StateDev &h, cudaStream_t st) {
  if (tb->comm) {
    const int e = prof_event(tb, st);
    NCCL_TRY(ncclAllReduce(h.sup, h.sup, (size_t)tb->R + 1, ncclUint8, ncclMax, tb->comm, st));
    prof_mark(tb, 4, e, st);
  }
  return CT_OK;
}

static ct_status enqueue_finalize(ct_table *tb, const StateDev *d_desc, int S, uint64_t *out_dom,
                                  uint64_t *out_pruned, int32_t *out_status, int use_state_out,
                                  cudaStream_t st) {
  const int e = prof_event(tb, st);
  k_finalize<<<dim3(1, S), kFinTPB, finalize_smem_bytes(tb->n, tb->Wd), st>>>(
      tb->dev, d_desc, out_dom, tb->Wd, out_pruned, out_status, use_state_out);
  prof_mark(tb, 5, e, st);
  CUDA_TRY(cudaGetLastError());
  return CT_OK;
}

// One call on a negative table (ct_neg.cuh).
static ct_status enqueue_neg(ct_table *tb, ct_state *s, const uint64_t *removed, int root_mode, uint64_t *out_dom,
                             uint64_t *out_pruned, int32_t *out_status, int use_state_out) {
  cudaStream_t st = s->stream;
  const StateDev *d = s->d_desc;
  int e = prof_event(tb, st);
  k_ingest<<<dim3(1, 1), kIngestTPB, ingest_smem_bytes(tb->n, tb->Wd), st>>>(tb->dev, d, removed, tb->Wd,
                                                                              root_mode);
  prof_mark(tb, 0, e, st);
  e = prof_event(tb, st);
  k_update<<<dim3(update_blocks(tb, 1), 1), kUpdTPB, 0, st>>>(tb->dev, d);
  prof_mark(tb, 1, e, st);
  e = prof_event(tb, st);
  k_neg_plan<<<1, kIngestTPB, (size_t)std::max(tb->n, 1) * 8, st>>>(tb->dev, d);
  prof_mark(tb, 2, e, st);
  e = prof_event(tb, st);
  k_neg_count<<<tb->sm_count * tb->neg_occ, kNegTPB, 0, st>>>(tb->dev, d);
  prof_mark(tb, 3, e, st);
  e = prof_event(tb, st);
  k_neg_finalize<<<1, kFinTPB, finalize_smem_bytes(tb->n, tb->Wd), st>>>(tb->dev, d, out_dom, out_pruned,
                                                                          out_status, use_state_out);
  prof_mark(tb, 5, e, st);
  CUDA_TRY(cudaGetLastError());
  return CT_OK;
}

// One single-state call.  Fused: one cooperative launch runs every phase (the
// finalize phase too unless the flags must first be combined across shards);
// otherwise one kernel per phase.  local_only stops before the combine.
// src (ct_propagate_from): the call's input state; the output is s.  k_fast
// reads src and writes s directly; every other launch shape copies first.
static ct_status enqueue_single(ct_table *tb, ct_state *s, const uint64_t *removed, int root_mode,
                                uint64_t *out_dom, uint64_t *out_pruned, int32_t *out_status, int use_state_out,
                                bool local_only, const ct_state *src = nullptr, const RemArg *ra = nullptr) {
  cudaStream_t st = s->stream;
  if (src && !(tb->use_fast && !tb->use_wide && !tb->use_small)) {
    CT_TRY(launch_state_copy(tb, s->mem, src->mem, st));
    src = nullptr;
  }
  if (tb->kind == CT_TABLE_NEGATIVE && !tb->use_fast) {   // ct_neg.cuh: shared ingest + update, counting filter
    CT_TRY(enqueue_neg(tb, s, removed, root_mode, out_dom, out_pruned, out_status, use_state_out));
    return CT_OK;
  }
  if (tb->use_wide) {
    const int fin_inside = (!tb->comm && !local_only) ? 1 : 0;
    const int e = prof_event(tb, st);
    k_wide<<<1, kWideTPB, tb->wide_smem, st>>>(tb->dev, (const StateDev *)s->d_desc, removed, root_mode, fin_inside,
                                               out_dom, out_pruned, out_status, use_state_out);
    // programmatic dependent launch: the filter grid is scheduled while k_wide
    // runs and waits for it at griddepcontrol.wait, hiding its launch latency
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)std::max(1, (tb->R + kWideFiltTPB - 1) / kWideFiltTPB));
    lc.blockDim = dim3(kWideFiltTPB);
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    CUDA_TRY(cudaLaunchKernelEx(&lc, k_wide_filter, tb->dev, (const StateDev *)s->d_desc, fin_inside, out_dom,
                                out_pruned, out_status, use_state_out));
    CUDA_TRY(cudaGetLastError());
    prof_mark(tb, 7, e, st);
    if (fin_inside || local_only) return CT_OK;
  } else if (tb->use_small) {
    const int fin_inside = (!tb->comm && !local_only) ? 1 : 0;
    const int e = prof_event(tb, st);
    k_small<<<1, kSmallTPB, tb->small_smem, st>>>(tb->dev, (const StateDev *)s->d_desc, removed, root_mode,
                                                  fin_inside, out_dom, out_pruned, out_status, use_state_out);
    CUDA_TRY(cudaGetLastError());
    prof_mark(tb, 7, e, st);
    if (fin_inside || local_only) return CT_OK;
  } else if (tb->use_fast) {
    // 2: shards combine their flags inside the kernel over NVLink (peer_combine)
    const int fin_inside = local_only ? 0 : tb->peer_on ? 2 : !tb->comm ? 1 : 0;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)tb->fast_grid);
    lc.blockDim = dim3(kFastTPB);
    lc.dynamicSmemBytes = tb->fast_smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = tb->coop;
    lc.attrs = attr;
    lc.numAttrs = 1;
    const int e = prof_event(tb, st);
    RemArg rarg;
    rarg.n = 0;
    if (ra) rarg = *ra;
    CUDA_TRY(cudaLaunchKernelEx(&lc, k_fast, tb->dev, (const StateDev *)s->d_desc, removed, root_mode, fin_inside,
                                out_dom, out_pruned, out_status, use_state_out,
                                src ? (const StateDev *)src->d_desc : (const StateDev *)nullptr, rarg));
    prof_mark(tb, 6, e, st);
    if (fin_inside || local_only) return CT_OK;
  } else if (tb->use_fused) {
    const int fin_inside = (!tb->comm && !local_only) ? 1 : 0;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)tb->fused_grid);
    lc.blockDim = dim3(kFusedTPB);
    lc.dynamicSmemBytes = tb->fused_smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = tb->coop;
    lc.attrs = attr;
    lc.numAttrs = 1;
    const int e = prof_event(tb, st);
    CUDA_TRY(cudaLaunchKernelEx(&lc, k_fused, tb->dev, (const StateDev *)s->d_desc, removed, root_mode, fin_inside,
                                out_dom, out_pruned, out_status, use_state_out));
    prof_mark(tb, 6, e, st);
    if (fin_inside || local_only) return CT_OK;
  } else {
    CT_TRY(enqueue_local(tb, s->d_desc, 1, removed, root_mode, st));
    if (local_only) return CT_OK;
  }
  CT_TRY(enqueue_combine(tb, s->h, st));
  return enqueue_finalize(tb, s->d_desc, 1, out_dom, out_pruned, out_status, use_state_out, st);
}

// Whole single-state call into the state's own out buffer, with host copies.
static ct_status enqueue_sync_call(ct_state *s, int root_mode) {
  ct_table *tb = s->tb;
  const uint64_t *removed = s->d_in_map;
  if (tb->use_fast && !tb->use_small && !tb->use_wide && tb->Wd) {
    // k_fast: one copy of the removal into device memory (a graph node) instead
    // of every CTA of the grid reading it over the host link (sync C3 bulk at
    // t = 1e7: ingest 9.3 us with the mapped reads vs ~3 us from device memory)
    uint64_t *slot = s->h.slot + 2 * (size_t)tb->Wd;
    CUDA_TRY(cudaMemcpyAsync(slot, s->h_in, (size_t)tb->Wd * 8, cudaMemcpyHostToDevice, s->stream));
    removed = slot;
  }
  return enqueue_single(tb, s, removed, root_mode, nullptr, nullptr, nullptr, 1, false);
}

// Wait for a sync call: the kernel writes the status word of the mapped output
// last (after a system-scope fence), so spinning on it replaces a stream sync.
// The stream is polled every so often so a failed launch cannot hang the host.
static ct_status wait_sync_call(ct_state *s) {
  volatile int32_t *st = (volatile int32_t *)s->h_out;
  for (uint64_t spin = 1;; ++spin) {
    if (*st != kPendingStatus) return CT_OK;
    if ((spin & 1023) == 0) {
      const cudaError_t e = cudaStreamQuery(s->stream);
      if (e == cudaSuccess) {
        if (*st != kPendingStatus) return CT_OK;
        return fail(CT_ECUDA, "propagation finished without writing its status");
      }
      if (e != cudaErrorNotReady) return fail(CT_ECUDA, "propagation failed: %s", cudaGetErrorString(e));
    }
  }
}

// ------------------------------------------------------------------ state lifetime
// served calls (ct_state_serve): the doorbell's layout
constexpr int kDoorCtl = 64;           // uint32 index of the control words (after 32 tagged request words)
constexpr size_t kDoorBytes = 2048;   // + 16 trace stamps at kDoorCtl + 64 (experiment builds), the tagged
                                      // outputs at kDoorCtl + kServeOutWord

// Stop a state's server (if running) before anything else touches the state.
static void quiesce(const ct_state *cs) {
  ct_state *s = const_cast<ct_state *>(cs);
  if (!s || !s->serving) return;
  *(volatile uint32_t *)(s->h_door + kDoorCtl) = 1u;
  cudaStreamSynchronize(s->srv_stream);
  *(volatile uint32_t *)(s->h_door + kDoorCtl) = 0u;
  s->serving = false;
}

static void free_state_mem(ct_state *s) {
  if (!s) return;
  ct_table *tb = s->tb;
  DeviceGuard g(tb->device);
  quiesce(s);
  if (s->srv_stream) cudaStreamDestroy(s->srv_stream);
  for (int b = 0; b < 2; ++b) {
    if (s->cp_done[b]) cudaEventDestroy(s->cp_done[b]);
    if (s->slot_free[b]) cudaEventDestroy(s->slot_free[b]);
  }
  if (s->cp_stream) cudaStreamDestroy(s->cp_stream);
  if (s->h_door) cudaFreeHost(s->h_door);
  // a synchronous call returns once its status word is visible, which the last
  // CTA may write before its final stores: wait for the stream before the
  // memory goes back to the allocator (the torch hook does not synchronize)
  if (s->stream) cudaStreamSynchronize(s->stream);
  if (s->gexec) cudaGraphExecDestroy(s->gexec);
  if (s->h_in) cudaFreeHost(s->h_in);
  if (s->h_out) cudaFreeHost(s->h_out);
  if (s->mem) tb->dfree(s->mem, tb->lay.total);
  tb->live--;
  delete s;
}

static ct_status new_state(ct_table *tb, ct_state **out) {
  ct_state *s = new (std::nothrow) ct_state();
  if (!s) return fail(CT_ENOMEM, "host allocation failed");
  s->tb = tb;
  s->stream = tb->stream;
  tb->live++;
  s->mem = (char *)tb->dalloc(tb->lay.total);
  if (!s->mem) {
    free_state_mem(s);
    return fail(CT_ENOMEM, "device allocation of %zu bytes for a state failed", tb->lay.total);
  }
  // mapped pinned staging: the sync path's kernels read `removed` from and write
  // status + domains to host memory directly (zero-copy, no memcpy nodes)
  if (cudaHostAlloc((void **)&s->h_in, std::max<size_t>(8, (size_t)tb->Wd * 8), cudaHostAllocMapped) !=
          cudaSuccess ||
      cudaHostAlloc((void **)&s->h_out, (size_t)(1 + 2 * tb->Wd) * 8, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void **)&s->d_in_map, s->h_in, 0) != cudaSuccess ||
      cudaHostGetDevicePointer((void **)&s->d_out_map, s->h_out, 0) != cudaSuccess) {
    cudaGetLastError();
    free_state_mem(s);
    return fail(CT_ENOMEM, "mapped pinned host allocation failed");
  }
  // per-call scratch starts zeroed (k_fast's tile statuses and miss list rely on it)
  if (cudaMemsetAsync(s->mem + tb->lay.persist, 0, tb->lay.total - tb->lay.persist, tb->stream) != cudaSuccess) {
    cudaGetLastError();
    free_state_mem(s);
    return fail(CT_ECUDA, "state scratch initialisation failed");
  }
  s->h = make_desc(tb, s->mem);
  s->h.out = s->d_out_map;
  s->d_desc = reinterpret_cast<StateDev *>(s->mem + tb->lay.desc);
  ct_status st = CT_OK;
  // after the scratch memset on the same stream (the descriptor lives in the
  // scratch region), then synchronous: it must be in place whichever stream
  // uses the state first
  if (cudaMemcpyAsync(s->d_desc, &s->h, sizeof(StateDev), cudaMemcpyHostToDevice, tb->stream) != cudaSuccess ||
      cudaStreamSynchronize(tb->stream) != cudaSuccess) {
    st = fail(CT_ECUDA, "descriptor upload failed: %s", cudaGetErrorString(cudaGetLastError()));
  }
  if (st != CT_OK) {
    free_state_mem(s);
    return st;
  }
  *out = s;
  return CT_OK;
}

// ------------------------------------------------------------------ table lifetime
static void free_table(ct_table *tb) {
  if (!tb) return;
  DeviceGuard g(tb->device);
  if (tb->stream) cudaStreamSynchronize(tb->stream);
  if (tb->comm) ncclCommDestroy(tb->comm);
  for (void *p : tb->peer_opened) cudaIpcCloseMemHandle(p);
  if (tb->d_peers) cudaFree(tb->d_peers);
  if (tb->peer_inbox) cudaFree(tb->peer_inbox);
  for (cudaEvent_t e : tb->ev_pool) cudaEventDestroy(e);
  if (tb->S) tb->dfree(tb->S, tb->S_bytes);
  if (tb->cells) tb->dfree(tb->cells, tb->cells_bytes);
  if (tb->meta) tb->dfree(tb->meta, tb->meta_bytes);
  if (tb->own_stream && tb->stream) cudaStreamDestroy(tb->stream);
  delete tb;
}

extern "C" {

void ct_config_init(ct_config *cfg) {
  if (!cfg) return;
  memset(cfg, 0, sizeof *cfg);
  cfg->device = 0;
  cfg->n_shards = 1;
  cfg->shard_rank = 0;
  cfg->update_policy = CT_POLICY_AUTO;
  cfg->use_residues = 1;
  cfg->use_index = 1;
  cfg->use_graph = 1;
  cfg->use_fused = 1;
  cfg->use_gather = 1;
  cfg->batch_cells = 1;
}

ct_status ct_shard_range(int64_t n_tuples, int32_t n_shards, int32_t rank, int64_t *word_begin, int64_t *words) {
  if (n_tuples < 0 || n_shards < 1 || rank < 0 || rank >= n_shards || !word_begin || !words)
    return fail(CT_EINVAL, "ct_shard_range: bad arguments");
  const int64_t wtot = (n_tuples + 63) / 64;
  // shard g owns words [b_g, b_{g+1}), b_g = floor(g*Wtot/G) rounded down to 16 words, b_G = Wtot
  auto bound = [&](int64_t g) -> int64_t {
    if (g >= n_shards) return wtot;
    return (int64_t)((__int128)wtot * g / n_shards) / 16 * 16;
  };
  *word_begin = bound(rank);
  *words = bound(rank + 1) - *word_begin;
  return CT_OK;
}

const char *ct_last_error(void) { return g_err; }

// Spin-watchdog diagnostics (ct_kernels.cuh spin_report): one host-mapped
// buffer per process, attached to a device's g_diag.
static unsigned long long *g_diag_host = nullptr;
ct_status ct_debug_diag_attach(int32_t device) {
  DeviceGuard g(device);
  if (!g_diag_host) {
    CUDA_TRY(cudaHostAlloc((void **)&g_diag_host, sizeof(unsigned long long) * kDiagWords, cudaHostAllocMapped |
                                                                                             cudaHostAllocPortable));
    memset(g_diag_host, 0, sizeof(unsigned long long) * kDiagWords);
  }
  unsigned long long *dp = nullptr;
  CUDA_TRY(cudaHostGetDevicePointer((void **)&dp, g_diag_host, 0));
  CUDA_TRY(cudaMemcpyToSymbol(g_diag, &dp, sizeof dp));
  CUDA_TRY(cudaDeviceSynchronize());
  return CT_OK;
}
ct_status ct_debug_spin_limit(int32_t device, double seconds) {
  if (!(seconds > 0)) return fail(CT_EINVAL, "spin limit must be > 0 s");
  DeviceGuard g(device);
  const unsigned long long ns = (unsigned long long)(seconds * 1e9);
  CUDA_TRY(cudaMemcpyToSymbol(g_spin_limit_ns, &ns, sizeof ns));
  CUDA_TRY(cudaDeviceSynchronize());
  return CT_OK;
}
int64_t ct_debug_diag_read(uint64_t *out, int64_t n_words) {
  if (!g_diag_host || !out) return 0;
  const int64_t n = std::min<int64_t>(n_words, kDiagWords);
  for (int64_t i = 0; i < n; ++i) out[i] = ((volatile unsigned long long *)g_diag_host)[i];
  return n;
}

const char *ct_version(void) { return "ct_b200 0.1 (sm_100a)"; }

ct_status ct_nccl_unique_id(void *out128) {
  if (!out128) return fail(CT_EINVAL, "ct_nccl_unique_id: NULL output");
  ncclUniqueId id;
  NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  memcpy(out128, &id, 128);
  return CT_OK;
}

// Negative tables list each forbidden assignment once (ct_neg.cuh counts
// currTable bits): the distinct tuples in order of first occurrence.  Rows are
// grouped by a 64-bit hash (sort of (hash, index) pairs), equal hashes compared
// exactly.
static std::vector<int32_t> distinct_tuples(int32_t n, int64_t t, const int32_t *tuples) {
  std::vector<std::pair<uint64_t, int64_t>> h((size_t)t);
  for (int64_t j = 0; j < t; ++j) {
    uint64_t x = 0x9E3779B97F4A7C15ull;
    for (int i = 0; i < n; ++i) {
      x ^= (uint32_t)tuples[j * n + i];
      x *= 0xBF58476D1CE4E5B9ull;
      x ^= x >> 31;
    }
    h[(size_t)j] = {x, j};
  }
  std::sort(h.begin(), h.end());
  std::vector<char> keep((size_t)t, 1);
  for (size_t a = 0; a < h.size();) {
    size_t b = a + 1;
    while (b < h.size() && h[b].first == h[a].first) ++b;
    for (size_t i = a + 1; i < b; ++i)       // run sorted by index: keep each row's first occurrence
      for (size_t k = a; k < i; ++k)
        if (keep[(size_t)h[k].second] &&
            !memcmp(tuples + h[i].second * n, tuples + h[k].second * n, sizeof(int32_t) * (size_t)n)) {
          keep[(size_t)h[i].second] = 0;
          break;
        }
    a = b;
  }
  std::vector<int32_t> out;
  for (int64_t j = 0; j < t; ++j)
    if (keep[(size_t)j]) out.insert(out.end(), tuples + j * n, tuples + (j + 1) * n);
  return out;
}

static ct_status create_impl(int32_t kind, int32_t n, const int32_t *scope, const int32_t *dom_lo,
                             const int32_t *dom_size, const uint64_t *init_dom, int64_t n_tuples,
                             const int32_t *tuples, const ct_config *cfg_in, ct_table **out_table,
                             ct_state **out_root, uint64_t *out_dom, ct_table *tb) {
  ct_config cfg;
  if (cfg_in) cfg = *cfg_in;
  else ct_config_init(&cfg);
  if (kind != CT_TABLE_POSITIVE && kind != CT_TABLE_SHORT && kind != CT_TABLE_NEGATIVE)
    return fail(CT_EINVAL, "bad table kind %d", kind);

  // ---------------- validation (include/ct.h)
  if (n < 1) return fail(CT_EINVAL, "n_vars must be >= 1 (got %d)", n);
  if (!dom_lo || !dom_size) return fail(CT_EINVAL, "dom_lo and dom_size are required");
  if (n_tuples < 0) return fail(CT_EINVAL, "n_tuples must be >= 0");
  if (n_tuples > 0 && !tuples) return fail(CT_EINVAL, "tuples is NULL");
  if (!out_table || !out_root) return fail(CT_EINVAL, "out_table and out_root are required");
  if (cfg.n_shards < 1 || cfg.shard_rank < 0 || cfg.shard_rank >= cfg.n_shards)
    return fail(CT_EINVAL, "bad shard config (n_shards=%d, shard_rank=%d)", cfg.n_shards, cfg.shard_rank);
  if (cfg.update_policy < 0 || cfg.update_policy > 2) return fail(CT_EINVAL, "bad update_policy");
  if (cfg.alloc && (!cfg.alloc->alloc || !cfg.alloc->free)) return fail(CT_EINVAL, "allocator hooks missing");
  int64_t R = 0;
  for (int i = 0; i < n; ++i) {
    if (dom_size[i] < 1) return fail(CT_EINVAL, "dom_size[%d] must be >= 1", i);
    if ((int64_t)dom_lo[i] + dom_size[i] - 1 > INT32_MAX) return fail(CT_EINVAL, "domain %d overflows int32", i);
    R += dom_size[i];
  }
  if (R >= (int64_t)kRowMask) return fail(CT_EINVAL, "too many support rows (%lld)", (long long)R);
  if (scope) {
    std::vector<int32_t> sc(scope, scope + n);
    std::sort(sc.begin(), sc.end());
    if (std::adjacent_find(sc.begin(), sc.end()) != sc.end())
      return fail(CT_EINVAL, "duplicate variable in scope (var(c) is a set, PAPER.md L48)");
  }
  if (kind == CT_TABLE_NEGATIVE && cfg.n_shards != 1)
    return fail(CT_EINVAL, "negative tables are not sharded (their filter counts; the shard combine is an OR)");
  std::vector<int32_t> distinct;
  if (kind == CT_TABLE_NEGATIVE && n_tuples > 0) {
    distinct = distinct_tuples(n, n_tuples, tuples);
    n_tuples = (int64_t)distinct.size() / n;
    tuples = distinct.data();
  }
  // short tables: a column with a star cell never takes the Δ-branch (use_delta)
  std::vector<int32_t> dom_only;
  if (kind == CT_TABLE_SHORT) {
    dom_only.assign(n, 0);
    for (int64_t j = 0; j < n_tuples; ++j)
      for (int i = 0; i < n; ++i)
        if (tuples[j * n + i] == CT_STAR) dom_only[i] = 1;
  }
  int ndev = 0;
  CUDA_TRY(cudaGetDeviceCount(&ndev));
  if (cfg.device < 0 || cfg.device >= ndev) return fail(CT_EINVAL, "device %d not present (%d devices)", cfg.device, ndev);

  // ---------------- geometry
  tb->device = cfg.device;
  tb->kind = kind;
  tb->n = n;
  tb->R = (int)R;
  tb->t = n_tuples;
  tb->policy = cfg.update_policy;
  tb->use_res = cfg.use_residues ? 1 : 0;
  tb->use_index = cfg.use_index ? 1 : 0;
  tb->use_graph = cfg.use_graph ? 1 : 0;
  tb->use_fused = cfg.use_fused ? 1 : 0;   // negative tables: k_fast's counting mode, else ct_neg.cuh's kernels
  if (cfg.launch_shape < 0 || cfg.launch_shape > CT_SHAPE_WIDE) return fail(CT_EINVAL, "bad launch_shape");
  if (cfg.launch_shape == CT_SHAPE_PHASES) tb->use_fused = 0;
  tb->fused_grid_override = std::max(0, cfg.grid_override);
  tb->n_shards = cfg.n_shards;
  tb->rank = cfg.shard_rank;
  if (cfg.alloc) {
    tb->alloc = *cfg.alloc;
    tb->has_alloc = true;
  }
  tb->lo.assign(dom_lo, dom_lo + n);
  tb->d.assign(dom_size, dom_size + n);
  if (scope) tb->scope.assign(scope, scope + n);
  tb->rowBase.assign(n + 1, 0);
  tb->domOff.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    tb->rowBase[i + 1] = tb->rowBase[i] + dom_size[i];
    tb->domOff[i + 1] = tb->domOff[i] + (dom_size[i] + 63) / 64;
  }
  tb->Wd = tb->domOff[n];
  tb->Wtot = (n_tuples + 63) / 64;
  CT_TRY(ct_shard_range(n_tuples, tb->n_shards, tb->rank, &tb->wbeg, &tb->W));
  if (tb->W > INT32_MAX - 1024) return fail(CT_EINVAL, "table shard too large (%lld words)", (long long)tb->W);
  tb->Wp = round_up(std::max<int64_t>(tb->W, 1), 16) + CT_SUP_PITCH_PAD;
  const int64_t j0 = std::min(tb->wbeg * 64, n_tuples), j1 = std::min((tb->wbeg + tb->W) * 64, n_tuples);
  tb->t_local = j1 - j0;
  tb->full_dom.assign(tb->Wd, 0ull);
  for (int i = 0; i < n; ++i)
    for (int a = 0; a < dom_size[i]; ++a) tb->full_dom[tb->domOff[i] + a / 64] |= 1ull << (a % 64);

  DeviceGuard guard(tb->device);
  if (cfg.stream) {
    tb->stream = (cudaStream_t)cfg.stream;
  } else {
    CUDA_TRY(cudaStreamCreateWithFlags(&tb->stream, cudaStreamNonBlocking));
    tb->own_stream = true;
  }
  CUDA_TRY(cudaDeviceGetAttribute(&tb->sm_count, cudaDevAttrMultiProcessorCount, tb->device));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tb->upd_occ, k_update, kUpdTPB, 0));
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tb->scan_occ, k_scan, kScanTPB, 0));
  tb->upd_occ = std::max(1, tb->upd_occ);
  {
    const size_t ib = ingest_smem_bytes(n, tb->Wd), fb = finalize_smem_bytes(n, tb->Wd);
    if (std::max(ib, fb) > 200 * 1024)
      return fail(CT_EINVAL, "table too wide for the single-block ingest (n=%d, %d domain words)", n, tb->Wd);
    CUDA_TRY(cudaFuncSetAttribute(k_ingest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(ib, 1)));
    CUDA_TRY(cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(fb, 1)));
    tb->fused_smem = std::max(ib, fb);
    CUDA_TRY(cudaFuncSetAttribute(k_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(tb->fused_smem, 1)));
    int occ = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused, kFusedTPB, tb->fused_smem));
    if (occ < 1) tb->use_fused = 0;
    tb->small_smem = small_smem_bytes(n, tb->Wd, (int)R);
    if (tb->small_smem <= 200 * 1024) {
      CUDA_TRY(cudaFuncSetAttribute(k_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb->small_smem));
    }
    tb->fused_occ = std::max(occ, 1);
  }
  tb->scan_occ = std::max(1, tb->scan_occ);
  if (kind == CT_TABLE_NEGATIVE) {
    CUDA_TRY(cudaFuncSetAttribute(k_neg_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, std::max(n, 1) * 8));
    CUDA_TRY(cudaFuncSetAttribute(k_neg_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(finalize_smem_bytes(n, tb->Wd), 1)));
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tb->neg_occ, k_neg_count, kNegTPB, 0));
    tb->neg_occ = std::max(1, tb->neg_occ);
  }

  // ---------------- NCCL (tuple-range sharding)
  if (cfg.nccl_unique_id) {
    ncclUniqueId id;
    memcpy(&id, cfg.nccl_unique_id, sizeof id);
    NCCL_TRY(ncclCommInitRank(&tb->comm, tb->n_shards, id, tb->rank));
  }

  // ---------------- table metadata on the device
  std::vector<int32_t> wordVar(std::max(tb->Wd, 1)), rowVar(std::max(tb->R, 1));
  for (int i = 0; i < n; ++i) {
    for (int k = tb->domOff[i]; k < tb->domOff[i + 1]; ++k) wordVar[k] = i;
    for (int r = tb->rowBase[i]; r < tb->rowBase[i + 1]; ++r) rowVar[r] = i;
  }
  std::vector<int32_t> meta;
  meta.insert(meta.end(), tb->rowBase.begin(), tb->rowBase.end());   // [0, n+1)
  meta.insert(meta.end(), tb->domOff.begin(), tb->domOff.end());     // [n+1, 2n+2)
  meta.insert(meta.end(), wordVar.begin(), wordVar.end());           // [2n+2, +Wd)
  meta.insert(meta.end(), rowVar.begin(), rowVar.end());             // [.., +R)
  meta.insert(meta.end(), tb->lo.begin(), tb->lo.end());
  meta.insert(meta.end(), tb->d.begin(), tb->d.end());
  const size_t dom_only_at = meta.size();
  meta.insert(meta.end(), dom_only.begin(), dom_only.end());
  tb->meta_bytes = meta.size() * 4;
  tb->meta = tb->dalloc(tb->meta_bytes);
  if (!tb->meta) return fail(CT_ENOMEM, "device allocation of table metadata failed");
  CUDA_TRY(cudaMemcpyAsync(tb->meta, meta.data(), tb->meta_bytes, cudaMemcpyHostToDevice, tb->stream));
  const int32_t *m = (const int32_t *)tb->meta;
  const int32_t *d_rowBase = m, *d_domOff = m + n + 1, *d_wordVar = m + 2 * n + 2;
  const int32_t *d_rowVar = d_wordVar + std::max(tb->Wd, 1);
  const int32_t *d_lo = d_rowVar + std::max(tb->R, 1), *d_d = d_lo + n;
  const bool any_star = std::find(dom_only.begin(), dom_only.end(), 1) != dom_only.end();

  tb->S_bytes = (size_t)tb->R * (size_t)tb->Wp * 8;
  tb->S = (uint64_t *)tb->dalloc(tb->S_bytes);
  if (!tb->S) return fail(CT_ENOMEM, "device allocation of %zu bytes of supports failed", tb->S_bytes);
  CUDA_TRY(cudaMemsetAsync(tb->S, 0, tb->S_bytes, tb->stream));

  TableDev &dv = tb->dev;
  dv.S = tb->S;
  dv.rowBase = d_rowBase;
  dv.domOff = d_domOff;
  dv.wordVar = d_wordVar;
  dv.rowVar = d_rowVar;
  dv.n = n;
  dv.R = tb->R;
  dv.Wd = tb->Wd;
  dv.W = (int32_t)tb->W;
  dv.W2 = (int32_t)((tb->W + 1) / 2);
  dv.Wp = tb->Wp;
  dv.policy = tb->policy;
  dv.domOnly = any_star ? m + dom_only_at : nullptr;
  dv.use_res = tb->use_res;
  dv.use_index = tb->use_index;
  dv.ntiles_max = (int32_t)((dv.W2 + kUpdTPB - 1) / kUpdTPB);
  tb->lay = make_layout(tb);
  // k_fused grid: every block co-resident (cooperative); at least one block per
  // SM for the filter phases, at most what the update can use beyond that.
  tb->fused_grid = std::min(tb->sm_count * tb->fused_occ, std::max(tb->sm_count, dv.ntiles_max));
  if (tb->fused_grid_override > 0) tb->fused_grid = std::min(tb->sm_count * tb->fused_occ, tb->fused_grid_override);
  // k_fast: per-CTA ingest lists in shared memory (tables with few support rows)
  {
    int fast_ok = (tb->use_fused && tb->R <= kLocalRowsMax) ? 1 : 0;
    if (cfg.launch_shape == CT_SHAPE_FUSED) fast_ok = 0;
    if (fast_ok) {
      tb->fast_smem = fast_smem_bytes(n, tb->Wd, tb->R);
      CUDA_TRY(cudaFuncSetAttribute(k_fast, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb->fast_smem));
      int occ = 0;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fast, kFastTPB, tb->fast_smem));
      if (occ >= 1) {
        tb->use_fast = 1;
        // an equal number of CTAs per SM, enough that one CTA's share of the
        // largest index (W2 entries) is at most kFastTPB entries
        const int per_sm = (int)((dv.W2 + (int64_t)tb->sm_count * kFastTPB - 1) / ((int64_t)tb->sm_count * kFastTPB));
        tb->fast_grid = tb->sm_count * std::max(1, std::min(occ, per_sm));
        // heavy calls on a short index (W2 x R >= 4M block-rows, e.g. t = 1e6 with
        // R = 800): the whole resident grid, its update splitting each entry's
        // rows over several lanes (fast_update_range_split)
        if ((int64_t)dv.W2 * tb->R >= (int64_t)1 << 22) tb->fast_grid = tb->sm_count * occ;
        if (tb->fused_grid_override > 0) tb->fast_grid = std::min(tb->sm_count * occ, tb->fused_grid_override);
      }
    }
  }
  // gather filter (k_fast, ct_fast.cuh): the local tuples' value offsets, 8 or
  // 16 bits per cell, for tables whose filter may scan many support rows
  {
    int maxd = 1;
    for (int i = 0; i < n; ++i) maxd = std::max(maxd, dom_size[i]);
    const bool star_free = kind == CT_TABLE_POSITIVE || (kind == CT_TABLE_SHORT && !any_star);
    // ... and for the batch update's cell route (8-bit cells, ct_batch.cuh)
    const bool batch_cells = cfg.batch_cells && !cfg.batch_per_state && kind == CT_TABLE_POSITIVE && maxd <= 256 &&
                             tb->R >= 1 && bupdate_smem_bytes(tb->R, 32) <= 200 * 1024;
    if (((cfg.use_gather && tb->use_fast) || batch_cells) && star_free && maxd <= 65536 && tb->t_local > 0) {
      const int bits = maxd <= 256 ? 8 : 16;
      const int words = (n * bits + 31) / 32;
      tb->cells_bytes = (size_t)tb->t_local * words * 4;
      tb->cells = (uint32_t *)tb->dalloc(tb->cells_bytes);
      if (!tb->cells) return fail(CT_ENOMEM, "device allocation of %zu bytes of gather cells failed", tb->cells_bytes);
      tb->dev.cells = tb->cells;
      tb->dev.cell_bits = bits;
      tb->dev.cell_words = words;
      tb->dev.gather = (cfg.use_gather && tb->use_fast) ? 1 : 0;
    }
  }

  // batches: tile-major update with the support tile in shared memory when all
  // R rows of a tile of >= 8 blocks fit (ct_batch.cuh)
  {
    int legacy = 0;
    legacy = cfg.batch_per_state ? 1 : 0;
    const size_t cap = 200 * 1024;
    int tw = 0;
    if (!legacy && tb->R >= 1) {
      if (bupdate_smem_bytes(tb->R, 32) <= cap) tw = 32;
      else if (bupdate_smem_bytes(tb->R, 16) <= cap) tw = 16;
      else if (bupdate_smem_bytes(tb->R, 8) <= cap) tw = 8;
    }
    if (tw) {
      tb->bt_smem = bupdate_smem_bytes(tb->R, tw);
      // cell route (ct_batch.cuh tile32_cells): the tile's tuple cells next to
      // the support tile, when the table has 8-bit cells and both fit
      tb->bt_cells = 0;
      if (tw == 32 && tb->cells && tb->dev.cell_bits == 8 && kind == CT_TABLE_POSITIVE && cfg.batch_cells) {
        const size_t cb = (size_t)4096 * tb->dev.cell_words * 4;
        if (tb->bt_smem + cb <= 216 * 1024) {
          tb->bt_smem += cb;
          tb->bt_cells = 1;
        }
      }
      int occ = 0;
      if (tw == 32) {
        CUDA_TRY(cudaFuncSetAttribute(k_bupdate<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb->bt_smem));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bupdate<32>, kBTPB, tb->bt_smem));
      } else if (tw == 16) {
        CUDA_TRY(cudaFuncSetAttribute(k_bupdate<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb->bt_smem));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bupdate<16>, kBTPB, tb->bt_smem));
      } else {
        CUDA_TRY(cudaFuncSetAttribute(k_bupdate<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb->bt_smem));
        CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bupdate<8>, kBTPB, tb->bt_smem));
      }
      const size_t ib = ingest_smem_bytes(n, tb->Wd), fb = finalize_smem_bytes(n, tb->Wd);
      CUDA_TRY(cudaFuncSetAttribute(k_bingest, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)std::max<size_t>(ib, 1)));
      CUDA_TRY(cudaFuncSetAttribute(k_bfinalize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)std::max<size_t>(fb, 1)));
      if (occ >= 1) {
        tb->bt_tw = tw;
        tb->bt_grid = tb->sm_count * occ;
      }
    }
  }
  // latency-bound tables: the whole call in one CTA (k_small)
  {
    int small_max = kSmallMaxPairs;
    if (cfg.launch_shape == CT_SHAPE_FUSED || cfg.launch_shape == CT_SHAPE_FAST) small_max = 0;
    tb->use_small = (tb->use_fused && dv.W2 <= small_max) ? 1 : 0;
    // ... but not when one call may stream more support rows than one CTA
    // should (W2 x R block-rows: a call removing from every variable reads up
    // to ~W2 x R / 2 of them; t = 1e6, R = 800: 100 MB in one CTA = 0.6 ms),
    // unless the table is a k_wide candidate (many rows over few words: the
    // filter dominates there and k_wide spreads it over a grid)
    if (tb->use_small && (int64_t)dv.W2 * tb->R > kSmallMaxWork && tb->R < kWideMinRows &&
        cfg.launch_shape != CT_SHAPE_SMALL)
      tb->use_small = 0;
  }
  // ... unless the filter dominates: many support rows over few words (k_wide)
  {
    int wide_ok = (tb->use_small && tb->R >= kWideMinRows) ? 1 : 0;
    if (cfg.launch_shape == CT_SHAPE_SMALL) wide_ok = 0;
    if (cfg.launch_shape == CT_SHAPE_WIDE) wide_ok = (tb->use_fused && dv.W2 <= kSmallMaxPairs) ? 1 : wide_ok;
    tb->wide_smem = wide_smem_bytes(n, tb->Wd);
    if (wide_ok && tb->wide_smem <= 200 * 1024) {
      CUDA_TRY(cudaFuncSetAttribute(k_wide, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb->wide_smem));
      tb->use_wide = 1;
      tb->use_small = 0;
    }
  }
  if (tb->use_small && tb->small_smem > 200 * 1024) tb->use_small = 0;   // k_small's on-chip lists do not fit
  if (kind == CT_TABLE_NEGATIVE) {   // only k_fast has the counting filter; otherwise k_ingest .. k_neg_finalize
    tb->use_small = tb->use_wide = 0;
    if (!tb->use_fast) tb->use_fused = 0;
    dv.negative = tb->use_fast;
  }

  // ---------------- root state + supports (a1)
  ct_state *root = nullptr;
  CT_TRY(new_state(tb, &root));
  *out_root = root;   // owned by the caller's cleanup path from here on
  CUDA_TRY(cudaMemsetAsync(root->mem, 0, tb->lay.persist, tb->stream));
  if (tb->t_local > 0) {
    const size_t tb_bytes = (size_t)tb->t_local * n * 4;
    void *d_tup = tb->dalloc(tb_bytes);
    if (!d_tup) return fail(CT_ENOMEM, "device allocation of %zu bytes of tuples failed", tb_bytes);
    cudaError_t e = cudaMemcpyAsync(d_tup, tuples + j0 * n, tb_bytes, cudaMemcpyHostToDevice, tb->stream);
    if (e == cudaSuccess) {
      const int threads = 256;
      const int64_t blocks = (tb->t_local + threads - 1) / threads;
      k_build<<<(unsigned)blocks, threads, 0, tb->stream>>>((const int32_t *)d_tup, tb->t_local, n, d_lo, d_d,
                                                            d_rowBase, tb->S, tb->Wp, (uint32_t *)root->h.T,
                                                            2 * tb->Wp, kind == CT_TABLE_SHORT ? 1 : 0);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess && tb->cells) {
      k_build_cells<<<(unsigned)((tb->t_local + 255) / 256), 256, 0, tb->stream>>>(
          (const int32_t *)d_tup, tb->t_local, n, d_lo, d_d, tb->cells, tb->dev.cell_bits, tb->dev.cell_words);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(tb->stream);   // tuples freed below
    tb->dfree(d_tup, tb_bytes);
    if (e != cudaSuccess) return fail(CT_ECUDA, "supports build failed: %s", cudaGetErrorString(e));
  }
  Ctl c0{};
  c0.L = tb->dev.W2;
  c0.identity = 1;
  c0.nvalid = (unsigned long long)tb->t_local;   // negative tables: bound on the root's valid forbidden tuples
  CUDA_TRY(cudaMemcpyAsync(root->h.ctl, &c0, sizeof c0, cudaMemcpyHostToDevice, tb->stream));
  if (tb->Wd)
    CUDA_TRY(cudaMemcpyAsync(root->h.dom, tb->full_dom.data(), (size_t)tb->Wd * 8, cudaMemcpyHostToDevice,
                             tb->stream));
  // root propagation: remove the holes of init_dom
  for (int k = 0; k < tb->Wd; ++k) root->h_in[k] = init_dom ? (tb->full_dom[k] & ~init_dom[k]) : 0ull;
  if (tb->n_shards > 1 && !tb->comm) {
    // caller-combined shard: the root verdict needs every shard's flags, so only
    // the local phase runs here; the caller combines and applies (include/ct.h)
    CT_TRY(enqueue_single(tb, root, root->d_in_map, /*root_mode=*/1, nullptr, nullptr, nullptr, 0, true));
    CUDA_TRY(cudaStreamSynchronize(tb->stream));   // h_in is reused by later calls
    root->pending = true;
    *out_table = tb;
    return CT_PENDING;
  }
  *(volatile int32_t *)root->h_out = kPendingStatus;
  CT_TRY(enqueue_sync_call(root, /*root_mode=*/1));
  CT_TRY(wait_sync_call(root));
  CUDA_TRY(cudaStreamSynchronize(tb->stream));
  const int32_t status = *(const int32_t *)root->h_out;
  if (status == CT_OK && out_dom && tb->Wd) memcpy(out_dom, root->h_out + 1, (size_t)tb->Wd * 8);
  *out_table = tb;
  return status == CT_OK ? CT_OK : CT_FAIL;
}

ct_status ct_create_table(int32_t kind, int32_t n_vars, const int32_t *scope, const int32_t *dom_lo,
                          const int32_t *dom_size, const uint64_t *init_dom, int64_t n_tuples,
                          const int32_t *tuples, const ct_config *cfg, ct_table **out_table, ct_state **out_root,
                          uint64_t *out_dom) {
  if (out_table) *out_table = nullptr;
  if (out_root) *out_root = nullptr;
  ct_table *tb = new (std::nothrow) ct_table();
  if (!tb) return fail(CT_ENOMEM, "host allocation failed");
  ct_state *root = nullptr;
  ct_table *tab = nullptr;
  ct_status s = create_impl(kind, n_vars, scope, dom_lo, dom_size, init_dom, n_tuples, tuples, cfg, &tab,
                            &root, out_dom, tb);
  if (s < 0) {
    if (root) free_state_mem(root);
    free_table(tb);
    return s;
  }
  *out_table = tab;
  *out_root = root;
  return s;
}

ct_status ct_create(int32_t n_vars, const int32_t *scope, const int32_t *dom_lo, const int32_t *dom_size,
                    const uint64_t *init_dom, int64_t n_tuples, const int32_t *tuples, const ct_config *cfg,
                    ct_table **out_table, ct_state **out_root, uint64_t *out_dom) {
  return ct_create_table(CT_TABLE_POSITIVE, n_vars, scope, dom_lo, dom_size, init_dom, n_tuples, tuples, cfg,
                         out_table, out_root, out_dom);
}

ct_status ct_table_info_get(const ct_table *t, ct_table_info *o) {
  if (!t || !o) return fail(CT_EINVAL, "NULL argument");
  o->n_vars = t->n;
  o->n_rows = t->R;
  o->dom_words = t->Wd;
  o->n_shards = t->n_shards;
  o->shard_rank = t->rank;
  o->n_tuples = t->t;
  o->words_total = t->Wtot;
  o->word_begin = t->wbeg;
  o->words = t->W;
  o->row_stride_words = t->Wp;
  o->device_bytes = (int64_t)(t->S_bytes + t->meta_bytes);
  o->state_bytes = (int64_t)t->lay.total;
  const bool neg_kernels = t->kind == CT_TABLE_NEGATIVE && !t->use_fast;
  o->kernel_path = neg_kernels ? 5 : t->use_wide ? 4 : t->use_small ? 3 : t->use_fast ? 2 : t->use_fused ? 1 : 0;
  o->grid = neg_kernels ? t->sm_count * t->neg_occ : t->use_wide ? 1 : t->use_small ? 1
          : t->use_fast ? t->fast_grid : t->use_fused ? t->fused_grid : 0;
  o->batch_tile = t->bt_tw;
  o->gather_cell_bits = t->dev.gather ? t->dev.cell_bits : 0;
  o->kind = t->kind;
  o->batch_cells = t->bt_cells;
  return CT_OK;
}

int32_t ct_dom_words(const ct_table *t) { return t ? t->Wd : -1; }
int32_t ct_dom_word_offset(const ct_table *t, int32_t i) {
  if (!t || i < 0 || i >= t->n) return -1;
  return t->domOff[i];
}

// ------------------------------------------------------------------ served calls (ct_state_serve)

static ct_status launch_server(ct_state *s, uint32_t last) {
  ct_table *tb = s->tb;
  CT_TRY(order_after(s->srv_stream, s->stream));   // after the state's earlier work
  *(volatile uint32_t *)(s->h_door + kDoorCtl + 1) = 1u;
  *(volatile uint32_t *)(s->h_door + kDoorCtl) = 0u;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  k_small_serve<<<1, kSmallTPB, tb->small_smem, s->srv_stream>>>(
      tb->dev, s->d_desc, reinterpret_cast<const unsigned long long *>(s->d_door), s->d_door + kDoorCtl, last,
      copy_layout(tb));
  CUDA_TRY(cudaGetLastError());
  s->serving = true;
  return CT_OK;
}

// One ct_propagate on a served state: inputs into the mapped staging, ring
// the doorbell, wait for the status word (relaunching the server if it had
// stopped on its idle limit before seeing the request).
// src != nullptr: a restore request (this state := src, served in place).
static ct_status served_call(ct_state *s, const ct_state *src = nullptr) {
  if (!s->serving) CT_TRY(launch_server(s, s->srv_seq));
  const uint32_t req = ++s->srv_seq;
  std::atomic_thread_fence(std::memory_order_seq_cst);   // the pending status first
  // the request: the removal's 32-bit halves, the operation and the source
  // state's address, each tagged with the sequence number
  const uint32_t *half = reinterpret_cast<const uint32_t *>(s->h_in);
  volatile unsigned long long *rq = reinterpret_cast<volatile unsigned long long *>(s->h_door);
  const int w2 = 2 * s->tb->Wd;
  const unsigned long long tg = (unsigned long long)req << 32;
  const unsigned long long sa = src ? (unsigned long long)(uintptr_t)src->mem : 0ull;
  for (int k = 0; k < w2; ++k) rq[k] = tg | (src ? 0u : half[k]);
  rq[w2] = tg | (src ? 1u : 0u);
  rq[w2 + 1] = tg | (uint32_t)sa;
  rq[w2 + 2] = tg | (uint32_t)(sa >> 32);
  // the outputs come back as tagged 32-bit halves (no fence on the device):
  // the status word first, then every dom / pruned half of this request
  const int Wd = s->tb->Wd;
  volatile const unsigned long long *to =
      reinterpret_cast<volatile const unsigned long long *>(s->h_door + kDoorCtl + kServeOutWord);
  auto done = [&]() -> bool {
    const unsigned long long w = to[4 * Wd];
    if ((uint32_t)(w >> 32) != req) return false;
    if (src) return true;   // a restore answers with its tagged status only
    const int32_t status = (int32_t)(uint32_t)w;
    if (status == CT_OK) {
      for (int k = 0; k < 4 * Wd; ++k)
        if ((uint32_t)(to[k] >> 32) != req) return false;
      uint32_t *o = reinterpret_cast<uint32_t *>(s->h_out + 1);
      for (int k = 0; k < 4 * Wd; ++k) o[k] = (uint32_t)to[k];
    }
    *(volatile int32_t *)s->h_out = status;
    return true;
  };
  for (uint64_t spin = 1;; ++spin) {
    if (done()) return CT_OK;
    if (*(volatile uint32_t *)(s->h_door + kDoorCtl + 1) == 2u) {   // the server stopped without serving this request
      if (done()) return CT_OK;
      CUDA_TRY(cudaStreamSynchronize(s->srv_stream));
      if (done()) return CT_OK;
      s->serving = false;
      CT_TRY(launch_server(s, req - 1));
    }
    if ((spin & 4095) == 0) {
      const cudaError_t e = cudaStreamQuery(s->srv_stream);
      if (e != cudaSuccess && e != cudaErrorNotReady) {
        s->serving = false;
        return fail(CT_ECUDA, "served propagation failed: %s", cudaGetErrorString(e));
      }
    }
  }
}

ct_status ct_state_serve(ct_state *s, int32_t on) {
  if (!s) return fail(CT_EINVAL, "NULL state");
  ct_table *tb = s->tb;
  DeviceGuard g(tb->device);
  if (!on) {
    quiesce(s);
    s->serve = false;
    return CT_OK;
  }
  if (!tb->use_small || tb->use_wide || tb->n_shards > 1 || tb->kind == CT_TABLE_NEGATIVE || tb->Wd > kServeMaxWd)
    return fail(CT_EINVAL, "served calls need the single-CTA launch shape (ct_table_info.kernel_path 3), one shard "
                           "and at most %d domain words", kServeMaxWd);
  if (s->pending) return fail(CT_ESTATE, "root of a caller-combined shard");
  const size_t ssm = tb->small_smem;
  if (ssm > 200 * 1024) return fail(CT_EINVAL, "table too large to serve (%zu bytes of shared memory)", ssm);
  CUDA_TRY(cudaFuncSetAttribute(k_small_serve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssm));
  if (!s->h_door) {
    if (cudaHostAlloc((void **)&s->h_door, kDoorBytes, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void **)&s->d_door, s->h_door, 0) != cudaSuccess) {
      cudaGetLastError();
      if (s->h_door) cudaFreeHost(s->h_door);
      s->h_door = nullptr;
      return fail(CT_ENOMEM, "mapped doorbell allocation failed");
    }
    memset(s->h_door, 0, kDoorBytes);
    s->srv_seq = 0;
  }
  if (!s->srv_stream) CUDA_TRY(cudaStreamCreateWithFlags(&s->srv_stream, cudaStreamNonBlocking));
  s->serve = true;
  return CT_OK;
}

ct_status ct_debug_serve_trace(const ct_state *s, int64_t *out16) {
  if (!s || !out16) return fail(CT_EINVAL, "NULL argument");
  for (int i = 0; i < 16; ++i)
    out16[i] = s->h_door ? (int64_t)((volatile unsigned long long *)(s->h_door + kDoorCtl + 64))[i] : 0;
  return CT_OK;
}

ct_status ct_debug_serve_idle(int64_t ns) {
  if (ns <= 0) return fail(CT_EINVAL, "idle limit must be positive");
  const unsigned long long v = (unsigned long long)ns;
  CUDA_TRY(cudaMemcpyToSymbol(g_serve_idle_ns, &v, sizeof v));
  return CT_OK;
}

// ------------------------------------------------------------------ propagation
ct_status ct_propagate(ct_state *s, const uint64_t *removed, uint64_t *out_dom, uint64_t *out_pruned) {
  if (!s) return fail(CT_EINVAL, "NULL state");
  ct_table *tb = s->tb;
  if (tb->n_shards > 1 && !tb->comm && !tb->peer_on)
    return fail(CT_EINVAL, "sharded table without NCCL: use ct_propagate_local_async/apply_async");
  DeviceGuard g(tb->device);
  if (tb->Wd) {
    if (removed) memcpy(s->h_in, removed, (size_t)tb->Wd * 8);
    else memset(s->h_in, 0, (size_t)tb->Wd * 8);
  }
  *(volatile int32_t *)s->h_out = kPendingStatus;
  if (s->serve) {
    CT_TRY(served_call(s));
  } else if (tb->use_graph) {
    if (s->gexec && s->gexec_gen != tb->graph_gen) {   // captured with stale kernel parameters
      cudaGraphExecDestroy(s->gexec);
      s->gexec = nullptr;
    }
    if (!s->gexec) {
      s->gexec_gen = tb->graph_gen;
      cudaGraph_t graph = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(s->stream, cudaStreamCaptureModeThreadLocal));
      ct_status st = enqueue_sync_call(s, 0);
      cudaError_t e = cudaStreamEndCapture(s->stream, &graph);
      if (st < 0) {
        if (graph) cudaGraphDestroy(graph);
        return st;
      }
      if (e != cudaSuccess) return fail(CT_ECUDA, "graph capture failed: %s", cudaGetErrorString(e));
      e = cudaGraphInstantiate(&s->gexec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) {
        s->gexec = nullptr;
        return fail(CT_ECUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
      }
    }
    CUDA_TRY(cudaGraphLaunch(s->gexec, s->stream));
  } else {
    CT_TRY(enqueue_sync_call(s, 0));
  }
  if (!s->serve) CT_TRY(wait_sync_call(s));
  const int32_t status = *(volatile const int32_t *)s->h_out;
  if (status == CT_OK) {
    if (out_dom && tb->Wd) memcpy(out_dom, s->h_out + 1, (size_t)tb->Wd * 8);
    if (out_pruned && tb->Wd) memcpy(out_pruned, s->h_out + 1 + tb->Wd, (size_t)tb->Wd * 8);
  }
  if (status == CT_ESTATE) return fail(CT_ESTATE, "state is dead (returned CT_FAIL); restore it with ct_state_copy");
  return (ct_status)status;
}

// A host-memory removal for an async call on s.  On the k_fast shape (and
// ra != nullptr) it is read now into *ra and travels with the launch by value
// (removed becomes nullptr).  Otherwise it is DMA'd into slot (cp_i & 1) on
// the state's copy stream once the call that last read that slot is done, and
// the state's stream waits for the copy -- so the copy for call i + 1 runs
// while call i propagates (one copy stream per state, two slots); removed
// becomes the device slot and slot_b the slot to mark free after the call
// (-1: none).
static ct_status stage_removed(ct_state *s, const uint64_t *&removed, int &slot_b, RemArg *ra = nullptr) {
  ct_table *tb = s->tb;
  slot_b = -1;
  if (ra) ra->n = 0;
  if (!removed || !tb->Wd) return CT_OK;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, removed) != cudaSuccess) {
    cudaGetLastError();
    a.type = cudaMemoryTypeUnregistered;
  }
  if (a.type != cudaMemoryTypeUnregistered && a.type != cudaMemoryTypeHost) return CT_OK;   // device memory
  // k_fast: a small removal travels by value with the launch (read here, at enqueue)
  if (ra && tb->use_fast && !tb->use_small && !tb->use_wide && tb->Wd <= kRemArgWords &&
      tb->kind != CT_TABLE_NEGATIVE) {
    memcpy(ra->w, removed, (size_t)tb->Wd * 8);
    ra->n = tb->Wd;
    removed = nullptr;
    return CT_OK;
  }
  if (!s->cp_stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(&s->cp_stream, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CUDA_TRY(cudaEventCreateWithFlags(&s->cp_done[b], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&s->slot_free[b], cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(s->slot_free[b], s->stream));
    }
  }
  const int b = (int)(s->cp_i++ & 1u);
  uint64_t *slot = s->h.slot + (size_t)b * tb->Wd;
  CUDA_TRY(cudaStreamWaitEvent(s->cp_stream, s->slot_free[b], 0));
  CUDA_TRY(cudaMemcpyAsync(slot, removed, (size_t)tb->Wd * 8, cudaMemcpyHostToDevice, s->cp_stream));
  CUDA_TRY(cudaEventRecord(s->cp_done[b], s->cp_stream));
  CUDA_TRY(cudaStreamWaitEvent(s->stream, s->cp_done[b], 0));
  removed = slot;
  slot_b = b;
  return CT_OK;
}

ct_status ct_propagate_async(ct_state *s, const uint64_t *removed, uint64_t *out_dom, uint64_t *out_pruned,
                             int32_t *out_status) {
  if (!s) return fail(CT_EINVAL, "NULL state");
  quiesce(s);
  ct_table *tb = s->tb;
  if (tb->n_shards > 1 && !tb->comm && !tb->peer_on)
    return fail(CT_EINVAL, "sharded table without NCCL: use ct_propagate_local_async/apply_async");
  DeviceGuard g(tb->device);
  // removals in host memory: one DMA into a device slot, overlapped with the
  // previous call (stage_removed), instead of every CTA reading them over the
  // host link (pinned removals read in place by every CTA: C3 bulk e2e 8.7k
  // vs 9.8k with a DMA)
  int slot_b;
  RemArg ra;
  CT_TRY(stage_removed(s, removed, slot_b, &ra));
  CT_TRY(enqueue_single(tb, s, removed, 0, out_dom, out_pruned, out_status, 0, false, nullptr, ra.n ? &ra : nullptr));
  if (slot_b >= 0) CUDA_TRY(cudaEventRecord(s->slot_free[slot_b], s->stream));
  return CT_OK;
}

ct_status ct_propagate_from_async(ct_state *dst, const ct_state *src, const uint64_t *removed, uint64_t *out_dom,
                                  uint64_t *out_pruned, int32_t *out_status) {
  if (!dst || !src) return fail(CT_EINVAL, "NULL state");
  quiesce(dst);
  quiesce(src);
  if (dst == src) return ct_propagate_async(dst, removed, out_dom, out_pruned, out_status);
  ct_table *tb = dst->tb;
  if (src->tb != tb) return fail(CT_ESTATE, "states belong to different tables");
  if (tb->n_shards > 1 && !tb->comm && !tb->peer_on)
    return fail(CT_EINVAL, "sharded table without NCCL: use ct_propagate_local_async/apply_async");
  if (src->pending || dst->pending) return fail(CT_ESTATE, "root of a caller-combined shard: combine and apply first");
  DeviceGuard g(tb->device);
  CT_TRY(order_after(dst->stream, src->stream));   // src's earlier work first
  int slot_b;
  RemArg ra;
  CT_TRY(stage_removed(dst, removed, slot_b, &ra));
  CT_TRY(enqueue_single(tb, dst, removed, 0, out_dom, out_pruned, out_status, 0, false, src, ra.n ? &ra : nullptr));
  if (slot_b >= 0) CUDA_TRY(cudaEventRecord(dst->slot_free[slot_b], dst->stream));
  return order_after(const_cast<ct_state *>(src)->stream, dst->stream);   // src's next writes wait for the call
}

ct_status ct_propagate_local_async(ct_state *s, const uint64_t *removed) {
  if (!s) return fail(CT_EINVAL, "NULL state");
  quiesce(s);
  if (s->tb->kind == CT_TABLE_NEGATIVE) return fail(CT_EINVAL, "negative tables have no shard-local phase");
  if (s->pending) return fail(CT_ESTATE, "root of a caller-combined shard: combine its flags and apply first");
  DeviceGuard g(s->tb->device);
  return enqueue_single(s->tb, s, removed, 0, nullptr, nullptr, nullptr, 0, true);
}

ct_status ct_state_flags(ct_state *s, uint8_t **flags_dev, int32_t *n_bytes) {
  if (!s || !flags_dev || !n_bytes) return fail(CT_EINVAL, "NULL argument");
  *flags_dev = s->h.sup;
  *n_bytes = s->tb->R + 1;
  return CT_OK;
}

ct_status ct_propagate_apply_async(ct_state *s, uint64_t *out_dom, uint64_t *out_pruned, int32_t *out_status) {
  if (!s) return fail(CT_EINVAL, "NULL state");
  quiesce(s);
  if (s->tb->kind == CT_TABLE_NEGATIVE) return fail(CT_EINVAL, "negative tables have no shard-local phase");
  DeviceGuard g(s->tb->device);
  CT_TRY(enqueue_finalize(s->tb, s->d_desc, 1, out_dom, out_pruned, out_status, 0, s->stream));
  s->pending = false;
  return CT_OK;
}

// ------------------------------------------------------------------ states
ct_status ct_state_clone(const ct_state *src, ct_state **out) {
  if (!src || !out) return fail(CT_EINVAL, "NULL argument");
  quiesce(src);
  if (src->pending) return fail(CT_ESTATE, "root of a caller-combined shard: combine its flags and apply first");
  ct_table *tb = src->tb;
  DeviceGuard g(tb->device);
  ct_state *s = nullptr;
  CT_TRY(new_state(tb, &s));
  s->stream = src->stream;
  const ct_status e = launch_state_copy(tb, s->mem, src->mem, s->stream);
  if (e != CT_OK) {
    free_state_mem(s);
    return e;
  }
  *out = s;
  return CT_OK;
}

ct_status ct_state_copy(ct_state *dst, const ct_state *src) {
  if (!dst || !src) return fail(CT_EINVAL, "NULL argument");
  if (dst->tb != src->tb) return fail(CT_ESTATE, "states belong to different tables");
  if (dst == src) return CT_OK;
  if (dst->serving && !src->pending) {
    // a served state restores in place (its server copies src and keeps
    // running); src's queued work first (a served src is idle between calls)
    DeviceGuard g(dst->tb->device);
    if (cudaStreamQuery(src->stream) != cudaSuccess) CUDA_TRY(cudaStreamSynchronize(src->stream));
    CT_TRY(served_call(dst, src));
    dst->pending = false;
    return CT_OK;
  }
  quiesce(dst);
  quiesce(src);
  if (src->pending) return fail(CT_ESTATE, "root of a caller-combined shard: combine its flags and apply first");
  DeviceGuard g(dst->tb->device);
  CT_TRY(order_after(dst->stream, src->stream));   // the copy reads src after its earlier work
  CT_TRY(launch_state_copy(dst->tb, dst->mem, src->mem, dst->stream));
  dst->pending = false;
  return order_after(src->stream, dst->stream);    // src's next writes wait for the copy
}

ct_status ct_state_set_stream(ct_state *s, void *stream) {
  if (!s) return fail(CT_EINVAL, "NULL state");
  if (!stream) return fail(CT_EINVAL, "stream must be a non-legacy cudaStream_t");
  quiesce(s);
  DeviceGuard g(s->tb->device);
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  s->stream = (cudaStream_t)stream;
  if (s->gexec) {
    cudaGraphExecDestroy(s->gexec);
    s->gexec = nullptr;
  }
  return CT_OK;
}

void *ct_state_stream(const ct_state *s) { return s ? (void *)s->stream : nullptr; }

ct_status ct_synchronize(ct_state *s) {
  if (!s) return fail(CT_EINVAL, "NULL state");
  DeviceGuard g(s->tb->device);
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  return CT_OK;
}

void ct_state_destroy(ct_state *s) {
  if (!s) return;
  {
    DeviceGuard g(s->tb->device);
    cudaStreamSynchronize(s->stream);
  }
  free_state_mem(s);
}

// ------------------------------------------------------------------ a10 over NVLink peer memory
static int peer_pw(const ct_table *tb) { return (int)round_up(((int64_t)tb->R + 1 + 3) / 4, 32); }

ct_status ct_peer_export(ct_table *tb, void *out_handle) {
  if (!tb || !out_handle) return fail(CT_EINVAL, "NULL argument");
  DeviceGuard g(tb->device);
  if (!tb->peer_inbox) {
    const size_t G = (size_t)std::max(tb->n_shards, 1);
    tb->peer_bytes = (2 * G * (size_t)peer_pw(tb) + 2 * G * 32 + 32) * 4;
    if (cudaMalloc(&tb->peer_inbox, tb->peer_bytes) != cudaSuccess) {
      tb->peer_inbox = nullptr;
      return fail(CT_ENOMEM, "peer inbox allocation of %zu bytes failed", tb->peer_bytes);
    }
    CUDA_TRY(cudaMemsetAsync(tb->peer_inbox, 0, tb->peer_bytes, tb->stream));   // on the table's (non-blocking) stream
    CUDA_TRY(cudaStreamSynchronize(tb->stream));   // zeroed before a peer attaches
  }
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, tb->peer_inbox));
  static_assert(sizeof h == CT_PEER_HANDLE_BYTES, "cudaIpcMemHandle_t size");
  memcpy(out_handle, &h, sizeof h);
  return CT_OK;
}

ct_status ct_peer_attach(ct_table *tb, int32_t n, const void *handles) {
  if (!tb || !handles) return fail(CT_EINVAL, "NULL argument");
  const int G = std::max(tb->n_shards, 1);
  if (n != G) return fail(CT_EINVAL, "ct_peer_attach: %d handles for %d shards", n, G);
  if (!tb->peer_inbox) return fail(CT_EINVAL, "ct_peer_attach before ct_peer_export");
  if (tb->peer_on) return fail(CT_EINVAL, "peers already attached");
  if (!tb->use_fast || tb->use_small || tb->use_wide || tb->kind == CT_TABLE_NEGATIVE)
    return fail(CT_EINVAL, "the in-kernel peer combine needs the k_fast launch shape (ct_table_info.kernel_path 2)");
  DeviceGuard dg(tb->device);
  CUDA_TRY(cudaStreamSynchronize(tb->stream));
  std::vector<uint32_t *> ptrs((size_t)G, nullptr);
  const char *hb = static_cast<const char *>(handles);
  for (int g = 0; g < G; ++g) {
    if (g == tb->rank) {
      ptrs[(size_t)g] = tb->peer_inbox;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, hb + (size_t)g * CT_PEER_HANDLE_BYTES, sizeof h);
    void *p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      for (void *q : tb->peer_opened) cudaIpcCloseMemHandle(q);
      tb->peer_opened.clear();
      return fail(CT_ECUDA, "cudaIpcOpenMemHandle of rank %d: %s", g, cudaGetErrorString(e));
    }
    tb->peer_opened.push_back(p);
    ptrs[(size_t)g] = static_cast<uint32_t *>(p);
  }
  CUDA_TRY(cudaMalloc(&tb->d_peers, (size_t)G * sizeof(uint32_t *)));
  CUDA_TRY(cudaMemcpy(tb->d_peers, ptrs.data(), (size_t)G * sizeof(uint32_t *), cudaMemcpyHostToDevice));
  const int pw = peer_pw(tb);
  tb->dev.peers = tb->d_peers;
  tb->dev.inbox = tb->peer_inbox;
  tb->dev.peer_epoch = tb->peer_inbox + 2 * (size_t)G * pw + 2 * (size_t)G * 32;
  tb->dev.peer_n = G;
  tb->dev.peer_rank = tb->rank;
  tb->dev.peer_pw = pw;
  tb->peer_on = true;
  tb->graph_gen += 1;   // every state's captured sync-call graph is re-captured with the new parameters
  return CT_OK;
}

void ct_table_destroy(ct_table *t) { free_table(t); }

// ------------------------------------------------------------------ batches
ct_status ct_batch_create(ct_table *tb, int32_t n_states, const ct_state *init, ct_batch **out) {
  if (!tb || !init || !out) return fail(CT_EINVAL, "NULL argument");
  if (init->tb != tb) return fail(CT_ESTATE, "init state belongs to another table");
  quiesce(init);
  if (n_states < 1 || n_states > 65535) return fail(CT_EINVAL, "n_states must be in [1, 65535]");
  if (tb->n_shards > 1) return fail(CT_EINVAL, "batches of sharded tables are not supported");
  if (tb->kind == CT_TABLE_NEGATIVE) return fail(CT_EINVAL, "batches of negative tables are not supported");
  DeviceGuard g(tb->device);
  ct_batch *b = new (std::nothrow) ct_batch();
  if (!b) return fail(CT_ENOMEM, "host allocation failed");
  b->tb = tb;
  b->S = n_states;
  b->bytes = tb->lay.total * (size_t)n_states;
  b->desc_bytes = sizeof(StateDev) * (size_t)n_states;
  const size_t io = (size_t)n_states * tb->Wd * 8;
  auto cleanup = [&](ct_status s) {
    if (b->mem) tb->dfree(b->mem, b->bytes);
    if (b->d_desc) tb->dfree(b->d_desc, b->desc_bytes);
    if (b->d_in) tb->dfree(b->d_in, io);
    if (b->d_dom) tb->dfree(b->d_dom, io);
    if (b->d_status) tb->dfree(b->d_status, (size_t)n_states * 4);
    if (b->d_bgo) tb->dfree(b->d_bgo, (size_t)n_states * 4);
    if (b->d_miss) tb->dfree(b->d_miss, b->miss_bytes);
    if (b->h_in) cudaFreeHost(b->h_in);
    if (b->h_dom) cudaFreeHost(b->h_dom);
    if (b->h_status) cudaFreeHost(b->h_status);
    delete b;
    return s;
  };
  b->mem = (char *)tb->dalloc(b->bytes);
  b->d_desc = (StateDev *)tb->dalloc(b->desc_bytes);
  b->d_in = (uint64_t *)tb->dalloc(io);
  b->d_dom = (uint64_t *)tb->dalloc(io);
  b->d_status = (int32_t *)tb->dalloc((size_t)n_states * 4);
  b->d_bgo = (int32_t *)tb->dalloc((size_t)n_states * 4);
  b->miss_bytes = 2 * (size_t)n_states * std::max(tb->R, 1) * sizeof(int2) + 80 + (size_t)n_states * sizeof(int2) +
                  (size_t)n_states * sizeof(int32_t);   // + the dense-state list
  b->d_miss = (int2 *)tb->dalloc(b->miss_bytes);
  if (b->d_miss && cudaMemsetAsync(b->d_miss, 0, b->miss_bytes, tb->stream) != cudaSuccess)
    return cleanup(fail(CT_ECUDA, "batch counter initialisation failed"));
  if (!b->mem || !b->d_desc || !b->d_in || !b->d_dom || !b->d_status || !b->d_bgo || !b->d_miss)
    return cleanup(fail(CT_ENOMEM, "device allocation of a %d-state batch (%zu bytes) failed", n_states, b->bytes));
  if (cudaHostAlloc((void **)&b->h_in, std::max<size_t>(io, 8), 0) != cudaSuccess ||
      cudaHostAlloc((void **)&b->h_dom, std::max<size_t>(io, 8), 0) != cudaSuccess ||
      cudaHostAlloc((void **)&b->h_status, (size_t)n_states * 4, 0) != cudaSuccess) {
    cudaGetLastError();
    return cleanup(fail(CT_ENOMEM, "pinned host allocation failed"));
  }
  b->h.resize(n_states);
  for (int i = 0; i < n_states; ++i) b->h[i] = make_desc(tb, b->mem + (size_t)i * tb->lay.total);
  {
    const StateLayout &L = tb->lay;
    BatchDev &bd = b->bd;
    bd.pool = b->mem;
    bd.pitch = (int64_t)L.total;
    bd.o_ctl = (int64_t)L.ctl;
    bd.o_T = (int64_t)L.T;
    bd.o_ulist = (int64_t)L.ulist;
    bd.o_items = (int64_t)L.items;
    bd.o_res = (int64_t)L.res;
    bd.o_sup = (int64_t)L.sup;
    bd.o_scan = (int64_t)L.scanlist;
    bd.o_idx0 = (int64_t)L.idx0;
    bd.o_idx1 = (int64_t)L.idx1;
    bd.o_bmask = (int64_t)L.bmask;
    bd.o_plist = (int64_t)L.plist;
    bd.plist_po = plist_po(tb->n);
    bd.bgo = b->d_bgo;
    const size_t nm = (size_t)n_states * std::max(tb->R, 1);
    bd.miss = b->d_miss;
    bd.miss2 = b->d_miss + nm;
    bd.nmiss = reinterpret_cast<int32_t *>(b->d_miss + 2 * nm);
    bd.nmiss2 = bd.nmiss + 1;
    bd.ndense = bd.nmiss + 2;                                                     // zeroed with the region
    bd.work = reinterpret_cast<unsigned long long *>(b->d_miss + 2 * nm + 2);   // 16-byte aligned
    bd.sinfo = b->d_miss + 2 * nm + 10;                                           // after work[8]
    bd.dense = reinterpret_cast<int32_t *>(bd.sinfo + n_states);
    bd.t_local = tb->t_local;
    bd.cell_route = tb->bt_cells;
  }
  if (cudaMemcpyAsync(b->d_desc, b->h.data(), b->desc_bytes, cudaMemcpyHostToDevice, tb->stream) != cudaSuccess)
    return cleanup(fail(CT_ECUDA, "descriptor upload failed"));
  if (init->pending) return cleanup(fail(CT_ESTATE, "init state is a pending shard root"));
  if (order_after(tb->stream, init->stream) != CT_OK) return cleanup(CT_ECUDA);
  // per-call scratch starts zeroed, as for single states
  if (cudaMemsetAsync(b->mem, 0, b->bytes, tb->stream) != cudaSuccess) return cleanup(fail(CT_ECUDA, "batch memset failed"));
  for (int i = 0; i < n_states; ++i)
    if (cudaMemcpyAsync(b->mem + (size_t)i * tb->lay.total, init->mem, tb->lay.persist, cudaMemcpyDeviceToDevice,
                        tb->stream) != cudaSuccess)
      return cleanup(fail(CT_ECUDA, "batch init copy failed"));
  if (order_after(init->stream, tb->stream) != CT_OK) return cleanup(CT_ECUDA);
  tb->live++;
  *out = b;
  return CT_OK;
}

int32_t ct_batch_size(const ct_batch *b) { return b ? b->S : -1; }

ct_status ct_batch_copy(ct_batch *b, int32_t i, const ct_state *src) {
  if (!b || !src) return fail(CT_EINVAL, "NULL argument");
  quiesce(src);
  if (src->tb != b->tb) return fail(CT_ESTATE, "state belongs to another table");
  if (i < 0 || i >= b->S) return fail(CT_EINVAL, "batch index %d out of range", i);
  if (src->pending) return fail(CT_ESTATE, "src is a pending shard root");
  DeviceGuard g(b->tb->device);
  CT_TRY(order_after(b->tb->stream, src->stream));
  CUDA_TRY(cudaMemcpyAsync(b->mem + (size_t)i * b->tb->lay.total, src->mem, b->tb->lay.persist,
                           cudaMemcpyDeviceToDevice, b->tb->stream));
  return order_after(src->stream, b->tb->stream);
}

ct_status ct_batch_copy_all(ct_batch *b, const ct_state *src) {
  if (!b || !src) return fail(CT_EINVAL, "NULL argument");
  quiesce(src);
  if (src->tb != b->tb) return fail(CT_ESTATE, "state belongs to another table");
  if (src->pending) return fail(CT_ESTATE, "src is a pending shard root");
  DeviceGuard g(b->tb->device);
  CT_TRY(order_after(b->tb->stream, src->stream));
  const size_t pitch = b->tb->lay.total;
  CUDA_TRY(cudaMemcpy2DAsync(b->mem, pitch, src->mem, 0, b->tb->lay.persist, (size_t)b->S,
                             cudaMemcpyDeviceToDevice, b->tb->stream));
  return order_after(src->stream, b->tb->stream);
}

ct_status ct_batch_restore_dead(ct_batch *b, const ct_state *src) {
  if (!b || !src) return fail(CT_EINVAL, "NULL argument");
  quiesce(src);
  if (src->tb != b->tb) return fail(CT_ESTATE, "state belongs to another table");
  if (src->pending) return fail(CT_ESTATE, "src is a pending shard root");
  DeviceGuard g(b->tb->device);
  CT_TRY(order_after(b->tb->stream, src->stream));
  k_restore_dead<<<b->S, 256, 0, b->tb->stream>>>(b->mem, b->tb->lay.total, src->mem, copy_layout(b->tb));
  CUDA_TRY(cudaGetLastError());
  return order_after(src->stream, b->tb->stream);
}

// Tile-major batch call (ct_batch.cuh): ingest, update, probe, scan, finalize.
static ct_status enqueue_batch_tiled(ct_batch *b, const uint64_t *removed, uint64_t *out_dom, int32_t *out_status) {
  ct_table *tb = b->tb;
  cudaStream_t st = tb->stream;
  const int S = b->S;
  int e = prof_event(tb, st);
  k_bingest<<<S, kBSmallTPB, ingest_smem_bytes(tb->n, tb->Wd), st>>>(tb->dev, b->d_desc, removed, tb->Wd, b->bd,
                                                                     tb->bt_tw == 32 ? 1 : 0);
  prof_mark(tb, 0, e, st);
  const int tw = tb->bt_tw;
  const int ntiles = (int)((tb->dev.W2 + tw - 1) / tw);
  const int G = tb->bt_grid;
  const int spw = 32 / tw;
  // units = tiles x state chunks: >= 16 per CTA for balance, chunks of at least
  // 4 states per warp slot so every warp of a CTA has work
  int nchunk = std::max(1, (16 * G + ntiles - 1) / std::max(ntiles, 1));
  const int min_chunk = 4 * (kBTPB / 32) * spw;
  nchunk = std::max(1, std::min(nchunk, (S + min_chunk - 1) / min_chunk));
  const int chunk_states = (S + nchunk - 1) / nchunk;
  nchunk = (S + chunk_states - 1) / chunk_states;
  e = prof_event(tb, st);
  if (ntiles > 0) {
    if (tw == 32)
      k_bupdate<32><<<G, kBTPB, tb->bt_smem, st>>>(tb->dev, b->bd, S, ntiles, nchunk, chunk_states);
    else if (tw == 16)
      k_bupdate<16><<<G, kBTPB, tb->bt_smem, st>>>(tb->dev, b->bd, S, ntiles, nchunk, chunk_states);
    else
      k_bupdate<8><<<G, kBTPB, tb->bt_smem, st>>>(tb->dev, b->bd, S, ntiles, nchunk, chunk_states);
  }
  k_bcompact<<<S, kBSmallTPB, 0, st>>>(tb->dev, b->bd);
  if (tb->bt_cells) k_bsparse<<<S, kBSparseTPB, 0, st>>>(tb->dev, b->bd);
  prof_mark(tb, 1, e, st);
  e = prof_event(tb, st);
  const int64_t pth = (int64_t)S * std::max(tb->R, 1);
  k_bprobe<<<(unsigned)((pth + kBProbeTPB - 1) / kBProbeTPB), kBProbeTPB, 0, st>>>(tb->dev, b->bd, S);
  prof_mark(tb, 2, e, st);
  e = prof_event(tb, st);
  k_bscan<<<tb->sm_count * 16, kBScanTPB, 0, st>>>(tb->dev, b->bd, 0);
  k_bscan<<<tb->sm_count * 8, kBScanTPB, 0, st>>>(tb->dev, b->bd, 1);
  prof_mark(tb, 3, e, st);
  e = prof_event(tb, st);
  k_bfinalize<<<S, kBSmallTPB, finalize_smem_bytes(tb->n, tb->Wd), st>>>(tb->dev, b->d_desc, out_dom, tb->Wd,
                                                                         out_status, b->bd);
  prof_mark(tb, 5, e, st);
  CUDA_TRY(cudaGetLastError());
  return CT_OK;
}

ct_status ct_propagate_many_async(ct_batch *b, const uint64_t *removed, uint64_t *out_dom, int32_t *out_status) {
  if (!b) return fail(CT_EINVAL, "NULL batch");
  ct_table *tb = b->tb;
  DeviceGuard g(tb->device);
  if (tb->bt_tw) return enqueue_batch_tiled(b, removed, out_dom, out_status);
  CT_TRY(enqueue_local(tb, b->d_desc, b->S, removed, 0, tb->stream));
  return enqueue_finalize(tb, b->d_desc, b->S, out_dom, nullptr, out_status, 0, tb->stream);
}

ct_status ct_propagate_many(ct_batch *b, const uint64_t *removed, uint64_t *out_dom, int32_t *out_status) {
  if (!b || !out_status) return fail(CT_EINVAL, "NULL argument");
  ct_table *tb = b->tb;
  DeviceGuard g(tb->device);
  const size_t io = (size_t)b->S * tb->Wd * 8;
  if (io) {
    if (removed) memcpy(b->h_in, removed, io);
    else memset(b->h_in, 0, io);
    CUDA_TRY(cudaMemcpyAsync(b->d_in, b->h_in, io, cudaMemcpyHostToDevice, tb->stream));
  }
  CT_TRY(ct_propagate_many_async(b, b->d_in, b->d_dom, b->d_status));
  if (io) CUDA_TRY(cudaMemcpyAsync(b->h_dom, b->d_dom, io, cudaMemcpyDeviceToHost, tb->stream));
  CUDA_TRY(cudaMemcpyAsync(b->h_status, b->d_status, (size_t)b->S * 4, cudaMemcpyDeviceToHost, tb->stream));
  CUDA_TRY(cudaStreamSynchronize(tb->stream));
  memcpy(out_status, b->h_status, (size_t)b->S * 4);
  if (out_dom && io) {
    // outputs are written for CT_OK states only (include/ct.h)
    for (int i = 0; i < b->S; ++i)
      if (b->h_status[i] == CT_OK)
        memcpy(out_dom + (size_t)i * tb->Wd, b->h_dom + (size_t)i * tb->Wd, (size_t)tb->Wd * 8);
  }
  return CT_OK;
}

void ct_batch_destroy(ct_batch *b) {
  if (!b) return;
  ct_table *tb = b->tb;
  DeviceGuard g(tb->device);
  cudaStreamSynchronize(tb->stream);
  const size_t io = (size_t)b->S * tb->Wd * 8;
  tb->dfree(b->mem, b->bytes);
  tb->dfree(b->d_desc, b->desc_bytes);
  tb->dfree(b->d_in, io);
  tb->dfree(b->d_dom, io);
  tb->dfree(b->d_status, (size_t)b->S * 4);
  tb->dfree(b->d_bgo, (size_t)b->S * 4);
  tb->dfree(b->d_miss, b->miss_bytes);
  cudaFreeHost(b->h_in);
  cudaFreeHost(b->h_dom);
  cudaFreeHost(b->h_status);
  tb->live--;
  delete b;
}

// ------------------------------------------------------------------ introspection
ct_status ct_state_read_table(const ct_state *s, uint64_t *out_bits) {
  if (!s || !out_bits) return fail(CT_EINVAL, "NULL argument");
  DeviceGuard g(s->tb->device);
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  if (s->tb->W) CUDA_TRY(cudaMemcpy(out_bits, s->h.T, (size_t)s->tb->W * 8, cudaMemcpyDeviceToHost));
  return CT_OK;
}

ct_status ct_batch_work(ct_batch *b, int64_t *out10, int32_t reset) {
  int64_t *out8 = out10;
  if (!b || !out10) return fail(CT_EINVAL, "NULL argument");
  DeviceGuard g(b->tb->device);
  CUDA_TRY(cudaStreamSynchronize(b->tb->stream));
  int64_t *out6 = out8;
  for (int i = 0; i < 10; ++i) out8[i] = -1;
  if (!b->tb->bt_tw) return CT_OK;
  int64_t w7[7];
  CUDA_TRY(cudaMemcpy(w7, b->bd.work, 7 * sizeof(int64_t), cudaMemcpyDeviceToHost));
  for (int i = 0; i < 4; ++i) out8[i] = w7[i];
  out8[6] = w7[4];
  out8[7] = w7[5];
  out8[8] = w7[6];
  out8[9] = 0;
  if (reset) {   // ordered before the next batch call's kernels on the table's stream
    CUDA_TRY(cudaMemsetAsync(b->bd.work, 0, 7 * sizeof(int64_t), b->tb->stream));
    CUDA_TRY(cudaStreamSynchronize(b->tb->stream));
  }
  // filter side of the last call: summed over the states' own counters
  std::vector<Ctl> c((size_t)b->S);
  CUDA_TRY(cudaMemcpy2D(c.data(), sizeof(Ctl), b->mem + b->tb->lay.ctl, b->tb->lay.total, sizeof(Ctl), (size_t)b->S,
                        cudaMemcpyDeviceToHost));
  std::vector<int32_t> bgo((size_t)b->S);
  CUDA_TRY(cudaMemcpy(bgo.data(), b->d_bgo, (size_t)b->S * 4, cudaMemcpyDeviceToHost));
  out6[4] = out6[5] = 0;
  for (int i = 0; i < b->S; ++i) {
    if (bgo[(size_t)i] < 0) continue;   // the state did not run the filter in the last call
    out6[4] += (int64_t)c[(size_t)i].scan_loads;
    out6[5] += c[(size_t)i].nscan;
  }
  return CT_OK;
}

ct_status ct_batch_read_table(const ct_batch *b, int32_t i, uint64_t *out_bits) {
  if (!b || !out_bits) return fail(CT_EINVAL, "NULL argument");
  if (i < 0 || i >= b->S) return fail(CT_EINVAL, "batch index %d out of range", i);
  DeviceGuard g(b->tb->device);
  CUDA_TRY(cudaStreamSynchronize(b->tb->stream));
  if (b->tb->W) CUDA_TRY(cudaMemcpy(out_bits, b->h[(size_t)i].T, (size_t)b->tb->W * 8, cudaMemcpyDeviceToHost));
  return CT_OK;
}

ct_status ct_table_read_supports(const ct_table *t, int32_t row, uint64_t *out_bits) {
  if (!t || !out_bits) return fail(CT_EINVAL, "NULL argument");
  if (row < 0 || row >= t->R) return fail(CT_EINVAL, "row %d out of range", row);
  DeviceGuard g(t->device);
  CUDA_TRY(cudaStreamSynchronize(t->stream));
  if (t->W) CUDA_TRY(cudaMemcpy(out_bits, t->S + (size_t)row * t->Wp, (size_t)t->W * 8, cudaMemcpyDeviceToHost));
  return CT_OK;
}

ct_status ct_state_read_dom(const ct_state *s, uint64_t *out_dom) {
  if (!s || !out_dom) return fail(CT_EINVAL, "NULL argument");
  DeviceGuard g(s->tb->device);
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  if (s->tb->Wd) CUDA_TRY(cudaMemcpy(out_dom, s->h.dom, (size_t)s->tb->Wd * 8, cudaMemcpyDeviceToHost));
  return CT_OK;
}

static void stats_from_ctl(const Ctl &c, ct_stats *o) {
  memset(o, 0, sizeof *o);
  o->calls = c.calls;
  o->last_status = c.last_status;
  o->noop = c.noop;
  o->n_changed = c.ngroups;
  o->n_update_rows = c.nrows;
  o->n_filter_items = c.nitems;
  o->n_residue_miss = c.nscan;
  o->words_in = c.L_in;
  o->words_out = c.L_out;
  o->update_support_words = (int64_t)c.upd_loads;
  o->update_table_writes = (int64_t)c.upd_writes;
  o->filter_support_words = (int64_t)c.scan_loads;
  o->filter_gathered_tuples = (int64_t)c.gathered;
  for (int i = 0; i < 7; ++i) o->phase_ns[i] = (c.tph[0] && c.tph[i + 1] >= c.tph[i]) ? (int64_t)(c.tph[i + 1] - c.tph[i]) : 0;
}

ct_status ct_state_stats(const ct_state *s, ct_stats *o) {
  if (!s || !o) return fail(CT_EINVAL, "NULL argument");
  DeviceGuard g(s->tb->device);
  CUDA_TRY(cudaStreamSynchronize(s->stream));
  Ctl c;
  CUDA_TRY(cudaMemcpy(&c, s->h.ctl, sizeof c, cudaMemcpyDeviceToHost));
  stats_from_ctl(c, o);
  return CT_OK;
}

ct_status ct_batch_stats(const ct_batch *b, ct_stats *o) {
  if (!b || !o) return fail(CT_EINVAL, "NULL argument");
  DeviceGuard g(b->tb->device);
  CUDA_TRY(cudaStreamSynchronize(b->tb->stream));
  std::vector<Ctl> c((size_t)b->S);
  CUDA_TRY(cudaMemcpy2D(c.data(), sizeof(Ctl), b->mem + b->tb->lay.ctl, b->tb->lay.total, sizeof(Ctl), (size_t)b->S,
                        cudaMemcpyDeviceToHost));
  for (int i = 0; i < b->S; ++i) stats_from_ctl(c[(size_t)i], o + i);
  return CT_OK;
}

ct_status ct_table_profile(ct_table *t, int32_t enable) {
  if (!t) return fail(CT_EINVAL, "NULL table");
  t->prof_on = enable != 0;
  return CT_OK;
}

ct_status ct_table_profile_read(ct_table *t, ct_kernel_times *out, int32_t reset) {
  if (!t || !out) return fail(CT_EINVAL, "NULL argument");
  DeviceGuard g(t->device);
  memset(out, 0, sizeof *out);
  CUDA_TRY(cudaDeviceSynchronize());
  for (const auto &m : t->marks) {
    float ms = 0.f;
    CUDA_TRY(cudaEventElapsedTime(&ms, t->ev_pool[m.e0], t->ev_pool[m.e1]));
    out->launches[m.kid] += 1;
    out->ms[m.kid] += ms;
  }
  if (reset) {
    t->marks.clear();
    t->ev_used = 0;
  }
  return CT_OK;
}

}  // extern "C"

// ================================================================== models (f1)
struct ct_model {
  int device = 0;
  int search_levels = 0;   // ct_config.search_levels
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int nv = 0, ntab = 0, Wg = 0;
  std::vector<int32_t> vlo, vd, gOff;
  std::vector<ct_table *> tabs;
  std::vector<size_t> off;        // table k's state block inside the pool
  char *pool = nullptr;           // all table states + shared domains (snapshot unit)
  size_t pool_bytes = 0, gdom_off = 0;
  char *meta = nullptr;           // TableDev[ntab] | StateDev[ntab] | ModelCtl | gword arrays
  size_t meta_bytes = 0;
  ModelDev md{};
  uint64_t *h_in = nullptr, *h_out = nullptr, *d_in = nullptr, *d_out = nullptr;   // mapped pinned
  int grid = 1;
  size_t smem = 0;
  std::vector<char *> snaps;      // device snapshot buffers, one per trail level
  std::vector<std::vector<uint64_t>> mirrors;
  int depth = 0;
  bool dead = false;
  std::vector<uint64_t> dom;      // host mirror of the shared domains
  // last fixpoint's counters
  int64_t last_iters = 0, last_calls = 0, last_ns = 0;
  // device-resident search (k_model_search), set up on first use
  uint4 *snap_dev = nullptr;
  int levels = 0;
  int32_t *d_goff = nullptr, *d_vlo = nullptr;
  long long *h_sout = nullptr, *d_sout = nullptr;   // mapped [16 + nv]
  int sgrid = 0;
  size_t ssmem = 0;
};

static void model_free(ct_model *m) {
  if (!m) return;
  DeviceGuard g(m->device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  for (char *sn : m->snaps) cudaFree(sn);
  if (m->snap_dev) cudaFree(m->snap_dev);
  if (m->d_goff) cudaFree(m->d_goff);
  if (m->h_sout) cudaFreeHost(m->h_sout);
  if (m->pool) cudaFree(m->pool);
  if (m->meta) cudaFree(m->meta);
  if (m->h_in) cudaFreeHost(m->h_in);
  if (m->h_out) cudaFreeHost(m->h_out);
  for (ct_table *t : m->tabs) free_table(t);
  if (m->own_stream && m->stream) cudaStreamDestroy(m->stream);
  delete m;
}

static ct_status model_launch(ct_model *m, bool with_input) {
  *(volatile int32_t *)m->h_out = kPendingStatus;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)m->grid);
  lc.blockDim = dim3(kFusedTPB);
  lc.dynamicSmemBytes = m->smem;
  lc.stream = m->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&lc, k_model_fixpoint, m->md, (const uint64_t *)(with_input ? m->d_in : nullptr),
                              m->d_out, 1 << 20));
  volatile int32_t *st = (volatile int32_t *)m->h_out;
  for (uint64_t spin = 1;; ++spin) {
    if (*st != kPendingStatus) break;
    if ((spin & 1023) == 0) {
      const cudaError_t e = cudaStreamQuery(m->stream);
      if (e == cudaSuccess && *st == kPendingStatus) return fail(CT_ECUDA, "model fixpoint ended without a status");
      if (e != cudaSuccess && e != cudaErrorNotReady)
        return fail(CT_ECUDA, "model fixpoint failed: %s", cudaGetErrorString(e));
    }
  }
  const int32_t status = *st;
  m->last_iters = (int64_t)m->h_out[1];
  m->last_calls = (int64_t)m->h_out[2];
  m->last_ns = (int64_t)m->h_out[3];
  if (status == 0) {
    memcpy(m->dom.data(), m->h_out + 4, (size_t)m->Wg * 8);
    return CT_OK;
  }
  m->dead = true;
  return CT_FAIL;
}

extern "C" {

ct_status ct_model_create(int32_t n_vars, const int32_t *var_lo, const int32_t *var_size, int32_t n_tables,
                          const int32_t *arity, const int32_t *scopes, const int64_t *n_tuples,
                          const int32_t *const *tuples, const ct_config *cfg_in, ct_model **out,
                          uint64_t *out_dom) {
  if (!out) return fail(CT_EINVAL, "out is NULL");
  *out = nullptr;
  if (n_vars < 1 || !var_lo || !var_size) return fail(CT_EINVAL, "bad variables");
  if (n_tables < 1 || n_tables > kMaxModelTables) return fail(CT_EINVAL, "n_tables must be in [1, %d]", kMaxModelTables);
  if (!arity || !scopes || !n_tuples || !tuples) return fail(CT_EINVAL, "NULL table arrays");
  ct_config cfg;
  if (cfg_in) cfg = *cfg_in;
  else ct_config_init(&cfg);
  if (cfg.n_shards != 1) return fail(CT_EINVAL, "models of sharded tables are not supported");
  ct_model *m = new (std::nothrow) ct_model();
  if (!m) return fail(CT_ENOMEM, "host allocation failed");
  auto bail = [&](ct_status s) {
    model_free(m);
    return s;
  };
  m->device = cfg.device;
  m->search_levels = cfg.search_levels;
  m->nv = n_vars;
  m->ntab = n_tables;
  m->vlo.assign(var_lo, var_lo + n_vars);
  m->vd.assign(var_size, var_size + n_vars);
  m->gOff.assign(n_vars + 1, 0);
  for (int v = 0; v < n_vars; ++v) {
    if (var_size[v] < 1) return bail(fail(CT_EINVAL, "var_size[%d] must be >= 1", v));
    m->gOff[v + 1] = m->gOff[v] + (var_size[v] + 63) / 64;
  }
  m->Wg = m->gOff[n_vars];
  DeviceGuard g(m->device);
  if (cfg.stream) {
    m->stream = (cudaStream_t)cfg.stream;
  } else {
    if (cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking) != cudaSuccess)
      return bail(fail(CT_ECUDA, "stream creation failed"));
    m->own_stream = true;
  }
  cfg.stream = m->stream;
  cfg.use_graph = 0;
  cfg.alloc = nullptr;   // the model owns its memory (plain cudaMalloc)
  const int model_grid = cfg.grid_override;
  cfg.grid_override = 0;   // the model's grid, not the tables'
  // ---- tables (each built and propagated at its own root)
  std::vector<uint64_t> gdom(m->Wg, 0ull);
  for (int v = 0; v < n_vars; ++v)
    for (int a = 0; a < var_size[v]; ++a) gdom[m->gOff[v] + a / 64] |= 1ull << (a % 64);
  std::vector<ct_state *> roots;
  bool root_fail = false;
  const int32_t *sc = scopes;
  for (int k = 0; k < n_tables; ++k) {
    const int n = arity[k];
    if (n < 1) return bail(fail(CT_EINVAL, "arity[%d] must be >= 1", k));
    std::vector<int32_t> lo(n), d(n);
    for (int i = 0; i < n; ++i) {
      if (sc[i] < 0 || sc[i] >= n_vars) return bail(fail(CT_EINVAL, "scope of table %d names var %d", k, sc[i]));
      lo[i] = var_lo[sc[i]];
      d[i] = var_size[sc[i]];
    }
    ct_table *t = nullptr;
    ct_state *r = nullptr;
    ct_status s = ct_create(n, sc, lo.data(), d.data(), nullptr, n_tuples[k], tuples[k], &cfg, &t, &r, nullptr);
    if (s < 0) {
      for (ct_state *x : roots) free_state_mem(x);
      return bail(s);
    }
    m->tabs.push_back(t);
    roots.push_back(r);
    if (s == CT_FAIL) root_fail = true;
    sc += n;
  }
  // ---- pool: every table state + the shared domains
  size_t o = 0;
  for (int k = 0; k < n_tables; ++k) {
    m->off.push_back(o);
    o += (size_t)round_up((int64_t)m->tabs[k]->lay.total, 256);
  }
  m->gdom_off = o;
  o += (size_t)round_up((int64_t)m->Wg * 8, 256);
  m->pool_bytes = o;
  if (cudaMalloc(&m->pool, m->pool_bytes) != cudaSuccess) {
    for (ct_state *x : roots) free_state_mem(x);
    return bail(fail(CT_ENOMEM, "model pool allocation failed"));
  }
  cudaMemsetAsync(m->pool, 0, m->pool_bytes, m->stream);   // scratch too: trail snapshots copy whole states
  for (int k = 0; k < n_tables; ++k) {
    cudaMemcpyAsync(m->pool + m->off[k], roots[k]->mem, m->tabs[k]->lay.persist, cudaMemcpyDeviceToDevice, m->stream);
  }
  cudaStreamSynchronize(m->stream);
  // root domains of each table -> shared domains
  sc = scopes;
  for (int k = 0; k < n_tables; ++k) {
    ct_table *t = m->tabs[k];
    std::vector<uint64_t> rd(std::max(t->Wd, 1));
    if (!root_fail) {
      if (ct_state_read_dom(roots[k], rd.data()) != CT_OK) {
        for (ct_state *x : roots) free_state_mem(x);
        return bail(CT_ECUDA);
      }
      for (int i = 0; i < t->n; ++i)
        for (int w = t->domOff[i]; w < t->domOff[i + 1]; ++w) gdom[m->gOff[sc[i]] + (w - t->domOff[i])] &= rd[w];
    }
    sc += t->n;
  }
  for (ct_state *x : roots) free_state_mem(x);
  // ---- device metadata
  const size_t tdev = sizeof(TableDev) * n_tables, sdev = sizeof(StateDev) * n_tables;
  size_t gw_total = 0;
  for (ct_table *t : m->tabs) gw_total += (size_t)std::max(t->Wd, 1);
  m->meta_bytes = (size_t)round_up((int64_t)(tdev + sdev), 256) + 256 + 2 * round_up((int64_t)gw_total * 4, 256) +
                  (size_t)kBarWords * 4;
  if (cudaMalloc(&m->meta, m->meta_bytes) != cudaSuccess) return bail(fail(CT_ENOMEM, "model metadata allocation failed"));
  if (cudaMemsetAsync(m->meta, 0, m->meta_bytes, m->stream) != cudaSuccess)
    return bail(fail(CT_ECUDA, "model metadata memset failed"));
  // the pool and metadata memsets (m->stream, non-blocking) finish before the
  // synchronous uploads below write into them
  if (cudaStreamSynchronize(m->stream) != cudaSuccess) return bail(fail(CT_ECUDA, "model stream sync failed"));
  TableDev *d_tabs = (TableDev *)m->meta;
  StateDev *d_sts = (StateDev *)(m->meta + tdev);
  ModelCtl *d_mc = (ModelCtl *)(m->meta + round_up((int64_t)(tdev + sdev), 256));
  int32_t *d_gw = (int32_t *)((char *)d_mc + 256);
  int32_t *d_gs = (int32_t *)((char *)d_gw + round_up((int64_t)gw_total * 4, 256));
  std::vector<int32_t> var_uses(n_vars, 0);   // scope positions per variable over all tables
  sc = scopes;
  for (int k = 0; k < n_tables; ++k) {
    for (int i = 0; i < m->tabs[k]->n; ++i) var_uses[sc[i]]++;
    sc += m->tabs[k]->n;
  }
  std::vector<TableDev> htabs(n_tables);
  std::vector<StateDev> hsts(n_tables);
  sc = scopes;
  size_t gpos = 0;
  for (int k = 0; k < n_tables; ++k) {
    ct_table *t = m->tabs[k];
    std::vector<int32_t> gw(std::max(t->Wd, 1), 0), gs(std::max(t->Wd, 1), 0);
    for (int i = 0; i < t->n; ++i)
      for (int w = t->domOff[i]; w < t->domOff[i + 1]; ++w) {
        gw[w] = m->gOff[sc[i]] + (w - t->domOff[i]);
        gs[w] = var_uses[sc[i]] > 1;
      }
    cudaMemcpy(d_gw + gpos, gw.data(), gw.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(d_gs + gpos, gs.data(), gs.size() * 4, cudaMemcpyHostToDevice);
    htabs[k] = t->dev;
    htabs[k].gword = d_gw + gpos;
    htabs[k].gshared = d_gs + gpos;
    hsts[k] = make_desc(t, m->pool + m->off[k]);
    gpos += gw.size();
    sc += t->n;
  }
  cudaMemcpy(d_tabs, htabs.data(), tdev, cudaMemcpyHostToDevice);
  cudaMemcpy(d_sts, hsts.data(), sdev, cudaMemcpyHostToDevice);
  cudaMemcpy(m->pool + m->gdom_off, gdom.data(), (size_t)m->Wg * 8, cudaMemcpyHostToDevice);
  m->md.ntab = n_tables;
  m->md.Wg = m->Wg;
  m->md.tabs = d_tabs;
  m->md.sts = d_sts;
  m->md.gdom = (uint64_t *)(m->pool + m->gdom_off);
  m->md.mc = d_mc;
  m->md.bar = (uint32_t *)((char *)d_gs + round_up((int64_t)gw_total * 4, 256));
  m->dom = gdom;
  // ---- launch geometry
  size_t smem = 0;
  int tiles = 0;
  for (ct_table *t : m->tabs) {
    smem = std::max({smem, ingest_smem_bytes(t->n, t->Wd), finalize_smem_bytes(t->n, t->Wd)});
    tiles += t->dev.ntiles_max;
  }
  m->smem = smem;
  CUDA_TRY(cudaFuncSetAttribute(k_model_fixpoint, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)std::max<size_t>(smem, 1)));
  int occ = 0, sms = 148;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_model_fixpoint, kFusedTPB, smem));
  CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device));
  if (occ < 1) return bail(fail(CT_EINVAL, "model kernel does not fit on an SM"));
  // one CTA per SM: the fixpoint is latency-bound (several grid barriers per
  // Jacobi round, per-table ingest / finalize by one CTA each), and a barrier
  // over 148 arrivals is ~2 us cheaper than over 444 (C5: 82 -> 72 us/node)
  (void)tiles;
  m->grid = sms;
  if (model_grid > 0) m->grid = std::max(1, std::min(sms * occ, model_grid));
  if (cudaHostAlloc((void **)&m->h_in, (size_t)std::max(m->Wg, 1) * 8, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostAlloc((void **)&m->h_out, (size_t)(4 + m->Wg) * 8, cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer((void **)&m->d_in, m->h_in, 0) != cudaSuccess ||
      cudaHostGetDevicePointer((void **)&m->d_out, m->h_out, 0) != cudaSuccess)
    return bail(fail(CT_ENOMEM, "mapped pinned allocation failed"));
  *out = m;
  if (root_fail) {
    m->dead = true;
    return CT_FAIL;
  }
  ct_status s = model_launch(m, false);
  if (s < 0) {
    *out = nullptr;
    return bail(s);
  }
  if (s == CT_OK && out_dom) memcpy(out_dom, m->dom.data(), (size_t)m->Wg * 8);
  return s;
}

int32_t ct_model_dom_words(const ct_model *m) { return m ? m->Wg : -1; }
int32_t ct_model_dom_word_offset(const ct_model *m, int32_t v) {
  if (!m || v < 0 || v >= m->nv) return -1;
  return m->gOff[v];
}

ct_status ct_model_fixpoint(ct_model *m, const uint64_t *dom_in, uint64_t *out_dom) {
  if (!m) return fail(CT_EINVAL, "NULL model");
  if (m->dead) return fail(CT_ESTATE, "model is dead (last fixpoint failed); ct_model_pop restores it");
  DeviceGuard g(m->device);
  if (dom_in)
    for (int w = 0; w < m->Wg; ++w) m->h_in[w] = m->dom[w] & dom_in[w];
  const ct_status s = model_launch(m, dom_in != nullptr);
  if (s == CT_OK && out_dom) memcpy(out_dom, m->dom.data(), (size_t)m->Wg * 8);
  return s;
}

ct_status ct_model_push(ct_model *m) {
  if (!m) return fail(CT_EINVAL, "NULL model");
  DeviceGuard g(m->device);
  if ((int)m->snaps.size() <= m->depth) {
    char *p = nullptr;
    if (cudaMalloc(&p, m->pool_bytes) != cudaSuccess) return fail(CT_ENOMEM, "snapshot allocation failed");
    m->snaps.push_back(p);
  }
  CUDA_TRY(cudaMemcpyAsync(m->snaps[m->depth], m->pool, m->pool_bytes, cudaMemcpyDeviceToDevice, m->stream));
  if ((int)m->mirrors.size() <= m->depth) m->mirrors.emplace_back();
  m->mirrors[m->depth] = m->dom;
  m->depth++;
  return CT_OK;
}

ct_status ct_model_pop(ct_model *m) {
  if (!m) return fail(CT_EINVAL, "NULL model");
  if (m->depth == 0) return fail(CT_EINVAL, "ct_model_pop without a matching push");
  DeviceGuard g(m->device);
  m->depth--;
  CUDA_TRY(cudaMemcpyAsync(m->pool, m->snaps[m->depth], m->pool_bytes, cudaMemcpyDeviceToDevice, m->stream));
  m->dom = m->mirrors[m->depth];
  m->dead = false;
  return CT_OK;
}

namespace {
struct Dfs {
  ct_model *m;
  int value_order;
  int64_t max_nodes, max_solutions;
  ct_search_stats st{};
  std::vector<int32_t> sol;
  bool stop = false;
  ct_status err = CT_OK;

  void hash(uint64_t x) {
    for (int i = 0; i < 8; ++i) {
      st.trace_hash ^= (x >> (8 * i)) & 0xff;
      st.trace_hash *= 1099511628211ull;
    }
  }
  void account(int depth, int var, int val, int branch, ct_status s) {
    st.nodes++;
    if (s == CT_FAIL) st.failures++;
    st.table_calls += m->last_calls;
    st.iterations += m->last_iters;
    st.device_ms += m->last_ns * 1e-6;
    if (depth > st.max_depth) st.max_depth = depth;
    hash((uint64_t)depth);
    hash((uint64_t)(int64_t)var);
    hash((uint64_t)(int64_t)val);
    hash((uint64_t)branch);
    hash((uint64_t)s);
  }
  // the model is at an OK fixpoint here
  void node(int depth) {
    if (stop) return;
    int x = -1;   // input_order: the lowest-index unbound variable
    for (int v = 0; v < m->nv && x < 0; ++v) {
      int c = 0;
      for (int w = m->gOff[v]; w < m->gOff[v + 1]; ++w) c += __builtin_popcountll(m->dom[w]);
      if (c > 1) x = v;
    }
    if (x < 0) {   // every variable bound: a solution
      st.solutions++;
      for (int v = 0; v < m->nv; ++v) {
        int a = 0;
        for (int w = m->gOff[v]; w < m->gOff[v + 1]; ++w)
          if (m->dom[w]) a = (w - m->gOff[v]) * 64 + __builtin_ctzll(m->dom[w]);
        sol[v] = m->vlo[v] + a;
      }
      if (max_solutions > 0 && st.solutions >= max_solutions) stop = true;
      return;
    }
    // value: indomain_max (0) or indomain_min (1)
    int a = -1;
    if (value_order == 0) {
      for (int w = m->gOff[x + 1] - 1; w >= m->gOff[x] && a < 0; --w)
        if (m->dom[w]) a = (w - m->gOff[x]) * 64 + 63 - __builtin_clzll(m->dom[w]);
    } else {
      for (int w = m->gOff[x]; w < m->gOff[x + 1] && a < 0; ++w)
        if (m->dom[w]) a = (w - m->gOff[x]) * 64 + __builtin_ctzll(m->dom[w]);
    }
    const int val = m->vlo[x] + a;
    const int wa = m->gOff[x] + a / 64;
    const uint64_t bit = 1ull << (a % 64);
    for (int branch = 0; branch < 2 && !stop; ++branch) {
      if (max_nodes > 0 && st.nodes >= max_nodes) {
        stop = true;
        return;
      }
      ct_status s = ct_model_push(m);
      if (s < 0) {
        err = s;
        stop = true;
        return;
      }
      std::vector<uint64_t> din(m->dom);
      if (branch == 0) {       // x = val
        for (int w = m->gOff[x]; w < m->gOff[x + 1]; ++w) din[w] = 0;
        din[wa] = bit;
      } else {                 // x != val
        din[wa] &= ~bit;
      }
      s = ct_model_fixpoint(m, din.data(), nullptr);
      if (s < 0) {
        err = s;
        stop = true;
        return;
      }
      account(depth + 1, x, val, branch, s);
      if (s == CT_OK) node(depth + 1);
      if (ct_model_pop(m) < 0) {
        err = CT_ECUDA;
        stop = true;
        return;
      }
    }
  }
};
}  // namespace

// Device-resident DFS: one cooperative launch (k_model_search).  Returns
// CT_OK / CT_FAIL like the host driver or an error; *fallback = true if the
// host driver must run instead (trail too short, no memory for it).
static ct_status model_search_device(ct_model *m, int32_t value_order, int64_t max_nodes, int64_t max_solutions,
                                     int32_t *out_solution, ct_search_stats *out_stats, bool *fallback) {
  *fallback = false;
  DeviceGuard g(m->device);
  const int64_t pool16 = (int64_t)((m->pool_bytes + 15) / 16);
  if (!m->snap_dev) {
    int64_t vals = 1;
    for (int v = 0; v < m->nv; ++v) vals += m->vd[v];
    m->levels = (int)std::min<int64_t>(kSearchMaxLevels, vals);
    if (m->search_levels > 0) m->levels = std::max(2, std::min(m->levels, m->search_levels));
    if (cudaMalloc(&m->snap_dev, (size_t)m->levels * pool16 * 16) != cudaSuccess) {
      cudaGetLastError();
      m->snap_dev = nullptr;
      *fallback = true;
      return CT_OK;
    }
    std::vector<int32_t> gv(m->gOff);
    gv.insert(gv.end(), m->vlo.begin(), m->vlo.end());
    CUDA_TRY(cudaMalloc(&m->d_goff, gv.size() * 4));
    CUDA_TRY(cudaMemcpy(m->d_goff, gv.data(), gv.size() * 4, cudaMemcpyHostToDevice));
    m->d_vlo = m->d_goff + m->gOff.size();
    CUDA_TRY(cudaHostAlloc((void **)&m->h_sout, (size_t)(16 + m->nv) * 8, cudaHostAllocMapped));
    CUDA_TRY(cudaHostGetDevicePointer((void **)&m->d_sout, m->h_sout, 0));
    m->ssmem = std::max(m->smem, (size_t)m->Wg * 8);
    CUDA_TRY(cudaFuncSetAttribute(k_model_search, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(m->ssmem, 1)));
    int occ = 0, sms = 148;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_model_search, kFusedTPB, m->ssmem));
    CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->device));
    if (occ < 1) {
      *fallback = true;
      return CT_OK;
    }
    m->sgrid = std::min(m->grid, sms * occ);
  }
  SearchDev sd{};
  sd.pool = reinterpret_cast<uint4 *>(m->pool);
  sd.pool16 = pool16;
  sd.snaps = m->snap_dev;
  sd.levels = m->levels;
  sd.gOff = m->d_goff;
  sd.vlo = m->d_vlo;
  sd.nv = m->nv;
  sd.value_order = value_order;
  sd.max_nodes = max_nodes;
  sd.max_solutions = max_solutions;
  sd.out = m->d_sout;
  volatile long long *st = m->h_sout;
  *st = kPendingStatus;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)m->sgrid);
  lc.blockDim = dim3(kFusedTPB);
  lc.dynamicSmemBytes = m->ssmem;
  lc.stream = m->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&lc, k_model_search, m->md, sd));
  CUDA_TRY(cudaStreamSynchronize(m->stream));
  if (*st == kPendingStatus) return fail(CT_ECUDA, "device search ended without a status");
  if (m->h_sout[9]) {   // deeper than the trail: the host driver takes over
    *fallback = true;
    return CT_OK;
  }
  ct_search_stats o{};
  o.nodes = m->h_sout[1];
  o.failures = m->h_sout[2];
  o.solutions = m->h_sout[3];
  o.table_calls = m->h_sout[4];
  o.iterations = m->h_sout[5];
  o.max_depth = m->h_sout[6];
  o.device_ms = (double)m->h_sout[7] * 1e-6;
  o.trace_hash = (uint64_t)m->h_sout[8];
  if (out_stats) *out_stats = o;
  if (o.solutions > 0 && out_solution)
    for (int v = 0; v < m->nv; ++v) out_solution[v] = (int32_t)m->h_sout[16 + v];
  return o.solutions > 0 ? CT_OK : CT_FAIL;
}

ct_status ct_model_search_phases(const ct_model *m, int64_t *out6) {
  if (!m || !out6) return fail(CT_EINVAL, "NULL argument");
  for (int i = 0; i < 6; ++i) out6[i] = m->h_sout ? (int64_t)m->h_sout[10 + i] : -1;
  return CT_OK;
}

ct_status ct_model_search(ct_model *m, int32_t value_order, int64_t max_nodes, int64_t max_solutions,
                          int32_t *out_solution, ct_search_stats *out_stats) {
  return ct_model_search_ex(m, value_order, max_nodes, max_solutions, 0, out_solution, out_stats);
}

ct_status ct_model_search_ex(ct_model *m, int32_t value_order, int64_t max_nodes, int64_t max_solutions,
                             int32_t driver, int32_t *out_solution, ct_search_stats *out_stats) {
  if (!m) return fail(CT_EINVAL, "NULL model");
  if (value_order < 0 || value_order > 1) return fail(CT_EINVAL, "value_order must be 0 (max) or 1 (min)");
  if (driver == 0 && !m->dead && m->depth == 0) {
    bool fallback = false;
    const ct_status s = model_search_device(m, value_order, max_nodes, max_solutions, out_solution, out_stats,
                                            &fallback);
    if (!fallback) return s;
  }
  Dfs d;
  d.m = m;
  d.value_order = value_order;
  d.max_nodes = max_nodes;
  d.max_solutions = max_solutions;
  d.sol.assign(m->nv, 0);
  d.st.trace_hash = 14695981039346656037ull;
  if (m->dead) {
    d.account(0, -1, 0, 2, CT_FAIL);
  } else {
    // the root is the model's current fixpoint (re-run: counts as the root node)
    ct_status s = ct_model_push(m);
    if (s < 0) return s;
    s = ct_model_fixpoint(m, nullptr, nullptr);
    if (s < 0) return s;
    d.account(0, -1, 0, 2, s);
    if (s == CT_OK) d.node(0);
    if (ct_model_pop(m) < 0) return CT_ECUDA;
  }
  if (d.err < 0) return d.err;
  if (out_stats) *out_stats = d.st;
  if (d.st.solutions > 0 && out_solution) memcpy(out_solution, d.sol.data(), (size_t)m->nv * 4);
  return d.st.solutions > 0 ? CT_OK : CT_FAIL;
}

void ct_model_destroy(ct_model *m) { model_free(m); }

}  // extern "C"

// ================================================================== placement ablation (f3)
#include "ct_placement.cuh"
