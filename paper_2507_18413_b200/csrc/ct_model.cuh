// ct_model.cuh -- on-device fixpoint of several table constraints sharing
// variables (the engine alternates search
// and propagation; each table's propagator runs until nothing changes).
//
// One cooperative persistent kernel per search node: Jacobi iterations over
// the tables -- every iteration runs the five CT phases of ALL tables at once
// (ingest: one block per table; update / probe / scan: the tiles, items and
// units of all tables pooled over the grid; finalize: one block per table,
// which ANDs the table's new domains into the shared domains).  A table whose
// scope lost no value since its last run is a no-op; the loop stops when every
// table is a no-op (greatest common fixpoint, unique -- SURVEY Q22) or one fails.
#pragma once
#include "ct_fast.cuh"

namespace ctk {

constexpr int kMaxModelTables = 64;

struct ModelCtl {
  int32_t fail;
  int32_t iters;                 // Jacobi iterations of the last fixpoint
  int32_t status;
  long long table_calls;         // non-no-op table propagations in the last fixpoint
  unsigned long long t0, t1;     // %globaltimer at start / end
  unsigned long long ph[6];      // device search: ns in ingest, update, probe, scan, finalize, trail copies
  // (the per-iteration verdicts -- active / failed tables, probe misses,
  // shared-domain changes -- travel on the grid barrier's arrivals)
};
static_assert(sizeof(ModelCtl) <= 256, "ModelCtl must fit its 256-byte slot");

struct ModelDev {
  int32_t ntab, Wg;
  const TableDev *tabs;   // [ntab]
  const StateDev *sts;    // [ntab]
  uint64_t *gdom;         // [Wg] shared domains
  ModelCtl *mc;
  uint32_t *bar;          // [kBarWords] grid barrier (k_fast's), zeroed at creation
};

// k_fast's grid barrier (one acq_rel arrival counter, per-group generation copies)
#define model_barrier(mc) fast_grid_barrier(md.bar)

// probe_item with the residue probe and the first round of the scan issued
// together (one round trip for most items instead of two).
__device__ __forceinline__ void probe_item_fused(const TableDev &tb, const StateDev &st, const FiltParams &f,
                                                 int item, uint32_t &n_loads, int32_t *miss_flag) {
  const int lane = threadIdx.x & 31;
  const ulonglong2 *__restrict__ T2 = reinterpret_cast<const ulonglong2 *>(st.T);
  const int row = __ldcg(st.items + item);
  const uint64_t *__restrict__ srow = tb.S + (int64_t)row * tb.Wp;
  const int r = (tb.use_res && lane == 0) ? st.res[row] : -1;
  const int L1 = min(f.L, 32 * kScanUnroll);   // the first round
  int pid[kScanUnroll];
#pragma unroll
  for (int q = 0; q < kScanUnroll; ++q) {
    const int k = q * 32 + lane;
    pid[q] = f.idx ? f.idx[k < L1 ? k : 0] : (k < L1 ? k : 0);
  }
  const int rr = r >= 0 ? r : pid[0];
  const ulonglong2 tr = __ldcg(T2 + rr), sr = ld_sup2(srow + 2 * (int64_t)rr);
  ulonglong2 t[kScanUnroll], sv[kScanUnroll];
#pragma unroll
  for (int q = 0; q < kScanUnroll; ++q) {
    t[q] = __ldcg(T2 + pid[q]);
    sv[q] = ld_sup2(srow + 2 * (int64_t)pid[q]);
  }
  n_loads += 2 * L1;
  if (__any_sync(0xffffffffu, r >= 0 && ((tr.x & sr.x) | (tr.y & sr.y)) != 0)) {
    if (lane == 0) st.sup[row] = 1;
    return;
  }
  int hit = -1;
#pragma unroll
  for (int q = kScanUnroll - 1; q >= 0; --q) {
    const bool in = q * 32 + lane < L1;
    const unsigned b = __ballot_sync(0xffffffffu, in && ((t[q].x & sv[q].x) | (t[q].y & sv[q].y)) != 0);
    if (b) hit = __shfl_sync(0xffffffffu, pid[q], __ffs(b) - 1);
  }
  if (hit < 0 && f.L > L1) hit = scan_pairs(f.idx, T2, srow, L1, min(f.L, kFirstScan), nullptr, lane, n_loads);
  if (lane == 0) {
    if (hit >= 0) {
      st.sup[row] = 1;
      st.res[row] = hit;
    } else if (f.L > kFirstScan) {
      st.scanlist[atomicAdd(&st.ctl->nscan, 1)] = row;
      *miss_flag = 1;
    }
  }
}

// Exclusive prefix of the per-table unit counts (thread 0, shared memory only),
// then a block barrier.
__device__ __forceinline__ void model_prefix(const int64_t *cnt, int64_t *pre, int ntab) {
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int k = 0; k < ntab; ++k) {
      pre[k] = acc;
      acc += cnt[k];
    }
    pre[ntab] = acc;
  }
  __syncthreads();
}

// table index k of pooled unit g given exclusive prefix pre[0..ntab]
__device__ __forceinline__ int find_table(const int64_t *pre, int ntab, int64_t g) {
  int k = 0;
  while (k + 1 < ntab && pre[k + 1] <= g) ++k;
  return k;
}

// The Jacobi fixpoint of the model from the current shared domains (md.gdom,
// already set and visible: the caller ends its set-up with a grid barrier, and
// block 0 has reset the control fields).  Every CTA of the cooperative grid
// calls it; it returns after a final grid barrier with mc->fail set iff some
// table failed.  Dynamic smem: max over tables of ingest/finalize smem.
__device__ void model_fixpoint_dev(const ModelDev &md, int max_iters, uint64_t *smem) {
  ModelCtl *mc = md.mc;
  const int tid = threadIdx.x;
  const int gw = blockIdx.x * (kFusedTPB / 32) + (tid >> 5), nw = gridDim.x * (kFusedTPB / 32);
  __shared__ UpdParams s_up[kMaxModelTables];
  __shared__ FiltParams s_fp[kMaxModelTables];
  __shared__ int64_t s_pre[kMaxModelTables + 1];
  __shared__ int64_t s_cnt[kMaxModelTables];
  __shared__ uint32_t s_woff[kUpdTPB / 32];
  __shared__ uint32_t s_excl;
  __shared__ int s_brk;
  __shared__ int s_miss;   // this CTA queued a probe miss (summed by the barrier)
  __shared__ int s_cnt_ing, s_cnt_fin;   // this CTA's ingest / finalize verdicts (summed by the barrier)
  const int ntab = md.ntab;
  const bool t0 = blockIdx.x == 0 && tid == 0;
  unsigned long long tp = t0 ? globaltimer() : 0ull;
  auto lap = [&](int i) {
    if (t0) {
      const unsigned long long t = globaltimer();
      mc->ph[i] += t - tp;
      tp = t;
    }
  };

  for (int it = 0; it < max_iters; ++it) {
    // ---- ingest (a2): one block per table, removals = values the shared domains lost.
    // Each CTA's verdicts ride on its barrier arrival (active tables + 256 x
    // failed tables); the releasing CTA decides whether the fixpoint stops
    // (a FAIL, or no table has anything to do) and keeps the statistics.
    set_loc(0x10000000u | ((uint32_t)it << 8) | 1u);
    if (tid == 0) s_cnt_ing = 0;
    for (int k = blockIdx.x; k < ntab; k += gridDim.x) {
      const int r = dev_ingest<kFusedTPB>(md.tabs[k], md.sts[k], nullptr, 0, smem, md.gdom);
      __syncthreads();
      if (tid == 0) s_cnt_ing += r == 2 ? 256 : (r == 0 ? 1 : 0);
    }
    {
      int leader = 0;
      const int brk = fast_grid_barrier_mode(
          md.bar,
          [&](uint32_t v) {
            const uint32_t active = v & 255u, fails = v >> 8;
            const int b = fails > 0 || active == 0;
            if (b) {
              mc->fail = fails > 0;
            } else {
              mc->iters = it + 1;
              mc->table_calls = __ldcg(&mc->table_calls) + (int)active;
            }
            return b;
          },
          leader, &s_brk, &s_cnt_ing);
      lap(0);
      if (brk) break;
    }
    set_loc(0x10000000u | ((uint32_t)it << 8) | 2u);
    // ---- update (a3-a5): tiles of all tables pooled over the grid
    // (every table's parameters loaded by its own thread: one round trip)
    if (tid < ntab) {
      s_up[tid] = load_upd_params(md.sts[tid].ctl);
      s_cnt[tid] = s_up[tid].go ? s_up[tid].ntiles : 0;
    }
    __syncthreads();
    model_prefix(s_cnt, s_pre, ntab);
    {
      uint32_t n_loads = 0, n_writes = 0;
      // static round-robin over the pooled tiles (no counter round trip per
      // tile; every CTA takes its tiles in increasing order, so the chained
      // scan's look-back only ever waits on lower tiles already taken)
      for (int64_t g = blockIdx.x; g < s_pre[ntab]; g += gridDim.x) {
        const int k = find_table(s_pre, ntab, g);
        update_tile(md.tabs[k], md.sts[k], s_up[k], (int)(g - s_pre[k]), s_woff, &s_excl, n_loads, n_writes);
      }
    }
    model_barrier(mc);
    lap(1);
    set_loc(0x10000000u | ((uint32_t)it << 8) | 3u);
    // ---- probe (a6a): items of all tables pooled over the warps
    if (tid < ntab) {
      s_fp[tid] = load_filt_params(md.tabs[tid], md.sts[tid]);
      s_cnt[tid] = (s_fp[tid].go && s_fp[tid].Lout > 0) ? s_fp[tid].nitems : 0;
    }
    if (tid == 0) s_miss = 0;
    __syncthreads();
    model_prefix(s_cnt, s_pre, ntab);
    if (blockIdx.x == 0 && tid < ntab && s_fp[tid].go) md.sts[tid].sup[md.tabs[tid].R] = s_fp[tid].Lout > 0;
    {
      uint32_t n_loads = 0;
      for (int64_t g = gw; g < s_pre[ntab]; g += nw) {
        const int k = find_table(s_pre, ntab, g);
        probe_item_fused(md.tabs[k], md.sts[k], s_fp[k], (int)(g - s_pre[k]), n_loads, &s_miss);
      }
    }
    // the barrier's last arrival checks whether any table queued a miss; if
    // none did, every CTA skips the scan phase and its barrier
    {
      int leader = 0;
      const int mode = fast_grid_barrier_mode(
          md.bar, [](uint32_t misses) { return misses ? 0 : 1; }, leader, &s_brk, &s_miss);
      lap(2);
      if (mode == 1) goto finalize_phase;
    }
    set_loc(0x10000000u | ((uint32_t)it << 8) | 4u);
    // ---- scan (a6b): misses x chunks of all tables pooled over the warps
    if (tid < ntab) {
      s_fp[tid] = load_filt_params(md.tabs[tid], md.sts[tid]);
      s_cnt[tid] = scan_units(s_fp[tid]);
    }
    __syncthreads();
    model_prefix(s_cnt, s_pre, ntab);
    {
      uint32_t n_loads = 0;
      for (int64_t g = gw; g < s_pre[ntab]; g += nw) {
        const int k = find_table(s_pre, ntab, g);
        scan_unit(md.tabs[k], md.sts[k], s_fp[k], g - s_pre[k], n_loads);
      }
    }
    model_barrier(mc);
    lap(3);
  finalize_phase:
    // ---- finalize (a6c-a7): one block per table; AND the new domains into the shared ones.
    // Verdicts on the barrier arrival again: CTAs that removed a value from
    // the shared domains + 256 x failed tables.
    set_loc(0x10000000u | ((uint32_t)it << 8) | 5u);
    if (tid == 0) s_cnt_fin = 0;
    for (int k = blockIdx.x; k < ntab; k += gridDim.x) {
      const TableDev &tb = md.tabs[k];
      const StateDev &st = md.sts[k];
      // in flight during dev_finalize
      const int gw0 = tid < tb.Wd ? tb.gword[tid] : 0, gs0 = tid < tb.Wd ? tb.gshared[tid] : 0;
      if (dev_finalize<kFusedTPB>(tb, st, nullptr, nullptr, nullptr, smem) != 0) {
        if (tid == 0) atomicAdd(&s_cnt_fin, 256);
      } else {
        for (int w = tid; w < tb.Wd; w += kFusedTPB) {
          const uint64_t nd = smem[w];   // dev_finalize's new domains (also stored in st.dom)
          const int gw = w == tid ? gw0 : tb.gword[w];
          if (nd != ~0ull) {
            const uint64_t old = atomicAnd(reinterpret_cast<unsigned long long *>(md.gdom + gw), nd);
            // a removal counts as a change only if another table constrains
            // the variable: a variable of this table alone cannot make any
            // table active in the next iteration (this one already has nd)
            if ((old & nd) != old && (w == tid ? gs0 : tb.gshared[w])) atomicOr(&s_cnt_fin, 1);
          }
        }
      }
      __syncthreads();
    }
    {
      // stop on a failure, or at the fixpoint: no table removed a value from
      // the shared domains, so every table is a no-op in the next iteration
      int leader = 0;
      const int brk = fast_grid_barrier_mode(
          md.bar,
          [&](uint32_t v) {
            const int b = (v >> 8) > 0 || (v & 255u) == 0;
            if (b) mc->fail = (v >> 8) > 0;
            return b;
          },
          leader, &s_brk, &s_cnt_fin);
      lap(4);
      if (brk) break;
    }
  }
  // the verdict and the statistics were written by the releasing CTA of the
  // deciding barrier: every CTA reads them after returning.  (The caller must
  // pass another grid barrier before the next model_reset_ctl.)
}

// Block 0: reset the per-fixpoint control fields (before a grid barrier).
__device__ __forceinline__ void model_reset_ctl(ModelCtl *mc) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    mc->fail = 0;
    mc->iters = 0;
    mc->table_calls = 0;
  }
}

// grid <= co-resident blocks (cooperative), kFusedTPB threads, dynamic smem =
// max over tables of ingest/finalize smem.  gdom_in (nullable, may be host
// mapped): new shared domains for this node (a search decision).  out (may be
// host mapped): [0] status (int32, written last), [1] Jacobi iterations,
// [2] non-no-op table propagations, [3] kernel ns, [4 ..) shared domains.
__global__ void __launch_bounds__(kFusedTPB, 3) k_model_fixpoint(ModelDev md, const uint64_t *__restrict__ gdom_in,
                                                                 uint64_t *__restrict__ out, int max_iters) {
  extern __shared__ __align__(16) uint64_t smem[];
  ModelCtl *mc = md.mc;
  const int tid = threadIdx.x;
  if (blockIdx.x == 0) {
    if (gdom_in)
      for (int w = tid; w < md.Wg; w += kFusedTPB) md.gdom[w] = gdom_in[w];
    if (tid == 0) mc->t0 = globaltimer();
  }
  model_reset_ctl(mc);
  model_barrier(mc);
  model_fixpoint_dev(md, max_iters, smem);
  if (blockIdx.x == 0) {
    const int status = __ldcg(&mc->fail) ? 1 : 0;
    if (status == 0)
      for (int w = tid; w < md.Wg; w += kFusedTPB) out[4 + w] = __ldcg(md.gdom + w);
    if (tid == 0) {
      mc->status = status;
      mc->t1 = globaltimer();
      out[1] = (uint64_t)__ldcg(&mc->iters);
      out[2] = (uint64_t)__ldcg(&mc->table_calls);
      out[3] = mc->t1 - mc->t0;
    }
    __threadfence_system();
    __syncthreads();
    if (tid == 0) *reinterpret_cast<int32_t *>(out) = status;
  }
}

// ------------------------------------------------------------------ device-resident DFS (config 5)
// The whole search in ONE cooperative launch: binary branching x = v / x != v,
// input_order (lowest-index unbound variable), indomain_max / indomain_min
// (SPEC S:L391), each node propagated to the common
// fixpoint with model_fixpoint_dev.  The trail is a snapshot of the state pool
// per level (all table states + shared domains), copied by the whole grid.
// Every CTA runs the same control flow (it depends only on the shared domains
// and the fixpoint verdicts, both read after grid barriers), so no decision
// has to be broadcast; block 0 thread 0 keeps the statistics, the trace hash
// (FNV-1a over (depth, var, value, branch, status), as the host driver) and
// the last solution.
constexpr int kSearchMaxLevels = 512;

struct SearchDev {
  uint4 *pool;                 // state pool, pool16 16-byte words
  int64_t pool16;
  uint4 *snaps;                // [levels][pool16]
  int32_t levels;
  const int32_t *gOff;         // [nv + 1] first shared-domain word of each variable
  const int32_t *vlo;          // [nv]
  int32_t nv, value_order;
  int64_t max_nodes, max_solutions;
  long long *out;              // [0] status (last), [1] nodes, [2] failures, [3] solutions, [4] table calls,
                               // [5] iterations, [6] max depth, [7] device ns, [8] trace hash,
                               // [9] error (1: deeper than `levels`), [10..15] ns per phase (ingest,
                               // update, probe, scan, finalize, trail copies), [16 ..) last solution (nv)
};

__device__ __forceinline__ void search_copy(uint4 *dst, const uint4 *src, int64_t n16) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride) dst[i] = __ldcg(src + i);
}

struct SearchFrame {
  int32_t x, a, branch, pad;
};

// Control state of the search, one copy per CTA (identical in every CTA).
struct SearchCtl {
  int state, d, x, a, fail, err;
  long long nodes, failures, solutions, calls, iters, maxd;
  unsigned long long hash;
};

enum { kSExpand = 0, kSBranch = 1, kSPop = 2, kSReturn = 3, kSDone = 4 };

__device__ __forceinline__ void search_fnv(unsigned long long &h, unsigned long long v) {
  for (int i = 0; i < 8; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= 1099511628211ull;
  }
}

// thread 0: count one fixpoint node (same fields and hash as the host driver)
__device__ __forceinline__ void search_account(SearchCtl &c, const ModelCtl *mc, int depth, int var, int val,
                                               int branch, int fail) {
  c.nodes++;
  if (fail) c.failures++;
  c.calls += __ldcg(&mc->table_calls);
  c.iters += __ldcg(&mc->iters);
  if (depth > c.maxd) c.maxd = depth;
  search_fnv(c.hash, (unsigned long long)depth);
  search_fnv(c.hash, (unsigned long long)(long long)var);
  search_fnv(c.hash, (unsigned long long)(long long)val);
  search_fnv(c.hash, (unsigned long long)branch);
  search_fnv(c.hash, (unsigned long long)(fail ? 1 : 0));
}

// grid <= co-resident blocks (cooperative; same geometry as k_model_fixpoint),
// kFusedTPB threads, dynamic smem = max(fixpoint smem, 8 * Wg).
__global__ void __launch_bounds__(kFusedTPB, 3) k_model_search(ModelDev md, SearchDev sd) {
  extern __shared__ __align__(16) uint64_t smem[];
  __shared__ SearchFrame fr[kSearchMaxLevels];
  __shared__ SearchCtl c;
  ModelCtl *mc = md.mc;
  const int tid = threadIdx.x;
  const unsigned long long t_start = globaltimer();
  // one fixpoint from the current shared domains; every CTA gets the verdict
  auto fixpoint = [&]() {
    model_reset_ctl(mc);
    model_barrier(mc);
    model_fixpoint_dev(md, 1 << 20, smem);
    if (tid == 0) c.fail = __ldcg(&mc->fail);
    __syncthreads();
  };
  if (blockIdx.x == 0 && tid == 0)
    for (int i = 0; i < 6; ++i) mc->ph[i] = 0;
  if (tid == 0) {
    c.d = 0;
    c.err = 0;
    c.nodes = c.failures = c.solutions = c.calls = c.iters = c.maxd = 0;
    c.hash = 14695981039346656037ull;
  }
  // the root: trail level 0, fixpoint of the current domains
  search_copy(sd.snaps, sd.pool, sd.pool16);
  fixpoint();
  if (tid == 0) {
    search_account(c, mc, 0, -1, 0, 2, c.fail);
    c.state = c.fail ? kSDone : kSExpand;
  }
  __syncthreads();
  while (true) {
    const int state = c.state;
    set_loc(0x20000000u | ((uint32_t)state << 16) | ((uint32_t)c.d & 0xffffu));
    // every thread has read the state (and the step before it read c) before
    // thread 0 may change it below
    __syncthreads();
    if (state == kSDone) break;
    if (state == kSExpand) {
      // the node at depth d is an OK fixpoint: pick x (input_order) and a
      // (indomain_max / min); the shared domains go to shared memory first
      for (int w = tid; w < md.Wg; w += kFusedTPB) smem[w] = __ldcg(md.gdom + w);
      __syncthreads();
      if (tid == 0) {
        int x = -1, a = -1;
        for (int v = 0; v < sd.nv && x < 0; ++v) {
          int cnt = 0;
          for (int w = sd.gOff[v]; w < sd.gOff[v + 1]; ++w) cnt += __popcll(smem[w]);
          if (cnt > 1) x = v;
        }
        if (x >= 0) {
          if (sd.value_order == 0) {
            for (int w = sd.gOff[x + 1] - 1; w >= sd.gOff[x] && a < 0; --w)
              if (smem[w]) a = (w - sd.gOff[x]) * 64 + 63 - __clzll(smem[w]);
          } else {
            for (int w = sd.gOff[x]; w < sd.gOff[x + 1] && a < 0; ++w)
              if (smem[w]) a = (w - sd.gOff[x]) * 64 + __ffsll(smem[w]) - 1;
          }
          if (c.d + 1 >= sd.levels) {   // the trail is full: report, stop
            c.err = 1;
            c.state = kSDone;
          } else {
            fr[c.d].x = x;
            fr[c.d].a = a;
            fr[c.d].branch = 0;
            c.state = kSBranch;
          }
        } else {   // every variable bound: a solution
          c.solutions++;
          if (blockIdx.x == 0)
            for (int v = 0; v < sd.nv; ++v) {
              int av = 0;
              for (int w = sd.gOff[v]; w < sd.gOff[v + 1]; ++w)
                if (smem[w]) av = (w - sd.gOff[v]) * 64 + __ffsll(smem[w]) - 1;
              sd.out[16 + v] = sd.vlo[v] + av;
            }
          c.state = (sd.max_solutions > 0 && c.solutions >= sd.max_solutions) ? kSDone : kSReturn;
        }
      }
      __syncthreads();
      // every CTA read the shared domains above; unless the next step is the
      // branch (whose snapshot barrier comes first), the next step may restore
      // the pool -- shared domains included -- so no CTA may move on before all
      // have read them (else a late CTA reads restored domains, picks another
      // step, and the grid's control flow splits)
      if (c.state != kSBranch) model_barrier(mc);
    } else if (state == kSBranch) {
      const SearchFrame f = fr[c.d];
      if (f.branch == 2) {
        if (tid == 0) c.state = kSReturn;
        __syncthreads();
        continue;
      }
      if (sd.max_nodes > 0 && c.nodes >= sd.max_nodes) {
        if (tid == 0) c.state = kSDone;
        __syncthreads();
        continue;
      }
      // push: trail level d + 1 = the state before this branch.  The second
      // branch comes straight from kSPop, which restored the pool FROM that
      // level (and ended with a barrier): the snapshot already holds it.
      if (f.branch == 0) {
        const unsigned long long tc = globaltimer();
        search_copy(sd.snaps + (int64_t)(c.d + 1) * sd.pool16, sd.pool, sd.pool16);
        model_barrier(mc);   // the snapshot is complete before the domains change
        if (blockIdx.x == 0 && tid == 0) mc->ph[5] += globaltimer() - tc;
      }
      // block 0 applies the decision to the shared domains (visible to all
      // after the fixpoint's opening barrier)
      if (blockIdx.x == 0) {
        const int w0 = sd.gOff[f.x], w1 = sd.gOff[f.x + 1];
        const int wa = w0 + f.a / 64;
        const uint64_t bit = 1ull << (f.a % 64);
        for (int w = w0 + tid; w < w1; w += kFusedTPB) {
          const uint64_t dw = md.gdom[w];
          md.gdom[w] = f.branch == 0 ? (w == wa ? bit : 0ull) : (w == wa ? dw & ~bit : dw);
        }
      }
      fixpoint();
      if (tid == 0) {
        search_account(c, mc, c.d + 1, f.x, sd.vlo[f.x] + f.a, f.branch, c.fail);
        if (!c.fail) {
          c.d += 1;
          c.state = kSExpand;
        } else {
          c.state = kSPop;
        }
      }
      __syncthreads();
    } else if (state == kSPop) {
      // restore the state before the branch, then the next branch
      const unsigned long long tc = globaltimer();
      search_copy(sd.pool, sd.snaps + (int64_t)(c.d + 1) * sd.pool16, sd.pool16);
      model_barrier(mc);
      if (blockIdx.x == 0 && tid == 0) mc->ph[5] += globaltimer() - tc;
      if (tid == 0) {
        fr[c.d].branch += 1;
        c.state = kSBranch;
      }
      __syncthreads();
    } else {   // kSReturn: the node at depth d is done
      if (tid == 0) {
        if (c.d == 0) {
          c.state = kSDone;
        } else {
          c.d -= 1;
          c.state = kSPop;
        }
      }
      __syncthreads();
    }
  }
  // leave the model as it was before the search (trail level 0)
  search_copy(sd.pool, sd.snaps, sd.pool16);
  model_barrier(mc);
  if (blockIdx.x == 0 && tid == 0) {
    sd.out[1] = c.nodes;
    sd.out[2] = c.failures;
    sd.out[3] = c.solutions;
    sd.out[4] = c.calls;
    sd.out[5] = c.iters;
    sd.out[6] = c.maxd;
    sd.out[7] = (long long)(globaltimer() - t_start);
    sd.out[8] = (long long)c.hash;
    sd.out[9] = c.err;
    for (int i = 0; i < 6; ++i) sd.out[10 + i] = (long long)mc->ph[i];
    __threadfence_system();
    sd.out[0] = c.err ? -1 : (c.solutions > 0 ? 0 : 1);
  }
}

}  // namespace ctk
