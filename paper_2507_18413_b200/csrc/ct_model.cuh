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
#include "ct_kernels.cuh"

namespace ctk {

constexpr int kMaxModelTables = 64;

struct ModelCtl {
  uint32_t bar_count, bar_gen;   // grid barrier
  int32_t active[2];             // tables with work, by iteration parity
  int32_t fail;
  int32_t iters;                 // Jacobi iterations of the last fixpoint
  int32_t tile_ctr;              // pooled update tiles
  int32_t status;
  long long table_calls;         // non-no-op table propagations in the last fixpoint
  unsigned long long t0, t1;     // %globaltimer at start / end
  int32_t pad[16];
};

struct ModelDev {
  int32_t ntab, Wg;
  const TableDev *tabs;   // [ntab]
  const StateDev *sts;    // [ntab]
  uint64_t *gdom;         // [Wg] shared domains
  ModelCtl *mc;
};

__device__ __forceinline__ void model_barrier(ModelCtl *mc) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t gen = ld_acquire_u32(&mc->bar_gen);
    __threadfence();
    if (atomicAdd(&mc->bar_count, 1u) == gridDim.x - 1) {
      mc->bar_count = 0;
      __threadfence();
      atomicAdd(&mc->bar_gen, 1u);
    } else {
      while (ld_acquire_u32(&mc->bar_gen) == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// table index k of pooled unit g given exclusive prefix pre[0..ntab]
__device__ __forceinline__ int find_table(const int64_t *pre, int ntab, int64_t g) {
  int k = 0;
  while (k + 1 < ntab && pre[k + 1] <= g) ++k;
  return k;
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
  const int tid = threadIdx.x, lane = tid & 31;
  const int gw = blockIdx.x * (kFusedTPB / 32) + (tid >> 5), nw = gridDim.x * (kFusedTPB / 32);
  __shared__ UpdParams s_up[kMaxModelTables];
  __shared__ FiltParams s_fp[kMaxModelTables];
  __shared__ int64_t s_pre[kMaxModelTables + 1];
  __shared__ int s_tile;
  __shared__ uint32_t s_woff[kUpdTPB / 32];
  __shared__ uint32_t s_excl;
  __shared__ int s_brk;
  const int ntab = md.ntab;

  if (blockIdx.x == 0) {
    if (gdom_in)
      for (int w = tid; w < md.Wg; w += kFusedTPB) md.gdom[w] = gdom_in[w];
    if (tid == 0) {
      mc->t0 = globaltimer();
      mc->fail = 0;
      mc->iters = 0;
      mc->table_calls = 0;
      mc->active[0] = mc->active[1] = 0;
      mc->tile_ctr = 0;
    }
  }
  model_barrier(mc);

  for (int it = 0; it < max_iters; ++it) {
    // ---- ingest (a2): one block per table, removals = values the shared domains lost
    if (blockIdx.x == 0 && tid == 0) mc->active[(it + 1) & 1] = 0;
    for (int k = blockIdx.x; k < ntab; k += gridDim.x) {
      dev_ingest<kFusedTPB>(md.tabs[k], md.sts[k], nullptr, 0, smem, md.gdom);
      __syncthreads();
      if (tid == 0) {
        const Ctl *c = md.sts[k].ctl;
        if (c->fail_fast) atomicExch(&mc->fail, 1);
        else if (!c->noop && !c->skip) atomicAdd(&mc->active[it & 1], 1);
      }
    }
    model_barrier(mc);
    if (tid == 0) s_brk = __ldcg(&mc->fail) || __ldcg(&mc->active[it & 1]) == 0;
    __syncthreads();
    if (s_brk) break;
    if (blockIdx.x == 0 && tid == 0) {
      mc->iters = it + 1;
      mc->table_calls += __ldcg(&mc->active[it & 1]);
    }
    // ---- update (a3-a5): tiles of all tables pooled over the grid
    if (tid == 0) {
      int64_t acc = 0;
      for (int k = 0; k < ntab; ++k) {
        s_up[k] = load_upd_params(md.sts[k].ctl);
        s_pre[k] = acc;
        acc += s_up[k].go ? s_up[k].ntiles : 0;
      }
      s_pre[ntab] = acc;
    }
    __syncthreads();
    {
      uint32_t n_loads = 0, n_writes = 0;
      while (true) {
        if (tid == 0) s_tile = atomicAdd(&mc->tile_ctr, 1);
        __syncthreads();
        const int g = s_tile;
        if (g >= s_pre[ntab]) break;
        const int k = find_table(s_pre, ntab, g);
        update_tile(md.tabs[k], md.sts[k], s_up[k], (int)(g - s_pre[k]), s_woff, &s_excl, n_loads, n_writes);
      }
    }
    model_barrier(mc);
    if (blockIdx.x == 0 && tid == 0) mc->tile_ctr = 0;
    // ---- probe (a6a): items of all tables pooled over the warps
    if (tid == 0) {
      int64_t acc = 0;
      for (int k = 0; k < ntab; ++k) {
        s_fp[k] = load_filt_params(md.tabs[k], md.sts[k]);
        s_pre[k] = acc;
        acc += (s_fp[k].go && s_fp[k].Lout > 0) ? s_fp[k].nitems : 0;
      }
      s_pre[ntab] = acc;
    }
    __syncthreads();
    if (blockIdx.x == 0 && tid < ntab && s_fp[tid].go) md.sts[tid].sup[md.tabs[tid].R] = s_fp[tid].Lout > 0;
    {
      uint32_t n_loads = 0;
      for (int64_t g = gw; g < s_pre[ntab]; g += nw) {
        const int k = find_table(s_pre, ntab, g);
        probe_item(md.tabs[k], md.sts[k], s_fp[k], (int)(g - s_pre[k]), n_loads);
      }
    }
    model_barrier(mc);
    // ---- scan (a6b): misses x chunks of all tables pooled over the warps
    if (tid == 0) {
      int64_t acc = 0;
      for (int k = 0; k < ntab; ++k) {
        s_fp[k] = load_filt_params(md.tabs[k], md.sts[k]);
        s_pre[k] = acc;
        acc += scan_units(s_fp[k]);
      }
      s_pre[ntab] = acc;
    }
    __syncthreads();
    {
      uint32_t n_loads = 0;
      for (int64_t g = gw; g < s_pre[ntab]; g += nw) {
        const int k = find_table(s_pre, ntab, g);
        scan_unit(md.tabs[k], md.sts[k], s_fp[k], g - s_pre[k], n_loads);
      }
    }
    model_barrier(mc);
    // ---- finalize (a6c-a7): one block per table; AND the new domains into the shared ones
    for (int k = blockIdx.x; k < ntab; k += gridDim.x) {
      const TableDev &tb = md.tabs[k];
      const StateDev &st = md.sts[k];
      dev_finalize<kFusedTPB>(tb, st, nullptr, nullptr, nullptr, smem);
      __syncthreads();
      if (__ldcg(&st.ctl->last_status) != 0) {
        if (tid == 0) atomicExch(&mc->fail, 1);
      } else {
        for (int w = tid; w < tb.Wd; w += kFusedTPB) {
          const uint64_t nd = __ldcg(st.dom + w);
          const uint64_t g0 = __ldcg(md.gdom + tb.gword[w]);
          if ((g0 & nd) != g0) atomicAnd(reinterpret_cast<unsigned long long *>(md.gdom + tb.gword[w]), nd);
        }
      }
      __syncthreads();
    }
    model_barrier(mc);
    if (tid == 0) s_brk = __ldcg(&mc->fail);
    __syncthreads();
    if (s_brk) break;
  }
  model_barrier(mc);
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
  (void)lane;
}

}  // namespace ctk
