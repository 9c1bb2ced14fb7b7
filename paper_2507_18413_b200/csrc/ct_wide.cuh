// ct_wide.cuh -- single-state propagation for tables with MANY support rows and
// FEW currTable words (the paper's own regime: knapsack tables with 80-200
// variables, domains up to 600-800 values and 5e3-1.5e4 tuples, PAPER.md
// L459-461, Table tbl:instances).  There R (sum of domain
// sizes, up to ~1e5 rows) is far larger than W (a few hundred words), so the
// call is dominated by filterDomains over up to R (x,a) items (P:L566-569:
// "filtering is where parallelisation helps most"), not by bandwidth.
//
//   k_wide        ONE CTA of kWideTPB threads: the word-level ingest of k_fast
//                 (per-domain-word popcount prefixes, lists written to global
//                 memory, no per-row scan over R), updateTable over the <= 8192
//                 active blocks + order-preserving compaction (block scan), the
//                 emptiness check; calls that end here (FAIL, dead state, no
//                 changed variable) are finalized here.
//   k_wide_filter ONE THREAD per filter item (item i -> CTA i % grid): residue
//                 probe; the misses of a CTA then go to its
//                 warps, one miss per warp, each scanned over the new index; a
//                 value without support is cleared from the state's domain with
//                 an atomic AND (x in s_sup by construction of the item list).
//                 The last CTA to finish writes the outputs (completion counter).
// Sharded tables: k_wide_filter only sets the per-row flags; the cross-shard
// OR and k_finalize follow as for the other shapes.
#pragma once
#include "ct_fast.cuh"

namespace ctk {

constexpr int kWideTPB = 1024;
constexpr int kWideWarps = kWideTPB / 32;
constexpr int kWideFiltTPB = 256;
constexpr int kWideMinRows = 2048;   // R above which a table takes this shape (if W2 <= kSmallMaxPairs)

// Shared memory of k_wide: the word arrays of cta_ingest (its row lists live in
// the state's global scratch).
__host__ __device__ inline size_t wide_smem_bytes(int n, int Wd) {
  return (size_t)Wd * 32 + (size_t)(Wd + 1) * 8 + (size_t)Wd * 4 + (size_t)(5 * n + 2) * 4 + 16;
}

__device__ __forceinline__ FastPtrs wide_ptrs(uint64_t *smem, const TableDev &tb, const StateDev &st) {
  FastPtrs p;
  const int Wd = tb.Wd, n = tb.n;
  p.din = smem;
  p.dl = p.din + Wd;
  p.bw = p.dl + Wd;
  p.iw = p.bw + Wd;
  p.upos = reinterpret_cast<int32_t *>(p.iw + Wd);
  p.ipos = p.upos + Wd + 1;
  p.wvar = p.ipos + Wd + 1;
  p.ulist = reinterpret_cast<uint32_t *>(st.ulist);   // global: up to R entries
  p.items = st.items;
  p.cd = p.wvar + Wd;
  p.cs = p.cd + n;
  p.vfl = p.cs + n;
  p.rb = p.vfl + n;
  p.dof = p.rb + n + 1;
  return p;
}

// Writes the call's outputs (domains from st.dom, pruned = din & ~dom) and the
// status; sys_fence: the outputs live in mapped host memory (sync call).
template <int NT>
__device__ void wide_write_ok(const TableDev &tb, const StateDev &st, uint64_t *out_dom, uint64_t *out_pruned,
                              int32_t *out_status, bool flip_index, int Lout, bool sys_fence) {
  Ctl *c = st.ctl;
  for (int k = threadIdx.x; k < tb.Wd; k += NT) {
    const uint64_t nd = __ldcg(st.dom + k);
    if (out_dom) out_dom[k] = nd;
    if (out_pruned) out_pruned[k] = __ldcg(st.din + k) & ~nd;
  }
  __syncthreads();   // then one cumulative system-scope fence by the status writer
  if (threadIdx.x == 0) {
    if (sys_fence) __threadfence_system();
    if (flip_index && tb.use_index) {
      c->parity ^= 1;
      c->L = Lout;
      c->identity = 0;
    }
    c->calls += 1;
    c->last_status = 0;
    if (out_status) *out_status = 0;
  }
}

__global__ void __launch_bounds__(kWideTPB, 1) k_wide(TableDev tb, const StateDev *__restrict__ states,
                                                     const uint64_t *__restrict__ removed, int root_mode,
                                                     int with_finalize, uint64_t *__restrict__ out_dom,
                                                     uint64_t *__restrict__ out_pruned,
                                                     int32_t *__restrict__ out_status, int use_state_out) {
  extern __shared__ __align__(16) uint64_t smem[];
  __shared__ FastShT<kWideWarps> fs;
  __shared__ StateDev s_st;
  __shared__ uint64_t s_warp[kWideWarps];
  if (threadIdx.x == 0) s_st = states[0];
  __syncthreads();
  const StateDev &st = s_st;
  Ctl *c = st.ctl;
  const int tid = threadIdx.x;
  const bool t0 = tid == 0;
  // let the dependent k_wide_filter grid launch now (it waits for this grid's
  // completion and memory flush at griddepcontrol.wait)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (t0) c->tph[0] = globaltimer();
  if (use_state_out) {
    out_dom = st.out + 1;
    out_pruned = st.out + 1 + tb.Wd;
    out_status = reinterpret_cast<int32_t *>(st.out);
  }
  const bool sys = use_state_out != 0;
  const FastPtrs p = wide_ptrs(smem, tb, st);
  cta_ingest<kWideTPB>(tb, st, removed, root_mode, p, fs, true);
  if (t0) c->tph[1] = globaltimer();
  // ---- calls that end without a filter (sharded tables: k_finalize decides
  // after the cross-shard OR, so nothing is finalized here)
  if (!with_finalize && (fs.dead || fs.fail || fs.noop)) return;
  if (fs.dead || fs.fail) {
    if (t0) {
      const int status = fs.dead ? -5 : 1;   // CT_ESTATE / CT_FAIL (some D_x empty)
      if (!fs.dead) {
        c->dead = 1;
        c->calls += 1;
      }
      c->last_status = status;
      if (with_finalize && out_status) {
        if (sys) __threadfence_system();
        *out_status = status;
      }
      for (int i = 2; i < 8; ++i) c->tph[i] = globaltimer();
    }
    return;
  }
  if (fs.noop) {   // no changed variable: the state is already at its fixpoint
    if (with_finalize) {
      for (int k = tid; k < tb.Wd; k += kWideTPB) st.dom[k] = p.din[k];
      __syncthreads();
      wide_write_ok<kWideTPB>(tb, st, out_dom, out_pruned, out_status, false, 0, sys);
    }
    if (t0)
      for (int i = 2; i < 8; ++i) c->tph[i] = globaltimer();
    return;
  }
  // ---- update + compaction (Alg. 2; RSparseBitSet index), one block
  const int Lout = block_update<kWideTPB>(tb, st, fs.L, fs.nrows, fs.ident, fs.par, s_warp);
  if (t0) {
    c->L_out = Lout;
    st.sup[tb.R] = Lout > 0;
    c->tph[2] = globaltimer();
  }
  if (Lout == 0 && with_finalize) {   // currTable empty: FAIL (Alg. 1 L5)
    if (t0) {
      c->dead = 1;
      c->calls += 1;
      c->last_status = 1;
      if (with_finalize && out_status) {
        if (sys) __threadfence_system();
        *out_status = 1;
      }
      for (int i = 3; i < 8; ++i) c->tph[i] = globaltimer();
    }
    return;
  }
  // the filter clears unsupported values from a copy of D (the new lastDom)
  if (with_finalize)
    for (int k = tid; k < tb.Wd; k += kWideTPB) st.dom[k] = p.din[k];
}

__global__ void __launch_bounds__(kWideFiltTPB) k_wide_filter(TableDev tb, const StateDev *__restrict__ states,
                                                             int with_finalize, uint64_t *__restrict__ out_dom,
                                                             uint64_t *__restrict__ out_pruned,
                                                             int32_t *__restrict__ out_status, int use_state_out) {
  __shared__ int s_last;
  __shared__ int s_cnt[kWideFiltTPB / 32];
  __shared__ int32_t s_miss[kWideFiltTPB];
  // launched as a programmatic dependent of k_wide: wait until it completed
  // and its writes are visible (a no-op when launched normally)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const StateDev &st = states[0];
  Ctl *c = st.ctl;
  const bool go = !(__ldcg(&c->skip) | __ldcg(&c->noop) | __ldcg(&c->fail_fast)) && __ldcg(&c->L_out) > 0;
  if (!go) return;   // k_wide ended the call
  const int lane = threadIdx.x & 31;
  const int nitems = __ldcg(&c->nitems);
  const int Lout = __ldcg(&c->L_out);
  const bool compact = tb.use_index != 0;
  const int par = __ldcg(&c->parity);
  const int32_t *__restrict__ idx = compact ? (par ? st.idx0 : st.idx1) : nullptr;
  const int L = compact ? Lout : tb.W2;
  const ulonglong2 *__restrict__ T2 = reinterpret_cast<const ulonglong2 *>(st.T);
  const int G = gridDim.x, warp = threadIdx.x >> 5;
  // item i -> CTA i % G, so every CTA gets an equal share; per round each
  // thread probes one item's residue, then the CTA's warps share its misses
  const int mine = (nitems - (int)blockIdx.x + G - 1) / G;   // items of this CTA
  uint32_t n_loads = 0;
  int nmiss = 0;
  for (int base = 0; base < mine; base += kWideFiltTPB) {
    const int j = base + threadIdx.x;
    int row = 0;
    bool miss = false;
    if (j < mine) {
      row = __ldcg(st.items + (int)blockIdx.x + j * G);
      miss = true;
      if (tb.use_res) {
        const int r = __ldcg(st.res + row);
        const ulonglong2 t = __ldcg(T2 + r);
        const ulonglong2 v = ld_sup2(tb.S + (int64_t)row * tb.Wp + 2 * (int64_t)r);
        if (((t.x & v.x) | (t.y & v.y)) != 0) {
          st.sup[row] = 1;
          miss = false;
        }
      }
    }
    // this round's misses -> shared list (ballot + popc per warp)
    const unsigned bm = __ballot_sync(0xffffffffu, miss);
    if (lane == 0) s_cnt[warp] = __popc(bm);
    __syncthreads();
    int off = 0, tot = 0;
    for (int w = 0; w < kWideFiltTPB / 32; ++w) {
      if (w < warp) off += s_cnt[w];
      tot += s_cnt[w];
    }
    if (miss) s_miss[off + __popc(bm & lanemask_lt())] = row;
    __syncthreads();
    // ... each scanned by one warp over the new index
    for (int m = warp; m < tot; m += kWideFiltTPB / 32) {
      const int mrow = s_miss[m];
      const int hit = scan_pairs(idx, T2, tb.S + (int64_t)mrow * tb.Wp, 0, L, nullptr, lane, n_loads);
      if (lane == 0) {
        if (hit >= 0) {
          st.sup[mrow] = 1;
          st.res[mrow] = hit;
        } else if (with_finalize) {   // a unsupported: remove it from dom(x) (Alg. 3 L3-4)
          const int x = tb.rowVar[mrow];
          const int a = mrow - tb.rowBase[x];
          atomicAnd(reinterpret_cast<unsigned long long *>(st.dom + tb.domOff[x] + (a >> 6)), ~(1ull << (a & 63)));
        }
      }
    }
    nmiss += tot;
    __syncthreads();   // s_cnt / s_miss are reused by the next round
  }
  if (lane == 0 && n_loads) atomicAdd(&c->scan_loads, (unsigned long long)n_loads);
  if (threadIdx.x == 0 && nmiss) atomicAdd(&c->nscan, nmiss);
  if (!with_finalize) return;
  // ---- completion: the last CTA writes the outputs
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&c->cta_done, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (use_state_out) {
    out_dom = st.out + 1;
    out_pruned = st.out + 1 + tb.Wd;
    out_status = reinterpret_cast<int32_t *>(st.out);
  }
  if (threadIdx.x == 0) {
    c->cta_done = 0;
    c->tph[3] = c->tph[4] = c->tph[5] = globaltimer();
  }
  wide_write_ok<kWideFiltTPB>(tb, st, out_dom, out_pruned, out_status, true, Lout, use_state_out != 0);
  if (threadIdx.x == 0) c->tph[6] = c->tph[7] = globaltimer();
}

}  // namespace ctk
