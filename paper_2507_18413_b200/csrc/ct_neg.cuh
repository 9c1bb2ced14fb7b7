// ct_neg.cuh -- negative tables (PAPER.md L66-68 footnote: "a
// table explicitly listing the disallowed tuples is said negative").
//
// The tuples are FORBIDDEN assignments; rel(c) = (product of the initial
// domains) minus the list.  By GAC's definition (L52-55) value a of x is
// supported iff some assignment of the current domains with x = a is not
// forbidden, i.e. iff
//     cnt[x,a] = |{ valid forbidden tuples with tau[x] = a }|  <  P_x = prod_{y != x} |D_y|.
// currTable keeps the valid forbidden tuples exactly as for a positive table
// (the list is deduplicated at creation, so a bit is one distinct assignment),
// and updateTable (Alg. 2) is unchanged -- it runs through k_ingest / k_update.
// Only filterDomains differs: residues cannot witness a support, so the filter
// COUNTS popc(currTable & supports[x,a]) over the active index.  A row needs
// counting only if P_x <= |V| (|V| = valid forbidden tuples; the previous
// call's |V| bounds this call's), which is what makes negative tables cheap
// while the domains are large.  One call:
//   k_ingest    (shared)  Δ / D_x / branch / update rows; a value the last call
//                         pruned is still in currTable and is fed back as a
//                         removal (StateDev::pend) so its tuples leave now
//   k_update    (shared)  T &= mask over the active index + compaction
//   k_neg_plan  (1 CTA)   P_x (saturating), the count-row list, cnt = 0
//   k_neg_count (grid)    cnt[row] += popc(T & S[row]) and |V| over the index:
//                         (index chunk x row group) work items, the chunk's
//                         currTable blocks held in registers across its rows,
//                         per-row partial sums in shared memory
//   k_neg_finalize (1 CTA) prune cnt >= P_x; FAIL iff a domain empties; outputs
// Single-state calls only (no batches, no sharding: counts would need a SUM
// combine, not the positive table's OR).
#pragma once
#include "ct_kernels.cuh"

namespace ctk {

constexpr int kNegTPB = 256;
constexpr int kNegE = 4;                          // index entries (16-byte blocks) per thread per chunk
constexpr int kNegChunk = kNegTPB * kNegE;        // entries per work item
constexpr int kNegGroupRows = 4096;               // count rows per work item (shared-memory partial sums)
constexpr unsigned long long kProdCap = 1ull << 62;

__device__ __forceinline__ unsigned long long mul_sat(unsigned long long a, unsigned long long b) {
  if (a == 0 || b == 0) return 0;
  return (a > kProdCap / b) ? kProdCap : a * b;
}

__device__ __forceinline__ bool neg_go(const Ctl *c) {
  return !(__ldcg(&c->skip) | __ldcg(&c->noop) | __ldcg(&c->fail_fast));
}

// One CTA (kIngestTPB threads), dynamic smem (n + 2) * 8 bytes.
__global__ void __launch_bounds__(kIngestTPB) k_neg_plan(TableDev tb, const StateDev *__restrict__ states) {
  extern __shared__ __align__(16) unsigned long long s_sz[];   // [n] |D_x|
  __shared__ uint64_t s_warp[kIngestTPB / 32];
  const StateDev st = states[0];
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, n = tb.n;
  if (!neg_go(c)) {
    if (tid == 0) c->nitems = 0;
    return;
  }
  for (int x = tid; x < n; x += kIngestTPB) s_sz[x] = (unsigned long long)__ldcg(st.varcnt + 2 * x + 1);
  __syncthreads();
  const unsigned long long bound = __ldcg(&c->nvalid);   // >= this call's |V|
  for (int x = tid; x < n; x += kIngestTPB) {
    unsigned long long p = 1;
    for (int y = 0; y < n; ++y)
      if (y != x) p = mul_sat(p, s_sz[y]);
    st.prod[x] = p;
  }
  __syncthreads();
  // count rows: (x, a) with a in D_x and P_x <= bound, in row order
  uint64_t carry = 0;
  for (int base = 0; base < tb.R; base += kIngestTPB) {
    const int r = base + tid;
    bool f = false;
    if (r < tb.R) {
      const int x = tb.rowVar[r];
      const int a = r - tb.rowBase[x];
      const uint64_t w = __ldcg(st.din + tb.domOff[x] + (a >> 6));
      f = ((w >> (a & 63)) & 1) && __ldcg(st.prod + x) <= bound;
      st.cnt[r] = 0;
    }
    uint64_t total;
    const uint64_t ex = block_excl_scan<kIngestTPB>((uint64_t)f, s_warp, total) + carry;
    if (f) st.items[(int)ex] = r;
    carry += total;
  }
  if (tid == 0) {
    c->nitems = (int32_t)carry;
    c->nvalid_new = 0;
    c->scan_loads = 0;
  }
}

// Grid of kNegTPB-thread CTAs (persistent over work items).
__global__ void __launch_bounds__(kNegTPB) k_neg_count(TableDev tb, const StateDev *__restrict__ states) {
  __shared__ uint32_t s_cnt[kNegGroupRows];
  __shared__ uint32_t s_nv;
  const StateDev st = states[0];
  Ctl *c = st.ctl;
  if (!neg_go(c)) return;
  const int tid = threadIdx.x, lane = tid & 31;
  const bool compact = tb.use_index != 0;
  const int L = compact ? __ldcg(&c->L_out) : tb.W2;
  const int32_t *__restrict__ idx = compact ? (__ldcg(&c->parity) ? st.idx0 : st.idx1) : nullptr;
  const int nitems = __ldcg(&c->nitems);
  const int nchunks = (L + kNegChunk - 1) / kNegChunk;
  if (nchunks == 0) return;
  // row groups: enough work items to cover the grid, each group's partial sums
  // in shared memory; |V| is counted by the group-0 items only
  int ngroups = max(1, (nitems + kNegGroupRows - 1) / kNegGroupRows);
  ngroups = max(ngroups, min(max(nitems, 1), (int)gridDim.x / nchunks));
  const int gsize = (max(nitems, 1) + ngroups - 1) / ngroups;
  const ulonglong2 *__restrict__ T2 = reinterpret_cast<const ulonglong2 *>(st.T);
  const int32_t *__restrict__ items = st.items;
  if (tid == 0) s_nv = 0;
  unsigned long long loads = 0;
  for (int w = blockIdx.x; w < nchunks * ngroups; w += gridDim.x) {
    const int chunk = w % nchunks, group = w / nchunks;
    const int r0 = min(nitems, group * gsize), r1 = min(nitems, r0 + gsize);
    for (int i = tid; i < r1 - r0; i += kNegTPB) s_cnt[i] = 0;
    int pid[kNegE];
    ulonglong2 t[kNegE];
    uint32_t nv = 0;
#pragma unroll
    for (int q = 0; q < kNegE; ++q) {
      const int k = chunk * kNegChunk + q * kNegTPB + tid;
      pid[q] = k < L ? (idx ? idx[k] : k) : -1;
      t[q] = pid[q] >= 0 ? T2[pid[q]] : make_ulonglong2(0ull, 0ull);
      nv += __popcll(t[q].x) + __popcll(t[q].y);
    }
    if (group == 0) {
      nv = __reduce_add_sync(0xffffffffu, nv);
      if (lane == 0 && nv) atomicAdd(&s_nv, nv);
    }
    __syncthreads();   // s_cnt zeroed
    int i = r0;
    for (; i + 1 < r1; i += 2) {   // two rows in flight: 2 * kNegE independent 16-byte loads
      const uint64_t *__restrict__ s0 = tb.S + (int64_t)__ldg(items + i) * tb.Wp;
      const uint64_t *__restrict__ s1 = tb.S + (int64_t)__ldg(items + i + 1) * tb.Wp;
      ulonglong2 a[kNegE], b[kNegE];
#pragma unroll
      for (int q = 0; q < kNegE; ++q) {
        a[q] = pid[q] >= 0 ? ld_sup2(s0 + 2 * (int64_t)pid[q]) : make_ulonglong2(0ull, 0ull);
        b[q] = pid[q] >= 0 ? ld_sup2(s1 + 2 * (int64_t)pid[q]) : make_ulonglong2(0ull, 0ull);
      }
      uint32_t ca = 0, cb = 0;
#pragma unroll
      for (int q = 0; q < kNegE; ++q) {
        ca += __popcll(t[q].x & a[q].x) + __popcll(t[q].y & a[q].y);
        cb += __popcll(t[q].x & b[q].x) + __popcll(t[q].y & b[q].y);
      }
      ca = __reduce_add_sync(0xffffffffu, ca);
      cb = __reduce_add_sync(0xffffffffu, cb);
      if (lane == 0) {
        if (ca) atomicAdd(&s_cnt[i - r0], ca);
        if (cb) atomicAdd(&s_cnt[i + 1 - r0], cb);
      }
    }
    if (i < r1) {
      const uint64_t *__restrict__ s0 = tb.S + (int64_t)__ldg(items + i) * tb.Wp;
      uint32_t ca = 0;
#pragma unroll
      for (int q = 0; q < kNegE; ++q) {
        const ulonglong2 a = pid[q] >= 0 ? ld_sup2(s0 + 2 * (int64_t)pid[q]) : make_ulonglong2(0ull, 0ull);
        ca += __popcll(t[q].x & a.x) + __popcll(t[q].y & a.y);
      }
      ca = __reduce_add_sync(0xffffffffu, ca);
      if (lane == 0 && ca) atomicAdd(&s_cnt[i - r0], ca);
    }
    if (tid == 0) loads += 2ull * (uint64_t)(r1 - r0) * (uint64_t)min(kNegChunk, L - chunk * kNegChunk);
    __syncthreads();
    for (int j = tid; j < r1 - r0; j += kNegTPB)
      if (s_cnt[j]) atomicAdd(st.cnt + __ldg(items + r0 + j), (unsigned long long)s_cnt[j]);
    __syncthreads();   // s_cnt is reused by the next work item
  }
  if (tid == 0) {
    if (s_nv) atomicAdd(&c->nvalid_new, (unsigned long long)s_nv);
    if (loads) atomicAdd(&c->scan_loads, loads);
  }
}

// One CTA (kFinTPB threads), dynamic smem finalize_smem_bytes(n, Wd).  Prunes
// (x, a) with cnt >= P_x; FAIL iff a domain empties (then every domain does:
// all assignments of D are forbidden).  Outputs as dev_finalize.
__global__ void __launch_bounds__(kFinTPB) k_neg_finalize(TableDev tb, const StateDev *__restrict__ states,
                                                          uint64_t *__restrict__ out_dom,
                                                          uint64_t *__restrict__ out_pruned,
                                                          int32_t *__restrict__ out_status, int use_state_out) {
  extern __shared__ __align__(16) uint64_t smem[];
  const StateDev st = states[0];
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, n = tb.n, Wd = tb.Wd;
  if (use_state_out) {
    out_dom = st.out + 1;
    out_pruned = st.out + 1 + Wd;
    out_status = reinterpret_cast<int32_t *>(st.out);
  }
  uint64_t *s_nd = smem;
  __shared__ int s_status, s_noop, s_empty;
  if (tid == 0) {
    const int skip = __ldcg(&c->skip), ff = __ldcg(&c->fail_fast), noop = __ldcg(&c->noop);
    s_status = skip ? -5 : (ff ? 1 : 0);
    s_noop = noop;
    s_empty = 0;
  }
  for (int k = tid; k < Wd; k += kFinTPB) s_nd[k] = __ldcg(st.din + k);
  __syncthreads();
  int status = s_status;
  const bool noop = s_noop != 0;
  if (status == 0 && !noop) {
    const int nitems = __ldcg(&c->nitems);
    for (int i = tid; i < nitems; i += kFinTPB) {
      const int r = __ldcg(st.items + i);
      const int x = tb.rowVar[r];
      if (__ldcg(st.cnt + r) >= __ldcg(st.prod + x)) {   // every assignment with x = a is forbidden
        const int a = r - tb.rowBase[x];
        const int w = tb.domOff[x] + (a >> 6);
        smem_clear_bit(s_nd + w, a & 63);
      }
    }
    __syncthreads();
    for (int x = tid; x < n; x += kFinTPB) {
      uint64_t any = 0;
      for (int w = tb.domOff[x]; w < tb.domOff[x + 1]; ++w) any |= s_nd[w];
      if (!any) s_empty = 1;
    }
    __syncthreads();
    if (s_empty) status = 1;
  }
  if (status != 0) {
    if (tid == 0) {
      if (status == 1) {
        c->dead = 1;
        c->calls += 1;
      }
      c->last_status = status;
      if (out_status) *out_status = status;
    }
    return;
  }
  for (int k = tid; k < Wd; k += kFinTPB) {
    const uint64_t nd = s_nd[k], di = __ldcg(st.din + k);
    st.dom[k] = nd;
    st.pend[k] = di & ~nd;   // pruned now, their tuples leave currTable next call
    if (out_dom) out_dom[k] = nd;
    if (out_pruned) out_pruned[k] = di & ~nd;
  }
  __syncthreads();
  if (tid == 0) {
    if (out_status) __threadfence_system();   // outputs visible before the status word (sync path)
    if (!noop) {
      c->nvalid = __ldcg(&c->nvalid_new);
      if (tb.use_index) {
        c->parity ^= 1;
        c->L = __ldcg(&c->L_out);
        c->identity = 0;
      }
    }
    c->calls += 1;
    c->last_status = 0;
    if (out_status) *out_status = 0;
  }
}

}  // namespace ctk
