// ct_fast.cuh -- k_fast: one whole single-state propagation (Alg. 1-3,
// L131-244) in ONE cooperative launch, for tables whose support-row count fits
// every CTA's shared memory (R <= kLocalRowsMax; BASELINE config 3 has R = 800).
//
// What it changes against k_fused (ct_kernels.cuh), phase by phase:
//   ingest   (a2) computed redundantly by EVERY CTA into its own shared memory:
//                 Δ_x, D_x, |Δ_x|, |D_x| and the update / filter row lists are a
//                 few KB derived from Wd domain words, so the update starts
//                 without a grid barrier.  A row's list position is a popcount
//                 over the branch words (no row-by-row block scans).  Block 0
//                 alone also publishes the per-call state (din, varcnt, control
//                 fields, cleared flags) that k_finalize (sharded tables) and the
//                 stats read.
//   update   (a3-a5) one thread per active 16-byte block, support rows in
//                 register batches of kFastUnroll 16-byte loads (the engine that
//                 reached 95 % of the measured copy bandwidth in tools/upd_bench.cu),
//                 tiles of kFastTPB entries assigned statically; a tile only
//                 publishes its survivor COUNT (__syncthreads_count).  The CTA is
//                 kept small (<= 85 registers, a few KB of shared memory) so at
//                 least 6 fit an SM: with a per-SM cap near the average CTAs per
//                 SM the hardware spreads the grid unevenly and the same loop
//                 loses ~30 % (tools/upd_bench.cu, pad=40K rows).
//   -- grid barrier --
//   compaction (a4) after the barrier: every CTA sums the tile counts before its
//                 tiles (one L2 pass, block reduction), re-reads its blocks'
//                 new currTable words and writes the order-preserving index.
//                 No chained-scan look-back chain on the update's critical path.
//   probe    (a6a) residue probe (L220) together with the first of up to
//                 kSelfRounds warp rounds over the PRE-update index (complete
//                 before the barrier, a superset of the survivors), so a value
//                 whose support lies early in the table never waits for the new
//                 index.  Values still unresolved are queued.
//   -- grid barrier (only if the probe rounds cannot cover the index) --
//   scan     (a6b) (miss, chunk) units of the new compacted index, strided over
//                 all warps (chunk-major): the queue holds the values that need a
//                 long or full scan, which is where the whole grid pays off.
//   finalize (a6c-a8) by the LAST CTA to finish (a completion counter instead of
//                 a third barrier), from the lists it holds in shared memory.
//                 Only the synchronous call, whose outputs live in mapped host
//                 memory, pays the system-scope fence.
// Work counters are reduced per CTA before one global atomic each.
#pragma once
#include "ct_kernels.cuh"

namespace ctk {

constexpr int kLocalRowsMax = 4096;                    // R limit of the per-CTA lists
#ifndef CT_FAST_TPB
#define CT_FAST_TPB 256
#endif
#ifndef CT_FAST_UNROLL
#define CT_FAST_UNROLL 12   // support rows in flight per lane (sweep 8/12/16/24: profiles/r02_fast_unroll.md)
#endif
#ifndef CT_FAST_MINB
#define CT_FAST_MINB 3
#endif
constexpr int kFastTPB = CT_FAST_TPB;                  // k_fast threads per CTA = index entries per tile
constexpr int kFastWarps = kFastTPB / 32;
constexpr int kFastUnroll = CT_FAST_UNROLL;            // support rows in flight per update thread
#ifndef CT_PROBE_UNROLL
#define CT_PROBE_UNROLL 6
#endif
constexpr int kProbeUnroll = CT_PROBE_UNROLL;          // index entries per lane per probe round
constexpr int kFirstScanFast = 32 * kProbeUnroll;      // index entries per probe round
#ifndef CT_SCAN_U
#define CT_SCAN_U 4
#endif
constexpr int kScanFastU = CT_SCAN_U;                  // index entries per lane per scan unit
constexpr int kFastChunk = 32 * kScanFastU;            // index entries per scan unit
#ifndef CT_SCAN_GROUP
#define CT_SCAN_GROUP 8
#endif
constexpr int kScanGroup = CT_SCAN_GROUP;              // probe misses per scan unit (<= 32)
constexpr int kSelfRounds = (32 + kProbeUnroll - 1) / kProbeUnroll;   // probe rounds before a miss is queued (~1024 entries)


// Static shared state of one k_fast CTA (NW warps; k_wide uses the same ingest
// with 32 warps).
template <int NW>
struct FastShT {
  int dead, fail, noop, go, ngroups, nrows, nitems;
  int L, ident, par, Lout, nscan, last, below, anymiss;
  uint32_t nvalid;               // valid tuples of this CTA's blocks after the update
  const StateDev *in;            // the call's INPUT state (the state itself, or the source of ct_propagate_from)
  int from;                      // 1: input and output states differ
  long long calls;               // the input state's call count
  unsigned long long nbound;     // negative tables: the input's valid forbidden tuples (bounds this call's)
  int red[NW];                   // block-reduction scratch
  uint32_t woff[NW];
  uint64_t scan[NW];
  unsigned long long cnt[3];     // update loads, update writes, filter loads (this CTA)
};
using FastSh = FastShT<kFastWarps>;

// Dynamic shared memory of one k_fast CTA.
struct FastPtrs {
  uint64_t *din;      // [Wd] D_x = dom ∧ ¬removed
  uint64_t *dl;       // [Wd] Δ_x = dom ∧ removed; finalize reuses it for the new domains
  uint64_t *bw;       // [Wd] update-branch words (Δ_x or D_x if x in s_val, else 0)
  uint64_t *iw;       // [Wd] filter words (D_x if x in s_sup, else 0)
  int32_t *upos;      // [Wd+1] exclusive prefix of popc(bw)
  int32_t *ipos;      // [Wd+1] exclusive prefix of popc(iw)
  int32_t *wvar;      // [Wd] variable of each domain word
  uint32_t *ulist;    // [R]  update list (row | kEndBit | kInvBit)
  int32_t *items;     // [R]  filter items (support rows)
  int32_t *cd, *cs;   // [n]  |Δ_x|, |D_x|
  int32_t *vfl;       // [n]  bit 0 Δ-branch, bit 1 x in s_val
  int32_t *rb, *dof;  // [n+1] rowBase, domOff
};

__host__ __device__ inline size_t fast_smem_bytes(int n, int Wd, int R) {
  return (size_t)Wd * 32 + (size_t)(Wd + 1) * 8 + (size_t)Wd * 4 + (size_t)R * 8 + (size_t)(5 * n + 2) * 4 + 16;
}

__device__ __forceinline__ FastPtrs fast_ptrs(uint64_t *smem, const TableDev &tb) {
  FastPtrs p;
  const int Wd = tb.Wd, n = tb.n;
  p.din = smem;
  p.dl = p.din + Wd;
  p.bw = p.dl + Wd;
  p.iw = p.bw + Wd;
  p.upos = reinterpret_cast<int32_t *>(p.iw + Wd);
  p.ipos = p.upos + Wd + 1;
  p.wvar = p.ipos + Wd + 1;
  p.ulist = reinterpret_cast<uint32_t *>(p.wvar + Wd);
  p.items = reinterpret_cast<int32_t *>(p.ulist + tb.R);
  p.cd = p.items + tb.R;
  p.cs = p.cd + n;
  p.vfl = p.cs + n;
  p.rb = p.vfl + n;
  p.dof = p.rb + n + 1;
  return p;
}

// Variable owning support row r: the last x with rb[x] <= r.
__device__ __forceinline__ int row_var(const int32_t *rb, int n, int r) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (rb[mid] <= r) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

// Grid barrier of k_fast (all CTAs co-resident).  Arrival counters taken with
// acq_rel atomics (release: this CTA's writes are visible before it counts;
// acquire + the L1 invalidate ptxas emits with it: it then reads the others'
// writes), one arrival counter, and a generation word with one copy per group
// of CTAs in lines of its own that the waiting CTAs poll (polling a counter's
// own line, or 740 CTAs polling one line, slows the release).  Each CTA may
// add a small count (*extra_flag, a shared int; the sum over the grid must stay
// below 2^16) with its arrival (e.g. "I queued a probe miss").  The
// last arrival resets the counter, computes the one-bit `mode` =
// leader_mode(sum of the flags) and bumps the generation, whose low bit
// carries the mode (no second word to read after the release); every CTA returns the mode and
// `leader` tells the releasing CTA it was the last.  Counters return to 0
// after each barrier, so the memory only has to be zeroed once (at state
// creation).
__device__ __forceinline__ uint32_t atom_add_acqrel(uint32_t *p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void st_release_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// rank / count: this CTA's rank among the `count` CTAs that meet at `bar`
// (default: the whole grid; the grouped model fixpoint uses per-table groups).
template <typename F>
__device__ __forceinline__ int fast_grid_barrier_mode(uint32_t *bar, F leader_mode, int &leader, int *s_mode,
                                                      const int *extra_flag = nullptr, int rank = -1,
                                                      int count = -1) {
  if (rank < 0) rank = blockIdx.x;
  if (count < 0) count = gridDim.x;
  __syncthreads();   // also orders the block's writes of *extra_flag before thread 0 reads it
  if (threadIdx.x == 0) {
    const uint32_t extra = extra_flag ? (uint32_t)*(volatile const int *)extra_flag : 0u;
    uint32_t *cnt = bar;
    // the generation word has kBarGroups copies (lines 1..kBarGroups): each CTA
    // polls its group's copy, so the polling is spread over several L2 slices.
    // Its low bit carries the mode, so nobody reads a second word after release.
    uint32_t *mygen = bar + (1 + rank % kBarGroups) * kBarLine;
    const uint32_t my_gen = ld_acquire_u32(mygen);
    int last = 0;
    uint32_t g;
    // low 16 bits: arrivals; high 16 bits: the sum of the CTAs' `extra` values
    const uint32_t old = atom_add_acqrel(cnt, 1u + (extra << 16));
    if ((old & 0xffffu) == (uint32_t)count - 1) {
      *cnt = 0;
      g = ((((my_gen >> 1) + 1u) << 1)) | ((uint32_t)leader_mode((old >> 16) + extra) & 1u);
      __threadfence();   // one release fence for all the generation copies
      for (int q = 0; q < kBarGroups; ++q) *(volatile uint32_t *)(bar + (1 + q) * kBarLine) = g;
      last = 1;
    } else {
      SpinGuard sg;
      while ((g = ld_acquire_u32(mygen)) == my_gen) {
        __nanosleep(32);
        spin_check(sg, 3, my_gen, *(volatile uint32_t *)cnt, old);
      }
    }
    *s_mode = (int)(g & 1u);
    leader = last;
    if (blockIdx.x < kDiagCtas) g_bseq[blockIdx.x] += 1;
  }
  __syncthreads();
  return *s_mode;
}

__device__ __forceinline__ void fast_grid_barrier(uint32_t *bar, int rank = -1, int count = -1) {
  __shared__ int s_mode;
  int leader;
  fast_grid_barrier_mode(bar, [](uint32_t) { return 0; }, leader, &s_mode, nullptr, rank, count);
}

// Adds a per-thread counter to a global 64-bit counter with ONE atomic per CTA
// (warp sums, then thread 0); every thread of the block must call it.
__device__ __forceinline__ void cta_count(uint32_t v, unsigned long long *dst, FastSh &fs) {
  v = warp_sum_u32(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) fs.woff[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < kFastWarps; ++w) t += fs.woff[w];
    if (t) atomicAdd(dst, t);
  }
  __syncthreads();   // fs.woff is free again
}

// Block-wide sum over kFastTPB threads (uses fs.red; every thread gets the total).
__device__ __forceinline__ int fast_block_sum(int v, FastSh &fs) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) fs.red[threadIdx.x >> 5] = v;
  __syncthreads();
  int t = 0;
#pragma unroll
  for (int w = 0; w < kFastWarps; ++w) t += fs.red[w];
  return t;
}

// ------------------------------------------------------------------ a2: per-CTA ingest
// Same decisions as dev_ingest (Alg. 1 L1-3, Alg. 2), results kept in this
// CTA's shared memory; `writer` (block 0) also publishes the per-call state.
template <int NT = kFastTPB>
__device__ void cta_ingest(const TableDev &tb, const StateDev &st, const uint64_t *__restrict__ rem, int root_mode,
                           const FastPtrs &p, FastShT<NT / 32> &fs, bool writer, const uint64_t *gdom = nullptr,
                           const StateDev *src = nullptr) {
  Ctl *c = st.ctl;
  const StateDev &in = src ? *src : st;   // ct_propagate_from: read the source, write st
  const Ctl *ci = in.ctl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = tb.n, Wd = tb.Wd, R = tb.R;
  // the first domain word of this thread is loaded before anything waits, so
  // the control fields, the table metadata and the domains cost one round trip
  uint64_t dm0 = 0, rm0 = 0;
  int x0 = 0;
  if (tid < Wd) {
    dm0 = in.dom[tid];
    // model tables: a value is removed iff the shared (global) domain lost it
    rm0 = gdom ? ~__ldcg(gdom + tb.gword[tid]) : (rem ? rem[tid] : 0ull);
    x0 = tb.wordVar[tid];
  }
  if (tid == 0) {
    fs.dead = ci->dead;
    fs.fail = 0;
    fs.ngroups = 0;
    fs.anymiss = 0;
    fs.nvalid = 0;
    fs.L = ci->L;
    fs.ident = ci->identity;
    fs.par = ci->parity;
    fs.in = &in;
    fs.from = src != nullptr;
    fs.calls = ci->calls;
    fs.nbound = ci->nvalid;
    fs.cnt[0] = fs.cnt[1] = fs.cnt[2] = 0;
  }
  for (int i = tid; i <= n; i += NT) {
    p.rb[i] = tb.rowBase[i];
    p.dof[i] = tb.domOff[i];
  }
  for (int x = tid; x < n; x += NT) p.cd[x] = p.cs[x] = 0;
  __syncthreads();
  if (fs.dead) {
    if (tid == 0) {
      fs.go = 0;
      fs.noop = 0;
      if (writer) {
        c->skip = 1;
        c->noop = 0;
        c->fail_fast = 0;
      }
    }
    __syncthreads();
    return;
  }
  if (writer) {   // sup[0..R] = 0, 16 bytes per store (sup is 256-byte aligned)
    uint4 *s4 = reinterpret_cast<uint4 *>(st.sup);
    for (int r = tid; r < (R + 16) / 16; r += NT) s4[r] = make_uint4(0u, 0u, 0u, 0u);
    if (src) {   // the residues and the persistent control fields start as the source's
      for (int r = tid; r < R; r += NT) st.res[r] = in.res[r];
      if (tid == 0) {
        c->dead = ci->dead;
        c->parity = ci->parity;
        c->identity = ci->identity;
        c->L = ci->L;
        c->calls = ci->calls;
      }
    }
  }
  // Δ_x = removed ∧ dom, D_x = dom ∧ ¬removed, sizes (Alg. 1 L1-2)
  for (int k = tid; k < Wd; k += NT) {
    uint64_t dm = k == tid ? dm0 : in.dom[k];
    uint64_t rm = k == tid ? rm0 : (gdom ? ~__ldcg(gdom + tb.gword[k]) : (rem ? rem[k] : 0ull));
    if (tb.negative) {   // values the last filter pruned leave currTable now (ct_neg.cuh's pend)
      const uint64_t pd = in.pend[k];
      dm |= pd;
      rm |= pd;
    }
    const int x = k == tid ? x0 : tb.wordVar[k];
    const uint64_t delta = rm & dm, di = dm & ~rm;
    p.din[k] = di;
    p.dl[k] = delta;
    p.wvar[k] = x;
    if (writer) st.din[k] = di;
    if (delta) atomicAdd(&p.cd[x], __popcll(delta));
    if (di) atomicAdd(&p.cs[x], __popcll(di));
  }
  __syncthreads();
  // per variable: s_val (Δ_x ≠ ∅), branch (Alg. 2: Δ-branch iff |Δ_x| < |D_x|), s_sup (|D_x| > 1)
  for (int x = tid; x < n; x += NT) {
    const int cd = p.cd[x], cs = p.cs[x];
    const bool useDelta = use_delta(tb, x, cd, cs);
    p.vfl[x] = (useDelta ? 1 : 0) | (cd > 0 ? 2 : 0);
    if (cd > 0) atomicAdd(&fs.ngroups, 1);
    if (cs == 0) fs.fail = 1;                   // D_x empty -> no valid tuple
    if (writer) {
      st.varcnt[2 * x] = cd;
      st.varcnt[2 * x + 1] = cs;
    }
  }
  __syncthreads();
  if (tb.negative) {
    // count rows (ct_neg.cuh): the values of x are counted iff P_x = prod_{y != x}
    // |D_y| <= the input's |V| (which bounds this call's); vfl bit 2
    const unsigned long long B = fs.nbound;
    for (int x = tid; x < n; x += NT) {
      unsigned long long P = 1;   // saturates at B + 1
      for (int y = 0; y < n; ++y) {
        if (y == x) continue;
        const unsigned long long cy = (unsigned long long)p.cs[y];
        if (cy == 0) {
          P = 0;
          break;
        }
        if (P > B / cy) {
          P = B + 1;
          break;
        }
        P *= cy;
      }
      if (P <= B) p.vfl[x] |= 4;
    }
    if (writer)
      for (int r = tid; r < R; r += NT) st.cnt[r] = 0;   // read after the first grid barrier
    __syncthreads();
  }
  const bool fail = fs.fail != 0;
  const bool noop = (fs.ngroups == 0) && !root_mode;
  int nrows = 0, nitems = 0;
  if (!(fail || noop)) {
    // branch / item words and their exclusive popcount prefixes (variables are
    // contiguous word runs, so the prefix groups the lists by variable)
    int carry_u = 0, carry_i = 0;
    for (int base = 0; base < Wd; base += NT) {
      const int k = base + tid;
      int cu = 0, ci = 0;
      if (k < Wd) {
        const int x = p.wvar[k], fl = p.vfl[x];
        const uint64_t b = (fl & 2) ? ((fl & 1) ? p.dl[k] : p.din[k]) : 0ull;
        const uint64_t it = (tb.negative ? (fl & 4) != 0 : p.cs[x] > 1) ? p.din[k] : 0ull;
        p.bw[k] = b;
        p.iw[k] = it;
        cu = __popcll(b);
        ci = __popcll(it);
      }
      const uint64_t v = ((uint64_t)cu << 32) | (uint64_t)ci;
      uint64_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) fs.scan[warp] = x;
      __syncthreads();
      uint64_t wb = 0, tot = 0;
#pragma unroll
      for (int w = 0; w < NT / 32; ++w) {
        if (w < warp) wb += fs.scan[w];
        tot += fs.scan[w];
      }
      const uint64_t ex = wb + x - v;
      if (k < Wd) {
        p.upos[k] = carry_u + (int)(ex >> 32);
        p.ipos[k] = carry_i + (int)(ex & 0xffffffffu);
      }
      carry_u += (int)(tot >> 32);
      carry_i += (int)(tot & 0xffffffffu);
      __syncthreads();
    }
    if (tid == 0) {
      p.upos[Wd] = carry_u;
      p.ipos[Wd] = carry_i;
    }
    nrows = carry_u;
    nitems = carry_i;
    __syncthreads();
    // one task per (domain word, byte): emit the rows of its set bits in order
    for (int j = tid; j < 8 * Wd; j += NT) {
      const int k = j >> 3, sh = (j & 7) * 8;
      const int x = p.wvar[k];
      const int rbase = p.rb[x] + 64 * (k - p.dof[x]) + sh;
      const uint64_t below = sh ? ((1ull << sh) - 1) : 0ull;
      uint32_t ub = (uint32_t)(p.bw[k] >> sh) & 0xffu;
      if (ub) {
        int pos = p.upos[k] + __popcll(p.bw[k] & below);
        const int uend = p.upos[p.dof[x + 1]] - 1;   // last entry of x's group
        const uint32_t inv = (p.vfl[x] & 1) ? kInvBit : 0u;
        while (ub) {
          const int b = __ffs(ub) - 1;
          ub &= ub - 1;
          p.ulist[pos] = (uint32_t)(rbase + b) | inv | (pos == uend ? kEndBit : 0u);
          ++pos;
        }
      }
      uint32_t ib = (uint32_t)(p.iw[k] >> sh) & 0xffu;
      if (ib) {
        int pos = p.ipos[k] + __popcll(p.iw[k] & below);
        while (ib) {
          const int b = __ffs(ib) - 1;
          ib &= ib - 1;
          p.items[pos++] = rbase + b;
        }
      }
    }
  }
  if (tid == 0) {
    fs.nrows = nrows;
    fs.nitems = nitems;
    fs.noop = noop && !fail;
    fs.go = !(fail || noop);
    if (writer) {
      c->skip = 0;
      c->noop = noop && !fail;
      c->fail_fast = fail;
      c->ngroups = fs.ngroups;
      c->nrows = nrows;
      c->nitems = nitems;
      c->L_in = fs.L;
      c->L_out = 0;
      c->nscan = 0;
      c->tile_ctr = 0;   // k_fast: the scan's unit counter
      c->upd_loads = 0;
      c->upd_writes = 0;
      c->scan_loads = 0;
      c->gathered = 0;
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------------ a3: update of one index entry
// Alg. 2 for index entry k (one 16-byte block per thread).  The block dies
// early (Alg. 2) once no valid tuple is left in it (checked between
// batches).  Returns the number of valid tuples the block keeps.
__device__ __forceinline__ uint32_t fast_update_entry(const TableDev &tb, const StateDev &st, const FastSh &fs,
                                                  const uint32_t *__restrict__ ulist, int k, uint32_t &n_loads,
                                                  uint32_t &n_writes) {
  const int nrows = fs.nrows;
  const StateDev &in = *fs.in;
  const int32_t *__restrict__ idx_in = fs.par ? in.idx1 : in.idx0;
  ulonglong2 *__restrict__ T2 = reinterpret_cast<ulonglong2 *>(st.T);
  const int64_t Wp = tb.Wp;
  const int pid = fs.ident ? k : idx_in[k];
  const ulonglong2 tw = reinterpret_cast<const ulonglong2 *>(in.T)[pid];
  const uint64_t *__restrict__ col = tb.S + 2 * (int64_t)pid;
  uint64_t mx = ~0ull, my = ~0ull, ax = 0, ay = 0;
  int p0 = 0;
  for (; p0 < nrows; p0 += kFastUnroll) {
    if (((tw.x & mx) | (tw.y & my)) == 0) break;   // Alg. 2, per 16-byte block
    ulonglong2 v[kFastUnroll];
#pragma unroll
    for (int q = 0; q < kFastUnroll; ++q)
      v[q] = (p0 + q < nrows) ? ld_sup2(col + (int64_t)(ulist[p0 + q] & kRowMask) * Wp)
                              : make_ulonglong2(0ull, 0ull);
#pragma unroll
    for (int q = 0; q < kFastUnroll; ++q) {
      if (p0 + q < nrows) {
        const uint32_t e = ulist[p0 + q];
        ax |= v[q].x;
        ay |= v[q].y;
        if (e & kEndBit) {
          if (e & kInvBit) {
            mx &= ~ax;
            my &= ~ay;
          } else {
            mx &= ax;
            my &= ay;
          }
          ax = ay = 0;
        }
      }
    }
  }
  n_loads += 2 * min(p0, nrows);   // rows issued before the block died or the list ended
  const ulonglong2 nt = make_ulonglong2(tw.x & mx, tw.y & my);
  if (nt.x != tw.x || nt.y != tw.y || fs.from) {
    T2[pid] = nt;
    ++n_writes;
  }
  return (uint32_t)(__popcll(nt.x) + __popcll(nt.y));
}

// The update of a CTA's index range [k_lo, k_hi) with Q lanes per entry: when
// the index is short against the grid's threads (a small table with many
// support rows, or a state deep in a search), one thread per entry would walk
// all of the entry's update rows alone (t = 1e6, R = 800: 400 dependent-ish
// loads, the grid mostly idle).  Here the Q lanes of an entry split each
// variable's rows (lane j: rows j, j + Q, ...; kSplitU in flight), OR-reduce
// the group with shuffles and AND it in (Alg. 2: the same
// per-variable OR, complemented for the Δ-branch, ANDed over the changed
// variables); a block that died skips the rest (L175).  The variables' groups
// come from the ingest's per-word list positions (upos, dof): no group table.
#ifndef CT_SPLIT_U
#define CT_SPLIT_U 8
#endif
constexpr int kSplitU = CT_SPLIT_U;   // rows in flight per lane (sweep 4 / 8 / 16)
template <int Q>
__device__ __forceinline__ void fast_update_range_split(const TableDev &tb, const StateDev &st, const FastSh &fs,
                                                        const FastPtrs &p, int k_lo, int k_hi, uint32_t &n_loads,
                                                        uint32_t &n_writes, uint32_t &nv, int &kept) {
  const int tid = threadIdx.x, sub = tid & (Q - 1);
  const StateDev &in = *fs.in;
  const int32_t *__restrict__ idx_in = fs.par ? in.idx1 : in.idx0;
  const ulonglong2 *__restrict__ Tin = reinterpret_cast<const ulonglong2 *>(in.T);
  ulonglong2 *__restrict__ T2 = reinterpret_cast<ulonglong2 *>(st.T);
  const int64_t Wp = tb.Wp;
  const int n = tb.n;
  for (int base = k_lo; base < k_hi; base += kFastTPB / Q) {
    const int k = base + tid / Q;
    const bool valid = k < k_hi;
    int pid = 0;
    ulonglong2 tw = make_ulonglong2(0ull, 0ull);
    if (valid) {
      pid = fs.ident ? k : idx_in[k];
      tw = Tin[pid];
    }
    const uint64_t *__restrict__ col = tb.S + 2 * (int64_t)pid;
    uint64_t mx = ~0ull, my = ~0ull;
    bool live = valid && (tw.x | tw.y) != 0ull;
    for (int x = 0; x < n; ++x) {
      const int s0 = p.upos[p.dof[x]], s1 = p.upos[p.dof[x + 1]];
      if (s0 == s1) continue;   // x not in s_val (shared-memory values: uniform)
      uint64_t ax = 0, ay = 0;
      if (live) {
        for (int r0 = s0 + sub; r0 < s1; r0 += Q * kSplitU) {
          ulonglong2 v[kSplitU];
#pragma unroll
          for (int u = 0; u < kSplitU; ++u) {
            const int r = r0 + u * Q;
            v[u] = r < s1 ? ld_sup2(col + (int64_t)(p.ulist[r] & kRowMask) * Wp) : make_ulonglong2(0ull, 0ull);
            n_loads += r < s1 ? 2u : 0u;
          }
#pragma unroll
          for (int u = 0; u < kSplitU; ++u) {
            ax |= v[u].x;
            ay |= v[u].y;
          }
        }
      }
#pragma unroll
      for (int o = Q / 2; o > 0; o >>= 1) {
        ax |= __shfl_xor_sync(0xffffffffu, ax, o);
        ay |= __shfl_xor_sync(0xffffffffu, ay, o);
      }
      const uint64_t inv = (p.vfl[x] & 1) ? ~0ull : 0ull;   // Δ-branch: AND the complement
      mx &= ax ^ inv;
      my &= ay ^ inv;
      live = live && ((tw.x & mx) | (tw.y & my)) != 0ull;
    }
    uint32_t cnt = 0;
    if (valid && sub == 0) {
      const ulonglong2 nt = make_ulonglong2(tw.x & mx, tw.y & my);
      if (nt.x != tw.x || nt.y != tw.y || fs.from) {
        T2[pid] = nt;
        ++n_writes;
      }
      cnt = (uint32_t)(__popcll(nt.x) + __popcll(nt.y));
    }
    nv += cnt;
    kept += __syncthreads_count(cnt != 0);
  }
}

// ct_propagate_from: blocks outside the source's index are zero in the source
// but stale in the output, so each CTA zeroes the gaps between its own index
// entries (the last CTA with entries also after the last one; rank 0 all of
// them when the index is empty): disjoint ranges, no barrier.
__device__ __forceinline__ void fast_zero_gaps(const TableDev &tb, const StateDev &st, const FastSh &fs, int k_lo,
                                               int k_hi, int rank) {
  ulonglong2 *__restrict__ T2 = reinterpret_cast<ulonglong2 *>(st.T);
  const ulonglong2 z = make_ulonglong2(0ull, 0ull);
  const int W2 = tb.W2, L = fs.L;
  const bool last = (k_lo < k_hi && k_hi == L) || (L == 0 && rank == 0);
  if (fs.ident) {   // entries 0..L-1
    if (last)
      for (int b = L + threadIdx.x; b < W2; b += blockDim.x) T2[b] = z;
    return;
  }
  const int32_t *__restrict__ idx = fs.par ? fs.in->idx1 : fs.in->idx0;
  for (int k = k_lo + threadIdx.x; k < k_hi; k += blockDim.x) {
    const int prev = k == 0 ? -1 : idx[k - 1];
    const int cur = idx[k];
    for (int b = prev + 1; b < cur; ++b) T2[b] = z;
  }
  if (last)
    for (int b = (L > 0 ? idx[L - 1] + 1 : 0) + threadIdx.x; b < W2; b += blockDim.x) T2[b] = z;
}

// ------------------------------------------------------------------ a4: index entries of one CTA's range
// The survivors of entries [k_lo, k_hi) go to the new index at positions
// fs.below + rank (order-preserving: fs.below = survivors of all lower CTAs).
__device__ __forceinline__ void fast_compact_range(const TableDev &tb, const StateDev &st, FastSh &fs, int k_lo,
                                                   int k_hi) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const ulonglong2 *__restrict__ T2 = reinterpret_cast<const ulonglong2 *>(st.T);
  const int32_t *__restrict__ idx_in = fs.par ? fs.in->idx1 : fs.in->idx0;
  int32_t *__restrict__ idx_out = fs.par ? st.idx0 : st.idx1;
  int below = fs.below;
  for (int base = k_lo; base < k_hi; base += kFastTPB) {
    const int k = base + tid;
    int pid = 0;
    bool keep = false;
    if (k < k_hi) {
      pid = fs.ident ? k : idx_in[k];
      const ulonglong2 t = __ldcg(T2 + pid);
      keep = (t.x | t.y) != 0;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    __syncthreads();
    if (lane == 0) fs.woff[warp] = __popc(bal);
    __syncthreads();
    uint32_t off = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kFastWarps; ++w) {
      if (w < warp) off += fs.woff[w];
      all += fs.woff[w];
    }
    if (keep) idx_out[below + off + __popc(bal & lanemask_lt())] = pid;
    below += (int)all;
  }
}

// ------------------------------------------------------------------ a6b': filter by gathering the valid tuples
// Alg. 3 asks, per unresolved (x,a), whether currTable & supports[x,a] != 0,
// i.e. (L189-193) whether some VALID tuple holds value a at x.  The same answer
// for every value at once: walk the valid tuples and mark the values they hold.
// When the valid tuples are few against the scans (|V| sectors of cells vs
// misses x L_out x 16 bytes of support words -- the banded C3b call reads
// ~3 MB instead of ~0.8 GB) every CTA walks the valid tuples of its own update
// range (their blocks were written by the same threads), reads their cells
// (value offsets, tb.cells) and marks (x, tau[x]) in a shared-memory bitmap in
// the domain layout; each queued miss then reads its bit.  A value is marked
// iff a valid tuple holds it, so the verdicts are Alg. 3's; a marked value's
// residue becomes a block holding such a tuple.
__device__ void fast_gather_range(const TableDev &tb, const StateDev &st, const FastSh &fs, const FastPtrs &p,
                                  int k_lo, int k_hi, uint32_t &n_tuples) {
  const int tid = threadIdx.x, n = tb.n, Wd = tb.Wd;
  uint64_t *mark = p.bw;                                   // [Wd] (free after the ingest)
  int32_t *rres = reinterpret_cast<int32_t *>(p.ulist);    // [R]  (free after the update)
  for (int k = tid; k < Wd; k += kFastTPB) mark[k] = 0;
  __syncthreads();
  const ulonglong2 *__restrict__ T2 = reinterpret_cast<const ulonglong2 *>(st.T);
  const int32_t *__restrict__ idx_in = fs.par ? fs.in->idx1 : fs.in->idx0;
  const int cw = tb.cell_words, bits = tb.cell_bits, per = 32 / bits;
  const uint32_t cmask = (1u << bits) - 1u;
  // per thread: its entries' valid tuples in batches of kGatherBatch, every
  // batch's cell loads issued before any is used (one DRAM round trip per
  // batch instead of one per cell word)
  constexpr int kGatherBatch = 4;
  const auto mark_word = [&](uint32_t wv, int q, int pid) {
    for (int e = 0; e < per; ++e) {
      const int i = q * per + e;
      if (i >= n) break;
      const int v = (int)((wv >> (e * bits)) & cmask);
      uint64_t *mw = mark + p.dof[i] + (v >> 6);
      if (!((*(volatile uint64_t *)mw >> (v & 63)) & 1ull)) {   // most values repeat: skip the atomic
        // the one thread that sets the bit records the residue
        unsigned int *m32 = reinterpret_cast<unsigned int *>(mw) + ((v & 63) >> 5);
        const unsigned int bit = 1u << (v & 31);
        if (!(atomicOr(m32, bit) & bit)) rres[p.rb[i] + v] = pid;
      }
    }
  };
  for (int k = k_lo + tid; k < k_hi; k += kFastTPB) {
    const int pid = fs.ident ? k : idx_in[k];
    const ulonglong2 t = T2[pid];   // written by this thread's own update
    uint64_t m0 = t.x, m1 = t.y;
    while (m0 | m1) {
      int64_t j[kGatherBatch];
      int nb = 0;
#pragma unroll
      for (int b = 0; b < kGatherBatch; ++b) {
        j[b] = -1;
        if (m0) {
          j[b] = (int64_t)(2 * pid) * 64 + (__ffsll(m0) - 1);
          m0 &= m0 - 1;
        } else if (m1) {
          j[b] = (int64_t)(2 * pid + 1) * 64 + (__ffsll(m1) - 1);
          m1 &= m1 - 1;
        }
        nb += j[b] >= 0;
      }
      n_tuples += nb;
      if (cw == 2) {   // the common case (n <= 8 at 8 bits, n <= 4 at 16): 2 words per tuple, 8 loads in flight
        uint2 w[kGatherBatch];
#pragma unroll
        for (int b = 0; b < kGatherBatch; ++b)
          w[b] = j[b] >= 0 ? __ldg(reinterpret_cast<const uint2 *>(tb.cells + j[b] * 2)) : make_uint2(0u, 0u);
#pragma unroll
        for (int b = 0; b < kGatherBatch; ++b)
          if (j[b] >= 0) {
            mark_word(w[b].x, 0, pid);
            mark_word(w[b].y, 1, pid);
          }
      } else {
        for (int q = 0; q < cw; ++q) {
          uint32_t w[kGatherBatch];
#pragma unroll
          for (int b = 0; b < kGatherBatch; ++b) w[b] = j[b] >= 0 ? __ldg(tb.cells + j[b] * cw + q) : 0u;
#pragma unroll
          for (int b = 0; b < kGatherBatch; ++b)
            if (j[b] >= 0) mark_word(w[b], q, pid);
        }
      }
    }
  }
  __syncthreads();
  for (int m = tid; m < fs.nscan; m += kFastTPB) {
    const int row = __ldcg(st.scanlist + m);
    const int x = row_var(p.rb, n, row), a = row - p.rb[x];
    if ((mark[p.dof[x] + (a >> 6)] >> (a & 63)) & 1ull) {
      st.sup[row] = 1;
      st.res[row] = rres[row];
    }
  }
}

// ------------------------------------------------------------------ a6a: probe of one row
// Alg. 3 L3 for one (x,a) by a warp: is some block b with T[b] & S[x,a][b] != 0?
// Lane 0's residue block r (L220; -1 = none) is tested together with the first
// round; each round covers kFirstScanFast entries of the PRE-update index (its
// blocks are a superset of the survivors, and it is complete before the
// barrier; nullptr = identity), at most kSelfRounds rounds.  Returns the hit
// block (r if the residue hit, else the lowest hit of the round) or -1.
__device__ __forceinline__ int probe_row(const int32_t *__restrict__ idx_old, int Lin,
                                         const ulonglong2 *__restrict__ T2, const uint64_t *__restrict__ srow,
                                         int r, int off, int lane, uint32_t &nl, int round0 = 0, int rstep = 1) {
  for (int round = round0; round < kSelfRounds; round += rstep) {
    const int kb = round * kFirstScanFast;
    if (kb >= Lin) break;
    // every load is issued unconditionally (out-of-range entries re-read a
    // valid one and are masked after): loads inside per-entry branches would
    // each wait for the previous one
    int pid[kProbeUnroll];
    uint64_t v[kProbeUnroll];
#pragma unroll
    for (int q = 0; q < kProbeUnroll; ++q) {
      const int j = kb + q * 32 + lane;
      int k = off + (j < Lin ? j : 0);
      if (k >= Lin) k -= Lin;
      pid[q] = idx_old ? idx_old[k] : k;
    }
    const int rr = r >= 0 ? r : pid[0];
    const ulonglong2 tr = __ldcg(T2 + rr);
    const ulonglong2 sr = ld_sup2(srow + 2 * (int64_t)rr);
    ulonglong2 t[kProbeUnroll], s[kProbeUnroll];
#pragma unroll
    for (int q = 0; q < kProbeUnroll; ++q) {
      t[q] = __ldcg(T2 + pid[q]);
      s[q] = ld_sup2(srow + 2 * (int64_t)pid[q]);
    }
    const bool rh = round == round0 && r >= 0 && ((tr.x & sr.x) | (tr.y & sr.y)) != 0;
    if (round == round0 && r >= 0) nl += 2;
#pragma unroll
    for (int q = 0; q < kProbeUnroll; ++q) {
      const bool in = kb + q * 32 + lane < Lin;
      v[q] = in ? ((t[q].x & s[q].x) | (t[q].y & s[q].y)) : 0ull;
    }
    nl += 2 * min(kFirstScanFast, Lin - kb);
    if (__any_sync(0xffffffffu, rh)) return __shfl_sync(0xffffffffu, r, 0);
    int hit = -1;
#pragma unroll
    for (int q = kProbeUnroll - 1; q >= 0; --q) {
      const unsigned b = __ballot_sync(0xffffffffu, v[q] != 0);
      if (b) hit = __shfl_sync(0xffffffffu, pid[q], __ffs(b) - 1);
    }
    if (hit >= 0) return hit;
  }
  return -1;
}

// ------------------------------------------------------------------ a10 over NVLink: in-kernel flag exchange
// Tuple-range shards combine their R+1 flag bytes ("row r
// supported by a valid tuple of my slice", "my slice is non-empty") by OR.
// With peer inboxes attached (ct_peer_attach) the finalizer CTA of k_fast does
// it itself instead of a separate all-reduce + finalize launch: it stores its
// flags into slot (epoch & 1, rank) of every rank's inbox over NVLink (peer
// pointers from CUDA IPC), publishes them with one system-scope release per
// rank, waits (acquire) for every rank's flags of the same epoch in its own
// inbox, and ORs them into st.sup.  Every rank makes the same sequence of
// sharded calls (SPMD), so the epochs agree; two slots suffice because a rank
// can write epoch e + 2 only after every rank published e + 1, i.e. finished
// reading e.  Returns the combined non-empty flag.  All threads of the CTA.
__device__ int peer_combine(const TableDev &tb, const StateDev &st) {
  const int tid = threadIdx.x, G = tb.peer_n, me = tb.peer_rank, pw = tb.peer_pw;
  const int nw = (tb.R + 1 + 3) >> 2;   // the flag bytes as 32-bit words (st.sup is padded to 256 bytes)
  // drawn by CTA 0 at kernel entry (k_fast), visible here after the completion counter
  const uint32_t ep = __ldcg(&st.ctl->peer_ep), slot = ep & 1u;
  const uint32_t *sw = reinterpret_cast<const uint32_t *>(st.sup);
  for (int g = 0; g < G; ++g) {
    uint32_t *dst = tb.peers[g] + ((size_t)slot * G + me) * pw;
    for (int w = tid; w < nw; w += blockDim.x) dst[w] = __ldcg(sw + w);
  }
  __syncthreads();
  const size_t fbase = (size_t)2 * G * pw;
  if (tid < G) {
    // the block barrier orders every thread's payload stores before this
    // thread's system-scope release (cumulative), which publishes them
    st_release_sys_u32(tb.peers[tid] + fbase + ((size_t)slot * G + me) * 32, ep);
    const uint32_t *f = tb.inbox + fbase + ((size_t)slot * G + tid) * 32;   // sender tid's flag here
    // the other ranks may reach this call a while later (their host work
    // between calls): a much longer limit than the grid barriers' watchdog
    const unsigned long long t0 = globaltimer();
    uint32_t n = 0;
    while (ld_acquire_sys_u32(f) != ep) {
      if ((++n & 1023u) == 0 && globaltimer() - t0 > 120000000000ull) {   // 120 s
        spin_report(5, ep, (unsigned long long)tid, 0);
        __trap();
      }
    }
  }
  __syncthreads();
  uint32_t *out = reinterpret_cast<uint32_t *>(st.sup);
  for (int w = tid; w < nw; w += blockDim.x) {
    uint32_t acc = 0;
    for (int g = 0; g < G; ++g) acc |= __ldcv(tb.inbox + ((size_t)slot * G + g) * pw + w);
    out[w] = acc;
  }
  __syncthreads();
  return *reinterpret_cast<volatile const uint8_t *>(st.sup + tb.R) != 0;
}

// ------------------------------------------------------------------ a6c-a8: finalize from shared memory
// Alg. 3 L3-4 over the filter items this CTA listed in its ingest: a value of
// x in s_sup leaves the domain iff its row is unsupported; lastDom <- dom.
// Returns the status; on CT_OK the new domains are left in p.dl (s_nd).
__device__ int cta_finalize(const TableDev &tb, const StateDev &st, const FastPtrs &p, const FastSh &fs,
                            uint64_t *__restrict__ out_dom, uint64_t *__restrict__ out_pruned,
                            int32_t *__restrict__ out_status, bool sys_fence, int nonempty = -1) {
  // ct_propagate_from: the output state's persistent fields are the input's,
  // advanced by this call (in place this is the same as updating them)
  constexpr int NT = kFastTPB;
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, Wd = tb.Wd;
  int status;
  if (fs.dead) status = -5;              // CT_ESTATE
  else if (fs.fail) status = 1;          // CT_FAIL: some D_x empty
  else if (fs.noop) status = 0;
  else if (nonempty >= 0) status = nonempty ? 0 : 1;   // shards: the combined flag (peer_combine)
  else status = fs.Lout > 0 ? 0 : 1;     // currTable empty <=> FAIL (Alg. 1 L5)
  if (status != 0) {
    if (tid == 0) {
      if (status == 1 || fs.from) {   // a dead source leaves a dead output
        c->dead = 1;
        c->calls = fs.calls + (status == 1 ? 1 : 0);
      }
      c->last_status = status;
      if (out_status) *out_status = status;
    }
    return status;
  }
  uint64_t *s_nd = p.dl;
  for (int k = tid; k < Wd; k += NT) s_nd[k] = p.din[k];
  __syncthreads();
  if (!fs.noop) {
    for (int i = tid; i < fs.nitems; i += NT) {
      const int r = p.items[i];
      if (!__ldcg(st.sup + r)) {                   // x in s_sup (Alg. 3 L1), a unsupported
        const int x = row_var(p.rb, tb.n, r);
        const int a = r - p.rb[x];
        const int w = p.dof[x] + (a >> 6);
        smem_clear_bit(s_nd + w, a & 63);
      }
    }
    __syncthreads();
  }
  for (int k = tid; k < Wd; k += NT) {
    const uint64_t nd = s_nd[k];
    st.dom[k] = nd;
    if (out_dom) out_dom[k] = nd;
    if (out_pruned) out_pruned[k] = p.din[k] & ~nd;
  }
  // the status word completes the host-mapped synchronous call: every output
  // write must be visible system-wide before it (block barrier, then ONE
  // cumulative system-scope fence by the thread that writes the status)
  __syncthreads();
  if (tid == 0) {
    if (sys_fence) __threadfence_system();
    if (!fs.noop && tb.use_index) {
      c->parity = fs.par ^ 1;
      c->L = fs.Lout;
      c->identity = 0;
    } else if (fs.from) {   // the source's index (copied by fast_call) and geometry
      c->parity = fs.par;
      c->L = fs.L;
      c->identity = fs.ident;
    }
    if (fs.from) c->dead = 0;
    c->calls = fs.calls + 1;
    c->last_status = 0;
    if (out_status) *out_status = 0;
  }
  return 0;
}


// The finalize of a negative table on the k_fast path (ct_neg.cuh's
// k_neg_finalize from this CTA's shared memory): (x, a) leaves the domain iff
// its count of valid forbidden tuples reached P_x = prod_{y != x} |D_y|; FAIL
// iff a domain empties; the pruned values are kept in `pend` so the next call
// removes their tuples; |V| = the CTAs' popcounts (tcnt[G + j]).
__device__ int cta_finalize_neg(const TableDev &tb, const StateDev &st, const FastPtrs &p, const FastSh &fs,
                                uint64_t *__restrict__ out_dom, uint64_t *__restrict__ out_pruned,
                                int32_t *__restrict__ out_status, bool sys_fence, int G) {
  constexpr int NT = kFastTPB;
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, Wd = tb.Wd, n = tb.n;
  __shared__ int s_empty;
  int status = fs.dead ? -5 : (fs.fail ? 1 : 0);
  uint64_t *s_nd = p.dl;
  unsigned long long *s_P = reinterpret_cast<unsigned long long *>(p.iw);   // [n] (n <= Wd; free after the ingest)
  for (int k = tid; k < Wd; k += NT) s_nd[k] = p.din[k];
  if (tid == 0) s_empty = 0;
  __syncthreads();
  if (status == 0 && !fs.noop) {
    for (int x = tid; x < n; x += NT) {   // exact for the counted variables (P_x <= |V| < 2^63)
      unsigned long long P = 1;
      for (int y = 0; y < n; ++y)
        if (y != x) P = (P > (1ull << 62) / max(1, p.cs[y])) ? (1ull << 62) : P * (unsigned long long)p.cs[y];
      s_P[x] = P;
    }
    __syncthreads();
    for (int i = tid; i < fs.nitems; i += NT) {
      const int r = p.items[i];
      const int x = row_var(p.rb, n, r);
      if (__ldcg(st.cnt + r) >= s_P[x]) {   // every assignment of D with x = a is forbidden
        const int a = r - p.rb[x];
        smem_clear_bit(s_nd + p.dof[x] + (a >> 6), a & 63);
      }
    }
    __syncthreads();
    for (int x = tid; x < n; x += NT) {
      uint64_t any = 0;
      for (int w = p.dof[x]; w < p.dof[x + 1]; ++w) any |= s_nd[w];
      if (!any) s_empty = 1;
    }
    __syncthreads();
    if (s_empty) status = 1;
  }
  if (status != 0) {
    if (tid == 0) {
      if (status == 1 || fs.from) {
        c->dead = 1;
        c->calls = fs.calls + (status == 1 ? 1 : 0);
      }
      c->last_status = status;
      if (out_status) *out_status = status;
    }
    return status;
  }
  for (int k = tid; k < Wd; k += NT) {
    const uint64_t nd = s_nd[k], di = p.din[k];
    st.dom[k] = nd;
    st.pend[k] = di & ~nd;
    if (out_dom) out_dom[k] = nd;
    if (out_pruned) out_pruned[k] = di & ~nd;
  }
  __syncthreads();
  if (tid == 0) {
    if (!fs.noop) {
      const uint32_t *tcnt = reinterpret_cast<const uint32_t *>(st.tilestat);
      unsigned long long nv = 0;
      for (int j = 0; j < G; ++j) nv += __ldcg(tcnt + G + j);
      c->nvalid = nv;
    } else if (fs.from) {
      c->nvalid = fs.nbound;
    }
    if (sys_fence) __threadfence_system();
    if (!fs.noop && tb.use_index) {
      c->parity = fs.par ^ 1;
      c->L = fs.Lout;
      c->identity = 0;
    } else if (fs.from) {
      c->parity = fs.par;
      c->L = fs.L;
      c->identity = fs.ident;
    }
    if (fs.from) c->dead = 0;
    c->calls = fs.calls + 1;
    c->last_status = 0;
    if (out_status) *out_status = 0;
  }
  return 0;
}

// ------------------------------------------------------------------ k_fast
// Cooperative launch (all CTAs co-resident), kFastTPB threads, dynamic smem
// fast_smem_bytes(n, Wd, R).  with_finalize = 0 for sharded tables (the flags are
// OR-combined across shards first and k_finalize runs after).  Filter items
// are spread CTA-major (item i -> CTA i % grid) so few items probe on many SMs.
// One whole single-state call by the G CTAs (ranks 0..G-1) that share the
// state: k_fast runs it on the whole grid, the grouped model fixpoint
// (ct_model.cuh) on one table's group of CTAs.  gdom != nullptr: a model
// table (removals = values the shared domains lost; no outputs).  Returns the
// call's status on the CTA that finalized (the last to finish), kNotFinalizer
// on the others; with_finalize = 0 (sharded tables) always kNotFinalizer.
constexpr int kNotFinalizer = -100;
__device__ __forceinline__ int fast_call(const TableDev &tb, const StateDev &st, FastSh &fs, const FastPtrs &p,
                                         const uint64_t *__restrict__ removed, const uint64_t *gdom, int root_mode,
                                         int with_finalize, uint64_t *__restrict__ out_dom,
                                         uint64_t *__restrict__ out_pruned, int32_t *__restrict__ out_status,
                                         int use_state_out, const int rank, const int G,
                                         const StateDev *src = nullptr) {
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool t0 = rank == 0 && tid == 0;
  int fstatus = kNotFinalizer;
  // phase timestamps of rank 0 go straight to tph[] (no registers held)
  if (t0) c->tph[0] = globaltimer();
  cta_ingest(tb, st, removed, root_mode, p, fs, rank == 0, gdom, src);
  if (t0) {
    const unsigned long long t = globaltimer();
    for (int i = 1; i < 6; ++i) c->tph[i] = t;
  }

  bool compact_after = false;   // the leader of a no-miss call writes its index entries after finalizing
  int leader_k_lo = 0, leader_k_hi = 0;
  if (fs.go) {
    uint32_t *__restrict__ tcnt = reinterpret_cast<uint32_t *>(st.tilestat);
    // ---- update (a3): CTA c owns index entries [c·ts, (c+1)·ts), ts = ceil(L / G)
    // (an equal share per CTA, so every SM streams the same number of blocks),
    // walked kFastTPB at a time; the CTA's survivor count goes to tcnt[c]
    const int ts = (fs.L + G - 1) / G;
    const int k_lo = min(fs.L, rank * ts), k_hi = min(fs.L, k_lo + ts);
    uint32_t n_loads = 0, n_writes = 0, f_loads = 0;
    {
      int kept = 0;
      uint32_t nv = 0;   // valid tuples of this thread's blocks (the gather filter's cost model)
      // lanes per index entry: 1, or more when the index is short against the grid
      int q = 1;
      while (q < 32 && (int64_t)(2 * q) * fs.L <= (int64_t)G * kFastTPB) q *= 2;
      switch (q) {
        case 1:
          for (int base = k_lo; base < k_hi; base += kFastTPB) {
            const int k = base + tid;
            const uint32_t cnt = k < k_hi ? fast_update_entry(tb, st, fs, p.ulist, k, n_loads, n_writes) : 0u;
            nv += cnt;
            kept += __syncthreads_count(cnt != 0);
          }
          break;
        case 2: fast_update_range_split<2>(tb, st, fs, p, k_lo, k_hi, n_loads, n_writes, nv, kept); break;
        case 4: fast_update_range_split<4>(tb, st, fs, p, k_lo, k_hi, n_loads, n_writes, nv, kept); break;
        case 8: fast_update_range_split<8>(tb, st, fs, p, k_lo, k_hi, n_loads, n_writes, nv, kept); break;
        case 16: fast_update_range_split<16>(tb, st, fs, p, k_lo, k_hi, n_loads, n_writes, nv, kept); break;
        default: fast_update_range_split<32>(tb, st, fs, p, k_lo, k_hi, n_loads, n_writes, nv, kept); break;
      }
      if (tid == 0) tcnt[rank] = (uint32_t)kept;
      if (tb.gather || tb.negative) {
        nv = warp_sum_u32(nv);
        if (lane == 0) atomicAdd(&fs.nvalid, nv);
      }
      if (fs.from) fast_zero_gaps(tb, st, fs, k_lo, k_hi, rank);
    }
    // update work counters now, while CTAs still finish at different times,
    // reduced per CTA first: when every CTA finishes its (short) update at
    // once, one same-address atomic per warp serialised into ~3.5 us before
    // barrier 1
    {
      const uint32_t wl = warp_sum_u32(n_loads), ww = warp_sum_u32(n_writes);
      if (lane == 0) fs.red[warp] = (int)wl;
      if (lane == 0) fs.woff[warp] = ww;
      __syncthreads();
      if (tid == 0) {
        unsigned long long tl = 0, tw = 0;
        for (int w = 0; w < kFastWarps; ++w) {
          tl += (uint32_t)fs.red[w];
          tw += fs.woff[w];
        }
        if (tl) atomicAdd(&c->upd_loads, tl);
        if (tw) atomicAdd(&c->upd_writes, tw);
      }
      __syncthreads();   // fs.red / fs.woff are free again
    }

    const ulonglong2 *__restrict__ T2 = reinterpret_cast<const ulonglong2 *>(st.T);
    fast_grid_barrier(st.bar, rank, G);
    if (t0) c->tph[2] = globaltimer();

    // ---- compaction (a4), part A: L_out and this CTA's prefix from the
    // per-CTA counts (the index entries themselves are written later, off the
    // critical path of a call without probe misses)
    {
      int tot = 0, below = 0;
      for (int j = tid; j < G; j += kFastTPB) {
        const int v = (int)__ldcg(tcnt + j);
        tot += v;
        if (j < rank) below += v;
      }
      tot = fast_block_sum(tot, fs);
      below = fast_block_sum(below, fs);
      if (tid == 0) {
        fs.Lout = tot;
        fs.below = below;
        if (rank == 0) c->L_out = tot;
      }
    }
    if ((tb.gather || tb.negative) && tid == 0) {   // this CTA's valid tuples -> the grid's (read later)
      tcnt[G + rank] = (uint32_t)fs.nvalid;
    }
    __syncthreads();
    if (tb.negative) {
      // ---- counting filter of a negative table (ct_neg.cuh): cnt[row] += popc(T & S[row])
      // over this CTA's own update range (blocks its own threads just wrote),
      // per-row partial sums in shared memory, one global atomic per row
      uint32_t *s_cnt = p.ulist;   // [nitems] (free after the update)
      for (int i = tid; i < fs.nitems; i += kFastTPB) s_cnt[i] = 0;
      __syncthreads();
      const int32_t *__restrict__ idx_in = fs.par ? fs.in->idx1 : fs.in->idx0;
      const int nit = fs.nitems;
      // a warp holds 32 x kNegE of the range's blocks in registers (lane l:
      // entries l, l + 32, ...) and streams the rows i = warp, warp + 8, ...
      // over them, two rows' loads in flight; row i belongs to one warp, so
      // its partial sum is a plain shared-memory update
      constexpr int kNegE = 8;
      for (int base = k_lo; base < k_hi; base += 32 * kNegE) {
        int pid[kNegE];
        ulonglong2 t[kNegE];
#pragma unroll
        for (int j = 0; j < kNegE; ++j) {
          const int k = base + 32 * j + lane;
          pid[j] = k < k_hi ? (fs.ident ? k : idx_in[k]) : -1;
          t[j] = pid[j] >= 0 ? T2[pid[j]] : make_ulonglong2(0ull, 0ull);
          if (pid[j] >= 0 && (t[j].x | t[j].y) == 0) pid[j] = -1;   // a dead block loads no row
        }
        for (int i = warp; i < nit; i += 2 * kFastWarps) {
          const int i2 = i + kFastWarps;
          const uint64_t *__restrict__ r0 = tb.S + (int64_t)p.items[i] * tb.Wp;
          const uint64_t *__restrict__ r1 = tb.S + (int64_t)p.items[i2 < nit ? i2 : i] * tb.Wp;
          ulonglong2 a[kNegE], b[kNegE];
#pragma unroll
          for (int j = 0; j < kNegE; ++j) {
            a[j] = pid[j] >= 0 ? ld_sup2(r0 + 2 * (int64_t)pid[j]) : make_ulonglong2(0ull, 0ull);
            b[j] = (pid[j] >= 0 && i2 < nit) ? ld_sup2(r1 + 2 * (int64_t)pid[j]) : make_ulonglong2(0ull, 0ull);
          }
          uint32_t ca = 0, cb = 0;
#pragma unroll
          for (int j = 0; j < kNegE; ++j) {
            ca += __popcll(t[j].x & a[j].x) + __popcll(t[j].y & a[j].y);
            cb += __popcll(t[j].x & b[j].x) + __popcll(t[j].y & b[j].y);
            if (pid[j] >= 0) f_loads += i2 < nit ? 4 : 2;
          }
          ca = __reduce_add_sync(0xffffffffu, ca);
          cb = __reduce_add_sync(0xffffffffu, cb);
          if (lane == 0) {
            s_cnt[i] += ca;
            if (i2 < nit) s_cnt[i2] += cb;
          }
        }
      }
      __syncthreads();
      for (int i = tid; i < nit; i += kFastTPB)
        if (s_cnt[i]) atomicAdd(st.cnt + p.items[i], (unsigned long long)s_cnt[i]);
      if (tb.use_index) fast_compact_range(tb, st, fs, k_lo, k_hi);
      if (t0) c->tph[3] = c->tph[4] = c->tph[5] = globaltimer();
      cta_count(f_loads, &c->scan_loads, fs);
      goto completion;
    }

    // ---- probe (a6a): residue + up to kSelfRounds rounds over the pre-update index.
    // Item i goes to CTA i % G; when there are few items per CTA, wpi warps of
    // the CTA share one item and take its rounds round-robin (warp q: rounds q,
    // q + wpi, ...), so an item costs one round trip instead of several.
    const int Lout = fs.Lout;
    const bool compact = tb.use_index != 0;
    const int32_t *__restrict__ idx = compact ? (fs.par ? st.idx0 : st.idx1) : nullptr;
    const int32_t *__restrict__ idx_old = fs.ident ? nullptr : (fs.par ? fs.in->idx1 : fs.in->idx0);
    const int Ls = compact ? Lout : tb.W2;
    const bool may_miss = fs.L > kSelfRounds * kFirstScanFast;   // the probe cannot cover the index
    if (t0) st.sup[tb.R] = Lout > 0;
    if (Lout > 0) {
      const int per_cta = (fs.nitems - rank + G - 1) / G;   // items of this CTA
      const int wpi = per_cta <= 1 ? kFastWarps : per_cta <= 2 ? kFastWarps / 2 : 1;
      const int slots = kFastWarps / wpi, slot = warp / wpi, q = warp % wpi;
      for (int j0 = 0; j0 < per_cta; j0 += slots) {
        const int j = j0 + slot;
        const int item = rank + j * G;
        int hit = -1, row = 0, r = -1;
        if (j < per_cta) {
          row = p.items[item];
          r = (tb.use_res && lane == 0 && q == 0) ? st.res[row] : -1;
          uint32_t nl = 0;
          hit = probe_row(idx_old, fs.L, T2, tb.S + (int64_t)row * tb.Wp, r, 0, lane, nl, q, wpi);
          if (lane == 0) {
            f_loads += nl;
            if (hit >= 0) {
              st.sup[row] = 1;
              if (hit != r) st.res[row] = hit;
            }
          }
        }
        if (wpi == 1) {
          if (j < per_cta && lane == 0 && hit < 0 && may_miss) {
            st.scanlist[atomicAdd(&c->nscan, 1)] = row;
            fs.anymiss = 1;
          }
        } else {
          // the item is a miss only if none of its wpi warps found a support
          __syncthreads();
          if (lane == 0) fs.red[warp] = hit >= 0;
          __syncthreads();
          if (j < per_cta && q == 0 && lane == 0 && may_miss) {
            int any = 0;
            for (int w = warp; w < warp + wpi; ++w) any |= fs.red[w];
            if (!any) {
              st.scanlist[atomicAdd(&c->nscan, 1)] = row;
              fs.anymiss = 1;
            }
          }
        }
      }
    }
    if (t0) c->tph[3] = c->tph[4] = globaltimer();
    cta_count(lane == 0 ? f_loads : 0u, &c->scan_loads, fs);   // probe rounds
    f_loads = 0;
    // ---- scan (a6b): misses x chunks of the compacted index, from entry 0.
    // The barrier's last arrival knows every probe is done: with no miss it
    // releases the others with mode 1 (they write their index entries and
    // exit) and finalizes at once, then writes its own entries.
    if (Lout > 0 && may_miss) {
      int leader = 0;
      const int mode = fast_grid_barrier_mode(st.bar, [](uint32_t misses) { return misses == 0 ? 1 : 0; }, leader,
                                              &fs.nscan, &fs.anymiss, rank, G);
      if (t0) c->tph[4] = globaltimer();
      if (mode == 1) {
        if (t0) c->tph[5] = globaltimer();   // no scan phase
        if (tid == 0) fs.last = leader;
        __syncthreads();
        if (!fs.last) {
          if (tb.use_index) fast_compact_range(tb, st, fs, k_lo, k_hi);
          return kNotFinalizer;
        }
        compact_after = tb.use_index != 0;
        leader_k_lo = k_lo;
        leader_k_hi = k_hi;
        goto finalize;
      }
      // misses: scan them (Alg. 3 over the new index) or gather the valid
      // tuples' values (fast_gather_range) -- whichever reads fewer bytes.  Both
      // inputs are final after the probe barrier, so every CTA decides alike.
      if (tb.gather) {
        __syncthreads();   // every thread has read the barrier's mode from fs.nscan
        if (tid == 0) fs.nscan = __ldcg(&c->nscan);
        unsigned long long v = 0;
        for (int j = tid; j < G; j += kFastTPB) v += __ldcg(tcnt + G + j);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        __syncthreads();
        if (lane == 0) fs.scan[warp] = v;
        __syncthreads();
        v = 0;
#pragma unroll
        for (int w = 0; w < kFastWarps; ++w) v += fs.scan[w];
        const unsigned long long scan_bytes = (unsigned long long)fs.nscan * (unsigned long long)Ls * 16ull;
        const unsigned long long gather_bytes = v * 32ull + (unsigned long long)Ls * 16ull;
        if (gather_bytes < scan_bytes) {
          if (tb.use_index) fast_compact_range(tb, st, fs, k_lo, k_hi);
          uint32_t ng = 0;
          fast_gather_range(tb, st, fs, p, k_lo, k_hi, ng);
          cta_count(ng, &c->gathered, fs);
          if (t0) c->tph[5] = globaltimer();
          goto completion;
        }
      }
      // the whole new index first (the scans read it)
      if (tb.use_index) fast_compact_range(tb, st, fs, k_lo, k_hi);
      fast_grid_barrier(st.bar, rank, G);
      if (tid == 0) fs.nscan = __ldcg(&c->nscan);
      __syncthreads();
      const int nscan = fs.nscan;
      // work unit = (chunk of kFastChunk index entries, group of kScanGroup misses),
      // chunk-major.  A warp loads the chunk's index entries and currTable
      // words ONCE and then streams the support words of every still
      // unresolved miss of its group over them (the next miss's words are in
      // flight while the current one is tested), so the currTable / index
      // traffic is amortised over the group and each miss costs one round trip.
      const int ngrp = (nscan + kScanGroup - 1) / kScanGroup;
      const int nch = (Ls + kFastChunk - 1) / kFastChunk;
      const int64_t total = (int64_t)nch * ngrp;
      // units handed out dynamically (one atomic per unit and warp): their cost
      // varies with how many misses of the group are still open, and a
      // static split of ~2-3 units per warp left the last warps ~40 us behind;
      // small groups keep one unit short (each open miss costs a round trip)
      for (;;) {
        int64_t u = 0;
        if (lane == 0) u = atomicAdd(&c->tile_ctr, 1);
        u = __shfl_sync(0xffffffffu, (int)u, 0);
        if (u >= total) break;
        const int chunk = (int)(u / ngrp), grp = (int)(u - (int64_t)chunk * ngrp);
        const int k0 = chunk * kFastChunk;
        const int m = grp * kScanGroup + lane;
        const int rowl = (lane < kScanGroup && m < nscan) ? __ldcg(st.scanlist + m) : -1;
        const int fl = rowl >= 0 ? *(volatile const uint8_t *)(st.sup + rowl) : 1;
        unsigned todo = __ballot_sync(0xffffffffu, fl == 0);
        if (!todo) continue;
        int pid[kScanFastU];
        ulonglong2 t[kScanFastU];
#pragma unroll
        for (int q = 0; q < kScanFastU; ++q) {
          const int k = k0 + q * 32 + lane;
          const int kk = k < Ls ? k : k0;
          pid[q] = idx ? __ldcg(idx + kk) : kk;
        }
#pragma unroll
        for (int q = 0; q < kScanFastU; ++q) t[q] = T2[pid[q]];
        const int nwords = 2 * min(kFastChunk, Ls - k0);
        int row = __shfl_sync(0xffffffffu, rowl, __ffs(todo) - 1);
        ulonglong2 sc[kScanFastU];
#pragma unroll
        for (int q = 0; q < kScanFastU; ++q) sc[q] = ld_sup2(tb.S + (int64_t)row * tb.Wp + 2 * (int64_t)pid[q]);
        while (todo) {
          const unsigned rest = todo & (todo - 1);
          int row_n = row;
          ulonglong2 sn[kScanFastU];
          if (rest) {
            row_n = __shfl_sync(0xffffffffu, rowl, __ffs(rest) - 1);
#pragma unroll
            for (int q = 0; q < kScanFastU; ++q)
              sn[q] = ld_sup2(tb.S + (int64_t)row_n * tb.Wp + 2 * (int64_t)pid[q]);
          }
          int hit = -1;
#pragma unroll
          for (int q = kScanFastU - 1; q >= 0; --q) {
            const bool in = k0 + q * 32 + lane < Ls;
            const uint64_t v = in ? ((t[q].x & sc[q].x) | (t[q].y & sc[q].y)) : 0ull;
            const unsigned b = __ballot_sync(0xffffffffu, v != 0);
            if (b) hit = __shfl_sync(0xffffffffu, pid[q], __ffs(b) - 1);
          }
          if (lane == 0) {
            f_loads += nwords;
            if (hit >= 0) {
              st.sup[row] = 1;
              st.res[row] = hit;
            }
          }
          todo = rest;
          row = row_n;
          if (rest) {
#pragma unroll
            for (int q = 0; q < kScanFastU; ++q) sc[q] = sn[q];
          }
        }
      }
    }
    if (!(Lout > 0 && may_miss) && tb.use_index)
      fast_compact_range(tb, st, fs, k_lo, k_hi);   // no scan phase: write the index now
    if (t0) c->tph[5] = globaltimer();
    // scan work counter, one atomic per CTA
    cta_count(lane == 0 ? f_loads : 0u, &c->scan_loads, fs);
  } else if (fs.from && fs.noop) {
    // ct_propagate_from with nothing to propagate: the output becomes a copy of
    // the source (its index entries and their blocks, the gaps zeroed)
    const int ts = (fs.L + G - 1) / G;
    const int k_lo = min(fs.L, rank * ts), k_hi = min(fs.L, k_lo + ts);
    const StateDev &in = *fs.in;
    const int32_t *__restrict__ idx_in = fs.par ? in.idx1 : in.idx0;
    int32_t *__restrict__ idx_out = fs.par ? st.idx1 : st.idx0;
    for (int k = k_lo + tid; k < k_hi; k += kFastTPB) {
      const int pid = fs.ident ? k : idx_in[k];
      reinterpret_cast<ulonglong2 *>(st.T)[pid] = reinterpret_cast<const ulonglong2 *>(in.T)[pid];
      if (!fs.ident) idx_out[k] = pid;
    }
    fast_zero_gaps(tb, st, fs, k_lo, k_hi, rank);
  }

  // ---- completion: the last CTA to get here finalizes
completion:
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    fs.last = atomicAdd(&c->cta_done, 1) == G - 1;
  }
  __syncthreads();
  if (!fs.last) return kNotFinalizer;
  __threadfence();
  if (tid == 0) c->cta_done = 0;
finalize:
  if (tid == 0) c->tph[6] = globaltimer();
  if (with_finalize) {
    if (use_state_out) {
      out_dom = st.out + 1;
      out_pruned = st.out + 1 + tb.Wd;
      out_status = reinterpret_cast<int32_t *>(st.out);
    }
    // with_finalize == 2: tuple-range shards with peer inboxes -- combine the
    // flags over NVLink first (every rank agrees on dead / fail / noop, so
    // they all skip the exchange alike)
    const int ne = (with_finalize == 2 && !(fs.dead || fs.fail || fs.noop)) ? peer_combine(tb, st) : -1;
    fstatus = tb.negative ? cta_finalize_neg(tb, st, p, fs, out_dom, out_pruned, out_status, use_state_out != 0, G)
                          : cta_finalize(tb, st, p, fs, out_dom, out_pruned, out_status, use_state_out != 0, ne);
  }
  if (tid == 0) c->tph[7] = globaltimer();
  if (compact_after) {   // the leader's own index entries, after the outputs
    __syncthreads();
    fast_compact_range(tb, st, fs, leader_k_lo, leader_k_hi);
  }
  return fstatus;
}

// grid = co-resident CTAs (cooperative launch), kFastTPB threads, dynamic smem
// fast_smem_bytes(n, Wd, R).
// A small removal bitmap passed by value with the launch (async calls whose
// removal sits in host memory): no copy node, no cross-stream event.
constexpr int kRemArgWords = 16;
struct RemArg {
  uint64_t w[kRemArgWords];
  int32_t n;   // words in use; 0: take `removed`
};

__global__ void __launch_bounds__(kFastTPB, CT_FAST_MINB) k_fast(TableDev tb, const StateDev *__restrict__ states,
                                                   const uint64_t *__restrict__ removed, int root_mode,
                                                   int with_finalize, uint64_t *__restrict__ out_dom,
                                                   uint64_t *__restrict__ out_pruned,
                                                   int32_t *__restrict__ out_status, int use_state_out,
                                                   const StateDev *__restrict__ src_state,
                                                   const __grid_constant__ RemArg ra) {
  extern __shared__ __align__(16) uint64_t smem[];
  if (ra.n) removed = ra.w;
  __shared__ FastSh fs;
  __shared__ StateDev s_st, s_src;   // the states' pointers live in shared memory, not in registers
  if (threadIdx.x == 0) {
    s_st = states[0];
    if (src_state) s_src = src_state[0];
    // tuple-range shards combining over NVLink: every call draws the next
    // epoch (dead / no-op calls too, alike on every rank); the finalizer reads it
    if (with_finalize == 2 && blockIdx.x == 0) s_st.ctl->peer_ep = atomicAdd(tb.peer_epoch, 1u) + 1u;
  }
  __syncthreads();
  fast_call(tb, s_st, fs, fast_ptrs(smem, tb), removed, nullptr, root_mode, with_finalize, out_dom, out_pruned,
            out_status, use_state_out, (int)blockIdx.x, (int)gridDim.x, src_state ? &s_src : nullptr);
}

}  // namespace ctk
