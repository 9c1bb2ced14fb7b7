// ct_kernels.cuh -- sm_100a device code of the Compact-Table propagation path.
//
// One propagation of a state (Alg. 1) runs five phases:
//
//   ingest   (a2)  removed ∧ dom -> Δ_x, D_x = dom ∧ ¬removed, |Δ_x|, |D_x|,
//                  s_val, s_sup (Alg. 1 L1-3), the Δ/dom branch of each changed
//                  var (Alg. 2), the update row list and the filter items.
//   update   (a3-a5) for every active 16-byte currTable block b:
//                  T[b] &= AND_{x in s_val} (Δ ? ¬OR_{a∈Δx} S[x,a][b] : OR_{a∈Dx} S[x,a][b])
//                  (Alg. 2; the per-variable ANDs commute, so all s_val vars
//                  are folded in one streaming pass), then order-preserving
//                  compaction of the non-zero blocks (the RSparseBitSet index)
//                  by a single-pass chained scan; L_out = 0 <=> FAIL (Alg. 1 L5).
//   probe    (a6a) per (x,a), x in s_sup: residue probe (L220), then the first
//                  kFirstScan index entries, warp-cooperatively.
//   scan     (a6b) probe misses: chunked warp-parallel intersect of S[x,a] with
//                  currTable over the compacted index (__ballot_sync "any").
//   finalize (a6c-a8) prune unsupported values (Alg. 3 L3-4), lastDom <- dom,
//                  outputs and status.
//
// Two launch shapes share these device functions:
//   * k_fused      one cooperative persistent kernel for a single state; the
//                  phases are separated by software grid barriers (all blocks
//                  are co-resident by construction of the cooperative launch);
//   * k_ingest / k_update / k_probe / k_scan / k_finalize -- one kernel per
//                  phase with a state dimension (blockIdx.y), used for batches
//                  of independent states (a9).
// Tuple-range sharding (a10) stops before finalize: the per-row flags sup[]
// written by probe/scan are OR-combined across shards (NCCL) and finalize runs
// as its own kernel.
#pragma once
#include <cstdint>

namespace ctk {

constexpr int kUpdTPB = 256;      // update threads per block = index entries per tile
constexpr int kIngestTPB = 1024;  // block size of the standalone ingest / finalize kernels
constexpr int kProbeTPB = 256;
constexpr int kScanTPB = 256;
constexpr int kFinTPB = 1024;
constexpr int kFusedTPB = 256;    // k_fused block size (= kUpdTPB)
#ifndef CT_UPD_UNROLL
#define CT_UPD_UNROLL 4
#endif
constexpr int kUpdUnroll = CT_UPD_UNROLL;   // support rows in flight per thread in update
constexpr int kScanUnroll = 4;    // index entries (16-byte blocks) per lane per scan round
constexpr int kFirstScan = 32 * kScanUnroll * 2;     // entries probe scans itself (2 rounds)
constexpr int kScanChunk = 32 * kScanUnroll * 2;     // entries per scan work unit (2 rounds)

constexpr int32_t kStar = INT32_MIN;          // short-table wildcard cell (CT_STAR, include/ct.h)
constexpr uint32_t kRowMask = 0x3FFFFFFFu;   // update-list entry: row id
constexpr uint32_t kEndBit = 1u << 30;        //   last row of its variable's group
constexpr uint32_t kInvBit = 1u << 31;        //   group uses the Δ-branch (complemented)

// k_fast's grid barrier: kBarGroups arrival counters and one top counter, each
// in its own 128-byte line, and the generation word in another.
constexpr int kBarGroups = 16;
constexpr int kBarLine = 32;                              // uint32 words per 128-byte line
constexpr int kBarWords = (kBarGroups + 3) * kBarLine;   // + one line for the leader's mode word

constexpr unsigned long long kFlagAgg = 1ull << 62;   // chained-scan tile status
constexpr unsigned long long kFlagPre = 2ull << 62;

// Device view of an immutable table (one shard).
struct TableDev {
  const uint64_t *S;        // supports [R][Wp], row = rowBase[x] + (a - lo[x])
  const int32_t *rowBase;   // [n+1]   first support row of each var (_supportJmp, L286)
  const int32_t *domOff;    // [n+1]   first domain word of each var
  const int32_t *wordVar;   // [Wd]    var owning each domain word
  const int32_t *rowVar;    // [R]     var owning each support row
  int32_t n, R, Wd;
  int32_t W;                // currTable words of this shard
  int32_t W2;               // 16-byte blocks of this shard = ceil(W/2) (index granularity)
  int64_t Wp;               // padded row stride in words (multiple of 16)
  int32_t policy;           // CT_POLICY_*
  int32_t use_res, use_index;
  int32_t ntiles_max;       // ceil(W2 / kUpdTPB)
  const int32_t *gword;     // [Wd] model tables only: global domain word of each domain word
  const int32_t *gshared;   // [Wd] model tables only: 1 if another table also constrains the word's variable
  const uint32_t *cells;    // [t_local][cell_words] or nullptr: tuple j's value offsets v - lo_i, cell_bits
                            // each, packed LSB-first (the gather filter of k_fast, ct_fast.cuh)
  int32_t cell_bits;        // 8 or 16
  int32_t cell_words;       // uint32 words per tuple
  int32_t gather;           // 1: k_fast's filter may use the cells (use_gather); they may also exist for
                            // the batch update's cell route only (ct_batch.cuh)
  // a10 over NVLink peer memory (ct_peer_attach): k_fast's finalizer CTA
  // exchanges the shard flags with every rank and ORs them itself (peer_combine)
  uint32_t *const *peers;   // [peer_n] every rank's exchange inbox (this rank's included), or nullptr
  uint32_t *inbox;          // this rank's inbox: payload [2][peer_n][peer_pw] words, flags [2][peer_n][32]
  uint32_t *peer_epoch;     // this rank's count of exchanged calls (identical on every rank: SPMD order)
  int32_t peer_n, peer_rank, peer_pw;
  int32_t negative;         // 1: a negative table (f4) on the k_fast path: counting filter (ct_fast.cuh)
  const int32_t *domOnly;   // [n] or nullptr: 1 if x's column has a star cell (short tables, f4), so the
                            // Δ-branch (which drops every tuple whose row has a removed value) is unsound
                            // for x: a star tuple is in every row of x and must survive
};

// Alg. 2: Δ-branch iff |Δ_x| < |D_x| (CT_POLICY_AUTO), or forced by the
// policy -- never for a starred column of a short table.
__device__ __forceinline__ bool use_delta(const TableDev &tb, int x, int cd, int cs) {
  return (tb.policy == 2 || (tb.policy == 0 && cd < cs)) && !(tb.domOnly && tb.domOnly[x]);
}

// Per-state control block (device).  The first fields up to last_status persist
// across calls (they are part of the state); the rest is per-call scratch.
struct Ctl {
  int32_t dead;        // 1 after CT_FAIL until restored by a copy
  int32_t parity;      // which index buffer holds the active index
  int32_t identity;    // 1: active index is implicitly 0..L-1 (root, or use_index=0)
  int32_t L;           // active 16-byte blocks (index entries)
  long long calls;
  int32_t last_status;
  // ---- per call
  int32_t skip;        // dead at entry
  int32_t noop;        // no changed variable: state already at fixpoint
  int32_t fail_fast;   // some D_x empty
  int32_t nrows;       // update-list length
  int32_t ngroups;     // |s_val|
  int32_t nitems;      // filter items
  int32_t L_in;
  int32_t L_out;       // active blocks after the update (this shard)
  int32_t tile_ctr;
  int32_t nscan;       // probe misses queued for scanning
  unsigned long long upd_loads;    // support words loaded by update (this call)
  unsigned long long upd_writes;   // currTable blocks rewritten by update
  unsigned long long scan_loads;   // support words loaded by probe + scan
  uint32_t bar_count;  // software grid barrier of k_fused
  uint32_t bar_gen;
  unsigned long long tph[8];   // phase timestamps (%globaltimer, ns); see ct_stats.phase_ns
  int32_t cta_done;    // k_fast: CTAs done with the filter; the last one finalizes
                       // and resets it to 0 (so a copied state always holds 0)
  uint32_t peer_ep;     // k_fast with peer inboxes: this call's exchange epoch (CTA 0 draws it at entry)
  // negative tables (ct_neg.cuh): valid forbidden tuples after the last call
  // (persists; copied with the state) and this call's running count
  unsigned long long nvalid;
  unsigned long long nvalid_new;
  unsigned long long gathered;   // k_fast gather filter: valid tuples whose cells it read (this call)
};
static_assert(sizeof(Ctl) <= 256, "Ctl must fit its 256-byte slot");

struct StateDev {
  Ctl *ctl;
  uint64_t *T;              // currTable [Wp]
  int32_t *idx0, *idx1;     // compacted index double buffer [Wp/2]
  int32_t *res;             // residues [R] (block ids of this shard)
  uint64_t *dom;            // current domains [Wd] (lastDom between calls)
  uint64_t *din;            // dom after the caller's removals [Wd]
  int32_t *ulist;           // update row list [R]
  int32_t *items;           // filter items (support rows) [R]
  int32_t *scanlist;        // probe misses [R]
  uint8_t *sup;             // [R+1]: per-row "supported", [R] = "currTable non-empty"
  int32_t *varcnt;          // [2n]: |Δ_x|, |D_x|
  unsigned long long *tilestat;  // [ntiles_max] chained-scan tile status
  uint64_t *out;            // [1 + 2 Wd]: status word, dom, pruned (sync path)
  uint64_t *slot;           // [Wd] removed (sync path, filled by an H2D copy)
  uint32_t *bar;            // [kBarWords] k_fast hierarchical grid barrier (zeroed at creation)
  // negative tables only (nullptr otherwise; ct_neg.cuh)
  uint64_t *pend;           // [Wd] values the last filter pruned whose tuples are still in currTable
  unsigned long long *cnt;  // [R] per-row count of valid forbidden tuples (this call)
  unsigned long long *prod; // [n] P_x = prod over y != x of |D_y| (saturating)
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ unsigned long long ld_acquire(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// Streaming read of support words: read-only path, no L1 allocation.
__device__ __forceinline__ ulonglong2 ld_sup2(const uint64_t *p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// One bit of a 64-bit word in SHARED memory, with the native 32-bit atomic on
// the word's half (a 64-bit shared-memory AND/OR compiles to a CAS loop, which
// serialises badly when many threads hit the same few words).
__device__ __forceinline__ void smem_clear_bit(uint64_t *w, int b) {
  atomicAnd(reinterpret_cast<unsigned int *>(w) + (b >> 5), ~(1u << (b & 31)));
}
__device__ __forceinline__ void smem_set_bit(uint64_t *w, int b) {
  atomicOr(reinterpret_cast<unsigned int *>(w) + (b >> 5), 1u << (b & 31));
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ------------------------------------------------------------------ spin watchdog
// Every software grid barrier and chained-scan look-back polls through
// spin_check: after kSpinLimitNs of waiting the CTA records where it waits
// (kind, its location marker, the words it polls) into the host-mapped
// diagnostic buffer (ct_debug_diag_attach / _read), the first reporter also
// copies every CTA's location and barrier count, and the kernel traps -- a lost
// arrival then surfaces as CT_ECUDA instead of a GPU spinning forever.
__device__ unsigned long long g_spin_limit_ns = 4000000000ull;   // 4 s: phases take us to ms
// experiment builds (-DCT_SERVE_TRACE): k_small_serve stamps points of each
// served call into its doorbell page (ct_debug_serve_trace)
#ifdef CT_SERVE_TRACE
__device__ unsigned long long *g_tr;
#define SERVE_TRACE(i) do { if (g_tr && threadIdx.x == 0) g_tr[i] = globaltimer(); } while (0)
#else
#define SERVE_TRACE(i) do { } while (0)
#endif
constexpr int kDiagCtas = 4096;
__device__ unsigned long long *g_diag;     // host-mapped [kDiagWords] or nullptr
__device__ uint32_t g_loc[kDiagCtas];      // per-CTA location marker (phase code)
__device__ uint32_t g_bseq[kDiagCtas];     // per-CTA grid-barrier count
__device__ uint32_t g_diag_n;              // reports written
constexpr int kDiagWords = 64 + 16 * 8 + 2 * kDiagCtas;   // header, 16 reports, loc + bseq

__device__ __forceinline__ void set_loc(uint32_t code) {
  if (threadIdx.x == 0 && blockIdx.x < kDiagCtas) g_loc[blockIdx.x] = code;
}

__device__ __noinline__ void spin_report(uint32_t kind, unsigned long long a, unsigned long long b,
                                         unsigned long long c) {
  unsigned long long *d = g_diag;
  if (!d) return;
  const uint32_t k = atomicAdd(&g_diag_n, 1u);
  if (k < 16) {
    unsigned long long *r = d + 64 + 8 * k;
    r[0] = kind;
    r[1] = blockIdx.x;
    r[2] = a;
    r[3] = b;
    r[4] = c;
    r[5] = blockIdx.x < kDiagCtas ? *(volatile uint32_t *)&g_loc[blockIdx.x] : 0;
    r[6] = blockIdx.x < kDiagCtas ? *(volatile uint32_t *)&g_bseq[blockIdx.x] : 0;
    r[7] = gridDim.x;
  }
  if (k == 0) {
    const int G = min((int)gridDim.x, kDiagCtas);
    for (int i = 0; i < G; ++i) {
      d[64 + 128 + i] = *(volatile uint32_t *)&g_loc[i];
      d[64 + 128 + kDiagCtas + i] = *(volatile uint32_t *)&g_bseq[i];
    }
  }
  __threadfence_system();
  if (k == 0) d[0] = 0xD1A6D1A6ull;   // header: a report is complete
  __threadfence_system();
}

struct SpinGuard {
  unsigned long long t0 = 0;
  uint32_t n = 0;
};
__device__ __forceinline__ void spin_check(SpinGuard &g, uint32_t kind, unsigned long long a, unsigned long long b,
                                           unsigned long long c) {
  if ((++g.n & 255u) != 0) return;
  const unsigned long long t = globaltimer();
  if (g.t0 == 0) {
    g.t0 = t;
    return;
  }
  if (t - g.t0 < g_spin_limit_ns) return;
  spin_report(kind, a, b, c);
  __trap();
}

// Exclusive block scan of a 64-bit value over NT threads (two packed 32-bit
// counters never overflow into each other here: each half sums to <= R < 2^30).
template <int NT>
__device__ __forceinline__ uint64_t block_excl_scan(uint64_t v, uint64_t *s_warp, uint64_t &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint64_t w = lane < NT / 32 ? s_warp[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) s_warp[lane] = w;
  }
  __syncthreads();
  const uint64_t base = warp > 0 ? s_warp[warp - 1] : 0;
  total = s_warp[NT / 32 - 1];
  __syncthreads();
  return base + x - v;
}

// Software grid barrier for k_fused (all blocks co-resident: cooperative launch).
// Sense by generation counter.  The gpu-scope fences also invalidate the SM's
// L1 (CCTL.IVALL), so after the barrier plain (L1-cached) loads see the data
// other SMs wrote before it; that is what lets the phases use ordinary loads
// for the update list, index and currTable.
__device__ __forceinline__ void grid_barrier(Ctl *c) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t gen = ld_acquire_u32(&c->bar_gen);
    __threadfence();
    if (atomicAdd(&c->bar_count, 1u) == gridDim.x - 1) {
      c->bar_count = 0;
      __threadfence();
      atomicAdd(&c->bar_gen, 1u);
    } else {
      SpinGuard sg;
      while (ld_acquire_u32(&c->bar_gen) == gen) {
        __nanosleep(20);
        spin_check(sg, 1, gen, c->bar_count, 0);
      }
    }
    __threadfence();
  }
  __syncthreads();
}

__host__ __device__ inline size_t ingest_smem_bytes(int n, int Wd) {
  return (size_t)Wd * 16 + (size_t)(5 * n + 3) * 4;
}
__host__ __device__ inline size_t finalize_smem_bytes(int n, int Wd) {
  return (size_t)Wd * 8 + (size_t)(3 * n + 2) * 4;
}

// ------------------------------------------------------------------ a1: supports builder
// One thread per tuple of this shard: sets bit j of row (x_i, tau_j[i]) for
// every in-range value (cell ([x_i,v], j) = 1 iff tau_j[i] = v),
// and the in-range validity of tau_j into the initial currTable (one ballot
// per 32 tuples -> one 32-bit half-word).  Out-of-range values create no row
// bit and make the tuple invalid forever.  A star cell (short
// tables, f4) sets bit j in every row of x_i.
__global__ void k_build(const int32_t *__restrict__ tuples, int64_t t_local, int n,
                        const int32_t *__restrict__ lo, const int32_t *__restrict__ d,
                        const int32_t *__restrict__ rowBase, uint64_t *__restrict__ S, int64_t Wp,
                        uint32_t *__restrict__ T32, int64_t n_half_words, int allow_star) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool valid = j < t_local;
  if (valid) {
    const int32_t *tau = tuples + j * n;
    const uint64_t bit = 1ull << (j & 63);
    const int64_t word = j >> 6;
    for (int i = 0; i < n; ++i) {
      if (allow_star && tau[i] == kStar) {   // short table: the cell matches every value of x_i
        for (int a = 0; a < d[i]; ++a)
          atomicOr(reinterpret_cast<unsigned long long *>(S + (int64_t)(rowBase[i] + a) * Wp + word),
                   (unsigned long long)bit);
        continue;
      }
      const int64_t v = (int64_t)tau[i] - lo[i];
      if (v >= 0 && v < d[i]) {
        atomicOr(reinterpret_cast<unsigned long long *>(S + (int64_t)(rowBase[i] + v) * Wp + word),
                 (unsigned long long)bit);
      } else {
        valid = false;
      }
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, valid);
  const int64_t hw = j >> 5;
  if ((threadIdx.x & 31) == 0 && hw < n_half_words) T32[hw] = bal;
}

// The gather filter's cells (ct_fast.cuh fast_gather_range): tuple j's value
// offsets v - lo_i, `bits` bits each, packed LSB-first into `words` uint32 per
// tuple.  Out-of-range values keep an all-ones cell (such a tuple is never
// valid, so never gathered).
__global__ void k_build_cells(const int32_t *__restrict__ tuples, int64_t t_local, int n,
                              const int32_t *__restrict__ lo, const int32_t *__restrict__ d,
                              uint32_t *__restrict__ cells, int bits, int words) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= t_local) return;
  const int per = 32 / bits;
  const uint32_t cmask = (1u << bits) - 1u;
  const int32_t *tau = tuples + j * n;
  for (int q = 0; q < words; ++q) {
    uint32_t w = 0;
    for (int e = 0; e < per; ++e) {
      const int i = q * per + e;
      if (i >= n) break;
      const int64_t v = (int64_t)tau[i] - lo[i];
      const uint32_t c = (v >= 0 && v < d[i]) ? (uint32_t)v : cmask;
      w |= (c & cmask) << (e * bits);
    }
    cells[j * words + q] = w;
  }
}

// ------------------------------------------------------------------ a2: ingest (one block)
// Row-parallel: every support row decides on its own whether it enters the
// update list (x in s_val, value in the chosen branch) and the filter list
// (x in s_sup, value in D_x); one block scan gives the ordered positions.
// Returns (every thread) 0: the call updates, 1: no-op, 2: FAIL (a domain
// became empty), 3: the state is dead (skip).
template <int NT>
__device__ int dev_ingest(const TableDev &tb, const StateDev &st, const uint64_t *__restrict__ rem,
                          int root_mode, uint64_t *smem, const uint64_t *gdom = nullptr) {
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, n = tb.n, Wd = tb.Wd;
  uint64_t *s_din = smem;                       // D_x = dom ∧ ¬removed
  uint64_t *s_dl = smem + Wd;                   // Δ_x = dom ∧ removed
  int32_t *s_cd = reinterpret_cast<int32_t *>(smem + 2 * Wd);   // |Δ_x|
  int32_t *s_cs = s_cd + n;                     // |D_x|
  int32_t *s_ust = s_cs + n;                    // [n+1] start of x's group in the update list
  int32_t *s_rb = s_ust + n + 1;                // [n+1] rowBase
  int32_t *s_do = s_rb + n + 1;                 // [n+1] domOff
  __shared__ int s_dead, s_fail, s_ngroups;
  __shared__ uint64_t s_warp[NT / 32];

  // this thread's first domain word and removal word are loaded before
  // anything waits: the removals may sit in mapped host memory (sync call)
  uint64_t dm0 = 0, rm0 = 0;
  int wv0 = 0, rv0 = 0;   // this thread's first word's / row's variable, in flight with the rest
  if (tid < Wd) {
    dm0 = st.dom[tid];
    rm0 = gdom ? ~__ldcg(gdom + tb.gword[tid]) : (rem ? rem[tid] : 0ull);
    wv0 = tb.wordVar[tid];
  }
  if (tid < tb.R) rv0 = tb.rowVar[tid];
  __shared__ int s_L;
  if (tid == 0) {
    s_L = c->L;
    s_dead = c->dead;
    s_fail = 0;
    s_ngroups = 0;
  }
  for (int i = tid; i <= n; i += NT) {
    s_rb[i] = tb.rowBase[i];
    s_do[i] = tb.domOff[i];
  }
  for (int x = tid; x < n; x += NT) s_cd[x] = s_cs[x] = 0;
  __syncthreads();
  if (s_dead) {
    if (tid == 0) {
      c->skip = 1;
      c->noop = 0;
      c->fail_fast = 0;
    }
    return 3;
  }
  // per-call scratch
  for (int r = tid; r <= tb.R; r += NT) st.sup[r] = 0;
  for (int k = tid; k < tb.ntiles_max; k += NT) st.tilestat[k] = 0;

  // phase 1 (Alg. 1 L1-2): Δ_x = removed ∧ dom, D_x = dom ∧ ¬removed, sizes
  for (int k = tid; k < Wd; k += NT) {
    uint64_t dm = k == tid ? dm0 : st.dom[k];
    // model tables: a value is removed iff the shared (global) domain lost it
    uint64_t rm = k == tid ? rm0 : (gdom ? ~__ldcg(gdom + tb.gword[k]) : (rem ? rem[k] : 0ull));
    if (st.pend) {   // negative table: values the last filter pruned leave currTable now
      const uint64_t pd = st.pend[k];
      dm |= pd;
      rm |= pd;
    }
    const int x = k == tid ? wv0 : tb.wordVar[k];
    const uint64_t delta = rm & dm, di = dm & ~rm;
    s_din[k] = di;
    s_dl[k] = delta;
    st.din[k] = di;
    if (delta) atomicAdd(&s_cd[x], __popcll(delta));
    if (di) atomicAdd(&s_cs[x], __popcll(di));
  }
  __syncthreads();
  // phase 2: per variable -- s_val membership, branch (Alg. 2), group sizes
  int carry = 0;
  for (int base = 0; base < n; base += NT) {
    const int x = base + tid;
    uint64_t ucnt = 0;
    if (x < n) {
      const int cd = s_cd[x], cs = s_cs[x];
      const bool useDelta = use_delta(tb, x, cd, cs);
      if (cd > 0) {
        ucnt = (uint64_t)(useDelta ? cd : cs);
        atomicAdd(&s_ngroups, 1);
      }
      if (cs == 0) s_fail = 1;                    // D_x empty -> no valid tuple
      st.varcnt[2 * x] = cd;
      st.varcnt[2 * x + 1] = cs;
    }
    uint64_t total;
    const uint64_t ex = block_excl_scan<NT>(ucnt, s_warp, total);
    if (x < n) s_ust[x] = carry + (int)ex;
    carry += (int)total;
  }
  if (tid == 0) s_ust[n] = carry;
  __syncthreads();
  const bool noop = (s_ngroups == 0) && !root_mode;
  int nrows = 0, nitems = 0;
  if (!(s_fail || noop)) {
    // phase 3: per support row -- update list (grouped by var, group end
    // marked) and filter items (Alg. 1 L3: s_sup), both in row order
    uint64_t rcarry = 0;
    for (int base = 0; base < tb.R; base += NT) {
      const int r = base + tid;
      bool u = false, f = false, useDelta = false;
      int x = 0;
      if (r < tb.R) {
        x = r == tid ? rv0 : tb.rowVar[r];
        const int a = r - s_rb[x];
        const int w = s_do[x] + (a >> 6), b = a & 63;
        const int cd = s_cd[x], cs = s_cs[x];
        useDelta = use_delta(tb, x, cd, cs);
        const bool inD = (s_din[w] >> b) & 1, inDl = (s_dl[w] >> b) & 1;
        u = cd > 0 && (useDelta ? inDl : inD);
        f = cs > 1 && inD;
      }
      uint64_t total;
      const uint64_t ex = block_excl_scan<NT>(((uint64_t)u << 32) | (uint64_t)f, s_warp, total) + rcarry;
      if (u) {
        const int up = (int)(ex >> 32);
        uint32_t e = (uint32_t)r | (useDelta ? kInvBit : 0u);
        if (up == s_ust[x + 1] - 1) e |= kEndBit;
        st.ulist[up] = (int32_t)e;
      }
      if (f) st.items[(int)(ex & 0xffffffffu)] = r;
      rcarry += total;
    }
    nrows = (int)(rcarry >> 32);
    nitems = (int)(rcarry & 0xffffffffu);
  }
  if (tid == 0) {
    c->skip = 0;
    c->noop = noop && !s_fail;
    c->fail_fast = s_fail;
    c->ngroups = s_ngroups;
    c->nrows = nrows;
    c->nitems = nitems;
    c->L_in = s_L;
    c->L_out = 0;
    c->tile_ctr = 0;
    c->nscan = 0;
    c->upd_loads = 0;
    c->upd_writes = 0;
    c->scan_loads = 0;
  }
  return s_fail ? 2 : (noop ? 1 : 0);
}

// ------------------------------------------------------------------ a2: ingest by one warp
// dev_ingest's decisions and outputs (same lists in the same order, same
// shared-memory layout) computed by warp 0 alone, with warp-level scans
// instead of block scans: for one-CTA calls on small tables (k_small) the
// ingest is latency-bound and 32 lanes cover its few words and rows.  Every
// thread of the block calls it; it ends with a block barrier.
// Shared-memory copies of what warp_ingest publishes (k_small keeps the whole
// call on chip: no global round trip between its phases).
struct SmallSh {
  int32_t *ulist, *items;   // [R] each
  int skip, noop, fail, nrows, nitems, L, ident, par;
};

__device__ void warp_ingest(const TableDev &tb, const StateDev &st, const uint64_t *__restrict__ rem,
                            int root_mode, uint64_t *smem, const uint64_t *gdom = nullptr,
                            SmallSh *sh = nullptr) {
  Ctl *c = st.ctl;
  const int n = tb.n, Wd = tb.Wd, R = tb.R;
  uint64_t *s_din = smem;
  uint64_t *s_dl = smem + Wd;
  int32_t *s_cd = reinterpret_cast<int32_t *>(smem + 2 * Wd);
  int32_t *s_cs = s_cd + n;
  int32_t *s_ust = s_cs + n;
  int32_t *s_rb = s_ust + n + 1;
  int32_t *s_do = s_rb + n + 1;
  constexpr int kRowWarps = 4;   // warps of the per-row pass
  __shared__ int s_wi[4];        // warp 0's verdicts: dead, fail, noop, groups
  __shared__ int s_wc[2 * kRowWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int rv0 = 0;   // this thread's row of the first round: its variable, requested at once
  if (warp < kRowWarps && warp * 32 + lane < R) rv0 = tb.rowVar[warp * 32 + lane];
  if (threadIdx.x < 32) {
    uint64_t dm0 = 0, rm0 = 0;
    int wv0 = 0;
    if (lane < Wd) {
      dm0 = st.dom[lane];
      // model tables: a value is removed iff the shared (global) domain lost it
      rm0 = gdom ? ~__ldcg(gdom + tb.gword[lane]) : (rem ? rem[lane] : 0ull);
      wv0 = tb.wordVar[lane];
    }
    const int dead = __shfl_sync(0xffffffffu, lane == 0 ? c->dead : 0, 0);
    SERVE_TRACE(2);
    for (int i = lane; i <= n; i += 32) {
      s_rb[i] = tb.rowBase[i];
      s_do[i] = tb.domOff[i];
    }
    for (int x = lane; x < n; x += 32) s_cd[x] = s_cs[x] = 0;
    if (dead) {
      if (lane == 0) {
        c->skip = 1;
        c->noop = 0;
        c->fail_fast = 0;
        if (sh) {
          sh->skip = 1;
          sh->noop = 0;
          sh->fail = 0;
        }
      }
    } else {
      uint4 *s4 = reinterpret_cast<uint4 *>(st.sup);   // sup[0..R] = 0 (256-byte aligned)
      for (int r = lane; r < (R + 16) / 16; r += 32) s4[r] = make_uint4(0u, 0u, 0u, 0u);
      for (int k = lane; k < tb.ntiles_max; k += 32) st.tilestat[k] = 0;   // chained-scan tile statuses
      __syncwarp();
      // Alg. 1 L1-2: Δ_x = removed ∧ dom, D_x = dom ∧ ¬removed, sizes
      for (int k = lane; k < Wd; k += 32) {
        const uint64_t dm = k == lane ? dm0 : st.dom[k];
        const uint64_t rm = k == lane ? rm0 : (gdom ? ~__ldcg(gdom + tb.gword[k]) : (rem ? rem[k] : 0ull));
        const int x = k == lane ? wv0 : tb.wordVar[k];
        const uint64_t delta = rm & dm, di = dm & ~rm;
        s_din[k] = di;
        s_dl[k] = delta;
        st.din[k] = di;
        if (delta) atomicAdd(&s_cd[x], __popcll(delta));
        if (di) atomicAdd(&s_cs[x], __popcll(di));
      }
      __syncwarp();
      SERVE_TRACE(3);
      // per variable: s_val, branch (Alg. 2), group sizes -> group starts
      int carry = 0, ngroups = 0, fail = 0;
      for (int base = 0; base < n; base += 32) {
        const int x = base + lane;
        int ucnt = 0;
        if (x < n) {
          const int cd = s_cd[x], cs = s_cs[x];
          const bool useDelta = use_delta(tb, x, cd, cs);
          if (cd > 0) ucnt = useDelta ? cd : cs;
          ngroups += cd > 0;
          fail |= cs == 0;
          st.varcnt[2 * x] = cd;
          st.varcnt[2 * x + 1] = cs;
        }
        int incl = ucnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        if (x < n) s_ust[x] = carry + incl - ucnt;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) s_ust[n] = carry;
      ngroups = __reduce_add_sync(0xffffffffu, ngroups);
      fail = __reduce_or_sync(0xffffffffu, fail);
      __syncwarp();
      const bool noop = ngroups == 0 && !root_mode;
      if (lane == 0) {
        s_wi[1] = fail;
        s_wi[2] = noop;
        s_wi[3] = ngroups;
      }
    }
    if (lane == 0) s_wi[0] = dead;
  }
  SERVE_TRACE(4);
  __syncthreads();
  // per support row: update list (grouped by var, group end marked) and filter
  // items (Alg. 1 L3: s_sup), both in row order -- kRowWarps warps, 32 x
  // kRowWarps rows per round, the warps' offsets from their ballot counts
  const int dead = s_wi[0], fail = s_wi[1], noop = s_wi[2];
  int nrows = 0, nitems = 0;
  if (!dead && !(fail || noop)) {
    int ucarry = 0, icarry = 0;
    for (int base = 0; base < R; base += 32 * kRowWarps) {   // uniform over the block (barriers inside)
      const int r = base + warp * 32 + lane;
      bool u = false, f = false, useDelta = false;
      int x = 0;
      if (warp < kRowWarps && r < R) {
        x = base == 0 ? rv0 : tb.rowVar[r];
        const int a = r - s_rb[x];
        const int w = s_do[x] + (a >> 6), b = a & 63;
        const int cd = s_cd[x], cs = s_cs[x];
        useDelta = use_delta(tb, x, cd, cs);
        const bool inD = (s_din[w] >> b) & 1, inDl = (s_dl[w] >> b) & 1;
        u = cd > 0 && (useDelta ? inDl : inD);
        f = cs > 1 && inD;
      }
      const unsigned bu = __ballot_sync(0xffffffffu, u), bf = __ballot_sync(0xffffffffu, f);
      if (lane == 0 && warp < kRowWarps) {
        s_wc[warp] = __popc(bu);
        s_wc[kRowWarps + warp] = __popc(bf);
      }
      __syncthreads();
      int uo = ucarry, io = icarry, ut = 0, it = 0;
#pragma unroll
      for (int q = 0; q < kRowWarps; ++q) {
        if (q < warp) {
          uo += s_wc[q];
          io += s_wc[kRowWarps + q];
        }
        ut += s_wc[q];
        it += s_wc[kRowWarps + q];
      }
      if (u) {
        const int up = uo + __popc(bu & lanemask_lt());
        uint32_t e = (uint32_t)r | (useDelta ? kInvBit : 0u);
        if (up == s_ust[x + 1] - 1) e |= kEndBit;
        if (sh) sh->ulist[up] = (int32_t)e;
        else st.ulist[up] = (int32_t)e;
      }
      if (f) {
        const int ip = io + __popc(bf & lanemask_lt());
        if (sh) sh->items[ip] = r;
        else st.items[ip] = r;
      }
      ucarry += ut;
      icarry += it;
      __syncthreads();   // s_wc is rewritten next round
    }
    nrows = ucarry;
    nitems = icarry;
  }
  if (threadIdx.x == 0 && !dead) {
    const int ngroups = s_wi[3];
    const int L0 = c->L;
    if (sh) {
      sh->skip = 0;
      sh->noop = noop && !fail;
      sh->fail = fail;
      sh->nrows = nrows;
      sh->nitems = nitems;
      sh->L = L0;
      sh->ident = c->identity;
      sh->par = c->parity;
    }
    c->skip = 0;
    c->noop = noop && !fail;
    c->fail_fast = fail;
    c->ngroups = ngroups;
    c->nrows = nrows;
    c->nitems = nitems;
    c->L_in = L0;
    c->L_out = 0;
    c->tile_ctr = 0;
    c->nscan = 0;
    c->upd_loads = 0;
    c->upd_writes = 0;
    c->scan_loads = 0;
  }
  SERVE_TRACE(5);
  __syncthreads();
}

// ------------------------------------------------------------------ a3-a5: update + compaction
// Chained-scan look-back (warp 0 of the block); returns the exclusive prefix.
__device__ __forceinline__ uint32_t tile_lookback(unsigned long long *ts, int tile, uint32_t agg, int lane) {
  if (tile == 0) {
    if (lane == 0) st_release(ts, kFlagPre | agg);
    return 0;
  }
  if (lane == 0) st_release(ts + tile, kFlagAgg | agg);
  uint32_t excl = 0;
  int base = tile - 1;
  while (true) {
    const int p = base - lane;
    unsigned long long s = kFlagPre;   // before tile 0: prefix 0
    if (p >= 0) {
      SpinGuard sg;
      do {
        s = ld_acquire(ts + p);
        if ((s >> 62) == 0) spin_check(sg, 2, (unsigned long long)tile, (unsigned long long)p, 0);
      } while ((s >> 62) == 0);
    }
    const unsigned pre = __ballot_sync(0xffffffffu, (s >> 62) == 2);
    uint32_t v = (uint32_t)s;
    if (pre) {
      const int f = __ffs(pre) - 1;
      if (lane > f) v = 0;
    }
    excl += warp_sum_u32(v);
    if (pre) break;
    base -= 32;
  }
  if (lane == 0) st_release(ts + tile, kFlagPre | (excl + agg));
  return excl;
}

// Per-call update parameters of one state (read once per block).
struct UpdParams {
  int go, nrows, L, ident, par, ntiles;
};

__device__ __forceinline__ UpdParams load_upd_params(const Ctl *c) {
  UpdParams u;
  u.go = !(__ldcg(&c->skip) | __ldcg(&c->noop) | __ldcg(&c->fail_fast));
  u.nrows = __ldcg(&c->nrows);
  u.L = __ldcg(&c->L);
  u.ident = __ldcg(&c->identity);
  u.par = __ldcg(&c->parity);
  u.ntiles = (u.L + kUpdTPB - 1) / kUpdTPB;
  return u;
}

// One tile (kUpdTPB index entries = 16-byte blocks, so every support/currTable
// access is an aligned 128-bit load) of one state's update, block-wide:
// new currTable blocks, then the tile's slot in the order-preserving compaction
// (chained scan over the state's tiles).  Requires blockDim.x == kUpdTPB.
// s_woff[kUpdTPB/32] and s_excl are block-shared scratch.
__device__ __forceinline__ void update_tile(const TableDev &tb, const StateDev &st, const UpdParams &u, int tile,
                                            uint32_t *s_woff, uint32_t *s_excl, uint32_t &n_loads,
                                            uint32_t &n_writes) {
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nrows = u.nrows, L = u.L;
  const int32_t *__restrict__ idx_in = u.par ? st.idx1 : st.idx0;
  int32_t *__restrict__ idx_out = u.par ? st.idx0 : st.idx1;
  const bool compact = tb.use_index != 0;
  const int32_t *__restrict__ ulist = st.ulist;
  const int64_t Wp = tb.Wp;
  ulonglong2 *__restrict__ T2 = reinterpret_cast<ulonglong2 *>(st.T);
  const int k = tile * kUpdTPB + tid;
  const bool valid = k < L;
  int pid = 0;
  ulonglong2 nt = make_ulonglong2(0ull, 0ull);
  if (valid) {
    pid = u.ident ? k : idx_in[k];
    const ulonglong2 tw = T2[pid];
    const uint64_t *__restrict__ col = tb.S + 2 * (int64_t)pid;
    uint64_t mx = ~0ull, my = ~0ull, ax = 0, ay = 0;
    uint32_t e[kUpdUnroll];
#pragma unroll
    for (int q = 0; q < kUpdUnroll; ++q) e[q] = (q < nrows) ? (uint32_t)ulist[q] : 0u;
    for (int p = 0; p < nrows; p += kUpdUnroll) {
      if (((tw.x & mx) | (tw.y & my)) == 0) break;   // Alg. 2, per 128-bit block
      ulonglong2 v[kUpdUnroll];
#pragma unroll
      for (int q = 0; q < kUpdUnroll; ++q)
        v[q] = (p + q < nrows) ? ld_sup2(col + (int64_t)(e[q] & kRowMask) * Wp) : make_ulonglong2(0ull, 0ull);
      n_loads += 2 * min(kUpdUnroll, nrows - p);
      uint32_t en[kUpdUnroll];
#pragma unroll
      for (int q = 0; q < kUpdUnroll; ++q)
        en[q] = (p + kUpdUnroll + q < nrows) ? (uint32_t)ulist[p + kUpdUnroll + q] : 0u;
#pragma unroll
      for (int q = 0; q < kUpdUnroll; ++q) {
        if (p + q < nrows) {
          ax |= v[q].x;
          ay |= v[q].y;
          if (e[q] & kEndBit) {
            if (e[q] & kInvBit) {
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
#pragma unroll
      for (int q = 0; q < kUpdUnroll; ++q) e[q] = en[q];
    }
    nt = make_ulonglong2(tw.x & mx, tw.y & my);
    if (nt.x != tw.x || nt.y != tw.y) {
      T2[pid] = nt;
      ++n_writes;
    }
  }
  const bool keep = valid && (nt.x | nt.y) != 0;
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  if (lane == 0) s_woff[warp] = __popc(bal);
  __syncthreads();
  if (warp == 0) {
    const uint32_t cnt = lane < kUpdTPB / 32 ? s_woff[lane] : 0u;
    uint32_t x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    const uint32_t agg = __shfl_sync(0xffffffffu, x, kUpdTPB / 32 - 1);
    if (lane < kUpdTPB / 32) s_woff[lane] = x - cnt;
    uint32_t excl = 0;
    if (compact) {
      excl = tile_lookback(st.tilestat, tile, agg, lane);
      if (lane == 0 && tile == u.ntiles - 1) c->L_out = (int32_t)(excl + agg);
    } else if (lane == 0 && agg) {
      atomicAdd(&c->L_out, (int32_t)agg);
    }
    if (lane == 0) *s_excl = excl;
  }
  __syncthreads();
  if (compact && keep) idx_out[*s_excl + s_woff[warp] + __popc(bal & lanemask_lt())] = pid;
  __syncthreads();   // s_woff / s_excl are reused by the next tile
}

__device__ __forceinline__ void flush_update_counts(Ctl *c, uint32_t n_loads, uint32_t n_writes) {
  n_loads = warp_sum_u32(n_loads);
  n_writes = warp_sum_u32(n_writes);
  if ((threadIdx.x & 31) == 0 && (n_loads | n_writes)) {
    atomicAdd(&c->upd_loads, (unsigned long long)n_loads);
    atomicAdd(&c->upd_writes, (unsigned long long)n_writes);
  }
}

// Block-level persistent loop over one state's tiles (atomic tile counter).
__device__ void dev_update(const TableDev &tb, const StateDev &st) {
  Ctl *c = st.ctl;
  __shared__ UpdParams s_u;
  __shared__ int s_tile;
  __shared__ uint32_t s_woff[kUpdTPB / 32];
  __shared__ uint32_t s_excl;
  if (threadIdx.x == 0) s_u = load_upd_params(c);
  __syncthreads();
  const UpdParams u = s_u;
  if (!u.go) return;
  uint32_t n_loads = 0, n_writes = 0;
  while (true) {
    if (threadIdx.x == 0) s_tile = atomicAdd(&c->tile_ctr, 1);
    __syncthreads();
    const int tile = s_tile;
    if (tile >= u.ntiles) break;
    update_tile(tb, st, u, tile, s_woff, &s_excl, n_loads, n_writes);
  }
  flush_update_counts(c, n_loads, n_writes);
}

// ------------------------------------------------------------------ a6: filter
// Warp-cooperative intersect of support row `srow` with currTable over index
// entries [k0, k1) (Alg. 3 L3 "currTable & supports[x,a] != 0", CT's
// intersectIndex): kScanUnroll blocks per lane per round, one __ballot_sync
// "any" per block.  Returns the first (lowest-entry) block with a common valid
// tuple, -1 if none, -2 if `supflag` was set by another warp meanwhile.
template <int U = kScanUnroll>
__device__ __forceinline__ int scan_pairs(const int32_t *__restrict__ idx, const ulonglong2 *__restrict__ T2,
                                          const uint64_t *__restrict__ srow, int k0, int k1,
                                          const uint8_t *supflag, int lane, uint32_t &n_loads) {
  for (int kb = k0; kb < k1; kb += 32 * U) {
    if (supflag && kb != k0) {
      const int f = lane == 0 ? *(volatile const uint8_t *)supflag : 0;
      if (__shfl_sync(0xffffffffu, f, 0)) return -2;
    }
    // loads are issued unconditionally (an out-of-range lane re-reads entry
    // k0 and is masked after): a load inside a per-entry branch would wait for
    // the previous one, serialising the round
    int pid[U];
    uint64_t v[U];
    ulonglong2 t[U], s[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int k = kb + q * 32 + lane;
      const int kk = k < k1 ? k : k0;
      pid[q] = idx ? idx[kk] : kk;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      t[q] = T2[pid[q]];   // L1-cacheable: the batch probes re-read a state's blocks
      s[q] = ld_sup2(srow + 2 * (int64_t)pid[q]);
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const bool in = kb + q * 32 + lane < k1;
      v[q] = in ? ((t[q].x & s[q].x) | (t[q].y & s[q].y)) : 0ull;
      if (!in) pid[q] = -1;
    }
    n_loads += 2 * min(32 * U, k1 - kb);
    int hit = -1;
#pragma unroll
    for (int q = U - 1; q >= 0; --q) {
      const unsigned b = __ballot_sync(0xffffffffu, v[q] != 0);
      if (b) hit = __shfl_sync(0xffffffffu, pid[q], __ffs(b) - 1);
    }
    if (hit >= 0) return hit;
  }
  return -1;
}

// Per-call filter parameters of one state.
struct FiltParams {
  int go, Lout, nitems, nscan, L;
  const int32_t *idx;   // index written by this call's update (nullptr: identity)
};

__device__ __forceinline__ FiltParams load_filt_params(const TableDev &tb, const StateDev &st) {
  const Ctl *c = st.ctl;
  FiltParams f;
  f.go = !(__ldcg(&c->skip) | __ldcg(&c->noop) | __ldcg(&c->fail_fast));
  f.Lout = __ldcg(&c->L_out);
  f.nitems = __ldcg(&c->nitems);
  f.nscan = __ldcg(&c->nscan);
  const bool compact = tb.use_index != 0;
  f.idx = compact ? (__ldcg(&c->parity) ? st.idx0 : st.idx1) : nullptr;
  f.L = compact ? f.Lout : tb.W2;
  return f;
}

// Warp-level, one (x,a) item: residue probe, then the first
// kFirstScan index entries; an item still unresolved goes to the scan list.
__device__ __forceinline__ void probe_item(const TableDev &tb, const StateDev &st, const FiltParams &f, int item,
                                           uint32_t &n_loads) {
  const int lane = threadIdx.x & 31;
  const ulonglong2 *__restrict__ T2 = reinterpret_cast<const ulonglong2 *>(st.T);
  const int row = __ldcg(st.items + item);
  const uint64_t *__restrict__ srow = tb.S + (int64_t)row * tb.Wp;
  if (tb.use_res) {
    int hit = 0;
    if (lane == 0) {
      const int r = st.res[row];
      const ulonglong2 t = __ldcg(T2 + r);
      const ulonglong2 s = ld_sup2(srow + 2 * (int64_t)r);
      hit = ((t.x & s.x) | (t.y & s.y)) != 0;
    }
    if (__shfl_sync(0xffffffffu, hit, 0)) {
      if (lane == 0) st.sup[row] = 1;
      return;
    }
  }
  const int hit = scan_pairs(f.idx, T2, srow, 0, min(f.L, kFirstScan), nullptr, lane, n_loads);
  if (lane == 0) {
    if (hit >= 0) {
      st.sup[row] = 1;
      st.res[row] = hit;
    } else if (f.L > kFirstScan) {
      st.scanlist[atomicAdd(&st.ctl->nscan, 1)] = row;
    }
  }
}

// Warp-level, one (miss, chunk) unit over index entries [kFirstScan, L).
__device__ __forceinline__ void scan_unit(const TableDev &tb, const StateDev &st, const FiltParams &f, int64_t u,
                                          uint32_t &n_loads) {
  const int lane = threadIdx.x & 31;
  const int chunk = (int)(u / f.nscan);
  const int item = (int)(u - (int64_t)chunk * f.nscan);
  const int row = __ldcg(st.scanlist + item);
  const int fl = lane == 0 ? *(volatile const uint8_t *)(st.sup + row) : 0;
  if (__shfl_sync(0xffffffffu, fl, 0)) return;
  const int k0 = kFirstScan + chunk * kScanChunk;
  const int k1 = min(k0 + kScanChunk, f.L);
  const ulonglong2 *__restrict__ T2 = reinterpret_cast<const ulonglong2 *>(st.T);
  const int hit = scan_pairs(f.idx, T2, tb.S + (int64_t)row * tb.Wp, k0, k1, st.sup + row, lane, n_loads);
  if (hit >= 0 && lane == 0) {
    st.sup[row] = 1;
    st.res[row] = hit;
  }
}

__device__ __forceinline__ int64_t scan_units(const FiltParams &f) {
  if (!f.go || f.nscan == 0 || f.Lout == 0 || f.L <= kFirstScan) return 0;
  return (int64_t)((f.L - kFirstScan + kScanChunk - 1) / kScanChunk) * f.nscan;
}

// Warp-level: items gw, gw + nw, ... of one state.  The warp with gw == 0 also
// publishes this shard's "non-empty" flag.
__device__ void dev_probe(const TableDev &tb, const StateDev &st, int gw, int nw) {
  const FiltParams f = load_filt_params(tb, st);
  if (!f.go) return;
  if (gw == 0 && (threadIdx.x & 31) == 0) st.sup[tb.R] = f.Lout > 0;
  if (f.Lout == 0) return;
  uint32_t n_loads = 0;
  for (int item = gw; item < f.nitems; item += nw) probe_item(tb, st, f, item, n_loads);
  if ((threadIdx.x & 31) == 0 && n_loads) atomicAdd(&st.ctl->scan_loads, (unsigned long long)n_loads);
}

// Warp-level: (miss, chunk) units gw, gw + nw, ... chunk-major so early chunks
// of every item go first; every round re-checks the item's flag so late chunks
// stop once any chunk hit.
__device__ void dev_scan(const TableDev &tb, const StateDev &st, int gw, int nw) {
  const FiltParams f = load_filt_params(tb, st);
  const int64_t total = scan_units(f);
  uint32_t n_loads = 0;
  for (int64_t u = gw; u < total; u += nw) scan_unit(tb, st, f, u, n_loads);
  if ((threadIdx.x & 31) == 0 && n_loads) atomicAdd(&st.ctl->scan_loads, (unsigned long long)n_loads);
}

// ------------------------------------------------------------------ a6c-a8: finalize (one block)
// Alg. 3 L3-4: a value of x in s_sup leaves the domain iff its support row has
// no valid tuple (sup[r] = 0 after the cross-shard OR); then lastDom <- dom.
// kDense: the state was updated densely (batch path, ct_batch.cuh): its index
// becomes the identity over all W2 blocks instead of the compacted one.
// Returns the call's status (every thread).  All inputs are final when it is
// entered, so they are loaded in one round trip up front.
template <int NT, bool kDense = false>
__device__ int dev_finalize(const TableDev &tb, const StateDev &st, uint64_t *__restrict__ out_dom,
                            uint64_t *__restrict__ out_pruned, int32_t *__restrict__ out_status, uint64_t *smem) {
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, n = tb.n, Wd = tb.Wd;
  uint64_t *s_nd = smem;
  int32_t *s_cs = reinterpret_cast<int32_t *>(smem + Wd);
  int32_t *s_rb = s_cs + n;
  int32_t *s_do = s_rb + n + 1;
  __shared__ int s_status, s_noop, s_lout;
  // this thread's first support row (flag + variable)
  uint8_t sp0 = 1;
  int x0 = 0;
  if (tid < tb.R) {
    sp0 = __ldcg(st.sup + tid);
    x0 = tb.rowVar[tid];
  }
  if (tid == 0) {
    // the flags are loaded together (one round trip, not a chain)
    const int skip = __ldcg(&c->skip), ff = __ldcg(&c->fail_fast), noop = __ldcg(&c->noop);
    const int nonempty = __ldcg(st.sup + tb.R);
    s_lout = __ldcg(&c->L_out);
    int s;
    if (skip) s = -5;                  // CT_ESTATE
    else if (ff) s = 1;                // CT_FAIL
    else if (noop) s = 0;
    else s = nonempty ? 0 : 1;         // global "currTable non-empty" (Alg. 1 L5)
    s_status = s;
    s_noop = noop;
  }
  for (int k = tid; k < Wd; k += NT) s_nd[k] = __ldcg(st.din + k);
  for (int x = tid; x < n; x += NT) s_cs[x] = __ldcg(st.varcnt + 2 * x + 1);
  for (int i = tid; i <= n; i += NT) {
    s_rb[i] = tb.rowBase[i];
    s_do[i] = tb.domOff[i];
  }
  __syncthreads();
  const int status = s_status;
  if (status != 0) {
    if (tid == 0) {
      if (status == 1) {
        c->dead = 1;
        c->calls += 1;
      }
      c->last_status = status;
      if (out_status) *out_status = status;
    }
    return status;
  }
  const bool noop = s_noop != 0;
  if (!noop) {
    for (int r = tid; r < tb.R; r += NT) {
      const uint8_t sp = r == tid ? sp0 : __ldcg(st.sup + r);
      const int x = r == tid ? x0 : tb.rowVar[r];
      if (!sp && s_cs[x] > 1) {                  // x in s_sup (Alg. 3 L1), a unsupported
        const int a = r - s_rb[x];
        const int w = s_do[x] + (a >> 6);
        const uint64_t bit = 1ull << (a & 63);
        if (s_nd[w] & bit) smem_clear_bit(s_nd + w, a & 63);
      }
    }
    __syncthreads();
  }
  for (int k = tid; k < Wd; k += NT) {
    const uint64_t nd = s_nd[k];
    st.dom[k] = nd;
    if (out_dom) out_dom[k] = nd;
    if (out_pruned) out_pruned[k] = __ldcg(st.din + k) & ~nd;
  }
  // the status word is the completion flag of the host-mapped sync path: every
  // thread's output writes must be visible system-wide before it.  The block
  // barrier makes them observed by thread 0, whose one system-scope fence is
  // cumulative (one MEMBAR.SYS instead of one per thread).
  __syncthreads();
  if (tid == 0) {
#ifndef CT_NO_SYSFENCE
    if (out_status) __threadfence_system();
#endif
    if (!noop && kDense) {
      c->L = tb.W2;
      c->identity = 1;
    } else if (!noop && tb.use_index) {
      c->parity ^= 1;
      c->L = s_lout;
      c->identity = 0;
    }
    c->calls += 1;
    c->last_status = 0;
    if (out_status) *out_status = 0;
  }
  return 0;
}

// ------------------------------------------------------------------ kernels: one per phase (batches)
// grid (1, S), kIngestTPB threads, dynamic smem ingest_smem_bytes().
__global__ void __launch_bounds__(kIngestTPB) k_ingest(TableDev tb, const StateDev *__restrict__ states,
                                                       const uint64_t *__restrict__ removed,
                                                       int64_t removed_stride, int root_mode) {
  extern __shared__ __align__(16) uint64_t smem[];
  const uint64_t *rem = removed ? removed + (int64_t)blockIdx.y * removed_stride : nullptr;
  dev_ingest<kIngestTPB>(tb, states[blockIdx.y], rem, root_mode, smem);
}

// grid (blocks, S), kUpdTPB threads.
__global__ void __launch_bounds__(kUpdTPB, 3) k_update(TableDev tb, const StateDev *__restrict__ states) {
  dev_update(tb, states[blockIdx.y]);
}

// grid (blocks, S), kProbeTPB threads: one warp per item.
__global__ void __launch_bounds__(kProbeTPB) k_probe(TableDev tb, const StateDev *__restrict__ states) {
  dev_probe(tb, states[blockIdx.y], blockIdx.x * (kProbeTPB / 32) + (threadIdx.x >> 5),
            gridDim.x * (kProbeTPB / 32));
}

// grid (blocks, S), kScanTPB threads.
__global__ void __launch_bounds__(kScanTPB) k_scan(TableDev tb, const StateDev *__restrict__ states) {
  dev_scan(tb, states[blockIdx.y], blockIdx.x * (kScanTPB / 32) + (threadIdx.x >> 5), gridDim.x * (kScanTPB / 32));
}

// grid (1, S), kFinTPB threads, dynamic smem finalize_smem_bytes().
__global__ void __launch_bounds__(kFinTPB) k_finalize(TableDev tb, const StateDev *__restrict__ states,
                                                      uint64_t *__restrict__ out_dom, int64_t dom_stride,
                                                      uint64_t *__restrict__ out_pruned,
                                                      int32_t *__restrict__ out_status, int use_state_out) {
  extern __shared__ __align__(16) uint64_t smem[];
  const StateDev st = states[blockIdx.y];
  if (use_state_out) {
    out_dom = st.out + 1;
    out_pruned = st.out + 1 + tb.Wd;
    out_status = reinterpret_cast<int32_t *>(st.out);
  } else {
    if (out_dom) out_dom += (int64_t)blockIdx.y * dom_stride;
    if (out_pruned) out_pruned += (int64_t)blockIdx.y * dom_stride;
    if (out_status) out_status += blockIdx.y;
  }
  dev_finalize<kFinTPB>(tb, st, out_dom, out_pruned, out_status, smem);
}

// ------------------------------------------------------------------ k_fused: one state, one launch
// Cooperative persistent kernel, kFusedTPB threads, grid <= co-resident blocks,
// dynamic smem max(ingest, finalize).  with_finalize = 0 for sharded tables
// (finalize runs after the cross-shard combine).
__global__ void __launch_bounds__(kFusedTPB, 3) k_fused(TableDev tb, const StateDev *__restrict__ states,
                                                     const uint64_t *__restrict__ removed, int root_mode,
                                                     int with_finalize, uint64_t *__restrict__ out_dom,
                                                     uint64_t *__restrict__ out_pruned,
                                                     int32_t *__restrict__ out_status, int use_state_out) {
  extern __shared__ __align__(16) uint64_t smem[];
  const StateDev st = states[0];
  const int gw = blockIdx.x * (kFusedTPB / 32) + (threadIdx.x >> 5), nw = gridDim.x * (kFusedTPB / 32);
  const bool t0 = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long ts[6];
  if (t0) ts[0] = globaltimer();
  if (blockIdx.x == 0) dev_ingest<kFusedTPB>(tb, st, removed, root_mode, smem);
  grid_barrier(st.ctl);
  if (t0) ts[1] = globaltimer();
  dev_update(tb, st);
  grid_barrier(st.ctl);
  if (t0) ts[2] = globaltimer();
  dev_probe(tb, st, gw, nw);
  grid_barrier(st.ctl);
  if (t0) ts[3] = globaltimer();
  dev_scan(tb, st, gw, nw);
  if (!with_finalize) {
    if (t0) {
      ts[4] = ts[5] = globaltimer();
      for (int i = 0; i < 8; ++i) st.ctl->tph[i] = ts[i < 6 ? i : 5];
    }
    return;
  }
  grid_barrier(st.ctl);
  if (t0) ts[4] = globaltimer();
  if (blockIdx.x == 0) {
    if (use_state_out) {
      out_dom = st.out + 1;
      out_pruned = st.out + 1 + tb.Wd;
      out_status = reinterpret_cast<int32_t *>(st.out);
    }
    dev_finalize<kFusedTPB>(tb, st, out_dom, out_pruned, out_status, smem);
    if (t0) {
      ts[5] = globaltimer();
      for (int i = 0; i < 8; ++i) st.ctl->tph[i] = ts[i < 6 ? i : 5];
    }
  }
}

// ------------------------------------------------------------------ a3-a4 in one block
// updateTable (Alg. 2) over the L active blocks and the order-preserving
// compaction of the survivors into the other index buffer, by ONE block of NT
// threads (tables of at most kSmallMaxPairs blocks).  Returns L_out.  Adds the
// work counters to the state.  s_warp: NT/32 words of shared scratch.
template <int NT, int U = kUpdUnroll>
__device__ int block_update(const TableDev &tb, const StateDev &st, int L, int nrows, int ident, int par,
                            uint64_t *s_warp, const int32_t *ulist = nullptr, int pid0 = -1) {
  if (!ulist) ulist = st.ulist;
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, lane = tid & 31;
  const int32_t *__restrict__ idx_in = par ? st.idx1 : st.idx0;
  int32_t *__restrict__ idx_out = par ? st.idx0 : st.idx1;
  const bool compact = tb.use_index != 0;
  ulonglong2 *__restrict__ T2 = reinterpret_cast<ulonglong2 *>(st.T);
  const int64_t Wp = tb.Wp;
  uint32_t n_loads = 0, n_writes = 0;
  uint64_t carry = 0;
  for (int base = 0; base < L; base += NT) {
    const int k = base + tid;
    int pid = 0;
    bool keep = false;
    if (k < L) {
      // pid0: this thread's first index entry, prefetched by the caller
      pid = ident ? k : (base == 0 && pid0 >= 0 ? pid0 : idx_in[k]);
      const ulonglong2 tw = T2[pid];
      const uint64_t *__restrict__ col = tb.S + 2 * (int64_t)pid;
      uint64_t mx = ~0ull, my = ~0ull, ax = 0, ay = 0;
      for (int p = 0; p < nrows; p += U) {
        if (p > 0 && ((tw.x & mx) | (tw.y & my)) == 0) break;
        uint32_t e[U];
        ulonglong2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) e[u] = (p + u < nrows) ? (uint32_t)ulist[p + u] : 0u;
#pragma unroll
        for (int u = 0; u < U; ++u)
          v[u] = (p + u < nrows) ? ld_sup2(col + (int64_t)(e[u] & kRowMask) * Wp) : make_ulonglong2(0ull, 0ull);
        n_loads += 2 * min(U, nrows - p);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (p + u < nrows) {
            ax |= v[u].x;
            ay |= v[u].y;
            if (e[u] & kEndBit) {
              if (e[u] & kInvBit) {
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
      const ulonglong2 nt = make_ulonglong2(tw.x & mx, tw.y & my);
      if (nt.x != tw.x || nt.y != tw.y) {
        T2[pid] = nt;
        ++n_writes;
      }
      keep = (nt.x | nt.y) != 0;
    }
    uint64_t total;
    const uint64_t ex = block_excl_scan<NT>((uint64_t)keep, s_warp, total);
    if (compact && keep) idx_out[carry + ex] = pid;
    carry += total;
  }
  n_loads = warp_sum_u32(n_loads);
  n_writes = warp_sum_u32(n_writes);
  if (lane == 0 && (n_loads | n_writes)) {
    atomicAdd(&c->upd_loads, (unsigned long long)n_loads);
    atomicAdd(&c->upd_writes, (unsigned long long)n_writes);
  }
  return (int)carry;
}

// ------------------------------------------------------------------ a6c-a8 inside one CTA after dev_ingest
// dev_finalize for a kernel whose single CTA also ran dev_ingest: the status
// is known, D (dom after the removals), |D_x|, rowBase and domOff are still in
// the ingest's shared-memory layout, so nothing is re-read from the state.
template <int NT>
__device__ void small_finalize(const TableDev &tb, const StateDev &st, int status, bool noop, int Lout,
                               uint64_t *__restrict__ out_dom, uint64_t *__restrict__ out_pruned,
                               int32_t *__restrict__ out_status, uint64_t *smem,
                               const uint8_t *s_sup = nullptr, unsigned long long *tout = nullptr,
                               uint32_t tag = 0) {
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, n = tb.n, Wd = tb.Wd;
  const uint64_t *s_din = smem;                                         // dev_ingest: D_x
  uint64_t *s_nd = smem + Wd;                                           // (was Δ_x)
  const int32_t *s_cs = reinterpret_cast<const int32_t *>(smem + 2 * Wd) + n;
  const int32_t *s_rb = s_cs + n + (n + 1);
  const int32_t *s_do = s_rb + n + 1;
  if (status != 0) {
    if (tid == 0) {
      if (status == 1) {
        c->dead = 1;
        c->calls += 1;
      }
      c->last_status = status;
      if (tout) tout[4 * Wd] = ((unsigned long long)tag << 32) | (uint32_t)status;
      else if (out_status) *out_status = status;
    }
    return;
  }
  for (int k = tid; k < Wd; k += NT) s_nd[k] = s_din[k];
  __syncthreads();
  if (!noop) {
    for (int r = tid; r < tb.R; r += NT) {
      const int x = tb.rowVar[r];
      if (!(s_sup ? s_sup[r] : __ldcg(st.sup + r)) && s_cs[x] > 1) {   // x in s_sup (Alg. 3 L1), a unsupported
        const int a = r - s_rb[x];
        smem_clear_bit(s_nd + s_do[x] + (a >> 6), a & 63);
      }
    }
    __syncthreads();
  }
  for (int k = tid; k < Wd; k += NT) {
    const uint64_t nd = s_nd[k];
    st.dom[k] = nd;
    if (tout) {
      // served calls: every output half carries the request's tag, so the host
      // knows when all have arrived and no system-scope fence is needed
      const unsigned long long tg = (unsigned long long)tag << 32;
      const uint64_t pr = s_din[k] & ~nd;
      tout[2 * k] = tg | (uint32_t)nd;
      tout[2 * k + 1] = tg | (uint32_t)(nd >> 32);
      tout[2 * Wd + 2 * k] = tg | (uint32_t)pr;
      tout[2 * Wd + 2 * k + 1] = tg | (uint32_t)(pr >> 32);
      continue;
    }
    if (out_dom) out_dom[k] = nd;
    if (out_pruned) out_pruned[k] = s_din[k] & ~nd;
  }
  __syncthreads();   // then one cumulative system-scope fence by the status writer
  if (tid == 0) {
    if (tout) tout[4 * Wd] = (unsigned long long)tag << 32;   // status CT_OK
    else if (out_status) __threadfence_system();
    if (!noop && tb.use_index) {
      c->parity ^= 1;
      c->L = Lout;
      c->identity = 0;
    }
    c->calls += 1;
    c->last_status = 0;
    if (out_status) *out_status = 0;
  }
}

// ------------------------------------------------------------------ k_small: one state, one CTA
// Tables of at most kSmallMaxPairs 16-byte blocks (e.g. BASELINE config 2,
// 1e5 tuples = 782 blocks) are latency-bound: every phase runs in ONE block of
// kSmallTPB threads, separated by __syncthreads instead of grid barriers, and
// the compaction is a plain block scan (no look-back).  Same phase semantics
// as k_fused; with_finalize = 0 for sharded tables.
#ifndef CT_SMALL_TPB
#define CT_SMALL_TPB 1024
#endif
constexpr int kSmallTPB = CT_SMALL_TPB;   // experiment builds: -DCT_SMALL_TPB=256|512
constexpr int kWarpIngestMaxRows = 1024;   // k_small ingests with one warp up to this many support rows
constexpr int kSmallMaxPairs = 8192;
constexpr int64_t kSmallMaxWork = 1 << 20;   // W2 x R block-rows above which a table leaves k_small (16 MB)

// Dynamic shared memory of k_small: the ingest / finalize region, then (warp
// ingest only) the update list, the filter items, the residues and the
// support flags, so no phase re-reads what an earlier one produced.
__host__ __device__ inline size_t small_region_bytes(int n, int Wd) {
  const size_t a = ingest_smem_bytes(n, Wd), b = finalize_smem_bytes(n, Wd);
  return ((a > b ? a : b) + 15) / 16 * 16;
}
__host__ __device__ inline size_t small_smem_bytes(int n, int Wd, int R) {
  return small_region_bytes(n, Wd) + (size_t)R * 12 + (size_t)R + 32;
}

// The whole call (k_small and its served form k_small_serve): `smem` = the
// dynamic shared memory, small_smem_bytes(n, Wd, R).
__device__ __forceinline__ void small_call(const TableDev &tb, const StateDev &st, const uint64_t *removed,
                                           int root_mode, int with_finalize, uint64_t *out_dom,
                                           uint64_t *out_pruned, int32_t *out_status, int use_state_out,
                                           uint64_t *smem, unsigned long long *tout = nullptr,
                                           uint32_t tag = 0) {
  Ctl *c = st.ctl;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool t0 = tid == 0;
  const int R = tb.R;
  const bool onchip = R <= kWarpIngestMaxRows;   // lists, residues and flags in shared memory
  __shared__ SmallSh sh;
  char *ext = reinterpret_cast<char *>(smem) + small_region_bytes(tb.n, tb.Wd);
  int32_t *s_res = reinterpret_cast<int32_t *>(ext) + 2 * R;
  uint8_t *s_sup = reinterpret_cast<uint8_t *>(s_res + R);
  if (t0) c->tph[0] = globaltimer();   // phase stamps straight to the state (no registers held)
  SERVE_TRACE(1);
  // everything the later phases need from the state is requested now, in
  // flight while warp 0 ingests: the residues, and each thread's first entry
  // of both index buffers (the parity is not known yet)
  int pid0a = -1, pid0b = -1;
  if (onchip) {
    sh.ulist = reinterpret_cast<int32_t *>(ext);
    sh.items = sh.ulist + R;
    for (int r = tid; r < R; r += kSmallTPB) {
      s_res[r] = st.res[r];
      s_sup[r] = 0;
    }
    if (tid < tb.W2) {
      pid0a = st.idx0[tid];
      pid0b = st.idx1[tid];
    }
    if (tb.R <= kWarpIngestMaxRows) warp_ingest(tb, st, removed, root_mode, smem, nullptr, &sh);
  } else {
    dev_ingest<kSmallTPB>(tb, st, removed, root_mode, smem);
  }
  __syncthreads();
  if (t0) c->tph[1] = globaltimer();
  SERVE_TRACE(6);
  __shared__ int s_go, s_L, s_nrows, s_ident, s_par, s_Lout, s_pre, s_nitems;
  __shared__ uint64_t s_warp[kSmallTPB / 32];
  if (t0) {
    if (onchip) {
      s_go = !(sh.skip | sh.noop | sh.fail);
      s_pre = sh.skip ? -5 : sh.fail ? 1 : sh.noop ? 2 : 0;   // status known before the update (2: no-op)
      s_L = sh.L;
      s_nrows = sh.nrows;
      s_ident = sh.ident;
      s_par = sh.par;
      s_nitems = sh.nitems;
    } else {
      s_go = !(c->skip | c->noop | c->fail_fast);
      s_pre = c->skip ? -5 : c->fail_fast ? 1 : c->noop ? 2 : 0;
      s_L = c->L;
      s_nrows = c->nrows;
      s_ident = c->identity;
      s_par = c->parity;
      s_nitems = c->nitems;
    }
  }
  __syncthreads();
  // ---- update + compaction (Alg. 2), all in this block; every listed row's
  // words are loaded together with the block's currTable word (one round trip)
  if (s_go) {
    const int Lout = onchip ? block_update<kSmallTPB, 8>(tb, st, s_L, s_nrows, s_ident, s_par, s_warp, sh.ulist,
                                                          s_par ? pid0b : pid0a)
                            : block_update<kSmallTPB>(tb, st, s_L, s_nrows, s_ident, s_par, s_warp);
    if (t0) {
      c->L_out = Lout;
      s_Lout = Lout;
    }
  }
  __syncthreads();
  if (t0) c->tph[2] = globaltimer();
  SERVE_TRACE(7);
  // ---- filter (Alg. 3 L3, residues L220): residue probes of every item at
  // once (rows and residues from shared memory: one round trip), then a warp
  // per miss over the new index
  if (s_go) {
    const int Lout = s_Lout;
    if (t0) st.sup[R] = Lout > 0;
    if (Lout > 0) {
      const bool compact = tb.use_index != 0;
      const int32_t *__restrict__ idx = compact ? (s_par ? st.idx0 : st.idx1) : nullptr;
      const int L = compact ? Lout : tb.W2;
      const ulonglong2 *__restrict__ T2 = reinterpret_cast<const ulonglong2 *>(st.T);
      const int nitems = s_nitems;
      uint32_t n_loads = 0;
      if (onchip) {
        // thread i probes item i's residue
        for (int i = tid; i < nitems; i += kSmallTPB) {
          const int row = sh.items[i];
          const int r = s_res[row];
          bool hit = false;
          if (tb.use_res) {
            const ulonglong2 t = T2[r];
            const ulonglong2 s2 = ld_sup2(tb.S + (int64_t)row * tb.Wp + 2 * (int64_t)r);
            hit = ((t.x & s2.x) | (t.y & s2.y)) != 0;
          }
          s_sup[row] = hit ? 1 : 0;
        }
        __syncthreads();
        for (int item = warp; item < nitems; item += kSmallTPB / 32) {
          const int row = sh.items[item];
          if (s_sup[row]) continue;
          const int hit = scan_pairs(idx, T2, tb.S + (int64_t)row * tb.Wp, 0, L, nullptr, lane, n_loads);
          if (lane == 0 && hit >= 0) {
            s_sup[row] = 1;
            st.res[row] = hit;
          }
        }
        __syncthreads();
        if (!with_finalize)   // sharded: k_finalize reads the flags after the combine
          for (int i = tid; i < nitems; i += kSmallTPB) st.sup[sh.items[i]] = s_sup[sh.items[i]];
      } else {
        for (int item = warp; item < nitems; item += kSmallTPB / 32) {
          const int row = st.items[item];
          const uint64_t *__restrict__ srow = tb.S + (int64_t)row * tb.Wp;
          if (tb.use_res) {
            int hit = 0;
            if (lane == 0) {
              const int r = st.res[row];
              const ulonglong2 t = T2[r];
              const ulonglong2 s2 = ld_sup2(srow + 2 * (int64_t)r);
              hit = ((t.x & s2.x) | (t.y & s2.y)) != 0;
            }
            if (__shfl_sync(0xffffffffu, hit, 0)) {
              if (lane == 0) st.sup[row] = 1;
              continue;
            }
          }
          const int hit = scan_pairs(idx, T2, srow, 0, L, nullptr, lane, n_loads);
          if (lane == 0 && hit >= 0) {
            st.sup[row] = 1;
            st.res[row] = hit;
          }
        }
      }
      if (lane == 0 && n_loads) atomicAdd(&c->scan_loads, (unsigned long long)n_loads);
    }
  }
  __syncthreads();
  if (t0) c->tph[3] = c->tph[4] = globaltimer();
  SERVE_TRACE(8);
  if (!with_finalize) {
    if (t0) c->tph[5] = c->tph[6] = c->tph[7] = c->tph[4];
    return;
  }
  if (use_state_out) {
    out_dom = st.out + 1;
    out_pruned = st.out + 1 + tb.Wd;
    out_status = reinterpret_cast<int32_t *>(st.out);
  }
  const int status = s_pre == 2 ? 0 : s_pre != 0 ? s_pre : (s_Lout > 0 ? 0 : 1);
  small_finalize<kSmallTPB>(tb, st, status, s_pre == 2, s_Lout, out_dom, out_pruned, out_status, smem,
                            onchip ? s_sup : nullptr, tout, tag);
  if (t0) c->tph[5] = c->tph[6] = c->tph[7] = globaltimer();
}

__global__ void __launch_bounds__(kSmallTPB, 1) k_small(TableDev tb, const StateDev *__restrict__ states,
                                                       const uint64_t *__restrict__ removed, int root_mode,
                                                       int with_finalize, uint64_t *__restrict__ out_dom,
                                                       uint64_t *__restrict__ out_pruned,
                                                       int32_t *__restrict__ out_status, int use_state_out) {
  extern __shared__ __align__(16) uint64_t smem[];
  const StateDev st = states[0];
  small_call(tb, st, removed, root_mode, with_finalize, out_dom, out_pruned, out_status, use_state_out, smem);
}

// ------------------------------------------------------------------ state copies (backtracking)
// Byte offsets / sizes of the persistent fields of a state block.
struct CopyLayout {
  int64_t T_bytes;           // currTable: W2 16-byte blocks
  int64_t o_T, o_idx0, o_idx1, o_res, o_dom;
  int64_t res_bytes, dom_bytes;
};

// Copies what a state needs from src to dst (threads [t0, t0 + nt) of the
// caller): the control block, currTable, the ACTIVE index buffer (only its L
// entries, none for an identity index), residues and domains -- not the
// other, scratch index buffer nor the per-call scratch.
__device__ __forceinline__ void copy_state_fields(char *__restrict__ dst, const char *__restrict__ src,
                                                  const CopyLayout &cl, int64_t t0, int64_t nt) {
  const Ctl *sc = reinterpret_cast<const Ctl *>(src);
  const int ident = __ldcg(&sc->identity), par = __ldcg(&sc->parity), L = __ldcg(&sc->L);
  const int64_t idx_bytes = ident ? 0 : (int64_t)L * 4;
  const int64_t o_idx = par ? cl.o_idx1 : cl.o_idx0;
  // segments, each a multiple of 16 bytes (the layout pads every field to 256)
  const int64_t seg_off[5] = {0, cl.o_T, o_idx, cl.o_res, cl.o_dom};
  const int64_t seg_len[5] = {256, cl.T_bytes, (idx_bytes + 15) / 16 * 16, (cl.res_bytes + 15) / 16 * 16,
                              (cl.dom_bytes + 15) / 16 * 16};
  for (int g = 0; g < 5; ++g) {
    const uint4 *s4 = reinterpret_cast<const uint4 *>(src + seg_off[g]);
    uint4 *d4 = reinterpret_cast<uint4 *>(dst + seg_off[g]);
    for (int64_t k = t0; k < seg_len[g] / 16; k += nt) d4[k] = __ldcg(s4 + k);
  }
}

// ct_state_copy / ct_state_clone: one state, the whole grid.
__global__ void __launch_bounds__(256) k_state_copy(char *__restrict__ dst, const char *__restrict__ src,
                                                    CopyLayout cl) {
  copy_state_fields(dst, src, cl, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

// ------------------------------------------------------------------ batch restart
// grid (S), 256 threads: state i := src iff state i is dead.
__global__ void __launch_bounds__(256) k_restore_dead(char *__restrict__ pool, size_t pitch,
                                                      const char *__restrict__ src, CopyLayout cl) {
  char *dst = pool + (size_t)blockIdx.x * pitch;
  // one read of `dead` for the whole block: the copy overwrites dst's control
  // block (dead = 0), so a thread reading it after that write would skip its share
  __shared__ int s_dead;
  if (threadIdx.x == 0) s_dead = reinterpret_cast<const Ctl *>(dst)->dead;
  __syncthreads();
  if (!s_dead) return;
  copy_state_fields(dst, src, cl, threadIdx.x, blockDim.x);
}

// ------------------------------------------------------------------ served calls (ct_state_serve)
// A persistent k_small for ONE state.  The request lives in mapped host memory
// as tagged 64-bit words, req[k] = seq << 32 | payload: k < 2 Wd the 32-bit
// halves of the removal bitmap, then the operation (0 propagate, 1 copy from
// another state of the table: the restore of a search, served in place so the
// server keeps running) and the source state's address (two halves).  Warp 0
// polls them in ONE read per lane, and a request is complete when every tag
// equals the next sequence number (the host writes the words in any order; a
// partly written request is simply not complete yet).
// ctl[0] = stop request (host), ctl[1] = 2 once the server has stopped.
// Each request runs small_call with the removal in shared memory and the
// outputs + status written to the mapped output, exactly as a launched
// synchronous call.  The server stops on request or after g_serve_idle_ns
// without one; either way it first marks ctl[1] = 2 and never serves again
// (the host relaunches it for a request it sees unserved), so no request is
// served twice.
constexpr int kServeMaxWd = 14;   // 2 Wd + 3 tagged words <= 32: one per lane of warp 0
constexpr int kServeOutWord = 192;  // uint32 offset from ctl of the tagged outputs: [4 Wd + 1] 64-bit words
__device__ unsigned long long g_serve_idle_ns = 200000000ull;   // 200 ms

__global__ void __launch_bounds__(kSmallTPB, 1) k_small_serve(TableDev tb, const StateDev *__restrict__ states,
                                                             const unsigned long long *req, uint32_t *ctl,
                                                             uint32_t last, CopyLayout cl) {
  extern __shared__ __align__(16) uint64_t smem[];
  __shared__ uint64_t s_rem[kServeMaxWd];
  __shared__ uint32_t s_cmd, s_last, s_op, s_src[2];
  const StateDev st = states[0];
  const int tid = threadIdx.x, lane = tid & 31;
  const int nreq = 2 * tb.Wd + 3;
#ifdef CT_SERVE_TRACE
  if (tid == 0) g_tr = reinterpret_cast<unsigned long long *>(ctl + 64);
#endif
  for (;;) {
    if (tid < 32) {
      const unsigned long long t0 = globaltimer();
      const uint32_t want = last + 1u;
      uint32_t cmd = 0, half = 0;
      for (;;) {
        unsigned long long w = 0;
        bool ok = true;
        if (lane < nreq) {
          w = *(volatile const unsigned long long *)(req + lane);
          ok = (uint32_t)(w >> 32) == want;
        }
        half = (uint32_t)w;
        if (__all_sync(0xffffffffu, ok)) {
          cmd = 1;
          break;
        }
        const uint32_t stop = lane == 0 ? *(volatile const uint32_t *)ctl : 0u;
        if (__shfl_sync(0xffffffffu, stop, 0)) {
          cmd = 2;
          break;
        }
        if (globaltimer() - t0 > g_serve_idle_ns) {
          cmd = 2;
          break;
        }
      }
      if (cmd == 1 && lane < 2 * tb.Wd) reinterpret_cast<uint32_t *>(s_rem)[lane] = half;
      if (cmd == 1 && lane == 2 * tb.Wd) s_op = half;
      if (cmd == 1 && lane > 2 * tb.Wd && lane < nreq) s_src[lane - 2 * tb.Wd - 1] = half;
      if (lane == 0) {
        s_cmd = cmd;
        s_last = want;
      }
    }
    __syncthreads();
    last = s_last;
    if (s_cmd == 2) {
      if (tid == 0) st_release_sys_u32(ctl + 1, 2u);
      return;
    }
    unsigned long long *tout = reinterpret_cast<unsigned long long *>(ctl + kServeOutWord);
    if (s_op == 1) {   // restore: this state := the source state (copy_state_fields), then the tagged OK
      const char *src = reinterpret_cast<const char *>(((unsigned long long)s_src[1] << 32) | s_src[0]);
      copy_state_fields(reinterpret_cast<char *>(st.ctl), src, cl, threadIdx.x, blockDim.x);
      __syncthreads();
      if (tid == 0) tout[4 * tb.Wd] = (unsigned long long)last << 32;
      continue;
    }
    SERVE_TRACE(0);
    small_call(tb, st, s_rem, 0, 1, nullptr, nullptr, nullptr, 1, smem, tout, last);
    SERVE_TRACE(15);
    __syncthreads();
  }
}

}  // namespace ctk
