// ct_batch.cuh -- batched propagation of S independent states of ONE table
// (ct_propagate_many), tile-major.
//
// The per-state kernels of ct_kernels.cuh give every state its own pass over
// its currTable, so each (support row, 16-byte block) pair is fetched once per
// state that needs it: on BASELINE config 4 (4096 states, 37.5 MB of supports)
// that is ~6.9 GB of support words per step, which does not stay in L2 next to
// 512 MB of streamed currTables.  Here the work is ordered the other way round:
//
//   k_bupdate  (a3-a5) a CTA owns a column tile of kTW 16-byte blocks, stages
//              ALL R support rows of that tile in shared memory once (R·kTW·16
//              bytes), then streams the currTable blocks of a whole range of
//              states through it.  Lanes map to (state, block): 32/kTW states
//              per warp, every support access is a conflict-free 16-byte
//              shared-memory load, every currTable access a coalesced 16-byte
//              global load.  Alg. 2 per block as in
//              update_tile: the per-variable OR of the listed rows, complemented
//              for the Δ-branch, ANDed over the changed variables, the block
//              dies early (L175) once nothing valid is left in it.  It visits
//              every block of the DENSE states (a zero block costs one 16-byte
//              read and no support load); a (state, tile) with few valid
//              tuples checks them against the new domains instead (the cell
//              route, tile32_cells).  The survivor bits go to a per-state
//              bitmap and k_bcompact builds the order-preserving index.
//   k_bsparse  (a3-a5) states whose input index is short are updated through
//              it, one CTA per state, their valid tuples checked against the
//              new domains, and compacted in the same pass.
//   k_bprobe   (a6a) one THREAD per (state, filter item): residue probe
//              (PAPER.md L220): T[res] & S[x,a][res] != 0 settles the value,
//              else the next few blocks; a miss goes to a global miss list.
//   k_bscan    (a6b) a quarter warp per miss over the first index entries,
//              then (miss, chunk) units over the rest for the misses still open.
//   k_bingest / k_bfinalize: dev_ingest / dev_finalize (ct_kernels.cuh) with
//              128-thread CTAs, one per state.
#pragma once
#include "ct_kernels.cuh"

namespace ctk {

#ifndef CT_BTPB
#define CT_BTPB 1024
#endif
constexpr int kBTPB = CT_BTPB;     // k_bupdate threads per CTA
constexpr int kBSmallTPB = 128;    // k_bingest / k_bfinalize threads per CTA (one state each)
constexpr int kBProbeTPB = 256;
constexpr int kBScanTPB = 256;
constexpr int kCellVars = 2;       // cell route: at most this many changed variables per state
#ifndef CT_SPARSE_DIV
#define CT_SPARSE_DIV 4
#endif
#ifndef CT_CELL_K
#define CT_CELL_K 4
#endif
constexpr int kSparseDiv = CT_SPARSE_DIV;   // sparse route iff active blocks L <= W2 / kSparseDiv
constexpr int kCellK = CT_CELL_K;           // cell route iff kCellK x (largest block popcount) <= P
constexpr int kBSparseTPB = 256;   // k_bsparse threads per CTA (one state each)
constexpr int kSpB = 4;            // k_bsparse: valid tuples whose cells one thread loads together

// Device view of a batch: S state blocks of `pitch` bytes in one pool, field
// offsets from ct_runtime.cu's StateLayout.
struct BatchDev {
  char *pool;
  int64_t pitch;
  int64_t o_ctl, o_T, o_ulist, o_items, o_res, o_sup, o_scan, o_idx0, o_idx1, o_bmask;
  int64_t o_plist;           // padded update list (kTW = 32 path), see k_bingest
  int64_t t_local;           // tuples of the table (shard): the cell tile's bound
  int32_t plist_po;          // its first padded entry (uint32 index)
  int32_t cell_route;        // 1: k_bupdate<32> stages the tile's tuple cells and may check valid tuples directly
  int32_t *bgo;              // [S] per call: (groups << 20) | update-list length, or -1 if the state does not update
  int2 *miss, *miss2;        // [S·R] global lists of (state, row) probe misses (pass 0 / pass 1 of k_bscan)
  int32_t *nmiss, *nmiss2;   // their lengths (zeroed by k_bingest)
  int32_t *dense, *ndense;   // [S] states k_bupdate updates (in k_bingest's arrival order) and their
                             // number; k_bfinalize zeroes the count for the next call
  int2 *sinfo;               // [S] per call: (index buffer parity, L_out) of each state, from k_bcompact
  unsigned long long *work;  // [7] whole batch, summed over calls until ct_batch_work resets them:
                             // update support words, currTable blocks read, blocks rewritten,
                             // support (and cell) bytes staged into shared memory, valid tuples
                             // checked by the cell routes, states updated by k_bsparse, the updating
                             // states' input active blocks (sum of L_in: the algorithmic currTable traffic)
};

__device__ __forceinline__ Ctl *bctl(const BatchDev &b, int s) {
  return reinterpret_cast<Ctl *>(b.pool + (int64_t)s * b.pitch + b.o_ctl);
}
template <typename T>
__device__ __forceinline__ T *bfield(const BatchDev &b, int s, int64_t off) {
  return reinterpret_cast<T *>(b.pool + (int64_t)s * b.pitch + off);
}

// ------------------------------------------------------------------ a2: ingest, one CTA per state
// dev_ingest (Alg. 1 L1-3, Alg. 2), then, for the kTW = 32 update, the
// update list re-laid out as ONE flat list of shared-memory byte offsets
// (row · 512) in groups padded to a multiple of 4 entries with the all-zero
// row R.  The Δ-branch variables share a single group: T & ¬OR(Δ_x1 rows) &
// ¬OR(Δ_x2 rows) = T & ¬OR(Δ_x1 rows ∪ Δ_x2 rows) (De Morgan), so however many
// variables take the Δ-branch they cost one group end; every dom-branch
// variable is a group of its own.  The last entry of a group carries kEndBit
// (and kInvBit for the Δ group), so k_bupdate walks the list without a group
// table:  plist[0] = padded total P,  plist[po + k] = padded entry k;
// bgo[s] = sparse route << 30 | P << 12 | update-list length (< 4096), or -1
// if the state does not update.
// The per-state work of the layout is paid once per call, not once per tile.
__global__ void __launch_bounds__(kBSmallTPB) k_bingest(TableDev tb, const StateDev *__restrict__ states,
                                                       const uint64_t *__restrict__ removed,
                                                       int64_t removed_stride, BatchDev bd, int build_plist) {
  extern __shared__ __align__(16) uint64_t smem[];
  const StateDev &st = states[blockIdx.x];
  const uint64_t *rem = removed ? removed + (int64_t)blockIdx.x * removed_stride : nullptr;
  dev_ingest<kBSmallTPB>(tb, st, rem, 0, smem);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *bd.nmiss = 0;
    *bd.nmiss2 = 0;
  }
  __shared__ int s_go, s_nrows;
  if (threadIdx.x == 0) {   // the thread that wrote the control fields
    Ctl *c = st.ctl;
    s_go = !(c->skip | c->noop | c->fail_fast);
    s_nrows = c->nrows;
  }
  __syncthreads();
  const int n = tb.n, Wd = tb.Wd;
  int P = 0;
  if (s_go && build_plist) {
    // dev_ingest's shared arrays: |Δ_x|, |D_x| and the group starts of the update list
    const int32_t *s_cd = reinterpret_cast<const int32_t *>(smem + 2 * Wd);
    const int32_t *s_cs = s_cd + n;
    const int32_t *s_ust = s_cs + n;
    __shared__ uint64_t s_warp[kBSmallTPB / 32];
    uint32_t *pl = bfield<uint32_t>(bd, blockIdx.x, bd.o_plist);
    uint32_t *pe = pl + bd.plist_po;
    const uint32_t zrow = (uint32_t)tb.R * 512u;
    const uint32_t *ul = reinterpret_cast<const uint32_t *>(st.ulist);
    // per variable: (dom-branch padded size << 32) | Δ-branch size
    auto sizes = [&](int x) -> uint64_t {
      if (x >= n) return 0ull;
      const int sz = s_ust[x + 1] - s_ust[x];
      if (!sz) return 0ull;
      return use_delta(tb, x, s_cd[x], s_cs[x]) ? (uint64_t)sz : ((uint64_t)((sz + 3) & ~3) << 32);
    };
    // pass 1: the Δ group's size (it goes first, the dom groups after it)
    uint64_t tot = 0;
    for (int base = 0; base < n; base += kBSmallTPB) {
      uint64_t t;
      block_excl_scan<kBSmallTPB>(sizes(base + threadIdx.x), s_warp, t);
      tot += t;
    }
    const int nd = (int)(tot & 0xffffffffu), pd = (nd + 3) & ~3;
    P = pd + (int)(tot >> 32);
    // pass 2: every variable writes its entries at its offset
    uint64_t carry = 0;
    for (int base = 0; base < n; base += kBSmallTPB) {
      const int x = base + threadIdx.x;
      const uint64_t v = sizes(x);
      uint64_t t;
      const uint64_t ex = block_excl_scan<kBSmallTPB>(v, s_warp, t) + carry;
      carry += t;
      if (v) {
        const bool dl = (v >> 32) == 0;
        const int sz = s_ust[x + 1] - s_ust[x];
        const int off = dl ? (int)(ex & 0xffffffffu) : pd + (int)(ex >> 32);
        for (int j = 0; j < sz; ++j) pe[off + j] = (ul[s_ust[x] + j] & kRowMask) * 512u;
        if (!dl) {
          const int psz = (sz + 3) & ~3;
          for (int j = sz; j < psz; ++j) pe[off + j] = zrow;
          pe[off + psz - 1] |= kEndBit;
        }
      }
    }
    if (threadIdx.x < pd - nd) pe[nd + threadIdx.x] = zrow;
    // cell-route descriptor (tile32_cells): the changed variables' cell
    // positions and new domains D'_x (dev_ingest's s_din), when there are at
    // most kCellVars of them and each domain is one 64-bit word:
    //   plist[1] = their number (0: rows only), plist[4 + k] = cell word << 8 |
    //   bit shift, plist[8 + 2k .. 9 + 2k] = D'_x lo/hi
    __shared__ int s_nchg, s_cok;
    if (threadIdx.x == 0) {
      s_nchg = 0;
      s_cok = bd.cell_route;
    }
    __syncthreads();   // also orders the Δ group's entries before its flags below
    for (int x = threadIdx.x; x < n; x += kBSmallTPB) {
      if (s_ust[x + 1] > s_ust[x]) {
        const int k = atomicAdd(&s_nchg, 1);
        const int w0 = tb.domOff[x];
        if (k >= kCellVars || tb.domOff[x + 1] - w0 != 1) {
          s_cok = 0;
        } else {
          const int bit = x * tb.cell_bits;
          pl[4 + k] = (uint32_t)((bit >> 5) << 8) | (uint32_t)(bit & 31);
          pl[8 + 2 * k] = (uint32_t)smem[w0];
          pl[9 + 2 * k] = (uint32_t)(smem[w0] >> 32);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (pd) pe[pd - 1] |= kEndBit | kInvBit;
      pl[0] = (uint32_t)P;
      pl[1] = s_cok ? (uint32_t)s_nchg : 0u;
    }
  }
  if (threadIdx.x == 0) {
    int sparse = 0;
    if (s_go && build_plist && bd.cell_route && tb.use_index) {
      // the sparse route (k_bsparse) for a state with few active blocks whose
      // changed variables the cell route can check (plist[1] > 0)
      const uint32_t *pl = bfield<const uint32_t>(bd, blockIdx.x, bd.o_plist);
      const Ctl *c = st.ctl;
      const int L = c->identity ? tb.W2 : c->L;
      sparse = (__ldcg(pl + 1) > 0u && (int64_t)L * kSparseDiv <= tb.W2) ? 1 : 0;
    }
    bd.bgo[blockIdx.x] = s_go ? (sparse << 30) | (P << 12) | s_nrows : -1;
    if (s_go) atomicAdd(bd.work + 6, (unsigned long long)(st.ctl->identity ? tb.W2 : st.ctl->L));
    if (s_go && !sparse) {
      const int at = atomicAdd(bd.ndense, 1);
      if (at < (int)gridDim.x) bd.dense[at] = blockIdx.x;   // (grid = S states)
    }
  }
}

// ------------------------------------------------------------------ a3-a5: tile-major update
// 16-byte shared-memory load at a 32-bit shared address.
__device__ __forceinline__ ulonglong2 lds128(uint32_t addr) {
  ulonglong2 v;
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];\n" : "=l"(v.x), "=l"(v.y) : "r"(addr));
  return v;
}
// The same, predicated on p != 0 (v keeps its value otherwise).
__device__ __forceinline__ void lds128p(uint32_t addr, uint32_t p, ulonglong2 &v) {
  asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %3, 0;\n @q ld.shared.v2.u64 {%0, %1}, [%2];\n}\n"
               : "+l"(v.x), "+l"(v.y) : "r"(addr), "r"(p));
}

// One state's tile when the tile is a full warp (kTW = 32): every lane works on
// the same state, so the walk over the flat padded list (k_bingest) is
// warp-uniform.  `pe` = lane k holds entry k of the first 32 (prefetched);
// later chunks of 32 are loaded from `pl`; the current chunk sits in this
// warp's shared slot `s_pl`, so one broadcast 16-byte load yields four row
// offsets.  Per step of four rows: four conflict-free 16-byte shared loads
// (predicated off for lanes whose block is dead: they cost no wavefront) and
// 3-input ORs; a group end (kEndBit on the step's 4th entry) ANDs the group's
// OR, complemented for the Δ group, into the mask and applies Alg. 2's early
// break per block.  `s_lane` = shared address of this lane's
// column of row 0.  Returns the new block value; adds to `nsteps` the steps
// this lane took while live (4 support rows each).
__device__ __forceinline__ ulonglong2 tile32_flat(uint32_t s_lane, uint32_t *s_pl, const uint32_t *pl, int P,
                                                  uint32_t pe, ulonglong2 tw, bool live, uint32_t &nsteps) {
  const int lane = threadIdx.x & 31;
  uint64_t mx = ~0ull, my = ~0ull, ax = 0, ay = 0;
  uint32_t lv = live ? 1u : 0u;
  ulonglong2 v0 = make_ulonglong2(0ull, 0ull), v1 = v0, v2 = v0, v3 = v0;
  for (int c = 0; c < P; c += 32) {
    if (c > 0) pe = __ldcg(pl + c + lane);
    __syncwarp();
    s_pl[lane] = pe;
    __syncwarp();
    const uint4 *rp = reinterpret_cast<const uint4 *>(s_pl);
    const int n4 = min(32, P - c) >> 2;
    for (int i = 0; i < n4; ++i) {
      const uint4 r = rp[i];
      // predicated (not branched) loads: a dead lane issues no shared-memory
      // access and ORs stale values, which is harmless: its mask only shrinks
      // (a Δ group ANDs a complement, a dom group an OR), and its block is 0
      lds128p(s_lane + r.x, lv, v0);
      lds128p(s_lane + r.y, lv, v1);
      lds128p(s_lane + r.z, lv, v2);
      lds128p(s_lane + (r.w & (kEndBit - 1u)), lv, v3);
      ax |= v0.x | v1.x;
      ay |= v0.y | v1.y;
      ax |= v2.x | v3.x;
      ay |= v2.y | v3.y;
      nsteps += lv;
      if (r.w & kEndBit) {                                  // warp-uniform: a group ends here
        const uint64_t inv = (r.w & kInvBit) ? ~0ull : 0ull; // Δ group: AND the complement
        mx &= ax ^ inv;
        my &= ay ^ inv;
        ax = ay = 0;
        live = live && ((tw.x & mx) | (tw.y & my)) != 0;    // Alg. 2, per block
        lv = live ? 1u : 0u;
        if (!__any_sync(0xffffffffu, live)) {
          __syncwarp();
          return make_ulonglong2(0ull, 0ull);
        }
      }
    }
  }
  __syncwarp();   // the slot is rewritten for the next state
  return make_ulonglong2(tw.x & mx, tw.y & my);
}

// The cell route: the same new block computed from the definition of a valid
// tuple instead of the support rows -- a tuple that was
// valid before the call stays valid iff its value of every CHANGED variable is
// still in D'_x (the unchanged variables' values were, and still are, in
// their domains).  Alg. 2's mask ANDed into T keeps exactly these tuples, so
// the result is the same block; k_bupdate takes this route for a (state, tile)
// when the warp's blocks hold so few valid tuples that checking each one is
// cheaper than OR-ing the update list's rows.  `s_cells` = the tile's cells in
// shared memory, [cell word][bit position 0..127][block 0..31] (a lane reads
// its own block's column: conflict-free); `dsc` = lane k holds plist[k]
// (k_bingest's descriptor); `maxc` = the warp's largest per-block popcount.
// Adds the tuples this lane checked to `nchk`.
__device__ __forceinline__ ulonglong2 tile32_cells(const uint32_t *s_cells, int nchg, uint32_t dsc, ulonglong2 tw,
                                                   bool live, int maxc, uint32_t &nchk) {
  const int lane = threadIdx.x & 31;
  const uint32_t ws0 = __shfl_sync(0xffffffffu, dsc, 4), ws1 = __shfl_sync(0xffffffffu, dsc, 5);
  const uint32_t d0l = __shfl_sync(0xffffffffu, dsc, 8), d0h = __shfl_sync(0xffffffffu, dsc, 9);
  const uint32_t d1l = __shfl_sync(0xffffffffu, dsc, 10), d1h = __shfl_sync(0xffffffffu, dsc, 11);
  const uint64_t dm0 = ((uint64_t)d0h << 32) | d0l;
  const uint64_t dm1 = nchg > 1 ? (((uint64_t)d1h << 32) | d1l) : ~0ull;   // one variable: accept all
  // (one changed variable: the second slot reads the first's word, harmlessly)
  const uint32_t *c0 = s_cells + (ws0 >> 8) * 4096 + lane;
  const uint32_t *c1 = s_cells + ((nchg > 1 ? ws1 : ws0) >> 8) * 4096 + lane;
  const uint32_t sh0 = ws0 & 31u, sh1 = nchg > 1 ? (ws1 & 31u) : 0u;
  // the block as four 32-bit words: the remaining bits (a, b, c, d) are
  // visited lowest first, one per iteration, and a failed tuple's bit is
  // cleared from the result words (ra .. rd)
  uint32_t a = 0, b = 0, c = 0, d = 0;
  if (live) {
    a = (uint32_t)tw.x;
    b = (uint32_t)(tw.x >> 32);
    c = (uint32_t)tw.y;
    d = (uint32_t)(tw.y >> 32);
  }
  uint32_t ra = a, rb = b, rc = c, rd = d;
  for (int it = 0; it < maxc; ++it) {
    const uint32_t w = a ? a : b ? b : c ? c : d;
    if (w) {
      const int q = a ? 0 : b ? 32 : c ? 64 : 96;
      const uint32_t bit = w & (0u - w);
      const int pos = q + __ffs(w) - 1;
      const uint32_t v0 = (c0[pos * 32] >> sh0) & 0xffu;
      const uint32_t v1 = (c1[pos * 32] >> sh1) & 0xffu;
      const uint32_t ok = (uint32_t)((dm0 >> v0) & (dm1 >> v1)) & 1u;
      const uint32_t kill = ok ? 0u : bit;
      if (q == 0) {
        a ^= bit;
        ra ^= kill;
      } else if (q == 32) {
        b ^= bit;
        rb ^= kill;
      } else if (q == 64) {
        c ^= bit;
        rc ^= kill;
      } else {
        d ^= bit;
        rd ^= kill;
      }
      ++nchk;
    }
  }
  if (!live) return make_ulonglong2(0ull, 0ull);
  return make_ulonglong2(((uint64_t)rb << 32) | ra, ((uint64_t)rd << 32) | rc);
}

// Persistent: CTA c processes the contiguous unit range [U·c/G, U·(c+1)/G) of
// the U = ntiles·nchunk units (tile-major: unit u = (tile u / nchunk, state
// chunk u % nchunk)), so it reloads its shared support tile at most a few
// times.  Dynamic shared memory: R·kTW 16-byte entries.  Per (state, tile) the
// survivor bits go to the state's block bitmap (k_bcompact builds the index).
template <int kTW>
__global__ void __launch_bounds__(kBTPB, 1) k_bupdate(TableDev tb, BatchDev bd, int S, int ntiles, int nchunk,
                                                     int chunk_states) {
  extern __shared__ __align__(16) ulonglong2 s_sup[];   // [R + 1][kTW], row R = 0; then the cell tile (kTW = 32)
  __shared__ __align__(16) uint32_t s_plw[kBTPB];        // per warp: 32 update-list entries (kTW = 32 path)
  constexpr int SPW = 32 / kTW;                         // states per warp
  const int R = tb.R, W2 = tb.W2;
  const int64_t Wp = tb.Wp, Wp2 = tb.Wp / 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const int sub = lane / kTW, bl = lane % kTW;
  const uint32_t s_lane = (uint32_t)__cvta_generic_to_shared(s_sup) + 16u * (uint32_t)bl;
  const int64_t units = (int64_t)ntiles * nchunk;
  const int64_t u0 = units * blockIdx.x / gridDim.x, u1 = units * (blockIdx.x + 1) / gridDim.x;
  int cur_tile = -1;
  const int nd = min(__ldcg(bd.ndense), S);   // states on the list (k_bingest)
  uint32_t w_loads = 0, w_writes = 0, w_reads = 0, w_cells = 0;   // this lane's share of the batch work counters
  unsigned long long w_staged = 0;
  for (int64_t u = u0; u < u1; ++u) {
    const int tile = (int)(u / nchunk), chunk = (int)(u - (int64_t)tile * nchunk);
    if (tile != cur_tile) {
      __syncthreads();   // every warp is done with the previous tile
      for (int i = threadIdx.x; i < (R + 1) * kTW; i += blockDim.x) {
        const int row = i / kTW;
        const int64_t blk = (int64_t)tile * kTW + (i - row * kTW);
        s_sup[i] = (row < R && blk < Wp2) ? ld_sup2(tb.S + (int64_t)row * Wp + 2 * blk)
                                          : make_ulonglong2(0ull, 0ull);
      }
      if (kTW == 32 && bd.cell_route) {
        // the tile's 4096 tuples' cells, [cell word][bit position][block]:
        // thread q reads 4 consecutive tuples of block q % 32 (whole sectors)
        uint32_t *s_cells = reinterpret_cast<uint32_t *>(s_sup + (R + 1) * kTW);
        const int cw = tb.cell_words;
        for (int q = threadIdx.x; q < 1024; q += blockDim.x) {
          const int b = q & 31, p4 = (q >> 5) * 4;
          const int64_t j0 = (int64_t)tile * 4096 + b * 128 + p4;
          const uint32_t *src = tb.cells + j0 * cw;
          for (int t = 0; t < 4; ++t) {
            const bool ok = j0 + t < bd.t_local;
            for (int w = 0; w < cw; ++w) s_cells[w * 4096 + (p4 + t) * 32 + b] = ok ? __ldg(src + t * cw + w) : 0u;
          }
        }
        w_staged += (unsigned long long)4096 * cw * 4;
      }
      __syncthreads();
      cur_tile = tile;
      w_staged += (unsigned long long)(R + 1) * kTW * 16;
    }
    // this unit's slice of the dense-state list (k_bingest: the updating
    // states that k_bsparse does not take)
    const int cs = (nd + nchunk - 1) / nchunk;
    const int s0 = chunk * cs, s1 = min(nd, s0 + cs);
    const int blk = tile * kTW + bl;
    const bool inblk = blk < W2;
    // software pipeline: the next state's go word, currTable block and first
    // update-list entries are in flight while the current state is processed,
    // and the state id after it (the list entry they depend on)
    const int step = nwarps * SPW;
    int i = s0 + warp * SPW + sub;
    int go_n = -1;
    ulonglong2 tw_n = make_ulonglong2(0ull, 0ull);
    uint32_t ev_n = 0, dsc_n = 0;
    auto fetch = [&](int ss) {
      go_n = -1;
      tw_n = make_ulonglong2(0ull, 0ull);
      ev_n = dsc_n = 0;
      if (ss >= 0) {
        const char *sb = bd.pool + (int64_t)ss * bd.pitch;
        go_n = __ldcg(bd.bgo + ss);
        if (inblk) tw_n = __ldcg(reinterpret_cast<const ulonglong2 *>(sb + bd.o_T) + blk);
        if constexpr (kTW == 32) {
          const uint32_t *pl = reinterpret_cast<const uint32_t *>(sb + bd.o_plist);
          ev_n = __ldcg(pl + bd.plist_po + lane);
          if (lane < 12) dsc_n = __ldcg(pl + lane);
        } else {
          if (bl < R) ev_n = __ldcg(reinterpret_cast<const uint32_t *>(sb + bd.o_ulist) + bl);
        }
      }
    };
    int id_c = i < s1 ? __ldcg(bd.dense + i) : -1;
    fetch(id_c);
    int id_n = i + step < s1 ? __ldcg(bd.dense + i + step) : -1;
    for (int base = s0 + warp * SPW; base < s1; base += step, i += step) {
      const int s = max(id_c, 0);
      const int go = go_n;
      const int nr = go < 0 ? -1 : (go & 0xfff);
      const ulonglong2 tw = tw_n;
      uint32_t ev = ev_n;
      const uint32_t dsc = dsc_n;
      fetch(id_n);
      id_c = id_n;
      id_n = i + 2 * step < s1 ? __ldcg(bd.dense + i + 2 * step) : -1;
      const bool upd = nr >= 0 && inblk;         // this lane's block takes part in the update
      const bool had = upd && (tw.x | tw.y) != 0;
      uint32_t nl = 0;
      char *sb = bd.pool + (int64_t)s * bd.pitch;
      const uint32_t *ul = reinterpret_cast<const uint32_t *>(sb + bd.o_ulist);
      ulonglong2 nt;
      if constexpr (kTW == 32) {
        if (nr < 0) continue;                    // warp-uniform: one state per warp
        const int P = (go >> 12) & 0x3ffff;
        const int nchg = __shfl_sync(0xffffffffu, dsc, 1);
        const int cnt = had ? __popcll(tw.x) + __popcll(tw.y) : 0;
        const int maxc = __reduce_max_sync(0xffffffffu, (unsigned)cnt);
        if (maxc == 0) {
          nt = make_ulonglong2(0ull, 0ull);
        } else if (nchg > 0 && kCellK * maxc <= P) {   // few valid tuples: check them (cost model: DESIGN §7)
          nt = tile32_cells(reinterpret_cast<const uint32_t *>(s_sup + (R + 1) * kTW), nchg, dsc, tw, had, maxc,
                            w_cells);
        } else {
          nt = tile32_flat(s_lane, s_plw + 32 * warp, reinterpret_cast<const uint32_t *>(sb + bd.o_plist) + bd.plist_po,
                           P, ev, tw, had, nl);
        }
      } else {
        bool live = had;
        uint64_t mx = ~0ull, my = ~0ull, ax = 0, ay = 0;
        const int maxn = __reduce_max_sync(0xffffffffu, live ? nr : 0);
        for (int p0 = 0; p0 < maxn; p0 += kTW) {
          if (p0 > 0) ev = (nr >= 0 && p0 + bl < nr) ? __ldcg(ul + p0 + bl) : 0u;
          const int cnt = min(kTW, maxn - p0);
          for (int q0 = 0; q0 < cnt; q0 += 8) {
#pragma unroll
            for (int q = q0; q < q0 + 8; ++q) {
              const uint32_t e = __shfl_sync(0xffffffffu, ev, sub * kTW + (q & (kTW - 1)));
              if (live && p0 + q < nr && q < kTW) {
                const ulonglong2 v = s_sup[(e & kRowMask) * kTW + bl];
                ++nl;
                ax |= v.x;
                ay |= v.y;
                if (e & kEndBit) {
                  if (e & kInvBit) {
                    mx &= ~ax;
                    my &= ~ay;
                  } else {
                    mx &= ax;
                    my &= ay;
                  }
                  ax = ay = 0;
                  live = ((tw.x & mx) | (tw.y & my)) != 0;   // Alg. 2, per block
                }
              }
            }
          }
          if (!__any_sync(0xffffffffu, live)) break;
        }
        nt = make_ulonglong2(tw.x & mx, tw.y & my);
      }
      const bool wr = had && (nt.x != tw.x || nt.y != tw.y);
      if (wr) reinterpret_cast<ulonglong2 *>(sb + bd.o_T)[blk] = nt;
      const bool keep = had && (nt.x | nt.y) != 0;
      const unsigned bk = __ballot_sync(0xffffffffu, keep);
      w_writes += wr ? 1u : 0u;
      w_reads += upd ? 1u : 0u;
      if constexpr (kTW == 32) {
        w_loads += 4u * nl;               // steps of 4 rows (padding rows included) while live
      } else {
        w_loads += nl;                    // per lane
      }
      if (bl == 0 && nr >= 0) {
        // survivor bits of this tile -> bits [tile·kTW, tile·kTW + kTW) of the bitmap
        uint8_t *bm = reinterpret_cast<uint8_t *>(sb + bd.o_bmask);
        const unsigned bits = kTW == 32 ? bk : (bk >> (sub * kTW)) & ((1u << kTW) - 1u);
        if (kTW == 32) reinterpret_cast<uint32_t *>(bm)[tile] = bits;
        else if (kTW == 16) reinterpret_cast<uint16_t *>(bm)[tile] = (uint16_t)bits;
        else bm[tile] = (uint8_t)bits;
      }
    }
  }
  // batch work counters: one reduction per warp for the whole launch
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    w_loads += __shfl_xor_sync(0xffffffffu, w_loads, o);
    w_writes += __shfl_xor_sync(0xffffffffu, w_writes, o);
    w_reads += __shfl_xor_sync(0xffffffffu, w_reads, o);
    w_cells += __shfl_xor_sync(0xffffffffu, w_cells, o);
  }
  if (lane == 0) {
    if (w_loads) atomicAdd(bd.work + 0, 2ull * w_loads);
    if (w_reads) atomicAdd(bd.work + 1, (unsigned long long)w_reads);
    if (w_writes) atomicAdd(bd.work + 2, (unsigned long long)w_writes);
    if (w_cells) atomicAdd(bd.work + 4, (unsigned long long)w_cells);
  }
  if (threadIdx.x == 0 && w_staged) atomicAdd(bd.work + 3, w_staged);
}

// ------------------------------------------------------------------ a4: index compaction, one CTA per state
// The order-preserving index of the non-zero blocks (RSparseBitSet, SURVEY
// §8(a) a4) from the survivor bitmap k_bupdate wrote, 128 bitmap words (4096
// blocks) per round: a block scan of the words' popcounts, then every warp
// expands 32 words, one word per step with the lanes as its bits, so the index
// stores are coalesced.  Writes L_out; the index goes to the buffer the
// single-state path would write (a batch state continues like a single state).
__global__ void __launch_bounds__(kBSmallTPB) k_bcompact(TableDev tb, BatchDev bd) {
  const int s = blockIdx.x;
  const int go = __ldcg(bd.bgo + s);
  if (go < 0 || (go >> 30)) return;   // no update, or k_bsparse compacted it
  __shared__ uint64_t s_warp[kBSmallTPB / 32];
  __shared__ uint32_t s_word[kBSmallTPB], s_pre[kBSmallTPB];
  Ctl *c = bctl(bd, s);
  const uint32_t *bm = bfield<const uint32_t>(bd, s, bd.o_bmask);
  int32_t *idx_out = bfield<int32_t>(bd, s, __ldcg(&c->parity) ? bd.o_idx0 : bd.o_idx1);
  const int nw = (tb.W2 + 31) >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t carry = 0;
  for (int base = 0; base < nw; base += kBSmallTPB) {
    const int k = base + threadIdx.x;
    uint32_t w = k < nw ? __ldcg(bm + k) : 0u;
    // k_bupdate writes only the tiles' bits: bits of the last word past W2 are never written
    if (k == nw - 1 && (tb.W2 & 31)) w &= (1u << (tb.W2 & 31)) - 1u;
    uint64_t total;
    const uint64_t ex = block_excl_scan<kBSmallTPB>((uint64_t)__popc(w), s_warp, total);
    if (tb.use_index) {
      s_word[threadIdx.x] = w;
      s_pre[threadIdx.x] = (uint32_t)(carry + ex);
      __syncthreads();
      for (int j = warp * 32; j < warp * 32 + 32; ++j) {
        const uint32_t wj = s_word[j];
        if ((wj >> lane) & 1u) idx_out[s_pre[j] + __popc(wj & lanemask_lt())] = (base + j) * 32 + lane;
      }
      __syncthreads();
    }
    carry += total;
  }
  if (threadIdx.x == 0) {
    c->L_out = (int32_t)carry;
    bd.sinfo[s] = make_int2(__ldcg(&c->parity), (int)carry);
  }
}

// ------------------------------------------------------------------ a3-a5, sparse states: one CTA per state
// A state whose active index holds few blocks (bgo bit 30, k_bingest) is
// updated through its index instead of densely: each active block's valid
// tuples are checked against the changed variables' new domains (the cell
// route's test, tile32_cells: a tuple valid before the call stays valid iff
// tau[x] in D'_x for every changed x, PAPER.md L189-193 -- the tuples Alg. 2's
// mask keeps), the block is rewritten if it changed, and the surviving blocks
// form the new order-preserving index at once (a4, chunks of 128 entries,
// block scan), so k_bcompact skips the state.  Reads L_in 16-byte blocks and
// one cell word per changed variable per valid tuple (the cells are
// L2-resident), instead of all W2 blocks.
__global__ void __launch_bounds__(kBSparseTPB) k_bsparse(TableDev tb, BatchDev bd) {
  const int s = blockIdx.x;
  const int go = __ldcg(bd.bgo + s);
  if (go < 0 || !(go >> 30)) return;
  __shared__ uint64_t s_warp[kBSparseTPB / 32];
  Ctl *c = bctl(bd, s);
  const uint32_t *pl = bfield<const uint32_t>(bd, s, bd.o_plist);
  const int nchg = (int)__ldcg(pl + 1);
  const uint32_t ws0 = __ldcg(pl + 4), ws1 = __ldcg(pl + 5);
  const uint64_t dm0 = ((uint64_t)__ldcg(pl + 9) << 32) | __ldcg(pl + 8);
  const uint64_t dm1 = nchg > 1 ? (((uint64_t)__ldcg(pl + 11) << 32) | __ldcg(pl + 10)) : ~0ull;
  const uint32_t sh0 = ws0 & 31u, sh1 = nchg > 1 ? (ws1 & 31u) : 0u;
  const int64_t cw = tb.cell_words;
  const uint32_t *cl0 = tb.cells + (ws0 >> 8), *cl1 = tb.cells + (nchg > 1 ? (ws1 >> 8) : (ws0 >> 8));
  const int ident = __ldcg(&c->identity), par = __ldcg(&c->parity);
  const int L = ident ? tb.W2 : __ldcg(&c->L);
  const int32_t *idx_in = ident ? nullptr : bfield<const int32_t>(bd, s, par ? bd.o_idx1 : bd.o_idx0);
  int32_t *idx_out = bfield<int32_t>(bd, s, par ? bd.o_idx0 : bd.o_idx1);
  ulonglong2 *T = bfield<ulonglong2>(bd, s, bd.o_T);
  uint32_t n_writes = 0, n_cells = 0;
  int carry = 0;
  for (int base = 0; base < L; base += kBSparseTPB) {
    const int i = base + threadIdx.x;
    bool keep = false;
    int b = 0;
    if (i < L) {
      b = idx_in ? __ldcg(idx_in + i) : i;
      const ulonglong2 t = __ldcg(T + b);
      uint64_t kx = 0, ky = 0;
      const int64_t j0 = (int64_t)b * 128;
      // the block's valid tuples in batches of kSpB: their cell loads are
      // independent, so a batch costs one round trip to L2
      uint64_t rx = t.x, ry = t.y;
      while (rx | ry) {
        int pos[kSpB];
        uint32_t c0[kSpB], c1[kSpB];
#pragma unroll
        for (int k = 0; k < kSpB; ++k) {
          pos[k] = -1;
          if (rx) {
            pos[k] = __ffsll((long long)rx) - 1;
            rx &= rx - 1;
          } else if (ry) {
            pos[k] = 64 + __ffsll((long long)ry) - 1;
            ry &= ry - 1;
          }
        }
#pragma unroll
        for (int k = 0; k < kSpB; ++k) {
          c0[k] = c1[k] = 0u;
          if (pos[k] >= 0) {
            c0[k] = __ldg(cl0 + (j0 + pos[k]) * cw);
            c1[k] = __ldg(cl1 + (j0 + pos[k]) * cw);
          }
        }
#pragma unroll
        for (int k = 0; k < kSpB; ++k) {
          if (pos[k] < 0) continue;
          const uint32_t v0 = (c0[k] >> sh0) & 0xffu, v1 = (c1[k] >> sh1) & 0xffu;
          if (!((dm0 >> v0) & (dm1 >> v1) & 1ull)) {
            if (pos[k] >= 64) ky |= 1ull << (pos[k] - 64);
            else kx |= 1ull << pos[k];
          }
          ++n_cells;
        }
      }
      const ulonglong2 nt = make_ulonglong2(t.x & ~kx, t.y & ~ky);
      if (kx | ky) {
        T[b] = nt;
        ++n_writes;
      }
      keep = (nt.x | nt.y) != 0ull;
    }
    uint64_t total;
    const uint64_t ex = block_excl_scan<kBSparseTPB>(keep ? 1ull : 0ull, s_warp, total);
    if (keep) idx_out[carry + (int)ex] = b;
    carry += (int)total;
  }
  if (threadIdx.x == 0) {
    c->L_out = carry;
    bd.sinfo[s] = make_int2(par, carry);
    atomicAdd(bd.work + 1, (unsigned long long)L);
    atomicAdd(bd.work + 5, 1ull);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    n_writes += __shfl_xor_sync(0xffffffffu, n_writes, o);
    n_cells += __shfl_xor_sync(0xffffffffu, n_cells, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (n_writes) atomicAdd(bd.work + 2, (unsigned long long)n_writes);
    if (n_cells) atomicAdd(bd.work + 4, (unsigned long long)n_cells);
  }
}

// ------------------------------------------------------------------ a6a: residue probe, one thread per item
// Appends (state, row) to a global miss list, one atomic per warp.
__device__ __forceinline__ void bmiss_push(const BatchDev &bd, int2 *list, int *count, bool miss, int s, int row) {
  const unsigned m = __ballot_sync(0xffffffffu, miss);
  if (!m) return;
  const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
  int base = 0;
  if (lane == leader) base = atomicAdd(count, __popc(m));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (miss) list[base + __popc(m & lanemask_lt())] = make_int2(s, row);
}

// grid = ceil(S·Rp / kBProbeTPB), Rp = max(R, 1): thread (s, i) takes item i
// of state s.  Residue probe; on a miss the same thread tries
// the kBProbeNext blocks after the residue (all loads in flight together: on
// tables with spread-out supports a support is usually a few blocks away), and
// only then queues the item for k_bscan.  Thread (s, 0) also publishes
// "currTable non-empty" (sup[R]).
#ifndef CT_BPROBE_NEXT
#define CT_BPROBE_NEXT 4
#endif
constexpr int kBProbeNext = CT_BPROBE_NEXT;
__global__ void __launch_bounds__(kBProbeTPB) k_bprobe(TableDev tb, BatchDev bd, int S) {
  const int Rp = max(tb.R, 1), W2 = tb.W2;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int s = (int)(gid / Rp), i = (int)(gid - (int64_t)s * Rp);
  bool miss = false;
  int row = 0;
  if (s < S && __ldcg(bd.bgo + s) >= 0) {
    Ctl *c = bctl(bd, s);
    const int Lout = __ldcg(&c->L_out);
    uint8_t *sup = bfield<uint8_t>(bd, s, bd.o_sup);
    if (i == 0) sup[tb.R] = Lout > 0;
    if (Lout > 0 && i < __ldcg(&c->nitems)) {
      row = __ldcg(bfield<int32_t>(bd, s, bd.o_items) + i);
      miss = true;
      if (tb.use_res) {
        int32_t *res = bfield<int32_t>(bd, s, bd.o_res);
        const ulonglong2 *T2 = bfield<const ulonglong2>(bd, s, bd.o_T);
        const uint64_t *srow = tb.S + (int64_t)row * tb.Wp;
        const int r = __ldcg(res + row);
        const ulonglong2 t = __ldcg(T2 + r);
        const ulonglong2 v = ld_sup2(srow + 2 * (int64_t)r);
        if (((t.x & v.x) | (t.y & v.y)) != 0) {
          sup[row] = 1;
          miss = false;
        } else {
          int blk[kBProbeNext];
          ulonglong2 tn[kBProbeNext], vn[kBProbeNext];
#pragma unroll
          for (int q = 0; q < kBProbeNext; ++q) {
            int k = r + 1 + q;
            blk[q] = k < W2 ? k : k % W2;
          }
#pragma unroll
          for (int q = 0; q < kBProbeNext; ++q) {
            tn[q] = __ldcg(T2 + blk[q]);
            vn[q] = ld_sup2(srow + 2 * (int64_t)blk[q]);
          }
          int hit = -1;
#pragma unroll
          for (int q = kBProbeNext - 1; q >= 0; --q)
            if (((tn[q].x & vn[q].x) | (tn[q].y & vn[q].y)) != 0) hit = blk[q];
          if (hit >= 0) {
            sup[row] = 1;
            res[row] = hit;
            miss = false;
          }
        }
      }
      if (miss) atomicAdd(&c->nscan, 1);
    }
  }
  bmiss_push(bd, bd.miss, bd.nmiss, miss, s, row);
}

// ------------------------------------------------------------------ a6b: scan of the probe misses
// Pass 0: one warp per miss of the global list, rounds of 32·kScanUnroll
// blocks from block 0 (CT's intersectIndex over the dense index), at most
// kBScanRounds rounds; a miss still unresolved goes to the second list.
// Pass 1: (miss, chunk) units of the second list, chunk-major over the
// remaining blocks (long scans: values that lost every support, correlated
// tables), each re-checking the miss's flag between rounds.
#ifndef CT_BSCAN_ROUNDS
#define CT_BSCAN_ROUNDS 4
#endif
constexpr int kBScanRounds = CT_BSCAN_ROUNDS;
constexpr int kBScanFirst = kBScanRounds * 32 * kScanUnroll;   // blocks scanned by pass 0
// Pass 0 with a HALF warp per miss (16 lanes x kScanUnroll entries = 64 index
// entries per round, the two halves of a warp on two misses), the next miss's
// list entry and index parameters loaded while the current one is scanned.
#ifndef CT_BSCAN_QW
#define CT_BSCAN_QW 8
#endif
constexpr int kBScanQW = CT_BSCAN_QW;   // lanes per miss in pass 0 (32 / kBScanQW misses per warp)
__device__ void bscan_pass0(const TableDev &tb, const BatchDev &bd, int gw, int nw) {
  constexpr int QW = kBScanQW, GW = 32 / QW;
  const int lane = threadIdx.x & 31, hl = lane % QW, grp = lane / QW;
  const int nm = __ldcg(bd.nmiss);
  constexpr int kR = QW * kScanUnroll;   // entries per round
  constexpr unsigned kGM = QW == 32 ? 0xffffffffu : ((1u << QW) - 1u);
  auto fetch = [&](int m, int2 &e, int2 &inf) {
    e = make_int2(0, 0);
    inf = make_int2(0, 0);
    if (m < nm) {
      e = __ldcg(bd.miss + m);
      inf = __ldcg(bd.sinfo + e.x);
    }
  };
  int2 e, inf, e_n, inf_n;
  int m = GW * gw + grp;
  fetch(m, e, inf);
  for (int mb = GW * gw; mb < nm; mb += GW * nw, m += GW * nw) {
    fetch(m + GW * nw, e_n, inf_n);
    const bool valid = m < nm;
    const int s = e.x, row = e.y;
    const int L = valid ? (tb.use_index ? inf.y : tb.W2) : 0;
    const int Lf = min(L, kBScanFirst);
    const int32_t *idx = tb.use_index ? bfield<const int32_t>(bd, s, inf.x ? bd.o_idx0 : bd.o_idx1) : nullptr;
    const ulonglong2 *T2 = bfield<const ulonglong2>(bd, s, bd.o_T);
    const uint64_t *srow = tb.S + (int64_t)row * tb.Wp;
    int hit = -1;
    uint32_t n_loads = 0;
    bool active = valid && Lf > 0;
    for (int k0 = 0; __any_sync(0xffffffffu, active); k0 += kR) {
      int pid[kScanUnroll];
      bool in[kScanUnroll];
#pragma unroll
      for (int q = 0; q < kScanUnroll; ++q) {
        const int k = k0 + q * QW + hl;
        in[q] = active && k < Lf;
        pid[q] = in[q] ? (idx ? __ldcg(idx + k) : k) : 0;
      }
      ulonglong2 t[kScanUnroll], v[kScanUnroll];
#pragma unroll
      for (int q = 0; q < kScanUnroll; ++q) {
        t[q] = in[q] ? __ldcg(T2 + pid[q]) : make_ulonglong2(0ull, 0ull);
        v[q] = in[q] ? ld_sup2(srow + 2 * (int64_t)pid[q]) : make_ulonglong2(0ull, 0ull);
      }
      if (active) n_loads += 2 * max(0, min(kR, Lf - k0));
#pragma unroll
      for (int q = kScanUnroll - 1; q >= 0; --q) {
        const unsigned b = __ballot_sync(0xffffffffu, ((t[q].x & v[q].x) | (t[q].y & v[q].y)) != 0);
        const unsigned hb = (b >> (QW * grp)) & kGM;
        const int src = hb ? (QW * grp + __ffs(hb) - 1) : lane;
        const int p = __shfl_sync(0xffffffffu, pid[q], src);
        if (hb && active) hit = p;
      }
      if (hit >= 0 || k0 + kR >= Lf) active = false;
    }
    if (valid && hl == 0) {
      uint8_t *sup = bfield<uint8_t>(bd, s, bd.o_sup);
      if (hit >= 0) {
        sup[row] = 1;
        bfield<int32_t>(bd, s, bd.o_res)[row] = hit;
      } else if (L > kBScanFirst) {
        bd.miss2[atomicAdd(bd.nmiss2, 1)] = e;
      }
      if (n_loads) atomicAdd(&bctl(bd, s)->scan_loads, (unsigned long long)n_loads);
    }
    e = e_n;
    inf = inf_n;
  }
}

__global__ void __launch_bounds__(kBScanTPB) k_bscan(TableDev tb, BatchDev bd, int pass) {
  const int lane = threadIdx.x & 31;
  if (pass == 0) {
    bscan_pass0(tb, bd, blockIdx.x * (kBScanTPB / 32) + (threadIdx.x >> 5), gridDim.x * (kBScanTPB / 32));
    return;
  }
  const int gw = blockIdx.x * (kBScanTPB / 32) + (threadIdx.x >> 5), nw = gridDim.x * (kBScanTPB / 32);
  const int Lmax = tb.W2;   // chunks are laid out over the largest possible index
  const int nm = __ldcg(pass == 0 ? bd.nmiss : bd.nmiss2);
  const int2 *list = pass == 0 ? bd.miss : bd.miss2;
  const int nch = pass == 0 ? 1 : (Lmax > kBScanFirst ? (Lmax - kBScanFirst + kScanChunk - 1) / kScanChunk : 0);
  const int64_t total = (int64_t)nm * nch;
  for (int64_t u = gw; u < total; u += nw) {
    const int chunk = (int)(u / nm);
    const int2 e = __ldcg(list + (int)(u - (int64_t)chunk * nm));
    const int s = e.x, row = e.y;
    uint8_t *sup = bfield<uint8_t>(bd, s, bd.o_sup);
    int k0 = 0, k1 = 0;
    if (pass != 0) {
      const int fl = lane == 0 ? *(volatile const uint8_t *)(sup + row) : 0;
      if (__shfl_sync(0xffffffffu, fl, 0)) continue;
      k0 = kBScanFirst + chunk * kScanChunk;
      k1 = k0 + kScanChunk;
    }
    uint32_t n_loads = 0;
    const ulonglong2 *T2 = bfield<const ulonglong2>(bd, s, bd.o_T);
    const int32_t *idx = tb.use_index ? bfield<const int32_t>(bd, s, __ldcg(&bctl(bd, s)->parity) ? bd.o_idx0 : bd.o_idx1)
                                      : nullptr;
    const int L = tb.use_index ? __ldcg(&bctl(bd, s)->L_out) : tb.W2;
    if (pass == 0) k1 = min(L, kBScanFirst);
    else k1 = min(k1, L);
    if (k0 >= k1) continue;
    const int hit = scan_pairs(idx, T2, tb.S + (int64_t)row * tb.Wp, k0, k1, pass ? sup + row : nullptr, lane,
                               n_loads);
    if (lane == 0) {
      if (hit >= 0) {
        sup[row] = 1;
        bfield<int32_t>(bd, s, bd.o_res)[row] = hit;
      } else if (pass == 0 && L > kBScanFirst) {   // (L: this state's index length)
        bd.miss2[atomicAdd(bd.nmiss2, 1)] = e;
      }
      if (n_loads) atomicAdd(&bctl(bd, s)->scan_loads, (unsigned long long)n_loads);
    }
  }
}

// ------------------------------------------------------------------ a6c-a8: finalize, one CTA per state
__global__ void __launch_bounds__(kBSmallTPB) k_bfinalize(TableDev tb, const StateDev *__restrict__ states,
                                                         uint64_t *__restrict__ out_dom, int64_t dom_stride,
                                                         int32_t *__restrict__ out_status, BatchDev bd) {
  extern __shared__ __align__(16) uint64_t smem[];
  const StateDev &st = states[blockIdx.x];
  if (out_dom) out_dom += (int64_t)blockIdx.x * dom_stride;
  if (out_status) out_status += blockIdx.x;
  if (blockIdx.x == 0 && threadIdx.x == 0) *bd.ndense = 0;   // k_bupdate is done with the list
  dev_finalize<kBSmallTPB>(tb, st, out_dom, nullptr, out_status, smem);
}

__host__ __device__ inline size_t bupdate_smem_bytes(int R, int tw) { return (size_t)(R + 1) * tw * 16; }

}  // namespace ctk
