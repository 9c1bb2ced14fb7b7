// ct_placement.cuh -- SURVEY §8(f) f3: the paper's serial CT propagator on the
// host and its three GPU-offloaded derivatives (§4):
//
//   CT      (CT_PLACE_HOST) the serial propagator: Alg. 1-3 with an RSparseBitSet
//           currTable and residues (RSparseBitSet as in the CT
//           paper), all on the host;
//   CT^u    (CT_PLACE_U)    updateTable on the device: currTable, s_val and the
//           domains go to the device, a kernel builds the mask (the AND over
//           s_val of the OR of the supports of dom(x), the paper's dom-branch
//           kernels updateTableGPU + reduce), the mask comes back and
//           the host ANDs it into currTable; filtering on the host;
//   CT^f    (CT_PLACE_F)    filterDomains on the device: the host updates
//           currTable, then currTable and the domains go to the device, a kernel
//           tests every (x,a), x in s_sup, a in dom(x), against currTable over the
//           whole row and returns a removal bitmap (filterDomainsGPU);
//   CT^uf   (CT_PLACE_UF)   both kernels, the paper's data movement: currTable,
//           s_val and domains in, mask and removal bitmap out.
//
// This is the placement ABLATION (the paper's central design trade-off: copies
// cost up to 50 % / 80 % of kernel time, and CT^u loses to the
// serial CT).  It is a separate, explicitly selected engine
// (ct_host_* in include/ct.h); ct_propagate / ct_propagate_many never route
// through it.  The device-resident path (ct_create / ct_propagate) is this
// library's CT^uf without the per-call currTable traffic.
//
// Kernels: 16-byte (two-word) blocks per thread, 128-bit loads, supports
// row-contiguous [R][Wp] as on the main path (the paper's transposed
// _supportsT_dev would stride single-row scans by R words).  Included once,
// from ct_runtime.cu.
#pragma once
#include <chrono>
#include <vector>

namespace ctk {

constexpr int kPlUpdTPB = 256;
constexpr int kPlFiltTPB = 256;

// CT^u / CT^uf: mask over all W2 16-byte blocks.  rows: the dom-branch row list
// of every x in s_val, grouped by variable (kEndBit marks a group's last row).
// mask[b] = AND_groups OR_rows S[row][b]; blocks whose currTable is already 0
// get mask 0 without loading supports (the host AND leaves them 0 anyway).
// T_out (nullable): currTable & mask for the device filter of CT^uf.
__global__ void __launch_bounds__(kPlUpdTPB) k_pl_update(const uint64_t *__restrict__ S, int64_t Wp, int W2,
                                                         const ulonglong2 *__restrict__ T,
                                                         const uint32_t *__restrict__ rows, int nrows,
                                                         ulonglong2 *__restrict__ mask_out,
                                                         ulonglong2 *__restrict__ T_out) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < W2; b += gridDim.x * blockDim.x) {
    const ulonglong2 t = T[b];
    uint64_t mx = 0, my = 0;
    if (t.x | t.y) {
      mx = my = ~0ull;
      uint64_t ax = 0, ay = 0;
      for (int k = 0; k < nrows; ++k) {
        const uint32_t e = rows[k];
        const ulonglong2 v = ld_sup2(S + (int64_t)(e & kRowMask) * Wp + 2 * (int64_t)b);
        ax |= v.x;
        ay |= v.y;
        if (e & kEndBit) {
          mx &= ax;
          my &= ay;
          ax = ay = 0;
        }
      }
    }
    mask_out[b] = make_ulonglong2(mx, my);
    if (T_out) T_out[b] = make_ulonglong2(t.x & mx, t.y & my);
  }
}

// CT^f / CT^uf: one warp per support row r = (x, a); a value of a variable in
// s_sup that is in dom(x) is removed iff S[r] & currTable = 0 over the whole
// row (Alg. 3 L3; the paper's kernel scans every word; here the
// warp stops at the first common tuple).  rem (Wd words) must be zeroed.
__global__ void __launch_bounds__(kPlFiltTPB) k_pl_filter(const uint64_t *__restrict__ S, int64_t Wp, int W2,
                                                          const ulonglong2 *__restrict__ T,
                                                          const uint64_t *__restrict__ dom,
                                                          const uint8_t *__restrict__ ssup,
                                                          const int32_t *__restrict__ rowVar,
                                                          const int32_t *__restrict__ rowBase,
                                                          const int32_t *__restrict__ domOff, int R,
                                                          unsigned long long *__restrict__ rem) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < R; r += nwarps) {
    const int x = rowVar[r];
    if (!ssup[x]) continue;
    const int a = r - rowBase[x];
    const int w = domOff[x] + (a >> 6);
    const uint64_t bit = 1ull << (a & 63);
    if (!(dom[w] & bit)) continue;
    const uint64_t *__restrict__ srow = S + (int64_t)r * Wp;
    bool hit = false;
    for (int b0 = 0; b0 < W2 && !hit; b0 += 64) {
      uint64_t v = 0;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int b = b0 + q * 32 + lane;
        if (b < W2) {
          const ulonglong2 t = T[b];
          const ulonglong2 s = ld_sup2(srow + 2 * (int64_t)b);
          v |= (t.x & s.x) | (t.y & s.y);
        }
      }
      hit = __any_sync(0xffffffffu, v != 0);
    }
    if (!hit && lane == 0) atomicOr(rem + w, (unsigned long long)bit);
  }
}

}  // namespace ctk

// ================================================================== host side
namespace ctpl {

using Clock = std::chrono::steady_clock;

inline int popc64(uint64_t x) { return __builtin_popcountll(x); }

// The reversible sparse bitset of CT (RSparseBitSet), without
// the trail: the solver's backtracking copies whole states (ct_host_copy).
struct SparseBitSet {
  std::vector<uint64_t> words, mask;
  std::vector<int32_t> index;   // index[0..limit] = the non-zero words
  int32_t limit = -1;

  void init(const std::vector<uint64_t> &w) {
    words = w;
    mask.assign(w.size(), 0ull);
    index.clear();
    for (int32_t i = 0; i < (int32_t)w.size(); ++i)
      if (w[(size_t)i]) index.push_back(i);
    const size_t nz = index.size();
    for (int32_t i = 0; i < (int32_t)w.size(); ++i)
      if (!w[(size_t)i]) index.push_back(i);
    limit = (int32_t)nz - 1;
  }
  bool empty() const { return limit < 0; }
  void clear_mask() {
    for (int32_t i = 0; i <= limit; ++i) mask[(size_t)index[(size_t)i]] = 0;
  }
  void add_to_mask(const uint64_t *m) {
    for (int32_t i = 0; i <= limit; ++i) {
      const int32_t o = index[(size_t)i];
      mask[(size_t)o] |= m[o];
    }
  }
  void reverse_mask() {
    for (int32_t i = 0; i <= limit; ++i) {
      const int32_t o = index[(size_t)i];
      mask[(size_t)o] = ~mask[(size_t)o];
    }
  }
  void intersect_with_mask() {
    for (int32_t i = limit; i >= 0; --i) {
      const int32_t o = index[(size_t)i];
      const uint64_t w = words[(size_t)o] & mask[(size_t)o];
      if (w != words[(size_t)o]) {
        words[(size_t)o] = w;
        if (w == 0) {
          index[(size_t)i] = index[(size_t)limit];
          index[(size_t)limit] = o;
          --limit;
        }
      }
    }
  }
  int32_t intersect_index(const uint64_t *m) const {
    for (int32_t i = 0; i <= limit; ++i) {
      const int32_t o = index[(size_t)i];
      if (words[(size_t)o] & m[o]) return o;
    }
    return -1;
  }
};

}  // namespace ctpl

struct ct_host_table {
  int placement = CT_PLACE_HOST;
  int n = 0, R = 0, Wd = 0;
  int64_t t = 0, W = 0, Wp = 0, W2 = 0;
  int policy = CT_POLICY_AUTO;
  std::vector<int32_t> lo, d, rowBase, domOff, rowVar;
  std::vector<uint64_t> S;          // host supports [R][W] (the serial CT's _supports)
  std::vector<uint64_t> full_dom;
  // device side (placements U / F / UF)
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint64_t *dS = nullptr;           // [R][Wp]
  int32_t *dmeta = nullptr;         // rowVar[R] | rowBase[n+1] | domOff[n+1]
  uint64_t *dT = nullptr, *dT2 = nullptr, *dMask = nullptr, *dDom = nullptr, *dRem = nullptr;
  uint32_t *dRows = nullptr;
  uint8_t *dSsup = nullptr;
  uint64_t *hT = nullptr, *hMask = nullptr, *hDom = nullptr, *hRem = nullptr;   // pinned staging
  uint32_t *hRows = nullptr;
  uint8_t *hSsup = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  int upd_grid = 1, filt_grid = 1;
  ct_place_stats st{};
  int live = 0;
};

struct ct_host_state {
  ct_host_table *tb = nullptr;
  ctpl::SparseBitSet T;
  std::vector<uint64_t> dom;
  std::vector<int32_t> res;         // residue word per support row
  bool dead = false;
};

namespace ctpl {

static void free_host_table(ct_host_table *tb) {
  if (!tb) return;
  if (tb->placement != CT_PLACE_HOST) {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(tb->device);
    if (tb->stream) cudaStreamSynchronize(tb->stream);
    for (void *p : {(void *)tb->dS, (void *)tb->dmeta, (void *)tb->dT, (void *)tb->dT2, (void *)tb->dMask,
                    (void *)tb->dDom, (void *)tb->dRem, (void *)tb->dRows, (void *)tb->dSsup})
      if (p) cudaFree(p);
    for (void *p : {(void *)tb->hT, (void *)tb->hMask, (void *)tb->hDom, (void *)tb->hRem, (void *)tb->hRows,
                    (void *)tb->hSsup})
      if (p) cudaFreeHost(p);
    for (cudaEvent_t e : tb->ev)
      if (e) cudaEventDestroy(e);
    if (tb->own_stream && tb->stream) cudaStreamDestroy(tb->stream);
    if (prev >= 0) cudaSetDevice(prev);
  }
  delete tb;
}

static double ms_since(Clock::time_point a) {
  return std::chrono::duration<double, std::milli>(Clock::now() - a).count();
}

// Alg. 2 on the host: one mask per changed variable (branch by |Δ| < |dom|,
// P:L163), intersect, stop when currTable empties.
static void host_update(ct_host_table *tb, ct_host_state *s, const std::vector<int> &sval,
                        const std::vector<uint64_t> &delta, const std::vector<int> &cdelta,
                        const std::vector<int> &csize) {
  SparseBitSet &T = s->T;
  for (int x : sval) {
    const bool useDelta = tb->policy == CT_POLICY_DELTA || (tb->policy == CT_POLICY_AUTO && cdelta[x] < csize[x]);
    const std::vector<uint64_t> &bits = useDelta ? delta : s->dom;
    T.clear_mask();
    for (int w = tb->domOff[x]; w < tb->domOff[x + 1]; ++w)
      for (uint64_t m = bits[(size_t)w]; m; m &= m - 1) {
        const int a = (w - tb->domOff[x]) * 64 + __builtin_ctzll(m);
        T.add_to_mask(tb->S.data() + (size_t)(tb->rowBase[x] + a) * tb->W);
      }
    if (useDelta) T.reverse_mask();
    T.intersect_with_mask();
    if (T.empty()) break;
  }
}

// Alg. 3 on the host with residues: values of x in s_sup without a valid tuple
// leave dom (written into s->dom).
static void host_filter(ct_host_table *tb, ct_host_state *s, const std::vector<int> &csize) {
  SparseBitSet &T = s->T;
  for (int x = 0; x < tb->n; ++x) {
    if (csize[x] <= 1) continue;   // x not in s_sup
    for (int w = tb->domOff[x]; w < tb->domOff[x + 1]; ++w)
      for (uint64_t m = s->dom[(size_t)w]; m; m &= m - 1) {
        const int a = (w - tb->domOff[x]) * 64 + __builtin_ctzll(m);
        const int r = tb->rowBase[x] + a;
        const uint64_t *row = tb->S.data() + (size_t)r * tb->W;
        int32_t q = s->res[(size_t)r];
        if (!(T.words[(size_t)q] & row[q])) {
          q = T.intersect_index(row);
          if (q >= 0) s->res[(size_t)r] = q;
          else s->dom[(size_t)w] &= ~(1ull << (a & 63));
        }
      }
  }
}

// Rows of the paper's device update for s_val (dom-branch only).
static int build_rows(ct_host_table *tb, ct_host_state *s, const std::vector<int> &sval) {
  int k = 0;
  for (int x : sval) {
    const int k0 = k;
    for (int w = tb->domOff[x]; w < tb->domOff[x + 1]; ++w)
      for (uint64_t m = s->dom[(size_t)w]; m; m &= m - 1) {
        const int a = (w - tb->domOff[x]) * 64 + __builtin_ctzll(m);
        tb->hRows[k++] = (uint32_t)(tb->rowBase[x] + a);
      }
    if (k > k0) tb->hRows[k - 1] |= ctk::kEndBit;
  }
  return k;
}

static float ev_ms(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

}  // namespace ctpl

static ct_status ct_host_propagate_impl(ct_host_state *s, const uint64_t *removed, uint64_t *out_dom,
                                        uint64_t *out_pruned, bool root_mode);

extern "C" {

ct_status ct_host_create(int32_t n, const int32_t *dom_lo, const int32_t *dom_size, const uint64_t *init_dom,
                         int64_t n_tuples, const int32_t *tuples, int32_t placement, const ct_config *cfg_in,
                         ct_host_table **out_table, ct_host_state **out_root, uint64_t *out_dom) {
  using namespace ctpl;
  if (out_table) *out_table = nullptr;
  if (out_root) *out_root = nullptr;
  if (n < 1 || !dom_lo || !dom_size || n_tuples < 0 || (n_tuples > 0 && !tuples) || !out_table || !out_root)
    return fail(CT_EINVAL, "ct_host_create: bad arguments");
  if (placement < CT_PLACE_HOST || placement > CT_PLACE_UF) return fail(CT_EINVAL, "bad placement %d", placement);
  ct_config cfg;
  if (cfg_in) cfg = *cfg_in;
  else ct_config_init(&cfg);
  if (cfg.update_policy < 0 || cfg.update_policy > 2) return fail(CT_EINVAL, "bad update_policy");
  ct_host_table *tb = new (std::nothrow) ct_host_table();
  if (!tb) return fail(CT_ENOMEM, "host allocation failed");
  auto bail = [&](ct_status s) {
    free_host_table(tb);
    return s;
  };
  tb->placement = placement;
  tb->policy = cfg.update_policy;
  tb->n = n;
  tb->t = n_tuples;
  tb->lo.assign(dom_lo, dom_lo + n);
  tb->d.assign(dom_size, dom_size + n);
  tb->rowBase.assign(n + 1, 0);
  tb->domOff.assign(n + 1, 0);
  for (int i = 0; i < n; ++i) {
    if (dom_size[i] < 1) return bail(fail(CT_EINVAL, "dom_size[%d] must be >= 1", i));
    tb->rowBase[i + 1] = tb->rowBase[i] + dom_size[i];
    tb->domOff[i + 1] = tb->domOff[i] + (dom_size[i] + 63) / 64;
  }
  tb->R = tb->rowBase[n];
  tb->Wd = tb->domOff[n];
  tb->W = std::max<int64_t>((n_tuples + 63) / 64, 1);
  tb->Wp = round_up(tb->W, 16);
  tb->W2 = tb->Wp / 2;
  tb->rowVar.assign(std::max(tb->R, 1), 0);
  for (int i = 0; i < n; ++i)
    for (int r = tb->rowBase[i]; r < tb->rowBase[i + 1]; ++r) tb->rowVar[(size_t)r] = i;
  tb->full_dom.assign(tb->Wd, 0ull);
  for (int i = 0; i < n; ++i)
    for (int a = 0; a < dom_size[i]; ++a) tb->full_dom[(size_t)(tb->domOff[i] + a / 64)] |= 1ull << (a % 64);
  // supports and the range-valid tuples
  try {
    tb->S.assign((size_t)tb->R * (size_t)tb->W, 0ull);
  } catch (...) {
    return bail(fail(CT_ENOMEM, "host supports allocation failed"));
  }
  std::vector<uint64_t> T0((size_t)tb->W, 0ull);
  for (int64_t j = 0; j < n_tuples; ++j) {
    bool ok = true;
    for (int i = 0; i < n; ++i) {
      const int64_t v = (int64_t)tuples[j * n + i] - dom_lo[i];
      if (v >= 0 && v < dom_size[i]) tb->S[(size_t)(tb->rowBase[i] + v) * tb->W + (size_t)(j >> 6)] |= 1ull << (j & 63);
      else ok = false;
    }
    if (ok) T0[(size_t)(j >> 6)] |= 1ull << (j & 63);
  }
  if (placement != CT_PLACE_HOST) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || cfg.device < 0 || cfg.device >= ndev) {
      cudaGetLastError();
      return bail(fail(CT_ECUDA, "placement %d needs CUDA device %d", placement, cfg.device));
    }
    tb->device = cfg.device;
    DeviceGuard g(tb->device);
    if (cfg.stream) {
      tb->stream = (cudaStream_t)cfg.stream;
    } else {
      CUDA_TRY(cudaStreamCreateWithFlags(&tb->stream, cudaStreamNonBlocking));
      tb->own_stream = true;
    }
    const size_t sb = (size_t)tb->R * (size_t)tb->Wp * 8, tbytes = (size_t)tb->Wp * 8;
    const size_t mbytes = ((size_t)tb->R + 2 * ((size_t)n + 1)) * 4;
    if (cudaMalloc(&tb->dS, std::max<size_t>(sb, 8)) != cudaSuccess || cudaMalloc(&tb->dmeta, mbytes) != cudaSuccess ||
        cudaMalloc(&tb->dT, tbytes) != cudaSuccess || cudaMalloc(&tb->dT2, tbytes) != cudaSuccess ||
        cudaMalloc(&tb->dMask, tbytes) != cudaSuccess || cudaMalloc(&tb->dDom, (size_t)tb->Wd * 8 + 8) != cudaSuccess ||
        cudaMalloc(&tb->dRem, (size_t)tb->Wd * 8 + 8) != cudaSuccess ||
        cudaMalloc(&tb->dRows, (size_t)tb->R * 4 + 4) != cudaSuccess || cudaMalloc(&tb->dSsup, (size_t)n + 1) != cudaSuccess ||
        cudaHostAlloc((void **)&tb->hT, tbytes, 0) != cudaSuccess ||
        cudaHostAlloc((void **)&tb->hMask, tbytes, 0) != cudaSuccess ||
        cudaHostAlloc((void **)&tb->hDom, (size_t)tb->Wd * 8 + 8, 0) != cudaSuccess ||
        cudaHostAlloc((void **)&tb->hRem, (size_t)tb->Wd * 8 + 8, 0) != cudaSuccess ||
        cudaHostAlloc((void **)&tb->hRows, (size_t)tb->R * 4 + 4, 0) != cudaSuccess ||
        cudaHostAlloc((void **)&tb->hSsup, (size_t)n + 1, 0) != cudaSuccess) {
      cudaGetLastError();
      return bail(fail(CT_ENOMEM, "placement %d: device / pinned allocation failed", placement));
    }
    memset(tb->hT, 0, tbytes);   // padding words stay 0 on the device copy
    for (int k = 0; k < 4; ++k) CUDA_TRY(cudaEventCreate(&tb->ev[k]));
    // device supports [R][Wp] from the host rows (one-time)
    CUDA_TRY(cudaMemset2DAsync(tb->dS, (size_t)tb->Wp * 8, 0, (size_t)tb->Wp * 8, (size_t)tb->R, tb->stream));
    if (tb->R)
      CUDA_TRY(cudaMemcpy2DAsync(tb->dS, (size_t)tb->Wp * 8, tb->S.data(), (size_t)tb->W * 8, (size_t)tb->W * 8,
                                 (size_t)tb->R, cudaMemcpyHostToDevice, tb->stream));
    std::vector<int32_t> meta(tb->rowVar.begin(), tb->rowVar.begin() + tb->R);
    meta.insert(meta.end(), tb->rowBase.begin(), tb->rowBase.end());
    meta.insert(meta.end(), tb->domOff.begin(), tb->domOff.end());
    CUDA_TRY(cudaMemcpyAsync(tb->dmeta, meta.data(), meta.size() * 4, cudaMemcpyHostToDevice, tb->stream));
    CUDA_TRY(cudaMemsetAsync(tb->dT, 0, tbytes, tb->stream));
    CUDA_TRY(cudaStreamSynchronize(tb->stream));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, tb->device);
    tb->upd_grid = (int)std::max<int64_t>(1, std::min<int64_t>((tb->W2 + kPlUpdTPB - 1) / kPlUpdTPB, 8 * sms));
    tb->filt_grid = (int)std::max<int64_t>(1, std::min<int64_t>(((int64_t)tb->R * 32 + kPlFiltTPB - 1) / kPlFiltTPB,
                                                                  16 * sms));
  }
  ct_host_state *root = new (std::nothrow) ct_host_state();
  if (!root) return bail(fail(CT_ENOMEM, "host allocation failed"));
  root->tb = tb;
  root->T.init(T0);
  root->dom = tb->full_dom;
  root->res.assign((size_t)std::max(tb->R, 1), 0);
  for (int r = 0; r < tb->R; ++r) {   // residue = the row's first support word
    const uint64_t *row = tb->S.data() + (size_t)r * tb->W;
    for (int64_t w = 0; w < tb->W; ++w)
      if (row[w]) {
        root->res[(size_t)r] = (int32_t)w;
        break;
      }
  }
  tb->live = 1;
  *out_table = tb;
  *out_root = root;
  // root propagation: remove the holes of init_dom, filter every variable
  std::vector<uint64_t> holes(tb->Wd, 0ull);
  if (init_dom)
    for (int k = 0; k < tb->Wd; ++k) holes[(size_t)k] = tb->full_dom[(size_t)k] & ~init_dom[k];
  const ct_status s = ct_host_propagate_impl(root, holes.data(), out_dom, nullptr, true);
  tb->st = ct_place_stats{};
  if (s < 0) {
    delete root;
    *out_root = nullptr;
    *out_table = nullptr;
    return bail(s);
  }
  return s;
}

}  // extern "C"

static ct_status ct_host_propagate_impl(ct_host_state *s, const uint64_t *removed, uint64_t *out_dom,
                                        uint64_t *out_pruned, bool root_mode) {
  using namespace ctpl;
  ct_host_table *tb = s->tb;
  if (s->dead) return fail(CT_ESTATE, "state is dead (returned CT_FAIL); restore it with ct_host_copy");
  const auto h0 = Clock::now();
  double host_ms = 0.0;
  const int n = tb->n;
  // Alg. 1 L1-3: Δ, dom after the removals, s_val, s_sup
  std::vector<uint64_t> delta((size_t)tb->Wd, 0ull);
  std::vector<int> cdelta(n, 0), csize(n, 0), sval;
  for (int x = 0; x < n; ++x) {
    for (int w = tb->domOff[x]; w < tb->domOff[x + 1]; ++w) {
      uint64_t rm = removed ? removed[w] : 0ull;
      if (w == tb->domOff[x + 1] - 1 && tb->d[x] % 64) rm &= (1ull << (tb->d[x] % 64)) - 1;
      const uint64_t dl = rm & s->dom[(size_t)w];
      delta[(size_t)w] = dl;
      s->dom[(size_t)w] &= ~dl;
      cdelta[x] += popc64(dl);
      csize[x] += popc64(s->dom[(size_t)w]);
    }
    if (cdelta[x]) sval.push_back(x);
  }
  std::vector<uint64_t> din(s->dom);
  tb->st.calls++;
  auto finish_fail = [&]() {
    s->dead = true;
    tb->st.host_ms += host_ms + ms_since(h0);
    return CT_FAIL;
  };
  for (int x = 0; x < n; ++x)
    if (csize[x] == 0) return finish_fail();   // a domain emptied: no valid tuple
  if (sval.empty() && !root_mode) {
    tb->st.noops++;
  } else if (tb->placement == CT_PLACE_HOST || tb->placement == CT_PLACE_F || sval.empty()) {
    host_update(tb, s, sval, delta, cdelta, csize);
    if (s->T.empty()) return finish_fail();
  }
  const bool work = !(sval.empty() && !root_mode);
  const bool dev_upd = work && (tb->placement == CT_PLACE_U || tb->placement == CT_PLACE_UF) && !sval.empty();
  const bool dev_filt = work && (tb->placement == CT_PLACE_F || tb->placement == CT_PLACE_UF);
  if (dev_upd || dev_filt) {
    DeviceGuard g(tb->device);
    // ---- host -> device: currTable (dense words), domains, s_val rows / s_sup
    int nrows = 0;
    memcpy(tb->hT, s->T.words.data(), (size_t)tb->W * 8);
    size_t h2d = (size_t)tb->W * 8;
    if (dev_upd) {
      nrows = build_rows(tb, s, sval);
      h2d += (size_t)nrows * 4;
    }
    if (dev_filt) {
      memcpy(tb->hDom, s->dom.data(), (size_t)tb->Wd * 8);
      for (int x = 0; x < n; ++x) tb->hSsup[x] = csize[x] > 1;
      h2d += (size_t)tb->Wd * 8 + (size_t)n;
    }
    host_ms += ms_since(h0);
    CUDA_TRY(cudaEventRecord(tb->ev[0], tb->stream));
    CUDA_TRY(cudaMemcpyAsync(tb->dT, tb->hT, (size_t)tb->W * 8, cudaMemcpyHostToDevice, tb->stream));
    if (dev_upd) CUDA_TRY(cudaMemcpyAsync(tb->dRows, tb->hRows, (size_t)nrows * 4, cudaMemcpyHostToDevice, tb->stream));
    if (dev_filt) {
      CUDA_TRY(cudaMemcpyAsync(tb->dDom, tb->hDom, (size_t)tb->Wd * 8, cudaMemcpyHostToDevice, tb->stream));
      CUDA_TRY(cudaMemcpyAsync(tb->dSsup, tb->hSsup, (size_t)n, cudaMemcpyHostToDevice, tb->stream));
    }
    CUDA_TRY(cudaEventRecord(tb->ev[1], tb->stream));
    // ---- kernels
    const ulonglong2 *Tf = reinterpret_cast<const ulonglong2 *>(tb->dT);
    if (dev_upd) {
      k_pl_update<<<tb->upd_grid, kPlUpdTPB, 0, tb->stream>>>(tb->dS, tb->Wp, (int)tb->W2, Tf, tb->dRows, nrows,
                                                              reinterpret_cast<ulonglong2 *>(tb->dMask),
                                                              dev_filt ? reinterpret_cast<ulonglong2 *>(tb->dT2) : nullptr);
      tb->st.kernel_launches++;
      if (dev_filt) Tf = reinterpret_cast<const ulonglong2 *>(tb->dT2);
    }
    if (dev_filt) {
      CUDA_TRY(cudaMemsetAsync(tb->dRem, 0, (size_t)tb->Wd * 8, tb->stream));
      const int32_t *rv = tb->dmeta, *rb = tb->dmeta + tb->R, *doff = rb + n + 1;
      k_pl_filter<<<tb->filt_grid, kPlFiltTPB, 0, tb->stream>>>(tb->dS, tb->Wp, (int)tb->W2, Tf, tb->dDom, tb->dSsup,
                                                                rv, rb, doff, tb->R,
                                                                reinterpret_cast<unsigned long long *>(tb->dRem));
      tb->st.kernel_launches++;
    }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaEventRecord(tb->ev[2], tb->stream));
    // ---- device -> host: mask (CT^u, CT^uf), removal bitmap (CT^f, CT^uf)
    size_t d2h = 0;
    if (dev_upd) {
      CUDA_TRY(cudaMemcpyAsync(tb->hMask, tb->dMask, (size_t)tb->W * 8, cudaMemcpyDeviceToHost, tb->stream));
      d2h += (size_t)tb->W * 8;
    }
    if (dev_filt) {
      CUDA_TRY(cudaMemcpyAsync(tb->hRem, tb->dRem, (size_t)tb->Wd * 8, cudaMemcpyDeviceToHost, tb->stream));
      d2h += (size_t)tb->Wd * 8;
    }
    CUDA_TRY(cudaEventRecord(tb->ev[3], tb->stream));
    CUDA_TRY(cudaEventSynchronize(tb->ev[3]));
    tb->st.h2d_ms += ev_ms(tb->ev[0], tb->ev[1]);
    tb->st.kernel_ms += ev_ms(tb->ev[1], tb->ev[2]);
    tb->st.d2h_ms += ev_ms(tb->ev[2], tb->ev[3]);
    tb->st.h2d_bytes += (int64_t)h2d;
    tb->st.d2h_bytes += (int64_t)d2h;
    const auto h1 = Clock::now();
    if (dev_upd) {   // "copied back to the host and combined bitwise with _currTable"
      SparseBitSet &T = s->T;
      for (int32_t i = 0; i <= T.limit; ++i) {
        const int32_t o = T.index[(size_t)i];
        T.mask[(size_t)o] = tb->hMask[o];
      }
      T.intersect_with_mask();
      if (T.empty()) {
        host_ms += ms_since(h1);
        s->dead = true;
        tb->st.host_ms += host_ms;
        return CT_FAIL;
      }
    }
    if (dev_filt) {
      for (int k = 0; k < tb->Wd; ++k) s->dom[(size_t)k] &= ~tb->hRem[k];
    } else {
      host_filter(tb, s, csize);
    }
    host_ms += ms_since(h1);
  } else {
    if (work) host_filter(tb, s, csize);
    host_ms += ms_since(h0);
  }
  tb->st.host_ms += host_ms;
  if (out_dom) memcpy(out_dom, s->dom.data(), (size_t)tb->Wd * 8);
  if (out_pruned)
    for (int k = 0; k < tb->Wd; ++k) out_pruned[k] = din[(size_t)k] & ~s->dom[(size_t)k];
  return CT_OK;
}

extern "C" {

ct_status ct_host_propagate(ct_host_state *s, const uint64_t *removed, uint64_t *out_dom, uint64_t *out_pruned) {
  if (!s) return fail(CT_EINVAL, "NULL state");
  return ct_host_propagate_impl(s, removed, out_dom, out_pruned, false);
}

ct_status ct_host_clone(const ct_host_state *src, ct_host_state **out) {
  if (!src || !out) return fail(CT_EINVAL, "NULL argument");
  ct_host_state *s = new (std::nothrow) ct_host_state(*src);
  if (!s) return fail(CT_ENOMEM, "host allocation failed");
  s->tb->live++;
  *out = s;
  return CT_OK;
}

ct_status ct_host_copy(ct_host_state *dst, const ct_host_state *src) {
  if (!dst || !src) return fail(CT_EINVAL, "NULL argument");
  if (dst->tb != src->tb) return fail(CT_ESTATE, "states belong to different tables");
  if (dst != src) {
    dst->T = src->T;
    dst->dom = src->dom;
    dst->res = src->res;
    dst->dead = src->dead;
  }
  return CT_OK;
}

ct_status ct_host_stats(ct_host_table *t, ct_place_stats *out, int32_t reset) {
  if (!t || !out) return fail(CT_EINVAL, "NULL argument");
  *out = t->st;
  if (reset) t->st = ct_place_stats{};
  return CT_OK;
}

int32_t ct_host_dom_words(const ct_host_table *t) { return t ? t->Wd : -1; }

void ct_host_state_destroy(ct_host_state *s) {
  if (!s) return;
  s->tb->live--;
  delete s;
}

void ct_host_table_destroy(ct_host_table *t) { ctpl::free_host_table(t); }

}  // extern "C"
