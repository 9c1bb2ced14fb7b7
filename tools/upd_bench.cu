// upd_bench.cu -- microbenchmark of update-loop engines on a C3-shaped problem
// (800 support rows x 156256 words = 1.0 GB, 400-row update list in 8 groups of
// 50, 78125 active 16-byte blocks).  Measures only the streaming AND/OR pass
// (no compaction) so engine choices can be compared in isolation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o upd_bench tools/upd_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

constexpr uint32_t kEnd = 1u << 30, kInv = 1u << 31, kRow = 0x3FFFFFFF;

__device__ __forceinline__ ulonglong2 ld2(const uint64_t *p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

// V1/V2: register batches of U rows, one thread per 16-byte block
template <int U>
__global__ void k_reg(const uint64_t *__restrict__ S, int64_t Wp, const uint32_t *__restrict__ ul, int nrows,
                      ulonglong2 *__restrict__ T2, int L) {
  __shared__ uint32_t s_ul[1024];
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) s_ul[i] = ul[i];
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  const uint64_t *col = S + 2 * (int64_t)k;
  const ulonglong2 tw = T2[k];
  uint64_t mx = ~0ull, my = ~0ull, ax = 0, ay = 0;
  for (int p = 0; p < nrows; p += U) {
    if (((tw.x & mx) | (tw.y & my)) == 0) break;
    ulonglong2 v[U];
#pragma unroll
    for (int q = 0; q < U; ++q)
      v[q] = (p + q < nrows) ? ld2(col + (int64_t)(s_ul[p + q] & kRow) * Wp) : make_ulonglong2(0, 0);
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (p + q < nrows) {
        const uint32_t e = s_ul[p + q];
        ax |= v[q].x; ay |= v[q].y;
        if (e & kEnd) {
          if (e & kInv) { mx &= ~ax; my &= ~ay; } else { mx &= ax; my &= ay; }
          ax = ay = 0;
        }
      }
    }
  }
  T2[k] = make_ulonglong2(tw.x & mx, tw.y & my);
}

// V3: register double buffer (U rows consumed while the next U are in flight)
template <int U>
__global__ void k_reg2(const uint64_t *__restrict__ S, int64_t Wp, const uint32_t *__restrict__ ul, int nrows,
                       ulonglong2 *__restrict__ T2, int L) {
  __shared__ uint32_t s_ul[1024 + 2 * U];
  for (int i = threadIdx.x; i < nrows + 2 * U; i += blockDim.x) s_ul[i] = i < nrows ? ul[i] : 0u;
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  const uint64_t *col = S + 2 * (int64_t)k;
  const ulonglong2 tw = T2[k];
  uint64_t mx = ~0ull, my = ~0ull, ax = 0, ay = 0;
  ulonglong2 a[U], b[U];
#pragma unroll
  for (int q = 0; q < U; ++q) a[q] = (q < nrows) ? ld2(col + (int64_t)(s_ul[q] & kRow) * Wp) : make_ulonglong2(0, 0);
  for (int p = 0; p < nrows; p += 2 * U) {
#pragma unroll
    for (int q = 0; q < U; ++q)
      b[q] = (p + U + q < nrows) ? ld2(col + (int64_t)(s_ul[p + U + q] & kRow) * Wp) : make_ulonglong2(0, 0);
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (p + q < nrows) {
        const uint32_t e = s_ul[p + q];
        ax |= a[q].x; ay |= a[q].y;
        if (e & kEnd) {
          if (e & kInv) { mx &= ~ax; my &= ~ay; } else { mx &= ax; my &= ay; }
          ax = ay = 0;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < U; ++q)
      a[q] = (p + 2 * U + q < nrows) ? ld2(col + (int64_t)(s_ul[p + 2 * U + q] & kRow) * Wp) : make_ulonglong2(0, 0);
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (p + U + q < nrows) {
        const uint32_t e = s_ul[p + U + q];
        ax |= b[q].x; ay |= b[q].y;
        if (e & kEnd) {
          if (e & kInv) { mx &= ~ax; my &= ~ay; } else { mx &= ax; my &= ay; }
          ax = ay = 0;
        }
      }
    }
    if (((tw.x & mx) | (tw.y & my)) == 0) break;
  }
  T2[k] = make_ulonglong2(tw.x & mx, tw.y & my);
}

// V4: cp.async ring of depth D
template <int D>
__global__ void k_ring(const uint64_t *__restrict__ S, int64_t Wp, const uint32_t *__restrict__ ul, int nrows,
                       ulonglong2 *__restrict__ T2, int L) {
  extern __shared__ __align__(16) ulonglong2 ring[];
  __shared__ uint32_t s_ul[1024];
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) s_ul[i] = ul[i];
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= L) return;
  const uint64_t *col = S + 2 * (int64_t)k;
  ulonglong2 *slot = ring + threadIdx.x;
  const int nt = blockDim.x;
#pragma unroll
  for (int q = 0; q < D - 1; ++q) {
    if (q < nrows) {
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(slot + q * nt);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(col + (int64_t)(s_ul[q] & kRow) * Wp) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  const ulonglong2 tw = T2[k];
  uint64_t mx = ~0ull, my = ~0ull, ax = 0, ay = 0;
  for (int r = 0; r < nrows; ++r) {
    const int q = r + D - 1;
    if (q < nrows) {
      const uint32_t d = (uint32_t)__cvta_generic_to_shared(slot + (q % D) * nt);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(col + (int64_t)(s_ul[q] & kRow) * Wp) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
    const ulonglong2 v = slot[(r % D) * nt];
    const uint32_t e = s_ul[r];
    ax |= v.x; ay |= v.y;
    if (e & kEnd) {
      if (e & kInv) { mx &= ~ax; my &= ~ay; } else { mx &= ax; my &= ay; }
      ax = ay = 0;
      if (((tw.x & mx) | (tw.y & my)) == 0) break;
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  T2[k] = make_ulonglong2(tw.x & mx, tw.y & my);
}

// V5: 8-byte granularity, one thread per word, register batches of U
template <int U>
__global__ void k_word(const uint64_t *__restrict__ S, int64_t Wp, const uint32_t *__restrict__ ul, int nrows,
                       uint64_t *__restrict__ T, int W) {
  __shared__ uint32_t s_ul[1024];
  for (int i = threadIdx.x; i < nrows; i += blockDim.x) s_ul[i] = ul[i];
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= W) return;
  const uint64_t *col = S + k;
  const uint64_t tw = T[k];
  uint64_t m = ~0ull, a = 0;
  for (int p = 0; p < nrows; p += U) {
    if ((tw & m) == 0) break;
    uint64_t v[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      uint64_t x = 0;
      if (p + q < nrows) asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(x) : "l"(col + (int64_t)(s_ul[p + q] & kRow) * Wp));
      v[q] = x;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      if (p + q < nrows) {
        const uint32_t e = s_ul[p + q];
        a |= v[q];
        if (e & kEnd) { m &= (e & kInv) ? ~a : a; a = 0; }
      }
    }
  }
  T[k] = tw & m;
}

// TLB probe: warp i reads 4 KB starting at S + i * stride_words (one 16-byte load
// per lane per round, 8 rounds in flight), like the filter's first probe round.
__global__ void k_tlb(const uint64_t *__restrict__ S, int64_t stride_words, int nwarps, unsigned long long *out) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nwarps) return;
  const uint64_t *base = S + (int64_t)w * stride_words;
  uint64_t acc = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const ulonglong2 v = ld2(base + 2 * (q * 32 + lane));
    acc ^= v.x ^ v.y;
  }
  if (acc == 0x12345) *out = acc;
}

// dependent-load latency: lane 0 chases n pointers through buf (index in the
// low word of each 16-byte cell); reports ns per hop from %globaltimer
__global__ void k_lat(const uint64_t *__restrict__ buf, int n, unsigned long long *out, int use_nc) {
  if (threadIdx.x != 0) return;
  uint64_t i = 0;
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int k = 0; k < n; ++k) {
    if (use_nc) i = ld2(buf + 2 * i).x;
    else i = __ldcg(reinterpret_cast<const ulonglong2 *>(buf) + i).x;
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  out[0] = (t1 - t0) / n;
  out[1] = i;
}

// copy kernel for a bandwidth reference
__global__ void k_copy(const ulonglong2 *__restrict__ a, ulonglong2 *__restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void k_read(const ulonglong2 *__restrict__ a, int64_t n, unsigned long long *out) {
  uint64_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    ulonglong2 v = ld2(reinterpret_cast<const uint64_t *>(a + i));
    acc ^= v.x ^ v.y;
  }
  if (acc == 0x12345) *out = acc;
}

int main() {
  const int R = 800, nrows = 400, W = 156250;
  const int64_t Wp = 156256;
  const int L = W / 2 + (W & 1);
  uint64_t *S, *T, *T0;
  uint32_t *ul;
  unsigned long long *dummy;
  CK(cudaMalloc(&S, (size_t)R * Wp * 8));
  CK(cudaMalloc(&T, Wp * 8));
  CK(cudaMalloc(&T0, Wp * 8));
  CK(cudaMalloc(&ul, 1024 * 4));
  CK(cudaMalloc(&dummy, 8));
  // supports of a C3-shaped i.i.d. table: t = 1e7 tuples, n = 8, d = 100, row
  // (i, v) bit j = [tau_j[i] = v]; update list = a random 50 of the 100 values
  // of every variable, ascending (dom-branch groups of 50, as ingest emits them)
  {
    const int64_t t = 10000000;
    std::vector<uint64_t> h((size_t)R * Wp, 0ull);
    uint64_t x = 0x9E3779B97F4A7C15ull;
    auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; };
    for (int64_t j = 0; j < t; ++j)
      for (int i = 0; i < 8; ++i) {
        const int v = (int)(((unsigned __int128)rnd() * 100) >> 64);
        h[(size_t)(i * 100 + v) * Wp + j / 64] |= 1ull << (j % 64);
      }
    CK(cudaMemcpy(S, h.data(), h.size() * 8, cudaMemcpyHostToDevice));
    std::vector<uint64_t> tv(Wp, 0ull);
    for (int64_t w = 0; w < W; ++w) tv[w] = (w < t / 64) ? ~0ull : ((1ull << (t % 64)) - 1);
    CK(cudaMemcpy(T0, tv.data(), Wp * 8, cudaMemcpyHostToDevice));
    std::vector<uint32_t> u;
    for (int g = 0; g < 8; ++g) {
      int pick[100];
      for (int a = 0; a < 100; ++a) pick[a] = a < 50;
      for (int a = 99; a > 0; --a) { const int b = (int)(rnd() % (a + 1)); std::swap(pick[a], pick[b]); }
      int cnt = 0;
      for (int a = 0; a < 100; ++a)
        if (pick[a]) {
          uint32_t e = (uint32_t)(g * 100 + a);
          if (++cnt == 50) e |= kEnd;
          u.push_back(e);
        }
    }
    CK(cudaMemcpy(ul, u.data(), nrows * 4, cudaMemcpyHostToDevice));
  }
  const double bytes = (double)L * 16 * (nrows + 2);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char *name, auto launch, int reps = 20) {
    for (int i = 0; i < 3; ++i) { cudaMemcpy(T, T0, Wp * 8, cudaMemcpyDeviceToDevice); launch(); }
    float tot = 0;
    for (int i = 0; i < reps; ++i) {
      cudaMemcpy(T, T0, Wp * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      tot += ms;
    }
    const double us = tot / reps * 1e3;
    cudaError_t err = cudaGetLastError();
    printf("%-28s %8.1f us  %7.0f GB/s  %s\n", name, us, bytes / (us * 1e-6) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
  ulonglong2 *T2 = reinterpret_cast<ulonglong2 *>(T);
  // occupancy / launch-mode probes of the best engine (dynamic smem pads the CTA)
  cudaFuncSetAttribute(k_reg<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int pad : {0, 20, 30, 40, 44, 56}) {
    char nm[64];
    snprintf(nm, sizeof nm, "reg U=16 tpb=128 pad=%dK", pad);
    run(nm, [&] { k_reg<16><<<(L + 127) / 128, 128, pad * 1024>>>(S, Wp, ul, nrows, T2, L); });
  }
  {
    void *args[] = {(void *)&S, (void *)&Wp, (void *)&ul, (void *)&nrows, (void *)&T2, (void *)&L};
    for (int pad : {0, 40}) {
      char nm[64];
      snprintf(nm, sizeof nm, "reg U=16 coop pad=%dK", pad);
      run(nm, [&] { cudaLaunchCooperativeKernel((void *)k_reg<16>, (L + 127) / 128, 128, args, pad * 1024, 0); });
    }
  }
  run("reg U=8 tpb=256", [&] { k_reg<8><<<(L + 255) / 256, 256>>>(S, Wp, ul, nrows, T2, L); });
  run("reg U=8 tpb=128", [&] { k_reg<8><<<(L + 127) / 128, 128>>>(S, Wp, ul, nrows, T2, L); });
  run("reg U=16 tpb=128", [&] { k_reg<16><<<(L + 127) / 128, 128>>>(S, Wp, ul, nrows, T2, L); });
  run("reg U=16 tpb=256", [&] { k_reg<16><<<(L + 255) / 256, 256>>>(S, Wp, ul, nrows, T2, L); });
  run("reg U=32 tpb=128", [&] { k_reg<32><<<(L + 127) / 128, 128>>>(S, Wp, ul, nrows, T2, L); });
  run("reg2 U=8 tpb=128", [&] { k_reg2<8><<<(L + 127) / 128, 128>>>(S, Wp, ul, nrows, T2, L); });
  run("reg2 U=8 tpb=256", [&] { k_reg2<8><<<(L + 255) / 256, 256>>>(S, Wp, ul, nrows, T2, L); });
  run("reg2 U=16 tpb=128", [&] { k_reg2<16><<<(L + 127) / 128, 128>>>(S, Wp, ul, nrows, T2, L); });
  cudaFuncSetAttribute(k_ring<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 256 * 16);
  cudaFuncSetAttribute(k_ring<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 256 * 16);
  cudaFuncSetAttribute(k_ring<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32 * 128 * 16);
  run("ring D=8 tpb=256", [&] { k_ring<8><<<(L + 255) / 256, 256, 8 * 256 * 16>>>(S, Wp, ul, nrows, T2, L); });
  run("ring D=16 tpb=256", [&] { k_ring<16><<<(L + 255) / 256, 256, 16 * 256 * 16>>>(S, Wp, ul, nrows, T2, L); });
  run("ring D=16 tpb=128", [&] { k_ring<16><<<(L + 127) / 128, 128, 16 * 128 * 16>>>(S, Wp, ul, nrows, T2, L); });
  run("ring D=32 tpb=128", [&] { k_ring<32><<<(L + 127) / 128, 128, 32 * 128 * 16>>>(S, Wp, ul, nrows, T2, L); });
  run("word U=8 tpb=256", [&] { k_word<8><<<(W + 255) / 256, 256>>>(S, Wp, ul, nrows, T, W); });
  run("word U=16 tpb=256", [&] { k_word<16><<<(W + 255) / 256, 256>>>(S, Wp, ul, nrows, T, W); });
  run("word U=16 tpb=128", [&] { k_word<16><<<(W + 127) / 128, 128>>>(S, Wp, ul, nrows, T, W); });
  run("word U=32 tpb=128", [&] { k_word<32><<<(W + 127) / 128, 128>>>(S, Wp, ul, nrows, T, W); });
  // TLB test: 400 warps x 4 KB at row starts (1.25 MB apart) vs packed (4 KB apart),
  // each right after a full 1-GB update pass (which leaves other pages in the TLB)
  for (int rep = 0; rep < 3; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      const int64_t stride = mode == 0 ? Wp : (mode == 1 ? 512 : Wp * 2);
      const int nw = mode == 2 ? 400 : 400;
      cudaMemcpy(T, T0, Wp * 8, cudaMemcpyDeviceToDevice);
      k_reg<16><<<(L + 127) / 128, 128>>>(S, Wp, ul, nrows, T2, L);
      cudaEventRecord(e0);
      k_tlb<<<(nw * 32 + 127) / 128, 128>>>(S + 2 * 1000, stride, mode == 2 ? 400 : nw, dummy);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("tlb probe %-22s %8.2f us\n", mode == 0 ? "rows 1.25 MB apart" : (mode == 1 ? "rows 4 KB apart" : "rows 2.5 MB apart"), ms * 1e3);
    }
  // pointer-chase latency through a random cycle over 1 GB (DRAM) and 1 MB (L2)
  {
    unsigned long long *dout;
    CK(cudaMalloc(&dout, 16));
    uint64_t *buf;
    const int64_t cells_big = (int64_t)R * Wp / 2, cells_small = 65536;
    CK(cudaMalloc(&buf, cells_big * 16));
    for (int which = 0; which < 2; ++which) {
      const int64_t cells = which ? cells_small : cells_big;
      const int hops = 200;
      std::vector<uint64_t> h(2 * hops, 0);
      // chain of `hops` random cells: cell c_k holds c_{k+1}
      std::vector<int64_t> c(hops + 1);
      uint64_t x = 12345;
      for (int k = 0; k <= hops; ++k) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; c[k] = k == 0 ? 0 : (int64_t)(x % cells); }
      for (int k = 0; k < hops; ++k) {
        uint64_t v[2] = {(uint64_t)c[k + 1], 0};
        CK(cudaMemcpy(buf + 2 * c[k], v, 16, cudaMemcpyHostToDevice));
      }
      for (int nc = 0; nc < 2; ++nc) {
        k_lat<<<1, 32>>>(buf, hops, dout, nc);   // warm TLB / L2
        k_lat<<<1, 32>>>(buf, hops, dout, nc);
        unsigned long long r[2];
        CK(cudaMemcpy(r, dout, 16, cudaMemcpyDeviceToHost));
        printf("latency %s %s: %llu ns per dependent load\n", which ? "L2 (1 MB)" : "1 GB", nc ? "ld.nc" : "ld.cg", r[0]);
      }
    }
    // the same right after a streaming pass (1 GB region, cold chain)
    cudaMemcpy(T, T0, Wp * 8, cudaMemcpyDeviceToDevice);
    k_reg<16><<<(L + 127) / 128, 128>>>(S, Wp, ul, nrows, T2, L);
    cudaDeviceSynchronize();
    cudaFree(buf);
  }
  // references: plain read and copy of the same 1 GB
  const int64_t n16 = (int64_t)R * Wp / 2;
  {
    const double b = (double)n16 * 16;
    for (int i = 0; i < 2; ++i) k_read<<<148 * 8, 256>>>(reinterpret_cast<ulonglong2 *>(S), n16, dummy);
    cudaEventRecord(e0);
    for (int i = 0; i < 10; ++i) k_read<<<148 * 8, 256>>>(reinterpret_cast<ulonglong2 *>(S), n16, dummy);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.1f us  %7.0f GB/s\n", "read 1 GB (grid-stride)", ms * 100, b / (ms / 10 * 1e-3) / 1e9);
  }
  return 0;
}
