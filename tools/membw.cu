// membw.cu -- read-bandwidth ceilings for the update phase's access pattern.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membw tools/membw.cu && ./membw
// (a) plain streaming read of 1 GB with 16-byte loads (grid-stride, unroll 8);
// (b) the update pattern: P 16-byte columns x R rows at stride Wp words, one
//     thread per column OR-ing its rows (unroll U), grid = one thread per column.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ ulonglong2 ld2(const uint64_t *p) {
  ulonglong2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(p));
  return v;
}

__global__ void k_stream(const ulonglong2 *a, size_t n, unsigned long long *sink) {
  uint64_t acc = 0;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i + 7 * st < n; i += 8 * st) {
    ulonglong2 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ld2((const uint64_t *)(a + i + u * st));
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y;
  }
  for (; i < n; i += st) acc ^= a[i].x;
  if (acc == 0x1234567) atomicAdd(sink, 1ull);
}

template <int U>
__global__ void k_cols(const uint64_t *S, int64_t Wp, int P, int R, unsigned long long *sink) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const uint64_t *col = S + 2 * (int64_t)p;
  uint64_t ax = 0, ay = 0;
  for (int r = 0; r < R; r += U) {
    ulonglong2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld2(col + (int64_t)(r + u) * Wp);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      ax |= v[u].x;
      ay |= v[u].y;
    }
  }
  if ((ax ^ ay) == 0x1234567) atomicAdd(sink, 1ull);
}

int main() {
  const size_t bytes = 1ull << 30;
  uint64_t *buf;
  unsigned long long *sink;
  cudaMalloc(&buf, bytes + (64 << 20));
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bpsm : {2, 4, 8}) {
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(e0);
      k_stream<<<sms * bpsm, 256>>>((const ulonglong2 *)buf, bytes / 16, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("stream read 1 GiB, %d blocks/SM x 256: %.1f us  %.0f GB/s\n", bpsm, best * 1e3, bytes / (best * 1e-3) / 1e9);
  }
  // update pattern: C3 shape, 800 rows x 156256 words; read 400 rows
  const int64_t Wp = 156256;
  const int P = 78125, R = 400;
  for (int tpb : {128, 256}) {
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(e0);
      k_cols<8><<<(P + tpb - 1) / tpb, tpb>>>(buf, Wp, P, R, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double b = (double)P * R * 16;
    printf("cols U=8 tpb=%d: %.1f us  %.0f GB/s\n", tpb, best * 1e3, b / (best * 1e-3) / 1e9);
  }
  for (int tpb : {128, 256}) {
    float best = 1e9;
    for (int it = 0; it < 10; ++it) {
      cudaEventRecord(e0);
      k_cols<16><<<(P + tpb - 1) / tpb, tpb>>>(buf, Wp, P, R, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double b = (double)P * R * 16;
    printf("cols U=16 tpb=%d: %.1f us  %.0f GB/s\n", tpb, best * 1e3, b / (best * 1e-3) / 1e9);
  }
  return 0;
}
