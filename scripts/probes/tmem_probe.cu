// TMEM read/write throughput probe: W warps per CTA (one CTA per SM) issue
// back-to-back tcgen05.ld / tcgen05.st 32x32b.x32 on their lane quarter.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2501_09767_b200/csrc \
//        scripts/probes/tmem_probe.cu -o scripts/probes/tmem_probe
#include "common.cuh"
#include <cstdio>
using namespace lemo;

template <int MODE>  // 0 = ld x32 (one wait per 2 loads), 1 = st x32, 2 = ld x16 pairs
__global__ void __launch_bounds__(512, 1) probe(int iters, unsigned long long* cyc, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = slot + (((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  float acc = 0.f;
  uint32_t v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = threadIdx.x * j;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (MODE == 0) {
      uint32_t a[32], b[32];
      tmem_ld_32x32b_x32(t, a);
      tmem_ld_32x32b_x32(t + 32, b);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) acc += __uint_as_float(a[j] ^ b[j]);
    } else {
      tmem_st_32x32b_x32(t, v);
      tmem_st_32x32b_x32(t + 32, v);
      tmem_st_wait();
      v[0] += 1;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  if (acc == 1.2345f) *sink = acc;
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(slot);
}

template <int MODE>
void run(const char* name, int warps) {
  unsigned long long* d; cudaMalloc(&d, 8);
  float* s; cudaMalloc(&s, 4);
  int iters = 2000;
  probe<MODE><<<148, warps * 32>>>(iters, d, s);
  probe<MODE><<<148, warps * 32>>>(iters, d, s);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = 2.0 * 4096 * warps * iters;  // two x32 ops of 4 KB per warp per iter
  printf("%-10s warps=%2d  %.1f B/clk/SM  err=%s\n", name, warps, bytes / c,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  for (int w : {4, 8, 16}) run<0>("ld", w);
  for (int w : {4, 8, 16}) run<1>("st", w);
  return 0;
}
