// Tensor-core throughput probe: one CTA per SM issues back-to-back tcgen05.mma
// of a given shape/operand source on resident (garbage) smem/TMEM data.
#include "common.cuh"
#include <cstdio>
using namespace lemo;

template <int N, bool TS, bool BMN>
__global__ void __launch_bounds__(128, 1) probe(int iters, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<512>(&slot);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, N, 0, BMN ? 1 : 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 65536);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t db = BMN ? umma_desc_mn_sw128(b + kk * 2048, 16384) : umma_desc_k_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32);
        if (TS) umma_bf16_ts(tmem, tmem + 256 + kk * 8, db, idesc, 1u);
        else umma_bf16_ss(tmem, umma_desc_k_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32), db, idesc, 1u);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int N, bool TS, bool BMN>
void run(const char* name) {
  unsigned long long* d; cudaMalloc(&d, 8);
  auto k = probe<N, TS, BMN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  int iters = 2000;
  k<<<148, 128, 140000>>>(iters, d);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<148, 128, 140000>>>(iters, d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  double flop = 2.0 * 128 * N * 16 * 8 * iters;
  printf("%-22s cycles/instr %.1f  flop/clk/SM %.0f  TFLOP/s %.0f  err=%s\n", name, (double)c / (8.0 * iters),
         flop / c, flop * 148 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main2();
int main() {
  main2();
  run<256, false, false>("SS N=256");
  run<128, false, false>("SS N=128");
  run<64, false, false>("SS N=64");
  run<32, false, false>("SS N=32");
  run<128, false, true>("SS N=128 B-MN");
  run<256, true, false>("TS N=256");
  run<128, true, false>("TS N=128");
  run<128, true, true>("TS N=128 B-MN");
  run<64, true, false>("TS N=64");
  run<32, true, false>("TS N=32");
  return 0;
}

// CTA-pair probe: leader issues M256 x N x K16 (cta_group::2) back to back.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe_pair(int iters, unsigned long long* cyc) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const bool leader = cluster_ctarank() == 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc_pair<512>(&slot);
  tc_fence_before(); cluster_sync(); tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0 && leader) {
    constexpr uint32_t idesc = umma_idesc_bf16(256, N, 0, 0);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 65536);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_bf16_ss_pair(tmem, umma_desc_k_sw128(a + (kk >> 2) * 16384 + (kk & 3) * 32),
                          umma_desc_k_sw128(b + (kk >> 2) * 16384 + (kk & 3) * 32), idesc, 1u);
    }
    umma_commit_pair(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
  }
  if (threadIdx.x == 0 && !leader) mbar_wait(&bar, 0);
  tc_fence_before(); cluster_sync(); tc_fence_after();
  if (warp == 0) tmem_dealloc_pair<512>(tmem);
}

template <int N>
void run_pair(const char* name) {
  unsigned long long* d; cudaMalloc(&d, 8);
  auto k = probe_pair<N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  int iters = 2000;
  k<<<148, 128, 140000>>>(iters, d);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<148, 128, 140000>>>(iters, d);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  double flop = 2.0 * 256 * N * 16 * 8 * iters;  // per pair
  printf("%-22s cycles/instr %.1f  flop/clk/pair %.0f  TFLOP/s %.0f  err=%s\n", name, (double)c / (8.0 * iters),
         flop / c, flop * 74 / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main2() {
  run_pair<256>("PAIR M256 N=256");
  run_pair<128>("PAIR M256 N=128");
  return 0;
}
