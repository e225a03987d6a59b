// TMEM hazard probe: does a tcgen05.mma that overwrites a TMEM region still
// being read as the A operand of the previous (TS) MMA drain the pipe?
// One CTA per SM issues the dK/dV backward pattern back to back on resident
// (garbage) data; cycles per M128·N128·K16 instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2501_09767_b200/csrc \
//        scripts/probes/hazard_probe.cu -o scripts/probes/hazard_probe
#include "common.cuh"
#include <cstdio>
using namespace lemo;

// mode 0: SS only, 4 distinct accumulators (no TMEM reuse)
// mode 1: bwd pattern  dV(A=S) S dP dK(A=P)  — A regions overwritten by the next S/dP
// mode 2: same shapes, A operands read from regions no MMA writes (dV/dK accumulators swapped)
// mode 3: SS → S then TS(A=S) → D, repeated (RAW + WAR on one region)
template <int MODE, int SPIN = 0>  // SPIN: extra warps polling an mbarrier during the run
__global__ void __launch_bounds__(512, 1) probe(int iters, unsigned long long* cyc, int fill) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar, bar2[4], spin;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&spin, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&bar2[i], 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&slot);
  if (fill) {  // random bf16 in [-2, 2) (non-trivial switching activity)
    uint32_t x = 0x9e3779b9u * (threadIdx.x + 1) + blockIdx.x;
    for (int i = threadIdx.x; i < 131072 / 4; i += 128) {
      x ^= x << 13; x ^= x >> 17; x ^= x << 5;
      const uint32_t lo = 0x3f80u | ((x & 0x7fu)) | ((x >> 7) & 1u) << 15;
      const uint32_t hi = 0x3f80u | ((x >> 8) & 0x7fu) | ((x >> 15) & 1u) << 15;
      reinterpret_cast<uint32_t*>(sm)[i] = lo | hi << 16;
    }
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot;
  if (fill) {  // TMEM A-operand regions: random packed bf16 too
    uint32_t v[32];
    uint32_t x = 0x85ebca6bu * (threadIdx.x + 7);
    for (int c = 0; c < 512; c += 32) {
      for (int j = 0; j < 32; ++j) { x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        v[j] = (0x3f80u | (x & 0x7fu)) | (0x3f80u | ((x >> 8) & 0x7fu) | ((x >> 16) & 1u) << 15) << 16; }
      tmem_st_32x32b_x32(slot + ((warp * 32) << 16) + c, v);
    }
    tmem_st_wait();
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tS = tmem, tP = tmem + 128, tV = tmem + 256, tK = tmem + 384;
  if (warp >= 4) {
    if (SPIN == 1) mbar_wait(&spin, 0);
    if (SPIN == 2) {  // polling with a nanosleep back-off
      while (!mbar_try_wait(&spin, 0)) __nanosleep(64);
    }
    if (SPIN == 3 || SPIN == 4) {  // element-wise warps streaming TMEM (ld, or ld + st) meanwhile
      const uint32_t row = slot + (((warp & 3) * 32) << 16) + ((warp >> 2) - 1) * 64;
      uint32_t v[32], acc = 0;
      while (!mbar_try_wait(&spin, 0)) {
        tmem_ld_32x32b_x32(row, v);
        uint32_t w[32];
        tmem_ld_32x32b_x32(row + 32, w);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) acc += v[j] ^ w[j];
        if (SPIN == 4) {
          uint32_t p16[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) p16[j] = v[j] + w[j];
          tmem_st_32x32b_x16(row, p16);
          tmem_st_wait();
        }
      }
      if (acc == 0x12345u) *cyc = acc;
    }
  }
  if (threadIdx.x == 0) {
    constexpr uint32_t id_k = umma_idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t id_mn = umma_idesc_bf16(128, 128, 0, 1);
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 65536);
    auto ss = [&](uint32_t d, int ra = 0, int rb = 0) {  // ra/rb: which 32 KB tile
      const uint32_t aa = a + ra * 32768, bb = b + rb * 32768;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_bf16_ss(d, umma_desc_k_sw128(aa + (kk >> 2) * 16384 + (kk & 3) * 32),
                     umma_desc_k_sw128(bb + (kk >> 2) * 16384 + (kk & 3) * 32), id_k, kk > 0);
    };
    auto ts = [&](uint32_t d, uint32_t at, int rb = 0) {
      const uint32_t bb = b + rb * 32768;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma_bf16_ts(d, at + kk * 8, umma_desc_mn_sw128(bb + kk * 2048, 16384), id_mn, 1u);
    };
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (MODE == 0) { ss(tS); ss(tP); ss(tV); ss(tK); }
      if (MODE == 1) { ts(tV, tS); ss(tS); ss(tP); ts(tK, tP); }
      if (MODE == 2) { ts(tV, tK); ss(tS); ss(tP); ts(tK, tV); }
      if (MODE == 3) { ss(tS); ts(tV, tS); ss(tP); ts(tK, tP); }
      if (MODE == 4) { ss(tS, 0, 0); ss(tP, 1, 1); ss(tV, 0, 1); ss(tK, 1, 0); }  // operands change
      if (MODE == 5) { ts(tV, tS, 0); ts(tK, tP, 1); ts(tV, tS, 1); ts(tK, tP, 0); }
      if (MODE == 7) {  // bwd pattern + one commit per MMA group (as the kernel does)
        ts(tV, tS, 0); umma_commit(&bar2[0]); ss(tS, 0, 1); umma_commit(&bar2[1]);
        ss(tP, 1, 0); umma_commit(&bar2[2]); ts(tK, tP, 1); umma_commit(&bar2[3]);
      }
      if (MODE == 8) {  // commits + the issuing thread waits for each group (no overlap)
        ts(tV, tS, 0); umma_commit(&bar2[0]); mbar_wait(&bar2[0], i & 1);
        ss(tS, 0, 1); umma_commit(&bar2[1]); mbar_wait(&bar2[1], i & 1);
        ss(tP, 1, 0); umma_commit(&bar2[2]); mbar_wait(&bar2[2], i & 1);
        ts(tK, tP, 1); umma_commit(&bar2[3]); mbar_wait(&bar2[3], i & 1);
      }
      if (MODE == 9 || MODE == 10) {  // the dK/dV kernel's smem map and operand forms
        const uint32_t base = smem_u32(sm);
        const uint32_t K = base, V = base + 32768, Q = base + 65536 + (i & 1) * 32768,
                       O = base + 131072 + (i & 1) * 32768, DS = base + 196608;
        auto kk_ss = [&](uint32_t d, uint32_t A, uint32_t B) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ss(d, umma_desc_k_sw128(A + (kk >> 2) * 16384 + (kk & 3) * 32),
                         umma_desc_k_sw128(B + (kk >> 2) * 16384 + (kk & 3) * 32), id_k, kk > 0);
        };
        auto tk = [&](uint32_t d, uint32_t at, uint32_t B) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ts(d, at + (kk >> 2) * 64 + (kk & 3) * 8,
                         umma_desc_mn_sw128(B + kk * 2048, 16384), id_mn, 1u);
        };
        tk(tV, tS, O);
        kk_ss(tS, K, Q);
        kk_ss(tP, V, O);
        if (MODE == 9) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            umma_bf16_ss(tK, umma_desc_k_sw128(DS + (kk >> 2) * 16384 + (kk & 3) * 32),
                         umma_desc_mn_sw128(Q + kk * 2048, 16384), id_mn, 1u);
        } else {
          tk(tK, tP, Q);
        }
      }
      if (MODE == 6) { ts(tV, tS, 0); ss(tS, 0, 1); ss(tP, 1, 0); ts(tK, tP, 1); }  // bwd, rotating
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cyc = t1 - t0;
    mbar_arrive(&spin);
  }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int MODE, int SPIN = 0>
void run(const char* name, int fill, int iters = 1000, int warps = 4) {
  unsigned long long* d; cudaMalloc(&d, 8);
  auto k = probe<MODE, SPIN>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 231424);
  k<<<148, warps * 32, 231424>>>(iters, d, fill);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, warps * 32, 231424>>>(iters, d, fill);
  cudaEventRecord(e1);
  cudaDeviceSynchronize();
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  if (iters > 1000)
    printf("  [%d iters: %.1f ms, SM clock %.0f MHz, %.0f TFLOP/s]\n", iters, ms, c / (ms * 1e3),
           2.0 * 128 * 128 * 16 * 32.0 * iters * 148 / (ms * 1e-3) / 1e12);
  printf("%s %-44s cycles/instr %.1f (ideal 64)  err=%s\n", fill ? "rand" : "zero", name, (double)c / (32.0 * iters),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<6, 3>("bwd pattern + 8 warps streaming tcgen05.ld", 1, 1000, 12);
  run<6, 4>("bwd pattern + 8 warps tcgen05.ld + st", 1, 1000, 12);
  run<0, 3>("SS x4 + 8 warps streaming tcgen05.ld", 1, 1000, 12);
  run<9>("kernel smem map, dK SS (A=dS smem)", 1);
  run<10>("kernel smem map, dK TS (A=dS TMEM)", 1);
  for (int fill = 0; fill < 2; ++fill) {
    run<0>("SS x4, distinct accumulators", fill);
    run<1>("dV(A=S) S dP dK(A=P): A overwritten next", fill);
    run<2>("dV(A=dK) S dP dK(A=dV): A never overwritten", fill);
    run<3>("S dV(A=S) dP dK(A=P): RAW+WAR", fill);
    run<4>("SS x4, operand tiles change every MMA", fill);
    run<5>("TS x4, B tile changes every MMA", fill);
    run<6>("bwd pattern, operand tiles change", fill);
    run<7>("bwd pattern + commit per group", fill);
    run<8>("commit + wait per group (latency)", fill);
  }
  return 0;
}
