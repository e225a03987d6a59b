// Per-SM issue throughput of the element-wise ops the attention kernels use:
// ex2.approx (MUFU), cvt.rn.bf16x2.f32 (F2FP), fma.rn.f32, fma.rn.f32x2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/probes/alu_probe.cu \
//        -o scripts/probes/alu_probe
#include <cstdio>
#include <cstdint>

template <int OP>
__global__ void __launch_bounds__(256, 1) probe(int iters, float* out, unsigned long long* cyc) {
  float x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3f + j * 1e-4f;
  uint32_t u = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[j]));
      if (OP == 1) {
        uint32_t r;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(x[j]), "f"(x[(j + 1) & 7]));
        u += r;
      }
      if (OP == 2) asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(x[j]));
      if (OP == 3) {
        uint64_t v = (uint64_t)__float_as_uint(x[j]) | ((uint64_t)__float_as_uint(x[(j + 1) & 7]) << 32);
        asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(v));
        x[j] = __uint_as_float((uint32_t)v);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + u;
}

template <int OP>
void run(const char* name) {
  float* o; cudaMalloc(&o, 148 * 256 * 4);
  unsigned long long* d; cudaMalloc(&d, 8);
  int iters = 4096;
  probe<OP><<<148, 256>>>(iters, o, d);
  probe<OP><<<148, 256>>>(iters, o, d);
  cudaDeviceSynchronize();
  unsigned long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("%-22s %.2f thread-ops/clk/SM  err=%s\n", name, 256.0 * 8 * iters / c,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  run<0>("ex2.approx.f32");
  run<1>("cvt.rn.bf16x2.f32");
  run<2>("fma.rn.f32");
  run<3>("fma.rn.f32x2");
  return 0;
}
