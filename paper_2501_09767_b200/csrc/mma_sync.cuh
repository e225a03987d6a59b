// Warp-level bf16 tensor-core helpers (mma.sync m16n8k16, ldmatrix, cp.async)
// and a 64-row swizzled shared-memory tile, shared by the attention and the
// exact block-score kernels.
#pragma once

#include "common.cuh"

namespace lemo {
namespace fa {

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Swizzled tile of 64 rows x D bf16 (row = D*2 bytes, 16-B chunks XOR row%8).
template <int D>
struct Tile {
  static constexpr int kRowBytes = D * 2;
  static constexpr int kChunks = D / 8;
  static constexpr int kBytes = 64 * kRowBytes;
  __device__ static __forceinline__ uint32_t off(int r, int col) {  // col multiple of 8
    return r * kRowBytes + (((col >> 3) ^ (r & 7)) << 4);
  }
  // rows [r0, r0+64) of a row-major [n, ld] matrix starting at column c0
  __device__ static __forceinline__ void load(uint32_t base, const __nv_bfloat16* g, int ld, int r0,
                                              int c0, int n, int tid, int nthreads) {
    for (int i = tid; i < 64 * kChunks; i += nthreads) {
      const int r = i / kChunks, c = i - r * kChunks;
      const int gr = r0 + r;
      const bool ok = gr < n;
      const __nv_bfloat16* src = g + (size_t)(ok ? gr : 0) * ld + c0 + c * 8;
      cp_async16(base + off(r, c * 8), src, ok);
    }
  }
};


}  // namespace fa
}  // namespace lemo
