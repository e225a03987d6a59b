// Exact attention block informativeness (sparsity.py:173-219, Eq. 2):
//   agg[i, j] = Σ_h max(q_i^h · k_j^h, 0) / H      (no 1/√d)
//   masked to 0 unless j <= i, i < n_valid, j < n_valid
//   score(m, n) = max over the b x b tile (query block m, key block n <= m)
// One CTA per (64-query, 64-key) tile pair on or below the diagonal; the
// head loop streams Q_h / K_h tiles (cp.async double buffer) and keeps the
// head-summed positive scores in registers; the epilogue reduces each
// 16x16 sub-tile to its max.  The s x s score matrix is never materialised.
#include "lemo_internal.h"
#include "mma_sync.cuh"

namespace lemo {
namespace fa {

template <int D>
__global__ void __launch_bounds__(128) exact_block_scores_kernel(
    const __nv_bfloat16* __restrict__ q, const __nv_bfloat16* __restrict__ k, int s, int h,
    int kv, int n_valid, float* __restrict__ out, int ldo) {
  using T = Tile<D>;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ[2] = {smem_u32(smem), smem_u32(smem) + T::kBytes};
  const uint32_t sK[2] = {smem_u32(smem) + 2 * T::kBytes, smem_u32(smem) + 3 * T::kBytes};
  // tile pair from the linear lower-triangle index
  const int t = blockIdx.x;
  int qt = (int)((sqrtf(8.f * t + 1.f) - 1.f) * 0.5f);
  while ((qt + 1) * (qt + 2) / 2 <= t) ++qt;
  while (qt * (qt + 1) / 2 > t) --qt;
  const int kt = t - qt * (qt + 1) / 2;
  const int q0 = qt * 64, k0 = kt * 64;
  const int H = h / D;
  const int group = h / kv;  // query heads per key head (grouped-query attention)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;

  float agg[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) agg[i][0] = agg[i][1] = agg[i][2] = agg[i][3] = 0.f;

  T::load(sQ[0], q, h, q0, 0, s, tid, 128);
  T::load(sK[0], k, kv, k0, 0, s, tid, 128);
  cp_async_commit();
  for (int hd = 0; hd < H; ++hd) {
    const int buf = hd & 1;
    if (hd + 1 < H) {
      T::load(sQ[buf ^ 1], q, h, q0, (hd + 1) * D, s, tid, 128);
      T::load(sK[buf ^ 1], k, kv, k0, ((hd + 1) / group) * D, s, tid, 128);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    float sc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) sc[i][0] = sc[i][1] = sc[i][2] = sc[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < D / 16; ++kk) {
      uint32_t a[4];
      const int r = warp * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
      ldsm_x4(sQ[buf] + T::off(r, kk * 16 + (lane >> 4) * 8), a);
#pragma unroll
      for (int nt2 = 0; nt2 < 4; ++nt2) {
        uint32_t b[4];
        const int key = nt2 * 16 + (lane & 7) + (lane >> 4) * 8;
        ldsm_x4(sK[buf] + T::off(key, kk * 16 + ((lane >> 3) & 1) * 8), b);
        mma16816(sc[2 * nt2], a, b[0], b[1]);
        mma16816(sc[2 * nt2 + 1], a, b[2], b[3]);
      }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int e = 0; e < 4; ++e) agg[i][e] += fmaxf(sc[i][e], 0.f);
    __syncthreads();
  }
  const float invH = 1.f / (float)H;
  // masked 16x16 tile maxima: warp w covers query sub-block (q0/16 + w);
  // n-tiles 2c, 2c+1 form key sub-block (k0/16 + c)
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    float mx = 0.f;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int nt = 2 * c + half;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int row = q0 + warp * 16 + g + (e >= 2 ? 8 : 0);
        const int col = k0 + nt * 8 + 2 * t4 + (e & 1);
        const bool keep = col <= row && row < n_valid && col < n_valid;
        const float v = keep ? agg[nt][e] * invH : 0.f;
        mx = fmaxf(mx, v);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int mb = (q0 >> 4) + warp, nb_ = (k0 >> 4) + c;
    const int nb_total = (s + 15) >> 4;
    if (lane == 0 && mb < nb_total && nb_ <= mb) out[(size_t)mb * ldo + nb_] = mx;
  }
}

}  // namespace fa
}  // namespace lemo

using namespace lemo;
using namespace lemo::fa;

extern "C" {

int lemo_exact_block_scores(const void* q, const void* k, int s, int h, int kv, int head_dim,
                            int block, int n_valid, float* out, int ldo, void* stream) {
  if (s <= 0) return 0;
  LEMO_ARG_CHECK(kv > 0 && kv <= h && h % kv == 0 && kv % head_dim == 0,
                 "lemo_exact_block_scores: bad k width");
  LEMO_ARG_CHECK(block == 16, "lemo_exact_block_scores: block size must be 16");
  LEMO_ARG_CHECK(head_dim == 64 || head_dim == 128, "lemo_exact_block_scores: head_dim 64/128");
  const int T = (s + 63) / 64;
  const int tiles = T * (T + 1) / 2;
  auto* qp = reinterpret_cast<const __nv_bfloat16*>(q);
  auto* kp = reinterpret_cast<const __nv_bfloat16*>(k);
  cudaStream_t st = (cudaStream_t)stream;
  if (head_dim == 128) {
    const int smem = 4 * Tile<128>::kBytes;
    static int once = (int)cudaFuncSetAttribute(exact_block_scores_kernel<128>,
                                                cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    (void)once;
    exact_block_scores_kernel<128><<<tiles, 128, smem, st>>>(qp, kp, s, h, kv, n_valid, out,
                                                              ldo);
  } else {
    const int smem = 4 * Tile<64>::kBytes;
    exact_block_scores_kernel<64><<<tiles, 128, smem, st>>>(qp, kp, s, h, kv, n_valid, out, ldo);
  }
  LEMO_CHECK_LAUNCH("lemo_exact_block_scores");
  return 0;
}

}  // extern "C"
