// tcgen05 FlashAttention forward over the compact retained sequence
// (tensor.py:646-691 semantics; see attention.cu for the masking rationale).
//
// One CTA = one 128-query tile of one head (head_dim 128).  Warp roles:
//   w0  TMA producer: Q once, then K/V tiles (128 keys) into a 2-deep ring
//   w1  MMA issuer (one thread): S_j = Q·K_jᵀ into a double-buffered TMEM S,
//       O += P_j·V_j with O resident in TMEM (V as an MN-major B operand)
//   w2  TMEM allocator (512 columns: S0 | S1 | O)
//   w4..w7  softmax: thread i owns query row i = TMEM lane i; online softmax
//       in fp32 registers, O rescaled in place in TMEM, P written to shared
//       memory in the SW128 K-major layout the next MMA reads.
// S_{j+1} is computed while the softmax warps work on S_j, and the softmax of
// S_j overlaps P_{j-1}·V_{j-1} on the tensor core.
#include "gemm.cuh"
#include "lemo_internal.h"

namespace lemo {
namespace fatc {

constexpr int kB = 128;                  // query rows = key rows per tile
constexpr int kD = 128;                  // head dim
constexpr int kBox = kB * 64 * 2;        // one [128 x 64] bf16 SW128 box = 16 KB
constexpr int kTile = 2 * kBox;          // [128 x 128] bf16 = 32 KB
constexpr int kSmem = kTile /*Q*/ + 2 * kTile /*K*/ + 2 * kTile /*V*/ + kTile /*P*/ + 1024 + 256;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__global__ void __launch_bounds__(256, 1)
    flash_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                        const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ o,
                        float* __restrict__ lse, int n, int h, float sl2) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = smem + kTile;          // 2 stages
  uint8_t* sV = smem + 3 * kTile;      // 2 stages
  uint8_t* sP = smem + 5 * kTile;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * kTile);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;    // [2]
  uint64_t* v_full = bars + 3;    // [2]
  uint64_t* kv_empty = bars + 5;  // [2]
  uint64_t* s_full = bars + 7;    // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* o_full = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 11);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qb = (int)(gridDim.x - 1 - blockIdx.x);  // heavy tiles first
  const int hd = blockIdx.y;
  const int q0 = qb * kB, c0 = hd * kD;
  const int nkv = qb + 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
    }
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS[2] = {tmem, tmem + 128};
  const uint32_t tO = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, kTile);
      tma_load_2d(&tmQ, q_full, sQ, c0, q0);
      tma_load_2d(&tmQ, q_full, sQ + kBox, c0 + 64, q0);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[st], kTile);
        tma_load_2d(&tmK, &k_full[st], sK + st * kTile, c0, j * kB);
        tma_load_2d(&tmK, &k_full[st], sK + st * kTile + kBox, c0 + 64, j * kB);
        mbar_arrive_expect_tx(&v_full[st], kTile);
        tma_load_2d(&tmV, &v_full[st], sV + st * kTile, c0, j * kB);
        tma_load_2d(&tmV, &v_full[st], sV + st * kTile + kBox, c0 + 64, j * kB);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(kB, kB, 0, 0);
    constexpr uint32_t idesc_o = umma_idesc_bf16(kB, kD, 0, 1);  // V: MN-major B
    const uint32_t aQ = smem_u32(sQ), aP = smem_u32(sP);
    mbar_wait(q_full, 0);
    auto issue_s = [&](int j) {
      const int st = j & 1;
      mbar_wait(&k_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t aK = smem_u32(sK + st * kTile);
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint32_t off = (kk >> 2) * kBox + (kk & 3) * 32;
          umma_bf16_ss(tS[st], umma_desc_k_sw128(aQ + off), umma_desc_k_sw128(aK + off), idesc_s,
                       kk > 0 ? 1u : 0u);
        }
        umma_commit(&s_full[st]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < nkv; ++j) {
      if (j + 1 < nkv) issue_s(j + 1);
      const int st = j & 1;
      mbar_wait(p_full, j & 1);
      mbar_wait(&v_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t aV = smem_u32(sV + st * kTile);
#pragma unroll
        for (int kk = 0; kk < kB / 16; ++kk) {
          const uint32_t offp = (kk >> 2) * kBox + (kk & 3) * 32;
          umma_bf16_ss(tO, umma_desc_k_sw128(aP + offp), umma_desc_mn_sw128(aV + kk * 2048, kBox),
                       idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
        }
        umma_commit(o_full);
        umma_commit(&kv_empty[st]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int wq = warp & 3;
    const int r = wq * 32 + lane;  // row within the tile == TMEM lane
    const int grow = q0 + r;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float s[kB];
      {
        uint32_t raw[kB];
#pragma unroll
        for (int c = 0; c < kB / 32; ++c)
          tmem_ld_32x32b_x32(tS[st] + lane_off + c * 32,
                             *reinterpret_cast<uint32_t(*)[32]>(raw + c * 32));
        tmem_ld_wait();  // one wait for all four loads
#pragma unroll
        for (int i = 0; i < kB; ++i) s[i] = __uint_as_float(raw[i]);
      }
      const int kv0 = j * kB;
      const bool edge = (j == qb) || (kv0 + kB > n);
      if (edge) {
#pragma unroll
        for (int i = 0; i < kB; ++i) {
          const int key = kv0 + i;
          if (key > grow || key >= n) s[i] = -INFINITY;
        }
      }
      // row max / row sum with 8 independent chains (ILP; one warp per SMSP)
      float mr[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) mr[t] = s[t];
#pragma unroll
      for (int i = 8; i < kB; ++i) mr[i & 7] = fmaxf(mr[i & 7], s[i]);
      const float mraw = fmaxf(fmaxf(fmaxf(mr[0], mr[1]), fmaxf(mr[2], mr[3])),
                               fmaxf(fmaxf(mr[4], mr[5]), fmaxf(mr[6], mr[7])));
      // lazy rescaling: keep the running max unless it grew by > 8 (log2
      // units); O / l / lse stay exact because they share the stale max
      const float mx = mraw * sl2;
      const float m_new = (m == -INFINITY || mx > m + 8.f) ? fmaxf(mx, m) : m;
      const float corr = (m == -INFINITY) ? 0.f : ex2_approx(m - m_new);
      float sm[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) sm[t] = 0.f;
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const float p = ex2_approx(fmaf(s[i], sl2, -m_new));
        s[i] = p;
        sm[i & 7] += p;
      }
      const float sum = ((sm[0] + sm[1]) + (sm[2] + sm[3])) + ((sm[4] + sm[5]) + (sm[6] + sm[7]));
      l = l * corr + sum;
      m = m_new;
      if (j > 0) {
        // P_{j-1}·V_{j-1} finished: P buffer is free and O is stable; rescale O
        mbar_wait(o_full, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < kD / 32; ++c) {
            uint32_t raw[32];
            tmem_ld_32x32b_x32(tO + lane_off + c * 32, raw);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) raw[i] = __float_as_uint(__uint_as_float(raw[i]) * corr);
            tmem_st_32x32b_x32(tO + lane_off + c * 32, raw);
          }
          tmem_st_wait();
        }
      }
      // P (bf16) -> shared memory, SW128 K-major [128 rows x 128 keys]
#pragma unroll
      for (int a = 0; a < 2; ++a) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float* pv = s + a * 64 + c * 8;
          const uint4 val = make_uint4(pack_bf16x2(pv[0], pv[1]), pack_bf16x2(pv[2], pv[3]),
                                       pack_bf16x2(pv[4], pv[5]), pack_bf16x2(pv[6], pv[7]));
          *reinterpret_cast<uint4*>(sP + a * kBox + r * 128 + ((c ^ (r & 7)) << 4)) = val;
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(o_full, (nkv - 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l;
#pragma unroll 1
    for (int c = 0; c < kD / 32; ++c) {
      uint32_t raw[32];
      tmem_ld_32x32b_x32(tO + lane_off + c * 32, raw);
      tmem_ld_wait();
      if (grow < n) {
        uint4* dst = reinterpret_cast<uint4*>(o + (size_t)grow * h + c0 + c * 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          dst[q] = make_uint4(
              pack_bf16x2(__uint_as_float(raw[8 * q + 0]) * inv_l, __uint_as_float(raw[8 * q + 1]) * inv_l),
              pack_bf16x2(__uint_as_float(raw[8 * q + 2]) * inv_l, __uint_as_float(raw[8 * q + 3]) * inv_l),
              pack_bf16x2(__uint_as_float(raw[8 * q + 4]) * inv_l, __uint_as_float(raw[8 * q + 5]) * inv_l),
              pack_bf16x2(__uint_as_float(raw[8 * q + 6]) * inv_l, __uint_as_float(raw[8 * q + 7]) * inv_l));
        }
      }
    }
    if (grow < n) lse[(size_t)hd * n + grow] = (m + log2f(l)) * kLn2;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace fatc
}  // namespace lemo

using namespace lemo;

extern "C" {

int lemo_flash_fwd_tc(const void* q, const void* k, const void* v, void* o, float* lse, int n,
                      int h, int head_dim, float scale, void* stream) {
  if (n <= 0) return 0;
  LEMO_ARG_CHECK(head_dim == fatc::kD, "lemo_flash_fwd_tc: head_dim must be 128");
  LEMO_ARG_CHECK(h % head_dim == 0, "lemo_flash_fwd_tc: h % head_dim");
  CUtensorMap tq, tk, tv;
  int rc = make_tma_bf16_2d(&tq, q, (uint64_t)n, (uint64_t)h, (uint64_t)h, fatc::kB);
  if (!rc) rc = make_tma_bf16_2d(&tk, k, (uint64_t)n, (uint64_t)h, (uint64_t)h, fatc::kB);
  if (!rc) rc = make_tma_bf16_2d(&tv, v, (uint64_t)n, (uint64_t)h, (uint64_t)h, fatc::kB);
  if (rc) LEMO_RETURN_RC("lemo_flash_fwd_tc", rc);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fatc::flash_fwd_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::kSmem);
    if (e != cudaSuccess) LEMO_RETURN_RC("lemo_flash_fwd_tc", (int)e);
    attr = true;
  }
  dim3 grid((n + fatc::kB - 1) / fatc::kB, h / head_dim);
  fatc::flash_fwd_tc_kernel<<<grid, 256, fatc::kSmem, (cudaStream_t)stream>>>(
      tq, tk, tv, reinterpret_cast<__nv_bfloat16*>(o), lse, n, h, scale * fatc::kLog2e);
  LEMO_CHECK_LAUNCH("lemo_flash_fwd_tc");
  return 0;
}

}  // extern "C"
