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

// ---------------------------------------------------------------------------
// backward (tensor.py:693-722), split into two atomic-free kernels that both
// recompute P from the saved log-sum-exp.

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Write one thread's row of 128 bf16 values into a SW128 K-major [128 x 128] tile.
__device__ __forceinline__ void store_row_sw128(uint8_t* tile, int r, const float (&v)[kB]) {
#pragma unroll
  for (int a = 0; a < 2; ++a) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float* pv = v + a * 64 + c * 8;
      const uint4 val = make_uint4(pack_bf16x2(pv[0], pv[1]), pack_bf16x2(pv[2], pv[3]),
                                   pack_bf16x2(pv[4], pv[5]), pack_bf16x2(pv[6], pv[7]));
      *reinterpret_cast<uint4*>(tile + a * kBox + r * 128 + ((c ^ (r & 7)) << 4)) = val;
    }
  }
}

__device__ __forceinline__ void tmem_row_load(uint32_t taddr, float (&v)[kB]) {
  uint32_t raw[kB];
#pragma unroll
  for (int c = 0; c < kB / 32; ++c)
    tmem_ld_32x32b_x32(taddr + c * 32, *reinterpret_cast<uint32_t(*)[32]>(raw + c * 32));
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < kB; ++i) v[i] = __uint_as_float(raw[i]);
}

// Issue D (+)= A·B over K = 128 with A K-major SW128 (two 64-col boxes) and B
// either K-major (b_mn = 0) or MN-major (b_mn = 1, two 64-col MN atoms).
template <uint32_t kIdesc, bool kBMN>
__device__ __forceinline__ void mma_k128(uint32_t d, uint32_t a, uint32_t b, bool acc) {
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint32_t offa = (kk >> 2) * kBox + (kk & 3) * 32;
    const uint64_t db = kBMN ? umma_desc_mn_sw128(b + kk * 2048, kBox)
                             : umma_desc_k_sw128(b + offa);
    umma_bf16_ss(d, umma_desc_k_sw128(a + offa), db, kIdesc, (acc || kk > 0) ? 1u : 0u);
  }
}

// Same with an MN-major A operand (A = Xᵀ for a [K rows x M cols] smem tile).
template <uint32_t kIdesc>
__device__ __forceinline__ void mma_k128_amn_bmn(uint32_t d, uint32_t a, uint32_t b, bool acc) {
#pragma unroll
  for (int kk = 0; kk < 8; ++kk)
    umma_bf16_ss(d, umma_desc_mn_sw128(a + kk * 2048, kBox), umma_desc_mn_sw128(b + kk * 2048, kBox),
                 kIdesc, (acc || kk > 0) ? 1u : 0u);
}

// dQ for one 128-query tile: for each key tile j <= diagonal
//   S = Q·K_jᵀ, dP = dO·V_jᵀ (TMEM), dS = P∘(dP − Δ) (threads, → smem),
//   dQ += dS·K_j (K_j as MN-major B), dQ resident in TMEM.
__global__ void __launch_bounds__(256, 1)
    flash_bwd_dq_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                           const __grid_constant__ CUtensorMap tmK,
                           const __grid_constant__ CUtensorMap tmV,
                           const __grid_constant__ CUtensorMap tmO, const float* __restrict__ lse,
                           const float* __restrict__ delta, float* __restrict__ dq, int n, int h,
                           float sl2, float scale) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sO = smem + kTile;      // dO tile
  uint8_t* sK = smem + 2 * kTile;  // [2]
  uint8_t* sV = smem + 4 * kTile;  // [2]
  uint8_t* sS = smem + 6 * kTile;  // dS tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 7 * kTile);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* ds_full = bars + 6;
  uint64_t* dq_done = bars + 7;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qb = (int)(gridDim.x - 1 - blockIdx.x);
  const int hd = blockIdx.y;
  const int q0 = qb * kB, c0 = hd * kD;
  const int nkv = qb + 1;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmO);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(ds_full, 4);
    mbar_init(dq_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 128, tQ = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, 2 * kTile);
      tma_load_2d(&tmQ, q_full, sQ, c0, q0);
      tma_load_2d(&tmQ, q_full, sQ + kBox, c0 + 64, q0);
      tma_load_2d(&tmO, q_full, sO, c0, q0);
      tma_load_2d(&tmO, q_full, sO + kBox, c0 + 64, q0);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[st], 2 * kTile);
        tma_load_2d(&tmK, &kv_full[st], sK + st * kTile, c0, j * kB);
        tma_load_2d(&tmK, &kv_full[st], sK + st * kTile + kBox, c0 + 64, j * kB);
        tma_load_2d(&tmV, &kv_full[st], sV + st * kTile, c0, j * kB);
        tma_load_2d(&tmV, &kv_full[st], sV + st * kTile + kBox, c0 + 64, j * kB);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(kB, kB, 0, 0);
    constexpr uint32_t idesc_q = umma_idesc_bf16(kB, kD, 0, 1);
    const uint32_t aQ = smem_u32(sQ), aO = smem_u32(sO), aS = smem_u32(sS);
    mbar_wait(q_full, 0);
    for (int j = 0; j < nkv; ++j) {
      const int st = j & 1;
      mbar_wait(&kv_full[st], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t aK = smem_u32(sK + st * kTile), aV = smem_u32(sV + st * kTile);
      if (lane == 0) {
        mma_k128<idesc_s, false>(tS, aQ, aK, false);
        mma_k128<idesc_s, false>(tP, aO, aV, false);
        umma_commit(s_full);
      }
      __syncwarp();
      mbar_wait(ds_full, j & 1);
      tc_fence_after();
      if (lane == 0) {
        mma_k128<idesc_q, true>(tQ, aS, aK, j > 0);
        umma_commit(dq_done);
        umma_commit(&kv_empty[st]);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int wq = warp & 3;
    const int r = wq * 32 + lane;
    const int grow = q0 + r;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const float lse2 = grow < n ? lse[(size_t)hd * n + grow] * kLog2e : 0.f;
    const float dl = grow < n ? delta[(size_t)hd * n + grow] : 0.f;
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      float p[kB];
      tmem_row_load(tS + lane_off, p);
      const int kv0 = j * kB;
#pragma unroll
      for (int i = 0; i < kB; ++i) {
        const int key = kv0 + i;
        float e = ex2_approx(fmaf(p[i], sl2, -lse2));
        if (key > grow || key >= n || grow >= n) e = 0.f;
        p[i] = e;
      }
#pragma unroll
      for (int c = 0; c < kB / 32; ++c) {
        uint32_t raw[32];
        tmem_ld_32x32b_x32(tP + lane_off + c * 32, raw);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) p[c * 32 + i] *= (__uint_as_float(raw[i]) - dl);
      }
      if (j > 0) mbar_wait(dq_done, (j - 1) & 1);  // dS buffer free
      store_row_sw128(sS, r, p);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
    }
    mbar_wait(dq_done, (nkv - 1) & 1);
    tc_fence_after();
#pragma unroll 1
    for (int c = 0; c < kD / 32; ++c) {
      uint32_t raw[32];
      tmem_ld_32x32b_x32(tQ + lane_off + c * 32, raw);
      tmem_ld_wait();
      if (grow < n) {
        float4* dst = reinterpret_cast<float4*>(dq + (size_t)grow * h + c0 + c * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          dst[q] = make_float4(__uint_as_float(raw[4 * q]) * scale, __uint_as_float(raw[4 * q + 1]) * scale,
                               __uint_as_float(raw[4 * q + 2]) * scale, __uint_as_float(raw[4 * q + 3]) * scale);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

// dK, dV for one 128-key tile (transposed formulation, thread = key row):
// for each query tile i >= diagonal
//   Sᵀ = K·Q_iᵀ, dPᵀ = V·dO_iᵀ (TMEM); Pᵀ = exp(Sᵀ − lse), dSᵀ = Pᵀ∘(dPᵀ − Δ)
//   (threads → smem, K-major over queries); dV += Pᵀ·dO_i, dK += dSᵀ·Q_i
//   (dO_i, Q_i as MN-major B).  dV, dK stay in TMEM across the whole loop.
__global__ void __launch_bounds__(256, 1)
    flash_bwd_dkdv_tc_kernel(const __grid_constant__ CUtensorMap tmQ,
                             const __grid_constant__ CUtensorMap tmK,
                             const __grid_constant__ CUtensorMap tmV,
                             const __grid_constant__ CUtensorMap tmO,
                             const float* __restrict__ lse, const float* __restrict__ delta,
                             float* __restrict__ dk, float* __restrict__ dv, int n, int h,
                             float sl2, float scale) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + kTile;
  uint8_t* sQ = smem + 2 * kTile;
  uint8_t* sO = smem + 3 * kTile;
  uint8_t* sPt = smem + 4 * kTile;
  uint8_t* sSt = smem + 5 * kTile;
  float* sL = reinterpret_cast<float*>(smem + 6 * kTile);  // [2][128] lse*log2e
  float* sD = sL + 256;                                    // [2][128] delta
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + 256);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;
  uint64_t* st_full = bars + 2;
  uint64_t* pt_full = bars + 3;
  uint64_t* mm_done = bars + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 5);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x, hd = blockIdx.y;
  const int k0 = kb * kB, c0 = hd * kD;
  const int nqb = (n + kB - 1) / kB;
  const int iters = nqb - kb;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmO);
    mbar_init(kv_full, 1);
    mbar_init(q_full, 1);
    mbar_init(st_full, 1);
    mbar_init(pt_full, 4);
    mbar_init(mm_done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tSt = tmem, tPt = tmem + 128, tdV = tmem + 256, tdK = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(kv_full, 2 * kTile);
      tma_load_2d(&tmK, kv_full, sK, c0, k0);
      tma_load_2d(&tmK, kv_full, sK + kBox, c0 + 64, k0);
      tma_load_2d(&tmV, kv_full, sV, c0, k0);
      tma_load_2d(&tmV, kv_full, sV + kBox, c0 + 64, k0);
      for (int it = 0; it < iters; ++it) {
        const int i = kb + it;
        if (it > 0) mbar_wait(mm_done, (it - 1) & 1);  // Q/dO single buffer free
        mbar_arrive_expect_tx(q_full, 2 * kTile);
        tma_load_2d(&tmQ, q_full, sQ, c0, i * kB);
        tma_load_2d(&tmQ, q_full, sQ + kBox, c0 + 64, i * kB);
        tma_load_2d(&tmO, q_full, sO, c0, i * kB);
        tma_load_2d(&tmO, q_full, sO + kBox, c0 + 64, i * kB);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(kB, kB, 0, 0);
    constexpr uint32_t idesc_g = umma_idesc_bf16(kB, kD, 0, 1);
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aQ = smem_u32(sQ), aO = smem_u32(sO);
    const uint32_t aPt = smem_u32(sPt), aSt = smem_u32(sSt);
    mbar_wait(kv_full, 0);
    for (int it = 0; it < iters; ++it) {
      mbar_wait(q_full, it & 1);
      tc_fence_after();
      if (lane == 0) {
        mma_k128<idesc_s, false>(tSt, aK, aQ, false);
        mma_k128<idesc_s, false>(tPt, aV, aO, false);
        umma_commit(st_full);
      }
      __syncwarp();
      mbar_wait(pt_full, it & 1);
      tc_fence_after();
      if (lane == 0) {
        mma_k128<idesc_g, true>(tdV, aPt, aO, it > 0);
        mma_k128<idesc_g, true>(tdK, aSt, aQ, it > 0);
        umma_commit(mm_done);
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int wq = warp & 3;
    const int r = wq * 32 + lane;  // key row within the tile
    const int key = k0 + r;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    for (int it = 0; it < iters; ++it) {
      const int i = kb + it;
      const int qrow0 = i * kB;
      const int buf = it & 1;
      {
        const int qr = qrow0 + r;
        sL[buf * 128 + r] = qr < n ? lse[(size_t)hd * n + qr] * kLog2e : 0.f;
        sD[buf * 128 + r] = qr < n ? delta[(size_t)hd * n + qr] : 0.f;
      }
      named_bar_sync(1, 128);
      mbar_wait(st_full, it & 1);
      tc_fence_after();
      float p[kB];
      tmem_row_load(tSt + lane_off, p);
#pragma unroll
      for (int c = 0; c < kB; ++c) {
        const int qr = qrow0 + c;
        float e = ex2_approx(fmaf(p[c], sl2, -sL[buf * 128 + c]));
        if (key > qr || qr >= n || key >= n) e = 0.f;
        p[c] = e;
      }
      if (it > 0) mbar_wait(mm_done, (it - 1) & 1);  // Pᵀ / dSᵀ tiles free
      store_row_sw128(sPt, r, p);
#pragma unroll
      for (int c = 0; c < kB / 32; ++c) {
        uint32_t raw[32];
        tmem_ld_32x32b_x32(tPt + lane_off + c * 32, raw);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e)
          p[c * 32 + e] *= (__uint_as_float(raw[e]) - sD[buf * 128 + c * 32 + e]);
      }
      store_row_sw128(sSt, r, p);
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(pt_full);
    }
    mbar_wait(mm_done, (iters - 1) & 1);
    tc_fence_after();
#pragma unroll 1
    for (int c = 0; c < kD / 32; ++c) {
      uint32_t rv[32], rk[32];
      tmem_ld_32x32b_x32(tdV + lane_off + c * 32, rv);
      tmem_ld_32x32b_x32(tdK + lane_off + c * 32, rk);
      tmem_ld_wait();
      if (key < n) {
        float4* dvp = reinterpret_cast<float4*>(dv + (size_t)key * h + c0 + c * 32);
        float4* dkp = reinterpret_cast<float4*>(dk + (size_t)key * h + c0 + c * 32);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          dvp[q] = make_float4(__uint_as_float(rv[4 * q]), __uint_as_float(rv[4 * q + 1]),
                               __uint_as_float(rv[4 * q + 2]), __uint_as_float(rv[4 * q + 3]));
          dkp[q] = make_float4(__uint_as_float(rk[4 * q]) * scale, __uint_as_float(rk[4 * q + 1]) * scale,
                               __uint_as_float(rk[4 * q + 2]) * scale, __uint_as_float(rk[4 * q + 3]) * scale);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

constexpr int kSmemDq = 7 * kTile + 1024 + 256;
constexpr int kSmemDkdv = 6 * kTile + 2048 + 1024 + 256;

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

int lemo_attn_delta(const void* o, const void* dout, float* delta, int n, int h, int head_dim,
                    void* stream);

int lemo_flash_bwd_tc(const void* q, const void* k, const void* v, const void* o,
                      const void* dout, const float* lse, float* delta, float* dq, float* dk,
                      float* dv, int n, int h, int head_dim, float scale, void* stream) {
  if (n <= 0) return 0;
  LEMO_ARG_CHECK(head_dim == fatc::kD, "lemo_flash_bwd_tc: head_dim must be 128");
  LEMO_ARG_CHECK(h % head_dim == 0, "lemo_flash_bwd_tc: h % head_dim");
  int rc = lemo_attn_delta(o, dout, delta, n, h, head_dim, stream);
  if (rc) return rc;
  CUtensorMap tq, tk, tv, tdo;
  rc = make_tma_bf16_2d(&tq, q, (uint64_t)n, (uint64_t)h, (uint64_t)h, fatc::kB);
  if (!rc) rc = make_tma_bf16_2d(&tk, k, (uint64_t)n, (uint64_t)h, (uint64_t)h, fatc::kB);
  if (!rc) rc = make_tma_bf16_2d(&tv, v, (uint64_t)n, (uint64_t)h, (uint64_t)h, fatc::kB);
  if (!rc) rc = make_tma_bf16_2d(&tdo, dout, (uint64_t)n, (uint64_t)h, (uint64_t)h, fatc::kB);
  if (rc) LEMO_RETURN_RC("lemo_flash_bwd_tc", rc);
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fatc::flash_bwd_dq_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         fatc::kSmemDq);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fatc::flash_bwd_dkdv_tc_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::kSmemDkdv);
    if (e != cudaSuccess) LEMO_RETURN_RC("lemo_flash_bwd_tc", (int)e);
    attr = true;
  }
  const float sl2 = scale * fatc::kLog2e;
  dim3 grid((n + fatc::kB - 1) / fatc::kB, h / head_dim);
  cudaStream_t st = (cudaStream_t)stream;
  fatc::flash_bwd_dkdv_tc_kernel<<<grid, 256, fatc::kSmemDkdv, st>>>(tq, tk, tv, tdo, lse, delta,
                                                                     dk, dv, n, h, sl2, scale);
  fatc::flash_bwd_dq_tc_kernel<<<grid, 256, fatc::kSmemDq, st>>>(tq, tk, tv, tdo, lse, delta, dq,
                                                                 n, h, sl2, scale);
  LEMO_CHECK_LAUNCH("lemo_flash_bwd_tc");
  return 0;
}

}  // extern "C"
