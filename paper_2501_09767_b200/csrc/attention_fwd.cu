// tcgen05 FlashAttention forward over the compact retained sequence
// (tensor.py:646-691: causal by compact index, q pre-scaled by 1/√d, online
// softmax, saves lse), head_dim D = 64 or 128 (template parameter; a D-wide
// tile is D/64 SW128 boxes of 64 columns).
//
// One CTA = two adjacent 128-query tiles (Q0, Q1) of one head sharing every
// K/V tile load; 320 threads:
//   w0-w3  softmax warpgroup 0 (rows of Q0),  w4-w7 softmax warpgroup 1 (Q1)
//   w8     TMA producer (Q0/Q1 once, K_j into a 3-deep ring, V_j into 2)
//   w9     MMA issuer + TMEM allocator (512 columns: S0 | S1 | O0 | O1)
// Per KV tile j the tensor core runs  S0(j) S1(j) | PV0(j) S0(j+1) PV1(j)
// S1(j+1) | …  so softmax WG0 works on S0 while the tensor core serves WG1 and
// vice versa (ping-pong).  P is written back as bf16 over its own S columns
// and read as the TMEM A operand of O += P·V (V_j as an MN-major B operand);
// a later S MMA overwriting those columns is ordered after the PV MMA that
// reads them because tcgen05.mma executes in issue order.  O rescales are
// lazy (only when the running max grows by > 8 in log2 units) and need no
// extra wait: when S_g(j) is complete, PV_g(j-1) is complete too.
// Measured timeline (scripts/fa_trace.py, 8K rows): softmax of a 128-key tile
// ≈ 1.85 k cycles per warpgroup (two warpgroups exponentiating at once), then
// ≈ 1.45 k until the next S is ready (PV + S on the tensor core + issue /
// commit latency): the loop is bound by E + L + 1024 per warpgroup.  An
// ablation without exponentials cuts E to 1.07 k; FMA-pipe polynomial or
// f16x2 exponentials and SFU turn-taking between the warpgroups all measured
// neutral or slower.  Row max with 3-input FMNMX3, scaling and
// row sums with packed FFMA2/FADD2.  The MMA warp issues warp-collectively;
// CTAs are dispatched in head groups of LEMO_FA_HEAD_GROUP, heavy pairs
// first; the first Q/K/V loads precede the TMEM allocation; O leaves through
// smem staging (over the finished Q tile) and TMA tile stores.
#include "gemm.cuh"
#include "lemo_internal.h"

#ifdef LEMO_FA_TRACE
// debug builds only (LEMO_EXTRA_NVCC_FLAGS=-DLEMO_FA_TRACE, scripts/fa_trace.py):
// per-iteration timestamps of the heaviest CTA's softmax warpgroups
__device__ unsigned long long g_fa_trace[2][4][64];  // [wg][event][iteration]
#endif

namespace lemo {
namespace faf {

constexpr int kT = 128;
#ifndef LEMO_FA_HEAD_GROUP
#define LEMO_FA_HEAD_GROUP 8
#endif
#ifndef LEMO_FA_POLY
#define LEMO_FA_POLY 0
#endif
constexpr int kPolyEvery = LEMO_FA_POLY;  // every k-th exponential pair on the FMA pipe (0 = none)
constexpr int kBox = kT * 64 * 2;   // [128 x 64] bf16 SW128 box = 16 KB
template <int D>
constexpr int kTile = (D / 64) * kBox;  // [128 x D]: 32 KB (D = 128) / 16 KB (D = 64)
constexpr int kKStages = 3, kVStages = 2;
constexpr int kThreads = 320;
template <int D>
constexpr int kSmem = (2 + kKStages + kVStages) * kTile<D> + 256;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ uint8_t* aligned_smem(uint8_t* raw) {
  if (smem_u32(raw) & 1023u) __trap();
  return raw;
}

// Warp-collective (the MMA warp stays converged, one elected lane issues);
// descriptor start addresses advance by (offset >> 4) in the low field.
template <uint32_t kIdesc, int D>
__device__ __forceinline__ void mma_qk(uint32_t d, uint32_t a, uint32_t b) {
  const uint64_t da = umma_desc_k_sw128(a), db = umma_desc_k_sw128(b);
#pragma unroll
  for (int kk = 0; kk < D / 16; ++kk) {
    const uint32_t off = ((kk >> 2) * kBox + (kk & 3) * 32) >> 4;
    umma_bf16_ss_w(d, da + off, db + off, kIdesc, kk > 0 ? 1u : 0u);
  }
}

// [128 x D] tile load: D/64 boxes of 64 columns, contiguous in smem.
template <int D>
__device__ __forceinline__ void load_tile(const CUtensorMap* map, uint64_t* bar, uint8_t* dst,
                                          int col, int row) {
#pragma unroll
  for (int b = 0; b < D / 64; ++b) tma_load_2d(map, bar, dst + b * kBox, col + 64 * b, row);
}

// O (+)= P·V: P = bf16 [128 x 128] packed in TMEM columns [p, p+64), V_j smem
// [128 keys x D] = MN-major B.
template <uint32_t kIdesc>
__device__ __forceinline__ void mma_pv(uint32_t d, uint32_t p, uint32_t b, bool acc) {
  const uint64_t db = umma_desc_mn_sw128(b, kBox);
#pragma unroll
  for (int kk = 0; kk < kT / 16; ++kk)
    umma_bf16_ts_w(d, p + kk * 8, db + kk * (2048 >> 4), kIdesc, (acc || kk > 0) ? 1u : 0u);
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    flash_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                     float* __restrict__ lse, int n, int h, int group, float sl2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = aligned_smem(smem_raw);
  constexpr int kTileD = kTile<D>;
  uint8_t* sQ = smem;                          // Q0 | Q1
  uint8_t* sK = smem + 2 * kTileD;             // [kKStages]
  uint8_t* sV = sK + kKStages * kTileD;        // [kVStages]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kVStages * kTileD);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;               // [kKStages]
  uint64_t* k_empty = k_full + kKStages;     // [kKStages]
  uint64_t* v_full = k_empty + kKStages;     // [kVStages]
  uint64_t* v_empty = v_full + kVStages;     // [kVStages]
  uint64_t* s_full = v_empty + kVStages;     // [2] per query tile
  uint64_t* p_full = s_full + 2;             // [2]
  uint64_t* o_done = p_full + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nt = (n + kT - 1) / kT;
  // 1-D grid over (pairs x heads), dispatched in index order: heads in groups
  // of LEMO_FA_HEAD_GROUP, heavy (late) pairs first within a group, so the
  // co-resident CTAs share a few heads' K/V in L2 and no heavy pair starts late
  const int heads = h / D, npairs = (int)gridDim.x / heads;
  const int G = heads < LEMO_FA_HEAD_GROUP ? heads : LEMO_FA_HEAD_GROUP;
  const int grp = (int)blockIdx.x / (npairs * G), gbase = grp * G;
  const int gsz = min(G, heads - gbase), rem = (int)blockIdx.x - grp * npairs * G;
  const int pair = npairs - 1 - rem / gsz;
  const int hd = gbase + rem % gsz, c0 = hd * D;
  const int ck = (hd / group) * D;  // key/value head of this query head
  const int qt0 = 2 * pair;
  const bool two = qt0 + 1 < nt;
  const int T = two ? qt0 + 2 : qt0 + 1;  // KV tiles; Q0 uses [0, qt0], Q1 uses [0, qt0+1]

  if (warp == 8 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1);
      mbar_init(&p_full[g], 4);
      mbar_init(&o_done[g], 1);
    }
    fence_barrier_init();
    // the first loads go out before the TMEM allocation / CTA barrier (first
    // pass over the rings: no empty-slot waits needed)
    mbar_arrive_expect_tx(q_full, (two ? 2 : 1) * kTileD);
    for (int g = 0; g < (two ? 2 : 1); ++g)
      load_tile<D>(&tmQ, q_full, sQ + g * kTileD, c0, (qt0 + g) * kT);
    for (int j = 0; j < min(T, kVStages); ++j) {
      mbar_arrive_expect_tx(&k_full[j], kTileD);
      load_tile<D>(&tmK, &k_full[j], sK + j * kTileD, ck, j * kT);
      mbar_arrive_expect_tx(&v_full[j], kTileD);
      load_tile<D>(&tmV, &v_full[j], sV + j * kTileD, ck, j * kT);
    }
  }
  if (warp == 9) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;  // S_g at 128·g, O_g at 256 + 128·g

  if (warp == 8) {
    if (lane == 0) {
      for (int j = min(T, kVStages); j < T; ++j) {
        const int sk = j % kKStages, sv = j % kVStages;
        mbar_wait(&k_empty[sk], ((j / kKStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[sk], kTileD);
        load_tile<D>(&tmK, &k_full[sk], sK + sk * kTileD, ck, j * kT);
        mbar_wait(&v_empty[sv], ((j / kVStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[sv], kTileD);
        load_tile<D>(&tmV, &v_full[sv], sV + sv * kTileD, ck, j * kT);
      }
    }
  } else if (warp == 9) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(kT, kT, 0, 0);
    constexpr uint32_t idesc_o = umma_idesc_bf16(kT, D, 0, 1);
    const uint32_t aQ = smem_u32(sQ), aK = smem_u32(sK), aV = smem_u32(sV);
    // tile g takes part in KV tile j iff j <= qt0 + g
    auto uses = [&](int g, int j) { return (g == 0 || two) && j <= qt0 + g; };
    auto last_k_user = [&](int j) { return uses(1, j) ? 1 : 0; };
    mbar_wait(q_full, 0);
    auto issue_s = [&](int g, int j) {
      const int sk = j % kKStages;
      if (g == 0) mbar_wait(&k_full[sk], (j / kKStages) & 1);
      tc_fence_after();
      mma_qk<idesc_s, D>(tmem + 128 * g, aQ + g * kTileD, aK + sk * kTileD);
      umma_commit_w(&s_full[g]);
      if (g == last_k_user(j)) umma_commit_w(&k_empty[sk]);
    };
    auto issue_pv = [&](int g, int j) {
      const int sv = j % kVStages;
      mbar_wait(&p_full[g], j & 1);
      if (g == 0 || !uses(0, j)) mbar_wait(&v_full[sv], (j / kVStages) & 1);
      tc_fence_after();
      mma_pv<idesc_o>(tmem + 256 + 128 * g, tmem + 128 * g, aV + sv * kTileD, j > 0);
      if (g == last_k_user(j)) umma_commit_w(&v_empty[sv]);
      if (j == qt0 + g) umma_commit_w(&o_done[g]);
    };
    issue_s(0, 0);
    if (two) issue_s(1, 0);
    for (int j = 0; j < T; ++j) {
      if (uses(0, j)) {
        issue_pv(0, j);
        if (uses(0, j + 1)) issue_s(0, j + 1);
      }
      if (uses(1, j)) {
        if (!uses(0, j + 1) && j + 1 < T) {  // Q0 is done: Q1 now waits for K itself
          const int sk = (j + 1) % kKStages;
          mbar_wait(&k_full[sk], ((j + 1) / kKStages) & 1);
        }
        issue_pv(1, j);
        if (j + 1 < T) issue_s(1, j + 1);
      }
    }
  } else {
    // softmax warpgroup g = warp / 4, thread = query row of tile g
    const int g = warp >> 2;
    if (g == 0 || two) {
      const int wq = warp & 3;
      const int r = wq * 32 + lane;
      const int qt = qt0 + g;
      const int qr = qt * kT + r;
      const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
      const uint32_t tS = tmem + 128 * g + lane_off, tO = tmem + 256 + 128 * g + lane_off;
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j <= qt; ++j) {
#ifdef LEMO_FA_TRACE
        const bool trace = blockIdx.x == 0 && r == 0 && j < 64;
        if (trace) g_fa_trace[g][0][j] = clock64();
#endif
        mbar_wait(&s_full[g], j & 1);
        tc_fence_after();
#ifdef LEMO_FA_TRACE
        if (trace) g_fa_trace[g][1][j] = clock64();
#endif
        float s[kT];
        {
          uint32_t raw[kT];
#pragma unroll
          for (int c = 0; c < kT / 32; ++c)
            tmem_ld_32x32b_x32(tS + c * 32, *reinterpret_cast<uint32_t(*)[32]>(raw + c * 32));
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < kT; ++i) s[i] = __uint_as_float(raw[i]);
        }
        const int kv0 = j * kT;
        const bool edge = (j == qt || kv0 + kT > n);
        if (edge) {
#pragma unroll
          for (int i = 0; i < kT; ++i)
            if (kv0 + i > qr || kv0 + i >= n) s[i] = -INFINITY;
        }
        float mr[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) mr[t] = fmax3(s[t], s[8 + t], s[16 + t]);
#pragma unroll
        for (int i = 24; i + 16 <= kT; i += 16)
#pragma unroll
          for (int t = 0; t < 8; ++t) mr[t] = fmax3(mr[t], s[i + t], s[i + 8 + t]);
#pragma unroll
        for (int t = 0; t < 8; ++t) mr[t] = fmaxf(mr[t], s[kT - 8 + t]);
        const float mraw = fmax3(fmax3(mr[0], mr[1], mr[2]), fmax3(mr[3], mr[4], mr[5]),
                                 fmaxf(mr[6], mr[7]));
        const float mx = mraw * sl2;
        const float m_new = (m == -INFINITY || mx > m + 8.f) ? fmaxf(mx, m) : m;
        const float corr = (m == -INFINITY) ? 0.f : ex2_approx(m - m_new);
        if (j > 0 && __any_sync(0xffffffffu, corr != 1.f)) {
          // PV_g(j-1) completed before S_g(j) did (issue order): O is stable
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t raw[32];
            tmem_ld_32x32b_x32(tO + c * 32, raw);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) raw[i] = __float_as_uint(__uint_as_float(raw[i]) * corr);
            tmem_st_32x32b_x32(tO + c * 32, raw);
          }
        }
        const float2 sl2x2 = make_float2(sl2, sl2), negm = make_float2(-m_new, -m_new);
        float2 sm[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) sm[t] = make_float2(0.f, 0.f);
#pragma unroll
        for (int c = 0; c < kT / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float2 x = ffma2(make_float2(s[32 * c + 2 * i], s[32 * c + 2 * i + 1]), sl2x2, negm);
            if (kPolyEvery && i % kPolyEvery == kPolyEvery - 1) {  // share off the SFU
              x.x = ex2_poly3(x.x);
              x.y = ex2_poly3(x.y);
            } else {
              x.x = ex2_approx(x.x);
              x.y = ex2_approx(x.y);
            }
            sm[i & 3] = fadd2(sm[i & 3], x);
            pk[i] = pack_bf16x2(x.x, x.y);
          }
          tmem_st_32x32b_x16(tS + 16 * c, pk);  // P over the already-read S columns
        }
        const float sum = ((sm[0].x + sm[0].y) + (sm[1].x + sm[1].y)) +
                          ((sm[2].x + sm[2].y) + (sm[3].x + sm[3].y));
        l = l * corr + sum;
        m = m_new;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[g]);
#ifdef LEMO_FA_TRACE
        if (trace) g_fa_trace[g][2][j] = clock64();
#endif
      }
      mbar_wait(&o_done[g], 0);
      tc_fence_after();
      const float inv_l = 1.f / l;
      // O_g = acc / l as bf16, staged over Q_g (every MMA reading it is done)
      // in two 64-column SW128 boxes, then written by TMA (rows ≥ n clipped)
      uint8_t* stage = sQ + g * kTileD;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t raw[32];
        tmem_ld_32x32b_x32(tO + c * 32, raw);
        tmem_ld_wait();
        uint8_t* row = stage + (c >> 1) * kBox + r * 128;
#pragma unroll
        for (int q = 0; q < 4; ++q)
          *reinterpret_cast<uint4*>(row + ((((c & 1) * 4 + q) ^ (r & 7)) << 4)) = make_uint4(
              pack_bf16x2(__uint_as_float(raw[8 * q + 0]) * inv_l, __uint_as_float(raw[8 * q + 1]) * inv_l),
              pack_bf16x2(__uint_as_float(raw[8 * q + 2]) * inv_l, __uint_as_float(raw[8 * q + 3]) * inv_l),
              pack_bf16x2(__uint_as_float(raw[8 * q + 4]) * inv_l, __uint_as_float(raw[8 * q + 5]) * inv_l),
              pack_bf16x2(__uint_as_float(raw[8 * q + 6]) * inv_l, __uint_as_float(raw[8 * q + 7]) * inv_l));
      }
      fence_proxy_async_smem();
      asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
      if (r == 0) {
#pragma unroll
        for (int b = 0; b < D / 64; ++b) tma_store_2d(&tmO, stage + b * kBox, c0 + 64 * b, qt * kT);
        tma_store_commit_and_wait_read();
      }
      if (qr < n) lse[(size_t)hd * n + qr] = (m + log2f(l)) * kLn2;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace faf
}  // namespace lemo

#ifdef LEMO_FA_TRACE
extern "C" int lemo_fa_trace_get(void* host) {
  return (int)cudaMemcpyFromSymbol(host, g_fa_trace, sizeof(g_fa_trace));
}
#endif

using namespace lemo;

extern "C" {

int lemo_flash_fwd_tc(const void* q, const void* k, const void* v, void* o, float* lse, int n,
                      int h, int kv, int head_dim, float scale, void* stream) {
  if (n <= 0) return 0;
  LEMO_ARG_CHECK(head_dim == 64 || head_dim == 128, "lemo_flash_fwd_tc: head_dim must be 64 or 128");
  LEMO_ARG_CHECK(h % head_dim == 0 && kv % head_dim == 0 && kv > 0 && h % kv == 0,
                 "lemo_flash_fwd_tc: h, kv must be multiples of head_dim with kv | h");
  CUtensorMap tq, tk, tv;
  int rc = make_tma_bf16_2d(&tq, q, (uint64_t)n, (uint64_t)h, (uint64_t)h, faf::kT);
  if (!rc) rc = make_tma_bf16_2d(&tk, k, (uint64_t)n, (uint64_t)kv, (uint64_t)kv, faf::kT);
  if (!rc) rc = make_tma_bf16_2d(&tv, v, (uint64_t)n, (uint64_t)kv, (uint64_t)kv, faf::kT);
  CUtensorMap to;  // output (TMA stores)
  if (!rc) rc = make_tma_bf16_2d(&to, o, (uint64_t)n, (uint64_t)h, (uint64_t)h, faf::kT);
  if (rc) LEMO_RETURN_RC("lemo_flash_fwd_tc", rc);
  const int nt = (n + faf::kT - 1) / faf::kT;
  dim3 grid((h / head_dim) * ((nt + 1) / 2));
  cudaStream_t st = (cudaStream_t)stream;
  const float sl2 = scale * faf::kLog2e;
  if (head_dim == 128) {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(faf::flash_fwd_kernel<128>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           faf::kSmem<128>);
      if (e != cudaSuccess) LEMO_RETURN_RC("lemo_flash_fwd_tc", (int)e);
      attr = true;
    }
    faf::flash_fwd_kernel<128><<<grid, faf::kThreads, faf::kSmem<128>, st>>>(
        tq, tk, tv, to, lse, n, h, h / kv, sl2);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(faf::flash_fwd_kernel<64>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           faf::kSmem<64>);
      if (e != cudaSuccess) LEMO_RETURN_RC("lemo_flash_fwd_tc", (int)e);
      attr = true;
    }
    faf::flash_fwd_kernel<64><<<grid, faf::kThreads, faf::kSmem<64>, st>>>(
        tq, tk, tv, to, lse, n, h, h / kv, sl2);
  }
  LEMO_CHECK_LAUNCH("lemo_flash_fwd_tc");
  return 0;
}

}  // extern "C"
