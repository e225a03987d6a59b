// tcgen05 FlashAttention backward over the compact retained sequence
// (tensor.py:693-722: P recomputed from the saved log-sum-exp,
// Δ = Σ dO∘O, dS = P∘(dP − Δ)), head_dim D = 64 or 128 (template parameter),
// atomic-free and deterministic.
//
// Two kernels on 128 x 128 tiles (tcgen05 reaches its full rate only for
// N >= 128: an M128·N64 MMA costs 48 cycles instead of 32, measured by
// scripts/probes/mma_probe.cu), 384 threads: w0 TMA producer, w1 MMA issuer,
// w2 TMEM allocator, w4-w7 / w8-w11 two element-wise warpgroups that split the
// 128 columns of every score tile (WG w owns columns 64w..64w+63).
//
//   dK/dV  CTA = one 128-key tile of one head, thread = key row.  Per
//          128-query tile t (diagonal first):
//            Sᵀ = K·Q_tᵀ, dPᵀ = V·dO_tᵀ                     (TMEM, fp32)
//            phase A: Pᵀ = exp2(Sᵀ·c − lse₂) → bf16 over the Sᵀ columns
//            phase B: dSᵀ = Pᵀ∘(dPᵀ − Δ)     → bf16 over the dPᵀ columns
//            dV += Pᵀ·dO_t, dK += dSᵀ·Q_t  (A operand read from TMEM)
//          issue order  S(0) dP(0) | dV(t) S(t+1) dK(t) dP(t+1) | …  so the
//          tensor core computes S(t+1) while phase B(t) runs and dP(t+1) while
//          phase A(t+1) runs; dV(t) goes out in two K halves as each half of
//          Pᵀ is stored.  dV, dK stay in TMEM (4 × 128 columns in all).
//   dQ     CTA = one 128-query tile, thread = query row.  Per key tile j:
//            S_j = Q·K_jᵀ (double-buffered), dP_j = dO·V_jᵀ,
//            phase A: P = exp2(S·c − lse₂) (registers), phase B: dS = P∘(dP − Δ)
//            → bf16 over the dP columns, dQ += dS·K_j (A from TMEM)
//          issue order  S(0) S(1) dP(0) | dQ(j) dP(j+1) S(j+2) | …
//
// A later MMA that overwrites TMEM columns still read (as bf16 A operand) by
// an earlier one is safe without a wait: tcgen05.mma executes in issue order.
// The MMA warp issues warp-collectively (umma_*_w: elect.sync inside the asm).
// CTAs are dispatched in head groups, heavy tiles first (cta_order); the first
// tiles are loaded before the TMEM allocation; gradients leave through smem
// staging + TMA tile stores (store_tile_f32_tma).  Timelines: scripts/
// fab_trace.py, fabq_trace.py, fab_cta.py (debug build, -DLEMO_FA_TRACE).
#include "gemm.cuh"
#include "lemo_internal.h"

#ifdef LEMO_FA_TRACE
// debug builds only.  Heaviest dK/dV CTA (key tile 0, head 0), [EW wg0, wg1,
// MMA warp][event][tile]: EW [0] before S wait, [1] S ready, [2] P arrive,
// [3] dP ready, [4] dS arrive; MMA [0] p_full seen, [1] dV,S issued, [2]
// ds_full seen, [3] dK,dP issued, [6]/[7] q_full/o_full seen.
__device__ unsigned long long g_fab_trace[3][8][128];
__device__ unsigned long long g_fabq_trace[2][5][128];  // dQ kernel [wg][event][key tile]
// per CTA [kernel][cta]: start, end, smid, units, first S seen, all MMAs done
__device__ unsigned long long g_fab_cta[2][8192][6];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#endif

namespace lemo {
namespace fab {

constexpr int kT = 128;                // rows per tile (keys or queries)
constexpr int kBox = kT * 64 * 2;      // [128 x 64] bf16 SW128 box = 16 KB
template <int D>
constexpr int kTile = (D / 64) * kBox;  // [128 x D] = D/64 boxes
constexpr int kThreads = 384;
constexpr float kLog2e = 1.4426950408889634f;
#ifndef LEMO_FAB_HEAD_GROUP
#define LEMO_FAB_HEAD_GROUP 4
#endif
#ifndef LEMO_FAB_POLY
#define LEMO_FAB_POLY 0
#endif
constexpr int kPolyEvery = LEMO_FAB_POLY;  // every k-th exponential on the FMA pipe (0 = none)
#ifndef LEMO_FABQ_POLY
#define LEMO_FABQ_POLY 0
#endif
constexpr int kPolyQ = LEMO_FABQ_POLY;  // the same for the dQ kernel's recomputed P

// D (+)= A·Bᵀ with A, B [128 x HD] K-major tiles (HD/64 16 KB boxes each).
// Warp-collective (the MMA warp stays converged; one elected lane issues).
// Descriptor start addresses advance by adding (offset >> 4) to the low field
// (smem addresses < 256 KB never carry out of its 14 bits).
template <uint32_t kIdesc, int HD>
__device__ __forceinline__ void mma_kk(uint32_t d, uint32_t a, uint32_t b) {
  const uint64_t da = umma_desc_k_sw128(a), db = umma_desc_k_sw128(b);
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    const uint32_t off = ((kk >> 2) * kBox + (kk & 3) * 32) >> 4;
    umma_bf16_ss_w(d, da + off, db + off, kIdesc, kk > 0 ? 1u : 0u);
  }
}

// D (+)= A·B, A = bf16 [128 x 128] in TMEM, packed as two 32-column groups at
// a_tmem and a_tmem + 64 (columns 64w..64w+31 hold WG w's 64 values); B =
// smem [128 (K) x HD (N)] row-major tile = MN-major, HD/64 16 KB 64-col atoms.
template <uint32_t kIdesc>
__device__ __forceinline__ void mma_tk(uint32_t d, uint32_t a_tmem, uint32_t b, bool acc) {
  const uint64_t db = umma_desc_mn_sw128(b, kBox);
#pragma unroll
  for (int kk = 0; kk < kT / 16; ++kk)
    umma_bf16_ts_w(d, a_tmem + (kk >> 2) * 64 + (kk & 3) * 8, db + kk * (2048 >> 4), kIdesc,
                   (acc || kk > 0) ? 1u : 0u);
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// [128 x HD] tile load: HD/64 boxes of 64 columns, contiguous in smem.
template <int HD>
__device__ __forceinline__ void load_tile(const CUtensorMap* map, uint64_t* bar, uint8_t* dst,
                                          int col, int row) {
#pragma unroll
  for (int b = 0; b < HD / 64; ++b) tma_load_2d(map, bar, dst + b * kBox, col + 64 * b, row);
}

// 32 values → 16 packed bf16x2 TMEM columns (element 2j in the low half).
__device__ __forceinline__ void st_bf16x32(uint32_t taddr, const float* v) {
  uint32_t p[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) p[j] = pack_bf16x2(v[2 * j], v[2 * j + 1]);
  tmem_st_32x32b_x16(taddr, p);
}

// A warpgroup's 128 rows x kCols fp32 accumulator (TMEM columns [0, kCols)
// at taddr, times scale) -> global via smem staging and TMA tile stores
// (boxes of 128 rows x 32 columns, SW128; rows past the tensor are clipped).
// Thread r of the warpgroup owns TMEM lane / tile row r.  Row-per-thread
// st.global of the same data (the previous epilogue) measured ≈ 22 GB/s per
// SM, 5.8 us per dK/dV CTA; this one takes 3.3 us (scripts/fab_cta.py).
template <int kCols>
__device__ __forceinline__ void store_tile_f32_tma(uint32_t taddr, uint8_t* stage,
                                                   const CUtensorMap* map, int x0, int y0,
                                                   float scale, int r, int bar_id) {
  // all TMEM loads in flight before one wait; each 32-column box is handed to
  // the TMA engine as soon as the warpgroup has staged it
  uint32_t raw[kCols / 32][32];
#pragma unroll
  for (int c = 0; c < kCols / 32; ++c) tmem_ld_32x32b_x32(taddr + c * 32, raw[c]);
  tmem_ld_wait();
#pragma unroll
  for (int c = 0; c < kCols / 32; ++c) {
    uint8_t* row = stage + c * 16384 + r * 128;
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<float4*>(row + ((j ^ (r & 7)) << 4)) =
          make_float4(__uint_as_float(raw[c][4 * j]) * scale,
                      __uint_as_float(raw[c][4 * j + 1]) * scale,
                      __uint_as_float(raw[c][4 * j + 2]) * scale,
                      __uint_as_float(raw[c][4 * j + 3]) * scale);
    fence_proxy_async_smem();
    named_bar_sync(bar_id, 128);
    if (r == 0) tma_store_2d(map, stage + c * 16384, x0 + 32 * c, y0);
  }
  if (r == 0) tma_store_commit_and_wait_read();
}

// The 227 KB budget leaves no room for a 1 KB alignment pad: the dynamic
// window must already be 1024-B aligned (it is when no static smem precedes it).
__device__ __forceinline__ uint8_t* aligned_smem(uint8_t* raw) {
  if (smem_u32(raw) & 1023u) __trap();
  return raw;
}

// CTA dispatch order of both backward kernels (1-D grid of tiles x heads).
// Blocks are dispatched in index order.  Heads are taken in groups of
// LEMO_FAB_HEAD_GROUP; within a group, tile rank k (heavy first) is the slow
// index and the head the fast one.  So (a) co-resident CTAs span only a few
// heads and share their Q/dO (dK/dV) or K/V (dQ) tiles in L2, and (b) every
// group's heavy CTAs start early -- with one group per head the last head's
// heaviest CTA started at the very end and left a ~80 us tail (measured
// with scripts/fab_cta.py); with all heads in one group the L2 reuse is lost
// (2-7 % slower).
struct CtaOrder {
  int tile, head;  // tile rank (0 = heaviest), head
};
__device__ __forceinline__ CtaOrder cta_order(int idx, int nblocks, int heads) {
  const int nt = nblocks / heads;
  const int G = heads < LEMO_FAB_HEAD_GROUP ? heads : LEMO_FAB_HEAD_GROUP;
  const int g = idx / (nt * G);
  const int base = g * G, gs = min(G, heads - base);
  const int rem = idx - g * nt * G;
  CtaOrder o;
  o.tile = rem / gs;
  o.head = base + rem % gs;
  return o;
}

// ---------------------------------------------------------------------------
// dK / dV

constexpr int kQStages = 3, kOStages = 2;
static_assert(kOStages <= kQStages, "the pre-barrier loads fill both rings' first kOStages slots");
template <int HD>
constexpr int kSmemKV = (2 + kQStages + kOStages) * kTile<HD> + 2 * 2 * kT * 4 + 256;

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    flash_bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tmQ,
                          const __grid_constant__ CUtensorMap tmK,
                          const __grid_constant__ CUtensorMap tmV,
                          const __grid_constant__ CUtensorMap tmO,
                          const float* __restrict__ lse, const float* __restrict__ delta,
                          const __grid_constant__ CUtensorMap tmdK,
                          const __grid_constant__ CUtensorMap tmdV, int n, int h, int kv,
                          float sl2, float scale) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = aligned_smem(smem_raw);
  constexpr int kTile = fab::kTile<HD>;
  uint8_t* sK = smem;
  uint8_t* sV = smem + kTile;
  uint8_t* sQ = smem + 2 * kTile;              // [kQStages]
  uint8_t* sO = sQ + kQStages * kTile;         // [kOStages]
  float* sLD = reinterpret_cast<float*>(sO + kOStages * kTile);  // [wg][buf][lse₂ 64 | Δ 64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sLD + 2 * 2 * kT);
  uint64_t* kv_full = bars;
  uint64_t* q_full = bars + 1;              // [kQStages]
  uint64_t* q_empty = q_full + kQStages;    // [kQStages]
  uint64_t* o_full = q_empty + kQStages;    // [kOStages]
  uint64_t* o_empty = o_full + kOStages;    // [kOStages]
  uint64_t* s_full = o_empty + kOStages;
  uint64_t* dp_full = s_full + 1;
  uint64_t* p_full = dp_full + 1;   // [2]: Pᵀ columns of query halves 0-31 / 32-63 of each WG
  uint64_t* ds_full = p_full + 2;
  uint64_t* mm_done = ds_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(mm_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // CTA = (key tile, key/value head); with grouped-query attention the loop
  // runs over the `group` query heads sharing this key head (u = g·T + t)
  const CtaOrder co = cta_order(blockIdx.x, gridDim.x, kv / HD);
  const int kb = co.tile, kvh = co.head;  // key tile 0 has the most query tiles
  const int group = h / kv;
  const int k0 = kb * kT, c0 = kvh * HD;
  const int T = (n - k0 + kT - 1) / kT;  // query tiles from the diagonal on
  const int U = group * T;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmO);
    mbar_init(kv_full, 1);
    for (int s = 0; s < kQStages; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < kOStages; ++s) {
      mbar_init(&o_full[s], 1);
      mbar_init(&o_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(dp_full, 1);
    mbar_init(&p_full[0], 8);
    mbar_init(&p_full[1], 8);
    mbar_init(ds_full, 8);
    mbar_init(mm_done, 1);
    fence_barrier_init();
    // the first loads go out before the TMEM allocation / CTA barrier (their
    // ring slots are free on the first pass, so no waits are needed)
    mbar_arrive_expect_tx(kv_full, 2 * kTile);
    load_tile<HD>(&tmK, kv_full, sK, c0, k0);
    load_tile<HD>(&tmV, kv_full, sV, c0, k0);
    for (int t = 0; t < min(U, kOStages); ++t) {
      const int q0 = k0 + (t % T) * kT, cq = (kvh * group + t / T) * HD;
      mbar_arrive_expect_tx(&q_full[t], kTile);
      load_tile<HD>(&tmQ, &q_full[t], sQ + t * kTile, cq, q0);
      mbar_arrive_expect_tx(&o_full[t], kTile);
      load_tile<HD>(&tmO, &o_full[t], sO + t * kTile, cq, q0);
    }
  }
#ifdef LEMO_FA_TRACE
  const int cta_id = blockIdx.x;
  if (threadIdx.x == 0 && cta_id < 8192) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_fab_cta[0][cta_id][0] = gtimer();
    g_fab_cta[0][cta_id][2] = smid;
    g_fab_cta[0][cta_id][3] = U;
  }
#endif
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tP = tmem + 128, tdV = tmem + 256, tdK = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      for (int t = min(U, kOStages); t < U; ++t) {
        const int q0 = k0 + (t % T) * kT, cq = (kvh * group + t / T) * HD;
        const int sq = t % kQStages, so = t % kOStages;
        mbar_wait(&q_empty[sq], ((t / kQStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[sq], kTile);
        load_tile<HD>(&tmQ, &q_full[sq], sQ + sq * kTile, cq, q0);
        mbar_wait(&o_empty[so], ((t / kOStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&o_full[so], kTile);
        load_tile<HD>(&tmO, &o_full[so], sO + so * kTile, cq, q0);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(kT, kT, 0, 0);
    constexpr uint32_t idesc_g = umma_idesc_bf16(kT, HD, 0, 1);
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
    const uint32_t aQ = smem_u32(sQ), aO = smem_u32(sO);
#ifdef LEMO_FA_TRACE
    const bool mtrace = blockIdx.x == 0 && blockIdx.y == 0 && lane == 0;
#define MT(i) if (mtrace && t < 128) g_fab_trace[2][i][t] = clock64();
#else
#define MT(i)
#endif
    mbar_wait(kv_full, 0);
    auto issue_s = [&](int t) {
      const int sq = t % kQStages;
      mbar_wait(&q_full[sq], (t / kQStages) & 1);
      MT(6)
      tc_fence_after();
      mma_kk<idesc_s, HD>(tS, aK, aQ + sq * kTile);
      umma_commit_w(s_full);
    };
    auto issue_dp = [&](int t) {
      const int so = t % kOStages;
      mbar_wait(&o_full[so], (t / kOStages) & 1);
      MT(7)
      tc_fence_after();
      mma_kk<idesc_s, HD>(tP, aV, aO + so * kTile);
      umma_commit_w(dp_full);
    };
    issue_s(0);
    issue_dp(0);
    const uint64_t dO0 = umma_desc_mn_sw128(aO, kBox);
    for (int t = 0; t < U; ++t) {
      // dV(t) in two K halves, each issued as soon as the element-wise warps
      // have stored that half of every warpgroup's Pᵀ columns
      const uint64_t dO = dO0 + (((t % kOStages) * kTile) >> 4);
#pragma unroll
      for (int hf = 0; hf < 2; ++hf) {
        mbar_wait(&p_full[hf], t & 1);
        if (hf == 0) MT(0)
        tc_fence_after();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int kk = (i >> 1) * 4 + hf * 2 + (i & 1);  // WG (i>>1), K-slice 2·hf + (i&1)
          umma_bf16_ts_w(tdV, tS + (kk >> 2) * 64 + (kk & 3) * 8, dO + kk * (2048 >> 4),
                         idesc_g, (t > 0 || kk > 0) ? 1u : 0u);
        }
      }
      umma_commit_w(&o_empty[t % kOStages]);
      if (t + 1 < U) issue_s(t + 1);
      MT(1)
      mbar_wait(ds_full, t & 1);
      MT(2)
      tc_fence_after();
      mma_tk<idesc_g>(tdK, tP, aQ + (t % kQStages) * kTile, t > 0);
      umma_commit_w(&q_empty[t % kQStages]);
      if (t == U - 1) umma_commit_w(mm_done);
      if (t + 1 < U) issue_dp(t + 1);
      MT(3)
    }
#undef MT
  } else if (warp >= 4) {
    const int wg = (warp - 4) >> 2;  // columns 64·wg … 64·wg + 63 of every query tile
    const int wq = warp & 3;
    const int r = wq * 32 + lane;    // key row within the tile == TMEM lane
    const int key = k0 + r;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t tSw = tS + lane_off + 64 * wg, tPw = tP + lane_off + 64 * wg;
    // thread r stages one of this WG's 64 lse₂ (r < 64) or Δ values of tile u;
    // the global load for u+1 is issued one phase ahead (latency hidden)
    // (raw load only: the log2e scaling is applied at the smem store, so no
    // arithmetic waits on the load before the next phase)
    const float* src = r < 64 ? lse : delta;
    const float stage_mul = r < 64 ? kLog2e : 1.f;
    auto stage_val = [&](int u) {
      const int q = k0 + (u % T) * kT + 64 * wg + (r & 63), hq = kvh * group + u / T;
      return __ldg(src + (size_t)hq * n + min(q, n - 1));  // q ≥ n: masked (P = 0) anyway
    };
    float lv = stage_val(0);
    for (int u = 0; u < U; ++u) {
      const int t = u % T;                   // query tile
      const int qw = k0 + t * kT + 64 * wg;  // first query of this WG's columns
      float* L = sLD + (wg * 2 + (u & 1)) * kT;
      L[r] = lv * stage_mul;
      named_bar_sync(1 + wg, 128);
      const bool edge = (t == 0) || (qw + 64 > n) || (key >= n);
      float p[64];
#ifdef LEMO_FA_TRACE
      const bool trace = blockIdx.x == 0 && blockIdx.y == 0 && r == 0 && u < 128;
      if (trace) g_fab_trace[wg][0][u] = clock64();
#endif
      // phase A: Pᵀ (both 32-column halves in flight before one wait)
      mbar_wait(s_full, u & 1);
      tc_fence_after();
#ifdef LEMO_FA_TRACE
      if (u == 0 && warp == 4 && lane == 0 && blockIdx.x < 8192)
        g_fab_cta[0][blockIdx.x][4] = gtimer();
#endif
#ifdef LEMO_FA_TRACE
      if (trace) g_fab_trace[wg][1][u] = clock64();
#endif
      {
        uint32_t raw[64];
        tmem_ld_32x32b_x32(tSw, *reinterpret_cast<uint32_t(*)[32]>(raw));
        tmem_ld_32x32b_x32(tSw + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
        tmem_ld_wait();
        // two halves of 32 columns, each stored (bf16, packed over the already
        // read fp32 columns) and signalled before the next is exponentiated
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
#pragma unroll
          for (int c = 32 * hf; c < 32 * hf + 32; ++c)
            p[c] = (kPolyEvery && c % kPolyEvery == kPolyEvery - 1)  // share of 2^x off the SFU
                       ? ex2_poly3(fmaf(__uint_as_float(raw[c]), sl2, -L[c]))
                       : ex2_approx(fmaf(__uint_as_float(raw[c]), sl2, -L[c]));
          if (edge) {
#pragma unroll
            for (int c = 32 * hf; c < 32 * hf + 32; ++c) {
              const int q = qw + c;
              if (key > q || q >= n || key >= n) p[c] = 0.f;
            }
          }
          st_bf16x32(tSw + 16 * hf, p + 32 * hf);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[hf]);
        }
      }
#ifdef LEMO_FA_TRACE
      if (trace) g_fab_trace[wg][2][u] = clock64();
#endif
      if (u + 1 < U) lv = stage_val(u + 1);
      // phase B: dSᵀ
      mbar_wait(dp_full, u & 1);
      tc_fence_after();
#ifdef LEMO_FA_TRACE
      if (trace) g_fab_trace[wg][3][u] = clock64();
#endif
      {
        uint32_t raw[64];
        tmem_ld_32x32b_x32(tPw, *reinterpret_cast<uint32_t(*)[32]>(raw));
        tmem_ld_32x32b_x32(tPw + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 64; ++c) p[c] *= (__uint_as_float(raw[c]) - L[64 + c]);
      }
      st_bf16x32(tPw, p);
      st_bf16x32(tPw + 16, p + 32);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
#ifdef LEMO_FA_TRACE
      if (trace) g_fab_trace[wg][4][u] = clock64();
#endif
    }
    mbar_wait(mm_done, 0);
    tc_fence_after();
#ifdef LEMO_FA_TRACE
    if (warp == 4 && lane == 0 && cta_id < 8192) g_fab_cta[0][cta_id][5] = gtimer();
#endif
    // operand buffers are all consumed: stage dV (WG0) / dK (WG1) in smem
    if (wg == 0)
      store_tile_f32_tma<HD>(tdV + lane_off, smem, &tmdV, c0, k0, 1.f, r, 1);
    else
      store_tile_f32_tma<HD>(tdK + lane_off, smem + HD * kT * 4, &tmdK, c0, k0, scale, r, 2);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
#ifdef LEMO_FA_TRACE
  if (threadIdx.x == 0 && cta_id < 8192) g_fab_cta[0][cta_id][1] = gtimer();
#endif
}

// ---------------------------------------------------------------------------
// dQ

constexpr int kKStages = 3, kVStages = 2;
static_assert(kVStages <= kKStages, "the pre-barrier loads fill both rings' first kVStages slots");
template <int HD>
constexpr int kSmemQ = (2 + kKStages + kVStages) * kTile<HD> + 256;

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    flash_bwd_dq_kernel(const __grid_constant__ CUtensorMap tmQ,
                        const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV,
                        const __grid_constant__ CUtensorMap tmO,
                        const float* __restrict__ lse, const float* __restrict__ delta,
                        const __grid_constant__ CUtensorMap tmdQ, int n, int h, int kv,
                        float sl2, float scale) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = aligned_smem(smem_raw);
  constexpr int kTile = fab::kTile<HD>;
  uint8_t* sQ = smem;
  uint8_t* sO = smem + kTile;
  uint8_t* sK = smem + 2 * kTile;              // [kKStages]
  uint8_t* sV = sK + kKStages * kTile;         // [kVStages]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + kVStages * kTile);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;               // [kKStages]
  uint64_t* k_empty = k_full + kKStages;     // [kKStages]
  uint64_t* v_full = k_empty + kKStages;     // [kVStages]
  uint64_t* v_empty = v_full + kVStages;     // [kVStages]
  uint64_t* s_full = v_empty + kVStages;     // [2]
  uint64_t* s_free = s_full + 2;             // [2]
  uint64_t* dp_full = s_free + 2;
  uint64_t* ds_full = dp_full + 1;
  uint64_t* dq_done = ds_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const CtaOrder co = cta_order(blockIdx.x, gridDim.x, h / HD);
  const int ntq = (int)gridDim.x / (h / HD);
  const int qb = ntq - 1 - co.tile, hd = co.head;  // the last query tile has the most key tiles
  const int q0 = qb * kT, c0 = hd * HD;
  const int ck = (hd / (h / kv)) * HD;  // key/value head of this query head
  const int T = qb + 1;  // key tiles 0 … diagonal

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    tma_prefetch_desc(&tmO);
    mbar_init(q_full, 1);
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_free[b], 8);
    }
    mbar_init(dp_full, 1);
    mbar_init(ds_full, 8);
    mbar_init(dq_done, 1);
    fence_barrier_init();
    // the first loads go out before the TMEM allocation / CTA barrier
    mbar_arrive_expect_tx(q_full, 2 * kTile);
    load_tile<HD>(&tmQ, q_full, sQ, c0, q0);
    load_tile<HD>(&tmO, q_full, sO, c0, q0);
    for (int j = 0; j < min(T, kVStages); ++j) {
      mbar_arrive_expect_tx(&k_full[j], kTile);
      load_tile<HD>(&tmK, &k_full[j], sK + j * kTile, ck, j * kT);
      mbar_arrive_expect_tx(&v_full[j], kTile);
      load_tile<HD>(&tmV, &v_full[j], sV + j * kTile, ck, j * kT);
    }
  }
#ifdef LEMO_FA_TRACE
  const int cta_id = blockIdx.x;
  if (threadIdx.x == 0 && cta_id < 8192) {
    unsigned int smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_fab_cta[1][cta_id][0] = gtimer();
    g_fab_cta[1][cta_id][2] = smid;
    g_fab_cta[1][cta_id][3] = T;
  }
#endif
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tP = tmem + 256, tdQ = tmem + 384;  // S[b] at 128·b

  if (warp == 0) {
    if (lane == 0) {
      for (int j = min(T, kVStages); j < T; ++j) {
        const int sk = j % kKStages, sv = j % kVStages;
        mbar_wait(&k_empty[sk], ((j / kKStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[sk], kTile);
        load_tile<HD>(&tmK, &k_full[sk], sK + sk * kTile, ck, j * kT);
        mbar_wait(&v_empty[sv], ((j / kVStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[sv], kTile);
        load_tile<HD>(&tmV, &v_full[sv], sV + sv * kTile, ck, j * kT);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = umma_idesc_bf16(kT, kT, 0, 0);
    constexpr uint32_t idesc_g = umma_idesc_bf16(kT, HD, 0, 1);
    const uint32_t aQ = smem_u32(sQ), aO = smem_u32(sO);
    const uint32_t aK = smem_u32(sK), aV = smem_u32(sV);
    mbar_wait(q_full, 0);
    auto issue_s = [&](int j) {
      const int sk = j % kKStages, b = j & 1;
      if (j >= 2) mbar_wait(&s_free[b], ((j - 2) >> 1) & 1);  // phase A of j-2 read it
      mbar_wait(&k_full[sk], (j / kKStages) & 1);
      tc_fence_after();
      mma_kk<idesc_s, HD>(tmem + 128 * b, aQ, aK + sk * kTile);
      umma_commit_w(&s_full[b]);
    };
    auto issue_dp = [&](int j) {
      const int sv = j % kVStages;
      mbar_wait(&v_full[sv], (j / kVStages) & 1);
      tc_fence_after();
      mma_kk<idesc_s, HD>(tP, aO, aV + sv * kTile);
      umma_commit_w(dp_full);
      umma_commit_w(&v_empty[sv]);
    };
    issue_s(0);
    if (T > 1) issue_s(1);
    issue_dp(0);
    for (int j = 0; j < T; ++j) {
      mbar_wait(ds_full, j & 1);
      tc_fence_after();
      mma_tk<idesc_g>(tdQ, tP, aK + (j % kKStages) * kTile, j > 0);
      umma_commit_w(&k_empty[j % kKStages]);
      if (j == T - 1) umma_commit_w(dq_done);
      if (j + 1 < T) issue_dp(j + 1);
      if (j + 2 < T) issue_s(j + 2);
    }
  } else if (warp >= 4) {
    const int wg = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;  // query row within the tile == TMEM lane
    const int qr = q0 + r;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t tPw = tP + lane_off + 64 * wg;
    const float lse2 = qr < n ? lse[(size_t)hd * n + qr] * kLog2e : 0.f;
    const float dl = qr < n ? delta[(size_t)hd * n + qr] : 0.f;
    for (int j = 0; j < T; ++j) {
      const int b = j & 1;
      const int kw = j * kT + 64 * wg;  // first key of this WG's columns
      const bool edge = (j == qb) || (kw + 64 > n) || (qr >= n);
      float p[64];
#ifdef LEMO_FA_TRACE
      const bool qtrace = blockIdx.x == 0 && r == 0 && j < 128;
      if (qtrace) g_fabq_trace[wg][0][j] = clock64();
#endif
      // phase A: P (registers only; both halves in flight before one wait)
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
#ifdef LEMO_FA_TRACE
      if (qtrace) g_fabq_trace[wg][1][j] = clock64();
#endif
      {
        uint32_t raw[64];
        const uint32_t ts = tmem + 128 * b + lane_off + 64 * wg;
        tmem_ld_32x32b_x32(ts, *reinterpret_cast<uint32_t(*)[32]>(raw));
        tmem_ld_32x32b_x32(ts + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 64; ++c)
          p[c] = (kPolyQ && c % kPolyQ == kPolyQ - 1)  // share of 2^x off the SFU
                     ? ex2_poly3(fmaf(__uint_as_float(raw[c]), sl2, -lse2))
                     : ex2_approx(fmaf(__uint_as_float(raw[c]), sl2, -lse2));
      }
      if (edge) {
#pragma unroll
        for (int c = 0; c < 64; ++c) {
          const int key = kw + c;
          if (key > qr || key >= n || qr >= n) p[c] = 0.f;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[b]);
#ifdef LEMO_FA_TRACE
      if (qtrace) g_fabq_trace[wg][2][j] = clock64();
#endif
      // phase B: dS
      mbar_wait(dp_full, j & 1);
      tc_fence_after();
#ifdef LEMO_FA_TRACE
      if (qtrace) g_fabq_trace[wg][3][j] = clock64();
#endif
      {
        uint32_t raw[64];
        tmem_ld_32x32b_x32(tPw, *reinterpret_cast<uint32_t(*)[32]>(raw));
        tmem_ld_32x32b_x32(tPw + 32, *reinterpret_cast<uint32_t(*)[32]>(raw + 32));
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 64; ++c) p[c] *= (__uint_as_float(raw[c]) - dl);
      }
      st_bf16x32(tPw, p);
      st_bf16x32(tPw + 16, p + 32);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
#ifdef LEMO_FA_TRACE
      if (qtrace) g_fabq_trace[wg][4][j] = clock64();
#endif
    }
    mbar_wait(dq_done, 0);
    tc_fence_after();
    constexpr int kHalf = HD / 2;  // each warpgroup stores half of dQ's columns
    store_tile_f32_tma<kHalf>(tdQ + lane_off + kHalf * wg, smem + wg * kHalf * kT * 4, &tmdQ,
                              c0 + kHalf * wg, q0, scale, r, 1 + wg);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
#ifdef LEMO_FA_TRACE
  if (threadIdx.x == 0 && cta_id < 8192) g_fab_cta[1][cta_id][1] = gtimer();
#endif
}

}  // namespace fab
}  // namespace lemo

#ifdef LEMO_FA_TRACE
extern "C" int lemo_fab_trace_get(void* host) {
  return (int)cudaMemcpyFromSymbol(host, g_fab_trace, sizeof(g_fab_trace));
}
extern "C" int lemo_fabq_trace_get(void* host) {
  return (int)cudaMemcpyFromSymbol(host, g_fabq_trace, sizeof(g_fabq_trace));
}
extern "C" int lemo_fab_cta_get(void* host) {
  return (int)cudaMemcpyFromSymbol(host, g_fab_cta, sizeof(g_fab_cta));
}
#endif

namespace lemo {
namespace fab {
// delta[hd, i] = Σ_d dO[i, hd·D + d] · O[i, hd·D + d]  (tensor.py:696): one CTA
// per row, 16-byte loads, a group of D/8 lanes per head, shuffle reduction.
template <int HD>
__global__ void __launch_bounds__(256) delta_kernel(const __nv_bfloat16* __restrict__ o,
                                                    const __nv_bfloat16* __restrict__ dout,
                                                    float* __restrict__ delta, int n, int h) {
  constexpr int kLanes = HD / 8;  // 16 (HD 128) or 8 (HD 64) lanes per head
  const int row = blockIdx.x;
  const int H = h / HD;
  const int sub = threadIdx.x % kLanes;
  for (int base = 0; base < H; base += blockDim.x / kLanes) {  // warp-uniform trip count
    const int hd = base + (int)threadIdx.x / kLanes;
    const bool ok = hd < H;
    const size_t off = (size_t)row * h + (size_t)(ok ? hd : 0) * HD + sub * 8;
    const uint4 a = ok ? *reinterpret_cast<const uint4*>(o + off) : make_uint4(0, 0, 0, 0);
    const uint4 b = ok ? *reinterpret_cast<const uint4*>(dout + off) : make_uint4(0, 0, 0, 0);
    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
    float acc = 0.f;
#pragma unroll
    for (int e = 0; e < 4; ++e)
      acc += bf16_lo(av[e]) * bf16_lo(bv[e]) + bf16_hi(av[e]) * bf16_hi(bv[e]);
#pragma unroll
    for (int m = kLanes / 2; m > 0; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if (ok && sub == 0) delta[(size_t)hd * n + row] = acc;
  }
}
}  // namespace fab
}  // namespace lemo

using namespace lemo;

extern "C" {

int lemo_attn_delta(const void* o, const void* dout, float* delta, int n, int h, int head_dim,
                    void* stream) {
  if (n <= 0) return 0;
  LEMO_ARG_CHECK(head_dim == 64 || head_dim == 128, "lemo_attn_delta: head_dim must be 64 or 128");
  auto* op = reinterpret_cast<const __nv_bfloat16*>(o);
  auto* dp = reinterpret_cast<const __nv_bfloat16*>(dout);
  cudaStream_t st = (cudaStream_t)stream;
  if (head_dim == 128)
    fab::delta_kernel<128><<<n, 256, 0, st>>>(op, dp, delta, n, h);
  else
    fab::delta_kernel<64><<<n, 256, 0, st>>>(op, dp, delta, n, h);
  LEMO_CHECK_LAUNCH("lemo_attn_delta");
  return 0;
}

}  // extern "C"

namespace {
template <int HD>
int launch_bwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
               const CUtensorMap& to, const float* lse, const float* delta,
               const CUtensorMap& tdq, const CUtensorMap& tdk, const CUtensorMap& tdv, int n, int h,
               int kv, float scale, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(fab::flash_bwd_dkdv_kernel<HD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         fab::kSmemKV<HD>);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fab::flash_bwd_dq_kernel<HD>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, fab::kSmemQ<HD>);
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  const float sl2 = scale * fab::kLog2e;
  const int nt = (n + fab::kT - 1) / fab::kT;
  fab::flash_bwd_dkdv_kernel<HD><<<nt * (kv / HD), fab::kThreads, fab::kSmemKV<HD>, st>>>(
      tq, tk, tv, to, lse, delta, tdk, tdv, n, h, kv, sl2, scale);
  fab::flash_bwd_dq_kernel<HD><<<nt * (h / HD), fab::kThreads, fab::kSmemQ<HD>, st>>>(
      tq, tk, tv, to, lse, delta, tdq, n, h, kv, sl2, scale);
  return (int)cudaGetLastError();
}
}  // namespace

extern "C" {

int lemo_flash_bwd_tc(const void* q, const void* k, const void* v, const void* o,
                      const void* dout, const float* lse, float* delta, float* dq, float* dk,
                      float* dv, int n, int h, int kv, int head_dim, float scale, void* stream) {
  if (n <= 0) return 0;
  LEMO_ARG_CHECK(head_dim == 64 || head_dim == 128, "lemo_flash_bwd_tc: head_dim must be 64 or 128");
  LEMO_ARG_CHECK(h % head_dim == 0 && kv % head_dim == 0 && kv > 0 && h % kv == 0,
                 "lemo_flash_bwd_tc: h, kv must be multiples of head_dim with kv | h");
  int rc = lemo_attn_delta(o, dout, delta, n, h, head_dim, stream);
  if (rc) return rc;
  CUtensorMap tq, tk, tv, to;
  rc = make_tma_bf16_2d(&tq, q, (uint64_t)n, (uint64_t)h, (uint64_t)h, fab::kT);
  if (!rc) rc = make_tma_bf16_2d(&tk, k, (uint64_t)n, (uint64_t)kv, (uint64_t)kv, fab::kT);
  if (!rc) rc = make_tma_bf16_2d(&tv, v, (uint64_t)n, (uint64_t)kv, (uint64_t)kv, fab::kT);
  if (!rc) rc = make_tma_bf16_2d(&to, dout, (uint64_t)n, (uint64_t)h, (uint64_t)h, fab::kT);
  CUtensorMap tdq, tdk, tdv;  // fp32 gradient outputs (TMA stores)
  if (!rc) rc = make_tma_f32_2d(&tdq, dq, (uint64_t)n, (uint64_t)h, (uint64_t)h, fab::kT);
  if (!rc) rc = make_tma_f32_2d(&tdk, dk, (uint64_t)n, (uint64_t)kv, (uint64_t)kv, fab::kT);
  if (!rc) rc = make_tma_f32_2d(&tdv, dv, (uint64_t)n, (uint64_t)kv, (uint64_t)kv, fab::kT);
  if (rc) LEMO_RETURN_RC("lemo_flash_bwd_tc", rc);
  cudaStream_t st = (cudaStream_t)stream;
  rc = head_dim == 128
           ? launch_bwd<128>(tq, tk, tv, to, lse, delta, tdq, tdk, tdv, n, h, kv, scale, st)
           : launch_bwd<64>(tq, tk, tv, to, lse, delta, tdq, tdk, tdv, n, h, kv, scale, st);
  LEMO_RETURN_RC("lemo_flash_bwd_tc", rc);
}

}  // extern "C"
