// Persistent warp-specialised tcgen05 GEMM for sm_100a:  C = A · Bᵀ
//
//   A : [M, K] bf16 row-major (K contiguous)      -> TMA box 128 x 64, SW128
//   B : [N, K] bf16 row-major (K contiguous)      -> TMA box BN  x 64, SW128
//   accumulator: fp32 in TMEM, two BN-column stages (MMA of tile i+1
//   overlaps the epilogue of tile i).
//
// Warp roles (384 threads):  w0 TMA producer · w1 MMA issuer · w2 TMEM
// allocator · w3 idle · w4..w11 epilogue (warp w owns TMEM lanes 32·(w%4)…
// and column half (w-4)/4 of the tile).
// Every epilogue thread owns one output row of the 128-row tile and pulls
// its accumulator row out of TMEM in 32-column chunks; the epilogue functor
// decides what to do with it (plain store, scatter-add into the residual
// stream at idx[row], RoPE + LoRA, SwiGLU scoring, …).  This is how the
// "index-remapped epilogue" of the permutation-free path is realised: the
// GEMM runs on the compact retained rows and the epilogue writes each row
// straight back to its original position.
#pragma once

#include "common.cuh"

namespace lemo {

constexpr int kBlockM = 128;
constexpr int kBlockK = 64;  // one 128-byte swizzle atom of bf16
constexpr int kUmmaK = 16;
constexpr int kGemmThreads = 384;
constexpr int kGroupM = 16;  // rasterisation group (L2 reuse of B tiles)

template <int BN>
struct GemmCfg {
  static constexpr int kStages = BN >= 256 ? 4 : (BN >= 128 ? 6 : 8);
  static constexpr int kABytes = kBlockM * kBlockK * 2;
  static constexpr int kBBytes = BN * kBlockK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;  // two accumulator stages
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
};

struct TileCoord {
  int m, n;
};

__device__ __forceinline__ TileCoord tile_coord(int t, int num_m, int num_n) {
  // grouped rasterisation: kGroupM m-tiles sweep all n before moving on
  const int per_group = kGroupM * num_n;
  const int g = t / per_group;
  const int first_m = g * kGroupM;
  const int gm = min(num_m - first_m, kGroupM);
  const int r = t - g * per_group;
  TileCoord c;
  c.m = first_m + (r % gm);
  c.n = r / gm;
  return c;
}

// Epilogue contract:
//   __device__ void operator()(int row, bool valid, int col0, uint32_t taddr, int part) const
// called by each epilogue thread for its row of the tile; `taddr` is the TMEM
// address of (this warp's lane base, first accumulator column of the tile).
// The functor must issue the same sequence of tcgen05.ld for every lane of
// the warp (they are warp-collective) and only store when `valid`.
// kPromote > 0: fp32-faithful accumulation.  The tcgen05 fp32 accumulator
// does not round to nearest when it adds into TMEM: every MMA step loses up
// to ~2^-23 of the running sum's magnitude toward zero, so a long K loop
// drifts by ~(K/16)·2^-24 relative (measured: 4e-5 at K = 12288, DESIGN §2,
// scripts/probes/acc_precision.py).  With kPromote = G the MMA warp restarts
// the TMEM accumulator every G k-blocks and the epilogue warps add each
// group's partial into fp32 registers with round-to-nearest adds (the
// "promotion" of partial sums to CUDA-core accumulators), then write the sum
// back into TMEM and run the epilogue as usual.  Used by the bf16x3 GEMMs
// (predictor, parity-mode scorers), where the operands carry fp32 precision.
template <int BN, class Epi, bool kBMN = false, int kPromote = 0>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_tn_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   int M, int N, int K, Epi epi) {
  using Cfg = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + Cfg::kStages * Cfg::kABytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStageBytes);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + Cfg::kStages;
  uint64_t* tfull_bar = bars + 2 * Cfg::kStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (M + kBlockM - 1) / kBlockM;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + kBlockK - 1) / kBlockK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < Cfg::kStages; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 8);  // one elected lane per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const TileCoord tc = tile_coord(t, num_m, num_n);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::kStageBytes);
          tma_load_2d(&tmA, &full_bar[stage], smem_a + stage * Cfg::kABytes, kb * kBlockK,
                      tc.m * kBlockM);
          if constexpr (!kBMN) {
            tma_load_2d(&tmB, &full_bar[stage], smem_b + stage * Cfg::kBBytes, kb * kBlockK,
                        tc.n * BN);
          } else {  // B is [K, N] (N contiguous): BN/64 MN-atoms of 64 N x 64 K
#pragma unroll
            for (int a = 0; a < BN / 64; ++a)
              tma_load_2d(&tmB, &full_bar[stage], smem_b + stage * Cfg::kBBytes + a * 8192,
                          tc.n * BN + a * 64, kb * kBlockK);
          }
          if (++stage == Cfg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one warp, one elected lane issues) ----------------
    constexpr uint32_t idesc = umma_idesc_bf16(kBlockM, BN, 0, kBMN ? 1 : 0);
    const int group = kPromote > 0 ? kPromote : num_kb;  // k-blocks per accumulator group
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;  // accumulator groups issued (one per tile unless promoting)
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      for (int kb0 = 0; kb0 < num_kb; kb0 += group, ++local) {
        const int kb1 = min(kb0 + group, num_kb);
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          {  // whole warp, one elected lane issues (descriptors stay uniform)
            const uint64_t da = umma_desc_k_sw128(smem_u32(smem_a + stage * Cfg::kABytes));
            const uint32_t b_addr = smem_u32(smem_b + stage * Cfg::kBBytes);
            const uint64_t db = kBMN ? umma_desc_mn_sw128(b_addr, 8192) : umma_desc_k_sw128(b_addr);
#pragma unroll
            for (int k = 0; k < kBlockK / kUmmaK; ++k) {
              // advancing K inside the 128-B swizzle atom = +32 B on the start address
              umma_bf16_ss_w(d_tmem, da + ((k * kUmmaK * 2) >> 4),
                             db + (kBMN ? (k * 2048) >> 4 : (k * kUmmaK * 2) >> 4), idesc,
                             (kb > kb0 || k != 0) ? 1u : 0u);
            }
            umma_commit_w(&empty_bar[stage]);
            if (kb == kb1 - 1) umma_commit_w(&tfull_bar[acc]);
          }
          if (++stage == Cfg::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int wq = warp & 3;
    const int part = (warp - 4) >> 2;
    int local = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const TileCoord tc = tile_coord(t, num_m, num_n);
      const int row = tc.m * kBlockM + wq * 32 + lane;
      if constexpr (kPromote > 0) {
        constexpr int kCols = BN / 2;  // this warp's half of the tile
        float sum[kCols];
#pragma unroll
        for (int i = 0; i < kCols; ++i) sum[i] = 0.f;
        const int ngroups = (num_kb + kPromote - 1) / kPromote;
        uint32_t taddr = 0;
        int acc = 0;
        for (int g = 0; g < ngroups; ++g, ++local) {
          acc = local & 1;
          mbar_wait(&tfull_bar[acc], (local >> 1) & 1);
          tc_fence_after();
          taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN;
#pragma unroll
          for (int c = 0; c < kCols / 32; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(taddr + part * kCols + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) sum[c * 32 + i] = __fadd_rn(sum[c * 32 + i], __uint_as_float(v[i]));
          }
          if (g + 1 < ngroups) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty_bar[acc]);
          }
        }
        // the promoted sum replaces the last group's partial, then the usual epilogue
#pragma unroll
        for (int c = 0; c < kCols / 32; ++c) {
          uint32_t v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(sum[c * 32 + i]);
          tmem_st_32x32b_x32(taddr + part * kCols + c * 32, v);
        }
        tmem_st_wait();
        // the epilogue functor may read columns the other half's warps wrote
        // (EpiGateUp pairs gate and up columns): all 8 warps first
        tc_fence_before();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        tc_fence_after();
        epi(row, row < M, tc.n * BN, taddr, part);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
      } else {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tfull_bar[acc], acc_phase);
        tc_fence_after();
        const uint32_t taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN;
        epi(row, row < M, tc.n * BN, taddr, part);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty_bar[acc]);
        ++local;
      }
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<Cfg::kTmemCols>(tmem_base);
  }
}

// --------------------------------------------------------------------------
// CTA-pair variant (cluster of 2, tcgen05 cta_group::2): one 256 x 256 output
// tile per pair; each CTA stages its 128-row half of the A tile and its
// 128-row half of the B tile (so per-SM operand traffic per FLOP drops by a
// third versus the 128 x 256 single-CTA tile), the leader CTA issues
// M256·N256·K16 MMAs that read both CTAs' smem and write each CTA's 128
// accumulator lanes; both CTAs' epilogues drain their own TMEM.
//   full[s]  (leader) : leader's expect_tx + the peer's remote arrive, TMA
//                       bytes of both CTAs
//   empty[s] (both)   : multicast commit
//   tfull[a] (both)   : multicast commit;  tempty[a] (leader): 16 epilogue warps

constexpr int kStagesPair = 6;
constexpr int kSmemPair = kStagesPair * 2 * kBlockM * kBlockK * 2 + 1024 + 256;

// Split-K tail.  Tiles are all the same cost, so T tiles on C clusters take
// ceil(T / C) tile-times even when the last wave holds a handful of tiles
// (M = 8208 rows at N = 4096 is 528 tiles = 7.14 waves -> 8).  When the last
// wave is at most half full, its R tiles are each cut into `split` K-ranges
// (R·split ≤ C units, one per cluster): every unit stores its fp32 partial
// accumulator to `ws` and bumps a per-(tile, CTA) counter; the unit whose
// arrival completes the count -- whichever finishes last; no unit ever waits
// for another -- sums all partials in chunk order (deterministic) into its
// TMEM accumulator and runs the epilogue.
constexpr int kPairTailMaxSplit = 4;  // the completing unit reads all partials: keep it short

struct PairTail {
  int full_tiles;  // tiles computed whole (the first full waves)
  int split;       // K-ranges per tail tile (1 = no split-K tail)
  float* ws;       // [unit][rank][part][c32][j][row] float4 partials
  int* ctr;        // [tail tile][rank] arrival counters (reset by the last unit)
};

// Epilogues that may take the split-K tail (specialised next to their
// definitions).  The heavy epilogues (GateUp, DGateUp, QKV) run at full
// register pressure already; the tail's partial-sum code would make them spill.
template <class Epi>
struct PairTailOK {
  static constexpr bool value = false;
};

// Epilogues whose split-K tail is finished by a separate kernel: the tail
// units only store their fp32 partials (no counting, no summing inside the
// GEMM, so the heavy epilogue loop does not grow), and the caller runs a
// fixed-order reduction + the epilogue's effect afterwards (the scatter-add
// GEMMs: lemo_gemm_scatter_add).
template <class Epi>
struct PairTailDeferred {
  static constexpr bool value = false;
};
constexpr int kPairTailMaxSplitDeferred = 16;

struct PairUnit {
  int tile, kb0, kb1, chunk;  // chunk = -1 for a whole tile
};

__device__ __forceinline__ PairUnit pair_unit(int u, const PairTail& tl, int num_kb) {
  PairUnit w;
  if (u < tl.full_tiles) {
    w.tile = u; w.kb0 = 0; w.kb1 = num_kb; w.chunk = -1;
  } else {
    const int v = u - tl.full_tiles;
    w.tile = tl.full_tiles + v / tl.split;
    w.chunk = v % tl.split;
    w.kb0 = w.chunk * num_kb / tl.split;
    w.kb1 = (w.chunk + 1) * num_kb / tl.split;
  }
  return w;
}

// kPromote > 0: promoted accumulation as in gemm_tn_kernel (every kPromote
// k-blocks the TMEM partial goes into the epilogue warps' fp32 registers);
// the split-K tail is not used with it.
template <class Epi, int kPromote = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm_tn_pair_kernel(const __grid_constant__ CUtensorMap tmA,
                        const __grid_constant__ CUtensorMap tmB, int M, int N, int K, Epi epi,
                        PairTail tl) {
  constexpr int BN = 256;
  constexpr int kHalf = kBlockM * kBlockK * 2;  // one 128 x 64 bf16 box = 16 KB
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* smem_a = smem;
  uint8_t* smem_b = smem + kStagesPair * kHalf;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kStagesPair * kHalf);
  uint64_t* full_bar = bars;
  uint64_t* empty_bar = bars + kStagesPair;
  uint64_t* tfull_bar = bars + 2 * kStagesPair;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int num_m = (M + 2 * kBlockM - 1) / (2 * kBlockM);  // 256-row tiles
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + kBlockK - 1) / kBlockK;
  const int cid = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int num_units = tl.full_tiles + (num_tiles - tl.full_tiles) * tl.split;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStagesPair; ++s) {
      mbar_init(&full_bar[s], 2);
      mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull_bar[s], 1);
      mbar_init(&tempty_bar[s], 16);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<512>(tmem_slot);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint32_t full0 = mapa_shared(smem_u32(full_bar), 0);  // the leader's barriers
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cid; u < num_units; u += nclusters) {
        const PairUnit w = pair_unit(u, tl, num_kb);
        const TileCoord tc = tile_coord(w.tile, num_m, num_n);
        for (int kb = w.kb0; kb < w.kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          const uint32_t fb = full0 + stage * 8;
          if (leader)
            mbar_arrive_expect_tx(&full_bar[stage], 4 * kHalf);
          else
            mbar_arrive_cluster(fb);
          tma_load_2d_pair(&tmA, fb, smem_a + stage * kHalf, kb * kBlockK,
                           tc.m * 2 * kBlockM + (int)rank * kBlockM);
          tma_load_2d_pair(&tmB, fb, smem_b + stage * kHalf, kb * kBlockK,
                           tc.n * BN + (int)rank * kBlockM);
          if (++stage == kStagesPair) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc = umma_idesc_bf16(2 * kBlockM, BN, 0, 0);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;  // accumulator groups (one per unit unless promoting)
      for (int u = cid; u < num_units; u += nclusters) {
        const PairUnit w = pair_unit(u, tl, num_kb);
        const int group = kPromote > 0 ? kPromote : (w.kb1 - w.kb0);
        for (int g0 = w.kb0; g0 < w.kb1; g0 += group, ++local) {
          const int g1 = min(g0 + group, w.kb1);
          const int acc = local & 1;
          mbar_wait(&tempty_bar[acc], ((local >> 1) & 1) ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * BN;
          for (int kb = g0; kb < g1; ++kb) {
            mbar_wait(&full_bar[stage], phase);
            tc_fence_after();
            {
              const uint64_t da = umma_desc_k_sw128(smem_u32(smem_a + stage * kHalf));
              const uint64_t db = umma_desc_k_sw128(smem_u32(smem_b + stage * kHalf));
#pragma unroll
              for (int k = 0; k < kBlockK / kUmmaK; ++k)
                umma_bf16_ss_pair_w(d_tmem, da + ((k * kUmmaK * 2) >> 4),
                                    db + ((k * kUmmaK * 2) >> 4), idesc,
                                    (kb > g0 || k > 0) ? 1u : 0u);
              umma_commit_pair_w(&empty_bar[stage]);
              if (kb == g1 - 1) umma_commit_pair_w(&tfull_bar[acc]);
            }
            if (++stage == kStagesPair) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp >= 4) {
    __shared__ int tail_last;  // split-K tail: this unit completed its tile
    const int wq = warp & 3;
    const int part = (warp - 4) >> 2;
    const uint32_t tempty0 = mapa_shared(smem_u32(tempty_bar), 0);
    int local = 0;
    for (int u = cid; u < num_units; u += nclusters, ++local) {
      const PairUnit w = pair_unit(u, tl, num_kb);
      const TileCoord tc = tile_coord(w.tile, num_m, num_n);
      const int row = tc.m * 2 * kBlockM + (int)rank * kBlockM + wq * 32 + lane;
      if constexpr (kPromote > 0) {
        // promoted accumulation (see gemm_tn_kernel): groups of kPromote k-blocks
        constexpr int kCols = BN / 2;
        float sum[kCols];
#pragma unroll
        for (int i = 0; i < kCols; ++i) sum[i] = 0.f;
        const int ngroups = (num_kb + kPromote - 1) / kPromote;
        uint32_t taddr = 0;
        int acc = 0;
        for (int g = 0; g < ngroups; ++g) {
          acc = local & 1;
          mbar_wait(&tfull_bar[acc], (local >> 1) & 1);
          tc_fence_after();
          taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN;
#pragma unroll
          for (int c = 0; c < kCols / 32; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(taddr + part * kCols + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i)
              sum[c * 32 + i] = __fadd_rn(sum[c * 32 + i], __uint_as_float(v[i]));
          }
          if (g + 1 < ngroups) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
            ++local;
          }
        }
#pragma unroll
        for (int c = 0; c < kCols / 32; ++c) {
          uint32_t v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(sum[c * 32 + i]);
          tmem_st_32x32b_x32(taddr + part * kCols + c * 32, v);
        }
        tmem_st_wait();
        tc_fence_before();
        asm volatile("bar.sync 1, 256;" ::: "memory");  // the epilogue may read the other half
        tc_fence_after();
        epi(row, row < M, tc.n * BN, taddr, part);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
        continue;
      }
      const int acc = local & 1;
      mbar_wait(&tfull_bar[acc], (local >> 1) & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(wq * 32) << 16) + acc * BN;
      bool run_epi = true;
      if constexpr (PairTailDeferred<Epi>::value) {
        if (w.chunk >= 0) {  // store this K-range's partial; the caller finishes the tile
          const int tail = w.tile - tl.full_tiles;
          const int r128 = wq * 32 + lane;
          float4* dst = reinterpret_cast<float4*>(tl.ws) +
                        (((size_t)(tail * tl.split + w.chunk) * 2 + rank) * 2 + part) * 4096;
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(taddr + part * 128 + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 8; ++j)
              __stcg(dst + (c * 8 + j) * 128 + r128,
                     make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                 __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
          }
          run_epi = false;
        }
      }
      if constexpr (PairTailOK<Epi>::value) {
      if (w.chunk >= 0) {
        // partial-sum slot of (unit, rank, part): [c32 4][j 8][row 128] float4
        const int tail = w.tile - tl.full_tiles, v0 = tail * tl.split;
        const int r128 = wq * 32 + lane;
        auto slot = [&](int c) {
          return reinterpret_cast<float4*>(tl.ws) + (((size_t)(v0 + c) * 2 + rank) * 2 + part) * 4096;
        };
        int* ctr = tl.ctr + tail * 2 + rank;
        // every unit stores its partial; the unit whose arrival completes the
        // tile's count (whichever finishes last -- no unit ever waits for
        // another) sums all partials in chunk order and runs the epilogue
        float4* dst = slot(w.chunk);
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(taddr + part * 128 + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            __stcg(dst + (c * 8 + j) * 128 + r128,
                   make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                               __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
        }
        __threadfence();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (threadIdx.x == 128) {
          const int old = atomicAdd(ctr, 1);
          tail_last = old == tl.split - 1;
          if (tail_last) {
            atomicExch(ctr, 0);  // ready for the next launch
            __threadfence();
          }
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (!tail_last) {
          run_epi = false;
        } else {
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            // per 8 columns, all partial loads in flight at once, then
            // ((p0 + p1) + p2) + p3: the same order whoever is last
            uint32_t v[32];
#pragma unroll
            for (int h = 0; h < 4; ++h) {
              float4 x[kPairTailMaxSplit][2];
#pragma unroll
              for (int k = 0; k < kPairTailMaxSplit; ++k)
                if (k < tl.split) {
                  const float4* src = slot(k);
#pragma unroll
                  for (int j = 0; j < 2; ++j)
                    x[k][j] = __ldcg(src + (c * 8 + 2 * h + j) * 128 + r128);
                }
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                float4 a = x[0][j];
#pragma unroll
                for (int k = 1; k < kPairTailMaxSplit; ++k)
                  if (k < tl.split) {
                    a.x += x[k][j].x; a.y += x[k][j].y; a.z += x[k][j].z; a.w += x[k][j].w;
                  }
                const int e = 4 * (2 * h + j);
                v[e] = __float_as_uint(a.x);
                v[e + 1] = __float_as_uint(a.y);
                v[e + 2] = __float_as_uint(a.z);
                v[e + 3] = __float_as_uint(a.w);
              }
            }
            tmem_st_32x32b_x32(taddr + part * 128 + c * 32, v);
          }
          tmem_st_wait();
        }
      }
      }
      if (run_epi) epi(row, row < M, tc.n * BN, taddr, part);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty0 + acc * 8);
    }
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tmem_base);
  }
}

// --------------------------------------------------------------------------
// host side

struct GemmShape {
  int M, N, K;
};

// Builds (or fetches from the per-process cache) a 2-D bf16 TMA descriptor
// over a row-major [rows, cols] matrix with a (box_rows x 64) SW128 box.
int make_tma_bf16_2d(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                     uint64_t ld_elems, uint32_t box_rows);
// fp32 row-major [rows, cols] with a (box_rows x 32) SW128 box (TMA stores)
int make_tma_f32_2d(CUtensorMap* out, const void* base, uint64_t rows, uint64_t cols,
                    uint64_t ld_elems, uint32_t box_rows);

int gemm_num_sms();

// Split-K tail scratch of the pair GEMM, one per stream (kernels on one stream
// are ordered, so they may share it): `units` partial slots of 2 x 128 x 256
// fp32 and `tiles` x 2 zeroed counters.  LEMO_GEMM_TAIL=0 disables the tail.
int pair_tail_workspace(cudaStream_t stream, int units, int tiles, float** ws, int** ctr);
bool pair_tail_enabled();

template <int BN, class Epi, bool kBMN = false, int kPromote = 0>
int launch_gemm_tn(const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                   const Epi& epi, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return 0;
  using Cfg = GemmCfg<BN>;
  CUtensorMap ta, tb;
  int rc = make_tma_bf16_2d(&ta, A, (uint64_t)M, (uint64_t)K, (uint64_t)lda, kBlockM);
  if (rc) return rc;
  if constexpr (kBMN)
    rc = make_tma_bf16_2d(&tb, B, (uint64_t)K, (uint64_t)N, (uint64_t)ldb, 64);
  else
    rc = make_tma_bf16_2d(&tb, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, BN);
  if (rc) return rc;
  static bool attr_set = false;  // one per template instantiation
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tn_kernel<BN, Epi, kBMN, kPromote>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::kSmemBytes);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  const int tiles = ((M + kBlockM - 1) / kBlockM) * ((N + BN - 1) / BN);
  const int grid = tiles < gemm_num_sms() ? tiles : gemm_num_sms();
  gemm_tn_kernel<BN, Epi, kBMN, kPromote><<<grid, kGemmThreads, Cfg::kSmemBytes, stream>>>(
      ta, tb, M, N, K, epi);
  return (int)cudaGetLastError();
}

// Pair-tile launch (BN = 256, non-transposed B): grid = 2 x (tiles capped at
// half the SMs), cluster dims fixed by __cluster_dims__.
// Deferred-tail epilogues report the tail they used through *deferred
// (split = 1: none) so the caller can finish those tiles.
template <class Epi, int kPromote = 0>
int launch_gemm_tn_pair(const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                        const Epi& epi, cudaStream_t stream, PairTail* deferred = nullptr) {
  if (M <= 0 || N <= 0) return 0;
  CUtensorMap ta, tb;
  int rc = make_tma_bf16_2d(&ta, A, (uint64_t)M, (uint64_t)K, (uint64_t)lda, kBlockM);
  if (!rc) rc = make_tma_bf16_2d(&tb, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb, kBlockM);
  if (rc) return rc;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tn_pair_kernel<Epi, kPromote>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemPair);
    if (e != cudaSuccess) return (int)e;
    attr_set = true;
  }
  const int tiles = ((M + 2 * kBlockM - 1) / (2 * kBlockM)) * ((N + 255) / 256);
  const int pairs = gemm_num_sms() / 2;
  const int clusters = tiles < pairs ? tiles : pairs;
  PairTail tl{tiles, 1, nullptr, nullptr};
  const int rem = tiles % clusters, num_kb = (K + kBlockK - 1) / kBlockK;
  constexpr bool kDefer = PairTailDeferred<Epi>::value;
  if (kPromote == 0 && (PairTailOK<Epi>::value || (kDefer && deferred != nullptr)) &&
      tiles > clusters && rem > 0 && 2 * rem <= clusters && pair_tail_enabled()) {
    int split = clusters / rem;
    const int max_split = kDefer ? kPairTailMaxSplitDeferred : kPairTailMaxSplit;
    if (split > max_split) split = max_split;
    if (split > num_kb / 4) split = num_kb / 4;  // keep ≥ 4 k-blocks per unit
    if (split >= 2) {
      rc = pair_tail_workspace(stream, rem * split, rem, &tl.ws, &tl.ctr);
      if (rc) return rc;
      tl.full_tiles = tiles - rem;
      tl.split = split;
    }
  }
  if (deferred != nullptr) *deferred = tl;
  gemm_tn_pair_kernel<Epi, kPromote><<<2 * clusters, kGemmThreads, kSmemPair, stream>>>(
      ta, tb, M, N, K, epi, tl);
  return (int)cudaGetLastError();
}

}  // namespace lemo
