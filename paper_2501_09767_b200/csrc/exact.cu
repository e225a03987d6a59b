// Exact attention block informativeness on tcgen05 (sparsity.py:173-219, Eq. 2):
//   agg[i, j]   = Σ_h max(q_i^h · k_j^h, 0)           (no 1/√d, heads in order)
//   score(m, n) = max over the 16 x 16 tile (m, n ≤ m) of agg / H, with
//                 entries outside  j ≤ i ∧ i < n_valid ∧ j < n_valid  set to 0
// The s x s score matrix is never materialised: one work item is a 128-query
// x 256-key tile; for every head the MMA warp computes S_h = Q_h·K_hᵀ into one
// of two 256-column TMEM buffers while eight epilogue warps fold the other
// buffer's max(S, 0) into per-thread registers (thread = query row, 128 of
// the tile's key columns).  After the last head the epilogue reduces each
// 16 x 16 sub-tile to its maximum (16-lane shuffles) and stores it.  Division
// by H is applied to the maximum: fl(a/H) is monotone, so max(a/H) == max(a)/H
// bit for bit.
//
// kSplit = 3 is the fp32-faithful variant for mask-parity runs: q and k are
// carried as bf16 hi/lo pairs (v ≈ hi + lo) and each head issues hi·hi +
// hi·lo + lo·hi into the same accumulator (the bf16x3 scheme of the predictor
// GEMMs), so the scores agree with the reference's f32 scores
// to ~1e-6 relative instead of the ~1e-3 of bf16 operands.
//
// Work items are rasterised in groups of kGroupQ query tiles sweeping the key
// tiles (key-major inside a group) so each K tile is fetched from HBM once per
// group and served from L2 to the group's CTAs; the kernel is persistent
// (static stride over items; every item costs the same H head-steps).
#include "gemm.cuh"
#include "lemo_internal.h"

namespace lemo {
namespace ex {

constexpr int kQ = 128;                 // query rows per item
constexpr int kN = 256;                 // key columns per item
constexpr int kBoxQ = kQ * 64 * 2;      // [128 x 64] bf16 SW128 = 16 KB
constexpr int kBoxK = kN * 64 * 2;      // [256 x 64] (two 128-row TMA boxes) = 32 KB
constexpr int kThreads = 320;           // w0 TMA, w1 MMA + TMEM, w2..w9 epilogue
constexpr int kGroupQ = 8;

template <int kSplit>
struct Cfg {
  static constexpr int kOps = kSplit == 3 ? 2 : 1;                // hi (+ lo) per operand
  static constexpr int kStageBytes = kOps * (kBoxQ + kBoxK);       // one 64-wide d chunk
  static constexpr int kStages = kSplit == 3 ? 2 : 4;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
};

struct Item {
  int qt, kt;  // query tile (128 rows), key tile (256 columns)
};

// item t -> (qt, kt): groups of kGroupQ query tiles, key-major inside a group;
// key tile kt is needed by query tile qt iff 2·kt <= qt (causal).
__device__ __forceinline__ Item decode_item(int t, int nq) {
  int g0 = 0;
  for (;;) {
    const int g1 = min(g0 + kGroupQ, nq);
    const int kmax = (g1 - 1) >> 1;
    int cnt = 0;
    for (int q = g0; q < g1; ++q) cnt += (q >> 1) + 1;
    if (t < cnt) {
      for (int kt = 0; kt <= kmax; ++kt) {
        const int n = g1 - max(g0, 2 * kt);
        if (t < n) return Item{max(g0, 2 * kt) + t, kt};
        t -= n;
      }
    }
    t -= cnt;
    g0 = g1;
  }
}

__host__ __device__ inline int num_items(int nq) {
  int c = 0;
  for (int q = 0; q < nq; ++q) c += (q >> 1) + 1;
  return c;
}

template <int kSplit, int D>
__global__ void __launch_bounds__(kThreads, 1)
    exact_scores_kernel(const __grid_constant__ CUtensorMap tmQ,
                        const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmQlo,
                        const __grid_constant__ CUtensorMap tmKlo, int s, int H, int group,
                        int n_valid, float* __restrict__ out, int ldo) {
  using C = Cfg<kSplit>;
  constexpr int kChunks = D / 64;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* full = bars;                    // [kStages]
  uint64_t* empty = full + C::kStages;      // [kStages]
  uint64_t* sfull = empty + C::kStages;     // [2]
  uint64_t* sempty = sfull + 2;             // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = (s + kQ - 1) / kQ;
  const int items = num_items(nq);
  const float fH = (float)H;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    if (kSplit == 3) {
      tma_prefetch_desc(&tmQlo);
      tma_prefetch_desc(&tmKlo);
    }
    for (int i = 0; i < C::kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sfull[i], 1);
      mbar_init(&sempty[i], 8);  // one arrive per epilogue warp
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < items; t += gridDim.x) {
        const Item it = decode_item(t, nq);
        for (int hd = 0; hd < H; ++hd) {
          const int cq = hd * D, ck = (hd / group) * D;
#pragma unroll 1
          for (int c = 0; c < kChunks; ++c) {
            mbar_wait(&empty[stage], phase ^ 1);
            mbar_arrive_expect_tx(&full[stage], C::kStageBytes);
            uint8_t* sq = smem + stage * C::kStageBytes;
            uint8_t* sk = sq + C::kOps * kBoxQ;
            tma_load_2d(&tmQ, &full[stage], sq, cq + c * 64, it.qt * kQ);
            tma_load_2d(&tmK, &full[stage], sk, ck + c * 64, it.kt * kN);
            tma_load_2d(&tmK, &full[stage], sk + kBoxK / 2, ck + c * 64, it.kt * kN + 128);
            if constexpr (kSplit == 3) {
              tma_load_2d(&tmQlo, &full[stage], sq + kBoxQ, cq + c * 64, it.qt * kQ);
              tma_load_2d(&tmKlo, &full[stage], sk + kBoxK, ck + c * 64, it.kt * kN);
              tma_load_2d(&tmKlo, &full[stage], sk + kBoxK + kBoxK / 2, ck + c * 64,
                          it.kt * kN + 128);
            }
            if (++stage == C::kStages) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (warp-collective, one elected lane) ----------------
    constexpr uint32_t idesc = umma_idesc_bf16(kQ, kN, 0, 0);
    int stage = 0;
    uint32_t phase = 0;
    uint32_t u = 0;  // head-steps issued by this CTA
    for (int t = blockIdx.x; t < items; t += gridDim.x) {
      for (int hd = 0; hd < H; ++hd, ++u) {
        const uint32_t buf = u & 1;
        mbar_wait(&sempty[buf], ((u >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + buf * kN;
#pragma unroll 1
        for (int c = 0; c < kChunks; ++c) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t aq = smem_u32(smem + stage * C::kStageBytes);
          const uint32_t ak = aq + C::kOps * kBoxQ;
          const uint64_t dq = umma_desc_k_sw128(aq), dk = umma_desc_k_sw128(ak);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint32_t off = (kk * 32) >> 4;  // +32 B per K16 step inside the atom
            umma_bf16_ss_w(d, dq + off, dk + off, idesc, (c | kk) != 0 ? 1u : 0u);
            if constexpr (kSplit == 3) {
              // hi·lo then lo·hi (the lo·lo term is below fp32 resolution)
              umma_bf16_ss_w(d, dq + off, dk + ((kBoxK) >> 4) + off, idesc, 1u);
              umma_bf16_ss_w(d, dq + ((kBoxQ) >> 4) + off, dk + off, idesc, 1u);
            }
          }
          umma_commit_w(&empty[stage]);
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_w(&sfull[buf]);
      }
    }
  } else {
    // ---------------- epilogue: 8 warps ----------------
    const int ew = warp - 2;             // 0..7
    const int wq = warp & 3;             // TMEM lane quarter this warp may access
    const int part = ew >> 2;            // key-column half of the tile
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const int nb = (s + 15) >> 4;
    uint32_t u = 0;
    for (int t = blockIdx.x; t < items; t += gridDim.x) {
      const Item it = decode_item(t, nq);
      float agg[128];
#pragma unroll
      for (int i = 0; i < 128; ++i) agg[i] = 0.f;
      for (int hd = 0; hd < H; ++hd, ++u) {
        const uint32_t buf = u & 1;
        mbar_wait(&sfull[buf], (u >> 1) & 1);
        tc_fence_after();
        const uint32_t ta = tmem + lane_off + buf * kN + part * 128;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(ta + c * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) agg[32 * c + i] += fmaxf(__uint_as_float(r[i]), 0.f);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[buf]);
      }
      // 16 x 16 sub-tile maxima of the masked aggregate
      const int row = it.qt * kQ + wq * 32 + lane;
      const int col0 = it.kt * kN + part * 128;
      const bool row_ok = row < n_valid;
      const int mb = (it.qt * kQ + wq * 32) / 16 + (lane >> 4);
#pragma unroll
      for (int g = 0; g < 8; ++g) {
        float mx = 0.f;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int col = col0 + g * 16 + i;
          if (row_ok && col <= row && col < n_valid) mx = fmaxf(mx, agg[g * 16 + i]);
        }
#pragma unroll
        for (int o = 1; o < 16; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const int nbk = col0 / 16 + g;
        if ((lane & 15) == 0 && mb < nb && nbk <= mb) out[(size_t)mb * ldo + nbk] = __fdiv_rn(mx, fH);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int kSplit, int D>
int launch(const void* q, const void* k, const void* qlo, const void* klo, int s, int h, int kv,
           int n_valid, float* out, int ldo, cudaStream_t st) {
  CUtensorMap tq, tk, tql, tkl;
  int rc = make_tma_bf16_2d(&tq, q, (uint64_t)s, (uint64_t)h, (uint64_t)h, 128);
  if (!rc) rc = make_tma_bf16_2d(&tk, k, (uint64_t)s, (uint64_t)kv, (uint64_t)kv, 128);
  if (!rc && kSplit == 3) rc = make_tma_bf16_2d(&tql, qlo, (uint64_t)s, (uint64_t)h, (uint64_t)h, 128);
  if (!rc && kSplit == 3) rc = make_tma_bf16_2d(&tkl, klo, (uint64_t)s, (uint64_t)kv, (uint64_t)kv, 128);
  if (rc) return rc;
  if (kSplit != 3) {
    tql = tq;
    tkl = tk;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(exact_scores_kernel<kSplit, D>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg<kSplit>::kSmem);
    if (e != cudaSuccess) return (int)e;
    attr = true;
  }
  const int items = num_items((s + kQ - 1) / kQ);
  const int grid = items < gemm_num_sms() ? items : gemm_num_sms();
  exact_scores_kernel<kSplit, D><<<grid, kThreads, Cfg<kSplit>::kSmem, st>>>(
      tq, tk, tql, tkl, s, h / D, h / kv, n_valid, out, ldo);
  return (int)cudaGetLastError();
}

}  // namespace ex
}  // namespace lemo

using namespace lemo;

extern "C" {

int lemo_exact_block_scores(const void* q, const void* k, const void* q_lo, const void* k_lo,
                            int s, int h, int kv, int head_dim, int block, int n_valid,
                            float* out, int ldo, void* stream) {
  if (s <= 0) return 0;
  LEMO_ARG_CHECK(kv > 0 && kv <= h && h % kv == 0 && kv % head_dim == 0,
                 "lemo_exact_block_scores: bad k width");
  LEMO_ARG_CHECK(block == 16, "lemo_exact_block_scores: block size must be 16");
  LEMO_ARG_CHECK(head_dim == 64 || head_dim == 128, "lemo_exact_block_scores: head_dim 64/128");
  LEMO_ARG_CHECK((q_lo == nullptr) == (k_lo == nullptr),
                 "lemo_exact_block_scores: q_lo and k_lo must be given together");
  cudaStream_t st = (cudaStream_t)stream;
  const bool x3 = q_lo != nullptr;
  int rc;
  if (head_dim == 128)
    rc = x3 ? ex::launch<3, 128>(q, k, q_lo, k_lo, s, h, kv, n_valid, out, ldo, st)
            : ex::launch<1, 128>(q, k, q_lo, k_lo, s, h, kv, n_valid, out, ldo, st);
  else
    rc = x3 ? ex::launch<3, 64>(q, k, q_lo, k_lo, s, h, kv, n_valid, out, ldo, st)
            : ex::launch<1, 64>(q, k, q_lo, k_lo, s, h, kv, n_valid, out, ldo, st);
  LEMO_RETURN_RC("lemo_exact_block_scores", rc);
}

}  // extern "C"
