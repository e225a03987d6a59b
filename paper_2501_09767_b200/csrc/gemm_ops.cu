// tcgen05 GEMM instantiations with the LeMo epilogues, exported through the
// C ABI declared in include/lemo.h.
//
// Reference semantics each epilogue reproduces:
//   EpiQKV        kernels.py:95-116 (_project + rope_rotate at positions idx;
//                 the LoRA term rides in a 64-column K-extension of the GEMM)
//   EpiScatterAdd tensor.py:536-550 (scatter_add_rows, in place, no atomics:
//                 retained rows are disjoint)
//   EpiGateUp     model.py:371-396 + sparsity.py:284-290 (SwiGLU inner and
//                 mean |inner| token informativeness, fused in the epilogue)
//   EpiDGateUp    tensor.py:283-292,377-384 (mul / silu backward)
//   EpiStoreF32   matmul forward/backward (tensor.py:316-327)
//   EpiSplit3     predictor layers in fp32-faithful bf16x3 form (predictor.py:83-89)
//
// Every epilogue runs on 8 warps: warp (4 + 4·part + q) owns TMEM lanes
// 32q..32q+31 (= output rows) and the `part`-th half of the tile's columns.
#include "gemm.cuh"
#include "lemo_internal.h"
#include <cstdlib>

namespace lemo {

__device__ __forceinline__ void load_chunk(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  __syncwarp();  // tcgen05.ld is warp-collective: reconverge after masked stores
  tmem_ld_32x32b_x32(taddr, r);
  tmem_ld_wait();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float (&v)[32]) {
  uint4* d = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    d[q] = make_uint4(pack_bf16x2(v[8 * q + 0], v[8 * q + 1]), pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                      pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
  }
}

__device__ __forceinline__ void load_bf16x32(const __nv_bfloat16* src, float (&v)[32]) {
  const uint4* s = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint4 u = s[q];
    v[8 * q + 0] = bf16_lo(u.x);
    v[8 * q + 1] = bf16_hi(u.x);
    v[8 * q + 2] = bf16_lo(u.y);
    v[8 * q + 3] = bf16_hi(u.y);
    v[8 * q + 4] = bf16_lo(u.z);
    v[8 * q + 5] = bf16_hi(u.z);
    v[8 * q + 6] = bf16_lo(u.w);
    v[8 * q + 7] = bf16_hi(u.w);
  }
}

// ---------------------------------------------------------------------------

struct EpiStoreBF16 {
  __nv_bfloat16* C;
  int ldc, N;
  template <int BN>
  __device__ void run(int row, bool valid, int col0, uint32_t taddr, int part) const {
#pragma unroll 1
    for (int c = part * (BN / 2); c < (part + 1) * (BN / 2); c += 32) {
      float v[32];
      load_chunk(taddr + c, v);
      if (valid && col0 + c < N) store_bf16x32(C + (size_t)row * ldc + col0 + c, v);
    }
  }
};

struct EpiStoreF32 {
  float* C;
  int ldc, N, accumulate;
  template <int BN>
  __device__ void run(int row, bool valid, int col0, uint32_t taddr, int part) const {
#pragma unroll 1
    for (int c = part * (BN / 2); c < (part + 1) * (BN / 2); c += 32) {
      float v[32];
      load_chunk(taddr + c, v);
      if (!valid || col0 + c >= N) continue;
      const int n = min(32, N - col0 - c);
      float* dst = C + (size_t)row * ldc + col0 + c;
      if (n == 32 && (ldc & 3) == 0) {
        float4* d = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          if (accumulate) {
            const float4 p = d[q];
            o.x += p.x; o.y += p.y; o.z += p.z; o.w += p.w;
          }
          d[q] = o;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < n) dst[i] = accumulate ? dst[i] + v[i] : v[i];
      }
    }
  }
};

// residual[idx[row]] += acc   (idx == nullptr: identity)
struct EpiScatterAdd {
  float* R;
  int ldr, N;
  const int* idx;
  template <int BN>
  __device__ void run(int row, bool valid, int col0, uint32_t taddr, int part) const {
    const int dst_row = valid ? (idx ? __ldg(idx + row) : row) : 0;
#pragma unroll 1
    for (int c = part * (BN / 2); c < (part + 1) * (BN / 2); c += 32) {
      float v[32];
      load_chunk(taddr + c, v);
      if (valid && col0 + c < N) {
        float4* d = reinterpret_cast<float4*>(R + (size_t)dst_row * ldr + col0 + c);
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 p = d[q];
          p.x += v[4 * q]; p.y += v[4 * q + 1]; p.z += v[4 * q + 2]; p.w += v[4 * q + 3];
          d[q] = p;
        }
      }
    }
  }
};

// Fused q/k/v projection epilogue (kernels.py:103-114).  The LoRA terms are
// already inside the accumulator: the GEMM runs over K = h + 64 with
// A = [xn | s·t_q | s·t_v | 0] and B = [W | B_qᵀ / B_vᵀ | 0] (lemo_lora_qkv_prep,
// lemo_lora_pack_b), so the epilogue only rotates q and k at the retained
// tokens' ORIGINAL positions (tensor.py:604-634).  cos/sin are computed on the
// fly: angle = pos · inv_freq in float64 (the reference's precision), reduced
// mod 2π in float64, then fp32 sincos of the reduced angle — no table gathers.
struct EpiQKV {
  __nv_bfloat16 *q, *k, *v;
  int h, kv, head_dim, rope;  // q width h, k / v width kv (grouped-query attention: kv < h)
  const double* inv_freq;  // [head_dim/2]
  const int* pos;
  const float* row_scale;  // optional RMSNorm 1/rms per row (A operand = bf16(x·w))
  template <int BN>
  __device__ void run(int row, bool valid, int col0, uint32_t taddr, int part) const {
    const int which = col0 < h ? 0 : (col0 < h + kv ? 1 : 2);
    const int cbase = col0 - (which == 0 ? 0 : (which == 1 ? h : h + kv));
    const int ld = which == 0 ? h : kv;
    __nv_bfloat16* out = which == 0 ? q : (which == 1 ? k : v);
    const double dp = (valid && rope) ? (double)__ldg(pos + row) : 0.0;
    const int half = head_dim >> 1;
    const int per_head = half >> 5;  // 32-column rotation chunks per head
    const int items = (BN / head_dim) * per_head;
#pragma unroll 1
    for (int it = part; it < items; it += 2) {
      const int hd = (it / per_head) * head_dim, cp = (it % per_head) * 32;
      float a[32], b[32];
      load_chunk(taddr + hd + cp, a);
      load_chunk(taddr + hd + half + cp, b);
      if (!valid) continue;
      if (row_scale != nullptr) {
        const float rs = __ldg(row_scale + row);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          a[i] *= rs;
          b[i] *= rs;
        }
      }
      const int ca = cbase + hd + cp, cb = ca + half;
      if (rope && which < 2) {  // only q and k are rotated (kernels.py:112-114)
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const double ang = dp * __ldg(inv_freq + cp + i);
          const double kq = rint(ang * 0.15915494309189535);
          const float red = (float)fma(-kq, 6.283185307179586476925, ang);
          float sn, cs;
          __sincosf(red, &sn, &cs);  // |red| <= pi: abs err < 2^-21
          const float xa = a[i], xb = b[i];
          a[i] = xa * cs - xb * sn;
          b[i] = xa * sn + xb * cs;
        }
      }
      store_bf16x32(out + (size_t)row * ld + ca, a);
      store_bf16x32(out + (size_t)row * ld + cb, b);
    }
  }
};

// SwiGLU / ReLU front half of the MLP with the token-informativeness
// reduction in the epilogue.  Weight columns are interleaved in 128-column
// chunks (gate chunk i at [256i, 256i+128), up chunk i at [256i+128, 256i+256)),
// so one BN=256 tile holds matching gate/up columns.
//   gu      : [M, N] bf16, same interleaved column order (saved for backward)
//   inner   : [M, N/2] bf16 (silu) or [M, N] (relu), optional
//   partial : [N/128, M] fp32 row sums of |inner| per half tile, optional
//   exact   : score from the fp32 accumulator instead of the bf16-rounded
//             gate/up (the fp32-faithful parity mode: the GEMM then runs on
//             bf16x3 operands, K = 3h, so the accumulator carries f32 precision)
//   row_scale : optional per-row factor applied to the accumulator (the RMSNorm
//             1/rms when the A operand is bf16(x·w), lemo_rmsnorm_gather_fold)
template <bool exact>
struct EpiGateUpT {
  __nv_bfloat16* gu;
  int ldgu;
  __nv_bfloat16* inner;
  int ldi;
  float* partial;
  int M, relu;
  const float* row_scale;
  template <int BN>
  __device__ void run(int row, bool valid, int col0, uint32_t taddr, int part) const {
    static_assert(BN == 256, "gate/up interleave assumes 256-column tiles");
    float score = 0.f;
    const float rs = (row_scale != nullptr && valid) ? __ldg(row_scale + row) : 1.f;
    if (!relu) {
#pragma unroll 1
      for (int c = part * 64; c < part * 64 + 64; c += 32) {
        float g[32], u[32];
        load_chunk(taddr + c, g);
        load_chunk(taddr + 128 + c, u);
        if (!valid) continue;
        if (row_scale != nullptr) {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            g[i] *= rs;
            u[i] *= rs;
          }
        }
        // inner from the bf16-rounded gate/up that are saved for backward, so the
        // dense path and the compaction path (mlp_compact) produce identical rows
        float in[32];
        if constexpr (exact) {  // the reference's two-branch logistic on expf (tensor.py:368-374)
#pragma unroll
          for (int i = 0; i < 32; ++i) score += fabsf(g[i] * sigmoid_stable(g[i]) * u[i]);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          g[i] = round_bf16(g[i]);
          u[i] = round_bf16(u[i]);
          in[i] = g[i] * sigmoid_fast(g[i]) * u[i];
          if (!exact) score += fabsf(in[i]);
        }
        if (gu) {
          store_bf16x32(gu + (size_t)row * ldgu + col0 + c, g);
          store_bf16x32(gu + (size_t)row * ldgu + col0 + 128 + c, u);
        }
        if (inner) store_bf16x32(inner + (size_t)row * ldi + (col0 >> 1) + c, in);
      }
    } else {
#pragma unroll 1
      for (int c = part * 128; c < part * 128 + 128; c += 32) {
        float u[32];
        load_chunk(taddr + c, u);
        if (!valid) continue;
        if (row_scale != nullptr) {
#pragma unroll
          for (int i = 0; i < 32; ++i) u[i] *= rs;
        }
        float in[32];
        if constexpr (exact) {
#pragma unroll
          for (int i = 0; i < 32; ++i) score += fmaxf(u[i], 0.f);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          u[i] = round_bf16(u[i]);
          in[i] = fmaxf(u[i], 0.f);
          if (!exact) score += in[i];
        }
        if (gu) store_bf16x32(gu + (size_t)row * ldgu + col0 + c, u);
        if (inner) store_bf16x32(inner + (size_t)row * ldi + col0 + c, in);
      }
    }
    if (valid && partial) partial[(size_t)((col0 / 256) * 2 + part) * M + row] = score;
  }
};
using EpiGateUp = EpiGateUpT<false>;
using EpiGateUpExact = EpiGateUpT<true>;

// dinner = dy · W_downᵀ ; epilogue turns it into d(gate), d(up) using the
// saved gate/up (silu:  dg = dinner·u·σ(g)(1+g(1-σ(g))),  du = dinner·g·σ(g);
// relu: du = dinner·[u>0]).  Output in the same interleaved layout as gu.
struct EpiDGateUp {
  const __nv_bfloat16* gu;
  int ldgu;
  __nv_bfloat16* dgu;
  int relu;
  template <int BN>
  __device__ void run(int row, bool valid, int col0, uint32_t taddr, int part) const {
#pragma unroll 1
    for (int c = part * (BN / 2); c < (part + 1) * (BN / 2); c += 32) {
      const int mc = col0 + c;
      const int gcol = relu ? mc : (mc >> 7) * 256 + (mc & 127);
      // issue the saved-activation loads before the TMEM load
      float g[32], u[32];
      if (valid) {
        load_bf16x32(gu + (size_t)row * ldgu + gcol, g);
        if (!relu) load_bf16x32(gu + (size_t)row * ldgu + gcol + 128, u);
      }
      float d[32];
      load_chunk(taddr + c, d);
      if (!valid) continue;
      if (!relu) {
        float dg[32], du[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float s = sigmoid_fast(g[i]);
          du[i] = d[i] * (g[i] * s);
          dg[i] = d[i] * u[i] * (s * (1.f + g[i] * (1.f - s)));
        }
        store_bf16x32(dgu + (size_t)row * ldgu + gcol, dg);
        store_bf16x32(dgu + (size_t)row * ldgu + gcol + 128, du);
      } else {
#pragma unroll
        for (int i = 0; i < 32; ++i) g[i] = g[i] > 0.f ? d[i] : 0.f;
        store_bf16x32(dgu + (size_t)row * ldgu + mc, g);
      }
    }
  }
};

// fp32-faithful GEMM chains on bf16 tensor cores ("bf16x3"): a fp32 value v
// is carried as hi = bf16(v), lo = bf16(v - hi); A·B ≈ Ahi·Bhi + Ahi·Blo +
// Alo·Bhi, realised as ONE GEMM over K' = 3K with A' = [hi|hi|lo] (pattern 0)
// and B' = [hi|lo|hi] (pattern 1).  This epilogue applies relu·mask (the
// Predictor hidden layers, predictor.py:83-89) and writes the split form of
// the result for the next GEMM of the chain, and/or the fp32 value.
struct EpiSplit3 {
  __nv_bfloat16* out;  // [M, 3N] (or null)
  int ldo;
  float* f32;  // [M, N] (or null)
  int ldf, N, pattern, relu;
  const unsigned char* mask;
  // dual output (nsplit > 0, a multiple of 32): columns >= nsplit belong to a
  // second product stacked along N (the key predictor's first layer next to
  // the query predictor's) and go to out2 [M, 3(N - nsplit)] instead
  __nv_bfloat16* out2 = nullptr;
  int ldo2 = 0, nsplit = 0;
  template <int BN>
  __device__ void run(int row, bool valid, int col0, uint32_t taddr, int part) const {
#pragma unroll 1
    for (int c = part * (BN / 2); c < (part + 1) * (BN / 2); c += 32) {
      float v[32];
      load_chunk(taddr + c, v);
      if (!valid || col0 + c >= N) continue;
      const bool second = nsplit > 0 && col0 + c >= nsplit;
      __nv_bfloat16* const base = second ? out2 : out;
      const int Nb = second ? N - nsplit : (nsplit > 0 ? nsplit : N);
      const int ldb = second ? ldo2 : ldo, cb = second ? col0 + c - nsplit : col0 + c;
      float hi[32], lo[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        float x = v[i];
        if (relu) x = fmaxf(x, 0.f);
        if (mask && !mask[min(col0 + c + i, N - 1)]) x = 0.f;
        v[i] = x;
        hi[i] = round_bf16(x);
        lo[i] = x - hi[i];
      }
      const int n = min(32, N - col0 - c);
      if (base) {
        __nv_bfloat16* o = base + (size_t)row * ldb + cb;
        if (n == 32 && (ldb & 7) == 0 && (Nb & 7) == 0) {
          store_bf16x32(o, hi);
          store_bf16x32(o + Nb, pattern ? lo : hi);
          store_bf16x32(o + 2 * Nb, pattern ? hi : lo);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            if (i < n) {
              o[i] = __float2bfloat16_rn(hi[i]);
              o[Nb + i] = __float2bfloat16_rn(pattern ? lo[i] : hi[i]);
              o[2 * Nb + i] = __float2bfloat16_rn(pattern ? hi[i] : lo[i]);
            }
          }
        }
      }
      if (f32) {
        float* d = f32 + (size_t)row * ldf + col0 + c;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (i < n) d[i] = v[i];
      }
    }
  }
};

// The kernel template calls epi(row, valid, col0, taddr, part); wrap run<BN>.
template <int BN, class Epi>
struct Bound {
  Epi e;
  __device__ void operator()(int row, bool valid, int col0, uint32_t taddr, int part) const {
    e.template run<BN>(row, valid, col0, taddr, part);
  }
};

template <> struct PairTailOK<Bound<256, EpiStoreF32>> { static constexpr bool value = true; };
template <> struct PairTailDeferred<Bound<256, EpiScatterAdd>> { static constexpr bool value = true; };

// Finish of the scatter-add GEMM's deferred split-K tail: one thread per
// float4 of a tail tile (tile, CTA half, column half, 32-column chunk, 4
// columns, row) sums the K-range partials in chunk order (deterministic) and
// adds the result into R[idx[row]] -- what the epilogue would have done with
// the whole tile's accumulator.  All partial loads of a thread are in flight
// at once (the reduction is latency-bound otherwise).
__global__ void __launch_bounds__(128) scatter_tail_finish_kernel(PairTail tl, int num_m,
                                                                  int num_n, int M, int N,
                                                                  float* __restrict__ R, int ldr,
                                                                  const int* __restrict__ idx) {
  const int cj = blockIdx.x & 31, half = (blockIdx.x >> 5) & 3, tail = blockIdx.x >> 7;
  const int rank = half >> 1, part = half & 1, c = cj >> 3, j = cj & 7;
  const int r128 = threadIdx.x;
  const TileCoord tc = tile_coord(tl.full_tiles + tail, num_m, num_n);
  const int row = tc.m * 2 * kBlockM + rank * kBlockM + r128;
  const int col = tc.n * 256 + part * 128 + c * 32 + 4 * j;
  if (row >= M || col >= N) return;
  const float4* src = reinterpret_cast<const float4*>(tl.ws) +
                      ((size_t)(tail * tl.split) * 2 + rank) * 2 * 4096 + part * 4096 +
                      (c * 8 + j) * 128 + r128;
  const size_t unit = (size_t)2 * 2 * 4096;  // float4 stride between K-range units
  float4 p[kPairTailMaxSplitDeferred];
#pragma unroll
  for (int k = 0; k < kPairTailMaxSplitDeferred; ++k)
    if (k < tl.split) p[k] = __ldcg(src + k * unit);
  float4 a = p[0];
#pragma unroll
  for (int k = 1; k < kPairTailMaxSplitDeferred; ++k)
    if (k < tl.split) { a.x += p[k].x; a.y += p[k].y; a.z += p[k].z; a.w += p[k].w; }
  float4* d = reinterpret_cast<float4*>(R + (size_t)(idx ? __ldg(idx + row) : row) * ldr + col);
  float4 q = *d;
  q.x += a.x; q.y += a.y; q.z += a.z; q.w += a.w;
  *d = q;
}
template <> struct PairTailOK<Bound<256, EpiStoreBF16>> { static constexpr bool value = true; };

// BN = 256 GEMMs run as CTA pairs (256 x 256 tiles) when M spans at least two
// row tiles; LEMO_GEMM_PAIR=0 forces the single-CTA kernel (A/B comparisons).
static bool use_pair(int M) {
  static const int env = getenv("LEMO_GEMM_PAIR") ? atoi(getenv("LEMO_GEMM_PAIR")) : 1;
  return env != 0 && M > kBlockM;
}

template <int BN, class Epi>
static int gemm(const void* A, int lda, const void* B, int ldb, int M, int N, int K, const Epi& e,
                cudaStream_t st) {
  Bound<BN, Epi> b{e};
  if constexpr (BN == 256) {
    if (use_pair(M)) return launch_gemm_tn_pair(A, lda, B, ldb, M, N, K, b, st);
  }
  return launch_gemm_tn<BN>(A, lda, B, ldb, M, N, K, b, st);
}

// Tile width: the widest BN whose tile count still fills the 148 SMs (wide
// tiles re-read A less and run the MMA at full rate; BN = 64 costs 48 instead
// of 32 cycles per MMA but doubles the CTAs of small GEMMs such as the
// predictor layers, Eq. 3 and the rank-r LoRA products).
static int pick_bn(int M, int N) {
  static const int forced = getenv("LEMO_GEMM_BN") ? atoi(getenv("LEMO_GEMM_BN")) : 0;
  if (forced) return forced;
  const int tm = (M + kBlockM - 1) / kBlockM;
  if (N <= 64) return 64;
  if (tm * ((N + 255) / 256) >= kNumSMs) return 256;
  if (tm * ((N + 127) / 128) >= kNumSMs) return 128;
  return 64;
}

// fp32-faithful accumulation (see kPromote in gemm.cuh): the TMEM partial is
// promoted into fp32 registers every kPromoteGroup k-blocks (K = 64 each).
#ifndef LEMO_PROMOTE_GROUP
#define LEMO_PROMOTE_GROUP 2
#endif
constexpr int kPromoteGroup = LEMO_PROMOTE_GROUP;

template <int BN, class Epi>
static int gemm_promoted(const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                         const Epi& e, cudaStream_t st) {
  Bound<BN, Epi> b{e};
  if constexpr (BN == 256) {  // CTA pairs when M spans two row tiles (as gemm<256>)
    if (use_pair(M))
      return launch_gemm_tn_pair<Bound<BN, Epi>, kPromoteGroup>(A, lda, B, ldb, M, N, K, b, st);
  }
  return launch_gemm_tn<BN, Bound<BN, Epi>, false, kPromoteGroup>(A, lda, B, ldb, M, N, K, b, st);
}

template <class Epi>
static int gemm_auto(const void* A, int lda, const void* B, int ldb, int M, int N, int K,
                     const Epi& e, cudaStream_t st) {
  switch (pick_bn(M, N)) {
    case 256: return gemm<256>(A, lda, B, ldb, M, N, K, e, st);
    case 128: return gemm<128>(A, lda, B, ldb, M, N, K, e, st);
    default: return gemm<64>(A, lda, B, ldb, M, N, K, e, st);
  }
}

}  // namespace lemo

using namespace lemo;

extern "C" {

int lemo_gemm_bf16(const void* A, int lda, const void* B, int ldb, void* C, int ldc, int M, int N,
                   int K, void* stream) {
  LEMO_ARG_CHECK(N % 32 == 0 && ldc % 8 == 0, "lemo_gemm_bf16: N and ldc must be multiples of 32/8");
  EpiStoreBF16 e{reinterpret_cast<__nv_bfloat16*>(C), ldc, N};
  LEMO_RETURN_RC("lemo_gemm_bf16", gemm_auto(A, lda, B, ldb, M, N, K, e, (cudaStream_t)stream));
}

int lemo_gemm_nn_bf16(const void* A, int lda, const void* B, int ldb, void* C, int ldc, int M,
                      int N, int K, void* stream) {
  LEMO_ARG_CHECK(N % 32 == 0 && ldc % 8 == 0, "lemo_gemm_nn_bf16: N%32, ldc%8");
  Bound<256, EpiStoreBF16> b{EpiStoreBF16{reinterpret_cast<__nv_bfloat16*>(C), ldc, N}};
  LEMO_RETURN_RC("lemo_gemm_nn_bf16", (launch_gemm_tn<256, Bound<256, EpiStoreBF16>, true>(
                                          A, lda, B, ldb, M, N, K, b, (cudaStream_t)stream)));
}

int lemo_gemm_f32(const void* A, int lda, const void* B, int ldb, float* C, int ldc, int M, int N,
                  int K, int accumulate, void* stream) {
  EpiStoreF32 e{C, ldc, N, accumulate};
  LEMO_RETURN_RC("lemo_gemm_f32", gemm_auto(A, lda, B, ldb, M, N, K, e, (cudaStream_t)stream));
}

int lemo_gemm_f32_exact(const void* A, int lda, const void* B, int ldb, float* C, int ldc, int M,
                        int N, int K, int accumulate, void* stream) {
  EpiStoreF32 e{C, ldc, N, accumulate};
  cudaStream_t st = (cudaStream_t)stream;
  int rc;
  switch (pick_bn(M, N)) {
    case 256: rc = gemm_promoted<256>(A, lda, B, ldb, M, N, K, e, st); break;
    case 128: rc = gemm_promoted<128>(A, lda, B, ldb, M, N, K, e, st); break;
    default: rc = gemm_promoted<64>(A, lda, B, ldb, M, N, K, e, st); break;
  }
  LEMO_RETURN_RC("lemo_gemm_f32_exact", rc);
}

int lemo_gemm_scatter_add(const void* A, int lda, const void* B, int ldb, float* R, int ldr,
                          const int* idx, int M, int N, int K, void* stream) {
  LEMO_ARG_CHECK(N % 32 == 0 && ldr % 4 == 0, "lemo_gemm_scatter_add: N%32, ldr%4");
  EpiScatterAdd e{R, ldr, N, idx};
  cudaStream_t st = (cudaStream_t)stream;
  if (pick_bn(M, N) == 256 && use_pair(M)) {
    // CTA-pair tiles with the deferred split-K tail: a last wave that is at
    // most half full runs as K-range units, finished by a second small kernel
    PairTail tl{};
    int rc = launch_gemm_tn_pair(A, lda, B, ldb, M, N, K, Bound<256, EpiScatterAdd>{e}, st, &tl);
    if (!rc && tl.split > 1) {
      const int num_m = (M + 2 * kBlockM - 1) / (2 * kBlockM), num_n = (N + 255) / 256;
      const int rem = num_m * num_n - tl.full_tiles;
      scatter_tail_finish_kernel<<<rem * 128, 128, 0, st>>>(tl, num_m, num_n, M, N, R, ldr, idx);
      rc = (int)cudaGetLastError();
    }
    LEMO_RETURN_RC("lemo_gemm_scatter_add", rc);
  }
  LEMO_RETURN_RC("lemo_gemm_scatter_add", gemm_auto(A, lda, B, ldb, M, N, K, e, st));
}

int lemo_gemm_qkv(const void* xn, int ldx, const void* w_qkv_t, int ldw, int M, int h, int kv,
                  int K, int nmat, void* q, void* k, void* v, int head_dim, int rope,
                  const double* inv_freq, const int* pos, const float* row_scale, void* stream) {
  LEMO_ARG_CHECK(head_dim % 64 == 0, "lemo_gemm_qkv: head_dim must be a multiple of 64");
  LEMO_ARG_CHECK(nmat == 2 || nmat == 3, "lemo_gemm_qkv: nmat must be 2 (q,k) or 3 (q,k,v)");
  LEMO_ARG_CHECK(kv > 0 && kv <= h && kv % head_dim == 0, "lemo_gemm_qkv: bad k/v width");
  EpiQKV e{reinterpret_cast<__nv_bfloat16*>(q), reinterpret_cast<__nv_bfloat16*>(k),
           reinterpret_cast<__nv_bfloat16*>(v), h, kv, head_dim, rope, inv_freq, pos, row_scale};
  const int N = h + (nmat - 1) * kv;
  int rc;
  if (h % 256 == 0 && kv % 256 == 0 && 256 % head_dim == 0)
    rc = gemm<256>(xn, ldx, w_qkv_t, ldw, M, N, K, e, (cudaStream_t)stream);
  else if (h % 128 == 0 && kv % 128 == 0 && 128 % head_dim == 0)
    rc = gemm<128>(xn, ldx, w_qkv_t, ldw, M, N, K, e, (cudaStream_t)stream);
  else {
    set_error_msg("lemo_gemm_qkv: hidden dim must be a multiple of 128 and of head_dim");
    return LEMO_ERR_REPORTED;
  }
  LEMO_RETURN_RC("lemo_gemm_qkv", rc);
}

int lemo_gemm_gateup(const void* xn, int ldx, const void* w_gu_t, int M, int N, int K, void* gu,
                     void* inner, float* partial, int relu, int exact_score,
                     const float* row_scale, void* stream) {
  LEMO_ARG_CHECK(N % 256 == 0, "lemo_gemm_gateup: N must be a multiple of 256 (padded mlp dim)");
  auto* gup = reinterpret_cast<__nv_bfloat16*>(gu);
  auto* inp = reinterpret_cast<__nv_bfloat16*>(inner);
  const int ldi = relu ? N : N / 2;
  cudaStream_t st = (cudaStream_t)stream;
  if (exact_score) {  // parity mode: bf16x3 operands, promoted accumulation
    EpiGateUpExact e{gup, N, inp, ldi, partial, M, relu, row_scale};
    LEMO_RETURN_RC("lemo_gemm_gateup", gemm_promoted<256>(xn, ldx, w_gu_t, K, M, N, K, e, st));
  }
  EpiGateUp e{gup, N, inp, ldi, partial, M, relu, row_scale};
  LEMO_RETURN_RC("lemo_gemm_gateup", gemm<256>(xn, ldx, w_gu_t, K, M, N, K, e, st));
}

int lemo_gemm_split3(const void* A, int lda, const void* B, int ldb, int M, int N, int K3,
                     int relu, const unsigned char* mask, int pattern, void* out, int ldo,
                     float* f32, int ldf, void* stream) {
  LEMO_ARG_CHECK(K3 % 3 == 0, "lemo_gemm_split3: K' must be 3K");
  EpiSplit3 e{reinterpret_cast<__nv_bfloat16*>(out), ldo, f32, ldf, N, pattern, relu, mask};
  // small in M (n_blocks): BN = 128 or 64 so the grid fills the SMs; fp32-faithful
  // operands, so the accumulation is promoted (gemm.cuh kPromote)
  cudaStream_t st = (cudaStream_t)stream;
  const int rc = pick_bn(M, N) == 64 ? gemm_promoted<64>(A, lda, B, ldb, M, N, K3, e, st)
                                     : gemm_promoted<128>(A, lda, B, ldb, M, N, K3, e, st);
  LEMO_RETURN_RC("lemo_gemm_split3", rc);
}

int lemo_gemm_split3_dual(const void* A, int lda, const void* B, int ldb, int M, int N, int K3,
                          int nsplit, int relu, const unsigned char* mask, void* out, int ldo,
                          void* out2, int ldo2, void* stream) {
  LEMO_ARG_CHECK(K3 % 3 == 0, "lemo_gemm_split3_dual: K' must be 3K");
  LEMO_ARG_CHECK(nsplit > 0 && nsplit < N && nsplit % 32 == 0,
                 "lemo_gemm_split3_dual: 0 < nsplit < N, nsplit % 32 == 0");
  EpiSplit3 e{reinterpret_cast<__nv_bfloat16*>(out), ldo, nullptr, 0, N, 0, relu, mask,
              reinterpret_cast<__nv_bfloat16*>(out2), ldo2, nsplit};
  // both first layers in one GEMM over the shared input: 256 x 256 CTA-pair
  // tiles read the [M, 3h] input and the stacked weights 4x / 2x less often
  // from L2 than two BN = 64 launches (the predictor GEMMs are L2-bound)
  cudaStream_t st = (cudaStream_t)stream;
  const int rc = use_pair(M) ? gemm_promoted<256>(A, lda, B, ldb, M, N, K3, e, st)
                             : gemm_promoted<128>(A, lda, B, ldb, M, N, K3, e, st);
  LEMO_RETURN_RC("lemo_gemm_split3_dual", rc);
}

int lemo_gemm_dgateup(const void* dy, const void* w_down, int M, int m_pad, int h, const void* gu,
                      void* dgu, int relu, void* stream) {
  LEMO_ARG_CHECK(m_pad % 128 == 0, "lemo_gemm_dgateup: padded mlp dim must be a multiple of 128");
  const int ldgu = relu ? m_pad : 2 * m_pad;
  EpiDGateUp e{reinterpret_cast<const __nv_bfloat16*>(gu), ldgu,
               reinterpret_cast<__nv_bfloat16*>(dgu), relu};
  int rc;
  if (m_pad % 256 == 0)
    rc = gemm<256>(dy, h, w_down, h, M, m_pad, h, e, (cudaStream_t)stream);
  else
    rc = gemm<128>(dy, h, w_down, h, M, m_pad, h, e, (cudaStream_t)stream);
  LEMO_RETURN_RC("lemo_gemm_dgateup", rc);
}

}  // extern "C"
