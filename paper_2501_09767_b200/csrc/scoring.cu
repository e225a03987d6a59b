// Pattern scoring and selection kernels (K1/K2 of the design):
//   block_embed      predictor.py:117-123 (block mean of the residual stream)
//   (the predictor GEMMs and Eq. 3 are fp32-faithful bf16x3 tcgen05 GEMMs with
//    promoted accumulation, gemm_ops.cu / gemm.cuh)
//   pack_tril        sparsity.py:35-69 packed lower triangle (+ clamp)
//   colsum_clamped   model.py:575-578 + sparsity.py:253-260 (clamp ≥ 0, f64
//                    column sums accumulated in ascending query block)
//   mlp_block_scores sparsity.py:284-305 (mean |inner| per token, block max)
//   select           sparsity.py:263-281 + 95-104 (>= threshold, sink force,
//                    block → token compaction; k stays on device)
//   quantile_lower   model.py:545-563 (np.quantile method="lower" as a radix
//                    select over order-preserving 64-bit keys)
#include <algorithm>

#include "common.cuh"
#include "lemo_internal.h"

namespace lemo {

// --------------------------------------------------------------------------
// block mean: one thread per (block, 4 columns); b independent float4 loads in
// flight per thread, sequential f32 sum in row order then / b — the same
// arithmetic numpy uses for mean over a non-contiguous axis.
// One CTA per token block: the b rows of the block are contiguous in HBM
// (b·h·4 bytes), so every CTA streams one contiguous region; each thread
// keeps b independent 16-B loads in flight (first batch issued before any add).
template <int B>
__global__ void __launch_bounds__(1024) block_embed_kernel(const float* __restrict__ x, int ldx,
                                                           int h, float* __restrict__ xb) {
  const int n = blockIdx.x;
  const int nv = h >> 2;
  const float4* base = reinterpret_cast<const float4*>(x + (size_t)n * B * ldx);
  const size_t stride = (size_t)ldx >> 2;
  for (int c = threadIdx.x; c < nv; c += blockDim.x) {
    float4 v[B];
#pragma unroll
    for (int i = 0; i < B; ++i) v[i] = __ldcs(base + i * stride + c);
    float4 acc = v[0];
#pragma unroll
    for (int i = 1; i < B; ++i) {
      acc.x += v[i].x; acc.y += v[i].y; acc.z += v[i].z; acc.w += v[i].w;
    }
    const float fb = (float)B;
    acc.x /= fb; acc.y /= fb; acc.z /= fb; acc.w /= fb;
    reinterpret_cast<float4*>(xb + (size_t)n * h)[c] = acc;
  }
}

__global__ void __launch_bounds__(256) block_embed_generic_kernel(const float* __restrict__ x,
                                                                  int ldx, int nb, int h, int b,
                                                                  float* __restrict__ xb) {
  const int nv = h >> 2;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)nb * nv) return;
  const int n = (int)(gid / nv), c = (int)(gid - (long long)n * nv);
  const float4* src = reinterpret_cast<const float4*>(x + (size_t)n * b * ldx) + c;
  const size_t stride = (size_t)ldx >> 2;
  float4 acc = __ldg(src);
  for (int i = 1; i < b; ++i) {
    const float4 v = __ldg(src + i * stride);
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  const float fb = (float)b;
  acc.x /= fb; acc.y /= fb; acc.z /= fb; acc.w /= fb;
  reinterpret_cast<float4*>(xb + (size_t)n * h)[c] = acc;
}

// vec[n] = Σ_{m=n}^{nb-1} (double)max(S[m,n], 0), ascending m (sparsity.py:256-259)
// One warp per column: the 32 lanes fetch 32 consecutive query blocks at once
// (all loads in flight), then the warp adds them in ascending m order through
// shuffles — the reference's exact f64 summation order, without its latency.
__global__ void colsum_clamped_kernel(const float* __restrict__ S, int lds, int nb,
                                      double* __restrict__ vec) {
  const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (n >= nb) return;
  double acc = 0.0;
  int m0 = n;
  float cur = m0 + lane < nb ? S[(size_t)(m0 + lane) * lds + n] : 0.f;
  while (m0 < nb) {
    const int m1 = m0 + 32;
    const float nxt = m1 + lane < nb ? S[(size_t)(m1 + lane) * lds + n] : 0.f;  // prefetch
    const double v = (double)fmaxf(cur, 0.f);
    const int cnt = min(32, nb - m0);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double x = __shfl_sync(0xffffffffu, v, j);
      if (j < cnt) acc += x;
    }
    cur = nxt;
    m0 = m1;
  }
  if (lane == 0) vec[n] = acc;
}

// Refined MLP scoring (scoring_precision "refined"): bf16 scores first, then
// only the rows that can decide a near-threshold block re-scored in the
// parity precision.  A block's decision is max_t score_t >= T, so inside
// a block whose bf16 score is within `margin` of T only the rows whose own
// bf16 token score is >= T - margin can decide it (a row below that cannot
// reach T under the same error bound); out[row] = 0 marks those rows (select
// with thr = 0, block size 1, compacts them in ascending order), -1 the rest.
__global__ void mlp_token_band_kernel(const float* __restrict__ partial, int n_tiles, int s,
                                      int n_valid, int b, float m_real,
                                      const double* __restrict__ vec, double thr, double margin,
                                      double* __restrict__ out) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= s) return;
  double o = -1.0;
  if (row < n_valid && fabs(__ldg(vec + row / b) - thr) <= margin) {
    float acc = 0.f;  // the token score exactly as mlp_block_scores forms it
    for (int t = 0; t < n_tiles; ++t) acc += partial[(size_t)t * s + row];
    if ((double)(acc / m_real) >= thr - margin) o = 0.0;
  }
  out[row] = o;
}

// vec[tok[i] / b] = max over the re-scored rows of that block (rows ascending,
// so a block's rows are contiguous).  One warp per compact row i; the warp of
// a block's first row reduces the block: lane l sums row i + l (the tile
// order of mlp_block_scores) and the maximum is a warp shuffle (b <= 32).
// count (optional): the number of valid rows when the GEMM ran on a capacity
// of `rows` (rows past the count are padding); *overflow = count > rows.
__global__ void mlp_patch_rows_kernel(const float* __restrict__ partial, int n_tiles, int rows,
                                      const int* __restrict__ tok, const int* __restrict__ count,
                                      int b, float m_real, double* __restrict__ vec,
                                      int* __restrict__ overflow) {
  const int i = (int)((blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int n = count ? min(__ldg(count), rows) : rows;
  if (overflow && blockIdx.x == 0 && threadIdx.x == 0) *overflow = count && __ldg(count) > rows;
  if (i >= n) return;
  const int blk = __ldg(tok + i) / b;
  if (i > 0 && __ldg(tok + i - 1) / b == blk) return;  // warp-uniform
  const int j = i + lane;
  float best = -INFINITY;
  if (j < n && __ldg(tok + j) / b == blk) {  // (partial rows are strided by `rows`)
    float acc = 0.f;
#pragma unroll 8
    for (int t = 0; t < n_tiles; ++t) acc += partial[(size_t)t * rows + j];
    best = acc / m_real;
  }
  for (int o = 16; o > 0; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
  if (lane == 0) vec[blk] = (double)best;
}

// Row-major packed lower triangle of a dense [nb, nb] fp32 matrix (element
// (m, n <= m) at m(m+1)/2 + n, sparsity.py:35-37), optionally clamped at 0
// (predict_scores, predictor.py:189-212), as f64 (BlockScoreMatrix) or f32.
__global__ void pack_tril_kernel(const float* __restrict__ S, int lds, int nb, int clamp,
                                 double* __restrict__ out64, float* __restrict__ out32) {
  const int m = blockIdx.x;
  const size_t base = (size_t)m * (m + 1) / 2;
  for (int n = threadIdx.x; n <= m; n += blockDim.x) {
    float v = S[(size_t)m * lds + n];
    if (clamp) v = fmaxf(v, 0.f);
    if (out64) out64[base + n] = (double)v;
    else out32[base + n] = v;
  }
}

// Same column sums straight from a packed f64 lower triangle (element (m, n)
// at m(m+1)/2 + n), e.g. reference-written or teacher score triangles.
__global__ void colsum_packed_kernel(const double* __restrict__ P, int nb,
                                     double* __restrict__ vec) {
  const int n = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (n >= nb) return;
  double acc = 0.0;
  for (int m0 = n; m0 < nb; m0 += 32) {
    const int m = m0 + lane;
    const double v = m < nb ? P[(size_t)m * (m + 1) / 2 + n] : 0.0;
    const int cnt = min(32, nb - m0);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double x = __shfl_sync(0xffffffffu, v, j);
      if (j < cnt) acc += x;
    }
  }
  if (lane == 0) vec[n] = acc;
}

// Token scores (one thread per row, coalesced over the per-tile partials, the
// same sequential tile order as before) and the block max via segmented warp
// shuffles (b a power of two <= 32).
__global__ void mlp_block_scores_warp_kernel(const float* __restrict__ partial, int n_tiles,
                                             int s, int n_valid, int b, float m_real,
                                             double* __restrict__ vec) {
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  const int lim = min(s, n_valid);
  float best = -INFINITY;
  if (row < lim) {
    float acc = 0.f;
    for (int t = 0; t < n_tiles; ++t) acc += partial[(size_t)t * s + row];
    best = acc / m_real;
  }
  for (int o = b >> 1; o > 0; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((row % b) == 0 && row < s) vec[row / b] = best == -INFINITY ? 0.0 : (double)best;
}

__global__ void mlp_block_scores_kernel(const float* __restrict__ partial, int n_tiles, int s,
                                        int n_valid, int b, float m_real,
                                        double* __restrict__ vec) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  const int nb = (s + b - 1) / b;
  if (n >= nb) return;
  const int t0 = n * b;
  const int t1 = min(min(t0 + b, s), n_valid);
  double best = 0.0;
  bool any = false;
  for (int row = t0; row < t1; ++row) {
    float acc = 0.f;
    for (int t = 0; t < n_tiles; ++t) acc += partial[(size_t)t * s + row];
    const double tok = (double)(acc / m_real);
    best = any ? fmax(best, tok) : tok;
    any = true;
  }
  vec[n] = any ? best : 0.0;
}

// --------------------------------------------------------------------------
// selection: one CTA; keep n iff vec[n] >= T (or forced sink block 0);
// blocks/tokens compacted in ascending order via a block-wide scan.
constexpr int kSelThreads = 1024;
__global__ void __launch_bounds__(kSelThreads) select_kernel(
    const double* __restrict__ vec, int nb, double thr, const double* __restrict__ thr_dev,
    const unsigned char* __restrict__ force, int b, int n_tokens, unsigned char* __restrict__ mask, int* __restrict__ blocks,
    int* __restrict__ tokens, int* __restrict__ counts, double* __restrict__ thr_out) {
  __shared__ int scan[kSelThreads];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  const double T = thr_dev ? *thr_dev : thr;
  const int per = (nb + kSelThreads - 1) / kSelThreads;
  const int start = min(tid * per, nb), end = min(start + per, nb);
  int cnt = 0;
  bool nonfinite = false;
  for (int n = start; n < end; ++n) {
    const double v = vec[n];
    if (!isfinite(v)) nonfinite = true;
    const bool keep = (v >= T) || (force && force[n]);
    mask[n] = keep ? 1 : 0;
    cnt += keep;
  }
  __syncthreads();
  if (nonfinite) atomicOr(&bad, 1);
  scan[tid] = cnt;
  __syncthreads();
  for (int o = 1; o < kSelThreads; o <<= 1) {
    const int v = tid >= o ? scan[tid - o] : 0;
    __syncthreads();
    scan[tid] += v;
    __syncthreads();
  }
  int off = scan[tid] - cnt;
  for (int n = start; n < end; ++n) {
    if (!mask[n]) continue;
    blocks[off] = n;
    const int t0 = n * b, t1 = min(t0 + b, n_tokens);
    for (int t = t0; t < t1; ++t) tokens[off * b + (t - t0)] = t;
    ++off;
  }
  if (tid == kSelThreads - 1) {
    const int total = scan[tid];
    const int short_tail = (nb > 0 && mask[nb - 1]) ? nb * b - n_tokens : 0;
    counts[0] = total * b - short_tail;
    counts[1] = total;
  }
  __syncthreads();
  if (tid == 0) {
    counts[2] = bad;
    if (thr_out) *thr_out = T;
  }
}

__device__ __forceinline__ unsigned long long f64_key(double x) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(x);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__device__ __forceinline__ double key_f64(unsigned long long k) {
  const unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}

__global__ void __launch_bounds__(1024) quantile_kernel(const double* __restrict__ data, int n,
                                                        long long rank, int plus_one,
                                                        double* __restrict__ out) {
  __shared__ unsigned int hist[256];
  __shared__ unsigned long long s_prefix, s_mask;
  __shared__ long long s_rank;
  if (threadIdx.x == 0) {
    s_prefix = 0;
    s_mask = 0;
    s_rank = rank;
  }
  __syncthreads();
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    const unsigned long long prefix = s_prefix, msk = s_mask;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const unsigned long long k = f64_key(data[i]);
      if ((k & msk) == prefix) atomicAdd(&hist[(k >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      long long r = s_rank;
      int d = 0;
      for (; d < 256; ++d) {
        if (r < (long long)hist[d]) break;
        r -= hist[d];
      }
      if (d > 255) d = 255;
      s_rank = r;
      s_prefix = prefix | ((unsigned long long)d << shift);
      s_mask = msk | (255ull << shift);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double v = key_f64(s_prefix);
    if (plus_one) v += 1.0;
    *out = v;
  }
}

// fp32 -> bf16x3 operand ([hi|hi|lo] pattern 0, [hi|lo|hi] pattern 1), see EpiSplit3.
__global__ void split_bf16x3_kernel(const float* __restrict__ A, int lda, int M, int K,
                                    int pattern, __nv_bfloat16* __restrict__ out) {
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)M * K) return;
  const int row = (int)(gid / K), c = (int)(gid - (long long)row * K);
  const float v = A[(size_t)row * lda + c];
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
  __nv_bfloat16* o = out + (size_t)row * 3 * K;
  o[c] = hi;
  o[K + c] = pattern ? lo : hi;
  o[2 * K + c] = pattern ? hi : lo;
}

}  // namespace lemo

using namespace lemo;

extern "C" {

int lemo_block_embed(const float* x, int ldx, int s, int h, int b, float* xb, void* stream) {
  LEMO_ARG_CHECK(b > 0 && s % b == 0, "lemo_block_embed: s must be a multiple of the block size");
  LEMO_ARG_CHECK(h % 4 == 0 && ldx % 4 == 0, "lemo_block_embed: h, ldx multiples of 4");
  const int nb = s / b;
  const long long total = (long long)nb * (h / 4);
  if (total == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const int threads = std::min(1024, std::max(32, ((h / 4 + 31) / 32) * 32));
  if (b == 16)
    block_embed_kernel<16><<<nb, threads, 0, st>>>(x, ldx, h, xb);
  else if (b == 8)
    block_embed_kernel<8><<<nb, threads, 0, st>>>(x, ldx, h, xb);
  else
    block_embed_generic_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(x, ldx, nb, h, b,
                                                                               xb);
  LEMO_CHECK_LAUNCH("lemo_block_embed");
  return 0;
}

int lemo_split_bf16x3(const float* A, int lda, int M, int K, int pattern, void* out,
                      void* stream) {
  const long long total = (long long)M * K;
  if (total == 0) return 0;
  split_bf16x3_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      A, lda, M, K, pattern, reinterpret_cast<__nv_bfloat16*>(out));
  LEMO_CHECK_LAUNCH("lemo_split_bf16x3");
  return 0;
}

int lemo_colsum_clamped(const float* S, int lds, int nb, double* vec, void* stream) {
  if (nb <= 0) return 0;
  colsum_clamped_kernel<<<(nb + 7) / 8, 256, 0, (cudaStream_t)stream>>>(S, lds, nb, vec);
  LEMO_CHECK_LAUNCH("lemo_colsum_clamped");
  return 0;
}

int lemo_mlp_token_band(const float* partial, int n_tiles, int s, int n_valid, int b, int m_real,
                        const double* vec, double thr, double margin, double* out, void* stream) {
  if (s <= 0) return 0;
  LEMO_ARG_CHECK(b > 0, "lemo_mlp_token_band: block size must be positive");
  mlp_token_band_kernel<<<(s + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      partial, n_tiles, s, n_valid, b, (float)m_real, vec, thr, margin, out);
  LEMO_CHECK_LAUNCH("lemo_mlp_token_band");
  return 0;
}

int lemo_mlp_patch_rows(const float* partial, int n_tiles, int rows, const int* tok,
                        const int* count, int b, int m_real, double* vec, int* overflow,
                        void* stream) {
  if (rows <= 0) return 0;
  LEMO_ARG_CHECK(b > 0 && b <= 32, "lemo_mlp_patch_rows: block size must be in [1, 32]");
  mlp_patch_rows_kernel<<<(unsigned)((rows * 32LL + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      partial, n_tiles, rows, tok, count, b, (float)m_real, vec, overflow);
  LEMO_CHECK_LAUNCH("lemo_mlp_patch_rows");
  return 0;
}

int lemo_pack_tril(const float* S, int lds, int nb, int clamp, double* out64, float* out32,
                   void* stream) {
  if (nb <= 0) return 0;
  LEMO_ARG_CHECK((out64 == nullptr) != (out32 == nullptr), "lemo_pack_tril: exactly one output");
  pack_tril_kernel<<<nb, 128, 0, (cudaStream_t)stream>>>(S, lds, nb, clamp, out64, out32);
  LEMO_CHECK_LAUNCH("lemo_pack_tril");
  return 0;
}

int lemo_colsum_packed(const double* packed, int nb, double* vec, void* stream) {
  if (nb <= 0) return 0;
  colsum_packed_kernel<<<(nb + 7) / 8, 256, 0, (cudaStream_t)stream>>>(packed, nb, vec);
  LEMO_CHECK_LAUNCH("lemo_colsum_packed");
  return 0;
}

int lemo_mlp_block_scores(const float* partial, int n_tiles, int s, int n_valid, int b, int m_real,
                          double* vec, void* stream) {
  const int nb = (s + b - 1) / b;
  if (nb <= 0) return 0;
  if (b <= 32 && (b & (b - 1)) == 0) {
    const long long rows = (long long)nb * b;
    mlp_block_scores_warp_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
        partial, n_tiles, s, n_valid, b, (float)m_real, vec);
  } else {
    mlp_block_scores_kernel<<<(nb + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
        partial, n_tiles, s, n_valid, b, (float)m_real, vec);
  }
  LEMO_CHECK_LAUNCH("lemo_mlp_block_scores");
  return 0;
}

int lemo_select(const double* vec, int nb, double thr, const double* thr_dev,
                const unsigned char* force, int b,
                int n_tokens, unsigned char* mask, int* blocks, int* tokens, int* counts,
                double* thr_out, void* stream) {
  LEMO_ARG_CHECK(nb == (n_tokens + b - 1) / b, "lemo_select: nb must equal ceil(n_tokens / b)");
  select_kernel<<<1, kSelThreads, 0, (cudaStream_t)stream>>>(vec, nb, thr, thr_dev, force, b,
                                                            n_tokens, mask, blocks, tokens,
                                                            counts, thr_out);
  LEMO_CHECK_LAUNCH("lemo_select");
  return 0;
}

int lemo_quantile_lower(const double* data, int n, long long rank, int plus_one, double* out,
                        void* stream) {
  LEMO_ARG_CHECK(n > 0 && rank >= 0 && rank < n, "lemo_quantile_lower: rank out of range");
  quantile_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(data, n, rank, plus_one, out);
  LEMO_CHECK_LAUNCH("lemo_quantile_lower");
  return 0;
}

}  // extern "C"
