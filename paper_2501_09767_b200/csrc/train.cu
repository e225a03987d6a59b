// Kernels of the offline predictor-training stage (predictor.py:215-433,
// fit_predictors): everything around the fp32-faithful bf16x3 tcgen05 GEMMs
// (gemm_ops.cu:EpiSplit3) that the forward and backward of the three-matrix
// predictors and of Eq. 3 are built from.
//
//   split_bf16x3_t   bf16x3 operand of Aᵀ (the K-major form of a transposed
//                    matrix: weight gradients are Xᵀ·dY products)
//   tril_mse         log1p-MSE of the packed lower triangle (tensor.py:495-505):
//                    per-row loss partials and the lower-triangular dL/dFull
//   relu_grad        dpre = dh · [h > 0] (ReLU·mask backward)
//   zero_count       per-neuron exact-zero counters (predictor.py:76-80, track=True)
#include "common.cuh"
#include "lemo_internal.h"

namespace lemo {

// out[c, :] = split(A[:, c]) : [C, 3R] from fp32 A [R, C] (32 x 32 smem tiles).
__global__ void __launch_bounds__(256) split_bf16x3_t_kernel(const float* __restrict__ A, int lda,
                                                             int R, int C, int pattern,
                                                             __nv_bfloat16* __restrict__ out) {
  __shared__ float t[32][33];
  const int r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    t[i][threadIdx.x] = (r < R && c < C) ? A[(size_t)r * lda + c] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (c >= C || r >= R) continue;
    const float v = t[threadIdx.x][i];
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    const __nv_bfloat16 lo = __float2bfloat16_rn(v - __bfloat162float(hi));
    __nv_bfloat16* o = out + (size_t)c * 3 * R;
    o[r] = hi;
    o[R + r] = pattern ? lo : hi;
    o[2 * R + r] = pattern ? hi : lo;
  }
}

// Row m of the nb x nb prediction: d = full[m, n] - label[m(m+1)/2 + n] for
// n <= m; dfull[m, n] = 2 d / T (0 above the diagonal); row_loss[m] = Σ d²
// (f64, fixed reduction order).  T = nb(nb+1)/2 packed elements.
__global__ void __launch_bounds__(256) tril_mse_kernel(const float* __restrict__ full, int ldf,
                                                       const float* __restrict__ label, int nb,
                                                       float inv_t2, float* __restrict__ dfull,
                                                       int ldd, double* __restrict__ row_loss) {
  __shared__ double red[8];
  const int m = blockIdx.x;
  const size_t base = (size_t)m * (m + 1) / 2;
  double acc = 0.0;
  for (int n = threadIdx.x; n < nb; n += blockDim.x) {
    float g = 0.f;
    if (n <= m) {
      const float d = full[(size_t)m * ldf + n] - label[base + n];
      acc += (double)d * (double)d;
      g = d * inv_t2;
    }
    dfull[(size_t)m * ldd + n] = g;
  }
  acc = warp_sum_d(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    row_loss[m] = s;
  }
}

__global__ void relu_grad_kernel(float* __restrict__ dh, const float* __restrict__ h, long long n) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < n && !(h[i] > 0.f)) dh[i] = 0.f;
}

// counts[c] += #{r : h[r, c] == 0}; one thread per column, rows streamed
// (coalesced across the warp), no atomics.
__global__ void zero_count_kernel(const float* __restrict__ h, int ldh, int M, int N,
                                  long long* __restrict__ counts) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  long long z = 0;
  for (int r = 0; r < M; ++r) z += h[(size_t)r * ldh + c] == 0.f;
  counts[c] += z;
}

// Backward of the per-block row mean (token pooling, predictor.py:126-135):
// out[i, :] = g[i / b, :] / b.
__global__ void block_expand_kernel(const float* __restrict__ g, int w, int b,
                                    float* __restrict__ out, long long total) {
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= total) return;
  const long long row = e / w, c = e - row * w;
  out[e] = g[(row / b) * w + c] / (float)b;
}

// out[slot] = Σ x (f64, one CTA, fixed order) — the per-record loss.
__global__ void sum_d_kernel(const double* __restrict__ x, int n, double scale,
                             double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    *out = t * scale;
  }
}

}  // namespace lemo

using namespace lemo;

extern "C" {

int lemo_split_bf16x3_t(const float* A, int lda, int R, int C, int pattern, void* out,
                        void* stream) {
  if (R <= 0 || C <= 0) return 0;
  dim3 grid((C + 31) / 32, (R + 31) / 32), block(32, 8);
  split_bf16x3_t_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(
      A, lda, R, C, pattern, reinterpret_cast<__nv_bfloat16*>(out));
  LEMO_CHECK_LAUNCH("lemo_split_bf16x3_t");
  return 0;
}

int lemo_tril_mse(const float* full, int ldf, const float* label, int nb, float* dfull, int ldd,
                  double* row_loss, void* stream) {
  if (nb <= 0) return 0;
  const double t = (double)nb * (nb + 1) / 2.0;
  tril_mse_kernel<<<nb, 256, 0, (cudaStream_t)stream>>>(full, ldf, label, nb, (float)(2.0 / t),
                                                        dfull, ldd, row_loss);
  LEMO_CHECK_LAUNCH("lemo_tril_mse");
  return 0;
}

int lemo_relu_grad(float* dh, const float* h, long long n, void* stream) {
  if (n <= 0) return 0;
  relu_grad_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(dh, h, n);
  LEMO_CHECK_LAUNCH("lemo_relu_grad");
  return 0;
}

int lemo_zero_count(const float* h, int ldh, int M, int N, long long* counts, void* stream) {
  if (M <= 0 || N <= 0) return 0;
  zero_count_kernel<<<(N + 127) / 128, 128, 0, (cudaStream_t)stream>>>(h, ldh, M, N, counts);
  LEMO_CHECK_LAUNCH("lemo_zero_count");
  return 0;
}

int lemo_block_expand(const float* g, int nb, int w, int b, float* out, void* stream) {
  const long long total = (long long)nb * b * w;
  if (total <= 0) return 0;
  block_expand_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      g, w, b, out, total);
  LEMO_CHECK_LAUNCH("lemo_block_expand");
  return 0;
}

int lemo_sum_d(const double* x, int n, double scale, double* out, void* stream) {
  sum_d_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(x, n, scale, out);
  LEMO_CHECK_LAUNCH("lemo_sum_d");
  return 0;
}

}  // extern "C"
