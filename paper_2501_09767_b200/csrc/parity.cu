// fp32-faithful scoring helpers (the "parity" precision of the scorers).
//
// Block selection is a `>=` against a threshold (sparsity.py:274-277), so a
// mask reproduces the reference's only if the scores carry the reference's
// f32 precision.  The production scorers run bf16 tensor-core operands; the
// parity path keeps every scoring operand as a bf16 hi/lo pair (bf16x3, see
// EpiSplit3 / the exact scorer) and the element-wise steps in fp32 with the
// reference's operation order:
//   rmsnorm_f32   model.py:333-335  x · inv · w, inv = 1/√(mean(x²) + eps)
//   qk_finish     model.py:338-353  q = xn·Wq + ((xn·A_q)·B_q)·s, then the
//                 rotate-half RoPE with the f64-derived cos/sin table cast to
//                 f32 (tensor.py:604-625), products and differences rounded
//                 separately (no FMA contraction, as NumPy evaluates them);
//                 emits the bf16 hi/lo split the exact scorer consumes
//   split_hilo    v -> (bf16(v), bf16(v - bf16(v)))
#include "common.cuh"
#include "lemo_internal.h"

namespace lemo {

__device__ __forceinline__ void split2(float v, __nv_bfloat16* hi, __nv_bfloat16* lo) {
  const __nv_bfloat16 h = __float2bfloat16_rn(v);
  *hi = h;
  *lo = __float2bfloat16_rn(v - __bfloat162float(h));
}

__global__ void __launch_bounds__(256) rmsnorm_f32_kernel(const float* __restrict__ x, int ldx,
                                                          const int* __restrict__ idx, int h,
                                                          const float* __restrict__ w,
                                                          float* __restrict__ out, int ldo,
                                                          float* __restrict__ inv_out) {
  __shared__ float red[8];
  const int row = blockIdx.x;
  const int src = idx ? __ldg(idx + row) : row;
  const float* xr = x + (size_t)src * ldx;
  float ss = 0.f;
  for (int c = threadIdx.x; c < h; c += blockDim.x) ss = fmaf(xr[c], xr[c], ss);
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  float tot = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) tot += red[i];
  const float inv = 1.f / sqrtf(tot / (float)h + 1e-6f);
  if (threadIdx.x == 0 && inv_out) inv_out[row] = inv;
  float* o = out + (size_t)row * ldo;
  for (int c = threadIdx.x; c < h; c += blockDim.x) o[c] = __fmul_rn(__fmul_rn(xr[c], inv), w[c]);
}

// one thread per rotation pair (row, head, j < half) of q (heads [0, H)) and
// k (heads [H, H + Hk)); without RoPE the pair is just two independent columns
__global__ void __launch_bounds__(256) qk_finish_kernel(
    const float* __restrict__ qk, int ldqk, const float* __restrict__ t, int ldt,
    const float* __restrict__ Bq, int r, float scale, const float* __restrict__ rope_tab, int s,
    int h, int kv, int D, int rope, __nv_bfloat16* __restrict__ q_hi,
    __nv_bfloat16* __restrict__ q_lo, __nv_bfloat16* __restrict__ k_hi,
    __nv_bfloat16* __restrict__ k_lo) {
  const int half = D >> 1;
  const int pairs_row = (h + kv) >> 1;
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)s * pairs_row) return;
  const int row = (int)(gid / pairs_row);
  const int p = (int)(gid - (long long)row * pairs_row);
  const bool is_q = p < (h >> 1);
  const int pp = is_q ? p : p - (h >> 1);
  const int head = pp / half, j = pp - head * half;
  const int ca = head * D + j, cb = ca + half;  // column inside q or k
  const float* src = qk + (size_t)row * ldqk + (is_q ? 0 : h);
  float a = src[ca], b = src[cb];
  if (is_q && Bq != nullptr) {
    // ((xn·A)·B)·scaling added to xn·W (model.py:338-342)
    const float* tr = t + (size_t)row * ldt;
    float la = 0.f, lb = 0.f;
    for (int i = 0; i < r; ++i) {
      la = fmaf(tr[i], Bq[(size_t)i * h + ca], la);
      lb = fmaf(tr[i], Bq[(size_t)i * h + cb], lb);
    }
    a = __fadd_rn(a, __fmul_rn(la, scale));
    b = __fadd_rn(b, __fmul_rn(lb, scale));
  }
  if (rope) {
    const float c = rope_tab[((size_t)row * half + j) * 2];
    const float sn = rope_tab[((size_t)row * half + j) * 2 + 1];
    const float na = __fsub_rn(__fmul_rn(a, c), __fmul_rn(b, sn));
    const float nb = __fadd_rn(__fmul_rn(a, sn), __fmul_rn(b, c));
    a = na;
    b = nb;
  }
  const int ld = is_q ? h : kv;
  __nv_bfloat16* hi = is_q ? q_hi : k_hi;
  __nv_bfloat16* lo = is_q ? q_lo : k_lo;
  split2(a, hi + (size_t)row * ld + ca, lo + (size_t)row * ld + ca);
  split2(b, hi + (size_t)row * ld + cb, lo + (size_t)row * ld + cb);
}

// [hi | lo] rows (K' = 2K): the A operand of x_hi·W + x_lo·W for bf16-exact W
__global__ void split_bf16x2_kernel(const float* __restrict__ a, int lda, int M, int K,
                                    __nv_bfloat16* __restrict__ out) {
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)M * K) return;
  const int row = (int)(gid / K), c = (int)(gid - (long long)row * K);
  __nv_bfloat16* o = out + (size_t)row * 2 * K;
  split2(a[(size_t)row * lda + c], o + c, o + K + c);
}

__global__ void split_hilo_kernel(const float* __restrict__ a, int lda, int M, int K,
                                  __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
  const long long gid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (gid >= (long long)M * K) return;
  const int row = (int)(gid / K), c = (int)(gid - (long long)row * K);
  split2(a[(size_t)row * lda + c], hi + (size_t)row * K + c, lo + (size_t)row * K + c);
}

}  // namespace lemo

using namespace lemo;

extern "C" {

int lemo_rmsnorm_f32(const float* x, int ldx, const int* idx, int M, int h, const float* w,
                     float* out, int ldo, float* inv, void* stream) {
  if (M <= 0) return 0;
  LEMO_ARG_CHECK(ldo >= h && ldx >= h, "lemo_rmsnorm_f32: bad row strides");
  rmsnorm_f32_kernel<<<M, 256, 0, (cudaStream_t)stream>>>(x, ldx, idx, h, w, out, ldo, inv);
  LEMO_CHECK_LAUNCH("lemo_rmsnorm_f32");
  return 0;
}

int lemo_qk_finish(const float* qk, int ldqk, const float* t, int ldt, const float* Bq, int r,
                   float scale, const float* rope_tab, int s, int h, int kv, int head_dim,
                   int rope, void* q_hi, void* q_lo, void* k_hi, void* k_lo, void* stream) {
  if (s <= 0) return 0;
  LEMO_ARG_CHECK(head_dim % 2 == 0 && h % head_dim == 0 && kv % head_dim == 0,
                 "lemo_qk_finish: bad head geometry");
  LEMO_ARG_CHECK(!rope || rope_tab != nullptr, "lemo_qk_finish: RoPE needs the cos/sin table");
  const long long total = (long long)s * ((h + kv) / 2);
  qk_finish_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      qk, ldqk, t, ldt, Bq, r, scale, rope_tab, s, h, kv, head_dim, rope,
      reinterpret_cast<__nv_bfloat16*>(q_hi), reinterpret_cast<__nv_bfloat16*>(q_lo),
      reinterpret_cast<__nv_bfloat16*>(k_hi), reinterpret_cast<__nv_bfloat16*>(k_lo));
  LEMO_CHECK_LAUNCH("lemo_qk_finish");
  return 0;
}

int lemo_split_bf16x2(const float* a, int lda, int M, int K, void* out, void* stream) {
  const long long total = (long long)M * K;
  if (total == 0) return 0;
  split_bf16x2_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      a, lda, M, K, reinterpret_cast<__nv_bfloat16*>(out));
  LEMO_CHECK_LAUNCH("lemo_split_bf16x2");
  return 0;
}

int lemo_split_hilo(const float* a, int lda, int M, int K, void* hi, void* lo, void* stream) {
  const long long total = (long long)M * K;
  if (total == 0) return 0;
  split_hilo_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      a, lda, M, K, reinterpret_cast<__nv_bfloat16*>(hi), reinterpret_cast<__nv_bfloat16*>(lo));
  LEMO_CHECK_LAUNCH("lemo_split_hilo");
  return 0;
}

}  // extern "C"
