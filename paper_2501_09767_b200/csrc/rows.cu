// Row-wise HBM-bound kernels of the LeMo step: fused gather+RMSNorm (+LoRA
// x·A factors), residual gathers, RMSNorm backward with index-remapped
// scatter-add, MLP retained-row compaction, q/k/v gradient preparation (RoPE
// backward + LoRA factors), LoRA weight gradients, embedding, segmented
// cross-entropy rows, Adam.  One CTA (or warp) per row, float4/16-B vector
// accesses, no atomics on the residual stream (retained rows are disjoint).
#include "common.cuh"
#include "lemo_internal.h"

namespace lemo {

constexpr float kEps = 1e-6f;  // tensor.py:387

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) t += red[i];
  return t;
}

// ---------------------------------------------------------------------------
// gather_rmsnorm (tensor.py:578-597).  idx == null: every row.  (The LoRA
// down-projection t = xn·[A_q|A_v] runs as a tcgen05 GEMM on the bf16 xn;
// see lemo_lora_pack.)

// kFold: write bf16(x·w) instead of bf16(x·inv·w) and leave inv to the GEMM
// epilogue (row scale).  The product of a row with a per-row scalar rounds
// correlatedly when x is bf16-valued (embedding rows, rows a sparse block did
// not update): bf16(x_i·inv) errors stop averaging out across the K sum
// (measured 3.7e-3 vs 3.5e-4 relative MLP-score error); bf16(x·w) is exact
// for such rows and no worse for the rest.
template <int VPT, bool kFold = false>
__global__ void __launch_bounds__(128) gather_rmsnorm_kernel(
    const float* __restrict__ x, int ldx, const int* __restrict__ idx, int h,
    const float* __restrict__ w, __nv_bfloat16* __restrict__ xn, int ldxn,
    __nv_bfloat16* __restrict__ xg, float* __restrict__ inv_out) {
  __shared__ float red[4];
  const int row = blockIdx.x;
  const int src = idx ? __ldg(idx + row) : row;
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)src * ldx);
  const int nv = h >> 2;
  float4 v[VPT];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    v[i] = c < nv ? xr[c] : make_float4(0.f, 0.f, 0.f, 0.f);
    ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
  }
  ss = block_sum<128>(ss, red);
  const float inv = 1.f / sqrtf(ss / (float)h + kEps);
  if (threadIdx.x == 0 && inv_out) inv_out[row] = inv;
  const float4* w4 = reinterpret_cast<const float4*>(w);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c >= nv) continue;
    const float4 ww = __ldg(w4 + c);
    const float sc = kFold ? 1.f : inv;
    float4 o;
    o.x = v[i].x * sc * ww.x;
    o.y = v[i].y * sc * ww.y;
    o.z = v[i].z * sc * ww.z;
    o.w = v[i].w * sc * ww.w;
    uint2 ob = make_uint2(pack_bf16x2(o.x, o.y), pack_bf16x2(o.z, o.w));
    reinterpret_cast<uint2*>(xn + (size_t)row * ldxn)[c] = ob;
    if (xg) {
      reinterpret_cast<uint2*>(xg + (size_t)row * h)[c] =
          make_uint2(pack_bf16x2(v[i].x, v[i].y), pack_bf16x2(v[i].z, v[i].w));
    }
  }
}

// LoRA down-projection operand for the tcgen05 GEMM: out[j, c] = bf16(A[c*lda + j])
// for j < 2r (A = [A_q | A_v] interleaved [h, 2r]), zero rows up to 32.
__global__ void lora_pack_kernel(const float* __restrict__ A, int lda, int h, int r2,
                                 __nv_bfloat16* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= h) return;
#pragma unroll 4
  for (int j = 0; j < 32; ++j)
    out[(size_t)j * h + c] = __float2bfloat16_rn(j < r2 ? A[(size_t)c * lda + j] : 0.f);
}

// LoRA as a K-extension of the q/k/v GEMM (64 extra K columns):
//   A-side: xn_ext[i, h + j] = bf16(scale · t[i, j]) for j < 2r, 0 for 2r <= j < 64
//   B-side: w_ext[c, h + j]          = bf16(Bq[j, c])   (q rows, j < r)
//           w_ext[2h + c, h + r + j] = bf16(Bv[j, c])   (v rows, j < r), all else 0
__global__ void lora_qkv_prep_kernel(const float* __restrict__ t, int ldt, int M, int r2,
                                     float scale, __nv_bfloat16* __restrict__ xn, int ldx,
                                     int h) {
  const int i = blockIdx.x * 4 + (threadIdx.x >> 6), j = threadIdx.x & 63;
  if (i >= M) return;
  xn[(size_t)i * ldx + h + j] = __float2bfloat16_rn(j < r2 ? scale * t[(size_t)i * ldt + j] : 0.f);
}

__global__ void lora_pack_b_kernel(const float* __restrict__ Bq, const float* __restrict__ Bv,
                                   int h, int kv, int r, __nv_bfloat16* __restrict__ w, int ldw) {
  const int row = blockIdx.x;  // 0 .. h+2kv-1: q rows, k rows, v rows
  const int j = threadIdx.x;   // 0 .. 63
  float val = 0.f;
  if (row < h && j < r) val = Bq[(size_t)j * h + row];
  if (row >= h + kv && j >= r && j < 2 * r) val = Bv[(size_t)(j - r) * kv + (row - h - kv)];
  w[(size_t)row * ldw + h + j] = __float2bfloat16_rn(val);
}

// dst[i] = bf16(src[idx[i]])
__global__ void gather_rows_bf16_kernel(const float* __restrict__ src, int ld,
                                        const int* __restrict__ idx, int h,
                                        __nv_bfloat16* __restrict__ dst) {
  const int row = blockIdx.x;
  const int s = idx ? __ldg(idx + row) : row;
  const float4* a = reinterpret_cast<const float4*>(src + (size_t)s * ld);
  uint2* d = reinterpret_cast<uint2*>(dst + (size_t)row * h);
  for (int c = threadIdx.x; c < (h >> 2); c += blockDim.x) {
    const float4 v = a[c];
    d[c] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
  }
}

// RMSNorm backward (tensor.py:396-400, 589-595) with the result scattered
// (added) into dx at idx[row]: the gather_rmsnorm backward writes only
// retained rows, so eliminated rows keep exactly the residual gradient.
template <bool kXBf16>
__global__ void __launch_bounds__(256) rmsnorm_bwd_kernel(
    const float* __restrict__ g, int ldg, const void* __restrict__ xv, int ldx,
    const float* __restrict__ inv_in, const float* __restrict__ w, const int* __restrict__ idx,
    int h, float gscale, float* __restrict__ dx, int lddx, int accumulate) {
  __shared__ float red[8];
  const int row = blockIdx.x;
  const float inv = inv_in[row];
  const float* gr = g + (size_t)row * ldg;
  float dot = 0.f;
  for (int c = threadIdx.x; c < h; c += blockDim.x) {
    float xv_;
    if (kXBf16)
      xv_ = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(xv)[(size_t)row * ldx + c]);
    else
      xv_ = reinterpret_cast<const float*>(xv)[(size_t)row * ldx + c];
    dot += gscale * gr[c] * w[c] * xv_;
  }
  dot = block_sum<256>(dot, red);
  const float coef = inv * inv * inv * dot / (float)h;
  const int dst = idx ? __ldg(idx + row) : row;
  float* d = dx + (size_t)dst * lddx;
  for (int c = threadIdx.x; c < h; c += blockDim.x) {
    float xv_;
    if (kXBf16)
      xv_ = __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(xv)[(size_t)row * ldx + c]);
    else
      xv_ = reinterpret_cast<const float*>(xv)[(size_t)row * ldx + c];
    const float val = gscale * gr[c] * w[c] * inv - xv_ * coef;
    d[c] = accumulate ? d[c] + val : val;
  }
}

// Vectorised variant: the row of g, x and w stays in registers between the
// dot product and the output pass (one read of each, 16-B accesses).
template <bool kXBf16, int VPT>
__global__ void __launch_bounds__(256) rmsnorm_bwd_vec_kernel(
    const float* __restrict__ g, int ldg, const void* __restrict__ xv, int ldx,
    const float* __restrict__ inv_in, const float* __restrict__ w, const int* __restrict__ idx,
    int h, float gscale, float* __restrict__ dx, int lddx, int accumulate) {
  __shared__ float red[8];
  const int row = blockIdx.x;
  const float inv = inv_in[row];
  const int nv = h >> 2;
  float4 gw[VPT], xr[VPT];
  float dot = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * 256;
    if (c < nv) {
      const float4 gg = reinterpret_cast<const float4*>(g + (size_t)row * ldg)[c];
      const float4 ww = __ldg(reinterpret_cast<const float4*>(w) + c);
      if (kXBf16) {
        const uint2 u = reinterpret_cast<const uint2*>(
            reinterpret_cast<const __nv_bfloat16*>(xv) + (size_t)row * ldx)[c];
        xr[i] = make_float4(bf16_lo(u.x), bf16_hi(u.x), bf16_lo(u.y), bf16_hi(u.y));
      } else {
        xr[i] = reinterpret_cast<const float4*>(reinterpret_cast<const float*>(xv) +
                                                (size_t)row * ldx)[c];
      }
      gw[i] = make_float4(gscale * gg.x * ww.x, gscale * gg.y * ww.y, gscale * gg.z * ww.z,
                          gscale * gg.w * ww.w);
      dot += gw[i].x * xr[i].x + gw[i].y * xr[i].y + gw[i].z * xr[i].z + gw[i].w * xr[i].w;
    }
  }
  dot = block_sum<256>(dot, red);
  const float coef = inv * inv * inv * dot / (float)h;
  const int dst = idx ? __ldg(idx + row) : row;
  float4* d = reinterpret_cast<float4*>(dx + (size_t)dst * lddx);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int c = threadIdx.x + i * 256;
    if (c < nv) {
      float4 val = make_float4(gw[i].x * inv - xr[i].x * coef, gw[i].y * inv - xr[i].y * coef,
                               gw[i].z * inv - xr[i].z * coef, gw[i].w * inv - xr[i].w * coef);
      if (accumulate) {
        const float4 o = d[c];
        val.x += o.x; val.y += o.y; val.z += o.z; val.w += o.w;
      }
      d[c] = val;
    }
  }
}

__global__ void embed_kernel(const int* __restrict__ ids, const float* __restrict__ table, int h,
                             const float* __restrict__ pos_table, float* __restrict__ x) {
  const int row = blockIdx.x;
  const float4* t = reinterpret_cast<const float4*>(table + (size_t)__ldg(ids + row) * h);
  const float4* p = pos_table ? reinterpret_cast<const float4*>(pos_table + (size_t)row * h) : nullptr;
  float4* o = reinterpret_cast<float4*>(x + (size_t)row * h);
  for (int c = threadIdx.x; c < (h >> 2); c += blockDim.x) {
    float4 v = t[c];
    if (p) {
      const float4 q = p[c];
      v.x += q.x; v.y += q.y; v.z += q.z; v.w += q.w;
    }
    o[c] = v;
  }
}

// Retained-row compaction after MLP scoring: copy gate/up rows (saved for
// backward), form the inner activation for the down projection, and save
// the raw gathered residual row + its inverse RMS.
__global__ void mlp_compact_kernel(const __nv_bfloat16* __restrict__ gu_all, int ldgu,
                                   const float* __restrict__ x, int ldx,
                                   const float* __restrict__ inv_all, const int* __restrict__ idx,
                                   int h, int m_pad, int relu, __nv_bfloat16* __restrict__ gu_out,
                                   __nv_bfloat16* __restrict__ inner_out,
                                   __nv_bfloat16* __restrict__ xg_out, float* __restrict__ inv_out) {
  const int row = blockIdx.x;
  const int s = __ldg(idx + row);
  const uint4* src = reinterpret_cast<const uint4*>(gu_all + (size_t)s * ldgu);
  uint4* dst = reinterpret_cast<uint4*>(gu_out + (size_t)row * ldgu);
  if (!relu && ldgu == 2 * m_pad) {
    // one pass: every 8-column gate chunk and its up chunk are read once,
    // copied to the compact row and turned into 8 SwiGLU outputs (the
    // epilogue's logistic, sigmoid_fast, as the dense path's gate/up GEMM)
#pragma unroll 2
    for (int c8 = threadIdx.x; c8 < (m_pad >> 3); c8 += blockDim.x) {
      const int mc = c8 * 8;
      const int gcol = (mc >> 7) * 256 + (mc & 127);
      const uint4 g = src[gcol >> 3];
      const uint4 u = src[(gcol + 128) >> 3];
      dst[gcol >> 3] = g;
      dst[(gcol + 128) >> 3] = u;
      const uint32_t gv[4] = {g.x, g.y, g.z, g.w}, uv[4] = {u.x, u.y, u.z, u.w};
      float in[8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float g0 = bf16_lo(gv[e]), g1 = bf16_hi(gv[e]);
        in[2 * e] = g0 * sigmoid_fast(g0) * bf16_lo(uv[e]);
        in[2 * e + 1] = g1 * sigmoid_fast(g1) * bf16_hi(uv[e]);
      }
      reinterpret_cast<uint4*>(inner_out + (size_t)row * m_pad)[c8] =
          make_uint4(pack_bf16x2(in[0], in[1]), pack_bf16x2(in[2], in[3]),
                     pack_bf16x2(in[4], in[5]), pack_bf16x2(in[6], in[7]));
    }
  } else {
  for (int c = threadIdx.x; c < (ldgu >> 3); c += blockDim.x) dst[c] = src[c];
  // inner: silu -> 8 columns at a time from one 8-col group of gate and up
  for (int c8 = threadIdx.x; c8 < (m_pad >> 3); c8 += blockDim.x) {
    const int mc = c8 * 8;
    float in[8];
    if (!relu) {
      const int gcol = (mc >> 7) * 256 + (mc & 127);
      const uint4 g = src[gcol >> 3];
      const uint4 u = src[(gcol + 128) >> 3];
      const uint32_t gv[4] = {g.x, g.y, g.z, g.w}, uv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float g0 = bf16_lo(gv[e]), g1 = bf16_hi(gv[e]);
        in[2 * e] = g0 * sigmoid_fast(g0) * bf16_lo(uv[e]);
        in[2 * e + 1] = g1 * sigmoid_fast(g1) * bf16_hi(uv[e]);
      }
    } else {
      const uint4 u = src[mc >> 3];
      const uint32_t uv[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        in[2 * e] = fmaxf(bf16_lo(uv[e]), 0.f);
        in[2 * e + 1] = fmaxf(bf16_hi(uv[e]), 0.f);
      }
    }
    reinterpret_cast<uint4*>(inner_out + (size_t)row * m_pad)[c8] =
        make_uint4(pack_bf16x2(in[0], in[1]), pack_bf16x2(in[2], in[3]),
                   pack_bf16x2(in[4], in[5]), pack_bf16x2(in[6], in[7]));
  }
  }
  const float4* xr = reinterpret_cast<const float4*>(x + (size_t)s * ldx);
  uint2* xo = reinterpret_cast<uint2*>(xg_out + (size_t)row * h);
  for (int c = threadIdx.x; c < (h >> 2); c += blockDim.x) {
    const float4 v = xr[c];
    xo[c] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
  }
  if (threadIdx.x == 0) inv_out[row] = inv_all[s];
}

// After FlashAttention backward: rotate dq/dk back (tensor.py:627-632), pack
// [dq|dk|dv] as bf16 rows (row stride ldo; the LoRA K-extension columns
// after 3h are filled separately) for the dX GEMM, and keep the fp32
// pre-rotation dq (in place) for the LoRA gradients.  Pure streaming.
__global__ void __launch_bounds__(256) qkv_grad_prep_kernel(
    float* __restrict__ dq, const float* __restrict__ dk, const float* __restrict__ dv, int h,
    int kv, int head_dim, int rope, const float2* __restrict__ rope_tab,
    const int* __restrict__ pos, __nv_bfloat16* __restrict__ dqkv, int ldo) {
  const int row = blockIdx.x;
  const int half = head_dim >> 1;
  const int p = rope ? __ldg(pos + row) : 0;
  float* dqr = dq + (size_t)row * h;
  const float* dkr = dk + (size_t)row * kv;
  const float* dvr = dv + (size_t)row * kv;
  __nv_bfloat16* o = dqkv + (size_t)row * ldo;
  // each thread: two consecutive rotation pairs (ca, ca+1) / (cb, cb+1) of one
  // head; items [0, h/4) are dq, [h/4, (h+kv)/4) are dk and dv (kv <= h)
  for (int e2 = threadIdx.x; e2 < ((h + kv) >> 2); e2 += blockDim.x) {
    const bool isq = e2 < (h >> 2);
    const int e = (isq ? e2 : e2 - (h >> 2)) * 2;
    const int hd = e / half, j = e - hd * half;
    const int ca = hd * head_dim + j, cb = ca + half;
    const float* src = isq ? dqr : dkr;
    float2 xa = *reinterpret_cast<const float2*>(src + ca);
    float2 xb = *reinterpret_cast<const float2*>(src + cb);
    if (rope) {
      const float4 cs = *reinterpret_cast<const float4*>(rope_tab + (size_t)p * half + j);
      // (cs.x, cs.y) = (cos, sin) of pair j, (cs.z, cs.w) of pair j+1
      const float t0 = xa.x * cs.x + xb.x * cs.y, t1 = -xa.x * cs.y + xb.x * cs.x;
      const float u0 = xa.y * cs.z + xb.y * cs.w, u1 = -xa.y * cs.w + xb.y * cs.z;
      xa = make_float2(t0, u0);
      xb = make_float2(t1, u1);
    }
    if (isq) {
      *reinterpret_cast<float2*>(dqr + ca) = xa;
      *reinterpret_cast<float2*>(dqr + cb) = xb;
      *reinterpret_cast<uint32_t*>(o + ca) = pack_bf16x2(xa.x, xa.y);
      *reinterpret_cast<uint32_t*>(o + cb) = pack_bf16x2(xb.x, xb.y);
    } else {
      const float2 va = *reinterpret_cast<const float2*>(dvr + ca);
      const float2 vb = *reinterpret_cast<const float2*>(dvr + cb);
      *reinterpret_cast<uint32_t*>(o + h + ca) = pack_bf16x2(xa.x, xa.y);
      *reinterpret_cast<uint32_t*>(o + h + cb) = pack_bf16x2(xb.x, xb.y);
      *reinterpret_cast<uint32_t*>(o + h + kv + ca) = pack_bf16x2(va.x, va.y);
      *reinterpret_cast<uint32_t*>(o + h + kv + cb) = pack_bf16x2(vb.x, vb.y);
    }
  }
}

// LoRA operands of the backward GEMMs:
//  Bt [32, 3h]:  row j < r: [Bq[j] | 0 | 0];  r <= j < 2r: [0 | 0 | Bv[j-r]]  (u = dqkv·Btᵀ)
//  A-extension of the dX weight: w[c, col0 + j] = A[c, j] (j < 2r), 0 up to 64.
__global__ void lora_pack_bt_kernel(const float* __restrict__ Bq, const float* __restrict__ Bv,
                                    int h, int kv, int r, __nv_bfloat16* __restrict__ out) {
  const int j = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int n = h + 2 * kv;
  if (c >= n) return;
  float val = 0.f;
  if (c < h && j < r) val = Bq[(size_t)j * h + c];
  if (c >= h + kv && j >= r && j < 2 * r) val = Bv[(size_t)(j - r) * kv + (c - h - kv)];
  out[(size_t)j * n + c] = __float2bfloat16_rn(val);
}

__global__ void lora_pack_a_ext_kernel(const float* __restrict__ A, int lda, int h, int r2,
                                       __nv_bfloat16* __restrict__ w, int ldw, int col0) {
  const int c = blockIdx.x * 4 + (threadIdx.x >> 6), j = threadIdx.x & 63;
  if (c >= h) return;
  w[(size_t)c * ldw + col0 + j] = __float2bfloat16_rn(j < r2 ? A[(size_t)c * lda + j] : 0.f);
}

// LoRA weight gradients (kernels.py:95-100 through tensor.py:324-325):
//   dA0[c,j] += s Σ_i xn[i,c] u0[i,j]     dB0[j,c] += s Σ_i t0[i,j] g0[i,c]
// (same for adapter 1), xn recomputed from the saved bf16 rows, inv, w.
constexpr int kLoraRows = 64;
constexpr int kLoraGroups = 32;  // row groups = partial sums reduced in fixed order
template <int R>
__global__ void __launch_bounds__(128) lora_grads_kernel(
    const __nv_bfloat16* __restrict__ xg, const float* __restrict__ inv, const float* __restrict__ w,
    const float* __restrict__ t, const float* __restrict__ u, int ld, const float* __restrict__ g0,
    const float* __restrict__ g1, int M, int h, int kv, float* __restrict__ part) {
  // per row: [t_q (R) | t_v (R)] and [u_q (R) | u_v (R)], read as float4 broadcasts
  __shared__ __align__(16) float st[kLoraRows][2 * R];
  __shared__ __align__(16) float su[kLoraRows][2 * R];
  __shared__ float sinv[kLoraRows];
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  float a0[R], b0[R], a1[R], b1[R];
#pragma unroll
  for (int j = 0; j < R; ++j) a0[j] = b0[j] = a1[j] = b1[j] = 0.f;
  const float wc = c < h ? w[c] : 0.f;
  // row-group g owns slabs g, g+G, g+2G, ... (fixed order: deterministic)
  for (int r0 = blockIdx.y * kLoraRows; r0 < M; r0 += gridDim.y * kLoraRows) {
  const int nrow = min(kLoraRows, M - r0);
  __syncthreads();
  for (int e = threadIdx.x; e < nrow * 2 * R; e += blockDim.x) {
    const int i = e / (2 * R), j = e - i * 2 * R;
    st[i][j] = t[(size_t)(r0 + i) * ld + j];
    su[i][j] = u[(size_t)(r0 + i) * ld + j];
  }
  for (int i = threadIdx.x; i < nrow; i += blockDim.x) sinv[i] = inv[r0 + i];
  __syncthreads();
  if (c < h) {
#pragma unroll 2
  for (int i = 0; i < nrow; ++i) {
    const size_t off = (size_t)(r0 + i) * h + c;
    const float xn = __bfloat162float(xg[off]) * sinv[i] * wc;
    const float q = g0[off], v = c < kv ? g1[(size_t)(r0 + i) * kv + c] : 0.f;
    float tv[2 * R], uv[2 * R];
#pragma unroll
    for (int j = 0; j < 2 * R; j += 4) {
      const float4 a = *reinterpret_cast<const float4*>(&st[i][j]);
      const float4 b = *reinterpret_cast<const float4*>(&su[i][j]);
      tv[j] = a.x; tv[j + 1] = a.y; tv[j + 2] = a.z; tv[j + 3] = a.w;
      uv[j] = b.x; uv[j + 1] = b.y; uv[j + 2] = b.z; uv[j + 3] = b.w;
    }
#pragma unroll
    for (int j = 0; j < R; ++j) {
      a0[j] = fmaf(xn, uv[j], a0[j]);
      a1[j] = fmaf(xn, uv[R + j], a1[j]);
      b0[j] = fmaf(tv[j], q, b0[j]);
      b1[j] = fmaf(tv[R + j], v, b1[j]);
    }
  }
  }
  }
  if (c >= h) return;
  // partials part[g][q][j][c], q = A0, A1, B0, B1 (coalesced over c)
  float* pg = part + (size_t)blockIdx.y * 4 * R * h + c;
#pragma unroll
  for (int j = 0; j < R; ++j) {
    pg[(size_t)(0 * R + j) * h] = a0[j];
    pg[(size_t)(1 * R + j) * h] = a1[j];
    pg[(size_t)(2 * R + j) * h] = b0[j];
    pg[(size_t)(3 * R + j) * h] = b1[j];
  }
}

// Fixed-order sum of the row-group partials (g ascending), scaled and added
// into the gradients: no atomics, so all-retain ≡ dense bitwise
// (tests/test_model.py:186-191) and repeated steps are reproducible.
__global__ void __launch_bounds__(256) lora_grads_reduce_kernel(
    const float* __restrict__ part, int G, int R, int h, int kv, float scale, int lda,
    float* __restrict__ dA0, float* __restrict__ dB0, float* __restrict__ dA1,
    float* __restrict__ dB1) {
  const int n = 4 * R * h;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n) return;
  float acc = 0.f;
  for (int g = 0; g < G; ++g) acc += part[(size_t)g * n + e];
  const int q = e / (R * h), rem = e - q * R * h, j = rem / h, c = rem - j * h;
  if (q == 3 && c >= kv) return;  // dB1 is [R, kv]
  float* dst = q == 0 ? dA0 + (size_t)c * lda + j
             : q == 1 ? dA1 + (size_t)c * lda + j
             : q == 2 ? dB0 + (size_t)j * h + c
                      : dB1 + (size_t)j * kv + c;
  *dst += scale * acc;
}

// Cross-entropy rows of segmented_loss_and_grad (kernels.py:256-273,
// tensor.py:446-468): per row lse, loss term, and dlogits = (p - onehot)/count.
template <int kThreads>
__device__ __forceinline__ float block_max(float v, float* red) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  float m = red[0];
#pragma unroll
  for (int i = 1; i < kThreads / 32; ++i) m = fmaxf(m, red[i]);
  __syncthreads();
  return m;
}

// One CTA per row, float4 loads / 4-wide bf16 stores.  kSmem: the row is
// read from HBM once into shared memory (V·4 bytes, e.g. 128 KB at V=32000)
// and the max / exp-sum / dlogits passes run from there; otherwise (very
// large vocabularies) the three passes re-read global memory.
template <bool kSmem>
__global__ void __launch_bounds__(512) ce_rows_kernel(const float* __restrict__ logits, int ldl,
                                                      const int* __restrict__ targets, int V,
                                                      int ignore, float inv_count,
                                                      __nv_bfloat16* __restrict__ dlogits, int ldd,
                                                      float* __restrict__ row_loss,
                                                      int* __restrict__ bad) {
  constexpr int kT = 512;
  extern __shared__ __align__(16) float srow[];
  __shared__ float red[kT / 32];
  const int row = blockIdx.x;
  const float* l = logits + (size_t)row * ldl;
  __nv_bfloat16* d = dlogits + (size_t)row * ldd;
  const int V4 = V >> 2;  // host guarantees V, ldl, ldd multiples of 4
  const float4* l4 = reinterpret_cast<const float4*>(l);
  uint2* d4 = reinterpret_cast<uint2*>(d);
  const int t = targets[row];
  if (t == ignore) {
    for (int c = threadIdx.x; c < V4; c += kT) d4[c] = make_uint2(0u, 0u);
    if (threadIdx.x == 0) row_loss[row] = 0.f;
    return;
  }
  if (t < 0 || t >= V) {  // (validated on the host first) the loss turns NaN, never silent
    for (int c = threadIdx.x; c < V4; c += kT) d4[c] = make_uint2(0u, 0u);
    if (threadIdx.x == 0) {
      row_loss[row] = __int_as_float(0x7fc00000);
      if (bad) atomicOr(bad, 1);
    }
    return;
  }
  const float4* src = kSmem ? reinterpret_cast<const float4*>(srow) : l4;
  float mx = -INFINITY;
  for (int c = threadIdx.x; c < V4; c += kT) {
    const float4 v = l4[c];
    if (kSmem) reinterpret_cast<float4*>(srow)[c] = v;
    mx = fmaxf(mx, fmaxf(fmaxf(v.x, v.y), fmaxf(v.z, v.w)));
  }
  mx = block_max<kT>(mx, red);  // (its __syncthreads also publishes srow)
  float se = 0.f;
  for (int c = threadIdx.x; c < V4; c += kT) {
    const float4 v = src[c];
    const float4 e = make_float4(expf(v.x - mx), expf(v.y - mx), expf(v.z - mx), expf(v.w - mx));
    if (kSmem) reinterpret_cast<float4*>(srow)[c] = e;  // the dlogits pass reuses them
    se += (e.x + e.y) + (e.z + e.w);
  }
  se = block_sum<kT>(se, red);
  const float inv_se = 1.f / se;
  for (int c = threadIdx.x; c < V4; c += kT) {
    const float4 v = src[c];
    float4 e;
    if (kSmem) {
      e = v;  // exp(v - max) stored by the previous pass
    } else {
      e = make_float4(expf(v.x - mx), expf(v.y - mx), expf(v.z - mx), expf(v.w - mx));
    }
    float p0 = e.x * inv_se, p1 = e.y * inv_se;
    float p2 = e.z * inv_se, p3 = e.w * inv_se;
    const int c0 = 4 * c;
    if (t == c0) p0 -= 1.f;
    if (t == c0 + 1) p1 -= 1.f;
    if (t == c0 + 2) p2 -= 1.f;
    if (t == c0 + 3) p3 -= 1.f;
    d4[c] = make_uint2(pack_bf16x2(p0 * inv_count, p1 * inv_count),
                       pack_bf16x2(p2 * inv_count, p3 * inv_count));
  }
  if (threadIdx.x == 0) row_loss[row] = logf(se) + mx - l[t];
}

__global__ void sum_f64_kernel(const float* __restrict__ x, int n, double* __restrict__ out,
                               int accumulate) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += (double)x[i];
  s = warp_sum_d(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
    *out = accumulate ? *out + t : t;
  }
}

// Adam (optim.py:37-53) over one flat buffer of all adapter parameters.
// guard (optional): skip the update when *guard_loss is not finite or an
// earlier guarded update was skipped (*latch != 0) -- a diverged predictor
// fit must not write NaN/Inf into the caller's weights before it raises
// (the reference checks each loss before stepping, predictor.py:405-410).
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                            float* __restrict__ m, float* __restrict__ v, long long n, float lr,
                            float b1, float b2, float eps, float wd, float bc1, float bc2,
                            const double* __restrict__ guard_loss, int* __restrict__ latch) {
  if (guard_loss != nullptr) {
    const bool bad = !isfinite(*guard_loss) || (latch != nullptr && *(volatile int*)latch);
    if (bad) {
      if (latch != nullptr && blockIdx.x == 0 && threadIdx.x == 0) *latch = 1;
      return;
    }
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    float pi = p[i];
    const float gi = g[i];
    if (wd != 0.f) pi *= 1.f - lr * wd;
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * (gi * gi);
    m[i] = mi;
    v[i] = vi;
    pi -= lr * ((mi / bc1) / (sqrtf(vi / bc2) + eps));
    p[i] = pi;
  }
}

}  // namespace lemo

using namespace lemo;

extern "C" {

int lemo_rmsnorm_gather_fold(const float* x, int ldx, const int* idx, int M, int h,
                             const float* w, void* xw, int ldxw, float* inv, void* stream) {
  LEMO_ARG_CHECK(ldxw % 4 == 0 && ldxw >= h && inv != nullptr,
                 "lemo_rmsnorm_gather_fold: bad output stride or missing inv");
  if (M <= 0) return 0;
  LEMO_ARG_CHECK(h % 4 == 0 && ldx % 4 == 0 && h <= 4 * 128 * 16,
                 "lemo_rmsnorm_gather_fold: h, ldx must be multiples of 4, h <= 8192");
  const int vpt = (h / 4 + 127) / 128;
  cudaStream_t st = (cudaStream_t)stream;
  auto* o = reinterpret_cast<__nv_bfloat16*>(xw);
#define LAUNCH(V) \
  gather_rmsnorm_kernel<V, true><<<M, 128, 0, st>>>(x, ldx, idx, h, w, o, ldxw, nullptr, inv)
  if (vpt <= 1) LAUNCH(1);
  else if (vpt <= 2) LAUNCH(2);
  else if (vpt <= 4) LAUNCH(4);
  else if (vpt <= 8) LAUNCH(8);
  else LAUNCH(16);
#undef LAUNCH
  LEMO_CHECK_LAUNCH("lemo_rmsnorm_gather_fold");
  return 0;
}

int lemo_rmsnorm_gather(const float* x, int ldx, const int* idx, int M, int h, const float* w,
                        void* xn, int ldxn, void* xg, float* inv, void* stream) {
  LEMO_ARG_CHECK(ldxn % 4 == 0 && ldxn >= h, "lemo_rmsnorm_gather: bad xn row stride");
  if (M <= 0) return 0;
  LEMO_ARG_CHECK(h % 4 == 0 && ldx % 4 == 0, "lemo_rmsnorm_gather: h, ldx must be multiples of 4");
  LEMO_ARG_CHECK(h <= 4 * 128 * 16, "lemo_rmsnorm_gather: h too large");
  const int nv = h / 4;
  const int vpt = (nv + 127) / 128;
  cudaStream_t st = (cudaStream_t)stream;
  auto* xnp = reinterpret_cast<__nv_bfloat16*>(xn);
  auto* xgp = reinterpret_cast<__nv_bfloat16*>(xg);
#define LAUNCH(V) \
  gather_rmsnorm_kernel<V><<<M, 128, 0, st>>>(x, ldx, idx, h, w, xnp, ldxn, xgp, inv)
  if (vpt <= 1) LAUNCH(1);
  else if (vpt <= 2) LAUNCH(2);
  else if (vpt <= 4) LAUNCH(4);
  else if (vpt <= 8) LAUNCH(8);
  else LAUNCH(16);
#undef LAUNCH
  LEMO_CHECK_LAUNCH("lemo_rmsnorm_gather");
  return 0;
}

int lemo_lora_qkv_prep(const float* t, int ldt, int M, int r2, float scale, void* xn_ext, int ldx,
                       int h, void* stream) {
  if (M <= 0) return 0;
  LEMO_ARG_CHECK(r2 <= 64 && ldx >= h + 64, "lemo_lora_qkv_prep: need 64 extension columns");
  lora_qkv_prep_kernel<<<(M + 3) / 4, 256, 0, (cudaStream_t)stream>>>(
      t, ldt, M, r2, scale, reinterpret_cast<__nv_bfloat16*>(xn_ext), ldx, h);
  LEMO_CHECK_LAUNCH("lemo_lora_qkv_prep");
  return 0;
}

int lemo_lora_pack_b(const float* Bq, const float* Bv, int h, int kv, int r, void* w_ext,
                     int ldw, void* stream) {
  LEMO_ARG_CHECK(2 * r <= 64 && ldw >= h + 64, "lemo_lora_pack_b: need 64 extension columns");
  lora_pack_b_kernel<<<h + 2 * kv, 64, 0, (cudaStream_t)stream>>>(
      Bq, Bv, h, kv, r, reinterpret_cast<__nv_bfloat16*>(w_ext), ldw);
  LEMO_CHECK_LAUNCH("lemo_lora_pack_b");
  return 0;
}

int lemo_lora_pack(const float* A, int lda, int h, int r2, void* out, void* stream) {
  LEMO_ARG_CHECK(r2 <= 32, "lemo_lora_pack: 2r must be <= 32");
  lora_pack_kernel<<<(h + 255) / 256, 256, 0, (cudaStream_t)stream>>>(
      A, lda, h, r2, reinterpret_cast<__nv_bfloat16*>(out));
  LEMO_CHECK_LAUNCH("lemo_lora_pack");
  return 0;
}

int lemo_gather_rows_bf16(const float* src, int ld, const int* idx, int M, int h, void* dst,
                          void* stream) {
  if (M <= 0) return 0;
  LEMO_ARG_CHECK(h % 4 == 0 && ld % 4 == 0, "lemo_gather_rows_bf16: h%4");
  gather_rows_bf16_kernel<<<M, 256, 0, (cudaStream_t)stream>>>(
      src, ld, idx, h, reinterpret_cast<__nv_bfloat16*>(dst));
  LEMO_CHECK_LAUNCH("lemo_gather_rows_bf16");
  return 0;
}

int lemo_rmsnorm_bwd(const float* g, int ldg, const void* x, int x_bf16, int ldx,
                     const float* inv, const float* w, const int* idx, int M, int h, float gscale,
                     float* dx, int lddx, int accumulate, void* stream) {
  if (M <= 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  const bool vec_ok = (h % 4 == 0) && (ldg % 4 == 0) && (ldx % 4 == 0) && (lddx % 4 == 0) &&
                      h <= 4 * 256 * 8;
  if (vec_ok) {
    const int vpt = (h / 4 + 255) / 256;
#define RB(XB, V)                                                                       \
  rmsnorm_bwd_vec_kernel<XB, V><<<M, 256, 0, st>>>(g, ldg, x, ldx, inv, w, idx, h, gscale, dx, \
                                                   lddx, accumulate)
    if (x_bf16) {
      if (vpt <= 1) RB(true, 1); else if (vpt <= 2) RB(true, 2); else if (vpt <= 4) RB(true, 4);
      else RB(true, 8);
    } else {
      if (vpt <= 1) RB(false, 1); else if (vpt <= 2) RB(false, 2); else if (vpt <= 4) RB(false, 4);
      else RB(false, 8);
    }
#undef RB
  } else if (x_bf16) {
    rmsnorm_bwd_kernel<true><<<M, 256, 0, st>>>(g, ldg, x, ldx, inv, w, idx, h, gscale, dx, lddx,
                                                accumulate);
  } else {
    rmsnorm_bwd_kernel<false><<<M, 256, 0, st>>>(g, ldg, x, ldx, inv, w, idx, h, gscale, dx, lddx,
                                                 accumulate);
  }
  LEMO_CHECK_LAUNCH("lemo_rmsnorm_bwd");
  return 0;
}

int lemo_embed(const int* ids, int n, const float* table, int h, const float* pos_table, float* x,
               void* stream) {
  if (n <= 0) return 0;
  LEMO_ARG_CHECK(h % 4 == 0, "lemo_embed: h%4");
  embed_kernel<<<n, 256, 0, (cudaStream_t)stream>>>(ids, table, h, pos_table, x);
  LEMO_CHECK_LAUNCH("lemo_embed");
  return 0;
}

int lemo_mlp_compact(const void* gu_all, const float* x, int ldx, const float* inv_all,
                     const int* idx, int M, int h, int m_pad, int relu, void* gu_out,
                     void* inner_out, void* xg_out, float* inv_out, void* stream) {
  if (M <= 0) return 0;
  LEMO_ARG_CHECK(m_pad % 128 == 0 && h % 4 == 0, "lemo_mlp_compact: m_pad%128, h%4");
  const int ldgu = relu ? m_pad : 2 * m_pad;
  mlp_compact_kernel<<<M, 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const __nv_bfloat16*>(gu_all), ldgu, x, ldx, inv_all, idx, h, m_pad, relu,
      reinterpret_cast<__nv_bfloat16*>(gu_out), reinterpret_cast<__nv_bfloat16*>(inner_out),
      reinterpret_cast<__nv_bfloat16*>(xg_out), inv_out);
  LEMO_CHECK_LAUNCH("lemo_mlp_compact");
  return 0;
}

int lemo_qkv_grad_prep(float* dq, const float* dk, const float* dv, int M, int h, int kv,
                       int head_dim, int rope, const void* rope_tab, const int* pos, void* dqkv,
                       int ldo, void* stream) {
  if (M <= 0) return 0;
  LEMO_ARG_CHECK(head_dim % 4 == 0 && kv <= h && kv % head_dim == 0 && ldo >= h + 2 * kv &&
                     ldo % 2 == 0,
                 "lemo_qkv_grad_prep: bad geometry");
  qkv_grad_prep_kernel<<<M, 256, 0, (cudaStream_t)stream>>>(
      dq, dk, dv, h, kv, head_dim, rope, reinterpret_cast<const float2*>(rope_tab), pos,
      reinterpret_cast<__nv_bfloat16*>(dqkv), ldo);
  LEMO_CHECK_LAUNCH("lemo_qkv_grad_prep");
  return 0;
}

int lemo_lora_pack_bt(const float* Bq, const float* Bv, int h, int kv, int r, void* out,
                      void* stream) {
  LEMO_ARG_CHECK(2 * r <= 32, "lemo_lora_pack_bt: 2r <= 32");
  dim3 grid((h + 2 * kv + 255) / 256, 32);
  lora_pack_bt_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      Bq, Bv, h, kv, r, reinterpret_cast<__nv_bfloat16*>(out));
  LEMO_CHECK_LAUNCH("lemo_lora_pack_bt");
  return 0;
}

int lemo_lora_pack_a_ext(const float* A, int lda, int h, int r2, void* w, int ldw, int col0,
                         void* stream) {
  LEMO_ARG_CHECK(r2 <= 64 && ldw >= col0 + 64, "lemo_lora_pack_a_ext: need 64 columns");
  lora_pack_a_ext_kernel<<<(h + 3) / 4, 256, 0, (cudaStream_t)stream>>>(
      A, lda, h, r2, reinterpret_cast<__nv_bfloat16*>(w), ldw, col0);
  LEMO_CHECK_LAUNCH("lemo_lora_pack_a_ext");
  return 0;
}

static int lora_row_groups(int M) {
  const int slabs = (M + kLoraRows - 1) / kLoraRows;
  return slabs < kLoraGroups ? slabs : kLoraGroups;
}

int lemo_lora_grads_workspace(int M, int h, int r) {
  if (M <= 0) return 0;
  return lora_row_groups(M) * 4 * r * h;
}

int lemo_lora_grads(const void* xg, const float* inv, const float* w, const float* t,
                    const float* u, int ld, const float* g0, const float* g1, int M, int h,
                    int kv, int r, float scale, int lda, float* dA0, float* dB0, float* dA1,
                    float* dB1, float* workspace, void* stream) {
  if (M <= 0) return 0;
  LEMO_ARG_CHECK(r <= 16, "lemo_lora_grads: LoRA rank <= 16");
  LEMO_ARG_CHECK(workspace != nullptr, "lemo_lora_grads: workspace required");
  const int G = lora_row_groups(M);
  dim3 grid((h + 127) / 128, G);
  cudaStream_t st = (cudaStream_t)stream;
  auto* xgp = reinterpret_cast<const __nv_bfloat16*>(xg);
#define LG(RR) \
  lora_grads_kernel<RR><<<grid, 128, 0, st>>>(xgp, inv, w, t, u, ld, g0, g1, M, h, kv, workspace)
  switch (r) {
    case 2: LG(2); break;
    case 4: LG(4); break;
    case 8: LG(8); break;
    case 16: LG(16); break;
    default: set_error_msg("lemo_lora_grads: LoRA rank must be 2, 4, 8 or 16"); return LEMO_ERR_REPORTED;
  }
#undef LG
  const int n = 4 * r * h;
  lora_grads_reduce_kernel<<<(n + 255) / 256, 256, 0, st>>>(workspace, G, r, h, kv, scale, lda,
                                                            dA0, dB0, dA1, dB1);
  LEMO_CHECK_LAUNCH("lemo_lora_grads");
  return 0;
}

int lemo_ce_rows(const float* logits, int ldl, const int* targets, int n, int V, int ignore,
                 float inv_count, void* dlogits, int ldd, float* row_loss, int* bad,
                 void* stream) {
  if (n <= 0) return 0;
  LEMO_ARG_CHECK(V % 4 == 0 && ldl % 4 == 0 && ldd % 4 == 0,
                 "lemo_ce_rows: V and the row strides must be multiples of 4");
  cudaStream_t st = (cudaStream_t)stream;
  auto* dl = reinterpret_cast<__nv_bfloat16*>(dlogits);
  const size_t smem = (size_t)V * sizeof(float);
  if (smem <= 200 * 1024) {
    static int attr = cudaFuncSetAttribute(ce_rows_kernel<true>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    (void)attr;
    ce_rows_kernel<true><<<n, 512, smem, st>>>(logits, ldl, targets, V, ignore, inv_count, dl, ldd,
                                               row_loss, bad);
  } else {
    ce_rows_kernel<false><<<n, 512, 0, st>>>(logits, ldl, targets, V, ignore, inv_count, dl, ldd,
                                             row_loss, bad);
  }
  LEMO_CHECK_LAUNCH("lemo_ce_rows");
  return 0;
}

int lemo_sum_f64(const float* x, int n, double* out, int accumulate, void* stream) {
  sum_f64_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(x, n, out, accumulate);
  LEMO_CHECK_LAUNCH("lemo_sum_f64");
  return 0;
}

int lemo_adam(float* p, const float* g, float* m, float* v, long long n, float lr, float b1,
              float b2, float eps, float wd, float bc1, float bc2, const double* guard_loss,
              int* guard_latch, void* stream) {
  if (n <= 0) return 0;
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  adam_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(p, g, m, v, n, lr, b1, b2, eps, wd,
                                                             bc1, bc2, guard_loss, guard_latch);
  LEMO_CHECK_LAUNCH("lemo_adam");
  return 0;
}

}  // extern "C"
