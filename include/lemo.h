/*
 * liblemo — C ABI of the B200 (sm_100a) LeMo contextual-token-sparsity hot path.
 *
 * This is the drop-in boundary for the reference `sparsetune` package
 * (arxiv 2501.09767 re-implementation, /root/reference/pkg/src/sparsetune).
 * The reference has no native code; its operator-plugin API is
 * `tensor.custom_op(out, op, inputs, saved, backward_fn)` (tensor.py:177-179)
 * and its hot-path entry points are the Python functions cited beside each
 * declaration below.  A host binding (ctypes in this repo, see
 * paper_2501_09767_b200/_lib.py and INTEGRATION.md) wraps these calls in the
 * reference's Python names.
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless stated otherwise.  The library
 *     never allocates or frees device memory: the caller owns every buffer
 *     and passes any workspace explicitly.
 *   - `stream` is a cudaStream_t passed as void*; every call is
 *     stream-ordered and asynchronous (no host synchronisation).
 *   - Matrices are row-major.  "bf16" buffers hold __nv_bfloat16.
 *   - Return value: 0 on success; nonzero on a launch / CUDA / argument
 *     error, with a description in lemo_last_error() (thread-local).
 *   - GEMM convention: C[M,N] = A[M,K] · B[N,K]^T (both operands K-contiguous).
 */
#ifndef LEMO_H_
#define LEMO_H_

#ifdef __cplusplus
extern "C" {
#endif

/* ---- library ------------------------------------------------------------ */
const char* lemo_last_error(void);
int lemo_version(void);
void lemo_clear_descriptor_cache(void);

/* ---- tcgen05 GEMMs with LeMo epilogues ---------------------------------- */

/* C(bf16) = A·Bᵀ.  tensor.py:316-327 (matmul forward). */
int lemo_gemm_bf16(const void* A, int lda, const void* B, int ldb, void* C, int ldc, int M, int N,
                   int K, void* stream);

/* C(f32) (+)= A·Bᵀ + scale · U[M,R] · S  where S(j, col) = S[j*s_rs + col*s_cs]
 * (rank-R side product = the LoRA term of kernels.py:95-100; R = 0 disables it). */
int lemo_gemm_f32(const void* A, int lda, const void* B, int ldb, float* C, int ldc, int M, int N,
                  int K, const float* U, int ldu, int R, const float* S, int s_rs, int s_cs,
                  float scale, int accumulate, void* stream);

/* R[idx[i], :] += (A·Bᵀ)[i, :]  — index-remapped in-place residual update,
 * replaces T.scatter_add_rows (tensor.py:536-550) after the output projections
 * of sparse_attention_fused / sparse_mlp_fused (kernels.py:153-222). idx may be
 * NULL (identity). Rows of idx must be distinct. */
int lemo_gemm_scatter_add(const void* A, int lda, const void* B, int ldb, float* R, int ldr,
                          const int* idx, int M, int N, int K, void* stream);

/* Fused q/k/v projection of attention_core (kernels.py:103-114):
 *   [q|k|v] = xn · W_qkv  (+ scale·(xn·A_q)·B_q on q, + scale·(xn·A_v)·B_v on v)
 *   then rope_rotate (tensor.py:610-634) at pos[i] (original token positions).
 * w_qkv_t: [3h, h] bf16 (rows = output features); tq/tv: [M, ldt] fp32 = xn·A;
 * Bq/Bv: [r, h] fp32; rope_tab: [max_pos, head_dim/2] float2 (cos, sin). */
int lemo_gemm_qkv(const void* xn, const void* w_qkv_t, int M, int h, void* q, void* k, void* v,
                  int head_dim, int rope, const void* rope_tab, const int* pos, const float* tq,
                  const float* tv, int ldt, int r, const float* Bq, const float* Bv, float scale,
                  void* stream);

/* Gate/up half of mlp_core (kernels.py:119-124) with the MLP token
 * informativeness (model.py:371-396, sparsity.py:284-290) in the epilogue.
 * w_gu_t: [N, K] bf16, gate/up columns interleaved in 128-column chunks
 * (silu) or up only (relu).  gu (optional): [M, N] bf16; inner (optional):
 * [M, N/2] (silu) or [M, N] (relu) bf16; partial (optional): [N/256, M] fp32
 * per-tile row sums of |inner|. */
int lemo_gemm_gateup(const void* xn, int ldx, const void* w_gu_t, int M, int N, int K, void* gu,
                     void* inner, float* partial, int relu, void* stream);

/* Backward of the MLP inner product: dinner = dy · W_downᵀ (w_down: [m_pad, h]
 * bf16, reference layout) turned into d(gate), d(up) (tensor.py:289-290,
 * 381-382) using the saved gu; dgu has gu's layout. */
int lemo_gemm_dgateup(const void* dy, const void* w_down, int M, int m_pad, int h, const void* gu,
                      void* dgu, int relu, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LEMO_H_ */
