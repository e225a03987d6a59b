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

/* C(bf16) = A·B with B [K, N] row-major (MN-major tcgen05 B operand). */
int lemo_gemm_nn_bf16(const void* A, int lda, const void* B, int ldb, void* C, int ldc, int M,
                      int N, int K, void* stream);

/* C(f32) (+)= A·Bᵀ (accumulate != 0 adds into C).  Any N; partial column
 * chunks are stored element-wise.  (LoRA terms of the dX GEMMs ride in a
 * K-extension of the operands — lemo_lora_pack_a_ext — not in the epilogue.) */
int lemo_gemm_f32(const void* A, int lda, const void* B, int ldb, float* C, int ldc, int M, int N,
                  int K, int accumulate, void* stream);

/* lemo_gemm_f32 with fp32-faithful accumulation: the TMEM partial sum is
 * restarted every 128 K-columns and promoted into round-to-nearest fp32
 * registers (the tcgen05 accumulator truncates; see gemm.cuh kPromote).  For
 * bf16x3 operand pairs (Eq. 3 of the predictor, parity-mode scorers). */
int lemo_gemm_f32_exact(const void* A, int lda, const void* B, int ldb, float* C, int ldc, int M,
                        int N, int K, int accumulate, void* stream);

/* R[idx[i], :] += (A·Bᵀ)[i, :]  — index-remapped in-place residual update,
 * replaces T.scatter_add_rows (tensor.py:536-550) after the output projections
 * of sparse_attention_fused / sparse_mlp_fused (kernels.py:153-222). idx may be
 * NULL (identity). Rows of idx must be distinct. */
int lemo_gemm_scatter_add(const void* A, int lda, const void* B, int ldb, float* R, int ldr,
                          const int* idx, int M, int N, int K, void* stream);

/* Fused q/k/v projection of attention_core (kernels.py:103-114):
 *   [q|k|v] = xn_ext · w_qkv_tᵀ over K columns, then rope_rotate
 *   (tensor.py:610-634) of q, k at pos[i] (original token positions).
 * With LoRA, K = h + 64: xn_ext = [xn | s·(xn·A_q) | s·(xn·A_v) | 0]
 * (lemo_lora_qkv_prep) and w_qkv_t = [W_qkvᵀ | B_qᵀ, B_vᵀ | 0]
 * (lemo_lora_pack_b), so q = xn·Wq + s·(xn·A_q)·B_q (kernels.py:95-100) is
 * accumulated by the tensor core itself.  Without LoRA, K = h.
 * w_qkv_t: [h + (nmat-1)·kv, ldw] bf16 (nmat = 2: q, k only, as layer_qk does,
 * model.py:356-368); q is [M, h], k and v are [M, kv] (kv = h for multi-head,
 * kv = n_kv_heads·head_dim < h for grouped-query attention, an extension
 * beyond the reference); inv_freq: [head_dim/2] float64 = base^(-j/half).
 * row_scale (optional, [M] fp32): per-row factor on the accumulator before
 * RoPE (RMSNorm folded into the epilogue, lemo_rmsnorm_gather_fold). */
int lemo_gemm_qkv(const void* xn, int ldx, const void* w_qkv_t, int ldw, int M, int h, int kv,
                  int K, int nmat, void* q, void* k, void* v, int head_dim, int rope,
                  const double* inv_freq, const int* pos, const float* row_scale, void* stream);

/* A-side LoRA K-extension: xn_ext[i, h+j] = bf16(scale·t[i, j]) (j < r2), 0 up to 64. */
int lemo_lora_qkv_prep(const float* t, int ldt, int M, int r2, float scale, void* xn_ext, int ldx,
                       int h, void* stream);

/* B-side LoRA K-extension of w_qkv_t [h+2kv, ldw]: columns h..h+63 ← B_qᵀ (q rows),
 * B_vᵀ (v rows, offset r; B_v is [r, kv]), zeros elsewhere.  Re-run after every
 * optimizer step. */
int lemo_lora_pack_b(const float* Bq, const float* Bv, int h, int kv, int r, void* w_ext,
                     int ldw, void* stream);

/* Gate/up half of mlp_core (kernels.py:119-124) with the MLP token
 * informativeness (model.py:371-396, sparsity.py:284-290) in the epilogue.
 * w_gu_t: [N, K] bf16, gate/up columns interleaved in 128-column chunks
 * (silu) or up only (relu).  gu (optional): [M, N] bf16; inner (optional):
 * [M, N/2] (silu) or [M, N] (relu) bf16; partial (optional): [N/256, M] fp32
 * per-tile row sums of |inner|.  exact_score != 0: the scores use the fp32
 * accumulator (parity mode: xn / w_gu_t given as bf16x3 operands, K = 3h, see
 * lemo_split_bf16x3) instead of the bf16-rounded gate/up that gu stores.
 * row_scale (optional, [M] fp32) multiplies each accumulator row first: the
 * RMSNorm 1/rms when xn is bf16(x·w) (lemo_rmsnorm_gather_fold). */
int lemo_gemm_gateup(const void* xn, int ldx, const void* w_gu_t, int M, int N, int K, void* gu,
                     void* inner, float* partial, int relu, int exact_score,
                     const float* row_scale, void* stream);

/* Backward of the MLP inner product: dinner = dy · W_downᵀ (w_down: [m_pad, h]
 * bf16, reference layout) turned into d(gate), d(up) (tensor.py:289-290,
 * 381-382) using the saved gu; dgu has gu's layout. */
int lemo_gemm_dgateup(const void* dy, const void* w_down, int M, int m_pad, int h, const void* gu,
                      void* dgu, int relu, void* stream);

/* ---- row kernels (HBM-bound) --------------------------------------------- */

/* Fused gather + RMSNorm (tensor.py:578-597; idx NULL = all rows): xn (bf16)
 * plus optional saved raw rows xg (bf16) and inv (fp32). */
int lemo_rmsnorm_gather(const float* x, int ldx, const int* idx, int M, int h, const float* w,
                        void* xn, int ldxn, void* xg, float* inv, void* stream);

/* As lemo_rmsnorm_gather, but xw = bf16(x[idx]·w) and inv = 1/sqrt(mean(x²)+eps)
 * separately: the normalisation is applied to the GEMM accumulator (row_scale of
 * lemo_gemm_gateup / lemo_gemm_qkv_scaled), so bf16-valued residual rows enter
 * the tensor cores exactly (scoring precision, model.py:333-335 + 371-396). */
int lemo_rmsnorm_gather_fold(const float* x, int ldx, const int* idx, int M, int h,
                             const float* w, void* xw, int ldxw, float* inv, void* stream);

/* LoRA down-projection operand: out[j, c] = bf16(A[c*lda + j]) for j < r2,
 * zero for r2 <= j < 32 (out: [32, h] bf16), so t = xn·[A_q|A_v]
 * (kernels.py:97-98) is one tcgen05 GEMM with N = 32. */
int lemo_lora_pack(const float* A, int lda, int h, int r2, void* out, void* stream);

/* dst[i] = bf16(src[idx[i]]) — gradient rows for the output-projection
 * backward (the g[idx] of scatter_add_rows backward, tensor.py:547-548). */
int lemo_gather_rows_bf16(const float* src, int ld, const int* idx, int M, int h, void* dst,
                          void* stream);

/* RMSNorm backward (tensor.py:396-400) of rows x (bf16 if x_bf16, else fp32),
 * result written (accumulate=0) or added (1) into dx at row idx[i]
 * (gather_rmsnorm backward, tensor.py:589-595). g is scaled by gscale. */
int lemo_rmsnorm_bwd(const float* g, int ldg, const void* x, int x_bf16, int ldx,
                     const float* inv, const float* w, const int* idx, int M, int h, float gscale,
                     float* dx, int lddx, int accumulate, void* stream);

/* x[i] = table[ids[i]] (+ pos_table[i])  (tensor.py:405-420, model.py:240-244). */
int lemo_embed(const int* ids, int n, const float* table, int h, const float* pos_table, float* x,
               void* stream);

/* Retained-row compaction after MLP scoring: gu_out[i] = gu_all[idx[i]],
 * inner_out[i] = silu(g)·u (or relu(u)), xg_out[i] = bf16(x[idx[i]]),
 * inv_out[i] = inv_all[idx[i]]. */
int lemo_mlp_compact(const void* gu_all, const float* x, int ldx, const float* inv_all,
                     const int* idx, int M, int h, int m_pad, int relu, void* gu_out,
                     void* inner_out, void* xg_out, float* inv_out, void* stream);

/* After attention backward: RoPE backward of dq/dk (tensor.py:627-632; dq is
 * rewritten in place pre-rotation) and packed bf16 [dq|dk|dv] rows (row stride
 * ldo >= h + 2kv; dq [M, h], dk/dv [M, kv]) for the dX GEMM. */
int lemo_qkv_grad_prep(float* dq, const float* dk, const float* dv, int M, int h, int kv,
                       int head_dim, int rope, const void* rope_tab, const int* pos, void* dqkv,
                       int ldo, void* stream);

/* out [32, h+2kv] bf16: row j < r = [Bq[j] | 0 | 0], r <= j < 2r = [0 | 0 | Bv[j-r]];
 * u = dqkv·outᵀ gives [dq·Bqᵀ | dv·Bvᵀ] (the LoRA backward factors of
 * kernels.py:95-100) as one tcgen05 GEMM. */
int lemo_lora_pack_bt(const float* Bq, const float* Bv, int h, int kv, int r, void* out,
                      void* stream);

/* w[c, col0 + j] = bf16(A[c*lda + j]) for j < r2, 0 up to 64 — the LoRA
 * K-extension of the dX weight, so dxn += s·u·Aᵀ runs inside the GEMM. */
int lemo_lora_pack_a_ext(const float* A, int lda, int h, int r2, void* w, int ldw, int col0,
                         void* stream);

/* LoRA weight gradients accumulated (+=) into dA0/dB0/dA1/dB1:
 * dA[c,j] = s·Σ xn[i,c]u[i,j], dB[j,c] = s·Σ t[i,j]g[i,c] (tensor.py:324-325).
 * Row-group partial sums go to `workspace` (lemo_lora_grads_workspace floats)
 * and are reduced in a fixed order: deterministic, no atomics. */
int lemo_lora_grads_workspace(int M, int h, int r); /* floats; not a status */
int lemo_lora_grads(const void* xg, const float* inv, const float* w, const float* t,
                    const float* u, int ld, const float* g0, const float* g1, int M, int h,
                    int kv, int r, float scale, int lda, float* dA0, float* dB0, float* dA1,
                    float* dB1, float* workspace, void* stream);

/* Cross-entropy rows of segmented_loss_and_grad (kernels.py:256-273): per-row
 * loss terms and dlogits = (softmax - onehot)·inv_count (bf16); ignore rows
 * get zeros; an out-of-range target makes its row loss NaN (so the summed
 * loss is NaN) and sets *bad when bad is non-NULL. */
int lemo_ce_rows(const float* logits, int ldl, const int* targets, int n, int V, int ignore,
                 float inv_count, void* dlogits, int ldd, float* row_loss, int* bad,
                 void* stream);

/* *out (+)= Σ x[i] in float64 (deterministic single-CTA reduction). */
int lemo_sum_f64(const float* x, int n, double* out, int accumulate, void* stream);

/* Adam step over a flat fp32 parameter buffer (optim.py:37-53).  guard_loss
 * (optional, device f64): the update is skipped when *guard_loss is not finite
 * or *guard_latch (optional) is set, and the latch is then set -- predictor
 * training checks each record's loss before stepping (predictor.py:405-410). */
int lemo_adam(float* p, const float* g, float* m, float* v, long long n, float lr, float b1,
              float b2, float eps, float wd, float bc1, float bc2, const double* guard_loss,
              int* guard_latch, void* stream);

/* ---- pattern scoring and selection ----------------------------------------- */

/* Block means xb[n] = mean(x[n*b:(n+1)*b]) (predictor.py:117-123). */
int lemo_block_embed(const float* x, int ldx, int s, int h, int b, float* xb, void* stream);

/* fp32-faithful bf16 tensor-core GEMMs ("bf16x3"): a fp32 matrix is carried
 * as hi = bf16(v), lo = bf16(v - hi) and A·B ≈ Ahi·Bhi + Ahi·Blo + Alo·Bhi is
 * one GEMM over K' = 3K with A' = [hi|hi|lo] (pattern 0) and B' = [hi|lo|hi]
 * (pattern 1).  lemo_split_bf16x3 builds an operand [M, 3K] from fp32 A. */
int lemo_split_bf16x3(const float* A, int lda, int M, int K, int pattern, void* out,
                      void* stream);

/* C = act(A'·B'ᵀ)·mask over K' = K3 (= 3K): writes the split form of C
 * (out [M, 3N], pattern as above) and/or fp32 C (f32 [M, N]); act = relu if
 * relu.  One Predictor layer (predictor.py:83-89) per call. */
int lemo_gemm_split3(const void* A, int lda, const void* B, int ldb, int M, int N, int K3,
                     int relu, const unsigned char* mask, int pattern, void* out, int ldo,
                     float* f32, int ldf, void* stream);

/* Two predictors' first layers (predictor.py:83-85) over the same input in
 * one GEMM: B' stacks both weight operands along N (rows [0, nsplit) = the
 * query predictor's, [nsplit, N) = the key predictor's), mask covers all N
 * columns; act = relu if relu.  Columns < nsplit are written in split form
 * (pattern 0) to out [M, 3·nsplit], the rest to out2 [M, 3·(N - nsplit)]. */
int lemo_gemm_split3_dual(const void* A, int lda, const void* B, int ldb, int M, int N, int K3,
                          int nsplit, int relu, const unsigned char* mask, void* out, int ldo,
                          void* out2, int ldo2, void* stream);

/* vec[n] = Σ_{m>=n} max(S[m,n], 0) in float64, ascending m
 * (model.py:575-578 + sparsity.py:253-260). */
int lemo_colsum_clamped(const float* S, int lds, int nb, double* vec, void* stream);

/* The same ascending-m f64 column sums from a packed lower triangle
 * (element (m, n) at m(m+1)/2 + n; sparsity.py:253-260). */
int lemo_colsum_packed(const double* packed, int nb, double* vec, void* stream);

/* out[m(m+1)/2 + n] = S[m, n] for n <= m (clamped at 0 when clamp != 0): the
 * packed lower triangle of sparsity.py:35-69 (BlockScoreMatrix) as f64 (out64)
 * or f32 (out32; exactly one of them non-NULL) — predicted_triangle /
 * predict_scores (predictor.py:176-212) and exact_block_scores. */
int lemo_pack_tril(const float* S, int lds, int nb, int clamp, double* out64, float* out32,
                   void* stream);

/* Token-level refinement candidates: out[row] = 0 for every row < n_valid
 * whose block score vec[row / b] lies within `margin` of thr AND whose own
 * token score Σ_t partial[t, row] / m_real is >= thr - margin; -1 otherwise
 * (select with thr = 0 and block size 1 compacts them).  Only these rows can
 * decide their block's >= (sparsity.py:274-277 on the block max,
 * sparsity.py:298-305); partial is [n_tiles, s]. */
int lemo_mlp_token_band(const float* partial, int n_tiles, int s, int n_valid, int b, int m_real,
                        const double* vec, double thr, double margin, double* out, void* stream);

/* vec[tok[i] / b] = max over the re-scored rows of that block of
 * Σ_t partial[t, i] / m_real (tok ascending; partial is [n_tiles, rows]) --
 * the token-level refinement written back (mlp_block_scores arithmetic).
 * count (device, may be NULL): the re-scored rows when the GEMM ran on a
 * capacity of `rows` (rows past *count are padding); overflow (device, may be
 * NULL) is set to *count > rows -- the caller then re-runs with the exact count. */
int lemo_mlp_patch_rows(const float* partial, int n_tiles, int rows, const int* tok,
                        const int* count, int b, int m_real, double* vec, int* overflow,
                        void* stream);

/* MLP block scores from per-tile row partials of lemo_gemm_gateup:
 * token score = Σ partial / m_real, block = max over rows < n_valid
 * (sparsity.py:284-305, model.py:383-395). */
int lemo_mlp_block_scores(const float* partial, int n_tiles, int s, int n_valid, int b, int m_real,
                          double* vec, void* stream);

/* eliminate (sparsity.py:263-281) + token_indices (sparsity.py:95-104):
 * keep block n iff vec[n] >= T (T = *thr_dev if thr_dev else thr), or
 * force[n] != 0 (force_blocks, e.g. the sink block; force may be NULL).  Writes mask[nb], ascending blocks[], tokens[] (int32) and
 * counts = {n_tokens_kept, n_blocks_kept, any_nonfinite}; thr_out = T. */
int lemo_select(const double* vec, int nb, double thr, const double* thr_dev,
                const unsigned char* force, int b, int n_tokens, unsigned char* mask, int* blocks, int* tokens, int* counts,
                double* thr_out, void* stream);

/* *out = sorted(data)[rank] (+1 if plus_one): np.quantile(..., method="lower")
 * with rank = floor((n-1)q) (model.py:562, predictor.py:276). */
int lemo_quantile_lower(const double* data, int n, long long rank, int plus_one, double* out,
                        void* stream);

/* Exact block informativeness (sparsity.py:173-219): out[m*ldo + n] (n <= m)
 * = max over the 16x16 tile of Σ_h max(q·k, 0)/H with the causal / n_valid
 * mask; q [s, h], k [s, kv] bf16 post-rotation (layer_qk, model.py:356-368;
 * query head hd reads key head hd / (h/kv)).  tcgen05 kernel: S per head in
 * TMEM, head sum / clamp / tile max in the epilogue.  q_lo, k_lo (both or
 * neither): bf16 residuals of fp32 q, k (v ≈ hi + lo) — the fp32-faithful
 * parity mode issues hi·hi + hi·lo + lo·hi per head.  Entries above the
 * diagonal are not written (the caller zero-fills out). */
int lemo_exact_block_scores(const void* q, const void* k, const void* q_lo, const void* k_lo,
                            int s, int h, int kv, int head_dim, int block, int n_valid,
                            float* out, int ldo, void* stream);

/* ---- fp32-faithful (parity-mode) scoring helpers ------------------------------ */

/* out[i, :] = x[idx[i]] · inv · w in fp32, inv = 1/sqrt(mean(x²) + 1e-6)
 * (model.py:333-335 _rmsnorm_np); idx may be NULL; inv (optional) [M]. */
int lemo_rmsnorm_f32(const float* x, int ldx, const int* idx, int M, int h, const float* w,
                     float* out, int ldo, float* inv, void* stream);

/* layer_qk tail in fp32 (model.py:338-368): q = qk[:, :h] + ((t[:, :r])·Bq)·scale,
 * k = qk[:, h:h+kv], RoPE at positions 0..s-1 from rope_tab [s, head_dim/2, 2]
 * (cos, sin; f64-computed, f32-cast as tensor.py:604-607) when rope != 0; Bq may
 * be NULL (no adapter).  Writes the bf16 hi/lo split of q [s, h] and k [s, kv]. */
int lemo_qk_finish(const float* qk, int ldqk, const float* t, int ldt, const float* Bq, int r,
                   float scale, const float* rope_tab, int s, int h, int kv, int head_dim,
                   int rope, void* q_hi, void* q_lo, void* k_hi, void* k_lo, void* stream);

/* out [M, 2K] = [hi | lo] of a fp32 [M, K]: the A operand of x_hi·W + x_lo·W
 * against a bf16-exact weight given as [W | W] (parity precision, 2 terms). */
int lemo_split_bf16x2(const float* a, int lda, int M, int K, void* out, void* stream);

/* hi = bf16(a), lo = bf16(a - hi) for a fp32 [M, K] (row stride lda). */
int lemo_split_hilo(const float* a, int lda, int M, int K, void* hi, void* lo, void* stream);

/* ---- offline predictor training (predictor.py:215-433) ----------------------- */

/* out [C, 3R] = bf16x3 split (pattern as lemo_split_bf16x3) of Aᵀ, A fp32 [R, C]:
 * the K-major operand of a transposed matrix (weight gradients Xᵀ·dY). */
int lemo_split_bf16x3_t(const float* A, int lda, int R, int C, int pattern, void* out,
                        void* stream);

/* MSE over the packed lower triangle of the nb x nb prediction `full` against
 * `label` (packed, tensor.py:495-505): row_loss[m] = Σ_{n<=m} d², dfull =
 * 2d/T below and on the diagonal, 0 above (T = nb(nb+1)/2). */
int lemo_tril_mse(const float* full, int ldf, const float* label, int nb, float* dfull, int ldd,
                  double* row_loss, void* stream);

/* dh[i] = 0 where h[i] <= 0 (ReLU·mask backward on the saved output). */
int lemo_relu_grad(float* dh, const float* h, long long n, void* stream);

/* counts[c] += #{r : h[r, c] == 0} (zero-frequency tracking, predictor.py:76-80). */
int lemo_zero_count(const float* h, int ldh, int M, int N, long long* counts, void* stream);

/* Backward of the per-block row mean of token pooling (predictor.py:126-135):
 * out [nb·b, w] rows i = g[i / b] / b. */
int lemo_block_expand(const float* g, int nb, int w, int b, float* out, void* stream);

/* *out = scale · Σ x (f64, fixed order). */
int lemo_sum_d(const double* x, int n, double scale, double* out, void* stream);

/* ---- attention over the compact retained sequence --------------------------- */

/* Causal softmax attention (tensor.py:646-691) on q [n, h], k/v [n, kv] bf16
 * (heads side by side; query head hd reads key/value head hd / (h/kv), i.e.
 * grouped-query attention when kv < h); o [n, h] bf16, lse [h/head_dim, n]
 * fp32 (natural log).  tcgen05 kernel: two query tiles per CTA ping-ponging
 * two softmax warpgroups, S/O in TMEM, P as a bf16 TMEM A operand,
 * warp-collective MMA issue; head_dim 64 or 128. */
int lemo_flash_fwd_tc(const void* q, const void* k, const void* v, void* o, float* lse, int n,
                      int h, int kv, int head_dim, float scale, void* stream);

/* delta[hd, i] = Σ_d dO[i, hd·D + d] · O[i, hd·D + d]  (tensor.py:696). */
int lemo_attn_delta(const void* o, const void* dout, float* delta, int n, int h, int head_dim,
                    void* stream);

/* Attention backward (tensor.py:693-722) on tcgen05 (head_dim 64 or 128): an
 * atomic-free dK/dV kernel (transposed formulation, dK/dV resident in TMEM,
 * Pᵀ/dSᵀ as bf16 TMEM A operands) and a dQ kernel, both recomputing P from lse
 * and pipelined so the element-wise phases overlap the MMAs.  dq [n, h], dk/dv
 * [n, kv] fp32; delta is a caller workspace [h/head_dim, n] fp32 (filled by
 * lemo_attn_delta); each dK/dV CTA accumulates over the h/kv query heads of
 * its group (grouped-query attention). */
int lemo_flash_bwd_tc(const void* q, const void* k, const void* v, const void* o,
                      const void* dout, const float* lse, float* delta, float* dq, float* dk,
                      float* dv, int n, int h, int kv, int head_dim, float scale, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* LEMO_H_ */
