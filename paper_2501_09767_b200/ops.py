"""Thin torch-tensor wrappers over the liblemo C ABI (include/lemo.h).

Each wrapper checks devices/dtypes/shapes on the host (raising the
reference's exception types) and calls the corresponding ``lemo_*`` entry
point on torch's current stream.  There is no non-CUDA path: a CPU tensor is
a ContractError and a missing library is a LemoError.
"""

from __future__ import annotations

import math

import torch

from ._lib import INSTRUMENT, call, lib, ptr, stream_ptr
from .errors import ContractError, DimensionError

BF16 = torch.bfloat16
F32 = torch.float32
F64 = torch.float64
I32 = torch.int32


def _check(*ts):
    for t in ts:
        if t is None:
            continue
        if not t.is_cuda:
            raise ContractError("liblemo operands must be CUDA tensors (there is no CPU path)")


def _dt(t, dtype, name):
    if t is not None and t.dtype != dtype:
        raise ContractError(f"{name} must be {dtype}, got {t.dtype}")


def _rowmajor(t, name):
    if t is not None and (t.dim() != 2 or t.stride(1) != 1):
        raise ContractError(f"{name} must be a row-major 2-D tensor")


def _s():
    return stream_ptr()


# ---------------------------------------------------------------------------
# tcgen05 GEMMs   C = A · Bᵀ  (B given as [N, K])


def _mnk(a, b):
    _check(a, b)
    _dt(a, BF16, "A")
    _dt(b, BF16, "B")
    _rowmajor(a, "A")
    _rowmajor(b, "B")
    M, K = a.shape
    N, K2 = b.shape
    if K != K2:
        raise DimensionError(f"matmul inner extents differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    return M, N, K


def gemm_bf16(a, b, out=None):
    M, N, K = _mnk(a, b)
    if out is None:
        out = torch.empty(M, N, dtype=BF16, device=a.device)
    call("lemo_gemm_bf16", ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(out), out.stride(0), M, N,
         K, _s())
    return out


def gemm_f32(a, b, out=None, *, accumulate=False):
    """out (+)= a·bᵀ in fp32."""
    M, N, K = _mnk(a, b)
    _check(out)
    if out is None:
        out = torch.empty(M, N, dtype=F32, device=a.device)
    call("lemo_gemm_f32", ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(out), out.stride(0), M, N,
         K, int(bool(accumulate)), _s())
    return out


def gemm_f32_exact(a, b, out=None, *, accumulate=False):
    """out (+)= a·bᵀ in fp32 with promoted (round-to-nearest) accumulation --
    for bf16x3 operand pairs whose product must keep fp32 precision."""
    M, N, K = _mnk(a, b)
    _check(out)
    if out is None:
        out = torch.empty(M, N, dtype=F32, device=a.device)
    call("lemo_gemm_f32_exact", ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(out), out.stride(0),
         M, N, K, int(bool(accumulate)), _s())
    return out


def gemm_scatter_add(a, b, resid, idx=None):
    """resid[idx] += a·bᵀ in place (idx None = identity rows)."""
    M, N, K = _mnk(a, b)
    _check(resid, idx)
    _dt(resid, F32, "resid")
    if idx is not None and idx.shape[0] != M:
        raise DimensionError("scatter index length must equal the GEMM row count")
    call("lemo_gemm_scatter_add", ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(resid),
         resid.stride(0), ptr(idx), M, N, K, _s())
    return resid


def gemm_qkv(xn, w_qkv_t, *, h, head_dim, rope, inv_freq, pos, nmat=3, kv=None, out=None,
             row_scale=None):
    """q [M, h], k(, v) [M, kv] = rope(xn·Wᵀ) at positions pos over K =
    xn.shape[1] columns (h, or h + 64 with the LoRA K-extension) — see
    lemo_gemm_qkv.  kv < h: grouped-query attention (kv = n_kv_heads·head_dim)."""
    M, K = xn.shape
    kv = h if kv is None else kv
    _check(xn, w_qkv_t, pos, inv_freq)
    if w_qkv_t.shape[1] < K or w_qkv_t.shape[0] < h + (nmat - 1) * kv:
        raise DimensionError("q/k/v weight does not cover the requested output")
    if out is None:
        out = [torch.empty(M, h if i == 0 else kv, dtype=BF16, device=xn.device)
               for i in range(nmat)]
    q, k = out[0], out[1]
    v = out[2] if nmat == 3 else None
    call("lemo_gemm_qkv", ptr(xn), xn.stride(0), ptr(w_qkv_t), w_qkv_t.stride(0), M, h, kv, K,
         nmat, ptr(q), ptr(k), ptr(v), head_dim, int(bool(rope)), ptr(inv_freq), ptr(pos),
         ptr(row_scale), _s())
    return out


def gemm_gateup(xn, w_gu_t, *, gu=None, inner=None, partial=None, relu=False, exact_score=False,
                row_scale=None):
    """exact_score=True: xn / w_gu_t are bf16x3 operands (K = 3h) and the MLP
    scores come from the fp32 accumulator (parity mode).  row_scale: per-row
    factor on the accumulator (xn given as bf16(x·w), rmsnorm_gather_fold)."""
    M, K = xn.shape
    N = w_gu_t.shape[0]
    _check(xn, w_gu_t, gu, inner, partial, row_scale)
    if w_gu_t.shape[1] != K or w_gu_t.stride(0) != K:
        raise DimensionError(f"gate/up weight {tuple(w_gu_t.shape)} does not match K = {K}")
    INSTRUMENT.note("lemo_gemm_gateup", (M, N, K, bool(exact_score)))
    call("lemo_gemm_gateup", ptr(xn), xn.stride(0), ptr(w_gu_t), M, N, K, ptr(gu), ptr(inner),
         ptr(partial), int(bool(relu)), int(bool(exact_score)), ptr(row_scale), _s())


def gemm_dgateup(dy, w_down, gu, dgu, *, m_pad, relu=False):
    M, h = dy.shape
    _check(dy, w_down, gu, dgu)
    call("lemo_gemm_dgateup", ptr(dy), ptr(w_down), M, m_pad, h, ptr(gu), ptr(dgu),
         int(bool(relu)), _s())


# ---------------------------------------------------------------------------
# row kernels


def rmsnorm_gather(x, w, idx=None, *, xn=None, xg=None, inv=None):
    """Fused gather + RMSNorm."""
    _check(x, w, idx)
    _dt(x, F32, "x")
    M = x.shape[0] if idx is None else idx.shape[0]
    h = x.shape[1]
    if xn is None:
        xn = torch.empty(M, h, dtype=BF16, device=x.device)
    call("lemo_rmsnorm_gather", ptr(x), x.stride(0), ptr(idx), M, h, ptr(w), ptr(xn),
         xn.stride(0), ptr(xg), ptr(inv), _s())
    return xn


LORA_K_EXT = 64  # extra K columns of the q/k/v GEMM carrying the LoRA terms


def rmsnorm_gather_fold(x, w, idx=None, *, inv, out=None):
    """bf16(x[idx]·w) rows and inv = 1/rms (the normalisation applied later as
    the GEMM epilogue's row scale)."""
    _check(x, w, idx, inv, out)
    _dt(x, F32, "x")
    M = x.shape[0] if idx is None else idx.shape[0]
    h = x.shape[1]
    if out is None:
        out = torch.empty(M, h, dtype=BF16, device=x.device)
    call("lemo_rmsnorm_gather_fold", ptr(x), x.stride(0), ptr(idx), M, h, ptr(w), ptr(out),
         out.stride(0), ptr(inv), _s())
    return out


def rmsnorm_f32(x, w, idx=None, *, out=None, inv=None):
    """fp32 RMSNorm rows (model.py:333-335), optionally gathered at idx."""
    _check(x, w, idx, out, inv)
    _dt(x, F32, "x")
    M = x.shape[0] if idx is None else idx.shape[0]
    h = x.shape[1]
    if out is None:
        out = torch.empty(M, h, dtype=F32, device=x.device)
    call("lemo_rmsnorm_f32", ptr(x), x.stride(0), ptr(idx), M, h, ptr(w), ptr(out), out.stride(0),
         ptr(inv), _s())
    return out


def qk_finish(qk, t, Bq, *, r, scale, rope_tab, h, kv, head_dim, rope):
    """fp32 layer_qk tail (LoRA add + RoPE) -> (q_hi, q_lo, k_hi, k_lo) bf16."""
    _check(qk, t, Bq, rope_tab)
    _dt(qk, F32, "qk")
    s = qk.shape[0]
    dev = qk.device
    q_hi, q_lo = (torch.empty(s, h, dtype=BF16, device=dev) for _ in range(2))
    k_hi, k_lo = (torch.empty(s, kv, dtype=BF16, device=dev) for _ in range(2))
    if rope and (rope_tab is None or rope_tab.shape[0] < s):
        raise ContractError("RoPE table shorter than the sequence")
    call("lemo_qk_finish", ptr(qk), qk.stride(0), ptr(t), 0 if t is None else t.stride(0),
         ptr(Bq), int(r), float(scale), ptr(rope_tab), s, h, kv, head_dim, int(bool(rope)),
         ptr(q_hi), ptr(q_lo), ptr(k_hi), ptr(k_lo), _s())
    return q_hi, q_lo, k_hi, k_lo


def split_bf16x2(a):
    """fp32 [M, K] -> bf16 [M, 2K] = [hi | lo] (A operand against [W | W])."""
    _check(a)
    _dt(a, F32, "a")
    _rowmajor(a, "a")
    M, K = a.shape
    out = torch.empty(M, 2 * K, dtype=BF16, device=a.device)
    call("lemo_split_bf16x2", ptr(a), a.stride(0), M, K, ptr(out), _s())
    return out


def split_hilo(a):
    """fp32 [M, K] -> (bf16 hi, bf16 lo) with a ≈ hi + lo."""
    _check(a)
    _dt(a, F32, "a")
    _rowmajor(a, "a")
    M, K = a.shape
    hi = torch.empty(M, K, dtype=BF16, device=a.device)
    lo = torch.empty_like(hi)
    call("lemo_split_hilo", ptr(a), a.stride(0), M, K, ptr(hi), ptr(lo), _s())
    return hi, lo


def lora_qkv_prep(t, r, scale, xn_ext, h):
    """xn_ext[:, h:h+64] = [s·t_q | s·t_v | 0] (bf16)."""
    _check(t, xn_ext)
    call("lemo_lora_qkv_prep", ptr(t), t.stride(0), xn_ext.shape[0], 2 * r, float(scale),
         ptr(xn_ext), xn_ext.stride(0), h, _s())


def lora_pack_b(Bq, Bv, r, w_ext, h):
    """w_ext[:, h:h+64] = [B_qᵀ | B_vᵀ | 0] on the q / v rows (bf16); B_v is [r, kv]."""
    _check(Bq, Bv, w_ext)
    call("lemo_lora_pack_b", ptr(Bq), ptr(Bv), h, Bv.shape[1], r, ptr(w_ext), w_ext.stride(0),
         _s())


LORA_T_COLS = 32  # t / u buffers are [k, 32] (2r <= 32, zero-padded)


def lora_pack(A, r, out=None):
    """[h, 2r] interleaved LoRA A (fp32) -> [32, h] bf16 GEMM operand."""
    _check(A, out)
    h = A.shape[0]
    if out is None:
        out = torch.empty(LORA_T_COLS, h, dtype=BF16, device=A.device)
    call("lemo_lora_pack", ptr(A), A.stride(0), h, 2 * r, ptr(out), _s())
    return out


def lora_down(xn, A_packed, t=None):
    """t = xn · [A_q | A_v]  ([k, 32] fp32, columns >= 2r are zero)."""
    return gemm_f32(xn, A_packed, out=t)


def gather_rows_bf16(src, idx, out=None):
    _check(src, idx)
    M = src.shape[0] if idx is None else idx.shape[0]
    h = src.shape[1]
    if out is None:
        out = torch.empty(M, h, dtype=BF16, device=src.device)
    call("lemo_gather_rows_bf16", ptr(src), src.stride(0), ptr(idx), M, h, ptr(out), _s())
    return out


def rmsnorm_bwd(g, x, inv, w, dx, idx=None, *, gscale=1.0, accumulate=True):
    _check(g, x, inv, w, dx, idx)
    M, h = g.shape
    call("lemo_rmsnorm_bwd", ptr(g), g.stride(0), ptr(x), int(x.dtype == BF16), x.stride(0),
         ptr(inv), ptr(w), ptr(idx), M, h, float(gscale), ptr(dx), dx.stride(0),
         int(bool(accumulate)), _s())
    return dx


def embed(ids, table, pos_table=None, out=None):
    _check(ids, table, pos_table)
    n = ids.shape[0]
    h = table.shape[1]
    if out is None:
        out = torch.empty(n, h, dtype=F32, device=table.device)
    call("lemo_embed", ptr(ids), n, ptr(table), h, ptr(pos_table), ptr(out), _s())
    return out


def mlp_compact(gu_all, x, inv_all, idx, *, m_pad, relu, gu_out, inner_out, xg_out, inv_out):
    _check(gu_all, x, inv_all, idx, gu_out, inner_out, xg_out, inv_out)
    M = idx.shape[0]
    h = x.shape[1]
    call("lemo_mlp_compact", ptr(gu_all), ptr(x), x.stride(0), ptr(inv_all), ptr(idx), M, h, m_pad,
         int(bool(relu)), ptr(gu_out), ptr(inner_out), ptr(xg_out), ptr(inv_out), _s())


def qkv_grad_prep(dq, dk, dv, *, head_dim, rope, rope_tab, pos, dqkv):
    """RoPE backward of dq (in place, fp32) / dk and the bf16 [dq|dk|dv] rows."""
    _check(dq, dk, dv, pos, dqkv)
    M, h = dq.shape
    call("lemo_qkv_grad_prep", ptr(dq), ptr(dk), ptr(dv), M, h, dk.shape[1], head_dim,
         int(bool(rope)), ptr(rope_tab), ptr(pos), ptr(dqkv), dqkv.stride(0), _s())
    return dqkv


def lora_pack_bt(Bq, Bv, r, h, out=None):
    """[32, h+2kv] bf16 LoRA B operand of u = dqkv·Btᵀ (lemo_lora_pack_bt)."""
    _check(Bq, Bv, out)
    kv = Bv.shape[1]
    if out is None:
        out = torch.empty(LORA_T_COLS, h + 2 * kv, dtype=BF16, device=Bq.device)
    call("lemo_lora_pack_bt", ptr(Bq), ptr(Bv), h, kv, r, ptr(out), _s())
    return out


def lora_pack_a_ext(A, r, w_ext, col0):
    """w_ext[:, col0:col0+64] = [A_q | A_v | 0] (bf16): LoRA K-extension of a dX weight."""
    _check(A, w_ext)
    call("lemo_lora_pack_a_ext", ptr(A), A.stride(0), A.shape[0], 2 * r, ptr(w_ext),
         w_ext.stride(0), col0, _s())


def lora_grads(xg, inv, w, t, u, g0, g1, *, r, scale, dA, dB0, dB1):
    """dA (= [h, 2r] interleaved q|v), dB0, dB1 accumulated in place."""
    _check(xg, inv, w, t, u, g0, g1, dA, dB0, dB1)
    M, h = xg.shape
    ws = torch.empty(max(1, lib().lemo_lora_grads_workspace(M, h, r)), dtype=torch.float32,
                     device=xg.device)
    call("lemo_lora_grads", ptr(xg), ptr(inv), ptr(w), ptr(t), ptr(u), t.stride(0), ptr(g0),
         ptr(g1), M, h, g1.shape[1], r, float(scale), dA.stride(0), ptr(dA), ptr(dB0),
         ptr(dA[:, r:]), ptr(dB1), ptr(ws), _s())


def ce_rows(logits, targets, *, V, ignore, inv_count, dlogits, row_loss, bad=None):
    """Targets are validated on the host (check_targets); an out-of-range one
    that reaches the kernel anyway makes the loss NaN (and sets `bad`)."""
    _check(logits, targets, dlogits, row_loss, bad)
    n = logits.shape[0]
    call("lemo_ce_rows", ptr(logits), logits.stride(0), ptr(targets), n, V, ignore,
         float(inv_count), ptr(dlogits), dlogits.stride(0), ptr(row_loss), ptr(bad), _s())


def sum_f64(x, out, accumulate=False):
    _check(x, out)
    call("lemo_sum_f64", ptr(x), x.numel(), ptr(out), int(bool(accumulate)), _s())
    return out


def adam(p, g, m, v, *, lr, b1, b2, eps, wd, bc1, bc2, guard_loss=None, guard_latch=None):
    """Adam step in place; with guard_loss (device f64 scalar) the update is
    skipped when the loss is not finite or guard_latch is already set."""
    _check(p, g, m, v, guard_loss, guard_latch)
    call("lemo_adam", ptr(p), ptr(g), ptr(m), ptr(v), p.numel(), float(lr), float(b1), float(b2),
         float(eps), float(wd), float(bc1), float(bc2), ptr(guard_loss), ptr(guard_latch), _s())


# ---------------------------------------------------------------------------
# scoring / selection


def block_embed(x, b, out=None):
    _check(x)
    _dt(x, F32, "x")
    s, h = x.shape
    if s % b != 0:
        raise ContractError(f"sequence length {s} not a multiple of block size {b}")
    if out is None:
        out = torch.empty(s // b, h, dtype=F32, device=x.device)
    call("lemo_block_embed", ptr(x), x.stride(0), s, h, b, ptr(out), _s())
    return out


def split_bf16x3(a, pattern, out=None):
    """fp32 [M, K] -> bf16 [M, 3K] operand ([hi|hi|lo] pattern 0, [hi|lo|hi] pattern 1)."""
    _check(a, out)
    _dt(a, F32, "a")
    M, K = a.shape
    if out is None:
        out = torch.empty(M, 3 * K, dtype=BF16, device=a.device)
    call("lemo_split_bf16x3", ptr(a), a.stride(0), M, K, int(pattern), ptr(out), _s())
    return out


def split_bf16x3_t(a, pattern, out=None):
    """fp32 [R, C] -> bf16 [C, 3R]: the bf16x3 operand of aᵀ."""
    _check(a, out)
    _dt(a, F32, "a")
    R, C = a.shape
    if out is None:
        out = torch.empty(C, 3 * R, dtype=BF16, device=a.device)
    call("lemo_split_bf16x3_t", ptr(a), a.stride(0), R, C, int(pattern), ptr(out), _s())
    return out


def tril_mse(full, label, *, dfull=None, row_loss=None, loss=None):
    """Packed-lower-triangle MSE of `full` [nb, nb] vs `label` [nb(nb+1)/2]:
    returns (loss f64 [1] device, dL/dfull [nb, nb])."""
    _check(full, label)
    _dt(full, F32, "full")
    _dt(label, F32, "label")
    nb = full.shape[0]
    if label.numel() != nb * (nb + 1) // 2:
        raise DimensionError(f"label has {label.numel()} entries, expected {nb * (nb + 1) // 2}")
    dev = full.device
    dfull = torch.empty(nb, nb, dtype=F32, device=dev) if dfull is None else dfull
    row_loss = torch.empty(nb, dtype=torch.float64, device=dev) if row_loss is None else row_loss
    loss = torch.empty(1, dtype=torch.float64, device=dev) if loss is None else loss
    call("lemo_tril_mse", ptr(full), full.stride(0), ptr(label), nb, ptr(dfull), dfull.stride(0),
         ptr(row_loss), _s())
    call("lemo_sum_d", ptr(row_loss), nb, 2.0 / (nb * (nb + 1)), ptr(loss), _s())
    return loss, dfull


def relu_grad(dh, h):
    """dh[h <= 0] = 0 in place (ReLU·mask backward)."""
    _check(dh, h)
    call("lemo_relu_grad", ptr(dh), ptr(h), dh.numel(), _s())
    return dh


def block_expand(g, b, out=None):
    """[nb, w] -> [nb·b, w], rows repeated b times and divided by b."""
    _check(g, out)
    nb, w = g.shape
    if out is None:
        out = torch.empty(nb * b, w, dtype=F32, device=g.device)
    call("lemo_block_expand", ptr(g), nb, w, b, ptr(out), _s())
    return out


def zero_count(h, counts):
    """counts[c] += #zeros in column c of h [M, N] (int64 counts)."""
    _check(h, counts)
    M, N = h.shape
    call("lemo_zero_count", ptr(h), h.stride(0), M, N, ptr(counts), _s())
    return counts


def gemm_split3(a3, b3, *, relu=False, mask=None, pattern=0, split_out=True, f32_out=False):
    """C = act(A·Bᵀ)·mask in fp32-faithful bf16x3; returns (split C or None, fp32 C or None)."""
    _check(a3, b3, mask)
    M, K3 = a3.shape
    N = b3.shape[0]
    if b3.shape[1] != K3:
        raise DimensionError(f"bf16x3 inner extents differ: {tuple(a3.shape)} vs {tuple(b3.shape)}")
    out = torch.empty(M, 3 * N, dtype=BF16, device=a3.device) if split_out else None
    f32 = torch.empty(M, N, dtype=F32, device=a3.device) if f32_out else None
    call("lemo_gemm_split3", ptr(a3), a3.stride(0), ptr(b3), b3.stride(0), M, N, K3,
         int(bool(relu)), ptr(mask), int(pattern), ptr(out), 0 if out is None else out.stride(0),
         ptr(f32), 0 if f32 is None else f32.stride(0), _s())
    return out, f32


def gemm_split3_dual(a3, b3, nsplit, *, relu=False, mask=None):
    """Two predictor layers over the same bf16x3 input in one GEMM (weights
    stacked along N): returns the split forms (pattern 0) of columns
    [0, nsplit) and [nsplit, N)."""
    _check(a3, b3, mask)
    M, K3 = a3.shape
    N = b3.shape[0]
    if b3.shape[1] != K3:
        raise DimensionError(f"bf16x3 inner extents differ: {tuple(a3.shape)} vs {tuple(b3.shape)}")
    out = torch.empty(M, 3 * nsplit, dtype=BF16, device=a3.device)
    out2 = torch.empty(M, 3 * (N - nsplit), dtype=BF16, device=a3.device)
    call("lemo_gemm_split3_dual", ptr(a3), a3.stride(0), ptr(b3), b3.stride(0), M, N, K3, nsplit,
         int(bool(relu)), ptr(mask), ptr(out), out.stride(0), ptr(out2), out2.stride(0), _s())
    return out, out2


def colsum_clamped(S, out=None):
    _check(S)
    nb = S.shape[0]
    if out is None:
        out = torch.empty(nb, dtype=F64, device=S.device)
    call("lemo_colsum_clamped", ptr(S), S.stride(0), nb, ptr(out), _s())
    return out


def pack_tril(S, *, clamp=False, dtype=F64):
    """Packed lower triangle (row-major, n <= m) of a dense fp32 [nb, nb]."""
    _check(S)
    _dt(S, F32, "S")
    nb = S.shape[0]
    out = torch.empty(nb * (nb + 1) // 2, dtype=dtype, device=S.device)
    call("lemo_pack_tril", ptr(S), S.stride(0), nb, int(bool(clamp)),
         ptr(out) if dtype == F64 else None, ptr(out) if dtype == F32 else None, _s())
    return out


def colsum_packed(packed, nb, out=None):
    """f64 column sums of a packed f64 lower triangle, ascending m."""
    _check(packed, out)
    _dt(packed, torch.float64, "packed")
    if packed.numel() != nb * (nb + 1) // 2:
        raise DimensionError(f"packed triangle has {packed.numel()} entries for {nb} blocks")
    if out is None:
        out = torch.empty(nb, dtype=torch.float64, device=packed.device)
    call("lemo_colsum_packed", ptr(packed), nb, ptr(out), _s())
    return out


def mlp_block_scores(partial, *, s, n_valid, b, m_real, out=None):
    _check(partial)
    nb = -(-s // b)
    if out is None:
        out = torch.empty(nb, dtype=F64, device=partial.device)
    call("lemo_mlp_block_scores", ptr(partial), partial.shape[0], s, n_valid, b, m_real, ptr(out),
         _s())
    return out


def mlp_token_band(partial, vec, thr, margin, *, n_valid, b, m_real, out=None):
    _check(partial, vec, out)
    _dt(vec, F64, "scores")
    s = partial.shape[1]
    out = torch.empty(s, dtype=F64, device=partial.device) if out is None else out
    call("lemo_mlp_token_band", ptr(partial), partial.shape[0], s, n_valid, b, m_real, ptr(vec),
         float(thr), float(margin), ptr(out), _s())
    return out


def mlp_patch_rows(partial, tok, *, b, m_real, vec, count=None, overflow=None):
    _check(partial, tok, vec, count, overflow)
    call("lemo_mlp_patch_rows", ptr(partial), partial.shape[0], partial.shape[1], ptr(tok),
         ptr(count), b, m_real, ptr(vec), ptr(overflow), _s())
    return vec


def select(vec, *, b, n_tokens, thr=0.0, thr_dev=None, force=None, mask, blocks, tokens, counts,
           thr_out=None):
    _check(vec, thr_dev, force, mask, blocks, tokens, counts, thr_out)
    _dt(vec, F64, "scores")
    nb = vec.shape[0]
    call("lemo_select", ptr(vec), nb, float(thr), ptr(thr_dev), ptr(force), b, n_tokens, ptr(mask),
         ptr(blocks), ptr(tokens), ptr(counts), ptr(thr_out), _s())


def quantile_lower(data, q, out, *, plus_one=False):
    """out = np.quantile(data, q, method='lower') (rank computed exactly like numpy)."""
    _check(data, out)
    n = data.numel()
    rank = n - 1 if plus_one else int(math.floor((n - 1) * q))
    call("lemo_quantile_lower", ptr(data), n, rank, int(bool(plus_one)), ptr(out), _s())
    return out


# ---------------------------------------------------------------------------
# attention


def flash_fwd(q, k, v, *, head_dim, scale, o=None, lse=None):
    """Causal attention forward on the tcgen05 kernel (head_dim 64 or 128);
    k, v may carry fewer heads than q (grouped-query attention)."""
    _check(q, k, v)
    n, h = q.shape
    if o is None:
        o = torch.empty(n, h, dtype=BF16, device=q.device)
    if lse is None:
        lse = torch.empty(h // head_dim, n, dtype=F32, device=q.device)
    INSTRUMENT.note("lemo_flash_fwd_tc", n)
    call("lemo_flash_fwd_tc", ptr(q), ptr(k), ptr(v), ptr(o), ptr(lse), n, h, k.shape[1],
         head_dim, float(scale), _s())
    return o, lse


def flash_bwd(q, k, v, o, dout, lse, *, head_dim, scale, dq=None, dk=None, dv=None):
    """Causal attention backward on the tcgen05 kernels (head_dim 64 or 128)."""
    _check(q, k, v, o, dout, lse)
    n, h = q.shape
    dev = q.device
    kv = k.shape[1]
    delta = torch.empty(h // head_dim, n, dtype=F32, device=dev)
    dq = torch.empty(n, h, dtype=F32, device=dev) if dq is None else dq
    dk = torch.empty(n, kv, dtype=F32, device=dev) if dk is None else dk
    dv = torch.empty(n, kv, dtype=F32, device=dev) if dv is None else dv
    INSTRUMENT.note("lemo_flash_bwd_tc", n)
    call("lemo_flash_bwd_tc", ptr(q), ptr(k), ptr(v), ptr(o), ptr(dout), ptr(lse), ptr(delta),
         ptr(dq), ptr(dk), ptr(dv), n, h, kv, head_dim, float(scale), _s())
    return dq, dk, dv
