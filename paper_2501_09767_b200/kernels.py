"""Permutation-free sparse execution and segment-based loss on the GPU.

Mirrors ``sparsetune.kernels`` (kernels.py:25-288).  The reference gathers
retained rows, runs the block on them and scatter-adds the result into a
copy of the residual stream; here every step is a liblemo kernel:

  attention block  gather+RMSNorm(+LoRA x·A)  → tcgen05 q/k/v GEMM with the
                   LoRA side term and RoPE at the ORIGINAL positions in its
                   epilogue → causal flash attention on the compact sequence
                   → tcgen05 output projection whose epilogue adds each row
                   into the residual at idx[row] (in place, no atomics)
  MLP block        gather+RMSNorm → tcgen05 gate/up GEMM (SwiGLU in the
                   epilogue) → tcgen05 down projection with the same
                   index-remapped residual epilogue; when the MLP scorer has
                   already produced gate/up for every row, the retained rows
                   are compacted instead of recomputed
  backward         only compact retained-row buffers are saved (tensor.py:
                   578-597 semantics); gradients are gathered from the
                   residual gradient, pushed through dX-only GEMMs (frozen
                   weights get no dW) and RMSNorm backward scatter-adds them
                   back at idx.

The block functions operate IN PLACE on a float32 residual stream `x`
[n_tokens, h]; the reference-named wrappers at the bottom keep the
reference's value semantics (they return a new tensor).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import ContractError

BF16, F32 = torch.bfloat16, torch.float32


class GatherPlan:
    """Sorted retained token indices within a sequence of n_tokens
    (kernels.py:25-55); indices live on the device as int32."""

    __slots__ = ("indices", "n_tokens", "k")

    def __init__(self, indices, n_tokens: int, *, device=None, _trusted: bool = False):
        if isinstance(indices, torch.Tensor) and indices.is_cuda and _trusted:
            self.indices = indices
            self.k = int(indices.shape[0])
            self.n_tokens = n_tokens
            return
        idx = np.asarray(indices.cpu() if isinstance(indices, torch.Tensor) else indices,
                         dtype=np.int64)
        if idx.ndim != 1:
            raise ContractError("plan indices must be one-dimensional")
        if idx.size:
            if (np.diff(idx) <= 0).any():
                raise ContractError("plan indices must be strictly increasing")
            if idx[0] < 0 or idx[-1] >= n_tokens:
                raise ContractError(f"plan indices out of range [0, {n_tokens})")
        dev = device or (indices.device if isinstance(indices, torch.Tensor) and indices.is_cuda
                         else torch.device("cuda"))
        self.indices = torch.as_tensor(idx.astype(np.int32)).to(dev)
        self.k = int(idx.size)
        self.n_tokens = n_tokens

    @staticmethod
    def full(n_tokens: int, device=None) -> "GatherPlan":
        dev = device or torch.device("cuda")
        return GatherPlan(torch.arange(n_tokens, dtype=torch.int32, device=dev), n_tokens,
                          _trusted=True)

    @staticmethod
    def empty(n_tokens: int, device=None) -> "GatherPlan":
        dev = device or torch.device("cuda")
        return GatherPlan(torch.empty(0, dtype=torch.int32, device=dev), n_tokens, _trusted=True)

    @staticmethod
    def from_pattern(pattern, n_tokens: int, device) -> "GatherPlan":
        """Device indices straight from the select kernel (already sorted)."""
        return GatherPlan(pattern.device_token_indices(device), n_tokens, _trusted=True)


@dataclass(frozen=True)
class SegmentPlan:
    """Contiguous partition of [0, n_tokens) into non-empty segments (kernels.py:58-88)."""

    n_tokens: int
    boundaries: tuple

    def __post_init__(self):
        b = tuple(int(x) for x in self.boundaries)
        object.__setattr__(self, "boundaries", b)
        if len(b) < 2 or b[0] != 0 or b[-1] != self.n_tokens:
            raise ContractError(f"boundaries must span [0, {self.n_tokens}], got {b}")
        if any(b[i + 1] <= b[i] for i in range(len(b) - 1)):
            raise ContractError(f"every segment must be non-empty, got {b}")

    @property
    def n_segments(self) -> int:
        return len(self.boundaries) - 1

    @property
    def segments(self):
        return [(self.boundaries[i], self.boundaries[i + 1]) for i in range(self.n_segments)]

    @staticmethod
    def even(n_tokens: int, n_segments: int) -> "SegmentPlan":
        if n_segments < 1 or n_segments > n_tokens:
            raise ContractError(f"cannot split {n_tokens} tokens into {n_segments} non-empty "
                                "segments")
        return SegmentPlan(n_tokens, tuple(round(i * n_tokens / n_segments)
                                           for i in range(n_segments + 1)))


# ---------------------------------------------------------------------------
# attention block


def attention_forward(x: torch.Tensor, plan: GatherPlan, layer, *, save: bool = True,
                      out: torch.Tensor | None = None, pos: torch.Tensor | None = None):
    """x[idx] += attention_core(gather_rmsnorm(x, idx)) in place; returns the
    compact saved state (or None when save=False / k == 0).  `out` (default
    x) receives the update instead; `pos` (default idx) are the RoPE
    positions -- the naive variant runs on a materialised compact copy whose
    row i sits at original position pos[i]."""
    if plan.k == 0:
        return None
    k, h = plan.k, x.shape[1]
    dev = x.device
    idx = plan.indices
    pos = idx if pos is None else pos
    r = layer.lora_rank
    xn = torch.empty(k, layer.w_qkv_t.shape[1], dtype=BF16, device=dev)  # [xn | LoRA ext]
    xg = torch.empty(k, h, dtype=BF16, device=dev) if save else None
    inv = torch.empty(k, dtype=F32, device=dev) if save else None
    ops.rmsnorm_gather(x, layer.attn_norm_w, idx, xn=xn, xg=xg, inv=inv)
    t = layer.qkv_input(xn) if r else None
    q, kk, v = ops.gemm_qkv(xn, layer.w_qkv_t, h=h, head_dim=layer.head_dim, rope=layer.rope,
                            inv_freq=layer.inv_freq, pos=pos, kv=layer.kv)
    del xn
    o, lse = ops.flash_fwd(q, kk, v, head_dim=layer.head_dim, scale=1.0 / math.sqrt(layer.head_dim))
    ops.gemm_scatter_add(o, layer.w_o_t, x if out is None else out, idx)
    if not save:
        return None
    return dict(idx=idx, pos=pos, xg=xg, inv=inv, t=t, q=q, k=kk, v=v, o=o, lse=lse)


_SIDE: dict = {}
_SERIAL = os.environ.get("LEMO_SERIAL_LORA_GRADS", "0") == "1"  # A/B switch


def _side_stream(dev) -> torch.cuda.Stream:
    """Per-device side stream for the memory-bound LoRA weight-gradient kernel,
    which then runs under the compute-bound dX GEMM of the same layer."""
    key = dev.index if dev.index is not None else torch.cuda.current_device()
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=dev)
    return _SIDE[key]


def attention_backward(dx: torch.Tensor, saved: dict, layer, grads):
    """dx[idx] += d(attention block)/dx (in place); LoRA grads accumulated
    into grads = (dA_qv, dBq, dBv) views of the flat gradient buffer.  The
    LoRA-gradient kernel runs on a side stream, overlapping the dX GEMM;
    returns the event the caller must wait on before reading `grads`
    (None when there is nothing pending)."""
    idx = saved["idx"]
    k, h = idx.shape[0], dx.shape[1]
    dev = dx.device
    r = layer.lora_rank
    dy = ops.gather_rows_bf16(dx, idx)
    d_o = ops.gemm_bf16(dy, layer.w_o)
    del dy
    dq, dk, dv = ops.flash_bwd(saved["q"], saved["k"], saved["v"], saved["o"], d_o, saved["lse"],
                               head_dim=layer.head_dim, scale=1.0 / math.sqrt(layer.head_dim))
    del d_o
    dqkv = torch.empty(k, layer.w_qkv.shape[1], dtype=BF16, device=dev)  # [dq|dk|dv|LoRA ext]
    ops.qkv_grad_prep(dq, dk, dv, head_dim=layer.head_dim, rope=layer.rope,
                      rope_tab=layer.rope_tab, pos=saved.get("pos", idx), dqkv=dqkv)
    done = None
    if r:
        u = layer.qkv_grad_input(dqkv)
        if grads is not None and not _SERIAL:
            dA, dBq, dBv = grads
            side = _side_stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                ops.lora_grads(saved["xg"], saved["inv"], layer.attn_norm_w, saved["t"], u, dq,
                               dv, r=r, scale=layer.lora_scaling, dA=dA, dB0=dBq, dB1=dBv)
                done = torch.cuda.Event()
                done.record(side)
            for t in (saved["xg"], saved["inv"], saved["t"], u, dq, dv):
                t.record_stream(side)  # allocator: in use on the side stream
        elif grads is not None:
            dA, dBq, dBv = grads
            ops.lora_grads(saved["xg"], saved["inv"], layer.attn_norm_w, saved["t"], u, dq, dv,
                           r=r, scale=layer.lora_scaling, dA=dA, dB0=dBq, dB1=dBv)
    del dq, dk, dv
    dxn = ops.gemm_f32(dqkv, layer.w_qkv)  # LoRA term inside the K-extension
    ops.rmsnorm_bwd(dxn, saved["xg"], saved["inv"], layer.attn_norm_w, dx, idx, accumulate=True)
    return done


# ---------------------------------------------------------------------------
# MLP block


def mlp_forward(x: torch.Tensor, plan: GatherPlan, layer, *, scored=None, save: bool = True,
                out: torch.Tensor | None = None):
    """x[idx] += mlp_core(gather_rmsnorm(x, idx)) in place (into `out` when
    given).  `scored` = (gu_all, inv_all) from the MLP scorer over every row
    of this same x: retained rows are then compacted instead of recomputed."""
    if plan.k == 0:
        return None
    k, h = plan.k, x.shape[1]
    dev = x.device
    idx = plan.indices
    N = layer.w_gu_t.shape[0]
    gu = torch.empty(k, N, dtype=BF16, device=dev)
    inner = torch.empty(k, layer.m_pad, dtype=BF16, device=dev)
    xg = torch.empty(k, h, dtype=BF16, device=dev)
    inv = torch.empty(k, dtype=F32, device=dev)
    if scored is not None:
        gu_all, inv_all = scored
        ops.mlp_compact(gu_all, x, inv_all, idx, m_pad=layer.m_pad, relu=layer.relu, gu_out=gu,
                        inner_out=inner, xg_out=xg, inv_out=inv)
    else:
        xn = ops.rmsnorm_gather(x, layer.mlp_norm_w, idx, xg=xg, inv=inv)
        ops.gemm_gateup(xn, layer.w_gu_t, gu=gu, inner=inner, relu=layer.relu)
        del xn
    ops.gemm_scatter_add(inner, layer.w_down_t, x if out is None else out, idx)
    if not save:
        return None
    return dict(idx=idx, xg=xg, inv=inv, gu=gu)


def mlp_backward(dx: torch.Tensor, saved: dict, layer) -> None:
    idx = saved["idx"]
    k = idx.shape[0]
    dy = ops.gather_rows_bf16(dx, idx)
    dgu = torch.empty(k, layer.w_gu_t.shape[0], dtype=BF16, device=dx.device)
    ops.gemm_dgateup(dy, layer.w_down, saved["gu"], dgu, m_pad=layer.m_pad, relu=layer.relu)
    del dy
    dxn = ops.gemm_f32(dgu, layer.w_gu)
    del dgu
    ops.rmsnorm_bwd(dxn, saved["xg"], saved["inv"], layer.mlp_norm_w, dx, idx, accumulate=True)


# ---------------------------------------------------------------------------
# segment-based loss (kernels.py:229-288): logits of one segment at a time,
# CE + dlogits + grad_hidden computed in the forward pass.


def segmented_loss_forward(hidden: torch.Tensor, lm_head_t: torch.Tensor, lm_head: torch.Tensor,
                           targets_dev: torch.Tensor, count: int, plan: SegmentPlan,
                           ignore_index: int = -1, need_grad: bool = True):
    """Returns (loss device scalar f64, grad_hidden f32 [n, h] or None)."""
    n, h = hidden.shape
    V = lm_head_t.shape[0]
    dev = hidden.device
    if count == 0:
        raise ContractError("segmented loss: no valid targets")
    grad_hidden = torch.empty(n, h, dtype=F32, device=dev) if need_grad else None
    row_loss = torch.empty(n, dtype=F32, device=dev)
    inv_count = 1.0 / count
    for a, b in plan.segments:
        logits = ops.gemm_f32(hidden[a:b], lm_head_t)
        dlog = torch.empty(b - a, V, dtype=BF16, device=dev)
        ops.ce_rows(logits, targets_dev[a:b], V=V, ignore=ignore_index, inv_count=inv_count,
                    dlogits=dlog, row_loss=row_loss[a:b])
        del logits
        if need_grad:
            ops.gemm_f32(dlog, lm_head, out=grad_hidden[a:b])
        del dlog
    loss_sum = torch.empty(1, dtype=torch.float64, device=dev)
    ops.sum_f64(row_loss, loss_sum)
    return loss_sum / count, grad_hidden


class _SegmentedLoss(torch.autograd.Function):
    """custom_op(loss, "segmented_cross_entropy", (hidden, lm_head), saved, bw)
    of kernels.py:281-288: the gradients are computed in the forward pass and
    the backward only scales them by g."""

    @staticmethod
    def forward(ctx, hidden, lm_head, targets_np, plan, ignore_index):
        n, h = hidden.shape
        V = lm_head.shape[1]
        dev = hidden.device
        count = check_targets(targets_np, V, ignore_index)
        if count == 0:
            raise ContractError("segmented loss: no valid targets")
        w = lm_head.detach()
        w_b = w.to(BF16).contiguous()                 # [h, V]: B operand of dlogits·Wᵀ
        w_t = w.t().contiguous().to(BF16)              # [V, h]: B operand of hidden·W
        hid = hidden.detach().to(BF16).contiguous()
        tg = torch.as_tensor(targets_np.astype(np.int32)).to(dev)
        need_w = lm_head.requires_grad
        loss, grad_hidden, grad_w = _segmented_loss(hid, w_t, w_b, tg, count, plan, ignore_index,
                                                    need_w=need_w)
        ctx.save_for_backward(grad_hidden, grad_w if need_w else None)
        ctx.need_w = need_w
        return loss.to(F32).reshape(())

    @staticmethod
    def backward(ctx, g):
        grad_hidden, grad_w = ctx.saved_tensors
        gw = g * grad_w if ctx.need_w else None
        return g * grad_hidden, gw, None, None, None


def _segmented_loss(hidden, lm_head_t, lm_head, targets_dev, count, plan, ignore_index, *,
                    need_w: bool):
    """segmented_loss_forward plus (optionally) the lm_head gradient
    Σ_seg hsegᵀ·dlogits / count (kernels.py:270-275)."""
    if not need_w:
        loss, gh = segmented_loss_forward(hidden, lm_head_t, lm_head, targets_dev, count, plan,
                                          ignore_index)
        return loss, gh, None
    n, h = hidden.shape
    V = lm_head_t.shape[0]
    dev = hidden.device
    grad_hidden = torch.empty(n, h, dtype=F32, device=dev)
    grad_w = torch.zeros(h, V, dtype=F32, device=dev)
    row_loss = torch.empty(n, dtype=F32, device=dev)
    for a, b in plan.segments:
        logits = ops.gemm_f32(hidden[a:b], lm_head_t)
        dlog = torch.empty(b - a, V, dtype=BF16, device=dev)
        ops.ce_rows(logits, targets_dev[a:b], V=V, ignore=ignore_index, inv_count=1.0 / count,
                    dlogits=dlog, row_loss=row_loss[a:b])
        del logits
        ops.gemm_f32(dlog, lm_head, out=grad_hidden[a:b])
        # grad_W += hsegᵀ·dlogits: K = segment rows (zero-padded to a multiple of
        # 8 for the 16-byte TMA row pitch), both operands transposed copies
        kp = -(-(b - a) // 8) * 8
        ht = torch.zeros(h, kp, dtype=BF16, device=dev)
        ht[:, : b - a] = hidden[a:b].t()
        dt = torch.zeros(V, kp, dtype=BF16, device=dev)
        dt[:, : b - a] = dlog.t()
        ops.gemm_f32(ht, dt, out=grad_w, accumulate=True)
        del ht, dt
        del dlog
    loss_sum = torch.empty(1, dtype=torch.float64, device=dev)
    ops.sum_f64(row_loss, loss_sum)
    return loss_sum / count, grad_hidden, grad_w


def segmented_loss_and_grad(hidden: torch.Tensor, lm_head, targets, plan: SegmentPlan,
                            ignore_index: int = -1) -> torch.Tensor:
    """kernels.py:229-288 (reference name and signature): mean token cross
    entropy of hidden·lm_head computed one segment at a time on the GPU (the
    logits of one segment are live at a time, tcgen05 GEMMs + the ce_rows
    kernel); grad_hidden (and grad_lm_head when lm_head.requires_grad) are
    formed in the forward pass, so backward is g·grad.  hidden [n, h] and
    lm_head [h, V] are CUDA tensors (lm_head may be a host array: frozen)."""
    targets = np.asarray(targets.cpu() if isinstance(targets, torch.Tensor) else targets)
    if not isinstance(hidden, torch.Tensor) or not hidden.is_cuda:
        raise ContractError("segmented_loss_and_grad: hidden must be a CUDA tensor")
    n = hidden.shape[0]
    if targets.shape != (n,):
        raise ContractError(f"targets shape {targets.shape} does not match {n} tokens")
    if plan.n_tokens != n:
        raise ContractError(f"segment plan covers {plan.n_tokens} tokens, input has {n}")
    if not isinstance(lm_head, torch.Tensor):
        lm_head = torch.as_tensor(np.asarray(lm_head, dtype=np.float32)).to(hidden.device)
    if lm_head.shape[0] != hidden.shape[1]:
        raise ContractError(f"lm_head {tuple(lm_head.shape)} does not match hidden "
                            f"{tuple(hidden.shape)}")
    return _SegmentedLoss.apply(hidden, lm_head, targets.astype(np.int64), plan, ignore_index)


def check_targets(targets: np.ndarray, vocab: int, ignore_index: int = -1) -> int:
    """IndexError for out-of-range targets (tensor.py:452-457); returns the
    number of valid targets."""
    valid = targets != ignore_index
    chk = targets[valid]
    if chk.size and (chk.min() < 0 or chk.max() >= vocab):
        raise IndexError(f"target index out of range [0, {vocab}): min={chk.min()}, "
                         f"max={chk.max()}")
    return int(valid.sum())


# ---------------------------------------------------------------------------
# reference-named entry points (value semantics: inputs are not modified)


class _SparseBlock(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, lora_flat, plan, layer, kind):
        out = x.detach().clone()
        if kind == "attention":
            saved = attention_forward(out, plan, layer)
        else:
            saved = mlp_forward(out, plan, layer)
        ctx.saved_state = saved
        ctx.plan, ctx.layer, ctx.kind = plan, layer, kind
        ctx.lora_shape = lora_flat.shape
        return out

    @staticmethod
    def backward(ctx, g):
        dx = g.detach().to(F32).clone().contiguous()
        dlora = torch.zeros(ctx.lora_shape, dtype=F32, device=dx.device)
        if ctx.saved_state is not None:
            if ctx.kind == "attention":
                ev = attention_backward(dx, ctx.saved_state, ctx.layer,
                                        ctx.layer.grad_views(dlora))
                if ev is not None:  # side-stream LoRA gradients must land first
                    torch.cuda.current_stream(dx.device).wait_event(ev)
            else:
                mlp_backward(dx, ctx.saved_state, ctx.layer)
        ctx.saved_state = None
        return dx, dlora, None, None, None


def _check_plan(x, plan):
    if plan.n_tokens != x.shape[0]:
        raise ContractError(f"plan covers {plan.n_tokens} tokens, input has {x.shape[0]}")


# ---------------------------------------------------------------------------
# the reference's duck-typed `layer` (model.py:83-117, kernels.py:295-313)

_SHADOWS: dict = {}


def _host(t):
    """Array behind a reference Tensor (`.data`), a torch tensor or an ndarray."""
    if isinstance(t, torch.Tensor):
        return t.detach()
    d = getattr(t, "data", t)
    return d.detach() if isinstance(d, torch.Tensor) else np.asarray(d)


def as_layer_state(layer, *, max_seq_len: int = 65536, device=None):
    """A LayerState for `layer`.  Accepts this package's LayerState as is, or
    any object with the reference's duck-typed fields (`wq wk wv wo
    attn_norm_w mlp_norm_w w_gate w_up w_down lora_q lora_v n_heads rope
    rope_base mlp_variant`, arrays or reference Tensors, [in, out] layout).
    The frozen weights are converted once (cached per layer object); the
    adapters are re-read on every call, since the caller's optimizer updates
    them.  LoRA gradients of the GPU blocks land in the shadow's flat
    `lora_param.grad` (reference names via `shadow_adapter_grads`)."""
    if hasattr(layer, "w_qkv_t"):
        return layer
    import weakref

    from .model import DecoderModel, ModelConfig

    ent = _SHADOWS.get(id(layer))
    st = ent[1] if ent is not None and ent[0]() is layer else None
    if st is None:
        wq, wk = _host(layer.wq), _host(layer.wk)
        h, kv = wq.shape[0], wk.shape[1]
        d = h // layer.n_heads
        lq = getattr(layer, "lora_q", None)
        r = int(_host(lq.a).shape[1]) if lq is not None else 0
        cfg = ModelConfig(n_layers=1, hidden_dim=h, n_heads=layer.n_heads, vocab_size=32,
                          max_seq_len=max_seq_len, mlp_variant=layer.mlp_variant,
                          mlp_dim=_host(layer.w_up).shape[1], lora_rank=r,
                          lora_alpha=(lq.scaling * r) if r else 16.0,
                          positions="rope" if layer.rope else "learned",
                          rope_base=float(layer.rope_base),
                          n_kv_heads=0 if kv == h else kv // d)
        arrays = {"embed": np.zeros((32, h), np.float32), "final_norm": np.ones(h, np.float32),
                  "lm_head": np.zeros((h, 32), np.float32)}
        names = {"wq": "wq", "wk": "wk", "wv": "wv", "wo": "wo", "attn_norm": "attn_norm_w",
                 "mlp_norm": "mlp_norm_w", "w_up": "w_up", "w_down": "w_down"}
        if layer.mlp_variant == "silu":
            names["w_gate"] = "w_gate"
        for ours, theirs in names.items():
            arrays[f"layer0.{ours}"] = _host(getattr(layer, theirs))
        if r:
            for tag in ("lora_q", "lora_v"):
                ad = getattr(layer, tag)
                arrays[f"layer0.{tag}.a"] = _host(ad.a)
                arrays[f"layer0.{tag}.b"] = _host(ad.b)
        shadow = DecoderModel(cfg, 0, arrays=arrays, device=device)
        st = shadow.layers[0]
        st.shadow_model = shadow
        _SHADOWS[id(layer)] = (weakref.ref(layer), st)
    if st.lora_rank:
        with torch.no_grad():
            for tag, ad in (("lora_q", st.lora_q), ("lora_v", st.lora_v)):
                src = getattr(layer, tag)
                ad.a.copy_(torch.as_tensor(_host(src.a)).to(ad.a.device, torch.float32))
                ad.b.copy_(torch.as_tensor(_host(src.b)).to(ad.b.device, torch.float32))
    return st


def shadow_adapter_grads(layer) -> dict:
    """LoRA gradients accumulated for a duck-typed layer ({"lora_q.a": ...})."""
    ent = _SHADOWS.get(id(layer))
    if ent is None or ent[0]() is not layer:
        return {}
    return {k.split(".", 1)[1]: v for k, v in ent[1].shadow_model.adapter_grads().items()}


def sparse_attention_fused(x: torch.Tensor, plan: GatherPlan, layer,
                           fuse_projections: bool = True) -> torch.Tensor:
    """kernels.py:153-177: k == 0 returns x itself; otherwise a new residual
    tensor with the attention output added at the retained rows.  `layer` is
    a LayerState or the reference's duck-typed layer (as_layer_state)."""
    _check_plan(x, plan)
    if plan.k == 0:
        return x
    layer = as_layer_state(layer, device=x.device)
    return _SparseBlock.apply(x, layer.lora_param, plan, layer, "attention")


def sparse_mlp_fused(x: torch.Tensor, plan: GatherPlan, layer,
                     fuse_projections: bool = True) -> torch.Tensor:
    """kernels.py:201-222"""
    _check_plan(x, plan)
    if plan.k == 0:
        return x
    layer = as_layer_state(layer, device=x.device)
    return _SparseBlock.apply(x, layer.lora_param, plan, layer, "mlp")


# ---------------------------------------------------------------------------
# naive variants (kernels.py:131-150, 180-198): the same block math on a
# MATERIALISED compact copy -- gather the retained rows into their own
# buffer, run the block there (RoPE still at the original positions), write
# its output into a zero [k, h] buffer, pad it to [s, h] and add.  Three
# transient buffers, no index-remapped epilogue: an independent data path
# that the fused kernels are checked against.


class _NaiveBlock(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, lora_flat, plan, layer, kind):
        idx = plan.indices.long()
        k = plan.k
        gathered = x.detach().index_select(0, idx).contiguous()   # transient 1
        small = torch.zeros_like(gathered)                        # transient 2
        compact = GatherPlan.full(k, x.device)
        if kind == "attention":
            saved = attention_forward(gathered, compact, layer, out=small, pos=plan.indices)
        else:
            saved = mlp_forward(gathered, compact, layer, out=small)
        padded = torch.zeros_like(x).index_copy_(0, idx, small)  # transient 3
        out = x.detach() + padded
        ctx.saved_state = saved
        ctx.plan, ctx.layer, ctx.kind = plan, layer, kind
        ctx.lora_shape = lora_flat.shape
        return out

    @staticmethod
    def backward(ctx, g):
        g = g.detach().to(F32)
        idx = ctx.plan.indices.long()
        dxc = g.index_select(0, idx).contiguous()  # d/dx of the compact copy, plus J^T g
        dlora = torch.zeros(ctx.lora_shape, dtype=F32, device=g.device)
        if ctx.kind == "attention":
            ev = attention_backward(dxc, ctx.saved_state, ctx.layer, ctx.layer.grad_views(dlora))
            if ev is not None:
                torch.cuda.current_stream(g.device).wait_event(ev)
        else:
            mlp_backward(dxc, ctx.saved_state, ctx.layer)
        ctx.saved_state = None
        dx = g.clone().index_copy_(0, idx, dxc)
        return dx, dlora, None, None, None


def sparse_attention_naive(x: torch.Tensor, plan: GatherPlan, layer) -> torch.Tensor:
    """kernels.py:131-150"""
    _check_plan(x, plan)
    if plan.k == 0:
        return x
    layer = as_layer_state(layer, device=x.device)
    return _NaiveBlock.apply(x, layer.lora_param, plan, layer, "attention")


def sparse_mlp_naive(x: torch.Tensor, plan: GatherPlan, layer) -> torch.Tensor:
    """kernels.py:180-198"""
    _check_plan(x, plan)
    if plan.k == 0:
        return x
    layer = as_layer_state(layer, device=x.device)
    return _NaiveBlock.apply(x, layer.lora_param, plan, layer, "mlp")
