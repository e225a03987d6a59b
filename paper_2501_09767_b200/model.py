"""Decoder model with LoRA adapters and the per-layer token-elimination hook.

Mirrors ``sparsetune.model`` (model.py:23-590): ModelConfig, LoraAdapter,
LayerState, DecoderModel.forward_step and the pattern sources.  Frozen
weights live on the GPU in bf16 in the two K-major layouts the tcgen05 GEMMs
need (forward: [out, in]; backward dX: [in, out]); the residual stream is
fp32; all LoRA parameters share one flat fp32 buffer (one Adam launch, one
NCCL all-reduce bucket).

`forward_step` runs the whole step through liblemo kernels and returns a
loss whose `.backward()` runs the sparse backward sweep (saved activations
are compact retained-row buffers only) and fills `model.lora_param.grad`.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, kernels, ledger, ops, predictor as predictor_mod, sparsity
from .errors import ContractError, DimensionError

PAD_TOKEN = 0
IGNORE_INDEX = -1
SCORING_PRECISIONS = ("bf16", "fp32", "refined")
BF16, F32 = torch.bfloat16, torch.float32


@dataclass
class ModelConfig:
    """Geometry, model.py:23-64 (same fields and validation)."""

    n_layers: int = 4
    hidden_dim: int = 64
    n_heads: int = 4
    vocab_size: int = 256
    max_seq_len: int = 2048
    mlp_variant: str = "silu"  # "relu" | "silu"
    mlp_dim: int = 256
    lora_rank: int = 8
    lora_alpha: float = 16.0
    block_size: int = 16
    positions: str = "rope"  # "rope" | "learned"
    rope_base: float = 10000.0
    dtype: str = "float32"
    # grouped-query attention (an extension beyond the reference; 0 = n_heads):
    # k / v carry n_kv_heads heads, query head i reads key head i // (H / n_kv)
    n_kv_heads: int = 0

    def __post_init__(self):
        if self.n_kv_heads and (self.n_kv_heads < 0 or self.n_heads % self.n_kv_heads):
            raise DimensionError(f"n_heads {self.n_heads} not a multiple of n_kv_heads "
                                 f"{self.n_kv_heads}")
        if self.hidden_dim % self.n_heads != 0:
            raise DimensionError(f"hidden_dim {self.hidden_dim} not divisible by {self.n_heads} heads")
        if self.positions == "rope" and self.head_dim % 2 != 0:
            raise DimensionError("rotary positions need an even head dim")
        if self.max_seq_len % self.block_size != 0:
            raise ContractError(f"max_seq_len {self.max_seq_len} must be a multiple of block "
                                f"size {self.block_size}")
        if self.mlp_variant not in ("relu", "silu"):
            raise ContractError(f"unknown mlp variant {self.mlp_variant!r}")
        if self.positions not in ("rope", "learned"):
            raise ContractError(f"unknown position mode {self.positions!r}")
        if self.dtype not in ("float32", "float64", "bfloat16"):
            raise ContractError(f"unsupported dtype {self.dtype!r}")

    @property
    def kv_heads(self) -> int:
        return self.n_kv_heads or self.n_heads

    @property
    def kv_dim(self) -> int:
        return self.kv_heads * self.head_dim

    @property
    def head_dim(self) -> int:
        return self.hidden_dim // self.n_heads

    @property
    def mlp_pad(self) -> int:
        return -(-self.mlp_dim // 128) * 128

    def check_gpu_geometry(self) -> None:
        """Tile constraints of the B200 kernels (reported, never silently padded)."""
        if self.head_dim not in (64, 128):
            raise ContractError(f"GPU kernels support head_dim 64 or 128, got {self.head_dim}")
        if self.hidden_dim % 128:
            raise ContractError("GPU kernels need hidden_dim % 128 == 0")
        if self.vocab_size % 32:
            raise ContractError("GPU kernels need vocab_size % 32 == 0")
        if self.lora_rank > 16:
            raise ContractError("GPU kernels support LoRA rank <= 16")
        if self.kv_dim % 128:
            raise ContractError("GPU kernels need n_kv_heads·head_dim % 128 == 0")


def llama2_7b(**kw) -> ModelConfig:
    """Llama2-7B geometry (BASELINE configs[1], north star at 16K)."""
    base = dict(n_layers=32, hidden_dim=4096, n_heads=32, vocab_size=32000, max_seq_len=16384,
                mlp_dim=11008, lora_rank=8, lora_alpha=16.0, block_size=16)
    base.update(kw)
    return ModelConfig(**base)


def llama3_8b(**kw) -> ModelConfig:
    """Llama3-8B geometry (BASELINE configs[2]): 32 query / 8 key-value heads
    (grouped-query attention, pinned through the repeated-head reference
    model), m=14336, V=128256, RoPE base 500000."""
    base = dict(n_layers=32, hidden_dim=4096, n_heads=32, n_kv_heads=8, vocab_size=128256,
                max_seq_len=16384, mlp_dim=14336, rope_base=500000.0, lora_rank=8,
                lora_alpha=16.0, block_size=16)
    base.update(kw)
    return ModelConfig(**base)


def mistral_7b(**kw) -> ModelConfig:
    """Mistral-7B geometry (BASELINE configs[3]): 32 / 8 heads, m=14336,
    V=32000.  Full causal attention: sliding-window attention is not part of
    the reference and is not modelled."""
    base = dict(n_layers=32, hidden_dim=4096, n_heads=32, n_kv_heads=8, vocab_size=32000,
                max_seq_len=32768, mlp_dim=14336, lora_rank=8, lora_alpha=16.0, block_size=16)
    base.update(kw)
    return ModelConfig(**base)


def opt_6_7b(**kw) -> ModelConfig:
    """OPT-6.7B geometry inside the reference's model family (BASELINE
    configs[4]): h=4096, 32 heads, ReLU MLP m=16384, learned positions,
    V=50272.  The reference has RMSNorm and no biases, so neither has this
    model (OPT's LayerNorm/bias are outside the reference)."""
    base = dict(n_layers=32, hidden_dim=4096, n_heads=32, vocab_size=50272, max_seq_len=65536,
                mlp_dim=16384, mlp_variant="relu", positions="learned", lora_rank=8,
                lora_alpha=16.0, block_size=16)
    base.update(kw)
    return ModelConfig(**base)


def tiny_t(**kw) -> ModelConfig:
    """Config T of SURVEY §8 (BASELINE configs[0])."""
    base = dict(n_layers=2, hidden_dim=256, n_heads=4, vocab_size=256, max_seq_len=2048,
                mlp_dim=688, lora_rank=8, lora_alpha=16.0, block_size=16)
    base.update(kw)
    return ModelConfig(**base)


# ---------------------------------------------------------------------------
# weights


def _interleave_gate_up(w_gate, w_up, m_pad):
    """[h, m] gate/up → [h, 2·m_pad] with 128-column chunks interleaved
    (gate chunk i, up chunk i, …); padded columns are zero (exact no-ops)."""
    h, m = w_up.shape
    out = torch.zeros(h, 2 * m_pad, dtype=w_up.dtype, device=w_up.device)
    g = torch.zeros(h, m_pad, dtype=w_up.dtype, device=w_up.device)
    u = torch.zeros_like(g)
    g[:, :m] = w_gate
    u[:, :m] = w_up
    out.view(h, m_pad // 128, 2, 128)[:, :, 0, :] = g.view(h, m_pad // 128, 128)
    out.view(h, m_pad // 128, 2, 128)[:, :, 1, :] = u.view(h, m_pad // 128, 128)
    return out


def rope_table(max_pos: int, head_dim: int, base: float, device) -> torch.Tensor:
    """(cos, sin) per (position, frequency) computed in float64 then cast —
    the table of tensor.py:604-607."""
    half = head_dim // 2
    inv_freq = base ** (-np.arange(half, dtype=np.float64) / half)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv_freq[None, :]
    tab = np.stack([np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)], axis=-1)
    return torch.as_tensor(np.ascontiguousarray(tab)).to(device)


class LoraAdapter:
    """Views of one adapter inside the model's flat LoRA buffer (model.py:67-80).
    a: [h, r] (strided view), b: [r, h]."""

    def __init__(self, a: torch.Tensor, b: torch.Tensor, scaling: float, grad_a, grad_b):
        self.a = a
        self.b = b
        self.rank = a.shape[1]
        self.scaling = scaling
        self._ga, self._gb = grad_a, grad_b

    @property
    def a_grad(self):
        return self._ga()

    @property
    def b_grad(self):
        return self._gb()

    def parameters(self):
        return [self.a, self.b]


class LayerState:
    """Frozen bf16 weights in GEMM layouts + LoRA views for one layer (model.py:83-130)."""

    def __init__(self, model: "DecoderModel", layer_id: int, arrays: dict):
        cfg = model.config
        dev = model.device
        h, m = cfg.hidden_dim, cfg.mlp_dim
        self.layer_id = layer_id
        self.n_heads = cfg.n_heads
        self.head_dim = cfg.head_dim
        self.kv = kv = cfg.kv_dim  # k / v width (= h unless grouped-query)
        self.rope = cfg.positions == "rope"
        self.rope_base = cfg.rope_base
        self.mlp_variant = cfg.mlp_variant
        self.relu = cfg.mlp_variant == "relu"
        self.m = m
        self.m_pad = cfg.mlp_pad
        self.rope_tab = model.rope_tab
        self.scoring_precision = model.scoring_precision
        self.refine_margin = model.refine_margin

        def g(name):
            a = arrays[name]
            t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
            return t.to(device=dev, dtype=F32)

        wq, wk, wv, wo = g("wq"), g("wk"), g("wv"), g("wo")
        w_qkv = torch.cat([wq, wk, wv], dim=1)  # [h, h+2kv]   (x·W layout)
        nq = h + 2 * kv
        kext = ops.LORA_K_EXT if cfg.lora_rank else 0
        # backward dX operand [h, h+2kv (+64: A_q|A_v, the LoRA term of dxn)]
        self.w_qkv = torch.zeros(h, nq + kext, dtype=BF16, device=dev)
        self.w_qkv[:, :nq] = w_qkv.to(BF16)
        # forward operand [h+2kv, h (+64 LoRA K-extension columns, see lemo_gemm_qkv)]
        self.w_qkv_t = torch.zeros(nq, h + kext, dtype=BF16, device=dev)
        self.w_qkv_t[:, :h] = w_qkv.t().to(BF16)
        self.inv_freq = model.inv_freq
        self.w_o = wo.to(BF16).contiguous()
        self.w_o_t = wo.t().contiguous().to(BF16)
        w_up = g("w_up")
        if self.relu:
            gu = torch.zeros(h, self.m_pad, device=dev)
            gu[:, :m] = w_up
        else:
            gu = _interleave_gate_up(g("w_gate"), w_up, self.m_pad)
        self.w_gu = gu.to(BF16).contiguous()
        self.w_gu_t = gu.t().contiguous().to(BF16)
        # fp32-faithful scoring (scoring_precision="fp32"): the bf16 residual
        # lo = bf16(w - hi) of the scoring weights, so hi + lo carries the fp32
        # weights into the bf16x3 GEMMs (gate/up, q/k)
        self.w_gu_t_lo = self.w_qk_t_lo = None
        self._gu_x3 = self._qk_x3 = None  # bf16xN operands, built on first fp32-precision use
        # parity_terms: 3 = hi·hi + hi·lo + lo·hi; 2 when the scoring weights are
        # bf16-representable (lo == 0 exactly, e.g. bf16 checkpoints): x_hi·W + x_lo·W
        self.parity_terms = 3
        if model.parity_weights:
            gut = gu.t().contiguous()
            lo_gu = (gut - self.w_gu_t.float()).to(BF16)
            del gut
            qk_t = w_qkv[:, :h + kv].t().contiguous()
            lo_qk = (qk_t - self.w_qkv_t[:h + kv, :h].float()).to(BF16)
            del qk_t
            if int(torch.count_nonzero(lo_gu)) == 0 and int(torch.count_nonzero(lo_qk)) == 0:
                self.parity_terms = 2
            else:
                self.w_gu_t_lo, self.w_qk_t_lo = lo_gu, lo_qk
            del lo_gu, lo_qk
        wd = torch.zeros(self.m_pad, h, device=dev)
        wd[:m] = g("w_down")
        self.w_down = wd.to(BF16).contiguous()
        self.w_down_t = wd.t().contiguous().to(BF16)
        del w_qkv, gu, wd
        self.attn_norm_w = g("attn_norm").contiguous()
        self.mlp_norm_w = g("mlp_norm").contiguous()
        # LoRA: views into the model's flat buffer
        r = cfg.lora_rank
        self.lora_rank = r
        self.lora_scaling = cfg.lora_alpha / r if r else 0.0
        self.lora_param = model.lora_param
        self.predictor_q: predictor_mod.Predictor | None = None
        self.predictor_k: predictor_mod.Predictor | None = None
        if r:
            self._off = model._lora_offset(layer_id)
            A, Bq, Bv = self._views(model.lora_param.data)
            self.lora_A, self.lora_Bq, self.lora_Bv = A, Bq, Bv
            self.lora_q = LoraAdapter(A[:, :r], Bq, self.lora_scaling,
                                      lambda: self._grad("Aq"), lambda: self._grad("Bq"))
            self.lora_v = LoraAdapter(A[:, r:], Bv, self.lora_scaling,
                                      lambda: self._grad("Av"), lambda: self._grad("Bv"))
        else:
            self.lora_q = self.lora_v = None

    def _views(self, flat):
        h, r, kv = self.head_dim * self.n_heads, self.lora_rank, self.kv
        o = self._off
        A = flat[o:o + 2 * h * r].view(h, 2 * r)
        Bq = flat[o + 2 * h * r:o + 3 * h * r].view(r, h)
        Bv = flat[o + 3 * h * r:o + 3 * h * r + kv * r].view(r, kv)
        return A, Bq, Bv

    def _require_parity(self):
        if self.w_gu_t_lo is None and self.parity_terms == 3:
            raise ContractError("fp32 scoring needs a model built with parity_weights=True")

    def gateup_x3(self) -> torch.Tensor:
        """B operand of the fp32-faithful gate/up GEMM, built on first use and
        kept (frozen weights): [hi | lo | hi] (K = 3h) or, for bf16-exact
        weights, [W | W] (K = 2h)."""
        self._require_parity()
        if self._gu_x3 is None:
            parts = ([self.w_gu_t, self.w_gu_t] if self.parity_terms == 2 else
                     [self.w_gu_t, self.w_gu_t_lo, self.w_gu_t])
            self._gu_x3 = torch.cat(parts, dim=1)
        return self._gu_x3

    def qk_x3(self) -> torch.Tensor:
        """B operand of the fp32-faithful q/k projections (kept, as above)."""
        self._require_parity()
        if self._qk_x3 is None:
            h = self.w_qkv.shape[0]
            hi = self.w_qkv_t[:h + self.kv, :h]
            parts = [hi, hi] if self.parity_terms == 2 else [hi, self.w_qk_t_lo, hi]
            self._qk_x3 = torch.cat(parts, dim=1)
        return self._qk_x3

    def split_input(self, xnf: torch.Tensor) -> torch.Tensor:
        """The A operand matching gateup_x3 / qk_x3: [hi | hi | lo] or [hi | lo]."""
        return ops.split_bf16x3(xnf, 0) if self.parity_terms == 3 else ops.split_bf16x2(xnf)

    def lora_A_packed(self) -> torch.Tensor:
        """[32, h] bf16 copy of [A_q | A_v] for the t = xn·A GEMM (re-packed each
        call: the adapters change every optimizer step)."""
        return ops.lora_pack(self.lora_A, self.lora_rank)

    def qkv_input(self, xn_ext: torch.Tensor) -> torch.Tensor:
        """Complete the q/k/v GEMM operands for LoRA (kernels.py:95-100): t = xn·A
        (fp32, saved for backward), s·t into xn_ext's 64 extension columns and
        the current B_q/B_v into the weight's extension columns.  Returns t."""
        h, r = self.w_qkv.shape[0], self.lora_rank
        t = ops.lora_down(xn_ext[:, :h], self.lora_A_packed())
        ops.lora_qkv_prep(t, r, self.lora_scaling, xn_ext, h)
        ops.lora_pack_b(self.lora_Bq, self.lora_Bv, r, self.w_qkv_t, h)
        return t

    def qkv_grad_input(self, dqkv_ext: torch.Tensor) -> torch.Tensor:
        """Backward counterpart: u = [dq·Bqᵀ | dv·Bvᵀ] (fp32 [k, 32], one GEMM),
        s·u into dqkv_ext's extension columns and A_q|A_v into the dX weight's,
        so dxn = dqkv·W_qkvᵀ + s·u·Aᵀ (kernels.py:95-100 backward) is one GEMM."""
        h, r = self.w_qkv.shape[0], self.lora_rank
        nq = h + 2 * self.kv
        u = ops.gemm_f32(dqkv_ext[:, :nq], ops.lora_pack_bt(self.lora_Bq, self.lora_Bv, r, h))
        ops.lora_qkv_prep(u, r, self.lora_scaling, dqkv_ext, nq)
        ops.lora_pack_a_ext(self.lora_A, r, self.w_qkv, nq)
        return u

    def grad_views(self, flat_grad):
        return self._views(flat_grad) if self.lora_rank else None

    def _grad(self, which):
        gr = self.lora_param.grad
        if gr is None:
            return None
        A, Bq, Bv = self._views(gr)
        r = self.lora_rank
        return {"Aq": A[:, :r], "Av": A[:, r:], "Bq": Bq, "Bv": Bv}[which]


def reference_init_arrays(cfg: ModelConfig, seed: int) -> dict:
    """Host arrays with the reference's exact draw order (model.py:86-153)."""
    rng = np.random.default_rng(seed)
    h, m = cfg.hidden_dim, cfg.mlp_dim
    std = 1.0 / np.sqrt(h)
    out = {"embed": (rng.standard_normal((cfg.vocab_size, h)) * std).astype(np.float32)}
    if cfg.positions == "learned":
        out["pos_embed"] = (rng.standard_normal((cfg.max_seq_len, h)) * std).astype(np.float32)
    for i in range(cfg.n_layers):
        p = f"layer{i}"

        def w(rows, cols):
            return (rng.standard_normal((rows, cols)) * std).astype(np.float32)
        kv = cfg.kv_dim
        out[f"{p}.wq"], out[f"{p}.wk"], out[f"{p}.wv"], out[f"{p}.wo"] = (
            w(h, h), w(h, kv), w(h, kv), w(h, h))
        out[f"{p}.attn_norm"] = np.ones(h, np.float32)
        out[f"{p}.mlp_norm"] = np.ones(h, np.float32)
        out[f"{p}.w_up"] = w(h, m)
        out[f"{p}.w_down"] = w(m, h)
        if cfg.mlp_variant == "silu":
            out[f"{p}.w_gate"] = w(h, m)
        if cfg.lora_rank > 0:
            for tag, width in (("lora_q", h), ("lora_v", cfg.kv_dim)):
                out[f"{p}.{tag}.a"] = (rng.standard_normal((h, cfg.lora_rank)) /
                                       np.sqrt(h)).astype(np.float32)
                out[f"{p}.{tag}.b"] = np.zeros((cfg.lora_rank, width), np.float32)
    out["final_norm"] = np.ones(h, np.float32)
    out["lm_head"] = (rng.standard_normal((h, cfg.vocab_size)) * std).astype(np.float32)
    return out


class _TorchInit:
    """Lazy on-device random init for large models (same distributions as the
    reference: N(0, 1/h) frozen weights, norms 1, LoRA A ~ N(0, 1/h), B = 0).
    Frozen weights are drawn in bf16 -- the precision they are stored and
    multiplied in -- so the fp32 model they define (what the reference would
    compute with) is exactly the bf16 one; LoRA A stays fp32."""

    def __init__(self, cfg: ModelConfig, seed: int, device):
        self.cfg, self.dev = cfg, device
        self.gen = torch.Generator(device=device)
        self.gen.manual_seed(seed)

    def normal(self, rows, cols, std, bf16: bool = True):
        w = torch.randn(rows, cols, generator=self.gen, device=self.dev) * std
        return w.to(BF16).float() if bf16 else w

    def layer(self, i):
        cfg = self.cfg
        h, m = cfg.hidden_dim, cfg.mlp_dim
        std = 1.0 / math.sqrt(h)
        kv = cfg.kv_dim
        d = {n: self.normal(h, h if n in ("wq", "wo") else kv, std)
             for n in ("wq", "wk", "wv", "wo")}
        d["w_up"] = self.normal(h, m, std)
        d["w_down"] = self.normal(m, h, std)
        if cfg.mlp_variant == "silu":
            d["w_gate"] = self.normal(h, m, std)
        d["attn_norm"] = torch.ones(h, device=self.dev)
        d["mlp_norm"] = torch.ones(h, device=self.dev)
        if cfg.lora_rank:
            for tag, width in (("lora_q", h), ("lora_v", kv)):
                d[f"{tag}.a"] = self.normal(h, cfg.lora_rank, std, bf16=False)
                d[f"{tag}.b"] = torch.zeros(cfg.lora_rank, width, device=self.dev)
        return d


class DecoderModel:
    """model.py:133-326 on the GPU.

    init="reference": numpy draws in the reference's order (bit-identical
    weights to sparsetune.DecoderModel(cfg, seed)); init="torch": on-device
    generator with the same distributions (for 7B-scale benches).
    """

    def __init__(self, cfg: ModelConfig, seed: int = 0, *, device=None, init: str = "torch",
                 arrays: dict | None = None, scoring_precision: str = "bf16",
                 parity_weights: bool | None = None, refine_margin: float = 2e-3):
        cfg.check_gpu_geometry()
        if scoring_precision not in SCORING_PRECISIONS:
            raise ContractError(f"unknown scoring precision {scoring_precision!r}")
        # default precision of the scorers the pattern sources call:
        #   "bf16"     production scorers on bf16 tensor-core operands
        #   "fp32"     the fp32-faithful parity scorers (reproduce the reference's masks)
        #   "refined"  bf16 scorers, then every MLP block whose score lies within
        #              refine_margin·|T| of its threshold T re-scored in the parity
        #              precision before selection (refine_mlp_block_scores)
        self.scoring_precision = scoring_precision
        self.refine_margin = float(refine_margin)
        # parity_weights: keep the bf16 residuals of the scoring weights (+~8 %
        # weight memory) so the fp32 precision can be used per call (e.g. by the
        # mask audit) while the sources default to bf16
        self.parity_weights = (scoring_precision != "bf16") if parity_weights is None \
            else bool(parity_weights)
        if scoring_precision != "bf16" and not self.parity_weights:
            raise ContractError(f"scoring_precision={scoring_precision!r} needs parity_weights")
        self.config = cfg
        self.seed = seed
        self.device = torch.device(device) if device is not None else torch.device("cuda")
        dev = self.device
        h, r, L = cfg.hidden_dim, cfg.lora_rank, cfg.n_layers
        self.rope_tab = rope_table(cfg.max_seq_len, cfg.head_dim, cfg.rope_base, dev) \
            if cfg.positions == "rope" else None
        half = cfg.head_dim // 2
        self.inv_freq = torch.as_tensor(
            cfg.rope_base ** (-np.arange(half, dtype=np.float64) / half)).to(dev)
        self.lora_param = torch.zeros(max((3 * h + cfg.kv_dim) * r * L, 1), dtype=F32,
                                      device=dev)
        if arrays is None and init == "reference":
            arrays = reference_init_arrays(cfg, seed)
        if arrays is not None:
            get = lambda n: arrays[n]  # noqa: E731
            layer_arrays = lambda i: {k.split(".", 1)[1]: v for k, v in arrays.items()  # noqa
                                      if k.startswith(f"layer{i}.")}
        else:
            ti = _TorchInit(cfg, seed, dev)
            std = 1.0 / math.sqrt(h)
            glob = {"embed": ti.normal(cfg.vocab_size, h, std)}
            if cfg.positions == "learned":
                glob["pos_embed"] = ti.normal(cfg.max_seq_len, h, std)
            get = glob.__getitem__
            layer_arrays = ti.layer
        f32 = lambda a: (a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))  # noqa
                         ).to(device=dev, dtype=F32).contiguous()
        self.embed = f32(get("embed"))
        self.pos_embed = f32(get("pos_embed")) if cfg.positions == "learned" else None
        self.layers = []
        for i in range(L):
            la = layer_arrays(i)
            layer = LayerState(self, i, la)
            if r:
                for tag, ad in (("lora_q", layer.lora_q), ("lora_v", layer.lora_v)):
                    ad.a.copy_(f32(la[f"{tag}.a"]))
                    ad.b.copy_(f32(la[f"{tag}.b"]))
            self.layers.append(layer)
            del la
        if arrays is not None:
            final, lm = arrays["final_norm"], arrays["lm_head"]
        else:
            final = torch.ones(h, device=dev)
            lm = ti.normal(h, cfg.vocab_size, 1.0 / math.sqrt(h))
        self.final_norm_w = f32(final)
        lm = f32(lm)
        self.lm_head = lm.to(BF16).contiguous()           # [h, V]  (dhidden GEMM)
        self.lm_head_t = lm.t().contiguous().to(BF16)      # [V, h]  (logits GEMM)
        del lm
        self.lora_param.requires_grad_(cfg.lora_rank > 0)
        # layer -> (step epoch, x address, (gu_all, inv_all)): full-sequence
        # gate/up rows the MLP scorer produced for the CURRENT step's residual;
        # mlp_forward compacts them instead of recomputing (see take_mlp_rows)
        self._mlp_scored = {}
        self._epoch = 0
        self.last_stats: dict = {}
        # data parallelism: called with each layer's LoRA-gradient slice as soon
        # as the backward sweep has finished it (parallel.BucketedGradReducer)
        self.grad_reducer = None

    # -- parameters -------------------------------------------------------------

    def _lora_offset(self, layer_id: int) -> int:
        c = self.config
        return (3 * c.hidden_dim + c.kv_dim) * c.lora_rank * layer_id

    def adapter_parameters(self):
        out = []
        for layer in self.layers:
            for ad in (layer.lora_q, layer.lora_v):
                if ad is not None:
                    out.extend(ad.parameters())
        return out

    def adapter_state(self) -> dict:
        """name -> host array of every adapter tensor (reference names)."""
        out = {}
        for layer in self.layers:
            for tag, ad in (("lora_q", layer.lora_q), ("lora_v", layer.lora_v)):
                if ad is not None:
                    out[f"layer{layer.layer_id}.{tag}.a"] = ad.a.cpu().numpy()
                    out[f"layer{layer.layer_id}.{tag}.b"] = ad.b.cpu().numpy()
        return out

    def adapter_grads(self) -> dict:
        out = {}
        for layer in self.layers:
            for tag, ad in (("lora_q", layer.lora_q), ("lora_v", layer.lora_v)):
                if ad is not None and ad.a_grad is not None:
                    out[f"layer{layer.layer_id}.{tag}.a"] = ad.a_grad.cpu().numpy()
                    out[f"layer{layer.layer_id}.{tag}.b"] = ad.b_grad.cpu().numpy()
        return out

    def load_adapter_state(self, state: dict) -> None:
        for layer in self.layers:
            for tag, ad in (("lora_q", layer.lora_q), ("lora_v", layer.lora_v)):
                if ad is None:
                    continue
                for ab, t in (("a", ad.a), ("b", ad.b)):
                    key = f"layer{layer.layer_id}.{tag}.{ab}"
                    if key in state:
                        t.copy_(torch.as_tensor(np.asarray(state[key], np.float32)))

    def attach_predictors(self, pairs: dict) -> None:
        for layer_id, (p_q, p_k) in pairs.items():
            self.layers[layer_id].predictor_q = p_q
            self.layers[layer_id].predictor_k = p_k

    # -- padding ------------------------------------------------------------------

    def pad_tokens(self, tokens, targets):
        """model.py:218-236 (host)."""
        tokens = np.asarray(tokens, dtype=np.int64)
        n = tokens.shape[0]
        if n == 0:
            raise ContractError("empty token sequence")
        if n > self.config.max_seq_len:
            raise ContractError(f"sequence length {n} exceeds max {self.config.max_seq_len}")
        if targets is None:
            targets = np.concatenate([tokens[1:], [IGNORE_INDEX]])
        else:
            targets = np.asarray(targets, dtype=np.int64)
            if targets.shape != tokens.shape:
                raise ContractError("targets must match token count")
        b = self.config.block_size
        n_pad = -(-n // b) * b
        if n_pad > n:
            tokens = np.concatenate([tokens, np.full(n_pad - n, PAD_TOKEN, dtype=np.int64)])
            targets = np.concatenate([targets, np.full(n_pad - n, IGNORE_INDEX, dtype=np.int64)])
        return tokens, targets, n

    # -- forward --------------------------------------------------------------------

    def stage_tokens(self, tokens, targets=None) -> "StagedBatch":
        return StagedBatch(self, tokens, targets)

    def forward_step(self, tokens, targets=None, *, pattern_source=None, segments: int = 1,
                     fused: bool = True, fuse_projections: bool = True):
        """model.py:246-297.  Returns (loss, hidden): loss is a CUDA scalar whose
        backward() runs the sparse backward sweep into lora_param.grad;
        hidden is the final normalised hidden state (bf16)."""
        step = _Step(self, tokens, targets, pattern_source, segments)
        if torch.is_grad_enabled():
            loss = _StepFn.apply(self.lora_param, step)
        else:
            with torch.no_grad():
                loss = step.forward(need_grad=False)
        return loss, step.hidden

    def set_scoring_precision(self, precision: str) -> None:
        """Switch the scorers' default precision (model and every layer)."""
        if precision not in SCORING_PRECISIONS:
            raise ContractError(f"unknown scoring precision {precision!r}")
        if precision != "bf16" and not self.parity_weights:
            raise ContractError(f"scoring_precision={precision!r} needs parity_weights")
        self.scoring_precision = precision
        for layer in self.layers:
            layer.scoring_precision = precision

    def stash_mlp_rows(self, layer_id: int, x: torch.Tensor, rows) -> None:
        self._mlp_scored[layer_id] = (self._epoch, x.data_ptr(), rows)

    def take_mlp_rows(self, layer_id: int, x: torch.Tensor):
        """The scorer's rows for this layer if they were computed from this very
        residual in this step (else None: the sparse MLP recomputes gate/up)."""
        ent = self._mlp_scored.pop(layer_id, None)
        if ent is None or ent[0] != self._epoch or ent[1] != x.data_ptr():
            return None
        return ent[2]

    @staticmethod
    def _plan_from(pattern, n_pad: int, device) -> kernels.GatherPlan:
        if pattern is None:
            return kernels.GatherPlan.full(n_pad, device)
        return kernels.GatherPlan.from_pattern(pattern, n_pad, device)


class StagedBatch:
    """A padded, validated token/target pair resident on the device
    (DecoderModel.stage_tokens); forward_step accepts it in place of host
    arrays so a caller can keep inputs in HBM across steps."""

    def __init__(self, model: "DecoderModel", tokens, targets=None):
        ids, tgts, n_valid = model.pad_tokens(tokens, targets)
        cfg = model.config
        if ids.min() < 0 or ids.max() >= cfg.vocab_size:
            raise IndexError(f"token id out of range [0, {cfg.vocab_size}): min={ids.min()}, "
                             f"max={ids.max()}")
        self.count = kernels.check_targets(tgts, cfg.vocab_size, IGNORE_INDEX)
        if self.count == 0:
            raise ContractError("segmented loss: no valid targets")
        self.n_valid = n_valid
        self.n_pad = len(ids)
        host = torch.empty(2, self.n_pad, dtype=torch.int32, pin_memory=True)
        host[0].copy_(torch.from_numpy(ids.astype(np.int32)))
        host[1].copy_(torch.from_numpy(tgts.astype(np.int32)))
        both = host.to(model.device, non_blocking=True)
        self.ids, self.tgts = both[0], both[1]
        self.h2d_bytes = host.numel() * 4


class _Step:
    """Saved state of one training step (the reference's tape, compacted)."""

    def __init__(self, model: DecoderModel, tokens, targets, source, segments):
        self.model = model
        self.source = source
        batch = tokens if isinstance(tokens, StagedBatch) else StagedBatch(model, tokens, targets)
        self.count = batch.count
        self.n_valid = batch.n_valid
        self.n_pad = batch.n_pad
        self.ids, self.tgts = batch.ids, batch.tgts
        self.h2d_bytes = 0 if batch is tokens else batch.h2d_bytes
        self.segments = max(1, segments)
        self.hidden = None

    def forward(self, need_grad: bool = True):
        m = self.model
        m._epoch += 1
        m._mlp_scored.clear()
        try:
            return self._forward(need_grad)
        finally:
            m._mlp_scored.clear()

    def _forward(self, need_grad: bool):
        m = self.model
        dev = m.device
        mem0 = _lib.memory_allocated(dev)
        x = ops.embed(self.ids, m.embed,
                      m.pos_embed[: self.n_pad].contiguous() if m.pos_embed is not None else None)
        saved = []
        src = self.source
        led = ledger.get()
        for layer in m.layers:
            pat = src.pattern(layer.layer_id, sparsity.ATTENTION, x, self.n_valid) \
                if src is not None else None
            plan = DecoderModel._plan_from(pat, self.n_pad, dev)
            sa = kernels.attention_forward(x, plan, layer, save=need_grad)
            ledger.retain_saved(led, f"layer{layer.layer_id}.attn", sa)
            pat = src.pattern(layer.layer_id, sparsity.MLP, x, self.n_valid) \
                if src is not None else None
            plan = DecoderModel._plan_from(pat, self.n_pad, dev)
            scored = m.take_mlp_rows(layer.layer_id, x)
            sm = kernels.mlp_forward(x, plan, layer, scored=scored, save=need_grad)
            ledger.retain_saved(led, f"layer{layer.layer_id}.mlp", sm)
            del scored
            saved.append((sa, sm))
        inv_f = torch.empty(self.n_pad, dtype=F32, device=dev)
        hidden = ops.rmsnorm_gather(x, m.final_norm_w, None, inv=inv_f)
        plan = kernels.SegmentPlan.even(self.n_pad, self.segments)
        loss, grad_hidden = kernels.segmented_loss_forward(
            hidden, m.lm_head_t, m.lm_head, self.tgts, self.count, plan, IGNORE_INDEX,
            need_grad=need_grad)
        self.hidden = hidden
        if need_grad:
            ledger.retain_saved(led, "head", {"x": x, "inv_f": inv_f, "grad_hidden": grad_hidden})
        led.mark("post_forward")
        # post_forward mark (model.py:296): activation bytes = everything still
        # allocated by this step that backward needs
        mark = _lib.memory_allocated(dev)
        m.last_stats = {"activation_bytes_post_forward": mark - mem0,
                        "retained": dict(src.last_fractions) if src is not None else {}}
        if need_grad:
            self.saved, self.x, self.inv_f, self.grad_hidden = saved, x, inv_f, grad_hidden
        return loss.to(F32).reshape(())

    def backward(self, g: torch.Tensor) -> torch.Tensor:
        m = self.model
        gval = float(g.item()) if isinstance(g, torch.Tensor) else float(g)
        grad = torch.zeros_like(m.lora_param)
        dx = torch.empty_like(self.x)
        ops.rmsnorm_bwd(self.grad_hidden, self.x, self.inv_f, m.final_norm_w, dx, None,
                        gscale=gval, accumulate=False)
        led = ledger.get()
        ledger.release_saved(led, {"x": self.x, "inv_f": self.inv_f,
                                   "grad_hidden": self.grad_hidden})
        self.grad_hidden = self.x = self.inv_f = None
        main = torch.cuda.current_stream(m.device)
        pending = []  # LoRA-gradient kernels still running on the side stream
        for layer, (sa, sm) in zip(reversed(m.layers), reversed(self.saved)):
            if sm is not None:
                kernels.mlp_backward(dx, sm, layer)
                ledger.release_saved(led, sm)
            if sa is not None:
                ev = kernels.attention_backward(dx, sa, layer, layer.grad_views(grad))
                if ev is not None:
                    pending.append(ev)
                ledger.release_saved(led, sa)
            if m.grad_reducer is not None and layer.lora_rank:
                for ev in pending:  # this layer's bucket must be final before it is reduced
                    main.wait_event(ev)
                pending = []
                off = m._lora_offset(layer.layer_id)
                m.grad_reducer.layer_ready(layer.layer_id,
                                           grad[off:off + m._lora_offset(1)])
            self.saved.pop()
        for ev in pending:
            main.wait_event(ev)
        self.saved = None
        if m.grad_reducer is not None:
            m.grad_reducer.finish()
        return grad


class _StepFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, lora_param, step):
        ctx.step = step
        return step.forward(need_grad=True)

    @staticmethod
    def backward(ctx, g):
        step = ctx.step
        ctx.step = None
        return step.backward(g), None


# ---------------------------------------------------------------------------
# scoring helpers (model.py:356-396)


def _precision(layer: LayerState, precision):
    """The precision one scorer call runs in ("refined" scores in bf16 first)."""
    p = precision or layer.scoring_precision
    if p not in SCORING_PRECISIONS:
        raise ContractError(f"unknown scoring precision {p!r}")
    return "bf16" if p == "refined" else p


def mlp_block_score_vector(layer: LayerState, x: torch.Tensor, block_size: int, n_valid: int,
                           *, keep_rows: bool = False, precision: str | None = None,
                           with_partial: bool = False):
    """Exact MLP block scores (model.py:371-396): RMSNorm of every row, the
    tcgen05 gate/up GEMM with |silu(g)·u| row sums in its epilogue, then
    mean/max per block.  With keep_rows=True also returns (gu_all, inv_all)
    so the sparse MLP can compact retained rows instead of recomputing;
    with_partial=True appends the per-tile row partials [n_tiles, s] (the
    token scores, for refine_mlp_block_scores).

    precision "fp32" (parity): fp32 RMSNorm, bf16x3 operands over K = 3h and
    scores from the fp32 accumulator -- the reference's f32 scores to ~1e-6."""
    s, h = x.shape
    dev = x.device
    N = layer.w_gu_t.shape[0]
    inv_all = torch.empty(s, dtype=F32, device=dev)
    gu_all = torch.empty(s, N, dtype=BF16, device=dev) if keep_rows else None
    partial = torch.empty(N // 128, s, dtype=F32, device=dev)
    if _precision(layer, precision) == "fp32":
        xnf = ops.rmsnorm_f32(x, layer.mlp_norm_w, inv=inv_all)
        a3 = layer.split_input(xnf)
        del xnf
        ops.gemm_gateup(a3, layer.gateup_x3(), gu=gu_all, partial=partial, relu=layer.relu,
                        exact_score=True)
        del a3
    else:
        # RMSNorm folded into the epilogue: bf16(x·w) in, ·1/rms on the accumulator
        xw_all = ops.rmsnorm_gather_fold(x, layer.mlp_norm_w, inv=inv_all)
        ops.gemm_gateup(xw_all, layer.w_gu_t, gu=gu_all, partial=partial, relu=layer.relu,
                        row_scale=inv_all)
        del xw_all
    vec = ops.mlp_block_scores(partial, s=s, n_valid=n_valid, b=block_size, m_real=layer.m)
    out = (vec,) + (((gu_all, inv_all),) if keep_rows else ()) + ((partial,) if with_partial else ())
    return out if len(out) > 1 else vec


def refine_mlp_block_scores(layer: LayerState, x: torch.Tensor, vec: torch.Tensor,
                            partial: torch.Tensor, thr: float, block_size: int, n_valid: int, *,
                            margin: float | None = None, capacity: int | None = None):
    """Refined MLP scoring (decisions of sparsity.py:274-277 on the block max
    of sparsity.py:298-305).  A block whose bf16 score lies within δ =
    margin·|thr| of the threshold is ambiguous; of its rows only those whose
    own bf16 token score is >= thr - δ can make max_t score_t >= thr (the
    rest are below thr even after a δ-sized error), so only those rows are
    re-scored in the fp32-faithful parity precision and the block's score in
    `vec` is replaced, in place, by their maximum -- the parity-precision
    decision.  `partial` is the bf16 scorer's per-tile row partials
    ([n_tiles, s], mlp_block_score_vector(..., with_partial=True)).  Returns
    the number of rows re-scored.

    The bf16 score error is measured at ≤ 5.2e-4 relative at Llama2-7B width
    (the bench's mask audit), so the default margin of 2e-3 leaves a 4×
    safety factor (tests/test_parity_gpu.py).  For a still-dropped block the
    patched value may differ from its full parity score (a non-re-scored row
    may hold the maximum); both are below the threshold.  One extra host
    read-back (the number of rows sizes the GEMM) -- or, with `capacity`,
    none: the GEMM runs on `capacity` rows and the device [count, overflow]
    pair is returned for the caller's own read-back (_refine_capacity)."""
    if not math.isfinite(thr):  # -inf retains every block, +inf none: nothing is ambiguous
        return 0
    margin = layer.refine_margin if margin is None else margin
    s = x.shape[0]
    band = ops.mlp_token_band(partial, vec, thr, margin * abs(thr), n_valid=n_valid,
                              b=block_size, m_real=layer.m)
    if capacity is not None:
        return _refine_capacity(layer, x, vec, band, block_size, capacity)
    cand = sparsity.select_device(band, 0.0, block_size=1, n_tokens=s)[0]
    rows = cand.k
    if rows == 0:
        return 0
    tok = cand.device_token_indices(x.device)
    _refine_rows(layer, x, vec, tok, rows, block_size)
    return rows


def _refine_rows(layer, x, vec, tok, rows, block_size, count=None, overflow=None):
    """Parity-precision gate/up scores of the rows tok[:rows] patched into vec."""
    xnf = ops.rmsnorm_f32(x, layer.mlp_norm_w, tok)
    a = layer.split_input(xnf)
    del xnf
    N = layer.w_gu_t.shape[0]
    part = torch.empty(N // 128, rows, dtype=F32, device=x.device)
    ops.gemm_gateup(a, layer.gateup_x3(), partial=part, relu=layer.relu, exact_score=True)
    ops.mlp_patch_rows(part, tok, b=block_size, m_real=layer.m, vec=vec, count=count,
                       overflow=overflow)


def _refine_capacity(layer, x, vec, band, block_size, capacity):
    """The refinement without a host read-back of the row count: the band rows
    are compacted on the device into a zero-padded index list, the parity GEMM
    runs on `capacity` rows (padding rows score row 0 and are ignored by the
    patch kernel) and the patch kernel raises a device flag when the true
    count exceeds the capacity.  Returns the device int32 [count, overflow]
    pair; the caller reads it back with its own selection read-back and
    re-runs the exact refinement on overflow (RefineCapacity)."""
    s = x.shape[0]
    dev = x.device
    capacity = max(1, min(int(capacity), s))  # the band never holds more than s rows
    ws = sparsity.SelectWorkspace(s, s, 1, dev)
    ws.tokens.zero_()
    ops.select(band, b=1, n_tokens=s, thr=0.0, mask=ws.mask, blocks=ws.blocks, tokens=ws.tokens,
               counts=ws.counts, thr_out=ws.thr)
    flags = torch.empty(2, dtype=torch.int32, device=dev)  # [count, overflow]
    flags[:1].copy_(ws.counts[:1])
    _refine_rows(layer, x, vec, ws.tokens[:capacity], capacity, block_size, count=flags[:1],
                 overflow=flags[1:])
    return flags


class RefineCapacity:
    """Per-layer capacity of the read-back-free refinement: the first call of
    a layer runs the exact path (one count read-back); later calls run on
    1.1 x the last count + 8 rows, rounded up to the GEMM's row tile (128
    rows for a single-CTA tile, else multiples of the 256-row CTA-pair tile),
    so the padding adds no tiles over the exact count in the common case (N*:
    ≈ 214 rows -> 256); an overflow re-runs the exact path from the bf16
    partials."""

    def __init__(self):
        self.cap: dict = {}

    def for_layer(self, layer_id):
        return self.cap.get(layer_id)

    def update(self, layer_id, count: int) -> None:
        target = int(count * 1.1) + 8
        self.cap[layer_id] = 128 if target <= 128 else -(-target // 256) * 256


def layer_qk(layer: LayerState, x: torch.Tensor, *, precision: str | None = None):
    """model.py:356-368: post-rotation Q (with LoRA) and K (without).

    "bf16": (q, k) bf16 [s, h] / [s, kv] from the tcgen05 q/k GEMM with RoPE
    in its epilogue.  "fp32" (parity): ((q_hi, q_lo), (k_hi, k_lo)) -- fp32
    RMSNorm, bf16x3 projections, LoRA and RoPE in fp32 (lemo_qk_finish)."""
    s, h = x.shape
    r = layer.lora_rank
    if _precision(layer, precision) == "fp32":
        xnf = ops.rmsnorm_f32(x, layer.attn_norm_w)
        qk = ops.gemm_f32_exact(layer.split_input(xnf), layer.qk_x3())
        t = None
        if r:  # the LoRA factors are fp32 (not bf16-exact): bf16x3 always
            a_t = ops.split_bf16x3_t(layer.lora_A.contiguous(), 1)  # [2r, 3h]
            t = ops.gemm_f32_exact(ops.split_bf16x3(xnf, 0), a_t)
        del xnf
        q_hi, q_lo, k_hi, k_lo = ops.qk_finish(
            qk, t, layer.lora_Bq if r else None, r=r, scale=layer.lora_scaling,
            rope_tab=layer.rope_tab, h=h, kv=layer.kv, head_dim=layer.head_dim, rope=layer.rope)
        return (q_hi, q_lo), (k_hi, k_lo)
    # RMSNorm folded into the epilogue (as the MLP scorer): bf16(x·w) in; the
    # LoRA term xw·A·B is linear in the row, so one row scale covers both
    xn = torch.empty(s, layer.w_qkv_t.shape[1], dtype=BF16, device=x.device)
    inv = torch.empty(s, dtype=F32, device=x.device)
    ops.rmsnorm_gather_fold(x, layer.attn_norm_w, inv=inv, out=xn)
    if r:
        layer.qkv_input(xn)
    pos = torch.arange(s, dtype=torch.int32, device=x.device)
    q, k = ops.gemm_qkv(xn, layer.w_qkv_t, h=h, head_dim=layer.head_dim, rope=layer.rope,
                        inv_freq=layer.inv_freq, pos=pos, nmat=2, kv=layer.kv, row_scale=inv)
    return q, k


# ---------------------------------------------------------------------------
# pattern sources (model.py:403-590)


class PatternSourceBase:
    """Interleaves scoring with the layer loop; records retained fractions
    (and, in the refined precision, how many MLP rows were re-scored)."""

    def __init__(self):
        self.last_fractions: dict = {}
        self.refined_rows: dict = {}

    def pattern(self, layer_id, component, x, n_valid):
        raise NotImplementedError

    def _note(self, layer_id, component, pattern):
        self.last_fractions[(layer_id, component)] = (
            1.0 if pattern is None else pattern.retained_fraction)
        return pattern


class AllRetainSource(PatternSourceBase):
    def pattern(self, layer_id, component, x, n_valid):
        return self._note(layer_id, component, None)


class FixedPatternSource(PatternSourceBase):
    """Serves pre-built patterns keyed by (layer, component)."""

    def __init__(self, patterns: dict):
        super().__init__()
        self.patterns = patterns

    def pattern(self, layer_id, component, x, n_valid):
        return self._note(layer_id, component, self.patterns.get((layer_id, component)))


class FractionSource(PatternSourceBase):
    """Evenly spaced fraction of blocks (model.py:437-451)."""

    def __init__(self, fraction: float, block_size: int):
        super().__init__()
        self.fraction = fraction
        self.block_size = block_size

    def pattern(self, layer_id, component, x, n_valid):
        s = x.shape[0]
        nb = sparsity.n_blocks_for(s, self.block_size)
        keep = max(1, int(round(nb * self.fraction)))
        blocks = tuple(np.unique(np.linspace(0, nb - 1, keep).round().astype(int)).tolist())
        return self._note(layer_id, component,
                          sparsity.SparsityPattern(layer_id, component, blocks, self.block_size, s))


class PredictedPatternSource(PatternSourceBase):
    """model.py:516-590 on the GPU: attention blocks from the predictor pair
    (fused block-pool → predictors → Eq. 3 → clamp → column sums), optional
    periodic re-derivation of the threshold as an order statistic over the
    last `history` score vectors (radix select), MLP blocks from the exact
    fused MLP scorer; selection by the liblemo select kernel."""

    def __init__(self, model: DecoderModel, pred_thresholds: sparsity.ThresholdSet, *,
                 mlp_scoring: bool = True, sink_first_block: bool = False, pooling: str = "mean",
                 target_retention: dict | None = None, recalibrate_every: int = 0,
                 history: int = 8, record: bool = False):
        super().__init__()
        self.model = model
        self.thresholds = pred_thresholds
        self.mlp_scoring = mlp_scoring
        self.sink_first_block = sink_first_block
        self.pooling = pooling
        self.target_retention = target_retention or {}
        self.recalibrate_every = recalibrate_every
        self.history = history
        self.record = record
        self.recorded_vectors: dict = {}
        self._recent: dict = {}
        self._calls: dict = {}
        self._refine_cap = RefineCapacity()

    def _maybe_recalibrate(self, layer_id, vec):
        """model.py:545-563; returns a device threshold or None."""
        if not self.recalibrate_every or layer_id not in self.target_retention:
            return None
        recent = self._recent.setdefault(layer_id, [])
        recent.append(vec)
        if len(recent) > self.history:
            recent.pop(0)
        self._calls[layer_id] = self._calls.get(layer_id, 0) + 1
        if self._calls[layer_id] % self.recalibrate_every != 0:
            return None
        retained = min(max(self.target_retention[layer_id], 0.0), 1.0)
        out = torch.empty(1, dtype=torch.float64, device=vec.device)
        if retained >= 1.0:
            out.fill_(float("-inf"))
            return out
        pooled = torch.cat(recent) if len(recent) > 1 else recent[0]
        if retained <= 0.0:
            return ops.quantile_lower(pooled, 1.0, out, plus_one=True)
        return ops.quantile_lower(pooled, 1.0 - retained, out)

    def pattern(self, layer_id, component, x, n_valid):
        b = self.model.config.block_size
        layer = self.model.layers[layer_id]
        thr_dev = None
        if component == sparsity.ATTENTION:
            if layer.predictor_q is None or layer.predictor_k is None:
                raise ContractError(f"layer {layer_id} has no attached predictors")
            vec = predictor_mod.predicted_block_vector(layer.predictor_q, layer.predictor_k, x, b,
                                                       self.pooling)
            thr_dev = self._maybe_recalibrate(layer_id, vec)
            thr = None if thr_dev is not None else self.thresholds.get(layer_id, component)
        else:
            if not self.mlp_scoring:
                return self._note(layer_id, component, None)
            vec, rows, partial = mlp_block_score_vector(layer, x, b, n_valid, keep_rows=True,
                                                        with_partial=True)
            self.model.stash_mlp_rows(layer_id, x, rows)
            thr = self.thresholds.get(layer_id, component)
            if layer.scoring_precision == "refined":
                return self._refined_mlp(layer, layer_id, x, vec, partial, thr, n_valid)
            del partial
        if self.record:
            self.recorded_vectors.setdefault((layer_id, component), []).append(vec)
        force = (0,) if self.sink_first_block else ()
        pat, used = sparsity.select_device(vec, thr, thr_dev=thr_dev, layer_id=layer_id,
                                           component=component, block_size=b,
                                           n_tokens=x.shape[0], force_blocks=force)
        if thr_dev is not None:
            self.thresholds.set(layer_id, sparsity.ATTENTION, used)
        return self._note(layer_id, component, pat)


    def _refined_mlp(self, layer, layer_id, x, vec, partial, thr, n_valid):
        """MLP pattern in the refined precision without a separate read-back
        of the refinement's row count: the parity re-scoring runs on the
        layer's capacity (RefineCapacity) and its [count, overflow] pair rides
        on the selection's read-back; an overflow (more band rows than the
        capacity) re-scores exactly from fresh bf16 block scores."""
        b = self.model.config.block_size
        cap = self._refine_cap.for_layer(layer_id)
        flags = refine_mlp_block_scores(layer, x, vec, partial, thr, b, n_valid, capacity=cap)
        force = (0,) if self.sink_first_block else ()
        sel = dict(layer_id=layer_id, component=sparsity.MLP, block_size=b, n_tokens=x.shape[0],
                   force_blocks=force)
        if isinstance(flags, torch.Tensor):
            pat, _, (count, overflow) = sparsity.select_device(vec, thr, extra=flags, **sel)
            if overflow:
                vec = ops.mlp_block_scores(partial, s=x.shape[0], n_valid=n_valid, b=b,
                                           m_real=layer.m)
                count = refine_mlp_block_scores(layer, x, vec, partial, thr, b, n_valid)
                pat, _ = sparsity.select_device(vec, thr, **sel)
        else:  # exact path (first call of the layer, or nothing ambiguous)
            count = flags
            pat, _ = sparsity.select_device(vec, thr, **sel)
        self._refine_cap.update(layer_id, count)
        self.refined_rows[layer_id] = count
        if self.record:
            self.recorded_vectors.setdefault((layer_id, sparsity.MLP), []).append(vec)
        del partial
        return self._note(layer_id, sparsity.MLP, pat)


class ExactPatternSource(PatternSourceBase):
    """model.py:454-513: exact attention scores from the layer's actual Q/K
    (tcgen05 projections + fused exact block scorer) and exact MLP scores;
    thresholds=None profiles only (retain all)."""

    def __init__(self, model: DecoderModel, thresholds: sparsity.ThresholdSet | None, *,
                 mlp_scoring: bool = True, sink_first_block: bool = False, record: bool = False,
                 record_inputs: bool = False):
        super().__init__()
        self.model = model
        self.thresholds = thresholds
        self.mlp_scoring = mlp_scoring
        self.sink_first_block = sink_first_block
        self.record = record
        self.record_inputs = record_inputs
        self.recorded_vectors: dict = {}
        self.recorded_matrices: list = []   # BlockScoreMatrix (device, packed f64) per call
        self.recorded_inputs: dict = {}     # layer -> [x clones] (teacher inputs)

    def pattern(self, layer_id, component, x, n_valid):
        from . import exact  # noqa: WPS433 (kernel module)

        b = self.model.config.block_size
        layer = self.model.layers[layer_id]
        if component == sparsity.ATTENTION:
            q, k = layer_qk(layer, x)
            if self.record and self.record_inputs:
                # teacher generation (pipeline.py:280-300): keep the packed
                # triangle and a copy of x (the residual is updated in place)
                bsm = exact.exact_block_scores(q, k, b, n_heads=layer.n_heads, n_valid=n_valid,
                                               layer_id=layer_id)
                vec = sparsity.token_block_scores(bsm)
                self.recorded_matrices.append(bsm)
                self.recorded_inputs.setdefault(layer_id, []).append(x.clone())
            else:
                vec = exact.exact_block_vector(q, k, b, n_heads=layer.n_heads, n_valid=n_valid)
        else:
            if not self.mlp_scoring:
                return self._note(layer_id, component, None)
            keep = self.thresholds is not None
            res = mlp_block_score_vector(layer, x, b, n_valid, keep_rows=keep, with_partial=keep)
            if keep:
                vec, rows, partial = res
                self.model.stash_mlp_rows(layer_id, x, rows)
                if layer.scoring_precision == "refined":
                    self.refined_rows[layer_id] = refine_mlp_block_scores(
                        layer, x, vec, partial, self.thresholds.get(layer_id, component), b,
                        n_valid)
                del partial
            else:
                vec = res
        if self.record:
            self.recorded_vectors.setdefault((layer_id, component), []).append(vec)
        if self.thresholds is None:
            return self._note(layer_id, component, None)
        force = (0,) if self.sink_first_block else ()
        pat, _ = sparsity.select_device(vec, self.thresholds.get(layer_id, component),
                                        layer_id=layer_id, component=component, block_size=b,
                                        n_tokens=x.shape[0], force_blocks=force)
        return self._note(layer_id, component, pat)
