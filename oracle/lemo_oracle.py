"""CPU oracle: a NumPy restatement of the reference LeMo hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs use it, and only as the checker (or as the timed CPU
baseline) — never as the thing measured for the GPU numbers.

It restates, function by function, the algorithm of the reference package
`sparsetune` (/root/reference/pkg/src/sparsetune, cited as `file.py:line`).
It is pinned against outputs of the reference itself: tests/golden/*.npz are
produced by tests/golden/make_golden.py, which imports the reference in the
build container, and tests/test_oracle.py checks this module against every
fixture and against the reference's own known-answer tests.

Arithmetic follows the reference's precision map: float32 model math,
float64 packed score triangles / column sums / threshold compares.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

EPS = 1e-6          # rmsnorm eps, tensor.py:387 / model.py:333
NEG_INF = -1e30     # masked-score sentinel, tensor.py:24
ATTENTION, MLP = "attention", "mlp"  # sparsity.py:20-21


class OracleContractError(ValueError):
    """Mirror of sparsetune.errors.ContractError for the oracle."""


# ---------------------------------------------------------------------------
# block geometry and selection  (sparsity.py)


def n_blocks_for(n_tokens: int, block_size: int) -> int:
    """sparsity.py:27-28"""
    return -(-n_tokens // block_size)


def tri_size(n_blocks: int) -> int:
    """sparsity.py:31-32"""
    return n_blocks * (n_blocks + 1) // 2


def tri_index(m: int, n: int) -> int:
    """sparsity.py:35-37"""
    return m * (m + 1) // 2 + n


def token_indices(blocks, block_size: int, n_tokens: int) -> np.ndarray:
    """SparsityPattern.token_indices, sparsity.py:95-104 (int64 ascending)."""
    chunks = [np.arange(n * block_size, min((n + 1) * block_size, n_tokens)) for n in blocks]
    if not chunks:
        return np.empty(0, dtype=np.int64)
    return np.concatenate(chunks).astype(np.int64)


def eliminate(block_scores, threshold: float, force_blocks=()) -> tuple[int, ...]:
    """Retain n iff score[n] >= T, union forced blocks — sparsity.py:263-281."""
    s = np.asarray(block_scores, dtype=np.float64)
    if s.size and not np.isfinite(s).all():
        raise OracleContractError("block scores must be finite")
    keep = set(np.nonzero(s >= threshold)[0].tolist())
    keep.update(int(b) for b in force_blocks)
    return tuple(sorted(keep))


def token_block_scores(packed, n_blocks: int) -> np.ndarray:
    """Column sums of the packed lower triangle, f64, ascending m — sparsity.py:253-260."""
    packed = np.asarray(packed, dtype=np.float64)
    out = np.zeros(n_blocks)
    for m in range(n_blocks):
        base = tri_index(m, 0)
        out[: m + 1] += packed[base: base + m + 1]
    return out


def column_sums_dense(dense: np.ndarray) -> np.ndarray:
    """Same column sum from a dense [nb, nb] matrix (lower triangle used),
    adding rows in ascending m exactly like token_block_scores."""
    dense = np.asarray(dense, dtype=np.float64)
    nb = dense.shape[0]
    out = np.zeros(nb)
    for m in range(nb):
        out[: m + 1] += dense[m, : m + 1]
    return out


def quantile_lower(pooled, q: float) -> float:
    """np.quantile(pooled, q, method="lower") = sorted[floor((n-1)q)]
    (numpy 2.3 'lower' rule, used by model.py:562 and predictor.py:276)."""
    a = np.sort(np.asarray(pooled, dtype=np.float64).reshape(-1))
    idx = int(np.floor((a.size - 1) * q))
    return float(a[idx])


def recalibrated_threshold(pooled, retention: float) -> float:
    """PredictedPatternSource._maybe_recalibrate threshold rule, model.py:555-562."""
    pooled = np.asarray(pooled, dtype=np.float64)
    retained = min(max(retention, 0.0), 1.0)
    if retained >= 1.0:
        return float("-inf")
    if retained <= 0.0:
        return float(pooled.max()) + 1.0
    return quantile_lower(pooled, 1.0 - retained)


def retention_matched_threshold(pred_scores, exact_scores, exact_threshold: float) -> float:
    """predictor.py:257-276"""
    pred = np.asarray(pred_scores, dtype=np.float64).reshape(-1)
    exact = np.asarray(exact_scores, dtype=np.float64).reshape(-1)
    if pred.size == 0 or exact.size == 0:
        raise OracleContractError("cannot match retention on empty score sets")
    retained = float((exact >= exact_threshold).mean())
    if retained >= 1.0:
        return float("-inf")
    if retained <= 0.0:
        return float(pred.max()) + 1.0
    return quantile_lower(pred, 1.0 - retained)


def mlp_block_scores(token_scores, block_size: int, n_valid: int | None = None) -> np.ndarray:
    """sparsity.py:293-305"""
    t = np.asarray(token_scores, dtype=np.float64)
    s = t.shape[0]
    n_valid = s if n_valid is None else n_valid
    nb = n_blocks_for(s, block_size)
    out = np.zeros(nb)
    for n in range(nb):
        t0, t1 = n * block_size, min((n + 1) * block_size, s, n_valid)
        if t1 > t0:
            out[n] = t[t0:t1].max()
    return out


# ---------------------------------------------------------------------------
# elementwise helpers  (tensor.py)


def sigmoid(x: np.ndarray) -> np.ndarray:
    """tensor.py:368-374 (stable two-branch logistic)."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def rmsnorm_fwd(x: np.ndarray, w: np.ndarray):
    """tensor.py:387-402 / model.py:333-335: returns (out, inv)."""
    inv = (1.0 / np.sqrt((x * x).mean(axis=-1, keepdims=True) + EPS)).astype(x.dtype)
    return x * inv * w, inv


def rmsnorm_bwd(g: np.ndarray, x: np.ndarray, inv: np.ndarray, w: np.ndarray) -> np.ndarray:
    """dx of tensor.py:396-400 (weights are frozen: dweight dropped)."""
    n = x.shape[-1]
    gw = g * w
    return gw * inv - x * (inv ** 3) * ((gw * x).sum(axis=-1, keepdims=True) / n)


def rope_tables(positions: np.ndarray, half: int, base: float, dtype):
    """tensor.py:604-607 (angles in float64, cast after cos/sin)."""
    inv_freq = base ** (-np.arange(half, dtype=np.float64) / half)
    ang = np.asarray(positions)[:, None].astype(np.float64) * inv_freq[None, :]
    return np.cos(ang).astype(dtype), np.sin(ang).astype(dtype)


def rope_fwd(x: np.ndarray, positions, n_heads: int, base: float) -> np.ndarray:
    """tensor.py:610-625 (rotate-half per head)."""
    n, h = x.shape
    d = h // n_heads
    half = d // 2
    c, s = rope_tables(positions, half, base, x.dtype)
    x3 = x.reshape(n, n_heads, d)
    xa, xb = x3[..., :half], x3[..., half:]
    ca, sa = c[:, None, :], s[:, None, :]
    return np.concatenate([xa * ca - xb * sa, xa * sa + xb * ca], axis=-1).reshape(n, h)


def rope_bwd(g: np.ndarray, positions, n_heads: int, base: float) -> np.ndarray:
    """tensor.py:627-632"""
    n, h = g.shape
    d = h // n_heads
    half = d // 2
    c, s = rope_tables(positions, half, base, g.dtype)
    g3 = g.reshape(n, n_heads, d)
    ga, gb = g3[..., :half], g3[..., half:]
    ca, sa = c[:, None, :], s[:, None, :]
    return np.concatenate([ga * ca + gb * sa, -ga * sa + gb * ca], axis=-1).reshape(n, h)


def causal_attention_fwd(q, k, v, n_heads: int):
    """Multi-head causal softmax attention (tensor.py:646-691), computed per
    head with a dense masked score matrix.  Returns (out [n,h], lse [H,n]).
    GQA extension (not in the reference): k, v narrower than q carry
    h/kv-fold fewer heads, query head hd reads key head hd // group — the
    same math as the reference on K/V heads repeated `group` times."""
    n, h = q.shape
    d = h // n_heads
    group = h // k.shape[1]
    dt = q.dtype
    scale = dt.type(1.0 / np.sqrt(d))
    out = np.empty_like(q)
    lse = np.empty((n_heads, n), dtype=dt)
    mask = np.tril(np.ones((n, n), dtype=bool))
    for hd in range(n_heads):
        sl = slice(hd * d, (hd + 1) * d)
        kl = slice((hd // group) * d, (hd // group + 1) * d)
        s = (q[:, sl] * scale) @ k[:, kl].T
        s = np.where(mask, s, dt.type(NEG_INF))
        mx = s.max(axis=-1, keepdims=True)
        with np.errstate(under="ignore"):
            e = np.exp(s - mx)
        l = e.sum(axis=-1, keepdims=True)
        out[:, sl] = (e / l) @ v[:, kl]
        lse[hd] = (mx + np.log(l))[:, 0]
    return out, lse


def causal_attention_bwd(g, q, k, v, out, lse, n_heads: int):
    """tensor.py:693-722 (P recomputed from lse, Δ = rowsum(dO·O))."""
    n, h = q.shape
    d = h // n_heads
    group = h // k.shape[1]
    dt = q.dtype
    scale = dt.type(1.0 / np.sqrt(d))
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    mask = np.tril(np.ones((n, n), dtype=bool))
    for hd in range(n_heads):
        sl = slice(hd * d, (hd + 1) * d)
        kl = slice((hd // group) * d, (hd // group + 1) * d)
        qs = q[:, sl] * scale
        s = np.where(mask, qs @ k[:, kl].T, dt.type(NEG_INF))
        with np.errstate(under="ignore"):
            p = np.exp(s - lse[hd][:, None])
        gi = g[:, sl]
        delta = (gi * out[:, sl]).sum(axis=-1, keepdims=True)
        dp = gi @ v[:, kl].T
        ds = p * (dp - delta)
        dq[:, sl] = ds @ k[:, kl] * scale
        dk[:, kl] += ds.T @ qs   # GQA: the group's query heads accumulate
        dv[:, kl] += p.T @ gi
    return dq, dk, dv


# ---------------------------------------------------------------------------
# model (model.py) — weights stored [in, out] like the reference


@dataclass
class Config:
    """ModelConfig fields, model.py:23-37."""
    n_layers: int = 4
    hidden_dim: int = 64
    n_heads: int = 4
    vocab_size: int = 256
    max_seq_len: int = 2048
    mlp_variant: str = "silu"
    mlp_dim: int = 256
    lora_rank: int = 8
    lora_alpha: float = 16.0
    block_size: int = 16
    positions: str = "rope"
    rope_base: float = 10000.0
    n_kv_heads: int = 0  # GQA extension (0 = n_heads, the reference's MHA)

    @property
    def head_dim(self) -> int:
        return self.hidden_dim // self.n_heads

    @property
    def kv_dim(self) -> int:
        return (self.n_kv_heads or self.n_heads) * self.head_dim


@dataclass
class Layer:
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    attn_norm: np.ndarray
    mlp_norm: np.ndarray
    w_up: np.ndarray
    w_down: np.ndarray
    w_gate: np.ndarray | None
    lora_q: list | None   # [a (h,r), b (r,h)]
    lora_v: list | None
    scaling: float
    n_heads: int
    rope: bool
    rope_base: float
    mlp_variant: str
    n_kv_heads: int = 0
    predictor_q: "Predictor | None" = None
    predictor_k: "Predictor | None" = None


@dataclass
class Model:
    cfg: Config
    embed: np.ndarray
    pos_embed: np.ndarray | None
    layers: list
    final_norm: np.ndarray
    lm_head: np.ndarray

    def adapter_names(self):
        out = []
        for i, L in enumerate(self.layers):
            for tag, ad in (("lora_q", L.lora_q), ("lora_v", L.lora_v)):
                if ad is not None:
                    out += [f"layer{i}.{tag}.a", f"layer{i}.{tag}.b"]
        return out

    def adapter(self, name):
        i, tag, ab = name.split(".")
        L = self.layers[int(i[5:])]
        ad = L.lora_q if tag == "lora_q" else L.lora_v
        return ad[0] if ab == "a" else ad[1]


def init_model(cfg: Config, seed: int = 0, dtype=np.float32, fast: bool = False) -> Model:
    """Same draw order as DecoderModel.__init__ / LayerState / LoraAdapter
    (model.py:67-153).  fast=True draws float32 normals directly (different
    values, same distribution) — used only for the timed CPU sample."""
    rng = np.random.default_rng(seed)
    if fast:
        gen = rng

        class _R:
            @staticmethod
            def standard_normal(shape):
                return gen.standard_normal(shape, dtype=np.float32)
        rng = _R()
    h, m = cfg.hidden_dim, cfg.mlp_dim
    std = 1.0 / np.sqrt(h)
    embed = (rng.standard_normal((cfg.vocab_size, h)) * std).astype(dtype)
    pos = None
    if cfg.positions == "learned":
        pos = (rng.standard_normal((cfg.max_seq_len, h)) * std).astype(dtype)
    layers = []
    for _ in range(cfg.n_layers):
        def w(rows, cols):
            return (rng.standard_normal((rows, cols)) * std).astype(dtype)
        kv = cfg.kv_dim
        wq, wk, wv, wo = w(h, h), w(h, kv), w(h, kv), w(h, h)
        w_up = w(h, m)
        w_down = w(m, h)
        w_gate = w(h, m) if cfg.mlp_variant == "silu" else None
        lq = lv = None
        if cfg.lora_rank > 0:
            lq = [(rng.standard_normal((h, cfg.lora_rank)) / np.sqrt(h)).astype(dtype),
                  np.zeros((cfg.lora_rank, h), dtype=dtype)]
            lv = [(rng.standard_normal((h, cfg.lora_rank)) / np.sqrt(h)).astype(dtype),
                  np.zeros((cfg.lora_rank, kv), dtype=dtype)]
        layers.append(Layer(wq, wk, wv, wo, np.ones(h, dtype), np.ones(h, dtype), w_up, w_down,
                            w_gate, lq, lv, cfg.lora_alpha / max(cfg.lora_rank, 1), cfg.n_heads,
                            cfg.positions == "rope", cfg.rope_base, cfg.mlp_variant,
                            cfg.n_kv_heads or cfg.n_heads))
    final = np.ones(h, dtype)
    lm = (rng.standard_normal((h, cfg.vocab_size)) * std).astype(dtype)
    return Model(cfg, embed, pos, layers, final, lm)


def perturb_lora_b(model: Model, seed: int, std: float = 0.1):
    """Nonzero B so dA != 0 (the parity variant of test_acceptance.py:144-145)."""
    rng = np.random.default_rng(seed)
    for L in model.layers:
        for ad in (L.lora_q, L.lora_v):
            if ad is not None:
                ad[1] = (rng.standard_normal(ad[1].shape) * std).astype(ad[1].dtype)


# ---------------------------------------------------------------------------
# predictor (predictor.py)


@dataclass
class Predictor:
    w1: np.ndarray
    w2: np.ndarray
    w3: np.ndarray
    mask1: np.ndarray = None
    mask2: np.ndarray = None

    def __post_init__(self):
        if self.mask1 is None:
            self.mask1 = np.ones(self.w1.shape[1], dtype=bool)
        if self.mask2 is None:
            self.mask2 = np.ones(self.w2.shape[1], dtype=bool)

    def predict(self, x: np.ndarray) -> np.ndarray:
        """predictor.py:83-89"""
        dt = self.w1.dtype
        x = np.asarray(x, dtype=dt)
        h1 = np.maximum(x @ self.w1, 0) * self.mask1.astype(dt)
        h2 = np.maximum(h1 @ self.w2, 0) * self.mask2.astype(dt)
        return h2 @ self.w3


def create_predictor(rng, h, r1, r2, d_pred, dtype=np.float32) -> Predictor:
    """Predictor.create, predictor.py:52-58"""
    def init(rows, cols):
        return (rng.standard_normal((rows, cols)) / np.sqrt(rows)).astype(dtype)
    return Predictor(init(h, r1), init(r1, r2), init(r2, d_pred))


def block_embed(x: np.ndarray, block_size: int) -> np.ndarray:
    """predictor.py:117-123"""
    s, h = x.shape
    if s % block_size != 0:
        raise OracleContractError(f"sequence length {s} not a multiple of block size {block_size}")
    return x.reshape(s // block_size, block_size, h).mean(axis=1)


def predicted_dense(p_q: Predictor, p_k: Predictor, x, block_size, pooling="mean") -> np.ndarray:
    """eq·ekᵀ of predicted_triangle (predictor.py:152-186), dense [nb, nb]."""
    if pooling == "mean":
        xb = np.asarray(block_embed(x, block_size), dtype=p_q.w1.dtype)
        eq, ek = p_q.predict(xb), p_k.predict(xb)
    elif pooling == "token":
        xt = np.asarray(x, dtype=p_q.w1.dtype)
        nb = xt.shape[0] // block_size
        eq = p_q.predict(xt).reshape(nb, block_size, -1).mean(axis=1)
        ek = p_k.predict(xt).reshape(nb, block_size, -1).mean(axis=1)
    else:
        raise OracleContractError(f"unknown pooling mode {pooling!r}")
    return eq @ ek.T


def predicted_triangle(p_q, p_k, x, block_size, pooling="mean") -> np.ndarray:
    """Packed lower triangle, unclamped (predictor.py:176-186)."""
    full = predicted_dense(p_q, p_k, x, block_size, pooling)
    r, c = np.tril_indices(full.shape[0])
    return full[r, c]


def predicted_block_vector(p_q, p_k, x, block_size, pooling="mean") -> np.ndarray:
    """model.py:572-578: clamp >= 0, BlockScoreMatrix (f64), column sums."""
    full = predicted_dense(p_q, p_k, x, block_size, pooling)
    return column_sums_dense(np.maximum(full, 0.0))


# ---------------------------------------------------------------------------
# scorers (model.py / sparsity.py)


def layer_qk(L: Layer, x: np.ndarray):
    """model.py:356-368 — [H, s, d] q (with LoRA) and k (without)."""
    n, h = x.shape
    xn, _ = rmsnorm_fwd(x, L.attn_norm)
    q = xn @ L.wq
    if L.lora_q is not None:
        q = q + (xn @ L.lora_q[0]) @ L.lora_q[1] * L.scaling
    k = xn @ L.wk
    nkv = L.n_kv_heads or L.n_heads
    if L.rope:
        pos = np.arange(n)
        q = rope_fwd(q, pos, L.n_heads, L.rope_base)
        k = rope_fwd(k, pos, nkv, L.rope_base)
    d = h // L.n_heads
    th = lambda a, H: np.ascontiguousarray(a.reshape(n, H, d).transpose(1, 0, 2))
    # GQA extension: key heads repeated to the query heads for Eq. 2
    return th(q, L.n_heads), np.repeat(th(k, nkv), L.n_heads // nkv, axis=0)


def exact_block_dense(q, k, block_size, n_valid=None, strip_blocks: int = 8) -> np.ndarray:
    """Dense [nb, nb] form of exact_block_scores (sparsity.py:173-219): per
    pair Σ_h max(q·k, 0)/H (no 1/√d), causal + n_valid mask, tile max.
    The reference forms one query-block strip at a time; here `strip_blocks`
    query blocks share one strip GEMM (the same per-element dot products and
    head sum; the tile maxima are taken by a reshape instead of a loop)."""
    if q.ndim == 2:
        q, k = q[None], k[None]
    H, s, _ = q.shape
    if block_size > s:
        raise OracleContractError(f"block size {block_size} exceeds sequence length {s}")
    n_valid = s if n_valid is None else n_valid
    b = block_size
    nb = n_blocks_for(s, b)
    out = np.zeros((nb, nb))
    for m0 in range(0, nb, strip_blocks):
        m1 = min(m0 + strip_blocks, nb)
        r0, r1 = m0 * b, min(m1 * b, s)
        strip = q[:, r0:r1] @ k[:, :r1].transpose(0, 2, 1)
        agg = np.maximum(strip, 0.0).sum(axis=0) / H
        rows = np.arange(r0, r1)[:, None]
        cols = np.arange(r1)[None, :]
        keep = (cols <= rows) & (rows < n_valid) & (cols < n_valid)
        agg = np.where(keep, agg, 0.0).astype(strip.dtype)
        nr, nc = m1 - m0, n_blocks_for(r1, b)
        pad = np.zeros((nr * b, nc * b), agg.dtype)  # masked / ragged entries are 0 anyway
        pad[: r1 - r0, :r1] = agg
        tiles = pad.reshape(nr, b, nc, b).max(axis=(1, 3))
        for i in range(nr):
            m = m0 + i
            out[m, : m + 1] = tiles[i, : m + 1]
    return out


def exact_block_scores(q, k, block_size, n_valid=None) -> np.ndarray:
    """Packed f64 triangle (sparsity.py:173-219)."""
    dense = exact_block_dense(q, k, block_size, n_valid)
    r, c = np.tril_indices(dense.shape[0])
    return dense[r, c].astype(np.float64)


def mlp_block_score_vector(L: Layer, x: np.ndarray, block_size: int, n_valid: int) -> np.ndarray:
    """model.py:371-396 (+ sparsity.py:284-290)."""
    s = x.shape[0]
    nb = n_blocks_for(s, block_size)
    out = np.zeros(nb)
    lim = min(s, n_valid)
    # rows are independent: stream a few blocks per GEMM (same per-row math as
    # the reference's one-block-at-a-time loop, better BLAS efficiency)
    per = block_size * max(1, 256 // block_size)
    for c0 in range(0, lim, per):
        c1 = min(c0 + per, lim)
        xn, _ = rmsnorm_fwd(x[c0:c1], L.mlp_norm)
        if L.mlp_variant == "silu":
            gate = xn @ L.w_gate
            inner = gate * sigmoid(gate) * (xn @ L.w_up)
        else:
            inner = np.maximum(xn @ L.w_up, 0)
        tok = np.abs(inner).mean(axis=-1).astype(np.float64)
        for blk in range(c0 // block_size, n_blocks_for(c1, block_size)):
            t0, t1 = blk * block_size, min((blk + 1) * block_size, c1)
            out[blk] = tok[t0 - c0:t1 - c0].max()
    return out


# ---------------------------------------------------------------------------
# pattern sources (model.py:403-590)


@dataclass
class PredictedSource:
    """PredictedPatternSource semantics (model.py:516-590)."""
    model: Model
    thresholds: dict            # (layer, comp) -> float
    mlp_scoring: bool = True
    sink_first_block: bool = False
    pooling: str = "mean"
    target_retention: dict = field(default_factory=dict)
    recalibrate_every: int = 0
    history: int = 8
    recent: dict = field(default_factory=dict)
    calls: dict = field(default_factory=dict)
    vectors: dict = field(default_factory=dict)   # last score vector per (l, c)

    def _maybe_recalibrate(self, layer_id, vec):
        if not self.recalibrate_every or layer_id not in self.target_retention:
            return
        recent = self.recent.setdefault(layer_id, [])
        recent.append(vec)
        if len(recent) > self.history:
            recent.pop(0)
        self.calls[layer_id] = self.calls.get(layer_id, 0) + 1
        if self.calls[layer_id] % self.recalibrate_every != 0:
            return
        self.thresholds[(layer_id, ATTENTION)] = recalibrated_threshold(
            np.concatenate(recent), self.target_retention[layer_id])

    def pattern(self, layer_id, component, x, n_valid):
        cfg = self.model.cfg
        b = cfg.block_size
        L = self.model.layers[layer_id]
        if component == ATTENTION:
            if L.predictor_q is None or L.predictor_k is None:
                raise OracleContractError(f"layer {layer_id} has no attached predictors")
            vec = predicted_block_vector(L.predictor_q, L.predictor_k, x, b, self.pooling)
            self._maybe_recalibrate(layer_id, vec)
            thr = self.thresholds[(layer_id, ATTENTION)]
        else:
            if not self.mlp_scoring:
                return None
            vec = mlp_block_score_vector(L, x, b, n_valid)
            thr = self.thresholds[(layer_id, MLP)]
        self.vectors[(layer_id, component)] = vec
        force = (0,) if self.sink_first_block else ()
        return eliminate(vec, thr, force)


@dataclass
class ExactSource:
    """ExactPatternSource semantics (model.py:454-513), thresholds optional."""
    model: Model
    thresholds: dict | None
    mlp_scoring: bool = True
    sink_first_block: bool = False
    vectors: dict = field(default_factory=dict)

    def pattern(self, layer_id, component, x, n_valid):
        b = self.model.cfg.block_size
        L = self.model.layers[layer_id]
        if component == ATTENTION:
            q, k = layer_qk(L, x)
            vec = token_block_scores(exact_block_scores(q, k, b, n_valid),
                                     n_blocks_for(x.shape[0], b))
        else:
            if not self.mlp_scoring:
                return None
            vec = mlp_block_score_vector(L, x, b, n_valid)
        self.vectors[(layer_id, component)] = vec
        if self.thresholds is None:
            return None
        force = (0,) if self.sink_first_block else ()
        return eliminate(vec, self.thresholds[(layer_id, component)], force)


@dataclass
class FixedSource:
    """FixedPatternSource (model.py:426-434): blocks per (layer, comp)."""
    patterns: dict

    def pattern(self, layer_id, component, x, n_valid):
        return self.patterns.get((layer_id, component))


# ---------------------------------------------------------------------------
# the training step (DecoderModel.forward_step + backward, model.py:246-297,
# kernels.py:153-288, tensor.py:208-245)


def pad_tokens(tokens, targets, block_size, max_seq_len):
    """model.py:218-236"""
    tokens = np.asarray(tokens, dtype=np.int64)
    n = tokens.shape[0]
    if n == 0:
        raise OracleContractError("empty token sequence")
    if n > max_seq_len:
        raise OracleContractError(f"sequence length {n} exceeds max {max_seq_len}")
    if targets is None:
        targets = np.concatenate([tokens[1:], [-1]])
    targets = np.asarray(targets, dtype=np.int64)
    n_pad = -(-n // block_size) * block_size
    if n_pad > n:
        tokens = np.concatenate([tokens, np.zeros(n_pad - n, dtype=np.int64)])
        targets = np.concatenate([targets, np.full(n_pad - n, -1, dtype=np.int64)])
    return tokens, targets, n


def segment_edges(n_tokens: int, n_segments: int):
    """SegmentPlan.even, kernels.py:81-88"""
    if n_segments < 1 or n_segments > n_tokens:
        raise OracleContractError("bad segment count")
    return [round(i * n_tokens / n_segments) for i in range(n_segments + 1)]


def segmented_loss_and_grad(hidden, lm_head, targets, n_segments, ignore_index=-1):
    """kernels.py:229-288 (+ _ce_terms tensor.py:446-468): returns
    (loss, grad_hidden) with grad_hidden computed in the forward pass."""
    edges = segment_edges(hidden.shape[0], n_segments)
    grad_hidden = np.zeros_like(hidden)
    loss_sum, count = 0.0, 0
    for a, b in zip(edges[:-1], edges[1:]):
        logits = hidden[a:b] @ lm_head
        t = targets[a:b]
        valid = t != ignore_index
        rowmax = logits.max(axis=-1, keepdims=True)
        with np.errstate(under="ignore"):
            e = np.exp(logits - rowmax)
        sums = e.sum(axis=-1, keepdims=True)
        probs = e / sums
        lse = np.log(sums[:, 0]) + rowmax[:, 0]
        rows = np.arange(logits.shape[0])
        per_row = lse - logits[rows, np.where(valid, t, 0)]
        loss_sum += per_row[valid].sum()
        count += int(valid.sum())
        d = probs
        d[rows[valid], t[valid]] -= 1.0
        d[~valid] = 0.0
        grad_hidden[a:b] = d @ lm_head.T
    if count == 0:
        raise OracleContractError("segmented loss: no valid targets")
    grad_hidden /= count
    return float(loss_sum / count), grad_hidden


def _attention_fwd(L: Layer, x, idx):
    xg = x[idx]
    xn, inv = rmsnorm_fwd(xg, L.attn_norm)
    s = L.scaling
    tq = tv = None
    q = xn @ L.wq
    if L.lora_q is not None:
        tq = xn @ L.lora_q[0]
        q = q + (tq @ L.lora_q[1]) * np.float32(s)
    k = xn @ L.wk
    v = xn @ L.wv
    if L.lora_v is not None:
        tv = xn @ L.lora_v[0]
        v = v + (tv @ L.lora_v[1]) * np.float32(s)
    if L.rope:
        q = rope_fwd(q, idx, L.n_heads, L.rope_base)
        k = rope_fwd(k, idx, L.n_kv_heads or L.n_heads, L.rope_base)
    att, lse = causal_attention_fwd(q, k, v, L.n_heads)
    out = att @ L.wo
    saved = dict(idx=idx, xg=xg, xn=xn, inv=inv, tq=tq, tv=tv, q=q, k=k, v=v, att=att, lse=lse)
    return out, saved


def _attention_bwd(L: Layer, dx, S, grads, li):
    idx = S["idx"]
    g = dx[idx]
    datt = g @ L.wo.T
    dq, dk, dv = causal_attention_bwd(datt, S["q"], S["k"], S["v"], S["att"], S["lse"], L.n_heads)
    if L.rope:
        dq = rope_bwd(dq, idx, L.n_heads, L.rope_base)
        dk = rope_bwd(dk, idx, L.n_kv_heads or L.n_heads, L.rope_base)
    xn = S["xn"]
    dxn = dq @ L.wq.T + dk @ L.wk.T + dv @ L.wv.T
    s = np.float32(L.scaling)
    for tag, ad, t, dout in (("lora_q", L.lora_q, S["tq"], dq), ("lora_v", L.lora_v, S["tv"], dv)):
        if ad is None:
            continue
        dd = dout * s                      # d(t @ B)
        grads[f"layer{li}.{tag}.b"] += t.T @ dd
        dt = dd @ ad[1].T
        grads[f"layer{li}.{tag}.a"] += xn.T @ dt
        dxn = dxn + dt @ ad[0].T
    dx[idx] += rmsnorm_bwd(dxn, S["xg"], S["inv"], L.attn_norm)


def _mlp_fwd(L: Layer, x, idx):
    xg = x[idx]
    xn, inv = rmsnorm_fwd(xg, L.mlp_norm)
    if L.mlp_variant == "silu":
        gate = xn @ L.w_gate
        sg = sigmoid(gate)
        silu = gate * sg
        up = xn @ L.w_up
        inner = silu * up
    else:
        gate = sg = silu = None
        up = xn @ L.w_up
        inner = np.maximum(up, 0)
    out = inner @ L.w_down
    return out, dict(idx=idx, xg=xg, inv=inv, gate=gate, sg=sg, silu=silu, up=up)


def _mlp_bwd(L: Layer, dx, S):
    idx = S["idx"]
    g = dx[idx]
    dinner = g @ L.w_down.T
    if L.mlp_variant == "silu":
        dsilu = dinner * S["up"]
        dup = dinner * S["silu"]
        sg, gate = S["sg"], S["gate"]
        dgate = dsilu * (sg * (1.0 + gate * (1.0 - sg)))
        dxn = dgate @ L.w_gate.T + dup @ L.w_up.T
    else:
        dup = dinner * (S["up"] > 0)
        dxn = dup @ L.w_up.T
    dx[idx] += rmsnorm_bwd(dxn, S["xg"], S["inv"], L.mlp_norm)


def train_step(model: Model, tokens, targets=None, *, source=None, segments: int = 1,
               return_hidden: bool = False):
    """forward_step + backward for the LoRA adapters.

    Returns dict(loss, grads{name: array}, patterns{(l,c): blocks|None},
    layer_inputs{(l,c): x before the block})."""
    cfg = model.cfg
    ids, tgts, n_valid = pad_tokens(tokens, targets, cfg.block_size, cfg.max_seq_len)
    n_pad = len(ids)
    if ids.min() < 0 or ids.max() >= cfg.vocab_size:
        raise IndexError("token id out of range")
    x = model.embed[ids].copy()
    if model.pos_embed is not None:
        x = x + model.pos_embed[np.arange(n_pad)]
    patterns, inputs, saved = {}, {}, []
    b = cfg.block_size
    for li, L in enumerate(model.layers):
        inputs[(li, ATTENTION)] = x.copy()
        pat = source.pattern(li, ATTENTION, x, n_valid) if source is not None else None
        patterns[(li, ATTENTION)] = pat
        idx = np.arange(n_pad) if pat is None else token_indices(pat, b, n_pad)
        sa = None
        if idx.size:
            out, sa = _attention_fwd(L, x, idx)
            x = x.copy()
            x[idx] += out
        inputs[(li, MLP)] = x.copy()
        pat = source.pattern(li, MLP, x, n_valid) if source is not None else None
        patterns[(li, MLP)] = pat
        idx = np.arange(n_pad) if pat is None else token_indices(pat, b, n_pad)
        sm = None
        if idx.size:
            out, sm = _mlp_fwd(L, x, idx)
            x = x.copy()
            x[idx] += out
        saved.append((sa, sm))
    hidden, inv_f = rmsnorm_fwd(x, model.final_norm)
    loss, grad_hidden = segmented_loss_and_grad(hidden, model.lm_head, tgts, segments)
    grads = {n: np.zeros_like(model.adapter(n)) for n in model.adapter_names()}
    dx = rmsnorm_bwd(grad_hidden, x, inv_f, model.final_norm)
    for li in reversed(range(len(model.layers))):
        L = model.layers[li]
        sa, sm = saved[li]
        if sm is not None:
            _mlp_bwd(L, dx, sm)
        if sa is not None:
            _attention_bwd(L, dx, sa, grads, li)
    out = dict(loss=loss, grads=grads, patterns=patterns, layer_inputs=inputs)
    if return_hidden:
        out["hidden"] = hidden
    return out


def adam_step(params: dict, grads: dict, state: dict, lr=1e-3, betas=(0.9, 0.999), eps=1e-8,
              weight_decay=0.0):
    """optim.py:37-53 (in place on params; state holds t, m, v)."""
    state["t"] = state.get("t", 0) + 1
    b1, b2 = betas
    bc1 = 1.0 - b1 ** state["t"]
    bc2 = 1.0 - b2 ** state["t"]
    for name, p in params.items():
        g = grads[name].astype(p.dtype, copy=False)
        m = state.setdefault(("m", name), np.zeros_like(p))
        v = state.setdefault(("v", name), np.zeros_like(p))
        if weight_decay:
            p *= 1.0 - lr * weight_decay
        m *= b1
        m += (1.0 - b1) * g
        v *= b2
        v += (1.0 - b2) * (g * g)
        p -= lr * ((m / bc1) / (np.sqrt(v / bc2) + eps)).astype(p.dtype)
