"""Low-rank sparsity-pattern predictors on the GPU.

Mirrors ``sparsetune.predictor`` (predictor.py:32-276): a predictor is three
matrices with ReLU·mask between successive products; the block embedding is
the block mean of the residual stream; Eq. 3 dots the query- and key-side
outputs.  The fused scoring path used by the elimination hook is
`predicted_block_vector`: block_embed → 2 × (3 GEMMs) → eq·ekᵀ → clamp →
float64 column sums, six liblemo launches, no host round trip.

All predictor math is fp32 (as in the reference) so predicted scores — and
therefore the selected masks — track the reference to float rounding.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .errors import ContractError
from .sparsity import ATTENTION, BlockScoreMatrix, n_blocks_for, tri_size


class Predictor:
    """Three-matrix low-rank network (predictor.py:32-89); weights fp32 on the GPU."""

    def __init__(self, w1, w2, w3, role: str = "q", layer_id: int = 0, device=None):
        dev = torch.device(device) if device is not None else torch.device("cuda")
        self.w1 = _dev_f32(w1, dev)
        self.w2 = _dev_f32(w2, dev)
        self.w3 = _dev_f32(w3, dev)
        if self.w1.shape[1] != self.w2.shape[0] or self.w2.shape[1] != self.w3.shape[0]:
            raise ContractError(f"predictor matrix chain mismatch: {tuple(self.w1.shape)} "
                                f"{tuple(self.w2.shape)} {tuple(self.w3.shape)}")
        self.role = role
        self.layer_id = layer_id
        self.mask1 = torch.ones(self.w1.shape[1], dtype=torch.uint8, device=dev)
        self.mask2 = torch.ones(self.w2.shape[1], dtype=torch.uint8, device=dev)
        # zero-frequency counters of the two hidden stages (predictor.py:48-50)
        self.zero_counts1 = torch.zeros(self.w1.shape[1], dtype=torch.int64, device=dev)
        self.zero_counts2 = torch.zeros(self.w2.shape[1], dtype=torch.int64, device=dev)
        self.observed = 0
        self._split = None

    def touch(self) -> None:
        """Weights were updated in place by a liblemo kernel (invisible to
        torch's version counter): drop the cached bf16x3 operands."""
        self._split = None

    def _weights3(self):
        """bf16x3 B-operands [N, 3K] (pattern 1) of W1ᵀ, W2ᵀ, W3ᵀ — rebuilt only
        when the weights change (predictors are frozen during fine-tuning)."""
        key = tuple(int(w._version) for w in (self.w1, self.w2, self.w3))
        if self._split is None or self._split[0] != key:
            ws = tuple(ops.split_bf16x3(w.t().contiguous(), 1) for w in (self.w1, self.w2, self.w3))
            self._split = (key, ws)
        return self._split[1]

    def hidden3(self, x3: torch.Tensor, h1: torch.Tensor | None = None) -> torch.Tensor:
        """relu/mask hidden layers on a bf16x3 input; returns split h2 [M, 3 r2].
        h1: the first layer's split output when already computed (pair_hidden1)."""
        w1, w2, _ = self._weights3()
        if h1 is None:
            h1, _ = ops.gemm_split3(x3, w1, relu=True, mask=self.mask1, pattern=0)
        h2, _ = ops.gemm_split3(h1, w2, relu=True, mask=self.mask2, pattern=0)
        return h2

    @staticmethod
    def create(rng: np.random.Generator, h: int, r1: int, r2: int, d_pred: int, role: str,
               layer_id: int, device=None) -> "Predictor":
        """Predictor.create (predictor.py:52-58): N(0, 1/rows) init, same draw order."""
        def init(rows, cols):
            return (rng.standard_normal((rows, cols)) / np.sqrt(rows)).astype(np.float32)
        return Predictor(init(h, r1), init(r1, r2), init(r2, d_pred), role, layer_id, device)

    @property
    def d_pred(self) -> int:
        return self.w3.shape[1]

    def parameters(self):
        return [self.w1, self.w2, self.w3]

    def set_masks(self, mask1, mask2) -> None:
        self.mask1 = torch.as_tensor(np.asarray(mask1, dtype=np.uint8)).to(self.w1.device)
        self.mask2 = torch.as_tensor(np.asarray(mask2, dtype=np.uint8)).to(self.w1.device)

    def active_param_count(self) -> int:
        h = self.w1.shape[0]
        a1 = int(self.mask1.sum())
        a2 = int(self.mask2.sum())
        return h * a1 + a1 * a2 + a2 * self.d_pred

    def predict(self, x: torch.Tensor) -> torch.Tensor:
        """h1 = relu(x·W1)·m1; h2 = relu(h1·W2)·m2; out = h2·W3 (predictor.py:83-89),
        fp32-faithful on bf16 tensor cores (bf16x3 tcgen05 GEMMs)."""
        x = _dev_f32(x, self.w1.device)
        h2 = self.hidden3(ops.split_bf16x3(x, 0))
        _, out = ops.gemm_split3(h2, self._weights3()[2], split_out=False, f32_out=True)
        return out

    def predict3(self, x3: torch.Tensor, pattern: int, h1: torch.Tensor | None = None) -> torch.Tensor:
        """Predictor output in split form (pattern 0: A-side, 1: B-side of Eq. 3)."""
        h2 = self.hidden3(x3, h1)
        out, _ = ops.gemm_split3(h2, self._weights3()[2], pattern=pattern)
        return out

    def forward(self, x, track: bool = False) -> torch.Tensor:
        """predictor.py:73-81: the same values as predict(); track=True also
        bumps the zero-frequency counters of both hidden stages (the
        elastic-pruning statistics, predictor.py:76-80)."""
        if not track:
            return self.predict(x)
        out, _ = self.forward_train(_dev_f32(x, self.w1.device), track=True)
        return out

    def state_arrays(self) -> dict:
        """Everything needed to resume training (predictor.py:91-102, same keys)."""
        return {"w1": self.w1.cpu().numpy(), "w2": self.w2.cpu().numpy(),
                "w3": self.w3.cpu().numpy(), "mask1": self.mask1.cpu().numpy().astype(bool),
                "mask2": self.mask2.cpu().numpy().astype(bool),
                "zero_counts1": self.zero_counts1.cpu().numpy(),
                "zero_counts2": self.zero_counts2.cpu().numpy(),
                "observed": np.asarray([self.observed], dtype=np.int64)}

    def load_state_arrays(self, state: dict) -> None:
        for name in ("w1", "w2", "w3"):
            t = getattr(self, name)
            if tuple(t.shape) != tuple(state[name].shape):
                raise ContractError(f"predictor {name} shape mismatch on load")
            t.copy_(torch.as_tensor(np.asarray(state[name], dtype=np.float32)))
        self.touch()
        if "mask1" in state:
            self.set_masks(state["mask1"], state["mask2"])
        dev = self.w1.device
        if "zero_counts1" in state:
            self.zero_counts1 = torch.as_tensor(
                np.asarray(state["zero_counts1"], dtype=np.int64)).to(dev)
            self.zero_counts2 = torch.as_tensor(
                np.asarray(state["zero_counts2"], dtype=np.int64)).to(dev)
        if "observed" in state:
            self.observed = int(np.asarray(state["observed"]).reshape(-1)[0])

    # -- training-side forward / backward (fit_predictors) -------------------

    def forward_train(self, x: torch.Tensor, track: bool = False):
        """Differentiable forward (predictor.py:73-81) on block rows x [M, h]
        fp32; returns (out [M, d_pred] fp32, saved) with saved = fp32 hidden
        activations for the backward.  track=True bumps the zero counters."""
        w1, w2, w3 = self._weights3()
        x3 = ops.split_bf16x3(x, 0)
        h1s, h1 = ops.gemm_split3(x3, w1, relu=True, mask=self.mask1, pattern=0, f32_out=True)
        h2s, h2 = ops.gemm_split3(h1s, w2, relu=True, mask=self.mask2, pattern=0, f32_out=True)
        _, out = ops.gemm_split3(h2s, w3, split_out=False, f32_out=True)
        if track:
            ops.zero_count(h1, self.zero_counts1)
            ops.zero_count(h2, self.zero_counts2)
            self.observed += x.shape[0]
        return out, (x, h1, h2)

    def backward_train(self, dout: torch.Tensor, saved, grads) -> None:
        """Weight gradients of forward_train (ReLU·mask backward through the
        saved outputs), all products as bf16x3 tcgen05 GEMMs: dW3 = h2ᵀ·dout,
        dh2 = dout·W3ᵀ, dW2 = h1ᵀ·dpre2, dh1 = dpre2·W2ᵀ, dW1 = xᵀ·dpre1."""
        x, h1, h2 = saved
        g1, g2, g3 = grads

        def mm_t(a, b):  # aᵀ·b, both [M, ·] fp32
            return ops.gemm_split3(ops.split_bf16x3_t(a, 0), ops.split_bf16x3_t(b, 1),
                                   split_out=False, f32_out=True)[1]

        def mm_wt(a, w):  # a·wᵀ, w [N, K] fp32 row-major
            return ops.gemm_split3(ops.split_bf16x3(a, 0), ops.split_bf16x3(w, 1),
                                   split_out=False, f32_out=True)[1]

        g3.copy_(mm_t(h2, dout))
        dh2 = ops.relu_grad(mm_wt(dout, self.w3), h2)
        g2.copy_(mm_t(h1, dh2))
        dh1 = ops.relu_grad(mm_wt(dh2, self.w2), h1)
        g1.copy_(mm_t(x, dh1))


def _dev_f32(a, device) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float32).contiguous()
    return torch.as_tensor(np.asarray(a, dtype=np.float32)).to(device).contiguous()


def block_embed(x, block_size: int) -> torch.Tensor:
    """Block means of the residual rows (predictor.py:117-123)."""
    x = _dev_f32(x, x.device if isinstance(x, torch.Tensor) and x.is_cuda else "cuda")
    return ops.block_embed(x, block_size)


def pair_block_outputs(p_q: Predictor, p_k: Predictor, x, block_size: int, pooling: str = "mean"):
    """eq, ek block embedding vectors (predictor.py:152-173)."""
    if pooling == "mean":
        xb = block_embed(x, block_size)
        return p_q.predict(xb), p_k.predict(xb)
    if pooling == "token":
        xt = _dev_f32(x, p_q.w1.device)
        if xt.shape[0] % block_size:
            raise ContractError(f"sequence length {xt.shape[0]} not a multiple of block size")
        return (ops.block_embed(p_q.predict(xt), block_size),
                ops.block_embed(p_k.predict(xt), block_size))
    raise ContractError(f"unknown pooling mode {pooling!r}")


def pair_hidden1(p_q: Predictor, p_k: Predictor, x3: torch.Tensor):
    """Both predictors' first layers (predictor.py:83-85) on the shared block
    embedding as ONE bf16x3 GEMM: W1_q and W1_k stacked along N (cached while
    neither weight changes), both masks side by side.  Returns the split
    first-layer outputs (h1_q, h1_k)."""
    wq, wk = p_q._weights3()[0], p_k._weights3()[0]
    cache = getattr(p_q, "_stack1", None)  # (W1_q operand, W1_k operand, stacked)
    if cache is None or cache[0] is not wq or cache[1] is not wk:
        # the operands are rebuilt whenever the weights change; once stacked, each
        # predictor's own W1 operand becomes a view into the stack (no second copy)
        r = wq.shape[0]
        stack = torch.cat([wq, wk], dim=0)
        vq, vk = stack[:r], stack[r:]
        for p, v in ((p_q, vq), (p_k, vk)):
            key, ws = p._split
            p._split = (key, (v,) + tuple(ws[1:]))
        cache = p_q._stack1 = (vq, vk, stack)
    mask = torch.cat([p_q.mask1, p_k.mask1])
    return ops.gemm_split3_dual(x3, cache[2], wq.shape[0], relu=True, mask=mask)


def predicted_dense(p_q, p_k, x, block_size: int, pooling: str = "mean") -> torch.Tensor:
    """Dense eq·ekᵀ [nb, nb] fp32 (unclamped), every product on tcgen05 in
    fp32-faithful bf16x3 form.  mean pooling: block_embed → split → both first
    layers in one GEMM → 2×2 predictor GEMMs → Eq. 3 GEMM, no fp32 round trip
    between them."""
    if pooling == "mean":
        xb = block_embed(x, block_size)
        x3 = ops.split_bf16x3(xb, 0)
        h1q = h1k = None
        if p_q.w1.shape == p_k.w1.shape and p_q.w1.shape[1] % 32 == 0:
            h1q, h1k = pair_hidden1(p_q, p_k, x3)
        eq3 = p_q.predict3(x3, 0, h1q)
        ek3 = p_k.predict3(x3, 1, h1k)
    else:
        eq, ek = pair_block_outputs(p_q, p_k, x, block_size, pooling)
        eq3, ek3 = ops.split_bf16x3(eq, 0), ops.split_bf16x3(ek, 1)
    return ops.gemm_f32_exact(eq3, ek3)


def predicted_triangle(p_q, p_k, x, block_size: int, pooling: str = "mean") -> torch.Tensor:
    """Packed lower triangle of predicted scores, unclamped (predictor.py:176-186)."""
    return ops.pack_tril(predicted_dense(p_q, p_k, x, block_size, pooling), dtype=torch.float32)


def predicted_block_vector(p_q, p_k, x, block_size: int, pooling: str = "mean") -> torch.Tensor:
    """The attention hook's scorer (model.py:572-578): clamp ≥ 0, float64
    column sums over query blocks — on device."""
    return ops.colsum_clamped(predicted_dense(p_q, p_k, x, block_size, pooling))


def predict_scores(p_q: Predictor, p_k: Predictor, x_blocks, *, layer_id=None) -> BlockScoreMatrix:
    """Clamped Eq. 3 dots as a BlockScoreMatrix with block_size=1 (predictor.py:189-212)."""
    if p_q.d_pred != p_k.d_pred:
        raise ContractError(f"predictor output dims differ: {p_q.d_pred} vs {p_k.d_pred}")
    eq = p_q.predict(x_blocks)
    ek = p_k.predict(x_blocks)
    full = ops.gemm_f32_exact(ops.split_bf16x3(eq, 0), ops.split_bf16x3(ek, 1))
    return BlockScoreMatrix(full.shape[0], 1, ops.pack_tril(full, clamp=True),
                            layer_id=p_q.layer_id if layer_id is None else layer_id,
                            component=ATTENTION)


def retention_matched_threshold(pred_scores, exact_scores, exact_threshold: float) -> float:
    """Predicted-side threshold at the exact side's retention (predictor.py:257-276);
    the order statistic runs on the GPU (radix select)."""
    pred = _dev_f64(pred_scores)
    exact = _dev_f64(exact_scores)
    if pred.numel() == 0 or exact.numel() == 0:
        raise ContractError("cannot match retention on empty score sets")
    retained = float((exact >= exact_threshold).double().mean().item())
    return quantile_threshold(pred, retained)


def quantile_threshold(pooled: torch.Tensor, retained: float) -> float:
    """The recalibration rule of model.py:555-562 on device data."""
    out = torch.empty(1, dtype=torch.float64, device=pooled.device)
    retained = min(max(retained, 0.0), 1.0)
    if retained >= 1.0:
        return float("-inf")
    if retained <= 0.0:
        ops.quantile_lower(pooled, 1.0, out, plus_one=True)
    else:
        ops.quantile_lower(pooled, 1.0 - retained, out)
    return float(out.item())


def _dev_f64(a) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda" if not a.is_cuda else a.device, dtype=torch.float64).reshape(-1)
    return torch.as_tensor(np.asarray(a, dtype=np.float64).reshape(-1)).cuda()


def recall(predicted, exact) -> float:
    """predictor.py:279-290"""
    if predicted.n_blocks != exact.n_blocks or predicted.block_size != exact.block_size:
        raise ContractError("pattern grids differ")
    es = set(exact.retained_blocks)
    if not es:
        return 1.0
    return len(es.intersection(predicted.retained_blocks)) / len(es)


def precision(predicted, exact) -> float:
    """predictor.py:293-301"""
    if predicted.n_blocks != exact.n_blocks or predicted.block_size != exact.block_size:
        raise ContractError("pattern grids differ")
    ps = set(predicted.retained_blocks)
    if not ps:
        return 1.0
    return len(ps.intersection(exact.retained_blocks)) / len(ps)


# ---------------------------------------------------------------------------
# offline training (predictor.py:215-433)


@dataclass
class PredictorTrainingRecord:
    epoch: int
    train_loss: float
    recall: float
    param_count: int


@dataclass
class TeacherRecord:
    """One (batch, layer) example (predictor.py:307-315): the layer input x
    [s, h] and the exact block scores as a packed lower triangle."""

    layer_id: int
    x: torch.Tensor
    teacher_packed: torch.Tensor
    n_tokens: int
    block_size: int


def track_zero_frequency(p: Predictor, batch) -> tuple:
    """Forward pass that only bumps the zero counters (predictor.py:215-219)."""
    p.forward_train(_dev_f32(batch, p.w1.device), track=True)
    return p.zero_counts1, p.zero_counts2


def _prune_stage(counts: np.ndarray, mask: np.ndarray, target_active: int) -> None:
    """predictor.py:222-238 (host: a few hundred neurons): highest zero
    frequency first, ties prune the lower index first."""
    n = mask.shape[0]
    if target_active < 1:
        raise ContractError("target would prune all neurons of a matrix")
    to_prune = int(mask.sum()) - target_active
    if to_prune <= 0:
        return
    pruned = 0
    for i in np.lexsort((np.arange(n), -counts)):
        if pruned == to_prune:
            break
        if mask[i]:
            mask[i] = False
            pruned += 1


def elastic_prune(p: Predictor, target_fraction: float) -> Predictor:
    """Mask the highest-zero-frequency neurons down to the target fraction
    (predictor.py:241-254), both hidden stages, in place."""
    if p.observed == 0:
        raise ContractError("elastic_prune requires populated zero-frequency counters")
    if not (0.0 < target_fraction <= 1.0):
        raise ContractError(f"target fraction must lie in (0, 1], got {target_fraction}")
    masks = []
    for counts, mask in ((p.zero_counts1, p.mask1), (p.zero_counts2, p.mask2)):
        m = mask.cpu().numpy().astype(bool)
        _prune_stage(counts.cpu().numpy(), m, int(np.floor(target_fraction * m.shape[0] + 1e-9)))
        masks.append(m)
    p.set_masks(*masks)
    return p


def _teacher_label(rec: TeacherRecord, log_scale: bool) -> torch.Tensor:
    t = rec.teacher_packed
    t = t if isinstance(t, torch.Tensor) else torch.as_tensor(np.asarray(t))
    t = t.to(device="cuda" if not t.is_cuda else t.device, dtype=torch.float64).reshape(-1)
    return (torch.log1p(t) if log_scale else t).to(torch.float32).contiguous()


def _eval_recall(pairs: dict, data: list, thresholds, pooling: str) -> tuple:
    """Recall / precision of predicted vs exact patterns (predictor.py:318-363),
    the predicted-side threshold matched to the exact side's retention."""
    from . import sparsity  # noqa: WPS433

    if not data:
        return float("nan"), float("nan")
    by_layer: dict = {}
    for rec in data:
        p_q, p_k = pairs[rec.layer_id]
        pred_vec = predicted_block_vector(p_q, p_k, rec.x, rec.block_size, pooling)
        nb = n_blocks_for(rec.n_tokens, rec.block_size)
        exact_vec = sparsity.token_block_scores(
            BlockScoreMatrix(nb, rec.block_size, _dev_f64(rec.teacher_packed)))
        by_layer.setdefault(rec.layer_id, []).append((rec, pred_vec, exact_vec))
    recalls, precisions = [], []
    for layer_id, items in by_layer.items():
        exact_all = torch.cat([e for _, _, e in items])
        if thresholds is not None:
            exact_thr = thresholds.get(layer_id, ATTENTION)
        else:
            exact_thr = float(exact_all.mean().item())
        pred_thr = retention_matched_threshold(torch.cat([p for _, p, _ in items]), exact_all,
                                               exact_thr)
        for rec, pv, ev in items:
            ep = sparsity.eliminate(ev, exact_thr, layer_id=layer_id, block_size=rec.block_size,
                                    n_tokens=rec.n_tokens)
            pp = sparsity.eliminate(pv, pred_thr, layer_id=layer_id, block_size=rec.block_size,
                                    n_tokens=rec.n_tokens)
            recalls.append(recall(pp, ep))
            precisions.append(precision(pp, ep))
    return float(np.mean(recalls)), float(np.mean(precisions))


class _PairAdam:
    """The reference Adam (optim.py:37-53) over all predictor matrices: one
    global step counter, and only the matrices of the record's layer carry a
    gradient (the others are skipped, moments untouched)."""

    def __init__(self, pairs: dict, lr: float, betas=(0.9, 0.999), eps: float = 1e-8):
        self.lr, self.eps = lr, eps
        self.b1, self.b2 = betas
        self.t = 0
        self.state = {}
        for layer_id, (p_q, p_k) in pairs.items():
            for p in (p_q, p_k):
                for w in p.parameters():
                    self.state[id(w)] = (torch.zeros_like(w), torch.zeros_like(w))

    def step(self, items, guard_loss=None, guard_latch=None) -> None:
        """items: [(predictor, [g1, g2, g3])] holding this step's gradients.
        guard_loss / guard_latch: device-side skip of a non-finite record (the
        reference raises before stepping; here the host learns it at the
        epoch's read-back, and no NaN update has been applied by then)."""
        self.t += 1
        bc1 = 1.0 - self.b1 ** self.t
        bc2 = 1.0 - self.b2 ** self.t
        for p, grads in items:
            for w, g in zip(p.parameters(), grads):
                m, v = self.state[id(w)]
                ops.adam(w, g, m, v, lr=self.lr, b1=self.b1, b2=self.b2, eps=self.eps, wd=0.0,
                         bc1=bc1, bc2=bc2, guard_loss=guard_loss, guard_latch=guard_latch)
            p.touch()


def fit_predictors(pairs: dict, train_data: list, *, epochs: int, lr: float, val_data=None,
                   thresholds=None, pooling: str = "mean", log_scale: bool = True,
                   prune_target: float = 1.0, prune_every: int = 50, prune_step: float = 0.10,
                   eval_every: int = 20, lr_decay: bool = True) -> list:
    """Regress predicted block scores onto exact scores, log1p-scaled MSE over
    the packed triangle (predictor.py:366-433), on the GPU: per record the
    block means, both predictors, Eq. 3 and the whole backward are bf16x3
    tcgen05 GEMMs (fp32-faithful), the loss/gradient of the packed triangle is
    one kernel, Adam one launch per matrix.  Every `prune_every` epochs
    `prune_step` of the remaining hidden neurons with the highest zero
    frequency are masked until `prune_target` is reached.  Losses are
    reduced on device and read back once per epoch."""
    if not train_data:
        raise ContractError("no teacher records to train on")
    if pooling not in ("mean", "token"):
        raise ContractError(f"unknown pooling mode {pooling!r}")
    opt = _PairAdam(pairs, lr)
    labels = [_teacher_label(rec, log_scale) for rec in train_data]
    grads = {}
    for p_q, p_k in pairs.values():
        for p in (p_q, p_k):
            grads[id(p)] = [torch.empty_like(w) for w in p.parameters()]
    history = []
    last_recall = float("nan")
    dev = next(iter(pairs.values()))[0].w1.device
    losses = torch.empty(len(train_data), dtype=torch.float64, device=dev)
    diverged = torch.zeros(1, dtype=torch.int32, device=dev)  # latched by the guarded Adam
    for epoch in range(1, epochs + 1):
        if lr_decay:
            opt.lr = lr * (0.02 + 0.98 * 0.5 * (1.0 + math.cos(math.pi * (epoch - 1) / epochs)))
        for i, rec in enumerate(train_data):
            p_q, p_k = pairs[rec.layer_id]
            b = rec.block_size
            if pooling == "mean":  # pool tokens, then predict (predictor.py:165-167)
                xb = block_embed(rec.x, b)
                eq, saved_q = p_q.forward_train(xb, track=True)
                ek, saved_k = p_k.forward_train(xb, track=True)
            else:  # predict per token, then block means (predictor.py:168-172)
                xt = _dev_f32(rec.x, p_q.w1.device)
                if xt.shape[0] % b:
                    raise ContractError(f"sequence length {xt.shape[0]} not a multiple of "
                                        "block size")
                oq, saved_q = p_q.forward_train(xt, track=True)
                ok, saved_k = p_k.forward_train(xt, track=True)
                eq, ek = ops.block_embed(oq, b), ops.block_embed(ok, b)
            full = ops.gemm_split3(ops.split_bf16x3(eq, 0), ops.split_bf16x3(ek, 1),
                                   split_out=False, f32_out=True)[1]
            _, dfull = ops.tril_mse(full, labels[i], loss=losses[i:i + 1])
            # d eq = dFull·ek, d ek = dFullᵀ·eq
            d_eq = ops.gemm_split3(ops.split_bf16x3(dfull, 0), ops.split_bf16x3_t(ek, 1),
                                   split_out=False, f32_out=True)[1]
            d_ek = ops.gemm_split3(ops.split_bf16x3_t(dfull, 0), ops.split_bf16x3_t(eq, 1),
                                   split_out=False, f32_out=True)[1]
            if pooling == "token":
                d_eq, d_ek = ops.block_expand(d_eq, b), ops.block_expand(d_ek, b)
            p_q.backward_train(d_eq, saved_q, grads[id(p_q)])
            p_k.backward_train(d_ek, saved_k, grads[id(p_k)])
            opt.step([(p_q, grads[id(p_q)]), (p_k, grads[id(p_k)])],
                     guard_loss=losses[i:i + 1], guard_latch=diverged)
        host_losses = losses.cpu().numpy()
        bad = np.flatnonzero(~np.isfinite(host_losses))
        if bad.size:
            rec = train_data[int(bad[0])]
            raise ContractError(f"predictor training diverged at epoch {epoch} "
                                f"(layer {rec.layer_id}, loss {float(host_losses[bad[0]])})")
        if prune_target < 1.0 and epoch % prune_every == 0:
            for p_q, p_k in pairs.values():
                for p in (p_q, p_k):
                    active = float(p.mask1.sum().item()) / p.mask1.shape[0]
                    nxt = max(prune_target, active * (1.0 - prune_step))
                    if nxt < active:
                        elastic_prune(p, nxt)
        if val_data is not None and (epoch % eval_every == 0 or epoch == epochs):
            last_recall, _ = _eval_recall(pairs, val_data, thresholds, pooling)
        param_count = sum(p.active_param_count() for pq, pk in pairs.values() for p in (pq, pk))
        history.append(PredictorTrainingRecord(epoch, float(np.mean(host_losses)), last_recall,
                                               param_count))
    return history


__all__ = ["Predictor", "block_embed", "pair_block_outputs", "predicted_dense",
           "predicted_triangle", "predicted_block_vector", "predict_scores",
           "retention_matched_threshold", "quantile_threshold", "recall", "precision",
           "n_blocks_for", "tri_size", "PredictorTrainingRecord", "TeacherRecord",
           "track_zero_frequency", "elastic_prune", "fit_predictors"]
