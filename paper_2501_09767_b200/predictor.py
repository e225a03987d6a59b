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
        self._split = None

    def _weights3(self):
        """bf16x3 B-operands [N, 3K] (pattern 1) of W1ᵀ, W2ᵀ, W3ᵀ — rebuilt only
        when the weights change (predictors are frozen during fine-tuning)."""
        key = tuple(int(w._version) for w in (self.w1, self.w2, self.w3))
        if self._split is None or self._split[0] != key:
            ws = tuple(ops.split_bf16x3(w.t().contiguous(), 1) for w in (self.w1, self.w2, self.w3))
            self._split = (key, ws)
        return self._split[1]

    def hidden3(self, x3: torch.Tensor) -> torch.Tensor:
        """relu/mask hidden layers on a bf16x3 input; returns split h2 [M, 3 r2]."""
        w1, w2, _ = self._weights3()
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

    def predict3(self, x3: torch.Tensor, pattern: int) -> torch.Tensor:
        """Predictor output in split form (pattern 0: A-side, 1: B-side of Eq. 3)."""
        h2 = self.hidden3(x3)
        out, _ = ops.gemm_split3(h2, self._weights3()[2], pattern=pattern)
        return out

    forward = predict

    def state_arrays(self) -> dict:
        return {"w1": self.w1.cpu().numpy(), "w2": self.w2.cpu().numpy(),
                "w3": self.w3.cpu().numpy(), "mask1": self.mask1.cpu().numpy().astype(bool),
                "mask2": self.mask2.cpu().numpy().astype(bool)}

    def load_state_arrays(self, state: dict) -> None:
        for name in ("w1", "w2", "w3"):
            t = getattr(self, name)
            if tuple(t.shape) != tuple(state[name].shape):
                raise ContractError(f"predictor {name} shape mismatch on load")
            t.copy_(torch.as_tensor(np.asarray(state[name], dtype=np.float32)))
        if "mask1" in state:
            self.set_masks(state["mask1"], state["mask2"])


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


def predicted_dense(p_q, p_k, x, block_size: int, pooling: str = "mean") -> torch.Tensor:
    """Dense eq·ekᵀ [nb, nb] fp32 (unclamped), every product on tcgen05 in
    fp32-faithful bf16x3 form.  mean pooling: block_embed → split → 2×3
    predictor GEMMs → Eq. 3 GEMM, no fp32 round trip between them."""
    if pooling == "mean":
        xb = block_embed(x, block_size)
        x3 = ops.split_bf16x3(xb, 0)
        eq3 = p_q.predict3(x3, 0)
        ek3 = p_k.predict3(x3, 1)
    else:
        eq, ek = pair_block_outputs(p_q, p_k, x, block_size, pooling)
        eq3, ek3 = ops.split_bf16x3(eq, 0), ops.split_bf16x3(ek, 1)
    return ops.gemm_f32(eq3, ek3)


def predicted_triangle(p_q, p_k, x, block_size: int, pooling: str = "mean") -> torch.Tensor:
    """Packed lower triangle of predicted scores, unclamped (predictor.py:176-186)."""
    full = predicted_dense(p_q, p_k, x, block_size, pooling)
    nb = full.shape[0]
    r, c = torch.tril_indices(nb, nb, device=full.device)
    return full[r, c]


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
    full = ops.gemm_f32(ops.split_bf16x3(eq, 0), ops.split_bf16x3(ek, 1))
    nb = full.shape[0]
    r, c = torch.tril_indices(nb, nb, device=full.device)
    packed = torch.clamp_min(full[r, c], 0.0)
    return BlockScoreMatrix(nb, 1, packed, layer_id=p_q.layer_id if layer_id is None else layer_id,
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


__all__ = ["Predictor", "block_embed", "pair_block_outputs", "predicted_dense",
           "predicted_triangle", "predicted_block_vector", "predict_scores",
           "retention_matched_threshold", "quantile_threshold", "recall", "precision",
           "n_blocks_for", "tri_size"]
