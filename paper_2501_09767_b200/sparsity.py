"""Block-wise token elimination: types and GPU selection.

Mirrors the public API of the reference module ``sparsetune.sparsity``
(/root/reference/pkg/src/sparsetune/sparsity.py).  Score vectors live on the
GPU as float64 tensors; `eliminate` runs the liblemo select kernel (>=
threshold, ties retained, forced blocks, block→token compaction) and returns
a `SparsityPattern` whose host view (retained_blocks / token_indices) is
materialised lazily from the device result.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Mapping, Sequence

import numpy as np
import torch

from . import ops
from .errors import ContractError

ATTENTION = "attention"
MLP = "mlp"
COMPONENTS = (ATTENTION, MLP)

NEG_INF = float("-inf")


def n_blocks_for(n_tokens: int, block_size: int) -> int:
    """sparsity.py:27-28"""
    return -(-n_tokens // block_size)


def tri_size(n_blocks: int) -> int:
    """sparsity.py:31-32"""
    return n_blocks * (n_blocks + 1) // 2


def tri_index(m: int, n: int) -> int:
    """sparsity.py:35-37: packed index of (query block m, key block n), n <= m."""
    return m * (m + 1) // 2 + n


class BlockScoreMatrix:
    """Packed lower-triangular block scores, float64, nonnegative
    (sparsity.py:40-69).  `scores` may be a CUDA tensor or array-like."""

    def __init__(self, n_blocks: int, block_size: int, scores, layer_id: int = 0,
                 component: str = ATTENTION):
        self.n_blocks = n_blocks
        self.block_size = block_size
        self.layer_id = layer_id
        self.component = component
        if isinstance(scores, torch.Tensor):
            sc = scores.to(torch.float64)
        else:
            sc = torch.as_tensor(np.asarray(scores, dtype=np.float64))
        if tuple(sc.shape) != (tri_size(n_blocks),):
            raise ContractError(f"packed triangle length {tuple(sc.shape)} does not match "
                                f"{n_blocks} blocks")
        if sc.numel() and bool((sc.min() < 0).item()):
            raise ContractError("block scores must be nonnegative")
        self.scores = sc

    def get(self, m: int, n: int) -> float:
        if n > m:
            raise ContractError(f"block ({m},{n}) is above the causal diagonal")
        return float(self.scores[tri_index(m, n)])

    def as_dense(self) -> torch.Tensor:
        nb = self.n_blocks
        r, c = torch.tril_indices(nb, nb, device=self.scores.device)
        dense = torch.zeros(nb, nb, dtype=torch.float64, device=self.scores.device)
        dense[r, c] = self.scores
        return dense


class SparsityPattern:
    """Retained token blocks for one (layer, component) — sparsity.py:72-117.

    Constructed either from host block ids (reference signature) or from the
    device result of the select kernel (`_from_device`); in the latter case
    the retained block list is copied to the host only when asked for.
    """

    __slots__ = ("layer_id", "component", "block_size", "n_tokens", "_blocks", "_dev_blocks",
                 "_dev_tokens", "_n_blocks_kept", "_k")

    def __init__(self, layer_id: int, component: str, retained_blocks: Sequence[int],
                 block_size: int, n_tokens: int):
        blocks = tuple(int(b) for b in retained_blocks)
        if list(blocks) != sorted(set(blocks)):
            raise ContractError("retained blocks must be sorted and unique")
        nb = n_blocks_for(n_tokens, block_size)
        if blocks and (blocks[0] < 0 or blocks[-1] >= nb):
            raise ContractError(f"retained blocks out of range [0, {nb})")
        self.layer_id = layer_id
        self.component = component
        self.block_size = block_size
        self.n_tokens = n_tokens
        self._blocks = blocks
        self._dev_blocks = None
        self._dev_tokens = None
        self._n_blocks_kept = len(blocks)
        self._k = None

    @classmethod
    def _from_device(cls, layer_id, component, block_size, n_tokens, dev_blocks, dev_tokens,
                     n_blocks_kept: int, k: int) -> "SparsityPattern":
        self = cls.__new__(cls)
        self.layer_id = layer_id
        self.component = component
        self.block_size = block_size
        self.n_tokens = n_tokens
        self._blocks = None
        self._dev_blocks = dev_blocks[:n_blocks_kept]
        self._dev_tokens = dev_tokens[:k]
        self._n_blocks_kept = n_blocks_kept
        self._k = k
        return self

    @property
    def retained_blocks(self) -> tuple[int, ...]:
        if self._blocks is None:
            self._blocks = tuple(self._dev_blocks.cpu().tolist())
        return self._blocks

    @property
    def n_blocks(self) -> int:
        return n_blocks_for(self.n_tokens, self.block_size)

    @property
    def k(self) -> int:
        """Number of retained tokens."""
        if self._k is None:
            b, n = self.block_size, self.n_tokens
            self._k = sum(min((x + 1) * b, n) - x * b for x in self.retained_blocks)
        return self._k

    @property
    def token_indices(self) -> np.ndarray:
        """int64 ascending retained token ids (host view), sparsity.py:95-104."""
        if self._dev_tokens is not None:
            return self._dev_tokens.cpu().numpy().astype(np.int64)
        b = self.block_size
        chunks = [np.arange(n * b, min((n + 1) * b, self.n_tokens)) for n in self.retained_blocks]
        if not chunks:
            return np.empty(0, dtype=np.int64)
        return np.concatenate(chunks).astype(np.int64)

    def device_token_indices(self, device) -> torch.Tensor:
        """int32 retained token ids on the device (no host round trip when the
        pattern came from the select kernel)."""
        if self._dev_tokens is None:
            self._dev_tokens = torch.as_tensor(self.token_indices.astype(np.int32), device=device)
        return self._dev_tokens

    @property
    def retained_fraction(self) -> float:
        return self.k / self.n_tokens

    def __eq__(self, other):
        if not isinstance(other, SparsityPattern):
            return NotImplemented
        return (self.layer_id, self.component, self.retained_blocks, self.block_size,
                self.n_tokens) == (other.layer_id, other.component, other.retained_blocks,
                                   other.block_size, other.n_tokens)

    def __repr__(self):
        return (f"SparsityPattern(layer={self.layer_id}, {self.component}, "
                f"blocks={self._n_blocks_kept}/{self.n_blocks}, b={self.block_size})")

    @staticmethod
    def full(n_tokens: int, block_size: int, layer_id: int = 0,
             component: str = ATTENTION) -> "SparsityPattern":
        nb = n_blocks_for(n_tokens, block_size)
        return SparsityPattern(layer_id, component, tuple(range(nb)), block_size, n_tokens)

    @staticmethod
    def empty(n_tokens: int, block_size: int, layer_id: int = 0,
              component: str = ATTENTION) -> "SparsityPattern":
        return SparsityPattern(layer_id, component, (), block_size, n_tokens)


@dataclass
class ThresholdSet:
    """One threshold per (layer, component) — sparsity.py:120-152 (host)."""

    values: dict = field(default_factory=dict)
    eps: float | None = None
    eta: float | None = None
    config_hash: str = ""

    def get(self, layer_id: int, component: str) -> float:
        return self.values[(layer_id, component)]

    def set(self, layer_id: int, component: str, value: float) -> None:
        self.values[(layer_id, component)] = value

    def copy(self) -> "ThresholdSet":
        return ThresholdSet(dict(self.values), self.eps, self.eta, self.config_hash)

    def to_dict(self) -> dict:
        return {
            "values": {f"{l}:{c}": v for (l, c), v in sorted(self.values.items())},
            "eps": self.eps,
            "eta": self.eta,
            "config_hash": self.config_hash,
        }

    @staticmethod
    def from_dict(d: dict) -> "ThresholdSet":
        values = {}
        for key, v in d["values"].items():
            layer, comp = key.split(":")
            values[(int(layer), comp)] = float(v)
        return ThresholdSet(values, d.get("eps"), d.get("eta"), d.get("config_hash", ""))


# ---------------------------------------------------------------------------
# selection on the GPU


class SelectWorkspace:
    """Buffers of one select call.  The retained block / token lists are fresh
    per call (the returned pattern keeps views of them); the scratch mask,
    counters and the pinned read-back slot are cached per (device, nb) -- they
    are consumed before select_device returns (it synchronises)."""

    _scratch: dict = {}

    def __init__(self, nb: int, n_tokens: int, block_size: int, device):
        self.nb = nb
        self.blocks = torch.empty(max(nb, 1), dtype=torch.int32, device=device)
        self.tokens = torch.empty(max(nb * block_size, 1), dtype=torch.int32, device=device)
        key = (str(device), nb)
        sc = SelectWorkspace._scratch.get(key)
        if sc is None:
            host_i = torch.empty(4, dtype=torch.int32, pin_memory=True)
            host_f = torch.empty(1, dtype=torch.float64, pin_memory=True)
            host_x = torch.empty(4, dtype=torch.int32, pin_memory=True)  # caller's extras
            sc = (torch.empty(max(nb, 1), dtype=torch.uint8, device=device),
                  torch.empty(4, dtype=torch.int32, device=device),
                  torch.empty(1, dtype=torch.float64, device=device), host_i, host_f,
                  host_i.numpy(), host_f.numpy(), host_x, host_x.numpy())
            SelectWorkspace._scratch[key] = sc
        (self.mask, self.counts, self.thr, self.host_i, self.host_f, self.host_i_np,
         self.host_f_np, self.host_x, self.host_x_np) = sc


def _force_mask(force_blocks, nb, device):
    force = [int(b) for b in force_blocks]
    if not force:
        return None
    if min(force) < 0 or max(force) >= nb:
        raise ContractError(f"retained blocks out of range [0, {nb})")
    m = torch.zeros(nb, dtype=torch.uint8)
    m[force] = 1
    return m.to(device, non_blocking=True)


def select_device(vec: torch.Tensor, threshold: float | None = None, *, thr_dev=None,
                  layer_id: int = 0, component: str = ATTENTION, block_size: int,
                  n_tokens: int, force_blocks: Sequence[int] = (), extra=None):
    """eliminate() on device scores; returns (pattern, threshold used).

    One host synchronisation: the retained count k (needed to size the
    compact activation buffers) and the threshold are read back together.
    `extra` (device int32, <= 4 values, e.g. the refinement's [count,
    overflow]) rides on the same read-back; then (pattern, threshold, extras)
    is returned.
    """
    nb = vec.shape[0]
    if nb != n_blocks_for(n_tokens, block_size):
        raise ContractError(f"{nb} scores for {n_blocks_for(n_tokens, block_size)} blocks")
    dev = vec.device
    ws = SelectWorkspace(nb, n_tokens, block_size, dev)
    force = _force_mask(force_blocks, nb, dev)
    thr = 0.0 if threshold is None else float(threshold)
    ops.select(vec, b=block_size, n_tokens=n_tokens, thr=thr, thr_dev=thr_dev, force=force,
               mask=ws.mask, blocks=ws.blocks, tokens=ws.tokens, counts=ws.counts, thr_out=ws.thr)
    ws.host_i.copy_(ws.counts, non_blocking=True)
    ws.host_f.copy_(ws.thr, non_blocking=True)
    if extra is not None:
        ws.host_x[:extra.numel()].copy_(extra, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    hi = ws.host_i_np  # numpy views of the pinned slots: no per-element tensor dispatch
    k, nkept, bad, used = int(hi[0]), int(hi[1]), int(hi[2]), float(ws.host_f_np[0])
    if bad:
        raise ContractError("block scores must be finite")
    pat = SparsityPattern._from_device(layer_id, component, block_size, n_tokens, ws.blocks,
                                       ws.tokens, nkept, k)
    if extra is not None:
        return pat, used, [int(v) for v in ws.host_x_np[:extra.numel()]]
    return pat, used


def _as_device_vec(block_scores, device=None) -> torch.Tensor:
    if isinstance(block_scores, torch.Tensor) and block_scores.is_cuda:
        return block_scores.to(torch.float64)
    dev = device or torch.device("cuda")
    return torch.as_tensor(np.asarray(block_scores, dtype=np.float64)).to(dev)


def eliminate(block_scores, threshold: float, *, layer_id: int = 0, component: str = ATTENTION,
              block_size: int, n_tokens: int, force_blocks: Sequence[int] = ()) -> SparsityPattern:
    """Retain every block whose score meets the threshold — sparsity.py:263-281,
    computed by the liblemo select kernel (ties retained, -inf keeps all,
    non-finite scores raise ContractError)."""
    vec = _as_device_vec(block_scores)
    return select_device(vec, threshold, layer_id=layer_id, component=component,
                         block_size=block_size, n_tokens=n_tokens, force_blocks=force_blocks)[0]


def token_block_scores(matrix: BlockScoreMatrix) -> torch.Tensor:
    """Column sums of the packed triangle, f64 in ascending m (sparsity.py:253-260),
    on the GPU (lemo_colsum_packed, one warp per column)."""
    packed = matrix.scores
    packed = (packed if packed.is_cuda else packed.to("cuda")).to(torch.float64).contiguous()
    return ops.colsum_packed(packed, matrix.n_blocks)


def _as_heads(a) -> torch.Tensor:
    """sparsity.py:159-166: [s, d] -> [1, s, d]; anything but 2-D/3-D raises."""
    t = a if isinstance(a, torch.Tensor) else torch.as_tensor(np.asarray(a))
    if t.dim() == 2:
        t = t[None]
    if t.dim() != 3:
        raise ContractError(f"expected [heads, s, d] scores input, got shape {tuple(t.shape)}")
    return t


def exact_block_scores(q, k, block_size: int, *, n_valid: int | None = None, layer_id: int = 0,
                       component: str = ATTENTION) -> BlockScoreMatrix:
    """sparsity.py:173-219 with the reference signature: q, k [H, s, d] (or
    [s, d]).  Runs the tcgen05 exact scorer (csrc/exact.cu); float inputs are
    scored in the fp32-faithful bf16x3 mode, bf16 CUDA inputs in bf16.  Head
    dims below 64/128 are zero-padded (q·k is unchanged)."""
    from . import exact  # kernel module (imports this one)

    qt, kt = _as_heads(q), _as_heads(k)
    if tuple(qt.shape) != tuple(kt.shape):
        raise ContractError(f"q/k shapes differ: {tuple(qt.shape)} vs {tuple(kt.shape)}")
    H, s, d = qt.shape
    if block_size > s:
        raise ContractError(f"block size {block_size} exceeds sequence length {s}")
    if d > 128:
        raise ContractError(f"head dim {d} > 128 is not supported by the exact scorer")
    dp = 64 if d <= 64 else 128
    dev = qt.device if qt.is_cuda else torch.device("cuda")
    bf16 = qt.dtype == torch.bfloat16 and qt.is_cuda

    def rows(t):  # [H, s, d] -> [s, H*dp], heads side by side
        out = torch.zeros(s, H, dp, dtype=torch.bfloat16 if bf16 else torch.float32, device=dev)
        out[:, :, :d] = t.to(device=dev, dtype=out.dtype).permute(1, 0, 2)
        return out.reshape(s, H * dp)

    qr, kr = rows(qt), rows(kt)
    if not bf16:
        qr, kr = ops.split_hilo(qr), ops.split_hilo(kr)
    return exact.exact_block_scores(qr, kr, block_size, n_heads=H, n_valid=n_valid,
                                    layer_id=layer_id, component=component)


def mlp_block_scores(token_scores, block_size: int, *, n_valid: int | None = None) -> np.ndarray:
    """Block score = max token score in the block (sparsity.py:293-305); host
    helper for already-reduced token scores (the fused GPU path is
    model.mlp_block_score_vector)."""
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


def init_thresholds(profile: Mapping, config_hash: str = "") -> ThresholdSet:
    """Algorithm 1 step 1: threshold = pooled mean of observed block scores
    (sparsity.py:360-376)."""
    if not profile:
        raise ContractError("empty profile")
    ts = ThresholdSet(config_hash=config_hash)
    for key, batches in profile.items():
        if not batches:
            raise ContractError(f"no profiled batches for {key}")
        pooled = []
        for item in batches:
            if isinstance(item, BlockScoreMatrix):
                item = token_block_scores(item)
            if isinstance(item, torch.Tensor):
                item = item.double().cpu().numpy()
            pooled.append(np.asarray(item, dtype=np.float64).reshape(-1))
        allv = np.concatenate(pooled)
        if allv.size == 0:
            raise ContractError(f"no scores observed for {key}")
        ts.values[key] = float(allv.mean())
    return ts


def tune_thresholds(acc_fn, thresholds: ThresholdSet, *, eps: float | None = None,
                    eta: float | None = None, rounds: int = 1) -> ThresholdSet:
    """Algorithm 1 step 2 (sparsity.py:379-417): per-threshold central finite
    difference of the accuracy proxy, T <- T + eta·G, keys in sorted order.
    eps defaults to 0.05·|T| + 1e-3; without eta the step is capped at 10 %
    of |T|.  `acc_fn(ThresholdSet) -> float` is where the GPU works (e.g.
    `pipeline.eval_accuracy`: eval forwards through the sparse path)."""
    tuned = thresholds.copy()
    tuned.eps = eps
    tuned.eta = eta
    for _ in range(max(rounds, 0)):
        for key in sorted(tuned.values):
            t = tuned.values[key]
            e = eps if eps is not None else 0.05 * abs(t) + 1e-3
            probe = tuned.copy()
            probe.values[key] = t + e
            acc_plus = float(acc_fn(probe))
            probe.values[key] = t - e
            acc_minus = float(acc_fn(probe))
            if not (np.isfinite(acc_plus) and np.isfinite(acc_minus)):
                raise ContractError(f"non-finite accuracy while tuning {key}: "
                                    f"acc(T+eps)={acc_plus}, acc(T-eps)={acc_minus}")
            grad = (acc_plus - acc_minus) / (2.0 * e)
            if eta is not None:
                step = eta * grad
            else:
                step = 0.1 * (abs(t) + 1e-3) / (abs(grad) + 1e-12) * grad
            tuned.values[key] = t + step
    return tuned
