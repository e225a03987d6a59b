"""Exact attention block scores on the GPU (sparsity.py:173-219, Eq. 2).

Used by ExactPatternSource (profiling, teacher labels, retain-all mode).
The fused kernel computes head-summed positive pre-softmax scores tile by
tile and keeps only each b x b tile's maximum; the column sums of the
resulting lower triangle are the token-block scores (sparsity.py:253-260).
"""

from __future__ import annotations

import torch

from . import ops
from ._lib import call, ptr, stream_ptr
from .errors import ContractError
from .sparsity import BlockScoreMatrix, n_blocks_for


def exact_block_dense(q: torch.Tensor, k: torch.Tensor, block_size: int, *, n_heads: int,
                      n_valid: int | None = None) -> torch.Tensor:
    """Dense [nb, nb] fp32 tile maxima (upper triangle zero).  q, k: [s, h] bf16."""
    if q.shape[0] != k.shape[0] or q.shape[1] % k.shape[1]:
        raise ContractError(f"q/k shapes incompatible: {tuple(q.shape)} vs {tuple(k.shape)}")
    s, h = q.shape
    if block_size > s:
        raise ContractError(f"block size {block_size} exceeds sequence length {s}")
    n_valid = s if n_valid is None else n_valid
    nb = n_blocks_for(s, block_size)
    out = torch.zeros(nb, nb, dtype=torch.float32, device=q.device)
    call("lemo_exact_block_scores", ptr(q.contiguous()), ptr(k.contiguous()), s, h, k.shape[1],
         h // n_heads, block_size, n_valid, ptr(out), out.stride(0), stream_ptr())
    return out


def exact_block_vector(q, k, block_size: int, *, n_heads: int, n_valid=None) -> torch.Tensor:
    """Token-block scores (f64 column sums, ascending query block)."""
    return ops.colsum_clamped(exact_block_dense(q, k, block_size, n_heads=n_heads,
                                                n_valid=n_valid))


def exact_block_scores(q, k, block_size: int, *, n_heads: int, n_valid=None, layer_id: int = 0,
                       component: str = "attention") -> BlockScoreMatrix:
    """Packed-triangle form (the reference's return type)."""
    dense = exact_block_dense(q, k, block_size, n_heads=n_heads, n_valid=n_valid)
    nb = dense.shape[0]
    r, c = torch.tril_indices(nb, nb, device=dense.device)
    return BlockScoreMatrix(nb, block_size, dense[r, c].double(), layer_id=layer_id,
                            component=component)
