"""Exact attention block scores on the GPU (sparsity.py:173-219, Eq. 2).

Used by ExactPatternSource (profiling, teacher labels, exact-mode
fine-tuning).  The tcgen05 kernel (csrc/exact.cu) computes head-summed
positive pre-softmax scores tile by tile in TMEM and keeps only each b x b
tile's maximum; the column sums of the resulting lower triangle are the
token-block scores (sparsity.py:253-260).

q and k are [s, h] / [s, kv] bf16 (production precision) or (hi, lo) bf16
pairs of fp32 values (the fp32-faithful parity precision: the kernel issues
hi·hi + hi·lo + lo·hi per head).
"""

from __future__ import annotations

import torch

from . import ops
from ._lib import call, ptr, stream_ptr
from .errors import ContractError
from .sparsity import BlockScoreMatrix, n_blocks_for


def _parts(t):
    if isinstance(t, (tuple, list)):
        hi, lo = t
        return hi.contiguous(), lo.contiguous()
    return t.contiguous(), None


def exact_block_dense(q, k, block_size: int, *, n_heads: int,
                      n_valid: int | None = None) -> torch.Tensor:
    """Dense [nb, nb] fp32 tile maxima (upper triangle zero)."""
    qh, ql = _parts(q)
    kh, kl = _parts(k)
    if (ql is None) != (kl is None):
        raise ContractError("q and k must both be bf16 or both be (hi, lo) pairs")
    for t in (qh, ql, kh, kl):
        if t is not None and (not t.is_cuda or t.dtype != torch.bfloat16):
            raise ContractError("exact scorer operands must be CUDA bf16 tensors")
    if qh.shape[0] != kh.shape[0] or qh.shape[1] % kh.shape[1]:
        raise ContractError(f"q/k shapes incompatible: {tuple(qh.shape)} vs {tuple(kh.shape)}")
    s, h = qh.shape
    if block_size > s:
        raise ContractError(f"block size {block_size} exceeds sequence length {s}")
    n_valid = s if n_valid is None else n_valid
    nb = n_blocks_for(s, block_size)
    out = torch.zeros(nb, nb, dtype=torch.float32, device=qh.device)
    call("lemo_exact_block_scores", ptr(qh), ptr(kh), ptr(ql), ptr(kl), s, h, kh.shape[1],
         h // n_heads, block_size, n_valid, ptr(out), out.stride(0), stream_ptr())
    return out


def exact_block_vector(q, k, block_size: int, *, n_heads: int, n_valid=None) -> torch.Tensor:
    """Token-block scores (f64 column sums, ascending query block)."""
    return ops.colsum_clamped(exact_block_dense(q, k, block_size, n_heads=n_heads,
                                                n_valid=n_valid))


def packed_from_dense(dense: torch.Tensor, block_size: int, *, layer_id: int = 0,
                      component: str = "attention") -> BlockScoreMatrix:
    return BlockScoreMatrix(dense.shape[0], block_size, ops.pack_tril(dense), layer_id=layer_id,
                            component=component)


def exact_block_scores(q, k, block_size: int, *, n_heads: int, n_valid=None, layer_id: int = 0,
                       component: str = "attention") -> BlockScoreMatrix:
    """Packed-triangle form (the reference's return type) of [s, h] operands."""
    dense = exact_block_dense(q, k, block_size, n_heads=n_heads, n_valid=n_valid)
    return packed_from_dense(dense, block_size, layer_id=layer_id, component=component)
