"""Thin torch-tensor wrappers over the liblemo C ABI.

Each wrapper validates shapes/dtypes/devices on the host (raising the
reference's exception types), then calls the corresponding ``lemo_*`` entry
point on torch's current stream.  No wrapper has a non-CUDA path.
"""

from __future__ import annotations

import torch

from ._lib import call, ptr, stream_ptr
from .errors import ContractError, DimensionError

BF16 = torch.bfloat16
F32 = torch.float32


def _cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ContractError("liblemo operands must be CUDA tensors (no CPU fallback)")


def _contig(*ts):
    for t in ts:
        if t is not None and not t.is_contiguous():
            raise ContractError("liblemo operands must be contiguous")


def _dt(t, dtype, name):
    if t is not None and t.dtype != dtype:
        raise ContractError(f"{name} must be {dtype}, got {t.dtype}")


# ---------------------------------------------------------------------------
# GEMMs  (C = A · Bᵀ, B given as [N, K])


def gemm_bf16(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    _cuda(a, b)
    _dt(a, BF16, "a")
    _dt(b, BF16, "b")
    M, K = a.shape
    N, K2 = b.shape
    if K != K2:
        raise DimensionError(f"gemm inner extents differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    if out is None:
        out = torch.empty(M, N, dtype=BF16, device=a.device)
    call("lemo_gemm_bf16", ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(out), out.stride(0),
         M, N, K, stream_ptr())
    return out


def gemm_f32(a, b, out=None, *, side_u=None, side_s=None, side_strides=(0, 0), scale=1.0,
             accumulate=False):
    """out (+)= a·bᵀ + scale·side_u·S, S(j, col) = side_s[j*s_rs + col*s_cs]."""
    _cuda(a, b, out, side_u, side_s)
    _dt(a, BF16, "a")
    _dt(b, BF16, "b")
    M, K = a.shape
    N, K2 = b.shape
    if K != K2:
        raise DimensionError(f"gemm inner extents differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    if out is None:
        out = torch.empty(M, N, dtype=F32, device=a.device)
    R = 0 if side_u is None else side_u.shape[1]
    ldu = 0 if side_u is None else side_u.stride(0)
    call("lemo_gemm_f32", ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(out), out.stride(0), M, N,
         K, ptr(side_u), ldu, R, ptr(side_s), int(side_strides[0]), int(side_strides[1]),
         float(scale), int(bool(accumulate)), stream_ptr())
    return out


def gemm_scatter_add(a, b, resid, idx=None):
    """resid[idx] += a·bᵀ (in place)."""
    _cuda(a, b, resid, idx)
    _dt(resid, F32, "resid")
    M, K = a.shape
    N = b.shape[0]
    if idx is not None and idx.shape[0] != M:
        raise DimensionError("scatter index length must equal the GEMM row count")
    call("lemo_gemm_scatter_add", ptr(a), a.stride(0), ptr(b), b.stride(0), ptr(resid),
         resid.stride(0), ptr(idx), M, N, K, stream_ptr())
    return resid
