"""Accumulation precision of the tcgen05 bf16 GEMM (kind::f16, fp32 TMEM
accumulator) vs float64: bf16-exact inputs (so every product is exact) and
the bf16x3 split of fp32 inputs."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2501_09767_b200 import ops  # noqa: E402

torch.manual_seed(0)
for K in (16, 64, 256, 4096, 12288):
    M, N = 512, 512
    a = torch.randn(M, K, device="cuda")
    b = torch.randn(N, K, device="cuda")
    ab, bb = a.bfloat16(), b.bfloat16()
    ref = ab.double() @ bb.double().t()
    got = ops.gemm_f32(ab, bb)
    err = (got.double() - ref).abs()
    scale = (ab.double().abs() @ bb.double().abs().t())
    print(f"K={K:6d} bf16-exact inputs: max|err|/sum|ab| = {(err / scale).max().item():.3e}  "
          f"max rel = {(err / ref.abs().clamp_min(1e-3)).max().item():.3e}")
    # bf16x3 of fp32 inputs
    ref32 = a.double() @ b.double().t()
    a3, b3 = ops.split_bf16x3(a, 0), ops.split_bf16x3(b, 1)
    _, g3 = ops.gemm_split3(a3, b3, split_out=False, f32_out=True)
    e3 = (g3.double() - ref32).abs()
    s3 = a.double().abs() @ b.double().abs().t()
    tf = (a @ b.t()).double()
    et = (tf - ref32).abs()
    print(f"          bf16x3: max|err|/sum|ab| = {(e3 / s3).max().item():.3e}   "
          f"torch fp32 (cuBLAS): {(et / s3).max().item():.3e}")
