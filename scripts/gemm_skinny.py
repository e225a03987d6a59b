"""Skinny GEMM timing (rank-r LoRA products, predictor layers), CUDA events."""
import sys, torch
sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops
def bench(fn, it=50):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
for M, N, K in ((8208, 32, 12352), (8208, 32, 4096), (16384, 32, 4096), (1024, 1024, 12288)):
    a = torch.randn(M, K, device='cuda').bfloat16(); b = torch.randn(N, K, device='cuda').bfloat16()
    out = torch.empty(M, N, device='cuda')
    t = bench(lambda: ops.gemm_f32(a, b, out=out))
    print(f"M={M} N={N} K={K}: {t*1e3:.1f} us {2*M*N*K/t/1e9:.0f} TF/s")
