"""GEMM micro-benchmark at the step's shapes (CUDA events, warm)."""
import sys, torch
sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops
def bench(fn, it=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it
shapes = [("attn dX", 8208, 4096, 12352), ("mlp dX", 7400, 4096, 22016), ("o-proj", 8208, 4096, 4096),
          ("down", 7400, 4096, 11008), ("qkv-like", 8208, 12288, 4160), ("dgateup-like", 7400, 11008, 4096)]
for name, M, N, K in shapes:
    a = torch.randn(M, K, device='cuda').bfloat16()
    b = torch.randn(N, K, device='cuda').bfloat16()
    out = torch.empty(M, N, device='cuda')
    t = bench(lambda: ops.gemm_f32(a, b, out=out))
    print(f"{name:14s} M={M} N={N} K={K}: {t*1e3:.1f} us  {2*M*N*K/t/1e9:.0f} TFLOP/s")
