"""Scatter-add epilogue GEMM (o-proj / down-proj shapes) timing, CUDA events."""
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
s, h = 16384, 4096
for k, K in ((8208, 4096), (7045, 11008), (8192, 4096)):
    idx = torch.randperm(s, device='cuda')[:k].sort().values.int()
    a = torch.randn(k, K, device='cuda').bfloat16(); b = torch.randn(h, K, device='cuda').bfloat16()
    resid = torch.randn(s, h, device='cuda')
    t = bench(lambda: ops.gemm_scatter_add(a, b, resid, idx))
    print(f"scatter k={k} K={K}: {t*1e3:.1f} us {2*k*h*K/t/1e9:.0f} TF/s")
