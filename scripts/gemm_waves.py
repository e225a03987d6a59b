"""Wave quantization of the CTA-pair GEMM: TFLOP/s vs M at N=4096 (CUDA events, warm)."""
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
N, K = 4096, 12352
for M in (7400, 7424, 8192, 8208, 8448, 9472, 9728, 18944):
    a = torch.randn(M, K, device='cuda').bfloat16()
    b = torch.randn(N, K, device='cuda').bfloat16()
    out = torch.empty(M, N, device='cuda')
    t = bench(lambda: ops.gemm_f32(a, b, out=out))
    tiles = -(-M // 256) * (N // 256)
    print(f"M={M:6d} tiles={tiles:4d} waves={tiles/74:5.2f}: {t*1e3:7.1f} us  {2*M*N*K/t/1e9:6.0f} TFLOP/s")
