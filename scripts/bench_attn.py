"""Isolated timing of the tcgen05 attention kernels (CUDA events, warm),
both head dims, 32 query heads (or h = 4096 at d = 64: 64 heads).

    python scripts/bench_attn.py [n ...]
"""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_09767_b200 import ops  # noqa: E402


def bench(fn, it=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


sizes = [int(a) for a in sys.argv[1:]] or [4096, 8192, 16384]
for d in (128, 64):
    H = 4096 // d
    for n in sizes:
        q, k, v = (torch.randn(n, H * d, device="cuda").bfloat16() for _ in range(3))
        fl = 2 * n * n * d * H  # causal forward FLOPs (QKᵀ + PV, half the square)
        sc = 1 / math.sqrt(d)
        t = bench(lambda: ops.flash_fwd(q, k, v, head_dim=d, scale=sc))
        o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=sc)
        do = torch.randn_like(o)
        tb = bench(lambda: ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=sc))
        g1 = ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=sc)
        g2 = ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=sc)
        det = all(torch.equal(a, b) for a, b in zip(g1, g2))
        print(f"d={d} n={n}: fwd {t:.3f} ms {fl / t / 1e9:.0f} TFLOP/s | bwd {tb:.3f} ms "
              f"{2.5 * fl / tb / 1e9:.0f} TFLOP/s algorithmic (5·n²·h/2), "
              f"{3.5 * fl / tb / 1e9:.0f} executed | deterministic={det}", flush=True)
