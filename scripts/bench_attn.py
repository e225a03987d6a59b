"""Micro-benchmark of the attention kernels (CUDA events, warm)."""
import math, sys, torch
sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops

def bench(fn, it=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it

impls = sys.argv[1].split(",") if len(sys.argv) > 1 else ["tc"]
for n in (4096, 8192, 16384):
    H, d = 32, 128
    q, k, v = (torch.randn(n, H * d, device='cuda').bfloat16() for _ in range(3))
    fl = 2 * n * n * d * H  # causal fwd flops (QK^T + PV, half)
    o1, l1 = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d), impl="tc")
    for fi in ("tc",):
        t = bench(lambda: ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d), impl=fi))
        o2, l2 = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d), impl=fi)
        e = float((o2.float() - o1.float()).norm() / o1.float().norm())
        print(f"fwd n={n} {fi}: {t:.3f} ms  {fl / t / 1e9:.0f} TFLOP/s  rel-vs-tc {e:.2e} "
              f"lse-maxdiff {float((l2 - l1).abs().max()):.2e}")
    o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
    do = torch.randn_like(o)
    ref = None
    for impl in impls:
        t = bench(lambda: ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=1 / math.sqrt(d), impl=impl))
        g = ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=1 / math.sqrt(d), impl=impl)
        g2 = ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=1 / math.sqrt(d), impl=impl)
        det = all(torch.equal(a, b) for a, b in zip(g, g2))
        if ref is None:
            ref = [x.clone() for x in g]
        errs = [float((a - b).norm() / b.norm()) for a, b in zip(g, ref)]
        print(f"bwd n={n} {impl}: {t:.3f} ms  {2.5 * fl / t / 1e9:.0f} TFLOP/s (2.5x fwd flops) "
              f"deterministic={det} rel-vs-first dq/dk/dv={errs}")
