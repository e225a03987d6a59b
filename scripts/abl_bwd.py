"""Backward attention variants (LEMO_FAB_POLY): timing and error vs fp32 torch (2 heads)."""
import math, os, sys, torch
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
H, d = 32, 128
for n in (8192, 16384):
    g = torch.Generator(device='cuda').manual_seed(0)
    q, k, v = (torch.randn(n, H * d, device='cuda', generator=g).bfloat16() for _ in range(3))
    o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
    do = torch.randn(n, H * d, device='cuda', generator=g).bfloat16()
    fl = 2.5 * 2 * n * n * d * H
    t = bench(lambda: ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=1 / math.sqrt(d)))
    dq, dk, dv = ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=1 / math.sqrt(d))
    # fp32 reference on 2 heads
    sl = slice(0, 2 * d)
    qr, kr, vr = (x[:, sl].float().view(n, 2, d).transpose(0, 1).requires_grad_(True) for x in (q, k, v))
    s = qr @ kr.transpose(1, 2) / math.sqrt(d)
    s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool, device='cuda'), 1), float('-inf'))
    out = torch.softmax(s, -1) @ vr
    out.backward(do[:, sl].float().view(n, 2, d).transpose(0, 1))
    errs = []
    for got, ref in ((dq, qr.grad), (dk, kr.grad), (dv, vr.grad)):
        ref = ref.transpose(0, 1).reshape(n, 2 * d)
        errs.append(float((got[:, sl] - ref).norm() / ref.norm()))
    print(f"poly={os.environ.get('LEMO_FAB_POLY')} n={n}: {t:.3f} ms {fl / t / 1e9:.0f} TF/s  rel dq/dk/dv {errs}")
    del s, out, qr, kr, vr
    torch.cuda.empty_cache()
