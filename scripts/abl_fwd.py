"""Forward attention variants (LEMO_FA_POLY) — timing and error vs fp32 torch."""
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
    q, k, v = (torch.randn(n, H * d, device='cuda').bfloat16() for _ in range(3))
    fl = 2 * n * n * d * H
    t = bench(lambda: ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d)))
    o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
    # reference on 2 heads
    qh, kh, vh = (x[:, :2 * d].float().view(n, 2, d).transpose(0, 1) for x in (q, k, v))
    s = qh @ kh.transpose(1, 2) / math.sqrt(d)
    s = s.masked_fill(torch.triu(torch.ones(n, n, dtype=torch.bool, device='cuda'), 1), float('-inf'))
    lref = torch.logsumexp(s, -1)
    oref = (torch.softmax(s, -1) @ vh).transpose(0, 1).reshape(n, 2 * d)
    e = float((o[:, :2 * d].float() - oref).norm() / oref.norm())
    el = float((lse[:2] - lref).abs().max())
    print(f"poly={os.environ.get('LEMO_FA_POLY')} n={n}: {t:.3f} ms {fl / t / 1e9:.0f} TFLOP/s  o-rel {e:.2e} lse-maxabs {el:.2e}")
