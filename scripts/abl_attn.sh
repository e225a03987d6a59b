python - <<'PY'
import math, sys, os, torch
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
n, H, d = 8192, 32, 128
q, k, v = (torch.randn(n, H * d, device='cuda').bfloat16() for _ in range(3))
o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
do = torch.randn_like(o)
t = bench(lambda: ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=1 / math.sqrt(d)))
print(os.environ.get("LEMO_FAB_MODE"), f"{t:.3f} ms")
PY
