"""One flash backward at n=8192, 32 heads (for ncu captures of the dK/dV and dQ kernels)."""
import math, sys, torch
sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops
n, H, d = 8192, 32, 128
q, k, v = (torch.randn(n, H * d, device='cuda').bfloat16() for _ in range(3))
o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
do = torch.randn_like(o)
for _ in range(2):
    ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=1 / math.sqrt(d))
torch.cuda.synchronize()
