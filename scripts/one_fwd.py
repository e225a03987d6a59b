import math, sys, torch
sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops
n, H, d = 8192, 32, 128
q, k, v = (torch.randn(n, H * d, device='cuda').bfloat16() for _ in range(3))
for _ in range(2):
    ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
torch.cuda.synchronize()
