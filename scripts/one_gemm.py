import sys, torch
sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops
M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (8208, 4096, 12352)
a = torch.randn(M, K, device='cuda').bfloat16(); b = torch.randn(N, K, device='cuda').bfloat16()
out = ops.gemm_f32(a, b); torch.cuda.synchronize()
