import sys, torch
sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops
torch.manual_seed(0)
for M, N, K in [(1024, 4096, 512), (8208, 4096, 1024), (300, 1024, 256)]:
    a = torch.randn(M, K, device='cuda').bfloat16(); b = torch.randn(N, K, device='cuda').bfloat16()
    out = ops.gemm_f32(a, b)
    ref = a.float() @ b.float().t()
    err = float((out - ref).abs().max() / ref.abs().max())
    # which half is wrong?
    e_rows = (out - ref).abs().amax(1) / ref.abs().max()
    e_cols = (out - ref).abs().amax(0) / ref.abs().max()
    print(M, N, K, "max rel err", err, "bad rows", int((e_rows > 1e-2).sum()), "bad cols", int((e_cols > 1e-2).sum()))
