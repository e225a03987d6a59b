"""Forward-attention timeline of one CTA (debug build: LEMO_EXTRA_NVCC_FLAGS=-DLEMO_FA_TRACE)."""
import ctypes, math, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops, _lib
n, H, d = 8192, 32, 128
q, k, v = (torch.randn(n, H * d, device='cuda').bfloat16() for _ in range(3))
for _ in range(3):
    ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
torch.cuda.synchronize()
buf = np.zeros((2, 4, 64), dtype=np.uint64)
_lib.lib().lemo_fa_trace_get(ctypes.c_void_p(buf.ctypes.data))
t = buf.astype(np.int64)
for g in range(2):
    start, sfull, pdone = t[g, 0], t[g, 1], t[g, 2]
    m = (pdone > 0)
    E = (pdone - sfull)[m][2:-2]
    W = (sfull[1:] - pdone[:-1])[m[1:]][2:-2]
    print(f"WG{g}: softmax E mean {E.mean():.0f} clk (min {E.min()}, max {E.max()}), "
          f"wait for next S mean {W.mean():.0f} clk; period {np.diff(pdone[m])[2:-2].mean():.0f}")
