"""dQ backward timeline of the heaviest CTA (debug build: -DLEMO_FA_TRACE)."""
import ctypes, math, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops, _lib
n, H, d = 8192, 32, 128
q, k, v = (torch.randn(n, H * d, device='cuda').bfloat16() for _ in range(3))
o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
do = torch.randn_like(o)
for _ in range(3):
    ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=1 / math.sqrt(d))
torch.cuda.synchronize()
buf = np.zeros((2, 5, 128), dtype=np.uint64)
_lib.lib().lemo_fabq_trace_get(ctypes.c_void_p(buf.ctypes.data))
t = buf.astype(np.int64)[:, :, 4:60]
for g in range(2):
    a0, s_rdy, a_end, dp_rdy, ds_arr = t[g]
    print(f"dQ WG{g}: wait S {np.mean(s_rdy - a0):.0f} | phase A {np.mean(a_end - s_rdy):.0f} | "
          f"wait dP {np.mean(dp_rdy - a_end):.0f} | phase B {np.mean(ds_arr - dp_rdy):.0f} | "
          f"period {np.mean(np.diff(ds_arr)):.0f} clk")
