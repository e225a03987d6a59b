"""dK/dV backward timeline of the heaviest CTA (debug build: -DLEMO_FA_TRACE)."""
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
buf = np.zeros((3, 8, 128), dtype=np.uint64)
_lib.lib().lemo_fab_trace_get(ctypes.c_void_p(buf.ctypes.data))
t = buf.astype(np.int64)[:, :, 4:60]
for g in range(2):
    a0, s_rdy, p_arr, dp_rdy, ds_arr = t[g][:5]
    print(f"WG{g}: wait S {np.mean(s_rdy - a0):.0f} | phase A {np.mean(p_arr - s_rdy):.0f} | "
          f"wait dP {np.mean(dp_rdy - p_arr):.0f} | phase B {np.mean(ds_arr - dp_rdy):.0f} | "
          f"period {np.mean(np.diff(ds_arr)):.0f} clk")
# MMA warp: [0] p_full seen, [1] dV+S(t+1) issued, [2] ds_full seen, [3] dK+dP(t+1) issued,
# [6] q_full(t) seen, [7] o_full(t) seen; one row per event, three consecutive tiles
m = t[2]
ev = {"MMA p_full seen": m[0], "MMA dV,S(t+1) issued": m[1], "MMA ds_full seen": m[2],
      "MMA dK,dP(t+1) issued": m[3], "MMA q_full(t+1) seen": np.roll(m[6], -1),
      "MMA o_full(t+1) seen": np.roll(m[7], -1),
      "EW0 S(t) seen": t[0][1], "EW0 p arrive": t[0][2], "EW0 dP(t) seen": t[0][3],
      "EW0 ds arrive": t[0][4]}
base = m[0][10]
for k, v in sorted(ev.items(), key=lambda kv: kv[1][10]):
    print(f"  {k:24s} " + " ".join(f"{int(x - base):6d}" for x in v[10:13]))
