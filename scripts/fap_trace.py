"""Timeline of the pair forward kernel's heaviest cluster (debug build:
LEMO_EXTRA_NVCC_FLAGS=-DLEMO_FA_TRACE): per KV tile, softmax wait / compute
per CTA and the leader's PV issue."""
import ctypes
import math
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops, _lib  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H, d = 32, 128
q, k, v = (torch.randn(n, H * d, device='cuda').bfloat16() for _ in range(3))
for _ in range(3):
    ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
torch.cuda.synchronize()
buf = np.zeros((3, 4, 128), dtype=np.uint64)
_lib.lib().lemo_fap_trace_get(ctypes.c_void_p(buf.ctypes.data))
t = buf.astype(np.int64)
T = int((t[0, 3] > 0).sum())
sl = slice(2, T - 2)
for r in range(2):
    w0, s_rdy, p_done, p_ann = (t[r, e, :T] for e in range(4))
    print(f"CTA{r}: S wait {np.mean((s_rdy - w0)[sl]):.0f}, softmax {np.mean((p_done - s_rdy)[sl]):.0f}, "
          f"pv wait+announce {np.mean((p_ann - p_done)[sl]):.0f}, period {np.mean(np.diff(p_ann)[sl]):.0f} clk")
a0 = t[0, 3, :T]
seen0, seen, pv_iss, s_iss = t[2, 2, :T], t[2, 0, :T], t[2, 3, :T], t[2, 1, :T]
print(f"MMA (CTA0 clock): own P announced -> seen {np.mean((seen0 - a0)[sl]):.0f}, "
      f"-> CTA1's P and V seen {np.mean((seen - seen0)[sl]):.0f}, PV issue {np.mean((pv_iss - seen)[sl]):.0f}, "
      f"next S issue {np.mean((s_iss - pv_iss)[sl]):.0f}; CTA0 sees PV(j) done "
      f"{np.mean((t[0, 3, 1:T] - t[0, 2, 1:T])[sl]):.0f} after P(j+1) computed; "
      f"PV(j) issued -> P(j+1) computed {np.mean((t[0, 2, 1:T] - pv_iss[:T-1])[sl]):.0f}")
print("T =", T)
wb = np.zeros((2, 4, 2, 128), dtype=np.uint64)
_lib.lib().lemo_fap_warp_get(ctypes.c_void_p(wb.ctypes.data))
w = wb.astype(np.int64)
for r in range(2):
    base = w[r, 0, 1, :T]
    print(f"CTA{r} per-warp (vs warp 0): P computed "
          + " ".join(f"{np.mean((w[r, k, 0, :T] - w[r, 0, 0, :T])[sl]):+.0f}" for k in range(4))
          + " | announced " + " ".join(f"{np.mean((w[r, k, 1, :T] - base)[sl]):+.0f}" for k in range(4)))
print("CTA0 last announce -> MMA sees own P:",
      f"{np.mean((seen0 - w[0, :, 1, :T].max(axis=0))[sl]):.0f}")
sb = np.zeros((4, 4, 128), dtype=np.uint64)
_lib.lib().lemo_fap_sub_get(ctypes.c_void_p(sb.ctypes.data))
u = sb.astype(np.int64)
for wi in range(4):
    print(f"CTA0 warp {wi}: S ready->in regs {np.mean((u[wi,1,:T]-u[wi,0,:T])[sl]):.0f}, "
          f"compute {np.mean((u[wi,2,:T]-u[wi,1,:T])[sl]):.0f}, P store wait {np.mean((u[wi,3,:T]-u[wi,2,:T])[sl]):.0f}, "
          f"S ready vs warp0 {np.mean((u[wi,0,:T]-u[0,0,:T])[sl]):+.0f}")
