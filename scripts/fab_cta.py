"""Per-CTA timing of the backward kernels (debug build -DLEMO_FA_TRACE): fixed
per-CTA cost vs per-tile cost, SM busy fraction, gaps between CTAs on an SM."""
import ctypes, math, sys
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2501_09767_b200 import ops, _lib
n, H, d = int(sys.argv[1]) if len(sys.argv) > 1 else 8192, 32, 128
q, k, v = (torch.randn(n, H * d, device='cuda').bfloat16() for _ in range(3))
o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
do = torch.randn_like(o)
for _ in range(3):
    ops.flash_bwd(q, k, v, o, do, lse, head_dim=d, scale=1 / math.sqrt(d))
torch.cuda.synchronize()
buf = np.zeros((2, 8192, 6), dtype=np.uint64)
_lib.lib().lemo_fab_cta_get(ctypes.c_void_p(buf.ctypes.data))
nt = (n + 127) // 128
for kname, kk in (("dK/dV", 0), ("dQ", 1)):
    b = buf[kk, :nt * H].astype(np.int64)
    t0, t1, sm, units = b[:, 0], b[:, 1], b[:, 2], b[:, 3]
    dur = (t1 - t0) / 1e3  # us
    A = np.stack([np.ones_like(units), units], 1).astype(float)
    (a0, a1), *_ = np.linalg.lstsq(A, dur, rcond=None)
    span = (t1.max() - t0.min()) / 1e3
    busy = np.zeros(int(sm.max()) + 1)
    for s_, du in zip(sm, dur):
        busy[s_] += du
    gaps = []
    for s_ in np.unique(sm):
        idx = np.where(sm == s_)[0]
        o_ = np.argsort(t0[idx])
        st, en = t0[idx][o_], t1[idx][o_]
        gaps.extend(((st[1:] - en[:-1]) / 1e3).tolist())
    print(f"{kname}: {len(b)} CTAs, span {span:.1f} us, CTA time = {a0:.2f} us + {a1:.3f} us/tile; "
          f"SM busy {busy.mean() / span * 100:.1f} % (min {busy.min() / span * 100:.1f} %), "
          f"mean gap between CTAs {np.mean(gaps):.2f} us, last CTA ends {(t1.max() - np.sort(t1)[-148]) / 1e3:.1f} us after the 148th-last")
b = buf[0, :nt * H].astype(np.int64)
pro = (b[:, 4] - b[:, 0]) / 1e3; epi = (b[:, 1] - b[:, 5]) / 1e3
print(f"dK/dV per CTA: start -> first S seen {pro.mean():.2f} us, all MMAs done -> exit {epi.mean():.2f} us")
