"""GPU timeline of one training step (torch.profiler / CUPTI): busy fraction,
idle gaps and what precedes them — host overhead vs kernel time."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from profile_step import setup  # noqa: E402
from paper_2501_09767_b200.optim import Adam  # noqa: E402

model, src, tokens = setup(16384, "lemo", "refined")
opt = Adam(model.lora_param, lr=1e-4)
batch = model.stage_tokens(tokens)


def step():
    loss, _ = model.forward_step(batch, pattern_source=src, segments=8)
    loss.backward()
    opt.step()
    opt.zero_grad()


for _ in range(2):
    step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    step()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ks = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda t: t[0])
span = ks[-1][1] - ks[0][0]
busy = 0
gaps = []
cur_end = ks[0][0]
prev = ""
for s, e, n in ks:
    if s > cur_end:
        gaps.append((s - cur_end, prev[:60]))
    busy += max(0, e - max(s, cur_end))
    if e > cur_end:
        cur_end = e
        prev = n
gaps.sort(reverse=True)
tot_gap = sum(g for g, _ in gaps)
print(f"kernels {len(ks)}  span {span / 1e3:.2f} ms  busy {busy / 1e3:.2f} ms "
      f"({busy / span * 100:.1f} %)  gaps {len(gaps)} total {tot_gap / 1e3:.2f} ms")
big = [g for g in gaps if g[0] > 20]
print(f"gaps > 20 us: {len(big)} totalling {sum(g for g, _ in big) / 1e3:.2f} ms")
for g, n in gaps[:15]:
    print(f"  {g:8.1f} us after {n}")
