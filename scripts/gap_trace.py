"""What the host does inside the GPU idle gaps of one step (torch.profiler, CPU+CUDA):
for the largest gaps, the CPU-side ops that ran between the GPU going idle and
the next kernel launch."""
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
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts, with_stack=True) as prof:
    step()
    torch.cuda.synchronize()
ev = prof.events()
gpu = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev
              if e.device_type == torch.autograd.DeviceType.CUDA), key=lambda t: t[0])
cpu = sorted(((e.time_range.start, e.time_range.end, e.name, e.stack) for e in ev
              if e.device_type == torch.autograd.DeviceType.CPU), key=lambda t: t[0])
gaps = []
end = gpu[0][1]
for s, e, n in gpu[1:]:
    if s - end > 30:
        gaps.append((s - end, end, s, n))
    end = max(end, e)
gaps.sort(reverse=True)
print(f"{len(gaps)} gaps > 30 us, total {sum(g[0] for g in gaps) / 1e3:.2f} ms")
for g, a, b, n in gaps[:6]:
    print(f"--- gap {g:.0f} us before {n[:50]}")
    inside = [c for c in cpu if c[0] >= a - 5 and c[0] <= b]
    for c in inside[:25]:
        st = ""
        if c[3]:
            fr = [f for f in c[3] if "paper_2501" in f]
            st = fr[0] if fr else ""
        print(f"   {c[0] - a:7.0f} {c[1] - c[0]:6.0f} us  {c[2][:40]:40s} {st[-70:]}")
