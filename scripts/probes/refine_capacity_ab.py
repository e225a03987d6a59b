"""A/B in one process: the refined MLP scorer with its own row-count read-back
(exact) vs the capacity path (count read back with the selection), N* step,
alternating 5-step timings; also the overflow count of the capacity path."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_09767_b200 import model as M  # noqa: E402
from paper_2501_09767_b200.optim import Adam  # noqa: E402
from profile_step import setup  # noqa: E402

model, src, tokens = setup(16384, "lemo", "refined")
opt = Adam(model.lora_param, lr=1e-4)
batch = model.stage_tokens(tokens)
real_for_layer = src._refine_cap.for_layer
overflows = {"n": 0}
orig = M.refine_mlp_block_scores


def counting(*a, **k):
    if k.get("capacity") is None and a[0] is not None:
        overflows["n"] += 1
    return orig(*a, **k)


M.refine_mlp_block_scores = counting


def step():
    loss, _ = model.forward_step(batch, pattern_source=src, segments=8)
    loss.backward()
    opt.step()
    opt.zero_grad()


def timed(mode, n=5):
    src._refine_cap.for_layer = real_for_layer if mode == "capacity" else (lambda l: None)
    step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    overflows["n"] = 0
    a.record()
    for _ in range(n):
        step()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n, overflows["n"]


for _ in range(2):
    step()
res = {"exact": [], "capacity": []}
for rep in range(4):
    for mode in (("exact", "capacity") if rep % 2 == 0 else ("capacity", "exact")):
        ms, ex = timed(mode)
        res[mode].append(ms)
        print(f"{mode:9s} {ms:.2f} ms/step  exact-path refinements per 5 steps: {ex}", flush=True)
print({k: round(float(np.mean(v)), 2) for k, v in res.items()}, "caps", dict(src._refine_cap.cap))
