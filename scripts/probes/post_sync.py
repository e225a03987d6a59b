"""Host latency from each count read-back (the select kernel's sync) to the
next liblemo launch in the N* step: the GPU idles for that long."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_09767_b200 import _lib, sparsity as S  # noqa: E402
from paper_2501_09767_b200.optim import Adam  # noqa: E402
from profile_step import setup  # noqa: E402

model, src, tokens = setup(16384, "lemo", "refined")
opt = Adam(model.lora_param, lr=1e-4)
batch = model.stage_tokens(tokens)
state = {"t": None, "lat": [], "names": []}
orig_sync = torch.cuda.Stream.synchronize
orig_call = _lib.call


def sync(self):
    orig_sync(self)
    state["t"] = time.perf_counter()


def call(name, *args):
    if state["t"] is not None:
        state["lat"].append((time.perf_counter() - state["t"]) * 1e6)
        state["names"].append(name)
        state["t"] = None
    return orig_call(name, *args)


torch.cuda.Stream.synchronize = sync
_lib.call = call
import paper_2501_09767_b200.ops as ops_mod  # noqa: E402
ops_mod.call = call


def step():
    loss, _ = model.forward_step(batch, pattern_source=src, segments=8)
    loss.backward()
    opt.step()
    opt.zero_grad()


for _ in range(3):
    step()
state["lat"].clear(); state["names"].clear()
step()
lat = np.array(state["lat"])
print(f"{len(lat)} read-backs: host latency to the next launch mean {lat.mean():.1f} us, "
      f"median {np.median(lat):.1f}, max {lat.max():.1f}, total {lat.sum() / 1e3:.2f} ms")
from collections import defaultdict  # noqa: E402
by = defaultdict(list)
for n, l in zip(state["names"], lat):
    by[n].append(l)
for n, v in sorted(by.items(), key=lambda kv: -sum(kv[1])):
    print(f"  next = {n:28s} n={len(v):3d} mean {np.mean(v):6.1f} us")
