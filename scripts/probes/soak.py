"""Soak run of the N* training step (refined scorers): 60 steps with a fresh
synthetic sequence each step, per-step CUDA-event time, loss, allocator
footprint and recalibrated thresholds -- steady state, no memory growth, no
non-finite loss."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_09767_b200.optim import Adam  # noqa: E402
from profile_step import setup  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 60
model, src, _ = setup(16384, "lemo", "refined")
opt = Adam(model.lora_param, lr=1e-4)
rng = np.random.default_rng(7)
rec = []
for i in range(steps):
    tokens = rng.integers(0, model.config.vocab_size, 16384)
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    loss, _ = model.forward_step(tokens, pattern_source=src, segments=8)
    loss.backward()
    opt.step()
    opt.zero_grad()
    b.record()
    lv = float(loss.detach())
    torch.cuda.synchronize()
    rec.append({"step": i, "ms": a.elapsed_time(b), "loss": lv,
                "alloc_gb": torch.cuda.memory_allocated() / 1e9,
                "retained_attn": float(np.mean([v for (l, c), v in src.last_fractions.items()
                                                if c == "attention"]))})
ms = np.array([r["ms"] for r in rec[3:]])
al = np.array([r["alloc_gb"] for r in rec])
out = {"steps": steps, "ms_mean": float(ms.mean()), "ms_min": float(ms.min()),
       "ms_max": float(ms.max()), "tokens_per_s_mean": 16384 / ms.mean() * 1e3,
       "alloc_gb_first": float(al[0]), "alloc_gb_last": float(al[-1]),
       "alloc_gb_max": float(al.max()), "loss_first": rec[0]["loss"], "loss_last": rec[-1]["loss"],
       "all_finite": bool(all(np.isfinite(r["loss"]) for r in rec)),
       "retained_attn_range": [float(min(r["retained_attn"] for r in rec)),
                               float(max(r["retained_attn"] for r in rec))],
       "peak_gb": torch.cuda.max_memory_allocated() / 1e9}
print(json.dumps(out))
