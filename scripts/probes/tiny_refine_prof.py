"""Where the refined precision's extra time goes at config T (torch.profiler)."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2501_09767_b200 import model as M, predictor as P, sparsity as S  # noqa: E402
from paper_2501_09767_b200.optim import Adam  # noqa: E402

dev = torch.device("cuda")
cfg = M.tiny_t()
model = M.DecoderModel(cfg, seed=0, device=dev, init="torch", scoring_precision="refined",
                       parity_weights=True)
h, rp = cfg.hidden_dim, cfg.hidden_dim // 4
g = torch.Generator(device=dev).manual_seed(1)
mk = lambda: P.Predictor(torch.randn(h, rp, generator=g, device=dev) / math.sqrt(h),  # noqa
                         torch.randn(rp, rp, generator=g, device=dev) / math.sqrt(rp),
                         torch.randn(rp, rp, generator=g, device=dev) / math.sqrt(rp), device=dev)
model.attach_predictors({l: (mk(), mk()) for l in range(cfg.n_layers)})
tokens = np.random.default_rng(0).integers(0, cfg.vocab_size, 2048)
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from bench import _mlp_only_profile  # noqa: E402

prof0 = M.ExactPatternSource(model, None, record=True)  # the bench's threshold protocol
prof0.pattern = _mlp_only_profile(prof0, S)
with torch.no_grad():
    model.forward_step(tokens, pattern_source=prof0, segments=8)
thr = S.init_thresholds(prof0.recorded_vectors)
for l in range(2):
    thr.set(l, S.ATTENTION, 0.0)
src = M.PredictedPatternSource(model, thr, target_retention={0: .5, 1: .5}, recalibrate_every=50)
opt = Adam(model.lora_param, lr=1e-4)
batch = model.stage_tokens(tokens)


def step():
    loss, _ = model.forward_step(batch, pattern_source=src, segments=8)
    loss.backward()
    opt.step()
    opt.zero_grad()


for prec in ("bf16", "refined"):
    model.set_scoring_precision(prec)
    for _ in range(5):
        step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(20):
        step()
    b.record()
    torch.cuda.synchronize()
    print(prec, "ms/step", a.elapsed_time(b) / 20, "refined rows", dict(src.refined_rows))
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts) as prof:
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    with torch.profiler.record_function("REFINE_ONLY"):
        x = torch.randn(2048, 256, device=dev)
        layer = model.layers[0]
        v, part = M.mlp_block_score_vector(layer, x, 16, 2048, precision="bf16", with_partial=True)
        M.refine_mlp_block_scores(layer, x, v, part, float(v.median()), 16, 2048)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=30))
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
