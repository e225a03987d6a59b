"""cProfile of the host side of a config-T LeMo step (host-bound regime)."""
import cProfile
import math
import pstats
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2501_09767_b200 import model as M, predictor as P, sparsity as S  # noqa: E402
from paper_2501_09767_b200.optim import Adam  # noqa: E402

dev = torch.device("cuda")
cfg = M.tiny_t()
model = M.DecoderModel(cfg, seed=0, device=dev, init="torch")
h, rp = cfg.hidden_dim, cfg.hidden_dim // 4
g = torch.Generator(device=dev).manual_seed(1)
mk = lambda: P.Predictor(torch.randn(h, rp, generator=g, device=dev) / math.sqrt(h),  # noqa
                         torch.randn(rp, rp, generator=g, device=dev) / math.sqrt(rp),
                         torch.randn(rp, rp, generator=g, device=dev) / math.sqrt(rp), device=dev)
model.attach_predictors({l: (mk(), mk()) for l in range(cfg.n_layers)})
tokens = np.random.default_rng(0).integers(0, cfg.vocab_size, 2048)
thr = S.ThresholdSet({(l, c): 0.0 for l in range(2) for c in S.COMPONENTS})
src = M.PredictedPatternSource(model, thr, target_retention={0: .5, 1: .5}, recalibrate_every=50)
opt = Adam(model.lora_param, lr=1e-4)
batch = model.stage_tokens(tokens)


def step(source):
    loss, _ = model.forward_step(batch, pattern_source=source, segments=8)
    loss.backward()
    opt.step()
    opt.zero_grad()


for mode, source in (("lemo", src), ("dense", None)):
    for _ in range(5):
        step(source)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(20):
        step(source)
    b.record()
    torch.cuda.synchronize()
    print(mode, "ms/step", a.elapsed_time(b) / 20)
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    step(src)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
