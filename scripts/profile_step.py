"""Set up the bench workload, warm up, then run ONE step inside
cudaProfilerStart/Stop so `ncu --profile-from-start off` sees exactly one
training step.  Usage (on the GPU box):

  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file gpurun_out/launches.csv python scripts/profile_step.py
  ncu --profile-from-start off --set full --clock-control none --import-source on \
      -k regex:EpiGateUp -c 1 -o gpurun_out/prof_gateup python scripts/profile_step.py
"""

import argparse
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2501_09767_b200 import model as M, predictor as P, sparsity as S  # noqa: E402
from paper_2501_09767_b200.optim import Adam  # noqa: E402


def setup(seq=16384, mode="lemo", precision="refined"):
    dev = torch.device("cuda")
    cfg = M.llama2_7b(max_seq_len=seq)
    # the bench's default: refined scorers (bf16 + parity re-scoring near the threshold)
    model = M.DecoderModel(cfg, seed=0, device=dev, init="torch", scoring_precision=precision,
                           parity_weights=precision != "bf16")
    h = cfg.hidden_dim
    rp = h // 4
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    pairs = {}
    for l in range(cfg.n_layers):
        mk = lambda: P.Predictor(torch.randn(h, rp, generator=gen, device=dev) / math.sqrt(h),  # noqa
                                 torch.randn(rp, rp, generator=gen, device=dev) / math.sqrt(rp),
                                 torch.randn(rp, rp, generator=gen, device=dev) / math.sqrt(rp),
                                 device=dev)
        pairs[l] = (mk(), mk())
    model.attach_predictors(pairs)
    tokens = np.random.default_rng(1000).integers(0, cfg.vocab_size, size=seq)
    if mode == "dense":
        return model, None, tokens
    prof = M.ExactPatternSource(model, None, record=True)
    orig = prof.pattern

    def mlp_only(layer_id, component, x, n_valid):
        if component == S.ATTENTION:
            return prof._note(layer_id, component, None)
        return orig(layer_id, component, x, n_valid)

    prof.pattern = mlp_only
    with torch.no_grad():
        model.forward_step(tokens, pattern_source=prof, segments=8)
    thr = S.init_thresholds(prof.recorded_vectors)
    for l in range(cfg.n_layers):
        thr.set(l, S.ATTENTION, 0.0)
    model._mlp_scored.clear()
    ret = {l: 0.5 for l in range(cfg.n_layers)}
    cal = M.PredictedPatternSource(model, thr.copy(), target_retention=ret, recalibrate_every=1)
    with torch.no_grad():
        model.forward_step(tokens, pattern_source=cal, segments=8)
    model._mlp_scored.clear()
    src = M.PredictedPatternSource(model, cal.thresholds.copy(), target_retention=ret,
                                   recalibrate_every=50)
    return model, src, tokens


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=16384)
    ap.add_argument("--mode", default="lemo", choices=["lemo", "dense"])
    ap.add_argument("--scoring-precision", default="refined", choices=["bf16", "fp32", "refined"])
    args = ap.parse_args()
    model, src, tokens = setup(args.seq, args.mode, args.scoring_precision)
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
    torch.cuda.cudart().cudaProfilerStart()
    step()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("retained", {k: round(v, 3) for k, v in (src.last_fractions.items() if src else [])})


if __name__ == "__main__":
    main()
