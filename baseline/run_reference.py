"""Time the UNMODIFIED reference (`sparsetune`, installed into baseline/_ref)
on this host's cores -- the reference arm of bench.py and its cpu_baseline.

Run as a subprocess with the BLAS thread pool sized by the environment
(OPENBLAS_NUM_THREADS / OMP_NUM_THREADS set by bench.py before NumPy loads):

    PYTHONPATH=baseline/_ref python baseline/run_reference.py --layer-seq 16384 ...

Everything timed goes through the reference's own public API and stock code
path (model.py:246-297 forward_step, tensor.backward, optim.Adam): no kernel
or module of this repository is imported.  Workload = BASELINE.md §3:
synthetic tokens `default_rng(seed).integers(0, V, s)`, reference init,
b=16, 8 loss segments, LeMo predicted mode (random predictors, ranks h/4;
attention retention 0.5 by the quantile rule re-derived on every call, MLP
threshold = pooled mean of exact MLP scores of a profiling sample).

Measurements (printed as one JSON object):
  tiny   config T (2 layers, h=256): the FULL training step (forward_step +
         backward + Adam), median of >= 5 steps after one warm-up step.
  layer  one Llama2-7B-width decoder layer (h=4096, 32 heads, m=11008,
         V=32000) at --layer-seq tokens: forward_step + backward of a
         1-layer model, repeated while --budget-s allows (>= 1 sample); the
         LM-head loss (segmented_loss_and_grad at the same shape) is timed
         separately so that  t_layer = t_sample - t_head  and the 32-layer
         step extrapolates as 32·t_layer + t_head.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

REF = Path(__file__).resolve().parent / "_ref"
if REF.exists():
    sys.path.insert(0, str(REF))

import numpy as np  # noqa: E402

from sparsetune import kernels, model as M, predictor as P, sparsity  # noqa: E402
from sparsetune import tensor as T  # noqa: E402
from sparsetune.optim import Adam  # noqa: E402

SEGMENTS = 8


def _source(model, cfg, tokens, mlp_profile_tokens: int, seed: int):
    """PredictedPatternSource with random predictors (ranks h/4) and the
    thresholds of BASELINE.md §3: MLP = pooled mean of the exact MLP scores
    of the embedded input (the reference's own scorer, model.py:371-396),
    attention = 50 % quantile re-derived on every call (model.py:545-563)."""
    h = cfg.hidden_dim
    r = h // 4
    rng = np.random.default_rng(seed + 1)
    pairs = {l: (P.Predictor.create(rng, h, r, r, r, "q", l),
                 P.Predictor.create(rng, h, r, r, r, "k", l)) for l in range(cfg.n_layers)}
    model.attach_predictors(pairs)
    x0 = model.embed.data[tokens[:mlp_profile_tokens]]
    mlp_thr = float(M.mlp_block_score_vector(model.layers[0], x0, cfg.block_size,
                                             x0.shape[0]).mean())
    ts = sparsity.ThresholdSet({(l, c): (mlp_thr if c == sparsity.MLP else 0.0)
                                for l in range(cfg.n_layers) for c in sparsity.COMPONENTS})
    return M.PredictedPatternSource(model, ts, target_retention={l: 0.5 for l in
                                                                 range(cfg.n_layers)},
                                    recalibrate_every=1)


def _train_step(model, tokens, src, opt=None):
    loss, _ = model.forward_step(tokens, pattern_source=src, segments=SEGMENTS)
    T.backward(loss)
    if opt is not None:
        opt.step()
        opt.zero_grad()
    return float(loss.data)


def tiny(steps: int, seed: int = 0) -> dict:
    cfg = M.ModelConfig(n_layers=2, hidden_dim=256, n_heads=4, vocab_size=256, max_seq_len=2048,
                        mlp_dim=688, block_size=16, lora_rank=8, lora_alpha=16.0)
    model = M.DecoderModel(cfg, seed=seed)
    tokens = np.random.default_rng(seed).integers(0, cfg.vocab_size, size=2048)
    src = _source(model, cfg, tokens, 2048, seed)
    opt = Adam(model.adapter_parameters(), lr=1e-4)
    _train_step(model, tokens, src, opt)  # warm-up
    times = []
    for _ in range(max(steps, 5)):
        t0 = time.perf_counter()
        _train_step(model, tokens, src, opt)
        times.append(time.perf_counter() - t0)
    med = float(np.median(times))
    return {"seq": 2048, "steps": len(times), "median_s": med, "tokens_per_s": 2048 / med,
            "step_s": times,
            "what": "config T full training step (2 layers, h=256): forward_step + backward + "
                    "Adam, LeMo predicted mode"}


def layer(seq: int, budget_s: float, seed: int = 0, max_samples: int = 8) -> dict:
    cfg = M.ModelConfig(n_layers=1, hidden_dim=4096, n_heads=32, vocab_size=32000,
                        max_seq_len=seq, mlp_dim=11008, block_size=16, lora_rank=8,
                        lora_alpha=16.0)
    t0 = time.perf_counter()
    model = M.DecoderModel(cfg, seed=seed)
    tokens = np.random.default_rng(seed).integers(0, cfg.vocab_size, size=seq)
    src = _source(model, cfg, tokens, min(seq, 2048), seed)
    setup = time.perf_counter() - t0
    # LM head alone (same shapes as inside the step): segmented_loss_and_grad
    hid = T.Tensor((np.random.default_rng(seed + 2).standard_normal((seq, 4096)) / 8)
                   .astype(np.float32), requires_grad=True)
    tg = np.concatenate([tokens[1:], [-1]])
    t0 = time.perf_counter()
    loss = kernels.segmented_loss_and_grad(hid, model.lm_head, tg,
                                           kernels.SegmentPlan.even(seq, SEGMENTS))
    T.backward(loss)
    t_head = time.perf_counter() - t0
    samples, fr = [], {}
    t_start = time.perf_counter()
    while len(samples) < max_samples:
        t0 = time.perf_counter()
        _train_step(model, tokens, src)
        samples.append(time.perf_counter() - t0)
        fr = {f"{l}:{c}": f for (l, c), f in src.last_fractions.items()}
        if time.perf_counter() - t_start + samples[-1] > budget_s:
            break
    t_sample = float(np.median(samples))
    t_layer = max(t_sample - t_head, 1e-9)
    step32 = 32 * t_layer + t_head
    return {"seq": seq, "samples": len(samples), "sample_s": samples, "median_sample_s": t_sample,
            "head_s": t_head, "layer_s": t_layer, "extrapolated_step_s": step32,
            "tokens_per_s": seq / step32, "setup_s": setup, "retained": fr,
            "what": f"1-layer Llama2-7B-width model (h=4096, 32 heads, m=11008, V=32000) at "
                    f"{seq} tokens: forward_step + backward in LeMo predicted mode; LM-head "
                    "loss timed alone; 32-layer step = 32·t_layer + t_head"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tiny-steps", type=int, default=5)
    ap.add_argument("--layer-seq", type=int, nargs="*", default=[16384])
    ap.add_argument("--budget-s", type=float, default=150.0)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    out = {"reference": str(REF), "numpy": np.__version__,
           "threads": os.environ.get("OPENBLAS_NUM_THREADS")}
    if a.tiny_steps > 0:
        out["tiny"] = tiny(a.tiny_steps, a.seed)
    for s in a.layer_seq:
        out[f"layer_{s}"] = layer(s, a.budget_s, a.seed)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
