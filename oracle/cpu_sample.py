"""Bounded CPU sample of the bench workload, timed with the oracle.

TEST/BENCH INFRASTRUCTURE ONLY (the cpu_baseline leg of bench.py and its
--impl reference arm).  The reference itself is Python and cannot travel to
the GPU box, so its algorithm runs here through the oracle restatement
(oracle/lemo_oracle.py, pinned to reference outputs by tests/test_oracle.py).

Sample: one decoder layer at the workload's full width (default Llama2-7B:
h=4096, 32 heads, m=11008, V=32000, LoRA r=8; bench.py passes the geometry of
the configuration it runs) on `sample_tokens` tokens, trained one
step in LeMo predicted mode (random predictors r1=r2=d_p=h/4, attention
retention 0.5 by the quantile rule, MLP threshold = pooled mean of the
exact MLP scores), forward + backward.  The LM-head/loss cost is timed
separately so tokens/s extrapolates as  s / (n_layers·t_layer + t_head).
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import lemo_oracle as O


class CpuSample:
    def __init__(self, *, hidden=4096, heads=32, mlp=11008, vocab=32000, n_layers_model=32,
                 sample_tokens=4096, block=16, lora_rank=8, seed=0, kv_heads=0,
                 mlp_variant="silu", positions="rope"):
        self.n_layers_model = n_layers_model
        self.s = sample_tokens
        self.geometry = dict(hidden=hidden, heads=heads, kv_heads=kv_heads or heads, mlp=mlp,
                             vocab=vocab, layers=n_layers_model, mlp_variant=mlp_variant,
                             positions=positions)
        cfg = O.Config(n_layers=1, hidden_dim=hidden, n_heads=heads, vocab_size=vocab,
                       max_seq_len=sample_tokens, mlp_dim=mlp, block_size=block,
                       lora_rank=lora_rank, lora_alpha=2.0 * lora_rank, n_kv_heads=kv_heads,
                       mlp_variant=mlp_variant, positions=positions)
        self.model = O.init_model(cfg, seed=seed, fast=True)
        rng = np.random.default_rng(seed + 1)
        L = self.model.layers[0]
        r = hidden // 4
        L.predictor_q = O.create_predictor(rng, hidden, r, r, r)
        L.predictor_k = O.create_predictor(rng, hidden, r, r, r)
        self.tokens = rng.integers(0, vocab, sample_tokens)
        # thresholds: MLP = pooled mean of exact MLP scores (init_thresholds,
        # sparsity.py:360-376); attention = quantile rule at 50% retention.
        x0 = self.model.embed[self.tokens]
        mlp_vec = O.mlp_block_score_vector(L, x0, block, sample_tokens)
        self.thresholds = {(0, O.ATTENTION): 0.0, (0, O.MLP): float(mlp_vec.mean())}
        self.hidden = (rng.standard_normal((sample_tokens, hidden)) / 8).astype(np.float32)

    def source(self):
        return O.PredictedSource(self.model, dict(self.thresholds), target_retention={0: 0.5},
                                 recalibrate_every=1)

    def time_head(self) -> float:
        tg = np.concatenate([self.tokens[1:], [-1]])
        t0 = time.perf_counter()
        O.segmented_loss_and_grad(self.hidden, self.model.lm_head, tg, 8)
        return time.perf_counter() - t0

    def time_step(self) -> tuple[float, dict]:
        t0 = time.perf_counter()
        res = O.train_step(self.model, self.tokens, source=self.source(), segments=8)
        return time.perf_counter() - t0, res

    def measure(self) -> dict:
        t_step, res = self.time_step()
        t_head = self.time_head()
        t_layer = max(t_step - t_head, 1e-9)
        per_step = self.n_layers_model * t_layer + t_head
        fr = {f"{l}:{c}": (1.0 if p is None else len(O.token_indices(p, 16, self.s)) / self.s)
              for (l, c), p in res["patterns"].items()}
        return {"tokens_per_s": self.s / per_step, "t_layer_s": t_layer, "t_head_s": t_head,
                "t_step_extrapolated_s": per_step, "retained": fr}


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
