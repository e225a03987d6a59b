"""The offline stages adjacent to the hot path, on the GPU (SURVEY.md §8f rows
1-2): exact-score teacher generation, predictor training, predicted-threshold
initialisation and Algorithm 1 threshold tuning.

Library entry points with the reference's names and argument meaning
(pipeline.py:178-367): everything that touches tensors runs through the
liblemo kernels — teacher scores are the fused exact block scorer on the
layer's tcgen05 Q/K projections, predictor training is fp32-faithful bf16x3
tcgen05 GEMMs (predictor.fit_predictors), tuning evaluates the sparse forward.
Orchestration (CLI, corpus loading, run directories) stays out of scope.
"""

from __future__ import annotations

import dataclasses

import numpy as np
import torch

from . import artifacts
from . import model as model_mod
from . import predictor as predictor_mod
from . import sparsity
from .errors import ContractError


def collect_teacher_records(model: model_mod.DecoderModel, seqs, n_batches: int,
                            block_size: int | None = None) -> list:
    """pipeline.py:280-300: exact block scores (packed triangles) and layer
    inputs for every layer of the first `n_batches` sequences.  `seqs` items
    are token arrays or (tokens, targets) pairs."""
    if block_size is not None and block_size != model.config.block_size:
        raise ContractError("teacher block size must equal the model's block size on the GPU")
    source = model_mod.ExactPatternSource(model, None, mlp_scoring=False, record=True,
                                          record_inputs=True)
    with torch.no_grad():
        for i in range(min(n_batches, len(seqs))):
            item = seqs[i]
            tokens, targets = item if isinstance(item, tuple) else (item, None)
            model.forward_step(tokens, targets, pattern_source=source)
    b = model.config.block_size
    per_layer: dict = {}
    for bsm in source.recorded_matrices:
        per_layer.setdefault(bsm.layer_id, []).append(bsm.scores)
    records = []
    for layer_id, tris in per_layer.items():
        for x, tri in zip(source.recorded_inputs[layer_id], tris):
            records.append(predictor_mod.TeacherRecord(layer_id, x, tri, x.shape[0], b))
    return records


def create_pairs(model: model_mod.DecoderModel, r1: int, r2: int, d_pred: int,
                 seed: int = 0) -> dict:
    """Predictor.create for every layer in the reference's draw order
    (pipeline.py:317-330)."""
    rng = np.random.default_rng(seed)
    h = model.config.hidden_dim
    dev = model.device
    return {l: (predictor_mod.Predictor.create(rng, h, r1, r2, d_pred, "q", l, dev),
                predictor_mod.Predictor.create(rng, h, r1, r2, d_pred, "k", l, dev))
            for l in range(model.config.n_layers)}


def train_predictors(model: model_mod.DecoderModel, shard, epochs: int, lr: float, *,
                     block_size: int | None = None, val_shard=None, thresholds=None,
                     r1: int = 16, r2: int = 16, d_pred: int = 16, seed: int = 0,
                     **fit_kwargs):
    """Library entry point (pipeline.py:303-333): teacher labels from the
    model's exact scores on `shard`, then offline regression.  Returns
    (pairs, history)."""
    records = collect_teacher_records(model, shard, len(shard), block_size)
    val = collect_teacher_records(model, val_shard, len(val_shard), block_size) \
        if val_shard else None
    pairs = create_pairs(model, r1, r2, d_pred, seed)
    history = predictor_mod.fit_predictors(pairs, records, epochs=epochs, lr=lr, val_data=val,
                                           thresholds=thresholds, **fit_kwargs)
    return pairs, history


def predicted_threshold_init(pairs: dict, records: list, exact_thresholds, *,
                             pooling: str = "mean", cfg_hash: str = ""):
    """pipeline.py:336-367: per layer, the predicted-side attention threshold
    retaining the fraction of blocks the exact threshold retains on the
    teacher shard; MLP thresholds carry over.  Returns (ThresholdSet,
    retention by layer)."""
    pred_by: dict = {}
    exact_by: dict = {}
    for rec in records:
        p_q, p_k = pairs[rec.layer_id]
        pred_by.setdefault(rec.layer_id, []).append(
            predictor_mod.predicted_block_vector(p_q, p_k, rec.x, rec.block_size, pooling))
        nb = sparsity.n_blocks_for(rec.n_tokens, rec.block_size)
        exact_by.setdefault(rec.layer_id, []).append(sparsity.token_block_scores(
            sparsity.BlockScoreMatrix(nb, rec.block_size, rec.teacher_packed)))
    ts = sparsity.ThresholdSet(config_hash=cfg_hash)
    retention = {}
    for layer_id, pv in pred_by.items():
        pred = torch.cat(pv)
        exact = torch.cat(exact_by[layer_id])
        thr = exact_thresholds.get(layer_id, sparsity.ATTENTION)
        ts.values[(layer_id, sparsity.ATTENTION)] = predictor_mod.retention_matched_threshold(
            pred, exact, thr)
        retention[layer_id] = float((exact >= thr).double().mean().item())
        if (layer_id, sparsity.MLP) in exact_thresholds.values:
            ts.values[(layer_id, sparsity.MLP)] = exact_thresholds.get(layer_id, sparsity.MLP)
    return ts, retention


def mean_eval_loss(model: model_mod.DecoderModel, eval_seqs, source, segments: int,
                   limit: int) -> float:
    """pipeline.py:178-187: mean loss of sparse eval forwards (no backward)."""
    losses = []
    with torch.no_grad():
        for item in eval_seqs[:limit]:
            tokens, targets = item if isinstance(item, tuple) else (item, None)
            loss, _ = model.forward_step(tokens, targets, pattern_source=source,
                                         segments=segments)
            losses.append(loss.detach())
    return float(torch.stack(losses).mean().item()) if losses else float("nan")


def tune_thresholds(model: model_mod.DecoderModel, thresholds, eval_seqs, *, segments: int = 1,
                    limit: int = 4, mlp_scoring: bool = True, sink_first_block: bool = False,
                    eps=None, eta=None, rounds: int = 1):
    """run_tune_thresholds (pipeline.py:190-223) minus the file IO: Algorithm 1
    step 2 with acc = −mean eval loss of exact-pattern sparse forwards."""
    def acc(ts):
        src = model_mod.ExactPatternSource(model, ts, mlp_scoring=mlp_scoring,
                                           sink_first_block=sink_first_block)
        return -mean_eval_loss(model, eval_seqs, src, segments, limit)

    return sparsity.tune_thresholds(acc, thresholds, eps=eps, eta=eta, rounds=rounds)


def save_predictors(path, model: model_mod.DecoderModel, pairs, pred_thresholds,
                    retention=None, *, mlp_scoring: bool = True, pooling: str = "mean") -> None:
    """predictors.ckpt exactly as the reference writes it, stamped with the
    reference's configuration hash of this model's geometry."""
    artifacts.save_predictors(path, pairs, pred_thresholds, retention, pooling=pooling,
                              cfg_hash=artifacts.config_hash(model.config, mlp_scoring),
                              config={"model": dataclasses.asdict(model.config)})


def load_predictors(path, model: model_mod.DecoderModel, *, mlp_scoring: bool = True,
                    attach: bool = True):
    """Reference-written predictors.ckpt onto this model's GPU (hash-checked)."""
    pairs, pt, retention, meta = artifacts.load_predictors(
        path, n_layers=model.config.n_layers, hidden_dim=model.config.hidden_dim,
        cfg_hash=artifacts.config_hash(model.config, mlp_scoring), device=model.device)
    if attach:
        model.attach_predictors(pairs)
    return pairs, pt, retention


__all__ = ["collect_teacher_records", "create_pairs", "train_predictors",
           "predicted_threshold_init", "mean_eval_loss", "tune_thresholds", "save_predictors",
           "load_predictors"]
