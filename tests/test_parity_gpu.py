"""Mask parity at the north-star width (Llama2-7B: h=4096, 32 heads, m=11008).

One decoder layer is teacher-forced with a seeded fp32 residual x at s=4096 and
s=16384 (the north-star context).  The oracle (oracle/lemo_oracle.py, NumPy
f32 -- the reference's precision, pinned to the reference by test_oracle.py)
computes the three score vectors the hook selects on:

  attention, exact      layer_qk + exact_block_scores + column sums
                        (model.py:356-368, sparsity.py:173-260)
  attention, predicted  block_embed + predictor pair + Eq. 3 + clamp + column
                        sums with the paper's predictor ranks r1=r2=d_p=1024
                        (predictor.py:117-212, model.py:572-578)
  MLP                   mlp_block_score_vector (model.py:371-396)

Thresholds follow the rule each mode uses in the reference:
  MLP        a fixed threshold, the pooled mean of the profile
             (init_thresholds, sparsity.py:360-376), given to both sides;
  exact      a fixed (tuned) threshold, given to both sides -- here the
             midpoint of the two oracle scores around the median, i.e. a value
             that is not itself a score, as a tuned T + eta·G is not;
  predicted  the recalibration rule (model.py:545-563): each side takes the
             50 % order statistic of ITS OWN score vector, so the masks agree
             iff the rank order at the boundary does.

Flips are classified as in SURVEY §8c's protocol: a flip whose oracle score
lies within 1e-5·|T| of the threshold is an ambiguous block (two correct f32
implementations -- the oracle itself differs from exact arithmetic by ~2e-7
-- may decide it either way); parity precision must show 0 non-ambiguous
flips, and the ambiguous ones are reported (≤ 1 per layer allowed).
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle import lemo_oracle as O
from paper_2501_09767_b200 import exact, model as M, predictor as P

pytestmark = pytest.mark.gpu

WIDTH = dict(n_layers=1, hidden_dim=4096, n_heads=32, vocab_size=512, mlp_dim=11008,
             block_size=16, lora_rank=8, lora_alpha=16.0)
B = 16
PARITY_SCORE_RTOL = 2e-5
BF16_FLIP_FRACTION = 0.01


def oracle_arrays(om):
    arrays = {"embed": om.embed, "final_norm": om.final_norm, "lm_head": om.lm_head}
    if om.pos_embed is not None:  # learned positions (the OPT configuration)
        arrays["pos_embed"] = om.pos_embed
    for i, L in enumerate(om.layers):
        p = f"layer{i}"
        arrays.update({f"{p}.wq": L.wq, f"{p}.wk": L.wk, f"{p}.wv": L.wv, f"{p}.wo": L.wo,
                       f"{p}.attn_norm": L.attn_norm, f"{p}.mlp_norm": L.mlp_norm,
                       f"{p}.w_up": L.w_up, f"{p}.w_down": L.w_down,
                       f"{p}.lora_q.a": L.lora_q[0], f"{p}.lora_q.b": L.lora_q[1],
                       f"{p}.lora_v.a": L.lora_v[0], f"{p}.lora_v.b": L.lora_v[1]})
        if L.w_gate is not None:
            arrays[f"{p}.w_gate"] = L.w_gate
    return arrays


def _flips(got: np.ndarray, ref: np.ndarray, thr: float):
    """(# mask differences, # of them with |ref - T| <= 1e-5 |T|)."""
    diff = (got >= thr) != (ref >= thr)
    amb = diff & (np.abs(ref - thr) <= 1e-5 * abs(thr))
    return int(diff.sum()), int(amb.sum())


def _rel(got: np.ndarray, ref: np.ndarray) -> float:
    return float(np.max(np.abs(got - ref)) / max(np.max(np.abs(ref)), 1e-30))


def _bf16_exact(a):
    return torch.as_tensor(a).to(torch.bfloat16).float().numpy()


@pytest.mark.parametrize("weights", ["fp32", "bf16"])
@pytest.mark.parametrize("s", [4096, 16384])
def test_north_star_width_masks(cuda, s, weights):
    """weights="fp32": reference-init fp32 weights, the parity scorers run
    bf16x3 (3 products); "bf16": bf16-representable weights (bf16
    checkpoints, the bench's init) -- the scorers detect lo == 0 and run the
    2-product form x_hi·W + x_lo·W."""
    cfg = dict(WIDTH, max_seq_len=s)
    om = O.init_model(O.Config(**cfg), seed=11, fast=True)
    O.perturb_lora_b(om, 12)
    L = om.layers[0]
    if weights == "bf16":
        for name in ("wq", "wk", "wv", "wo", "w_up", "w_down", "w_gate"):
            setattr(L, name, _bf16_exact(getattr(L, name)))
    model = M.DecoderModel(M.ModelConfig(**cfg), 0, arrays=oracle_arrays(om),
                           scoring_precision="fp32")
    layer = model.layers[0]
    assert layer.parity_terms == (2 if weights == "bf16" else 3)
    rng = np.random.default_rng(13)
    x = rng.standard_normal((s, 4096), dtype=np.float32)
    n_valid = s - 7  # ragged tail: the last block is partly padding
    prng = np.random.default_rng(14)
    ws = [[(prng.standard_normal(sh, dtype=np.float32) / np.sqrt(sh[0])).astype(np.float32)
           for sh in ((4096, 1024), (1024, 1024), (1024, 1024))] for _ in range(2)]

    # ---- oracle (CPU, f32) --------------------------------------------------
    ref = {}
    ref["mlp"] = O.mlp_block_score_vector(L, x, B, n_valid)
    q, k = O.layer_qk(L, x)
    ref["exact"] = O.column_sums_dense(O.exact_block_dense(q, k, B, n_valid))
    del q, k
    ref["predicted"] = O.predicted_block_vector(O.Predictor(*ws[0]), O.Predictor(*ws[1]), x, B)
    srt = np.sort(ref["exact"])
    mid = (len(srt) - 1) // 2
    thr = {"mlp": float(np.mean(ref["mlp"])),
           "exact": float(0.5 * (srt[mid] + srt[mid + 1])),
           "predicted": None}  # recalibrated per side

    # ---- GPU ------------------------------------------------------------------
    xd = torch.as_tensor(x).cuda()
    pq, pk = P.Predictor(*ws[0]), P.Predictor(*ws[1])
    got = {}
    for prec in ("fp32", "bf16"):
        got[(prec, "mlp")] = M.mlp_block_score_vector(layer, xd, B, n_valid, precision=prec)
        qq, kk = M.layer_qk(layer, xd, precision=prec)
        got[(prec, "exact")] = exact.exact_block_vector(qq, kk, B, n_heads=32, n_valid=n_valid)
        del qq, kk
    # refined: bf16 scores, the rows that can decide a near-threshold block re-scored
    # in parity precision
    v, part = M.mlp_block_score_vector(layer, xd, B, n_valid, precision="bf16", with_partial=True)
    n_ref = M.refine_mlp_block_scores(layer, xd, v, part, thr["mlp"], B, n_valid)
    del part
    got[("refined", "mlp")] = v
    # the predictor path is fp32-faithful in production already (bf16x3)
    got[("fp32", "predicted")] = got[("bf16", "predicted")] = P.predicted_block_vector(
        pq, pk, xd, B)
    torch.cuda.synchronize()

    report = {"s": s, "weights": weights, "parity_terms": layer.parity_terms,
              "n_blocks": len(ref["mlp"]), "refined_rows": n_ref}
    for (prec, mode), vec in got.items():
        g = vec.cpu().numpy()
        t_got = None
        if thr[mode] is None:  # recalibration: each side's own 50 % order statistic
            t_ref, t_got = O.quantile_lower(ref[mode], 0.5), O.quantile_lower(g, 0.5)
            flips = int(((g >= t_got) != (ref[mode] >= t_ref)).sum())
            amb = int((((g >= t_got) != (ref[mode] >= t_ref))
                       & (np.abs(ref[mode] - t_ref) <= 1e-5 * abs(t_ref))).sum())
        else:
            t_ref = thr[mode]
            flips, amb = _flips(g, ref[mode], t_ref)
        diff = (g >= (t_got if thr[mode] is None else t_ref)) != (ref[mode] >= t_ref)
        margin = (float(np.max(np.abs(ref[mode][diff] - t_ref)) / abs(t_ref))
                  if diff.any() else None)
        report[f"{prec}_{mode}"] = {"flips": flips, "ambiguous": amb,
                                    "score_rel_err": _rel(g, ref[mode]),
                                    "max_flip_margin_rel": margin,
                                    "retained": float(np.mean(ref[mode] >= t_ref))}
    print("mask parity", json.dumps(report))
    out = os.environ.get("LEMO_PARITY_OUT")
    if out:
        with open(os.path.join(out, f"parity_{s}_{weights}.json"), "w") as f:
            json.dump(report, f, indent=1)
    nb = report["n_blocks"]
    for prec, mode in (("fp32", "mlp"), ("fp32", "exact"), ("fp32", "predicted"),
                       ("refined", "mlp")):
        r = report[f"{prec}_{mode}"]
        assert r["flips"] - r["ambiguous"] == 0 and r["ambiguous"] <= 1, (prec, mode, r)
        if prec == "fp32":  # refined only re-scores the blocks near the threshold
            assert r["score_rel_err"] <= PARITY_SCORE_RTOL, (mode, r)
        rb = report[f"bf16_{mode}"]
        assert rb["flips"] <= BF16_FLIP_FRACTION * nb, (mode, rb)


@pytest.mark.parametrize("variant,mlp_dim", [("silu", 14336), ("relu", 16384)])
def test_mlp_masks_other_baseline_widths(cuda, variant, mlp_dim):
    """MLP mask parity at the other BASELINE widths: Llama3-8B / Mistral-7B
    (SwiGLU, m = 14336) and OPT-6.7B in the reference family (ReLU,
    m = 16384), h = 4096, s = 4096, one layer teacher-forced with a seeded
    residual.  Parity and refined precision: 0 non-ambiguous flips against
    the oracle (f32, model.py:371-396); bf16 flips bounded."""
    s = 4096
    cfg = dict(WIDTH, max_seq_len=s, mlp_dim=mlp_dim, mlp_variant=variant)
    om = O.init_model(O.Config(**cfg), seed=21, fast=True)
    model = M.DecoderModel(M.ModelConfig(**cfg), 0, arrays=oracle_arrays(om),
                           scoring_precision="fp32")
    layer = model.layers[0]
    x = np.random.default_rng(22).standard_normal((s, 4096), dtype=np.float32)
    n_valid = s - 3
    ref = O.mlp_block_score_vector(om.layers[0], x, B, n_valid)
    thr = float(np.mean(ref))
    xd = torch.as_tensor(x).cuda()
    got = {p: M.mlp_block_score_vector(layer, xd, B, n_valid, precision=p)
           for p in ("fp32", "bf16")}
    v, part = M.mlp_block_score_vector(layer, xd, B, n_valid, precision="bf16", with_partial=True)
    rows = M.refine_mlp_block_scores(layer, xd, v, part, thr, B, n_valid)
    got["refined"] = v
    report = {"variant": variant, "mlp_dim": mlp_dim, "refined_rows": rows}
    for p, vec in got.items():
        g = vec.cpu().numpy()
        flips, amb = _flips(g, ref, thr)
        report[p] = {"flips": flips, "ambiguous": amb, "score_rel_err": _rel(g, ref)}
    print("mlp mask parity", json.dumps(report))
    for p in ("fp32", "refined"):
        assert report[p]["flips"] - report[p]["ambiguous"] == 0 and report[p]["ambiguous"] <= 1, \
            (p, report)
    assert report["fp32"]["score_rel_err"] <= PARITY_SCORE_RTOL, report
    assert report["bf16"]["flips"] <= BF16_FLIP_FRACTION * len(ref), report


@pytest.mark.parametrize("geometry", ["gqa", "learned_positions"])
def test_exact_attention_masks_gqa_width(cuda, geometry):
    """Exact-attention mask parity at the other BASELINE geometries, s = 4096:
    "gqa" = Llama3-8B / Mistral-7B (grouped-query attention, 32 query / 8
    key-value heads, RoPE base 500000); "learned_positions" = the OPT-6.7B
    configuration in the reference family (no RoPE in layer_qk).  layer_qk +
    the tcgen05 exact scorer + column sums vs the oracle (model.py:356-368,
    sparsity.py:173-260; key heads repeated for GQA, the extension pinned in
    test_step_gpu).  Parity precision 0 non-ambiguous flips, bf16 bounded."""
    s = 4096
    cfg = (dict(WIDTH, max_seq_len=s, n_kv_heads=8, rope_base=500000.0) if geometry == "gqa"
           else dict(WIDTH, max_seq_len=s, positions="learned"))
    om = O.init_model(O.Config(**cfg), seed=31, fast=True)
    O.perturb_lora_b(om, 32)
    model = M.DecoderModel(M.ModelConfig(**cfg), 0, arrays=oracle_arrays(om),
                           scoring_precision="fp32")
    layer = model.layers[0]
    x = np.random.default_rng(33).standard_normal((s, 4096), dtype=np.float32)
    n_valid = s - 5
    q, k = O.layer_qk(om.layers[0], x)
    ref = O.column_sums_dense(O.exact_block_dense(q, k, B, n_valid))
    del q, k
    srt = np.sort(ref)
    mid = (len(srt) - 1) // 2
    thr = float(0.5 * (srt[mid] + srt[mid + 1]))
    xd = torch.as_tensor(x).cuda()
    report = {"geometry": geometry}
    for prec in ("fp32", "bf16"):
        qq, kk = M.layer_qk(layer, xd, precision=prec)
        g = exact.exact_block_vector(qq, kk, B, n_heads=32, n_valid=n_valid).cpu().numpy()
        del qq, kk
        flips, amb = _flips(g, ref, thr)
        report[prec] = {"flips": flips, "ambiguous": amb, "score_rel_err": _rel(g, ref)}
    print("gqa exact mask parity", json.dumps(report))
    r = report["fp32"]
    assert r["flips"] - r["ambiguous"] == 0 and r["ambiguous"] <= 1, report
    assert r["score_rel_err"] <= PARITY_SCORE_RTOL, report
    assert report["bf16"]["flips"] <= BF16_FLIP_FRACTION * len(ref), report
