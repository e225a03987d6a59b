"""Whole-step parity: GPU forward_step + sparse backward vs the reference.

The golden fixtures hold the reference's own loss / LoRA gradients / masks
for a 2-layer model (tests/golden/make_golden.py); the oracle (pinned to the
same fixtures by test_oracle.py) supplies extra cases at full Llama width.

Two geometries: head_dim 64 (h=128, H=2; suffix "") and head_dim 128
(h=256, H=2; suffix "_d128", the production attention kernels' head size).

Tolerances (bf16 GEMM operands, fp32 accumulation, fp32 residual stream):
  loss       relative error <= 1e-2   (measured <= 3.6e-4)
  LoRA grads relative L2 error (per tensor) <= 3e-2
SURVEY §8c proposes 2e-2 for bf16 runs; the measured worst case is 2.6e-2
(layer1.lora_q.a of the GQA fixture; 1.6e-2..2.4e-2 on the golden steps): the
attention backward consumes dO, P and dS as bf16 tensor-core operands and the
residual gradient enters every dX GEMM rounded to bf16, and layer 1's A_q
gradient is the deepest product of those roundings.  The errors are printed
(pytest -s) so the slack stays visible.
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import lemo_oracle as O
from paper_2501_09767_b200 import model as M, predictor as P, sparsity as S
from paper_2501_09767_b200.optim import Adam

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"

STEP_CFG = dict(n_layers=2, hidden_dim=128, n_heads=2, vocab_size=128, max_seq_len=256,
                mlp_dim=344, block_size=16, lora_rank=8, lora_alpha=16.0)
STEP_VARIANTS = {"": STEP_CFG, "_d128": dict(STEP_CFG, hidden_dim=256)}
LOSS_RTOL = 1e-2
GRAD_RL2 = 3e-2


def _model_and_oracle(suffix="", scoring_precision="bf16"):
    cfg = STEP_VARIANTS[suffix]
    om = O.init_model(O.Config(**cfg), seed=17)
    O.perturb_lora_b(om, 23)
    arrays = M.reference_init_arrays(M.ModelConfig(**cfg), 17)
    for name in om.adapter_names():
        arrays[name] = om.adapter(name)
    return M.DecoderModel(M.ModelConfig(**cfg), 17, arrays=arrays,
                          scoring_precision=scoring_precision), om


def _rl2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def _source(mode, model, z):
    if mode == "dense":
        return None
    if mode == "fraction":
        return M.FractionSource(0.5, 16)
    thr = S.ThresholdSet({(l, c): float(z[f"thr_{l}_{c}"]) for l in range(2)
                          for c in (S.ATTENTION, S.MLP)})
    if mode == "exact":
        return M.ExactPatternSource(model, thr)
    pairs = {l: (P.Predictor(z[f"pred{l}_q_w1"], z[f"pred{l}_q_w2"], z[f"pred{l}_q_w3"], "q", l),
                 P.Predictor(z[f"pred{l}_k_w1"], z[f"pred{l}_k_w2"], z[f"pred{l}_k_w3"], "k", l))
             for l in range(2)}
    model.attach_predictors(pairs)
    return M.PredictedPatternSource(model, thr, target_retention={0: 0.5, 1: 0.5},
                                    recalibrate_every=1)


@pytest.mark.parametrize("suffix", ["", "_d128"])
@pytest.mark.parametrize("mode", ["dense", "fraction", "predicted", "exact"])
def test_step_matches_reference(cuda, mode, suffix):
    z = np.load(G / f"step_{mode}{suffix}.npz")
    model, _ = _model_and_oracle(suffix)
    src = _source(mode, model, z)
    loss, hidden = model.forward_step(z["tokens"], pattern_source=src, segments=2)
    loss.backward()
    got = float(loss)
    loss_err = abs(got - z["losses"][0]) / abs(z["losses"][0])
    grads = model.adapter_grads()
    errs = {name: _rl2(g, z[f"grad__{name}"]) for name, g in grads.items()}
    print(f"step {mode}{suffix}: loss rel err {loss_err:.2e}, max grad rel-L2 "
          f"{max(errs.values()):.2e}")
    assert loss_err <= LOSS_RTOL, (got, z["losses"][0])
    for name, e in errs.items():
        assert e <= GRAD_RL2, (name, e)
    if src is not None and mode in ("fraction",):
        frac = json.loads(str(z["fractions"]))
        for key, f in frac.items():
            l, c = key.split(":")
            assert src.last_fractions[(int(l), c)] == pytest.approx(f)
    # one Adam step (lr 1e-2), then the second loss of the reference trajectory
    opt = Adam(model.lora_param, lr=1e-2)
    opt.step()
    opt.zero_grad()
    with torch.no_grad():
        loss2, _ = model.forward_step(z["tokens"], pattern_source=src, segments=2)
    assert abs(float(loss2) - z["losses"][1]) <= LOSS_RTOL * abs(z["losses"][1])


@pytest.mark.parametrize("precision", ["bf16", "fp32"])
@pytest.mark.parametrize("suffix", ["", "_d128"])
@pytest.mark.parametrize("mode", ["predicted", "exact"])
def test_layer_masks_teacher_forced(cuda, mode, suffix, precision):
    """Feeding the reference's own per-layer input x_l to the GPU hook gives
    the reference's retained blocks (scores computed on the GPU), in the
    production bf16 scorers and the fp32-faithful parity precision."""
    z = np.load(G / f"patterns_{mode}{suffix}.npz")
    zs = np.load(G / f"step_{mode}{suffix}.npz")
    model, _ = _model_and_oracle(suffix, precision)
    src = _source(mode, model, zs)
    flips = 0
    for l in range(2):
        for c in (S.ATTENTION, S.MLP):
            x = torch.as_tensor(z[f"x_{l}_{c}"]).cuda()
            pat = src.pattern(l, c, x, 150)
            want = set(z[f"blocks_{l}_{c}"].tolist())
            flips += len(set(pat.retained_blocks) ^ want)
    assert flips == 0


@pytest.mark.parametrize("suffix", ["", "_d128"])
def test_all_retain_equals_dense_bitwise(cuda, suffix):
    """tests/test_model.py:186-191: all-retain patterns ≡ dense, bitwise."""
    z = np.load(G / f"step_dense{suffix}.npz")
    m1, _ = _model_and_oracle(suffix)
    l1, _ = m1.forward_step(z["tokens"], segments=2)
    l1.backward()
    m2, _ = _model_and_oracle(suffix)
    l2, _ = m2.forward_step(z["tokens"], pattern_source=M.AllRetainSource(), segments=2)
    l2.backward()
    assert float(l1) == float(l2)
    assert torch.equal(m1.lora_param.grad, m2.lora_param.grad)


def test_segment_count_invariance(cuda):
    """tests/test_kernels.py:190-211: N in {1,2,4,8} within 1e-6 (here: bf16 GEMM, fp32 CE)."""
    z = np.load(G / "step_dense.npz")
    losses = []
    for seg in (1, 2, 4, 8):
        m, _ = _model_and_oracle()
        with torch.no_grad():
            loss, _ = m.forward_step(z["tokens"], segments=seg)
        losses.append(float(loss))
    assert max(losses) - min(losses) <= 1e-5 * abs(losses[0])


def test_empty_pattern_is_identity(cuda):
    """k == 0 leaves the residual untouched (kernels.py:161-162)."""
    z = np.load(G / "step_dense.npz")
    m, om = _model_and_oracle()
    pats = {(l, c): S.SparsityPattern.empty(160, 16, l, c) for l in range(2)
            for c in (S.ATTENTION, S.MLP)}
    loss, _ = m.forward_step(z["tokens"], pattern_source=M.FixedPatternSource(pats), segments=2)
    ores = O.train_step(om, z["tokens"], source=O.FixedSource({k: () for k in pats}), segments=2)
    assert abs(float(loss) - ores["loss"]) <= 1e-3 * abs(ores["loss"])


@pytest.mark.parametrize("frac", [0.25, 0.5, 1.0])
def test_full_width_layer_vs_oracle(cuda, frac):
    """One Llama2-7B-width layer (h=4096, 32 heads, m=11008) at s=512 against
    the oracle with identical weights and patterns."""
    cfg = dict(n_layers=1, hidden_dim=4096, n_heads=32, vocab_size=512, max_seq_len=512,
               mlp_dim=11008, block_size=16, lora_rank=8, lora_alpha=16.0)
    om = O.init_model(O.Config(**cfg), seed=5)
    O.perturb_lora_b(om, 6)
    arrays = M.reference_init_arrays(M.ModelConfig(**cfg), 5)
    for name in om.adapter_names():
        arrays[name] = om.adapter(name)
    model = M.DecoderModel(M.ModelConfig(**cfg), 5, arrays=arrays)
    tokens = np.random.default_rng(7).integers(0, 512, 512)
    nb = 32
    keep = max(1, int(round(nb * frac)))
    blocks = tuple(np.unique(np.linspace(0, nb - 1, keep).round().astype(int)).tolist())
    oref = O.train_step(om, tokens, source=O.FixedSource({(0, c): blocks for c in ("attention", "mlp")}),
                        segments=2)
    src = M.FractionSource(frac, 16)
    loss, _ = model.forward_step(tokens, pattern_source=src, segments=2)
    loss.backward()
    assert abs(float(loss) - oref["loss"]) <= LOSS_RTOL * abs(oref["loss"])
    for name, g in model.adapter_grads().items():
        assert _rl2(g, oref["grads"][name]) <= GRAD_RL2, (name, _rl2(g, oref["grads"][name]))


def _oracle_arrays(om):
    arrays = {"embed": om.embed, "final_norm": om.final_norm, "lm_head": om.lm_head}
    for i, L in enumerate(om.layers):
        p = f"layer{i}"
        arrays.update({f"{p}.wq": L.wq, f"{p}.wk": L.wk, f"{p}.wv": L.wv, f"{p}.wo": L.wo,
                       f"{p}.attn_norm": L.attn_norm, f"{p}.mlp_norm": L.mlp_norm,
                       f"{p}.w_up": L.w_up, f"{p}.w_down": L.w_down, f"{p}.w_gate": L.w_gate,
                       f"{p}.lora_q.a": L.lora_q[0], f"{p}.lora_q.b": L.lora_q[1],
                       f"{p}.lora_v.a": L.lora_v[0], f"{p}.lora_v.b": L.lora_v[1]})
    return arrays


@pytest.mark.parametrize("mode", ["dense", "fraction"])
def test_gqa_step_matches_reference_repeated_heads(cuda, mode):
    """Grouped-query attention (4 query heads over 2 key/value heads) vs the
    reference run on the equivalent repeated-head MHA model (step_gqa.npz)."""
    z = np.load(G / "step_gqa.npz")
    cfg = dict(n_layers=2, hidden_dim=512, n_heads=4, vocab_size=256, max_seq_len=512,
               mlp_dim=344, block_size=16, lora_rank=8, lora_alpha=16.0, n_kv_heads=2)
    om = O.init_model(O.Config(**cfg), seed=5)
    O.perturb_lora_b(om, 6)
    model = M.DecoderModel(M.ModelConfig(**cfg), 0, arrays=_oracle_arrays(om))
    src = M.FractionSource(0.5, 16) if mode == "fraction" else None
    loss, _ = model.forward_step(z["tokens"], pattern_source=src, segments=2)
    loss.backward()
    ref_loss = float(z[f"{mode}_loss"])
    assert abs(float(loss.detach()) - ref_loss) <= LOSS_RTOL * abs(ref_loss)
    for name, g in model.adapter_grads().items():
        ref = z[f"{mode}_grad__{name}"]
        assert g.shape == ref.shape, name
        assert _rl2(g, ref) <= GRAD_RL2, (name, _rl2(g, ref))


@pytest.mark.parametrize("sink,pooling", [(False, "mean"), (True, "token")])
def test_full_width_predicted_step_refined(cuda, sink, pooling):
    """The bench's production path at the north-star width: 2 Llama2-7B-width
    layers (h=4096, 32 heads, m=11008), s=1024, PredictedPatternSource with
    recalibrated attention thresholds (model.py:545-563) and fixed MLP
    thresholds, `refined` scorers -- against the oracle's PredictedSource on
    the same weights, predictors (ranks 1024) and tokens: identical retained
    blocks for every (layer, component), loss and LoRA gradients within the
    bf16 tolerance.  Second case: the sink block forced and token pooling of
    the predictor outputs (predictor.py:126-173)."""
    cfg = dict(n_layers=2, hidden_dim=4096, n_heads=32, vocab_size=512, max_seq_len=1024,
               mlp_dim=11008, block_size=16, lora_rank=8, lora_alpha=16.0)
    om = O.init_model(O.Config(**cfg), seed=41, fast=True)
    O.perturb_lora_b(om, 42)
    model = M.DecoderModel(M.ModelConfig(**cfg), 0, arrays=_oracle_arrays(om),
                           scoring_precision="refined")
    prng = np.random.default_rng(43)
    ws = {l: [[(prng.standard_normal(sh, dtype=np.float32) / np.sqrt(sh[0])).astype(np.float32)
               for sh in ((4096, 1024), (1024, 1024), (1024, 1024))] for _ in range(2)]
          for l in range(2)}
    model.attach_predictors({l: (P.Predictor(*ws[l][0]), P.Predictor(*ws[l][1]))
                             for l in range(2)})
    for l in range(2):
        om.layers[l].predictor_q, om.layers[l].predictor_k = (O.Predictor(*ws[l][0]),
                                                              O.Predictor(*ws[l][1]))
    tokens = np.random.default_rng(44).integers(0, 512, 1024)
    # MLP thresholds: midpoints between neighbouring scores of a retain-all
    # profile near its mean (a tuned threshold is not itself a score)
    prof = O.ExactSource(om, None)
    O.train_step(om, tokens, source=prof, segments=2)
    thr = {}
    for l in range(2):
        v = np.sort(prof.vectors[(l, "mlp")])
        i = int(np.searchsorted(v, v.mean()))
        thr[(l, "mlp")] = float(0.5 * (v[i - 1] + v[i]))
        thr[(l, "attention")] = 0.0  # recalibrated at every call
    osrc = O.PredictedSource(om, dict(thr), target_retention={0: 0.5, 1: 0.5},
                             recalibrate_every=1, sink_first_block=sink, pooling=pooling)
    ores = O.train_step(om, tokens, source=osrc, segments=2)
    src = M.PredictedPatternSource(model, S.ThresholdSet(dict(thr)),
                                   target_retention={0: 0.5, 1: 0.5}, recalibrate_every=1,
                                   sink_first_block=sink, pooling=pooling)
    got, inner = {}, src.pattern

    def record(layer_id, component, x, n_valid):
        pat = inner(layer_id, component, x, n_valid)
        got[(layer_id, component)] = None if pat is None else tuple(pat.retained_blocks)
        return pat

    src.pattern = record
    loss, _ = model.forward_step(tokens, pattern_source=src, segments=2)
    loss.backward()
    errs = {n: _rl2(g, ores["grads"][n]) for n, g in model.adapter_grads().items()}
    print("full-width predicted step", json.dumps({
        "loss": float(loss), "oracle": ores["loss"], "grad_rl2": errs,
        "retained": {f"{l}_{c}": len(b) for (l, c), b in got.items()},
        "refined_rows": dict((f"{k}", v) for k, v in src.refined_rows.items())}))
    for key, blocks in ores["patterns"].items():
        assert got[key] == tuple(blocks), (key, got[key], blocks)
    assert abs(float(loss) - ores["loss"]) <= LOSS_RTOL * abs(ores["loss"])
    for n, e in errs.items():
        assert e <= GRAD_RL2, (n, e)


def test_refined_source_capacity_and_overflow(cuda):
    """PredictedPatternSource in the refined precision: the first step counts
    the refinement rows (exact path), later steps run on the per-layer
    capacity without that read-back, and a forced overflow (capacity below the
    band) falls back to the exact path -- the same patterns and the same loss
    every time."""
    z = np.load(G / "step_predicted_d128.npz")
    m, _ = _model_and_oracle("_d128", scoring_precision="refined")
    src = _source("predicted", m, z)
    got = []
    for trial in range(3):
        if trial == 2:
            for l in range(2):
                src._refine_cap.cap[l] = 1  # below any band: overflow -> exact re-run
        pats, inner = {}, src.pattern

        def record(layer_id, component, x, n_valid, inner=inner, pats=pats):
            pat = inner(layer_id, component, x, n_valid)
            pats[(layer_id, component)] = None if pat is None else tuple(pat.retained_blocks)
            return pat

        src.pattern = record
        with torch.no_grad():
            loss, _ = m.forward_step(z["tokens"], pattern_source=src, segments=2)
        src.pattern = inner
        got.append((pats, float(loss)))
        assert all(v >= 0 for v in src.refined_rows.values())
    assert got[0] == got[1] == got[2]
