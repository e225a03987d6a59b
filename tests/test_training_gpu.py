"""GPU parity of the offline stages next to the hot path:
predictor training (fit_predictors) against the reference's own run, loading
reference-written predictors.ckpt, teacher generation and Algorithm 1 tuning
through the sparse forward.  Fixtures: tests/golden/make_golden.py."""

import math
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2501_09767_b200 import artifacts as A
from paper_2501_09767_b200 import model as M
from paper_2501_09767_b200 import pipeline
from paper_2501_09767_b200 import predictor as P
from paper_2501_09767_b200 import sparsity as S

G = Path(__file__).resolve().parent / "golden"
pytestmark = pytest.mark.gpu


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


@pytest.mark.parametrize("pooling", ["mean", "token"])
def test_fit_predictors_matches_reference(cuda, pooling):
    z = np.load(G / ("predictor_train.npz" if pooling == "mean" else f"predictor_train_{pooling}.npz"))
    pairs = {}
    for l in range(2):
        pair = []
        for role in ("q", "k"):
            p = P.Predictor(z[f"init_{l}_{role}_w1"], z[f"init_{l}_{role}_w2"],
                            z[f"init_{l}_{role}_w3"], role, l, cuda)
            pair.append(p)
        pairs[l] = tuple(pair)
    records = []
    for i in range(4):
        records.append(P.TeacherRecord(int(z[f"layer_{i}"][0]),
                                       torch.as_tensor(z[f"x_{i}"]).to(cuda),
                                       torch.as_tensor(z[f"teacher_{i}"]).to(cuda), 128, 8))
    hist = P.fit_predictors(pairs, records, epochs=6, lr=1e-2, val_data=records,
                            prune_target=0.6, prune_every=2, prune_step=0.2, eval_every=3,
                            pooling=pooling)
    loss = np.array([h.train_loss for h in hist])
    assert np.allclose(loss, z["loss"], rtol=1e-3, atol=0), (loss, z["loss"])
    assert [h.param_count for h in hist] == z["params"].tolist()
    rec = np.array([h.recall for h in hist])
    assert np.array_equal(np.isnan(rec), np.isnan(z["recall"]))
    assert np.allclose(rec[~np.isnan(rec)], z["recall"][~np.isnan(z["recall"])], atol=0.1)
    for l, pq in pairs.items():
        for p in pq:
            st = p.state_arrays()
            for name in ("mask1", "mask2", "zero_counts1", "zero_counts2", "observed"):
                assert np.array_equal(st[name], z[f"final_{l}_{p.role}_{name}"]), (l, p.role, name)
            for name in ("w1", "w2", "w3"):
                assert _rel(st[name], z[f"final_{l}_{p.role}_{name}"]) < 2e-3, (l, p.role, name)


def test_fit_predictors_divergence_leaves_weights_finite(cuda):
    """A non-finite record loss raises ContractError and no NaN/Inf update
    reaches the caller's predictors (the reference checks every loss before
    stepping, predictor.py:405-410; here Adam is guarded on the device)."""
    from paper_2501_09767_b200.errors import ContractError

    rng = np.random.default_rng(3)
    pairs = {0: (P.Predictor.create(rng, 64, 16, 16, 16, "q", 0, cuda),
                 P.Predictor.create(rng, 64, 16, 16, 16, "k", 0, cuda))}
    before = [w.clone() for p in pairs[0] for w in p.parameters()]
    x = torch.randn(128, 64, device=cuda)
    bad = torch.full((16 * 17 // 2,), float("nan"), dtype=torch.float64, device=cuda)
    good = torch.rand(16 * 17 // 2, dtype=torch.float64, device=cuda)
    recs = [P.TeacherRecord(0, x, bad, 128, 8), P.TeacherRecord(0, x, good, 128, 8)]
    with pytest.raises(ContractError):
        P.fit_predictors(pairs, recs, epochs=2, lr=1e-2)
    after = [w for p in pairs[0] for w in p.parameters()]
    for a, b in zip(after, before):
        assert torch.equal(a, b)  # the NaN record and every later one were skipped


def test_load_reference_predictors_ckpt(cuda):
    z = np.load(G / "artifacts.npz")
    pairs, pt, retention, meta = A.load_predictors(G / "predictors.ckpt", n_layers=2,
                                                   hidden_dim=64, cfg_hash=str(z["hash"][0]),
                                                   device=cuda)
    assert retention == {0: 0.5, 1: 0.4} and pt.get(0, "attention") == 1.25
    tensors, _, _ = A.load_container(G / "predictors.ckpt")
    for l, (p_q, p_k) in pairs.items():
        for p in (p_q, p_k):
            for name, arr in p.state_arrays().items():
                assert np.array_equal(arr, tensors[f"pred/L{l}/{p.role}/{name}"]), name
        vec = P.predicted_block_vector(p_q, p_k, torch.as_tensor(z["x"]).to(cuda), 8)
        ref = z[f"vec_{l}"]
        assert float((vec.cpu() - torch.as_tensor(ref)).abs().max()) <= 1e-5 * max(
            float(np.abs(ref).max()), 1.0)
    # written back through our writer: the reference's own bytes
    out = Path("/tmp") / f"lemo_pred_{torch.cuda.current_device()}.ckpt"
    A.save_predictors(out, pairs, pt, retention, cfg_hash=meta["config_hash"])
    t2, _, m2 = A.load_container(out)
    assert set(t2) == set(tensors) and all(np.array_equal(t2[k], tensors[k]) for k in t2)
    assert m2 == meta


def _tiny_model(cuda):
    cfg = M.ModelConfig(n_layers=2, hidden_dim=256, n_heads=2, vocab_size=256, max_seq_len=512,
                        mlp_dim=688, block_size=16, lora_rank=8, lora_alpha=16.0)
    return M.DecoderModel(cfg, 3, device=cuda)


def test_teacher_generation_training_and_threshold_init(cuda):
    model = _tiny_model(cuda)
    rng = np.random.default_rng(0)
    seqs = [rng.integers(0, 256, 256) for _ in range(3)]
    records = pipeline.collect_teacher_records(model, seqs, 2)
    assert len(records) == 2 * 2 and {r.layer_id for r in records} == {0, 1}
    nb = 256 // 16
    for r in records:
        assert r.teacher_packed.numel() == nb * (nb + 1) // 2
        assert r.x.shape == (256, 256) and bool(torch.isfinite(r.x).all())
    # teacher rows agree with the retain-all exact scorer of the same input
    q, k = M.layer_qk(model.layers[0], records[0].x)
    from paper_2501_09767_b200 import exact
    vec = exact.exact_block_vector(q, k, 16, n_heads=2)
    vec2 = S.token_block_scores(S.BlockScoreMatrix(nb, 16, records[0].teacher_packed))
    assert torch.equal(vec, vec2)
    pairs = pipeline.create_pairs(model, 64, 64, 64, seed=1)
    hist = P.fit_predictors(pairs, records, epochs=8, lr=1e-2, val_data=records[:2],
                            prune_target=0.8, prune_every=4, eval_every=4)
    assert hist[-1].train_loss < hist[0].train_loss
    assert all(math.isfinite(h.train_loss) for h in hist)
    exact_thr = S.ThresholdSet({(l, S.ATTENTION): 0.0 for l in range(2)})
    for l in range(2):
        vecs = [S.token_block_scores(S.BlockScoreMatrix(nb, 16, r.teacher_packed))
                for r in records if r.layer_id == l]
        exact_thr.set(l, S.ATTENTION, float(torch.cat(vecs).mean()))
    pt, retention = pipeline.predicted_threshold_init(pairs, records, exact_thr)
    assert set(pt.values) == {(0, S.ATTENTION), (1, S.ATTENTION)}
    assert all(0.0 < r <= 1.0 for r in retention.values())
    model.attach_predictors(pairs)
    src = M.PredictedPatternSource(model, pt, mlp_scoring=False)
    loss, _ = model.forward_step(seqs[2], pattern_source=src)
    assert math.isfinite(float(loss.detach()))


def test_tune_thresholds_through_sparse_forward(cuda):
    model = _tiny_model(cuda)
    rng = np.random.default_rng(1)
    seqs = [rng.integers(0, 256, 256) for _ in range(2)]
    prof = M.ExactPatternSource(model, None, record=True)
    with torch.no_grad():
        model.forward_step(seqs[0], pattern_source=prof)
    ts = S.init_thresholds(prof.recorded_vectors)
    calls = []
    orig = pipeline.mean_eval_loss

    def counting(*a, **kw):
        calls.append(1)
        return orig(*a, **kw)

    pipeline.mean_eval_loss = counting
    try:
        tuned = pipeline.tune_thresholds(model, ts, seqs, limit=2, rounds=1)
    finally:
        pipeline.mean_eval_loss = orig
    assert len(calls) == 2 * len(ts.values)
    assert set(tuned.values) == set(ts.values)
    assert all(math.isfinite(v) for v in tuned.values.values())
    # one round moves each threshold by at most 10 % of |T| + 1e-3 (auto eta)
    for key, v in ts.values.items():
        assert abs(tuned.values[key] - v) <= 0.1 * (abs(v) + 1e-3) + 1e-12
