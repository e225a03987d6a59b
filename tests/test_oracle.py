"""Pin the CPU oracle (oracle/lemo_oracle.py) to the reference.

1. Golden fixtures produced by running the reference itself
   (tests/golden/make_golden.py) — selection, quantile recalibration, column
   sums, predictor, scorers, whole training steps and per-layer masks.
2. The reference test-suite's own known-answer cases (cited by file:line).
"""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import lemo_oracle as O

G = Path(__file__).resolve().parent / "golden"

STEP_CFG = dict(n_layers=2, hidden_dim=128, n_heads=2, vocab_size=128, max_seq_len=256,
                mlp_dim=344, block_size=16, lora_rank=8, lora_alpha=16.0)
# "" = head_dim 64 (h=128), "_d128" = head_dim 128 (h=256): make_golden.STEP_VARIANTS
STEP_VARIANTS = {"": STEP_CFG, "_d128": dict(STEP_CFG, hidden_dim=256)}


def _split(flat, lens):
    out, o = [], 0
    for n in lens:
        out.append(flat[o:o + n])
        o += n
    return out


# ---------------------------------------------------------------- goldens


def test_select_golden():
    z = np.load(G / "select.npz")
    vecs = _split(z["vec"], z["vec_len"])
    masks = _split(z["mask"], z["vec_len"])
    toks = _split(z["tok"], z["tok_len"])
    for v, thr, sink, n, b, m, t in zip(vecs, z["thr"], z["sink"], z["n_tokens"], z["block"],
                                        masks, toks):
        blocks = O.eliminate(v, float(thr), (0,) if sink else ())
        assert blocks == tuple(np.nonzero(m)[0].tolist())
        np.testing.assert_array_equal(O.token_indices(blocks, int(b), int(n)), t)


def test_quantile_recalibration_golden():
    z = np.load(G / "quantile.npz")
    flat, o = z["vecs"], 0
    for nb, thr_seq, ret in zip(z["nb"], z["thr"], z["ret"]):
        src = O.PredictedSource(model=None, thresholds={}, target_retention={0: float(ret)},
                                recalibrate_every=1)
        for call in range(len(thr_seq)):
            v = flat[o:o + nb]
            o += nb
            src._maybe_recalibrate(0, v)
            got = src.thresholds[(0, O.ATTENTION)]
            assert got == thr_seq[call] or (np.isinf(got) and np.isinf(thr_seq[call]))


def test_column_sums_golden():
    z = np.load(G / "colsum.npz")
    nbs = list(z["nb"])
    packs = _split(z["packed"], [O.tri_size(n) for n in nbs])
    vecs = _split(z["vec"], nbs)
    for nb, p, v in zip(nbs, packs, vecs):
        np.testing.assert_array_equal(O.token_block_scores(p, nb), v)  # same order: bitwise
        d = np.zeros((nb, nb))
        r, c = np.tril_indices(nb)
        d[r, c] = p
        np.testing.assert_array_equal(O.column_sums_dense(d), v)


def _pred(z, side):
    return O.Predictor(z[f"{side}_w1"], z[f"{side}_w2"], z[f"{side}_w3"], z[f"{side}_m1"],
                       z[f"{side}_m2"])


def test_predictor_golden():
    z = np.load(G / "predictor.npz")
    pq, pk = _pred(z, "q"), _pred(z, "k")
    b = int(z["b"])
    np.testing.assert_allclose(O.block_embed(z["x"], b), z["block_embed"], rtol=1e-6, atol=1e-7)
    np.testing.assert_allclose(O.predicted_triangle(pq, pk, z["x"], b), z["packed"], rtol=1e-5,
                               atol=1e-6)
    np.testing.assert_allclose(O.predicted_triangle(pq, pk, z["x"], b, "token"),
                               z["packed_token"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(O.predicted_block_vector(pq, pk, z["x"], b), z["vec"], rtol=1e-5,
                               atol=1e-6)


def _scorer_layer(seed, **kw):
    cfg = O.Config(n_layers=1, hidden_dim=128, n_heads=2, vocab_size=64, max_seq_len=256,
                   block_size=16, **kw)
    return O.init_model(cfg, seed=seed).layers[0]


def test_scorers_golden():
    z = np.load(G / "scorers.npz")
    L = _scorer_layer(3, mlp_dim=344, lora_rank=4, lora_alpha=8.0)
    L.lora_q[1] = z["lora_q_b"]
    x, nv = z["x"], int(z["n_valid"])
    np.testing.assert_allclose(O.mlp_block_score_vector(L, x, 16, nv), z["mlp_vec"], rtol=1e-5)
    q, k = O.layer_qk(L, x)
    np.testing.assert_allclose(q, z["q"], rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(k, z["k"], rtol=1e-4, atol=1e-5)
    packed = O.exact_block_scores(z["q"], z["k"], 16, nv)
    np.testing.assert_allclose(packed, z["exact_packed"], rtol=1e-5, atol=1e-7)
    nb = O.n_blocks_for(x.shape[0], 16)
    np.testing.assert_allclose(O.token_block_scores(z["exact_packed"], nb), z["exact_vec"],
                               rtol=0, atol=0)
    zr = np.load(G / "scorers_relu.npz")
    Lr = _scorer_layer(4, mlp_dim=256, mlp_variant="relu")
    np.testing.assert_allclose(O.mlp_block_score_vector(Lr, zr["x"], 16, nv), zr["mlp_vec"],
                               rtol=1e-5)


def step_model(mode, suffix=""):
    z = np.load(G / f"step_{mode}{suffix}.npz")
    model = O.init_model(O.Config(**STEP_VARIANTS[suffix]), seed=17)
    O.perturb_lora_b(model, 23)
    source = None
    if mode == "fraction":
        nb = O.n_blocks_for(160, 16)
        keep = max(1, int(round(nb * 0.5)))
        blocks = tuple(np.unique(np.linspace(0, nb - 1, keep).round().astype(int)).tolist())
        source = O.FixedSource({(l, c): blocks for l in range(2) for c in (O.ATTENTION, O.MLP)})
    elif mode in ("predicted", "exact"):
        thr = {(l, c): float(z[f"thr_{l}_{c}"]) for l in range(2) for c in (O.ATTENTION, O.MLP)}
        if mode == "exact":
            source = O.ExactSource(model, thr)
        else:
            for l in range(2):
                model.layers[l].predictor_q = O.Predictor(
                    z[f"pred{l}_q_w1"], z[f"pred{l}_q_w2"], z[f"pred{l}_q_w3"])
                model.layers[l].predictor_k = O.Predictor(
                    z[f"pred{l}_k_w1"], z[f"pred{l}_k_w2"], z[f"pred{l}_k_w3"])
            source = O.PredictedSource(model, dict(thr), target_retention={0: 0.5, 1: 0.5},
                                       recalibrate_every=1)
    return z, model, source


@pytest.mark.parametrize("suffix", ["", "_d128"])
@pytest.mark.parametrize("mode", ["dense", "fraction", "predicted", "exact"])
def test_train_step_golden(mode, suffix):
    z, model, source = step_model(mode, suffix)
    res = O.train_step(model, z["tokens"], source=source, segments=2, return_hidden=True)
    np.testing.assert_allclose(res["loss"], z["losses"][0], rtol=2e-6)
    np.testing.assert_allclose(res["hidden"], z["hidden"], rtol=1e-4, atol=1e-5)
    for name in model.adapter_names():
        ref = z[f"grad__{name}"]
        got = res["grads"][name]
        tol = 1e-4 * np.abs(ref).max() + 1e-9
        assert np.abs(got - ref).max() <= tol, (name, np.abs(got - ref).max(), tol)
    # one Adam step (optim.py:37-53, lr 1e-2) then the second loss
    params = {n: model.adapter(n) for n in model.adapter_names()}
    O.adam_step(params, res["grads"], {}, lr=1e-2)
    res2 = O.train_step(model, z["tokens"], source=source, segments=2)
    np.testing.assert_allclose(res2["loss"], z["losses"][1], rtol=1e-5)
    if source is not None and mode != "fraction":
        frac = json.loads(str(z["fractions"]))
        for key, f in frac.items():
            l, c = key.split(":")
            pat = res2["patterns"][(int(l), c)]
            got = 1.0 if pat is None else len(O.token_indices(pat, 16, 160)) / 160
            assert got == pytest.approx(f)


@pytest.mark.parametrize("suffix", ["", "_d128"])
@pytest.mark.parametrize("mode", ["predicted", "exact"])
def test_layer_patterns_golden(mode, suffix):
    """Teacher-forced per-layer masks: feeding the reference's own layer input
    x_l to the oracle's scorer reproduces the reference's retained blocks."""
    z = np.load(G / f"patterns_{mode}{suffix}.npz")
    _, model, source = step_model(mode, suffix)
    for l in range(2):
        for c in (O.ATTENTION, O.MLP):
            x = z[f"x_{l}_{c}"]
            got = source.pattern(l, c, x, 150)
            want = tuple(z[f"blocks_{l}_{c}"].tolist())
            assert got == want, (l, c, got, want)


# -------------------------------------------- reference known-answer tests


def test_token_block_scores_known_answer():
    # tests/test_sparsity.py:121-123
    np.testing.assert_array_equal(O.token_block_scores([1.0, 2.0, 5.0], 2), [3.0, 5.0])


def test_last_block_is_diagonal():
    # tests/test_sparsity.py:126-132: last column sum == the diagonal entry
    nb = 6
    p = np.arange(1, O.tri_size(nb) + 1, dtype=np.float64)
    v = O.token_block_scores(p, nb)
    assert v[-1] == p[O.tri_index(nb - 1, nb - 1)]


def test_eliminate_known_answers():
    # tests/test_sparsity.py:135-156
    v = np.array([3.0, 5.0])
    assert O.eliminate(v, float("-inf")) == (0, 1)
    assert O.eliminate(v, 6.0) == ()
    assert O.eliminate(v, 4.0) == (1,)
    np.testing.assert_array_equal(O.token_indices((1,), 2, 4), [2, 3])
    assert O.eliminate(v, 4.0, (0,)) == (0, 1)


def test_eliminate_monotone():
    # tests/test_sparsity.py:159-168
    rng = np.random.default_rng(0)
    v = rng.random(50)
    prev = None
    for t in np.sort(rng.random(20)):
        cur = set(O.eliminate(v, t))
        if prev is not None:
            assert cur <= prev
        prev = cur


def test_token_indices_known_answers():
    # tests/test_sparsity.py:202-209
    np.testing.assert_array_equal(O.token_indices((0, 2), 4, 12), [0, 1, 2, 3, 8, 9, 10, 11])
    np.testing.assert_array_equal(O.token_indices((2,), 4, 10), [8, 9])  # ragged tail


def test_mlp_known_answers():
    # tests/test_sparsity.py:230-248
    inner = np.array([[-4.0, 8.0]])
    assert np.abs(inner).mean(axis=-1)[0] == 6.0
    np.testing.assert_array_equal(O.mlp_block_scores([1, 5, 2, 0.5], 2), [5, 2])


def test_zero_qk_scores_zero():
    # tests/test_sparsity.py:17-20
    q = np.zeros((2, 32, 8))
    assert O.exact_block_scores(q, q, 8).max() == 0.0


def test_exact_matches_brute_force():
    # tests/test_sparsity.py:23-28, 53-65 (1e-12 in f64)
    rng = np.random.default_rng(4)
    q = rng.standard_normal((3, 40, 8))
    k = rng.standard_normal((3, 40, 8))
    full = np.einsum("hid,hjd->hij", q, k)
    agg = np.maximum(full, 0).sum(0) / 3
    agg = np.where(np.tril(np.ones((40, 40), dtype=bool)), agg, 0)
    dense = O.exact_block_dense(q, k, 8)
    for m in range(5):
        for n in range(m + 1):
            assert abs(dense[m, n] - agg[8 * m:8 * m + 8, 8 * n:8 * n + 8].max()) < 1e-12


def test_attention_matches_dense_oracle():
    # tests/test_tensor.py:300-317 / tests/oracles.py:10-24
    rng = np.random.default_rng(8)
    q, k, v = (rng.standard_normal((20, 8)) for _ in range(3))
    out, _ = O.causal_attention_fwd(q, k, v, 2)
    ref = []
    for hd in range(2):
        sl = slice(4 * hd, 4 * hd + 4)
        s = q[:, sl] @ k[:, sl].T / 2.0
        s = np.where(np.tril(np.ones((20, 20), dtype=bool)), s, -np.inf)
        p = np.exp(s - s.max(-1, keepdims=True))
        ref.append((p / p.sum(-1, keepdims=True)) @ v[:, sl])
    np.testing.assert_allclose(out, np.concatenate(ref, 1), rtol=1e-12, atol=1e-12)


def test_attention_bwd_finite_difference():
    # gradient check in float64 (tests/test_tensor.py:194-293 methodology)
    rng = np.random.default_rng(9)
    q, k, v = (rng.standard_normal((12, 8)) for _ in range(3))
    g = rng.standard_normal((12, 8))
    out, lse = O.causal_attention_fwd(q, k, v, 2)
    dq, dk, dv = O.causal_attention_bwd(g, q, k, v, out, lse, 2)
    eps = 1e-6
    for arr, grad in ((q, dq), (k, dk), (v, dv)):
        for i in [(0, 0), (5, 3), (11, 7)]:
            old = arr[i]
            arr[i] = old + eps
            fp = (O.causal_attention_fwd(q, k, v, 2)[0] * g).sum()
            arr[i] = old - eps
            fm = (O.causal_attention_fwd(q, k, v, 2)[0] * g).sum()
            arr[i] = old
            assert abs((fp - fm) / (2 * eps) - grad[i]) < 1e-6


def test_quantile_lower_rule():
    # numpy 'lower' = sorted[floor((n-1) q)] (model.py:562)
    rng = np.random.default_rng(1)
    for n in (1, 2, 7, 100):
        a = rng.standard_normal(n)
        for q in (0.0, 0.1, 0.5, 0.999, 1.0):
            assert O.quantile_lower(a, q) == np.quantile(a, q, method="lower")


def test_oracle_gqa_matches_reference_on_repeated_heads():
    """GQA is an extension; the reference pins it through the equivalent MHA
    model with repeated K/V (and LoRA B_v) head blocks (make_golden.gqa_case)."""
    z = np.load(G / "step_gqa.npz")
    cfg = dict(n_layers=2, hidden_dim=512, n_heads=4, vocab_size=256, max_seq_len=512,
               mlp_dim=344, block_size=16, lora_rank=8, lora_alpha=16.0, n_kv_heads=2)
    for mode in ("dense", "fraction"):
        om = O.init_model(O.Config(**cfg), seed=5)
        O.perturb_lora_b(om, 6)
        src = None
        if mode == "fraction":  # FractionSource(0.5, 16) on the padded 304 tokens
            nb = O.n_blocks_for(304, 16)
            keep = max(1, int(round(nb * 0.5)))
            blocks = tuple(np.unique(np.linspace(0, nb - 1, keep).round().astype(int)).tolist())
            src = O.FixedSource({(l, c): blocks for l in range(2) for c in (O.ATTENTION, O.MLP)})
        ref = O.train_step(om, z["tokens"], source=src, segments=2)
        assert abs(ref["loss"] - float(z[f"{mode}_loss"])) <= 1e-5 * abs(float(z[f"{mode}_loss"]))
        for name, g in ref["grads"].items():
            r = z[f"{mode}_grad__{name}"]
            assert g.shape == r.shape, name
            assert np.linalg.norm(g - r) <= 1e-4 * max(np.linalg.norm(r), 1e-30), name
