"""Per-kernel parity of liblemo against the oracle / a plain fp32 torch reference."""

import math
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import lemo_oracle as O
from paper_2501_09767_b200 import ops, predictor as P, sparsity as S
from paper_2501_09767_b200.model import DecoderModel, ModelConfig, mlp_block_score_vector, layer_qk
from paper_2501_09767_b200 import exact

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def _split(flat, lens):
    out, o = [], 0
    for n in lens:
        out.append(flat[o:o + n])
        o += n
    return out


# ------------------------------------------------------------------ selection


def test_select_bit_exact_on_reference_scores(cuda):
    """Given the reference's own score vectors and thresholds, retained blocks
    and token indices are bit-identical (sparsity.py:263-281, 95-104)."""
    z = np.load(G / "select.npz")
    vecs = _split(z["vec"], z["vec_len"])
    masks = _split(z["mask"], z["vec_len"])
    toks = _split(z["tok"], z["tok_len"])
    for v, thr, sink, n, b, m, t in zip(vecs, z["thr"], z["sink"], z["n_tokens"], z["block"],
                                        masks, toks):
        pat = S.eliminate(v, float(thr), block_size=int(b), n_tokens=int(n),
                          force_blocks=(0,) if sink else ())
        assert pat.retained_blocks == tuple(np.nonzero(m)[0].tolist())
        np.testing.assert_array_equal(pat.token_indices, t)
        assert pat.k == len(t)


def test_select_rejects_nonfinite(cuda):
    from paper_2501_09767_b200.errors import ContractError
    with pytest.raises(ContractError):
        S.eliminate(np.array([1.0, np.nan, 2.0]), 0.5, block_size=4, n_tokens=12)
    with pytest.raises(ContractError):
        S.eliminate(np.array([1.0, np.inf]), 0.5, block_size=4, n_tokens=8)


def test_select_large_random(cuda):
    rng = np.random.default_rng(3)
    for nb in (1, 1023, 1024, 1025, 4096, 5000):
        v = rng.integers(0, 50, nb).astype(np.float64) * 0.25
        thr = float(np.quantile(v, 0.5, method="lower"))
        pat = S.eliminate(v, thr, block_size=16, n_tokens=nb * 16 - 5)
        assert pat.retained_blocks == O.eliminate(v, thr)
        np.testing.assert_array_equal(pat.token_indices,
                                      O.token_indices(O.eliminate(v, thr), 16, nb * 16 - 5))


def test_quantile_recalibration_bit_exact(cuda):
    z = np.load(G / "quantile.npz")
    flat, o = z["vecs"], 0
    for nb, thr_seq, ret in zip(z["nb"], z["thr"], z["ret"]):
        recent = []
        for call in range(len(thr_seq)):
            v = flat[o:o + nb]
            o += nb
            recent.append(v)
            recent = recent[-8:]
            got = P.quantile_threshold(torch.as_tensor(np.concatenate(recent)).cuda(), float(ret))
            assert got == thr_seq[call] or (np.isinf(got) and np.isinf(thr_seq[call]))


def test_colsum_golden(cuda):
    z = np.load(G / "colsum.npz")
    nbs = list(z["nb"])
    for nb, p, v in zip(nbs, _split(z["packed"], [O.tri_size(n) for n in nbs]), _split(z["vec"], nbs)):
        d = np.zeros((nb, nb), np.float32)
        r, c = np.tril_indices(nb)
        d[r, c] = p
        got = ops.colsum_clamped(torch.as_tensor(d).cuda()).cpu().numpy()
        np.testing.assert_array_equal(got, v)  # same f64 order: bitwise


# ------------------------------------------------------------------ predictor


def test_block_embed_bitwise(cuda):
    z = np.load(G / "predictor.npz")
    got = ops.block_embed(torch.as_tensor(z["x"]).cuda(), int(z["b"])).cpu().numpy()
    np.testing.assert_array_equal(got, z["block_embed"])


def test_predictor_golden(cuda):
    z = np.load(G / "predictor.npz")
    pq = P.Predictor(z["q_w1"], z["q_w2"], z["q_w3"])
    pq.set_masks(z["q_m1"], z["q_m2"])
    pk = P.Predictor(z["k_w1"], z["k_w2"], z["k_w3"])
    pk.set_masks(z["k_m1"], z["k_m2"])
    x = torch.as_tensor(z["x"]).cuda()
    b = int(z["b"])
    # fp32-faithful bf16x3 products: |err| <= 1e-5 of the output scale
    scale = np.abs(z["packed"]).max()
    np.testing.assert_allclose(P.predicted_triangle(pq, pk, x, b).cpu().numpy(), z["packed"],
                               rtol=1e-5, atol=1e-5 * scale)
    np.testing.assert_allclose(P.predicted_triangle(pq, pk, x, b, "token").cpu().numpy(),
                               z["packed_token"], rtol=1e-5, atol=1e-5 * scale)
    np.testing.assert_allclose(P.predicted_block_vector(pq, pk, x, b).cpu().numpy(), z["vec"],
                               rtol=1e-5, atol=1e-5 * np.abs(z["vec"]).max())
    # Predictor.forward(x, track) (predictor.py:73-81) ≡ predict, and track=True
    # counts exact zeros of both hidden stages (pruned neurons always count)
    xb = P.block_embed(x, b)
    out = pq.forward(xb, track=True)
    torch.testing.assert_close(out, pq.predict(xb), rtol=0, atol=0)
    assert pq.observed == xb.shape[0]
    op = O.Predictor(z["q_w1"], z["q_w2"], z["q_w3"], z["q_m1"].astype(bool),
                     z["q_m2"].astype(bool))
    xbn = xb.cpu().numpy()
    h1 = np.maximum(xbn @ op.w1, 0) * op.mask1
    h2 = np.maximum(h1 @ op.w2, 0) * op.mask2
    assert np.abs(pq.zero_counts1.cpu().numpy() - (h1 == 0).sum(0)).max() <= 1
    assert np.abs(pq.zero_counts2.cpu().numpy() - (h2 == 0).sum(0)).max() <= 1
    # predict_scores (predictor.py:189-212): clamped Eq. 3 dots, block_size 1
    bsm = P.predict_scores(pq, pk, xb)
    full = op.predict(xbn) @ O.Predictor(z["k_w1"], z["k_w2"], z["k_w3"], z["k_m1"].astype(bool),
                                         z["k_m2"].astype(bool)).predict(xbn).T
    r, c = np.tril_indices(full.shape[0])
    ref = np.maximum(full[r, c], 0.0)
    assert bsm.block_size == 1 and bsm.n_blocks == full.shape[0]
    np.testing.assert_allclose(bsm.scores.cpu().numpy(), ref, rtol=1e-4, atol=5e-5 * ref.max())


# ------------------------------------------------------------------ scorers


def _scorer_model(seed, **kw):
    cfg = ModelConfig(n_layers=1, hidden_dim=128, n_heads=2, vocab_size=64, max_seq_len=256,
                      block_size=16, **kw)
    ocfg = O.Config(n_layers=1, hidden_dim=128, n_heads=2, vocab_size=64, max_seq_len=256,
                    block_size=16, **kw)
    om = O.init_model(ocfg, seed=seed)
    return DecoderModel(cfg, seed, init="reference"), om


@pytest.mark.parametrize("nb,h,r", [(96, 256, 64), (1024, 512, 256)])
def test_pair_first_layer_equals_separate(cuda, nb, h, r):
    """Both predictors' first layers as one stacked bf16x3 GEMM (CTA-pair
    tiles when nb spans two row tiles) == the two separate layer GEMMs, with
    distinct masks; and the predicted block vector through it matches the
    per-predictor path."""
    g = torch.Generator(device="cuda").manual_seed(3)
    mk = lambda: P.Predictor(*(torch.randn(a, b, generator=g, device="cuda") / math.sqrt(a)  # noqa
                               for a, b in ((h, r), (r, r), (r, r))))
    pq, pk = mk(), mk()
    pq.set_masks(np.arange(r) % 7 != 3, np.ones(r, bool))
    pk.set_masks(np.arange(r) % 5 != 1, np.ones(r, bool))
    x3 = ops.split_bf16x3(torch.randn(nb, h, device="cuda"), 0)
    hq, hk = P.pair_hidden1(pq, pk, x3)
    sq, _ = ops.gemm_split3(x3, pq._weights3()[0], relu=True, mask=pq.mask1, pattern=0)
    sk, _ = ops.gemm_split3(x3, pk._weights3()[0], relu=True, mask=pk.mask1, pattern=0)
    for got, ref in ((hq, sq), (hk, sk)):
        a = got[:, :r].float() + got[:, 2 * r:].float()
        b = ref[:, :r].float() + ref[:, 2 * r:].float()
        torch.testing.assert_close(a, b, rtol=2e-6, atol=2e-6 * float(b.abs().max()))
    x = torch.randn(nb * 16, h, device="cuda")
    v = P.predicted_block_vector(pq, pk, x, 16)
    xb3 = ops.split_bf16x3(P.block_embed(x, 16), 0)
    ref = ops.colsum_clamped(ops.gemm_f32_exact(pq.predict3(xb3, 0), pk.predict3(xb3, 1)))
    torch.testing.assert_close(v, ref, rtol=1e-5, atol=1e-5 * float(ref.abs().max()))


def test_mlp_scores_golden(cuda):
    z = np.load(G / "scorers.npz")
    m, _ = _scorer_model(3, mlp_dim=344, lora_rank=4, lora_alpha=8.0)
    x = torch.as_tensor(z["x"]).cuda()
    got = mlp_block_score_vector(m.layers[0], x, 16, int(z["n_valid"])).cpu().numpy()
    # bf16 GEMM operands: token scores are means over m products -> ~1e-3 relative
    np.testing.assert_allclose(got, z["mlp_vec"], rtol=2e-2)
    zr = np.load(G / "scorers_relu.npz")
    mr, _ = _scorer_model(4, mlp_dim=256, mlp_variant="relu")
    got = mlp_block_score_vector(mr.layers[0], x, 16, int(zr["n_valid"])).cpu().numpy()
    np.testing.assert_allclose(got, zr["mlp_vec"], rtol=2e-2)


def test_exact_scores_golden(cuda):
    z = np.load(G / "scorers.npz")
    H, s, d = z["q"].shape
    q = torch.as_tensor(z["q"].transpose(1, 0, 2).reshape(s, H * d)).cuda().bfloat16()
    k = torch.as_tensor(z["k"].transpose(1, 0, 2).reshape(s, H * d)).cuda().bfloat16()
    nv = int(z["n_valid"])
    bsm = exact.exact_block_scores(q, k, 16, n_heads=H, n_valid=nv)
    ref = z["exact_packed"]
    np.testing.assert_allclose(bsm.scores.cpu().numpy(), ref, rtol=2e-2, atol=2e-2 * ref.max())
    vec = exact.exact_block_vector(q, k, 16, n_heads=H, n_valid=nv).cpu().numpy()
    np.testing.assert_allclose(vec, z["exact_vec"], rtol=2e-2)


def test_layer_qk_matches_oracle(cuda):
    z = np.load(G / "scorers.npz")
    m, om = _scorer_model(3, mlp_dim=344, lora_rank=4, lora_alpha=8.0)
    m.layers[0].lora_q.b.copy_(torch.as_tensor(z["lora_q_b"]))
    x = torch.as_tensor(z["x"]).cuda()
    q, k = layer_qk(m.layers[0], x)
    H, s, d = z["q"].shape
    qref = z["q"].transpose(1, 0, 2).reshape(s, H * d)
    kref = z["k"].transpose(1, 0, 2).reshape(s, H * d)
    np.testing.assert_allclose(q.float().cpu().numpy(), qref, rtol=3e-2, atol=3e-2)
    np.testing.assert_allclose(k.float().cpu().numpy(), kref, rtol=3e-2, atol=3e-2)


# fp32-faithful (parity) precision: bf16x3 operands, fp32 element-wise steps


def _scorer_model_fp32(seed, **kw):
    cfg = ModelConfig(n_layers=1, hidden_dim=128, n_heads=2, vocab_size=64, max_seq_len=256,
                      block_size=16, **kw)
    return DecoderModel(cfg, seed, init="reference", scoring_precision="fp32")


def test_mlp_scores_golden_fp32(cuda):
    z = np.load(G / "scorers.npz")
    m = _scorer_model_fp32(3, mlp_dim=344, lora_rank=4, lora_alpha=8.0)
    x = torch.as_tensor(z["x"]).cuda()
    got = mlp_block_score_vector(m.layers[0], x, 16, int(z["n_valid"])).cpu().numpy()
    np.testing.assert_allclose(got, z["mlp_vec"], rtol=1e-5)
    zr = np.load(G / "scorers_relu.npz")
    mr = _scorer_model_fp32(4, mlp_dim=256, mlp_variant="relu")
    got = mlp_block_score_vector(mr.layers[0], x, 16, int(zr["n_valid"])).cpu().numpy()
    np.testing.assert_allclose(got, zr["mlp_vec"], rtol=1e-5)


def test_parity_weights_keep_bf16_default(cuda):
    """parity_weights=True only enables the fp32 precision per call: the
    sources' default (scoring_precision) stays the production bf16 scorer."""
    z = np.load(G / "scorers.npz")
    cfg = ModelConfig(n_layers=1, hidden_dim=128, n_heads=2, vocab_size=64, max_seq_len=256,
                      block_size=16, mlp_dim=344, lora_rank=4, lora_alpha=8.0)
    m = DecoderModel(cfg, 3, init="reference", parity_weights=True)
    x = torch.as_tensor(z["x"]).cuda()
    nv = int(z["n_valid"])
    default = mlp_block_score_vector(m.layers[0], x, 16, nv)
    bf16 = mlp_block_score_vector(m.layers[0], x, 16, nv, precision="bf16")
    fp32 = mlp_block_score_vector(m.layers[0], x, 16, nv, precision="fp32")
    assert torch.equal(default, bf16) and not torch.equal(default, fp32)
    np.testing.assert_allclose(fp32.cpu().numpy(), z["mlp_vec"], rtol=1e-5)


@pytest.mark.parametrize("margin", [2e-3, 5e-2])
def test_refined_mlp_decisions_equal_parity(cuda, margin):
    """Token-level refinement (refine_mlp_block_scores): bf16 block scores,
    then only the rows that can decide a near-threshold block re-scored in the
    parity precision -> the same >= decisions as the fp32 scorer at every
    threshold tried; a wide margin (5e-2) re-scores many rows and must agree
    too, and every re-scored block that is retained carries its fp32 score (its
    maximum row is among the re-scored ones)."""
    from paper_2501_09767_b200.model import refine_mlp_block_scores
    cfg = ModelConfig(n_layers=1, hidden_dim=256, n_heads=2, vocab_size=64, max_seq_len=1024,
                      block_size=16, mlp_dim=688, lora_rank=4, lora_alpha=8.0)
    m = DecoderModel(cfg, 5, init="reference", parity_weights=True)
    L = m.layers[0]
    x = torch.randn(1024, 256, device="cuda")
    nv = 1024 - 5
    fp32 = mlp_block_score_vector(L, x, 16, nv, precision="fp32")
    total = 0
    for q in (0.3, 0.5, 0.7):
        thr = float(torch.quantile(fp32, q))
        vec, part = mlp_block_score_vector(L, x, 16, nv, precision="bf16", with_partial=True)
        before = vec.clone()
        rows = refine_mlp_block_scores(L, x, vec, part, thr, 16, nv, margin=margin)
        total += rows
        assert torch.equal(vec >= thr, fp32 >= thr), (q, margin, rows)
        touched = (vec != before) & (vec >= thr)
        np.testing.assert_allclose(vec[touched].cpu().numpy(), fp32[touched].cpu().numpy(),
                                   rtol=2e-6)
        # blocks outside the band are left as scored
        far = (before - thr).abs() > margin * abs(thr)
        assert torch.equal(vec[far], before[far])
    assert total > 0
    for thr in (float("-inf"), float("inf")):  # nothing ambiguous: no rows, scores untouched
        vec, part = mlp_block_score_vector(L, x, 16, nv, precision="bf16", with_partial=True)
        before = vec.clone()
        assert refine_mlp_block_scores(L, x, vec, part, thr, 16, nv, margin=margin) == 0
        assert torch.equal(vec, before)


def test_refine_capacity_matches_exact(cuda):
    """The read-back-free refinement (capacity rows, device [count, overflow])
    patches exactly what the counted path patches when the capacity covers
    the band; a capacity below the count raises the overflow flag."""
    from paper_2501_09767_b200.model import refine_mlp_block_scores
    cfg = ModelConfig(n_layers=1, hidden_dim=256, n_heads=2, vocab_size=64, max_seq_len=1024,
                      block_size=16, mlp_dim=688, lora_rank=4, lora_alpha=8.0)
    m = DecoderModel(cfg, 5, init="reference", parity_weights=True)
    L = m.layers[0]
    x = torch.randn(1024, 256, device="cuda")
    nv = 1024 - 5
    v0, part = mlp_block_score_vector(L, x, 16, nv, precision="bf16", with_partial=True)
    thr = float(torch.quantile(v0, 0.5))
    exact_vec = v0.clone()
    rows = refine_mlp_block_scores(L, x, exact_vec, part, thr, 16, nv, margin=5e-2)
    assert rows > 8
    cap_vec = v0.clone()
    flags = refine_mlp_block_scores(L, x, cap_vec, part, thr, 16, nv, margin=5e-2,
                                    capacity=rows + 37)
    count, overflow = (int(v) for v in flags.cpu())
    assert (count, overflow) == (rows, 0)
    assert torch.equal(cap_vec, exact_vec)
    small = v0.clone()
    flags = refine_mlp_block_scores(L, x, small, part, thr, 16, nv, margin=5e-2, capacity=8)
    assert [int(v) for v in flags.cpu()] == [rows, 1]
    big = v0.clone()  # a capacity beyond the sequence is clamped to it
    flags = refine_mlp_block_scores(L, x, big, part, thr, 16, nv, margin=5e-2, capacity=5000)
    assert [int(v) for v in flags.cpu()] == [rows, 0] and torch.equal(big, exact_vec)


def test_ce_rows_out_of_range_target_is_nan(cuda):
    """A target that escapes host validation makes its row loss NaN (the
    summed loss turns NaN) instead of being dropped silently."""
    V = 64
    logits = torch.randn(4, V, device="cuda")
    tg = torch.tensor([3, -1, V + 5, 7], dtype=torch.int32, device="cuda")
    dl = torch.empty(4, V, dtype=torch.bfloat16, device="cuda")
    rl = torch.empty(4, dtype=torch.float32, device="cuda")
    bad = torch.zeros(1, dtype=torch.int32, device="cuda")
    ops.ce_rows(logits, tg, V=V, ignore=-1, inv_count=1.0, dlogits=dl, row_loss=rl, bad=bad)
    r = rl.cpu()
    assert torch.isfinite(r[[0, 3]]).all() and r[1] == 0 and torch.isnan(r[2])
    assert int(bad) == 1 and not dl[2].float().abs().any()
    ops.ce_rows(logits, tg, V=V, ignore=-1, inv_count=1.0, dlogits=dl, row_loss=rl)
    assert torch.isnan(rl[2])


def test_layer_qk_fp32_matches_reference(cuda):
    z = np.load(G / "scorers.npz")
    m = _scorer_model_fp32(3, mlp_dim=344, lora_rank=4, lora_alpha=8.0)
    m.layers[0].lora_q.b.copy_(torch.as_tensor(z["lora_q_b"]))
    x = torch.as_tensor(z["x"]).cuda()
    (qh, ql), (kh, kl) = layer_qk(m.layers[0], x)
    H, s, d = z["q"].shape
    qref = z["q"].transpose(1, 0, 2).reshape(s, H * d)
    kref = z["k"].transpose(1, 0, 2).reshape(s, H * d)
    q = (qh.float() + ql.float()).cpu().numpy()
    k = (kh.float() + kl.float()).cpu().numpy()
    np.testing.assert_allclose(q, qref, rtol=0, atol=2e-5 * np.abs(qref).max())
    np.testing.assert_allclose(k, kref, rtol=0, atol=2e-5 * np.abs(kref).max())


def test_exact_scores_reference_signature_fp32(cuda):
    """sparsity.exact_block_scores(q, k, block_size, *, n_valid, ...) on the
    reference's own [H, s, d] f32 q/k (sparsity.py:173-181): the tcgen05
    scorer in bf16x3 mode reproduces the f32 scores to ~1e-6."""
    z = np.load(G / "scorers.npz")
    nv = int(z["n_valid"])
    bsm = S.exact_block_scores(z["q"], z["k"], 16, n_valid=nv, layer_id=3)
    ref = z["exact_packed"]
    assert bsm.layer_id == 3 and bsm.n_blocks == 11
    np.testing.assert_allclose(bsm.scores.cpu().numpy(), ref, rtol=1e-5, atol=1e-6 * ref.max())
    vec = S.token_block_scores(bsm).cpu().numpy()
    np.testing.assert_allclose(vec, z["exact_vec"], rtol=1e-5)
    # [s, d] input = one head; shape mismatch / bad rank raise like the reference
    one = S.exact_block_scores(z["q"][0], z["k"][0], 16)
    assert one.n_blocks == 11
    from paper_2501_09767_b200.errors import ContractError
    with pytest.raises(ContractError):
        S.exact_block_scores(z["q"], z["k"][:1], 16)
    with pytest.raises(ContractError):
        S.exact_block_scores(z["q"][None], z["k"][None], 16)
    with pytest.raises(ContractError):
        S.exact_block_scores(z["q"][:, :8], z["k"][:, :8], 16)


@pytest.mark.parametrize("s,H,Hk,d", [(300, 4, 4, 64), (1000, 2, 2, 128), (777, 8, 2, 128),
                                      (2048, 4, 4, 64)])
def test_exact_scorer_vs_oracle_shapes(cuda, s, H, Hk, d):
    """tcgen05 exact scorer (both precisions) on ragged lengths, GQA and both
    head dims against the oracle's dense tile maxima."""
    rng = np.random.default_rng(s + H)
    q = rng.standard_normal((H, s, d)).astype(np.float32) * 0.3
    kk = rng.standard_normal((Hk, s, d)).astype(np.float32) * 0.3
    nv = s - 3
    ref = O.exact_block_dense(q, np.repeat(kk, H // Hk, axis=0), 16, nv)
    rows = lambda a: torch.as_tensor(a.transpose(1, 0, 2).reshape(s, -1)).cuda()  # noqa: E731
    qh, ql = ops.split_hilo(rows(q))
    kh, kl = ops.split_hilo(rows(kk))
    dense = exact.exact_block_dense((qh, ql), (kh, kl), 16, n_heads=H, n_valid=nv).cpu().numpy()
    np.testing.assert_allclose(dense, ref, rtol=1e-5, atol=1e-6 * ref.max())
    dense16 = exact.exact_block_dense(rows(q).bfloat16(), rows(kk).bfloat16(), 16, n_heads=H,
                                      n_valid=nv).cpu().numpy()
    np.testing.assert_allclose(dense16, ref, rtol=3e-2, atol=1e-2 * ref.max())


# ------------------------------------------------------------------ attention


def _torch_attn(q, k, v, H):
    n, h = q.shape
    d = h // H
    qh = q.float().view(n, H, d).transpose(0, 1)
    kh = k.float().view(n, H, d).transpose(0, 1)
    vh = v.float().view(n, H, d).transpose(0, 1)
    s = qh @ kh.transpose(1, 2) / math.sqrt(d)
    mask = torch.ones(n, n, dtype=torch.bool, device=q.device).tril()
    s = s.masked_fill(~mask, float("-inf"))
    p = torch.softmax(s, -1)
    lse = torch.logsumexp(s, -1)
    return (p @ vh).transpose(0, 1).reshape(n, h), lse


@pytest.mark.parametrize("n,H,d", [(1, 2, 64), (17, 2, 64), (64, 4, 128), (100, 2, 128),
                                   (257, 4, 64), (1000, 2, 128)])
def test_flash_fwd_bwd_vs_torch(cuda, n, H, d):
    g = torch.Generator(device=cuda).manual_seed(n)
    h = H * d
    q, k, v = (torch.randn(n, h, device=cuda, generator=g).bfloat16() for _ in range(3))
    o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
    qr, kr, vr = (t.float().requires_grad_(True) for t in (q, k, v))
    oref, lref = _torch_attn(qr, kr, vr, H)
    torch.testing.assert_close(o.float(), oref, rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(lse, lref, rtol=1e-3, atol=1e-3)
    dout = torch.randn(n, h, device=cuda, generator=g).bfloat16()
    oref.backward(dout.float())
    dq, dk, dv = ops.flash_bwd(q, k, v, o, dout, lse, head_dim=d, scale=1 / math.sqrt(d))
    floor = 1e-2 * dout.float().norm()  # dq = dk = 0 exactly for a single token
    for got, ref in ((dq, qr.grad), (dk, kr.grad), (dv, vr.grad)):
        err = (got - ref).norm() / torch.maximum(ref.norm(), floor)
        assert err < 2e-2, float(err)


# ------------------------------------------------------------------ rows


def test_rmsnorm_gather_lora(cuda):
    g = torch.Generator(device=cuda).manual_seed(1)
    s, h, r = 300, 512, 8
    x = torch.randn(s, h, device=cuda, generator=g)
    w = torch.rand(h, device=cuda, generator=g) + 0.5
    A = torch.randn(h, 2 * r, device=cuda, generator=g) / math.sqrt(h)
    idx = torch.arange(0, s, 3, device=cuda, dtype=torch.int32)
    k = idx.numel()
    xg = torch.empty(k, h, dtype=torch.bfloat16, device=cuda)
    inv = torch.empty(k, device=cuda)
    xn = ops.rmsnorm_gather(x, w, idx, xg=xg, inv=inv)
    t = ops.lora_down(xn, ops.lora_pack(A, r))
    xr = x[idx.long()]
    invr = 1 / torch.sqrt((xr * xr).mean(-1, keepdim=True) + 1e-6)
    xnr = xr * invr * w
    torch.testing.assert_close(xn.float(), xnr, rtol=1e-2, atol=1e-2)
    torch.testing.assert_close(inv, invr[:, 0], rtol=1e-5, atol=1e-6)
    assert t.shape == (k, 32) and float(t[:, 2 * r:].abs().max()) == 0.0
    torch.testing.assert_close(t[:, :2 * r], xn.float() @ A.bfloat16().float(), rtol=1e-3,
                               atol=1e-3)
    torch.testing.assert_close(xg.float(), xr, rtol=1e-2, atol=1e-2)


def test_gateup_and_dgateup_vs_torch(cuda):
    g = torch.Generator(device=cuda).manual_seed(2)
    M, h, m = 200, 256, 344
    cfg = ModelConfig(n_layers=1, hidden_dim=h, n_heads=4, vocab_size=64, mlp_dim=m)
    model = DecoderModel(cfg, 0)
    L = model.layers[0]
    xn = torch.randn(M, h, device=cuda, generator=g).bfloat16()
    N = L.w_gu_t.shape[0]
    gu = torch.empty(M, N, dtype=torch.bfloat16, device=cuda)
    inner = torch.empty(M, L.m_pad, dtype=torch.bfloat16, device=cuda)
    part = torch.empty(N // 128, M, device=cuda)
    ops.gemm_gateup(xn, L.w_gu_t, gu=gu, inner=inner, partial=part)
    full = xn.float() @ L.w_gu_t.float().t()
    gate = full.view(M, L.m_pad // 128, 2, 128)[:, :, 0].reshape(M, -1)
    up = full.view(M, L.m_pad // 128, 2, 128)[:, :, 1].reshape(M, -1)
    innr = torch.nn.functional.silu(gate) * up
    torch.testing.assert_close(inner.float(), innr, rtol=3e-2, atol=3e-2)
    torch.testing.assert_close(part.sum(0) / m, innr.abs().sum(-1) / m, rtol=1e-2, atol=1e-3)
    dy = torch.randn(M, h, device=cuda, generator=g).bfloat16()
    dgu = torch.empty_like(gu)
    ops.gemm_dgateup(dy, L.w_down, gu, dgu, m_pad=L.m_pad)
    dinner = dy.float() @ L.w_down.float().t()
    gb = gu.float().view(M, L.m_pad // 128, 2, 128)
    gg, uu = gb[:, :, 0].reshape(M, -1), gb[:, :, 1].reshape(M, -1)
    sg = torch.sigmoid(gg)
    dg = dinner * uu * sg * (1 + gg * (1 - sg))
    du = dinner * gg * sg
    got = dgu.float().view(M, L.m_pad // 128, 2, 128)
    torch.testing.assert_close(got[:, :, 0].reshape(M, -1), dg, rtol=3e-2, atol=3e-2)
    torch.testing.assert_close(got[:, :, 1].reshape(M, -1), du, rtol=3e-2, atol=3e-2)


def test_qkv_rope_lora_vs_oracle(cuda):
    """q/k/v projection epilogue = _project + rope_rotate at original positions."""
    rng = np.random.default_rng(0)
    h, H, r, M = 256, 4, 8, 96
    d = h // H
    cfg = ModelConfig(n_layers=1, hidden_dim=h, n_heads=H, vocab_size=64, mlp_dim=256, lora_rank=r)
    model = DecoderModel(cfg, 0)
    L = model.layers[0]
    L.lora_q.b.copy_(torch.randn(r, h, device=cuda) * 0.1)
    L.lora_v.b.copy_(torch.randn(r, h, device=cuda) * 0.1)
    xn_ext = torch.empty(M, h + 64, dtype=torch.bfloat16, device=cuda)
    xn_ext[:, :h] = torch.as_tensor(rng.standard_normal((M, h)).astype(np.float32)).cuda().bfloat16()
    xn = xn_ext[:, :h]
    pos_np = np.sort(rng.choice(1000, M, replace=False))
    pos = torch.as_tensor(pos_np.astype(np.int32)).cuda()
    t = L.qkv_input(xn_ext)
    q, k, v = ops.gemm_qkv(xn_ext, L.w_qkv_t, h=h, head_dim=d, rope=True, inv_freq=L.inv_freq,
                           pos=pos)
    xf = xn.float().cpu().numpy()
    W = L.w_qkv[:, :3 * h].float().cpu().numpy()
    s = L.lora_scaling
    np.testing.assert_allclose(t[:, :2 * r].cpu().numpy(),
                               xf @ L.lora_A.bfloat16().float().cpu().numpy(), rtol=1e-3, atol=1e-3)
    qr = xf @ W[:, :h] + (t[:, :r].cpu().numpy() @ L.lora_Bq.cpu().numpy()) * s
    kr = xf @ W[:, h:2 * h]
    vr = xf @ W[:, 2 * h:] + (t[:, r:2 * r].cpu().numpy() @ L.lora_Bv.cpu().numpy()) * s
    qr = O.rope_fwd(qr.astype(np.float32), pos_np, H, 10000.0)
    kr = O.rope_fwd(kr.astype(np.float32), pos_np, H, 10000.0)
    for got, ref in ((q, qr), (k, kr), (v, vr)):
        np.testing.assert_allclose(got.float().cpu().numpy(), ref, rtol=2e-2, atol=2e-2)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("n,H", [(1, 1), (63, 1), (65, 2), (100, 2), (128, 1), (191, 1), (257, 2),
                                 (1000, 2), (2049, 1)])
def test_flash_tc_vs_torch(cuda, n, H, d):
    """tcgen05 attention forward + backward (both head dims) vs fp32 torch on
    ragged lengths (partial tiles, odd tile counts, a single token)."""
    g = torch.Generator(device=cuda).manual_seed(n + 11 + d)
    h = H * d
    q, k, v = (torch.randn(n, h, device=cuda, generator=g).bfloat16() for _ in range(3))
    o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
    qr, kr, vr = (t.float().requires_grad_(True) for t in (q, k, v))
    oref, lref = _torch_attn(qr, kr, vr, H)
    torch.testing.assert_close(o.float(), oref, rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(lse, lref, rtol=1e-3, atol=1e-3)
    dout = torch.randn(n, h, device=cuda, generator=g).bfloat16()
    oref.backward(dout.float())
    dq, dk, dv = ops.flash_bwd(q, k, v, o, dout, lse, head_dim=d, scale=1 / math.sqrt(d))
    floor = 1e-2 * dout.float().norm()
    for name, got, ref in (("dq", dq, qr.grad), ("dk", dk, kr.grad), ("dv", dv, vr.grad)):
        err = (got - ref).norm() / torch.maximum(ref.norm(), floor)
        assert err < 2e-2, (name, float(err))


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("n,H,Hkv", [(100, 4, 2), (257, 4, 1), (1000, 8, 2), (2049, 4, 4)])
def test_flash_gqa_vs_torch(cuda, n, H, Hkv, d):
    """Grouped-query attention on the tcgen05 kernels: fwd + bwd vs fp32 torch
    on K/V heads repeated to the query heads (dK/dV summed over the group)."""
    g = torch.Generator(device=cuda).manual_seed(n + H)
    h, kv = H * d, Hkv * d
    q = torch.randn(n, h, device=cuda, generator=g).bfloat16()
    k = torch.randn(n, kv, device=cuda, generator=g).bfloat16()
    v = torch.randn(n, kv, device=cuda, generator=g).bfloat16()
    o, lse = ops.flash_fwd(q, k, v, head_dim=d, scale=1 / math.sqrt(d))
    rep = lambda t: t.view(n, Hkv, d).repeat_interleave(H // Hkv, dim=1).reshape(n, h)  # noqa
    qr = q.float().requires_grad_(True)
    kr = k.float().requires_grad_(True)
    vr = v.float().requires_grad_(True)
    oref, lref = _torch_attn(qr, rep(kr), rep(vr), H)
    torch.testing.assert_close(o.float(), oref, rtol=2e-2, atol=2e-2)
    torch.testing.assert_close(lse, lref, rtol=1e-3, atol=1e-3)
    dout = torch.randn(n, h, device=cuda, generator=g).bfloat16()
    oref.backward(dout.float())
    dq, dk, dv = ops.flash_bwd(q, k, v, o, dout, lse, head_dim=d, scale=1 / math.sqrt(d))
    assert dk.shape == (n, kv) and dv.shape == (n, kv)
    floor = 1e-2 * dout.float().norm()
    for name, got, ref in (("dq", dq, qr.grad), ("dk", dk, kr.grad), ("dv", dv, vr.grad)):
        err = (got - ref).norm() / torch.maximum(ref.norm(), floor)
        assert err < 2e-2, (name, float(err))
