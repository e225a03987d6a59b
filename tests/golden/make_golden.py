"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is importable there, read-only):

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden.py

Writes small .npz files next to this script.  They pin the oracle
(oracle/lemo_oracle.py) and, through it, the GPU path; nothing at test or
bench time reads /root/reference.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from sparsetune import kernels, model as model_mod, predictor as pred_mod, sparsity  # noqa: E402
from sparsetune import tensor as T  # noqa: E402
from sparsetune.optim import Adam  # noqa: E402

OUT = Path(__file__).resolve().parent


def select_cases():
    rng = np.random.default_rng(1234)
    vecs, thrs, forces, ns, bs, masks, toks = [], [], [], [], [], [], []
    for case in range(64):
        b = int(rng.choice([1, 4, 8, 16]))
        n_tokens = int(rng.integers(1, 400))
        nb = sparsity.n_blocks_for(n_tokens, b)
        kind = case % 4
        if kind == 0:
            v = rng.standard_normal(nb) ** 2
        elif kind == 1:
            v = rng.integers(0, 5, nb).astype(np.float64)  # many ties
        elif kind == 2:
            v = np.abs(rng.standard_normal(nb)) * 10 ** rng.uniform(-8, 8)
        else:
            v = np.zeros(nb)
        choice = case % 5
        if choice == 0:
            thr = float("-inf")
        elif choice == 1:
            thr = float(v.max()) + 1.0
        elif choice == 2 and nb:
            thr = float(v[rng.integers(0, nb)])  # exact tie with a score
        else:
            thr = float(np.quantile(v, rng.uniform(0, 1))) if nb else 0.0
        force = (0,) if case % 3 == 0 else ()
        pat = sparsity.eliminate(v, thr, block_size=b, n_tokens=n_tokens, force_blocks=force)
        m = np.zeros(nb, dtype=np.uint8)
        m[list(pat.retained_blocks)] = 1
        vecs.append(v)
        thrs.append(thr)
        forces.append(1 if force else 0)
        ns.append(n_tokens)
        bs.append(b)
        masks.append(m)
        toks.append(pat.token_indices)
    np.savez_compressed(
        OUT / "select.npz",
        vec=np.concatenate(vecs), vec_len=np.array([len(v) for v in vecs]),
        thr=np.array(thrs), sink=np.array(forces), n_tokens=np.array(ns), block=np.array(bs),
        mask=np.concatenate(masks), tok=np.concatenate(toks),
        tok_len=np.array([len(t) for t in toks]))


def quantile_cases():
    """_maybe_recalibrate threshold sequence (model.py:545-563)."""
    rng = np.random.default_rng(99)
    out_vecs, out_thr, out_ret, out_nb = [], [], [], []
    for case in range(24):
        nb = int(rng.integers(1, 300))
        ret = [0.0, 1.0, 0.5, 0.25, 0.9, 0.37][case % 6]
        src = model_mod.PredictedPatternSource(
            None, sparsity.ThresholdSet(), target_retention={0: ret}, recalibrate_every=1,
            history=8)
        thr_seq = []
        vecs = []
        for call in range(11):
            if case % 2:
                v = rng.integers(0, 4, nb).astype(np.float64)
            else:
                v = rng.standard_normal(nb) ** 2
            src._maybe_recalibrate(0, v)
            thr_seq.append(src.thresholds.get(0, sparsity.ATTENTION))
            vecs.append(v)
        out_vecs.append(np.stack(vecs))
        out_thr.append(thr_seq)
        out_ret.append(ret)
        out_nb.append(nb)
    np.savez_compressed(OUT / "quantile.npz",
                        vecs=np.concatenate([v.reshape(-1) for v in out_vecs]),
                        nb=np.array(out_nb), thr=np.array(out_thr), ret=np.array(out_ret))


def column_sum_cases():
    rng = np.random.default_rng(7)
    packed, nbs, outs = [], [], []
    for nb in (1, 2, 5, 33, 128):
        p = np.abs(rng.standard_normal(sparsity.tri_size(nb))).astype(np.float32)
        bsm = sparsity.BlockScoreMatrix(nb, 16, p)
        packed.append(p.astype(np.float64))
        nbs.append(nb)
        outs.append(sparsity.token_block_scores(bsm))
    np.savez_compressed(OUT / "colsum.npz", packed=np.concatenate(packed), nb=np.array(nbs),
                        vec=np.concatenate(outs))


def predictor_case():
    rng = np.random.default_rng(11)
    h, r1, r2, dp, b, s = 128, 32, 24, 16, 16, 256
    pq = pred_mod.Predictor.create(rng, h, r1, r2, dp, "q", 0)
    pk = pred_mod.Predictor.create(rng, h, r1, r2, dp, "k", 0)
    pq.mask1[::5] = False  # exercise pruned neurons (exact zeros)
    pk.mask2[1::7] = False
    x = rng.standard_normal((s, h)).astype(np.float32)
    packed = pred_mod.predicted_triangle(pq, pk, x, b).data
    packed_tok = pred_mod.predicted_triangle(pq, pk, x, b, pooling="token").data
    nb = s // b
    vec = sparsity.token_block_scores(sparsity.BlockScoreMatrix(nb, b, np.maximum(packed, 0.0)))
    np.savez_compressed(
        OUT / "predictor.npz", x=x, b=b,
        q_w1=pq.w1.data, q_w2=pq.w2.data, q_w3=pq.w3.data, q_m1=pq.mask1, q_m2=pq.mask2,
        k_w1=pk.w1.data, k_w2=pk.w2.data, k_w3=pk.w3.data, k_m1=pk.mask1, k_m2=pk.mask2,
        packed=packed, packed_token=packed_tok, vec=vec,
        block_embed=pred_mod.block_embed(x, b))


def scorer_cases():
    cfg = model_mod.ModelConfig(n_layers=1, hidden_dim=128, n_heads=2, vocab_size=64,
                                max_seq_len=256, mlp_dim=344, block_size=16, lora_rank=4,
                                lora_alpha=8.0)
    m = model_mod.DecoderModel(cfg, seed=3)
    layer = m.layers[0]
    rng = np.random.default_rng(5)
    layer.lora_q.b.data[...] = rng.standard_normal(layer.lora_q.b.shape).astype(np.float32) * 0.1
    x = rng.standard_normal((176, 128)).astype(np.float32)
    n_valid = 170
    mlp_vec = model_mod.mlp_block_score_vector(layer, x, 16, n_valid)
    q, k = model_mod.layer_qk(layer, x)
    bsm = sparsity.exact_block_scores(q, k, 16, n_valid=n_valid)
    np.savez_compressed(
        OUT / "scorers.npz", x=x, n_valid=n_valid, mlp_vec=mlp_vec, q=q, k=k,
        exact_packed=bsm.scores, exact_vec=sparsity.token_block_scores(bsm),
        lora_q_b=layer.lora_q.b.data)
    relu_cfg = model_mod.ModelConfig(n_layers=1, hidden_dim=128, n_heads=2, vocab_size=64,
                                     max_seq_len=256, mlp_dim=256, block_size=16,
                                     mlp_variant="relu")
    rm = model_mod.DecoderModel(relu_cfg, seed=4)
    np.savez_compressed(OUT / "scorers_relu.npz", x=x, n_valid=n_valid,
                        mlp_vec=model_mod.mlp_block_score_vector(rm.layers[0], x, 16, n_valid))


STEP_CFG = dict(n_layers=2, hidden_dim=128, n_heads=2, vocab_size=128, max_seq_len=256,
                mlp_dim=344, block_size=16, lora_rank=8, lora_alpha=16.0)
# head_dim 128: the geometry of the production (Llama-class) attention kernels
STEP_CFG_D128 = dict(n_layers=2, hidden_dim=256, n_heads=2, vocab_size=128, max_seq_len=256,
                     mlp_dim=344, block_size=16, lora_rank=8, lora_alpha=16.0)
STEP_VARIANTS = {"": STEP_CFG, "_d128": STEP_CFG_D128}


def _perturb_b(m, seed):
    rng = np.random.default_rng(seed)
    for layer in m.layers:
        for ad in (layer.lora_q, layer.lora_v):
            ad.b.data[...] = (rng.standard_normal(ad.b.shape) * 0.1).astype(np.float32)


def _grads(m):
    out = {}
    for layer in m.layers:
        for tag, ad in (("lora_q", layer.lora_q), ("lora_v", layer.lora_v)):
            out[f"layer{layer.layer_id}.{tag}.a"] = ad.a.grad.copy()
            out[f"layer{layer.layer_id}.{tag}.b"] = ad.b.grad.copy()
    return out


def step_cases(suffix=""):
    base = STEP_VARIANTS[suffix]
    h = base["hidden_dim"]
    rng = np.random.default_rng(21)
    tokens = rng.integers(0, base["vocab_size"], size=150)
    cases = {}
    for mode in ("dense", "fraction", "predicted", "exact"):
        cfg = model_mod.ModelConfig(**base)
        m = model_mod.DecoderModel(cfg, seed=17)
        _perturb_b(m, 23)
        source = None
        extra = {}
        if mode == "fraction":
            source = model_mod.FractionSource(0.5, cfg.block_size)
        elif mode in ("predicted", "exact"):
            # MLP thresholds: pooled mean of a 1-batch exact profile (init_thresholds)
            prof = model_mod.ExactPatternSource(m, None, record=True)
            with T.no_grad():
                m.forward_step(tokens, segments=2, pattern_source=prof)
            ts = sparsity.init_thresholds(prof.recorded_vectors)
            if mode == "exact":
                source = model_mod.ExactPatternSource(m, ts)
            else:
                prng = np.random.default_rng(31)
                pairs = {}
                for l in range(cfg.n_layers):
                    pairs[l] = (pred_mod.Predictor.create(prng, h, 32, 32, 32, "q", l),
                                pred_mod.Predictor.create(prng, h, 32, 32, 32, "k", l))
                m.attach_predictors(pairs)
                for l, (pq, pk) in pairs.items():
                    for tag, p in (("q", pq), ("k", pk)):
                        extra[f"pred{l}_{tag}_w1"] = p.w1.data
                        extra[f"pred{l}_{tag}_w2"] = p.w2.data
                        extra[f"pred{l}_{tag}_w3"] = p.w3.data
                source = model_mod.PredictedPatternSource(
                    m, ts.copy(), target_retention={0: 0.5, 1: 0.5}, recalibrate_every=1)
            for (l, c), v in ts.values.items():
                extra[f"thr_{l}_{c}"] = np.array(v)
        led_losses = []
        opt = Adam(m.adapter_parameters(), lr=1e-2)
        loss, hidden = m.forward_step(tokens, segments=2, pattern_source=source)
        T.backward(loss)
        grads = _grads(m)
        pats = {}
        if source is not None:
            # re-derive the masks recorded by this step from last_fractions is lossy;
            # record them by re-running the hook in a FixedPatternSource-free way:
            pass
        opt.step()
        opt.zero_grad()
        loss2, _ = m.forward_step(tokens, segments=2, pattern_source=source)
        T.release_tape(loss2)
        led_losses = [float(loss.data), float(loss2.data)]
        arrays = {f"grad__{k}": v for k, v in grads.items()}
        arrays.update(extra)
        frac = {f"{l}:{c}": f for (l, c), f in (source.last_fractions.items() if source else [])}
        np.savez_compressed(OUT / f"step_{mode}{suffix}.npz", tokens=tokens,
                            losses=np.array(led_losses),
                            hidden=hidden.data, fractions=json.dumps(frac), **arrays)
        cases[mode] = led_losses
    return cases


def step_pattern_cases(suffix=""):
    """Per-(layer, component) retained blocks of the predicted step, captured
    through a recording wrapper around the reference source."""
    base = STEP_VARIANTS[suffix]
    h = base["hidden_dim"]
    rng = np.random.default_rng(21)
    tokens = rng.integers(0, base["vocab_size"], size=150)
    cfg = model_mod.ModelConfig(**base)
    out = {}
    for mode in ("predicted", "exact"):
        m = model_mod.DecoderModel(cfg, seed=17)
        _perturb_b(m, 23)
        prof = model_mod.ExactPatternSource(m, None, record=True)
        with T.no_grad():
            m.forward_step(tokens, segments=2, pattern_source=prof)
        ts = sparsity.init_thresholds(prof.recorded_vectors)
        if mode == "predicted":
            prng = np.random.default_rng(31)
            pairs = {l: (pred_mod.Predictor.create(prng, h, 32, 32, 32, "q", l),
                         pred_mod.Predictor.create(prng, h, 32, 32, 32, "k", l))
                     for l in range(cfg.n_layers)}
            m.attach_predictors(pairs)
            src = model_mod.PredictedPatternSource(m, ts.copy(), target_retention={0: 0.5, 1: 0.5},
                                                  recalibrate_every=1)
        else:
            src = model_mod.ExactPatternSource(m, ts)
        orig = src.pattern
        rec = {}

        def recording(layer_id, component, x_np, n_valid, _orig=orig, _rec=rec):
            p = _orig(layer_id, component, x_np, n_valid)
            _rec[(layer_id, component)] = (tuple(p.retained_blocks) if p is not None else None,
                                           x_np.copy())
            return p

        src.pattern = recording
        with T.no_grad():
            m.forward_step(tokens, segments=2, pattern_source=src)
        arrays = {}
        for (l, c), (blocks, x) in rec.items():
            arrays[f"blocks_{l}_{c}"] = np.array(blocks if blocks is not None else [-1])
            arrays[f"x_{l}_{c}"] = x
        if mode == "predicted":
            arrays["thr_attn"] = np.array([src.thresholds.get(l, "attention") for l in range(2)])
        np.savez_compressed(OUT / f"patterns_{mode}{suffix}.npz", **arrays)
        out[mode] = {k: v[0] for k, v in rec.items()}
    return out


def predictor_train_case(pooling="mean"):
    """fit_predictors (predictor.py:366-433) on fixed teacher records: per-epoch
    losses / recall / active params and the final weights, masks, counters."""
    rng = np.random.default_rng(77)
    h, r, b, s, n_layers = 64, 16, 8, 128, 2
    nb = s // b
    tsz = nb * (nb + 1) // 2
    pairs = {l: (pred_mod.Predictor.create(rng, h, r, r, r, "q", l),
                 pred_mod.Predictor.create(rng, h, r, r, r, "k", l)) for l in range(n_layers)}
    init = {f"init_{l}_{p.role}_{n}": a.copy() for l, pq in pairs.items() for p in pq
            for n, a in p.state_arrays().items()}
    records, arrays = [], {}
    for i in range(2 * n_layers):
        l = i % n_layers
        x = rng.standard_normal((s, h)).astype(np.float32)
        teacher = (np.abs(rng.standard_normal(tsz)) * 3.0).astype(np.float64)
        records.append(pred_mod.TeacherRecord(l, x, teacher, s, b))
        arrays[f"x_{i}"] = x
        arrays[f"teacher_{i}"] = teacher
        arrays[f"layer_{i}"] = np.array([l])
    hist = pred_mod.fit_predictors(pairs, records, epochs=6, lr=1e-2, val_data=records,
                                   prune_target=0.6, prune_every=2, prune_step=0.2, eval_every=3,
                                   pooling=pooling)
    arrays.update(init)
    arrays["loss"] = np.array([hr.train_loss for hr in hist])
    arrays["recall"] = np.array([hr.recall for hr in hist])
    arrays["params"] = np.array([hr.param_count for hr in hist])
    for l, pq in pairs.items():
        for p in pq:
            for n, a in p.state_arrays().items():
                arrays[f"final_{l}_{p.role}_{n}"] = a
    suffix = "" if pooling == "mean" else "_" + pooling
    np.savez_compressed(OUT / f"predictor_train{suffix}.npz", **arrays)
    return arrays["loss"].tolist()


def artifact_case():
    """Reference-written artifacts: predictors.ckpt (STCHKPT container,
    pred/L{l}/{role}/{name} keys, pipeline.py:370-418), thresholds.json,
    config hashes; plus the reference's predicted scores on a fixed input."""
    from sparsetune import checkpoint, pipeline
    from sparsetune.config import RunConfig

    cfg = RunConfig()
    cfg.model = model_mod.ModelConfig(n_layers=2, hidden_dim=64, n_heads=4, vocab_size=256,
                                      mlp_dim=256, block_size=8, max_seq_len=512)
    rng = np.random.default_rng(5)
    pairs = {l: (pred_mod.Predictor.create(rng, 64, 16, 16, 16, "q", l),
                 pred_mod.Predictor.create(rng, 64, 16, 16, 16, "k", l)) for l in range(2)}
    for pq in pairs.values():
        for p in pq:
            pred_mod.track_zero_frequency(p, rng.standard_normal((40, 64)).astype(np.float32))
            pred_mod.elastic_prune(p, 0.75)
    pt = sparsity.ThresholdSet({(0, "attention"): 1.25, (1, "attention"): -0.5,
                                (0, "mlp"): 0.125, (1, "mlp"): 3.0}, config_hash=cfg.config_hash())
    pipeline.save_predictors(OUT / "predictors.ckpt", cfg, pairs, pt, {0: 0.5, 1: 0.4})
    ts = sparsity.ThresholdSet({(0, "attention"): 2.5, (0, "mlp"): 0.75, (1, "attention"): 1e-3,
                                (1, "mlp"): 7.0}, eps=0.01, eta=None, config_hash=cfg.config_hash())
    (OUT / "thresholds.json").write_text(json.dumps(ts.to_dict(), indent=2) + "\n")
    x = rng.standard_normal((128, 64)).astype(np.float32)
    vecs = {}
    for l, (p_q, p_k) in pairs.items():
        tri = pred_mod.predicted_triangle(p_q, p_k, x, 8).data
        bsm = sparsity.BlockScoreMatrix(16, 8, np.maximum(tri, 0.0))
        vecs[f"vec_{l}"] = sparsity.token_block_scores(bsm)
    hashes = {}
    for name, kw in (("tiny", dict(n_layers=2, hidden_dim=256, n_heads=4, vocab_size=256,
                                   mlp_dim=688, block_size=16)),
                     ("llama2_7b", dict(n_layers=32, hidden_dim=4096, n_heads=32,
                                        vocab_size=32000, mlp_dim=11008, block_size=16,
                                        max_seq_len=16384)),
                     ("relu_learned", dict(mlp_variant="relu", positions="learned"))):
        c = RunConfig()
        c.model = model_mod.ModelConfig(**kw)
        hashes[name] = [kw, c.config_hash()]
        c.sparsity.mlp_scoring = False
        hashes[name + "_nomlp"] = [kw, c.config_hash()]
    (OUT / "config_hashes.json").write_text(json.dumps(hashes, indent=1) + "\n")
    # a container with mixed dtypes / shapes, written by the reference
    tensors = {"a/f32": rng.standard_normal((3, 5)).astype(np.float32),
               "b/i64": np.arange(7, dtype=np.int64), "c/bool": np.array([True, False, True]),
               "d/f64": np.array(3.5), "e/empty": np.zeros((0, 4), dtype=np.float32)}
    checkpoint.save_container(OUT / "mixed.ckpt", tensors, {"k": 1}, {"m": "x"})
    np.savez_compressed(OUT / "artifacts.npz", x=x, hash=np.array([cfg.config_hash()]), **vecs,
                        **{"t_" + k.replace("/", "_"): v for k, v in tensors.items()})


def tune_case():
    """tune_thresholds (sparsity.py:379-417) on a smooth synthetic accuracy proxy."""
    ts = sparsity.ThresholdSet({(0, "attention"): 1.0, (0, "mlp"): -2.0, (1, "attention"): 0.0,
                                (1, "mlp"): 5.0})

    def acc(t):
        v = t.values
        return -sum((val - 0.3 * (i + 1)) ** 2 + 0.1 * val ** 3 / (1 + val ** 2)
                    for i, (_, val) in enumerate(sorted(v.items())))

    out = {}
    for name, kw in (("auto", dict(rounds=2)), ("fixed", dict(eps=0.05, eta=0.2, rounds=3))):
        tuned = sparsity.tune_thresholds(acc, ts, **kw)
        out[name] = tuned.to_dict()
    (OUT / "tune.json").write_text(json.dumps({"init": ts.to_dict(), **out}, indent=1) + "\n")


GQA_CFG = dict(n_layers=2, hidden_dim=512, n_heads=4, vocab_size=256, max_seq_len=512,
               mlp_dim=344, block_size=16, lora_rank=8, lora_alpha=16.0)
GQA_KV_HEADS = 2


def gqa_case():
    """Grouped-query attention is not in the reference; pin it through the
    equivalent multi-head model: K/V (and LoRA B_v) head blocks repeated
    `group` times.  The oracle's GQA model (seed 5) supplies the weights; the
    reference runs the repeated MHA model; gradients of the repeated blocks
    are folded back (summed) to the GQA shapes."""
    sys.path.insert(0, str(OUT.parent.parent))
    from oracle import lemo_oracle as O

    om = O.init_model(O.Config(**GQA_CFG, n_kv_heads=GQA_KV_HEADS), seed=5)
    O.perturb_lora_b(om, 6)
    h, H = GQA_CFG["hidden_dim"], GQA_CFG["n_heads"]
    d, g = h // H, H // GQA_KV_HEADS
    rep = lambda w: np.concatenate([w[..., (hd // g) * d:(hd // g + 1) * d]  # noqa: E731
                                    for hd in range(H)], axis=-1)
    state = {"embed": om.embed, "final_norm": om.final_norm, "lm_head": om.lm_head}
    for i, L in enumerate(om.layers):
        p = f"layer{i}"
        state.update({f"{p}.wq": L.wq, f"{p}.wk": rep(L.wk), f"{p}.wv": rep(L.wv),
                      f"{p}.wo": L.wo, f"{p}.attn_norm": L.attn_norm, f"{p}.mlp_norm": L.mlp_norm,
                      f"{p}.w_up": L.w_up, f"{p}.w_down": L.w_down, f"{p}.w_gate": L.w_gate,
                      f"{p}.lora_q.a": L.lora_q[0], f"{p}.lora_q.b": L.lora_q[1],
                      f"{p}.lora_v.a": L.lora_v[0], f"{p}.lora_v.b": rep(L.lora_v[1])})
    rng = np.random.default_rng(8)
    tokens = rng.integers(0, GQA_CFG["vocab_size"], size=300)
    out = {"tokens": tokens}
    for mode in ("dense", "fraction"):
        m = model_mod.DecoderModel(model_mod.ModelConfig(**GQA_CFG), seed=0)
        m.load_state_arrays({k: np.asarray(v, np.float32) for k, v in state.items()})
        src = model_mod.FractionSource(0.5, 16) if mode == "fraction" else None
        loss, _ = m.forward_step(tokens, segments=2, pattern_source=src)
        T.backward(loss)
        out[f"{mode}_loss"] = np.array(float(loss.data))
        for name, gr in _grads(m).items():
            if name.endswith("lora_v.b"):  # fold the repeated head blocks
                gr = np.concatenate([sum(gr[:, hd * d:(hd + 1) * d]
                                         for hd in range(kvh * g, (kvh + 1) * g))
                                     for kvh in range(GQA_KV_HEADS)], axis=-1)
            out[f"{mode}_grad__{name}"] = gr
    np.savez_compressed(OUT / "step_gqa.npz", **out)
    return {k: float(v) for k, v in out.items() if k.endswith("_loss")}


CASES = {"select": select_cases, "quantile": quantile_cases, "colsum": column_sum_cases,
         "predictor": predictor_case, "scorers": scorer_cases, "steps": step_cases,
         "patterns": step_pattern_cases, "steps_d128": lambda: step_cases("_d128"),
         "patterns_d128": lambda: step_pattern_cases("_d128"), "predictor_train": predictor_train_case,
         "predictor_train_token": lambda: predictor_train_case("token"),
         "artifacts": artifact_case, "tune": tune_case, "gqa": gqa_case}


def main():
    np.show_config() if "-v" in sys.argv else None
    names = [a for a in sys.argv[1:] if not a.startswith("-")] or list(CASES)
    for name in names:
        print(name, CASES[name]())
    print("wrote", sorted(p.name for p in OUT.glob("*.*")))


if __name__ == "__main__":
    main()
