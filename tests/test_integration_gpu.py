"""The INTEGRATION.md binding exercised from the reference's own code.

The unmodified reference (`sparsetune`, installed into baseline/_ref; the
test skips when it is absent) runs a whole training step -- its own model,
pattern sources, tape and backward -- twice: as shipped, and with
`sparsity.eliminate` and `kernels.segmented_loss_and_grad` rerouted through
liblemo by the maintainer-side ctypes stub (tests/lemo_ffi_stub.py, which
does not import this repository's package).  The masks must be identical
(selection is bit-exact given the same scores), the loss and every LoRA
gradient within the bf16 tolerance of the logits GEMM.
"""

import importlib
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "baseline" / "_ref"
LIB = ROOT / "paper_2501_09767_b200" / "liblemo.so"

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sparsetune():
    if not (REF / "sparsetune" / "__init__.py").exists():
        pytest.skip("reference not installed into baseline/_ref")
    sys.path.insert(0, str(REF))
    try:
        mods = {n: importlib.import_module(f"sparsetune.{n}")
                for n in ("model", "sparsity", "kernels", "tensor", "predictor")}
    finally:
        sys.path.remove(str(REF))
    return mods


def _run(st, tokens, patched_ops=None):
    M, S, K, T, P = (st[n] for n in ("model", "sparsity", "kernels", "tensor", "predictor"))
    saved = (S.eliminate, K.segmented_loss_and_grad)
    if patched_ops is not None:
        S.eliminate = patched_ops.eliminate
        K.segmented_loss_and_grad = patched_ops.segmented_loss_and_grad
    try:
        cfg = M.ModelConfig(n_layers=2, hidden_dim=256, n_heads=2, vocab_size=512,
                            max_seq_len=512, mlp_dim=688, block_size=16, lora_rank=8,
                            lora_alpha=16.0)
        m = M.DecoderModel(cfg, seed=4)
        rng = np.random.default_rng(9)
        for layer in m.layers:  # nonzero B so every adapter carries gradient
            for ad in (layer.lora_q, layer.lora_v):
                ad.b.data[...] = (rng.standard_normal(ad.b.shape) * 0.1).astype(np.float32)
        prng = np.random.default_rng(10)
        m.attach_predictors({l: (P.Predictor.create(prng, 256, 64, 64, 64, "q", l),
                                 P.Predictor.create(prng, 256, 64, 64, 64, "k", l))
                             for l in range(2)})
        x0 = m.embed.data[tokens]
        t_mlp = float(M.mlp_block_score_vector(m.layers[0], x0, 16, len(tokens)).mean())
        ts = S.ThresholdSet({(l, c): (t_mlp if c == S.MLP else 0.0)
                             for l in range(2) for c in S.COMPONENTS})
        src = M.PredictedPatternSource(m, ts, target_retention={0: 0.5, 1: 0.5},
                                       recalibrate_every=1)
        patterns = {}
        orig = src.pattern

        def recording(layer_id, component, x, n_valid):
            p = orig(layer_id, component, x, n_valid)
            patterns[(layer_id, component)] = None if p is None else p.retained_blocks
            return p

        src.pattern = recording
        loss, _ = m.forward_step(tokens, pattern_source=src, segments=4)
        T.backward(loss)
        grads = {f"{l}.{tag}.{ab}": getattr(getattr(layer, tag), ab).grad.copy()
                 for l, layer in enumerate(m.layers) for tag in ("lora_q", "lora_v")
                 for ab in ("a", "b")}
        return float(loss.data), grads, patterns
    finally:
        S.eliminate, K.segmented_loss_and_grad = saved


def test_reference_step_through_the_ctypes_binding(cuda, sparsetune):
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from lemo_ffi_stub import LemoOps

    ops = LemoOps(LIB, sparsetune["sparsity"], sparsetune["tensor"])
    tokens = np.random.default_rng(3).integers(0, 512, size=400)
    loss_ref, g_ref, pat_ref = _run(sparsetune, tokens)
    loss_gpu, g_gpu, pat_gpu = _run(sparsetune, tokens, ops)
    assert pat_gpu == pat_ref and len(pat_ref) == 4           # identical masks
    assert any(p is not None and len(p) < 25 for p in pat_ref.values())  # real sparsity
    assert abs(loss_gpu - loss_ref) <= 1e-2 * abs(loss_ref), (loss_gpu, loss_ref)
    for name, r in g_ref.items():
        err = np.linalg.norm(g_gpu[name] - r) / max(np.linalg.norm(r), 1e-30)
        assert err <= 3e-2, (name, err)
    # the binding's eliminate is bit-exact against the reference on raw vectors
    S = sparsetune["sparsity"]
    rng = np.random.default_rng(5)
    for nb in (1, 7, 64, 1000):
        v = rng.integers(0, 6, nb).astype(np.float64)
        for thr in (float("-inf"), 2.0, 9.0):
            want = S.eliminate(v, thr, block_size=16, n_tokens=nb * 16 - 3, force_blocks=(0,))
            got = ops.eliminate(v, thr, block_size=16, n_tokens=nb * 16 - 3, force_blocks=(0,))
            assert got.retained_blocks == want.retained_blocks
            assert np.array_equal(got.token_indices, want.token_indices)


@pytest.mark.parametrize("block", ["attention", "mlp"])
def test_fused_blocks_accept_the_reference_layer(cuda, sparsetune, block):
    """sparse_attention_fused / sparse_mlp_fused(x, plan, layer) called with
    the REFERENCE's own LayerState (duck-typed fields, kernels.py:295-313):
    output, input gradient and LoRA gradients vs the reference's fused block
    on its tape."""
    import torch

    from paper_2501_09767_b200 import kernels as K

    M, Kr, T = sparsetune["model"], sparsetune["kernels"], sparsetune["tensor"]
    cfg = M.ModelConfig(n_layers=1, hidden_dim=256, n_heads=2, vocab_size=64, max_seq_len=512,
                        mlp_dim=344, block_size=16, lora_rank=8, lora_alpha=16.0)
    ref_model = M.DecoderModel(cfg, seed=2)
    layer = ref_model.layers[0]
    rng = np.random.default_rng(4)
    for ad in (layer.lora_q, layer.lora_v):
        ad.b.data[...] = (rng.standard_normal(ad.b.shape) * 0.1).astype(np.float32)
    s = 320
    x = rng.standard_normal((s, 256)).astype(np.float32)
    up = rng.standard_normal((s, 256)).astype(np.float32)
    idx = np.concatenate([np.arange(0, 96), np.arange(160, 224), np.arange(288, 320)])
    # reference
    xt = T.Tensor(x, requires_grad=True)
    fn_ref = Kr.sparse_attention_fused if block == "attention" else Kr.sparse_mlp_fused
    out_ref = fn_ref(xt, Kr.GatherPlan(idx, s), layer)
    loss = T.sum_all(T.mul(out_ref, T.Tensor(up)))
    T.backward(loss)
    # ours, same layer object
    xd = torch.as_tensor(x).cuda().requires_grad_(True)
    fn = K.sparse_attention_fused if block == "attention" else K.sparse_mlp_fused
    out = fn(xd, K.GatherPlan(idx, s), layer)
    (out * torch.as_tensor(up).cuda()).sum().backward()
    np.testing.assert_allclose(out.detach().cpu().numpy(), out_ref.data, rtol=2e-2, atol=2e-2)
    gx = xd.grad.cpu().numpy()
    assert np.linalg.norm(gx - xt.grad) <= 2e-2 * np.linalg.norm(xt.grad)
    if block == "attention":
        grads = K.shadow_adapter_grads(layer)
        for tag in ("lora_q", "lora_v"):
            for ab in ("a", "b"):
                r = getattr(getattr(layer, tag), ab).grad
                g = grads[f"{tag}.{ab}"]
                assert np.linalg.norm(g - r) <= 3e-2 * np.linalg.norm(r), (tag, ab)
