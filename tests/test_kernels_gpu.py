"""Hot-path equivalences of the reference's own test strategy on the GPU path
(SURVEY.md §4): value semantics and bit-exact eliminated rows of the fused
blocks (tests/test_kernels.py:117-124), the eliminated-token gradient
(tests/test_model.py:269-314), fused ≡ naive (tests/test_kernels.py:61-114),
segment-plan independence (tests/test_kernels.py:190-260) and LoRA at init ≡
frozen (tests/test_model.py:34-50)."""

import numpy as np
import pytest
import torch

from paper_2501_09767_b200 import kernels as K, model as M

pytestmark = pytest.mark.gpu
CFG = dict(n_layers=2, hidden_dim=256, n_heads=2, vocab_size=256, max_seq_len=512, mlp_dim=688,
           block_size=16, lora_rank=8, lora_alpha=16.0)


def _model(cuda, **kw):
    cfg = M.ModelConfig(**{**CFG, **kw})
    m = M.DecoderModel(cfg, 11, device=cuda, init="reference")
    if cfg.lora_rank:
        with torch.no_grad():  # nonzero B so the LoRA path carries gradient
            g = torch.Generator(device=cuda).manual_seed(5)
            m.lora_param.add_(0.05 * torch.randn(m.lora_param.shape, generator=g, device=cuda))
    return m


@pytest.mark.parametrize("block", ["attention", "mlp"])
def test_fused_block_semantics_and_eliminated_rows(cuda, block):
    model = _model(cuda)
    layer = model.layers[0]
    g = torch.Generator(device=cuda).manual_seed(3)
    s = 304
    x = torch.randn(s, 256, device=cuda, generator=g)
    idx = np.unique(np.concatenate([np.arange(0, 64), np.arange(128, 176), np.arange(288, 304)]))
    plan = K.GatherPlan(idx, s)
    fn = K.sparse_attention_fused if block == "attention" else K.sparse_mlp_fused
    naive = K.sparse_attention_naive if block == "attention" else K.sparse_mlp_naive
    x0 = x.clone()
    xr = x.clone().requires_grad_(True)
    out = fn(xr, plan, layer)
    assert torch.equal(x, x0)                     # inputs are not modified
    keep = np.setdiff1d(np.arange(s), idx)
    assert torch.equal(out[keep], x[keep])         # eliminated rows bit-exact
    assert not torch.equal(out[idx], x[idx])
    # fused ≡ naive (tests/test_kernels.py:61-114): the naive path gathers into
    # a materialised compact copy, runs the block there with RoPE at the
    # original positions and pads/adds through two more buffers
    xn_ = x.clone().requires_grad_(True)
    out2 = naive(xn_, plan, layer)
    torch.testing.assert_close(out.detach(), out2.detach(), rtol=1e-6, atol=1e-6)
    # eliminated-token gradient: a row the block did not process passes the
    # upstream gradient through unchanged
    up = torch.randn(s, 256, device=cuda, generator=g)
    out.backward(up)
    assert torch.equal(xr.grad[keep], up[keep])
    assert not torch.equal(xr.grad[idx], up[idx])
    lora_fused = model.lora_param.grad.clone()
    model.lora_param.grad = None
    out2.backward(up)                              # grads fused ≡ naive (:163-176)
    torch.testing.assert_close(xn_.grad, xr.grad, rtol=1e-5, atol=1e-6)
    torch.testing.assert_close(model.lora_param.grad, lora_fused, rtol=1e-5, atol=1e-7)
    if block == "attention":
        assert float(lora_fused.abs().sum()) > 0


def test_empty_plan_returns_input(cuda):
    model = _model(cuda)
    x = torch.randn(64, 256, device=cuda)
    assert K.sparse_attention_fused(x, K.GatherPlan.empty(64), model.layers[0]) is x
    assert K.sparse_mlp_fused(x, K.GatherPlan.empty(64), model.layers[0]) is x


def test_segment_plan_independence(cuda):
    """Uneven, even and single-segment plans give the same loss (the segment
    partition only bounds the logits buffer)."""
    model = _model(cuda)
    tokens = np.random.default_rng(4).integers(0, 256, 300)
    losses = []
    for seg in (1, 3, 8):
        loss, _ = model.forward_step(tokens, segments=seg)
        losses.append(float(loss.detach()))
    assert max(abs(l - losses[0]) for l in losses) <= 1e-5 * abs(losses[0])


def test_lora_at_init_equals_frozen(cuda):
    """B = 0 at init: the LoRA model computes the frozen model's loss exactly."""
    cfg = M.ModelConfig(**CFG)
    arrays = M.reference_init_arrays(cfg, 2)       # reference init: B = 0
    with_lora = M.DecoderModel(cfg, 2, arrays=arrays, device=cuda)
    frozen_arrays = {k: v for k, v in arrays.items() if ".lora_" not in k}
    frozen = M.DecoderModel(M.ModelConfig(**{**CFG, "lora_rank": 0}), 2, arrays=frozen_arrays,
                            device=cuda)
    tokens = np.random.default_rng(6).integers(0, 256, 200)
    a, _ = with_lora.forward_step(tokens, segments=2)
    b, _ = frozen.forward_step(tokens, segments=2)
    assert float(a.detach()) == float(b.detach())


@pytest.mark.parametrize("trainable_head", [False, True])
def test_segmented_loss_and_grad_reference_api(cuda, trainable_head):
    """kernels.segmented_loss_and_grad(hidden, lm_head, targets, plan,
    ignore_index=-1) -- the reference's custom_op client (kernels.py:229-288):
    loss, d hidden (and d lm_head when it requires grad) vs the oracle, the
    reference's contract errors, and segment-count independence."""
    from oracle import lemo_oracle as O
    from paper_2501_09767_b200.errors import ContractError

    rng = np.random.default_rng(9)
    n, h, V = 300, 256, 512
    hid = (rng.standard_normal((n, h)) * 0.5).astype(np.float32)
    W = (rng.standard_normal((h, V)) / 16).astype(np.float32)
    tg = rng.integers(0, V, n)
    tg[::7] = -1
    # the oracle on the bf16-rounded operands the GPU GEMMs consume
    hb = torch.as_tensor(hid).bfloat16().float().numpy()
    Wb = torch.as_tensor(W).bfloat16().float().numpy()
    ref_loss, ref_gh = O.segmented_loss_and_grad(hb, Wb, tg, 3)
    hidden = torch.as_tensor(hid).cuda().requires_grad_(True)
    lm = torch.as_tensor(W).cuda().requires_grad_(trainable_head)
    for seg in (1, 3, 8):
        loss = K.segmented_loss_and_grad(hidden, lm, tg, K.SegmentPlan.even(n, seg))
        assert abs(float(loss) - ref_loss) <= 1e-4 * abs(ref_loss)
    hidden.grad = None
    loss = K.segmented_loss_and_grad(hidden, lm, tg, K.SegmentPlan.even(n, 3))
    (2.0 * loss).backward()
    gh = hidden.grad.cpu().numpy()
    assert np.linalg.norm(gh - 2 * ref_gh) <= 1e-2 * np.linalg.norm(2 * ref_gh)
    if trainable_head:
        # dW = hiddenᵀ·dlogits / count, from the same per-segment dlogits
        probs = np.exp(hb @ Wb - (hb @ Wb).max(1, keepdims=True))
        probs /= probs.sum(1, keepdims=True)
        valid = tg != -1
        probs[np.nonzero(valid)[0], tg[valid]] -= 1.0
        probs[~valid] = 0.0
        ref_gw = 2 * hb.T @ probs / valid.sum()
        gw = lm.grad.cpu().numpy()
        assert np.linalg.norm(gw - ref_gw) <= 1e-2 * np.linalg.norm(ref_gw)
    else:
        assert lm.grad is None
    with pytest.raises(ContractError):
        K.segmented_loss_and_grad(hidden, lm, tg[:-1], K.SegmentPlan.even(n, 2))
    with pytest.raises(ContractError):
        K.segmented_loss_and_grad(hidden, lm, tg, K.SegmentPlan.even(n + 1, 2))
    with pytest.raises(ContractError):
        K.segmented_loss_and_grad(hidden, lm, np.full(n, -1), K.SegmentPlan.even(n, 2))
    with pytest.raises(IndexError):
        K.segmented_loss_and_grad(hidden, lm, np.full(n, V), K.SegmentPlan.even(n, 2))
