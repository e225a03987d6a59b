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
    out2 = naive(x.clone(), plan, layer)
    assert torch.equal(out.detach(), out2)         # fused ≡ naive
    # eliminated-token gradient: a row the block did not process passes the
    # upstream gradient through unchanged
    up = torch.randn(s, 256, device=cuda, generator=g)
    out.backward(up)
    assert torch.equal(xr.grad[keep], up[keep])
    assert not torch.equal(xr.grad[idx], up[idx])
    if block == "attention":
        assert float(model.lora_param.grad.abs().sum()) > 0


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
