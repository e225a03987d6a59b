"""Ledger host logic (reference tests/test_ledger.py:12-80 restated) and, on the
GPU, the memory law of acceptance criterion 9 (tests/test_acceptance.py:511-553):
block activation bytes linear in the retained fraction, the activation peak
affine in the sequence length."""

import gc
import numpy as np
import pytest

from paper_2501_09767_b200 import ledger as L
from paper_2501_09767_b200.errors import AccountingError


def test_alloc_free_returns_to_baseline():
    led = L.Ledger()
    h = led.alloc(100, L.TRANSIENT)
    assert led.live_bytes() == 100
    led.free(h)
    assert led.live_bytes() == 0


def test_free_without_alloc_is_accounting_error():
    with pytest.raises(AccountingError):
        L.Ledger().free(12345)


def test_nested_scopes_attribute_to_innermost():
    led = L.Ledger()
    with led.scope("outer"):
        with led.scope("inner"):
            led.alloc(64, L.TRANSIENT)
    assert led.peak_by_site.get("inner") == 64 and "outer" not in led.peak_by_site


def test_refcounted_retention_counts_once():
    led = L.Ledger()
    arr = np.zeros(10, dtype=np.float32)
    led.retain_array(arr, L.ACTIVATION)
    led.retain_array(arr, L.ACTIVATION)
    assert led.live_bytes() == arr.nbytes
    led.release_array(arr)
    assert led.live_bytes() == arr.nbytes
    led.release_array(arr)
    assert led.live_bytes() == 0
    with pytest.raises(AccountingError):
        led.release_array(arr)


def test_peaks_dominate_instantaneous_sums():
    led = L.Ledger()
    h1 = led.alloc(100, L.TRANSIENT)
    h2 = led.alloc(50, L.ACTIVATION)
    led.free(h1)
    led.free(h2)
    rep = led.report()
    assert rep.peak_total_bytes == 150
    assert all(rep.peak_total_bytes >= v for v in rep.peak_by_category.values())
    assert all(live <= rep.peak_total_bytes for _, live in rep.series)


def test_model_states_bytes():
    assert L.model_states_bytes(175e9) == 2.8e12 and L.model_states_bytes(7e9) == 112e9
    with pytest.raises(ValueError):
        L.model_states_bytes(0)


def test_affine_fit_exact_line():
    a, c, r2 = L.affine_fit([1.0, 2.0, 3.0], [5.0, 7.0, 9.0])
    assert (a, c, r2) == (2.0, 3.0, 1.0)


@pytest.mark.gpu
def test_memory_law_on_gpu(cuda):
    from paper_2501_09767_b200 import model as M

    cfg = M.ModelConfig(n_layers=2, hidden_dim=256, n_heads=2, vocab_size=256,
                        max_seq_len=2048, mlp_dim=688, block_size=16)
    model = M.DecoderModel(cfg, 0, device=cuda)
    scopes = [f"layer{i}.{c}" for i in range(cfg.n_layers) for c in ("attn", "mlp")]
    rng = np.random.default_rng(0)

    def step(tokens, source):
        # objects left by earlier tests must not be collected inside the step:
        # their frees would shrink the allocator delta the ledger is checked against
        gc.collect()
        gc.disable()
        try:
            led = L.Ledger(keep_series=False)
            with L.use(led):
                loss, _ = model.forward_step(tokens, pattern_source=source)
                post = led.marks["post_forward"]
                loss.backward()
            rep = led.report()
        finally:
            gc.enable()
        assert rep.leaked_bytes == 0 and led.live_bytes() == 0
        return rep, post

    tokens = rng.integers(0, 256, size=1024)
    fracs = [1.0, 0.5, 0.25]
    nbytes = []
    for f in fracs:
        rep, post = step(tokens, M.FractionSource(f, cfg.block_size))
        nbytes.append(float(rep.activation_bytes(*scopes)))
        # the logical ledger accounts for what the allocator holds at the mark
        alloc = model.last_stats["activation_bytes_post_forward"]
        assert 0.8 * alloc <= post <= alloc * 1.001, (post, alloc)
    slope, intercept, _ = L.affine_fit(fracs, nbytes)
    for f, b in zip(fracs, nbytes):
        assert abs((b - intercept) - slope * f) <= 0.05 * max(slope * f, 1.0)
    ratio = (nbytes[1] - intercept) / (nbytes[0] - intercept)
    assert abs(ratio - 0.5) <= 0.035
    peaks = []
    sizes = [256, 512, 1024, 2048]
    for s in sizes:
        rep, _ = step(rng.integers(0, 256, size=s), None)
        peaks.append(float(rep.peak_by_category[L.ACTIVATION]))
    _, _, r2 = L.affine_fit([float(s) for s in sizes], peaks)
    assert r2 > 0.99
