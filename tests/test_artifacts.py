"""Artifact compatibility with the reference pipeline and
threshold tuning (§8f row 2, Algorithm 1) — host-side, CPU-only.

Fixtures in tests/golden/ were written by the reference itself
(make_golden.py: artifact_case, tune_case)."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2501_09767_b200 import artifacts as A
from paper_2501_09767_b200 import sparsity as S
from paper_2501_09767_b200.errors import ContractError, DependencyError, LoadError
from paper_2501_09767_b200.model import ModelConfig

G = Path(__file__).resolve().parent / "golden"


def test_container_reads_reference_file_and_rewrites_it_bytewise(tmp_path):
    tensors, config, meta = A.load_container(G / "mixed.ckpt")
    z = np.load(G / "artifacts.npz")
    for name, arr in tensors.items():
        ref = z["t_" + name.replace("/", "_")]
        if ref.shape == ():  # the reference loader returns 0-d tensors as shape (1,)
            ref = ref.reshape(1)
        assert arr.dtype == ref.dtype and arr.shape == ref.shape
        assert np.array_equal(arr, ref)
    assert config == {"k": 1} and meta == {"m": "x"}
    A.save_container(tmp_path / "m.ckpt", tensors, config, meta)
    assert (tmp_path / "m.ckpt").read_bytes() == (G / "mixed.ckpt").read_bytes()


def test_predictors_ckpt_layout_and_bytewise_roundtrip(tmp_path):
    tensors, config, meta = A.load_container(G / "predictors.ckpt")
    for l in range(2):
        for role in ("q", "k"):
            for name in ("w1", "w2", "w3", "mask1", "mask2", "zero_counts1", "zero_counts2",
                         "observed"):
                assert f"pred/L{l}/{role}/{name}" in tensors
    assert meta["ranks"] == [16, 16, 16] and meta["pooling"] == "mean"
    assert S.ThresholdSet.from_dict(meta["pred_thresholds"]).get(1, "attention") == -0.5
    A.save_container(tmp_path / "p.ckpt", tensors, config, meta)
    assert (tmp_path / "p.ckpt").read_bytes() == (G / "predictors.ckpt").read_bytes()


def test_thresholds_json_roundtrip(tmp_path):
    z = np.load(G / "artifacts.npz")
    ts = A.load_thresholds(G / "thresholds.json", cfg_hash=str(z["hash"][0]))
    assert ts.get(1, "mlp") == 7.0 and ts.eps == 0.01 and ts.eta is None
    A.save_thresholds(tmp_path / "t.json", ts)
    assert (tmp_path / "t.json").read_text() == (G / "thresholds.json").read_text()
    with pytest.raises(ContractError):
        A.load_thresholds(G / "thresholds.json", cfg_hash="0" * 16)
    with pytest.raises(DependencyError):
        A.load_thresholds(tmp_path / "missing.json")


def test_config_hash_matches_reference():
    hashes = json.loads((G / "config_hashes.json").read_text())
    for name, (kw, h) in hashes.items():
        cfg = ModelConfig(**kw)
        assert A.config_hash(cfg, mlp_scoring=not name.endswith("_nomlp")) == h, name


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b[:10], "truncated header"),
    (lambda b: b"XXXXXXXX" + b[8:], "bad magic"),
    (lambda b: b[:8] + (2).to_bytes(4, "little") + b[12:], "unsupported container version"),
    (lambda b: b[:-3], "extends past end"),
])
def test_container_load_errors(tmp_path, mutate, msg):
    blob = (G / "mixed.ckpt").read_bytes()
    bad = tmp_path / "bad.ckpt"
    bad.write_bytes(mutate(blob))
    with pytest.raises(LoadError, match=msg):
        A.load_container(bad)


def test_container_overlap_rejected(tmp_path):
    A.save_container(tmp_path / "o.ckpt", {"a": np.arange(4, dtype=np.int32),
                                           "b": np.arange(4, dtype=np.int32)})
    blob = (tmp_path / "o.ckpt").read_bytes()
    hl = int.from_bytes(blob[12:20], "little")
    header = json.loads(blob[20:20 + hl])
    header["tensors"][1]["offset"] = 8  # overlaps "a"
    hb = json.dumps(header).encode()
    (tmp_path / "o.ckpt").write_bytes(blob[:12] + len(hb).to_bytes(8, "little") + hb +
                                      blob[20 + hl:])
    with pytest.raises(LoadError, match="overlap"):
        A.load_container(tmp_path / "o.ckpt")


def test_tune_thresholds_matches_reference():
    ref = json.loads((G / "tune.json").read_text())
    ts = S.ThresholdSet.from_dict(ref["init"])

    def acc(t):
        v = t.values
        return -sum((val - 0.3 * (i + 1)) ** 2 + 0.1 * val ** 3 / (1 + val ** 2)
                    for i, (_, val) in enumerate(sorted(v.items())))

    for name, kw in (("auto", dict(rounds=2)), ("fixed", dict(eps=0.05, eta=0.2, rounds=3))):
        got = S.tune_thresholds(acc, ts, **kw).to_dict()
        assert got == ref[name], name  # bitwise: same float operation order


def test_tune_thresholds_rejects_nonfinite():
    ts = S.ThresholdSet({(0, "attention"): 1.0})
    with pytest.raises(ContractError):
        S.tune_thresholds(lambda t: float("nan"), ts)
