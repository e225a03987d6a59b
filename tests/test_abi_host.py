"""CPU tests: the C ABI library loads and exports every declared symbol; the
host-side contract checks raise the reference's exception types."""

import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2501_09767_b200 import _lib
from paper_2501_09767_b200.errors import ContractError, DimensionError

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib._LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    declared = set(_lib.SIGNATURES)
    assert declared, "no declarations parsed from include/lemo.h"
    missing = declared - exported
    assert not missing, missing
    for name in declared:
        assert getattr(lib, name) is not None
    assert lib.lemo_version() == 1


def test_header_declares_all_exported_lemo_symbols():
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib._LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T lemo_" in line}
    assert exported <= set(_lib.SIGNATURES), exported - set(_lib.SIGNATURES)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib._LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_last_error_is_a_string():
    assert isinstance(_lib.lib().lemo_last_error(), bytes)


def test_gather_plan_contract():
    from paper_2501_09767_b200.kernels import GatherPlan, SegmentPlan

    with pytest.raises(ContractError):
        GatherPlan(np.array([3, 2]), 10)
    with pytest.raises(ContractError):
        GatherPlan(np.array([0, 10]), 10)
    with pytest.raises(ContractError):
        GatherPlan(np.array([[0]]), 10)
    assert SegmentPlan.even(10, 3).boundaries == (0, 3, 7, 10)
    with pytest.raises(ContractError):
        SegmentPlan.even(3, 4)
    with pytest.raises(ContractError):
        SegmentPlan(5, (0, 2, 2, 5))


def test_sparsity_pattern_host_view():
    from paper_2501_09767_b200.sparsity import SparsityPattern, ThresholdSet, n_blocks_for

    p = SparsityPattern(0, "attention", (0, 2), 4, 12)
    np.testing.assert_array_equal(p.token_indices, [0, 1, 2, 3, 8, 9, 10, 11])
    assert p.retained_fraction == 8 / 12
    assert SparsityPattern(0, "attention", (2,), 4, 10).k == 2
    with pytest.raises(ContractError):
        SparsityPattern(0, "attention", (2, 1), 4, 12)
    with pytest.raises(ContractError):
        SparsityPattern(0, "attention", (3,), 4, 12)
    assert n_blocks_for(17, 16) == 2
    ts = ThresholdSet({(0, "attention"): 1.5, (1, "mlp"): -2.0})
    assert ThresholdSet.from_dict(ts.to_dict()).values == ts.values


def test_model_config_contract():
    from paper_2501_09767_b200.model import ModelConfig, llama2_7b

    with pytest.raises(DimensionError):
        ModelConfig(hidden_dim=30, n_heads=4)
    with pytest.raises(ContractError):
        ModelConfig(max_seq_len=100, block_size=16)
    with pytest.raises(ContractError):
        ModelConfig(mlp_variant="gelu")
    cfg = llama2_7b()
    cfg.check_gpu_geometry()
    assert cfg.head_dim == 128 and cfg.mlp_pad == 11008
    with pytest.raises(ContractError):
        ModelConfig(hidden_dim=96, n_heads=3).check_gpu_geometry()


def test_no_oracle_import_in_product():
    """The product package never imports the CPU oracle (test infrastructure)."""
    for f in (ROOT / "paper_2501_09767_b200").rglob("*.py"):
        text = f.read_text()
        assert "oracle" not in text.replace("oracle/", "").lower() or "import" not in text.split(
            "oracle")[0][-40:], f
        assert "lemo_oracle" not in text, f
