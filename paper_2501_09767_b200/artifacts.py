"""Artifact compatibility with the reference pipeline.

The GPU path consumes — and writes — the reference's own artifacts, so masks
can be compared across implementations on trained predictors:

* the ``STCHKPT`` binary container (checkpoint.py:17-104): magic, version,
  header length, JSON header (endianness, tensor directory, config, meta),
  little-endian payloads, tensors sorted by name; byte-identical round trip;
* ``predictors.ckpt`` (pipeline.py:370-418): keys ``pred/L{l}/{role}/{name}``,
  meta ``config_hash``, ``pred_thresholds``, ``target_retention``, ``ranks``,
  ``pooling``;
* ``thresholds.json`` (pipeline.py:226-244): ``ThresholdSet.to_dict``;
* the configuration hash the pipeline stamps into every artifact
  (config.py:84-99).

Host-side file IO only (bytes and JSON); tensors land on the GPU through
`Predictor.load_state_arrays`.
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np

from .errors import ContractError, DependencyError, LoadError
from .sparsity import ThresholdSet

MAGIC = b"STCHKPT\x01"
VERSION = 1
PREDICTORS_FILE = "predictors.ckpt"
THRESHOLDS_FILE = "thresholds.json"


# ---------------------------------------------------------------------------
# container


def save_container(path, tensors: dict, config: dict | None = None,
                   meta: dict | None = None) -> None:
    """checkpoint.py:22-58: tensors in name order, contiguous little-endian."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    directory, payloads, offset = [], [], 0
    for name in sorted(tensors):
        arr = np.ascontiguousarray(tensors[name])
        if arr.dtype.byteorder == ">":
            arr = arr.astype(arr.dtype.newbyteorder("<"))
        payload = arr.tobytes()
        directory.append({"name": name, "dtype": arr.dtype.str, "shape": list(arr.shape),
                          "offset": offset, "nbytes": len(payload)})
        payloads.append(payload)
        offset += len(payload)
    header = json.dumps({"endianness": "little", "tensors": directory, "config": config or {},
                         "meta": meta or {}}).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(VERSION.to_bytes(4, "little"))
        fh.write(len(header).to_bytes(8, "little"))
        fh.write(header)
        for payload in payloads:
            fh.write(payload)


def load_container(path) -> tuple[dict, dict, dict]:
    """checkpoint.py:61-104, with the same LoadError checks (truncation, magic,
    version, header JSON, endianness, out-of-range / overlapping entries,
    payload size)."""
    path = Path(path)
    try:
        blob = path.read_bytes()
    except OSError as exc:
        raise LoadError(f"cannot read checkpoint {path}: {exc}") from exc
    if len(blob) < len(MAGIC) + 12:
        raise LoadError(f"{path}: truncated header")
    if blob[:len(MAGIC)] != MAGIC:
        raise LoadError(f"{path}: bad magic, not a checkpoint container")
    version = int.from_bytes(blob[8:12], "little")
    if version != VERSION:
        raise LoadError(f"{path}: unsupported container version {version}")
    header_end = 20 + int.from_bytes(blob[12:20], "little")
    if len(blob) < header_end:
        raise LoadError(f"{path}: truncated header block")
    try:
        header = json.loads(blob[20:header_end].decode("utf-8"))
    except (UnicodeDecodeError, json.JSONDecodeError) as exc:
        raise LoadError(f"{path}: corrupt header json: {exc}") from exc
    if header.get("endianness") != "little":
        raise LoadError(f"{path}: unsupported endianness {header.get('endianness')!r}")
    payload = memoryview(blob)[header_end:]
    spans = []
    for e in header["tensors"]:
        end = e["offset"] + e["nbytes"]
        if end > len(payload):
            raise LoadError(f"{path}: tensor {e['name']!r} extends past end of file")
        spans.append((e["offset"], end, e["name"]))
    spans.sort()
    for (_, e0, n0), (s1, _, n1) in zip(spans, spans[1:]):
        if s1 < e0:
            raise LoadError(f"{path}: directory entries {n0!r} and {n1!r} overlap")
    tensors = {}
    for e in header["tensors"]:
        arr = np.frombuffer(payload[e["offset"]:e["offset"] + e["nbytes"]],
                            dtype=np.dtype(e["dtype"]))
        expected = int(np.prod(e["shape"])) if e["shape"] else 1
        if arr.size != expected:
            raise LoadError(f"{path}: tensor {e['name']!r} payload size mismatch")
        tensors[e["name"]] = arr.reshape(e["shape"]).copy()
    return tensors, header.get("config", {}), header.get("meta", {})


# ---------------------------------------------------------------------------
# configuration hash


def config_hash(model_cfg, mlp_scoring: bool = True) -> str:
    """RunConfig.config_hash (config.py:84-99): sha256 of the pattern-relevant
    geometry, first 16 hex digits."""
    m = model_cfg
    fields = {"block_size": m.block_size, "n_layers": m.n_layers,
              "hidden_dim": m.hidden_dim, "n_heads": m.n_heads,
              "vocab_size": m.vocab_size, "mlp_variant": m.mlp_variant,
              "mlp_dim": m.mlp_dim, "positions": m.positions,
              "mlp_scoring": mlp_scoring}
    # grouped-query attention (beyond the reference) changes the exact scores
    # and so the thresholds / predictors: it enters the key only when present,
    # so multi-head configurations keep the reference's hash
    kv = getattr(m, "n_kv_heads", 0)
    if kv and kv != m.n_heads:
        fields["n_kv_heads"] = kv
    key = json.dumps(fields, sort_keys=True)
    return hashlib.sha256(key.encode()).hexdigest()[:16]


# ---------------------------------------------------------------------------
# predictors.ckpt / thresholds.json


def save_predictors(path, pairs: dict, pred_thresholds: ThresholdSet,
                    retention: dict | None = None, *, ranks=None, pooling: str = "mean",
                    cfg_hash: str = "", config: dict | None = None) -> None:
    """pipeline.py:370-385: same keys and meta as the reference writer."""
    tensors = {}
    for layer_id, (p_q, p_k) in pairs.items():
        for p in (p_q, p_k):
            for name, arr in p.state_arrays().items():
                tensors[f"pred/L{layer_id}/{p.role}/{name}"] = arr
    if ranks is None:
        p0 = next(iter(pairs.values()))[0]
        ranks = [int(p0.w1.shape[1]), int(p0.w2.shape[1]), int(p0.w3.shape[1])]
    meta = {"config_hash": cfg_hash, "pred_thresholds": pred_thresholds.to_dict(),
            "target_retention": {str(k): v for k, v in (retention or {}).items()},
            "ranks": list(ranks), "pooling": pooling}
    save_container(path, tensors, config or {}, meta)


def load_predictors(path, *, n_layers: int, hidden_dim: int, cfg_hash: str | None = None,
                    device=None):
    """pipeline.py:388-418 onto the GPU: returns (pairs, pred_thresholds,
    target_retention, meta).  A config-hash mismatch is a ContractError, a
    missing file a DependencyError, as in the reference."""
    from .predictor import Predictor  # noqa: WPS433 (device-side class)

    path = Path(path)
    if path.is_dir():
        path = path / PREDICTORS_FILE
    if not path.exists():
        raise DependencyError(
            f"missing predictor artifact {path}; run the `train-predictors` step first")
    tensors, _, meta = load_container(path)
    if cfg_hash is not None and meta.get("config_hash") != cfg_hash:
        raise ContractError("predictors were generated under a different configuration; "
                            "rerun `train-predictors`")
    r1, r2, d_pred = meta["ranks"]
    pairs = {}
    for layer_id in range(n_layers):
        pair = []
        for role in ("q", "k"):
            prefix = f"pred/L{layer_id}/{role}/"
            state = {n[len(prefix):]: a for n, a in tensors.items() if n.startswith(prefix)}
            if not state:
                raise ContractError(f"predictor for layer {layer_id}/{role} missing")
            p = Predictor(np.zeros((hidden_dim, r1), np.float32), np.zeros((r1, r2), np.float32),
                          np.zeros((r2, d_pred), np.float32), role, layer_id, device)
            p.load_state_arrays(state)
            pair.append(p)
        pairs[layer_id] = tuple(pair)
    pred_thresholds = ThresholdSet.from_dict(meta["pred_thresholds"])
    retention = {int(k): float(v) for k, v in meta.get("target_retention", {}).items()}
    return pairs, pred_thresholds, retention, meta


def save_thresholds(path, ts: ThresholdSet) -> None:
    """pipeline.py:226: indent-2 JSON of ThresholdSet.to_dict + newline."""
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text(json.dumps(ts.to_dict(), indent=2) + "\n")


def load_thresholds(path, cfg_hash: str | None = None) -> ThresholdSet:
    """pipeline.py:230-244."""
    path = Path(path)
    if path.is_dir():
        path = path / THRESHOLDS_FILE
    if not path.exists():
        raise DependencyError(
            f"missing thresholds artifact {path}; run the `tune-thresholds` step first")
    ts = ThresholdSet.from_dict(json.loads(path.read_text()))
    if cfg_hash is not None and ts.config_hash != cfg_hash:
        raise ContractError("thresholds were generated under a different configuration "
                            f"(hash {ts.config_hash} != {cfg_hash}); rerun the pipeline")
    return ts


__all__ = ["MAGIC", "VERSION", "save_container", "load_container", "config_hash",
           "save_predictors", "load_predictors", "save_thresholds", "load_thresholds"]
