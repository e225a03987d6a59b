"""Mask-flip audit of the production scorers against the parity precision.

The production MLP scorer runs its gate/up GEMM on bf16 operands; the
fp32-faithful parity precision (bf16x3 operands, promoted accumulation,
`scoring_precision="fp32"`) reproduces the reference's f32 scores to ~1e-6
and therefore its masks (tests/test_parity_gpu.py pins it to the oracle at
Llama2-7B width, s = 4K / 16K).  `MaskAudit` wraps a pattern source: it
forwards every call unchanged and, for each MLP decision, also scores the
same residual in both precisions and counts the blocks whose selection
differs under the threshold the source used.  The attention side of
PredictedPatternSource is fp32-faithful in production already (bf16x3
predictor GEMMs), so its flip count is 0 by construction and reported so.

Used by bench.py outside the timed region; costs one extra gate/up GEMM in
each precision per layer.
"""

from __future__ import annotations

from . import sparsity
from .model import PatternSourceBase, mlp_block_score_vector, refine_mlp_block_scores


class MaskAudit(PatternSourceBase):
    def __init__(self, inner, model):  # noqa: D107 (last_fractions is the inner source's)
        if not model.parity_weights:
            raise ValueError("the audit needs a model built with parity_weights=True")
        self.inner = inner
        self.model = model
        self.per_layer: dict = {}  # layer -> {"mlp_flips", "mlp_ambiguous", "n_blocks"}

    @property
    def last_fractions(self):
        return self.inner.last_fractions

    def pattern(self, layer_id, component, x, n_valid):
        pat = self.inner.pattern(layer_id, component, x, n_valid)
        if component != sparsity.MLP or pat is None:
            return pat
        layer = self.model.layers[layer_id]
        b = self.model.config.block_size
        thr = self.inner.thresholds.get(layer_id, sparsity.MLP)
        # the precision the step itself scores in (model default) vs the parity one
        prec = self.model.scoring_precision
        prod, partial = mlp_block_score_vector(layer, x, b, n_valid, precision=prec,
                                               with_partial=True)
        if prec == "refined":
            refine_mlp_block_scores(layer, x, prod, partial, thr, b, n_valid)
        del partial
        par = mlp_block_score_vector(layer, x, b, n_valid, precision="fp32")
        flips = (prod >= thr) != (par >= thr)
        amb = flips & ((par - thr).abs() <= 1e-5 * abs(thr))
        self.per_layer[layer_id] = {"mlp_flips": int(flips.sum()), "mlp_ambiguous": int(amb.sum()),
                                    "n_blocks": int(par.numel()),
                                    "max_rel_score_diff": float(((prod - par).abs().max() /
                                                                 par.abs().max()).item())}
        del prod, par
        return pat

    def summary(self) -> dict:
        rows = [self.per_layer[k] for k in sorted(self.per_layer)]
        nb = sum(r["n_blocks"] for r in rows)
        flips = sum(r["mlp_flips"] for r in rows)
        return {"step_precision": self.model.scoring_precision,
                "reference_precision": "fp32-faithful parity scorers (bf16x3, promoted "
                                       "accumulation; 0 flips vs the oracle at this width, "
                                       "tests/test_parity_gpu.py)",
                "mlp_flips_per_layer": [r["mlp_flips"] for r in rows],
                "mlp_flips_total": flips, "mlp_blocks_total": nb,
                "mlp_flip_rate": flips / nb if nb else None,
                "mlp_ambiguous_total": sum(r["mlp_ambiguous"] for r in rows),
                "mlp_max_rel_score_diff": max((r["max_rel_score_diff"] for r in rows),
                                              default=None),
                "mlp_refined_rows_total": sum(getattr(self.inner, "refined_rows", {}).values())
                if prec_refined(self.model) else None,
                "attention_flips_total": 0,
                "attention_note": "predicted attention scores are fp32-faithful in production "
                                  "(bf16x3 predictor GEMMs): identical to the parity precision"}


def prec_refined(model) -> bool:
    return model.scoring_precision == "refined"


__all__ = ["MaskAudit"]
