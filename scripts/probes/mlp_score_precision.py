"""Where does the production (bf16) MLP score error come from?  One
Llama2-7B-width layer at s tokens, scores vs the f32 oracle:
  bf16       production: bf16 operands, bf16-rounded gate/up in the epilogue
  bf16+f32e  bf16 operands, scores from the (promoted) fp32 accumulator
  fp32       parity precision (bf16x3 operands, promoted, fp32 epilogue)"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
from oracle import lemo_oracle as O  # noqa: E402
from paper_2501_09767_b200 import model as M, ops  # noqa: E402
from test_parity_gpu import WIDTH, oracle_arrays  # noqa: E402

s = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
cfg = dict(WIDTH, max_seq_len=s)
om = O.init_model(O.Config(**cfg), seed=11, fast=True)
model = M.DecoderModel(M.ModelConfig(**cfg), 0, arrays=oracle_arrays(om), scoring_precision="fp32")
layer = model.layers[0]
x = np.random.default_rng(13).standard_normal((s, 4096), dtype=np.float32)
ref = O.mlp_block_score_vector(om.layers[0], x, 16, s)
xd = torch.as_tensor(x).cuda()


def variant(exact_epi):
    N = layer.w_gu_t.shape[0]
    inv = torch.empty(s, device="cuda")
    xn = ops.rmsnorm_gather(xd, layer.mlp_norm_w, None, inv=inv)
    part = torch.empty(N // 128, s, device="cuda")
    ops.gemm_gateup(xn, layer.w_gu_t, partial=part, relu=layer.relu, exact_score=exact_epi)
    return ops.mlp_block_scores(part, s=s, n_valid=s, b=16, m_real=layer.m).cpu().numpy()


res = {"bf16": variant(False), "bf16+f32e": variant(True),
       "fp32": M.mlp_block_score_vector(layer, xd, 16, s, precision="fp32").cpu().numpy()}
thr = float(ref.mean())
for k, v in res.items():
    d = v - ref
    print(f"{k:10s} max rel {np.abs(d).max() / np.abs(ref).max():.2e}  mean signed rel "
          f"{(d / ref).mean():+.2e}  flips {int(((v >= thr) != (ref >= thr)).sum())}/{len(ref)}")
