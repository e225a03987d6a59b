"""Which side drifts in the bench's early layers: bf16 scores, parity scores
or neither?  Llama2-7B width, torch init (bf16-valued weights), real residual
stream (embedding + attention of layer 0), s = 4096; MLP scores of layer 0
vs the f32 oracle computed from the same weights."""
import math
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from oracle import lemo_oracle as O  # noqa: E402
from paper_2501_09767_b200 import kernels, model as M, ops  # noqa: E402

s = 4096
cfg = M.llama2_7b(n_layers=1, max_seq_len=s)
model = M.DecoderModel(cfg, seed=0, init="torch", parity_weights=True)
layer = model.layers[0]
print("parity_terms", layer.parity_terms)
tokens = np.random.default_rng(1000).integers(0, cfg.vocab_size, size=s)
ids = torch.as_tensor(tokens.astype(np.int32)).cuda()
x = ops.embed(ids, model.embed, None)
def f32e(xx):
    N = layer.w_gu_t.shape[0]
    inv = torch.empty(s, device="cuda")
    xn = ops.rmsnorm_gather(xx, layer.mlp_norm_w, None, inv=inv)
    part = torch.empty(N // 128, s, device="cuda")
    ops.gemm_gateup(xn, layer.w_gu_t, partial=part, exact_score=True)
    return ops.mlp_block_scores(part, s=s, n_valid=s, b=16, m_real=layer.m).cpu().numpy()


for name, xx in (("embedding", x), ("embedding x64", x * 64), ("random", torch.randn(s, 4096, device="cuda"))):
    v16 = M.mlp_block_score_vector(layer, xx, 16, s, precision="bf16").cpu().numpy()
    v32 = M.mlp_block_score_vector(layer, xx, 16, s, precision="fp32").cpu().numpy()
    # oracle from the weights as stored (bf16 values, interleaved gate/up undone)
    m = cfg.mlp_dim
    gu = layer.w_gu_t.float().cpu().numpy()  # [2*m_pad, h]
    mp = layer.m_pad
    g_t = gu.reshape(mp // 128, 2, 128, 4096)[:, 0].reshape(mp, 4096)[:m]
    u_t = gu.reshape(mp // 128, 2, 128, 4096)[:, 1].reshape(mp, 4096)[:m]
    L = O.Layer(None, None, None, None, np.ones(4096, np.float32), layer.mlp_norm_w.cpu().numpy(),
                np.ascontiguousarray(u_t.T), None, np.ascontiguousarray(g_t.T), None, None, 1.0, 32,
                True, 1e4, "silu")
    vo = O.mlp_block_score_vector(L, xx.cpu().numpy(), 16, s)
    sc = np.abs(vo).max()
    ve = f32e(xx)
    print(f"{name}: bf16-operands+fp32-epilogue vs oracle {np.abs(ve - vo).max() / np.abs(vo).max():.2e}")
    print(f"{name}: bf16 vs oracle {np.abs(v16 - vo).max() / sc:.2e}, fp32 vs oracle "
          f"{np.abs(v32 - vo).max() / sc:.2e}, bf16 vs fp32 {np.abs(v16 - v32).max() / sc:.2e}, "
          f"score spread {(vo.max() - vo.min()) / vo.mean():.3f}", flush=True)
