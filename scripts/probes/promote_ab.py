"""A/B of the promotion group: parity-mode gate/up GEMM time at Llama2-7B
width (s = 16384, bf16-exact weights -> 2-term form) and the MLP score
error vs the f32 oracle at s = 4096."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[2] / "tests"))
from oracle import lemo_oracle as O  # noqa: E402
from paper_2501_09767_b200 import model as M  # noqa: E402
from test_parity_gpu import WIDTH, oracle_arrays  # noqa: E402

for weights in ("bf16", "fp32"):
    s = 4096
    cfg = dict(WIDTH, max_seq_len=16384)
    om = O.init_model(O.Config(**cfg), seed=11, fast=True)
    L = om.layers[0]
    if weights == "bf16":
        for n in ("wq", "wk", "wv", "wo", "w_up", "w_down", "w_gate"):
            setattr(L, n, torch.as_tensor(getattr(L, n)).bfloat16().float().numpy())
    model = M.DecoderModel(M.ModelConfig(**cfg), 0, arrays=oracle_arrays(om), scoring_precision="fp32")
    layer = model.layers[0]
    x = np.random.default_rng(13).standard_normal((s, 4096), dtype=np.float32)
    ref = O.mlp_block_score_vector(L, x, 16, s)
    got = M.mlp_block_score_vector(layer, torch.as_tensor(x).cuda(), 16, s).cpu().numpy()
    xb = torch.randn(16384, 4096, device="cuda")
    f = lambda: M.mlp_block_score_vector(layer, xb, 16, 16384)  # noqa: E731
    f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(5):
        f()
    b.record()
    torch.cuda.synchronize()
    print(f"weights={weights} terms={layer.parity_terms}: score max rel err "
          f"{np.abs(got - ref).max() / np.abs(ref).max():.2e}, 16K scoring "
          f"{a.elapsed_time(b) / 5:.2f} ms", flush=True)
