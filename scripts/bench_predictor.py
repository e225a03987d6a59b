"""Predictor path micro-benchmark at Llama2-7B width (CUDA events, warm):
predicted_block_vector (block_embed -> 2 x 3 bf16x3 GEMMs -> Eq. 3 -> column
sums) at s = 16384 (nb = 1024 blocks, h = 4096, r1 = r2 = d_p = 1024), and the
single bf16x3 predictor GEMMs.  LEMO_LIB selects an A/B build."""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2501_09767_b200 import ops, predictor as P  # noqa: E402


def bench(fn, it=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3  # us


h, r, s = 4096, 1024, 16384
g = torch.Generator(device="cuda").manual_seed(0)
mk = lambda: P.Predictor(*(torch.randn(a, b, generator=g, device="cuda") / math.sqrt(a)  # noqa
                           for a, b in ((h, r), (r, r), (r, r))))
pq, pk = mk(), mk()
x = torch.randn(s, h, device="cuda")
t = bench(lambda: P.predicted_block_vector(pq, pk, x, 16, "mean"))
print(f"predicted_block_vector s={s}: {t:.1f} us")
xb = torch.randn(s // 16, h, device="cuda")
x3 = ops.split_bf16x3(xb, 0)
w1, w2, w3 = pq._weights3()
h1, _ = ops.gemm_split3(x3, w1, relu=True, mask=pq.mask1, pattern=0)
for name, a, w in (("layer1 K=3h", x3, w1), ("layer2 K=3r", h1, w2)):
    M, N, K = a.shape[0], w.shape[0], a.shape[1]
    tt = bench(lambda: ops.gemm_split3(a, w, relu=True, mask=pq.mask1, pattern=0))
    print(f"{name}: M={M} N={N} K'={K}: {tt:.1f} us  {2 * M * N * K / tt / 1e6:.0f} TFLOP/s executed")
