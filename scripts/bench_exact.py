"""Isolated timing of the tcgen05 exact block scorer (sparsity.py:173-219) at
Llama2-7B width (32 heads x 128): production bf16 operands and the
fp32-faithful bf16x3 parity mode.  Work = Σ over causal 128x256 items of
H · 2·128·256·d FLOPs (the kernel's executed MMA work; x3 for bf16x3).

    python scripts/bench_exact.py [s ...]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2501_09767_b200 import exact, ops  # noqa: E402


def bench(fn, it=5):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / it


H, d = 32, 128
for s in [int(a) for a in sys.argv[1:]] or [4096, 16384]:
    nq = (s + 127) // 128
    items = sum(q // 2 + 1 for q in range(nq))
    fl = items * H * 2 * 128 * 256 * d
    alg = s * s * H * d  # causal half of the 2·s²·h product
    qf = torch.randn(s, H * d, device="cuda") * 0.1
    kf = torch.randn(s, H * d, device="cuda") * 0.1
    q16, k16 = qf.bfloat16(), kf.bfloat16()
    qs, ks = ops.split_hilo(qf), ops.split_hilo(kf)
    t1 = bench(lambda: exact.exact_block_dense(q16, k16, 16, n_heads=H))
    t3 = bench(lambda: exact.exact_block_dense(qs, ks, 16, n_heads=H))
    print(f"s={s}: bf16 {t1:.3f} ms {fl / t1 / 1e9:.0f} TFLOP/s executed "
          f"({alg / t1 / 1e9:.0f} algorithmic) | bf16x3 {t3:.3f} ms "
          f"{3 * fl / t3 / 1e9:.0f} TFLOP/s executed", flush=True)
