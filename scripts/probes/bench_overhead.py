"""Does the bench's measurement apparatus perturb the timed step?  One setup
(the bench's N* workload, refined scorers), then 5-step timings with and
without per-call CUDA-event instrumentation and the nvidia-smi sampler."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_2501_09767_b200 import _lib  # noqa: E402
from paper_2501_09767_b200.optim import Adam  # noqa: E402
from profile_step import setup  # noqa: E402

model, src, tokens = setup(16384, "lemo", "refined")
opt = Adam(model.lora_param, lr=1e-4)
staged = model.stage_tokens(tokens)


def step():
    loss, _ = model.forward_step(staged, pattern_source=src, segments=8)
    loss.backward()
    opt.step()
    opt.zero_grad()


def timed(inst, smi, steps=5):
    ins = _lib.INSTRUMENT
    torch.cuda.synchronize()
    ck = bench.Clocks(0) if smi else None
    if ck:
        ck.start()
    ins.reset(("lemo_gemm_gateup", "lemo_block_embed", "lemo_flash_fwd_tc", "lemo_flash_bwd_tc")
              if inst else ())
    ins.enabled = inst
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(steps):
        step()
    b.record()
    torch.cuda.synchronize()
    ins.enabled = False
    c = ck.stop() if ck else None
    return a.elapsed_time(b) / steps, c


for _ in range(3):
    step()
for rep in range(2):
    for inst, smi in ((False, False), (True, False), (False, True), (True, True)):
        ms, c = timed(inst, smi)
        print(f"inst={inst} smi={smi}: {ms:.1f} ms/step  {16384 / ms * 1e3:.0f} tok/s  "
              f"{c and (c['sm_mhz'], c['reasons'])}", flush=True)
