"""Host-side (Python) cost of one training step: cProfile, top functions by own time."""
import cProfile, pstats, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from profile_step import setup  # noqa: E402
from paper_2501_09767_b200.optim import Adam  # noqa: E402
model, src, tokens = setup(16384, "lemo", "refined")
opt = Adam(model.lora_param, lr=1e-4)
batch = model.stage_tokens(tokens)
def step():
    loss, _ = model.forward_step(batch, pattern_source=src, segments=8)
    loss.backward(); opt.step(); opt.zero_grad()
for _ in range(2): step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable(); step(); torch.cuda.synchronize(); pr.disable()
st = pstats.Stats(pr); st.sort_stats("tottime").print_stats(25)
