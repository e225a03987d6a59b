import numpy as np, torch, math, sys
sys.path.insert(0, '.')
from oracle import lemo_oracle as O
from paper_2501_09767_b200 import ops
from paper_2501_09767_b200.model import DecoderModel, ModelConfig
cuda = torch.device('cuda')
rng = np.random.default_rng(0)
h, H, r, M = 256, 4, 8, 96
d = h // H
cfg = ModelConfig(n_layers=1, hidden_dim=h, n_heads=H, vocab_size=64, mlp_dim=256, lora_rank=r)
model = DecoderModel(cfg, 0)
L = model.layers[0]
L.lora_q.b.copy_(torch.randn(r, h, device=cuda) * 0.1)
L.lora_v.b.copy_(torch.randn(r, h, device=cuda) * 0.1)
xn = torch.as_tensor(rng.standard_normal((M, h)).astype(np.float32)).cuda().bfloat16()
pos_np = np.sort(rng.choice(1000, M, replace=False))
pos = torch.as_tensor(pos_np.astype(np.int32)).cuda()
t = (xn.float() @ L.lora_A).contiguous()
for rope in (False, True):
  for use_lora in (False, True):
    q, k, v = ops.gemm_qkv(xn, L.w_qkv_t, h=h, head_dim=d, rope=rope, rope_tab=L.rope_tab, pos=pos,
                           t=t if use_lora else None, r=r if use_lora else 0, Bq=L.lora_Bq, Bv=L.lora_Bv, scale=L.lora_scaling)
    torch.cuda.synchronize()
    xf = xn.float().cpu().numpy(); W = L.w_qkv.float().cpu().numpy(); s = L.lora_scaling
    qr = xf @ W[:, :h]; kr = xf @ W[:, h:2*h]; vr = xf @ W[:, 2*h:]
    if use_lora:
        qr = qr + (t[:, :r].cpu().numpy() @ L.lora_Bq.cpu().numpy()) * s
        vr = vr + (t[:, r:].cpu().numpy() @ L.lora_Bv.cpu().numpy()) * s
    if rope:
        qr = O.rope_fwd(qr.astype(np.float32), pos_np, H, 10000.0); kr = O.rope_fwd(kr.astype(np.float32), pos_np, H, 10000.0)
    for nm, got, ref in (('q', q, qr), ('k', k, kr), ('v', v, vr)):
        g = got.float().cpu().numpy()
        err = np.abs(g - ref)
        print(f"rope={rope} lora={use_lora} {nm}: maxerr {err.max():.4f} at {np.unravel_index(err.argmax(), err.shape)} refmax {np.abs(ref).max():.3f}")
