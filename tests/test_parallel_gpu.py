"""Data parallelism on the GPU path (SURVEY.md §8e equality check): W=2 ranks
(one process each, both on cuda:0, gloo for the exchange since one box has
one GPU here) each train their own sequence, average the LoRA gradients and
step Adam; the result equals a single process averaging the two sequences'
gradients, and both ranks hold bitwise-identical adapters."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

CFG = dict(n_layers=2, hidden_dim=256, n_heads=2, vocab_size=256, max_seq_len=512, mlp_dim=688,
           block_size=16, lora_rank=8, lora_alpha=16.0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _seqs():
    rng = np.random.default_rng(42)
    return [rng.integers(0, 256, 300) for _ in range(2)]


def _model():
    from paper_2501_09767_b200 import model as M
    m = M.DecoderModel(M.ModelConfig(**CFG), 7, device="cuda:0", init="reference")
    with torch.no_grad():  # nonzero B so every adapter has a gradient
        g = torch.Generator(device="cuda:0").manual_seed(3)
        m.lora_param.add_(0.05 * torch.randn(m.lora_param.shape, generator=g, device="cuda:0"))
    return m


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2501_09767_b200 import model as M, parallel
        from paper_2501_09767_b200.optim import Adam
        model = _model()
        opt = Adam(model.lora_param, lr=1e-2)
        step = parallel.DataParallelStep(model, opt, M.FractionSource(0.5, 16), segments=2)
        step(_seqs())
        out[rank] = model.lora_param.detach().cpu().numpy()
    finally:
        dist.destroy_process_group()


def test_two_ranks_equal_single_process_average(cuda):
    from paper_2501_09767_b200 import model as M
    from paper_2501_09767_b200.optim import Adam
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.get_context("spawn")
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert np.array_equal(out[0], out[1])  # identical update on every rank
    # single process: average of the two sequences' gradients, one Adam step
    model = _model()
    grads = []
    for seq in _seqs():
        loss, _ = model.forward_step(seq, pattern_source=M.FractionSource(0.5, 16), segments=2)
        loss.backward()
        grads.append(model.lora_param.grad.clone())
        model.lora_param.grad = None
    model.lora_param.grad = (grads[0] + grads[1]) / 2
    opt = Adam(model.lora_param, lr=1e-2)
    opt.step()
    ref = model.lora_param.detach().cpu().numpy()
    assert np.abs(out[0] - ref).max() <= 1e-6 * max(np.abs(ref).max(), 1.0)
