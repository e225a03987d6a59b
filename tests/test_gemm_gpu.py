"""tcgen05 GEMM + epilogues vs a plain PyTorch fp32 reference."""

import pytest
import torch

from paper_2501_09767_b200 import ops

pytestmark = pytest.mark.gpu


def _ref(a, b):
    return a.float() @ b.float().T


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 128), (300, 256, 4096),
                                   (1000, 768, 320), (16, 128, 64), (4096, 4096, 4096),
                                   (2048, 32000, 4096), (77, 96, 200)])
def test_gemm_bf16(cuda, M, N, K):
    g = torch.Generator(device=cuda).manual_seed(M * 7 + N)
    a = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    b = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    c = ops.gemm_bf16(a, b)
    torch.cuda.synchronize()
    ref = _ref(a, b)
    err = (c.float() - ref).abs().max().item()
    scale = ref.abs().max().item()
    assert err <= 1e-2 * scale + 1e-3, (err, scale)


@pytest.mark.parametrize("M,N,K,acc", [(256, 512, 256, True), (333, 250, 512, False),
                                       (128, 4096, 4096, True), (1024, 10, 3072, False),
                                       (2085, 2560, 320, True), (4099, 4096, 1088, False)])
def test_gemm_f32(cuda, M, N, K, acc):
    g = torch.Generator(device=cuda).manual_seed(3)
    a = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    b = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    out = torch.randn(M, N, device=cuda, generator=g)
    base = out.clone()
    ops.gemm_f32(a, b, out, accumulate=acc)
    torch.cuda.synchronize()
    ref = (base if acc else 0) + _ref(a, b)
    err = (out - ref).abs().max().item()
    assert err <= 1e-3 * ref.abs().max().item() + 1e-3


@pytest.mark.parametrize("s,h,K,k", [(1024, 512, 256, 400), (8192, 4096, 512, 4111)])
def test_gemm_scatter_add(cuda, s, h, K, k):
    """(the second case runs as 256 x 256 CTA-pair tiles)"""
    g = torch.Generator(device=cuda).manual_seed(5)
    idx = torch.randperm(s, device=cuda, generator=g)[:k].sort().values.int()
    a = torch.randn(k, K, device=cuda, generator=g).bfloat16()
    b = torch.randn(h, K, device=cuda, generator=g).bfloat16()
    resid = torch.randn(s, h, device=cuda, generator=g)
    ref = resid.clone()
    ref[idx.long()] += _ref(a, b)
    ops.gemm_scatter_add(a, b, resid, idx)
    torch.cuda.synchronize()
    assert torch.allclose(resid, ref, atol=1e-3, rtol=1e-3)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (300, 512, 4096), (1000, 768, 320)])
def test_gemm_nn_mn_major_b(cuda, M, N, K):
    """MN-major B operand descriptors (used by the attention kernels)."""
    from paper_2501_09767_b200._lib import call, ptr, stream_ptr
    g = torch.Generator(device=cuda).manual_seed(11)
    a = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    b = torch.randn(K, N, device=cuda, generator=g).bfloat16()
    c = torch.empty(M, N, device=cuda, dtype=torch.bfloat16)
    call("lemo_gemm_nn_bf16", ptr(a), K, ptr(b), N, ptr(c), N, M, N, K, stream_ptr())
    torch.cuda.synchronize()
    ref = a.float() @ b.float()
    err = (c.float() - ref).abs().max().item()
    assert err <= 1e-2 * ref.abs().max().item() + 1e-3, err


@pytest.mark.parametrize("M,N,K,acc", [(8208, 4096, 1024, False), (7045, 4096, 2048, True),
                                       (4096, 4096, 4096, False)])
def test_gemm_pair_split_k_tail(cuda, M, N, K, acc):
    """Shapes whose last wave of 256 x 256 pair tiles is at most half full run
    that wave as split-K units (partials summed in a fixed order): same result
    as the fp32 reference, and bit-identical run to run."""
    tiles = -(-M // 256) * (N // 256)
    assert tiles % 74 and 2 * (tiles % 74) <= 74  # the tail path is taken on 148 SMs
    g = torch.Generator(device=cuda).manual_seed(11)
    a = torch.randn(M, K, device=cuda, generator=g).bfloat16()
    b = torch.randn(N, K, device=cuda, generator=g).bfloat16()
    base = torch.randn(M, N, device=cuda, generator=g)
    outs = []
    for _ in range(2):
        out = base.clone()
        ops.gemm_f32(a, b, out, accumulate=acc)
        outs.append(out)
    torch.cuda.synchronize()
    ref = (base if acc else 0) + _ref(a, b)
    assert (outs[0] - ref).abs().max().item() <= 1e-3 * ref.abs().max().item() + 1e-3
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("K", [1024, 11008])
def test_gemm_scatter_add_split_k_tail(cuda, K):
    """The down-projection shape (k = 7045 retained rows -> 448 pair tiles =
    6 full waves + 4): the last wave runs as deferred split-K units whose
    partials a second kernel sums in a fixed order and scatter-adds
    (lemo_gemm_scatter_add) -- same result as the fp32 reference, rows outside
    idx untouched, bit-identical run to run."""
    s, h, k = 16384, 4096, 7045
    g = torch.Generator(device=cuda).manual_seed(12)
    idx = torch.randperm(s, device=cuda, generator=g)[:k].sort().values.int()
    a = torch.randn(k, K, device=cuda, generator=g).bfloat16()
    b = torch.randn(h, K, device=cuda, generator=g).bfloat16()
    resid0 = torch.randn(s, h, device=cuda, generator=g)
    ref = resid0.clone()
    ref[idx.long()] += _ref(a, b)
    outs = []
    for _ in range(2):
        resid = resid0.clone()
        ops.gemm_scatter_add(a, b, resid, idx)
        outs.append(resid)
    torch.cuda.synchronize()
    tol = 1e-3 * float(ref.abs().max())
    assert (outs[0] - ref).abs().max().item() <= tol
    assert torch.equal(outs[0], outs[1])
    untouched = torch.ones(s, dtype=torch.bool, device=cuda)
    untouched[idx.long()] = False
    assert torch.equal(outs[0][untouched], resid0[untouched])
