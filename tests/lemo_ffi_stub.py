"""The binding a `sparsetune` maintainer adds, verbatim in
spirit: plain ctypes on liblemo.so, torch only for device buffers and the
stream.  It does NOT import this repository's Python package -- it is what
the reference would ship as `sparsetune/lemo_ffi.py`.

Two reference ops are routed through the C ABI:
  eliminate(block_scores, threshold, *, layer_id, component, block_size,
            n_tokens, force_blocks)                      (sparsity.py:263-281)
      -> lemo_select on the device, returns the reference's SparsityPattern
  segmented_loss_and_grad(hidden, lm_head, targets, plan, ignore_index=-1)
                                                          (kernels.py:229-288)
      -> lemo_gemm_f32 (logits) + lemo_ce_rows + lemo_gemm_f32 (grad_hidden)
         + lemo_sum_f64, registered on the reference's tape with
         tensor.custom_op (tensor.py:177-179) exactly as the reference does
"""

from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np
import torch

P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
_SIGS = {
    "lemo_select": [P, I, D, P, P, I, I, P, P, P, P, P, P],
    "lemo_gemm_f32": [P, I, P, I, P, I, I, I, I, I, P],
    "lemo_ce_rows": [P, I, P, I, I, I, ctypes.c_float, P, I, P, P, P],
    "lemo_sum_f64": [P, I, P, I, P],
}


def load(path: Path):
    lib = ctypes.CDLL(str(path))
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    lib.lemo_last_error.restype = ctypes.c_char_p
    return lib


class LemoOps:
    def __init__(self, lib_path: Path, sparsity_mod, tensor_mod):
        self.lib = load(lib_path)
        self.S = sparsity_mod
        self.T = tensor_mod
        self.dev = torch.device("cuda")

    def _ok(self, rc):
        if rc:
            raise RuntimeError(self.lib.lemo_last_error().decode())

    def _stream(self):
        return torch.cuda.current_stream().cuda_stream

    # sparsity.eliminate ---------------------------------------------------------
    def eliminate(self, block_scores, threshold, *, layer_id=0, component="attention",
                  block_size, n_tokens, force_blocks=()):
        v = torch.as_tensor(np.asarray(block_scores, dtype=np.float64)).to(self.dev)
        nb = v.numel()
        force = None
        if len(force_blocks):
            f = torch.zeros(nb, dtype=torch.uint8)
            f[list(force_blocks)] = 1
            force = f.to(self.dev)
        mask = torch.empty(max(nb, 1), dtype=torch.uint8, device=self.dev)
        blocks = torch.empty(max(nb, 1), dtype=torch.int32, device=self.dev)
        tokens = torch.empty(max(nb * block_size, 1), dtype=torch.int32, device=self.dev)
        counts = torch.zeros(4, dtype=torch.int32, device=self.dev)
        self._ok(self.lib.lemo_select(v.data_ptr(), nb, float(threshold), None,
                                      None if force is None else force.data_ptr(), block_size,
                                      n_tokens, mask.data_ptr(), blocks.data_ptr(),
                                      tokens.data_ptr(), counts.data_ptr(), None, self._stream()))
        k, nkept, bad = counts.cpu().tolist()[:3]
        if bad:
            raise self.S.ContractError("block scores must be finite")
        kept = tuple(blocks[:nkept].cpu().tolist())
        return self.S.SparsityPattern(layer_id, component, kept, block_size, n_tokens)

    # kernels.segmented_loss_and_grad ----------------------------------------------
    def segmented_loss_and_grad(self, hidden, lm_head, targets, plan, ignore_index=-1):
        T = self.T
        targets = np.asarray(targets)
        n, h = hidden.shape
        V = lm_head.shape[1]
        valid = targets != ignore_index
        if valid.any() and (targets[valid].min() < 0 or targets[valid].max() >= V):
            raise IndexError("target index out of range")
        count = int(valid.sum())
        dev, st = self.dev, self._stream()
        hid = torch.as_tensor(hidden.data).to(dev).to(torch.bfloat16).contiguous()
        w = torch.as_tensor(lm_head.data).to(dev)
        w_t = w.t().contiguous().to(torch.bfloat16)   # [V, h]
        w_b = w.to(torch.bfloat16).contiguous()       # [h, V]
        tg = torch.as_tensor(targets.astype(np.int32)).to(dev)
        gh = torch.empty(n, h, dtype=torch.float32, device=dev)
        row_loss = torch.empty(n, dtype=torch.float32, device=dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        for a, b in plan.segments:
            logits = torch.empty(b - a, V, dtype=torch.float32, device=dev)
            self._ok(self.lib.lemo_gemm_f32(hid[a:b].data_ptr(), h, w_t.data_ptr(), h,
                                            logits.data_ptr(), V, b - a, V, h, 0, st))
            dlog = torch.empty(b - a, V, dtype=torch.bfloat16, device=dev)
            self._ok(self.lib.lemo_ce_rows(logits.data_ptr(), V, tg[a:b].data_ptr(), b - a, V,
                                           ignore_index, 1.0 / max(count, 1), dlog.data_ptr(), V,
                                           row_loss[a:b].data_ptr(), bad.data_ptr(), st))
            self._ok(self.lib.lemo_gemm_f32(dlog.data_ptr(), V, w_b.data_ptr(), V,
                                            gh[a:b].data_ptr(), h, b - a, h, V, 0, st))
        total = torch.empty(1, dtype=torch.float64, device=dev)
        self._ok(self.lib.lemo_sum_f64(row_loss.data_ptr(), n, total.data_ptr(), 0, st))
        if count == 0:
            raise self.S.ContractError("segmented loss: no valid targets")
        loss = float(total.item()) / count
        grad_hidden = gh.cpu().numpy().astype(hidden.data.dtype)

        def bw(g):
            return (g * grad_hidden, None)

        return T.custom_op(np.asarray(loss, dtype=hidden.data.dtype),
                           "segmented_cross_entropy", (hidden, lm_head), (grad_hidden,), bw)
