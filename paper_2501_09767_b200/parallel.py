"""Data parallelism for the LeMo fine-tuning step.

The path shards by independent sequences: rank r trains sequence
`step·W + r`; predictors are frozen, so the ONLY exchange is the average of
the LoRA gradients — fp32, bucketed per layer and all-reduced (NCCL over
NVLink) while the backward sweep is still working on the layers below
(`BucketedGradReducer`), then an identical Adam step on every rank.
Recalibration history stays rank-local (each rank behaves like a
single-process reference on its own stream of sequences).
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_index(step: int, rank: int, world: int) -> int:
    """Sequence index of `rank` at `step` (pipeline.py:470 with W ranks)."""
    return step * world + rank


def allreduce_mean_(grad: torch.Tensor, group=None) -> torch.Tensor:
    """In-place mean over ranks of one flat gradient bucket.  NCCL uses its
    native AVG; other backends (gloo, used by the CPU tests) SUM then scale."""
    if not dist.is_available() or not dist.is_initialized():
        return grad
    world = dist.get_world_size(group)
    if world == 1:
        return grad
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(grad, op=dist.ReduceOp.AVG, group=group)
    else:
        dist.all_reduce(grad, op=dist.ReduceOp.SUM, group=group)
        grad.div_(world)
    return grad


class BucketedGradReducer:
    """Per-layer LoRA-gradient buckets all-reduced asynchronously as the
    backward sweep finishes each layer (DecoderModel.grad_reducer): the
    collective of layer l runs on NCCL's stream while the sweep computes layer
    l-1.  finish() makes the compute stream wait for every bucket (no host
    block) and applies the 1/W of non-NCCL backends."""

    def __init__(self, group=None):
        self.group = group
        self.pending = []

    def _active(self) -> bool:
        return dist.is_available() and dist.is_initialized() and \
            dist.get_world_size(self.group) > 1

    def layer_ready(self, layer_id: int, grad_slice: torch.Tensor) -> None:
        if not self._active():
            return
        nccl = dist.get_backend(self.group) == "nccl"
        op = dist.ReduceOp.AVG if nccl else dist.ReduceOp.SUM
        work = dist.all_reduce(grad_slice, op=op, group=self.group, async_op=True)
        self.pending.append((work, grad_slice, nccl))

    def finish(self) -> None:
        world = dist.get_world_size(self.group) if self._active() else 1
        for work, sl, nccl in self.pending:
            work.wait()
            if not nccl:
                sl.div_(world)
        self.pending = []


class DataParallelStep:
    """forward_step + sparse backward + LoRA-gradient all-reduce + Adam, one
    sequence per rank.  `sequences` is indexable; rank r of W takes
    sequences[shard_index(step, r, W) % len(sequences)]."""

    def __init__(self, model, optimizer, pattern_source=None, *, segments: int = 8, group=None,
                 overlap: bool = True):
        self.model = model
        self.opt = optimizer
        self.source = pattern_source
        self.segments = segments
        self.group = group
        self.overlap = overlap
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.step_idx = 0

    def __call__(self, sequences):
        seq = sequences[shard_index(self.step_idx, self.rank, self.world) % len(sequences)]
        loss, _ = self.model.forward_step(seq, pattern_source=self.source,
                                          segments=self.segments)
        if self.overlap:  # buckets reduced inside the backward sweep
            self.model.grad_reducer = BucketedGradReducer(self.group)
        try:
            loss.backward()
        finally:
            self.model.grad_reducer = None
        g = self.model.lora_param.grad
        if g is not None and not self.overlap:
            allreduce_mean_(g, self.group)
        self.opt.step()
        self.opt.zero_grad()
        self.step_idx += 1
        return loss.detach()
