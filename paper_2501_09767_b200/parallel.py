"""Data parallelism for the LeMo fine-tuning step.

The path shards by independent sequences: rank r trains sequence
`step·W + r`; predictors are frozen, so the ONLY exchange is the average of
the LoRA gradients — one flat fp32 bucket (`model.lora_param.grad`), one
NCCL all-reduce over NVLink — followed by an identical Adam step on every
rank.  Recalibration history stays rank-local (each rank behaves like a
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


class DataParallelStep:
    """forward_step + sparse backward + LoRA-gradient all-reduce + Adam, one
    sequence per rank.  `sequences` is indexable; rank r of W takes
    sequences[shard_index(step, r, W) % len(sequences)]."""

    def __init__(self, model, optimizer, pattern_source=None, *, segments: int = 8, group=None):
        self.model = model
        self.opt = optimizer
        self.source = pattern_source
        self.segments = segments
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.step_idx = 0

    def __call__(self, sequences):
        seq = sequences[shard_index(self.step_idx, self.rank, self.world) % len(sequences)]
        loss, _ = self.model.forward_step(seq, pattern_source=self.source,
                                          segments=self.segments)
        loss.backward()
        g = self.model.lora_param.grad
        if g is not None:
            allreduce_mean_(g, self.group)
        self.opt.step()
        self.opt.zero_grad()
        self.step_idx += 1
        return loss.detach()
