"""Multi-GPU layout of the hot path: one process per GPU.

The sampler, inspector and executor shard by *superbatch*: every batch's RNG
stream depends only on its global batch index (sampler.hpp:216), so rank r can
run superbatches r, r+P, r+2P, ... of the epoch plan independently and its
outputs are bit-identical to the single-GPU run of the same superbatches. No
data-path collective is needed (weak scaling); the only communication is the
timing/statistics reduction, done here with torch.distributed (NCCL on the GPU
box, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List, Sequence


def assign_superbatches(num_superbatches: int, rank: int, world: int, steps: int,
                        start: int = 0) -> List[int]:
    """Superbatch indices rank `rank` runs for `steps` consecutive steps."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if num_superbatches < 1:
        raise ValueError("empty plan")
    return [(rank + (start + k) * world) % num_superbatches for k in range(steps)]


def first_global_batch(sb_index: int, superbatch_size: int) -> int:
    """Global index of the first batch of a superbatch (TrainingRunner::run, pipeline.hpp:214-228)."""
    return sb_index * superbatch_size


def reduce_stats(values: Sequence[float], ops: Sequence[str], device=None) -> List[float]:
    """All-reduce a small vector of floats with per-entry op in {"max", "sum"}."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(values)
    out = []
    for v, op in zip(values, ops):
        t = torch.tensor([float(v)], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        out.append(float(t.item()))
    return out
