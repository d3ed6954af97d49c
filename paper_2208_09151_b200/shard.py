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

from typing import List, NamedTuple, Optional, Sequence


def assign_superbatches(num_superbatches: int, rank: int, world: int, steps: int,
                        start: int = 0) -> List[int]:
    """Superbatch indices rank `rank` runs for `steps` consecutive steps."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if num_superbatches < 1:
        raise ValueError("empty plan")
    return [(rank + (start + k) * world) % num_superbatches for k in range(steps)]


class Job(NamedTuple):
    """One (epoch, superbatch) job of TrainingRunner::run (pipeline.hpp:206-228)."""
    epoch: int
    seq: int                 # position in the flattened job list
    first_global_batch: int  # batches of all earlier jobs, short final superbatches included
    lo: int                  # batch range [lo, hi) of the epoch's seed plan
    hi: int


def superbatch_jobs(batches_per_epoch: Sequence[int], superbatch_size: int) -> List[Job]:
    """The flattened job list of TrainingRunner::run (pipeline.hpp:212-228):
    every epoch's plan is cut into superbatches of `superbatch_size` batches
    (the last one may be short) and first_global_batch counts the batches of
    all earlier jobs, so batch seeds stay the reference's across epochs."""
    if superbatch_size < 1:
        raise ValueError("superbatch_size must be >= 1")
    jobs: List[Job] = []
    g = 0
    for e, nb in enumerate(batches_per_epoch):
        for off in range(0, nb, superbatch_size):
            end = min(off + superbatch_size, nb)
            jobs.append(Job(e, len(jobs), g, off, end))
            g += end - off
    return jobs


def first_global_batch(sb_index: int, superbatch_size: int,
                       batches_per_epoch: Optional[Sequence[int]] = None) -> int:
    """Global index of the first batch of job `sb_index` (pipeline.hpp:214-228).
    Without `batches_per_epoch` the job is taken from epoch 0 (sb_index * S);
    with it, from the flattened multi-epoch job list (short final superbatches
    of earlier epochs counted as the reference counts them)."""
    if batches_per_epoch is None:
        return sb_index * superbatch_size
    return superbatch_jobs(batches_per_epoch, superbatch_size)[sb_index].first_global_batch


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


def batch_block(num_batches: int, rank: int, world: int) -> range:
    """Contiguous block of a superbatch's batches that rank `rank` samples when
    the superbatch's batches are split by rank (north_star / SURVEY §8e):
    [S*r/P, S*(r+1)/P). Batch i of the block keeps its global index
    first_global_batch + i, so its RNG stream is the single-GPU one
    (sampler.hpp:216)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return range(num_batches * rank // world, num_batches * (rank + 1) // world)


def partition_graph(graph, rank: int, world: int, group=None):
    """Row-partition a GraphFile over the ranks of `group` (collective): every
    rank keeps its edge-balanced share of the in-neighbour lists, exports the
    CUDA IPC handle of that share, and maps every peer's share, so the sampler
    reads remote lists straight from the owner's HBM over NVLink
    (gx_graph_partition / gx_graph_attach_peers, include/gx_b200.h). Handles
    travel through torch.distributed (all_gather_object)."""
    import torch.distributed as dist
    graph.partition(world, rank)
    if world == 1:
        return graph
    mine = graph.ipc_handle()
    handles = [None] * world
    dist.all_gather_object(handles, mine, group=group)
    graph.attach_peers(handles)
    return graph
