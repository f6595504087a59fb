"""Multi-GPU plumbing for independent frame streams.

The path shards by frame stream: a stream's stereo and local-map search only
touch that stream's frame and map (reference tracker.py:1-7, one tracker per
stream), so there is no exchange step and no collective on the data path.
Stream s runs on rank s mod world; torch.distributed (NCCL on the GPU box,
gloo in the CPU tests) carries only the start barrier and the max-over-ranks
timing reduction.
"""

from __future__ import annotations


def streams_of_rank(n_streams: int, world: int, rank: int) -> list[int]:
    """Global stream ids owned by `rank` (round robin: s mod world == rank)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    return list(range(rank, n_streams, world))


def rank_of_stream(s: int, world: int) -> int:
    return s % world


def max_over_ranks(values, dist=None, device=None):
    """Element-wise max of a list of floats across ranks (the timing rule:
    the job takes as long as its slowest rank)."""
    import torch
    vals = [float(v) for v in values]
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return vals
    if dist.get_backend() == "gloo":
        device = None  # gloo reduces host tensors
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


def job_frames_per_s(frames_per_rank: int, world: int, max_ms: float) -> float:
    """Whole-job throughput: every rank's frames over the slowest rank's time."""
    return frames_per_rank * world / (max_ms / 1e3)
