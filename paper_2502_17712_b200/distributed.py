"""Multi-GPU throughput for independent views.

A single frame does not shard: union-find is global over the visible mesh
(charts.py:362-386) and the scale search is global over all charts
(packing.py:295-345).  Throughput therefore scales over independent views:
each rank (one process per GPU) keeps a mesh replica and renders a contiguous
block of views.  There is no collective on the data path.  torch.distributed
is used only for the barrier around the timed region and for the max-over-
ranks reduction of the per-rank device time.
"""

from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def view_shard(n_views: int, rank: int, world_size: int) -> range:
    """Contiguous block of views for `rank` (sizes differ by at most one)."""
    if world_size < 1 or not (0 <= rank < world_size):
        raise ValueError("bad rank / world size")
    base, extra = divmod(int(n_views), world_size)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def step_views(steps: int, rank: int, n_pool: int = 64) -> list:
    """Weak scaling: every rank renders `steps` views, rank r taking pool
    indices r*steps .. r*steps+steps-1 (mod the pool size)."""
    return [(rank * steps + s) % n_pool for s in range(steps)]


def max_over_ranks(values, device=None):
    """Element-wise MAX all-reduce of a list of floats (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.cpu()]


def sum_over_ranks(values, device=None):
    """Element-wise SUM all-reduce of a list of floats (identity when not distributed)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(v) for v in values], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.cpu()]


def barrier(device=None):
    import torch
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()
    if device is not None and torch.cuda.is_available():
        torch.cuda.synchronize(device)


def run_views(engine_factory, views, render_view):
    """Render `views` with one engine (one GPU); returns the per-view results.
    `render_view(engine, view)` performs one frame."""
    eng = engine_factory()
    return [render_view(eng, v) for v in views]
