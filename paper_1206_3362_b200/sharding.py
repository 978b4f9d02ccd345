"""Frame sharding across ranks (one process per GPU) and the counter all-reduce.

Frames are independent (reference SPEC.md:169,431) and each frame's noise is
keyed by its GLOBAL index (channel.py:39-50), so a rank's result for a frame
does not depend on the world size.  The only exchange is the int64 counter
vector (frames, bit/word errors, iterations, flips, stalls, ...) per step.
"""

from __future__ import annotations

from typing import Tuple


def frame_shard(first: int, count: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [start, start + n) slice of [first, first + count) for `rank`.

    Slices are balanced to within one frame and tile the range in rank order."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("need 0 <= rank < world")
    if count < 0:
        raise ValueError("count must be nonnegative")
    base, extra = divmod(count, world)
    start = first + rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def reduce_counters(t, group=None):
    """Sum a counter tensor over all ranks in place (no-op when not distributed)."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t
