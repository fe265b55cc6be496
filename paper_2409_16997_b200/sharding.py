"""(b,h)-slice sharding across GPUs.

Every (b,h) slice is an independent attention problem (the reference's
harness loops them, eval.cpp:167-168; V's tensor scale is per slice,
eval.cpp:101), so the multi-GPU layout is a contiguous split of the flat
slice index with no collective on the data path.  NCCL is used only to
gather per-rank results for verification and to sum per-rank MRE partials.
"""
from __future__ import annotations

from typing import List, Tuple


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [lo, hi) slice range of `rank`: sizes differ by at most 1,
    larger shards first (slice g -> rank owning it is deterministic)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world {world}")
    if total < 0:
        raise ValueError("negative slice count")
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def owner_of(slice_index: int, total: int, world: int) -> int:
    """Rank that owns flat slice `slice_index` under shard_range."""
    for r in range(world):
        lo, hi = shard_range(total, world, r)
        if lo <= slice_index < hi:
            return r
    raise ValueError("slice index out of range")


def gather_slices(local, total: int, world: int, rank: int, group=None) -> List:
    """All-gather per-rank tensors of shape [hi-lo, ...] into a list ordered by
    slice (verification only).  Pads to the largest shard for the collective."""
    import torch
    import torch.distributed as dist

    sizes = [shard_range(total, world, r) for r in range(world)]
    maxn = max(hi - lo for lo, hi in sizes)
    pad = torch.zeros((maxn,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return [bufs[r][: hi - lo] for r, (lo, hi) in enumerate(sizes)]


def allreduce_error(acc, group=None):
    """Sum every rank's ErrorAccum (num, den) into a whole-job accumulator
    (f64 all-reduce): the normalized L1 error composes
    exactly as eval.cpp:55-75 accumulates it across slices."""
    import torch
    import torch.distributed as dist
    from .evaluation import ErrorAccum

    t = torch.tensor([acc.num, acc.den], dtype=torch.float64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    out = ErrorAccum()
    out.num, out.den = float(t[0]), float(t[1])
    return out
