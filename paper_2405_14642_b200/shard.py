"""Instance sharding across GPUs (host logic; no data-path collective).

Instances are independent (``bbadd`` is a map), so the
batch is partitioned by contiguous global instance ranges.  Two schemes:

* weak scaling (bench.py default): every rank owns ``per_rank`` instances,
  rank r -> [r * per_rank, (r + 1) * per_rank);
* strong scaling: a global batch of ``n`` instances, rank r ->
  [floor(r n / W), floor((r + 1) n / W)) — sizes differ by at most one.

Inputs are generated from *global* instance indices
(``inputs.make_operands(..., inst0=start)``), so every shard is bit-identical
to the corresponding rows of a single-GPU run.  The only collectives used by
the benchmark are the timing barrier and the max-over-ranks reduction
(``max_over_ranks``), which are plumbing, not the hot path.
"""
from __future__ import annotations


def weak_range(rank: int, world: int, per_rank: int):
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return rank * per_rank, (rank + 1) * per_rank


def strong_range(rank: int, world: int, n: int):
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return (rank * n) // world, ((rank + 1) * n) // world


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (e.g. a kernel time) over all ranks."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def plan(rank: int, world: int, n: int, scaling: str):
    """This rank's global instance range [lo, hi) and the job's total.

    weak:   n instances per rank (the paper batch per GPU), total = n * world;
    strong: a global batch of n instances split floor(r n / W), total = n."""
    if scaling == "weak":
        lo, hi = weak_range(rank, world, n)
        return lo, hi, n * world
    if scaling == "strong":
        lo, hi = strong_range(rank, world, n)
        return lo, hi, n
    raise ValueError("scaling must be 'weak' or 'strong'")


def checksum(t) -> int:
    """Wrapping 64-bit sum of a limb tensor's bytes read as int64 words (any
    device).  Additive over row ranges, so the sum of the per-rank checksums
    (mod 2^64) equals the single-GPU checksum of the same global rows."""
    import torch
    flat = t.contiguous().view(-1)
    if flat.dtype != torch.int64:
        flat = flat.view(torch.int32)
        if flat.numel() % 2:
            flat = torch.cat([flat, flat.new_zeros(1)])
        flat = flat.view(torch.int64)
    return int(flat.sum().item()) & ((1 << 64) - 1)


def combine_checksums(parts) -> int:
    """Global checksum from per-rank ones (mod 2^64)."""
    return sum(int(p) for p in parts) & ((1 << 64) - 1)


def gather_objects(obj, dist=None):
    """All ranks' `obj` in rank order (a list of one at world size 1)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return [obj]
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, obj)
    return out
