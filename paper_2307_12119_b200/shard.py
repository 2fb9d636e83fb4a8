"""Sample sharding over ranks (configs 1-3 shard by independent
pairs / traces, no collective on the data path).

Each rank owns a contiguous range of global sample indices; inputs are a pure
function of the global index (inputs.sample_seed), so a sample's result does
not depend on the world size. Collectives are used only for bookkeeping:
the max-over-ranks step time and an optional gather of per-sample scalars.
"""
from __future__ import annotations


def shard_range(rank: int, world: int, per_rank: int, weak: bool = True, total: int | None = None) -> tuple[int, int]:
    """Global [start, stop) of `rank`. weak: every rank gets `per_rank` samples;
    strong: `total` samples split as evenly as possible."""
    if weak:
        return rank * per_rank, (rank + 1) * per_rank
    assert total is not None
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def max_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_scalars(values, device=None):
    """All-gather a per-rank 1-D float64 array of equal length -> concatenated in rank order."""
    import torch
    import torch.distributed as dist
    t = torch.as_tensor(values, dtype=torch.float64, device=device).contiguous()
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t.cpu().numpy()
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return torch.cat(parts).cpu().numpy()
