"""Multi-GPU layout: batch x head (attention) / token-row (FFN) sharding.

The EFTA path has no data exchange between units (heads are independent,
SPEC.md:352/473 in the reference; src/campaign.cpp:175 loops them), so ranks
own contiguous ranges of the flattened (b, h) index and run the fused kernel on
their range with no collective. The only collectives are control-plane: a
barrier around timed regions and a max-reduce of per-rank device times.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    start: int   # first flat unit (b*H + h, or token row) owned by this rank
    count: int   # units owned

    @property
    def stop(self) -> int:
        return self.start + self.count


def shard_units(n_units: int, world: int, rank: int) -> Shard:
    """Contiguous, balanced split of n_units over world ranks (sizes differ by <= 1)."""
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("shard_units: bad rank/world")
    base, extra = divmod(n_units, world)
    start = rank * base + min(rank, extra)
    return Shard(rank, world, start, base + (1 if rank < extra else 0))


def shard_tokens(n_tokens: int, world: int, rank: int, align: int = 128) -> Shard:
    """Token-row split of an FFN activation [n_tokens, d] for the strided-ABFT GEMM: contiguous
    blocks of `align` rows (the GEMM's 128-row tile), balanced to within one block. Weights and
    their checksum rows are replicated, so every rank verifies its own rows (no exchange)."""
    if n_tokens % align:
        raise ValueError("shard_tokens: n_tokens must be a multiple of align")
    blk = shard_units(n_tokens // align, world, rank)
    return Shard(rank, world, blk.start * align, blk.count * align)


def gather_units(local, dist=None):
    """Concatenate per-rank lists of unit results in rank order (host-side, small objects:
    outputs of sampled units, event logs). The data path itself never exchanges anything."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return list(local)
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, list(local))
    return [x for part in parts for x in part]


def route_faults(specs, shard: Shard):
    """Keep the fault specs whose flat head lies in this shard, re-indexed locally."""
    out = []
    for f in specs:
        if shard.start <= f.head < shard.stop:
            g = type(f)(**{**f.__dict__, "head": f.head - shard.start})
            out.append(g)
    return out


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the max over ranks)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
