"""Request sharding across GPUs: decode shards by request with
no collective on the data path. Each rank owns its requests' KV pool, digests,
tables and recall stream; collectives appear only around the timed region
(max-over-ranks timing) and for verification (checksum gather)."""
from __future__ import annotations

import torch


def request_shard(global_batch: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous split of global_batch requests: (first request, count) of rank."""
    if world <= 0 or not 0 <= rank < world or global_batch < 0:
        raise ValueError("request_shard: bad world / rank / batch")
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def unit_range(global_batch: int, hkv: int, world: int, rank: int) -> tuple[int, int]:
    """(first unit, count) where unit = request * hkv + kv_head."""
    s, n = request_shard(global_batch, world, rank)
    return s * hkv, n * hkv


def max_over_ranks(x: float, device=None) -> float:
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_checksums(out: torch.Tensor) -> list[float]:
    """Verification only (outside timing): every rank's output checksum."""
    import torch.distributed as dist

    c = out.double().sum().reshape(1)
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return [float(c.item())]
    got = [torch.zeros_like(c) for _ in range(dist.get_world_size())]
    dist.all_gather(got, c)
    return [float(g.item()) for g in got]
