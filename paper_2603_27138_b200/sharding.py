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


def request_seed(seed: int, request: int, salt: int) -> int:
    """Seed of one request's synthetic data: a function of the GLOBAL request
    index, so every rank's shard is a slice of one seeded global workload
    (the same request gets the same data whatever the world size)."""
    return ((int(seed) * 1_000_003 + int(request)) * 1_009 + int(salt)) & 0x7FFF_FFFF_FFFF_FFFF


def gather_per_request(values: torch.Tensor, global_batch: int, world: int, rank: int) -> torch.Tensor:
    """Verification only (outside timing): this rank's per-request values
    [n_local, ...] into a [global_batch, ...] tensor on every rank (all_gather
    of request_shard slices, padded to the largest shard)."""
    import torch.distributed as dist

    start, n = request_shard(global_batch, world, rank)
    if values.shape[0] != n:
        raise ValueError("gather_per_request: expected this rank's shard of values")
    if not dist.is_available() or not dist.is_initialized() or world == 1:
        return values.clone()
    width = max(request_shard(global_batch, world, r)[1] for r in range(world))
    pad = torch.zeros((width,) + tuple(values.shape[1:]), dtype=values.dtype, device=values.device)
    pad[:n] = values
    got = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(got, pad)
    out = [got[r][:request_shard(global_batch, world, r)[1]] for r in range(world)]
    return torch.cat(out, dim=0)
