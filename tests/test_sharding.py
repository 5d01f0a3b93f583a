"""Multi-process (gloo, world_size 2, CPU) coverage of the N>1 host path:
request sharding, max-over-ranks timing, checksum gather."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2603_27138_b200.sharding import gather_checksums, max_over_ranks, request_shard, unit_range


@pytest.mark.parametrize("gb,world", [(128, 2), (128, 8), (7, 3), (1, 4), (0, 2)])
def test_request_shard_partitions(gb, world):
    seen = []
    for r in range(world):
        s, n = request_shard(gb, world, r)
        seen += list(range(s, s + n))
    assert seen == list(range(gb))
    counts = [request_shard(gb, world, r)[1] for r in range(world)]
    assert max(counts) - min(counts) <= 1


def test_unit_range_and_errors():
    assert unit_range(128, 8, 4, 1) == (32 * 8, 32 * 8)
    with pytest.raises(ValueError):
        request_shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, n = request_shard(128, world, rank)
        t = max_over_ranks(10.0 + rank)               # the slowest rank sets the step time
        out = torch.full((n, 4), float(rank + 1))      # this rank's attention outputs
        sums = gather_checksums(out)
        q.put((rank, s, n, t, sums))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [(r[1], r[2]) for r in res] == [(0, 64), (64, 64)]
    assert all(r[3] == 11.0 for r in res)
    assert all(r[4] == [64 * 4 * 1.0, 64 * 4 * 2.0] for r in res)


def test_request_seed_depends_on_global_request_only():
    from paper_2603_27138_b200.sharding import request_seed

    # the same request gets the same seed whatever shard it lands in; distinct
    # requests and salts differ
    seeds = {request_seed(1234, r, s) for r in range(64) for s in range(4)}
    assert len(seeds) == 256
    assert request_seed(1234, 7, 1) == request_seed(1234, 7, 1)
    assert all(0 <= x < 2**63 for x in seeds)


def _gather_worker(rank, world, port, q):
    from paper_2603_27138_b200.sharding import gather_per_request

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gb = 7  # uneven shards: 4 + 3
        s, n = request_shard(gb, world, rank)
        vals = torch.arange(s, s + n, dtype=torch.float64) * 10.0  # "per-request output sums" of this shard
        got = gather_per_request(vals, gb, world, rank)
        q.put((rank, got.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_gather_per_request_slices_one_global_workload():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, got in res:  # every rank sees the global vector, in global request order
        assert got == [10.0 * r for r in range(7)]


def test_gather_per_request_single_rank_and_shape_check():
    from paper_2603_27138_b200.sharding import gather_per_request

    v = torch.arange(5.0)
    assert torch.equal(gather_per_request(v, 5, 1, 0), v)
    with pytest.raises(ValueError):
        gather_per_request(torch.arange(3.0), 5, 1, 0)
