"""Multi-process (gloo, world_size 2) tests of the host-side sharding logic
used by bench.py for replicas (cfg1-cfg3) and the by-matrix batch split (cfg4)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2402_19147_b200.sharding import shard_range


def test_shard_range_partitions_exactly():
    for total in (1, 7, 64, 65):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                seen.extend(shard_range(total, world, r))
            assert seen == list(range(total))
    assert list(shard_range(64, 8, 3)) == list(range(24, 32))
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank: int, world: int, port: int, q):
    import torch.distributed as dist

    from paper_2402_19147_b200.sharding import gather_results, max_over_ranks, shard_range

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    owned = shard_range(64, world, rank)
    local = {b: float(b * b) for b in owned}          # stand-in per-matrix result
    allres = gather_results(local, 64)
    slowest = max_over_ranks(10.0 + rank)
    q.put((rank, list(owned), allres, slowest))
    dist.destroy_process_group()


def test_gloo_world2_batch_split_and_timing():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    out.sort()
    assert out[0][1] == list(range(32)) and out[1][1] == list(range(32, 64))
    for _, _, allres, slowest in out:
        assert allres == [float(b * b) for b in range(64)]
        assert slowest == 11.0
