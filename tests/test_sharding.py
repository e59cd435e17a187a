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


CFG4_SMALL = dict(m=96, n=80, rank=6, noise=1e-4, relative=True, strategy="uniform", c=12, r=12, plan_seed=0,
                  gen_seed=20240301, batch=16)


def cfg4_row(b):
    """One matrix of bench.py's cfg4 recipe (reduced size) through the CPU oracle stand-in:
    (relative error, J, I)."""
    import sys
    import numpy as np

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path[:0] = [root, os.path.join(root, "oracle")]
    import bench
    import oracle as O

    cfg = CFG4_SMALL
    planes = bench.host_lowrank(cfg, cfg["gen_seed"] + 1000 * b)
    res = O.approx(planes, cfg["strategy"], cfg["rank"], cfg["plan_seed"] + b, cfg["c"], cfg["r"])
    return np.concatenate([[res["rel_err"]], res["cols"], res["rows"]])


def _split_worker(rank: int, world: int, port: int, q):
    import torch.distributed as dist

    from paper_2402_19147_b200.sharding import run_batch_split

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    table = run_batch_split(CFG4_SMALL["batch"], cfg4_row, 1 + CFG4_SMALL["c"] + CFG4_SMALL["r"])
    q.put((rank, table))
    dist.destroy_process_group()


def test_gloo_world2_cfg4_split_end_to_end():
    """The bench's cfg4 split end to end with CPU stand-ins: each of 2 gloo ranks approximates its
    half of the batch; both receive the full table, equal to a single-process run."""
    import numpy as np

    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    want = np.stack([cfg4_row(b) for b in range(CFG4_SMALL["batch"])])
    for _, table in out:
        assert np.array_equal(table, want)
