"""Row-block sharded QMCUR (cfg5 design): the orchestration in
paper_2402_19147_b200/rowshard.py run with numpy ops on CPU — single process
and gloo world_size 2 — against the single-process oracle on the full matrix.
Bars as everywhere: indices, C rows and R bit-exact; U within 1e-9; error
within 1e-10 (the Gram all-reduce changes only the summation order)."""
import math
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle as O
from paper_2402_19147_b200.rowshard import SingleComm, approx_rowsharded, combine_subtrees, subtree_aligned

M, N, K, C, R = 64, 48, 5, 10, 12


def full_matrix(seed=21):
    p = O.lowrank_planes(np.random.default_rng(seed), M, N, K)
    g = np.random.default_rng(seed + 1)
    return tuple(x + 1e-3 * g.standard_normal(x.shape) for x in p)


def as_tensor(planes, rows=None):
    a = np.stack(planes, axis=-1)
    if rows is not None:
        a = a[rows]
    return torch.from_numpy(np.ascontiguousarray(a))


def check(res, planes, strategy, seed, rows=None):
    want = O.approx(planes, strategy, K, seed, C, R)
    assert np.array_equal(res["J"].numpy(), want["cols"])
    assert np.array_equal(res["I"].numpy(), want["rows"])
    got_r = res["R"].numpy()
    for s in range(4):
        assert np.array_equal(got_r[..., s], want["r"][s])
    got_c = res["Cb"].numpy()
    for s in range(4):
        assert np.array_equal(got_c[..., s], want["c"][s][rows] if rows is not None else want["c"][s])
    u = tuple(np.ascontiguousarray(res["U"].numpy()[..., s]) for s in range(4))
    assert O.rel_fro(u, want["u"]) <= 1e-9
    assert abs(res["rel_err"] - want["rel_err"]) <= 1e-10 * want["rel_err"]


def test_subtree_alignment():
    assert subtree_aligned(M * N, 2) and subtree_aligned(32768 * 32768, 8)
    assert subtree_aligned(4000 * 4000, 4)
    assert not subtree_aligned(10 * 13, 2)
    assert not subtree_aligned(4000 * 4000, 3)
    a = np.random.default_rng(0).random(M * N)
    halves = [float(a[: M * N // 2].sum()), float(a[M * N // 2:].sum())]
    assert combine_subtrees(halves) == float(a.sum())


@pytest.mark.parametrize("strategy", ["length", "uniform"])
def test_single_rank_matches_oracle(strategy):
    from rowshard_cpu_ops import CpuOps

    planes = full_matrix()
    res = approx_rowsharded(CpuOps(), SingleComm(), as_tensor(planes), M, strategy, 4, C, R)
    check(res, planes, strategy, 4)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, strategy, q):
    import os
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    sys.path.insert(0, here)
    sys.path.insert(0, os.path.join(os.path.dirname(here), "oracle"))
    import torch.distributed as dist

    from rowshard_cpu_ops import CpuOps

    from paper_2402_19147_b200.rowshard import Comm, approx_rowsharded

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        planes = full_matrix()
        rows = slice(rank * M // world, (rank + 1) * M // world)
        res = approx_rowsharded(CpuOps(), Comm(), as_tensor(planes, rows), M, strategy, 4, C, R)
        check(res, planes, strategy, 4, rows)
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("strategy", ["length", "uniform"])
def test_gloo_world2_matches_single_process_oracle(strategy):
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, strategy, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    assert out == [(0, "ok"), (1, "ok")], out
