"""qcur_approx_batched: a batch of same-shape matrices through the whole pipeline
in one ABI call (lanes overlapping one another, capturable as one CUDA graph) gives, matrix by
matrix, the bits of one-at-a-time qcur_approx, and the oracle's indices / U / error."""
import math

import numpy as np
import pytest
import torch

import oracle as O
from paper_2402_19147_b200 import _native
from paper_2402_19147_b200.cur import DeviceApprox, DeviceBatch
from paper_2402_19147_b200.quat import to_device
from helpers import lowrank

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strategy,lanes,graph", [("uniform", 4, False), ("length", 3, True), ("length", 1, False)])
def test_batched_equals_single_and_oracle(strategy, lanes, graph):
    dev = _native.device()
    B, m, n, c, r = 6, 300, 260, 24, 20
    hosts = [lowrank(m, n, 8, seed=100 + b, noise=1e-3) for b in range(B)]
    xs = [to_device(h, dev) for h in hosts]
    seeds = [7 + b for b in range(B)]
    batch = DeviceBatch(B, m, n, c, r, dev, lanes=lanes)
    batch.run(xs, strategy, seeds, graph=graph)
    if graph:
        batch.run(xs, strategy, seeds, graph=True)  # a replay
    batch.check()
    one = DeviceApprox(m, n, c, r, dev)
    for b in range(B):
        one.run(xs[b], strategy, seeds[b])
        one.check()
        assert torch.equal(batch.J[b], one.J) and torch.equal(batch.I[b], one.I)
        assert torch.equal(batch.C[b], one.C) and torch.equal(batch.R[b], one.R)
        assert torch.equal(batch.U[b], one.U)
        assert torch.equal(batch.err4[b], one.err4)
    # matrix 2 against the oracle
    res = O.approx(tuple(hosts[2].planes), strategy, 8, seeds[2], c, r)
    assert np.array_equal(batch.J[2].cpu().numpy(), res["cols"]) and np.array_equal(batch.I[2].cpu().numpy(), res["rows"])
    u = batch.U[2].cpu().numpy()
    assert O.rel_fro(tuple(u[..., k] for k in range(4)), res["u"]) <= 1e-9
    assert abs(batch.rel_errors()[2] - res["rel_err"]) <= 1e-10 * res["rel_err"]


def test_batched_status_reports_sampling_error():
    import paper_2402_19147_b200 as q

    dev = _native.device()
    m, n = 40, 30
    xs = [to_device(q.QMatrix.zeros(m, n), dev), to_device(lowrank(m, n, 3, seed=5), dev)]
    batch = DeviceBatch(2, m, n, 4, 4, dev, lanes=2)
    batch.run(xs, "length", [1, 2])
    with pytest.raises(q.QcurError):
        batch.check()
    batch.run(xs[1:] * 2, "length", [1, 2])
    batch.check()  # the failure bit was consumed; a clean batch reports clean
