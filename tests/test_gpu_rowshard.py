"""The row-block orchestrator (rowshard.py) on the GPU ops (C ABI), one rank:
must reproduce the monolithic device path (qcur_approx) and the oracle."""
import math

import numpy as np
import pytest

import oracle as O
import paper_2402_19147_b200 as q
from paper_2402_19147_b200 import _native
from paper_2402_19147_b200.cur import DeviceApprox
from paper_2402_19147_b200.rowshard import GpuOps, SingleComm, approx_rowsharded
from helpers import lowrank

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strategy", ["length", "uniform"])
def test_rowshard_gpu_single_rank_matches_monolithic(strategy):
    m, n, k, c, r, seed = 256, 192, 8, 40, 36, 9
    x = lowrank(m, n, k, seed, noise=1e-3)
    dev = _native.device()
    xd = dev.upload_planes(x.planes)
    res = approx_rowsharded(GpuOps(dev), SingleComm(), xd, m, strategy, seed, c, r)
    mono = DeviceApprox(m, n, c, r, dev)
    mono.run(xd, strategy, seed)
    mono.check()
    assert np.array_equal(res["J"].cpu().numpy(), mono.J.cpu().numpy())
    assert np.array_equal(res["I"].cpu().numpy(), mono.I.cpu().numpy())
    assert np.array_equal(res["R"].cpu().numpy(), mono.R.cpu().numpy())
    assert np.array_equal(res["Cb"].cpu().numpy(), mono.C.cpu().numpy())
    u1, u2 = res["U"].cpu().numpy(), mono.U.cpu().numpy()
    assert np.max(np.abs(u1 - u2)) <= 1e-12 * np.max(np.abs(u2))
    assert abs(res["rel_err"] - mono.rel_error()) <= 1e-12 * mono.rel_error()
    # and the oracle
    plan = q.make_plan(x, strategy, k, seed, num_rows=r, num_cols=c)
    rows, cols, C, U, R = O.qmcur(tuple(x.planes), plan.col_probs, plan.row_probs, c, r, seed)
    assert np.array_equal(res["J"].cpu().numpy(), cols) and np.array_equal(res["I"].cpu().numpy(), rows)
    uu = tuple(np.ascontiguousarray(u1[..., s]) for s in range(4))
    assert O.rel_fro(uu, U) <= 1e-9
    e2, x2 = O.cur_error(tuple(x.planes), C, U, R)
    assert abs(res["rel_err"] - math.sqrt(e2 / x2)) <= 1e-10 * math.sqrt(e2 / x2)
