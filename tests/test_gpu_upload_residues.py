"""The drop-in path forms the INT8 X Q_R's residues of X while make_plan uploads X (qcur_upload_length_xq)
and qmcur consumes them (qcur_qmcur_host_xq): the factors must be bit-identical to the plain path, which
forms the residues inside qmcur; a plan with another row count, or a matrix below the INT8 threshold,
falls back to the plain path."""
import numpy as np
import pytest

import paper_2402_19147_b200 as q
from helpers import lowrank

pytestmark = pytest.mark.gpu


def factors(f):
    return (np.stack(f.c.planes), np.stack(f.u.planes), np.stack(f.r.planes), f.row_indices, f.col_indices)


def test_upload_residues_bitwise_equal_plain_path():
    x = lowrank(1500, 1300, 20, seed=41, noise=1e-3)
    plan = q.make_plan(x, "length", 20, 5, num_rows=200, num_cols=180)
    assert x._xq is not None and x._xq[1] == 200  # INT8 X Q_R at this size: residues formed at upload
    fa = factors(q.qmcur(x, plan))
    ea = q.cur_relative_error(x, q.qmcur(x, plan))
    x._xq = None  # the plain path: residues formed inside qmcur
    fb = factors(q.qmcur(x, plan))
    eb = q.cur_relative_error(x, q.qmcur(x, plan))
    for a, b in zip(fa, fb):
        assert np.array_equal(a, b)
    assert ea == eb


def test_upload_residues_other_row_count_falls_back():
    x = lowrank(1200, 1000, 10, seed=42, noise=1e-3)
    plan = q.make_plan(x, "length", 10, 6, num_rows=120, num_cols=100)
    other = q.SamplingPlan(strategy="length", rank=10, num_rows=90, num_cols=100, seed=6,
                           row_probs=plan.row_probs, col_probs=plan.col_probs)
    f1 = factors(q.qmcur(x, other))  # r = 90 != 120: the upload-time residues are not used
    x._xq = None
    f2 = factors(q.qmcur(x, other))
    for a, b in zip(f1, f2):
        assert np.array_equal(a, b)


def test_small_matrix_has_no_upload_residues():
    x = lowrank(120, 100, 5, seed=43, noise=1e-3)
    q.make_plan(x, "length", 5, 1, num_rows=20, num_cols=20)
    assert x._xq is None  # below the INT8 threshold: nothing formed at upload


def test_upload_residues_after_graph_replays():
    # a graph capture of qcur_approx records the side stream's join event inside the capture; the
    # drop-in path with upload-time residues must not wait on that captured record
    from paper_2402_19147_b200 import _native
    from paper_2402_19147_b200.cur import DeviceApprox
    from paper_2402_19147_b200.quat import drop_device_copy, to_device

    dev = _native.device()
    x = lowrank(1500, 1300, 20, seed=44, noise=1e-3)
    xd = to_device(x, dev)
    da = DeviceApprox(1500, 1300, 200, 200, dev)
    for _ in range(2):
        da.run(xd, "length", 3, graph=True)
    dev.synchronize()
    drop_device_copy(x)
    plan = q.make_plan(x, "length", 20, 3, num_rows=200, num_cols=200)
    assert x._xq is not None
    f = q.qmcur(x, plan)
    assert np.isfinite(np.stack(f.u.planes)).all()
