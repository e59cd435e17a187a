"""approx_stream (upload of matrix k+1 overlapped with the approximation of matrix k)
returns exactly what the one-at-a-time public API returns."""
import numpy as np
import pytest

import paper_2402_19147_b200 as q
from helpers import lowrank

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("strategy", ["length", "uniform"])
def test_stream_matches_sequential_api(strategy):
    xs = [lowrank(300, 260, 8, seed=40 + k, noise=1e-3) for k in range(5)]
    seeds = [7 + k for k in range(5)]
    got = list(q.approx_stream(xs, strategy, 8, seeds, num_rows=40, num_cols=32))
    assert [r.index for r in got] == list(range(5))
    for x, s, r in zip(xs, seeds, got):
        plan = q.make_plan(x, strategy, 8, s, num_rows=40, num_cols=32)
        f = q.qmcur(x, plan)
        assert np.array_equal(r.row_indices, f.row_indices) and np.array_equal(r.col_indices, f.col_indices)
        assert all(np.array_equal(a, b) for a, b in zip(r.u.planes, f.u.planes))
        assert r.rel_err == q.cur_relative_error(x, f)
        c, u, rr = r.factors(x)
        assert all(np.array_equal(a, b) for a, b in zip(c.planes, f.c.planes))


def test_stream_reports_degenerate_input():
    xs = [lowrank(50, 40, 3, seed=1), q.QMatrix.zeros(50, 40)]
    it = q.approx_stream(xs, "length", 3, 0)
    with pytest.raises(q.DegenerateDistributionError):
        list(it)


def test_stream_rejects_mixed_shapes():
    with pytest.raises(q.ShapeError):
        list(q.approx_stream([lowrank(20, 20, 2, seed=1), lowrank(21, 20, 2, seed=2)], "uniform", 2, 0))
