"""Host-side contract of the drop-in API (validation and error classes), which
needs no GPU: mirrors the reference's test_cur.py / test_quat.py validation."""
import numpy as np
import pytest

import paper_2402_19147_b200 as q
from paper_2402_19147_b200 import errors


def test_error_hierarchy_matches_reference():
    assert issubclass(errors.ShapeError, ValueError) and issubclass(errors.ShapeError, errors.QcurError)
    assert issubclass(errors.ParameterError, ValueError)
    assert issubclass(errors.DegenerateDistributionError, ValueError)
    assert issubclass(errors.SamplingError, RuntimeError)
    assert issubclass(errors.DegenerateSamplingError, errors.SamplingError)


@pytest.mark.parametrize("k,m,n,want", [(50, 500, 500, (196, 196)), (5, 100, 100, (9, 9)), (1, 10, 10, (1, 1)),
                                        (2, 10, 10, (2, 2)), (10, 12, 40, (12, 12))])
def test_default_sample_counts_kats(k, m, n, want):
    assert q.default_sample_counts(k, m, n) == want


def test_default_sample_counts_rejects():
    with pytest.raises(q.ParameterError):
        q.default_sample_counts(13, 12, 40)
    with pytest.raises(q.ParameterError):
        q.default_sample_counts(0, 12, 40)


def test_plan_validation():
    with pytest.raises(q.ParameterError):
        q.SamplingPlan("length", 1, 1, 1, 0, np.array([0.5, 0.6]), np.array([1.0]))
    with pytest.raises(q.ParameterError):
        q.SamplingPlan("leverage", 1, 1, 1, 0, np.array([1.0]), np.array([1.0]))
    with pytest.raises(q.ParameterError):
        q.SamplingPlan("length", 4, 3, 4, 0, np.full(10, 0.1), np.full(10, 0.1))
    with pytest.raises(q.ParameterError):
        q.SamplingPlan("length", 1, 11, 1, 0, np.full(10, 0.1), np.full(10, 0.1))
    plan = q.SamplingPlan("uniform", 1, 2, 2, 5, np.full(4, 0.25), np.full(4, 0.25))
    assert not plan.row_probs.flags.writeable


def test_make_plan_rejects_bad_strategy_before_gpu():
    x = q.QMatrix.zeros(4, 4)
    with pytest.raises(q.ParameterError):
        q.make_plan(x, "leverage", 2, seed=0)


def test_qmatrix_contract():
    with pytest.raises(q.ShapeError):
        q.QMatrix(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 3)))
    with pytest.raises(q.ShapeError):
        q.QMatrix(np.zeros((2, 3)), np.zeros((3, 2)), np.zeros((2, 3)), np.zeros((2, 3)))
    a = np.ones((2, 3))
    x = q.QMatrix(a, a, a, a)
    a[0, 0] = 5.0
    assert x.a0[0, 0] == 1.0 and not x.a0.flags.writeable
    assert x[1, 2] == q.Quaternion(1, 1, 1, 1)
    assert x.take_cols([2, 0]).shape == (2, 2)
    with pytest.raises(q.ShapeError):
        x.take_rows([])


def test_quaternion_hamilton():
    i, j, k = q.Quaternion(0, 1), q.Quaternion(0, 0, 1), q.Quaternion(0, 0, 0, 1)
    assert i * j == k and j * k == i and k * i == j
    assert j * i == -k
    assert (i * i).a0 == -1.0


def test_cur_factors_shape_check():
    u = q.QMatrix.zeros(3, 2)
    c = q.QMatrix.zeros(5, 3)
    r = q.QMatrix.zeros(2, 4)
    q.CURFactors(np.arange(2), np.arange(3), c, u, r)
    with pytest.raises(q.ShapeError):
        q.CURFactors(np.arange(3), np.arange(3), c, u, r)


def test_draw_indices_validation_before_gpu():
    with pytest.raises(q.ShapeError):
        q.draw_indices(np.array([]), 1, 0)
    with pytest.raises(q.ParameterError):
        q.draw_indices(np.array([0.5, -0.1]), 1, 0)
    with pytest.raises(q.ParameterError):
        q.draw_indices(np.array([0.5, 0.5]), 0, 0)
    with pytest.raises(q.SamplingError):
        q.draw_indices(np.array([0.5, 0.0, 0.5]), 3, 0)
