"""QSVD (linalg.py:226-310), numerical_rank (:370-378), lowrank_truncate (:381-383), save_qsvd and
perturbation_bounds (cur.py:306-388) on the GPU, against the oracle and the reference's goldens.

The reference's own invariants (test_linalg.py:62-200) are the bars: singular values equal to
the complex adjoint's (one per pair) to 1e-10 relative, quaternion-orthonormal W and V,
A = W S V^H, truncation is a prefix, rank-deficient and zero inputs, Eckart-Young tail energy.
"""
import os

import numpy as np
import pytest

import oracle as O
import paper_2402_19147_b200 as q
from golden import cases
from helpers import lowrank, rand_mat, rel_fro_err

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def orth_defect(a: q.QMatrix) -> float:
    """max |W^H W - I| over the quaternion Gram."""
    g = a.conj_transpose() @ a
    eye = np.eye(a.cols)
    return float(max(np.abs(g.planes[0] - eye).max(), *(np.abs(p).max() for p in g.planes[1:])))


@pytest.mark.parametrize("name", sorted(cases.QSVD_CASES))
def test_qsvd_matches_reference_sigma(name):
    a = q.QMatrix(*cases.qsvd_input(cases.QSVD_CASES[name]))
    res = q.qsvd(a)
    want = G[f"{name}/sigma"]
    assert res.sigma.shape == want.shape
    assert np.allclose(res.sigma, want, rtol=1e-10, atol=1e-12 * want[0])
    assert q.numerical_rank(a) == int(G[f"{name}/rank"][0])
    assert orth_defect(res.w) < 1e-12 and orth_defect(res.v) < 1e-12
    assert rel_fro_err(res.reconstruct(), a) < 1e-12


@pytest.mark.parametrize("m,n", [(40, 30), (30, 40), (64, 64), (130, 17), (1, 6), (6, 1), (200, 120)])
def test_qsvd_invariants_random(m, n):
    a = rand_mat(m, n, seed=m * 1000 + n)
    res = q.qsvd(a)
    assert res.w.shape == (m, min(m, n)) and res.v.shape == (n, min(m, n))
    s_ref = O.singular_values(tuple(a.planes))
    assert np.allclose(res.sigma, s_ref, rtol=1e-10, atol=1e-12 * s_ref[0])
    assert np.all(np.diff(res.sigma) <= 0)
    assert orth_defect(res.w) < 1e-11 and orth_defect(res.v) < 1e-11
    assert rel_fro_err(res.reconstruct(), a) < 1e-12


def test_qsvd_truncation_prefix_and_bad_k():
    a = rand_mat(7, 6, seed=25)
    full, part = q.qsvd(a), q.qsvd(a, 3)
    assert np.allclose(part.sigma, full.sigma[:3], rtol=1e-12)
    assert part.w.shape == (7, 3) and orth_defect(part.w) < 1e-12
    for bad in (0, -1, 7):
        with pytest.raises(q.ParameterError):
            q.qsvd(a, bad)


def test_qsvd_rank_deficient_zero_and_ties():
    a = lowrank(10, 8, 3, seed=27)
    res = q.qsvd(a)
    assert np.all(res.sigma[3:] < 1e-10 * res.sigma[0])
    assert rel_fro_err(res.reconstruct(), a) < 1e-10
    assert orth_defect(res.w) < 1e-10 and orth_defect(res.v) < 1e-10
    z = q.qsvd(q.QMatrix.zeros(3, 2))
    assert np.all(z.sigma == 0.0) and orth_defect(z.w) == 0.0 and orth_defect(z.v) == 0.0
    eye = q.QMatrix(np.eye(5), np.zeros((5, 5)), np.zeros((5, 5)), np.zeros((5, 5)))
    r = q.qsvd(eye)  # five tied singular values
    assert np.allclose(r.sigma, 1.0, rtol=0, atol=1e-15)
    assert orth_defect(r.w) < 1e-14 and rel_fro_err(r.reconstruct(), eye) < 1e-14


def test_lowrank_truncate_tail_energy_and_numerical_rank():
    a = rand_mat(7, 6, seed=33)
    sigma = q.qsvd(a).sigma
    for k in (1, 3, 5):
        resid = (a - q.lowrank_truncate(a, k)).frobenius_norm()
        assert resid == pytest.approx(float(np.sqrt(np.sum(sigma[k:] ** 2))), rel=1e-8)
    assert q.numerical_rank(lowrank(20, 16, 4, seed=3)) == 4
    assert q.numerical_rank(q.QMatrix.zeros(4, 4)) == 0
    assert q.numerical_rank(a, tol=float(sigma[2]) * 1.0000001) == 2


def test_save_qsvd_round_trip(tmp_path):
    res = q.qsvd(rand_mat(5, 4, seed=29))
    q.save_qsvd(res, tmp_path)
    w, v = q.read_qmat(tmp_path / "w.qmat"), q.read_qmat(tmp_path / "v.qmat")
    sigma = np.array([float(t) for t in (tmp_path / "sigma.txt").read_text().split()])
    assert all(np.array_equal(a, b) for a, b in zip(w.planes, res.w.planes))
    assert all(np.array_equal(a, b) for a, b in zip(v.planes, res.v.planes))
    assert np.array_equal(sigma, res.sigma)


FIELDS = ["lhs", "bound_a", "bound_b", "noise_norm", "xrp_norm", "cx_norm", "wsub_pinv_norm", "vsub_pinv_norm"]


@pytest.mark.parametrize("name", sorted(cases.PERT_CASES))
def test_perturbation_bounds_match_reference(name):
    case = cases.PERT_CASES[name]
    x, e, rows, cols = cases.pert_input(case)
    b = q.perturbation_bounds(q.QMatrix(*x), q.QMatrix(*e), rows, cols, case[2], norm=case[7])
    want = G[f"{name}/fields"]
    for f, w in zip(FIELDS, want):
        # lhs: a small residual of a noisy projection (see test_oracle_golden); spectral norms by Lanczos
        assert getattr(b, f) == pytest.approx(w, rel=1e-7), f
    if case[7] == "spectral":
        assert b.lhs <= b.bound_a <= b.bound_b


def test_perturbation_bounds_errors():
    x, e, rows, cols = cases.pert_input(cases.PERT_CASES["pb_spec_40x36"])
    X, E = q.QMatrix(*x), q.QMatrix(*e)
    with pytest.raises(q.ParameterError):
        q.perturbation_bounds(X, E, rows, cols, 3, norm="nuclear")
    with pytest.raises(q.ShapeError):
        q.perturbation_bounds(X, q.QMatrix.zeros(40, 35), rows, cols, 3)
    with pytest.raises(q.ParameterError):
        q.perturbation_bounds(X, E, rows, cols, 4)  # numerical rank is 3
    with pytest.raises(q.ParameterError):
        q.perturbation_bounds(X, E, rows[:2], cols, 3)


def test_qsvd_truncated_early_stop_matches_full():
    """qsvd(x, k) may stop once the top k columns are certified (qcur_qsvd_jacobi_top); the
    triplets must agree with the fully converged decomposition."""
    g = np.random.default_rng(41)
    m, n, r = 160, 120, 6
    pf = q.QMatrix(*(g.standard_normal((m, r)) for _ in range(4)))
    qf = q.QMatrix(*(g.standard_normal((r, n)) for _ in range(4)))
    s = pf @ qf
    x = q.QMatrix(*(p + 1e-4 * g.standard_normal((m, n)) for p in s.planes))
    full = q.qsvd(x)
    sw_full = q.linalg._last_sweeps
    for k in (1, 3, 6):
        part = q.qsvd(x, k)
        sw_part = q.linalg._last_sweeps
        assert sw_part <= sw_full
        assert np.allclose(part.sigma, full.sigma[:k], rtol=1e-12, atol=0)
        assert orth_defect(part.w) < 1e-12 and orth_defect(part.v) < 1e-12
        # same rank-k truncation (singular vectors up to a unit quaternion phase per column)
        wk = q.QMatrix(*(p[:, :k].copy() for p in full.w.planes))
        vk = q.QMatrix(*(p[:, :k].copy() for p in full.v.planes))
        assert rel_fro_err(part.reconstruct(), q.QSVDResult(wk, full.sigma[:k], vk).reconstruct()) < 1e-10
    assert q.linalg._last_sweeps < sw_full  # k = 6 (the signal rank) stops early
    s_ref = O.singular_values(tuple(x.planes))
    assert np.allclose(q.qsvd(x, 6).sigma, s_ref[:6], rtol=1e-10)
