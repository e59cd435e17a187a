"""Pin the CPU oracle against golden outputs of the reference package
(tests/golden/golden.npz, made by tests/golden/make_golden.py from qcur)."""
import math
import os

import numpy as np
import pytest

import oracle as O
from golden import cases

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


@pytest.mark.parametrize("name", sorted(cases.QMCUR_CASES))
def test_oracle_qmcur_matches_reference(name):
    m, n, k, noise, gseed, strategy, pseed, nr, nc = cases.QMCUR_CASES[name]
    planes = cases.qmcur_input(cases.QMCUR_CASES[name])
    d_r, d_c = O.default_sample_counts(k, m, n)
    nr = d_r if nr is None else nr
    nc = d_c if nc is None else nc
    res = O.approx(planes, strategy, k, pseed, nc, nr)
    assert np.array_equal(res["col_probs"], G[f"{name}/col_probs"])
    assert np.array_equal(res["row_probs"], G[f"{name}/row_probs"])
    assert np.array_equal(res["cols"], G[f"{name}/cols"])
    assert np.array_equal(res["rows"], G[f"{name}/rows"])
    u_ref = tuple(G[f"{name}/u"])
    assert O.rel_fro(res["u"], u_ref) <= 1e-9
    ref = float(G[f"{name}/rel_err"][0])
    assert abs(res["rel_err"] - ref) <= max(1e-10 * ref, 1e-14)


@pytest.mark.parametrize("name", sorted(cases.DIST_CASES))
def test_oracle_distributions_bitwise(name):
    col, row = O.length_distributions(cases.dist_input(cases.DIST_CASES[name]))
    assert np.array_equal(col, G[f"{name}/col"]) and np.array_equal(row, G[f"{name}/row"])


@pytest.mark.parametrize("name", sorted(cases.DRAW_CASES))
def test_oracle_draws_exact(name):
    p, count, seed = cases.draw_input(cases.DRAW_CASES[name])
    assert np.array_equal(O.draw_indices(p, count, np.random.default_rng(seed)), G[f"{name}/idx"])


@pytest.mark.parametrize("name", sorted(cases.PINV_CASES))
def test_oracle_pinv(name):
    got = O.pinv(cases.pinv_input(cases.PINV_CASES[name]))
    assert O.rel_fro(got, tuple(G[f"{name}/pinv"])) <= 1e-10


def test_oracle_error_definition():
    # relative error = ||X - CUR||_F / ||X||_F with planes summed in order
    planes = cases.qmcur_input(cases.QMCUR_CASES["small_10x8"])
    e2, x2 = O.cur_error(planes, planes, tuple(np.zeros((8, 8)) + (1.0 if s == 0 else 0.0) * np.eye(8) for s in range(4)),
                         tuple(np.eye(8) * (1.0 if s == 0 else 0.0) for s in range(4)))
    assert e2 == pytest.approx(0.0, abs=1e-24) and math.sqrt(x2) > 0


# ---- completion: oracle restatement vs the reference's complete() ----
@pytest.mark.parametrize("name", sorted(cases.COMPLETION_CASES))
def test_oracle_completion_matches_reference(name):
    m, n, k, gseed, ratio, mseed, strategy, policy, seed, iters, tol = cases.COMPLETION_CASES[name]
    truth, observed, y = cases.completion_input(cases.COMPLETION_CASES[name])
    assert np.array_equal(observed, G[f"{name}/mask"])  # random_mask, bit for bit
    x, hist, conv = O.complete(y, observed, k, strategy, iters, tol, policy, seed)
    ref_hist = G[f"{name}/history"]
    assert len(hist) == len(ref_hist) and conv == bool(G[f"{name}/converged"][0])
    # late sweeps measure differences of nearly equal iterates: relative agreement ~1e-7
    assert np.max(np.abs(np.array(hist) - ref_hist) / np.abs(ref_hist)) <= 1e-6
    xs = tuple(G[f"{name}/x_star"][i] for i in range(4))
    assert O.rel_fro(x, xs) <= 1e-8
    assert all(np.array_equal(a[observed], b[observed]) for a, b in zip(x, xs))


def test_oracle_derive_seed_matches_reference():
    got = [O.derive_seed(s, *parts) for s, parts in cases.DERIVE_SEED_CASES]
    assert np.array_equal(np.array(got, dtype=np.uint64), G["derive_seed"])


@pytest.mark.parametrize("name", sorted(cases.QSVD_CASES))
def test_oracle_singular_values_and_rank(name):
    a = cases.qsvd_input(cases.QSVD_CASES[name])
    s = O.singular_values(a)
    want = G[f"{name}/sigma"]
    assert np.allclose(s[: want.size], want, rtol=1e-12, atol=1e-14 * want[0])
    assert O.numerical_rank(a) == int(G[f"{name}/rank"][0])


@pytest.mark.parametrize("name", sorted(cases.PERT_CASES))
def test_oracle_perturbation_bounds(name):
    case = cases.PERT_CASES[name]
    x, e, rows, cols = cases.pert_input(case)
    got = O.perturbation_bounds(x, e, rows, cols, case[2], norm=case[7])
    keys = ["lhs", "bound_a", "bound_b", "noise_norm", "xrp_norm", "cx_norm", "wsub_pinv_norm", "vsub_pinv_norm"]
    want = G[f"{name}/fields"]
    # lhs = ||X - C U R|| of a noisy projection: two correct pseudoinverses (the reference's
    # QSVD + Gram-Schmidt, the oracle's complex-adjoint pinv) differ by ~1e-13 in U, which the
    # small residual amplifies to ~1e-8; every other field is a norm of a well-conditioned factor
    for k, w in zip(keys, want):
        assert got[k] == pytest.approx(w, rel=1e-7 if k == "lhs" else 1e-9), k
    assert got["lhs"] <= got["bound_a"] <= got["bound_b"] or case[7] != "spectral"
