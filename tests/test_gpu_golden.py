"""GPU path against the REFERENCE's own outputs (tests/golden/golden.npz,
generated from the reference package by tests/golden/make_golden.py)."""
import hashlib
import os

import numpy as np
import pytest

import oracle as O
import paper_2402_19147_b200 as q
from golden import cases
from helpers import assert_error_parity, exact_rel_error

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def planes_hash(planes) -> str:
    h = hashlib.sha256()
    for p in planes:
        h.update(np.ascontiguousarray(p, dtype="<f8").tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", sorted(cases.QMCUR_CASES))
def test_qmcur_matches_reference_golden(name):
    m, n, k, noise, gseed, strategy, pseed, nr, nc = cases.QMCUR_CASES[name]
    x = q.QMatrix(*cases.qmcur_input(cases.QMCUR_CASES[name]))
    plan = q.make_plan(x, strategy, k, pseed, num_rows=nr, num_cols=nc)
    assert np.array_equal(plan.col_probs, G[f"{name}/col_probs"])
    assert np.array_equal(plan.row_probs, G[f"{name}/row_probs"])
    f = q.qmcur(x, plan)
    assert np.array_equal(f.col_indices, G[f"{name}/cols"])
    assert np.array_equal(f.row_indices, G[f"{name}/rows"])
    assert planes_hash(f.c.planes) == str(G[f"{name}/c_sha"][0])
    assert planes_hash(f.r.planes) == str(G[f"{name}/r_sha"][0])
    assert O.rel_fro(tuple(f.u.planes), tuple(G[f"{name}/u"])) <= 1e-9
    ref = float(G[f"{name}/rel_err"][0])
    got = q.cur_relative_error(x, f)
    if ref > 1e-12:
        xp = tuple(x.planes)
        cols, rows = G[f"{name}/cols"], G[f"{name}/rows"]
        exact_ref = exact_rel_error(xp, tuple(p[:, cols] for p in xp), tuple(G[f"{name}/u"]),
                                    tuple(p[rows, :] for p in xp))
        exact_got = exact_rel_error(xp, tuple(f.c.planes), tuple(f.u.planes), tuple(f.r.planes))
        assert_error_parity(got, ref, exact_got, exact_ref)
    else:  # exactly recovered rank-deficient input: both at rounding level
        assert got <= 1e-12


@pytest.mark.parametrize("name", sorted(cases.DIST_CASES))
def test_distributions_match_reference_bitwise(name):
    col, row = q.length_distributions(q.QMatrix(*cases.dist_input(cases.DIST_CASES[name])))
    assert np.array_equal(col, G[f"{name}/col"]) and np.array_equal(row, G[f"{name}/row"])


@pytest.mark.parametrize("name", sorted(cases.DRAW_CASES))
def test_draws_match_reference(name):
    p, count, seed = cases.draw_input(cases.DRAW_CASES[name])
    assert np.array_equal(q.draw_indices(p, count, seed), G[f"{name}/idx"])


@pytest.mark.parametrize("name", sorted(cases.PINV_CASES))
def test_pinv_matches_reference(name):
    got = q.pseudoinverse(q.QMatrix(*cases.pinv_input(cases.PINV_CASES[name])))
    assert O.rel_fro(tuple(got.planes), tuple(G[f"{name}/pinv"])) <= 1e-10
