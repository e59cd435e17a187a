"""The robust factorization path (rank-deficient or ill-conditioned C / R; the reference's
pinv with its eps max(m, n) sigma_max cutoff, linalg.py:346-362): one-sided Jacobi on the
tall block on a 16-CTA cluster (k_robust.cu), forced with qcur_force_robust or reached by
rank-deficient input, against the oracle."""
import math

import numpy as np
import pytest

import oracle as O
import paper_2402_19147_b200 as q
from paper_2402_19147_b200 import _native
from helpers import exact_rel_error, lowrank, rand_mat

pytestmark = pytest.mark.gpu


class forced_robust:
    def __enter__(self):
        self.dev = _native.device()
        self.dev.lib.qcur_force_robust(self.dev.handle, 1)

    def __exit__(self, *a):
        self.dev.lib.qcur_force_robust(self.dev.handle, 0)


@pytest.mark.parametrize("m,n,k,c,r,strategy", [(300, 260, 12, 36, 48, "length"), (1000, 1000, 10, 40, 40, "uniform"),
                                                (1200, 1100, 30, 120, 110, "length"),
                                                (1000, 900, 20, 200, 196, "length")])
def test_forced_robust_qmcur_matches_oracle(m, n, k, c, r, strategy):
    x = lowrank(m, n, k, seed=m + k, noise=1e-3)
    plan = q.make_plan(x, strategy, k, 7, num_rows=r, num_cols=c)
    with forced_robust():
        f = q.qmcur(x, plan)
        err = q.cur_relative_error(x, f)
    rows, cols, C, U, R = O.qmcur(tuple(x.planes), plan.col_probs, plan.row_probs, c, r, 7)
    assert np.array_equal(f.col_indices, cols) and np.array_equal(f.row_indices, rows)
    assert O.rel_fro(tuple(f.u.planes), U) <= 1e-9
    e2, x2 = O.cur_error(tuple(x.planes), C, U, R)
    ref = math.sqrt(e2 / x2)
    assert abs(err - ref) <= 1e-10 * ref


@pytest.mark.parametrize("m,n,rank", [(400, 60, 20), (60, 400, 20), (1000, 80, 5)])
def test_rank_deficient_pinv_matches_oracle(m, n, rank):
    # exactly rank-deficient: the cutoff drops the zero singular values, as the reference's pinv
    a = lowrank(m, n, rank, seed=m * n)
    got = q.pseudoinverse(a)
    want = O.pinv(tuple(a.planes))
    assert O.rel_fro(tuple(got.planes), want) <= 1e-9


def test_exact_recovery_through_robust_path():
    # rank 5 with c = r = 12: C and R are rank-deficient, the fast path's guard sends them here
    x = lowrank(500, 450, 5, seed=77)
    plan = q.make_plan(x, "length", 5, 3, num_rows=12, num_cols=12)
    f = q.qmcur(x, plan)
    assert q.cur_relative_error(x, f) <= 1e-10


@pytest.mark.parametrize("c,r", [(200, 200), (160, 240)])
def test_rank_deficient_large_blocks_reach_robust_path(c, r):
    # rank 40, c, r >= 160: the Grams are singular, so the cluster Cholesky (the pipelined variant from
    # q = 192) breaks down or the kappa guard trips, and both blocks go through the merged robust launches
    x = lowrank(900, 800, 40, seed=2024)
    plan = q.make_plan(x, "length", 40, 11, num_rows=r, num_cols=c)
    f = q.qmcur(x, plan)
    err = q.cur_relative_error(x, f)
    rows, cols, C, U, R = O.qmcur(tuple(x.planes), plan.col_probs, plan.row_probs, c, r, 11)
    assert np.array_equal(f.col_indices, cols) and np.array_equal(f.row_indices, rows)
    assert O.rel_fro(tuple(f.u.planes), U) <= 1e-9
    assert err <= 1e-10
