"""The INT8 tensor-core contraction (tcgen05 kind::i8, Ozaki scheme II) behind Y = X Q_R.

The product is computed exactly in integers from X and B rounded to `bits` significant bits
relative to their row / column maxima, so its error must sit at FP64 level: checked against an
extended-precision host product, against the FP64 DMMA GEMM, on edge shapes (K and N not
multiples of the tile, m < 256, a single row) and on extreme row scales.  qmcur with the
INT8 engine forced must meet the same oracle bars as the FP64 engine (U 1e-9, error 1e-10).
"""
import numpy as np
import pytest
import torch

import oracle as O
import paper_2402_19147_b200 as q
from paper_2402_19147_b200 import _native
from helpers import lowrank, rand_mat
from test_gpu_parity import check_against_oracle

pytestmark = pytest.mark.gpu


def default_mode() -> int:
    """The engine new contexts start with (QCUR_GEMM), restored after a test forces one."""
    import os
    return {"dmma": 1, "int8": 2}.get(os.environ.get("QCUR_GEMM", ""), 0)

SIGNS = {0: (1, -1, -1, -1), 1: (1, 1, 1, -1), 2: (1, -1, 1, 1), 3: (1, 1, -1, 1)}


def ref_product(x, b):
    """(m, n, 4) x (n, r, 4) quaternion product in long double (Hamilton: (xb)_t = sum_s +-x_s b_{s^t})."""
    xl, bl = x.astype(np.longdouble), b.astype(np.longdouble)
    y = np.zeros((x.shape[0], b.shape[1], 4), dtype=np.longdouble)
    for t in range(4):
        for s in range(4):
            y[:, :, t] += SIGNS[t][s] * (xl[:, :, s] @ bl[:, :, s ^ t])
    return y


def run_int8(x, b, nmod=0):
    dev = _native.device()
    m, n, r = x.shape[0], x.shape[1], b.shape[1]
    dx, db = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    y = dev.empty_q(m, r)
    dev.call("qcur_qgemm_int8", m, r, n, dx.data_ptr(), n, db.data_ptr(), r, y.data_ptr(), r, nmod)
    return y.cpu().numpy()


def run_fp64(x, b):
    dev = _native.device()
    m, n, r = x.shape[0], x.shape[1], b.shape[1]
    dx, db = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
    y = dev.empty_q(m, r)
    dev.call("qcur_qgemm", 0, 0, m, r, n, 1.0, dx.data_ptr(), n, db.data_ptr(), r, 0.0, y.data_ptr(), r)
    return y.cpu().numpy()


def scaled_err(y, ref, x, b):
    scale = np.sqrt((x ** 2).sum(axis=(1, 2)))[:, None] * np.sqrt((b ** 2).sum(axis=(0, 2)))[None, :]
    scale = np.where(scale > 0, scale, 1.0)
    return float((np.abs(y - ref).max(axis=2) / scale).max())


@pytest.mark.parametrize("m,n,r", [(1, 1, 1), (5, 3, 2), (8, 8, 4), (129, 257, 52), (300, 500, 40),
                                   (257, 33, 67), (1000, 1000, 40)])
@pytest.mark.parametrize("nmod", [14, 15])
def test_int8_gemm_fp64_accuracy(m, n, r, nmod):
    g = np.random.default_rng(m * 7 + n * 3 + r)
    x, b = g.standard_normal((m, n, 4)), g.standard_normal((n, r, 4))
    ref = ref_product(x, b)
    e8 = scaled_err(run_int8(x, b, nmod), ref, x, b)
    ed = scaled_err(run_fp64(x, b), ref, x, b)
    # FP64 level: within a small multiple of the DMMA error and of the unit roundoff
    assert e8 <= max(20 * ed, 4e-15), (e8, ed)


def test_int8_gemm_extreme_row_scales_and_zeros():
    g = np.random.default_rng(5)
    x = g.standard_normal((70, 90, 4)) * np.exp(g.uniform(-300, 300, size=(70, 1, 1)))
    x[3] = 0.0                                   # an all-zero row
    x[4, 10:, :] = 0.0                           # a mostly-zero row
    b = g.standard_normal((90, 20, 4)) * np.exp(g.uniform(-200, 200, size=(1, 20, 1)))
    b[:, 7] = 0.0                                # an all-zero column
    ref = ref_product(x, b)
    y = run_int8(x, b)
    assert np.all(y[3] == 0.0) and np.all(y[:, 7] == 0.0)
    assert scaled_err(y, ref, x, b) <= 4e-15


def test_int8_gemm_bitwise_deterministic():
    g = np.random.default_rng(9)
    x, b = g.standard_normal((300, 260, 4)), g.standard_normal((260, 36, 4))
    assert np.array_equal(run_int8(x, b), run_int8(x, b))


def test_int8_gemm_rejects_bad_arguments():
    dev = _native.device()
    x = torch.zeros((4, 4, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(q.ParameterError):
        dev.call("qcur_qgemm_int8", 4, 4, 4, x.data_ptr(), 4, x.data_ptr(), 4, x.data_ptr(), 4, 3)
    with pytest.raises(q.ParameterError):
        dev.call("qcur_qgemm_int8", 4, 4, 4, x.data_ptr(), 4, x.data_ptr(), 4, x.data_ptr(), 4, 16)
    with pytest.raises(q.ShapeError):
        dev.call("qcur_qgemm_int8", 0, 4, 4, x.data_ptr(), 4, x.data_ptr(), 4, x.data_ptr(), 4, 0)


@pytest.fixture
def int8_engine():
    dev = _native.device()
    dev.call("qcur_set_gemm_mode", 2)
    yield
    dev.call("qcur_set_gemm_mode", default_mode())


@pytest.mark.parametrize("m,n,k,strategy,seed,counts", [
    (10, 8, 3, "length", 41, None),
    (200, 150, 10, "uniform", 3, (40, 30)),
    (300, 260, 12, "length", 11, (48, 36)),
    (1000, 1000, 10, "uniform", 0, (40, 40)),
])
def test_qmcur_int8_engine_matches_oracle(int8_engine, m, n, k, strategy, seed, counts):
    x = lowrank(m, n, k, seed, noise=1e-3)
    kw = {} if counts is None else dict(num_rows=counts[0], num_cols=counts[1])
    plan = q.make_plan(x, strategy, k, seed, **kw)
    check_against_oracle(x, plan, q.qmcur(x, plan))


def test_qmcur_int8_engine_close_to_fp64_engine():
    x = rand_mat(600, 500, seed=77)
    plan = q.make_plan(x, "length", 20, 5, num_rows=80, num_cols=60)
    dev = _native.device()
    dev.call("qcur_set_gemm_mode", 1)
    try:
        f64 = q.qmcur(x, plan)
        dev.call("qcur_set_gemm_mode", 2)
        f8 = q.qmcur(x, plan)
    finally:
        dev.call("qcur_set_gemm_mode", default_mode())
    assert np.array_equal(f64.col_indices, f8.col_indices)
    assert O.rel_fro(tuple(f8.u.planes), tuple(f64.u.planes)) <= 1e-11


def error_stats(x, c, u, r, mode, psnr_scale=0.0):
    """{||X - C U R||^2, ||X||^2, imaginary part, u8-image sum} through qcur_cur_error on one engine."""
    dev = _native.device()
    m, n = x.shape[0], x.shape[1]
    cq, rq = c.shape[1], r.shape[0]
    dx, dc, du, dr = (torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (x, c, u, r))
    out = dev.empty(4)
    dev.call("qcur_set_gemm_mode", mode)
    try:
        dev.call("qcur_cur_error", dx.data_ptr(), m, n, dc.data_ptr(), cq, du.data_ptr(), dr.data_ptr(), rq,
                 psnr_scale, out.data_ptr())
    finally:
        dev.call("qcur_set_gemm_mode", default_mode())
    return out.cpu().numpy()


def exact_err2(x, c, u, r):
    p = ref_product(c, u).astype(np.float64)
    pr = ref_product(p, r)
    return float(((x.astype(np.longdouble) - pr) ** 2).sum())


@pytest.mark.parametrize("m,n,cq,rq", [(37, 53, 5, 7), (129, 300, 20, 12), (300, 257, 40, 40), (700, 900, 64, 48)])
def test_int8_error_matches_fp64_engine_and_exact(m, n, cq, rq):
    g = np.random.default_rng(m + n + cq)
    x = lowrank(m, n, 6, seed=m, noise=1e-3)
    xi = np.stack(x.planes, axis=-1)
    J = g.choice(n, cq, replace=False)
    I = g.choice(m, rq, replace=False)
    c, r = xi[:, J], xi[I, :]
    u = g.standard_normal((cq, rq, 4)) * 1e-2
    s8 = error_stats(xi, c, u, r, 2)
    s64 = error_stats(xi, c, u, r, 1)
    ex = exact_err2(xi, c, u, r)
    assert abs(s8[0] - ex) <= 1e-12 * ex + 1e-300
    assert abs(s8[0] - s64[0]) <= 1e-12 * s64[0]
    assert abs(s8[1] - s64[1]) <= 1e-13 * s64[1]
    assert abs(s8[2] - s64[2]) <= 1e-12 * s64[2]


def test_int8_error_u8_image_statistic():
    g = np.random.default_rng(3)
    m, n, k = 96, 130, 8
    xi = np.clip(np.stack(lowrank(m, n, k, seed=4).planes, axis=-1) * 0.1 + 0.5, 0.0, 1.0)
    J, I = g.choice(n, 24, replace=False), g.choice(m, 20, replace=False)
    c, r = xi[:, J], xi[I, :]
    u = g.standard_normal((24, 20, 4)) * 1e-3
    s8 = error_stats(xi, c, u, r, 2, psnr_scale=255.0)
    s64 = error_stats(xi, c, u, r, 1, psnr_scale=255.0)
    # integer sums of squared u8 differences; a rint() at an exact half-way point may differ
    assert abs(s8[3] - s64[3]) <= 4.0 * max(1.0, 1e-9 * s64[3])
    assert abs(s8[0] - s64[0]) <= 1e-12 * s64[0]


def ref_herm(a, b):
    """A^H B for (p, qa, 4) and (p, qb, 4) in long double."""
    x = np.transpose(a.astype(np.longdouble), (1, 0, 2)).copy()
    x[:, :, 1:] *= -1  # conj(A)^T as a qa x p quaternion matrix
    bl = b.astype(np.longdouble)
    y = np.zeros((x.shape[0], b.shape[1], 4), dtype=np.longdouble)
    for t in range(4):
        for s in range(4):
            y[:, :, t] += SIGNS[t][s] * (x[:, :, s] @ bl[:, :, s ^ t])
    return y


@pytest.mark.parametrize("p,qa,qb,same", [(40, 7, 7, True), (300, 40, 40, True), (257, 33, 20, False),
                                          (1000, 64, 64, True), (4000, 50, 30, False), (5, 1, 1, False)])
def test_int8_hermitian_product(p, qa, qb, same):
    g = np.random.default_rng(p + qa + qb)
    a = g.standard_normal((p, qa, 4))
    b = a if same else g.standard_normal((p, qb, 4))
    dev = _native.device()
    da = torch.from_numpy(a).cuda()
    db = da if same else torch.from_numpy(b).cuda()
    c8 = dev.empty_q(qa, qb)
    dev.call("qcur_qgemm_herm_int8", qa, qb, p, da.data_ptr(), qa, db.data_ptr(), qb, c8.data_ptr(), qb)
    cd = dev.empty_q(qa, qb)
    dev.call("qcur_qgemm", 1, 0, qa, qb, p, 1.0, da.data_ptr(), qa, db.data_ptr(), qb, 0.0, cd.data_ptr(), qb)
    ref = ref_herm(a, b)
    scale = np.sqrt((a ** 2).sum(axis=(0, 2)))[:, None] * np.sqrt((b ** 2).sum(axis=(0, 2)))[None, :]
    e8 = float((np.abs(c8.cpu().numpy() - ref).max(axis=2) / scale).max())
    ed = float((np.abs(cd.cpu().numpy() - ref).max(axis=2) / scale).max())
    assert e8 <= max(20 * ed, 4e-15), (e8, ed)
