"""The small quaternion product kernel (k_qgemm_small.cu: one 8-CTA cluster per 32 x 32 output tile,
k split across the cluster, partials added in rank order through distributed shared memory) behind
qcur_qgemm for M, N, K <= 256: every op(A) / op(B) combination, alpha / beta, ragged sizes, against a
long-double product; determinism and independence of the pairing (the k split depends on K only)."""
import numpy as np
import pytest
import torch

from paper_2402_19147_b200 import _native
from test_gpu_int8 import SIGNS

pytestmark = pytest.mark.gpu


def qprod_ld(a, b):
    al, bl = a.astype(np.longdouble), b.astype(np.longdouble)
    y = np.zeros((a.shape[0], b.shape[1], 4), dtype=np.longdouble)
    for t in range(4):
        for s in range(4):
            y[:, :, t] += SIGNS[t][s] * (al[:, :, s] @ bl[:, :, s ^ t])
    return y


def conj_t(a):
    out = np.transpose(a, (1, 0, 2)).copy()
    out[:, :, 1:] *= -1.0
    return out


def run(opa, opb, M, N, K, alpha, beta, a, b, c0):
    dev = _native.device()
    da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
    dc = torch.from_numpy(c0.copy()).cuda()
    lda, ldb = a.shape[1], b.shape[1]
    dev.call("qcur_qgemm", opa, opb, M, N, K, alpha, da.data_ptr(), lda, db.data_ptr(), ldb, beta, dc.data_ptr(), N)
    return dc.cpu().numpy()


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (3, 5, 2), (7, 33, 9), (40, 40, 40), (80, 80, 80), (200, 200, 200),
                                   (256, 256, 256), (31, 200, 129), (200, 17, 256)])
@pytest.mark.parametrize("opa,opb", [(0, 0), (1, 0), (0, 1), (1, 1)])
def test_small_product_matches_long_double(M, N, K, opa, opb):
    g = np.random.default_rng(M * 1000 + N * 10 + K + 7 * opa + 3 * opb)
    a = g.standard_normal((M, K, 4) if opa == 0 else (K, M, 4))
    b = g.standard_normal((K, N, 4) if opb == 0 else (N, K, 4))
    c0 = g.standard_normal((M, N, 4))
    alpha, beta = -0.75, 1.5
    got = run(opa, opb, M, N, K, alpha, beta, a, b, c0)
    A = a if opa == 0 else conj_t(a)
    B = b if opb == 0 else conj_t(b)
    ref = alpha * qprod_ld(A, B) + beta * c0.astype(np.longdouble)
    scale = abs(alpha) * np.sqrt((A ** 2).sum(axis=(1, 2)))[:, None] * np.sqrt((B ** 2).sum(axis=(0, 2)))[None, :]
    scale = scale + abs(beta) * np.abs(c0).max(axis=2)
    err = (np.abs(got - ref).max(axis=2) / scale).max()
    assert err <= 8 * K * 2.0 ** -53 + 1e-16


def test_small_product_beta_zero_ignores_garbage_and_is_deterministic():
    g = np.random.default_rng(5)
    a, b = g.standard_normal((200, 200, 4)), g.standard_normal((200, 200, 4))
    c0 = np.full((200, 200, 4), np.nan)
    outs = [run(0, 1, 200, 200, 200, 1.0, 0.0, a, b, c0) for _ in range(5)]
    assert np.isfinite(outs[0]).all()
    for o in outs[1:]:
        assert np.array_equal(o, outs[0])


def test_small_product_bits_do_not_depend_on_m():
    # the k split depends on K only: the first 40 rows of a 200-row product equal a 40-row product
    g = np.random.default_rng(9)
    a, b = g.standard_normal((200, 150, 4)), g.standard_normal((150, 120, 4))
    z = np.zeros((200, 120, 4))
    full = run(0, 0, 200, 120, 150, 1.0, 0.0, a, b, z)
    part = run(0, 0, 40, 120, 150, 1.0, 0.0, a[:40].copy(), b, z[:40].copy())
    assert np.array_equal(full[:40], part)
