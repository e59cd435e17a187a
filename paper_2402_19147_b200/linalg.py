"""Pseudoinverse on the GPU — mirror of ``qcur.linalg.pseudoinverse``
(pkg/src/qcur/linalg.py:346-362) for the QMCUR path.

pinv(A) = V diag(1/sigma_i, sigma_i > cutoff) W^H with the default cutoff
eps * max(m, n) * sigma_max (linalg.py:338-339).  Device method: CholeskyQR2
with a kappa guard (no sigma can reach the cutoff) or, otherwise and whenever
``tol`` is given, Householder QR + one-sided Jacobi SVD with the cutoff
applied exactly (csrc/k_dense.cu).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import ParameterError
from .quat import QMatrix, from_device, to_device

__all__ = ["pseudoinverse", "spectral_norm"]


def pseudoinverse(a, tol: float | None = None) -> QMatrix:
    dev = _native.device()
    m, n = (int(v) for v in a.shape)
    ad = to_device(a, dev)
    if tol is not None and float(tol) < 0:
        # the reference returns zeros for the zero matrix before validating tol
        ss = ctypes.c_double()
        dev.call("qcur_frobenius_sq", ad.data_ptr(), m, n, ctypes.byref(ss))
        if ss.value == 0.0:
            return QMatrix.zeros(n, m)
        raise ParameterError(f"tol must be nonnegative, got {tol}")
    out = dev.empty_q(n, m)
    dev.call("qcur_pseudoinverse", ad.data_ptr(), m, n, -1.0 if tol is None else float(tol), out.data_ptr())
    return from_device(out, dev)



# ---------------------------------------------------------------------------
# spectral norm (linalg.py:365-367): largest singular value over right scalars
# ---------------------------------------------------------------------------
def _cdot(u: np.ndarray, v: np.ndarray) -> complex:
    """Complex inner product of quaternion vectors viewed in the complex adjoint
    representation: the 1, i part of sum conj(u_k) v_k."""
    w = u[:, 0] * v[:, 0] + u[:, 1] * v[:, 1] + u[:, 2] * v[:, 2] + u[:, 3] * v[:, 3]
    x = u[:, 0] * v[:, 1] - u[:, 1] * v[:, 0] - u[:, 2] * v[:, 3] + u[:, 3] * v[:, 2]
    return complex(float(w.sum()), float(x.sum()))


def _rmul_c(v: np.ndarray, a: complex) -> np.ndarray:
    """v * a for a complex scalar a = (re, im, 0, 0) acting on the right."""
    re, im = a.real, a.imag
    out = np.empty_like(v)
    out[:, 0] = v[:, 0] * re - v[:, 1] * im
    out[:, 1] = v[:, 0] * im + v[:, 1] * re
    out[:, 2] = v[:, 2] * re + v[:, 3] * im
    out[:, 3] = -v[:, 2] * im + v[:, 3] * re
    return out


def spectral_norm(a, max_iter: int = 300, tol: float = 1e-15) -> float:
    """Largest singular value of a quaternion matrix (linalg.py:365-367).

    The reference takes the top singular value of the complex adjoint chi(A)
    from a full SVD.  Here: Lanczos with full reorthogonalisation on
    chi(A)^H chi(A), whose complex-linear action is a quaternion A^H (A v) with
    complex scalars acting on the right; the two matrix-vector products per step
    run on the device (qcur_qgemv, one HBM pass over A each), the Krylov
    bookkeeping on the host.  Stops when the top Ritz value is stable to `tol`
    (relative) twice in a row or the Krylov space is exhausted."""
    dev = _native.device()
    m, n = (int(v) for v in a.shape)
    ad = to_device(a, dev)
    t = dev.torch
    xd = dev.empty(n, 4)
    yd = dev.empty(m, 4)
    zd = dev.empty(n, 4)

    def apply(v: np.ndarray) -> np.ndarray:
        xd.copy_(t.from_numpy(np.ascontiguousarray(v)))
        dev.call("qcur_qgemv", 0, m, n, ad.data_ptr(), n, xd.data_ptr(), yd.data_ptr())
        dev.call("qcur_qgemv", 1, m, n, ad.data_ptr(), n, yd.data_ptr(), zd.data_ptr())
        return zd.cpu().numpy()

    v = np.random.default_rng(0x5EC7).standard_normal((n, 4))
    v /= np.sqrt((v * v).sum())
    basis = [v]
    alphas: list[float] = []
    betas: list[float] = []
    w = apply(v)
    lam_prev, stable, lam = None, 0, 0.0
    kmax = min(max_iter, 2 * n)
    for j in range(kmax):
        alpha = _cdot(basis[j], w).real
        alphas.append(alpha)
        w = w - basis[j] * alpha
        if j > 0:
            w = w - basis[j - 1] * betas[j - 1]
        for _ in range(2):  # full reorthogonalisation (classical Gram-Schmidt, twice)
            for q in basis:
                w = w - _rmul_c(q, _cdot(q, w))
        beta = float(np.sqrt((w * w).sum()))
        tri = np.diag(alphas) + np.diag(betas, 1) + np.diag(betas, -1)
        lam = float(np.linalg.eigvalsh(tri)[-1])
        if lam_prev is not None and abs(lam - lam_prev) <= tol * abs(lam):
            stable += 1
            if stable >= 2:
                break
        else:
            stable = 0
        lam_prev = lam
        if beta <= 1e-14 * max(abs(lam), 1e-300):
            break  # invariant subspace: the Ritz values are exact
        betas.append(beta)
        v = w / beta
        basis.append(v)
        w = apply(v)
    return float(np.sqrt(max(lam, 0.0)))
