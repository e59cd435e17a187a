"""Pseudoinverse, QSVD, numerical rank and spectral norm on the GPU — mirrors of
``qcur.linalg`` (pkg/src/qcur/linalg.py).

  pseudoinverse     linalg.py:346-362   -> qcur_pseudoinverse (CholeskyQR2 / Householder + Jacobi)
  qsvd              linalg.py:226-310   -> qcur_qsvd_jacobi (quaternion one-sided Jacobi)
  numerical_rank    linalg.py:370-378   -> the same singular values, the pinv cutoff
  lowrank_truncate  linalg.py:381-383   -> W_k diag(sigma_k) V_k^H (GPU quaternion GEMMs)
  spectral_norm     linalg.py:365-367   -> Lanczos on the device (qcur_qgemv)
  save_qsvd         linalg.py:406-420   (host file output)

pinv(A) = V diag(1/sigma_i, sigma_i > cutoff) W^H with the default cutoff
eps * max(m, n) * sigma_max (linalg.py:338-339).  Device method: CholeskyQR2
with a kappa guard (no sigma can reach the cutoff) or, otherwise and whenever
``tol`` is given, Householder QR + one-sided Jacobi SVD with the cutoff
applied exactly (csrc/k_dense.cu).
"""
from __future__ import annotations

import ctypes

import numpy as np

from dataclasses import dataclass

from . import _native
from .errors import ParameterError, ShapeError
from .quat import QMatrix, from_device, to_device

__all__ = ["QSVDResult", "qsvd", "pseudoinverse", "spectral_norm", "numerical_rank", "lowrank_truncate",
           "save_qsvd", "ComplexAdjoint", "to_complex_adjoint", "orthonormalize_columns"]

_EPS = float(np.finfo(np.float64).eps)


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


# ---------------------------------------------------------------------------
# QSVD (linalg.py:226-310) by quaternion one-sided Jacobi on the device
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class QSVDResult:
    """Economy quaternion SVD factors A ~ W diag(sigma) V^H (linalg.py:191-214)."""

    w: QMatrix
    sigma: np.ndarray
    v: QMatrix

    def __post_init__(self) -> None:
        sig = np.array(self.sigma, dtype=np.float64, copy=True)
        sig.setflags(write=False)
        object.__setattr__(self, "sigma", sig)
        if sig.ndim != 1:
            raise ShapeError("sigma must be 1-D")
        if self.w.cols != sig.size or self.v.cols != sig.size:
            raise ShapeError("factor widths disagree with sigma length")

    @property
    def rank_used(self) -> int:
        return int(self.sigma.size)

    def reconstruct(self) -> QMatrix:
        return self.w.scale_columns(self.sigma) @ self.v.conj_transpose()


_last_sweeps = 0  # sweeps of the last Jacobi run (diagnostics)


def _jacobi(a, want_v: bool, k: int = 0):
    """One-sided Jacobi on the device for a (m x n, m >= n): returns (AV columns (n, m, 4),
    V columns (n, n, 4) or None, sigma (n,)) as host arrays, columns unsorted.  0 < k < n: only
    the k largest columns are guaranteed converged (qcur_qsvd_jacobi_top)."""
    dev = _native.device()
    m, n = (int(v) for v in a.shape)
    ad = to_device(a, dev)
    acm = dev.empty(n, m, 4)
    vcm = dev.empty(n, n, 4) if want_v else None
    sig = dev.empty(n)
    sweeps = ctypes.c_int()
    dev.call("qcur_qsvd_jacobi_top", ad.data_ptr(), m, n, n, acm.data_ptr(), vcm.data_ptr() if want_v else None,
             sig.data_ptr(), int(k), ctypes.byref(sweeps))
    global _last_sweeps
    _last_sweeps = sweeps.value
    return acm.cpu().numpy(), (vcm.cpu().numpy() if want_v else None), sig.cpu().numpy()


def _qdot(u: np.ndarray, v: np.ndarray) -> np.ndarray:
    """sum_i conj(u_i) v_i for quaternion vectors stored (len, 4)."""
    a0, a1, a2, a3 = u[:, 0], -u[:, 1], -u[:, 2], -u[:, 3]
    b0, b1, b2, b3 = v[:, 0], v[:, 1], v[:, 2], v[:, 3]
    return np.array([np.sum(a0 * b0 - a1 * b1 - a2 * b2 - a3 * b3), np.sum(a0 * b1 + a1 * b0 + a2 * b3 - a3 * b2),
                     np.sum(a0 * b2 - a1 * b3 + a2 * b0 + a3 * b1), np.sum(a0 * b3 + a1 * b2 - a2 * b1 + a3 * b0)])


def _rmul(u: np.ndarray, q: np.ndarray) -> np.ndarray:
    """u * q (quaternion vector times a quaternion scalar on the right)."""
    a0, a1, a2, a3 = u[:, 0], u[:, 1], u[:, 2], u[:, 3]
    b0, b1, b2, b3 = q
    return np.stack([a0 * b0 - a1 * b1 - a2 * b2 - a3 * b3, a0 * b1 + a1 * b0 + a2 * b3 - a3 * b2,
                     a0 * b2 - a1 * b3 + a2 * b0 + a3 * b1, a0 * b3 + a1 * b2 - a2 * b1 + a3 * b0], axis=1)


def _complete(cols: list, dim: int, need: int) -> list:
    """Extend orthonormal quaternion columns by `need` unit vectors orthogonal to them
    (twice-applied Gram-Schmidt over the canonical basis, as _complete_basis, linalg.py:313-335)."""
    out = list(cols)
    for i in range(dim):
        if len(out) >= len(cols) + need:
            break
        e = np.zeros((dim, 4))
        e[i, 0] = 1.0
        for _ in range(2):
            for q in out:
                e = e - _rmul(q, _qdot(q, e))
        nr = float(np.sqrt(np.sum(e * e)))
        if nr > 1e-3:
            out.append(e / nr)
    if len(out) < len(cols) + need:
        raise ParameterError("failed to complete an orthonormal basis")
    return out[len(cols):]


def _to_qmat(cols: list, dim: int) -> QMatrix:
    arr = np.stack(cols, axis=1) if cols else np.zeros((dim, 0, 4))
    return QMatrix._wrap(*(np.ascontiguousarray(arr[:, :, t]) for t in range(4)))


def qsvd(a, k: int | None = None) -> QSVDResult:
    """Quaternion SVD (linalg.py:226-310): W (m x r), V (n x r) with quaternion-orthonormal
    columns and sigma nonincreasing, r = k or min(m, n).  Computed by one-sided Jacobi on the
    quaternion columns (of A, or of A^H when m < n), so each singular value appears once; the
    zero-singular-value columns of W are completed to an orthonormal set."""
    m, n = (int(v) for v in a.shape)
    r_full = min(m, n)
    if k is None:
        k = r_full
    else:
        k = int(k)
        if not 1 <= k <= r_full:
            raise ParameterError(f"k={k} outside 1..min(m,n)={r_full}")
    tall = m >= n
    src = a if tall else QMatrix._wrap(*_planes_conj_t(a))
    p, q = (m, n) if tall else (n, m)  # src is p x q, p >= q
    av, vc, sig = _jacobi(src, True, k)
    order = np.argsort(-sig, kind="stable")
    sig = sig[order]
    smax = float(sig[0]) if sig.size else 0.0
    if smax == 0.0:
        eye_w = QMatrix._wrap(np.eye(m, k), np.zeros((m, k)), np.zeros((m, k)), np.zeros((m, k)))
        eye_v = QMatrix._wrap(np.eye(n, k), np.zeros((n, k)), np.zeros((n, k)), np.zeros((n, k)))
        return QSVDResult(eye_w, np.zeros(k), eye_v)
    zero_tol = max(2 * m, 2 * n) * _EPS * smax
    left = [av[j] / sig[i] for i, j in enumerate(order[:k]) if sig[i] > zero_tol]
    nz = len(left)
    if nz < k:
        left = left + _complete(left, p, k - nz)
    right = [vc[j] for j in order[:k]]
    w_src, v_src = _to_qmat(left, p), _to_qmat(right, q)
    if tall:
        return QSVDResult(w_src, sig[:k], v_src)
    return QSVDResult(v_src, sig[:k], w_src)  # A^H = W' S V'^H  =>  A = V' S W'^H


def _planes_conj_t(a):
    from .quat import as_planes

    a0, a1, a2, a3 = as_planes(a)
    return a0.T.copy(), -a1.T, -a2.T, -a3.T


def _singular_values(a) -> np.ndarray:
    m, n = (int(v) for v in a.shape)
    src = a if m >= n else QMatrix._wrap(*_planes_conj_t(a))
    _, _, sig = _jacobi(src, False)
    return np.sort(sig)[::-1]


def numerical_rank(a, tol: float | None = None) -> int:
    """Number of singular values above the pseudoinverse cutoff eps max(m, n) sigma_max
    (linalg.py:370-378)."""
    sigma = _singular_values(a)
    smax = float(sigma[0])
    if smax == 0.0:
        return 0
    cutoff = _EPS * max(a.shape) * smax if tol is None else float(tol)
    return int(np.sum(sigma > cutoff))


def lowrank_truncate(a, k: int) -> QMatrix:
    """Best rank-k approximation W_k diag(sigma_k) V_k^H (linalg.py:381-383)."""
    return qsvd(a, k).reconstruct()


def save_qsvd(result: QSVDResult, directory) -> None:
    """W and V as .qmat files plus sigma as a plain-text list (linalg.py:406-420)."""
    from pathlib import Path

    from .quat import write_qmat

    out = Path(directory)
    out.mkdir(parents=True, exist_ok=True)
    write_qmat(result.w, out / "w.qmat")
    write_qmat(result.v, out / "v.qmat")
    with open(out / "sigma.txt", "w") as fh:
        for s_ in result.sigma:
            fh.write(f"{s_:.17g}\n")


# ---------------------------------------------------------------------------
# the complex adjoint and column orthonormalisation (linalg.py:136-164, 385-404)
# ---------------------------------------------------------------------------
@dataclass(frozen=True)
class ComplexAdjoint:
    """The 2m-by-2n complex image chi(A) of an m-by-n quaternion matrix (linalg.py:136-148)."""

    matrix: np.ndarray
    source_rows: int
    source_cols: int

    def __post_init__(self) -> None:
        self.matrix.setflags(write=False)

    @property
    def shape(self) -> tuple[int, int]:
        return self.matrix.shape


def to_complex_adjoint(a) -> ComplexAdjoint:
    """chi(A) = [[A_a, A_b], [-conj(A_b), conj(A_a)]] built on the device (k_complex_adjoint;
    sign flips only, so the block relations hold bit for bit as in linalg.py:151-164)."""
    dev = _native.device()
    m, n = (int(v) for v in a.shape)
    ad = to_device(a, dev)
    chi = dev.empty(2 * m, 2 * n, 2)
    dev.call("qcur_complex_adjoint", ad.data_ptr(), m, n, chi.data_ptr())
    out = chi.cpu().numpy().view(np.complex128).reshape(2 * m, 2 * n).copy()
    return ComplexAdjoint(out, m, n)


def orthonormalize_columns(a) -> QMatrix:
    """An orthonormal basis of A's columns, the Q of A = Q T with T upper triangular and a positive
    real diagonal (the frame the reference's twice-applied Gram-Schmidt produces, linalg.py:385-404;
    QR with a positive diagonal is unique).  On the device: CholeskyQR2 (qcur_factor), the
    Householder path when the kappa guard trips.  ShapeError for more columns than rows;
    ParameterError when a column is numerically dependent on the others."""
    m, n = (int(v) for v in a.shape)
    if n > m:
        raise ShapeError(f"cannot orthonormalize {n} columns in dimension {m}")
    sigma = _singular_values(a)
    from .quat import as_planes

    colnorm2 = sum(p * p for p in as_planes(a)).sum(axis=0)
    scale = max(float(np.sqrt(colnorm2.max())), 1.0)
    if not float(sigma[-1]) > 1e-12 * scale:
        raise ParameterError("columns are numerically dependent on earlier columns")
    dev = _native.device()
    z = to_device(a, dev)
    # qcur_factor returns pinv(Z) = F Q^H with Q = Z L1^-H (one Cholesky pass, orthonormal to
    # kappa^2 u); factoring that Q once more gives Z (L' L1)^-H, orthonormal to u
    for _ in range(2):
        Q, F = dev.empty_q(m, n), dev.empty_q(n, n)
        dev.call("qcur_factor", z.data_ptr(), 0, m, n, Q.data_ptr(), F.data_ptr())
        z = Q
    dev.call("qcur_check")
    return from_device(Q, dev)
