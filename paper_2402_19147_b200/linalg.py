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

from . import _native
from .errors import ParameterError
from .quat import QMatrix, from_device, to_device

__all__ = ["pseudoinverse"]


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

