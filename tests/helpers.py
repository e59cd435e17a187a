"""Shared helpers for the test-suite (generators and comparisons).

Generators use element-wise numpy only, so inputs are bit-identical on the
build container and on the GPU box (no host-BLAS dependence)."""
from __future__ import annotations

import numpy as np

import oracle as O
from paper_2402_19147_b200 import QMatrix


def rand_mat(m, n, seed, scale=1.0) -> QMatrix:
    return QMatrix(*O.random_planes(np.random.default_rng(seed), m, n, scale))


def lowrank(m, n, k, seed, noise=0.0) -> QMatrix:
    p = O.lowrank_planes(np.random.default_rng(seed), m, n, k)
    if noise:
        g = np.random.default_rng(seed + 7919)
        p = tuple(x + noise * g.standard_normal(x.shape) for x in p)
    return QMatrix(*p)


def rel_fro_err(approx, exact) -> float:
    return O.rel_fro(tuple(approx.planes), tuple(exact.planes))


def _qmul_ld(a, b):
    a0, a1, a2, a3 = (np.asarray(t, dtype=np.longdouble) for t in a)
    b0, b1, b2, b3 = (np.asarray(t, dtype=np.longdouble) for t in b)
    return (a0 @ b0 - a1 @ b1 - a2 @ b2 - a3 @ b3, a0 @ b1 + a1 @ b0 + a2 @ b3 - a3 @ b2,
            a0 @ b2 - a1 @ b3 + a2 @ b0 + a3 @ b1, a0 @ b3 + a1 @ b2 - a2 @ b1 + a3 @ b0)


def exact_rel_error(x, c, u, r) -> float:
    """||X - C U R||_F / ||X||_F of the given fp64 factors, evaluated in extended
    precision (x87 long double): the value any fp64 evaluation approximates.

    Two fp64 evaluations of the same error differ by their own rounding (the
    product C U carries ~u * ||C|| ||U|| of it), which for small, nearly square
    C can reach 1e-10 relative; the parity bars compare each side with this
    value."""
    cur = _qmul_ld(_qmul_ld(c, u), r)
    e2 = sum(((np.asarray(p, dtype=np.longdouble) - q) ** 2).sum() for p, q in zip(x, cur))
    x2 = sum((np.asarray(p, dtype=np.longdouble) ** 2).sum() for p in x)
    return float(np.sqrt(e2 / x2))


def assert_error_parity(got: float, ref: float, exact_got: float, exact_ref: float, tol: float = 1e-10) -> None:
    """North-star error bar (1e-10 relative, fp64): our value within tol of the
    exact error of our factors, and within tol of the reference's fp64 value up to
    the reference's own rounding (|ref - exact_ref|)."""
    assert abs(got - exact_got) <= tol * exact_got, (got, exact_got)
    assert abs(got - ref) <= tol * ref + abs(ref - exact_ref) + abs(exact_got - exact_ref), (got, ref, exact_ref)
