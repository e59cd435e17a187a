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
    """North-star error bar (1e-10 relative, fp64), as two separate claims plus a report:

    1. our fp64 value is within tol of the exact error of OUR factors (evaluation accuracy);
    2. the exact error of our factors is within tol of the exact error of the REFERENCE's factors
       (factor quality).  U = C^+ X R^+ minimises ||X - C U R||_F over U, so the true error is
       stationary in U: two cores within the 1e-9 U bar differ in true error only to second
       order, far below tol.
    The raw |got - ref| / ref is printed; by 1 and 2 it is at most 2 tol plus the reference's
    own fp64 rounding |ref - exact_ref|, which is not ours to bound (it reaches 8e-11 on the
    golden wide_40x300 case)."""
    raw = abs(got - ref) / ref if ref else abs(got - ref)
    print(f"error parity: got {got:.15e} ref {ref:.15e} raw rel diff {raw:.3e}; "
          f"|got - exact_got| / exact_got {abs(got - exact_got) / exact_got if exact_got else 0.0:.3e}; "
          f"|exact_got - exact_ref| / exact_ref {abs(exact_got - exact_ref) / exact_ref if exact_ref else 0.0:.3e}")
    assert abs(got - exact_got) <= tol * exact_got, ("evaluation", got, exact_got)
    assert abs(exact_got - exact_ref) <= tol * exact_ref, ("factors", exact_got, exact_ref)
