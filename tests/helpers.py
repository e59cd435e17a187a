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
