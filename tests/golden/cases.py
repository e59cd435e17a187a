"""Golden-case definitions shared by make_golden.py (run once, in the build
container, against the reference package) and the tests (which regenerate the
same inputs with element-wise numpy and compare against the stored outputs)."""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
import oracle as O  # noqa: E402

# name: (m, n, rank, noise, gen_seed, strategy, plan_seed, num_rows, num_cols)
QMCUR_CASES = {
    "small_10x8": (10, 8, 3, 1e-3, 41, "length", 41, None, None),
    "small_15x11": (15, 11, 4, 0.0, 45, "length", 123, None, None),
    "shape_12x9": (12, 9, 2, 1e-3, 44, "length", 7, 4, 3),
    "rankdef_100_length": (100, 100, 5, 0.0, 31, "length", 31, None, None),
    "rankdef_100_uniform": (100, 100, 5, 0.0, 31, "uniform", 31, None, None),
    "mid_200x150_uniform": (200, 150, 10, 1e-3, 3, "uniform", 3, 40, 30),
    "mid_300x260_length": (300, 260, 12, 1e-3, 11, "length", 11, 48, 36),
    "cfg1_like_1000": (1000, 1000, 10, 1e-3, 2024, "uniform", 0, 40, 40),
    "wide_40x300_length": (40, 300, 6, 1e-3, 9, "length", 9, 20, 30),
}
DIST_CASES = {"d_6x5": (6, 5, 10), "d_37x1029": (37, 1029, 1), "d_129x7": (129, 7, 7), "d_1x1": (1, 1, 8),
              "d_300x8200": (300, 8200, 6)}
DRAW_CASES = {"w_20_12": (20, 12, 99), "w_4000_200": (4000, 200, 1), "w_33_30": (33, 30, 3),
              "w_1100_1000": (1100, 1000, 8), "w_9_9": (9, 9, 5)}
PINV_CASES = {"p_10x8": (10, 8, 1), "p_8x10": (8, 10, 2), "p_64x40": (64, 40, 3), "p_1x5": (1, 5, 4)}
RNG_SEEDS = [0, 1, 7, 12345, 2 ** 40 + 3, 2 ** 70 + 5]
# completion (completion.py): name: (m, n, rank, gen_seed, missing_ratio, mask_seed,
#                                    strategy, index_policy, seed, max_iters, rel_tol)
COMPLETION_CASES = {
    "comp_uniform_40x36": (40, 36, 3, 21, 0.3, 22, "uniform", "resample_each_iter", 4, 200, 1e-4),
    "comp_length_30x30": (30, 30, 3, 23, 0.3, 24, "length", "resample_each_iter", 2, 200, 1e-4),
    "comp_fixed_30x28": (30, 28, 2, 25, 0.4, 26, "length", "fixed", 3, 20, 1e-4),
    "comp_budget_24x20": (24, 20, 2, 27, 0.5, 28, "uniform", "resample_each_iter", 7, 3, 1e-14),
}
SPECTRAL_CASES = {"s_30x20": (30, 20, 0, 31), "s_lowrank_40": (40, 40, 3, 32), "s_1x5": (1, 5, 0, 33),
                  "s_64x12": (64, 12, 0, 34)}
QSVD_CASES = {"q_9x6": (9, 6, 0, 41), "q_6x9": (6, 9, 0, 42), "q_lowrank_10x8": (10, 8, 3, 43),
              "q_30x30": (30, 30, 0, 44), "q_1x4": (1, 4, 0, 45)}
# (m, n, k, noise, seed, |I|, |J|, norm)
PERT_CASES = {"pb_spec_40x36": (40, 36, 3, 1e-4, 51, 12, 10, "spectral"),
              "pb_fro_40x36": (40, 36, 3, 1e-4, 51, 12, 10, "frobenius"),
              "pb_spec_60x50": (60, 50, 4, 1e-3, 52, 16, 14, "spectral")}
DERIVE_SEED_CASES = [(0, ("draw",)), (5, ("sweep", 0)), (5, ("sweep", 17)), (2 ** 63 + 11, ("batch", 3))]


def qmcur_input(case):
    m, n, k, noise, gseed = case[:5]
    p = O.lowrank_planes(np.random.default_rng(gseed), m, n, k)
    if noise:
        g = np.random.default_rng(gseed + 7919)
        p = tuple(x + noise * g.standard_normal(x.shape) for x in p)
    return p


def dist_input(case):
    m, n, seed = case
    return O.random_planes(np.random.default_rng(seed), m, n)


def draw_input(case):
    size, count, seed = case
    p = np.random.default_rng(seed).random(size) ** 3
    return p / p.sum(), count, seed


def pinv_input(case):
    m, n, seed = case
    return O.random_planes(np.random.default_rng(100 + seed), m, n)


def completion_input(case):
    """(truth planes, observed mask, y = truth on the observed entries, zeros elsewhere)."""
    m, n, k, gseed, ratio, mseed = case[:6]
    truth = O.lowrank_planes(np.random.default_rng(gseed), m, n, k)
    observed = O.random_mask(m, n, ratio, mseed)
    y = O.project_observed(tuple(np.zeros((m, n)) for _ in range(4)), observed, truth)
    return truth, observed, y


def spectral_input(case):
    m, n, k, seed = case
    g = np.random.default_rng(seed)
    if k:
        p = O.lowrank_planes(g, m, n, k)
        return tuple(x + 1e-6 * g.standard_normal(x.shape) for x in p)
    return O.random_planes(g, m, n)


def qsvd_input(case):
    m, n, k, seed = case
    g = np.random.default_rng(seed)
    return O.lowrank_planes(g, m, n, k) if k else O.random_planes(g, m, n)


def pert_input(case):
    """(clean rank-k X, noise E, rows I, cols J)."""
    m, n, k, noise, seed, nr, nc = case[:7]
    g = np.random.default_rng(seed)
    x = O.lowrank_planes(g, m, n, k)
    e = tuple(noise * g.standard_normal((m, n)) for _ in range(4))
    rows = np.sort(g.choice(m, nr, replace=False)).astype(np.int64)
    cols = np.sort(g.choice(n, nc, replace=False)).astype(np.int64)
    return x, e, rows, cols
