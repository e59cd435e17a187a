"""Completion host-side contract (no GPU): masks, config validation, seeds —
the reference's test_completion.py semantics for the parts that run on the host."""
import numpy as np
import pytest

from golden import cases
from paper_2402_19147_b200 import ParameterError, ShapeError
from paper_2402_19147_b200.completion import (CompletionConfig, CompletionResult, ObservationMask, derive_seed,
                                              random_mask)
from paper_2402_19147_b200.quat import QMatrix

G = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden", "golden.npz"))


def test_mask_counts_and_ratio():
    arr = np.zeros((4, 5), dtype=bool)
    arr[0, :] = True
    mask = ObservationMask(arr)
    assert (mask.rows, mask.cols) == (4, 5) and mask.num_observed == 5
    assert abs(mask.missing_ratio - 0.75) <= 1e-12


def test_mask_copies_and_freezes():
    arr = np.ones((2, 2), dtype=bool)
    mask = ObservationMask(arr)
    arr[0, 0] = False
    assert mask.num_observed == 4
    with pytest.raises(ValueError):
        mask.observed[0, 0] = False


def test_mask_validation():
    with pytest.raises(ParameterError):
        ObservationMask(np.ones((2, 2)))
    with pytest.raises(ShapeError):
        ObservationMask(np.ones(4, dtype=bool))


def test_random_mask_exact_and_deterministic():
    assert random_mask(6, 7, 0.0, seed=0).num_observed == 42
    mask = random_mask(512, 768, 0.9, seed=1)
    assert mask.observed.size - mask.num_observed == 353_894
    assert np.array_equal(random_mask(20, 20, 0.5, 9).observed, random_mask(20, 20, 0.5, 9).observed)
    with pytest.raises(ParameterError):
        random_mask(3, 3, 1.0, 0)
    with pytest.raises(ParameterError):
        random_mask(0, 3, 0.1, 0)


@pytest.mark.parametrize("name", sorted(cases.COMPLETION_CASES))
def test_random_mask_matches_reference(name):
    m, n, _, _, ratio, mseed = cases.COMPLETION_CASES[name][:6]
    assert np.array_equal(random_mask(m, n, ratio, mseed).observed, G[f"{name}/mask"])


def test_derive_seed_matches_reference():
    got = [derive_seed(s, *parts) for s, parts in cases.DERIVE_SEED_CASES]
    assert np.array_equal(np.array(got, dtype=np.uint64), G["derive_seed"])


def test_config_defaults_and_validation():
    cfg = CompletionConfig(rank=3)
    assert (cfg.strategy, cfg.max_iters, cfg.rel_tol, cfg.index_policy, cfg.seed) == (
        "length", 200, 1e-4, "resample_each_iter", 0)
    for bad in (dict(rank=0), dict(rank=2, max_iters=0), dict(rank=2, rel_tol=0.0),
                dict(rank=2, index_policy="sometimes"), dict(rank=2, strategy="leverage")):
        with pytest.raises(ParameterError):
            CompletionConfig(**bad)


def test_result_history_length_checked():
    with pytest.raises(ParameterError):
        CompletionResult(x_star=QMatrix.zeros(2, 2), iterations_run=2, rel_change_history=(0.5,), converged=False)
