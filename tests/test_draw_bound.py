"""The draw kernel's proof bound (k_draw.cu) on weights with a large dynamic range.

A dominant weight drawn first leaves rounding of its own size in every later
prefix while the remaining mass is 1e-13 of it; the bound must follow the
totals seen so far, not today's total (round-1 advisor finding).  The kernel's
arithmetic is restated in tests/draw_sim.py; the GPU test of the same inputs
is test_gpu_parity.py::test_draw_dynamic_range."""
import numpy as np
import pytest

from draw_sim import dev_draw, np_draw


def _weights(kind: str, n: int, g):
    if kind == "dominant":
        p = g.random(n)
        p[g.integers(n)] *= 1e13
    elif kind == "geometric":
        p = 10.0 ** (-g.random(n) * 30)
    else:
        p = g.random(n) ** 3
    return p / p.sum()


@pytest.mark.parametrize("kind,n,count,trials", [("dominant", 64, 40, 150), ("geometric", 64, 40, 60),
                                                  ("dominant", 300, 100, 8), ("plain", 300, 100, 8)])
def test_tree_decisions_match_numpy(kind, n, count, trials):
    for s in range(trials):
        p = _weights(kind, n, np.random.default_rng(s))
        uni = np.random.default_rng(1000 + s).random(count)
        assert dev_draw(p, count, uni, use_new=True) == np_draw(p, count, uni), (kind, s)


def test_previous_bound_was_unsound():
    # the round-1 rule (delta relative to today's total) accepts wrong indices here
    bad = 0
    for s in range(60):
        p = _weights("geometric", 64, np.random.default_rng(s))
        uni = np.random.default_rng(1000 + s).random(40)
        bad += dev_draw(p, 40, uni, use_new=False) != np_draw(p, 40, uni)
    assert bad > 0
