"""Parity at the BASELINE.json configurations on the production path (VERDICT r1 "next" #1).

Every case runs the public API (make_plan + qmcur + cur_relative_error, the C ABI underneath)
twice: in the default engine mode (the INT8 tensor-core engine where its size thresholds
trigger: X Q_R and the fused error when m n r >= 3e7, the CholeskyQR2 Grams when p q^2 >= 1e6)
and with the FP64 DMMA engine forced.  Against the oracle (oracle/oracle.py, pinned to the
reference) on the same input bits:

  probabilities bit-exact, I / J equal, C / R bit-exact, U within 1e-9 relative Frobenius,
  relative error within 1e-10 of the oracle's value (raw |got - ref| / ref, no slack term:
  at these sizes the error is ~1e-3 of ||X|| and both fp64 evaluations sit ~1e-14 from the
  exact value).

Configurations (bench.py CONFIGS): cfg2 (4000^2, rank 50, length, c = r = 200, plan seed 1),
cfg3 at c = r = 256 (2048^2 image-like), one cfg4 matrix (1024^2, uniform, c = r = 80) and
the cfg5 twin (8192^2 from the on-device cfg5 generator, rank 200, length, c = r = 250).
The 16-CTA cluster Cholesky runs at q = 80 / 200 / 250 / 256 here.
"""
import math

import numpy as np
import pytest
import torch

import oracle as O
import paper_2402_19147_b200 as q
from paper_2402_19147_b200 import _native
from paper_2402_19147_b200.quat import from_device

from bench import CONFIGS, host_lowrank

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

U_TOL = 1e-9
ERR_TOL = 1e-10


def default_mode() -> int:
    import os
    return {"dmma": 1, "int8": 2}.get(os.environ.get("QCUR_GEMM", ""), 0)


_oracle_cache: dict = {}


def cfg5_twin_planes():
    m = n = 8192
    dev = _native.device()
    x = dev.empty_q(m, n)
    dev.call("qcur_synth_lowrank_rows", m, n, 200, CONFIGS["cfg5"]["gen_seed"], 1e-3, 0, m, x.data_ptr())
    planes = tuple(p.copy() for p in from_device(x, dev).planes)
    del x
    torch.cuda.empty_cache()
    return planes


CASES = {
    # name: (planes factory, strategy, rank, plan seed, c, r)
    "cfg2": (lambda: host_lowrank(CONFIGS["cfg2"], CONFIGS["cfg2"]["gen_seed"]), "length", 50, 1, 200, 200),
    "cfg3_c256": (lambda: host_lowrank(CONFIGS["cfg3"], CONFIGS["cfg3"]["gen_seed"]), "length", 64, 3, 256, 256),
    "cfg4_b0": (lambda: host_lowrank(CONFIGS["cfg4"], CONFIGS["cfg4"]["gen_seed"]), "uniform", 20, 0, 80, 80),
    "cfg5_twin": (cfg5_twin_planes, "length", 200, 5, 250, 250),
}


def oracle_case(name):
    if name not in _oracle_cache:
        _oracle_cache.clear()  # keep one large case resident at a time
        make, strategy, rank, seed, c, r = CASES[name]
        planes = tuple(np.ascontiguousarray(p, dtype=np.float64) for p in make())
        ref = O.approx(planes, strategy, rank, seed, c, r)
        _oracle_cache[name] = (planes, ref)
    return _oracle_cache[name]


@pytest.mark.parametrize("mode", ["auto", "fp64"])
@pytest.mark.parametrize("name", list(CASES))
def test_baseline_config_parity(name, mode):
    planes, ref = oracle_case(name)
    _, strategy, rank, seed, c, r = CASES[name]
    dev = _native.device()
    dev.call("qcur_set_gemm_mode", 1 if mode == "fp64" else default_mode())
    try:
        x = q.QMatrix(*planes)
        plan = q.make_plan(x, strategy, rank, seed, num_rows=r, num_cols=c)
        f = q.qmcur(x, plan)
        err = q.cur_relative_error(x, f)
    finally:
        dev.call("qcur_set_gemm_mode", default_mode())
    assert np.array_equal(plan.col_probs, ref["col_probs"]) and np.array_equal(plan.row_probs, ref["row_probs"])
    assert np.array_equal(f.col_indices, ref["cols"])
    assert np.array_equal(f.row_indices, ref["rows"])
    for got, want in zip(f.c.planes, ref["c"]):
        assert np.array_equal(got, want)
    for got, want in zip(f.r.planes, ref["r"]):
        assert np.array_equal(got, want)
    du = O.rel_fro(tuple(f.u.planes), ref["u"])
    derr = abs(err - ref["rel_err"]) / ref["rel_err"]
    print(f"{name} [{mode}]: U rel diff {du:.3e}, error {err:.15e} vs oracle {ref['rel_err']:.15e} "
          f"(rel diff {derr:.3e})")
    assert du <= U_TOL, du
    assert derr <= ERR_TOL, (err, ref["rel_err"])
    assert math.isfinite(err) and err < 1.0
