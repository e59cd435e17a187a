"""Opt-in kernel variants kept for A/B timing must stay correct: each is run in a subprocess with its
environment switch and compared with the default path on the same input.

* QCUR_OZ_BMC=1: the modular GEMM on CTA pairs sharing B by multicast with double-buffered
  accumulators (k_oz_gemm_bmc) gives the bits of the single-CTA kernel (same integer products).
* QCUR_INT8_MIN_Q1=1: Q_1 = Z L_1^-H on the INT8 engine (launch_ozaki_pair); U and the error stay
  within the oracle bars (different rounding from the DMMA product, so not bitwise).
* QCUR_CHOL_PIPE=0 / 1, QCUR_CHOL_BULK=1 and QCUR_SMALL_GEMM=0: the one-column / pipelined / bulk-copy
  cluster Cholesky give identical factors; the DMMA GEMM for the q x q products stays within the bars.
* QCUR_RDIG_EARLY=0, QCUR_PREPB_BCOL=0, QCUR_NATIVE_GRAPH=1: scheduling / launch-shape variants with
  the same bits (the last only affects DeviceApprox graph replays, not this public-API run).
* QCUR_BRES_FAST=0 (with and without QCUR_PREPB_BCOL=0) and =3: the FP64-quotient residues of the right
  operand, and the FP32-limb kernel with a shared-memory transpose tile; the default FP32-limb residues may store the other centred representative of a residue,
  and the products reduce modulo p, so the factors are bitwise equal."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np
sys.path[:0] = [{root!r}, {root!r} + "/tests", {root!r} + "/oracle"]
import paper_2402_19147_b200 as q
from helpers import lowrank
x = lowrank(1500, 1300, 20, seed=3, noise=1e-3)
plan = q.make_plan(x, "length", 20, 4, num_rows=200, num_cols=200)
f = q.qmcur(x, plan)
err = q.cur_relative_error(x, f)
np.savez(sys.argv[1], u=np.stack(f.u.planes), err=np.array([err]), I=f.row_indices, J=f.col_indices)
"""


def run(env_extra, out):
    env = dict(os.environ, **env_extra)
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT), out], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return np.load(out)


@pytest.fixture(scope="module")
def default_run(tmp_path_factory):
    return run({}, str(tmp_path_factory.mktemp("d") / "default.npz"))


@pytest.mark.parametrize("env,bitwise", [({"QCUR_OZ_BMC": "1"}, True), ({"QCUR_CHOL_PIPE": "0"}, True),
                                         ({"QCUR_CHOL_BULK": "1"}, True), ({"QCUR_RDIG_EARLY": "0"}, True),
                                         ({"QCUR_PREPB_BCOL": "0"}, True), ({"QCUR_NATIVE_GRAPH": "1"}, True),
                                         ({"QCUR_CHOL_PIPE": "1"}, True), ({"QCUR_INT8_MIN_Q1": "1"}, False),
                                         ({"QCUR_SMALL_GEMM": "0"}, False), ({"QCUR_BRES_FAST": "0"}, True),
                                         ({"QCUR_BRES_FAST": "0", "QCUR_PREPB_BCOL": "0"}, True),
                                         ({"QCUR_BRES_FAST": "3", "QCUR_PREPB_BCOL": "0"}, True)])
def test_optin_variant_matches_default(tmp_path, default_run, env, bitwise):
    got = run(env, str(tmp_path / "v.npz"))
    assert np.array_equal(got["I"], default_run["I"]) and np.array_equal(got["J"], default_run["J"])
    if bitwise:
        assert np.array_equal(got["u"], default_run["u"]) and np.array_equal(got["err"], default_run["err"])
    else:
        du = np.sqrt(((got["u"] - default_run["u"]) ** 2).sum() / (default_run["u"] ** 2).sum())
        assert du <= 1e-9
        assert abs(got["err"][0] - default_run["err"][0]) <= 1e-10 * default_run["err"][0]
