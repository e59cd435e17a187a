"""CLI `approx` end to end (cli.py:169-189, test_cli.py TestApprox semantics) and the
Krylov spectral norm against the reference's SVD-based spectral_norm (linalg.py:365-367)."""
import os

import numpy as np
import pytest

import paper_2402_19147_b200 as q
from golden import cases
from helpers import lowrank
from paper_2402_19147_b200.cli import main

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


@pytest.mark.parametrize("name", sorted(cases.SPECTRAL_CASES))
def test_spectral_norm_matches_reference(name):
    x = q.QMatrix(*cases.spectral_input(cases.SPECTRAL_CASES[name]))
    ref = float(G[f"{name}/sigma"][0])
    got = q.spectral_norm(x)
    assert abs(got - ref) <= 1e-12 * ref, (got, ref)


@pytest.fixture
def qmat_file(tmp_path):
    path = tmp_path / "input.qmat"
    q.write_qmat(lowrank(10, 8, 2, seed=77), path)
    return path


def test_exact_factorization(qmat_file, tmp_path):
    out = tmp_path / "out"
    assert main(["approx", str(qmat_file), "--rank", "2", "--seed", "3", "--out", str(out)]) == 0
    for name in ("C.qmat", "U.qmat", "R.qmat", "reconstruction.qmat", "metrics.csv"):
        assert (out / name).is_file()
    header, row = (out / "metrics.csv").read_text().splitlines()
    assert header == "rel_err_fro,err_spec,time_s"
    rel_err, err_spec, elapsed = (float(v) for v in row.split(","))
    assert rel_err <= 1e-8 and err_spec <= 1e-7 and elapsed == 0.0
    x = q.read_qmat(qmat_file)
    rec = q.read_qmat(out / "reconstruction.qmat")
    assert all(np.max(np.abs(a - b)) <= 1e-8 for a, b in zip(x.planes, rec.planes))


def test_byte_reproducible(qmat_file, tmp_path):
    outs = [tmp_path / "a", tmp_path / "b"]
    for out in outs:
        assert main(["approx", str(qmat_file), "--rank", "2", "--seed", "9", "--out", str(out)]) == 0
    for name in ("C.qmat", "U.qmat", "R.qmat", "reconstruction.qmat", "metrics.csv"):
        assert (outs[0] / name).read_bytes() == (outs[1] / name).read_bytes()


def test_timing_flag_and_infeasible_rank(qmat_file, tmp_path, capsys):
    out = tmp_path / "timed"
    assert main(["approx", str(qmat_file), "--rank", "2", "--time", "--out", str(out)]) == 0
    assert float((out / "metrics.csv").read_text().splitlines()[1].split(",")[2]) > 0.0
    assert main(["approx", str(qmat_file), "--rank", "99", "--out", str(tmp_path / "x")]) == 2
    assert "exceeds" in capsys.readouterr().err
