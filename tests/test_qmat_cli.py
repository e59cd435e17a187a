"""`.qmat` wire format (quat.py:310-338) and the CLI's host-side contract (no GPU)."""
import os

import numpy as np
import pytest

from golden import cases
from paper_2402_19147_b200 import FileFormatError, QMatrix, read_qmat, write_qmat
from paper_2402_19147_b200.cli import main

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def test_qmat_bytes_match_reference(tmp_path):
    x = QMatrix(*cases.spectral_input(cases.SPECTRAL_CASES["s_1x5"]))
    path = tmp_path / "x.qmat"
    write_qmat(x, path)
    assert path.read_bytes() == G["qmat/s_1x5_bytes"].tobytes()


def test_qmat_round_trip(tmp_path):
    x = QMatrix(*cases.spectral_input(cases.SPECTRAL_CASES["s_30x20"]))
    path = tmp_path / "x.qmat"
    write_qmat(x, path)
    y = read_qmat(path)
    assert y.shape == (30, 20) and all(np.array_equal(a, b) for a, b in zip(x.planes, y.planes))


@pytest.mark.parametrize("payload", [b"", b"QMAT1\x00" + b"\x00" * 8, b"QMAX1\x00" + b"\x00" * 16,
                                     b"QMAT1\x00" + np.array([0, 3], "<u8").tobytes(),
                                     b"QMAT1\x00" + np.array([2, 3], "<u8").tobytes() + b"\x00" * 8])
def test_qmat_rejects_malformed(tmp_path, payload):
    path = tmp_path / "bad.qmat"
    path.write_bytes(payload)
    with pytest.raises(FileFormatError):
        read_qmat(path)


def test_cli_malformed_and_missing_input(tmp_path, capsys):
    bad = tmp_path / "bad.qmat"
    bad.write_bytes(b"not a matrix at all")
    assert main(["approx", str(bad), "--rank", "1"]) == 2
    assert "error:" in capsys.readouterr().err
    assert main(["approx", str(tmp_path / "ghost.qmat"), "--rank", "1"]) == 2
