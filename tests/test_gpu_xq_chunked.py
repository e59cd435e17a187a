"""Y = X Q_R in row chunks (the cfg5 path: the residue planes of a 34 GB X exceed the one-shot
workspace) must give the bits of the one-shot INT8 product: rows are independent (each is
scaled by its own maximum), and the last chunk, which overlaps its predecessor, recomputes
identical rows.  The caps are lowered through the environment so a small problem chunks."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys, numpy as np, torch
sys.path[:0] = [{root!r}, {root!r} + "/tests", {root!r} + "/oracle"]
from paper_2402_19147_b200 import _native
from paper_2402_19147_b200.quat import to_device
from helpers import rand_mat
dev = _native.device()
m, n, r = 2300, 700, 48
x = to_device(rand_mat(m, n, seed=5), dev)
qr = to_device(rand_mat(n, r, seed=6), dev)
y = dev.empty_q(m, r)
dev.call("qcur_xq", x.data_ptr(), m, n, n, qr.data_ptr(), r, y.data_ptr())
dev.synchronize()
np.save(sys.argv[1], y.cpu().numpy())
"""


def run(env_extra, out):
    env = dict(os.environ, **env_extra)
    code = SCRIPT.format(root=ROOT)
    r = subprocess.run([sys.executable, "-c", code, out], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]


def test_chunked_xq_bitwise_equals_one_shot(tmp_path):
    import numpy as np

    one = str(tmp_path / "one.npy")
    chunked = str(tmp_path / "chunked.npy")
    run({"QCUR_GEMM": "int8"}, one)
    # one-shot cap below this problem's workspace, chunk cap for ~3 chunks of 768 rows
    run({"QCUR_GEMM": "int8", "QCUR_OZ_ONESHOT_CAP": "5e7", "QCUR_OZ_CHUNK_CAP": "3.5e7"}, chunked)
    a, b = np.load(one), np.load(chunked)
    assert a.shape == b.shape and np.array_equal(a, b)
