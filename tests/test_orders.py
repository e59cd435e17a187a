"""numpy's summation orders, restated in C (oracle/numpy_order.c), pinned
against numpy itself; and the library's compiled pairwise program (the exact
tree the K1 kernels run) evaluated on the host."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
D = ctypes.POINTER(ctypes.c_double)


@pytest.fixture(scope="module")
def olib():
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
    lib = ctypes.CDLL(os.path.join(ROOT, "oracle", "libqcur_oracle.so"))
    lib.qo_pairwise.restype = ctypes.c_double
    lib.qo_pairwise.argtypes = [D, ctypes.c_int64, ctypes.c_int64]
    lib.qo_length_distributions.argtypes = [D, D, D, D, ctypes.c_int64, ctypes.c_int64, D, D, D, D]
    return lib


def p(a):
    return a.ctypes.data_as(D)


@pytest.mark.parametrize("m,n,seed", [(6, 5, 0), (37, 1029, 1), (200, 300, 2), (129, 7, 7), (1, 1, 8), (3, 9000, 9)])
def test_c_oracle_matches_numpy(olib, m, n, seed):
    rng = np.random.default_rng(seed)
    planes = [rng.standard_normal((m, n)) for _ in range(4)]
    sq = sum(q * q for q in planes)
    total = float(sq.sum())
    col = sq.sum(axis=0) / total
    row = sq.sum(axis=1) / total
    sqo, colo, rowo, tot = np.empty(m * n), np.empty(n), np.empty(m), np.empty(1)
    olib.qo_length_distributions(*(p(q) for q in planes), m, n, p(sqo), p(colo), p(rowo), p(tot))
    assert tot[0] == total
    assert np.array_equal(colo, col / col.sum())
    assert np.array_equal(rowo, row / row.sum())


@pytest.mark.parametrize("n", [0, 1, 7, 8, 9, 127, 128, 129, 1000, 8192, 8193, 20000, 123457, 1 << 20])
def test_compiled_pairwise_program_matches_numpy(n):
    from paper_2402_19147_b200 import _native

    lib = _native.load_library()
    a = np.random.default_rng(n).random(n) ** 2
    out = ctypes.c_double()
    assert lib.qcur_pairwise_host(a.ctypes.data, n, ctypes.byref(out)) == 0
    assert out.value == float(a.sum())
