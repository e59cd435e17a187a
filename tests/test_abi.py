"""The C ABI library loads without a GPU and exports every declared symbol;
host-only entry points (numpy-compatible RNG) work on the CPU."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2402_19147_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "qcur_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qcur_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = _native.load_library()
    syms = header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTS)
    assert lib.qcur_abi_version() == 1


def test_create_without_device_fails_cleanly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a device")
    lib = _native.load_library()
    h = ctypes.c_void_p()
    assert lib.qcur_create(0, ctypes.byref(h)) == 5  # QCUR_E_CUDA


def test_device_raises_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a device")
    with pytest.raises(_native.NativeUnavailable):
        _native.Device(0)


@pytest.mark.parametrize("seed", [0, 1, 7, 12345, 2 ** 40 + 3, 2 ** 70 + 5])
def test_rng_matches_numpy_default_rng(seed):
    st = _native.state_from_seed(seed)
    g = np.random.default_rng(seed)
    assert np.array_equal(_native.state_from_generator(g), st)
    assert np.array_equal(_native.rng_random(st.copy(), 64), g.random(64))


def test_rng_advance_matches_numpy():
    g = np.random.default_rng(99)
    st = _native.state_from_generator(g)
    lib = _native.load_library()
    lib.qcur_rng_advance(st.ctypes.data_as(_native._u64p), 1000)
    g.bit_generator.advance(1000)
    assert np.array_equal(_native.state_from_generator(g), st)


def test_store_generator_state_keeps_stream():
    g = np.random.default_rng(3)
    g.integers(0, 10)  # leaves a buffered uint32
    st = _native.state_from_generator(g)
    _native.store_generator_state(g, st)
    assert g.bit_generator.state["has_uint32"] in (0, 1)


def test_seed_words():
    assert list(_native.seed_words(0)) == [0]
    assert list(_native.seed_words(2 ** 32 + 5)) == [5, 1]
    with pytest.raises(ValueError):
        _native.seed_words(-1)
