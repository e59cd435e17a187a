"""CPU checks of the host restatement of the device generator (tests/synth_host.py)."""
import numpy as np

from synth_host import normals, uniforms


def test_uniform_ranges_and_determinism():
    u1, u2 = uniforms(20240305, 3, np.arange(0, 4096, dtype=np.uint64))
    assert (u1 > 0).all() and (u1 <= 1).all() and (u2 >= 0).all() and (u2 < 1).all()
    v1, v2 = uniforms(20240305, 3, np.arange(0, 4096, dtype=np.uint64))
    assert np.array_equal(u1, v1) and np.array_equal(u2, v2)
    w1, _ = uniforms(20240306, 3, np.arange(0, 4096, dtype=np.uint64))
    assert not np.array_equal(u1, w1)


def test_blocks_are_slices_of_the_stream():
    whole = normals(7, 1, 0, 10000)
    assert np.array_equal(whole[2468:2468 + 1000], normals(7, 1, 2468, 1000))


def test_normal_moments():
    z = normals(11, 2, 0, 200000)
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01
