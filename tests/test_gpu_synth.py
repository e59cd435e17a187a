"""The on-device generator behind cfg5 (and every bench input), SURVEY 8(c) cfg5 row.

* its normal stream equals the host restatement (tests/synth_host.py): Philox integers and
  uniforms bit-exact, normals to a few ulps (device log / sincospi vs host libm);
* a row block of the generated matrix equals the host restatement of that block;
* row blocks generated independently, as the G ranks of a row-sharded run do, concatenate
  bit for bit to the G = 1 matrix (the product S = P Q^H is summed over k in one fixed order
  per element, whatever the block's height).
"""
import numpy as np
import pytest
import torch

from paper_2402_19147_b200 import _native
from synth_host import lowrank_rows, normals

pytestmark = pytest.mark.gpu


def dev_normals(seed, stream, offset, count):
    dev = _native.device()
    out = dev.empty(count)
    dev.call("qcur_synth_normals", seed, stream, offset, count, 1.0, out.data_ptr())
    return out.cpu().numpy()


@pytest.mark.parametrize("stream,offset,count", [(1, 0, 4096), (2, 123456, 3001), (3, 2 ** 33, 2048)])
def test_normals_match_host_restatement(stream, offset, count):
    got = dev_normals(20240305, stream, offset, count)
    want = normals(20240305, stream, offset, count)
    assert np.max(np.abs(got - want)) <= 8 * np.finfo(float).eps * np.max(np.abs(want))


def gen_rows(m, n, k, seed, noise, row0, rows):
    dev = _native.device()
    x = dev.empty_q(rows, n)
    dev.call("qcur_synth_lowrank_rows", m, n, k, seed, noise, row0, rows, x.data_ptr())
    return x


@pytest.mark.parametrize("row0,rows", [(0, 64), (1000, 64), (4032, 64)])
def test_row_block_matches_host(row0, rows):
    m, n, k = 4096, 512, 200
    got = gen_rows(m, n, k, 20240305, 1e-3, row0, rows).cpu().numpy()
    want = lowrank_rows(m, n, k, 20240305, 1e-3, row0, rows)
    scale = np.sqrt(4.0 * k)  # typical |S| entry
    assert np.max(np.abs(got - want)) <= 1e-13 * scale


@pytest.mark.parametrize("G", [2, 4, 8])
def test_row_blocks_concatenate_bitwise(G):
    m, n, k = 2048, 1024, 200
    whole = gen_rows(m, n, k, 20240305, 1e-3, 0, m)
    b = m // G
    parts = [gen_rows(m, n, k, 20240305, 1e-3, g * b, b) for g in range(G)]
    assert torch.equal(torch.cat(parts, 0), whole)


def test_cfg5_shape_row_blocks_bitwise():
    # the cfg5 generator at its full width (n = 32768, k = 200): rank 7 of 8's first rows equal
    # the same rows cut from a taller block
    m = n = 32768
    k = 200
    tall = gen_rows(m, n, k, 20240305, 1e-3, 7 * 4096, 256)
    short = gen_rows(m, n, k, 20240305, 1e-3, 7 * 4096 + 64, 64)
    assert torch.equal(tall[64:128], short)
