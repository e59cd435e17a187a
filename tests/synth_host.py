"""Host (numpy) restatement of the on-device synthetic generator (csrc/k_synth.cu).

Test infrastructure: lets any block of a generated BASELINE matrix (cfg5 is
34 GB and exists only on the device, in row blocks) be regenerated on the host
and spot-checked.  Philox4x32-10 keyed by the 64-bit seed, counter = (pair
index, stream), two 53-bit uniforms per counter and Box-Muller, exactly as
`normal_pair` in k_synth.cu.  The integer stream and the uniforms are
bit-exact; log / sin / cos come from the host libm, so the normals agree with
the device's to a few ulps (the device uses CUDA's log and sincospi)."""
from __future__ import annotations

import numpy as np

_M32 = np.uint64(0xFFFFFFFF)
_M53 = np.uint64((1 << 53) - 1)


def philox4x32_10(c0, c1, c2, c3, seed: int):
    """Ten Philox rounds on uint64 arrays holding 32-bit counter words."""
    k0, k1 = seed & 0xFFFFFFFF, (seed >> 32) & 0xFFFFFFFF
    m0, m1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    for _ in range(10):
        p0 = m0 * c0
        p1 = m1 * c2
        hi0, lo0 = p0 >> np.uint64(32), p0 & _M32
        hi1, lo1 = p1 >> np.uint64(32), p1 & _M32
        c0, c1, c2, c3 = hi1 ^ c1 ^ np.uint64(k0), lo1, hi0 ^ c3 ^ np.uint64(k1), lo0
        k0 = (k0 + 0x9E3779B9) & 0xFFFFFFFF
        k1 = (k1 + 0xBB67AE85) & 0xFFFFFFFF
    return c0, c1, c2, c3


def uniforms(seed: int, stream: int, pairs: np.ndarray):
    """(u1 in (0, 1], u2 in [0, 1)) of counters `pairs` of `stream` (bit-exact with the device)."""
    idx = pairs.astype(np.uint64)
    c0, c1 = idx & _M32, idx >> np.uint64(32)
    c2 = np.full_like(idx, stream & 0xFFFFFFFF)
    c3 = np.full_like(idx, (stream >> 32) & 0xFFFFFFFF)
    c0, c1, c2, c3 = philox4x32_10(c0, c1, c2, c3, seed)
    a = ((c0 << np.uint64(21)) ^ c1) & _M53
    b = ((c2 << np.uint64(21)) ^ c3) & _M53
    u1 = (a.astype(np.float64) + 1.0) * (1.0 / 9007199254740992.0)
    u2 = b.astype(np.float64) * (1.0 / 9007199254740992.0)
    return u1, u2


def normals(seed: int, stream: int, offset: int, count: int, scale: float = 1.0) -> np.ndarray:
    """Elements [offset, offset + count) of a generator stream (offset even), as k_normal_fill writes them."""
    assert offset % 2 == 0
    p0 = offset // 2
    npairs = (count + 1) // 2
    u1, u2 = uniforms(seed, stream, np.arange(p0, p0 + npairs, dtype=np.uint64))
    rad = np.sqrt(-2.0 * np.log(u1))
    ang = np.pi * (2.0 * u2)
    z = np.empty(2 * npairs)
    z[0::2] = rad * np.cos(ang)
    z[1::2] = rad * np.sin(ang)
    return scale * z[:count]


def _qmul_conj(p, q):
    """S = P Q^H for interleaved (.., 4) quaternion arrays P (a x k), Q (b x k)."""
    a0, a1, a2, a3 = (p[:, :, t] for t in range(4))
    b0, b1, b2, b3 = (q[:, :, t].T for t in range(4))
    b1, b2, b3 = -b1, -b2, -b3  # conj
    s = np.empty((p.shape[0], q.shape[0], 4))
    s[:, :, 0] = a0 @ b0 - a1 @ b1 - a2 @ b2 - a3 @ b3
    s[:, :, 1] = a0 @ b1 + a1 @ b0 + a2 @ b3 - a3 @ b2
    s[:, :, 2] = a0 @ b2 - a1 @ b3 + a2 @ b0 + a3 @ b1
    s[:, :, 3] = a0 @ b3 + a1 @ b2 - a2 @ b1 + a3 @ b0
    return s


def lowrank_rows(m: int, n: int, k: int, seed: int, noise: float, row0: int, rows: int, cols=None) -> np.ndarray:
    """Rows [row0, row0 + rows) (optionally columns `cols`) of qcur_synth_lowrank_rows' matrix, interleaved
    (rows x n x 4): P Q^H + sigma Z with sigma = noise * sqrt(4k)."""
    p = normals(seed, 1, row0 * k * 4, rows * k * 4).reshape(rows, k, 4)
    q = normals(seed, 2, 0, n * k * 4).reshape(n, k, 4)
    x = _qmul_conj(p, q)
    if noise > 0.0:
        x = x + (noise * np.sqrt(4.0 * k)) * normals(seed, 3, row0 * n * 4, rows * n * 4).reshape(rows, n, 4)
    return x if cols is None else x[:, cols, :]
