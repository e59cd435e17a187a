"""numpy stand-in for rowshard.GpuOps (TEST INFRASTRUCTURE: exercises the
row-block orchestration and its collectives with gloo on CPU).  Same
operations, same shapes, torch CPU tensors; the arithmetic follows the oracle
(and numpy's own summation orders, which the GPU kernels reproduce)."""
from __future__ import annotations

import numpy as np
import torch

import oracle as O
from paper_2402_19147_b200 import _native


def planes(t):
    a = t.numpy()
    return tuple(np.ascontiguousarray(a[..., s]) for s in range(4))


def stack(p):
    return torch.from_numpy(np.ascontiguousarray(np.stack(p, axis=-1)))


def qchol_inv(g):
    """Quaternion Cholesky G = L L^H (lower, real diagonal), returns L^{-1}."""
    q = g[0].shape[0]
    L = [np.zeros((q, q)) for _ in range(4)]
    for j in range(q):
        if j:
            row_j = tuple(p[j:j + 1, :j] for p in L)
            d = g[0][j, j] - O.frob2(row_j)
            lower = tuple(p[j:, :j] for p in L)
            s = O.qmatmul(lower, O.conj_t(row_j))  # (q-j) x 1
        else:
            d = g[0][0, 0]
            s = tuple(np.zeros((q, 1)) for _ in range(4))
        ljj = np.sqrt(d)
        for k in range(4):
            L[k][j:, j] = (g[k][j:, j] - s[k][:, 0]) / ljj
        L[0][j, j] = ljj
        for k in (1, 2, 3):
            L[k][j, j] = 0.0
    # forward substitution for X = L^{-1}
    X = [np.zeros((q, q)) for _ in range(4)]
    for i in range(q):
        X[0][i, i] = 1.0 / L[0][i, i]
        if i:
            row = tuple(p[i:i + 1, :i] for p in L)
            prev = tuple(p[:i, :] for p in X)
            s = O.qmatmul(row, prev)  # 1 x q
            for k in range(4):
                X[k][i, :i] = -s[k][0, :i] / L[0][i, i]
    return tuple(X)


def lh(e):
    q = e[0].shape[0]
    out = [np.tril(p, -1) for p in e]
    out[0] = out[0] + np.diag(0.5 * np.diag(e[0]))
    return tuple(out)


class CpuOps:
    def vec(self, n):
        return torch.empty(int(n), dtype=torch.float64)

    def colsums_seq(self, xb, acc):
        a0, a1, a2, a3 = planes(xb)
        sq = ((a0 * a0 + a1 * a1) + a2 * a2) + a3 * a3
        col = np.zeros(sq.shape[1]) if acc is None else acc.numpy().copy()
        for i in range(sq.shape[0]):  # numpy's sequential axis-0 order
            col = col + sq[i]
        return torch.from_numpy(np.ascontiguousarray(sq.ravel())), torch.from_numpy(col)

    def colsums_chunk(self, xb, c0, c1, acc, colsum, sq):
        a0, a1, a2, a3 = planes(xb[:, c0:c1])
        blk = ((a0 * a0 + a1 * a1) + a2 * a2) + a3 * a3
        col = np.zeros(c1 - c0) if acc is None else acc.numpy().copy()
        for i in range(blk.shape[0]):  # numpy's sequential axis-0 order
            col = col + blk[i]
        colsum[c0:c1] = torch.from_numpy(col)
        n = xb.shape[1]
        sq.view(xb.shape[0], n)[:, c0:c1] = torch.from_numpy(np.ascontiguousarray(blk))

    def pairwise(self, data, nseg, length):
        return torch.from_numpy(np.ascontiguousarray(data.numpy().reshape(nseg, length).sum(axis=1)))

    def div(self, v, denom):
        d = float(denom) if not isinstance(denom, torch.Tensor) else float(denom.reshape(-1)[0])
        return torch.from_numpy(v.numpy() / d)

    def scalar(self, t):
        return float(t.reshape(-1)[0])

    def uniform(self, m, n):
        return torch.full((n,), 1.0 / n, dtype=torch.float64), torch.full((m,), 1.0 / m, dtype=torch.float64)

    def draw(self, probs, count, state):
        g = np.random.default_rng()
        s = g.bit_generator.state
        s["state"]["state"] = (int(state[0]) << 64) | int(state[1])
        s["state"]["inc"] = (int(state[2]) << 64) | int(state[3])
        g.bit_generator.state = s
        idx = O.draw_indices(probs.numpy(), count, g)
        state[:] = _native.state_from_generator(g)
        return torch.from_numpy(idx.astype(np.int64))

    def gather_cols(self, xb, J):
        return xb[:, J, :].contiguous()

    def gather_rows(self, xb, local_rows):
        return xb[local_rows].contiguous()

    def index_tensor(self, values):
        return torch.tensor(list(values), dtype=torch.int64)

    def to_host_int(self, t):
        return t.numpy()

    def gemm(self, A, B, opA=0, opB=0, alpha=1.0, flags=0):
        a, b = planes(A), planes(B)
        if opA:
            a = O.conj_t(a)
        if opB:
            b = O.conj_t(b)
        return stack(tuple(alpha * p for p in O.qmatmul(a, b)))

    def xq(self, xb, QR):
        return self.gemm(xb, QR)

    def chol_inv(self, G):
        return stack(qchol_inv(planes(G)))

    def series(self, G2):
        g = planes(G2)
        q = g[0].shape[0]
        e = (g[0] - np.eye(q),) + g[1:]
        m0 = lh(e)
        p = O.qmatmul(m0, O.conj_t(m0))
        m1 = lh(tuple(x - y for x, y in zip(e, p)))
        p2 = O.qmatmul(m1, m1)
        out = tuple(-x + y for x, y in zip(m1, p2))
        out = (out[0] + np.eye(q),) + out[1:]
        return stack(tuple(np.tril(x) for x in out))

    def series_inv(self, G2):
        g = planes(G2)
        q = g[0].shape[0]
        lo = tuple(np.tril(x) for x in g)  # Hermitian from the lower triangle
        full = tuple(l + (np.tril(l, -1).T * (1 if k == 0 else -1)) for k, l in enumerate(lo))
        e = (full[0] - np.eye(q),) + full[1:]
        e2 = O.qmatmul(e, e)
        s = tuple(-a + b for a, b in zip(e, e2))
        return stack((s[0] + np.eye(q),) + s[1:])

    def kappa(self, G1, F):
        return None

    def fast_failed(self):
        return False

    def factor(self, Z, zh):
        z = planes(Z)
        if zh:
            z = O.conj_t(z)
        zt = stack(z)
        g1 = self.gemm(zt, zt, opA=1)
        x1 = self.chol_inv(g1)
        q1 = self.gemm(zt, x1, opB=1)
        l2i = self.series(self.gemm(q1, q1, opA=1))
        return self.gemm(q1, l2i, opB=1), self.gemm(x1, l2i, opA=1, opB=1)

    def error_stats(self, xb, Cb, U, R, psnr_scale=0.0):
        x = planes(xb)
        rec = O.qmatmul(O.qmatmul(planes(Cb), planes(U)), planes(R))
        d = tuple(a - b for a, b in zip(x, rec))
        return torch.tensor([O.frob2(d), O.frob2(x), O.frob2(d[1:]), 0.0], dtype=torch.float64)

    def stack_stats(self, t):
        return t.reshape(1, 4)
