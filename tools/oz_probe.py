"""Probe the INT8 (Ozaki II) quaternion GEMM against the FP64 DMMA GEMM and an
extended-precision host product: accuracy on small shapes, timing at cfg2's Y = X Q_R."""
from __future__ import annotations

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2402_19147_b200 import _native  # noqa: E402

SIGNS = {  # (x b)_t = sum_s sign * x_s b_{s^t}
    0: (1, -1, -1, -1), 1: (1, 1, 1, -1), 2: (1, -1, 1, 1), 3: (1, 1, -1, 1)}


def ref_product(x, b):
    """x: (m, n, 4), b: (n, r, 4) -> (m, r, 4) in long double."""
    xl = x.astype(np.longdouble)
    bl = b.astype(np.longdouble)
    m, r = x.shape[0], b.shape[1]
    y = np.zeros((m, r, 4), dtype=np.longdouble)
    for t in range(4):
        for s in range(4):
            y[:, :, t] += SIGNS[t][s] * (xl[:, :, s] @ bl[:, :, s ^ t])
    return y


def run(dev, m, n, r, nmod, seed=0, scale_rows=False):
    g = np.random.default_rng(seed)
    x = g.standard_normal((m, n, 4))
    if scale_rows:
        x *= np.exp(g.uniform(-20, 20, size=(m, 1, 1)))
    b = g.standard_normal((n, r, 4))
    dx = torch.from_numpy(x).cuda()
    db = torch.from_numpy(b).cuda()
    y8 = dev.empty_q(m, r)
    yd = dev.empty_q(m, r)
    dev.call("qcur_qgemm_int8", m, r, n, dx.data_ptr(), n, db.data_ptr(), r, y8.data_ptr(), r, nmod)
    dev.call("qcur_qgemm", 0, 0, m, r, n, 1.0, dx.data_ptr(), n, db.data_ptr(), r, 0.0, yd.data_ptr(), r)
    torch.cuda.synchronize()
    ref = ref_product(x, b)
    # error relative to the natural scale |x_i| |b_j| (row / column norms)
    scale = np.sqrt((x ** 2).sum(axis=(1, 2)))[:, None] * np.sqrt((b ** 2).sum(axis=(0, 2)))[None, :]
    e8 = np.abs(y8.cpu().numpy() - ref).max(axis=2) / scale
    ed = np.abs(yd.cpu().numpy() - ref).max(axis=2) / scale
    print(f"m={m} n={n} r={r} L={nmod} rows_scaled={scale_rows}: int8 max {float(e8.max()):.3e} mean "
          f"{float(e8.mean()):.3e} | dmma max {float(ed.max()):.3e} mean {float(ed.mean()):.3e}", flush=True)
    return float(e8.max()), float(ed.max())


def timing(dev, m, n, r, nmod, reps=20):
    dx = torch.randn((m, n, 4), dtype=torch.float64, device="cuda")
    db = torch.randn((n, r, 4), dtype=torch.float64, device="cuda")
    y = dev.empty_q(m, r)
    out = {}
    for name in ("int8", "dmma"):
        def call():
            if name == "int8":
                dev.call("qcur_qgemm_int8", m, r, n, dx.data_ptr(), n, db.data_ptr(), r, y.data_ptr(), r, nmod)
            else:
                dev.call("qcur_qgemm", 0, 0, m, r, n, 1.0, dx.data_ptr(), n, db.data_ptr(), r, 0.0, y.data_ptr(), r)
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            call()
        e1.record()
        torch.cuda.synchronize()
        out[name] = e0.elapsed_time(e1) / reps
    flop = 32.0 * m * n * r
    print(f"timing m={m} n={n} r={r} L={nmod}: int8 {out['int8']:.3f} ms ({flop / out['int8'] / 1e9:.1f} TF/s fp64-eq)"
          f" | dmma {out['dmma']:.3f} ms ({flop / out['dmma'] / 1e9:.1f} TF/s)", flush=True)


def main():
    dev = _native.device()
    for (m, n, r) in [(8, 8, 4), (300, 500, 40), (129, 257, 52), (1000, 1000, 40)]:
        for L in (14, 15):
            run(dev, m, n, r, L)
    run(dev, 300, 500, 40, 15, scale_rows=True)
    for L in (14, 15):
        timing(dev, 4000, 4000, 200, L)
    timing(dev, 1000, 1000, 40, 15)
    timing(dev, 2048, 2048, 128, 15)


if __name__ == "__main__":
    main()
