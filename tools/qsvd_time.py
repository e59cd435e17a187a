"""Time qsvd / numerical_rank on the device at a few sizes (CUDA sync around each call)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2402_19147_b200 as q  # noqa: E402

for m, n in [(200, 200), (500, 500), (1000, 1000), (2000, 500), (3000, 600)]:
    g = np.random.default_rng(m + n)
    a = q.QMatrix(*(g.standard_normal((m, n)) for _ in range(4)))
    q.qsvd(a, 10)
    t0 = time.perf_counter()
    res = q.qsvd(a, 10)
    t1 = time.perf_counter()
    sw = q.linalg._last_sweeps
    r = q.numerical_rank(a)
    t2 = time.perf_counter()
    print(f"{m}x{n}: qsvd(k=10) {t1 - t0:.3f} s, numerical_rank {t2 - t1:.3f} s, sigma0 {res.sigma[0]:.6f} rank {r} sweeps {sw}",
          flush=True)

# rank-10 + noise (the bench matrix): the truncated path can stop before full convergence
for m, n in [(500, 500), (1000, 1000)]:
    g = np.random.default_rng(20240229)
    pf = q.QMatrix(*(g.standard_normal((m, 10)) for _ in range(4)))
    qf = q.QMatrix(*(g.standard_normal((10, n)) for _ in range(4)))
    x = q.QMatrix(*(p + 1e-3 * g.standard_normal((m, n)) for p in (pf @ qf).planes))
    for k in (10, None):
        q.qsvd(x, k)
        t0 = time.perf_counter()
        q.qsvd(x, k)
        print(f"lowrank {m}x{n} k={k}: {time.perf_counter() - t0:.3f} s, sweeps {q.linalg._last_sweeps}", flush=True)
