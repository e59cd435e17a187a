"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck): the smoke case, a
cfg1-shaped approximation on both engines (FP64 DMMA and INT8 tcgen05, incl. the 2-CTA cluster
error kernel and the 16-CTA cluster Cholesky), a batched call and a draw with a dominant weight."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import numpy as np  # noqa: E402

import paper_2402_19147_b200 as q  # noqa: E402
from paper_2402_19147_b200 import _native  # noqa: E402
from paper_2402_19147_b200.cur import DeviceBatch  # noqa: E402
from paper_2402_19147_b200.quat import to_device  # noqa: E402
from helpers import lowrank  # noqa: E402

dev = _native.device()
x = lowrank(96, 80, 6, seed=11, noise=1e-3)
plan = q.make_plan(x, "length", 6, 5, num_rows=20, num_cols=16)
print("smoke", q.cur_relative_error(x, q.qmcur(x, plan)))
x = lowrank(1000, 1000, 10, seed=2024, noise=1e-3)
for mode in (1, 2):
    dev.call("qcur_set_gemm_mode", mode)
    plan = q.make_plan(x, "length", 10, 0, num_rows=40, num_cols=40)
    print("cfg1 mode", mode, q.cur_relative_error(x, q.qmcur(x, plan)))
dev.call("qcur_set_gemm_mode", 0)
xs = [to_device(lowrank(200, 180, 5, seed=s, noise=1e-3), dev) for s in (1, 2)]
b = DeviceBatch(2, 200, 180, 16, 16, dev, lanes=2)
b.run(xs, "uniform", [3, 4])
b.check()
print("batch", b.rel_errors())
p = np.random.default_rng(0).random(64)
p[5] *= 1e13
p /= p.sum()
print("draw", q.draw_indices(p, 40, 3)[:5])
dev.synchronize()
print("done")
