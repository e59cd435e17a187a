"""Accuracy of the fused relative error on each engine against the extended-precision value of the
same factors (x87 long double), on the blocked-path case and lower-noise variants (smaller errors
amplify any evaluation rounding).  Prints one JSON line per (case, engine)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]
import paper_2402_19147_b200 as q  # noqa: E402
from paper_2402_19147_b200 import _native  # noqa: E402
from helpers import exact_rel_error, lowrank  # noqa: E402

cases = [(1300, 1100, 60, 1e-3, 330, 320), (1300, 1100, 60, 1e-5, 330, 320), (2000, 2000, 40, 1e-4, 200, 200)]
dev = _native.device()
for (m, n, k, noise, r, c) in cases:
    x = lowrank(m, n, k, seed=8, noise=noise)
    plan = q.make_plan(x, "length", k, 8, num_rows=r, num_cols=c)
    for mode in (1, 2):
        dev.call("qcur_set_gemm_mode", mode)
        f = q.qmcur(x, plan)
        got = q.cur_relative_error(x, f)
        ex = exact_rel_error(tuple(x.planes), tuple(f.c.planes), tuple(f.u.planes), tuple(f.r.planes))
        print(json.dumps({"m": m, "n": n, "k": k, "noise": noise, "r": r, "c": c,
                          "engine": {1: "fp64", 2: "int8"}[mode], "err": got, "exact": ex,
                          "rel_dev": abs(got - ex) / ex}), flush=True)
    dev.call("qcur_set_gemm_mode", 0)
