"""What the host delivery costs in the drop-in qmcur at cfg2: qcur_qmcur_ex (device outputs) vs
qcur_qmcur_host (C, R, indices streamed out while U is computed, U at the end), same resident input,
same plan; wall time per call after warm-up (both synchronise at the end)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_19147_b200 import _native  # noqa: E402

cfg = bench.CONFIGS["cfg2"]
dev = _native.device(0)
m, n, c, r = cfg["m"], cfg["n"], cfg["c"], cfg["r"]
x = dev.empty_q(m, n)
dev.call("qcur_synth_lowrank", m, n, cfg["rank"], cfg["gen_seed"], cfg["noise"], 1, x.data_ptr())
col, row = dev.empty(n), dev.empty(m)
dev.call("qcur_length_distributions", x.data_ptr(), m, n, col.data_ptr(), row.data_ptr())
state = _native.state_from_seed(cfg["plan_seed"])
J, I = dev.empty(c, dtype=torch.int64), dev.empty(r, dtype=torch.int64)
C, U, R = dev.empty_q(m, c), dev.empty_q(c, r), dev.empty_q(r, n)
hj, hi = dev.pinned_vec(c), dev.pinned_vec(r)
hc, hu, hr = dev.pinned_planes(m, c), dev.pinned_planes(c, r), dev.pinned_planes(r, n)
ptrs = [_native._c_dp4(*(p.ctypes.data for p in planes)) for planes in (hc, hu, hr)]


def ex():
    dev.call("qcur_qmcur_ex", x.data_ptr(), m, n, col.data_ptr(), row.data_ptr(), c, r,
             state.ctypes.data_as(_native._u64p), 0, J.data_ptr(), I.data_ptr(), C.data_ptr(), U.data_ptr(), R.data_ptr())
    dev.synchronize()


def host():
    dev.call("qcur_qmcur_host", x.data_ptr(), m, n, col.data_ptr(), row.data_ptr(), c, r,
             state.ctypes.data_as(_native._u64p), 0, J.data_ptr(), I.data_ptr(), C.data_ptr(), U.data_ptr(),
             R.data_ptr(), hj.ctypes.data, hi.ctypes.data, *ptrs)


for name, fn in (("qmcur_ex", ex), ("qmcur_host", host), ("qmcur_ex", ex), ("qmcur_host", host)):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(10):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    print(f"{name}: median {1e3 * np.median(ts):.3f} ms, min {1e3 * min(ts):.3f} ms")
dev.profile(True)
for _ in range(5):
    host()
print("host phases:", {k: round(v[0] / v[1], 4) for k, v in dev.profile_read().items()})
dev.profile(False)
