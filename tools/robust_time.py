"""Time of one cfg2 approximation on the robust factorization path (qcur_force_robust: Householder QR +
one-sided Jacobi SVD with the reference's cutoff, the path rank-deficient inputs take) against the
CholeskyQR2 fast path, device-resident, phases per approximation.  One JSON line."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_19147_b200 import _native  # noqa: E402
from paper_2402_19147_b200.cur import DeviceApprox  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = bench.CONFIGS[name]
dev = _native.device(0)
m, n, c, r = cfg["m"], cfg["n"], cfg["c"], cfg["r"]
x = dev.empty_q(m, n)
dev.call("qcur_synth_lowrank", m, n, cfg["rank"], cfg["gen_seed"], cfg["noise"], 1 if cfg["relative"] else 0,
         x.data_ptr())
out = {}
for robust in (0, 1):
    dev.call("qcur_force_robust", robust)
    o = DeviceApprox(m, n, c, r, dev)
    for _ in range(2):
        o.run(x, cfg["strategy"], cfg["plan_seed"])
    o.check()
    torch.cuda.synchronize()
    dev.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        o.run(x, cfg["strategy"], cfg["plan_seed"])
    e1.record()
    torch.cuda.synchronize()
    ph = dev.profile_read()
    dev.profile(False)
    o.check()
    out["robust" if robust else "fast"] = {"ms_per_approx": e0.elapsed_time(e1) / 3,
                                           "phases_ms": {k: v[0] / max(v[1], 1) for k, v in ph.items()},
                                           "rel_err": o.rel_error()}
dev.call("qcur_force_robust", 0)
print(json.dumps({"config": name, **out}))
