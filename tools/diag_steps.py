"""Per-step phase times of repeated cfg2 approximations (diagnostics)."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2402_19147_b200 import _native  # noqa: E402
from paper_2402_19147_b200.cur import DeviceApprox  # noqa: E402

cfg = bench.CONFIGS["cfg2"]
m, n = cfg["m"], cfg["n"]
dev = _native.device(0)
x = dev.empty_q(m, n)
dev.call("qcur_synth_lowrank", m, n, cfg["rank"], cfg["gen_seed"], cfg["noise"], 1, x.data_ptr())
out = DeviceApprox(m, n, cfg["c"], cfg["r"], dev)
for _ in range(3):
    out.run(x, "length", 1)
torch.cuda.synchronize()
dev.profile(True)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    t0 = time.perf_counter()
    out.run(x, "length", 1)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    out.check()
    info = dev.info()
    ph = dev.profile_read()
    slow = {k: round(v[0], 2) for k, v in ph.items() if v[0] > 5.0}
    print(f"step {i}: {ms:.2f} ms info={info}", slow if ms > 20 else "")
