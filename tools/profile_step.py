"""Run one cfg2 QMCUR approximation inside cudaProfilerStart/Stop (for ncu
--profile-from-start off).  Usage: python tools/profile_step.py [cfg2|cfg1]"""
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
m, n = cfg["m"], cfg["n"]
x = dev.empty_q(m, n)
dev.call("qcur_synth_lowrank", m, n, cfg["rank"], cfg["gen_seed"], cfg["noise"], 1 if cfg["relative"] else 0,
         x.data_ptr())
out = DeviceApprox(m, n, cfg["c"], cfg["r"], dev)
for _ in range(3):
    out.run(x, cfg["strategy"], cfg["plan_seed"])
out.check()
torch.cuda.synchronize()
torch.cuda.profiler.start()
out.run(x, cfg["strategy"], cfg["plan_seed"])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
out.check()
print("rel_err", out.rel_error())
