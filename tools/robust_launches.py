"""One cfg2 approximation on the forced robust path inside cudaProfilerStart/Stop (for the ncu launch list)."""
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
dev.call("qcur_force_robust", 1)
o = DeviceApprox(m, n, c, r, dev)
o.run(x, cfg["strategy"], cfg["plan_seed"])
torch.cuda.synchronize()
torch.cuda.profiler.start()
o.run(x, cfg["strategy"], cfg["plan_seed"])
torch.cuda.synchronize()
torch.cuda.profiler.stop()
o.check()
print("rel_err", o.rel_error())
