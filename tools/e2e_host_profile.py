"""Host-side time inside the drop-in calls (make_plan / qmcur / cur_relative_error) at cfg2: cProfile of a
few e2e steps after warm-up, to separate Python/ctypes overhead from the device-bound ABI calls."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_19147_b200 import _native, make_plan, qmcur, cur_relative_error  # noqa: E402
from paper_2402_19147_b200.quat import QMatrix, drop_device_copy  # noqa: E402

cfg = bench.CONFIGS["cfg2"]
dev = _native.device(0)
m, n, c, r = cfg["m"], cfg["n"], cfg["c"], cfg["r"]
x = dev.empty_q(m, n)
dev.call("qcur_synth_lowrank", m, n, cfg["rank"], cfg["gen_seed"], cfg["noise"], 1, x.data_ptr())
pinned = [torch.empty((m, n), dtype=torch.float64, pin_memory=True) for _ in range(4)]
hp = [p.numpy() for p in pinned]
dev.download_planes(x, m, n, pinned_out=hp)
xh = QMatrix._wrap(*hp)


def step():
    drop_device_copy(xh)
    plan = make_plan(xh, cfg["strategy"], cfg["rank"], cfg["plan_seed"], num_rows=r, num_cols=c)
    f = qmcur(xh, plan)
    return cur_relative_error(xh, f)


for _ in range(3):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
