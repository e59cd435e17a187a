"""Does replaying one cfg2 approximation as a CUDA graph beat stream launches? (diagnostics)"""
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
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(3):
        out.run(x, "length", 1)
torch.cuda.synchronize()


def timed(fn, k=20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


print("stream launches: %.3f ms" % timed(lambda: out.run(x, "length", 1)))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    out.run(x, "length", 1)
torch.cuda.synchronize()
print("graph replay:    %.3f ms" % timed(g.replay))
out.check()
print("rel_err", out.rel_error())
