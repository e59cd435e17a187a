"""Throughput with K approximations in flight (K native contexts, K streams, K resident inputs)."""
import sys
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2402_19147_b200 import _native  # noqa: E402
from paper_2402_19147_b200.cur import DeviceApprox  # noqa: E402

cfg = bench.CONFIGS["cfg2"]
m, n, c, r = cfg["m"], cfg["n"], cfg["c"], cfg["r"]
for K in (1, 2, 3):
    devs = [_native.device(0)] + [_native.Device(0) for _ in range(K - 1)]
    xs, outs, sts = [], [], []
    for k in range(K):
        x = devs[k].empty_q(m, n)
        devs[k].call("qcur_synth_lowrank", m, n, cfg["rank"], cfg["gen_seed"] + k, cfg["noise"], 1, x.data_ptr())
        xs.append(x)
        outs.append(DeviceApprox(m, n, c, r, devs[k]))
        sts.append(torch.cuda.Stream())
    torch.cuda.synchronize()
    def step(s):
        k = s % K
        with torch.cuda.stream(sts[k]):
            outs[k].run(xs[k], cfg["strategy"], cfg["plan_seed"], 0.0, graph=True)
    for s in range(3 * K):
        step(s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 60
    e0.record()
    for st in sts:
        st.wait_event(e0)
    for s in range(steps):
        step(s)
    for st in sts:
        torch.cuda.current_stream().wait_stream(st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"in flight {K}: {steps / (ms / 1e3):.1f} approx/s, rel_err {[round(o.rel_error(), 12) for o in outs]}",
          flush=True)
