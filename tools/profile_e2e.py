"""Break the bench e2e step (public API, pinned host planes) into its parts.
Usage: python tools/profile_e2e.py [cfg2]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_19147_b200 import _native, make_plan, qmcur, cur_relative_error  # noqa: E402
from paper_2402_19147_b200.quat import QMatrix, drop_device_copy, to_device  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cfg = bench.CONFIGS[name]
dev = _native.device(0)
m, n, c, r = cfg["m"], cfg["n"], cfg["c"], cfg["r"]
x = dev.empty_q(m, n)
dev.call("qcur_synth_lowrank", m, n, cfg["rank"], cfg["gen_seed"], cfg["noise"], 1 if cfg["relative"] else 0,
         x.data_ptr())
pinned = [torch.empty((m, n), dtype=torch.float64, pin_memory=True) for _ in range(4)]
hp = [p.numpy() for p in pinned]
dev.download_planes(x, m, n, pinned_out=hp)
xh = QMatrix._wrap(*hp)


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, (time.perf_counter() - t0) * 1e3


# raw copies
buf = torch.empty(m * n, dtype=torch.float64, device="cuda")
_, h2d = t(lambda: buf.copy_(pinned[0].view(-1), non_blocking=True))
_, h2d = t(lambda: buf.copy_(pinned[0].view(-1), non_blocking=True))
pg = torch.empty(m * n, dtype=torch.float64)
_, d2h_pg = t(lambda: pg.copy_(buf))
_, d2h_pg = t(lambda: pg.copy_(buf))
_, d2h_pin = t(lambda: pinned[1].view(-1).copy_(buf))
print(f"raw H2D pinned plane {8*m*n/1e6:.0f} MB: {h2d:.2f} ms ({8*m*n/h2d/1e6:.1f} GB/s)")
print(f"raw D2H pageable: {d2h_pg:.2f} ms ({8*m*n/d2h_pg/1e6:.1f} GB/s); pinned: {d2h_pin:.2f} ms")
dev.download_planes(x, m, n, pinned_out=hp)

for it in range(4):
    drop_device_copy(xh)
    _, t_up = t(lambda: to_device(xh, dev))
    plan, t_plan = t(lambda: make_plan(xh, cfg["strategy"], cfg["rank"], cfg["plan_seed"], num_rows=r, num_cols=c))
    f, t_q = t(lambda: qmcur(xh, plan))
    e, t_e = t(lambda: cur_relative_error(xh, f))
    drop_device_copy(xh)
    tot0 = time.perf_counter()
    plan = make_plan(xh, cfg["strategy"], cfg["rank"], cfg["plan_seed"], num_rows=r, num_cols=c)
    f = qmcur(xh, plan)
    e = cur_relative_error(xh, f)
    torch.cuda.synchronize()
    tot = (time.perf_counter() - tot0) * 1e3
    print(f"iter {it}: upload {t_up:.2f}  make_plan {t_plan:.2f}  qmcur {t_q:.2f}  error {t_e:.2f}  "
          f"(sum {t_up + t_plan + t_q + t_e:.2f}); whole step {tot:.2f} ms; err {e:.3e}")

print("--- whole step with marks (no extra syncs)")
for it in range(3):
    drop_device_copy(xh)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = make_plan(xh, cfg["strategy"], cfg["rank"], cfg["plan_seed"], num_rows=r, num_cols=c)
    t1 = time.perf_counter()
    f = qmcur(xh, plan)
    t2 = time.perf_counter()
    e = cur_relative_error(xh, f)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"make_plan {1e3*(t1-t0):.2f} qmcur {1e3*(t2-t1):.2f} error {1e3*(t3-t2):.2f} tail {1e3*(t4-t3):.2f}")
print("--- same, f deleted before the next step")
for it in range(3):
    del f
    drop_device_copy(xh)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = make_plan(xh, cfg["strategy"], cfg["rank"], cfg["plan_seed"], num_rows=r, num_cols=c)
    t1 = time.perf_counter()
    f = qmcur(xh, plan)
    t2 = time.perf_counter()
    e = cur_relative_error(xh, f)
    t3 = time.perf_counter()
    print(f"make_plan {1e3*(t1-t0):.2f} qmcur {1e3*(t2-t1):.2f} error {1e3*(t3-t2):.2f}")
