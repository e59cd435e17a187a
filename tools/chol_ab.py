"""A/B of a factorization variant selected by environment (e.g. QCUR_CHOL_FLAT=0/1): one JSON line per
config with the device-resident time per approximation, the factor phase, and a sha256 of U and of the
error words, so two runs with different settings can be compared for bitwise-identical results."""
import hashlib
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_19147_b200 import _native  # noqa: E402
from paper_2402_19147_b200.cur import DeviceApprox  # noqa: E402

dev = _native.device(0)
for name in sys.argv[1:] or ["cfg1", "cfg2"]:
    cfg = dict(bench.CONFIGS[name.split(":")[0]])
    if ":" in name:
        cfg["c"] = cfg["r"] = int(name.split(":")[1])
    m, n, c, r = cfg["m"], cfg["n"], cfg["c"], cfg["r"]
    x = dev.empty_q(m, n)
    dev.call("qcur_synth_lowrank", m, n, cfg["rank"], cfg["gen_seed"], cfg["noise"], 1 if cfg["relative"] else 0,
             x.data_ptr())
    o = DeviceApprox(m, n, c, r, dev)
    for _ in range(3):
        o.run(x, cfg["strategy"], cfg["plan_seed"])
    o.check()
    torch.cuda.synchronize()
    reps = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        o.run(x, cfg["strategy"], cfg["plan_seed"])
    e1.record()
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1) / reps
    dev.profile(True)
    for _ in range(5):
        o.run(x, cfg["strategy"], cfg["plan_seed"])
    torch.cuda.synchronize()
    ph = dev.profile_read()
    dev.profile(False)
    o.check()
    print(json.dumps({"config": name, "env": {k: v for k, v in os.environ.items() if k.startswith("QCUR_")},
                      "ms_per_approx": total,
                      "phases_ms": {k: round(v[0] / max(v[1], 1), 4) for k, v in ph.items()},
                      "sha_U": hashlib.sha256(o.U.cpu().numpy().tobytes()).hexdigest()[:16],
                      "sha_err": hashlib.sha256(o.err4.cpu().numpy().tobytes()).hexdigest()[:16],
                      "rel_err": o.rel_error()}), flush=True)
