"""Repeat the CholeskyQR2 steps of pinv(C) at cfg2 and report any run-to-run bit
differences (diagnostics for intermittent robust-path fallbacks)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2402_19147_b200 import _native  # noqa: E402
from paper_2402_19147_b200.cur import DeviceApprox  # noqa: E402

cfg = bench.CONFIGS["cfg2"]
m, n, c = cfg["m"], cfg["n"], cfg["c"]
dev = _native.device(0)
x = dev.empty_q(m, n)
dev.call("qcur_synth_lowrank", m, n, cfg["rank"], cfg["gen_seed"], cfg["noise"], 1, x.data_ptr())
out = DeviceApprox(m, n, c, cfg["r"], dev)
out.run(x, "length", 1)
out.check()
C = dev.empty_q(m, c)
dev.call("qcur_gather_cols", x.data_ptr(), m, n, out.J.data_ptr(), c, C.data_ptr())
lower = torch.tril(torch.ones(c, c, dtype=torch.bool, device="cuda"))


def step():
    G1 = torch.zeros(c, c, 4, dtype=torch.float64, device="cuda")
    dev.call("qcur_qgemm_ex", 1, 0, c, c, m, 1.0, C.data_ptr(), c, C.data_ptr(), c, 0.0, G1.data_ptr(), c, 2)
    L1i = dev.empty_q(c, c)
    dev.call("qcur_chol_inv", G1.data_ptr(), c, L1i.data_ptr())
    Q1 = dev.empty_q(m, c)
    dev.call("qcur_qgemm_ex", 0, 1, m, c, c, 1.0, C.data_ptr(), c, L1i.data_ptr(), c, 0.0, Q1.data_ptr(), c, 1)
    G2 = torch.zeros(c, c, 4, dtype=torch.float64, device="cuda")
    dev.call("qcur_qgemm_ex", 1, 0, c, c, m, 1.0, Q1.data_ptr(), c, Q1.data_ptr(), c, 0.0, G2.data_ptr(), c, 2)
    torch.cuda.synchronize()
    return G1 * lower[..., None], L1i, Q1, G2 * lower[..., None]


ref = step()
eye = torch.zeros(c, c, 4, dtype=torch.float64, device="cuda")
eye[torch.arange(c), torch.arange(c), 0] = 1.0
print("G2-I max", float((ref[3] - eye * lower[..., None]).abs().max()))
bad = {}
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 40):
    cur = step()
    for name, a, b in zip(("G1", "L1i", "Q1", "G2"), ref, cur):
        d = (a != b).sum().item()
        if d:
            bad.setdefault(name, []).append((i, d, float((a - b).abs().max())))
print({k: v[:5] for k, v in bad.items()}, {k: len(v) for k, v in bad.items()})
