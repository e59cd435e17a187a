"""Run the INT8 quaternion GEMM at cfg2's Y = X Q_R shape a few times (for ncu launch lists)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2402_19147_b200 import _native

m, n, r = (int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (4000, 4000, 200)))
L = int(sys.argv[4]) if len(sys.argv) > 4 else 15
dev = _native.device()
dx = torch.randn((m, n, 4), dtype=torch.float64, device="cuda")
db = torch.randn((n, r, 4), dtype=torch.float64, device="cuda")
y = dev.empty_q(m, r)
for _ in range(3):
    dev.call("qcur_qgemm_int8", m, r, n, dx.data_ptr(), n, db.data_ptr(), r, y.data_ptr(), r, L)
torch.cuda.synchronize()
print("ok")
