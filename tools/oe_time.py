"""Time the fused error ||X - C U R|| at cfg2 shapes on both engines (CUDA events), for A/B and ncu runs."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2402_19147_b200 import _native

m, n, c, r = 4000, 4000, 200, 200
dev = _native.device()
x = torch.randn((m, n, 4), dtype=torch.float64, device="cuda")
C = x[:, :c].contiguous()
R = x[:r, :].contiguous()
U = torch.randn((c, r, 4), dtype=torch.float64, device="cuda") * 1e-3
out = dev.empty(4)
for mode in (2, 1):
    dev.call("qcur_set_gemm_mode", mode)
    def call():
        dev.call("qcur_cur_error", x.data_ptr(), m, n, C.data_ptr(), c, U.data_ptr(), R.data_ptr(), r, 0.0, out.data_ptr())
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        call()
    e1.record()
    torch.cuda.synchronize()
    print("mode", mode, "ms", e0.elapsed_time(e1) / 10, "stats", out.cpu().numpy())
