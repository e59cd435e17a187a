import sys, torch
sys.path.insert(0, ".")
from paper_2402_19147_b200 import _native
dev = _native.device()
for (K, q) in [(10, 3), (64, 8), (4000, 200)]:
    a = torch.randn((K, q, 4), dtype=torch.float64, device="cuda")
    c = torch.zeros((q, q, 4), dtype=torch.float64, device="cuda")
    try:
        dev.call("qcur_qgemm_herm_int8", q, q, K, a.data_ptr(), q, a.data_ptr(), q, c.data_ptr(), q)
        torch.cuda.synchronize()
        # reference
        A = a.cpu()
        w, x, y, z = A[..., 0], A[..., 1], A[..., 2], A[..., 3]
        G0 = w.T @ w + x.T @ x + y.T @ y + z.T @ z
        print(K, q, "ok", float((c.cpu()[..., 0] - G0).abs().max()), flush=True)
    except Exception as e:
        print(K, q, "ERR", e, flush=True)
        break
