import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04083_b200 import kernels as k
a = torch.randn(128, 32, device="cuda"); b = torch.randn(32, 16, device="cuda")
for (ta, tb, A, B) in [(False, False, a, b), (False, True, a, b.t().contiguous()), (True, False, a.t().contiguous(), b.t().contiguous().t().contiguous())]:
    out = torch.full((128, 16), float("nan"), device="cuda")
    if ta:
        A = torch.randn(32, 128, device="cuda"); B = torch.randn(32, 16, device="cuda")
        want = A.t() @ B
    elif tb:
        want = A @ B.t()
    else:
        want = A @ B
    k.gemm(A, B, ta, tb, mode=k.PK_MODE_FAST, out=out)
    torch.cuda.synchronize()
    print(ta, tb, "nan:", torch.isnan(out).sum().item(), "zeros:", (out == 0).sum().item(), "err:", (out - want).abs().max().item())
    print(out[0, :8].tolist(), want[0, :8].tolist())
