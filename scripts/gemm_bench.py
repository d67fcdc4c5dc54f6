"""Times the dense transforms of one products-shaped epoch (1x1x1, N=2,097,152,
dims 100-256-256-47) through pk_gemm_f32 FAST (tcgen05 3xTF32) and PARITY,
beside cuBLAS fp32 (torch.matmul, TF32 off) as a vendor comparison point.
Reports ms and algorithmic GB/s (4*(MK+KN+MN) bytes) per shape."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04083_b200 import kernels as k

torch.backends.cuda.matmul.allow_tf32 = False
N = 2_097_152
dims = [100, 256, 256, 47]
shapes = []
for l in range(3):
    din, dout = dims[l], dims[l + 1]
    shapes.append(("NN", N, dout, din))      # Q = H W
    shapes.append(("TN", din, dout, N))      # dW = H^T dQ
    shapes.append(("NT", N, din, dout))      # dH = dQ W^T

def timeit(fn, it=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(it):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return min(ts)

args = [a for a in sys.argv[1:] if not a.startswith("--only=")]
only = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--only=")]
modes = args or ["fast", "cublas"]
if only:  # e.g. --only=NN,2097152,256,256
    f, m_, n_, k_ = only[0].split(",")
    shapes = [(f, int(m_), int(n_), int(k_))]
tot = {m: 0.0 for m in modes}
for form, m, n, kk in shapes:
    ta, tb = form[0] == "T", form[1] == "T"
    a = torch.rand((kk, m) if ta else (m, kk), device="cuda")
    b = torch.rand((n, kk) if tb else (kk, n), device="cuda")
    out = torch.empty(m, n, device="cuda")
    byts = 4 * (m * kk + kk * n + m * n)
    row = dict(form=form, m=m, n=n, k=kk)
    for mode in modes:
        if mode == "cublas":
            A = a.t() if ta else a
            B = b.t() if tb else b
            fn = lambda: torch.matmul(A, B, out=out)
        else:
            md = k.PK_MODE_FAST if mode == "fast" else k.PK_MODE_PARITY
            fn = lambda: k.gemm(a, b, ta, tb, mode=md, out=out)
        ms = timeit(fn)
        tot[mode] += ms
        row[mode + "_ms"] = round(ms, 4)
        row[mode + "_gbs"] = round(byts / ms / 1e6, 1)
        row[mode + "_tflops"] = round(2 * m * n * kk / ms / 1e9, 1)
    print(json.dumps(row), flush=True)
print(json.dumps({"total_ms": tot}))
