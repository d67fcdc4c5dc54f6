"""Per-role barrier-wait breakdown of the tcgen05 GEMM (library built with
-DPK_TC_PROF, see scripts/tc_prof.sh) for the epoch's GEMM shapes."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04083_b200 import _capi, kernels as k  # noqa: E402

lib = _capi.lib()
lib.pk_tc_prof.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
N = 2_097_152
shapes = [("NN", N, 256, 100), ("TN", 100, 256, N), ("NT", N, 100, 256), ("NN", N, 256, 256),
          ("TN", 256, 256, N), ("NN", N, 47, 256), ("TN", 256, 47, N), ("NT", N, 256, 47)]
for form, m, n, kk in shapes:
    ta, tb = form[0] == "T", form[1] == "T"
    # padded leading dimensions like the engine's buffers (16-B rows)
    def mat(r, c):
        return torch.rand((r, (c + 3) // 4 * 4), device="cuda")[:, :c]
    a = mat(kk, m) if ta else mat(m, kk)
    b = mat(n, kk) if tb else mat(kk, n)
    out = torch.empty(m, n, device="cuda")
    k.gemm(a, b, ta, tb, mode=k.PK_MODE_FAST, out=out)
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 8)()
    lib.pk_tc_prof(buf, 1)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    k.gemm(a, b, ta, tb, mode=k.PK_MODE_FAST, out=out)
    e1.record()
    torch.cuda.synchronize()
    lib.pk_tc_prof(buf, 1)
    v = list(buf)
    ctas = 148
    kern = v[5] / ctas
    stages = v[7] / ctas
    def pct(x):
        return f"{100 * x / kern:5.1f}%" if kern else "-"
    print(f"{form} m={m} n={n} k={kk}: {e0.elapsed_time(e1):.3f} ms, stages/CTA {stages:.0f}, "
          f"cyc/stage {kern / max(stages, 1):.0f} | waits per CTA: producer/empty {pct(v[0] / ctas)}"
          f" conv/raw {pct(v[1] / ctas / int(os.environ.get("CONV", "7")))} mma/raw {pct(v[2] / ctas)}"
          f" mma/full {pct(v[6] / ctas)} mma/tempty {pct(v[3] / ctas)}"
          f" epi/tfull {pct(v[4] / ctas / 4)}", flush=True)
