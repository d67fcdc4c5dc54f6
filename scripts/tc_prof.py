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
    a = torch.rand((kk, m) if ta else (m, kk), device="cuda")
    b = torch.rand((n, kk) if tb else (kk, n), device="cuda")
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
          f" conv/raw {pct(v[1] / ctas / 128)} mma/raw {pct(v[2] / ctas / 32)}"
          f" mma/full {pct(v[6] / ctas / 32)} mma/tempty {pct(v[3] / ctas / 32)}"
          f" epi/tfull {pct(v[4] / ctas / 128)}", flush=True)
