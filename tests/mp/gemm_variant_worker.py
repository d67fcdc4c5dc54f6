"""Computes a fixed set of FAST-mode GEMMs (NN / NT / TN, tile counts that
leave phantom tiles for 2- and 4-CTA clusters) and saves them to an npz, so
tests can compare environment variants (PK_TC_CLUSTER, PK_TC_TMA) of the
same process-level settings bit for bit."""
import sys

import numpy as np
import torch

sys.path.insert(0, sys.argv[2])
from paper_2505_04083_b200 import kernels as k  # noqa: E402

SHAPES = [("NN", 19067, 256, 100), ("NN", 4737, 47, 256), ("NT", 4737, 256, 256),
          ("NT", 19067, 100, 47), ("NN", 300, 256, 64), ("TN", 256, 47, 70001)]


def main():
    out = {}
    for i, (form, m, n, kk) in enumerate(SHAPES):
        ta, tb = form[0] == "T", form[1] == "T"
        g = torch.Generator().manual_seed(i)
        a = torch.randn((kk, m) if ta else (m, kk), generator=g).cuda()
        b = torch.randn((n, kk) if tb else (kk, n), generator=g).cuda()
        out[f"c{i}"] = k.gemm(a, b, ta, tb, mode=k.PK_MODE_FAST).cpu().numpy()
        out[f"r{i}"] = k.gemm(a, b, ta, tb, mode=k.PK_MODE_FAST, relu=True).cpu().numpy()
    np.savez(sys.argv[1], **out)


if __name__ == "__main__":
    main()
