"""Minimal SpMM driver for ncu captures: build the products-shaped graph on
the GPU, then run the planned (hub-split) SpMM `iters` times at width d.

    python scripts/spmm_kernel.py --scale 21 --edges 62000000 --d 256 --iters 3
"""

import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_04083_b200 import graph, kernels  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=21)
    ap.add_argument("--edges", type=int, default=62_000_000)
    ap.add_argument("--d", type=int, default=256)
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    pre = graph.preprocess(graph.synth_rmat(args.scale, args.edges, 16, 4, seed=1), 1)
    a = pre.a_even
    x = torch.rand(a.cols, args.d, device="cuda")
    y = torch.empty(a.rows, args.d, device="cuda")
    plan = a.plan()
    for _ in range(args.iters):
        kernels.spmm(a, x, out=y, plan=plan)
    torch.cuda.synchronize()
    print("spmm_kernel: ok", a.rows, a.nnz, args.d, plan.info())


if __name__ == "__main__":
    main()
