"""Column-blocked SpMM probe (products-shaped C2 graph, FAST plans): time
A.X at width D as one pass against B passes over column blocks of A whose
X rows fit L2 (each block its own CSR and plan, outputs added), to see
whether L2-resident gathers beat the random-row DRAM gathers of the narrow
transform-first passes (D = 48: 403 MB of X).

    python scripts/colblock_probe.py --widths 48,100 --blocks 1,2,4,8
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2505_04083_b200 import graph, kernels  # noqa: E402


def timed(fn, iters=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    ts = []
    for _ in range(iters):
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--widths", default="48,100")
    ap.add_argument("--blocks", default="1,2,4,8")
    args = ap.parse_args()
    ds = graph.synth_rmat(21, 62_000_000, 100, 47, seed=1)
    pre = graph.preprocess(ds, perm_seed=1)
    del ds
    a = pre.a_even
    rp = a.row_ptr.to(torch.int64)
    ci = a.col_idx.to(torch.int64)
    vals = a.values
    rows = rp.numel() - 1
    row_of = torch.repeat_interleave(torch.arange(rows, device="cuda"), rp[1:] - rp[:-1])
    for nb in [int(b) for b in args.blocks.split(",")]:
        subs = []
        for b in range(nb):
            c0, c1 = a.cols * b // nb, a.cols * (b + 1) // nb
            sel = (ci >= c0) & (ci < c1)
            r = row_of[sel]
            cnt = torch.bincount(r, minlength=rows)
            srp = torch.zeros(rows + 1, dtype=torch.int64, device="cuda")
            srp[1:] = torch.cumsum(cnt, 0)
            sub = kernels.DeviceCsr(rows, a.cols, srp.contiguous(), ci[sel].to(torch.int32).contiguous(),
                                    vals[sel].contiguous())
            subs.append((sub, kernels.SpmmPlan(sub, 0, mode=kernels.PK_MODE_FAST)))
        for d in [int(w) for w in args.widths.split(",")]:
            x = torch.rand(a.cols, d, device="cuda")
            ys = [torch.empty(rows, d, device="cuda") for _ in range(min(nb, 2))]
            def run():
                for i, (sub, plan) in enumerate(subs):
                    kernels.spmm(sub, x, out=ys[i % len(ys)], plan=plan)
                    if i:
                        ys[0].add_(ys[1])
            ms = timed(run)
            print(json.dumps({"d": d, "blocks": nb, "ms": round(ms, 3)}), flush=True)
        del subs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
