"""SpMM throughput probe on a products-shaped RMAT graph (C2: scale 21,
62M edges) generated and preprocessed on the GPU. Prints algorithmic GB/s
per width with and without the hub plan, and the shard-builder timings.

    python scripts/spmm_probe.py [--scale 21] [--edges 62000000]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_04083_b200 import graph, kernels  # noqa: E402


def timed(fn, iters=5, warmup=2):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ts = []
    for _ in range(iters):
        ev[0].record()
        fn()
        ev[1].record()
        torch.cuda.synchronize()
        ts.append(ev[0].elapsed_time(ev[1]))
    return float(np.median(ts)), float(np.min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=21)
    ap.add_argument("--edges", type=int, default=62_000_000)
    ap.add_argument("--widths", default="50,100,128,256")
    ap.add_argument("--thresholds", default="0")
    ap.add_argument("--fast", action="store_true", help="FAST plans (segmented hub rows)")
    args = ap.parse_args()
    t0 = time.time()
    ds = graph.synth_rmat(args.scale, args.edges, 100, 47, seed=1)
    torch.cuda.synchronize()
    t1 = time.time()
    pre = graph.preprocess(ds, perm_seed=1)
    torch.cuda.synchronize()
    t2 = time.time()
    a = pre.a_even
    rp = a.row_ptr.cpu().numpy()
    lens = np.diff(rp)
    out = dict(n=a.rows, nnz=a.nnz, synth_s=t1 - t0, preprocess_s=t2 - t1,
               row_len=dict(mean=float(lens.mean()), median=float(np.median(lens)),
                            p99=float(np.percentile(lens, 99)), max=int(lens.max()),
                            rows_ge_4096=int((lens >= 4096).sum()),
                            nnz_share_ge_4096=float(lens[lens >= 4096].sum() / lens.sum())))
    t3 = time.time()
    at = graph.csr_transpose(a)
    torch.cuda.synchronize()
    out["transpose_s"] = time.time() - t3
    del at
    res = []
    for d in [int(w) for w in args.widths.split(",")]:
        x = torch.rand(a.cols, d, device="cuda")
        y = torch.empty(a.rows, d, device="cuda")
        byts = 8 * a.nnz + 8 * (a.rows + 1) + 4 * a.nnz * d + 4 * a.rows * d
        for t in [int(v) for v in args.thresholds.split(",")]:
            plan = (kernels.SpmmPlan(a, t, mode=kernels.PK_MODE_FAST) if args.fast
                    else a.plan(t))
            planned = timed(lambda: kernels.spmm(a, x, out=y, plan=plan))
            hubs, thr = plan.info()
            res.append(dict(d=d, bytes=byts, plan_ms=planned, hubs=hubs, hub_threshold=thr,
                            plan_gbs=byts / planned[1] / 1e6))
            print(json.dumps(res[-1]), flush=True)
            del plan
    out["spmm"] = res
    print(json.dumps(out))


if __name__ == "__main__":
    main()
