"""Per-rank compute of a multi-GPU grid measured on ONE B200: every rank of
the grid is loaded in turn from the same preprocessed dataset, in
measurement mode (pk_engine_comm_init_solo: collectives keep only the rank's
own contribution, so the epoch is the rank's compute alone), and trained a
few epochs. Against the real N-GPU epoch this separates the compute (and its
imbalance across ranks) from the exposed collective time.

    python scripts/solo_ranks.py --config c2 --grid 2,1,2
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import bench  # noqa: E402
from paper_2505_04083_b200 import layout, trainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--grid", default="2,1,2")
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--epochs", type=int, default=5)
    ap.add_argument("--ranks", default="")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    cfg = bench.CONFIGS[args.config]
    pre = bench.build_dataset(cfg, 0)
    grid = layout.GridConfig(*[int(x) for x in args.grid.split(",")])
    ranks = [int(r) for r in args.ranks.split(",")] if args.ranks else range(grid.size)
    for r in ranks:
        opts = trainer.TrainOptions(hidden_dims=cfg["hidden"], mode=trainer.PK_MODE_FAST)
        eng = trainer.RankEngine(pre.n, pre.feat_dim, pre.num_classes, grid, r, opts, 0)
        eng.comm_init_solo()
        eng.load(pre)
        for e in range(args.warmup):
            eng.train_epoch(e)
        torch.cuda.synchronize()
        stream = torch.cuda.ExternalStream(eng.stream_ptr())
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        ms = eng.train_epochs(args.warmup, args.epochs)
        ev1.record(stream)
        torch.cuda.synchronize()
        phases = {k: round(float(np.mean([m[k] for m in ms])) * 1e3, 3) for k in
                  ("forward_spmm_s", "forward_gemm_s", "backward_s", "optimizer_s",
                   "collectives_s", "spmm_s")}
        print("SOLO " + json.dumps({"config": args.config, "grid": args.grid, "rank": r,
                                    "epoch_ms": ev0.elapsed_time(ev1) / args.epochs,
                                    "phases_ms": phases}), flush=True)
        eng.close()
        del eng
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
