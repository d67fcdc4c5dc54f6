"""Driver for ncu captures of the epoch: builds the products-shaped graph
(or --config), runs `--warmup` untimed epochs, then `--epochs` epochs inside
cudaProfilerStart/Stop so `ncu --profile-from-start off` sees exactly the
epoch's launches.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv \
        python scripts/epoch_driver.py --config c2
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2505_04083_b200 import layout, trainer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--epochs", type=int, default=1)
    ap.add_argument("--mode", default="fast")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    pre = bench.build_dataset(cfg, 0)
    mode = trainer.PK_MODE_FAST if args.mode == "fast" else trainer.PK_MODE_PARITY
    opts = trainer.TrainOptions(hidden_dims=cfg["hidden"], mode=mode)
    eng = trainer.RankEngine(pre.n, pre.feat_dim, pre.num_classes, layout.GridConfig(1, 1, 1),
                             0, opts, 0)
    eng.load(pre)
    for e in range(args.warmup):
        eng.train_epoch(e)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    for e in range(args.epochs):
        m = eng.train_epoch(args.warmup + e)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("epoch_driver: ok", {k: m[k] for k in ("loss", "epoch_s", "spmm_s", "kernel_launches")})
    eng.close()


if __name__ == "__main__":
    main()
