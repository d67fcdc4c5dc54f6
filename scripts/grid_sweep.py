"""C5: the 3D grid-configuration sweep (BASELINE.json configs[4]).

Runs every ordered factorization of the world size on the products-shaped
graph (one process per GPU, torchrun), measures epoch time and its SpMM /
collective phases per grid (max over ranks), then checks the performance
model (csrc/perf_model.cpp, the reference's rank_configs) against the
measurements: the ranking with the reference's default coefficients, and
with coefficients refit on these B200 SpMM timings (fit_regression over
n,nnz,dims,gx,gy,gz,seconds samples, perf_model.cpp:301-331). Prints one
JSON line per grid and a summary line with Spearman rank correlations.

    torchrun --nproc-per-node 4 scripts/grid_sweep.py --epochs 3
"""
import argparse
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2505_04083_b200 import distributed as D, layout, perf_model as pm, trainer  # noqa: E402


def spearman(a, b):
    ra = np.argsort(np.argsort(a))
    rb = np.argsort(np.argsort(b))
    if len(a) < 2:
        return 1.0
    return float(np.corrcoef(ra, rb)[0, 1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    args = ap.parse_args()
    rank, world, local = D.dist_env()
    torch.cuda.set_device(local)
    D.init_control_plane()
    cfg = bench.CONFIGS[args.config]
    pre = bench.build_dataset(cfg, local)
    dims = [cfg["feat"], *cfg["hidden"], cfg["classes"]]
    opts = trainer.TrainOptions(hidden_dims=cfg["hidden"], mode=trainer.PK_MODE_FAST)
    rows = []
    for shape in pm.enumerate_configs(world):
        grid = layout.GridConfig(*shape)
        eng = trainer.RankEngine(pre.n, pre.feat_dim, pre.num_classes, grid, rank, opts, local)
        if world > 1:
            eng.comm_init(D.broadcast_unique_id(trainer.nccl_unique_id), world)
        eng.load(pre)
        for e in range(args.warmup):
            eng.train_epoch(e)
        ms = []
        for e in range(args.epochs):
            m = eng.train_epoch(args.warmup + e)
            ms.append([m["epoch_s"], m["spmm_s"], m["collectives_s"]])
        eng.close()
        t = torch.tensor(np.mean(ms, axis=0), device="cuda", dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        epoch_s, spmm_s, comm_s = t.tolist()
        rows.append(dict(grid=list(shape), epoch_ms=epoch_s * 1e3, spmm_ms=spmm_s * 1e3,
                         collectives_ms=comm_s * 1e3))
        if rank == 0:
            print(json.dumps(rows[-1]), flush=True)
    if rank == 0:
        stats = pm.DatasetStats(pre.n, pre.a_even.nnz, dims)
        machine = pm.MachineParams(**bench.B200_MACHINE)
        shapes = [tuple(r["grid"]) for r in rows]
        measured = [r["epoch_ms"] for r in rows]
        default = pm.rank_configs(world, stats, machine, pm.default_coefficients())
        pred_default = {p.shape: p.total_seconds for p in default}
        out = {"world": world, "measured_best": list(shapes[int(np.argmin(measured))]),
               "default_pick": list(default[0].shape),
               "spearman_default": spearman([pred_default[s] for s in shapes], measured)}
        if len(rows) >= 3:
            samples = [pm.RegressionSample(pm.comp_features(stats, s), r["spmm_ms"] * 1e-3)
                       for s, r in zip(shapes, rows)]
            try:
                fit = pm.fit_regression(samples)
                refit = pm.rank_configs(world, stats, machine, fit)
                pred_fit = {p.shape: p.total_seconds for p in refit}
                out.update(refit_coeffs=[fit.c1, fit.c2, fit.c3], refit_r2=fit.train_r2,
                           refit_pick=list(refit[0].shape),
                           spearman_refit=spearman([pred_fit[s] for s in shapes], measured))
            except Exception as exc:  # rank-deficient on few configs
                out["refit_error"] = str(exc)
        print("SWEEP " + json.dumps(out), flush=True)
    dist.barrier() if world > 1 else None
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
