"""Breaks the bench's e2e number (train from a pinned-host dataset) into
phases: engine creation, load (H2D + shards + plans; PK_TIMING=1 prints the
load's own phases), and each epoch's wall time."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2505_04083_b200 import layout, trainer

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
pre = bench.build_dataset(cfg, 0)
host = trainer.HostDataset.from_device(pre, pin=True)
opts = trainer.TrainOptions(hidden_dims=cfg["hidden"], mode=trainer.PK_MODE_FAST)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng = trainer.RankEngine(host.n, host.feat_dim, host.num_classes, layout.GridConfig(1, 1, 1), 0, opts, 0)
    t1 = time.perf_counter()
    eng.load(host)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ep = []
    for e in range(5):
        a = time.perf_counter(); eng.train_epoch(e); ep.append((time.perf_counter() - a) * 1e3)
    eng.close()
    print(f"rep {rep}: create {1e3*(t1-t0):.1f} ms, load {1e3*(t2-t1):.1f} ms, epochs ms {[round(x,1) for x in ep]}", flush=True)
