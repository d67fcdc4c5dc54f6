"""torchrun worker for the abort test (tests/test_multigpu_gpu.py): every
rank trains on NCCL axis communicators; rank --fail-rank raises from its host
code after epoch --fail-epoch (train_distributed's epoch hook). The failing
rank must report its own error and every other rank ClusterAborted naming
it — within seconds, not by hanging in a collective (cluster.hpp:67-71,
240, 434)."""
import argparse
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2505_04083_b200 import _capi, distributed as D, graph, trainer  # noqa: E402
from paper_2505_04083_b200.layout import GridConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="2,1,1")
    ap.add_argument("--fail-rank", type=int, default=1)
    ap.add_argument("--fail-epoch", type=int, default=1)
    args = ap.parse_args()
    grid = GridConfig(*[int(g) for g in args.grid.split(",")])
    rank, world, local = D.dist_env()
    torch.cuda.set_device(local)
    D.init_control_plane()
    pre = graph.preprocess(graph.synth_rmat(12, 40000, 16, 5, seed=2), perm_seed=2)
    opts = trainer.TrainOptions(hidden_dims=[32, 32], mode=trainer.PK_MODE_FAST, epochs=50)

    def hook(e):
        if rank == args.fail_rank and e == args.fail_epoch:
            raise ValueError(f"injected failure on rank {rank}")
    t0 = time.time()
    kind, msg = "none", ""
    try:
        D.train_distributed(lambda: pre, grid, opts, epoch_hook=hook)
    except _capi.ClusterAborted as exc:
        kind, msg = "ClusterAborted", str(exc)
    except ValueError as exc:
        kind, msg = "ValueError", str(exc)
    dt = time.time() - t0
    ok = (kind == "ValueError") if rank == args.fail_rank else \
        (kind == "ClusterAborted" and f"rank {args.fail_rank}" in msg)
    print(f"ABORTRESULT rank={rank} kind={kind} ok={int(ok)} s={dt:.1f} msg={msg[:200]}",
          flush=True)
    os._exit(0 if ok else 1)  # no teardown of aborted communicators / process groups


if __name__ == "__main__":
    main()
