"""train_distributed (trainer.hpp:541-687) for one process per GPU.

The reference runs every rank of the grid as a thread of one process
(`Cluster::run`, cluster.hpp:405-442) and reassembles the result on the host.
Here each rank is its own process (torchrun), drives one GPU through its
`pk_engine` (csrc/engine.cu), and the engine's collectives run on NCCL per-
axis communicators. torch.distributed (gloo, host memory) is only the control
plane: it broadcasts the NCCL unique id and gathers the per-rank metrics and
parameter shards for the same host-side reassembly the reference does
(trainer.hpp:636-686) — global loss from rank 0, phase times = max over
ranks, FLOPs and bytes summed, W / F0 stitched from weight_slice /
feature_slice.

`engine_factory` lets tests drive this host logic with a stand-in engine on
CPU (tests/test_distributed_cpu.py, world size 2 over gloo).
"""

import os
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional

import numpy as np

from .layout import GridConfig, feature_slice, plan_layouts, weight_slice

MAX_KEYS = ("forward_spmm_s", "forward_gemm_s", "backward_s", "optimizer_s", "collectives_s",
            "epoch_s", "spmm_s")
SUM_KEYS = ("spmm_flops", "gemm_flops", "allreduce_bytes", "allgather_bytes",
            "reducescatter_bytes", "spmm_bytes", "spmm_compulsory_bytes", "kernel_launches")


@dataclass
class TrainResult:
    """TrainResult (trainer.hpp:529-539), host side."""
    global_metrics: List[Dict] = field(default_factory=list)
    per_rank: List[List[Dict]] = field(default_factory=list)
    weights: List[np.ndarray] = field(default_factory=list)
    features: Optional[np.ndarray] = None
    # CommStats per rank (cluster.hpp:35-65): (calls, ring bytes), [axis][op]
    stats: List = field(default_factory=list)


def dist_env():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def init_control_plane(backend="gloo"):
    """Host control plane (uid broadcast, metric gathers). Idempotent."""
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group(backend, rank=rank, world_size=world)
    return rank, world


def broadcast_unique_id(make_uid: Callable[[], bytes]):
    """Rank 0 creates the 128-byte ncclUniqueId; every rank receives it."""
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world == 1:
        return None
    obj = [make_uid() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def reduce_epoch_metrics(per_rank: List[List[Dict]]) -> List[Dict]:
    """trainer.hpp:660-686: loss/accuracy from rank 0, times max over ranks,
    counters summed."""
    out = []
    for e in range(len(per_rank[0])):
        g = {"epoch": per_rank[0][e]["epoch"], "loss": per_rank[0][e]["loss"],
             "accuracy": per_rank[0][e]["accuracy"]}
        for k in MAX_KEYS:
            g[k] = max(r[e].get(k, 0.0) for r in per_rank)
        for k in SUM_KEYS:
            g[k] = sum(r[e].get(k, 0) for r in per_rank)
        out.append(g)
    return out


def reassemble(grid: GridConfig, n: int, dims: List[int], w_shards: List[List[np.ndarray]],
               f0_shards: List[np.ndarray]):
    """trainer.hpp:642-659: full W per layer and F0 from the rank shards."""
    lays = plan_layouts(len(dims) - 1)
    weights = []
    for l in range(len(dims) - 1):
        w = np.zeros((dims[l], dims[l + 1]), np.float32)
        for r in range(grid.size):
            r0, r1, c0, c1 = weight_slice(grid, lays[l], grid.coords_of(r), dims[l], dims[l + 1])
            w[r0:r1, c0:c1] = w_shards[r][l]
        weights.append(w)
    f = np.zeros((n, dims[0]), np.float32)
    for r in range(grid.size):
        r0, r1, c0, c1 = feature_slice(grid, grid.coords_of(r), n, dims[0])
        f[r0:r1, c0:c1] = f0_shards[r]
    return weights, f


def train_distributed(load_dataset: Callable[[], object], grid: GridConfig, opts,
                      engine_factory: Optional[Callable] = None,
                      reassemble_params: bool = True,
                      epoch_hook: Optional[Callable[[int], None]] = None) -> TrainResult:
    """Collective call on every rank (world size == grid.size). Returns the
    reassembled TrainResult on rank 0 and per-rank metrics everywhere."""
    import torch.distributed as dist
    rank, world = init_control_plane()
    if world != grid.size:
        raise ValueError(f"train_distributed: world size {world} != grid size {grid.size}")
    pre = load_dataset()
    if engine_factory is None:
        import torch

        from . import trainer
        _, _, local = dist_env()
        torch.cuda.set_device(local)

        def engine_factory(pre_, grid_, rank_, opts_):
            e = trainer.RankEngine(pre_.n, pre_.feat_dim, pre_.num_classes, grid_, rank_, opts_,
                                   local)
            if grid_.size > 1:
                e.comm_init(broadcast_unique_id(trainer.nccl_unique_id), grid_.size)
            e.load(pre_)
            return e
    eng = engine_factory(pre, grid, rank, opts)
    mine = []
    try:
        for e in range(opts.epochs):
            mine.append(eng.train_epoch(e))
            if epoch_hook is not None:
                epoch_hook(e)
    except Exception as exc:
        # a failure on this rank takes the grid down (cluster.hpp:240, 434):
        # peers blocked in their epoch raise ClusterAborted instead of hanging
        from ._capi import ClusterAborted
        if not isinstance(exc, ClusterAborted) and hasattr(eng, "abort"):
            eng.abort(f"{type(exc).__name__}: {exc}")
        raise
    L = len(eng.dims) - 1
    w_mine = [np.asarray(_host(eng.tensor(0, l))) for l in range(L)] if reassemble_params else []
    f_mine = np.asarray(_host(eng.tensor(2))) if reassemble_params else None
    dims = list(eng.dims)
    stats = eng.comm_stats() if hasattr(eng, "comm_stats") else None
    eng.close()
    if world > 1:
        gathered = [None] * world
        dist.all_gather_object(gathered, (mine, w_mine, f_mine, stats))
    else:
        gathered = [(mine, w_mine, f_mine, stats)]
    res = TrainResult(per_rank=[g[0] for g in gathered], stats=[g[3] for g in gathered])
    res.global_metrics = reduce_epoch_metrics(res.per_rank)
    if reassemble_params:
        res.weights, res.features = reassemble(grid, pre.n, dims, [g[1] for g in gathered],
                                               [g[2] for g in gathered])
    return res


def _host(t):
    try:
        return t.detach().cpu().numpy()
    except AttributeError:
        return t


__all__ = ["TrainResult", "train_distributed", "reduce_epoch_metrics", "reassemble",
           "broadcast_unique_id", "init_control_plane", "dist_env"]
