"""In-process cluster: `Cluster` / `Cluster::run` (cluster.hpp:188-250,
405-442) and `train_distributed` (trainer.hpp:541-687) with every rank of
the grid a host thread of this process driving its own engine — the
reference's own execution model, on the B200 engine.

Ranks may share one GPU (every grid of 2, 4 or 8 ranks fits on one B200 at
test sizes) or spread over the visible devices (`devices`). Collectives are
the library's ordered device sums / copies sequenced by CUDA events that the
members of an axis group swap at a host rendezvous (csrc/local.cu), so
results equal the reference's coordinate-order combine bit for bit. A rank
that fails aborts the cluster; the others fail with ClusterAborted naming it
(cluster.hpp:67-71, 240, 434).

The multi-process path (one process per GPU, NCCL + NVLink peer memory) is
`distributed.py`; this one needs no second GPU, so the engine's multi-rank
schedule runs wherever one B200 does.
"""

import ctypes as C
import threading
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _capi
from ._capi import ClusterAborted, call
from .distributed import TrainResult, reassemble, reduce_epoch_metrics
from .layout import GridConfig

_capi.register({
    "pk_cluster_create": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "pk_cluster_abort": (C.c_int, [C.c_void_p, C.c_int, C.c_char_p]),
    "pk_cluster_aborted": (C.c_int, [C.c_void_p, C.POINTER(C.c_int)]),
    "pk_cluster_destroy": (C.c_int, [C.c_void_p]),
    "pk_engine_comm_init_local": (C.c_int, [C.c_void_p, C.c_void_p]),
})


class Cluster:
    """G = gx*gy*gz ranks as threads of this process (ClusterOptions'
    `max_running` has no counterpart: every rank has its own stream)."""

    def __init__(self, grid: GridConfig, devices: Optional[Sequence[int]] = None):
        import torch
        self.grid = grid
        self.devices = list(devices) if devices else [torch.cuda.current_device()]
        h = C.c_void_p()
        call("pk_cluster_create", grid.gx, grid.gy, grid.gz, C.byref(h))
        self.h = h

    def device_of(self, rank: int) -> int:
        return self.devices[rank % len(self.devices)]

    def engine(self, n, feat_dim, classes, rank, opts):
        """A RankEngine bound to this cluster as `rank`."""
        from . import trainer
        e = trainer.RankEngine(n, feat_dim, classes, self.grid, rank, opts, self.device_of(rank))
        call("pk_engine_comm_init_local", e.h, self.h)
        return e

    def run(self, fn: Callable[[int], object]) -> List[object]:
        """Cluster::run: fn(rank) on one thread per rank; returns the results
        in rank order. The first failure is re-raised (the reference
        rethrows the primary exception, cluster.hpp:436-441); ranks that
        failed only because of it raise ClusterAborted."""
        import torch
        out: List[object] = [None] * self.grid.size
        errs: List[Optional[BaseException]] = [None] * self.grid.size

        def body(r):
            try:
                torch.cuda.set_device(self.device_of(r))
                out[r] = fn(r)
            except BaseException as exc:  # noqa: BLE001 - reported below
                errs[r] = exc
                try:
                    call("pk_cluster_abort", self.h, r, str(exc).encode()[:1000])
                except Exception:
                    pass

        threads = [threading.Thread(target=body, args=(r,), daemon=True)
                   for r in range(self.grid.size)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
        primary = [e for e in errs if e is not None and not _is_aborted(e)]
        if primary:
            raise primary[0]
        if any(e is not None for e in errs):
            raise next(e for e in errs if e is not None)
        return out

    def aborted(self) -> bool:
        v = C.c_int()
        call("pk_cluster_aborted", self.h, C.byref(v))
        return bool(v.value)

    def close(self):
        if getattr(self, "h", None):
            call("pk_cluster_destroy", self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _is_aborted(exc) -> bool:
    return isinstance(exc, ClusterAborted)


def distributed_pass(pre, grid: GridConfig, opts, devices=None):
    """rank_forward_backward (trainer.hpp:478-527) on every rank of `grid`,
    reassembled like test_engine.cpp:30-84: (loss, accuracy, logits, dW,
    dF0, per-rank losses)."""
    from . import trainer
    cl = Cluster(grid, devices)
    dims = trainer.model_dims(pre.feat_dim, list(opts.hidden_dims), pre.num_classes)
    L = len(dims) - 1

    def rank_pass(r):
        e = cl.engine(pre.n, pre.feat_dim, pre.num_classes, r, opts)
        try:
            e.load(pre)
            loss, acc = e.forward_backward(0)
            return {"fout": e.tensor(trainer.PK_T_FOUT).cpu().numpy(),
                    "dw": [e.tensor(trainer.PK_T_DW, l).cpu().numpy() for l in range(L)],
                    "df0": e.tensor(trainer.PK_T_DF0).cpu().numpy(), "loss": loss, "acc": acc,
                    "comm": e.comm_stats()}
        finally:
            e.close()
    try:
        per = cl.run(rank_pass)
    finally:
        cl.close()
    logits, dw, df0 = trainer.gather_rank_pass(per, grid, pre.n, dims)
    return dict(loss=per[0]["loss"], accuracy=per[0]["acc"], logits=logits, dw=dw, df0=df0,
                rank_losses=[p["loss"] for p in per],
                comm_calls=np.array([p["comm"][0] for p in per]),
                comm_bytes=np.array([p["comm"][1] for p in per]))


def train_distributed(pre, grid: GridConfig, opts, devices=None) -> TrainResult:
    """train_distributed (trainer.hpp:541-687) with in-process ranks: global
    init sliced per rank, opts.epochs of pass + Adam, metrics reduced like
    trainer.hpp:660-686, W and F0 reassembled from the rank shards."""
    from . import trainer
    cl = Cluster(grid, devices)
    dims = trainer.model_dims(pre.feat_dim, list(opts.hidden_dims), pre.num_classes)
    L = len(dims) - 1

    def rank_train(r):
        e = cl.engine(pre.n, pre.feat_dim, pre.num_classes, r, opts)
        try:
            e.load(pre)
            metrics = [e.train_epoch(ep) for ep in range(opts.epochs)]
            w = [e.tensor(trainer.PK_T_W, l).cpu().numpy() for l in range(L)]
            f = e.tensor(trainer.PK_T_F0).cpu().numpy()
            return metrics, w, f
        finally:
            e.close()
    try:
        per = cl.run(rank_train)
    finally:
        cl.close()
    res = TrainResult(per_rank=[p[0] for p in per])
    res.global_metrics = reduce_epoch_metrics(res.per_rank)
    res.weights, res.features = reassemble(grid, pre.n, dims, [p[1] for p in per],
                                           [p[2] for p in per])
    return res





def train_distributed_generated(spec, grid: GridConfig, opts, devices=None) -> TrainResult:
    """train_distributed with the file_handle-style per-rank loader replaced
    by per-rank generation (rank_gen.generate_rank_tensors): no rank, and no
    host, ever holds the global graph."""
    from . import rank_gen, trainer
    cl = Cluster(grid, devices)
    dims = trainer.model_dims(spec.feat_dim, list(opts.hidden_dims), spec.classes)
    L = len(dims) - 1
    pieces = rank_gen.global_pieces(spec, 0, grid.size)

    def rank_train(r):
        e = cl.engine(spec.n, spec.feat_dim, spec.classes, r, opts)
        try:
            e.load_rank(rank_gen.generate_rank_tensors(spec, grid, r, L, pieces), adopt=True)
            metrics = [e.train_epoch(ep) for ep in range(opts.epochs)]
            w = [e.tensor(trainer.PK_T_W, l).cpu().numpy() for l in range(L)]
            f = e.tensor(trainer.PK_T_F0).cpu().numpy()
            return metrics, w, f
        finally:
            e.close()
    try:
        per = cl.run(rank_train)
    finally:
        cl.close()
    res = TrainResult(per_rank=[p[0] for p in per])
    res.global_metrics = reduce_epoch_metrics(res.per_rank)
    res.weights, res.features = reassemble(grid, spec.n, dims, [p[1] for p in per],
                                           [p[2] for p in per])
    return res
__all__ = ["Cluster", "ClusterAborted", "distributed_pass", "train_distributed", "train_distributed_generated"]
