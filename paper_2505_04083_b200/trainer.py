"""Host mirror of the reference trainer API (trainer.hpp): TrainOptions,
EpochMetrics, the per-rank engine and train_distributed, over the C++ engine
in libplexus_b200.so (one engine per GPU; NCCL per-axis communicators).

Process model: one process per GPU (torchrun). Rank 0 creates the NCCL
unique id and every rank receives it through torch.distributed (gloo or
nccl) — torch is only the bootstrap; all collectives of the hot path are
issued by the C++ engine.
"""

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from . import _capi
from ._capi import PK_MODE_FAST, PK_MODE_PARITY, call
from .graph import PreprocessedDataset
from .layout import GridConfig, feature_slice, label_row_range, model_dims, plan_layouts, \
    weight_slice

PK_MAX_LAYERS = 15
PK_T_W, PK_T_DW, PK_T_F0, PK_T_DF0, PK_T_FOUT, PK_T_H, PK_T_Q, PK_T_ACT = range(8)


class pk_engine_config(C.Structure):
    _fields_ = [("gx", C.c_int), ("gy", C.c_int), ("gz", C.c_int), ("rank", C.c_int),
                ("device", C.c_int), ("num_layers", C.c_int),
                ("dims", C.c_int64 * (PK_MAX_LAYERS + 1)), ("n", C.c_int64),
                ("seed", C.c_uint64), ("lr", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("block_count", C.c_int),
                ("mode", C.c_int), ("fault_epoch", C.c_int), ("hub_threshold", C.c_int64)]


class pk_dataset_view(C.Structure):
    _fields_ = [("n", C.c_int64), ("feat_dim", C.c_int64), ("num_classes", C.c_uint32),
                ("a_even", _capi.pk_csr), ("a_odd", _capi.pk_csr), ("features", C.c_void_p),
                ("ld_features", C.c_int64), ("labels_row", C.c_void_p),
                ("labels_col", C.c_void_p), ("mask_row", C.c_void_p), ("mask_col", C.c_void_p)]


class pk_epoch_metrics(C.Structure):
    _fields_ = [("epoch", C.c_int), ("loss", C.c_double), ("accuracy", C.c_double),
                ("forward_spmm_s", C.c_double), ("forward_gemm_s", C.c_double),
                ("backward_s", C.c_double), ("optimizer_s", C.c_double),
                ("collectives_s", C.c_double), ("epoch_s", C.c_double),
                ("spmm_s", C.c_double), ("spmm_bytes", C.c_double),
                ("kernel_launches", C.c_uint64),
                ("spmm_flops", C.c_uint64), ("gemm_flops", C.c_uint64),
                ("allreduce_bytes", C.c_double), ("allgather_bytes", C.c_double),
                ("reducescatter_bytes", C.c_double), ("spmm_compulsory_bytes", C.c_double)]


class pk_rank_view(C.Structure):
    _fields_ = [("adj", _capi.pk_csr * 6), ("f0", C.c_void_p), ("f0_rows", C.c_int64),
                ("f0_cols", C.c_int64), ("ld_f0", C.c_int64), ("labels", C.c_void_p),
                ("mask", C.c_void_p), ("label_rows", C.c_int64)]


class pk_tensor_view(C.Structure):
    _fields_ = [("data", C.c_void_p), ("rows", C.c_int64), ("cols", C.c_int64),
                ("ld", C.c_int64)]


_SIGS = {
    "pk_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "pk_engine_create": (C.c_int, [C.POINTER(pk_engine_config), C.POINTER(C.c_void_p)]),
    "pk_engine_comm_init": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "pk_engine_load": (C.c_int, [C.c_void_p, C.POINTER(pk_dataset_view)]),
    "pk_engine_load_host": (C.c_int, [C.c_void_p, C.POINTER(pk_dataset_view)]),
    "pk_engine_load_rank": (C.c_int, [C.c_void_p, C.POINTER(pk_rank_view)]),
    "pk_engine_load_rank_adopt": (C.c_int, [C.c_void_p, C.POINTER(pk_rank_view),
                                            C.POINTER(_capi.pk_csr_owned)]),
    "pk_engine_forward_backward": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_double),
                                             C.POINTER(C.c_double)]),
    "pk_engine_optimizer_step": (C.c_int, [C.c_void_p]),
    "pk_engine_train_epoch": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(pk_epoch_metrics)]),
    "pk_engine_forward_only": (C.c_int, [C.c_void_p]),
    "pk_engine_train_epochs": (C.c_int, [C.c_void_p, C.c_int, C.c_int,
                                         C.POINTER(pk_epoch_metrics)]),
    "pk_engine_tensor": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.POINTER(pk_tensor_view)]),
    "pk_engine_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "pk_engine_destroy": (C.c_int, [C.c_void_p]),
    "pk_engine_abort": (C.c_int, [C.c_void_p, C.c_char_p]),
    "pk_engine_comm_init_solo": (C.c_int, [C.c_void_p]),
    "pk_engine_comm_stats": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
}
_capi.register(_SIGS)


def _d2h_threads():
    v = os.environ.get("PK_D2H_THREADS")
    return max(1, int(v)) if v else 1


@dataclass
class TrainOptions:
    """TrainOptions (trainer.hpp:31-38) + the engine knobs (EngineOptions,
    engine.hpp:123-127): GEMM mode and the SpMM hub threshold."""
    epochs: int = 10
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    seed: int = 0
    block_count: int = 0
    hidden_dims: List[int] = field(default_factory=lambda: [128, 128])
    fault_epoch: int = -1
    mode: int = PK_MODE_PARITY
    hub_threshold: int = 0


METRIC_KEYS = ("epoch", "loss", "accuracy", "forward_spmm_s", "forward_gemm_s", "backward_s",
               "optimizer_s", "collectives_s", "epoch_s", "spmm_s", "spmm_bytes",
               "kernel_launches", "spmm_flops", "gemm_flops",
               "allreduce_bytes", "allgather_bytes", "reducescatter_bytes",
               "spmm_compulsory_bytes")


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    call("pk_nccl_unique_id", C.cast(buf, C.c_void_p))
    return bytes(buf)


def _csr_struct(a):
    return _capi.pk_csr(a.rows, a.cols, a.nnz, a.row_ptr.data_ptr(),
                        a.col_idx.data_ptr() if a.nnz else 0,
                        a.values.data_ptr() if a.nnz else 0)


def dataset_view(pre: PreprocessedDataset):
    """pk_dataset_view over a device-resident PreprocessedDataset."""
    f = pre.features
    v = pk_dataset_view(pre.n, pre.feat_dim, pre.num_classes, _csr_struct(pre.a_even),
                        _csr_struct(pre.a_odd), f.data_ptr(), f.stride(0),
                        pre.labels_row_order.data_ptr(), pre.labels_col_order.data_ptr(),
                        pre.mask_row_order.data_ptr(), pre.mask_col_order.data_ptr())
    return v


@dataclass
class HostDataset:
    """A PreprocessedDataset held in (pinned) host memory: numpy arrays."""
    n: int
    feat_dim: int
    num_classes: int
    even: tuple
    odd: tuple
    features: np.ndarray
    labels_row: np.ndarray
    labels_col: np.ndarray
    mask_row: np.ndarray
    mask_col: np.ndarray

    @classmethod
    def from_device(cls, pre: PreprocessedDataset, pin=True):
        def host(t):
            h = torch.empty(t.shape, dtype=t.dtype, pin_memory=pin)
            h.copy_(t)
            return h
        keep = []

        def csr(a):
            parts = [host(a.row_ptr), host(a.col_idx), host(a.values)]
            keep.extend(parts)
            return tuple(p.numpy() for p in parts)
        feats = host(pre.features)
        ds = cls(pre.n, pre.feat_dim, pre.num_classes, csr(pre.a_even), csr(pre.a_odd),
                 feats.numpy(), host(pre.labels_row_order).numpy(),
                 host(pre.labels_col_order).numpy(), host(pre.mask_row_order).numpy(),
                 host(pre.mask_col_order).numpy())
        ds._keep = keep + [feats]
        return ds

    def nbytes(self):
        return sum(a.nbytes for a in (*self.even, *self.odd, self.features, self.labels_row,
                                      self.labels_col, self.mask_row, self.mask_col))

    def view(self):
        def csr(t):
            rp, ci, v = t
            return _capi.pk_csr(self.n, self.n, ci.size, rp.ctypes.data, ci.ctypes.data,
                                v.ctypes.data)
        p = lambda a: a.ctypes.data  # noqa: E731
        return pk_dataset_view(self.n, self.feat_dim, self.num_classes, csr(self.even),
                               csr(self.odd), p(self.features), self.features.shape[1],
                               p(self.labels_row), p(self.labels_col), p(self.mask_row),
                               p(self.mask_col))


class RankEngine:
    """One rank of the 3D grid on one GPU (the per-rank lambda of
    train_distributed, trainer.hpp:562-633)."""

    def __init__(self, n, feat_dim, classes, grid: GridConfig, rank: int,
                 opts: TrainOptions = None, device: Optional[int] = None):
        self.opts = opts or TrainOptions()
        self.grid = grid
        self.rank = rank
        self.dims = model_dims(feat_dim, list(self.opts.hidden_dims), classes)
        if len(self.dims) - 1 > PK_MAX_LAYERS:
            raise _capi.ContractError("too many layers")
        self.n = n
        self.device = torch.cuda.current_device() if device is None else device
        cfg = pk_engine_config()
        cfg.gx, cfg.gy, cfg.gz = grid.gx, grid.gy, grid.gz
        cfg.rank, cfg.device, cfg.num_layers = rank, self.device, len(self.dims) - 1
        for i, d in enumerate(self.dims):
            cfg.dims[i] = d
        cfg.n, cfg.seed = n, self.opts.seed
        cfg.lr, cfg.beta1, cfg.beta2, cfg.eps = (self.opts.lr, self.opts.beta1, self.opts.beta2,
                                                 self.opts.eps)
        cfg.block_count, cfg.mode = self.opts.block_count, self.opts.mode
        cfg.fault_epoch, cfg.hub_threshold = self.opts.fault_epoch, self.opts.hub_threshold
        h = C.c_void_p()
        call("pk_engine_create", C.byref(cfg), C.byref(h))
        self.h = h

    def comm_init(self, uid: bytes, world_size: int):
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        call("pk_engine_comm_init", self.h, C.cast(buf, C.c_void_p), world_size)

    def comm_stats(self):
        """CommStats since the load: (calls, ring bytes), each [axis][op]
        (op: all_gather, all_reduce, reduce_scatter)."""
        calls = np.zeros(9, np.uint64)
        byts = np.zeros(9, np.float64)
        call("pk_engine_comm_stats", self.h, calls.ctypes.data_as(C.c_void_p),
             byts.ctypes.data_as(C.c_void_p))
        return calls.reshape(3, 3), byts.reshape(3, 3)

    def comm_init_solo(self):
        """Measurement mode (pk_engine_comm_init_solo): this rank alone;
        collectives keep only its own contribution."""
        call("pk_engine_comm_init_solo", self.h)

    def load(self, pre):
        """A PreprocessedDataset (device), a HostDataset (pinned host), or a
        shard manifest — the file_handle path (trainer.hpp:461-466): this
        rank reads only its blocks (shard_io.load_rank_shards)."""
        from . import shard_io
        if isinstance(pre, shard_io.ShardManifest):
            rt = shard_io.load_rank_shards(pre, self.grid, self.grid.coords_of(self.rank),
                                           len(self.dims) - 1)
            self.load_rank(rt)
            return
        if isinstance(pre, HostDataset):
            v = pre.view()
            call("pk_engine_load_host", self.h, C.byref(v))
        else:
            v = dataset_view(pre)
            torch.cuda.synchronize()
            call("pk_engine_load", self.h, C.byref(v))

    def load_rank(self, rt, adopt=False):
        """RankTensors (shard_io.RankTensors) -> pk_engine_load_rank. With
        adopt=True, library-allocated blocks (rank_gen / shard builder
        outputs) are handed to the engine instead of copied
        (pk_engine_load_rank_adopt); those DeviceCsr objects are spent."""
        v = pk_rank_view()
        for (plane, parity), (blk, _) in rt.adj.items():
            v.adj[plane * 2 + parity] = blk._view
        f0 = rt.f0.contiguous()
        v.f0 = f0.data_ptr() if f0.numel() else None
        v.f0_rows, v.f0_cols, v.ld_f0 = f0.shape[0], f0.shape[1], f0.shape[1]
        v.labels = rt.labels.data_ptr() if rt.labels.numel() else None
        v.mask = rt.mask.data_ptr() if rt.mask.numel() else None
        v.label_rows = rt.labels.numel()
        torch.cuda.synchronize()
        if not adopt:
            call("pk_engine_load_rank", self.h, C.byref(v))
            return
        owned = (_capi.pk_csr_owned * 6)()
        taken, seen = [], set()
        for (plane, parity), (blk, _) in rt.adj.items():
            keep = getattr(blk, "_owned", None)
            if keep is None or id(keep) in seen or not keep.owned.row_ptr:
                continue
            seen.add(id(keep))
            owned[plane * 2 + parity] = keep.owned
            taken.append(keep)
        call("pk_engine_load_rank_adopt", self.h, C.byref(v), owned)
        for keep in taken:  # the engine owns those arrays now
            keep.owned = _capi.pk_csr_owned()

    def forward_backward(self, epoch=0):
        loss, acc = C.c_double(), C.c_double()
        call("pk_engine_forward_backward", self.h, epoch, C.byref(loss), C.byref(acc))
        return loss.value, acc.value

    def optimizer_step(self):
        call("pk_engine_optimizer_step", self.h)

    def train_epoch(self, epoch):
        m = pk_epoch_metrics()
        call("pk_engine_train_epoch", self.h, epoch, C.byref(m))
        return {k: getattr(m, k) for k in METRIC_KEYS}

    def abort(self, why: str):
        """This rank failed: take the grid down (pk_engine_abort) — the other
        ranks' pending epoch fails with ClusterAborted naming this rank."""
        call("pk_engine_abort", self.h, str(why).encode()[:500])

    def train_epochs(self, first, count):
        """`count` epochs with one host wait (pk_engine_train_epochs)."""
        arr = (pk_epoch_metrics * count)()
        call("pk_engine_train_epochs", self.h, first, count, arr)
        return [{k: getattr(m, k) for k in METRIC_KEYS} for m in arr]

    def tensor(self, which, layer=0) -> torch.Tensor:
        """Copy of an engine tensor (rows x cols) as a CUDA tensor."""
        v = pk_tensor_view()
        call("pk_engine_tensor", self.h, which, layer, C.byref(v))
        if v.rows == 0 or v.cols == 0:
            return torch.zeros((v.rows, v.cols), dtype=torch.float32, device="cuda")

        class _Arr:
            __cuda_array_interface__ = {"shape": (int(v.rows), int(v.ld)), "typestr": "<f4",
                                        "data": (int(v.data), False), "version": 3,
                                        "strides": None}
        return torch.as_tensor(_Arr(), device="cuda")[:, :v.cols].clone()

    def _result_shapes(self):
        out = []
        for which, layers in ((PK_T_W, range(len(self.dims) - 1)), (PK_T_F0, [0])):
            for l in layers:
                v = pk_tensor_view()
                call("pk_engine_tensor", self.h, which, l, C.byref(v))
                out.append((which, l, int(v.rows), int(v.cols)))
        return out

    def prepare_result_buffers(self):
        """Allocate the host buffers of this rank's TrainResult share on a
        helper thread while the GPU trains, and fault their pages in: first
        touch of ~1 GB of fresh host memory costs more than the copy. (Not
        pinned: cudaHostAlloc holds the driver lock and stalls the training
        thread's launches for as long as it runs.)"""
        import threading
        shapes = self._result_shapes()
        self._result_bufs = None

        def alloc():
            bufs = []
            for _, _, r, c in shapes:
                h = np.empty((r, c), np.float32)
                h.fill(0)
                bufs.append(torch.from_numpy(h))
            self._result_bufs = bufs
        self._result_thread = threading.Thread(target=alloc, daemon=True)
        self._result_thread.start()

    def download_params(self):
        """This rank's share of TrainResult (trainer.hpp:636-686): its W
        shards and F0 shard as host numpy arrays (into the pinned buffers of
        prepare_result_buffers when they exist)."""
        t = getattr(self, "_result_thread", None)
        if t is None:
            return [self.tensor(which, l).cpu().numpy()
                    for which, l, _, _ in self._result_shapes()]
        t.join()
        out = []
        jobs = []
        for (which, l, _, _), h in zip(self._result_shapes(), self._result_bufs):
            d = self.tensor(which, l)
            # PK_D2H_THREADS=N copies the big F0 shard as N row chunks, each
            # on its own thread and stream; measured slower than one copy
            # (C2: 86.8 vs 67.6 ms for 8 threads), so 1 by default
            n = _d2h_threads() if h.numel() * 4 >= (64 << 20) else 1
            rows = h.shape[0]
            for i in range(n):
                r0, r1 = rows * i // n, rows * (i + 1) // n
                if r1 > r0:
                    jobs.append((h[r0:r1], d[r0:r1]))
            out.append(h.numpy())
        if len(jobs) <= len(out):
            for h, d in jobs:
                h.copy_(d)
        else:
            import concurrent.futures as cf
            dev = torch.cuda.current_device()

            def run(job):
                h, d = job
                torch.cuda.set_device(dev)
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    h.copy_(d)
                s.synchronize()
            with cf.ThreadPoolExecutor(max_workers=_d2h_threads()) as ex:
                list(ex.map(run, jobs))
        return out

    def forward_only(self):
        """SerialTrainer::forward_only (trainer.hpp:126-135): the forward of
        every layer with the current parameters, no loss / gradients /
        optimizer step; returns this rank's logits block (device tensor)."""
        call("pk_engine_forward_only", self.h)
        return self.tensor(PK_T_FOUT)

    def stream_ptr(self):
        s = C.c_void_p()
        call("pk_engine_stream", self.h, C.byref(s))
        return s.value

    def close(self):
        if getattr(self, "h", None):
            call("pk_engine_destroy", self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def train_single(pre, opts: TrainOptions, epochs=None):
    """train_distributed on grid 1x1x1 (one GPU): per-epoch metrics, final
    weights and features."""
    eng = RankEngine(pre.n, pre.feat_dim, pre.num_classes, GridConfig(1, 1, 1), 0, opts)
    eng.load(pre)
    out = [eng.train_epoch(e) for e in range(opts.epochs if epochs is None else epochs)]
    w = [eng.tensor(PK_T_W, l) for l in range(len(eng.dims) - 1)]
    f0 = eng.tensor(PK_T_F0)
    eng.close()
    return out, w, f0


def gather_rank_pass(engines_or_tensors, grid, n, dims):
    """Reassemble logits / dW / dF0 from per-rank tensors the way the
    reference's engine tests do (test_engine.cpp:30-84). Input: list indexed
    by rank of dicts {fout, dw[list], df0} as numpy arrays."""
    L = len(dims) - 1
    lays = plan_layouts(L)
    last = lays[-1]
    logits = np.zeros((n, dims[-1]), np.float32)
    dw = [np.zeros((dims[l], dims[l + 1]), np.float32) for l in range(L)]
    df0 = np.zeros((n, dims[0]), np.float32)
    from .layout import chunk_start
    for r, t in enumerate(engines_or_tensors):
        c = grid.coords_of(r)
        r0 = chunk_start(n, grid.extent(last.row_shard), c[last.row_shard])
        c0 = chunk_start(dims[-1], grid.extent(last.inner), c[last.inner])
        fo = t["fout"]
        logits[r0:r0 + fo.shape[0], c0:c0 + fo.shape[1]] = fo
        for l in range(L):
            ws = weight_slice(grid, lays[l], c, dims[l], dims[l + 1])
            dw[l][ws[0]:ws[1], ws[2]:ws[3]] = t["dw"][l]
        fs = feature_slice(grid, c, n, dims[0])
        df0[fs[0]:fs[1], fs[2]:fs[3]] = t["df0"]
    return logits, dw, df0


__all__ = ["TrainOptions", "RankEngine", "HostDataset", "train_single", "nccl_unique_id",
           "gather_rank_pass", "PK_MODE_FAST", "PK_MODE_PARITY", "label_row_range"]
