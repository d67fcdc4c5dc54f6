"""Per-rank synthetic shards: one rank's RankTensors (trainer.hpp:217-224)
generated on its own GPU from synth_rmat's indexable Philox streams
(csrc/rank_gen.cu), bit-identical to
    synth_rmat (graph.hpp:291-322) -> preprocess (356-384) ->
    slice_rank_tensors (trainer.hpp:234-250)
without ever building the global graph — the per-rank shard generation a
billion-edge grid needs (the papers-shaped C4).

Global information is two u32 vectors of n: the normalisation degrees and
the label degrees. Each rank counts the nodes of its own ceil-split range
and the vectors are all-gathered (`allgather`, e.g. torch.distributed over
NCCL); with `allgather=None` this process counts every range itself (one
process, or one rank measured alone).
"""

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from . import _capi
from ._capi import call
from .graph import generate_permutation_pair
from ._capi import pk_csr_owned
from .kernels import DeviceCsr
from .layout import (GridConfig, adjacency_block_range, chunk_start, feature_slice,
                     final_output_parity, label_row_range, needed_adjacency_keys)
from .shard_io import RankTensors


class pk_rmat_spec(C.Structure):
    _fields_ = [("scale", C.c_int), ("undirected", C.c_int), ("edges", C.c_uint64),
                ("a", C.c_double), ("b", C.c_double), ("c", C.c_double), ("seed", C.c_uint64)]


_capi.register({
    "pk_rmat_node_degrees": (C.c_int, [C.POINTER(pk_rmat_spec), C.c_int, C.c_int64, C.c_int64,
                                       C.c_void_p, C.c_void_p]),
    "pk_invert_permutation": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "pk_rmat_block": (C.c_int, [C.POINTER(pk_rmat_spec), C.c_int, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_int64,
                                C.c_int64, C.c_int64, C.POINTER(pk_csr_owned), C.c_void_p]),
    "pk_rmat_features_permuted": (C.c_int, [C.c_uint64, C.c_int64, C.c_void_p, C.c_int64,
                                            C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                            C.c_int64, C.c_void_p]),
    "pk_labels_from_degrees": (C.c_int, [C.c_void_p, C.c_int64, C.c_uint32, C.c_void_p,
                                         C.c_void_p]),
    "pk_gather_u32": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
})


@dataclass
class RmatSpec:
    """synth_rmat's inputs (RmatParams, graph.hpp:189-193; feature / class
    counts, seed) plus the dataset orientation and preprocess' perm seed."""
    scale: int
    edges: int
    feat_dim: int
    classes: int
    seed: int = 1
    a: float = 0.57
    b: float = 0.19
    c: float = 0.19
    undirected: bool = True
    perm_seed: Optional[int] = None  # default: the data seed (main.cpp:258)

    @property
    def n(self):
        return 1 << self.scale

    def c_spec(self):
        return pk_rmat_spec(self.scale, int(self.undirected), self.edges, self.a, self.b, self.c,
                            self.seed)


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return C.c_void_p(t.data_ptr())


def node_degrees(spec: RmatSpec, kind: int, node0: int, node1: int) -> torch.Tensor:
    """Degrees of nodes [node0, node1): kind 0 = normalize_adjacency's,
    kind 1 = degree_quantile_labels' (int32 tensor holding u32 bits)."""
    out = torch.empty(max(node1 - node0, 1), dtype=torch.int32, device="cuda")
    call("pk_rmat_node_degrees", C.byref(spec.c_spec()), kind, node0, node1, _p(out), _stream())
    return out[:node1 - node0]


def global_degrees(spec: RmatSpec, kind: int, rank: int, world: int,
                   allgather: Optional[Callable] = None) -> torch.Tensor:
    """All n degrees: this rank's ceil-split range, then `allgather(part,
    counts)` -> the full vector in range order; without it, every range here."""
    n = spec.n
    if allgather is None:
        return torch.cat([node_degrees(spec, kind, chunk_start(n, world, r),
                                       chunk_start(n, world, r + 1)) for r in range(world)])
    part = node_degrees(spec, kind, chunk_start(n, world, rank), chunk_start(n, world, rank + 1))
    counts = [chunk_start(n, world, r + 1) - chunk_start(n, world, r) for r in range(world)]
    return allgather(part, counts)


@dataclass
class GlobalPieces:
    """What every rank shares: the permutation pair (graph.hpp:84-93), its
    inverses, the normalisation degrees and the labels."""
    row_perm: torch.Tensor
    col_perm: torch.Tensor
    inv_row: torch.Tensor
    inv_col: torch.Tensor
    norm_degree: torch.Tensor
    labels: torch.Tensor


def global_pieces(spec: RmatSpec, rank: int = 0, world: int = 1,
                  allgather: Optional[Callable] = None) -> GlobalPieces:
    n = spec.n
    perm_seed = spec.seed if spec.perm_seed is None else spec.perm_seed
    rp, cp = generate_permutation_pair(n, perm_seed)
    dev = lambda a: torch.from_numpy(a.view(np.int32)).cuda()  # noqa: E731
    row_perm, col_perm = dev(rp), dev(cp)
    inv_row = torch.empty_like(row_perm)
    inv_col = torch.empty_like(col_perm)
    call("pk_invert_permutation", _p(row_perm), n, _p(inv_row), _stream())
    call("pk_invert_permutation", _p(col_perm), n, _p(inv_col), _stream())
    norm = global_degrees(spec, 0, rank, world, allgather)
    lab_deg = global_degrees(spec, 1, rank, world, allgather)
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    call("pk_labels_from_degrees", _p(lab_deg), n, spec.classes, _p(labels), _stream())
    del lab_deg
    return GlobalPieces(row_perm, col_perm, inv_row, inv_col, norm, labels)


def rank_block(spec: RmatSpec, g: GlobalPieces, parity: int, r0, r1, c0, c1) -> DeviceCsr:
    """Block [r0, r1) x [c0, c1) of A_even / A_odd, local columns."""
    out = pk_csr_owned()
    call("pk_rmat_block", C.byref(spec.c_spec()), parity, _p(g.row_perm), _p(g.col_perm),
         _p(g.inv_row), _p(g.inv_col), _p(g.norm_degree), r0, r1, c0, c1, C.byref(out),
         _stream())
    return DeviceCsr._from_owned(out)


def generate_rank_tensors(spec: RmatSpec, grid: GridConfig, rank: int, num_layers: int,
                          pieces: Optional[GlobalPieces] = None,
                          allgather: Optional[Callable] = None) -> RankTensors:
    """slice_rank_tensors (trainer.hpp:234-250) of rank `rank`, generated:
    its adjacency blocks per needed (plane, parity) key (blocks of the same
    range and parity are generated once), its F0 slice (feature_slice,
    model.hpp:53-67) and the labels / mask of its logit rows. The mask is
    all ones (synth_rmat's default train_fraction = 1)."""
    n = spec.n
    c = grid.coords_of(rank)
    if pieces is None:
        pieces = global_pieces(spec, rank, grid.size, allgather)
    adj, made = {}, {}
    for plane, parity in needed_adjacency_keys(num_layers):
        r = adjacency_block_range(grid, plane, c, n)
        key = (parity, *r)
        if key not in made:
            made[key] = rank_block(spec, pieces, parity, *r)
        adj[(plane, parity)] = (made[key], None)
    fr0, fr1, fc0, fc1 = feature_slice(grid, c, n, spec.feat_dim)
    f0 = torch.empty((fr1 - fr0, fc1 - fc0), dtype=torch.float32, device="cuda")
    call("pk_rmat_features_permuted", spec.seed, spec.feat_dim, _p(pieces.col_perm), fr0, fr1,
         fc0, fc1, C.c_void_p(f0.data_ptr() if f0.numel() else 0), max(fc1 - fc0, 1), _stream())
    lr0, lr1 = label_row_range(grid, c, n, num_layers)
    perm = pieces.row_perm if final_output_parity(num_layers) == 0 else pieces.col_perm
    labels = torch.empty(max(lr1 - lr0, 1), dtype=torch.int32, device="cuda")
    call("pk_gather_u32", _p(pieces.labels), C.c_void_p(perm.data_ptr() + 4 * lr0), lr1 - lr0,
         _p(labels), _stream())
    return RankTensors(adj=adj, f0=f0, labels=labels[:lr1 - lr0],
                       mask=torch.ones(lr1 - lr0, dtype=torch.uint8, device="cuda"))


__all__ = ["RmatSpec", "GlobalPieces", "global_pieces", "generate_rank_tensors", "rank_block",
           "node_degrees", "global_degrees"]
