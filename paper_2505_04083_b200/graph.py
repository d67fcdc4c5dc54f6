"""Host mirror of the reference's graph preprocessing and shard builder
(graph.hpp, csr.hpp:78-120), running on the GPU through the C ABI.

Everything here is bit-exact with the reference: RMAT edges, features and
labels (graph.hpp:197-322), normalize_adjacency (40-76), the permutation pair
(84-93), permute_csr (101-131), preprocess (356-384), CSR transpose / block.
"""

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from ._capi import ContractError, call, pk_csr_owned
from .kernels import DeviceCsr, _ptr, _stream

__all__ = ["csr_transpose", "csr_block", "normalize_adjacency", "permute_csr",
           "generate_permutation_pair", "invert_permutation", "synth_rmat", "preprocess",
           "GraphDataset", "PreprocessedDataset", "balance_metric"]


def _owned_call(name, *args):
    out = pk_csr_owned()
    call(name, *args, C.byref(out), _stream())
    return DeviceCsr._from_owned(out)


def csr_transpose(a: DeviceCsr) -> DeviceCsr:
    """CsrMatrix::transpose (csr.hpp:78-95)."""
    return _owned_call("pk_csr_transpose", a.view())


def csr_block(a: DeviceCsr, r0, r1, c0, c1) -> DeviceCsr:
    """CsrMatrix::block (csr.hpp:97-120)."""
    if not (0 <= r0 <= r1 <= a.rows and 0 <= c0 <= c1 <= a.cols):
        raise ContractError("csr block: range out of bounds")
    return _owned_call("pk_csr_block", a.view(), r0, r1, c0, c1)


def normalize_adjacency(n, edges: torch.Tensor, undirected=True) -> DeviceCsr:
    """normalize_adjacency (graph.hpp:40-76); edges is an (m, 2) int32 CUDA
    tensor holding u32 endpoints."""
    e = edges.contiguous()
    return _owned_call("pk_normalize_adjacency", n, _ptr(e), e.shape[0], int(undirected))


def permute_csr(a: DeviceCsr, row_perm: torch.Tensor, col_perm: torch.Tensor) -> DeviceCsr:
    """permute_csr (graph.hpp:101-131): result[i, j] = a[row_perm[i], col_perm[j]]."""
    if a.rows != a.cols:
        raise ContractError("permute_csr: matrix must be square")
    if row_perm.numel() != a.rows or col_perm.numel() != a.cols:
        raise ContractError("permute_csr: permutation length mismatch")
    return _owned_call("pk_permute_csr", a.view(), _ptr(row_perm), _ptr(col_perm))


def generate_permutation_pair(n, seed):
    """generate_permutation_pair (graph.hpp:84-93): host Fisher-Yates on the
    Philox streams 1 and 2 (sequential by definition). Returns numpy u32."""
    if n < 1:
        raise ContractError("generate_permutation_pair: n must be >= 1")
    r, c = np.empty(n, np.uint32), np.empty(n, np.uint32)
    call("pk_permutation_pair_host", n, seed, r.ctypes.data_as(C.c_void_p),
         c.ctypes.data_as(C.c_void_p))
    return r, c


def invert_permutation(p):
    inv = np.empty_like(p)
    inv[p] = np.arange(p.size, dtype=p.dtype)
    return inv


@dataclass
class GraphDataset:
    """GraphDataset<float> (graph.hpp:19-38) with device arrays."""
    num_nodes: int
    edges: torch.Tensor          # (m, 2) int32 (u32 bits), may contain duplicates
    features: torch.Tensor       # (n, D0) float32
    labels: torch.Tensor         # (n,) int32 (u32 bits)
    num_classes: int
    train_mask: torch.Tensor     # (n,) uint8
    undirected: bool = True


def synth_rmat(scale, edges, feat_dim, classes, seed, a=0.57, b=0.19, c=0.19,
               train_fraction=1.0, device="cuda") -> GraphDataset:
    """synth_rmat (graph.hpp:291-322) + assemble_synth (224-249) on the GPU."""
    if not (1 <= scale < 31):
        raise ContractError("rmat: scale out of range")
    if not (a > 0 and b >= 0 and c >= 0 and a + b + c < 1.0):
        raise ContractError("rmat: quadrant probabilities must sum below 1")
    if classes < 1:
        raise ContractError("synth: need at least one class")
    n = 1 << scale
    target = edges if edges else 8 * n
    uv = torch.empty((target, 2), dtype=torch.int32, device=device)
    kept = C.c_uint64()
    call("pk_rmat_edges", scale, target, a, b, c, seed, _ptr(uv), C.byref(kept), _stream())
    uv = uv[:kept.value]
    feats = torch.empty((n, feat_dim), dtype=torch.float32, device=device)
    call("pk_rmat_features", seed, n, feat_dim, _ptr(feats), feat_dim, _stream())
    labels = torch.empty(n, dtype=torch.int32, device=device)
    call("pk_degree_quantile_labels", _ptr(uv), uv.shape[0], n, classes, _ptr(labels),
         _stream())
    if train_fraction < 1.0:
        # stream 4 mask (graph.hpp:238-246) is sequential and tiny: host side
        mask = _host_mask(seed, n, train_fraction)
        mask_t = torch.from_numpy(mask).to(device)
    else:
        mask_t = torch.ones(n, dtype=torch.uint8, device=device)
    return GraphDataset(n, uv, feats, labels, classes, mask_t, True)


def _assemble(n, uv, feat_dim, classes, seed, train_fraction, device):
    """assemble_synth (graph.hpp:224-249) on the device: Philox(seed, 3)
    features, degree-quantile labels, Philox(seed, 4) training mask."""
    if classes < 1:
        raise ContractError("synth: need at least one class")
    feats = torch.empty((n, feat_dim), dtype=torch.float32, device=device)
    call("pk_rmat_features", seed, n, feat_dim, _ptr(feats), feat_dim, _stream())
    labels = torch.empty(n, dtype=torch.int32, device=device)
    call("pk_degree_quantile_labels", _ptr(uv), uv.shape[0], n, classes, _ptr(labels),
         _stream())
    if train_fraction < 1.0:
        mask_t = torch.from_numpy(_host_mask(seed, n, train_fraction)).to(device)
    else:
        mask_t = torch.ones(n, dtype=torch.uint8, device=device)
    return GraphDataset(n, uv, feats, labels, classes, mask_t, True)


def _pair_graph(fn, args, n, feat_dim, classes, seed, train_fraction, device):
    if classes < 1:
        raise ContractError("synth: need at least one class")
    cnt = C.c_uint64()
    call(fn, *args, seed, None, 0, C.byref(cnt), _stream())
    uv = torch.empty((max(cnt.value, 1), 2), dtype=torch.int32, device=device)
    call(fn, *args, seed, _ptr(uv), cnt.value, C.byref(cnt), _stream())
    return _assemble(n, uv[:cnt.value], feat_dim, classes, seed, train_fraction, device)


def synth_sbm(n, communities, p_in, p_out, feat_dim, classes, seed, train_fraction=1.0,
              device="cuda") -> GraphDataset:
    """synth_sbm (graph.hpp:254-274) + assemble_synth on the GPU: bit-exact
    with the reference (edge order included)."""
    return _pair_graph("pk_sbm_edges", (n, communities, p_in, p_out), n, feat_dim, classes,
                       seed, train_fraction, device)


def synth_erdos(n, p, feat_dim, classes, seed, train_fraction=1.0,
                device="cuda") -> GraphDataset:
    """synth_erdos (graph.hpp:276-289) + assemble_synth on the GPU."""
    return _pair_graph("pk_erdos_edges", (n, p), n, feat_dim, classes, seed, train_fraction,
                       device)


def _host_mask(seed, n, frac):
    # Philox(seed, 4).next_double() < frac per node; never empty.
    from .philox import philox_doubles
    d = philox_doubles(seed, 4, n)
    m = (d < frac).astype(np.uint8)
    if not m.any():
        m[0] = 1
    return m


@dataclass
class PreprocessedDataset:
    """PreprocessedDataset<float> (graph.hpp:327-350), device resident."""
    n: int
    feat_dim: int
    num_classes: int
    perm_seed: int
    a_even: DeviceCsr
    a_odd: DeviceCsr
    features: torch.Tensor      # col_perm order
    labels_row_order: torch.Tensor
    labels_col_order: torch.Tensor
    mask_row_order: torch.Tensor
    mask_col_order: torch.Tensor
    row_perm: np.ndarray = field(default=None, repr=False)
    col_perm: np.ndarray = field(default=None, repr=False)

    def labels_for_parity(self, parity):
        return self.labels_row_order if parity == 0 else self.labels_col_order

    def mask_for_parity(self, parity):
        return self.mask_row_order if parity == 0 else self.mask_col_order


def preprocess(ds: GraphDataset, perm_seed) -> PreprocessedDataset:
    """preprocess (graph.hpp:356-384): normalize, double permutation,
    attribute alignment — all on the device except Fisher-Yates."""
    a = normalize_adjacency(ds.num_nodes, ds.edges, ds.undirected)
    rperm, cperm = generate_permutation_pair(ds.num_nodes, perm_seed)
    dev = ds.features.device
    rp = torch.from_numpy(rperm.view(np.int32)).to(dev)
    cp = torch.from_numpy(cperm.view(np.int32)).to(dev)
    even = permute_csr(a, rp, cp)
    odd = permute_csr(a, cp, rp)
    del a
    # attribute alignment (graph.hpp:373-380): library gathers, so a C++
    # caller can run the whole preprocess through the ABI
    n, d0 = ds.num_nodes, ds.features.shape[1]
    feats = torch.empty((n, d0), dtype=torch.float32, device=dev)
    f_src = ds.features.contiguous()
    call("pk_gather_rows_f32", _ptr(f_src), d0, _ptr(cp), n, d0, _ptr(feats), d0, _stream())
    lab = ds.labels.contiguous()
    msk = ds.train_mask.contiguous()
    out = {}
    for name, perm in (("row", rp), ("col", cp)):
        lo = torch.empty(n, dtype=torch.int32, device=dev)
        mo = torch.empty(n, dtype=torch.uint8, device=dev)
        call("pk_gather_u32", _ptr(lab), _ptr(perm), n, _ptr(lo), _stream())
        call("pk_gather_u8", _ptr(msk), _ptr(perm), n, _ptr(mo), _stream())
        out[name] = (lo, mo)
    return PreprocessedDataset(
        n=n, feat_dim=d0, num_classes=ds.num_classes,
        perm_seed=perm_seed, a_even=even, a_odd=odd, features=feats,
        labels_row_order=out["row"][0], labels_col_order=out["col"][0],
        mask_row_order=out["row"][1], mask_col_order=out["col"][1],
        row_perm=rperm, col_perm=cperm)


def balance_metric(a: DeviceCsr, p, q):
    """balance_metric (graph.hpp:157-172): max/mean nnz over a p x q
    ceil-split block partition, counted on the device (pk_balance_metric)."""
    out = C.c_double()
    call("pk_balance_metric", a.view(), p, q, C.byref(out), _stream())
    return out.value
