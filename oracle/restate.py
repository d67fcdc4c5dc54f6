"""TEST INFRASTRUCTURE ONLY — ctypes view of the C restatement
(``oracle/plexus_oracle.c`` -> ``oracle/_build/liboracle.so``). float32 only.

Each wrapper names the reference function (file:line under
/root/reference/proj/include/plexuskit) that the C code restates.
"""

import ctypes as C
import os

import numpy as np

from . import ORACLE_LIB

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_LIB):
            raise RuntimeError(f"oracle restatement not built: {ORACLE_LIB}")
        _lib = C.CDLL(ORACLE_LIB)
        for n in ("ora_rmat_edges", "ora_normalize_f32", "ora_csr_block_f32"):
            getattr(_lib, n).restype = C.c_uint64
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


U64 = C.c_uint64


def philox_u64(seed, stream, count):
    """rng.hpp:17-104"""
    out = np.empty(count, np.uint64)
    lib().ora_philox_u64(U64(seed), U64(stream), U64(count), _p(out))
    return out


def permutation_pair(n, seed):
    """generate_permutation_pair, graph.hpp:84-93"""
    r, c = np.empty(n, np.uint32), np.empty(n, np.uint32)
    lib().ora_permutation_pair(U64(n), U64(seed), _p(r), _p(c))
    return r, c


def rmat_edges(scale, edges, seed, a=0.57, b=0.19, c=0.19):
    """synth_rmat edge loop, graph.hpp:291-322"""
    uv = np.empty((edges, 2), np.uint32)
    kept = lib().ora_rmat_edges(C.c_int(scale), U64(edges), C.c_double(a), C.c_double(b),
                                C.c_double(c), U64(seed), _p(uv))
    return uv[:kept].copy()


def features(seed, n, d):
    """assemble_synth features, graph.hpp:233-236"""
    out = np.empty((n, d), np.float32)
    lib().ora_features_f32(U64(seed), U64(n * d), _p(out))
    return out


def train_mask(seed, n, train_fraction=1.0):
    """assemble_synth mask, graph.hpp:238-246"""
    out = np.empty(n, np.uint8)
    lib().ora_train_mask(U64(seed), U64(n), C.c_double(train_fraction), _p(out))
    return out


def degree_quantile_labels(edges, n, classes):
    """graph.hpp:197-222"""
    uv = np.ascontiguousarray(edges, np.uint32)
    out = np.empty(n, np.uint32)
    lib().ora_degree_quantile_labels(_p(uv), U64(uv.shape[0]), U64(n), C.c_uint32(classes),
                                     _p(out))
    return out


def synth_rmat(scale, edges, feat, classes, seed, a=0.57, b=0.19, c=0.19,
               train_fraction=1.0):
    """synth_rmat + assemble_synth, graph.hpp:224-322"""
    n = 1 << scale
    uv = rmat_edges(scale, edges, seed, a, b, c)
    return dict(n=n, edges=uv, features=features(seed, n, feat),
                labels=degree_quantile_labels(uv, n, classes), classes=classes,
                mask=train_mask(seed, n, train_fraction))


def chunk_index(total, parts, pos):
    """graph.hpp:151-155 (ceil-split chunk holding pos), vectorised"""
    base, rem = total // parts, total % parts
    pos = np.asarray(pos, np.int64)
    return np.where(pos < rem * (base + 1), pos // (base + 1),
                    rem + (pos - rem * (base + 1)) // max(base, 1))


def sbm_edges(n, communities, p_in, p_out, seed):
    """synth_sbm / synth_erdos edge loop, graph.hpp:254-289: pairs (u, v),
    u < v, in lexicographic order, one next_double() of Philox(seed, 5) each
    (u64 >> 11 scaled by 2^-53), kept below p_in (same community) or p_out.
    Small n only (all n(n-1)/2 draws are materialised)."""
    u, v = np.triu_indices(n, k=1)
    r = (philox_u64(seed, 5, u.size) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    same = chunk_index(n, communities, u) == chunk_index(n, communities, v)
    keep = r < np.where(same, p_in, p_out)
    return np.stack([u[keep], v[keep]], 1).astype(np.uint32)


def synth_sbm(n, communities, p_in, p_out, feat, classes, seed, train_fraction=1.0):
    """synth_sbm + assemble_synth, graph.hpp:224-274"""
    uv = sbm_edges(n, communities, p_in, p_out, seed)
    return dict(n=n, edges=uv, features=features(seed, n, feat),
                labels=degree_quantile_labels(uv, n, classes), classes=classes,
                mask=train_mask(seed, n, train_fraction))


def synth_erdos(n, p, feat, classes, seed, train_fraction=1.0):
    """synth_erdos + assemble_synth, graph.hpp:224-249, 276-289 (one community)"""
    return synth_sbm(n, 1, p, p, feat, classes, seed, train_fraction)


def normalize(n, edges, undirected=True):
    """normalize_adjacency, graph.hpp:40-76"""
    uv = np.ascontiguousarray(edges, np.uint32)
    nnz = lib().ora_normalize_f32(U64(n), _p(uv), U64(uv.shape[0]), C.c_int(int(undirected)),
                                  None, None, None)
    rp, ci, v = np.empty(n + 1, np.uint64), np.empty(nnz, np.uint32), np.empty(nnz, np.float32)
    lib().ora_normalize_f32(U64(n), _p(uv), U64(uv.shape[0]), C.c_int(int(undirected)),
                            _p(rp), _p(ci), _p(v))
    return rp, ci, v


def csr_transpose(rows, cols, rp, ci, v):
    """CsrMatrix::transpose, csr.hpp:78-95"""
    nnz = int(rp[rows])
    orp, oci, ov = (np.empty(cols + 1, np.uint64), np.empty(nnz, np.uint32),
                    np.empty(nnz, np.float32))
    lib().ora_csr_transpose_f32(U64(rows), U64(cols), _p(np.ascontiguousarray(rp, np.uint64)),
                                _p(np.ascontiguousarray(ci, np.uint32)),
                                _p(np.ascontiguousarray(v, np.float32)), _p(orp), _p(oci),
                                _p(ov))
    return orp, oci, ov


def csr_block(rp, ci, v, r0, r1, c0, c1):
    """CsrMatrix::block, csr.hpp:97-120"""
    rp = np.ascontiguousarray(rp, np.uint64)
    ci = np.ascontiguousarray(ci, np.uint32)
    v = np.ascontiguousarray(v, np.float32)
    orp = np.empty(r1 - r0 + 1, np.uint64)
    nnz = lib().ora_csr_block_f32(_p(rp), _p(ci), _p(v), U64(r0), U64(r1), U64(c0), U64(c1),
                                  _p(orp), None, None)
    oci, ov = np.empty(nnz, np.uint32), np.empty(nnz, np.float32)
    lib().ora_csr_block_f32(_p(rp), _p(ci), _p(v), U64(r0), U64(r1), U64(c0), U64(c1),
                            _p(orp), _p(oci), _p(ov))
    return orp, oci, ov


def permute_csr(n, rp, ci, v, row_perm, col_perm):
    """permute_csr, graph.hpp:101-131"""
    nnz = int(rp[n])
    orp, oci, ov = np.empty(n + 1, np.uint64), np.empty(nnz, np.uint32), np.empty(nnz, np.float32)
    lib().ora_permute_csr_f32(U64(n), _p(np.ascontiguousarray(rp, np.uint64)),
                              _p(np.ascontiguousarray(ci, np.uint32)),
                              _p(np.ascontiguousarray(v, np.float32)),
                              _p(np.ascontiguousarray(row_perm, np.uint32)),
                              _p(np.ascontiguousarray(col_perm, np.uint32)),
                              _p(orp), _p(oci), _p(ov))
    return orp, oci, ov


def preprocess(ds, perm_seed):
    """preprocess, graph.hpp:356-384"""
    n = ds["n"]
    a = normalize(n, ds["edges"], ds.get("undirected", True))
    rperm, cperm = permutation_pair(n, perm_seed)
    even = permute_csr(n, *a, rperm, cperm)
    odd = permute_csr(n, *a, cperm, rperm)
    return dict(n=n, classes=ds["classes"], even=even, odd=odd,
                features=np.ascontiguousarray(ds["features"][cperm]),
                labels_row=ds["labels"][rperm], labels_col=ds["labels"][cperm],
                mask_row=ds["mask"][rperm], mask_col=ds["mask"][cperm],
                row_perm=rperm, col_perm=cperm)


def spmm_rows(rp, ci, v, x, r0, r1):
    """spmm_rows, kernels.hpp:39-62"""
    x = np.ascontiguousarray(x, np.float32)
    out = np.empty((r1 - r0, x.shape[1]), np.float32)
    lib().ora_spmm_rows_f32(_p(np.ascontiguousarray(rp, np.uint64)),
                            _p(np.ascontiguousarray(ci, np.uint32)),
                            _p(np.ascontiguousarray(v, np.float32)), _p(x),
                            U64(x.shape[1]), U64(r0), U64(r1), _p(out))
    return out


def gemm(a, b, ta=False, tb=False):
    """gemm, kernels.hpp:64-92"""
    a = np.ascontiguousarray(a, np.float32)
    b = np.ascontiguousarray(b, np.float32)
    m = a.shape[1] if ta else a.shape[0]
    n = b.shape[0] if tb else b.shape[1]
    out = np.empty((m, n), np.float32)
    lib().ora_gemm_f32(_p(a), U64(a.shape[0]), U64(a.shape[1]), _p(b), U64(b.shape[0]),
                       U64(b.shape[1]), C.c_int(int(ta)), C.c_int(int(tb)), _p(out))
    return out


def relu_forward(q):
    """kernels.hpp:94-100"""
    q = np.ascontiguousarray(q, np.float32)
    out = np.empty_like(q)
    lib().ora_relu_forward_f32(_p(q), U64(q.size), _p(out))
    return out


def relu_backward(q, df):
    """kernels.hpp:102-111"""
    q = np.ascontiguousarray(q, np.float32)
    df = np.ascontiguousarray(df, np.float32)
    out = np.empty_like(q)
    lib().ora_relu_backward_f32(_p(q), _p(df), U64(q.size), _p(out))
    return out


def ce_sums(logits, labels, mask):
    """softmax_cross_entropy_sums, kernels.hpp:117-158"""
    logits = np.ascontiguousarray(logits, np.float32)
    ls, cnt, cor = C.c_double(), U64(), U64()
    d = np.empty_like(logits)
    rc = lib().ora_ce_sums_f32(_p(logits), U64(logits.shape[0]), U64(logits.shape[1]),
                               _p(np.ascontiguousarray(labels, np.uint32)),
                               _p(np.ascontiguousarray(mask, np.uint8)), C.byref(ls),
                               C.byref(cnt), C.byref(cor), _p(d))
    if rc:
        raise ValueError("cross entropy: label out of range")
    return ls.value, cnt.value, cor.value, d


def adam_step(p, g, m, v, step, lr=1e-2, b1=0.9, b2=0.999, eps=1e-8):
    """adam_step, model.hpp:88-111 (in place; `step` = count after increment)"""
    lib().ora_adam_f32(_p(p), _p(np.ascontiguousarray(g, np.float32)), _p(m), _p(v),
                       U64(p.size), U64(step), C.c_double(lr), C.c_double(b1),
                       C.c_double(b2), C.c_double(eps))


def init_weights(dims, seed):
    """init_weights, model.hpp:17-33"""
    d = np.asarray(dims, np.uint64)
    out = np.empty(sum(dims[l] * dims[l + 1] for l in range(len(dims) - 1)), np.float32)
    lib().ora_init_weights_f32(_p(d), C.c_int(len(dims)), U64(seed), _p(out))
    res, off = [], 0
    for l in range(len(dims) - 1):
        sz = dims[l] * dims[l + 1]
        res.append(out[off:off + sz].reshape(dims[l], dims[l + 1]))
        off += sz
    return res


def serial_forward_backward(pre, weights):
    """SerialTrainer::forward_backward, trainer.hpp:137-169"""
    n = pre["n"]
    dims = [weights[0].shape[0]] + [w.shape[1] for w in weights]
    d = np.asarray(dims, np.uint64)
    et = csr_transpose(n, n, *pre["even"])
    ot = csr_transpose(n, n, *pre["odd"])
    w_cat = np.concatenate([np.ascontiguousarray(w, np.float32).ravel() for w in weights])
    L = len(weights)
    parity = (L - 1) % 2
    labels = pre["labels_row"] if parity == 0 else pre["labels_col"]
    mask = pre["mask_row"] if parity == 0 else pre["mask_col"]
    loss, acc = C.c_double(), C.c_double()
    logits = np.empty((n, dims[-1]), np.float32)
    dw = np.empty_like(w_cat)
    df0 = np.empty((n, dims[0]), np.float32)
    arrs = [np.ascontiguousarray(a) for a in (*pre["even"], *pre["odd"], *et, *ot)]
    rc = lib().ora_serial_forward_backward_f32(
        U64(n), _p(d), C.c_int(len(dims)), *[_p(a) for a in arrs],
        _p(np.ascontiguousarray(pre["features"], np.float32)), _p(w_cat),
        _p(np.ascontiguousarray(labels, np.uint32)), _p(np.ascontiguousarray(mask, np.uint8)),
        C.byref(loss), C.byref(acc), _p(logits), _p(dw), _p(df0))
    if rc:
        raise RuntimeError(f"serial forward_backward failed rc={rc}")
    dws, off = [], 0
    for l in range(L):
        sz = dims[l] * dims[l + 1]
        dws.append(dw[off:off + sz].reshape(dims[l], dims[l + 1]))
        off += sz
    return dict(loss=loss.value, accuracy=acc.value, logits=logits, dw=dws, df0=df0)
