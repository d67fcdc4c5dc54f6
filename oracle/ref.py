"""TEST INFRASTRUCTURE ONLY — ctypes view of the compiled reference
(``oracle/_ref/libplexus_ref.so``, built from the unmodified
/root/reference/proj sources by oracle/Makefile; shim in ref_capi.cpp).

Arrays are numpy; scalar type float32 unless ``f64=True``.
"""

import ctypes as C
import os

import numpy as np

from . import REF_LIB

_u64p = C.POINTER(C.c_uint64)
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(REF_LIB):
            raise RuntimeError(f"reference oracle not built: {REF_LIB}")
        _lib = C.CDLL(REF_LIB)
        _lib.ref_last_error.restype = C.c_char_p
        for name in ("ref_synth_rmat", "ref_synth_sbm", "ref_synth_erdos", "ref_graph_from_arrays",
                     "ref_normalize", "ref_csr_from_arrays", "ref_csr_transpose",
                     "ref_csr_block", "ref_permute_csr", "ref_preprocess",
                     "ref_pre_csr", "ref_pre_from_arrays", "ref_serial_create"):
            getattr(_lib, name).restype = C.c_void_p
        _lib.ref_synth_rmat.argtypes = [C.c_int, C.c_uint64, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, C.c_uint32, C.c_uint64,
                                        C.c_double, C.c_int]
        _lib.ref_synth_sbm.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double,
                                       C.c_uint64, C.c_uint32, C.c_uint64, C.c_double,
                                       C.c_int]
        _lib.ref_synth_erdos.argtypes = [C.c_uint64, C.c_double, C.c_uint64, C.c_uint32,
                                         C.c_uint64, C.c_double, C.c_int]
        _lib.ref_balance_metric.restype = C.c_double
        _lib.ref_balance_metric.argtypes = [C.c_void_p, C.c_int, C.c_int]
        _lib.ref_predict_comm.restype = C.c_double
        for name in ("ref_graph_free", "ref_csr_free", "ref_pre_free", "ref_serial_free"):
            getattr(_lib, name).argtypes = [C.c_void_p]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _dt(f64):
    return np.float64 if f64 else np.float32


def _check(rc):
    if rc != 0:
        raise RuntimeError(lib().ref_last_error().decode())


class _Handle:
    _free = None

    def __init__(self, h, f64):
        if not h:
            raise RuntimeError(lib().ref_last_error().decode())
        self.h = C.c_void_p(h)
        self.f64 = f64

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            getattr(_lib, self._free)(self.h)
            self.h = None


class Graph(_Handle):
    _free = "ref_graph_free"

    def info(self):
        n, e, f = C.c_uint64(), C.c_uint64(), C.c_uint64()
        c = C.c_uint32()
        lib().ref_graph_info(self.h, C.byref(n), C.byref(e), C.byref(f), C.byref(c))
        return n.value, e.value, f.value, c.value

    def arrays(self):
        n, e, f, _ = self.info()
        uv = np.empty((e, 2), np.uint32)
        feats = np.empty((n, f), _dt(self.f64))
        labels = np.empty(n, np.uint32)
        mask = np.empty(n, np.uint8)
        lib().ref_graph_copy(self.h, _p(uv), _p(feats), _p(labels), _p(mask))
        return dict(edges=uv, features=feats, labels=labels, mask=mask)

    def set_undirected(self, undirected: bool):
        lib().ref_graph_set_undirected(self.h, C.c_int(int(undirected)))

    def normalize(self):
        return Csr(lib().ref_normalize(self.h), self.f64)

    def preprocess(self, perm_seed):
        return Pre(lib().ref_preprocess(self.h, C.c_uint64(perm_seed)), self.f64)


class Csr(_Handle):
    _free = "ref_csr_free"

    @classmethod
    def from_arrays(cls, rows, cols, rp, ci, vals):
        f64 = vals.dtype == np.float64
        rp = np.ascontiguousarray(rp, np.uint64)
        ci = np.ascontiguousarray(ci, np.uint32)
        vals = np.ascontiguousarray(vals)
        return cls(lib().ref_csr_from_arrays(C.c_uint64(rows), C.c_uint64(cols), _p(rp),
                                             _p(ci), _p(vals), C.c_int(int(f64))), f64)

    def info(self):
        r, c, z = C.c_uint64(), C.c_uint64(), C.c_uint64()
        lib().ref_csr_info(self.h, C.byref(r), C.byref(c), C.byref(z))
        return r.value, c.value, z.value

    def arrays(self):
        r, _, z = self.info()
        rp = np.empty(r + 1, np.uint64)
        ci = np.empty(z, np.uint32)
        v = np.empty(z, _dt(self.f64))
        lib().ref_csr_copy(self.h, _p(rp), _p(ci), _p(v))
        return rp, ci, v

    def transpose(self):
        return Csr(lib().ref_csr_transpose(self.h), self.f64)

    def block(self, r0, r1, c0, c1):
        return Csr(lib().ref_csr_block(self.h, *[C.c_uint64(x) for x in (r0, r1, c0, c1)]),
                   self.f64)

    def permute(self, row_perm, col_perm):
        rp = np.ascontiguousarray(row_perm, np.uint32)
        cp = np.ascontiguousarray(col_perm, np.uint32)
        return Csr(lib().ref_permute_csr(self.h, _p(rp), _p(cp)), self.f64)

    def balance(self, p, q):
        return lib().ref_balance_metric(self.h, p, q)

    def spmm_rows(self, x, r0=None, r1=None):
        rows, cols, _ = self.info()
        r0 = 0 if r0 is None else r0
        r1 = rows if r1 is None else r1
        x = np.ascontiguousarray(x, _dt(self.f64))
        out = np.empty((r1 - r0, x.shape[1]), x.dtype)
        fl = C.c_uint64(0)
        _check(lib().ref_spmm_h(self.h, _p(x), C.c_uint64(x.shape[0]), C.c_uint64(x.shape[1]),
                                C.c_uint64(r0), C.c_uint64(r1), _p(out), C.byref(fl)))
        return out, fl.value


class Pre(_Handle):
    _free = "ref_pre_free"

    @classmethod
    def from_arrays(cls, n, feat, classes, even, odd, features, labels_row, labels_col,
                    mask_row, mask_col):
        f64 = features.dtype == np.float64
        ep, ei, ev = [np.ascontiguousarray(a) for a in even]
        op, oi, ov = [np.ascontiguousarray(a) for a in odd]
        arrs = [np.ascontiguousarray(a) for a in (features, labels_row, labels_col,
                                                  mask_row, mask_col)]
        h = lib().ref_pre_from_arrays(C.c_uint64(n), C.c_uint64(feat), C.c_uint32(classes),
                                      _p(ep), _p(ei), _p(ev), _p(op), _p(oi), _p(ov),
                                      *[_p(a) for a in arrs], C.c_int(int(f64)))
        return cls(h, f64)

    def info(self):
        n, f, ne, no = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        c = C.c_uint32()
        lib().ref_pre_info(self.h, C.byref(n), C.byref(f), C.byref(c), C.byref(ne),
                           C.byref(no))
        return dict(n=n.value, feat=f.value, classes=c.value, nnz_even=ne.value,
                    nnz_odd=no.value)

    def csr(self, parity):
        return Csr(lib().ref_pre_csr(self.h, C.c_int(parity)), self.f64)

    def arrays(self):
        i = self.info()
        n = i["n"]
        feats = np.empty((n, i["feat"]), _dt(self.f64))
        lr, lc = np.empty(n, np.uint32), np.empty(n, np.uint32)
        mr, mc = np.empty(n, np.uint8), np.empty(n, np.uint8)
        lib().ref_pre_copy(self.h, _p(feats), _p(lr), _p(lc), _p(mr), _p(mc))
        return dict(features=feats, labels_row=lr, labels_col=lc, mask_row=mr, mask_col=mc)

    def serial(self, hidden=(128, 128), seed=0, epochs=10, lr=1e-2):
        return Serial(self, hidden, seed, epochs, lr)

    def train_distributed(self, grid, hidden=(128, 128), seed=0, epochs=10, lr=1e-2,
                          block_count=0, fault_epoch=-1, max_running=0, params=False):
        i = self.info()
        dims = [i["feat"], *hidden, i["classes"]]
        hid = np.asarray(hidden, np.uint64)
        losses, accs = np.empty(epochs), np.empty(epochs)
        phase = np.empty((epochs, 5))
        flops = np.empty((epochs, 2), np.uint64)
        byts = np.empty((epochs, 3))
        w = f = None
        if params:
            w = np.empty(sum(dims[l] * dims[l + 1] for l in range(len(dims) - 1)),
                         _dt(self.f64))
            f = np.empty((i["n"], i["feat"]), _dt(self.f64))
        _check(lib().ref_train_distributed(
            self.h, *[C.c_int(g) for g in grid], _p(hid), C.c_int(len(hidden)),
            C.c_uint64(seed), C.c_int(epochs), C.c_double(lr), C.c_int(block_count),
            C.c_int(fault_epoch), C.c_int(max_running), _p(losses), _p(accs), _p(phase),
            _p(flops), _p(byts), _p(w), _p(f)))
        out = dict(loss=losses, accuracy=accs, phase_s=phase, flops=flops, bytes=byts)
        if params:
            out["weights"] = split_weights(w, dims)
            out["features"] = f
        return out

    def epoch_sample(self, hidden, rows, threads):
        """ref_epoch_sample: (estimated full-epoch seconds, sampled wall seconds)."""
        hid = np.asarray(hidden, np.uint64)
        out = np.zeros(2)
        _check(lib().ref_epoch_sample(self.h, _p(hid), C.c_int(len(hidden)), C.c_uint64(rows),
                                      C.c_int(threads), _p(out)))
        return float(out[0]), float(out[1])

    def serial_pass_parallel(self, hidden, threads, seed=0, want_h0=False, sample_cols=0):
        """SerialTrainer::forward_backward(0) composed from the reference
        kernels over `threads` row blocks (ref_serial_pass_parallel): rows
        bitwise the serial pass's, the CE loss sum reduced blockwise, dW in
        float64 (the reference gemm at T = double)."""
        i = self.info()
        dims = [i["feat"], *hidden, i["classes"]]
        n = i["n"]
        hid = np.asarray(hidden, np.uint64)
        loss, acc = C.c_double(), C.c_double()
        logits = np.empty((n, dims[-1]), np.float32)
        dw = np.empty(sum(dims[l] * dims[l + 1] for l in range(len(dims) - 1)), np.float64)
        df0 = np.empty((n, dims[0]), np.float32)
        h0 = np.empty((n, dims[0]), np.float32) if want_h0 else None
        L = len(dims) - 1
        dmax = max(dims)
        dws = np.zeros((L, dmax, sample_cols), np.float32) if sample_cols else None
        _check(lib().ref_serial_pass_parallel(
            self.h, _p(hid), C.c_int(len(hidden)), C.c_uint64(seed), C.c_int(threads),
            C.byref(loss), C.byref(acc), _p(logits), _p(dw), _p(df0), _p(h0),
            C.c_int(sample_cols), _p(dws)))
        out = dict(loss=loss.value, accuracy=acc.value, logits=logits,
                   dw=split_weights(dw, dims), df0=df0, h0=h0)
        if sample_cols:
            # serial fp32 chain dW[:, :sample_cols] per layer
            out["dw_serial_cols"] = [dws[l, :dims[l], :min(sample_cols, dims[l + 1])]
                                     for l in range(L)]
        return out

    def distributed_pass(self, grid, hidden=(128, 128), seed=0, block_count=0):
        i = self.info()
        dims = [i["feat"], *hidden, i["classes"]]
        hid = np.asarray(hidden, np.uint64)
        dt = _dt(self.f64)
        loss, acc = C.c_double(), C.c_double()
        logits = np.empty((i["n"], dims[-1]), dt)
        dw = np.empty(sum(dims[l] * dims[l + 1] for l in range(len(dims) - 1)), dt)
        df0 = np.empty((i["n"], dims[0]), dt)
        flops = np.empty(2, np.uint64)
        g = grid[0] * grid[1] * grid[2]
        comm = np.empty((g, 3, 3, 2))
        _check(lib().ref_distributed_pass(
            self.h, *[C.c_int(g) for g in grid], _p(hid), C.c_int(len(hidden)),
            C.c_uint64(seed), C.c_int(block_count), C.byref(loss), C.byref(acc),
            _p(logits), _p(dw), _p(df0), _p(flops), _p(comm)))
        return dict(loss=loss.value, accuracy=acc.value, logits=logits,
                    dw=split_weights(dw, dims), df0=df0, flops=flops,
                    comm_calls=comm[..., 0], comm_bytes=comm[..., 1])


def split_weights(cat, dims):
    out, off = [], 0
    for l in range(len(dims) - 1):
        sz = dims[l] * dims[l + 1]
        out.append(cat[off:off + sz].reshape(dims[l], dims[l + 1]))
        off += sz
    return out


class Serial(_Handle):
    _free = "ref_serial_free"

    def __init__(self, pre, hidden, seed, epochs, lr):
        i = pre.info()
        self.pre = pre
        self.dims = [i["feat"], *hidden, i["classes"]]
        self.n = i["n"]
        hid = np.asarray(hidden, np.uint64)
        super().__init__(lib().ref_serial_create(pre.h, _p(hid), C.c_int(len(hidden)),
                                                 C.c_uint64(seed), C.c_int(epochs),
                                                 C.c_double(lr)), pre.f64)

    def forward_backward(self, epoch=0):
        dt = _dt(self.f64)
        d = self.dims
        loss, acc = C.c_double(), C.c_double()
        logits = np.empty((self.n, d[-1]), dt)
        dw = np.empty(sum(d[l] * d[l + 1] for l in range(len(d) - 1)), dt)
        df0 = np.empty((self.n, d[0]), dt)
        sf, gf = C.c_uint64(), C.c_uint64()
        _check(lib().ref_serial_forward_backward(self.h, C.c_int(epoch), C.byref(loss),
                                                 C.byref(acc), _p(logits), _p(dw), _p(df0),
                                                 C.byref(sf), C.byref(gf)))
        return dict(loss=loss.value, accuracy=acc.value, logits=logits,
                    dw=split_weights(dw, d), df0=df0, spmm_flops=sf.value,
                    gemm_flops=gf.value)

    def forward_only(self):
        logits = np.empty((self.n, self.dims[-1]), _dt(self.f64))
        _check(lib().ref_serial_forward_only(self.h, _p(logits)))
        return logits

    def train(self, epochs):
        losses, accs = np.empty(epochs), np.empty(epochs)
        _check(lib().ref_serial_train(self.h, C.c_int(epochs), _p(losses), _p(accs)))
        return losses, accs

    def params(self):
        d = self.dims
        dt = _dt(self.f64)
        w = np.empty(sum(d[l] * d[l + 1] for l in range(len(d) - 1)), dt)
        f = np.empty((self.n, d[0]), dt)
        lib().ref_serial_params(self.h, _p(w), _p(f))
        return split_weights(w, d), f


# --------------------------------------------------------------------------
# free functions

def synth_rmat(scale, edges, feat, classes, seed, a=0.57, b=0.19, c=0.19,
               train_fraction=1.0, f64=False):
    return Graph(lib().ref_synth_rmat(scale, edges, a, b, c, feat, classes, seed,
                                      train_fraction, int(f64)), f64)


def synth_sbm(n, communities, p_in, p_out, feat, classes, seed, train_fraction=1.0,
              f64=False):
    return Graph(lib().ref_synth_sbm(n, communities, p_in, p_out, feat, classes, seed,
                                     train_fraction, int(f64)), f64)


def synth_erdos(n, p, feat, classes, seed, train_fraction=1.0, f64=False):
    return Graph(lib().ref_synth_erdos(n, p, feat, classes, seed, train_fraction, int(f64)), f64)


def graph_from_arrays(n, edges, features, labels, classes, mask, undirected=True):
    f64 = features.dtype == np.float64
    uv = np.ascontiguousarray(edges, np.uint32)
    features = np.ascontiguousarray(features)
    labels = np.ascontiguousarray(labels, np.uint32)
    mask = np.ascontiguousarray(mask, np.uint8)
    lib().ref_graph_from_arrays.restype = C.c_void_p
    return Graph(lib().ref_graph_from_arrays(
        C.c_uint64(n), C.c_uint64(uv.shape[0]), _p(uv), C.c_int(int(undirected)),
        _p(features), C.c_uint64(features.shape[1]), _p(labels), C.c_uint32(classes),
        _p(mask), C.c_int(int(f64))), f64)


def permutation_pair(n, seed):
    r, c = np.empty(n, np.uint32), np.empty(n, np.uint32)
    lib().ref_permutation_pair(C.c_uint64(n), C.c_uint64(seed), _p(r), _p(c))
    return r, c


def philox_u64(seed, stream, count):
    out = np.empty(count, np.uint64)
    lib().ref_philox_u64(C.c_uint64(seed), C.c_uint64(stream), C.c_uint64(count), _p(out))
    return out


def spmm_rows(rows, cols, rp, ci, vals, x, r0=0, r1=None):
    f64 = vals.dtype == np.float64
    r1 = rows if r1 is None else r1
    rp = np.ascontiguousarray(rp, np.uint64)
    ci = np.ascontiguousarray(ci, np.uint32)
    x = np.ascontiguousarray(x, vals.dtype)
    out = np.empty((r1 - r0, x.shape[1]), vals.dtype)
    fl = C.c_uint64(0)
    _check(lib().ref_spmm_rows(C.c_uint64(rows), C.c_uint64(cols), _p(rp), _p(ci),
                               _p(np.ascontiguousarray(vals)), _p(x),
                               C.c_uint64(x.shape[0]), C.c_uint64(x.shape[1]),
                               C.c_uint64(r0), C.c_uint64(r1), _p(out), C.byref(fl),
                               C.c_int(int(f64))))
    return out, fl.value


def gemm(a, b, ta=False, tb=False):
    f64 = a.dtype == np.float64
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b, a.dtype)
    m = a.shape[1] if ta else a.shape[0]
    n = b.shape[0] if tb else b.shape[1]
    out = np.empty((m, n), a.dtype)
    fl = C.c_uint64(0)
    _check(lib().ref_gemm(_p(a), C.c_uint64(a.shape[0]), C.c_uint64(a.shape[1]), _p(b),
                          C.c_uint64(b.shape[0]), C.c_uint64(b.shape[1]), C.c_int(int(ta)),
                          C.c_int(int(tb)), _p(out), C.byref(fl), C.c_int(int(f64))))
    return out, fl.value


def relu_forward(q):
    q = np.ascontiguousarray(q)
    out = np.empty_like(q)
    _check(lib().ref_relu_forward(_p(q), C.c_uint64(q.shape[0]), C.c_uint64(q.shape[1]),
                                  _p(out), C.c_int(int(q.dtype == np.float64))))
    return out


def relu_backward(q, df):
    q = np.ascontiguousarray(q)
    df = np.ascontiguousarray(df, q.dtype)
    out = np.empty_like(q)
    _check(lib().ref_relu_backward(_p(q), _p(df), C.c_uint64(q.shape[0]),
                                   C.c_uint64(q.shape[1]), _p(out),
                                   C.c_int(int(q.dtype == np.float64))))
    return out


def ce_sums(logits, labels, mask):
    logits = np.ascontiguousarray(logits)
    labels = np.ascontiguousarray(labels, np.uint32)
    mask = np.ascontiguousarray(mask, np.uint8)
    ls, cnt, cor = C.c_double(), C.c_uint64(), C.c_uint64()
    d = np.empty_like(logits)
    _check(lib().ref_ce_sums(_p(logits), C.c_uint64(logits.shape[0]),
                             C.c_uint64(logits.shape[1]), _p(labels), _p(mask), C.byref(ls),
                             C.byref(cnt), C.byref(cor), _p(d),
                             C.c_int(int(logits.dtype == np.float64))))
    return ls.value, cnt.value, cor.value, d


def adam_step(param, grad, m, v, step, lr=1e-2, b1=0.9, b2=0.999, eps=1e-8):
    """In-place on param/m/v (float arrays, 2-D). `step` = count before."""
    r, c = param.shape
    _check(lib().ref_adam_step(_p(param), _p(np.ascontiguousarray(grad, param.dtype)),
                               _p(m), _p(v), C.c_uint64(r), C.c_uint64(c),
                               C.c_uint64(step), C.c_double(lr), C.c_double(b1),
                               C.c_double(b2), C.c_double(eps),
                               C.c_int(int(param.dtype == np.float64))))


def init_weights(dims, seed, f64=False):
    d = np.asarray(dims, np.uint64)
    out = np.empty(sum(dims[l] * dims[l + 1] for l in range(len(dims) - 1)), _dt(f64))
    _check(lib().ref_init_weights(_p(d), C.c_int(len(dims)), C.c_uint64(seed), _p(out),
                                  C.c_int(int(f64))))
    return split_weights(out, dims)


def plan_layout(layer):
    i, c, r = C.c_int(), C.c_int(), C.c_int()
    lib().ref_plan_layout(C.c_int(layer), C.byref(i), C.byref(c), C.byref(r))
    return i.value, c.value, r.value


def layer_shapes(grid, layer, coords, n, d_in, d_out):
    out = np.empty(10, np.uint64)
    lib().ref_layer_shapes(*[C.c_int(g) for g in grid], C.c_int(layer),
                           *[C.c_int(x) for x in coords], C.c_uint64(n), C.c_uint64(d_in),
                           C.c_uint64(d_out), _p(out))
    keys = ("a_rows", "a_cols", "f_rows", "f_cols", "w_rows", "w_cols", "h_rows",
            "h_cols", "q_rows", "q_cols")
    return dict(zip(keys, (int(x) for x in out)))


def weight_slice(grid, layer, coords, d_in, d_out):
    out = np.empty(4, np.uint64)
    lib().ref_weight_slice(*[C.c_int(g) for g in grid], C.c_int(layer),
                           *[C.c_int(x) for x in coords], C.c_uint64(d_in),
                           C.c_uint64(d_out), _p(out))
    return tuple(int(x) for x in out)


def feature_slice(grid, coords, n, d0):
    out = np.empty(4, np.uint64)
    lib().ref_feature_slice(*[C.c_int(g) for g in grid], *[C.c_int(x) for x in coords],
                            C.c_uint64(n), C.c_uint64(d0), _p(out))
    return tuple(int(x) for x in out)


def block_range(grid, plane, coords, n):
    out = np.empty(4, np.uint64)
    lib().ref_block_range(*[C.c_int(g) for g in grid], C.c_int(plane),
                          *[C.c_int(x) for x in coords], C.c_uint64(n), _p(out))
    return tuple(int(x) for x in out)


def label_row_range(grid, coords, n, layers):
    out = np.empty(2, np.uint64)
    lib().ref_label_row_range(*[C.c_int(g) for g in grid], *[C.c_int(x) for x in coords],
                              C.c_uint64(n), C.c_int(layers), _p(out))
    return int(out[0]), int(out[1])


def collective_volumes(grid, n, dims):
    d = np.asarray(dims, np.uint64)
    cnt = lib().ref_collective_volumes(*[C.c_int(g) for g in grid], C.c_uint64(n), _p(d),
                                       C.c_int(len(dims)), None)
    out = np.empty((cnt, 5), np.uint64)
    lib().ref_collective_volumes(*[C.c_int(g) for g in grid], C.c_uint64(n), _p(d),
                                 C.c_int(len(dims)), _p(out))
    return out


def rank_configs(g, n, nnz, dims, g_node=4, beta_intra=200e9, beta_inter=25e9,
                 bytes_per_scalar=4, coeffs=(7.8e-4, 7.8e-10, -2.6e-10)):
    d = np.asarray(dims, np.uint64)
    out = np.empty((64, 7))
    cnt = lib().ref_rank_configs(C.c_int(g), C.c_uint64(n), C.c_uint64(nnz), _p(d),
                                 C.c_int(len(dims)), C.c_int(g_node), C.c_double(beta_intra),
                                 C.c_double(beta_inter), C.c_int(bytes_per_scalar),
                                 *[C.c_double(c) for c in coeffs], _p(out))
    if cnt < 0:
        raise RuntimeError(lib().ref_last_error().decode())
    return out[:cnt]


def comp_features(n, nnz, dims, grid):
    d = np.asarray(dims, np.uint64)
    out = np.empty(3)
    lib().ref_comp_features(C.c_uint64(n), C.c_uint64(nnz), _p(d), C.c_int(len(dims)),
                            *[C.c_int(g) for g in grid], _p(out))
    return out


def predict_comm(n, nnz, dims, grid, g_node=4, beta_intra=200e9, beta_inter=25e9,
                 bytes_per_scalar=4):
    d = np.asarray(dims, np.uint64)
    lib().ref_predict_comm.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_int]
    return lib().ref_predict_comm(n, nnz, _p(d), len(dims), *grid, g_node, beta_intra,
                                  beta_inter, bytes_per_scalar)


def fit_regression(features, seconds):
    f = np.ascontiguousarray(features, np.float64)
    s = np.ascontiguousarray(seconds, np.float64)
    out = np.empty(5)
    _check(lib().ref_fit_regression(_p(f), _p(s), C.c_int(len(s)), _p(out)))
    return out


# ---------------------------------------------------------------------------
# shard files (shard_io.hpp, trainer.hpp:252-438)

def _io_check(rc):
    """IoError codes come back as 10 + IoErrorCode (common.hpp:28-35)."""
    if rc != 0:
        raise RuntimeError(f"rc={rc}: " + lib().ref_last_error().decode())


def write_shards(pre, p, q, directory, name="dataset"):
    """shard_io::write_shards (shard_io.hpp:278-414)."""
    _io_check(lib().ref_write_shards(pre.h, C.c_int(p), C.c_int(q),
                                     str(directory).encode(), name.encode()))


def load_preprocessed(directory):
    """load_manifest + load_preprocessed (shard_io.hpp:416-486, trainer.hpp:386-438)."""
    lib().ref_load_preprocessed.restype = C.c_void_p
    lib().ref_load_preprocessed.argtypes = [C.c_char_p]
    h = lib().ref_load_preprocessed(str(directory).encode())
    if not h:
        raise RuntimeError(lib().ref_last_error().decode())
    # precision from the manifest
    import json
    with open(os.path.join(str(directory), "manifest.json")) as f:
        f64 = json.load(f)["precision"] == "f64"
    return Pre(h, f64)


class RankShards(_Handle):
    """load_rank_shards (trainer.hpp:256-384) for one rank."""
    _free = "ref_rank_free"

    @classmethod
    def load(cls, directory, grid, coords, layers, f64=False):
        lib().ref_load_rank_shards.restype = C.c_void_p
        lib().ref_load_rank_shards.argtypes = [C.c_char_p] + [C.c_int] * 7
        lib().ref_rank_adj.restype = C.c_void_p
        lib().ref_rank_adj.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        lib().ref_rank_free.argtypes = [C.c_void_p]
        h = lib().ref_load_rank_shards(str(directory).encode(), *grid, *coords, layers)
        return cls(h, f64)

    def adj(self, plane, parity, transposed=False):
        return Csr(lib().ref_rank_adj(self.h, plane, parity, int(transposed)), self.f64)

    def info(self):
        fr, fc, nl = C.c_uint64(), C.c_uint64(), C.c_uint64()
        files, nbytes = C.c_int(), C.c_uint64()
        lib().ref_rank_info(self.h, C.byref(fr), C.byref(fc), C.byref(nl), C.byref(files),
                            C.byref(nbytes))
        return dict(f0_rows=fr.value, f0_cols=fc.value, labels=nl.value, files_read=files.value,
                    bytes_read=nbytes.value)

    def arrays(self):
        i = self.info()
        f0 = np.empty((i["f0_rows"], i["f0_cols"]), _dt(self.f64))
        lab = np.empty(i["labels"], np.uint32)
        mask = np.empty(i["labels"], np.uint8)
        lib().ref_rank_copy(self.h, _p(f0), _p(lab), _p(mask))
        return f0, lab, mask
