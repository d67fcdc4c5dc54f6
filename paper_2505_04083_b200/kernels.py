"""Host mirror of the reference kernel API (kernels.hpp, model.hpp:69-111)
over CUDA tensors, calling the sm_100a kernels through the C ABI.

Same names, argument meaning and error behaviour as the reference:
``spmm(a, x)``, ``spmm_rows(a, x, r0, r1)``, ``gemm(a, b, ta, tb)``,
``relu_forward(q)``, ``relu_backward(q, df)``,
``softmax_cross_entropy_sums(logits, labels, mask)``,
``adam_step(param, grad, state, params)``. Shape violations raise
``ContractError`` with the reference's message. FLOP counters are optional
one-element lists incremented like the reference's ``u64*`` out-params.
"""

import ctypes as C
from dataclasses import dataclass

import torch

from . import _capi
from ._capi import PK_MODE_FAST, PK_MODE_PARITY, PK_SPMM_PAIRED, ContractError, call

__all__ = ["DeviceCsr", "spmm", "spmm_rows", "gemm", "relu_forward", "relu_backward",
           "softmax_cross_entropy_sums", "softmax_cross_entropy", "AdamParams", "AdamState",
           "adam_step", "SpmmPlan", "PK_MODE_FAST", "PK_MODE_PARITY"]


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else C.c_void_p(
        t.data_ptr() if t is not None else 0)


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ld(t):
    """Leading dimension (elements) of a row-major 2-D view."""
    if t.dim() != 2:
        raise ContractError(f"expected a matrix, got {tuple(t.shape)}")
    if t.shape[1] > 1 and t.stride(1) != 1:
        raise ContractError("matrix must be row-major (unit column stride)")
    return max(t.stride(0), t.shape[1]) if t.shape[0] > 1 else max(t.shape[1], 1)


class DeviceCsr:
    """CsrMatrix<float> (csr.hpp:14-149) resident in HBM: u64 row_ptr
    (held in an int64 tensor), u32 col_idx (int32 tensor, same bits),
    f32 values."""

    def __init__(self, rows, cols, row_ptr, col_idx, values, _owned=None):
        self.rows, self.cols = int(rows), int(cols)
        self.row_ptr, self.col_idx, self.values = row_ptr, col_idx, values
        self._owned = _owned  # pk_csr_owned to free, when the library allocated it
        self._view = _capi.pk_csr(self.rows, self.cols, self.nnz, row_ptr.data_ptr(),
                                  col_idx.data_ptr() if col_idx.numel() else 0,
                                  values.data_ptr() if values.numel() else 0)
        self._plan = None

    @property
    def nnz(self):
        return int(self.col_idx.numel())

    def view(self):
        return C.byref(self._view)

    @classmethod
    def from_host(cls, rows, cols, row_ptr, col_idx, values, device="cuda"):
        import numpy as np
        rp = torch.from_numpy(np.ascontiguousarray(row_ptr).astype(np.uint64).view(np.int64))
        ci = torch.from_numpy(np.ascontiguousarray(col_idx).astype(np.uint32).view(np.int32))
        v = torch.from_numpy(np.ascontiguousarray(values, dtype=np.float32))
        return cls(rows, cols, rp.to(device), ci.to(device), v.to(device))

    @classmethod
    def _from_owned(cls, owned):
        """Wrap library-allocated arrays (pk_csr_owned) without copying."""
        rows, cols, nnz = owned.rows, owned.cols, owned.nnz
        keep = _OwnedCsr(owned)
        rp = _wrap_device(owned.row_ptr, rows + 1, torch.int64, keep)
        ci = _wrap_device(owned.col_idx, nnz, torch.int32, keep)
        v = _wrap_device(owned.values, nnz, torch.float32, keep)
        return cls(rows, cols, rp, ci, v, _owned=keep)

    def to_host(self):
        import numpy as np
        return (self.row_ptr.cpu().numpy().view(np.uint64), self.col_idx.cpu().numpy().view(
            np.uint32), self.values.cpu().numpy())

    def plan(self, hub_threshold=0, mode=PK_MODE_PARITY):
        """The cached exact plan, or a new plan for a given threshold / mode."""
        if hub_threshold or mode != PK_MODE_PARITY:
            return SpmmPlan(self, hub_threshold, mode=mode)
        if self._plan is None:
            self._plan = SpmmPlan(self)
        return self._plan


class _OwnedCsr:
    def __init__(self, owned):
        self.owned = owned

    def __del__(self):
        try:
            _capi.lib().pk_csr_free(C.byref(self.owned))
        except Exception:
            pass


def _wrap_device(ptr, count, dtype, keepalive):
    """Zero-copy torch view of `count` elements at a library-owned device pointer."""
    if count == 0 or not ptr:
        return torch.empty(0, dtype=dtype, device="cuda")
    # __cuda_array_interface__ lets torch adopt external device memory
    typestr = {torch.int64: "<i8", torch.int32: "<i4", torch.float32: "<f4"}[dtype]

    class _Arr:
        __cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                    "data": (int(ptr), False), "version": 3, "strides": None}
    t = torch.as_tensor(_Arr(), device="cuda")
    t._pk_keepalive = keepalive  # the library buffer outlives the view
    return t


class SpmmPlan:
    """pk_spmm_plan: hub rows split off (one per matrix). mode PARITY keeps
    every row one exact chain (bit-identical); FAST cuts hub rows into
    segments combined in a fixed order (fp32-level difference)."""

    def __init__(self, a: DeviceCsr, hub_threshold=0, stream=None, mode=PK_MODE_PARITY):
        self.a = a
        h = C.c_void_p()
        call("pk_spmm_plan_create_mode", a.view(), hub_threshold, mode, _stream(stream),
             C.byref(h))
        self.h = h

    def info(self):
        hub, thr = C.c_int64(), C.c_int64()
        call("pk_spmm_plan_info", self.h, C.byref(hub), C.byref(thr))
        return hub.value, thr.value

    def __del__(self):
        try:
            if self.h:
                _capi.lib().pk_spmm_plan_destroy(self.h)
        except Exception:
            pass


def _flops_out(flops):
    return C.c_uint64(0) if flops is not None else None


def spmm_rows(a: DeviceCsr, x: torch.Tensor, r0: int, r1: int, flops=None, out=None,
              plan=None, stream=None, paired=False):
    """spmm_rows (kernels.hpp:39-62): rows [r0, r1) of A . X, bit-exact.
    paired=True (a PK_MODE_FAST plan; rows of <= 64 columns): each row as two
    interleaved chains added at the row end (PK_SPMM_PAIRED) — fp32-level
    difference, deterministic."""
    d = x.shape[1]
    if a.cols != x.shape[0]:
        raise ContractError(f"spmm_rows: A is {a.rows}x{a.cols} but X is {x.shape[0]}x{d}")
    if out is None:
        out = torch.empty((r1 - r0, d), dtype=torch.float32, device=x.device)
    fl = _flops_out(flops)
    args = [a.view(), r0, r1, _ptr(x), x.shape[0], _ld(x), d, _ptr(out), _ld(out),
            C.byref(fl) if fl is not None else None, _stream(stream)]
    if paired:
        if plan is None:
            raise ContractError("spmm_rows: paired=True needs a PK_MODE_FAST plan")
        call("pk_spmm_plan_rows_ex_f32", plan.h, *args[:-2], PK_SPMM_PAIRED, *args[-2:])
    elif plan is not None:
        call("pk_spmm_plan_rows_f32", plan.h, *args)
    else:
        call("pk_spmm_rows_f32", *args)
    if flops is not None:
        flops[0] += fl.value
    return out


def spmm_rows_relu_backward(a: DeviceCsr, x: torch.Tensor, r0: int, r1: int, mask, plan,
                            flops=None, out=None, stream=None):
    """relu_backward(mask, spmm_rows(A, X, r0, r1)) in one pass
    (kernels.hpp:39-62 then 103-111): the backward's dF of a layer, masked by
    the previous layer's cached relu(Q)."""
    d = x.shape[1]
    if a.cols != x.shape[0]:
        raise ContractError(f"spmm_rows: A is {a.rows}x{a.cols} but X is {x.shape[0]}x{d}")
    if tuple(mask.shape) != (r1 - r0, d):
        raise ContractError(f"relu_backward: mask is {tuple(mask.shape)}, want {(r1 - r0, d)}")
    if out is None:
        out = torch.empty((r1 - r0, d), dtype=torch.float32, device=x.device)
    fl = _flops_out(flops)
    call("pk_spmm_plan_rows_relu_bwd_f32", plan.h, a.view(), r0, r1, _ptr(x), x.shape[0], _ld(x),
         d, _ptr(mask), _ld(mask), _ptr(out), _ld(out), C.byref(fl) if fl is not None else None,
         _stream(stream))
    if flops is not None:
        flops[0] += fl.value
    return out


def spmm(a: DeviceCsr, x: torch.Tensor, flops=None, out=None, plan=None, stream=None,
         paired=False):
    """spmm (kernels.hpp:16-37): A . X, bit-exact (paired: see spmm_rows)."""
    if a.cols != x.shape[0]:
        raise ContractError(f"spmm: A is {a.rows}x{a.cols} but X is {x.shape[0]}x{x.shape[1]}")
    return spmm_rows(a, x, 0, a.rows, flops=flops, out=out, plan=plan, stream=stream,
                     paired=paired)


def gemm(a, b, transpose_a=False, transpose_b=False, flops=None, mode=PK_MODE_PARITY, out=None,
         stream=None, relu=False):
    """gemm (kernels.hpp:64-92): op(A) . op(B). PARITY is bit-exact with the
    reference loop; FAST is the tensor-core path. relu=True returns
    relu_forward(op(A) . op(B)) from one fused call (pk_gemm_relu_f32)."""
    m = a.shape[1] if transpose_a else a.shape[0]
    ka = a.shape[0] if transpose_a else a.shape[1]
    kb = b.shape[1] if transpose_b else b.shape[0]
    n = b.shape[0] if transpose_b else b.shape[1]
    if ka != kb:
        raise ContractError(
            f"gemm: inner dimensions disagree: {a.shape[0]}x{a.shape[1]}"
            f"{'^T' if transpose_a else ''} * {b.shape[0]}x{b.shape[1]}"
            f"{'^T' if transpose_b else ''}")
    if out is None:
        out = torch.empty((m, n), dtype=torch.float32, device=a.device)
    fl = _flops_out(flops)
    call("pk_gemm_relu_f32" if relu else "pk_gemm_f32", int(transpose_a), int(transpose_b), m, n,
         ka, _ptr(a), _ld(a), _ptr(b),
         _ld(b), _ptr(out), _ld(out), mode, C.byref(fl) if fl is not None else None,
         _stream(stream))
    if flops is not None:
        flops[0] += fl.value
    return out


def relu_forward(q, out=None, stream=None):
    """relu_forward (kernels.hpp:94-100)."""
    if out is None:
        out = torch.empty_like(q)
    call("pk_relu_forward_f32", _ptr(q), _ld(q), q.shape[0], q.shape[1], _ptr(out), _ld(out),
         _stream(stream))
    return out


def relu_backward(q, df, out=None, stream=None):
    """relu_backward (kernels.hpp:102-111)."""
    if tuple(q.shape) != tuple(df.shape):
        raise ContractError(f"relu_backward: Q is {q.shape[0]}x{q.shape[1]} but dF is "
                            f"{df.shape[0]}x{df.shape[1]}")
    if out is None:
        out = torch.empty_like(q)
    call("pk_relu_backward_f32", _ptr(q), _ld(q), _ptr(df), _ld(df), q.shape[0], q.shape[1],
         _ptr(out), _ld(out), _stream(stream))
    return out


@dataclass
class CrossEntropySums:
    """CrossEntropySums<T> (kernels.hpp:117-123)."""
    loss_sum: float
    count: int
    correct: int
    dlogits: torch.Tensor
    sums_dev: torch.Tensor  # the device 1x3 double block


def softmax_cross_entropy_sums(logits, labels, mask, stream=None):
    """softmax_cross_entropy_sums (kernels.hpp:125-158)."""
    rows, c = logits.shape
    if labels.numel() != rows:
        raise ContractError(f"cross entropy: labels length {labels.numel()} != rows {rows}")
    if mask.numel() != rows:
        raise ContractError("cross entropy: mask length mismatch")
    d = torch.empty_like(logits)
    sums = torch.zeros(3, dtype=torch.float64, device=logits.device)
    call("pk_softmax_ce_sums_f32", _ptr(logits), _ld(logits), rows, c, _ptr(labels), _ptr(mask),
         _ptr(d), _ld(d), _ptr(sums), _stream(stream))
    h = sums.cpu()
    return CrossEntropySums(float(h[0]), int(h[1]), int(h[2]), d, sums)


def softmax_cross_entropy(logits, labels, mask, stream=None):
    """softmax_cross_entropy (kernels.hpp:160-173): mean loss and scaled dlogits."""
    s = softmax_cross_entropy_sums(logits, labels, mask, stream)
    if s.count == 0:
        raise ContractError("cross entropy: no rows selected by the mask")
    call("pk_scale_by_count_f32", _ptr(s.dlogits), _ld(s.dlogits), s.dlogits.shape[0],
         s.dlogits.shape[1], _ptr(s.sums_dev), _stream(stream))
    return s.loss_sum / s.count, s.dlogits


@dataclass
class AdamParams:
    """AdamParams (model.hpp:69-74)."""
    lr: float = 1e-2
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


class AdamState:
    """AdamState<T> (model.hpp:76-86): moments sharded like the parameter."""

    def __init__(self, m, v, step=0):
        self.m, self.v, self.step = m, v, step

    @classmethod
    def like(cls, param):
        return cls(torch.zeros_like(param), torch.zeros_like(param), 0)


def adam_step(param, grad, state: AdamState, opts: AdamParams = AdamParams(), stream=None):
    """adam_step (model.hpp:88-111), in place, bit-exact."""
    if tuple(param.shape) != tuple(grad.shape) or tuple(param.shape) != tuple(state.m.shape):
        raise ContractError(
            f"adam_step: parameter {param.shape[0]}x{param.shape[1]}, gradient "
            f"{grad.shape[0]}x{grad.shape[1]} and state shapes must agree")
    for t in (param, grad, state.m, state.v):
        if not t.is_contiguous():
            raise ContractError("adam_step: tensors must be contiguous")
    state.step += 1
    call("pk_adam_step_f32", _ptr(param), _ptr(grad), _ptr(state.m), _ptr(state.v),
         param.numel(), state.step, opts.lr, opts.beta1, opts.beta2, opts.eps, _stream(stream))
