"""ctypes binding of libplexus_b200.so (include/plexus_b200.h).

The library is the product: there is no Python or CPU fallback. Loading
fails loudly when the shared object is missing; every call raises the
reference's exception type when the C ABI returns an error.
"""

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libplexus_b200.so")

(PK_OK, PK_ERR_CONTRACT, PK_ERR_CUDA, PK_ERR_NCCL, PK_ERR_MEMORY, PK_ERR_TRAINING,
 PK_ERR_ABORTED) = range(7)
PK_MODE_PARITY, PK_MODE_FAST = 0, 1
PK_SPMM_PAIRED = 1  # pk_spmm_plan_rows_ex_f32 flags


class ContractError(RuntimeError):
    """plexuskit::ContractError (common.hpp:16-20)."""


class MemoryError_(RuntimeError):
    """plexuskit::MemoryError (common.hpp:22-26)."""


class TrainingError(RuntimeError):
    """plexuskit::TrainingError (trainer.hpp:26-29)."""


class CudaError(RuntimeError):
    pass


class NcclError(RuntimeError):
    pass


class ClusterAborted(RuntimeError):
    """plexuskit::ClusterAborted (cluster.hpp:67-71): another rank failed."""


class IoError(RuntimeError):
    """plexuskit::IoError (common.hpp:28-41); `code` is the IoErrorCode name."""
    CODES = {10: "MissingFile", 11: "TruncatedFile", 12: "ChecksumMismatch",
             13: "ManifestMismatch", 14: "BadFormat", 15: "WriteFailed"}

    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def _io_error(rc):
    return lambda msg: IoError(IoError.CODES[rc], msg)


_ERRORS = {PK_ERR_CONTRACT: ContractError, PK_ERR_CUDA: CudaError, PK_ERR_NCCL: NcclError,
           PK_ERR_MEMORY: MemoryError_, PK_ERR_TRAINING: TrainingError,
           PK_ERR_ABORTED: ClusterAborted}
_ERRORS.update({rc: _io_error(rc) for rc in IoError.CODES})


class pk_csr(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_uint64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class pk_plxs_csr_host(C.Structure):
    _fields_ = [("rows", C.c_uint64), ("cols", C.c_uint64), ("nnz", C.c_uint64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class pk_csr_owned(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_uint64),
                ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


P = C.c_void_p
I64 = C.c_int64
U64 = C.c_uint64
U32 = C.c_uint32
INT = C.c_int
DBL = C.c_double
U64P = C.POINTER(C.c_uint64)
I64P = C.POINTER(C.c_int64)

# name -> (restype, argtypes); mirrors include/plexus_b200.h
SIGNATURES = {
    "pk_last_error": (C.c_char_p, []),
    "pk_abi_version": (INT, []),
    "pk_kernel_launch_count": (U64, []),
    "pk_device_cache_release": (INT, []),
    "pk_device_sm_count": (INT, [INT]),
    "pk_spmm_rows_f32": (INT, [C.POINTER(pk_csr), I64, I64, P, I64, I64, I64, P, I64, U64P, P]),
    "pk_spmm_f32": (INT, [C.POINTER(pk_csr), P, I64, I64, I64, P, I64, U64P, P]),
    "pk_spmm_plan_create": (INT, [C.POINTER(pk_csr), I64, P, C.POINTER(P)]),
    "pk_spmm_plan_create_mode": (INT, [C.POINTER(pk_csr), I64, INT, P, C.POINTER(P)]),
    "pk_spmm_plan_destroy": (INT, [P]),
    "pk_spmm_plan_rows_f32": (INT, [P, C.POINTER(pk_csr), I64, I64, P, I64, I64, I64, P, I64,
                                    U64P, P]),
    "pk_spmm_plan_rows_relu_bwd_f32": (INT, [P, C.POINTER(pk_csr), I64, I64, P, I64, I64, I64,
                                             P, I64, P, I64, U64P, P]),
    "pk_spmm_plan_rows_ex_f32": (INT, [P, C.POINTER(pk_csr), I64, I64, P, I64, I64, I64, P,
                                       I64, INT, U64P, P]),
    "pk_spmm_plan_info": (INT, [P, I64P, I64P]),
    "pk_gemm_f32": (INT, [INT, INT, I64, I64, I64, P, I64, P, I64, P, I64, INT, U64P, P]),
    "pk_gemm_relu_f32": (INT, [INT, INT, I64, I64, I64, P, I64, P, I64, P, I64, INT, U64P, P]),
    "pk_relu_forward_f32": (INT, [P, I64, I64, I64, P, I64, P]),
    "pk_relu_backward_f32": (INT, [P, I64, P, I64, I64, I64, P, I64, P]),
    "pk_softmax_ce_sums_f32": (INT, [P, I64, I64, I64, P, P, P, I64, P, P]),
    "pk_scale_by_count_f32": (INT, [P, I64, I64, I64, P, P]),
    "pk_adam_step_f32": (INT, [P, P, P, P, I64, U64, DBL, DBL, DBL, DBL, P]),
    "pk_csr_transpose": (INT, [C.POINTER(pk_csr), C.POINTER(pk_csr_owned), P]),
    "pk_csr_block": (INT, [C.POINTER(pk_csr), I64, I64, I64, I64, C.POINTER(pk_csr_owned), P]),
    "pk_normalize_adjacency": (INT, [I64, P, U64, INT, C.POINTER(pk_csr_owned), P]),
    "pk_permute_csr": (INT, [C.POINTER(pk_csr), P, P, C.POINTER(pk_csr_owned), P]),
    "pk_csr_free": (None, [C.POINTER(pk_csr_owned)]),
    "pk_csr_hconcat": (INT, [C.POINTER(pk_csr), P, INT, U64, U64, C.POINTER(pk_csr_owned), P]),
    "pk_plxs_write": (INT, [C.c_char_p, P, C.c_uint32, C.POINTER(pk_plxs_csr_host),
                            C.POINTER(pk_plxs_csr_host), U64, U64, P, U64, P, P, P, P, P]),
    "pk_plxs_open": (INT, [C.c_char_p, P, C.c_uint32, C.POINTER(C.c_void_p)]),
    "pk_plxs_close": (INT, [P]),
    "pk_plxs_info": (INT, [P, P, P, P]),
    "pk_plxs_csr_extent": (INT, [P, INT, U64, U64, P, P, P, P, P]),
    "pk_plxs_read_csr_rows": (INT, [P, INT, U64, U64, U64, P, P, P, INT, P]),
    "pk_plxs_read_feature_rows": (INT, [P, U64, U64, U64, P, INT, P]),
    "pk_plxs_read_labels": (INT, [P, U64, U64, U64, P, P, P, P]),
    "pk_permutation_pair_host": (INT, [U64, U64, P, P]),
    "pk_philox_permutation_host": (INT, [U64, U64, U64, P]),
    "pk_rmat_edges": (INT, [INT, U64, DBL, DBL, DBL, U64, P, U64P, P]),
    "pk_sbm_edges": (INT, [U64, INT, C.c_double, C.c_double, U64, P, U64, U64P, P]),
    "pk_erdos_edges": (INT, [U64, C.c_double, U64, P, U64, U64P, P]),
    "pk_rmat_features": (INT, [U64, I64, I64, P, I64, P]),
    "pk_degree_quantile_labels": (INT, [P, U64, I64, U32, P, P]),
    "pk_gather_rows_f32": (INT, [P, I64, P, I64, I64, P, I64, P]),
    "pk_gather_u32": (INT, [P, P, I64, P, P]),
    "pk_gather_u8": (INT, [P, P, I64, P, P]),
    "pk_balance_metric": (INT, [C.POINTER(pk_csr), INT, INT, C.POINTER(DBL), P]),
}

_lib = None


def lib():
    """Load libplexus_b200.so; raise if it is not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (no CPU fallback exists)")
        lib_ = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib_, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib_
    return _lib


def register(sigs):
    """Add signatures declared by another module (applied now if loaded)."""
    SIGNATURES.update(sigs)
    if _lib is not None:
        for name, (res, args) in sigs.items():
            fn = getattr(_lib, name)
            fn.restype = res
            fn.argtypes = args


def call(name, *args):
    rc = getattr(lib(), name)(*args)
    if rc not in (None, PK_OK):
        msg = lib().pk_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, RuntimeError)(msg)
    return rc
