"""Host mirror of the reference performance model API (perf_model.hpp:18-127)
over libplexus_b200.so's native implementation (csrc/perf_model.cpp).

Same names and argument meaning as the reference: DatasetStats,
MachineParams, PerfCoefficients, comp_features, predict_spmm_time,
effective_bandwidth, ring_collective_seconds, predict_comm_time,
fit_regression, fit_with_split, rank_configs, plus the machine/coefficient
JSON files and the sample CSV (perf_model.cpp:231-339). Errors raise the
reference's exception types (ContractError; IoError for files).
"""

import ctypes as C
import json
import math
from dataclasses import dataclass, field
from typing import List, Sequence

from . import _capi
from ._capi import ContractError, call
from .layout import GridConfig

PK_MAX_LAYERS = 15
AXES = {"X": 0, "Y": 1, "Z": 2}
COLL_OPS = {"all_gather": 0, "all_reduce": 1, "reduce_scatter": 2}


IoError = _capi.IoError  # plexuskit::IoError (common.hpp:28-45); code = IoErrorCode name


class pk_dataset_stats(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_uint64), ("num_dims", C.c_int),
                ("dims", C.c_int64 * (PK_MAX_LAYERS + 1))]


class pk_machine(C.Structure):
    _fields_ = [("g_node", C.c_int), ("beta_intra", C.c_double), ("beta_inter", C.c_double),
                ("bytes_per_scalar", C.c_int)]


class pk_perf_coeffs(C.Structure):
    _fields_ = [("c1", C.c_double), ("c2", C.c_double), ("c3", C.c_double),
                ("train_r2", C.c_double), ("train_rmse", C.c_double)]


class pk_config_prediction(C.Structure):
    _fields_ = [("gx", C.c_int), ("gy", C.c_int), ("gz", C.c_int), ("clamped", C.c_int),
                ("spmm_seconds", C.c_double), ("comm_seconds", C.c_double),
                ("total_seconds", C.c_double)]


class pk_collective_volume(C.Structure):
    _fields_ = [("layer", C.c_int), ("forward", C.c_int), ("op", C.c_int), ("axis", C.c_int),
                ("elems", C.c_uint64)]


_P = C.POINTER
_capi.register({
    "pk_perf_default_coefficients": (C.c_int, [_P(pk_perf_coeffs)]),
    "pk_perf_comp_features": (C.c_int, [_P(pk_dataset_stats), C.c_int, C.c_int, C.c_int,
                                        _P(C.c_double)]),
    "pk_perf_predict_spmm": (C.c_int, [_P(C.c_double), _P(pk_perf_coeffs), _P(C.c_double),
                                       _P(C.c_int)]),
    "pk_perf_effective_bandwidth": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int,
                                              _P(pk_machine), _P(C.c_double)]),
    "pk_perf_ring_seconds": (C.c_int, [C.c_int, C.c_double, C.c_int, C.c_double,
                                       _P(C.c_double)]),
    "pk_perf_predict_comm": (C.c_int, [_P(pk_dataset_stats), C.c_int, C.c_int, C.c_int,
                                       _P(pk_machine), _P(C.c_double)]),
    "pk_collective_volumes": (C.c_int, [C.c_int, C.c_int, C.c_int, _P(pk_dataset_stats),
                                        _P(pk_collective_volume), C.c_int, _P(C.c_int)]),
    "pk_perf_fit_regression": (C.c_int, [_P(C.c_double), _P(C.c_double), C.c_int,
                                         _P(pk_perf_coeffs)]),
    "pk_enumerate_configs": (C.c_int, [C.c_int, _P(C.c_int), C.c_int, _P(C.c_int)]),
    "pk_perf_rank_configs": (C.c_int, [C.c_int, _P(pk_dataset_stats), _P(pk_machine),
                                       _P(pk_perf_coeffs), _P(pk_config_prediction), C.c_int,
                                       _P(C.c_int)]),
})


@dataclass
class DatasetStats:
    n: int
    nnz: int
    dims: List[int]

    def c(self):
        if len(self.dims) > PK_MAX_LAYERS + 1:
            raise ContractError("perf model: too many layers")
        s = pk_dataset_stats(self.n, self.nnz, len(self.dims))
        for i, d in enumerate(self.dims):
            s.dims[i] = d
        return s


@dataclass
class MachineParams:
    g_node: int = 4
    beta_intra: float = 200e9
    beta_inter: float = 25e9
    bytes_per_scalar: int = 4

    def c(self):
        return pk_machine(self.g_node, self.beta_intra, self.beta_inter, self.bytes_per_scalar)


@dataclass
class PerfCoefficients:
    c1: float = 0.0
    c2: float = 0.0
    c3: float = 0.0
    train_r2: float = 0.0
    train_rmse: float = 0.0

    def c(self):
        return pk_perf_coeffs(self.c1, self.c2, self.c3, self.train_r2, self.train_rmse)

    @classmethod
    def from_c(cls, p):
        return cls(p.c1, p.c2, p.c3, p.train_r2, p.train_rmse)


@dataclass
class ConfigPrediction:
    shape: tuple
    spmm_seconds: float
    comm_seconds: float
    total_seconds: float
    clamped: bool


@dataclass
class RegressionSample:
    features: tuple
    seconds: float


@dataclass
class SplitReport:
    coeffs: PerfCoefficients
    test_r2: float = 0.0
    test_rmse: float = 0.0


def _shape(grid):
    if isinstance(grid, GridConfig):
        return grid.gx, grid.gy, grid.gz
    return tuple(int(g) for g in grid)


def default_coefficients() -> PerfCoefficients:
    out = pk_perf_coeffs()
    call("pk_perf_default_coefficients", C.byref(out))
    return PerfCoefficients.from_c(out)


def comp_features(stats: DatasetStats, grid) -> tuple:
    f = (C.c_double * 3)()
    call("pk_perf_comp_features", C.byref(stats.c()), *_shape(grid), f)
    return tuple(f)


def predict_spmm_time(features: Sequence[float], coeffs: PerfCoefficients):
    """Returns (seconds, clamped)."""
    f = (C.c_double * 3)(*features)
    s, cl = C.c_double(), C.c_int()
    call("pk_perf_predict_spmm", f, C.byref(coeffs.c()), C.byref(s), C.byref(cl))
    return s.value, bool(cl.value)


def effective_bandwidth(axis, grid, machine: MachineParams) -> float:
    a = AXES[axis] if isinstance(axis, str) else int(axis)
    out = C.c_double()
    call("pk_perf_effective_bandwidth", a, *_shape(grid), C.byref(machine.c()), C.byref(out))
    return out.value


def ring_collective_seconds(op, m_bytes: float, g: int, beta: float) -> float:
    o = COLL_OPS[op] if isinstance(op, str) else int(op)
    out = C.c_double()
    call("pk_perf_ring_seconds", o, float(m_bytes), int(g), float(beta), C.byref(out))
    return out.value


def predict_comm_time(grid, stats: DatasetStats, machine: MachineParams) -> float:
    out = C.c_double()
    call("pk_perf_predict_comm", C.byref(stats.c()), *_shape(grid), C.byref(machine.c()),
         C.byref(out))
    return out.value


def training_collective_volumes(grid, n: int, dims: Sequence[int]):
    """(layer, forward, op, axis, elems) tuples (layout.hpp:123-157)."""
    st = DatasetStats(n, 0, list(dims)).c()
    cnt = C.c_int()
    call("pk_collective_volumes", *_shape(grid), C.byref(st), None, 0, C.byref(cnt))
    arr = (pk_collective_volume * max(1, cnt.value))()
    call("pk_collective_volumes", *_shape(grid), C.byref(st), arr, cnt.value, C.byref(cnt))
    return [(v.layer, bool(v.forward), v.op, v.axis, v.elems) for v in arr[:cnt.value]]


def fit_regression(samples: Sequence[RegressionSample]) -> PerfCoefficients:
    n = len(samples)
    f = (C.c_double * (3 * max(n, 1)))(*[x for s in samples for x in s.features])
    y = (C.c_double * max(n, 1))(*[s.seconds for s in samples])
    out = pk_perf_coeffs()
    call("pk_perf_fit_regression", f, y, n, C.byref(out))
    return PerfCoefficients.from_c(out)


def fit_with_split(samples: Sequence[RegressionSample], train_fraction: float,
                   seed: int) -> SplitReport:
    """Random train/test split (perf_model.cpp:168-205): Philox(seed, 17)
    permutation, the first max(3, fraction*n) samples train."""
    if not 0 < train_fraction < 1:
        raise ContractError("fit_with_split: fraction must be in (0,1)")
    order = (C.c_uint32 * max(1, len(samples)))()
    call("pk_philox_permutation_host", len(samples), int(seed), 17, order)
    order = list(order)[:len(samples)]
    n_train = max(3, int(train_fraction * len(samples)))
    if n_train >= len(samples):
        raise ContractError("fit_with_split: test split is empty")
    train = [samples[i] for i in order[:n_train]]
    test = [samples[i] for i in order[n_train:]]
    coeffs = fit_regression(train)
    pred = [coeffs.c1 * s.features[0] + coeffs.c2 * s.features[1] + coeffs.c3 * s.features[2]
            for s in test]
    mean = sum(s.seconds for s in test) / len(test)
    ss_res = sum((s.seconds - p) ** 2 for s, p in zip(test, pred))
    ss_tot = sum((s.seconds - mean) ** 2 for s in test)
    return SplitReport(coeffs, 1.0 - ss_res / ss_tot if ss_tot > 0 else 1.0,
                       math.sqrt(ss_res / len(test)))


def enumerate_configs(g: int):
    cnt = C.c_int()
    call("pk_enumerate_configs", int(g), None, 0, C.byref(cnt))
    arr = (C.c_int * (3 * max(1, cnt.value)))()
    call("pk_enumerate_configs", int(g), arr, cnt.value, C.byref(cnt))
    return [tuple(arr[3 * i:3 * i + 3]) for i in range(cnt.value)]


def rank_configs(g: int, stats: DatasetStats, machine: MachineParams,
                 coeffs: PerfCoefficients) -> List[ConfigPrediction]:
    cap = len(enumerate_configs(g))
    arr = (pk_config_prediction * max(1, cap))()
    cnt = C.c_int()
    call("pk_perf_rank_configs", int(g), C.byref(stats.c()), C.byref(machine.c()),
         C.byref(coeffs.c()), arr, cap, C.byref(cnt))
    return [ConfigPrediction((p.gx, p.gy, p.gz), p.spmm_seconds, p.comm_seconds,
                             p.total_seconds, bool(p.clamped)) for p in arr[:cnt.value]]


# --------------------------------------------------------------- files
# IoErrorCode (common.hpp:28-37) by name: MissingFile, BadFormat, WriteFailed

def _read_json(path, what):
    try:
        with open(path) as f:
            return json.load(f)
    except FileNotFoundError:
        raise IoError("MissingFile", f"cannot open {what} file {path}")
    except (json.JSONDecodeError, UnicodeDecodeError) as exc:
        raise IoError("BadFormat", f"{what} file {path}: {exc}")


def machine_from_json_file(path) -> MachineParams:
    j = _read_json(path, "machine")
    m = MachineParams()
    m.g_node = int(j.get("g_node", m.g_node))
    m.beta_intra = float(j.get("beta_intra", m.beta_intra))
    m.beta_inter = float(j.get("beta_inter", m.beta_inter))
    m.bytes_per_scalar = int(j.get("bytes_per_scalar", m.bytes_per_scalar))
    if not (m.g_node >= 1 and m.beta_intra > 0 and m.beta_inter > 0 and m.bytes_per_scalar > 0):
        raise ContractError(f"machine file {path}: invalid values")
    return m


def coefficients_from_json_file(path) -> PerfCoefficients:
    j = _read_json(path, "coefficients")
    try:
        return PerfCoefficients(float(j["c1"]), float(j["c2"]), float(j["c3"]),
                                float(j.get("train_r2", 0.0)), float(j.get("train_rmse", 0.0)))
    except KeyError as exc:
        raise IoError("BadFormat", f"coefficients file {path}: missing {exc}")


def coefficients_to_json_file(c: PerfCoefficients, path):
    try:
        with open(path, "w") as f:
            json.dump({"c1": c.c1, "c2": c.c2, "c3": c.c3, "train_r2": c.train_r2,
                       "train_rmse": c.train_rmse}, f, indent=2)
            f.write("\n")
    except OSError:
        raise IoError("WriteFailed", f"cannot write coefficients file {path}")


def samples_from_csv_file(path) -> List[RegressionSample]:
    """Feature rows `f1,f2,f3,seconds` or raw rows `n,nnz,dims,gx,gy,gz,seconds`
    (dims like 100-128-128-47), perf_model.cpp:285-339."""
    try:
        lines = open(path).read().splitlines()
    except FileNotFoundError:
        raise IoError("MissingFile", f"cannot open sample log {path}")
    head = lines[0].split(",") if lines else []
    if len(head) == 4 and head[0] == "f1":
        raw = False
    elif len(head) == 7 and head[0] == "n":
        raw = True
    else:
        raise IoError("BadFormat", f"sample log {path}: expected header f1,f2,f3,seconds or "
                         "n,nnz,dims,gx,gy,gz,seconds")
    out = []
    for line in lines[1:]:
        if not line:
            continue
        f = line.split(",")
        try:
            if not raw:
                if len(f) != 4:
                    raise ValueError("bad field count")
                out.append(RegressionSample((float(f[0]), float(f[1]), float(f[2])),
                                            float(f[3])))
            else:
                if len(f) != 7:
                    raise ValueError("bad field count")
                st = DatasetStats(int(f[0]), int(f[1]), [int(d) for d in f[2].split("-")])
                out.append(RegressionSample(comp_features(st, (int(f[3]), int(f[4]), int(f[5]))),
                                            float(f[6])))
        except (ValueError, ContractError) as exc:
            raise IoError("BadFormat", f"sample log {path}: bad row '{line}': {exc}")
    return out


__all__ = ["DatasetStats", "MachineParams", "PerfCoefficients", "ConfigPrediction",
           "RegressionSample", "SplitReport", "IoError", "default_coefficients",
           "comp_features", "predict_spmm_time", "effective_bandwidth",
           "ring_collective_seconds", "predict_comm_time", "training_collective_volumes",
           "fit_regression", "fit_with_split", "enumerate_configs", "rank_configs",
           "machine_from_json_file", "coefficients_from_json_file",
           "coefficients_to_json_file", "samples_from_csv_file"]
