"""PLXS dataset shard files and the per-rank file loader — the reference's
shard_io.hpp (26-486) and trainer.hpp:252-438 (load_rank_shards,
load_preprocessed, file_handle) over the library's C ABI.

Files are written and read by the library (csrc/shard_io.cpp: byte-identical
writer, FNV-1a 64 checked reader that streams sections into HBM through a
pinned double buffer); blocks are cut and merged on the GPU (pk_csr_block,
pk_csr_hconcat). The JSON manifest is handled here, in the reference's
format (nlohmann dump(2): sorted keys, two-space indent).
"""

import ctypes as C
import json
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from . import _capi, graph
from ._capi import ContractError, IoError, call
from .kernels import DeviceCsr
from .layout import (GridConfig, adjacency_block_range, chunk_start, feature_slice,
                     label_row_range, needed_adjacency_keys)

SECTIONS = ("even", "odd", "features", "labels")
CSR_EVEN, CSR_ODD, FEATURES, LABELS = range(4)


@dataclass
class ShardFileInfo:
    """shard_io.hpp:37-45."""
    i: int
    j: int
    path: str
    row0: int
    row1: int
    col0: int
    col1: int
    fcol0: int
    fcol1: int
    nnz_even: int = 0
    nnz_odd: int = 0
    checksum: List[int] = field(default_factory=lambda: [0, 0, 0, 0])

    def ranges(self):
        return [self.row0, self.row1, self.col0, self.col1, self.fcol0, self.fcol1]


@dataclass
class ShardManifest:
    """shard_io.hpp:47-65."""
    dataset: str
    dir: str
    precision: int
    n: int
    feat_dim: int
    classes: int
    p: int
    q: int
    perm_seed: int
    nnz_even: int
    nnz_odd: int
    files: List[ShardFileInfo]

    @property
    def num_classes(self):  # DatasetHandle's shape metadata (trainer.hpp:443-450)
        return self.classes

    def file(self, i, j) -> ShardFileInfo:
        if not (0 <= i < self.p and 0 <= j < self.q):
            raise ContractError("manifest: shard index out of range")
        return self.files[i * self.q + j]

    def file_path(self, i, j):
        return os.path.join(self.dir, self.file(i, j).path)


def _manifest_json(m: ShardManifest):
    files = []
    for f in m.files:
        files.append({"i": f.i, "j": f.j, "path": f.path, "row0": f.row0, "row1": f.row1,
                      "col0": f.col0, "col1": f.col1, "fcol0": f.fcol0, "fcol1": f.fcol1,
                      "nnz_even": f.nnz_even, "nnz_odd": f.nnz_odd,
                      "sum_even": format(f.checksum[CSR_EVEN], "x"),
                      "sum_odd": format(f.checksum[CSR_ODD], "x"),
                      "sum_features": format(f.checksum[FEATURES], "x"),
                      "sum_labels": format(f.checksum[LABELS], "x")})
    return {"format": "plxs-1", "dataset": m.dataset, "rng": "philox4x32-10",
            "perm_seed": m.perm_seed, "precision": "f32" if m.precision == 4 else "f64",
            "n": m.n, "feat_dim": m.feat_dim, "classes": m.classes, "p": m.p, "q": m.q,
            "nnz_even": m.nnz_even, "nnz_odd": m.nnz_odd, "checksum": "fnv1a64",
            "files": files}


def _host(t: torch.Tensor) -> np.ndarray:
    return np.ascontiguousarray(t.detach().cpu().numpy())


def write_shards(pre: "graph.PreprocessedDataset", p: int, q: int, directory: str,
                 dataset_name: str) -> ShardManifest:
    """write_shards (shard_io.hpp:278-414): a p x q grid of PLXS files — rows
    of both adjacency variants by chunk(n, p), columns by chunk(n, q),
    feature columns by chunk(feat_dim, q), the row block's labels and masks
    in every file of the stripe — plus manifest.json. Blocks are cut on the
    GPU; the files are byte-identical to the reference's."""
    if p < 1 or q < 1:
        raise ContractError("write_shards: p and q must be >= 1")
    os.makedirs(directory, exist_ok=True)
    m = ShardManifest(dataset_name, directory, 4, pre.n, pre.feat_dim, pre.num_classes, p, q,
                      pre.perm_seed, pre.a_even.nnz, pre.a_odd.nnz, [])
    for i in range(p):
        r0, r1 = chunk_start(pre.n, p, i), chunk_start(pre.n, p, i + 1)
        lab = [_host(t[r0:r1]) for t in (pre.labels_row_order, pre.labels_col_order,
                                         pre.mask_row_order, pre.mask_col_order)]
        lab[0], lab[1] = lab[0].view(np.uint32), lab[1].view(np.uint32)
        for j in range(q):
            c0, c1 = chunk_start(pre.n, q, j), chunk_start(pre.n, q, j + 1)
            f0, f1 = chunk_start(pre.feat_dim, q, j), chunk_start(pre.feat_dim, q, j + 1)
            info = ShardFileInfo(i, j, f"shard_{i}_{j}.plxs", r0, r1, c0, c1, f0, f1)
            blocks = [graph.csr_block(a, r0, r1, c0, c1) for a in (pre.a_even, pre.a_odd)]
            info.nnz_even, info.nnz_odd = blocks[0].nnz, blocks[1].nnz
            host = [b.to_host() for b in blocks]
            keep = []

            def csr_struct(b, h):
                rp, ci, v = (np.ascontiguousarray(x) for x in h)
                keep.extend([rp, ci, v])
                return _capi.pk_plxs_csr_host(b.rows, b.cols, b.nnz, rp.ctypes.data,
                                              ci.ctypes.data, v.ctypes.data)
            even, odd = (csr_struct(b, h) for b, h in zip(blocks, host))
            feats = np.ascontiguousarray(_host(pre.features[r0:r1, f0:f1]), np.float32)
            ranges = np.array(info.ranges(), np.uint64)
            sums = np.zeros(4, np.uint64)
            call("pk_plxs_write", os.path.join(directory, info.path).encode(),
                 ranges.ctypes.data, 4, C.byref(even), C.byref(odd), feats.shape[0],
                 feats.shape[1], feats.ctypes.data, r1 - r0, lab[0].ctypes.data,
                 lab[1].ctypes.data, lab[2].ctypes.data, lab[3].ctypes.data, sums.ctypes.data)
            info.checksum = [int(x) for x in sums]
            m.files.append(info)
    path = os.path.join(directory, "manifest.json")
    try:
        with open(path, "w") as f:
            f.write(json.dumps(_manifest_json(m), indent=2, sort_keys=True) + "\n")
    except OSError as exc:
        raise IoError("WriteFailed", f"cannot write manifest {path}: {exc}")
    return m


def load_manifest(path_or_dir: str) -> ShardManifest:
    """load_manifest (shard_io.hpp:416-486), with the reference's structural
    checks and error codes."""
    path = path_or_dir
    if os.path.isdir(path):
        path = os.path.join(path, "manifest.json")
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise IoError("MissingFile", f"cannot open manifest {path}")
    try:
        j = json.loads(text)
        files = [ShardFileInfo(int(x["i"]), int(x["j"]), str(x["path"]), int(x["row0"]),
                               int(x["row1"]), int(x["col0"]), int(x["col1"]),
                               int(x["fcol0"]), int(x["fcol1"]), int(x["nnz_even"]),
                               int(x["nnz_odd"]),
                               [int(x["sum_even"], 16), int(x["sum_odd"], 16),
                                int(x["sum_features"], 16), int(x["sum_labels"], 16)])
                 for x in j["files"]]
        m = ShardManifest(j.get("dataset", ""), os.path.dirname(path) or ".",
                          4 if j["precision"] == "f32" else 8, int(j["n"]), int(j["feat_dim"]),
                          int(j["classes"]), int(j["p"]), int(j["q"]), int(j["perm_seed"]),
                          int(j["nnz_even"]), int(j["nnz_odd"]), files)
    except (ValueError, KeyError, TypeError) as exc:
        raise IoError("BadFormat", f"manifest {path}: {exc}")
    if len(m.files) != m.p * m.q:
        raise IoError("ManifestMismatch", f"manifest lists {len(m.files)} files but the grid "
                                          f"is {m.p}x{m.q}")
    ordered: List[Optional[ShardFileInfo]] = [None] * (m.p * m.q)
    for f in m.files:
        if not (0 <= f.i < m.p and 0 <= f.j < m.q) or ordered[f.i * m.q + f.j] is not None:
            raise IoError("ManifestMismatch", "manifest shard indices are not a p x q grid")
        ordered[f.i * m.q + f.j] = f
    m.files = ordered
    if sum(f.nnz_even for f in m.files) != m.nnz_even or \
            sum(f.nnz_odd for f in m.files) != m.nnz_odd:
        raise IoError("ManifestMismatch", "per-shard nnz does not sum to the manifest total")
    return m


class ShardFileReader:
    """ShardFileReader (shard_io.hpp:90-276); sections stream into HBM."""

    def __init__(self, manifest: ShardManifest, i: int, j: int):
        self.info = manifest.file(i, j)
        self.path = manifest.file_path(i, j)
        self.precision = manifest.precision
        ranges = np.array(self.info.ranges(), np.uint64)
        h = C.c_void_p()
        call("pk_plxs_open", self.path.encode(), ranges.ctypes.data, manifest.precision,
             C.byref(h))
        self.h = h

    def close(self):
        if self.h:
            _capi.lib().pk_plxs_close(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def bytes_read(self):
        out = C.c_uint64()
        call("pk_plxs_info", self.h, None, None, C.byref(out))
        return out.value

    def _stream(self):
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def read_csr_rows(self, section: int, r0: int, r1: int, device=True):
        """Rows [r0, r1) of one adjacency variant (shard_io.hpp:120-151):
        into HBM as a DeviceCsr, or (device=False) host arrays
        (rows, cols, row_ptr, col_idx, values)."""
        rows, cols, e0, e1 = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        call("pk_plxs_csr_extent", self.h, section, r0, r1, C.byref(rows), C.byref(cols), None,
             C.byref(e0), C.byref(e1))
        nnz = e1.value - e0.value
        if not device:
            rp = np.empty(r1 - r0 + 1, np.uint64)
            ci = np.empty(nnz, np.uint32)
            v = np.empty(nnz, np.float32 if self.precision == 4 else np.float64)
            call("pk_plxs_read_csr_rows", self.h, section, r0, r1, self.info.checksum[section],
                 rp.ctypes.data, ci.ctypes.data, v.ctypes.data, 0, None)
            return r1 - r0, cols.value, rp, ci, v
        if self.precision != 4:
            raise ContractError("read_csr_rows: device reads hold f32 shards")
        rp = np.empty(r1 - r0 + 1, np.uint64)
        ci = torch.empty(nnz, dtype=torch.int32, device="cuda")
        v = torch.empty(nnz, dtype=torch.float32, device="cuda")
        call("pk_plxs_read_csr_rows", self.h, section, r0, r1, self.info.checksum[section],
             rp.ctypes.data, ci.data_ptr() if nnz else None, v.data_ptr() if nnz else None, 1,
             self._stream())
        rpt = torch.from_numpy(rp.view(np.int64)).cuda()
        return DeviceCsr(r1 - r0, cols.value, rpt, ci, v)

    def read_feature_rows(self, r0: int, r1: int, device=True):
        """Feature rows [r0, r1) of the file's column chunk (shard_io.hpp:158-176)."""
        cols = self.info.fcol1 - self.info.fcol0
        if not device:
            out = np.empty((r1 - r0, cols), np.float32 if self.precision == 4 else np.float64)
            call("pk_plxs_read_feature_rows", self.h, r0, r1, self.info.checksum[FEATURES],
                 out.ctypes.data, 0, None)
            return out
        out = torch.empty((r1 - r0, cols), dtype=torch.float32, device="cuda")
        call("pk_plxs_read_feature_rows", self.h, r0, r1, self.info.checksum[FEATURES],
             out.data_ptr() if out.numel() else None, 1, self._stream())
        return out

    def read_labels(self, r0: int, r1: int):
        n = r1 - r0
        lr, lc = np.empty(n, np.uint32), np.empty(n, np.uint32)
        mr, mc = np.empty(n, np.uint8), np.empty(n, np.uint8)
        call("pk_plxs_read_labels", self.h, r0, r1, self.info.checksum[LABELS], lr.ctypes.data,
             lc.ctypes.data, mr.ctypes.data, mc.ctypes.data)
        return lr, lc, mr, mc


def _vstack(blocks: List[DeviceCsr], cols: int) -> DeviceCsr:
    """Row-wise concatenation of CSR blocks with equal column counts."""
    if len(blocks) == 1:
        return blocks[0]
    rps, base = [], 0
    for k, b in enumerate(blocks):
        rp = b.row_ptr if k == 0 else b.row_ptr[1:]
        rps.append(rp + base)
        base += b.nnz
    return DeviceCsr(sum(b.rows for b in blocks), cols, torch.cat(rps),
                     torch.cat([b.col_idx for b in blocks]), torch.cat([b.values for b in blocks]))


def _merge(pieces: List[DeviceCsr], col0: List[int], c0: int, c1: int) -> DeviceCsr:
    """Per-row merge of column pieces, kept columns in [c0, c1) renumbered
    from c0 (trainer.hpp:296-306) — pk_csr_hconcat on the device."""
    arr = (_capi.pk_csr * len(pieces))(*[p._view for p in pieces])
    origins = np.array(col0, np.uint64)
    out = _capi.pk_csr_owned()
    call("pk_csr_hconcat", arr, origins.ctypes.data, len(pieces), c0, c1, C.byref(out),
         C.c_void_p(torch.cuda.current_stream().cuda_stream))
    return DeviceCsr._from_owned(out)


@dataclass
class RankTensors:
    """RankTensors (trainer.hpp:217-224), device resident."""
    adj: dict                 # (plane, parity) -> (block, transpose)
    f0: torch.Tensor
    labels: torch.Tensor      # int32 (u32 bits)
    mask: torch.Tensor        # uint8
    bytes_read: int = 0
    files_read: int = 0


def load_rank_shards(mani: ShardManifest, grid: GridConfig, coords, num_layers: int
                     ) -> RankTensors:
    """load_rank_shards (trainer.hpp:256-384): reads only the stripe / section
    slices overlapping this rank's blocks and merges them on the device;
    blocks shared by several planes are assembled once."""
    if mani.precision != 4:
        raise ContractError("load_rank_shards: scalar type does not match manifest precision")
    n = mani.n
    readers = {}

    def reader(i, j):
        if (i, j) not in readers:
            readers[(i, j)] = ShardFileReader(mani, i, j)
        return readers[(i, j)]

    def assemble(sec, r0, r1, c0, c1):
        stripes = []
        for i in range(mani.p):
            stripe = mani.file(i, 0)
            sr0, sr1 = max(r0, stripe.row0), min(r1, stripe.row1)
            if sr0 >= sr1:
                continue
            pieces, origins = [], []
            for j in range(mani.q):
                info = mani.file(i, j)
                if info.col1 <= c0 or info.col0 >= c1:
                    continue
                pieces.append(reader(i, j).read_csr_rows(sec, sr0 - info.row0, sr1 - info.row0))
                origins.append(info.col0)
            stripes.append(_merge(pieces, origins, c0, c1))
        if not stripes:  # zero-extent block
            return DeviceCsr(r1 - r0, c1 - c0, torch.zeros(r1 - r0 + 1, dtype=torch.int64,
                                                           device="cuda"),
                             torch.empty(0, dtype=torch.int32, device="cuda"),
                             torch.empty(0, dtype=torch.float32, device="cuda"))
        return _vstack(stripes, c1 - c0)

    coords = tuple(coords)
    memo, adj = {}, {}
    for plane, parity in needed_adjacency_keys(num_layers):
        sec = CSR_ODD if parity else CSR_EVEN
        r0, r1, c0, c1 = adjacency_block_range(grid, plane, coords, n)
        key = (sec, r0, r1, c0, c1)
        if key not in memo:
            memo[key] = assemble(sec, r0, r1, c0, c1)
        block = memo[key]
        adj[(plane, parity)] = (block, graph.csr_transpose(block))

    # trainable feature shard
    fr0, fr1, fc0, fc1 = feature_slice(grid, coords, n, mani.feat_dim)
    f0 = torch.zeros((fr1 - fr0, fc1 - fc0), dtype=torch.float32, device="cuda")
    for i in range(mani.p):
        stripe = mani.file(i, 0)
        sr0, sr1 = max(fr0, stripe.row0), min(fr1, stripe.row1)
        if sr0 >= sr1:
            continue
        for j in range(mani.q):
            info = mani.file(i, j)
            sc0, sc1 = max(fc0, info.fcol0), min(fc1, info.fcol1)
            if sc0 >= sc1:
                continue
            rows = reader(i, j).read_feature_rows(sr0 - info.row0, sr1 - info.row0)
            f0[sr0 - fr0:sr1 - fr0, sc0 - fc0:sc1 - fc0] = \
                rows[:, sc0 - info.fcol0:sc1 - info.fcol0]

    # final-parity labels and mask of this rank's logit rows
    parity = (num_layers - 1) % 2
    lr0, lr1 = label_row_range(grid, coords, n, num_layers)
    labels = np.zeros(lr1 - lr0, np.uint32)
    mask = np.zeros(lr1 - lr0, np.uint8)
    for i in range(mani.p):
        stripe = mani.file(i, 0)
        sr0, sr1 = max(lr0, stripe.row0), min(lr1, stripe.row1)
        if sr0 >= sr1:
            continue
        j_pick = 0  # labels repeat across the stripe: a file the feature columns overlap
        for j in range(mani.q):
            info = mani.file(i, j)
            if info.fcol1 > fc0 and info.fcol0 < fc1:
                j_pick = j
                break
        lr, lc, mr, mc = reader(i, j_pick).read_labels(sr0 - stripe.row0, sr1 - stripe.row0)
        labels[sr0 - lr0:sr1 - lr0] = lc if parity else lr
        mask[sr0 - lr0:sr1 - lr0] = mc if parity else mr
    out = RankTensors(adj, f0, torch.from_numpy(labels.view(np.int32)).cuda(),
                      torch.from_numpy(mask).cuda())
    out.files_read = len(readers)
    out.bytes_read = sum(r.bytes_read() for r in readers.values())
    return out


def load_preprocessed(mani: ShardManifest) -> "graph.PreprocessedDataset":
    """load_preprocessed (trainer.hpp:386-438): the whole dataset back into
    HBM, every section checksum verified (full-range reads)."""
    if mani.precision != 4:
        raise ContractError("load_preprocessed: f32 manifests only")
    n = mani.n
    variants = []
    for sec in (CSR_EVEN, CSR_ODD):
        stripes = []
        for i in range(mani.p):
            pieces, origins = [], []
            for j in range(mani.q):
                info = mani.file(i, j)
                pieces.append(ShardFileReader(mani, i, j).read_csr_rows(
                    sec, 0, info.row1 - info.row0))
                origins.append(info.col0)
            stripes.append(_merge(pieces, origins, 0, n))
        variants.append(_vstack(stripes, n))
    features = torch.zeros((n, mani.feat_dim), dtype=torch.float32, device="cuda")
    lab = [np.zeros(n, np.uint32), np.zeros(n, np.uint32), np.zeros(n, np.uint8),
           np.zeros(n, np.uint8)]
    for i in range(mani.p):
        for j in range(mani.q):
            info = mani.file(i, j)
            rd = ShardFileReader(mani, i, j)
            features[info.row0:info.row1, info.fcol0:info.fcol1] = \
                rd.read_feature_rows(0, info.row1 - info.row0)
            got = rd.read_labels(0, info.row1 - info.row0)  # verifies every file's labels
            if j == 0:
                for dst, src in zip(lab, got):
                    dst[info.row0:info.row1] = src
    t = [torch.from_numpy(x.view(np.int32) if x.dtype == np.uint32 else x).cuda() for x in lab]
    return graph.PreprocessedDataset(n, mani.feat_dim, mani.classes, mani.perm_seed,
                                     variants[0], variants[1], features, t[0], t[1], t[2], t[3])
