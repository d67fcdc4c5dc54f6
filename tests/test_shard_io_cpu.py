"""PLXS shard files on the host (shard_io.hpp): the library's reader on
files the compiled reference wrote — manifest, CSR / feature / label
sections, checksums, bytes read — and the reference's error codes for
missing, corrupt, truncated and inconsistent files. CPU only; device reads,
the writer and the per-rank loader are in test_shard_io_gpu.py."""

import json
import os
import shutil

import numpy as np
import pytest

from oracle import ref
from paper_2505_04083_b200 import shard_io
from paper_2505_04083_b200._capi import IoError


@pytest.fixture(scope="module")
def written(tmp_path_factory):
    d = tmp_path_factory.mktemp("plxs")
    pre = ref.synth_rmat(9, 3000, 8, 5, seed=2).preprocess(1)
    ref.write_shards(pre, 2, 3, str(d), "rmat9")
    return pre, str(d)


def test_manifest_matches_reference(written):
    pre, d = written
    m = shard_io.load_manifest(d)
    info = pre.info()
    assert (m.p, m.q, m.n, m.feat_dim, m.classes, m.precision) == (2, 3, info["n"],
                                                                    info["feat"], 5, 4)
    assert (m.nnz_even, m.nnz_odd) == (info["nnz_even"], info["nnz_odd"])
    assert [(f.i, f.j) for f in m.files] == [(i, j) for i in range(2) for j in range(3)]
    raw = json.load(open(os.path.join(d, "manifest.json")))
    assert m.files[4].checksum[0] == int(raw["files"][4]["sum_even"], 16)


def test_host_reads_match_reference_blocks(written):
    pre, d = written
    m = shard_io.load_manifest(d)
    arrays = pre.arrays()
    for f in m.files:
        r = shard_io.ShardFileReader(m, f.i, f.j)
        for sec in (0, 1):
            rows, cols, rp, ci, v = r.read_csr_rows(sec, 0, f.row1 - f.row0, device=False)
            want = pre.csr(sec).block(f.row0, f.row1, f.col0, f.col1).arrays()
            assert np.array_equal(rp, want[0]) and np.array_equal(ci, want[1])
            assert np.array_equal(v.view(np.uint32), want[2].view(np.uint32))
            # partial row range, rebased
            rows, cols, rp, ci, v = r.read_csr_rows(sec, 3, 40, device=False)
            pw = pre.csr(sec).block(f.row0 + 3, f.row0 + 40, f.col0, f.col1).arrays()
            assert np.array_equal(rp, pw[0]) and np.array_equal(ci, pw[1])
        feats = r.read_feature_rows(0, f.row1 - f.row0, device=False)
        assert np.array_equal(feats, arrays["features"][f.row0:f.row1, f.fcol0:f.fcol1])
        lr, lc, mr, mc = r.read_labels(0, f.row1 - f.row0)
        assert np.array_equal(lr, arrays["labels_row"][f.row0:f.row1])
        assert np.array_equal(mc, arrays["mask_col"][f.row0:f.row1])


def _copy(d, tmp_path):
    out = tmp_path / "copy"
    shutil.copytree(d, out)
    return str(out)


def test_error_codes(written, tmp_path):
    _, d = written
    m = shard_io.load_manifest(d)
    f = m.files[0]
    rows = f.row1 - f.row0
    # checksum mismatch: one flipped byte inside the feature values (the
    # label section, 8 + 10 * rows bytes, closes the file)
    c = _copy(d, tmp_path)
    path = os.path.join(c, f.path)
    blob = bytearray(open(path, "rb").read())
    blob[-(rows * 10 + 8) - 100] ^= 0x40
    open(path, "wb").write(bytes(blob))
    mc = shard_io.load_manifest(c)
    r = shard_io.ShardFileReader(mc, 0, 0)
    with pytest.raises(IoError) as e:
        r.read_csr_rows(1, 0, rows, device=False)
        r.read_feature_rows(0, rows, device=False)
        r.read_labels(0, rows)
    assert e.value.code == "ChecksumMismatch"
    # truncated file
    open(path, "wb").write(bytes(blob[:200]))
    with pytest.raises(IoError) as e:
        shard_io.ShardFileReader(mc, 0, 0).read_csr_rows(0, 0, rows, device=False)
    assert e.value.code == "TruncatedFile"
    # not a shard file
    open(path, "wb").write(b"XXXX" + bytes(blob[4:]))
    with pytest.raises(IoError) as e:
        shard_io.ShardFileReader(mc, 0, 0)
    assert e.value.code == "BadFormat"
    # missing file / manifest
    os.remove(path)
    with pytest.raises(IoError) as e:
        shard_io.ShardFileReader(mc, 0, 0)
    assert e.value.code == "MissingFile"
    with pytest.raises(IoError) as e:
        shard_io.load_manifest(str(tmp_path / "nowhere"))
    assert e.value.code == "MissingFile"
    # manifest inconsistencies
    j = json.load(open(os.path.join(d, "manifest.json")))
    j["nnz_even"] += 1
    bad = tmp_path / "bad"
    bad.mkdir()
    (bad / "manifest.json").write_text(json.dumps(j))
    with pytest.raises(IoError) as e:
        shard_io.load_manifest(str(bad))
    assert e.value.code == "ManifestMismatch"
    j["nnz_even"] -= 1
    j["files"][2]["row1"] += 1  # ranges disagree with the file header
    (bad / "manifest.json").write_text(json.dumps(j))
    for f2 in m.files:
        shutil.copy(os.path.join(d, f2.path), bad / f2.path)
    mb = shard_io.load_manifest(str(bad))
    with pytest.raises(IoError) as e:
        shard_io.ShardFileReader(mb, 0, 2)
    assert e.value.code == "ManifestMismatch"
