"""PLXS shard files on the GPU: the writer (blocks cut on the device) is
byte-identical to the reference's write_shards, device reads stream the
sections into HBM with checksums verified, and load_rank_shards /
load_preprocessed assemble exactly what the reference's do (trainer.hpp:
252-438) on every rank of several grids — including bytes and files read."""

import os

import numpy as np
import pytest

from oracle import ref

pytestmark = pytest.mark.gpu


def _mods():
    from paper_2505_04083_b200 import graph, layout, shard_io
    return graph, layout, shard_io


def _csr_eq(dev, want):
    rp, ci, v = dev.to_host()
    assert np.array_equal(rp.astype(np.uint64), want[0])
    assert np.array_equal(ci.astype(np.uint32), want[1])
    assert np.array_equal(np.asarray(v, np.float32).view(np.uint32), want[2].view(np.uint32))


@pytest.fixture(scope="module")
def datasets(tmp_path_factory):
    graph, _, shard_io = _mods()
    pre = graph.preprocess(graph.synth_rmat(10, 9000, 11, 6, seed=3), perm_seed=3)
    rpre = ref.synth_rmat(10, 9000, 11, 6, seed=3).preprocess(3)
    ours = str(tmp_path_factory.mktemp("ours"))
    theirs = str(tmp_path_factory.mktemp("theirs"))
    shard_io.write_shards(pre, 3, 2, ours, "rmat10")
    ref.write_shards(rpre, 3, 2, theirs, "rmat10")
    return pre, rpre, ours, theirs


def test_writer_byte_identical(cuda, datasets):
    _, _, ours, theirs = datasets
    names = sorted(os.listdir(theirs))
    assert sorted(os.listdir(ours)) == names
    for name in names:
        with open(os.path.join(ours, name), "rb") as a, open(os.path.join(theirs, name), "rb") as b:
            assert a.read() == b.read(), name


def test_load_preprocessed_matches_reference(cuda, datasets):
    _, _, shard_io = _mods()
    _, rpre, _, theirs = datasets
    got = shard_io.load_preprocessed(shard_io.load_manifest(theirs))
    want = ref.load_preprocessed(theirs)
    for parity, a in ((0, got.a_even), (1, got.a_odd)):
        _csr_eq(a, want.csr(parity).arrays())
    arr = want.arrays()
    assert np.array_equal(got.features.cpu().numpy(), arr["features"])
    assert np.array_equal(got.labels_row_order.cpu().numpy().view(np.uint32), arr["labels_row"])
    assert np.array_equal(got.mask_col_order.cpu().numpy(), arr["mask_col"])


@pytest.mark.parametrize("grid", [(1, 1, 1), (2, 1, 2), (1, 3, 2), (2, 2, 2), (4, 1, 1)])
@pytest.mark.parametrize("layers", [2, 3])
def test_load_rank_shards_matches_reference(cuda, datasets, grid, layers):
    _, layout, shard_io = _mods()
    _, _, _, theirs = datasets
    mani = shard_io.load_manifest(theirs)
    g = layout.GridConfig(*grid)
    for r in range(g.size):
        c = g.coords_of(r)
        got = shard_io.load_rank_shards(mani, g, c, layers)
        want = ref.RankShards.load(theirs, grid, c, layers)
        for (plane, parity), (blk, blk_t) in got.adj.items():
            _csr_eq(blk, want.adj(plane, parity).arrays())
            _csr_eq(blk_t, want.adj(plane, parity, transposed=True).arrays())
        f0, labels, mask = want.arrays()
        assert np.array_equal(got.f0.cpu().numpy(), f0)
        assert np.array_equal(got.labels.cpu().numpy().view(np.uint32), labels)
        assert np.array_equal(got.mask.cpu().numpy(), mask)
        info = want.info()
        assert (got.files_read, got.bytes_read) == (info["files_read"], info["bytes_read"]), c


def test_device_read_detects_corruption(cuda, datasets, tmp_path):
    _, _, shard_io = _mods()
    from paper_2505_04083_b200._capi import IoError
    import shutil
    _, _, ours, _ = datasets
    c = tmp_path / "c"
    shutil.copytree(ours, c)
    mani = shard_io.load_manifest(str(c))
    f = mani.file(1, 1)
    path = os.path.join(str(c), f.path)
    blob = bytearray(open(path, "rb").read())
    rows = f.row1 - f.row0
    blob[-(rows * 10 + 8) - 40] ^= 0x01  # a feature value
    open(path, "wb").write(bytes(blob))
    r = shard_io.ShardFileReader(mani, 1, 1)
    r.read_csr_rows(0, 0, rows)          # intact sections still read
    with pytest.raises(IoError) as e:
        r.read_feature_rows(0, rows)
    assert e.value.code == "ChecksumMismatch"
    r.read_feature_rows(2, 9)            # partial reads are not checksummed (reference too)


def test_engine_from_shard_files_matches_in_memory_load(cuda, datasets):
    """The file_handle path: an engine loaded with only this rank's blocks
    read from the files runs the same pass as one loaded from the in-memory
    dataset (1x1x1; multi-rank grids go through test_multigpu_gpu.py)."""
    _, layout, shard_io = _mods()
    from paper_2505_04083_b200 import trainer as tr
    pre, _, ours, _ = datasets
    mani = shard_io.load_manifest(ours)
    opts = tr.TrainOptions(hidden_dims=[16, 16], mode=tr.PK_MODE_PARITY, hub_threshold=64)
    outs = []
    for src in (pre, mani):
        eng = tr.RankEngine(pre.n, pre.feat_dim, pre.num_classes, layout.GridConfig(1, 1, 1), 0,
                            opts)
        eng.load(src)
        m = [eng.train_epoch(e) for e in range(2)]
        outs.append(([x["loss"] for x in m], eng.tensor(tr.PK_T_FOUT).cpu().numpy()))
        eng.close()
    assert outs[0][0] == outs[1][0]
    assert np.array_equal(outs[0][1].view(np.uint32), outs[1][1].view(np.uint32))
