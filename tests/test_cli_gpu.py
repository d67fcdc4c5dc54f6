"""CLI end to end on the GPU: preprocess writes the same PLXS set as the
reference's `preprocess` would (write_shards of the same dataset), train
reads it back per rank and writes metrics.csv / summary.csv / model.plxm."""

import os
import struct
import subprocess
import sys

import numpy as np
import pytest

from oracle import ref

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args):
    r = subprocess.run([sys.executable, "-m", "paper_2505_04083_b200", *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    return r.returncode, r.stdout, r.stderr


def test_preprocess_then_train(cuda, tmp_path):
    shards, run = str(tmp_path / "shards"), str(tmp_path / "run")
    rc, out, err = _cli("preprocess", "--synth", "rmat:scale=10,edges=9000", "--feat-dim", "11",
                        "--classes", "6", "--p", "2", "--q", "2", "--seed", "3", "--out", shards,
                        "--name", "cli")
    assert rc == 0, err
    theirs = str(tmp_path / "theirs")
    ref.write_shards(ref.synth_rmat(10, 9000, 11, 6, seed=3).preprocess(3), 2, 2, theirs, "cli")
    for name in sorted(os.listdir(theirs)):
        assert open(os.path.join(shards, name), "rb").read() == \
            open(os.path.join(theirs, name), "rb").read(), name
    rc, out, err = _cli("train", "--manifest", shards, "--grid", "1,1,1", "--epochs", "3",
                        "--layers", "16,16", "--mode", "parity", "--out", run)
    assert rc == 0, err
    rows = open(os.path.join(run, "metrics.csv")).read().splitlines()
    assert rows[0].startswith("epoch,rank,loss,accuracy") and len(rows) == 1 + 3 * 2
    assert os.path.exists(os.path.join(run, "summary.csv"))
    comm = open(os.path.join(run, "comm_stats.csv")).read().splitlines()
    assert comm[0] == "rank,axis,collective,calls,ring_bytes" and len(comm) == 1 + 9
    blob = open(os.path.join(run, "model.plxm"), "rb").read()
    assert blob[:4] == b"PLXM" and struct.unpack("<III", blob[4:16]) == (1, 4, 3)
    # the loss curve is the reference serial trainer's (PARITY, 1x1x1)
    want, _ = ref.synth_rmat(10, 9000, 11, 6, seed=3).preprocess(3).serial(
        hidden=(16, 16), seed=0).train(3)
    got = [float(r.split(",")[2]) for r in rows[1:] if r.split(",")[1] == "global"]
    assert np.allclose(got, want, rtol=1e-5), (got, want)


@pytest.mark.parametrize("spec,want", [
    ("sbm:n=600,k=4,p_in=0.2,p_out=0.01", lambda: ref.synth_sbm(600, 4, 0.2, 0.01, 9, 5, 4,
                                                                 train_fraction=0.8)),
    ("erdos:n=500,p=0.02", lambda: ref.synth_erdos(500, 0.02, 9, 5, 4, train_fraction=0.8)),
])
def test_preprocess_sbm_erdos_shards_match_reference(cuda, tmp_path, spec, want):
    """tools/main.cpp:70-93 synth kinds: the shard set of an SBM / Erdős
    dataset is byte-identical to the reference's write_shards."""
    shards, theirs = str(tmp_path / "shards"), str(tmp_path / "theirs")
    rc, out, err = _cli("preprocess", "--synth", spec, "--feat-dim", "9", "--classes", "5",
                        "--train-fraction", "0.8", "--p", "2", "--q", "3", "--seed", "4",
                        "--out", shards, "--name", "pairs")
    assert rc == 0, err
    ref.write_shards(want().preprocess(4), 2, 3, theirs, "pairs")
    for name in sorted(os.listdir(theirs)):
        assert open(os.path.join(shards, name), "rb").read() == \
            open(os.path.join(theirs, name), "rb").read(), name


def test_preprocess_unknown_synth_kind(cuda, tmp_path):
    rc, out, err = _cli("preprocess", "--synth", "kron:n=5", "--out", str(tmp_path / "x"))
    assert rc != 0 and "expected sbm, erdos or rmat" in err
