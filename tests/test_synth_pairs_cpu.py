"""The SBM / Erdős restatement (oracle/restate.py sbm_edges / synth_sbm /
synth_erdos, graph.hpp:254-289) and the closed-form pair-draw indexing the
device generators use (csrc/rmat.cu pair_rows_kernel: pair (u, v), u < v,
takes u64 draw t = sum_{i<u} (n - 1 - i) + (v - u - 1) of Philox(seed, 5)),
pinned to the compiled reference's synth_sbm / synth_erdos on CPU —
features, labels and mask included."""
import numpy as np
import pytest

from oracle import ref
from paper_2505_04083_b200.philox import philox_doubles


def chunk_index(total, parts, pos):
    base, rem = total // parts, total % parts
    pos = np.asarray(pos, np.int64)
    return np.where(pos < rem * (base + 1), pos // (base + 1),
                    rem + (pos - rem * (base + 1)) // max(base, 1))


def pair_edges(n, communities, p_in, p_out, seed):
    u, v = np.triu_indices(n, k=1)          # lexicographic (u, v), u < v
    t = u * (n - 1) - u * (u - 1) // 2 + (v - u - 1)
    assert np.array_equal(t, np.arange(t.size))  # closed form = running index
    r = philox_doubles(seed, 5, t.size)
    same = chunk_index(n, communities, u) == chunk_index(n, communities, v)
    keep = r < np.where(same, p_in, p_out)
    return np.stack([u[keep], v[keep]], 1).astype(np.uint32)


@pytest.mark.parametrize("n,c,pi,po,seed", [(200, 4, 0.2, 0.02, 23), (97, 3, 0.5, 0.05, 7),
                                            (64, 64, 0.9, 0.01, 2)])
def test_sbm_pair_indexing_matches_reference(n, c, pi, po, seed):
    want = ref.synth_sbm(n, c, pi, po, 2, 2, seed).arrays()["edges"]
    assert np.array_equal(pair_edges(n, c, pi, po, seed), want)


@pytest.mark.parametrize("n,p,seed", [(50, 0.1, 21), (120, 0.03, 7), (8, 0.4, 13)])
def test_erdos_pair_indexing_matches_reference(n, p, seed):
    want = ref.synth_erdos(n, p, 2, 2, seed).arrays()["edges"]
    assert np.array_equal(pair_edges(n, 1, p, p, seed), want)


@pytest.mark.parametrize("n,c,pi,po,seed,frac", [(300, 4, 0.2, 0.02, 31, 1.0),
                                                 (48, 4, 0.3, 0.02, 3, 0.7)])
def test_restated_synth_sbm_matches_reference(n, c, pi, po, seed, frac):
    from oracle import restate
    got = restate.synth_sbm(n, c, pi, po, 6, 3, seed, frac)
    want = ref.synth_sbm(n, c, pi, po, 6, 3, seed, train_fraction=frac).arrays()
    assert np.array_equal(got["edges"], want["edges"])
    assert np.array_equal(got["features"], want["features"])
    assert np.array_equal(got["labels"], want["labels"])
    assert np.array_equal(got["mask"], want["mask"])


def test_restated_synth_erdos_matches_reference():
    from oracle import restate
    got = restate.synth_erdos(200, 0.05, 4, 2, 7)
    want = ref.synth_erdos(200, 0.05, 4, 2, 7).arrays()
    assert np.array_equal(got["edges"], want["edges"])
    assert np.array_equal(got["labels"], want["labels"])
