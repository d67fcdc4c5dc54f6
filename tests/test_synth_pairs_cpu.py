"""The pair-draw indexing the device SBM / Erdős generators use
(csrc/rmat.cu pair_rows_kernel: pair (u, v), u < v, takes u64 draw
t = sum_{i<u} (n - 1 - i) + (v - u - 1) of Philox(seed, 5)), restated in
numpy and pinned to the compiled reference's synth_sbm / synth_erdos
(graph.hpp:254-289) on CPU."""
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
