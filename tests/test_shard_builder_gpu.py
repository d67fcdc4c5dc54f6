"""GPU shard builder vs the compiled reference (oracle/_ref): RMAT edges,
features, labels, normalize_adjacency, permutation pair, permute_csr,
preprocess, CSR transpose and block — all bit-exact
(reference cases: proj/tests/test_graph.cpp, test_kernels.cpp:154-173)."""

import numpy as np
import pytest
import torch

from oracle import ref

pytestmark = pytest.mark.gpu


def _g():
    from paper_2505_04083_b200 import graph
    return graph


def _k():
    from paper_2505_04083_b200 import kernels
    return kernels


def assert_csr_equal(dev, want):
    rp, ci, v = dev.to_host()
    wrp, wci, wv = want
    assert np.array_equal(rp, wrp)
    assert np.array_equal(ci, wci)
    assert np.array_equal(v.view(np.uint32), np.asarray(wv, np.float32).view(np.uint32))


@pytest.mark.parametrize("scale,edges,a,b,c", [(10, 20000, 0.57, 0.19, 0.19),
                                               (12, 50000, 0.25, 0.25, 0.25),
                                               (6, 1000, 0.45, 0.15, 0.15)])
def test_synth_rmat_bitwise(cuda, scale, edges, a, b, c):
    ds = _g().synth_rmat(scale, edges, 7, 5, seed=11, a=a, b=b, c=c)
    want = ref.synth_rmat(scale, edges, 7, 5, seed=11, a=a, b=b, c=c).arrays()
    assert np.array_equal(ds.edges.cpu().numpy().view(np.uint32), want["edges"])
    assert np.array_equal(ds.features.cpu().numpy(), want["features"])
    assert np.array_equal(ds.labels.cpu().numpy().view(np.uint32), want["labels"])


def test_normalize_known_answers(cuda):
    """test_graph.cpp:57-82: K2 -> 0.5 everywhere; star center 1/sqrt(8)."""
    g = _g()
    e = torch.tensor([[0, 1]], dtype=torch.int32, device=cuda)
    a = g.normalize_adjacency(2, e)
    rp, ci, v = a.to_host()
    assert rp.tolist() == [0, 2, 4] and ci.tolist() == [0, 1, 0, 1]
    assert np.all(v == 0.5)
    star = torch.tensor([[0, i] for i in range(1, 8)], dtype=torch.int32, device=cuda)
    s = g.normalize_adjacency(8, star)
    rp, ci, v = s.to_host()
    assert abs(v[0] - np.float32(1 / 8)) == 0  # (0,0): 1/sqrt(8*8)
    assert v[1] == np.float32(1.0 / np.sqrt(8.0 * 2.0))


@pytest.mark.parametrize("undirected", [True, False])
def test_normalize_bitwise(cuda, undirected):
    gr = ref.synth_rmat(11, 30000, 4, 3, seed=5)
    gr.set_undirected(undirected)
    want = gr.normalize().arrays()
    edges = torch.from_numpy(gr.arrays()["edges"].view(np.int32)).to(cuda)
    got = _g().normalize_adjacency(1 << 11, edges, undirected)
    assert_csr_equal(got, want)


def test_permutation_pair_bitwise():
    for n, seed in [(1, 0), (2, 3), (1000, 1), (100003, 9)]:
        r, c = _g().generate_permutation_pair(n, seed)
        wr, wc = ref.permutation_pair(n, seed)
        assert np.array_equal(r, wr) and np.array_equal(c, wc)


def test_preprocess_bitwise(cuda):
    ds = _g().synth_rmat(12, 40000, 16, 6, seed=3)
    pre = _g().preprocess(ds, perm_seed=7)
    rpre = ref.synth_rmat(12, 40000, 16, 6, seed=3).preprocess(7)
    assert_csr_equal(pre.a_even, rpre.csr(0).arrays())
    assert_csr_equal(pre.a_odd, rpre.csr(1).arrays())
    w = rpre.arrays()
    assert np.array_equal(pre.features.cpu().numpy(), w["features"])
    for got, key in ((pre.labels_row_order, "labels_row"), (pre.labels_col_order, "labels_col")):
        assert np.array_equal(got.cpu().numpy().view(np.uint32), w[key])
    assert np.array_equal(pre.mask_row_order.cpu().numpy(), w["mask_row"])


def test_csr_transpose_and_block_bitwise(cuda):
    rng = np.random.default_rng(0)
    rpre = ref.synth_rmat(10, 8000, 4, 3, seed=2).preprocess(1)
    a_ref = rpre.csr(0)
    rows, cols, _ = a_ref.info()
    a = _k().DeviceCsr.from_host(rows, cols, *a_ref.arrays())
    assert_csr_equal(_g().csr_transpose(a), a_ref.transpose().arrays())
    ranges = [tuple(sorted(rng.integers(0, rows + 1, size=2))) +
              tuple(sorted(rng.integers(0, cols + 1, size=2))) for _ in range(6)]
    # all columns (the row-range copy path), whole matrix, empty row range
    ranges += [(0, rows, 0, cols), (17, 700, 0, cols), (5, 5, 0, cols)]
    for r0, r1, c0, c1 in ranges:
        blk = _g().csr_block(a, int(r0), int(r1), int(c0), int(c1))
        want = a_ref.block(int(r0), int(r1), int(c0), int(c1))
        assert_csr_equal(blk, want.arrays())
        assert_csr_equal(_g().csr_transpose(blk), want.transpose().arrays())


def test_transpose_involution_and_empty(cuda):
    k, g = _k(), _g()
    e = k.DeviceCsr.from_host(3, 2, np.zeros(4, np.uint64), np.zeros(0, np.uint32),
                              np.zeros(0, np.float32))
    t = g.csr_transpose(e)
    assert (t.rows, t.cols, t.nnz) == (2, 3, 0)
    single = k.DeviceCsr.from_host(2, 3, np.array([0, 1, 1]), np.array([2]),
                                   np.array([5], np.float32))
    st = g.csr_transpose(single)
    rp, ci, v = st.to_host()
    assert rp.tolist() == [0, 0, 0, 1] and ci.tolist() == [0] and v.tolist() == [5.0]
