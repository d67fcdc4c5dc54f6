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


# the reference's own SBM / Erdős cases (test_graph.cpp:92, 189-231,
# test_engine.cpp:16, test_trainer.cpp:15-17, 185, 229) plus a partial mask
@pytest.mark.parametrize("kind,args,feat,classes,seed,frac", [
    ("sbm", (4096, 8, 0.2, 0.001), 8, 4, 31, 1.0),
    ("sbm", (128, 4, 0.2, 0.02), 16, 8, 23, 1.0),
    ("sbm", (48, 4, 0.3, 0.02), 6, 3, 3, 0.7),
    ("sbm", (1000, 2, 0.4, 0.1), 5, 3, 9, 1.0),
    ("sbm", (300, 300, 0.9, 0.0), 2, 2, 4, 1.0),   # every node its own community
    ("erdos", (50, 0.1), 4, 3, 21, 1.0),
    ("erdos", (1000, 0.01), 4, 2, 7, 1.0),
    ("erdos", (8, 0.4), 4, 3, 13, 1.0),
    ("erdos", (1, 0.5), 2, 1, 1, 1.0),              # no pairs at all
])
def test_synth_sbm_erdos_bitwise(cuda, kind, args, feat, classes, seed, frac):
    g = _g()
    if kind == "sbm":
        ds = g.synth_sbm(*args, feat, classes, seed, train_fraction=frac)
        want = ref.synth_sbm(*args, feat, classes, seed, train_fraction=frac).arrays()
    else:
        ds = g.synth_erdos(*args, feat, classes, seed, train_fraction=frac)
        want = ref.synth_erdos(*args, feat, classes, seed, train_fraction=frac).arrays()
    assert np.array_equal(ds.edges.cpu().numpy().view(np.uint32).reshape(-1, 2),
                          want["edges"].reshape(-1, 2))
    assert np.array_equal(ds.features.cpu().numpy(), want["features"])
    assert np.array_equal(ds.labels.cpu().numpy().view(np.uint32), want["labels"])
    assert np.array_equal(ds.train_mask.cpu().numpy(), want["mask"])


def test_synth_sbm_erdos_contract_errors(cuda):
    """test_graph.cpp:230-231"""
    g = _g()
    from paper_2505_04083_b200._capi import ContractError
    with pytest.raises(ContractError):
        g.synth_erdos(0, 0.5, 2, 2, 1)
    with pytest.raises(ContractError):
        g.synth_sbm(10, 0, 0.5, 0.1, 2, 2, 1)
    with pytest.raises(ContractError):
        g.synth_sbm(10, 2, 1.5, 0.1, 2, 2, 1)


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
