"""Every grid of 2, 4 and 8 ranks on ONE B200: the in-process cluster
(paper_2505_04083_b200/cluster.py, csrc/local.cu) runs each rank of the grid
as a host thread with its own engine, the way the reference's Cluster runs
its ranks as threads (cluster.hpp:405-442). Checked against the reference's
own distributed pass / train_distributed at the same grid (oracle/_ref) —
the reassembly of test_engine.cpp:30-84 and the grids of
test_trainer.cpp:275-294 — plus the zero-extent shards of
test_engine.cpp:173-188 and the abort propagation of
test_collectives.cpp:190-199 (ClusterAborted).

The engine's multi-rank schedule (shards per plane, weight / feature slices,
which collective runs on which axis, the logits column gather, the
reduce-scatters of dW and dF0) is the same code the multi-GPU runs use; only
the transport differs (ordered device sums over events instead of NVLink
peer memory / NCCL), and it sums in the reference's coordinate order, so
PARITY logits are bit-identical on every grid.
"""

import numpy as np
import pytest

from oracle import ref

pytestmark = pytest.mark.gpu


def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def grids(g):
    out = []
    for gx in range(1, g + 1):
        if g % gx:
            continue
        for gy in range(1, g // gx + 1):
            if (g // gx) % gy == 0:
                out.append((gx, gy, g // gx // gy))
    return out


ALL = grids(2) + grids(4) + grids(8)


@pytest.fixture(scope="module")
def data(cuda):
    from paper_2505_04083_b200 import graph
    pre = graph.preprocess(graph.synth_rmat(11, 20000, 12, 5, seed=2), perm_seed=2)
    rpre = ref.synth_rmat(11, 20000, 12, 5, seed=2).preprocess(2)
    return pre, rpre


@pytest.mark.parametrize("grid", ALL, ids=lambda g: "x".join(map(str, g)))
def test_cluster_pass_matches_reference(data, grid):
    from paper_2505_04083_b200 import cluster, trainer
    from paper_2505_04083_b200.layout import GridConfig
    pre, rpre = data
    hidden = [16, 16]
    opts = trainer.TrainOptions(hidden_dims=hidden, mode=trainer.PK_MODE_PARITY,
                                hub_threshold=64)
    got = cluster.distributed_pass(pre, GridConfig(*grid), opts)
    want = rpre.distributed_pass(grid, hidden=hidden, seed=0)
    assert np.array_equal(got["logits"].view(np.uint32), want["logits"].view(np.uint32))
    assert len(set(got["rank_losses"])) == 1  # every rank reports the same loss
    assert abs(got["loss"] - want["loss"]) <= 1e-6 * abs(want["loss"])
    for a, b in zip(got["dw"], want["dw"]):
        assert nrel(a, b) <= 1e-5
    assert nrel(got["df0"], want["df0"]) <= 1e-5


@pytest.mark.parametrize("grid", [(2, 1, 1), (1, 2, 2), (2, 2, 2), (8, 1, 1), (1, 1, 8)],
                         ids=lambda g: "x".join(map(str, g)))
def test_cluster_train_distributed_tracks_reference(data, grid):
    """train_distributed: loss curve, final W and F0 vs the reference's
    train_distributed at the same grid (test_trainer.cpp:256-294)."""
    from paper_2505_04083_b200 import cluster, trainer
    from paper_2505_04083_b200.layout import GridConfig
    pre, rpre = data
    opts = trainer.TrainOptions(hidden_dims=[16, 16], mode=trainer.PK_MODE_PARITY, epochs=4,
                                hub_threshold=64)
    res = cluster.train_distributed(pre, GridConfig(*grid), opts)
    want = rpre.train_distributed(grid, hidden=(16, 16), seed=0, epochs=4, params=True)
    got = np.array([m["loss"] for m in res.global_metrics])
    assert np.max(np.abs(got - want["loss"]) / want["loss"]) <= 1e-5, (got, want["loss"])
    for a, b in zip(res.weights, want["weights"]):
        assert nrel(a, b) <= 1e-4
    assert nrel(res.features, want["features"]) <= 1e-4
    # FLOP counters summed over ranks equal the reference's (acceptance crit. 4)
    assert res.global_metrics[0]["spmm_flops"] == int(want["flops"][0][0])
    assert res.global_metrics[0]["gemm_flops"] == int(want["flops"][0][1])


@pytest.mark.parametrize("grid", [(2, 2, 2), (4, 1, 2)], ids=lambda g: "x".join(map(str, g)))
def test_cluster_fast_mode(data, grid):
    """FAST mode (tcgen05 3xTF32 GEMMs, segmented SpMM plans) on 8 ranks."""
    from paper_2505_04083_b200 import cluster, trainer
    from paper_2505_04083_b200.layout import GridConfig
    pre, rpre = data
    opts = trainer.TrainOptions(hidden_dims=[16, 16], mode=trainer.PK_MODE_FAST,
                                hub_threshold=64)
    got = cluster.distributed_pass(pre, GridConfig(*grid), opts)
    want = rpre.distributed_pass(grid, hidden=[16, 16], seed=0)
    assert abs(got["loss"] - want["loss"]) <= 1e-5 * abs(want["loss"])
    assert nrel(got["logits"], want["logits"]) <= 1e-4
    for a, b in zip(got["dw"], want["dw"]):
        assert nrel(a, b) <= 1e-4
    assert nrel(got["df0"], want["df0"]) <= 1e-4


@pytest.mark.parametrize("grid", grids(4), ids=lambda g: "x".join(map(str, g)))
def test_cluster_zero_extent_shards(cuda, grid):
    """test_engine.cpp:173-188: N=13, dims 5-7-3 on every grid of 4 — some
    ranks hold 0-row / 0-column blocks (e.g. W 7x0, a 13x0 logits chunk) and
    still enter every collective."""
    import torch

    from paper_2505_04083_b200 import cluster, graph, trainer
    from paper_2505_04083_b200.layout import GridConfig
    rng = np.random.default_rng(5)
    n = 13
    edges = np.array([(u, v) for u in range(n) for v in range(n) if u != v and rng.random() < .3],
                     np.uint32)
    feats = rng.random((n, 5)).astype(np.float32)
    labels = rng.integers(0, 3, n).astype(np.uint32)
    g = ref.graph_from_arrays(n, edges, feats, labels, 3, np.ones(n, np.uint8))
    rpre = g.preprocess(7)
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    pre = graph.preprocess(graph.GraphDataset(n, dev(edges.view(np.int32)), dev(feats),
                                              dev(labels.view(np.int32)), 3,
                                              dev(np.ones(n, np.uint8)), True), 7)
    opts = trainer.TrainOptions(hidden_dims=[7], mode=trainer.PK_MODE_PARITY)
    got = cluster.distributed_pass(pre, GridConfig(*grid), opts)
    want = rpre.distributed_pass(grid, hidden=[7], seed=0)
    assert np.array_equal(got["logits"].view(np.uint32), want["logits"].view(np.uint32))
    for a, b in zip(got["dw"], want["dw"]):
        assert nrel(a, b) <= 1e-5
    assert nrel(got["df0"], want["df0"]) <= 1e-5


def test_cluster_abort_propagates(data):
    """A rank that fails takes the cluster down: the failure is re-raised,
    every other rank ends with ClusterAborted naming it instead of waiting
    forever in a collective (cluster.hpp:67-71, 240, 434;
    test_collectives.cpp:190-199)."""
    from paper_2505_04083_b200 import _capi, cluster, trainer
    from paper_2505_04083_b200.layout import GridConfig
    pre, _ = data
    grid = GridConfig(2, 2, 1)
    cl = cluster.Cluster(grid)
    opts = trainer.TrainOptions(hidden_dims=[16, 16], mode=trainer.PK_MODE_PARITY)
    seen = {}

    def body(r):
        e = cl.engine(pre.n, pre.feat_dim, pre.num_classes, r, opts)
        try:
            e.load(pre)
            e.train_epoch(0)
            if r == 2:
                raise ValueError("rank 2 injected failure")
            try:
                for ep in range(1, 4):
                    e.train_epoch(ep)
            except _capi.ClusterAborted as exc:
                seen[r] = str(exc)
                raise
        finally:
            e.close()
    with pytest.raises(ValueError, match="injected"):
        cl.run(body)
    assert cl.aborted()
    assert sorted(seen) == [0, 1, 3]
    assert all("rank 2" in m for m in seen.values())
    cl.close()


@pytest.mark.parametrize("grid", [(2, 1, 1), (2, 2, 2), (1, 4, 2)],
                         ids=lambda g: "x".join(map(str, g)))
def test_cluster_comm_stats_match_reference(data, grid):
    """CommStats (cluster.hpp:35-65) of one pass on every rank — calls and
    ring-model bytes per axis and collective — equal the reference's, with
    the blocked aggregation's block count fixed on both sides
    (engine.hpp:135-138)."""
    from paper_2505_04083_b200 import cluster, trainer
    from paper_2505_04083_b200.layout import GridConfig
    pre, rpre = data
    opts = trainer.TrainOptions(hidden_dims=[16, 16], mode=trainer.PK_MODE_PARITY,
                                hub_threshold=64, block_count=2)
    got = cluster.distributed_pass(pre, GridConfig(*grid), opts)
    want = rpre.distributed_pass(grid, hidden=[16, 16], seed=0, block_count=2)
    assert np.array_equal(got["comm_calls"], want["comm_calls"].astype(np.uint64))
    assert np.allclose(got["comm_bytes"], want["comm_bytes"], rtol=0, atol=0.5)
