"""Per-rank shard generation (paper_2505_04083_b200/rank_gen.py,
csrc/rank_gen.cu) against the reference's whole-graph pipeline:
synth_rmat -> preprocess -> block / slice_rank_tensors (graph.hpp:40-148,
291-384; engine.hpp:96-113; trainer.hpp:234-250), for every rank of several
grids, undirected (synth_rmat's default) and directed (the papers-shaped
C4 orientation, SURVEY 8e'): adjacency blocks, F0 slices and labels must be
byte-identical. Then a directed graph trains from generated shards on an
in-process 2x2x2 cluster and tracks the reference's train_distributed."""

import numpy as np
import pytest

from oracle import ref

pytestmark = pytest.mark.gpu

SCALE, EDGES, FEAT, CLASSES, SEED = 10, 9000, 12, 5, 4
GRIDS = [(1, 1, 1), (2, 2, 2), (2, 1, 2), (1, 4, 2), (4, 1, 1), (1, 2, 3)]


def nrel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (den if den > 0 else 1.0))


def reference(undirected):
    g = ref.synth_rmat(SCALE, EDGES, FEAT, CLASSES, seed=SEED)
    if not undirected:
        g.set_undirected(False)
    return g.preprocess(SEED)


@pytest.mark.parametrize("undirected", [True, False], ids=["undirected", "directed"])
def test_generated_rank_tensors_bit_exact(cuda, undirected):
    from paper_2505_04083_b200 import rank_gen
    from paper_2505_04083_b200.layout import (GridConfig, adjacency_block_range, feature_slice,
                                              final_output_parity, label_row_range,
                                              needed_adjacency_keys)
    rpre = reference(undirected)
    arr = rpre.arrays()
    spec = rank_gen.RmatSpec(SCALE, EDGES, FEAT, CLASSES, seed=SEED, undirected=undirected)
    n = spec.n
    pieces = rank_gen.global_pieces(spec)
    variants = {0: rpre.csr(0), 1: rpre.csr(1)}
    for L in (3, 4):
        for gt in GRIDS:
            grid = GridConfig(*gt)
            for r in range(grid.size):
                c = grid.coords_of(r)
                rt = rank_gen.generate_rank_tensors(spec, grid, r, L, pieces)
                for plane, parity in needed_adjacency_keys(L):
                    r0, r1, c0, c1 = adjacency_block_range(grid, plane, c, n)
                    want = variants[parity].block(r0, r1, c0, c1).arrays()
                    got = rt.adj[(plane, parity)][0].to_host()
                    for g, w in zip(got, want):
                        assert np.array_equal(np.asarray(g).view(np.uint8),
                                              np.asarray(w).view(np.uint8)), (gt, r, plane, parity)
                fr0, fr1, fc0, fc1 = feature_slice(grid, c, n, FEAT)
                assert np.array_equal(rt.f0.cpu().numpy().view(np.uint32),
                                      arr["features"][fr0:fr1, fc0:fc1].view(np.uint32))
                lr0, lr1 = label_row_range(grid, c, n, L)
                key = "labels_row" if final_output_parity(L) == 0 else "labels_col"
                assert np.array_equal(rt.labels.cpu().numpy().view(np.uint32),
                                      arr[key][lr0:lr1])
                assert np.all(rt.mask.cpu().numpy() == 1)


def test_degrees_by_range_equal_whole(cuda):
    """All-gathering per-range degree counts gives the whole vector (the
    multi-rank path): 1 range vs 7 uneven ranges."""
    from paper_2505_04083_b200 import rank_gen
    spec = rank_gen.RmatSpec(SCALE, EDGES, FEAT, CLASSES, seed=SEED, undirected=False)
    for kind in (0, 1):
        whole = rank_gen.global_degrees(spec, kind, 0, 1)
        split = rank_gen.global_degrees(spec, kind, 0, 7)
        assert np.array_equal(whole.cpu().numpy(), split.cpu().numpy())


def test_directed_training_from_generated_shards(cuda):
    """C4's orientation end to end at small scale: 8 in-process ranks load
    their generated shards and train; the loss curve, W and F0 follow the
    reference's train_distributed on the directed dataset."""
    from paper_2505_04083_b200 import cluster, rank_gen, trainer
    from paper_2505_04083_b200.layout import GridConfig
    spec = rank_gen.RmatSpec(SCALE, EDGES, FEAT, CLASSES, seed=SEED, undirected=False)
    opts = trainer.TrainOptions(hidden_dims=[16, 16], mode=trainer.PK_MODE_PARITY, epochs=4,
                                hub_threshold=64)
    res = cluster.train_distributed_generated(spec, GridConfig(2, 2, 2), opts)
    want = reference(False).train_distributed((2, 2, 2), hidden=(16, 16), seed=0, epochs=4,
                                              params=True)
    got = np.array([m["loss"] for m in res.global_metrics])
    assert np.max(np.abs(got - want["loss"]) / want["loss"]) <= 1e-5, (got, want["loss"])
    for a, b in zip(res.weights, want["weights"]):
        assert nrel(a, b) <= 1e-4
    assert nrel(res.features, want["features"]) <= 1e-4
