"""Grid and layer-layout algebra (grid.hpp, layout.hpp, model.hpp:35-67,
engine.hpp:70-92, trainer.hpp:226-232) against the compiled reference on
every rank of every factorization of 1..8 ranks, plus the reference's own
known answers (test_grid.cpp). CPU only. The C++ engine carries the same
algebra (csrc/layout.h); its use is pinned by the GPU engine tests."""

import numpy as np
import pytest

from oracle import ref
from paper_2505_04083_b200 import layout as L

GRIDS = [g for G in range(1, 9) for g in L.enumerate_configs(G)]


def test_grid_known_answers():
    """test_grid.cpp:12-59, 85-135: x fastest, chunk algebra, rotation."""
    g = L.GridConfig(2, 3, 4)
    assert g.size == 24
    for r in range(24):
        c = g.coords_of(r)
        assert c == (r % 2, (r // 2) % 3, r // 6)
    assert [L.chunk_size(10, 4, i) for i in range(4)] == [3, 3, 2, 2]
    assert [L.chunk_start(10, 4, i) for i in range(5)] == [0, 3, 6, 8, 10]
    assert [L.chunk_size(2, 4, i) for i in range(4)] == [1, 1, 0, 0]   # zero-extent chunks
    lays = L.plan_layouts(4)
    assert [(x.inner, x.col_shard, x.row_shard) for x in lays] == [
        (L.X, L.Y, L.Z), (L.Z, L.X, L.Y), (L.Y, L.Z, L.X), (L.X, L.Y, L.Z)]
    assert len(L.enumerate_configs(8)) == 10 and len(L.enumerate_configs(4)) == 6
    assert L.enumerate_configs(4)[0] == (1, 1, 4)


@pytest.mark.parametrize("grid_t", GRIDS)
def test_layout_matches_reference_every_rank(grid_t):
    grid = L.GridConfig(*grid_t)
    n, dims = 37, [13, 7, 9, 5]
    layers = len(dims) - 1
    lays = L.plan_layouts(layers)
    for l, lay in enumerate(lays):
        assert ref.plan_layout(l) == (lay.inner, lay.col_shard, lay.row_shard)
    for r in range(grid.size):
        c = grid.coords_of(r)
        for l, lay in enumerate(lays):
            assert L.layer_shapes(grid, lay, c, n, dims[l], dims[l + 1]) == \
                ref.layer_shapes(grid_t, l, c, n, dims[l], dims[l + 1])
            assert tuple(L.weight_slice(grid, lay, c, dims[l], dims[l + 1])) == \
                ref.weight_slice(grid_t, l, c, dims[l], dims[l + 1])
        assert tuple(L.feature_slice(grid, c, n, dims[0])) == ref.feature_slice(grid_t, c, n,
                                                                              dims[0])
        for plane in range(3):
            assert tuple(L.adjacency_block_range(grid, plane, c, n)) == \
                ref.block_range(grid_t, plane, c, n)
        assert tuple(L.label_row_range(grid, c, n, layers)) == \
            ref.label_row_range(grid_t, c, n, layers)
    vols = L.training_collective_volumes(grid, n, dims)
    rv = ref.collective_volumes(grid_t, n, dims)
    assert [tuple(int(x) for x in v) for v in vols] == [tuple(int(x) for x in v) for v in rv]


@pytest.mark.parametrize("grid_t", [g for g in GRIDS if np.prod(g) in (4, 8)])
def test_slices_partition_the_tensors(grid_t):
    """Every W element and every F0 element is owned by exactly one rank
    (the reassembly of trainer.hpp:642-659 covers each once)."""
    grid = L.GridConfig(*grid_t)
    n, dims = 29, [11, 6, 5]
    lays = L.plan_layouts(2)
    f_cover = np.zeros((n, dims[0]), int)
    w_cover = [np.zeros((dims[l], dims[l + 1]), int) for l in range(2)]
    for r in range(grid.size):
        c = grid.coords_of(r)
        r0, r1, c0, c1 = L.feature_slice(grid, c, n, dims[0])
        f_cover[r0:r1, c0:c1] += 1
        for l in range(2):
            r0, r1, c0, c1 = L.weight_slice(grid, lays[l], c, dims[l], dims[l + 1])
            w_cover[l][r0:r1, c0:c1] += 1
    assert (f_cover == 1).all()
    # W shards are replicated across the axis that is neither row nor inner
    for l in range(2):
        assert (w_cover[l] == grid.size // (grid.extent(lays[l].col_shard) *
                                            grid.extent(lays[l].row_shard) *
                                            grid.extent(lays[l].inner))).all()
