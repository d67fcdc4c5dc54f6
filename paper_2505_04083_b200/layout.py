"""Grid and layer-layout algebra (grid.hpp, layout.hpp, model.hpp:35-67,
engine.hpp:70-92, trainer.hpp:226-232) — pure host integer logic shared by
the Python driver, the perf model and the tests. The C++ engine carries the
same algebra (csrc/layout.h); tests pin both against the reference.
"""

from dataclasses import dataclass

import numpy as np

X, Y, Z = 0, 1, 2
AXIS_NAMES = "XYZ"


def chunk_start(total, parts, idx):
    """layout.hpp:16-21: ceil split, earlier chunks get the extra element."""
    base, rem = divmod(total, parts)
    return idx * base + min(idx, rem)


def chunk_size(total, parts, idx):
    return chunk_start(total, parts, idx + 1) - chunk_start(total, parts, idx)


def chunk_index(total, parts, pos):
    """graph.hpp:150-155"""
    base, rem = divmod(total, parts)
    if pos < rem * (base + 1):
        return pos // (base + 1)
    return rem + (pos - rem * (base + 1)) // max(base, 1)


def chunk_index_array(total, parts, pos):
    base, rem = divmod(total, parts)
    pos = np.asarray(pos, dtype=np.int64)
    lo = pos // (base + 1)
    hi = rem + (pos - rem * (base + 1)) // max(base, 1)
    return np.where(pos < rem * (base + 1), lo, hi)


@dataclass(frozen=True)
class GridConfig:
    """GridConfig (grid.hpp:39-102): x fastest-varying."""
    gx: int
    gy: int
    gz: int

    def __post_init__(self):
        if min(self.gx, self.gy, self.gz) < 1:
            raise ValueError("grid: all dimensions must be >= 1")

    @property
    def size(self):
        return self.gx * self.gy * self.gz

    def extent(self, axis):
        return (self.gx, self.gy, self.gz)[axis]

    def coords_of(self, rank):
        if not 0 <= rank < self.size:
            raise ValueError("grid: rank out of range")
        return (rank % self.gx, (rank // self.gx) % self.gy, rank // (self.gx * self.gy))

    def rank_of(self, c):
        return c[0] + self.gx * (c[1] + self.gy * c[2])

    def group_id(self, axis, c):
        x, y, z = c
        return (y + self.gy * z, x + self.gx * z, x + self.gx * y)[axis]

    def group_members(self, axis, gid):
        out = []
        for i in range(self.extent(axis)):
            if axis == X:
                c = (i, gid % self.gy, gid // self.gy)
            elif axis == Y:
                c = (gid % self.gx, i, gid // self.gx)
            else:
                c = (gid % self.gx, gid // self.gx, i)
            out.append(self.rank_of(c))
        return out

    def __str__(self):
        return f"{self.gx}x{self.gy}x{self.gz}"


def enumerate_configs(g):
    """grid.hpp:112-123: ordered factorizations, lexicographic (gx, gy, gz)."""
    out = []
    for gx in range(1, g + 1):
        if g % gx:
            continue
        rest = g // gx
        for gy in range(1, rest + 1):
            if rest % gy == 0:
                out.append((gx, gy, rest // gy))
    return out


@dataclass(frozen=True)
class LayerLayout:
    """LayerLayout (layout.hpp:28-43)."""
    layer: int
    inner: int
    col_shard: int
    row_shard: int

    @property
    def plane(self):
        return self.layer % 3

    @property
    def parity(self):
        return self.layer % 2


def plan_layouts(num_layers):
    """layout.hpp:53-66: (inner, col, row) rotates (X,Y,Z) -> (Z,X,Y) -> ..."""
    out = []
    inner, col, row = X, Y, Z
    for l in range(num_layers):
        out.append(LayerLayout(l, inner, col, row))
        inner, col, row = row, inner, col
    return out


def layer_shapes(grid, lay, c, n, d_in, d_out):
    """layout.hpp:82-101"""
    g_in, g_col, g_row = grid.extent(lay.inner), grid.extent(lay.col_shard), grid.extent(lay.row_shard)
    a_rows = chunk_size(n, g_row, c[lay.row_shard])
    a_cols = chunk_size(n, g_in, c[lay.inner])
    f_cols = chunk_size(d_in, g_col, c[lay.col_shard])
    w_rows = chunk_size(f_cols, g_row, c[lay.row_shard])
    w_cols = chunk_size(d_out, g_in, c[lay.inner])
    return dict(a_rows=a_rows, a_cols=a_cols, f_rows=a_cols, f_cols=f_cols, w_rows=w_rows,
                w_cols=w_cols, h_rows=a_rows, h_cols=f_cols, q_rows=a_rows, q_cols=w_cols)


def weight_slice(grid, lay, c, d_in, d_out):
    """model.hpp:35-51: rows by col_shard then row_shard, cols by inner."""
    g_col, g_row, g_in = grid.extent(lay.col_shard), grid.extent(lay.row_shard), grid.extent(lay.inner)
    outer0 = chunk_start(d_in, g_col, c[lay.col_shard])
    outer_len = chunk_size(d_in, g_col, c[lay.col_shard])
    r0 = outer0 + chunk_start(outer_len, g_row, c[lay.row_shard])
    r1 = outer0 + chunk_start(outer_len, g_row, c[lay.row_shard] + 1)
    return (r0, r1, chunk_start(d_out, g_in, c[lay.inner]), chunk_start(d_out, g_in, c[lay.inner] + 1))


def feature_slice(grid, c, n, d0):
    """model.hpp:53-67: rows by X then Z, cols by Y."""
    outer0 = chunk_start(n, grid.gx, c[0])
    outer_len = chunk_size(n, grid.gx, c[0])
    r0 = outer0 + chunk_start(outer_len, grid.gz, c[2])
    r1 = outer0 + chunk_start(outer_len, grid.gz, c[2] + 1)
    return (r0, r1, chunk_start(d0, grid.gy, c[1]), chunk_start(d0, grid.gy, c[1] + 1))


def adjacency_block_range(grid, plane, c, n):
    """engine.hpp:85-92"""
    lay = plan_layouts(plane + 1)[-1]
    g_row, g_in = grid.extent(lay.row_shard), grid.extent(lay.inner)
    cr, ci = c[lay.row_shard], c[lay.inner]
    return (chunk_start(n, g_row, cr), chunk_start(n, g_row, cr + 1), chunk_start(n, g_in, ci),
            chunk_start(n, g_in, ci + 1))


def needed_adjacency_keys(num_layers):
    """engine.hpp:70-78"""
    keys = []
    for l in range(num_layers):
        k = (l % 3, l % 2)
        if k not in keys:
            keys.append(k)
        if len(keys) == 6:
            break
    return keys


def label_row_range(grid, c, n, num_layers):
    """trainer.hpp:226-232"""
    last = plan_layouts(num_layers)[-1]
    g, pos = grid.extent(last.row_shard), c[last.row_shard]
    return chunk_start(n, g, pos), chunk_start(n, g, pos + 1)


def final_output_parity(num_layers):
    """graph.hpp:352-354"""
    return (num_layers - 1) % 2


ALL_GATHER, ALL_REDUCE, REDUCE_SCATTER = 0, 1, 2


def training_collective_volumes(grid, n, dims):
    """layout.hpp:123-157: (layer, forward, op, axis, elems) as seen by rank 0."""
    layers = len(dims) - 1
    out = []
    origin = (0, 0, 0)
    for l, lay in enumerate(plan_layouts(layers)):
        s = layer_shapes(grid, lay, origin, n, dims[l], dims[l + 1])
        f = s["f_rows"] * s["f_cols"]
        h = s["h_rows"] * s["h_cols"]
        q = s["q_rows"] * s["q_cols"]
        w = s["f_cols"] * s["w_cols"]
        if l == 0:
            out.append((l, True, ALL_GATHER, lay.row_shard, f))
        out += [(l, True, ALL_REDUCE, lay.inner, h), (l, True, ALL_GATHER, lay.row_shard, w),
                (l, True, ALL_REDUCE, lay.col_shard, q),
                (l, False, REDUCE_SCATTER, lay.row_shard, w),
                (l, False, ALL_GATHER, lay.row_shard, w), (l, False, ALL_REDUCE, lay.inner, h)]
        out.append((l, False, REDUCE_SCATTER if l == 0 else ALL_REDUCE, lay.row_shard, f))
    return out


def model_dims(d0, hidden, classes):
    """trainer.hpp:51-59"""
    return [d0, *hidden, classes]
