// Grid / layer-layout algebra of the 3D decomposition (grid.hpp,
// layout.hpp, model.hpp:35-67, engine.hpp:70-92, trainer.hpp:226-232),
// restated for the C++ engine. Pure integer logic, host only.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <utility>
#include <vector>

namespace pk {

enum Axis : int { kX = 0, kY = 1, kZ = 2 };

struct Coords {
  int c[3] = {0, 0, 0};
  int along(int axis) const { return c[axis]; }
};

inline int64_t chunk_start(int64_t total, int parts, int idx) {
  const int64_t base = total / parts, rem = total % parts;
  return static_cast<int64_t>(idx) * base + std::min<int64_t>(idx, rem);
}
inline int64_t chunk_size(int64_t total, int parts, int idx) {
  return chunk_start(total, parts, idx + 1) - chunk_start(total, parts, idx);
}

struct Grid {
  int g[3] = {1, 1, 1};
  int size() const { return g[0] * g[1] * g[2]; }
  int extent(int axis) const { return g[axis]; }
  Coords coords_of(int rank) const {
    Coords c;
    c.c[0] = rank % g[0];
    c.c[1] = (rank / g[0]) % g[1];
    c.c[2] = rank / (g[0] * g[1]);
    return c;
  }
  int rank_of(const Coords& c) const { return c.c[0] + g[0] * (c.c[1] + g[1] * c.c[2]); }
  // grid.hpp:67-73: ranks sharing the other two coordinates
  int group_id(int axis, const Coords& c) const {
    switch (axis) {
      case kX: return c.c[1] + g[1] * c.c[2];
      case kY: return c.c[0] + g[0] * c.c[2];
      default: return c.c[0] + g[0] * c.c[1];
    }
  }
};

struct Layout {
  int layer = 0, inner = kX, col = kY, row = kZ;
  int plane() const { return layer % 3; }
  int parity() const { return layer % 2; }
};

// layout.hpp:53-66
inline std::vector<Layout> plan_layouts(int layers) {
  std::vector<Layout> out;
  Layout cur;
  for (int l = 0; l < layers; ++l) {
    cur.layer = l;
    out.push_back(cur);
    cur = Layout{l + 1, cur.row, cur.inner, cur.col};
  }
  return out;
}

struct Shapes {
  int64_t a_rows, a_cols, f_rows, f_cols, w_rows, w_cols, h_rows, h_cols, q_rows, q_cols;
};

// layout.hpp:82-101
inline Shapes layer_shapes(const Grid& g, const Layout& l, const Coords& c, int64_t n,
                           int64_t d_in, int64_t d_out) {
  Shapes s;
  s.a_rows = chunk_size(n, g.extent(l.row), c.along(l.row));
  s.a_cols = chunk_size(n, g.extent(l.inner), c.along(l.inner));
  s.f_rows = s.a_cols;
  s.f_cols = chunk_size(d_in, g.extent(l.col), c.along(l.col));
  s.w_rows = chunk_size(s.f_cols, g.extent(l.row), c.along(l.row));
  s.w_cols = chunk_size(d_out, g.extent(l.inner), c.along(l.inner));
  s.h_rows = s.a_rows;
  s.h_cols = s.f_cols;
  s.q_rows = s.a_rows;
  s.q_cols = s.w_cols;
  return s;
}

struct Slice {
  int64_t r0, r1, c0, c1;
};

// model.hpp:35-51
inline Slice weight_slice(const Grid& g, const Layout& l, const Coords& c, int64_t d_in,
                          int64_t d_out) {
  const int gc = g.extent(l.col), gr = g.extent(l.row), gi = g.extent(l.inner);
  const int64_t outer0 = chunk_start(d_in, gc, c.along(l.col));
  const int64_t outer_len = chunk_size(d_in, gc, c.along(l.col));
  return {outer0 + chunk_start(outer_len, gr, c.along(l.row)),
          outer0 + chunk_start(outer_len, gr, c.along(l.row) + 1),
          chunk_start(d_out, gi, c.along(l.inner)), chunk_start(d_out, gi, c.along(l.inner) + 1)};
}

// model.hpp:53-67
inline Slice feature_slice(const Grid& g, const Coords& c, int64_t n, int64_t d0) {
  const int64_t outer0 = chunk_start(n, g.g[0], c.c[0]);
  const int64_t outer_len = chunk_size(n, g.g[0], c.c[0]);
  return {outer0 + chunk_start(outer_len, g.g[2], c.c[2]),
          outer0 + chunk_start(outer_len, g.g[2], c.c[2] + 1), chunk_start(d0, g.g[1], c.c[1]),
          chunk_start(d0, g.g[1], c.c[1] + 1)};
}

// engine.hpp:85-92
inline Slice adjacency_block_range(const Grid& g, int plane, const Coords& c, int64_t n) {
  const Layout l = plan_layouts(plane + 1).back();
  const int gr = g.extent(l.row), gi = g.extent(l.inner);
  return {chunk_start(n, gr, c.along(l.row)), chunk_start(n, gr, c.along(l.row) + 1),
          chunk_start(n, gi, c.along(l.inner)), chunk_start(n, gi, c.along(l.inner) + 1)};
}

// engine.hpp:70-78
inline std::vector<std::pair<int, int>> needed_adjacency_keys(int layers) {
  std::vector<std::pair<int, int>> keys;
  for (int l = 0; l < layers && keys.size() < 6; ++l) {
    std::pair<int, int> k{l % 3, l % 2};
    if (std::find(keys.begin(), keys.end(), k) == keys.end()) keys.push_back(k);
  }
  return keys;
}

// trainer.hpp:226-232
inline std::pair<int64_t, int64_t> label_row_range(const Grid& g, const Coords& c, int64_t n,
                                                   int layers) {
  const Layout last = plan_layouts(layers).back();
  const int gr = g.extent(last.row), pos = c.along(last.row);
  return {chunk_start(n, gr, pos), chunk_start(n, gr, pos + 1)};
}

// engine.hpp:135-138
inline int resolve_block_count(int requested, int64_t rows) {
  if (requested > 0) return requested;
  return static_cast<int>(std::max<int64_t>(1, (rows + 16383) / 16384));
}

}  // namespace pk
