// Performance model that picks the 3D grid (perf_model.hpp:18-127,
// src/perf_model.cpp:33-229): SpMM cost features with the paper's shape
// penalties, a ring model of every collective the engine
// issues (layout.hpp:123-157) with per-axis effective bandwidth, an OLS fit
// of the three SpMM coefficients, and the ranking of all ordered
// factorizations of G. Host-only C++ (it runs once, before training); the
// B200 part is the calibration: bench.py feeds it measured NVLink bus
// bandwidth and SpMM timings.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <tuple>
#include <vector>

#include "layout.h"
#include "pk_common.cuh"

namespace pk {

namespace {

struct Stats {
  double n = 0, nnz = 0;
  std::vector<int64_t> dims;
};

Stats read_stats(const pk_dataset_stats* s) {
  check(s != nullptr, "perf model: null dataset stats");
  check(s->n >= 1, "perf model: node count must be positive");
  check(s->num_dims >= 2 && s->num_dims <= PK_MAX_LAYERS + 1,
        "perf model: need at least two layer dims");
  Stats out;
  out.n = static_cast<double>(s->n);
  out.nnz = static_cast<double>(s->nnz);
  for (int i = 0; i < s->num_dims; ++i) {
    check(s->dims[i] >= 1, "perf model: zero layer dimension");
    out.dims.push_back(s->dims[i]);
  }
  return out;
}

Grid read_grid(int gx, int gy, int gz) {
  check(gx >= 1 && gy >= 1 && gz >= 1, "perf model: grid dims must be >= 1");
  Grid g;
  g.g[0] = gx, g.g[1] = gy, g.g[2] = gz;
  return g;
}

// Per-layer SpMM features: sqrt(nnz * D) and that root times the forward and
// backward shape penalties (n / g_inner or n / g_row) * (g_col / D).
std::array<double, 3> features(const Stats& st, const Grid& g) {
  const int L = static_cast<int>(st.dims.size()) - 1;
  const auto lays = plan_layouts(L);
  std::array<double, 3> f{0, 0, 0};
  for (int l = 0; l < L; ++l) {
    const double d = static_cast<double>(st.dims[l]);
    const double root = std::sqrt(st.nnz * d);
    const double gi = g.extent(lays[l].inner), gc = g.extent(lays[l].col),
                 gr = g.extent(lays[l].row);
    f[0] += root;
    f[1] += root * ((st.n / gi) * (gc / d));
    f[2] += root * ((st.n / gr) * (gc / d));
  }
  return f;
}

double beta_of(int axis, const Grid& g, const pk_machine& m) {
  check(m.beta_intra > 0 && m.beta_inter > 0 && m.g_node >= 1,
        "perf model: invalid machine parameters");
  const int ext = g.extent(axis);
  if (ext == 1) return m.beta_intra;
  // ranks fill nodes Y first, then X, then Z
  double inner_ranks = 1;
  if (axis == kX) inner_ranks = g.extent(kY);
  if (axis == kZ) inner_ranks = static_cast<double>(g.extent(kX)) * g.extent(kY);
  if (inner_ranks * ext <= m.g_node) return m.beta_intra;
  return m.beta_inter / std::min<double>(m.g_node, inner_ranks);
}

double ring_seconds(int op, double bytes, int g, double beta) {
  check(g >= 1 && beta > 0, "ring_collective_seconds: invalid arguments");
  const double passes = op == PK_COLL_ALL_REDUCE ? 2.0 : 1.0;
  return passes * (static_cast<double>(g - 1) / g) * bytes / beta;
}

// layout.hpp:123-157 at the coordinate-0 rank
std::vector<pk_collective_volume> volumes(const Grid& g, int64_t n,
                                          const std::vector<int64_t>& dims) {
  check(dims.size() >= 2, "need at least input and output dims");
  const int L = static_cast<int>(dims.size()) - 1;
  const auto lays = plan_layouts(L);
  const Coords o;
  std::vector<pk_collective_volume> v;
  auto add = [&](int l, int fwd, int op, int axis, int64_t elems) {
    v.push_back(pk_collective_volume{l, fwd, op, axis, static_cast<uint64_t>(elems)});
  };
  for (int l = 0; l < L; ++l) {
    const Layout& y = lays[l];
    const Shapes s = layer_shapes(g, y, o, n, dims[l], dims[l + 1]);
    const int64_t fe = s.f_rows * s.f_cols, he = s.h_rows * s.h_cols,
                  qe = s.q_rows * s.q_cols, we = s.f_cols * s.w_cols;
    if (l == 0) add(l, 1, PK_COLL_ALL_GATHER, y.row, fe);
    add(l, 1, PK_COLL_ALL_REDUCE, y.inner, he);
    add(l, 1, PK_COLL_ALL_GATHER, y.row, we);
    add(l, 1, PK_COLL_ALL_REDUCE, y.col, qe);
    add(l, 0, PK_COLL_REDUCE_SCATTER, y.row, we);
    add(l, 0, PK_COLL_ALL_GATHER, y.row, we);
    add(l, 0, PK_COLL_ALL_REDUCE, y.inner, he);
    add(l, 0, l == 0 ? PK_COLL_REDUCE_SCATTER : PK_COLL_ALL_REDUCE, y.row, fe);
  }
  return v;
}

double comm_total(const Grid& g, const Stats& st, const pk_machine& m) {
  double t = 0;
  for (const auto& c : volumes(g, static_cast<int64_t>(st.n), st.dims))
    t += ring_seconds(c.op, static_cast<double>(c.elems) * m.bytes_per_scalar,
                      g.extent(c.axis), beta_of(c.axis, g, m));
  return t;
}

// Least squares y ~ X c for three features, X columns scaled to unit norm
// (the raw features span ~10 orders of magnitude), solved by Householder QR
// of the scaled design matrix. Rank deficiency is a contract error naming
// the cause, like the reference (perf_model.cpp:104-165).
pk_perf_coeffs ols3(const double* x3, const double* y, int count) {
  check(count >= 3, "fit_regression: need at least 3 samples, got " + std::to_string(count));
  const int m = count;
  std::vector<double> a(static_cast<size_t>(m) * 3), b(y, y + m);
  double scale[3];
  for (int j = 0; j < 3; ++j) {
    double s = 0;
    for (int i = 0; i < m; ++i) s += x3[i * 3 + j] * x3[i * 3 + j];
    scale[j] = std::sqrt(s);
    check(scale[j] > 0, "fit_regression: feature " + std::to_string(j + 1) +
                            " is identically zero; supply more diverse configurations");
    for (int i = 0; i < m; ++i) a[i * 3 + j] = x3[i * 3 + j] / scale[j];
  }
  double rdiag[3];
  for (int k = 0; k < 3; ++k) {
    double norm = 0;
    for (int i = k; i < m; ++i) norm += a[i * 3 + k] * a[i * 3 + k];
    norm = std::sqrt(norm);
    check(norm > 1e-10, "fit_regression: features are rank deficient; supply more diverse "
                        "configurations");
    const double alpha = a[k * 3 + k] > 0 ? -norm : norm;
    // v = x - alpha e1, stored in place
    a[k * 3 + k] -= alpha;
    double vnorm2 = 0;
    for (int i = k; i < m; ++i) vnorm2 += a[i * 3 + k] * a[i * 3 + k];
    auto reflect = [&](auto&& get) {
      double dot = 0;
      for (int i = k; i < m; ++i) dot += a[i * 3 + k] * get(i);
      return 2.0 * dot / vnorm2;
    };
    for (int j = k + 1; j < 3; ++j) {
      const double f = reflect([&](int i) { return a[i * 3 + j]; });
      for (int i = k; i < m; ++i) a[i * 3 + j] -= f * a[i * 3 + k];
    }
    const double fb = reflect([&](int i) { return b[i]; });
    for (int i = k; i < m; ++i) b[i] -= fb * a[i * 3 + k];
    rdiag[k] = alpha;
  }
  double c[3];
  for (int k = 2; k >= 0; --k) {
    double r = b[k];
    for (int j = k + 1; j < 3; ++j) r -= a[k * 3 + j] * c[j];
    c[k] = r / rdiag[k];
  }
  pk_perf_coeffs out{};
  out.c1 = c[0] / scale[0];
  out.c2 = c[1] / scale[1];
  out.c3 = c[2] / scale[2];
  double mean = 0;
  for (int i = 0; i < m; ++i) mean += y[i];
  mean /= m;
  double res = 0, tot = 0;
  for (int i = 0; i < m; ++i) {
    const double p = out.c1 * x3[i * 3] + out.c2 * x3[i * 3 + 1] + out.c3 * x3[i * 3 + 2];
    res += (y[i] - p) * (y[i] - p);
    tot += (y[i] - mean) * (y[i] - mean);
  }
  out.train_rmse = std::sqrt(res / m);
  out.train_r2 = tot > 0 ? 1.0 - res / tot : 1.0;
  return out;
}

}  // namespace

}  // namespace pk

using namespace pk;

extern "C" {

int pk_perf_default_coefficients(pk_perf_coeffs* out) {
  return guard([&] {
    check(out != nullptr, "perf model: null output");
    // perf_model.hpp:38-40 (the paper's Perlmutter fit)
    *out = pk_perf_coeffs{7.8e-4, 7.8e-10, -2.6e-10, 0, 0};
  });
}

int pk_perf_comp_features(const pk_dataset_stats* stats, int gx, int gy, int gz,
                          double* features3) {
  return guard([&] {
    const auto f = features(read_stats(stats), read_grid(gx, gy, gz));
    std::memcpy(features3, f.data(), sizeof(double) * 3);
  });
}

int pk_perf_predict_spmm(const double* f, const pk_perf_coeffs* c, double* seconds,
                         int* clamped) {
  return guard([&] {
    const double t = c->c1 * f[0] + c->c2 * f[1] + c->c3 * f[2];
    *seconds = t < 0 ? 0.0 : t;
    if (clamped) *clamped = t < 0;
  });
}

int pk_perf_effective_bandwidth(int axis, int gx, int gy, int gz, const pk_machine* m,
                                double* out) {
  return guard([&] {
    check(axis >= 0 && axis < 3, "perf model: bad axis");
    *out = beta_of(axis, read_grid(gx, gy, gz), *m);
  });
}

int pk_perf_ring_seconds(int op, double bytes, int g, double beta, double* out) {
  return guard([&] { *out = ring_seconds(op, bytes, g, beta); });
}

int pk_perf_predict_comm(const pk_dataset_stats* stats, int gx, int gy, int gz,
                         const pk_machine* m, double* total) {
  return guard([&] { *total = comm_total(read_grid(gx, gy, gz), read_stats(stats), *m); });
}

int pk_collective_volumes(int gx, int gy, int gz, const pk_dataset_stats* stats,
                          pk_collective_volume* out, int cap, int* count) {
  return guard([&] {
    const Stats st = read_stats(stats);
    const auto v = volumes(read_grid(gx, gy, gz), static_cast<int64_t>(st.n), st.dims);
    *count = static_cast<int>(v.size());
    check(out == nullptr || cap >= *count, "collective volumes: output too small");
    if (out) std::copy(v.begin(), v.end(), out);
  });
}

int pk_perf_fit_regression(const double* features3, const double* seconds, int count,
                           pk_perf_coeffs* out) {
  return guard([&] { *out = ols3(features3, seconds, count); });
}

int pk_enumerate_configs(int g, int* gxyz, int cap, int* count) {
  return guard([&] {
    check(g >= 1, "enumerate_configs: g must be >= 1");
    int k = 0;
    for (int x = 1; x <= g; ++x)
      for (int y = 1; x * y <= g; ++y)
        if (g % (x * y) == 0) {
          if (gxyz && k < cap) {
            gxyz[3 * k] = x, gxyz[3 * k + 1] = y, gxyz[3 * k + 2] = g / (x * y);
          }
          ++k;
        }
    *count = k;
    check(gxyz == nullptr || cap >= k, "enumerate_configs: output too small");
  });
}

int pk_perf_rank_configs(int g, const pk_dataset_stats* stats, const pk_machine* m,
                         const pk_perf_coeffs* c, pk_config_prediction* out, int cap,
                         int* count) {
  return guard([&] {
    const Stats st = read_stats(stats);
    int n = 0;
    check(pk_enumerate_configs(g, nullptr, 0, &n) == PK_OK, pk_last_error());
    std::vector<int> xyz(3 * n);
    check(pk_enumerate_configs(g, xyz.data(), n, &n) == PK_OK, pk_last_error());
    std::vector<pk_config_prediction> preds;
    for (int i = 0; i < n; ++i) {
      const Grid grid = read_grid(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
      pk_config_prediction p{};
      p.gx = grid.g[0], p.gy = grid.g[1], p.gz = grid.g[2];
      const auto f = features(st, grid);
      const double t = c->c1 * f[0] + c->c2 * f[1] + c->c3 * f[2];
      p.clamped = t < 0;
      p.spmm_seconds = t < 0 ? 0.0 : t;
      p.comm_seconds = comm_total(grid, st, *m);
      p.total_seconds = p.spmm_seconds + p.comm_seconds;
      preds.push_back(p);
    }
    std::stable_sort(preds.begin(), preds.end(), [](const auto& a, const auto& b) {
      if (a.total_seconds != b.total_seconds) return a.total_seconds < b.total_seconds;
      return std::tie(a.gz, a.gx, a.gy) < std::tie(b.gz, b.gx, b.gy);
    });
    *count = static_cast<int>(preds.size());
    check(cap >= *count, "rank_configs: output too small");
    std::copy(preds.begin(), preds.end(), out);
  });
}

}  // extern "C"
