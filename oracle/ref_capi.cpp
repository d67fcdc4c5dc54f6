// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Thin extern "C" shim over the UNMODIFIED reference headers in
// /root/reference/proj/include (plexuskit). It is compiled by oracle/Makefile
// with the reference's own flags (-O2 -g -DNDEBUG -std=gnu++20, no -march, so
// the reference kernels are scalar mulss+addss with no FMA) into
// oracle/_ref/libplexus_ref.so. tests/, bench.py's reference arm and
// tests/golden/make_golden.py load it through ctypes (oracle/ref.py).
//
// Nothing here re-implements reference logic: every function marshals plain
// arrays into the reference's types and calls the reference entry point named
// in its comment.

#include <algorithm>
#include <cstring>
#include <memory>
#include <thread>
#include <string>
#include <vector>

#include "plexuskit/perf_model.hpp"
#include "plexuskit/trainer.hpp"

using namespace plexuskit;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ContractError& e) {
    g_err = std::string("ContractError: ") + e.what();
    return 1;
  } catch (const TrainingError& e) {
    g_err = std::string("TrainingError: ") + e.what();
    return 5;
  } catch (const MemoryError& e) {
    g_err = std::string("MemoryError: ") + e.what();
    return 4;
  } catch (const IoError& e) {  // 10 + IoErrorCode (common.hpp:28-35)
    g_err = std::string("IoError: ") + e.what();
    return 10 + static_cast<int>(e.code());
  } catch (const std::exception& e) {
    g_err = std::string("Error: ") + e.what();
    return 9;
  }
}

template <typename T>
DenseMatrix<T> dense_in(const void* p, std::size_t r, std::size_t c) {
  const T* t = static_cast<const T*>(p);
  return DenseMatrix<T>(r, c, std::vector<T>(t, t + r * c));
}

template <typename T>
void dense_out(const DenseMatrix<T>& m, void* p) {
  if (m.size()) std::memcpy(p, m.data(), m.size() * sizeof(T));
}

template <typename T>
CsrMatrix<T> csr_in(std::size_t rows, std::size_t cols, const u64* rp,
                    const u32* ci, const void* v) {
  const u64 nnz = rp[rows];
  const T* tv = static_cast<const T*>(v);
  return CsrMatrix<T>(rows, cols, std::vector<u64>(rp, rp + rows + 1),
                      std::vector<u32>(ci, ci + nnz),
                      std::vector<T>(tv, tv + nnz));
}

// Opaque holders. `f64` selects the scalar type.
struct Graph {
  int f64 = 0;
  GraphDataset<float> f;
  GraphDataset<double> d;
};
struct Pre {
  int f64 = 0;
  PreprocessedDataset<float> f;
  PreprocessedDataset<double> d;
};
struct Csr {
  int f64 = 0;
  CsrMatrix<float> f;
  CsrMatrix<double> d;
};

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// ---------------------------------------------------------------------------
// synthetic datasets: synth_rmat / synth_sbm (graph.hpp:253-322)

void* ref_synth_rmat(int scale, u64 edges, double a, double b, double c,
                     u64 feat, u32 classes, u64 seed, double train_fraction,
                     int f64) {
  auto* g = new Graph;
  g->f64 = f64;
  int rc = guarded([&] {
    RmatParams p;
    p.scale = scale;
    p.edges = edges;
    p.a = a;
    p.b = b;
    p.c = c;
    if (f64)
      g->d = synth_rmat<double>(p, feat, classes, seed, train_fraction);
    else
      g->f = synth_rmat<float>(p, feat, classes, seed, train_fraction);
  });
  if (rc) {
    delete g;
    return nullptr;
  }
  return g;
}

void* ref_synth_sbm(u64 n, int communities, double p_in, double p_out, u64 feat,
                    u32 classes, u64 seed, double train_fraction, int f64) {
  auto* g = new Graph;
  g->f64 = f64;
  int rc = guarded([&] {
    SbmParams p;
    p.n = n;
    p.communities = communities;
    p.p_in = p_in;
    p.p_out = p_out;
    if (f64)
      g->d = synth_sbm<double>(p, feat, classes, seed, train_fraction);
    else
      g->f = synth_sbm<float>(p, feat, classes, seed, train_fraction);
  });
  if (rc) {
    delete g;
    return nullptr;
  }
  return g;
}

void* ref_synth_erdos(u64 n, double prob, u64 feat, u32 classes, u64 seed,
                      double train_fraction, int f64) {
  auto* g = new Graph;
  g->f64 = f64;
  int rc = guarded([&] {
    ErdosParams p;
    p.n = n;
    p.p = prob;
    if (f64)
      g->d = synth_erdos<double>(p, feat, classes, seed, train_fraction);
    else
      g->f = synth_erdos<float>(p, feat, classes, seed, train_fraction);
  });
  if (rc) {
    delete g;
    return nullptr;
  }
  return g;
}

// Builds a dataset from caller arrays (edges as u,v pairs).
void* ref_graph_from_arrays(u64 n, u64 num_edges, const u32* uv, int undirected,
                            const void* features, u64 feat, const u32* labels,
                            u32 classes, const u8* mask, int f64) {
  auto* g = new Graph;
  g->f64 = f64;
  auto fill = [&](auto& ds, auto tag) {
    using T = decltype(tag);
    ds.num_nodes = n;
    ds.edges.resize(num_edges);
    for (u64 e = 0; e < num_edges; ++e) ds.edges[e] = {uv[2 * e], uv[2 * e + 1]};
    ds.undirected = undirected != 0;
    ds.features = dense_in<T>(features, n, feat);
    ds.labels.assign(labels, labels + n);
    ds.num_classes = classes;
    ds.train_mask.assign(mask, mask + n);
  };
  if (f64)
    fill(g->d, double{});
  else
    fill(g->f, float{});
  return g;
}

void ref_graph_set_undirected(void* h, int undirected) {
  auto* g = static_cast<Graph*>(h);
  g->f.undirected = g->d.undirected = undirected != 0;
}

void ref_graph_info(void* h, u64* n, u64* num_edges, u64* feat, u32* classes) {
  auto* g = static_cast<Graph*>(h);
  auto info = [&](auto& ds) {
    *n = ds.num_nodes;
    *num_edges = ds.edges.size();
    *feat = ds.features.cols();
    *classes = ds.num_classes;
  };
  if (g->f64)
    info(g->d);
  else
    info(g->f);
}

void ref_graph_copy(void* h, u32* uv, void* features, u32* labels, u8* mask) {
  auto* g = static_cast<Graph*>(h);
  auto copy = [&](auto& ds) {
    for (std::size_t e = 0; e < ds.edges.size(); ++e) {
      uv[2 * e] = ds.edges[e].first;
      uv[2 * e + 1] = ds.edges[e].second;
    }
    if (features) dense_out(ds.features, features);
    if (labels) std::memcpy(labels, ds.labels.data(), ds.labels.size() * 4);
    if (mask) std::memcpy(mask, ds.train_mask.data(), ds.train_mask.size());
  };
  if (g->f64)
    copy(g->d);
  else
    copy(g->f);
}

void ref_graph_free(void* h) { delete static_cast<Graph*>(h); }

// ---------------------------------------------------------------------------
// CSR holders: normalize_adjacency (graph.hpp:44-76), transpose / block
// (csr.hpp:78-120), permute_csr (graph.hpp:101-131)

void* ref_normalize(void* gh) {
  auto* g = static_cast<Graph*>(gh);
  auto* c = new Csr;
  c->f64 = g->f64;
  int rc = guarded([&] {
    if (g->f64)
      c->d = normalize_adjacency(g->d);
    else
      c->f = normalize_adjacency(g->f);
  });
  if (rc) {
    delete c;
    return nullptr;
  }
  return c;
}

void* ref_csr_from_arrays(u64 rows, u64 cols, const u64* rp, const u32* ci,
                          const void* vals, int f64) {
  auto* c = new Csr;
  c->f64 = f64;
  int rc = guarded([&] {
    if (f64)
      c->d = csr_in<double>(rows, cols, rp, ci, vals);
    else
      c->f = csr_in<float>(rows, cols, rp, ci, vals);
  });
  if (rc) {
    delete c;
    return nullptr;
  }
  return c;
}

void ref_csr_info(void* h, u64* rows, u64* cols, u64* nnz) {
  auto* c = static_cast<Csr*>(h);
  if (c->f64) {
    *rows = c->d.rows(), *cols = c->d.cols(), *nnz = c->d.nnz();
  } else {
    *rows = c->f.rows(), *cols = c->f.cols(), *nnz = c->f.nnz();
  }
}

void ref_csr_copy(void* h, u64* rp, u32* ci, void* vals) {
  auto* c = static_cast<Csr*>(h);
  auto copy = [&](auto& m) {
    std::memcpy(rp, m.row_ptr().data(), m.row_ptr().size() * 8);
    if (m.nnz()) {
      std::memcpy(ci, m.col_idx().data(), m.nnz() * 4);
      std::memcpy(vals, m.values().data(), m.nnz() * sizeof(m.values()[0]));
    }
  };
  if (c->f64)
    copy(c->d);
  else
    copy(c->f);
}

void* ref_csr_transpose(void* h) {
  auto* c = static_cast<Csr*>(h);
  auto* o = new Csr;
  o->f64 = c->f64;
  if (c->f64)
    o->d = c->d.transpose();
  else
    o->f = c->f.transpose();
  return o;
}

void* ref_csr_block(void* h, u64 r0, u64 r1, u64 c0, u64 c1) {
  auto* c = static_cast<Csr*>(h);
  auto* o = new Csr;
  o->f64 = c->f64;
  int rc = guarded([&] {
    if (c->f64)
      o->d = c->d.block(r0, r1, c0, c1);
    else
      o->f = c->f.block(r0, r1, c0, c1);
  });
  if (rc) {
    delete o;
    return nullptr;
  }
  return o;
}

void* ref_permute_csr(void* h, const u32* row_perm, const u32* col_perm) {
  auto* c = static_cast<Csr*>(h);
  auto* o = new Csr;
  o->f64 = c->f64;
  const u64 n = c->f64 ? c->d.rows() : c->f.rows();
  std::vector<u32> rp(row_perm, row_perm + n), cp(col_perm, col_perm + n);
  int rc = guarded([&] {
    if (c->f64)
      o->d = permute_csr(c->d, rp, cp);
    else
      o->f = permute_csr(c->f, rp, cp);
  });
  if (rc) {
    delete o;
    return nullptr;
  }
  return o;
}

double ref_balance_metric(void* h, int p, int q) {
  auto* c = static_cast<Csr*>(h);
  double out = -1;
  guarded([&] { out = c->f64 ? balance_metric(c->d, p, q) : balance_metric(c->f, p, q); });
  return out;
}

void ref_csr_free(void* h) { delete static_cast<Csr*>(h); }

// generate_permutation_pair (graph.hpp:84-93)
void ref_permutation_pair(u64 n, u64 seed, u32* row_perm, u32* col_perm) {
  auto p = generate_permutation_pair(n, seed);
  std::memcpy(row_perm, p.row_perm.data(), n * 4);
  std::memcpy(col_perm, p.col_perm.data(), n * 4);
}

// Philox stream dump (rng.hpp:17-104): `count` u64 draws.
void ref_philox_u64(u64 seed, u64 stream, u64 count, u64* out) {
  Philox r(seed, stream);
  for (u64 i = 0; i < count; ++i) out[i] = r.next_u64();
}

void ref_philox_double(u64 seed, u64 stream, u64 count, double* out) {
  Philox r(seed, stream);
  for (u64 i = 0; i < count; ++i) out[i] = r.next_double();
}

// ---------------------------------------------------------------------------
// preprocess (graph.hpp:356-384)

void* ref_preprocess(void* gh, u64 perm_seed) {
  auto* g = static_cast<Graph*>(gh);
  auto* p = new Pre;
  p->f64 = g->f64;
  int rc = guarded([&] {
    if (g->f64)
      p->d = preprocess(g->d, perm_seed);
    else
      p->f = preprocess(g->f, perm_seed);
  });
  if (rc) {
    delete p;
    return nullptr;
  }
  return p;
}

void ref_pre_info(void* h, u64* n, u64* feat, u32* classes, u64* nnz_even,
                  u64* nnz_odd) {
  auto* p = static_cast<Pre*>(h);
  auto info = [&](auto& d) {
    *n = d.n;
    *feat = d.feat_dim;
    *classes = d.num_classes;
    *nnz_even = d.a_even.nnz();
    *nnz_odd = d.a_odd.nnz();
  };
  if (p->f64)
    info(p->d);
  else
    info(p->f);
}

// parity 0 -> a_even, 1 -> a_odd
void* ref_pre_csr(void* h, int parity) {
  auto* p = static_cast<Pre*>(h);
  auto* c = new Csr;
  c->f64 = p->f64;
  if (p->f64)
    c->d = parity ? p->d.a_odd : p->d.a_even;
  else
    c->f = parity ? p->f.a_odd : p->f.a_even;
  return c;
}

void ref_pre_copy(void* h, void* features, u32* labels_row, u32* labels_col,
                  u8* mask_row, u8* mask_col) {
  auto* p = static_cast<Pre*>(h);
  auto copy = [&](auto& d) {
    if (features) dense_out(d.features, features);
    std::memcpy(labels_row, d.labels_row_order.data(), d.n * 4);
    std::memcpy(labels_col, d.labels_col_order.data(), d.n * 4);
    std::memcpy(mask_row, d.mask_row_order.data(), d.n);
    std::memcpy(mask_col, d.mask_col_order.data(), d.n);
  };
  if (p->f64)
    copy(p->d);
  else
    copy(p->f);
}

// Builds a PreprocessedDataset from caller arrays (e.g. the GPU shard
// builder's output) so the reference trainers can run on it.
void* ref_pre_from_arrays(u64 n, u64 feat, u32 classes, const u64* ep,
                          const u32* ei, const void* ev, const u64* op,
                          const u32* oi, const void* ov, const void* features,
                          const u32* labels_row, const u32* labels_col,
                          const u8* mask_row, const u8* mask_col, int f64) {
  auto* p = new Pre;
  p->f64 = f64;
  auto fill = [&](auto& d, auto tag) {
    using T = decltype(tag);
    d.n = n;
    d.feat_dim = feat;
    d.num_classes = classes;
    d.a_even = csr_in<T>(n, n, ep, ei, ev);
    d.a_odd = csr_in<T>(n, n, op, oi, ov);
    d.features = dense_in<T>(features, n, feat);
    d.labels_row_order.assign(labels_row, labels_row + n);
    d.labels_col_order.assign(labels_col, labels_col + n);
    d.mask_row_order.assign(mask_row, mask_row + n);
    d.mask_col_order.assign(mask_col, mask_col + n);
  };
  int rc = guarded([&] {
    if (f64)
      fill(p->d, double{});
    else
      fill(p->f, float{});
  });
  if (rc) {
    delete p;
    return nullptr;
  }
  return p;
}

void ref_pre_free(void* h) { delete static_cast<Pre*>(h); }

// ---------------------------------------------------------------------------
// kernels (kernels.hpp:16-173) on caller arrays

int ref_spmm_rows(u64 rows, u64 cols, const u64* rp, const u32* ci,
                  const void* vals, const void* x, u64 x_rows, u64 x_cols,
                  u64 r0, u64 r1, void* out, u64* flops, int f64) {
  return guarded([&] {
    if (f64) {
      auto a = csr_in<double>(rows, cols, rp, ci, vals);
      auto m = dense_in<double>(x, x_rows, x_cols);
      dense_out(spmm_rows(a, m, r0, r1, flops), out);
    } else {
      auto a = csr_in<float>(rows, cols, rp, ci, vals);
      auto m = dense_in<float>(x, x_rows, x_cols);
      dense_out(spmm_rows(a, m, r0, r1, flops), out);
    }
  });
}

int ref_spmm(u64 rows, u64 cols, const u64* rp, const u32* ci, const void* vals,
             const void* x, u64 x_rows, u64 x_cols, void* out, u64* flops,
             int f64) {
  return guarded([&] {
    if (f64) {
      auto a = csr_in<double>(rows, cols, rp, ci, vals);
      dense_out(spmm(a, dense_in<double>(x, x_rows, x_cols), flops), out);
    } else {
      auto a = csr_in<float>(rows, cols, rp, ci, vals);
      dense_out(spmm(a, dense_in<float>(x, x_rows, x_cols), flops), out);
    }
  });
}

// Same as ref_spmm but on an already-built CSR holder (no per-call copy of A).
int ref_spmm_h(void* h, const void* x, u64 x_rows, u64 x_cols, u64 r0, u64 r1,
               void* out, u64* flops) {
  auto* c = static_cast<Csr*>(h);
  return guarded([&] {
    if (c->f64)
      dense_out(spmm_rows(c->d, dense_in<double>(x, x_rows, x_cols), r0, r1, flops), out);
    else
      dense_out(spmm_rows(c->f, dense_in<float>(x, x_rows, x_cols), r0, r1, flops), out);
  });
}

int ref_gemm(const void* a, u64 ar, u64 ac, const void* b, u64 br, u64 bc,
             int ta, int tb, void* out, u64* flops, int f64) {
  return guarded([&] {
    if (f64)
      dense_out(gemm(dense_in<double>(a, ar, ac), dense_in<double>(b, br, bc),
                     ta != 0, tb != 0, flops),
                out);
    else
      dense_out(gemm(dense_in<float>(a, ar, ac), dense_in<float>(b, br, bc),
                     ta != 0, tb != 0, flops),
                out);
  });
}

int ref_relu_forward(const void* q, u64 r, u64 c, void* out, int f64) {
  return guarded([&] {
    if (f64)
      dense_out(relu_forward(dense_in<double>(q, r, c)), out);
    else
      dense_out(relu_forward(dense_in<float>(q, r, c)), out);
  });
}

int ref_relu_backward(const void* q, const void* df, u64 r, u64 c, void* out,
                      int f64) {
  return guarded([&] {
    if (f64)
      dense_out(relu_backward(dense_in<double>(q, r, c), dense_in<double>(df, r, c)), out);
    else
      dense_out(relu_backward(dense_in<float>(q, r, c), dense_in<float>(df, r, c)), out);
  });
}

int ref_ce_sums(const void* logits, u64 r, u64 c, const u32* labels,
                const u8* mask, double* loss_sum, u64* count, u64* correct,
                void* dlogits, int f64) {
  return guarded([&] {
    std::vector<u32> lab(labels, labels + r);
    std::vector<u8> msk(mask, mask + r);
    auto run = [&](auto tag) {
      using T = decltype(tag);
      auto s = softmax_cross_entropy_sums(dense_in<T>(logits, r, c), lab, msk);
      *loss_sum = s.loss_sum;
      *count = s.count;
      *correct = s.correct;
      dense_out(s.dlogits, dlogits);
    };
    if (f64)
      run(double{});
    else
      run(float{});
  });
}

// adam_step (model.hpp:88-111). `step` is the state's step count BEFORE the
// call; the reference increments it.
int ref_adam_step(void* param, const void* grad, void* m, void* v, u64 r, u64 c,
                  u64 step, double lr, double b1, double b2, double eps,
                  int f64) {
  return guarded([&] {
    AdamParams ap{lr, b1, b2, eps};
    auto run = [&](auto tag) {
      using T = decltype(tag);
      auto p = dense_in<T>(param, r, c);
      AdamState<T> st{dense_in<T>(m, r, c), dense_in<T>(v, r, c), step};
      adam_step(p, dense_in<T>(grad, r, c), st, ap);
      dense_out(p, param);
      dense_out(st.m, m);
      dense_out(st.v, v);
    };
    if (f64)
      run(double{});
    else
      run(float{});
  });
}

// init_weights (model.hpp:17-33); output is every layer's W concatenated.
int ref_init_weights(const u64* dims, int ndims, u64 seed, void* out, int f64) {
  return guarded([&] {
    std::vector<std::size_t> d(dims, dims + ndims);
    std::size_t off = 0;
    if (f64) {
      for (auto& w : init_weights<double>(d, seed)) {
        std::memcpy(static_cast<double*>(out) + off, w.data(), w.size() * 8);
        off += w.size();
      }
    } else {
      for (auto& w : init_weights<float>(d, seed)) {
        std::memcpy(static_cast<float*>(out) + off, w.data(), w.size() * 4);
        off += w.size();
      }
    }
  });
}

// ---------------------------------------------------------------------------
// grid / layout algebra (grid.hpp, layout.hpp, model.hpp:35-67)

void ref_plan_layout(int layer, int* inner, int* col_shard, int* row_shard) {
  auto l = plan_layouts(layer + 1).back();
  *inner = static_cast<int>(l.inner);
  *col_shard = static_cast<int>(l.col_shard);
  *row_shard = static_cast<int>(l.row_shard);
}

// out: a_rows a_cols f_rows f_cols w_rows w_cols h_rows h_cols q_rows q_cols
void ref_layer_shapes(int gx, int gy, int gz, int layer, int x, int y, int z,
                      u64 n, u64 d_in, u64 d_out, u64* out) {
  GridConfig g(gx, gy, gz);
  auto l = plan_layouts(layer + 1).back();
  auto s = layer_shapes(g, l, Coords{x, y, z}, n, d_in, d_out);
  u64 v[10] = {s.a_rows, s.a_cols, s.f_rows, s.f_cols, s.w_rows,
               s.w_cols, s.h_rows, s.h_cols, s.q_rows, s.q_cols};
  std::memcpy(out, v, sizeof v);
}

void ref_weight_slice(int gx, int gy, int gz, int layer, int x, int y, int z,
                      u64 d_in, u64 d_out, u64* out) {
  GridConfig g(gx, gy, gz);
  auto l = plan_layouts(layer + 1).back();
  auto s = weight_slice(g, l, Coords{x, y, z}, d_in, d_out);
  out[0] = s.r0, out[1] = s.r1, out[2] = s.c0, out[3] = s.c1;
}

void ref_feature_slice(int gx, int gy, int gz, int x, int y, int z, u64 n,
                       u64 d0, u64* out) {
  GridConfig g(gx, gy, gz);
  auto s = feature_slice(g, Coords{x, y, z}, n, d0);
  out[0] = s.r0, out[1] = s.r1, out[2] = s.c0, out[3] = s.c1;
}

void ref_block_range(int gx, int gy, int gz, int plane, int x, int y, int z,
                     u64 n, u64* out) {
  GridConfig g(gx, gy, gz);
  auto r = adjacency_block_range(g, plane, Coords{x, y, z}, n);
  out[0] = r.row0, out[1] = r.row1, out[2] = r.col0, out[3] = r.col1;
}

void ref_label_row_range(int gx, int gy, int gz, int x, int y, int z, u64 n,
                         int layers, u64* out) {
  GridConfig g(gx, gy, gz);
  auto [a, b] = label_row_range(g, Coords{x, y, z}, n, layers);
  out[0] = a, out[1] = b;
}

// training_collective_volumes (layout.hpp:123-157): rows of
// (layer, forward, op, axis, elems); returns the count (call with out=NULL
// to size).
int ref_collective_volumes(int gx, int gy, int gz, u64 n, const u64* dims,
                           int ndims, u64* out) {
  GridConfig g(gx, gy, gz);
  std::vector<std::size_t> d(dims, dims + ndims);
  auto v = training_collective_volumes(g, n, d);
  if (out)
    for (std::size_t i = 0; i < v.size(); ++i) {
      out[5 * i + 0] = v[i].layer;
      out[5 * i + 1] = v[i].forward;
      out[5 * i + 2] = static_cast<u64>(v[i].op);
      out[5 * i + 3] = static_cast<u64>(v[i].axis);
      out[5 * i + 4] = v[i].elems;
    }
  return static_cast<int>(v.size());
}

// ---------------------------------------------------------------------------
// perf model (perf_model.hpp / src/perf_model.cpp)

// rank_configs; out rows: gx gy gz spmm_s comm_s total_s clamped
int ref_rank_configs(int g, u64 n, u64 nnz, const u64* dims, int ndims,
                     int g_node, double beta_intra, double beta_inter,
                     int bytes_per_scalar, double c1, double c2, double c3,
                     double* out) {
  DatasetStats st{n, nnz, std::vector<std::size_t>(dims, dims + ndims)};
  MachineParams mp{g_node, beta_intra, beta_inter, bytes_per_scalar};
  PerfCoefficients pc{c1, c2, c3, 0, 0};
  std::vector<ConfigPrediction> r;
  int rc = guarded([&] { r = rank_configs(g, st, mp, pc); });
  if (rc) return -rc;
  for (std::size_t i = 0; i < r.size(); ++i) {
    double* o = out + 7 * i;
    o[0] = r[i].shape.gx, o[1] = r[i].shape.gy, o[2] = r[i].shape.gz;
    o[3] = r[i].spmm_seconds, o[4] = r[i].comm_seconds,
    o[5] = r[i].total_seconds, o[6] = r[i].clamped;
  }
  return static_cast<int>(r.size());
}

void ref_comp_features(u64 n, u64 nnz, const u64* dims, int ndims, int gx,
                       int gy, int gz, double* out) {
  DatasetStats st{n, nnz, std::vector<std::size_t>(dims, dims + ndims)};
  auto f = comp_features(st, GridShape{gx, gy, gz});
  out[0] = f.f[0], out[1] = f.f[1], out[2] = f.f[2];
}

double ref_predict_comm(u64 n, u64 nnz, const u64* dims, int ndims, int gx,
                        int gy, int gz, int g_node, double beta_intra,
                        double beta_inter, int bytes_per_scalar) {
  DatasetStats st{n, nnz, std::vector<std::size_t>(dims, dims + ndims)};
  MachineParams mp{g_node, beta_intra, beta_inter, bytes_per_scalar};
  return predict_comm_time(GridShape{gx, gy, gz}, st, mp).total;
}

int ref_fit_regression(const double* features3, const double* seconds, int n,
                       double* out5) {
  std::vector<RegressionSample> s(n);
  for (int i = 0; i < n; ++i) {
    s[i].features = {features3[3 * i], features3[3 * i + 1], features3[3 * i + 2]};
    s[i].seconds = seconds[i];
  }
  return guarded([&] {
    auto c = fit_regression(s);
    out5[0] = c.c1, out5[1] = c.c2, out5[2] = c.c3, out5[3] = c.train_r2,
    out5[4] = c.train_rmse;
  });
}

// ---------------------------------------------------------------------------
// trainers (trainer.hpp:96-211, 478-687)

struct SerialHolder {
  int f64 = 0;
  std::unique_ptr<SerialTrainer<float>> f;
  std::unique_ptr<SerialTrainer<double>> d;
};

static TrainOptions make_opts(const u64* hidden, int nh, u64 seed, int epochs,
                              double lr, int block_count, int fault_epoch) {
  TrainOptions o;
  o.hidden_dims.assign(hidden, hidden + nh);
  o.seed = seed;
  o.epochs = epochs;
  o.adam.lr = lr;
  o.block_count = block_count;
  o.fault_epoch = fault_epoch;
  return o;
}

void* ref_serial_create(void* pre, const u64* hidden, int nh, u64 seed,
                        int epochs, double lr) {
  auto* p = static_cast<Pre*>(pre);
  auto* s = new SerialHolder;
  s->f64 = p->f64;
  auto o = make_opts(hidden, nh, seed, epochs, lr, 0, -1);
  if (p->f64)
    s->d = std::make_unique<SerialTrainer<double>>(p->d, o);
  else
    s->f = std::make_unique<SerialTrainer<float>>(p->f, o);
  return s;
}

// SerialTrainer::forward_backward (trainer.hpp:137-169). Outputs: loss/acc,
// logits (n x C), dW per layer concatenated, dF0 (n x D0), flop counters.
int ref_serial_forward_backward(void* h, int epoch, double* loss, double* acc,
                                void* logits, void* dw_cat, void* df0,
                                u64* spmm_flops, u64* gemm_flops) {
  auto* s = static_cast<SerialHolder*>(h);
  return guarded([&] {
    auto run = [&](auto& tr, auto tag) {
      using T = decltype(tag);
      auto pass = tr->forward_backward(epoch);
      *loss = pass.loss;
      *acc = pass.accuracy;
      if (logits) dense_out(pass.logits, logits);
      if (dw_cat) {
        std::size_t off = 0;
        for (auto& w : pass.dw) {
          dense_out(w, static_cast<T*>(dw_cat) + off);
          off += w.size();
        }
      }
      if (df0) dense_out(pass.df0, df0);
      if (spmm_flops) *spmm_flops = pass.spmm_flops;
      if (gemm_flops) *gemm_flops = pass.gemm_flops;
    };
    if (s->f64)
      run(s->d, double{});
    else
      run(s->f, float{});
  });
}

// SerialTrainer::train; per-epoch loss and accuracy.
// SerialTrainer::forward_only (trainer.hpp:126-135): logits (n x C) of the
// current parameters, no loss, no gradients.
int ref_serial_forward_only(void* h, void* logits) {
  auto* s = static_cast<SerialHolder*>(h);
  return guarded([&] {
    if (s->f64)
      dense_out(s->d->forward_only(), logits);
    else
      dense_out(s->f->forward_only(), logits);
  });
}

int ref_serial_train(void* h, int epochs, double* losses, double* accs) {
  auto* s = static_cast<SerialHolder*>(h);
  return guarded([&] {
    auto run = [&](auto& tr) {
      for (int e = 0; e < epochs; ++e) {
        auto m = tr->run_epoch(e);
        losses[e] = m.loss;
        accs[e] = m.accuracy;
      }
    };
    if (s->f64)
      run(s->d);
    else
      run(s->f);
  });
}

// Current weights (concatenated) and features of the serial trainer.
void ref_serial_params(void* h, void* w_cat, void* features) {
  auto* s = static_cast<SerialHolder*>(h);
  auto run = [&](auto& tr, auto tag) {
    using T = decltype(tag);
    std::size_t off = 0;
    for (auto& w : tr->weights()) {
      dense_out(w, static_cast<T*>(w_cat) + off);
      off += w.size();
    }
    if (features) dense_out(tr->features(), features);
  };
  if (s->f64)
    run(s->d, double{});
  else
    run(s->f, float{});
}

void ref_serial_free(void* h) { delete static_cast<SerialHolder*>(h); }

// train_distributed (trainer.hpp:541-687) on the in-memory handle.
// per-epoch outputs (arrays of length epochs): loss, accuracy, and the phase
// seconds max-over-ranks: fwd_spmm, fwd_gemm, backward, optimizer,
// collectives (5*epochs, row-major per epoch). Optional reassembled weights
// (concatenated) and features.
int ref_train_distributed(void* pre, int gx, int gy, int gz, const u64* hidden,
                          int nh, u64 seed, int epochs, double lr,
                          int block_count, int fault_epoch, int max_running,
                          double* losses, double* accs, double* phase_s,
                          u64* flops2, double* bytes3, void* w_cat,
                          void* features) {
  auto* p = static_cast<Pre*>(pre);
  return guarded([&] {
    auto o = make_opts(hidden, nh, seed, epochs, lr, block_count, fault_epoch);
    ClusterOptions co;
    co.max_running = max_running;
    auto run = [&](auto& d, auto tag) {
      using T = decltype(tag);
      auto r = train_distributed(memory_handle(d), GridConfig(gx, gy, gz), o, co);
      for (int e = 0; e < epochs; ++e) {
        const auto& g = r.global[e];
        losses[e] = g.loss;
        accs[e] = g.accuracy;
        if (phase_s) {
          phase_s[5 * e + 0] = g.forward_spmm_s;
          phase_s[5 * e + 1] = g.forward_gemm_s;
          phase_s[5 * e + 2] = g.backward_s;
          phase_s[5 * e + 3] = g.optimizer_s;
          phase_s[5 * e + 4] = g.collectives_s;
        }
        if (flops2) {
          flops2[2 * e] = g.spmm_flops;
          flops2[2 * e + 1] = g.gemm_flops;
        }
        if (bytes3) {
          bytes3[3 * e] = g.allreduce_bytes;
          bytes3[3 * e + 1] = g.allgather_bytes;
          bytes3[3 * e + 2] = g.reducescatter_bytes;
        }
      }
      if (w_cat) {
        std::size_t off = 0;
        for (auto& w : r.weights) {
          dense_out(w, static_cast<T*>(w_cat) + off);
          off += w.size();
        }
      }
      if (features) dense_out(r.features, features);
    };
    if (p->f64)
      run(p->d, double{});
    else
      run(p->f, float{});
  });
}

// One distributed forward+backward pass (rank_forward_backward,
// trainer.hpp:478-527) on every rank of the grid, outputs reassembled the way
// the reference's engine tests do (test_engine.cpp:30-84): logits in full
// (n x C), dW per layer in full (concatenated), dF0 in full (n x D0).
int ref_distributed_pass(void* pre, int gx, int gy, int gz, const u64* hidden,
                         int nh, u64 seed, int block_count, double* loss,
                         double* acc, void* logits, void* dw_cat, void* df0,
                         u64* flops2, double* comm) {
  auto* p = static_cast<Pre*>(pre);
  return guarded([&] {
    auto run = [&](auto& d, auto tag) {
      using T = decltype(tag);
      GridConfig grid(gx, gy, gz);
      TrainOptions o = make_opts(hidden, nh, seed, 1, 1e-2, block_count, -1);
      const auto dims = model_dims(d.feat_dim, o.hidden_dims, d.num_classes);
      const int layers = static_cast<int>(dims.size()) - 1;
      const auto layouts = plan_layouts(layers);
      const auto gw = init_weights<T>(dims, seed);
      std::vector<DenseMatrix<T>> dw_full;
      for (int l = 0; l < layers; ++l)
        dw_full.push_back(DenseMatrix<T>::zeros(dims[l], dims[l + 1]));
      auto lg = DenseMatrix<T>::zeros(d.n, dims.back());
      auto f0g = DenseMatrix<T>::zeros(d.n, d.feat_dim);
      std::mutex mu;
      double lo = 0, ac = 0;
      Cluster cluster(grid, ClusterOptions{});
      auto stats = cluster.run([&](RankCtx& ctx) {
        const Coords c = ctx.coords();
        auto tensors = slice_rank_tensors(d, grid, c, layers);
        std::vector<GcnLayerState<T>> states(layers);
        for (int l = 0; l < layers; ++l) {
          auto ws = weight_slice(grid, layouts[l], c, dims[l], dims[l + 1]);
          states[l].w = gw[l].block(ws.r0, ws.r1, ws.c0, ws.c1);
        }
        EngineOptions eo;
        eo.block_count = block_count;
        auto pass = rank_forward_backward(ctx, layouts, states, tensors,
                                          tensors.f0, dims, eo, 0);
        std::lock_guard lk(mu);
        if (ctx.rank() == 0) lo = pass.loss, ac = pass.accuracy;
        const auto& last = layouts.back();
        const std::size_t r0 = chunk_start(d.n, grid.extent(last.row_shard),
                                           c.along(last.row_shard));
        const std::size_t c0 = chunk_start(dims.back(), grid.extent(last.inner),
                                           c.along(last.inner));
        for (std::size_t i = 0; i < pass.f_out.rows(); ++i)
          for (std::size_t j = 0; j < pass.f_out.cols(); ++j)
            lg.at(r0 + i, c0 + j) = pass.f_out.at(i, j);
        for (int l = 0; l < layers; ++l) {
          auto ws = weight_slice(grid, layouts[l], c, dims[l], dims[l + 1]);
          for (std::size_t i = 0; i < pass.dw[l].rows(); ++i)
            for (std::size_t j = 0; j < pass.dw[l].cols(); ++j)
              dw_full[l].at(ws.r0 + i, ws.c0 + j) = pass.dw[l].at(i, j);
        }
        auto fs = feature_slice(grid, c, d.n, d.feat_dim);
        for (std::size_t i = 0; i < pass.df0.rows(); ++i)
          for (std::size_t j = 0; j < pass.df0.cols(); ++j)
            f0g.at(fs.r0 + i, fs.c0 + j) = pass.df0.at(i, j);
      });
      *loss = lo;
      *acc = ac;
      if (logits) dense_out(lg, logits);
      if (dw_cat) {
        std::size_t off = 0;
        for (auto& w : dw_full) {
          dense_out(w, static_cast<T*>(dw_cat) + off);
          off += w.size();
        }
      }
      if (df0) dense_out(f0g, df0);
      if (flops2) {
        flops2[0] = flops2[1] = 0;
        for (auto& s : stats) flops2[0] += s.spmm_flops, flops2[1] += s.gemm_flops;
      }
      if (comm)  // per rank, [axis][op]: calls, ring bytes (CommStats::bytes)
        for (std::size_t r = 0; r < stats.size(); ++r)
          for (int a = 0; a < 3; ++a)
            for (int o = 0; o < 3; ++o) {
              const auto ax = static_cast<Axis>(a);
              const auto op = static_cast<CollOp>(o);
              comm[(r * 9 + a * 3 + o) * 2] = static_cast<double>(stats[r].at(ax, op).calls);
              comm[(r * 9 + a * 3 + o) * 2 + 1] = stats[r].bytes(ax, op, grid);
            }
    };
    if (p->f64)
      run(p->d, double{});
    else
      run(p->f, float{});
  });
}

// ---------------------------------------------------------------------------
// CPU baseline sampler (bench.py): the reference's own per-layer ops of one
// 1x1x1 training epoch (SerialTrainer::forward_backward + adam_step,
// trainer.hpp:137-176; same op list as train_distributed on 1x1x1) timed on
// a bounded sample of `rows` consecutive rows per thread, `threads` threads
// on disjoint row blocks, every op linear in the rows it touches. The
// backward aggregation uses A^T = the other permutation variant, which holds
// exactly for the symmetric (undirected) normalized adjacency
// (P_r A P_c^T)^T = P_c A P_r^T. Returns the wall seconds of the sampled
// region; out[0] = estimated full-epoch seconds = wall * n / (threads*rows).
int ref_epoch_sample(void* pre, const u64* hidden, int nh, u64 rows, int threads,
                     double* out) {
  auto* p = static_cast<Pre*>(pre);
  return guarded([&] {
    check(!p->f64, "ref_epoch_sample: float datasets only");
    auto& d = p->f;
    std::vector<std::size_t> dims{d.feat_dim};
    for (int i = 0; i < nh; ++i) dims.push_back(hidden[i]);
    dims.push_back(d.num_classes);
    const int L = static_cast<int>(dims.size()) - 1;
    const std::size_t n = d.n;
    std::size_t dmax = 0;
    for (auto x : dims) dmax = std::max(dmax, x);
    // one shared dense operand at the widest width; the narrower layers read
    // its leading columns (content does not change the op cost)
    auto x_full = DenseMatrix<float>::zeros(n, dmax);
    for (std::size_t i = 0; i < x_full.size(); ++i) x_full.data()[i] = 0.001f * (i % 997);
    std::vector<DenseMatrix<float>> xs;
    for (int l = 0; l < L; ++l) xs.push_back(x_full.block(0, n, 0, dims[l]));
    x_full = DenseMatrix<float>();
    auto ws = init_weights<float>(dims, 0);
    std::vector<u32> labels(rows, 0);
    std::vector<u8> mask(rows, 1);
    AdamParams ap;
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
      pool.emplace_back([&, t] {
        const std::size_t r0 = (static_cast<std::size_t>(t) * rows) % (n > rows ? n - rows : 1);
        const std::size_t r1 = std::min(n, r0 + rows);
        std::vector<DenseMatrix<float>> h(L), q(L);
        for (int l = 0; l < L; ++l) {
          const auto& a = l % 2 ? d.a_odd : d.a_even;
          h[l] = spmm_rows(a, xs[l], r0, r1);
          q[l] = gemm(h[l], ws[l]);
          if (l + 1 < L) q[l] = relu_forward(q[l]);
        }
        auto sums = softmax_cross_entropy_sums(
            q[L - 1], std::vector<u32>(labels.begin(), labels.begin() + (r1 - r0)),
            std::vector<u8>(mask.begin(), mask.begin() + (r1 - r0)));
        DenseMatrix<float> df = std::move(sums.dlogits);
        for (int l = L - 1; l >= 0; --l) {
          auto dq = l == L - 1 ? df : relu_backward(q[l], df);
          auto dw = gemm(dq, h[l], true, false).transposed();
          auto dh = gemm(dq, ws[l], false, true);
          const auto& at = l % 2 ? d.a_even : d.a_odd;
          df = spmm_rows(at, xs[l], r0, r1);
          (void)dw;
          (void)dh;
        }
        auto f0 = d.features.block(r0, r1, 0, dims[0]);
        auto st = AdamState<float>::like(f0);
        adam_step(f0, df, st, ap);
      });
    for (auto& th : pool) th.join();
    const double wall =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    out[0] = wall * static_cast<double>(n) / (static_cast<double>(threads) * rows);
    out[1] = wall;
  });
}

// SerialTrainer::forward_backward (trainer.hpp:137-169) with the reference's
// own kernels composed over `threads` row blocks — the checker for passes too
// large for one thread (C2: 116.6M nonzeros, 100-256-256-47). Row-local ops
// (spmm_rows, the NN / NT gemms, relu, per-row CE) are bitwise those of the
// serial pass: every output row is the same loop over the same operands.
// The two cross-row reductions are not: the CE loss_sum (double; blocks
// summed in order) and dW = H^T dQ over K = n rows, which is returned in
// double (the reference's gemm at T = double on the fp32 operands, block
// partials summed in double) — at K = 2M rows the serial fp32 chain's own
// rounding is ~1e-4 normwise, so dW is gated against this fp64 value.
// Outputs: loss, accuracy, logits (n x C), dW (f64) concatenated, dF0
// (n x F), H of layer 0.
int ref_serial_pass_parallel(void* pre, const u64* hidden, int nh, u64 seed, int threads,
                             double* loss, double* acc, float* logits, double* dw_cat,
                             float* df0, float* h0, int sample_cols, float* dw_serial) {
  auto* p = static_cast<Pre*>(pre);
  return guarded([&] {
    check(!p->f64, "ref_serial_pass_parallel: float datasets only");
    const auto& d = p->f;
    std::vector<std::size_t> dims{d.feat_dim};
    for (int i = 0; i < nh; ++i) dims.push_back(hidden[i]);
    dims.push_back(d.num_classes);
    const int L = static_cast<int>(dims.size()) - 1;
    const std::size_t n = d.n;
    const int T = std::max(1, threads);
    std::size_t dims_max_ = 0;
    for (auto x : dims) dims_max_ = std::max(dims_max_, x);
    auto ws = init_weights<float>(dims, seed);
    const CsrMatrix<float> at_even = d.a_even.transpose(), at_odd = d.a_odd.transpose();
    auto par = [&](auto&& body) {
      std::vector<std::thread> pool;
      for (int t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
          const std::size_t r0 = n * t / T, r1 = n * (t + 1) / T;
          body(t, r0, r1);
        });
      for (auto& th : pool) th.join();
    };
    auto put = [&](DenseMatrix<float>& dst, std::size_t r0, const DenseMatrix<float>& blk) {
      if (blk.size()) std::memcpy(dst.data() + r0 * dst.cols(), blk.data(), blk.size() * sizeof(float));
    };
    std::vector<DenseMatrix<float>> h(L), q(L);
    DenseMatrix<float> f = d.features;
    for (int l = 0; l < L; ++l) {
      const auto& a = l % 2 ? d.a_odd : d.a_even;
      h[l] = DenseMatrix<float>::zeros(n, dims[l]);
      q[l] = DenseMatrix<float>::zeros(n, dims[l + 1]);
      DenseMatrix<float> fn = l + 1 < L ? DenseMatrix<float>::zeros(n, dims[l + 1])
                                        : DenseMatrix<float>();
      par([&](int, std::size_t r0, std::size_t r1) {
        auto hb = spmm_rows(a, f, r0, r1);
        auto qb = gemm(hb, ws[l]);
        put(h[l], r0, hb);
        put(q[l], r0, qb);
        if (l + 1 < L) put(fn, r0, relu_forward(qb));
      });
      if (l + 1 < L) f = std::move(fn);
    }
    const int parity = final_output_parity(L);
    const auto& labels = d.labels_for_parity(parity);
    const auto& mask = d.mask_for_parity(parity);
    std::vector<double> lsum(T);
    std::vector<u64> cnt(T), cor(T);
    auto df = DenseMatrix<float>::zeros(n, dims[L]);
    par([&](int t, std::size_t r0, std::size_t r1) {
      auto s = softmax_cross_entropy_sums(
          q[L - 1].block(r0, r1, 0, dims[L]),
          std::vector<u32>(labels.begin() + r0, labels.begin() + r1),
          std::vector<u8>(mask.begin() + r0, mask.begin() + r1));
      lsum[t] = s.loss_sum, cnt[t] = s.count, cor[t] = s.correct;
      put(df, r0, s.dlogits);
    });
    double sum = 0;
    u64 count = 0, correct = 0;
    for (int t = 0; t < T; ++t) sum += lsum[t], count += cnt[t], correct += cor[t];
    CrossEntropySums<float> all;
    all.dlogits = std::move(df);
    auto lr = detail::finalize_loss<float>(std::move(all), sum, count, correct, 0);
    *loss = lr.loss;
    *acc = lr.accuracy;
    std::memcpy(logits, q[L - 1].data(), q[L - 1].size() * sizeof(float));
    if (h0) std::memcpy(h0, h[0].data(), h[0].size() * sizeof(float));
    df = std::move(lr.dlogits);
    std::vector<std::size_t> off(L, 0);
    for (int l = 1; l < L; ++l) off[l] = off[l - 1] + dims[l - 1] * dims[l];
    for (int l = L - 1; l >= 0; --l) {
      const auto& at = l % 2 ? at_odd : at_even;
      auto dq = l == L - 1 ? std::move(df) : DenseMatrix<float>::zeros(n, dims[l + 1]);
      auto dh = DenseMatrix<float>::zeros(n, dims[l]);
      std::vector<DenseMatrix<double>> dwp(T);
      par([&](int t, std::size_t r0, std::size_t r1) {
        DenseMatrix<float> dqb = l == L - 1 ? dq.block(r0, r1, 0, dims[l + 1])
                                            : relu_backward(q[l].block(r0, r1, 0, dims[l + 1]),
                                                            df.block(r0, r1, 0, dims[l + 1]));
        if (l != L - 1) put(dq, r0, dqb);
        // dW = H^T dQ in T = double: the reference's own gemm at double
        // precision on the fp32 operands, block partials summed in double
        auto hb = h[l].block(r0, r1, 0, dims[l]);
        dwp[t] = gemm(DenseMatrix<double>(hb.rows(), hb.cols(),
                                          std::vector<double>(hb.data(), hb.data() + hb.size())),
                      DenseMatrix<double>(dqb.rows(), dqb.cols(),
                                          std::vector<double>(dqb.data(), dqb.data() + dqb.size())),
                      true, false);
        put(dh, r0, gemm(dqb, ws[l], false, true));
      });
      // the serial trainer's own fp32 dW for the first `sample_cols`
      // columns: gemm(h, dq[:, j], true) over all n rows in one k chain,
      // one column per thread (trainer.hpp:163)
      if (dw_serial && sample_cols > 0) {
        const int sc = std::min<int>(sample_cols, static_cast<int>(dims[l + 1]));
        std::vector<std::thread> cols;
        std::vector<DenseMatrix<float>> res(sc);
        for (int j = 0; j < sc; ++j)
          cols.emplace_back([&, j] { res[j] = gemm(h[l], dq.block(0, n, j, j + 1), true, false); });
        for (auto& th : cols) th.join();
        float* dst = dw_serial + l * dims_max_ * sample_cols;
        for (int j = 0; j < sc; ++j)
          for (std::size_t i = 0; i < dims[l]; ++i) dst[i * sample_cols + j] = res[j].at(i, 0);
      }
      DenseMatrix<double> dw = std::move(dwp[0]);
      for (int t = 1; t < T; ++t)
        for (std::size_t i = 0; i < dw.size(); ++i) dw.data()[i] += dwp[t].data()[i];
      for (std::size_t i = 0; i < dw.size(); ++i) dw_cat[off[l] + i] = dw.data()[i];
      auto dfn = DenseMatrix<float>::zeros(n, dims[l]);
      par([&](int, std::size_t r0, std::size_t r1) { put(dfn, r0, spmm_rows(at, dh, r0, r1)); });
      df = std::move(dfn);
    }
    std::memcpy(df0, df.data(), df.size() * sizeof(float));
  });
}

// ---------------------------------------------------------------------------
// shard files (shard_io.hpp:278-536, trainer.hpp:252-438): the reference's
// writer and readers, for byte-level parity of the PLXS files and the
// per-rank loader

int ref_write_shards(void* pre, int p, int q, const char* dir, const char* name) {
  auto* h = static_cast<Pre*>(pre);
  return guarded([&] {
    if (h->f64)
      shard_io::write_shards(h->d, p, q, dir, name);
    else
      shard_io::write_shards(h->f, p, q, dir, name);
  });
}

void* ref_load_preprocessed(const char* dir) {
  auto* out = new Pre;
  int rc = guarded([&] {
    auto m = shard_io::load_manifest(dir);
    out->f64 = m.precision == 8;
    if (out->f64)
      out->d = load_preprocessed<double>(m);
    else
      out->f = load_preprocessed<float>(m);
  });
  if (rc) {
    delete out;
    return nullptr;
  }
  return out;
}

struct RankHolder {
  int f64 = 0;
  RankTensors<float> f;
  RankTensors<double> d;
};

void* ref_load_rank_shards(const char* dir, int gx, int gy, int gz, int x, int y, int z,
                           int layers) {
  auto* out = new RankHolder;
  int rc = guarded([&] {
    auto m = shard_io::load_manifest(dir);
    out->f64 = m.precision == 8;
    if (out->f64)
      out->d = load_rank_shards<double>(m, GridConfig(gx, gy, gz), Coords{x, y, z}, layers);
    else
      out->f = load_rank_shards<float>(m, GridConfig(gx, gy, gz), Coords{x, y, z}, layers);
  });
  if (rc) {
    delete out;
    return nullptr;
  }
  return out;
}

// the (plane, parity) adjacency block (0) or its transpose (1) as a Csr handle
void* ref_rank_adj(void* h, int plane, int parity, int transposed) {
  auto* r = static_cast<RankHolder*>(h);
  auto* c = new Csr;
  c->f64 = r->f64;
  LayerLayout lay;  // get() keys by (layer % 3, layer % 2)
  for (int l = 0; l < 6; ++l)
    if (l % 3 == plane && l % 2 == parity) lay.layer = l;
  int rc = guarded([&] {
    if (r->f64) {
      const auto& s = r->d.adj.get(lay);
      c->d = transposed ? s.at : s.a;
    } else {
      const auto& s = r->f.adj.get(lay);
      c->f = transposed ? s.at : s.a;
    }
  });
  if (rc) {
    delete c;
    return nullptr;
  }
  return c;
}

void ref_rank_info(void* h, u64* f0_rows, u64* f0_cols, u64* labels, int* files_read,
                   u64* bytes_read) {
  auto* r = static_cast<RankHolder*>(h);
  auto info = [&](auto& t) {
    *f0_rows = t.f0.rows();
    *f0_cols = t.f0.cols();
    *labels = t.labels.size();
    *files_read = t.files_read;
    *bytes_read = t.bytes_read;
  };
  if (r->f64)
    info(r->d);
  else
    info(r->f);
}

void ref_rank_copy(void* h, void* f0, u32* labels, u8* mask) {
  auto* r = static_cast<RankHolder*>(h);
  auto copy = [&](auto& t) {
    dense_out(t.f0, f0);
    if (!t.labels.empty()) std::memcpy(labels, t.labels.data(), t.labels.size() * 4);
    if (!t.mask.empty()) std::memcpy(mask, t.mask.data(), t.mask.size());
  };
  if (r->f64)
    copy(r->d);
  else
    copy(r->f);
}

void ref_rank_free(void* h) { delete static_cast<RankHolder*>(h); }

}  // extern "C"
