// plexuskit_b200.hpp — the reference's own C++ entry points, forwarded to
// the B200 library (libplexus_b200.so) through its C ABI (plexus_b200.h).
//
// A maintainer drops this header next to the reference's headers
// (/root/reference/proj/include/plexuskit; paths below are relative to it)
// and calls plexuskit::b200::X where the reference calls plexuskit::X — same
// argument types, same value semantics (host DenseMatrix / CsrMatrix in,
// fresh matrices out), same exception types (ContractError, MemoryError,
// TrainingError, IoError, ClusterAborted). Each function uploads its
// operands, runs the sm_100a kernels and downloads the result; the device
// engine path (train_distributed) keeps everything resident across epochs.
// Link: -lplexus_b200 -lcudart. float only (the library's T = float).
//
//   kernels.hpp:17-19   spmm                 kernels.hpp:41-43  spmm_rows
//   kernels.hpp:66-69   gemm                 kernels.hpp:94-111 relu_forward/backward
//   kernels.hpp:125-128 softmax_cross_entropy_sums
//   model.hpp:88-90     adam_step            csr.hpp:78-95      transpose
//   trainer.hpp:541-545 train_distributed (DatasetHandle loader per rank,
//                       one engine per rank, in-process cluster over the
//                       visible GPUs; ClusterOptions accepted, scheduling is
//                       the GPU's)
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "plexus_b200.h"
#include "plexuskit/trainer.hpp"

namespace plexuskit::b200 {

namespace detail {

// pk_status -> the reference's exception types (common.hpp:16-45,
// trainer.hpp:26-29, cluster.hpp:67-71)
inline void rethrow(int rc) {
  if (rc == PK_OK) return;
  const std::string msg = pk_last_error();
  switch (rc) {
    case PK_ERR_CONTRACT: throw ContractError(msg);
    case PK_ERR_MEMORY: throw MemoryError(msg);
    case PK_ERR_TRAINING: throw TrainingError(msg);
    case PK_ERR_ABORTED: throw ClusterAborted();
    default:
      if (rc >= PK_ERR_IO_MISSING && rc <= PK_ERR_IO_WRITE)
        throw IoError(static_cast<IoErrorCode>(rc - PK_ERR_IO_MISSING), msg);
      throw std::runtime_error("libplexus_b200 (status " + std::to_string(rc) + "): " + msg);
  }
}

inline void cuda(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation) throw MemoryError(std::string(what) + ": out of device memory");
  throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

// A device array owned for the duration of one forwarded call.
template <typename T>
class Dev {
 public:
  explicit Dev(std::size_t n) : n_(n) {
    if (n_) cuda(cudaMalloc(&p_, n_ * sizeof(T)), "cudaMalloc");
  }
  Dev(const T* host, std::size_t n) : Dev(n) {
    if (n_) cuda(cudaMemcpy(p_, host, n_ * sizeof(T), cudaMemcpyHostToDevice), "upload");
  }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  ~Dev() {
    if (p_) cudaFree(p_);
  }
  T* get() const { return p_; }
  void download(T* host) const {
    if (n_) cuda(cudaMemcpy(host, p_, n_ * sizeof(T), cudaMemcpyDeviceToHost), "download");
  }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

// A CsrMatrix<float> resident on the device for one call.
struct DevCsr {
  Dev<u64> rp;
  Dev<u32> ci;
  Dev<float> v;
  pk_csr view{};
  explicit DevCsr(const CsrMatrix<float>& a)
      : rp(a.row_ptr().data(), a.row_ptr().size()),
        ci(a.col_idx().data(), a.col_idx().size()),
        v(a.values().data(), a.values().size()) {
    view.rows = static_cast<int64_t>(a.rows());
    view.cols = static_cast<int64_t>(a.cols());
    view.nnz = a.nnz();
    view.row_ptr = rp.get();
    view.col_idx = ci.get();
    view.values = v.get();
  }
};

inline DenseMatrix<float> download(const Dev<float>& d, std::size_t rows, std::size_t cols) {
  auto out = DenseMatrix<float>::zeros(rows, cols);
  d.download(out.data());
  return out;
}

}  // namespace detail

// ---------------------------------------------------------------------------
// kernels (kernels.hpp)

inline DenseMatrix<float> spmm_rows(const CsrMatrix<float>& a, const DenseMatrix<float>& f,
                                    std::size_t r0, std::size_t r1, u64* flops = nullptr) {
  detail::DevCsr da(a);
  detail::Dev<float> x(f.data(), f.size());
  detail::Dev<float> y(std::max<std::size_t>(r1 > r0 ? r1 - r0 : 0, 0) * f.cols());
  detail::rethrow(pk_spmm_rows_f32(&da.view, static_cast<int64_t>(r0), static_cast<int64_t>(r1),
                                   x.get(), static_cast<int64_t>(f.rows()),
                                   static_cast<int64_t>(f.cols()), static_cast<int64_t>(f.cols()),
                                   y.get(), static_cast<int64_t>(f.cols()), flops, nullptr));
  return detail::download(y, r1 - r0, f.cols());
}

inline DenseMatrix<float> spmm(const CsrMatrix<float>& a, const DenseMatrix<float>& f,
                               u64* flops = nullptr) {
  detail::DevCsr da(a);
  detail::Dev<float> x(f.data(), f.size());
  detail::Dev<float> y(a.rows() * f.cols());
  detail::rethrow(pk_spmm_f32(&da.view, x.get(), static_cast<int64_t>(f.rows()),
                              static_cast<int64_t>(f.cols()), static_cast<int64_t>(f.cols()),
                              y.get(), static_cast<int64_t>(f.cols()), flops, nullptr));
  return detail::download(y, a.rows(), f.cols());
}

// mode: PK_MODE_PARITY (default) reproduces the reference's loop bit for bit;
// PK_MODE_FAST runs the tcgen05 3xTF32 tensor-core path.
inline DenseMatrix<float> gemm(const DenseMatrix<float>& a, const DenseMatrix<float>& b,
                               bool transpose_a = false, bool transpose_b = false,
                               u64* flops = nullptr, int mode = PK_MODE_PARITY) {
  const std::size_t m = transpose_a ? a.cols() : a.rows();
  const std::size_t k = transpose_a ? a.rows() : a.cols();
  const std::size_t kb = transpose_b ? b.cols() : b.rows();
  const std::size_t n = transpose_b ? b.rows() : b.cols();
  check(k == kb, "gemm: inner dimensions disagree (" + a.shape_str() +
                     (transpose_a ? "^T" : "") + " x " + b.shape_str() +
                     (transpose_b ? "^T" : "") + ")");
  detail::Dev<float> da(a.data(), a.size()), db(b.data(), b.size()), dc(m * n);
  detail::rethrow(pk_gemm_f32(transpose_a, transpose_b, static_cast<int64_t>(m),
                              static_cast<int64_t>(n), static_cast<int64_t>(k), da.get(),
                              static_cast<int64_t>(a.cols()), db.get(),
                              static_cast<int64_t>(b.cols()), dc.get(), static_cast<int64_t>(n),
                              mode, flops, nullptr));
  return detail::download(dc, m, n);
}

inline DenseMatrix<float> relu_forward(const DenseMatrix<float>& q) {
  detail::Dev<float> dq(q.data(), q.size()), out(q.size());
  const auto c = static_cast<int64_t>(q.cols());
  detail::rethrow(pk_relu_forward_f32(dq.get(), c, static_cast<int64_t>(q.rows()), c, out.get(),
                                      c, nullptr));
  return detail::download(out, q.rows(), q.cols());
}

inline DenseMatrix<float> relu_backward(const DenseMatrix<float>& q, const DenseMatrix<float>& df) {
  check(q.same_shape(df), "relu_backward: shapes " + q.shape_str() + " and " + df.shape_str() +
                              " differ");
  detail::Dev<float> dq(q.data(), q.size()), ddf(df.data(), df.size()), out(q.size());
  const auto c = static_cast<int64_t>(q.cols());
  detail::rethrow(pk_relu_backward_f32(dq.get(), c, ddf.get(), c,
                                       static_cast<int64_t>(q.rows()), c, out.get(), c, nullptr));
  return detail::download(out, q.rows(), q.cols());
}

inline CrossEntropySums<float> softmax_cross_entropy_sums(const DenseMatrix<float>& logits,
                                                          const std::vector<u32>& labels,
                                                          const std::vector<u8>& mask) {
  check(labels.size() == logits.rows() && mask.size() == logits.rows(),
        "softmax_cross_entropy_sums: labels/mask length must equal logits rows");
  detail::Dev<float> dl(logits.data(), logits.size()), dd(logits.size());
  detail::Dev<u32> lab(labels.data(), labels.size());
  detail::Dev<u8> msk(mask.data(), mask.size());
  detail::Dev<double> sums(3);
  const auto c = static_cast<int64_t>(logits.cols());
  detail::rethrow(pk_softmax_ce_sums_f32(dl.get(), c, static_cast<int64_t>(logits.rows()), c,
                                         lab.get(), msk.get(), dd.get(), c, sums.get(), nullptr));
  double h[3];
  sums.download(h);
  CrossEntropySums<float> out;
  out.loss_sum = h[0];
  out.count = static_cast<u64>(h[1]);
  out.correct = static_cast<u64>(h[2]);
  out.dlogits = detail::download(dd, logits.rows(), logits.cols());
  return out;
}

// model.hpp:88-111: the step counter advances here, bias terms in double
inline void adam_step(DenseMatrix<float>& param, const DenseMatrix<float>& grad,
                      AdamState<float>& state, const AdamParams& opts) {
  check(param.same_shape(grad) && param.same_shape(state.m),
        "adam_step: parameter " + param.shape_str() + ", gradient " + grad.shape_str() +
            " and state shapes must agree");
  detail::Dev<float> p(param.data(), param.size()), g(grad.data(), grad.size());
  detail::Dev<float> m(state.m.data(), state.m.size()), v(state.v.data(), state.v.size());
  detail::rethrow(pk_adam_step_f32(p.get(), g.get(), m.get(), v.get(),
                                   static_cast<int64_t>(param.size()), state.step + 1, opts.lr,
                                   opts.beta1, opts.beta2, opts.eps, nullptr));
  state.step++;
  p.download(param.data());
  m.download(state.m.data());
  v.download(state.v.data());
}

// csr.hpp:78-95
inline CsrMatrix<float> transpose(const CsrMatrix<float>& a) {
  detail::DevCsr da(a);
  pk_csr_owned t{};
  detail::rethrow(pk_csr_transpose(&da.view, &t, nullptr));
  std::vector<u64> rp(static_cast<std::size_t>(t.rows) + 1);
  std::vector<u32> ci(t.nnz);
  std::vector<float> v(t.nnz);
  detail::cuda(cudaMemcpy(rp.data(), t.row_ptr, rp.size() * 8, cudaMemcpyDeviceToHost), "download");
  if (t.nnz) {
    detail::cuda(cudaMemcpy(ci.data(), t.col_idx, t.nnz * 4, cudaMemcpyDeviceToHost), "download");
    detail::cuda(cudaMemcpy(v.data(), t.values, t.nnz * 4, cudaMemcpyDeviceToHost), "download");
  }
  const auto rows = static_cast<std::size_t>(t.rows), cols = static_cast<std::size_t>(t.cols);
  pk_csr_free(&t);
  return CsrMatrix<float>(rows, cols, std::move(rp), std::move(ci), std::move(v));
}

// ---------------------------------------------------------------------------
// train_distributed (trainer.hpp:541-687)

struct DeviceOptions {
  int mode = PK_MODE_FAST;      // dense transforms: tcgen05 3xTF32 or PARITY
  int64_t hub_threshold = 0;    // SpMM hub rows (0 = automatic)
  std::vector<int> devices;     // rank r runs on devices[r % size]; empty = all visible
};

inline TrainResult<float> train_distributed(const DatasetHandle<float>& data,
                                            const GridConfig& grid, const TrainOptions& opts,
                                            const ClusterOptions& = {},
                                            const DeviceOptions& eng = {}) {
  const auto dims = model_dims(data.feat_dim, opts.hidden_dims, data.classes);
  const int layers = static_cast<int>(dims.size()) - 1;
  check(layers <= PK_MAX_LAYERS, "train_distributed: too many layers");
  const auto layouts = plan_layouts(layers);
  std::vector<int> devices = eng.devices;
  if (devices.empty()) {
    int n = 0;
    detail::cuda(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
    for (int d = 0; d < n; ++d) devices.push_back(d);
  }
  check(!devices.empty(), "train_distributed: no CUDA device");
  pk_cluster* cl = nullptr;
  detail::rethrow(pk_cluster_create(grid.gx(), grid.gy(), grid.gz(), &cl));

  struct RankOut {
    std::vector<EpochMetrics> epochs;
    std::vector<DenseMatrix<float>> w_shards;
    DenseMatrix<float> f0;
    u64 bytes_read = 0;
    int files_read = 0;
    double load_s = 0;
    std::exception_ptr err;
    bool aborted = false;
  };
  std::vector<RankOut> outs(grid.size());
  auto rank_body = [&](int r) {
    RankOut& mine = outs[r];
    pk_engine* e = nullptr;
    try {
      detail::cuda(cudaSetDevice(devices[r % devices.size()]), "cudaSetDevice");
      pk_engine_config cfg{};
      cfg.gx = grid.gx(), cfg.gy = grid.gy(), cfg.gz = grid.gz();
      cfg.rank = r;
      cfg.device = devices[r % devices.size()];
      cfg.num_layers = layers;
      for (int i = 0; i <= layers; ++i) cfg.dims[i] = static_cast<int64_t>(dims[i]);
      cfg.n = static_cast<int64_t>(data.n);
      cfg.seed = opts.seed;
      cfg.lr = opts.adam.lr, cfg.beta1 = opts.adam.beta1, cfg.beta2 = opts.adam.beta2;
      cfg.eps = opts.adam.eps;
      cfg.block_count = opts.block_count;
      cfg.mode = eng.mode;
      cfg.fault_epoch = opts.fault_epoch;
      cfg.hub_threshold = eng.hub_threshold;
      detail::rethrow(pk_engine_create(&cfg, &e));
      detail::rethrow(pk_engine_comm_init_local(e, cl));
      const auto t0 = std::chrono::steady_clock::now();
      RankTensors<float> t = data.loader(grid, grid.coords_of(r), layers);
      mine.bytes_read = t.bytes_read;
      mine.files_read = t.files_read;
      // the rank's tensors go to its device once; the engine copies them
      std::vector<std::unique_ptr<detail::DevCsr>> blocks;
      pk_rank_view rv{};
      for (int plane = 0; plane < 3; ++plane)
        for (int parity = 0; parity < 2; ++parity) {
          if (!t.adj.has(plane, parity)) continue;
          LayerLayout lay{};
          lay.layer = plane % 2 == parity ? plane : plane + 3;  // a layer with this key
          blocks.push_back(std::make_unique<detail::DevCsr>(t.adj.get(lay).a));
          rv.adj[plane * 2 + parity] = blocks.back()->view;
        }
      detail::Dev<float> f0(t.f0.data(), t.f0.size());
      detail::Dev<u32> lab(t.labels.data(), t.labels.size());
      detail::Dev<u8> msk(t.mask.data(), t.mask.size());
      rv.f0 = f0.get();
      rv.f0_rows = static_cast<int64_t>(t.f0.rows());
      rv.f0_cols = rv.ld_f0 = static_cast<int64_t>(t.f0.cols());
      rv.labels = lab.get();
      rv.mask = msk.get();
      rv.label_rows = static_cast<int64_t>(t.labels.size());
      detail::rethrow(pk_engine_load_rank(e, &rv));
      mine.load_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      for (int ep = 0; ep < opts.epochs; ++ep) {
        pk_epoch_metrics pm{};
        detail::rethrow(pk_engine_train_epoch(e, ep, &pm));
        EpochMetrics m;
        m.epoch = ep;
        m.loss = pm.loss;
        m.accuracy = pm.accuracy;
        m.load_s = ep == 0 ? mine.load_s : 0;
        m.forward_spmm_s = pm.forward_spmm_s;
        m.forward_gemm_s = pm.forward_gemm_s;
        m.backward_s = pm.backward_s;
        m.optimizer_s = pm.optimizer_s;
        m.collectives_s = pm.collectives_s;
        m.spmm_flops = pm.spmm_flops;
        m.gemm_flops = pm.gemm_flops;
        m.allreduce_bytes = pm.allreduce_bytes;
        m.allgather_bytes = pm.allgather_bytes;
        m.reducescatter_bytes = pm.reducescatter_bytes;
        mine.epochs.push_back(m);
      }
      auto fetch = [&](int which, int l) {
        pk_tensor_view v{};
        detail::rethrow(pk_engine_tensor(e, which, l, &v));
        auto out = DenseMatrix<float>::zeros(static_cast<std::size_t>(v.rows),
                                             static_cast<std::size_t>(v.cols));
        if (v.rows && v.cols)
          detail::cuda(cudaMemcpy2D(out.data(), v.cols * sizeof(float), v.data,
                                    v.ld * sizeof(float), v.cols * sizeof(float), v.rows,
                                    cudaMemcpyDeviceToHost),
                       "download");
        return out;
      };
      for (int l = 0; l < layers; ++l) mine.w_shards.push_back(fetch(PK_T_W, l));
      mine.f0 = fetch(PK_T_F0, 0);
    } catch (const ClusterAborted&) {
      mine.aborted = true;
      mine.err = std::current_exception();
    } catch (...) {
      mine.err = std::current_exception();
      pk_cluster_abort(cl, r, "rank failed");
    }
    if (e) pk_engine_destroy(e);
  };
  std::vector<std::thread> pool;
  for (int r = 0; r < grid.size(); ++r) pool.emplace_back(rank_body, r);
  for (auto& th : pool) th.join();
  pk_cluster_destroy(cl);
  // the primary failure wins over the ClusterAborted it caused (cluster.hpp:436-441)
  for (auto& o : outs)
    if (o.err && !o.aborted) std::rethrow_exception(o.err);
  for (auto& o : outs)
    if (o.err) std::rethrow_exception(o.err);

  // host-side reassembly, as the reference does it (trainer.hpp:636-686)
  TrainResult<float> result;
  result.per_rank.resize(grid.size());
  for (int r = 0; r < grid.size(); ++r) {
    result.per_rank[r] = outs[r].epochs;
    result.bytes_read.push_back(outs[r].bytes_read);
    result.files_read.push_back(outs[r].files_read);
    result.load_seconds = std::max(result.load_seconds, outs[r].load_s);
  }
  for (int l = 0; l < layers; ++l) {
    auto w = DenseMatrix<float>::zeros(dims[l], dims[l + 1]);
    for (int r = 0; r < grid.size(); ++r) {
      auto ws = weight_slice(grid, layouts[l], grid.coords_of(r), dims[l], dims[l + 1]);
      const auto& sh = outs[r].w_shards[l];
      for (std::size_t i = 0; i < sh.rows(); ++i)
        for (std::size_t j = 0; j < sh.cols(); ++j) w.at(ws.r0 + i, ws.c0 + j) = sh.at(i, j);
    }
    result.weights.push_back(std::move(w));
  }
  result.features = DenseMatrix<float>::zeros(data.n, data.feat_dim);
  for (int r = 0; r < grid.size(); ++r) {
    auto fs = feature_slice(grid, grid.coords_of(r), data.n, data.feat_dim);
    const auto& sh = outs[r].f0;
    for (std::size_t i = 0; i < sh.rows(); ++i)
      for (std::size_t j = 0; j < sh.cols(); ++j)
        result.features.at(fs.r0 + i, fs.c0 + j) = sh.at(i, j);
  }
  for (int ep = 0; ep < opts.epochs; ++ep) {
    EpochMetrics g;
    g.epoch = ep;
    g.loss = outs[0].epochs[ep].loss;
    g.accuracy = outs[0].epochs[ep].accuracy;
    for (int r = 0; r < grid.size(); ++r) {
      const auto& m = outs[r].epochs[ep];
      g.load_s = std::max(g.load_s, m.load_s);
      g.forward_spmm_s = std::max(g.forward_spmm_s, m.forward_spmm_s);
      g.forward_gemm_s = std::max(g.forward_gemm_s, m.forward_gemm_s);
      g.backward_s = std::max(g.backward_s, m.backward_s);
      g.optimizer_s = std::max(g.optimizer_s, m.optimizer_s);
      g.collectives_s = std::max(g.collectives_s, m.collectives_s);
      g.spmm_flops += m.spmm_flops;
      g.gemm_flops += m.gemm_flops;
      g.allreduce_bytes += m.allreduce_bytes;
      g.allgather_bytes += m.allgather_bytes;
      g.reducescatter_bytes += m.reducescatter_bytes;
    }
    result.global.push_back(g);
  }
  return result;
}

}  // namespace plexuskit::b200
