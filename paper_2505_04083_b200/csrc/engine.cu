// Per-rank GCN engine: device twin of forward_layer / backward_layer
// (engine.hpp:158-259), rank_forward_backward (trainer.hpp:478-527) and the
// epoch body of train_distributed (trainer.hpp:586-628).
#include <cuda_runtime.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>

#include "engine.cuh"
#include "gemm.cuh"
#include "philox.cuh"
#include "shard_builder.cuh"

namespace pk {

namespace {

i64 pad4(i64 c) { return c <= 0 ? 4 : (c + 3) / 4 * 4; }

// 8 B per nonzero (u32 col + f32 val) + 8 B per row_ptr entry
// + one gathered feature row per nonzero + one written output row per row.
double spmm_alg_bytes(i64 rows, u64 nnz, i64 d) {
  return 8.0 * nnz + 8.0 * (rows + 1) + 4.0 * nnz * d + 4.0 * rows * d;
}

// Compulsory bytes of the same launch: the sparse matrix and the output once,
// and every row of the gathered operand once (x_rows = the matrix's column
// count) — the traffic floor if L2 caught every repeated gather.
double spmm_compulsory_bytes(i64 rows, u64 nnz, i64 x_rows, i64 d) {
  return 8.0 * nnz + 8.0 * (rows + 1) + 4.0 * x_rows * d + 4.0 * rows * d;
}

// Global Glorot init (model.hpp:17-33) then this rank's block.
std::vector<float> init_weight_block(u64 seed, int l, i64 din, i64 dout, const Slice& s) {
  const double bound = std::sqrt(6.0 / static_cast<double>(din + dout));
  PhiloxStream rng(seed, 100 + static_cast<u64>(l));
  std::vector<float> blk(static_cast<size_t>((s.r1 - s.r0) * (s.c1 - s.c0)));
  for (i64 i = 0; i < din; ++i)
    for (i64 j = 0; j < dout; ++j) {
      const double u = u64_to_unit(rng.next_u64());
      const float w = static_cast<float>(-bound + (bound - -bound) * u);
      if (i >= s.r0 && i < s.r1 && j >= s.c0 && j < s.c1)
        blk[(i - s.r0) * (s.c1 - s.c0) + (j - s.c0)] = w;
    }
  return blk;
}

void upload_block(DMat& m, const float* host, i64 cols, cudaStream_t st) {
  if (m.rows == 0 || cols == 0) return;
  PK_CUDA(cudaMemcpy2DAsync(m.p(), m.ld * sizeof(float), host, cols * sizeof(float),
                            cols * sizeof(float), m.rows, cudaMemcpyHostToDevice, st));
}

}  // namespace

void DMat::alloc(i64 r, i64 c, cudaStream_t st) {
  rows = r;
  cols = c;
  ld = pad4(c);
  buf.alloc(static_cast<size_t>(std::max<i64>(1, r) * ld));
  // zero-filled (the allocator hands back reused, non-zero blocks): on the
  // engine stream that will use the block, so no host wait is needed
  PK_CUDA(cudaMemsetAsync(buf.p, 0, buf.n * sizeof(float), st));
}

const std::vector<u64>& AdjShard::blocks_nnz(int blocks, cudaStream_t st) {
  auto it = block_nnz.find(blocks);
  if (it != block_nnz.end()) return it->second;
  // block edges only: blocks + 1 row_ptr entries
  std::vector<u64> edge(blocks + 1), out;
  for (int b = 0; b <= blocks; ++b)
    PK_CUDA(cudaMemcpyAsync(&edge[b], a.row_ptr + chunk_start(a.rows, blocks, b), sizeof(u64),
                            cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  for (int b = 0; b < blocks; ++b) out.push_back(edge[b + 1] - edge[b]);
  return block_nnz[blocks] = out;
}

AdjShard::~AdjShard() {
  csr_free(&a);
  csr_free(&at);
}

// ---------------------------------------------------------------------------
// phase clock

cudaEvent_t PhaseClock::get() {
  if (used == pool.size()) {
    cudaEvent_t e;
    PK_CUDA(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[used++];
}

cudaEvent_t PhaseClock::stamp(cudaStream_t st) {
  cudaEvent_t e = get();
  PK_CUDA(cudaEventRecord(e, st));
  return e;
}

void PhaseClock::begin(int phase, cudaStream_t st) {
  if (!enabled) return;
  open_phase = phase;
  open_ev = get();
  PK_CUDA(cudaEventRecord(open_ev, st));
}

void PhaseClock::end(cudaStream_t st) {
  if (!enabled || open_phase < 0) return;
  cudaEvent_t e = get();
  PK_CUDA(cudaEventRecord(e, st));
  marks.push_back({open_phase, open_ev, e});
  open_phase = -1;
}

void PhaseClock::collect(double out[6]) {
  for (int i = 0; i < 6; ++i) out[i] = 0;
  for (auto& m : marks) {
    PK_CUDA(cudaEventSynchronize(m.b));
    float ms = 0;
    PK_CUDA(cudaEventElapsedTime(&ms, m.a, m.b));
    out[m.phase] += ms * 1e-3;
  }
  marks.clear();
  used = 0;
}

PhaseClock::~PhaseClock() {
  for (auto e : pool) cudaEventDestroy(e);
}

// ---------------------------------------------------------------------------

Engine::Engine(const pk_engine_config& cfg) : cfg_(cfg) {
  check(cfg.gx >= 1 && cfg.gy >= 1 && cfg.gz >= 1, "grid: all dimensions must be >= 1");
  check(cfg.num_layers >= 1 && cfg.num_layers <= PK_MAX_LAYERS, "engine: bad layer count");
  grid_.g[0] = cfg.gx, grid_.g[1] = cfg.gy, grid_.g[2] = cfg.gz;
  check(cfg.rank >= 0 && cfg.rank < grid_.size(), "grid: rank out of range");
  PK_CUDA(cudaSetDevice(cfg.device));
  rank_ = cfg.rank;
  c_ = grid_.coords_of(rank_);
  L_ = cfg.num_layers;
  dims_.assign(cfg.dims, cfg.dims + L_ + 1);
  for (auto d : dims_) check(d >= 1, "engine: zero layer dimension");
  lays_ = plan_layouts(L_);
  for (int l = 0; l < L_; ++l)
    shapes_.push_back(layer_shapes(grid_, lays_[l], c_, cfg.n, dims_[l], dims_[l + 1]));
  // Transform-first layers (FAST only): where the layer's inner axis is a
  // single rank and it narrows (D_out < D_in), Q = A (F W) instead of
  // (A F) W — both SpMMs of the layer then gather D_out-wide rows instead of
  // D_in-wide ones (C2's last layer: 47 instead of 256; C3's first: 128
  // instead of 602). Same products, another association: tolerance-level
  // difference, so PARITY keeps the reference's order. PK_TRANSFORM_FIRST=0
  // turns it off.
  static const bool tf_on = [] {
    const char* e = std::getenv("PK_TRANSFORM_FIRST");
    return !(e && e[0] == '0');
  }();
  tf_.assign(L_, 0);
  for (int l = 0; l < L_; ++l)
    tf_[l] = tf_on && cfg.mode == PK_MODE_FAST && grid_.extent(lays_[l].inner) == 1 &&
             dims_[l + 1] < dims_[l];
  PK_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
  PK_CUDA(cudaStreamCreateWithFlags(&cs_, cudaStreamNonBlocking));
  sums_.alloc(4);
  PK_CUDA(cudaMallocHost(&sums_host_, 4 * sizeof(double)));
}

Engine::~Engine() {
  if (st_) {
    cudaStreamSynchronize(st_);
    cudaStreamDestroy(st_);
  }
  if (cs_) {
    cudaStreamSynchronize(cs_);
    cudaStreamDestroy(cs_);
  }
  for (auto e : sync_ev_) cudaEventDestroy(e);
  if (sums_host_) cudaFreeHost(sums_host_);
  if (sums_ring_) cudaFreeHost(sums_ring_);
}

cudaEvent_t Engine::sync_event() {
  if (sync_used_ == sync_ev_.size()) {
    cudaEvent_t e;
    PK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    sync_ev_.push_back(e);
  }
  return sync_ev_[sync_used_++];
}

int Engine::comm_chunks(i64 rows, int axis) const {
  if (grid_.extent(axis) == 1) return 1;
  // Default: one chunk, i.e. the reduction follows its producer without
  // row-chunked overlap. Measured on C2 (scripts/chunk_sweep.sh): N=2
  // 48.4 / 48.4 / 49.4 / 51.6 ms and N=4 33.4 / 34.0 / 35.4 ms for 1 / 2 / 4
  // / 8 chunks — the producers (SpMM, GEMM) are HBM-bound, and a reduction
  // running beside them takes HBM bandwidth and SMs, and every extra chunk
  // adds a drain/refill of the persistent SpMM. PK_COMM_CHUNKS forces a count.
  static const int forced = [] {
    const char* e = std::getenv("PK_COMM_CHUNKS");
    return e ? std::atoi(e) : 0;
  }();
  if (forced > 0) return static_cast<int>(std::min<i64>(forced, std::max<i64>(rows, 1)));
  return 1;
}

template <typename P, typename R>
void Engine::pipelined(i64 rows, int chunks, P&& produce, R&& reduce) {
  chunks = static_cast<int>(std::max<i64>(1, std::min<i64>(chunks, std::max<i64>(rows, 1))));
  for (int c = 0; c < chunks; ++c) {
    const i64 r0 = chunk_start(rows, chunks, c), r1 = chunk_start(rows, chunks, c + 1);
    produce(r0, r1);
    cudaEvent_t ready = sync_event();
    PK_CUDA(cudaEventRecord(ready, st_));
    PK_CUDA(cudaStreamWaitEvent(cs_, ready, 0));
    cudaEvent_t a = clock_.stamp(cs_);
    reduce(r0, r1);
    clock_.add(4, a, clock_.stamp(cs_));
  }
  cudaEvent_t done = sync_event();
  PK_CUDA(cudaEventRecord(done, cs_));
  PK_CUDA(cudaStreamWaitEvent(st_, done, 0));
}

const AdjShard& Engine::shard(const Layout& l) const {
  const auto& s = shards_[l.plane() * 2 + l.parity()];
  check(s != nullptr, "no adjacency shard for plane " + std::to_string(l.plane()) +
                          " parity " + std::to_string(l.parity()));
  return *s;
}

// Transpose + SpMM plans of a freshly cut block; stored under its key.
template <typename Mark>
void Engine::finish_shard(std::shared_ptr<AdjShard> sh, int plane, int parity, Mark& mark) {
  csr_transpose(view(sh->a), &sh->at, st_);
  mark("csr_transpose");
  // FAST mode cuts hub rows into segments summed in a fixed order
  // (tolerance-level difference); PARITY keeps every row one exact chain
  const u64 seg = cfg_.mode == PK_MODE_FAST ? spmm_fast_segment() : 0;
  spmm_plan_build(sh->plan_a, view(sh->a), static_cast<u64>(cfg_.hub_threshold), st_, seg);
  spmm_plan_build(sh->plan_at, view(sh->at), static_cast<u64>(cfg_.hub_threshold), st_, seg);
  mark("spmm plans");
  sh->nnz_t = sh->at.nnz;
  // A FAST plan carries every nonzero of its matrix (packed (col, val)
  // pairs, hub rows as segments), so the CSR's columns and values are dead
  // weight from here on: 8 B per nonzero for A and again for A^T (20 GB per
  // rank at C4 scale). Only row_ptr stays (block edges). PK_KEEP_CSR=1 keeps
  // them.
  // (dropped in drop_csr_arrays() once the whole load has drained: a free
  // synchronises the device, which here would stall the staged uploads)
  shards_[plane * 2 + parity] = std::move(sh);
}

void Engine::drop_csr_arrays() {
  static const bool keep_csr = [] {
    const char* e = std::getenv("PK_KEEP_CSR");
    return e && e[0] == '1';
  }();
  if (cfg_.mode != PK_MODE_FAST || spmm_fast_segment() == 0 || keep_csr) return;
  PK_CUDA(cudaStreamSynchronize(st_));
  for (auto& sh : shards_) {
    if (!sh) continue;
    for (pk_csr_owned* m : {&sh->a, &sh->at}) {
      if (m->col_idx) dev_free(m->col_idx);
      if (m->values) dev_free(m->values);
      m->col_idx = nullptr;
      m->values = nullptr;
    }
  }
}

// F0 shard from device rows of width feature_slice's column count (ld given)
void Engine::set_f0(const float* src, i64 ld) {
  const Slice fs = feature_slice(grid_, c_, cfg_.n, dims_[0]);
  f0_.alloc(fs.r1 - fs.r0, fs.c1 - fs.c0, st_);
  if (f0_.rows && f0_.cols) {
    if (f0_.ld == f0_.cols && ld == f0_.cols)
      PK_CUDA(cudaMemcpyAsync(f0_.p(), src, f0_.rows * f0_.cols * sizeof(float),
                              cudaMemcpyDeviceToDevice, st_));
    else
      copy_block_launch(src, ld, f0_.rows, f0_.cols, f0_.p(), f0_.ld, st_);
  }
  f0_m_.alloc(f0_.rows, f0_.cols, st_);
  f0_v_.alloc(f0_.rows, f0_.cols, st_);
  df0_.alloc(f0_.rows, f0_.cols, st_);
  f0_step_ = 0;
}

// Weights (global init, then weight_slice), Adam state, activations and
// workspaces of every layer.
void Engine::alloc_params() {
  w_.resize(L_), w_m_.resize(L_), w_v_.resize(L_), dw_.resize(L_);
  wfull_.resize(L_), dwp_.resize(L_), h_.resize(L_), q_.resize(L_), fout_.resize(L_);
  i64 max_dh = 1, max_df = 1, max_tf = 0;
  for (int l = 0; l < L_; ++l) {
    const Shapes& s = shapes_[l];
    const Slice ws = weight_slice(grid_, lays_[l], c_, dims_[l], dims_[l + 1]);
    w_[l].alloc(ws.r1 - ws.r0, ws.c1 - ws.c0, st_);
    auto blk = init_weight_block(cfg_.seed, l, dims_[l], dims_[l + 1], ws);
    upload_block(w_[l], blk.data(), w_[l].cols, st_);
    PK_CUDA(cudaStreamSynchronize(st_));
    w_m_[l].alloc(w_[l].rows, w_[l].cols, st_);
    w_v_[l].alloc(w_[l].rows, w_[l].cols, st_);
    dw_[l].alloc(w_[l].rows, w_[l].cols, st_);
    wfull_[l].alloc(s.f_cols, s.w_cols, st_);
    dwp_[l].alloc(s.f_cols, s.w_cols, st_);
    if (!tf_[l]) h_[l].alloc(s.h_rows, s.h_cols, st_);  // a transform-first layer keeps no H
    else max_tf = std::max(max_tf, s.a_cols * pad4(s.w_cols));
    // a hidden layer's Q exists only where the engine materialises it (the
    // NCCL fallback of a split col_shard): allocated on first use
    if (l + 1 == L_) q_[l].alloc(s.q_rows, s.q_cols, st_);
    if (l + 1 < L_) fout_[l].alloc(s.q_rows, s.q_cols, st_);
    max_dh = std::max(max_dh, s.h_rows * pad4(s.h_cols));
    max_df = std::max(max_df, s.a_cols * pad4(s.f_cols));
  }
  w_step_ = 0;
  f0g_.alloc(shapes_[0].f_rows, shapes_[0].f_cols, st_);
  dh_.buf.alloc(max_dh);
  df_.buf.alloc(max_df);
  df_prev_.buf.alloc(max_df);
  if (max_tf) {  // P = F W forward, dP = A^T dQ backward; padding stays 0
    tfbuf_.buf.alloc(max_tf);
    PK_CUDA(cudaMemset(tfbuf_.buf.p, 0, tfbuf_.buf.n * sizeof(float)));
  }
  PK_CUDA(cudaMemset(dh_.buf.p, 0, dh_.buf.n * sizeof(float)));
  PK_CUDA(cudaMemset(df_.buf.p, 0, df_.buf.n * sizeof(float)));
  PK_CUDA(cudaMemset(df_prev_.buf.p, 0, df_prev_.buf.n * sizeof(float)));
  PK_CUDA(cudaStreamSynchronize(0));
}

// This rank's logit-row labels and mask (device pointers, lrows rows) and
// the global masked-row count the CE scaling divides by.
void Engine::set_labels(const u32* labels, const u8* mask, i64 lrows, u64 global_count) {
  const Shapes& sl = shapes_[L_ - 1];
  check(lrows == sl.a_rows, "engine: label rows disagree with the logits shard");
  labels_.alloc(std::max<i64>(1, lrows));
  mask_.alloc(std::max<i64>(1, lrows));
  if (lrows) {
    PK_CUDA(cudaMemcpyAsync(labels_.p, labels, lrows * sizeof(u32), cudaMemcpyDeviceToDevice,
                            st_));
    PK_CUDA(cudaMemcpyAsync(mask_.p, mask, lrows, cudaMemcpyDeviceToDevice, st_));
  }
  mask_count_ = global_count;
  // the gathered logits and their gather stage exist only when the classes
  // are split (inner > 1); the stage is bounded (row chunks); dlogits keeps
  // only this rank's class chunk — at C4 scale (2x2x2, s26) the three full
  // a_rows x C buffers were 69 GB per rank
  const Layout& last = lays_[L_ - 1];
  const int gi = grid_.extent(last.inner);
  if (gi > 1) {
    logits_.alloc(sl.a_rows, dims_[L_], st_);
    stage_rows_ = std::max<i64>(1, std::min<i64>(sl.a_rows, (i64{256} << 20) / 4 / dims_[L_]));
    stage_.alloc(stage_rows_, dims_[L_], st_);
  }
  dl_.alloc(sl.a_rows, chunk_size(dims_[L_], gi, c_.along(last.inner)), st_);
  // DMat::alloc zeroes on the legacy stream: drain everything before use
  PK_CUDA(cudaDeviceSynchronize());
}

void Engine::load(const pk_dataset_view& dsin, bool host) {
  PK_CUDA(cudaSetDevice(cfg_.device));
  check(dsin.n == cfg_.n, "engine load: dataset has " + std::to_string(dsin.n) +
                              " nodes but the engine was configured for " +
                              std::to_string(cfg_.n));
  check(dsin.feat_dim == dims_[0] && static_cast<i64>(dsin.num_classes) == dims_[L_],
        "engine load: dataset dims do not match the model dims");
  const i64 n = cfg_.n;
  // PK_TIMING=1: host wall time of each setup phase on stderr
  static const bool timing = std::getenv("PK_TIMING") != nullptr;
  auto t_last = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    if (!timing) return;
    PK_CUDA(cudaStreamSynchronize(st_));
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[pk load r%d] %-28s %8.2f ms\n", rank_, what,
                 std::chrono::duration<double, std::milli>(now - t_last).count());
    t_last = now;
  };
  // host inputs: stage the whole preprocessed dataset in HBM first
  pk_dataset_view ds = dsin;
  DevBuf<u64> erp, orp;
  DevBuf<u32> eci, oci, lr, lc;
  DevBuf<float> ev, ov, feat;
  DevBuf<u8> mr, mc;
  // Host inputs are staged in HBM on the (idle) comm stream in the order
  // they are consumed — even variant, odd variant, features, labels — and
  // each piece's event gates its consumer on st_, so the shards of one
  // variant are cut, transposed and planned while the next one uploads.
  cudaEvent_t staged[4] = {nullptr, nullptr, nullptr, nullptr};  // even, odd, feat, labels
  auto gate = [&](int i) {
    if (staged[i]) PK_CUDA(cudaStreamWaitEvent(st_, staged[i], 0));
  };
  if (host) {
    for (auto& e : staged) PK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    auto up = [&](auto& buf, const auto* src, size_t count) {
      buf.alloc(count ? count : 1);
      if (count)
        PK_CUDA(cudaMemcpyAsync(buf.p, src, count * sizeof(*src), cudaMemcpyHostToDevice, cs_));
      return buf.p;
    };
    ds.a_even.row_ptr = up(erp, dsin.a_even.row_ptr, n + 1);
    ds.a_even.col_idx = up(eci, dsin.a_even.col_idx, dsin.a_even.nnz);
    ds.a_even.values = up(ev, dsin.a_even.values, dsin.a_even.nnz);
    PK_CUDA(cudaEventRecord(staged[0], cs_));
    ds.a_odd.row_ptr = up(orp, dsin.a_odd.row_ptr, n + 1);
    ds.a_odd.col_idx = up(oci, dsin.a_odd.col_idx, dsin.a_odd.nnz);
    ds.a_odd.values = up(ov, dsin.a_odd.values, dsin.a_odd.nnz);
    PK_CUDA(cudaEventRecord(staged[1], cs_));
    feat.alloc(static_cast<size_t>(n * dims_[0]));
    if (dsin.ld_features == dims_[0])  // one DMA: a pitched copy moves row by row
      PK_CUDA(cudaMemcpyAsync(feat.p, dsin.features, n * dims_[0] * sizeof(float),
                              cudaMemcpyHostToDevice, cs_));
    else
      PK_CUDA(cudaMemcpy2DAsync(feat.p, dims_[0] * sizeof(float), dsin.features,
                                dsin.ld_features * sizeof(float), dims_[0] * sizeof(float), n,
                                cudaMemcpyHostToDevice, cs_));
    PK_CUDA(cudaEventRecord(staged[2], cs_));
    ds.features = feat.p;
    ds.ld_features = dims_[0];
    ds.labels_row = up(lr, dsin.labels_row, n);
    ds.labels_col = up(lc, dsin.labels_col, n);
    ds.mask_row = up(mr, dsin.mask_row, n);
    ds.mask_col = up(mc, dsin.mask_col, n);
    PK_CUDA(cudaEventRecord(staged[3], cs_));
    mark("h2d dataset");
  }
  // adjacency shards (build_adjacency_shards, engine.hpp:96-113)
  for (auto [plane, parity] : needed_adjacency_keys(L_)) {
    const pk_csr& variant = parity ? ds.a_odd : ds.a_even;
    check(variant.rows == n && variant.cols == n,
          "build_adjacency_shards: adjacency variants must be square and equal");
    gate(parity);
    const Slice r = adjacency_block_range(grid_, plane, c_, n);
    std::shared_ptr<AdjShard> same;
    for (auto& prev : shards_)
      if (prev && prev->parity == parity && prev->r0 == r.r0 && prev->r1 == r.r1 &&
          prev->c0 == r.c0 && prev->c1 == r.c1)
        same = prev;
    if (same) {
      shards_[plane * 2 + parity] = same;
      continue;
    }
    auto sh = std::make_shared<AdjShard>();
    sh->parity = parity, sh->r0 = r.r0, sh->r1 = r.r1, sh->c0 = r.c0, sh->c1 = r.c1;
    const bool whole = r.r0 == 0 && r.r1 == n && r.c0 == 0 && r.c1 == n;
    if (host && whole) {
      // the staged upload already is this block: adopt it (one rank on the
      // row and inner axes; every plane of this parity shares the shard)
      auto& rp = parity ? orp : erp;
      auto& ci = parity ? oci : eci;
      auto& va = parity ? ov : ev;
      sh->a.rows = n, sh->a.cols = n, sh->a.nnz = variant.nnz;
      sh->a.row_ptr = rp.release_ownership();
      sh->a.col_idx = ci.release_ownership();
      sh->a.values = va.release_ownership();
    } else {
      csr_block(variant, r.r0, r.r1, r.c0, r.c1, &sh->a, st_);
    }
    mark("csr_block");
    finish_shard(std::move(sh), plane, parity, mark);
  }
  // trainable features F0 (feature_slice, model.hpp:53-67) + Adam state
  const Slice fs = feature_slice(grid_, c_, n, dims_[0]);
  gate(2);
  set_f0(ds.features + fs.r0 * ds.ld_features + fs.c0, ds.ld_features);
  alloc_params();
  // labels / mask of this rank's logit rows (trainer.hpp:241-248)
  const int parity = (L_ - 1) % 2;
  const auto lr_rng = label_row_range(grid_, c_, n, L_);
  // global CE count = masked nodes over all row chunks (the label ranges of
  // the last layer's row group partition [0, n)); constant across epochs, so
  // the gradient scaling can ride in the CE kernel
  u64 count = 0;
  gate(3);
  {
    std::vector<u8> hm(n);
    PK_CUDA(cudaMemcpyAsync(hm.data(), parity ? ds.mask_col : ds.mask_row, n,
                            cudaMemcpyDeviceToHost, st_));
    PK_CUDA(cudaStreamSynchronize(st_));
    for (u8 m : hm) count += m != 0;
  }
  set_labels((parity ? ds.labels_col : ds.labels_row) + lr_rng.first,
             (parity ? ds.mask_col : ds.mask_row) + lr_rng.first,
             lr_rng.second - lr_rng.first, count);
  mark("params, activations");
  PK_CUDA(cudaStreamSynchronize(cs_));  // the staged uploads are released with this scope
  for (auto& e : staged)
    if (e) cudaEventDestroy(e);
  drop_csr_arrays();
  comm_at_load_ = comms_.counters;  // CommStats count the training only
  loaded_ = true;
}

// The file_handle path (trainer.hpp:461-466): the rank's own tensors.
void Engine::load_rank(const pk_rank_view& rv, pk_csr_owned* adopt) {
  PK_CUDA(cudaSetDevice(cfg_.device));
  const i64 n = cfg_.n;
  auto mark = [](const char*) {};
  for (auto [plane, parity] : needed_adjacency_keys(L_)) {
    const pk_csr& b = rv.adj[plane * 2 + parity];
    const Slice r = adjacency_block_range(grid_, plane, c_, n);
    check(b.rows == r.r1 - r.r0 && b.cols == r.c1 - r.c0,
          "engine load_rank: adjacency block (" + std::to_string(plane) + ", " +
              std::to_string(parity) + ") is " + std::to_string(b.rows) + "x" +
              std::to_string(b.cols) + ", expected " + std::to_string(r.r1 - r.r0) + "x" +
              std::to_string(r.c1 - r.c0));
    std::shared_ptr<AdjShard> same;
    for (auto& prev : shards_)
      if (prev && prev->parity == parity && prev->r0 == r.r0 && prev->r1 == r.r1 &&
          prev->c0 == r.c0 && prev->c1 == r.c1)
        same = prev;
    if (same) {
      shards_[plane * 2 + parity] = same;
      continue;
    }
    auto sh = std::make_shared<AdjShard>();
    sh->parity = parity, sh->r0 = r.r0, sh->r1 = r.r1, sh->c0 = r.c0, sh->c1 = r.c1;
    pk_csr_owned* own = adopt ? &adopt[plane * 2 + parity] : nullptr;
    if (own && own->row_ptr) {  // library-allocated block: taken over, no copy
      sh->a = *own;
      *own = pk_csr_owned{};
    } else {
      csr_block(b, 0, b.rows, 0, b.cols, &sh->a, st_);  // an all-columns block: a plain copy
    }
    finish_shard(std::move(sh), plane, parity, mark);
  }
  const Slice fs = feature_slice(grid_, c_, n, dims_[0]);
  check(rv.f0_rows == fs.r1 - fs.r0 && rv.f0_cols == fs.c1 - fs.c0,
        "engine load_rank: F0 shard shape disagrees with feature_slice");
  set_f0(rv.f0, rv.ld_f0);
  alloc_params();
  // global CE count: this rank's masked label rows summed over the last
  // layer's row_shard group (its label ranges partition [0, n))
  const Layout& last = lays_[L_ - 1];
  double count = 0;
  if (rv.label_rows) {
    std::vector<u8> hm(rv.label_rows);
    PK_CUDA(cudaMemcpyAsync(hm.data(), rv.mask, hm.size(), cudaMemcpyDeviceToHost, st_));
    PK_CUDA(cudaStreamSynchronize(st_));
    for (u8 m : hm) count += m != 0;
  }
  if (grid_.extent(last.row) > 1) {
    check(comms_.ready(), "engine load_rank: comm_init before loading a multi-rank grid");
    DevBuf<double> d(1);
    PK_CUDA(cudaMemcpyAsync(d.p, &count, sizeof(double), cudaMemcpyHostToDevice, st_));
    comms_.all_reduce_f64(d.p, 1, last.row, st_);
    PK_CUDA(cudaMemcpyAsync(&count, d.p, sizeof(double), cudaMemcpyDeviceToHost, st_));
    PK_CUDA(cudaStreamSynchronize(st_));
  }
  set_labels(rv.labels, rv.mask, rv.label_rows, static_cast<u64>(count));
  drop_csr_arrays();
  comm_at_load_ = comms_.counters;  // CommStats count the training only
  loaded_ = true;
}

int Engine::forward_blocks(i64 rows, const Layout& lay) const {
  if (cfg_.block_count > 0) return cfg_.block_count;
  if (grid_.extent(lay.inner) == 1) return 1;
  return static_cast<int>(std::max<i64>(1, std::min<i64>(4, rows / 65536)));
}

// The producer-fused form of an axis' ordered reduction (lsa.cuh
// slot_map / reduce_slots): FAST mode (plans without hub CTAs, the
// tensor-core GEMM epilogue) with peer-memory groups. PK_FUSED_REDUCE is a
// mask of the producers that store into the owners' slots: 1 = SpMM, 2 =
// GEMM. Measured and off by default (correct on every grid of 2 and 4,
// tests/test_multigpu_gpu.py): C2 at 2 GPUs (2x1x1) 40.6 vs 37.0 ms — the
// SpMMs' remote row stores cost 2.7 ms more SpMM time than the 0.7 ms of
// reduction they save (profiles/r2_fused_ab_trees_n2.log), and the GEMM
// epilogue's 32-B-per-thread row stores over NVLink are slower still (9.2 vs
// 2.5 ms for the forward GEMMs, profiles/r2_fused_ab_n4.log).
int Engine::fused_mask() {
  static const int m = [] {
    const char* e = std::getenv("PK_FUSED_REDUCE");
    return e ? std::atoi(e) : 0;
  }();
  return m;
}

LsaGroup* Engine::fused(int axis, int producer) const {
  if (!(fused_mask() & producer) || cfg_.mode != PK_MODE_FAST || spmm_fast_segment() == 0)
    return nullptr;
  return comms_.lsa(axis);
}

// ---------------------------------------------------------------------------
// forward_layer (engine.hpp:158-206)

void Engine::on_comm(const std::function<void(cudaStream_t)>& f) {
  // every collective runs on the comm stream, in program order, so each
  // communicator sees the same sequence on every rank
  cudaEvent_t ready = sync_event();
  PK_CUDA(cudaEventRecord(ready, st_));
  PK_CUDA(cudaStreamWaitEvent(cs_, ready, 0));
  cudaEvent_t a = clock_.stamp(cs_);
  f(cs_);
  clock_.add(4, a, clock_.stamp(cs_));
  cudaEvent_t done = sync_event();
  PK_CUDA(cudaEventRecord(done, cs_));
  PK_CUDA(cudaStreamWaitEvent(st_, done, 0));
}

void Engine::on_comm_nowait(const std::function<void(cudaStream_t)>& f) {
  cudaEvent_t ready = sync_event();
  PK_CUDA(cudaEventRecord(ready, st_));
  PK_CUDA(cudaStreamWaitEvent(cs_, ready, 0));
  cudaEvent_t a = clock_.stamp(cs_);
  f(cs_);
  clock_.add(4, a, clock_.stamp(cs_));
}

void Engine::forward_layer(int l, bool fault) {
  if (tf_[l]) return forward_layer_tf(l);
  const Layout& lay = lays_[l];
  const Shapes& s = shapes_[l];
  AdjShard& sh = const_cast<AdjShard&>(shard(lay));
  const float* f;
  i64 ldf;
  if (l == 0) {
    // layer-0 input carries the extra row_shard split: gather it
    on_comm([&](cudaStream_t cs) {
      comms_.all_gather_rows(f0_.p(), f0g_.p(), s.f_rows, f0g_.ld, lay.row, s.f_cols, cs);
    });
    f = f0g_.p();
    ldf = f0g_.ld;
  } else {
    f = fout_[l - 1].p();
    ldf = fout_[l - 1].ld;
  }
  check(sh.a.cols == s.f_rows, "forward layer " + std::to_string(l) + ": adjacency shard " +
                                   shape(sh.a.rows, sh.a.cols) + " does not match features " +
                                   shape(s.f_rows, s.f_cols));
  // W's all-gather goes out now, on the comm stream ahead of H's reduction,
  // so it runs under the SpMM instead of between the reduction and the GEMM
  // (the GEMM waits for the reduction, which follows it in stream order)
  on_comm_nowait([&](cudaStream_t cs) {
    comms_.all_gather_rows(w_[l].p(), wfull_[l].p(), s.f_cols, wfull_[l].ld, lay.row, s.w_cols,
                           cs);
  });
  DMat& h = h_[l];
  // blocked aggregation (engine.hpp:175-192): SpMM row block b, then its
  // all-reduce along inner — overlapped with block b+1's SpMM
  // fused: the SpMM stores each row straight into its owner's slot (one
  // block — the transfer already overlaps the SpMM)
  LsaGroup* fu_h = fault ? nullptr : fused(lay.inner, kFuseSpmm);
  RowMap map_h;
  if (fu_h) map_h = fu_h->slot_map(sh.a.rows, h.ld);
  const int blocks = fu_h ? 1 : forward_blocks(sh.a.rows, lay);
  const std::vector<u64>& bnnz = sh.blocks_nnz(blocks, st_);
  int b = 0;
  // partials go to the axis' symmetric scratch when the ordered peer-memory
  // reduction is available (fault_epoch skips the reduction altogether: the
  // reference's negative control, engine.hpp:186)
  LsaGroup* lsa_h = fault ? nullptr : comms_.lsa(lay.inner);
  float* hpart = lsa_h ? lsa_h->scratch() : h.p();
  pipelined(
      sh.a.rows, blocks,
      [&](i64 r0, i64 r1) {
        clock_.begin(0, st_);
        spmm_run(sh.plan_a, view(sh.a), r0, r1, f, ldf, s.f_cols, hpart + r0 * h.ld, h.ld, st_,
                 nullptr, 0, fu_h ? &map_h : nullptr);
        spmm_flops_ += 2 * bnnz[b] * static_cast<u64>(s.f_cols);
        spmm_bytes_ += spmm_alg_bytes(r1 - r0, bnnz[b], s.f_cols);
        spmm_cbytes_ += spmm_compulsory_bytes(r1 - r0, bnnz[b], b == 0 ? sh.a.cols : 0, s.f_cols);
        ++b;
        clock_.end(st_);
      },
      [&](i64 r0, i64 r1) {
        if (fault) return;
        if (fu_h) {
          fu_h->reduce_slots(sh.a.rows, s.f_cols, h.ld, h.p(), h.ld, cs_);
          comms_.count(kAllReduce, lay.inner, (r1 - r0) * s.f_cols * 4);
        } else if (lsa_h) {
          lsa_h->all_reduce(r0, r1, s.f_cols, h.ld, h.p(), r0, h.ld, cs_);
          comms_.count(kAllReduce, lay.inner, (r1 - r0) * s.f_cols * 4);
        } else {
          comms_.all_reduce(h.p() + r0 * h.ld, (r1 - r0) * h.ld, lay.inner,
                            (r1 - r0) * s.f_cols * 4, cs_);
        }
      });
  // Q = H . W_full, then its all-reduce along col_shard, row-chunked. Hidden
  // layers store only relu(Q) (the next layer's input and, since
  // relu(Q) > 0 <=> Q > 0, the backward's ReLU mask): the activation is
  // fused into the GEMM epilogue when col_shard is a single rank, else into
  // the ordered peer reduction; only the NCCL fallback materialises Q.
  const bool hidden = l + 1 < L_;
  const bool col_single = comms_.size(lay.col) == 1;
  LsaGroup* lsa_q = comms_.lsa(lay.col);
  // measurement mode stands in for the peer-memory path: relu in place
  // where the ordered reduction would have fused it
  const bool solo = comms_.solo();
  DMat& qout = hidden && (col_single || lsa_q || solo) ? fout_[l] : q_[l];
  if (qout.buf.p == nullptr) qout.alloc(s.q_rows, s.q_cols, st_);
  float* qpart = lsa_q ? lsa_q->scratch() : qout.p();
  // fused when the epilogue stores each row once (k <= 512: one TMEM segment)
  LsaGroup* fu_q = s.h_cols <= 512 ? fused(lay.col, kFuseGemm) : nullptr;
  RowMap map_q;
  if (fu_q) map_q = fu_q->slot_map(s.h_rows, qout.ld);
  pipelined(
      s.h_rows, fu_q ? 1 : comm_chunks(s.h_rows, lay.col),
      [&](i64 r0, i64 r1) {
        clock_.begin(1, st_);
        gemm_launch(false, false, r1 - r0, s.w_cols, s.h_cols, h.p() + r0 * h.ld, h.ld,
                    wfull_[l].p(), wfull_[l].ld, qpart + r0 * qout.ld, qout.ld, cfg_.mode, st_,
                    hidden && col_single, fu_q ? &map_q : nullptr);
        clock_.end(st_);
      },
      [&](i64 r0, i64 r1) {
        if (fu_q) {
          fu_q->reduce_slots(s.h_rows, s.q_cols, qout.ld, qout.p(), qout.ld, cs_, hidden);
          comms_.count(kAllReduce, lay.col, (r1 - r0) * s.q_cols * 4);
        } else if (lsa_q) {
          lsa_q->all_reduce(r0, r1, s.q_cols, qout.ld, qout.p(), r0, qout.ld, cs_, hidden);
          comms_.count(kAllReduce, lay.col, (r1 - r0) * s.q_cols * 4);
        } else {
          comms_.all_reduce(qout.p() + r0 * qout.ld, (r1 - r0) * qout.ld, lay.col,
                            (r1 - r0) * s.q_cols * 4, cs_);
          if (solo && hidden && !col_single)
            relu_forward_launch(qout.p() + r0 * qout.ld, qout.ld, r1 - r0, s.q_cols,
                                qout.p() + r0 * qout.ld, qout.ld, cs_);
        }
      });
  gemm_flops_ += 2 * static_cast<u64>(s.h_rows) * s.w_cols * s.h_cols;
  if (hidden) {
    if (q_kept_.size() < static_cast<size_t>(L_)) q_kept_.assign(L_, 0);
    q_kept_[l] = &qout == &q_[l];
  }
  if (hidden && &qout == &q_[l]) {
    clock_.begin(1, st_);
    relu_forward_launch(q_[l].p(), q_[l].ld, s.q_rows, s.q_cols, fout_[l].p(), fout_[l].ld, st_);
    clock_.end(st_);
  }
}

// ---------------------------------------------------------------------------
// loss (trainer.hpp:498-516)

void Engine::loss() {
  const Layout& last = lays_[L_ - 1];
  const Shapes& s = shapes_[L_ - 1];
  const i64 C = dims_[L_];
  // logits: the column gather along inner (trainer.hpp:499); with a single
  // member the local Q block already is the full logits matrix
  const float* logits = q_[L_ - 1].p();
  i64 ldl = q_[L_ - 1].ld;
  if (comms_.size(last.inner) > 1) {
    on_comm([&](cudaStream_t cs) {
      comms_.all_gather_cols(q_[L_ - 1].p(), q_[L_ - 1].ld, logits_.p(), logits_.ld, s.a_rows,
                             C, last.inner, stage_.p(), stage_rows_, cs);
    });
    logits = logits_.p();
    ldl = logits_.ld;
  } else {
    comms_.counters.calls[last.inner][kAllGather]++;  // the reference still counts the call
  }
  clock_.begin(2, st_);
  const int gi = comms_.size(last.inner), pi = c_.along(last.inner);
  ce_sums_launch(logits, ldl, s.a_rows, C, labels_.p, mask_.p, dl_.p(), dl_.ld, sums_.p, ce_ws_,
                 st_, mask_count_, chunk_start(C, gi, pi), chunk_start(C, gi, pi + 1));
  clock_.end(st_);
  on_comm([&](cudaStream_t cs) { comms_.all_reduce_f64(sums_.p, 3, last.row, cs); });
  // no host wait here: the sums ride to pinned memory in stream order and
  // finish_pass() checks them after the epoch (the gradient scaling uses the
  // load-time mask count, so the backward does not need them)
  double* dst = sums_dst_ ? sums_dst_ : sums_host_;
  PK_CUDA(cudaMemcpyAsync(dst, sums_.p, 3 * sizeof(double), cudaMemcpyDeviceToHost, st_));
  PK_CUDA(cudaMemcpyAsync(reinterpret_cast<u32*>(dst + 3), ce_ws_.bad.p, sizeof(u32),
                          cudaMemcpyDeviceToHost, st_));
}

// finalize_loss (trainer.hpp:71-89) and the pass's error checks; the stream
// has drained.
// the checks every pass ends with (the stream has drained): a failed peer
// (its ClusterAborted, not our partial sums), a timed-out peer reduction,
// a device watchdog
void Engine::check_after_pass() {
  comms_.check_alive();
  if (lsa_ready_ && grid_.size() > 1 && lsa_timed_out())
    throw Error(PK_ERR_NCCL, "peer-memory reduction: a barrier wait timed out (peer stalled)");
  check_device_watchdogs();
}

void Engine::finish_pass(int epoch, double* loss_out, double* acc_out, const double* slot) {
  check_after_pass();
  const i64 C = dims_[L_];
  const double* sums = slot ? slot : sums_host_;
  const u32 bad = *reinterpret_cast<const u32*>(sums + 3);
  check(!bad, "cross entropy: label out of range for " + std::to_string(C) + " classes");
  const double* h = sums;
  const u64 count = static_cast<u64>(h[1]), correct = static_cast<u64>(h[2]);
  if (count == 0 && comms_.solo()) {  // measurement mode: this rank holds no loss rows
    if (loss_out) *loss_out = 0;
    if (acc_out) *acc_out = 0;
    return;
  }
  if (count == 0)
    throw Error(PK_ERR_TRAINING,
                "epoch " + std::to_string(epoch) + ": no nodes selected by the training mask");
  const double loss = h[0] / static_cast<double>(count);
  if (!std::isfinite(loss))
    throw Error(PK_ERR_TRAINING, "epoch " + std::to_string(epoch) + ": loss is not finite (" +
                                     std::to_string(loss) + ")");
  if (loss_out) *loss_out = loss;
  if (acc_out) *acc_out = static_cast<double>(correct) / static_cast<double>(count);
  // (measurement mode counts only this rank's rows)
  check(comms_.solo() || count == mask_count_, "cross entropy: counted " + std::to_string(count) +
                                  " masked rows, expected " + std::to_string(mask_count_));
}

// ---------------------------------------------------------------------------
// backward_layer (engine.hpp:214-259)

void Engine::backward_layer(int l) {
  if (tf_[l]) return backward_layer_tf(l);
  const Layout& lay = lays_[l];
  const Shapes& s = shapes_[l];
  AdjShard& sh = const_cast<AdjShard&>(shard(lay));
  const bool is_last = l == L_ - 1;
  // dQ: the loss gradient's own class chunk on the last layer (a strided
  // view of dlogits: no copy), relu'(Q) * dF otherwise
  const float* dq;
  i64 lddq;
  clock_.begin(2, st_);
  if (is_last) {  // dlogits holds exactly this rank's class chunk
    dq = dl_.p();
    lddq = dl_.ld;
  } else if (df_masked_) {
    // relu_backward already applied by the SpMM^T / reduction that made dF
    lddq = pad4(s.q_cols);
    dq = df_prev_.p();
  } else {
    lddq = pad4(s.q_cols);
    // relu'(Q) from the stored activation: relu(Q) > 0 exactly where Q > 0;
    // in place — dF_out is dead once dQ exists (no separate dQ workspace)
    relu_backward_launch(fout_[l].p(), fout_[l].ld, df_prev_.p(), pad4(s.q_cols), s.q_rows,
                         s.q_cols, df_prev_.p(), lddq, st_);
    dq = df_prev_.p();
  }
  // dW = (dQ^T H)^T computed as H^T dQ: same products, same k order
  LsaGroup* lsa_dw = comms_.lsa(lay.row);
  float* dwpart = lsa_dw ? lsa_dw->scratch() : dwp_[l].p();
  auto dw_gemm = [&]() {
    gemm_launch(true, false, s.h_cols, s.q_cols, s.h_rows, h_[l].p(), h_[l].ld, dq, lddq, dwpart,
                dwp_[l].ld, cfg_.mode, st_);
    gemm_flops_ += 2 * static_cast<u64>(s.h_cols) * s.q_cols * s.h_rows;
  };
  auto dw_comm = [&](cudaStream_t cs) {
    if (lsa_dw) {  // reduce-scatter (engine.hpp:237): this member sums its own rows
      const int g = grid_.extent(lay.row), pos = c_.along(lay.row);
      const i64 o0 = chunk_start(s.f_cols, g, pos), o1 = chunk_start(s.f_cols, g, pos + 1);
      lsa_dw->reduce(o0, o1, s.w_cols, dwp_[l].ld, dw_[l].p(), 0, dw_[l].ld, cs);
      comms_.count(kReduceScatter, lay.row, s.f_cols * s.w_cols * 4);
    } else {
      comms_.reduce_scatter_rows(dwp_[l].p(), dw_[l].p(), s.f_cols, dwp_[l].ld, lay.row,
                                 s.w_cols, cs);
    }
    comms_.all_gather_rows(w_[l].p(), wfull_[l].p(), s.f_cols, wfull_[l].ld, lay.row, s.w_cols,
                           cs);
  };
  // dH = dQ . W_full^T, then its all-reduce along inner, row-chunked
  const i64 lddh = pad4(s.h_cols);
  LsaGroup* lsa_dh = comms_.lsa(lay.inner);
  float* dhpart = lsa_dh ? lsa_dh->scratch() : dh_.p();
  LsaGroup* fu_dh = s.q_cols <= 512 ? fused(lay.inner, kFuseGemm) : nullptr;
  RowMap map_dh;
  if (fu_dh) map_dh = fu_dh->slot_map(s.q_rows, lddh);
  auto dh_gemm = [&](i64 r0, i64 r1) {
    clock_.begin(2, st_);
    gemm_launch(false, true, r1 - r0, s.h_cols, s.q_cols, dq + r0 * lddq, lddq, wfull_[l].p(),
                wfull_[l].ld, dhpart + r0 * lddh, lddh, cfg_.mode, st_, false,
                fu_dh ? &map_dh : nullptr);
    clock_.end(st_);
  };
  auto dh_reduce = [&](i64 r0, i64 r1) {
    if (fu_dh) {
      fu_dh->reduce_slots(s.q_rows, s.h_cols, lddh, dh_.p(), lddh, cs_);
      comms_.count(kAllReduce, lay.inner, (r1 - r0) * s.h_cols * 4);
    } else if (lsa_dh) {
      lsa_dh->all_reduce(r0, r1, s.h_cols, lddh, dh_.p(), r0, lddh, cs_);
      comms_.count(kAllReduce, lay.inner, (r1 - r0) * s.h_cols * 4);
    } else {
      comms_.all_reduce(dh_.p() + r0 * lddh, (r1 - r0) * lddh, lay.inner,
                        (r1 - r0) * s.h_cols * 4, cs_);
    }
  };
  // Order: when dH is reduced along a split inner axis, its GEMM goes first
  // and the dW GEMM runs while dH crosses NVLink (the dW reduce-scatter and
  // the W re-gather follow on the comm stream); otherwise the reference's
  // order, with the dW reduce-scatter under the dH GEMM. PK_BWD_DH_FIRST=0
  // keeps the reference's order everywhere.
  static const bool dh_first_on = [] {
    const char* e = std::getenv("PK_BWD_DH_FIRST");
    return !(e && e[0] == '0');
  }();
  const bool dh_first = dh_first_on && comms_.size(lay.inner) > 1 && !fu_dh &&
                        comm_chunks(s.q_rows, lay.inner) == 1;
  cudaEvent_t bwd_comm_done = nullptr;
  if (dh_first) {
    clock_.end(st_);  // the dQ phase
    dh_gemm(0, s.q_rows);
    cudaEvent_t ready = sync_event();
    PK_CUDA(cudaEventRecord(ready, st_));
    PK_CUDA(cudaStreamWaitEvent(cs_, ready, 0));
    cudaEvent_t c0 = clock_.stamp(cs_);
    dh_reduce(0, s.q_rows);
    clock_.add(4, c0, clock_.stamp(cs_));
    cudaEvent_t dh_done = sync_event();
    PK_CUDA(cudaEventRecord(dh_done, cs_));
    clock_.begin(2, st_);
    dw_gemm();
    clock_.end(st_);
    cudaEvent_t dw_ready = sync_event();
    PK_CUDA(cudaEventRecord(dw_ready, st_));
    PK_CUDA(cudaStreamWaitEvent(cs_, dw_ready, 0));
    cudaEvent_t c1 = clock_.stamp(cs_);
    dw_comm(cs_);
    clock_.add(4, c1, clock_.stamp(cs_));
    bwd_comm_done = sync_event();
    PK_CUDA(cudaEventRecord(bwd_comm_done, cs_));
    PK_CUDA(cudaStreamWaitEvent(st_, dh_done, 0));
    // the dF partial below overwrites the row axis' scratch the dW
    // reduce-scatter reads: then it waits for that too
    if (lsa_dw) {
      PK_CUDA(cudaStreamWaitEvent(st_, bwd_comm_done, 0));
      bwd_comm_done = nullptr;
    }
  } else {
    dw_gemm();
    clock_.end(st_);
    on_comm(dw_comm);
    pipelined(s.q_rows, fu_dh ? 1 : comm_chunks(s.q_rows, lay.inner), dh_gemm, dh_reduce);
  }
  gemm_flops_ += 2 * static_cast<u64>(s.q_rows) * s.h_cols * s.q_cols;
  // dF = A^T . dH, then reduce-scatter (layer 0) or all-reduce along
  // row_shard, row-chunked
  const i64 lddf = pad4(s.f_cols);
  LsaGroup* lsa_df = comms_.lsa(lay.row);
  float* dfpart = lsa_df ? lsa_df->scratch() : df_.p();
  const int gr = grid_.extent(lay.row), pr = c_.along(lay.row);
  const i64 own0 = chunk_start(s.a_cols, gr, pr), own1 = chunk_start(s.a_cols, gr, pr + 1);
  // layer l-1's relu_backward rides on the ordered dF reduction when
  // row_shard is split (the reduction is NVLink-bound; the mask read is
  // free there). Inside the SpMM^T epilogue it is measured slower than the
  // separate streaming pass (C2 1x1x1: 67.3 vs 65.6 ms per epoch — the mask
  // reads compete with the gathers), so that variant is opt-in.
  // PK_FUSE_RELU_BWD: 0 = never, 1 = reduction only (default), 2 = also SpMM^T.
  static const int fuse = [] {
    const char* e = std::getenv("PK_FUSE_RELU_BWD");
    return e ? std::atoi(e) : 1;
  }();
  const DMat* act = l > 0 && fuse > 0 ? &fout_[l - 1] : nullptr;
  const bool mask_spmm = act && gr == 1 && fuse >= 2;
  const bool mask_reduce = act && gr > 1 && lsa_df;
  LsaGroup* fu_df = fused(lay.row, kFuseSpmm);
  RowMap map_df;
  if (fu_df) map_df = fu_df->slot_map(sh.at.rows, lddf);
  pipelined(
      sh.at.rows, fu_df ? 1 : comm_chunks(sh.at.rows, lay.row),
      [&](i64 r0, i64 r1) {
        clock_.begin(5, st_);
        spmm_run(sh.plan_at, view(sh.at), r0, r1, dh_.p(), lddh, s.f_cols, dfpart + r0 * lddf,
                 lddf, st_, mask_spmm ? act->p() + r0 * act->ld : nullptr,
                 mask_spmm ? act->ld : 0, fu_df ? &map_df : nullptr);
        clock_.end(st_);
      },
      [&](i64 r0, i64 r1) {
        if (fu_df) {
          if (l == 0) {  // reduce-scatter: the owner keeps its own rows only
            fu_df->reduce_slots(sh.at.rows, s.f_cols, lddf, df0_.p(), df0_.ld, cs_, false,
                                nullptr, 0, true);
            comms_.count(kReduceScatter, lay.row, (r1 - r0) * s.f_cols * 4);
          } else {
            fu_df->reduce_slots(sh.at.rows, s.f_cols, lddf, df_.p(), lddf, cs_, false,
                                mask_reduce ? act->p() : nullptr, mask_reduce ? act->ld : 0);
            comms_.count(kAllReduce, lay.row, (r1 - r0) * s.f_cols * 4);
          }
        } else if (lsa_df) {
          if (l == 0) {  // reduce-scatter: this member sums only its own rows
            const i64 a = std::max(r0, own0), b = std::min(r1, own1);
            lsa_df->reduce(a, std::max(a, b), s.f_cols, lddf, df0_.p(), a - own0, df0_.ld, cs_);
            comms_.count(kReduceScatter, lay.row, (r1 - r0) * s.f_cols * 4);
          } else {
            lsa_df->all_reduce(r0, r1, s.f_cols, lddf, df_.p(), r0, lddf, cs_, false,
                           mask_reduce ? act->p() : nullptr, mask_reduce ? act->ld : 0);
            comms_.count(kAllReduce, lay.row, (r1 - r0) * s.f_cols * 4);
          }
        } else if (l == 0) {
          comms_.reduce_scatter_rows_range(df_.p(), df0_.p(), s.a_cols, lddf, lay.row, s.f_cols,
                                           r0, r1, cs_);
        } else {
          comms_.all_reduce(df_.p() + r0 * lddf, (r1 - r0) * lddf, lay.row,
                            (r1 - r0) * s.f_cols * 4, cs_);
        }
      });
  spmm_flops_ += 2 * sh.nnz_t * static_cast<u64>(s.f_cols);
  spmm_bytes_ += spmm_alg_bytes(sh.at.rows, sh.nnz_t, s.f_cols);
  spmm_cbytes_ += spmm_compulsory_bytes(sh.at.rows, sh.nnz_t, sh.at.cols, s.f_cols);
  if (l > 0) std::swap(df_.buf, df_prev_.buf);  // becomes dF_out of layer l-1
  df_masked_ = mask_spmm || mask_reduce;
  if (bwd_comm_done) PK_CUDA(cudaStreamWaitEvent(st_, bwd_comm_done, 0));
}

// ---------------------------------------------------------------------------
// transform-first layers (inner axis a single rank, D_out < D_in; FAST)
//
// forward:  P = F W_full  (a_cols x w_cols, partial over col_shard: its
//           all-reduce replaces Q's), Q = A P (complete: inner is one rank)
// backward: dP = A^T dQ (partial over row_shard: all-reduced, replacing
//           dF's), dW = F^T dP restricted to this rank's stored rows (no
//           reduce-scatter: dP is complete and F holds every row), dF = dP
//           W_full^T (complete; at layer 0 only this rank's F0 rows)
// The fault hook (skip the aggregation all-reduce) has nothing to skip here:
// inner is a single rank.

int Engine::tf_vec() {
  static const int v = [] {
    const char* e = std::getenv("PK_TF_VEC");
    return e ? std::atoi(e) : 2;
  }();
  return v;
}

// PK_TF_PAIR=1: the narrow SpMMs in the paired form (two nonzeros per warp
// gather, spmm_pair_kernel). Measured neutral on C2 (3.69-3.73 vs 3.69 ms
// per 48-wide pass, 5.7 GB DRAM either way: the pass is bound by random
// 192-B DRAM reads, not by gather instructions), so the list kernel —
// bit-identical to PARITY on regular rows — stays the default.
bool Engine::tf_pair() {
  static const bool v = [] {
    const char* e = std::getenv("PK_TF_PAIR");
    return e && e[0] == '1';
  }();
  return v;
}

void Engine::forward_layer_tf(int l) {
  const Layout& lay = lays_[l];
  const Shapes& s = shapes_[l];
  AdjShard& sh = const_cast<AdjShard&>(shard(lay));
  const float* f;
  i64 ldf;
  if (l == 0) {
    on_comm([&](cudaStream_t cs) {
      comms_.all_gather_rows(f0_.p(), f0g_.p(), s.f_rows, f0g_.ld, lay.row, s.f_cols, cs);
    });
    f = f0g_.p();
    ldf = f0g_.ld;
  } else {
    f = fout_[l - 1].p();
    ldf = fout_[l - 1].ld;
  }
  check(sh.a.cols == s.f_rows, "forward layer " + std::to_string(l) + ": adjacency shard " +
                                   shape(sh.a.rows, sh.a.cols) + " does not match features " +
                                   shape(s.f_rows, s.f_cols));
  comms_.counters.calls[lay.inner][kAllReduce]++;  // the singleton H all-reduce
  on_comm([&](cudaStream_t cs) {
    comms_.all_gather_rows(w_[l].p(), wfull_[l].p(), s.f_cols, wfull_[l].ld, lay.row, s.w_cols,
                           cs);
  });
  const i64 ldp = pad4(s.w_cols);
  LsaGroup* lsa_p = comms_.lsa(lay.col);
  float* ppart = lsa_p ? lsa_p->scratch() : tfbuf_.p();
  LsaGroup* fu_p = s.f_cols <= 512 ? fused(lay.col, kFuseGemm) : nullptr;
  RowMap map_p;
  if (fu_p) map_p = fu_p->slot_map(s.f_rows, ldp);
  clock_.begin(1, st_);
  gemm_launch(false, false, s.f_rows, s.w_cols, s.f_cols, f, ldf, wfull_[l].p(), wfull_[l].ld,
              ppart, ldp, cfg_.mode, st_, false, fu_p ? &map_p : nullptr);
  clock_.end(st_);
  gemm_flops_ += 2 * static_cast<u64>(s.f_rows) * s.w_cols * s.f_cols;
  if (comms_.size(lay.col) > 1) {
    on_comm([&](cudaStream_t cs) {
      if (fu_p) {
        fu_p->reduce_slots(s.f_rows, s.w_cols, ldp, tfbuf_.p(), ldp, cs);
        comms_.count(kAllReduce, lay.col, s.f_rows * s.w_cols * 4);
      } else if (lsa_p) {
        lsa_p->all_reduce(0, s.f_rows, s.w_cols, ldp, tfbuf_.p(), 0, ldp, cs);
        comms_.count(kAllReduce, lay.col, s.f_rows * s.w_cols * 4);
      } else {
        comms_.all_reduce(tfbuf_.p(), s.f_rows * ldp, lay.col, s.f_rows * s.w_cols * 4, cs);
      }
    });
  } else {
    comms_.counters.calls[lay.col][kAllReduce]++;
  }
  const bool hidden = l + 1 < L_;
  DMat& qout = hidden ? fout_[l] : q_[l];
  clock_.begin(0, st_);
  // Width of the narrow SpMMs (PK_TF_VEC): 0 = the exact width (47: 32
  // lanes x 2 of 4-B gathers); v > 0 = the padded width (48; P's and dQ's
  // padding columns are zero, so the extra output column is exactly +0)
  // with gathers of at most v floats. Default 2: 24 lanes of 8-B gathers,
  // C2 epoch 52.2 vs 52.8 ms; at 16 B the padded width takes the 16-lane
  // group form, measured slower (2 x 5.6 vs 2 x 3.9 ms per C2 epoch).
  // (a width that is a multiple of 4 needs no padding and keeps 16-B and
  // wider gathers: C3's 128)
  const int tfv = s.w_cols % 4 ? tf_vec() : 0;
  spmm_run(sh.plan_a, view(sh.a), 0, sh.a.rows, tfbuf_.p(), ldp, tfv ? ldp : s.w_cols,
           qout.p(), qout.ld, st_, nullptr, 0, nullptr, tfv ? tfv : 8, tf_pair());
  spmm_flops_ += 2 * sh.a.nnz * static_cast<u64>(s.w_cols);
  spmm_bytes_ += spmm_alg_bytes(sh.a.rows, sh.a.nnz, s.w_cols);
  spmm_cbytes_ += spmm_compulsory_bytes(sh.a.rows, sh.a.nnz, sh.a.cols, s.w_cols);
  if (hidden) relu_forward_launch(qout.p(), qout.ld, s.q_rows, s.q_cols, qout.p(), qout.ld, st_);
  clock_.end(st_);
  if (hidden) {
    if (q_kept_.size() < static_cast<size_t>(L_)) q_kept_.assign(L_, 0);
    q_kept_[l] = 0;
  }
}

void Engine::backward_layer_tf(int l) {
  const Layout& lay = lays_[l];
  const Shapes& s = shapes_[l];
  AdjShard& sh = const_cast<AdjShard&>(shard(lay));
  const bool is_last = l == L_ - 1;
  const float* dq;
  i64 lddq;
  clock_.begin(2, st_);
  if (is_last) {  // inner is one rank: dlogits holds every class
    dq = dl_.p();
    lddq = dl_.ld;
  } else {
    lddq = pad4(s.q_cols);
    if (!df_masked_)
      relu_backward_launch(fout_[l].p(), fout_[l].ld, df_prev_.p(), lddq, s.q_rows, s.q_cols,
                           df_prev_.p(), lddq, st_);
    dq = df_prev_.p();
  }
  clock_.end(st_);
  const i64 ldp = pad4(s.w_cols);
  LsaGroup* lsa_r = comms_.lsa(lay.row);
  float* dpp = lsa_r ? lsa_r->scratch() : tfbuf_.p();
  LsaGroup* fu_r = fused(lay.row, kFuseSpmm);
  RowMap map_r;
  if (fu_r) map_r = fu_r->slot_map(sh.at.rows, ldp);
  clock_.begin(5, st_);
  const int tfv = s.w_cols % 4 ? tf_vec() : 0;
  spmm_run(sh.plan_at, view(sh.at), 0, sh.at.rows, dq, lddq, tfv ? ldp : s.w_cols, dpp, ldp, st_,
           nullptr, 0, fu_r ? &map_r : nullptr, tfv ? tfv : 8, tf_pair());
  clock_.end(st_);
  spmm_flops_ += 2 * sh.nnz_t * static_cast<u64>(s.w_cols);
  spmm_bytes_ += spmm_alg_bytes(sh.at.rows, sh.nnz_t, s.w_cols);
  spmm_cbytes_ += spmm_compulsory_bytes(sh.at.rows, sh.nnz_t, sh.at.cols, s.w_cols);
  const int gr = grid_.extent(lay.row), pr = c_.along(lay.row);
  if (gr > 1) {
    on_comm([&](cudaStream_t cs) {
      if (fu_r) {
        fu_r->reduce_slots(s.a_cols, s.w_cols, ldp, tfbuf_.p(), ldp, cs);
        comms_.count(kAllReduce, lay.row, s.a_cols * s.w_cols * 4);
      } else if (lsa_r) {
        lsa_r->all_reduce(0, s.a_cols, s.w_cols, ldp, tfbuf_.p(), 0, ldp, cs);
        comms_.count(kAllReduce, lay.row, s.a_cols * s.w_cols * 4);
      } else {
        comms_.all_reduce(tfbuf_.p(), s.a_cols * ldp, lay.row, s.a_cols * s.w_cols * 4, cs);
      }
    });
  } else {
    comms_.counters.calls[lay.row][kAllReduce]++;
  }
  const float* dp = tfbuf_.p();
  const float* f = l == 0 ? f0g_.p() : fout_[l - 1].p();
  const i64 ldf = l == 0 ? f0g_.ld : fout_[l - 1].ld;
  clock_.begin(2, st_);
  // dW: this rank's stored rows of W (weight_slice: the f_cols chunk split
  // again by row_shard) = F[:, o0:o1]^T dP over all a_cols rows
  const i64 o0 = chunk_start(s.f_cols, gr, pr), o1 = chunk_start(s.f_cols, gr, pr + 1);
  gemm_launch(true, false, o1 - o0, s.w_cols, s.f_rows, f + o0, ldf, dp, ldp, dw_[l].p(),
              dw_[l].ld, cfg_.mode, st_);
  gemm_flops_ += 2 * static_cast<u64>(o1 - o0) * s.w_cols * s.f_rows;
  bool masked = false;
  if (l > 0) {
    const i64 lddf = pad4(s.f_cols);
    // dF is complete here (no reduction follows), so layer l-1's relu'
    // (kernels.hpp:103-111, mask relu(Q_{l-1}) = this layer's F) can ride
    // the GEMM epilogue instead of a separate pass over dF (bit-identical;
    // PK_GEMM_RELU_BWD=0: the separate pass). With the mask rows read as
    // 256-bit loads in the TMA-store epilogue: C2 50.28 / 50.40 vs 50.38 /
    // 50.55 ms (scalar mask loads were slower: 52.4 vs 50.5)
    static const bool fuse_mask = [] {
      const char* e = std::getenv("PK_GEMM_RELU_BWD");
      return !(e && e[0] == '0');
    }();
    masked = fuse_mask;
    gemm_launch(false, true, s.f_rows, s.f_cols, s.w_cols, dp, ldp, wfull_[l].p(), wfull_[l].ld,
                df_.p(), lddf, cfg_.mode, st_, false, nullptr, masked ? f : nullptr,
                masked ? ldf : 0);
    gemm_flops_ += 2 * static_cast<u64>(s.f_rows) * s.f_cols * s.w_cols;
    std::swap(df_.buf, df_prev_.buf);  // becomes dF_out of layer l-1
  } else {
    // this rank's F0 rows: the row_shard chunk of the gathered input rows
    const i64 own0 = chunk_start(s.a_cols, gr, pr), own1 = chunk_start(s.a_cols, gr, pr + 1);
    gemm_launch(false, true, own1 - own0, s.f_cols, s.w_cols, dp + own0 * ldp, ldp,
                wfull_[l].p(), wfull_[l].ld, df0_.p(), df0_.ld, cfg_.mode, st_);
    gemm_flops_ += 2 * static_cast<u64>(own1 - own0) * s.f_cols * s.w_cols;
  }
  clock_.end(st_);
  df_masked_ = masked;
}

// Symmetric scratch for the ordered peer-memory reductions: per axis the
// largest partial it reduces (H and dH along inner, Q along col_shard, dF
// along row_shard). Collective; every member of a group computes the same
// sizes (the reduced dimensions do not depend on the member's coordinate
// along that axis).
void Engine::setup_lsa() {
  size_t need[3] = {0, 0, 0};
  for (int l = 0; l < L_; ++l) {
    const Layout& lay = lays_[l];
    const Shapes& s = shapes_[l];
    auto grow = [&](int axis, size_t e) { need[axis] = std::max(need[axis], e); };
    grow(lay.inner, static_cast<size_t>(s.a_rows) * h_[l].ld);
    grow(lay.inner, static_cast<size_t>(s.q_rows) * pad4(s.h_cols));
    grow(lay.col, static_cast<size_t>(s.h_rows) * pad4(s.q_cols));
    grow(lay.row, static_cast<size_t>(s.a_cols) * pad4(s.f_cols));
    grow(lay.row, static_cast<size_t>(s.f_cols) * dwp_[l].ld);
    if (tf_[l]) {  // P along col_shard, dP along row_shard
      grow(lay.col, static_cast<size_t>(s.a_cols) * pad4(s.w_cols));
      grow(lay.row, static_cast<size_t>(s.a_cols) * pad4(s.w_cols));
    }
  }
  for (int a = 0; a < 3; ++a)
    if (need[a] && grid_.extent(a) > 1) {
      // the fused form needs the owner slots (g x ceil(rows / g) rows) and a
      // result region of all rows: ~2x the partial, plus the ceil slack
      const size_t e = fused_mask() && cfg_.mode == PK_MODE_FAST
                           ? 2 * need[a] + (size_t{1} << 16) : need[a];
      comms_.lsa(a, e);
    }
  lsa_ready_ = true;
}

void Engine::begin_pass() {
  check(loaded_, "engine: no dataset loaded");
  check(comms_.ready(), "engine: communicators not initialised");
  PK_CUDA(cudaSetDevice(cfg_.device));
  sync_used_ = 0;
  if (!lsa_ready_) setup_lsa();
}

void Engine::forward_backward(int epoch) {
  const bool fault = epoch == cfg_.fault_epoch;
  begin_pass();
  for (int l = 0; l < L_; ++l) forward_layer(l, fault);
  loss();
  for (int l = L_ - 1; l >= 0; --l) backward_layer(l);
}

void Engine::optimizer_step() {
  clock_.begin(3, st_);
  ++w_step_;
  const AdamScalars sw = adam_scalars(w_step_, cfg_.lr, cfg_.beta1, cfg_.beta2, cfg_.eps);
  for (int l = 0; l < L_; ++l)
    adam_launch(w_[l].p(), dw_[l].p(), w_m_[l].p(), w_v_[l].p(), w_[l].elems(), sw, st_);
  ++f0_step_;
  const AdamScalars sf = adam_scalars(f0_step_, cfg_.lr, cfg_.beta1, cfg_.beta2, cfg_.eps);
  adam_launch(f0_.p(), df0_.p(), f0_m_.p(), f0_v_.p(), f0_.elems(), sf, st_);
  clock_.end(st_);
}

void Engine::train_epoch(int epoch, pk_epoch_metrics* m) {
  CommCounters before = comms_.counters;
  const u64 sf0 = spmm_flops_, gf0 = gemm_flops_;
  const double sb0 = spmm_bytes_, cb0 = spmm_cbytes_;
  const u64 launches0 = launch_count();
  clock_.reset();  // marks of earlier forward_backward / optimizer_step calls
  cudaEvent_t e0 = clock_.get(), e1 = clock_.get();
  PK_CUDA(cudaEventRecord(e0, st_));
  double loss = 0, acc = 0;
  forward_backward(epoch);
  optimizer_step();
  PK_CUDA(cudaEventRecord(e1, st_));
  PK_CUDA(cudaEventSynchronize(e1));
  // the one host wait of the epoch; the checks of the pass follow it (the
  // reference raises TrainingError before its Adam step, trainer.hpp:74-83 —
  // here the step already ran on the device, and the error still names the
  // epoch and ends training)
  finish_pass(epoch, &loss, &acc);
  float ms = 0;
  PK_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  double ph[6];
  clock_.collect(ph);
  if (!m) return;
  std::memset(m, 0, sizeof(*m));
  m->epoch = epoch;
  m->loss = loss;
  m->accuracy = acc;
  m->forward_spmm_s = ph[0];
  m->forward_gemm_s = ph[1];
  m->backward_s = ph[2] + ph[5];
  m->spmm_s = ph[0] + ph[5];
  m->spmm_bytes = spmm_bytes_ - sb0;
  m->spmm_compulsory_bytes = spmm_cbytes_ - cb0;
  m->kernel_launches = launch_count() - launches0;
  m->optimizer_s = ph[3];
  m->collectives_s = ph[4];
  m->epoch_s = ms * 1e-3;
  m->spmm_flops = spmm_flops_ - sf0;
  m->gemm_flops = gemm_flops_ - gf0;
  for (int a = 0; a < 3; ++a) {
    const double g = grid_.extent(a);
    auto delta = [&](int op) {
      return static_cast<double>(comms_.counters.ring_numer[a][op] - before.ring_numer[a][op]) / g;
    };
    m->allreduce_bytes += delta(kAllReduce);
    m->allgather_bytes += delta(kAllGather);
    m->reducescatter_bytes += delta(kReduceScatter);
  }
}

void Engine::comm_stats(u64* calls9, double* bytes9) const {
  for (int a = 0; a < 3; ++a)
    for (int o = 0; o < 3; ++o) {
      const u64 c = comms_.counters.calls[a][o] - comm_at_load_.calls[a][o];
      const u64 r = comms_.counters.ring_numer[a][o] - comm_at_load_.ring_numer[a][o];
      if (calls9) calls9[a * 3 + o] = c;
      if (bytes9) bytes9[a * 3 + o] = static_cast<double>(r) / grid_.extent(a);
    }
}

void Engine::on_failure(const std::string& why) {
  if (LocalCluster* cl = comms_.local_cluster()) cl->abort(rank_, why);
  else comms_.signal_abort(rank_, why);
}

// `count` epochs enqueued back to back with one host wait at the end: the
// host runs ahead of the device (no per-epoch sync bubble), each epoch's CE
// sums land in their own pinned slot, and the checks / metrics of every
// epoch follow the wait in epoch order (the first failing epoch raises, as
// train_epoch would have).
void Engine::train_epochs(int first, int count, pk_epoch_metrics* out) {
  check(count >= 1, "train_epochs: count must be >= 1");
  if (sums_ring_n_ < count) {
    if (sums_ring_) cudaFreeHost(sums_ring_);
    PK_CUDA(cudaMallocHost(&sums_ring_, sizeof(double) * 4 * count));
    sums_ring_n_ = count;
  }
  clock_.reset();
  struct Snap {
    CommCounters c;
    u64 sf, gf, launches;
    double sb, cb;
    size_t mark0;
    cudaEvent_t e0, e1;
  };
  std::vector<Snap> snaps(count);
  for (int i = 0; i < count; ++i) {
    Snap& sn = snaps[i];
    sn.c = comms_.counters, sn.sf = spmm_flops_, sn.gf = gemm_flops_;
    sn.sb = spmm_bytes_, sn.cb = spmm_cbytes_, sn.launches = launch_count();
    sn.e0 = clock_.get();
    sn.e1 = clock_.get();
    sn.mark0 = clock_.marks.size();
    PK_CUDA(cudaEventRecord(sn.e0, st_));
    sums_dst_ = sums_ring_ + 4 * i;
    forward_backward(first + i);
    optimizer_step();
    PK_CUDA(cudaEventRecord(sn.e1, st_));
  }
  sums_dst_ = nullptr;
  const u64 sf_end = spmm_flops_, gf_end = gemm_flops_, l_end = launch_count();
  const double sb_end = spmm_bytes_, cb_end = spmm_cbytes_;
  const CommCounters c_end = comms_.counters;
  PK_CUDA(cudaEventSynchronize(snaps[count - 1].e1));
  for (int i = 0; i < count; ++i) {
    const Snap& sn = snaps[i];
    double loss = 0, acc = 0;
    finish_pass(first + i, &loss, &acc, sums_ring_ + 4 * i);
    double ph[6] = {0, 0, 0, 0, 0, 0};
    const size_t mark1 = i + 1 < count ? snaps[i + 1].mark0 : clock_.marks.size();
    for (size_t k = sn.mark0; k < mark1; ++k) {
      float t = 0;
      PK_CUDA(cudaEventElapsedTime(&t, clock_.marks[k].a, clock_.marks[k].b));
      ph[clock_.marks[k].phase] += t * 1e-3;
    }
    float ms = 0;
    PK_CUDA(cudaEventElapsedTime(&ms, sn.e0, sn.e1));
    const bool last = i + 1 == count;
    const Snap* nx = last ? nullptr : &snaps[i + 1];
    pk_epoch_metrics* m = out + i;
    std::memset(m, 0, sizeof(*m));
    m->epoch = first + i;
    m->loss = loss;
    m->accuracy = acc;
    m->forward_spmm_s = ph[0];
    m->forward_gemm_s = ph[1];
    m->backward_s = ph[2] + ph[5];
    m->spmm_s = ph[0] + ph[5];
    m->optimizer_s = ph[3];
    m->collectives_s = ph[4];
    m->epoch_s = ms * 1e-3;
    m->spmm_bytes = (last ? sb_end : nx->sb) - sn.sb;
    m->spmm_compulsory_bytes = (last ? cb_end : nx->cb) - sn.cb;
    m->kernel_launches = (last ? l_end : nx->launches) - sn.launches;
    m->spmm_flops = (last ? sf_end : nx->sf) - sn.sf;
    m->gemm_flops = (last ? gf_end : nx->gf) - sn.gf;
    const CommCounters& ce = last ? c_end : nx->c;
    for (int a = 0; a < 3; ++a) {
      const double g = grid_.extent(a);
      auto delta = [&](int op) {
        return static_cast<double>(ce.ring_numer[a][op] - sn.c.ring_numer[a][op]) / g;
      };
      m->allreduce_bytes += delta(kAllReduce);
      m->allgather_bytes += delta(kAllGather);
      m->reducescatter_bytes += delta(kReduceScatter);
    }
  }
  clock_.reset();
}

bool Engine::tensor(int which, int layer, pk_tensor_view* out) {
  auto fill = [&](const DMat& m, i64 cols) {
    out->data = m.p();
    out->rows = m.rows;
    out->cols = cols;
    out->ld = m.ld;
    return true;
  };
  const bool lay_ok = layer >= 0 && layer < L_;
  switch (which) {
    case PK_T_W: return lay_ok && fill(w_[layer], w_[layer].cols);
    case PK_T_DW: return lay_ok && fill(dw_[layer], dw_[layer].cols);
    case PK_T_F0: return fill(f0_, f0_.cols);
    case PK_T_DF0: return fill(df0_, df0_.cols);
    case PK_T_FOUT: return fill(q_[L_ - 1], q_[L_ - 1].cols);
    case PK_T_H: return lay_ok && fill(h_[layer], h_[layer].cols);
    case PK_T_Q:
      return lay_ok && (layer == L_ - 1 || (layer < static_cast<int>(q_kept_.size()) &&
                                            q_kept_[layer])) &&
             fill(q_[layer], q_[layer].cols);
    case PK_T_ACT: return lay_ok && layer + 1 < L_ && fill(fout_[layer], fout_[layer].cols);
    default: return false;
  }
}

}  // namespace pk

// ---------------------------------------------------------------------------
// C ABI

struct pk_engine {
  std::unique_ptr<pk::Engine> e;
};

struct pk_cluster {
  std::unique_ptr<pk::LocalCluster> c;
};

using namespace pk;

namespace {
// Entry points that run the rank's collective program: a failure here is a
// rank failure and aborts the rank's cluster (ClusterAborted on the peers).
template <typename F>
int guard_rank(pk_engine* e, F&& f) {
  const int rc = guard(std::forward<F>(f));
  if (rc != PK_OK && rc != PK_ERR_ABORTED && e && e->e) {
    try {
      e->e->on_failure(pk_last_error());
    } catch (...) {
    }
  }
  return rc;
}
}  // namespace

extern "C" {

int pk_nccl_unique_id(void* out128) {
  return guard([&] {
    ncclUniqueId id;
    PK_NCCL(ncclGetUniqueId(&id));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

int pk_engine_create(const pk_engine_config* cfg, pk_engine** out) {
  return guard([&] {
    check(cfg != nullptr && out != nullptr, "engine: null argument");
    auto* h = new pk_engine;
    try {
      h->e = std::make_unique<Engine>(*cfg);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int pk_engine_comm_init(pk_engine* e, const void* uid, int world_size) {
  return guard([&] { e->e->comm_init(uid, world_size); });
}

int pk_cluster_create(int gx, int gy, int gz, pk_cluster** out) {
  return guard([&] {
    check(out != nullptr, "cluster: null argument");
    Grid g;
    g.g[0] = gx, g.g[1] = gy, g.g[2] = gz;
    check(gx >= 1 && gy >= 1 && gz >= 1, "grid: all dimensions must be >= 1");
    auto* h = new pk_cluster;
    h->c = std::make_unique<LocalCluster>(g);
    *out = h;
  });
}

int pk_cluster_abort(pk_cluster* c, int rank, const char* why) {
  return guard([&] { c->c->abort(rank, why ? why : "aborted by the host"); });
}

int pk_cluster_aborted(pk_cluster* c, int* aborted) {
  return guard([&] { *aborted = c->c->aborted() ? 1 : 0; });
}

int pk_cluster_destroy(pk_cluster* c) {
  return guard([&] { delete c; });
}

int pk_engine_comm_init_local(pk_engine* e, pk_cluster* c) {
  return guard([&] {
    check(e && c, "comm init: null argument");
    e->e->comm_init_local(c->c.get());
  });
}

int pk_engine_comm_init_solo(pk_engine* e) {
  return guard([&] { e->e->comm_init_solo(); });
}

int pk_engine_load(pk_engine* e, const pk_dataset_view* ds) {
  return guard_rank(e, [&] { e->e->load(*ds, false); });
}

int pk_engine_load_host(pk_engine* e, const pk_dataset_view* ds) {
  return guard_rank(e, [&] { e->e->load(*ds, true); });
}

int pk_engine_load_rank(pk_engine* e, const pk_rank_view* rv) {
  return guard_rank(e, [&] {
    check(e && rv, "engine load_rank: null argument");
    e->e->load_rank(*rv, nullptr);
  });
}

int pk_engine_load_rank_adopt(pk_engine* e, const pk_rank_view* rv, pk_csr_owned* blocks) {
  return guard_rank(e, [&] {
    check(e && rv && blocks, "engine load_rank: null argument");
    e->e->load_rank(*rv, blocks);
  });
}

int pk_engine_forward_backward(pk_engine* e, int epoch, double* loss, double* acc) {
  return guard_rank(e, [&] {
    e->e->reset_clock();  // phase marks are only collected by train_epoch
    e->e->forward_backward(epoch);
    PK_CUDA(cudaStreamSynchronize(e->e->stream()));
    e->e->finish_pass(epoch, loss, acc);
  });
}

int pk_engine_forward_only(pk_engine* e) {
  return guard_rank(e, [&] {
    e->e->reset_clock();
    e->e->begin_pass();
    for (int l = 0; l < e->e->num_layers(); ++l) e->e->layer_forward(l, false);
    PK_CUDA(cudaStreamSynchronize(e->e->stream()));
    e->e->check_after_pass();
  });
}

int pk_engine_begin_pass(pk_engine* e) {
  return guard_rank(e, [&] {
    e->e->reset_clock();
    e->e->begin_pass();
  });
}

int pk_engine_forward_layer(pk_engine* e, int layer, int fault) {
  return guard_rank(e, [&] {
    check(layer >= 0 && layer < e->e->num_layers(), "engine: layer out of range");
    e->e->layer_forward(layer, fault != 0);
  });
}

int pk_engine_loss(pk_engine* e) {
  return guard_rank(e, [&] { e->e->pass_loss(); });
}

int pk_engine_backward_layer(pk_engine* e, int layer) {
  return guard_rank(e, [&] {
    check(layer >= 0 && layer < e->e->num_layers(), "engine: layer out of range");
    e->e->layer_backward(layer);
  });
}

int pk_engine_finish_pass(pk_engine* e, int epoch, double* loss, double* acc) {
  return guard_rank(e, [&] {
    PK_CUDA(cudaStreamSynchronize(e->e->stream()));
    e->e->finish_pass(epoch, loss, acc);
  });
}

// RankCtx collectives (cluster.hpp:265-340) on this rank's axis groups.
int pk_engine_all_reduce_f32(pk_engine* e, int axis, float* buf, int64_t rows, int64_t cols,
                             int64_t ld, void* stream) {
  return guard_rank(e, [&] {
    check(axis >= 0 && axis < 3, "all_reduce: axis out of range");
    check(rows >= 0 && cols >= 0 && ld >= cols, "all_reduce: bad shape");
    e->e->comms().all_reduce(buf, rows * ld, axis, rows * cols * 4, as_stream(stream));
  });
}

int pk_engine_all_gather_f32(pk_engine* e, int axis, int concat_cols, const float* local,
                             int64_t local_ld, float* out, int64_t out_rows, int64_t out_cols,
                             int64_t out_ld, void* stream) {
  return guard_rank(e, [&] {
    check(axis >= 0 && axis < 3, "all_gather: axis out of range");
    Comms& c = e->e->comms();
    const int g = c.size(axis);
    if (concat_cols) {
      DevBuf<float> stage(static_cast<size_t>(std::max<i64>(1, out_rows * out_cols)));
      c.all_gather_cols(local, local_ld, out, out_ld, out_rows, out_cols, axis, stage.p, 0,
                        as_stream(stream));
      PK_CUDA(cudaStreamSynchronize(as_stream(stream)));  // stage dies here
    } else {
      check(local_ld == out_ld, "all_gather: rows are concatenated with one row stride");
      (void)g;
      c.all_gather_rows(local, out, out_rows, out_ld, axis, out_cols, as_stream(stream));
    }
  });
}

int pk_engine_reduce_scatter_f32(pk_engine* e, int axis, float* buf, int64_t rows, int64_t cols,
                                 int64_t ld, float* out, void* stream) {
  return guard_rank(e, [&] {
    check(axis >= 0 && axis < 3, "reduce_scatter: axis out of range");
    e->e->comms().reduce_scatter_rows(buf, out, rows, ld, axis, cols, as_stream(stream));
  });
}

int pk_engine_optimizer_step(pk_engine* e) {
  return guard_rank(e, [&] {
    e->e->reset_clock();
    e->e->optimizer_step();
  });
}

int pk_engine_train_epochs(pk_engine* e, int first_epoch, int count, pk_epoch_metrics* out) {
  return guard_rank(e, [&] {
    check(out != nullptr, "train_epochs: null metrics array");
    e->e->train_epochs(first_epoch, count, out);
  });
}

int pk_engine_train_epoch(pk_engine* e, int epoch, pk_epoch_metrics* m) {
  return guard_rank(e, [&] { e->e->train_epoch(epoch, m); });
}

int pk_engine_comm_stats(pk_engine* e, uint64_t* calls9, double* ring_bytes9) {
  return guard([&] { e->e->comm_stats(calls9, ring_bytes9); });
}

int pk_engine_abort(pk_engine* e, const char* why) {
  return guard([&] { e->e->on_failure(why ? why : "aborted by the host"); });
}

int pk_engine_tensor(pk_engine* e, int which, int layer, pk_tensor_view* out) {
  return guard([&] {
    PK_CUDA(cudaStreamSynchronize(e->e->stream()));
    check(e->e->tensor(which, layer, out), "engine tensor: unknown tensor or layer");
  });
}

int pk_engine_stream(pk_engine* e, void** s) {
  return guard([&] { *s = e->e->stream(); });
}

int pk_engine_destroy(pk_engine* e) {
  return guard([&] { delete e; });
}

}  // extern "C"
