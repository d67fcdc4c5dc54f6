// extern "C" entry points of libplexus_b200.so (include/plexus_b200.h).
// Each validates shapes with the reference's error wording, then launches.
#include <cuda_runtime.h>

#include <atomic>
#include <string>

#include "elementwise.cuh"
#include "gemm.cuh"
#include "philox.cuh"
#include "pk_common.cuh"
#include "shard_builder.cuh"
#include "spmm.cuh"

namespace pk {

namespace {
thread_local std::string g_last_error;
}

void set_last_error(const std::string& msg) { g_last_error = msg; }

namespace {
std::atomic<u64> g_launches{0};
}
u64 count_launch() { return g_launches.fetch_add(1, std::memory_order_relaxed) + 1; }
u64 launch_count() { return g_launches.load(std::memory_order_relaxed); }

void check_device_watchdogs() {
  if (const unsigned s = spmm_watchdog())
    throw Error(PK_ERR_CUDA, "spmm: hub pipeline watchdog fired " + std::to_string(s) +
                                 " time(s); results are incomplete");
  if (const unsigned g = gemm_watchdog())
    throw Error(PK_ERR_CUDA, "gemm_tc: pipeline watchdog fired " + std::to_string(g) +
                                 " time(s); results are incomplete");
}

SideStream& side_stream() {
  struct Holder {
    SideStream s;
    int device = -1;
    ~Holder() {
      // streams die with the context at process exit; nothing to do
    }
  };
  static thread_local Holder h;
  int dev = 0;
  PK_CUDA(cudaGetDevice(&dev));
  if (h.s.stream == nullptr || h.device != dev) {
    PK_CUDA(cudaStreamCreateWithFlags(&h.s.stream, cudaStreamNonBlocking));
    PK_CUDA(cudaEventCreateWithFlags(&h.s.fork, cudaEventDisableTiming));
    PK_CUDA(cudaEventCreateWithFlags(&h.s.join, cudaEventDisableTiming));
    h.device = dev;
  }
  return h.s;
}

namespace {

void check_csr(const pk_csr* a, const char* who) {
  check(a != nullptr, std::string(who) + ": null matrix");
  check(a->rows >= 0 && a->cols >= 0, std::string(who) + ": negative shape");
  check(a->rows == 0 || a->row_ptr != nullptr, std::string(who) + ": null row_ptr");
}

std::string csr_shape(const pk_csr* a) { return shape(a->rows, a->cols); }

u64 nnz_of_rows(const pk_csr* a, i64 r0, i64 r1, cudaStream_t st) {
  if (r0 == r1) return 0;
  u64 b = 0, e = 0;
  PK_CUDA(cudaMemcpyAsync(&b, a->row_ptr + r0, sizeof(u64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaMemcpyAsync(&e, a->row_ptr + r1, sizeof(u64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  return e - b;
}

void spmm_common(const pk_csr* a, i64 r0, i64 r1, const float* x, i64 x_rows, i64 ldx, i64 d,
                 float* y, i64 ldy, u64* flops, cudaStream_t st, SpmmPlan* plan,
                 const char* who, const float* mask = nullptr, i64 ldm = 0,
                 bool paired = false) {
  check_csr(a, who);
  check(a->cols == x_rows, std::string(who) + ": A is " + csr_shape(a) + " but X is " +
                               shape(x_rows, d));
  check(r0 >= 0 && r0 <= r1 && r1 <= a->rows, std::string(who) + ": row range out of bounds");
  check(d >= 0 && ldx >= d && ldy >= d, std::string(who) + ": leading dimension smaller than width");
  check(!mask || ldm >= d, std::string(who) + ": mask leading dimension smaller than width");
  if (plan) {
    spmm_run(*plan, *a, r0, r1, x, ldx, d, y, ldy, st, mask, ldm, nullptr, 8, paired);
  } else {
    // a one-off call builds a throwaway plan (the engine keeps one per shard)
    SpmmPlan tmp;
    spmm_plan_build(tmp, *a, 0, st);
    spmm_run(tmp, *a, r0, r1, x, ldx, d, y, ldy, st, mask, ldm);
    PK_CUDA(cudaStreamSynchronize(st));
  }
  if (flops) *flops += 2 * nnz_of_rows(a, r0, r1, st) * static_cast<u64>(d);
}

}  // namespace
}  // namespace pk

struct pk_spmm_plan {
  pk::SpmmPlan plan;
};

using namespace pk;

extern "C" {

const char* pk_last_error(void) { return g_last_error.c_str(); }

int pk_abi_version(void) { return 2; }  // 2: pk_epoch_metrics.spmm_compulsory_bytes, clusters, per-layer calls

uint64_t pk_kernel_launch_count(void) { return g_launches.load(); }

int pk_device_watchdogs(uint32_t* spmm, uint32_t* gemm) {
  return guard([&] {
    if (spmm) *spmm = spmm_watchdog();
    if (gemm) *gemm = gemm_watchdog();
  });
}

int pk_device_cache_release(void) {
  return guard([&] { dev_trim(); });
}

int pk_device_sm_count(int device) {
  int n = 0;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return n;
}

int pk_spmm_rows_f32(const pk_csr* a, int64_t r0, int64_t r1, const float* x, int64_t x_rows,
                     int64_t ldx, int64_t d, float* y, int64_t ldy, uint64_t* flops_host,
                     void* stream) {
  return guard([&] {
    spmm_common(a, r0, r1, x, x_rows, ldx, d, y, ldy, flops_host, as_stream(stream), nullptr,
                "spmm_rows");
  });
}

int pk_spmm_f32(const pk_csr* a, const float* x, int64_t x_rows, int64_t ldx, int64_t d,
                float* y, int64_t ldy, uint64_t* flops_host, void* stream) {
  return guard([&] {
    check(a != nullptr, "spmm: null matrix");
    spmm_common(a, 0, a->rows, x, x_rows, ldx, d, y, ldy, flops_host, as_stream(stream),
                nullptr, "spmm");
  });
}

int pk_spmm_plan_create(const pk_csr* a, int64_t hub_threshold, void* stream,
                        pk_spmm_plan** out) {
  return guard([&] {
    check_csr(a, "spmm plan");
    auto* p = new pk_spmm_plan;
    try {
      spmm_plan_build(p->plan, *a, static_cast<u64>(hub_threshold), as_stream(stream));
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

int pk_spmm_plan_create_mode(const pk_csr* a, int64_t hub_threshold, int mode, void* stream,
                             pk_spmm_plan** out) {
  return guard([&] {
    check_csr(a, "spmm plan");
    check(mode == PK_MODE_PARITY || mode == PK_MODE_FAST, "spmm plan: unknown mode");
    auto* p = new pk_spmm_plan;
    try {
      spmm_plan_build(p->plan, *a, static_cast<u64>(hub_threshold), as_stream(stream),
                      mode == PK_MODE_FAST ? spmm_fast_segment() : 0);
    } catch (...) {
      delete p;
      throw;
    }
    *out = p;
  });
}

int pk_spmm_plan_destroy(pk_spmm_plan* plan) {
  return guard([&] { delete plan; });
}

int pk_spmm_plan_rows_f32(const pk_spmm_plan* plan, const pk_csr* a, int64_t r0, int64_t r1,
                          const float* x, int64_t x_rows, int64_t ldx, int64_t d, float* y,
                          int64_t ldy, uint64_t* flops_host, void* stream) {
  return guard([&] {
    check(plan != nullptr, "spmm plan: null plan");
    check(a != nullptr && plan->plan.rows == a->rows, "spmm plan: plan built for another matrix");
    spmm_common(a, r0, r1, x, x_rows, ldx, d, y, ldy, flops_host, as_stream(stream),
                const_cast<SpmmPlan*>(&plan->plan), "spmm_rows");
  });
}

int pk_spmm_plan_rows_relu_bwd_f32(const pk_spmm_plan* plan, const pk_csr* a, int64_t r0,
                                   int64_t r1, const float* x, int64_t x_rows, int64_t ldx,
                                   int64_t d, const float* mask, int64_t ldm, float* y,
                                   int64_t ldy, uint64_t* flops_host, void* stream) {
  return guard([&] {
    check(plan != nullptr, "spmm plan: null plan");
    check(a != nullptr && plan->plan.rows == a->rows, "spmm plan: plan built for another matrix");
    check(mask != nullptr, "spmm relu_backward: null mask");
    spmm_common(a, r0, r1, x, x_rows, ldx, d, y, ldy, flops_host, as_stream(stream),
                const_cast<SpmmPlan*>(&plan->plan), "spmm_rows_relu_backward", mask, ldm);
  });
}

int pk_spmm_plan_rows_ex_f32(const pk_spmm_plan* plan, const pk_csr* a, int64_t r0, int64_t r1,
                             const float* x, int64_t x_rows, int64_t ldx, int64_t d, float* y,
                             int64_t ldy, int flags, uint64_t* flops_host, void* stream) {
  return guard([&] {
    check(plan != nullptr, "spmm plan: null plan");
    check(a != nullptr && plan->plan.rows == a->rows, "spmm plan: plan built for another matrix");
    check((flags & ~PK_SPMM_PAIRED) == 0, "spmm_rows_ex: unknown flags");
    check(!(flags & PK_SPMM_PAIRED) || plan->plan.segment,
          "spmm_rows_ex: PK_SPMM_PAIRED needs a PK_MODE_FAST plan");
    spmm_common(a, r0, r1, x, x_rows, ldx, d, y, ldy, flops_host, as_stream(stream),
                const_cast<SpmmPlan*>(&plan->plan), "spmm_rows_ex", nullptr, 0,
                (flags & PK_SPMM_PAIRED) != 0);
  });
}

int pk_spmm_plan_info(const pk_spmm_plan* plan, int64_t* hub_rows, int64_t* hub_threshold) {
  return guard([&] {
    check(plan != nullptr, "spmm plan: null plan");
    if (hub_rows) *hub_rows = plan->plan.hub_count;
    if (hub_threshold) *hub_threshold = static_cast<int64_t>(plan->plan.threshold);
  });
}

namespace {
int gemm_entry(int ta, int tb, int64_t m, int64_t n, int64_t k, const float* a, int64_t lda,
               const float* b, int64_t ldb, float* c, int64_t ldc, int mode,
               uint64_t* flops_host, void* stream, bool relu) {
  return guard([&] {
    check(m >= 0 && n >= 0 && k >= 0, "gemm: negative dimension");
    check(mode == PK_MODE_PARITY || mode == PK_MODE_FAST, "gemm: unknown mode");
    check(lda >= (ta ? m : k) && ldb >= (tb ? k : n) && ldc >= n,
          "gemm: leading dimension smaller than the stored width");
    gemm_launch(ta != 0, tb != 0, m, n, k, a, lda, b, ldb, c, ldc, mode, as_stream(stream),
                relu);
    if (flops_host) *flops_host += 2 * static_cast<u64>(m) * n * k;
  });
}

}  // namespace

int pk_gemm_f32(int ta, int tb, int64_t m, int64_t n, int64_t k, const float* a, int64_t lda,
                const float* b, int64_t ldb, float* c, int64_t ldc, int mode,
                uint64_t* flops_host, void* stream) {
  return gemm_entry(ta, tb, m, n, k, a, lda, b, ldb, c, ldc, mode, flops_host, stream, false);
}

int pk_gemm_relu_f32(int ta, int tb, int64_t m, int64_t n, int64_t k, const float* a,
                     int64_t lda, const float* b, int64_t ldb, float* c, int64_t ldc, int mode,
                     uint64_t* flops_host, void* stream) {
  return gemm_entry(ta, tb, m, n, k, a, lda, b, ldb, c, ldc, mode, flops_host, stream, true);
}

int pk_relu_forward_f32(const float* q, int64_t ldq, int64_t rows, int64_t cols, float* out,
                        int64_t ldo, void* stream) {
  return guard([&] {
    check(rows >= 0 && cols >= 0 && ldq >= cols && ldo >= cols, "relu_forward: bad shape");
    relu_forward_launch(q, ldq, rows, cols, out, ldo, as_stream(stream));
  });
}

int pk_relu_backward_f32(const float* q, int64_t ldq, const float* df, int64_t lddf,
                         int64_t rows, int64_t cols, float* out, int64_t ldo, void* stream) {
  return guard([&] {
    check(rows >= 0 && cols >= 0 && ldq >= cols && lddf >= cols && ldo >= cols,
          "relu_backward: Q is " + shape(rows, cols) + " but dF leading dimension is " +
              std::to_string(lddf));
    relu_backward_launch(q, ldq, df, lddf, rows, cols, out, ldo, as_stream(stream));
  });
}

int pk_softmax_ce_sums_f32(const float* logits, int64_t ldl, int64_t rows, int64_t classes,
                           const uint32_t* labels, const uint8_t* mask, float* dlogits,
                           int64_t ldd, double* sums_dev, void* stream) {
  return guard([&] {
    check(rows >= 0 && classes >= 0 && ldl >= classes && ldd >= classes,
          "cross entropy: bad shape");
    static thread_local CeWorkspace ws;
    auto st = as_stream(stream);
    ce_sums_launch(logits, ldl, rows, classes, labels, mask, dlogits, ldd, sums_dev, ws, st);
    u32 bad = 0;
    PK_CUDA(cudaMemcpyAsync(&bad, ws.bad.p, sizeof(u32), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    check(!bad, "cross entropy: label out of range for " + std::to_string(classes) + " classes");
  });
}

int pk_scale_by_count_f32(float* d, int64_t ldd, int64_t rows, int64_t cols,
                          const double* sums_dev, void* stream) {
  return guard([&] {
    check(rows >= 0 && cols >= 0 && ldd >= cols, "scale: bad shape");
    scale_by_count_launch(d, ldd, rows, cols, sums_dev, as_stream(stream));
  });
}

int pk_adam_step_f32(float* param, const float* grad, float* m, float* v, int64_t n,
                     uint64_t step, double lr, double beta1, double beta2, double eps,
                     void* stream) {
  return guard([&] {
    check(n >= 0 && step >= 1, "adam_step: step must be >= 1");
    adam_launch(param, grad, m, v, n, adam_scalars(step, lr, beta1, beta2, eps),
                as_stream(stream));
  });
}

int pk_csr_transpose(const pk_csr* a, pk_csr_owned* out, void* stream) {
  return guard([&] {
    check_csr(a, "csr transpose");
    csr_transpose(*a, out, as_stream(stream));
  });
}

int pk_csr_block(const pk_csr* a, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                 pk_csr_owned* out, void* stream) {
  return guard([&] {
    check_csr(a, "csr block");
    csr_block(*a, r0, r1, c0, c1, out, as_stream(stream));
  });
}

int pk_csr_hconcat(const pk_csr* pieces, const uint64_t* col0, int count, uint64_t c0,
                   uint64_t c1, pk_csr_owned* out, void* stream) {
  return guard([&] {
    check(pieces && col0 && out, "csr hconcat: null argument");
    for (int k = 0; k < count; ++k) check_csr(&pieces[k], "csr hconcat");
    csr_hconcat(pieces, col0, count, c0, c1, out, as_stream(stream));
  });
}

int pk_normalize_adjacency(int64_t n, const uint32_t* edges_uv, uint64_t num_edges,
                           int undirected, pk_csr_owned* out, void* stream) {
  return guard([&] {
    normalize_adjacency(n, edges_uv, num_edges, undirected != 0, out, as_stream(stream));
  });
}

int pk_permute_csr(const pk_csr* a, const uint32_t* row_perm, const uint32_t* col_perm,
                   pk_csr_owned* out, void* stream) {
  return guard([&] {
    check_csr(a, "permute_csr");
    permute_csr(*a, row_perm, col_perm, out, as_stream(stream));
  });
}

void pk_csr_free(pk_csr_owned* m) { csr_free(m); }

int pk_permutation_pair_host(uint64_t n, uint64_t seed, uint32_t* row_perm_host,
                             uint32_t* col_perm_host) {
  return guard([&] {
    check(n >= 1, "generate_permutation_pair: n must be >= 1");
    // rng.hpp:57-66 Fisher-Yates, streams 1 (rows) and 2 (columns)
    auto shuffle = [&](u64 stream, u32* p) {
      PhiloxStream rng(seed, stream);
      for (u64 i = 0; i < n; ++i) p[i] = static_cast<u32>(i);
      for (u64 i = n; i > 1; --i) {
        const u64 j = rng.randint(i);
        const u32 t = p[i - 1];
        p[i - 1] = p[j];
        p[j] = t;
      }
    };
    shuffle(1, row_perm_host);
    shuffle(2, col_perm_host);
  });
}

int pk_philox_permutation_host(uint64_t n, uint64_t seed, uint64_t stream, uint32_t* out) {
  return guard([&] {
    // Philox::permutation (rng.hpp:57-66): identity, then Fisher-Yates from
    // the top with rejection-sampled randint
    PhiloxStream rng(seed, stream);
    for (u64 i = 0; i < n; ++i) out[i] = static_cast<u32>(i);
    for (u64 i = n; i > 1; --i) std::swap(out[i - 1], out[rng.randint(i)]);
  });
}

int pk_rmat_edges(int scale, uint64_t edges, double a, double b, double c, uint64_t seed,
                  uint32_t* edges_uv, uint64_t* kept_host, void* stream) {
  return guard([&] {
    *kept_host = rmat_edges(scale, edges, a, b, c, seed, edges_uv, as_stream(stream));
  });
}

int pk_sbm_edges(uint64_t n, int communities, double p_in, double p_out, uint64_t seed,
                 uint32_t* edges_uv, uint64_t capacity, uint64_t* count_host, void* stream) {
  return guard([&] {
    check(count_host != nullptr, "sbm: null count");
    *count_host = pair_edges(n, communities, p_in, p_out, seed, edges_uv, capacity,
                             as_stream(stream));
  });
}

int pk_erdos_edges(uint64_t n, double p, uint64_t seed, uint32_t* edges_uv, uint64_t capacity,
                   uint64_t* count_host, void* stream) {
  return guard([&] {
    check(count_host != nullptr, "erdos: null count");
    check(n >= 1, "erdos: n must be >= 1");
    check(p >= 0 && p <= 1, "erdos: probability must be in [0,1]");
    *count_host = pair_edges(n, 1, p, p, seed, edges_uv, capacity, as_stream(stream));
  });
}

int pk_rmat_features(uint64_t seed, int64_t n, int64_t d, float* out, int64_t ldo,
                     void* stream) {
  return guard([&] {
    check(n >= 0 && d >= 0 && ldo >= d, "features: bad shape");
    rmat_features(seed, n, d, out, ldo, as_stream(stream));
  });
}

int pk_degree_quantile_labels(const uint32_t* edges_uv, uint64_t num_edges, int64_t n,
                              uint32_t classes, uint32_t* labels, void* stream) {
  return guard([&] {
    degree_quantile_labels(edges_uv, num_edges, n, classes, labels, as_stream(stream));
  });
}

}  // extern "C"
