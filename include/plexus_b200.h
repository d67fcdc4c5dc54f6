/*
 * plexus_b200.h — C ABI of the B200-native Plexus GCN hot path
 * (libplexus_b200.so, built from paper_2505_04083_b200/csrc).
 *
 * Drop-in boundary for the reference's header-only C++ API in
 * /root/reference/proj/include/plexuskit (paths below are relative to it).
 * Every entry point names the reference function it replaces. The reference
 * has no FFI of its own; INTEGRATION.md shows the C++ forwarding shim a
 * maintainer adds to kernels.hpp / engine.hpp / trainer.hpp to call these.
 *
 * Conventions
 *   - Plain pointers and sizes only. Pointers are DEVICE pointers unless the
 *     parameter name ends in `_host`. Dense matrices are row-major with an
 *     explicit leading dimension (elements).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *   - Return value: a pk_status. On failure pk_last_error() (thread-local)
 *     holds a message naming the shapes, in the reference's wording.
 *   - The caller owns every buffer passed in; the library owns only the
 *     workspaces inside pk_spmm_plan / pk_engine objects.
 *   - Zero-extent operands are legal (reference test_engine.cpp:173-188):
 *     an empty output launches nothing; a GEMM with k = 0 writes zeros.
 *   - float32 only (the reference's T = float instantiation).
 */
#ifndef PLEXUS_B200_H
#define PLEXUS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pk_status {
  PK_OK = 0,
  PK_ERR_CONTRACT = 1, /* ContractError (common.hpp:16-20)            */
  PK_ERR_CUDA = 2,     /* CUDA runtime / launch failure               */
  PK_ERR_NCCL = 3,     /* NCCL failure                                */
  PK_ERR_MEMORY = 4,   /* MemoryError (common.hpp:22-26), device OOM  */
  PK_ERR_TRAINING = 5  /* TrainingError (trainer.hpp:26-29)           */
} pk_status;

/* Numeric mode of the dense transforms. PARITY reproduces the reference's
 * scalar loop order bit-for-bit (kernels.hpp:84-89: acc from 0, k ascending,
 * separate mul and add). FAST uses the sm_100a tensor-core path (3xTF32,
 * fp32-level error, tolerance-checked). SpMM is bit-exact in both modes. */
typedef enum pk_mode { PK_MODE_PARITY = 0, PK_MODE_FAST = 1 } pk_mode;

/* CsrMatrix<float> (csr.hpp:14-149): u64 row_ptr, u32 col_idx (strictly
 * increasing within a row), f32 values. Device pointers. */
typedef struct pk_csr {
  int64_t rows;
  int64_t cols;
  uint64_t nnz;
  const uint64_t* row_ptr;
  const uint32_t* col_idx;
  const float* values;
} pk_csr;

/* Mutable CSR produced by the shard builder; arrays are allocated by the
 * library (cudaMalloc) and released with pk_csr_free. */
typedef struct pk_csr_owned {
  int64_t rows;
  int64_t cols;
  uint64_t nnz;
  uint64_t* row_ptr;
  uint32_t* col_idx;
  float* values;
} pk_csr_owned;

const char* pk_last_error(void);
int pk_abi_version(void);
int pk_device_sm_count(int device);

/* ------------------------------------------------------------------ */
/* Sparse aggregation                                                  */

/* spmm_rows (kernels.hpp:39-62): y[0:r1-r0, 0:d] = A[r0:r1, :] . x.
 * x is a.cols x d (ldx), y is (r1-r0) x d (ldy). Bit-exact with the
 * reference. flops (optional, host) += 2 * nnz(A[r0:r1]) * d. */
int pk_spmm_rows_f32(const pk_csr* a, int64_t r0, int64_t r1, const float* x,
                     int64_t x_rows, int64_t ldx, int64_t d, float* y,
                     int64_t ldy, uint64_t* flops_host, void* stream);

/* spmm (kernels.hpp:16-37) = spmm_rows over all rows. */
int pk_spmm_f32(const pk_csr* a, const float* x, int64_t x_rows, int64_t ldx,
                int64_t d, float* y, int64_t ldy, uint64_t* flops_host,
                void* stream);

/* A reusable schedule for one sparse matrix (hub rows split off and
 * ordered longest-first, short rows packed). Same results as the plain
 * calls; built once per adjacency shard (engine.hpp:96-113 precomputes its
 * shards the same way). */
typedef struct pk_spmm_plan pk_spmm_plan;
/* hub_threshold: rows with at least this many nonzeros take the hub path;
 * 0 = automatic (max(4096, 64 x mean row length)). */
int pk_spmm_plan_create(const pk_csr* a, int64_t hub_threshold, void* stream,
                        pk_spmm_plan** out);
int pk_spmm_plan_destroy(pk_spmm_plan* plan);
int pk_spmm_plan_rows_f32(const pk_spmm_plan* plan, const pk_csr* a, int64_t r0,
                          int64_t r1, const float* x, int64_t x_rows,
                          int64_t ldx, int64_t d, float* y, int64_t ldy,
                          uint64_t* flops_host, void* stream);
/* number of hub rows and the hub threshold the plan chose */
int pk_spmm_plan_info(const pk_spmm_plan* plan, int64_t* hub_rows,
                      int64_t* hub_threshold);

/* ------------------------------------------------------------------ */
/* Dense transform                                                     */

/* gemm (kernels.hpp:64-92): C(m x n) = op(A) . op(B) with op = transpose
 * when ta / tb is set; A is stored (ta ? k x m : m x k), B is stored
 * (tb ? n x k : k x n). Row-major with leading dimensions. k == 0 writes
 * zeros. flops (optional, host) += 2*m*n*k. */
int pk_gemm_f32(int ta, int tb, int64_t m, int64_t n, int64_t k,
                const float* a, int64_t lda, const float* b, int64_t ldb,
                float* c, int64_t ldc, int mode, uint64_t* flops_host,
                void* stream);

/* ------------------------------------------------------------------ */
/* Fused elementwise                                                   */

/* relu_forward (kernels.hpp:94-100): out = q > 0 ? q : 0 (rows x cols) */
int pk_relu_forward_f32(const float* q, int64_t ldq, int64_t rows,
                        int64_t cols, float* out, int64_t ldo, void* stream);
/* relu_backward (kernels.hpp:102-111): out = q > 0 ? df : 0 */
int pk_relu_backward_f32(const float* q, int64_t ldq, const float* df,
                         int64_t lddf, int64_t rows, int64_t cols, float* out,
                         int64_t ldo, void* stream);

/* softmax_cross_entropy_sums (kernels.hpp:117-158). Writes dlogits
 * (softmax - onehot on masked rows, 0 elsewhere) and the three sums into
 * DEVICE scalars sums_dev = {loss_sum (double), count (as double),
 * correct (as double)} — the 1x3 double block the trainer all-reduces
 * (trainer.hpp:501-504). Out-of-range labels on masked rows -> contract
 * error (checked on the host after the launch). */
int pk_softmax_ce_sums_f32(const float* logits, int64_t ldl, int64_t rows,
                           int64_t classes, const uint32_t* labels,
                           const uint8_t* mask, float* dlogits, int64_t ldd,
                           double* sums_dev, void* stream);

/* finalize_loss scaling (trainer.hpp:84-87): d *= (float)1/(float)count,
 * count read from the device sums block. */
int pk_scale_by_count_f32(float* d, int64_t ldd, int64_t rows, int64_t cols,
                          const double* sums_dev, void* stream);

/* adam_step (model.hpp:88-111) on `n` contiguous elements. `step` is the
 * step count AFTER the increment; bias terms are formed in double on the
 * host exactly as the reference does. Bit-exact. */
int pk_adam_step_f32(float* param, const float* grad, float* m, float* v,
                     int64_t n, uint64_t step, double lr, double beta1,
                     double beta2, double eps, void* stream);

/* ------------------------------------------------------------------ */
/* Shard builder (graph.hpp, csr.hpp) — bit-exact with the reference     */

/* CsrMatrix::transpose (csr.hpp:78-95) */
int pk_csr_transpose(const pk_csr* a, pk_csr_owned* out, void* stream);
/* CsrMatrix::block (csr.hpp:97-120) with local column ids */
int pk_csr_block(const pk_csr* a, int64_t r0, int64_t r1, int64_t c0,
                 int64_t c1, pk_csr_owned* out, void* stream);
/* normalize_adjacency (graph.hpp:40-76): edges are device u32 pairs */
int pk_normalize_adjacency(int64_t n, const uint32_t* edges_uv,
                           uint64_t num_edges, int undirected,
                           pk_csr_owned* out, void* stream);
/* permute_csr (graph.hpp:101-131): result[i,j] = a[row_perm[i], col_perm[j]]
 * (device permutations) */
int pk_permute_csr(const pk_csr* a, const uint32_t* row_perm,
                   const uint32_t* col_perm, pk_csr_owned* out, void* stream);
void pk_csr_free(pk_csr_owned* m);

/* generate_permutation_pair (graph.hpp:84-93): Philox Fisher-Yates on the
 * host (sequential by definition); host output arrays of length n. */
int pk_permutation_pair_host(uint64_t n, uint64_t seed, uint32_t* row_perm_host,
                             uint32_t* col_perm_host);

/* synth_rmat edge draw (graph.hpp:291-322) on the device: Philox(seed, 5),
 * `scale` doubles per edge, self loops dropped (stable). Device output
 * buffer must hold 2*edges u32; *kept_host receives the kept count. */
int pk_rmat_edges(int scale, uint64_t edges, double a, double b, double c,
                  uint64_t seed, uint32_t* edges_uv, uint64_t* kept_host,
                  void* stream);
/* features (graph.hpp:233-236): (float)next_double() of Philox(seed, 3) */
int pk_rmat_features(uint64_t seed, int64_t n, int64_t d, float* out,
                     int64_t ldo, void* stream);
/* degree_quantile_labels (graph.hpp:197-222) */
int pk_degree_quantile_labels(const uint32_t* edges_uv, uint64_t num_edges,
                              int64_t n, uint32_t classes, uint32_t* labels,
                              void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PLEXUS_B200_H */
