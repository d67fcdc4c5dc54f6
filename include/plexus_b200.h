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
  PK_ERR_TRAINING = 5, /* TrainingError (trainer.hpp:26-29)           */
  PK_ERR_ABORTED = 6,  /* ClusterAborted (cluster.hpp:67-71): another
                          rank of the grid failed                      */
  /* IoError (common.hpp:28-41): 10 + IoErrorCode                        */
  PK_ERR_IO_MISSING = 10,   /* MissingFile                              */
  PK_ERR_IO_TRUNCATED = 11, /* TruncatedFile                            */
  PK_ERR_IO_CHECKSUM = 12,  /* ChecksumMismatch                         */
  PK_ERR_IO_MANIFEST = 13,  /* ManifestMismatch                         */
  PK_ERR_IO_FORMAT = 14,    /* BadFormat                                */
  PK_ERR_IO_WRITE = 15      /* WriteFailed                              */
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
int pk_abi_version(void); /* 2 */
/* total kernels launched by this library in the process (evidence counter) */
uint64_t pk_kernel_launch_count(void);
/* Device watchdog counters (process-wide): non-zero when an SpMM hub
 * pipeline or a tcgen05 GEMM pipeline abandoned a barrier wait (its output
 * is incomplete). The engine checks them after every epoch / pass and
 * fails with PK_ERR_CUDA; exposed for callers of the plain kernels. */
int pk_device_watchdogs(uint32_t* spmm, uint32_t* gemm);

/* Device memory the library freed is kept in a per-process cache and reused
 * by the next allocation of the same size (a rebuilt engine allocates
 * nothing new). This returns every cached block to the driver. */
int pk_device_cache_release(void);
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
/* The same with a numeric mode: PK_MODE_PARITY is the call above
 * (bit-identical); PK_MODE_FAST cuts hub rows into fixed segments whose sums
 * are combined in a fixed order (deterministic, fp32-level difference). */
int pk_spmm_plan_create_mode(const pk_csr* a, int64_t hub_threshold, int mode,
                             void* stream, pk_spmm_plan** out);
int pk_spmm_plan_destroy(pk_spmm_plan* plan);
int pk_spmm_plan_rows_f32(const pk_spmm_plan* plan, const pk_csr* a, int64_t r0,
                          int64_t r1, const float* x, int64_t x_rows,
                          int64_t ldx, int64_t d, float* y, int64_t ldy,
                          uint64_t* flops_host, void* stream);
/* spmm_rows then relu_backward in one pass (the backward's dF of layer l+1
 * feeding layer l): y = mask > 0 ? (A . X)[r0:r1] : 0, mask (r1 - r0) x d
 * with leading dimension ldm (the cached relu(Q) of layer l). Bit-identical
 * to pk_spmm_plan_rows_f32 followed by pk_relu_backward_f32. */
int pk_spmm_plan_rows_relu_bwd_f32(const pk_spmm_plan* plan, const pk_csr* a,
                                   int64_t r0, int64_t r1, const float* x,
                                   int64_t x_rows, int64_t ldx, int64_t d,
                                   const float* mask, int64_t ldm, float* y,
                                   int64_t ldy, uint64_t* flops_host,
                                   void* stream);
/* pk_spmm_plan_rows_f32 with flags. PK_SPMM_PAIRED (PK_MODE_FAST plans):
 * rows of at most 16 gathered vectors (16-B, 8-B or 4-B, by alignment: up
 * to 64 columns) are summed as two interleaved chains — the even and the
 * odd nonzeros of each 32-nonzero window, each in the reference's order —
 * added at the row end; a warp then gathers two rows per instruction.
 * Deterministic; another association of the same sum (fp32-level
 * difference, like the FAST plan's hub segments). Wider rows, and flags 0,
 * are pk_spmm_plan_rows_f32. */
#define PK_SPMM_PAIRED 1
int pk_spmm_plan_rows_ex_f32(const pk_spmm_plan* plan, const pk_csr* a,
                             int64_t r0, int64_t r1, const float* x,
                             int64_t x_rows, int64_t ldx, int64_t d, float* y,
                             int64_t ldy, int flags, uint64_t* flops_host,
                             void* stream);
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

/* gemm followed by relu_forward in one pass (the forward of a hidden layer:
 * C = relu(op(A) . op(B))); FAST applies it in the tensor-core epilogue,
 * PARITY as an in-place pass. Same results as pk_gemm_f32 then
 * pk_relu_forward_f32. */
int pk_gemm_relu_f32(int ta, int tb, int64_t m, int64_t n, int64_t k,
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

/* Philox(seed, stream).permutation(n) (rng.hpp:57-66) on the host */
int pk_philox_permutation_host(uint64_t n, uint64_t seed, uint64_t stream,
                               uint32_t* out_host);

/* synth_rmat edge draw (graph.hpp:291-322) on the device: Philox(seed, 5),
 * `scale` doubles per edge, self loops dropped (stable). Device output
 * buffer must hold 2*edges u32; *kept_host receives the kept count. */
int pk_rmat_edges(int scale, uint64_t edges, double a, double b, double c,
                  uint64_t seed, uint32_t* edges_uv, uint64_t* kept_host,
                  void* stream);
/* synth_sbm edge draw (graph.hpp:254-274) on the device: pair (u, v), u < v,
 * in lexicographic order takes the next double of Philox(seed, 5) and is
 * kept below p_in (same ceil-split community, graph.hpp:151-155) or p_out.
 * The kept pairs come out in the reference's order as u32 [u, v] pairs.
 * edges_uv == NULL: count only (*count_host = the edge count); otherwise the
 * device buffer holds `capacity` pairs (2 * capacity u32). */
int pk_sbm_edges(uint64_t n, int communities, double p_in, double p_out,
                 uint64_t seed, uint32_t* edges_uv, uint64_t capacity,
                 uint64_t* count_host, void* stream);
/* synth_erdos (graph.hpp:276-289): the same walk with one probability */
int pk_erdos_edges(uint64_t n, double p, uint64_t seed, uint32_t* edges_uv,
                   uint64_t capacity, uint64_t* count_host, void* stream);
/* features (graph.hpp:233-236): (float)next_double() of Philox(seed, 3) */
int pk_rmat_features(uint64_t seed, int64_t n, int64_t d, float* out,
                     int64_t ldo, void* stream);
/* degree_quantile_labels (graph.hpp:197-222) */
int pk_degree_quantile_labels(const uint32_t* edges_uv, uint64_t num_edges,
                              int64_t n, uint32_t classes, uint32_t* labels,
                              void* stream);

/* ------------------------------------------------------------------ */
/* Per-rank shard generation (billion-edge grids): one rank's blocks,    */
/* features and labels straight from synth_rmat's indexable Philox       */
/* streams, bit-identical to synth_rmat -> preprocess ->                 */
/* build_adjacency_shards / slice_rank_tensors (graph.hpp:40-148, 291-384,*/
/* engine.hpp:96-113, trainer.hpp:234-250) without the global graph.     */

/* RmatParams (graph.hpp:189-193) + the dataset's orientation: synth_rmat
 * always symmetrises (graph.hpp:23); undirected = 0 keeps the drawn
 * orientation with row degrees (the papers-shaped C4, SURVEY 8e'). */
typedef struct pk_rmat_spec {
  int scale;
  int undirected;
  uint64_t edges; /* 0 = 8 * 2^scale (graph.hpp:298) */
  double a, b, c;
  uint64_t seed;
} pk_rmat_spec;

/* Degrees of nodes [node0, node1) (device u32 out). kind 0: the degree
 * normalize_adjacency uses (distinct row entries incl. the self loop,
 * graph.hpp:44-61); kind 1: degree_quantile_labels' distinct undirected
 * neighbours without self loops (graph.hpp:197-210). Ranks compute their
 * node ranges and all-gather. */
int pk_rmat_node_degrees(const pk_rmat_spec* spec, int kind, int64_t node0,
                         int64_t node1, uint32_t* degree, void* stream);
/* inv[perm[i]] = i (invert_permutation, graph.hpp:95-99) */
int pk_invert_permutation(const uint32_t* perm, int64_t n, uint32_t* inv,
                          void* stream);
/* Block [r0, r1) x [c0, c1) of A_even (parity 0) or A_odd (1) with local
 * column ids — variant.block(...) of the reference (engine.hpp:108) —
 * from the permutation pair, its inverses and the all-gathered kind-0
 * degrees (device arrays of n). Allocates out (pk_csr_free). */
int pk_rmat_block(const pk_rmat_spec* spec, int parity, const uint32_t* row_perm,
                  const uint32_t* col_perm, const uint32_t* inv_row,
                  const uint32_t* inv_col, const uint32_t* norm_degree, int64_t r0,
                  int64_t r1, int64_t c0, int64_t c1, pk_csr_owned* out, void* stream);
/* features in permuted order (graph.hpp:233-236, 373-376): out[i - r0, j - c0]
 * = (float) next_double number perm[i] * feat_dim + j of Philox(seed, 3) */
int pk_rmat_features_permuted(uint64_t seed, int64_t feat_dim, const uint32_t* perm,
                              int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                              float* out, int64_t ldo, void* stream);
/* degree_quantile_labels (graph.hpp:212-221) from all n kind-1 degrees */
int pk_labels_from_degrees(const uint32_t* label_degree, int64_t n, uint32_t classes,
                           uint32_t* labels, void* stream);
/* out[i] = src[idx[i]] (labels / masks into a permuted order) */
int pk_gather_u32(const uint32_t* src, const uint32_t* idx, int64_t n, uint32_t* out,
                  void* stream);
int pk_gather_u8(const uint8_t* src, const uint32_t* idx, int64_t n, uint8_t* out,
                 void* stream);
/* dst row i = src row idx[i] (cols floats): preprocess' feature alignment,
 * features in col_perm order (graph.hpp:373-376) */
int pk_gather_rows_f32(const float* src, int64_t ld_src, const uint32_t* idx, int64_t n,
                       int64_t cols, float* dst, int64_t ld_dst, void* stream);
/* balance_metric (graph.hpp:157-172): max / mean nonzeros over the p x q
 * ceil-split block partition, counted on the device */
int pk_balance_metric(const pk_csr* a, int p, int q, double* out_host, void* stream);

/* ------------------------------------------------------------------ */
/* 3D-parallel GCN engine: one per rank (one per GPU)                   */
/*                                                                     */
/* Replaces the per-rank body of train_distributed (trainer.hpp:562-633):*/
/* RankTensors slicing (trainer.hpp:234-250), weight/feature slices      */
/* (model.hpp:35-67), forward_layer / backward_layer (engine.hpp:158-259),*/
/* rank_forward_backward (trainer.hpp:478-527) and Adam (598-599).       */
/* Collectives run on NCCL per-axis communicators (Cluster/RankCtx,      */
/* cluster.hpp:198-403, in-process threads in the reference).            */

#define PK_MAX_LAYERS 15

typedef struct pk_engine pk_engine;

typedef struct pk_engine_config {
  int gx, gy, gz;     /* GridConfig (grid.hpp:39-102)                   */
  int rank;           /* x fastest-varying (grid.hpp:58-63)             */
  int device;         /* CUDA device this rank runs on                  */
  int num_layers;     /* L                                              */
  int64_t dims[PK_MAX_LAYERS + 1]; /* model_dims (trainer.hpp:51-59)    */
  int64_t n;          /* nodes                                          */
  uint64_t seed;      /* TrainOptions.seed: weight init (model.hpp:17)  */
  double lr, beta1, beta2, eps;    /* AdamParams (model.hpp:69-74)       */
  int block_count;    /* EngineOptions.block_count, 0 = auto            */
  int mode;           /* pk_mode of the dense transforms                */
  int fault_epoch;    /* TrainOptions.fault_epoch (-1 = none)           */
  int64_t hub_threshold; /* SpMM hub rows (0 = automatic)               */
} pk_engine_config;

/* PreprocessedDataset<float> (graph.hpp:327-350). Device pointers for
 * pk_engine_load, host pointers for pk_engine_load_host. */
typedef struct pk_dataset_view {
  int64_t n;
  int64_t feat_dim;
  uint32_t num_classes;
  pk_csr a_even, a_odd;       /* n x n, permuted (graph.hpp:133-148)      */
  const float* features;      /* n x feat_dim, col_perm order             */
  int64_t ld_features;
  const uint32_t* labels_row; /* labels_row_order / labels_col_order      */
  const uint32_t* labels_col;
  const uint8_t* mask_row;
  const uint8_t* mask_col;
} pk_dataset_view;

/* RankTensors (trainer.hpp:217-224) in device memory: what a per-rank
 * loader (load_rank_shards, the file_handle path) produces. adj[plane * 2 +
 * parity] holds the block A[rows(row_shard), cols(inner)] of every key
 * needed_adjacency_keys lists (others: rows = cols = 0). */
typedef struct pk_rank_view {
  pk_csr adj[6];
  const float* f0;            /* feature_slice rows x cols, row-major       */
  int64_t f0_rows, f0_cols, ld_f0;
  const uint32_t* labels;     /* final-parity labels of label_row_range     */
  const uint8_t* mask;
  int64_t label_rows;
} pk_rank_view;

/* EpochMetrics (trainer.hpp:40-49); phase seconds are device time of this
 * rank (CUDA events), byte counters use the reference's ring model. */
typedef struct pk_epoch_metrics {
  int epoch;
  double loss, accuracy;
  double forward_spmm_s, forward_gemm_s, backward_s, optimizer_s, collectives_s;
  double epoch_s;
  double spmm_s;        /* device time of all SpMM launches (fwd + bwd)  */
  double spmm_bytes;    /* their algorithmic bytes (SURVEY 8d formula)    */
  uint64_t kernel_launches; /* libplexus kernels launched in the epoch    */
  uint64_t spmm_flops, gemm_flops;
  double allreduce_bytes, allgather_bytes, reducescatter_bytes;
  double spmm_compulsory_bytes; /* SpMM traffic floor: sparse matrix, output
                                   and each gathered row once             */
} pk_epoch_metrics;

typedef struct pk_tensor_view {
  float* data;
  int64_t rows, cols, ld;
} pk_tensor_view;

/* which tensor pk_engine_tensor returns */
enum {
  PK_T_W = 0,      /* stored W shard of layer l (weight_slice)           */
  PK_T_DW = 1,     /* dW shard of the last pass                          */
  PK_T_F0 = 2,     /* trainable feature shard (feature_slice)            */
  PK_T_DF0 = 3,    /* its gradient                                       */
  PK_T_FOUT = 4,   /* last layer's raw logits shard (RankPass.f_out)     */
  PK_T_H = 5,      /* cached H of layer l (valid after forward)          */
  PK_T_Q = 6,      /* cached Q of layer l: the last layer's, or a hidden
                      layer's when the engine materialised it (NCCL
                      fallback on a split col_shard); else an error     */
  PK_T_ACT = 7     /* relu(Q) of hidden layer l (next layer's input; the
                      backward's ReLU mask, relu(Q) > 0 <=> Q > 0)      */
};

/* 128-byte ncclUniqueId for rank 0 to broadcast (any bootstrap works). */
int pk_nccl_unique_id(void* out128);
int pk_engine_create(const pk_engine_config* cfg, pk_engine** out);
/* world_size 1 needs no call; otherwise every rank passes rank 0's id. */
int pk_engine_comm_init(pk_engine* e, const void* unique_id128, int world_size);
/* In-process cluster (Cluster, cluster.hpp:188-250, 405-442): every rank
 * of the grid is a host thread of this process with its own engine; several
 * ranks may share one GPU. Collectives are ordered device sums / copies
 * sequenced by CUDA events the members swap at a host rendezvous
 * (GroupChannel::exchange, cluster.hpp:140-168) — the reference's
 * coordinate-order combine bit for bit for any group size. When a rank's
 * load / pass / epoch fails, its cluster aborts: every other rank's pending
 * or next collective returns PK_ERR_ABORTED naming the failed rank
 * (ClusterAborted, cluster.hpp:67-71, 240, 434). */
typedef struct pk_cluster pk_cluster;
int pk_cluster_create(int gx, int gy, int gz, pk_cluster** out);
int pk_cluster_abort(pk_cluster* c, int rank, const char* why);
int pk_cluster_aborted(pk_cluster* c, int* aborted);
/* after every engine of the cluster is destroyed */
int pk_cluster_destroy(pk_cluster* c);
/* instead of pk_engine_comm_init: this engine is rank cfg.rank of `c` */
int pk_engine_comm_init_local(pk_engine* e, pk_cluster* c);
/* Measurement mode: rank cfg.rank of a grid larger than the machine runs
 * alone — every collective only puts this rank's own contribution in place
 * (results are NOT the GCN's), the ring-model byte counters still follow the
 * real grid. Measures one rank's memory and compute share (e.g. one rank of
 * 2x2x2 at billion-edge scale on one GPU). */
int pk_engine_comm_init_solo(pk_engine* e);
int pk_engine_load(pk_engine* e, const pk_dataset_view* ds);
int pk_engine_load_host(pk_engine* e, const pk_dataset_view* ds_host);
/* The file_handle path (trainer.hpp:461-466): this rank's tensors only
 * (e.g. from load_rank_shards); blocks are copied, the global CE count is
 * summed over the last layer's row_shard group (comm_init first when the
 * grid has more than one rank). */
int pk_engine_load_rank(pk_engine* e, const pk_rank_view* rank_tensors);
/* The same, taking over the blocks in `blocks[plane * 2 + parity]` (arrays
 * allocated by this library, e.g. pk_rmat_block / pk_csr_block) instead of
 * copying them — a billion-edge rank cannot hold its blocks twice. Taken
 * entries are zeroed; entries left with a NULL row_ptr are copied from
 * rank_tensors->adj as usual. */
int pk_engine_load_rank_adopt(pk_engine* e, const pk_rank_view* rank_tensors,
                              pk_csr_owned* blocks);
int pk_engine_forward_backward(pk_engine* e, int epoch, double* loss_host,
                               double* accuracy_host);
int pk_engine_optimizer_step(pk_engine* e);

/* SerialTrainer::forward_only (trainer.hpp:126-135) on the engine: the
 * forward of every layer with the current parameters — no loss, no
 * gradients, no optimizer step — then the pass's error checks. The logits
 * are this rank's last-layer output block (pk_engine_tensor PK_T_FOUT of the
 * last layer; the full n x C matrix on a 1x1x1 grid). Collective. */
int pk_engine_forward_only(pk_engine* e);
/* rank_forward_backward one piece at a time (forward_layer, engine.hpp:
 * 158-206; backward_layer, engine.hpp:214-259): begin_pass; forward_layer
 * l = 0..L-1 (fault = EngineOptions.fault_skip_h_allreduce); loss (logits
 * column gather + CE + the 1x3 sums all-reduce, trainer.hpp:498-516);
 * backward_layer l = L-1..0; finish_pass (stream sync, finalize_loss checks,
 * loss / accuracy). The same as pk_engine_forward_backward. The layer's
 * tensors (PK_T_H / PK_T_Q / PK_T_ACT / PK_T_DW) are readable after it. */
int pk_engine_begin_pass(pk_engine* e);
int pk_engine_forward_layer(pk_engine* e, int layer, int fault);
int pk_engine_loss(pk_engine* e);
int pk_engine_backward_layer(pk_engine* e, int layer);
int pk_engine_finish_pass(pk_engine* e, int epoch, double* loss_host,
                          double* accuracy_host);

/* RankCtx collectives (cluster.hpp:265-340) over this rank's axis group
 * (axis 0/1/2 = X/Y/Z; members in ascending coordinate order), on device
 * buffers, enqueued on `stream`; singleton axes short-circuit but are still
 * counted, like the reference. Every member of the group must make the same
 * call. Sums are the reference's coordinate-order combine (in-process
 * clusters and peer-memory groups) or NCCL's sum (two-member axes: equal).
 *   all_reduce     (cluster.hpp:307-321): buf rows x cols (ld) summed in place
 *   all_gather     (cluster.hpp:268-305): member j's block (chunk_size(out_rows
 *                  or out_cols, g, j) rows / columns) concatenated by rows
 *                  (concat_cols = 0) or columns (1) into out
 *   reduce_scatter (cluster.hpp:323-340): sum of buf (rows x cols), this
 *                  member keeps row chunk chunk_start(rows, g, pos).. in out */
int pk_engine_all_reduce_f32(pk_engine* e, int axis, float* buf, int64_t rows,
                             int64_t cols, int64_t ld, void* stream);
int pk_engine_all_gather_f32(pk_engine* e, int axis, int concat_cols,
                             const float* local, int64_t local_ld, float* out,
                             int64_t out_rows, int64_t out_cols, int64_t out_ld,
                             void* stream);
int pk_engine_reduce_scatter_f32(pk_engine* e, int axis, float* buf, int64_t rows,
                                 int64_t cols, int64_t ld, float* out,
                                 void* stream);
int pk_engine_train_epoch(pk_engine* e, int epoch, pk_epoch_metrics* out_host);
/* `count` epochs (first_epoch, first_epoch + 1, ...) enqueued back to back
 * with one host wait at the end (no per-epoch sync bubble); out_host[count]
 * receives each epoch's metrics, and the first epoch that fails the loss
 * checks raises (PK_ERR_TRAINING naming it) after the wait. */
int pk_engine_train_epochs(pk_engine* e, int first_epoch, int count,
                           pk_epoch_metrics* out_host);
/* This rank failed outside the library (e.g. its host code threw): take the
 * grid down like the reference's Cluster does (cluster.hpp:240, 434). In
 * an in-process cluster every other rank's collectives return
 * PK_ERR_ABORTED; across processes (pk_engine_comm_init) the failure is
 * published in a node-local shared-memory block named after the NCCL unique
 * id, every rank aborts its communicators and peer-memory waits, and their
 * pending epoch returns PK_ERR_ABORTED naming this rank. Failures inside
 * pk_engine_load* / forward_backward / train_epoch do this on their own. */
int pk_engine_abort(pk_engine* e, const char* why);
/* CommStats (cluster.hpp:35-65) of this rank since its load: calls and
 * ring-model bytes (CommStats::bytes, cluster.hpp:53-55) per [axis * 3 + op],
 * op 0 all_gather, 1 all_reduce, 2 reduce_scatter — comm_stats.csv of the
 * CLI (main.cpp:353-366). */
int pk_engine_comm_stats(pk_engine* e, uint64_t* calls9, double* ring_bytes9);
int pk_engine_tensor(pk_engine* e, int which, int layer, pk_tensor_view* out);
int pk_engine_stream(pk_engine* e, void** stream_out);
int pk_engine_destroy(pk_engine* e);

/* ------------------------------------------------------------------ */
/* Performance model: picks the grid (perf_model.hpp:18-127,            */
/* src/perf_model.cpp:33-229). Host-only; no device work.               */

/* DatasetStats (perf_model.hpp:18-22) */
typedef struct pk_dataset_stats {
  int64_t n;
  uint64_t nnz;
  int num_dims;                       /* L + 1                          */
  int64_t dims[PK_MAX_LAYERS + 1];
} pk_dataset_stats;

/* MachineParams (perf_model.hpp:24-29); reference defaults
 * {4, 200e9, 25e9, 4}. */
typedef struct pk_machine {
  int g_node;
  double beta_intra, beta_inter;
  int bytes_per_scalar;
} pk_machine;

/* PerfCoefficients (perf_model.hpp:31-41) */
typedef struct pk_perf_coeffs {
  double c1, c2, c3, train_r2, train_rmse;
} pk_perf_coeffs;

/* ConfigPrediction (perf_model.hpp:98-104) */
typedef struct pk_config_prediction {
  int gx, gy, gz, clamped;
  double spmm_seconds, comm_seconds, total_seconds;
} pk_config_prediction;

/* CollOp / CollectiveVolume (layout.hpp:105-121) */
enum { PK_COLL_ALL_GATHER = 0, PK_COLL_ALL_REDUCE = 1, PK_COLL_REDUCE_SCATTER = 2 };
typedef struct pk_collective_volume {
  int layer, forward, op, axis; /* axis 0/1/2 = X/Y/Z                 */
  uint64_t elems;               /* full buffer M (pre-scatter for RS) */
} pk_collective_volume;

/* default_coefficients (perf_model.hpp:38-40) */
int pk_perf_default_coefficients(pk_perf_coeffs* out);
/* comp_features (perf_model.cpp:33-56): 3 doubles */
int pk_perf_comp_features(const pk_dataset_stats* stats, int gx, int gy, int gz,
                          double* features3);
/* predict_spmm_time (perf_model.cpp:58-64): negative -> 0, clamped = 1 */
int pk_perf_predict_spmm(const double* features3, const pk_perf_coeffs* c,
                         double* seconds, int* clamped);
/* effective_bandwidth (perf_model.cpp:66-78) */
int pk_perf_effective_bandwidth(int axis, int gx, int gy, int gz,
                                const pk_machine* m, double* out);
/* ring_collective_seconds (perf_model.cpp:80-85) */
int pk_perf_ring_seconds(int op, double bytes, int g, double beta, double* out);
/* predict_comm_time(...).total (perf_model.cpp:87-102) */
int pk_perf_predict_comm(const pk_dataset_stats* stats, int gx, int gy, int gz,
                         const pk_machine* m, double* total_seconds);
/* training_collective_volumes (layout.hpp:123-157); out may be NULL to
 * query the count */
int pk_collective_volumes(int gx, int gy, int gz, const pk_dataset_stats* stats,
                          pk_collective_volume* out, int cap, int* count);
/* fit_regression (perf_model.cpp:104-166): features row-major count x 3 */
int pk_perf_fit_regression(const double* features3, const double* seconds,
                           int count, pk_perf_coeffs* out);
/* enumerate_configs (grid.hpp:112-123): triples in (gx, gy) lexicographic
 * order; gxyz may be NULL to query the count */
int pk_enumerate_configs(int g, int* gxyz, int cap, int* count);
/* rank_configs (perf_model.cpp:207-229): ascending total, ties by
 * (gz, gx, gy) */
int pk_perf_rank_configs(int g, const pk_dataset_stats* stats,
                         const pk_machine* m, const pk_perf_coeffs* c,
                         pk_config_prediction* out, int cap, int* count);

/* ------------------------------------------------------------------ */
/* PLXS shard files (shard_io.hpp:26-414, trainer.hpp:252-438)         */

/* One CSR block in host memory for the writer; values are `precision`
 * bytes each (4 = f32, 8 = f64). */
typedef struct pk_plxs_csr_host {
  uint64_t rows, cols, nnz;
  const uint64_t* row_ptr;
  const uint32_t* col_idx;
  const void* values;
} pk_plxs_csr_host;

/* write_shards' per-file body (shard_io.hpp:311-361): header, CSR even,
 * CSR odd, feature block, labels/masks of the row block; byte-identical to
 * the reference. checksums_out = the four sections' FNV-1a 64. */
int pk_plxs_write(const char* path, const uint64_t ranges[6], uint32_t precision,
                  const pk_plxs_csr_host* even, const pk_plxs_csr_host* odd,
                  uint64_t f_rows, uint64_t f_cols, const void* features,
                  uint64_t label_count, const uint32_t* labels_row,
                  const uint32_t* labels_col, const uint8_t* mask_row,
                  const uint8_t* mask_col, uint64_t checksums_out[4]);

/* ShardFileReader (shard_io.hpp:90-276). open checks magic, version,
 * precision (0 = any) and the block ranges against the manifest (NULL =
 * skip). Reads of a whole section verify its checksum (`expected`);
 * partial reads cannot, like the reference. `device` = 1 streams col_idx /
 * values / features into device memory through a pinned double buffer on
 * `stream`. */
typedef struct pk_plxs pk_plxs;
int pk_plxs_open(const char* path, const uint64_t expect_ranges[6], uint32_t precision,
                 pk_plxs** out);
int pk_plxs_close(pk_plxs* h);
int pk_plxs_info(const pk_plxs* h, uint64_t ranges_out[6], uint32_t* precision,
                 uint64_t* bytes_read);
int pk_plxs_csr_extent(pk_plxs* h, int section, uint64_t r0, uint64_t r1, uint64_t* rows,
                       uint64_t* cols, uint64_t* nnz, uint64_t* e0, uint64_t* e1);
int pk_plxs_read_csr_rows(pk_plxs* h, int section, uint64_t r0, uint64_t r1,
                          uint64_t expected, uint64_t* row_ptr, uint32_t* col_idx,
                          void* values, int device, void* stream);
int pk_plxs_read_feature_rows(pk_plxs* h, uint64_t r0, uint64_t r1, uint64_t expected,
                              void* dst, int device, void* stream);
int pk_plxs_read_labels(pk_plxs* h, uint64_t r0, uint64_t r1, uint64_t expected,
                        uint32_t* labels_row, uint32_t* labels_col, uint8_t* mask_row,
                        uint8_t* mask_col);

/* load_rank_shards' row merge (trainer.hpp:276-309) on the device: pieces
 * k = 0..count-1 hold the same rows (row_ptr on the device, rebased), with
 * column origin col0[k] in the global numbering; out = for each row, the
 * pieces' entries in piece order whose global column lies in [c0, c1),
 * renumbered from c0. Allocates out (free with pk_csr_free). */
int pk_csr_hconcat(const pk_csr* pieces, const uint64_t* col0, int count, uint64_t c0,
                   uint64_t c1, pk_csr_owned* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* PLEXUS_B200_H */
