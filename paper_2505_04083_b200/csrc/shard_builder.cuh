// Internal interface of the GPU shard builder (shard_builder.cu, rmat.cu).
#pragma once

#include "pk_common.cuh"

namespace pk {

void csr_transpose(const pk_csr& a, pk_csr_owned* out, cudaStream_t st);
void csr_block(const pk_csr& a, i64 r0, i64 r1, i64 c0, i64 c1, pk_csr_owned* out,
               cudaStream_t st);
void normalize_adjacency(i64 n, const u32* uv, u64 m, bool undirected, pk_csr_owned* out,
                         cudaStream_t st);
void permute_csr(const pk_csr& a, const u32* row_perm, const u32* col_perm, pk_csr_owned* out,
                 cudaStream_t st);
void csr_free(pk_csr_owned* m);
// load_rank_shards' row merge of column pieces (trainer.hpp:276-309)
void csr_hconcat(const pk_csr* pieces, const u64* col0, int count, u64 c0, u64 c1,
                 pk_csr_owned* out, cudaStream_t st);

u64 rmat_edges(int scale, u64 edges, double a, double b, double c, u64 seed, u32* uv,
               cudaStream_t st);
// synth_sbm / synth_erdos edge lists (graph.hpp:254-289; Erdős = one
// community): uv == nullptr counts only; returns the edge count
u64 pair_edges(u64 n, int communities, double p_in, double p_out, u64 seed, u32* uv,
               u64 capacity, cudaStream_t st);
void rmat_features(u64 seed, i64 n, i64 d, float* out, i64 ldo, cudaStream_t st);
void degree_quantile_labels(const u32* uv, u64 m, i64 n, u32 classes, u32* labels,
                            cudaStream_t st);

inline pk_csr view(const pk_csr_owned& m) {
  return pk_csr{m.rows, m.cols, m.nnz, m.row_ptr, m.col_idx, m.values};
}

}  // namespace pk
