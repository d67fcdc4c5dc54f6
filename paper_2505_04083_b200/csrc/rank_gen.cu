// Per-rank synthetic shard generation: one rank's adjacency blocks, F0 slice
// and labels straight from the generator's indexable Philox streams, never
// materialising the global graph — what a billion-edge grid needs (SURVEY
// 8a S18/S19, 8e; the papers-shaped C4 target). Bit-identical to
//   synth_rmat (graph.hpp:291-322) -> preprocess (356-384) ->
//   build_adjacency_shards / slice_rank_tensors (engine.hpp:96-113,
//   trainer.hpp:234-250).
//
// Why this is possible without a global sort:
//  * edge e of synth_rmat is a closed-form function of e (philox.cuh), so a
//    rank regenerates all edges in registers and keeps only those that land
//    in its blocks;
//  * normalize_adjacency's value for (u, v) needs only the two degrees
//    (graph.hpp:57-73), and a degree needs only the rows of that node:
//    ranks count the distinct neighbours of their own node range and the
//    degree vectors are all-gathered (pk_rmat_node_degrees);
//  * A_even[i, j] = A[row_perm[i], col_perm[j]] (graph.hpp:101-131): an edge
//    (u, v) maps to (inv_row[u], inv_col[v]); duplicates collapse with the
//    block's own sort + unique, exactly like the reference's global
//    sort + unique restricted to the block;
//  * degree_quantile_labels (graph.hpp:197-222) needs every node's
//    undirected distinct-neighbour degree (same all-gather) and one sort of
//    n (degree, id) keys.
// Generation work is two passes over the edge stream per output (count, then
// fill), all in registers: no edge list, no global key array.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "philox.cuh"
#include "pk_common.cuh"
#include "shard_builder.cuh"

namespace pk {

namespace {

unsigned grid_for(u64 n) {
  return static_cast<unsigned>(std::max<u64>(1, std::min<u64>((n + 255) / 256, 148u * 64)));
}

struct RmatDev {
  int scale;
  int undirected;
  u64 edges;
  double a, ab, abc;
  u64 seed;
};

// edge e of synth_rmat (graph.hpp:300-320); false for a dropped self loop
__device__ __forceinline__ bool rmat_edge(const RmatDev& s, u64 e, u32& u, u32& v) {
  u = 0, v = 0;
  u64 t = e * static_cast<u64>(s.scale);
  u64 cur = ~0ull;
  Philox4 blk{};
  for (int bit = 0; bit < s.scale; ++bit, ++t) {
    if ((t >> 1) != cur) {
      cur = t >> 1;
      blk = philox_at(s.seed, 5, cur);
    }
    const int k = static_cast<int>(t & 1) * 2;
    const double r = u64_to_unit(static_cast<u64>(blk.v[k]) | (static_cast<u64>(blk.v[k + 1]) << 32));
    u <<= 1;
    v <<= 1;
    if (r < s.a) {
    } else if (r < s.ab) {
      v |= 1;
    } else if (r < s.abc) {
      u |= 1;
    } else {
      u |= 1;
      v |= 1;
    }
  }
  return u != v;
}

// Warp-aggregated append: every lane of the warp calls it the same number
// of times (uniform loop bounds); lanes with `want` get consecutive slots.
__device__ __forceinline__ void append(bool want, u64 key, u64* out, unsigned long long* count) {
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  const int lane = threadIdx.x & 31;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(count, static_cast<unsigned long long>(__popc(m)));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (want && out) out[base + __popc(m & ((1u << lane) - 1u))] = key;
}

// kind 0: normalize_adjacency's rows (graph.hpp:44-61) — E, plus E^T when
// undirected; kind 1: degree_quantile_labels' neighbours (197-210) — E and
// E^T always. Keys ((u - node0) << 32) | v for rows u in [node0, node1).
__global__ void degree_keys_kernel(RmatDev s, int kind, u32 node0, u32 node1, u64* out,
                                   unsigned long long* count) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  const u64 first = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) & ~31ull;
  const bool both = kind == 1 || s.undirected;
  for (u64 base = first; base < s.edges; base += stride) {
    const u64 e = base + (threadIdx.x & 31);
    u32 u = 0, v = 0;
    const bool ok = e < s.edges && rmat_edge(s, e, u, v);
    append(ok && u >= node0 && u < node1, (static_cast<u64>(u - node0) << 32) | v, out, count);
    append(ok && both && v >= node0 && v < node1, (static_cast<u64>(v - node0) << 32) | u, out,
           count);
  }
}

// Entries of one block of A_parity: edges (and their mirrors when
// undirected) mapped through the inverse permutations, plus the self loops
// normalize_adjacency adds for every node (graph.hpp:52-53).
struct BlockMap {
  const u32* inv_r;  // inverse of the permutation applied to rows
  const u32* inv_c;  // ... to columns
  u32 r0, r1, c0, c1;
};

__device__ __forceinline__ bool map_entry(const BlockMap& m, u32 u, u32 v, u64& key) {
  const u32 i = m.inv_r[u], j = m.inv_c[v];
  if (i < m.r0 || i >= m.r1 || j < m.c0 || j >= m.c1) return false;
  key = (static_cast<u64>(i - m.r0) << 32) | (j - m.c0);
  return true;
}

__global__ void block_keys_kernel(RmatDev s, BlockMap m, u64* out, unsigned long long* count) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  const u64 first = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) & ~31ull;
  for (u64 base = first; base < s.edges; base += stride) {
    const u64 e = base + (threadIdx.x & 31);
    u32 u = 0, v = 0;
    const bool ok = e < s.edges && rmat_edge(s, e, u, v);
    u64 k1 = 0, k2 = 0;
    const bool w1 = ok && map_entry(m, u, v, k1);
    const bool w2 = ok && s.undirected && map_entry(m, v, u, k2);
    append(w1, k1, out, count);
    append(w2, k2, out, count);
  }
}

__global__ void self_loop_keys_kernel(u64 n, BlockMap m, u64* out, unsigned long long* count) {
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  const u64 first = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) & ~31ull;
  for (u64 base = first; base < n; base += stride) {
    const u64 u = base + (threadIdx.x & 31);
    u64 k = 0;
    const bool w = u < n && map_entry(m, static_cast<u32>(u), static_cast<u32>(u), k);
    append(w, k, out, count);
  }
}

__global__ void count_rows_kernel(const u64* keys, u64 k, u32* deg) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < k;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    atomicAdd(&deg[keys[i] >> 32], 1u);
}

__global__ void add_scalar_kernel(u32* deg, u64 n, u32 add) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    deg[i] += add;
}

__global__ void row_counts_u64_kernel(const u64* keys, u64 k, u64* counts) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < k;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&counts[(keys[i] >> 32) + 1]), 1ull);
}

// col_idx and the normalised value (graph.hpp:66-70) of every unique key;
// the global node ids come back through the forward permutations
__global__ void block_entries_kernel(const u64* keys, u64 k, const u32* perm_r, const u32* perm_c,
                                     u32 r0, u32 c0, const u32* degree, u32* col, float* val) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < k;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 li = static_cast<u32>(keys[i] >> 32), lj = static_cast<u32>(keys[i]);
    const u32 u = perm_r[r0 + li], v = perm_c[c0 + lj];
    col[i] = lj;
    val[i] = static_cast<float>(1.0 / sqrt(static_cast<double>(degree[u]) *
                                           static_cast<double>(degree[v])));
  }
}

// out[i - r0, j - c0] = (float) next_double of Philox(seed, 3) number
// perm[i] * d + j — row perm[i] of the features (graph.hpp:233-236) in the
// permuted order (features travel with col_perm, graph.hpp:373-376)
__global__ void features_perm_kernel(u64 seed, i64 d, const u32* perm, i64 r0, i64 r1, i64 c0,
                                     i64 c1, float* out, i64 ldo) {
  const i64 w = c1 - c0;
  const u64 total = static_cast<u64>(r1 - r0) * w;
  for (u64 t = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<u64>(gridDim.x) * blockDim.x) {
    const i64 i = static_cast<i64>(t / w), j = static_cast<i64>(t % w);
    const u64 idx = static_cast<u64>(perm[r0 + i]) * d + (c0 + j);
    out[i * ldo + j] = static_cast<float>(u64_to_unit(philox_u64_at(seed, 3, idx)));
  }
}

__global__ void invert_kernel(const u32* p, u64 n, u32* inv) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    inv[p[i]] = static_cast<u32>(i);
}

__global__ void degree_id_keys_kernel(const u32* degree, u64 n, u64* keys) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    keys[i] = (static_cast<u64>(degree[i]) << 32) | i;
}

__global__ void assign_labels_kernel(const u64* sorted, u64 n, u32 classes, u32* labels) {
  for (u64 pos = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; pos < n;
       pos += static_cast<u64>(gridDim.x) * blockDim.x)
    labels[static_cast<u32>(sorted[pos])] = static_cast<u32>(pos * classes / n);
}

__global__ void gather_u32_kernel(const u32* src, const u32* idx, u64 n, u32* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = src[idx[i]];
}

template <typename F>
void cub_run(F&& f, cudaStream_t st) {
  size_t bytes = 0;
  PK_CUDA(f(nullptr, bytes));
  DevBuf<unsigned char> tmp(bytes ? bytes : 1);
  PK_CUDA(f(tmp.p, bytes));
  PK_CUDA(cudaStreamSynchronize(st));  // tmp dies here
}

RmatDev to_dev(const pk_rmat_spec& s) {
  check(s.scale >= 1 && s.scale < 31, "rmat: scale out of range");
  check(s.a > 0 && s.b >= 0 && s.c >= 0 && s.a + s.b + s.c < 1.0,
        "rmat: quadrant probabilities must sum below 1");
  RmatDev d;
  d.scale = s.scale;
  d.undirected = s.undirected ? 1 : 0;
  d.edges = s.edges ? s.edges : 8ull << s.scale;  // graph.hpp:298
  d.a = s.a, d.ab = s.a + s.b, d.abc = s.a + s.b + s.c;  // same order as the reference
  d.seed = s.seed;
  return d;
}

int bits_for(u64 x) {
  int b = 1;
  while (b < 64 && (x >> b)) ++b;
  return b;
}

// count pass, allocate exactly, fill pass; then sort + unique. Returns the
// unique key count; keys end up in `out`.
template <typename Launch>
u64 collect_unique(Launch&& launch, int key_bits, DevBuf<u64>& out, cudaStream_t st) {
  DevBuf<unsigned long long> cnt(1);
  PK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
  launch(static_cast<u64*>(nullptr), cnt.p);
  unsigned long long k = 0;
  PK_CUDA(cudaMemcpyAsync(&k, cnt.p, sizeof(k), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  DevBuf<u64> raw(k ? k : 1), sorted(k ? k : 1);
  PK_CUDA(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
  launch(raw.p, cnt.p);
  if (k) {
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortKeys(t, b, raw.p, sorted.p, static_cast<i64>(k), 0,
                                            key_bits, st);
    }, st);
    DevBuf<i64> nsel(1);
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceSelect::Unique(t, b, sorted.p, raw.p, nsel.p, static_cast<i64>(k), st);
    }, st);
    i64 u = 0;
    PK_CUDA(cudaMemcpyAsync(&u, nsel.p, sizeof(u), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    k = static_cast<unsigned long long>(u);
  }
  out = std::move(raw);
  return k;
}

}  // namespace

}  // namespace pk

using namespace pk;

extern "C" {

int pk_rmat_node_degrees(const pk_rmat_spec* spec, int kind, int64_t node0, int64_t node1,
                         uint32_t* degree, void* stream) {
  return guard([&] {
    check(spec != nullptr, "rmat: null spec");
    check(kind == 0 || kind == 1, "rmat degrees: kind must be 0 (normalize) or 1 (labels)");
    const RmatDev s = to_dev(*spec);
    const i64 n = i64{1} << s.scale;
    check(node0 >= 0 && node0 <= node1 && node1 <= n, "rmat degrees: node range out of bounds");
    cudaStream_t st = as_stream(stream);
    const u64 rows = static_cast<u64>(node1 - node0);
    if (!rows) return;
    PK_CUDA(cudaMemsetAsync(degree, 0, rows * sizeof(u32), st));
    DevBuf<u64> keys;
    const u64 k = collect_unique(
        [&](u64* out, unsigned long long* cnt) {
          degree_keys_kernel<<<grid_for(s.edges), 256, 0, st>>>(
              s, kind, static_cast<u32>(node0), static_cast<u32>(node1), out, cnt);
          PK_LAUNCH("rmat degree keys");
        },
        32 + bits_for(rows), keys, st);
    if (k) {
      count_rows_kernel<<<grid_for(k), 256, 0, st>>>(keys.p, k, degree);
      PK_LAUNCH("rmat degree count");
    }
    if (kind == 0) {  // the self loop every node gets (graph.hpp:52-53)
      add_scalar_kernel<<<grid_for(rows), 256, 0, st>>>(degree, rows, 1u);
      PK_LAUNCH("rmat degree self loop");
    }
    PK_CUDA(cudaStreamSynchronize(st));
  });
}

int pk_invert_permutation(const uint32_t* perm, int64_t n, uint32_t* inv, void* stream) {
  return guard([&] {
    if (n <= 0) return;
    invert_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(perm, static_cast<u64>(n), inv);
    PK_LAUNCH("invert permutation");
  });
}

int pk_rmat_block(const pk_rmat_spec* spec, int parity, const uint32_t* row_perm,
                  const uint32_t* col_perm, const uint32_t* inv_row, const uint32_t* inv_col,
                  const uint32_t* norm_degree, int64_t r0, int64_t r1, int64_t c0, int64_t c1,
                  pk_csr_owned* out, void* stream) {
  return guard([&] {
    check(spec && out, "rmat block: null argument");
    const RmatDev s = to_dev(*spec);
    const i64 n = i64{1} << s.scale;
    check(0 <= r0 && r0 <= r1 && r1 <= n && 0 <= c0 && c0 <= c1 && c1 <= n,
          "rmat block: range out of bounds");
    cudaStream_t st = as_stream(stream);
    // A_even = P_r A P_c^T: rows through row_perm, columns through col_perm;
    // A_odd = P_c A P_r^T the other way round (graph.hpp:139-148)
    const u32* perm_r = parity ? col_perm : row_perm;
    const u32* perm_c = parity ? row_perm : col_perm;
    BlockMap m;
    m.inv_r = parity ? inv_col : inv_row;
    m.inv_c = parity ? inv_row : inv_col;
    m.r0 = static_cast<u32>(r0), m.r1 = static_cast<u32>(r1);
    m.c0 = static_cast<u32>(c0), m.c1 = static_cast<u32>(c1);
    const i64 rows = r1 - r0;
    DevBuf<u64> keys;
    const u64 k = collect_unique(
        [&](u64* o, unsigned long long* cnt) {
          block_keys_kernel<<<grid_for(s.edges), 256, 0, st>>>(s, m, o, cnt);
          PK_LAUNCH("rmat block keys");
          self_loop_keys_kernel<<<grid_for(n), 256, 0, st>>>(static_cast<u64>(n), m, o, cnt);
          PK_LAUNCH("rmat block self loops");
        },
        32 + bits_for(static_cast<u64>(std::max<i64>(rows, 1))), keys, st);
    pk_csr_owned res{};
    res.rows = rows, res.cols = c1 - c0, res.nnz = k;
    res.row_ptr = static_cast<u64*>(dev_alloc((rows + 1) * sizeof(u64)));
    res.col_idx = static_cast<u32*>(dev_alloc(std::max<u64>(k, 1) * sizeof(u32)));
    res.values = static_cast<float*>(dev_alloc(std::max<u64>(k, 1) * sizeof(float)));
    PK_CUDA(cudaMemsetAsync(res.row_ptr, 0, (rows + 1) * sizeof(u64), st));
    if (k) {
      row_counts_u64_kernel<<<grid_for(k), 256, 0, st>>>(keys.p, k, res.row_ptr);
      PK_LAUNCH("rmat block row counts");
      cub_run([&](void* t, size_t& b) {
        return cub::DeviceScan::InclusiveSum(t, b, res.row_ptr, res.row_ptr, rows + 1, st);
      }, st);
      block_entries_kernel<<<grid_for(k), 256, 0, st>>>(keys.p, k, perm_r, perm_c, m.r0, m.c0,
                                                         norm_degree, res.col_idx, res.values);
      PK_LAUNCH("rmat block entries");
    }
    PK_CUDA(cudaStreamSynchronize(st));
    *out = res;
  });
}

int pk_rmat_features_permuted(uint64_t seed, int64_t feat_dim, const uint32_t* perm, int64_t r0,
                              int64_t r1, int64_t c0, int64_t c1, float* out, int64_t ldo,
                              void* stream) {
  return guard([&] {
    check(0 <= r0 && r0 <= r1 && 0 <= c0 && c0 <= c1 && c1 <= feat_dim && ldo >= c1 - c0,
          "rmat features: bad slice");
    const u64 total = static_cast<u64>(r1 - r0) * (c1 - c0);
    if (!total) return;
    features_perm_kernel<<<grid_for(total), 256, 0, as_stream(stream)>>>(seed, feat_dim, perm, r0,
                                                                         r1, c0, c1, out, ldo);
    PK_LAUNCH("rmat features permuted");
  });
}

int pk_labels_from_degrees(const uint32_t* label_degree, int64_t n, uint32_t classes,
                           uint32_t* labels, void* stream) {
  return guard([&] {
    check(classes >= 1, "synth: need at least one class");
    if (n <= 0) return;
    cudaStream_t st = as_stream(stream);
    DevBuf<u64> k(n), ks(n);
    degree_id_keys_kernel<<<grid_for(n), 256, 0, st>>>(label_degree, n, k.p);
    PK_LAUNCH("label order keys");
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortKeys(t, b, k.p, ks.p, n, 0, 64, st);
    }, st);
    assign_labels_kernel<<<grid_for(n), 256, 0, st>>>(ks.p, static_cast<u64>(n), classes, labels);
    PK_LAUNCH("assign labels");
    PK_CUDA(cudaStreamSynchronize(st));
  });
}

int pk_gather_u32(const uint32_t* src, const uint32_t* idx, int64_t n, uint32_t* out,
                  void* stream) {
  return guard([&] {
    if (n <= 0) return;
    gather_u32_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(src, idx, static_cast<u64>(n),
                                                                  out);
    PK_LAUNCH("gather u32");
  });
}

}  // extern "C"

// ---------------------------------------------------------------------------
// preprocess' attribute alignment (graph.hpp:373-380) and balance_metric
// (graph.hpp:157-172) on the device

namespace pk {
namespace {

__global__ void gather_rows_kernel(const float* __restrict__ src, i64 ld_src,
                                   const u32* __restrict__ idx, i64 n, i64 cols,
                                   float* __restrict__ dst, i64 ld_dst) {
  const u64 total = static_cast<u64>(n) * cols;
  for (u64 t = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<u64>(gridDim.x) * blockDim.x) {
    const i64 i = static_cast<i64>(t / cols), j = static_cast<i64>(t % cols);
    dst[i * ld_dst + j] = src[static_cast<i64>(idx[i]) * ld_src + j];
  }
}

__global__ void gather_u8_kernel(const u8* __restrict__ src, const u32* __restrict__ idx, u64 n,
                                 u8* __restrict__ out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = src[idx[i]];
}

// chunk_index (graph.hpp:150-155)
__device__ __forceinline__ u64 chunk_of(u64 total, u64 parts, u64 pos) {
  const u64 base = total / parts, rem = total % parts;
  if (pos < rem * (base + 1)) return pos / (base + 1);
  return rem + (pos - rem * (base + 1)) / (base > 0 ? base : 1);
}

__global__ void block_nnz_kernel(const u64* __restrict__ rp, const u32* __restrict__ ci, u64 rows,
                                 u64 cols, int p, int q, unsigned long long* __restrict__ counts) {
  for (u64 r = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 bi = chunk_of(rows, p, r);
    for (u64 k = rp[r]; k < rp[r + 1]; ++k)
      atomicAdd(&counts[bi * q + chunk_of(cols, q, ci[k])], 1ull);
  }
}

}  // namespace
}  // namespace pk

extern "C" {

int pk_gather_rows_f32(const float* src, int64_t ld_src, const uint32_t* idx, int64_t n,
                       int64_t cols, float* dst, int64_t ld_dst, void* stream) {
  return guard([&] {
    if (n <= 0 || cols <= 0) return;
    gather_rows_kernel<<<grid_for(static_cast<u64>(n) * cols), 256, 0, as_stream(stream)>>>(
        src, ld_src, idx, n, cols, dst, ld_dst);
    PK_LAUNCH("gather rows");
  });
}

int pk_gather_u8(const uint8_t* src, const uint32_t* idx, int64_t n, uint8_t* out, void* stream) {
  return guard([&] {
    if (n <= 0) return;
    gather_u8_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(src, idx, static_cast<u64>(n),
                                                               out);
    PK_LAUNCH("gather u8");
  });
}

int pk_balance_metric(const pk_csr* a, int p, int q, double* out_host, void* stream) {
  return guard([&] {
    check(p >= 1 && q >= 1, "balance_metric: p and q must be >= 1");
    check(a && a->nnz > 0, "balance_metric: matrix has no nonzeros");
    cudaStream_t st = as_stream(stream);
    const size_t nb = static_cast<size_t>(p) * q;
    DevBuf<unsigned long long> counts(nb);
    PK_CUDA(cudaMemsetAsync(counts.p, 0, nb * sizeof(unsigned long long), st));
    block_nnz_kernel<<<grid_for(a->rows), 256, 0, st>>>(a->row_ptr, a->col_idx,
                                                        static_cast<u64>(a->rows),
                                                        static_cast<u64>(a->cols), p, q, counts.p);
    PK_LAUNCH("balance block counts");
    std::vector<unsigned long long> h(nb);
    PK_CUDA(cudaMemcpyAsync(h.data(), counts.p, nb * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    const unsigned long long mx = *std::max_element(h.begin(), h.end());
    *out_host = static_cast<double>(mx) / (static_cast<double>(a->nnz) / static_cast<double>(nb));
  });
}

}  // extern "C"
