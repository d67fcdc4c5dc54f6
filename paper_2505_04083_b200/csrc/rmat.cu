// Device synthetic-graph generator, bit-exact with the reference's
// synth_rmat / assemble_synth (graph.hpp:197-322).
//
// Edge e consumes u64 draws e*scale .. e*scale+scale-1 of Philox(seed, 5)
// (no rejection anywhere), so each thread derives its own draws in closed
// form (philox.cuh). Self loops are dropped with a stable compaction, which
// keeps the reference's edge order.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include "philox.cuh"
#include "pk_common.cuh"
#include "shard_builder.cuh"

namespace pk {

namespace {

unsigned grid_for(u64 n) {
  return static_cast<unsigned>(std::max<u64>(1, std::min<u64>((n + 255) / 256, 1u << 20)));
}

// One thread per edge. Draws of an edge share Philox blocks pairwise, so a
// thread computes each block once.
__global__ void rmat_kernel(u64 edges, int scale, double a, double ab, double abc, u64 seed,
                            u64* packed, u8* keep) {
  for (u64 e = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; e < edges;
       e += static_cast<u64>(gridDim.x) * blockDim.x) {
    u32 u = 0, v = 0;
    u64 t = e * static_cast<u64>(scale);
    u64 cur_block = ~0ull;
    Philox4 blk{};
    for (int bit = 0; bit < scale; ++bit, ++t) {
      if ((t >> 1) != cur_block) {
        cur_block = t >> 1;
        blk = philox_at(seed, 5, cur_block);
      }
      const int s = static_cast<int>(t & 1) * 2;
      const u64 x = static_cast<u64>(blk.v[s]) | (static_cast<u64>(blk.v[s + 1]) << 32);
      const double r = u64_to_unit(x);
      u <<= 1;
      v <<= 1;
      // graph.hpp:308-316; a+b and a+b+c formed on the host in the same order
      if (r < a) {
      } else if (r < ab) {
        v |= 1;
      } else if (r < abc) {
        u |= 1;
      } else {
        u |= 1;
        v |= 1;
      }
    }
    // little-endian: u64 (v << 32 | u) is the u32 pair [u, v]
    packed[e] = (static_cast<u64>(v) << 32) | u;
    keep[e] = u != v ? 1 : 0;
  }
}

__global__ void features_kernel(u64 seed, i64 n, i64 d, float* out, i64 ldo) {
  const u64 total = static_cast<u64>(n) * d;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const double x = u64_to_unit(philox_u64_at(seed, 3, i));
    out[(i / d) * ldo + i % d] = static_cast<float>(x);
  }
}

__global__ void label_keys(const u32* uv, u64 m, u64* keys, u8* keep) {
  for (u64 e = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; e < m;
       e += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 u = uv[2 * e], v = uv[2 * e + 1];
    keys[2 * e] = (u << 32) | v;
    keys[2 * e + 1] = (v << 32) | u;
    keep[2 * e] = keep[2 * e + 1] = u != v ? 1 : 0;
  }
}

__global__ void degree_count(const u64* keys, u64 n, u32* degree) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    atomicAdd(&degree[keys[i] >> 32], 1u);
}

__global__ void degree_id_keys(const u32* degree, i64 n, u64* keys) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    keys[i] = (static_cast<u64>(degree[i]) << 32) | static_cast<u64>(i);
}

__global__ void assign_labels(const u64* sorted, i64 n, u32 classes, u32* labels) {
  for (i64 pos = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; pos < n;
       pos += static_cast<i64>(gridDim.x) * blockDim.x) {
    const u32 node = static_cast<u32>(sorted[pos]);
    labels[node] = static_cast<u32>(static_cast<u64>(pos) * classes / static_cast<u64>(n));
  }
}

// chunk_index (graph.hpp:151-155): which of `parts` ceil-split chunks of
// [0, total) holds pos
__device__ __forceinline__ int chunk_index_dev(u64 total, int parts, u64 pos) {
  const u64 base = total / parts, rem = total % parts;
  if (pos < rem * (base + 1)) return static_cast<int>(pos / (base + 1));
  return static_cast<int>(rem + (pos - rem * (base + 1)) / (base > 0 ? base : 1));
}

// synth_sbm / synth_erdos (graph.hpp:254-289): pair (u, v), u < v, in
// lexicographic order consumes u64 draw t(u, v) = sum_{i<u} (n - 1 - i) +
// (v - u - 1) of Philox(seed, 5) and keeps the edge when the draw's unit
// double falls below p_in (same community) or p_out. One warp per row u
// walks v in 32-wide steps; a ballot orders the kept pairs, so the emitted
// edge list is the reference's, in its order. COUNT pass first (per-row
// counts -> exclusive scan), then EMIT.
template <bool EMIT>
__global__ void pair_rows_kernel(u64 n, int communities, double p_in, double p_out, u64 seed,
                                 const u64* __restrict__ offsets, u64* __restrict__ counts,
                                 u64* __restrict__ packed) {
  const int lane = threadIdx.x % 32;
  const u64 warps = static_cast<u64>(gridDim.x) * (blockDim.x / 32);
  for (u64 u = blockIdx.x * static_cast<u64>(blockDim.x / 32) + threadIdx.x / 32; u < n;
       u += warps) {
    const u64 base = u * (n - 1) - u * (u - 1) / 2;  // draws of rows 0 .. u-1
    const int cu = chunk_index_dev(n, communities, u);
    u64 cnt = 0;
    const u64 out0 = EMIT ? offsets[u] : 0;
    for (u64 v0 = u + 1; v0 < n; v0 += 32) {
      const u64 v = v0 + lane;
      bool keep = false;
      if (v < n) {
        const double r = u64_to_unit(philox_u64_at(seed, 5, base + (v - u - 1)));
        keep = r < (chunk_index_dev(n, communities, v) == cu ? p_in : p_out);
      }
      const unsigned ballot = __ballot_sync(0xffffffffu, keep);
      if (EMIT && keep)
        packed[out0 + cnt + __popc(ballot & ((1u << lane) - 1u))] = (v << 32) | u;
      cnt += static_cast<u64>(__popc(ballot));
    }
    if (!EMIT && lane == 0) counts[u] = cnt;
  }
}

template <typename F>
void cub_call(F&& f, cudaStream_t st) {
  size_t bytes = 0;
  PK_CUDA(f(nullptr, bytes));
  DevBuf<unsigned char> tmp(bytes ? bytes : 1);
  PK_CUDA(f(tmp.p, bytes));
  PK_CUDA(cudaStreamSynchronize(st));
}

}  // namespace

u64 rmat_edges(int scale, u64 edges, double a, double b, double c, u64 seed, u32* uv,
               cudaStream_t st) {
  check(scale >= 1 && scale < 31, "rmat: scale out of range");
  check(a > 0 && b >= 0 && c >= 0 && a + b + c < 1.0,
        "rmat: quadrant probabilities must sum below 1");
  if (edges == 0) return 0;
  DevBuf<u64> packed(edges);
  DevBuf<u8> keep(edges);
  rmat_kernel<<<grid_for(edges), 256, 0, st>>>(edges, scale, a, a + b, a + b + c, seed, packed.p,
                                               keep.p);
  PK_LAUNCH("rmat edges");
  DevBuf<i64> nsel(1);
  u64* out = reinterpret_cast<u64*>(uv);
  cub_call([&](void* t, size_t& bytes) {
    return cub::DeviceSelect::Flagged(t, bytes, packed.p, keep.p, out, nsel.p,
                                      static_cast<i64>(edges), st);
  }, st);
  i64 kept = 0;
  PK_CUDA(cudaMemcpyAsync(&kept, nsel.p, sizeof(i64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  return static_cast<u64>(kept);
}

u64 pair_edges(u64 n, int communities, double p_in, double p_out, u64 seed, u32* uv,
               u64 capacity, cudaStream_t st) {
  check(n >= 1, "sbm: n must be >= 1");
  check(communities >= 1 && static_cast<u64>(communities) <= n, "sbm: invalid community count");
  check(p_in >= 0 && p_in <= 1 && p_out >= 0 && p_out <= 1,
        "sbm: probabilities must be in [0,1]");
  check(n < (1ull << 32), "sbm: node ids are u32");
  DevBuf<u64> counts(n), offsets(n);
  const unsigned grid = static_cast<unsigned>(std::max<u64>(1, std::min<u64>((n + 7) / 8, 1u << 20)));
  pair_rows_kernel<false><<<grid, 256, 0, st>>>(n, communities, p_in, p_out, seed, nullptr,
                                                 counts.p, nullptr);
  PK_LAUNCH("pair edges count");
  cub_call([&](void* t, size_t& bytes) {
    return cub::DeviceScan::ExclusiveSum(t, bytes, counts.p, offsets.p, static_cast<i64>(n), st);
  }, st);
  u64 last[2] = {0, 0};
  PK_CUDA(cudaMemcpyAsync(&last[0], offsets.p + (n - 1), sizeof(u64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaMemcpyAsync(&last[1], counts.p + (n - 1), sizeof(u64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  const u64 total = last[0] + last[1];
  if (uv == nullptr) return total;
  check(total <= capacity, "sbm: edge buffer too small (" + std::to_string(total) + " edges)");
  pair_rows_kernel<true><<<grid, 256, 0, st>>>(n, communities, p_in, p_out, seed, offsets.p,
                                                nullptr, reinterpret_cast<u64*>(uv));
  PK_LAUNCH("pair edges emit");
  PK_CUDA(cudaStreamSynchronize(st));
  return total;
}

void rmat_features(u64 seed, i64 n, i64 d, float* out, i64 ldo, cudaStream_t st) {
  if (n * d == 0) return;
  features_kernel<<<grid_for(static_cast<u64>(n) * d), 256, 0, st>>>(seed, n, d, out, ldo);
  PK_LAUNCH("rmat features");
}

void degree_quantile_labels(const u32* uv, u64 m, i64 n, u32 classes, u32* labels,
                            cudaStream_t st) {
  check(classes >= 1, "synth: need at least one class");
  DevBuf<u32> degree(n);
  PK_CUDA(cudaMemsetAsync(degree.p, 0, n * sizeof(u32), st));
  if (m) {
    DevBuf<u64> keys(2 * m), sel(2 * m);
    DevBuf<u8> keep(2 * m);
    DevBuf<i64> nsel(1);
    label_keys<<<grid_for(m), 256, 0, st>>>(uv, m, keys.p, keep.p);
    PK_LAUNCH("label keys");
    cub_call([&](void* t, size_t& bytes) {
      return cub::DeviceSelect::Flagged(t, bytes, keys.p, keep.p, sel.p, nsel.p,
                                        static_cast<i64>(2 * m), st);
    }, st);
    i64 k = 0;
    PK_CUDA(cudaMemcpyAsync(&k, nsel.p, sizeof(i64), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    cub_call([&](void* t, size_t& bytes) {
      return cub::DeviceRadixSort::SortKeys(t, bytes, sel.p, keys.p, k, 0, 64, st);
    }, st);
    cub_call([&](void* t, size_t& bytes) {
      return cub::DeviceSelect::Unique(t, bytes, keys.p, sel.p, nsel.p, k, st);
    }, st);
    PK_CUDA(cudaMemcpyAsync(&k, nsel.p, sizeof(i64), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    degree_count<<<grid_for(k), 256, 0, st>>>(sel.p, k, degree.p);
    PK_LAUNCH("label degree");
  }
  // order nodes by (distinct-neighbour degree, id): unique composite keys
  DevBuf<u64> dk(n), ds(n);
  degree_id_keys<<<grid_for(n), 256, 0, st>>>(degree.p, n, dk.p);
  PK_LAUNCH("label order keys");
  cub_call([&](void* t, size_t& bytes) {
    return cub::DeviceRadixSort::SortKeys(t, bytes, dk.p, ds.p, n, 0, 64, st);
  }, st);
  assign_labels<<<grid_for(n), 256, 0, st>>>(ds.p, n, classes, labels);
  PK_LAUNCH("assign labels");
  PK_CUDA(cudaStreamSynchronize(st));
}

}  // namespace pk
