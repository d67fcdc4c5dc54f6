// GPU shard builder: the reference's graph preprocessing and CSR
// restructuring, bit-exact (integer work + one IEEE double expression).
//
//   normalize_adjacency (graph.hpp:40-76): u64 keys (u<<32|v), both
//     directions when undirected, plus self loops -> radix sort -> unique ->
//     degree histogram -> row_ptr scan -> value (float)(1/sqrt(du*dv)) in
//     IEEE double (device sqrt/div are correctly rounded without fast-math).
//   permute_csr (graph.hpp:101-131): key (inv_r<<32 | inv_c) is unique per
//     entry, so a radix sort by key reproduces the reference's std::sort on
//     (r, c) exactly.
//   CsrMatrix::transpose (csr.hpp:78-95): stable radix sort of column ids
//     (LSD radix sort is stable, so ties keep row order = counting-sort
//     order of the reference).
//   CsrMatrix::block (csr.hpp:97-120): entry flags + exclusive scan; the
//     compaction keeps the original order.
//
// These run once per dataset / shard (setup), so they favour simplicity:
// one CUB call per step, temporaries sized per call.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <cmath>

#include "pk_common.cuh"
#include "shard_builder.cuh"

namespace pk {

namespace {

int bits_for(u64 maxval) {
  int b = 1;
  while (b < 64 && (maxval >> b) != 0) ++b;
  return b;
}

template <typename F>
void cub_call(F&& f, cudaStream_t st) {
  size_t bytes = 0;
  PK_CUDA(f(nullptr, bytes));
  DevBuf<unsigned char> tmp(bytes ? bytes : 1);
  PK_CUDA(f(tmp.p, bytes));
  (void)st;
  PK_CUDA(cudaStreamSynchronize(st));  // tmp is released at scope exit
}

unsigned grid_for(u64 n) {
  return static_cast<unsigned>(std::max<u64>(1, std::min<u64>((n + 255) / 256, 1u << 20)));
}

// row id of every entry: count row starts landing on each position, then an
// inclusive scan (rows with no entries contribute nothing).
__global__ void row_start_marks(const u64* rp, i64 rows, u64 base, u64 nnz, u32* marks) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x + 1; i < rows;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const u64 p = rp[i] - base;
    if (p < nnz) atomicAdd(&marks[p], 1u);
  }
}

__global__ void histogram_u32(const u32* keys, u64 n, u64* counts) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&counts[keys[i]]), 1ull);
}

__global__ void histogram_hi(const u64* keys, u64 n, u64* counts) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&counts[keys[i] >> 32]), 1ull);
}

__global__ void iota_u32(u32* p, u64 n) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    p[i] = static_cast<u32>(i);
}

__global__ void transpose_scatter(const u32* perm, const u32* rows, const float* val, u64 n,
                                  u32* oci, float* ov) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 src = perm[i];
    oci[i] = rows[src];
    ov[i] = val[src];
  }
}

// ------------------------------------------------------------------------

// Expands row_ptr into per-entry row ids for entries [rp[r0], rp[r1]).
DevBuf<u32> expand_rows(const pk_csr& a, i64 r0, i64 r1, cudaStream_t st) {
  u64 b = 0, e = 0;
  PK_CUDA(cudaMemcpyAsync(&b, a.row_ptr + r0, sizeof(u64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaMemcpyAsync(&e, a.row_ptr + r1, sizeof(u64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  const u64 n = e - b;
  DevBuf<u32> marks(n ? n : 1);
  PK_CUDA(cudaMemsetAsync(marks.p, 0, marks.n * sizeof(u32), st));
  if (r1 - r0 > 1 && n) {
    row_start_marks<<<grid_for(r1 - r0), 256, 0, st>>>(a.row_ptr + r0, r1 - r0, b, n, marks.p);
    PK_LAUNCH("row start marks");
  }
  DevBuf<u32> rows(n ? n : 1);
  if (n)
    cub_call([&](void* t, size_t& bytes) {
      return cub::DeviceScan::InclusiveSum(t, bytes, marks.p, rows.p, static_cast<i64>(n), st);
    }, st);
  return rows;  // local row index (0 = r0)
}

void alloc_owned(pk_csr_owned* out, i64 rows, i64 cols, u64 nnz) {
  out->rows = rows;
  out->cols = cols;
  out->nnz = nnz;
  out->row_ptr = nullptr;
  out->col_idx = nullptr;
  out->values = nullptr;
  out->row_ptr = static_cast<u64*>(dev_alloc((rows + 1) * sizeof(u64)));
  if (nnz) {
    out->col_idx = static_cast<u32*>(dev_alloc(nnz * sizeof(u32)));
    out->values = static_cast<float*>(dev_alloc(nnz * sizeof(float)));
  }
}

// counts[0..len) -> exclusive prefix into row_ptr[0..len] (row_ptr[len] = total)
void counts_to_row_ptr(u64* counts, i64 len, u64* row_ptr, cudaStream_t st) {
  // counts has len+1 slots with counts[len] = 0, so the exclusive scan's last
  // element is the total.
  cub_call([&](void* t, size_t& bytes) {
    return cub::DeviceScan::ExclusiveSum(t, bytes, counts, row_ptr, static_cast<i64>(len + 1), st);
  }, st);
}

__global__ void rebase_row_ptr(const u64* rp, i64 count, u64 base, u64* out) {
  const i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (i < count) out[i] = rp[i] - base;
}

__global__ void block_flags(const u32* ci, u64 n, u32 c0, u32 c1, u32* flags) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    flags[i] = (ci[i] >= c0 && ci[i] < c1) ? 1u : 0u;
}

__global__ void block_row_ptr(const u64* rp, i64 r0, i64 rows, u64 base, const u64* pos,
                              u64 total, u64* orp) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i <= rows;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const u64 p = rp[r0 + i] - base;
    orp[i] = i == rows ? total : pos[p];
  }
}

__global__ void block_scatter(const u32* ci, const float* v, const u32* flags, const u64* pos,
                              u64 n, u32 c0, u32* oci, float* ov) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    if (flags[i]) {
      oci[pos[i]] = ci[i] - c0;
      ov[pos[i]] = v[i];
    }
}

__global__ void edge_keys(const u32* uv, u64 m, i64 n, int undirected, u64* keys) {
  const u64 stride = undirected ? 2 : 1;
  for (u64 e = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; e < m + n;
       e += static_cast<u64>(gridDim.x) * blockDim.x) {
    if (e < m) {
      const u64 u = uv[2 * e], v = uv[2 * e + 1];
      keys[stride * e] = (u << 32) | v;
      if (undirected) keys[stride * e + 1] = (v << 32) | u;
    } else {
      const u64 u = e - m;  // self loop
      keys[stride * m + u] = (u << 32) | u;
    }
  }
}

__global__ void normalize_values(const u64* keys, u64 nnz, const u64* degree, u32* ci,
                                 float* val) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 k = keys[i];
    const u32 u = static_cast<u32>(k >> 32), v = static_cast<u32>(k);
    ci[i] = v;
    // graph.hpp:71-72, IEEE double sqrt and division
    const double prod = __dmul_rn(static_cast<double>(degree[u]), static_cast<double>(degree[v]));
    val[i] = __double2float_rn(__ddiv_rn(1.0, __dsqrt_rn(prod)));
  }
}

__global__ void invert_perm(const u32* p, i64 n, u32* inv) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    inv[p[i]] = static_cast<u32>(i);
}

__global__ void permute_keys(const u32* rows, const u32* ci, u64 nnz, const u32* inv_r,
                             const u32* inv_c, u64* keys) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    keys[i] = (static_cast<u64>(inv_r[rows[i]]) << 32) | inv_c[ci[i]];
}

__global__ void low_words(const u64* keys, u64 n, u32* out) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    out[i] = static_cast<u32>(keys[i]);
}

}  // namespace

void csr_transpose(const pk_csr& a, pk_csr_owned* out, cudaStream_t st) {
  alloc_owned(out, a.cols, a.rows, a.nnz);
  const u64 n = a.nnz;
  // temporaries from the per-thread scratch arena (row ids, iota, sorted
  // keys, permutation, counts, cub workspaces): nothing to allocate per call
  Scratch& sc = Scratch::get();
  auto cub_temp = [&](auto&& f) {  // cub call with its workspace in the arena
    size_t bytes = 0;
    PK_CUDA(f(nullptr, bytes));
    const size_t m = sc.mark();
    PK_CUDA(f(sc.take<unsigned char>(bytes), bytes));
    PK_CUDA(cudaStreamSynchronize(st));
    sc.release_to(m);
  };
  size_t sort_bytes = 0;
  if (n)
    PK_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, a.col_idx, (u32*)nullptr,
                                            (u32*)nullptr, (u32*)nullptr, static_cast<i64>(n),
                                            0, 32, st));
  sc.reset(5 * (n + 1) * sizeof(u32) + (a.cols + 1) * sizeof(u64) + sort_bytes +
           (size_t{64} << 20));
  u64* counts = sc.take<u64>(a.cols + 1);
  PK_CUDA(cudaMemsetAsync(counts, 0, (a.cols + 1) * sizeof(u64), st));
  if (n) {
    histogram_u32<<<grid_for(n), 256, 0, st>>>(a.col_idx, n, counts);
    PK_LAUNCH("transpose histogram");
  }
  cub_temp([&](void* t, size_t& bytes) {
    return cub::DeviceScan::ExclusiveSum(t, bytes, counts, out->row_ptr,
                                         static_cast<i64>(a.cols + 1), st);
  });
  if (!n) return;
  // row id of every entry (expand_rows, in the arena)
  u32* marks = sc.take<u32>(n);
  u32* rows = sc.take<u32>(n);
  PK_CUDA(cudaMemsetAsync(marks, 0, n * sizeof(u32), st));
  if (a.rows > 1) {
    u64 base = 0;
    PK_CUDA(cudaMemcpyAsync(&base, a.row_ptr, sizeof(u64), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    row_start_marks<<<grid_for(a.rows), 256, 0, st>>>(a.row_ptr, a.rows, base, n, marks);
    PK_LAUNCH("row start marks");
  }
  cub_temp([&](void* t, size_t& bytes) {
    return cub::DeviceScan::InclusiveSum(t, bytes, marks, rows, static_cast<i64>(n), st);
  });
  u32* idx = sc.take<u32>(n);
  u32* keys_out = sc.take<u32>(n);
  u32* perm = sc.take<u32>(n);
  iota_u32<<<grid_for(n), 256, 0, st>>>(idx, n);
  PK_LAUNCH("iota");
  const int end_bit = bits_for(a.cols > 0 ? a.cols - 1 : 0);
  cub_temp([&](void* t, size_t& bytes) {
    return cub::DeviceRadixSort::SortPairs(t, bytes, a.col_idx, keys_out, idx, perm,
                                           static_cast<i64>(n), 0, end_bit, st);
  });
  transpose_scatter<<<grid_for(n), 256, 0, st>>>(perm, rows, a.values, n, out->col_idx,
                                                 out->values);
  PK_LAUNCH("transpose scatter");
  PK_CUDA(cudaStreamSynchronize(st));
}

void csr_block(const pk_csr& a, i64 r0, i64 r1, i64 c0, i64 c1, pk_csr_owned* out,
               cudaStream_t st) {
  check(r0 >= 0 && r0 <= r1 && r1 <= a.rows && c0 >= 0 && c0 <= c1 && c1 <= a.cols,
        "csr block: range out of bounds");
  u64 b = 0, e = 0;
  PK_CUDA(cudaMemcpyAsync(&b, a.row_ptr + r0, sizeof(u64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaMemcpyAsync(&e, a.row_ptr + r1, sizeof(u64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  const u64 n = e - b;
  if (c0 == 0 && c1 == a.cols) {
    // every column kept (the inner axis is one rank): a row range is a plain
    // copy with the row pointers rebased
    alloc_owned(out, r1 - r0, c1 - c0, n);
    rebase_row_ptr<<<grid_for(r1 - r0 + 1), 256, 0, st>>>(a.row_ptr + r0, r1 - r0 + 1, b,
                                                          out->row_ptr);
    PK_LAUNCH("block row_ptr rebase");
    if (n) {
      PK_CUDA(cudaMemcpyAsync(out->col_idx, a.col_idx + b, n * sizeof(u32),
                              cudaMemcpyDeviceToDevice, st));
      PK_CUDA(cudaMemcpyAsync(out->values, a.values + b, n * sizeof(float),
                              cudaMemcpyDeviceToDevice, st));
    }
    PK_CUDA(cudaStreamSynchronize(st));
    return;
  }
  DevBuf<u32> flags(n ? n : 1);
  DevBuf<u64> pos(n + 1);
  u64 total = 0;
  if (n) {
    block_flags<<<grid_for(n), 256, 0, st>>>(a.col_idx + b, n, static_cast<u32>(c0),
                                             static_cast<u32>(c1), flags.p);
    PK_LAUNCH("block flags");
    cub_call([&](void* t, size_t& bytes) {
      return cub::DeviceScan::ExclusiveSum(t, bytes, flags.p, pos.p, static_cast<i64>(n), st);
    }, st);
    u64 last_pos = 0;
    u32 last_flag = 0;
    PK_CUDA(cudaMemcpyAsync(&last_pos, pos.p + n - 1, sizeof(u64), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaMemcpyAsync(&last_flag, flags.p + n - 1, sizeof(u32), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    total = last_pos + last_flag;
  }
  PK_CUDA(cudaMemcpyAsync(pos.p + n, &total, sizeof(u64), cudaMemcpyHostToDevice, st));
  alloc_owned(out, r1 - r0, c1 - c0, total);
  block_row_ptr<<<grid_for(r1 - r0 + 1), 256, 0, st>>>(a.row_ptr, r0, r1 - r0, b, pos.p, total,
                                                       out->row_ptr);
  PK_LAUNCH("block row_ptr");
  if (total) {
    block_scatter<<<grid_for(n), 256, 0, st>>>(a.col_idx + b, a.values + b, flags.p, pos.p, n,
                                               static_cast<u32>(c0), out->col_idx, out->values);
    PK_LAUNCH("block scatter");
  }
  PK_CUDA(cudaStreamSynchronize(st));
}

void normalize_adjacency(i64 n, const u32* uv, u64 m, bool undirected, pk_csr_owned* out,
                         cudaStream_t st) {
  check(n >= 1, "normalize_adjacency: n must be >= 1");
  const u64 nk = (undirected ? 2 * m : m) + static_cast<u64>(n);
  DevBuf<u64> keys(nk), sorted(nk);
  edge_keys<<<grid_for(m + n), 256, 0, st>>>(uv, m, n, undirected ? 1 : 0, keys.p);
  PK_LAUNCH("edge keys");
  const int end_bit = 32 + bits_for(static_cast<u64>(n - 1));
  cub_call([&](void* t, size_t& bytes) {
    return cub::DeviceRadixSort::SortKeys(t, bytes, keys.p, sorted.p, static_cast<i64>(nk), 0,
                                          end_bit, st);
  }, st);
  DevBuf<i64> nsel(1);
  cub_call([&](void* t, size_t& bytes) {
    return cub::DeviceSelect::Unique(t, bytes, sorted.p, keys.p, nsel.p, static_cast<i64>(nk), st);
  }, st);
  i64 nnz = 0;
  PK_CUDA(cudaMemcpyAsync(&nnz, nsel.p, sizeof(i64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  sorted.release();
  DevBuf<u64> degree(n + 1);
  PK_CUDA(cudaMemsetAsync(degree.p, 0, degree.n * sizeof(u64), st));
  histogram_hi<<<grid_for(nnz), 256, 0, st>>>(keys.p, nnz, degree.p);
  PK_LAUNCH("degree histogram");
  alloc_owned(out, n, n, static_cast<u64>(nnz));
  counts_to_row_ptr(degree.p, n, out->row_ptr, st);
  normalize_values<<<grid_for(nnz), 256, 0, st>>>(keys.p, nnz, degree.p, out->col_idx,
                                                  out->values);
  PK_LAUNCH("normalize values");
  PK_CUDA(cudaStreamSynchronize(st));
}

void permute_csr(const pk_csr& a, const u32* row_perm, const u32* col_perm, pk_csr_owned* out,
                 cudaStream_t st) {
  check(a.rows == a.cols, "permute_csr: matrix must be square");
  const i64 n = a.rows;
  const u64 nnz = a.nnz;
  DevBuf<u32> inv_r(n), inv_c(n);
  invert_perm<<<grid_for(n), 256, 0, st>>>(row_perm, n, inv_r.p);
  invert_perm<<<grid_for(n), 256, 0, st>>>(col_perm, n, inv_c.p);
  PK_LAUNCH("invert permutation");
  alloc_owned(out, n, n, nnz);
  DevBuf<u64> counts(n + 1);
  PK_CUDA(cudaMemsetAsync(counts.p, 0, counts.n * sizeof(u64), st));
  if (nnz) {
    DevBuf<u64> keys(nnz), sorted(nnz);
    {
      DevBuf<u32> rows = expand_rows(a, 0, n, st);
      permute_keys<<<grid_for(nnz), 256, 0, st>>>(rows.p, a.col_idx, nnz, inv_r.p, inv_c.p,
                                                  keys.p);
      PK_LAUNCH("permute keys");
      PK_CUDA(cudaStreamSynchronize(st));
    }
    const int end_bit = 32 + bits_for(static_cast<u64>(n - 1));
    cub_call([&](void* t, size_t& bytes) {
      return cub::DeviceRadixSort::SortPairs(t, bytes, keys.p, sorted.p, a.values, out->values,
                                             static_cast<i64>(nnz), 0, end_bit, st);
    }, st);
    histogram_hi<<<grid_for(nnz), 256, 0, st>>>(sorted.p, nnz, counts.p);
    PK_LAUNCH("permute histogram");
    low_words<<<grid_for(nnz), 256, 0, st>>>(sorted.p, nnz, out->col_idx);
    PK_LAUNCH("permute columns");
  }
  counts_to_row_ptr(counts.p, n, out->row_ptr, st);
  PK_CUDA(cudaStreamSynchronize(st));
}

// ---------------------------------------------------------------------------
// row merge of column pieces (load_rank_shards' assemble_csr,
// trainer.hpp:276-309): columns within a piece row ascend, so the entries
// that fall in [c0, c1) are one contiguous run found by two binary searches

constexpr int kMaxPieces = 64;

struct Pieces {
  const u64* rp[kMaxPieces];
  const u32* ci[kMaxPieces];
  const float* v[kMaxPieces];
  u64 col0[kMaxPieces];
  int count;
};

__device__ u64 lower_bound_col(const u32* ci, u64 lo, u64 hi, u64 key) {
  while (lo < hi) {
    const u64 mid = lo + (hi - lo) / 2;
    if (ci[mid] < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// the run of piece k's row r whose global column is in [c0, c1)
__device__ void piece_run(const Pieces& P, int k, i64 r, u64 c0, u64 c1, u64& lo, u64& hi) {
  const u64 b = P.rp[k][r], e = P.rp[k][r + 1];
  const u64 o = P.col0[k];
  const u64 klo = c0 > o ? c0 - o : 0, khi = c1 > o ? c1 - o : 0;
  lo = lower_bound_col(P.ci[k], b, e, klo);
  hi = lower_bound_col(P.ci[k], lo, e, khi);
}

__global__ void hconcat_count(Pieces P, i64 rows, u64 c0, u64 c1, u64* counts) {
  for (i64 r = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<i64>(gridDim.x) * blockDim.x) {
    u64 total = 0;
    for (int k = 0; k < P.count; ++k) {
      u64 lo, hi;
      piece_run(P, k, r, c0, c1, lo, hi);
      total += hi - lo;
    }
    counts[r] = total;
  }
}

// one warp per row: runs copied in piece order, lanes over entries
__global__ void hconcat_fill(Pieces P, i64 rows, u64 c0, u64 c1, const u64* out_rp,
                             u32* out_ci, float* out_v) {
  const int lane = threadIdx.x % 32;
  const i64 warps = static_cast<i64>(gridDim.x) * (blockDim.x / 32);
  for (i64 r = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) / 32; r < rows;
       r += warps) {
    u64 pos = out_rp[r];
    for (int k = 0; k < P.count; ++k) {
      u64 lo, hi;
      piece_run(P, k, r, c0, c1, lo, hi);
      const u64 shift = P.col0[k] - c0;  // global = col0 + local; out = global - c0
      for (u64 i = lo + lane; i < hi; i += 32) {
        out_ci[pos + (i - lo)] = static_cast<u32>(P.ci[k][i] + shift);
        out_v[pos + (i - lo)] = P.v[k][i];
      }
      pos += hi - lo;
    }
  }
}

void csr_hconcat(const pk_csr* pieces, const u64* col0, int count, u64 c0, u64 c1,
                 pk_csr_owned* out, cudaStream_t st) {
  check(count >= 1 && count <= kMaxPieces, "csr hconcat: 1.." + std::to_string(kMaxPieces) +
                                               " pieces");
  check(c0 <= c1, "csr hconcat: empty column range");
  const i64 rows = pieces[0].rows;
  Pieces P{};
  P.count = count;
  for (int k = 0; k < count; ++k) {
    check(pieces[k].rows == rows, "csr hconcat: pieces must hold the same rows");
    check(col0[k] <= c0 || col0[k] - c0 < (u64{1} << 32), "csr hconcat: column origin");
    P.rp[k] = pieces[k].row_ptr;
    P.ci[k] = pieces[k].col_idx;
    P.v[k] = pieces[k].values;
    P.col0[k] = col0[k];
  }
  DevBuf<u64> counts(rows + 1);
  PK_CUDA(cudaMemsetAsync(counts.p + rows, 0, sizeof(u64), st));
  if (rows) {
    hconcat_count<<<grid_for(rows), 256, 0, st>>>(P, rows, c0, c1, counts.p);
    PK_LAUNCH("hconcat count");
  }
  DevBuf<u64> rp(rows + 1);
  counts_to_row_ptr(counts.p, rows, rp.p, st);
  u64 nnz = 0;
  PK_CUDA(cudaMemcpyAsync(&nnz, rp.p + rows, sizeof(u64), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  alloc_owned(out, rows, static_cast<i64>(c1 - c0), nnz);
  PK_CUDA(cudaMemcpyAsync(out->row_ptr, rp.p, (rows + 1) * sizeof(u64),
                          cudaMemcpyDeviceToDevice, st));
  if (rows && nnz) {
    hconcat_fill<<<grid_for(rows * 32), 256, 0, st>>>(P, rows, c0, c1, out->row_ptr,
                                                      out->col_idx, out->values);
    PK_LAUNCH("hconcat fill");
  }
  PK_CUDA(cudaStreamSynchronize(st));
}

void csr_free(pk_csr_owned* m) {
  if (!m) return;
  if (m->row_ptr) dev_free(m->row_ptr);
  if (m->col_idx) dev_free(m->col_idx);
  if (m->values) dev_free(m->values);
  m->row_ptr = nullptr;
  m->col_idx = nullptr;
  m->values = nullptr;
  m->rows = m->cols = 0;
  m->nnz = 0;
}

}  // namespace pk
