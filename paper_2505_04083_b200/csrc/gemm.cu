// Dense transform GEMMs of the GCN layer (kernels.hpp:64-92):
//   forward  Q  = H . W            (NN, engine.hpp:198)
//   backward dW = (dQ^T . H)^T     (TN, engine.hpp:233-235; K = adjacency rows)
//            dH = dQ . W^T         (NT, engine.hpp:242)
//
// PARITY mode: one thread owns a 4x4 register tile of C, operands staged in
// shared memory, k strictly ascending, acc from +0, __fmul_rn then __fadd_rn
// — the reference's loop (kernels.hpp:84-89) element for element, so C is
// bit-identical. For a tall reduction (dW, small m*n, huge k) the per-element
// chain is inherently sequential; the kernel then uses 1x1 tiles to expose
// m*n independent chains.
//
// FAST mode: the tensor-core kernels in gemm_tc.cu (tcgen05 3xTF32); shapes
// they do not cover fall back to the FFMA SIMT kernel below with a
// deterministic split-K for tall reductions.
#include <cuda_runtime.h>

#include "elementwise.cuh"
#include "gemm.cuh"
#include "pk_common.cuh"

namespace pk {

namespace {

constexpr int kBM = 64, kBN = 64, kBK = 16;

template <bool TA, bool TB, bool EXACT>
__global__ void __launch_bounds__(256)
gemm_simt_kernel(i64 m, i64 n, i64 k_total, i64 k_chunk, const float* __restrict__ a,
                 i64 lda, const float* __restrict__ b, i64 ldb, float* __restrict__ c,
                 i64 ldc) {
  // split z covers k in [z*k_chunk, min(k_total, (z+1)*k_chunk))
  const i64 k_begin = static_cast<i64>(blockIdx.z) * k_chunk;
  const i64 k_end = min(k_total, k_begin + k_chunk);
  __shared__ float as[kBK][kBM + 4];
  __shared__ float bs[kBK][kBN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const i64 m0 = static_cast<i64>(blockIdx.y) * kBM, n0 = static_cast<i64>(blockIdx.x) * kBN;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;

  for (i64 k0 = k_begin; k0 < k_end; k0 += kBK) {
    // stage A tile (kBM x kBK) as as[kk][mm]
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int idx = threadIdx.x + t * 256;
      int mm, kk;
      if (TA) {  // A stored k x m: consecutive threads along m
        mm = idx % kBM, kk = idx / kBM;
      } else {   // A stored m x k: consecutive threads along k
        kk = idx % kBK, mm = idx / kBK;
      }
      const i64 gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < m && gk < k_end) v = TA ? a[gk * lda + gm] : a[gm * lda + gk];
      as[kk][mm] = v;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int idx = threadIdx.x + t * 256;
      int nn, kk;
      if (TB) {  // B stored n x k
        kk = idx % kBK, nn = idx / kBK;
      } else {   // B stored k x n
        nn = idx % kBN, kk = idx / kBN;
      }
      const i64 gn = n0 + nn, gk = k0 + kk;
      float v = 0.f;
      if (gn < n && gk < k_end) v = TB ? b[gn * ldb + gk] : b[gk * ldb + gn];
      bs[kk][nn] = v;
    }
    __syncthreads();
    const int kmax = static_cast<int>(min(static_cast<i64>(kBK), k_end - k0));
    if (kmax == kBK) {
#pragma unroll
      for (int kk = 0; kk < kBK; ++kk) {
        float av[4], bv[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) av[i] = as[kk][ty + 16 * i];
#pragma unroll
        for (int j = 0; j < 4; ++j) bv[j] = bs[kk][tx + 16 * j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j)
            acc[i][j] = EXACT ? __fadd_rn(acc[i][j], __fmul_rn(av[i], bv[j]))
                              : fmaf(av[i], bv[j], acc[i][j]);
      }
    } else {
      for (int kk = 0; kk < kmax; ++kk) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float x = as[kk][ty + 16 * i], y = bs[kk][tx + 16 * j];
            acc[i][j] = EXACT ? __fadd_rn(acc[i][j], __fmul_rn(x, y)) : fmaf(x, y, acc[i][j]);
          }
      }
    }
    __syncthreads();
  }
  const i64 zoff = static_cast<i64>(blockIdx.z) * m * ldc;  // split-K partials
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const i64 gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
      if (gm < m && gn < n) c[zoff + gm * ldc + gn] = acc[i][j];
    }
}

// Tall reduction in parity mode: one thread per C element, k ascending over
// the full K. Operands are staged kTK rows at a time; every thread of the
// block reads the same staged rows (16 x 16 output tile per block).
constexpr int kTK = 64;

template <bool TA, bool TB>
__global__ void __launch_bounds__(256)
gemm_tall_exact_kernel(i64 m, i64 n, i64 k, const float* __restrict__ a, i64 lda,
                       const float* __restrict__ b, i64 ldb, float* __restrict__ c, i64 ldc) {
  __shared__ float as[kTK][17];
  __shared__ float bs[kTK][17];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const i64 m0 = static_cast<i64>(blockIdx.y) * 16, n0 = static_cast<i64>(blockIdx.x) * 16;
  float acc = 0.f;
  for (i64 k0 = 0; k0 < k; k0 += kTK) {
    for (int idx = threadIdx.x; idx < kTK * 16; idx += 256) {
      const int kk = idx / 16, mm = idx % 16;
      const i64 gk = k0 + kk, gm = m0 + mm, gn = n0 + mm;
      float av = 0.f, bv = 0.f;
      if (gk < k) {
        if (gm < m) av = TA ? a[gk * lda + gm] : a[gm * lda + gk];
        if (gn < n) bv = TB ? b[gn * ldb + gk] : b[gk * ldb + gn];
      }
      as[kk][mm] = av;
      bs[kk][mm] = bv;
    }
    __syncthreads();
    const int kmax = static_cast<int>(min(static_cast<i64>(kTK), k - k0));
    for (int kk = 0; kk < kmax; ++kk)
      acc = __fadd_rn(acc, __fmul_rn(as[kk][ty], bs[kk][tx]));
    __syncthreads();
  }
  const i64 gm = m0 + ty, gn = n0 + tx;
  if (gm < m && gn < n) c[gm * ldc + gn] = acc;
}

// Deterministic split-K combine: C = sum over splits in ascending order.
__global__ void splitk_reduce_kernel(const float* __restrict__ part, int splits, i64 m, i64 n,
                                     i64 ldp, float* __restrict__ c, i64 ldc) {
  const i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (idx >= m * n) return;
  const i64 i = idx / n, j = idx % n;
  float s = part[i * ldp + j];
  for (int z = 1; z < splits; ++z) s += part[static_cast<i64>(z) * m * ldp + i * ldp + j];
  c[i * ldc + j] = s;
}

__global__ void zero_kernel(float* c, i64 m, i64 n, i64 ldc) {
  const i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (idx < m * n) c[(idx / n) * ldc + idx % n] = 0.f;
}

template <bool TA, bool TB, bool EXACT>
void launch_simt(i64 m, i64 n, i64 k, i64 k_chunk, const float* a, i64 lda, const float* b,
                 i64 ldb, float* c, i64 ldc, int splits, cudaStream_t st) {
  dim3 grid(ceil_div(n, kBN), ceil_div(m, kBM), splits);
  check(grid.y < 65536, "gemm: m too large for one launch");
  gemm_simt_kernel<TA, TB, EXACT><<<grid, 256, 0, st>>>(m, n, k, k_chunk, a, lda, b, ldb, c,
                                                         ldc);
  PK_LAUNCH("gemm simt kernel");
}

template <bool TA, bool TB>
void gemm_simt_dispatch(i64 m, i64 n, i64 k, const float* a, i64 lda, const float* b, i64 ldb,
                        float* c, i64 ldc, int mode, cudaStream_t st) {
  const i64 tiles = static_cast<i64>(ceil_div(m, kBM)) * ceil_div(n, kBN);
  const i64 want = static_cast<i64>(sm_count()) * 4;
  if (mode == PK_MODE_PARITY) {
    if (tiles < want / 4 && k > 4 * kTK) {
      dim3 grid(ceil_div(n, 16), ceil_div(m, 16));
      gemm_tall_exact_kernel<TA, TB><<<grid, 256, 0, st>>>(m, n, k, a, lda, b, ldb, c, ldc);
      PK_LAUNCH("gemm tall exact kernel");
    } else {
      launch_simt<TA, TB, true>(m, n, k, k, a, lda, b, ldb, c, ldc, 1, st);
    }
    return;
  }
  // FAST fallback: FFMA with split-K for tall reductions.
  int splits = 1;
  if (tiles < want && k >= 4096) {
    splits = static_cast<int>(std::min<i64>(std::min<i64>(want / tiles, 64), k / 1024));
    if (splits < 1) splits = 1;
  }
  if (splits == 1) {
    launch_simt<TA, TB, false>(m, n, k, k, a, lda, b, ldb, c, ldc, 1, st);
    return;
  }
  // each split covers a contiguous k range (multiple of kBK)
  const i64 chunk = ((k + splits - 1) / splits + kBK - 1) / kBK * kBK;
  splits = static_cast<int>((k + chunk - 1) / chunk);
  static thread_local DevBuf<float> part;
  part.ensure(static_cast<size_t>(splits) * m * n);
  launch_simt<TA, TB, false>(m, n, k, chunk, a, lda, b, ldb, part.p, n, splits, st);
  splitk_reduce_kernel<<<ceil_div(m * n, 256), 256, 0, st>>>(part.p, splits, m, n, n, c, ldc);
  PK_LAUNCH("gemm split-k reduce");
}

}  // namespace

void gemm_launch(bool ta, bool tb, i64 m, i64 n, i64 k, const float* a, i64 lda, const float* b,
                 i64 ldb, float* c, i64 ldc, int mode, cudaStream_t st, bool relu,
                 const RowMap* map, const float* mask, i64 ldm) {
  if (m == 0 || n == 0) return;
  check(!mask || (!relu && !map), "gemm: a mask epilogue goes without relu / mapped rows");
  if (mask && k > 0 && mode == PK_MODE_FAST &&
      gemm_tc_launch(ta, tb, m, n, k, a, lda, b, ldb, c, ldc, st, false, nullptr, mask, ldm))
    return;
  if (mask) {  // then the plain product and a separate relu_backward pass
    gemm_launch(ta, tb, m, n, k, a, lda, b, ldb, c, ldc, mode, st);
    relu_backward_launch(mask, ldm, c, ldc, m, n, c, ldc, st);
    return;
  }
  if (map) {  // a reduction fused into the epilogue: tensor-core path only
    check(mode == PK_MODE_FAST && k > 0 &&
              gemm_tc_launch(ta, tb, m, n, k, a, lda, b, ldb, c, ldc, st, relu, map),
          "gemm: mapped output rows need the tensor-core path");
    return;
  }
  if (k == 0) {  // reference writes acc = 0 (kernels.hpp:84-89); relu(0) = 0
    zero_kernel<<<ceil_div(m * n, 256), 256, 0, st>>>(c, m, n, ldc);
    PK_LAUNCH("gemm zero fill");
    return;
  }
  if (mode == PK_MODE_FAST && gemm_tc_launch(ta, tb, m, n, k, a, lda, b, ldb, c, ldc, st, relu))
    return;
  if (!ta && !tb)
    gemm_simt_dispatch<false, false>(m, n, k, a, lda, b, ldb, c, ldc, mode, st);
  else if (ta && !tb)
    gemm_simt_dispatch<true, false>(m, n, k, a, lda, b, ldb, c, ldc, mode, st);
  else if (!ta && tb)
    gemm_simt_dispatch<false, true>(m, n, k, a, lda, b, ldb, c, ldc, mode, st);
  else
    gemm_simt_dispatch<true, true>(m, n, k, a, lda, b, ldb, c, ldc, mode, st);
  if (relu) relu_forward_launch(c, ldc, m, n, c, ldc, st);
}

}  // namespace pk
