// Fused elementwise kernels of the GCN layer: ReLU forward/backward
// (kernels.hpp:94-111), masked softmax cross-entropy sums (kernels.hpp:117-158)
// with the finalize_loss scaling (trainer.hpp:84-87), and Adam
// (model.hpp:88-111). All are HBM-streaming; ReLU and Adam are bit-exact.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "elementwise.cuh"
#include "pk_common.cuh"

namespace pk {

namespace {

// ReLU kernels. Contiguous operands (ld == cols, 16-B aligned) stream as
// flat float4 arrays; strided views go row by row (a warp per row, lanes over
// columns), never dividing per element.
__device__ __forceinline__ float relu1(float v) { return v > 0.f ? v : 0.f; }

__global__ void relu_fwd_flat_kernel(const float4* __restrict__ q, i64 n4,
                                     float4* __restrict__ out) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const float4 v = __ldcs(q + i);
    __stcs(out + i, make_float4(relu1(v.x), relu1(v.y), relu1(v.z), relu1(v.w)));
  }
}

__global__ void relu_bwd_flat_kernel(const float4* __restrict__ q, const float4* __restrict__ df,
                                     i64 n4, float4* __restrict__ out) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const float4 a = __ldcs(q + i), d = __ldcs(df + i);
    __stcs(out + i, make_float4(a.x > 0.f ? d.x : 0.f, a.y > 0.f ? d.y : 0.f,
                                a.z > 0.f ? d.z : 0.f, a.w > 0.f ? d.w : 0.f));
  }
}

__global__ void relu_fwd_kernel(const float* __restrict__ q, i64 ldq, i64 rows, i64 cols,
                                float* __restrict__ out, i64 ldo) {
  const int lane = threadIdx.x % 32;
  const i64 nw = static_cast<i64>(gridDim.x) * (blockDim.x / 32);
  for (i64 r = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) / 32; r < rows; r += nw)
    for (i64 c = lane; c < cols; c += 32) out[r * ldo + c] = relu1(q[r * ldq + c]);
}

__global__ void relu_bwd_kernel(const float* __restrict__ q, i64 ldq,
                                const float* __restrict__ df, i64 lddf, i64 rows, i64 cols,
                                float* __restrict__ out, i64 ldo) {
  const int lane = threadIdx.x % 32;
  const i64 nw = static_cast<i64>(gridDim.x) * (blockDim.x / 32);
  for (i64 r = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) / 32; r < rows; r += nw)
    for (i64 c = lane; c < cols; c += 32)
      out[r * ldo + c] = q[r * ldq + c] > 0.f ? df[r * lddf + c] : 0.f;
}

bool flat4(const void* p, i64 ld, i64 cols) {
  return ld == cols && cols % 4 == 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
}

unsigned stream_grid(i64 n) {
  const i64 cap = static_cast<i64>(sm_count()) * 8;
  return static_cast<unsigned>(std::max<i64>(1, std::min<i64>(cap, (n + 255) / 256)));
}

// ---------------------------------------------------------------------------
// cross entropy: a CTA stages a tile of kCeRows logits rows in shared memory
// with coalesced loads (row stride padded to an odd word count: the per-row
// passes below are bank-conflict free), then each thread owns one row and
// walks it in ascending class order exactly like the reference loop; the
// dlogits tile goes back out through the same buffer with coalesced stores.
// Fixed grid, per-thread double partials reduced in a fixed tree ->
// run-to-run deterministic.

constexpr int kCeRows = 128;  // rows per tile = threads per CTA
constexpr int kCeMaxClasses = 384;  // tile <= 193 KB of shared memory

__host__ __device__ inline int ce_stride(int classes) { return classes | 1; }

__global__ void __launch_bounds__(kCeRows)
ce_kernel(const float* __restrict__ logits, i64 ldl, i64 rows, int classes,
          const u32* __restrict__ labels, const u8* __restrict__ mask,
          float* __restrict__ dl, i64 ldd, int dc0, int dc1, double* __restrict__ partial,
          u32* __restrict__ bad_label, u64 scale_count) {
  extern __shared__ float tile[];  // [kCeRows][ce_stride(classes)]
  // (T)1 / (T)global_count (trainer.hpp:84), applied as the reference's
  // separate multiply, fl(d * s)
  const float s = scale_count ? __fdiv_rn(1.f, static_cast<float>(scale_count)) : 1.f;
  const int t = threadIdx.x;
  const int stride = ce_stride(classes);
  double loss = 0, count = 0, correct = 0;
  for (i64 r0 = static_cast<i64>(blockIdx.x) * kCeRows; r0 < rows;
       r0 += static_cast<i64>(gridDim.x) * kCeRows) {
    const int nr = static_cast<int>(rows - r0 < kCeRows ? rows - r0 : kCeRows);
    const int elems = nr * classes;
    // coalesced stage-in: flat element e of the tile -> (row, class)
    for (int e = t; e < elems; e += kCeRows) {
      const int rr = e / classes, c = e - rr * classes;
      tile[rr * stride + c] = __ldcs(logits + (r0 + rr) * ldl + c);
    }
    const i64 r = r0 + t;
    const bool live = t < nr;
    const u8 m = live ? mask[r] : 0;
    const u32 lab = live ? labels[r] : 0;
    __syncthreads();
    float* x = tile + t * stride;
    if (live) {
      if (!m || lab >= static_cast<u32>(classes)) {
        if (m) atomicExch(bad_label, 1u);
        for (int j = 0; j < classes; ++j) x[j] = 0.f;
      } else {
        // first max, lowest index on ties (kernels.hpp:142-145)
        float mx = x[0];
        int am = 0;
        for (int j = 1; j < classes; ++j)
          if (x[j] > mx) mx = x[j], am = j;
        const float xl = x[lab];
        // denominator summed in ascending class order like the reference
        float denom = 0.f;
        for (int j = 0; j < classes; ++j) {
          const float e = expf(x[j] - mx);
          x[j] = e;
          denom = __fadd_rn(denom, e);
        }
        loss += static_cast<double>(__fsub_rn(logf(denom), __fsub_rn(xl, mx)));
        count += 1;
        if (am == static_cast<int>(lab)) correct += 1;
        // one reciprocal per row instead of a divide per class: within 1 ulp
        // of the reference's exp/denom (CE is tolerance-checked anyway:
        // expf/logf differ from glibc in the last ulp)
        const float rden = __frcp_rn(denom);
        for (int j = 0; j < classes; ++j) {
          float d = __fmul_rn(x[j], rden);
          if (j == static_cast<int>(lab)) d = __fsub_rn(d, 1.f);
          x[j] = scale_count ? __fmul_rn(d, s) : d;
        }
      }
    }
    __syncthreads();
    // only the class window [dc0, dc1) of dlogits leaves the CTA: the rank's
    // own chunk of the last layer's classes (trainer.hpp:517-520)
    const int w = dc1 - dc0;
    for (int e = t; e < nr * w; e += kCeRows) {
      const int rr = e / w, c = e - rr * w;
      __stcs(dl + (r0 + rr) * ldd + c, tile[rr * stride + dc0 + c]);
    }
    __syncthreads();
  }
  // fixed-order tree over the CTA's threads
  __shared__ double sh[kCeRows][3];
  sh[t][0] = loss, sh[t][1] = count, sh[t][2] = correct;
  __syncthreads();
  for (int h = kCeRows / 2; h > 0; h >>= 1) {
    if (t < h)
      for (int k = 0; k < 3; ++k) sh[t][k] += sh[t + h][k];
    __syncthreads();
  }
  if (t == 0) {
    partial[3 * blockIdx.x] = sh[0][0];
    partial[3 * blockIdx.x + 1] = sh[0][1];
    partial[3 * blockIdx.x + 2] = sh[0][2];
  }
}

// one CTA: thread t sums blocks t, t + 256, ... in order, then a fixed tree
// (deterministic; the per-block partials were summed in a fixed order too)
constexpr int kCeFinishThreads = 256;

__global__ void __launch_bounds__(kCeFinishThreads)
ce_finish_kernel(const double* __restrict__ partial, int blocks, double* __restrict__ sums) {
  __shared__ double sh[kCeFinishThreads][3];
  const int t = threadIdx.x;
  double a = 0, b = 0, c = 0;
  for (int i = t; i < blocks; i += kCeFinishThreads)
    a += partial[3 * i], b += partial[3 * i + 1], c += partial[3 * i + 2];
  sh[t][0] = a, sh[t][1] = b, sh[t][2] = c;
  __syncthreads();
  for (int h = kCeFinishThreads / 2; h > 0; h >>= 1) {
    if (t < h)
      for (int k = 0; k < 3; ++k) sh[t][k] += sh[t + h][k];
    __syncthreads();
  }
  if (t == 0) sums[0] = sh[0][0], sums[1] = sh[0][1], sums[2] = sh[0][2];
}

__global__ void scale_kernel(float* __restrict__ d, i64 ldd, i64 rows, i64 cols,
                             const double* __restrict__ sums) {
  // (T)1 / (T)global_count (trainer.hpp:84)
  const float s = __fdiv_rn(1.f, static_cast<float>(static_cast<u64>(sums[1])));
  const i64 n = rows * cols;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = i / cols, c = i % cols;
    d[r * ldd + c] = __fmul_rn(d[r * ldd + c], s);
  }
}

__device__ __forceinline__ void adam1(float& p, float g, float& m, float& v,
                                      const AdamScalars& s) {
  // m = b1*m + (1-b1)*g ; v = b2*v + ((1-b2)*g)*g   (model.hpp:97-98)
  m = __fadd_rn(__fmul_rn(s.b1, m), __fmul_rn(s.omb1, g));
  v = __fadd_rn(__fmul_rn(s.b2, v), __fmul_rn(__fmul_rn(s.omb2, g), g));
  const float mh = __fdiv_rn(m, s.bias1);
  const float vh = __fdiv_rn(v, s.bias2);
  // p -= (lr*m_hat) / (sqrt(v_hat) + eps)   (model.hpp:101)
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(s.lr, mh), __fadd_rn(__fsqrt_rn(vh), s.eps)));
}

// float4 body over [0, n4) plus a scalar tail [4*n4, n); four streams in,
// three out, all in-place
__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                            float* __restrict__ m, float* __restrict__ v, i64 n, AdamScalars s) {
  const i64 n4 = n / 4;
  const i64 step = static_cast<i64>(gridDim.x) * blockDim.x;
  const i64 t0 = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  float4* p4 = reinterpret_cast<float4*>(p);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* m4 = reinterpret_cast<float4*>(m);
  float4* v4 = reinterpret_cast<float4*>(v);
  for (i64 i = t0; i < n4; i += step) {
    float4 pi = p4[i], mi = m4[i], vi = v4[i];
    const float4 gi = __ldcs(g4 + i);
    adam1(pi.x, gi.x, mi.x, vi.x, s);
    adam1(pi.y, gi.y, mi.y, vi.y, s);
    adam1(pi.z, gi.z, mi.z, vi.z, s);
    adam1(pi.w, gi.w, mi.w, vi.w, s);
    p4[i] = pi, m4[i] = mi, v4[i] = vi;
  }
  for (i64 i = 4 * n4 + t0; i < n; i += step) adam1(p[i], g[i], m[i], v[i], s);
}

__global__ void adam_scalar_kernel(float* __restrict__ p, const float* __restrict__ g,
                                   float* __restrict__ m, float* __restrict__ v, i64 n,
                                   AdamScalars s) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    adam1(p[i], g[i], m[i], v[i], s);
}

}  // namespace

void relu_forward_launch(const float* q, i64 ldq, i64 rows, i64 cols, float* out, i64 ldo,
                         cudaStream_t st) {
  if (rows * cols == 0) return;
  if (flat4(q, ldq, cols) && flat4(out, ldo, cols)) {
    const i64 n4 = rows * cols / 4;
    relu_fwd_flat_kernel<<<stream_grid(n4), 256, 0, st>>>(reinterpret_cast<const float4*>(q), n4,
                                                          reinterpret_cast<float4*>(out));
  } else {
    relu_fwd_kernel<<<stream_grid(rows * 32), 256, 0, st>>>(q, ldq, rows, cols, out, ldo);
  }
  PK_LAUNCH("relu forward");
}

void relu_backward_launch(const float* q, i64 ldq, const float* df, i64 lddf, i64 rows,
                          i64 cols, float* out, i64 ldo, cudaStream_t st) {
  if (rows * cols == 0) return;
  if (flat4(q, ldq, cols) && flat4(df, lddf, cols) && flat4(out, ldo, cols)) {
    const i64 n4 = rows * cols / 4;
    relu_bwd_flat_kernel<<<stream_grid(n4), 256, 0, st>>>(reinterpret_cast<const float4*>(q),
                                                          reinterpret_cast<const float4*>(df), n4,
                                                          reinterpret_cast<float4*>(out));
  } else {
    relu_bwd_kernel<<<stream_grid(rows * 32), 256, 0, st>>>(q, ldq, df, lddf, rows, cols, out,
                                                            ldo);
  }
  PK_LAUNCH("relu backward");
}

void ce_sums_launch(const float* logits, i64 ldl, i64 rows, i64 classes, const u32* labels,
                    const u8* mask, float* dl, i64 ldd, double* sums, CeWorkspace& ws,
                    cudaStream_t st, u64 scale_count, i64 dc0, i64 dc1) {
  if (dc1 < 0) dc1 = classes;
  check(0 <= dc0 && dc0 <= dc1 && dc1 <= classes, "cross entropy: bad class window");
  const size_t smem = sizeof(float) * kCeRows * ce_stride(static_cast<int>(classes));
  check(classes <= kCeMaxClasses, "cross entropy: at most " + std::to_string(kCeMaxClasses) +
                                      " classes supported");
  static const bool attr = [] {
    PK_CUDA(cudaFuncSetAttribute(ce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(sizeof(float) * kCeRows *
                                                  ce_stride(kCeMaxClasses))));
    return true;
  }();
  (void)attr;
  // CTAs resident per SM by shared memory (<= 8), times the SM count
  const int per_sm = static_cast<int>(std::max<size_t>(1, std::min<size_t>(8, (200u << 10) / smem)));
  const int blocks =
      std::max(1, std::min<int>(sm_count() * per_sm, ceil_div(rows, kCeRows)));
  ws.partial.ensure(3 * static_cast<size_t>(blocks));
  ws.bad.ensure(1);
  PK_CUDA(cudaMemsetAsync(ws.bad.p, 0, sizeof(u32), st));
  if (rows > 0 && classes > 0) {
    ce_kernel<<<blocks, kCeRows, smem, st>>>(logits, ldl, rows, static_cast<int>(classes), labels,
                                             mask, dl, ldd, static_cast<int>(dc0),
                                             static_cast<int>(dc1), ws.partial.p, ws.bad.p,
                                             scale_count);
    PK_LAUNCH("cross entropy");
    ce_finish_kernel<<<1, kCeFinishThreads, 0, st>>>(ws.partial.p, blocks, sums);
  } else {
    PK_CUDA(cudaMemsetAsync(sums, 0, 3 * sizeof(double), st));
  }
  PK_LAUNCH("cross entropy finish");
}

void scale_by_count_launch(float* d, i64 ldd, i64 rows, i64 cols, const double* sums,
                           cudaStream_t st) {
  if (rows * cols == 0) return;
  scale_kernel<<<stream_grid(rows * cols), 256, 0, st>>>(d, ldd, rows, cols, sums);
  PK_LAUNCH("scale dlogits");
}

AdamScalars adam_scalars(u64 step, double lr, double beta1, double beta2, double eps) {
  // model.hpp:93-96: beta/lr/eps cast to T; bias terms in double then cast
  AdamScalars s;
  s.b1 = static_cast<float>(beta1);
  s.b2 = static_cast<float>(beta2);
  s.omb1 = 1.0f - s.b1;
  s.omb2 = 1.0f - s.b2;
  s.bias1 = static_cast<float>(1.0 - std::pow(beta1, static_cast<double>(step)));
  s.bias2 = static_cast<float>(1.0 - std::pow(beta2, static_cast<double>(step)));
  s.lr = static_cast<float>(lr);
  s.eps = static_cast<float>(eps);
  return s;
}

void adam_launch(float* p, const float* g, float* m, float* v, i64 n, const AdamScalars& s,
                 cudaStream_t st) {
  if (n == 0) return;
  const bool a16 = ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g) |
                     reinterpret_cast<uintptr_t>(m) | reinterpret_cast<uintptr_t>(v)) & 15) == 0;
  if (a16)
    adam_kernel<<<stream_grid((n + 3) / 4), 256, 0, st>>>(p, g, m, v, n, s);
  else
    adam_scalar_kernel<<<stream_grid(n), 256, 0, st>>>(p, g, m, v, n, s);
  PK_LAUNCH("adam");
}

}  // namespace pk
