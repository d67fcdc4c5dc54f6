// Fused elementwise kernels of the GCN layer: ReLU forward/backward
// (kernels.hpp:94-111), masked softmax cross-entropy sums (kernels.hpp:117-158)
// with the finalize_loss scaling (trainer.hpp:84-87), and Adam
// (model.hpp:88-111). All are HBM-streaming; ReLU and Adam are bit-exact.
#include <cuda_runtime.h>

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
// cross entropy: one warp per row (grid-stride, fixed grid so the double
// partial sums reduce in a fixed order -> run-to-run deterministic).

constexpr int kCeWarps = 8;
constexpr int kCeMaxPerLane = 8;  // up to 256 classes per row in registers

__global__ void __launch_bounds__(kCeWarps * 32)
ce_kernel(const float* __restrict__ logits, i64 ldl, i64 rows, int classes,
          const u32* __restrict__ labels, const u8* __restrict__ mask,
          float* __restrict__ dl, i64 ldd, double* __restrict__ partial,
          u32* __restrict__ bad_label, u64 scale_count) {
  // (T)1 / (T)global_count (trainer.hpp:84), applied as the reference's
  // separate multiply, fl(d * s)
  const float s = scale_count ? __fdiv_rn(1.f, static_cast<float>(scale_count)) : 1.f;
  const int lane = threadIdx.x % 32, w = threadIdx.x / 32;
  const i64 gw = static_cast<i64>(blockIdx.x) * kCeWarps + w;
  const i64 nw = static_cast<i64>(gridDim.x) * kCeWarps;
  double loss = 0, count = 0, correct = 0;
  // the next row's mask, label and logits are loaded before the current row
  // is processed: one memory latency per row instead of three serial ones
  const int nt = (classes + 31) / 32;
  auto fetch = [&](i64 r, u8& m, u32& lab, float (&x)[kCeMaxPerLane]) {
    m = 0, lab = 0;
    if (r >= rows) return;
    m = mask[r];
    lab = labels[r];
    const float* row = logits + r * ldl;
#pragma unroll
    for (int t = 0; t < kCeMaxPerLane; ++t) {
      const int j = lane + 32 * t;
      x[t] = (t < nt && j < classes) ? row[j] : -INFINITY;
    }
  };
  u8 m_next;
  u32 lab_next;
  float x_next[kCeMaxPerLane];
  fetch(gw, m_next, lab_next, x_next);
  for (i64 r = gw; r < rows; r += nw) {
    const u8 m = m_next;
    const u32 lab = lab_next;
    float xv[kCeMaxPerLane];
#pragma unroll
    for (int t = 0; t < kCeMaxPerLane; ++t) xv[t] = x_next[t];
    fetch(r + nw, m_next, lab_next, x_next);
    float* drow = dl + r * ldd;
    if (!m) {
      for (int j = lane; j < classes; j += 32) drow[j] = 0.f;
      continue;
    }
    if (lab >= static_cast<u32>(classes)) {
      if (lane == 0) atomicExch(bad_label, 1u);
      for (int j = lane; j < classes; j += 32) drow[j] = 0.f;
      continue;
    }
    // first max, lowest index on ties (kernels.hpp:142-145)
    float mx = -INFINITY;
    int am = 0x7fffffff;
#pragma unroll
    for (int t = 0; t < kCeMaxPerLane; ++t) {
      const int j = lane + 32 * t;
      if (j < classes && (xv[t] > mx || am == 0x7fffffff)) mx = xv[t], am = j;
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float om = __shfl_xor_sync(0xffffffffu, mx, off);
      const int oa = __shfl_xor_sync(0xffffffffu, am, off);
      if (om > mx || (om == mx && oa < am)) mx = om, am = oa;
    }
    // denominator summed in ascending class order like the reference loop
    float ev[kCeMaxPerLane];
#pragma unroll
    for (int t = 0; t < kCeMaxPerLane; ++t) {
      const int j = lane + 32 * t;
      ev[t] = j < classes ? expf(xv[t] - mx) : 0.f;
    }
    float denom = 0.f;
#pragma unroll
    for (int t = 0; t < kCeMaxPerLane; ++t) {
      if (32 * t >= classes) break;
      for (int src = 0; src < 32; ++src) {
        const float e = __shfl_sync(0xffffffffu, ev[t], src);
        if (32 * t + src < classes) denom = __fadd_rn(denom, e);
      }
    }
    const float xl = __shfl_sync(0xffffffffu, xv[lab / 32], lab % 32);
    if (lane == 0) {
      loss += static_cast<double>(__fsub_rn(logf(denom), __fsub_rn(xl, mx)));
      count += 1;
      if (am == static_cast<int>(lab)) correct += 1;
    }
    // one reciprocal per row instead of a divide per class: within 1 ulp of
    // the reference's exp/denom (CE is tolerance-checked anyway: expf/logf
    // differ from glibc in the last ulp)
    const float rden = __frcp_rn(denom);
#pragma unroll
    for (int t = 0; t < kCeMaxPerLane; ++t) {
      const int j = lane + 32 * t;
      if (j < classes) {
        float d = __fmul_rn(ev[t], rden);
        if (j == static_cast<int>(lab)) d = __fsub_rn(d, 1.f);
        drow[j] = scale_count ? __fmul_rn(d, s) : d;
      }
    }
  }
  // block partials in warp order
  __shared__ double sh[kCeWarps][3];
  if (lane == 0) sh[w][0] = loss, sh[w][1] = count, sh[w][2] = correct;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0, b = 0, c = 0;
    for (int i = 0; i < kCeWarps; ++i) a += sh[i][0], b += sh[i][1], c += sh[i][2];
    partial[3 * blockIdx.x] = a;
    partial[3 * blockIdx.x + 1] = b;
    partial[3 * blockIdx.x + 2] = c;
  }
}

__global__ void ce_finish_kernel(const double* __restrict__ partial, int blocks,
                                 double* __restrict__ sums) {
  if (threadIdx.x != 0) return;
  double a = 0, b = 0, c = 0;
  for (int i = 0; i < blocks; ++i)
    a += partial[3 * i], b += partial[3 * i + 1], c += partial[3 * i + 2];
  sums[0] = a, sums[1] = b, sums[2] = c;
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

__global__ void adam_kernel(float* __restrict__ p, const float* __restrict__ g,
                            float* __restrict__ m, float* __restrict__ v, i64 n, AdamScalars s) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const float gi = g[i];
    // m = b1*m + (1-b1)*g ; v = b2*v + ((1-b2)*g)*g   (model.hpp:97-98)
    const float mi = __fadd_rn(__fmul_rn(s.b1, m[i]), __fmul_rn(s.omb1, gi));
    const float vi = __fadd_rn(__fmul_rn(s.b2, v[i]), __fmul_rn(__fmul_rn(s.omb2, gi), gi));
    m[i] = mi;
    v[i] = vi;
    const float mh = __fdiv_rn(mi, s.bias1);
    const float vh = __fdiv_rn(vi, s.bias2);
    // p -= (lr*m_hat) / (sqrt(v_hat) + eps)   (model.hpp:101)
    p[i] = __fsub_rn(p[i], __fdiv_rn(__fmul_rn(s.lr, mh), __fadd_rn(__fsqrt_rn(vh), s.eps)));
  }
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
                    cudaStream_t st, u64 scale_count) {
  check(classes <= 32 * kCeMaxPerLane,
        "cross entropy: at most " + std::to_string(32 * kCeMaxPerLane) + " classes supported");
  const int blocks = std::max(1, std::min<int>(sm_count() * 4, ceil_div(rows, kCeWarps)));
  ws.partial.ensure(3 * static_cast<size_t>(blocks));
  ws.bad.ensure(1);
  PK_CUDA(cudaMemsetAsync(ws.bad.p, 0, sizeof(u32), st));
  if (rows > 0 && classes > 0) {
    ce_kernel<<<blocks, kCeWarps * 32, 0, st>>>(logits, ldl, rows, static_cast<int>(classes),
                                               labels, mask, dl, ldd, ws.partial.p, ws.bad.p,
                                               scale_count);
    PK_LAUNCH("cross entropy");
    ce_finish_kernel<<<1, 32, 0, st>>>(ws.partial.p, blocks, sums);
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
  adam_kernel<<<stream_grid(n), 256, 0, st>>>(p, g, m, v, n, s);
  PK_LAUNCH("adam");
}

}  // namespace pk
