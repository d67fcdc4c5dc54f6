// CSR SpMM for the GCN aggregation H = A . F (and dF = A^T . dH with the
// precomputed transpose), sm_100a.
//
// Reference semantics (kernels.hpp:16-62): out row i starts at +0 and, for k
// ascending over the row's nonzeros, out[i][j] = fl(out[i][j] + fl(v_k *
// x[c_k][j])) with no FMA. Every kernel here keeps exactly that order for
// every output element — one lane owns one column chain of one row — so the
// result is bit-identical to the CPU reference. All parallelism is across
// rows and columns, never across k.
//
// The operation is HBM/gather bound (8 B per nonzero of index +
// value, plus one gathered feature row per nonzero). Design:
//   * short rows ("warp path"): a LANES-wide lane group owns a row; lanes
//     span the feature columns with 16-B (or 8-/4-B) vector loads so each
//     gathered row is read with full sectors; the (col, val) pairs are
//     fetched coalesced, LANES at a time, and broadcast with shuffles; the
//     gathers are unrolled U deep so each lane keeps U*NV loads in flight.
//   * hub rows (RMAT degree skew: median 3, max 155,518 nnz per row at the
//     products shape): a whole CTA serves one (row, 32*VEC-column slice);
//     seven loader warps stream the gathered row slices into a shared-memory
//     ring with cp.async so hundreds of gathers are in flight for the single
//     sequential chain that the consumer warp runs. Hub CTAs are the first
//     blocks of the same launch, longest row first, so they overlap the
//     short-row work.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "pk_common.cuh"
#include "spmm.cuh"

namespace pk {

namespace {

template <int VEC>
struct Vec;
template <>
struct Vec<1> {
  using T = float;
  static __device__ __forceinline__ T zero() { return 0.f; }
};
template <>
struct Vec<2> {
  using T = float2;
  static __device__ __forceinline__ T zero() { return make_float2(0.f, 0.f); }
};
template <>
struct Vec<4> {
  using T = float4;
  static __device__ __forceinline__ T zero() { return make_float4(0.f, 0.f, 0.f, 0.f); }
};

// acc = fl(acc + fl(v * x)), element-wise, never contracted to FMA.
__device__ __forceinline__ void madd(float& a, float v, float x) {
  a = __fadd_rn(a, __fmul_rn(v, x));
}
__device__ __forceinline__ void madd(float2& a, float v, float2 x) {
  madd(a.x, v, x.x);
  madd(a.y, v, x.y);
}
__device__ __forceinline__ void madd(float4& a, float v, float4 x) {
  madd(a.x, v, x.x);
  madd(a.y, v, x.y);
  madd(a.z, v, x.z);
  madd(a.w, v, x.w);
}

template <typename T>
__device__ __forceinline__ T ldg(const float* p) {
  return __ldg(reinterpret_cast<const T*>(p));
}

constexpr int kThreads = 256;

// Set (and reported once with printf) when a kernel bails out of a wait or
// loop that should have terminated; read back by pk_spmm_watchdog().
__device__ unsigned g_spmm_watchdog = 0;

// ---------------------------------------------------------------------------
// short-row path: persistent nnz-balanced stream
//
// [r0, r1) is cut into chunks of ~equal nonzeros (whole rows, empty rows
// included). Each lane group grabs chunks from an atomic counter and walks
// its chunk's nonzeros as one contiguous stream in windows of LANES entries:
// the (col, val) window is a single coalesced load (the next one prefetched),
// and U gathers are in flight regardless of where rows begin and end. Row
// boundaries are tracked from a LANES-wide batch of row_ptr values; a row's
// accumulator is stored the moment its last entry is consumed, so every
// output element still sums its own k terms strictly in order.

__global__ void spmm_partition_kernel(const u64* __restrict__ rp, i64 r0, i64 r1, int nchunks,
                                      i64* __restrict__ bounds, int* __restrict__ counters,
                                      int nslices) {
  const i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (t < nslices) counters[t] = 0;
  if (t > nchunks) return;
  if (t == 0 || t == nchunks) {
    bounds[t] = t == 0 ? r0 : r1;
    return;
  }
  const u64 base = rp[r0], total = rp[r1] - base;
  const u64 target = base + total / nchunks * t + (total % nchunks) * t / nchunks;
  i64 lo = r0, hi = r1;  // first row with rp[row] >= target
  while (lo < hi) {
    const i64 mid = lo + (hi - lo) / 2;
    if (rp[mid] < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  bounds[t] = lo;
}

template <int VEC, int LANES, int NV, int U>
__device__ __forceinline__ void stream_rows(const SpmmArgs& a, i64 rs, i64 re, int lane,
                                            unsigned gmask, int vbase, const bool (&valid)[NV]) {
  using V = typename Vec<VEC>::T;
  const u64 hub_t = a.hub_threshold;
  // ends[i] = rp[rb + 1 + i]: end of row rb + i
  i64 rb = rs;
  u64 ends = __ldg(a.rp + min(rb + 1 + lane, re));
  u64 s = __ldg(a.rp + rs);
  u64 e = __shfl_sync(gmask, ends, 0, LANES);
  const u64 kend = __ldg(a.rp + re);
  i64 r = rs;
  V acc[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) acc[t] = Vec<VEC>::zero();

  auto store = [&](i64 row) {
    float* yrow = a.y + (row - a.r0) * a.ldy;
#pragma unroll
    for (int t = 0; t < NV; ++t)
      if (valid[t]) *reinterpret_cast<V*>(yrow + (vbase + t * LANES + lane) * VEC) = acc[t];
  };
  auto next_row = [&]() {
    ++r;
    s = e;
    if (r < re) {
      if (r - rb >= LANES) {
        rb = r;
        ends = __ldg(a.rp + min(rb + 1 + lane, re));
      }
      e = __shfl_sync(gmask, ends, static_cast<int>(r - rb), LANES);
    }
  };
  // skip empty rows (store zeros) and hub rows (owned by hub CTAs); returns
  // true when a hub was skipped, i.e. the nonzero stream jumps forward
  auto settle = [&]() {
    bool jumped = false;
    while (r < re) {
      if (s == e) {
        store(r);  // acc is zero here
        next_row();
      } else if (e - s >= hub_t) {
        next_row();
        jumped = true;
      } else {
        break;
      }
    }
    return jumped;
  };

  settle();
  u64 kb = s;
  u32 c = 0;
  float v = 0.f;
  if (r < re && kb + lane < kend) {
    c = __ldcs(a.ci + kb + lane);
    v = __ldcs(a.val + kb + lane);
  }
  // every window either consumes >= 1 entry or jumps forward, so a chunk
  // takes at most (its nonzeros + its rows) windows
  u64 guard = (kend - kb) + static_cast<u64>(re - rs) + 2;
  while (r < re) {
    if (guard-- == 0) {
      if (atomicAdd(&g_spmm_watchdog, 1u) == 0)
        printf("spmm stream watchdog: rows [%lld, %lld) stuck at row %lld kb %llu\n",
               static_cast<long long>(rs), static_cast<long long>(re),
               static_cast<long long>(r), static_cast<unsigned long long>(kb));
      return;
    }
    // prefetch the next window
    u32 cn = 0;
    float vn = 0.f;
    if (kb + LANES + lane < kend) {
      cn = __ldcs(a.ci + kb + LANES + lane);
      vn = __ldcs(a.val + kb + LANES + lane);
    }
    const int cnt = static_cast<int>(min(static_cast<u64>(LANES), kend - kb));
    bool jumped = false;
    for (int j = 0; j < cnt && !jumped && r < re; j += U) {
      V xv[U][NV];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const u32 cj = __shfl_sync(gmask, c, (j + u) % LANES, LANES);
        const float* xrow = a.x + static_cast<i64>(cj) * a.ldx;
        const bool in = j + u < cnt;
#pragma unroll
        for (int t = 0; t < NV; ++t)
          xv[u][t] = (valid[t] && in) ? ldg<V>(xrow + (vbase + t * LANES + lane) * VEC)
                                      : Vec<VEC>::zero();
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float vj = __shfl_sync(gmask, v, (j + u) % LANES, LANES);
        if (j + u < cnt && !jumped && r < re) {
#pragma unroll
          for (int t = 0; t < NV; ++t) madd(acc[t], vj, xv[u][t]);
          if (kb + j + u + 1 == e) {  // last entry of row r
            store(r);
#pragma unroll
            for (int t = 0; t < NV; ++t) acc[t] = Vec<VEC>::zero();
            next_row();
            jumped = settle();
          }
        }
      }
    }
    if (r >= re) break;
    if (jumped) {  // restart the window at the next regular row
      kb = s;
      c = kb + lane < kend ? __ldcs(a.ci + kb + lane) : 0u;
      v = kb + lane < kend ? __ldcs(a.val + kb + lane) : 0.f;
    } else {
      kb += cnt;
      c = cn;
      v = vn;
    }
  }
}

template <int VEC, int LANES, int NV, int U>
__global__ void __launch_bounds__(kThreads)
spmm_stream_kernel(SpmmArgs args, const i64* __restrict__ bounds, int nchunks,
                   int* __restrict__ counters) {
  const int lane = threadIdx.x % LANES;
  const unsigned gmask =
      LANES == 32 ? 0xffffffffu
                  : (((1u << LANES) - 1u) << ((threadIdx.x % 32) / LANES * LANES));
  const int vbase = static_cast<int>(blockIdx.y) * (NV * LANES);
  bool valid[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) valid[t] = vbase + t * LANES + lane < args.nvec;
  int* counter = counters + blockIdx.y;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(counter, 1);
    t = __shfl_sync(gmask, t, 0, LANES);
    if (t >= nchunks) break;
    const i64 rs = bounds[t], re = bounds[t + 1];
    if (rs < re) stream_rows<VEC, LANES, NV, U>(args, rs, re, lane, gmask, vbase, valid);
  }
}

// ---------------------------------------------------------------------------
// hub path: one CTA per (hub row, column slice of 32*VEC floats)
//
// Ring of kStages stages, each holding kBatch consecutive nonzeros' gathered
// slices (kBatch x 32 lanes x VEC floats). Warps 1..7 fill stages with
// cp.async (stage i by warp 1 + i % 7) and signal `full[i % kStages]` through
// cp.async.mbarrier.arrive; warp 0 consumes stages in order, running the
// sequential chain, and releases them through `empty`.

constexpr int kHubBatch = 32;
constexpr int kHubStages = 8;

__device__ __forceinline__ void mbar_init(u64* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar))),
               "r"(count));
}
__device__ __forceinline__ void mbar_arrive(u64* bar) {
  asm volatile(
      "{ .reg .b64 st; mbarrier.arrive.shared::cta.b64 st, [%0]; }" ::"r"(
          static_cast<unsigned>(__cvta_generic_to_shared(bar)))
      : "memory");
}
// Bounded wait: a protocol bug must surface as an error, never as a GPU that
// spins until the job is killed. ~2^28 polls is seconds of wall time.
__device__ __forceinline__ bool mbar_try(unsigned a, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(a), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(u64* bar, unsigned parity) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(bar));
  for (unsigned spins = 0; !mbar_try(a, parity); ++spins) {
    if (spins == (1u << 28)) {
      if (atomicAdd(&g_spmm_watchdog, 1u) == 0)
        printf("spmm hub watchdog: block %d thread %d stuck on barrier parity %u\n",
               blockIdx.x, threadIdx.x, parity);
      return;
    }
  }
}
// arrive on `bar` once all of this thread's prior cp.async copies land
__device__ __forceinline__ void cp_async_arrive(u64* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(
                   static_cast<unsigned>(__cvta_generic_to_shared(bar)))
               : "memory");
}
template <int BYTES>
__device__ __forceinline__ void cp_async(void* smem, const void* gmem, bool pred) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int src_bytes = pred ? BYTES : 0;  // zero-fill when out of range
  if constexpr (BYTES == 16)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem),
                 "r"(src_bytes)
                 : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(s), "l"(gmem),
                 "n"(BYTES), "r"(src_bytes)
                 : "memory");
}

// Stage count per vector width: 6 stages of 16-B slices (96 KB) lets two hub
// CTAs share an SM.
template <int VEC>
constexpr int hub_stages() {
  return VEC == 4 ? 6 : kHubStages;
}
// Loader warps = stages - 1. A loader may run ahead of the consumer by at
// most its own stride of stages; with stride <= stages - 1 it can never
// reach a ring slot two phases ahead, which mbarrier parity waits cannot
// tell apart from the phase it is waiting for.
template <int VEC>
constexpr int hub_loaders() {
  return hub_stages<VEC>() - 1;
}
template <int VEC>
constexpr int hub_threads() {
  return 32 * (hub_loaders<VEC>() + 1);
}

template <int VEC>
size_t hub_smem_bytes() {
  return static_cast<size_t>(hub_stages<VEC>()) * kHubBatch * (32 * VEC + 1) * sizeof(float);
}

template <int VEC>
__global__ void __launch_bounds__(hub_threads<VEC>())
spmm_hub_kernel(SpmmArgs args) {
  using V = typename Vec<VEC>::T;
  constexpr int kSliceVec = 32;  // vectors per slice (one per consumer lane)
  constexpr int kStages = hub_stages<VEC>();
  constexpr int kHubLoaders = hub_loaders<VEC>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  V* ring = reinterpret_cast<V*>(smem_raw);  // [stage][batch][32] gathered slices
  float* vring = reinterpret_cast<float*>(ring + kStages * kHubBatch * kSliceVec);  // [stage][batch]
  __shared__ u64 full[kStages], empty[kStages];

  const int hb = blockIdx.x;
  if (hb >= args.hub_blocks) return;
  const int slices = args.hub_slices;
  const i64 r = args.hub_rows[hb / slices];  // absolute row id
  const int slice = hb % slices;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int vcol = slice * kSliceVec + lane;
  const bool valid = vcol < args.nvec;
  const u64 s = __ldg(args.rp + r), e = __ldg(args.rp + r + 1);
  const u64 nb = (e - s + kHubBatch - 1) / kHubBatch;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 32);  // every loader lane arrives once per stage
      mbar_init(&empty[i], 1);  // consumer lane 0 releases
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp > 0) {
    // loaders: stage i handled by warp 1 + i % kHubLoaders. The column ids of
    // the loader's next stage are fetched before it blocks on `empty`, so the
    // index latency overlaps the wait.
    u64 i = warp - 1;
    u32 c_next = 0;
    if (i < nb) {
      const u64 k = s + i * kHubBatch + lane;
      c_next = k < e ? __ldcs(args.ci + k) : 0u;
    }
    for (; i < nb; i += kHubLoaders) {
      const int st = static_cast<int>(i % kStages);
      const unsigned use = static_cast<unsigned>(i / kStages);
      const u32 c = c_next;
      const u64 i2 = i + kHubLoaders;
      if (i2 < nb) {
        const u64 k2 = s + i2 * kHubBatch + lane;
        c_next = k2 < e ? __ldcs(args.ci + k2) : 0u;
      }
      if (use > 0) mbar_wait(&empty[st], (use - 1) & 1);
      V* stage = ring + static_cast<size_t>(st) * kHubBatch * kSliceVec;
      const u64 kbase = s + i * kHubBatch;
      // the lane's own value rides the same async group as the gathers
      cp_async<4>(vring + st * kHubBatch + lane, args.val + (kbase + lane < e ? kbase + lane : s),
                  kbase + lane < e);
#pragma unroll 8
      for (int j = 0; j < kHubBatch; ++j) {
        const u32 cj = __shfl_sync(0xffffffffu, c, j);
        const bool ok = valid && (kbase + j < e);
        const float* src = args.x + static_cast<i64>(cj) * args.ldx + vcol * VEC;
        cp_async<sizeof(V)>(stage + j * kSliceVec + lane, ok ? src : args.x, ok);
      }
      cp_async_arrive(&full[st]);
    }
  } else {
    V acc = Vec<VEC>::zero();
    for (u64 i = 0; i < nb; ++i) {
      const int st = static_cast<int>(i % kStages);
      const unsigned use = static_cast<unsigned>(i / kStages);
      const int cnt = static_cast<int>(min(static_cast<u64>(kHubBatch), e - s - i * kHubBatch));
      mbar_wait(&full[st], use & 1);
      const V* stage = ring + static_cast<size_t>(st) * kHubBatch * kSliceVec;
      const float* vs = vring + st * kHubBatch;
      if (cnt == kHubBatch) {
#pragma unroll
        for (int j = 0; j < kHubBatch; ++j) madd(acc, vs[j], stage[j * kSliceVec + lane]);
      } else {
        for (int j = 0; j < cnt; ++j) madd(acc, vs[j], stage[j * kSliceVec + lane]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (valid) {
      const i64 rr = r - args.r0;
      *reinterpret_cast<V*>(args.y + rr * args.ldy + vcol * VEC) = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// launch selection

struct StreamWorkspace {
  DevBuf<i64> bounds;
  DevBuf<int> counters;
};

template <int VEC, int LANES, int NV>
void launch_stream(const SpmmArgs& a, cudaStream_t st) {
  constexpr int U0 = NV >= 4 ? 2 : (NV == 2 ? 4 : 8);
  constexpr int U = U0 < LANES ? U0 : LANES;
  auto kernel = spmm_stream_kernel<VEC, LANES, NV, U>;
  const int slices = ceil_div(a.nvec, NV * LANES);
  // ~1-2K nonzeros per chunk at the products shape; never more chunks than rows
  const i64 nchunks64 = std::max<i64>(1, std::min<i64>(a.nrows, static_cast<i64>(sm_count()) * 512));
  const int nchunks = static_cast<int>(nchunks64);
  static thread_local StreamWorkspace ws;
  ws.bounds.ensure(nchunks + 1);
  ws.counters.ensure(std::max(slices, 1));
  spmm_partition_kernel<<<ceil_div(nchunks + 1, 256), 256, 0, st>>>(a.rp, a.r0, a.r0 + a.nrows,
                                                                    nchunks, ws.bounds.p,
                                                                    ws.counters.p, slices);
  PK_LAUNCH("spmm partition");
  static thread_local int occ = 0;
  if (occ == 0) {
    PK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0));
    occ = std::max(occ, 1);
  }
  const i64 groups_per_block = kThreads / LANES;
  const i64 blocks = std::max<i64>(
      1, std::min<i64>(static_cast<i64>(sm_count()) * occ,
                       (nchunks + groups_per_block - 1) / groups_per_block));
  dim3 grid(static_cast<unsigned>(blocks), slices);
  kernel<<<grid, kThreads, 0, st>>>(a, ws.bounds.p, nchunks, ws.counters.p);
  PK_LAUNCH("spmm stream kernel");
}

template <int VEC>
void launch_hub(const SpmmArgs& a, cudaStream_t st) {
  if (a.hub_blocks == 0) return;
  const size_t smem = hub_smem_bytes<VEC>();
  static thread_local bool attr_set = false;
  if (!attr_set) {
    PK_CUDA(cudaFuncSetAttribute(spmm_hub_kernel<VEC>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    attr_set = true;
  }
  spmm_hub_kernel<VEC><<<a.hub_blocks, hub_threads<VEC>(), smem, st>>>(a);
  PK_LAUNCH("spmm hub kernel");
}

template <int VEC>
void dispatch_vec(const SpmmArgs& a, cudaStream_t st) {
  const int nv = a.nvec;
  // Hub CTAs go first on a forked stream so they hold their SMs while the
  // short-row blocks stream through the rest of the machine.
  SideStream& side = side_stream();
  if (a.hub_blocks > 0) {
    PK_CUDA(cudaEventRecord(side.fork, st));
    PK_CUDA(cudaStreamWaitEvent(side.stream, side.fork, 0));
    launch_hub<VEC>(a, side.stream);
    PK_CUDA(cudaEventRecord(side.join, side.stream));
  }
  // lane-group width: smallest power of two covering the row's vectors
  if (nv <= 4)
    launch_stream<VEC, 4, 1>(a, st);
  else if (nv <= 8)
    launch_stream<VEC, 8, 1>(a, st);
  else if (nv <= 16)
    launch_stream<VEC, 16, 1>(a, st);
  else if (nv <= 32)
    launch_stream<VEC, 32, 1>(a, st);
  else if (nv <= 64)
    launch_stream<VEC, 32, 2>(a, st);
  else
    launch_stream<VEC, 32, 4>(a, st);  // wider rows split across blockIdx.y
  if (a.hub_blocks > 0) PK_CUDA(cudaStreamWaitEvent(st, side.join, 0));
}

int pick_vec(const float* x, i64 ldx, const float* y, i64 ldy, i64 d) {
  auto aligned = [](const void* p, int bytes) {
    return (reinterpret_cast<uintptr_t>(p) % bytes) == 0;
  };
  if (d % 4 == 0 && ldx % 4 == 0 && ldy % 4 == 0 && aligned(x, 16) && aligned(y, 16))
    return 4;
  if (d % 2 == 0 && ldx % 2 == 0 && ldy % 2 == 0 && aligned(x, 8) && aligned(y, 8))
    return 2;
  return 1;
}

}  // namespace

void spmm_launch(SpmmArgs a, i64 d, cudaStream_t st) {
  if (a.nrows == 0 || d == 0) return;
  const int vec = pick_vec(a.x, a.ldx, a.y, a.ldy, d);
  a.nvec = static_cast<int>(d / vec);
  // hub CTAs serve 32 vectors per slice
  a.hub_slices = ceil_div(a.nvec, 32);
  a.hub_blocks = a.hub_count * a.hub_slices;
  if (vec == 4)
    dispatch_vec<4>(a, st);
  else if (vec == 2)
    dispatch_vec<2>(a, st);
  else
    dispatch_vec<1>(a, st);
}

// ---------------------------------------------------------------------------
// plan: hub rows (nnz >= threshold) sorted longest first


void spmm_plan_build(SpmmPlan& plan, const pk_csr& a, u64 threshold, cudaStream_t st) {
  plan.rows = a.rows;
  plan.hub_rows.release();
  plan.hub_count = 0;
  if (a.rows == 0) return;
  // Threshold: a row is a hub when a single lane chain over it would outlast
  // the short-row work spread over the whole GPU several times over.
  const u64 avg = a.nnz / std::max<i64>(1, a.rows);
  plan.threshold = threshold ? threshold : std::max<u64>(4096, 64 * avg);
  // host scan of row_ptr is the simplest exact selection; it runs once per
  // shard at setup (like the reference's precomputed transposes)
  std::vector<u64> rp(a.rows + 1);
  PK_CUDA(cudaMemcpyAsync(rp.data(), a.row_ptr, (a.rows + 1) * sizeof(u64),
                          cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  std::vector<std::pair<u64, i64>> hubs;
  for (i64 i = 0; i < a.rows; ++i) {
    const u64 len = rp[i + 1] - rp[i];
    if (len >= plan.threshold) hubs.push_back({len, i});
  }
  std::stable_sort(hubs.begin(), hubs.end(),
                   [](const auto& x, const auto& y) { return x.first > y.first; });
  std::vector<i64> ids(hubs.size());
  for (size_t i = 0; i < hubs.size(); ++i) ids[i] = hubs[i].second;
  plan.hub_count = static_cast<int>(ids.size());
  if (!ids.empty()) {
    plan.hub_rows.alloc(ids.size());
    PK_CUDA(cudaMemcpyAsync(plan.hub_rows.p, ids.data(), ids.size() * sizeof(i64),
                            cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaStreamSynchronize(st));
  }
}

// Hub rows restricted to [r0, r1): the plan's list is global, so a row-range
// call filters it on the host (cached per range).
const i64* spmm_plan_range(SpmmPlan& plan, i64 r0, i64 r1, int* count,
                           cudaStream_t st) {
  if (plan.hub_count == 0) {
    *count = 0;
    return nullptr;
  }
  if (r0 == 0 && r1 == plan.rows) {
    *count = plan.hub_count;
    return plan.hub_rows.p;
  }
  for (auto& c : plan.range_cache)
    if (c.r0 == r0 && c.r1 == r1) {
      *count = c.count;
      return c.rows.p;
    }
  std::vector<i64> all(plan.hub_count);
  PK_CUDA(cudaMemcpyAsync(all.data(), plan.hub_rows.p, all.size() * sizeof(i64),
                          cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  std::vector<i64> sel;
  for (i64 r : all)
    if (r >= r0 && r < r1) sel.push_back(r);
  SpmmPlan::Range rg;
  rg.r0 = r0, rg.r1 = r1, rg.count = static_cast<int>(sel.size());
  if (!sel.empty()) {
    rg.rows.alloc(sel.size());
    PK_CUDA(cudaMemcpyAsync(rg.rows.p, sel.data(), sel.size() * sizeof(i64),
                            cudaMemcpyHostToDevice, st));
    PK_CUDA(cudaStreamSynchronize(st));
  }
  plan.range_cache.push_back(std::move(rg));
  *count = plan.range_cache.back().count;
  return plan.range_cache.back().rows.p;
}

}  // namespace pk
