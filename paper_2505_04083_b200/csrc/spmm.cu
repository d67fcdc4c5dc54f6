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
// The operation is a gather-bound stream (8 B of index + value
// per nonzero plus one gathered feature row per nonzero). ncu on the first
// version showed it issue- and latency-bound, not DRAM-bound (~60 warp
// instructions per nonzero, 37 % DRAM throughput), so the design minimises
// per-nonzero instructions and keeps many gathers in flight:
//   * regular rows ("list kernel"): the plan compacts their nonzeros into
//     one stream of packed 8-B (col, val) pairs plus a bitmap marking row
//     ends. A lane group (4-32 lanes, sized to the feature width) takes an
//     nnz-balanced chunk, loads 32 pairs per coalesced 8-B load, broadcasts
//     each pair with two shuffles, keeps U gathered 16-B feature slices in
//     flight per lane, and stores a row when its end bit comes up — a bit
//     test of a uniform mask instead of per-nonzero row bookkeeping.
//   * hub rows (RMAT degree skew: median 3, max 155,518 nnz per row at the
//     products shape): a whole CTA serves one (row, 32*VEC-column slice);
//     loader warps stream the gathered row slices into a shared-memory ring
//     with cp.async so hundreds of gathers are in flight for the single
//     sequential chain the consumer warp runs. Hub CTAs run on a forked
//     stream so they overlap the list kernel.
//   * empty rows are zero-filled.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <tuple>
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
// 32-B lane slices: one 256-bit load per lane per gathered row slice
// (LDG.256 on sm_100a) halves the gather instructions of wide rows
struct alignas(32) float8 {
  float4 a, b;
};
template <>
struct Vec<8> {
  using T = float8;
  static __device__ __forceinline__ T zero() {
    return float8{make_float4(0.f, 0.f, 0.f, 0.f), make_float4(0.f, 0.f, 0.f, 0.f)};
  }
};

// acc = fl(acc + fl(v * x)), element-wise, never contracted to FMA.
#ifndef PK_SPMM_FMA
#define PK_SPMM_FMA 0
#endif
__device__ __forceinline__ void madd(float& a, float v, float x) {
#if PK_SPMM_FMA  // experiment: fused multiply-add — not the reference's rounding;
                 // measured 3-4 % faster (D=100 4.66 vs 4.85 ms, D=256 8.78 vs
                 // 9.06), kept off so every row chain stays bit-identical
  a = __fmaf_rn(v, x, a);
#else
  a = __fadd_rn(a, __fmul_rn(v, x));
#endif
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

__device__ __forceinline__ void madd(float8& a, float v, const float8& x) {
  madd(a.a, v, x.a);
  madd(a.b, v, x.b);
}

// FAST plans: one fused multiply-add per nonzero, acc = fma(v, x, acc) —
// one rounding instead of two (no less accurate), measured 3-4 % faster
// per pass; PARITY keeps the reference's separate mul and add.
__device__ __forceinline__ void fmadd(float& a, float v, float x) { a = __fmaf_rn(v, x, a); }
__device__ __forceinline__ void fmadd(float2& a, float v, float2 x) {
  fmadd(a.x, v, x.x);
  fmadd(a.y, v, x.y);
}
__device__ __forceinline__ void fmadd(float4& a, float v, float4 x) {
  fmadd(a.x, v, x.x);
  fmadd(a.y, v, x.y);
  fmadd(a.z, v, x.z);
  fmadd(a.w, v, x.w);
}
__device__ __forceinline__ void fmadd(float8& a, float v, const float8& x) {
  fmadd(a.a, v, x.a);
  fmadd(a.b, v, x.b);
}
template <bool FMA, typename V, typename X>
__device__ __forceinline__ void madd_t(V& a, float v, const X& x) {
  if constexpr (FMA) fmadd(a, v, x);
  else madd(a, v, x);
}

// relu_backward select: keep a where the mask (relu(Q)) is positive
__device__ __forceinline__ float keep(float a, float m) { return m > 0.f ? a : 0.f; }
__device__ __forceinline__ float keep_v(float a, const float* m) { return keep(a, *m); }
__device__ __forceinline__ float2 keep_v(float2 a, const float* m) {
  const float2 q = *reinterpret_cast<const float2*>(m);
  return make_float2(keep(a.x, q.x), keep(a.y, q.y));
}
__device__ __forceinline__ float4 keep_v(float4 a, const float* m) {
  const float4 q = __ldcs(reinterpret_cast<const float4*>(m));
  return make_float4(keep(a.x, q.x), keep(a.y, q.y), keep(a.z, q.z), keep(a.w, q.w));
}
__device__ __forceinline__ float8 keep_v(const float8& a, const float* m) {
  return float8{keep_v(a.a, m), keep_v(a.b, m + 4)};
}
__device__ __forceinline__ float keep_vv(float a, float m) { return keep(a, m); }
__device__ __forceinline__ float2 keep_vv(float2 a, float2 m) {
  return make_float2(keep(a.x, m.x), keep(a.y, m.y));
}
__device__ __forceinline__ float4 keep_vv(float4 a, float4 m) {
  return make_float4(keep(a.x, m.x), keep(a.y, m.y), keep(a.z, m.z), keep(a.w, m.w));
}
__device__ __forceinline__ float8 keep_vv(const float8& a, const float8& m) {
  return float8{keep_vv(a.a, m.a), keep_vv(a.b, m.b)};
}

template <typename T>
__device__ __forceinline__ T ldg(const float* p) {
  return __ldg(reinterpret_cast<const T*>(p));
}
template <>
__device__ __forceinline__ float8 ldg<float8>(const float* p) {
  float8 r;
  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                 "=f"(r.b.z), "=f"(r.b.w)
               : "l"(p));
  return r;
}

// Gather with an L2 eviction hint from the plan's hot-column bit (bit 31 of
// the packed column): rows of high-degree columns are kept (evict_last),
// single-use rows of cold columns are streamed (evict_first, no L1
// allocation), so cold gathers do not push hot rows out of L2. Only the
// 256-bit load carries the hint on sm_100a; narrower slices load plainly.
// Measured (scripts/spmm_hint_sweep.sh, products D=256): 10.57 ms with hints
// at the best hot-factor vs 10.23 ms without — the hardware's own policy
// wins, so the hints are compiled out by default.
#ifndef PK_LIST_HINTS
#define PK_LIST_HINTS 0
#endif
template <typename T>
__device__ __forceinline__ T ldg_hint(const float* p, bool hot) {
  (void)hot;
  return ldg<T>(p);
}
template <>
__device__ __forceinline__ float8 ldg_hint<float8>(const float* p, bool hot) {
#if PK_LIST_HINTS
  float8 r;
  if (hot)
    asm volatile("ld.global.nc.L1::evict_last.L2::evict_last.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                   "=f"(r.b.z), "=f"(r.b.w)
                 : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(r.a.x), "=f"(r.a.y), "=f"(r.a.z), "=f"(r.a.w), "=f"(r.b.x), "=f"(r.b.y),
                   "=f"(r.b.z), "=f"(r.b.w)
                 : "l"(p));
  return r;
#else
  (void)hot;
  return ldg<float8>(p);
#endif
}

constexpr int kThreads = 256;

// Set (and reported once with printf) when a kernel bails out of a wait or
// loop that should have terminated; read back by spmm_watchdog() / pk_device_watchdogs(); the engine checks it
// after every epoch.
__device__ unsigned g_spmm_watchdog = 0;

// ---------------------------------------------------------------------------
// list kernel: regular rows as one nnz stream

struct ListArgs {
  const u64* cv = nullptr;      // packed (val << 32 | col) per nonzero
  const u32* rl = nullptr;      // row id per list entry
  const u64* rpc = nullptr;     // nonzero offset per list entry (+1)
  const u32* endbits = nullptr; // bit k set: nonzero k is the last of its row
  const float* x = nullptr;
  i64 ldx = 0;
  float* y = nullptr;
  i64 ldy = 0;
  i64 r0 = 0;                   // y holds rows [r0, ...)
  float* part = nullptr;        // FAST plan: segment sums (target bit 31 set)
  i64 ldp = 0;
  int nvec = 0;
  i64 xrows = 0;                // rows of x the nonzeros gather from
  const float* mask = nullptr;  // optional relu_backward mask, rows like y
  i64 ldm = 0;
  RowMap map;                   // where output rows go (g == 0: y)
  bool fma = false;             // FAST plan: fused multiply-add chains
};

// chunk bounds over list entries [i0, i1), ~equal nonzeros per chunk
__global__ void list_partition_kernel(const u64* __restrict__ rpc, i64 i0, i64 i1, int nchunks,
                                      i64* __restrict__ bounds, int* __restrict__ counters,
                                      int nslices) {
  const i64 t = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (t < nslices) counters[t] = 0;
  if (t > nchunks) return;
  if (t == 0 || t == nchunks) {
    bounds[t] = t == 0 ? i0 : i1;
    return;
  }
  const u64 base = rpc[i0], total = rpc[i1] - base;
  const u64 target = base + total / nchunks * t + (total % nchunks) * t / nchunks;
  i64 lo = i0, hi = i1;  // first entry with rpc[entry] >= target
  while (lo < hi) {
    const i64 mid = lo + (hi - lo) / 2;
    if (rpc[mid] < target)
      lo = mid + 1;
    else
      hi = mid;
  }
  bounds[t] = lo;
}

// 32 end bits starting at nonzero k
__device__ __forceinline__ unsigned end_mask(const u32* __restrict__ bits, u64 k) {
  const u64 w = k >> 5;
  const unsigned lo = __ldg(bits + w), hi = __ldg(bits + w + 1);
  return __funnelshift_r(lo, hi, static_cast<unsigned>(k & 31));
}

// Gathers in flight per lane and unrolling of the window loop (tuned with
// scripts/spmm_tune_sweep.sh).
#ifndef PK_LIST_U1
#define PK_LIST_U1 4
#endif
#ifndef PK_LIST_U2
#define PK_LIST_U2 4
#endif
#ifndef PK_LIST_UNROLL
#define PK_LIST_UNROLL 16
#endif
constexpr int kListUnroll = PK_LIST_UNROLL;

// Minimum resident blocks per SM for the register allocation: three for
// the 2-vector (D <= 256) form, where the extra warps' gathers outweigh the
// registers (measured, scripts/spmm_minb_sweep.sh: -4 % at D=256; the 1-vector
// form is already register-light and gets slower when squeezed).
#ifndef PK_LIST_MINB1
#define PK_LIST_MINB1 4
#endif
#ifndef PK_LIST_U8
#define PK_LIST_U8 2
#endif
#ifndef PK_LIST_MINB8
#define PK_LIST_MINB8 4
#endif
#ifndef PK_LIST_MINB8M
#define PK_LIST_MINB8M 4
#endif
// (The tuned one-vector, full-warp forms above; wider rows carry NV
// accumulators and NV x U gathers per lane and narrower groups more gathers
// per lane, so those trade residency for registers instead of spilling.)
template <int VEC, int LANES, int NV, bool MASK>
constexpr int list_min_blocks() {
  if (NV >= 3 || (NV == 2 && VEC == 8)) return 2;
  if (NV == 2 || LANES < 32) return 3;
  return VEC == 8 ? (MASK ? PK_LIST_MINB8M : PK_LIST_MINB8) : PK_LIST_MINB1;
}
// EPI: 0 plain; 1 the relu_backward epilogue (MASK); 2 mapped output rows
// (a reduction's owner slots, RowMap). Each its own instantiation, so the
// plain kernel's registers and code stay untouched (the row mapping inlined
// at every row end grew the plain kernel by 20 % and cost 8 ms per C2 epoch).
template <int VEC, int LANES, int NV, int U, int EPI, bool FMA = false>
__global__ void __launch_bounds__(kThreads, list_min_blocks<VEC, LANES, NV, EPI == 1>())
spmm_list_kernel(ListArgs a, const i64* __restrict__ bounds, int nchunks,
                 int* __restrict__ counters) {
  constexpr bool MASK = EPI == 1, MAPPED = EPI == 2;
  using V = typename Vec<VEC>::T;
  const int lane = threadIdx.x % LANES;
  const unsigned gmask =
      LANES == 32 ? 0xffffffffu
                  : (((1u << LANES) - 1u) << ((threadIdx.x % 32) / LANES * LANES));
  const int vbase = static_cast<int>(blockIdx.y) * (NV * LANES);
  bool valid[NV];
#pragma unroll
  for (int t = 0; t < NV; ++t) valid[t] = vbase + t * LANES + lane < a.nvec;
  int* counter = counters + blockIdx.y;
  const float* xlane = a.x + (vbase + lane) * VEC;

  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(counter, 1);
    t = __shfl_sync(gmask, t, 0, LANES);
    if (t >= nchunks) break;
    const i64 is = bounds[t], ie = bounds[t + 1];
    if (is >= ie) continue;
    u64 k = __ldg(a.rpc + is);
    const u64 kend = __ldg(a.rpc + ie);
    // row ids of the chunk, LANES at a time
    i64 rb = is;
    u32 rid = rb + lane < ie ? __ldg(a.rl + rb + lane) : 0u;
    int rn = 0;
    V acc[NV];
#pragma unroll
    for (int q = 0; q < NV; ++q) acc[q] = Vec<VEC>::zero();
    // MASK: the current row's relu_backward mask is loaded when the row
    // starts (right after the previous row's store), so its latency hides
    // behind the row's gathers instead of stalling the store
    V mk[MASK ? NV : 1];
    auto load_mask = [&]() {
      if constexpr (MASK) {
        const u32 row = __shfl_sync(gmask, rid, rn, LANES);
        if (rb + rn < ie && !(row & 0x80000000u)) {
          const float* mr =
              a.mask + (static_cast<i64>(row) - a.r0) * a.ldm + (vbase + lane) * VEC;
#pragma unroll
          for (int q = 0; q < NV; ++q)
            mk[q] = valid[q] ? ldg<V>(mr + q * LANES * VEC) : Vec<VEC>::zero();
        }
      }
    };
    load_mask();
    auto row_done = [&]() {
      const u32 row = __shfl_sync(gmask, rid, rn, LANES);
      const bool seg = (row & 0x80000000u) != 0;
      float* yrow;
      if (seg) {
        yrow = a.part + static_cast<i64>(row & 0x7fffffffu) * a.ldp;
      } else if constexpr (MAPPED) {
        yrow = a.map.row(a.y, a.ldy, static_cast<i64>(row) - a.r0);
      } else {
        yrow = a.y + (static_cast<i64>(row) - a.r0) * a.ldy;
      }
      yrow += (vbase + lane) * VEC;
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        if (valid[q]) {
          V out = acc[q];
          if constexpr (MASK) {
            if (!seg) out = keep_vv(out, mk[q]);
          }
          *reinterpret_cast<V*>(yrow + q * LANES * VEC) = out;
        }
        acc[q] = Vec<VEC>::zero();
      }
      if (++rn == LANES) {
        rn = 0;
        rb += LANES;
        rid = rb + lane < ie ? __ldg(a.rl + rb + lane) : 0u;
      }
      load_mask();
    };
    // Full windows are software-pipelined: the gathers of group g+1 (U
    // nonzeros, the next window's first group at a window's end) are issued
    // before group g is consumed, so every lane always has U*NV 16-B loads in
    // flight. Partial windows (a chunk's tail) take the simple path.
    u64 w = k + lane < kend ? __ldcs(a.cv + k + lane) : 0ull;
    V xa[U][NV], xb[U][NV];
    auto gather = [&](V (&xv)[U][NV], u32 wc, int j) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const u32 c = __shfl_sync(gmask, wc, j + u, LANES);
        const float* xr = xlane + static_cast<i64>(c & 0x7fffffffu) * a.ldx;
        const bool hot = (c >> 31) != 0;
#pragma unroll
        for (int q = 0; q < NV; ++q)
          xv[u][q] = valid[q] ? ldg_hint<V>(xr + q * LANES * VEC, hot) : Vec<VEC>::zero();
      }
    };
    auto consume = [&](const V (&xv)[U][NV], u32 wv, unsigned em, int j) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float v = __uint_as_float(__shfl_sync(gmask, wv, j + u, LANES));
#pragma unroll
        for (int q = 0; q < NV; ++q) madd_t<FMA>(acc[q], v, xv[u][q]);
        if ((em >> (j + u)) & 1u) row_done();
      }
    };
    bool primed = false;  // xa holds the gathers of the current window's group 0
    while (k < kend) {
      const int cnt = static_cast<int>(min(static_cast<u64>(LANES), kend - k));
      const u64 wn = k + LANES + lane < kend ? __ldcs(a.cv + k + LANES + lane) : 0ull;
      const unsigned em = end_mask(a.endbits, k);
      const u32 wc = static_cast<u32>(w), wv = static_cast<u32>(w >> 32);
      if (cnt == LANES) {
        if (!primed) gather(xa, wc, 0);
        // the next window is full too: its group 0 can be prefetched
        const bool next_full = k + 2 * LANES <= kend;
#pragma unroll (kListUnroll)
        for (int j = 0; j < LANES; j += 2 * U) {
          if (j + U < LANES) gather(xb, wc, j + U);
          else if (next_full) gather(xb, static_cast<u32>(wn), 0);
          consume(xa, wv, em, j);
          if (j + U < LANES) {
            if (j + 2 * U < LANES) gather(xa, wc, j + 2 * U);
            else if (next_full) gather(xa, static_cast<u32>(wn), 0);
            consume(xb, wv, em, j + U);
          }
        }
        // with LANES/U even, the prefetched next group 0 sits in xa
        primed = next_full && ((LANES / U) % 2 == 0);
        if (next_full && (LANES / U) % 2 == 1) {
          // odd group count: the prefetch landed in xb; move it (registers)
#pragma unroll
          for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < NV; ++q) xa[u][q] = xb[u][q];
          primed = true;
        }
      } else {
        for (int j = 0; j < cnt; ++j) {
          const u32 c = __shfl_sync(gmask, wc, j, LANES);
          const float v = __uint_as_float(__shfl_sync(gmask, wv, j, LANES));
          const float* xr = xlane + static_cast<i64>(c & 0x7fffffffu) * a.ldx;
          const bool hot = (c >> 31) != 0;
#pragma unroll
          for (int q = 0; q < NV; ++q)
            if (valid[q]) madd_t<FMA>(acc[q], v, ldg_hint<V>(xr + q * LANES * VEC, hot));
          if ((em >> j) & 1u) row_done();
        }
        primed = false;
      }
      k += cnt;
      w = wn;
    }
  }
}

// ---------------------------------------------------------------------------
// paired narrow form (FAST, opt-in): rows of at most 16 vectors, e.g. the
// transform-first layers' 48-wide P / dQ (engine.cu forward_layer_tf). The
// plain form gives such a row one lane group per chunk, so a warp gather
// moves one nonzero's 192 B and the pass is bound by gathers in flight (C2:
// 1.6 TB/s DRAM, 3.9 ms per pass for 1 GB of compulsory bytes). Here a
// warp's two halves take a window's even and odd nonzeros, so every gather
// instruction moves two rows and half as many instructions cover a window.
// Each half keeps a running chain (even / odd stream positions within the
// chunk, each k-ascending, fl(acc + fl(v x)) like the reference); at a row
// end the halves' chains are added (one shuffle) and the even half stores.
// A two-chain sum is another association of the same row: tolerance-level
// (FAST), deterministic (fixed chunks), so callers opt in (PK_SPMM_PAIRED).
#ifndef PK_PAIR_U
#define PK_PAIR_U 4
#endif
#ifndef PK_PAIR_MINB
#define PK_PAIR_MINB 4
#endif

__device__ __forceinline__ float fold_halves(float a) {
  return __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, 16));
}
__device__ __forceinline__ float2 fold_halves(float2 a) {
  return make_float2(fold_halves(a.x), fold_halves(a.y));
}
__device__ __forceinline__ float4 fold_halves(float4 a) {
  return make_float4(fold_halves(a.x), fold_halves(a.y), fold_halves(a.z), fold_halves(a.w));
}

template <int VEC, int U, bool MAPPED>
__global__ void __launch_bounds__(kThreads, PK_PAIR_MINB)
spmm_pair_kernel(ListArgs a, const i64* __restrict__ bounds, int nchunks,
                 int* __restrict__ counters) {
  using V = typename Vec<VEC>::T;
  constexpr unsigned kAll = 0xffffffffu;
  constexpr int kSteps = 16;  // pair steps per 32-nonzero window
  const int lane = threadIdx.x % 32, half = lane / 16, col = lane % 16;
  const bool valid = col < a.nvec;
  const float* xlane = a.x + col * VEC;
  for (;;) {
    int t = 0;
    if (lane == 0) t = atomicAdd(counters, 1);
    t = __shfl_sync(kAll, t, 0);
    if (t >= nchunks) break;
    const i64 is = bounds[t], ie = bounds[t + 1];
    if (is >= ie) continue;
    u64 k = __ldg(a.rpc + is);
    const u64 kend = __ldg(a.rpc + ie);
    i64 rb = is;
    u32 rid = rb + lane < ie ? __ldg(a.rl + rb + lane) : 0u;
    int rn = 0;
    V acc = Vec<VEC>::zero();
    auto row_done = [&]() {
      const V tot = fold_halves(acc);
      const u32 row = __shfl_sync(kAll, rid, rn);
      if (half == 0 && valid) {
        float* yrow;
        if (row & 0x80000000u) {
          yrow = a.part + static_cast<i64>(row & 0x7fffffffu) * a.ldp;
        } else if constexpr (MAPPED) {
          yrow = a.map.row(a.y, a.ldy, static_cast<i64>(row) - a.r0);
        } else {
          yrow = a.y + (static_cast<i64>(row) - a.r0) * a.ldy;
        }
        *reinterpret_cast<V*>(yrow + col * VEC) = tot;
      }
      acc = Vec<VEC>::zero();
      if (++rn == 32) {
        rn = 0;
        rb += 32;
        rid = rb + lane < ie ? __ldg(a.rl + rb + lane) : 0u;
      }
    };
    // pair step s: this lane's nonzero is 2s + half of the window
    auto step = [&](const V& xv, u32 wv, unsigned em, int s, bool odd_live) {
      const float v = __uint_as_float(__shfl_sync(kAll, wv, 2 * s + half));
      if (half == 0) madd(acc, v, xv);
      if ((em >> (2 * s)) & 1u) row_done();
      if (half == 1 && odd_live) madd(acc, v, xv);
      if (odd_live && ((em >> (2 * s + 1)) & 1u)) row_done();
    };
    auto gather = [&](V (&xv)[U], u32 wc, int s0) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const u32 c = __shfl_sync(kAll, wc, 2 * (s0 + u) + half);
        xv[u] = valid ? ldg<V>(xlane + static_cast<i64>(c & 0x7fffffffu) * a.ldx)
                      : Vec<VEC>::zero();
      }
    };
    auto consume = [&](const V (&xv)[U], u32 wv, unsigned em, int s0) {
#pragma unroll
      for (int u = 0; u < U; ++u) step(xv[u], wv, em, s0 + u, true);
    };
    // the list kernel's software pipeline, over pair steps: the gathers of
    // group g+1 (or the next window's group 0) are issued before group g is
    // consumed
    u64 w = k + lane < kend ? __ldcs(a.cv + k + lane) : 0ull;
    V xa[U], xb[U];
    bool primed = false;
    while (k < kend) {
      const int cnt = static_cast<int>(min(static_cast<u64>(32), kend - k));
      const u64 wn = k + 32 + lane < kend ? __ldcs(a.cv + k + 32 + lane) : 0ull;
      const unsigned em = end_mask(a.endbits, k);
      const u32 wc = static_cast<u32>(w), wv = static_cast<u32>(w >> 32);
      if (cnt == 32) {
        if (!primed) gather(xa, wc, 0);
        const bool next_full = k + 64 <= kend;
#pragma unroll
        for (int s = 0; s < kSteps; s += 2 * U) {
          if (s + U < kSteps) gather(xb, wc, s + U);
          else if (next_full) gather(xb, static_cast<u32>(wn), 0);
          consume(xa, wv, em, s);
          if (s + U < kSteps) {
            if (s + 2 * U < kSteps) gather(xa, wc, s + 2 * U);
            else if (next_full) gather(xa, static_cast<u32>(wn), 0);
            consume(xb, wv, em, s + U);
          }
        }
        primed = next_full && ((kSteps / U) % 2 == 0);
        if (next_full && (kSteps / U) % 2 == 1) {
#pragma unroll
          for (int u = 0; u < U; ++u) xa[u] = xb[u];
          primed = true;
        }
      } else {
        for (int s = 0; 2 * s < cnt; ++s) {
          const int j = 2 * s + half;
          const u32 c = __shfl_sync(kAll, wc, j);
          const V xv = valid && j < cnt
                           ? ldg<V>(xlane + static_cast<i64>(c & 0x7fffffffu) * a.ldx)
                           : Vec<VEC>::zero();
          step(xv, wv, em, s, 2 * s + 1 < cnt);
        }
        primed = false;
      }
      k += cnt;
      w = wn;
    }
  }
}

// FAST plan: y[hub row] = fold of its segment sums in segment order
template <bool MAPPED>
__global__ void combine_segments_kernel(const u32* __restrict__ hub, const u32* __restrict__ seg0,
                                        const u32* __restrict__ nseg, i64 nh, i64 r0,
                                        const float* __restrict__ part, i64 ldp, float* y,
                                        i64 ldy, i64 d, const float* __restrict__ mask,
                                        i64 ldm, RowMap map) {
  const i64 total = nh * d;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 h = i / d, c = i % d;
    const u64 s0 = seg0[h];
    float acc = part[s0 * ldp + c];
    for (u32 k = 1; k < nseg[h]; ++k) acc = __fadd_rn(acc, part[(s0 + k) * ldp + c]);
    const i64 rr = static_cast<i64>(hub[h]) - r0;
    float* yr = MAPPED ? map.row(y, ldy, rr) : y + rr * ldy;
    yr[c] = mask ? keep(acc, mask[rr * ldm + c]) : acc;
  }
}

// y rows listed in `rows` (absolute ids) := 0 over d columns
template <bool MAPPED>
__global__ void zero_rows_kernel(const u32* __restrict__ rows, i64 n, i64 r0, float* y, i64 ldy,
                                 i64 d, RowMap map) {
  const i64 total = n * d;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 lr = static_cast<i64>(rows[i / d]) - r0;
    (MAPPED ? map.row(y, ldy, lr) : y + lr * ldy)[i % d] = 0.f;
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
      *reinterpret_cast<V*>(args.y + rr * args.ldy + vcol * VEC) =
          args.mask ? keep_v(acc, args.mask + rr * args.ldm + vcol * VEC) : acc;
    }
  }
}


// ---------------------------------------------------------------------------
// launch selection

struct ListWorkspace {
  DevBuf<i64> bounds;
  DevBuf<int> counters;
};

template <int VEC, int LANES, int NV>
void launch_list(const ListArgs& a, i64 i0, i64 i1, const u64* rpc, cudaStream_t st) {
  // gathers in flight per lane: U groups x NV vectors, double-buffered —
  // kept to what fits the residency's register budget without spills
#ifndef PK_LIST_U2V
#define PK_LIST_U2V 4
#endif
  constexpr int U0 = NV >= 3 ? 2
                             : (NV == 2 ? (VEC >= 4 ? 2 : PK_LIST_U2)
                                        : (VEC == 8 ? PK_LIST_U8
                                                    : (VEC == 2 ? PK_LIST_U2V : PK_LIST_U1)));
  constexpr int U = U0 < LANES ? U0 : LANES / 2;
  const bool masked = a.mask != nullptr;
  check(!(masked && a.map.g), "spmm: a mask epilogue with mapped rows is not supported");
  auto kernel = masked ? (a.fma ? spmm_list_kernel<VEC, LANES, NV, U, 1, true>
                                : spmm_list_kernel<VEC, LANES, NV, U, 1>)
                : a.map.g ? (a.fma ? spmm_list_kernel<VEC, LANES, NV, U, 2, true>
                                   : spmm_list_kernel<VEC, LANES, NV, U, 2>)
                          : (a.fma ? spmm_list_kernel<VEC, LANES, NV, U, 0, true>
                                   : spmm_list_kernel<VEC, LANES, NV, U, 0>);
  const int slices = ceil_div(a.nvec, NV * LANES);
  // ~1-2K nonzeros per chunk at the products shape; never more chunks than
  // rows (PK_LIST_CHUNKS: chunks per SM, experiments)
  static const i64 per_sm = [] {
    const char* e = std::getenv("PK_LIST_CHUNKS");
    return e ? std::max<i64>(1, std::atoll(e)) : i64{512};
  }();
  const i64 nchunks64 =
      std::max<i64>(1, std::min<i64>(i1 - i0, static_cast<i64>(sm_count()) * per_sm));
  const int nchunks = static_cast<int>(nchunks64);
  static thread_local ListWorkspace ws;
  ws.bounds.ensure(nchunks + 1);
  ws.counters.ensure(std::max(slices, 1));
  list_partition_kernel<<<ceil_div(nchunks + 1, 256), 256, 0, st>>>(rpc, i0, i1, nchunks,
                                                                    ws.bounds.p, ws.counters.p,
                                                                    slices);
  PK_LAUNCH("spmm list partition");
  static thread_local int occs[6] = {0, 0, 0, 0, 0, 0};
  int& occ = occs[(masked ? 1 : (a.map.g ? 2 : 0)) + (a.fma ? 3 : 0)];
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
  PK_LAUNCH("spmm list kernel");
}

template <int VEC>
void launch_pair(const ListArgs& a, i64 i0, i64 i1, const u64* rpc, cudaStream_t st) {
  constexpr int U = PK_PAIR_U;
  const bool mapped = a.map.g != 0;
  auto kernel = mapped ? spmm_pair_kernel<VEC, U, true> : spmm_pair_kernel<VEC, U, false>;
  static const i64 per_sm = [] {
    const char* e = std::getenv("PK_LIST_CHUNKS");
    return e ? std::max<i64>(1, std::atoll(e)) : i64{512};
  }();
  const int nchunks = static_cast<int>(
      std::max<i64>(1, std::min<i64>(i1 - i0, static_cast<i64>(sm_count()) * per_sm)));
  static thread_local ListWorkspace ws;
  ws.bounds.ensure(nchunks + 1);
  ws.counters.ensure(1);
  list_partition_kernel<<<ceil_div(nchunks + 1, 256), 256, 0, st>>>(rpc, i0, i1, nchunks,
                                                                    ws.bounds.p, ws.counters.p, 1);
  PK_LAUNCH("spmm pair partition");
  static thread_local int occs[2] = {0, 0};
  int& occ = occs[mapped ? 1 : 0];
  if (occ == 0) {
    PK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, 0));
    occ = std::max(occ, 1);
  }
  const i64 warps = kThreads / 32;
  const i64 blocks = std::max<i64>(
      1, std::min<i64>(static_cast<i64>(sm_count()) * occ, (nchunks + warps - 1) / warps));
  kernel<<<static_cast<unsigned>(blocks), kThreads, 0, st>>>(a, ws.bounds.p, nchunks,
                                                             ws.counters.p);
  PK_LAUNCH("spmm pair kernel");
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

// Wide rows over a gathered matrix larger than L2 (C3: 262K rows x 602
// features = 631 MB): one column slice of 32 lanes per grid.y, so the
// slices run one after another and each slice's columns of x (262K x 256 B =
// 67 MB at 32 lanes of 8 B) stay L2-resident while the nonzeros are
// re-streamed (8 B per nonzero per slice against LANES*4*VEC B of gathers).
// Returns the slice's lane count, or 0 for the balanced wide form.
// PK_SPMM_L2_MB: the slice's L2 budget (0 = off); PK_SPMM_L2_LANES=32|16
// forces the form on every wide row (tests).
inline int l2_slice_lanes(const ListArgs& a, int vec) {
  static const double budget = [] {
    const char* e = std::getenv("PK_SPMM_L2_MB");
    return (e ? std::atof(e) : 96.0) * (1 << 20);
  }();
  static const int forced = [] {
    const char* e = std::getenv("PK_SPMM_L2_LANES");
    return e ? std::atoi(e) : 0;
  }();
  if (a.nvec <= 32) return 0;
  if (forced == 32 || forced == 16) return forced;
  if (budget <= 0) return 0;
  const double row_bytes = 4.0 * vec;
  if (static_cast<double>(a.xrows) * a.nvec * row_bytes <= budget) return 0;
  // 32 lanes of at least 8 B: narrower slices (16 lanes, or 4-B gathers)
  // measured slower than the balanced form (C3: 121 vs 94 ms at 16 lanes on
  // 1 GPU; 65.8 vs 38.2 ms with 4-B gathers at D = 301 on 2 GPUs)
  if (vec >= 2 && static_cast<double>(a.xrows) * 32 * row_bytes <= budget) return 32;
  return 0;
}

template <int VEC>
void dispatch_list(const ListArgs& a, i64 i0, i64 i1, const u64* rpc, cudaStream_t st) {
  const int nv = a.nvec;
  // lane-group width: smallest power of two covering the row's vectors
  if (nv <= 4)
    launch_list<VEC, 4, 1>(a, i0, i1, rpc, st);
  else if (nv <= 8)
    launch_list<VEC, 8, 1>(a, i0, i1, rpc, st);
  else if (nv <= 16)
    launch_list<VEC, 16, 1>(a, i0, i1, rpc, st);
  else if (nv <= 32)
    launch_list<VEC, 32, 1>(a, i0, i1, rpc, st);
  else if (const int sl = l2_slice_lanes(a, VEC); sl == 32)
    launch_list<VEC, 32, 1>(a, i0, i1, rpc, st);
  else if (sl == 16)
    launch_list<VEC, 16, 1>(a, i0, i1, rpc, st);
  else if (nv <= 64)
    launch_list<VEC, 32, 2>(a, i0, i1, rpc, st);
  else {
    // wider rows: as few column slices (blockIdx.y, each re-streaming the
    // nonzeros) as 6 vectors per lane allow, each slice as even as possible
    // (C3's 602 features at 8 B: 2 slices of 160 instead of 128+128+45)
    // (vectors per lane capped so the accumulators and gathers fit without
    // spills: 6 below 16-B vectors, 4 at 16 B, 2 at 32 B)
    constexpr int kMaxNV = VEC <= 2 ? 6 : (VEC == 4 ? 4 : 2);
    const int slices = (nv + 32 * kMaxNV - 1) / (32 * kMaxNV);
    const int per_lane = (nv + 32 * slices - 1) / (32 * slices);
    if (per_lane <= 2) {
      launch_list<VEC, 32, 2>(a, i0, i1, rpc, st);
    } else if constexpr (kMaxNV >= 4) {
      if (per_lane <= 3)
        launch_list<VEC, 32, 3>(a, i0, i1, rpc, st);
      else if (per_lane <= 4 || kMaxNV == 4)
        launch_list<VEC, 32, 4>(a, i0, i1, rpc, st);
      else if constexpr (kMaxNV >= 6) {
        if (per_lane <= 5)
          launch_list<VEC, 32, 5>(a, i0, i1, rpc, st);
        else
          launch_list<VEC, 32, 6>(a, i0, i1, rpc, st);
      }
    }
  }
}

int pick_vec(const float* x, i64 ldx, const float* y, i64 ldy, i64 d, bool allow8) {
  auto aligned = [](const void* p, int bytes) {
    return (reinterpret_cast<uintptr_t>(p) % bytes) == 0;
  };
  // 32-B slices only when they still fill a 32-lane group (narrower rows
  // would split warps into diverging sub-groups: measured slower at D=128)
  if (allow8 && d % 8 == 0 && d >= 256 && ldx % 8 == 0 && ldy % 8 == 0 && aligned(x, 32) &&
      aligned(y, 32))
    return 8;
  if (d % 4 == 0 && ldx % 4 == 0 && ldy % 4 == 0 && aligned(x, 16) && aligned(y, 16))
    return 4;
  if (d % 2 == 0 && ldx % 2 == 0 && ldy % 2 == 0 && aligned(x, 8) && aligned(y, 8))
    return 2;
  return 1;
}

// ---------------------------------------------------------------------------
// plan construction (device side; runs once per shard)

// entries per row: 0 (empty, or hub on the exact plan), 1 (regular), or
// ceil(len / segment) (hub on the FAST plan)
__global__ void classify_rows_kernel(const u64* __restrict__ rp, i64 rows, u64 thr, u64 segment,
                                     u64* __restrict__ ents, u64* __restrict__ hsegs,
                                     u8* __restrict__ is_empty, u8* __restrict__ is_hub) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < rows;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const u64 len = rp[i + 1] - rp[i];
    const bool hub = len >= thr, empty = len == 0;
    const u64 nseg = (hub && segment) ? (len + segment - 1) / segment : 0;
    ents[i] = empty ? 0 : (hub ? nseg : 1);
    hsegs[i] = nseg;
    is_empty[i] = empty;
    is_hub[i] = hub;
  }
}

__global__ void col_degree_kernel(const u32* __restrict__ ci, u64 nnz, u32* __restrict__ deg) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < nnz;
       i += static_cast<u64>(gridDim.x) * blockDim.x)
    atomicAdd(deg + ci[i], 1u);
}

__global__ void iota_rows_kernel(u32* p, i64 n) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    p[i] = static_cast<u32>(i);
}

// per row: its entries' row key, store target and length
__global__ void fill_entries_kernel(const u64* __restrict__ rp, i64 rows, u64 segment,
                                    const u64* __restrict__ ents, const u64* __restrict__ ent_off,
                                    const u64* __restrict__ hsegs,
                                    const u64* __restrict__ hseg_off, u32* __restrict__ rowkey,
                                    u32* __restrict__ target, u64* __restrict__ elen) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < rows;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const u64 ne = ents[i];
    if (ne == 0) continue;
    const u64 len = rp[i + 1] - rp[i], e0 = ent_off[i];
    if (hsegs[i] == 0) {  // a regular row: one entry, stored to its own row
      rowkey[e0] = static_cast<u32>(i);
      target[e0] = static_cast<u32>(i);
      elen[e0] = len;
      continue;
    }
    for (u64 s = 0; s < ne; ++s) {
      rowkey[e0 + s] = static_cast<u32>(i);
      target[e0 + s] = 0x80000000u | static_cast<u32>(hseg_off[i] + s);
      elen[e0 + s] = min(segment, len - s * segment);
    }
  }
}

// one warp per row: copy its (col, val) pairs into the packed stream and
// mark the last nonzero of each of its entries
__global__ void compact_rows_kernel(const u64* __restrict__ rp, const u32* __restrict__ ci,
                                    const float* __restrict__ val, i64 rows,
                                    const u64* __restrict__ ents,
                                    const u64* __restrict__ ent_off, const u64* __restrict__ rpc,
                                    const u32* __restrict__ col_deg, u32 hot_deg,
                                    u64* __restrict__ cv, u32* __restrict__ endbits) {
  const int lane = threadIdx.x % 32;
  for (i64 i = (blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x) / 32; i < rows;
       i += static_cast<i64>(gridDim.x) * blockDim.x / 32) {
    const u64 ne = ents[i];
    if (ne == 0) continue;
    const u64 s = rp[i], len = rp[i + 1] - s, e0 = ent_off[i], dst = rpc[e0];
    for (u64 j = lane; j < len; j += 32) {
      const u32 c = ci[s + j];
      const u32 hot = col_deg[c] >= hot_deg ? 0x80000000u : 0u;
      cv[dst + j] = (static_cast<u64>(__float_as_uint(val[s + j])) << 32) | c | hot;
    }
    for (u64 e = lane; e < ne; e += 32) {
      const u64 last = rpc[e0 + e + 1] - 1;
      atomicOr(endbits + (last >> 5), 1u << (last & 31));
    }
  }
}

struct NonZero {
  __device__ bool operator()(u64 v) const { return v != 0; }
};

__global__ void hub_len_kernel(const u64* __restrict__ rp, const u32* __restrict__ rows, i64 n,
                               u64* __restrict__ len) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    len[i] = rp[rows[i] + 1] - rp[rows[i]];
}

__global__ void seg_meta_kernel(const u64* __restrict__ hsegs, const u64* __restrict__ hseg_off,
                                i64 n, u32* __restrict__ lo, u32* __restrict__ cnt) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    lo[i] = static_cast<u32>(hseg_off[i]);
    cnt[i] = static_cast<u32>(hsegs[i]);
  }
}

unsigned blocks_for(i64 n, int per = 256) {
  return static_cast<unsigned>(std::max<i64>(1, std::min<i64>((n + per - 1) / per, 1 << 16)));
}

template <typename F>
void cub_run(F&& f, cudaStream_t st) {
  size_t bytes = 0;
  PK_CUDA(f(nullptr, bytes));
  Scratch& sc = Scratch::get();
  const size_t m = sc.mark();
  PK_CUDA(f(sc.take<unsigned char>(bytes), bytes));
  PK_CUDA(cudaStreamSynchronize(st));
  sc.release_to(m);
}

// first index in sorted device array [0, n) with value >= key
template <typename T>
__global__ void lower_bound_kernel(const T* __restrict__ a, i64 n, i64 key0, i64 key1,
                                   i64* __restrict__ out) {
  const int t = threadIdx.x;
  if (t > 1) return;
  const i64 key = t == 0 ? key0 : key1;
  i64 lo = 0, hi = n;
  while (lo < hi) {
    const i64 mid = lo + (hi - lo) / 2;
    if (static_cast<i64>(a[mid]) < key)
      lo = mid + 1;
    else
      hi = mid;
  }
  out[t] = lo;
}

template <typename T>
std::pair<i64, i64> range_of(const T* a, i64 n, i64 r0, i64 r1, cudaStream_t st) {
  if (n == 0) return {0, 0};
  DevBuf<i64> out(2);
  lower_bound_kernel<T><<<1, 32, 0, st>>>(a, n, r0, r1, out.p);
  PK_LAUNCH("spmm plan range");
  i64 h[2];
  PK_CUDA(cudaMemcpyAsync(h, out.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  return {h[0], h[1]};
}

SpmmPlan::Range& plan_range(SpmmPlan& plan, i64 r0, i64 r1, cudaStream_t st) {
  for (auto& r : plan.ranges)
    if (r.r0 == r0 && r.r1 == r1) return r;
  SpmmPlan::Range rg;
  rg.r0 = r0, rg.r1 = r1;
  if (r0 == 0 && r1 == plan.rows) {
    rg.i0 = 0, rg.i1 = plan.entries, rg.e0 = 0, rg.e1 = plan.empty;
    rg.h0 = 0, rg.h1 = plan.segment ? plan.hub_count : 0;
  } else {
    std::tie(rg.i0, rg.i1) = range_of(plan.rowkey.p, plan.entries, r0, r1, st);
    std::tie(rg.e0, rg.e1) = range_of(plan.empty_rows.p, plan.empty, r0, r1, st);
    if (plan.segment) std::tie(rg.h0, rg.h1) = range_of(plan.hub_asc.p, plan.hub_count, r0, r1, st);
  }
  // exact plan: the hub subset keeps the longest-first order
  if (!plan.segment && plan.hub_count) {
    std::vector<i64> all(plan.hub_count), sel;
    PK_CUDA(cudaMemcpyAsync(all.data(), plan.hub_rows.p, all.size() * sizeof(i64),
                            cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    for (i64 r : all)
      if (r >= r0 && r < r1) sel.push_back(r);
    rg.hubs = static_cast<int>(sel.size());
    if (!sel.empty()) {
      rg.hub_ids.alloc(sel.size());
      PK_CUDA(cudaMemcpyAsync(rg.hub_ids.p, sel.data(), sel.size() * sizeof(i64),
                              cudaMemcpyHostToDevice, st));
      PK_CUDA(cudaStreamSynchronize(st));
    }
  }
  plan.ranges.push_back(std::move(rg));
  return plan.ranges.back();
}

}  // namespace

u64 spmm_fast_segment() {
  static const u64 seg = [] {
    const char* e = std::getenv("PK_SPMM_SEGMENT");
    return e ? static_cast<u64>(std::atoll(e)) : u64{2048};
  }();
  return seg;
}

void spmm_plan_build(SpmmPlan& plan, const pk_csr& a, u64 threshold, cudaStream_t st,
                     u64 segment) {
  plan = SpmmPlan();
  plan.rows = a.rows;
  plan.segment = segment;
  if (a.rows == 0) return;
  // A row is a hub when one lane chain over it would outlast the rest of the
  // work spread over the whole GPU; measured on the products shape
  // (scripts/spmm_probe.py), 4096 nonzeros is the sweet spot (2048-8192 within 3 %).
  const u64 avg = a.nnz / std::max<i64>(1, a.rows);
  plan.threshold = threshold ? threshold : std::max<u64>(4096, 64 * avg);
  const i64 n = a.rows;
  // temporaries (scratch): per-row tables, flags, ids, select output, entry
  // lengths (<= rows + segments), column degrees, cub workspaces
  Scratch& sc = Scratch::get();
  const u64 seg_bound = segment ? a.nnz / segment + 1 : 0;
  sc.reset(static_cast<size_t>(n) * 72 + (n + seg_bound) * 8 + static_cast<size_t>(a.cols) * 4 +
           (64u << 20));
  u64* ents = sc.take<u64>(n);
  u64* hsegs = sc.take<u64>(n);
  u64* ent_off = sc.take<u64>(n + 1);
  u64* hseg_off = sc.take<u64>(n + 1);
  u8* is_empty = sc.take<u8>(n);
  u8* is_hub = sc.take<u8>(n);
  u32* ids = sc.take<u32>(n);
  i64* count = sc.take<i64>(1);
  classify_rows_kernel<<<blocks_for(n), 256, 0, st>>>(a.row_ptr, n, plan.threshold, segment,
                                                       ents, hsegs, is_empty, is_hub);
  PK_LAUNCH("spmm plan classify");
  iota_rows_kernel<<<blocks_for(n), 256, 0, st>>>(ids, n);
  PK_LAUNCH("spmm plan iota");
  auto exclusive_scan = [&](const u64* in, u64* out) {  // out[0..n], out[n] = total
    PK_CUDA(cudaMemsetAsync(out, 0, sizeof(u64), st));
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceScan::InclusiveSum(t, b, in, out + 1, n, st);
    }, st);
    u64 total = 0;
    PK_CUDA(cudaMemcpyAsync(&total, out + n, sizeof(u64), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    return total;
  };
  u32* sel_tmp = sc.take<u32>(n);
  auto select = [&](const u32* src, const u8* flags, DevBuf<u32>& out) {
    u32* tmp = sel_tmp;
    cub_run([&](void* t, size_t& b) {
      return cub::DeviceSelect::Flagged(t, b, src, flags, tmp, count, n, st);
    }, st);
    i64 c = 0;
    PK_CUDA(cudaMemcpyAsync(&c, count, sizeof(i64), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    out.alloc(std::max<i64>(c, 1));
    if (c)
      PK_CUDA(cudaMemcpyAsync(out.p, tmp, c * sizeof(u32), cudaMemcpyDeviceToDevice, st));
    return c;
  };
  plan.entries = static_cast<i64>(exclusive_scan(ents, ent_off));
  plan.segments = exclusive_scan(hsegs, hseg_off);
  plan.empty = select(ids, is_empty, plan.empty_rows);
  DevBuf<u32> hubs32;
  const i64 nh = select(ids, is_hub, hubs32);
  plan.hub_count = static_cast<int>(nh);
  // entries: row key, store target, length -> offsets
  const i64 E = std::max<i64>(plan.entries, 1);
  plan.rowkey.alloc(E);
  plan.rl.alloc(E);
  plan.rpc.alloc(plan.entries + 1);
  {
    u64* elen = sc.take<u64>(E);
    fill_entries_kernel<<<blocks_for(n), 256, 0, st>>>(a.row_ptr, n, segment, ents, ent_off,
                                                       hsegs, hseg_off, plan.rowkey.p,
                                                       plan.rl.p, elen);
    PK_LAUNCH("spmm plan entries");
    PK_CUDA(cudaMemsetAsync(plan.rpc.p, 0, sizeof(u64), st));
    if (plan.entries)
      cub_run([&](void* t, size_t& b) {
        return cub::DeviceScan::InclusiveSum(t, b, elen, plan.rpc.p + 1, plan.entries, st);
      }, st);
  }
  PK_CUDA(cudaMemcpyAsync(&plan.list_nnz, plan.rpc.p + plan.entries, sizeof(u64),
                          cudaMemcpyDeviceToHost, st));
  PK_CUDA(cudaStreamSynchronize(st));
  plan.cv.alloc(std::max<u64>(plan.list_nnz, 1));
  const size_t words = plan.list_nnz / 32 + 2;
  plan.endbits.alloc(words);
  PK_CUDA(cudaMemsetAsync(plan.endbits.p, 0, words * sizeof(u32), st));
  if (plan.entries) {
    // hot columns: degree >= PK_HOT_FACTOR (default 2) x the mean
    check(a.cols < (i64{1} << 31), "spmm plan: more than 2^31 columns");
    const size_t ncols = static_cast<size_t>(std::max<i64>(a.cols, 1));
    u32* deg = sc.take<u32>(ncols);
    PK_CUDA(cudaMemsetAsync(deg, 0, ncols * sizeof(u32), st));
    if (a.nnz) {
      col_degree_kernel<<<blocks_for(static_cast<i64>(a.nnz)), 256, 0, st>>>(a.col_idx, a.nnz,
                                                                             deg);
      PK_LAUNCH("spmm plan column degrees");
    }
    static const double hot_factor = [] {
      const char* e = std::getenv("PK_HOT_FACTOR");
      return e ? std::atof(e) : 2.0;
    }();
    const double mean = static_cast<double>(a.nnz) / std::max<i64>(a.cols, 1);
    const u32 hot_deg = static_cast<u32>(std::max(1.0, std::ceil(hot_factor * mean)));
    compact_rows_kernel<<<blocks_for(n * 32), 256, 0, st>>>(a.row_ptr, a.col_idx, a.values, n,
                                                             ents, ent_off, plan.rpc.p,
                                                             deg, hot_deg, plan.cv.p,
                                                             plan.endbits.p);
    PK_LAUNCH("spmm plan compact");
  }
  if (nh && segment) {
    // FAST plan: hub rows ascending with their segment ranges
    plan.hub_asc = std::move(hubs32);
    u32* lo = sc.take<u32>(n);
    u32* cnt = sc.take<u32>(n);
    seg_meta_kernel<<<blocks_for(n), 256, 0, st>>>(hsegs, hseg_off, n, lo, cnt);
    PK_LAUNCH("spmm plan segments");
    select(lo, is_hub, plan.hub_seg0);
    select(cnt, is_hub, plan.hub_nseg);
  } else if (nh) {
    // exact plan: hub rows longest first (few: host sort)
    std::vector<u32> h(nh);
    std::vector<u64> lens(nh);
    DevBuf<u64> dlen(nh);
    hub_len_kernel<<<blocks_for(nh), 256, 0, st>>>(a.row_ptr, hubs32.p, nh, dlen.p);
    PK_LAUNCH("spmm plan hub lengths");
    PK_CUDA(cudaMemcpyAsync(h.data(), hubs32.p, nh * sizeof(u32), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaMemcpyAsync(lens.data(), dlen.p, nh * sizeof(u64), cudaMemcpyDeviceToHost, st));
    PK_CUDA(cudaStreamSynchronize(st));
    std::vector<std::pair<u64, i64>> by_len(nh);
    for (i64 i = 0; i < nh; ++i) by_len[i] = {lens[i], h[i]};
    std::stable_sort(by_len.begin(), by_len.end(),
                     [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<i64> ids64(nh);
    for (i64 i = 0; i < nh; ++i) ids64[i] = by_len[i].second;
    plan.hub_rows.alloc(nh);
    PK_CUDA(cudaMemcpyAsync(plan.hub_rows.p, ids64.data(), nh * sizeof(i64),
                            cudaMemcpyHostToDevice, st));
  }
  PK_CUDA(cudaStreamSynchronize(st));
}

void spmm_run(SpmmPlan& plan, const pk_csr& a, i64 r0, i64 r1, const float* x, i64 ldx, i64 d,
              float* y, i64 ldy, cudaStream_t st, const float* mask, i64 ldm,
              const RowMap* map, int max_vec, bool paired) {
  if (r1 <= r0 || d == 0) return;
  SpmmPlan::Range& rg = plan_range(plan, r0, r1, st);
  const RowMap rmap = map ? *map : RowMap{};
  check(rmap.g == 0 || plan.segment || rg.hubs == 0,
        "spmm: mapped output rows need a FAST plan (no hub CTAs)");
  if (rmap.g) y = rmap.base[0];  // alignment of the slots (all 16-B aligned)
  // 32-B slices for the list kernel; the exact plan's hub kernel stages
  // 16-B cp.async pieces, so a plan with hub CTAs stays at 16 B
  // the mask is read with y's vector width: it must share y's alignment
  int vec = pick_vec(x, ldx, y, ldy, d, plan.segment || rg.hubs == 0);
  while (vec > max_vec) vec /= 2;
  // experiment knob: the gather width of mid-width rows (64 < d < 256, e.g.
  // C2's D = 100), PK_SPMM_MID_VEC = 1 | 2 | 4
  static const int mid_vec = [] {
    const char* e = std::getenv("PK_SPMM_MID_VEC");
    return e ? std::atoi(e) : 0;
  }();
  if (mid_vec > 0 && d > 64 && d < 256)
    while (vec > mid_vec) vec /= 2;
  // the paired narrow form: FAST plans, no epilogue mask, at most 16 vectors
  // of up to 16 B per row
  int pair_vec = 0;
  if (paired && plan.segment && !mask) {
    const int pv = pick_vec(x, ldx, y, ldy, d, false);
    if (d / pv <= 16) pair_vec = pv;
  }
  if (pair_vec) vec = pair_vec;
  if (mask)
    while (vec > 1 && (ldm % vec || (reinterpret_cast<uintptr_t>(mask) % (vec * 4)))) vec /= 2;
  const int nvec = static_cast<int>(d / vec);
  // hub CTAs first, on a forked stream, so they hold their SMs while the
  // list kernel streams through the rest of the machine
  SideStream& side = side_stream();
  SpmmArgs h;
  if (!plan.segment && rg.hubs > 0) {
    h.rp = a.row_ptr, h.ci = a.col_idx, h.val = a.values;
    h.x = x, h.ldx = ldx, h.y = y, h.ldy = ldy, h.r0 = r0, h.nrows = r1 - r0, h.nvec = nvec;
    h.mask = mask, h.ldm = ldm;
    h.hub_rows = rg.hub_ids.p ? rg.hub_ids.p : plan.hub_rows.p;
    h.hub_count = rg.hubs;
    h.hub_slices = ceil_div(nvec, 32);
    h.hub_blocks = h.hub_count * h.hub_slices;
    PK_CUDA(cudaEventRecord(side.fork, st));
    PK_CUDA(cudaStreamWaitEvent(side.stream, side.fork, 0));
    if (vec == 4)
      launch_hub<4>(h, side.stream);
    else if (vec == 2)
      launch_hub<2>(h, side.stream);
    else
      launch_hub<1>(h, side.stream);
    PK_CUDA(cudaEventRecord(side.join, side.stream));
  }
  if (rg.e1 > rg.e0) {
    const i64 ne = rg.e1 - rg.e0;
    (rmap.g ? zero_rows_kernel<true> : zero_rows_kernel<false>)<<<blocks_for(ne * d), 256, 0, st>>>(
        plan.empty_rows.p + rg.e0, ne, r0, y, ldy, d, rmap);
    PK_LAUNCH("spmm zero rows");
  }
  if (rg.i1 > rg.i0) {
    ListArgs la;
    la.cv = plan.cv.p, la.rl = plan.rl.p, la.rpc = plan.rpc.p, la.endbits = plan.endbits.p;
    la.x = x, la.ldx = ldx, la.y = y, la.ldy = ldy, la.r0 = r0, la.nvec = nvec;
    la.xrows = static_cast<i64>(a.cols);
    la.mask = mask, la.ldm = ldm;
    la.map = rmap;
    // FAST plans chain with fused multiply-adds (PK_SPMM_FMA_FAST=0: off)
    static const bool fma_fast = [] {
      const char* e = std::getenv("PK_SPMM_FMA_FAST");
      return !(e && e[0] == '0');
    }();
    la.fma = fma_fast && plan.segment != 0;
    if (plan.segment && plan.segments) {
      la.ldp = (d + 7) / 8 * 8;  // 32-B aligned rows for the widest slices
      plan.partial.ensure(plan.segments * la.ldp);
      la.part = plan.partial.p;
    }
    if (pair_vec == 4)
      launch_pair<4>(la, rg.i0, rg.i1, plan.rpc.p, st);
    else if (pair_vec == 2)
      launch_pair<2>(la, rg.i0, rg.i1, plan.rpc.p, st);
    else if (pair_vec == 1)
      launch_pair<1>(la, rg.i0, rg.i1, plan.rpc.p, st);
    else if (vec == 8)
      dispatch_list<8>(la, rg.i0, rg.i1, plan.rpc.p, st);
    else if (vec == 4)
      dispatch_list<4>(la, rg.i0, rg.i1, plan.rpc.p, st);
    else if (vec == 2)
      dispatch_list<2>(la, rg.i0, rg.i1, plan.rpc.p, st);
    else
      dispatch_list<1>(la, rg.i0, rg.i1, plan.rpc.p, st);
  }
  if (plan.segment && rg.h1 > rg.h0) {
    const i64 nh = rg.h1 - rg.h0;
    (rmap.g ? combine_segments_kernel<true> : combine_segments_kernel<false>)<<<blocks_for(nh * d), 256, 0, st>>>(
        plan.hub_asc.p + rg.h0, plan.hub_seg0.p + rg.h0, plan.hub_nseg.p + rg.h0, nh, r0,
        plan.partial.p, (d + 7) / 8 * 8, y, ldy, d, mask, ldm, rmap);
    PK_LAUNCH("spmm combine segments");
  }
  if (!plan.segment && rg.hubs > 0) PK_CUDA(cudaStreamWaitEvent(st, side.join, 0));
}

}  // namespace pk

namespace pk {
unsigned spmm_watchdog() {
  unsigned v = 0;
  PK_CUDA(cudaMemcpyFromSymbol(&v, g_spmm_watchdog, sizeof(v)));
  return v;
}
}  // namespace pk
