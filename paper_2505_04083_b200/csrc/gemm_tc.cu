// Tensor-core dense transforms of the GCN layer on sm_100a: tcgen05.mma
// (kind::tf32) with fp32 accumulators in TMEM, 3xTF32 operand splitting.
//
// The reference multiplies in fp32 with a plain k-ascending loop
// (kernels.hpp:64-92). TF32 alone (10-bit mantissa) misses the 1e-4
// normwise budget (~3e-4 per GEMM), so every operand is
// split x = hi + lo (hi = tf32 part, lo = tf32 of the remainder), and
//     C = A_lo.B_hi + A_hi.B_lo + A_hi.B_hi
// accumulated in TMEM (error ~2^-21 relative per product, i.e. fp32-level).
//
// Feeding the big operands. The tensor core reads an fp32 operand by
// truncating it to tf32 (measured, scripts/tf32_round_probe.cu), so a raw
// fp32 tile already is the "hi" operand of hi = trunc(x), lo = x - hi. TMA
// (cp.async.bulk.tensor) streams raw tiles straight into swizzled shared
// memory — K-major with the 128-B swizzle, MN-major in 32-wide atoms with the
// 128-B/32-B-atom swizzle tf32 needs — and four converter warps derive each
// stage's lo tile in shared memory (lo = rna_tf32(x - trunc(x))), then fence
// and release the stage to the MMA. Converters never hold outstanding global
// loads, so their proxy fence is cheap; the first version staged operands
// through registers, where every fence waited for the prefetched loads and
// the pipeline collapsed to ~one stage in flight (kept for unaligned
// operands, PK_TC_TMA=0). The small weight operand of NN / NT is split once
// per call into per-stage hi/lo tile images that ride the same TMA barrier
// (cp.async.bulk). One elected thread issues the MMAs; epilogue warps drain
// the double-buffered TMEM accumulator with tcgen05.ld and store rows.
//
// Persistent CTAs walk a static tile schedule (m tile, n tile, k split). A
// k split > 1 writes fp32 partials that a deterministic fixed-order reduce
// combines (dW = H^T dQ reduces over all adjacency rows, engine.hpp:233-235).
//
// Operand forms (row-major storage; "T" = storage runs along M/N):
//   NN  Q  = H . W        A = H   (K-major tile)  B = W   (pre-split image)
//   NT  dH = dQ . W^T     A = dQ  (K-major tile)  B = W   (pre-split image)
//   TN  dW = H^T . dQ     A = H^T (MN-major tile) B = dQ  (MN-major tile)
#include <cuda.h>  // CUtensorMap (type only; the encoder comes from the runtime's entry point)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "elementwise.cuh"
#include "gemm.cuh"
#include "pk_common.cuh"

namespace pk {

namespace {

constexpr int kBM = 128;        // UMMA M (one CTA, cta_group::1)
constexpr int kBK = 32;         // k per stage: one 128-B swizzle row of fp32
constexpr int kLoaderWarps = 8;
constexpr int kMmaWarp = kLoaderWarps;          // warp 8
constexpr int kThreadsTc = 32 * (kLoaderWarps + 1 + 4);
constexpr int kLoaderThreads = 32 * kLoaderWarps;
#ifndef PK_CONV_WARPS
#define PK_CONV_WARPS 7
#endif
// TMA path: warps 8-PK_CONV_WARPS..7 derive the lo tiles (warp 0 lane 0 is
// the TMA producer)
constexpr int kConvWarps = PK_CONV_WARPS;
static_assert(kConvWarps >= 1 && kConvWarps <= kLoaderWarps - 1, "converter warps");
constexpr int kConvRingWarps = kLoaderWarps - 2;  // ring mode: warps 2..7
// k-stages accumulated in TMEM before the epilogue folds the partial into
// the output with round-to-nearest fp32 adds. The tensor core's fp32
// accumulation does not round to nearest, so its error grows with the chain
// length; 16 stages (512 k) keep the tall dW reduction (K = adjacency rows,
// up to millions) at fp32-level error (tests/test_gemm_tc_gpu.py).
constexpr int kSegStages = 16;
#ifndef PK_TC_RB
#define PK_TC_RB 2
#endif
#ifndef PK_EPI_V8
#define PK_EPI_V8 1
#endif
#ifndef PK_TC_RB_NARROW
#define PK_TC_RB_NARROW 8  // BN <= 64: the K = 256 weight images fit (resident mode)
#endif

__device__ unsigned g_gemm_watchdog = 0;

// PK_TC_PROF builds (scripts/tc_prof.sh): cycles each role spends in its
// barrier waits, lane 0 of each warp, summed over CTAs — 0 producer/empty,
// 1 converters/raw (x4 warps), 2 MMA/raw, 6 MMA/full, 3 MMA/tempty, 4
// epilogue/tfull (x4 warps); 5 kernel cycles (thread 0); 7 stages issued.
#ifdef PK_TC_PROF
__device__ unsigned long long g_tc_prof[8];
#define TC_PROF_WAIT(slot, call)          \
  do {                                    \
    const long long t0_ = clock64();      \
    call;                                 \
    prof_acc[slot] += clock64() - t0_;    \
  } while (0)
#else
#define TC_PROF_WAIT(slot, call) call
#endif

// ---------------------------------------------------------------- PTX glue

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(u64* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive(u64* bar) {
  asm volatile("{ .reg .b64 st; mbarrier.arrive.release.cta.shared::cta.b64 st, [%0]; }" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Bounded parity wait: a protocol error must surface as a flagged error, not
// as a GPU that spins until the job is killed.
__device__ __forceinline__ void mbar_wait(u64* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  for (unsigned spins = 0;; ++spins) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n"
        " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return;
    if (spins == (1u << 26)) {
      if (atomicAdd(&g_gemm_watchdog, 1u) == 0)
        printf("gemm_tc watchdog: block %d thread %d stuck on barrier parity %u\n", blockIdx.x,
               threadIdx.x, parity);
      return;
    }
  }
}

__device__ __forceinline__ void mbar_expect_tx(u64* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// 1-D bulk copy global -> shared (TMA engine, no tensor map), completing
// `bytes` of transaction count on `bar`.
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, unsigned bytes,
                                              u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// TMA tile loads (tensor maps built on the host per call)
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            u64* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<u64>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// shared -> global tensor store (bulk async group); the box lands clipped
// to the tensor's bounds
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0,
                                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
          reinterpret_cast<u64>(map)),
      "r"(c0), "r"(c1), "r"(smem_u32(src))
      : "memory");
}

__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
// bulk copy into the same smem offset of every CTA in `mask`, completing
// `bytes` on each one's barrier at `bar`'s offset
__device__ __forceinline__ void bulk_copy_g2s_mc(void* dst, const void* src, unsigned bytes,
                                                 u64* bar, unsigned short mask) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void tc_commit_mc(u64* bar, unsigned short mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

// arrive on the barrier at the same smem offset in cluster CTA `rank`
__device__ __forceinline__ void mbar_arrive_cluster(u64* bar, unsigned rank) {
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
// CTA-pair commit: arrives on `bar` in both CTAs of the pair
__device__ __forceinline__ void tc_commit_pair(u64* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(static_cast<unsigned short>(3))
      : "memory");
}
__device__ __forceinline__ void tc_mma_tf32_pair(unsigned d_tmem, u64 adesc, u64 bdesc,
                                                 unsigned idesc, unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tc_commit(u64* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_mma_tf32(unsigned d_tmem, u64 adesc, u64 bdesc, unsigned idesc,
                                            unsigned accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// 32 lanes x 32 bit, 8 consecutive columns per thread
__device__ __forceinline__ void tmem_ld8(unsigned taddr, float (&v)[8]) {
  unsigned r[8];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 32 lanes x 32 bit, 16 / 32 consecutive columns per thread, one wait
__device__ __forceinline__ void tmem_ld16(unsigned taddr, float (&v)[16]) {
  unsigned r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld32(unsigned taddr, float (&v)[32]) {
  unsigned r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Shared-memory matrix descriptor (tcgen05 "version 1"), 128-B swizzle.
__device__ __forceinline__ u64 smem_desc(unsigned addr, unsigned lbo, unsigned sbo) {
  u64 d = 0;
  d |= static_cast<u64>((addr >> 4) & 0x3FFF);
  d |= static_cast<u64>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<u64>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  d |= 2ull << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor: fp32 accumulate, tf32 A and B, M = 128; bits 15/16
// mark an MN-major operand (staged in the 32-B-atom swizzle, see below).
__host__ __device__ constexpr unsigned instr_desc(int n, bool a_mn, bool b_mn, int m = kBM) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<unsigned>(a_mn) << 15) |
         (static_cast<unsigned>(b_mn) << 16) | (static_cast<unsigned>(n >> 3) << 17) |
         (static_cast<unsigned>(m >> 4) << 24);
}

// ------------------------------------------------------------ tile layout
//
// K-major SW128: row r (an M or N index) holds 32 fp32 of k in one 128-B
// line; 8-row atoms of 1024 B; 16-B chunk c (= k/4) of row r lives at
// r*128 + ((c ^ r%8) * 16). UMMA k-step t (8 k) starts 32*t bytes into the
// tile; SBO (next 8-row group) = 1024, LBO unused for swizzled K-major.

__device__ __forceinline__ unsigned kmajor_offset(int row, int kc) {
  return static_cast<unsigned>(row * 128 + ((kc ^ (row & 7)) << 4));
}
__device__ __forceinline__ u64 kmajor_desc(unsigned base, int kstep) {
  return smem_desc(base + 32u * kstep, 16u, 1024u);
}

// One operand's view for the loaders; storage is row-major `p[r * ld + c]`.
//  T = false ("K-contiguous"): r = m/n index (extent `mn`), c = k.
//  T = true  ("MN-contiguous"): r = k, c = m/n index (extent `mn`).
struct OperandSrc {
  const float* p;
  i64 ld;
  i64 mn;      // extent of the M/N index
  bool vec;    // base and ld allow 16-B loads
};

__device__ __forceinline__ float4 split_hi(float4 v) {
  return make_float4(tf32_rna(v.x), tf32_rna(v.y), tf32_rna(v.z), tf32_rna(v.w));
}
__device__ __forceinline__ float4 split_lo(float4 v, float4 h) {
  return make_float4(tf32_rna(v.x - h.x), tf32_rna(v.y - h.y), tf32_rna(v.z - h.z),
                     tf32_rna(v.w - h.w));
}

// 4 consecutive elements of storage row r starting at column c, masked to
// [0, c_end) (zero fill); 16-B load when the whole quad is in range.
__device__ __forceinline__ float4 load_quad(const OperandSrc& s, i64 r, i64 c, i64 c_end) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  const float* p = s.p + r * s.ld + c;
  if (s.vec && c + 3 < c_end) return __ldg(reinterpret_cast<const float4*>(p));
  if (c < c_end) v.x = __ldg(p);
  if (c + 1 < c_end) v.y = __ldg(p + 1);
  if (c + 2 < c_end) v.z = __ldg(p + 2);
  if (c + 3 < c_end) v.w = __ldg(p + 3);
  return v;
}

// Loader work for one operand tile of ROWS (M/N) x 32 (k) per stage.
//
// K-contiguous source: item = one 16-B chunk (row, k-chunk); 8 consecutive
// threads read one row's 128 B; stored as-is (one 16-B st.shared each).
//
// MN-contiguous source: item = a 4 (k) x 4 (mn) block read as 4 float4 rows
// and transposed in registers into 4 k-quads. Lane l of a warp takes mn
// block l%8 and k-chunk l/8 (+4 for the second half), so each 16-B store
// row-group hits 8 distinct swizzle chunks: conflict-free, and every k row
// is still read as 128 contiguous bytes by 8 lanes.
// MN-major "128-B swizzle, 32-B atom" tile (layout type 1, the tf32 MN-major
// form; the plain 128-B swizzle reads back zeros for tf32 MN-major operands,
// measured with scripts/tc_probe.cu): atoms of 4 k-rows x 128 B (32 M/N
// values); the 32-B chunk (mn%32)/8 of row k is XOR-ed with k%4; MN atoms
// are 512 B apart (LBO), 4-row k groups are SBO = (ROWS/32)*512 apart. A
// UMMA k-step (8 k) spans two k groups.
template <int ROWS>
__device__ __forceinline__ unsigned mnmajor_offset(int mn, int k) {
  constexpr unsigned kSbo = (ROWS / 32) * 512;
  const int a = mn >> 5, c = (mn & 31) >> 3, half = (mn >> 2) & 1, r = k & 3, g = k >> 2;
  return static_cast<unsigned>(g * kSbo + a * 512 + r * 128 + ((c ^ r) << 5) + half * 16);
}
template <int ROWS>
__device__ __forceinline__ u64 mnmajor_desc(unsigned base, int kstep) {
  constexpr unsigned kSbo = (ROWS / 32) * 512;
  u64 d = smem_desc(base + 2u * kSbo * kstep, 512u, kSbo);
  d &= ~(7ull << 61);
  return d | (1ull << 61);  // SWIZZLE_128B_BASE32B
}

// MN-major tile as TMA writes it: one {32 mn x 32 k} box per 32-wide mn atom,
// 4 KB each (k row r at r*128, 32-B chunks swizzled in 4-row groups), so
// mn atoms are 4096 B apart (LBO) and 4-row k groups 512 B (SBO).
__device__ __forceinline__ u64 mnmajor_tma_desc(unsigned base, int kstep) {
  u64 d = smem_desc(base + 1024u * kstep, 4096u, 512u);
  d &= ~(7ull << 61);
  return d | (1ull << 61);  // SWIZZLE_128B_BASE32B
}

// lo = x - trunc_tf32(x), rounded to tf32: the tensor core reads an fp32
// operand by truncating it to tf32 (scripts/tf32_round_probe.cu), so the raw
// tile itself serves as "hi" and only lo is computed.
__device__ __forceinline__ float4 lo_of_raw(float4 v) {
  auto one = [](float x) {
    const float t = __uint_as_float(__float_as_uint(x) & 0xffffe000u);
    return tf32_rna(x - t);
  };
  return make_float4(one(v.x), one(v.y), one(v.z), one(v.w));
}

// Loader work for one operand tile of ROWS (M/N) x 32 (k) per stage. Each
// item is one 16-B chunk of the row-major source, stored (split into hi/lo)
// without any transposition:
//  T = false, K-contiguous source: chunk (row, k quad) -> K-major tile; 8
//    consecutive threads read one row's 128 B.
//  T = true, MN-contiguous source: chunk (k row, 4 mn) -> MN-major tile;
//    consecutive threads read one k row's consecutive 16-B pieces.
template <bool T, int ROWS>
struct TileLoader {
  static constexpr int kItems = 8 * ROWS;
  static constexpr int kPer = (kItems + kLoaderThreads - 1) / kLoaderThreads;
  static constexpr int kRegs = kPer;

  static __device__ __forceinline__ void item_coords(int q, int& mn, int& k) {
    if (!T) {
      mn = q >> 3;
      k = (q & 7) << 2;
    } else {
      constexpr int per_k = ROWS / 4;
      k = q / per_k;
      mn = (q % per_k) << 2;
    }
  }

  static __device__ __forceinline__ void load(const OperandSrc& s, i64 mn0, i64 k0, i64 k_end,
                                              int tid, float4 (&r)[kRegs]) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int q = tid + i * kLoaderThreads;
      int mn, k;
      item_coords(q, mn, k);
      const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
      if (!T) {
        const i64 gr = mn0 + mn;
        r[i] = (q < kItems && gr < s.mn) ? load_quad(s, gr, k0 + k, k_end) : z;
      } else {
        const i64 gk = k0 + k;
        r[i] = (q < kItems && gk < k_end) ? load_quad(s, gk, mn0 + mn, s.mn) : z;
      }
    }
  }

  static __device__ __forceinline__ void store(unsigned char* hi, unsigned char* lo, int tid,
                                               const float4 (&r)[kRegs]) {
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int q = tid + i * kLoaderThreads;
      if (q >= kItems) continue;
      int mn, k;
      item_coords(q, mn, k);
      const unsigned off = T ? mnmajor_offset<ROWS>(mn, k) : kmajor_offset(mn, k >> 2);
      const float4 h = split_hi(r[i]);
      *reinterpret_cast<float4*>(hi + off) = h;
      *reinterpret_cast<float4*>(lo + off) = split_lo(r[i], h);
    }
  }

  static __device__ __forceinline__ u64 desc(unsigned base, int kstep) {
    if constexpr (T) return mnmajor_desc<ROWS>(base, kstep);
    return kmajor_desc(base, kstep);
  }
};

struct TcParams {
  OperandSrc a, b;
  // NN / NT: B (the weight) pre-split into per-k-stage [hi | lo] K-major
  // swizzled tile images, bulk-copied straight into shared memory
  const unsigned char* b_image;
  i64 b_stages;     // k stages per n tile in b_image
  i64 m, n, k;
  i64 k_chunk;      // k per split (multiple of kBK)
  int m_tiles, n_tiles, splits;
  float* c;         // output (splits == 1) or partials [split][m][ldc]
  i64 ldc;
  i64 split_stride; // elements between split partials
  int resident_ok = 0;  // weight-resident ring allowed (PK_TC_RESIDENT=1)
  const float* mask = nullptr;  // relu_backward epilogue: keep where mask > 0
  i64 ldm = 0;
  int tma_store = 0;  // ring kernel: the epilogue stores 32 x 32 boxes by TMA
  int relu;         // 1: the final value is stored as relu(v) (v > 0 ? v : 0)
  RowMap map;       // output row placement (g == 0: c + row * ldc)
};

template <bool A_T, bool B_T, int BN, int STAGES, bool B_PRE>
struct TcConfig {
  // stored N extent: a multiple of 16 (UMMA N) — and of 32 when the loader
  // transposes, whose items cover 32 rows per lane group
  static constexpr int kRowsB = (B_T && !B_PRE) ? ((BN + 31) / 32) * 32 : BN;
  static constexpr int kTileA = kBM * kBK * 4;  // bytes, one of hi/lo
  static constexpr int kTileB = kRowsB * kBK * 4;
  static constexpr int kStage = 2 * kTileA + 2 * kTileB;
  using LoadA = TileLoader<A_T, kBM>;
  using LoadB = TileLoader<B_T, kRowsB>;
  static constexpr int kTmemCols = BN <= 32 ? 64 : (BN <= 64 ? 128 : (BN <= 128 ? 256 : 512));
  static constexpr int kAccStride = kTmemCols / 2;  // two accumulator buffers
  static constexpr size_t kSmem = static_cast<size_t>(STAGES) * kStage + 1024;
  // Ring layout (TMA + weight image, single-CTA): the raw A tiles, their lo
  // tiles and the weight images live in three rings of their own depth, so
  // the DRAM-fed raw ring can run far ahead of the L2-fed weight ring.
  // weight images (hi | lo): L2-fed, so a narrow tile's ring needs more
  // slots in flight to cover the L2 latency (PK_TC_RB / PK_TC_RB_NARROW)
  static constexpr int kRB = BN <= 64 ? PK_TC_RB_NARROW : PK_TC_RB;
  static constexpr int kRL = 2;                 // converted lo tiles
  static constexpr int kRingBudget = 224 * 1024;
  // epilogue staging for the TMA stores: one 32 x 32 fp32 box per epilogue warp
  static constexpr int kStgBytes = 4 * 4096;
  static constexpr int kRA =
      std::min(8, (kRingBudget - kStgBytes - kRB * 2 * kTileB - kRL * kTileA) / kTileA);
  static constexpr size_t kSmemRing = static_cast<size_t>(kRA + kRL) * kTileA +
                                      static_cast<size_t>(kRB) * 2 * kTileB + kStgBytes + 1024;
  // CTA-pair rings: each CTA keeps half of every weight image (its N/2 rows)
  static constexpr int kRAPair = std::min(8, (kRingBudget - kRB * kTileB - kRL * kTileA) / kTileA);
  static constexpr size_t kSmemPair =
      static_cast<size_t>(kRAPair + kRL) * kTileA + static_cast<size_t>(kRB) * kTileB + 1024;
};

// TMA: the big operands arrive by TMA as raw fp32 tiles (the tensor core's
// own truncation makes them the "hi" operand); four converter warps derive
// each stage's lo tile from shared memory. Otherwise they are register-staged
// by eight loader warps (unaligned operands, or PK_TC_TMA=0).
// CS > 1 (TMA + pre-split B, one n tile, no k split): clusters of CS CTAs
// on consecutive m tiles share each stage's weight image — every CTA bulk-
// copies 1/CS of it multicast into all CTAs of the cluster, and a stage is
// refilled only when every CTA's MMAs are done with it (commit multicast to
// all `empty` barriers). The weight's L2 -> SM traffic drops CS-fold. A CTA
// whose own tile runs past the end follows its cluster through a phantom
// tile (A zero-filled by TMA, nothing stored).
//
// PAIR (TMA + weight image, one n tile, no k split; launched as 2-CTA
// clusters): the ring kernel as a CTA pair — tcgen05.mma.cta_group::2 with
// M = 256, each CTA supplying its 128 A rows and half of the weight image's
// N rows, so each SM's shared memory feeds a third less operand traffic per
// MMA. The leader (rank 0) issues the MMAs; both CTAs load, convert and
// drain their own TMEM half; the peer's converters and epilogue warps
// arrive on the leader's barriers across the cluster, and the leader's
// commits release both CTAs' stages.
template <bool A_T, bool B_T, int BN, int STAGES, bool B_PRE, bool TMA, int CS, bool PAIR = false>
__global__ void __launch_bounds__(kThreadsTc, 1)
    gemm_tc_kernel(TcParams p, const __grid_constant__ CUtensorMap tma_a,
                   const __grid_constant__ CUtensorMap tma_b,
                   const __grid_constant__ CUtensorMap tma_c) {
  using Cfg = TcConfig<A_T, B_T, BN, STAGES, B_PRE>;
  static_assert(!TMA || B_PRE || B_T, "TMA path: a streamed B must be MN-major");
  static_assert(CS == 1 || (TMA && B_PRE), "clusters need the TMA + weight-image path");
  static_assert(!PAIR || (TMA && B_PRE && CS == 2 && !A_T && BN % 32 == 0),
                "CTA pairs: TMA K-major A, weight image, 2-CTA clusters, BN % 32 == 0");
  constexpr unsigned short kMask = static_cast<unsigned short>((1u << CS) - 1u);
  const int crank = CS > 1 ? static_cast<int>(cluster_rank()) : 0;
  constexpr bool kRing = TMA && B_PRE && (CS == 1 || PAIR);
  constexpr int kRA = PAIR ? Cfg::kRAPair : Cfg::kRA, kRL = Cfg::kRL, kRB = Cfg::kRB;
  constexpr int kBSlot = PAIR ? Cfg::kTileB : 2 * Cfg::kTileB;  // bytes of one weight slot
  const bool leader = !PAIR || crank == 0;
  // pair mode walks pair tiles: one index per cluster, CTA rank picks the half
  const int tile_first = PAIR ? static_cast<int>(blockIdx.x) / 2 : static_cast<int>(blockIdx.x);
  const int tile_step = PAIR ? static_cast<int>(gridDim.x) / 2 : static_cast<int>(gridDim.x);
  static_assert(!kRing || kRA >= 2, "ring layout: at least two raw stages");
#ifdef PK_TC_PROF
  const long long t_kernel = clock64();
  long long prof_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  extern __shared__ unsigned char smem_raw[];
  // 1024-B alignment for the swizzle atoms
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  __shared__ u64 full[STAGES], empty[STAGES], raw[STAGES], tfull[2], tempty[2];
  // ring mode: raw A full/empty, lo full/empty, weight image full/empty
  __shared__ u64 ra_full[kRing ? kRA : 1], ra_empty[kRing ? kRA : 1];
  __shared__ u64 rl_full[kRing ? kRL : 1], rl_empty[kRing ? kRL : 1];
  __shared__ u64 rb_full[kRing ? kRB : 1], rb_empty[kRing ? kRB : 1];
  __shared__ unsigned tmem_base;

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], TMA ? kConvWarps : kLoaderWarps);
      mbar_init(&empty[s], CS);  // every cluster CTA's MMAs release the stage
      mbar_init(&raw[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 8 : 4);  // pair: both CTAs' epilogue warps
    }
    if constexpr (kRing) {
      for (int i = 0; i < kRA; ++i) mbar_init(&ra_full[i], 1), mbar_init(&ra_empty[i], 1);
      for (int i = 0; i < kRL; ++i)
        mbar_init(&rl_full[i], (PAIR ? 2 : 1) * kConvRingWarps), mbar_init(&rl_empty[i], 1);
      for (int i = 0; i < kRB; ++i) mbar_init(&rb_full[i], 1), mbar_init(&rb_empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kMmaWarp) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base)),
                   "n"(Cfg::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(&tmem_base)),
                   "n"(Cfg::kTmemCols));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CS > 1) cluster_sync();  // peers' barriers initialised before any multicast
  tc_fence_after();
  const unsigned tmem = tmem_base;

  const int total_tiles = PAIR ? (p.m_tiles + 1) / 2 : p.m_tiles * p.n_tiles * p.splits;
  // Weight-resident ring: one n tile, no k split, and every k-stage's
  // weight image fits the ring — each CTA loads the images once and keeps
  // them (slot = k-stage) instead of re-streaming them from L2 for every m
  // tile (C2: T = H W3 and dH3 = dT W3^T, where the images were as many
  // bytes per tile as the A rows).
  const int nk_all = static_cast<int>((p.k + kBK - 1) / kBK);
  const bool resident =
      kRing && !PAIR && p.resident_ok && p.n_tiles == 1 && p.splits == 1 && nk_all > 0 &&
      nk_all <= kRB;
  // a tile index is live while its cluster leader's is (phantoms beyond)
  auto live = [&](int t) { return PAIR ? t < total_tiles : t - crank < total_tiles; };
  // n tile fastest: the CTAs that share an A row block (several n tiles)
  // run side by side, so A comes from DRAM once and from L2 after
  auto tile_coords = [&](int t, int& mt, int& nt, int& sp) {
    if (PAIR) {  // the pair's 256 rows: this CTA's 128 (zero-filled past m)
      mt = 2 * t + crank, nt = 0, sp = 0;
      return;
    }
    if (CS > 1 && t >= total_tiles) {  // phantom: past the last m tile
      mt = p.m_tiles, nt = 0, sp = 0;
      return;
    }
    nt = t % p.n_tiles;
    mt = (t / p.n_tiles) % p.m_tiles;
    sp = t / (p.m_tiles * p.n_tiles);
  };
  auto k_range = [&](int sp, i64& kb, i64& ke) {
    kb = static_cast<i64>(sp) * p.k_chunk;
    ke = min(p.k, kb + p.k_chunk);
  };

  // k-stage walk shared by the loaders / producer / converters
  struct Pos {
    int t, kk, nk, nt;
    i64 kb, ke, m0, n0;
  };
  auto start = [&](Pos& q, int t) {
    q.t = t;
    q.kk = 0;
    q.nk = 0;
    while (live(q.t)) {
      int mt, nt, sp;
      tile_coords(q.t, mt, nt, sp);
      k_range(sp, q.kb, q.ke);
      q.m0 = static_cast<i64>(mt) * kBM;
      q.nt = nt;
      q.n0 = static_cast<i64>(nt) * BN;
      q.nk = static_cast<int>((q.ke - q.kb + kBK - 1) / kBK);
      if (q.nk > 0) return;
      q.t += tile_step;  // empty k range: the MMA warp signals it without stages
    }
  };
  auto advance = [&](Pos& q) {
    if (++q.kk == q.nk) start(q, q.t + tile_step);
  };
  auto valid = [&](const Pos& q) { return live(q.t); };

  // smem of the rings: [raw A x kRA][lo A x kRL][weight image (hi|lo) x kRB]
  auto ra_slot = [&](int i) { return smem + static_cast<size_t>(i) * Cfg::kTileA; };
  auto rl_slot = [&](int i) { return smem + static_cast<size_t>(kRA + i) * Cfg::kTileA; };
  auto rb_slot = [&](int i) {
    return smem + static_cast<size_t>(kRA + kRL) * Cfg::kTileA + static_cast<size_t>(i) * kBSlot;
  };

  if (kRing && warp < kLoaderWarps) {
    if constexpr (kRing) {
      if (warp == 0 && lane == 0) {
        // ------------------------------------------- raw A producer (DRAM)
        Pos q;
        start(q, tile_first);
        for (u64 s = 0; valid(q); ++s) {
          const int i = static_cast<int>(s % kRA);
          const unsigned ph = static_cast<unsigned>((s / kRA) & 1);
          TC_PROF_WAIT(0, mbar_wait(&ra_empty[i], ph ^ 1u));
          const i64 k0 = q.kb + static_cast<i64>(q.kk) * kBK;
          mbar_expect_tx(&ra_full[i], Cfg::kTileA);
          tma_load_2d(ra_slot(i), &tma_a, static_cast<int>(k0), static_cast<int>(q.m0),
                      &ra_full[i]);
          mbar_arrive(&ra_full[i]);
          advance(q);
        }
      } else if (warp == 1 && lane == 0) {
        // ------------------------------------- weight image producer (L2)
        Pos q;
        start(q, tile_first);
        if (resident) {
          // every stage's image once, into slot kk, for all of this CTA's tiles
          if (valid(q))
            for (int i = 0; i < nk_all; ++i) {
              mbar_expect_tx(&rb_full[i], 2u * Cfg::kTileB);
              bulk_copy_g2s(rb_slot(i), p.b_image + static_cast<i64>(i) * 2 * Cfg::kTileB,
                            2u * Cfg::kTileB, &rb_full[i]);
              mbar_arrive(&rb_full[i]);
            }
        } else
        for (u64 s = 0; valid(q); ++s) {
          const int i = static_cast<int>(s % kRB);
          const unsigned ph = static_cast<unsigned>((s / kRB) & 1);
          mbar_wait(&rb_empty[i], ph ^ 1u);
          const i64 k0 = q.kb + static_cast<i64>(q.kk) * kBK;
          const i64 g = q.nt * p.b_stages + k0 / kBK;
          if constexpr (PAIR) {
            // this CTA's N/2 rows of the hi and the lo image (K-major rows
            // are contiguous 128-B lines, so each half is one block)
            constexpr unsigned kHalf = Cfg::kTileB / 2;
            const unsigned char* img = p.b_image + g * 2 * Cfg::kTileB + crank * kHalf;
            mbar_expect_tx(&rb_full[i], 2u * kHalf);
            bulk_copy_g2s(rb_slot(i), img, kHalf, &rb_full[i]);
            bulk_copy_g2s(rb_slot(i) + kHalf, img + Cfg::kTileB, kHalf, &rb_full[i]);
          } else {
            mbar_expect_tx(&rb_full[i], 2u * Cfg::kTileB);
            bulk_copy_g2s(rb_slot(i), p.b_image + g * 2 * Cfg::kTileB, 2u * Cfg::kTileB,
                          &rb_full[i]);
          }
          mbar_arrive(&rb_full[i]);
          advance(q);
        }
      } else if (warp >= 2) {
        // ------------------------------------------------------ converters
        const int ct = threadIdx.x - 64;
        constexpr int kStep = 32 * kConvRingWarps;
        Pos q;
        start(q, tile_first);
        for (u64 s = 0; valid(q); ++s) {
          const int ia = static_cast<int>(s % kRA), il = static_cast<int>(s % kRL);
          TC_PROF_WAIT(1, mbar_wait(&ra_full[ia], static_cast<unsigned>((s / kRA) & 1)));
          mbar_wait(&rl_empty[il], static_cast<unsigned>((s / kRL) & 1) ^ 1u);
          const unsigned s0 = smem_u32(ra_slot(ia)), d0 = smem_u32(rl_slot(il));
          for (int i0 = ct; i0 < Cfg::kTileA / 16; i0 += 4 * kStep) {
            float4 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int i = i0 + j * kStep;
              if (i < Cfg::kTileA / 16)
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v[j].x), "=f"(v[j].y), "=f"(v[j].z), "=f"(v[j].w)
                             : "r"(s0 + 16u * i));
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int i = i0 + j * kStep;
              if (i < Cfg::kTileA / 16) {
                const float4 l = lo_of_raw(v[j]);
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(d0 + 16u * i),
                             "f"(l.x), "f"(l.y), "f"(l.z), "f"(l.w)
                             : "memory");
              }
            }
          }
          fence_async_smem();
          if constexpr (PAIR) {
            // the leader's MMA reads this CTA's weight half and lo tile too:
            // signal it once both are in place
            mbar_wait(&rb_full[static_cast<int>(s % kRB)],
                      static_cast<unsigned>((s / kRB) & 1));
          }
          __syncwarp();
          if (lane == 0) {
            if (PAIR && crank != 0)
              mbar_arrive_cluster(&rl_full[il], 0);
            else
              mbar_arrive(&rl_full[il]);
          }
          advance(q);
        }
      }
    }
  } else if (TMA && warp < kLoaderWarps) {
    if constexpr (TMA) {
      if (warp == 0 && lane == 0) {
        // ---------------------------------------------------- TMA producer
        int stage = 0;
        unsigned phase = 0;
        Pos q;
        start(q, tile_first);
        constexpr unsigned kBytes =
            Cfg::kTileA + (B_PRE ? 2u * Cfg::kTileB : static_cast<unsigned>(Cfg::kTileB));
        while (valid(q)) {
          TC_PROF_WAIT(0, mbar_wait(&empty[stage], phase ^ 1u));
          unsigned char* st = smem + static_cast<size_t>(stage) * Cfg::kStage;
          const i64 k0 = q.kb + static_cast<i64>(q.kk) * kBK;
          mbar_expect_tx(&raw[stage], kBytes);
          if constexpr (!A_T) {
            tma_load_2d(st, &tma_a, static_cast<int>(k0), static_cast<int>(q.m0), &raw[stage]);
          } else {
#pragma unroll
            for (int a = 0; a < kBM / 32; ++a)
              tma_load_2d(st + a * 4096, &tma_a, static_cast<int>(q.m0 + a * 32),
                          static_cast<int>(k0), &raw[stage]);
          }
          if constexpr (B_PRE) {
            const i64 g = q.nt * p.b_stages + k0 / kBK;
            if constexpr (CS > 1) {
              constexpr unsigned kPiece = 2u * Cfg::kTileB / CS;
              bulk_copy_g2s_mc(st + 2 * Cfg::kTileA + crank * kPiece,
                               p.b_image + g * 2 * Cfg::kTileB + crank * kPiece, kPiece,
                               &raw[stage], kMask);
            } else {
              bulk_copy_g2s(st + 2 * Cfg::kTileA, p.b_image + g * 2 * Cfg::kTileB,
                            2u * Cfg::kTileB, &raw[stage]);
            }
          } else {
#pragma unroll
            for (int a = 0; a < Cfg::kRowsB / 32; ++a)
              tma_load_2d(st + 2 * Cfg::kTileA + a * 4096, &tma_b,
                          static_cast<int>(q.n0 + a * 32), static_cast<int>(k0), &raw[stage]);
          }
          mbar_arrive(&raw[stage]);
          advance(q);
          if (++stage == STAGES) stage = 0, phase ^= 1u;
        }
      } else if (warp >= kLoaderWarps - kConvWarps) {
        // ------------------------------------------------------ converters
        const int ct = threadIdx.x - 32 * (kLoaderWarps - kConvWarps);
        int stage = 0;
        unsigned phase = 0;
        Pos q;
        start(q, tile_first);
        // shared-window addresses: explicit ld/st.shared (generic pointers
        // compiled to generic LD/ST, measured as the converters' stall)
        // Batches of 4 chunks per thread: four loads in flight, then the
        // math and four stores.
        auto convert = [&](unsigned char* src, unsigned char* dst, int bytes) {
          const unsigned s0 = smem_u32(src), d0 = smem_u32(dst);
          constexpr int kStep = 32 * kConvWarps;
          for (int i0 = ct; i0 < bytes / 16; i0 += 4 * kStep) {
            float4 v[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int i = i0 + j * kStep;
              if (i < bytes / 16)
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(v[j].x), "=f"(v[j].y), "=f"(v[j].z), "=f"(v[j].w)
                             : "r"(s0 + 16u * i));
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int i = i0 + j * kStep;
              if (i < bytes / 16) {
                const float4 l = lo_of_raw(v[j]);
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(d0 + 16u * i),
                             "f"(l.x), "f"(l.y), "f"(l.z), "f"(l.w)
                             : "memory");
              }
            }
          }
        };
        while (valid(q)) {
          TC_PROF_WAIT(1, mbar_wait(&raw[stage], phase));
          unsigned char* st = smem + static_cast<size_t>(stage) * Cfg::kStage;
          convert(st, st + Cfg::kTileA, Cfg::kTileA);
          if constexpr (!B_PRE)
            convert(st + 2 * Cfg::kTileA, st + 2 * Cfg::kTileA + Cfg::kTileB, Cfg::kTileB);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(&full[stage]);
          advance(q);
          if (++stage == STAGES) stage = 0, phase ^= 1u;
        }
      }
    }
  } else if (warp < kLoaderWarps) {
    // ------------------------------------------------------------ loaders
    // A (and B when it streams) go through registers two k-stages ahead,
    // across tile boundaries, in two alternating register sets; a pre-split
    // B arrives by one bulk copy per stage.
    const int lt = threadIdx.x;
    int stage = 0;
    unsigned phase = 0;
    constexpr int kRB = B_PRE ? 1 : Cfg::LoadB::kRegs;
    struct Regs {
      float4 a[Cfg::LoadA::kRegs];
      float4 b[kRB];
    };
    // prefetch depth: three register sets when only A streams (NN / NT), two
    // when A and B both do (TN)
    constexpr int kDepth = B_PRE ? 3 : 2;
    Regs rs[kDepth];
    auto load = [&](Regs& r, const Pos& q) {
      if (!valid(q)) return;
      const i64 k0 = q.kb + static_cast<i64>(q.kk) * kBK;
      Cfg::LoadA::load(p.a, q.m0, k0, q.ke, lt, r.a);
      if constexpr (!B_PRE) Cfg::LoadB::load(p.b, q.n0, k0, q.ke, lt, r.b);
    };
    Pos cur, pre;
    start(cur, tile_first);
    pre = cur;
#pragma unroll
    for (int d = 0; d < kDepth; ++d) {
      load(rs[d], pre);
      if (valid(pre)) advance(pre);
    }
    auto step = [&](Regs& r) {
      mbar_wait(&empty[stage], phase ^ 1u);
      unsigned char* st = smem + static_cast<size_t>(stage) * Cfg::kStage;
      if constexpr (B_PRE) {
        if (threadIdx.x == 0) {
          const i64 g = cur.nt * p.b_stages + (cur.kb + static_cast<i64>(cur.kk) * kBK) / kBK;
          mbar_expect_tx(&full[stage], 2u * Cfg::kTileB);
          bulk_copy_g2s(st + 2 * Cfg::kTileA, p.b_image + g * 2 * Cfg::kTileB,
                        2u * Cfg::kTileB, &full[stage]);
        }
      }
      Cfg::LoadA::store(st, st + Cfg::kTileA, lt, r.a);
      if constexpr (!B_PRE)
        Cfg::LoadB::store(st + 2 * Cfg::kTileA, st + 2 * Cfg::kTileA + Cfg::kTileB, lt, r.b);
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[stage]);
      if (++stage == STAGES) stage = 0, phase ^= 1u;
      advance(cur);
      load(r, pre);  // kDepth stages ahead
      if (valid(pre)) advance(pre);
    };
    while (valid(cur)) {
#pragma unroll
      for (int d = 0; d < kDepth; ++d) {
        if (!valid(cur)) break;
        step(rs[d]);
      }
    }
  } else if (warp == kMmaWarp) {
    // ------------------------------------------------------------ MMA issuer
    if (!leader) goto mma_done;  // the pair's MMAs are the leader's
    {
    constexpr unsigned idesc = instr_desc(BN, A_T, B_T && !B_PRE, PAIR ? 2 * kBM : kBM);
    int stage = 0;
    unsigned phase = 0;
    u64 ring_s = 0;  // ring mode: k-stages consumed so far
    int acc = 0;
    unsigned acc_phase = 0;
    for (int t = tile_first; live(t); t += tile_step) {
      int mt, nt, sp;
      tile_coords(t, mt, nt, sp);
      i64 kb, ke;
      k_range(sp, kb, ke);
      const int nk = static_cast<int>((ke - kb + kBK - 1) / kBK);
      const int nseg = nk == 0 ? 1 : (nk + kSegStages - 1) / kSegStages;
      for (int sg = 0; sg < nseg; ++sg) {
        TC_PROF_WAIT(3, mbar_wait(&tempty[acc], acc_phase ^ 1u));
        tc_fence_after();
        const unsigned d = tmem + static_cast<unsigned>(acc * Cfg::kAccStride);
        const int k_lo = sg * kSegStages, k_hi = min(nk, k_lo + kSegStages);
        for (int kk = k_lo; kk < k_hi; ++kk) {
          if constexpr (kRing) {
            const int ia = static_cast<int>(ring_s % kRA), il = static_cast<int>(ring_s % kRL),
                      ib = resident ? kk : static_cast<int>(ring_s % kRB);
            TC_PROF_WAIT(2, mbar_wait(&ra_full[ia], static_cast<unsigned>((ring_s / kRA) & 1)));
            TC_PROF_WAIT(6, mbar_wait(&rl_full[il], static_cast<unsigned>((ring_s / kRL) & 1)));
            mbar_wait(&rb_full[ib], resident ? 0u : static_cast<unsigned>((ring_s / kRB) & 1));
            tc_fence_after();
            if (lane == 0) {
              const unsigned a_hi = smem_u32(ra_slot(ia)), a_lo = smem_u32(rl_slot(il));
              const unsigned b_hi = smem_u32(rb_slot(ib)), b_lo = b_hi + kBSlot / 2;
#pragma unroll
              for (int ks = 0; ks < kBK / 8; ++ks) {
                const u64 dah = kmajor_desc(a_hi, ks), dal = kmajor_desc(a_lo, ks);
                const u64 dbh = kmajor_desc(b_hi, ks), dbl = kmajor_desc(b_lo, ks);
                const unsigned first = (kk == k_lo && ks == 0) ? 0u : 1u;
                if constexpr (PAIR) {
                  tc_mma_tf32_pair(d, dal, dbh, idesc, first);
                  tc_mma_tf32_pair(d, dah, dbl, idesc, 1u);
                  tc_mma_tf32_pair(d, dah, dbh, idesc, 1u);
                } else {
                  tc_mma_tf32(d, dal, dbh, idesc, first);  // small terms first
                  tc_mma_tf32(d, dah, dbl, idesc, 1u);
                  tc_mma_tf32(d, dah, dbh, idesc, 1u);
                }
              }
#ifdef PK_TC_PROF
              prof_acc[7] += 1;
#endif
              if constexpr (PAIR) {  // release the stage in both CTAs
                tc_commit_pair(&ra_empty[ia]);
                tc_commit_pair(&rl_empty[il]);
                tc_commit_pair(&rb_empty[ib]);
              } else {
                tc_commit(&ra_empty[ia]);
                tc_commit(&rl_empty[il]);
                if (!resident) tc_commit(&rb_empty[ib]);
              }
            }
            __syncwarp();
            ++ring_s;
            continue;
          }
          if constexpr (TMA) TC_PROF_WAIT(2, mbar_wait(&raw[stage], phase));  // TMA landed
          TC_PROF_WAIT(6, mbar_wait(&full[stage], phase));
          tc_fence_after();
          if (lane == 0) {
            const unsigned base = smem_u32(smem + static_cast<size_t>(stage) * Cfg::kStage);
            const unsigned a_hi = base, a_lo = base + Cfg::kTileA;
            const unsigned b_hi = base + 2 * Cfg::kTileA, b_lo = b_hi + Cfg::kTileB;
#pragma unroll
            for (int ks = 0; ks < kBK / 8; ++ks) {
              u64 dah, dal, dbh, dbl;
              if constexpr (TMA && A_T) {
                dah = mnmajor_tma_desc(a_hi, ks), dal = mnmajor_tma_desc(a_lo, ks);
              } else {
                dah = Cfg::LoadA::desc(a_hi, ks), dal = Cfg::LoadA::desc(a_lo, ks);
              }
              if constexpr (B_PRE) {
                dbh = kmajor_desc(b_hi, ks), dbl = kmajor_desc(b_lo, ks);
              } else if constexpr (TMA) {
                dbh = mnmajor_tma_desc(b_hi, ks), dbl = mnmajor_tma_desc(b_lo, ks);
              } else {
                dbh = Cfg::LoadB::desc(b_hi, ks), dbl = Cfg::LoadB::desc(b_lo, ks);
              }
              const unsigned first = (kk == k_lo && ks == 0) ? 0u : 1u;
              tc_mma_tf32(d, dal, dbh, idesc, first);  // small terms first
              tc_mma_tf32(d, dah, dbl, idesc, 1u);
              tc_mma_tf32(d, dah, dbh, idesc, 1u);
            }
#ifdef PK_TC_PROF
            prof_acc[7] += 1;
#endif
            // frees the smem stage (in every cluster CTA) when the MMAs finish
            if constexpr (CS > 1)
              tc_commit_mc(&empty[stage], kMask);
            else
              tc_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) stage = 0, phase ^= 1u;
        }
        if (lane == 0) {
          if (k_hi == k_lo) {
            // empty k range: the epilogue writes zeros without reading TMEM
            mbar_arrive(&tfull[acc]);
          } else if constexpr (PAIR) {
            tc_commit_pair(&tfull[acc]);  // both CTAs' epilogues
          } else {
            tc_commit(&tfull[acc]);
          }
        }
        __syncwarp();
        if (++acc == 2) acc = 0, acc_phase ^= 1u;
      }
    }
    }
  mma_done:;
  } else {
    // ------------------------------------------------------------ epilogue
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int row = quad * 32 + lane;
    int acc = 0;
    unsigned acc_phase = 0;
    for (int t = tile_first; live(t); t += tile_step) {
      int mt, nt, sp;
      tile_coords(t, mt, nt, sp);
      i64 kb, ke;
      k_range(sp, kb, ke);
      const int nk = static_cast<int>((ke - kb + kBK - 1) / kBK);
      const int nseg = nk == 0 ? 1 : (nk + kSegStages - 1) / kSegStages;
      const i64 gm = static_cast<i64>(mt) * kBM + row;
      const i64 n0 = static_cast<i64>(nt) * BN;
      float* out = p.c + static_cast<i64>(sp) * p.split_stride;
      const bool vec_out = (p.ldc % 4 == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
      // 32-B row pieces as one 256-bit store (a full sector per thread: half
      // the L2 write requests of two 16-B stores; the epilogue is what bounds
      // the wide-N small-K tiles, PK_TC_PROF)
      const bool v8_out = PK_EPI_V8 && p.ldc % 8 == 0 && !p.map.g &&
                          ((reinterpret_cast<uintptr_t>(out) & 31) == 0) &&
                          (!p.mask || (p.ldm % 8 == 0 &&
                                       (reinterpret_cast<uintptr_t>(p.mask) & 31) == 0));
      // segments of one tile land in order: the first stores, later ones add
      // (fp32 round-to-nearest in registers, fixed order: deterministic); the
      // fused ReLU applies to the last segment's sum (never to split partials)
      for (int sg = 0; sg < nseg; ++sg) {
        const bool zero = nk == 0;
        const bool relu = p.relu && p.splits == 1 && sg == nseg - 1;
        // relu_backward (kernels.hpp:103-111) of the finished sum
        const bool masked = p.mask && p.splits == 1 && sg == nseg - 1;
        TC_PROF_WAIT(4, mbar_wait(&tfull[acc], acc_phase));
        tc_fence_after();
        const unsigned taddr = tmem + (static_cast<unsigned>(quad * 32) << 16) +
                               static_cast<unsigned>(acc * Cfg::kAccStride);
        if constexpr (kRing && !PAIR) {
          // TMA-store epilogue (one k segment, no split, no row map): each
          // warp stages its 32 rows x 32 columns in shared memory (128-B
          // swizzle: conflict-free row writes) and one lane stores the box —
          // full 128-B lines instead of a 32-B piece per thread per row
          if (p.tma_store && nseg == 1) {
            unsigned char* stgp = rb_slot(kRB) + quad * 4096;
            const unsigned stg = smem_u32(stgp);
            const i64 mrow0 = static_cast<i64>(mt) * kBM + quad * 32;
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 32) {
              float v[32];
              tmem_ld32(taddr + static_cast<unsigned>(c0), v);
              if (relu) {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = v[i] > 0.f ? v[i] : 0.f;
              }
              if (masked && gm < p.m) {
                const float* mr = p.mask + gm * p.ldm + n0 + c0;
                const i64 left = p.n - (n0 + c0);
                if (left >= 32 && p.ldm % 8 == 0 &&
                    (reinterpret_cast<uintptr_t>(p.mask) & 31) == 0) {
                  // the row's 32 mask values as four 256-bit loads
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    float q[8];
                    asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                                 : "=f"(q[0]), "=f"(q[1]), "=f"(q[2]), "=f"(q[3]), "=f"(q[4]),
                                   "=f"(q[5]), "=f"(q[6]), "=f"(q[7])
                                 : "l"(mr + 8 * j));
#pragma unroll
                    for (int i = 0; i < 8; ++i) v[8 * j + i] = q[i] > 0.f ? v[8 * j + i] : 0.f;
                  }
                } else {
#pragma unroll
                  for (int i = 0; i < 32; ++i)
                    if (i < left && !(__ldg(mr + i) > 0.f)) v[i] = 0.f;
                }
              }
              if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
              __syncwarp();
#pragma unroll
              for (int j = 0; j < 8; ++j)
                asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(
                                 stg + static_cast<unsigned>(lane) * 128u +
                                 (static_cast<unsigned>(j ^ (lane & 7)) << 4)),
                             "f"(v[4 * j]), "f"(v[4 * j + 1]), "f"(v[4 * j + 2]),
                             "f"(v[4 * j + 3])
                             : "memory");
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&tma_c, stgp, static_cast<int>(n0 + c0), static_cast<int>(mrow0));
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
              }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            if (++acc == 2) acc = 0, acc_phase ^= 1u;
            continue;
          }
        }
        // CH columns per step: one TMEM load and, for a later segment, all
        // CH/4 old-value loads in flight together (RMW latency once per step)
#ifndef PK_EPI_CH
#define PK_EPI_CH 8  // measured: 8 beats 32 (11.0 vs 11.7 ms per epoch's GEMMs)
#endif
        constexpr int CH = (BN % PK_EPI_CH == 0) ? PK_EPI_CH : (BN % 16 == 0 ? 16 : 8);
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += CH) {
          float v[CH];
          if (zero) {
#pragma unroll
            for (int i = 0; i < CH; ++i) v[i] = 0.f;
          } else if constexpr (CH == 32) {
            tmem_ld32(taddr + static_cast<unsigned>(c0), v);
          } else if constexpr (CH == 16) {
            tmem_ld16(taddr + static_cast<unsigned>(c0), v);
          } else {
            tmem_ld8(taddr + static_cast<unsigned>(c0), v);
          }
          if (gm < p.m) {
            float* dst = p.map.row(out, p.ldc, gm) + n0 + c0;
            const i64 left = p.n - (n0 + c0);
            if (v8_out && left >= CH) {
#pragma unroll
              for (int j = 0; j < CH / 8; ++j) {
                float* d8 = dst + 8 * j;
                float* w = v + 8 * j;
                if (sg > 0) {
                  float o[8];
                  asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                               : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]),
                                 "=f"(o[5]), "=f"(o[6]), "=f"(o[7])
                               : "l"(d8));
#pragma unroll
                  for (int i = 0; i < 8; ++i) w[i] += o[i];
                }
                if (relu) {
#pragma unroll
                  for (int i = 0; i < 8; ++i) w[i] = w[i] > 0.f ? w[i] : 0.f;
                }
                if (masked) {
                  const float* m8 = p.mask + gm * p.ldm + n0 + c0 + 8 * j;
                  float q[8];
                  asm volatile("ld.global.nc.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                               : "=f"(q[0]), "=f"(q[1]), "=f"(q[2]), "=f"(q[3]), "=f"(q[4]),
                                 "=f"(q[5]), "=f"(q[6]), "=f"(q[7])
                               : "l"(m8));
#pragma unroll
                  for (int i = 0; i < 8; ++i) w[i] = q[i] > 0.f ? w[i] : 0.f;
                }
                asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(d8),
                             "f"(w[0]), "f"(w[1]), "f"(w[2]), "f"(w[3]), "f"(w[4]), "f"(w[5]),
                             "f"(w[6]), "f"(w[7])
                             : "memory");
              }
            } else if (vec_out && left >= CH) {
              float4* d4 = reinterpret_cast<float4*>(dst);
              if (sg > 0) {
                float4 o[CH / 4];
#pragma unroll
                for (int j = 0; j < CH / 4; ++j) o[j] = d4[j];
#pragma unroll
                for (int j = 0; j < CH / 4; ++j) {
                  v[4 * j] += o[j].x, v[4 * j + 1] += o[j].y;
                  v[4 * j + 2] += o[j].z, v[4 * j + 3] += o[j].w;
                }
              }
              if (relu) {
#pragma unroll
                for (int i = 0; i < CH; ++i) v[i] = v[i] > 0.f ? v[i] : 0.f;
              }
              if (masked) {
                const float* mr = p.mask + gm * p.ldm + n0 + c0;
#pragma unroll
                for (int i = 0; i < CH; ++i) v[i] = __ldg(mr + i) > 0.f ? v[i] : 0.f;
              }
#pragma unroll
              for (int j = 0; j < CH / 4; ++j)
                d4[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            } else {
#pragma unroll
              for (int i = 0; i < CH; ++i)
                if (i < left) {
                  const float x = sg > 0 ? dst[i] + v[i] : v[i];
                  const float y = relu ? (x > 0.f ? x : 0.f) : x;
                  dst[i] = masked && !(__ldg(p.mask + gm * p.ldm + n0 + c0 + i) > 0.f) ? 0.f : y;
                }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR && crank != 0)
            mbar_arrive_cluster(&tempty[acc], 0);  // the leader reuses the pair's TMEM
          else
            mbar_arrive(&tempty[acc]);
        }
        if (++acc == 2) acc = 0, acc_phase ^= 1u;
      }
    }
    // the TMA stores have read their staging (and landed) before the CTA
    // releases its shared memory
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }

  tc_fence_before();
  __syncthreads();
#ifdef PK_TC_PROF
  if (threadIdx.x == 0) prof_acc[5] = clock64() - t_kernel;
  if (lane == 0)  // one sample per warp (lane 0 waits like its warp)
    for (int i = 0; i < 8; ++i)
      if (prof_acc[i]) atomicAdd(&g_tc_prof[i], static_cast<unsigned long long>(prof_acc[i]));
#endif
  if constexpr (CS > 1) cluster_sync();  // no CTA leaves while peers may still multicast into it
  if (warp == kMmaWarp) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "n"(Cfg::kTmemCols));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "n"(Cfg::kTmemCols));
  }
}

// B image for NN (W stored k x n) / NT (W stored n x k): per 32-k stage g,
// [hi tile | lo tile], each `rows` x 128 B, K-major 128-B swizzled, zero
// padded past n and k. One thread per (g, row, 16-B chunk).
__global__ void b_image_kernel(const float* __restrict__ w, i64 ldw, bool w_is_kxn, i64 n, i64 k,
                               int rows, i64 stages, int n_tiles, unsigned char* __restrict__ img) {
  // layout [n tile][stage][hi | lo]; n tile t covers rows [t*rows, (t+1)*rows)
  const i64 total = static_cast<i64>(n_tiles) * stages * rows * 8;
  const unsigned tile = static_cast<unsigned>(rows) * 128u;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % 8);
    const int r = static_cast<int>((i / 8) % rows);
    const i64 g = (i / (8 * rows)) % stages;
    const i64 t = i / (8 * rows * stages);
    const i64 gr = t * rows + r;
    float v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const i64 kk = g * kBK + c * 4 + j;
      v[j] = (gr < n && kk < k) ? (w_is_kxn ? w[kk * ldw + gr] : w[gr * ldw + kk]) : 0.f;
    }
    const float4 x = make_float4(v[0], v[1], v[2], v[3]);
    const float4 h = split_hi(x);
    unsigned char* base = img + (t * stages + g) * 2 * tile;
    const unsigned off = kmajor_offset(r, c);
    *reinterpret_cast<float4*>(base + off) = h;
    *reinterpret_cast<float4*>(base + tile + off) = split_lo(x, h);
  }
}

// Deterministic split combine: C = partial[0] + partial[1] + ... in order.
__global__ void tc_split_reduce_kernel(const float* __restrict__ part, int splits, i64 m, i64 n,
                                       i64 ldp, i64 stride, float* __restrict__ c, i64 ldc,
                                       int relu) {
  const i64 idx = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x;
  if (idx >= m * n) return;
  const i64 i = idx / n, j = idx % n;
  float s = part[i * ldp + j];
  for (int z = 1; z < splits; ++z) s += part[z * stride + i * ldp + j];
  c[i * ldc + j] = relu ? (s > 0.f ? s : 0.f) : s;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda
// link). fp32 row-major operand `rows x cols` (cols contiguous, ld elements),
// box {32 cols, box_rows}, zero fill out of bounds.
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static const EncodeTiledFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<EncodeTiledFn>(f);
  }();
  return fn;
}

bool make_map(CUtensorMap* map, const float* base, i64 rows, i64 cols, i64 ld, int box_rows,
              bool mn_major) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(float)};
  const cuuint32_t box[2] = {32u, static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1u, 1u};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the output for the TMA-store epilogue: {n, m}, box {32 cols, 32 rows},
// 128-B swizzle (the staging layout)
bool make_c_map(CUtensorMap* map, float* base, i64 rows, i64 cols, i64 ld) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(float)};
  const cuuint32_t box[2] = {32u, 32u};
  const cuuint32_t estr[2] = {1u, 1u};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool tma_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PK_TC_TMA");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <bool A_T, bool B_T, int BN, bool B_PRE>
void launch_bn(const TcParams& p0, cudaStream_t st) {
  constexpr int kStageBytes = TcConfig<A_T, B_T, BN, 1, B_PRE>::kStage;
  constexpr int STAGES = std::min(6, std::max(2, (200 * 1024) / kStageBytes));
  using Cfg = TcConfig<A_T, B_T, BN, STAGES, B_PRE>;
  // TMA maps: K-major A {k, m} box {32, 128}; MN-major A {m, k} / B {n, k}
  // box {32, 32} per 32-wide atom. Needs 16-B aligned bases and ld % 4 == 0.
  CUtensorMap map_a, map_b, map_c;
  std::memset(&map_a, 0, sizeof(map_a));
  std::memset(&map_b, 0, sizeof(map_b));
  std::memset(&map_c, 0, sizeof(map_c));
  bool tma = tma_enabled() && p0.a.vec && (B_PRE || p0.b.vec);
  if (tma)
    tma = A_T ? make_map(&map_a, p0.a.p, p0.k, p0.a.mn, p0.a.ld, 32, true)
              : make_map(&map_a, p0.a.p, p0.a.mn, p0.k, p0.a.ld, kBM, false);
  if (tma && !B_PRE) tma = make_map(&map_b, p0.b.p, p0.k, p0.b.mn, p0.b.ld, 32, true);
  // weight-image multicast across a cluster of CS CTAs (PK_TC_CLUSTER)
  static const int cluster_pref = [] {
    const char* e = std::getenv("PK_TC_CLUSTER");
    const int v = e ? std::atoi(e) : 1;  // measured neutral at 2, slower at 4
    return v >= 4 ? 4 : (v >= 2 ? 2 : 1);
  }();
  // CTA pairs (tcgen05 cta_group::2, M = 256) for the weight-image forms:
  // bit-identical, but measured slower on the epoch's shapes (NN 256x256
  // 1.77 vs 1.44 ms: the leader waits for the slower CTA's conversion every
  // stage), so opt-in with PK_TC_PAIR=1
  static const bool pair_pref = [] {
    const char* e = std::getenv("PK_TC_PAIR");
    return e && e[0] == '1';
  }();
  int cs = 1;
  if (B_PRE && tma && p0.n_tiles == 1 && p0.splits == 1)
    while (cs < cluster_pref && p0.m_tiles >= 4 * cs * 2) cs *= 2;
  const bool pair = B_PRE && !A_T && BN % 32 == 0 && tma && pair_pref && cs == 1 &&
                    p0.n_tiles == 1 && p0.splits == 1 && p0.m_tiles >= 4;
  if (pair) cs = 2;
  using KernelT = void (*)(TcParams, const CUtensorMap, const CUtensorMap, const CUtensorMap);
  KernelT kernel;
  int variant;
  if (!tma) {
    kernel = gemm_tc_kernel<A_T, B_T, BN, STAGES, B_PRE, false, 1>, variant = 0;
  } else if constexpr (B_PRE && !A_T && BN % 32 == 0) {
    if (pair)
      kernel = gemm_tc_kernel<A_T, B_T, BN, STAGES, B_PRE, true, 2, true>, variant = 4;
    else if (cs == 4)
      kernel = gemm_tc_kernel<A_T, B_T, BN, STAGES, B_PRE, true, 4>, variant = 3;
    else if (cs == 2)
      kernel = gemm_tc_kernel<A_T, B_T, BN, STAGES, B_PRE, true, 2>, variant = 2;
    else
      kernel = gemm_tc_kernel<A_T, B_T, BN, STAGES, B_PRE, true, 1>, variant = 1;
  } else if constexpr (B_PRE) {
    if (cs == 4)
      kernel = gemm_tc_kernel<A_T, B_T, BN, STAGES, B_PRE, true, 4>, variant = 3;
    else if (cs == 2)
      kernel = gemm_tc_kernel<A_T, B_T, BN, STAGES, B_PRE, true, 2>, variant = 2;
    else
      kernel = gemm_tc_kernel<A_T, B_T, BN, STAGES, B_PRE, true, 1>, variant = 1;
  } else {
    kernel = gemm_tc_kernel<A_T, B_T, BN, STAGES, B_PRE, true, 1>, variant = 1;
  }
  // the single-CTA TMA + weight-image kernel runs the ring layout
  const size_t smem = variant == 4 ? Cfg::kSmemPair
                                    : ((B_PRE && variant == 1) ? Cfg::kSmemRing : Cfg::kSmem);
  static thread_local bool attr[5] = {false, false, false, false, false};
  if (!attr[variant]) {
    PK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    attr[variant] = true;
  }
  TcParams p = p0;
  // TMA-store epilogue (PK_TC_TMA_STORE, default on): the single-CTA ring
  // kernel, one k segment, no split / row map, output boxes that stay inside
  // the tile (one n tile, or 32-multiple tile widths), 16-B aligned rows
  static const bool tma_store_pref = [] {
    const char* e = std::getenv("PK_TC_TMA_STORE");
    return !(e && e[0] == '0');
  }();
  p.tma_store = 0;
  if (tma_store_pref && B_PRE && !A_T && variant == 1 && p.splits == 1 && !p.map.g &&
      p.k <= static_cast<i64>(kSegStages) * kBK && (p.n_tiles == 1 || BN % 32 == 0) &&
      p.ldc % 4 == 0 && (reinterpret_cast<uintptr_t>(p.c) & 15) == 0)
    p.tma_store = make_c_map(&map_c, p.c, p.m, p.n, p.ldc) ? 1 : 0;
  // measured neutral (C2: NN 2M x 47 x 256 1.05 vs 1.07 ms, NT 2M x 256 x 47
  // 0.88 vs 0.86; epoch within noise): opt-in
  static const int resident_ok = [] {
    const char* e = std::getenv("PK_TC_RESIDENT");
    return e && e[0] == '1' ? 1 : 0;
  }();
  p.resident_ok = resident_ok;
  if (B_PRE) {
    // split the weight once per call into its per-stage tile images
    const i64 stages = (p.k + kBK - 1) / kBK;
    static thread_local DevBuf<unsigned char> img;
    img.ensure(static_cast<size_t>(p.n_tiles) * stages * 2 * Cfg::kTileB);
    const i64 items = static_cast<i64>(p.n_tiles) * stages * Cfg::kRowsB * 8;
    b_image_kernel<<<ceil_div(items, 256), 256, 0, st>>>(p.b.p, p.b.ld, B_T, p.n, p.k,
                                                         Cfg::kRowsB, stages, p.n_tiles, img.p);
    p.b_stages = stages;
    PK_LAUNCH("gemm tcgen05 b image");
    p.b_image = img.p;
  }
  const i64 tiles = pair ? 2 * ((p.m_tiles + 1) / 2)  // one CTA per half of a pair tile
                        : static_cast<i64>(p.m_tiles) * p.n_tiles * p.splits;
  int grid = static_cast<int>(std::min<i64>(tiles, sm_count()));
  if (cs > 1) {
    grid = std::max(cs, grid / cs * cs);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kThreadsTc);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(cs);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PK_CUDA(cudaLaunchKernelEx(&cfg, kernel, p, map_a, map_b, map_c));
  } else {
    kernel<<<grid, kThreadsTc, smem, st>>>(p, map_a, map_b, map_c);
  }
  PK_LAUNCH("gemm tcgen05 kernel");
}

template <bool A_T, bool B_T, bool B_PRE>
void launch_forms(const TcParams& p, int bn, cudaStream_t st) {
  switch (bn) {
    case 16: return launch_bn<A_T, B_T, 16, B_PRE>(p, st);
    case 32: return launch_bn<A_T, B_T, 32, B_PRE>(p, st);
    case 48: return launch_bn<A_T, B_T, 48, B_PRE>(p, st);
    case 64: return launch_bn<A_T, B_T, 64, B_PRE>(p, st);
    case 96: return launch_bn<A_T, B_T, 96, B_PRE>(p, st);
    case 128: return launch_bn<A_T, B_T, 128, B_PRE>(p, st);
    case 192: return launch_bn<A_T, B_T, 192, B_PRE>(p, st);
    default: return launch_bn<A_T, B_T, 256, B_PRE>(p, st);
  }
}

int pick_bn(i64 n) {
  static const int opts[] = {16, 32, 48, 64, 96, 128, 192, 256};
  for (int b : opts)
    if (n <= b) return b;
  return 256;
}

bool aligned16(const void* p, i64 ld) {
  return (reinterpret_cast<uintptr_t>(p) & 15) == 0 && ld % 4 == 0;
}

}  // namespace

bool gemm_tc_launch(bool ta, bool tb, i64 m, i64 n, i64 k, const float* a, i64 lda,
                    const float* b, i64 ldb, float* c, i64 ldc, cudaStream_t st, bool relu,
                    const RowMap* map, const float* mask, i64 ldm) {
  if (ta && tb) return false;  // not used by the layer
  TcParams p{};
  p.mask = mask;
  p.ldm = ldm;
  if (map) {
    p.map = *map;
    c = map->base[0];  // alignment of the slots (all 16-B aligned)
  }
  p.m = m, p.n = n, p.k = k;
  p.relu = relu ? 1 : 0;
  // A: NN/NT -> K-major (storage m x k); TN -> MN-major (storage k x m)
  p.a = OperandSrc{a, lda, m, aligned16(a, lda)};
  // B: NN -> MN-major (storage k x n); NT -> K-major (storage n x k); TN -> MN-major
  p.b = OperandSrc{b, ldb, n, aligned16(b, ldb)};
  // TN tile width (both operands stream through registers): PK_TN_BN caps it
  // for experiments; default 128 (measured faster than 256: two register
  // sets of 128-wide tiles fit without spills)
  // TMA-fed TN holds no operand registers: 256-wide tiles (each H row block
  // read once) measured 2.1 vs 2.8 ms for the 256x256 dW
  static const int tn_cap = [] {
    const char* e = std::getenv("PK_TN_BN");
    return e ? std::atoi(e) : 0;
  }();
  const bool tn_tma = tma_enabled() && aligned16(a, lda) && aligned16(b, ldb);
  const int tn_width = tn_cap > 0 ? tn_cap : (tn_tma ? 256 : 128);
  static const int nn_cap = [] {  // NN / NT tile width cap (experiments)
    const char* e = std::getenv("PK_NN_BN");
    return e ? std::atoi(e) : 256;
  }();
  const int bn =
      (ta && !tb) ? pick_bn(std::min<i64>(n, tn_width)) : pick_bn(std::min<i64>(n, nn_cap));
  p.m_tiles = static_cast<int>((m + kBM - 1) / kBM);
  p.n_tiles = static_cast<int>((n + bn - 1) / bn);
  const i64 tiles = static_cast<i64>(p.m_tiles) * p.n_tiles;
  // split k when the output alone cannot fill the machine and k is long
  int splits = 1;
  const i64 sms = sm_count();
  if (tiles < sms && k >= 8 * kBK) {
    splits = static_cast<int>(std::min<i64>((sms + tiles - 1) / tiles * 2, k / (4 * kBK)));
    splits = std::max(splits, 1);
  }
  p.k_chunk = ((k + splits - 1) / splits + kBK - 1) / kBK * kBK;
  splits = static_cast<int>((k + p.k_chunk - 1) / p.k_chunk);
  p.splits = splits;
  check(!map || splits == 1, "gemm: mapped output rows need an unsplit k");
  static thread_local DevBuf<float> part;
  if (splits > 1) {
    const i64 ldp = static_cast<i64>(p.n_tiles) * bn;
    p.split_stride = m * ldp;
    part.ensure(static_cast<size_t>(splits) * p.split_stride);
    p.c = part.p;
    p.ldc = ldp;
  } else {
    p.c = c;
    p.ldc = ldc;
    p.split_stride = 0;
  }
  if (!ta && !tb)
    launch_forms<false, true, true>(p, bn, st);
  else if (!ta && tb)
    launch_forms<false, false, true>(p, bn, st);
  else
    launch_forms<true, true, false>(p, bn, st);
  if (splits > 1) {
    tc_split_reduce_kernel<<<ceil_div(m * n, 256), 256, 0, st>>>(part.p, splits, m, n, p.ldc,
                                                                 p.split_stride, c, ldc, p.relu);
    PK_LAUNCH("gemm tcgen05 split reduce");
    if (mask) relu_backward_launch(mask, ldm, c, ldc, m, n, c, ldc, st);
  }
  return true;
}

}  // namespace pk

#ifdef PK_TC_PROF
extern "C" int pk_tc_prof(unsigned long long* out8, int reset) {
  cudaMemcpyFromSymbol(out8, pk::g_tc_prof, sizeof(unsigned long long) * 8);
  if (reset) {
    unsigned long long z[8] = {};
    cudaMemcpyToSymbol(pk::g_tc_prof, z, sizeof(z));
  }
  return 0;
}
#endif

namespace pk {
unsigned gemm_watchdog() {
  unsigned v = 0;
  PK_CUDA(cudaMemcpyFromSymbol(&v, g_gemm_watchdog, sizeof(v)));
  return v;
}
}  // namespace pk
