// Deterministic all-reduce / reduce-scatter over NVLink peer memory.
//
// The reference combines partial sums in ascending coordinate order:
// acc = s[0]; acc += s[1]; ... (cluster.hpp:345-373). NCCL's ring / tree /
// NVLS orders differ for groups of three or more, so the engine's large
// reductions run here instead: every member of an axis group writes its
// partial into a symmetric buffer (ncclMemAlloc + ncclCommWindowRegister,
// NCCL_WIN_COLL_SYMMETRIC), and one kernel per member reads all members'
// partials straight out of their HBM through NVLink (load/store-accessible
// peer mappings) and sums them in coordinate order. The result is the
// reference's, bit for bit, for any group size — and no NCCL kernel shares
// the SMs with the overlapped SpMM / GEMM.
//
// Synchronisation: per-CTA flag barriers in a small symmetric flag buffer.
// CTA b of every member arrives by storing the call's epoch into slot
// [me][b] of every peer's flags (release, system scope) and waits until all
// peers' slots [p][b] in its own flags reach the epoch (acquire). One
// barrier before the reads (all partials complete), one after (nobody reads
// a buffer its owner is about to overwrite). Waits are bounded: a protocol
// failure sets an error flag that the host checks, never a hung GPU.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <mutex>
#include <type_traits>
#include <cstdlib>
#include <cstring>

#include "layout.h"
#include "lsa.cuh"

namespace pk {

namespace {

__device__ unsigned g_lsa_timeout = 0;

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ void flag_store(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned flag_load(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// flags of member m: [g][kLsaBlocks] u32; slot [src][b] is written by src
// Waits are bounded by wall time (%globaltimer), not by a poll count: a
// peer whose host thread pauses for a while (logging, a checkpoint, GC)
// only delays the group; a peer that never arrives within timeout_ns
// (PK_LSA_TIMEOUT_S, default 120 s) sets the error flag the engine checks.
__device__ void barrier(const LsaPeers& P, int b, unsigned epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < P.g; ++p)
      if (p != P.me) flag_store(P.flags[p] + P.me * kLsaBlocks + b, epoch);
    const unsigned long long t0 = globaltimer_ns();
    for (int p = 0; p < P.g; ++p) {
      if (p == P.me) continue;
      const unsigned* f = P.flags[P.me] + p * kLsaBlocks + b;
      unsigned spins = 0;
      while (static_cast<int>(flag_load(f) - epoch) < 0) {
        if ((++spins & 255u) == 0 &&
            (globaltimer_ns() - t0 > P.timeout_ns || (P.abort && *P.abort))) {
          atomicExch(&g_lsa_timeout, 1u);
          break;
        }
        __nanosleep(spins < 64 ? 32 : 256);
      }
    }
  }
  __syncthreads();
}

// out[r, c] = sum_j part_j[r, c] in ascending j, rows [r0, r1) of the
// partial buffers (ld_p) -> out rows starting at out_r0 (ld_o)
// VEC floats per thread per element group: 1, 4 (128-bit) or 8 (256-bit
// loads and stores: half the NVLink read requests of 128-bit ones).
template <int VEC>
struct LsaVec {
  float f[VEC];
};
template <int VEC>
__device__ __forceinline__ LsaVec<VEC> lsa_ld(const float* p) {
  LsaVec<VEC> r;
  if constexpr (VEC == 8) {
    asm volatile("ld.global.cg.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(r.f[0]), "=f"(r.f[1]), "=f"(r.f[2]), "=f"(r.f[3]), "=f"(r.f[4]),
                   "=f"(r.f[5]), "=f"(r.f[6]), "=f"(r.f[7])
                 : "l"(p));
  } else if constexpr (VEC == 4) {
    const float4 v = __ldcg(reinterpret_cast<const float4*>(p));
    r.f[0] = v.x, r.f[1] = v.y, r.f[2] = v.z, r.f[3] = v.w;
  } else {
    r.f[0] = __ldcg(p);
  }
  return r;
}
template <int VEC>
__device__ __forceinline__ LsaVec<VEC> lsa_ld_plain(const float* p) {
  LsaVec<VEC> r;
  if constexpr (VEC == 8) {
    asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=f"(r.f[0]), "=f"(r.f[1]), "=f"(r.f[2]), "=f"(r.f[3]), "=f"(r.f[4]),
                   "=f"(r.f[5]), "=f"(r.f[6]), "=f"(r.f[7])
                 : "l"(p));
  } else if constexpr (VEC == 4) {
    const float4 v = *reinterpret_cast<const float4*>(p);
    r.f[0] = v.x, r.f[1] = v.y, r.f[2] = v.z, r.f[3] = v.w;
  } else {
    r.f[0] = *p;
  }
  return r;
}
template <int VEC>
__device__ __forceinline__ void lsa_st(float* p, const LsaVec<VEC>& v) {
  if constexpr (VEC == 8) {
    asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p),
                 "f"(v.f[0]), "f"(v.f[1]), "f"(v.f[2]), "f"(v.f[3]), "f"(v.f[4]), "f"(v.f[5]),
                 "f"(v.f[6]), "f"(v.f[7])
                 : "memory");
  } else if constexpr (VEC == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v.f[0], v.f[1], v.f[2], v.f[3]);
  } else {
    *p = v.f[0];
  }
}

#ifndef PK_LSA_UNROLL
#define PK_LSA_UNROLL 4
#endif

template <int VEC, int G>
__global__ void __launch_bounds__(256) lsa_reduce_kernel(LsaPeers P, i64 r0, i64 r1, i64 cols,
                                                         i64 ld_p, float* __restrict__ out,
                                                         i64 out_r0, i64 ld_o, int relu,
                                                         const float* __restrict__ mask,
                                                         i64 ldm, unsigned epoch) {
  barrier(P, blockIdx.x, epoch);
  const i64 cv = cols / VEC;
  const i64 total = (r1 - r0) * cv;
  const i64 stride = static_cast<i64>(gridDim.x) * blockDim.x;
  using V = LsaVec<VEC>;
  // kUnroll grid-stride elements per pass, all members' loads issued before
  // the ordered adds: remote NVLink loads are latency-bound, so each thread
  // keeps kUnroll x g of them in flight
  constexpr int kUnroll = PK_LSA_UNROLL;
  for (i64 base = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; base < total;
       base += stride * kUnroll) {
    V x[kUnroll][G];
    i64 off[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const i64 i = base + u * stride;
      const i64 r = r0 + i / cv, c = (i % cv) * VEC;
      off[u] = i < total ? r * ld_p + c : -1;
#pragma unroll
      for (int j = 0; j < G; ++j)
        if (j < P.g && off[u] >= 0) x[u][j] = lsa_ld<VEC>(P.data[j] + off[u]);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (off[u] < 0) continue;
      const i64 i = base + u * stride;
      const i64 r = r0 + i / cv, c = (i % cv) * VEC;
      V acc = x[u][0];
#pragma unroll
      for (int j = 1; j < G; ++j) {
        if (j >= P.g) break;
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc.f[e] = __fadd_rn(acc.f[e], x[u][j].f[e]);
      }
      if (relu) {  // fused relu_forward of the reduced Q (kernels.hpp:94-101)
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc.f[e] = acc.f[e] > 0.f ? acc.f[e] : 0.f;
      }
      const i64 ro = r - r0 + out_r0;
      if (mask) {  // fused relu_backward: keep where relu(Q) > 0
        const V m = lsa_ld_plain<VEC>(mask + ro * ldm + c);
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc.f[e] = m.f[e] > 0.f ? acc.f[e] : 0.f;
      }
      lsa_st<VEC>(out + ro * ld_o + c, acc);
    }
  }
  barrier(P, blockIdx.x, epoch + 1);
}

// Two-member all-pull with the peer's partial streamed by the TMA engine
// (PK_LSA_BULK=1): each CTA walks blocks of whole rows (contiguous in the
// scratch: rows x ld_p floats), one thread issues 1-D bulk copies of the
// peer's block into a 4-stage shared-memory ring (mbarrier transaction
// counts), and every thread adds its own partial (local loads) and the
// staged peer values in coordinate order. The NVLink reads become a few
// large transfers per CTA instead of one 16-B load per thread per element.
// Same row -> CTA assignment on both members, same two barriers as
// lsa_reduce_kernel, same sums bit for bit.
constexpr int kBulkStages = 4;
constexpr int kBulkBytes = 8192;  // per stage (static shared memory: 4 x 8 KB)

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ bool bulk_wait(unsigned long long* bar, unsigned parity,
                                          const LsaPeers& P) {
  const unsigned a = smem_addr(bar);
  const unsigned long long t0 = globaltimer_ns();
  for (unsigned spins = 0;; ++spins) {
    unsigned ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
    if (ok) return true;
    if ((spins & 255u) == 255u &&
        (globaltimer_ns() - t0 > P.timeout_ns || (P.abort && *P.abort))) {
      atomicExch(&g_lsa_timeout, 1u);
      return false;
    }
  }
}

__global__ void __launch_bounds__(256) lsa_reduce2_bulk_kernel(
    LsaPeers P, i64 r0, i64 r1, i64 cols, i64 ld_p, float* __restrict__ out, i64 out_r0,
    i64 ld_o, int relu, const float* __restrict__ mask, i64 ldm, unsigned epoch) {
  __shared__ __align__(128) float stage[kBulkStages][kBulkBytes / 4];
  __shared__ __align__(8) unsigned long long full[kBulkStages];
  barrier(P, blockIdx.x, epoch);
  const int peer = 1 - P.me;
  const float* own = P.data[P.me];
  const float* rem = P.data[peer];
  const i64 rb = std::max<i64>(1, (kBulkBytes / 4) / ld_p);  // rows per block
  const i64 nblk = (r1 - r0 + rb - 1) / rb;
  // this CTA's blocks: blockIdx.x, + gridDim.x, ...
  const i64 mine = blockIdx.x < nblk ? (nblk - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kBulkStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](i64 j) {  // j-th block of this CTA into stage j % S
    const i64 b = blockIdx.x + j * gridDim.x;
    const i64 a0 = r0 + b * rb, a1 = std::min<i64>(r1, a0 + rb);
    const unsigned bytes = static_cast<unsigned>((a1 - a0) * ld_p * 4);
    const int st = static_cast<int>(j % kBulkStages);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     smem_addr(&full[st])),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_addr(stage[st])),
        "l"(rem + a0 * ld_p), "r"(bytes), "r"(smem_addr(&full[st]))
        : "memory");
  };
  if (threadIdx.x == 0)
    for (i64 j = 0; j < std::min<i64>(mine, kBulkStages); ++j) issue(j);
  __shared__ int s_ok;
  for (i64 j = 0; j < mine; ++j) {
    const int st = static_cast<int>(j % kBulkStages);
    // thread 0 waits for the stage (bounded: a timeout / abort is flagged and
    // the CTA stops reading); the block barrier hands the data to the rest
    if (threadIdx.x == 0)
      s_ok = bulk_wait(&full[st], static_cast<unsigned>((j / kBulkStages) & 1), P) ? 1 : 0;
    __syncthreads();
    if (!s_ok) break;
    const i64 b = blockIdx.x + j * gridDim.x;
    const i64 a0 = r0 + b * rb, a1 = std::min<i64>(r1, a0 + rb);
    const i64 cv = cols / 4;
    const i64 total = (a1 - a0) * cv;
    for (i64 i = threadIdx.x; i < total; i += blockDim.x) {
      const i64 rr = i / cv, c = (i % cv) * 4;
      const float4 x = __ldcg(reinterpret_cast<const float4*>(own + (a0 + rr) * ld_p + c));
      const float4 y = *reinterpret_cast<const float4*>(&stage[st][rr * ld_p + c]);
      const float4 s0 = P.me == 0 ? x : y, s1 = P.me == 0 ? y : x;  // coordinate order
      float4 acc = make_float4(__fadd_rn(s0.x, s1.x), __fadd_rn(s0.y, s1.y),
                               __fadd_rn(s0.z, s1.z), __fadd_rn(s0.w, s1.w));
      if (relu) {
        acc.x = acc.x > 0.f ? acc.x : 0.f, acc.y = acc.y > 0.f ? acc.y : 0.f;
        acc.z = acc.z > 0.f ? acc.z : 0.f, acc.w = acc.w > 0.f ? acc.w : 0.f;
      }
      const i64 ro = a0 + rr - r0 + out_r0;
      if (mask) {
        const float4 m = *reinterpret_cast<const float4*>(mask + ro * ldm + c);
        acc.x = m.x > 0.f ? acc.x : 0.f, acc.y = m.y > 0.f ? acc.y : 0.f;
        acc.z = m.z > 0.f ? acc.z : 0.f, acc.w = m.w > 0.f ? acc.w : 0.f;
      }
      *reinterpret_cast<float4*>(out + ro * ld_o + c) = acc;
    }
    __syncthreads();  // the stage is free again
    if (threadIdx.x == 0 && j + kBulkStages < mine) issue(j + kBulkStages);
  }
  barrier(P, blockIdx.x, epoch + 1);
}

// All-reduce at ring cost: 2 (g - 1) / g x M NVLink bytes per member instead
// of the all-pull reduce's (g - 1) x M. Rows [r0, r1) are ceil-split over
// the members; member i
//   phase 1: sums its own chunk over all members' partials (coordinate order,
//            the reference's sum_combine), applies the fused relu / mask,
//            stores the result to its output and pushes it into every
//            peer's scratch at the same place (posted NVLink stores; a peer
//            only ever reads its own chunk there, and only in phase 1);
//   barrier;
//   phase 2: copies the other members' chunks out of its own scratch.
// Element e of a chunk is handled by CTA (e mod stride) / blockDim in both
// phases on every member, so the per-CTA barrier orders each phase-2 read
// after the phase-1 store that produced it. Two barriers, like the reduce.
template <int VEC, int G>
__global__ void __launch_bounds__(256) lsa_allreduce_kernel(LsaPeers P, i64 r0, i64 r1, i64 cols,
                                                            i64 ld_p, float* __restrict__ out,
                                                            i64 out_r0, i64 ld_o, int relu,
                                                            const float* __restrict__ mask,
                                                            i64 ldm, unsigned epoch) {
  using V = typename std::conditional<VEC == 4, float4, float>::type;
  barrier(P, blockIdx.x, epoch);
  const i64 cv = cols / VEC;
  const i64 stride = static_cast<i64>(gridDim.x) * blockDim.x;
  const i64 rows = r1 - r0;
  const i64 base_rows = rows / P.g, rem = rows % P.g;
  auto chunk0 = [&](int k) { return r0 + k * base_rows + (k < rem ? k : rem); };
  const i64 a = chunk0(P.me), b = chunk0(P.me + 1);
  {
    const i64 total = (b - a) * cv;
    constexpr int kUnroll = 4;
    for (i64 base = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; base < total;
         base += stride * kUnroll) {
      V x[kUnroll][G];
      i64 off[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const i64 i = base + u * stride;
        const i64 r = a + i / cv, c = (i % cv) * VEC;
        off[u] = i < total ? r * ld_p + c : -1;
#pragma unroll
        for (int j = 0; j < G; ++j)
          if (j < P.g && off[u] >= 0) x[u][j] = __ldcg(reinterpret_cast<const V*>(P.data[j] + off[u]));
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        if (off[u] < 0) continue;
        const i64 i = base + u * stride;
        const i64 r = a + i / cv, c = (i % cv) * VEC;
        V acc = x[u][0];
#pragma unroll
        for (int j = 1; j < G; ++j) {
          if (j >= P.g) break;
          if constexpr (VEC == 4) {
            acc.x = __fadd_rn(acc.x, x[u][j].x), acc.y = __fadd_rn(acc.y, x[u][j].y);
            acc.z = __fadd_rn(acc.z, x[u][j].z), acc.w = __fadd_rn(acc.w, x[u][j].w);
          } else {
            acc = __fadd_rn(acc, x[u][j]);
          }
        }
        const i64 ro = r - r0 + out_r0;
        if (relu) {
          if constexpr (VEC == 4) {
            acc.x = acc.x > 0.f ? acc.x : 0.f, acc.y = acc.y > 0.f ? acc.y : 0.f;
            acc.z = acc.z > 0.f ? acc.z : 0.f, acc.w = acc.w > 0.f ? acc.w : 0.f;
          } else {
            acc = acc > 0.f ? acc : 0.f;
          }
        }
        if (mask) {
          const V m = *reinterpret_cast<const V*>(mask + ro * ldm + c);
          if constexpr (VEC == 4) {
            acc.x = m.x > 0.f ? acc.x : 0.f, acc.y = m.y > 0.f ? acc.y : 0.f;
            acc.z = m.z > 0.f ? acc.z : 0.f, acc.w = m.w > 0.f ? acc.w : 0.f;
          } else {
            acc = m > 0.f ? acc : 0.f;
          }
        }
        *reinterpret_cast<V*>(out + ro * ld_o + c) = acc;
#pragma unroll
        for (int j = 0; j < G; ++j)
          if (j < P.g && j != P.me)
            __stcg(reinterpret_cast<V*>(const_cast<float*>(P.data[j]) + off[u]), acc);
      }
    }
  }
  __threadfence_system();  // every thread's pushes before the CTA's arrival
  barrier(P, blockIdx.x, epoch + 1);
  for (int k = 0; k < P.g; ++k) {
    if (k == P.me) continue;
    const i64 ka = chunk0(k), kb = chunk0(k + 1);
    const i64 total = (kb - ka) * cv;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total; i += stride) {
      const i64 r = ka + i / cv, c = (i % cv) * VEC;
      *reinterpret_cast<V*>(out + (r - r0 + out_r0) * ld_o + c) =
          __ldcg(reinterpret_cast<const V*>(P.data[P.me] + r * ld_p + c));
    }
  }
}

// Producer-fused reduction (reduce_slots): member i's scratch holds g slots
// of S rows (slot j = member j's partial of chunk i's rows) followed by a
// result region indexed by global row. Phase 1 sums the slots of the own
// chunk in coordinate order, stores out and (unless scatter) pushes to every
// peer's result region; phase 2 copies the other chunks' results. Element e
// of a chunk is handled by the same CTA slot in both phases on every member.
template <int VEC, int G>
__global__ void __launch_bounds__(256) lsa_slots_kernel(LsaPeers P, i64 rows, i64 cols, i64 ld,
                                                        i64 S, float* __restrict__ out,
                                                        i64 ld_o, int relu,
                                                        const float* __restrict__ mask, i64 ldm,
                                                        int scatter, unsigned epoch) {
  using V = typename std::conditional<VEC == 4, float4, float>::type;
  barrier(P, blockIdx.x, epoch);
  const i64 cv = cols / VEC;
  const i64 stride = static_cast<i64>(gridDim.x) * blockDim.x;
  const i64 base_rows = rows / P.g, rem = rows % P.g;
  auto chunk0 = [&](int k) { return k * base_rows + (k < rem ? k : rem); };
  const i64 a = chunk0(P.me), b = chunk0(P.me + 1);
  const float* mine = P.data[P.me];
  const i64 res = static_cast<i64>(P.g) * S * ld;  // result region offset
  {
    const i64 total = (b - a) * cv;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total; i += stride) {
      const i64 lr = i / cv, c = (i % cv) * VEC;
      V x[G];
#pragma unroll
      for (int j = 0; j < G; ++j)
        if (j < P.g) x[j] = __ldcg(reinterpret_cast<const V*>(mine + (j * S + lr) * ld + c));
      V acc = x[0];
#pragma unroll
      for (int j = 1; j < G; ++j) {
        if (j >= P.g) break;
        if constexpr (VEC == 4) {
          acc.x = __fadd_rn(acc.x, x[j].x), acc.y = __fadd_rn(acc.y, x[j].y);
          acc.z = __fadd_rn(acc.z, x[j].z), acc.w = __fadd_rn(acc.w, x[j].w);
        } else {
          acc = __fadd_rn(acc, x[j]);
        }
      }
      const i64 r = a + lr;
      if (relu) {
        if constexpr (VEC == 4) {
          acc.x = acc.x > 0.f ? acc.x : 0.f, acc.y = acc.y > 0.f ? acc.y : 0.f;
          acc.z = acc.z > 0.f ? acc.z : 0.f, acc.w = acc.w > 0.f ? acc.w : 0.f;
        } else {
          acc = acc > 0.f ? acc : 0.f;
        }
      }
      if (mask) {
        const V m = *reinterpret_cast<const V*>(mask + r * ldm + c);
        if constexpr (VEC == 4) {
          acc.x = m.x > 0.f ? acc.x : 0.f, acc.y = m.y > 0.f ? acc.y : 0.f;
          acc.z = m.z > 0.f ? acc.z : 0.f, acc.w = m.w > 0.f ? acc.w : 0.f;
        } else {
          acc = m > 0.f ? acc : 0.f;
        }
      }
      // scatter (a reduce-scatter): out holds only the own chunk's rows
      *reinterpret_cast<V*>(out + (scatter ? lr : r) * ld_o + c) = acc;
      if (!scatter) {
#pragma unroll
        for (int j = 0; j < G; ++j)
          if (j < P.g && j != P.me)
            __stcg(reinterpret_cast<V*>(const_cast<float*>(P.data[j]) + res + r * ld + c), acc);
      }
    }
  }
  if (scatter) {
    barrier(P, blockIdx.x, epoch + 1);  // slots may be rewritten only after all reads
    return;
  }
  __threadfence_system();
  barrier(P, blockIdx.x, epoch + 1);
  // (a trailing barrier follows phase 2: the next producer writes into the
  // peers' scratch without a barrier of its own, and a later reduction's
  // slots may overlap this one's result region)
  for (int k = 0; k < P.g; ++k) {
    if (k == P.me) continue;
    const i64 ka = chunk0(k), kb = chunk0(k + 1);
    const i64 total = (kb - ka) * cv;
    for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < total; i += stride) {
      const i64 r = ka + i / cv, c = (i % cv) * VEC;
      *reinterpret_cast<V*>(out + r * ld_o + c) =
          __ldcg(reinterpret_cast<const V*>(mine + res + r * ld + c));
    }
  }
  barrier(P, blockIdx.x, epoch + 2);
}

__global__ void lsa_peer_ptrs_kernel(ncclWindow_t win, int g, void** out) {
  const int j = threadIdx.x;
  if (j < g) out[j] = ncclGetLsaPointer(win, 0, j);
}

void peer_pointers(ncclWindow_t win, int g, void** host_out) {
  void** d = nullptr;
  PK_CUDA(cudaMalloc(&d, sizeof(void*) * g));
  lsa_peer_ptrs_kernel<<<1, 32>>>(win, g, d);
  PK_LAUNCH("lsa peer pointers");
  PK_CUDA(cudaMemcpy(host_out, d, sizeof(void*) * g, cudaMemcpyDeviceToHost));
  PK_CUDA(cudaFree(d));
}

// one host-mapped abort word per process (zero until a rank fails)
unsigned* g_abort_host = nullptr;
std::mutex g_abort_mu;

const volatile unsigned* abort_flag_device() {
  std::lock_guard<std::mutex> lk(g_abort_mu);
  if (!g_abort_host) {
    PK_CUDA(cudaHostAlloc(&g_abort_host, sizeof(unsigned), cudaHostAllocMapped));
    *g_abort_host = 0;
  }
  unsigned* d = nullptr;
  PK_CUDA(cudaHostGetDevicePointer(&d, g_abort_host, 0));
  return d;
}

}  // namespace

void lsa_signal_abort() {
  std::lock_guard<std::mutex> lk(g_abort_mu);
  if (g_abort_host) __atomic_store_n(g_abort_host, 1u, __ATOMIC_RELEASE);
}

LsaGroup::~LsaGroup() {
  // windows and ncclMemAlloc buffers are released with the communicator
  // (process lifetime, see Comms); nothing to do per engine
}

bool LsaGroup::init(ncclComm_t comm, int g, int me, size_t scratch_elems) {
  g_ = g, me_ = me;
  if (g < 2 || g > kLsaMaxMembers) return false;
  ncclTeam_t lsa = ncclTeamLsa(comm);
  if (lsa.nRanks != g || lsa.rank != me) return false;  // not one node-local group
  scratch_bytes_ = ((scratch_elems * sizeof(float)) + 4095) / 4096 * 4096;
  const size_t flag_bytes = ((g * kLsaBlocks * sizeof(unsigned)) + 4095) / 4096 * 4096;
  if (ncclMemAlloc(&scratch_, scratch_bytes_) != ncclSuccess) return false;
  if (ncclMemAlloc(reinterpret_cast<void**>(&flags_), flag_bytes) != ncclSuccess) return false;
  PK_CUDA(cudaMemset(flags_, 0, flag_bytes));
  PK_CUDA(cudaDeviceSynchronize());
  if (ncclCommWindowRegister(comm, scratch_, scratch_bytes_, &data_win_,
                             NCCL_WIN_COLL_SYMMETRIC) != ncclSuccess)
    return false;
  if (ncclCommWindowRegister(comm, flags_, flag_bytes, &flag_win_, NCCL_WIN_COLL_SYMMETRIC) !=
      ncclSuccess)
    return false;
  void* dp[kLsaMaxMembers] = {};
  void* fp[kLsaMaxMembers] = {};
  peer_pointers(data_win_, g, dp);
  peer_pointers(flag_win_, g, fp);
  peers_.g = g, peers_.me = me;
  static const double timeout_s = [] {
    const char* e = std::getenv("PK_LSA_TIMEOUT_S");
    const double v = e ? std::atof(e) : 120.0;
    return v > 0 ? v : 120.0;
  }();
  peers_.timeout_ns = static_cast<unsigned long long>(timeout_s * 1e9);
  peers_.abort = abort_flag_device();
  for (int j = 0; j < g; ++j) {
    peers_.data[j] = static_cast<const float*>(dp[j]);
    peers_.flags[j] = static_cast<unsigned*>(fp[j]);
  }
  ready_ = true;
  return true;
}

void LsaGroup::reduce(i64 r0, i64 r1, i64 cols, i64 ld_p, float* out, i64 out_r0, i64 ld_o,
                      cudaStream_t st, bool relu, const float* mask, i64 ldm) {
  check(ready_, "lsa reduce: group not initialised");
  check((r1 > 0 ? r1 : 0) * ld_p * sizeof(float) <= scratch_bytes_,
        "lsa reduce: partial exceeds the symmetric scratch");
  const unsigned epoch = epoch_;
  epoch_ += 2;
  const bool v4 = cols % 4 == 0 && ld_p % 4 == 0 && ld_o % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                  (!mask || (ldm % 4 == 0 && (reinterpret_cast<uintptr_t>(mask) & 15) == 0));
  // CTAs per reduce: every member must launch the same count (the barrier
  // slots are per CTA). PK_LSA_CTAS trades NVLink/HBM parallelism against
  // the SMs the overlapped SpMM / GEMM keep.
  static const int ctas = [] {
    const char* e = std::getenv("PK_LSA_CTAS");
    // 296 (2 per SM): C2 at 2 GPUs 7.65 vs 8.46 ms of reductions at 148,
    // 13.3 at 74; NCCL 8.25 (profiles/r2_lsa_ctas_ab_n2.log)
    const int v = e ? std::atoi(e) : 296;
    return std::max(1, std::min(v, kLsaBlocks));
  }();
  auto launch = [&](auto vec_tag, auto g_tag) {
    constexpr int V = decltype(vec_tag)::value, Gm = decltype(g_tag)::value;
    lsa_reduce_kernel<V, Gm><<<ctas, 256, 0, st>>>(peers_, r0, r1, cols, ld_p, out, out_r0, ld_o,
                                                  relu ? 1 : 0, mask, ldm, epoch);
  };
  using V4 = std::integral_constant<int, 4>;
  using V1 = std::integral_constant<int, 1>;
  // 256-bit element groups for two-member groups (PK_LSA_VEC=8)
  static const int vec_pref = [] {
    const char* e = std::getenv("PK_LSA_VEC");
    return e ? std::atoi(e) : 4;
  }();
  const bool v8 = vec_pref >= 8 && cols % 8 == 0 && ld_p % 8 == 0 && ld_o % 8 == 0 &&
                  (reinterpret_cast<uintptr_t>(out) & 31) == 0 &&
                  (!mask || (ldm % 8 == 0 && (reinterpret_cast<uintptr_t>(mask) & 31) == 0));
  static const bool bulk_pref = [] {
    const char* e = std::getenv("PK_LSA_BULK");
    return e && e[0] == '1';
  }();
  if (g_ == 2 && bulk_pref && v4 && ld_p * 4 <= kBulkBytes && ld_p % 4 == 0) {
    lsa_reduce2_bulk_kernel<<<ctas, 256, 0, st>>>(peers_, r0, r1, cols, ld_p, out, out_r0, ld_o,
                                                  relu ? 1 : 0, mask, ldm, epoch);
  } else if (g_ <= 2 && v8) {
    launch(std::integral_constant<int, 8>{}, std::integral_constant<int, 2>{});
  } else if (g_ <= 2) {
    if (v4) launch(V4{}, std::integral_constant<int, 2>{});
    else launch(V1{}, std::integral_constant<int, 2>{});
  } else if (g_ <= 4) {
    if (v4) launch(V4{}, std::integral_constant<int, 4>{});
    else launch(V1{}, std::integral_constant<int, 4>{});
  } else {
    if (v4) launch(V4{}, std::integral_constant<int, 8>{});
    else launch(V1{}, std::integral_constant<int, 8>{});
  }
  PK_LAUNCH("lsa ordered reduce");
}

void LsaGroup::all_reduce(i64 r0, i64 r1, i64 cols, i64 ld_p, float* out, i64 out_r0, i64 ld_o,
                          cudaStream_t st, bool relu, const float* mask, i64 ldm) {
  // Owner-push pays off from three members up: C2 at 4 GPUs, collectives
  // per epoch 1x1x4 26.3 -> 19.5 ms, 4x1x1 28.7 -> 19.5, 1x4x1 42.5 ->
  // 29.5; with two members both move M per member and the all-pull is
  // faster (2x1x1 10.6 vs 13.0 ms; profiles/r2_lsa_push_ab_n4.log).
  // PK_LSA_PUSH=0 never pushes, 1 always, default from g >= 3.
  static const int push = [] {
    const char* e = std::getenv("PK_LSA_PUSH");
    return e ? std::atoi(e) : -1;
  }();
  if (push == 0 || (push < 0 && g_ < 3))
    return reduce(r0, r1, cols, ld_p, out, out_r0, ld_o, st, relu, mask, ldm);
  check(ready_, "lsa all_reduce: group not initialised");
  check((r1 > 0 ? r1 : 0) * ld_p * sizeof(float) <= scratch_bytes_,
        "lsa all_reduce: partial exceeds the symmetric scratch");
  const unsigned epoch = epoch_;
  epoch_ += 2;
  const bool v4 = cols % 4 == 0 && ld_p % 4 == 0 && ld_o % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                  (!mask || (ldm % 4 == 0 && (reinterpret_cast<uintptr_t>(mask) & 15) == 0));
  static const int ctas = [] {
    const char* e = std::getenv("PK_LSA_CTAS");
    const int v = e ? std::atoi(e) : 296;
    return std::max(1, std::min(v, kLsaBlocks));
  }();
  auto launch = [&](auto vec_tag, auto g_tag) {
    constexpr int V = decltype(vec_tag)::value, Gm = decltype(g_tag)::value;
    lsa_allreduce_kernel<V, Gm><<<ctas, 256, 0, st>>>(peers_, r0, r1, cols, ld_p, out, out_r0,
                                                     ld_o, relu ? 1 : 0, mask, ldm, epoch);
  };
  using V4 = std::integral_constant<int, 4>;
  using V1 = std::integral_constant<int, 1>;
  if (g_ <= 2) {
    if (v4) launch(V4{}, std::integral_constant<int, 2>{});
    else launch(V1{}, std::integral_constant<int, 2>{});
  } else if (g_ <= 4) {
    if (v4) launch(V4{}, std::integral_constant<int, 4>{});
    else launch(V1{}, std::integral_constant<int, 4>{});
  } else {
    if (v4) launch(V4{}, std::integral_constant<int, 8>{});
    else launch(V1{}, std::integral_constant<int, 8>{});
  }
  PK_LAUNCH("lsa ring all-reduce");
}

RowMap LsaGroup::slot_map(i64 rows, i64 ld) const {
  RowMap m;
  m.g = g_;
  const i64 S = (rows + g_ - 1) / g_;
  for (int k = 0; k <= g_; ++k) m.start[k] = chunk_start(rows, g_, k);
  for (int k = 0; k < g_; ++k)
    m.base[k] = const_cast<float*>(peers_.data[k]) + static_cast<i64>(me_) * S * ld;
  return m;
}

i64 LsaGroup::slot_scratch_elems(i64 rows, i64 ld) const {
  const i64 S = (rows + g_ - 1) / g_;
  return (static_cast<i64>(g_) * S + rows) * ld;
}

void LsaGroup::reduce_slots(i64 rows, i64 cols, i64 ld, float* out, i64 ld_o, cudaStream_t st,
                            bool relu, const float* mask, i64 ldm, bool scatter) {
  check(ready_, "lsa reduce_slots: group not initialised");
  check(slot_scratch_elems(rows, ld) * sizeof(float) <= scratch_bytes_,
        "lsa reduce_slots: slots exceed the symmetric scratch");
  const unsigned epoch = epoch_;
  epoch_ += 3;
  const i64 S = (rows + g_ - 1) / g_;
  const bool v4 = cols % 4 == 0 && ld % 4 == 0 && ld_o % 4 == 0 &&
                  (reinterpret_cast<uintptr_t>(out) & 15) == 0 &&
                  (!mask || (ldm % 4 == 0 && (reinterpret_cast<uintptr_t>(mask) & 15) == 0));
  static const int ctas = [] {
    const char* e = std::getenv("PK_LSA_CTAS");
    const int v = e ? std::atoi(e) : 296;
    return std::max(1, std::min(v, kLsaBlocks));
  }();
  auto launch = [&](auto vec_tag, auto g_tag) {
    constexpr int V = decltype(vec_tag)::value, Gm = decltype(g_tag)::value;
    lsa_slots_kernel<V, Gm><<<ctas, 256, 0, st>>>(peers_, rows, cols, ld, S, out, ld_o,
                                                 relu ? 1 : 0, mask, ldm, scatter ? 1 : 0, epoch);
  };
  using V4 = std::integral_constant<int, 4>;
  using V1 = std::integral_constant<int, 1>;
  if (g_ <= 2) {
    if (v4) launch(V4{}, std::integral_constant<int, 2>{});
    else launch(V1{}, std::integral_constant<int, 2>{});
  } else if (g_ <= 4) {
    if (v4) launch(V4{}, std::integral_constant<int, 4>{});
    else launch(V1{}, std::integral_constant<int, 4>{});
  } else {
    if (v4) launch(V4{}, std::integral_constant<int, 8>{});
    else launch(V1{}, std::integral_constant<int, 8>{});
  }
  PK_LAUNCH("lsa slot reduce");
}

bool lsa_timed_out() {
  unsigned v = 0;
  PK_CUDA(cudaMemcpyFromSymbol(&v, g_lsa_timeout, sizeof(v)));
  return v != 0;
}

void lsa_clear_timeout() {
  const unsigned z = 0;
  PK_CUDA(cudaMemcpyToSymbol(g_lsa_timeout, &z, sizeof(z)));
}

}  // namespace pk
