// Standalone probe of the tcgen05 building blocks used by gemm_tc.cu:
//   1. TMEM alloc + tcgen05.st / tcgen05.ld round trip
//   2. one kind::tf32 MMA (M=128, N=16, K=8) from K-major SW128 tiles
//   3. the same with an MN-major SW128 B operand
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o scripts/tc_probe scripts/tc_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(unsigned addr, unsigned lbo, unsigned sbo, int layout) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= (uint64_t)layout << 61;
  return d;
}

// mode 0: TMEM round trip; mode 1: MMA K-major A and B; mode 2: MMA K-major A, MN-major B
__global__ void probe(int mode, float* out, unsigned idesc_override) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* s = (unsigned char*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
  __shared__ unsigned tbase;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(su(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  // A: 128 x 8 (k) values a[m][k] = m + 1 (so D[m][n] = sum_k a*b)
  // B: 16 (n) x 8 (k) values b[n][k] = (k == n % 8) ? 1 : 0   -> D[m][n] = m + 1
  float* As = (float*)s;                 // 128 rows x 32 floats (K-major SW128)
  float* Bs = (float*)(s + 16384);       // K-major: 16 rows x 32 floats; MN-major: 32 k x 32 n
  for (int i = threadIdx.x; i < 4096 * 2; i += blockDim.x) ((float*)s)[i] = 0.f;
  __syncthreads();
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
    int m = i / 8, k = i % 8;
    unsigned off = m * 128 + ((((k >> 2) ^ (m & 7))) << 4) + (k & 3) * 4;
    *(float*)((unsigned char*)As + off) = (float)(m + 1);
  }
  for (int i = threadIdx.x; i < 16 * 8; i += blockDim.x) {
    int n = i / 8, k = i % 8;
    float v = (k == n % 8) ? 1.f : 0.f;
    if (n >= 8) v *= 2.f;
    unsigned off;
    if (mode != 2) {
      off = n * 128 + ((((k >> 2) ^ (n & 7))) << 4) + (k & 3) * 4;
    } else {
      int c = n >> 2;  // chunk of 4 n
      off = k * 128 + ((c ^ k) << 4) + (n & 3) * 4;
    }
    *(float*)((unsigned char*)Bs + off) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned t = tbase;
  if (mode == 0) {
    // each warp writes its lane quadrant: value = lane_row * 100 + col
    if (warp < 4) {
      unsigned r[8];
      for (int c = 0; c < 8; ++c) r[c] = __float_as_uint((float)((warp * 32 + lane) * 100 + c));
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::
                   "r"(t + ((warp * 32) << 16)), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]),
                   "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  } else if (warp == 0) {
    const unsigned idesc = idesc_override ? idesc_override
        : ((1u << 4) | (2u << 7) | (2u << 10) | ((mode == 2 ? 1u : 0u) << 16) | ((16u >> 3) << 17) | ((128u >> 4) << 24));
    uint64_t da = desc(su(As), 16, 1024, 2);
    uint64_t db = mode == 2 ? desc(su(Bs), 1024, 1024, 2) : desc(su(Bs), 16, 1024, 2);
    if (lane == 0) {
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                   " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(t), "l"(da), "l"(db), "r"(idesc), "r"(0u));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
    }
    __syncwarp();
  }
  if (mode != 0) {
    // wait for the MMA
    unsigned ok = 0;
    for (int spin = 0; spin < (1 << 24) && !ok; ++spin)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(su(&bar)) : "memory");
    if (!ok && threadIdx.x == 0) printf("probe: mma barrier never completed\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    unsigned r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                   "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                 : "r"(t + ((warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int c = 0; c < 16; ++c) out[(warp * 32 + lane) * 16 + c] = __uint_as_float(r[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(t));
}

int main() {
  float* d;
  CK(cudaMalloc(&d, 128 * 16 * 4));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  std::vector<float> h(128 * 16);
  for (int mode = 0; mode < 3; ++mode) {
    CK(cudaMemset(d, 0xff, 128 * 16 * 4));
    probe<<<1, 128, 64 * 1024>>>(mode, d, 0);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < 128; ++m)
      for (int c = 0; c < 16; ++c) {
        float want = mode == 0 ? (c < 8 ? (float)(m * 100 + c) : h[m * 16 + c]) : (float)(m + 1) * (c >= 8 ? 2.f : 1.f);
        if (h[m * 16 + c] != want) ++bad;
      }
    printf("mode %d: bad %d | row0: ", mode, bad);
    for (int c = 0; c < 16; ++c) printf("%g ", h[c]);
    printf("| row77: ");
    for (int c = 0; c < 16; ++c) printf("%g ", h[77 * 16 + c]);
    printf("\n");
  }
  return 0;
}
