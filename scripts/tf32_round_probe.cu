// Probe: how does tcgen05.mma kind::tf32 reduce an fp32 operand with low
// mantissa bits set — truncation, round-to-nearest, or full precision?
// A[m][k] = 1 + m * 2^-14 (+ sign flip on odd m), B = selector (1.0 on k == n%8),
// so D[m][n] = tf32(A[m][n%8]). Prints how many rows match trunc / rn / exact.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o scripts/tf32_round_probe scripts/tf32_round_probe.cu
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstring>

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

// byte offset of (mn, k) in a tile with `rows` mn extent (k < 8 here)
__device__ unsigned off_k(int mn, int k) { return mn * 128 + ((((k >> 2) ^ (mn & 7))) << 4) + (k & 3) * 4; }
__device__ unsigned off_mn(int mn, int k, int rows) {
  (void)rows;
  const int a = mn >> 5, c = (mn & 31) >> 2;
  return a * 1024 + k * 128 + ((c ^ k) << 4) + (mn & 3) * 4;
}

struct Case { int a_mn, b_mn, n, swap; int b32 = 0; };
__host__ __device__ inline float aval(int m) {
  const float v = 1.0f + (float)m * (1.0f / 16384.0f);
  return (m & 1) ? -v : v;
}

// SWIZZLE_128B_BASE32B MN-major (layout type 1): atoms of 4 k-rows x 128 B
// (32 MN values); 32-B chunk (mn%32)/8 XOR (k%4); k-groups of 4 at SBO.
__device__ unsigned off_mn32(int mn, int k, unsigned sbo) {
  const int a = mn >> 5, c = (mn & 31) >> 3, r = k & 3, g = k >> 2;
  return g * sbo + a * 512 + r * 128 + ((c ^ r) << 5) + (mn & 7) * 4;
}

__global__ void probe(Case cs, float* out) {
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
  unsigned char* As = s;           // 16 KB
  unsigned char* Bs = s + 16384;   // 16 KB
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) ((float*)s)[i] = 0.f;
  __syncthreads();
  // a[m][k] = m + 1 + k/16 ; b[n][k] = (k == n % 8) * (1 + n / 8)
  for (int i = threadIdx.x; i < 128 * 8; i += blockDim.x) {
    int m = i / 8, k = i % 8;
    *(float*)(As + (cs.a_mn ? (cs.b32 ? off_mn32(m, k, 2048) : off_mn(m, k, 128)) : off_k(m, k))) = aval(m);
  }
  for (int i = threadIdx.x; i < cs.n * 8; i += blockDim.x) {
    int n = i / 8, k = i % 8;
    float v = (k == n % 8) ? 1.f : 0.f;
    *(float*)(Bs + (cs.b_mn ? (cs.b32 ? off_mn32(n, k, 1024) : off_mn(n, k, 64)) : off_k(n, k))) = v;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned t = tbase;
  if (warp == 0) {
    const unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)cs.a_mn << 15) |
                           ((unsigned)cs.b_mn << 16) | ((unsigned)(cs.n >> 3) << 17) | ((128u >> 4) << 24);
    unsigned la = cs.a_mn ? 1024 : 16, sa = cs.a_mn ? 8192 : 1024;
    unsigned lb = cs.b_mn ? 1024 : 16, sb = cs.b_mn ? 8192 : 1024;
    if (cs.swap) {
      if (cs.a_mn) { unsigned x = la; la = sa; sa = x; }
      if (cs.b_mn) { unsigned x = lb; lb = sb; sb = x; }
    }
    if (cs.b32) {  // atoms of 512 B along MN; k-groups of 4 rows
      if (cs.a_mn) { la = 512; sa = 2048; }
      if (cs.b_mn) { lb = 512; sb = 1024; }
      if (cs.swap) {
        if (cs.a_mn) { unsigned x = la; la = sa; sa = x; }
        if (cs.b_mn) { unsigned x = lb; lb = sb; sb = x; }
      }
    }
    uint64_t da = desc(su(As), la, sa, cs.a_mn && cs.b32 ? 1 : 2),
             db = desc(su(Bs), lb, sb, cs.b_mn && cs.b32 ? 1 : 2);
    if (lane == 0) {
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                   " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n"
                   ::"r"(t), "l"(da), "l"(db), "r"(idesc), "r"(0u));
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)) : "memory");
    }
    __syncwarp();
  }
  unsigned ok = 0;
  for (int spin = 0; spin < (1 << 24) && !ok; ++spin)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(su(&bar)) : "memory");
  if (!ok && threadIdx.x == 0) printf("probe: mma barrier never completed\n");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    for (int c0 = 0; c0 < cs.n; c0 += 8) {
      unsigned r[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(t + ((warp * 32) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int c = 0; c < 8; ++c) out[(warp * 32 + lane) * 64 + c0 + c] = __uint_as_float(r[c]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(t));
}

static float trunc_tf32(float x) { unsigned u; memcpy(&u, &x, 4); u &= 0xffffe000u; float y; memcpy(&y, &u, 4); return y; }
static float rn_tf32(float x) {  // round half to even at bit 13
  unsigned u; memcpy(&u, &x, 4);
  const unsigned lsb = (u >> 13) & 1u;
  u += 0xfffu + lsb; u &= 0xffffe000u;
  float y; memcpy(&y, &u, 4); return y;
}
static float rna_tf32(float x) { unsigned u; memcpy(&u, &x, 4); u += 0x1000u; u &= 0xffffe000u; float y; memcpy(&y, &u, 4); return y; }

int main() {
  float* d;
  CK(cudaMalloc(&d, 128 * 64 * 4));
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  std::vector<float> h(128 * 64);
  const Case cases[] = {{0, 0, 16, 0}, {1, 0, 16, 0, 1}};
  for (const Case& cs : cases) {
    CK(cudaMemset(d, 0xff, 128 * 64 * 4));
    probe<<<1, 128, 64 * 1024>>>(cs, d);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost));
    int tr = 0, rn = 0, ra = 0, ex = 0, tot = 0;
    for (int m = 0; m < 128; ++m)
      for (int c = 0; c < cs.n; ++c) {
        const float a = aval(m), g = h[m * 64 + c];
        tr += g == trunc_tf32(a); rn += g == rn_tf32(a); ra += g == rna_tf32(a); ex += g == a; ++tot;
      }
    printf("a_mn %d: of %d: trunc %d rn-even %d rna %d exact %d | m=3: a=%.9g got %.9g trunc %.9g rn %.9g\n",
           cs.a_mn, tot, tr, rn, ra, ex, aval(3), h[3 * 64], trunc_tf32(aval(3)), rn_tf32(aval(3)));
  }
  return 0;
}
