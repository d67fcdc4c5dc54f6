// Shared plumbing for the sm_100a kernels: status codes, the thread-local
// error string behind pk_last_error(), CUDA checks and a small device
// allocation helper. Exceptions never cross the C ABI: every extern "C"
// entry point wraps its body in pk_guard().
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "plexus_b200.h"

namespace pk {

using u8 = uint8_t;
using u32 = uint32_t;
using u64 = uint64_t;
using i64 = int64_t;

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// Reference ContractError wording (common.hpp:47-49).
inline void check(bool ok, const std::string& msg) {
  if (!ok) throw Error(PK_ERR_CONTRACT, msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation)
    throw Error(PK_ERR_MEMORY, std::string(what) + ": " + cudaGetErrorString(e));
  throw Error(PK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

#define PK_CUDA(x) ::pk::cuda_check((x), #x)
// Every kernel launch of the library is followed by PK_LAUNCH, which also
// counts it (pk_kernel_launch_count(); bench.py reports the per-step count).
u64 count_launch();
u64 launch_count();
#define PK_LAUNCH(what) (::pk::count_launch(), ::pk::cuda_check(cudaGetLastError(), what))

void set_last_error(const std::string& msg);

// Device-side watchdogs: a kernel that gave up on a wait it should never
// have had to abandon leaves partial results; these counters say so.
unsigned spmm_watchdog();  // spmm.cu (hub pipeline mbarrier waits)
unsigned gemm_watchdog();  // gemm_tc.cu (tcgen05 pipeline barrier waits)
// Throws PK_ERR_CUDA naming the kernel when a watchdog fired (a sync point:
// call after the work has completed).
void check_device_watchdogs();

template <typename F>
int guard(F&& f) {
  try {
    f();
    return PK_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return PK_ERR_MEMORY;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PK_ERR_CUDA;
  }
}

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Where a producer kernel stores output row lr (0-based in its output): its
// own buffer (g == 0: y + lr * ld), or — for a reduction fused into the
// producer — the slot this rank owns in the symmetric scratch of the member
// that owns the row's chunk: base[k] + (lr - start[k]) * ld for the k with
// start[k] <= lr < start[k + 1] (lsa.cu; remote rows travel over NVLink as
// the producer writes them).
constexpr int kMaxRowOwners = 8;
struct RowMap {
  float* base[kMaxRowOwners] = {};
  i64 start[kMaxRowOwners + 1] = {};
  int g = 0;
#ifdef __CUDACC__
  __device__ __forceinline__ float* row(float* y, i64 ld, i64 lr) const {
    if (g == 0) return y + lr * ld;
    int k = 0;
#pragma unroll
    for (int j = 1; j < kMaxRowOwners; ++j)
      if (j < g && lr >= start[j]) k = j;
    return base[k] + (lr - start[k]) * ld;
  }
#endif
};

inline std::string shape(i64 r, i64 c) {
  return std::to_string(r) + "x" + std::to_string(c);
}

// Device memory of the library: a caching allocator over cudaMalloc
// (memory.cu). dev_free synchronises the device like cudaFree; dev_trim
// returns every cached block to the driver.
void* dev_alloc(size_t bytes);
void dev_free(void* p);
void dev_trim();

// Device buffer owned by RAII; used for workspaces.
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    release();
    p = o.p, n = o.n;
    o.p = nullptr, o.n = 0;
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T)));
  }
  void ensure(size_t count) {
    if (count > n) alloc(count);
  }
  void release() {
    if (p) dev_free(p);
    p = nullptr;
    n = 0;
  }
  T* release_ownership() {
    T* q = p;
    p = nullptr;
    n = 0;
    return q;
  }
};

// Device scratch for setup work (SpMM plans, transposes): one buffer per
// host thread, grown to the largest need and kept, bump-allocated, reset by
// each user at its start. Setup then allocates only its results — the
// temporaries' cudaMalloc/cudaFree pairs were most of the engine's load time.
class Scratch {
 public:
  static Scratch& get() {
    static thread_local Scratch s;
    return s;
  }
  void reset(size_t reserve) {
    extra_.clear();
    if (buf_.n < reserve) buf_.alloc(reserve);
    off_ = 0;
  }
  template <typename T>
  T* take(size_t count) {
    const size_t b = (std::max<size_t>(count, 1) * sizeof(T) + 255) / 256 * 256;
    if (off_ + b > buf_.n) {  // beyond the reservation: a dedicated buffer until reset
      extra_.emplace_back(b);
      return reinterpret_cast<T*>(extra_.back().p);
    }
    T* p = reinterpret_cast<T*>(buf_.p + off_);
    off_ += b;
    return p;
  }
  size_t mark() const { return off_; }
  void release_to(size_t m) { off_ = m; }

 private:
  DevBuf<unsigned char> buf_;
  size_t off_ = 0;
  std::vector<DevBuf<unsigned char>> extra_;
};

inline int sm_count() {
  static thread_local int cached = -1;
  if (cached < 0) {
    int dev = 0;
    PK_CUDA(cudaGetDevice(&dev));
    PK_CUDA(cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev));
  }
  return cached;
}

inline unsigned ceil_div(u64 a, u64 b) { return static_cast<unsigned>((a + b - 1) / b); }

}  // namespace pk
