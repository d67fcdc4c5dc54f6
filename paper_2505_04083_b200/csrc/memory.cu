// Device memory for every buffer the library owns (pk_common.cuh).
//
// The stream-ordered pool of each device keeps freed blocks mapped
// (release threshold = max), so tearing an engine down and building the
// next one — the e2e load after a warm run, a re-shard, a second trainer in
// the same process — recycles mappings instead of going back to the driver.
// Calls are serialised through one private non-blocking stream per device and
// synchronised, which keeps cudaMalloc / cudaFree semantics for callers that
// hand the pointer to any stream.
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "pk_common.cuh"

namespace pk {

namespace {

constexpr int kMaxDevices = 64;

struct PoolState {
  std::once_flag once[kMaxDevices];
  cudaStream_t stream[kMaxDevices] = {};
  std::mutex mu;
};

PoolState& state() {
  static PoolState* s = new PoolState();  // leaked: outlives static destructors
  return *s;
}

cudaStream_t pool_stream(int dev) {
  PoolState& s = state();
  std::call_once(s.once[dev], [&] {
    cudaMemPool_t pool;
    PK_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t keep = ~0ull;
    PK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    PK_CUDA(cudaStreamCreateWithFlags(&s.stream[dev], cudaStreamNonBlocking));
  });
  return s.stream[dev];
}

}  // namespace

bool pool_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PK_POOL");
    return !(e && e[0] == '0');
  }();
  return on;
}

void* dev_alloc(size_t bytes) {
  void* p = nullptr;
  if (!bytes) return p;
  if (!pool_enabled()) {
    PK_CUDA(cudaMalloc(&p, bytes));
    return p;
  }
  int dev = 0;
  PK_CUDA(cudaGetDevice(&dev));
  check(dev < kMaxDevices, "dev_alloc: device ordinal out of range");
  cudaStream_t st = pool_stream(dev);
  std::lock_guard<std::mutex> lock(state().mu);
  PK_CUDA(cudaMallocAsync(&p, bytes, st));
  PK_CUDA(cudaStreamSynchronize(st));
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  if (!pool_enabled()) {
    cudaFree(p);
    return;
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= kMaxDevices) return;
  // like cudaFree: no kernel still using p may be in flight on any stream
  if (cudaDeviceSynchronize() != cudaSuccess) return;
  cudaStream_t st = pool_stream(dev);
  std::lock_guard<std::mutex> lock(state().mu);
  cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
}

}  // namespace pk
