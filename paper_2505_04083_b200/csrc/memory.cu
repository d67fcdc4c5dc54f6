// Device allocations of the library (DevBuf, owned CSR arrays): a caching
// allocator over cudaMalloc.
//
// Engine construction allocates tens of large buffers (shards, plans,
// activations, Adam state); cudaMalloc / cudaFree of GB-sized blocks cost
// milliseconds each and far more while the driver reclaims memory another
// engine just released (measured: the same load 137 ms fresh, 312 ms right
// after an engine freed ~20 GB, up to 1.7 s in the bench). Freed blocks
// therefore go to a per-process free list keyed by (device, rounded size) and
// are handed back to the next allocation of that size — a re-built engine of
// the same shape allocates nothing new. A free still synchronises the device
// first, like cudaFree, so a block is never reused under a running kernel.
// The cache is bounded (PK_ALLOC_CACHE_GB, default half the device): going
// over it releases cached blocks until it fits; an out-of-memory cudaMalloc
// releases all of them and retries.
// PK_ALLOC_CACHE=0 selects plain cudaMalloc / cudaFree.
#include <cuda_runtime.h>

#include <cstdlib>
#include <iterator>
#include <map>
#include <mutex>
#include <unordered_map>
#include <utility>
#include <vector>

#include "pk_common.cuh"

namespace pk {

namespace {

struct Block {
  int dev;
  size_t bytes;
};

struct Cache {
  std::mutex mu;
  std::unordered_map<void*, Block> live;
  std::map<std::pair<int, size_t>, std::vector<void*>> free;
  size_t cached = 0;
};

Cache& cache() {
  static Cache* c = new Cache();  // leaked: outlives static destructors
  return *c;
}

bool caching() {
  static const bool on = [] {
    const char* e = std::getenv("PK_ALLOC_CACHE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// default: half of the device's memory (an engine of the bench shape holds
// tens of GB; a smaller cap would drop it on close and defeat the reuse)
size_t cache_cap() {
  static const size_t cap = [] {
    const char* e = std::getenv("PK_ALLOC_CACHE_GB");
    if (e) return static_cast<size_t>(std::atof(e) * (1ull << 30));
    size_t free_b = 0, total = 0;
    if (cudaMemGetInfo(&free_b, &total) != cudaSuccess) total = size_t{64} << 30;
    return total / 2;
  }();
  return cap;
}

// 512-B steps below 1 MiB, 2 MiB steps above (the driver's own granularity)
size_t round_size(size_t b) {
  if (b < (size_t{1} << 20)) return (b + 511) / 512 * 512;
  const size_t g = size_t{2} << 20;
  return (b + g - 1) / g * g;
}

// release cached blocks until `keep` bytes or fewer stay cached
void trim_to_locked(Cache& c, size_t keep) {
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto it = c.free.begin(); it != c.free.end() && c.cached > keep;) {
    cudaSetDevice(it->first.first);
    auto& blocks = it->second;
    while (!blocks.empty() && c.cached > keep) {
      cudaFree(blocks.back());
      blocks.pop_back();
      c.cached -= it->first.second;
    }
    it = blocks.empty() ? c.free.erase(it) : std::next(it);
  }
  cudaSetDevice(cur);
}

void trim_locked(Cache& c) {
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& [key, blocks] : c.free) {
    cudaSetDevice(key.first);
    for (void* p : blocks) cudaFree(p);
  }
  cudaSetDevice(cur);
  c.free.clear();
  c.cached = 0;
}

}  // namespace

void* dev_alloc(size_t bytes) {
  if (!bytes) return nullptr;
  void* p = nullptr;
  if (!caching()) {
    PK_CUDA(cudaMalloc(&p, bytes));
    return p;
  }
  int dev = 0;
  PK_CUDA(cudaGetDevice(&dev));
  const size_t sz = round_size(bytes);
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  auto it = c.free.find({dev, sz});
  if (it != c.free.end() && !it->second.empty()) {
    p = it->second.back();
    it->second.pop_back();
    c.cached -= sz;
  } else if (cudaMalloc(&p, sz) != cudaSuccess) {
    cudaGetLastError();  // clear the OOM and retry with the cache released
    trim_locked(c);
    PK_CUDA(cudaMalloc(&p, sz));
  }
  c.live[p] = Block{dev, sz};
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  if (!caching()) {
    cudaFree(p);
    return;
  }
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  auto it = c.live.find(p);
  if (it == c.live.end()) {  // not ours
    cudaFree(p);
    return;
  }
  const Block b = it->second;
  c.live.erase(it);
  // like cudaFree: nothing still running may touch the block once reused
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != b.dev) cudaSetDevice(b.dev);
  const bool ok = cudaDeviceSynchronize() == cudaSuccess;
  if (cur != b.dev) cudaSetDevice(cur);
  if (!ok) return;  // a failed context: drop the block rather than reuse it
  const size_t cap = cache_cap();
  if (b.bytes > cap) {  // never cache a block bigger than the whole cache
    cudaFree(p);
    return;
  }
  if (c.cached + b.bytes > cap) trim_to_locked(c, cap - b.bytes);
  c.free[{b.dev, b.bytes}].push_back(p);
  c.cached += b.bytes;
}

void dev_trim() {
  Cache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  trim_locked(c);
}

}  // namespace pk
