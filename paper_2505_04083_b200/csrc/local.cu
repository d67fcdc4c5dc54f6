// In-process cluster (local.cuh): rendezvous, abort propagation and the
// event-ordered collectives of ranks that share a process.
#include <cuda_runtime.h>

#include <type_traits>

#include "local.cuh"

namespace pk {

namespace {

constexpr int kMaxMembers = 8;

template <typename T>
struct SrcSet {
  const T* p[kMaxMembers];
};

__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// out[r, c] = src_0[r0 + r, c] + src_1[...] + ... in ascending member order
template <typename T>
__global__ void ordered_sum_kernel(SrcSet<T> s, int g, i64 r0, i64 rows, i64 cols, i64 ld_src,
                                   T* __restrict__ out, i64 ld_out) {
  const i64 n = rows * cols;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = i / cols, c = i % cols;
    const i64 off = (r0 + r) * ld_src + c;
    T acc = s.p[0][off];
    for (int j = 1; j < g; ++j) acc = add_rn(acc, s.p[j][off]);
    out[r * ld_out + c] = acc;
  }
}

unsigned grid_for(i64 n) {
  return static_cast<unsigned>(std::max<i64>(1, std::min<i64>((n + 255) / 256, 148 * 8)));
}

}  // namespace

// ---------------------------------------------------------------------------
// rendezvous

std::vector<LocalSlot> LocalGroup::exchange(int me, const LocalSlot& s) {
  std::unique_lock<std::mutex> lk(mu_);
  if (cl_->aborted()) throw Error(PK_ERR_ABORTED, cl_->abort_message());
  const unsigned long long my = gen_;
  slots_[me] = s;
  if (++arrived_ == g_) {
    result_ = slots_;
    arrived_ = 0;
    ++gen_;
    cv_.notify_all();
    return result_;
  }
  cv_.wait(lk, [&] { return gen_ != my || cl_->aborted(); });
  if (gen_ == my) throw Error(PK_ERR_ABORTED, cl_->abort_message());
  return result_;  // nobody can complete the next generation before we leave
}

void LocalGroup::wake() {
  std::lock_guard<std::mutex> lk(mu_);
  cv_.notify_all();
}

LocalCluster::LocalCluster(const Grid& grid) : grid_(grid) {
  check(grid.size() >= 1 && grid.size() <= 64, "cluster: grid size out of range");
  for (int a = 0; a < 3; ++a) {
    const int groups = grid.size() / grid.extent(a);
    check(grid.extent(a) <= kMaxMembers, "cluster: at most 8 ranks per axis");
    for (int i = 0; i < groups; ++i)
      groups_[a].push_back(std::make_unique<LocalGroup>(this, grid.extent(a)));
  }
}

void LocalCluster::abort(int rank, const std::string& why) {
  {
    std::lock_guard<std::mutex> lk(mu_);
    if (aborted_.load()) return;
    why_ = "cluster aborted: rank " + std::to_string(rank) + " failed: " + why;
    aborted_.store(true);
  }
  for (auto& axis : groups_)
    for (auto& g : axis) g->wake();
}

std::string LocalCluster::abort_message() const {
  std::lock_guard<std::mutex> lk(mu_);
  return why_;
}

// ---------------------------------------------------------------------------
// member side

LocalComm::~LocalComm() {
  if (ready_) cudaEventDestroy(ready_);
  if (done_) cudaEventDestroy(done_);
}

void LocalComm::init(LocalCluster* cl, const Grid& grid, int rank) {
  cl_ = cl;
  grid_ = grid;
  c_ = grid.coords_of(rank);
  PK_CUDA(cudaGetDevice(&device_));
  PK_CUDA(cudaEventCreateWithFlags(&ready_, cudaEventDisableTiming));
  PK_CUDA(cudaEventCreateWithFlags(&done_, cudaEventDisableTiming));
}

std::vector<LocalSlot> LocalComm::rendezvous(int axis, const void* src, i64 ld,
                                             cudaStream_t st) {
  PK_CUDA(cudaEventRecord(ready_, st));
  LocalSlot s;
  s.src = src, s.ev = ready_, s.device = device_, s.ld = ld;
  auto peers = cl_->group(axis, grid_.group_id(axis, c_))->exchange(c_.along(axis), s);
  for (auto& p : peers) {
    if (p.device != device_) {
      int ok = 0;
      PK_CUDA(cudaDeviceCanAccessPeer(&ok, device_, p.device));
      check(ok != 0, "cluster: device " + std::to_string(device_) + " cannot access device " +
                         std::to_string(p.device));
      const cudaError_t e = cudaDeviceEnablePeerAccess(p.device, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else PK_CUDA(e);
    }
    PK_CUDA(cudaStreamWaitEvent(st, p.ev, 0));
  }
  return peers;
}

void LocalComm::done(int axis, cudaStream_t st) {
  PK_CUDA(cudaEventRecord(done_, st));
  LocalSlot s;
  s.ev = done_, s.device = device_;
  auto peers = cl_->group(axis, grid_.group_id(axis, c_))->exchange(c_.along(axis), s);
  for (auto& p : peers) PK_CUDA(cudaStreamWaitEvent(st, p.ev, 0));
}

template <typename T>
void LocalComm::ordered_sum(int axis, const T* src, i64 ld_src, i64 r0, i64 r1, i64 cols,
                            T* out, i64 ld_out, cudaStream_t st) {
  auto peers = rendezvous(axis, src, ld_src, st);
  const int g = static_cast<int>(peers.size());
  SrcSet<T> s{};
  for (int j = 0; j < g; ++j) {
    check(peers[j].ld == ld_src, "cluster: members disagree on a reduction's row stride");
    s.p[j] = static_cast<const T*>(peers[j].src);
  }
  if (r1 > r0 && cols > 0) {
    ordered_sum_kernel<T><<<grid_for((r1 - r0) * cols), 256, 0, st>>>(s, g, r0, r1 - r0, cols,
                                                                      ld_src, out, ld_out);
    PK_LAUNCH("cluster ordered sum");
  }
  done(axis, st);
}

template <typename T>
void LocalComm::all_reduce(int axis, T* buf, i64 rows, i64 cols, i64 ld, cudaStream_t st) {
  const size_t bytes = static_cast<size_t>(std::max<i64>(rows, 1) * ld) * sizeof(T);
  if (tmp_.n < bytes) tmp_.alloc(bytes);
  T* tmp = reinterpret_cast<T*>(tmp_.p);
  ordered_sum<T>(axis, buf, ld, 0, rows, cols, tmp, ld, st);
  if (rows && cols)
    PK_CUDA(cudaMemcpy2DAsync(buf, ld * sizeof(T), tmp, ld * sizeof(T), cols * sizeof(T), rows,
                              cudaMemcpyDeviceToDevice, st));
}

void LocalComm::all_gather_rows(int axis, const float* local, float* out, i64 total_rows, i64 ld,
                                cudaStream_t st) {
  auto peers = rendezvous(axis, local, ld, st);
  const int g = static_cast<int>(peers.size());
  for (int j = 0; j < g; ++j) {
    const i64 off = chunk_start(total_rows, g, j), rows = chunk_size(total_rows, g, j);
    float* dst = out + off * ld;
    if (!rows || peers[j].src == dst) continue;
    check(peers[j].ld == ld, "cluster: members disagree on an all-gather's row stride");
    PK_CUDA(cudaMemcpyAsync(dst, peers[j].src, rows * ld * sizeof(float), cudaMemcpyDefault, st));
  }
  done(axis, st);
}

void LocalComm::all_gather_cols(int axis, const float* local, i64 ld_in, float* out, i64 ld_out,
                                i64 rows, i64 total_cols, cudaStream_t st) {
  auto peers = rendezvous(axis, local, ld_in, st);
  const int g = static_cast<int>(peers.size());
  for (int j = 0; j < g; ++j) {
    const i64 c0 = chunk_start(total_cols, g, j), cj = chunk_size(total_cols, g, j);
    if (!rows || !cj) continue;
    PK_CUDA(cudaMemcpy2DAsync(out + c0, ld_out * sizeof(float), peers[j].src,
                              peers[j].ld * sizeof(float), cj * sizeof(float), rows,
                              cudaMemcpyDefault, st));
  }
  done(axis, st);
}

template void LocalComm::ordered_sum<float>(int, const float*, i64, i64, i64, i64, float*, i64,
                                            cudaStream_t);
template void LocalComm::ordered_sum<double>(int, const double*, i64, i64, i64, i64, double*, i64,
                                             cudaStream_t);
template void LocalComm::all_reduce<float>(int, float*, i64, i64, i64, cudaStream_t);
template void LocalComm::all_reduce<double>(int, double*, i64, i64, i64, cudaStream_t);

}  // namespace pk
