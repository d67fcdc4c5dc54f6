#include <cuda_runtime.h>
#include <nccl.h>

#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <thread>

#include "comm.cuh"

namespace pk {

namespace {

// out[r, off_j + c] = stage_j[r, c] for member blocks stacked in `stage`
__global__ void pack_cols_kernel(const float* __restrict__ stage, i64 rows, i64 total_cols,
                                 int g, float* __restrict__ out, i64 ld_out) {
  const i64 n = rows * total_cols;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    const i64 r = i / total_cols, c = i % total_cols;
    // locate the member owning column c (ceil split)
    const i64 base = total_cols / g, rem = total_cols % g;
    int j;
    i64 c0;
    if (c < rem * (base + 1)) {
      j = static_cast<int>(c / (base + 1));
      c0 = j * (base + 1);
    } else {
      j = static_cast<int>(rem + (c - rem * (base + 1)) / base);
      c0 = j * base + rem;
    }
    const i64 cj = j < rem ? base + 1 : base;
    const i64 blk = rows * c0;  // blocks before j hold rows * c0 floats in total
    out[r * ld_out + c] = stage[blk + r * cj + (c - c0)];
  }
}

__global__ void copy_block_kernel(const float* __restrict__ src, i64 ld_src, i64 rows, i64 cols,
                                  float* __restrict__ dst, i64 ld_dst) {
  const i64 n = rows * cols;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<i64>(gridDim.x) * blockDim.x)
    dst[(i / cols) * ld_dst + i % cols] = src[(i / cols) * ld_src + i % cols];
}

unsigned small_grid(i64 n) {
  return static_cast<unsigned>(std::max<i64>(1, std::min<i64>((n + 255) / 256, 4096)));
}

}  // namespace

void copy_block_launch(const float* src, i64 ld_src, i64 rows, i64 cols, float* dst, i64 ld_dst,
                       cudaStream_t st) {
  if (rows == 0 || cols == 0) return;
  copy_block_kernel<<<small_grid(rows * cols), 256, 0, st>>>(src, ld_src, rows, cols, dst,
                                                             ld_dst);
  PK_LAUNCH("copy block");
}

// Abort propagation across the processes of one node (ClusterAborted,
// cluster.hpp:67-71, 240, 434, for one process per GPU): a small POSIX
// shared-memory block named after the NCCL unique id. A rank that fails
// publishes itself there; every rank's monitor thread sees it within a
// millisecond and aborts its communicators (NCCL kernels waiting on the dead
// peer exit) and raises the peer-memory reductions' abort flag (their
// barrier waits exit), so blocked host waits return and the engine raises
// PK_ERR_ABORTED naming the failed rank instead of hanging.
struct AbortBlock {
  unsigned flag;  // 0 = running; set once, by the first failing rank
  int rank;
  char why[504];
};

struct CommSet {
  ncclComm_t world = nullptr;
  std::array<ncclComm_t, 3> axes{nullptr, nullptr, nullptr};
  // symmetric scratch per axis (grows; re-registered when a larger one is
  // needed) — lives as long as the communicators
  std::array<std::unique_ptr<LsaGroup>, 3> lsa;
  std::array<size_t, 3> lsa_elems{0, 0, 0};
  std::array<bool, 3> lsa_failed{false, false, false};
  AbortBlock* ab = nullptr;
  std::thread monitor;
  std::atomic<bool> stop{false}, dead{false};
  std::mutex mu;

  void kill() {
    std::lock_guard<std::mutex> lk(mu);
    if (dead.exchange(true)) return;
    lsa_signal_abort();
    for (auto& c : axes)
      if (c) ncclCommAbort(c), c = nullptr;
    if (world) ncclCommAbort(world), world = nullptr;
  }
  std::string why() const {
    if (!ab) return "cluster aborted";
    char buf[sizeof(ab->why) + 1];
    std::memcpy(buf, ab->why, sizeof(ab->why));
    buf[sizeof(ab->why)] = 0;
    return "cluster aborted: rank " + std::to_string(ab->rank) + " failed: " + buf;
  }
  void publish(int rank, const std::string& msg) {
    if (!ab) return;
    unsigned zero = 0;
    if (__atomic_compare_exchange_n(&ab->flag, &zero, 2u, false, __ATOMIC_ACQ_REL,
                                    __ATOMIC_ACQUIRE)) {
      ab->rank = rank;
      std::strncpy(ab->why, msg.c_str(), sizeof(ab->why) - 1);
      __atomic_store_n(&ab->flag, 1u, __ATOMIC_RELEASE);
    }
  }
  ~CommSet() {
    stop = true;
    if (monitor.joinable()) monitor.join();
    if (!dead) {
      for (auto& c : axes)
        if (c) ncclCommDestroy(c);
      if (world) ncclCommDestroy(world);
    }
    if (ab) munmap(ab, sizeof(AbortBlock));
  }
};

namespace {
std::string abort_block_name(const void* uid) {
  // FNV-1a of the 128-byte unique id
  unsigned long long h = 1469598103934665603ull;
  const auto* p = static_cast<const unsigned char*>(uid);
  for (int i = 0; i < 128; ++i) h = (h ^ p[i]) * 1099511628211ull;
  char name[64];
  std::snprintf(name, sizeof(name), "/pk_abort_%016llx", h);
  return name;
}

AbortBlock* open_abort_block(const std::string& name) {
  const int fd = shm_open(name.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) return nullptr;
  if (ftruncate(fd, sizeof(AbortBlock)) != 0) {
    close(fd);
    return nullptr;
  }
  void* p = mmap(nullptr, sizeof(AbortBlock), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  return p == MAP_FAILED ? nullptr : static_cast<AbortBlock*>(p);
}
}  // namespace

namespace {
std::mutex g_comm_mu;
// intentionally leaked: no NCCL teardown during static destruction at exit
auto& g_comm_cache = *new std::map<std::array<int, 6>, std::shared_ptr<CommSet>>();
bool comm_cache_on() {
  static const bool on = [] {
    const char* e = std::getenv("PK_NCCL_CACHE");
    return !(e && e[0] == '0');
  }();
  return on;
}
}  // namespace

Comms::~Comms() {
  set_.reset();  // cached sets stay alive in the registry until process exit
}

void Comms::init(const Grid& grid, int rank, const void* uid, int world_size) {
  grid_ = grid;
  coords_ = grid.coords_of(rank);
  check(world_size == grid.size(), "comm init: world size " + std::to_string(world_size) +
                                       " != grid size " + std::to_string(grid.size()));
  if (world_size == 1) return;
  int dev = 0;
  PK_CUDA(cudaGetDevice(&dev));
  const std::array<int, 6> key{dev, world_size, rank, grid.g[0], grid.g[1], grid.g[2]};
  {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    auto it = g_comm_cache.find(key);
    if (comm_cache_on() && it != g_comm_cache.end()) set_ = it->second;
  }
  if (!set_) {
    auto fresh = std::make_shared<CommSet>();
    ncclUniqueId id;
    std::memcpy(&id, uid, sizeof(id));
    // every rank maps the block before the (collective) init; rank 0 unlinks
    // the name once init has returned on all ranks — the mappings stay
    const std::string ab_name = abort_block_name(uid);
    fresh->ab = open_abort_block(ab_name);
    // NCCL's CTAs share the SMs with the SpMM / GEMM they overlap.
    // PK_NCCL_MAX_CTAS caps them; the default (NCCL's own choice) measured
    // best: a 16-CTA cap slowed the 2-GPU epoch from 52.9 to 56.6 ms.
    const char* mc = std::getenv("PK_NCCL_MAX_CTAS");
    const int max_ctas = mc ? std::atoi(mc) : 0;
    ncclConfig_t wcfg = NCCL_CONFIG_INITIALIZER;
    if (max_ctas > 0) wcfg.maxCTAs = max_ctas;
    PK_NCCL(ncclCommInitRankConfig(&fresh->world, world_size, id, rank, &wcfg));
    for (int a = 0; a < 3; ++a) {
      if (grid.extent(a) == 1) continue;  // singleton: identity, nothing moves
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      if (max_ctas > 0) cfg.maxCTAs = max_ctas;
      PK_NCCL(ncclCommSplit(fresh->world, grid.group_id(a, coords_), coords_.along(a),
                            &fresh->axes[a], &cfg));
      int n = 0, r = 0;
      PK_NCCL(ncclCommCount(fresh->axes[a], &n));
      PK_NCCL(ncclCommUserRank(fresh->axes[a], &r));
      check(n == grid.extent(a) && r == coords_.along(a), "comm split: inconsistent axis group");
    }
    if (rank == 0) shm_unlink(ab_name.c_str());
    if (fresh->ab) {
      CommSet* cs = fresh.get();
      cs->monitor = std::thread([cs] {
        while (!cs->stop.load()) {
          if (__atomic_load_n(&cs->ab->flag, __ATOMIC_ACQUIRE) == 1u) {
            cs->kill();
            return;
          }
          std::this_thread::sleep_for(std::chrono::milliseconds(1));
        }
      });
    }
    set_ = fresh;
    if (comm_cache_on()) {
      std::lock_guard<std::mutex> lk(g_comm_mu);
      g_comm_cache[key] = fresh;
    }
  }
  world_ = set_->world;
  axes_ = set_->axes;
}

void Comms::init_local(const Grid& grid, int rank, LocalCluster* cluster) {
  check(cluster != nullptr, "comm init: null cluster");
  const Grid& cg = cluster->grid();
  check(cg.g[0] == grid.g[0] && cg.g[1] == grid.g[1] && cg.g[2] == grid.g[2],
        "comm init: the cluster's grid differs from the engine's");
  grid_ = grid;
  coords_ = grid.coords_of(rank);
  local_ = true;
  lc_.init(cluster, grid, rank);
}

void Comms::init_solo(const Grid& grid, int rank) {
  grid_ = grid;
  coords_ = grid.coords_of(rank);
  solo_ = true;
}

void Comms::signal_abort(int rank, const std::string& why) {
  if (!set_) return;
  set_->publish(rank, why);
  abort_nccl();
}

void Comms::check_alive() const {
  if (set_ && set_->dead.load()) throw Error(PK_ERR_ABORTED, set_->why());
}

void Comms::abort_nccl() {
  if (!set_) return;
  // ncclCommAbort ends in-flight operations instead of waiting for them;
  // the set leaves the process cache so no later engine reuses it
  set_->kill();
  {
    std::lock_guard<std::mutex> lk(g_comm_mu);
    for (auto it = g_comm_cache.begin(); it != g_comm_cache.end();)
      it = it->second == set_ ? g_comm_cache.erase(it) : std::next(it);
  }
  world_ = nullptr;
  axes_ = {nullptr, nullptr, nullptr};
}

LsaGroup* Comms::lsa(int axis, size_t elems) {
  const int g = grid_.extent(axis);
  if (g == 1 || !set_) return nullptr;
  static const bool on = [] {
    const char* e = std::getenv("PK_LSA");
    return !(e && e[0] == '0');
  }();
  if (!on || set_->lsa_failed[axis]) return nullptr;
  if (set_->lsa[axis] && set_->lsa_elems[axis] >= elems) return set_->lsa[axis].get();
  // (re)create: collective over the axis communicator, same order on all
  // members (engine load), sizes identical across the group
  auto grp = std::make_unique<LsaGroup>();
  if (!grp->init(axes_[axis], g, coords_.along(axis), elems)) {
    set_->lsa_failed[axis] = true;
    std::fprintf(stderr, "[pk] axis %d: NVLink peer-memory reductions unavailable, using NCCL\n",
                 axis);
    return nullptr;
  }
  set_->lsa[axis] = std::move(grp);
  set_->lsa_elems[axis] = elems;
  return set_->lsa[axis].get();
}

LsaGroup* Comms::lsa(int axis) const {
  if (!set_ || grid_.extent(axis) == 1) return nullptr;
  return set_->lsa[axis] && set_->lsa[axis]->ready() ? set_->lsa[axis].get() : nullptr;
}

void Comms::count(int op, int axis, i64 logical_bytes) {
  const int g = grid_.extent(axis);
  counters.calls[axis][op]++;
  counters.ring_numer[axis][op] += (op == kAllReduce ? 2 : 1) * static_cast<u64>(g - 1) *
                                   static_cast<u64>(logical_bytes);
}

void Comms::all_reduce(float* buf, i64 count, int axis, i64 logical_bytes, cudaStream_t st) {
  const int g = grid_.extent(axis);
  counters.calls[axis][kAllReduce]++;
  counters.ring_numer[axis][kAllReduce] += 2 * static_cast<u64>(g - 1) * logical_bytes;
  if (g == 1 || solo_) return;
  if (local_) return lc_.all_reduce<float>(axis, buf, 1, count, count, st);
  if (count == 0) return;
  check_alive();
  PK_NCCL(ncclAllReduce(buf, buf, count, ncclFloat32, ncclSum, axes_[axis], st));
}

void Comms::all_reduce_f64(double* buf, i64 count, int axis, cudaStream_t st) {
  const int g = grid_.extent(axis);
  // the reference counts the loss sums' 1x3 all-reduce like any other
  // (cluster.hpp:316: 2 (g - 1) x its bytes)
  counters.calls[axis][kAllReduce]++;
  counters.ring_numer[axis][kAllReduce] += 2 * static_cast<u64>(g - 1) * count * sizeof(double);
  if (g == 1 || solo_) return;
  if (local_) return lc_.all_reduce<double>(axis, buf, 1, count, count, st);
  if (count == 0) return;
  check_alive();
  PK_NCCL(ncclAllReduce(buf, buf, count, ncclFloat64, ncclSum, axes_[axis], st));
}

void Comms::all_gather_rows(const float* local, float* out, i64 total_rows, i64 ld, int axis,
                            i64 logical_cols, cudaStream_t st) {
  const int g = grid_.extent(axis), pos = coords_.along(axis);
  counters.calls[axis][kAllGather]++;
  counters.ring_numer[axis][kAllGather] +=
      static_cast<u64>(g - 1) * static_cast<u64>(total_rows) * logical_cols * sizeof(float);
  const i64 own0 = chunk_start(total_rows, g, pos), own_rows = chunk_size(total_rows, g, pos);
  if (g == 1 || solo_) {
    if (local != out + own0 * ld && own_rows)
      PK_CUDA(cudaMemcpyAsync(out + own0 * ld, local, own_rows * ld * sizeof(float),
                              cudaMemcpyDeviceToDevice, st));
    return;
  }
  if (local_) return lc_.all_gather_rows(axis, local, out, total_rows, ld, st);
  check_alive();
  PK_NCCL(ncclGroupStart());
  for (int j = 0; j < g; ++j) {
    const i64 off = chunk_start(total_rows, g, j), rows = chunk_size(total_rows, g, j);
    const float* send = j == pos ? local : out + off * ld;
    PK_NCCL(ncclBroadcast(send, out + off * ld, rows * ld, ncclFloat32, j, axes_[axis], st));
  }
  PK_NCCL(ncclGroupEnd());
  (void)own0;
}

void Comms::all_gather_cols(const float* local, i64 ld_in, float* out, i64 ld_out, i64 rows,
                            i64 total_cols, int axis, float* stage, i64 stage_rows,
                            cudaStream_t st) {
  const int g = grid_.extent(axis), pos = coords_.along(axis);
  counters.calls[axis][kAllGather]++;
  counters.ring_numer[axis][kAllGather] +=
      static_cast<u64>(g - 1) * static_cast<u64>(rows) * total_cols * sizeof(float);
  if (g > 1 && local_) return lc_.all_gather_cols(axis, local, ld_in, out, ld_out, rows, total_cols, st);
  if (rows == 0 || total_cols == 0) return;
  if (g == 1) {
    copy_block_kernel<<<small_grid(rows * total_cols), 256, 0, st>>>(local, ld_in, rows,
                                                                     total_cols, out, ld_out);
    PK_LAUNCH("gather cols copy");
    return;
  }
  if (solo_) {
    const i64 c0 = chunk_start(total_cols, g, pos), cj = chunk_size(total_cols, g, pos);
    if (cj) {
      copy_block_kernel<<<small_grid(rows * cj), 256, 0, st>>>(local, ld_in, rows, cj, out + c0,
                                                               ld_out);
      PK_LAUNCH("gather cols copy");
    }
    return;
  }
  check_alive();
  // per row chunk: own block -> its contiguous slot of `stage`, grouped
  // broadcasts of every member's slot, then pack into the output columns
  const i64 my_c0 = chunk_start(total_cols, g, pos), my_c = chunk_size(total_cols, g, pos);
  const i64 step = stage_rows > 0 ? stage_rows : rows;
  for (i64 q0 = 0; q0 < rows; q0 += step) {
    const i64 nr = std::min(step, rows - q0);
    if (my_c) {
      copy_block_kernel<<<small_grid(nr * my_c), 256, 0, st>>>(local + q0 * ld_in, ld_in, nr,
                                                               my_c, stage + nr * my_c0, my_c);
      PK_LAUNCH("gather cols stage");
    }
    PK_NCCL(ncclGroupStart());
    for (int j = 0; j < g; ++j) {
      const i64 c0 = chunk_start(total_cols, g, j), cj = chunk_size(total_cols, g, j);
      float* slot = stage + nr * c0;
      PK_NCCL(ncclBroadcast(slot, slot, nr * cj, ncclFloat32, j, axes_[axis], st));
    }
    PK_NCCL(ncclGroupEnd());
    pack_cols_kernel<<<small_grid(nr * total_cols), 256, 0, st>>>(stage, nr, total_cols, g,
                                                                  out + q0 * ld_out, ld_out);
    PK_LAUNCH("gather cols pack");
  }
}

void Comms::reduce_scatter_rows(float* buf, float* out, i64 rows, i64 ld, int axis,
                                i64 logical_cols, cudaStream_t st) {
  const int g = grid_.extent(axis), pos = coords_.along(axis);
  counters.calls[axis][kReduceScatter]++;
  counters.ring_numer[axis][kReduceScatter] +=
      static_cast<u64>(g - 1) * static_cast<u64>(rows) * logical_cols * sizeof(float);
  const i64 own0 = chunk_start(rows, g, pos), own_rows = chunk_size(rows, g, pos);
  if (g == 1 || solo_) {
    if (buf != out && own_rows)
      PK_CUDA(cudaMemcpyAsync(out, buf + own0 * ld, own_rows * ld * sizeof(float),
                              cudaMemcpyDeviceToDevice, st));
    return;
  }
  if (local_) return lc_.ordered_sum<float>(axis, buf, ld, own0, own0 + own_rows, logical_cols, out, ld, st);
  PK_NCCL(ncclGroupStart());
  for (int j = 0; j < g; ++j) {
    const i64 off = chunk_start(rows, g, j), cnt = chunk_size(rows, g, j);
    PK_NCCL(ncclReduce(buf + off * ld, j == pos ? out : buf + off * ld, cnt * ld, ncclFloat32,
                       ncclSum, j, axes_[axis], st));
  }
  PK_NCCL(ncclGroupEnd());
}

void Comms::reduce_scatter_rows_range(float* buf, float* out, i64 rows, i64 ld, int axis,
                                      i64 logical_cols, i64 r0, i64 r1, cudaStream_t st) {
  const int g = grid_.extent(axis), pos = coords_.along(axis);
  counters.calls[axis][kReduceScatter]++;
  counters.ring_numer[axis][kReduceScatter] +=
      static_cast<u64>(g - 1) * static_cast<u64>(r1 - r0) * logical_cols * sizeof(float);
  const i64 own0 = chunk_start(rows, g, pos), own1 = chunk_start(rows, g, pos + 1);
  if (g == 1 || solo_) {
    const i64 a = std::max(r0, own0), b = std::min(r1, own1);
    if (buf != out && b > a)
      PK_CUDA(cudaMemcpyAsync(out + (a - own0) * ld, buf + a * ld, (b - a) * ld * sizeof(float),
                              cudaMemcpyDeviceToDevice, st));
    return;
  }
  if (local_) {
    const i64 a = std::max(r0, own0), b = std::max(a, std::min(r1, own1));
    return lc_.ordered_sum<float>(axis, buf, ld, a, b, logical_cols, out + (a - own0) * ld, ld, st);
  }
  PK_NCCL(ncclGroupStart());
  for (int j = 0; j < g; ++j) {
    const i64 a = std::max(r0, chunk_start(rows, g, j)), b = std::min(r1, chunk_start(rows, g, j + 1));
    if (a >= b) continue;
    float* dst = j == pos ? out + (a - own0) * ld : buf + a * ld;
    PK_NCCL(ncclReduce(buf + a * ld, dst, (b - a) * ld, ncclFloat32, ncclSum, j, axes_[axis], st));
  }
  PK_NCCL(ncclGroupEnd());
  (void)own1;
}

}  // namespace pk
