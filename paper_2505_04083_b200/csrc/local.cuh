// In-process cluster: every rank of the grid is a host thread of one
// process, driving its own engine on a device of this process (several ranks
// may share one GPU) — the reference's execution model, `Cluster::run`
// (cluster.hpp:405-442), with its channel rendezvous (GroupChannel::exchange,
// cluster.hpp:140-168) and abort propagation (ClusterAborted,
// cluster.hpp:67-71, 144, 240, 434).
//
// Collectives are device work ordered by CUDA events that the members of an
// axis group swap through a host rendezvous: member i records "ready" on its
// stream, the rendezvous hands every member all members' buffers and events,
// each member's stream waits for all of them and runs the reduction /
// gather kernel reading its peers' buffers directly (same device, or peer
// access between devices of the process), then a second rendezvous of
// "done reading" events keeps every member from overwriting a buffer a peer
// is still reading. Sums run in ascending coordinate order — the reference's
// sum_combine (cluster.hpp:345-373) bit for bit, for any group size.
#pragma once

#include <atomic>
#include <condition_variable>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "layout.h"
#include "pk_common.cuh"

namespace pk {

struct LocalSlot {
  const void* src = nullptr;
  cudaEvent_t ev = nullptr;
  int device = 0;
  i64 ld = 0;
};

class LocalCluster;

// One axis group: a generation rendezvous over g member threads.
class LocalGroup {
 public:
  LocalGroup(LocalCluster* cl, int g) : cl_(cl), g_(g), slots_(g), result_(g) {}
  int size() const { return g_; }
  // Blocks until every member posted its slot for this generation; returns
  // all slots in coordinate order. Throws ClusterAborted (PK_ERR_ABORTED)
  // when another rank failed.
  std::vector<LocalSlot> exchange(int me, const LocalSlot& s);
  void wake();

 private:
  LocalCluster* cl_;
  int g_;
  std::mutex mu_;
  std::condition_variable cv_;
  unsigned long long gen_ = 0;
  int arrived_ = 0;
  std::vector<LocalSlot> slots_, result_;
};

class LocalCluster {
 public:
  explicit LocalCluster(const Grid& grid);
  const Grid& grid() const { return grid_; }
  LocalGroup* group(int axis, int group_id) { return groups_[axis][group_id].get(); }
  // First failure wins; every rank blocked in (or later entering) a
  // rendezvous throws ClusterAborted naming it.
  void abort(int rank, const std::string& why);
  bool aborted() const { return aborted_.load(); }
  std::string abort_message() const;

 private:
  Grid grid_;
  std::vector<std::unique_ptr<LocalGroup>> groups_[3];
  std::atomic<bool> aborted_{false};
  mutable std::mutex mu_;
  std::string why_;
};

// Per-member helper used by Comms in local mode.
class LocalComm {
 public:
  ~LocalComm();
  void init(LocalCluster* cl, const Grid& grid, int rank);
  LocalCluster* cluster() const { return cl_; }
  // out rows [0, r1 - r0) = ordered sum of all members' src rows [r0, r1)
  // (src ld = ld_src, out ld = ld_out); T = float or double. The members'
  // src pointers are exchanged; `src` stays readable until the call's
  // second rendezvous has passed on every member.
  template <typename T>
  void ordered_sum(int axis, const T* src, i64 ld_src, i64 r0, i64 r1, i64 cols, T* out,
                   i64 ld_out, cudaStream_t st);
  // in-place all-reduce of buf (rows x cols, ld) through a member scratch
  template <typename T>
  void all_reduce(int axis, T* buf, i64 rows, i64 cols, i64 ld, cudaStream_t st);
  // out rows of member j's chunk [off_j, off_j + rows_j) = member j's local
  void all_gather_rows(int axis, const float* local, float* out, i64 total_rows, i64 ld,
                       cudaStream_t st);
  // out[:, c0_j : c0_j + c_j] = member j's rows x c_j block (its ld_in)
  void all_gather_cols(int axis, const float* local, i64 ld_in, float* out, i64 ld_out, i64 rows,
                       i64 total_cols, cudaStream_t st);

 private:
  std::vector<LocalSlot> rendezvous(int axis, const void* src, i64 ld, cudaStream_t st);
  void done(int axis, cudaStream_t st);
  LocalCluster* cl_ = nullptr;
  Grid grid_;
  Coords c_;
  int device_ = 0;
  cudaEvent_t ready_ = nullptr, done_ = nullptr;
  DevBuf<unsigned char> tmp_;
};

}  // namespace pk
