// Per-axis NCCL communicators and the reference's three collectives
// (cluster.hpp:265-340) on device buffers, plus the ring-model byte
// counters of CommStats (cluster.hpp:35-65).
//
// One communicator per grid axis, split from the world communicator with
// color = group_id(axis) and key = coordinate along the axis, so NCCL rank
// order inside a group is the reference's ascending-coordinate order
// (grid.hpp:77-93) and row/column concatenation needs no reordering. Ragged
// ceil-split chunks (layout.hpp:16-26) are handled without padding:
// all-gather = grouped ncclBroadcast into each member's offset,
// reduce-scatter = grouped ncclReduce of each member's row chunk. Singleton
// axes short-circuit like the reference (cluster.hpp:380-386) but still count
// calls. With two members per axis (every axis of 2x2x2) a sum is a+b = b+a,
// so results are bit-identical to the reference's ordered combine.
#pragma once

#include <nccl.h>

#include <array>
#include <memory>

#include "layout.h"
#include "local.cuh"
#include "lsa.cuh"
#include "pk_common.cuh"

namespace pk {

inline void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess || r == ncclInProgress) return;
  throw Error(PK_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
#define PK_NCCL(x) ::pk::nccl_check((x), #x)

// dst[r, c] = src[r, c] for a rows x cols block (strided on both sides)
void copy_block_launch(const float* src, i64 ld_src, i64 rows, i64 cols, float* dst, i64 ld_dst,
                       cudaStream_t st);

enum CollOp : int { kAllGather = 0, kAllReduce = 1, kReduceScatter = 2 };

struct CommCounters {
  u64 calls[3][3] = {};       // [axis][op]
  u64 ring_numer[3][3] = {};  // g * bytes under the ring model
};

class Comms {
 public:
  Comms() = default;
  Comms(const Comms&) = delete;
  Comms& operator=(const Comms&) = delete;
  ~Comms();

  // world_size == 1: no NCCL at all. Otherwise `uid` is the 128-byte
  // ncclUniqueId from rank 0.
  void init(const Grid& grid, int rank, const void* uid, int world_size);
  // In-process cluster (local.cuh): the ranks are threads of this process.
  void init_local(const Grid& grid, int rank, LocalCluster* cluster);
  // Measurement mode: this rank of `grid` runs alone; every collective
  // puts only the rank's own contribution in place (results are not the
  // GCN's) while the byte counters still follow the real grid. Used to
  // measure one rank's share of a grid larger than the machine at hand.
  void init_solo(const Grid& grid, int rank);
  bool ready() const { return world_ != nullptr || local_ || solo_ || grid_.size() == 1; }
  LocalCluster* local_cluster() const { return local_ ? lc_.cluster() : nullptr; }
  bool solo() const { return solo_; }
  // Tear down after a failure (ClusterAborted semantics): NCCL
  // communicators are aborted so no later call can block on them.
  void abort_nccl();
  // This rank failed: tell every rank of the node (shared-memory abort
  // block) and abort the communicators.
  void signal_abort(int rank, const std::string& why);
  // Throws PK_ERR_ABORTED when a rank of the communicator set failed.
  void check_alive() const;
  int size(int axis) const { return grid_.extent(axis); }
  int pos(int axis) const { return coords_.along(axis); }

  // In-place sum over the axis group (cluster.hpp:307-321).
  void all_reduce(float* buf, i64 count, int axis, i64 logical_bytes, cudaStream_t st);
  void all_reduce_f64(double* buf, i64 count, int axis, cudaStream_t st);
  // Row concatenation in coordinate order (cluster.hpp:268-305): member j
  // contributes chunk_size(total_rows, g, j) rows of width `ld` floats;
  // `local` may alias out + own offset.
  void all_gather_rows(const float* local, float* out, i64 total_rows, i64 ld, int axis,
                       i64 logical_cols, cudaStream_t st);
  // Column concatenation (trainer.hpp:499): member j holds rows x c_j
  // (ld_in) with c_j = chunk_size(total_cols, g, j); output rows x total_cols
  // (ld_out). `stage` holds stage_rows * total_cols floats; the rows go
  // through it in chunks of stage_rows (0 = all at once).
  void all_gather_cols(const float* local, i64 ld_in, float* out, i64 ld_out, i64 rows,
                       i64 total_cols, int axis, float* stage, i64 stage_rows, cudaStream_t st);
  // Sum over the group, keep this member's row chunk (cluster.hpp:323-340):
  // buf is rows x ld (clobbered); out receives chunk rows x ld.
  void reduce_scatter_rows(float* buf, float* out, i64 rows, i64 ld, int axis, i64 logical_cols,
                           cudaStream_t st);
  // The part of reduce_scatter_rows covering rows [r0, r1) of the buffer:
  // chunked calls over a partition of [0, rows) add up to the full one.
  void reduce_scatter_rows_range(float* buf, float* out, i64 rows, i64 ld, int axis,
                                 i64 logical_cols, i64 r0, i64 r1, cudaStream_t st);

  // Deterministic ordered reductions over NVLink peer memory (lsa.cu) for
  // one axis: collective setup with the largest partial this axis reduces.
  // Returns the group, or nullptr when the axis is a singleton or peer
  // load/store access is unavailable (callers then use NCCL).
  LsaGroup* lsa(int axis, size_t scratch_elems);
  LsaGroup* lsa(int axis) const;
  // ring-model byte accounting of an all-reduce / reduce-scatter done
  // outside NCCL (cluster.hpp:298-333)
  void count(int op, int axis, i64 logical_bytes);

  CommCounters counters;

 private:
  ncclComm_t axis_comm(int axis) const { return axes_[axis]; }
  bool local_ = false, solo_ = false;
  LocalComm lc_;
  Grid grid_;
  Coords coords_;
  ncclComm_t world_ = nullptr;
  std::array<ncclComm_t, 3> axes_{nullptr, nullptr, nullptr};
  // Communicators are a process-level runtime resource (like the CUDA
  // context): a later engine of the same (device, grid, rank) reuses them
  // instead of paying ncclCommInitRank + three splits again. Every rank runs
  // the same sequence of engine creations, so all ranks take the same
  // branch. PK_NCCL_CACHE=0 turns this off.
  std::shared_ptr<struct CommSet> set_;
};

}  // namespace pk
