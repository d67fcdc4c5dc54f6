// Deterministic ordered reductions over NVLink peer memory (lsa.cu).
#pragma once

#include <nccl.h>

#include "pk_common.cuh"

namespace pk {

constexpr int kLsaMaxMembers = 8;
constexpr int kLsaBlocks = 148 * 4;  // max CTAs of a reduce (barrier slots per member)

struct LsaPeers {
  const float* data[kLsaMaxMembers];  // each member's symmetric scratch
  unsigned* flags[kLsaMaxMembers];    // each member's barrier flags
  int g = 0, me = 0;
  unsigned long long timeout_ns = 0;  // bounded barrier waits (wall time)
  const volatile unsigned* abort = nullptr;  // host-mapped: a rank failed
};

// One axis group's symmetric scratch + barrier flags.
class LsaGroup {
 public:
  ~LsaGroup();
  // Collective over `comm` (every member calls it in the same order).
  // Returns false when the group cannot use load/store peer access (then
  // the caller keeps NCCL for this axis).
  bool init(ncclComm_t comm, int g, int me, size_t scratch_elems);
  bool ready() const { return ready_; }
  // This member's partial goes here (row-major, the caller's ld).
  float* scratch() const { return static_cast<float*>(scratch_); }
  size_t scratch_elems() const { return scratch_bytes_ / sizeof(float); }
  // out rows [out_r0, out_r0 + r1 - r0) = sum over members, in coordinate
  // order, of their scratch rows [r0, r1). Collective (same call sequence on
  // every member); runs on `st`. relu: store relu(sum) (the forward's
  // activation fused into the Q reduction). mask (rows indexed like out,
  // ld = ldm): store mask > 0 ? sum : 0 (the backward's relu_backward fused
  // into the dF reduction).
  void reduce(i64 r0, i64 r1, i64 cols, i64 ld_p, float* out, i64 out_r0, i64 ld_o,
              cudaStream_t st, bool relu = false, const float* mask = nullptr, i64 ldm = 0);
  // The same result for a row range every member passes identically (an
  // all-reduce), at ring cost: each member sums its own ceil-split chunk and
  // pushes it to the peers (lsa.cu). The scratch then holds the reduced
  // rows of the other members' chunks. Bit-identical to reduce().
  void all_reduce(i64 r0, i64 r1, i64 cols, i64 ld_p, float* out, i64 out_r0, i64 ld_o,
                  cudaStream_t st, bool relu = false, const float* mask = nullptr, i64 ldm = 0);

  // Producer-fused reduction over rows [0, rows) (ld floats per row). The
  // producer (SpMM / GEMM epilogue) stores its partial of row r straight into
  // the scratch of the member owning r's ceil-split chunk, at this member's
  // slot: slot_map() is that RowMap. reduce_slots() then sums each owner's
  // slots locally in coordinate order (the reference's combine, bit for
  // bit), applies relu / mask, stores the owner's rows and — unless only
  // this member's rows are wanted (scatter: a reduce-scatter) — pushes them
  // to every peer, which copies the other chunks out of its own HBM. NVLink
  // then carries the partials while the producer runs and only the reduced
  // chunks afterwards.
  RowMap slot_map(i64 rows, i64 ld) const;
  i64 slot_scratch_elems(i64 rows, i64 ld) const;  // what slot_map + results need
  void reduce_slots(i64 rows, i64 cols, i64 ld, float* out, i64 ld_o, cudaStream_t st,
                    bool relu = false, const float* mask = nullptr, i64 ldm = 0,
                    bool scatter = false);

 private:
  int g_ = 0, me_ = 0;
  bool ready_ = false;
  void* scratch_ = nullptr;
  size_t scratch_bytes_ = 0;
  unsigned* flags_ = nullptr;
  ncclWindow_t data_win_ = nullptr, flag_win_ = nullptr;
  LsaPeers peers_;
  unsigned epoch_ = 1;
};

// true when a barrier wait gave up (a protocol error; results are invalid)
bool lsa_timed_out();
// Raise the process's abort flag: every peer-memory barrier wait exits.
void lsa_signal_abort();
void lsa_clear_timeout();

}  // namespace pk
