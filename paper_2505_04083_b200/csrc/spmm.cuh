// Internal interface of the SpMM kernels (spmm.cu).
#pragma once

#include <vector>

#include "pk_common.cuh"

namespace pk {

// Arguments of the hub kernel (one CTA per hub row and column slice).
struct SpmmArgs {
  const u64* rp = nullptr;   // CSR row_ptr (absolute rows)
  const u32* ci = nullptr;   // CSR col_idx
  const float* val = nullptr;
  const float* x = nullptr;  // dense operand, row-major, ld = ldx
  i64 ldx = 0;
  float* y = nullptr;        // output rows [r0, r0+nrows), ld = ldy
  i64 ldy = 0;
  i64 r0 = 0;
  i64 nrows = 0;
  int nvec = 0;              // d / VEC
  const i64* hub_rows = nullptr;  // absolute ids, longest first
  int hub_count = 0;
  int hub_slices = 0;
  int hub_blocks = 0;
};

// A reusable schedule of one CSR matrix (built once per adjacency shard,
// like the reference precomputes its shards, engine.hpp:96-113):
//  * hub rows (nnz >= threshold): served by whole CTAs, longest first;
//  * regular rows: a compacted copy of their nonzeros as packed (col, val)
//    pairs, their row ids, offsets, and a bitmap marking the last nonzero of
//    every row, so the list kernel walks one contiguous nonzero stream;
//  * empty rows: zero-filled.
struct SpmmPlan {
  i64 rows = 0;
  u64 threshold = ~0ull;
  int hub_count = 0;
  DevBuf<i64> hub_rows;   // sorted by length, descending
  i64 regular = 0;        // number of regular (non-empty, non-hub) rows
  u64 reg_nnz = 0;
  DevBuf<u32> rl;         // regular row ids, ascending
  DevBuf<u64> rpc;        // offsets into cv, regular + 1
  DevBuf<u64> cv;         // (val bits << 32) | col, per regular nonzero
  DevBuf<u32> endbits;    // bit k: nonzero k ends its row
  i64 empty = 0;
  DevBuf<u32> empty_rows; // ascending
  struct Range {
    i64 r0 = 0, r1 = 0;
    i64 i0 = 0, i1 = 0;   // regular list range
    i64 e0 = 0, e1 = 0;   // empty list range
    int hubs = 0;
    DevBuf<i64> hub_ids;  // subset, longest first
  };
  std::vector<Range> ranges;
};

void spmm_plan_build(SpmmPlan& plan, const pk_csr& a, u64 threshold, cudaStream_t st);

// y[0:r1-r0, 0:d] = A[r0:r1, :] . x, bit-identical to the reference's loop
// (kernels.hpp:39-62). Launches on `st` (hub CTAs on a forked stream joined
// back into `st`).
void spmm_run(SpmmPlan& plan, const pk_csr& a, i64 r0, i64 r1, const float* x, i64 ldx, i64 d,
              float* y, i64 ldy, cudaStream_t st);

// Per-thread fork/join stream used to overlap hub CTAs with the list kernel.
struct SideStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_stream();

}  // namespace pk
