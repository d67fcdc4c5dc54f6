// Internal interface of the SpMM kernels (spmm.cu).
#pragma once

#include <vector>

#include "pk_common.cuh"

namespace pk {

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
  int nvec = 0;              // d / VEC (set by spmm_launch)
  int rows_per_group = 0;    // 0 = auto
  u64 hub_threshold = ~0ull; // rows with nnz >= this are served by hub CTAs
  const i64* hub_rows = nullptr;  // absolute ids, longest first
  int hub_count = 0;
  int hub_slices = 0;        // set by spmm_launch
  int hub_blocks = 0;        // set by spmm_launch
};

// Launches the short-row kernel on `st` and, when the args carry hub rows,
// the hub kernel on a forked stream joined back into `st`.
void spmm_launch(SpmmArgs a, i64 d, cudaStream_t st);

struct SpmmPlan {
  i64 rows = 0;
  u64 threshold = ~0ull;
  int hub_count = 0;
  DevBuf<i64> hub_rows;
  struct Range {
    i64 r0 = 0, r1 = 0;
    int count = 0;
    DevBuf<i64> rows;
  };
  std::vector<Range> range_cache;
};

void spmm_plan_build(SpmmPlan& plan, const pk_csr& a, u64 threshold, cudaStream_t st);
const i64* spmm_plan_range(SpmmPlan& plan, i64 r0, i64 r1, int* count, cudaStream_t st);

// Per-thread fork/join stream used to overlap hub CTAs with short rows.
struct SideStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_stream();

}  // namespace pk
