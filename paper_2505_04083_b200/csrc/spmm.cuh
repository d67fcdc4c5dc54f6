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
  const float* mask = nullptr;  // optional: y = mask > 0 ? y : 0 (rows as y)
  i64 ldm = 0;
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
  // 0: exact plan — hub rows run on the hub kernel (bit-identical chains).
  // > 0: FAST plan — hub rows are cut into segments of this many nonzeros
  // that the list kernel sums as virtual rows; a fixed-order combine adds a
  // row's segment sums (deterministic, fp32-level difference from the
  // reference's single chain).
  u64 segment = 0;
  int hub_count = 0;
  DevBuf<i64> hub_rows;   // exact plan: sorted by length, descending
  DevBuf<u32> hub_asc;    // FAST plan: hub rows ascending ...
  DevBuf<u32> hub_seg0;   // ... their first segment ...
  DevBuf<u32> hub_nseg;   // ... and segment count
  u64 segments = 0;
  DevBuf<float> partial;  // segments x ld_partial (FAST plan workspace)
  i64 entries = 0;        // list entries: regular rows (+ hub segments)
  u64 list_nnz = 0;
  DevBuf<u32> rowkey;     // row id of every entry, ascending
  DevBuf<u32> rl;         // store target: row id, or 0x80000000 | segment
  DevBuf<u64> rpc;        // nonzero offset of every entry (+1)
  DevBuf<u64> cv;         // (val bits << 32) | col, per list nonzero
  DevBuf<u32> endbits;    // bit k: nonzero k ends its entry
  i64 empty = 0;
  DevBuf<u32> empty_rows; // ascending
  struct Range {
    i64 r0 = 0, r1 = 0;
    i64 i0 = 0, i1 = 0;   // list entry range
    i64 e0 = 0, e1 = 0;   // empty list range
    i64 h0 = 0, h1 = 0;   // FAST plan: hub_asc range
    int hubs = 0;         // exact plan: hub rows in range ...
    DevBuf<i64> hub_ids;  // ... longest first
  };
  std::vector<Range> ranges;
};

// Segment length of FAST plans: 2048 nonzeros, PK_SPMM_SEGMENT overrides
// (0 = exact plans in FAST mode too).
u64 spmm_fast_segment();

// segment = 0: exact plan; > 0: FAST plan with hub rows cut into segments.
void spmm_plan_build(SpmmPlan& plan, const pk_csr& a, u64 threshold, cudaStream_t st,
                     u64 segment = 0);

// y[0:r1-r0, 0:d] = A[r0:r1, :] . x, bit-identical to the reference's loop
// (kernels.hpp:39-62). Launches on `st` (hub CTAs on a forked stream joined
// back into `st`).
// mask (optional, rows laid out like y, ld = ldm): every stored row value
// becomes mask > 0 ? value : 0 — relu_backward (kernels.hpp:103-111) of the
// previous layer fused into this SpMM^T's epilogue.
// map (optional, FAST / hub-free plans only): output row lr = row - r0 goes
// to map->row(y, ldy, lr) — a reduction's owner slots (RowMap).
// max_vec caps the gather width in floats (8 = no cap). paired (FAST plans,
// rows of at most 16 vectors, no mask): each row summed as two interleaved
// chains added at the row end (spmm_pair_kernel) — tolerance-level.
void spmm_run(SpmmPlan& plan, const pk_csr& a, i64 r0, i64 r1, const float* x, i64 ldx, i64 d,
              float* y, i64 ldy, cudaStream_t st, const float* mask = nullptr, i64 ldm = 0,
              const RowMap* map = nullptr, int max_vec = 8, bool paired = false);

// Per-thread fork/join stream used to overlap hub CTAs with the list kernel.
struct SideStream {
  cudaStream_t stream = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_stream();

}  // namespace pk
