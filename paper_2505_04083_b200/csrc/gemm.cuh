// Internal interface of the dense-transform GEMMs (gemm.cu, gemm_tc.cu).
#pragma once

#include "pk_common.cuh"

namespace pk {

// C(m x n, ldc) = op(A) . op(B); A stored (ta ? k x m : m x k), B stored
// (tb ? n x k : k x n). mode: PK_MODE_PARITY (bit-exact) or PK_MODE_FAST.
// relu: store relu(C) instead (relu_forward, kernels.hpp:94-101), fused into
// the tensor-core epilogue, else a separate in-place pass.
// map (FAST only): output row r goes to map->row(c, ldc, r) (RowMap).
// mask: store relu_backward(mask, C) instead (kernels.hpp:103-111: C where
// mask > 0, else 0; mask m x n, ldm) — in the tensor-core epilogue, else a
// separate pass. Not with relu or map.
void gemm_launch(bool ta, bool tb, i64 m, i64 n, i64 k, const float* a, i64 lda,
                 const float* b, i64 ldb, float* c, i64 ldc, int mode, cudaStream_t st,
                 bool relu = false, const RowMap* map = nullptr, const float* mask = nullptr,
                 i64 ldm = 0);

// Tensor-core (tcgen05, 3xTF32) path; returns false when the shape or
// alignment is not covered and the caller should fall back.
bool gemm_tc_launch(bool ta, bool tb, i64 m, i64 n, i64 k, const float* a, i64 lda,
                    const float* b, i64 ldb, float* c, i64 ldc, cudaStream_t st,
                    bool relu = false, const RowMap* map = nullptr, const float* mask = nullptr,
                    i64 ldm = 0);

}  // namespace pk
