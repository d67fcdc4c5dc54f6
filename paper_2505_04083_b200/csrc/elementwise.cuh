// Internal interface of the fused elementwise kernels (elementwise.cu).
#pragma once

#include "pk_common.cuh"

namespace pk {

void relu_forward_launch(const float* q, i64 ldq, i64 rows, i64 cols, float* out, i64 ldo,
                         cudaStream_t st);
void relu_backward_launch(const float* q, i64 ldq, const float* df, i64 lddf, i64 rows,
                          i64 cols, float* out, i64 ldo, cudaStream_t st);

struct CeWorkspace {
  DevBuf<double> partial;
  DevBuf<u32> bad;  // set when a masked-in label is out of range
};

// sums = {loss_sum, count, correct} as doubles on the device.
// scale: 0 writes the unscaled softmax - onehot; otherwise the gradient is
// multiplied by (float)1/(float)scale in the same pass (finalize_loss,
// trainer.hpp:84-87, with the global count known in advance). Only the
// class columns [dc0, dc1) of dlogits are written (dl column 0 = class dc0);
// dc1 < 0 = all classes.
void ce_sums_launch(const float* logits, i64 ldl, i64 rows, i64 classes, const u32* labels,
                    const u8* mask, float* dl, i64 ldd, double* sums, CeWorkspace& ws,
                    cudaStream_t st, u64 scale_count = 0, i64 dc0 = 0, i64 dc1 = -1);
void scale_by_count_launch(float* d, i64 ldd, i64 rows, i64 cols, const double* sums,
                           cudaStream_t st);

struct AdamScalars {
  float b1, b2, omb1, omb2, bias1, bias2, lr, eps;
};
AdamScalars adam_scalars(u64 step, double lr, double beta1, double beta2, double eps);
void adam_launch(float* p, const float* g, float* m, float* v, i64 n, const AdamScalars& s,
                 cudaStream_t st);

}  // namespace pk
