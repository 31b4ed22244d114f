// FP64 GEMM on the DMMA tensor path (mma.sync.m8n8k4.f64; sm_100a has no f64 kind of
// tcgen05, so DMMA is the FP64 tensor-core path: 37.07 TF measured, profiles/fp64_peak_r01.json).
// Column-major operands, grouped problems, optional split-K with a deterministic reduce.
#pragma once
#include "common.cuh"

namespace ttb {

struct GemmDesc {
  int64_t M = 0, N = 0, K = 0;
  const double* A = nullptr;
  int64_t lda = 0;
  bool ta = false;  // A stored K x M (use A^T)
  const double* B = nullptr;
  int64_t ldb = 0;
  bool tb = false;  // B stored N x K (use B^T)
  double* C = nullptr;
  int64_t ldc = 0;
  // Optional two-level column addressing of C: column j lives at
  //   (j / ncol_split) * ldc_hi + (j % ncol_split) * ldc      (ncol_split > 0)
  int64_t ncol_split = 0;
  int64_t ldc_hi = 0;
  double alpha = 1.0, beta = 0.0;
};

// C = alpha op(A) op(B) + beta C.  Splits K when the tile grid is small.
void gemm(tt_ctx ctx, const GemmDesc& g);
// Several independent problems in one launch (all must share ta/tb).
void gemm_grouped(tt_ctx ctx, const std::vector<GemmDesc>& gs);

}  // namespace ttb
