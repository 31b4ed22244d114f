// Truncated SVD of a core unfolding for the left-to-right sweep of TT-rounding
// (SURVEY §8(a) a5): column-pivoted Householder QR until the trailing Frobenius mass is
// below theta*tau, LQ of the kept rows, one-sided Jacobi SVD of the small triangle,
// rank decided on sum_{j>rho} sigma_j^2 + e^2 <= tau^2 (exact-SVD decision; ambiguous
// cases resume the QRCP until resolved).
#pragma once
#include "common.cuh"

namespace ttb {

// One-sided Jacobi SVD of the rows x k column-major A (rows >= k) in one CTA:
// A V = U diag(sigma); outputs sorted descending.  U (rows x k), V (k x k), sigma (k), all
// device buffers.  Throws TT_ENOCONV after max_sweeps.
void jacobi_svd(tt_ctx ctx, const double* A, int64_t lda, int64_t rows, int64_t k, double* U, double* V,
                double* sigma);

struct TruncResult {
  int64_t rho = 0;
  int64_t qrcp_steps = 0;
  int64_t resumes = 0;
};

// Y: m x c ROW-major (a core in (rho_{k-1}, n_k, R'_k) layout).  On return:
//   Ucore (m x rho row-major, i.e. core (rho_{k-1}, n_k, rho) layout, alloc'd here),
//   SV    (rho x c row-major) = S_rho V_rho^T.
// keep_all (delta = 0): plain QR, rho = min(m, c).  max_rank > 0 caps rho.
// The QRCP stops once ||R_22||_F <= stop_abs (= min(theta tau, 1e-12 s(x)) from round_sum):
// the SVD of the kept rows then equals the exact truncated SVD to stop_abs.
TruncResult truncated_svd(tt_ctx ctx, const double* Y, int64_t m, int64_t c, double tau, bool keep_all,
                          int64_t max_rank, double stop_abs, DBuf& Ucore, DBuf& SV);

}  // namespace ttb
