// TT-vector kernels: block-diagonal TT-sum access, contractions, dots, elements, norms.
#pragma once
#include "common.cuh"

namespace ttb {

constexpr int MAXT = 64;  // terms per gather launch (more terms -> several launches)

// One term of a TT-sum as seen by a core-k kernel.
struct TermCore {
  const double* ptr;  // core k of the term (device)
  int64_t r0, r1;     // its ranks around core k
  int64_t off0, off1; // offsets of its block in the concatenated ranks R_{k-1}, R_k
  double coef;        // c_l (applied on the first core only)
};

// Panel of the last core: A (n_d x R_{d-1}, col-major, lda): A[i, off_l + a] = X_d^(l)(a, i).
void gather_last(tt_ctx ctx, const std::vector<TermCore>& terms, int64_t n, double* A, int64_t lda);
// Concatenated first core M1 (R_1 x n_1 col-major): M1[off_l + b, i] = c_l X_1^(l)(i, b).
void gather_first(tt_ctx ctx, const std::vector<TermCore>& terms, int64_t n, double* M1, int64_t R1);
// Materialised TT-sum core k (R_{k-1} x n x R_k, C order) for tt_sum; zeros off the blocks.
void materialise_core(tt_ctx ctx, const std::vector<TermCore>& terms, int64_t n, int64_t R0, int64_t R1,
                      bool first, bool last, double* out);

// out (cols x rows, col-major, ld cols) = in^T where in is rows x cols col-major (ld rows)
void transpose(tt_ctx ctx, const double* in, int64_t ldin, int64_t rows, int64_t cols, double* out, int64_t ldout);
// sum of squares of n doubles -> *out_dev (deterministic two-stage reduction)
void sumsq(tt_ctx ctx, const double* x, int64_t n, double* out_dev);
void scale_inplace(tt_ctx ctx, double* x, int64_t n, double alpha);
// y = x (device-to-device)
void copy_d2d(tt_ctx ctx, double* y, const double* x, int64_t n);
// out = sum_l coef_l x_l for K equally shaped arrays
void lincomb(tt_ctx ctx, const std::vector<const double*>& xs, const std::vector<double>& coef, int64_t n, double* out);

// Batched TT inner products.  Each pair p: x-cores xc[p*d + k], ranks xr[p*(d+1) + k].
struct DotBatch {
  int d = 0;
  std::vector<int64_t> n;
  std::vector<const double*> xc, yc;
  std::vector<int64_t> xr, yr;
  int P = 0;
};
// traces_dev (optional, P*(d+1)): for x == y pairs, trace(W_k) = ||left part of x through
// core k||_F^2 after every core (entry 0 = 1).
void dot_batch(tt_ctx ctx, const DotBatch& b, double* out_dev, double* traces_dev = nullptr);
// y = A x for a TT-matrix A (cores (ra_k, n_k, n_k, ra_{k+1}), row index then column index) and
// a TT-vector x: a new tensor with ranks ra_k rx_k (the Krylov workload).
// z = x (.) y elementwise (cores: Kronecker products of the slices, ranks multiply).
tt_tensor hadamard(tt_ctx ctx, int d, const std::vector<int64_t>& n, const std::vector<int64_t>& rx,
                   const std::vector<const double*>& xc, const std::vector<int64_t>& ry,
                   const std::vector<const double*>& yc);
tt_tensor matvec(tt_ctx ctx, int d, const std::vector<int64_t>& n, const std::vector<int64_t>& ra,
                 const std::vector<const double*>& acore, const std::vector<int64_t>& rx,
                 const std::vector<const double*>& xcore);
// Same dots through grouped DMMA GEMMs per core (dot_batch takes this route above rank 32).
void dot_batch_gemm(tt_ctx ctx, const DotBatch& b, double* out_dev, double* traces_dev = nullptr);
// Elements x(i_1..i_d) for 0-based multi-indices idx[t*d + k].
void elements(tt_ctx ctx, int d, const std::vector<int64_t>& n, const std::vector<const double*>& core,
              const std::vector<int64_t>& r, const std::vector<int64_t>& idx, int nidx, double* out_dev);

}  // namespace ttb
