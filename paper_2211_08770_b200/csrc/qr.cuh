// Blocked Householder QR in FP64 for the right-to-left orthogonalisation sweep of
// TT-rounding: tall-skinny panels factored by TSQR (Householder QR of
// 256-row chunks in shared memory, reduced up a tree), converted back to compact-WY
// Householder form by Householder reconstruction, trailing updates and the explicit Q
// as DMMA GEMMs.
#pragma once
#include "common.cuh"

namespace ttb {

constexpr int QR_NB = 32;      // panel width
constexpr int QR_LEAF = 256;   // TSQR leaf chunk rows

struct QRFactors {
  int64_t m = 0, c = 0, kmax = 0;
  DBuf Y;  // m x kmax, ld m: explicit unit-lower-trapezoidal Householder vectors per panel
  DBuf T;  // QR_NB x kmax, ld QR_NB: upper-triangular T of each panel (compact WY)
  std::vector<int64_t> pan_s;  // panel start columns
  std::vector<int> pan_w;      // panel widths (<= QR_NB)
};

// Cluster-resident panel factorisation (panel.cu): m x w panel at A (ld lda) -> explicit Y,
// T (ld ldt) and R in the panel's top w x w block.  Returns false when m exceeds what one
// 16-CTA cluster holds in registers (8192 rows at w <= 32, 16384 rows at w <= 16).
bool panel_qr_cluster(tt_ctx ctx, double* A, int64_t lda, int64_t m, int w, double* Y, int64_t ldy, double* T,
                      int64_t ldt);
int panel_cluster_max_rows(int w);

// In-place QR of the m x c column-major matrix A: on exit the upper trapezoid of
// A[0:kmax, 0:c] holds R (kmax = min(m, c)); the strict lower part is garbage.
void geqrf(tt_ctx ctx, double* A, int64_t lda, int64_t m, int64_t c, QRFactors& f);
// Explicit Q (m x kmax, ld ldq) with orthonormal columns, A = Q R.
void orgqr(tt_ctx ctx, const QRFactors& f, double* Q, int64_t ldq);
// B (m x nb, ld ldb) <- H B with H = H_0 H_1 ... H_{kmax-1} the full m x m orthogonal factor
// (so Q X = H [X; 0]); compact-WY panels applied last to first, 3 DMMA GEMMs each.
void ormqr_left(tt_ctx ctx, const QRFactors& f, double* B, int64_t ldb, int64_t nb);
// R (kmax x c, ld ldr) = upper trapezoid of A with explicit zeros below.
void copy_upper(tt_ctx ctx, const double* A, int64_t lda, int64_t rows, int64_t cols, double* R, int64_t ldr);

// Unblocked Householder QR with column pivoting of the m x c matrix Y (in place, column-
// major, one CTA, LAPACK dlaqp2 norms with exact recomputation), stopping as soon as the
// Frobenius mass of the trailing block drops to stop2 or after kcap steps.
// On exit: *k_done steps, Householder vectors below the diagonal of Y[:, 0:k], R_1 in
// rows 0..k-1 (permuted column order), perm[j] = original column of position j,
// *e2 = exact ||R_22||_F^2 of the trailing block.
struct QRCPState {
  int64_t m = 0, c = 0;
  DBuf tau;    // c
  DBuf norms;  // 2c: current and reference column norms^2
  IBuf perm;   // c
  DBuf scalars;  // [k_done, e2] as doubles
  int k = 0;
  double e2 = 0.0;
  int cluster = -1;  // -1 undecided, 1 cluster-resident path, 0 single-CTA path
};
// m x c fits the distributed shared memory of one <= 16-CTA cluster
bool qrcp_cluster_fits(int64_t m, int64_t c);
// out[:, perm[j]] = in[:, j] (undo a column pivoting)
void unpermute_cols(tt_ctx ctx, const double* in, int64_t ldi, int64_t rows, int64_t c, const int* perm, double* out,
                    int64_t ldo);
// One launch of the cluster-resident QRCP (qrcp_cluster.cu); false if the matrix does not fit.
bool qrcp_cluster_run(tt_ctx ctx, double* Y, int64_t ldy, int64_t m, int64_t c, int k_start, double stop2, int kcap,
                      double* tau, int* perm2c, double* scalars);
// Grid-cooperative QRCP (qrcp_grid.cu) for matrices beyond one cluster; same layout and stopping
// test as the single-CTA kernel; norms (2c) and perm live in global memory.  False if the
// cooperative launch is not possible.
bool qrcp_grid_run(tt_ctx ctx, double* Y, int64_t ldy, int64_t m, int64_t c, int k_start, double stop2, int kcap,
                   double* tau, double* norms, int* perm, double* scalars);
void qrcp_init(tt_ctx ctx, QRCPState& st, double* Y, int64_t ldy, int64_t m, int64_t c);
void qrcp_run(tt_ctx ctx, QRCPState& st, double* Y, int64_t ldy, double stop2, int kcap);
// target (m x nc) <- H_0 H_1 ... H_{k-1} target, reflectors of a QRCP (unblocked).
void apply_reflectors_left(tt_ctx ctx, const double* Y, int64_t ldy, const double* tau, int64_t m, int k,
                           double* target, int64_t ldt, int64_t nc);

}  // namespace ttb
