// The six orthogonalization drivers of PAPER.md §2 in lazy-coefficient form.
#pragma once
#include "common.cuh"
#include "round.cuh"

namespace ttb {

// Borrowed single TT (input view or library tensor).
struct TTRef {
  int d = 0;
  std::vector<int64_t> n, r;
  std::vector<const double*> core;
  double norm = NAN;
  static TTRef of(const tt_view& v);
  static TTRef of(tt_tensor t);
};

// <x_p, y_p> for all pairs, returned on the host (synchronises).
std::vector<double> dots_host(tt_ctx ctx, const std::vector<std::pair<const TTRef*, const TTRef*>>& pairs);
void dots_device(tt_ctx ctx, const std::vector<std::pair<const TTRef*, const TTRef*>>& pairs, double* out_dev);

// Host dense helpers (m <= a few hundred).
// Cholesky G = L L^T (row-major m x m); returns -1 or the failing pivot.
int cholesky_host(std::vector<double>& G, int m);
double loo_host(const std::vector<double>& Gq, int m, int k);  // ||I_k - Gq[:k,:k]||_2

tt_status orth_run(tt_ctx ctx, tt_orth_kind kind, int m, const tt_view* a, const tt_orth_opts& o,
                   tt_tensor* q_out, double* R_host, tt_orth_report* rep);

tt_tensor make_canonical(tt_ctx ctx, const std::vector<int64_t>& n, int64_t lin1);

}  // namespace ttb
