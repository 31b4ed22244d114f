// TT-rounding of a TT-sum.
#pragma once
#include "common.cuh"

namespace ttb {

// A borrowed TT-sum x = sum_l coef[l] y_l.
struct SumInput {
  int d = 0;
  std::vector<int64_t> n;
  std::vector<std::vector<int64_t>> r;            // r[l][0..d]
  std::vector<std::vector<const double*>> core;   // core[l][0..d-1]
  std::vector<double> coef;
  std::vector<double> norm;                       // ||y_l|| or NaN
  int K() const { return (int)coef.size(); }
  void add(const tt_view& v, double c);           // validates against the first term
  void add_tensor(tt_tensor t, double c);
};

struct RoundStats {
  int64_t calls = 0;
  int64_t qrcp_steps = 0;
  int64_t resumes = 0;
};

tt_tensor round_sum(tt_ctx ctx, const SumInput& in, const tt_round_opts& o, tt_round_info* info);
// ||x|| of the sum through the right-to-left QR sweep (no truncation).
double sweep_norm(tt_ctx ctx, const SumInput& in);
// materialised TT-sum (block concatenation)
tt_tensor materialise_sum(tt_ctx ctx, const SumInput& in);
tt_round_opts default_round_opts();

}  // namespace ttb
