// Batched TT-rounding of uniformly shaped TT-sums (batch_round.cu).
#pragma once
#include <string>
#include <vector>

#include "round.cuh"

namespace ttb {

// B items sharing d, n, K and the term ranks.  tab[(b*K + l)*d + k] = device pointer to core k
// of term l of item b; coef / norm [b*K + l] (norm NaN = unknown, computed on the device).
struct BatchDesc {
  int B = 0, K = 0, d = 0;
  std::vector<int64_t> n;
  std::vector<std::vector<int64_t>> r;  // r[l][0..d]
  std::vector<const double*> tab;
  std::vector<double> coef, norm;
};

// Results: item b's core k at core[b*d + k] (inside arenas[w] of its wave), ranks[b*(d+1) + k].
struct BatchOut {
  int B = 0, d = 0;
  std::vector<int64_t> n;
  std::vector<int64_t> ranks;
  std::vector<double*> core;
  std::vector<double> norm, tau, scale;  // ||x||, the truncation threshold and s(x) per item
  std::vector<void*> arenas;   // one exact-size allocation per wave (caller frees)
  std::vector<int64_t> arena_size;  // doubles in each arena (items in order, cores in order)
  std::vector<int> wave_first; // first item of each wave
};

// d >= 2, every formal rank R_k <= 64, K <= 16.
bool batch_shape_supported(int d, int K, const std::vector<std::vector<int64_t>>& r, std::string* why);
bool batch_uniform_supported(int B, const std::vector<SumInput>& items, std::string* why);
void run_batch(tt_ctx ctx, const BatchDesc& in, const tt_round_opts& o, BatchOut& res);
// Fill in.B/K/d/n/r from the C-ABI shape arguments of tt_round_batch_strided / _host, validated
// (TT_ESHAPE for bad ranks or modes, TT_ENOTSUP outside batch_shape_supported).
void batch_desc_shape(BatchDesc& in, int B, int K, int d, const int64_t* n, const int64_t* r);
// host_pipe.cu: release the context's host-pipeline streams and staging buffers.
void host_pipe_release(tt_ctx ctx);
// out[b] = TT-round(items[b]) as library tensors (sharing one refcounted arena per wave).
// info (optional, B entries): ||x||, s(x) and tau of each item.
void round_batch_uniform(tt_ctx ctx, const std::vector<SumInput>& items, const tt_round_opts& o, tt_tensor* out,
                         int64_t* ranks_out, tt_round_info* info = nullptr);

}  // namespace ttb
