// Batched TT-rounding of uniformly shaped TT-sums (batch_round.cu).
#pragma once
#include <string>
#include <vector>

#include "round.cuh"

namespace ttb {

// All items share d, n, K and the term ranks; d >= 2; formal ranks <= 64; K <= 16.
bool batch_uniform_supported(int B, const std::vector<SumInput>& items, std::string* why);
// out[b] = TT-round(items[b]) for every b (library-owned tensors sharing one arena per wave);
// ranks_out (host, B*(d+1)) optional.  Throws ttb::Error.
void round_batch_uniform(tt_ctx ctx, const std::vector<SumInput>& items, const tt_round_opts& o, tt_tensor* out,
                         int64_t* ranks_out);

}  // namespace ttb
