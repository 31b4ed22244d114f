// Pair-tiled TT-dot Gram matrix of equally shaped TT-vectors (gram.cu).
#pragma once
#include <vector>

#include "common.cuh"

namespace ttb {

// cores[t*d + k]: core k of tensor t (device); every tensor has modes n[0..d-1], ranks r[0..d].
bool gram_tiled_supported(const std::vector<const double*>& cores, int m, int d, const std::vector<int64_t>& n,
                          const std::vector<int64_t>& r);
// G_dev (m x m row-major, device) = <a_i, a_j>, symmetric; enqueued on the ctx stream.
void gram_tiled(tt_ctx ctx, const std::vector<const double*>& cores, int m, int d, const std::vector<int64_t>& n,
                const std::vector<int64_t>& r, double* G_dev);

// Pair blocks (i0, j0, bi, bj) (blk: 4 ints each): block b's pairs row-major at packed_dev + the
// sizes of the previous blocks (the tt_gram_blocks layout).  rj (optional): rank profile of the
// J-side tensors (the tensors j0..j0+bj-1 of every block) when it differs from the I side's r.
void gram_tiled_blocks(tt_ctx ctx, const std::vector<const double*>& cores, int m, int d,
                       const std::vector<int64_t>& n, const std::vector<int64_t>& r, int nblk, const int32_t* blk,
                       double* packed_dev, const std::vector<int64_t>* rj = nullptr);

}  // namespace ttb
