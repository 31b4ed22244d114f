// TT-dot Gram matrix of m equally shaped TT-vectors, pair-tiled (Alg. 5 lines 2-6, Eq. (3):
// G(i,j) = <a_i, a_j>; PAPER.md:19 dot through the core contraction).
//
// One CTA per tile of TI x TJ pairs (i in I, j in J, tiles of the lower triangle).  Per pair the
// left-to-right recursion W_k = sum_s X^(i)_k(s)^T W_{k-1} X^(j)_k(s) runs with every pair's
// W and the mode slice U = W X^(j)(s) in shared memory and the new W accumulated in registers:
// per slice s the tile's tensors' slices X(s) are staged once and reused by all pairs of the
// tile.  Each thread owns 4 x 4 micro-tiles (FP64 FMA, register blocked).  Summation order is
// fixed (deterministic).
#include <cuda_pipeline.h>

#include <algorithm>

#include "gram.cuh"

namespace ttb {

namespace {

constexpr int GT_I = 2, GT_J = 2, GT_P = GT_I * GT_J;  // pairs per tile
constexpr int GT_MAXD = 128;

// One CTA's work: pairs (i, j) with i in [i0, i0 + GT_I), j in [j0, j0 + GT_J).  mode 0: write
// G(i, j) and G(j, i) for i >= j (symmetric m x m output); mode 1: write the pairs with
// i < ilim, j < jlim to out[off + (i - bi0) * bj + (j - bj0)] (packed pair block).
struct GramTile {
  int i0, j0, ilim, jlim, bi0, bj0, bj, mode;
  int64_t off;
};

struct GramShape {
  int d;
  int n[GT_MAXD];
  int r[GT_MAXD + 1];
};

__host__ __device__ inline int ceil4(int x) { return (x + 3) & ~3; }

template <int GT_T>  // threads per CTA; one V micro-tile per thread
__global__ void __launch_bounds__(GT_T) gram_tile_kernel(const double* const* __restrict__ cores, GramShape sh, int m,
                                                          int nbj, const GramTile* __restrict__ tiles, int RP,
                                                          int S, int PS, double* __restrict__ G) {
  extern __shared__ __align__(16) double gsm[];
  // smem blocks of PS doubles (per pair / per staged tensor), rows of stride S >= RP: padded so
  // the 4x4 micro-tile accesses of a warp spread over the banks
  const int RR = PS;
  double* W = gsm;                 // [p][c][a]  (column-major W: W[p][c * RP + a] = W(a, c))
  double* U = W + GT_P * RR;       // [p][a][c'] (row-major)
  double* XB = U + GT_P * RR;      // 2 buffers x [t][a][a'] (row-major slices X(a, s, a')), I then J
  const double** rowsrc = reinterpret_cast<const double**>(XB + 2 * (GT_I + GT_J) * RR);  // <= 4 * 32 rows
  int* rowdst = reinterpret_cast<int*>(rowsrc + (GT_I + GT_J) * 32);
  const int tid = threadIdx.x;
  const GramTile tl = tiles[blockIdx.x];
  const int i0 = tl.i0, j0 = tl.j0;
  const int d = sh.d;
  for (int idx = tid; idx < GT_P * RR; idx += GT_T) W[idx] = (idx % RR == 0) ? 1.0 : 0.0;  // W_0 = 1 (1 x 1)
#pragma unroll 1
  for (int k = 0; k < d; ++k) {
    const int n = sh.n[k], R0 = sh.r[k], R1 = sh.r[k + 1];
    const int T0 = ceil4(R0) / 4, T1 = ceil4(R1) / 4;
    const int nU = GT_P * T0 * T1, nV = GT_P * T1 * T1;
    for (int idx = tid; idx < 2 * (GT_I + GT_J) * RR; idx += GT_T) XB[idx] = 0.0;  // pads stay zero
    double acc[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) acc[e] = 0.0;
    __syncthreads();
    // slices X(:, s, :) of the tile's tensors, staged asynchronously one slice ahead
    // slices X(:, s, :) of the tile's tensors, staged asynchronously one slice ahead: 16-byte
    // copies when R1 is even (rows stay 16-byte aligned), per-row source bases tabulated once
    const bool v16 = (R1 & 1) == 0;
    const int cpr = v16 ? R1 / 2 : R1;             // copies per slice row
    const int nrow = (GT_I + GT_J) * R0;
    for (int rid = tid; rid < nrow; rid += GT_T) {
      const int t = rid / R0, a = rid - t * R0;
      int tens = t < GT_I ? i0 + t : j0 + (t - GT_I);
      if (tens >= m) tens = m - 1;  // padding tensor: its pairs are never written
      rowsrc[rid] = cores[(int64_t)tens * d + k] + (int64_t)a * n * R1;
      rowdst[rid] = t * RR + a * S;
    }
    __syncthreads();
    auto stage = [&](int s, double* buf) {
      for (int idx = tid; idx < nrow * cpr; idx += GT_T) {
        const int rid = idx / cpr, c = idx - rid * cpr;
        const double* src = rowsrc[rid] + (int64_t)s * R1;
        double* dst = buf + rowdst[rid];
        if (v16) __pipeline_memcpy_async(dst + 2 * c, src + 2 * c, 2 * sizeof(double));
        else __pipeline_memcpy_async(dst + c, src + c, sizeof(double));
      }
      __pipeline_commit();
    };
    stage(0, XB);
#pragma unroll 1
    for (int s = 0; s < n; ++s) {
      double* XI = XB + (s & 1) * (GT_I + GT_J) * RR;
      double* XJ = XI + GT_I * RR;
      __pipeline_wait_prior(0);
      __syncthreads();  // slice s visible; V of slice s-1 done (its buffer may be refilled)
      if (s + 1 < n) stage(s + 1, XB + ((s + 1) & 1) * (GT_I + GT_J) * RR);
      // U_p = W_p X^(j_p)(s): (R0 x R0) x (R0 x R1)
      for (int u = tid; u < nU; u += GT_T) {
        const int p = u / (T0 * T1), rem = u % (T0 * T1), ta = rem / T1, tc = rem % T1;
        const double* Wp = W + p * RR;
        const double* Xj = XJ + (p % GT_J) * RR;
        double c4[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) c4[x][y] = 0.0;
#pragma unroll 2
        for (int c = 0; c < R0; ++c) {
          const double2 w01 = *reinterpret_cast<const double2*>(Wp + c * S + 4 * ta);
          const double2 w23 = *reinterpret_cast<const double2*>(Wp + c * S + 4 * ta + 2);
          const double2 x01 = *reinterpret_cast<const double2*>(Xj + c * S + 4 * tc);
          const double2 x23 = *reinterpret_cast<const double2*>(Xj + c * S + 4 * tc + 2);
          const double wv[4] = {w01.x, w01.y, w23.x, w23.y}, xv[4] = {x01.x, x01.y, x23.x, x23.y};
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) c4[x][y] += wv[x] * xv[y];
        }
        double* Up = U + p * RR;
#pragma unroll
        for (int x = 0; x < 4; ++x) {
          *reinterpret_cast<double2*>(Up + (4 * ta + x) * S + 4 * tc) = make_double2(c4[x][0], c4[x][1]);
          *reinterpret_cast<double2*>(Up + (4 * ta + x) * S + 4 * tc + 2) = make_double2(c4[x][2], c4[x][3]);
        }
      }
      __syncthreads();
      // V_p += X^(i_p)(s)^T U_p: (R1 x R0) x (R0 x R1), accumulated in registers
      {
        const int v = tid;
        if (v < nV) {
          const int p = v / (T1 * T1), rem = v % (T1 * T1), ta = rem / T1, tc = rem % T1;
          const double* Xi = XI + (p / GT_J) * RR;
          const double* Up = U + p * RR;
#pragma unroll 2
          for (int a = 0; a < R0; ++a) {
            const double2 x01 = *reinterpret_cast<const double2*>(Xi + a * S + 4 * ta);
            const double2 x23 = *reinterpret_cast<const double2*>(Xi + a * S + 4 * ta + 2);
            const double2 u01 = *reinterpret_cast<const double2*>(Up + a * S + 4 * tc);
            const double2 u23 = *reinterpret_cast<const double2*>(Up + a * S + 4 * tc + 2);
            const double xv[4] = {x01.x, x01.y, x23.x, x23.y}, uv[4] = {u01.x, u01.y, u23.x, u23.y};
#pragma unroll
            for (int x = 0; x < 4; ++x)
#pragma unroll
              for (int y = 0; y < 4; ++y) acc[x * 4 + y] += xv[x] * uv[y];
          }
        }
      }
    }
    __syncthreads();
    // W_k (column-major) <- V
    for (int idx = tid; idx < GT_P * RR; idx += GT_T) W[idx] = 0.0;
    __syncthreads();
    {
      const int v = tid;
      if (v < nV) {
        const int p = v / (T1 * T1), rem = v % (T1 * T1), ta = rem / T1, tc = rem % T1;
        double* Wp = W + p * RR;
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) {
            const int a1 = 4 * ta + x, c1 = 4 * tc + y;
            if (a1 < R1 && c1 < R1) Wp[c1 * S + a1] = acc[x * 4 + y];
          }
      }
    }
    __syncthreads();
  }
  if (tid < GT_P) {
    const int i = i0 + tid / GT_J, j = j0 + tid % GT_J;
    const double g = W[tid * RR];
    if (tl.mode == 0) {
      if (i < m && j < m && i >= j) {
        G[(int64_t)i * m + j] = g;
        G[(int64_t)j * m + i] = g;
      }
    } else if (i < tl.ilim && j < tl.jlim) {
      G[tl.off + (int64_t)(i - tl.bi0) * tl.bj + (j - tl.bj0)] = g;
    }
  }
  (void)nbj;
}

}  // namespace

bool gram_tiled_supported(const std::vector<const double*>& cores, int m, int d, const std::vector<int64_t>& n,
                          const std::vector<int64_t>& r) {
  (void)cores;
  if (m < 1 || d < 1 || d > GT_MAXD) return false;
  int rmax = 1;
  for (int k = 0; k <= d; ++k) rmax = std::max<int>(rmax, (int)r[(size_t)k]);
  for (int k = 0; k < d; ++k)
    if (n[(size_t)k] < 1) return false;
  // one V micro-tile per thread: GT_P * (ceil4(R)/4)^2 <= 256 (R <= 32)
  return GT_P * (ceil4(rmax) / 4) * (ceil4(rmax) / 4) <= 256;
}

static void gram_launch(tt_ctx ctx, const std::vector<const double*>& cores, int m, int d,
                        const std::vector<int64_t>& n, const std::vector<int64_t>& r,
                        const std::vector<GramTile>& tiles, double npairs, double* out) {
  GramShape sh{};
  sh.d = d;
  int rmax = 1;
  double flops = 0.0;
  for (int k = 0; k < d; ++k) {
    sh.n[k] = (int)n[(size_t)k];
    const double R0 = (double)r[(size_t)k], R1 = (double)r[(size_t)k + 1];
    flops += 2.0 * (double)n[(size_t)k] * (R0 * R0 * R1 + R0 * R1 * R1);  // per pair
  }
  for (int k = 0; k <= d; ++k) {
    sh.r[k] = (int)r[(size_t)k];
    rmax = std::max<int>(rmax, (int)r[(size_t)k]);
  }
  if (tiles.empty()) return;
  const int RP = ceil4(rmax);
  // row stride / block stride chosen for the fewest shared-memory bank conflicts (offline model)
  const int S = (RP == 8 || RP == 12 || RP == 20 || RP == 24) ? RP + 2 : RP;
  const int PS = S * RP + 2;
  BBuf dt, dc;
  dt.upload(ctx, tiles.data(), tiles.size() * sizeof(GramTile));
  dc.upload(ctx, cores.data(), cores.size() * sizeof(double*));
  const size_t smem = sizeof(double) * (size_t)(2 * GT_P + 2 * (GT_I + GT_J)) * PS +
                      (sizeof(double*) + sizeof(int)) * (GT_I + GT_J) * 32;
  double bytes = 0.0;
  for (int k = 0; k < d; ++k) bytes += 8.0 * (double)m * r[(size_t)k] * n[(size_t)k] * r[(size_t)k + 1];
  const int nv = GT_P * (RP / 4) * (RP / 4);
  const int ntiles = (int)tiles.size();
  const GramTile* tp = static_cast<const GramTile*>(dt.p);
  if (nv <= 128) {
    TTB_CUDA(cudaFuncSetAttribute(gram_tile_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TTB_RUN(ctx, "tt_gram_tiled", flops * npairs, bytes,
            gram_tile_kernel<128><<<ntiles, 128, smem, ctx->stream>>>(static_cast<const double* const*>(dc.p), sh, m,
                                                                        0, tp, RP, S, PS, out));
  } else {
    TTB_CUDA(cudaFuncSetAttribute(gram_tile_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TTB_RUN(ctx, "tt_gram_tiled", flops * npairs, bytes,
            gram_tile_kernel<256><<<ntiles, 256, smem, ctx->stream>>>(static_cast<const double* const*>(dc.p), sh, m,
                                                                        0, tp, RP, S, PS, out));
  }
}

void gram_tiled(tt_ctx ctx, const std::vector<const double*>& cores, int m, int d, const std::vector<int64_t>& n,
                const std::vector<int64_t>& r, double* G_dev) {
  std::vector<GramTile> tiles;
  for (int i0 = 0; i0 < m; i0 += GT_I)
    for (int j0 = 0; j0 < m; j0 += GT_J)
      if (i0 + GT_I - 1 >= j0) tiles.push_back(GramTile{i0, j0, m, m, 0, 0, 0, 0, 0});  // holds a pair i >= j
  gram_launch(ctx, cores, m, d, n, r, tiles, 0.5 * m * (m + 1.0), G_dev);
}

void gram_tiled_blocks(tt_ctx ctx, const std::vector<const double*>& cores, int m, int d,
                       const std::vector<int64_t>& n, const std::vector<int64_t>& r, int nblk, const int32_t* blk,
                       double* packed_dev) {
  std::vector<GramTile> tiles;
  int64_t off = 0;
  double npairs = 0.0;
  for (int b = 0; b < nblk; ++b) {
    const int i0 = blk[4 * b], j0 = blk[4 * b + 1], bi = blk[4 * b + 2], bj = blk[4 * b + 3];
    for (int ti = i0; ti < i0 + bi; ti += GT_I)
      for (int tj = j0; tj < j0 + bj; tj += GT_J) tiles.push_back(GramTile{ti, tj, i0 + bi, j0 + bj, i0, j0, bj, 1, off});
    off += (int64_t)bi * bj;
    npairs += (double)bi * bj;
  }
  gram_launch(ctx, cores, m, d, n, r, tiles, npairs, packed_dev);
}

}  // namespace ttb
