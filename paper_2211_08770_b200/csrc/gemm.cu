// FP64 DMMA GEMM.  64x64 CTA tile, BK = 16, 4 warps each owning a 32x32 sub-tile made of
// 4x4 m8n8k4 DMMA fragments; operands staged through shared memory (double-buffered,
// register prefetch of the next K tile).  Shared rows padded to 68 doubles so the
// half-warp fragment loads (4 k-rows x 4 consecutive doubles) hit 32 distinct banks.
#include <algorithm>

#include "gemm.cuh"

namespace ttb {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, THREADS = 128, LDS = BM + 4;
constexpr int MAXP = 40;

struct Prob {
  const double* A;
  const double* B;
  double* C;
  double* Cpart;  // split-K partials (splits x M x N) or null
  int64_t lda, ldb, ldc, ldc_hi, ncol_split;
  int M, N, K;
  int kchunk, tiles_m, tiles_n, tile_begin;
  double alpha, beta;
};

struct Batch {
  Prob p[MAXP];
  int nprob;
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(THREADS) gemm_kernel(const __grid_constant__ Batch bt) {
  int bid = blockIdx.x;
  int pi = 0;
  while (pi + 1 < bt.nprob && bid >= bt.p[pi + 1].tile_begin) ++pi;
  const Prob& P = bt.p[pi];
  int t = bid - P.tile_begin;
  const int tps = P.tiles_m * P.tiles_n;
  const int split = t / tps;
  t -= split * tps;
  const int m0 = (t % P.tiles_m) * BM, n0 = (t / P.tiles_m) * BN;
  const int kbeg = split * P.kchunk;
  const int kend = min(P.K, kbeg + P.kchunk);

  __shared__ __align__(16) double As[2][BK][LDS];
  __shared__ __align__(16) double Bs[2][BK][LDS];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tg = lane & 3;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[8], rb[8];
  auto load_tile = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int idx = tid + q * THREADS;
      int ml, kl;
      if (!TA) { ml = idx & 63; kl = idx >> 6; } else { kl = idx & 15; ml = idx >> 4; }
      int m = m0 + ml, k = k0 + kl;
      double v = 0.0;
      if (m < P.M && k < kend) v = TA ? P.A[(int64_t)k + (int64_t)m * P.lda] : P.A[(int64_t)m + (int64_t)k * P.lda];
      ra[q] = v;
      int nl, kb;
      if (!TB) { kb = idx & 15; nl = idx >> 4; } else { nl = idx & 63; kb = idx >> 6; }
      int n = n0 + nl, kk = k0 + kb;
      double w = 0.0;
      if (n < P.N && kk < kend) w = TB ? P.B[(int64_t)n + (int64_t)kk * P.ldb] : P.B[(int64_t)kk + (int64_t)n * P.ldb];
      rb[q] = w;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      int idx = tid + q * THREADS;
      int ml, kl;
      if (!TA) { ml = idx & 63; kl = idx >> 6; } else { kl = idx & 15; ml = idx >> 4; }
      As[buf][kl][ml] = ra[q];
      int nl, kb;
      if (!TB) { kb = idx & 15; nl = idx >> 4; } else { nl = idx & 63; kb = idx >> 6; }
      Bs[buf][kb][nl] = rb[q];
    }
  };

  const int nk = (kend > kbeg) ? (kend - kbeg + BK - 1) / BK : 0;
  if (nk > 0) {
    load_tile(kbeg);
    store_tile(0);
    __syncthreads();
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_tile(kbeg + (kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][kk + tg][wm + i * 8 + g];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][kk + tg][wn + j * 8 + g];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (kt + 1 < nk) {
      store_tile(buf ^ 1);
    }
    __syncthreads();
  }

  // epilogue
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + wm + i * 8 + g;
    if (row >= P.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = n0 + wn + j * 8 + 2 * tg + e;
        if (col >= P.N) continue;
        const double v = acc[i][j][e];
        if (P.Cpart) {
          P.Cpart[((int64_t)split * P.N + col) * P.M + row] = v;
        } else {
          int64_t addr = P.ncol_split > 0 ? (col / P.ncol_split) * P.ldc_hi + (col % P.ncol_split) * P.ldc
                                          : (int64_t)col * P.ldc;
          addr += row;
          double o = P.alpha * v;
          if (P.beta != 0.0) o += P.beta * P.C[addr];
          P.C[addr] = o;
        }
      }
    }
  }
}

__global__ void splitk_reduce_kernel(const double* __restrict__ part, int splits, int M, int N, double* C,
                                     int64_t ldc, int64_t ncol_split, int64_t ldc_hi, double alpha,
                                     double beta) {
  const int64_t total = (int64_t)M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(idx % M), col = (int)(idx / M);
    double s = 0.0;
    for (int q = 0; q < splits; ++q) s += part[(int64_t)q * total + idx];  // fixed order
    int64_t addr = ncol_split > 0 ? (col / ncol_split) * ldc_hi + (col % ncol_split) * ldc : (int64_t)col * ldc;
    addr += row;
    double o = alpha * s;
    if (beta != 0.0) o += beta * C[addr];
    C[addr] = o;
  }
}

void launch_batch(tt_ctx ctx, Batch& b, int total_tiles, bool ta, bool tb) {
  if (total_tiles <= 0) return;
  dim3 grid(total_tiles), block(THREADS);
  double fl = 0.0, by = 0.0;
  for (int i = 0; i < b.nprob; ++i) {
    const Prob& p = b.p[i];
    fl += 2.0 * p.M * p.N * (double)p.K;
    by += 8.0 * ((double)p.M * p.K + (double)p.K * p.N + (p.beta != 0.0 ? 2.0 : 1.0) * (double)p.M * p.N);
  }
  if (!ta && !tb) TTB_RUN(ctx, "gemm_dmma", fl, by, gemm_kernel<false, false><<<grid, block, 0, ctx->stream>>>(b));
  else if (ta && !tb) TTB_RUN(ctx, "gemm_dmma", fl, by, gemm_kernel<true, false><<<grid, block, 0, ctx->stream>>>(b));
  else if (!ta && tb) TTB_RUN(ctx, "gemm_dmma", fl, by, gemm_kernel<false, true><<<grid, block, 0, ctx->stream>>>(b));
  else TTB_RUN(ctx, "gemm_dmma", fl, by, gemm_kernel<true, true><<<grid, block, 0, ctx->stream>>>(b));
}

Prob make_prob(const GemmDesc& g) {
  Prob p{};
  p.A = g.A; p.B = g.B; p.C = g.C; p.Cpart = nullptr;
  p.lda = g.lda; p.ldb = g.ldb; p.ldc = g.ldc; p.ldc_hi = g.ldc_hi; p.ncol_split = g.ncol_split;
  p.M = (int)g.M; p.N = (int)g.N; p.K = (int)g.K;
  p.kchunk = (int)std::max<int64_t>(g.K, 1);
  p.tiles_m = (int)ceil_div(g.M, BM);
  p.tiles_n = (int)ceil_div(g.N, BN);
  p.alpha = g.alpha; p.beta = g.beta;
  return p;
}

// C = beta C (K == 0 case)
__global__ void scale_kernel(int M, int N, double* C, int64_t ldc, int64_t ncol_split, int64_t ldc_hi, double beta) {
  const int64_t total = (int64_t)M * N;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(idx % M), col = (int)(idx / M);
    int64_t addr = (ncol_split > 0 ? (col / ncol_split) * ldc_hi + (col % ncol_split) * ldc : (int64_t)col * ldc) + row;
    C[addr] = beta == 0.0 ? 0.0 : beta * C[addr];
  }
}

}  // namespace

void gemm(tt_ctx ctx, const GemmDesc& g) {
  if (g.M <= 0 || g.N <= 0) return;
  if (g.K <= 0) {
    int blocks = (int)std::min<int64_t>(ceil_div(g.M * g.N, 256), 4096);
    TTB_RUN(ctx, "aux", 0, 16.0 * g.M * g.N,
            scale_kernel<<<blocks, 256, 0, ctx->stream>>>((int)g.M, (int)g.N, g.C, g.ldc, g.ncol_split, g.ldc_hi, g.beta));
    return;
  }
  Batch b{};
  b.nprob = 1;
  Prob p = make_prob(g);
  const int tiles = p.tiles_m * p.tiles_n;
  int splits = 1;
  if (tiles < ctx->num_sms && g.K >= 512) {
    splits = (int)std::min<int64_t>(ceil_div(2 * ctx->num_sms, tiles), g.K / 256);
    splits = std::max(1, std::min(splits, 64));
  }
  DBuf part;
  if (splits > 1) {
    int64_t kc = ceil_div(g.K, splits);
    kc = ceil_div(kc, BK) * BK;
    splits = (int)ceil_div(g.K, kc);
    p.kchunk = (int)kc;
    part.alloc(ctx, (size_t)splits * g.M * g.N);
    p.Cpart = part.p;
  }
  p.tile_begin = 0;
  b.p[0] = p;
  launch_batch(ctx, b, tiles * splits, g.ta, g.tb);
  if (splits > 1) {
    int blocks = (int)std::min<int64_t>(ceil_div(g.M * g.N, 256), 2048);
    TTB_RUN(ctx, "gemm_splitk_reduce", (double)splits * g.M * g.N, 8.0 * (splits + 2.0) * g.M * g.N,
            splitk_reduce_kernel<<<blocks, 256, 0, ctx->stream>>>(part.p, splits, (int)g.M, (int)g.N, g.C, g.ldc,
                                                          g.ncol_split, g.ldc_hi, g.alpha, g.beta));
  }
}

void gemm_grouped(tt_ctx ctx, const std::vector<GemmDesc>& gs) {
  if (gs.empty()) return;
  const bool ta = gs[0].ta, tb = gs[0].tb;
  Batch b{};
  int tiles = 0;
  b.nprob = 0;
  for (const GemmDesc& g : gs) {
    if (g.ta != ta || g.tb != tb) fail(TT_EINVAL, "gemm_grouped: mixed transposes");
    if (g.M <= 0 || g.N <= 0) continue;
    if (g.K <= 0) { gemm(ctx, g); continue; }
    if (b.nprob == MAXP) {
      launch_batch(ctx, b, tiles, ta, tb);
      b.nprob = 0;
      tiles = 0;
    }
    Prob p = make_prob(g);
    p.tile_begin = tiles;
    tiles += p.tiles_m * p.tiles_n;
    b.p[b.nprob++] = p;
  }
  if (b.nprob > 0) launch_batch(ctx, b, tiles, ta, tb);
}

}  // namespace ttb
