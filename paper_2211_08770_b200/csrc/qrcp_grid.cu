// Householder QR with column pivoting over the whole GPU (cooperative launch, grid-wide
// synchronisation), for right-to-left panels too large for one cluster's shared memory (C3:
// 1280 x 1000, C5: 480 x 3131).  Same arithmetic, stopping test and output layout as the
// single-CTA qrcp_kernel (qr.cu): LAPACK dlarfg reflectors, column norms downdated with exact
// recomputation when cancellation sets in and before any decision near the threshold, columns
// physically swapped into pivot order, perm[j] = original column at position j.
//
// Per step two grid barriers: (1) every warp applies reflector s-1 to its columns (columns are
// dealt round-robin over all warps of the grid), downdates their norms and contributes to its
// CTA's candidate (mass, best norm, position); (2) every CTA reduces the G candidates in the same
// fixed order (identical decisions everywhere), CTA 0 swaps the pivot column into place and forms
// reflector s.
#include <cooperative_groups.h>

#include <algorithm>

#include "qr.cuh"

namespace cg = cooperative_groups;

namespace ttb {

namespace {

constexpr int QG_T = 256;
constexpr int QG_W = QG_T / 32;

struct QGCand {
  double mass, val;
  int pos, pad;
};

__device__ __forceinline__ bool qg_better(double v, int p, double bv, int bp) { return v > bv || (v == bv && p < bp); }

// CTA-wide reduction of (mass, best) -> cand[blockIdx.x]
__device__ void qg_publish(double mass, double bv, int bp, QGCand* cand, QGCand* wbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  mass = warp_sum(mass);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int op = __shfl_xor_sync(0xffffffffu, bp, o);
    if (qg_better(ov, op, bv, bp)) { bv = ov; bp = op; }
  }
  if (lane == 0) wbuf[warp] = QGCand{mass, bv, bp, 0};
  __syncthreads();
  if (warp == 0) {
    QGCand cd = lane < QG_W ? wbuf[lane] : QGCand{0.0, -1.0, 0x7fffffff, 0};
    double ms = warp_sum(cd.mass), v = cd.val;
    int p = cd.pos;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int op = __shfl_xor_sync(0xffffffffu, p, o);
      if (qg_better(ov, op, v, p)) { v = ov; p = op; }
    }
    if (lane == 0) cand[blockIdx.x] = QGCand{ms, v, p, 0};
  }
  __syncthreads();
}

// Every CTA: total mass and global pivot from the G candidates.  Warp 0 reads them in parallel
// (lane q: candidates q, q + 32, ...) and reduces in a fixed order (deterministic; identical in
// every CTA); the result is broadcast through shared memory.
__device__ void qg_decide(const QGCand* cand, double& tot, int& gp, QGCand* wbuf) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
    double ms = 0.0, v = -1.0;
    int p = 0x7fffffff;
    for (int q = lane; q < (int)gridDim.x; q += 32) {
      const QGCand cd = cand[q];
      ms += cd.mass;
      if (qg_better(cd.val, cd.pos, v, p)) { v = cd.val; p = cd.pos; }
    }
    ms = warp_sum(ms);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int op = __shfl_xor_sync(0xffffffffu, p, o);
      if (qg_better(ov, op, v, p)) { v = ov; p = op; }
    }
    if (lane == 0) wbuf[QG_W] = QGCand{ms, v, p, 0};
  }
  __syncthreads();
  tot = wbuf[QG_W].mass;
  gp = wbuf[QG_W].pos;
  __syncthreads();
}

__global__ void __launch_bounds__(QG_T) qrcp_grid_kernel(double* Y, int64_t ldy, int m, int c, int k_start, double stop2,
                                                         int kcap, double* tau, double* norms, int* perm,
                                                         double* scalars, QGCand* cand) {
  cg::grid_group grid = cg::this_grid();
  __shared__ QGCand wbuf[QG_W + 1];
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gw = blockIdx.x * QG_W + warp, nwg = gridDim.x * QG_W;
  double* nrm = norms;
  double* nrm0 = norms + c;
  const int kmax = min(min(m, c), kcap);
  // exact norms of the trailing columns (rows >= s) + this CTA's candidate
  auto recompute = [&](int s) {
    double mass = 0.0, bv = -1.0;
    int bp = 0x7fffffff;
    for (int j = s + gw; j < c; j += nwg) {
      double q = 0.0;
      for (int i = s + lane; i < m; i += 32) { const double v = Y[i + (int64_t)j * ldy]; q += v * v; }
      q = warp_sum(q);
      if (lane == 0) { nrm[j] = q; nrm0[j] = q; }
      mass += (lane == 0) ? q : 0.0;
      if (lane == 0 && qg_better(q, j, bv, bp)) { bv = q; bp = j; }
    }
    qg_publish(mass, bv, bp, cand, wbuf);
  };
  if (k_start == 0)
    for (int j = blockIdx.x * QG_T + tid; j < c; j += gridDim.x * QG_T) perm[j] = j;
  recompute(k_start);
  grid.sync();
  int s = k_start;
#pragma unroll 1
  for (; s < kmax; ++s) {
    double tot;
    int gp;
    qg_decide(cand, tot, gp, wbuf);
    if (tot <= 4.0 * stop2 && s > k_start) {  // near the threshold: exact norms before deciding
      grid.sync();                              // every CTA has read the candidates
      recompute(s);
      grid.sync();
      qg_decide(cand, tot, gp, wbuf);
    }
    if (tot <= stop2 || gp >= c) break;
    // CTA 0: pivot column into position s, reflector of column s (rows s..m-1)
    if (blockIdx.x == 0) {
      if (gp != s) {
        for (int i = tid; i < m; i += QG_T) {
          const double a = Y[i + (int64_t)s * ldy];
          Y[i + (int64_t)s * ldy] = Y[i + (int64_t)gp * ldy];
          Y[i + (int64_t)gp * ldy] = a;
        }
        if (tid == 0) {
          double t = nrm[s]; nrm[s] = nrm[gp]; nrm[gp] = t;
          t = nrm0[s]; nrm0[s] = nrm0[gp]; nrm0[gp] = t;
          const int q = perm[s]; perm[s] = perm[gp]; perm[gp] = q;
        }
        __syncthreads();
      }
      double pp = 0.0;
      for (int i = s + 1 + tid; i < m; i += QG_T) { const double v = Y[i + (int64_t)s * ldy]; pp += v * v; }
      const double sigma = block_sum(pp, red);
      const double alpha = Y[s + (int64_t)s * ldy];
      double t = 0.0, beta = alpha, scal = 0.0;
      if (sigma != 0.0) {
        const double nr = sqrt(alpha * alpha + sigma);
        beta = alpha >= 0.0 ? -nr : nr;
        t = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      for (int i = s + 1 + tid; i < m; i += QG_T) Y[i + (int64_t)s * ldy] *= scal;
      __syncthreads();
      if (tid == 0) { Y[s + (int64_t)s * ldy] = beta; tau[s] = t; }
    }
    grid.sync();
    // every warp: apply reflector s to its columns j > s, downdate norms, next candidate
    const double t = tau[s];
    const double* v = Y + (int64_t)s * ldy;
    double mass = 0.0, bv = -1.0;
    int bp = 0x7fffffff;
    for (int j = s + 1 + gw; j < c; j += nwg) {
      double* col = Y + (int64_t)j * ldy;
      if (t != 0.0) {
        double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;  // four independent chains in flight
        int i = s + 1 + lane;
        for (; i + 96 < m; i += 128) {
          q0 += v[i] * col[i];
          q1 += v[i + 32] * col[i + 32];
          q2 += v[i + 64] * col[i + 64];
          q3 += v[i + 96] * col[i + 96];
        }
        for (; i < m; i += 32) q0 += v[i] * col[i];
        double q = warp_sum((q0 + q1) + (q2 + q3));
        q = t * (q + col[s]);
        for (i = s + 1 + lane; i + 96 < m; i += 128) {
          const double a0 = col[i], a1 = col[i + 32], a2 = col[i + 64], a3 = col[i + 96];
          col[i] = a0 - q * v[i];
          col[i + 32] = a1 - q * v[i + 32];
          col[i + 64] = a2 - q * v[i + 64];
          col[i + 96] = a3 - q * v[i + 96];
        }
        for (; i < m; i += 32) col[i] -= q * v[i];
        __syncwarp();
        if (lane == 0) col[s] -= q;
        __syncwarp();
      }
      const double rs = col[s];
      double nn = nrm[j] - rs * rs;
      if (!(nn > 1e-8 * nrm0[j])) {
        double q = 0.0;
        for (int i = s + 1 + lane; i < m; i += 32) { const double x = col[i]; q += x * x; }
        nn = warp_sum(q);
        if (lane == 0) nrm0[j] = nn;
      }
      __syncwarp();
      if (lane == 0) nrm[j] = nn;
      if (lane == 0) {
        mass += nn;
        if (qg_better(nn, j, bv, bp)) { bv = nn; bp = j; }
      }
    }
    qg_publish(mass, bv, bp, cand, wbuf);
    grid.sync();
  }
  // exact trailing mass (rows >= s of the unpivoted columns)
  double part = 0.0;
  for (int j = s + gw; j < c; j += nwg)
    for (int i = s + lane; i < m; i += 32) { const double x = Y[i + (int64_t)j * ldy]; part += x * x; }
  qg_publish(part, -1.0, 0x7fffffff, cand, wbuf);
  grid.sync();
  if (blockIdx.x == 0 && tid == 0) {
    double e2 = 0.0;
    for (int q = 0; q < (int)gridDim.x; ++q) e2 += cand[q].mass;
    scalars[0] = (double)s;
    scalars[1] = e2;
  }
}

}  // namespace

bool qrcp_grid_run(tt_ctx ctx, double* Y, int64_t ldy, int64_t m, int64_t c, int k_start, double stop2, int kcap,
                   double* tau, double* norms, int* perm, double* scalars) {
  int per_sm = 0;
  TTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrcp_grid_kernel, QG_T, 0));
  if (per_sm < 1) return false;
  const int G = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->num_sms * per_sm,
                                                            std::min<int64_t>(ctx->num_sms, ceil_div(c, QG_W))));
  DBuf cand(ctx, (size_t)G * 3);
  QGCand* cp = reinterpret_cast<QGCand*>(cand.p);
  int mi = (int)m, ci = (int)c;
  void* args[] = {&Y, &ldy, &mi, &ci, &k_start, &stop2, &kcap, &tau, &norms, &perm, &scalars, &cp};
  TTB_RUN(ctx, "qrcp_grid", 0, 16.0 * m * c,
          TTB_CUDA(cudaLaunchCooperativeKernel((const void*)qrcp_grid_kernel, dim3(G), dim3(QG_T), args, 0,
                                               ctx->stream)));
  return true;
}

}  // namespace ttb
