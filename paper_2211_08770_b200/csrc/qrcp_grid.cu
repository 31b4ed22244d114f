// Householder QR with column pivoting over the whole GPU (cooperative launch, grid-wide
// synchronisation), for right-to-left panels too large for one cluster's shared memory (C3:
// 1280 x 1000, 14000 x 440; C5: 480 x 3131).  Same arithmetic, stopping test and output layout
// as the single-CTA qrcp_kernel (qr.cu): LAPACK dlarfg reflectors, pivot = largest remaining
// column norm (ties: lowest position), stop once the trailing Frobenius mass drops to stop2,
// columns in pivot order on exit, perm[j] = original column at position j.
//
// Work decomposition (the column-per-warp sweep is latency bound: one warp streams a whole
// 14000-row column twice per step).  The panel is cut into RC row chunks of CH rows; a work item
// is one (column, chunk) pair, dealt round-robin over every warp of the grid.  Per step:
//   top     every CTA reduces the exact column masses n1[j] (rows >= s) of the unprocessed
//           columns to (total mass, pivot p) -- identical decisions everywhere -- and forms the
//           reflector of column p redundantly (alpha = Y[s,p], sigma = n2[p] = mass of rows > s,
//           kept exactly, never by subtraction).
//   phase 1 each pair: partial of w_j = v^T Y[s:, j] (v read from the raw pivot column, scaled on
//           the fly).
//   sync
//   phase 2 each pair: w_j = the chunk partials summed in chunk order (by every chunk of column
//           j), Y[s:, j] -= tau w_j v, then the partial masses of rows >= s+1 and >= s+2
//           of the updated values (no downdating: exact norms every step at no extra traffic);
//           the last chunk for column j writes n1[j], n2[j].
//   sync
// Columns are not swapped during the sweep (the pivot column is scaled into its reflector one
// step later, when nobody reads it any more); one gather at the end puts them in pivot order.
// Panels up to ~80 MB stay in L2 across steps.  All reductions run in a fixed order
// (deterministic, run to run).
#include <cooperative_groups.h>
#include <cuda/atomic>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "qr.cuh"

namespace cg = cooperative_groups;

namespace ttb {

namespace {

constexpr int QG_T = 256;
constexpr int QG_W = QG_T / 32;

struct QGArgs {
  double* Y;
  int64_t ldy;
  int m, c, k_start, kcap;
  double stop2;
  double* tau;
  int* perm;
  double* scalars;
  int CH, RC;  // rows per chunk, chunks
  double* wpart;   // RC x c
  double* n1part;  // RC x c
  double* n2part;  // RC x c
  double* w;       // c
  double* n1;      // c: mass of rows >= s of column j
  double* n2;      // c: mass of rows >= s+1
  int* cnt;        // c (counters, zero on entry and on exit)
  double* tmp;     // m x c gather buffer
  int* order;      // c
  int* ptmp;       // c
};

__device__ __forceinline__ bool qg_better(double v, int p, double bv, int bp) { return v > bv || (v == bv && p < bp); }

// Sum of squares of rows [a, r1) of column col (lane-strided, 4 chains, whole warp).
__device__ __forceinline__ double qg_sumsq(const double* col, int a, int r1, int lane) {
  double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
  int i = a + lane;
  for (; i + 96 < r1; i += 128) {
    const double x0 = col[i], x1 = col[i + 32], x2 = col[i + 64], x3 = col[i + 96];
    q0 += x0 * x0; q1 += x1 * x1; q2 += x2 * x2; q3 += x3 * x3;
  }
  for (; i < r1; i += 32) { const double x = col[i]; q0 += x * x; }
  return warp_sum((q0 + q1) + (q2 + q3));
}

// Last-arriver reduction of RC partials (chunks lo..RC-1) of column j into out[j] (fixed order).
// Called by the whole warp; lane 0 has written part[chunk * c + j] already.
__device__ __forceinline__ bool qg_arrive(int* cnt, int j, int nact, int lane) {
  int last = 0;
  if (lane == 0) {  // acq_rel RMW: releases this lane's partial, acquires the others' (no full fence)
    cuda::atomic_ref<int, cuda::thread_scope_device> r(cnt[j]);
    last = (r.fetch_add(1, cuda::memory_order_acq_rel) == nact - 1);
    if (last) r.store(0, cuda::memory_order_relaxed);
  }
  return __shfl_sync(0xffffffffu, last, 0) != 0;
}

__device__ __forceinline__ double qg_sum_parts(const double* part, int c, int j, int lo, int RC, int lane) {
  double v = 0.0;
  for (int q = lo + lane; q < RC; q += 32) v += __ldcg(part + (int64_t)q * c + j);
  return warp_sum(v);  // fixed shuffle tree: deterministic
}

__global__ void __launch_bounds__(QG_T, 4) qrcp_grid_kernel(QGArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ unsigned char qg_smem[];
  // unprocessed columns as a list (alist[0..nalive), apos = position of a column in it): the
  // (column, chunk) pairs are dealt over the live columns and live chunks only, so every warp
  // gets the same number of pairs (+-1) at every step; identical in every CTA
  int* alist = reinterpret_cast<int*>(qg_smem);
  int* apos = alist + a.c;
  unsigned char* done = reinterpret_cast<unsigned char*>(apos + a.c);  // c flags
  __shared__ double red_v[QG_W], red_m[QG_W];
  __shared__ int red_p[QG_W];
  __shared__ int piv_s, nalive;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gw = blockIdx.x * QG_W + warp, nwg = gridDim.x * QG_W;
  const int m = a.m, c = a.c, CH = a.CH, RC = a.RC;
  const int64_t ldy = a.ldy;
  double* Y = a.Y;
  const int kmax = min(min(m, c), a.kcap);
  for (int j = tid; j < c; j += QG_T) {
    done[j] = (j < a.k_start) ? 1 : 0;
    if (j >= a.k_start) { alist[j - a.k_start] = j; apos[j] = j - a.k_start; }
  }
  if (tid == 0) nalive = c - a.k_start;
  if (a.k_start == 0)
    for (int j = blockIdx.x * QG_T + tid; j < c; j += gridDim.x * QG_T) a.perm[j] = j;
  __syncthreads();
  // exact masses of rows >= k_start and >= k_start + 1
  {
    const int s = a.k_start, lo = s / CH, nact = RC - lo, na = nalive;
    for (int q = gw; q < nact * na; q += nwg) {
      const int ch = lo + q / na, j = alist[q % na];
      const int r0 = max(ch * CH, s), r1 = min(m, (ch + 1) * CH);
      const double* col = Y + (int64_t)j * ldy;
      double m1 = 0.0, m2 = 0.0;
      if (r0 < r1) {
        if (r0 == s) {  // row s peeled off: rows > s summed on their own (no subtraction)
          const double x = col[s];
          m2 = qg_sumsq(col, r0 + 1, r1, lane);
          m1 = m2 + x * x;
        } else {
          m1 = m2 = qg_sumsq(col, r0, r1, lane);
        }
      }
      if (lane == 0) { a.n1part[(int64_t)ch * c + j] = m1; a.n2part[(int64_t)ch * c + j] = m2; }
      if (qg_arrive(a.cnt, j, nact, lane)) {
        const double t1 = qg_sum_parts(a.n1part, c, j, lo, RC, lane);
        const double t2 = qg_sum_parts(a.n2part, c, j, lo, RC, lane);
        if (lane == 0) { a.n1[j] = t1; a.n2[j] = t2; }
      }
    }
  }
  grid.sync();
  int s = a.k_start, prev_p = -1;
  double prev_scal = 0.0, prev_beta = 0.0, mass = 0.0;
#pragma unroll 1
  for (;; ++s) {
    // ---- top: total mass and pivot over the unprocessed columns (same result in every CTA)
    {
      double ms = 0.0, bv = -1.0;
      int bp = 0x7fffffff;
      for (int t = tid; t < nalive; t += QG_T) {
        const int j = alist[t];
        const double v = a.n1[j];
        ms += v;
        if (qg_better(v, j, bv, bp)) { bv = v; bp = j; }
      }
      ms = warp_sum(ms);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (qg_better(ov, op, bv, bp)) { bv = ov; bp = op; }
      }
      if (lane == 0) { red_v[warp] = bv; red_p[warp] = bp; red_m[warp] = ms; }
      __syncthreads();
      if (tid == 0) {
        double tv = -1.0, tm = 0.0;
        int tp = 0x7fffffff;
        for (int w = 0; w < QG_W; ++w) {
          tm += red_m[w];
          if (qg_better(red_v[w], red_p[w], tv, tp)) { tv = red_v[w]; tp = red_p[w]; }
        }
        red_m[0] = tm;
        piv_s = tp;
      }
      __syncthreads();
      mass = red_m[0];
    }
    const int p = piv_s;
    if (s >= kmax || mass <= a.stop2 || p >= c) break;
    // ---- reflector of column p, rows s..m-1 (dlarfg), formed redundantly in every CTA
    const double alpha = Y[s + (int64_t)p * ldy];
    const double sigma = a.n2[p];
    double t = 0.0, beta = alpha, scal = 0.0;
    if (sigma != 0.0) {
      const double nr = sqrt(alpha * alpha + sigma);
      beta = alpha >= 0.0 ? -nr : nr;
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    if (blockIdx.x == 0 && tid == 0) {
      a.tau[s] = t;
      a.order[s] = p;  // pivot sequence (the gather at the end reads it)
    }
    __syncthreads();  // every thread has read piv_s / red_m before done[] and the list change
    if (tid == 0) {  // swap-remove p from the live list
      done[p] = 1;
      const int ip = apos[p], last = alist[nalive - 1];
      alist[ip] = last;
      apos[last] = ip;
      nalive = nalive - 1;
    }
    // previous pivot column -> its reflector (nobody reads it any more)
    if (prev_p >= 0) {
      double* col = Y + (int64_t)prev_p * ldy;
      for (int i = s + blockIdx.x * QG_T + tid; i < m; i += gridDim.x * QG_T) col[i] *= prev_scal;
      if (blockIdx.x == 0 && tid == 0) col[s - 1] = prev_beta;
    }
    __syncthreads();
    const double* vcol = Y + (int64_t)p * ldy;
    const int lo = s / CH, nact = RC - lo, na = nalive;
    // ---- phase 1: w_j = v^T Y[s:, j] with v = [1; scal * Y[s+1:, p]]
    for (int q = gw; q < nact * na; q += nwg) {
      const int ch = lo + q / na, j = alist[q % na];
      const int r0 = max(ch * CH, s + 1), r1 = min(m, (ch + 1) * CH);
      const double* col = Y + (int64_t)j * ldy;
      double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
      int i = r0 + lane;
      for (; i + 96 < r1; i += 128) {
        q0 += vcol[i] * col[i];
        q1 += vcol[i + 32] * col[i + 32];
        q2 += vcol[i + 64] * col[i + 64];
        q3 += vcol[i + 96] * col[i + 96];
      }
      for (; i < r1; i += 32) q0 += vcol[i] * col[i];
      double part = scal * warp_sum((q0 + q1) + (q2 + q3));
      if (ch == lo) part += col[s];
      if (lane == 0) a.wpart[(int64_t)ch * c + j] = part;
    }
    grid.sync();
    // ---- phase 2: Y[s:, j] -= tau w_j v; exact masses of rows >= s+1 and >= s+2
    for (int q = gw; q < nact * na; q += nwg) {
      const int ch = lo + q / na, j = alist[q % na];
      const int r0 = max(ch * CH, s + 1), r1 = min(m, (ch + 1) * CH);
      double* col = Y + (int64_t)j * ldy;
      // w_j = sum of the chunk partials in chunk order (read by every chunk of column j: no
      // atomics or fences in phase 1, the grid barrier orders the partials)
      const double qj = t * qg_sum_parts(a.wpart, c, j, lo, RC, lane);
      const double qv = qj * scal;
      // row s+1 (first row of the chunk that holds it) peeled off: rows >= s+2 summed on their own
      int b = r0;
      double e1 = 0.0;
      if (r0 == s + 1 && r0 < r1) {
        const double x = col[r0] - qv * vcol[r0];
        e1 = x * x;
        __syncwarp();
        if (lane == 0) col[r0] = x;
        b = r0 + 1;
      }
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
      int i = b + lane;
      if (qj != 0.0) {
        for (; i + 96 < r1; i += 128) {
          const double x0 = col[i] - qv * vcol[i], x1 = col[i + 32] - qv * vcol[i + 32];
          const double x2 = col[i + 64] - qv * vcol[i + 64], x3 = col[i + 96] - qv * vcol[i + 96];
          col[i] = x0; col[i + 32] = x1; col[i + 64] = x2; col[i + 96] = x3;
          s0 += x0 * x0; s1 += x1 * x1; s2 += x2 * x2; s3 += x3 * x3;
        }
        for (; i < r1; i += 32) { const double x = col[i] - qv * vcol[i]; col[i] = x; s0 += x * x; }
      } else {
        for (; i + 96 < r1; i += 128) {
          const double x0 = col[i], x1 = col[i + 32], x2 = col[i + 64], x3 = col[i + 96];
          s0 += x0 * x0; s1 += x1 * x1; s2 += x2 * x2; s3 += x3 * x3;
        }
        for (; i < r1; i += 32) { const double x = col[i]; s0 += x * x; }
      }
      const double m2 = warp_sum((s0 + s1) + (s2 + s3));
      const double m1 = m2 + e1;
      if (ch == lo && lane == 0) col[s] -= qj;
      if (lane == 0) { a.n1part[(int64_t)ch * c + j] = m1; a.n2part[(int64_t)ch * c + j] = m2; }
      if (qg_arrive(a.cnt, j, nact, lane)) {
        const double t1 = qg_sum_parts(a.n1part, c, j, lo, RC, lane);
        const double t2 = qg_sum_parts(a.n2part, c, j, lo, RC, lane);
        if (lane == 0) { a.n1[j] = t1; a.n2[j] = t2; }
      }
    }
    grid.sync();
    prev_p = p;
    prev_scal = scal;
    prev_beta = beta;
  }
  const int k = s;
  if (prev_p >= 0) {
    double* col = Y + (int64_t)prev_p * ldy;
    for (int i = k + blockIdx.x * QG_T + tid; i < m; i += gridDim.x * QG_T) col[i] *= prev_scal;
    if (blockIdx.x == 0 && tid == 0) col[k - 1] = prev_beta;
  }
  // ---- gather into pivot order: positions k_start..k-1 the pivots, then the rest ascending
  if (blockIdx.x == 0 && tid == 0) {
    int pos = k;
    for (int j = a.k_start; j < c; ++j)
      if (!done[j]) a.order[pos++] = j;
    a.scalars[0] = (double)k;
    a.scalars[1] = mass;  // exact mass of the unprocessed columns (rows >= k)
  }
  grid.sync();
  const int ncols = c - a.k_start;
  const int64_t tot = (int64_t)ncols * m;
  for (int64_t e = (int64_t)blockIdx.x * QG_T + tid; e < tot; e += (int64_t)gridDim.x * QG_T) {
    const int jj = (int)(e / m), i = (int)(e - (int64_t)jj * m);
    a.tmp[e] = Y[i + (int64_t)a.order[a.k_start + jj] * ldy];
  }
  for (int jj = blockIdx.x * QG_T + tid; jj < ncols; jj += gridDim.x * QG_T) a.ptmp[jj] = a.perm[a.order[a.k_start + jj]];
  grid.sync();
  for (int64_t e = (int64_t)blockIdx.x * QG_T + tid; e < tot; e += (int64_t)gridDim.x * QG_T) {
    const int jj = (int)(e / m), i = (int)(e - (int64_t)jj * m);
    Y[i + (int64_t)(a.k_start + jj) * ldy] = a.tmp[e];
  }
  for (int jj = blockIdx.x * QG_T + tid; jj < ncols; jj += gridDim.x * QG_T) a.perm[a.k_start + jj] = a.ptmp[jj];
}

}  // namespace

bool qrcp_grid_run(tt_ctx ctx, double* Y, int64_t ldy, int64_t m, int64_t c, int k_start, double stop2, int kcap,
                   double* tau, double* norms, int* perm, double* scalars) {
  const size_t smem = (size_t)c * (1 + 2 * sizeof(int)) + 16;
  if (smem > 160 * 1024) return false;
  if (smem > 48 * 1024)
    TTB_CUDA(cudaFuncSetAttribute(qrcp_grid_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  TTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, qrcp_grid_kernel, QG_T, smem));
  if (per_sm < 1) return false;
  static const char* ps_env = std::getenv("TT_B200_QG_PERSM");
  per_sm = std::min(per_sm, ps_env ? std::max(1, std::atoi(ps_env)) : 4);
  const int G = ctx->num_sms * per_sm;
  const int64_t nwg = (int64_t)G * QG_W;
  // rows per chunk: about two (column, chunk) pairs per warp, 128-row multiples, 128..4096
  static const char* chm_env = std::getenv("TT_B200_QG_PAIRS");  // (column, chunk) pairs per warp
  const double ppw = chm_env ? std::max(0.05, std::atof(chm_env)) : 1.0;
  int64_t CH = ceil_div((int64_t)std::ceil((double)m * c / (ppw * (double)nwg)), 128) * 128;
  CH = std::max<int64_t>(128, std::min<int64_t>(CH, 4096));
  const int64_t RC = ceil_div(m, CH);
  DBuf parts(ctx, (size_t)(3 * RC * c + 2 * c + (size_t)m * c));
  IBuf ints(ctx, (size_t)(3 * c));
  TTB_CUDA(cudaMemsetAsync(ints.p, 0, sizeof(int) * (size_t)c, ctx->stream));
  QGArgs a;
  a.Y = Y;
  a.ldy = ldy;
  a.m = (int)m;
  a.c = (int)c;
  a.k_start = k_start;
  a.kcap = kcap;
  a.stop2 = stop2;
  a.tau = tau;
  a.perm = perm;
  a.scalars = scalars;
  a.CH = (int)CH;
  a.RC = (int)RC;
  a.wpart = parts.p;
  a.n1part = parts.p + RC * c;
  a.n2part = parts.p + 2 * RC * c;
  a.w = parts.p + 3 * RC * c;
  a.n1 = norms;
  a.n2 = norms + c;
  a.tmp = parts.p + 3 * RC * c + c;
  a.cnt = ints.p;
  a.order = ints.p + c;
  a.ptmp = ints.p + 2 * c;
  void* args[] = {&a};
  TTB_RUN(ctx, "qrcp_grid", 0, 16.0 * m * c,
          TTB_CUDA(cudaLaunchCooperativeKernel((const void*)qrcp_grid_kernel, dim3(G), dim3(QG_T), args, smem,
                                               ctx->stream)));
  return true;
}

}  // namespace ttb
