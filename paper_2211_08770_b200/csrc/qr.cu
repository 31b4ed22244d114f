// Householder QR kernels (FP64, sm_100a).
//
//  * tsqr_leaf_reg_kernel: one CTA factors a <=256-row chunk of a <=32-column panel with
//                         the rows held in registers (LAPACK dgeqr2 arithmetic), writes its R
//                         to the stack of the next tree level and its explicit Q.
//  * tsqr_combine_kernel: Q_panel(chunk p) = Q_leaf(chunk p) * Q_next(p-th w x w block).
//  * hr_kernel          : Householder reconstruction (LU with sign choice of Q_1 - S) so the
//                         TSQR panel becomes compact-WY (Y, T) with H[:, :w] = Q S, R_h = S R.
//  * qrcp_kernel        : unblocked Householder QR with column pivoting and a Frobenius
//                         stopping test (truncated-SVD stage of the left-to-right sweep).
#include <algorithm>
#include <cstdlib>

#include "gemm.cuh"
#include "qr.cuh"

namespace ttb {

namespace {

// a[j] / a[j] = v for a runtime j without dynamic register indexing (32 predicated moves)
__device__ __forceinline__ double sel32(const double (&a)[32], int j) {
  double r = 0.0;
#pragma unroll
  for (int c = 0; c < 32; ++c)
    if (c == j) r = a[c];
  return r;
}
__device__ __forceinline__ void put32(double (&a)[32], int j, double v) {
#pragma unroll
  for (int c = 0; c < 32; ++c)
    if (c == j) a[c] = v;
}

// Sum a per-lane array p[0..31] over the warp, scattered: on return p[0] of lane l holds
// sum_lanes p_in[l] (butterfly reduce-scatter: 16 + 8 + 4 + 2 + 1 shuffles).
__device__ __forceinline__ void warp_reduce_scatter32(double (&p)[32], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool hi = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < o; ++i) {
      const double send = hi ? p[i] : p[o + i];
      const double keep = hi ? p[o + i] : p[i];
      p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

// Register-resident Householder QR of one <= 256-row chunk of a <= 32-column panel:
// thread t owns row t (32 doubles).  Per column: one block reduction for the norm, one
// butterfly reduce-scatter + one cross-warp pass for the 31 dot products, 32 FMAs.
// Writes R (w x w, to the next level's stack) and the explicit Q chunk (h x w).
constexpr int REG_THREADS = 256;
__global__ void __launch_bounds__(REG_THREADS) tsqr_leaf_reg_kernel(const double* __restrict__ A, int64_t lda,
                                                                    int m, int w, int P, double* Qout, int64_t ldq,
                                                                    double* Rst, int64_t ldr) {
  constexpr int NW = REG_THREADS / 32;
  __shared__ double red[NW][33];
  __shared__ double bc[34];
  __shared__ double tau_s[32];
  const int p = blockIdx.x;
  const int base = m / P, rem = m % P;
  const int r0 = p * base + min(p, rem);
  const int h = base + (p < rem ? 1 : 0);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = (t < h && c < w) ? A[(int64_t)(r0 + t) + (int64_t)c * lda] : 0.0;
  // ---------------- factorisation (LAPACK dgeqr2 arithmetic).  The column loop stays rolled
  // (an unrolled body is ~360 KB of SASS and thrashes the instruction cache); register
  // entries are addressed through static selects.
#pragma unroll 1
  for (int j = 0; j < 32; ++j) {
    const double aj = sel32(a, j);
    double x = (t > j) ? aj : 0.0;
    double s = warp_sum(x * x);
    if (lane == 0) red[warp][32] = s;
    if (t == j) bc[32] = aj;
    __syncthreads();
    double sigma = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) sigma += red[q][32];
    const double alpha = bc[32];
    double tj = 0.0, beta = alpha, scal = 0.0;
    if (sigma != 0.0) {
      const double nrm = sqrt(alpha * alpha + sigma);
      beta = alpha >= 0.0 ? -nrm : nrm;
      tj = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    const double v = (t > j) ? aj * scal : (t == j ? 1.0 : 0.0);
    put32(a, j, (t > j) ? v : (t == j ? beta : aj));
    if (t == 0) tau_s[j] = tj;
    if (j < 31 && tj != 0.0) {
      double pp[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) pp[c] = (c > j) ? v * a[c] : 0.0;
      warp_reduce_scatter32(pp, lane);
      red[warp][lane] = pp[0];
      __syncthreads();
      if (warp == 0) {
        double wc = 0.0;
#pragma unroll
        for (int q = 0; q < NW; ++q) wc += red[q][lane];
        bc[lane] = tj * wc;
      }
      __syncthreads();
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c > j) a[c] -= v * bc[c];
    } else {
      __syncthreads();
    }
  }
  // R rows 0..w-1 -> stack rows [p*w, p*w + w)
  if (t < w) {
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (c < w) Rst[(int64_t)(p * w + t) + (int64_t)c * ldr] = (c >= t) ? a[c] : 0.0;
  }
  // ---------------- explicit Q = H_0 ... H_31 [I; 0] (backward accumulation)
  double qv[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) qv[c] = (t == c) ? 1.0 : 0.0;
#pragma unroll 1
  for (int j = 31; j >= 0; --j) {
    const double tj = tau_s[j];
    if (tj == 0.0) continue;  // uniform across the block
    const double v = (t > j) ? sel32(a, j) : (t == j ? 1.0 : 0.0);
    double pp[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) pp[c] = (c >= j) ? v * qv[c] : 0.0;
    warp_reduce_scatter32(pp, lane);
    __syncthreads();
    red[warp][lane] = pp[0];
    __syncthreads();
    if (warp == 0) {
      double wc = 0.0;
#pragma unroll
      for (int q = 0; q < NW; ++q) wc += red[q][lane];
      bc[lane] = tj * wc;
    }
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (c >= j) qv[c] -= v * bc[c];
  }
  if (t < h) {
#pragma unroll
    for (int c = 0; c < 32; ++c)
      if (c < w) Qout[(int64_t)(r0 + t) + (int64_t)c * ldq] = qv[c];
  }
}

__global__ void __launch_bounds__(256) tsqr_combine_kernel(const double* __restrict__ Ql, int64_t ldl,
                                                           const double* __restrict__ QS, int64_t lds, int m, int w,
                                                           int P, double* Qout, int64_t ldq) {
  __shared__ double Bs[32 * 33];
  const int p = blockIdx.x;
  const int base = m / P, rem = m % P;
  const int r0 = p * base + min(p, rem);
  const int h = base + (p < rem ? 1 : 0);
  for (int idx = threadIdx.x; idx < w * w; idx += blockDim.x) {
    const int c = idx / w, k = idx - c * w;
    Bs[c * 33 + k] = QS[(int64_t)(p * w + k) + (int64_t)c * lds];
  }
  __syncthreads();
  for (int row = threadIdx.x; row < h; row += blockDim.x) {
    double a[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) a[k] = (k < w) ? Ql[(int64_t)(r0 + row) + (int64_t)k * ldl] : 0.0;
    for (int c = 0; c < w; ++c) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 32; ++k) s += a[k] * Bs[c * 33 + k];
      Qout[(int64_t)(r0 + row) + (int64_t)c * ldq] = s;
    }
  }
}

// Householder reconstruction (Ballard et al.): choose S = diag(+-1) during an LU without
// pivoting of W = [I; 0] - Q S (pivots 1 + |.| >= 1), so W = Y U with Y unit lower
// trapezoidal; then T = U Y_1^{-T} and I - Y T Y^T has first columns Q S, R_h = S R.
// Warp 0 of every CTA eliminates the w x w top block right-looking (lane i holds row i in
// registers), inverts U and Y_1 into shared memory; every thread then writes its rows
// Y_2(i, :) = -Q_2(i, :) S U^{-1} (statically indexed 32 x 32 product).
__global__ void __launch_bounds__(256) hr_kernel(const double* __restrict__ Q, int64_t ldq, int m, int w,
                                                 const double* __restrict__ Rp, int64_t ldrp, double* Y,
                                                 int64_t ldy, double* T, int64_t ldt, double* Rh, int64_t ldrh) {
  __shared__ double Us[32][33];   // U (upper, final)
  __shared__ double Ls[32][33];   // Y_1 = L (unit lower)
  __shared__ double Ss[32];
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid < 32) {
    double z[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) z[c] = (lane < w && c < w) ? Q[lane + (int64_t)c * ldq] : 0.0;
    Ss[lane] = 1.0;
#pragma unroll 1
    for (int j = 0; j < w; ++j) {  // rolled: the unrolled body thrashes the instruction cache
      const double zj = sel32(z, j);
      const double piv = __shfl_sync(0xffffffffu, zj, j);
      const double s = (piv >= 0.0) ? -1.0 : 1.0;
      const double ujj = 1.0 + fabs(piv);
      if (lane == 0) Ss[j] = s;
      const double lij = (lane > j && lane < w) ? (-s * zj / ujj) : 0.0;
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const double rjc = __shfl_sync(0xffffffffu, z[c], j);
        if (c > j) z[c] -= lij * rjc;
      }
      put32(z, j, lane == j ? ujj : (lane > j ? lij : zj));
    }
    __syncwarp();
    // row `lane`: z[c] holds L(lane, c) for c < lane, U(lane, lane) at c == lane, and the
    // raw eliminated M(lane, c) for c > lane with U(lane, c) = -s_c M(lane, c)
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const bool in = (lane < w && c < w);
      Ls[lane][c] = !in ? (lane == c ? 1.0 : 0.0) : (c < lane ? z[c] : (c == lane ? 1.0 : 0.0));
      Us[lane][c] = !in ? (lane == c ? 1.0 : 0.0) : (c < lane ? 0.0 : (c == lane ? z[c] : -Ss[c] * z[c]));
    }
    __syncwarp();
  }
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + tid; i < m; i += gridDim.x * blockDim.x) {
    if (i < w) {
      for (int c = 0; c < w; ++c) Y[i + (int64_t)c * ldy] = Ls[i][c];
    } else {
      // row solve y U = -q S (forward substitution over columns, y in registers)
      double y[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        y[c] = 0.0;
        if (c < w) {
          double acc = -Ss[c] * Q[i + (int64_t)c * ldq];
#pragma unroll
          for (int k = 0; k < c; ++k) acc -= y[k] * Us[k][c];
          y[c] = acc / Us[c][c];
          Y[i + (int64_t)c * ldy] = y[c];
        }
      }
    }
  }
  if (blockIdx.x == 0) {
    if (tid < 32 && tid < w) {
      // T Y_1^T = U, row `tid`: T(i, j) = U(i, j) - sum_{k<j} T(i, k) Y_1(j, k) (T upper)
      double trow[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        double acc = (j < w && j >= tid) ? Us[tid][j] : 0.0;
#pragma unroll
        for (int k = 0; k < j; ++k) acc -= trow[k] * Ls[j][k];
        trow[j] = (j >= tid) ? acc : 0.0;
        if (j < w) T[tid + (int64_t)j * ldt] = trow[j];
      }
    }
    for (int idx = tid; idx < w * w; idx += blockDim.x) {
      const int c = idx / w, r = idx - c * w;
      if (r <= c) Rh[r + (int64_t)c * ldrh] = Ss[r] * Rp[r + (int64_t)c * ldrp];
    }
  }
}

__global__ void copy_upper_kernel(const double* A, int64_t lda, int rows, int cols, double* R, int64_t ldr) {
  const int64_t total = (int64_t)rows * cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx % rows), c = (int)(idx / rows);
    R[r + (int64_t)c * ldr] = (r <= c) ? A[r + (int64_t)c * lda] : 0.0;
  }
}

// Merge two compact-WY blocks (dlarft's forward accumulation): with Q1 = I - Y1 T1 Y1^T and
// Q2 = I - Y2 T2 Y2^T, Q1 Q2 = I - [Y1 Y2] T [Y1 Y2]^T, T = [[T1, -T1 G T2], [0, T2]], G = Y1^T Y2.
// T points at the merged block (ld ldt): T1 in rows [0, w1) of columns [0, w1), T2 on entry in rows
// [0, w2) of columns [w1, w1 + w2); on exit T2 sits in rows [w1, w1 + w2).  One CTA of 1024.
__global__ void __launch_bounds__(1024) merge_t_kernel(double* T, int64_t ldt, const double* __restrict__ G,
                                                       int64_t ldg, int w1, int w2) {
  __shared__ double t1[32][33], t2[32][33], g[32][33], h[32][33];
  const int tid = threadIdx.x, r = tid & 31, c = tid >> 5;
  t1[r][c] = (r < w1 && c < w1) ? T[r + (int64_t)c * ldt] : 0.0;
  t2[r][c] = (r < w2 && c < w2) ? T[r + (int64_t)(w1 + c) * ldt] : 0.0;
  g[r][c] = (r < w1 && c < w2) ? G[r + (int64_t)c * ldg] : 0.0;
  __syncthreads();
  double acc = 0.0;  // H = G T2
  for (int k = 0; k < w2; ++k) acc = fma(g[r][k], t2[k][c], acc);
  h[r][c] = acc;
  __syncthreads();
  acc = 0.0;  // T12 = -T1 H
  for (int k = 0; k < w1; ++k) acc = fma(t1[r][k], h[k][c], acc);
  if (c < w2) {
    if (r < w1) T[r + (int64_t)(w1 + c) * ldt] = -acc;
    if (r < w2) T[w1 + r + (int64_t)(w1 + c) * ldt] = t2[r][c];
  }
  if (c < w1 && r < w2) T[w1 + r + (int64_t)c * ldt] = 0.0;
}

__global__ void set_identity_kernel(double* Q, int64_t ldq, int m, int k) {
  const int64_t total = (int64_t)m * k;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx % m), c = (int)(idx / m);
    Q[r + (int64_t)c * ldq] = (r == c) ? 1.0 : 0.0;
  }
}

int grid_for(int64_t n, int threads, int cap = 4096) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), cap));
}

// Recursive TSQR of the m x w matrix A (w <= 32): explicit Q (m x w) and R (w x w, ld w).
void tsqr(tt_ctx ctx, const double* A, int64_t lda, int64_t m, int w, double* Qout, int64_t ldq, double* Rout) {
  if (m <= QR_LEAF) {
    TTB_RUN(ctx, "tsqr_leaf", 4.0 * m * w * w, 16.0 * m * w,
            tsqr_leaf_reg_kernel<<<1, REG_THREADS, 0, ctx->stream>>>(A, lda, (int)m, w, 1, Qout, ldq, Rout, w));
    return;
  }
  const int P = (int)ceil_div(m, QR_LEAF);
  const int64_t ms = (int64_t)P * w;
  DBuf Qleaf(ctx, (size_t)m * w), S(ctx, (size_t)ms * w), QS(ctx, (size_t)ms * w);
  TTB_RUN(ctx, "tsqr_leaf", 4.0 * m * w * w, 16.0 * m * w + 8.0 * ms * w,
          tsqr_leaf_reg_kernel<<<P, REG_THREADS, 0, ctx->stream>>>(A, lda, (int)m, w, P, Qleaf.p, m, S.p, ms));
  tsqr(ctx, S.p, ms, ms, w, QS.p, ms, Rout);
  TTB_RUN(ctx, "tsqr_combine", 2.0 * m * w * w, 16.0 * m * w + 8.0 * ms * w,
          tsqr_combine_kernel<<<P, 256, 0, ctx->stream>>>(Qleaf.p, m, QS.p, ms, (int)m, w, P, Qout, ldq));
}

// ---------------------------------------------------------------- QRCP
__global__ void __launch_bounds__(1024) qrcp_kernel(double* Y, int64_t ldy, int m, int c, int k_start, double stop2,
                                                    int kcap, double* tau, double* norms_g, int* perm_g,
                                                    double* scalars) {
  extern __shared__ double sm[];
  double* nrm = sm;
  double* nrm0 = sm + c;
  int* perm = reinterpret_cast<int*>(sm + 2 * c);
  __shared__ double red[32];
  __shared__ double redv[32];
  __shared__ int redi[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;

  if (k_start == 0) {
    for (int j = warp; j < c; j += nw) {
      double s = 0.0;
      for (int i = lane; i < m; i += 32) { const double v = Y[i + (int64_t)j * ldy]; s += v * v; }
      s = warp_sum(s);
      if (lane == 0) { nrm[j] = s; nrm0[j] = s; perm[j] = j; }
    }
  } else {
    for (int j = tid; j < c; j += blockDim.x) { nrm[j] = norms_g[j]; nrm0[j] = norms_g[c + j]; perm[j] = perm_g[j]; }
  }
  __syncthreads();
  const int kmax = min(min(m, c), kcap);
  int s = k_start;
  for (; s < kmax; ++s) {
    double part = 0.0;
    for (int j = s + tid; j < c; j += blockDim.x) part += nrm[j];
    double tot = block_sum(part, red);
    if (tot <= 4.0 * stop2 || s == k_start) {
      // exact recomputation of the trailing column norms (rows >= s)
      for (int j = s + warp; j < c; j += nw) {
        double q = 0.0;
        for (int i = s + lane; i < m; i += 32) { const double v = Y[i + (int64_t)j * ldy]; q += v * v; }
        q = warp_sum(q);
        if (lane == 0) { nrm[j] = q; nrm0[j] = q; }
      }
      __syncthreads();
      part = 0.0;
      for (int j = s + tid; j < c; j += blockDim.x) part += nrm[j];
      tot = block_sum(part, red);
    }
    if (tot <= stop2) break;
    // pivot: argmax_{j >= s} nrm[j], ties -> smallest j
    double bv = -1.0;
    int bi = c;
    for (int j = s + tid; j < c; j += blockDim.x) {
      const double v = nrm[j];
      if (v > bv || (v == bv && j < bi)) { bv = v; bi = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (lane == 0) { redv[warp] = bv; redi[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      bv = (lane < nw) ? redv[lane] : -1.0;
      bi = (lane < nw) ? redi[lane] : c;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
      }
      if (lane == 0) redi[0] = bi;
    }
    __syncthreads();
    const int pv = redi[0];
    __syncthreads();
    if (pv != s) {
      for (int i = tid; i < m; i += blockDim.x) {
        const double a = Y[i + (int64_t)s * ldy];
        Y[i + (int64_t)s * ldy] = Y[i + (int64_t)pv * ldy];
        Y[i + (int64_t)pv * ldy] = a;
      }
      if (tid == 0) {
        double t = nrm[s]; nrm[s] = nrm[pv]; nrm[pv] = t;
        t = nrm0[s]; nrm0[s] = nrm0[pv]; nrm0[pv] = t;
        const int q = perm[s]; perm[s] = perm[pv]; perm[pv] = q;
      }
      __syncthreads();
    }
    // Householder vector of column s (rows s..m-1), LAPACK dlarfg
    double pp = 0.0;
    for (int i = s + 1 + tid; i < m; i += blockDim.x) { const double v = Y[i + (int64_t)s * ldy]; pp += v * v; }
    const double sigma = block_sum(pp, red);
    const double alpha = Y[s + (int64_t)s * ldy];
    double t = 0.0, beta = alpha, scal = 0.0;
    if (sigma != 0.0) {
      const double nr = sqrt(alpha * alpha + sigma);
      beta = alpha >= 0.0 ? -nr : nr;
      t = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    for (int i = s + 1 + tid; i < m; i += blockDim.x) Y[i + (int64_t)s * ldy] *= scal;
    __syncthreads();
    if (tid == 0) { Y[s + (int64_t)s * ldy] = beta; tau[s] = t; }
    // apply to the trailing columns and downdate their norms
    for (int j = s + 1 + warp; j < c; j += nw) {
      double* col = Y + (int64_t)j * ldy;
      if (t != 0.0) {
        double q = 0.0;
        for (int i = s + 1 + lane; i < m; i += 32) q += Y[i + (int64_t)s * ldy] * col[i];
        q = warp_sum(q);
        q = t * (q + col[s]);
        for (int i = s + 1 + lane; i < m; i += 32) col[i] -= q * Y[i + (int64_t)s * ldy];
        __syncwarp();
        if (lane == 0) col[s] -= q;
        __syncwarp();
      }
      const double rs = col[s];
      double nn = nrm[j] - rs * rs;
      if (!(nn > 1e-8 * nrm0[j])) {
        double q = 0.0;
        for (int i = s + 1 + lane; i < m; i += 32) { const double v = col[i]; q += v * v; }
        q = warp_sum(q);
        nn = q;
        if (lane == 0) nrm0[j] = q;
      }
      __syncwarp();
      if (lane == 0) nrm[j] = nn;
    }
    __syncthreads();
  }
  // exact trailing mass
  double part = 0.0;
  for (int j = s + warp; j < c; j += nw)
    for (int i = s + lane; i < m; i += 32) { const double v = Y[i + (int64_t)j * ldy]; part += v * v; }
  const double e2 = block_sum(part, red);
  for (int j = tid; j < c; j += blockDim.x) { norms_g[j] = nrm[j]; norms_g[c + j] = nrm0[j]; perm_g[j] = perm[j]; }
  if (tid == 0) { scalars[0] = (double)s; scalars[1] = e2; }
}

__global__ void __launch_bounds__(1024) apply_reflectors_kernel(const double* __restrict__ Y, int64_t ldy,
                                                                const double* __restrict__ tau, int m, int k,
                                                                double* X, int64_t ldx, int nc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = k - 1; j >= 0; --j) {
    const double t = tau[j];
    if (t != 0.0) {
      for (int c = warp; c < nc; c += nw) {
        double* col = X + (int64_t)c * ldx;
        double q = 0.0;
        for (int i = j + 1 + lane; i < m; i += 32) q += Y[i + (int64_t)j * ldy] * col[i];
        q = warp_sum(q);
        q = t * (q + col[j]);
        for (int i = j + 1 + lane; i < m; i += 32) col[i] -= q * Y[i + (int64_t)j * ldy];
        __syncwarp();
        if (lane == 0) col[j] -= q;
      }
    }
    __syncthreads();
  }
}

// One CTA per target column (columns are independent): the column lives in shared memory while
// the k reflectors are applied last to first, each dot product one block reduction.
__global__ void __launch_bounds__(256) apply_reflectors_col_kernel(const double* __restrict__ Y, int64_t ldy,
                                                                   const double* __restrict__ tau, int m, int k,
                                                                   double* X, int64_t ldx) {
  extern __shared__ double xs[];
  __shared__ double red[32];
  const int tid = threadIdx.x;
  double* col = X + (int64_t)blockIdx.x * ldx;
  for (int i = tid; i < m; i += 256) xs[i] = col[i];
  __syncthreads();
  for (int j = k - 1; j >= 0; --j) {
    const double t = __ldg(tau + j);
    if (t == 0.0) continue;  // uniform
    const double* v = Y + (int64_t)j * ldy;
    double q0 = 0.0, q1 = 0.0;
    int i = j + 1 + tid;
    for (; i + 256 < m; i += 512) { q0 += __ldg(v + i) * xs[i]; q1 += __ldg(v + i + 256) * xs[i + 256]; }
    if (i < m) q0 += __ldg(v + i) * xs[i];
    const double q = t * (block_sum(q0 + q1, red) + xs[j]);
    for (int r = j + 1 + tid; r < m; r += 256) xs[r] -= q * __ldg(v + r);
    if (tid == 0) xs[j] -= q;
    __syncthreads();
  }
  for (int r = tid; r < m; r += 256) col[r] = xs[r];
}

// Same application with the column in registers: thread t owns rows t + T i (i < RPT), fixed
// for all reflectors, so a reflector's dot and update touch only the thread's own rows (the
// implicit 1 of v at row j is folded into the thread's v values); the one cross-thread step is
// the dot's reduction (warp sums, one __syncthreads, every thread adds the T/32 warp sums in the
// same order; double-buffered).
template <int T, int RPT>  // T threads, RPT rows per thread
__global__ void __launch_bounds__(T) apply_reflectors_reg_kernel(const double* __restrict__ Y, int64_t ldy,
                                                                 const double* __restrict__ tau, int m, int k,
                                                                 double* X, int64_t ldx) {
  constexpr int NW = T / 32;
  __shared__ double red[2][NW];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* col = X + (int64_t)blockIdx.x * ldx;
  double x[RPT];
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = tid + T * i;
    x[i] = r < m ? col[r] : 0.0;
  }
  int b = 0;
#pragma unroll 1
  for (int j = k - 1; j >= 0; --j) {
    const double t = __ldg(tau + j);
    if (t == 0.0) continue;  // uniform
    const double* v = Y + (int64_t)j * ldy;
    constexpr bool KEEP = (T <= 256);  // v kept in registers (larger CTAs: read again from L2)
    double vv[KEEP ? RPT : 1];
    double q0 = 0.0, q1 = 0.0;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      const int r = tid + T * i;
      const double vi = (r > j && r < m) ? __ldg(v + r) : (r == j ? 1.0 : 0.0);
      if constexpr (KEEP) vv[i] = vi;
      if (i & 1) q1 += vi * x[i]; else q0 += vi * x[i];
    }
    const double ws = warp_sum(q0 + q1);
    if (lane == 0) red[b][warp] = ws;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) tot += red[b][w];
    const double q = t * tot;
#pragma unroll
    for (int i = 0; i < RPT; ++i) {
      if constexpr (KEEP) {
        x[i] -= q * vv[i];
      } else {
        const int r = tid + T * i;
        x[i] -= q * ((r > j && r < m) ? __ldg(v + r) : (r == j ? 1.0 : 0.0));
      }
    }
    b ^= 1;
  }
#pragma unroll
  for (int i = 0; i < RPT; ++i) {
    const int r = tid + T * i;
    if (r < m) col[r] = x[i];
  }
}

}  // namespace

void copy_upper(tt_ctx ctx, const double* A, int64_t lda, int64_t rows, int64_t cols, double* R, int64_t ldr) {
  if (rows <= 0 || cols <= 0) return;
  TTB_RUN(ctx, "aux", 0, 16.0 * rows * cols,
          copy_upper_kernel<<<grid_for(rows * cols, 256), 256, 0, ctx->stream>>>(A, lda, (int)rows, (int)cols, R, ldr));
}

void geqrf(tt_ctx ctx, double* A, int64_t lda, int64_t m, int64_t c, QRFactors& f) {
  f.m = m;
  f.c = c;
  f.kmax = std::min(m, c);
  if (f.kmax <= 0) return;
  f.Y.alloc(ctx, (size_t)m * f.kmax);
  f.T.alloc(ctx, (size_t)QR_NB * f.kmax);
  DBuf Qp(ctx, (size_t)m * QR_NB), Rp(ctx, (size_t)QR_NB * QR_NB);
  DBuf W(ctx, (size_t)QR_NB * std::max<int64_t>(c, 1)), W2(ctx, (size_t)QR_NB * std::max<int64_t>(c, 1));
  // rows above the panel inside Y must read as zero for the explicit-Y GEMMs
  TTB_CUDA(cudaMemsetAsync(f.Y.p, 0, sizeof(double) * (size_t)m * f.kmax, ctx->stream));
  f.pan_s.clear();
  f.pan_w.clear();
  // One panel: Householder QR of the ms x w block at (s, s) into Y / T (ld QR_NB at column s).
  auto factor = [&](int64_t s, int w) {
    const int64_t ms = m - s;
    double* P = A + s + s * lda;
    double* Yp = f.Y.p + s + s * m;
    double* Tp = f.T.p + s * QR_NB;
    if (!panel_qr_cluster(ctx, P, lda, ms, w, Yp, m, Tp, QR_NB)) {
      // taller than a cluster: TSQR tree + Householder reconstruction
      tsqr(ctx, P, lda, ms, w, Qp.p, ms, Rp.p);
      TTB_RUN(ctx, "householder_reconstruct", 1.0 * ms * w * w, 16.0 * ms * w,
              hr_kernel<<<grid_for(ms, 256, 1024), 256, 0, ctx->stream>>>(Qp.p, ms, (int)ms, w, Rp.p, w, Yp, m, Tp,
                                                                          QR_NB, P, lda));
    }
  };
  // C (rows [s, m), n2 columns starting at column c0) <- (I - Y T Y^T)^T C for the panel at s.
  auto update = [&](int64_t s, int w, int64_t c0, int64_t n2) {
    if (n2 <= 0) return;
    const int64_t ms = m - s;
    const double* Yp = f.Y.p + s + s * m;
    const double* Tp = f.T.p + s * QR_NB;
    double* C = A + s + c0 * lda;
    GemmDesc g1;  // W = Y^T C
    g1.M = w; g1.N = n2; g1.K = ms; g1.A = Yp; g1.lda = m; g1.ta = true; g1.B = C; g1.ldb = lda; g1.C = W.p; g1.ldc = w;
    gemm(ctx, g1);
    GemmDesc g2;  // W2 = T^T W
    g2.M = w; g2.N = n2; g2.K = w; g2.A = Tp; g2.lda = QR_NB; g2.ta = true; g2.B = W.p; g2.ldb = w; g2.C = W2.p; g2.ldc = w;
    gemm(ctx, g2);
    GemmDesc g3;  // C -= Y W2
    g3.M = ms; g3.N = n2; g3.K = w; g3.A = Yp; g3.lda = m; g3.B = W2.p; g3.ldb = w; g3.C = C; g3.ldc = lda;
    g3.alpha = -1.0; g3.beta = 1.0;
    gemm(ctx, g3);
  };
  static const bool merge_on = [] {
    const char* e = std::getenv("TT_B200_QR_MERGE");
    return !(e && e[0] == '0');
  }();
  for (int64_t s = 0; s < f.kmax;) {
    const int64_t ms = m - s;
    int w = (int)std::min<int64_t>(QR_NB, f.kmax - s);
    // narrower panels when that lets one cluster hold the panel
    if (ms > panel_cluster_max_rows(w) && ms <= panel_cluster_max_rows(16)) w = std::min(w, 16);
    const int w2 = (int)std::min<int64_t>(QR_NB - w, f.kmax - s - w);
    if (merge_on && w < QR_NB && w2 > 0 && c - s - w - w2 > 0) {
      // Two narrow panels, one wide trailing update: the second panel is brought up to date
      // alone, factored, and the two compact-WY blocks merged (T = [[T1, -T1 Y1^T Y2 T2], [0, T2]])
      // so that the trailing matrix -- the HBM traffic of the factorization -- is read and
      // written once per QR_NB columns instead of once per w.
      factor(s, w);
      update(s, w, s + w, w2);
      factor(s + w, w2);
      GemmDesc gg;  // G = Y1^T Y2 over rows [s, m) (Y2 is zero above row s + w)
      gg.M = w; gg.N = w2; gg.K = ms; gg.A = f.Y.p + s + s * m; gg.lda = m; gg.ta = true;
      gg.B = f.Y.p + s + (s + w) * m; gg.ldb = m; gg.C = W.p; gg.ldc = w;
      gemm(ctx, gg);
      TTB_RUN(ctx, "aux", 0, 8.0 * 3 * QR_NB * QR_NB,
              merge_t_kernel<<<1, 1024, 0, ctx->stream>>>(f.T.p + s * QR_NB, QR_NB, W.p, w, w, w2));
      w += w2;
    } else {
      factor(s, w);
    }
    f.pan_s.push_back(s);
    f.pan_w.push_back(w);
    update(s, w, s + w, c - s - w);
    s += w;
  }
}

void orgqr(tt_ctx ctx, const QRFactors& f, double* Q, int64_t ldq) {
  const int64_t m = f.m, kq = f.kmax;
  if (kq <= 0) return;
  TTB_RUN(ctx, "aux", 0, 8.0 * m * kq,
          set_identity_kernel<<<grid_for(m * kq, 256), 256, 0, ctx->stream>>>(Q, ldq, (int)m, (int)kq));
  DBuf W(ctx, (size_t)QR_NB * kq), W2(ctx, (size_t)QR_NB * kq);
  for (int64_t pnl = (int64_t)f.pan_s.size() - 1; pnl >= 0; --pnl) {
    const int64_t s = f.pan_s[(size_t)pnl];
    const int w = f.pan_w[(size_t)pnl];
    const int64_t ms = m - s, ncols = kq - s;
    const double* Yp = f.Y.p + s + s * m;
    const double* Tp = f.T.p + s * QR_NB;
    double* E = Q + s + s * ldq;
    GemmDesc g1;  // W = Y^T E
    g1.M = w; g1.N = ncols; g1.K = ms; g1.A = Yp; g1.lda = m; g1.ta = true; g1.B = E; g1.ldb = ldq; g1.C = W.p; g1.ldc = w;
    gemm(ctx, g1);
    GemmDesc g2;  // W2 = T W
    g2.M = w; g2.N = ncols; g2.K = w; g2.A = Tp; g2.lda = QR_NB; g2.B = W.p; g2.ldb = w; g2.C = W2.p; g2.ldc = w;
    gemm(ctx, g2);
    GemmDesc g3;  // E -= Y W2
    g3.M = ms; g3.N = ncols; g3.K = w; g3.A = Yp; g3.lda = m; g3.B = W2.p; g3.ldb = w; g3.C = E; g3.ldc = ldq;
    g3.alpha = -1.0; g3.beta = 1.0;
    gemm(ctx, g3);
  }
}

void ormqr_left(tt_ctx ctx, const QRFactors& f, double* B, int64_t ldb, int64_t nb) {
  const int64_t m = f.m, kq = f.kmax;
  if (kq <= 0 || nb <= 0) return;
  DBuf W(ctx, (size_t)QR_NB * nb), W2(ctx, (size_t)QR_NB * nb);
  for (int64_t pnl = (int64_t)f.pan_s.size() - 1; pnl >= 0; --pnl) {
    const int64_t s = f.pan_s[(size_t)pnl];
    const int w = f.pan_w[(size_t)pnl];
    const int64_t ms = m - s;
    const double* Yp = f.Y.p + s + s * m;
    const double* Tp = f.T.p + s * QR_NB;
    double* E = B + s;
    GemmDesc g1;  // W = Y^T E
    g1.M = w; g1.N = nb; g1.K = ms; g1.A = Yp; g1.lda = m; g1.ta = true; g1.B = E; g1.ldb = ldb; g1.C = W.p; g1.ldc = w;
    gemm(ctx, g1);
    GemmDesc g2;  // W2 = T W
    g2.M = w; g2.N = nb; g2.K = w; g2.A = Tp; g2.lda = QR_NB; g2.B = W.p; g2.ldb = w; g2.C = W2.p; g2.ldc = w;
    gemm(ctx, g2);
    GemmDesc g3;  // E -= Y W2
    g3.M = ms; g3.N = nb; g3.K = w; g3.A = Yp; g3.lda = m; g3.B = W2.p; g3.ldb = w; g3.C = E; g3.ldc = ldb;
    g3.alpha = -1.0; g3.beta = 1.0;
    gemm(ctx, g3);
  }
}

void qrcp_init(tt_ctx ctx, QRCPState& st, double* Y, int64_t ldy, int64_t m, int64_t c) {
  (void)Y; (void)ldy;
  st.m = m;
  st.c = c;
  st.tau.alloc(ctx, (size_t)std::max<int64_t>(c, 1));
  st.norms.alloc(ctx, (size_t)2 * std::max<int64_t>(c, 1));
  st.perm.alloc(ctx, (size_t)2 * std::max<int64_t>(c, 1));  // second half: write-back scratch
  std::vector<int> ident((size_t)std::max<int64_t>(c, 1));
  for (int64_t j = 0; j < c; ++j) ident[(size_t)j] = (int)j;
  TTB_CUDA(cudaMemcpyAsync(st.perm.p, ident.data(), sizeof(int) * ident.size(), cudaMemcpyHostToDevice, ctx->stream));
  TTB_CUDA(cudaStreamSynchronize(ctx->stream));  // `ident` is pageable and local
  st.scalars.alloc(ctx, 2);
  st.k = 0;
  st.e2 = 0.0;
  st.cluster = -1;
}

void qrcp_run(tt_ctx ctx, QRCPState& st, double* Y, int64_t ldy, double stop2, int kcap) {
  // cluster-resident QRCP when the matrix fits the distributed shared memory of <= 16 CTAs
  if (st.cluster != 0) {
    const int kmax = (int)std::min<int64_t>(std::min(st.m, st.c), kcap);
    bool ok = true;
    while (ok) {
      ok = qrcp_cluster_run(ctx, Y, ldy, st.m, st.c, st.k, stop2, kcap, st.tau.p, st.perm.p, st.scalars.p);
      if (!ok) break;
      double h[2];
      d2h_small(ctx, h, st.scalars.p, 2);
      const int before = st.k;
      st.k = (int)h[0];
      st.e2 = h[1];
      st.cluster = 1;
      if (st.k >= kmax || st.e2 <= stop2 || st.k == before) return;  // else: step cap per launch hit
    }
    if (st.cluster == 1) fail(TT_ENOTSUP, "QRCP: cluster path lost mid-factorisation");
    st.cluster = 0;
  }
  // large panels (beyond one cluster): the grid-cooperative QRCP over every SM
  if (st.m * st.c >= (int64_t)1 << 17 &&
      qrcp_grid_run(ctx, Y, ldy, st.m, st.c, st.k, stop2, kcap, st.tau.p, st.norms.p, st.perm.p, st.scalars.p)) {
    double h[2];
    d2h_small(ctx, h, st.scalars.p, 2);
    st.k = (int)h[0];
    st.e2 = h[1];
    return;
  }
  const size_t smem = (size_t)st.c * (2 * sizeof(double) + sizeof(int)) + 16;
  if (smem > 200 * 1024) fail(TT_ENOTSUP, "QRCP: too many columns for the shared-memory norm cache");
  if (smem > 48 * 1024)  // idempotent and thread-safe (several contexts may run concurrently)
    TTB_CUDA(cudaFuncSetAttribute(qrcp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(200 * 1024 + 64)));
  TTB_RUN(ctx, "qrcp", 0, 16.0 * st.m * st.c,
          qrcp_kernel<<<1, 1024, smem, ctx->stream>>>(Y, ldy, (int)st.m, (int)st.c, st.k, stop2, kcap, st.tau.p, st.norms.p,
                                              st.perm.p, st.scalars.p));
  double h[2];
  d2h_small(ctx, h, st.scalars.p, 2);
  st.k = (int)h[0];
  st.e2 = h[1];
}

void apply_reflectors_left(tt_ctx ctx, const double* Y, int64_t ldy, const double* tau, int64_t m, int k,
                           double* target, int64_t ldt, int64_t nc) {
  if (k <= 0 || nc <= 0) return;
  if (m <= 16384) {  // one CTA per target column, the column in registers (<= 16 rows per thread)
    const bool big = m > 4096;  // 1024 threads (measured faster than 512 with twice the rows)
    const int T = big ? 1024 : 256;
    const int rpt = (int)ceil_div(m, T);
    auto kern = big ? (rpt <= 8 ? apply_reflectors_reg_kernel<1024, 8> : apply_reflectors_reg_kernel<1024, 16>)
              : rpt <= 2 ? apply_reflectors_reg_kernel<256, 2> : rpt <= 4 ? apply_reflectors_reg_kernel<256, 4>
              : rpt <= 8 ? apply_reflectors_reg_kernel<256, 8> : apply_reflectors_reg_kernel<256, 16>;
    TTB_RUN(ctx, "apply_reflectors", 4.0 * m * k * nc, 8.0 * (m * k + 2.0 * m * nc),
            kern<<<(unsigned)nc, T, 0, ctx->stream>>>(Y, ldy, tau, (int)m, k, target, ldt));
    return;
  }
  const size_t smem = sizeof(double) * (size_t)m;
  if (smem <= 200 * 1024) {  // one CTA per target column, the column in shared memory
    if (smem > 48 * 1024)
      TTB_CUDA(cudaFuncSetAttribute(apply_reflectors_col_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)(200 * 1024)));
    TTB_RUN(ctx, "apply_reflectors", 4.0 * m * k * nc, 8.0 * (m * k + 2.0 * m * nc),
            apply_reflectors_col_kernel<<<(unsigned)nc, 256, smem, ctx->stream>>>(Y, ldy, tau, (int)m, k, target, ldt));
    return;
  }
  TTB_RUN(ctx, "apply_reflectors", 4.0 * m * k * nc, 8.0 * (m * k + 2.0 * m * nc),
          apply_reflectors_kernel<<<1, 1024, 0, ctx->stream>>>(Y, ldy, tau, (int)m, k, target, ldt, (int)nc));
}

}  // namespace ttb
