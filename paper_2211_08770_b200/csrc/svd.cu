// Truncated SVD for the left-to-right TT-rounding sweep (FP64, sm_100a).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>

#include "gemm.cuh"
#include "qr.cuh"
#include "svd.cuh"
#include "ttops.cuh"

namespace ttb {

namespace {

constexpr int JAC_THREADS = 1024;
constexpr int JAC_MAX_SWEEPS = 60;

// One-sided (Hestenes) Jacobi with the round-robin (circle) ordering: every round has
// k/2 disjoint column pairs, one warp per pair.  Pairs rotate when
// |<a_p,a_q>| > tol sqrt(<a_p,a_p><a_q,a_q>), tol = sqrt(rows) u.
__global__ void __launch_bounds__(JAC_THREADS) jacobi_kernel(const double* __restrict__ Ain, int64_t lda, int rows,
                                                             int k, double* Ug, double* Vg, double* sig,
                                                             double* work, int use_smem, int* info) {
  extern __shared__ double sm[];
  double* A = use_smem ? sm : work;
  double* V = A + (int64_t)rows * k;
  double* nrm = V + (int64_t)k * k;
  __shared__ int rotated;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int64_t idx = tid; idx < (int64_t)rows * k; idx += blockDim.x) {
    const int64_t c = idx / rows, r = idx % rows;
    A[idx] = Ain[r + c * lda];
  }
  for (int64_t idx = tid; idx < (int64_t)k * k; idx += blockDim.x) V[idx] = (idx % k == idx / k) ? 1.0 : 0.0;
  __syncthreads();
  const double tol = sqrt((double)max(rows, 1)) * U_ROUND;
  const int kk = k + (k & 1);
  int sweep = 0;
  bool conv = (k < 2);
  for (; sweep < JAC_MAX_SWEEPS && !conv; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int r = 0; r < kk - 1; ++r) {
      for (int q = warp; q < kk / 2; q += nw) {
        int a, b;
        if (q == 0) { a = kk - 1; b = r; }
        else { a = (r + q) % (kk - 1); b = (r + kk - 1 - q) % (kk - 1); }
        if (a >= k || b >= k) continue;
        if (a > b) { const int t = a; a = b; b = t; }
        double* ca = A + (int64_t)a * rows;
        double* cb = A + (int64_t)b * rows;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < rows; i += 32) {
          const double x = ca[i], y = cb[i];
          al += x * x; be += y * y; ga += x * y;
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        if (ga != 0.0 && fabs(ga) > tol * sqrt(al) * sqrt(be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int i = lane; i < rows; i += 32) {
            const double x = ca[i], y = cb[i];
            ca[i] = c * x - s * y;
            cb[i] = s * x + c * y;
          }
          double* va = V + (int64_t)a * k;
          double* vb = V + (int64_t)b * k;
          for (int i = lane; i < k; i += 32) {
            const double x = va[i], y = vb[i];
            va[i] = c * x - s * y;
            vb[i] = s * x + c * y;
          }
          if (lane == 0) rotated = 1;
        }
      }
      __syncthreads();
    }
    conv = (rotated == 0);
    __syncthreads();
  }
  if (tid == 0) *info = conv ? 0 : 1;
  for (int j = warp; j < k; j += nw) {
    double s = 0.0;
    for (int i = lane; i < rows; i += 32) { const double x = A[(int64_t)j * rows + i]; s += x * x; }
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);
  }
  __syncthreads();
  for (int j = tid; j < k; j += blockDim.x) {
    const double v = nrm[j];
    int rank = 0;
    for (int i = 0; i < k; ++i) {
      const double w = nrm[i];
      if (w > v || (w == v && i < j)) ++rank;
    }
    sig[rank] = v;
    const double inv = v > 0.0 ? 1.0 / v : 0.0;
    for (int i = 0; i < rows; ++i) Ug[(int64_t)rank * rows + i] = A[(int64_t)j * rows + i] * inv;
    for (int i = 0; i < k; ++i) Vg[(int64_t)rank * k + i] = V[(int64_t)j * k + i];
  }
}

// The same Jacobi over the whole GPU for large k (C5: k ~ 1000, where one CTA would take
// seconds per SVD): cooperative launch, the k/2 disjoint pairs of a round dealt one per warp
// over the grid, one grid barrier per round; A and V in global memory (L2-resident).  Same
// ordering, threshold and rotation formulas as jacobi_kernel, so the result is identical.
constexpr int JG_T = 256;
__global__ void __launch_bounds__(JG_T) jacobi_grid_kernel(const double* __restrict__ Ain, int64_t lda, int rows,
                                                           int k, double* A, double* V, double* nrm, int* flags,
                                                           double* Ug, double* Vg, double* sig, int* info) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int64_t gtid = (int64_t)blockIdx.x * JG_T + threadIdx.x, nth = (int64_t)gridDim.x * JG_T;
  const int gw = (int)(gtid >> 5), nwg = (int)(nth >> 5);
  for (int64_t idx = gtid; idx < (int64_t)rows * k; idx += nth) {
    const int64_t c = idx / rows, r = idx % rows;
    A[idx] = Ain[r + c * lda];
  }
  for (int64_t idx = gtid; idx < (int64_t)k * k; idx += nth) V[idx] = (idx % k == idx / k) ? 1.0 : 0.0;
  grid.sync();
  const double tol = sqrt((double)max(rows, 1)) * U_ROUND;
  const int kk = k + (k & 1);
  int sweep = 0;
  bool conv = (k < 2);
  for (; sweep < JAC_MAX_SWEEPS && !conv; ++sweep) {
    for (int r = 0; r < kk - 1; ++r) {
      for (int q = gw; q < kk / 2; q += nwg) {
        int a, b;
        if (q == 0) { a = kk - 1; b = r; }
        else { a = (r + q) % (kk - 1); b = (r + kk - 1 - q) % (kk - 1); }
        if (a >= k || b >= k) continue;
        if (a > b) { const int t = a; a = b; b = t; }
        double* ca = A + (int64_t)a * rows;
        double* cb = A + (int64_t)b * rows;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < rows; i += 32) {
          const double x = ca[i], y = cb[i];
          al += x * x; be += y * y; ga += x * y;
        }
        al = warp_sum(al); be = warp_sum(be); ga = warp_sum(ga);
        if (ga != 0.0 && fabs(ga) > tol * sqrt(al) * sqrt(be)) {
          const double zeta = (be - al) / (2.0 * ga);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + hypot(1.0, zeta));
          const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
          for (int i = lane; i < rows; i += 32) {
            const double x = ca[i], y = cb[i];
            ca[i] = c * x - s * y;
            cb[i] = s * x + c * y;
          }
          double* va = V + (int64_t)a * k;
          double* vb = V + (int64_t)b * k;
          for (int i = lane; i < k; i += 32) {
            const double x = va[i], y = vb[i];
            va[i] = c * x - s * y;
            vb[i] = s * x + c * y;
          }
          if (lane == 0) flags[sweep] = 1;
        }
      }
      grid.sync();
    }
    conv = (flags[sweep] == 0);  // read after the sweep's last barrier: the same in every thread
  }
  if (gtid == 0) *info = conv ? 0 : 1;
  for (int j = gw; j < k; j += nwg) {
    double s = 0.0;
    for (int i = lane; i < rows; i += 32) { const double x = A[(int64_t)j * rows + i]; s += x * x; }
    s = warp_sum(s);
    if (lane == 0) nrm[j] = sqrt(s);
  }
  grid.sync();
  for (int j = gw; j < k; j += nwg) {  // one warp per column: rank, then U and V columns
    const double v = nrm[j];
    int rank = 0;
    for (int i = lane; i < k; i += 32) {
      const double w = nrm[i];
      if (w > v || (w == v && i < j)) ++rank;
    }
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (lane == 0) sig[rank] = v;
    const double inv = v > 0.0 ? 1.0 / v : 0.0;
    for (int i = lane; i < rows; i += 32) Ug[(int64_t)rank * rows + i] = A[(int64_t)j * rows + i] * inv;
    for (int i = lane; i < k; i += 32) Vg[(int64_t)rank * k + i] = V[(int64_t)j * k + i];
  }
}

// SV[j, perm[i]] = sigma[j] * B[i + j ldb]   (SV row-major rho x c)
__global__ void scale_unpermute_kernel(const double* __restrict__ B, int64_t ldb, const double* __restrict__ sigma,
                                       const int* __restrict__ perm, int c, int rho, double* SV) {
  const int64_t total = (int64_t)c * rho;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(idx % c), j = (int)(idx / c);
    SV[(int64_t)j * c + perm[i]] = sigma[j] * B[i + (int64_t)j * ldb];
  }
}

}  // namespace

void jacobi_svd(tt_ctx ctx, const double* A, int64_t lda, int64_t rows, int64_t k, double* U, double* V,
                double* sigma) {
  if (k <= 0) return;
  if (k >= 128) {  // whole-GPU Jacobi
    int per_sm = 0;
    TTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_grid_kernel, JG_T, 0));
    if (per_sm >= 1) {
      const int kk = (int)(k + (k & 1));
      const int G = std::max(1, std::min(ctx->num_sms * per_sm, (kk / 2 + JG_T / 32 - 1) / (JG_T / 32)));
      DBuf work(ctx, (size_t)(rows * k + k * k + k));
      IBuf flags(ctx, (size_t)JAC_MAX_SWEEPS + 1);
      TTB_CUDA(cudaMemsetAsync(flags.p, 0, sizeof(int) * (JAC_MAX_SWEEPS + 1), ctx->stream));
      double* Aw = work.p;
      double* Vw = work.p + rows * k;
      double* nw = Vw + k * k;
      int* fl = flags.p;
      int* inf = flags.p + JAC_MAX_SWEEPS;
      int ri = (int)rows, ki = (int)k;
      void* args[] = {(void*)&A, (void*)&lda, &ri, &ki, &Aw, &Vw, &nw, &fl, &U, &V, &sigma, &inf};
      TTB_RUN(ctx, "jacobi_svd", 0, 16.0 * rows * k,
              TTB_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_grid_kernel, dim3(G), dim3(JG_T), args, 0,
                                                   ctx->stream)));
      int h = 0;
      d2h_small_int(ctx, &h, inf, 1);
      if (h != 0) fail(TT_ENOCONV, "one-sided Jacobi SVD did not converge in " + std::to_string(JAC_MAX_SWEEPS) + " sweeps");
      return;
    }
  }
  const size_t need = sizeof(double) * (size_t)(rows * k + k * k + k);
  int use_smem = need <= 200 * 1024;
  DBuf work;
  size_t smem = 0;
  if (use_smem) {
    smem = need;
    if (smem > 48 * 1024)
      TTB_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  } else {
    work.alloc(ctx, (size_t)(rows * k + k * k + k));
  }
  IBuf info(ctx, 1);
  TTB_RUN(ctx, "jacobi_svd", 0, 16.0 * rows * k,
          jacobi_kernel<<<1, JAC_THREADS, smem, ctx->stream>>>(A, lda, (int)rows, (int)k, U, V, sigma, work.p, use_smem,
                                                       info.p));
  int h = 0;
  d2h_small_int(ctx, &h, info.p, 1);
  if (h != 0) fail(TT_ENOCONV, "one-sided Jacobi SVD did not converge in " + std::to_string(JAC_MAX_SWEEPS) + " sweeps");
}

TruncResult truncated_svd(tt_ctx ctx, const double* Y, int64_t m, int64_t c, double tau, bool keep_all,
                          int64_t max_rank, double stop_abs, DBuf& Ucore, DBuf& SV) {
  TruncResult res;
  const int64_t kq = std::min(m, c);
  DBuf Ycm(ctx, (size_t)m * c);
  transpose(ctx, Y, c, c, m, Ycm.p, m);  // row-major m x c -> column-major m x c
  if (keep_all && max_rank <= 0) {
    QRFactors f;
    geqrf(ctx, Ycm.p, m, m, c, f);
    DBuf Q(ctx, (size_t)m * kq), R(ctx, (size_t)kq * c);
    orgqr(ctx, f, Q.p, m);
    copy_upper(ctx, Ycm.p, m, kq, c, R.p, kq);
    Ucore.alloc(ctx, (size_t)m * kq);
    transpose(ctx, Q.p, m, m, kq, Ucore.p, kq);
    SV.alloc(ctx, (size_t)kq * c);
    transpose(ctx, R.p, kq, kq, c, SV.p, c);
    res.rho = kq;
    return res;
  }
  QRCPState st;
  qrcp_init(ctx, st, Ycm.p, m, m, c);
  double stop2 = keep_all ? -1.0 : stop_abs * stop_abs;
  qrcp_run(ctx, st, Ycm.p, m, stop2, (int)kq);
  if (st.k == 0) qrcp_run(ctx, st, Ycm.p, m, -1.0, 1);
  const double tau2 = tau * tau;
  std::vector<double> hs;
  DBuf QL, UJ, VJ, sig;
  int64_t rho = 0;
  for (;;) {
    const int64_t k = st.k;
    DBuf R1(ctx, (size_t)k * c), R1t(ctx, (size_t)c * k);
    copy_upper(ctx, Ycm.p, m, k, c, R1.p, k);
    transpose(ctx, R1.p, k, k, c, R1t.p, c);
    QRFactors fl;
    geqrf(ctx, R1t.p, c, c, k, fl);
    QL.alloc(ctx, (size_t)c * k);
    orgqr(ctx, fl, QL.p, c);
    DBuf RL(ctx, (size_t)k * k);
    copy_upper(ctx, R1t.p, c, k, k, RL.p, k);
    UJ.alloc(ctx, (size_t)k * k);
    VJ.alloc(ctx, (size_t)k * k);
    sig.alloc(ctx, (size_t)k);
    jacobi_svd(ctx, RL.p, k, k, k, UJ.p, VJ.p, sig.p);
    hs.assign((size_t)k, 0.0);
    d2h_small(ctx, hs.data(), sig.p, (size_t)k);
    std::vector<double> suf((size_t)k + 1, 0.0);  // suf[j] = sum_{i >= j} sigma_i^2, smallest first
    for (int64_t j = k - 1; j >= 0; --j) suf[(size_t)j] = suf[(size_t)j + 1] + hs[(size_t)j] * hs[(size_t)j];
    const double e2 = st.e2;
    if (keep_all) {
      rho = k;
      break;
    }
    rho = 0;
    for (int64_t r = 1; r <= k; ++r)
      if (suf[(size_t)r] + e2 <= tau2) { rho = r; break; }
    // exact decision test: tail^2(rho-1) lies in [suf[rho-1], suf[rho-1] + e2]
    const bool unresolved = (rho == 0) || (rho > 1 && e2 > 0.0 && suf[(size_t)rho - 1] <= tau2);
    if (unresolved && st.k < kq) {
      const int before = st.k;
      stop2 = (stop2 > 0.0) ? stop2 / 16.0 : stop2;
      qrcp_run(ctx, st, Ycm.p, m, stop2, (int)kq);
      if (st.k == before) qrcp_run(ctx, st, Ycm.p, m, -1.0, before + 1);
      res.resumes++;
      continue;
    }
    if (rho == 0) rho = k;
    break;
  }
  if (max_rank > 0) rho = std::min(rho, max_rank);
  rho = std::max<int64_t>(rho, 1);
  const int64_t k = st.k;
  res.rho = rho;
  res.qrcp_steps = k;
  // left vectors: Q_1 [V_J(:, :rho); 0]
  DBuf Ucm(ctx, (size_t)m * rho);
  TTB_CUDA(cudaMemsetAsync(Ucm.p, 0, sizeof(double) * (size_t)m * rho, ctx->stream));
  TTB_CUDA(cudaMemcpy2DAsync(Ucm.p, sizeof(double) * m, VJ.p, sizeof(double) * k, sizeof(double) * k, (size_t)rho,
                             cudaMemcpyDeviceToDevice, ctx->stream));
  apply_reflectors_left(ctx, Ycm.p, m, st.tau.p, m, (int)k, Ucm.p, m, rho);
  Ucore.alloc(ctx, (size_t)m * rho);
  transpose(ctx, Ucm.p, m, m, rho, Ucore.p, rho);
  // right factor: S_rho (Q_L U_J)(:, :rho)^T, columns un-permuted
  DBuf B(ctx, (size_t)c * rho);
  GemmDesc g;
  g.M = c; g.N = rho; g.K = k; g.A = QL.p; g.lda = c; g.B = UJ.p; g.ldb = k; g.C = B.p; g.ldc = c;
  gemm(ctx, g);
  SV.alloc(ctx, (size_t)rho * c);
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(c * rho, 256), 2048));
  TTB_RUN(ctx, "aux", 0, 16.0 * c * rho,
          scale_unpermute_kernel<<<blocks, 256, 0, ctx->stream>>>(B.p, c, sig.p, st.perm.p, (int)c, (int)rho, SV.p));
  return res;
}

}  // namespace ttb
