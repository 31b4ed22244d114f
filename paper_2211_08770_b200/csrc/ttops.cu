// TT-vector kernels (FP64): in-kernel block-diagonal TT-sum access,
// batched TT inner products, elements X_1(i_1)...X_d(i_d),
// norms and small helpers.
#include <algorithm>
#include <cstdlib>

#include "gemm.cuh"
#include "ttops.cuh"

namespace ttb {

namespace {

struct TermTab {
  const double* ptr[MAXT];
  int64_t r0[MAXT], r1[MAXT], off0[MAXT], off1[MAXT];
  double coef[MAXT];
  int K;
};

int grid_for(int64_t n, int threads, int cap = 4096) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), cap));
}

// out[((off0+a) n + i) R1 + off1 + b] = c * X(a, i, b) for every term (block-diagonal TT-sum core)
__global__ void scatter_blocks_kernel(const __grid_constant__ TermTab tab, int64_t n, int64_t R1, bool use_coef,
                                      double* out) {
  const int l = blockIdx.y;
  const double* X = tab.ptr[l];
  const int64_t r0 = tab.r0[l], r1 = tab.r1[l];
  const int64_t total = r0 * n * r1;
  const double c = use_coef ? tab.coef[l] : 1.0;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx % r1, t = idx / r1;
    const int64_t i = t % n, a = t / n;
    out[((tab.off0[l] + a) * n + i) * R1 + tab.off1[l] + b] = c * X[idx];
  }
}

// A[i + (off0 + a) lda] = X_d(a, i)  (last core, r1 = 1)
__global__ void gather_last_kernel(const __grid_constant__ TermTab tab, int64_t n, double* A, int64_t lda) {
  const int l = blockIdx.y;
  const double* X = tab.ptr[l];
  const int64_t total = tab.r0[l] * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = idx / n, i = idx % n;
    A[i + (tab.off0[l] + a) * lda] = tab.coef[l] * X[idx];
  }
}

// M1[(off1 + b) + i R1] = c_l X_1(i, b)  (first core, r0 = 1)
__global__ void gather_first_kernel(const __grid_constant__ TermTab tab, int64_t n, double* M1, int64_t R1) {
  const int l = blockIdx.y;
  const double* X = tab.ptr[l];
  const int64_t r1 = tab.r1[l];
  const int64_t total = n * r1;
  const double c = tab.coef[l];
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / r1, b = idx % r1;
    M1[(tab.off1[l] + b) + i * R1] = c * X[idx];  // callers pass coef = 1 when c_l sits on the last core
  }
}

template <typename F>
void for_each_chunk(const std::vector<TermCore>& terms, F f) {
  for (size_t s = 0; s < terms.size(); s += MAXT) {
    TermTab tab{};
    tab.K = (int)std::min<size_t>(MAXT, terms.size() - s);
    int64_t maxe = 0;
    for (int l = 0; l < tab.K; ++l) {
      const TermCore& t = terms[s + l];
      tab.ptr[l] = t.ptr; tab.r0[l] = t.r0; tab.r1[l] = t.r1; tab.off0[l] = t.off0; tab.off1[l] = t.off1;
      tab.coef[l] = t.coef;
      maxe = std::max(maxe, t.r0 * t.r1);
    }
    f(tab, maxe);
  }
}

__global__ void transpose_kernel(const double* __restrict__ in, int64_t ldin, int rows, int cols, double* out,
                                 int64_t ldout) {
  __shared__ double tile[32][33];
  const int r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int r = r0 + threadIdx.x, c = c0 + j;
    if (r < rows && c < cols) tile[j][threadIdx.x] = in[r + (int64_t)c * ldin];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int c = c0 + threadIdx.x, r = r0 + j;
    if (r < rows && c < cols) out[c + (int64_t)r * ldout] = tile[threadIdx.x][j];
  }
}

__global__ void sumsq_partial_kernel(const double* __restrict__ x, int64_t n, double* part) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = x[i];
    s += v * v;
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_final_kernel(const double* __restrict__ part, int np, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) *out = s;
}

__global__ void scale_kernel(double* x, int64_t n, double a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) x[i] *= a;
}

struct LinTab {
  const double* x[MAXT];
  double c[MAXT];
  int K;
};

__global__ void lincomb_kernel(const __grid_constant__ LinTab tab, int64_t n, double* out, bool accumulate) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double s = accumulate ? out[i] : 0.0;
    for (int l = 0; l < tab.K; ++l) s += tab.c[l] * tab.x[l][i];
    out[i] = s;
  }
}

// ------------------------------------------------------------------ TT-dot
// One CTA per pair.  W_{k} = sum_i X_k(i)^T W_{k-1} Y_k(i) (row-major rx x ry), staged as
// T(a, i, c) = sum_b W(a, b) Y(b, i, c) over chunks of mode indices, then
// W'(a', c) += sum_{a, i} X(a, i, a') T(a, i, c).  Fixed summation order (deterministic).
__global__ void __launch_bounds__(256) dot_kernel(int d, const int64_t* __restrict__ n,
                                                  const double* const* __restrict__ xc,
                                                  const double* const* __restrict__ yc,
                                                  const int64_t* __restrict__ xr, const int64_t* __restrict__ yr,
                                                  double* out, double* scratch, int64_t wcap, int64_t tcap,
                                                  int use_smem, double* traces) {
  extern __shared__ double sm[];
  const int p = blockIdx.x;
  double* base = use_smem ? sm : scratch + (int64_t)p * (2 * wcap + tcap);
  double* W = base;
  double* Wn = base + wcap;
  double* T = base + 2 * wcap;
  const int tid = threadIdx.x;
  if (tid == 0) W[0] = 1.0;
  __syncthreads();
  for (int k = 0; k < d; ++k) {
    const int64_t nk = n[k];
    const int64_t rx0 = xr[(int64_t)p * (d + 1) + k], rx1 = xr[(int64_t)p * (d + 1) + k + 1];
    const int64_t ry0 = yr[(int64_t)p * (d + 1) + k], ry1 = yr[(int64_t)p * (d + 1) + k + 1];
    const double* __restrict__ X = xc[(int64_t)p * d + k];
    const double* __restrict__ Y = yc[(int64_t)p * d + k];
    for (int64_t idx = tid; idx < rx1 * ry1; idx += blockDim.x) Wn[idx] = 0.0;
    const int64_t rr = rx0 * ry1 > 0 ? rx0 * ry1 : 1;
    const int64_t ic = tcap / rr > 0 ? tcap / rr : 1;
    for (int64_t i0 = 0; i0 < nk; i0 += ic) {
      const int64_t ni = (ic < nk - i0) ? ic : (nk - i0);
      for (int64_t idx = tid; idx < rx0 * ni * ry1; idx += blockDim.x) {
        const int64_t c = idx % ry1, t = idx / ry1;
        const int64_t ii = t % ni, a = t / ni;
        double s = 0.0;
        for (int64_t b = 0; b < ry0; ++b) s += W[a * ry0 + b] * Y[(b * nk + i0 + ii) * ry1 + c];
        T[idx] = s;
      }
      __syncthreads();
      for (int64_t idx = tid; idx < rx1 * ry1; idx += blockDim.x) {
        const int64_t c = idx % ry1, a1 = idx / ry1;
        double s = 0.0;
        for (int64_t a = 0; a < rx0; ++a)
          for (int64_t ii = 0; ii < ni; ++ii) s += X[(a * nk + i0 + ii) * rx1 + a1] * T[(a * ni + ii) * ry1 + c];
        Wn[idx] += s;
      }
      __syncthreads();
    }
    double* tmp = W;
    W = Wn;
    Wn = tmp;
    if (traces && tid == 0) {  // x == y: trace(W_k) = ||left part through core k||_F^2
      double tr = 0.0;
      for (int64_t a = 0; a < rx1 && a < ry1; ++a) tr += W[a * ry1 + a];
      traces[(int64_t)p * (d + 1) + k + 1] = tr;
    }
  }
  if (tid == 0) {
    out[p] = W[0];
    if (traces) traces[(int64_t)p * (d + 1)] = 1.0;
  }
}

__global__ void __launch_bounds__(256) element_kernel(int d, const int64_t* __restrict__ n,
                                                      const double* const* __restrict__ core,
                                                      const int64_t* __restrict__ r, const int64_t* __restrict__ idx,
                                                      double* out, double* scratch, int64_t rmax, int use_smem) {
  extern __shared__ double sm[];
  const int t = blockIdx.x;
  double* v = use_smem ? sm : scratch + (int64_t)t * 2 * rmax;
  double* vn = v + rmax;
  if (threadIdx.x == 0) v[0] = 1.0;
  __syncthreads();
  for (int k = 0; k < d; ++k) {
    const int64_t i = idx[(int64_t)t * d + k], r0 = r[k], r1 = r[k + 1], nk = n[k];
    const double* X = core[k];
    for (int64_t b = threadIdx.x; b < r1; b += blockDim.x) {
      double s = 0.0;
      for (int64_t a = 0; a < r0; ++a) s += v[a] * X[(a * nk + i) * r1 + b];
      vn[b] = s;
    }
    __syncthreads();
    double* tmp = v;
    v = vn;
    vn = tmp;
  }
  if (threadIdx.x == 0) out[t] = v[0];
}

}  // namespace

void gather_last(tt_ctx ctx, const std::vector<TermCore>& terms, int64_t n, double* A, int64_t lda) {
  for_each_chunk(terms, [&](const TermTab& tab, int64_t maxe) {
    dim3 grid(grid_for(maxe * n, 256, 1024), tab.K);
    TTB_RUN(ctx, "tt_sum_gather", 0, 16.0 * maxe * n * tab.K,
            gather_last_kernel<<<grid, 256, 0, ctx->stream>>>(tab, n, A, lda));
  });
}

void gather_first(tt_ctx ctx, const std::vector<TermCore>& terms, int64_t n, double* M1, int64_t R1) {
  for_each_chunk(terms, [&](const TermTab& tab, int64_t maxe) {
    dim3 grid(grid_for(maxe * n, 256, 1024), tab.K);
    TTB_RUN(ctx, "tt_sum_gather", 0, 16.0 * maxe * n * tab.K,
            gather_first_kernel<<<grid, 256, 0, ctx->stream>>>(tab, n, M1, R1));
  });
}

void materialise_core(tt_ctx ctx, const std::vector<TermCore>& terms, int64_t n, int64_t R0, int64_t R1, bool first,
                      bool last, double* out) {
  (void)last;
  TTB_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)(R0 * n * R1), ctx->stream));
  for_each_chunk(terms, [&](const TermTab& tab, int64_t maxe) {
    dim3 grid(grid_for(maxe * n, 256, 1024), tab.K);
    TTB_RUN(ctx, "tt_sum_gather", 0, 16.0 * maxe * n * tab.K,
            scatter_blocks_kernel<<<grid, 256, 0, ctx->stream>>>(tab, n, R1, first, out));
  });
}

void transpose(tt_ctx ctx, const double* in, int64_t ldin, int64_t rows, int64_t cols, double* out, int64_t ldout) {
  if (rows <= 0 || cols <= 0) return;
  dim3 grid((unsigned)ceil_div(rows, 32), (unsigned)ceil_div(cols, 32)), block(32, 8);
  TTB_RUN(ctx, "aux", 0, 16.0 * rows * cols,
          transpose_kernel<<<grid, block, 0, ctx->stream>>>(in, ldin, (int)rows, (int)cols, out, ldout));
}

void sumsq(tt_ctx ctx, const double* x, int64_t n, double* out_dev) {
  const int nb = grid_for(n, 256, 512);
  DBuf part(ctx, nb);
  TTB_RUN(ctx, "aux", 2.0 * n, 8.0 * n, sumsq_partial_kernel<<<nb, 256, 0, ctx->stream>>>(x, n, part.p));
  TTB_RUN(ctx, "aux", nb, 8.0 * nb, sum_final_kernel<<<1, 256, 0, ctx->stream>>>(part.p, nb, out_dev));
}

void scale_inplace(tt_ctx ctx, double* x, int64_t n, double alpha) {
  if (n <= 0) return;
  TTB_RUN(ctx, "aux", n, 16.0 * n, scale_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(x, n, alpha));
}

void copy_d2d(tt_ctx ctx, double* y, const double* x, int64_t n) {
  if (n <= 0) return;
  TTB_CUDA(cudaMemcpyAsync(y, x, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, ctx->stream));
}

void lincomb(tt_ctx ctx, const std::vector<const double*>& xs, const std::vector<double>& coef, int64_t n, double* out) {
  for (size_t s = 0; s < xs.size(); s += MAXT) {
    LinTab tab{};
    tab.K = (int)std::min<size_t>(MAXT, xs.size() - s);
    for (int l = 0; l < tab.K; ++l) { tab.x[l] = xs[s + l]; tab.c[l] = coef[s + l]; }
    TTB_RUN(ctx, "aux", 2.0 * n * tab.K, 8.0 * n * (tab.K + 1),
            lincomb_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(tab, n, out, s > 0));
  }
}

namespace {

// Y_k((a, alpha), i, (b, beta)) = sum_j A_k(a, i, j, b) X_k(alpha, j, beta): one thread per output
// element (a short sum over the n column indices; the operator cores are tiny and L1-resident).
__global__ void matvec_core_kernel(const double* __restrict__ Ak, const double* __restrict__ Xk, int ra0, int ra1,
                                   int rx0, int rx1, int n, double* __restrict__ Yk) {
  const int64_t r1 = (int64_t)ra1 * rx1;
  const int64_t total = (int64_t)ra0 * rx0 * n * r1;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c1 = idx % r1, t = idx / r1;
    const int i = (int)(t % n);
    const int64_t c0 = t / n;
    const int a = (int)(c0 / rx0), al = (int)(c0 % rx0), b = (int)(c1 / rx1), be = (int)(c1 % rx1);
    const double* ap = Ak + (((int64_t)a * n + i) * n) * ra1 + b;  // A_k(a, i, j, b), j stride ra1
    const double* xp = Xk + (int64_t)al * n * rx1 + be;             // X_k(alpha, j, beta), j stride rx1
    double s = 0.0;
    for (int j = 0; j < n; ++j) s += ap[(int64_t)j * ra1] * xp[(int64_t)j * rx1];
    Yk[idx] = s;
  }
}

}  // namespace

tt_tensor matvec(tt_ctx ctx, int d, const std::vector<int64_t>& n, const std::vector<int64_t>& ra,
                 const std::vector<const double*>& acore, const std::vector<int64_t>& rx,
                 const std::vector<const double*>& xcore) {
  std::vector<int64_t> ry((size_t)d + 1);
  for (int k = 0; k <= d; ++k) ry[(size_t)k] = ra[(size_t)k] * rx[(size_t)k];
  tt_tensor y = tensor_alloc(ctx, d, n, ry);
  for (int k = 0; k < d; ++k) {
    const int64_t total = ry[(size_t)k] * n[(size_t)k] * ry[(size_t)k + 1];
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 4096));
    TTB_RUN(ctx, "tt_matvec", 2.0 * total * n[(size_t)k],
            8.0 * (total + ra[(size_t)k] * n[(size_t)k] * n[(size_t)k] * ra[(size_t)k + 1] +
                   rx[(size_t)k] * n[(size_t)k] * rx[(size_t)k + 1]),
            matvec_core_kernel<<<blocks, 256, 0, ctx->stream>>>(
                acore[(size_t)k], xcore[(size_t)k], (int)ra[(size_t)k], (int)ra[(size_t)k + 1], (int)rx[(size_t)k],
                (int)rx[(size_t)k + 1], (int)n[(size_t)k], y->core[(size_t)k]));
  }
  return y;
}

namespace {

// Z_k((a, c), i, (b, e)) = X_k(a, i, b) Y_k(c, i, e): the slices' Kronecker product (elementwise
// product of the two tensors), one thread per output element.
__global__ void hadamard_core_kernel(const double* __restrict__ Xk, const double* __restrict__ Yk, int rx0, int rx1,
                                     int ry0, int ry1, int n, double* __restrict__ Zk) {
  const int64_t r1 = (int64_t)rx1 * ry1;
  const int64_t total = (int64_t)rx0 * ry0 * n * r1;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c1 = idx % r1, t = idx / r1;
    const int i = (int)(t % n);
    const int64_t c0 = t / n;
    const int a = (int)(c0 / ry0), c = (int)(c0 % ry0), b = (int)(c1 / ry1), e = (int)(c1 % ry1);
    Zk[idx] = Xk[((int64_t)a * n + i) * rx1 + b] * Yk[((int64_t)c * n + i) * ry1 + e];
  }
}

}  // namespace

tt_tensor hadamard(tt_ctx ctx, int d, const std::vector<int64_t>& n, const std::vector<int64_t>& rx,
                   const std::vector<const double*>& xc, const std::vector<int64_t>& ry,
                   const std::vector<const double*>& yc) {
  std::vector<int64_t> rz((size_t)d + 1);
  for (int k = 0; k <= d; ++k) rz[(size_t)k] = rx[(size_t)k] * ry[(size_t)k];
  tt_tensor z = tensor_alloc(ctx, d, n, rz);
  for (int k = 0; k < d; ++k) {
    const int64_t total = rz[(size_t)k] * n[(size_t)k] * rz[(size_t)k + 1];
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(total, 256), 4096));
    TTB_RUN(ctx, "tt_hadamard", (double)total, 24.0 * total,
            hadamard_core_kernel<<<blocks, 256, 0, ctx->stream>>>(
                xc[(size_t)k], yc[(size_t)k], (int)rx[(size_t)k], (int)rx[(size_t)k + 1], (int)ry[(size_t)k],
                (int)ry[(size_t)k + 1], (int)n[(size_t)k], z->core[(size_t)k]));
  }
  return z;
}

namespace {

__global__ void dot_init_kernel(double* W, const int64_t* __restrict__ wo, int P) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) W[wo[p]] = 1.0;
}
__global__ void dot_out_kernel(const double* W, const int64_t* __restrict__ wo, int P, double* out) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) out[p] = W[wo[p]];
}
// traces[p (d+1) + k + 1] = trace(W_p) (rx1 x ry1, ld rx1), one warp per pair
__global__ void dot_trace_kernel(const double* W, const int64_t* __restrict__ wo, const int64_t* __restrict__ xr,
                                 const int64_t* __restrict__ yr, int d, int k, int P, double* traces) {
  const int p = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
  if (p >= P) return;
  const int64_t rx1 = xr[(int64_t)p * (d + 1) + k + 1], ry1 = yr[(int64_t)p * (d + 1) + k + 1];
  const int64_t nd = rx1 < ry1 ? rx1 : ry1;
  double t = 0.0;
  for (int64_t a = lane; a < nd; a += 32) t += W[wo[p] + a + a * rx1];
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) {
    traces[(int64_t)p * (d + 1) + k + 1] = t;
    if (k == 0) traces[(int64_t)p * (d + 1)] = 1.0;
  }
}

}  // namespace

// Large ranks: the per-core recursion of every pair as two grouped DMMA GEMMs per core (gemm.cu),
// W (rx_k x ry_k, column-major) -> S^T = X_k^T W  (rows (i, a'), columns b: M = n rx1, K = rx0,
// N = ry0) -> W' = S Y_k with K = (b, i) (M = rx1, N = ry1): both products read the cores in
// place (no transposes), O(n rx ry (rx + ry)) flops per core on the tensor pipe.
void dot_batch_gemm(tt_ctx ctx, const DotBatch& b, double* out_dev, double* traces_dev) {
  const int d = b.d, P = b.P;
  if (P <= 0) return;
  // per-pair workspace: W (max rx_k ry_k) and S^T (max n_k rx_{k+1} ry_k), exact offsets; pairs
  // are processed in groups of <= 2 GiB of workspace
  std::vector<int64_t> wsz((size_t)P), ssz((size_t)P);
  for (int p = 0; p < P; ++p) {
    int64_t w = 1, sc = 1;
    for (int k = 0; k < d; ++k) {
      const int64_t rx0 = b.xr[(size_t)p * (d + 1) + k], rx1 = b.xr[(size_t)p * (d + 1) + k + 1];
      const int64_t ry0 = b.yr[(size_t)p * (d + 1) + k], ry1 = b.yr[(size_t)p * (d + 1) + k + 1];
      w = std::max(w, std::max(rx0 * ry0, rx1 * ry1));
      sc = std::max(sc, b.n[(size_t)k] * rx1 * ry0);
    }
    wsz[(size_t)p] = (w + 1) & ~int64_t(1);  // 16-byte aligned blocks
    ssz[(size_t)p] = (sc + 1) & ~int64_t(1);
  }
  const int64_t budget = (int64_t)1 << 28;  // doubles (2 GiB)
  std::vector<GemmDesc> g1, g2;
  for (int p0 = 0; p0 < P;) {
    int p1 = p0;
    int64_t wt = 0, st = 0;
    while (p1 < P && (p1 == p0 || wt + st + wsz[(size_t)p1] + ssz[(size_t)p1] <= budget)) {
      wt += wsz[(size_t)p1];
      st += ssz[(size_t)p1];
      ++p1;
    }
    const int Pg = p1 - p0;
    std::vector<int64_t> wo((size_t)Pg), so((size_t)Pg);
    int64_t a0 = 0, b0 = 0;
    for (int q = 0; q < Pg; ++q) { wo[(size_t)q] = a0; so[(size_t)q] = b0; a0 += wsz[(size_t)(p0 + q)]; b0 += ssz[(size_t)(p0 + q)]; }
    DBuf W(ctx, (size_t)wt), S(ctx, (size_t)st);
    BBuf dxr, dyr;
    if (traces_dev) {
      dxr.upload(ctx, b.xr.data() + (size_t)p0 * (d + 1), sizeof(int64_t) * (size_t)Pg * (d + 1));
      dyr.upload(ctx, b.yr.data() + (size_t)p0 * (d + 1), sizeof(int64_t) * (size_t)Pg * (d + 1));
    }
    BBuf dwo;
    dwo.upload(ctx, wo.data(), sizeof(int64_t) * wo.size());
    TTB_RUN(ctx, "aux", 0, 8.0 * Pg,  // W_0 = 1 (1 x 1) for every pair
            dot_init_kernel<<<(Pg + 127) / 128, 128, 0, ctx->stream>>>(W.p, (const int64_t*)dwo.p, Pg));
    for (int k = 0; k < d; ++k) {
      const int64_t n = b.n[(size_t)k];
      g1.clear();
      g2.clear();
      for (int q = 0; q < Pg; ++q) {
        const int p = p0 + q;
        const int64_t rx0 = b.xr[(size_t)p * (d + 1) + k], rx1 = b.xr[(size_t)p * (d + 1) + k + 1];
        const int64_t ry0 = b.yr[(size_t)p * (d + 1) + k], ry1 = b.yr[(size_t)p * (d + 1) + k + 1];
        const double* X = b.xc[(size_t)p * d + k];
        const double* Y = b.yc[(size_t)p * d + k];
        double* Wp = W.p + wo[(size_t)q];
        double* Sp = S.p + so[(size_t)q];
        GemmDesc a;  // S^T (n rx1 x ry0, ld n rx1) = X^T (n rx1 x rx0, ld n rx1) W (rx0 x ry0, ld rx0)
        a.M = n * rx1; a.N = ry0; a.K = rx0;
        a.A = X; a.lda = n * rx1;
        a.B = Wp; a.ldb = rx0;
        a.C = Sp; a.ldc = n * rx1;
        g1.push_back(a);
        GemmDesc c;  // W' (rx1 x ry1, ld rx1) = S (rx1 x (ry0 n), ld rx1) Y ((ry0 n) x ry1, stored ry1 x (ry0 n))
        c.M = rx1; c.N = ry1; c.K = ry0 * n;
        c.A = Sp; c.lda = rx1;
        c.B = Y; c.ldb = ry1; c.tb = true;
        c.C = Wp; c.ldc = rx1;
        g2.push_back(c);
      }
      gemm_grouped(ctx, g1);
      gemm_grouped(ctx, g2);
      if (traces_dev)
        TTB_RUN(ctx, "aux", 0, 8.0 * Pg, dot_trace_kernel<<<(Pg + 7) / 8, 256, 0, ctx->stream>>>(
                                             W.p, (const int64_t*)dwo.p, (const int64_t*)dxr.p, (const int64_t*)dyr.p,
                                             d, k, Pg, traces_dev + (int64_t)p0 * (d + 1)));
    }
    TTB_RUN(ctx, "aux", 0, 16.0 * Pg,
            dot_out_kernel<<<(Pg + 127) / 128, 128, 0, ctx->stream>>>(W.p, (const int64_t*)dwo.p, Pg, out_dev + p0));
    p0 = p1;
  }
}

void dot_batch(tt_ctx ctx, const DotBatch& b, double* out_dev, double* traces_dev) {
  if (b.P <= 0) return;
  static const bool pairwise = std::getenv("TT_B200_DOT_PAIRWISE") != nullptr;
  // Route: per-core grouped DMMA GEMMs when a pair's recursion is long enough to amortise two
  // launches per core (one CTA per pair runs at ~15 GFLOP/s; a grouped launch costs ~10 us):
  // flops per pair > 0.3 MFLOP x d, or ranks beyond the one-CTA workspace (> 32).
  int64_t rmax = 1;
  double fl_pair = 0.0;
  for (int p = 0; p < b.P; ++p) {
    double f = 0.0;
    for (int k = 0; k < b.d; ++k) {
      const double rx0 = (double)b.xr[(size_t)p * (b.d + 1) + k], rx1 = (double)b.xr[(size_t)p * (b.d + 1) + k + 1];
      const double ry0 = (double)b.yr[(size_t)p * (b.d + 1) + k], ry1 = (double)b.yr[(size_t)p * (b.d + 1) + k + 1];
      f += 2.0 * b.n[(size_t)k] * (rx0 * ry0 * ry1 + rx0 * rx1 * ry1);
    }
    fl_pair = std::max(fl_pair, f);
  }
  for (int64_t v : b.xr) rmax = std::max(rmax, v);
  for (int64_t v : b.yr) rmax = std::max(rmax, v);
  if (!pairwise && (rmax > 32 || fl_pair > 0.3e6 * b.d)) {
    dot_batch_gemm(ctx, b, out_dev, traces_dev);
    return;
  }
  const int d = b.d;
  int64_t wcap = 1, tcap = 1;
  for (int p = 0; p < b.P; ++p)
    for (int k = 0; k <= d; ++k) wcap = std::max(wcap, b.xr[(size_t)p * (d + 1) + k] * b.yr[(size_t)p * (d + 1) + k]);
  for (int p = 0; p < b.P; ++p)
    for (int k = 0; k < d; ++k)
      tcap = std::max(tcap, b.xr[(size_t)p * (d + 1) + k] * b.yr[(size_t)p * (d + 1) + k + 1]);
  tcap = std::min<int64_t>(std::max<int64_t>(tcap, 1) * 8, std::max<int64_t>(tcap, 8192));
  BBuf dn, dxc, dyc, dxr, dyr;
  dn.upload(ctx, b.n.data(), sizeof(int64_t) * d);
  dxc.upload(ctx, b.xc.data(), sizeof(double*) * b.xc.size());
  dyc.upload(ctx, b.yc.data(), sizeof(double*) * b.yc.size());
  dxr.upload(ctx, b.xr.data(), sizeof(int64_t) * b.xr.size());
  dyr.upload(ctx, b.yr.data(), sizeof(int64_t) * b.yr.size());
  // algorithmic work: 2 n (rx0 ry0 ry1 + rx0 rx1 ry1) per pair and core; bytes = cores read once
  double dot_flops = 0.0, dot_bytes = 0.0;
  for (int p = 0; p < b.P; ++p)
    for (int k = 0; k < d; ++k) {
      const double rx0 = (double)b.xr[(size_t)p * (d + 1) + k], rx1 = (double)b.xr[(size_t)p * (d + 1) + k + 1];
      const double ry0 = (double)b.yr[(size_t)p * (d + 1) + k], ry1 = (double)b.yr[(size_t)p * (d + 1) + k + 1];
      dot_flops += 2.0 * b.n[(size_t)k] * (rx0 * ry0 * ry1 + rx0 * rx1 * ry1);
      dot_bytes += 8.0 * b.n[(size_t)k] * (rx0 * rx1 + ry0 * ry1);
    }
  size_t smem = sizeof(double) * (size_t)(2 * wcap + tcap);
  int use_smem = smem <= 200 * 1024;
  DBuf scratch;
  if (!use_smem) {
    tcap = std::max<int64_t>(tcap, 1);
    scratch.alloc(ctx, (size_t)b.P * (2 * wcap + tcap));
    smem = 0;
  } else if (smem > 48 * 1024) {
    TTB_CUDA(cudaFuncSetAttribute(dot_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  TTB_RUN(ctx, "tt_dot", dot_flops, dot_bytes,
          dot_kernel<<<b.P, 256, smem, ctx->stream>>>(d, (const int64_t*)dn.p, (const double* const*)dxc.p,
                                              (const double* const*)dyc.p, (const int64_t*)dxr.p,
                                              (const int64_t*)dyr.p, out_dev, scratch.p, wcap, tcap, use_smem,
                                              traces_dev));
}

void elements(tt_ctx ctx, int d, const std::vector<int64_t>& n, const std::vector<const double*>& core,
              const std::vector<int64_t>& r, const std::vector<int64_t>& idx, int nidx, double* out_dev) {
  if (nidx <= 0) return;
  int64_t rmax = 1;
  for (int64_t v : r) rmax = std::max(rmax, v);
  BBuf dn, dc, dr, di;
  dn.upload(ctx, n.data(), sizeof(int64_t) * d);
  dc.upload(ctx, core.data(), sizeof(double*) * d);
  dr.upload(ctx, r.data(), sizeof(int64_t) * (d + 1));
  di.upload(ctx, idx.data(), sizeof(int64_t) * idx.size());
  size_t smem = sizeof(double) * 2 * (size_t)rmax;
  int use_smem = smem <= 48 * 1024;
  DBuf scratch;
  if (!use_smem) {
    scratch.alloc(ctx, (size_t)nidx * 2 * rmax);
    smem = 0;
  }
  TTB_RUN(ctx, "tt_element", 2.0 * nidx * rmax * rmax * d, 8.0 * nidx * rmax * rmax * d,
          element_kernel<<<nidx, 256, smem, ctx->stream>>>(d, (const int64_t*)dn.p, (const double* const*)dc.p,
                                                   (const int64_t*)dr.p, (const int64_t*)di.p, out_dev, scratch.p, rmax,
                                                   use_smem));
}

}  // namespace ttb
