// Panel factorisation of the blocked Householder QR on ONE thread-block cluster (sm_100a):
// the m x w panel (w <= NB) lives in registers spread over a cluster of up to 16 CTAs
// (one row per thread); each Householder column costs ONE cluster-wide reduction.
//
// For column j every thread contributes x_r a_r[c] (x_r = a_r[j] for r >= j) to NB slots:
//   slot c > j : d_c = sum_{r>=j} a_r[j] a_r[c]      (gives v^T a_c = (d_c - beta a_j[c]) / (alpha - beta))
//   slot c < j : e_c = sum_{r>=j} a_r[j] v^(c)_r     (gives (V^T v_j)_c = (e_c - beta v^(c)_j) / (alpha - beta))
//   slot j     : sigma = sum_{r>j} a_r[j]^2          (LAPACK dlarfg: beta = -sign(alpha) sqrt(alpha^2 + sigma))
// so the norm, the trailing dot products and the T column all come out of one butterfly
// reduce-scatter per warp, one cross-warp pass and one all-to-all DSMEM exchange of the CTA
// partials (double-buffered, one cluster barrier per column).  CTA 0 also broadcasts row j.
// Output: explicit unit-lower Y (m x w), T (w x w, compact WY, dlarft recurrence), and R in
// the upper triangle of the panel's top w x w block (A = (I - Y T Y^T)[:, :w] R).
#include <cooperative_groups.h>

#include <algorithm>

#include "qr.cuh"

namespace cg = cooperative_groups;

namespace ttb {

namespace {

constexpr int MAX_CS = 16;

template <int NB>
__device__ __forceinline__ double selN(const double (&a)[NB], int j) {
  double r = 0.0;
#pragma unroll
  for (int c = 0; c < NB; ++c)
    if (c == j) r = a[c];
  return r;
}

template <int NB>
__device__ __forceinline__ void putN(double (&a)[NB], int j, double v) {
#pragma unroll
  for (int c = 0; c < NB; ++c)
    if (c == j) a[c] = v;
}

// butterfly reduce-scatter of NB (power of 2, <= 32) slots: lane l (l < NB) ends with the
// warp sum of slot l in p[0] (lanes l >= NB hold duplicates)
template <int NB>
__device__ __forceinline__ void reduce_scatter(double (&p)[NB], int lane) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (o >= NB) {  // more lanes than slots: plain butterfly sum at this level
#pragma unroll
      for (int i = 0; i < NB; ++i) p[i] += __shfl_xor_sync(0xffffffffu, p[i], o);
    } else {
      const bool hi = (lane & o) != 0;
#pragma unroll
      for (int i = 0; i < o; ++i) {
        const double send = hi ? p[i] : p[o + i];
        const double keep = hi ? p[o + i] : p[i];
        p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
  }
}

template <int NB, int NT>
__global__ void __launch_bounds__(NT, 1) panel_qr_cluster_kernel(double* A, int64_t lda, int m, int w, double* Y,
                                                                 int64_t ldy, double* T, int64_t ldt) {
  constexpr int NWARP = NT / 32;
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  __shared__ double part[2][MAX_CS][NB];  // CTA partial sums, from every CTA of the cluster
  __shared__ double rowj[2][NB];          // row j, broadcast by CTA 0
  __shared__ double red[NWARP][NB];
  __shared__ double fin[NB], fin2[NB];
  __shared__ double Ts[NB][NB + 1];
  __shared__ double rowloc[NB];
  const int base = m / CS, rem = m % CS;
  const int r0 = rank * base + min(rank, rem);
  const int h = base + (rank < rem ? 1 : 0);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int row = r0 + t;
  const bool live = t < h;
  double a[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c) a[c] = (live && c < w) ? A[(int64_t)row + (int64_t)c * lda] : 0.0;
  cluster.sync();  // every CTA is resident before the first DSMEM store
#pragma unroll 1
  for (int j = 0; j < w; ++j) {
    const int buf = j & 1;
    const double aj = selN<NB>(a, j);
    const double x = (live && row >= j) ? aj : 0.0;
    double pp[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) pp[c] = (c == j) ? ((row > j) ? x * x : 0.0) : x * a[c];
    reduce_scatter<NB>(pp, lane);
    if (lane < NB) red[warp][lane] = pp[0];
    if (rank == 0 && row == j) {
#pragma unroll
      for (int c = 0; c < NB; ++c) rowloc[c] = a[c];
    }
    __syncthreads();
    if (warp == 0 && lane < NB) {
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < NWARP; ++q) s += red[q][lane];
      for (int dst = 0; dst < CS; ++dst) {
        double* rp = cluster.map_shared_rank(&part[buf][rank][lane], dst);
        *rp = s;
        if (rank == 0) {
          double* rq = cluster.map_shared_rank(&rowj[buf][lane], dst);
          *rq = rowloc[lane];
        }
      }
    }
    cluster.sync();
    if (warp == 0) {
      double s = 0.0, rj = 0.0;
      if (lane < NB) {
        for (int src = 0; src < CS; ++src) s += part[buf][src][lane];  // fixed order: deterministic
        rj = rowj[buf][lane];
      }
      // every lane derives the reflector from slot j, then lane c forms its coefficient
      const double sigma_ = __shfl_sync(0xffffffffu, s, j);
      const double alpha_ = __shfl_sync(0xffffffffu, rj, j);
      double tj_ = 0.0, beta_ = alpha_, scal_ = 0.0;
      if (sigma_ != 0.0) {
        const double nrm = sqrt(alpha_ * alpha_ + sigma_);
        beta_ = alpha_ >= 0.0 ? -nrm : nrm;
        tj_ = (beta_ - alpha_) / beta_;
        scal_ = 1.0 / (alpha_ - beta_);
      }
      if (lane < NB) {
        const double z = (s - beta_ * rj) * scal_;  // c > j: v^T a_c ; c < j: (V^T v_j)_c
        fin[lane] = (lane > j) ? tj_ * z : z;       // trailing update coefficient tau w_c
      }
      if (lane == 0) { fin2[0] = beta_; fin2[1] = tj_; fin2[2] = scal_; }
    }
    __syncthreads();
    const double beta = fin2[0], tj = fin2[1], scal = fin2[2];
    const double v = (row > j) ? x * scal : (row == j ? 1.0 : 0.0);
    if (tj != 0.0) {
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c > j) a[c] -= v * fin[c];
    }
    if (live) putN<NB>(a, j, (row > j) ? v : (row == j ? beta : aj));
    // T column j (dlarft): T(j,j) = tau_j, T(0:j, j) = -tau_j T(0:j, 0:j) (V^T v_j)
    if (rank == 0 && warp == 1 && lane < NB) {
      const int i = lane;
      double acc = 0.0;
      if (i < j && tj != 0.0) {
        for (int k = i; k < j; ++k) acc += Ts[i][k] * fin[k];
        acc = -tj * acc;
      }
      Ts[i][j] = (i == j) ? tj : (i < j ? acc : 0.0);
    }
  }
  __syncthreads();
  if (live) {
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c < w) {
        Y[(int64_t)row + (int64_t)c * ldy] = (row > c) ? a[c] : (row == c ? 1.0 : 0.0);
        if (row < w) A[(int64_t)row + (int64_t)c * lda] = (c >= row) ? a[c] : 0.0;  // R
      }
    }
  }
  if (rank == 0) {
    for (int idx = t; idx < w * w; idx += NT) {
      const int c = idx / w, r = idx - c * w;
      T[r + (int64_t)c * ldt] = (r <= c) ? Ts[r][c] : 0.0;
    }
  }
  cluster.sync();  // no CTA leaves while DSMEM traffic to it may be in flight
}

template <int NB, int NT>
void launch_panel(tt_ctx ctx, double* A, int64_t lda, int64_t m, int w, double* Y, int64_t ldy, double* T,
                  int64_t ldt, int CS) {
  auto kern = panel_qr_cluster_kernel<NB, NT>;
  if (CS > 8) TTB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static const std::string cls = "panel_qr_cluster<" + std::to_string(NB) + "," + std::to_string(NT) + ">";
  TTB_RUN(ctx, cls.c_str(), 4.0 * m * w * w, 16.0 * m * w,
          TTB_CUDA(cudaLaunchKernelEx(&cfg, kern, A, lda, (int)m, w, Y, ldy, T, ldt)));
}

}  // namespace

int panel_cluster_max_rows(int w) { return w <= 16 ? 16 * 1024 : 16 * 512; }

// The smallest CTA that keeps the cluster within 16 CTAs: fewer rows per SM make each
// column step cheaper (the per-step cost is ~ rows-per-CTA issue slots + two barriers).
bool panel_qr_cluster(tt_ctx ctx, double* A, int64_t lda, int64_t m, int w, double* Y, int64_t ldy, double* T,
                      int64_t ldt) {
  if (w > 32) return false;
  if (m <= 16 * 128) {
    launch_panel<32, 128>(ctx, A, lda, m, w, Y, ldy, T, ldt, (int)ceil_div(m, 128));
  } else if (m <= 16 * 256) {
    launch_panel<32, 256>(ctx, A, lda, m, w, Y, ldy, T, ldt, (int)ceil_div(m, 256));
  } else if (m <= 16 * 512) {
    launch_panel<32, 512>(ctx, A, lda, m, w, Y, ldy, T, ldt, (int)ceil_div(m, 512));
  } else if (w <= 16 && m <= 16 * 1024) {
    launch_panel<16, 1024>(ctx, A, lda, m, w, Y, ldy, T, ldt, (int)ceil_div(m, 1024));
  } else {
    return false;
  }
  return true;
}

}  // namespace ttb
