// Householder QR with column pivoting held entirely in the shared memory of ONE thread-block
// cluster (sm_100a, up to 16 CTAs, distributed shared memory).  Used by the rank-revealing
// right-to-left orthogonalisation and by the truncated SVD of the left-to-right sweep.
//
// CTA q owns a contiguous block of the c columns (all m rows) in its shared memory.  Per
// Householder step s:
//   A  every CTA reduces its active columns' trailing mass and its best pivot candidate and
//      writes them into every CTA's slot (DSMEM), one cluster barrier;
//   B  all CTAs take the same decision (stop when the trailing Frobenius mass <= stop2; exact
//      norm recomputation before deciding near the threshold, LAPACK dlaqp2 style), the owner of
//      the pivot column forms the reflector (dlarfg) and broadcasts v and tau into every CTA
//      (double-buffered), one cluster barrier;
//   C  every CTA applies the reflector to its active columns and downdates their norms.
// Columns are never moved during the loop; the pivot order is replicated in every CTA and the
// final write-back puts pivoted columns at positions k_start.. and the rest after them, so the
// global layout equals the one of an explicitly swapping QRCP (qrcp_kernel in qr.cu).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "qr.cuh"

namespace cg = cooperative_groups;

namespace ttb {

namespace {

constexpr int QC_THREADS = 512;
constexpr int QC_MAXCS = 16;
constexpr int QC_SMEM = 200 * 1024;  // dynamic shared memory per CTA
constexpr int QC_MAXSTEPS = 512;     // pivots per launch

struct Cand {
  double mass, val;
  int pos;
  int pad;
};

__device__ __forceinline__ bool better(double v, int p, double bv, int bp) { return v > bv || (v == bv && p < bp); }

__global__ void __launch_bounds__(QC_THREADS, 1) qrcp_cluster_kernel(double* Y, int64_t ldy, int m, int c, int k_start,
                                                                     double stop2, int kcap, double* tau_g,
                                                                     int* perm_g, double* scalars) {
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks();
  const int rank = (int)cluster.block_rank();
  extern __shared__ double smem[];
  __shared__ Cand slot[2][QC_MAXCS];
  __shared__ double slot2[QC_MAXCS];
  __shared__ double taus[2];
  __shared__ int piv_pos[QC_MAXSTEPS];
  __shared__ double red[32];
  __shared__ Cand wbest[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = QC_THREADS / 32;
  // columns [g0, g0 + cq) of positions k_start..c-1 belong to this CTA
  const int act = c - k_start;
  const int base = act / CS, rem = act % CS;
  const int g0 = k_start + rank * base + min(rank, rem);
  const int cq = base + (rank < rem ? 1 : 0);
  // vb first: it is written remotely, so its offset must not depend on this CTA's cq
  double* vb = smem;                             // 2 x m reflector buffers
  double* A = vb + 2 * (size_t)m;                // m x cq, column-major (ld m)
  double* nrm = A + (size_t)m * cq;              // cq
  double* nrm0 = nrm + cq;                       // cq
  int* flag = reinterpret_cast<int*>(nrm0 + cq); // cq: 1 = active
  for (int64_t idx = tid; idx < (int64_t)m * cq; idx += QC_THREADS) {
    const int jl = (int)(idx / m), r = (int)(idx % m);
    A[idx] = Y[(int64_t)r + (int64_t)(g0 + jl) * ldy];
  }
  __syncthreads();
  // exact trailing norms (rows >= k_start)
  for (int jl = warp; jl < cq; jl += NW) {
    double q = 0.0;
    for (int r = k_start + lane; r < m; r += 32) { const double v = A[(int64_t)jl * m + r]; q += v * v; }
    q = warp_sum(q);
    if (lane == 0) { nrm[jl] = q; nrm0[jl] = q; flag[jl] = 1; }
  }
  cluster.sync();  // all CTAs loaded (global reads done) and resident for DSMEM
  const int kmax = min(min(m, c), kcap);
  int s = k_start;
  int nsteps = 0;
#pragma unroll 1
  for (; s < kmax && nsteps < QC_MAXSTEPS; ++s, ++nsteps) {
    const int buf = s & 1;
    // ---- A: local mass and best candidate
    double mass = 0.0, bv = -1.0;
    int bp = 0x7fffffff;
    for (int jl = tid; jl < cq; jl += QC_THREADS) {
      if (flag[jl]) {
        const double v = nrm[jl];
        mass += v;
        if (better(v, g0 + jl, bv, bp)) { bv = v; bp = g0 + jl; }
      }
    }
    mass = warp_sum(mass);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int op = __shfl_xor_sync(0xffffffffu, bp, o);
      if (better(ov, op, bv, bp)) { bv = ov; bp = op; }
    }
    if (lane == 0) { Cand cd; cd.mass = mass; cd.val = bv; cd.pos = bp; cd.pad = 0; wbest[warp] = cd; }
    __syncthreads();
    if (warp == 0) {
      Cand cd = (lane < NW) ? wbest[lane] : Cand{0.0, -1.0, 0x7fffffff, 0};
      double ms = cd.mass, v = cd.val;
      int p = cd.pos;
      ms = warp_sum(ms);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int op = __shfl_xor_sync(0xffffffffu, p, o);
        if (better(ov, op, v, p)) { v = ov; p = op; }
      }
      if (lane < CS) {
        Cand out;
        out.mass = ms; out.val = v; out.pos = p; out.pad = 0;
        Cand* dst = cluster.map_shared_rank(&slot[buf][rank], lane);
        *dst = out;
      }
    }
    cluster.sync();
    // ---- B: global decision (identical in every CTA)
    double tot = 0.0, gv = -1.0;
    int gp = 0x7fffffff;
    for (int q = 0; q < CS; ++q) {  // fixed order: deterministic
      const Cand cd = slot[buf][q];
      tot += cd.mass;
      if (better(cd.val, cd.pos, gv, gp)) { gv = cd.val; gp = cd.pos; }
    }
    if (tot <= 4.0 * stop2) {
      // exact recomputation before trusting downdated norms near the threshold
      for (int jl = warp; jl < cq; jl += NW) {
        if (!flag[jl]) continue;
        double q = 0.0;
        for (int r = s + lane; r < m; r += 32) { const double v = A[(int64_t)jl * m + r]; q += v * v; }
        q = warp_sum(q);
        if (lane == 0) { nrm[jl] = q; nrm0[jl] = q; }
      }
      __syncthreads();
      double lm = 0.0;
      for (int jl = tid; jl < cq; jl += QC_THREADS)
        if (flag[jl]) lm += nrm[jl];
      lm = block_sum(lm, red);
      if (tid < CS) *cluster.map_shared_rank(&slot2[rank], tid) = lm;
      cluster.sync();
      tot = 0.0;
      for (int q = 0; q < CS; ++q) tot += slot2[q];
      // the candidate may have changed by the recomputation
      bv = -1.0;
      bp = 0x7fffffff;
      for (int jl = tid; jl < cq; jl += QC_THREADS)
        if (flag[jl] && better(nrm[jl], g0 + jl, bv, bp)) { bv = nrm[jl]; bp = g0 + jl; }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int op = __shfl_xor_sync(0xffffffffu, bp, o);
        if (better(ov, op, bv, bp)) { bv = ov; bp = op; }
      }
      __syncthreads();
      if (lane == 0) { Cand cd; cd.mass = 0.0; cd.val = bv; cd.pos = bp; cd.pad = 0; wbest[warp] = cd; }
      __syncthreads();
      if (warp == 0) {
        Cand cd = (lane < NW) ? wbest[lane] : Cand{0.0, -1.0, 0x7fffffff, 0};
        double v = cd.val;
        int p = cd.pos;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ov = __shfl_xor_sync(0xffffffffu, v, o);
          const int op = __shfl_xor_sync(0xffffffffu, p, o);
          if (better(ov, op, v, p)) { v = ov; p = op; }
        }
        if (lane < CS) {
          Cand out;
          out.mass = 0.0; out.val = v; out.pos = p; out.pad = 0;
          *cluster.map_shared_rank(&slot[buf ^ 1][rank], lane) = out;
        }
      }
      cluster.sync();
      gv = -1.0;
      gp = 0x7fffffff;
      for (int q = 0; q < CS; ++q) {
        const Cand cd = slot[buf ^ 1][q];
        if (better(cd.val, cd.pos, gv, gp)) { gv = cd.val; gp = cd.pos; }
      }
      cluster.sync();  // slot[buf^1] is reused by the next step
    }
    if (tot <= stop2 || gp == 0x7fffffff) break;
    if (tid == 0) piv_pos[nsteps] = gp;
    // ---- owner forms the reflector from its column gp (rows s..m-1) and broadcasts it
    const bool owner = (gp >= g0 && gp < g0 + cq);
    if (owner) {
      const int jl = gp - g0;
      double* col = A + (int64_t)jl * m;
      double pp = 0.0;
      for (int r = s + 1 + tid; r < m; r += QC_THREADS) { const double v = col[r]; pp += v * v; }
      const double sigma = block_sum(pp, red);
      const double alpha = col[s];
      double t = 0.0, beta = alpha, scal = 0.0;
      if (sigma != 0.0) {
        const double nr = sqrt(alpha * alpha + sigma);
        beta = alpha >= 0.0 ? -nr : nr;
        t = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      for (int r = s + 1 + tid; r < m; r += QC_THREADS) col[r] *= scal;
      __syncthreads();
      if (tid == 0) { col[s] = beta; flag[jl] = 0; tau_g[s] = t; }
      // broadcast v (v_s = 1) and tau to every CTA's buffer `buf`
      for (int64_t idx = tid; idx < (int64_t)(m - s) * CS; idx += QC_THREADS) {
        const int dst = (int)(idx / (m - s)), r = s + (int)(idx % (m - s));
        const double v = (r == s) ? 1.0 : col[r];
        *cluster.map_shared_rank(&vb[(int64_t)buf * m + r], dst) = v;
      }
      if (tid < CS) *cluster.map_shared_rank(&taus[buf], tid) = t;
    }
    cluster.sync();
    // ---- C: apply H = I - tau v v^T to the active local columns, downdate their norms
    const double t = taus[buf];
    const double* v = vb + (int64_t)buf * m;
    for (int jl = warp; jl < cq; jl += NW) {
      if (!flag[jl]) continue;
      double* col = A + (int64_t)jl * m;
      if (t != 0.0) {
        double q = 0.0;
        for (int r = s + lane; r < m; r += 32) q += v[r] * col[r];
        q = t * warp_sum(q);
        for (int r = s + lane; r < m; r += 32) col[r] -= q * v[r];
      }
      __syncwarp();
      const double rs = col[s];
      double nn = nrm[jl] - rs * rs;
      if (!(nn > 1e-8 * nrm0[jl])) {
        double q = 0.0;
        for (int r = s + 1 + lane; r < m; r += 32) { const double x = col[r]; q += x * x; }
        nn = warp_sum(q);
        if (lane == 0) nrm0[jl] = nn;
      }
      __syncwarp();
      if (lane == 0) nrm[jl] = nn;
    }
    __syncthreads();
  }
  const int k = s;
  // exact trailing mass of the unpivoted columns (rows >= k)
  double part = 0.0;
  for (int jl = warp; jl < cq; jl += NW) {
    if (!flag[jl]) continue;
    for (int r = k + lane; r < m; r += 32) { const double x = A[(int64_t)jl * m + r]; part += x * x; }
  }
  part = block_sum(part, red);
  if (tid < CS) *cluster.map_shared_rank(&slot2[rank], tid) = part;
  cluster.sync();
  // ---- write-back in pivoted order: positions k_start.. for pivots, then the rest in order
  const int npiv = k - k_start;
  for (int jl = 0; jl < cq; ++jl) {
    const int g = g0 + jl;
    int dst = -1;
    if (!flag[jl]) {
      for (int q = 0; q < npiv; ++q)
        if (piv_pos[q] == g) { dst = k_start + q; break; }
    } else {
      int before = 0;
      for (int q = 0; q < npiv; ++q) before += (piv_pos[q] < g);
      dst = k + (g - k_start) - before;
    }
    for (int r = tid; r < m; r += QC_THREADS) Y[(int64_t)r + (int64_t)dst * ldy] = A[(int64_t)jl * m + r];
  }
  // perm and tau: every CTA reads the old perm of its own columns (global, before any write
  // to it: perm is written to a scratch half and copied by CTA 0 after a barrier)
  int* newperm = perm_g + c;
  for (int jl = tid; jl < cq; jl += QC_THREADS) {
    const int g = g0 + jl;
    int dst;
    if (!flag[jl]) {
      dst = -1;
      for (int q = 0; q < npiv; ++q)
        if (piv_pos[q] == g) { dst = k_start + q; break; }
    } else {
      int before = 0;
      for (int q = 0; q < npiv; ++q) before += (piv_pos[q] < g);
      dst = k + (g - k_start) - before;
    }
    newperm[dst] = perm_g[g];
  }
  cluster.sync();
  if (rank == 0) {
    for (int j = k_start + tid; j < c; j += QC_THREADS) perm_g[j] = newperm[j];
    if (tid == 0) {
      double e2 = 0.0;
      for (int q = 0; q < CS; ++q) e2 += slot2[q];
      scalars[0] = (double)k;
      scalars[1] = e2;
    }
  }
  cluster.sync();
}

size_t qc_smem(int64_t m, int64_t cq) {
  return sizeof(double) * (size_t)(m * cq + 2 * m + 2 * cq) + sizeof(int) * (size_t)cq + 64;
}

__global__ void unpermute_cols_kernel(const double* __restrict__ in, int64_t ldi, int rows, int c,
                                      const int* __restrict__ perm, double* out, int64_t ldo) {
  const int64_t total = (int64_t)rows * c;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total; idx += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(idx % rows), j = (int)(idx / rows);
    out[(int64_t)r + (int64_t)perm[j] * ldo] = in[(int64_t)r + (int64_t)j * ldi];
  }
}

}  // namespace

bool qrcp_cluster_fits(int64_t m, int64_t c) {
  return c >= 1 && qc_smem(m, ceil_div(c, QC_MAXCS)) <= (size_t)QC_SMEM;
}

void unpermute_cols(tt_ctx ctx, const double* in, int64_t ldi, int64_t rows, int64_t c, const int* perm, double* out,
                    int64_t ldo) {
  if (rows <= 0 || c <= 0) return;
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(rows * c, 256), 2048));
  TTB_RUN(ctx, "aux", 0, 16.0 * rows * c,
          unpermute_cols_kernel<<<blocks, 256, 0, ctx->stream>>>(in, ldi, (int)rows, (int)c, perm, out, ldo));
}

bool qrcp_cluster_run(tt_ctx ctx, double* Y, int64_t ldy, int64_t m, int64_t c, int k_start, double stop2, int kcap,
                      double* tau, int* perm2c, double* scalars) {
  const int64_t act = c - k_start;
  if (act <= 0) return false;
  int CS = 0;
  for (int cs = 1; cs <= QC_MAXCS; ++cs)
    if (qc_smem(m, ceil_div(act, cs)) <= (size_t)QC_SMEM) { CS = cs; break; }
  if (CS == 0) return false;
  // spread over more CTAs when that shortens the per-step column work (<= 48 columns per CTA)
  while (CS < QC_MAXCS && ceil_div(act, CS) > 48) ++CS;
  if (const char* f = std::getenv("TT_B200_QRCP_CS")) {  // debugging: force the cluster size
    const int want = std::atoi(f);
    if (want >= 1 && want <= QC_MAXCS && qc_smem(m, ceil_div(act, want)) <= (size_t)QC_SMEM) CS = want;
  }
  CS = (int)std::min<int64_t>(CS, act);
  const size_t smem = qc_smem(m, ceil_div(act, CS));
  TTB_CUDA(cudaFuncSetAttribute(qrcp_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, QC_SMEM + 64));
  if (CS > 8) TTB_CUDA(cudaFuncSetAttribute(qrcp_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(CS, 1, 1);
  cfg.blockDim = dim3(QC_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TTB_RUN(ctx, "qrcp_cluster", 0, 16.0 * m * c,
          TTB_CUDA(cudaLaunchKernelEx(&cfg, qrcp_cluster_kernel, Y, ldy, (int)m, (int)c, k_start, stop2, kcap, tau,
                                      perm2c, scalars)));
  return true;
}

}  // namespace ttb
