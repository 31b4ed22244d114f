// Batched TT-rounding of many independent, uniformly shaped TT-sums (BASELINE.json
// configs[3], "C4": 4096 sums of 4 rank-16 TTs).  PAPER.md:64 (TT-sum ranks add; rounding
// contract ||x - x~|| <= delta ||x||), PAPER.md:69 (O(d n r^3) rounding); algorithm =
// Oseledets' TT-SVD rounding (readings A1-A3, A11, A12).
//
// One CTA per item; each launch runs ONE phase of the rounding for every item of a wave, so
// the GPU is filled by the batch, not by the (small) matrices of one item:
//
//   br_r2l_kernel (core k = d..2)  assembles the right-to-left panel A_k = C_k^T
//       ((n_k R'_k) x R_{k-1}) stack by stack straight from the terms' cores (block-diagonal
//       TT-sum read in-kernel; coefficient c_l applied on term l's last core) and factors it
//       by a flat-tree Householder QR: a 64-row R block in shared memory plus 128-row chunks
//       held in registers (warp w owns columns w, w+8, ...; lane owns rows lane+32t).  One
//       __syncthreads per reflector.  Reflectors go to HBM, R is passed to core k-1.
//   br_l2r_kernel (split k = 1..d-1)  Y_k ((rho_{k-1} n_k) x R'_k) -> Householder QR when it
//       has more than 64 rows -> one-sided Jacobi SVD (<= 64 x 64, shared memory) -> rho_k =
//       smallest rho with sqrt(sum_{j>rho} sigma_j^2) <= tau -> output core k = Q_Y U_rho and
//       Z_{k+1} = H_{k+1} [(S_rho V_rho^T)^T; 0]: the right-orthonormal core k+1 is never
//       formed, its reflectors are applied to the thin S V^T.
//   br_compact_kernel  moves the cores from the worst-case workspace to the exact-size arena
//       shared by the batch's result tensors (ranks are known only after the sweep).
//
// Unlike round.cu, the right-to-left QR is not rank-revealing: panels keep their structural
// ranks R'_{k-1} = min(n_k R'_k, R_{k-1}) (identical tensor; the truncation decisions come from
// the same SVDs).  Supported shapes: d >= 2, every formal rank R_k <= 64, K <= 16 terms.
#include <algorithm>
#include <cstddef>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "batch_round.cuh"
#include "batch_wy.cuh"
#include "ttops.cuh"

namespace ttb {

namespace {

constexpr int BR_T = 256;              // threads per CTA
constexpr int BR_W = BR_T / 32;        // warps
constexpr int BR_C = 64;               // max columns (formal ranks)
constexpr int BR_CH = 128;             // chunk rows held in registers
constexpr int BR_RPL = BR_CH / 32;     // chunk rows per lane
constexpr int BR_CPW = BR_C / BR_W;    // columns per warp
constexpr int BR_S0 = BR_C + BR_CH;    // rows of stack 0 (R block + first chunk)
constexpr int BR_SL = 8;               // reflectors per staged slice of the applications
constexpr int BR_APPLY_NS = 2;         // target columns per warp and pass of the applications
constexpr int BR_MAXD = 64;
constexpr int BR_MAXK = 16;
constexpr int BR_JAC_SWEEPS = 60;

struct BRShape {
  int d, K;
  int n[BR_MAXD];
  int R[BR_MAXD + 1];             // formal ranks R_k = sum_l r_k^(l)
  int Rp[BR_MAXD + 1];            // ranks after the right-to-left sweep
  int r[BR_MAXK][BR_MAXD + 1];    // term ranks
  int off[BR_MAXD + 1][BR_MAXK];  // offset of term l inside R_k
  int64_t voff[BR_MAXD];          // core index kc: offset of its panel reflectors (per item)
  int64_t toff[BR_MAXD];          // core index kc: offset of its taus (per item)
  int64_t ooff[BR_MAXD];          // core index kc: worst-case output core offset (per item)
  int64_t vstride, tstride, ystride, ytstride, zstride, ostride;
  int wyni[BR_MAXD];              // WY engine: mode indices per chunk of panel kc (chunk rows wyni * Rp[kc+1])
};

struct LBuf {  // long long device buffer (debug counters)
  tt_ctx ctx = nullptr;
  long long* p = nullptr;
  void alloc(tt_ctx c, size_t n) { ctx = c; TTB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), n * sizeof(long long), c->stream)); }
  ~LBuf() { if (p) cudaFreeAsync(p, ctx->stream); }
};

struct BRArgs {
  const BRShape* sh;
  const double* const* cores;  // [gitem][l][kc]
  const double* coef;          // [gitem][l]
  const double* scale;         // [gitem] s(x)
  double* V;                   // right-to-left reflectors   [item][vstride]
  double* T;                   // their taus                 [item][tstride]
  double* L;                   // R factors, 2 slots         [item][2][64*64]
  double* YV;                  // left-to-right QR reflectors [item][ystride]
  double* YT;                  // their taus                 [item][ytstride]
  double* Z;                   // Y_{k+1} staging, 2 slots   [item][2][zstride]
  double* out;                 // worst-case output cores    [item][ostride]
  double* JM;                  // l2r: Jacobi input (R_Y or Y), 64 x 64 per item
  double* QX;                  // l2r: QRCP of R_Y^T (factors 64 x 64 + 64 taus) per item
  double* TT;                  // l2r: apply targets U_rho and V_rho S, 2 x 64 x 64 per item
  int* ranks;                  // [item][d+1]
  double* scal;                // [item][4]: ||x||, tau, s, zero flag
  int* info;                   // [item]: 1 = Jacobi hit its sweep limit
  int* gemm;                   // [item]: 1 = output core of this split by U = Y V S^-1 (DMMA)
  double rel_tol, floor_c;
  int64_t max_rank;
  int keep_all;
  int jac_t;                   // tall splits: one-sided Jacobi on R_Y^T (rows of R) instead of R_Y
  int qrcp_svd;                // tall splits: rank-revealing QR of R_Y^T before the Jacobi (truncated)
  int jac_lpp;                 // lanes per Jacobi column pair (0: by the pair count; TT_B200_BR_JLPP)
  int item0;                   // global index of this wave's first item
  int b0 = 0;                  // first item of this launch inside the wave (half-wave launches)
  long long* dbg;              // TT_B200_BR_DEBUG: CTA 0 phase cycle counters (else null)
};

__host__ __device__ inline int br_stacks(int64_t m) {
  return m <= BR_S0 ? 1 : 1 + (int)((m - BR_S0 + BR_CH - 1) / BR_CH);
}
__host__ __device__ inline int64_t br_stack_off(int q, int c) {  // reflector storage offset of stack q
  return q == 0 ? 0 : (int64_t)BR_S0 * c + (int64_t)BR_CH * c * (q - 1);
}
__host__ __device__ inline int64_t br_vsize(int64_t m, int c) { return br_stack_off(br_stacks(m), c); }

template <int N>
__device__ __forceinline__ double sel(const double (&a)[N], int j) {
  double r = 0.0;
#pragma unroll
  for (int c = 0; c < N; ++c)
    if (c == j) r = a[c];
  return r;
}

// ---- 1-D bulk copies global -> shared (TMA engine) completing on an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
  }
}

// Reflector slices (8 consecutive reflectors of one stack, stored contiguously) staged in shared
// memory by the TMA engine, double-buffered; the next slice is in flight while one is applied.
struct VStage {
  alignas(16) double buf[2][BR_SL * BR_S0];
  uint64_t bar[2];
  uint32_t phase[2];  // (kept per thread, uniform)
};

// Shared-memory work areas of one CTA.
struct BRSmem {
  double Rs[BR_C * BR_C];     // R block (column-major, ld 64); Jacobi matrix in the l2r kernel
  double Aux[BR_C * BR_C];    // L^T for the panel assembly; V of the Jacobi SVD
  double vb[2][BR_S0];        // reflector broadcast (double-buffered)
  double tb[2];
  double sig[BR_C];
  double red[32];
  int perm[BR_C];
  int cterm[BR_C], ca[BR_C];
  int flag;
  int rho;
  uint64_t qfull[2], qempty[2];  // split-phase reflector hand-off of the later stacks (br_stack_qr_later_async)
  double xst[BR_W][32];       // r2l panel assembly: the term-core values of one column, per warp
  VStage vst;
};

// Sums over the 32 lanes of eight per-lane values v[0..7] (one total per column), returned in
// every lane: a transposed butterfly halves the set per level (4 + 2 + 1 exchanges), two more
// finish the sums, one broadcast per column -- 17 shuffles instead of 8 x 5.
__device__ __forceinline__ void warp_sum8(double (&v)[8]) {
  const int lane = threadIdx.x & 31;
  const bool b4 = (lane & 16) != 0, b3 = (lane & 8) != 0, b2 = (lane & 4) != 0;
  double u4[4], u2[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double keep = b4 ? v[4 + k] : v[k], send = b4 ? v[k] : v[4 + k];
    u4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);  // column 4 b4 + k
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double keep = b3 ? u4[2 + k] : u4[k], send = b3 ? u4[k] : u4[2 + k];
    u2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);   // column 4 b4 + 2 b3 + k
  }
  double u1 = (b2 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u2[0] : u2[1], 4);  // column 4 b4 + 2 b3 + b2
  u1 += __shfl_xor_sync(0xffffffffu, u1, 2);
  u1 += __shfl_xor_sync(0xffffffffu, u1, 1);
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = __shfl_sync(0xffffffffu, u1, ((c >> 2) & 1) * 16 + ((c >> 1) & 1) * 8 + (c & 1) * 4);
}

// Two per-lane values summed over the warp (one total each, in every lane): one exchange
// halves the pair, four more finish, two broadcasts -- 7 shuffles instead of 2 x 5.
__device__ __forceinline__ void warp_sum2(double (&v)[2]) {
  const int lane = threadIdx.x & 31;
  const bool b4 = (lane & 16) != 0;
  double u = (b4 ? v[1] : v[0]) + __shfl_xor_sync(0xffffffffu, b4 ? v[0] : v[1], 16);  // column b4
#pragma unroll
  for (int o = 8; o > 0; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
  v[0] = __shfl_sync(0xffffffffu, u, 0);
  v[1] = __shfl_sync(0xffffffffu, u, 16);
}

// Flat-tree Householder QR step over one stack: R block in sm.Rs (rows 0..63, column-major;
// a full block for stack 0, upper triangular afterwards) stacked on the 128-row chunk in
// registers a[t][s] (row 32t + lane, column 8s + warp).  LAPACK dlarfg arithmetic per column j;
// on return the strictly lower part of Rs holds stack 0's R-block reflector parts, a[][] holds
// the chunk reflector parts, taus go to tau_out[j] (global).
__device__ void br_stack_qr_first(double (&a)[BR_RPL][BR_CPW], BRSmem& sm, int ncol, double* tau_out, long long* sdbg) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long c0 = 0, c1 = 0, c2 = 0;
  // j = 8 S + ww: the slot S of column j in its owner warp ww is a compile-time index
#pragma unroll
  for (int S = 0; S < BR_CPW; ++S) {
#pragma unroll 1
    for (int ww = 0; ww < BR_W; ++ww) {
      const int j = S * BR_W + ww;
      if (j >= ncol) break;
      const int buf = j & 1;
      if (sdbg) c0 = clock64();
      if (warp == ww) {
        double* Rc = sm.Rs + j * BR_C;
        const double r0 = Rc[lane], r1 = Rc[lane + 32];
        double ss = 0.0;
        if (lane > j) ss += r0 * r0;
        if (lane + 32 > j) ss += r1 * r1;
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) ss += a[t][S] * a[t][S];
        const double sigma = warp_sum(ss);
        const double alpha = Rc[j];
        double tau = 0.0, beta = alpha, scal = 0.0;
        if (sigma != 0.0) {
          // dlarfg with one reciprocal: inv = 1 / (beta (alpha - beta)) (never 0: signs differ)
          const double nr = sqrt(alpha * alpha + sigma);
          beta = alpha >= 0.0 ? -nr : nr;
          const double am = alpha - beta;
          const double inv = 1.0 / (beta * am);
          tau = -am * am * inv;  // (beta - alpha) / beta
          scal = beta * inv;     // 1 / (alpha - beta)
        }
        const double v0 = lane > j ? r0 * scal : (lane == j ? 1.0 : 0.0);
        const double v1 = lane + 32 > j ? r1 * scal : (lane + 32 == j ? 1.0 : 0.0);
        sm.vb[buf][lane] = v0;
        sm.vb[buf][lane + 32] = v1;
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) {
          a[t][S] *= scal;
          sm.vb[buf][BR_C + 32 * t + lane] = a[t][S];
        }
        __syncwarp();
        if (lane > j) Rc[lane] = v0;
        if (lane + 32 > j) Rc[lane + 32] = v1;
        if (lane == j) Rc[lane] = beta;
        if (lane + 32 == j) Rc[lane + 32] = beta;
        if (lane == 0) { sm.tb[buf] = tau; tau_out[j] = tau; }
      }
      if (sdbg) c1 = clock64();
      __syncthreads();
      if (sdbg) c2 = clock64();
      const double tau = sm.tb[buf];
      if (tau != 0.0) {
        const double* v = sm.vb[buf];
        const double v0 = v[lane], v1 = v[lane + 32];
        double vc[BR_RPL];
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) vc[t] = v[BR_C + 32 * t + lane];
        // columns 8s + warp > j (slots below S are done): all partial dots first, the
        // reductions interleaved (branch-free: an inactive column gets a zero update)
        double dt[BR_CPW], r0[BR_CPW], r1[BR_CPW];
#pragma unroll
        for (int s = S; s < BR_CPW; ++s) {
          const int col = min(s * BR_W + warp, BR_C - 1);
          r0[s] = sm.Rs[col * BR_C + lane];
          r1[s] = sm.Rs[col * BR_C + lane + 32];
          double q = (v0 * r0[s] + v1 * r1[s]) + (vc[0] * a[0][s] + vc[1] * a[1][s]);
#pragma unroll
          for (int t = 2; t < BR_RPL; ++t) q += vc[t] * a[t][s];
          dt[s] = q;
        }
        if (S < 5) {  // >= 4 live slots: transposed butterfly over all 8
#pragma unroll
          for (int s = 0; s < S; ++s) dt[s] = 0.0;
          warp_sum8(dt);
        } else {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int s = S; s < BR_CPW; ++s) dt[s] += __shfl_xor_sync(0xffffffffu, dt[s], o);
        }
#pragma unroll
        for (int s = S; s < BR_CPW; ++s) {
          const int col = s * BR_W + warp;
          const bool act = (s > S || warp > ww) && col < ncol;
          const double w = act ? tau * dt[s] : 0.0;
          if (act) {
            sm.Rs[col * BR_C + lane] = r0[s] - w * v0;
            sm.Rs[col * BR_C + lane + 32] = r1[s] - w * v1;
          }
#pragma unroll
          for (int t = 0; t < BR_RPL; ++t) a[t][s] -= w * vc[t];
        }
      }
      if (sdbg && tid == 0) {
        const long long c3 = clock64();
        if (ww == 0) { sdbg[0] += c1 - c0; sdbg[3] += 1; } else { sdbg[4] += c1 - c0; }
        sdbg[1] += c2 - c1;
        sdbg[2] += c3 - c2;
      }
    }
  }
  __syncthreads();
}

// Stacks after the first: the R block is upper triangular, so the reflector's R-block part is
// the unit vector e_j: the R block enters the column dot products and updates only through row j.
__device__ void br_stack_qr_later(double (&a)[BR_RPL][BR_CPW], BRSmem& sm, int ncol, double* tau_out, long long* sdbg) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  long long c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
  for (int S = 0; S < BR_CPW; ++S) {
#pragma unroll 1
    for (int ww = 0; ww < BR_W; ++ww) {
      const int j = S * BR_W + ww;
      if (j >= ncol) break;
      const int buf = j & 1;
      if (sdbg) c0 = clock64();
      if (warp == ww) {
        double* Rc = sm.Rs + j * BR_C;
        double ss = 0.0;
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) ss += a[t][S] * a[t][S];
        const double sigma = warp_sum(ss);
        const double alpha = Rc[j];
        double tau = 0.0, beta = alpha, scal = 0.0;
        if (sigma != 0.0) {
          const double nr = sqrt(alpha * alpha + sigma);
          beta = alpha >= 0.0 ? -nr : nr;
          const double am = alpha - beta;
          const double inv = 1.0 / (beta * am);
          tau = -am * am * inv;
          scal = beta * inv;
        }
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) {
          a[t][S] *= scal;
          sm.vb[buf][BR_C + 32 * t + lane] = a[t][S];
        }
        __syncwarp();
        if (lane == 0) { Rc[j] = beta; sm.tb[buf] = tau; tau_out[j] = tau; }
      }
      if (sdbg) c1 = clock64();
      __syncthreads();
      if (sdbg) c2 = clock64();
      const double tau = sm.tb[buf];
      if (tau != 0.0) {
        const double* v = sm.vb[buf];
        double vc[BR_RPL];
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) vc[t] = v[BR_C + 32 * t + lane];
        double dt[BR_CPW], rj[BR_CPW];
#pragma unroll
        for (int s = S; s < BR_CPW; ++s) {
          const int col = min(s * BR_W + warp, BR_C - 1);
          rj[s] = sm.Rs[col * BR_C + j];  // broadcast: row j of the R block
          double q = vc[0] * a[0][s] + vc[1] * a[1][s];
#pragma unroll
          for (int t = 2; t < BR_RPL; ++t) q += vc[t] * a[t][s];
          dt[s] = q;
        }
        if (S < 5) {  // >= 4 live slots: transposed butterfly over all 8
#pragma unroll
          for (int s = 0; s < S; ++s) dt[s] = 0.0;
          warp_sum8(dt);
        } else {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1)
#pragma unroll
            for (int s = S; s < BR_CPW; ++s) dt[s] += __shfl_xor_sync(0xffffffffu, dt[s], o);
        }
#pragma unroll
        for (int s = S; s < BR_CPW; ++s) {
          const int col = s * BR_W + warp;
          const bool act = (s > S || warp > ww) && col < ncol;
          const double w = act ? tau * (rj[s] + dt[s]) : 0.0;
          if (act && lane == 0) sm.Rs[col * BR_C + j] = rj[s] - w;
#pragma unroll
          for (int t = 0; t < BR_RPL; ++t) a[t][s] -= w * vc[t];
        }
      }
      if (sdbg && tid == 0) {
        const long long c3 = clock64();
        if (ww == 0) { sdbg[0] += c1 - c0; sdbg[3] += 1; } else { sdbg[4] += c1 - c0; }
        sdbg[1] += c2 - c1;
        sdbg[2] += c3 - c2;
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Later stacks (R block upper triangular, reflector R-block part e_j), split-phase version of
// br_stack_qr_later: reflector j is handed over through buffer j & 1 guarded by two mbarriers
// (qfull: the owner warp's 32 lanes arrive after writing it; qempty: every thread arrives once
// it holds it in registers) instead of a __syncthreads per reflector.  The owner of column j+1
// applies reflector j to that column first, forms reflector j+1 and publishes it, then updates
// its other columns; every other warp updates its columns as soon as reflector j is out.  Every
// column is touched by its owner warp only, so nothing else needs ordering.  Same arithmetic.
template <int SL>
__device__ __forceinline__ void br_gen_later(double (&a)[BR_RPL][BR_CPW], BRSmem& sm, int j, double* tau_out,
                                             int lane) {
  const int buf = j & 1;
  double* Rc = sm.Rs + j * BR_C;
  double ss = 0.0;
#pragma unroll
  for (int t = 0; t < BR_RPL; ++t) ss += a[t][SL] * a[t][SL];
  const double sigma = warp_sum(ss);
  const double alpha = Rc[j];
  double tau = 0.0, beta = alpha, scal = 0.0;
  if (sigma != 0.0) {
    const double nr = sqrt(alpha * alpha + sigma);
    beta = alpha >= 0.0 ? -nr : nr;
    const double am = alpha - beta;
    const double inv = 1.0 / (beta * am);
    tau = -am * am * inv;
    scal = beta * inv;
  }
#pragma unroll
  for (int t = 0; t < BR_RPL; ++t) {
    a[t][SL] *= scal;
    sm.vb[buf][BR_C + 32 * t + lane] = a[t][SL];
  }
  __syncwarp();
  if (lane == 0) { Rc[j] = beta; sm.tb[buf] = tau; tau_out[j] = tau; }
}

template <int SL>
__device__ __forceinline__ void br_upd_one_later(double (&a)[BR_RPL][BR_CPW], BRSmem& sm, int j, double tau,
                                                 const double (&vc)[BR_RPL], int lane, int warp) {
  const int col = SL * BR_W + warp;
  const double rj = sm.Rs[col * BR_C + j];
  double q = vc[0] * a[0][SL] + vc[1] * a[1][SL];
#pragma unroll
  for (int t = 2; t < BR_RPL; ++t) q += vc[t] * a[t][SL];
  q = warp_sum(q);
  const double w = tau * (rj + q);
  __syncwarp();
  if (lane == 0) sm.Rs[col * BR_C + j] = rj - w;
#pragma unroll
  for (int t = 0; t < BR_RPL; ++t) a[t][SL] -= w * vc[t];
}

template <int S>
__device__ __forceinline__ void br_later_async_slot(double (&a)[BR_RPL][BR_CPW], BRSmem& sm, int ncol,
                                                    double* tau_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
  for (int ww = 0; ww < BR_W; ++ww) {
    const int j = S * BR_W + ww;
    if (j >= ncol) return;
    const int buf = j & 1;
    mbar_wait(&sm.qfull[buf], (uint32_t)((j >> 1) & 1));
    const double tau = sm.tb[buf];
    const double* v = sm.vb[buf];
    double vc[BR_RPL];
#pragma unroll
    for (int t = 0; t < BR_RPL; ++t) vc[t] = v[BR_C + 32 * t + lane];
    mbar_arrive(&sm.qempty[buf]);  // reflector j is in registers: its buffer may be reused
    const int j1 = j + 1;
    const bool own = j1 < ncol && warp == (j1 & (BR_W - 1));
    if (own) {  // look-ahead: column j+1 first, reflector j+1 published, then the other columns
      if (ww < BR_W - 1) {
        if (tau != 0.0) br_upd_one_later<S>(a, sm, j, tau, vc, lane, warp);
      } else {
        if constexpr (S + 1 < BR_CPW)
          if (tau != 0.0) br_upd_one_later<S + 1>(a, sm, j, tau, vc, lane, warp);
      }
      if (j1 >= 2) mbar_wait(&sm.qempty[j1 & 1], (uint32_t)(((j1 - 2) >> 1) & 1));
      __syncwarp();
      if (ww < BR_W - 1) {
        br_gen_later<S>(a, sm, j1, tau_out, lane);
      } else {
        if constexpr (S + 1 < BR_CPW) br_gen_later<S + 1>(a, sm, j1, tau_out, lane);
      }
      __syncwarp();
      mbar_arrive(&sm.qfull[j1 & 1]);
    }
    if (tau != 0.0) {
      double dt[BR_CPW], rj[BR_CPW];
#pragma unroll
      for (int s = S; s < BR_CPW; ++s) {
        const int col = min(s * BR_W + warp, BR_C - 1);
        rj[s] = sm.Rs[col * BR_C + j];  // broadcast: row j of the R block
        double q = vc[0] * a[0][s] + vc[1] * a[1][s];
#pragma unroll
        for (int t = 2; t < BR_RPL; ++t) q += vc[t] * a[t][s];
        dt[s] = q;
      }
      if (S < 5) {  // >= 4 live slots: transposed butterfly over all 8
#pragma unroll
        for (int s = 0; s < S; ++s) dt[s] = 0.0;
        warp_sum8(dt);
      } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int s = S; s < BR_CPW; ++s) dt[s] += __shfl_xor_sync(0xffffffffu, dt[s], o);
      }
#pragma unroll
      for (int s = S; s < BR_CPW; ++s) {
        const int col = s * BR_W + warp;
        const bool act = (s > S || warp > ww) && col < ncol && !(own && col == j1);
        const double w = act ? tau * (rj[s] + dt[s]) : 0.0;
        if (act && lane == 0) sm.Rs[col * BR_C + j] = rj[s] - w;
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) a[t][s] -= w * vc[t];
      }
    }
  }
  if constexpr (S + 1 < BR_CPW) br_later_async_slot<S + 1>(a, sm, ncol, tau_out);
}

__device__ void br_stack_qr_later_async(double (&a)[BR_RPL][BR_CPW], BRSmem& sm, int ncol, double* tau_out) {
  const int tid = threadIdx.x;
  if (ncol <= 0) return;
  if (tid == 0) {
    mbar_init(&sm.qfull[0], 32);
    mbar_init(&sm.qfull[1], 32);
    mbar_init(&sm.qempty[0], BR_T);
    mbar_init(&sm.qempty[1], BR_T);
  }
  __syncthreads();
  if ((tid >> 5) == 0) {  // reflector 0: warp 0, slot 0
    br_gen_later<0>(a, sm, 0, tau_out, tid & 31);
    __syncwarp();
    mbar_arrive(&sm.qfull[0]);
  }
  br_later_async_slot<0>(a, sm, ncol, tau_out);
  __syncthreads();  // every warp done (every barrier phase consumed) before the stack is stored
}

// Store one stack's reflectors (column-major, ld = stack rows) and, for stack 0, move the
// R-block reflector parts out of Rs (its strictly lower part is zeroed for the next stacks).
__device__ void br_store_stack(const double (&a)[BR_RPL][BR_CPW], BRSmem& sm, int q, int ncol, double* Vq) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ld = q == 0 ? BR_S0 : BR_CH, roff = q == 0 ? BR_C : 0;
#pragma unroll
  for (int s = 0; s < BR_CPW; ++s) {
    const int col = s * BR_W + warp;
    if (col < ncol) {
#pragma unroll
      for (int t = 0; t < BR_RPL; ++t) Vq[(int64_t)col * ld + roff + 32 * t + lane] = a[t][s];
    }
  }
  if (q == 0) {
    for (int idx = tid; idx < BR_C * ncol; idx += BR_T) {
      const int col = idx / BR_C, row = idx % BR_C;
      if (row > col) {
        Vq[(int64_t)col * ld + row] = sm.Rs[col * BR_C + row];
        sm.Rs[col * BR_C + row] = 0.0;
      }
    }
  }
  __syncthreads();
}

// target <- H_q target for one stack's reflectors (j = ncol-1 .. 0).  The target's R-block
// rows live in tr[0/1][s] (rows lane, lane+32), its chunk rows in tc[t][s]; column 8s + warp.
// target <- H_q target for one stack's reflectors (j = ncol-1 .. 0), reflector vectors read
// from the staged slices.  The target's R-block rows live in tr[0/1][s] (rows lane, lane+32),
// its chunk rows in tc[t][s]; column 8s + warp.
template <int NS, bool FIRST>
__device__ void br_stack_apply(double (&tr)[2][NS], double (&tc)[BR_RPL][NS], const double* __restrict__ Vq,
                               const double* __restrict__ tq, int q, int ncol, int ntgt, VStage& vs,
                               uint32_t (&ph)[2]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ld = q == 0 ? BR_S0 : BR_CH, roff = q == 0 ? BR_C : 0;
  const int nsl = (ncol + BR_SL - 1) / BR_SL;
  auto issue = [&](int sl, int b) {
    const int j0 = sl * BR_SL, cnt = min(BR_SL, ncol - j0);
    bulk_load(vs.buf[b], Vq + (int64_t)j0 * ld, (uint32_t)(cnt * ld * sizeof(double)), &vs.bar[b]);
  };
  __syncthreads();  // previous users of both buffers are done
  if (threadIdx.x == 0) issue(nsl - 1, 0);
#pragma unroll 1
  for (int sl = nsl - 1, b = 0; sl >= 0; --sl, b ^= 1) {
    if (sl > 0) {
      __syncthreads();  // everyone finished reading buffer b^1 (slice sl+1)
      if (threadIdx.x == 0) issue(sl - 1, b ^ 1);
    }
    mbar_wait(&vs.bar[b], ph[b]);
    ph[b] ^= 1u;
    const double* sv = vs.buf[b];
    const int j0 = sl * BR_SL, j1 = min(j0 + BR_SL, ncol);
#pragma unroll 1
    for (int j = j1 - 1; j >= j0; --j) {
      const double tau = __ldg(tq + j);
      if (tau == 0.0) continue;
      const double* v = sv + (j - j0) * ld;
      double v0 = 0.0, v1 = 0.0;
      if (FIRST) {
        v0 = lane > j ? v[lane] : (lane == j ? 1.0 : 0.0);
        v1 = lane + 32 > j ? v[lane + 32] : (lane + 32 == j ? 1.0 : 0.0);
      }
      double vc[BR_RPL];
#pragma unroll
      for (int t = 0; t < BR_RPL; ++t) vc[t] = v[roff + 32 * t + lane];
      // inactive target columns are zero and stay zero: no branches, reductions interleaved
      double dt[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        // later stacks: the reflector's R-block part is e_j (row j held by lane j & 31)
        const double rpart = FIRST ? (v0 * tr[0][s] + v1 * tr[1][s])
                                   : (lane == (j & 31) ? (j < 32 ? tr[0][s] : tr[1][s]) : 0.0);
        double q = rpart + (vc[0] * tc[0][s] + vc[1] * tc[1][s]);
#pragma unroll
        for (int t = 2; t < BR_RPL; ++t) q += vc[t] * tc[t][s];
        dt[s] = q;
      }
      if constexpr (NS == 2) {
        warp_sum2(dt);
      } else {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int s = 0; s < NS; ++s) dt[s] += __shfl_xor_sync(0xffffffffu, dt[s], o);
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const double w = tau * dt[s];
        if (FIRST) {
          tr[0][s] -= w * v0;
          tr[1][s] -= w * v1;
        } else if (lane == (j & 31)) {
          if (j < 32) tr[0][s] -= w; else tr[1][s] -= w;
        }
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) tc[t][s] -= w * vc[t];
      }
    }
  }
}

// out(row, col) = Q [T; 0] for the m-row factor whose stacks are at V (taus Tq, ncol reflectors
// per stack); this warp's target columns col0 + 8 s + warp (s < 4, col < ntgt) with the R-block
// rows of T in tr on entry.  Output address: out[row * rs + col * cs].
template <int NS>
__device__ __noinline__ void br_apply_q(double (&tr)[2][NS], const double* V, const double* Tq, int64_t m, int ncol,
                                        int col0, int ntgt, double* out, int64_t rs, int64_t cs, VStage& vs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nst = br_stacks(m);
  uint32_t ph[2] = {vs.phase[0], vs.phase[1]};
  double tc[BR_RPL][NS];
#pragma unroll 1
  for (int q = nst - 1; q >= 0; --q) {
#pragma unroll
    for (int t = 0; t < BR_RPL; ++t)
#pragma unroll
      for (int s = 0; s < NS; ++s) tc[t][s] = 0.0;
    if (q == 0) br_stack_apply<NS, true>(tr, tc, V + br_stack_off(q, ncol), Tq + (int64_t)q * BR_C, q, ncol, ntgt - col0, vs, ph);
    else br_stack_apply<NS, false>(tr, tc, V + br_stack_off(q, ncol), Tq + (int64_t)q * BR_C, q, ncol, ntgt - col0, vs, ph);
    const int64_t base = q == 0 ? BR_C : BR_S0 + (int64_t)BR_CH * (q - 1);
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int col = col0 + s * BR_W + warp;
      if (col < ntgt) {
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) {
          const int64_t row = base + 32 * t + lane;
          if (row < m) out[row * rs + col * cs] = tc[t][s];
        }
        if (q == 0) {
          if (lane < m) out[(int64_t)lane * rs + col * cs] = tr[0][s];
          if (lane + 32 < m) out[(int64_t)(lane + 32) * rs + col * cs] = tr[1][s];
        }
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) { vs.phase[0] = ph[0]; vs.phase[1] = ph[1]; }
  __syncthreads();
}

// Q [T; 0] for the rho target columns stored in src (column-major, ld 64, rows < cp), in passes
// of 8 BR_APPLY_NS columns (BR_APPLY_NS per warp: 2 keeps the application within 80 registers
// at 3 CTAs per SM without spilling; more passes re-stream the reflectors from L2).
__device__ void br_apply_targets(const double* __restrict__ src, int rho, int cp, const double* V, const double* Tq,
                                 int64_t m, int ncol, double* out, int64_t rs, int64_t cs, VStage& vs) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll 1
  for (int col0 = 0; col0 < rho; col0 += BR_APPLY_NS * BR_W) {
    double tr[2][BR_APPLY_NS];
#pragma unroll
    for (int s = 0; s < BR_APPLY_NS; ++s) {
      const int col = col0 + s * BR_W + warp;
      const bool ok = col < rho;
      tr[0][s] = (ok && lane < cp) ? src[col * BR_C + lane] : 0.0;
      tr[1][s] = (ok && lane + 32 < cp) ? src[col * BR_C + lane + 32] : 0.0;
    }
    br_apply_q(tr, V, Tq, m, ncol, col0, rho, out, rs, cs, vs);
  }
}

// Flat-tree QR of an m x ncol matrix given by elem(row, col) (zero outside); reflectors to V,
// taus to Tq; on return sm.Rs holds R (upper triangle; strictly lower part zero).
template <class Elem>
__device__ __noinline__ void br_qr(const Elem& elem, int64_t m, int ncol, BRSmem& sm, double* V, double* Tq,
                                   long long* dbg) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nst = br_stacks(m);
  long long c0 = clock64();
  double a[BR_RPL][BR_CPW];
#pragma unroll 1
  for (int q = 0; q < nst; ++q) {
    if (q == 0) {
      for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) {
        const int col = idx / BR_C, row = idx % BR_C;
        sm.Rs[idx] = (row < m && col < ncol) ? elem(row, col) : 0.0;
      }
    }
    const int64_t base = q == 0 ? BR_C : BR_S0 + (int64_t)BR_CH * (q - 1);
    elem.chunk(a, base, m, ncol);
    __syncthreads();
    const long long c1 = clock64();
    if (q == 0) br_stack_qr_first(a, sm, ncol, Tq, dbg ? dbg + 16 : nullptr);
    else if (dbg) br_stack_qr_later(a, sm, ncol, Tq + (int64_t)q * BR_C, dbg + 16);  // (debug counters)
    else br_stack_qr_later_async(a, sm, ncol, Tq + (int64_t)q * BR_C);
    const long long c2 = clock64();
    br_store_stack(a, sm, q, ncol, V + br_stack_off(q, ncol));
    if (dbg && tid == 0) { dbg[0] += c1 - c0; dbg[1] += c2 - c1; dbg[2] += clock64() - c2; }
    c0 = clock64();
  }
}

// A_k[(i, b'), col] = sum_beta L_{k+1}[b', off_l + beta] X_k^(l)[a, i, beta], col = off_{k-1,l} + a;
// for k = d: c_l X_d^(l)[a, i, 0].  LT (smem) = L^T, column-major ld 64 (LT[c*64 + b']).
struct PanelElem {
  const double* const* cores;  // this item's [l][kc]
  const BRShape* sh;
  const double* LT;
  double* xst;                 // BR_W x 32 staging (shared memory)
  const int* cterm;
  const int* ca;
  int kc, d, n, Rpk, last;
  __device__ double operator()(int64_t row, int col) const {
    const int i = (int)(row / Rpk), bp = (int)(row % Rpk);
    const int l = cterm[col], aa = ca[col];
    const double* X = cores[l * d + kc];
    if (last) return LT[l * BR_C] * __ldg(X + (int64_t)aa * n + i);
    const int rl = sh->r[l][kc + 1], o = sh->off[kc + 1][l];
    const double* xp = X + ((int64_t)aa * n + i) * rl;
    const double* lp = LT + (int64_t)o * BR_C + bp;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;  // four chains: loads in flight together
    int be = 0;
    for (; be + 4 <= rl; be += 4) {
      s0 += lp[be * BR_C] * __ldg(xp + be);
      s1 += lp[(be + 1) * BR_C] * __ldg(xp + be + 1);
      s2 += lp[(be + 2) * BR_C] * __ldg(xp + be + 2);
      s3 += lp[(be + 3) * BR_C] * __ldg(xp + be + 3);
    }
    for (; be < rl; ++be) s0 += lp[be * BR_C] * __ldg(xp + be);
    return (s0 + s1) + (s2 + s3);
  }

  // chunk loader: per column (term l, index a) the four rows' beta sums run as four
  // independent chains (loads of both operands in flight together)
  __device__ void chunk(double (&a)[BR_RPL][BR_CPW], int64_t base, int64_t m, int ncol) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // rows of this lane: row_t = base + 32 t + lane -> (i_t, b'_t); packed in one int each
    int ib[BR_RPL];
#pragma unroll
    for (int t = 0; t < BR_RPL; ++t) {
      const int64_t row = base + 32 * t + lane;
      ib[t] = row < m ? (int)((row / Rpk) << 8 | (row % Rpk)) : -1;
    }
    // the chunk's rows cover mode indices i in [ilo, ilo + ni): per column the ni x rl term-core
    // values X(a, i, beta) are loaded once, one per lane, into the warp's staging row, instead of
    // one dependent L2 load per (row, beta) in the FMA loop (the term cores do not fit in L1)
    const int64_t rlast = (base + BR_CH < m ? base + BR_CH : m) - 1;
    const int ilo = (int)(base / Rpk), ni = rlast >= base ? (int)(rlast / Rpk) - ilo + 1 : 0;
    int xi[BR_RPL];
#pragma unroll
    for (int t = 0; t < BR_RPL; ++t) xi[t] = ib[t] < 0 ? 0 : (ib[t] >> 8) - ilo;
    double* xw = xst + warp * 32;
#pragma unroll
    for (int s = 0; s < BR_CPW; ++s) {
      const int col = s * BR_W + warp;
      if (col >= ncol) {
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) a[t][s] = 0.0;
        continue;
      }
      const int l = cterm[col], aa = ca[col];
      const double* X = cores[l * d + kc];
      if (last) {
        const double c = LT[l * BR_C];
#pragma unroll
        for (int t = 0; t < BR_RPL; ++t) a[t][s] = ib[t] >= 0 ? c * __ldg(X + (int64_t)aa * n + (ib[t] >> 8)) : 0.0;
        continue;
      }
      const int rl = sh->r[l][kc + 1], o = sh->off[kc + 1][l];
      const double* xa = X + (int64_t)aa * n * rl;
      double acc[BR_RPL];
#pragma unroll
      for (int t = 0; t < BR_RPL; ++t) acc[t] = 0.0;
      if (ni * rl <= 32) {
        __syncwarp();
        if (lane < ni * rl) xw[lane] = __ldg(xa + (int64_t)(ilo + lane / rl) * rl + lane % rl);
        __syncwarp();
#pragma unroll 2
        for (int be = 0; be < rl; ++be) {
          const double* lrow = LT + (int64_t)(o + be) * BR_C;
#pragma unroll
          for (int t = 0; t < BR_RPL; ++t) {
            const int q = ib[t] < 0 ? 0 : ib[t];
            acc[t] += lrow[q & 255] * xw[xi[t] * rl + be];
          }
        }
      } else {
#pragma unroll 2
        for (int be = 0; be < rl; ++be) {
          const double* lrow = LT + (int64_t)(o + be) * BR_C;
#pragma unroll
          for (int t = 0; t < BR_RPL; ++t) {
            const int q = ib[t] < 0 ? 0 : ib[t];
            acc[t] += lrow[q & 255] * __ldg(xa + (int64_t)(q >> 8) * rl + be);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < BR_RPL; ++t) a[t][s] = ib[t] >= 0 ? acc[t] : 0.0;
    }
  }
};

// Y_1[i, b'] = sum_{l, beta} X_1^(l)[0, i, beta] L_2[b', off_{1,l} + beta]
struct FirstElem {
  const double* const* cores;
  const BRShape* sh;
  const double* LT;
  int d, K;
  __device__ double operator()(int64_t row, int col) const {
    double s = 0.0;
    for (int l = 0; l < K; ++l) {
      const int rl = sh->r[l][1], o = sh->off[1][l];
      const double* xp = cores[l * d] + row * rl;
      const double* lp = LT + (int64_t)o * BR_C + col;
      for (int be = 0; be < rl; ++be) s += lp[be * BR_C] * __ldg(xp + be);
    }
    return s;
  }

  // chunk rows base + 32t + lane, columns 8s + warp (zero outside the matrix)
  __device__ void chunk(double (&a)[BR_RPL][BR_CPW], int64_t base, int64_t m, int ncol) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int s = 0; s < BR_CPW; ++s) {
      const int col = s * BR_W + warp;
#pragma unroll
      for (int t = 0; t < BR_RPL; ++t) {
        const int64_t row = base + 32 * t + lane;
        a[t][s] = (row < m && col < ncol) ? (*this)(row, col) : 0.0;
      }
    }
  }
};

struct RowMajorElem {  // Y[row, col] = Z[row * ld + col]
  const double* Z;
  int ld;
  __device__ double operator()(int64_t row, int col) const { return Z[row * ld + col]; }

  // chunk rows base + 32t + lane, columns 8s + warp (zero outside the matrix)
  __device__ void chunk(double (&a)[BR_RPL][BR_CPW], int64_t base, int64_t m, int ncol) const {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int s = 0; s < BR_CPW; ++s) {
      const int col = s * BR_W + warp;
#pragma unroll
      for (int t = 0; t < BR_RPL; ++t) {
        const int64_t row = base + 32 * t + lane;
        a[t][s] = (row < m && col < ncol) ? (*this)(row, col) : 0.0;
      }
    }
  }
};

// Load L^T (rows x cols of the row-major ld-64 L) into sm.Aux: Aux[c * 64 + b'] = L[b' * 64 + c].
__device__ void br_load_lt(BRSmem& sm, const double* L, int rows, int cols) {
  for (int idx = threadIdx.x; idx < BR_C * BR_C; idx += BR_T) {
    const int c = idx / BR_C, bp = idx % BR_C;
    sm.Aux[idx] = (bp < rows && c < cols) ? L[bp * BR_C + c] : 0.0;
  }
}

__global__ void __launch_bounds__(BR_T, 2) br_r2l_kernel(BRArgs A, int kc) {
  extern __shared__ __align__(16) unsigned char br_smem_raw[];
  BRSmem& sm = *reinterpret_cast<BRSmem*>(br_smem_raw);
  const BRShape* S = A.sh;
  const int b = blockIdx.x + A.b0, gb = A.item0 + b;
  const int d = S->d, K = S->K;
  const int k = kc + 1;                 // 1-based core index, 2..d
  const int n = S->n[kc], Rpk = S->Rp[k], c = S->R[k - 1];
  const int64_t m = (int64_t)n * Rpk;
  const bool last = (k == d);
  const int tid = threadIdx.x;
  if (tid < BR_C) {
    int l = 0;
    while (l + 1 < K && tid >= S->off[k - 1][l + 1]) ++l;
    sm.cterm[tid] = l;
    sm.ca[tid] = tid - S->off[k - 1][l];
  }
  if (last) {
    for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) sm.Aux[idx] = 0.0;
    __syncthreads();
    if (tid < K) sm.Aux[tid * BR_C] = A.coef[(int64_t)gb * K + tid];
  } else {
    br_load_lt(sm, A.L + (int64_t)b * 2 * BR_C * BR_C + ((k + 1) & 1) * BR_C * BR_C, Rpk, S->R[k]);
  }
  __syncthreads();
  PanelElem e{A.cores + (int64_t)gb * K * d, S, sm.Aux, &sm.xst[0][0], sm.cterm, sm.ca, kc, d, n, Rpk, last ? 1 : 0};
  double* V = A.V + (int64_t)b * S->vstride + S->voff[kc];
  double* Tq = A.T + (int64_t)b * S->tstride + S->toff[kc];
  br_qr(e, m, c, sm, V, Tq, (A.dbg && blockIdx.x == 0) ? A.dbg + 32 : nullptr);
  // R (R'_{k-1} x c, row-major ld 64) -> L slot (k & 1)
  double* Lout = A.L + (int64_t)b * 2 * BR_C * BR_C + (k & 1) * BR_C * BR_C;
  const int rows = S->Rp[k - 1];
  for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) {
    const int row = idx / BR_C, col = idx % BR_C;
    Lout[idx] = (row < rows && col < c && row <= col) ? sm.Rs[col * BR_C + row] : 0.0;
  }
}

// One-sided (Hestenes) Jacobi SVD of the rows x nc matrix in sm.Rs (column-major, ld 64),
// round-robin pair ordering, one warp per pair; V (nc x nc) in sm.Aux.  On return
// sm.sig[j] = j-th largest singular value, sm.perm[j] = its column; returns false on
// non-convergence (|<c_i,c_j>| <= sqrt(rows) u ||c_i|| ||c_j||).
// Pairs whose columns both have squared norm <= tail2 (tail2 = tau^2 / nc: even all such columns
// together lie inside the truncation tail) are not rotated: their mutual orthogonality is never
// used.  The big-small pairs still converge, so the small columns span the orthogonal
// complement of the kept subspace and their squared norms sum to the exact tail mass: the rank
// decision, U_rho and S V^T are those of the full Jacobi.
// LPP lanes per column pair (8, 16 or 32: 4, 2 or 1 pairs per warp), each lane holding 64 / LPP
// rows -- the caller picks LPP so that a round's kk / 2 pairs fill the 8 warps.
template <int LPP>
__device__ __forceinline__ bool br_jacobi_rounds(BRSmem& sm, int nc, double tol, double negl, double tail2,
                                                 long long* nsweeps) {
  constexpr int RPL = BR_C / LPP, NPW = 32 / LPP;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kk = nc + (nc & 1);
  bool conv = nc < 2;
#pragma unroll 1
  // Squared column norms are kept in n2 across a sweep (a rotation by t = tan(theta) that zeroes
  // gamma moves them to alpha - t gamma and beta + t gamma) and recomputed exactly when a sweep
  // starts -- so the sweep that declares convergence (no rotation at all) tests exact norms, and a
  // rotation costs one dot product and one reduction instead of three.
  double* n2 = sm.vb[1];
  const double tol2 = tol * tol;
  // A sweep whose rotations were all tiny also ends the iteration (no confirming sweep): with
  // rho_ij = |<c_i, c_j>| / (||c_i|| ||c_j||), a rotation of (p, q) moves rho_pj by at most
  // kappa rho_qj, kappa = |sin| max(||c_p|| / ||c_q||, ||c_q|| / ||c_p||).  If every pair had
  // rho <= e at its visit and every rotation kappa <= e, e^2 = tol / (32 kk), then no rho exceeds
  // 2 e during the sweep (2 kk e << 1) and each drifts by at most 2 kk e 2 e = tol / 8 after its
  // visit: all pairs end at <= 1.125 tol (A23).
  const double tiny2 = tol / (32.0 * (double)kk);
  for (int sweep = 0; sweep < BR_JAC_SWEEPS && !conv; ++sweep) {
    for (int j = warp; j < nc; j += BR_W) {
      const double x0 = sm.Rs[j * BR_C + lane], x1 = sm.Rs[j * BR_C + lane + 32];
      const double sq = warp_sum(x0 * x0 + x1 * x1);
      if (lane == 0) n2[j] = sq;
    }
    // Small-small pairs are skipped for the first 12 sweeps only: when the threshold falls inside a
    // cluster (tau at the noise level of a cancelling sum), skipped pairs of strongly correlated
    // small columns couple the big-small rotations to first order and the iteration turns linear;
    // from sweep 12 on every pair rotates (plain one-sided Jacobi, quadratic again).
    const double tl2 = sweep < 12 ? tail2 : -1.0;
    if (tid == 0) { sm.flag = 0; sm.rho = 0; }  // sm.rho: a rotation of this sweep was not tiny (below)
    __syncthreads();
#pragma unroll 1
    for (int r = 0; r < kk - 1; ++r) {
      // lane = LPP pp + rl holds rows LPP ((t + pp) mod RPL) + rl (the stagger keeps the pairs of
      // a warp on different banks)
      const int pp = lane / LPP, rl = lane % LPP;
      const int q = warp + pp * BR_W;
      int p0, p1;
      if (q == 0) { p0 = kk - 1; p1 = r; }
      else {  // (r + q) mod (kk - 1) and (r - q) mod (kk - 1): both sums lie below 2 (kk - 1)
        p0 = r + q; p1 = r + kk - 1 - q;
        if (p0 >= kk - 1) p0 -= kk - 1;
        if (p1 >= kk - 1) p1 -= kk - 1;
      }
      if (p0 > p1) { const int t = p0; p0 = p1; p1 = t; }
      const bool act = q < kk / 2 && p1 < nc && pp < NPW;
      double* ca = sm.Rs + (act ? p0 : 0) * BR_C;
      double* cb = sm.Rs + (act ? p1 : 0) * BR_C;
      double x[RPL], y[RPL];
#pragma unroll
      for (int t = 0; t < RPL; ++t) {
        const int row = LPP * ((t + pp) % RPL) + rl;
        x[t] = act ? ca[row] : 0.0;
        y[t] = act ? cb[row] : 0.0;
      }
      const double al = act ? n2[p0] : 0.0, be = act ? n2[p1] : 0.0;
      double ga = 0.0;
#pragma unroll
      for (int t = 0; t < RPL; ++t) ga += x[t] * y[t];
#pragma unroll
      for (int o = LPP / 2; o > 0; o >>= 1) ga += __shfl_xor_sync(0xffffffffu, ga, o);
      const bool rot = act && ga != 0.0 && al > negl && be > negl && (al > tl2 || be > tl2) &&
                       ga * ga > tol2 * (al * be);
      bool big = false;
      if (rot) {
        // tan(2 theta) = 2 gamma / (beta - alpha), the smaller angle: with h = hypot(dd, 2 gamma),
        // cos^2 = (1 + |dd| / h) / 2, sin = sgn gamma / (h cos), t = sin / cos -- no cancellation in
        // either, and two reciprocal square roots in sequence instead of sqrt -> divide -> rsqrt
        const double dd = be - al;
        const double gs = dd >= 0.0 ? ga : -ga;
        const double rh = rsqrt(dd * dd + 4.0 * ga * ga);
        const double c2 = 0.5 + 0.5 * (fabs(dd) * rh);
        const double rc = rsqrt(c2);
        const double cs = c2 * rc, sn = (gs * rh) * rc;
        const double t = sn * rc;
        big = ga * ga > tiny2 * (al * be) || sn * sn * fmax(al, be) > tiny2 * fmin(al, be);
        if (rl == 0) {
          n2[p0] = al - t * ga;
          n2[p1] = be + t * ga;
        }
        double* va = sm.Aux + p0 * BR_C;
        double* vbp = sm.Aux + p1 * BR_C;
#pragma unroll
        for (int u = 0; u < RPL; ++u) {
          const int row = LPP * ((u + pp) % RPL) + rl;
          ca[row] = cs * x[u] - sn * y[u];
          cb[row] = sn * x[u] + cs * y[u];
          if (row < nc) {  // V = Aux starts as I: rows >= nc of its first nc columns stay zero
            const double a0 = va[row], b0 = vbp[row];
            va[row] = cs * a0 - sn * b0;
            vbp[row] = sn * a0 + cs * b0;
          }
        }
      }
      if (__any_sync(0xffffffffu, rot)) {
        const bool anybig = __any_sync(0xffffffffu, big);
        if (lane == 0) { sm.flag = 1; if (anybig) sm.rho = 1; }
      }
      __syncthreads();
    }
    conv = (sm.flag == 0) || (sm.rho == 0);
    if (nsweeps && tid == 0) *nsweeps += 1;
    __syncthreads();
  }
  return conv;
}

__device__ __noinline__ bool br_jacobi(BRSmem& sm, int rows, int nc, double tail2, int lpp, long long* nsweeps = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) sm.Aux[idx] = (idx % BR_C == idx / BR_C) ? 1.0 : 0.0;
  const double tol = sqrt((double)max(rows, 1)) * U_ROUND;
  // Columns with ||c||_2 <= u ||A||_F are numerically zero: rotating them against the others
  // only shrinks them geometrically (each projection leaves rounding residue) and the
  // relative test never settles, so they are left alone (their sigma stays <= u ||A||_F).
  double fro = 0.0;
  for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) { const double v = sm.Rs[idx]; fro += v * v; }
  double fro2 = block_sum(fro, sm.red);
  // The rounds test products of squared norms (gamma^2 against alpha beta): a matrix whose
  // ||A||_F^2 is far from 1 is scaled by a power of two first (exact) and scaled back after the
  // rounds, so the tests neither underflow nor overflow for matrices whose squared norms are
  // representable (||A||_F within ~1e-150 .. 1e150); ordinary inputs skip both passes.
  int ek = (fro2 > 0.0 && fro2 <= 1.7e308) ? ilogb(fro2) / 2 : 0;
  ek = ek > 500 ? 500 : (ek < -500 ? -500 : ek);
  const bool scaled = ek >= 64 || ek <= -64;
  __syncthreads();  // block_sum's scratch is reused below
  if (scaled) {
    const double f = scalbn(1.0, -ek);
    for (int idx = tid; idx < BR_C * nc; idx += BR_T) sm.Rs[idx] *= f;
    fro2 *= f * f;
    tail2 *= f * f;
  }
  const double negl = fro2 * U_ROUND * U_ROUND;
  __syncthreads();
  const int pairs = (nc + (nc & 1)) / 2;
  bool conv;
  // lpp = 0: the widest layout whose pairs fill the 8 warps (shortest round); lpp = 8 / 16 / 32
  // forces a layout (fewer, fuller warps issue fewer instructions per round: TT_B200_BR_JLPP)
  if (lpp == 0) lpp = pairs <= BR_W ? 32 : pairs <= 2 * BR_W ? 16 : 8;
  if (lpp == 32 && pairs > BR_W) lpp = 16;
  if (lpp == 16 && pairs > 2 * BR_W) lpp = 8;
  if (lpp == 32) conv = br_jacobi_rounds<32>(sm, nc, tol, negl, tail2, nsweeps);
  else if (lpp == 16) conv = br_jacobi_rounds<16>(sm, nc, tol, negl, tail2, nsweeps);
  else conv = br_jacobi_rounds<8>(sm, nc, tol, negl, tail2, nsweeps);
  if (scaled) {
    const double f = scalbn(1.0, ek);
    for (int idx = tid; idx < BR_C * nc; idx += BR_T) sm.Rs[idx] *= f;
    __syncthreads();
  }
  // singular values = column norms, sorted descending (ties: lower column first)
  for (int j = warp; j < nc; j += BR_W) {
    const double x0 = sm.Rs[j * BR_C + lane], x1 = sm.Rs[j * BR_C + lane + 32];
    const double s = warp_sum(x0 * x0 + x1 * x1);
    if (lane == 0) sm.vb[0][j] = sqrt(s);
  }
  __syncthreads();
  if (tid < nc) {
    const double v = sm.vb[0][tid];
    int rk = 0;
    for (int i = 0; i < nc; ++i) {
      const double w = sm.vb[0][i];
      if (w > v || (w == v && i < tid)) ++rk;
    }
    sm.sig[rk] = v;
    sm.perm[rk] = tid;
  }
  __syncthreads();
  return conv;
}

// Column-pivoted Householder QR of the rows x nc matrix X in sm.Rs (column-major, ld 64), stopped
// at the first step s whose remaining columns carry squared mass <= stop2 (LAPACK dlaqp2
// arithmetic; masses recomputed exactly after every step, no downdating).  Reflectors below the
// diagonal, taus in tau_s[], pivot order in piv[] (pivoted column j = original column piv[j]);
// returns the number of steps k, the remaining mass in *e2.  Warp w owns the columns j = w mod 8.
__device__ int br_qrcp(BRSmem& sm, int rows, int nc, double stop2, double* tau_s, int* piv, double* nrm2,
                       double* e2) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = warp; j < nc; j += BR_W) {
    const double x0 = sm.Rs[j * BR_C + lane], x1 = sm.Rs[j * BR_C + lane + 32];
    const double q = warp_sum(x0 * x0 + x1 * x1);
    if (lane == 0) { nrm2[j] = q; piv[j] = j; }
  }
  __syncthreads();
  int s = 0;
#pragma unroll 1
  for (; s < nc && s < rows; ++s) {
    if (warp == 0) {  // remaining mass and the pivot (largest mass, lowest index on ties)
      const int j0 = s + lane, j1 = s + lane + 32;
      const double v0 = j0 < nc ? nrm2[j0] : -1.0, v1 = j1 < nc ? nrm2[j1] : -1.0;
      double tot = (v0 > 0.0 ? v0 : 0.0) + (v1 > 0.0 ? v1 : 0.0);
      double bv = v1 > v0 ? v1 : v0;
      int bj = v1 > v0 ? j1 : j0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        tot += __shfl_xor_sync(0xffffffffu, tot, o);
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ov > bv || (ov == bv && oj < bj)) { bv = ov; bj = oj; }
      }
      if (lane == 0) { sm.red[0] = tot; sm.flag = bj; }
    }
    __syncthreads();
    const double tot = sm.red[0];
    const int p = sm.flag;
    if (tot <= stop2) break;
    if (p != s) {  // swap columns s and p
      for (int r = tid; r < BR_C; r += BR_T) {
        const double t = sm.Rs[s * BR_C + r];
        sm.Rs[s * BR_C + r] = sm.Rs[p * BR_C + r];
        sm.Rs[p * BR_C + r] = t;
      }
      if (tid == 0) {
        const double t = nrm2[s]; nrm2[s] = nrm2[p]; nrm2[p] = t;
        const int ti = piv[s]; piv[s] = piv[p]; piv[p] = ti;
      }
      __syncthreads();
    }
    if (warp == (s & (BR_W - 1))) {  // reflector of column s, rows s..63 (dlarfg)
      double* cs = sm.Rs + s * BR_C;
      const double x0 = cs[lane], x1 = cs[lane + 32];
      const double sig = warp_sum((lane > s ? x0 * x0 : 0.0) + (lane + 32 > s ? x1 * x1 : 0.0));
      const double alpha = cs[s];
      double beta = alpha, tau = 0.0, scal = 0.0;
      if (sig != 0.0) {
        const double nr = sqrt(alpha * alpha + sig);
        beta = alpha >= 0.0 ? -nr : nr;
        const double am = alpha - beta;
        const double inv = 1.0 / (beta * am);
        tau = -am * am * inv;
        scal = beta * inv;
      }
      __syncwarp();
      if (lane > s) cs[lane] = x0 * scal;
      if (lane + 32 > s) cs[lane + 32] = x1 * scal;
      if (lane == 0) { cs[s] = beta; tau_s[s] = tau; }
    }
    __syncthreads();
    const double tau = tau_s[s];
    const double* v = sm.Rs + s * BR_C;
    const double v0 = lane > s ? v[lane] : (lane == s ? 1.0 : 0.0);
    const double v1 = lane + 32 > s ? v[lane + 32] : (lane + 32 == s ? 1.0 : 0.0);
    {  // this warp's columns j > s (j = j0 + 8 t, at most 8): dots and masses through one
       // transposed butterfly each instead of two warp reductions per column
      const int j0 = s + 1 + ((warp - s - 1) & (BR_W - 1));
      const int ncj = j0 < nc ? (nc - j0 + BR_W - 1) / BR_W : 0;
      double x0[8], x1[8], dq[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double* cj = sm.Rs + (t < ncj ? j0 + BR_W * t : 0) * BR_C;
        x0[t] = t < ncj ? cj[lane] : 0.0;
        x1[t] = t < ncj ? cj[lane + 32] : 0.0;
      }
      if (tau != 0.0 && ncj > 0) {
#pragma unroll
        for (int t = 0; t < 8; ++t) dq[t] = v0 * x0[t] + v1 * x1[t];
        wy::warp_sum8v(dq);
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const double w = tau * dq[t];
          x0[t] -= w * v0;
          x1[t] -= w * v1;
          if (t < ncj) {
            double* cj = sm.Rs + (j0 + BR_W * t) * BR_C;
            cj[lane] = x0[t];
            cj[lane + 32] = x1[t];
          }
        }
      }
      if (ncj > 0) {
#pragma unroll
        for (int t = 0; t < 8; ++t) dq[t] = (lane > s ? x0[t] * x0[t] : 0.0) + (lane + 32 > s ? x1[t] * x1[t] : 0.0);
        wy::warp_sum8v(dq);
        if (lane == 0)
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (t < ncj) nrm2[j0 + BR_W * t] = dq[t];
      }
    }
    __syncthreads();
  }
  double rest = 0.0;
  for (int j = s; j < nc; ++j) rest += nrm2[j];
  *e2 = rest;
  return s;
}

// y (64-vector in shared or global memory, per warp) <- Q [y] with Q = H_0 .. H_{k-1} the
// reflectors stored below the diagonal of F (column-major ld 64) and taus t (H_{k-1} applied first).
__device__ __forceinline__ void br_apply_qx(double& y0, double& y1, const double* __restrict__ F,
                                            const double* __restrict__ t, int k) {
  const int lane = threadIdx.x & 31;
#pragma unroll 1
  for (int i = k - 1; i >= 0; --i) {
    const double tau = t[i];
    if (tau == 0.0) continue;
    const double* v = F + i * BR_C;
    const double v0 = lane > i ? v[lane] : (lane == i ? 1.0 : 0.0);
    const double v1 = lane + 32 > i ? v[lane + 32] : (lane + 32 == i ? 1.0 : 0.0);
    const double w = tau * warp_sum(v0 * y0 + v1 * y1);
    y0 -= w * v0;
    y1 -= w * v1;
  }
}

// ---- left-to-right step at split k, in three launches over the batch:
//   br_l2r_qr_kernel     Y_k -> (tall: flat-tree QR, reflectors to YV/YT) -> Jacobi input JM;
//                        split 1 also computes ||x|| and tau
//   br_l2r_svd_kernel    one-sided Jacobi of JM, rank rho_k, targets U_rho and V_rho S to TT
//                        (short Y_k: output core k written directly)
//   br_l2r_apply_kernel  output core k = Q_Y [U_rho; 0] and Z_{k+1} = H_{k+1} [(S V^T)^T; 0]
// (split so that the register-light Jacobi and applications run three CTAs per SM).
__global__ void __launch_bounds__(BR_T, 2) br_l2r_qr_kernel(BRArgs A, int k) {
  extern __shared__ __align__(16) unsigned char br_smem_raw[];
  BRSmem& sm = *reinterpret_cast<BRSmem*>(br_smem_raw);
  const BRShape* S = A.sh;
  const int b = blockIdx.x + A.b0, gb = A.item0 + b;
  const int d = S->d, K = S->K;
  const int kc = k - 1;
  const int tid = threadIdx.x;
  int* rk = A.ranks + (int64_t)b * (d + 1);
  double* sc = A.scal + (int64_t)b * 4;
  double* out = A.out + (int64_t)b * S->ostride;
  const int n = S->n[kc], cp = S->Rp[k];
  if (k > 1 && sc[3] != 0.0) {  // ||x|| = 0: rank-1 zero tensor
    for (int i = tid; i < n; i += BR_T) out[S->ooff[kc] + i] = 0.0;
    if (k + 1 == d)
      for (int i = tid; i < S->n[d - 1]; i += BR_T) out[S->ooff[d - 1] + i] = 0.0;
    if (tid == 0) { rk[k] = 1; if (k + 1 == d) rk[d] = 1; }
    return;
  }
  const int64_t p = (k == 1) ? (int64_t)n : (int64_t)rk[k - 1] * n;
  double* YV = A.YV + (int64_t)b * S->ystride;
  double* YT = A.YT + (int64_t)b * S->ytstride;
  const bool tall = p > BR_C;
  if (k == 1) {
    br_load_lt(sm, A.L + (int64_t)b * 2 * BR_C * BR_C + 0, cp, S->R[1]);  // L_2 lives in slot 0
    __syncthreads();
    FirstElem e{A.cores + (int64_t)gb * K * d, S, sm.Aux, d, K};
    if (tall) br_qr(e, p, cp, sm, YV, YT, (A.dbg && blockIdx.x == 0) ? A.dbg + 4 : nullptr);
    else {
      for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) {
        const int col = idx / BR_C, row = idx % BR_C;
        sm.Rs[idx] = (row < p && col < cp) ? e(row, col) : 0.0;
      }
      __syncthreads();
    }
  } else {
    RowMajorElem e{A.Z + (int64_t)b * 2 * S->zstride + (k & 1) * S->zstride, cp};
    if (tall) br_qr(e, p, cp, sm, YV, YT, (A.dbg && blockIdx.x == 0) ? A.dbg + 4 : nullptr);
    else {
      for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) {
        const int col = idx / BR_C, row = idx % BR_C;
        sm.Rs[idx] = (row < p && col < cp) ? e(row, col) : 0.0;
      }
      __syncthreads();
    }
  }
  if (k == 1) {
    double q = 0.0;
    for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) { const double v = sm.Rs[idx]; q += v * v; }
    const double nrm = sqrt(block_sum(q, sm.red));
    if (tid == 0) {
      const double s = A.scale[gb];
      double tau = 0.0;
      if (!A.keep_all) tau = fmax(A.rel_tol * nrm / sqrt((double)(d - 1)), A.floor_c * U_ROUND * s);
      sc[0] = nrm;
      sc[1] = tau;
      sc[2] = s;
      sc[3] = nrm == 0.0 ? 1.0 : 0.0;
      rk[0] = 1;
      rk[d] = 1;
    }
    if (nrm == 0.0) {
      for (int i = tid; i < n; i += BR_T) out[S->ooff[0] + i] = 0.0;
      if (d == 2)
        for (int i = tid; i < S->n[1]; i += BR_T) out[S->ooff[1] + i] = 0.0;
      if (tid == 0) { rk[1] = 1; rk[d] = 1; }
      return;
    }
  }
  double* jm = A.JM + (int64_t)b * BR_C * BR_C;
  for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) jm[idx] = sm.Rs[idx];
}

__global__ void __launch_bounds__(BR_T, 3) br_l2r_svd_kernel(BRArgs A, int k) {
  extern __shared__ __align__(16) unsigned char br_smem_raw[];
  BRSmem& sm = *reinterpret_cast<BRSmem*>(br_smem_raw);
  const BRShape* S = A.sh;
  const int b = blockIdx.x + A.b0;
  const int d = S->d;
  const int kc = k - 1;
  const int tid = threadIdx.x;
  int* rk = A.ranks + (int64_t)b * (d + 1);
  const double* sc = A.scal + (int64_t)b * 4;
  if (sc[3] != 0.0) return;
  const int n = S->n[kc], cp = S->Rp[k];
  const int64_t p = (k == 1) ? (int64_t)n : (int64_t)rk[k - 1] * n;
  const bool tall = p > BR_C;
  const int jrows = tall ? cp : (int)p;
  const double* jm = A.JM + (int64_t)b * BR_C * BR_C;
  // Tall splits: Jacobi on X = R_Y^T (R_Y = W S V^T  <=>  X = V S W^T): the accumulated rotations
  // are R_Y's left singular vectors W (what Q_Y is applied to), the rotated columns are V S
  // (the next core's target, no division) -- and the rows of the triangular factor converge in
  // fewer sweeps than its columns.
  const bool jt = tall && A.jac_t;
  for (int idx = tid; idx < BR_C * BR_C; idx += BR_T)
    sm.Rs[idx] = jt ? jm[(idx % BR_C) * BR_C + idx / BR_C] : jm[idx];
  __syncthreads();
  static_assert(BR_C == 64, "QRCP path assumes 64-row columns");
  if (jt && !A.keep_all && A.max_rank <= 0 && A.qrcp_svd) {
    // Truncated SVD through a rank-revealing QR of X = R_Y^T: X P = Q_X [T; E]
    // with ||E||_F^2 = e2 <= (theta tau)^2, theta = 1e-3, then one-sided Jacobi on T^T (cp x kq,
    // kq ~ the kept rank instead of 64).  Ky Fan: tail(rho)^2 lies in [sum_{j>=rho} sigma_j(T)^2,
    // that + e2], so the decision equals the exact-SVD decision unless tau^2 falls inside the
    // interval for rho - 1 (then the full Jacobi below decides).  U_rho (R_Y's left vectors) =
    // P (T^T J) / sigma, V_rho S = Q_X [J Sigma; 0] (or Q_X [J Sigma^-1; 0] for U = Y W).
    const double tau = sc[1];
    double* qx = A.QX + (int64_t)b * (BR_C * BR_C + BR_C);
    double* taus = sm.vb[1];
    double* nrm2 = sm.vb[0];
    double e2 = 0.0;
    const bool prof = A.dbg && blockIdx.x == 0 && tid == 0;  // CTA 0 phase cycles (TT_B200_BR_DEBUG)
    long long pt = prof ? clock64() : 0;
    // theta = min(1e-3, 1e-7 ||x|| / tau): the left vectors of [T^T E^T] are those of T^T up to
    // ||E||^2 / gap (M M^T = T^T T + E^T E), so (theta tau)^2 <= 1e-14 ||x||^2 keeps that
    // perturbation within ~100 u ||x||^2 / gap of the exact SVD's own sensitivity, for any delta;
    // the first-order term E U~ enters the next core's target below.
    const double th = fmin(1e-3, 1e-7 * sc[0] / tau);
    const int kq = br_qrcp(sm, cp, cp, th * th * tau * tau, taus, sm.cterm, nrm2, &e2);
    if (prof) { const long long t = clock64(); A.dbg[80] += t - pt; A.dbg[84] += kq; A.dbg[85] += 1; pt = t; }
    for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) qx[idx] = sm.Rs[idx];
    if (tid < BR_C) qx[BR_C * BR_C + tid] = tid < kq ? taus[tid] : 0.0;
    __syncthreads();
    for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) {  // C = T^T: column i = row i of T (j >= i)
      const int i = idx / BR_C, j = idx % BR_C;
      sm.Rs[idx] = (i < kq && j < cp && j >= i) ? qx[j * BR_C + i] : 0.0;
    }
    __syncthreads();
    const bool conv = kq < 1 || br_jacobi(sm, cp, kq, tau * tau / (double)(kq > 0 ? kq : 1), A.jac_lpp,
                                          (A.dbg && blockIdx.x == 0) ? A.dbg + 11 : nullptr);
    if (prof) { const long long t = clock64(); A.dbg[81] += t - pt; pt = t; }
    if (tid == 0) {
      int rho = kq;
      double t2 = e2;
      for (int r = kq - 1; r >= 1; --r) {
        t2 += sm.sig[r] * sm.sig[r];
        if (t2 <= tau * tau) rho = r; else break;
      }
      rho = rho < 1 ? 1 : rho;
      double lo = 0.0;  // lower bound of the exact tail at rho - 1
      for (int r = rho - 1; r < kq; ++r) lo += sm.sig[r] * sm.sig[r];
      const bool amb = kq < 1 || (rho > 1 && lo <= tau * tau);
      if (!conv && !amb) A.info[b] = 1;
      sm.flag = amb ? 1 : 0;
      sm.rho = rho;
    }
    __syncthreads();
    if (!sm.flag) {
      const int rho = sm.rho;
      if (tid == 0) rk[k] = rho;
      const bool use_gemm = sm.sig[rho - 1] >= 1e-3 * sm.sig[0];
      if (tid == 0) A.gemm[b] = use_gemm ? 1 : 0;
      double* tt = A.TT + (int64_t)b * 2 * BR_C * BR_C;
      if (!use_gemm)  // U_rho = P (C J)[:, perm] / sigma  (C J = the rotated columns in Rs)
        for (int idx = tid; idx < BR_C * rho; idx += BR_T) {
          const int col = idx / BR_C, j = idx % BR_C;
          const double sg = sm.sig[col];
          if (j < cp) tt[col * BR_C + sm.cterm[j]] = sg > 0.0 ? sm.Rs[sm.perm[col] * BR_C + j] / sg : 0.0;
          else tt[col * BR_C + j] = 0.0;
        }
      // V_rho S = R_Y^T U_rho = Q_X [T; E] U~ = Q_X [J Sigma; E U~] (second slot) with U~ = C J / sigma
      // (pivoted coordinates; E = the unreduced trailing block left in qx: rows and columns >= kq)
      // and, for U = Y W, W = V_rho S Sigma^-2 = Q_X [J Sigma^-1; E U~ Sigma^-2] (first slot).
      // Targets of this warp: its columns col = warp + 8 i, each as J Sigma (second slot) and, for
      // U = Y W, J Sigma^-1 (first slot); up to 8 targets at a time take each reflector together
      // (one transposed butterfly per reflector for all of them).
      const int lane = tid & 31, warp = tid >> 5;
      // E (rows and columns >= kq of the QRCP remainder) into the columns of Aux that J leaves free
      for (int idx = tid + kq * BR_C; idx < cp * BR_C; idx += BR_T) sm.Aux[idx] = qx[idx];
      __syncthreads();
      const int ncw = rho > warp ? (rho - warp + BR_W - 1) / BR_W : 0;
      const int ntg = ncw * (use_gemm ? 2 : 1);
      const double* taus_x = qx + BR_C * BR_C;
#pragma unroll 1
      for (int g0 = 0; g0 < ntg; g0 += 8) {
        double y0[8], y1[8], dq[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int tg = g0 + t;
          const int col = warp + BR_W * (use_gemm ? tg >> 1 : tg);
          const bool live = tg < ntg;
          const double sg = live ? sm.sig[col] : 0.0;
          const double f = (use_gemm && (tg & 1)) ? (sg > 0.0 ? 1.0 / sg : 0.0) : sg;
          const int pc = live ? sm.perm[col] : 0;
          y0[t] = live && lane < kq ? sm.Aux[pc * BR_C + lane] * f : 0.0;
          y1[t] = live && lane + 32 < kq ? sm.Aux[pc * BR_C + lane + 32] * f : 0.0;
        }
        if (kq < cp) {  // rows >= kq: E U~ (times sigma^-2 for the W targets)
          const bool in0 = lane >= kq && lane < cp, in1 = lane + 32 >= kq && lane + 32 < cp;
          const double* ccol[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int tg = g0 + t;
            const int col = warp + BR_W * (use_gemm ? tg >> 1 : tg);
            ccol[t] = sm.Rs + (tg < ntg ? sm.perm[col] : 0) * BR_C;
          }
          if (use_gemm) {  // targets 2 u and 2 u + 1 share their column: one sum for both
#pragma unroll 1
            for (int j = kq; j < cp; ++j) {
              const double e0 = in0 ? sm.Aux[j * BR_C + lane] : 0.0;
              const double e1 = in1 ? sm.Aux[j * BR_C + lane + 32] : 0.0;
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const double c = ccol[2 * u][j];
                y0[2 * u] += e0 * c;
                y1[2 * u] += e1 * c;
              }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              if (in0) y0[2 * u + 1] = y0[2 * u];
              if (in1) y1[2 * u + 1] = y1[2 * u];
            }
          } else {
#pragma unroll 1
            for (int j = kq; j < cp; ++j) {
              const double e0 = in0 ? sm.Aux[j * BR_C + lane] : 0.0;
              const double e1 = in1 ? sm.Aux[j * BR_C + lane + 32] : 0.0;
#pragma unroll
              for (int t = 0; t < 8; ++t) {
                const double c = ccol[t][j];
                y0[t] += e0 * c;
                y1[t] += e1 * c;
              }
            }
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int tg = g0 + t;
            const int col = warp + BR_W * (use_gemm ? tg >> 1 : tg);
            const double sg = tg < ntg ? sm.sig[col] : 0.0;
            const double h = sg > 0.0 ? 1.0 / sg : 0.0;
            const bool wt = use_gemm && (tg & 1);  // one factor at a time: h^3 alone may overflow
            if (in0) { y0[t] *= h; if (wt) { y0[t] *= h; y0[t] *= h; } }
            if (in1) { y1[t] *= h; if (wt) { y1[t] *= h; y1[t] *= h; } }
          }
        }
#pragma unroll 1
        for (int i = kq - 1; i >= 0; --i) {  // Q_X = H_0 .. H_{kq-1}: H_{kq-1} first
          const double tau = taus_x[i];
          if (tau == 0.0) continue;
          const double* vq = qx + i * BR_C;
          const double v0 = lane > i ? vq[lane] : (lane == i ? 1.0 : 0.0);
          const double v1 = lane + 32 > i ? vq[lane + 32] : (lane + 32 == i ? 1.0 : 0.0);
#pragma unroll
          for (int t = 0; t < 8; ++t) dq[t] = v0 * y0[t] + v1 * y1[t];
          wy::warp_sum8v(dq);
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const double w = tau * dq[t];
            y0[t] -= w * v0;
            y1[t] -= w * v1;
          }
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int tg = g0 + t;
          if (tg < ntg) {
            const int col = warp + BR_W * (use_gemm ? tg >> 1 : tg);
            double* dst = tt + ((use_gemm && (tg & 1)) ? 0 : BR_C * BR_C) + col * BR_C;
            dst[lane] = lane < cp ? y0[t] : 0.0;
            dst[lane + 32] = lane + 32 < cp ? y1[t] : 0.0;
          }
        }
      }
      if (prof) A.dbg[82] += clock64() - pt;
      return;
    }
    if (prof) A.dbg[83] += 1;
    // ambiguous decision: the full Jacobi on X decides (reload R_Y^T)
    for (int idx = tid; idx < BR_C * BR_C; idx += BR_T) sm.Rs[idx] = jm[(idx % BR_C) * BR_C + idx / BR_C];
    __syncthreads();
  }
  const long long cj0 = clock64();
  static_assert(BR_C == 64, "tail2 below assumes nc <= 64");
  const double tail2 = (A.keep_all || A.max_rank > 0) ? 0.0 : sc[1] * sc[1] / (double)(cp > 0 ? cp : 1);
  const bool conv = br_jacobi(sm, jrows, cp, tail2, A.jac_lpp, (A.dbg && blockIdx.x == 0) ? A.dbg + 11 : nullptr);
  if (A.dbg && blockIdx.x == 0 && tid == 0) A.dbg[8] += clock64() - cj0;
  if (tid == 0) {
    if (!conv) A.info[b] = 1;
    const int nsv = (int)(p < cp ? p : cp);
    int rho = nsv;
    if (!A.keep_all) {
      const double tau = sc[1];
      // tail[rho] = sqrt(sum_{j >= rho} sigma_j^2), accumulated from the smallest value up
      double tail2 = 0.0;
      rho = nsv;
      // A short wide Y_k (more columns than rows) leaves cp - nsv columns that are zero in exact
      // arithmetic; with the small-small pairs not rotated they share the small columns' mass,
      // which belongs to the tail (only the group's total is exact).
      for (int r = cp - 1; r >= nsv; --r) tail2 += sm.sig[r] * sm.sig[r];
      for (int r = nsv - 1; r >= 1; --r) {
        tail2 += sm.sig[r] * sm.sig[r];
        if (sqrt(tail2) <= tau) rho = r; else break;
      }
    }
    if (A.max_rank > 0 && rho > A.max_rank) rho = (int)A.max_rank;
    rho = rho < 1 ? 1 : rho;
    sm.rho = rho;
    rk[k] = rho;
  }
  __syncthreads();
  const int rho = sm.rho;
  double* tt = A.TT + (int64_t)b * 2 * BR_C * BR_C;
  // Well-separated kept singular values (sigma_rho >= 1e-3 sigma_1): U_rho = Y V_rho S_rho^-1 is
  // accurate to u sigma_1 / sigma_rho <= 1e-13 and is a plain GEMM (DMMA) instead of applying
  // Q_Y's reflectors; W = V_rho S_rho^-1 goes to the first target slot.
  const bool use_gemm = tall && sm.sig[rho - 1] >= 1e-3 * sm.sig[0];
  if (tid == 0) A.gemm[b] = use_gemm ? 1 : 0;
  if (use_gemm) {  // V_rho S^-1
    for (int idx = tid; idx < BR_C * rho; idx += BR_T) {
      const int col = idx / BR_C, row = idx % BR_C;
      const double sg = sm.sig[col];
      tt[idx] = row < cp ? (jt ? sm.Rs[sm.perm[col] * BR_C + row] / (sg * sg) : sm.Aux[sm.perm[col] * BR_C + row] / sg)
                         : 0.0;
    }
  } else if (tall) {  // U_rho (cp x rho), the target of Q_Y
    for (int idx = tid; idx < BR_C * rho; idx += BR_T) {
      const int col = idx / BR_C, row = idx % BR_C;
      const double sg = sm.sig[col];
      tt[idx] = row >= cp ? 0.0
                          : jt ? sm.Aux[sm.perm[col] * BR_C + row]
                               : (sg > 0.0 ? sm.Rs[sm.perm[col] * BR_C + row] / sg : 0.0);
    }
  } else {  // short Y_k: output core k = U_rho directly ((rho_{k-1} n_k) x rho, row-major)
    double* ok = A.out + (int64_t)b * S->ostride + S->ooff[kc];
    for (int idx = tid; idx < p * rho; idx += BR_T) {
      const int row = idx / rho, col = idx % rho;
      const double sg = sm.sig[col];
      ok[idx] = sg > 0.0 ? sm.Rs[sm.perm[col] * BR_C + row] / sg : 0.0;
    }
  }
  for (int idx = tid; idx < BR_C * rho; idx += BR_T) {  // V_rho S (cp x rho), the target of H_{k+1}
    const int col = idx / BR_C, row = idx % BR_C;
    tt[BR_C * BR_C + idx] = row >= cp ? 0.0
                                      : jt ? sm.Rs[sm.perm[col] * BR_C + row]
                                           : sm.Aux[sm.perm[col] * BR_C + row] * sm.sig[col];
  }
}

// out (p x rho, row-major) = Y (p x cp, row-major ld cp) W (cp x rho, column-major ld 64) on the FP64
// tensor cores (mma.sync m8n8k4): warp w takes 8-row tiles w, w+8, ...; per tile the rho columns
// in 8-column tiles (accumulators in registers), K = cp in steps of 4.
__device__ void br_gemm_yw(const double* __restrict__ Y, int p, int cp, const double* __restrict__ W, int rho,
                           double* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ar = lane >> 2, ak = lane & 3;  // A fragment: row ar, k ak; B fragment: k ak, col ar
  const int nct = (rho + 7) / 8;            // <= 8 column tiles
#pragma unroll 1
  for (int rt = warp; rt * 8 < p; rt += BR_W) {
    const int row = rt * 8 + ar;
    double acc[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = 0.0;
#pragma unroll 1
    for (int k0 = 0; k0 < cp; k0 += 4) {
      const int kk = k0 + ak;
      const double a = (row < p && kk < cp) ? __ldg(Y + (int64_t)row * cp + kk) : 0.0;
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (c < nct) {
          const int col = c * 8 + ar;
          const double bv = (col < rho && kk < cp) ? __ldg(W + col * BR_C + kk) : 0.0;
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(acc[c][0]), "+d"(acc[c][1])
                       : "d"(a), "d"(bv));
        }
      }
    }
    // D fragment: row ar, columns 2 ak, 2 ak + 1 of each 8-column tile
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < nct && row < p) {
        const int col = c * 8 + 2 * ak;
        if (col < rho) out[(int64_t)row * rho + col] = acc[c][0];
        if (col + 1 < rho) out[(int64_t)row * rho + col + 1] = acc[c][1];
      }
    }
  }
}

struct BRSmemA {
  VStage vst;
};

__global__ void __launch_bounds__(BR_T, 3) br_l2r_apply_kernel(BRArgs A, int k) {
  extern __shared__ __align__(16) unsigned char br_smem_raw[];
  BRSmemA& sm = *reinterpret_cast<BRSmemA*>(br_smem_raw);
  const BRShape* S = A.sh;
  const int b = blockIdx.x + A.b0;
  const int d = S->d;
  const int kc = k - 1;
  const int tid = threadIdx.x;
  const int* rk = A.ranks + (int64_t)b * (d + 1);
  const double* sc = A.scal + (int64_t)b * 4;
  if (sc[3] != 0.0) return;
  if (tid == 0) {
    mbar_init(&sm.vst.bar[0], 1);
    mbar_init(&sm.vst.bar[1], 1);
    sm.vst.phase[0] = sm.vst.phase[1] = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  double* out = A.out + (int64_t)b * S->ostride;
  const int n = S->n[kc], cp = S->Rp[k];
  const int64_t p = (k == 1) ? (int64_t)n : (int64_t)rk[k - 1] * n;
  const bool tall = p > BR_C;
  const int rho = rk[k];
  const double* tt = A.TT + (int64_t)b * 2 * BR_C * BR_C;
  const long long co0 = clock64();
  if (tall && A.gemm[b]) {
    br_gemm_yw(A.Z + (int64_t)b * 2 * S->zstride + (k & 1) * S->zstride, (int)p, cp, tt, rho, out + S->ooff[kc]);
  } else if (tall) {
    const double* YV = A.YV + (int64_t)b * S->ystride;
    const double* YT = A.YT + (int64_t)b * S->ytstride;
    br_apply_targets(tt, rho, cp, YV, YT, p, cp, out + S->ooff[kc], rho, 1, sm.vst);
  }
  if (A.dbg && blockIdx.x == 0 && tid == 0) A.dbg[9] += clock64() - co0;
  const long long cz0 = clock64();
  const int kn = kc + 1;  // core index of core k+1
  const int64_t m1 = (int64_t)S->n[kn] * S->Rp[k + 1];
  const int c1 = S->R[k];
  double* dst = (k + 1 == d) ? out + S->ooff[kn] : A.Z + (int64_t)b * 2 * S->zstride + ((k + 1) & 1) * S->zstride;
  const double* V = A.V + (int64_t)b * S->vstride + S->voff[kn];
  const double* Tq = A.T + (int64_t)b * S->tstride + S->toff[kn];
  br_apply_targets(tt + BR_C * BR_C, rho, cp, V, Tq, m1, c1, dst, 1, m1, sm.vst);
  if (A.dbg && blockIdx.x == 0 && tid == 0) A.dbg[10] += clock64() - cz0;
}


// ================================================================ compact-WY engine (batch_wy.cuh)
// The same three phases as above with the blocked, tensor-core QR and applications.

// r2l chunk of panel kc (core k = kc + 1 < d), mode indices [i0, i0 + ni): rows (i - i0) Rpk + b',
// column off_{k-1,l} + a:  sum_beta L_{k+1}[b'][off_{k,l} + beta] X_k^(l)[a, i, beta] as DMMA tiles
// (M = b', N = a, K = beta), L read from the item's L slot (row-major ld 64, L2-resident).
// Loader of the right-to-left panel of core k = kc + 1 (wy::factor_panel): stack q holds mode
// indices [q ni, q ni + nq), rows (i - i0) Rpk + b'; column off_{k-1,l} + a of term l is
//   A[(i, b'), col] = sum_beta L_{k+1}[b'][off_{k,l} + beta] X_k^(l)[a, i, beta]   (k < d)
//   A[i, col]      = c_l X_d^(l)[a, i, 0]                                         (k = d)
// (the TT-sum's block-diagonal cores read in place).  A warp fills its own 8 columns: as DMMA tiles
// (M = b', N = a, K = beta; L from the item's L slot, row-major ld 64, L2-resident) when they belong
// to one term, else element by element.
// CTAs per SM of the panel kernels (shared memory: packed R block + PW staging buffers)
#ifndef WY_PANEL_CTAS
#define WY_PANEL_CTAS 4
#endif

struct R2LLoader {
  const BRShape* S;
  const double* const* cores;
  const double* L;
  const double* coef;
  int kc, n, Rpk, c, ni, last, K, d;
  __device__ int stacks() const { return (n + ni - 1) / ni; }
  __device__ int crow(int q) const { return min(ni, n - q * ni) * Rpk; }
  __device__ int term(int col) const {
    int l = 0;
    while (l + 1 < K && col >= S->off[kc][l + 1]) ++l;
    return l;
  }
  // L2 prefetch of the term-core rows cell (q, jb) will read (issued a cell ahead, before the
  // previous cell's factorisation)
  __device__ void prefetch(int q, int jb) const {
    if (last) return;
    const int lane = threadIdx.x & 31, r8 = lane & 7;
    const int i0 = q * ni, nq = min(ni, n - i0);
    const int c0 = wy::NB * jb;
    const int l0 = term(c0);
    const int ra = S->r[l0][kc], rb = S->r[l0][kc + 1], a0 = c0 - S->off[kc][l0];
    if (a0 + r8 >= ra) return;
    for (int ii = lane >> 3; ii < nq; ii += 4) {
      const char* p = reinterpret_cast<const char*>(cores[l0 * d + kc] + ((int64_t)(a0 + r8) * n + i0 + ii) * rb);
      for (int off = 0; off < rb * 8; off += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + off));
    }
  }
  __device__ void load(double* __restrict__ buf, int q, int jb) const {
    const int lane = threadIdx.x & 31, q4 = lane & 3, r8 = lane >> 2;
    const int i0 = q * ni, nq = min(ni, n - i0);
    const int c0 = wy::NB * jb, c1 = min(c0 + wy::NB, c);
    wy::zero_buf(buf);
    if (last) {
      for (int idx = lane; idx < nq * wy::NB; idx += 32) {
        const int ii = idx / wy::NB, col = c0 + idx % wy::NB;
        if (col < c1) {
          const int l = term(col), a = col - S->off[kc][l];
          buf[(col - c0) * wy::VLD + ii] = coef[l] * __ldg(cores[l * d + kc] + (int64_t)a * n + i0 + ii);
        }
      }
      __syncwarp();
      return;
    }
    const int l0 = term(c0), l1 = term(c1 - 1);
    if (l0 == l1) {  // one term: D (b' x 8) = L[:, ob + beta] X[a0 + (0..7)][i][beta]^T
      const int ra = S->r[l0][kc], rb = S->r[l0][kc + 1], ob = S->off[kc + 1][l0];
      const int a0 = c0 - S->off[kc][l0];
      const double* X = cores[l0 * d + kc];
      const int mtiles = (Rpk + 7) >> 3;
      const bool bok = a0 + r8 < ra && c0 + r8 < c1;
      if (rb <= 16) {
        // one 16-wide beta slab: the L fragments of a tile group serve every mode index of the
        // stack -- loaded once per group, then one short X load per mode index
#pragma unroll 1
        for (int mg = 0; mg < mtiles; mg += 4) {
          double af[4][4];
#pragma unroll
          for (int s4 = 0; s4 < 4; ++s4) {
            const int beta = 4 * s4 + q4;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int bp = 8 * (mg + t) + r8;
              af[t][s4] = (beta < rb && bp < Rpk) ? __ldg(L + (int64_t)bp * BR_C + ob + beta) : 0.0;
            }
          }
#pragma unroll 2
          for (int ii = 0; ii < nq; ++ii) {
            const double* xr = X + ((int64_t)(a0 + r8) * n + i0 + ii) * rb;
            double bf[4];
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4) {
              const int beta = 4 * s4 + q4;
              bf[s4] = (bok && beta < rb) ? __ldg(xr + beta) : 0.0;
            }
            double acc[4][2];
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = 0.0;
#pragma unroll
            for (int s4 = 0; s4 < 4; ++s4)
#pragma unroll
              for (int t = 0; t < 4; ++t) wy::dmma(acc[t][0], acc[t][1], af[t][s4], bf[s4]);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int bp = 8 * (mg + t) + r8;
              if (bp < Rpk) {
                const int ca = 2 * q4;
                double* dst = buf + ca * wy::VLD + ii * Rpk + bp;
                if (c0 + ca < c1 && a0 + ca < ra) dst[0] = acc[t][0];
                if (c0 + ca + 1 < c1 && a0 + ca + 1 < ra) dst[wy::VLD] = acc[t][1];
              }
            }
          }
        }
      } else {
#pragma unroll 1
        for (int ii = 0; ii < nq; ++ii) {
          const double* xr = X + ((int64_t)(a0 + r8) * n + i0 + ii) * rb;
  #pragma unroll 1
          for (int mg = 0; mg < mtiles; mg += 4) {
            double acc[4][2];
  #pragma unroll
            for (int t = 0; t < 4; ++t) acc[t][0] = acc[t][1] = 0.0;
  #pragma unroll 1
            for (int be = 0; be < rb; be += 16) {
              double af[4][4], bf[4];
  #pragma unroll
              for (int s4 = 0; s4 < 4; ++s4) {
                const int beta = be + 4 * s4 + q4;
                const bool kok = beta < rb;
                bf[s4] = (bok && kok) ? __ldg(xr + beta) : 0.0;
  #pragma unroll
                for (int t = 0; t < 4; ++t) {
                  const int bp = 8 * (mg + t) + r8;
                  af[t][s4] = (kok && bp < Rpk) ? __ldg(L + (int64_t)bp * BR_C + ob + beta) : 0.0;
                }
              }
  #pragma unroll
              for (int s4 = 0; s4 < 4; ++s4)
  #pragma unroll
                for (int t = 0; t < 4; ++t) wy::dmma(acc[t][0], acc[t][1], af[t][s4], bf[s4]);
            }
  #pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int bp = 8 * (mg + t) + r8;
              if (bp < Rpk) {
                const int ca = 2 * q4;
                double* dst = buf + ca * wy::VLD + ii * Rpk + bp;
                if (c0 + ca < c1 && a0 + ca < ra) dst[0] = acc[t][0];
                if (c0 + ca + 1 < c1 && a0 + ca + 1 < ra) dst[wy::VLD] = acc[t][1];
              }
            }
          }
        }
      }
    } else {  // columns of several terms: element by element, lane = row
      const int rows = nq * Rpk;
#pragma unroll 1
      for (int col = c0; col < c1; ++col) {
        const int l = term(col), a = col - S->off[kc][l];
        const int rb = S->r[l][kc + 1], ob = S->off[kc + 1][l];
        const double* X = cores[l * d + kc];
        for (int r = lane; r < rows; r += 32) {
          const int ii = r / Rpk, bp = r % Rpk;
          const double* xp = X + ((int64_t)a * n + i0 + ii) * rb;
          const double* lp = L + (int64_t)bp * BR_C + ob;
          double acc = 0.0;
          for (int be = 0; be < rb; ++be) acc += __ldg(lp + be) * __ldg(xp + be);
          buf[(col - c0) * wy::VLD + r] = acc;
        }
      }
    }
    __syncwarp();
  }
};

__global__ void __launch_bounds__(wy::PT, WY_PANEL_CTAS) br_r2l_wy_kernel(BRArgs A, int kc) {
  extern __shared__ __align__(16) unsigned char br_smem_raw[];
  wy::Smem& sm = *reinterpret_cast<wy::Smem*>(br_smem_raw);
  const BRShape* S = A.sh;
  const int b = blockIdx.x + A.b0, gb = A.item0 + b;
  const int d = S->d, K = S->K;
  const int k = kc + 1;                 // 1-based core index, 2..d
  const int n = S->n[kc], Rpk = S->Rp[k], c = S->R[k - 1];
  const int64_t m = (int64_t)n * Rpk;
  const int tid = threadIdx.x;
  R2LLoader ld{S, A.cores + (int64_t)gb * K * d, A.L + (int64_t)b * 2 * BR_C * BR_C + ((k + 1) & 1) * BR_C * BR_C,
               A.coef + (int64_t)gb * K, kc, n, Rpk, c, S->wyni[kc], k == d ? 1 : 0, K, d};
  double* Lout = A.L + (int64_t)b * 2 * BR_C * BR_C + (k & 1) * BR_C * BR_C;
  const int rows = S->Rp[k - 1];
  if (m < c) {
    // fewer rows than columns (one stack): A_k = I_m A_k -- the identity is a valid orthogonal Q and
    // R = A_k exactly (an augmented factorisation with m reflectors for c > m columns would lose
    // the columns whose leading block is rank deficient)
    const int w = tid >> 5, lane = tid & 31;
    for (int idx = tid; idx < BR_C * BR_C; idx += wy::PT) Lout[idx] = 0.0;
    __syncthreads();
    for (int jb = w; 8 * jb < c; jb += wy::PW) {  // block by block through the warp's staging buffer
      ld.load(sm.Vb[w], 0, jb);
      for (int idx = lane; idx < 8 * rows; idx += 32) {
        const int cc = idx / rows, row = idx % rows, col = 8 * jb + cc;
        if (col < c) Lout[row * BR_C + col] = sm.Vb[w][cc * wy::VLD + row];
      }
      __syncwarp();
    }
    return;
  }
  wy::factor_panel(sm, ld, c, A.V + (int64_t)b * S->vstride + S->voff[kc],
                   (A.dbg && blockIdx.x == 0) ? A.dbg + 32 : nullptr);
  // R (R'_{k-1} x c, row-major ld 64) -> L slot (k & 1)
  for (int idx = tid; idx < BR_C * BR_C; idx += wy::PT) {
    const int row = idx / BR_C, col = idx % BR_C;
    Lout[idx] = (row < rows && col < c && row <= col) ? sm.st[wy::ridx(row, col)] : 0.0;
  }
}

// Loader of a tall left-to-right Y_k (p rows, cp columns) in stacks of 128 rows.
struct YLoader {
  const BRShape* S;
  const double* Z;       // k > 1: Y_k row-major ld cp
  const double* L2;      // k = 1: L_2 (row-major ld 64)
  const double* const* cores;
  int k, p, cp, K, d;
  __device__ int stacks() const { return (p + wy::CH - 1) / wy::CH; }
  __device__ int crow(int q) const { return min(wy::CH, p - q * wy::CH); }
  __device__ double el(int64_t row, int col) const {
    if (k > 1) return Z[row * cp + col];
    double s = 0.0;  // Y_1[i, b'] = sum_l sum_beta X_1^(l)[0, i, beta] L_2[b'][off_{1,l} + beta]
    const double* Lr = L2 + (int64_t)col * BR_C;
    for (int l = 0; l < K; ++l) {
      const int rl = S->r[l][1], o = S->off[1][l];
      const double* xp = cores[l * d] + row * rl;
      for (int be = 0; be < rl; ++be) s += Lr[o + be] * __ldg(xp + be);
    }
    return s;
  }
  __device__ void prefetch(int q, int jb) const {
    if (k == 1) return;
    const int lane = threadIdx.x & 31;
    const int rows = crow(q);
    for (int r = lane; r < rows; r += 32)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(Z + ((int64_t)q * wy::CH + r) * cp + wy::NB * jb));
  }
  __device__ void load(double* __restrict__ buf, int q, int jb) const {
    const int lane = threadIdx.x & 31;
    const int rows = crow(q), c0 = wy::NB * jb, c1 = min(c0 + wy::NB, cp);
    wy::zero_buf(buf);
    for (int r = lane; r < rows; r += 32)
      for (int col = c0; col < c1; ++col) buf[(col - c0) * wy::VLD + r] = el((int64_t)q * wy::CH + r, col);
    __syncwarp();
  }
};

// Left-to-right QR of a tall Y_k (p > 64 rows, cp columns) with the WY engine; R -> JM.
__global__ void __launch_bounds__(wy::PT, WY_PANEL_CTAS) br_l2r_qr_wy_kernel(BRArgs A, int k) {
  extern __shared__ __align__(16) unsigned char br_smem_raw[];
  wy::Smem& sm = *reinterpret_cast<wy::Smem*>(br_smem_raw);
  const BRShape* S = A.sh;
  const int b = blockIdx.x + A.b0, gb = A.item0 + b;
  const int d = S->d, K = S->K;
  const int kc = k - 1;
  const int tid = threadIdx.x;
  int* rk = A.ranks + (int64_t)b * (d + 1);
  double* sc = A.scal + (int64_t)b * 4;
  double* out = A.out + (int64_t)b * S->ostride;
  const int n = S->n[kc], cp = S->Rp[k];
  if (k > 1 && sc[3] != 0.0) {  // ||x|| = 0: rank-1 zero tensor
    for (int i = tid; i < n; i += wy::PT) out[S->ooff[kc] + i] = 0.0;
    if (k + 1 == d)
      for (int i = tid; i < S->n[d - 1]; i += wy::PT) out[S->ooff[d - 1] + i] = 0.0;
    if (tid == 0) { rk[k] = 1; if (k + 1 == d) rk[d] = 1; }
    return;
  }
  const int64_t p = (k == 1) ? (int64_t)n : (int64_t)rk[k - 1] * n;
  const bool tall = p > BR_C;
  const double* Lin = A.L;  // k == 1: L_2 in slot 0
  const double* Z = A.Z + (int64_t)b * 2 * S->zstride + (k & 1) * S->zstride;
  const double* const* cores = A.cores + (int64_t)gb * K * d;
  YLoader ld{S, Z, Lin + (int64_t)b * 2 * BR_C * BR_C, cores, k, (int)p, cp, K, d};
  // the 64 x 64 matrix handed to the SVD (column-major ld 64), in the staging area: R of the tall
  // Y_k unpacked, or a short Y_k itself
  double* dense = &sm.Vb[0][0];
  static_assert(sizeof(sm.Vb) >= sizeof(double) * BR_C * BR_C, "staging area holds the dense block");
  if (tall) {
    wy::factor_panel(sm, ld, cp, A.YV + (int64_t)b * S->ystride);
    for (int idx = tid; idx < BR_C * BR_C; idx += wy::PT) {
      const int col = idx / BR_C, row = idx % BR_C;
      dense[idx] = row <= col ? sm.st[wy::ridx(row, col)] : 0.0;
    }
  } else {
    for (int idx = tid; idx < BR_C * BR_C; idx += wy::PT) dense[idx] = 0.0;
    __syncthreads();
    for (int idx = tid; idx < p * cp; idx += wy::PT) {
      const int r = idx / cp, col = idx % cp;
      dense[col * BR_C + r] = ld.el(r, col);  // short Y_k: the Jacobi input is Y itself
    }
  }
  __syncthreads();
  if (k == 1) {
    double q = 0.0;
    for (int idx = tid; idx < BR_C * BR_C; idx += wy::PT) {
      const double v = dense[idx];
      q += v * v;
    }
    const double nrm = sqrt(block_sum(q, sm.red));
    if (tid == 0) {
      const double s = A.scale[gb];
      double tau = 0.0;
      if (!A.keep_all) tau = fmax(A.rel_tol * nrm / sqrt((double)(d - 1)), A.floor_c * U_ROUND * s);
      sc[0] = nrm;
      sc[1] = tau;
      sc[2] = s;
      sc[3] = nrm == 0.0 ? 1.0 : 0.0;
      rk[0] = 1;
      rk[d] = 1;
    }
    if (nrm == 0.0) {
      for (int i = tid; i < n; i += wy::PT) out[S->ooff[0] + i] = 0.0;
      if (d == 2)
        for (int i = tid; i < S->n[1]; i += wy::PT) out[S->ooff[1] + i] = 0.0;
      if (tid == 0) { rk[1] = 1; rk[d] = 1; }
      return;
    }
  }
  double* jm = A.JM + (int64_t)b * BR_C * BR_C;  // column-major ld 64, zero outside
  for (int idx = tid; idx < BR_C * BR_C; idx += wy::PT) {
    const int col = idx / BR_C, row = idx % BR_C;
    jm[idx] = (col < cp && row <= (tall ? col : BR_C)) ? dense[col * BR_C + row] : 0.0;
  }
}

__global__ void __launch_bounds__(wy::T, 3) br_l2r_apply_wy_kernel(BRArgs A, int k) {
  extern __shared__ __align__(16) unsigned char br_smem_raw[];
  wy::ASmem& sm = *reinterpret_cast<wy::ASmem*>(br_smem_raw);
  const BRShape* S = A.sh;
  const int b = blockIdx.x + A.b0;
  const int d = S->d;
  const int kc = k - 1;
  const int* rk = A.ranks + (int64_t)b * (d + 1);
  const double* sc = A.scal + (int64_t)b * 4;
  if (sc[3] != 0.0) return;
  wy::apply_init(sm);
  uint32_t ph[wy::NBUF] = {};
  double* out = A.out + (int64_t)b * S->ostride;
  const int n = S->n[kc], cp = S->Rp[k];
  const int64_t p = (k == 1) ? (int64_t)n : (int64_t)rk[k - 1] * n;
  const bool tall = p > BR_C;
  const int rho = rk[k];
  const double* tt = A.TT + (int64_t)b * 2 * BR_C * BR_C;
  if (tall && A.gemm[b]) {
    br_gemm_yw(A.Z + (int64_t)b * 2 * S->zstride + (k & 1) * S->zstride, (int)p, cp, tt, rho, out + S->ooff[kc]);
    __syncthreads();
  } else if (tall) {  // output core k = Q_Y [U_rho; 0]  ((rho_{k-1} n_k) x rho, row-major)
    wy::apply(sm, ph, tt, cp, rho, A.YV + (int64_t)b * S->ystride, p, wy::CH, cp, cp, out + S->ooff[kc], rho, 1);
  }
  // Z_{k+1} = Q_{k+1} [(S V^T)^T; 0] (panel rows (i, b') of core k+1 -> core layout (a, i, b'))
  const int kn = kc + 1;
  const int64_t m1 = (int64_t)S->n[kn] * S->Rp[k + 1];
  const int c1 = S->R[k];
  double* dst = (k + 1 == d) ? out + S->ooff[kn] : A.Z + (int64_t)b * 2 * S->zstride + ((k + 1) & 1) * S->zstride;
  const double* V = A.V + (int64_t)b * S->vstride + S->voff[kn];
  const int cr = S->wyni[kn] * S->Rp[k + 1];
  if (m1 < c1) {  // Q_{k+1} = I (br_r2l_wy_kernel): the panel rows are the target rows (cp = m1)
    const double* src = tt + BR_C * BR_C;
    for (int idx = threadIdx.x; idx < rho * m1; idx += wy::T) {
      const int col = idx / (int)m1, row = idx % (int)m1;
      dst[row + (int64_t)col * m1] = src[col * BR_C + row];
    }
    return;
  }
  wy::apply(sm, ph, tt + BR_C * BR_C, cp, rho, V, m1, cr, c1, c1, dst, 1, m1,
            (A.dbg && blockIdx.x == 0) ? A.dbg + 72 : nullptr);
}

// Copy item b's cores from the worst-case workspace to the exact-size arena.
__global__ void br_compact_kernel(const double* __restrict__ work, int64_t ostride, const int64_t* __restrict__ ooff,
                                  const int64_t* __restrict__ dst_off, const int64_t* __restrict__ sizes, int d,
                                  double* arena) {
  const int b = blockIdx.x;
  for (int kc = 0; kc < d; ++kc) {
    const double* src = work + (int64_t)b * ostride + ooff[kc];
    double* dst = arena + dst_off[(int64_t)b * d + kc];
    const int64_t sz = sizes[(int64_t)b * d + kc];
    for (int64_t i = threadIdx.x; i < sz; i += blockDim.x) dst[i] = src[i];
  }
}

}  // namespace

bool batch_uniform_supported(int B, const std::vector<SumInput>& items, std::string* why) {
  auto no = [&](const char* w) { if (why) *why = w; return false; };
  if (B < 1) return no("empty batch");
  const SumInput& f = items[0];
  for (const SumInput& it : items)
    if (it.d != f.d || it.K() != f.K() || it.n != f.n || it.r != f.r) return no("items differ in shape");
  return batch_shape_supported(f.d, f.K(), f.r, why);
}

bool batch_shape_supported(int d, int K, const std::vector<std::vector<int64_t>>& r, std::string* why) {
  auto no = [&](const char* w) { if (why) *why = w; return false; };
  if (d < 2) return no("d < 2");
  if (d > BR_MAXD) return no("d > 64");
  if (K < 1 || K > BR_MAXK) return no("K outside 1..16");
  for (int k = 1; k < d; ++k) {
    int64_t R = 0;
    for (int l = 0; l < K; ++l) R += r[(size_t)l][(size_t)k];
    if (R > BR_C) return no("formal rank > 64");
  }
  return true;
}

void batch_desc_shape(BatchDesc& in, int B, int K, int d, const int64_t* n, const int64_t* r) {
  if (B < 0 || K < 1 || d < 1 || !n || !r) fail(TT_EINVAL, "batch: bad shape arguments");
  in.B = B;
  in.K = K;
  in.d = d;
  in.n.assign(n, n + d);
  in.r.resize((size_t)K);
  for (int l = 0; l < K; ++l) {
    in.r[(size_t)l].assign(r + (size_t)l * (d + 1), r + (size_t)(l + 1) * (d + 1));
    if (in.r[(size_t)l][0] != 1 || in.r[(size_t)l][(size_t)d] != 1) fail(TT_ESHAPE, "boundary ranks must be 1");
    for (int k = 0; k < d; ++k)
      if (n[k] < 1 || in.r[(size_t)l][(size_t)k] < 1) fail(TT_ESHAPE, "mode sizes and ranks must be >= 1");
  }
  std::string why;
  if (!batch_shape_supported(d, K, in.r, &why)) fail(TT_ENOTSUP, "batched engine: " + why);
}

void run_batch(tt_ctx ctx, const BatchDesc& in, const tt_round_opts& o, BatchOut& res) {
  TTB_RANGE("tt_round_batch");
  const char* hdbg = std::getenv("TT_B200_BR_DEBUG");
  const bool hd = hdbg && hdbg[0] == '1';
  const auto t_start = std::chrono::steady_clock::now();
  auto stamp = [&](const char* what) {
    if (!hd) return;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
    std::fprintf(stderr, "[br_host] %8.2f ms  %s\n", ms, what);
  };
  const int B = in.B, d = in.d, K = in.K;
  // ---------------------------------------------------------------- shape tables (uniform)
  BRShape sh;
  std::memset(&sh, 0, sizeof(sh));
  sh.d = d;
  sh.K = K;
  for (int k = 0; k < d; ++k) sh.n[k] = (int)in.n[(size_t)k];
  for (int k = 0; k <= d; ++k) {
    int s = 0;
    for (int l = 0; l < K; ++l) {
      sh.r[l][k] = (int)in.r[(size_t)l][(size_t)k];
      sh.off[k][l] = s;
      s += sh.r[l][k];
    }
    sh.R[k] = s;
  }
  sh.R[0] = 1;
  sh.R[d] = 1;
  sh.Rp[d] = 1;
  for (int k = d; k >= 2; --k) sh.Rp[k - 1] = (int)std::min<int64_t>((int64_t)sh.n[k - 1] * sh.Rp[k], sh.R[k - 1]);
  sh.Rp[0] = 1;
  int64_t v = 0, t = 0, omax = 0, yv = 0, zmax = 0;
  for (int kc = 1; kc < d; ++kc) {  // panels of cores 2..d
    const int64_t m = (int64_t)sh.n[kc] * sh.Rp[kc + 1];
    const int c = sh.R[kc];
    sh.voff[kc] = v;
    sh.toff[kc] = t;
    v += br_vsize(m, c);
    t += (int64_t)br_stacks(m) * BR_C;
  }
  for (int kc = 0; kc < d; ++kc) {
    sh.ooff[kc] = omax;
    omax += (int64_t)sh.Rp[kc] * sh.n[kc] * sh.Rp[kc + 1];
  }
  int64_t yt = 0;
  for (int k = 1; k < d; ++k) {  // left-to-right QR of Y_k, p <= Rp_{k-1} n_k
    const int64_t p = (int64_t)sh.Rp[k - 1] * sh.n[k - 1];
    if (p > BR_C) {
      yv = std::max<int64_t>(yv, br_vsize(p, sh.Rp[k]));
      yt = std::max<int64_t>(yt, (int64_t)br_stacks(p) * BR_C);
    }
    if (k + 1 < d) zmax = std::max<int64_t>(zmax, (int64_t)sh.n[k] * sh.Rp[k + 1] * sh.Rp[k]);
  }
  static const bool use_wy = [] {
    const char* e = std::getenv("TT_B200_BR_WY");
    return !(e && e[0] == '0');
  }();
  if (use_wy) {  // compact-WY engine: stacks of whole mode indices (<= 128 rows), V + T per stack
    v = 0;
    yv = 0;
    for (int kc = 1; kc < d; ++kc) {
      const int Rpk = sh.Rp[kc + 1];
      const int ni = std::max(1, std::min(sh.n[kc], wy::CH / Rpk));
      sh.wyni[kc] = ni;
      sh.voff[kc] = v;
      v += (int64_t)((sh.n[kc] + ni - 1) / ni) * wy::stack_doubles(sh.R[kc]);
    }
    for (int k = 1; k < d; ++k) {
      const int64_t p = (int64_t)sh.Rp[k - 1] * sh.n[k - 1];
      if (p > BR_C) yv = std::max<int64_t>(yv, ((p + wy::CH - 1) / wy::CH) * wy::stack_doubles(sh.Rp[k]));
    }
    t = 2;
    yt = 2;
  }
  sh.vstride = (std::max<int64_t>(v, 2) + 1) & ~(int64_t)1;
  sh.tstride = (std::max<int64_t>(t, 2) + 1) & ~(int64_t)1;
  sh.ystride = (std::max<int64_t>(yv, 2) + 1) & ~(int64_t)1;
  sh.ytstride = (std::max<int64_t>(yt, 2) + 1) & ~(int64_t)1;
  sh.zstride = (std::max<int64_t>(zmax, 2) + 1) & ~(int64_t)1;
  sh.ostride = omax;
  const int64_t per_item = sh.vstride + sh.tstride + 6 * BR_C * BR_C + BR_C + sh.ystride + sh.ytstride + 2 * sh.zstride +
                           sh.ostride + 8;
  // ---------------------------------------------------------------- s(x) per item
  const bool keep_all = (o.rel_tol == 0.0);
  std::vector<double> scale((size_t)B, 0.0);
  {
    std::vector<int64_t> need;  // b * K + l with unknown ||y_l||
    for (int64_t q = 0; q < (int64_t)B * K; ++q)
      if (!(in.norm[(size_t)q] == in.norm[(size_t)q])) need.push_back(q);
    std::vector<double> nn(need.size(), 0.0);
    if (!need.empty() && !keep_all && o.floor_c > 0.0) {
      DotBatch db;
      db.d = d;
      db.n = in.n;
      db.P = (int)need.size();
      for (int64_t q : need) {
        const int l = (int)(q % K);
        for (int k = 0; k < d; ++k) {
          db.xc.push_back(in.tab[(size_t)q * d + k]);
          db.yc.push_back(in.tab[(size_t)q * d + k]);
        }
        for (int k = 0; k <= d; ++k) {
          db.xr.push_back(in.r[(size_t)l][(size_t)k]);
          db.yr.push_back(in.r[(size_t)l][(size_t)k]);
        }
      }
      DBuf dd(ctx, need.size());
      dot_batch(ctx, db, dd.p, nullptr);
      d2h_small(ctx, nn.data(), dd.p, nn.size());
      for (double& x : nn) x = std::sqrt(std::max(x, 0.0));
    }
    size_t q2 = 0;
    for (int64_t q = 0; q < (int64_t)B * K; ++q) {
      double nl = in.norm[(size_t)q];
      if (!(nl == nl)) nl = nn[q2++];
      scale[(size_t)(q / K)] += std::fabs(in.coef[(size_t)q]) * nl;
    }
  }
  // ---------------------------------------------------------------- device tables
  BBuf dsh, dtab, dcoef, dscale;
  dsh.upload(ctx, &sh, sizeof(sh), true);
  dtab.upload(ctx, in.tab.data(), in.tab.size() * sizeof(double*), true);
  dcoef.upload(ctx, in.coef.data(), in.coef.size() * sizeof(double), true);
  dscale.upload(ctx, scale.data(), scale.size() * sizeof(double), true);
  // ---------------------------------------------------------------- waves
  stamp("tables uploaded");
  auto ws_for = [&](int nbm) {
    return (size_t)nbm * ((size_t)sh.vstride + sh.tstride + 6 * BR_C * BR_C + BR_C + sh.ystride + sh.ytstride +
                          2 * sh.zstride + std::max<int64_t>(sh.ostride, 1) + 4) +
           (size_t)nbm * (d + 3) + 64;
  };
  // one wave when the whole batch fits in ~60 % of the device (the workspace is the context's
  // grow-only scratch: no allocation churn between calls).  A batch the scratch already holds
  // skips the free-memory query (cudaMemGetInfo costs 0.2-2 ms: the serial drivers' one-item
  // batches would pay it on every rounding).
  size_t free_b = 0, total_b = 0;
  int W = B;
  if (ws_for(B) * sizeof(double) > ctx->scratch_bytes) {
    TTB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const double budget = std::min<double>(0.6 * ((double)free_b + (double)ctx->scratch_bytes), 100e9);
    W = (int)std::max<int64_t>(1, std::min<int64_t>(B, (int64_t)(budget / (8.0 * (double)per_item))));
  }
  const int nb_max = std::min(W, B);
  const size_t ws_doubles = ws_for(nb_max);
  double* ws = static_cast<double*>(ctx_scratch(ctx, ws_doubles * sizeof(double)));
  // kernels that do not stage reflector slices leave out the VStage buffers
  const size_t smem = offsetof(BRSmem, vst), smem_q = offsetof(BRSmem, vst), smem_a = sizeof(BRSmemA);
  const size_t smem_wy = sizeof(wy::Smem), smem_wya = sizeof(wy::ASmem);
  static uint64_t attr_set = 0;  // devices whose kernel attributes are set (once per process)
  if (!(attr_set >> (ctx->device & 63) & 1)) {
    attr_set |= (uint64_t)1 << (ctx->device & 63);
    TTB_CUDA(cudaFuncSetAttribute(br_r2l_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    TTB_CUDA(cudaFuncSetAttribute(br_l2r_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_q));
    TTB_CUDA(cudaFuncSetAttribute(br_l2r_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_q));
    TTB_CUDA(cudaFuncSetAttribute(br_l2r_apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a));
    TTB_CUDA(cudaFuncSetAttribute(br_r2l_wy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_wy));
    TTB_CUDA(cudaFuncSetAttribute(br_l2r_qr_wy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_wy));
    TTB_CUDA(cudaFuncSetAttribute(br_l2r_apply_wy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_wya));
  }
  res.B = B;
  res.d = d;
  res.n = in.n;
  res.ranks.assign((size_t)B * (d + 1), 1);
  res.norm.assign((size_t)B, 0.0);
  res.tau.assign((size_t)B, 0.0);
  res.scale.assign((size_t)B, 0.0);
  res.core.assign((size_t)B * d, nullptr);
  res.wave_first.clear();
  res.arenas.clear();
  res.arena_size.clear();
  try {
    if (hd) std::fprintf(stderr, "[br_host] W = %d of B = %d, per item %.1f MB, free %.1f GB\n", W, B, 8e-6 * per_item, 1e-9 * free_b);
    for (int w0 = 0; w0 < B; w0 += W) {
      const int nb = std::min(W, B - w0);
      stamp("wave start");
      struct { double* p; } V, T, L, YV, YT, Z, O, SC, JM, TT, QX;
      struct { int* p; } RK, INF, GM;
      {
        double* w = ws;  // carve the scratch (every piece a multiple of 2 doubles: 16-B aligned)
        auto take = [&](size_t n) { double* r = w; w += (n + 1) & ~(size_t)1; return r; };
        V.p = take((size_t)nb * sh.vstride);
        T.p = take((size_t)nb * sh.tstride);
        L.p = take((size_t)nb * 2 * BR_C * BR_C);
        YV.p = take((size_t)nb * sh.ystride);
        YT.p = take((size_t)nb * sh.ytstride);
        Z.p = take((size_t)nb * 2 * sh.zstride);
        O.p = take((size_t)nb * std::max<int64_t>(sh.ostride, 1));
        JM.p = take((size_t)nb * BR_C * BR_C);
        TT.p = take((size_t)nb * 2 * BR_C * BR_C);
        QX.p = take((size_t)nb * (BR_C * BR_C + BR_C));
        SC.p = take((size_t)nb * 4);
        RK.p = reinterpret_cast<int*>(take(((size_t)nb * (d + 1) + 1) / 2));
        INF.p = reinterpret_cast<int*>(take(((size_t)nb + 1) / 2));
        GM.p = reinterpret_cast<int*>(take(((size_t)nb + 1) / 2));
      }
      TTB_CUDA(cudaMemsetAsync(INF.p, 0, sizeof(int) * nb, ctx->stream));
      BRArgs a;
      a.sh = static_cast<const BRShape*>(dsh.p);
      a.cores = static_cast<const double* const*>(dtab.p);
      a.coef = static_cast<const double*>(dcoef.p);
      a.scale = static_cast<const double*>(dscale.p);
      a.V = V.p; a.T = T.p; a.L = L.p; a.YV = YV.p; a.YT = YT.p; a.Z = Z.p; a.out = O.p; a.JM = JM.p; a.TT = TT.p; a.QX = QX.p;
      a.ranks = RK.p; a.scal = SC.p; a.info = INF.p; a.gemm = GM.p;
      a.rel_tol = o.rel_tol;
      a.floor_c = o.floor_c;
      a.max_rank = o.max_rank;
      a.keep_all = keep_all ? 1 : 0;
      {
        static const char* jt = std::getenv("TT_B200_BR_JACT");
        a.jac_t = (jt && jt[0] == '0') ? 0 : 1;
        static const char* qs = std::getenv("TT_B200_BR_QRCP");
        a.qrcp_svd = (qs && qs[0] == '0') ? 0 : 1;
        static const char* jl = std::getenv("TT_B200_BR_JLPP");
        const int jlv = jl ? std::atoi(jl) : 0;
        a.jac_lpp = (jlv == 8 || jlv == 16 || jlv == 32) ? jlv : 0;
      }
      a.item0 = w0;
      const char* dbe = std::getenv("TT_B200_BR_DEBUG");
      LBuf dbg;
      if (dbe && dbe[0] == '1') {
        dbg.alloc(ctx, 96);
        TTB_CUDA(cudaMemsetAsync(dbg.p, 0, 96 * sizeof(long long), ctx->stream));
      }
      a.dbg = dbg.p;
      a.b0 = 0;
      // the whole sweep of one range of the wave's items on one stream
      auto run_seq = [&](const BRArgs& ah, int nh, cudaStream_t st) {
      nvtxRangePushA("tt_round_batch: right-to-left orthogonalisation");
      for (int kc = d - 1; kc >= 1; --kc) {
          const int64_t m = (int64_t)sh.n[kc] * sh.Rp[kc + 1];
          const double c = sh.R[kc];
          double rl = 0.0;  // panel assembly: 2 r_k^(l) flops per element of term l's columns
          for (int l = 0; l < K; ++l) rl += (double)sh.r[l][kc] * sh.r[l][kc + 1];
          const double mm = (double)m;
          const double fl = nh * (2.0 * mm * rl + (mm >= c ? 2.0 * mm * c * c - 2.0 * c * c * c / 3.0
                                                           : 2.0 * c * mm * mm - 2.0 * mm * mm * mm / 3.0));
          if (use_wy)
            TTB_RUN(ctx, "batch_r2l_qr", fl, 8.0 * nh * (mm * c) * 2.0,
                    br_r2l_wy_kernel<<<nh, wy::PT, smem_wy, st>>>(ah, kc));
          else
            TTB_RUN(ctx, "batch_r2l_qr", fl, 8.0 * nh * (mm * c) * 2.0,
                    br_r2l_kernel<<<nh, BR_T, smem, st>>>(ah, kc));
          static const char* dump = std::getenv("TT_B200_BR_DUMP");  // debugging: item 0's R factors
          if (dump && w0 == 0) {
            std::vector<double> h(BR_C * BR_C);
            TTB_CUDA(cudaMemcpyAsync(h.data(), L.p + ((kc + 1) & 1) * BR_C * BR_C, sizeof(double) * h.size(),
                                     cudaMemcpyDeviceToHost, ctx->stream));
            TTB_CUDA(cudaStreamSynchronize(ctx->stream));
            FILE* f = std::fopen(dump, kc == d - 1 ? "wb" : "ab");
            if (f) { std::fwrite(h.data(), sizeof(double), h.size(), f); std::fclose(f); }
          }
        }
        nvtxRangePop();
        TTB_RANGE("tt_round_batch: left-to-right truncation");
        for (int k = 1; k < d; ++k) {
          if (use_wy)
            TTB_RUN(ctx, "batch_l2r_qr", 0.0, 0.0, br_l2r_qr_wy_kernel<<<nh, wy::PT, smem_wy, st>>>(ah, k));
          else
            TTB_RUN(ctx, "batch_l2r_qr", 0.0, 0.0, br_l2r_qr_kernel<<<nh, BR_T, smem_q, st>>>(ah, k));
          TTB_RUN(ctx, "batch_l2r_svd", 0.0, 0.0, br_l2r_svd_kernel<<<nh, BR_T, smem_q, st>>>(ah, k));
          if (use_wy)
            TTB_RUN(ctx, "batch_l2r_apply", 0.0, 0.0, br_l2r_apply_wy_kernel<<<nh, wy::T, smem_wya, st>>>(ah, k));
          else
            TTB_RUN(ctx, "batch_l2r_apply", 0.0, 0.0, br_l2r_apply_kernel<<<nh, BR_T, smem_a, st>>>(ah, k));
        }
      };
      // The wave in two (TT_B200_BR_SPLIT) parts on as many streams (items are independent): when a kernel of one half drains its
      // last CTAs, the SMs it leaves take CTAs of the other half's kernel instead of idling, and
      // kernels with different bottlenecks (DMMA applications, latency-bound Jacobi) share SMs.
      // One stream when per-kernel timing (tt_ctx_profile), debugging or the dump is on.
      static const char* split_env = std::getenv("TT_B200_BR_SPLIT");  // parts (1 = off), default 2
      int parts = split_env ? std::atoi(split_env) : 2;
      parts = std::max(1, std::min(parts, 4));
      const bool split = use_wy && parts > 1 && !ctx->prof && !ctx->debug_sync && !dbg.p && nb >= 16 * ctx->num_sms &&
                         !std::getenv("TT_B200_BR_DUMP");
      if (split) {
        if (!ctx->br_fork) TTB_CUDA(cudaEventCreateWithFlags(&ctx->br_fork, cudaEventDisableTiming));
        for (int i = 0; i + 1 < parts; ++i)
          if (!ctx->br_aux[i]) {
            TTB_CUDA(cudaStreamCreateWithFlags(&ctx->br_aux[i], cudaStreamNonBlocking));
            TTB_CUDA(cudaEventCreateWithFlags(&ctx->br_join[i], cudaEventDisableTiming));
          }
        TTB_CUDA(cudaEventRecord(ctx->br_fork, ctx->stream));
        for (int i = 0; i < parts; ++i) {
          const int lo = (int)((int64_t)nb * i / parts), hi = (int)((int64_t)nb * (i + 1) / parts);
          BRArgs ai = a;
          ai.b0 = lo;
          cudaStream_t st = i == 0 ? ctx->stream : ctx->br_aux[i - 1];
          if (i > 0) TTB_CUDA(cudaStreamWaitEvent(st, ctx->br_fork, 0));
          run_seq(ai, hi - lo, st);
          if (i > 0) {
            TTB_CUDA(cudaEventRecord(ctx->br_join[i - 1], st));
          }
        }
        for (int i = 0; i + 1 < parts; ++i) TTB_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->br_join[i], 0));
      } else {
        run_seq(a, nb, ctx->stream);
      }
      if (dbg.p) {
        long long h[96];
        TTB_CUDA(cudaMemcpyAsync(h, dbg.p, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
        TTB_CUDA(cudaStreamSynchronize(ctx->stream));
        if (use_wy)
          std::fprintf(stderr, "[br_debug] l2r SVD, CTA 0 (%lld tall splits, kq sum %lld, %lld ambiguous): QRCP %.2f Mcycles, "
                       "Jacobi %.2f (%lld sweeps), Q_X applications %.2f\n", h[85], h[84], h[83], 1e-6 * h[80],
                       1e-6 * h[81], h[11], 1e-6 * h[82]);
        if (use_wy && !WY_PROF) {
          std::fprintf(stderr, "[br_debug] WY cycle counters: rebuild with TT_B200_NVCC_EXTRA=-DWY_PROF=1\n");
        } else if (use_wy) {
          std::fprintf(stderr, "[br_debug] WY r2l, CTA 0, per warp (wait / update / factor / store+release+load, Mcycles):");
          for (int w = 0; w < 8; ++w)
            std::fprintf(stderr, " w%d %.2f/%.2f/%.2f/%.2f", w, 1e-6 * h[32 + 4 * w], 1e-6 * h[33 + 4 * w],
                         1e-6 * h[34 + 4 * w], 1e-6 * h[35 + 4 * w]);
          std::fprintf(stderr, "\n[br_debug] warp 3 block factorisation (Mcycles): dots + reduction %.2f dlarfg %.2f update %.2f T + R row %.2f writeback %.2f\n",
                       1e-6 * h[64], 1e-6 * h[65], 1e-6 * h[66], 1e-6 * h[67], 1e-6 * h[68]);
          std::fprintf(stderr, "[br_debug] Z application, CTA 0 thread 0 (Mcycles): staging wait %.2f, W %.2f, barrier %.2f, "
                       "W' + update %.2f, end barrier + issue %.2f\n",
                       1e-6 * h[72], 1e-6 * h[73], 1e-6 * h[74], 1e-6 * h[75], 1e-6 * h[76]);
        } else {
        std::fprintf(stderr, "[br_debug] r2l: assemble %lld qr %lld store %lld | l2r: assemble %lld qr %lld store %lld | jacobi %lld (%lld sweeps) outcore %lld nextcore %lld (cycles, CTA 0) | qr steps: owner(w0) %lld x%lld, pre-barrier(w0 not owner) %lld, barrier %lld, update %lld\n",
                     h[0], h[1], h[2], h[4], h[5], h[6], h[8], h[11], h[9], h[10], h[16], h[19], h[20], h[17], h[18]);
        }
      }
      // ranks (the one host synchronisation of the wave), then compaction
      std::vector<int> hr((size_t)nb * (d + 1)), hinf((size_t)nb);
      stamp("launched");
      // SC, RK, INF and GM are consecutive pieces of the scratch: one read-back
      std::vector<double> hblk((size_t)((reinterpret_cast<double*>(GM.p) - SC.p) + (nb + 1) / 2));
      d2h_small(ctx, hblk.data(), SC.p, hblk.size());
      stamp("synced (ranks)");
      auto piece = [&](const void* dp) { return reinterpret_cast<const char*>(hblk.data()) + (reinterpret_cast<const char*>(dp) - reinterpret_cast<const char*>(SC.p)); };
      std::memcpy(hr.data(), piece(RK.p), sizeof(int) * hr.size());
      std::memcpy(hinf.data(), piece(INF.p), sizeof(int) * hinf.size());
      for (int b = 0; b < nb; ++b)
        if (hinf[(size_t)b]) fail(TT_ENOCONV, "Jacobi SVD did not converge (batch item " + std::to_string(w0 + b) + ")");
      std::vector<double> hsc((size_t)nb * 4);
      std::memcpy(hsc.data(), piece(SC.p), sizeof(double) * hsc.size());
      for (int b = 0; b < nb; ++b)  // value range (tt_b200.h): squared norms must be representable
        if (!std::isfinite(hsc[(size_t)b * 4])) fail(TT_EINVAL, "batch item " + std::to_string(w0 + b) + ": ||x|| is not finite (input outside the value range, see tt_b200.h)");
      std::vector<int> hgm((size_t)nb);
      std::memcpy(hgm.data(), piece(GM.p), sizeof(int) * hgm.size());
      std::vector<int64_t> dst((size_t)nb * d), sz((size_t)nb * d);
      int64_t tot = 0;
      double l2r_svd_fl = 0.0, l2r_qr_fl = 0.0, l2r_ap_fl = 0.0;
      for (int b = 0; b < nb; ++b) {
        const int* r = hr.data() + (size_t)b * (d + 1);
        for (int kc = 0; kc < d; ++kc) {
          dst[(size_t)b * d + kc] = tot;
          sz[(size_t)b * d + kc] = (int64_t)r[kc] * sh.n[kc] * r[kc + 1];
          tot += sz[(size_t)b * d + kc];
        }
        if (hsc[(size_t)b * 4 + 3] != 0.0) continue;
        for (int k = 1; k < d; ++k) {  // LAPACK-standard counts of the l2r operations
          const double pp = (double)r[k - 1] * sh.n[k - 1], cp = sh.Rp[k], rho = r[k];
          const double a1 = std::max(pp, cp), b1 = std::min(pp, cp);
          const double m1 = (double)sh.n[k] * sh.Rp[k + 1], c1 = sh.R[k];
          // R-SVD (GVL nominal 6ab^2 + 11b^3): the QR part 2ab^2 - 2b^3/3 is the qr
          // launch, the rest the svd launch
          const double qrf = (pp > BR_C) ? 2.0 * a1 * b1 * b1 - 2.0 * b1 * b1 * b1 / 3.0 : 0.0;
          l2r_qr_fl += qrf;
          l2r_svd_fl += 6.0 * a1 * b1 * b1 + 11.0 * b1 * b1 * b1 - qrf;
          // output core: Householder application (ormqr count) or the GEMM Y W (2 p c' rho); the
          // flag of the last split is what the host holds -- the choice is per (item, split), so
          // count the application for every split whose flag is unknown (an upper bound)
          if (pp > BR_C) l2r_ap_fl += (k == d - 1 && hgm[(size_t)b]) ? 2.0 * pp * cp * rho
                                                                     : 4.0 * pp * cp * rho - 2.0 * cp * cp * rho;
          l2r_ap_fl += 4.0 * m1 * std::min(m1, c1) * rho - 2.0 * std::min(m1, c1) * std::min(m1, c1) * rho;
        }
      }
      prof_credit(ctx, "batch_l2r_svd", l2r_svd_fl);
      prof_credit(ctx, "batch_l2r_qr", l2r_qr_fl);
      prof_credit(ctx, "batch_l2r_apply", l2r_ap_fl);
      void* arena = nullptr;
      if (cudaMallocAsync(&arena, (size_t)std::max<int64_t>(tot, 1) * sizeof(double), ctx->stream) != cudaSuccess) {
        // the stream-ordered pool keeps freed blocks cached: give them back and retry once
        (void)cudaGetLastError();
        cudaMemPool_t pool;
        TTB_CUDA(cudaStreamSynchronize(ctx->stream));
        TTB_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
        TTB_CUDA(cudaMemPoolTrimTo(pool, 0));
        if (cudaMallocAsync(&arena, (size_t)std::max<int64_t>(tot, 1) * sizeof(double), ctx->stream) != cudaSuccess) {
          (void)cudaGetLastError();
          fail(TT_ENOMEM, "batch result arena allocation failed");
        }
      }
      res.arenas.push_back(arena);
      res.arena_size.push_back(tot);
      res.wave_first.push_back(w0);
      BBuf ddst, dsz, dooff;
      ddst.upload(ctx, dst.data(), dst.size() * sizeof(int64_t), true);
      dsz.upload(ctx, sz.data(), sz.size() * sizeof(int64_t), true);
      dooff.upload(ctx, sh.ooff, sizeof(int64_t) * d, true);
      stamp("arena allocated");
      TTB_RUN(ctx, "batch_compact", 0.0, 16.0 * (double)tot,
              br_compact_kernel<<<nb, 256, 0, ctx->stream>>>(O.p, sh.ostride, static_cast<const int64_t*>(dooff.p),
                                                             static_cast<const int64_t*>(ddst.p),
                                                             static_cast<const int64_t*>(dsz.p), d,
                                                             static_cast<double*>(arena)));
      for (int b = 0; b < nb; ++b) {
        for (int k = 0; k <= d; ++k) res.ranks[(size_t)(w0 + b) * (d + 1) + k] = hr[(size_t)b * (d + 1) + k];
        for (int kc = 0; kc < d; ++kc)
          res.core[(size_t)(w0 + b) * d + kc] = static_cast<double*>(arena) + dst[(size_t)b * d + kc];
        res.norm[(size_t)(w0 + b)] = hsc[(size_t)b * 4 + 0];
        res.tau[(size_t)(w0 + b)] = hsc[(size_t)b * 4 + 1];
        res.scale[(size_t)(w0 + b)] = hsc[(size_t)b * 4 + 2];
      }
      stamp("wave done (host)");
    }
  } catch (...) {
    for (void* p : res.arenas) cudaFreeAsync(p, ctx->stream);
    res.arenas.clear();
    throw;
  }
}

void round_batch_uniform(tt_ctx ctx, const std::vector<SumInput>& items, const tt_round_opts& o, tt_tensor* out,
                         int64_t* ranks_out, tt_round_info* info) {
  BatchDesc in;
  const SumInput& f = items[0];
  in.B = (int)items.size();
  in.K = f.K();
  in.d = f.d;
  in.n = f.n;
  in.r = f.r;
  const int B = in.B, K = in.K, d = in.d;
  in.tab.resize((size_t)B * K * d);
  in.coef.resize((size_t)B * K);
  in.norm.resize((size_t)B * K);
  for (int b = 0; b < B; ++b)
    for (int l = 0; l < K; ++l) {
      in.coef[(size_t)b * K + l] = items[(size_t)b].coef[(size_t)l];
      in.norm[(size_t)b * K + l] = items[(size_t)b].norm[(size_t)l];
      for (int k = 0; k < d; ++k) in.tab[((size_t)b * K + l) * d + k] = items[(size_t)b].core[(size_t)l][(size_t)k];
    }
  BatchOut res;
  run_batch(ctx, in, o, res);
  // one refcount per wave arena, shared by that wave's tensors
  for (size_t w = 0; w < res.arenas.size(); ++w) {
    const int b0 = res.wave_first[w];
    const int b1 = (w + 1 < res.arenas.size()) ? res.wave_first[w + 1] : B;
    int64_t* refs = new int64_t(b1 - b0);
    for (int b = b0; b < b1; ++b) {
      tt_tensor tt = new tt_tensor_s();
      tt->d = d;
      tt->n = f.n;
      tt->r.assign(res.ranks.begin() + (size_t)b * (d + 1), res.ranks.begin() + (size_t)(b + 1) * (d + 1));
      tt->core.assign(res.core.begin() + (size_t)b * d, res.core.begin() + (size_t)(b + 1) * d);
      tt->core_c.assign(tt->core.begin(), tt->core.end());
      tt->norm = res.norm[(size_t)b];
      tt->arena = res.arenas[w];
      tt->arena_refs = refs;
      out[b] = tt;
      if (info) {
        info[b] = tt_round_info{};
        info[b].norm = res.norm[(size_t)b];
        info[b].scale = res.scale[(size_t)b];
        info[b].tau = res.tau[(size_t)b];
      }
      if (ranks_out)
        for (int k = 0; k <= d; ++k) ranks_out[(size_t)b * (d + 1) + k] = tt->r[(size_t)k];
    }
  }
}

}  // namespace ttb
