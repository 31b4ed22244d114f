// TT-dot Gram matrix of m equally shaped TT-vectors, pair-tiled (Alg. 5 lines 2-6, Eq. (3):
// G(i,j) = <a_i, a_j>; PAPER.md:19 dot through the core contraction).
//
// One CTA per tile of 2 x 2 pairs (i in I, j in J, tiles of the lower triangle), one warp per
// pair.  Per pair the left-to-right recursion W_k = sum_s X^(i)_k(s)^T W_{k-1} X^(j)_k(s) runs as
// two small GEMMs per mode slice on the FP64 tensor cores (DMMA): U = W X^(j)(s), V += X^(i)(s)^T U;
// the tile's four tensors' slices X(s) are staged once (cp.async) and reused by all its pairs.
// A tile runs on a cluster of CS CTAs that split the mode slices of every core (more CTAs in
// flight and better balance: the C3 Gram has only 325 tiles for 148 SMs); the partial V of each
// CTA meet through distributed shared memory once per core, summed in cluster-rank order.
// Summation order is fixed (deterministic).
#include <cooperative_groups.h>
#include <cuda_pipeline.h>

#include <algorithm>

#include "gram.cuh"

namespace cg = cooperative_groups;

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

struct GramShape {  // modes and the rank profiles of the I-side (r) and J-side (q) tensors
  int d;
  int n[GT_MAXD];
  int r[GT_MAXD + 1];
  int q[GT_MAXD + 1];
};


// ---- FP64 tensor-core (DMMA, mma.sync m8n8k4) kernel: one warp per pair of the 2 x 2 tile.
// Warp p = 2 i + j keeps W and V in DMMA fragments (registers) for the whole core; per mode
// slice s it forms U^T = X^(j)(s)^T W^T and then V += X^(i)(s)^T U -- no cross-warp dependency
// inside a slice, one __syncthreads per slice for the staged slices (cp.async from a per-core copy
// list in shared memory: one 16-byte copy per list entry and thread, no per-copy index
// arithmetic; double buffered, the next core's first slice prefetched during the last slice of
// the current one).  One warp per SM sub-partition with >= 2 independent accumulators saturates
// the DMMA pipe (tools/dmma_bench: latency 26 cycles, 16 cycles per DMMA per sub-partition).
// Ranks are padded to 8 NT with zeros; the row stride L = 4 or 12 (mod 16) keeps the fragment
// loads free of bank conflicts.  C3 Gram (profiles/ncu_r02_v2.md): DMMA sub-pipe 62 % busy;
// the padding 20 -> 24 on M and N costs the rest.
__device__ __forceinline__ void gmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

constexpr int GM_T = 128;  // threads per CTA: one warp per pair

// ---- register-chained version: the two GEMMs of a slice pass U through registers.  U^T =
// X_j(s)^T W^T leaves U^T in C fragments (thread (g, tg) holds U^T[8x + g][8y + 2tg + e]); read
// as B[k][n] of V += X_i(s)^T U with the k positions of a k-step taken as 8z + 2tg + e (e fixed)
// -- a relabelling of the contraction index, matched by the A fragments' row offsets -- they are
// exactly the B fragments, and likewise V's C fragments are next core's W^T B fragments.  No
// shared-memory round trip of U, no fragment shuffles.  A rank whose last 8-block is at most half
// full places that block's entries on the even positions (rc_pos), so the odd k-step of the
// block is all padding and skipped: K steps = ceil(r / 4), as with natural k-steps of 4.
__device__ __forceinline__ int rc_pos(int p, int nt, bool half) {
  const int b = 8 * (nt - 1);
  if (!half || p < b || p >= b + 8) return p;
  const int l = p - b;
  return b + ((l & 1) ? 4 + (l >> 1) : (l >> 1));
}

template <int NT>
__global__ void __launch_bounds__(GM_T, NT >= 4 ? 1 : 3) gram_rc_kernel(const double* const* __restrict__ cores,
                                                                      GramShape sh, int m,
                                                                      const GramTile* __restrict__ tiles, int L,
                                                                      double* __restrict__ G) {
  extern __shared__ __align__(16) double gsm[];
  constexpr int RP = 8 * NT;
  const int MB = RP * L;                    // one matrix block
  double* U = gsm;                          // [pair][a][c'] row-major, stride L (also W at core ends)
  double* XB = U + GT_P * MB;               // 2 buffers x [I0, I1, J0, J1][a][a']
  // copy list of the staged slices (16-byte cp.async, even ranks): entry q = {offset of the
  // chunk inside its tensor's core (doubles, without the slice term), destination | slot << 24}
  int2* gdesc = reinterpret_cast<int2*>(XB + 2 * (GT_I + GT_J) * MB);
  __shared__ const double* gbase[2][GT_I + GT_J];  // core pointers of the tile's tensors, by core parity
  const int tid = threadIdx.x, lane = tid & 31, p = tid >> 5, g = lane >> 2, tg = lane & 3;
  const int pi = p / GT_J, pj = p % GT_J;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), crank = (int)cl.block_rank();
  const GramTile tl = tiles[blockIdx.x / CS];
  const int i0 = tl.i0, j0 = tl.j0, d = sh.d;
  double* Up = U + p * MB;
  // W as the C fragments of the previous core's V (W[8x + g][8y + 2tg + e]); W_0 = 1 (1 x 1)
  double wf[NT][NT][2];
#pragma unroll
  for (int x = 0; x < NT; ++x)
#pragma unroll
    for (int y = 0; y < NT; ++y) wf[x][y][0] = wf[x][y][1] = 0.0;
  wf[0][0][0] = (g == 0 && tg == 0) ? 1.0 : 0.0;
  double gv = 0.0;
  // Staged rows of core kk: the tile's I tensors (R0i rows of R1i doubles) then its J tensors
  // (R0j rows of R1j), clamped into the tile's block, so a padding tensor has its side's shape
  // (its pairs are never written).
  auto set_bases = [&](int kk) {
    if (tid < GT_I + GT_J) {
      const int tens = tid < GT_I ? min(i0 + tid, tl.ilim - 1) : min(j0 + tid - GT_I, tl.jlim - 1);
      gbase[kk & 1][tid] = cores[(int64_t)tens * d + kk];
    }
  };
  auto even = [&](int kk) { return ((sh.r[kk + 1] | sh.q[kk + 1]) & 1) == 0; };
  auto nq_of = [&](int kk) { return GT_I * sh.r[kk] * (sh.r[kk + 1] / 2) + GT_J * sh.q[kk] * (sh.q[kk + 1] / 2); };
  auto build = [&](int kk) {  // copy list of core kk's shape (n, R0i, R1i, R0j, R1j)
    const int nk = sh.n[kk], R0i = sh.r[kk], R1i = sh.r[kk + 1], R0j = sh.q[kk], R1j = sh.q[kk + 1];
    const int nI = GT_I * R0i * (R1i / 2), nq = nI + GT_J * R0j * (R1j / 2);
    for (int q = tid; q < nq; q += GM_T) {
      const bool iside = q < nI;
      const int qq = iside ? q : q - nI, cpr = (iside ? R1i : R1j) / 2, R0 = iside ? R0i : R0j;
      const int row = qq / cpr, c = qq - row * cpr, tt = row / R0, a = row - tt * R0;
      const int slot = iside ? tt : GT_I + tt;
      gdesc[q] = make_int2(a * nk * (iside ? R1i : R1j) + 2 * c, (slot * MB + a * L + 2 * c) | (slot << 24));
    }
  };
  auto stage = [&](int kk, int s, int b) {
    double* buf = XB + b * (GT_I + GT_J) * MB;
    const int R1i = sh.r[kk + 1], R1j = sh.q[kk + 1];
    if (even(kk)) {
      const int nq = nq_of(kk);
      for (int q = tid; q < nq; q += GM_T) {
        const int2 e = gdesc[q];
        const int slot = e.y >> 24;
        const double* src = gbase[kk & 1][slot] + e.x + (int64_t)s * (slot < GT_I ? R1i : R1j);
        __pipeline_memcpy_async(buf + (e.y & 0xffffff), src, 2 * sizeof(double));
      }
    } else {  // odd ranks: 8-byte copies, indices decoded per element
      const int nk = sh.n[kk], R0i = sh.r[kk], R0j = sh.q[kk];
      const int eI = GT_I * R0i * R1i, tot = eI + GT_J * R0j * R1j;
      for (int q = tid; q < tot; q += GM_T) {
        const bool iside = q < eI;
        const int qq = iside ? q : q - eI, R1 = iside ? R1i : R1j, R0 = iside ? R0i : R0j;
        const int row = qq / R1, c = qq - row * R1, tt = row / R0, a = row - tt * R0;
        const int slot = iside ? tt : GT_I + tt;
        __pipeline_memcpy_async(buf + slot * MB + a * L + c,
                                gbase[kk & 1][slot] + ((int64_t)a * nk + s) * R1 + c, sizeof(double));
      }
    }
    __pipeline_commit();
  };
  auto srange = [&](int kk, int& b0, int& b1) {
    b0 = (int)((int64_t)crank * sh.n[kk] / CS);
    b1 = (int)((int64_t)(crank + 1) * sh.n[kk] / CS);
  };
  int bufc = 0;           // buffer of the next slice to consume
  bool staged = false;    // core k's first slice already in flight (prefetched by core k-1)
#pragma unroll 1
  for (int k = 0; k < d; ++k) {
    int sb, se;
    srange(k, sb, se);
    // the next core can be prefetched when its staged slices have the same shape (same copy
    // list; pads stay zero)
    const bool pre_next = k + 1 < d && sh.n[k + 1] == sh.n[k] && sh.r[k + 1] == sh.r[k] &&
                          sh.r[k + 2] == sh.r[k + 1] && sh.q[k + 1] == sh.q[k] && sh.q[k + 2] == sh.q[k + 1];
    if (!staged) {
      __syncthreads();  // every warp is done reading the previous core's slices and copy list
      for (int idx = tid; idx < 2 * (GT_I + GT_J) * MB; idx += GM_T) XB[idx] = 0.0;  // pads stay zero
      if (even(k)) build(k);
      set_bases(k);
      __syncthreads();
      if (sb < se) stage(k, sb, bufc);
    }
    if (pre_next) set_bases(k + 1);  // read after the slice loop's first barrier
    staged = false;
    // rank spaces of this core: a = r_{k-1} (rows of the slices), a' = r_k (columns), per side
    const int nti0 = (sh.r[k] + 7) >> 3, nti1 = (sh.r[k + 1] + 7) >> 3;
    const int ntj0 = (sh.q[k] + 7) >> 3, ntj1 = (sh.q[k + 1] + 7) >> 3;
    const bool pi0 = sh.r[k] - 8 * (nti0 - 1) <= 4, pi1 = sh.r[k + 1] - 8 * (nti1 - 1) <= 4;
    const bool pj0 = sh.q[k] - 8 * (ntj0 - 1) <= 4, pj1 = sh.q[k + 1] - 8 * (ntj1 - 1) <= 4;
    // fragment offsets inside a staged slice: rows at the k-step positions 8z + 2tg + e, columns
    // at the M positions 8x + g (rc_pos: the half-full last block on the even positions)
    int ci[NT], cj[NT], ri[NT][2], rj[NT][2];
#pragma unroll
    for (int x = 0; x < NT; ++x) {
      ci[x] = rc_pos(8 * x + g, nti1, pi1);
      cj[x] = rc_pos(8 * x + g, ntj1, pj1);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        ri[x][e] = rc_pos(8 * x + 2 * tg + e, nti0, pi0) * L;
        rj[x][e] = rc_pos(8 * x + 2 * tg + e, ntj0, pj0) * L;
      }
    }
    double v[NT][NT][2];
#pragma unroll
    for (int x = 0; x < NT; ++x)
#pragma unroll
      for (int y = 0; y < NT; ++y) v[x][y][0] = v[x][y][1] = 0.0;
#pragma unroll 1
    for (int s = sb; s < se; ++s) {
      const double* XS = XB + bufc * (GT_I + GT_J) * MB;
      __pipeline_wait_prior(0);
      __syncthreads();  // slice s visible to all; everyone is done with the other buffer
      if (s + 1 < se) {
        stage(k, s + 1, bufc ^ 1);
      } else if (pre_next) {  // first slice of the next core, overlapped with this slice's math
        int nb, ne;
        srange(k + 1, nb, ne);
        if (nb < ne) stage(k + 1, nb, bufc ^ 1);
        staged = true;
      }
      bufc ^= 1;
      const double* Xi = XS + pi * MB;
      const double* Xj = XS + (GT_I + pj) * MB;
      // U^T = X_j(s)^T W^T: A[c'][c] = X_j[c][c'] (smem), B[c][a] = W[a][c] (registers, the C
      // fragments of the previous core's V: k positions 8z + 2tg + e)
      double u[NT][NT][2];
#pragma unroll
      for (int x = 0; x < NT; ++x)
#pragma unroll
        for (int y = 0; y < NT; ++y) u[x][y][0] = u[x][y][1] = 0.0;
#pragma unroll
      for (int z = 0; z < NT; ++z) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (z < ntj0 && !(e == 1 && z == ntj0 - 1 && pj0)) {
            double af[NT];
#pragma unroll
            for (int x = 0; x < NT; ++x) af[x] = Xj[rj[z][e] + cj[x]];
#pragma unroll
            for (int x = 0; x < NT; ++x)
#pragma unroll
              for (int y = 0; y < NT; ++y)
                gmma(u[x][y][0], u[x][y][1], af[x], wf[y][z][e]);  // pad tiles: zero operands
          }
        }
      }
      // V += X_i(s)^T U: A[a'][a] = X_i[a][a'] (smem), B[a][c'] = U^T[c'][a] (the C fragments of u)
#pragma unroll
      for (int z = 0; z < NT; ++z) {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (z < nti0 && !(e == 1 && z == nti0 - 1 && pi0)) {
            double af[NT];
#pragma unroll
            for (int x = 0; x < NT; ++x) af[x] = Xi[ri[z][e] + ci[x]];
#pragma unroll
            for (int x = 0; x < NT; ++x)
#pragma unroll
              for (int y = 0; y < NT; ++y)
                gmma(v[x][y][0], v[x][y][1], af[x], u[y][z][e]);
          }
        }
      }
    }
    // W_k = V (summed over the cluster's slice ranges, cluster-rank order): C fragments in place
    if (CS > 1) {
#pragma unroll
      for (int x = 0; x < NT; ++x)
#pragma unroll
        for (int y = 0; y < NT; ++y)
          *reinterpret_cast<double2*>(Up + (8 * x + g) * L + 8 * y + 2 * tg) = make_double2(v[x][y][0], v[x][y][1]);
      cl.sync();  // every CTA's partial is complete
#pragma unroll
      for (int x = 0; x < NT; ++x)
#pragma unroll
        for (int y = 0; y < NT; ++y) {
          double w0 = 0.0, w1 = 0.0;
          for (int c = 0; c < CS; ++c) {
            const double2 t = *reinterpret_cast<const double2*>(cl.map_shared_rank(Up, c) + (8 * x + g) * L + 8 * y + 2 * tg);
            w0 += t.x;
            w1 += t.y;
          }
          wf[x][y][0] = w0;
          wf[x][y][1] = w1;
        }
      cl.sync();  // partials read everywhere before they are rewritten
    } else {
#pragma unroll
      for (int x = 0; x < NT; ++x)
#pragma unroll
        for (int y = 0; y < NT; ++y) {
          wf[x][y][0] = v[x][y][0];
          wf[x][y][1] = v[x][y][1];
        }
    }
    if (k == d - 1) gv = wf[0][0][0];
  }
  if (lane == 0 && crank == 0) {
    const int i = i0 + pi, j = j0 + pj;
    if (tl.mode == 0) {
      if (i < m && j < m && i >= j) {
        G[(int64_t)i * m + j] = gv;
        G[(int64_t)j * m + i] = gv;
      }
    } else if (i < tl.ilim && j < tl.jlim) {
      G[tl.off + (int64_t)(i - tl.bi0) * tl.bj + (j - tl.bj0)] = gv;
    }
  }
}

}  // namespace

bool gram_tiled_supported(const std::vector<const double*>& cores, int m, int d, const std::vector<int64_t>& n,
                          const std::vector<int64_t>& r) {
  if (m < 1 || d < 1 || d > GT_MAXD) return false;
  for (const double* c : cores)  // 16-byte cp.async rows
    if (reinterpret_cast<uintptr_t>(c) & 15) return false;
  int rmax = 1;
  for (int k = 0; k <= d; ++k) rmax = std::max<int>(rmax, (int)r[(size_t)k]);
  for (int k = 0; k < d; ++k)
    if (n[(size_t)k] < 1) return false;
  return rmax <= 32;  // ranks padded to 8 NT, NT <= 4 (one pair's fragments per warp)
}

static void gram_launch(tt_ctx ctx, const std::vector<const double*>& cores, int m, int d,
                        const std::vector<int64_t>& n, const std::vector<int64_t>& r, const std::vector<int64_t>& q,
                        const std::vector<GramTile>& tiles, double npairs, double* out) {
  GramShape sh{};
  sh.d = d;
  int rmax = 1;
  double flops = 0.0;
  for (int k = 0; k < d; ++k) {
    sh.n[k] = (int)n[(size_t)k];
    const double Ri0 = (double)r[(size_t)k], Ri1 = (double)r[(size_t)k + 1];
    const double Rj0 = (double)q[(size_t)k], Rj1 = (double)q[(size_t)k + 1];
    // per pair: U = W X_j (Ri0 Rj0 Rj1), V = X_i^T U (Ri0 Ri1 Rj1)
    flops += 2.0 * (double)n[(size_t)k] * (Ri0 * Rj0 * Rj1 + Ri0 * Ri1 * Rj1);
  }
  for (int k = 0; k <= d; ++k) {
    sh.r[k] = (int)r[(size_t)k];
    sh.q[k] = (int)q[(size_t)k];
    rmax = std::max<int>(rmax, (int)std::max(r[(size_t)k], q[(size_t)k]));
  }
  if (tiles.empty()) return;
  BBuf dt, dc;
  dt.upload(ctx, tiles.data(), tiles.size() * sizeof(GramTile));
  dc.upload(ctx, cores.data(), cores.size() * sizeof(double*));
  double bytes = 0.0;
  for (int k = 0; k < d; ++k) bytes += 8.0 * (double)m * r[(size_t)k] * n[(size_t)k] * r[(size_t)k + 1];
  const int ntiles = (int)tiles.size();
  const GramTile* tp = static_cast<const GramTile*>(dt.p);
  const int NT = (rmax + 7) / 8;
  int L = 8 * NT;  // row stride: 4 or 12 (mod 16) keeps the fragment loads conflict-free
  while (L % 16 != 4 && L % 16 != 12) ++L;
  const size_t smem_m = sizeof(double) * (size_t)(GT_P + 2 * (GT_I + GT_J)) * (8 * NT) * L +
                        sizeof(int2) * (size_t)(GT_I + GT_J) * (8 * NT) * (4 * NT);  // copy list
  auto kern = NT == 1 ? gram_rc_kernel<1> : NT == 2 ? gram_rc_kernel<2> : NT == 3 ? gram_rc_kernel<3>
                                                                                 : gram_rc_kernel<4>;
  const int T = GM_T;
  TTB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_m));
  TTB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  // slice split: the smallest cluster size that fills every resident slot once
  // (>= 2 slices per CTA, <= 8 CTAs per cluster)
  int per_sm = 1;
  TTB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, T, smem_m));
  int nmin = 1 << 30;
  for (int k = 0; k < d; ++k) nmin = std::min(nmin, (int)n[(size_t)k]);
  static const char* cs_env = std::getenv("TT_B200_GRAM_CS");
  int CS = 1;
  while (CS < 8 && 2 * CS <= nmin / 2 && (int64_t)ntiles * CS < (int64_t)ctx->num_sms * std::max(per_sm, 1)) CS *= 2;
  if (cs_env) CS = std::max(1, std::min(8, std::atoi(cs_env)));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(ntiles * CS));
  cfg.blockDim = dim3((unsigned)T);
  cfg.dynamicSmemBytes = smem_m;
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)CS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const double* const* cp = static_cast<const double* const*>(dc.p);
  TTB_RUN(ctx, "tt_gram_tiled", flops * npairs, bytes,
          TTB_CUDA(cudaLaunchKernelEx(&cfg, kern, cp, sh, m, tp, L, out)));
}

void gram_tiled(tt_ctx ctx, const std::vector<const double*>& cores, int m, int d, const std::vector<int64_t>& n,
                const std::vector<int64_t>& r, double* G_dev) {
  std::vector<GramTile> tiles;
  for (int i0 = 0; i0 < m; i0 += GT_I)
    for (int j0 = 0; j0 < m; j0 += GT_J)
      if (i0 + GT_I - 1 >= j0) tiles.push_back(GramTile{i0, j0, m, m, 0, 0, 0, 0, 0});  // holds a pair i >= j
  gram_launch(ctx, cores, m, d, n, r, r, tiles, 0.5 * m * (m + 1.0), G_dev);
}

void gram_tiled_blocks(tt_ctx ctx, const std::vector<const double*>& cores, int m, int d,
                       const std::vector<int64_t>& n, const std::vector<int64_t>& r, int nblk, const int32_t* blk,
                       double* packed_dev, const std::vector<int64_t>* rj) {
  const std::vector<int64_t>& q = rj ? *rj : r;
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
  gram_launch(ctx, cores, m, d, n, r, q, tiles, npairs, packed_dev);
}

}  // namespace ttb
