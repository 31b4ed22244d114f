// Blocked (compact-WY) Householder QR of tall panels on the FP64 tensor cores, one CTA per item
// (the batched engine, batch_round.cu).  PAPER.md:69 (rounding = QR sweeps of the core
// unfoldings), north star "core x R ... as FP64 DMMA tensor-core tiles".
//
// Flat tree over row chunks ("stacks"): the panel is cut into chunks of up to 128 rows and
//      [R; chunk]  ->  [R'; 0]
// is factored per stack with reflectors v = [e_j; v_chunk] (the 64-row R block is upper
// triangular, so a reflector's R part is the unit vector of its own row).  Stack 0 starts from
// R = 0: the panel is factored as [0; A] (an augmented panel with 64 virtual zero rows on top), so
// every stack has the same structure; A = Q R with Q = rows 64.. of the product of all reflectors
// applied to [I; 0] (the virtual rows of that product vanish wherever R has full row rank).
//
// Columns come in blocks of 8.  A *cell* (q, jb) -- column block jb of stack q -- is the work of
// one warp: load the 128 x 8 chunk, apply the published reflector blocks jb' < jb of the stack to
// it (W = R[8jb'.., blk jb] + V^T A, W' = T^T W, A -= V W', R rows -= W': mma.sync.m8n8k4.f64),
// factor it (8 reflectors, LAPACK dlarfg arithmetic) with its T (compact WY: H_1..H_8 = I - V T V^T),
// store V / T into the stack's factor in global memory and publish the cell.  Cell (q, jb) depends
// on (q, jb' < jb) (their V / T) and on (q - 1, jb) (the R rows of the block): a 2-D wavefront.
//
// Decoupled wavefront: the chunk of a cell lives in its warp's REGISTERS as transposed DMMA
// accumulator fragments (A^T tiles, 8 columns x 8 rows; a C fragment doubles as the A operand of
// the next product, contracting over its column index, so W^T = A^T V, W'^T = W^T T and
// A^T -= W'^T V^T chain through registers), shared memory holds only the R block and one staging
// buffer per warp, and a published block's V / T are read back from global memory (L2) by TMA bulk
// copies into the consumer's staging buffer.  So nothing ever waits for a consumer: warp w runs its
// own loop over the stacks, cell (q, (w + q) mod nblk) -- the rotation balances the cells' cost
// (jb updates + one factorisation) over the warps -- and waits only for pub[jb'] > q.
//
// Stored per stack and column block: V (WY_CH x 8, column-major ld VLD, rows beyond the chunk and
// columns beyond the panel zero) and T (8 x 8, row-major) behind it -- wy::apply applies them to
// thin targets.
#pragma once

#include "common.cuh"

// Cycle counters of factor_panel / factor_block / apply (CTA 0, TT_B200_BR_DEBUG): compiled in only
// with -DWY_PROF=1 (tools/wy_check time builds), so the production kernels carry no counters.
#ifndef WY_PROF
#define WY_PROF 0
#endif

namespace ttb {
namespace wy {

constexpr int T = 256;        // threads per CTA of the application kernel
constexpr int W = T / 32;     // its warps
#ifndef WY_PT
#define WY_PT 128
#endif
constexpr int PT = WY_PT;     // threads per CTA of the panel factorisation
constexpr int PW = PT / 32;   // its warps
constexpr int C = 64;         // max columns
constexpr int NB = 8;         // columns per reflector block
constexpr int CH = 128;       // max chunk rows per stack
constexpr int RR = 64;        // rows of the R block
constexpr int RT = (C / NB) * (C / NB + 1) / 2 * 64;  // doubles of the packed R block: the 36 upper 8 x 8 tiles
constexpr int VLD = CH + 4;   // ld of a staged V block / chunk buffer (132 = 4 mod 16)
constexpr int VBUF = NB * VLD + 64;  // staging buffer: V block (column-major ld VLD) + T (8 x 8 row-major)

// doubles of one stack's stored factor: one record of VBUF doubles per column block -- V (CH x 8,
// column-major ld VLD: the staging layout, so a block moves with ONE bulk copy) and its T behind it
__host__ __device__ inline int64_t stack_doubles(int ncol) { return (int64_t)VBUF * ((ncol + NB - 1) / NB); }

// Packed R block: tile (bi <= bj) at (bj (bj + 1) / 2 + bi) * 64, column-major inside the tile (the
// lower part of a diagonal tile stays zero).
__host__ __device__ inline int ridx(int row, int col) {
  const int bi = row >> 3, bj = col >> 3;
  return (bj * (bj + 1) / 2 + bi) * 64 + (col & 7) * 8 + (row & 7);
}

struct Smem {
  double st[RT];          // the R block, packed upper 8 x 8 tiles (ridx)
  double Vb[PW][VBUF];    // per-warp staging: the cell's chunk (loader / factorisation) or a staged V + T
  double red[32];
  uint64_t bar[PW];       // per-warp TMA completion barrier
  int pub[C / NB];        // stacks of block jb whose V / T are in global memory (monotone)
  int next;               // next unclaimed cell (wavefront order)
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done)
                 : "r"(su32(b)), "r"(parity)
                 : "memory");
  }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void pub_store(int* p, int v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(su32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int pub_load(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(su32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void pub_wait(const int* p, int need) {
  while (pub_load(p) < need) __nanosleep(64);
}

// Sum of eight per-lane values over the warp, every lane gets all eight (transposed butterfly).
__device__ __forceinline__ void warp_sum8v(double (&v)[8]) {
  const int lane = threadIdx.x & 31;
  const bool b4 = (lane & 16) != 0, b3 = (lane & 8) != 0, b2 = (lane & 4) != 0;
  double u4[4], u2[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double keep = b4 ? v[4 + k] : v[k], send = b4 ? v[k] : v[4 + k];
    u4[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double keep = b3 ? u4[2 + k] : u4[k], send = b3 ? u4[k] : u4[2 + k];
    u2[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  double u1 = (b2 ? u2[1] : u2[0]) + __shfl_xor_sync(0xffffffffu, b2 ? u2[0] : u2[1], 4);
  u1 += __shfl_xor_sync(0xffffffffu, u1, 2);
  u1 += __shfl_xor_sync(0xffffffffu, u1, 1);
#pragma unroll
  for (int c = 0; c < 8; ++c) v[c] = __shfl_sync(0xffffffffu, u1, ((c >> 2) & 1) * 16 + ((c >> 1) & 1) * 8 + (c & 1) * 4);
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- the cell's chunk as transposed accumulator fragments
// Lane (r8 = lane >> 2, q4 = lane & 3) keeps a[mt][e] = A[8 mt + P(2 q4 + e)][column r8 of the
// block], P(s) = s ^ (s >> 2) (slots 4..7 hold rows 5, 4, 7, 6): tile mt is the C fragment of the
// 8 x 8 tile A^T[column][slot].  The slot permutation makes every staged-V access below hit 16
// distinct banks per half-warp with the column-major ld VLD = 4 (mod 16).
__device__ __forceinline__ int slot_row(int s) { return s ^ (s >> 2); }

// buf (column-major ld VLD, 128 x 8) -> fragments
__device__ __forceinline__ void frag_load(double (&a)[CH / 8][2], const double* __restrict__ buf) {
  const int lane = threadIdx.x & 31, q4 = lane & 3, r8 = lane >> 2;
  const double* p = buf + r8 * VLD;
  const int o0 = slot_row(2 * q4), o1 = slot_row(2 * q4 + 1);
#pragma unroll
  for (int mt = 0; mt < CH / 8; ++mt) {
    a[mt][0] = p[8 * mt + o0];
    a[mt][1] = p[8 * mt + o1];
  }
}
__device__ __forceinline__ void frag_store(const double (&a)[CH / 8][2], double* __restrict__ buf) {
  const int lane = threadIdx.x & 31, q4 = lane & 3, r8 = lane >> 2;
  double* p = buf + r8 * VLD;
  const int o0 = slot_row(2 * q4), o1 = slot_row(2 * q4 + 1);
#pragma unroll
  for (int mt = 0; mt < CH / 8; ++mt) {
    p[8 * mt + o0] = a[mt][0];
    p[8 * mt + o1] = a[mt][1];
  }
}

// Apply the block staged in Vs (V column-major ld VLD, T behind it: block jb of the current stack)
// to the cell's fragments (column block blk): all three products chain through registers.
__device__ __forceinline__ void update_cell(Smem& sm, const double* __restrict__ Vs, double (&a)[CH / 8][2], int blk,
                                            int jb) {
  const int lane = threadIdx.x & 31, q4 = lane & 3, r8 = lane >> 2;
  // W^T[c][i] = R[8jb + i][8blk + c] + sum_rows A[row][c] V[row][i]   (C fragment: c = r8, i = 2 q4 + e)
  double* rp = sm.st + ridx(8 * jb, 8 * blk + r8);  // rows 8jb .. 8jb + 7 of the column: contiguous in tile (jb, blk)
  double c0 = rp[2 * q4], c1 = rp[2 * q4 + 1];
  double e0 = 0.0, e1 = 0.0, f0 = 0.0, f1 = 0.0, g0 = 0.0, g1 = 0.0;  // four independent chains
  const double* v1 = Vs + r8 * VLD;
  const int o0 = slot_row(2 * q4), o1 = slot_row(2 * q4 + 1);
#pragma unroll
  for (int mt = 0; mt < CH / 8; mt += 2) {
    dmma(c0, c1, a[mt][0], v1[8 * mt + o0]);
    dmma(e0, e1, a[mt][1], v1[8 * mt + o1]);
    dmma(f0, f1, a[mt + 1][0], v1[8 * mt + 8 + o0]);
    dmma(g0, g1, a[mt + 1][1], v1[8 * mt + 8 + o1]);
  }
  c0 += e0 + (f0 + g0);
  c1 += e1 + (f1 + g1);
  // W'^T[c][i'] = sum_i W^T[c][i] T[i][i'], i' = pi(2 q4 + e) = q4 + 4 e (B fragment column r8 -> i' = pi(r8))
  const double* Ts = Vs + NB * VLD;
  const int pr = (r8 >> 1) + 4 * (r8 & 1);
  double d0 = 0.0, d1 = 0.0;
  dmma(d0, d1, c0, Ts[(2 * q4) * 8 + pr]);
  dmma(d0, d1, c1, Ts[(2 * q4 + 1) * 8 + pr]);
  rp[q4] -= d0;
  rp[q4 + 4] -= d1;
  // A^T[c][slot] -= sum_i' W'^T[c][i'] V[row(slot)][i']
  const double n0 = -d0, n1 = -d1;
  const double* v2 = Vs + q4 * VLD + slot_row(r8);
#pragma unroll
  for (int mt = 0; mt < CH / 8; ++mt) {
    dmma(a[mt][0], a[mt][1], n0, v2[8 * mt]);
    dmma(a[mt][0], a[mt][1], n1, v2[4 * VLD + 8 * mt]);
  }
}

// The warp factors column block blk of the current stack from buf (its chunk, column-major ld VLD,
// rows >= the stack's rows zero): reflectors j = 8 blk + jj, T of the block; V (CH x 8, ld VLD) and
// T (8 x 8 row-major) go from the registers to Vout / Tout (global).  T is built
// column by column as the reflectors appear (T(0:jj, jj) = -tau_jj T(0:jj, 0:jj) V(:, 0:jj)^T v_jj,
// lane r keeping row r): the dots v_c^T v_jj (c < jj) ride in the same butterfly as the update dots
// v_jj^T a_c (c > jj) and the column mass sigma: one warp reduction per reflector.
template <bool PROF>
__device__ __forceinline__ void factor_block(Smem& sm, const double* __restrict__ buf, int blk, int nr,
                                             double* __restrict__ Vout, double* __restrict__ Tout, long long* fp) {
  // Columns jj >= nr of a partial block are zero (chunk and R rows), so their steps below are
  // exact no-ops (sigma = alpha = 0: tau = 0, beta = 0): the loop runs all NB steps branch-free.
  const int lane = threadIdx.x & 31;
  long long f0 = PROF ? clock64() : 0, facc[5] = {0, 0, 0, 0, 0};  // phase cycles (flushed at the end)
  auto tick = [&](int slot) {
    if (PROF) {
      const long long t = clock64();
      facc[slot] += t - f0;
      f0 = t;
    }
  };
  double* st = sm.st;
  const int db = ridx(8 * blk, 8 * blk);  // the block's diagonal tile
  double x[4][NB];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int c = 0; c < NB; ++c) x[t][c] = buf[c * VLD + 32 * t + lane];
  double trow[NB];  // row `lane` of T (lanes 0..7)
#pragma unroll
  for (int c = 0; c < NB; ++c) trow[c] = 0.0;
#pragma unroll
  for (int jj = 0; jj < NB; ++jj) {
    // R row 8 blk + jj of this block (only reflector jj touches it: loads off the dependency chain)
    const double alpha = st[db + jj * 8 + jj];
    double rj[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) rj[c] = c > jj ? st[db + c * 8 + jj] : 0.0;
    // one reduction for sigma = ||x_jj||^2 (slot jj), the dots x_jj^T a_c (c > jj: the update)
    // and x_jj^T v_c (c < jj: for T), all with the unscaled x_jj
    double dt[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const double p0 = x[0][jj] * x[0][c] + x[1][jj] * x[1][c];
      const double p1 = x[2][jj] * x[2][c] + x[3][jj] * x[3][c];
      dt[c] = p0 + p1;
    }
    warp_sum8v(dt);
    tick(0);
    const double sigma = dt[jj];
    // dlarfg with one reciprocal, branch-free (sigma = 0: H = I, beta = alpha)
    const double nrm = sqrt(fma(alpha, alpha, sigma));
    const double beta0 = alpha >= 0.0 ? -nrm : nrm;
    const double am = alpha - beta0;
    const double inv = 1.0 / (beta0 * am);
    const bool live = sigma != 0.0;
    const double tj = live ? -am * am * inv : 0.0;
    const double scal = live ? beta0 * inv : 0.0;
    const double beta = live ? beta0 : alpha;
    tick(1);
#pragma unroll
    for (int c = 0; c < NB; ++c) dt[c] *= scal;  // v_jj^T a_c (c > jj), v_c^T v_jj (c < jj)
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      if (c > jj) {
        const double wv = tj * (rj[c] + dt[c]);
        const double wsc = wv * scal;
#pragma unroll
        for (int t = 0; t < 4; ++t) x[t][c] -= wsc * x[t][jj];
        rj[c] -= wv;
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      x[t][jj] *= scal;
      __stcg(Vout + jj * VLD + 32 * t + lane, x[t][jj]);  // v_jj is final: its store drains behind the chain
    }
    tick(2);
    {  // T(lane, jj) for lane < jj, T(jj, jj) = tau
      double tv = 0.0;
#pragma unroll
      for (int q = 0; q < NB; ++q)
        if (q < jj && q >= lane) tv += trow[q] * dt[q];
      trow[jj] = lane < jj ? -tj * tv : (lane == jj ? tj : 0.0);
    }
    if (lane == 0) {
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c > jj) st[db + c * 8 + jj] = rj[c];
      st[db + jj * 8 + jj] = beta;
    }
    tick(3);
  }
  (void)nr;  // columns >= nr are zero and stored as such (consumers copy whole records)
  if (lane < NB) {
#pragma unroll
    for (int i = 0; i < NB; ++i) __stcg(Tout + lane * 8 + i, trow[i]);
  }
  tick(4);
  if (PROF && lane == 0)
#pragma unroll
    for (int i = 0; i < 5; ++i) fp[i] += facc[i];
}

// Zero the R block (all threads; the caller synchronises).
__device__ __forceinline__ void init(Smem& sm) {
  for (int idx = threadIdx.x; idx < RT; idx += PT) sm.st[idx] = 0.0;
  __syncthreads();
}

// Zero a chunk buffer (the warp's staging buffer) before a loader fills it (warp-synchronous).
__device__ __forceinline__ void zero_buf(double* buf) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int c = 0; c < NB; ++c)
#pragma unroll
    for (int t = 0; t < CH / 32; ++t) buf[c * VLD + 32 * t + lane] = 0.0;
  __syncwarp();
}

// ---------------------------------------------------------------- pipelined panel
// The whole flat tree of a panel, one loop per warp, no CTA barrier between stacks (see the top).
//   L.stacks(), L.crow(q) (rows of stack q), L.load(buf, q, jb) (the warp fills buf = the 128 x 8
//   chunk of column block jb of stack q, column-major ld VLD, rows >= crow and columns >= ncol
//   zero; warp-synchronous), L.prefetch(q, jb) (L2 prefetch hints for that load), out + q * stack_doubles(ncol).
// On return (after a CTA barrier) sm.st holds R (packed: ridx).
template <class Loader>
__device__ void factor_panel(Smem& sm, const Loader& L, int ncol, double* __restrict__ out,
                             long long* __restrict__ prof = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int nact = (ncol + NB - 1) / NB;  // active column blocks (all factored: nrefl = ncol)
  const int S = L.stacks();
  const int64_t sd = stack_doubles(ncol);
  if (tid < C / NB) sm.pub[tid] = 0;
  if (tid < PW) bar_init(&sm.bar[tid], 1);
  if (tid == 0) sm.next = 0;
  for (int idx = tid; idx < RT; idx += PT) sm.st[idx] = 0.0;  // R block = 0
  if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  {
    // prof (debugging, CTA 0): per warp cycles waiting for blocks (flag + TMA), applying them,
    // factoring + storing, and loading
    long long t0 = (WY_PROF && prof) ? clock64() : 0, tw = 0, tu = 0, tf = 0, tl = 0;
    double* buf = sm.Vb[w];
    uint32_t ph = 0;
    // Cells are claimed in wavefront order (anti-diagonals t = q + jb, heavy cells -- large jb --
    // first): every cell a claimed one depends on has a smaller index, so it is done or in the hands
    // of a warp that waits for smaller indices only; the warps' loads stay balanced whatever jb costs.
    const int ncell = S * nact;
    int td = 0, base = 0;  // current diagonal and the index of its first cell
    auto claim = [&](int& cq, int& cjb) {  // next cell in wavefront order; false: none left
      int idx = 0;
      if (lane == 0) idx = atomicAdd(&sm.next, 1);
      idx = __shfl_sync(0xffffffffu, idx, 0);
      if (idx >= ncell) return false;
      while (true) {
        const int ds = min(S - 1, td) - max(0, td - (nact - 1)) + 1;
        if (idx < base + ds) break;
        base += ds;
        ++td;
      }
      cq = max(0, td - (nact - 1)) + (idx - base);
      cjb = td - cq;
      return true;
    };
    int q = 0, jb = 0, qn = 0, jbn = 0;
    bool more = claim(q, jb);
#pragma unroll 1
    while (more) {
      double* o = out + (int64_t)q * sd;
      L.load(buf, q, jb);
      if (WY_PROF && prof) { const long long t = clock64(); tl += t - t0; t0 = t; }
      if (jb > 0) {
        double a[CH / 8][2];
        frag_load(a, buf);
        pub_wait(&sm.pub[jb], q);  // R rows of the block from stack q - 1
#pragma unroll 1
        for (int j2 = 0; j2 < jb; ++j2) {
          pub_wait(&sm.pub[j2], q + 1);
          if (WY_PROF && prof && w == 0 && lane == 0) prof[37] += clock64() - t0;  // flag part of warp 0's wait
          __syncwarp();
          if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            bar_expect(&sm.bar[w], (uint32_t)(VBUF * sizeof(double)));
            bulk_g2s(buf, o + (int64_t)j2 * VBUF, VBUF * sizeof(double), &sm.bar[w]);
          }
          bar_wait(&sm.bar[w], ph);
          ph ^= 1u;
          if (WY_PROF && prof) { const long long t = clock64(); tw += t - t0; t0 = t; }
          update_cell(sm, buf, a, jb, j2);
          __syncwarp();
          if (WY_PROF && prof) { const long long t = clock64(); tu += t - t0; t0 = t; }
        }
        frag_store(a, buf);
        __syncwarp();
      } else {
        pub_wait(&sm.pub[0], q);
      }
      double* Vo = o + (int64_t)jb * VBUF;
      double* To = Vo + NB * VLD;
      // the next cell is claimed before the factorisation so that its operands can be prefetched
      // (L2) behind it
      more = claim(qn, jbn);
      if (more) L.prefetch(qn, jbn);
      if (WY_PROF && prof && w == 3)
        factor_block<true>(sm, buf, jb, min(NB, ncol - NB * jb), Vo, To, prof + 32);
      else
        factor_block<false>(sm, buf, jb, min(NB, ncol - NB * jb), Vo, To, nullptr);
      __threadfence();
      asm volatile("fence.proxy.async;" ::: "memory");
      __syncwarp();
      if (lane == 0) pub_store(&sm.pub[jb], q + 1);
      if (WY_PROF && prof) { const long long t = clock64(); tf += t - t0; t0 = t; }
      q = qn;
      jb = jbn;
    }
    if (WY_PROF && prof && lane == 0) {
      prof[4 * w + 0] += tw;
      prof[4 * w + 1] += tu;
      prof[4 * w + 2] += tf;
      prof[4 * w + 3] += tl;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- applications
// Q [X; 0] for a factored panel: Q = (stack 0 blocks)(stack 1 blocks)..., each block
// I - V T V^T, so the last stack's last block is applied first; the target's R-block rows start
// as X and its chunk rows as 0 per stack (each chunk's rows are touched by its own stack only and
// are final once that stack is applied).  Target columns in passes of AN.
//
// The chunk rows of the target live in REGISTERS as transposed accumulator fragments (C^T tiles,
// 8 target columns x 8 rows, the slot permutation of frag_load): warp w keeps column tile
// w mod ntl4 and a 1/ksp share of the rows.  Per block: W^T = Rt^T + C^T V (partial over the warp's
// rows; the ksp partials of a column tile meet through shared memory -- the one CTA barrier of the
// block), W'^T = W^T T^T, Rt rows -= W', C^T -= W'^T V^T, all DMMA with the accumulators doubling as
// A operands.  V / T records arrive by one TMA bulk copy each, one block ahead (ring of NBUF).
constexpr int AN = 32;           // target columns per pass
constexpr int RLD = RR;          // ld of the R-block target (few accesses: no padding)
constexpr int NBUF = 2;          // staging ring depth
struct ASmem {
  double Rt[AN * RLD];           // R-block rows of the target (column-major)
  double VT[NBUF][VBUF];         // staged block records (V column-major ld VLD, then T)
  double Wp[2][W][64];           // partial W^T fragments (lane-major), double-buffered by block parity
  uint64_t bar[NBUF];
};

__device__ __forceinline__ void apply_init(ASmem& sm) {
  if (threadIdx.x == 0) {
    for (int b = 0; b < NBUF; ++b) bar_init(&sm.bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
}

// Stage block jb of the stack factor F into buffer b (thread 0).
__device__ __forceinline__ void stage_block(ASmem& sm, const double* F, int jb, int b) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  bar_expect(&sm.bar[b], (uint32_t)(VBUF * sizeof(double)));
  bulk_g2s(sm.VT[b], F + (int64_t)jb * VBUF, VBUF * sizeof(double), &sm.bar[b]);
}

// out[row * rs + col * cs] = (Q [X; 0])[row][col] for the m panel rows, X = src (ncx x nt,
// column-major ld 64, global).  Stack q holds panel rows [q cr, min(m, (q+1) cr)), factor at
// F + q * stack_doubles(ncol).  ph[]: the staging barriers' phase bits (kept across calls).
__device__ void apply(ASmem& sm, uint32_t (&ph)[NBUF], const double* __restrict__ src, int ncx, int nt,
                      const double* __restrict__ F0, int64_t m, int cr, int ncol, int nrefl, double* __restrict__ out,
                      int64_t rs, int64_t cs, long long* ap = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, q4 = lane & 3, r8 = lane >> 2;
  long long a0 = (WY_PROF && ap && tid == 0) ? clock64() : 0, aacc[5] = {0, 0, 0, 0, 0};
  auto tk = [&](int slot) {
    if (WY_PROF && ap && tid == 0) {
      const long long t = clock64();
      aacc[slot] += t - a0;
      a0 = t;
    }
  };
  const int S = (int)((m + cr - 1) / cr);
  const int nbr = (nrefl + NB - 1) / NB;
  const int64_t sd = stack_doubles(ncol);
  const int tot = S * nbr;
  const int o0 = slot_row(2 * q4), o1 = slot_row(2 * q4 + 1), pr8 = slot_row(r8);
  const int pr = (r8 >> 1) + 4 * (r8 & 1);  // i' of B-fragment column r8 (W'^T comes out with i' = q4 + 4 e)
#pragma unroll 1
  for (int t0 = 0; t0 < nt; t0 += AN) {
    const int ntp = min(AN, nt - t0), ntl = (ntp + 7) >> 3;
    const int ntl4 = ntl == 3 ? 4 : ntl;  // a divisor of 8: each warp keeps one column tile
    const int ksp = 8 / ntl4;             // row shares per column tile
    const int ntile = (CH / 8) / ksp;     // 8-row tiles per warp (2, 4 or 8)
    const int nti = w % ntl4, rsp = w / ntl4, mt0 = rsp * ntile;
    const bool on = nti < ntl;
    __syncthreads();  // the previous pass is done with Rt and the ring
    for (int idx = tid; idx < AN * RR; idx += T) {
      const int c = idx / RR, r = idx % RR;
      sm.Rt[c * RLD + r] = (c < ntp && r < ncx) ? src[(int64_t)(t0 + c) * 64 + r] : 0.0;
    }
    if (tid == 0) stage_block(sm, F0 + (int64_t)(S - 1) * sd, nbr - 1, 0);
    __syncthreads();
    double* rt = sm.Rt + (8 * nti + r8) * RLD;
#pragma unroll 1
    for (int q = S - 1; q >= 0; --q) {
      const int64_t row0 = (int64_t)q * cr;
      const int crow = (int)(m - row0 < cr ? m - row0 : cr);
      double ct[CH / 16][2];
#pragma unroll
      for (int u = 0; u < CH / 16; ++u) ct[u][0] = ct[u][1] = 0.0;
#pragma unroll 1
      for (int jb = nbr - 1; jb >= 0; --jb) {
        // block sequence index over the whole pass (stacks descending, blocks descending)
        const int tq = (S - 1 - q) * nbr + (nbr - 1 - jb), b = tq % NBUF;
        tk(4);
        bar_wait(&sm.bar[b], ph[b]);
        ph[b] ^= 1u;
        tk(0);
        const double* Vs = sm.VT[b];
        // ---- partial W^T[c][i] = Rt[8jb + i][c] (first row share) + sum over the warp's rows C^T V
        if (on) {
          double c0 = 0.0, c1 = 0.0, e0 = 0.0, e1 = 0.0;
          if (rsp == 0) {
            c0 = rt[8 * jb + 2 * q4];
            c1 = rt[8 * jb + 2 * q4 + 1];
          }
          if (jb != nbr - 1) {  // (the chunk rows are still zero at a stack's first block)
            const double* v1 = Vs + r8 * VLD + 8 * mt0;
#pragma unroll
            for (int u = 0; u < CH / 16; ++u)
              if (u < ntile) {
                dmma(c0, c1, ct[u][0], v1[8 * u + o0]);
                dmma(e0, e1, ct[u][1], v1[8 * u + o1]);
              }
          }
          *reinterpret_cast<double2*>(&sm.Wp[tq & 1][w][2 * lane]) = make_double2(c0 + e0, c1 + e1);
        }
        tk(1);
        __syncthreads();
        tk(2);
        // the ring: block tq + 1 goes into the buffer block tq - 1 used (every warp is past it)
        if (tid == 0 && tq + 1 < tot) {
          const int u = tq + 1, uq = S - 1 - u / nbr, ujb = nbr - 1 - u % nbr;
          stage_block(sm, F0 + (int64_t)uq * sd, ujb, u % NBUF);
        }
        if (on) {
          double s0 = 0.0, s1 = 0.0;
          for (int ks = 0; ks < ksp; ++ks) {
            const double2 pv = *reinterpret_cast<const double2*>(&sm.Wp[tq & 1][nti + ks * ntl4][2 * lane]);
            s0 += pv.x;
            s1 += pv.y;
          }
          // W'^T[c][i'] = sum_i W^T[c][i] T[i'][i]
          const double* Ts = Vs + NB * VLD + pr * 8;
          double d0 = 0.0, d1 = 0.0;
          dmma(d0, d1, s0, Ts[2 * q4]);
          dmma(d0, d1, s1, Ts[2 * q4 + 1]);
          if (rsp == 0) {
            rt[8 * jb + q4] -= d0;
            rt[8 * jb + q4 + 4] -= d1;
          }
          const double n0 = -d0, n1 = -d1;
          const double* v2 = Vs + q4 * VLD + 8 * mt0 + pr8;
#pragma unroll
          for (int u = 0; u < CH / 16; ++u)
            if (u < ntile) {
              dmma(ct[u][0], ct[u][1], n0, v2[8 * u]);
              dmma(ct[u][0], ct[u][1], n1, v2[4 * VLD + 8 * u]);
            }
        }
        tk(3);
      }
      // the stack's rows are final: registers -> out
      const int col = 8 * nti + r8;
      if (on && col < ntp) {
        double* op = out + (int64_t)(t0 + col) * cs;
#pragma unroll
        for (int u = 0; u < CH / 16; ++u)
          if (u < ntile) {
            const int ra = 8 * (mt0 + u) + o0, rb = 8 * (mt0 + u) + o1;
            if (ra < crow) op[(row0 + ra) * rs] = ct[u][0];
            if (rb < crow) op[(row0 + rb) * rs] = ct[u][1];
          }
      }
    }
  }
  __syncthreads();
  if (WY_PROF && ap && tid == 0)
#pragma unroll
    for (int i = 0; i < 5; ++i) ap[i] += aacc[i];
}

}  // namespace wy
}  // namespace ttb
