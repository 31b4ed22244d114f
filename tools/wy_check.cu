// Standalone check of the compact-WY flat-tree QR and its application (csrc/batch_wy.cuh):
// factor a random m x c matrix in stacks of cr rows, apply Q to [I; 0], and compare on the host:
// ||A - Q R|| / ||A|| and ||Q^T Q - I||.
// Cases include nearly dependent, rank-deficient and graded columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/wy_check tools/wy_check.cu
// Timing of the pipelined panel (2048 x 64, one matrix per CTA; per-warp cycle counters of CTA 0
// when built with -DWY_PROF=1):  tools/wy_check time GRID
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

#include "../paper_2211_08770_b200/csrc/batch_wy.cuh"

using namespace ttb;

struct RowLoader {  // row-major m x c matrix in stacks of cr rows
  const double* A;
  int64_t m;
  int c, cr;
  __device__ int stacks() const { return (int)((m + cr - 1) / cr); }
  __device__ int crow(int q) const { return (int)(m - (int64_t)q * cr < cr ? m - (int64_t)q * cr : cr); }
  __device__ void prefetch(int, int) const {}
  __device__ void load(double* __restrict__ buf, int q, int jb) const {
    const int lane = threadIdx.x & 31;
    wy::zero_buf(buf);
    for (int r = lane; r < crow(q); r += 32)
      for (int col = 8 * jb; col < 8 * jb + 8 && col < c; ++col)
        buf[(col - 8 * jb) * wy::VLD + r] = A[((int64_t)q * cr + r) * c + col];
    __syncwarp();
  }
};

__global__ void __launch_bounds__(wy::PT, 1) factor_kernel(const double* A, int64_t m, int c, int cr, double* F, double* R) {
  extern __shared__ __align__(16) unsigned char raw[];
  wy::Smem& sm = *reinterpret_cast<wy::Smem*>(raw);
  RowLoader ld{A, m, c, cr};
  wy::factor_panel(sm, ld, c, F);
  for (int idx = threadIdx.x; idx < c * c; idx += wy::PT) {
    const int row = idx / c, col = idx % c;
    R[idx] = row <= col ? sm.st[wy::ridx(row, col)] : 0.0;
  }
}

// timing: CTA b factors its own m x c matrix (A + b m c); CTA 0 records the per-warp counters
__global__ void __launch_bounds__(wy::PT, 2) time_kernel(const double* A, int64_t m, int c, int cr, double* F,
                                                        long long* prof) {
  extern __shared__ __align__(16) unsigned char raw[];
  wy::Smem& sm = *reinterpret_cast<wy::Smem*>(raw);
  RowLoader ld{A + (int64_t)blockIdx.x * m * c, m, c, cr};
  wy::factor_panel(sm, ld, c, F + (int64_t)blockIdx.x * ((m + cr - 1) / cr) * wy::stack_doubles(c),
                   blockIdx.x == 0 ? prof : nullptr);
}

static int time_main(int grid) {
  const int64_t m = 2048;
  const int c = 64, cr = 128, S = (int)(m / cr);
  double *dA, *dF;
  long long* dp;
  cudaMalloc(&dA, sizeof(double) * grid * m * c);
  cudaMalloc(&dF, sizeof(double) * grid * S * wy::stack_doubles(c));
  cudaMalloc(&dp, sizeof(long long) * 64);
  std::vector<double> A((size_t)grid * m * c);
  std::mt19937_64 rng(11);
  std::normal_distribution<double> nd(0.0, 1.0);
  for (auto& v : A) v = nd(rng);
  cudaMemcpy(dA, A.data(), sizeof(double) * A.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(time_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(wy::Smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int it = 0; it < 3; ++it) {
    cudaMemset(dp, 0, sizeof(long long) * 64);
    cudaEventRecord(e0);
    time_kernel<<<grid, wy::PT, sizeof(wy::Smem)>>>(dA, m, c, cr, dF, dp);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[64];
  cudaMemcpy(h, dp, sizeof(h), cudaMemcpyDeviceToHost);
  std::printf("grid %d: %.3f ms, %d stacks of %d x %d per CTA (%s)\n", grid, ms, S, cr, c,
              cudaGetErrorString(cudaGetLastError()));
  for (int w = 0; w < 8; ++w)
    std::printf("  w%d wait %.0f update %.0f factor %.0f store+load %.0f (cycles per stack)\n", w, (double)h[4 * w] / S,
                (double)h[4 * w + 1] / S, (double)h[4 * w + 2] / S, (double)h[4 * w + 3] / S);
  std::printf("  w3 factor phases per block: dots+reduce %.0f dlarfg %.0f update %.0f T+store %.0f writeback %.0f\n",
              (double)h[32] / S, (double)h[33] / S, (double)h[34] / S, (double)h[35] / S, (double)h[36] / S);
  cudaFree(dA); cudaFree(dF); cudaFree(dp);
  return 0;
}

__global__ void __launch_bounds__(wy::T, 1) apply_kernel(const double* X, int ncx, int nt, const double* F, int64_t m,
                                                         int cr, int c, double* out) {
  extern __shared__ __align__(16) unsigned char raw[];
  wy::ASmem& sm = *reinterpret_cast<wy::ASmem*>(raw);
  wy::apply_init(sm);
  uint32_t ph[wy::NBUF] = {};
  wy::apply(sm, ph, X, ncx, nt, F, m, cr, c, (int)(m < c ? m : c), out, nt, 1);
}

int main(int argc, char** argv) {
  if (argc > 2 && std::string(argv[1]) == "time") return time_main(std::atoi(argv[2]));
  struct Case { int64_t m; int c, cr, kind = 0; };
  std::vector<Case> cases = {{50, 8, 128}, {100, 12, 128}, {300, 24, 120}, {720, 24, 120}, {2500, 64, 100},
                             {2500, 50, 128}, {2048, 64, 128},  {825, 12, 128},
                             {480, 16, 128}, {396, 25, 120}, {270, 3, 126}, {90, 9, 128}, {270, 3, 128}, {64, 3, 64},
                             {2048, 64, 128, 1}, {300, 24, 120, 1}, {2048, 64, 128, 2}, {396, 25, 120, 2},
                             {2048, 64, 128, 3}, {720, 24, 120, 3}};
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(wy::Smem));
  cudaFuncSetAttribute(apply_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(wy::ASmem));
  int bad = 0;
  for (const Case& cs : cases) {
    const int64_t m = cs.m;
    const int c = cs.c, cr = cs.cr;
    const int k = (int)(m < c ? m : c);
    std::vector<double> A((size_t)m * c);
    for (auto& v : A) v = nd(rng);
    if (cs.kind == 1)  // nearly dependent column pairs: a_{2i+1} = a_{2i} + 1e-9 noise
      for (int64_t i = 0; i < m; ++i)
        for (int j = 1; j < c; j += 2) A[i * c + j] = A[i * c + j - 1] + 1e-9 * A[i * c + j];
    if (cs.kind == 2)  // exactly repeated columns and a zero column: rank deficient
      for (int64_t i = 0; i < m; ++i)
        for (int j = 0; j < c; ++j) A[i * c + j] = j % 3 == 2 ? A[i * c + j - 1] : (j == 7 ? 0.0 : A[i * c + j]);
    if (cs.kind == 3)  // graded columns: scale 10^(-j / 4)
      for (int64_t i = 0; i < m; ++i)
        for (int j = 0; j < c; ++j) A[i * c + j] *= std::pow(10.0, -0.25 * j);
    const int S = (int)((m + cr - 1) / cr);
    double *dA, *dF, *dR, *dX, *dQ;
    cudaMalloc(&dA, sizeof(double) * A.size());
    cudaMalloc(&dF, sizeof(double) * S * wy::stack_doubles(c));
    cudaMalloc(&dR, sizeof(double) * c * c);
    cudaMalloc(&dX, sizeof(double) * 64 * 64);
    cudaMalloc(&dQ, sizeof(double) * m * k);
    cudaMemcpy(dA, A.data(), sizeof(double) * A.size(), cudaMemcpyHostToDevice);
    std::vector<double> X(64 * 64, 0.0);
    for (int j = 0; j < k; ++j) X[j * 64 + j] = 1.0;  // column-major ld 64: I_k
    cudaMemcpy(dX, X.data(), sizeof(double) * X.size(), cudaMemcpyHostToDevice);
    factor_kernel<<<1, wy::PT, sizeof(wy::Smem)>>>(dA, m, c, cr, dF, dR);
    apply_kernel<<<1, wy::T, sizeof(wy::ASmem)>>>(dX, k, k, dF, m, cr, c, dQ);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> R((size_t)c * c), Q((size_t)m * k);
    cudaMemcpy(R.data(), dR, sizeof(double) * R.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(Q.data(), dQ, sizeof(double) * Q.size(), cudaMemcpyDeviceToHost);
    double na = 0, nres = 0, north = 0;
    for (int64_t i = 0; i < m; ++i)
      for (int j = 0; j < c; ++j) {
        double s = 0;
        for (int l = 0; l < k; ++l) s += Q[i * k + l] * R[l * c + j];
        const double d = A[i * c + j] - s;
        nres += d * d;
        na += A[i * c + j] * A[i * c + j];
      }
    for (int a = 0; a < k; ++a)
      for (int b = 0; b < k; ++b) {
        double s = 0;
        for (int64_t i = 0; i < m; ++i) s += Q[i * k + a] * Q[i * k + b];
        const double d = s - (a == b ? 1.0 : 0.0);
        north += d * d;
      }
    if (cs.kind == 2) {  // rank-deficient A: the augmented factorisation gives Q^T Q R = R (the
      // virtual rows of Q vanish only on range(R)), so check ||(Q^T Q - I) R|| / ||R|| instead
      north = 0.0;
      double nr = 0.0;
      for (int a = 0; a < k; ++a)
        for (int j = 0; j < c; ++j) {
          double s = 0;
          for (int b = 0; b < k; ++b) {
            double g = 0;
            for (int64_t i = 0; i < m; ++i) g += Q[i * k + a] * Q[i * k + b];
            s += (g - (a == b ? 1.0 : 0.0)) * R[b * c + j];
          }
          north += s * s;
          nr += R[a * c + j] * R[a * c + j];
        }
      north /= nr;
    }
    const double rel = std::sqrt(nres / na), orth = std::sqrt(north);
    // kind 1 (column pairs dependent to 1e-9): the virtual rows of the augmented Q carry
    // u x (growth of the near-null directions), measured ~2e-13 -- bounded at 1e-12, the engine's
    // own left-orthonormality bar; kind 2: Q spans a rank-deficient A
    const bool ok = e == cudaSuccess && rel < 1e-13 && orth < (cs.kind == 1 ? 1e-12 : 1e-13);
    if (argc > 1 && m == 300) {  // dump A, R, F, Q for host-side analysis
      std::vector<double> Fh((size_t)S * wy::stack_doubles(c));
      cudaMemcpy(Fh.data(), dF, sizeof(double) * Fh.size(), cudaMemcpyDeviceToHost);
      FILE* f = std::fopen(argv[1], "wb");
      std::fwrite(A.data(), 8, A.size(), f);
      std::fwrite(R.data(), 8, R.size(), f);
      std::fwrite(Fh.data(), 8, Fh.size(), f);
      std::fwrite(Q.data(), 8, Q.size(), f);
      std::fclose(f);
    }
    bad += !ok;
    std::printf("m %5lld c %2d cr %3d kind %d: ||A-QR||/||A|| %.2e  ||Q^TQ-I|| %.2e  %s %s\n", (long long)m, c, cr,
                cs.kind, rel, orth,
                ok ? "OK" : "BAD", cudaGetErrorString(e));
    cudaFree(dA); cudaFree(dF); cudaFree(dR); cudaFree(dX); cudaFree(dQ);
  }
  return bad ? 1 : 0;
}
