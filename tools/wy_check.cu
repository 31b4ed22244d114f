// Standalone check of the compact-WY flat-tree QR and its application (csrc/batch_wy.cuh):
// factor a random m x c matrix in stacks of cr rows, apply Q to [I; 0], and compare on the host:
// ||A - Q R|| / ||A|| and ||Q^T Q - I||.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -o tools/wy_check tools/wy_check.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_2211_08770_b200/csrc/batch_wy.cuh"

using namespace ttb;

struct RowLoader {  // row-major m x c matrix in stacks of cr rows
  const double* A;
  int64_t m;
  int c, cr;
  __device__ int stacks() const { return (int)((m + cr - 1) / cr); }
  __device__ int crow(int q) const { return (int)(m - (int64_t)q * cr < cr ? m - (int64_t)q * cr : cr); }
  __device__ void load(wy::Smem& sm, int q, int w) const {
    const int lane = threadIdx.x & 31;
    wy::zero_cols(sm, w);
    for (int r = lane; r < crow(q); r += 32)
      for (int col = 8 * w; col < 8 * w + 8 && col < c; ++col)
        sm.st[col * wy::LD + wy::RR + r] = A[((int64_t)q * cr + r) * c + col];
    __syncwarp();
  }
};

__global__ void __launch_bounds__(wy::T, 1) factor_kernel(const double* A, int64_t m, int c, int cr, double* F, double* R) {
  extern __shared__ __align__(16) unsigned char raw[];
  wy::Smem& sm = *reinterpret_cast<wy::Smem*>(raw);
  RowLoader ld{A, m, c, cr};
  wy::factor_panel(sm, ld, c, F);
  for (int idx = threadIdx.x; idx < c * c; idx += wy::T) {
    const int row = idx / c, col = idx % c;
    R[idx] = row <= col ? sm.st[col * wy::LD + row] : 0.0;
  }
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
  struct Case { int64_t m; int c, cr; };
  std::vector<Case> cases = {{50, 8, 128}, {100, 12, 128}, {300, 24, 120}, {720, 24, 120}, {2500, 64, 100},
                             {2500, 50, 128}, {2048, 64, 128},  {825, 12, 128},
                             {480, 16, 128}, {396, 25, 120}, {270, 3, 126}, {90, 9, 128}, {270, 3, 128}, {64, 3, 64}};
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
    factor_kernel<<<1, wy::T, sizeof(wy::Smem)>>>(dA, m, c, cr, dF, dR);
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
    const double rel = std::sqrt(nres / na), orth = std::sqrt(north);
    const bool ok = e == cudaSuccess && rel < 1e-13 && orth < 1e-13;
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
    std::printf("m %5lld c %2d cr %3d: ||A-QR||/||A|| %.2e  ||Q^TQ-I|| %.2e  %s %s\n", (long long)m, c, cr, rel, orth,
                ok ? "OK" : "BAD", cudaGetErrorString(e));
    cudaFree(dA); cudaFree(dF); cudaFree(dR); cudaFree(dX); cudaFree(dQ);
  }
  return bad ? 1 : 0;
}
