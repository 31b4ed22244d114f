// DMMA (mma.sync m8n8k4 f64) latency / throughput probe: grid = #SMs, W warps per CTA, each warp
// runs C independent accumulator chains for N steps.  Prints DMMA per clock per SM.
#include <cstdio>
#include <cuda_runtime.h>

template <int C>
__global__ void probe(int n, double* out, long long* clk) {
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  double c0[C], c1[C];
#pragma unroll
  for (int i = 0; i < C; ++i) { c0[i] = i; c1[i] = -i; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < C; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c0[i]), "+d"(c1[i]) : "d"(a), "d"(b));
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < C; ++i) s += c0[i] + c1[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int C>
void run(int warps, int sms, double* out, long long* clk) {
  const int n = 4096;
  probe<C><<<sms, warps * 32>>>(n, out, clk);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, clk, sizeof(h), cudaMemcpyDeviceToHost);
  const double dmma = (double)n * C * warps;
  printf("chains %2d warps %2d: %.1f cyc per chain step, %.3f DMMA/clk/SM\n", C, warps, (double)h / n, dmma / h);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  long long* clk;
  cudaMalloc(&out, sizeof(double) * sms * 1024);
  cudaMalloc(&clk, sizeof(long long) * sms);
  for (int w : {1, 2, 4, 8, 16}) {
    run<1>(w, sms, out, clk);
    run<4>(w, sms, out, clk);
    run<9>(w, sms, out, clk);
    run<16>(w, sms, out, clk);
  }
  return 0;
}
