// FP64 peak microbenchmark for B200 (sm_100a): FFMA (DFMA) and DMMA (mma.sync f64).
// MEASURED_PEAKS.json carries no FP64 entry; the roofline denominator for every
// hot-path kernel of this repo is the max of the two sustained rates measured here.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int ILP>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m8n8k4_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-12, b = 1.0 - threadIdx.x * 1e-12;
  double c[4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m16n8k4_kernel(double* out, int iters) {
  double a0 = 1.0 + threadIdx.x * 1e-12, a1 = a0 * 0.5, b = 1.0 - threadIdx.x * 1e-12;
  double c[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3]) : "d"(a0), "d"(a1), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_m16n8k16_kernel(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + (threadIdx.x + i) * 1e-12;
#pragma unroll
  for (int i = 0; i < 4; ++i) b[i] = 1.0 - (threadIdx.x + i) * 1e-12;
  double c[2][4];
#pragma unroll
  for (int i = 0; i < 2; ++i) for (int j = 0; j < 4; ++j) c[i][j] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]), "+d"(c[i][2]), "+d"(c[i][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 2; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", p.name, sms);
  double* out;
  CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // DFMA
  {
    const int ILP = 8, threads = 256, iters = 20000;
    int blocks = sms * 8;
    for (int rep = 0; rep < 2; ++rep) dfma_kernel<ILP><<<blocks, threads>>>(out, iters / 10, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      dfma_kernel<ILP><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double tf = 2.0 * ILP * (double)iters * threads * blocks / (ms * 1e-3) / 1e12;
      if (tf > best) best = tf;
    }
    printf(", \"dfma_tflops\": %.3f", best);
  }
  // DMMA variants
  {
    const int threads = 256, iters = 20000;
    int blocks = sms * 8;
    double best = 0;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      dmma_m8n8k4_kernel<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 8 * 4 * 4.0 * iters * (threads / 32) * blocks;
      double tf = flops / (ms * 1e-3) / 1e12;
      if (rep > 0 && tf > best) best = tf;
    }
    printf(", \"dmma_m8n8k4_tflops\": %.3f", best);
    best = 0;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      dmma_m16n8k4_kernel<<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * 8 * 4 * 4.0 * iters * (threads / 32) * blocks;
      double tf = flops / (ms * 1e-3) / 1e12;
      if (rep > 0 && tf > best) best = tf;
    }
    printf(", \"dmma_m16n8k4_tflops\": %.3f", best);
    best = 0;
    for (int rep = 0; rep < 6; ++rep) {
      cudaEventRecord(e0);
      dmma_m16n8k16_kernel<<<blocks, threads>>>(out, iters / 2);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * 8 * 16 * 2.0 * (iters / 2) * (threads / 32) * blocks;
      double tf = flops / (ms * 1e-3) / 1e12;
      if (rep > 0 && tf > best) best = tf;
    }
    printf(", \"dmma_m16n8k16_tflops\": %.3f", best);
  }
  CK(cudaGetLastError());
  printf("}\n");
  return 0;
}
