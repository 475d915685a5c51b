// FP64 peak microbenchmark for the roofline denominator of the FP64-bound
// kernels (MEASURED_PEAKS.json has no FP64 entry): DMMA (mma.sync m8n8k4 f64,
// the FP64 tensor path; tcgen05 has no f64 kind) and plain DFMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-7;
  double c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int blocksPerSM : {1, 2, 4}) {
    for (int threads : {128, 256, 512}) {
      dim3 grid(sms * blocksPerSM);
      k_dmma<<<grid, threads>>>(d, 100);
      cudaEventRecord(e0);
      k_dmma<<<grid, threads>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double warps = (double)grid.x * threads / 32;
      double flops = warps * iters * 8 * (8.0 * 8 * 4 * 2);
      printf("{\"kind\":\"dmma_m8n8k4\",\"blocks_per_sm\":%d,\"threads\":%d,\"tflops\":%.2f}\n", blocksPerSM, threads,
             flops / ms / 1e9);
      k_dfma<<<grid, threads>>>(d, 100);
      cudaEventRecord(e0);
      k_dfma<<<grid, threads>>>(d, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = (double)grid.x * threads * iters * 8 * 2;
      printf("{\"kind\":\"dfma\",\"blocks_per_sm\":%d,\"threads\":%d,\"tflops\":%.2f}\n", blocksPerSM, threads,
             flops / ms / 1e9);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("{\"status\":\"%s\"}\n", cudaGetErrorString(err));
  return 0;
}
