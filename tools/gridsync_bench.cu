// Micro-benchmark: cost of one grid-wide barrier step on B200 (148 CTAs),
// cooperative-groups grid.sync vs a hand-rolled flag barrier, with and
// without the partial-sum publish/read that an Arnoldi step needs.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_sync(int iters, int mode, double* part, unsigned* bar, const double2* vec, long long vlen) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double tot;
  __shared__ double2 buf[2][1024];
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (mode >= 3) {
      // prefetch one element per thread of a rotating 2 MB vector (as k_mgs1 does)
      const long long e = ((long long)(it % 64) * gridDim.x * blockDim.x + blockIdx.x * blockDim.x + threadIdx.x) % vlen;
      const unsigned sa = (unsigned)__cvta_generic_to_shared(&buf[it & 1][threadIdx.x]);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(vec + e));
      asm volatile("cp.async.commit_group;");
      if (mode == 4) asm volatile("cp.async.wait_group 0;");
      acc += buf[(it + 1) & 1][threadIdx.x].x;
    }
    if (mode >= 1 && threadIdx.x == 0) part[(it & 1) * gridDim.x + blockIdx.x] = it + blockIdx.x;
    if (mode == 2) {
      // flag barrier: one atomic per CTA, spin on the generation counter
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        unsigned target = (unsigned)(it + 1) * gridDim.x;
        atomicAdd(bar, 1u);
        while (true) {
          unsigned v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar));
          if (v >= target) break;
        }
      }
      __syncthreads();
    } else {
      grid.sync();
    }
    if (mode >= 3) asm volatile("cp.async.wait_group 0;");
    if (mode >= 1 && threadIdx.x < 32) {
      double s = 0;
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        int q = threadIdx.x + 32 * u;
        v[u] = q < (int)gridDim.x ? __ldcg(part + (it & 1) * gridDim.x + q) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(~0u, s, o);
      if (threadIdx.x == 0) tot = s;
    }
    __syncthreads();
    acc += tot;
  }
  if (acc == -1) part[0] = acc;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* part;
  unsigned* bar;
  cudaMalloc(&part, 4096 * sizeof(double));
  cudaMalloc(&bar, sizeof(unsigned));
  long long vlen = 1 << 20;
  double2* vec;
  cudaMalloc(&vec, vlen * sizeof(double2));
  cudaMemset(vec, 0, vlen * sizeof(double2));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int bd : {128, 512, 864, 1024})
    for (int mode : {0, 1, 2, 3, 4}) {
      int iters = 2000;
      float best = 1e30f;
      for (int rep = 0; rep < 3; ++rep) {
        cudaMemset(bar, 0, sizeof(unsigned));
        void* args[] = {&iters, &mode, &part, &bar, &vec, &vlen};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_sync, nsm, bd, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("{\"block\": %d, \"mode\": \"%s\", \"us_per_step\": %.3f, \"err\": \"%s\"}\n", bd,
             mode == 0 ? "grid.sync" : mode == 1 ? "grid.sync+partials" : mode == 2 ? "flag+partials"
             : mode == 3 ? "grid.sync+partials+cp.async in flight" : "grid.sync+partials+cp.async waited",
             best * 1000.0 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
