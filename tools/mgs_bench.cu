// Arnoldi-kernel timing outside the profiler: random orthonormal-ish basis of
// L complex elements, one Arnoldi step at each k, CUDA events around each
// launch (caches as in a real solve: w just written, older v_j wherever they
// are).  Compares k_mgs + k_givens (grid) with k_mgs1 (fused Givens).
//   build: see tools/gpu_mgs_bench.sh;  run: ./tools/mgs_bench L KMAX
#include <cstdio>
#include <cstdlib>
#include <vector>

#define main allreduce_main
#include "allreduce_bench.cu"
#undef main
#include "hsb200.h"
#include "../paper_2209_10886_b200/csrc/hs_ctx.h"
#include "../paper_2209_10886_b200/csrc/hs_kernels.h"

using namespace hs;

__global__ void k_fill(double2* x, long long n, unsigned long long seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull ^ seed;
    z ^= z >> 31; z *= 0xBF58476D1CE4E5B9ull; z ^= z >> 29;
    x[i] = make_double2((double)(z & 0xffff) / 65536.0 - 0.5, (double)((z >> 16) & 0xffff) / 65536.0 - 0.5);
  }
}

int main(int argc, char** argv) {
  const long long L = argc > 1 ? atoll(argv[1]) : 499712;
  const int KMAX = argc > 2 ? atoi(argv[2]) : 100;
  hs_ctx* hc = nullptr;
  if (hs_create(&hc, 0, 4, 4, 32, 1.0 / 128, 80.0, 0.0, 80.0, 0, 1)) { printf("create failed\n"); return 1; }
  Ctx& c = *(Ctx*)hc;
  GmresDev G{};
  G.LR = L; G.R = 1; G.tol = 1e-300;
  const int maxit = KMAX + 1;
  cudaMalloc(&G.V, (size_t)(maxit + 1) * L * sizeof(double2));
  cudaMalloc(&G.H, (size_t)(maxit * (maxit + 3) / 2 + 2) * sizeof(double2));
  cudaMalloc(&G.cs, maxit * sizeof(double));
  cudaMalloc(&G.sn, maxit * sizeof(double2));
  cudaMalloc(&G.g, (maxit + 1) * sizeof(double2));
  cudaMalloc(&G.hist, (maxit + 1) * sizeof(double));
  cudaMalloc(&G.beta, sizeof(double));
  cudaMalloc(&G.wnorm0, sizeof(double));
  int* ints;
  cudaMalloc(&ints, 8 * sizeof(int));
  G.active = ints; G.iters = ints + 1; G.conv = ints + 2; G.brk = ints + 3; G.nactive = ints + 4;
  cudaMalloc(&G.partial, (size_t)2 * (4 * c.num_sms) * sizeof(double2));
  cudaMalloc(&G.y, maxit * sizeof(double2));
  double2* W;
  cudaMalloc(&W, L * sizeof(double2));
  k_fill<<<1024, 256, 0, c.stream>>>(G.V, (maxit + 1) * L, 7);
  k_fill<<<1024, 256, 0, c.stream>>>(W, L, 11);
  std::vector<double> h1 = {1.0};
  cudaMemcpyAsync(G.beta, h1.data(), sizeof(double), cudaMemcpyHostToDevice, c.stream);
  static int one[5] = {1, 0, 0, 0, 1};
  cudaMemcpyAsync(ints, one, 5 * sizeof(int), cudaMemcpyHostToDevice, c.stream);
  cudaStreamSynchronize(c.stream);
  int chunk = 0, m1chunk = 0, E = 0, bd = 0;
  const int grid = gmres_coop_grid(c, L, 1, &chunk);
  const int m1grid = gmres_mgs1_plan(c, L, 1, maxit, &m1chunk, &E, &bd);
  int ccchunk = 0, c1chunk = 0, c1E = 0, c1bd = 0;
  const int ccs = gmres_cluster_size(L, 1, &ccchunk);
  const int c1cs = gmres_mgs1c_plan(L, 1, maxit, &c1chunk, &c1E, &c1bd);
  std::vector<cudaEvent_t> ev(2 * (KMAX + 1));
  for (auto& e : ev) cudaEventCreate(&e);
  printf("{\"L\": %lld, \"grid\": %d, \"mgs1_grid\": %d, \"E\": %d, \"block\": %d}\n", L, grid, m1grid, E, bd);
  const char* names[] = {"k_mgs+k_givens", "k_mgs1", "k_mgs_cluster", "k_mgs1c"};
  for (int variant = 0; variant < 4; ++variant) {
    if ((variant == 1 && m1grid <= 0) || (variant == 2 && ccs <= 0) || (variant == 3 && c1cs <= 0)) continue;
    // all launches back to back (the GPU stays busy, clocks stay up), events read at the end
    for (int k = 0; k <= KMAX; ++k) {
      cudaMemcpyAsync(G.V + (long long)(k + 1) * L, W, L * sizeof(double2), cudaMemcpyDeviceToDevice, c.stream);
      cudaEventRecord(ev[2 * k], c.stream);
      cudaError_t e;
      if (variant == 0) { e = gmres_arnoldi(c, G, k, grid, chunk); if (!e) e = gmres_givens(c, G, k); }
      else if (variant == 1) e = gmres_arnoldi1(c, G, k, m1grid, m1chunk, E, bd);
      else if (variant == 2) e = gmres_arnoldi_cluster(c, G, k, ccs, ccchunk);
      else e = gmres_arnoldi1c(c, G, k, c1cs, c1chunk, c1E, c1bd);
      cudaEventRecord(ev[2 * k + 1], c.stream);
      if (e) { printf("launch error %s\n", cudaGetErrorString(e)); return 1; }
    }
    cudaStreamSynchronize(c.stream);
    double sum = 0, s10 = 0, s50 = 0;
    for (int k = 0; k <= KMAX; ++k) {
      float ms;
      cudaEventElapsedTime(&ms, ev[2 * k], ev[2 * k + 1]);
      sum += ms;
      if (k == 10) s10 = ms;
      if (k == 50) s50 = ms;
    }
    printf("{\"variant\": \"%s\", \"total_ms\": %.3f, \"k10_us\": %.1f, \"k50_us\": %.1f, \"per_j_us\": %.2f}\n",
           names[variant], sum, s10 * 1e3, s50 * 1e3, (s50 - s10) * 1e3 / 40);
  }
  {
    // the exchange micro-benchmark kernel (mode 1: grid.sync + component-major partials), same process/stream
    double *part, *out;
    unsigned long long* sl;
    cudaMalloc(&part, 2 * 32 * MAXG * sizeof(double));
    cudaMalloc(&out, MAXG * sizeof(double));
    cudaMalloc(&sl, (2 * 6 * MAXG + 16) * sizeof(unsigned long long));
    // after a k_mgs1 launch c.mgs1_slots exists: run the exchange kernel on that buffer too
    double* bufs[2] = {part, (double*)c.mgs1_slots};
    for (int bi = 0; bi < 2; ++bi) {
    part = bufs[bi];
    if (!part) continue;
    for (size_t smem : {(size_t)0}) {
      cudaFuncSetAttribute((const void*)k_ar, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      int iters = 2000, mode = 1;
      unsigned seq = 1;
      void* args[] = {&iters, &mode, &part, &sl, &seq, &out};
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      for (cudaStream_t st : {(cudaStream_t)0, c.stream}) {
        cudaEventRecord(a, st);
        cudaError_t e = cudaLaunchCooperativeKernel((void*)k_ar, c.num_sms, 256, args, smem, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("{\"exchange_bench\": \"grid.sync+SoA\", \"buffer\": \"%s\", \"smem\": %zu, \"stream\": \"%s\", \"us_per_step\": %.3f, \"err\": \"%s\"}\n",
               bi ? "mgs1_slots" : "own", smem, st ? "ctx" : "default", ms * 1e3 / iters, cudaGetErrorString(e));
      }
    }
    }
  }
  hs_destroy(hc);
  return 0;
}
