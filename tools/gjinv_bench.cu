// Microbenchmark of the panel inverse k_gj_inv (hs_schur.cu) on one 32 x 32
// panel of a random diagonally-shifted matrix: mean kernel time over many
// launches and the inverse's residual.  Variants by -DGJ_EXP=n (timing only:
// 1 drops the reciprocal, 2 the pivot search) to see what a step is made of.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -I include \
//        -o tools/_bin/gjinv_bench tools/gjinv_bench.cu
#include "../paper_2209_10886_b200/csrc/hs_schur.cu"

#include <complex>
#include <random>

namespace hs {
// hs_zmma.cu is not linked here
bool zgemm_dmma(cudaStream_t, int, int, int, double2, const double2*, int, long long, const double2*, int, long long, double2,
                double2*, int, long long, int) {
  return false;
}
}  // namespace hs

int main() {
  using namespace hs;
  const int n = 256, nb = 32, j0 = 64;
  std::vector<double2> A((size_t)n * n);
  std::mt19937_64 rng(1);
  std::normal_distribution<double> nd;
  for (auto& v : A) v = make_double2(nd(rng), nd(rng));
  for (int i = 0; i < n; ++i) A[(size_t)i * n + i].x += 8.0;
  double2 *dA, *dP, *dB, *dC;
  int* dbad;
  const long long pstride = 32LL * n + 32 * 32;
  cudaMalloc(&dA, A.size() * sizeof(double2));
  cudaMalloc(&dP, pstride * sizeof(double2));
  cudaMalloc(&dB, pstride * sizeof(double2));
  cudaMalloc(&dC, pstride * sizeof(double2));
  cudaMalloc(&dbad, sizeof(int));
  cudaMemset(dbad, 0, sizeof(int));
  cudaMemcpy(dA, A.data(), A.size() * sizeof(double2), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 2000;
  for (int grid : {1, 9}) {
    for (int w = 0; w < 50; ++w) k_gj_inv<<<dim3(grid, 1), kGjThreads>>>(dA, 0, 0, n, j0, nb, dP, dB, dC, pstride, dbad);
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_gj_inv<<<dim3(grid, 1), kGjThreads>>>(dA, 0, 0, n, j0, nb, dP, dB, dC, pstride, dbad);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"grid\": %d, \"threads\": %d, \"us_per_launch\": %.3f, \"err\": \"%s\"}\n", grid, kGjThreads,
           1e3 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<double2> P(32 * 32);
  cudaMemcpy(P.data(), dP, P.size() * sizeof(double2), cudaMemcpyDeviceToHost);
  double worst = 0;
  for (int i = 0; i < 32; ++i)
    for (int j = 0; j < 32; ++j) {
      std::complex<double> s = 0;
      for (int k = 0; k < 32; ++k)
        s += std::complex<double>(P[i * 32 + k].x, P[i * 32 + k].y) *
             std::complex<double>(A[(size_t)(j0 + k) * n + j0 + j].x, A[(size_t)(j0 + k) * n + j0 + j].y);
      worst = std::max(worst, std::abs(s - (i == j ? 1.0 : 0.0)));
    }
  printf("{\"max_abs_PinvP_minus_I\": %.3e}\n", worst);
  return 0;
}
