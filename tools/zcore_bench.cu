// Micro-benchmark of complex128 DMMA contraction cores (the k_zmma main loop
// redesign): a CTA tile of 32 map rows x BN columns, K streamed in chunks of KC
// through an S-stage ring filled by a producer warp with per-row bulk copies
// (cp.async.bulk + mbarrier complete_tx) into padded shared rows (conflict-free
// 128-bit fragment loads), consumer warps owning TM x TN 8x8 DMMA tiles over
// the whole chunk (no intra-CTA K split), 3M complex product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/zcore_bench tools/zcore_bench.cu
// Prints one JSON line per variant: fraction of the measured DMMA peak.
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("{\"error\":\"%s\",\"line\":%d}\n", cudaGetErrorString(e_), __LINE__); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  unsigned ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int BN, int TM, int TN, int KC, int S, int AMODE = 0, bool NMAJ = false>
struct Cfg {
  static constexpr int WM = 32 / (8 * TM), WN = BN / (8 * TN), NWC = WM * WN;
  // AMODE 0: one bulk copy per k row into padded rows (2k + m (mod 8) distinct in a
  // 128-bit phase); AMODE 1: the whole 32 x 32 chunk as ONE 16 KB copy, unpadded
  static constexpr int SA = AMODE == 0 ? 32 + 2 : 32;
  static constexpr int SB = NMAJ ? KC + 4 : BN + 2;
  static constexpr int BROWS = NMAJ ? BN : KC;
  static constexpr int STAGE = KC * SA + BROWS * SB;
  static constexpr size_t SMEM = sizeof(double2) * S * STAGE;
};

// tasks t = blockIdx.x, blockIdx.x + gridDim.x, ...: strip (t % nstrips) of A
// ([K][32] per strip) times B panel (t % nb) ([K][BN]), output tile t.
template <int BN, int TM, int TN, int KC, int S, int AMODE, bool NMAJ>
__global__ void __launch_bounds__((Cfg<BN, TM, TN, KC, S, AMODE, NMAJ>::NWC + 1) * 32)
    k_core(const double2* __restrict__ A, const double2* __restrict__ B, double2* C, int K, int ntasks, int nstrips,
           int nb) {
  using F = Cfg<BN, TM, TN, KC, S, AMODE, NMAJ>;
  extern __shared__ __align__(128) double2 sm[];
  __shared__ __align__(8) unsigned long long full[S], empty[S];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], F::NWC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int nk = K / KC;
  if (warp == F::NWC) {  // producer
    long long g = 0;
    for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
      const double2* As = A + (long long)(t % nstrips) * K * 32;
      const double2* Bs = B + (long long)(t % nb) * K * BN;
      for (int kc = 0; kc < nk; ++kc, ++g) {
        const int st = (int)(g % S);
        mbar_wait(&empty[st], (unsigned)((g / S) & 1) ^ 1);
        if (lane == 0) mbar_expect_tx(&full[st], (unsigned)(KC * (32 + BN) * sizeof(double2)));
        __syncwarp();
        double2* sa = sm + (size_t)st * F::STAGE;
        double2* sb = sa + KC * F::SA;
        if (AMODE == 1) {
          if (lane == 0) bulk_g2s(sa, As + (long long)kc * KC * 32, KC * 32 * sizeof(double2), &full[st]);
        } else {
          for (int r = lane; r < KC; r += 32)
            bulk_g2s(sa + r * F::SA, As + (long long)(kc * KC + r) * 32, 32 * sizeof(double2), &full[st]);
        }
        if (NMAJ) {  // column j: KC consecutive positions of "subdomain" column j
          for (int j = lane; j < BN; j += 32)
            bulk_g2s(sb + j * F::SB, Bs + (long long)j * K + kc * KC, KC * sizeof(double2), &full[st]);
        } else {
          for (int r = lane; r < KC; r += 32)
            bulk_g2s(sb + r * F::SB, Bs + (long long)(kc * KC + r) * BN, BN * sizeof(double2), &full[st]);
        }
      }
    }
    return;
  }
  const int wm = warp / F::WN, wn = warp % F::WN;
  const int gid = lane >> 2, tig = lane & 3;
  long long g = 0;
  for (int t = blockIdx.x; t < ntasks; t += gridDim.x) {
    double cr[TM][TN][2], ci[TM][TN][2], p3[TM][TN][2];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b)
#pragma unroll
        for (int c = 0; c < 2; ++c) cr[a][b][c] = ci[a][b][c] = p3[a][b][c] = 0.0;
    for (int kc = 0; kc < nk; ++kc, ++g) {
      const int st = (int)(g % S);
      mbar_wait(&full[st], (unsigned)((g / S) & 1));
      const double2* sa = sm + (size_t)st * F::STAGE;
      const double2* sb = sa + KC * F::SA;
#pragma unroll
      for (int k4 = 0; k4 < KC; k4 += 4) {
        double2 a[TM], b[TN];
#pragma unroll
        for (int mt = 0; mt < TM; ++mt) a[mt] = sa[(k4 + tig) * F::SA + (wm * TM + mt) * 8 + gid];
#pragma unroll
        for (int nt = 0; nt < TN; ++nt)
          b[nt] = NMAJ ? sb[((wn * TN + nt) * 8 + gid) * F::SB + k4 + tig] : sb[(k4 + tig) * F::SB + (wn * TN + nt) * 8 + gid];
        double s_b[TN];
#pragma unroll
        for (int nt = 0; nt < TN; ++nt) s_b[nt] = b[nt].x + b[nt].y;
#pragma unroll
        for (int mt = 0; mt < TM; ++mt) {
          const double s_a = a[mt].x + a[mt].y;
#pragma unroll
          for (int nt = 0; nt < TN; ++nt) dmma(cr[mt][nt][0], cr[mt][nt][1], a[mt].x, b[nt].x);
#pragma unroll
          for (int nt = 0; nt < TN; ++nt) dmma(ci[mt][nt][0], ci[mt][nt][1], a[mt].y, b[nt].y);
#pragma unroll
          for (int nt = 0; nt < TN; ++nt) dmma(p3[mt][nt][0], p3[mt][nt][1], s_a, s_b[nt]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    double2* Ct = C + (long long)t * 32 * BN;
#pragma unroll
    for (int mt = 0; mt < TM; ++mt)
#pragma unroll
      for (int nt = 0; nt < TN; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = (wm * TM + mt) * 8 + gid, col = (wn * TN + nt) * 8 + 2 * tig + h;
          const double s1 = cr[mt][nt][h], s2 = ci[mt][nt][h];
          Ct[row * BN + col] = make_double2(s1 - s2, p3[mt][nt][h] - s1 - s2);
        }
  }
}

template <int BN, int TM, int TN, int KC, int S, int AMODE = 0, bool NMAJ = false>
int run(const char* name, const double2* A, const double2* B, double2* C, int K, int nstrips, int nb, int sms,
        int ctas_per_sm, int tasks_per_cta, cudaEvent_t e0, cudaEvent_t e1) {
  using F = Cfg<BN, TM, TN, KC, S, AMODE, NMAJ>;
  auto kern = k_core<BN, TM, TN, KC, S, AMODE, NMAJ>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F::SMEM));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, (F::NWC + 1) * 32, F::SMEM));
  if (occ < ctas_per_sm) {
    printf("{\"variant\":\"%s\",\"skip\":\"occupancy %d < %d\"}\n", name, occ, ctas_per_sm);
    return 0;
  }
  const int grid = sms * ctas_per_sm;
  const int ntasks = grid * tasks_per_cta;
  kern<<<grid, (F::NWC + 1) * 32, F::SMEM>>>(A, B, C, K, ntasks, nstrips, nb);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  const int reps = 10;
  CK(cudaEventRecord(e0));
  for (int i = 0; i < reps; ++i) kern<<<grid, (F::NWC + 1) * 32, F::SMEM>>>(A, B, C, K, ntasks, nstrips, nb);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  const double dmma_flops = (double)reps * ntasks * 32.0 * BN * K * 3 * 2;  // 3M: 3 real MACs per complex MAC
  const double tf = dmma_flops / (ms * 1e-3) / 1e12;
  printf(
      "{\"variant\":\"%s\",\"BN\":%d,\"TM\":%d,\"TN\":%d,\"KC\":%d,\"S\":%d,\"warps\":%d,\"ctas_per_sm\":%d,\"K\":%d,"
      "\"tasks_per_cta\":%d,\"us_per_launch\":%.2f,\"dmma_tflops\":%.2f,\"frac_dmma_peak\":%.3f}\n",
      name, BN, TM, TN, KC, S, F::NWC, ctas_per_sm, K, tasks_per_cta, ms * 1e3 / reps, tf, tf / 37.17);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int Kmax = 1024, nstrips = 64, nb = 64;
  double2 *A, *B, *C;
  CK(cudaMalloc(&A, sizeof(double2) * (size_t)nstrips * Kmax * 32));
  CK(cudaMalloc(&B, sizeof(double2) * (size_t)nb * Kmax * 64));
  CK(cudaMalloc(&C, sizeof(double2) * (size_t)sms * 2 * 64 * 32 * 64));
  {
    std::vector<double2> h((size_t)nb * Kmax * 64);
    for (size_t i = 0; i < h.size(); ++i) h[i] = make_double2(1e-3 * (i % 97), -1e-3 * (i % 89));
    CK(cudaMemcpy(B, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(A, h.data(), sizeof(double2) * (size_t)nstrips * Kmax * 32, cudaMemcpyHostToDevice));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int K : {256, 1024}) {
    const int tpc = K == 256 ? 16 : 4;
    run<64, 2, 2, 32, 4>("bn64_w8_s4", A, B, C, K, nstrips, nb, sms, 1, tpc, e0, e1);
    run<64, 2, 2, 32, 3>("bn64_w8_s3", A, B, C, K, nstrips, nb, sms, 1, tpc, e0, e1);
    run<64, 2, 2, 32, 4, 1>("bn64_w8_s4_a1copy", A, B, C, K, nstrips, nb, sms, 1, tpc, e0, e1);
    run<64, 2, 2, 32, 3, 0, true>("bn64_w8_s3_nmaj", A, B, C, K, nstrips, nb, sms, 1, tpc, e0, e1);
    run<64, 2, 2, 32, 3, 1, true>("bn64_w8_s3_nmaj_a1copy", A, B, C, K, nstrips, nb, sms, 1, tpc, e0, e1);
    run<32, 1, 2, 32, 3>("bn32_w8_s3_2cta", A, B, C, K, nstrips, nb, sms, 2, tpc, e0, e1);
    run<32, 1, 2, 32, 3>("bn32_w8_s3_1cta", A, B, C, K, nstrips, nb, sms, 1, tpc, e0, e1);
    run<32, 1, 2, 32, 3, 0, true>("bn32_w8_s3_nmaj_2cta", A, B, C, K, nstrips, nb, sms, 2, tpc, e0, e1);
    run<32, 1, 2, 32, 3, 1, true>("bn32_w8_s3_nmaj_a1_2cta", A, B, C, K, nstrips, nb, sms, 2, tpc, e0, e1);
  }
  printf("{\"status\":\"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
