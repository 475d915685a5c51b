// Micro-benchmark: one grid-wide sum of 3 doubles per step across 148 CTAs
// (the Arnoldi inner-product exchange), several exchange designs.  Prints
// microseconds per step.  Deterministic designs only (fixed summation order).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
constexpr int MAXG = 256;

__device__ __forceinline__ void st_rlx(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wsum3(double& a, double& b, double& c) {
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(~0u, a, o); b += __shfl_xor_sync(~0u, b, o); c += __shfl_xor_sync(~0u, c, o);
  }
}
// pack/unpack a double into two tagged words
__device__ __forceinline__ void put(unsigned long long* w0, unsigned long long* w1, double v, unsigned tag) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v), hi = (unsigned long long)tag << 32;
  st_rlx(w0, hi | (b & 0xffffffffull)); st_rlx(w1, hi | (b >> 32));
}

__global__ void k_ar(int iters, int mode, double* part, unsigned long long* slots, unsigned seq0, double* out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[32][3], red2[8][3], tot[3];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5, nb = gridDim.x;
  const int nwr = (nb + 31) / 32;
  double acc = 0;
  for (int it = 0; it < iters; ++it) {
    const unsigned tag = seq0 + it;
    double a = tid * 1e-3 + it, b = blockIdx.x * 1.0, c = 1.0;
    wsum3(a, b, c);
    if (lane == 0) { red[wid][0] = a; red[wid][1] = b; red[wid][2] = c; }
    __syncthreads();
    double A = 0, B = 0, C = 0;
    if (wid == 0) {
      A = lane < nw ? red[lane][0] : 0; B = lane < nw ? red[lane][1] : 0; C = lane < nw ? red[lane][2] : 0;
      wsum3(A, B, C);
    }
    double* P = part + (it & 1) * 3 * MAXG;
    unsigned long long* S = slots + (size_t)(it & 1) * 6 * MAXG;
    if (mode == 0 || mode == 1) {  // grid.sync; 0: AoS strided reads, 1: SoA coalesced reads
      if (wid == 0 && lane == 0) {
        if (mode == 0) { P[blockIdx.x * 3] = A; P[blockIdx.x * 3 + 1] = B; P[blockIdx.x * 3 + 2] = C; }
        else { P[blockIdx.x] = A; P[MAXG + blockIdx.x] = B; P[2 * MAXG + blockIdx.x] = C; }
      }
      grid.sync();
      if (wid == 0) {
        double x[8][3];
        for (int u = 0; u < 8; ++u) {
          int q = lane + 32 * u;
          for (int m = 0; m < 3; ++m)
            x[u][m] = q < nb ? __ldcg(mode == 0 ? P + q * 3 + m : P + m * MAXG + q) : 0.0;
        }
        A = B = C = 0;
        for (int u = 0; u < 8; ++u) { A += x[u][0]; B += x[u][1]; C += x[u][2]; }
        wsum3(A, B, C);
        if (lane == 0) { tot[0] = A; tot[1] = B; tot[2] = C; }
      }
      __syncthreads();
    } else if (mode == 8 || mode == 9) {  // own counter barrier (8: one counter; 9: counter per 32 B apart, read by all)
      if (wid == 0 && lane == 0) { P[blockIdx.x] = A; P[MAXG + blockIdx.x] = B; P[2 * MAXG + blockIdx.x] = C; }
      __syncthreads();
      if (tid == 0) {
        unsigned* bar = (unsigned*)(slots + 2 * 6 * MAXG + 16 - 4);
        __threadfence();
        atomicAdd(bar, 1u);
        const unsigned target = (unsigned)(it + 1) * nb;
        unsigned v;
        do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory"); } while (v < target);
      }
      __syncthreads();
      if (wid == 0) {
        double x[8][3];
        for (int u = 0; u < 8; ++u) {
          int q = lane + 32 * u;
          for (int m = 0; m < 3; ++m) x[u][m] = q < nb ? __ldcg(P + m * MAXG + q) : 0.0;
        }
        A = B = C = 0;
        for (int u = 0; u < 8; ++u) { A += x[u][0]; B += x[u][1]; C += x[u][2]; }
        wsum3(A, B, C);
        if (lane == 0) { tot[0] = A; tot[1] = B; tot[2] = C; }
      }
      __syncthreads();
    } else if (mode == 7) {  // SoA partials indexed by SM id (lines written by neighbouring SMs)
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      if (wid == 0 && lane == 0) { P[smid] = A; P[MAXG + smid] = B; P[2 * MAXG + smid] = C; }
      grid.sync();
      if (wid == 0) {
        double x[8][3];
        for (int u = 0; u < 8; ++u) {
          int q = lane + 32 * u;
          for (int m = 0; m < 3; ++m) x[u][m] = q < nb ? __ldcg(P + m * MAXG + q) : 0.0;
        }
        A = B = C = 0;
        for (int u = 0; u < 8; ++u) { A += x[u][0]; B += x[u][1]; C += x[u][2]; }
        wsum3(A, B, C);
        if (lane == 0) { tot[0] = A; tot[1] = B; tot[2] = C; }
      }
      __syncthreads();
    } else if (mode >= 4) {  // 4: {a,b} double2 + c; 5: one 128-B line per CTA; 6: {a,b} only
      double2* P2 = (double2*)(part + (size_t)(it & 1) * 32 * MAXG);
      double* P3 = part + (size_t)(it & 1) * 32 * MAXG + 2 * MAXG;
      double* PL = part + (size_t)(it & 1) * 16 * MAXG;
      if (wid == 0 && lane == 0) {
        if (mode == 5) { PL[blockIdx.x * 16] = A; PL[blockIdx.x * 16 + 1] = B; PL[blockIdx.x * 16 + 2] = C; }
        else { P2[blockIdx.x] = make_double2(A, B); if (mode == 4) P3[blockIdx.x] = C; }
      }
      grid.sync();
      if (wid == 0) {
        double x[8][3];
        for (int u = 0; u < 8; ++u) {
          int q = lane + 32 * u;
          if (q < nb) {
            if (mode == 5) { x[u][0] = __ldcg(PL + q * 16); x[u][1] = __ldcg(PL + q * 16 + 1); x[u][2] = __ldcg(PL + q * 16 + 2); }
            else { double2 v = __ldcg(P2 + q); x[u][0] = v.x; x[u][1] = v.y; x[u][2] = mode == 4 ? __ldcg(P3 + q) : 0.0; }
          } else x[u][0] = x[u][1] = x[u][2] = 0.0;
        }
        A = B = C = 0;
        for (int u = 0; u < 8; ++u) { A += x[u][0]; B += x[u][1]; C += x[u][2]; }
        wsum3(A, B, C);
        if (lane == 0) { tot[0] = A; tot[1] = B; tot[2] = C; }
      }
      __syncthreads();
    } else if (mode == 2) {  // tagged words, every CTA polls all (threads t < nb, one slot each)
      if (wid == 0 && lane == 0) {
        put(S + 0 * MAXG + blockIdx.x, S + 1 * MAXG + blockIdx.x, A, tag);
        put(S + 2 * MAXG + blockIdx.x, S + 3 * MAXG + blockIdx.x, B, tag);
        put(S + 4 * MAXG + blockIdx.x, S + 5 * MAXG + blockIdx.x, C, tag);
      }
      if (wid < nwr) {
        double x[3] = {0, 0, 0};
        if (tid < nb) {
          unsigned long long w[6];
          for (;;) {
            for (int m = 0; m < 6; ++m) w[m] = ld_rlx(S + m * MAXG + tid);
            bool ok = true;
            for (int m = 0; m < 6; ++m) ok &= (unsigned)(w[m] >> 32) == tag;
            if (ok) break;
          }
          for (int m = 0; m < 3; ++m) x[m] = __longlong_as_double((long long)((w[2 * m + 1] << 32) | (w[2 * m] & 0xffffffffull)));
        }
        wsum3(x[0], x[1], x[2]);
        if (lane == 0) { red2[wid][0] = x[0]; red2[wid][1] = x[1]; red2[wid][2] = x[2]; }
      }
      __syncthreads();
      if (tid == 0) { tot[0] = tot[1] = tot[2] = 0; for (int q = 0; q < nwr; ++q) for (int m = 0; m < 3; ++m) tot[m] += red2[q][m]; }
      __syncthreads();
    } else {  // mode 3: tagged words, CTA 0 collects and publishes the total, others poll the total
      if (wid == 0 && lane == 0) {
        put(S + 0 * MAXG + blockIdx.x, S + 1 * MAXG + blockIdx.x, A, tag);
        put(S + 2 * MAXG + blockIdx.x, S + 3 * MAXG + blockIdx.x, B, tag);
        put(S + 4 * MAXG + blockIdx.x, S + 5 * MAXG + blockIdx.x, C, tag);
      }
      unsigned long long* T = slots + (size_t)2 * 6 * MAXG + (it & 1) * 8;  // total: 6 words
      if (blockIdx.x == 0) {
        if (wid < nwr) {
          double x[3] = {0, 0, 0};
          if (tid < nb) {
            unsigned long long w[6];
            for (;;) {
              for (int m = 0; m < 6; ++m) w[m] = ld_rlx(S + m * MAXG + tid);
              bool ok = true;
              for (int m = 0; m < 6; ++m) ok &= (unsigned)(w[m] >> 32) == tag;
              if (ok) break;
            }
            for (int m = 0; m < 3; ++m) x[m] = __longlong_as_double((long long)((w[2 * m + 1] << 32) | (w[2 * m] & 0xffffffffull)));
          }
          wsum3(x[0], x[1], x[2]);
          if (lane == 0) { red2[wid][0] = x[0]; red2[wid][1] = x[1]; red2[wid][2] = x[2]; }
        }
        __syncthreads();
        if (tid == 0) {
          double t[3] = {0, 0, 0};
          for (int q = 0; q < nwr; ++q) for (int m = 0; m < 3; ++m) t[m] += red2[q][m];
          for (int m = 0; m < 3; ++m) { tot[m] = t[m]; put(T + 2 * m, T + 2 * m + 1, t[m], tag); }
        }
        __syncthreads();
      } else {
        if (tid < 6) {
          unsigned long long w;
          do { w = ld_rlx(T + tid); } while ((unsigned)(w >> 32) != tag);
          ((unsigned long long*)red2)[tid] = w;
        }
        __syncthreads();
        if (tid == 0) {
          unsigned long long* w = (unsigned long long*)red2;
          for (int m = 0; m < 3; ++m) tot[m] = __longlong_as_double((long long)((w[2 * m + 1] << 32) | (w[2 * m] & 0xffffffffull)));
        }
        __syncthreads();
      }
    }
    acc += tot[0];
  }
  if (tid == 0) out[blockIdx.x] = acc;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double *part, *out;
  unsigned long long* slots;
  cudaMalloc(&part, 2 * 32 * MAXG * sizeof(double));
  cudaMalloc(&out, MAXG * sizeof(double));
  cudaMalloc(&slots, (2 * 6 * MAXG + 16) * sizeof(unsigned long long));
  cudaMemset(slots, 0, (2 * 6 * MAXG + 16) * sizeof(unsigned long long));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  unsigned seq = 1;
  const char* names[] = {"grid.sync + AoS strided", "grid.sync + SoA coalesced", "tagged words, all poll all",
                         "tagged words, CTA 0 collects + broadcasts", "grid.sync + double2{a,b} + c",
                         "grid.sync + one 128B line per CTA", "grid.sync + double2{a,b} only", "grid.sync + SoA by smid", "own counter barrier + SoA"};
  for (int bd : {256})
    for (int mode : {1, 1, 1, 1, 1, 8, 8, 8, 8, 8, 8, 8, 8}) {
      int iters = 2000;
      float best = 1e30f;
      for (int rep = 0; rep < 1; ++rep) {
        cudaMemset(slots, 0, (2 * 6 * MAXG + 16) * sizeof(unsigned long long));
        void* args[] = {&iters, &mode, &part, &slots, &seq, &out};
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_ar, nsm, bd, args, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        seq += iters;
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
      }
      printf("{\"block\": %d, \"design\": \"%s\", \"us_per_step\": %.3f, \"err\": \"%s\"}\n", bd, names[mode],
             best * 1000.0 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
