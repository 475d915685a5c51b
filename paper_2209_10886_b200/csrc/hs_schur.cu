// One-shot subdomain factorisation on the GPU: interface Schur maps.
//
// Replaces LocalOperator.__init__ + splu (discretization.py:126-174) and the
// per-apply solve_local + extract_outgoing_trace (discretization.py:264-312)
// by the dense map
//     T = -(s/d) I - (2 tau / (h^3 d^2)) E^T A^{-1} E
// (SURVEY.md §7), computed once per DISTINCT operator: the matrix depends
// only on (n, h, kappa, tau, Dirichlet cells) (discretization.py:221-256), so
// every subdomain without scatterer cells shares one operator.
//
// A is taken row-block by row-block (grid rows y = k, n cells each): it is
// block tridiagonal, A = tridiag(C_{k-1}, D_k, C_k) with diagonal couplings
// C_k = -1/h^2 (zero at Dirichlet cells, which are eliminated: identity rows
// AND columns, their known value moved to the right-hand side).  Block
// elimination without inter-block pivoting (accurate for these operators,
// SURVEY.md §7 hard part 1) in the TWISTED order: the rows above the middle
// row m = n/2 are eliminated downwards and the rows below it upwards -- two
// independent chains of half the length, run concurrently on two streams (the
// panel chain of a row is latency-bound and leaves the GPU mostly idle) -- and
// row m couples them:
//     S_k = D_k - C_{k-1} X_{k-1} C_{k-1}                        (k < m)
//     S_k = D_k - C_k X_{k+1} C_k                                (k > m)
//     S_m = D_m - C_{m-1} X_{m-1} C_{m-1} - C_m X_{m+1} C_m,     X_k = S_k^{-1}
// X_k by blocked in-place Gauss-Jordan (32-wide panels, partial pivoting
// inside the diagonal panel block).  Then for the R right-hand sides (one unit
// vector per boundary cell, plus lifting data), "prev" being the rows already
// eliminated next to k (k-1 above m, k+1 below, both at m):
//     Y_k = X_k (F_k - sum_prev C Y_prev)                         (towards m)
//     U_m = Y_m,  U_k = Y_k - X_k C U_next                        (away from m)
// and the boundary rows of U give E^T A^{-1} E.  All dense work is batched
// over the distinct operators; the products are complex GEMMs.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "hs_common.cuh"
#include "hs_kernels.h"

namespace hs {

struct OpParams {
  int n;
  double ih2;      // 1/h^2
  double dre, dim; // diagonal base: (4/h^2 - kappa^2) - (1/h^2)(s/d) per ghost: dre + g * (gre, gim)
  double gre, gim; // -(1/h^2)(s/d)
};

__device__ __forceinline__ bool dmask(const uint8_t* m, int n, int k, int x) { return m[k * n + x] != 0; }

// Programmatic dependent launch for the panel chain (k_formS -> k_gj_inv ->
// k_gj_update -> k_gj_inv ...): every kernel lets its successor launch at once
// and waits for its predecessor's completion before touching memory, so the
// successor's launch latency hides behind the running kernel.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() {
  pdl_trigger();
  pdl_wait();
}
template <class... KArgs, class... Args>
static void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  static const bool pdl = !(getenv("HS_FACTOR_PDL") && atoi(getenv("HS_FACTOR_PDL")) == 0);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, KArgs(args)...);
}

// coupling between row k and k+1 at column x
__device__ __forceinline__ double coupling(const uint8_t* m, int n, int k, int x, double ih2) {
  return (dmask(m, n, k, x) || dmask(m, n, k + 1, x)) ? 0.0 : -ih2;
}

// coupling between rows k and kp (|k - kp| = 1) at column x
__device__ __forceinline__ double coupling2(const uint8_t* m, int n, int k, int kp, int x, double ih2) {
  return coupling(m, n, k < kp ? k : kp, x, ih2);
}

// S_k = D_k - sum over the eliminated neighbour rows kp of C X_kp C, written
// into X_k (kp1, kp2: neighbour rows or -1).   grid (n, ncls), block 128
__global__ void k_formS(double2* X, long long xstride, const uint8_t* masks, OpParams P, int k, int kp1, int kp2) {
  pdl_enter();
  const int n = P.n;
  const int i = blockIdx.x;
  const int c = blockIdx.y;
  const uint8_t* m = masks + (long long)c * n * n;
  double2* Xk = X + c * xstride + (long long)k * n * n;
  const int kp[2] = {kp1, kp2};
  const double2* Xp[2];
  double ci[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    Xp[q] = kp[q] >= 0 ? X + c * xstride + (long long)kp[q] * n * n : nullptr;
    ci[q] = kp[q] >= 0 ? coupling2(m, n, k, kp[q], i, P.ih2) : 0.0;
  }
  const bool di = dmask(m, n, k, i);
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double2 v = make_double2(0, 0);
    const bool dj = dmask(m, n, k, j);
    if (i == j) {
      if (di) v = make_double2(1, 0);
      else {
        double g = (i == 0) + (i == n - 1) + (k == 0) + (k == n - 1);
        v = make_double2(P.dre + g * P.gre, g * P.gim);
      }
    } else if ((j == i + 1 || j == i - 1) && !di && !dj) {
      v = make_double2(-P.ih2, 0);
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (ci[q] == 0.0) continue;
      const double cj = coupling2(m, n, k, kp[q], j, P.ih2);
      if (cj != 0.0) {
        const double2 xv = Xp[q][(long long)i * n + j];
        v.x -= ci[q] * xv.x * cj;
        v.y -= ci[q] * xv.y * cj;
      }
    }
    Xk[(long long)i * n + j] = v;
  }
}

// panel inverse: columns per warp and threads (32 columns, lane = row)
#ifndef GJ_CW
#define GJ_CW 2
#endif
constexpr int kGjCW = GJ_CW, kGjThreads = 32 / kGjCW * 32;

// Panel step of blocked Gauss-Jordan on A = X_k (n x n, in place), panel
// columns J = [j0, j0+nb), in two kernels:
//   k_gj_inv:    CTA 0: P^{-1} of P = A[J,J] by Gauss-Jordan with partial
//                pivoting (max |re| + |im|, ties to the lower row) -> Pinv;
//                the other CTAs copy the panels A[J, :] and A[:, J];
//   k_gj_update: each 32 x 32 tile forms its row-panel tile P^{-1} A[J, cols]
//                and applies the trailing update.
// k_gj_inv keeps P in registers (in place: see the kernel): warp w owns kGjCW
// columns, lane = row.  The warp owning column p finds the pivot and
// publishes the column and the pivot's inverse (double-buffered by step
// parity); every warp then scales the pivot row and eliminates its columns
// with warp shuffles, one barrier per step (the shared-memory form had five
// and took 57 us per panel, the augmented [P | I] register form 23, this one
// ~16).
// grid (1 + 8 copy CTAs, ncls), block kGjThreads
__global__ void __launch_bounds__(kGjThreads) k_gj_inv(const double2* X, long long xstride, int k, int n, int j0,
                                                int nb, double2* Pinv, double2* Bp, double2* Cp,
                                                long long pstride, int* bad) {
  __shared__ double2 gj_f[2][32];
  __shared__ double2 gj_inv[2];
  __shared__ int gj_piv[2], gj_pos[2];
  // the successor (k_gj_update: a CTA per tile, 68 KB of shared memory each) is
  // let in only after the pivot loop: launched at entry it would sit on the
  // SMs for the whole panel inverse and starve the forward solves' GEMMs
  pdl_wait();
  const int c = blockIdx.y;
  const double2* A = X + c * xstride + (long long)k * n * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (blockIdx.x > 0) {
    // the other CTAs copy the row panel Bp = A[J, :] and the column panel
    // Cp = A[:, J] before the update overwrites A
    const int nc = gridDim.x - 1, b = blockIdx.x - 1;
    double2* B = Bp + c * pstride;
    double2* Cpp = Cp + c * pstride;
    for (int i = b * kGjThreads + tid; i < nb * n; i += nc * kGjThreads) {
      const int t = i / n, col = i % n;
      B[(long long)t * n + col] = A[(long long)(j0 + t) * n + col];
    }
    for (int i = b * kGjThreads + tid; i < n * nb; i += nc * kGjThreads) {
      const int r = i / nb, t = i % nb;
      Cpp[(long long)r * 32 + t] = A[(long long)r * n + j0 + t];
    }
    return;
  }
  // In-place Gauss-Jordan: warp w owns columns [CW w, CW w + CW) of P, lane =
  // row.  The identity column that the augmented form [P | I] would bring in at
  // step p (the pivot row's) takes the place of column p, which that step turns
  // into a unit vector.  A step is a dependent chain (read the published
  // pivot -> update the next pivot column -> reciprocal and search -> publish
  // -> barrier) of ~470 ns whatever the columns per warp (tools/gjinv_bench.cu:
  // 1, 2, 4, 8 columns within 10 %; 2 is the in-situ best by a little).
  // perm[u]: which column of P^{-1} the register column holds at the end.
  constexpr int CW = kGjCW;
  double2 a[CW];
  int perm[CW];
#pragma unroll
  for (int u = 0; u < CW; ++u) {
    const int q = warp * CW + u;
    double2 v = make_double2(0, 0);
    if (lane < nb && q < nb) v = A[(long long)(j0 + lane) * n + j0 + q];
    else if (q == lane) v = make_double2(1, 0);  // pad rows / columns: identity, never pivoted
    a[u] = v;
    perm[u] = q;
  }
  // Rows are not moved: each lane keeps its row's logical position (the
  // position row swaps would give it) and the pivot row is only broadcast.
  int mypos = lane;
  bool used = false;
  // pivot search on column value v of the rows not yet pivoted, by the warp
  // that owns the column; publishes the column, the pivot lane, the position
  // the pivot row had and the pivot's inverse into buffer par
  int gj_next = 0;  // (bench variants only)
  (void)gj_next;
  auto find_pivot = [&](const double2 v, int par) {
    // every row's reciprocal, formed while the pivot reduction runs (only the
    // pivot row's is used)
#if defined(GJ_EXP) && GJ_EXP == 1  // bench only: no reciprocal
    const double rden = 1e-2;
#else
    const double rden = 1.0 / (v.x * v.x + v.y * v.y);
#endif
    // pivot = max |re| + |im| over the rows not yet pivoted, in one warp
    // reduction: the magnitude's high word (non-negative doubles order like
    // their bit patterns) with the low 5 bits replaced by 31 - position, so ties
    // (to 2^-15 relative) go to the lower (swapped) row.  Keys of candidate rows
    // are distinct, so the one lane whose key is the maximum publishes itself:
    // no ballot / find-first on the critical chain.
    unsigned key = 0;
    if (!used && lane < nb) key = ((unsigned)__double2hiint(fabs(v.x) + fabs(v.y)) & ~31u) | (31u - (unsigned)mypos);
#if defined(GJ_EXP) && GJ_EXP == 2  // bench only: no pivot search (diagonal pivots)
    const unsigned best = __shfl_sync(0xffffffffu, key, gj_next);
#else
    const unsigned best = __reduce_max_sync(0xffffffffu, key);
#endif
    gj_f[par][lane] = v;
    if (key == best && (best & ~31u) != 0u) {
      gj_piv[par] = lane;
      gj_pos[par] = mypos;
      gj_inv[par] = make_double2(v.x * rden, -v.y * rden);
    }
    if (lane == 0 && (best & ~31u) == 0u) {  // zero pivot column: flagged, the panel's result is not used
      gj_piv[par] = 0;
      gj_pos[par] = 0;
      gj_inv[par] = make_double2(0, 0);
      if (bad) atomicExch(bad, 1);
    }
  };
  if (warp == 0) find_pivot(a[0], 0);
  __syncthreads();
  // p = CW pb + pu with pu unrolled: the pivot column is a static register.
  // Row update a -= (f / pivot) * (pivot row), the pivot row itself becoming
  // (pivot row) / pivot: with g = f / pivot (pivot row: g = -1 / pivot on a zero
  // base) that is 4 FMAs per entry.  The warp owning column p + 1 updates that
  // column first and searches the next pivot at once, so the search overlaps
  // the other warps' updates: one barrier per step, the search off the
  // critical path.
#pragma unroll 1
  for (int pb = 0; pb * CW < nb; ++pb)
#pragma unroll
  for (int pu = 0; pu < CW; ++pu) {
    const int p = pb * CW + pu;
    if (p >= nb) break;
    const int par = p & 1;
    const int pl = gj_piv[par], q = gj_pos[par];
    const double2 inv = gj_inv[par];
    const double2 f = gj_f[par][lane];
    const bool piv_lane = lane == pl;
    const double2 g = piv_lane ? make_double2(-inv.x, -inv.y) : (lane < nb ? cmul(f, inv) : make_double2(0, 0));
    auto upd = [&](double2& x) {
      double2 pv;  // the pivot row of this column
      pv.x = __shfl_sync(0xffffffffu, x.x, pl);
      pv.y = __shfl_sync(0xffffffffu, x.y, pl);
      double bx = piv_lane ? 0.0 : x.x, by = piv_lane ? 0.0 : x.y;
      bx = fma(-g.x, pv.x, bx);
      bx = fma(g.y, pv.y, bx);
      by = fma(-g.x, pv.y, by);
      by = fma(-g.y, pv.x, by);
      x = make_double2(bx, by);
    };
    // bookkeeping of the row swap of step p (needed by the next search)
    if (piv_lane) {
      mypos = p;
      used = true;
    } else if (mypos == p) {
      mypos = q;  // the row at position p moves to the pivot's position
    }
    const int pun = (pu + 1) % CW;  // column p + 1 in its owner's registers
    const bool next_owner = p + 1 < nb && warp == (pu == CW - 1 ? pb + 1 : pb);
    gj_next = p + 1;
    if (next_owner) {
      upd(a[pun]);
      find_pivot(a[pun], par ^ 1);
    }
#pragma unroll
    for (int u = 0; u < CW; ++u) {
      if (u == pu && warp == pb) {
        // the pivot column: the pivot row's identity column after this step
        a[u] = make_double2(-g.x, -g.y);
        perm[u] = pl;
      } else if (!(next_owner && u == pun)) {
        upd(a[u]);
      }
    }
#if !(defined(GJ_EXP) && GJ_EXP == 4)  // (bench only: 4 = no barrier, racy)
    __syncthreads();
#endif
  }
  pdl_trigger();
  // row = the lane's position, column = the identity column the register holds
  double2* Pi = Pinv + c * pstride;
#pragma unroll
  for (int u = 0; u < CW; ++u) Pi[mypos * 32 + perm[u]] = a[u];
}

constexpr size_t kGjUpdSmem = 4 * 32 * 33 * sizeof(double2);

// Trailing update of the GJ panel step.  grid (ceil(n/32), ceil(n/32), ncls), block 256
__global__ void __launch_bounds__(256) k_gj_update(double2* X, long long xstride, int k, int n,
                                                   int j0, int nb, const double2* Pinv, const double2* Bp,
                                                   const double2* Cp, long long pstride) {
  extern __shared__ double2 upd_sm[];  // Cs, Rs, Ps, Bs: 4 x [32][33]
  auto Cs = reinterpret_cast<double2 (*)[33]>(upd_sm);
  auto Rs = reinterpret_cast<double2 (*)[33]>(upd_sm + 32 * 33);
  auto Ps = reinterpret_cast<double2 (*)[33]>(upd_sm + 2 * 32 * 33);
  auto Bs = reinterpret_cast<double2 (*)[33]>(upd_sm + 3 * 32 * 33);
  pdl_enter();
  const int c = blockIdx.z;
  double2* A = X + c * xstride + (long long)k * n * n;
  const double2* B = Bp + c * pstride;
  const double2* C = Cp + c * pstride;
  const double2* Pi = Pinv + c * pstride;
  const int r0 = blockIdx.y * 32, q0 = blockIdx.x * 32;
  const int tid = threadIdx.x;
  for (int i = tid; i < 32 * 32; i += 256) {
    int a = i / 32, b = i % 32;
    Cs[a][b] = (r0 + a < n && b < nb) ? C[(long long)(r0 + a) * 32 + b] : make_double2(0, 0);
    Ps[a][b] = Pi[i];
    Bs[a][b] = (a < nb && q0 + b < n) ? B[(long long)a * n + q0 + b] : make_double2(0, 0);
  }
  // this thread's four elements of the tile, fetched before the inner products
  double2 aold[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int r = r0 + (tid >> 5) + 8 * m, qq = q0 + (tid & 31);
    aold[m] = (r < n && qq < n) ? A[(long long)r * n + qq] : make_double2(0, 0);
  }
  __syncthreads();
  // row panel tile R = P^{-1} A[J, cols] (cols outside J) or P^{-1}[:, cols - j0].
  // A thread owns one column and four rows (w, w + 8, ...): every shared-memory
  // operand of the inner products is loaded once per four complex FMAs (the
  // one-output-per-pass form was bound by shared-memory bandwidth).
  const int ql = tid & 31, w = tid >> 5;
  const int q = q0 + ql;
  {
    double2 v[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) v[m] = make_double2(0, 0);
#pragma unroll 8
    for (int u = 0; u < 32; ++u) {
      const double2 bs = Bs[u][ql];
#pragma unroll
      for (int m = 0; m < 4; ++m) cfma(v[m], Ps[w + 8 * m][u], bs);
    }
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int t = w + 8 * m;
      double2 r = make_double2(0, 0);
      if (t < nb && q < n) r = (q >= j0 && q < j0 + nb) ? Ps[t][q - j0] : v[m];
      Rs[t][ql] = r;
    }
  }
  __syncthreads();
  double2 sacc[4];
#pragma unroll
  for (int m = 0; m < 4; ++m) sacc[m] = make_double2(0, 0);
  for (int t = 0; t < nb; ++t) {
    const double2 r = Rs[t][ql];
#pragma unroll
    for (int m = 0; m < 4; ++m) cfma(sacc[m], Cs[w + 8 * m][t], r);
  }
#pragma unroll
  for (int m = 0; m < 4; ++m) {
    const int a = w + 8 * m;
    const int r = r0 + a;
    if (r >= n || q >= n) continue;
    double2 v;
    if (r >= j0 && r < j0 + nb) {
      v = Rs[r - j0][ql];
    } else {
      v = (q >= j0 && q < j0 + nb) ? make_double2(0, 0) : aold[m];
      v = csub(v, sacc[m]);
    }
    A[(long long)r * n + q] = v;
  }
}

// Complex GEMM, batched over blockIdx.z:  C = alpha * A * B + beta * C
// A: M x K (lda), B: K x N (ldb), C: M x N (ldc); 64 x 64 tiles, 256 threads,
// 4 x 4 complex outputs per thread (rows ty + 16 i, cols tx + 16 j).
__global__ void __launch_bounds__(256) k_zgemm(int M, int N, int K, double2 alpha,
                                               const double2* A, int lda, long long sa,
                                               const double2* B, int ldb, long long sb,
                                               double2 beta, double2* C, int ldc, long long sc) {
  __shared__ double2 As[16][64];
  __shared__ double2 Bs[16][64];
  const int z = blockIdx.z;
  A += z * sa;
  B += z * sb;
  C += z * sc;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0, 0);
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = tid; i < 16 * 64; i += 256) {
      int kk = i & 15, mm = i >> 4;  // A tile: 64 rows x 16 k
      int gr = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gr < M && gk < K) ? A[(long long)gr * lda + gk] : make_double2(0, 0);
      int kb = i >> 6, nn = i & 63;  // B tile: 16 k x 64 cols
      int bk = k0 + kb, bc = n0 + nn;
      Bs[kb][nn] = (bk < K && bc < N) ? B[(long long)bk * ldb + bc] : make_double2(0, 0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < 16; ++kk) {
      double2 a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cfma(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
  const bool zero_beta = beta.x == 0.0 && beta.y == 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = m0 + ty + 16 * i;
    if (r >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int q = n0 + tx + 16 * j;
      if (q >= N) continue;
      double2 v = cmul(alpha, acc[i][j]);
      long long o = (long long)r * ldc + q;
      if (!zero_beta) v = cadd(v, cmul(beta, C[o]));
      C[o] = v;
    }
  }
}

// Forward right-hand side of row k: B = F_k - sum over the eliminated
// neighbour rows kp of C Y_kp (kp1, kp2: rows or -1); F_k's unit part for the
// 4n boundary columns (faces W,S,N,E, position p) is analytic.
// grid (n, ncls), block 256
__global__ void k_rhs_fwd(double2* Bk, long long bstride, const double2* Y, long long ystride,
                          const uint8_t* masks, int n, int R, int nunit, double ih2, int k, int kp1, int kp2) {
  const int x = blockIdx.x, c = blockIdx.y;
  const uint8_t* m = masks + (long long)c * n * n;
  const int kp[2] = {kp1, kp2};
  double cx[2];
  const double2* Yp[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    cx[q] = kp[q] >= 0 ? coupling2(m, n, k, kp[q], x, ih2) : 0.0;
    Yp[q] = Y + c * ystride + ((long long)(kp[q] >= 0 ? kp[q] : 0) * n + x) * R;
  }
  double2* B = Bk + c * bstride + (long long)x * R;
  for (int col = threadIdx.x; col < R; col += blockDim.x) {
    double2 v = make_double2(0, 0);
    if (col < nunit) {
      int f = col / n, p = col - f * n;
      bool hit = (f == 0 && k == p && x == 0) || (f == 1 && k == 0 && x == p) ||
                 (f == 2 && k == n - 1 && x == p) || (f == 3 && k == p && x == n - 1);
      if (hit) v.x = 1.0;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (cx[q] != 0.0) {
        const double2 y = Yp[q][col];
        v.x -= cx[q] * y.x;
        v.y -= cx[q] * y.y;
      }
    }
    B[col] = v;
  }
}

// Forward right-hand side of row k for the field solves of several subdomains
// (one column each): F_k = rhs_coeff * (incoming traces scattered to the face
// cells, corners get two faces; discretization.py:278-285) - sum over the
// eliminated neighbour rows kp of C Y_kp.
// face_off[4 * col + f]: element offset of the subdomain's incoming block for
// face f (W,S,N,E) in g, or -1.   grid (n, 1), block <= 256
__global__ void k_rhs_traces(double2* Bk, const double2* Y, const uint8_t* mask, int n, int R, double ih2,
                             int k, int kp1, int kp2, const double2* g, const int* face_off, double2 coeff) {
  const int x = blockIdx.x;
  const int kp[2] = {kp1, kp2};
  double cx[2];
  const double2* Yp[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    cx[q] = kp[q] >= 0 ? coupling2(mask, n, k, kp[q], x, ih2) : 0.0;
    Yp[q] = Y + ((long long)(kp[q] >= 0 ? kp[q] : 0) * n + x) * R;
  }
  double2* B = Bk + (long long)x * R;
  for (int col = threadIdx.x; col < R; col += blockDim.x) {
    const int* fo = face_off + 4 * col;
    double2 t = make_double2(0, 0);
    if (x == 0 && fo[0] >= 0) t = cadd(t, g[fo[0] + k]);          // W, position k
    if (k == 0 && fo[1] >= 0) t = cadd(t, g[fo[1] + x]);          // S, position x
    if (k == n - 1 && fo[2] >= 0) t = cadd(t, g[fo[2] + x]);      // N, position x
    if (x == n - 1 && fo[3] >= 0) t = cadd(t, g[fo[3] + k]);      // E, position k
    double2 v = cmul(coeff, t);
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (cx[q] != 0.0) {
        const double2 y = Yp[q][col];
        v.x -= cx[q] * y.x;
        v.y -= cx[q] * y.y;
      }
    }
    B[col] = v;
  }
}

// Stitch solved fields Y[k][x][col] into the global grid (y slow):
// field[(b-1) n + k][(a-1) n + x] (+)= Y, one column per subdomain.
__global__ void k_scatter_field(double2* field, int nx_total, const double2* Y, int n, int R,
                                const int* col_ab, int accumulate) {
  const long long total = (long long)n * n * R;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int col = (int)(i % R);
    const long long cell = i / R;
    const int k = (int)(cell / n), x = (int)(cell % n);
    const int a = col_ab[2 * col], b = col_ab[2 * col + 1];
    const long long o = ((long long)(b - 1) * n + k) * nx_total + (long long)(a - 1) * n + x;
    field[o] = accumulate ? cadd(field[o], Y[i]) : Y[i];
  }
}

// Sparse additions to F_k (Dirichlet data and its coupling to free cells).
__global__ void k_rhs_extra(double2* Bk, long long bstride, int R, const int* ex_x, const int* ex_col,
                            const double2* ex_val, int cnt, int c) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cnt) return;
  double2* B = Bk + c * bstride;
  long long o = (long long)ex_x[i] * R + ex_col[i];
  B[o] = cadd(B[o], ex_val[i]);
}

// Backward: B = C U_kn, kn the neighbour row towards the middle.  grid (n, ncls)
__global__ void k_rhs_bwd(double2* Bk, long long bstride, const double2* Y, long long ystride,
                          const uint8_t* masks, int n, int R, double ih2, int k, int kn) {
  const int x = blockIdx.x, c = blockIdx.y;
  const uint8_t* m = masks + (long long)c * n * n;
  const double cx = coupling2(m, n, k, kn, x, ih2);
  const double2* Yn = Y + c * ystride + ((long long)kn * n + x) * R;
  double2* B = Bk + c * bstride + (long long)x * R;
  for (int col = threadIdx.x; col < R; col += blockDim.x) {
    double2 y = Yn[col];
    B[col] = make_double2(cx * y.x, cx * y.y);
  }
}

// Boundary values G[4n][R] (faces W,S,N,E; increasing coordinate) of U.
__global__ void k_extract(double2* G, long long gstride, const double2* Y, long long ystride, int n,
                          int R) {
  const int row = blockIdx.x, c = blockIdx.y;
  const int f = row / n, p = row - f * n;
  int k, x;
  if (f == 0) { k = p; x = 0; }
  else if (f == 1) { k = 0; x = p; }
  else if (f == 2) { k = n - 1; x = p; }
  else { k = p; x = n - 1; }
  const double2* src = Y + c * ystride + ((long long)k * n + x) * R;
  double2* dst = G + c * gstride + (long long)row * R;
  for (int col = threadIdx.x; col < R; col += blockDim.x) dst[col] = src[col];
}

// T4 = a I + b G[:, :4n]   (a = -s/d, b = -2 tau/(h^3 d^2))
__global__ void k_make_T4(double2* T4, const double2* G, int n4, int R, double2 a, double2 b) {
  const int row = blockIdx.x;
  for (int col = threadIdx.x; col < n4; col += blockDim.x) {
    double2 v = cmul(b, G[(long long)row * R + col]);
    if (row == col) v = cadd(v, a);
    T4[(long long)row * n4 + col] = v;
  }
}

// Scatter compact per-subdomain maps (tile-major) from the class maps.
// One CTA per (sub, tile) via the tile list; face[] maps compact -> global face.
__global__ void __launch_bounds__(256) k_scatter_T(const int2* tl, const DevSub* subs,
                                                   const int* sub_faces, const int* sub_cls,
                                                   double2* const* T4s, double2* T, int n) {
  __shared__ double2 buf[32][33];
  const int2 st = tl[blockIdx.x];
  const int s = st.x, tile = st.y;
  const DevSub sb = subs[s];
  const int K = sb.k * n;
  const int n4 = 4 * n;
  const double2* T4 = T4s[sub_cls[s]];
  const int* fc = sub_faces + 4 * s;
  double2* out = T + sb.T_off + (long long)tile * K * kRowTile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int c0 = 0; c0 < K; c0 += 32) {
    // read rows (tile) x cols c0..c0+31 coalesced along columns
    for (int a = warp; a < 32; a += 8) {
      int r = tile * 32 + a;
      int col = c0 + lane;
      double2 v = make_double2(0, 0);
      if (r < K && col < K) {
        int gr = fc[r / n] * n + r % n;
        int gc = fc[col / n] * n + col % n;
        v = T4[(long long)gr * n4 + gc];
      }
      buf[a][lane] = v;
    }
    __syncthreads();
    for (int cc = warp; cc < 32; cc += 8) {
      int col = c0 + cc;
      if (col < K) out[(long long)col * kRowTile + lane] = buf[lane][cc];
    }
    __syncthreads();
  }
}

// Lifting traces of the home subdomain into b: b[m(j,home)] = coef * U_face(lift col).
__global__ void k_lift_b(double2* b, const double2* G, int Rtot, int col0, int nrhs, int n,
                         const int* face_tgt /*4: element offsets or -1*/, double2 coef) {
  const int row = blockIdx.x;  // 0..4n
  const int f = row / n, p = row - f * n;
  const int off = face_tgt[f];
  if (off < 0) return;
  for (int j = threadIdx.x; j < nrhs; j += blockDim.x) {
    double2 g = G[(long long)row * Rtot + col0 + j];
    b[((long long)off + p) * nrhs + j] = cmul(coef, g);
  }
}

// ---------------------------------------------------------------------------
// host drivers

static OpParams op_params(const Ctx& c) {
  OpParams P;
  P.n = c.n;
  P.ih2 = 1.0 / (c.h * c.h);
  // d = 1/h - tau/2, s = 1/h + tau/2, ratio = s/d (discretization.py:139-140, 245)
  double dr = 1.0 / c.h - c.tau_re / 2, di = -c.tau_im / 2;
  double sr = 1.0 / c.h + c.tau_re / 2, si = c.tau_im / 2;
  double den = dr * dr + di * di;
  double rr = (sr * dr + si * di) / den, ri = (si * dr - sr * di) / den;
  P.dre = 4.0 * P.ih2 - c.kappa * c.kappa;
  P.dim = 0;
  P.gre = -P.ih2 * rr;
  P.gim = -P.ih2 * ri;
  return P;
}

void zgemm(cudaStream_t st, int M, int N, int K, double2 alpha, const double2* A, int lda,
           long long sa, const double2* B, int ldb, long long sb, double2 beta, double2* C, int ldc,
           long long sc, int batch) {
  static const bool use_dmma = !(getenv("HS_ZGEMM_FMA") && atoi(getenv("HS_ZGEMM_FMA")) != 0);
  if (use_dmma && zgemm_dmma(st, M, N, K, alpha, A, lda, sa, B, ldb, sb, beta, C, ldc, sc, batch)) return;
  dim3 grid((N + 63) / 64, (M + 63) / 64, batch);
  k_zgemm<<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, sa, B, ldb, sb, beta, C, ldc, sc);
}

// The twisted elimination order (file header): row m = n / 2 is the middle; the
// top chain runs k = 0 .. m-1 (previous row k-1), the bottom chain k = n-1 ..
// m+1 (previous row k+1), row m has both neighbours as previous rows.
struct Twist {
  int n, m;
  explicit Twist(int n_) : n(n_), m(n_ / 2) {}
  int ntop() const { return m; }
  int nbot() const { return n - 1 - m; }
  int top(int i) const { return i; }
  int bot(int i) const { return n - 1 - i; }
  int mid_prev1() const { return m >= 1 ? m - 1 : -1; }
  int mid_prev2() const { return m + 1 < n ? m + 1 : -1; }
};

// Factorisation interleaved with the forward sweep of the boundary solves.
// Four streams: one per chain for the panel steps (the chains are independent
// until row m; high priority, so their small latency-bound kernels are not
// queued behind full-grid GEMMs), and one per chain for the forward solve step
// of row k (it only needs X_k) while the chain factors its next rows.  Row m,
// the backward sweeps (again one stream per half) and the extraction follow.
// Rp / Cp / Bk hold two slices (2 * ncls classes' worth), one per chain.
cudaError_t factor_and_solve_boundary(Ctx& c, double2* X, long long xstride, const uint8_t* dmasks, int ncls,
                                      double2* Rp, double2* Cp, long long pstride, int* dbad, int R, int nunit,
                                      const ExtraRHS* extras, double2* Y, long long ystride, double2* Bk,
                                      long long bstride, double2* G, long long gstride) {
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_gj_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGjUpdSmem);
  if (attr != cudaSuccess) return attr;
  const int n = c.n;
  const double ih2 = 1.0 / (c.h * c.h);
  const long long nn = (long long)n * n;
  const int rthreads = R < 256 ? ((R + 31) / 32) * 32 : 256;
  const OpParams P = op_params(c);
  const Twist tw(n);
  // top / bottom chain (high priority: their small latency-bound kernels go ahead
  // of the forward solves' full-grid GEMMs), forward solves of the two chains
  cudaStream_t sa = nullptr, sb = nullptr, fa = nullptr, fb = nullptr;
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (getenv("HS_FACTOR_PRIO") && atoi(getenv("HS_FACTOR_PRIO")) == 0) prio_hi = prio_lo;
  cudaError_t e = cudaStreamCreateWithPriority(&sa, cudaStreamNonBlocking, prio_hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&sb, cudaStreamNonBlocking, prio_hi);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&fa, cudaStreamNonBlocking, prio_lo);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&fb, cudaStreamNonBlocking, prio_lo);
  if (e != cudaSuccess) {
    for (cudaStream_t st : {sa, sb, fa, fb})
      if (st) cudaStreamDestroy(st);
    return e;
  }
  std::vector<cudaEvent_t> ev(n);
  for (auto& x : ev) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  // HS_FACTOR_TIMING=1: phase times of the call on stderr (diagnostics)
  static const bool timing = getenv("HS_FACTOR_TIMING") && atoi(getenv("HS_FACTOR_TIMING")) != 0;
  cudaEvent_t join[8];
  for (auto& x : join) cudaEventCreateWithFlags(&x, timing ? cudaEventDefault : cudaEventDisableTiming);
  cudaEvent_t tend = nullptr;
  if (timing) cudaEventCreate(&tend);
  double2 *RpB = Rp + pstride * ncls, *CpB = Cp + pstride * ncls, *BkB = Bk + bstride * ncls;
  auto factor_row = [&](cudaStream_t st, int k, int kp1, int kp2, double2* rp, double2* cp) {
    launch_pdl(k_formS, dim3(n, ncls), dim3(128), 0, st, X, xstride, dmasks, P, k, kp1, kp2);
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int nb = n - j0 < 32 ? n - j0 : 32;
      // rp slice of a class: the row panel A[J, :] (32 x n), then P^{-1} (32 x 32)
      launch_pdl(k_gj_inv, dim3(1 + 8, ncls), dim3(kGjThreads), 0, st, X, xstride, k, n, j0, nb, rp + 32LL * n, rp, cp,
                 pstride, dbad);
      launch_pdl(k_gj_update, dim3((n + 31) / 32, (n + 31) / 32, ncls), dim3(256), kGjUpdSmem, st, X, xstride, k, n,
                 j0, nb, rp + 32LL * n, rp, cp, pstride);
    }
  };
  // The unit columns (faces W, S, N, E; position p) of a chain's forward sweep
  // are zero until the sweep reaches their cell's row: at row k of the top
  // chain only W / E positions <= k and the S face are nonzero, of the bottom
  // chain W / E positions >= k and the N face.  The block solves skip the zero
  // column ranges (Y is zeroed once): 2.7x fewer flops in the sweeps that share
  // the GPU with the latency-bound panel chains.  Not with sparse extras (their
  // columns can be nonzero in neighbouring rows) or odd sizes.
  bool skip = nunit == 4 * n && R == 4 * n && n % 32 == 0;
  for (int cl = 0; cl < ncls; ++cl) skip = skip && extras[cl].row_ptr.empty();
  if (skip) {
    for (int cl = 0; cl < ncls; ++cl)
      cudaMemsetAsync(Y + cl * ystride, 0, (size_t)nn * R * sizeof(double2), c.stream);
  }
  auto gemm_cols = [&](cudaStream_t st, int k, double2* bk, int c0, int nc) {
    if (nc > 0)
      zgemm(st, n, nc, n, make_double2(1, 0), X + k * nn, n, xstride, bk + c0, R, bstride, make_double2(0, 0),
            Y + (long long)k * n * R + c0, R, ystride, ncls);
  };
  // chain: 0 top, 1 bottom, 2 the middle row (all columns)
  auto forward_row = [&](cudaStream_t st, int k, int kp1, int kp2, double2* bk, int chain) {
    k_rhs_fwd<<<dim3(n, ncls), rthreads, 0, st>>>(bk, bstride, Y, ystride, dmasks, n, R, nunit, ih2, k, kp1, kp2);
    for (int cl = 0; cl < ncls; ++cl) {
      const ExtraRHS& ex = extras[cl];
      if (ex.row_ptr.empty()) continue;
      const int b0 = ex.row_ptr[k], b1 = ex.row_ptr[k + 1];
      if (b1 > b0)
        k_rhs_extra<<<(b1 - b0 + 255) / 256, 256, 0, st>>>(bk, bstride, R, ex.d_x + b0, ex.d_col + b0, ex.d_val + b0,
                                                            b1 - b0, cl);
    }
    if (!skip || chain == 2) {
      gemm_cols(st, k, bk, 0, R);
    } else if (chain == 0) {
      const int cw = std::min(n, (k + 1 + 31) / 32 * 32);
      gemm_cols(st, k, bk, 0, cw);          // W, positions 0 .. k
      gemm_cols(st, k, bk, n, n);           // S
      gemm_cols(st, k, bk, 3 * n, cw);      // E, positions 0 .. k
    } else {
      const int p0 = k / 32 * 32;
      gemm_cols(st, k, bk, p0, n - p0);          // W, positions k .. n-1
      gemm_cols(st, k, bk, 2 * n, n);            // N
      gemm_cols(st, k, bk, 3 * n + p0, n - p0);  // E, positions k .. n-1
    }
  };
  auto backward_row = [&](cudaStream_t st, int k, int kn, double2* bk) {
    k_rhs_bwd<<<dim3(n, ncls), rthreads, 0, st>>>(bk, bstride, Y, ystride, dmasks, n, R, ih2, k, kn);
    zgemm(st, n, R, n, make_double2(-1, 0), X + k * nn, n, xstride, bk, R, bstride, make_double2(1, 0),
          Y + (long long)k * n * R, R, ystride, ncls);
  };
  cudaEventRecord(join[0], c.stream);  // the other streams start after everything queued before
  for (cudaStream_t st : {sa, sb, fa, fb}) cudaStreamWaitEvent(st, join[0], 0);
  const int nt = tw.ntop(), nbt = tw.nbot();
  auto top_row = [&](int i) {
    const int k = tw.top(i), kp = i > 0 ? k - 1 : -1;
    factor_row(sa, k, kp, -1, Rp, Cp);
    cudaEventRecord(ev[k], sa);  // X_k complete
    cudaStreamWaitEvent(fa, ev[k], 0);
    forward_row(fa, k, kp, -1, Bk, 0);
  };
  auto bottom_row = [&](int i) {
    const int k = tw.bot(i), kp = i > 0 ? k + 1 : -1;
    factor_row(sb, k, kp, -1, RpB, CpB);
    cudaEventRecord(ev[k], sb);
    cudaStreamWaitEvent(fb, ev[k], 0);
    forward_row(fb, k, kp, -1, BkB, 1);
  };
  // (enqueueing the chains from two host threads was measured: 48.0 vs 49.0 ms
  // at cfg5 -- the chains are bound by the GPU's dependent-launch latency)
  for (int i = 0; i < (nt > nbt ? nt : nbt); ++i) {  // launches of the two chains interleaved
    if (i < nt) top_row(i);
    if (i < nbt) bottom_row(i);
  }
  // row m couples the chains
  cudaEventRecord(join[1], sb);
  if (timing) cudaEventRecord(join[7], sa);
  cudaStreamWaitEvent(sa, join[1], 0);
  factor_row(sa, tw.m, tw.mid_prev1(), tw.mid_prev2(), Rp, Cp);
  cudaEventRecord(join[2], fa);
  cudaEventRecord(join[3], fb);
  cudaStreamWaitEvent(sa, join[2], 0);
  cudaStreamWaitEvent(sa, join[3], 0);
  forward_row(sa, tw.m, tw.mid_prev1(), tw.mid_prev2(), Bk, 2);
  // backward sweeps, away from row m
  cudaEventRecord(join[4], sa);
  cudaStreamWaitEvent(sb, join[4], 0);
  for (int i = 0; i < (nt > nbt ? nt : nbt); ++i) {
    if (i < nt) backward_row(sa, tw.m - 1 - i, tw.m - i, Bk);
    if (i < nbt) backward_row(sb, tw.m + 1 + i, tw.m + i, BkB);
  }
  cudaEventRecord(join[5], sb);
  cudaStreamWaitEvent(sa, join[5], 0);
  k_extract<<<dim3(4 * n, ncls), rthreads, 0, sa>>>(G, gstride, Y, ystride, n, R);
  cudaEventRecord(join[6], sa);  // back on the context stream
  cudaStreamWaitEvent(c.stream, join[6], 0);
  e = cudaGetLastError();
  if (timing) cudaEventRecord(tend, c.stream);
  // before the streams and their events go away
  for (cudaStream_t st : {sa, sb, fa, fb}) cudaStreamSynchronize(st);
  if (timing) {
    cudaEventSynchronize(tend);
    float top = 0, bot = 0, ffa = 0, ffb = 0, mid = 0, back = 0;
    cudaEventElapsedTime(&top, join[0], join[7]);  // the chains' last panel steps
    cudaEventElapsedTime(&bot, join[0], join[1]);
    cudaEventElapsedTime(&ffa, join[0], join[2]);  // their forward solves
    cudaEventElapsedTime(&ffb, join[0], join[3]);
    cudaEventElapsedTime(&mid, join[0], join[4]);
    cudaEventElapsedTime(&back, join[4], tend);
    fprintf(stderr,
            "[hs_factor] n=%d classes=%d: chains %.3f / %.3f ms, their forward solves %.3f / %.3f ms, through row m "
            "%.3f ms, backward %.3f ms\n",
            n, ncls, top, bot, ffa, ffb, mid, back);
    cudaEventDestroy(tend);
  }
  for (auto& x : ev) cudaEventDestroy(x);
  for (auto& x : join) cudaEventDestroy(x);
  for (cudaStream_t st : {sa, sb, fa, fb}) cudaStreamDestroy(st);
  return e;
}

// Solve the factored block-tridiagonal systems for R right-hand sides (twisted
// order, one stream) and extract the boundary values G (4n x R) per class.
cudaError_t solve_boundary(Ctx& c, const double2* X, long long xstride, const uint8_t* dmasks,
                           int ncls, int R, int nunit, const ExtraRHS* extras, double2* Y,
                           long long ystride, double2* Bk, long long bstride, double2* G,
                           long long gstride) {
  const int n = c.n;
  const double ih2 = 1.0 / (c.h * c.h);
  const long long nn = (long long)n * n;
  const int rthreads = R < 256 ? ((R + 31) / 32) * 32 : 256;
  const Twist tw(n);
  auto forward_row = [&](int k, int kp1, int kp2) {
    k_rhs_fwd<<<dim3(n, ncls), rthreads, 0, c.stream>>>(Bk, bstride, Y, ystride, dmasks, n, R, nunit, ih2, k, kp1,
                                                        kp2);
    for (int cl = 0; cl < ncls; ++cl) {
      const ExtraRHS& e = extras[cl];
      if (e.row_ptr.empty()) continue;
      const int b0 = e.row_ptr[k], b1 = e.row_ptr[k + 1];
      if (b1 > b0)
        k_rhs_extra<<<(b1 - b0 + 255) / 256, 256, 0, c.stream>>>(Bk, bstride, R, e.d_x + b0, e.d_col + b0,
                                                                 e.d_val + b0, b1 - b0, cl);
    }
    zgemm(c.stream, n, R, n, make_double2(1, 0), X + k * nn, n, xstride, Bk, R, bstride, make_double2(0, 0),
          Y + (long long)k * n * R, R, ystride, ncls);
  };
  auto backward_row = [&](int k, int kn) {
    k_rhs_bwd<<<dim3(n, ncls), rthreads, 0, c.stream>>>(Bk, bstride, Y, ystride, dmasks, n, R, ih2, k, kn);
    zgemm(c.stream, n, R, n, make_double2(-1, 0), X + k * nn, n, xstride, Bk, R, bstride, make_double2(1, 0),
          Y + (long long)k * n * R, R, ystride, ncls);
  };
  for (int i = 0; i < tw.ntop(); ++i) forward_row(tw.top(i), i > 0 ? tw.top(i) - 1 : -1, -1);
  for (int i = 0; i < tw.nbot(); ++i) forward_row(tw.bot(i), i > 0 ? tw.bot(i) + 1 : -1, -1);
  forward_row(tw.m, tw.mid_prev1(), tw.mid_prev2());
  for (int k = tw.m - 1; k >= 0; --k) backward_row(k, k + 1);
  for (int k = tw.m + 1; k < n; ++k) backward_row(k, k - 1);
  k_extract<<<dim3(4 * n, ncls), rthreads, 0, c.stream>>>(G, gstride, Y, ystride, n, R);
  return cudaGetLastError();
}

// Full fields of R subdomains of one operator class driven by their incoming
// traces in g (+ sparse extras: the lifting's Dirichlet data), Y = n x n x R.
cudaError_t solve_fields(Ctx& c, const double2* X, const uint8_t* dmask, int R, const double2* g,
                         const int* face_off, double2 coeff, const ExtraRHS& extras, double2* Y, double2* Bk) {
  const int n = c.n;
  const double ih2 = 1.0 / (c.h * c.h);
  const long long nn = (long long)n * n;
  const int rthreads = R < 256 ? ((R + 31) / 32) * 32 : 256;
  const Twist tw(n);
  auto forward_row = [&](int k, int kp1, int kp2) {
    c.launches++;
    k_rhs_traces<<<n, rthreads, 0, c.stream>>>(Bk, Y, dmask, n, R, ih2, k, kp1, kp2, g, face_off, coeff);
    if (!extras.row_ptr.empty()) {
      const int b0 = extras.row_ptr[k], b1 = extras.row_ptr[k + 1];
      if (b1 > b0) {
        c.launches++;
        k_rhs_extra<<<(b1 - b0 + 255) / 256, 256, 0, c.stream>>>(Bk, 0, R, extras.d_x + b0, extras.d_col + b0,
                                                                 extras.d_val + b0, b1 - b0, 0);
      }
    }
    c.launches++;
    zgemm(c.stream, n, R, n, make_double2(1, 0), X + k * nn, n, 0, Bk, R, 0, make_double2(0, 0),
          Y + (long long)k * n * R, R, 0, 1);
  };
  auto backward_row = [&](int k, int kn) {
    c.launches += 2;
    k_rhs_bwd<<<dim3(n, 1), rthreads, 0, c.stream>>>(Bk, 0, Y, 0, dmask, n, R, ih2, k, kn);
    zgemm(c.stream, n, R, n, make_double2(-1, 0), X + k * nn, n, 0, Bk, R, 0, make_double2(1, 0),
          Y + (long long)k * n * R, R, 0, 1);
  };
  for (int i = 0; i < tw.ntop(); ++i) forward_row(tw.top(i), i > 0 ? tw.top(i) - 1 : -1, -1);
  for (int i = 0; i < tw.nbot(); ++i) forward_row(tw.bot(i), i > 0 ? tw.bot(i) + 1 : -1, -1);
  forward_row(tw.m, tw.mid_prev1(), tw.mid_prev2());
  for (int k = tw.m - 1; k >= 0; --k) backward_row(k, k + 1);
  for (int k = tw.m + 1; k < n; ++k) backward_row(k, k - 1);
  return cudaGetLastError();
}

void launch_scatter_field(Ctx& c, double2* field, int nx_total, const double2* Y, int R, const int* col_ab,
                          int accumulate) {
  c.launches++;
  k_scatter_field<<<4 * c.num_sms, 256, 0, c.stream>>>(field, nx_total, Y, c.n, R, col_ab, accumulate);
}

// flag |= 2 when any of the count values is not finite
__global__ void k_finite_check(const double2* v, long long count, int* flag) {
  bool bad = false;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x) {
    const double2 x = v[i];
    bad |= !isfinite(x.x) || !isfinite(x.y);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 2);
}

void launch_finite_check(Ctx& c, const double2* v, long long count, int* flag) {
  k_finite_check<<<2 * c.num_sms, 256, 0, c.stream>>>(v, count, flag);
}

void launch_make_T4(Ctx& c, double2* T4, const double2* G, int R, double2 a, double2 b) {
  k_make_T4<<<4 * c.n, 256, 0, c.stream>>>(T4, G, 4 * c.n, R, a, b);
}

void launch_scatter_T(Ctx& c, const int2* tl, int ntiles, const int* sub_faces, const int* sub_cls,
                      double2* const* T4s) {
  if (ntiles > 0)
    k_scatter_T<<<ntiles, 256, 0, c.stream>>>(tl, c.dsubs, sub_faces, sub_cls, T4s, c.T, c.n);
}

void launch_lift_b(Ctx& c, double2* b, const double2* G, int Rtot, int col0, int nrhs,
                   const int* face_tgt, double2 coef) {
  int th = nrhs < 32 ? 32 : (nrhs > 256 ? 256 : nrhs);
  k_lift_b<<<4 * c.n, th, 0, c.stream>>>(b, G, Rtot, col0, nrhs, c.n, face_tgt, coef);
}

HS_DBG_ACCESSOR(hs_dbg_take_schur)

}  // namespace hs
