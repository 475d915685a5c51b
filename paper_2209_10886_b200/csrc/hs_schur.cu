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
// AND columns, their known value moved to the right-hand side).  Natural-order
// block elimination without inter-block pivoting (accurate for these
// operators, SURVEY.md §7 hard part 1):
//     S_0 = D_0,   S_k = D_k - C_{k-1} X_{k-1} C_{k-1},   X_k = S_k^{-1}
// X_k by blocked in-place Gauss-Jordan (32-wide panels, partial pivoting
// inside the diagonal panel block).  Then for the R right-hand sides (one unit
// vector per boundary cell, plus lifting data):
//     Y_0 = X_0 F_0,  Y_k = X_k (F_k - C_{k-1} Y_{k-1})         (forward)
//     U_{n-1} = Y_{n-1},  U_k = Y_k - X_k C_k U_{k+1}            (backward)
// and the boundary rows of U give E^T A^{-1} E.  All dense work is batched
// over the distinct operators; the products are complex GEMMs.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

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

// coupling between row k and k+1 at column x
__device__ __forceinline__ double coupling(const uint8_t* m, int n, int k, int x, double ih2) {
  return (dmask(m, n, k, x) || dmask(m, n, k + 1, x)) ? 0.0 : -ih2;
}

// S_k = D_k - C X_{k-1} C  written into X_k.   grid (n, ncls), block 256
__global__ void k_formS(double2* X, long long xstride, const uint8_t* masks, OpParams P, int k) {
  const int n = P.n;
  const int i = blockIdx.x;
  const int c = blockIdx.y;
  const uint8_t* m = masks + (long long)c * n * n;
  double2* Xk = X + c * xstride + (long long)k * n * n;
  const double2* Xp = Xk - (long long)n * n;
  const bool di = dmask(m, n, k, i);
  const double ci = k > 0 ? coupling(m, n, k - 1, i, P.ih2) : 0.0;
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
    if (k > 0 && ci != 0.0) {
      const double cj = coupling(m, n, k - 1, j, P.ih2);
      if (cj != 0.0) {
        double2 xv = Xp[(long long)i * n + j];
        v.x -= ci * xv.x * cj;
        v.y -= ci * xv.y * cj;
      }
    }
    Xk[(long long)i * n + j] = v;
  }
}

// Panel step of blocked Gauss-Jordan on A = X_k (n x n, in place), panel
// columns J = [j0, j0+nb), in two kernels:
//   k_gj_inv:    CTA 0: P^{-1} of P = A[J,J] by Gauss-Jordan with partial
//                pivoting (max |re| + |im|, ties to the lower row) -> Pinv;
//                the other CTAs copy the panels A[J, :] and A[:, J];
//   k_gj_update: each 32 x 32 tile forms its row-panel tile P^{-1} A[J, cols]
//                and applies the trailing update.
// k_gj_inv keeps [P | I] in registers: warp w owns columns [8w, 8w + 8),
// lane = row.  Per pivot step the warp owning column p finds the pivot and
// publishes the column and the pivot's inverse (double-buffered by step
// parity), one barrier, then every warp swaps rows p and pr, scales the pivot
// row and eliminates its columns with warp shuffles: one barrier per step
// (the shared-memory form had five and took 57 us per panel).
// grid (ncls), block 256
__global__ void __launch_bounds__(256) k_gj_inv(const double2* X, long long xstride, int k, int n, int j0,
                                                int nb, double2* Pinv, double2* Bp, double2* Cp,
                                                long long pstride, int* bad) {
  __shared__ double2 gj_f[2][32];
  __shared__ double2 gj_inv[2];
  __shared__ int gj_piv[2], gj_pos[2];
  const int c = blockIdx.y;
  const double2* A = X + c * xstride + (long long)k * n * n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (blockIdx.x > 0) {
    // the other CTAs copy the row panel Bp = A[J, :] and the column panel
    // Cp = A[:, J] before the update overwrites A
    const int nc = gridDim.x - 1, b = blockIdx.x - 1;
    double2* B = Bp + c * pstride;
    double2* Cpp = Cp + c * pstride;
    for (int i = b * 256 + tid; i < nb * n; i += nc * 256) {
      const int t = i / n, col = i % n;
      B[(long long)t * n + col] = A[(long long)(j0 + t) * n + col];
    }
    for (int i = b * 256 + tid; i < n * nb; i += nc * 256) {
      const int r = i / nb, t = i % nb;
      Cpp[(long long)r * 32 + t] = A[(long long)r * n + j0 + t];
    }
    return;
  }
  double2 a[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int q = warp * 8 + u;
    double2 v = make_double2(0, 0);
    if (lane < nb) {
      if (q < nb) v = A[(long long)(j0 + lane) * n + j0 + q];
      else if (q - 32 == lane) v = make_double2(1, 0);
    } else if (q == lane || q - 32 == lane) {
      v = make_double2(q == lane ? 1 : 0, 0);  // pad rows: identity, never pivoted into
    }
    a[u] = v;
  }
  // Rows are not moved: each lane keeps its row's logical position (the
  // position row swaps would give it) and the pivot row is only broadcast.
  int mypos = lane;
  bool used = false;
  // p = 8 pb + pu with pu unrolled: the pivot column is a static register
#pragma unroll 1
  for (int pb = 0; pb * 8 < nb; ++pb)
#pragma unroll
  for (int pu = 0; pu < 8; ++pu) {
    const int p = pb * 8 + pu;
    if (p >= nb) break;
    const int par = p & 1;
    if (warp == pb) {
      const double2 v = a[pu];
      // pivot = max |re| + |im| over the rows not yet pivoted, in one warp
      // reduction: the magnitude rounded to float (non-negative floats order
      // like their bit patterns) with the low 5 bits replaced by 31 - position,
      // so ties go to the lower (swapped) row
      unsigned key = 0;
      if (!used && lane < nb) {
        const float m = (float)(fabs(v.x) + fabs(v.y));
        key = (__float_as_uint(m) & ~31u) | (31u - (unsigned)mypos);
      }
      const unsigned best = __reduce_max_sync(0xffffffffu, key);
      const int pl = __ffs(__ballot_sync(0xffffffffu, key == best)) - 1;
      gj_f[par][lane] = v;
      if (lane == 0) {
        gj_piv[par] = pl;
        gj_pos[par] = 31 - (int)(best & 31u);
        if ((best & ~31u) == 0u && bad) atomicExch(bad, 1);  // zero pivot column
      }
      if (lane == pl) {
        const double rden = 1.0 / (v.x * v.x + v.y * v.y);
        gj_inv[par] = make_double2(v.x * rden, -v.y * rden);
      }
    }
    __syncthreads();
    const int pl = gj_piv[par], q = gj_pos[par];
    const double2 inv = gj_inv[par];
    const double2 f = gj_f[par][lane];
    const bool fz = f.x == 0.0 && f.y == 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      double2 pv;  // the pivot row of this column
      pv.x = __shfl_sync(0xffffffffu, a[u].x, pl);
      pv.y = __shfl_sync(0xffffffffu, a[u].y, pl);
      const double2 np = cmul(pv, inv);  // scaled pivot row
      if (lane == pl) a[u] = np;
      else if (lane < nb && !fz) a[u] = csub(a[u], cmul(f, np));
    }
    if (lane == pl) {
      mypos = p;
      used = true;
    } else if (mypos == p) {
      mypos = q;  // the row at position p moves to the pivot's position
    }
  }
  if (warp >= 4) {  // columns 32..63 hold P^{-1}, row = the lane's position
    double2* Pi = Pinv + c * pstride;
#pragma unroll
    for (int u = 0; u < 8; ++u) Pi[mypos * 32 + (warp - 4) * 8 + u] = a[u];
  }
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
  __syncthreads();
  // row panel tile R = P^{-1} A[J, cols] (cols outside J) or P^{-1}[:, cols - j0]
  for (int i = tid; i < 32 * 32; i += 256) {
    const int t = i / 32, b = i % 32, col = q0 + b;
    double2 v = make_double2(0, 0);
    if (t < nb && col < n) {
      if (col >= j0 && col < j0 + nb) {
        v = Ps[t][col - j0];
      } else {
#pragma unroll
        for (int u = 0; u < 32; ++u) cfma(v, Ps[t][u], Bs[u][b]);
      }
    }
    Rs[t][b] = v;
  }
  __syncthreads();
  const int ql = tid & 31;
  const int q = q0 + ql;
  for (int a = tid >> 5; a < 32; a += 8) {
    const int r = r0 + a;
    if (r >= n || q >= n) continue;
    double2 v;
    if (r >= j0 && r < j0 + nb) {
      v = Rs[r - j0][ql];
    } else {
      v = (q >= j0 && q < j0 + nb) ? make_double2(0, 0) : A[(long long)r * n + q];
      double2 s = make_double2(0, 0);
      for (int t = 0; t < nb; ++t) cfma(s, Cs[a][t], Rs[t][ql]);
      v = csub(v, s);
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

// Forward right-hand side of row k: B = F_k - C_{k-1} Y_{k-1}; F_k's unit part
// for the 4n boundary columns (faces W,S,N,E, position p) is analytic.
// grid (n, ncls), block 256
__global__ void k_rhs_fwd(double2* Bk, long long bstride, const double2* Y, long long ystride,
                          const uint8_t* masks, int n, int R, int nunit, double ih2, int k) {
  const int x = blockIdx.x, c = blockIdx.y;
  const uint8_t* m = masks + (long long)c * n * n;
  const double cx = k > 0 ? coupling(m, n, k - 1, x, ih2) : 0.0;
  const double2* Yp = Y + c * ystride + ((long long)(k - 1) * n + x) * R;
  double2* B = Bk + c * bstride + (long long)x * R;
  for (int col = threadIdx.x; col < R; col += blockDim.x) {
    double2 v = make_double2(0, 0);
    if (col < nunit) {
      int f = col / n, p = col - f * n;
      bool hit = (f == 0 && k == p && x == 0) || (f == 1 && k == 0 && x == p) ||
                 (f == 2 && k == n - 1 && x == p) || (f == 3 && k == p && x == n - 1);
      if (hit) v.x = 1.0;
    }
    if (cx != 0.0) {
      double2 y = Yp[col];
      v.x -= cx * y.x;
      v.y -= cx * y.y;
    }
    B[col] = v;
  }
}

// Forward right-hand side of row k for the field solves of several subdomains
// (one column each): F_k = rhs_coeff * (incoming traces scattered to the face
// cells, corners get two faces; discretization.py:278-285) - C_{k-1} Y_{k-1}.
// face_off[4 * col + f]: element offset of the subdomain's incoming block for
// face f (W,S,N,E) in g, or -1.   grid (n, 1), block <= 256
__global__ void k_rhs_traces(double2* Bk, const double2* Y, const uint8_t* mask, int n, int R, double ih2,
                             int k, const double2* g, const int* face_off, double2 coeff) {
  const int x = blockIdx.x;
  const double cx = k > 0 ? coupling(mask, n, k - 1, x, ih2) : 0.0;
  const double2* Yp = Y + ((long long)(k - 1) * n + x) * R;
  double2* B = Bk + (long long)x * R;
  for (int col = threadIdx.x; col < R; col += blockDim.x) {
    const int* fo = face_off + 4 * col;
    double2 t = make_double2(0, 0);
    if (x == 0 && fo[0] >= 0) t = cadd(t, g[fo[0] + k]);          // W, position k
    if (k == 0 && fo[1] >= 0) t = cadd(t, g[fo[1] + x]);          // S, position x
    if (k == n - 1 && fo[2] >= 0) t = cadd(t, g[fo[2] + x]);      // N, position x
    if (x == n - 1 && fo[3] >= 0) t = cadd(t, g[fo[3] + k]);      // E, position k
    double2 v = cmul(coeff, t);
    if (cx != 0.0) {
      const double2 y = Yp[col];
      v.x -= cx * y.x;
      v.y -= cx * y.y;
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

// Backward: B = C_k U_{k+1}.  grid (n, ncls)
__global__ void k_rhs_bwd(double2* Bk, long long bstride, const double2* Y, long long ystride,
                          const uint8_t* masks, int n, int R, double ih2, int k) {
  const int x = blockIdx.x, c = blockIdx.y;
  const uint8_t* m = masks + (long long)c * n * n;
  const double cx = coupling(m, n, k, x, ih2);
  const double2* Yn = Y + c * ystride + ((long long)(k + 1) * n + x) * R;
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

// X_k = S_k^{-1} for all rows and all classes (batched over the classes).
cudaError_t factor_blocks(Ctx& c, double2* X, long long xstride, const uint8_t* dmasks, int ncls,
                          double2* Rp, double2* Cp, long long pstride, int* dbad) {
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_gj_update, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGjUpdSmem);
  if (attr != cudaSuccess) return attr;
  const int n = c.n;
  OpParams P = op_params(c);
  for (int k = 0; k < n; ++k) {
    k_formS<<<dim3(n, ncls), 128, 0, c.stream>>>(X, xstride, dmasks, P, k);
    for (int j0 = 0; j0 < n; j0 += 32) {
      int nb = n - j0 < 32 ? n - j0 : 32;
      // Rp slice of a class: the row panel A[J, :] (32 x n), then P^{-1} (32 x 32)
      k_gj_inv<<<dim3(1 + 8, ncls), 256, 0, c.stream>>>(X, xstride, k, n, j0, nb, Rp + 32LL * n, Rp, Cp,
                                                          pstride, dbad);
      k_gj_update<<<dim3((n + 31) / 32, (n + 31) / 32, ncls), 256, kGjUpdSmem, c.stream>>>(
          X, xstride, k, n, j0, nb, Rp + 32LL * n, Rp, Cp, pstride);
    }
  }
  return cudaGetLastError();
}

void zgemm(cudaStream_t st, int M, int N, int K, double2 alpha, const double2* A, int lda,
           long long sa, const double2* B, int ldb, long long sb, double2 beta, double2* C, int ldc,
           long long sc, int batch) {
  static const bool use_dmma = !(getenv("HS_ZGEMM_FMA") && atoi(getenv("HS_ZGEMM_FMA")) != 0);
  if (use_dmma && zgemm_dmma(st, M, N, K, alpha, A, lda, sa, B, ldb, sb, beta, C, ldc, sc, batch)) return;
  dim3 grid((N + 63) / 64, (M + 63) / 64, batch);
  k_zgemm<<<grid, 256, 0, st>>>(M, N, K, alpha, A, lda, sa, B, ldb, sb, beta, C, ldc, sc);
}

// Factorisation interleaved with the forward sweep of the boundary solves:
// row k's forward step only needs X_k, so it runs on a side stream while the
// main stream factors rows k+1.. (the panel chain is latency-bound and leaves
// the GPU mostly idle); the backward sweep and the extraction follow.
// Same kernels and arithmetic as factor_blocks + solve_boundary.
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
  OpParams P = op_params(c);
  cudaStream_t side;
  cudaError_t e = cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking);
  if (e != cudaSuccess) return e;
  std::vector<cudaEvent_t> ev(n);
  for (auto& x : ev) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  cudaEvent_t start, done;
  cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&done, cudaEventDisableTiming);
  cudaEventRecord(start, c.stream);  // the side stream starts after everything queued before
  cudaStreamWaitEvent(side, start, 0);
  for (int k = 0; k < n; ++k) {
    k_formS<<<dim3(n, ncls), 128, 0, c.stream>>>(X, xstride, dmasks, P, k);
    for (int j0 = 0; j0 < n; j0 += 32) {
      int nb = n - j0 < 32 ? n - j0 : 32;
      k_gj_inv<<<dim3(1 + 8, ncls), 256, 0, c.stream>>>(X, xstride, k, n, j0, nb, Rp + 32LL * n, Rp, Cp,
                                                          pstride, dbad);
      k_gj_update<<<dim3((n + 31) / 32, (n + 31) / 32, ncls), 256, kGjUpdSmem, c.stream>>>(
          X, xstride, k, n, j0, nb, Rp + 32LL * n, Rp, Cp, pstride);
    }
    cudaEventRecord(ev[k], c.stream);  // X_k complete
    cudaStreamWaitEvent(side, ev[k], 0);
    k_rhs_fwd<<<dim3(n, ncls), rthreads, 0, side>>>(Bk, bstride, Y, ystride, dmasks, n, R, nunit, ih2, k);
    for (int cl = 0; cl < ncls; ++cl) {
      const ExtraRHS& ex = extras[cl];
      if (ex.row_ptr.empty()) continue;
      int b0 = ex.row_ptr[k], b1 = ex.row_ptr[k + 1];
      if (b1 > b0)
        k_rhs_extra<<<(b1 - b0 + 255) / 256, 256, 0, side>>>(Bk, bstride, R, ex.d_x + b0, ex.d_col + b0,
                                                              ex.d_val + b0, b1 - b0, cl);
    }
    zgemm(side, n, R, n, make_double2(1, 0), X + k * nn, n, xstride, Bk, R, bstride, make_double2(0, 0),
          Y + (long long)k * n * R, R, ystride, ncls);
  }
  cudaEventRecord(done, side);
  cudaStreamWaitEvent(c.stream, done, 0);
  for (int k = n - 2; k >= 0; --k) {
    k_rhs_bwd<<<dim3(n, ncls), rthreads, 0, c.stream>>>(Bk, bstride, Y, ystride, dmasks, n, R, ih2, k);
    zgemm(c.stream, n, R, n, make_double2(-1, 0), X + k * nn, n, xstride, Bk, R, bstride,
          make_double2(1, 0), Y + (long long)k * n * R, R, ystride, ncls);
  }
  k_extract<<<dim3(4 * n, ncls), rthreads, 0, c.stream>>>(G, gstride, Y, ystride, n, R);
  e = cudaGetLastError();
  cudaStreamSynchronize(side);  // before the side stream and its events go away
  for (auto& x : ev) cudaEventDestroy(x);
  cudaEventDestroy(start);
  cudaEventDestroy(done);
  cudaStreamDestroy(side);
  return e;
}

// Solve the factored block-tridiagonal systems for R right-hand sides and
// extract the boundary values G (4n x R) per class.
cudaError_t solve_boundary(Ctx& c, const double2* X, long long xstride, const uint8_t* dmasks,
                           int ncls, int R, int nunit, const ExtraRHS* extras, double2* Y,
                           long long ystride, double2* Bk, long long bstride, double2* G,
                           long long gstride) {
  const int n = c.n;
  const double ih2 = 1.0 / (c.h * c.h);
  const long long nn = (long long)n * n;
  const int rthreads = R < 256 ? ((R + 31) / 32) * 32 : 256;
  for (int k = 0; k < n; ++k) {
    k_rhs_fwd<<<dim3(n, ncls), rthreads, 0, c.stream>>>(Bk, bstride, Y, ystride, dmasks, n, R, nunit,
                                                        ih2, k);
    for (int cl = 0; cl < ncls; ++cl) {
      const ExtraRHS& e = extras[cl];
      if (e.row_ptr.empty()) continue;
      int b0 = e.row_ptr[k], b1 = e.row_ptr[k + 1];
      if (b1 > b0)
        k_rhs_extra<<<(b1 - b0 + 255) / 256, 256, 0, c.stream>>>(Bk, bstride, R, e.d_x + b0,
                                                                 e.d_col + b0, e.d_val + b0, b1 - b0,
                                                                 cl);
    }
    zgemm(c.stream, n, R, n, make_double2(1, 0), X + k * nn, n, xstride, Bk, R, bstride,
          make_double2(0, 0), Y + (long long)k * n * R, R, ystride, ncls);
  }
  for (int k = n - 2; k >= 0; --k) {
    k_rhs_bwd<<<dim3(n, ncls), rthreads, 0, c.stream>>>(Bk, bstride, Y, ystride, dmasks, n, R, ih2, k);
    zgemm(c.stream, n, R, n, make_double2(-1, 0), X + k * nn, n, xstride, Bk, R, bstride,
          make_double2(1, 0), Y + (long long)k * n * R, R, ystride, ncls);
  }
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
  for (int k = 0; k < n; ++k) {
    c.launches++;
    k_rhs_traces<<<n, rthreads, 0, c.stream>>>(Bk, Y, dmask, n, R, ih2, k, g, face_off, coeff);
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
  }
  for (int k = n - 2; k >= 0; --k) {
    c.launches += 2;
    k_rhs_bwd<<<dim3(n, 1), rthreads, 0, c.stream>>>(Bk, 0, Y, 0, dmask, n, R, ih2, k);
    zgemm(c.stream, n, R, n, make_double2(-1, 0), X + k * nn, n, 0, Bk, R, 0, make_double2(1, 0),
          Y + (long long)k * n * R, R, 0, 1);
  }
  return cudaGetLastError();
}

void launch_scatter_field(Ctx& c, double2* field, int nx_total, const double2* Y, int R, const int* col_ab,
                          int accumulate) {
  c.launches++;
  k_scatter_field<<<4 * c.num_sms, 256, 0, c.stream>>>(field, nx_total, Y, c.n, R, col_ab, accumulate);
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
