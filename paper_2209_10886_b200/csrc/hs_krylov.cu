// GMRES on the device: right-preconditioned, full (no restart), modified
// Gram-Schmidt Arnoldi, complex Givens rotations (the
// conventions are written out in oracle/gmres.py and mirrored here exactly).
//
// The Arnoldi step of iteration k is ONE cooperative kernel: each CTA keeps
// its slice of w = A M v_k in shared memory, and for j = 0..k computes its
// partial <v_j, w>, meets the other CTAs at a grid barrier, reduces the
// partials in a fixed order (deterministic, no atomics) and subtracts
// h_jk v_j.  HBM traffic is one read of each v_j plus one read/write of w.
// Multi-RHS (R columns, RHS fastest) runs R independent processes in lockstep
// (batched GMRES); a thread always sees the same column r = e mod R.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "hs_common.cuh"
#include "hs_kernels.h"

namespace cg = cooperative_groups;

namespace hs {

__device__ __forceinline__ long long hoff(int k, int R) { return (long long)R * ((long long)k * (k + 3) / 2); }

// Grid barrier of a cooperative launch on the context's own monotone counter
// (cooperative groups' grid.sync was bimodal per launch on B200 -- 2.2 or 5.9
// us per step with the same code, tools/allreduce_bench.cu -- while a fixed
// counter is a stable 2.2 us).  Every CTA adds 1; barrier number s of a
// launch completes at base + (s + 1) * gridDim.x (modulo 2^32).  Thread 0
// fences its own prior writes (the CTA's partials are written by thread 0
// or published to it through the bar.sync before).
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    unsigned v;
#ifdef HS_DEVICE_CHECKS
    unsigned long long spins = 0;
#endif
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
#ifdef HS_DEVICE_CHECKS
      if ((int)(v - target) < 0 && ++spins > (1ull << 28)) {
        hs_dbg_fail(DBG_GRIDBAR, __LINE__);
        break;
      }
#endif
    } while ((int)(v - target) < 0);
  }
  __syncthreads();
}

// Block-level per-column reduction: red[tid] holds a thread value, threads
// with equal tid % R share a column; P = blockDim / R is a power of two.
__device__ void block_colsum(double2* red, int R) {
  const int tid = threadIdx.x;
  for (int s = blockDim.x / 2; s >= R; s >>= 1) {
    __syncthreads();
    if (tid < s) red[tid] = cadd(red[tid], red[tid + s]);
  }
  __syncthreads();
}

// Grid-level reduction of partials[b][r] (b < nblk) into out[r] (shared),
// fixed summation order.  Uses red (blockDim) as scratch.
__device__ void grid_colsum(const double2* partials, int nblk, int R, double2* red, double2* out) {
  const int tid = threadIdx.x;
  const int r = tid % R, i = tid / R, P = blockDim.x / R;
  // four independent accumulators keep four L2 loads in flight per thread
  // (the partials are read by every CTA at every step); fixed order
  double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
  int b = i;
  for (; b + 3 * P < nblk; b += 4 * P) {
    a0 = cadd(a0, __ldcg(&partials[(long long)b * R + r]));
    a1 = cadd(a1, __ldcg(&partials[(long long)(b + P) * R + r]));
    a2 = cadd(a2, __ldcg(&partials[(long long)(b + 2 * P) * R + r]));
    a3 = cadd(a3, __ldcg(&partials[(long long)(b + 3 * P) * R + r]));
  }
  for (; b < nblk; b += P) a0 = cadd(a0, __ldcg(&partials[(long long)b * R + r]));
  const double2 acc = cadd(cadd(a0, a1), cadd(a2, a3));
  red[tid] = acc;
  block_colsum(red, R);
  if (tid < R) out[tid] = red[tid];
  __syncthreads();
}

__global__ void k_mgs(GmresDev G, int k, int chunk, unsigned* bar, unsigned bar_base) {
  unsigned nbar = 0;
  extern __shared__ double2 sm[];
  const int R = G.R;
  double2* ws = sm;                    // chunk
  double2* red = ws + chunk;           // blockDim
  double2* hsh = red + blockDim.x;     // R
  const long long LR = G.LR;
  const long long e0 = (long long)blockIdx.x * chunk;
  const int cnt = (int)max(0LL, min((long long)chunk, LR - e0));
  const int tid = threadIdx.x;
  const int nblk = gridDim.x;
  double2* w = G.V + (long long)(k + 1) * LR;
  double2* part = G.partial;
  int pb = 0;
  for (int i = tid; i < cnt; i += blockDim.x) ws[i] = w[e0 + i];
  // ||w|| before orthogonalisation (breakdown test)
  {
    double2 acc = make_double2(0, 0);
    for (int i = tid; i < cnt; i += blockDim.x) acc.x += ws[i].x * ws[i].x + ws[i].y * ws[i].y;
    red[tid] = acc;
    block_colsum(red, R);
    if (tid < R) part[(long long)pb * nblk * R + (long long)blockIdx.x * R + tid] = red[tid];
    grid_barrier(bar, bar_base + (++nbar) * (unsigned)nblk);
    grid_colsum(part + (long long)pb * nblk * R, nblk, R, red, hsh);
    if (blockIdx.x == 0 && tid < R) G.wnorm0[tid] = sqrt(hsh[tid].x);
    pb ^= 1;
  }
  double2* Hk = G.H + hoff(k, R);
  for (int j = 0; j <= k; ++j) {
    const double2* v = G.V + (long long)j * LR + e0;
    double2 acc = make_double2(0, 0);
    for (int i = tid; i < cnt; i += blockDim.x) cfma_conj(acc, v[i], ws[i]);
    red[tid] = acc;
    block_colsum(red, R);
    if (tid < R) part[(long long)pb * nblk * R + (long long)blockIdx.x * R + tid] = red[tid];
    grid_barrier(bar, bar_base + (++nbar) * (unsigned)nblk);
    grid_colsum(part + (long long)pb * nblk * R, nblk, R, red, hsh);
    pb ^= 1;
    if (blockIdx.x == 0 && tid < R) Hk[(long long)j * R + tid] = hsh[tid];
    for (int i = tid; i < cnt; i += blockDim.x) {
      const double2 h = hsh[(int)((e0 + i) % R)];
      double2 vv = v[i];
      // w = w - h v   (oracle: w - H[j,k] * V[j])
      ws[i] = csub(ws[i], cmul(h, vv));
    }
    __syncthreads();
  }
  {
    double2 acc = make_double2(0, 0);
    for (int i = tid; i < cnt; i += blockDim.x) acc.x += ws[i].x * ws[i].x + ws[i].y * ws[i].y;
    red[tid] = acc;
    block_colsum(red, R);
    if (tid < R) part[(long long)pb * nblk * R + (long long)blockIdx.x * R + tid] = red[tid];
    grid_barrier(bar, bar_base + (++nbar) * (unsigned)nblk);
    grid_colsum(part + (long long)pb * nblk * R, nblk, R, red, hsh);
  }
  if (tid < R) {
    double hn = sqrt(hsh[tid].x);
    hsh[tid].x = hn;
    if (blockIdx.x == 0) Hk[(long long)(k + 1) * R + tid] = make_double2(hn, 0);
  }
  __syncthreads();
  for (int i = tid; i < cnt; i += blockDim.x) {
    const double hn = hsh[(int)((e0 + i) % R)].x;
    w[e0 + i] = hn > 0 ? make_double2(ws[i].x / hn, ws[i].y / hn) : make_double2(0, 0);
  }
}

// Givens update of column k of right-hand side r (if still active); returns
// whether r stays active.  Hc[j * hs] is entry j of the column and cs/sn[j *
// st] the rotations of r: the global arrays, or a shared-memory copy
// (k_mgs1); the new rotation, g, history and flags always go to G.
__device__ bool givens_column_at(const GmresDev& G, int k, int r, double2* Hc, int hs, const double* csp,
                                 const double2* snp, int st) {
  const int R = G.R;
  const double eps = 2.220446049250313e-16;
  if (!G.active[r]) return false;
  const double hn = Hc[(long long)(k + 1) * hs].x;
  for (int j = 0; j < k; ++j) {
    const double c = csp[(long long)j * st];
    const double2 s = snp[(long long)j * st];
    const double2 a = Hc[(long long)j * hs], b = Hc[(long long)(j + 1) * hs];
    // t = c a + s b ;  b' = -conj(s) a + c b
    double2 t = cadd(make_double2(c * a.x, c * a.y), cmul(s, b));
    double2 sc = make_double2(-s.x, s.y);  // -conj(s)
    double2 b2 = cadd(cmul(sc, a), make_double2(c * b.x, c * b.y));
    Hc[(long long)j * hs] = t;
    Hc[(long long)(j + 1) * hs] = b2;
  }
  const double2 a = Hc[(long long)k * hs];
  const double bb = Hc[(long long)(k + 1) * hs].x;
  double c;
  double2 s;
  const double aa = hypot(a.x, a.y);
  if (aa == 0.0) {
    c = 0.0;
    s = make_double2(1.0, 0.0);
  } else {
    const double rho = hypot(aa, fabs(bb));
    c = aa / rho;
    // s = (a/|a|) * conj(b) / rho, b real
    s = make_double2(a.x / aa * bb / rho, a.y / aa * bb / rho);
  }
  G.cs[(long long)k * R + r] = c;
  G.sn[(long long)k * R + r] = s;
  Hc[(long long)k * hs] = cadd(make_double2(c * a.x, c * a.y), make_double2(s.x * bb, s.y * bb));
  Hc[(long long)(k + 1) * hs] = make_double2(0, 0);
  const double2 gk = G.g[(long long)k * R + r];
  // g[k+1] = -conj(s) g[k];  g[k] = c g[k]
  G.g[(long long)(k + 1) * R + r] = cmul(make_double2(-s.x, s.y), gk);
  G.g[(long long)k * R + r] = make_double2(c * gk.x, c * gk.y);
  const double2 gn = G.g[(long long)(k + 1) * R + r];
  const double res = hypot(gn.x, gn.y) / G.beta[r];
  G.hist[(long long)(k + 1) * R + r] = res;
  G.iters[r] = k + 1;
  if (res <= G.tol) {
    G.conv[r] = 1;
    G.active[r] = 0;
    return false;
  }
  if (hn <= 16 * eps * G.wnorm0[r]) {
    G.brk[r] = 1;
    G.active[r] = 0;
    return false;
  }
  return true;
}

__device__ bool givens_column(const GmresDev& G, int k, int r) {
  return givens_column_at(G, k, r, G.H + hoff(k, G.R) + r, G.R, G.cs + r, G.sn + r, G.R);
}

// Givens update of column k for every active right-hand side.
__global__ void k_givens(GmresDev G, int k) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < G.R; r += blockDim.x)
    if (givens_column(G, k, r)) atomicAdd(&cnt, 1);
  __syncthreads();
  if (threadIdx.x == 0) *G.nactive = cnt;
}

// Arnoldi step + Givens on one thread-block cluster (<= 16 CTAs): each CTA
// keeps its slice of w in shared memory; the per-j partial sums are exchanged
// through distributed shared memory and reduced in rank order by every CTA
// (deterministic, identical on all CTAs), with one cluster barrier per j --
// far cheaper than a grid-wide barrier for the small interface vectors of
// configs 1-3.  CTA 0 then applies the Givens rotations of column k.
__global__ void __launch_bounds__(1024) k_mgs_cluster(GmresDev G, int k, int chunk) {
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  extern __shared__ double2 sm[];
  const int R = G.R;
  double2* ws = sm;                       // chunk
  double2* red = ws + chunk;              // blockDim
  double2* pub = red + blockDim.x;        // 2 x R published partials (parity)
  double2* hsh = pub + 2 * R;             // R
  __shared__ int cnt;
  const long long LR = G.LR;
  const long long e0 = (long long)rank * chunk;
  const int n_el = (int)max(0LL, min((long long)chunk, LR - e0));
  const int tid = threadIdx.x;
  double2* w = G.V + (long long)(k + 1) * LR;
  int par = 0;
  auto exchange = [&](double2 acc) {
    // block reduce -> publish -> cluster barrier -> every CTA sums the ranks in order
    red[tid] = acc;
    block_colsum(red, R);
    if (tid < R) pub[par * R + tid] = red[tid];
    cl.sync();
    for (int r = tid; r < R; r += blockDim.x) {
      double2 s2 = make_double2(0, 0);
      for (int q = 0; q < CS; ++q) s2 = cadd(s2, cl.map_shared_rank(pub, q)[par * R + r]);
      hsh[r] = s2;
    }
    __syncthreads();
    par ^= 1;
  };
  for (int i = tid; i < n_el; i += blockDim.x) ws[i] = w[e0 + i];
  {
    double2 acc = make_double2(0, 0);
    for (int i = tid; i < n_el; i += blockDim.x) acc.x += ws[i].x * ws[i].x + ws[i].y * ws[i].y;
    exchange(acc);
    if (rank == 0 && tid < R) G.wnorm0[tid] = sqrt(hsh[tid].x);
  }
  double2* Hk = G.H + hoff(k, R);
  for (int j = 0; j <= k; ++j) {
    const double2* v = G.V + (long long)j * LR + e0;
    double2 acc = make_double2(0, 0);
    for (int i = tid; i < n_el; i += blockDim.x) cfma_conj(acc, v[i], ws[i]);
    exchange(acc);
    if (rank == 0 && tid < R) Hk[(long long)j * R + tid] = hsh[tid];
    for (int i = tid; i < n_el; i += blockDim.x) {
      const double2 h = hsh[(int)((e0 + i) % R)];
      ws[i] = csub(ws[i], cmul(h, v[i]));
    }
    __syncthreads();
  }
  {
    double2 acc = make_double2(0, 0);
    for (int i = tid; i < n_el; i += blockDim.x) acc.x += ws[i].x * ws[i].x + ws[i].y * ws[i].y;
    exchange(acc);
  }
  if (tid < R) {
    const double hn = sqrt(hsh[tid].x);
    hsh[tid].x = hn;
    if (rank == 0) Hk[(long long)(k + 1) * R + tid] = make_double2(hn, 0);
  }
  __syncthreads();
  for (int i = tid; i < n_el; i += blockDim.x) {
    const double hn = hsh[(int)((e0 + i) % R)].x;
    w[e0 + i] = hn > 0 ? make_double2(ws[i].x / hn, ws[i].y / hn) : make_double2(0, 0);
  }
  if (rank == 0) {
    if (tid == 0) cnt = 0;
    __syncthreads();
    for (int r = tid; r < R; r += blockDim.x)
      if (givens_column(G, k, r)) atomicAdd(&cnt, 1);
    __syncthreads();
    if (tid == 0) *G.nactive = cnt;
  }
  cl.sync();  // peers' shared memory must outlive the last remote read
}

// beta = ||b|| per column (two-pass deterministic), V0 = b / beta, state init.
__global__ void k_colnorm_partial(const double2* x, long long LR, int R, int chunk, double2* part) {
  extern __shared__ double2 red[];
  const long long e0 = (long long)blockIdx.x * chunk;
  const int cnt = (int)max(0LL, min((long long)chunk, LR - e0));
  double2 acc = make_double2(0, 0);
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    double2 v = x[e0 + i];
    acc.x += v.x * v.x + v.y * v.y;
  }
  red[threadIdx.x] = acc;
  block_colsum(red, R);
  if (threadIdx.x < R) part[(long long)blockIdx.x * R + threadIdx.x] = red[threadIdx.x];
}

// nblk >= 0: reduce G.partial[nblk][R]; nblk < 0: pre[r].x already holds |b_r|^2
__global__ void k_gmres_init(GmresDev G, int nblk, const double2* pre) {
  extern __shared__ double2 red[];
  double2* out = red + blockDim.x;
  if (nblk >= 0) {
    grid_colsum(G.partial, nblk, G.R, red, out);
  } else {
    for (int r = threadIdx.x; r < G.R; r += blockDim.x) out[r] = pre[r];
    __syncthreads();
  }
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int r = threadIdx.x; r < G.R; r += blockDim.x) {
    double b = sqrt(out[r].x);
    G.beta[r] = b;
    G.g[r] = make_double2(b, 0);
    G.hist[r] = 1.0;
    G.iters[r] = 0;
    G.brk[r] = 0;
    G.conv[r] = b == 0.0 ? 1 : 0;
    G.active[r] = b == 0.0 ? 0 : 1;
    if (b != 0.0) atomicAdd(&cnt, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) *G.nactive = cnt;
}

__global__ void k_scale_cols(double2* V, const double2* b, const double* beta, long long LR, int R) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < LR;
       i += (long long)gridDim.x * blockDim.x) {
    double bt = beta[i % R];
    double2 v = b[i];
    V[i] = bt > 0 ? make_double2(v.x / bt, v.y / bt) : make_double2(0, 0);
  }
}

// Back substitution H y = g (rotated, upper triangular, m = iters[r]).
__global__ void k_trisolve(GmresDev G) {
  const int R = G.R;
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    const int m = G.iters[r];
    for (int i = m - 1; i >= 0; --i) {
      double2 acc = G.g[(long long)i * R + r];
      for (int j = i + 1; j < m; ++j) {
        const double2 hij = G.H[hoff(j, R) + (long long)i * R + r];
        acc = csub(acc, cmul(hij, G.y[(long long)j * R + r]));
      }
      const double2 d = G.H[hoff(i, R) + (long long)i * R + r];
      const double den = d.x * d.x + d.y * d.y;
      G.y[(long long)i * R + r] =
          make_double2((acc.x * d.x + acc.y * d.y) / den, (acc.y * d.x - acc.x * d.y) / den);
    }
  }
}

// u = sum_{j < m_r} y_j v_j
__global__ void k_combine(GmresDev G, int mmax, double2* u) {
  const long long LR = G.LR;
  const int R = G.R;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < LR;
       e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e % R);
    const int m = G.iters[r];
    double2 acc = make_double2(0, 0);
    for (int j = 0; j < mmax && j < m; ++j) cfma(acc, G.y[(long long)j * R + r], G.V[(long long)j * LR + e]);
    u[e] = acc;
  }
}

// k_mgs1 partials [2][6][kMgs1MaxGrid] followed by the grid-barrier counter
// shared by k_mgs and k_mgs1 (same stream: launches never overlap).
static constexpr int kGridScratch = 2 * 20 * 256 + 16;  // doubles: k_mgs1 partials [2][20][256] + barrier counter
cudaError_t ensure_grid_scratch(Ctx& c) {
  if (c.mgs1_slots) return cudaSuccess;
  cudaError_t e = cudaMalloc((void**)&c.mgs1_slots, (size_t)kGridScratch * sizeof(double));
  if (e == cudaSuccess) e = cudaMemsetAsync(c.mgs1_slots, 0, (size_t)kGridScratch * sizeof(double), c.stream);
  c.mgs1_bar = 0;
  return e;
}
static unsigned* grid_bar(Ctx& c) { return (unsigned*)(c.mgs1_slots + 2 * 20 * 256); }

static int pow2_floor(int x) {
  int p = 1;
  while (p * 2 <= x) p *= 2;
  return p;
}

static int coop_block(int R) { return R * pow2_floor(1024 / R); }

int gmres_coop_grid(Ctx& c, long long LR, int R, int* chunk) {
  const int bs = coop_block(R);
  int dev = c.device;
  int per_sm = 1;
  // aim for 1 CTA per SM with <= 160 KB of w slice
  long long nb = c.num_sms;
  long long ch = (LR + nb - 1) / nb;
  ch = ((ch + R - 1) / R) * R;
  size_t smem = (size_t)(ch + bs + R) * sizeof(double2);
  if (smem > 200 * 1024) {
    per_sm = 2;
    nb = (long long)c.num_sms * 2;
    ch = ((LR + nb - 1) / nb + R - 1) / R * R;
    smem = (size_t)(ch + bs + R) * sizeof(double2);
    if (smem > 110 * 1024) return -1;
  }
  (void)dev;
  (void)per_sm;
  *chunk = (int)ch;
  return (int)((LR + ch - 1) / ch);
}

cudaError_t gmres_init(Ctx& c, GmresDev& G, const double2* b) {
  const int R = G.R;
  const int bs = coop_block(R);
  long long nb = c.num_sms * 2;
  long long ch = ((G.LR + nb - 1) / nb + R - 1) / R * R;
  int nblk = (int)((G.LR + ch - 1) / ch);
  c.launches += 3;
  k_colnorm_partial<<<nblk, bs, bs * sizeof(double2), c.stream>>>(b, G.LR, R, (int)ch, G.partial);
  k_gmres_init<<<1, bs, (bs + R) * sizeof(double2), c.stream>>>(G, nblk, nullptr);
  int g2 = (int)std::min<long long>((G.LR + 255) / 256, (long long)c.num_sms * 8);
  k_scale_cols<<<g2 > 0 ? g2 : 1, 256, 0, c.stream>>>(G.V, b, G.beta, G.LR, R);
  return cudaGetLastError();
}

// Cluster size / slice for k_mgs_cluster: the smallest power of two such that
// a CTA holds <= 12288 elements of w and has >= 2048 to stream; 0 when the
// vector is too large for one 16-CTA cluster (then the grid-wide kernel runs).
int gmres_cluster_size(long long LR, int R, int* chunk) {
  // beyond ~32k elements the k basis vectors per iteration need the whole
  // GPU's bandwidth more than cheap barriers (measured: cfg3 slower on 16 CTAs)
  if (LR > 32768) return 0;
  int cs = 1;
  while (cs < 16 && ((LR + cs - 1) / cs > 12288 || (LR + cs - 1) / cs > 2048)) cs *= 2;
  long long ch = (LR + cs - 1) / cs;
  ch = ((ch + R - 1) / R) * R;
  if (ch > 12288 + R) return 0;
  *chunk = (int)ch;
  return cs;
}

cudaError_t gmres_arnoldi_cluster(Ctx& c, GmresDev& G, int k, int cs, int chunk) {
  const int bs = coop_block(G.R);
  const size_t smem = (size_t)(chunk + bs + 3 * G.R) * sizeof(double2);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_mgs_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    cudaFuncSetAttribute(k_mgs_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  c.launches++;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(bs);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_mgs_cluster, G, k, chunk);
}

cudaError_t gmres_arnoldi(Ctx& c, GmresDev& G, int k, int grid, int chunk) {
  const int bs = coop_block(G.R);
  size_t smem = (size_t)(chunk + bs + G.R) * sizeof(double2);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_mgs, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    attr_set = true;
  }
  if (cudaError_t e = ensure_grid_scratch(c)) return e;
  unsigned* bar = grid_bar(c);
  unsigned bar_base = c.mgs1_bar;
  c.mgs1_bar += (unsigned)(k + 3) * (unsigned)grid;  // k + 3 barriers
  c.launches++;
  void* args[] = {(void*)&G, (void*)&k, (void*)&chunk, (void*)&bar, (void*)&bar_base};
  return cudaLaunchCooperativeKernel((const void*)k_mgs, dim3(grid), dim3(bs), args, smem, c.stream);
}

cudaError_t gmres_givens(Ctx& c, GmresDev& G, int k) {
  int bs = G.R < 1024 ? ((G.R + 31) / 32) * 32 : 1024;
  c.launches++;
  k_givens<<<1, bs, 0, c.stream>>>(G, k);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// MGS across row bands (and the single-GPU host-driven variant of the same
// algorithm): each rank owns whole blocks of every Krylov vector.  For every j
// one kernel applies the previous projection and forms this rank's partial
// inner products over its owned blocks (fixed-order block reduction), one
// CTA reduces the partials in a fixed order, and -- with several ranks -- one
// ncclAllReduce of R complex values makes h_jk identical on every rank, so
// the Givens rotations (k_givens) stay replicated.  No host round trip per j.

// mode 0: out = (|w|^2, <v_j, w>)            (j = 0; |w| before orthogonalisation)
// mode 1: w -= h v_{j-1}; out = <v_j, w>      (1 <= j <= k)
// mode 2: w -= h v_k; out = |w|^2
// mode 3: w /= |w| (h = allreduced |w|^2), writes H[k+1] and wnorm0 handled by caller
__global__ void k_mgs_dist(GmresDev G, const int* __restrict__ blocks, int nb, int nR, int k, int j,
                           int mode, const double2* __restrict__ h, double2* part) {
  extern __shared__ double2 red[];
  const int R = G.R;
  const long long LR = G.LR;
  double2* w = G.V + (long long)(k + 1) * LR;
  const double2* vj = G.V + (long long)j * LR;
  const double2* vp = mode == 1 ? G.V + (long long)(j - 1) * LR : (mode == 2 ? G.V + (long long)k * LR : nullptr);
  const long long total = (long long)nb * nR;
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = (long long)blocks[i / nR] * nR + i % nR;
    const int r = (int)(e % R);
    double2 x = w[e];
    if (mode == 1 || mode == 2) {
      x = csub(x, cmul(h[r], vp[e]));
      w[e] = x;
    } else if (mode == 3) {
      const double hn = sqrt(h[r].x);
      w[e] = hn > 0 ? make_double2(x.x / hn, x.y / hn) : make_double2(0, 0);
      continue;
    }
    if (mode == 0) {
      a0.x += x.x * x.x + x.y * x.y;
      cfma_conj(a1, vj[e], x);
    } else if (mode == 1) {
      cfma_conj(a1, vj[e], x);
    } else {
      a0.x += x.x * x.x + x.y * x.y;
    }
  }
  if (mode == 3) return;
  // per-column block reduction (thread's column fixed: blockDim % R == 0, nR % R == 0)
  red[threadIdx.x] = a0;
  block_colsum(red, R);
  if (threadIdx.x < R) part[(long long)blockIdx.x * 2 * R + threadIdx.x] = red[threadIdx.x];
  __syncthreads();
  red[threadIdx.x] = a1;
  block_colsum(red, R);
  if (threadIdx.x < R) part[(long long)blockIdx.x * 2 * R + R + threadIdx.x] = red[threadIdx.x];
}

// out[0..2R) = fixed-order sum of part[g][0..2R) over g < ngrid
__global__ void k_mgs_reduce(const double2* part, int ngrid, int R, double2* out) {
  for (int t = threadIdx.x; t < 2 * R; t += blockDim.x) {
    double2 s = make_double2(0, 0);
    for (int g = 0; g < ngrid; ++g) s = cadd(s, part[(long long)g * 2 * R + t]);
    out[t] = s;
  }
}

// record the allreduced values: j == 0 -> wnorm0 and H[0]; 1..k -> H[j]; j == k+1 -> H[k+1] = |w|
__global__ void k_mgs_commit(GmresDev G, int k, int j, const double2* out) {
  const int R = G.R;
  double2* Hk = G.H + hoff(k, R);
  for (int r = threadIdx.x; r < R; r += blockDim.x) {
    if (j == 0) {
      G.wnorm0[r] = sqrt(out[r].x);
      Hk[r] = out[R + r];
    } else if (j <= k) {
      Hk[(long long)j * R + r] = out[R + r];
    } else {
      Hk[(long long)(k + 1) * R + r] = make_double2(sqrt(out[r].x), 0);
    }
  }
}

cudaError_t gmres_arnoldi_dist(Ctx& c, GmresDev& G, int k, const int* blocks, int nb, double2* part,
                               double2* out, void* nccl_comm) {
  const int R = G.R;
  const int bs = coop_block(R);
  const int nR = c.n * R;
  const int grid = c.num_sms * 2;
  const size_t smem = bs * sizeof(double2);
  auto allreduce = [&]() -> cudaError_t {
    if (!nccl_comm) return cudaSuccess;
    return allreduce_sum_doubles(c, (double*)out, 4 * R, nccl_comm);
  };
  // j = 0: (|w|^2, <v_0, w>)
  c.launches += 3;
  k_mgs_dist<<<grid, bs, smem, c.stream>>>(G, blocks, nb, nR, k, 0, 0, out, part);
  k_mgs_reduce<<<1, 256, 0, c.stream>>>(part, grid, R, out);
  if (cudaError_t e = allreduce()) return e;
  k_mgs_commit<<<1, 256, 0, c.stream>>>(G, k, 0, out);
  for (int j = 1; j <= k; ++j) {
    // h_{j-1} = out[R..2R)
    c.launches += 3;
    k_mgs_dist<<<grid, bs, smem, c.stream>>>(G, blocks, nb, nR, k, j, 1, out + R, part);
    k_mgs_reduce<<<1, 256, 0, c.stream>>>(part, grid, R, out);
    if (cudaError_t e = allreduce()) return e;
    k_mgs_commit<<<1, 256, 0, c.stream>>>(G, k, j, out);
  }
  c.launches += 4;
  k_mgs_dist<<<grid, bs, smem, c.stream>>>(G, blocks, nb, nR, k, k, 2, out + R, part);
  k_mgs_reduce<<<1, 256, 0, c.stream>>>(part, grid, R, out);
  if (cudaError_t e = allreduce()) return e;
  k_mgs_commit<<<1, 256, 0, c.stream>>>(G, k, k + 1, out);
  k_mgs_dist<<<grid, bs, smem, c.stream>>>(G, blocks, nb, nR, k, k, 3, out, part);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// CGS2 Arnoldi (one RHS): classical Gram-Schmidt with one reorthogonalisation,
// h = V^H w; w -= V h; h' = V^H w; w -= V h'; H[:,k] = h + h'.  All k+1 inner
// products of a pass are formed in one kernel (one warp per basis vector, over
// this CTA's slice of the owned blocks, shuffle-reduced: no block barriers),
// reduced over CTAs in a fixed order, and -- across row bands -- summed with
// ONE allreduce per pass instead of k+1.
// part: [grid][kp1 + 1] (the extra slot: |w|^2 for the breakdown test).
// inner products for j in [jbeg, jend); j == k+1 is |w|^2
__global__ void k_cgs_dots(GmresDev G, const int* __restrict__ blocks, int nb, int n, int k, int jbeg, int jend,
                           double2* part) {
  const long long LR = G.LR;
  const double2* w = G.V + (long long)(k + 1) * LR;
  const long long total = (long long)nb * n;
  const long long per = (total + gridDim.x - 1) / gridDim.x;
  const long long i0 = blockIdx.x * per, i1 = min(total, i0 + per);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int kp1 = k + 1;
  for (int j = jbeg + warp; j < jend; j += nw) {
    double2 acc = make_double2(0, 0);
    const double2* v = G.V + (long long)(j < kp1 ? j : 0) * LR;
    for (long long i = i0 + lane; i < i1; i += 32) {
      const long long e = (long long)blocks[i / n] * n + i % n;
      const double2 x = w[e];
      if (j < kp1) cfma_conj(acc, v[e], x);
      else acc.x += x.x * x.x + x.y * x.y;
    }
    for (int o = 16; o > 0; o >>= 1) {
      acc.x += __shfl_down_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_down_sync(0xffffffffu, acc.y, o);
    }
    if (lane == 0) part[(long long)blockIdx.x * (kp1 + 1) + j] = acc;
  }
}

// out[j] = sum over CTAs of part[g][j] (fixed order), j < cnt
__global__ void k_cgs_reduce(const double2* part, int ngrid, int stride, int cnt, double2* out) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += gridDim.x * blockDim.x) {
    double2 s = make_double2(0, 0);
    for (int g = 0; g < ngrid; ++g) s = cadd(s, part[(long long)g * stride + j]);
    out[j] = s;
  }
}

// w -= sum_j h_j v_j over owned elements; pass 0 stores h, pass 1 adds h' into H[:,k]
__global__ void k_cgs_update(GmresDev G, const int* __restrict__ blocks, int nb, int n, int k, const double2* h,
                             int pass) {
  const long long LR = G.LR;
  double2* w = G.V + (long long)(k + 1) * LR;
  const long long total = (long long)nb * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = (long long)blocks[i / n] * n + i % n;
    double2 x = w[e];
    for (int j = 0; j <= k; ++j) x = csub(x, cmul(h[j], G.V[(long long)j * LR + e]));
    w[e] = x;
  }
  if (blockIdx.x == 0) {
    double2* Hk = G.H + hoff(k, 1);
    for (int j = threadIdx.x; j <= k; j += blockDim.x) Hk[j] = pass == 0 ? h[j] : cadd(Hk[j], h[j]);
    if (pass == 0 && threadIdx.x == 0) G.wnorm0[0] = sqrt(h[k + 1].x);
  }
}

// nrm2 = [h'_0 .. h'_k, |w'|^2] (pyth = 1: |w''|^2 = |w'|^2 - |h'|^2, the
// second pass's coefficients being O(eps) |w'| -- no cancellation) or
// [|w''|^2] (pyth = 0: a third reduction formed it directly)
__global__ void k_cgs_normalize(GmresDev G, const int* __restrict__ blocks, int nb, int n, int k,
                                const double2* nrm2, int pyth) {
  const long long LR = G.LR;
  double2* w = G.V + (long long)(k + 1) * LR;
  double q = pyth ? nrm2[k + 1].x : nrm2[0].x;
  if (pyth)
    for (int j = 0; j <= k; ++j) q -= nrm2[j].x * nrm2[j].x + nrm2[j].y * nrm2[j].y;
  const double hn = sqrt(q > 0 ? q : 0.0);
  const long long total = (long long)nb * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = (long long)blocks[i / n] * n + i % n;
    const double2 x = w[e];
    w[e] = hn > 0 ? make_double2(x.x / hn, x.y / hn) : make_double2(0, 0);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) G.H[hoff(k, 1) + k + 1] = make_double2(hn, 0);
}

// ---------------------------------------------------------------------------
// CGS2 with ONE reduction per iteration (arnoldi "cgs2g", the row-band
// default): pass 0's inner products also give the new Gram row, and the
// reorthogonalisation is done on the coefficients instead of a second pass,
//   h  = V^H w,  g_k = V^H v_k (the Gram row of the newest basis vector),
//   h' = V^H (w - V h) = h - G h,   c = h + h' = 2 h - G h,
//   w'' = w - V c,  ||w''||^2 = ||w||^2 - 2 Re(c^H h) + c^H G c,
// with G = V^H V kept on the device (rows added as the basis grows).  In exact
// arithmetic this is CGS2; the second pass's re-projection of w's rounding
// error (O(eps ||w||)) is what it omits.  One reduction of 2 (k + 1) + 1
// values, one pass over V for the products and one for the update (+ the
// normalisation, whose norm is already known).
// Owned element i -> vector element: the owned blocks in order (row bands), or
// the identity (blocks == nullptr: one rank owns everything).  32-bit index
// arithmetic (a 64-bit division per element dominated these passes).
__device__ __forceinline__ long long owned_elem(const int* __restrict__ blocks, int n, long long i) {
  if (!blocks) return i;
  const int ii = (int)i, q = ii / n;
  return (long long)blocks[q] * n + (ii - q * n);
}

// part: [grid][2 (k+1) + 1]: h_j, g_kj, then ||w||^2
__global__ void k_cgsg_dots(GmresDev G, const int* __restrict__ blocks, int nb, int n, int k, double2* part,
                            int stride) {
  extern __shared__ double2 sw[];  // this CTA's slice of w and v_k
  const long long LR = G.LR;
  const double2* w = G.V + (long long)(k + 1) * LR;
  const double2* vk = G.V + (long long)k * LR;
  const long long total = (long long)nb * n;
  const long long per = (total + gridDim.x - 1) / gridDim.x;
  const long long i0 = blockIdx.x * per, i1 = min(total, i0 + per);
  const int cnt = (int)max(0ll, i1 - i0);
  double2* sws = sw;
  double2* svk = sw + per;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const long long e = owned_elem(blocks, n, i0 + i);
    sws[i] = w[e];
    svk[i] = vk[e];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int kp1 = k + 1;
  for (int j = warp; j <= kp1; j += nw) {  // j = k + 1: ||w||^2
    double2 a = make_double2(0, 0), b = make_double2(0, 0);
    if (j < kp1) {
      const double2* v = G.V + (long long)j * LR;
      for (int i = lane; i < cnt; i += 32) {
        const double2 x = v[owned_elem(blocks, n, i0 + i)];
        cfma_conj(a, x, sws[i]);
        cfma_conj(b, x, svk[i]);
      }
    } else {
      for (int i = lane; i < cnt; i += 32) a.x += sws[i].x * sws[i].x + sws[i].y * sws[i].y;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a.x += __shfl_down_sync(0xffffffffu, a.x, o);
      a.y += __shfl_down_sync(0xffffffffu, a.y, o);
      b.x += __shfl_down_sync(0xffffffffu, b.x, o);
      b.y += __shfl_down_sync(0xffffffffu, b.y, o);
    }
    if (lane == 0) {
      double2* P = part + (long long)blockIdx.x * stride;
      if (j < kp1) {
        P[j] = a;
        P[kp1 + j] = b;
      } else {
        P[2 * kp1] = a;
      }
    }
  }
}

// out[j] = sum over CTAs of part[g][j]: one warp per entry, lane l summing
// partials l, l + 32, ... then a shuffle tree (a fixed order: deterministic)
__global__ void k_cgsg_reduce(const double2* __restrict__ part, int ngrid, int stride, int cnt, double2* out) {
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= cnt) return;
  double2 a = make_double2(0, 0);
  for (int g = lane; g < ngrid; g += 32) a = cadd(a, __ldcg(part + (long long)g * stride + j));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a.x += __shfl_xor_sync(0xffffffffu, a.x, o);
    a.y += __shfl_xor_sync(0xffffffffu, a.y, o);
  }
  if (lane == 0) out[j] = a;
}

// One CTA: the new Gram row, the coefficients c = 2 h - G h, the new norm by
// expansion, H[:, k] and ||w|| (breakdown test), then the Givens update of the
// column (as k_givens; fused here, the column in shared memory).
// red = [h_0..h_k, g_k0..g_kk, ||w||^2] (reduced over CTAs / ranks); Gm is the
// full Hermitian (maxit + 1)^2 Gram matrix, row-major: Gm[i ldg + j] = v_i^H v_j.
__global__ void __launch_bounds__(1024) k_cgsg_coef(GmresDev G, int k, const double2* red, double2* Gm, int ldg, double2* cbuf) {
  extern __shared__ double2 sh[];  // h, c, Gh, Gc (k+1 each), column (k+2), 2 (k+1) terms, sn, cs
  const int kp1 = k + 1;
  double2* h = sh;
  double2* cc = sh + kp1;
  double2* gh = sh + 2 * kp1;
  double2* gc = sh + 3 * kp1;
  double2* col = sh + 4 * kp1;
  double* t1 = (double*)(col + kp1 + 1);
  double* t2 = t1 + kp1;
  double2* sns = (double2*)(t1 + 2 * kp1 + 2);  // the previous rotations, staged for thread 0 (16-byte aligned)
  double* css = (double*)(sns + kp1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    css[j] = G.cs[j];
    sns[j] = G.sn[j];
  }
  for (int j = threadIdx.x; j < kp1; j += blockDim.x) {
    h[j] = red[j];
    const double2 g = red[kp1 + j];                        // v_j^H v_k
    Gm[(long long)j * ldg + k] = g;                        // G[j][k]
    Gm[(long long)k * ldg + j] = make_double2(g.x, -g.y);  // G[k][j] = conj
  }
  __syncthreads();
  // warp per row: (G x)_i = sum_j G[i][j] x_j, lanes over j (coalesced), shuffle tree
  auto matvec = [&](const double2* x, double2* y) {
    for (int i = warp; i < kp1; i += nw) {
      double2 acc = make_double2(0, 0);
      const double2* row = Gm + (long long)i * ldg;
      for (int j = lane; j < kp1; j += 32) acc = cadd(acc, cmul(row[j], x[j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (lane == 0) y[i] = acc;
    }
  };
  matvec(h, gh);
  __syncthreads();
  for (int i = threadIdx.x; i < kp1; i += blockDim.x) cc[i] = csub(make_double2(2.0 * h[i].x, 2.0 * h[i].y), gh[i]);
  __syncthreads();
  matvec(cc, gc);
  __syncthreads();
  for (int i = threadIdx.x; i < kp1; i += blockDim.x) {  // Re(c^H h), c^H G c termwise
    t1[i] = cc[i].x * h[i].x + cc[i].y * h[i].y;
    t2[i] = cc[i].x * gc[i].x + cc[i].y * gc[i].y;
    col[i] = cc[i];
    cbuf[i] = cc[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < kp1; ++i) s1 += t1[i], s2 += t2[i];  // index order: deterministic
    const double w2 = red[2 * kp1].x;
    const double q = w2 - 2.0 * s1 + s2;
    const double hn = sqrt(q > 0 ? q : 0.0);
    G.wnorm0[0] = sqrt(w2);
    col[kp1] = make_double2(hn, 0);
    cbuf[kp1] = make_double2(hn, 0);
    // the Givens update of column k on the shared copy (k_givens' arithmetic)
    *G.nactive = givens_column_at(G, k, 0, col, 1, css, sns, 1) ? 1 : 0;
  }
  __syncthreads();
  double2* Hk = G.H + hoff(k, 1);
  for (int j = threadIdx.x; j <= kp1; j += blockDim.x) Hk[j] = col[j];
}

// w'' = (w - V c) / ||w''|| over the owned elements
__global__ void k_cgsg_update(GmresDev G, const int* __restrict__ blocks, int nb, int n, int k, const double2* cbuf) {
  const long long LR = G.LR;
  double2* w = G.V + (long long)(k + 1) * LR;
  const double hn = cbuf[k + 1].x;
  const long long total = (long long)nb * n;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long e = owned_elem(blocks, n, i);
    double2 x = w[e];
    for (int j = 0; j <= k; ++j) x = csub(x, cmul(cbuf[j], G.V[(long long)j * LR + e]));
    w[e] = hn > 0 ? make_double2(x.x / hn, x.y / hn) : make_double2(0, 0);
  }
}

cudaError_t gmres_arnoldi_cgsg(Ctx& c, GmresDev& G, int k, const int* blocks, int nb, double2* part,
                               double2* red, double2* Gm, int ldg, void* nccl_comm) {
  const int grid = 2 * c.num_sms;
  const int kp1 = k + 1;
  const int cnt = 2 * kp1 + 1;
  const long long total = (long long)nb * c.n;
  const long long per = (total + grid - 1) / grid;
  const size_t smem = (size_t)2 * per * sizeof(double2);
  if (smem > 200 * 1024) return cudaErrorInvalidValue;
  static cudaError_t attr = [] {
    cudaError_t e = cudaFuncSetAttribute(k_cgsg_dots, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_cgsg_coef, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return e;
  }();
  if (attr != cudaSuccess) return attr;
  if ((size_t)(8 * kp1 + 2) * sizeof(double2) > 200 * 1024) return cudaErrorInvalidValue;
  c.launches += 4;
  k_cgsg_dots<<<grid, 256, smem, c.stream>>>(G, blocks, nb, c.n, k, part, cnt);
  k_cgsg_reduce<<<(cnt + 7) / 8, 256, 0, c.stream>>>(part, grid, cnt, cnt, red);
  if (nccl_comm) {
    if (cudaError_t e = allreduce_sum_doubles(c, (double*)red, 2 * (size_t)cnt, nccl_comm)) return e;
  }
  double2* cbuf = red + cnt;  // c (k+1) + ||w''||
  k_cgsg_coef<<<1, 1024, (size_t)(8 * kp1 + 2) * sizeof(double2), c.stream>>>(G, k, red, Gm, ldg, cbuf);
  const int ug = std::min(grid * 4, std::max(1, (int)((total + 255) / 256)));
  k_cgsg_update<<<ug, 256, 0, c.stream>>>(G, blocks, nb, c.n, k, cbuf);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// The same Gram-corrected one-reduction CGS2 for R right-hand sides on one
// rank (element e = position * R + r; every column r runs its own Arnoldi
// process with its own Gram matrix Gm[r]).  It replaces the cooperative k_mgs
// (one grid barrier, two block trees and a 148 x R partial read per CTA *per
// basis vector*: ~12 us per j at cfg4, where the vector itself streams in 2 us)
// by four launches per iteration: all inner products in one pass over V,
// one reduction over the CTAs, the coefficients per right-hand side, one
// update pass; the Givens update rides in the coefficient kernel.
//   part: [grid][2 (k+1) + 1][R]   red: [2 (k+1) + 1][R]   cbuf: [k + 2][R]
template <int NC>
__global__ void __launch_bounds__(256) k_cgsgR_dots(GmresDev G, int k, long long npos, long long per, double2* part,
                                                    int cnt) {
  extern __shared__ double2 sw[];  // this CTA's positions of w and v_k, all R columns
  const int R = G.R;
  const long long LR = G.LR;
  const double2* w = G.V + (long long)(k + 1) * LR;
  const double2* vk = G.V + (long long)k * LR;
  const long long p0 = blockIdx.x * per, p1 = min(npos, p0 + per);
  const int np = (int)max(0ll, p1 - p0);
  const int ne = np * R;
  double2* sws = sw;
  double2* svk = sw + per * R;
  for (int i = threadIdx.x; i < ne; i += blockDim.x) {
    sws[i] = w[p0 * R + i];
    svk[i] = vk[p0 * R + i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int kp1 = k + 1;
  double2* P = part + (long long)blockIdx.x * cnt * R;
  // a warp per basis vector; lane l owns columns l, l + 32, ...: no cross-lane
  // reduction, positions summed in order (deterministic)
  for (int j = warp; j <= kp1; j += nw) {  // j = k + 1: ||w||^2
    double2 a[NC], b[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) a[c] = b[c] = make_double2(0, 0);
    if (j < kp1) {
      const double2* v = G.V + (long long)j * LR + p0 * R;
      // PB positions' loads issued before their products: PB * NC 16-byte loads
      // in flight per lane (the one-position loop ran at DRAM latency per step)
      constexpr int PB = 8;
      int rr[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) rr[c] = lane + 32 * c < R ? lane + 32 * c : -1;
      for (int pq = 0; pq < np; pq += PB) {
        double2 x[PB][NC];
#pragma unroll
        for (int u = 0; u < PB; ++u)
#pragma unroll
          for (int c = 0; c < NC; ++c)
            x[u][c] = (pq + u < np && rr[c] >= 0) ? __ldg(v + (pq + u) * R + rr[c]) : make_double2(0, 0);
#pragma unroll
        for (int u = 0; u < PB; ++u) {
          if (pq + u >= np) break;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            if (rr[c] < 0) continue;
            cfma_conj(a[c], x[u][c], sws[(pq + u) * R + rr[c]]);
            cfma_conj(b[c], x[u][c], svk[(pq + u) * R + rr[c]]);
          }
        }
      }
    } else {
      for (int p = 0; p < np; ++p) {
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const int r = lane + 32 * c;
          if (r < R) {
            const double2 x = sws[p * R + r];
            a[c].x += x.x * x.x + x.y * x.y;
          }
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int r = lane + 32 * c;
      if (r >= R) continue;
      if (j < kp1) {
        P[(long long)j * R + r] = a[c];
        P[(long long)(kp1 + j) * R + r] = b[c];
      } else {
        P[(long long)2 * kp1 * R + r] = a[c];
      }
    }
  }
}

// out[e] = sum over CTAs g of part[g][e], e < total: 32 consecutive entries per
// block (coalesced), warp w sums CTAs w, w + 8, ... with four loads in flight,
// the eight warp sums added in warp order (a fixed order: deterministic)
__global__ void __launch_bounds__(256) k_cgsgR_reduce(const double2* __restrict__ part, int ngrid, long long total,
                                                      double2* out) {
  __shared__ double2 s[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long long e = (long long)blockIdx.x * 32 + lane;
  double2 a0 = make_double2(0, 0), a1 = a0, a2 = a0, a3 = a0;
  if (e < total) {
    int g = warp;
    for (; g + 24 < ngrid; g += 32) {
      a0 = cadd(a0, __ldcg(part + (long long)g * total + e));
      a1 = cadd(a1, __ldcg(part + (long long)(g + 8) * total + e));
      a2 = cadd(a2, __ldcg(part + (long long)(g + 16) * total + e));
      a3 = cadd(a3, __ldcg(part + (long long)(g + 24) * total + e));
    }
    for (; g < ngrid; g += 8) a0 = cadd(a0, __ldcg(part + (long long)g * total + e));
  }
  s[warp][lane] = cadd(cadd(a0, a1), cadd(a2, a3));
  __syncthreads();
  if (warp == 0 && e < total) {
    double2 t = s[0][lane];
#pragma unroll
    for (int q = 1; q < 8; ++q) t = cadd(t, s[q][lane]);
    out[e] = t;
  }
}

// One CTA per right-hand side r: its new Gram row, c = 2 h - G h, the new norm
// by expansion, H[:, k] and ||w|| (k_cgsg_coef's arithmetic; the Givens update
// is k_givens').  Gm: R matrices of ldg x ldg, row-major, Hermitian.
// The Givens update of the column follows in the same CTA (thread 0, as
// k_givens does per column); the CTAs count the still-active right-hand sides
// through sync[0] and a ticket sync[1] (the last one publishes the count and
// resets both).
__global__ void __launch_bounds__(256) k_cgsgR_coef(GmresDev G, int k, const double2* red, double2* Gm, int ldg,
                                                    double2* cbuf, int* sync) {
  extern __shared__ double2 sh[];  // h, c, Gh, Gc (k+1 each), 2 (k+1) terms
  const int R = G.R, r = blockIdx.x;
  const int kp1 = k + 1;
  double2* h = sh;
  double2* cc = sh + kp1;
  double2* gh = sh + 2 * kp1;
  double2* gc = sh + 3 * kp1;
  double* t1 = (double*)(sh + 4 * kp1);
  double* t2 = t1 + kp1;
  double2* Gr = Gm + (long long)r * ldg * ldg;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int j = threadIdx.x; j < kp1; j += blockDim.x) {
    h[j] = red[(long long)j * R + r];
    const double2 g = red[(long long)(kp1 + j) * R + r];   // v_j^H v_k
    Gr[(long long)j * ldg + k] = g;                        // G[j][k]
    Gr[(long long)k * ldg + j] = make_double2(g.x, -g.y);  // G[k][j] = conj
  }
  __syncthreads();
  auto matvec = [&](const double2* x, double2* y) {
    for (int i = warp; i < kp1; i += nw) {
      double2 acc = make_double2(0, 0);
      const double2* row = Gr + (long long)i * ldg;
      for (int j = lane; j < kp1; j += 32) acc = cadd(acc, cmul(row[j], x[j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
        acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
      }
      if (lane == 0) y[i] = acc;
    }
  };
  matvec(h, gh);
  __syncthreads();
  for (int i = threadIdx.x; i < kp1; i += blockDim.x) cc[i] = csub(make_double2(2.0 * h[i].x, 2.0 * h[i].y), gh[i]);
  __syncthreads();
  matvec(cc, gc);
  __syncthreads();
  double2* Hk = G.H + hoff(k, R);
  for (int i = threadIdx.x; i < kp1; i += blockDim.x) {  // Re(c^H h), c^H G c termwise
    t1[i] = cc[i].x * h[i].x + cc[i].y * h[i].y;
    t2[i] = cc[i].x * gc[i].x + cc[i].y * gc[i].y;
    cbuf[(long long)i * R + r] = cc[i];
    Hk[(long long)i * R + r] = cc[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < kp1; ++i) s1 += t1[i], s2 += t2[i];  // index order: deterministic
    const double w2 = red[(long long)2 * kp1 * R + r].x;
    const double q = w2 - 2.0 * s1 + s2;
    const double hn = sqrt(q > 0 ? q : 0.0);
    G.wnorm0[r] = sqrt(w2);
    cbuf[(long long)kp1 * R + r] = make_double2(hn, 0);
    Hk[(long long)kp1 * R + r] = make_double2(hn, 0);
    // (the column's entries above were written by this CTA's other threads before the barrier)
    const int act = givens_column(G, k, r) ? 1 : 0;
    atomicAdd(&sync[0], act);
    __threadfence();
    if (atomicAdd(&sync[1], 1) == R - 1) {
      *G.nactive = atomicAdd(&sync[0], 0);
      sync[0] = 0;
      sync[1] = 0;
    }
  }
}

// w'' = (w - V c) / ||w''||, column by column
__global__ void __launch_bounds__(256) k_cgsgR_update(GmresDev G, int k, const double2* __restrict__ cbuf) {
  const int R = G.R;
  const long long LR = G.LR;
  double2* w = G.V + (long long)(k + 1) * LR;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < LR; e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e % R);
    double2 x = w[e];
#pragma unroll 4
    for (int j = 0; j <= k; ++j) x = csub(x, cmul(cbuf[(long long)j * R + r], G.V[(long long)j * LR + e]));
    const double hn = cbuf[(long long)(k + 1) * R + r].x;
    w[e] = hn > 0 ? make_double2(x.x / hn, x.y / hn) : make_double2(0, 0);
  }
}

static int cgsgR_grid(Ctx& c) { return 2 * c.num_sms; }

bool gmres_cgsgR_ok(Ctx& c, long long LR, int R, int maxit) {
  if (R < 2 || R > 128 || LR % R) return false;
  const long long npos = LR / R, per = (npos + cgsgR_grid(c) - 1) / cgsgR_grid(c);
  if ((size_t)2 * per * R * sizeof(double2) > 200 * 1024) return false;
  if ((size_t)(5 * (maxit + 1) + 2) * sizeof(double2) > 200 * 1024) return false;
  return (double)R * (maxit + 1) * (maxit + 1) * sizeof(double2) <= 2e9;  // the Gram matrices
}

cudaError_t gmres_arnoldi_cgsgR(Ctx& c, GmresDev& G, int k, double2* part, double2* red, double2* Gm, int ldg,
                                int* sync) {
  const int grid = cgsgR_grid(c), R = G.R;
  const int kp1 = k + 1, cnt = 2 * kp1 + 1;
  const long long npos = G.LR / R, per = (npos + grid - 1) / grid;
  const size_t smem = (size_t)2 * per * R * sizeof(double2);
  static cudaError_t attr = [] {
    cudaError_t e = cudaFuncSetAttribute(k_cgsgR_dots<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_cgsgR_dots<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_cgsgR_dots<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_cgsgR_dots<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(k_cgsgR_coef, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return e;
  }();
  if (attr != cudaSuccess) return attr;
  c.launches += 4;
  switch ((R + 31) / 32) {
    case 1: k_cgsgR_dots<1><<<grid, 256, smem, c.stream>>>(G, k, npos, per, part, cnt); break;
    case 2: k_cgsgR_dots<2><<<grid, 256, smem, c.stream>>>(G, k, npos, per, part, cnt); break;
    case 3: k_cgsgR_dots<3><<<grid, 256, smem, c.stream>>>(G, k, npos, per, part, cnt); break;
    default: k_cgsgR_dots<4><<<grid, 256, smem, c.stream>>>(G, k, npos, per, part, cnt); break;
  }
  const long long total = (long long)cnt * R;
  k_cgsgR_reduce<<<(unsigned)((total + 31) / 32), 256, 0, c.stream>>>(part, grid, total, red);
  double2* cbuf = red + total;  // c (k+1 rows of R) + ||w''||
  k_cgsgR_coef<<<R, 256, (size_t)(5 * kp1 + 2) * sizeof(double2), c.stream>>>(G, k, red, Gm, ldg, cbuf, sync);
  const int ug = (int)std::min<long long>((long long)grid * 4, std::max<long long>(1, (G.LR + 255) / 256));
  k_cgsgR_update<<<ug, 256, 0, c.stream>>>(G, k, cbuf);
  return cudaGetLastError();
}

cudaError_t gmres_arnoldi_cgs2(Ctx& c, GmresDev& G, int k, const int* blocks, int nb, double2* part,
                               double2* hbuf, void* nccl_comm) {
  const int grid = 2 * c.num_sms;
  const int kp1 = k + 1;
  auto allreduce = [&](int cnt) -> cudaError_t {
    if (!nccl_comm) return cudaSuccess;
    return allreduce_sum_doubles(c, (double*)hbuf, 2 * (size_t)cnt, nccl_comm);
  };
  const int ug = std::min(grid * 4, std::max(1, (int)(((long long)nb * c.n + 255) / 256)));
  // Two reductions per iteration: pass 0 forms h and |w|^2 (breakdown test),
  // pass 1 h' and |w'|^2, and the new norm follows by Pythagoras.
  // HS_CGS2_DIRECT=1: a third reduction forms |w''|^2 directly.
  static const bool direct = getenv("HS_CGS2_DIRECT") && atoi(getenv("HS_CGS2_DIRECT")) != 0;
  for (int pass = 0; pass < 2; ++pass) {
    const int cnt = kp1 + (pass == 0 || !direct ? 1 : 0);
    c.launches += 3;
    k_cgs_dots<<<grid, 256, 0, c.stream>>>(G, blocks, nb, c.n, k, 0, cnt, part);
    k_cgs_reduce<<<(cnt + 127) / 128, 128, 0, c.stream>>>(part, grid, kp1 + 1, cnt, hbuf);
    if (cudaError_t e = allreduce(cnt)) return e;
    k_cgs_update<<<ug, 256, 0, c.stream>>>(G, blocks, nb, c.n, k, hbuf, pass);
  }
  if (direct) {  // |w|^2 -> normalise
    c.launches += 2;
    k_cgs_dots<<<grid, 256, 0, c.stream>>>(G, blocks, nb, c.n, k, kp1, kp1 + 1, part);
    k_cgs_reduce<<<1, 32, 0, c.stream>>>(part + kp1, grid, kp1 + 1, 1, hbuf);
    if (cudaError_t e = allreduce(1)) return e;
  }
  c.launches++;
  k_cgs_normalize<<<ug, 256, 0, c.stream>>>(G, blocks, nb, c.n, k, hbuf, direct ? 0 : 1);
  return cudaGetLastError();
}

// beta over owned blocks (+ allreduce), then the usual init
cudaError_t gmres_init_dist(Ctx& c, GmresDev& G, const double2* b, const int* blocks, int nb,
                            double2* part, double2* out, void* nccl_comm) {
  const int R = G.R;
  const int bs = coop_block(R);
  const int nR = c.n * R;
  const int grid = c.num_sms * 2;
  // |b|^2 via mode 2 on a scratch copy is avoidable: reuse k_mgs_dist on V[0] = b
  cudaError_t e = cudaMemcpyAsync(G.V, b, G.LR * sizeof(double2), cudaMemcpyDeviceToDevice, c.stream);
  if (e != cudaSuccess) return e;
  // mode 0 with k = -1: w = V[0], v_j = V[0] -> out[0..R) = |b|^2
  c.launches += 2;
  k_mgs_dist<<<grid, bs, bs * sizeof(double2), c.stream>>>(G, blocks, nb, nR, -1, 0, 0, out, part);
  k_mgs_reduce<<<1, 256, 0, c.stream>>>(part, grid, R, out);
  if (nccl_comm) {
    e = allreduce_sum_doubles(c, (double*)out, 4 * R, nccl_comm);
    if (e != cudaSuccess) return e;
  }
  c.launches += 2;
  k_gmres_init<<<1, bs, (bs + R) * sizeof(double2), c.stream>>>(G, -1, out);
  int g2 = (int)std::min<long long>((G.LR + 255) / 256, (long long)c.num_sms * 8);
  k_scale_cols<<<g2 > 0 ? g2 : 1, 256, 0, c.stream>>>(G.V, b, G.beta, G.LR, R);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// One right-hand side, vectors too large for one cluster (configs 3 and 5):
// k_mgs1<E>, one CTA per SM, each thread owning E elements of w in registers.
// Per j the CTA forms its partial <v_j, w>, the partials meet at one grid
// barrier and every CTA sums them in the same fixed order (deterministic,
// identical everywhere).  The update w -= h_j v_j and the next inner product
// <v_{j+1}, w> are one pass, and v_{j+2} streams into shared memory
// (cp.async, issued before step j's barrier) while the CTA waits, so each v_j
// is read from HBM once and a step costs one barrier plus one coalesced read
// of the partials.  ||w|| before orthogonalisation rides on step j = 0: k + 2
// barriers in all (k_mgs: k + 3, each with two shared-memory tree
// reductions).  CTA 0 then applies the Givens rotations from a shared-memory
// copy of the column (no k_givens).  Exchange designs measured on B200
// (tools/allreduce_bench.cu, 148 CTAs, per step): counter barrier +
// component-major partials 2.2 us; CTA-major partials 7 us; barrier-free
// tagged 64-bit words polled by every CTA 8.7 us (polling traffic); one
// collector CTA + broadcast 5.4 us.  In the Arnoldi step (tools/mgs_bench.cu):
// 3.3 us per j at L = 122880 and 4.5 us at L = 499712, against 5.0 and 8.0
// for k_mgs + k_givens.
static __device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
static __device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
static __device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

static __device__ __forceinline__ void warp_sum3(double& a, double& b, double& c) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
}

constexpr int kMgs1MaxGrid = 256;   // partials: [2 parities][kMgs1Comp components][kMgs1MaxGrid]
constexpr int kMgs1MaxM = 4;        // MGS steps per grid barrier (blocks of M basis vectors)
constexpr int kMgs1Comp = 2 * kMgs1MaxM + kMgs1MaxM * (kMgs1MaxM - 1);  // alpha (M complex) + gamma (M(M-1)/2 complex)
static_assert(kGridScratch == 2 * kMgs1Comp * kMgs1MaxGrid + 16, "grid scratch layout");
constexpr int kMgs1MaxBlock = 896;  // 72 registers per thread

template <int E, int M>
__global__ void __launch_bounds__(kMgs1MaxBlock, 1) k_mgs1(GmresDev G, int k, int chunk, int nbuf, double* slots, unsigned* bar, unsigned bar_base) {
  // M MGS steps per grid barrier (compile time: the block arrays stay in
  // registers); nbuf = 2 M slices (the pending block and the next one), or
  // 2 / 3 slices for M = 1
  constexpr int NCM = M >= 2 ? 2 * M + M * (M - 1) : 3;  // components per barrier
  static_assert(M == 1 || M == 2 || M == 4, "block size");
  extern __shared__ __align__(16) double2 sm1[];
  __shared__ double red[32][kMgs1Comp];
  __shared__ double red2[kMgs1Comp];
  const int BD = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = BD >> 5;
  auto buf = [&](int j) { return sm1 + (size_t)(j % nbuf) * chunk; };  // v_j (nbuf slices)
  double2* hs = sm1 + (size_t)nbuf * chunk;  // k + 2: the column (CTA 0)
  double2* sns = hs + (k + 2);     // k
  double* css = (double*)(sns + k);  // k
  const long long LR = G.LR;
  const long long e0 = (long long)blockIdx.x * chunk;
  const long long eend = min(e0 + (long long)chunk, LR);
  const int nblk = gridDim.x;
  double2* w = G.V + (long long)(k + 1) * LR;
  double2 wr[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const long long e = e0 + tid + (long long)i * BD;
    wr[i] = e < eend ? w[e] : make_double2(0, 0);
  }
  auto prefetch = [&](int j) {
    const double2* v = G.V + (long long)j * LR;
    double2* b = buf(j);
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const long long e = e0 + tid + (long long)i * BD;
      if (e < eend) cpa16(b + tid + i * BD, v + e);
    }
    cpa_commit();
  };
  int step = 0;
  // block sum, publish, grid barrier, collect: x[0..nc) summed over the grid
  // in a fixed order, returned identically to every thread of every CTA.
  // Partials are stored component-major so the collecting warps' loads are
  // fully coalesced (a CTA-major layout is 3.5x slower: 7 vs 2 us per step,
  // tools/allreduce_bench.cu).  Basis vectors [pf, pf + npf) are prefetched
  // while the CTA waits at the barrier.
  auto reduce = [&](double (&x)[NCM], int nc, int pf, int npf) {
    double* P = slots + (size_t)(step & 1) * kMgs1Comp * kMgs1MaxGrid;
#pragma unroll
    for (int q = 0; q < NCM; ++q)
      if (q < nc)
#pragma unroll
        for (int o = 16; o; o >>= 1) x[q] += __shfl_xor_sync(0xffffffffu, x[q], o);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < NCM; ++q)
        if (q < nc) red[wid][q] = x[q];
    __syncthreads();
    for (int q = wid; q < nc; q += nw) {  // warp q: component q over the CTA's warps
      double v = lane < nw ? red[lane][q] : 0.0;
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) P[q * kMgs1MaxGrid + blockIdx.x] = v;
    }
    // a basis vector issued here streams while the CTA waits at the barrier;
    // issued after the barrier its loads would queue ahead of the partials
    for (int j = pf; j < pf + npf; ++j) prefetch(j);
    grid_barrier(bar, bar_base + (unsigned)(step + 1) * (unsigned)nblk);
    for (int q = wid; q < nc; q += nw) {  // warp q collects component q (fixed order)
      double xs[kMgs1MaxGrid / 32];
#pragma unroll
      for (int u = 0; u < kMgs1MaxGrid / 32; ++u) {
        const int t = lane + 32 * u;
        xs[u] = t < nblk ? __ldcg(P + q * kMgs1MaxGrid + t) : 0.0;
      }
      double v = 0.0;
#pragma unroll
      for (int u = 0; u < kMgs1MaxGrid / 32; ++u) v += xs[u];
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red2[q] = v;
    }
    __syncthreads();
    ++step;
#pragma unroll
    for (int q = 0; q < NCM; ++q) x[q] = q < nc ? red2[q] : 0.0;
  };
  double x[NCM];
  // initial lead: v_0 and the first block v_1..v_M (one step per barrier: v_0..v_{nbuf-1})
  const int lead = M >= 2 ? M + 1 : nbuf;
  for (int j = 0; j < lead && j <= k; ++j) prefetch(j);
  if (blockIdx.x == 0)
    for (int j = tid; j < k; j += BD) { css[j] = G.cs[j]; sns[j] = G.sn[j]; }
  {  // v_0 landed: the groups issued after it may still be in flight
    const int later = min(lead, k + 1) - 1;
    switch (later >= 4 ? 4 : later) {
      case 4: cpa_wait<4>(); break;
      case 3: cpa_wait<3>(); break;
      case 2: cpa_wait<2>(); break;
      case 1: cpa_wait<1>(); break;
      default: cpa_wait<0>(); break;
    }
  }
  // j = 0: <v_0, w> and ||w||^2 before orthogonalisation
  {
    double2 acc = make_double2(0, 0);
    double nrm = 0;
    const double2* v0 = buf(0);
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (e0 + tid + (long long)i * BD < eend) {
        cfma_conj(acc, v0[tid + i * BD], wr[i]);
        nrm += wr[i].x * wr[i].x + wr[i].y * wr[i].y;
      }
#pragma unroll
    for (int q = 0; q < NCM; ++q) x[q] = 0.0;
    x[0] = acc.x; x[1] = acc.y; x[2] = nrm;
    reduce(x, 3, 0, 0);
  }
  double2 h = make_double2(x[0], x[1]);
  if (blockIdx.x == 0 && tid == 0) {
    G.wnorm0[0] = sqrt(x[2]);
    hs[0] = h;
  }
  double hn2 = 0;
  if constexpr (M >= 2) {
    // M MGS steps per barrier.  With the pending update w -= sum_p h_p v_p
    // (the previous block) applied, one pass forms alpha_q = <v_{a+q}, w> and
    // gamma_qr = <v_{a+q}, v_{a+r}> (r < q) for the next block; then
    //   h_{a+q} = <v_{a+q}, w - sum_{r<q} h_{a+r} v_{a+r}> = alpha_q - sum_{r<q} h_{a+r} gamma_qr,
    // exactly the MGS coefficients (rounding differs at the 1e-16 level).  The
    // last pass (no vectors left) applies the final update and forms ||w||^2.
    int pb0 = 0, pbn = 1;
    double2 hp[M];
    hp[0] = h;
#pragma unroll
    for (int q = 1; q < M; ++q) hp[q] = make_double2(0, 0);
    for (int a = 1;; a += M) {
      const int mb = max(0, min(M, k + 1 - a));
      cpa_wait<0>();  // the block (issued before the previous barrier)
      double2 al[M], ga[M * (M - 1) / 2];
#pragma unroll
      for (int q = 0; q < M; ++q) al[q] = make_double2(0, 0);
#pragma unroll
      for (int q = 0; q < M * (M - 1) / 2; ++q) ga[q] = make_double2(0, 0);
      double nrm = 0;
#pragma unroll
      for (int i = 0; i < E; ++i)
        if (e0 + tid + (long long)i * BD < eend) {
          const int o = tid + i * BD;
#pragma unroll
          for (int p = 0; p < M; ++p)
            if (p < pbn) wr[i] = csub(wr[i], cmul(hp[p], buf(pb0 + p)[o]));
          if (mb > 0) {
            double2 xv[M];
#pragma unroll
            for (int q = 0; q < M; ++q) xv[q] = q < mb ? buf(a + q)[o] : make_double2(0, 0);
#pragma unroll
            for (int q = 0; q < M; ++q)
              if (q < mb) cfma_conj(al[q], xv[q], wr[i]);
#pragma unroll
            for (int q = 1; q < M; ++q)
#pragma unroll
              for (int r = 0; r < q; ++r)
                if (q < mb) cfma_conj(ga[q * (q - 1) / 2 + r], xv[q], xv[r]);
          } else {
            nrm += wr[i].x * wr[i].x + wr[i].y * wr[i].y;
          }
        }
      int nc;
      if (mb > 0) {
#pragma unroll
        for (int q = 0; q < M; ++q) x[2 * q] = al[q].x, x[2 * q + 1] = al[q].y;
#pragma unroll
        for (int q = 0; q < M * (M - 1) / 2; ++q)
          x[2 * M + 2 * q] = ga[q].x, x[2 * M + 2 * q + 1] = ga[q].y;
        nc = NCM;
      } else {
#pragma unroll
        for (int q = 0; q < NCM; ++q) x[q] = 0.0;
        x[0] = nrm;
        nc = 1;
      }
      // the pending block's slices are free: the block after (a..) goes into them
      const int pf = a + M, npf = max(0, min(M, k + 1 - pf));
      reduce(x, nc, pf, npf);
      if (mb == 0) {
        hn2 = x[0];
        break;
      }
      double2 hb[M];
#pragma unroll
      for (int q = 0; q < M; ++q) {
        double2 v = make_double2(x[2 * q], x[2 * q + 1]);
#pragma unroll
        for (int r = 0; r < q; ++r) {
          const int g = 2 * M + 2 * (q * (q - 1) / 2 + r);
          v = csub(v, cmul(hb[r], make_double2(x[g], x[g + 1])));
        }
        hb[q] = q < mb ? v : make_double2(0, 0);
      }
      if (blockIdx.x == 0 && tid == 0)
        for (int q = 0; q < mb; ++q) hs[a + q] = hb[q];
      pb0 = a;
      pbn = mb;
#pragma unroll
      for (int q = 0; q < M; ++q) hp[q] = hb[q];
    }
  } else {
    for (int j = 0; j <= k; ++j) {
      const double2* vj = buf(j);
      const double2* vn = buf(j + 1);
      const bool more = j + 1 <= k;
      if (more) {  // v_{j+1} landed (each thread reads only what it copied); v_{j+2} may be in flight
        if (nbuf == 3 && j + 2 <= k) cpa_wait<1>(); else cpa_wait<0>();
      }
      double2 acc = make_double2(0, 0);
      double nrm = 0;
#pragma unroll
      for (int i = 0; i < E; ++i)
        if (e0 + tid + (long long)i * BD < eend) {
          wr[i] = csub(wr[i], cmul(h, vj[tid + i * BD]));  // w - H[j,k] V[j]
          if (more) cfma_conj(acc, vn[tid + i * BD], wr[i]);
          else nrm += wr[i].x * wr[i].x + wr[i].y * wr[i].y;
        }
      // v_j's slice is free: the vector nbuf steps ahead goes into it
#pragma unroll
      for (int q = 0; q < NCM; ++q) x[q] = 0.0;
      x[0] = acc.x; x[1] = acc.y; x[2] = nrm;
      reduce(x, 3, j + nbuf, j + nbuf <= k ? 1 : 0);
      if (more) {
        h = make_double2(x[0], x[1]);
        if (blockIdx.x == 0 && tid == 0) hs[j + 1] = h;
      } else {
        hn2 = x[2];
      }
    }
  }
  const double hn = sqrt(hn2);
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const long long e = e0 + tid + (long long)i * BD;
    if (e < eend) w[e] = hn > 0 ? make_double2(wr[i].x / hn, wr[i].y / hn) : make_double2(0, 0);
  }
  if (blockIdx.x == 0) {
    if (tid == 0) {
      hs[k + 1] = make_double2(hn, 0);
      *G.nactive = givens_column_at(G, k, 0, hs, 1, css, sns, 1) ? 1 : 0;
    }
    __syncthreads();
    double2* Hk = G.H + hoff(k, 1);
    for (int j = tid; j <= k + 1; j += BD) Hk[j] = hs[j];
  }
}

// Shared-memory bytes of k_mgs1 at iteration k with nbuf basis slices.
static size_t mgs1_smem(int chunk, int k, int nbuf) {
  return (size_t)nbuf * chunk * sizeof(double2) + (size_t)(k + 2) * sizeof(double2) +
         (size_t)k * (sizeof(double2) + sizeof(double));
}

static constexpr size_t kMgs1SmemMax = 220 * 1024;  // + static smem + the 1 KB per-CTA reserve <= 228 KB

int gmres_mgs1_plan(Ctx& c, long long LR, int R, int maxit, int* chunk, int* E, int* bd) {
  if (R != 1 || c.num_sms > kMgs1MaxGrid) return 0;
  const long long nb = c.num_sms;
  const long long ch = (LR + nb - 1) / nb;
  int e = 1;
  while (e < 8 && ch > (long long)e * kMgs1MaxBlock) e *= 2;
  if (ch > (long long)e * kMgs1MaxBlock) return 0;
  if (mgs1_smem((int)ch, maxit, 2) > kMgs1SmemMax) return 0;
  *chunk = (int)ch;
  *E = e;
  *bd = (int)(((ch + e - 1) / e + 31) / 32 * 32);
  return (int)((LR + ch - 1) / ch);
}

cudaError_t gmres_arnoldi1(Ctx& c, GmresDev& G, int k, int grid, int chunk, int E, int bd) {
  static cudaError_t attr = [] {
    cudaError_t e = cudaSuccess;
    for (const void* f : {(const void*)k_mgs1<1, 1>, (const void*)k_mgs1<2, 1>, (const void*)k_mgs1<4, 1>, (const void*)k_mgs1<8, 1>,
                          (const void*)k_mgs1<1, 2>, (const void*)k_mgs1<2, 2>, (const void*)k_mgs1<4, 2>, (const void*)k_mgs1<8, 2>,
                          (const void*)k_mgs1<1, 4>, (const void*)k_mgs1<2, 4>, (const void*)k_mgs1<4, 4>, (const void*)k_mgs1<8, 4>})
      if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMgs1SmemMax);
    return e;
  }();
  if (attr != cudaSuccess) return attr;
  if (cudaError_t e = ensure_grid_scratch(c)) return e;
  c.launches++;
  double* slots = (double*)c.mgs1_slots;
  unsigned* bar = grid_bar(c);
  unsigned bar_base = c.mgs1_bar;  // counter value before this launch (wraps modulo 2^32)
  // 2 M basis slices: M MGS steps per grid barrier (the pending block and the
  // next one), M = 4 where the slices fit in shared memory (L <= ~250k), else
  // 2; M = 1: two slices, one step per barrier (three measured no faster).
  // HS_MGS1_BLOCK = 1 | 2 | 4 caps M (HS_MGS1_PAIRS=0: M = 1).
  static const int mcap = [] {
    const char* p = getenv("HS_MGS1_PAIRS");
    if (p && atoi(p) == 0) return 1;
    const char* e = getenv("HS_MGS1_BLOCK");
    return e ? std::max(1, std::min(kMgs1MaxM, atoi(e))) : kMgs1MaxM;
  }();
  int M = 1;
  for (int m = mcap; m >= 2; m /= 2)
    if (mgs1_smem(chunk, k, 2 * m) <= kMgs1SmemMax) { M = m; break; }
  int nbuf = M >= 2 ? 2 * M : 2;
  const unsigned nbar = M >= 2 ? (unsigned)((k + M - 1) / M + 2) : (unsigned)(k + 2);
  c.mgs1_bar += nbar * (unsigned)grid;
  void* args[] = {(void*)&G, (void*)&k, (void*)&chunk, (void*)&nbuf, (void*)&slots, (void*)&bar, (void*)&bar_base};
  const size_t smem = mgs1_smem(chunk, k, nbuf);
  static const void* fns[3][4] = {
      {(const void*)k_mgs1<1, 1>, (const void*)k_mgs1<2, 1>, (const void*)k_mgs1<4, 1>, (const void*)k_mgs1<8, 1>},
      {(const void*)k_mgs1<1, 2>, (const void*)k_mgs1<2, 2>, (const void*)k_mgs1<4, 2>, (const void*)k_mgs1<8, 2>},
      {(const void*)k_mgs1<1, 4>, (const void*)k_mgs1<2, 4>, (const void*)k_mgs1<4, 4>, (const void*)k_mgs1<8, 4>}};
  const void* fn = fns[M == 4 ? 2 : M == 2 ? 1 : 0][E == 1 ? 0 : E == 2 ? 1 : E == 4 ? 2 : 3];
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(bd), args, smem, c.stream);
}

// One right-hand side, small vectors (configs 1 and 2, L <= 32768): k_mgs1c<E>
// runs the k_mgs1 algorithm on one thread-block cluster of CS <= 16 CTAs
// (CS = 1: a single CTA, no cluster barrier).  The per-step partials are
// exchanged through distributed shared memory -- each CTA publishes its
// partial in its own shared memory, one cluster barrier, every CTA reads the
// CS partials in rank order -- so a step costs a cluster barrier instead of a
// grid barrier.  k_mgs_cluster (any R) needs ~5 us per step for the same work
// (shared-memory tree reductions, unprefetched basis reads).
template <int E>
__global__ void __launch_bounds__(kMgs1MaxBlock, 1) k_mgs1c(GmresDev G, int k, int chunk, int nbuf) {
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks(), rank = (int)cl.block_rank();
  extern __shared__ __align__(16) double2 sm1[];
  __shared__ double red[32][kMgs1Comp];
  __shared__ double pub[2][kMgs1Comp];  // this CTA's partial, by parity (read by the cluster)
  __shared__ double tot6[kMgs1Comp];
  const int BD = blockDim.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = BD >> 5;
  const bool pairs = nbuf == 4;  // two MGS steps per cluster barrier (see k_mgs1)
  auto buf = [&](int j) { return sm1 + (size_t)(j % nbuf) * chunk; };  // v_j
  double2* hs = sm1 + (size_t)nbuf * chunk;  // k + 2: the column (rank 0)
  double2* sns = hs + (k + 2);               // k
  double* css = (double*)(sns + k);          // k
  const long long LR = G.LR;
  const long long e0 = (long long)rank * chunk;
  const long long eend = min(e0 + (long long)chunk, LR);
  double2* w = G.V + (long long)(k + 1) * LR;
  double2 wr[E];
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const long long e = e0 + tid + (long long)i * BD;
    wr[i] = e < eend ? w[e] : make_double2(0, 0);
  }
  auto prefetch = [&](int j) {
    const double2* v = G.V + (long long)j * LR;
    double2* b = buf(j);
#pragma unroll
    for (int i = 0; i < E; ++i) {
      const long long e = e0 + tid + (long long)i * BD;
      if (e < eend) cpa16(b + tid + i * BD, v + e);
    }
    cpa_commit();
  };
  int step = 0;
  const int nc = pairs ? kMgs1Comp : 3;
  auto reduce = [&](double (&x)[kMgs1Comp], int pf0, int pf1) {
    const int par = step & 1;
    warp_sum3(x[0], x[1], x[2]);
    if (pairs) warp_sum3(x[3], x[4], x[5]);
    if (lane == 0)
      for (int q = 0; q < nc; ++q) red[wid][q] = x[q];
    __syncthreads();
    if (wid == 0) {
      for (int q = 0; q < nc; ++q) x[q] = lane < nw ? red[lane][q] : 0.0;
      warp_sum3(x[0], x[1], x[2]);
      if (pairs) warp_sum3(x[3], x[4], x[5]);
      if (lane == 0)
        for (int q = 0; q < nc; ++q) {
          if (CS > 1) pub[par][q] = x[q];
          else tot6[q] = x[q];
        }
    }
    if (pf0 >= 0) prefetch(pf0);
    if (pf1 >= 0) prefetch(pf1);
    if (CS > 1) {
      cl.sync();
      if (wid == 0) {
        // rank q's partial to lane q, summed in rank order by the butterfly
        double y[kMgs1Comp] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        if (lane < CS) {
          const double* pq = cl.map_shared_rank(&pub[par][0], lane);
          for (int q = 0; q < nc; ++q) y[q] = pq[q];
        }
        warp_sum3(y[0], y[1], y[2]);
        if (pairs) warp_sum3(y[3], y[4], y[5]);
        if (lane == 0)
          for (int q = 0; q < nc; ++q) tot6[q] = y[q];
      }
    }
    __syncthreads();
    ++step;
    for (int q = 0; q < kMgs1Comp; ++q) x[q] = q < nc ? tot6[q] : 0.0;
  };
  double x[kMgs1Comp];
  const int lead = pairs ? 3 : 2;
  for (int j = 0; j < lead && j <= k; ++j) prefetch(j);
  if (rank == 0)
    for (int j = tid; j < k; j += BD) { css[j] = G.cs[j]; sns[j] = G.sn[j]; }
  {
    const int later = min(lead, k + 1) - 1;
    if (later >= 2) cpa_wait<2>(); else if (later == 1) cpa_wait<1>(); else cpa_wait<0>();
  }
  {
    double2 acc = make_double2(0, 0);
    double nrm = 0;
#pragma unroll
    for (int i = 0; i < E; ++i)
      if (e0 + tid + (long long)i * BD < eend) {
        cfma_conj(acc, buf(0)[tid + i * BD], wr[i]);
        nrm += wr[i].x * wr[i].x + wr[i].y * wr[i].y;
      }
    x[0] = acc.x; x[1] = acc.y; x[2] = nrm; x[3] = x[4] = x[5] = 0.0;
    reduce(x, -1, -1);
  }
  double2 h = make_double2(x[0], x[1]);
  if (rank == 0 && tid == 0) {
    G.wnorm0[0] = sqrt(x[2]);
    hs[0] = h;
  }
  double hn2 = 0;
  if (pairs) {
    int p0 = 0, p1 = -1;
    double2 hp0 = h, hp1 = make_double2(0, 0);
    for (int a = 1;; a += 2) {
      const int bb = a + 1;
      const bool ha = a <= k, hb = bb <= k;
      cpa_wait<0>();
      const double2* vp0 = buf(p0);
      const double2* vp1 = p1 >= 0 ? buf(p1) : vp0;
      const double2* va = buf(a);
      const double2* vb = buf(bb);
      double2 al = make_double2(0, 0), be = al, ga = al;
      double nrm = 0;
#pragma unroll
      for (int i = 0; i < E; ++i)
        if (e0 + tid + (long long)i * BD < eend) {
          const int o = tid + i * BD;
          wr[i] = csub(wr[i], cmul(hp0, vp0[o]));
          if (p1 >= 0) wr[i] = csub(wr[i], cmul(hp1, vp1[o]));
          if (ha) {
            const double2 xa = va[o];
            cfma_conj(al, xa, wr[i]);
            if (hb) {
              const double2 xb = vb[o];
              cfma_conj(be, xb, wr[i]);
              cfma_conj(ga, xb, xa);
            }
          } else {
            nrm += wr[i].x * wr[i].x + wr[i].y * wr[i].y;
          }
        }
      x[0] = al.x; x[1] = al.y; x[2] = ha ? be.x : nrm; x[3] = be.y; x[4] = ga.x; x[5] = ga.y;
      reduce(x, bb + 1 <= k ? bb + 1 : -1, bb + 2 <= k ? bb + 2 : -1);
      if (!ha) {
        hn2 = x[2];
        break;
      }
      const double2 h_a = make_double2(x[0], x[1]);
      const double2 h_b = csub(make_double2(x[2], x[3]), cmul(h_a, make_double2(x[4], x[5])));
      if (rank == 0 && tid == 0) {
        hs[a] = h_a;
        if (hb) hs[bb] = h_b;
      }
      p0 = a; hp0 = h_a;
      p1 = hb ? bb : -1; hp1 = h_b;
    }
  } else {
    for (int j = 0; j <= k; ++j) {
      const double2* vj = buf(j);
      const double2* vn = buf(j + 1);
      const bool more = j + 1 <= k;
      if (more) cpa_wait<0>();
      double2 acc = make_double2(0, 0);
      double nrm = 0;
#pragma unroll
      for (int i = 0; i < E; ++i)
        if (e0 + tid + (long long)i * BD < eend) {
          wr[i] = csub(wr[i], cmul(h, vj[tid + i * BD]));  // w - H[j,k] V[j]
          if (more) cfma_conj(acc, vn[tid + i * BD], wr[i]);
          else nrm += wr[i].x * wr[i].x + wr[i].y * wr[i].y;
        }
      x[0] = acc.x; x[1] = acc.y; x[2] = nrm; x[3] = x[4] = x[5] = 0.0;
      reduce(x, j + 2 <= k ? j + 2 : -1, -1);
      if (more) {
        h = make_double2(x[0], x[1]);
        if (rank == 0 && tid == 0) hs[j + 1] = h;
      } else {
        hn2 = x[2];
      }
    }
  }
  const double hn = sqrt(hn2);
#pragma unroll
  for (int i = 0; i < E; ++i) {
    const long long e = e0 + tid + (long long)i * BD;
    if (e < eend) w[e] = hn > 0 ? make_double2(wr[i].x / hn, wr[i].y / hn) : make_double2(0, 0);
  }
  if (rank == 0) {
    if (tid == 0) {
      hs[k + 1] = make_double2(hn, 0);
      *G.nactive = givens_column_at(G, k, 0, hs, 1, css, sns, 1) ? 1 : 0;
    }
    __syncthreads();
    double2* Hk = G.H + hoff(k, 1);
    for (int j = tid; j <= k + 1; j += BD) Hk[j] = hs[j];
  }
  if (CS > 1) cl.sync();  // peers' shared memory must outlive the last remote read
}

// Cluster size / slice for k_mgs1c: one CTA up to 2048 elements, else the
// smallest power of two <= 16 with at most 1024 elements per CTA; 0 beyond
// 32768 elements (k_mgs1 then).
int gmres_mgs1c_plan(long long LR, int R, int maxit, int* chunk, int* E, int* bd) {
  if (R != 1 || LR > 32768) return 0;
  // measured (tools/mgs_bench.cu, us per step): L = 1536: 1 CTA 1.36, 2 CTAs
  // 1.90; L = 14336: 16 CTAs 2.29, 8 CTAs 2.59, 4 CTAs 3.17
  int cs = 1;
  if (LR > 2048)
    while (cs < 16 && (LR + cs - 1) / cs > 1024) cs *= 2;
  const long long ch = (LR + cs - 1) / cs;
  int e = 1;
  while (e < 4 && ch > (long long)e * kMgs1MaxBlock) e *= 2;
  if (ch > (long long)e * kMgs1MaxBlock || mgs1_smem((int)ch, maxit, 2) > kMgs1SmemMax) return 0;
  *chunk = (int)ch;
  *E = e;
  *bd = (int)(((ch + e - 1) / e + 31) / 32 * 32);
  return cs;
}

cudaError_t gmres_arnoldi1c(Ctx& c, GmresDev& G, int k, int cs, int chunk, int E, int bd) {
  static cudaError_t attr = [] {
    cudaError_t e = cudaSuccess;
    for (const void* f : {(const void*)k_mgs1c<1>, (const void*)k_mgs1c<2>, (const void*)k_mgs1c<4>}) {
      if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMgs1SmemMax);
      if (e == cudaSuccess) e = cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    return e;
  }();
  if (attr != cudaSuccess) return attr;
  c.launches++;
  static const bool pairs_ok = [] {
    const char* e = getenv("HS_MGS1_PAIRS");
    return !e || atoi(e) != 0;
  }();
  int nbuf = pairs_ok && mgs1_smem(chunk, k, 4) <= kMgs1SmemMax ? 4 : 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(bd);
  cfg.dynamicSmemBytes = mgs1_smem(chunk, k, nbuf);
  cfg.stream = c.stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (E == 1) return cudaLaunchKernelEx(&cfg, k_mgs1c<1>, G, k, chunk, nbuf);
  if (E == 2) return cudaLaunchKernelEx(&cfg, k_mgs1c<2>, G, k, chunk, nbuf);
  return cudaLaunchKernelEx(&cfg, k_mgs1c<4>, G, k, chunk, nbuf);
}

// Back substitution for one right-hand side with m <= blockDim: thread t owns
// row t, the columns are swept from the last (entry (t, i) prefetched one
// column ahead) with one barrier per column.
__global__ void __launch_bounds__(1024) k_trisolve1(GmresDev G) {
  __shared__ double2 ysh[2];
  const int m = G.iters[0];
  const int t = threadIdx.x;
  double2 acc = t < m ? G.g[t] : make_double2(0, 0);
  double2 hcur = (m >= 1 && t <= m - 1) ? G.H[hoff(m - 1, 1) + t] : make_double2(0, 0);
  for (int i = m - 1; i >= 0; --i) {
    const double2 hnx = (i >= 1 && t <= i - 1) ? G.H[hoff(i - 1, 1) + t] : make_double2(0, 0);
    if (t == i) {
      const double den = hcur.x * hcur.x + hcur.y * hcur.y;
      const double2 y = make_double2((acc.x * hcur.x + acc.y * hcur.y) / den, (acc.y * hcur.x - acc.x * hcur.y) / den);
      ysh[i & 1] = y;
      G.y[i] = y;
    }
    __syncthreads();
    if (t < i) acc = csub(acc, cmul(hcur, ysh[i & 1]));
    hcur = hnx;
  }
}

cudaError_t gmres_finish(Ctx& c, GmresDev& G, int mmax, double2* u) {
  int bs = G.R < 1024 ? ((G.R + 31) / 32) * 32 : 1024;
  c.launches += 2;
  if (G.R == 1 && mmax <= 1024) k_trisolve1<<<1, ((mmax + 31) / 32) * 32, 0, c.stream>>>(G);
  else k_trisolve<<<1, bs, 0, c.stream>>>(G);
  int g2 = (int)std::min<long long>((G.LR + 255) / 256, (long long)c.num_sms * 8);
  k_combine<<<g2 > 0 ? g2 : 1, 256, 0, c.stream>>>(G, mmax, u);
  return cudaGetLastError();
}

}  // namespace hs

namespace hs {
// ---------------------------------------------------------------------------
// Peer-memory all-reduce of the sharded Arnoldi's inner products (replaces the
// ncclAllReduce calls: one kernel, no host involvement, fixed rank order).
// Rank r: (1) wait until every peer has consumed epoch - 2 (the previous use
// of this parity of r's area); (2) write its partials into its own area; (3)
// release-publish the epoch on its flag (system scope); (4) acquire every
// rank's flag >= epoch; (5) sum the G areas in rank order 0..G-1 -- the same
// additions on every rank, so all ranks hold bitwise the same sums; (6)
// release its consumed counter.  Peers are reached through the CUDA-IPC
// mappings of hs_peer_open (NVLink loads); the areas sit at the tail of the
// exported region.
static __device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
static __device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(256) k_peer_allreduce(PeerRedArgs a) {
  const int r = a.self >= 0 ? a.self : (int)blockIdx.x;
  for (int it = 0; it < a.repeats; ++it) {
    const unsigned e = a.epoch + (unsigned)it;
    const int par = (int)(e & 1);
    double* mine = a.data[r] + (size_t)par * kPeerRedCap;
    double* buf = a.buf[a.self >= 0 ? 0 : r] + (long long)it * a.stride;
    if (threadIdx.x == 0 && e >= 2)
      for (int g = 0; g < a.G; ++g)
        if (g != r) HS_WAIT(ld_acquire_sys(a.consumed[g]) < e - 2, 64, DBG_PEER);
    __syncthreads();
    for (int j = threadIdx.x; j < a.count; j += blockDim.x) mine[j] = buf[j];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      st_release_sys(a.flag[r] + par, e);
      for (int g = 0; g < a.G; ++g) HS_WAIT(ld_acquire_sys(a.flag[g] + par) < e, 32, DBG_PEER);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < a.count; j += blockDim.x) {
      double s = 0.0;
      for (int g = 0; g < a.G; ++g) s += __ldcv(a.data[g] + (size_t)par * kPeerRedCap + j);
      buf[j] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      st_release_sys(a.consumed[r], e);
    }
  }
}

cudaError_t launch_peer_allreduce(Ctx& c, const PeerRedArgs& a) {
  if (a.count > kPeerRedCap || a.G < 1 || a.G > kMaxRanks) return cudaErrorInvalidValue;
  c.launches++;
  if (a.self >= 0) {
    k_peer_allreduce<<<1, 256, 0, c.stream>>>(a);
    return cudaGetLastError();
  }
  // emulation: the G CTAs wait on one another -> a cooperative launch keeps them co-resident
  PeerRedArgs aa = a;
  void* args[] = {(void*)&aa};
  return cudaLaunchCooperativeKernel((const void*)k_peer_allreduce, dim3(a.G), dim3(256), args, 0, c.stream);
}
HS_DBG_ACCESSOR(hs_dbg_take_krylov)

}  // namespace hs
