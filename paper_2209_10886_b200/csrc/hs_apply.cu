// Batched step-apply kernels: every subdomain solve-application of one sweep
// step (all concurrent windows at once) as one launch.
//
// Replaces _scatter_one / restricted_apply / apply_scattering
// (interface_system.py:115-162): for each item (subdomain s, output rows
// [rlo, rhi) of its map) y = T_s[rlo:rhi, :] * g_in(s), where g_in(s) is the
// contiguous m-order slab of s's incoming blocks; each output face is routed
// to the block m(j, s) it owns (interface_system.py:128-133) with the step's
// epilogue fused in.
//
// Single right-hand side: an HBM-bound batched ZGEMV.  One CTA owns one
// 32-row strip of one map (a contiguous K*512 B run in the tile-major layout);
// lane = row, the 8 warps split the K columns, partial sums meet in shared
// memory.  Map elements are read once with 128-bit streaming loads.
#include <cuda_runtime.h>

#include <algorithm>

#include "hs_common.cuh"
#include "hs_kernels.h"

namespace hs {

template <int NW>
__global__ void __launch_bounds__(NW * 32) k_step1(const DevTile* __restrict__ tiles,
                                                   const DevItem* __restrict__ items,
                                                   const DevSub* __restrict__ subs,
                                                   const double2* __restrict__ T,
                                                   const double2* srcA, const double2* srcB, Epi e,
                                                   int n) {
  extern __shared__ double2 sm[];
  const DevTile tl = tiles[blockIdx.x];
  const DevItem it = items[tl.item];
  const DevSub sb = subs[it.s];
  const int K = sb.k * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double2* xs = sm;            // K incoming values
  double2* part = sm + K;      // NW x 32 partial sums
  const double2* x = (it.alt ? srcB : srcA) + sb.in_off;
  for (int i = threadIdx.x; i < K; i += NW * 32) xs[i] = x[i];
  __syncthreads();

  const double2* Tt = T + sb.T_off + (long long)tl.tile * K * kRowTile + lane;
  const int per = (K + NW - 1) / NW;
  const int c0 = warp * per;
  const int c1 = min(K, c0 + per);
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  int c = c0;
  for (; c + 8 <= c1; c += 8) {
    double2 t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = ld_stream(Tt + (long long)(c + u) * kRowTile);
#pragma unroll
    for (int u = 0; u < 8; u += 2) {
      cfma(a0, t[u], xs[c + u]);
      cfma(a1, t[u + 1], xs[c + u + 1]);
    }
  }
  for (; c < c1; ++c) cfma(a0, ld_stream(Tt + (long long)c * kRowTile), xs[c]);
  part[warp * 32 + lane] = cadd(a0, a1);
  __syncthreads();
  if (warp == 0) {
    double2 y = part[lane];
#pragma unroll
    for (int w = 1; w < NW; ++w) y = cadd(y, part[w * 32 + lane]);
    const int r = tl.tile * kRowTile + lane;
    if (r >= it.rlo && r < it.rhi) {
      const int q = r / n, p = r - q * n;
      const int slot = it.slot[q];
      if (slot == -1) epi_apply(e, (long long)sb.tgt[q] + p, y);
      else if (slot >= 0) e.send_up[(long long)slot * n + p] = y;
      else e.send_dn[(long long)(-slot - 2) * n + p] = y;
    }
  }
}

// ---------------------------------------------------------------------------
// The whole BSP apply (forward half, intermediate residual, backward half) as
// ONE persistent dataflow launch.  Tiles are claimed in schedule order from
// an atomic ticket; a tile first waits until every block it reads (its
// subdomain's incoming slab) or read-modify-writes (its output blocks) has
// received all the tile-writes the schedule puts before it (per-block
// completion counters), then runs exactly the k_step1 computation.  Step
// t+1 of one window therefore streams while step t of another window drains,
// and the 13-17 launches + ramps per apply disappear.  Deadlock-free: a
// dependency always points to an earlier ticket, held by a running CTA.
// Same arithmetic and summation order as k_step1 (bitwise identical result).
struct FusedArgs {
  const FusedTile* tiles;
  const DevItem* items;
  const FusedDep* deps;
  const DevSub* subs;
  const double2* T;
  const double2* r;
  double2* zL;
  double2* rp;
  double2* w;
  double2* z;
  int* done;
  int* ticket;
  int ntiles, n;
};

// RT = 32-row strips per tile (RT * K ~ 1024 columns-strips keeps the fixed
// per-tile cost -- ticket, dependency check, slab load, epilogue -- amortised).
template <int NW, int RT>
__global__ void __launch_bounds__(NW * 32) k_bsp_fused(FusedArgs a) {
  extern __shared__ double2 sm[];
  __shared__ int s_t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = a.n;
  for (;;) {
    if (threadIdx.x == 0) s_t = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int t = s_t;
    if (t >= a.ntiles) return;
    const FusedTile ft = a.tiles[t];
    const DevItem it = a.items[ft.item];
    const DevSub sb = a.subs[it.s];
    for (int d = threadIdx.x; d < ft.ndep; d += blockDim.x) {
      const FusedDep dp = a.deps[ft.dep0 + d];
      const volatile int* p = a.done + dp.block;
      while (*p < dp.count) __nanosleep(32);
    }
    __threadfence();
    __syncthreads();
    const int K = sb.k * n;
    const double2* src;
    if (ft.phase == 0) src = it.alt ? a.r : a.zL;
    else if (ft.phase == 1) src = a.zL;
    else src = it.alt ? a.rp : a.w;
    src += sb.in_off;
    double2* xs = sm;
    double2* part = sm + K;
    for (int i = threadIdx.x; i < K; i += NW * 32) xs[i] = __ldcg(src + i);
    __syncthreads();
    // strips beyond the map (RT > 1 at the last rows) are skipped
    const int nstrip = (K + kRowTile - 1) / kRowTile;
    const int s0 = ft.tile * RT;
    const double2* Tt = a.T + sb.T_off + (long long)s0 * K * kRowTile + lane;
    const int per = (K + NW - 1) / NW;
    const int c0 = warp * per;
    const int c1 = min(K, c0 + per);
    double2 acc[RT][2];
#pragma unroll
    for (int q = 0; q < RT; ++q) acc[q][0] = acc[q][1] = make_double2(0, 0);
    int c = c0;
    for (; c + 8 <= c1; c += 8) {
#pragma unroll
      for (int q = 0; q < RT; ++q) {
        if (s0 + q >= nstrip) break;
        const double2* Tq = Tt + (long long)q * K * kRowTile;
        double2 tv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) tv[u] = ld_stream(Tq + (long long)(c + u) * kRowTile);
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          cfma(acc[q][0], tv[u], xs[c + u]);
          cfma(acc[q][1], tv[u + 1], xs[c + u + 1]);
        }
      }
    }
    for (; c < c1; ++c)
#pragma unroll
      for (int q = 0; q < RT; ++q)
        if (s0 + q < nstrip) cfma(acc[q][0], ld_stream(Tt + (long long)q * K * kRowTile + (long long)c * kRowTile), xs[c]);
#pragma unroll
    for (int q = 0; q < RT; ++q) part[(q * NW + warp) * 32 + lane] = cadd(acc[q][0], acc[q][1]);
    __syncthreads();
    if (warp < RT) {
      // warp q finalises strip q: fixed-order sum over the warps' partials
      const int q = warp;
      double2 y = part[(q * NW) * 32 + lane];
#pragma unroll
      for (int ww = 1; ww < NW; ++ww) y = cadd(y, part[(q * NW + ww) * 32 + lane]);
      const int row = (s0 + q) * kRowTile + lane;
      if (row >= it.rlo && row < it.rhi) {
        const int f = row / n, p = row - f * n;
        const long long off = (long long)sb.tgt[f] + p;
        if (ft.phase == 0) {
          a.zL[off] = cadd(__ldcg(a.zL + off), y);
        } else if (ft.phase == 1) {
          const double2 zl = __ldcg(a.zL + off);
          const double2 v = csub(a.r[off], csub(zl, y));
          a.rp[off] = v;
          a.w[off] = v;
          a.z[off] = cadd(zl, v);
        } else {
          a.w[off] = cadd(__ldcg(a.w + off), y);
          a.z[off] = cadd(__ldcg(a.z + off), y);
        }
      }
      __threadfence();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      // one completion per (tile, written block); all strips' stores are fenced above
      const int r0 = max(it.rlo, s0 * kRowTile), r1 = min(it.rhi, (s0 + RT) * kRowTile);
      for (int f = r0 / n; f * n < r1; ++f) atomicAdd(a.done + sb.tgt[f] / n, 1);
    }
  }
}

// Multi right-hand side (vectors [L][R], RHS fastest): Y = T_rows * X with
// X = K x R slab.  Generic smem-tiled FP64 FMA version: 32 rows x 32 RHS per
// pass, K in chunks of 32.  (The DMMA kernel for R % 8 == 0 is k_stepR_dmma.)
__global__ void __launch_bounds__(256) k_stepR(const DevTile* __restrict__ tiles,
                                               const DevItem* __restrict__ items,
                                               const DevSub* __restrict__ subs,
                                               const double2* __restrict__ T, const double2* srcA,
                                               const double2* srcB, Epi e, int n, int R) {
  __shared__ double2 Ts[32][32];
  __shared__ double2 Xs[32][33];
  const DevTile tl = tiles[blockIdx.x];
  const DevItem it = items[tl.item];
  const DevSub sb = subs[it.s];
  const int K = sb.k * n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double2* x = (it.alt ? srcB : srcA) + (long long)sb.in_off * R;
  const double2* Tt = T + sb.T_off + (long long)tl.tile * K * kRowTile;
  const int r = tl.tile * kRowTile + lane;
  for (int r0 = 0; r0 < R; r0 += 32) {
    double2 acc[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] = make_double2(0, 0);
    for (int k0 = 0; k0 < K; k0 += 32) {
      const int kc = min(32, K - k0);
      for (int i = threadIdx.x; i < 32 * 32; i += 256) {
        int cc = i >> 5, ll = i & 31;
        Ts[cc][ll] = cc < kc ? Tt[(long long)(k0 + cc) * kRowTile + ll] : make_double2(0, 0);
        int rr = r0 + ll;
        Xs[cc][ll] = (cc < kc && rr < R) ? x[(long long)(k0 + cc) * R + rr] : make_double2(0, 0);
      }
      __syncthreads();
#pragma unroll 4
      for (int cc = 0; cc < 32; ++cc) {
        double2 t = Ts[cc][lane];
#pragma unroll
        for (int i = 0; i < 4; ++i) cfma(acc[i], t, Xs[cc][warp * 4 + i]);
      }
      __syncthreads();
    }
    if (r >= it.rlo && r < it.rhi) {
      const int q = r / n, p = r - q * n;
      const int slot = it.slot[q];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int rr = r0 + warp * 4 + i;
        if (rr >= R) continue;
        if (slot == -1) epi_apply(e, ((long long)sb.tgt[q] + p) * R + rr, acc[i]);
        else if (slot >= 0) e.send_up[((long long)slot * n + p) * R + rr] = acc[i];
        else e.send_dn[((long long)(-slot - 2) * n + p) * R + rr] = acc[i];
      }
    }
  }
}

// Epilogue for outputs received from neighbouring row bands.
__global__ void k_recv_epi(const DevRecv* __restrict__ recv, int nrecv, const double2* rdn,
                           const double2* rup, Epi e, int n, int R) {
  const long long per = (long long)n * R;
  const long long total = per * nrecv;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / per);
    const long long w = i - j * per;
    const DevRecv rv = recv[j];
    const double2* src = rv.dir == 0 ? rdn : rup;
    epi_apply(e, rv.off * R + w, src[(long long)rv.slot * per + w]);
  }
}

// Elementwise helpers over L*R elements.
__global__ void k_vec(int op, long long len, double2* o1, double2* o2, const double2* a,
                      const double2* b) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len;
       i += (long long)gridDim.x * blockDim.x) {
    switch (op) {
      case VEC_ADD: o1[i] = cadd(a[i], b[i]); break;                      // o1 = a + b
      case VEC_COPY2: o1[i] = a[i]; o2[i] = a[i]; break;                 // o1 = o2 = a
      case VEC_INIT_BWD: o1[i] = a[i]; o2[i] = cadd(b[i], a[i]); break;  // w = r, z = zL + r
    }
  }
}

// Literal seam mode: z += r on the blocks of the seam groups.
__global__ void k_seam_add(const int* __restrict__ blocks, int nb, double2* z, const double2* r,
                           int n, int R) {
  const long long per = (long long)n * R;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per * nb;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / per);
    const long long t = (long long)blocks[j] * per + (i - j * per);
    z[t] = cadd(z[t], r[t]);
  }
}

static int grid_for(long long len, int sms) {
  long long g = (len + 255) / 256;
  long long cap = (long long)sms * 8;
  return (int)(g < cap ? (g > 0 ? g : 1) : cap);
}

void launch_step(Ctx& c, const DevStep& st, const double2* srcA, const double2* srcB,
                 const Epi& e, int R) {
  if (st.ntiles > 0) {
    if (R == 1) {
      constexpr int NW = 16;  // same column split as the fused kernel (bitwise identical sums)
      size_t smem = (size_t)(st.maxK + NW * 32) * sizeof(double2);
      c.launches++;
      k_step1<NW><<<st.ntiles, NW * 32, smem, c.stream>>>(st.tiles, st.items, c.dsubs, c.T, srcA,
                                                          srcB, e, c.n);
    } else {
      c.launches++;
      k_stepR<<<st.ntiles, 256, 0, c.stream>>>(st.tiles, st.items, c.dsubs, c.T, srcA, srcB, e,
                                              c.n, R);
    }
  }
}

void launch_recv_epi(Ctx& c, const DevStep& st, const Epi& e, int R) {
  if (st.nrecv == 0) return;
  long long len = (long long)st.nrecv * c.n * R;
  c.launches++;
  k_recv_epi<<<grid_for(len, c.num_sms), 256, 0, c.stream>>>(st.recv, st.nrecv, c.recv_dn,
                                                             c.recv_up, e, c.n, R);
}

void launch_vec(Ctx& c, int op, long long len, double2* o1, double2* o2, const double2* a,
                const double2* b) {
  if (len <= 0) return;
  c.launches++;
  k_vec<<<grid_for(len, c.num_sms), 256, 0, c.stream>>>(op, len, o1, o2, a, b);
}

void launch_seam_add(Ctx& c, int dir, double2* z, const double2* r, int R) {
  if (c.n_seam[dir] == 0) return;
  long long len = (long long)c.n_seam[dir] * c.n * R;
  c.launches++;
  k_seam_add<<<grid_for(len, c.num_sms), 256, 0, c.stream>>>(c.d_seam[dir], c.n_seam[dir], z, r,
                                                             c.n, R);
}

cudaError_t set_step_smem_limit() {
  cudaFuncSetAttribute(k_bsp_fused<8, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_bsp_fused<16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_bsp_fused<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  return cudaFuncSetAttribute(k_step1<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              200 * 1024);
}

cudaError_t launch_bsp_fused(Ctx& c, const DevFused& f, const double2* r, double2* zL, double2* rp,
                             double2* w, double2* z) {
  // variant: 0 = 8 warps x 1 strip, 1 = 16 warps x 1 strip, 2 = 8 warps x 2 strips
  const int var = f.rt == 2 ? 2 : (f.nw == 16 ? 1 : 0);
  const int NWv = var == 1 ? 16 : 8;
  const size_t smem = (size_t)(f.maxK + NWv * 32 * f.rt) * sizeof(double2);
  static int per_sm[3] = {0, 0, 0};
  static size_t per_sm_smem[3] = {0, 0, 0};
  if (per_sm[var] == 0 || per_sm_smem[var] != smem) {
    if (var == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[var], k_bsp_fused<8, 2>, 256, smem);
    else if (var == 1) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[var], k_bsp_fused<16, 1>, 512, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[var], k_bsp_fused<8, 1>, 256, smem);
    per_sm_smem[var] = smem;
    if (per_sm[var] < 1) per_sm[var] = 1;
  }
  cudaError_t e = cudaMemsetAsync(f.counters, 0, (c.plan.npairs + 1) * sizeof(int), c.stream);
  if (e != cudaSuccess) return e;
  FusedArgs a;
  a.tiles = f.tiles; a.items = f.items; a.deps = f.deps; a.subs = c.dsubs; a.T = c.T;
  a.r = r; a.zL = zL; a.rp = rp; a.w = w; a.z = z;
  a.done = f.counters; a.ticket = f.counters + c.plan.npairs;
  a.ntiles = f.ntiles; a.n = c.n;
  const int grid = std::max(1, std::min(f.ntiles, per_sm[var] * c.num_sms));
  c.launches++;
  if (var == 2) k_bsp_fused<8, 2><<<grid, 256, smem, c.stream>>>(a);
  else if (var == 1) k_bsp_fused<16, 1><<<grid, 512, smem, c.stream>>>(a);
  else k_bsp_fused<8, 1><<<grid, 256, smem, c.stream>>>(a);
  return cudaGetLastError();
}

}  // namespace hs
