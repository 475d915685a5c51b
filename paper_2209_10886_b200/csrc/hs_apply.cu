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

#include <cstdio>
#include <cstdlib>
#include <vector>

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

  // column c belongs to warp (c % 32) / (32 / NW) and accumulator c & 1: the
  // order of the TMA-staged fused kernel, which consumes 32-column chunks
  const double2* Tt = T + sb.T_off + (long long)tl.tile * K * kRowTile + lane;
  const unsigned long long pol = l2_evict_first();
  constexpr int CPW = 32 / NW;
  double2 a0 = make_double2(0, 0), a1 = make_double2(0, 0);
  constexpr int U = 8 / CPW;  // chunks per unrolled batch: 8 loads in flight
  const int nch = (K + 31) / 32;
  int ch = 0;
  for (; ch + U <= nch && (ch + U) * 32 <= K; ch += U) {
    double2 t[U][CPW];
#pragma unroll
    for (int v = 0; v < U; ++v)
#pragma unroll
      for (int u = 0; u < CPW; ++u) t[v][u] = ld_stream(Tt + (long long)((ch + v) * 32 + warp * CPW + u) * kRowTile, pol);
#pragma unroll
    for (int v = 0; v < U; ++v)
#pragma unroll
      for (int u = 0; u < CPW; ++u) {
        const int col = (ch + v) * 32 + warp * CPW + u;
        if (col & 1) cfma(a1, t[v][u], xs[col]);
        else cfma(a0, t[v][u], xs[col]);
      }
  }
  for (; ch < nch; ++ch)
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
      const int col = ch * 32 + warp * CPW + u;
      if (col < K) {
        if (col & 1) cfma(a1, ld_stream(Tt + (long long)col * kRowTile, pol), xs[col]);
        else cfma(a0, ld_stream(Tt + (long long)col * kRowTile, pol), xs[col]);
      }
    }
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
// Row-band ranks (multi-rank instantiations, MR): every block lives -- all its
// vectors and its completion counter -- on its owner rank; a tile reads its
// subdomain's slab on its own rank and writes its output blocks, and signals
// their counters, on the owners' ranks (peer memory across GPUs).  self >= 0:
// all CTAs are that rank (one GPU per rank); self < 0: CTA c emulates rank
// c % G on one GPU (one launch over all ranks' data).
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
  double2* wout;  // phase 3 output (I - S) z (GMRES: the next basis vector), else null
  int* done;
  int* ticket;
  int ntiles, n, maxK;
  int nv;  // slab vectors per tile at most (shared-memory layout)
  unsigned long long* trace;  // per ticket: claim, inputs ready, map streamed, signalled (globaltimer ns), sm<<32|tile
  int direct_signal;          // TMA kernel: warp 0 signals itself (latency-bound plans), else the signaller warp
  int map_keep;               // maps re-read by many tiles (aliased per-kind maps): keep them in L2
  double2* split_buf;         // split-K partial sums [pair][half][32 rows][2]
  int* split_cnt;             // split-K arrivals per pair (odd arrival combines)
  MultiRankArgs mr;
  long long L = 0, T_elems = 0;  // bounds of the device checks (debug library)
  int prefetch = 0;              // k_bsp_tma: L2-prefetch each tile's chunks beyond the ring at its claim
  int nitems = 0, nsub = 0, npairs = 0;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}

// Rank view of a CTA: its tile list and the owner-rank addressing of blocks.
template <bool MR>
struct RankView {
  const FusedArgs& a;
  int cr;
  __device__ explicit RankView(const FusedArgs& args)
      : a(args), cr(MR ? (args.mr.self >= 0 ? args.mr.self : (int)(blockIdx.x % args.mr.G)) : 0) {}
  __device__ const FusedTile* tiles() const { return MR ? a.mr.tiles[cr] : a.tiles; }
  __device__ int* ticket() const { return MR ? a.mr.ticket[cr] : a.ticket; }
  __device__ int ntiles() const { return MR ? a.mr.ntiles[cr] : a.ntiles; }
  __device__ int owner(int block) const { return MR ? a.mr.blk_rank[block] : 0; }
  __device__ int* done(int block) const { return (MR ? a.mr.done[owner(block)] : a.done) + block; }
  __device__ int* wdone(int block) const { return a.mr.wdone[owner(block)] + block; }
  // completion count a dependency waits for (epoch protocol: counters accumulate)
  __device__ int target(const FusedDep& dp) const {
    return MR && a.mr.epoch ? dp.count + (int)(a.mr.epoch - 1) * a.mr.wtot[dp.block] : dp.count;
  }
  // epoch protocol: wait until every rank has posted this apply's inputs
  __device__ void wait_inputs() const {
    if (!MR || !a.mr.epoch) return;
    for (int g = 0; g < a.mr.G; ++g) {
      const volatile int* f = a.mr.inflag[g];
      while (*f < (int)a.mr.epoch) __nanosleep(64);
    }
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  }
  // epoch protocol: this rank's blocks have received every write of this apply
  // (some come from other ranks' tiles); threads [i0, +stride) share the list
  __device__ void drain(int i0, int stride) const {
    if (!MR || !a.mr.epoch) return;
    for (int i = i0; i < a.mr.n_own; i += stride) {
      const int b = a.mr.own_blocks[i];
      const volatile int* p = a.mr.done[cr] + b;
      const int want = (int)a.mr.epoch * a.mr.wtot[b];
      while (*p < want) __nanosleep(64);
      if (a.mr.ims_epoch && a.mr.wwtot) {  // A M v: the wout rows other ranks write
        const volatile int* q = a.mr.wdone[cr] + b;
        const int wq = (int)a.mr.ims_epoch * a.mr.wwtot[b];
        while (*q < wq) __nanosleep(64);
      }
    }
    asm volatile("fence.acq_rel.sys;" ::: "memory");
  }
  __device__ double2* vec(int k, int rk) const {
    if (MR) return a.mr.v[k][rk];
    switch (k) {
      case FV_R: return const_cast<double2*>(a.r);
      case FV_ZL: return a.zL;
      case FV_RP: return a.rp;
      case FV_W: return a.w;
      case FV_Z: return a.z;
      default: return a.wout;
    }
  }
  // release (a tile's stores before its signals) / acquire (the producers'
  // stores before a tile's reads) -- acq_rel, not the sequentially consistent
  // __threadfence(); system scope when the owners are other GPUs
  __device__ void fence() const {
    if (MR && a.mr.self >= 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
    else asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
};

// Epilogue operands of one output row (phase table in hs_ctx.h), fetched
// before the tile's products are needed: o = the output block's rank, off =
// element offset, low = the row feeds a lower neighbour (W/S face), zr = zL
// of the output face not yet written (read r).
template <bool MR>
__device__ __forceinline__ void epi_fetch(const RankView<MR>& rv, int phase, int flags, bool low, bool zr, int o,
                                          long long off, double2& e1, double2& e2, double2& e3) {
  const double2* r_o = rv.vec(FV_R, o);
  const double2* zb = zr ? r_o : rv.vec(FV_ZL, o);
  switch (phase) {
    case 0: e1 = __ldcg(zb + off); break;
    case 1: e1 = __ldcg(zb + off); e2 = r_o[off]; break;
    case 2:
      if (low) { e1 = __ldcg(rv.vec(FV_W, o) + off); e2 = __ldcg(rv.vec(FV_Z, o) + off); }
      if (flags & FT_WOUT) e3 = r_o[off];
      break;
    case 3: e1 = __ldcg(rv.vec(FV_Z, o) + off); break;
    case 4:
      if (low) e1 = __ldcg(zb + off);
      e2 = r_o[off];
      break;
    default:
      e1 = r_o[off];
      if (low && !(flags & FT_DIFF)) { e2 = __ldcg(rv.vec(FV_RP, o) + off); e3 = __ldcg(rv.vec(FV_W, o) + off); }
  }
}

template <bool MR>
__device__ __forceinline__ void epi_store(const RankView<MR>& rv, int phase, int flags, bool low, int o, long long off,
                                          double2 y1, double2 y2, double2 e1, double2 e2, double2 e3) {
  const double2 zero = make_double2(0, 0);
  switch (phase) {
    case 0: {
      const double2 zn = cadd(e1, y1);
      rv.vec(FV_ZL, o)[off] = zn;
      if (flags & FT_ZERO) {  // r' = 0 exactly: the window's substitution was exact here
        rv.vec(FV_RP, o)[off] = zero;
        rv.vec(FV_W, o)[off] = zero;
        rv.vec(FV_Z, o)[off] = zn;
      }
      break;
    }
    case 1: {
      const double2 v = (flags & FT_DIFF) ? y1 : csub(e2, csub(e1, y1));  // T_up (zL - r), or r - (zL - S zL)
      rv.vec(FV_RP, o)[off] = v;
      rv.vec(FV_W, o)[off] = v;
      rv.vec(FV_Z, o)[off] = cadd(e1, v);
      break;
    }
    case 2:
      if (low) {
        rv.vec(FV_W, o)[off] = cadd(e1, y1);
        rv.vec(FV_Z, o)[off] = cadd(e2, y1);
        if (flags & FT_WOUT) rv.vec(FV_WOUT, o)[off] = e3;
      } else {
        rv.vec(FV_WOUT, o)[off] = csub(e3, y1);
      }
      break;
    case 3: rv.vec(FV_WOUT, o)[off] = csub(e1, y1); break;  // EPI_IMS on the final z
    case 4:
      if (low) {
        const double2 v = csub(e2, csub(e1, y1));
        rv.vec(FV_RP, o)[off] = v;
        rv.vec(FV_W, o)[off] = cadd(v, y2);
        rv.vec(FV_Z, o)[off] = cadd(cadd(e1, v), y2);
        if (flags & FT_WOUT) rv.vec(FV_WOUT, o)[off] = e2;
      } else {
        rv.vec(FV_WOUT, o)[off] = csub(e2, y2);
      }
      break;
    default:
      rv.vec(FV_WOUT, o)[off] = (low && !(flags & FT_DIFF)) ? cadd(csub(e1, e2), csub(e3, y1)) : csub(e1, y1);
  }
}

// Slab value i of a tile: X1 (r where zL is not written yet, bit q of rmask),
// zero outside the item's column range; FT_DIFF subtracts r (phase 1) or rp
// (phase 5).
template <bool MR>
__device__ __forceinline__ double2 slab_value(const RankView<MR>& rv, int cr, const double2* x1, const double2* rsrc,
                                              int i, int n, int rmask, int c0, int c1, int phase, int flags,
                                              int in_off) {
  if (i < c0 || i >= c1) return make_double2(0, 0);
  double2 v = __ldcg(((rmask >> (i / n)) & 1 ? rsrc : x1) + i);
  if (flags & FT_DIFF) v = csub(v, __ldcg((phase == 1 ? rsrc : rv.vec(FV_RP, cr) + in_off) + i));
  return v;
}

// Slab sources of a tile: X1 (and X2 for phase 4) on this CTA's rank.
template <bool MR>
__device__ __forceinline__ void slab_srcs(const RankView<MR>& rv, int phase, int alt, int cr, const double2*& x1,
                                          const double2*& x2) {
  x2 = nullptr;
  switch (phase) {
    case 0: x1 = rv.vec(alt ? FV_R : FV_ZL, cr); break;
    case 1: x1 = rv.vec(FV_ZL, cr); break;
    case 2: x1 = rv.vec(alt ? FV_RP : FV_W, cr); break;
    case 3: x1 = rv.vec(FV_Z, cr); break;
    case 4: x1 = rv.vec(FV_ZL, cr); x2 = rv.vec(alt ? FV_RP : FV_W, cr); break;
    default: x1 = rv.vec(FV_W, cr);
  }
}

// Signal the blocks a tile completed (phases 0-2 and 4; lower faces only for
// phases 2 and 4, whose upper rows write wout).  One fence by the signalling
// thread publishes the epilogue stores the barrier ordered before it
// (cumulativity), instead of a fence per storing lane.
// Row bands with the epoch protocol also count the wout writes (phases 3 and
// 5, phases 2 / 4 with FT_WOUT) per block, so the owner can drain them.
// phase < 0: nothing (the first half of a split-K pair).
template <bool MR>
__device__ __forceinline__ void tile_signal(const RankView<MR>& rv, int phase, int flags, int r0, int r1, int n,
                                            int nlow, const int* tgt) {
  if (phase < 0) return;
  const bool wout = phase == 3 || phase == 5 || ((phase == 2 || phase == 4) && (flags & FT_WOUT));
  const bool counts = MR && wout && rv.a.mr.wdone[0] != nullptr;
  if ((phase == 3 || phase == 5) && !counts) return;
  rv.fence();
  for (int f = r0 / n; f * n < r1; ++f) {
    if (phase <= 1 || ((phase == 2 || phase == 4) && f < nlow)) atomicAdd(rv.done(tgt[f] / n), 1);
    if (counts) atomicAdd(rv.wdone(tgt[f] / n), 1);
  }
}

// Register-streaming contraction of RT strips with NV slab vectors (xs,
// xs + K); column c into warp (c % 32) / (32 / NW), accumulator c & 1.
template <int NW, int RT, int NV>
__device__ __forceinline__ void contract_regs(const double2* __restrict__ Tt, const double2* xs, int K, int nstrip,
                                              int s0, int warp, int ch0, int nch, double2 (&acc)[RT][NV][2]) {
  constexpr int CPW = 32 / NW;
  constexpr int U = 8 / CPW;  // chunks per unrolled batch: 8 loads in flight per strip
  const unsigned long long pol = l2_evict_first();
#pragma unroll
  for (int q = 0; q < RT; ++q)
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[q][v][0] = acc[q][v][1] = make_double2(0, 0);
  int ch = ch0;
  for (; ch + U <= nch && (ch + U) * 32 <= K; ch += U) {
#pragma unroll
    for (int q = 0; q < RT; ++q) {
      if (s0 + q >= nstrip) break;
      const double2* Tq = Tt + (long long)q * K * kRowTile;
      double2 tv[U][CPW];
#pragma unroll
      for (int v = 0; v < U; ++v)
#pragma unroll
        for (int u = 0; u < CPW; ++u) tv[v][u] = ld_stream(Tq + (long long)((ch + v) * 32 + warp * CPW + u) * kRowTile, pol);
#pragma unroll
      for (int v = 0; v < U; ++v)
#pragma unroll
        for (int u = 0; u < CPW; ++u) {
          const int col = (ch + v) * 32 + warp * CPW + u;
#pragma unroll
          for (int x = 0; x < NV; ++x) cfma(acc[q][x][col & 1], tv[v][u], xs[x * K + col]);
        }
    }
  }
  for (; ch < nch; ++ch)
#pragma unroll
    for (int u = 0; u < CPW; ++u) {
      const int col = ch * 32 + warp * CPW + u;
      if (col < K)
#pragma unroll
        for (int q = 0; q < RT; ++q)
          if (s0 + q < nstrip) {
            const double2 t = ld_stream(Tt + (long long)q * K * kRowTile + (long long)col * kRowTile, pol);
#pragma unroll
            for (int x = 0; x < NV; ++x) cfma(acc[q][x][col & 1], t, xs[x * K + col]);
          }
    }
}

// RT = 32-row strips per tile (RT * K ~ 1024 columns-strips keeps the fixed
// per-tile cost -- ticket, dependency check, slab load, epilogue -- amortised).
// 6 CTAs of 8 warps per SM for the one-strip form: the map stream needs the
// bytes in flight (5 CTAs per SM measured ~10 % slower at cfg5).  Phase-4
// tiles (map-once plan, RT = 1) multiply two slab vectors per map read.
template <int NW, int RT, bool MR>
__global__ void __launch_bounds__(NW * 32, RT == 1 ? 6 : 1) k_bsp_fused(FusedArgs a) {
  extern __shared__ double2 sm[];
  __shared__ int s_t;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int n = a.n;
  const RankView<MR> rv(a);
  const int cr = rv.cr;
  const FusedTile* tiles = rv.tiles();
  const int ntiles = rv.ntiles();
  if (threadIdx.x == 0) rv.wait_inputs();
  __syncthreads();
  for (;;) {
    if (threadIdx.x == 0) s_t = atomicAdd(rv.ticket(), 1);
    __syncthreads();
    const int t = s_t;
    if (t >= ntiles) {
      rv.drain(blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
      return;
    }
    unsigned long long* tr = (a.trace && !MR) ? a.trace + 6ll * t : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = tr[1] = gtimer();
    const FusedTile ft = tiles[t];
    HS_DCHECK(ft.item >= 0 && ft.item < a.nitems, DBG_INDEX);
    const DevItem it = a.items[ft.item];
    HS_DCHECK(it.s >= 0 && it.s < a.nsub, DBG_INDEX);
    const DevSub sb = a.subs[it.s];
    HS_DCHECK(sb.T_off >= 0 && sb.T_off + (long long)sb.k * n * ((sb.k * n + kRowTile - 1) / kRowTile * kRowTile) <= a.T_elems,
              DBG_MAP);
    HS_DCHECK(sb.in_off >= 0 && sb.in_off + (long long)sb.k * n <= a.L, DBG_VEC);
    for (int d = threadIdx.x; d < ft.ndep; d += blockDim.x) {
      const FusedDep dp = a.deps[ft.dep0 + d];
      HS_DCHECK(dp.block >= 0 && dp.block < a.npairs, DBG_COUNTER);
      const volatile int* p = rv.done(dp.block);
      HS_WAIT(*p < rv.target(dp), 32, DBG_DEPWAIT);
    }
    rv.fence();  // acquire: the producers' stores before this CTA's reads
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[2] = gtimer();
    const int K = sb.k * n;
    const int nv = (RT == 1 && ft.phase == 4) ? 2 : 1;
    // the slab (this subdomain's incoming blocks) lives on this CTA's rank
    const double2 *x1, *x2;
    slab_srcs(rv, ft.phase, it.alt, cr, x1, x2);
    x1 += sb.in_off;
    const double2* rsrc = rv.vec(FV_R, cr) + sb.in_off;
    double2* xs = sm;
    // the partial sums reuse the slab's shared memory once every warp is done
    // with it (one barrier): 6 CTAs per SM fit with two 1024-column slabs
    double2* part = sm;
    // zL starts as r without a copy: faces of zL not yet written read r
    for (int i = threadIdx.x; i < K; i += NW * 32)
      xs[i] = slab_value(rv, cr, x1, rsrc, i, n, ft.rmask, ft.c0, ft.c1, ft.phase, ft.flags, sb.in_off);
    if (nv == 2)
      for (int i = threadIdx.x; i < K; i += NW * 32) xs[K + i] = __ldcg(x2 + sb.in_off + i);
    __syncthreads();
    const int ch0 = ft.c0 / 32, nch = (ft.c1 + 31) / 32;
    // strips beyond the map (RT > 1 at the last rows) are skipped
    const int nstrip = (K + kRowTile - 1) / kRowTile;
    const int s0 = ft.tile * RT;
    const double2* Tt = a.T + sb.T_off + (long long)s0 * K * kRowTile + lane;
    if (RT == 1 && nv == 2) {
      double2 acc[1][2][2];
      contract_regs<NW, 1, 2>(Tt, xs, K, nstrip, s0, warp, ch0, nch, acc);
      __syncthreads();
#pragma unroll
      for (int x = 0; x < 2; ++x) part[(x * NW + warp) * 32 + lane] = cadd(acc[0][x][0], acc[0][x][1]);
    } else {
      double2 acc[RT][1][2];
      contract_regs<NW, RT, 1>(Tt, xs, K, nstrip, s0, warp, ch0, nch, acc);
      __syncthreads();
#pragma unroll
      for (int q = 0; q < RT; ++q) part[(q * NW + warp) * 32 + lane] = cadd(acc[q][0][0], acc[q][0][1]);
    }
    __syncthreads();
    if (tr && threadIdx.x == 0) tr[3] = gtimer();
    if (warp < RT) {
      // warp q finalises strip q: fixed-order sum over the warps' partials
      const int q = warp;
      double2 y1 = part[(q * NW) * 32 + lane], y2 = make_double2(0, 0);
#pragma unroll
      for (int ww = 1; ww < NW; ++ww) y1 = cadd(y1, part[(q * NW + ww) * 32 + lane]);
      if (nv == 2) {
        y2 = part[NW * 32 + lane];
#pragma unroll
        for (int ww = 1; ww < NW; ++ww) y2 = cadd(y2, part[(NW + ww) * 32 + lane]);
      }
      const int row = (s0 + q) * kRowTile + lane;
      if (row >= it.rlo && row < it.rhi) {
        const int f = row / n, p = row - f * n;
        const long long off = (long long)sb.tgt[f] + p;
        HS_DCHECK(f < sb.k && off >= 0 && off < a.L, DBG_VEC);
        const int o = rv.owner(sb.tgt[f] / n);  // the output block's rank
        const bool low = f < sb.nlow, zr = (ft.rmask >> (4 + f)) & 1;
        double2 e1 = make_double2(0, 0), e2 = e1, e3 = e1;
        epi_fetch(rv, ft.phase, ft.flags, low, zr, o, off, e1, e2, e3);
        epi_store(rv, ft.phase, ft.flags, low, o, off, y1, y2, e1, e2, e3);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      tile_signal(rv, ft.phase, ft.flags, max(it.rlo, s0 * kRowTile), min(it.rhi, (s0 + RT) * kRowTile), n, sb.nlow,
                  sb.tgt);
      if (tr) {
        tr[4] = gtimer();
        tr[5] = ((unsigned long long)smid() << 32) | ((unsigned)blockIdx.x << 8) | (unsigned)ft.phase;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// The fused BSP apply with the maps staged by the Tensor Memory Accelerator:
// a producer warp claims tiles (ticket order), and for each issues bulk
// copies (cp.async.bulk, one elected thread) of the tile's 32-column chunks
// -- 16 KB each, contiguous in the strip-major layout -- into a ring of S
// shared-memory stages with mbarrier full/empty handshakes.  NW consumer warps
// wait for the tile's dependencies, load its incoming slab and consume the
// chunks as they land.  The map stream never waits on a dependency: while the
// consumers wait (or run the epilogue) the producer keeps filling the ring
// with this tile's and the next tile's chunks, so HBM stays busy (the
// register-streaming kernel idles ~30 % of a tile's time at cfg3 on the
// dependency wait, slab load and epilogue; profiles/r01/fused_trace_summary.txt).
// Warps: producer (NW), signaller (NW + 1: takes each tile's release fence and
// completion atomics off the consumers' path, or idle when the plan has the
// consumers signal directly), consumers 0..NW-1 (warp 0 finishes the rows).
// Map chunks carry an L2 evict-first policy (evict-last for aliased per-kind
// maps).  Phase-4 tiles multiply two slabs per map read; split-K pairs (opt-in)
// meet in `split_buf`.  Per-step plan: the k_step1 arithmetic order (bitwise
// identical); map-once plan: the same column split, other phases (hs_ctx.h).
constexpr int kSigStop = -99;  // SigRec.phase: the consumers are done (phase -1: a record with nothing to signal)
struct SigRec {  // a tile's completions, handed from the consumers to the signaller warp
  int phase, flags, nlow, r0, r1;
  int tgt[4];
  unsigned long long* tr;
};

struct TileDesc {
  long long map_off;  // element offset of the tile's 32-row strip
  int t, K, phase, flags, alt, in_off, rlo, rhi, row0, dep0, ndep, rmask, nlow, c0, c1, ks, pair;
  int tgt[4];
  unsigned long long claimed;  // globaltimer at the producer's claim (trace only)
};

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
#ifdef HS_DEVICE_CHECKS
  unsigned long long spins = 0;
#endif
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
#ifdef HS_DEVICE_CHECKS
    if (!ok && ++spins > (1ull << 28)) {
      hs_dbg_fail(DBG_MBAR, __LINE__);
      break;
    }
#endif
  } while (!ok);
}
// Map chunks are read exactly once per apply: evict them from L2 first, so the
// interface vectors (a few x 8 MB, re-read by every tile) stay L2-resident.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                         unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void consumers_sync(int nthreads) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

constexpr int kChunk = 32 * kRowTile;  // elements of one 32-column chunk of a strip

template <int NW, int S, bool MR>
__global__ void __maxnreg__(96) k_bsp_tma(FusedArgs a) {  // 96: two 10-warp CTAs per SM (per-SMSP register file)
  const RankView<MR> rv(a);
  const int cr = rv.cr;
  extern __shared__ __align__(128) double2 smt[];
  double2* stage = smt;                // S x kChunk
  double2* xs = stage + S * kChunk;    // maxK
  double2* part = xs;                  // nv x NW x 32 partial sums, reusing the slab once consumed
  __shared__ __align__(8) unsigned long long full[S], empty[S], dfull[2], dempty[2], sfull[2], sempty[2];
  __shared__ TileDesc desc[2];
  __shared__ SigRec sig[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NT = NW * 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], NW); }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&dfull[i], 1); mbar_init(&dempty[i], NW);
      mbar_init(&sfull[i], 1); mbar_init(&sempty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NW + 1) {  // ---- signaller: publishes each tile's completions off the consumers' path
    if (lane == 0 && !a.direct_signal) {
      for (int q = 0;; ++q) {
        const int d = q & 1;
        mbar_wait(&sfull[d], (q >> 1) & 1);  // acquire: warp 0's epilogue stores
        const SigRec r = sig[d];
        mbar_arrive(&sempty[d]);
        if (r.phase == kSigStop) break;
        tile_signal(rv, r.phase, r.flags, r.r0, r.r1, a.n, r.nlow, r.tgt);
        if (r.tr) r.tr[4] = gtimer();
      }
    }
    return;
  }
  if (warp == NW) {  // ---- producer
    if (lane == 0) {
      const unsigned long long pol = a.map_keep ? l2_evict_last() : l2_evict_first();
      long long g = 0;
      for (int q = 0;; ++q) {
        const int d = q & 1;
        mbar_wait(&dempty[d], ((q >> 1) & 1) ^ 1);
        TileDesc td;
        td.t = atomicAdd(rv.ticket(), 1);
        if (a.trace) td.claimed = gtimer();
        if (td.t < rv.ntiles()) {
          const FusedTile ft = rv.tiles()[td.t];
          HS_DCHECK(ft.item >= 0 && ft.item < a.nitems, DBG_INDEX);
          const DevItem it = a.items[ft.item];
          HS_DCHECK(it.s >= 0 && it.s < a.nsub, DBG_INDEX);
          const DevSub sb = a.subs[it.s];
          HS_DCHECK(sb.T_off >= 0 && sb.T_off + (long long)(ft.tile + 1) * sb.k * a.n * kRowTile <= a.T_elems, DBG_MAP);
          HS_DCHECK(sb.in_off >= 0 && sb.in_off + (long long)sb.k * a.n <= a.L, DBG_VEC);
          HS_DCHECK(ft.c0 >= 0 && ft.c0 <= ft.c1 && ft.c1 <= sb.k * a.n, DBG_INDEX);
          td.K = sb.k * a.n;
          td.row0 = ft.tile * kRowTile;
          td.map_off = sb.T_off + (long long)ft.tile * td.K * kRowTile;
          td.phase = ft.phase; td.flags = ft.flags; td.alt = it.alt; td.in_off = sb.in_off; td.nlow = sb.nlow;
          td.c0 = ft.c0; td.c1 = ft.c1; td.ks = ft.ks; td.pair = ft.pair;
          td.rlo = it.rlo; td.rhi = it.rhi; td.dep0 = ft.dep0; td.ndep = ft.ndep; td.rmask = ft.rmask;
          for (int f = 0; f < 4; ++f) td.tgt[f] = sb.tgt[f];
        }
        desc[d] = td;
        mbar_arrive(&dfull[d]);
        if (td.t >= rv.ntiles()) break;
        const int nch = (td.c1 + 31) / 32;
        const double2* src = a.T + td.map_off;
        if (a.prefetch) {
          // the chunks beyond the ring stream into L2 now, while the consumers
          // wait for the tile's dependencies: the bulk copies of those chunks
          // then hit L2 (a critical-path tile streams at L2 rather than at its
          // share of HBM bandwidth; the bytes from HBM are the same)
          const int cp0 = td.c0 / 32 + S;
          if (cp0 < nch) {
            const long long e0 = (long long)cp0 * kChunk;
            // prefetch = 1: the whole rest of the tile; 2: the next ring's worth
            const int cp1 = a.prefetch == 2 ? min(nch, cp0 + S) : nch;
            const long long e1 = (long long)min(td.K, 32 * cp1) * kRowTile;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src + e0),
                         "r"((unsigned)((e1 - e0) * sizeof(double2)))
                         : "memory");
          }
        }
        for (int ch = td.c0 / 32; ch < nch; ++ch, ++g) {
          const int st = (int)(g % S);
          mbar_wait(&empty[st], (unsigned)((g / S) & 1) ^ 1);
          const unsigned bytes = (unsigned)min(32, td.K - 32 * ch) * kRowTile * sizeof(double2);
          mbar_expect_tx(&full[st], bytes);
          bulk_g2s(stage + (size_t)st * kChunk, src + (long long)ch * kChunk, bytes, &full[st], pol);
        }
      }
    }
    return;
  }
  // ---- consumers
  constexpr int CPW = 32 / NW;
  const int n = a.n;
  long long g = 0;
  if (threadIdx.x == 0) rv.wait_inputs();
  consumers_sync(NT);
  for (int q = 0;; ++q) {
    const int d = q & 1;
    mbar_wait(&dfull[d], (q >> 1) & 1);
    const TileDesc td = desc[d];
    __syncwarp();
    if (lane == 0) mbar_arrive(&dempty[d]);
    if (td.t >= rv.ntiles()) {
      if (threadIdx.x == 0 && !a.direct_signal) {  // tell the signaller to stop
        mbar_wait(&sempty[q & 1], ((q >> 1) & 1) ^ 1);
        sig[q & 1].phase = kSigStop;
        mbar_arrive(&sfull[q & 1]);
      }
      rv.drain(blockIdx.x * NT + threadIdx.x, gridDim.x * NT);
      break;
    }
    unsigned long long* tr = (a.trace && !MR) ? a.trace + 6ll * td.t : nullptr;
    if (tr && threadIdx.x == 0) {
      tr[0] = td.claimed;
      tr[1] = gtimer();
    }
    for (int i = threadIdx.x; i < td.ndep; i += NT) {
      const FusedDep dp = a.deps[td.dep0 + i];
      HS_DCHECK(dp.block >= 0 && dp.block < a.npairs, DBG_COUNTER);
      const volatile int* p = rv.done(dp.block);
      HS_WAIT(*p < rv.target(dp), 32, DBG_DEPWAIT);
    }
    rv.fence();  // acquire: the producers' stores before this CTA's reads
    consumers_sync(NT);
    if (tr && threadIdx.x == 0) tr[2] = gtimer();
    // warp 0 (lane = output row) fetches its epilogue operands now, in the
    // shadow of the slab load and the contraction, not after them
    const int erow = td.row0 + lane;
    const bool erow_ok = warp == 0 && erow >= td.rlo && erow < td.rhi;
    const int ef = erow / n;
    const long long eoff = erow_ok ? (long long)td.tgt[ef] + (erow - ef * n) : 0;
    HS_DCHECK(!erow_ok || (ef < 4 && eoff >= 0 && eoff < a.L), DBG_VEC);
    const int eo = erow_ok ? rv.owner(td.tgt[ef] / n) : cr;  // the output block's rank
    const bool elow = ef < td.nlow;
    double2 e1 = make_double2(0, 0), e2 = e1, e3 = e1;
    if (erow_ok) epi_fetch(rv, td.phase, td.flags, elow, (td.rmask >> (4 + ef)) & 1, eo, eoff, e1, e2, e3);
    const int K = td.K;
    const int nv = td.phase == 4 ? 2 : 1;
    // the slab (this subdomain's incoming blocks) lives on this CTA's rank
    const double2 *x1, *x2;
    slab_srcs(rv, td.phase, td.alt, cr, x1, x2);
    x1 += td.in_off;
    const double2* rsrc = rv.vec(FV_R, cr) + td.in_off;
    // zL starts as r without a copy: faces of zL not yet written read r
    for (int i = threadIdx.x; i < K; i += NT)
      xs[i] = slab_value(rv, cr, x1, rsrc, i, n, td.rmask, td.c0, td.c1, td.phase, td.flags, td.in_off);
    if (nv == 2)
      for (int i = threadIdx.x; i < K; i += NT) xs[K + i] = __ldcg(x2 + td.in_off + i);
    consumers_sync(NT);
    double2 a0 = make_double2(0, 0), a1 = a0, b0 = a0, b1 = a0;
    const int ch0 = td.c0 / 32, nch = (td.c1 + 31) / 32;
    if (nv == 2) {
      for (int ch = ch0; ch < nch; ++ch, ++g) {
        const int st = (int)(g % S);
        mbar_wait(&full[st], (unsigned)((g / S) & 1));
        const double2* Ts = stage + (size_t)st * kChunk;
#pragma unroll
        for (int u = 0; u < CPW; ++u) {
          const int cc = warp * CPW + u, col = ch * 32 + cc;
          if (col < K) {
            const double2 tv = Ts[cc * kRowTile + lane];
            if (col & 1) { cfma(a1, tv, xs[col]); cfma(b1, tv, xs[K + col]); }
            else { cfma(a0, tv, xs[col]); cfma(b0, tv, xs[K + col]); }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
    } else {
      for (int ch = ch0; ch < nch; ++ch, ++g) {
        const int st = (int)(g % S);
        mbar_wait(&full[st], (unsigned)((g / S) & 1));
        const double2* Ts = stage + (size_t)st * kChunk;
#pragma unroll
        for (int u = 0; u < CPW; ++u) {
          const int cc = warp * CPW + u, col = ch * 32 + cc;
          if (col < K) {
            if (col & 1) cfma(a1, Ts[cc * kRowTile + lane], xs[col]);
            else cfma(a0, Ts[cc * kRowTile + lane], xs[col]);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
      }
    }
    consumers_sync(NT);  // every consumer is done with the slab
    part[warp * 32 + lane] = cadd(a0, a1);
    if (nv == 2) part[(NW + warp) * 32 + lane] = cadd(b0, b1);
    consumers_sync(NT);
    if (tr && threadIdx.x == 0) tr[3] = gtimer();
    if (warp == 0) {
      double2 y1 = part[lane], y2 = make_double2(0, 0);
#pragma unroll
      for (int w = 1; w < NW; ++w) y1 = cadd(y1, part[w * 32 + lane]);
      if (nv == 2) {
        y2 = part[NW * 32 + lane];
#pragma unroll
        for (int w = 1; w < NW; ++w) y2 = cadd(y2, part[(NW + w) * 32 + lane]);
      }
      bool finish = true;
      if (td.ks >= 0) {
        // split-K: publish this half's partial sums; the second of the pair to
        // arrive adds them in half order (deterministic) and finishes the rows
        double2* mine = a.split_buf + ((size_t)td.pair * 2 + td.ks) * 64;
        mine[lane] = y1;
        mine[32 + lane] = y2;
        __syncwarp();
        int old = 0;
        if (lane == 0) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          old = atomicAdd(a.split_cnt + td.pair, 1);
        }
        old = __shfl_sync(0xffffffffu, old, 0);
        finish = old & 1;
        if (finish) {
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
          const double2* other = a.split_buf + ((size_t)td.pair * 2 + (1 - td.ks)) * 64;
          const double2 o1 = __ldcg(other + lane), o2 = __ldcg(other + 32 + lane);
          y1 = td.ks == 0 ? cadd(y1, o1) : cadd(o1, y1);
          y2 = td.ks == 0 ? cadd(y2, o2) : cadd(o2, y2);
        }
      }
      if (finish && erow_ok) epi_store(rv, td.phase, td.flags, elow, eo, eoff, y1, y2, e1, e2, e3);
      const int sphase = finish ? td.phase : -1;  // the first half of a pair signals nothing
      __syncwarp();
      if (lane == 0 && a.direct_signal) {  // latency-bound plans: no hand-off hop
        tile_signal(rv, sphase, td.flags, max(td.rlo, td.row0), min(td.rhi, td.row0 + kRowTile), n, td.nlow, td.tgt);
        if (tr) {
          tr[4] = gtimer();
          tr[5] = ((unsigned long long)smid() << 32) | ((unsigned)blockIdx.x << 8) | (unsigned)td.phase;
        }
      } else if (lane == 0) {  // hand the completion signals to the signaller warp
        mbar_wait(&sempty[q & 1], ((q >> 1) & 1) ^ 1);
        SigRec& r = sig[q & 1];
        r.phase = sphase; r.flags = td.flags; r.nlow = td.nlow;
        r.r0 = max(td.rlo, td.row0); r.r1 = min(td.rhi, td.row0 + kRowTile);
        for (int f = 0; f < 4; ++f) r.tgt[f] = td.tgt[f];
        r.tr = tr;
        if (tr) tr[5] = ((unsigned long long)smid() << 32) | ((unsigned)blockIdx.x << 8) | (unsigned)td.phase;
        mbar_arrive(&sfull[q & 1]);  // release: this warp's epilogue stores
      }
    }
    // no CTA barrier here: the next tile's slab overwrites the partial sums only
    // after the next consumers_sync, which warp 0 joins after its epilogue
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

// Blocks finished without a map read (map-once per-step plan): mode 0:
// o1 = o2 = 0, o3 = a (rp = w = 0, z = zL); mode 1: o1 = a ((I - S) z = r).
__global__ void k_block_fill(const int* __restrict__ blocks, int nb, int mode, double2* o1, double2* o2, double2* o3,
                             const double2* a, int n, int R) {
  const long long per = (long long)n * R;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < per * nb;
       i += (long long)gridDim.x * blockDim.x) {
    const int j = (int)(i / per);
    const long long t = (long long)blocks[j] * per + (i - j * per);
    if (mode == 0) {
      o1[t] = make_double2(0, 0);
      o2[t] = make_double2(0, 0);
      o3[t] = a[t];
    } else {
      o1[t] = a[t];
    }
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
      constexpr int NW = kSumWarps;  // same column split as the fused kernels (bitwise identical sums)
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

void launch_block_fill(Ctx& c, const int* blocks, int nb, int mode, double2* o1, double2* o2, double2* o3,
                       const double2* a, int R, cudaStream_t st) {
  if (nb == 0) return;
  long long len = (long long)nb * c.n * R;
  c.launches++;
  k_block_fill<<<grid_for(len, c.num_sms), 256, 0, st ? st : c.stream>>>(blocks, nb, mode, o1, o2, o3, a, c.n, R);
}

void launch_seam_add(Ctx& c, int dir, double2* z, const double2* r, int R) {
  if (c.n_seam[dir] == 0) return;
  long long len = (long long)c.n_seam[dir] * c.n * R;
  c.launches++;
  k_seam_add<<<grid_for(len, c.num_sms), 256, 0, c.stream>>>(c.d_seam[dir], c.n_seam[dir], z, r,
                                                             c.n, R);
}

cudaError_t set_step_smem_limit() {
  cudaFuncSetAttribute(k_bsp_fused<8, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_bsp_fused<8, 2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  return cudaFuncSetAttribute(k_step1<kSumWarps>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              200 * 1024);
}

// TMA-staged fused kernel with an ST-stage ring: the grid is every CTA that
// fits (ST = 5: two CTAs per SM, the map stream's bytes in flight; ST = 12:
// one CTA per SM holding up to 192 KB of a tile's map while it waits for its
// inputs -- for critical-path-bound plans).  G > 1: emulated ranks, grid a
// multiple of G.
template <int ST, bool MR>
cudaError_t launch_tma(Ctx& c, const DevFused& f, const FusedArgs& a, int G) {
  constexpr int NWt = kSumWarps;
  const size_t smem = (size_t)(ST * kChunk + f.nv * std::max(f.maxK, NWt * 32)) * sizeof(double2);
  static int per_sm = 0;
  static size_t per_sm_smem = 0;
  if (per_sm == 0 || per_sm_smem != smem) {
    cudaError_t ae = cudaFuncSetAttribute(k_bsp_tma<NWt, ST, MR>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (ae != cudaSuccess) return ae;  // does not fit one CTA per SM
    cudaFuncSetAttribute(k_bsp_tma<NWt, ST, MR>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bsp_tma<NWt, ST, MR>, (NWt + 2) * 32, smem);
    if (getenv("HS_DEBUG")) fprintf(stderr, "k_bsp_tma<%d>: smem %zu per_sm %d (%s)\n", ST, smem, per_sm, cudaGetErrorString(oe));
    per_sm = std::max(1, per_sm);
    per_sm_smem = smem;
  }
  const int grid = G > 1 ? std::max(G, (per_sm * c.num_sms / G) * G) : std::max(1, std::min(std::max(1, f.ntiles), per_sm * c.num_sms));
  c.launches++;
  k_bsp_tma<NWt, ST, MR><<<grid, (NWt + 2) * 32, smem, c.stream>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_bsp_fused(Ctx& c, const DevFused& f, const double2* r, double2* zL, double2* rp,
                             double2* w, double2* z, double2* wout) {
  // TMA-staged (k_bsp_tma) or register streaming (k_bsp_fused: variant 0 = 1 strip
  // per tile, 2 = 2 strips per tile)
  if (f.tma) {
    // 8 consumer warps, 5 x 16 KB stages: 2 CTAs per SM (measured on B200 against
    // 16 warps, 3 or 10 stages; tools/run_bsp_variants.sh)
    cudaError_t e = cudaMemsetAsync(f.counters, 0, (c.plan.npairs + 1) * sizeof(int), c.stream);
    if (e != cudaSuccess) return e;
    FusedArgs a;
    a.tiles = f.tiles; a.items = f.items; a.deps = f.deps; a.subs = c.dsubs; a.T = c.T;
    a.r = r; a.zL = zL; a.rp = rp; a.w = w; a.z = z; a.wout = wout;
    a.done = f.counters; a.ticket = f.counters + c.plan.npairs;
    a.ntiles = f.ntiles; a.n = c.n; a.maxK = f.maxK; a.nv = f.nv;
  a.L = c.plan.L; a.T_elems = (long long)c.T_elems;
  { static const int pf = getenv("HS_TMA_PREFETCH") ? atoi(getenv("HS_TMA_PREFETCH")) : 0; a.prefetch = pf; } a.nitems = f.nitems; a.nsub = c.plan.nsub; a.npairs = c.plan.npairs;
    a.direct_signal = f.direct_signal;
    a.split_buf = f.split_buf; a.split_cnt = f.split_cnt;
    a.map_keep = c.map_mode == 2;
    a.trace = (c.trace_on && c.trace && c.trace_cap >= (size_t)f.ntiles) ? c.trace : nullptr;
    if (a.trace) c.trace_rows = f.ntiles;
    return f.stages == 12 ? launch_tma<12, false>(c, f, a, 1) : launch_tma<5, false>(c, f, a, 1);
  }
  static_assert(kSumWarps == 8, "register-streaming fused kernels are instantiated for 8 warps");
  const int var = f.rt == 2 ? 2 : 0;
  const int NWv = 8;
  const size_t smem = (size_t)std::max(f.nv * f.maxK, NWv * 32 * std::max(f.rt, f.nv)) * sizeof(double2);
  static int per_sm[3] = {0, 0, 0};
  static size_t per_sm_smem[3] = {0, 0, 0};
  if (per_sm[var] == 0 || per_sm_smem[var] != smem) {
    if (var == 2) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[var], k_bsp_fused<8, 2, false>, 256, smem);
    else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[var], k_bsp_fused<8, 1, false>, 256, smem);
    per_sm_smem[var] = smem;
    if (per_sm[var] < 1) per_sm[var] = 1;
  }
  cudaError_t e = cudaMemsetAsync(f.counters, 0, (c.plan.npairs + 1) * sizeof(int), c.stream);
  if (e != cudaSuccess) return e;
  FusedArgs a;
  a.tiles = f.tiles; a.items = f.items; a.deps = f.deps; a.subs = c.dsubs; a.T = c.T;
  a.r = r; a.zL = zL; a.rp = rp; a.w = w; a.z = z; a.wout = wout;
  a.done = f.counters; a.ticket = f.counters + c.plan.npairs;
  a.ntiles = f.ntiles; a.n = c.n; a.maxK = f.maxK; a.nv = f.nv;
  a.L = c.plan.L; a.T_elems = (long long)c.T_elems;
  { static const int pf = getenv("HS_TMA_PREFETCH") ? atoi(getenv("HS_TMA_PREFETCH")) : 0; a.prefetch = pf; } a.nitems = f.nitems; a.nsub = c.plan.nsub; a.npairs = c.plan.npairs;
    a.trace = (c.trace_on && c.trace && c.trace_cap >= (size_t)f.ntiles) ? c.trace : nullptr;
    if (a.trace) c.trace_rows = f.ntiles;
  const int grid = std::max(1, std::min(f.ntiles, per_sm[var] * c.num_sms));
  c.launches++;
  if (var == 2) k_bsp_fused<8, 2, false><<<grid, 256, smem, c.stream>>>(a);
  else k_bsp_fused<8, 1, false><<<grid, 256, smem, c.stream>>>(a);
  return cudaGetLastError();
}

// out[block b] = the copy of block b held by its owner rank (emulated ranks).
struct RankBases {
  const double2* p[kMaxRanks];
};
__global__ void k_gather_blocks(double2* out, RankBases src, const int* __restrict__ blk_rank, int n, long long L) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < L; i += (long long)gridDim.x * blockDim.x)
    out[i] = src.p[blk_rank[i / n]][i];
}

void launch_gather_blocks(Ctx& c, double2* out, const double2* const* src, int G, const int* blk_rank, long long L) {
  RankBases b;
  for (int g = 0; g < kMaxRanks; ++g) b.p[g] = g < G ? src[g] : nullptr;
  c.launches++;
  k_gather_blocks<<<grid_for(L, c.num_sms), 256, 0, c.stream>>>(out, b, blk_rank, c.n, L);
}

// The fused apply over row-band ranks: `mr` carries every rank's vectors,
// counters and tile list.  Emulation (mr.self < 0): one launch, CTA c works
// for rank c % G.  (The caller zeroes the counters.)
cudaError_t launch_bsp_fused_ranks(Ctx& c, const DevFused& f, const MultiRankArgs& mr) {
  FusedArgs a;
  a.tiles = nullptr; a.items = f.items; a.deps = f.deps; a.subs = c.dsubs; a.T = c.T;
  a.r = nullptr; a.zL = a.rp = a.w = a.z = a.wout = nullptr;
  a.done = nullptr; a.ticket = nullptr;
  a.ntiles = 0; a.n = c.n; a.maxK = f.maxK; a.nv = f.nv; a.trace = nullptr;
  a.L = c.plan.L; a.T_elems = (long long)c.T_elems;
  { static const int pf = getenv("HS_TMA_PREFETCH") ? atoi(getenv("HS_TMA_PREFETCH")) : 0; a.prefetch = pf; } a.nitems = f.nitems; a.nsub = c.plan.nsub; a.npairs = c.plan.npairs;
  a.direct_signal = f.direct_signal;
  a.split_buf = f.split_buf; a.split_cnt = f.split_cnt;
  a.map_keep = c.map_mode == 2;
  a.mr = mr;
  const int G = mr.self < 0 ? mr.G : 1;
  if (f.tma) {
    return f.stages == 12 ? launch_tma<12, true>(c, f, a, G) : launch_tma<5, true>(c, f, a, G);
  }
  c.launches++;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_bsp_fused<8, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  const size_t smem = (size_t)std::max(f.nv * f.maxK, 8 * 32 * f.nv) * sizeof(double2);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bsp_fused<8, 1, true>, 256, smem);
  const int grid = std::max(G, (std::max(1, per_sm) * c.num_sms / G) * G);
  k_bsp_fused<8, 1, true><<<grid, 256, smem, c.stream>>>(a);
  return cudaGetLastError();
}

// A deliberately failing check (hs_debug_selftest): proves that the debug
// library's instrumentation reports (and the release library's is compiled out).
__global__ void k_dbg_selftest(int n) { HS_DCHECK(n < 0, DBG_INDEX); }

cudaError_t launch_dbg_selftest(Ctx& c) {
  c.launches++;
  k_dbg_selftest<<<1, 32, 0, c.stream>>>(1);
  return cudaGetLastError();
}

HS_DBG_ACCESSOR(hs_dbg_take_apply)

}  // namespace hs
