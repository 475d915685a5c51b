// Complex128 GEMM on the FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64; tcgen05
// has no f64 kind) for the dense contractions of the sweeps:
//   * K4, multi-RHS: Y = T_s[rows, :] * X_s (K x R), X_s the subdomain's
//     incoming slab of the [L][R] vector (interface_system.py:115-133 for R
//     right-hand sides at once);
//   * the shared-operator variant: every subdomain with the same operator
//     (discretization.py:224-229: the matrix does not depend on which faces
//     couple) uses its class map T4 (4n x 4n), so a step is ONE contraction
//     Y = T4[rows, :] * [x_s1 ... x_sm] with missing faces read as zero and
//     their outputs dropped -- FP64-bound with the map L2-resident.
//
// Kernels (a complex MAC is 3 real DMMAs by the 3M (Gauss) product in all):
//   * k_zmma2 (default, per step): bulk-copy (TMA) staged, producer warp +
//     mbarrier ring, one task per CTA with cluster split-K or persistent;
//   * k_zmma2_df (default for R right-hand sides; the shared maps with one
//     right-hand side on request, hs_set_fused bit 3): the whole BSP apply as
//     one persistent dataflow launch on the same core (tickets, per-(block,
//     32-RHS chunk) completion counters, the map-once residual with fill tasks);
//   * k_zmma / k_zmma_fused (round 1, cp.async core: tasks of 32 rows x 32
//     columns, 4 output quadrants x 2 K halves): the shared maps with several
//     right-hand sides (n-major columns of stride R are not bulk-copyable) and
//     HS_ZMMA2=0;
//   * k_zgemm_dmma: the factorisation's batched block solves.
// A task's A operand is a 32-row strip of the strip-major map layout (K x 32,
// contiguous); B columns come from the vector through column descriptors
// (per-face element offset or -1, stride R between consecutive positions).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "hs_common.cuh"
#include "hs_kernels.h"

namespace cg = cooperative_groups;

namespace hs {

namespace {

constexpr int BM = 32, BN = 32, KC = 32, STAGES = 3, THREADS = 256;
// row stride 34 (not 32): the 8 lanes of a 128-bit shared-load phase (4 k rows x
// 2 columns) then hit 8 distinct 16-byte bank groups
constexpr int SA = BM + 2, SB = BN + 2;
constexpr int kStageElems = KC * (SA + SB);

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// column descriptors of the current task, staged in shared memory
struct ZCols {
  long long in[BN][4];
  long long out[BN][4];
  int slot[BN][4];
  int r[BN];
  int alt[BN];
};

__device__ __forceinline__ void zmma_cols(const MmaTask& tk, const MmaCol* __restrict__ cols, ZCols& zc) {
  const int tid = threadIdx.x;
  if (tid < BN) {
    if (tid < tk.ncols) {
      const MmaCol c = cols[tk.col0 + tid];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        zc.in[tid][q] = c.in[q];
        zc.out[tid][q] = c.out[q];
        zc.slot[tid][q] = c.slot[q];
      }
      zc.r[tid] = c.r;
      zc.alt[tid] = c.alt;
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) zc.in[tid][q] = zc.out[tid][q] = -1, zc.slot[tid][q] = -1;
      zc.r[tid] = 0;
      zc.alt[tid] = 0;
    }
  }
}

// K chunks [kc0, kc0 + nk) of the task; on return the wk == 0 warps hold the
// summed tile (cre/cim), and shared memory may be reused.
__device__ __forceinline__ double2& zAs(double2* dyn, int st, int k, int m) { return dyn[st * kStageElems + k * SA + m]; }
__device__ __forceinline__ double2& zBs(double2* dyn, int st, int k, int j) {
  return dyn[st * kStageElems + KC * SA + k * SB + j];
}

// The pipelined contraction of K chunks [kc0, kc0 + nk): load(stage, kc) stages
// chunk kc's A tile ([k][m], 32 x 32) and B tile ([k][j], 32 x 32) with
// cp.async; on return the wk == 0 warps hold the summed 32 x 32 tile.
template <class Load>
__device__ __forceinline__ void zmma_core(double2* dyn, Load load, int kc0, int nk, double (&cre)[2][2][2],
                                          double (&cim)[2][2][2]);

__device__ __forceinline__ void zmma_main(const MmaTask& tk, const ZCols& zc, double2* dyn,
                                          const double2* __restrict__ A, const double2* srcA,
                                          const double2* srcB, int n, int R, int kc0, int nk,
                                          double (&cre)[2][2][2], double (&cim)[2][2][2]) {
  const int tid = threadIdx.x;
  const double2* Ab = A + tk.a_off;  // strip containing rows r0..r0+31: [K][32]
  auto As = [&](int st, int k, int m) -> double2& { return zAs(dyn, st, k, m); };
  auto Bs = [&](int st, int k, int j) -> double2& { return zBs(dyn, st, k, j); };
  auto load = [&](int stage, int kc) {
    const int k0 = kc * KC;
    const double2* asrc = Ab + (long long)k0 * BM;
#pragma unroll
    for (int i = 0; i < (KC * BM) / THREADS; ++i) {
      const int el = tid + i * THREADS;
      cp16(&As(stage, el / BM, el % BM), asrc + el);
    }
    const int q = k0 / n, p0 = k0 - q * n;
#pragma unroll
    for (int i = 0; i < (KC * BN) / THREADS; ++i) {
      const int el = tid + i * THREADS;
      const int kk = el / BN, j = el % BN;
      const long long off = zc.in[j][q];
      double2* dst = &Bs(stage, kk, j);
      if (off >= 0) cp16(dst, (zc.alt[j] ? srcB : srcA) + off + (long long)(p0 + kk) * R);
      else *dst = make_double2(0.0, 0.0);
    }
  };
  zmma_core(dyn, load, kc0, nk, cre, cim);
}

template <class Load>
__device__ __forceinline__ void zmma_core(double2* dyn, Load load, int kc0, int nk, double (&cre)[2][2][2],
                                          double (&cim)[2][2][2]) {
  const int tid = threadIdx.x;
  auto As = [&](int st, int k, int m) -> double2& { return zAs(dyn, st, k, m); };
  auto Bs = [&](int st, int k, int j) -> double2& { return zBs(dyn, st, k, j); };
  const int lane = tid & 31, warp = tid >> 5;
  const int wk = warp >> 2, wq = warp & 3;
  const int wm = wq >> 1, wn = wq & 1;
  const int gid = lane >> 2, tig = lane & 3;
  // 3M (Gauss) complex product: s1 = sum ar br, s2 = sum ai bi, p3 = sum (ar + ai)(br + bi);
  // re = s1 - s2, im = p3 - s1 - s2: 3 DMMAs per complex MAC instead of 4
  double p3[2][2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) cre[a][b][c] = cim[a][b][c] = p3[a][b][c] = 0.0;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load(s, kc0 + s);
    cp_commit();
  }
  for (int i = 0; i < nk; ++i) {
    cp_wait<STAGES - 2>();
    __syncthreads();
    const int nxt = i + STAGES - 1;
    if (nxt < nk) load(nxt % STAGES, kc0 + nxt);
    cp_commit();
    const int st = i % STAGES;
    const int kb = wk * (KC / 2);
    double2 a[2], b[2], an[2], bn[2];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) a[mt] = As(st, kb + tig, wm * 16 + mt * 8 + gid);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) b[nt] = Bs(st, kb + tig, wn * 16 + nt * 8 + gid);
#pragma unroll
    for (int k4 = 0; k4 < KC / 2; k4 += 4) {
      if (k4 + 4 < KC / 2) {  // prefetch the next fragments before issuing this step's DMMAs
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) an[mt] = As(st, kb + k4 + 4 + tig, wm * 16 + mt * 8 + gid);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) bn[nt] = Bs(st, kb + k4 + 4 + tig, wn * 16 + nt * 8 + gid);
      }
      double sb[2];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) sb[nt] = b[nt].x + b[nt].y;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const double sa = a[mt].x + a[mt].y;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) dmma(cre[mt][nt][0], cre[mt][nt][1], a[mt].x, b[nt].x);  // s1
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) dmma(cim[mt][nt][0], cim[mt][nt][1], a[mt].y, b[nt].y);  // s2
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) dmma(p3[mt][nt][0], p3[mt][nt][1], sa, sb[nt]);
      }
      if (k4 + 4 < KC / 2) {
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) a[mt] = an[mt];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) b[nt] = bn[nt];
      }
    }
  }
  cp_wait<0>();
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const double s1 = cre[a][b][c], s2 = cim[a][b][c];
        cre[a][b][c] = s1 - s2;
        cim[a][b][c] = p3[a][b][c] - s1 - s2;
      }
  __syncthreads();
  // reduce the two K halves: the wk = 1 warps hand their tiles to wk = 0
  double2* red = dyn;
  if (wk == 1) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          red[(wq * 8 + (mt * 4 + nt * 2 + h)) * 32 + lane] = make_double2(cre[mt][nt][h], cim[mt][nt][h]);
  }
  __syncthreads();
  if (wk == 0) {
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double2 o = red[(wq * 8 + (mt * 4 + nt * 2 + h)) * 32 + lane];
          cre[mt][nt][h] += o.x;
          cim[mt][nt][h] += o.y;
        }
  }
}

}  // namespace

// grid = ntasks * KS, cluster (KS, 1, 1); task = blockIdx.x / KS
__global__ void __launch_bounds__(THREADS) k_zmma(const MmaTask* __restrict__ tasks,
                                                  const MmaCol* __restrict__ cols,
                                                  const double2* __restrict__ A,
                                                  const double2* srcA, const double2* srcB, Epi e,
                                                  int n, int R, int KS) {
  extern __shared__ __align__(16) double2 dyn[];
  __shared__ ZCols zc;
  // programmatic dependent launch: the next step's grid may launch now and
  // run up to its own wait (task and column descriptors) while this one works
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int rank = KS > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const MmaTask tk = tasks[blockIdx.x / KS];
  const int tid = threadIdx.x;
  zmma_cols(tk, cols, zc);
  // the previous step's outputs (this step's inputs and epilogue operands) are
  // complete and visible past this point
  asm volatile("griddepcontrol.wait;" ::: "memory");
  __syncthreads();
  const int nk_all = tk.K / KC;
  const int kc0 = (int)((long long)nk_all * rank / KS), kc1 = (int)((long long)nk_all * (rank + 1) / KS);
  double cre[2][2][2], cim[2][2][2];
  zmma_main(tk, zc, dyn, A, srcA, srcB, n, R, kc0, kc1 - kc0, cre, cim);
  const int lane = tid & 31, warp = tid >> 5;
  const int wk = warp >> 2, wq = warp & 3;
  const int wm = wq >> 1, wn = wq & 1;
  const int gid = lane >> 2, tig = lane & 3;
  double2* red = dyn;
  if (KS > 1) {
    // cluster split-K: ranks > 0 publish their tile, rank 0 sums in rank order
    cg::cluster_group cl = cg::this_cluster();
    __syncthreads();
    if (wk == 0 && rank > 0) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            red[(wq * 8 + (mt * 4 + nt * 2 + h)) * 32 + lane] = make_double2(cre[mt][nt][h], cim[mt][nt][h]);
    }
    cl.sync();
    if (rank == 0 && wk == 0) {
      for (int src = 1; src < KS; ++src) {
        const double2* rem = cl.map_shared_rank(red, src);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double2 o = rem[(wq * 8 + (mt * 4 + nt * 2 + h)) * 32 + lane];
              cre[mt][nt][h] += o.x;
              cim[mt][nt][h] += o.y;
            }
      }
    }
    cl.sync();  // keep remote shared memory alive until rank 0 has read it
    if (rank != 0) return;
  }
  if (wk != 0) return;
  // epilogue: C(row gid, cols 2 tig + {0,1}) of each 8x8 tile
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int row = tk.r0 + wm * 16 + mt * 8 + gid;
    if (row < tk.rlo || row >= tk.rhi) continue;
    const int q = row / n, p = row - q * n;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = wn * 16 + nt * 8 + 2 * tig + h;
        if (j >= tk.ncols) continue;
        const double2 y = make_double2(cre[mt][nt][h], cim[mt][nt][h]);
        const int slot = zc.slot[j][q];
        if (slot == -1) {
          const long long off = zc.out[j][q];
          if (off >= 0) epi_apply(e, off + (long long)p * R, y);
        } else if (slot >= 0) {
          e.send_up[((long long)slot * n + p) * R + zc.r[j]] = y;
        } else {
          e.send_dn[((long long)(-slot - 2) * n + p) * R + zc.r[j]] = y;
        }
      }
  }
}

// ---------------------------------------------------------------------------
// k_zmma2: the per-step contraction with bulk-copy (TMA) staging.
//
// One task = 32 map rows x BN columns (64: all 64 right-hand sides of a
// subdomain's slab, or 64 subdomain columns of a shared-map step; 32 for
// smaller steps).  A producer warp streams K in chunks of KC (32, or 64 for
// the n-major form) through an S-stage ring with cp.async.bulk copies
// (mbarrier complete_tx):
//   A [k][m]  one copy per chunk (unpadded, see Z2::SA);
//   B rows padded so the 128-bit fragment loads are conflict-free:
//   B k-major [k][j] (R RHS of one slab: one contiguous row per position)
//             stride BN + 2: units 2 tig + gid (mod 8), distinct;
//   B n-major [j][k] (shared maps, one column per subdomain: its KC positions
//             of the chunk's face are one contiguous run) stride KC + 4:
//             units 4 gid + tig (mod 8), distinct.
// Absent faces read a zero buffer.  Consumer warps own TM x TN 8x8 DMMA tiles
// of the output over the chunk (KG warp groups split the chunk's k range),
// 3M complex product.  Launch forms (launch_zmma): one task per CTA, K split
// over a thread-block cluster when the step leaves SMs idle (partial tiles
// summed by rank 0 through DSMEM in rank order -- deterministic), or
// persistent (PERS: tasks claimed from a ticket counter, the next task's
// chunks streaming while the current one finishes).  The map chunks do not
// depend on the previous step, so the producer issues the first stages' map
// copies before griddepcontrol.wait (programmatic dependent launch) and the
// vector rows after it.  tools/zcore_bench.cu: this core sustains 0.80-0.86
// of the DMMA peak on L2-resident operands (the cp.async core: ~0.4).
constexpr int Z2KC = 32;

template <int BN, int TM, int TN, bool NMAJ, int S, bool PERS, int KG = 1, int KC_ = Z2KC>
struct Z2 {
  static constexpr int KC = KC_;  // k rows per chunk (64: the n-major shared-map form, half the copies per k)
  // KG warp groups split every chunk's k range (each group owns the whole tile;
  // group 1's partial is added to group 0's through shared memory): a 32 x 32
  // tile then keeps 8 warps x 12 accumulator chains in flight, which the DMMA
  // pipe needs to stay busy (tools/zcore_bench.cu: 4 warps x 12 reach ~0.4)
  static constexpr int WM = 32 / (8 * TM), WN = BN / (8 * TN), NWQ = WM * WN, NWC = NWQ * KG,
                       THREADS = (NWC + 1) * 32;

  // A: the chunk's 32 k rows x 32 map rows are one contiguous 16 KB run of the
  // strip-major layout -> ONE bulk copy, unpadded (a small copy costs the TMA
  // unit ~60 cycles whatever its size, so 32 padded row copies made the
  // n-major contraction copy-bound; the 4-way bank conflicts of the unpadded
  // fragment loads are hidden behind the DMMAs, tools/zcore_bench.cu)
  static constexpr int SA = 32;
  static constexpr int SB = NMAJ ? KC + 4 : BN + 2;
  static constexpr int BROWS = NMAJ ? BN : KC;
  static constexpr int STAGE = KC * SA + BROWS * SB;
  static constexpr int YS = BN + 1;  // output tile row stride (conflict-free fragment writes and row/column reads)
  static constexpr int RING = S * STAGE;
  static constexpr int NTR = TM * TN * 2;  // accumulator pairs per lane
  // persistent: a separate output tile and warp-group reduction area (the ring
  // already holds the next task's chunks); one task per CTA: the drained ring
  static constexpr size_t SMEM =
      sizeof(double2) * (RING + (PERS ? 32 * YS + (KG > 1 ? NWQ * NTR * 32 : 0) : 0));
  static constexpr int ND = PERS ? 2 : 1;  // task descriptor buffers
  static constexpr int EPT = 32 * BN / (NWC * 32);  // epilogue elements per consumer thread
  static_assert(WM * TM * 8 == 32 && WN * TN * 8 == BN, "tile split");
  static_assert(PERS || RING >= 32 * YS, "output tile must fit in the ring");
};

template <int BN>
struct ZCols2 {
  MmaTask tk;
  int stop;  // persistent form: no more tickets
  long long in[BN][4];
  long long out[BN][4];
  int slot[BN][4];
  int r[BN];
  int alt[BN];
};

template <int N>
__device__ __forceinline__ void consumers_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ unsigned long long z2_gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned z2_smem(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void z2_bar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(z2_smem(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void z2_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(z2_smem(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void z2_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(z2_smem(b)) : "memory");
}
__device__ __forceinline__ void z2_wait(unsigned long long* b, unsigned parity) {
  unsigned ok = 0;
#ifdef HS_DEVICE_CHECKS
  unsigned long long spins = 0;
#endif
  do {
#ifdef HS_DEVICE_CHECKS
    if (++spins > (1ull << 28)) {
      hs_dbg_fail(DBG_MBAR, __LINE__);
      break;
    }
#endif
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(z2_smem(b)), "r"(parity)
        : "memory");
  } while (!ok);
}
// CTA-local destination and mbarrier (.shared::cta).  The .shared::cluster
// form with shared::cta-window addresses gave wrong blocks in cluster launches
// (even of cluster size 1) once two CTAs shared an SM (round 2,
// tools/zmma_check.py); the CTA-window form is the one these addresses denote.
__device__ __forceinline__ void z2_copy(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   z2_smem(dst)),
               "l"(src), "r"(bytes), "r"(z2_smem(bar))
               : "memory");
}

// Epilogue operands of one output element, loaded before any store so a lane's
// up to 2 TM TN loads are in flight together (the epilogue is on every sweep
// step's critical path).
struct EpiIn {
  double2 u, v;
};
__device__ __forceinline__ EpiIn epi_load(const Epi& e, long long t) {
  EpiIn x;
  switch (e.mode) {
    case EPI_ACC: x.u = e.o1[t]; break;
    case EPI_IMS: x.u = e.a[t]; break;
    case EPI_RESID: x.u = e.a[t]; x.v = e.b[t]; break;
    case EPI_LATE: x.u = csub(e.a[t], e.b[t]); x.v = e.c[t]; break;
    case EPI_ACC2: x.u = e.o1[t]; x.v = e.o2[t]; break;
    default: break;
  }
  return x;
}
// the arithmetic of epi_apply (hs_common.cuh), same operation order
__device__ __forceinline__ void epi_store(const Epi& e, long long t, double2 y, const EpiIn& x) {
  switch (e.mode) {
    case EPI_SET: e.o1[t] = y; break;
    case EPI_ACC: e.o1[t] = cadd(x.u, y); break;
    case EPI_IMS: e.o1[t] = csub(x.u, y); break;
    case EPI_RESID: {
      const double2 v = csub(x.u, csub(x.v, y));
      e.o1[t] = v;
      e.o2[t] = v;
      e.o3[t] = cadd(x.v, v);
    } break;
    case EPI_LATE: e.o1[t] = cadd(x.u, csub(x.v, y)); break;
    case EPI_ACC2:
      e.o1[t] = cadd(x.u, y);
      e.o2[t] = cadd(x.v, y);
      break;
  }
}

// The kernel.  PERS = false: one task (or one split-K slice of it) per CTA,
// grid = ntasks x KS.  PERS = true (steps with at least one task per SM):
// grid <= #SMs, CTA b runs tasks b, b + grid, ... with the producer streaming
// the next task's chunks while the consumers finish the current one (task
// descriptors double-buffered, mbarrier dfull / dempty).  Epilogue: the tile
// goes through shared memory and is finished by all consumer threads with
// coalesced accesses (k-major: consecutive right-hand sides of a row are
// consecutive elements; n-major: consecutive rows of a column are).
template <int BN, int TM, int TN, bool NMAJ, int S, bool PERS, int KG, int KCT = Z2KC>
__global__ void __launch_bounds__(Z2<BN, TM, TN, NMAJ, S, PERS, KG, KCT>::THREADS, (!PERS && KG == 1 && BN == 32) ? 2 : 1)
    k_zmma2(const MmaTask* __restrict__ tasks, int ntasks, const MmaCol* __restrict__ cols,
            const double2* __restrict__ A, const double2* srcA, const double2* srcB,
            const double2* __restrict__ zeros, Epi e, int n, int R, int KS, unsigned long long* tr, int seq,
            long long Aelems, long long LR, unsigned* ticket, unsigned tbase) {
  using F = Z2<BN, TM, TN, NMAJ, S, PERS, KG, KCT>;
  constexpr int KC = F::KC;
  extern __shared__ __align__(128) double2 sm[];
  __shared__ __align__(8) unsigned long long full[S], empty[S], dfull[2], dempty[2];
  __shared__ ZCols2<BN> zcs[F::ND];
  double2* ys = PERS ? sm + F::RING : sm;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = (!PERS && KS > 1) ? (int)cg::this_cluster().block_rank() : 0;
  // persistent form: tasks claimed from a ticket counter (this launch's slot
  // of a ring of counters, never reset: tickets tbase, tbase + 1, ...), so
  // CTAs that start late -- the previous step's CTAs still hold their SMs --
  // take fewer tasks; one task per CTA otherwise
  const int t0 = PERS ? 0 : (int)blockIdx.x / KS;
  // trace row (hs_set_trace): start, setup done, first chunk landed, contraction
  // done, end, (seq << 40 | smid << 32 | block)
  unsigned long long* trow = tr ? tr + 6ull * blockIdx.x : nullptr;
  if (trow && tid == 0) trow[0] = z2_gtimer();
  auto kslice = [&](const MmaTask& tk, int& kc0, int& nk) {
    const int nk_all = tk.K / KC;
    kc0 = (int)((long long)nk_all * rank / KS);
    nk = (int)((long long)nk_all * (rank + 1) / KS) - kc0;
  };
  auto stage_cols = [&](ZCols2<BN>& zc, const MmaTask& tk, int j0, int jstep) {
    for (int j = j0; j < BN; j += jstep) {
      if (j < tk.ncols) {
        const MmaCol c = cols[tk.col0 + j];
#pragma unroll
        for (int q = 0; q < 4; ++q) zc.in[j][q] = c.in[q], zc.out[j][q] = c.out[q], zc.slot[j][q] = c.slot[q];
        zc.r[j] = c.r;
        zc.alt[j] = c.alt;
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) zc.in[j][q] = zc.out[j][q] = -1, zc.slot[j][q] = -1;
        zc.r[j] = 0;
        zc.alt[j] = 0;
      }
    }
  };
  if (warp == F::NWC && lane == 0) {
    for (int i = 0; i < S; ++i) z2_bar_init(&full[i], 1), z2_bar_init(&empty[i], F::NWC);
    for (int i = 0; i < 2; ++i) z2_bar_init(&dfull[i], 1), z2_bar_init(&dempty[i], F::NWC);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (!PERS) {
    // one task: the consumers stage its column table while the producer starts
    // the map stream (the maps depend neither on it nor on the previous step)
    if (warp < F::NWC) {
      if (tid == 0) zcs[0].tk = tasks[t0];
      stage_cols(zcs[0], tasks[t0], tid, F::NWC * 32);
    }
  }
  __syncthreads();
  if (trow && tid == 0) trow[1] = z2_gtimer();
  if (warp == F::NWC) {  // ---------------- producer
    long long g = 0;
    for (int it = 0; PERS || it == 0; ++it) {
      const int d = PERS ? (it & 1) : 0;
      ZCols2<BN>& zc = zcs[d];
      int t = t0;
      if (PERS) {
        z2_wait(&dempty[d], (unsigned)((it >> 1) & 1) ^ 1);
        unsigned raw = 0;
        if (lane == 0) raw = atomicAdd(ticket, 1u);
        t = (int)(__shfl_sync(0xffffffffu, raw, 0) - tbase);
        HS_DCHECK(t >= 0, DBG_INDEX);
        if (t >= ntasks || t < 0) {
          if (lane == 0) {
            zc.stop = 1;
            z2_arrive(&dfull[d]);
          }
          break;
        }
      }
      const MmaTask tk = tasks[t];
      HS_DCHECK(tk.a_off >= 0 && tk.a_off + (long long)tk.K * 32 <= Aelems && tk.K % KC == 0, DBG_MAP);
      HS_DCHECK(tk.ncols >= 1 && tk.ncols <= BN, DBG_INDEX);
      if (PERS) {
        if (lane == 0) zc.tk = tk, zc.stop = 0;
        stage_cols(zc, tk, lane, 32);
        __syncwarp();
        if (lane == 0) z2_arrive(&dfull[d]);  // release: the table is visible to the consumers
      }
      int kc0, nk;
      kslice(tk, kc0, nk);
      const unsigned bytesB =
          NMAJ ? (unsigned)(BN * KC * sizeof(double2)) : (unsigned)(KC * tk.ncols * sizeof(double2));
      const unsigned bytes = (unsigned)(KC * 32 * sizeof(double2)) + bytesB;
      const double2* Ab = A + tk.a_off;
      auto issueA = [&](int st, int kc) {
        if (lane == 0)
          z2_copy(sm + (size_t)st * F::STAGE, Ab + (long long)kc * KC * 32, KC * 32 * sizeof(double2), &full[st]);
      };
      auto issueB = [&](int st, int kc) {
        double2* sb = sm + (size_t)st * F::STAGE + KC * F::SA;
        const int k0 = kc * KC, q = k0 / n, p0 = k0 - q * n;
        if (NMAJ) {
          for (int j = lane; j < BN; j += 32) {
            const long long off = zc.in[j][q];
            HS_DCHECK(off < 0 || off + (long long)(p0 + KC - 1) * R < LR, DBG_VEC);
            const double2* src = off >= 0 ? (zc.alt[j] ? srcB : srcA) + off + (long long)p0 * R : zeros;
            z2_copy(sb + j * F::SB, src, KC * sizeof(double2), &full[st]);
          }
        } else {
          // one slab: positions k0.. of the compact faces are consecutive rows of R
          HS_DCHECK(zc.in[0][0] >= 0 && zc.in[0][0] + (long long)(k0 + KC - 1) * R + tk.ncols - 1 < LR, DBG_VEC);
          const double2* base = (zc.alt[0] ? srcB : srcA) + zc.in[0][0] + (long long)k0 * R;
          for (int r = lane; r < KC; r += 32)
            z2_copy(sb + r * F::SB, base + (long long)r * R, tk.ncols * sizeof(double2), &full[st]);
        }
      };
      int i = 0;
      if (it == 0) {
        // first task: its first stages' map rows before the dependency wait
        const int pre = nk < S ? nk : S;
        for (int k = 0; k < pre; ++k) {
          if (lane == 0) z2_expect_tx(&full[k], bytes);
          __syncwarp();
          issueA(k, kc0 + k);
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int k = 0; k < pre; ++k) issueB(k, kc0 + k);
        i = pre;
        g = pre;
      }
      for (; i < nk; ++i, ++g) {
        const int st = (int)(g % S);
        if (g >= S) z2_wait(&empty[st], (unsigned)((g / S) & 1) ^ 1);
        if (lane == 0) z2_expect_tx(&full[st], bytes);
        __syncwarp();
        issueA(st, kc0 + i);
        issueB(st, kc0 + i);
      }
    }
  } else {  // ---------------- consumers
    asm volatile("griddepcontrol.wait;" ::: "memory");  // epilogue operands: the previous step's outputs
    const int kg = warp / F::NWQ, wq = warp % F::NWQ;
    const int wm = wq / F::WN, wn = wq % F::WN;
    const int gid = lane >> 2, tig = lane & 3;
    const int ctid = tid;  // consumers are warps 0 .. NWC - 1
    constexpr int KH = KC / KG;  // k rows of a chunk per warp group
    long long g = 0;
    for (int it = 0; PERS || it == 0; ++it) {
      const int d = PERS ? (it & 1) : 0;
      if (PERS) z2_wait(&dfull[d], (unsigned)((it >> 1) & 1));
      const ZCols2<BN>& zc = zcs[d];
      if (PERS && zc.stop) break;
      const MmaTask tk = zc.tk;
      int kc0, nk;
      kslice(tk, kc0, nk);
      double cr[TM][TN][2], ci[TM][TN][2], p3[TM][TN][2];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b)
#pragma unroll
          for (int c = 0; c < 2; ++c) cr[a][b][c] = ci[a][b][c] = p3[a][b][c] = 0.0;
      for (int i = 0; i < nk; ++i, ++g) {
        const int st = (int)(g % S);
        z2_wait(&full[st], (unsigned)((g / S) & 1));
        if (trow && tid == 0 && g == 0) trow[2] = z2_gtimer();
        const double2* sa = sm + (size_t)st * F::STAGE;
        const double2* sb = sa + KC * F::SA;
#pragma unroll
        for (int kk = 0; kk < KH; kk += 4) {
          const int k4 = kg * KH + kk;
          double2 a[TM], b[TN];
#pragma unroll
          for (int mt = 0; mt < TM; ++mt) a[mt] = sa[(k4 + tig) * F::SA + (wm * TM + mt) * 8 + gid];
#pragma unroll
          for (int nt = 0; nt < TN; ++nt)
            b[nt] = NMAJ ? sb[((wn * TN + nt) * 8 + gid) * F::SB + k4 + tig]
                         : sb[(k4 + tig) * F::SB + (wn * TN + nt) * 8 + gid];
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
        if (lane == 0) z2_arrive(&empty[st]);
      }
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const double s1 = cr[a][b][c], s2 = ci[a][b][c];
            cr[a][b][c] = s1 - s2;
            ci[a][b][c] = p3[a][b][c] - s1 - s2;
          }
      if (trow && tid == 0 && it == 0) trow[3] = z2_gtimer();
      constexpr int NT = TM * TN * 2;  // accumulator pairs per lane
      if (KG > 1) {
        // group g > 0 hands its partial tile to group 0 (the drained ring holds
        // it; the persistent form has its own area past the output tile)
        double2* gred = PERS ? ys + 32 * F::YS : sm;
        consumers_bar<F::NWC * 32>();
        if (kg > 0) {
#pragma unroll
          for (int a = 0; a < TM; ++a)
#pragma unroll
            for (int b = 0; b < TN; ++b)
#pragma unroll
              for (int c = 0; c < 2; ++c)
                gred[((warp - F::NWQ) * NT + (a * TN + b) * 2 + c) * 32 + lane] = make_double2(cr[a][b][c], ci[a][b][c]);
        }
        consumers_bar<F::NWC * 32>();
        if (kg == 0) {
#pragma unroll
          for (int a = 0; a < TM; ++a)
#pragma unroll
            for (int b = 0; b < TN; ++b)
#pragma unroll
              for (int c = 0; c < 2; ++c) {
                const double2 o = gred[(warp * NT + (a * TN + b) * 2 + c) * 32 + lane];
                cr[a][b][c] += o.x;
                ci[a][b][c] += o.y;
              }
        }
      }
      if (!PERS && KS > 1) {
        // cluster split-K: ranks > 0 publish their tile (in their drained
        // ring, past the group-reduction area), rank 0 sums in rank order.
        // Consumers only: the producer has left its loop and issues nothing more.
        cg::cluster_group cl = cg::this_cluster();
        double2* red = sm + F::NWQ * NT * 32;
        if (rank > 0 && kg == 0) {
#pragma unroll
          for (int a = 0; a < TM; ++a)
#pragma unroll
            for (int b = 0; b < TN; ++b)
#pragma unroll
              for (int c = 0; c < 2; ++c)
                red[(warp * NT + (a * TN + b) * 2 + c) * 32 + lane] = make_double2(cr[a][b][c], ci[a][b][c]);
        }
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (rank == 0 && kg == 0) {
          for (int src = 1; src < KS; ++src) {
            const double2* rem = cl.map_shared_rank(red, src);
            double2 o[NT];
#pragma unroll
            for (int i = 0; i < NT; ++i) o[i] = rem[(warp * NT + i) * 32 + lane];
#pragma unroll
            for (int a = 0; a < TM; ++a)
#pragma unroll
              for (int b = 0; b < TN; ++b)
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                  cr[a][b][c] += o[(a * TN + b) * 2 + c].x;
                  ci[a][b][c] += o[(a * TN + b) * 2 + c].y;
                }
          }
        }
        // keep remote shared memory alive until rank 0 has read it
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        if (rank != 0) break;
      }
      // ---- epilogue through the output tile
      consumers_bar<F::NWC * 32>();  // the previous task's tile readers (and group partials) are done
      if (kg == 0) {
#pragma unroll
        for (int mt = 0; mt < TM; ++mt)
#pragma unroll
          for (int nt = 0; nt < TN; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              ys[((wm * TM + mt) * 8 + gid) * F::YS + (wn * TN + nt) * 8 + 2 * tig + h] =
                  make_double2(cr[mt][nt][h], ci[mt][nt][h]);
      }
      consumers_bar<F::NWC * 32>();
      long long toff[F::EPT];
      EpiIn xin[F::EPT];
#pragma unroll
      for (int u = 0; u < F::EPT; ++u) {
        const int el = u * F::NWC * 32 + ctid;
        const int rr = NMAJ ? el % 32 : el / BN, j = NMAJ ? el / 32 : el % BN;
        const int row = tk.r0 + rr;
        long long t = -1;
        if (row >= tk.rlo && row < tk.rhi && j < tk.ncols) {
          const int q = row / n, p = row - q * n;
          const int slot = zc.slot[j][q];
          if (slot == -1) {
            const long long off = zc.out[j][q];
            if (off >= 0) t = off + (long long)p * R;
          } else {
            // row-band exchange buffers: encoded as -2 - (2 index + (down ? 1 : 0))
            t = slot >= 0 ? -2 - 2 * (((long long)slot * n + p) * R + zc.r[j])
                          : -3 - 2 * (((long long)(-slot - 2) * n + p) * R + zc.r[j]);
          }
        }
        toff[u] = t;
        HS_DCHECK(t < LR, DBG_VEC);
        if (t >= 0) xin[u] = epi_load(e, t);
      }
#pragma unroll
      for (int u = 0; u < F::EPT; ++u) {
        const int el = u * F::NWC * 32 + ctid;
        const int rr = NMAJ ? el % 32 : el / BN, j = NMAJ ? el / 32 : el % BN;
        const long long t = toff[u];
        const double2 y = ys[rr * F::YS + j];
        if (t >= 0) {
          epi_store(e, t, y, xin[u]);
        } else if (t <= -2) {
          const long long v = -2 - t;
          if (v & 1) e.send_dn[v >> 1] = y;
          else e.send_up[v >> 1] = y;
        }
      }
      if (PERS) {
        __syncwarp();
        if (lane == 0) z2_arrive(&dempty[d]);  // this warp is done with the task's table
      }
    }
  }
  if (!PERS && KS > 1 && warp == F::NWC) {
    // the producer warp takes part in both cluster barriers
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (trow && tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    trow[4] = z2_gtimer();
    trow[5] = ((unsigned long long)seq << 40) | ((unsigned long long)smid << 32) | blockIdx.x;
  }
}

// The whole BSP apply for R right-hand sides (or on the shared class maps) as
// one persistent dataflow launch; see k_bsp_fused for the protocol.
__global__ void __launch_bounds__(THREADS) k_zmma_fused(FusedMmaArgs a) {
  extern __shared__ __align__(16) double2 dyn[];
  __shared__ ZCols zc;
  __shared__ int s_t;
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wk = warp >> 2, wq = warp & 3;
  const int wm = wq >> 1, wn = wq & 1;
  const int gid = lane >> 2, tig = lane & 3;
  const int n = a.n, R = a.R;
  for (;;) {
    if (tid == 0) s_t = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int t = s_t;
    if (t >= a.ntasks) return;
    const FusedMmaTask ft = a.tasks[t];
    const MmaTask tk = ft.task;
    for (int d = tid; d < ft.ndep; d += blockDim.x) {
      const FusedDep dp = a.deps[ft.dep0 + d];
      const volatile int* p = a.done + dp.block;
      while (*p < dp.count) __nanosleep(32);
    }
    __threadfence();
    zmma_cols(tk, a.cols, zc);
    __syncthreads();
    const double2* srcA = ft.phase == 0 ? a.zL : (ft.phase == 1 ? a.zL : a.w);
    const double2* srcB = ft.phase == 0 ? a.r : (ft.phase == 1 ? a.zL : a.rp);
    double cre[2][2][2], cim[2][2][2];
    zmma_main(tk, zc, dyn, a.A, srcA, srcB, n, R, 0, tk.K / KC, cre, cim);
    if (wk == 0) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int row = tk.r0 + wm * 16 + mt * 8 + gid;
        if (row < tk.rlo || row >= tk.rhi) continue;
        const int q = row / n, p = row - q * n;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = wn * 16 + nt * 8 + 2 * tig + h;
            if (j >= tk.ncols) continue;
            const long long o0 = zc.out[j][q];
            if (o0 < 0) continue;
            const long long off = o0 + (long long)p * R;
            const double2 y = make_double2(cre[mt][nt][h], cim[mt][nt][h]);
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
      }
      __threadfence();
    }
    __syncthreads();
    for (int i = tid; i < ft.ninc; i += blockDim.x) atomicAdd(a.done + a.incs[ft.inc0 + i], 1);
  }
}

// The fused apply with every task's K range split over a thread-block cluster
// of KS CTAs: rank 0 claims the ticket and hands it to the cluster through
// distributed shared memory, every rank waits for the task's dependencies and
// contracts its share of the K chunks, ranks > 0 publish their partial tile
// and rank 0 sums them in rank order (deterministic), runs the epilogue and
// signals completion.  A subdomain step is then spread over KS x more SMs, so
// the sweep's dependency chain (17 steps at cfg4) is paced by KS x shorter
// tasks -- the per-step launches could split K the same way but pay a launch
// and a ramp per step, and the unsplit fused kernel runs each task's whole K
// on one SM.
template <int KS>
__global__ void __launch_bounds__(THREADS) k_zmma_fused_ks(FusedMmaArgs a) {
  extern __shared__ __align__(16) double2 dyn[];
  __shared__ ZCols zc;
  __shared__ int s_t;
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank();
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int wk = warp >> 2, wq = warp & 3;
  const int wm = wq >> 1, wn = wq & 1;
  const int gid = lane >> 2, tig = lane & 3;
  const int n = a.n, R = a.R;
  for (;;) {
    if (rank == 0 && tid == 0) {
      // push the ticket into every rank's own shared memory before the barrier:
      // no rank reads a peer's shared memory after it (a peer may have exited)
      const int tt = atomicAdd(a.ticket, 1);
      for (int q = 0; q < KS; ++q) *cl.map_shared_rank(&s_t, q) = tt;
    }
    cl.sync();
    const int t = s_t;
    if (t >= a.ntasks) return;  // the whole cluster leaves together
    const FusedMmaTask ft = a.tasks[t];
    const MmaTask tk = ft.task;
    for (int d = tid; d < ft.ndep; d += blockDim.x) {
      const FusedDep dp = a.deps[ft.dep0 + d];
      const volatile int* p = a.done + dp.block;
      while (*p < dp.count) __nanosleep(32);
    }
    __threadfence();
    zmma_cols(tk, a.cols, zc);
    __syncthreads();
    const double2* srcA = ft.phase == 0 ? a.zL : (ft.phase == 1 ? a.zL : a.w);
    const double2* srcB = ft.phase == 0 ? a.r : (ft.phase == 1 ? a.zL : a.rp);
    const int nk_all = tk.K / KC;
    const int kc0 = nk_all * rank / KS, kc1 = nk_all * (rank + 1) / KS;
    double cre[2][2][2], cim[2][2][2];
    zmma_main(tk, zc, dyn, a.A, srcA, srcB, n, R, kc0, kc1 - kc0, cre, cim);
    double2* red = dyn;
    __syncthreads();
    if (wk == 0 && rank > 0) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            red[(wq * 8 + (mt * 4 + nt * 2 + h)) * 32 + lane] = make_double2(cre[mt][nt][h], cim[mt][nt][h]);
    }
    cl.sync();
    if (rank == 0 && wk == 0) {
      for (int src = 1; src < KS; ++src) {
        const double2* rem = cl.map_shared_rank(red, src);
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const double2 o = rem[(wq * 8 + (mt * 4 + nt * 2 + h)) * 32 + lane];
              cre[mt][nt][h] += o.x;
              cim[mt][nt][h] += o.y;
            }
      }
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int row = tk.r0 + wm * 16 + mt * 8 + gid;
        if (row < tk.rlo || row >= tk.rhi) continue;
        const int q = row / n, p = row - q * n;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int j = wn * 16 + nt * 8 + 2 * tig + h;
            if (j >= tk.ncols) continue;
            const long long o0 = zc.out[j][q];
            if (o0 < 0) continue;
            const long long off = o0 + (long long)p * R;
            const double2 y = make_double2(cre[mt][nt][h], cim[mt][nt][h]);
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
      }
      __threadfence();
    }
    cl.sync();  // remote partials read; s_t free for the next ticket
    if (rank == 0) {
      for (int i = tid; i < ft.ninc; i += blockDim.x) atomicAdd(a.done + a.incs[ft.inc0 + i], 1);
    }
  }
}

// Batched complex GEMM on the DMMA pipe for the factorisation's solves
// (C = alpha A B + beta C, row-major, M, N, K multiples of 32): the
// contraction core above with tiles loaded straight from the matrices.
// grid (N / 32, M / 32, batch), 256 threads
__global__ void __launch_bounds__(THREADS) k_zgemm_dmma(int K, double2 alpha, const double2* __restrict__ A,
                                                        int lda, long long sa, const double2* __restrict__ B,
                                                        int ldb, long long sb, double2 beta, double2* C, int ldc,
                                                        long long sc) {
  extern __shared__ __align__(16) double2 dyn[];
  const int z = blockIdx.z;
  const double2* Ab = A + z * sa + (long long)blockIdx.y * 32 * lda;
  const double2* Bb = B + z * sb + (long long)blockIdx.x * 32;
  const int tid = threadIdx.x;
  auto load = [&](int stage, int kc) {
    const int k0 = kc * KC;
#pragma unroll
    for (int i = 0; i < (KC * BM) / THREADS; ++i) {  // A[m][k0 + kk] -> As[kk][m]
      const int el = tid + i * THREADS, m = el / KC, kk = el % KC;
      cp16(&zAs(dyn, stage, kk, m), Ab + (long long)m * lda + k0 + kk);
    }
#pragma unroll
    for (int i = 0; i < (KC * BN) / THREADS; ++i) {  // B[k0 + kk][j] -> Bs[kk][j]
      const int el = tid + i * THREADS, kk = el / BN, j = el % BN;
      cp16(&zBs(dyn, stage, kk, j), Bb + (long long)(k0 + kk) * ldb + j);
    }
  };
  double cre[2][2][2], cim[2][2][2];
  zmma_core(dyn, load, 0, K / KC, cre, cim);
  const int lane = tid & 31, warp = tid >> 5;
  const int wk = warp >> 2, wq = warp & 3;
  const int wm = wq >> 1, wn = wq & 1;
  const int gid = lane >> 2, tig = lane & 3;
  if (wk != 0) return;
  double2* Cb = C + z * sc + (long long)blockIdx.y * 32 * ldc + blockIdx.x * 32;
  const bool b0 = beta.x == 0.0 && beta.y == 0.0;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = wm * 16 + mt * 8 + gid, col = wn * 16 + nt * 8 + 2 * tig + h;
        double2* cp = Cb + (long long)row * ldc + col;
        const double2 acc = make_double2(cre[mt][nt][h], cim[mt][nt][h]);
        double2 v = cmul(alpha, acc);
        if (!b0) v = cadd(v, cmul(beta, *cp));
        *cp = v;
      }
}

bool zgemm_dmma(cudaStream_t st, int M, int N, int K, double2 alpha, const double2* A, int lda, long long sa,
                const double2* B, int ldb, long long sb, double2 beta, double2* C, int ldc, long long sc,
                int batch) {
  if (M % 32 || N % 32 || K % 32 || M == 0 || N == 0 || K == 0) return false;
  static const cudaError_t attr =
      cudaFuncSetAttribute(k_zgemm_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)(sizeof(double2) * STAGES * kStageElems));
  if (attr != cudaSuccess) return false;
  k_zgemm_dmma<<<dim3(N / 32, M / 32, batch), THREADS, sizeof(double2) * STAGES * kStageElems, st>>>(
      K, alpha, A, lda, sa, B, ldb, sb, beta, C, ldc, sc);
  return true;
}

constexpr size_t kZmmaSmem = sizeof(double2) * STAGES * kStageElems;

// k_zmma2 instantiations: (BN, TM, TN, n-major B, stages, persistent).
// 64-column tasks (steps with >= 1 task per SM): persistent, one CTA per SM;
// 32-column tasks (smaller steps): one task per CTA (one per SM: 4-stage ring,
// two warp groups splitting each chunk's k range), cluster split-K.
using Z2Slab64 = Z2<64, 2, 2, false, 3, true>;
using Z2Slab32 = Z2<32, 2, 2, false, 4, false, 2>;
using Z2Cols64 = Z2<64, 2, 2, true, 3, true>;
using Z2Cols32 = Z2<32, 2, 2, true, 4, false, 2>;
using Z2Cols32P = Z2<32, 2, 2, true, 4, true, 2>;
// n-major with 64-row k chunks (n % 64 == 0): one 32 KB map copy + 32 column
// copies of 1 KB per chunk, half the copies per k of the 32-row form (the
// n-major contraction is bound by the TMA unit's per-copy cost otherwise)
using Z2Cols32K = Z2<32, 2, 2, true, 2, false, 2, 64>;
using Z2Cols32PK = Z2<32, 2, 2, true, 2, true, 2, 64>;
#define Z2K_SLAB64 k_zmma2<64, 2, 2, false, 3, true, 1>
#define Z2K_SLAB32 k_zmma2<32, 2, 2, false, 4, false, 2>
#define Z2K_COLS64 k_zmma2<64, 2, 2, true, 3, true, 1>
#define Z2K_COLS32 k_zmma2<32, 2, 2, true, 4, false, 2>
#define Z2K_COLS32P k_zmma2<32, 2, 2, true, 4, true, 2>
#define Z2K_COLS32K k_zmma2<32, 2, 2, true, 2, false, 2, 64>
#define Z2K_COLS32PK k_zmma2<32, 2, 2, true, 2, true, 2, 64>

void launch_zmma(Ctx& c, const DevMma& m, const double2* A, const double2* srcA, const double2* srcB,
                 const double2* zeros, const Epi& e, int R) {
  if (m.ntasks == 0) return;
  static const bool pdl = !(getenv("HS_ZMMA_PDL") && atoi(getenv("HS_ZMMA_PDL")) == 0);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap with the previous step's tail
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 2 : 1;
  cfg.stream = c.stream;
  c.launches++;
  if (m.kind != 0) {
    int KS = 1;
    // persistent: 64-column slab tasks, or 32-column shared-map tasks when the
    // step has at least one per SM
    const bool pers = m.bn == 64 || (m.kind == 2 && m.ntasks >= c.num_sms);
    if (pers) {
      cfg.gridDim = dim3(std::min(m.ntasks, c.num_sms));
    } else {
      // split K over a cluster while the step's tasks leave SMs idle and every
      // rank keeps >= 2 chunks (HS_ZMMA2_KS caps the cluster size)
      static const int ks_cap = getenv("HS_ZMMA2_KS") ? atoi(getenv("HS_ZMMA2_KS")) : 8;
      while (KS < ks_cap && (long long)m.ntasks * KS * 2 <= c.num_sms && m.minK / Z2KC >= 4 * KS) KS *= 2;
      cfg.gridDim = dim3(m.ntasks * KS);
    }
    attr[0].val.clusterDim.x = KS;
    static const int test2 = getenv("HS_ZMMA2_TEST2CTA") ? atoi(getenv("HS_ZMMA2_TEST2CTA")) : 0;
    if (KS == 1 && test2 != 2) {  // no cluster launch at all when K is not split
      cfg.attrs = attr + 1;
      cfg.numAttrs = pdl ? 1 : 0;
    }
    // ticket slot of a persistent launch (a ring: consecutive, possibly
    // overlapping launches never share a counter); its claims = tasks + grid
    unsigned* ticket = nullptr;
    unsigned tbase = 0;
    if (pers) {  // the counters are allocated (zeroed) with the contraction tables (make_mma)
      const int slot = (int)(c.z2_seq++ % kZ2TicketSlots);
      ticket = c.z2_tickets + slot;
      tbase = c.z2_base[slot];
    }
    const long long Aelems = (long long)(A == c.Tcls ? c.Tcls_elems : c.T_elems);
    const long long LR = c.plan.L * (long long)R;
    unsigned long long* tr = nullptr;
    const int seq = (int)(c.launches & 0xFFFFFF);
    if (c.trace_on && c.trace && (size_t)c.trace_rows + cfg.gridDim.x <= c.trace_cap) {
      tr = c.trace + 6ull * c.trace_rows;
      c.trace_rows += (int)cfg.gridDim.x;
    }
#define Z2_LAUNCH(F, K)                                                                                         \
  do {                                                                                                          \
    cfg.blockDim = dim3(F::THREADS);                                                                            \
    cfg.dynamicSmemBytes = F::SMEM;                                                                             \
    cudaLaunchKernelEx(&cfg, K, (const MmaTask*)m.tasks, m.ntasks, (const MmaCol*)m.cols, A, srcA, srcB, zeros, \
                       e, c.n, R, KS, tr, seq, Aelems, LR, ticket, tbase);                                      \
  } while (0)
    // a persistent launch's claims are tasks + grid (every CTA's last claim
    // fails); counted only when the launch was accepted, so a failed launch
    // cannot shift the next launch's ticket base on this slot
    struct Claims {
      Ctx& c;
      bool pers;
      int slot, claims;
      ~Claims() {
        if (pers && cudaPeekAtLastError() == cudaSuccess) c.z2_base[slot] += (unsigned)claims;
      }
    } claims_{c, pers, (int)((c.z2_seq + kZ2TicketSlots - 1) % kZ2TicketSlots), m.ntasks + (int)cfg.gridDim.x};
    if (test2 && m.kind == 1 && m.bn == 32 && !pers) {  // diagnostics: the 2-CTA-per-SM form of round 2's first version
      using FT = Z2<32, 1, 2, false, 3, false, 1>;
      static const cudaError_t at = cudaFuncSetAttribute(k_zmma2<32, 1, 2, false, 3, false, 1>,
                                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FT::SMEM);
      (void)at;
      Z2_LAUNCH(FT, (k_zmma2<32, 1, 2, false, 3, false, 1>));
      return;
    }
    static const bool kc64 = !(getenv("HS_ZMMA2_KC64") && atoi(getenv("HS_ZMMA2_KC64")) == 0);
    const bool k64 = kc64 && m.kind == 2 && c.n % 64 == 0 && m.minK % 64 == 0;
    if (m.kind == 2 && m.bn == 64) Z2_LAUNCH(Z2Cols64, Z2K_COLS64);
    else if (m.kind == 2 && pers && k64) Z2_LAUNCH(Z2Cols32PK, Z2K_COLS32PK);
    else if (m.kind == 2 && pers) Z2_LAUNCH(Z2Cols32P, Z2K_COLS32P);
    else if (k64) Z2_LAUNCH(Z2Cols32K, Z2K_COLS32K);
    else if (m.kind == 2) Z2_LAUNCH(Z2Cols32, Z2K_COLS32);
    else if (m.bn == 64) Z2_LAUNCH(Z2Slab64, Z2K_SLAB64);
    else Z2_LAUNCH(Z2Slab32, Z2K_SLAB32);
#undef Z2_LAUNCH
    return;
  }
  // split K over a cluster when the step has too few tasks to fill the GPU
  const int minK = m.minK;
  int KS = 1;
  static int ks_max = getenv("HS_ZMMA_KS") ? atoi(getenv("HS_ZMMA_KS")) : 4;
  static int min_chunks = getenv("HS_ZMMA_MINCH") ? atoi(getenv("HS_ZMMA_MINCH")) : 4;
  while (KS < ks_max && (long long)m.ntasks * KS < 2LL * c.num_sms && minK / KC >= 2 * KS * min_chunks / 2) KS *= 2;
  attr[0].val.clusterDim.x = KS;
  cfg.gridDim = dim3(m.ntasks * KS);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = kZmmaSmem;
  cudaLaunchKernelEx(&cfg, k_zmma, (const MmaTask*)m.tasks, (const MmaCol*)m.cols, A, srcA, srcB, e,
                     c.n, R, KS);
}

// ---------------------------------------------------------------------------
// k_zmma2_df: the whole R-RHS BSP apply as ONE persistent dataflow launch on
// the k_zmma2 core (k-major slabs of R right-hand sides, or NMAJ: the shared
// class maps, one column per subdomain, KC = 64-row chunks where the faces
// allow).  The plan is build_fused_mma's: every 32-row x 32-column task of
// the forward steps (phase 0), the map-once residual step (1: only the rows
// where r' can be nonzero, as the per-step path) with fill tasks (3: rp = w =
// 0, z = zL on the other blocks; no contraction) and the backward steps (2)
// in schedule order (a topological order), with per-(block, 32-RHS chunk)
// completion counters it waits for / completes.  One CTA per SM: a producer
// warp claims tickets, stages the task's column table (double-buffered),
// streams the map chunks -- the first S before the task's dependencies are
// met, since maps depend on nothing -- waits for the dependencies, then
// streams the slab rows (after fence.proxy.async: generic-proxy stores of
// other CTAs, async-proxy reads here).  Two groups of 4 consumer warps split
// each chunk's k range; the tile goes through shared memory to a coalesced
// epilogue; warp 0 then releases the task's completion counters.  A task
// waits only for lower tickets, held by running CTAs: deadlock-free with every
// CTA resident (grid <= #SMs).  Phase arithmetic (k_zmma_fused's):
//   0 forward   y = T (zL | r):  zL += y
//   1 residual  y = T zL:        v = r - (zL - y); rp = w = v; z = zL + v
//   2 backward  y = T (w | rp):  w += y; z += y
//   3 fill      (no y):          rp = w = 0; z = zL
constexpr int kDfStages = 4;
template <int BN>
struct DfCols {
  ZCols2<BN> c;
  int phase, inc0, ninc, stop, ks, pair;
  unsigned long long* tr;
};

// BN = 16 (k-major slabs only): 32 x 16 tasks on four warp groups of two
// quadrant warps (8 warps x 12 accumulator chains again), per-(block, 16-RHS
// chunk) counters: twice the tasks at half the contraction each, for applies
// that are bound by their dependency chain rather than by the flops.
template <int S, bool NMAJ, int KC, int BN = 32>
__global__ void __launch_bounds__(Z2<BN, 2, 2, NMAJ, S, false, 64 / BN, KC>::THREADS, 1)
    k_zmma2_df(const __grid_constant__ FusedMmaArgs a) {
  constexpr int KG = 64 / BN;  // warp groups splitting each chunk's k range
  using F = Z2<BN, 2, 2, NMAJ, S, false, KG, KC>;
  static_assert(BN == 32 || (BN == 16 && !NMAJ), "task width");
  extern __shared__ __align__(128) double2 sm[];
  __shared__ __align__(8) unsigned long long full[S], empty[S], dfull[2], dempty[2];
  __shared__ DfCols<BN> zcs[2];
  double2* ys = sm + F::RING;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n, R = a.R;
  if (warp == F::NWC && lane == 0) {
    for (int i = 0; i < S; ++i) z2_bar_init(&full[i], 1), z2_bar_init(&empty[i], F::NWC);
    for (int i = 0; i < 2; ++i) z2_bar_init(&dfull[i], 1), z2_bar_init(&dempty[i], F::NWC);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == F::NWC) {  // ---------------- producer
    long long g = 0;
    for (int it = 0;; ++it) {
      const int d = it & 1;
      DfCols<BN>& zd = zcs[d];
      z2_wait(&dempty[d], (unsigned)((it >> 1) & 1) ^ 1);
      int t = 0;
      if (lane == 0) t = atomicAdd(a.ticket, 1);
      t = __shfl_sync(0xffffffffu, t, 0);
      if (t >= a.ntasks) {
        if (lane == 0) {
          zd.stop = 1;
          z2_arrive(&dfull[d]);
        }
        break;
      }
      unsigned long long* tr = a.trace ? a.trace + 6ull * t : nullptr;
      if (tr && lane == 0) tr[0] = z2_gtimer();
      const FusedMmaTask ft = a.tasks[t];
      const MmaTask tk = ft.task;
      // fill tasks (phase 3) carry no columns and no contraction
      HS_DCHECK(ft.phase == 3 ? tk.ncols == 0 && tk.K == 0 : tk.ncols >= 1 && tk.ncols <= BN && tk.K % KC == 0, DBG_INDEX);
      for (int j = lane; j < BN; j += 32) {
        if (j < tk.ncols) {
          const MmaCol c = a.cols[tk.col0 + j];
#pragma unroll
          for (int q = 0; q < 4; ++q) zd.c.in[j][q] = c.in[q], zd.c.out[j][q] = c.out[q], zd.c.slot[j][q] = c.slot[q];
          zd.c.r[j] = c.r;
          zd.c.alt[j] = c.alt;
        } else {
#pragma unroll
          for (int q = 0; q < 4; ++q) zd.c.in[j][q] = zd.c.out[j][q] = -1, zd.c.slot[j][q] = -1;
          zd.c.r[j] = 0;
          zd.c.alt[j] = 0;
        }
      }
      if (lane == 0) {
        zd.c.tk = tk;
        zd.phase = ft.phase;
        zd.inc0 = ft.inc0;
        zd.ninc = ft.ninc;
        zd.stop = 0;
        zd.tr = tr;
        zd.ks = ft.ks;
        zd.pair = ft.pair;
      }
      if (ft.phase == 3) {
        // fill task (map-once residual: rp = w = 0, z = zL on blocks the
        // residual does not reach): no contraction, no ring; the consumers
        // start it once its inputs are final
        for (int q = lane; q < ft.ndep; q += 32) {
          const FusedDep dp = a.deps[ft.dep0 + q];
          const volatile int* pc = a.done + dp.block;
          HS_WAIT(*pc < dp.count, 32, DBG_DEPWAIT);
        }
        __syncwarp();
        __threadfence();
        if (tr && lane == 0) tr[1] = tr[2] = z2_gtimer();
        __syncwarp();
        if (lane == 0) z2_arrive(&dfull[d]);
        continue;
      }
      __syncwarp();
      if (lane == 0) z2_arrive(&dfull[d]);  // release: the table is visible to the consumers
      const double2* srcA = ft.phase == 0 ? a.zL : (ft.phase == 1 ? a.zL : a.w);
      const double2* srcB = ft.phase == 0 ? a.r : (ft.phase == 1 ? a.zL : a.rp);
      const int nkall = tk.K / KC;
      const int kc0 = ft.ks == 1 ? nkall / 2 : 0;
      const int nk = ft.ks == 0 ? nkall / 2 : nkall - kc0;
      // n-major: all 32 column rows (absent faces and padding columns read zeros)
      // (a tensor copy of the slab rows always delivers its whole box: BN + 2 columns)
      const bool tmb = !NMAJ && a.use_tm;
      const unsigned bytes = (unsigned)(KC * 32 * sizeof(double2)) +
                             (unsigned)(KC * (NMAJ ? 32 : (tmb ? BN + 2 : tk.ncols)) * sizeof(double2));
      const double2* Ab = a.A + tk.a_off;
      const double2* base = NMAJ ? nullptr : (zd.c.alt[0] ? srcB : srcA) + zd.c.in[0][0];
      // tensor-copy coordinates of the slab: vector (zL, r, w, rp), first row, first column (in doubles)
      const int tmi = ft.phase == 2 ? (zd.c.alt[0] ? 3 : 2) : ((ft.phase == 0 && zd.c.alt[0]) ? 1 : 0);
      const int tmx = 2 * zd.c.r[0];
      const int tmy = NMAJ ? 0 : (int)((zd.c.in[0][0] - zd.c.r[0]) / R);
      auto issueA = [&](int st, int kc) {
        if (lane == 0)
          z2_copy(sm + (size_t)st * F::STAGE, Ab + (long long)kc * KC * 32, KC * 32 * sizeof(double2), &full[st]);
      };
      auto issueB = [&](int st, int kc) {
        double2* sb = sm + (size_t)st * F::STAGE + KC * F::SA;
        if (NMAJ) {
          // column j (a subdomain): the chunk's KC positions of face q, one run
          const int k0 = kc * KC, q = k0 / n, p0 = k0 - q * n;
          const int j = lane;
          const long long off = zd.c.in[j][q];
          HS_DCHECK(off < 0 || off + (long long)(p0 + KC - 1) * R < a.LR, DBG_VEC);
          const double2* src = off >= 0 ? (zd.c.alt[j] ? srcB : srcA) + off + (long long)p0 * R : a.zeros;
          z2_copy(sb + j * F::SB, src, KC * sizeof(double2), &full[st]);
        } else {
          if (tmb) {
            // ONE tensor copy of the chunk's KC slab rows x (BN + 2) columns (the
            // padded row stride of the fragment loads; columns past R read as
            // zeros).  A bulk copy per row kept the TMA unit busy ~60 cycles per
            // row, ~1 us per chunk: that, not the DMMAs, bounded a contraction.
            HS_DCHECK(tmy >= 0 && (long long)(tmy + (kc + 1) * KC) * R <= a.LR, DBG_VEC);
            if (lane == 0)
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                      z2_smem(sb)),
                  "l"(&a.tm[tmi]), "r"(tmx), "r"(tmy + kc * KC), "r"(z2_smem(&full[st]))
                  : "memory");
          } else {
            const double2* b0 = base + (long long)kc * KC * R;
            for (int r = lane; r < KC; r += 32)
              z2_copy(sb + r * F::SB, b0 + (long long)r * R, tk.ncols * sizeof(double2), &full[st]);
          }
        }
      };
      // the map chunks of the first stages stream while the dependencies settle
      const int pre = nk < S ? nk : S;
      const long long g0 = g;
      for (int i = 0; i < pre; ++i, ++g) {
        const int st = (int)(g % S);
        if (g >= S) z2_wait(&empty[st], (unsigned)((g / S) & 1) ^ 1);
        if (lane == 0) z2_expect_tx(&full[st], bytes);
        __syncwarp();
        issueA(st, kc0 + i);
      }
      for (int q = lane; q < ft.ndep; q += 32) {
        const FusedDep dp = a.deps[ft.dep0 + q];
        const volatile int* pc = a.done + dp.block;
        HS_WAIT(*pc < dp.count, 32, DBG_DEPWAIT);
      }
      __syncwarp();
      __threadfence();
      asm volatile("fence.proxy.async.global;" ::: "memory");
      if (tr && lane == 0) tr[1] = z2_gtimer();
      for (int i = 0; i < pre; ++i) issueB((int)((g0 + i) % S), kc0 + i);
      for (int i = pre; i < nk; ++i, ++g) {
        const int st = (int)(g % S);
        z2_wait(&empty[st], (unsigned)((g / S) & 1) ^ 1);
        if (lane == 0) z2_expect_tx(&full[st], bytes);
        __syncwarp();
        issueA(st, kc0 + i);
        issueB(st, kc0 + i);
      }
    }
    return;
  }
  // ---------------- consumers (warps 0 .. 7: two groups of 4 quadrant warps)
  const int kg = warp / F::NWQ, wq = warp % F::NWQ;
  const int wm = wq / F::WN, wn = wq % F::WN;
  const int gid = lane >> 2, tig = lane & 3;
  constexpr int KH = KC / KG;
  constexpr int NT = 2 * 2 * 2;
  // output element el of the 32 x 32 tile: k-major row-major (consecutive
  // right-hand sides), n-major column-major (consecutive rows of a column)
  auto el_rr = [](int el) { return NMAJ ? el % 32 : el / BN; };
  auto el_j = [](int el) { return NMAJ ? el / 32 : el % BN; };
  long long g = 0;
  for (int it = 0;; ++it) {
    const int d = it & 1;
    z2_wait(&dfull[d], (unsigned)((it >> 1) & 1));
    const DfCols<BN>& zd = zcs[d];
    if (zd.stop) break;
    const MmaTask tk = zd.c.tk;
    const int phase = zd.phase, ks = zd.ks;
    unsigned long long* tr = zd.tr;
    if (phase == 3) {
      // fill: counter k2 = block * nch + RHS chunk covers positions 0..n-1 of
      // the block, right-hand sides BN ch .. BN ch + BN - 1 (< R)
      const int nch = (R + BN - 1) / BN, cw = R < BN ? R : BN;
      const int per = n * cw;
      for (int i = 0; i < zd.ninc; ++i) {
        const int k2 = a.incs[zd.inc0 + i];
        const int blk = k2 / nch, r0 = (k2 - blk * nch) * BN;
        for (int e = tid; e < per; e += F::NWC * 32) {
          const int p = e / cw, r = r0 + e - (e / cw) * cw;
          if (r >= R) continue;
          const long long t = ((long long)blk * n + p) * R + r;
          HS_DCHECK(t < a.LR, DBG_VEC);
          a.rp[t] = make_double2(0.0, 0.0);
          a.w[t] = make_double2(0.0, 0.0);
          a.z[t] = __ldcg(a.zL + t);
        }
      }
      if (tr && tid == 0) tr[3] = z2_gtimer();
      consumers_bar<F::NWC * 32>();  // every fill store issued
      if (warp == 0) {
        __threadfence();
        for (int i = lane; i < zd.ninc; i += 32) atomicAdd(a.done + a.incs[zd.inc0 + i], 1);
        if (tr && lane == 0) {
          unsigned smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          tr[4] = z2_gtimer();
          tr[5] = ((unsigned long long)smid << 32) | ((unsigned long long)blockIdx.x << 8) | 3u;
        }
      }
      __syncwarp();
      if (lane == 0) z2_arrive(&dempty[d]);
      continue;
    }
    const int nk = ks == 0 ? tk.K / KC / 2 : (ks == 1 ? tk.K / KC - tk.K / KC / 2 : tk.K / KC);
    double cr[2][2][2], ci[2][2][2], p3[2][2][2];
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int c = 0; c < 2; ++c) cr[x][y][c] = ci[x][y][c] = p3[x][y][c] = 0.0;
    long long toff[F::EPT];
    double2 u1[F::EPT], u2[F::EPT];
    for (int i = 0; i < nk; ++i, ++g) {
      const int st = (int)(g % S);
      z2_wait(&full[st], (unsigned)((g / S) & 1));
      if (i == 0) {
        if (tr && tid == 0) tr[2] = z2_gtimer();
        // the first chunk landed, so the producer saw every dependency met: the
        // epilogue operands are final -- fetch them now, in the contraction's shadow
#pragma unroll
        for (int u = 0; u < F::EPT; ++u) {
          const int el = u * F::NWC * 32 + tid;
          const int rr = el_rr(el), j = el_j(el);
          const int row = tk.r0 + rr;
          long long t = -1;
          if (row >= tk.rlo && row < tk.rhi && j < tk.ncols) {
            const int q = row / n, p = row - q * n;
            const long long off = zd.c.out[j][q];
            if (off >= 0) t = off + (long long)p * R;
          }
          toff[u] = t;
          if (t >= 0) {
            if (phase == 0) u1[u] = __ldcg(a.zL + t);
            else if (phase == 1) { u1[u] = __ldcg(a.r + t); u2[u] = __ldcg(a.zL + t); }
            else { u1[u] = __ldcg(a.w + t); u2[u] = __ldcg(a.z + t); }
          }
        }
      }
      const double2* sa = sm + (size_t)st * F::STAGE;
      const double2* sb = sa + KC * F::SA;
#pragma unroll
      for (int kk = 0; kk < KH; kk += 4) {
        const int k4 = kg * KH + kk;
        double2 av[2], bv[2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) av[mt] = sa[(k4 + tig) * F::SA + (wm * 2 + mt) * 8 + gid];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
          bv[nt] = NMAJ ? sb[((wn * 2 + nt) * 8 + gid) * F::SB + k4 + tig] : sb[(k4 + tig) * F::SB + (wn * 2 + nt) * 8 + gid];
        double s_b[2];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) s_b[nt] = bv[nt].x + bv[nt].y;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          const double s_a = av[mt].x + av[mt].y;
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) dmma(cr[mt][nt][0], cr[mt][nt][1], av[mt].x, bv[nt].x);
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) dmma(ci[mt][nt][0], ci[mt][nt][1], av[mt].y, bv[nt].y);
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) dmma(p3[mt][nt][0], p3[mt][nt][1], s_a, s_b[nt]);
        }
      }
      __syncwarp();
      if (lane == 0) z2_arrive(&empty[st]);
    }
#pragma unroll
    for (int x = 0; x < 2; ++x)
#pragma unroll
      for (int y = 0; y < 2; ++y)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          const double s1 = cr[x][y][c], s2 = ci[x][y][c];
          cr[x][y][c] = s1 - s2;
          ci[x][y][c] = p3[x][y][c] - s1 - s2;
        }
    if (tr && tid == 0) tr[3] = z2_gtimer();
    // groups 1 .. KG-1 hand their partial tiles to group 0 through the area past
    // the output tile; group 0 adds them in group order and writes the tile
    double2* red = ys + 32 * F::YS;
    consumers_bar<F::NWC * 32>();  // the previous task's tile readers are done
    if (kg > 0) {
      double2* mine = red + (size_t)(kg - 1) * F::NWQ * NT * 32;
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y)
#pragma unroll
          for (int c = 0; c < 2; ++c) mine[(wq * NT + (x * 2 + y) * 2 + c) * 32 + lane] = make_double2(cr[x][y][c], ci[x][y][c]);
    }
    consumers_bar<F::NWC * 32>();
    if (kg == 0) {
#pragma unroll
      for (int x = 0; x < 2; ++x)
#pragma unroll
        for (int y = 0; y < 2; ++y)
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            double2 t = make_double2(cr[x][y][c], ci[x][y][c]);
#pragma unroll
            for (int g2 = 1; g2 < KG; ++g2) {
              const double2 o = red[(size_t)(g2 - 1) * F::NWQ * NT * 32 + (wq * NT + (x * 2 + y) * 2 + c) * 32 + lane];
              t.x += o.x;
              t.y += o.y;
            }
            ys[((wm * 2 + x) * 8 + gid) * F::YS + (wn * 2 + y) * 8 + 2 * tig + c] = t;
          }
    }
    consumers_bar<F::NWC * 32>();
    bool finish = true;
    const double2* other = nullptr;
    if (ks >= 0) {
      // split-K: publish this half's tile; the pair's second arrival adds the
      // halves in half order (deterministic) and finishes the task
      __shared__ int s_old;
      double2* mine = a.split_buf + ((size_t)zd.pair * 2 + ks) * 1024;
#pragma unroll
      for (int u = 0; u < F::EPT; ++u) {
        const int el = u * F::NWC * 32 + tid;
        mine[el] = ys[el_rr(el) * F::YS + el_j(el)];
      }
      consumers_bar<F::NWC * 32>();
      if (tid == 0) {
        __threadfence();
        s_old = atomicAdd(a.split_cnt + zd.pair, 1);
        __threadfence();
      }
      consumers_bar<F::NWC * 32>();
      finish = s_old & 1;
      other = a.split_buf + ((size_t)zd.pair * 2 + (1 - ks)) * 1024;
    }
    // coalesced epilogue (el_rr / el_j)
#pragma unroll
    for (int u = 0; u < F::EPT; ++u) {
      const long long t = toff[u];
      if (t < 0 || !finish) continue;
      const int el = u * F::NWC * 32 + tid;
      double2 y = ys[el_rr(el) * F::YS + el_j(el)];
      if (ks >= 0) {
        const double2 o = __ldcg(other + el);
        y = ks == 0 ? cadd(y, o) : cadd(o, y);
      }
      if (phase == 0) {
        a.zL[t] = cadd(u1[u], y);
      } else if (phase == 1) {
        const double2 v = csub(u1[u], csub(u2[u], y));
        a.rp[t] = v;
        a.w[t] = v;
        a.z[t] = cadd(u2[u], v);
      } else {
        a.w[t] = cadd(u1[u], y);
        a.z[t] = cadd(u2[u], y);
      }
    }
    consumers_bar<F::NWC * 32>();  // every epilogue store of the task issued
    if (warp == 0) {
      // release the task's outputs, then count them done: one counter per lane
      // (a shared-map task completes up to 32 blocks; one thread walking the
      // list serialised a dependent load per counter, ~10 us per task)
      if (finish) {
        __threadfence();
        for (int i = lane; i < zd.ninc; i += 32) atomicAdd(a.done + a.incs[zd.inc0 + i], 1);
      }
      if (tr && lane == 0) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        tr[4] = z2_gtimer();
        tr[5] = ((unsigned long long)smid << 32) | ((unsigned long long)blockIdx.x << 8) | (unsigned)phase;
      }
    }
    __syncwarp();
    if (lane == 0) z2_arrive(&dempty[d]);
  }
}

// vec as a [L][2 R] FP64 tensor, box = (2 cols doubles) x rows; false when the
// driver entry point or the encoding is not available (the caller falls back
// to a bulk copy per row)
static bool encode_slab_tensor(CUtensorMap* tm, const double2* vec, long long L, int R, int cols, int rows) {
  typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Encode enc = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (Encode)fn;
  }();
  if (!enc || ((uintptr_t)vec & 15) || L <= 0) return false;
  const cuuint64_t gdim[2] = {(cuuint64_t)2 * R, (cuuint64_t)L};
  const cuuint64_t gstr[1] = {(cuuint64_t)R * sizeof(double2)};
  const cuuint32_t box[2] = {(cuuint32_t)2 * cols, (cuuint32_t)rows};
  const cuuint32_t estr[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)vec, gdim, gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_zmma_fused(Ctx& c, const DevFusedMma& f, FusedMmaArgs a) {
  cudaError_t e = cudaMemsetAsync(f.counters, 0, (f.ncounters + 1) * sizeof(int), c.stream);
  if (e != cudaSuccess) return e;
  a.tasks = f.tasks; a.cols = f.cols; a.deps = f.deps; a.incs = f.incs;
  a.split_buf = f.split_buf; a.split_cnt = f.split_cnt;
  a.done = f.counters; a.ticket = f.counters + f.ncounters;
  a.ntasks = f.ntasks; a.n = c.n;
  // the k_zmma2 core for per-subdomain slabs (32-column tasks of consecutive
  // right-hand sides); HS_ZMMA2=0 keeps k_zmma_fused
  static const bool z2 = !(getenv("HS_ZMMA2") && atoi(getenv("HS_ZMMA2")) == 0);
  // the shared class maps with one right-hand side: the n-major form (one
  // column per subdomain), 64-row k chunks when the faces allow (half the
  // bulk copies per k, two stages), else 32-row chunks in four stages
  static const bool kc64 = !(getenv("HS_ZMMA2_KC64") && atoi(getenv("HS_ZMMA2_KC64")) == 0);
  const bool nmaj = z2 && f.shared && f.R == 1 && c.zeros;
  if (z2 && (!f.shared || nmaj)) {
    if (c.trace_on && c.trace && (size_t)f.ntasks <= c.trace_cap) {
      a.trace = c.trace;
      c.trace_rows = f.ntasks;
    }
    a.zeros = c.zeros;
    a.LR = c.plan.L * (long long)f.R;
    // the slab rows of the k-major form by tensor copies (HS_ZMMA2_DF_TM=0: a bulk copy per row)
    static const bool tm_env = !(getenv("HS_ZMMA2_DF_TM") && atoi(getenv("HS_ZMMA2_DF_TM")) == 0);
    if (!nmaj && tm_env) {  // (a box wider than the R columns reads zeros past them: tests at R = 16)
      const double2* vecs[4] = {a.zL, a.r, a.w, a.rp};
      a.use_tm = 1;
      for (int i = 0; i < 4 && a.use_tm; ++i)
        if (!encode_slab_tensor(&a.tm[i], vecs[i], c.plan.L, f.R, f.cw + 2, 32)) a.use_tm = 0;
    }
    auto go = [&](auto kern, auto tag) -> cudaError_t {
      using F = decltype(tag);
      constexpr size_t smem =
          F::SMEM + sizeof(double2) * 32 * F::YS + sizeof(double2) * (F::NWC / F::NWQ - 1) * F::NWQ * 8 * 32;
      const cudaError_t at = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (at != cudaSuccess) return at;
      c.launches++;
      kern<<<std::min(f.ntasks, c.num_sms), F::THREADS, smem, c.stream>>>(a);
      return cudaGetLastError();
    };
    if (!nmaj && f.cw == 16) return go(k_zmma2_df<kDfStages, false, 32, 16>, Z2<16, 2, 2, false, kDfStages, false, 4>());
    if (!nmaj) return go(k_zmma2_df<kDfStages, false, 32>, Z2<32, 2, 2, false, kDfStages, false, 2>());
    if (kc64 && c.n % 64 == 0 && f.minK % 64 == 0)
      return go(k_zmma2_df<2, true, 64>, Z2<32, 2, 2, true, 2, false, 2, 64>());
    return go(k_zmma2_df<kDfStages, true, 32>, Z2<32, 2, 2, true, kDfStages, false, 2>());
  }
  // K split over a cluster: KS ranks each keep >= 2 K chunks (HS_ZMMA_FUSED_KS overrides)
  static const int ks_env = getenv("HS_ZMMA_FUSED_KS") ? atoi(getenv("HS_ZMMA_FUSED_KS")) : 0;
  int KS = ks_env > 0 ? ks_env : 1;
  if (ks_env <= 0)
    while (KS < 4 && f.minK / KC >= 4 * KS) KS *= 2;
  KS = KS >= 4 ? 4 : (KS >= 2 ? 2 : 1);
  c.launches++;
  if (KS == 1) {
    static int per_sm = 0;
    if (per_sm == 0) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_zmma_fused, THREADS, kZmmaSmem);
      if (per_sm < 1) per_sm = 1;
    }
    const int grid = std::max(1, std::min(f.ntasks, per_sm * c.num_sms));
    k_zmma_fused<<<grid, THREADS, kZmmaSmem, c.stream>>>(a);
    return cudaGetLastError();
  }
  const void* fn = KS == 2 ? (const void*)k_zmma_fused_ks<2> : (const void*)k_zmma_fused_ks<4>;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = kZmmaSmem;
  cfg.stream = c.stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = KS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  static int max_clusters[5] = {0, 0, 0, 0, 0};
  if (max_clusters[KS] == 0) {
    cfg.gridDim = dim3(KS * c.num_sms);
    cudaOccupancyMaxActiveClusters(&max_clusters[KS], fn, &cfg);
    if (max_clusters[KS] < 1) max_clusters[KS] = 1;
  }
  cfg.gridDim = dim3(KS * std::max(1, std::min(f.ntasks, max_clusters[KS])));
  void* args[] = {(void*)&a};
  return cudaLaunchKernelExC(&cfg, fn, args);
}

cudaError_t set_zmma_smem_limit() {
  cudaFuncSetAttribute(k_zmma_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kZmmaSmem);
  cudaFuncSetAttribute(k_zmma_fused_ks<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kZmmaSmem);
  cudaFuncSetAttribute(k_zmma_fused_ks<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kZmmaSmem);
  cudaFuncSetAttribute(Z2K_SLAB64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Slab64::SMEM);
  cudaFuncSetAttribute(Z2K_SLAB32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Slab32::SMEM);
  cudaFuncSetAttribute(Z2K_COLS64, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cols64::SMEM);
  cudaFuncSetAttribute(Z2K_COLS32, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cols32::SMEM);
  cudaFuncSetAttribute(Z2K_COLS32P, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cols32P::SMEM);
  cudaFuncSetAttribute(Z2K_COLS32K, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cols32K::SMEM);
  cudaFuncSetAttribute(Z2K_COLS32PK, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z2Cols32PK::SMEM);
  return cudaFuncSetAttribute(k_zmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kZmmaSmem);
}

// Row-major (rows x cols) map -> strip-major [rows/32][cols][32], zero-padded rows.
__global__ void k_pack_strips(const double2* T4, double2* out, int rows, int cols) {
  const long long strips = (rows + 31) / 32;
  const long long total = strips * cols * 32;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const int lane = (int)(i % 32);
    const long long rest = i / 32;
    const int col = (int)(rest % cols);
    const int strip = (int)(rest / cols);
    const int row = strip * 32 + lane;
    out[i] = row < rows ? T4[(long long)row * cols + col] : make_double2(0, 0);
  }
}

void launch_pack_strips(Ctx& c, const double2* T4, double2* out, int rows, int cols) {
  c.launches++;
  k_pack_strips<<<4 * c.num_sms, 256, 0, c.stream>>>(T4, out, rows, cols);
}

HS_DBG_ACCESSOR(hs_dbg_take_zmma)

}  // namespace hs
