// Device helpers shared by the kernels.
#pragma once
#include <cuda_runtime.h>

#include "hs_ctx.h"

namespace hs {

// ---- device-side checks (the debug library, -DHS_DEVICE_CHECKS:
// libhsb200_debug.so; compute-sanitizer is unavailable on this GPU pool).
// HS_DCHECK: index / range asserts on every table and vector access of the
// dataflow kernels; HS_WAIT: every spin-wait of a cross-CTA protocol (block
// completion counters, grid barriers, mbarrier rings, peer flags) with a
// watchdog (~2 s) so a protocol bug reports instead of hanging.  The first
// failure of a translation unit is kept as (line << 8 | tag); hs_debug_check
// collects them.  In the release library both macros are the plain code.
enum DbgTag { DBG_INDEX = 1, DBG_MAP = 2, DBG_VEC = 3, DBG_COUNTER = 4, DBG_DEPWAIT = 5, DBG_MBAR = 6,
              DBG_GRIDBAR = 7, DBG_PEER = 8, DBG_SMEM = 9 };
#ifdef HS_DEVICE_CHECKS
static __device__ unsigned long long g_hs_dbg;
static __device__ __noinline__ void hs_dbg_fail(unsigned tag, unsigned line) {
  atomicCAS(&g_hs_dbg, 0ull, (1ull << 63) | ((unsigned long long)line << 8) | tag);
}
#define HS_DCHECK(cond, tag)                     \
  do {                                           \
    if (!(cond)) ::hs::hs_dbg_fail((tag), __LINE__); \
  } while (0)
#define HS_WAIT(still_waiting, ns, tag)                        \
  do {                                                         \
    unsigned long long hs_n_ = 0;                              \
    while (still_waiting) {                                    \
      __nanosleep(ns);                                         \
      if (++hs_n_ > (1ull << 26)) {                            \
        ::hs::hs_dbg_fail((tag), __LINE__);                    \
        break;                                                 \
      }                                                        \
    }                                                          \
  } while (0)
// one accessor per translation unit: the first failure, then cleared
#define HS_DBG_ACCESSOR(name)                                             \
  unsigned long long name() {                                             \
    unsigned long long v = 0, z = 0;                                      \
    cudaMemcpyFromSymbol(&v, ::hs::g_hs_dbg, sizeof(v));                  \
    cudaMemcpyToSymbol(::hs::g_hs_dbg, &z, sizeof(z));                    \
    return v;                                                             \
  }
#else
#define HS_DCHECK(cond, tag) \
  do {                       \
  } while (0)
#define HS_WAIT(still_waiting, ns, tag) \
  do {                                  \
    while (still_waiting) __nanosleep(ns); \
  } while (0)
#define HS_DBG_ACCESSOR(name) \
  unsigned long long name() { return 0; }
#endif

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// acc += a * b
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
// acc += conj(a) * b
__device__ __forceinline__ void cfma_conj(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(-a.y, b.x, acc.y);
}

// Streaming 128-bit load of a map element: read-only path, no L1 allocation.
__device__ __forceinline__ double2 ld_stream(const double2* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
// The same with an L2 cache policy (map elements are read once per apply:
// evict-first keeps the re-read interface vectors L2-resident).
__device__ __forceinline__ unsigned long long l2_evict_first() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ unsigned long long l2_evict_last() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double2 ld_stream(const double2* p, unsigned long long pol) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(v.x), "=d"(v.y)
               : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ void epi_apply(const Epi& e, long long t, double2 y) {
  switch (e.mode) {
    case EPI_SET: e.o1[t] = y; break;
    case EPI_ACC: e.o1[t] = cadd(e.o1[t], y); break;
    case EPI_IMS: e.o1[t] = csub(e.a[t], y); break;
    case EPI_RESID: {
      // r' = b - (zL - S zL)  (SPEC.md:343 with interface_system.py:144-146 order)
      double2 zl = e.b[t];
      double2 v = csub(e.a[t], csub(zl, y));
      e.o1[t] = v;
      e.o2[t] = v;
      e.o3[t] = cadd(zl, v);
    } break;
    case EPI_LATE: e.o1[t] = cadd(csub(e.a[t], e.b[t]), csub(e.c[t], y)); break;
    case EPI_ACC2:
      e.o1[t] = cadd(e.o1[t], y);
      e.o2[t] = cadd(e.o2[t], y);
      break;
  }
}

// Send-buffer routing of a face's output (row-band exchange); returns true if routed.
__device__ __forceinline__ bool epi_route(const Epi& e, int slot, long long p, double2 y) {
  if (slot == -1) return false;
  if (slot >= 0) e.send_up[p + 0] = y;
  else e.send_dn[p + 0] = y;
  return true;
}

}  // namespace hs
