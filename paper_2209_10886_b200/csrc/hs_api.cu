// C ABI (include/hsb200.h): context lifecycle, factorisation driver, sweep
// orchestration, GMRES loop, introspection and the row-band exchange.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdlib>
#include <cstring>
#include <map>
#include <queue>
#include <type_traits>
#include <tuple>
#include <set>
#include <string>
#include <vector>

#include "../../include/hsb200.h"
#include "hs_ctx.h"
#include "hs_kernels.h"

using namespace hs;

struct hs_ctx : public Ctx {};

namespace hs {
// One in-place sum over the ranks of the context (GMRES inner products): the
// peer-memory all-reduce when the ranks' regions are mapped (hs_peer_open) --
// one kernel, fixed rank order, no host call -- else ncclAllReduce.
cudaError_t allreduce_sum_doubles(Ctx& c, double* buf, size_t count, void* comm) {
  PeerRanks& p = c.peer;
  if (p.G > 1 && p.red_on && count <= (size_t)kPeerRedCap) {
    PeerRedArgs a;
    a.G = p.G;
    a.self = c.plan.rank;
    a.count = (int)count;
    a.epoch = ++p.red_epoch;
    for (int g = 0; g < p.G; ++g) {
      a.data[g] = p.red_data[g];
      a.flag[g] = p.red_flag[g];
      a.consumed[g] = p.red_consumed[g];
    }
    a.buf[0] = buf;
    return launch_peer_allreduce(c, a);
  }
  ncclResult_t r = ncclAllReduce(buf, buf, count, ncclDouble, ncclSum, (ncclComm_t)comm, c.stream);
  if (r != ncclSuccess) {
    c.err = std::string("ncclAllReduce: ") + ncclGetErrorString(r);
    return cudaErrorUnknown;
  }
  return cudaSuccess;
}
}  // namespace hs

static std::string g_create_err;

#define HS_VERSION "hsb200 0.1.0 sm_100a complex128"

namespace {

int fail(Ctx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  else g_create_err = msg;
  return code;
}

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess)                                                           \
      return fail(c, -1, std::string(#call) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define NK(call)                                                                     \
  do {                                                                               \
    ncclResult_t r_ = (call);                                                        \
    if (r_ != ncclSuccess)                                                           \
      return fail(c, -2, std::string(#call) + ": " + ncclGetErrorString(r_));       \
  } while (0)

#define NEED_GPU(c)                                                                  \
  do {                                                                               \
    if ((c)->device < 0) return fail(c, 2, "plan-only context (device -1) cannot run kernels"); \
  } while (0)

// Every entry point that can touch the GPU runs on the context's device and
// restores the caller's current device on return: two contexts on two GPUs in
// one process, or a torch.cuda.set_device between calls, must not launch into
// another device's streams or allocate the workspace on the wrong GPU.
struct DeviceScope {
  int prev = -1;
  bool restore = false;
  explicit DeviceScope(const Ctx* c) {
    if (!c || c->device < 0) return;
    if (cudaGetDevice(&prev) == cudaSuccess && prev != c->device)
      restore = cudaSetDevice(c->device) == cudaSuccess;
  }
  ~DeviceScope() {
    if (restore) cudaSetDevice(prev);
  }
};
#define DEV_SCOPE(c) DeviceScope dev_scope_(c)

// Device allocations of a context are tracked by pointer so hs_memory is exact
// whatever the caller passes as size to dfree.
cudaError_t dalloc(Ctx* c, void** p, size_t bytes) {
  cudaError_t e = cudaMalloc(p, bytes > 0 ? bytes : 16);
  if (e == cudaSuccess) {
    c->alloc_sz[*p] = bytes;
    c->dev_bytes += (int64_t)bytes;
  }
  return e;
}

void dfree(Ctx* c, void* p, size_t /*bytes*/) {
  if (!p) return;
  auto it = c->alloc_sz.find(p);
  if (it != c->alloc_sz.end()) {
    c->dev_bytes -= (int64_t)it->second;
    c->alloc_sz.erase(it);
  }
  cudaFree(p);
}

// Temporaries of one call, freed when it returns (including error returns).
struct TmpAllocs {
  Ctx* c;
  std::vector<void*> p;
  explicit TmpAllocs(Ctx* ctx) : c(ctx) {}
  ~TmpAllocs() {
    for (void* q : p) dfree(c, q, 0);
  }
  template <class T>
  cudaError_t alloc(T** out, size_t bytes) {
    *out = nullptr;
    cudaError_t e = dalloc(c, (void**)out, bytes);
    if (e == cudaSuccess) p.push_back(*out);
    return e;
  }
  void add(void* q) {
    if (q) p.push_back(q);
  }
};

// Named, grow-only device work buffers.
int ws_get(Ctx* c, const std::string& name, size_t elems, double2** out) {
  Workspace& w = c->ws[name];
  if (w.cap < elems) {
    dfree(c, w.p, w.cap * sizeof(double2));
    w.p = nullptr;
    w.cap = 0;
    CK(dalloc(c, (void**)&w.p, elems * sizeof(double2)));
    w.cap = elems;
  }
  *out = w.p;
  return 0;
}

template <class T>
int upload(Ctx* c, T** dptr, const std::vector<T>& v) {
  if (v.empty()) {
    *dptr = nullptr;
    return 0;
  }
  CK(dalloc(c, (void**)dptr, v.size() * sizeof(T)));
  // Stream-ordered: the kernels run on a non-blocking stream, which does not
  // order against a legacy-stream cudaMemcpy (whose pageable H2D copy may
  // return before the DMA lands).  Pageable source -> staged before return.
  CK(cudaMemcpyAsync(*dptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, c->stream));
  return 0;
}

void free_step(Ctx* c, DevStep& s) {
  dfree(c, s.items, s.nitems * sizeof(DevItem));
  dfree(c, s.tiles, s.ntiles * sizeof(DevTile));
  dfree(c, s.recv, s.nrecv * sizeof(DevRecv));
  for (auto& kv : s.mma) {
    dfree(c, kv.second.tasks, kv.second.ntasks * sizeof(MmaTask));
    dfree(c, kv.second.cols, kv.second.ncols * sizeof(MmaCol));
  }
  s = DevStep();
}

// DMMA contraction tasks of a step (host vectors).  shared = false:
// per-subdomain maps (compact faces, rows of T_s), R right-hand sides per slab.
// shared = true: the class maps (4 faces W,S,N,E), one column per (subdomain,
// RHS), items of the same class and face range batched into one contraction.
void build_mma_host(Ctx* c, const StepTable& host, int R, bool shared, std::vector<MmaTask>& tasks,
                    std::vector<MmaCol>& cols, double& flops, int bn = 32) {
  const Plan& P = c->plan;
  const int n = c->n;
  auto col_for = [&](const Item& item, int r, bool global_faces) {
    const SubPlan& sp = P.subs[item.s];
    MmaCol col;
    for (int q = 0; q < 4; ++q) { col.in[q] = -1; col.out[q] = -1; col.slot[q] = -1; }
    for (int q = 0; q < sp.k; ++q) {
      const int f = global_faces ? sp.face[q] : q;
      col.in[f] = ((long long)sp.first_block * n + (long long)q * n) * R + r;
      const int r0 = q * n, r1 = (q + 1) * n;
      if (r1 <= item.rlo || r0 >= item.rhi) continue;  // face not produced by this item
      col.out[f] = (long long)sp.tgt_block[q] * n * R + r;
      col.slot[f] = item.slot[q];
    }
    col.r = r;
    col.alt = item.alt;
    return col;
  };
  if (!shared) {
    for (const Item& item : host.items) {
      const SubPlan& sp = P.subs[item.s];
      const int K = sp.k * n;
      for (int r0 = (item.rlo / 32) * 32; r0 < item.rhi; r0 += 32)
        for (int c0 = 0; c0 < R; c0 += bn) {
          MmaTask tk;
          tk.a_off = sp.T_off + (long long)(r0 / 32) * K * 32;
          tk.K = K; tk.r0 = r0; tk.rlo = item.rlo; tk.rhi = item.rhi;
          tk.col0 = (int)cols.size();
          tk.ncols = std::min(bn, R - c0);
          for (int r = c0; r < c0 + tk.ncols; ++r) cols.push_back(col_for(item, r, false));
          tasks.push_back(tk);
          flops += 8.0 * 32 * tk.ncols * K;
        }
    }
    return;
  }
  // group by (class, global face-row range)
  std::map<std::tuple<int, int, int>, std::vector<int>> groups;
  for (size_t i = 0; i < host.items.size(); ++i) {
    const Item& item = host.items[i];
    const SubPlan& sp = P.subs[item.s];
    int glo, ghi;
    if (item.rlo == 0 && item.rhi == sp.k * n) { glo = 0; ghi = 4 * n; }
    else if (item.rlo == 0) { glo = 0; ghi = 2 * n; }      // lower faces W,S
    else { glo = 2 * n; ghi = 4 * n; }                      // upper faces N,E
    groups[std::make_tuple(c->sub_class[item.s], glo, ghi)].push_back((int)i);
  }
  const int K = 4 * n;
  for (auto& g : groups) {
    const int cls = std::get<0>(g.first), glo = std::get<1>(g.first), ghi = std::get<2>(g.first);
    std::vector<MmaCol> gc;
    for (int i : g.second)
      for (int r = 0; r < R; ++r) gc.push_back(col_for(host.items[i], r, true));
    for (size_t c0 = 0; c0 < gc.size(); c0 += bn) {
      const int nc = (int)std::min<size_t>(bn, gc.size() - c0);
      const int base = (int)cols.size();
      cols.insert(cols.end(), gc.begin() + c0, gc.begin() + c0 + nc);
      for (int r0 = (glo / 32) * 32; r0 < ghi; r0 += 32) {
        MmaTask tk;
        tk.a_off = c->Tcls_off[cls] + (long long)(r0 / 32) * K * 32;
        tk.K = K; tk.r0 = r0; tk.rlo = glo; tk.rhi = ghi;
        tk.col0 = base;
        tk.ncols = nc;
        tasks.push_back(tk);
        flops += 8.0 * 32 * nc * K;
      }
    }
  }
}

// bounds validation of every descriptor (a bad table must fail here, not fault)
int validate_mma(Ctx* c, const std::vector<MmaTask>& tasks, const std::vector<MmaCol>& cols, int R, bool shared) {
  const int n = c->n;
  const long long LR = c->plan.L * (long long)R;
  const size_t Aelems = shared ? c->Tcls_elems : c->T_elems;
  for (const MmaTask& tk : tasks) {
    if (tk.K % 32 || tk.a_off < 0 || (size_t)(tk.a_off + (long long)tk.K * 32) > Aelems)
      return fail(c, -4, "internal: contraction task reads outside the maps");
    for (int j = 0; j < tk.ncols; ++j) {
      const MmaCol& col = cols[tk.col0 + j];
      for (int q = 0; q < 4; ++q) {
        if (col.in[q] >= 0 && col.in[q] + (long long)(n - 1) * R >= LR)
          return fail(c, -4, "internal: contraction column reads outside the vector");
        if (col.out[q] >= 0 && col.out[q] + (long long)(n - 1) * R >= LR)
          return fail(c, -4, "internal: contraction column writes outside the vector");
      }
    }
  }
  return 0;
}

// k_zmma2's k-major operand form needs every task's columns to be consecutive
// right-hand sides of one slab read from one source: B row k is then one
// contiguous run at in[0] + k R.
bool slab_rows(const std::vector<MmaTask>& tasks, const std::vector<MmaCol>& cols) {
  for (const MmaTask& tk : tasks) {
    const MmaCol& c0 = cols[tk.col0];
    if (c0.in[0] < 0) return false;
    for (int j = 1; j < tk.ncols; ++j) {
      const MmaCol& cj = cols[tk.col0 + j];
      if (cj.alt != c0.alt) return false;
      for (int q = 0; q < 4; ++q)
        if ((c0.in[q] < 0) != (cj.in[q] < 0) || (c0.in[q] >= 0 && cj.in[q] != c0.in[q] + j)) return false;
    }
  }
  return true;
}

int make_mma(Ctx* c, DevStep& st, int R, bool shared, DevMma** out) {
  const int key = shared ? -R : R;
  auto it = st.mma.find(key);
  if (it != st.mma.end()) {
    *out = &it->second;
    return 0;
  }
  std::vector<MmaTask> tasks;
  std::vector<MmaCol> cols;
  double flops = 0;
  // k_zmma2 (bulk-copy staged): slabs of R RHS (64-column tasks when R > 32) or
  // shared maps with one RHS (64 subdomain columns); k_zmma otherwise.
  // HS_ZMMA2=0 keeps k_zmma everywhere.
  static const bool z2 = !(getenv("HS_ZMMA2") && atoi(getenv("HS_ZMMA2")) == 0);
  int kind = 0, bn = 32;
  if (z2 && !shared) kind = 1, bn = R > 32 ? 64 : 32;
  else if (z2 && shared && R == 1) kind = 2, bn = 64;
  build_mma_host(c, st.host, R, shared, tasks, cols, flops, bn);
  static const int bn_env = getenv("HS_ZMMA2_BN") ? atoi(getenv("HS_ZMMA2_BN")) : 0;  // 32 / 64: fixed
  // shared maps: 32-column tasks (finer tasks balance the persistent residual
  // step; the n-major 64-column tile is copy-bound); slabs: 32 when a step
  // has fewer 64-column tasks than SMs
  if (bn == 64 && (bn_env == 32 || (bn_env != 64 && (kind == 2 || (int)tasks.size() < c->num_sms)))) {
    // a step with fewer 64-column tasks than SMs: 32-column tasks, twice the CTAs
    tasks.clear(); cols.clear(); flops = 0; bn = 32;
    build_mma_host(c, st.host, R, shared, tasks, cols, flops, bn);
  }
  if (validate_mma(c, tasks, cols, R, shared)) return -1;
  if (kind == 1 && !slab_rows(tasks, cols)) return fail(c, -4, "internal: contraction task columns are not one slab");
  if (kind != 0 && !c->zeros) {
    CK(dalloc(c, (void**)&c->zeros, 64 * sizeof(double2)));
    CK(cudaMemsetAsync(c->zeros, 0, 64 * sizeof(double2), c->stream));
  }
  if (kind != 0 && !c->z2_tickets) {  // k_zmma2 persistent launches' ticket counters (never reset)
    CK(dalloc(c, (void**)&c->z2_tickets, kZ2TicketSlots * sizeof(unsigned)));
    CK(cudaMemsetAsync(c->z2_tickets, 0, kZ2TicketSlots * sizeof(unsigned), c->stream));
  }
  DevMma m;
  m.kind = kind;
  m.bn = bn;
  if (upload(c, &m.tasks, tasks) || upload(c, &m.cols, cols)) return -1;
  m.ntasks = (int)tasks.size();
  m.ncols = (int)cols.size();
  m.flops = flops;
  m.minK = tasks.empty() ? 0 : tasks[0].K;
  for (const MmaTask& tk : tasks) m.minK = std::min(m.minK, tk.K);
  auto res = st.mma.emplace(key, m);
  *out = &res.first->second;
  return 0;
}

void free_fused_mma(Ctx* c) {
  DevFusedMma& f = c->fused_mma;
  dfree(c, f.tasks, f.ntasks * sizeof(FusedMmaTask));
  dfree(c, f.cols, f.ncols * sizeof(MmaCol));
  dfree(c, f.deps, f.ndeps * sizeof(FusedDep));
  dfree(c, f.incs, f.nincs * sizeof(int));
  dfree(c, f.counters, (f.ncounters + 1) * sizeof(int));
  dfree(c, f.split_buf, 0);
  dfree(c, f.split_cnt, 0);
  f = DevFusedMma();
}

template <class Tile>
std::vector<Tile> list_schedule(const std::vector<Tile>& tiles, const std::vector<FusedDep>& deps,
                                const std::vector<std::vector<int>>& tile_inc, const std::vector<double>& cost,
                                int nblocks, int workers, double fixed, double rate);

// Dataflow plan of one BSP apply on the DMMA contraction: every task of the
// forward steps, the residual and the backward steps in schedule order, with
// per-(block, 32-RHS chunk) completion counts it waits for / completes.
bool map_once_steps(const Ctx* c);

int build_fused_mma(Ctx* c, int R, bool shared) {
  free_fused_mma(c);
  DevFusedMma& f = c->fused_mma;
  const int n = c->n;
  // fill tasks and split-K pairs are k_zmma2_df's (launch_zmma_fused): not with
  // HS_ZMMA2=0 or the shared maps with R > 1 (k_zmma_fused)
  static const bool z2 = !(getenv("HS_ZMMA2") && atoi(getenv("HS_ZMMA2")) == 0);
  const bool df = z2 && (!shared || R == 1);
  // task / counter width in right-hand sides: 16 for the per-subdomain slabs
  // (k_zmma2_df<.., 16>: the apply is bound by its dependency chain, so twice
  // the tasks at half the contraction each; HS_ZMMA2_DF_BN=32: 32-column tasks)
  static const int bn_env = getenv("HS_ZMMA2_DF_BN") ? atoi(getenv("HS_ZMMA2_DF_BN")) : 16;
  const int cwd = (df && !shared && R > 16 && bn_env == 16) ? 16 : 32;
  const int nch = (R + cwd - 1) / cwd;
  const int ncnt = c->plan.npairs * nch;
  std::vector<FusedMmaTask> ftasks;
  std::vector<MmaCol> cols;
  std::vector<FusedDep> deps;
  std::vector<int> incs;
  std::vector<int> written(ncnt, 0);
  double flops = 0;
  auto counter = [&](long long off, int r) { return (int)((off - r) / ((long long)n * R)) * nch + r / cwd; };
  auto add = [&](const DevStep& st, int phase) {
    std::vector<MmaTask> tasks;
    std::vector<MmaCol> sc;
    build_mma_host(c, st.host, R, shared, tasks, sc, flops, cwd);
    std::vector<int> inc_step;
    const int cbase = (int)cols.size();
    cols.insert(cols.end(), sc.begin(), sc.end());
    for (MmaTask tk : tasks) {
      FusedMmaTask ft;
      ft.phase = phase;
      ft.dep0 = (int)deps.size(); ft.ndep = 0;
      ft.inc0 = (int)incs.size(); ft.ninc = 0;
      std::set<int> rd, wr;
      const int r0 = std::max(tk.rlo, tk.r0), r1 = std::min(tk.rhi, tk.r0 + 32);
      for (int j = 0; j < tk.ncols; ++j) {
        const MmaCol& col = sc[tk.col0 + j];
        for (int q = 0; q < 4; ++q)
          if (col.in[q] >= 0) rd.insert(counter(col.in[q], col.r));
        for (int q = r0 / n; q * n < r1; ++q)
          if (q < 4 && col.out[q] >= 0) wr.insert(counter(col.out[q], col.r));
      }
      std::set<int> all(rd);
      all.insert(wr.begin(), wr.end());
      for (int k2 : all)
        if (written[k2] > 0) { deps.push_back({k2, written[k2]}); ft.ndep++; }
      for (int k2 : wr) { incs.push_back(k2); ft.ninc++; inc_step.push_back(k2); }
      tk.col0 += cbase;
      ft.task = tk;
      ftasks.push_back(ft);
    }
    for (int k2 : inc_step) written[k2]++;
  };
  for (auto& st : c->fwd) add(st, 0);
  // map-once residual (as the per-step path, do_precond): the residual tasks
  // cover only the rows where r' can be nonzero; fill tasks set rp = w = 0,
  // z = zL on the other blocks (after the residual tasks in plan order, so no
  // residual task waits on a fill).  HS_ZMMA2_DF_MO=0: the full residual step.
  static const bool mo_env = !(getenv("HS_ZMMA2_DF_MO") && atoi(getenv("HS_ZMMA2_DF_MO")) == 0);
  const bool mo = mo_env && df && map_once_steps(c);
  if (mo) {
    add(c->mo_resid, 1);
    std::vector<int> fc;
    for (int b : c->mo_zero_host)
      for (int ch = 0; ch < nch; ++ch) fc.push_back(b * nch + ch);
    // ~4k elements per fill task
    const int per = std::max(1, 4096 / (n * std::min(R, cwd)));
    for (size_t i = 0; i < fc.size(); i += per) {
      FusedMmaTask ft;
      ft.task = MmaTask();
      ft.task.a_off = 0; ft.task.K = 0; ft.task.ncols = 0; ft.task.col0 = 0;
      ft.phase = 3;
      ft.dep0 = (int)deps.size(); ft.ndep = 0;
      ft.inc0 = (int)incs.size(); ft.ninc = 0;
      for (size_t j = i; j < std::min(fc.size(), i + per); ++j) {
        const int k2 = fc[j];
        if (written[k2] > 0) { deps.push_back({k2, written[k2]}); ft.ndep++; }
        incs.push_back(k2); ft.ninc++;
      }
      ftasks.push_back(ft);
    }
    for (int k2 : fc) written[k2]++;
  } else {
    add(c->full, 1);
  }
  for (auto& st : c->bwd) add(st, 2);
  // k_zmma2_df split-K (opt-in, HS_ZMMA2_SPLIT=1): the sweep steps' tasks (the
  // dependency chain) in two K halves on two CTAs; the later arrival adds the
  // halves in half order and finishes the task.  cfg4: 0.208 ms either way
  // (the chain's links shrink, the extra tickets and partial exchange eat it);
  // the shared maps (K = 4n, 16 chunks per task): cfg5 0.490 -> 0.384 ms.
  static const bool split = getenv("HS_ZMMA2_SPLIT") && atoi(getenv("HS_ZMMA2_SPLIT")) != 0;
  int npairs = 0;
  if (split && df) {
    std::vector<FusedMmaTask> sp;
    sp.reserve(ftasks.size() * 2);
    for (const FusedMmaTask& ft : ftasks) {
      if (ft.phase == 1 || ft.phase == 3 || ft.task.K / 32 < 4) {
        sp.push_back(ft);
        continue;
      }
      FusedMmaTask h = ft;
      h.pair = npairs++;
      h.ks = 0;
      sp.push_back(h);
      h.ks = 1;
      sp.push_back(h);
    }
    ftasks.swap(sp);
  }
  {
    // ticket order: list-scheduled on one CTA per SM (HS_FUSED_ORDER=0: plan
    // order); a task costs ~1 us per 32-column k chunk + ~3 us of latency
    static const bool reorder = !(getenv("HS_FUSED_ORDER") && atoi(getenv("HS_FUSED_ORDER")) == 0);
    if (reorder) {
      std::vector<std::vector<int>> tinc(ftasks.size());
      std::vector<double> cost(ftasks.size());
      for (size_t t = 0; t < ftasks.size(); ++t) {
        // a pair's completions are its second arrival's: counted once, on half 1
        if (ftasks[t].ks != 0)
          tinc[t].assign(incs.begin() + ftasks[t].inc0, incs.begin() + ftasks[t].inc0 + ftasks[t].ninc);
        // us: a 32-position chunk of a 16-column task contracts in ~0.55 us, of a
        // 32-column task in ~0.9 us (tensor-copy staged slabs; zmma_df_trace)
        static const double us16 = getenv("HS_DF_COST16") ? atof(getenv("HS_DF_COST16")) : 0.55;
        const double per_chunk = shared ? 1.0 : (cwd == 16 ? us16 : 0.9);
        cost[t] = ftasks[t].phase == 3 ? 0.5 : per_chunk * (ftasks[t].task.K / 32) / (ftasks[t].ks >= 0 ? 2 : 1);
      }
      static const double fixed_us = getenv("HS_DF_FIXED") ? atof(getenv("HS_DF_FIXED")) : 3.0;
      ftasks = list_schedule(ftasks, deps, tinc, cost, ncnt, c->num_sms, fixed_us * 1e-6, 1e6);
    }
  }
  {
    std::vector<MmaTask> plain;
    for (auto& ft : ftasks) plain.push_back(ft.task);
    if (validate_mma(c, plain, cols, R, shared)) return -1;
  }
  if (upload(c, &f.tasks, ftasks) || upload(c, &f.cols, cols) || upload(c, &f.deps, deps) ||
      upload(c, &f.incs, incs))
    return -1;
  CK(dalloc(c, (void**)&f.counters, (ncnt + 1) * sizeof(int)));
  if (shared && !c->zeros) {  // the n-major form's zero rows (absent faces, padding columns)
    CK(dalloc(c, (void**)&c->zeros, 64 * sizeof(double2)));
    CK(cudaMemsetAsync(c->zeros, 0, 64 * sizeof(double2), c->stream));
  }
  f.npairs_split = npairs;
  if (npairs > 0) {
    CK(dalloc(c, (void**)&f.split_buf, (size_t)npairs * 2 * 32 * 32 * sizeof(double2)));
    CK(dalloc(c, (void**)&f.split_cnt, (size_t)npairs * sizeof(int)));
    CK(cudaMemsetAsync(f.split_cnt, 0, (size_t)npairs * sizeof(int), c->stream));
  }
  f.ntasks = (int)ftasks.size();
  f.ncols = (int)cols.size();
  f.ndeps = (int)deps.size();
  f.nincs = (int)incs.size();
  f.ncounters = ncnt;
  f.flops = flops;
  f.minK = 1 << 30;
  for (const auto& ft : ftasks)
    if (ft.phase != 3) f.minK = std::min(f.minK, ft.task.K);
  f.R = R;
  f.cw = cwd;
  f.shared = shared;
  f.built = true;
  return 0;
}

int make_step(Ctx* c, const StepTable& t, DevStep& out) {
  std::vector<DevItem> items;
  std::vector<DevTile> tiles;
  std::vector<DevRecv> recv;
  double mapb = 0, vecb = 0;
  int maxK = 0;
  for (size_t i = 0; i < t.items.size(); ++i) {
    const Item& it = t.items[i];
    DevItem d;
    d.s = it.s; d.rlo = it.rlo; d.rhi = it.rhi; d.alt = it.alt;
    for (int q = 0; q < 4; ++q) d.slot[q] = it.slot[q];
    d.c0 = 0; d.c1 = c->plan.subs[it.s].k * c->n;
    items.push_back(d);
    const int K = c->plan.subs[it.s].k * c->n;
    maxK = std::max(maxK, K);
    for (int tl = it.rlo / kRowTile; tl * kRowTile < it.rhi; ++tl) tiles.push_back({(int)i, tl});
    const double rows = it.rhi - it.rlo;
    // 16 (rows cols + cols + 2 rows) bytes per solve-application
    mapb += 16.0 * rows * K;
    vecb += 16.0 * (K + 2.0 * rows);
  }
  for (const RecvSlot& r : t.recv) recv.push_back({r.dir, r.slot, (long long)r.off});
  free_step(c, out);
  if (upload(c, &out.items, items)) return -1;
  if (upload(c, &out.tiles, tiles)) return -1;
  if (upload(c, &out.recv, recv)) return -1;
  out.nitems = (int)items.size();
  out.ntiles = (int)tiles.size();
  out.nrecv = (int)recv.size();
  out.nsend_up = t.nsend_up; out.nsend_dn = t.nsend_dn;
  out.nrecv_up = t.nrecv_up; out.nrecv_dn = t.nrecv_dn;
  out.maxK = maxK;
  out.bytes_per_rhs_map = mapb;
  out.bytes_per_rhs_vec = vecb;
  out.host = t;
  return 0;
}

void free_fused(Ctx* c) {
  for (DevFused* fp : {&c->fused, &c->fused_ims}) {
    DevFused& f = *fp;
    dfree(c, f.split_buf, 0);
    dfree(c, f.split_cnt, 0);
    dfree(c, f.items, f.nitems * sizeof(DevItem));
    dfree(c, f.tiles, f.ntiles * sizeof(FusedTile));
    dfree(c, f.deps, f.ndeps * sizeof(FusedDep));
    dfree(c, f.counters, (c->plan.npairs + 1) * sizeof(int));
    f = DevFused();
  }
}

// Ticket order of a fused plan.  CTAs claim tiles in ticket order and wait
// for their dependencies, so a ticket claimed long before its inputs exist
// idles a CTA that could stream another tile's map.  List-schedule the tiles
// on `workers` simulated CTAs (duration = fixed cost + streamed bytes at the
// per-CTA share of HBM bandwidth): whenever a CTA frees up, it takes, among
// the tiles whose inputs are complete by then, the one with the longest path
// to the end of the apply (else the one that becomes ready first).  The
// result is a topological order of the dependency graph (a tile's
// predecessors are the first `count` writers of each block it waits on), so
// any such order keeps the plan deadlock-free and the arithmetic unchanged.
// Ticket order of a dataflow plan: list-schedule the dependency graph on
// `workers` resident CTAs, greedy by the longest path to the end (bottom
// level), and return the tasks in the order they would start.  Any
// topological order is deadlock-free; every writer of a block depends on the
// block's earlier writers, so the per-block completion counts keep their
// meaning.  dur[t] = fixed + cost[t] / rate.
template <class Tile>
std::vector<Tile> list_schedule(const std::vector<Tile>& tiles, const std::vector<FusedDep>& deps,
                                const std::vector<std::vector<int>>& tile_inc, const std::vector<double>& cost,
                                int nblocks, int workers, double fixed, double rate);

std::vector<FusedTile> schedule_tickets(const std::vector<FusedTile>& tiles, const std::vector<FusedDep>& deps,
                                        const std::vector<std::vector<int>>& tile_inc,
                                        const std::vector<double>& cost, int nblocks, int workers) {
  return list_schedule(tiles, deps, tile_inc, cost, nblocks, workers, 3e-6, 6.5e12 / std::max(1, workers));
}

// Predecessor lists of a plan in plan order (a dependency (block, count) =
// the block's first `count` writers).
static std::vector<std::vector<int>> plan_preds(const std::vector<FusedTile>& tiles, const std::vector<FusedDep>& deps,
                                                const std::vector<std::vector<int>>& tile_inc, int nblocks) {
  const int T = (int)tiles.size();
  std::vector<std::vector<int>> writers(nblocks), pre(T);
  for (int t = 0; t < T; ++t)
    for (int b : tile_inc[t]) writers[b].push_back(t);
  for (int t = 0; t < T; ++t) {
    for (int d = 0; d < tiles[t].ndep; ++d) {
      const FusedDep& dp = deps[tiles[t].dep0 + d];
      for (int i = 0; i < dp.count && i < (int)writers[dp.block].size(); ++i) pre[t].push_back(writers[dp.block][i]);
    }
    std::sort(pre[t].begin(), pre[t].end());
    pre[t].erase(std::unique(pre[t].begin(), pre[t].end()), pre[t].end());
  }
  return pre;
}

// Longest modelled path from a tile to the end (including it) / from the start
// to it (excluding it); dur = fixed + cost / rate.
std::vector<double> bottom_levels(const std::vector<FusedTile>& tiles, const std::vector<FusedDep>& deps,
                                  const std::vector<std::vector<int>>& tile_inc, const std::vector<double>& cost,
                                  int nblocks, double fixed, double rate) {
  const auto pre = plan_preds(tiles, deps, tile_inc, nblocks);
  const int T = (int)tiles.size();
  std::vector<double> bl(T, 0.0);
  std::vector<std::vector<int>> succ(T);
  for (int t = 0; t < T; ++t)
    for (int p : pre[t]) succ[p].push_back(t);
  for (int t = T - 1; t >= 0; --t) {
    double m = 0;
    for (int q : succ[t]) m = std::max(m, bl[q]);
    bl[t] = fixed + cost[t] / rate + m;
  }
  return bl;
}

std::vector<double> top_levels(const std::vector<FusedTile>& tiles, const std::vector<FusedDep>& deps,
                               const std::vector<std::vector<int>>& tile_inc, const std::vector<double>& cost,
                               int nblocks, double fixed, double rate) {
  const auto pre = plan_preds(tiles, deps, tile_inc, nblocks);
  const int T = (int)tiles.size();
  std::vector<double> tl(T, 0.0);
  for (int t = 0; t < T; ++t)
    for (int p : pre[t]) tl[t] = std::max(tl[t], tl[p] + fixed + cost[p] / rate);
  return tl;
}

template <class Tile>
std::vector<Tile> list_schedule(const std::vector<Tile>& tiles, const std::vector<FusedDep>& deps,
                                const std::vector<std::vector<int>>& tile_inc, const std::vector<double>& cost,
                                int nblocks, int workers, double fixed, double rate) {
  const int T = (int)tiles.size();
  std::vector<std::vector<int>> writers(nblocks);
  for (int t = 0; t < T; ++t)
    for (int b : tile_inc[t]) writers[b].push_back(t);
  std::vector<std::vector<int>> succ(T);
  std::vector<int> npred(T, 0);
  for (int t = 0; t < T; ++t) {
    std::vector<int> pre;
    for (int d = 0; d < tiles[t].ndep; ++d) {
      const FusedDep& dp = deps[tiles[t].dep0 + d];
      for (int i = 0; i < dp.count; ++i) pre.push_back(writers[dp.block][i]);
    }
    std::sort(pre.begin(), pre.end());
    pre.erase(std::unique(pre.begin(), pre.end()), pre.end());
    npred[t] = (int)pre.size();
    for (int p : pre) succ[p].push_back(t);
  }
  std::vector<double> dur(T), bl(T, 0.0), ready(T, 0.0);
  for (int t = 0; t < T; ++t) dur[t] = fixed + cost[t] / rate;
  for (int t = T - 1; t >= 0; --t) {  // successors come later in plan order
    double m = 0;
    for (int s : succ[t]) m = std::max(m, bl[s]);
    bl[t] = dur[t] + m;
  }
  using Q = std::pair<double, int>;
  std::priority_queue<Q, std::vector<Q>, std::greater<Q>> waiting, freew;  // by ready time / free time
  std::priority_queue<Q> avail;                                             // by bottom level
  for (int w = 0; w < workers; ++w) freew.push({0.0, w});
  for (int t = 0; t < T; ++t)
    if (npred[t] == 0) waiting.push({0.0, t});
  // split-K pairs (ks = 0 / 1, adjacent in plan order, the same
  // dependencies): emitted together -- consecutive tickets, so both halves
  // stream at once -- and every successor (it depends on half 1, the pair's
  // writer) gets a later ticket than BOTH halves: the completion is signalled
  // by whichever half arrives second, and a successor ticketed before a half
  // could spin on a counter no running CTA will bump.
  std::vector<char> emitted(T, 0);
  std::vector<Tile> out;
  out.reserve(T);
  auto partner = [&](int t) -> int {
    if (tiles[t].ks == 0 && t + 1 < T && tiles[t + 1].ks == 1 && tiles[t + 1].pair == tiles[t].pair) return t + 1;
    if (tiles[t].ks == 1 && t > 0 && tiles[t - 1].ks == 0 && tiles[t - 1].pair == tiles[t].pair) return t - 1;
    return -1;
  };
  auto finish = [&](int t, double fin) {
    freew.push({fin, 0});
    for (int s : succ[t]) {
      ready[s] = std::max(ready[s], fin);
      if (--npred[s] == 0) waiting.push({ready[s], s});
    }
  };
  while ((int)out.size() < T) {
    const double tau = freew.top().first;
    freew.pop();
    while (!waiting.empty() && waiting.top().first <= tau) {
      avail.push({bl[waiting.top().second], waiting.top().second});
      waiting.pop();
    }
    int t = -1;
    while (t < 0 && !avail.empty()) {
      if (!emitted[avail.top().second]) t = avail.top().second;
      avail.pop();
    }
    while (t < 0 && !waiting.empty()) {
      if (!emitted[waiting.top().second]) t = waiting.top().second;
      waiting.pop();
    }
    if (t < 0) {  // everything left is a partner already emitted
      freew.push({tau, 0});
      continue;
    }
    const int q = partner(t);
    const int first = q >= 0 ? std::min(t, q) : t;
    const double fin = std::max(tau, ready[t]) + dur[t];
    emitted[t] = 1;
    if (q < 0) {
      out.push_back(tiles[t]);
      finish(t, fin);
      continue;
    }
    // the pair: half 0 first, the partner on the next free CTA
    const double tau2 = freew.top().first;
    freew.pop();
    const double fin2 = std::max(tau2, ready[q]) + dur[q];
    emitted[q] = 1;
    out.push_back(tiles[first]);
    out.push_back(tiles[first == t ? q : t]);
    finish(t, fin);
    finish(q, fin2);
  }
  return out;
}

// Dataflow plan of one BSP apply: every tile of the forward steps, the
// residual step and the backward steps in schedule order, each with the
// per-block completion counts it waits for (all earlier tile-writes to the
// blocks it reads or read-modify-writes; counts taken before its own step,
// since the tiles of one step are independent).  ims: append the (I - S) z
// step (GMRES's A M v in one launch): its tiles wait for the final z of the
// blocks they read and of their output rows, and signal nothing.
//
// Two plans (FusedTile phases, hs_ctx.h):
//  * per-step (c->fused_mode & 4): forward, full residual, backward, full
//    (I - S) z -- the k_step1 arithmetic in the same order, bitwise equal.
//  * map-once (default): the same z (and (I - S) z) with each map row read
//    about once.  Within a forward window the substitution is exact, so
//    r' = r - (I - S) zL vanishes on every W/S block whose writer read the
//    final zL of its slab (every forward writer but the window starts at
//    seams, whose residual rows are recomputed: phase 1 "a").  On N/E blocks
//    r' = T_low zL, which shares the map rows of the backward step: both
//    products come from one read (phase 4), except for writers whose output
//    feeds a backward window start (phase 1 "b" early + phase 2 late).  With
//    (I - S) z = (r - r') + (I - S) w and w the backward state, (I - S) z is
//    r on N/E blocks whose writer read its final w, and r - T_up w on W/S
//    blocks: phase 4 / 2 tiles read the whole map (upper rows on the final w)
//    when their slab is final; the backward window starts (slab read from
//    rp, final w later) and subdomains without lower faces get phase 5.
// keep_rank >= 0: keep only the tiles of that rank's subdomains (sub_rank),
// in the global ticket order (row-band ranks on separate GPUs).
// Partial-sum slots and arrival counters of the split-K pairs (zeroed once:
// arrivals are counted modulo 2, so they are never reset).
int alloc_split(Ctx* c, DevFused& f) {
  if (f.npairs_split == 0) return 0;
  CK(dalloc(c, (void**)&f.split_buf, (size_t)f.npairs_split * 2 * 32 * 2 * sizeof(double2)));
  CK(dalloc(c, (void**)&f.split_cnt, (size_t)f.npairs_split * sizeof(int)));
  CK(cudaMemsetAsync(f.split_cnt, 0, (size_t)f.npairs_split * sizeof(int), c->stream));
  return 0;
}

struct FusedHost {
  std::vector<DevItem> items;
  std::vector<FusedTile> tiles;
  std::vector<FusedDep> deps;
};

int fused_plan_host(const Ctx* c, const Plan& P, const std::vector<StepTable>& fwd, const StepTable& full,
                    const std::vector<StepTable>& bwd, bool ims, DevFused& f, FusedHost& H,
                    const std::vector<int>* sub_rank = nullptr, int keep_rank = -1) {
  const int n = c->n;
  std::vector<DevItem>& items = H.items;
  std::vector<FusedTile>& tiles = H.tiles;
  std::vector<FusedDep>& deps = H.deps;
  std::vector<int> written(P.npairs, 0), zl_written(P.npairs, 0);
  f.map_once = !(c->fused_mode & 4);
  // tile shape: one 32-row strip, kSumWarps warps splitting its columns
  // (2 strips per tile -- 80 registers, half the occupancy -- was slower at
  // cfg3; HS_FUSED_RT=2 selects it, per-step plan only).
  f.rt = 1;
  f.nw = kSumWarps;
  f.nv = 1;
  if (const char* e = getenv("HS_FUSED_RT")) f.rt = std::max(1, std::min(2, atoi(e)));
  if (f.map_once) f.rt = 1;
  // TMA-staged maps (k_bsp_tma) up to 512 map columns, register streaming beyond
  // (measured on B200, ms per apply, TMA vs streaming: cfg1 0.044/0.046, cfg2
  // 0.091/0.094, cfg3 0.334/0.355, cfg5 2.37/2.25).  HS_FUSED_TMA=0/1 overrides.
  f.tma = f.rt == 1;  // decided on maxK below
  f.bytes = 0;
  const int TR = kRowTile * f.rt;
  struct VItem {
    Item it;
    int phase, flags;
    int c0 = 0, c1 = -1;  // column range (-1: all K columns)
  };
  // one virtual step: tiles of independent items (counts taken before the step)
  std::vector<std::vector<int>> tile_inc;  // blocks each tile completes
  std::vector<double> tile_cost;           // bytes each tile streams
  auto add = [&](const std::vector<VItem>& step) {
    std::vector<int> inc;
    size_t inc0 = 0;
    for (const VItem& v : step) {
      const Item& it = v.it;
      const int phase = v.phase;
      const SubPlan& sp = P.subs[it.s];
      const int K = sp.k * n;
      DevItem d;
      d.s = it.s; d.rlo = it.rlo; d.rhi = it.rhi; d.alt = it.alt;
      for (int q = 0; q < 4; ++q) d.slot[q] = -1;
      d.c0 = v.c0; d.c1 = v.c1 < 0 ? K : v.c1;
      const int idx = (int)items.size();
      items.push_back(d);
      const int KC = d.c1 - d.c0;  // columns streamed
      f.maxK = std::max(f.maxK, K);
      const int nv = phase == 4 ? 2 : 1;
      f.nv = std::max(f.nv, nv);
      f.bytes += 16.0 * ((double)(it.rhi - it.rlo) * KC + nv * KC + 2.0 * (it.rhi - it.rlo));
      for (int tl = it.rlo / TR; tl * TR < it.rhi; ++tl) {
        FusedTile ft;
        ft.item = idx; ft.tile = tl; ft.phase = phase; ft.flags = v.flags;
        ft.c0 = d.c0; ft.c1 = d.c1; ft.ks = -1; ft.pair = -1;
        ft.dep0 = (int)deps.size(); ft.ndep = 0;
        ft.rmask = 0;
        if (phase <= 1 || phase == 4) {  // zL is never initialised: blocks without a forward write read r
          if (phase != 0 || !it.alt)
            for (int q = 0; q < sp.k; ++q)
              if (zl_written[sp.first_block + q] == 0) ft.rmask |= 1 << q;
          for (int q = 0; q < sp.k; ++q)
            if (zl_written[sp.tgt_block[q]] == 0) ft.rmask |= 1 << (4 + q);
        }
        std::set<int> blocks;
        for (int q = 0; q < sp.k; ++q) blocks.insert(sp.first_block + q);
        const int r0 = std::max(it.rlo, tl * TR), r1 = std::min(it.rhi, (tl + 1) * TR);
        for (int q = r0 / n; q * n < r1; ++q) {
          blocks.insert(sp.tgt_block[q]);
          // phases 2 and 4 complete their lower-face blocks only (upper rows write wout)
          const bool signals = phase <= 1 || ((phase == 2 || phase == 4) && q < sp.nlower);
          if (signals) inc.push_back(sp.tgt_block[q]);
        }
        for (int b : blocks)
          if (written[b] > 0) {
            deps.push_back({b, written[b]});
            ft.ndep++;
          }
        tiles.push_back(ft);
        tile_inc.push_back(std::vector<int>(inc.begin() + inc0, inc.end()));
        tile_cost.push_back(16.0 * ((double)(r1 - r0) * KC + nv * KC));
        inc0 = inc.size();
      }
    }
    for (int b : inc) written[b]++;
    return inc;
  };
  auto vstep = [](const StepTable& st, int phase, int flags) {
    std::vector<VItem> v;
    for (const Item& it : st.items) v.push_back({it, phase, flags});
    return v;
  };
  auto mark_zl = [&](const std::vector<int>& inc) {
    for (int b : inc) zl_written[b]++;
  };
  if (!f.map_once) {
    for (auto& st : fwd) mark_zl(add(vstep(st, 0, 0)));
    add(vstep(full, 1, 0));
    for (auto& st : bwd) add(vstep(st, 2, 0));
    if (ims) add(vstep(full, 3, 0));
  } else {
    // backward window starts below the top group (their slab is read from rp)
    std::set<int> bstart;
    for (auto& w : P.win_upper)
      if (w.second < P.ng + 1) bstart.insert(w.second);
    std::vector<VItem> resid;
    for (auto& st : fwd) {
      std::vector<VItem> step;
      for (const Item& it : st.items) {
        const bool seam = it.alt && P.subs[it.s].nlower > 0;  // slab zL != r: residual rows recomputed
        step.push_back({it, 0, seam ? 0 : FT_ZERO});
        if (seam) {  // r' = T_up (zL - r): zL differs from r on the W/S slab faces only
          Item r = it;
          r.alt = 0;
          resid.push_back({r, 1, FT_DIFF, 0, P.subs[it.s].nlower * n});
        }
      }
      mark_zl(add(step));
    }
    std::vector<bool> has_bwd(P.nsub, false), late(P.nsub, false);
    std::vector<std::vector<VItem>> bsteps;
    for (auto& st : bwd) {
      std::vector<VItem> step;
      for (const Item& it : st.items) {
        const SubPlan& sp = P.subs[it.s];
        has_bwd[it.s] = true;
        const bool final_slab = !it.alt || sp.k == sp.nlower;  // reads its final w
        if (!final_slab) late[it.s] = true;
        Item b = it;
        int flags = 0;
        if (ims && final_slab) {
          flags = FT_WOUT;
          b.rhi = sp.k * n;  // upper rows too: wout = r - T_up w
        }
        if (bstart.count(sp.group - 1)) {  // feeds a backward window start: residual early
          Item r = it;
          r.alt = 0;
          resid.push_back({r, 1, 0});
          step.push_back({b, 2, flags});
        } else {
          step.push_back({b, 4, flags});
        }
      }
      bsteps.push_back(step);
    }
    add(resid);
    for (auto& st : bsteps) add(st);
    if (ims) {
      std::vector<VItem> lt;
      for (int s = 0; s < P.nsub; ++s) {
        const SubPlan& sp = P.subs[s];
        if (late[s] || (!has_bwd[s] && sp.k > sp.nlower)) {
          Item it;
          it.s = s; it.alt = 0;
          it.rlo = sp.nlower * n; it.rhi = sp.k * n;  // upper rows: wout = r - T_up w
          if (it.rhi > it.rlo) lt.push_back({it, 5, 0});
          if (late[s]) {  // lower rows: wout = r - T_low (w - rp), nonzero on the N/E slab faces only
            it.rlo = 0; it.rhi = sp.nlower * n;
            lt.push_back({it, 5, FT_DIFF, sp.nlower * n, sp.k * n});
          }
        }
      }
      add(lt);
    }
  }
  // per-step plan: TMA up to 512 map columns; map-once plan: TMA at every
  // width (cfg5, 1024 columns, ms per apply TMA / register streaming: 1.43 / 1.50)
  f.tma = f.tma && (f.map_once || f.maxK <= 512);
  if (const char* e = getenv("HS_FUSED_TMA")) f.tma = atoi(e) != 0 && f.rt == 1;
  // TMA ring: 5 stages / 2 CTAs per SM, or 12 stages / 1 CTA per SM for small
  // plans (< 2 tiles per 5-stage CTA), where a tile's map is prefetched while it
  // waits (ms per apply, 5 / 12 stages: cfg2 0.100 / 0.087, cfg3 0.205 / 0.249,
  // cfg5 1.32 / 1.63)
  f.stages = (int)tiles.size() < 4 * c->num_sms ? 12 : 5;
  if (const char* e = getenv("HS_TMA_STAGES")) f.stages = atoi(e) == 12 ? 12 : 5;
  // the signaller warp takes the fence + atomics off the consumers' path; on
  // smaller (critical-path-bound) plans its extra hop sits on the chain (ms per
  // apply, signaller / direct: cfg5 1.311 / 1.335, cfg3 0.208 / 0.205)
  f.direct_signal = (int)tiles.size() < 32 * c->num_sms ? 1 : 0;
  if (const char* e = getenv("HS_DIRECT_SIGNAL")) f.direct_signal = atoi(e) != 0;
  if (f.stages == 12 && (12 * 1024 + f.nv * std::max(f.maxK, 256)) * 16 > 225 * 1024) f.stages = 5;  // must fit one CTA
  // split-K (opt-in, HS_SPLITK=1): each strip of >= 8 chunks is streamed by
  // two CTAs, the later one adding the two halves in a fixed order.  Meant for
  // plans near their critical path (row bands on many GPUs: the conservative
  // model, tools/scaling_model.py --split, gives cfg5 on 8 GPUs 0.26 -> 0.21
  // ms), but the doubled per-tile cost measured on one GPU (cfg5 1.30 -> 1.50
  // ms, cfg3 0.207 -> 0.274 ms) is far above the model's, so it stays off until
  // it can be measured on real row bands.
  // HS_SPLITK=2: only the tiles on (or within 15 % of) the modelled critical
  // path are split -- the chain links of a critical-path-bound plan (cfg3's 8 +
  // 8 window steps) stream at two CTAs' rate while the throughput-bound rest
  // keeps one tile per strip.
  {
    int split_mode = 0;
    if (const char* e = getenv("HS_SPLITK")) split_mode = f.tma ? atoi(e) : 0;
    f.npairs_split = 0;
    std::vector<char> crit(tiles.size(), 1);
    if (split_mode == 2) {
      const int workers = (f.stages == 12 ? 1 : 2) * c->num_sms;
      const std::vector<double> bl =
          bottom_levels(tiles, deps, tile_inc, tile_cost, P.npairs, 3e-6, 6.5e12 / std::max(1, workers));
      const double mx = bl.empty() ? 0.0 : *std::max_element(bl.begin(), bl.end());
      // a tile is critical when its bottom level plus the longest path into it
      // is within 15 % of the plan's critical path (top levels: forward pass)
      const std::vector<double> tl =
          top_levels(tiles, deps, tile_inc, tile_cost, P.npairs, 3e-6, 6.5e12 / std::max(1, workers));
      for (size_t i = 0; i < tiles.size(); ++i) crit[i] = tl[i] + bl[i] >= 0.85 * mx;
    }
    if (split_mode != 0) {
      std::vector<FusedTile> t2;
      std::vector<std::vector<int>> inc2;
      std::vector<double> cost2;
      for (size_t i = 0; i < tiles.size(); ++i) {
        const FusedTile& t = tiles[i];
        const int nch = (t.c1 + 31) / 32 - t.c0 / 32;
        if (nch < 8 || !crit[i]) {
          t2.push_back(t); inc2.push_back(tile_inc[i]); cost2.push_back(tile_cost[i]);
          continue;
        }
        const int mid = (t.c0 / 32 + nch / 2) * 32;
        FusedTile a = t, b = t;
        a.c1 = mid; b.c0 = mid;
        a.ks = 0; b.ks = 1;
        a.pair = b.pair = f.npairs_split++;
        t2.push_back(a); inc2.push_back({}); cost2.push_back(tile_cost[i] * (mid - t.c0) / (t.c1 - t.c0));
        t2.push_back(b); inc2.push_back(tile_inc[i]); cost2.push_back(tile_cost[i] * (t.c1 - mid) / (t.c1 - t.c0));
      }
      tiles.swap(t2);
      tile_inc.swap(inc2);
      tile_cost.swap(cost2);
    }
  }
  bool reorder = true;
  if (const char* e = getenv("HS_FUSED_ORDER")) reorder = atoi(e) != 0;
  if (reorder) {
    const int workers = (f.tma ? (f.stages == 12 ? 1 : 2) : (f.rt == 1 ? 6 : 1)) * c->num_sms;
    tiles = schedule_tickets(tiles, deps, tile_inc, tile_cost, P.npairs, workers);
  }
  // wout writes per block per apply (tile faces of phases 3 / 5 and FT_WOUT 2 / 4)
  f.wwtot.assign(P.npairs, 0);
  for (const FusedTile& t : tiles) {
    if (t.ks == 0) continue;  // a split-K pair writes once (its second arrival)
    const bool wo = t.phase == 3 || t.phase == 5 || ((t.phase == 2 || t.phase == 4) && (t.flags & FT_WOUT));
    if (!wo) continue;
    const DevItem& it = items[t.item];
    const SubPlan& sp = P.subs[it.s];
    const int r0 = std::max(it.rlo, t.tile * kRowTile * f.rt), r1 = std::min(it.rhi, (t.tile + 1) * kRowTile * f.rt);
    for (int q = r0 / n; q * n < r1; ++q) f.wwtot[sp.tgt_block[q]]++;
  }
  if (keep_rank >= 0) {
    std::vector<FusedTile> mine;
    double own_bytes = 0, all_bytes = 0;
    for (const FusedTile& t : tiles) {  // streamed bytes of a tile (map rows x its columns + slabs)
      const DevItem& it = items[t.item];
      const int r0 = std::max(it.rlo, t.tile * kRowTile * f.rt), r1 = std::min(it.rhi, (t.tile + 1) * kRowTile * f.rt);
      const double b = 16.0 * ((double)(r1 - r0) * (t.c1 - t.c0) + (t.phase == 4 ? 2 : 1) * (t.c1 - t.c0));
      all_bytes += b;
      if ((*sub_rank)[it.s] == keep_rank) {
        mine.push_back(t);
        own_bytes += b;
      }
    }
    if (all_bytes > 0) f.bytes *= own_bytes / all_bytes;  // this rank's share of the apply's bytes
    tiles.swap(mine);
  }
  f.nitems = (int)items.size();
  f.ntiles = (int)tiles.size();
  f.ndeps = (int)deps.size();
  f.wtot = written;  // signals per block per apply (every rank's tiles)

  return 0;
}

int build_fused_plan(Ctx* c, const Plan& P, const std::vector<StepTable>& fwd, const StepTable& full,
                     const std::vector<StepTable>& bwd, bool ims, DevFused& f,
                     const std::vector<int>* sub_rank = nullptr, int keep_rank = -1) {
  FusedHost H;
  if (int e = fused_plan_host(c, P, fwd, full, bwd, ims, f, H, sub_rank, keep_rank)) return e;
  if (upload(c, &f.items, H.items) || upload(c, &f.tiles, H.tiles) || upload(c, &f.deps, H.deps)) return -1;
  CK(dalloc(c, (void**)&f.counters, (P.npairs + 1) * sizeof(int)));
  if (int e = alloc_split(c, f)) return e;
  f.built = true;
  return 0;
}

int build_fused(Ctx* c, bool ims) {
  std::vector<StepTable> fwd, bwd;
  for (auto& st : c->fwd) fwd.push_back(st.host);
  for (auto& st : c->bwd) bwd.push_back(st.host);
  return build_fused_plan(c, c->plan, fwd, c->full.host, bwd, ims, ims ? c->fused_ims : c->fused);
}

// Global (not yet localized) tables of the map-once per-step form and this
// rank's blocks filled without a map read:
//   rs   -- residual rows: every lower face, plus the upper faces of the forward
//           window starts past group 2 (their slab z_L != r at the forward read)
//   up   -- (I - S) z: every subdomain's upper rows on the final w
//   late -- (I - S) z: lower rows of the backward window starts below the top
//   zero -- W/S blocks of exact forward writers (r' = 0: rp = w = 0, z = z_L)
//   rfill-- N/E blocks of final backward writers ((I - S) z = r)
void map_once_tables(const Plan& P, int n, StepTable& rs, StepTable& up, StepTable& late, std::vector<int>& zero,
                     std::vector<int>& rfill) {
  std::set<int> fseam, bstart;  // forward window starts past group 2; backward starts below the top
  for (auto& w : P.win_lower)
    if (w.first > 2) fseam.insert(w.first);
  for (auto& w : P.win_upper)
    if (w.second < P.ng + 1) bstart.insert(w.second);
  for (int s2 = 0; s2 < P.nsub; ++s2) {
    const SubPlan& sp = P.subs[s2];
    const int nl = sp.nlower, K = sp.k * n;
    const bool seam = fseam.count(sp.group) && nl > 0 && sp.k > nl;
    const bool late_b = bstart.count(sp.group) && nl > 0 && sp.k > nl;
    Item it;
    it.s = s2;
    if (nl > 0) { it.rlo = 0; it.rhi = nl * n; rs.items.push_back(it); }
    if (seam) { it.rlo = nl * n; it.rhi = K; rs.items.push_back(it); }
    if (sp.k > nl) { it.rlo = nl * n; it.rhi = K; up.items.push_back(it); }
    if (late_b) { it.rlo = 0; it.rhi = nl * n; late.items.push_back(it); }
    for (int q = 0; q < sp.k; ++q) {
      const int tb = sp.tgt_block[q];
      if (P.subs[P.block_sub[tb]].rank != P.rank) continue;  // own blocks only
      if (q >= nl && !seam) zero.push_back(tb);
      if (q < nl && !late_b) rfill.push_back(tb);
    }
  }
}

void free_emu(Ctx* c);
void free_peer_plans(Ctx* c);
void free_peer(Ctx* c);

int build_steps(Ctx* c) {
  if (!c->steps_dirty) return 0;
  free_fused(c);
  free_emu(c);
  free_peer_plans(c);
  free_fused_mma(c);
  for (auto& s : c->fwd) free_step(c, s);
  for (auto& s : c->bwd) free_step(c, s);
  for (auto& s : c->sp_fwd) free_step(c, s);
  for (auto& s : c->sp_bwd) free_step(c, s);
  free_step(c, c->full);
  free_step(c, c->mo_resid);
  free_step(c, c->mo_ims_up);
  free_step(c, c->mo_ims_late);
  dfree(c, c->mo_zero_blocks, 0); c->mo_zero_blocks = nullptr; c->n_mo_zero = 0; c->mo_zero_host.clear();
  dfree(c, c->mo_r_blocks, 0); c->mo_r_blocks = nullptr; c->n_mo_r = 0;
  Plan& P = c->plan;
  auto f = P.half_steps(0), b = P.half_steps(1);
  for (auto* v : {&f, &b})
    for (const auto& st : *v) {
      const std::string bad = P.check_step(st, true);
      if (!bad.empty()) return fail(c, 1, "windows give an unsafe sweep: " + bad);
    }
  c->fwd.assign(f.size(), DevStep());
  c->bwd.assign(b.size(), DevStep());
  for (size_t i = 0; i < f.size(); ++i) if (make_step(c, f[i], c->fwd[i])) return -1;
  for (size_t i = 0; i < b.size(); ++i) if (make_step(c, b[i], c->bwd[i])) return -1;
  // SP = one window per direction
  auto wl = P.win_lower, wu = P.win_upper;
  P.win_lower.clear(); P.win_upper.clear();
  if (P.ng >= 2) {
    P.win_lower.push_back({2, P.ng + 1});
    P.win_upper.push_back({2, P.ng + 1});
  }
  auto sf = P.half_steps(0), sb = P.half_steps(1);
  P.win_lower = wl; P.win_upper = wu;
  c->sp_fwd.assign(sf.size(), DevStep());
  c->sp_bwd.assign(sb.size(), DevStep());
  for (size_t i = 0; i < sf.size(); ++i) if (make_step(c, sf[i], c->sp_fwd[i])) return -1;
  for (size_t i = 0; i < sb.size(); ++i) if (make_step(c, sb[i], c->sp_bwd[i])) return -1;
  if (make_step(c, P.full_step(), c->full)) return -1;
  // map-once per-step tables (see do_precond / do_ims_mo)
  {
    StepTable rs, up, late;
    std::vector<int> zero, rfill;
    map_once_tables(P, c->n, rs, up, late, zero, rfill);
    if (make_step(c, P.localize(rs), c->mo_resid) || make_step(c, P.localize(up), c->mo_ims_up) ||
        make_step(c, P.localize(late), c->mo_ims_late))
      return -1;
    if (upload(c, &c->mo_zero_blocks, zero) || upload(c, &c->mo_r_blocks, rfill)) return -1;
    c->n_mo_zero = (int)zero.size();
    c->mo_zero_host = zero;
    c->n_mo_r = (int)rfill.size();
  }
  // seam blocks (literal mode): groups shared by consecutive windows
  for (int dir = 0; dir < 2; ++dir) {
    const auto& W = dir == 0 ? P.win_lower : P.win_upper;
    std::set<int> seams;
    for (size_t i = 0; i + 1 < W.size(); ++i) {
      if (dir == 0) seams.insert(W[i].second);   // lower: hi of window i == lo of i+1
      else seams.insert(W[i].first);             // upper: lo of window i == hi of i+1
    }
    std::vector<int> blocks;
    for (int m = 0; m < P.npairs; ++m)
      if (seams.count(P.block_group[m]) && P.subs[P.block_sub[m]].rank == P.rank) blocks.push_back(m);
    dfree(c, c->d_seam[dir], c->n_seam[dir] * sizeof(int));
    c->d_seam[dir] = nullptr;
    if (upload(c, &c->d_seam[dir], blocks)) return -1;
    c->n_seam[dir] = (int)blocks.size();
  }
  // exchange buffers
  size_t need = 0;
  auto upd = [&](const std::vector<DevStep>& v) {
    for (auto& s : v) need = std::max(need, (size_t)std::max(std::max(s.nsend_up, s.nsend_dn), std::max(s.nrecv_up, s.nrecv_dn)));
  };
  upd(c->fwd); upd(c->bwd); upd(c->sp_fwd); upd(c->sp_bwd);
  upd({c->mo_resid, c->mo_ims_up, c->mo_ims_late});
  need = std::max(need, (size_t)std::max(std::max(c->full.nsend_up, c->full.nsend_dn), std::max(c->full.nrecv_up, c->full.nrecv_dn)));
  c->xbuf_cap = need * c->n;  // per RHS; grown with R in ensure_xbuf
  c->steps_dirty = false;
  return 0;
}

int ensure_xbuf(Ctx* c, int R) {
  if (c->plan.nranks == 1) return 0;
  size_t elems = c->xbuf_cap * R;
  double2* p;
  if (ws_get(c, "xsu", elems, &p)) return -1;
  c->send_up = p;
  if (ws_get(c, "xsd", elems, &p)) return -1;
  c->send_dn = p;
  if (ws_get(c, "xru", elems, &p)) return -1;
  c->recv_up = p;
  if (ws_get(c, "xrd", elems, &p)) return -1;
  c->recv_dn = p;
  return 0;
}

cudaEvent_t ev_get(Ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

// One sweep step: batched apply + (row bands) exchange + receive epilogue.
int run_step(Ctx* c, DevStep& st, const double2* srcA, const double2* srcB, Epi e, int R) {
  e.send_up = c->send_up;
  e.send_dn = c->send_dn;
  // kernel choice: shared class maps -> DMMA contraction; per-subdomain maps:
  // one RHS -> HBM ZGEMV (k_step1), several -> DMMA contraction (FFMA fallback
  // when n is not a multiple of the 16-wide K chunk)
  DevMma* mm = nullptr;
  const bool shared = c->map_mode == 1;
  if (st.nitems > 0 && (shared || (R > 1 && c->n % 32 == 0)))
    if (make_mma(c, st, R, shared, &mm)) return -1;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing && st.ntiles > 0) {
    e0 = ev_get(c);
    e1 = ev_get(c);
    cudaEventRecord(e0, c->stream);
  }
  if (mm) launch_zmma(*c, *mm, shared ? c->Tcls : c->T, srcA, srcB, c->zeros, e, R);
  else launch_step(*c, st, srcA, srcB, e, R);
  if (e1) {
    cudaEventRecord(e1, c->stream);
    c->ev_pending.push_back({e0, e1});
    c->ev_bytes.push_back(shared ? 0.0 : st.bytes_per_rhs_map + R * st.bytes_per_rhs_vec);
    c->ev_flops.push_back(mm ? mm->flops : 8.0 * st.bytes_per_rhs_map / 16.0 * R);
  }
  CK(cudaGetLastError());
  if (c->plan.nranks > 1) {
    ncclComm_t comm = (ncclComm_t)c->nccl;
    if (!comm) return fail(c, -2, "sharded context without hs_comm_init");
    const size_t per = (size_t)c->n * R * 2;  // doubles per slot
    const int rk = c->plan.rank;
    NK(ncclGroupStart());
    if (st.nsend_up) NK(ncclSend(c->send_up, per * st.nsend_up, ncclDouble, rk + 1, comm, c->stream));
    if (st.nsend_dn) NK(ncclSend(c->send_dn, per * st.nsend_dn, ncclDouble, rk - 1, comm, c->stream));
    if (st.nrecv_up) NK(ncclRecv(c->recv_up, per * st.nrecv_up, ncclDouble, rk + 1, comm, c->stream));
    if (st.nrecv_dn) NK(ncclRecv(c->recv_dn, per * st.nrecv_dn, ncclDouble, rk - 1, comm, c->stream));
    NK(ncclGroupEnd());
    launch_recv_epi(*c, st, e, R);
    CK(cudaGetLastError());
  }
  return 0;
}

Epi epi(int mode, double2* o1, double2* o2 = nullptr, double2* o3 = nullptr,
        const double2* a = nullptr, const double2* b = nullptr, const double2* cc = nullptr) {
  Epi e;
  e.mode = mode; e.o1 = o1; e.o2 = o2; e.o3 = o3; e.a = a; e.b = b; e.c = cc;
  e.send_up = e.send_dn = nullptr;
  return e;
}

long long LRof(Ctx* c, int R) { return c->plan.L * (long long)R; }

// ---- device pointer in/out for host or device caller buffers
int dev_in(Ctx* c, const double* p, long long elems, int mem, const char* name, const double2** out) {
  if (mem == HS_MEM_DEVICE) {
    *out = (const double2*)p;
    return 0;
  }
  if (mem != HS_MEM_HOST) return fail(c, 1, "mem must be HS_MEM_HOST or HS_MEM_DEVICE");
  double2* d;
  if (ws_get(c, name, elems, &d)) return -1;
  if (elems) CK(cudaMemcpyAsync(d, p, elems * sizeof(double2), cudaMemcpyHostToDevice, c->stream));
  *out = d;
  return 0;
}

int dev_out(Ctx* c, double* p, long long elems, int mem, const char* name, double2** out) {
  if (mem == HS_MEM_DEVICE) {
    *out = (double2*)p;
    return 0;
  }
  if (mem != HS_MEM_HOST) return fail(c, 1, "mem must be HS_MEM_HOST or HS_MEM_DEVICE");
  return ws_get(c, name, elems, out);
}

int finish_out(Ctx* c, double* p, const double2* d, long long elems, int mem) {
  if (mem == HS_MEM_HOST) {
    if (elems) CK(cudaMemcpyAsync(p, d, elems * sizeof(double2), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  } else if (!c->async_mode) {
    CK(cudaStreamSynchronize(c->stream));
  }
  return 0;
}

int check_ready(Ctx* c, int R) {
  NEED_GPU(c);
  if (!c->factored) return fail(c, 1, "hs_factor has not been called");
  if (R < 1 || R > 1024) return fail(c, 1, "nrhs must be in 1..1024");
  if (int e_ = build_steps(c)) return e_;
  if (ensure_xbuf(c, R)) return -1;
  return 0;
}

// ---- preconditioners on device vectors
int do_half(Ctx* c, int dir, const double2* r, double2* z, int R) {
  const long long LR = LRof(c, R);
  CK(cudaMemcpyAsync(z, r, LR * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
  auto& steps = dir == 0 ? c->fwd : c->bwd;
  for (auto& st : steps)
    if (int e_ = run_step(c, st, z, r, epi(EPI_ACC, z), R)) return e_;
  if (c->seam == HS_SEAM_LITERAL) launch_seam_add(*c, dir, z, r, R);
  return 0;
}

void free_emu(Ctx* c) {
  EmuRanks& e = c->emu;
  dfree(c, e.blk_rank, 0);
  for (int g = 0; g < kMaxRanks; ++g) dfree(c, e.tiles[g], 0);
  dfree(c, e.buf, 0);
  dfree(c, e.counters, 0);
  const int G = e.G;
  e = EmuRanks();
  e.G = G;
}

// Per-rank tile lists, owners and buffers of the emulated row bands (the
// row-band partition of Plan::build with G ranks).
int build_emu(Ctx* c) {
  EmuRanks& e = c->emu;
  free_emu(c);
  const Plan& P = c->plan;
  const DevFused& f = c->fused;
  Plan pg;
  std::string err = pg.build(P.n1, P.n2, P.n, 0, e.G);
  if (!err.empty()) return fail(c, 1, "emulated ranks: " + err);
  e.sub_rank.assign(P.nsub, 0);
  for (int s = 0; s < P.nsub; ++s) e.sub_rank[s] = pg.subs[s].rank;
  std::vector<int> br(P.npairs);
  for (int b = 0; b < P.npairs; ++b) br[b] = e.sub_rank[P.block_sub[b]];
  if (upload(c, &e.blk_rank, br)) return -1;
  std::vector<FusedTile> tiles(f.ntiles);
  std::vector<DevItem> items(f.nitems);
  CK(cudaMemcpy(tiles.data(), f.tiles, tiles.size() * sizeof(FusedTile), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(items.data(), f.items, items.size() * sizeof(DevItem), cudaMemcpyDeviceToHost));
  std::vector<std::vector<FusedTile>> per(e.G);
  for (const FusedTile& t : tiles) per[e.sub_rank[items[t.item].s]].push_back(t);
  for (int g = 0; g < e.G; ++g) {
    e.ntiles[g] = (int)per[g].size();
    if (upload(c, &e.tiles[g], per[g])) return -1;
  }
  CK(dalloc(c, (void**)&e.buf, (size_t)e.G * 5 * P.L * sizeof(double2)));
  CK(dalloc(c, (void**)&e.counters, (size_t)e.G * (P.npairs + 1) * sizeof(int)));
  e.built = true;
  return 0;
}

// The fused BSP apply over G emulated row-band ranks on this GPU: every rank
// has its own copy of r, zL, rp, w, z and of the completion counters, uses
// only the blocks it owns, and reaches other ranks' blocks through their
// buffers -- the multi-GPU peer-memory protocol in one launch.
int do_precond_emulated(Ctx* c, const double2* r, double2* z) {
  EmuRanks& e = c->emu;
  if (!e.built && build_emu(c)) return -1;
  const Plan& P = c->plan;
  const long long L = P.L;
  MultiRankArgs mr;
  mr.G = e.G;
  mr.self = -1;
  mr.blk_rank = e.blk_rank;
  const double2* zsrc[kMaxRanks];
  CK(cudaMemsetAsync(e.counters, 0, (size_t)e.G * (P.npairs + 1) * sizeof(int), c->stream));
  for (int g = 0; g < e.G; ++g) {
    double2* base = e.buf + (size_t)g * 5 * L;
    CK(cudaMemcpyAsync(base, r, L * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
    for (int k = 0; k < 5; ++k) mr.v[k][g] = base + (size_t)k * L;  // r, zL, rp, w, z
    mr.v[FV_WOUT][g] = nullptr;
    mr.done[g] = e.counters + (size_t)g * (P.npairs + 1);
    mr.ticket[g] = mr.done[g] + P.npairs;
    mr.tiles[g] = e.tiles[g];
    mr.ntiles[g] = e.ntiles[g];
    zsrc[g] = mr.v[FV_Z][g];
  }
  CK(launch_bsp_fused_ranks(*c, c->fused, mr));
  launch_gather_blocks(*c, z, zsrc, e.G, e.blk_rank, L);
  return cudaGetLastError() == cudaSuccess ? 0 : fail(c, -1, "emulated ranks: launch failed");
}

// ---- row-band ranks on separate GPUs: the fused apply over CUDA IPC ----
void free_peer_plans(Ctx* c) {
  PeerRanks& p = c->peer;
  for (DevFused* fp : {&p.plan, &p.plan_ims}) {
    DevFused& f = *fp;
    dfree(c, f.split_buf, 0);
    dfree(c, f.split_cnt, 0);
    dfree(c, f.items, 0);
    dfree(c, f.tiles, 0);
    dfree(c, f.deps, 0);
    dfree(c, f.counters, 0);
    f = DevFused();
  }
  dfree(c, p.wtot, 0);
  p.wtot = nullptr;
  dfree(c, p.wwtot, 0);
  p.wwtot = nullptr;
}

int peer_barrier(Ctx* c);

// New plans (other windows / plan kind): the epoch counters restart from zero.
// Every rank rebuilds at the same point of its call sequence; one barrier so no
// peer still signals the old epochs, the reset, one barrier so no peer signals
// the new ones before it.
int peer_restart_epochs(Ctx* c) {
  PeerRanks& p = c->peer;
  if (p.epoch == 0) return 0;
  CK(cudaStreamSynchronize(c->stream));
  if (int e = peer_barrier(c)) return e;
  CK(cudaMemsetAsync(p.counters[c->plan.rank], 0, (2 * c->plan.npairs + 2) * sizeof(int), c->stream));
  if (int e = peer_barrier(c)) return e;
  p.epoch = 0;
  p.ims_epoch = 0;
  p.epochs = !(getenv("HS_PEER_BARRIERS") && atoi(getenv("HS_PEER_BARRIERS")) != 0);
  return 0;
}

void free_peer(Ctx* c) {
  PeerRanks& p = c->peer;
  free_peer_plans(c);
  for (int g = 0; g < kMaxRanks; ++g)
    if (p.opened[g]) cudaIpcCloseMemHandle(p.opened[g]);
  dfree(c, p.own, 0);
  dfree(c, p.blk_rank, 0);
  dfree(c, p.own_blocks, 0);
  dfree(c, p.wtot, 0);
  dfree(c, p.bar, 0);
  p = PeerRanks();
}

// Global plan of the row bands (all ranks' tiles in one ticket order) keeping
// the tiles of `rank` (host part; plan-only contexts too).
int peer_plan_host(const Ctx* c, bool ims, int rank, DevFused& f, FusedHost& H) {
  Plan pg;
  std::string err = pg.build(c->n1, c->n2, c->n, 0, 1);
  if (!err.empty()) return fail(const_cast<Ctx*>(c), 1, "peer plan: " + err);
  pg.win_lower = c->plan.win_lower;
  pg.win_upper = c->plan.win_upper;
  std::vector<StepTable> fwd = pg.half_steps(0), bwd = pg.half_steps(1);
  std::vector<int> sub_rank(c->plan.nsub);
  for (int s = 0; s < c->plan.nsub; ++s) sub_rank[s] = c->plan.subs[s].rank;
  return fused_plan_host(c, pg, fwd, pg.full_step(), bwd, ims, f, H, &sub_rank, rank);
}

int build_peer_plan(Ctx* c, bool ims) {
  PeerRanks& p = c->peer;
  DevFused& f = ims ? p.plan_ims : p.plan;
  if (!p.plan.built && !p.plan_ims.built)
    if (int e = peer_restart_epochs(c)) return e;
  FusedHost H;
  if (int e = peer_plan_host(c, ims, c->plan.rank, f, H)) return e;
  if (upload(c, &f.items, H.items) || upload(c, &f.tiles, H.tiles) || upload(c, &f.deps, H.deps)) return -1;
  if (int e = alloc_split(c, f)) return e;
  // the epoch protocol needs the same signals per block from every plan
  // (the BSP and the A M v plans signal the same blocks the same number of times)
  const DevFused& other = ims ? p.plan : p.plan_ims;
  if (other.built && other.wtot != f.wtot) p.epochs = false;
  if (!p.wtot && upload(c, &p.wtot, f.wtot)) return -1;
  if (ims && !p.wwtot && upload(c, &p.wwtot, f.wwtot)) return -1;
  f.built = true;
  return 0;
}

__global__ void k_post_epoch(int* flag, int e) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");  // this rank's inputs (copied before, stream order) first
  *(volatile int*)flag = e;
}

// Stream-ordered barrier of the row-band ranks (a one-element all-reduce).
int peer_barrier(Ctx* c) {
  if (c->peer.G <= 1) return 0;
  ncclComm_t comm = (ncclComm_t)c->nccl;
  if (!comm) return fail(c, -2, "peer ranks without hs_comm_init");
  NK(ncclAllReduce(c->peer.bar, c->peer.bar, 1, ncclDouble, ncclSum, comm, c->stream));
  return 0;
}

// z = M r (and wout = (I - S) z when wout != null) with every rank's tiles on
// its own GPU: inputs into this rank's region, counters reset, barrier (no
// rank signals a peer before the peer has reset), one launch, barrier (every
// write into this rank's blocks has landed), outputs copied back.
int do_precond_peer(Ctx* c, const double2* r, double2* z, double2* wout) {
  PeerRanks& p = c->peer;
  const bool ims = wout != nullptr;
  DevFused& f = ims ? p.plan_ims : p.plan;
  if (!f.built && build_peer_plan(c, ims)) return -1;
  const Plan& P = c->plan;
  const long long L = P.L;
  const int me = P.rank;
  double2* mine = p.vec[me];
  MultiRankArgs mr;
  CK(cudaMemcpyAsync(mine + FV_R * L, r, L * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
  if (p.epochs) {
    // no barrier: post this rank's inputs for the epoch; the kernel's CTAs wait
    // for every rank's post, dependencies count from the epoch's base, and the
    // kernel drains this rank's blocks before it ends
    mr.epoch = ++p.epoch;
    mr.wtot = p.wtot;
    mr.own_blocks = p.own_blocks;
    mr.n_own = p.n_own;
    for (int g = 0; g < p.G; ++g) {
      mr.inflag[g] = p.inflag[g];
      mr.wdone[g] = p.wdone[g];
    }
    if (ims) {  // the A M v apply also drains the wout rows other ranks write
      mr.ims_epoch = ++p.ims_epoch;
      mr.wwtot = p.wwtot;
    }
    CK(cudaMemsetAsync(p.counters[me] + P.npairs, 0, sizeof(int), c->stream));  // own ticket only
    c->launches++;
    k_post_epoch<<<1, 1, 0, c->stream>>>(p.inflag[me], (int)mr.epoch);
  } else {
    CK(cudaMemsetAsync(p.counters[me], 0, (P.npairs + 1) * sizeof(int), c->stream));
    if (int e = peer_barrier(c)) return e;
  }
  mr.G = p.G;
  mr.self = me;
  mr.blk_rank = p.blk_rank;
  for (int g = 0; g < p.G; ++g) {
    for (int k = 0; k < FV_N; ++k) mr.v[k][g] = p.vec[g] + (size_t)k * L;
    mr.done[g] = p.counters[g];
    mr.ticket[g] = p.counters[g] + P.npairs;
  }
  mr.tiles[me] = f.tiles;
  mr.ntiles[me] = f.ntiles;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (c->timing) {
    e0 = ev_get(c);
    e1 = ev_get(c);
    cudaEventRecord(e0, c->stream);
  }
  CK(launch_bsp_fused_ranks(*c, f, mr));
  if (e1) {  // this rank's kernel and its share of the algorithmic bytes
    cudaEventRecord(e1, c->stream);
    c->ev_pending.push_back({e0, e1});
    c->ev_bytes.push_back(f.bytes);
    c->ev_flops.push_back(f.bytes / 2.0);
  }
  if (!p.epochs)
    if (int e = peer_barrier(c)) return e;
  CK(cudaMemcpyAsync(z, mine + FV_Z * L, L * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
  if (ims) CK(cudaMemcpyAsync(wout, mine + FV_WOUT * L, L * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
  return 0;
}

bool fused_bsp_ok(const Ctx* c, int R) {
  return (c->fused_mode & 1) && R == 1 && c->map_mode != 1 && (c->plan.nranks == 1 || c->peer.G > 0) && c->inter &&
         c->seam == HS_SEAM_DEDUP && c->full.nitems > 0;
}

// GMRES's w = (I - S) M r with M = BSP as ONE dataflow launch (z = M r is
// left in z).  Bitwise identical to do_precond + do_apply(HS_APPLY_IMS).
int do_precond_ims(Ctx* c, const double2* r, double2* z, double2* wout) {
  const long long L = c->plan.L;
  double2 *zl, *rp, *w;
  if (ws_get(c, "zL", L, &zl) || ws_get(c, "rp", L, &rp) || ws_get(c, "w", L, &w)) return -1;
  if (c->peer.G > 0) return do_precond_peer(c, r, z, wout);
  if (!c->fused_ims.built && build_fused(c, true)) return -1;
  CK(launch_bsp_fused(*c, c->fused_ims, r, zl, rp, w, z, wout));
  return 0;
}

// The per-step BSP in map-once form (dedup seams, intermediate residual, not
// the literal-arithmetic mask bit 2).
bool mma_fused_path(const Ctx* c, int R) {
  // R right-hand sides on the per-subdomain maps: k_zmma2_df (bit 1, default
  // on); the shared class maps only on request (bit 3: k_zmma2_df n-major for
  // one right-hand side, else k_zmma_fused) -- the per-step k_zmma2 with
  // cluster split-K measured faster there (cfg5 0.393 vs 0.490 ms, 0.384 with
  // HS_ZMMA2_SPLIT=1; cfg3 0.198 vs 0.37 / 0.29)
  return (c->fused_mode & 2) && ((R > 1 && c->map_mode != 1) || (c->map_mode == 1 && (c->fused_mode & 8))) &&
         c->n % 32 == 0 && c->plan.nranks == 1 && c->inter &&
         c->seam == HS_SEAM_DEDUP && c->full.nitems > 0;
}

bool map_once_steps(const Ctx* c) {
  return c->inter && c->seam == HS_SEAM_DEDUP && !(c->fused_mode & 4) && c->mo_resid.host.items.size() > 0;
}

// wout = (I - S) z right after the per-step map-once BSP apply of r (whose
// zL, rp and w are still in the workspace): r on the N/E blocks of final
// backward writers, r - T_up w on every W/S block, (r - rp) + (w - T_low w) on
// the lower rows of the backward window starts -- about half the map reads of
// a full (I - S) step.
int do_ims_mo(Ctx* c, const double2* r, double2* wout, int R) {
  const long long LR = LRof(c, R);
  double2 *zl, *rp, *w;
  if (ws_get(c, "zL", LR, &zl) || ws_get(c, "rp", LR, &rp) || ws_get(c, "w", LR, &w)) return -1;
  launch_block_fill(*c, c->mo_r_blocks, c->n_mo_r, 1, wout, nullptr, nullptr, r, R);
  if (int e_ = run_step(c, c->mo_ims_up, w, w, epi(EPI_IMS, wout, nullptr, nullptr, r), R)) return e_;
  return run_step(c, c->mo_ims_late, w, w, epi(EPI_LATE, wout, nullptr, nullptr, r, rp, w), R);
}

int do_precond(Ctx* c, int kind, const double2* r, double2* z, int R) {
  const long long LR = LRof(c, R);
  if (kind == HS_PC_NONE) {
    CK(cudaMemcpyAsync(z, r, LR * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
    return 0;
  }
  if (kind == HS_PC_SP) {
    double2* zl;
    if (ws_get(c, "zL", LR, &zl)) return -1;
    CK(cudaMemcpyAsync(zl, r, LR * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
    for (auto& st : c->sp_fwd)
      if (int e_ = run_step(c, st, zl, r, epi(EPI_ACC, zl), R)) return e_;
    CK(cudaMemcpyAsync(z, zl, LR * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
    for (auto& st : c->sp_bwd)
      if (int e_ = run_step(c, st, z, zl, epi(EPI_ACC, z), R)) return e_;
    return 0;
  }
  if (kind != HS_PC_BSP) return fail(c, 1, "unknown preconditioner kind");
  double2 *zl, *rp, *w;
  if (ws_get(c, "zL", LR, &zl) || ws_get(c, "rp", LR, &rp) || ws_get(c, "w", LR, &w)) return -1;
  if (fused_bsp_ok(c, R)) {
    // the whole apply as one dataflow launch (bitwise identical to the step sequence)
    if (c->peer.G > 0) return do_precond_peer(c, r, z, nullptr);
    if (!c->fused.built && build_fused(c, false)) return -1;
    if (c->emu.G > 1) return do_precond_emulated(c, r, z);
    // no zL = r copy: the plan's rmask makes tiles read r for blocks zL has not received yet
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {
      e0 = ev_get(c);
      e1 = ev_get(c);
      cudaEventRecord(e0, c->stream);
    }
    CK(launch_bsp_fused(*c, c->fused, r, zl, rp, w, z));
    if (e1) {
      cudaEventRecord(e1, c->stream);
      c->ev_pending.push_back({e0, e1});
      c->ev_bytes.push_back(c->fused.bytes);
      c->ev_flops.push_back(c->fused.bytes / 2.0);
    }
    return 0;
  }
  const bool shared = c->map_mode == 1;
  if (mma_fused_path(c, R)) {
    // the whole apply on the DMMA contraction as one dataflow launch
    if (!c->fused_mma.built || c->fused_mma.R != R || c->fused_mma.shared != shared)
      if (int e_ = build_fused_mma(c, R, shared)) return e_;
    CK(cudaMemcpyAsync(zl, r, LR * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
    FusedMmaArgs a;
    a.A = shared ? c->Tcls : c->T;
    a.r = r; a.zL = zl; a.rp = rp; a.w = w; a.z = z; a.R = R;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (c->timing) {
      e0 = ev_get(c);
      e1 = ev_get(c);
      cudaEventRecord(e0, c->stream);
    }
    CK(launch_zmma_fused(*c, c->fused_mma, a));
    if (e1) {
      cudaEventRecord(e1, c->stream);
      c->ev_pending.push_back({e0, e1});
      c->ev_bytes.push_back(0.0);
      c->ev_flops.push_back(c->fused_mma.flops);
    }
    return 0;
  }
  if (int e_ = do_half(c, 0, r, zl, R)) return e_;
  const double2* rsrc;
  if (map_once_steps(c)) {
    // map-once: r' = 0 on the W/S blocks of exact forward writers (no map read);
    // the residual step covers only the rows where r' can be nonzero
    // (the fill touches other blocks than the residual step: it runs beside it)
    if (!c->aux) {
      CK(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&c->aux_fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&c->aux_join, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(c->aux_fork, c->stream));
    CK(cudaStreamWaitEvent(c->aux, c->aux_fork, 0));
    launch_block_fill(*c, c->mo_zero_blocks, c->n_mo_zero, 0, rp, w, z, zl, R, c->aux);
    CK(cudaEventRecord(c->aux_join, c->aux));
    const int e_res = run_step(c, c->mo_resid, zl, zl, epi(EPI_RESID, rp, w, z, r, zl), R);
    // join the side stream on every path: the fill may still be writing rp/w/z
    // when a failed residual step returns, and the caller may then reuse them
    CK(cudaStreamWaitEvent(c->stream, c->aux_join, 0));
    if (e_res) return e_res;
    rsrc = rp;
  } else if (c->inter) {
    if (int e_ = run_step(c, c->full, zl, zl, epi(EPI_RESID, rp, w, z, r, zl), R)) return e_;
    rsrc = rp;
  } else {
    launch_vec(*c, VEC_INIT_BWD, LR, w, z, r, zl);
    rsrc = r;
  }
  for (auto& st : c->bwd)
    if (int e_ = run_step(c, st, w, rsrc, epi(EPI_ACC2, w, z), R)) return e_;
  if (c->seam == HS_SEAM_LITERAL) launch_seam_add(*c, 1, z, rsrc, R);
  return 0;
}

int do_apply(Ctx* c, int mode, const double2* g, double2* out, int R) {
  if (mode == HS_APPLY_S) return run_step(c, c->full, g, g, epi(EPI_SET, out), R);
  if (mode == HS_APPLY_IMS) return run_step(c, c->full, g, g, epi(EPI_IMS, out, nullptr, nullptr, g), R);
  return fail(c, 1, "unknown apply mode");
}

// ---- factorisation
int build_classes(Ctx* c) {
  const int n = c->n;
  c->classes.clear();
  OpClass gen;
  gen.mask.assign((size_t)n * n, 0);
  c->classes.push_back(gen);
  c->sub_class.assign(c->plan.nsub, 0);
  for (auto& kv : c->dcells) {
    if (kv.second.empty()) continue;
    std::vector<uint8_t> m((size_t)n * n, 0);
    for (int cell : kv.second) m[cell] = 1;
    int found = -1;
    for (size_t i = 0; i < c->classes.size(); ++i)
      if (c->classes[i].mask == m) found = (int)i;
    if (found < 0) {
      OpClass oc;
      oc.mask = m;
      oc.dcells = kv.second;
      c->classes.push_back(oc);
      found = (int)c->classes.size() - 1;
    }
    c->sub_class[kv.first] = found;
  }
  return 0;
}

// Sparse RHS entries for the unit columns of Dirichlet boundary cells (rare:
// a scatterer cell on the subdomain edge) -- eliminated form, SURVEY.md §7.
void dirichlet_boundary_extras(Ctx* c, const OpClass& oc, std::map<std::tuple<int, int, int>, double2>& ex) {
  const int n = c->n;
  const double ih2 = 1.0 / (c->h * c->h);
  auto isd = [&](int k, int x) { return oc.mask[(size_t)k * n + x] != 0; };
  for (int f = 0; f < 4; ++f)
    for (int p = 0; p < n; ++p) {
      int k, x;
      if (f == 0) { k = p; x = 0; } else if (f == 1) { k = 0; x = p; }
      else if (f == 2) { k = n - 1; x = p; } else { k = p; x = n - 1; }
      if (!isd(k, x)) continue;
      const int col = f * n + p;
      const int nb[4][2] = {{k - 1, x}, {k + 1, x}, {k, x - 1}, {k, x + 1}};
      for (auto& q : nb) {
        if (q[0] < 0 || q[0] >= n || q[1] < 0 || q[1] >= n || isd(q[0], q[1])) continue;
        double2& v = ex[std::make_tuple(q[0], q[1], col)];
        v.x += ih2;
      }
    }
}

int upload_extras(Ctx* c, const std::map<std::tuple<int, int, int>, double2>& ex, ExtraRHS& e,
                  std::vector<void*>& owned) {
  const int n = c->n;
  e.row_ptr.assign(n + 1, 0);
  if (ex.empty()) {
    e.row_ptr.clear();
    return 0;
  }
  std::vector<int> xs, cols;
  std::vector<double2> vals;
  for (auto& kv : ex) e.row_ptr[std::get<0>(kv.first) + 1]++;
  for (int k = 0; k < n; ++k) e.row_ptr[k + 1] += e.row_ptr[k];
  for (auto& kv : ex) {  // map is ordered by (k, x, col)
    xs.push_back(std::get<1>(kv.first));
    cols.push_back(std::get<2>(kv.first));
    vals.push_back(kv.second);
  }
  e.d_x = nullptr; e.d_col = nullptr; e.d_val = nullptr;
  const int up = upload(c, &e.d_x, xs) || upload(c, &e.d_col, cols) || upload(c, &e.d_val, vals);
  for (void* q : {(void*)e.d_x, (void*)e.d_col, (void*)e.d_val})
    if (q) owned.push_back(q);
  return up ? -1 : 0;
}

}  // namespace

// ===========================================================================
extern "C" {

const char* hs_version(void) { return HS_VERSION; }

const char* hs_last_error(const hs_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int hs_create(hs_ctx** out, int device, int n1, int n2, int n, double h, double kappa, double tau_re,
              double tau_im, int rank, int nranks) {
  Ctx* c = nullptr;
  if (!out) return fail(nullptr, 1, "null context pointer");
  *out = nullptr;
  if (!(h > 0)) return fail(nullptr, 1, "h must be positive");
  if (!(kappa > 0)) return fail(nullptr, 1, "kappa must be positive");
  if (tau_im == 0) return fail(nullptr, 1, "impedance coefficient must have nonzero imaginary part");
  hs_ctx* x = new hs_ctx();
  std::string e = x->plan.build(n1, n2, n, rank, nranks);
  if (!e.empty()) {
    delete x;
    return fail(nullptr, 1, e);
  }
  x->device = device;
  x->n1 = n1; x->n2 = n2; x->n = n;
  x->h = h; x->kappa = kappa; x->tau_re = tau_re; x->tau_im = tau_im;
  int prev_dev = -1;
  if (device >= 0 && cudaGetDevice(&prev_dev) != cudaSuccess) prev_dev = -1;
  struct Restore {  // the caller's current device is left as it was
    int d;
    ~Restore() {
      if (d >= 0) cudaSetDevice(d);
    }
  } restore_dev{prev_dev};
  if (device >= 0) {
    c = x;
    cudaError_t ce = cudaSetDevice(device);
    if (ce != cudaSuccess) {
      std::string m = std::string("cudaSetDevice: ") + cudaGetErrorString(ce);
      delete x;
      return fail(nullptr, -1, m);
    }
    cudaStreamCreateWithFlags(&x->stream, cudaStreamNonBlocking);
    cudaDeviceGetAttribute(&x->num_sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&x->coop_ok, cudaDevAttrCooperativeLaunch, device);
    set_step_smem_limit();
    set_zmma_smem_limit();
    // per-subdomain records (T_off filled by hs_factor)
    std::vector<DevSub> subs(x->plan.nsub);
    long long off = 0;
    for (int s = 0; s < x->plan.nsub; ++s) {
      const SubPlan& sp = x->plan.subs[s];
      DevSub d;
      d.k = sp.k;
      d.nlow = sp.nlower;
      d.in_off = sp.first_block * n;
      for (int q = 0; q < 4; ++q) d.tgt[q] = q < sp.k ? sp.tgt_block[q] * n : -1;
      const long long K = (long long)sp.k * n;
      // row bands: a rank stores the maps of its own subdomains only
      d.T_off = sp.rank == x->plan.rank ? off : -1;
      if (sp.rank == x->plan.rank) off += ((K + kRowTile - 1) / kRowTile) * kRowTile * K;
      x->plan.subs[s].T_off = d.T_off;
      subs[s] = d;
    }
    x->T_elems = (size_t)off;
    if (upload(x, &x->dsubs, subs)) {
      std::string m = x->err;
      delete x;
      return fail(nullptr, -1, m);
    }
    cudaError_t le = cudaGetLastError();
    if (le != cudaSuccess) {
      std::string m = std::string("device setup: ") + cudaGetErrorString(le);
      delete x;
      return fail(nullptr, -1, m);
    }
  }
  *out = x;
  return 0;
}

int hs_destroy(hs_ctx* c) {
  if (!c) return 0;
  DEV_SCOPE(c);
  if (c->device >= 0) {
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    for (auto& s : c->fwd) free_step(c, s);
    for (auto& s : c->bwd) free_step(c, s);
    for (auto& s : c->sp_fwd) free_step(c, s);
    for (auto& s : c->sp_bwd) free_step(c, s);
    free_step(c, c->full);
    free_fused(c);
    free_fused_mma(c);
    free_peer(c);
    if (c->h_flags) cudaFreeHost(c->h_flags);
    if (c->flag_ev[0]) cudaEventDestroy(c->flag_ev[0]);
    if (c->flag_ev[1]) cudaEventDestroy(c->flag_ev[1]);
    if (c->mgs1_slots) cudaFree(c->mgs1_slots);
    // everything else (maps, work buffers, factors, tables) is in the allocation map
    for (auto& kv : c->alloc_sz) cudaFree(kv.first);
    c->alloc_sz.clear();
    for (auto& p : c->ev_pending) { cudaEventDestroy(p.first); cudaEventDestroy(p.second); }
    for (auto e : c->ev_pool) cudaEventDestroy(e);
    if (c->nccl) ncclCommDestroy((ncclComm_t)c->nccl);
    for (auto e : c->bev)
      if (e) cudaEventDestroy(e);
    if (c->aux_fork) cudaEventDestroy(c->aux_fork);
    if (c->aux_join) cudaEventDestroy(c->aux_join);
    if (c->aux) cudaStreamDestroy(c->aux);
    if (c->copy_in) cudaStreamDestroy(c->copy_in);
    if (c->copy_out) cudaStreamDestroy(c->copy_out);
    cudaStreamDestroy(c->stream);
  }
  delete c;
  return 0;
}

int hs_set_dirichlet(hs_ctx* c, int i1, int i2, const int32_t* cells, int ncells) {
  if (!c) return fail(nullptr, 1, "null context");
  if (i1 < 1 || i1 > c->n1 || i2 < 1 || i2 > c->n2) return fail(c, 1, "subdomain out of range");
  if (ncells < 0 || (ncells > 0 && !cells)) return fail(c, 1, "bad cell list");
  std::vector<int32_t> v(cells, cells + ncells);
  for (int x : v)
    if (x < 0 || x >= c->n * c->n) return fail(c, 1, "Dirichlet cell index out of range");
  std::sort(v.begin(), v.end());
  v.erase(std::unique(v.begin(), v.end()), v.end());
  c->dcells[c->plan.ordinal(i1, i2)] = v;
  c->factored = false;
  return 0;
}

// Map storage offsets for map modes 0 (every own subdomain its own map) and 2
// (one map per distinct (class, face set); aliases share it).  Rewrites the
// device subdomain records and reallocates the map storage when its size
// changes; `rep` = the subdomains whose maps are materialised.
int assign_map_offsets(Ctx* c, std::vector<int>& rep) {
  Plan& P = c->plan;
  const int n = c->n;
  std::map<std::pair<int, int>, long long> kind_off;  // (class, face mask) -> offset
  std::vector<DevSub> subs(P.nsub);
  CK(cudaMemcpy(subs.data(), c->dsubs, subs.size() * sizeof(DevSub), cudaMemcpyDeviceToHost));
  long long off = 0;
  rep.clear();
  for (int s = 0; s < P.nsub; ++s) {
    SubPlan& sp = P.subs[s];
    const long long K = (long long)sp.k * n;
    const long long sz = ((K + kRowTile - 1) / kRowTile) * kRowTile * K;
    long long o = -1;
    if (sp.rank == P.rank) {
      if (c->map_mode == 2) {
        int mask = 0;
        for (int q = 0; q < sp.k; ++q) mask |= 1 << sp.face[q];
        auto key = std::make_pair(c->sub_class[s], mask);
        auto it = kind_off.find(key);
        if (it == kind_off.end()) {
          kind_off[key] = o = off;
          off += sz;
          rep.push_back(s);
        } else {
          o = it->second;
        }
      } else {
        o = off;
        off += sz;
        rep.push_back(s);
      }
    }
    sp.T_off = o;
    subs[s].T_off = o;
  }
  if ((size_t)off != c->T_elems) {
    dfree(c, c->T, 0);
    c->T = nullptr;
    c->T_elems = (size_t)off;
  }
  CK(cudaMemcpy(c->dsubs, subs.data(), subs.size() * sizeof(DevSub), cudaMemcpyHostToDevice));
  return 0;
}

int hs_factor(hs_ctx* c) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  NEED_GPU(c);
  CK(cudaSetDevice(c->device));
  const int n = c->n;
  // a refactorisation replaces the previous class factors and maps
  for (auto& oc : c->classes) {
    dfree(c, oc.T4, 0);
    oc.T4 = nullptr;
  }
  if (c->ws.count("__X")) {
    dfree(c, c->ws["__X"].p, 0);
    c->ws.erase("__X");
  }
  c->factored = false;
  build_classes(c);
  const int ncls = (int)c->classes.size();
  const long long nn = (long long)n * n;
  TmpAllocs tmp(c);  // factorisation temporaries, released on every return path
  // masks
  std::vector<uint8_t> masks;
  for (auto& oc : c->classes) masks.insert(masks.end(), oc.mask.begin(), oc.mask.end());
  uint8_t* dmasks = nullptr;
  if (upload(c, &dmasks, masks)) return -1;
  tmp.add(dmasks);
  // X_k for all classes (kept: lifting solves reuse them; freed at destroy / refactor)
  double2* X;
  const long long xstride = nn * n;
  CK(dalloc(c, (void**)&X, (size_t)xstride * ncls * sizeof(double2)));
  c->ws["__X"].p = X;
  c->ws["__X"].cap = (size_t)xstride * ncls;
  double2 *Rp, *Cp;
  const long long pstride = 32LL * n + 32 * 32;  // row/column panel + the panel inverse
  // two slices each: the twisted elimination runs two chains at once
  CK(tmp.alloc(&Rp, (size_t)pstride * ncls * 2 * sizeof(double2)));
  CK(tmp.alloc(&Cp, (size_t)pstride * ncls * 2 * sizeof(double2)));
  int* dbad;
  CK(tmp.alloc(&dbad, sizeof(int)));
  CK(cudaMemsetAsync(dbad, 0, sizeof(int), c->stream));
  // boundary responses for the 4n unit columns, the forward sweep overlapped
  // with the factorisation (factor_and_solve_boundary)
  const int R = 4 * n;
  double2 *Y, *Bk, *G;
  const long long ystride = nn * R, bstride = (long long)n * R, gstride = 4LL * n * R;
  CK(tmp.alloc(&Y, (size_t)ystride * ncls * sizeof(double2)));
  CK(tmp.alloc(&Bk, (size_t)bstride * ncls * 2 * sizeof(double2)));
  CK(tmp.alloc(&G, (size_t)gstride * ncls * sizeof(double2)));
  std::vector<ExtraRHS> extras(ncls);
  for (int k = 0; k < ncls; ++k) {
    std::map<std::tuple<int, int, int>, double2> ex;
    dirichlet_boundary_extras(c, c->classes[k], ex);
    if (upload_extras(c, ex, extras[k], tmp.p)) return -1;
  }
  static const bool timing = getenv("HS_FACTOR_TIMING") && atoi(getenv("HS_FACTOR_TIMING")) != 0;
  auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
  const double t_pre = now();
  CK(factor_and_solve_boundary(*c, X, xstride, dmasks, ncls, Rp, Cp, pstride, dbad, R, R, extras.data(), Y, ystride,
                               Bk, bstride, G, gstride));
  const double t_fac = now();
  // T4 = -(s/d) I - (2 tau / (h^3 d^2)) G
  const std::complex<double> tau(c->tau_re, c->tau_im);
  const double h = c->h;
  const std::complex<double> d = 1.0 / h - tau / 2.0, s = 1.0 / h + tau / 2.0;
  const std::complex<double> a = -(s / d), b = -(2.0 * tau) / (h * h * h * d * d);
  std::vector<double2*> T4s(ncls);
  for (int k = 0; k < ncls; ++k) {
    CK(dalloc(c, (void**)&c->classes[k].T4, (size_t)16 * nn * sizeof(double2)));
    launch_make_T4(*c, c->classes[k].T4, G + k * gstride, R, make_double2(a.real(), a.imag()),
                   make_double2(b.real(), b.imag()));
    T4s[k] = c->classes[k].T4;
    c->classes[k].X = X + k * xstride;  // view; X freed as a whole at destroy
  }
  // class maps, strip-major (shared-operator mode reads them directly)
  {
    const long long strips = (4LL * n + 31) / 32;
    const long long per = strips * 32 * 4LL * n;
    dfree(c, c->Tcls, c->Tcls_elems * sizeof(double2));
    c->Tcls = nullptr;
    c->Tcls_elems = (size_t)per * ncls;
    CK(dalloc(c, (void**)&c->Tcls, c->Tcls_elems * sizeof(double2)));
    c->Tcls_off.assign(ncls, 0);
    for (int k = 0; k < ncls; ++k) {
      c->Tcls_off[k] = per * k;
      launch_pack_strips(*c, c->classes[k].T4, c->Tcls + per * k, 4 * n, 4 * n);
    }
  }
  // per-subdomain maps, tile-major (the HBM-streamed path); map mode 2: one
  // compact map per distinct (operator class, face set), every subdomain's
  // record pointing at its own kind's
  int2* dtl = nullptr;
  int *dfaces = nullptr, *dcls = nullptr;
  double2** dT4s = nullptr;
  if (c->map_mode == 0 || c->map_mode == 2) {
    std::vector<int> rep;  // subdomains whose maps are materialised
    if (int e = assign_map_offsets(c, rep)) return e;
    if (!c->T) CK(dalloc(c, (void**)&c->T, c->T_elems * sizeof(double2)));
    std::vector<int2> tl;
    std::vector<int> faces(4 * c->plan.nsub, 0), cls(c->plan.nsub, 0);
    for (int s2 : rep)
      for (int t = 0; t * kRowTile < c->plan.subs[s2].k * n; ++t) tl.push_back(make_int2(s2, t));
    for (int s2 = 0; s2 < c->plan.nsub; ++s2) {
      const SubPlan& sp = c->plan.subs[s2];
      for (int q = 0; q < sp.k; ++q) faces[4 * s2 + q] = sp.face[q];
      cls[s2] = c->sub_class[s2];
    }
    const int up = upload(c, &dtl, tl) || upload(c, &dfaces, faces) || upload(c, &dcls, cls) || upload(c, &dT4s, T4s);
    tmp.add(dtl); tmp.add(dfaces); tmp.add(dcls); tmp.add(dT4s);
    if (up) return -1;
    launch_scatter_T(*c, dtl, (int)tl.size(), dfaces, dcls, dT4s);
  } else if (n % 32 != 0) {
    return fail(c, 1, "shared-map mode needs cells_per_side divisible by 32");
  }
  // finite check of the class maps, on the device (flag bit 1)
  for (int k = 0; k < ncls; ++k) launch_finite_check(*c, c->classes[k].T4, 16 * nn, dbad);
  CK(cudaGetLastError());
  int bad = 0;
  CK(cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const double t_maps = now();
  if (timing)
    fprintf(stderr, "[hs_factor] host: elimination + boundary solves %.3f ms, maps + finite check %.3f ms\n", t_fac - t_pre,
            t_maps - t_fac);
  for (auto& oc : c->classes) oc.factored = true;
  if (bad) return fail(c, -3, "singular or non-finite subdomain factorisation");
  c->factored = true;
  c->steps_dirty = true;
  return 0;
}

int hs_lifting_rhs(hs_ctx* c, const double* vals, int nrhs, double* bout, int mem) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (int e = check_ready(c, nrhs)) return e;
  CK(cudaSetDevice(c->device));
  const int n = c->n;
  const long long LR = LRof(c, nrhs);
  double2* b;
  if (int e = dev_out(c, bout, LR, mem, "out", &b)) return e;
  CK(cudaMemsetAsync(b, 0, LR * sizeof(double2), c->stream));
  const double ih2 = 1.0 / (c->h * c->h);
  const std::complex<double> tau(c->tau_re, c->tau_im);
  const std::complex<double> d = 1.0 / c->h - tau / 2.0;
  const std::complex<double> coef = -(2.0 * tau) / (c->h * d);
  size_t vpos = 0;
  for (auto& kv : c->dcells) {
    const auto& cells = kv.second;
    if (cells.empty()) continue;
    const int s = kv.first;
    const SubPlan& sp = c->plan.subs[s];
    const OpClass& oc = c->classes[c->sub_class[s]];
    std::map<std::tuple<int, int, int>, double2> ex;
    auto isd = [&](int k, int x) { return oc.mask[(size_t)k * n + x] != 0; };
    for (size_t ci = 0; ci < cells.size(); ++ci) {
      const int k = cells[ci] / n, x = cells[ci] % n;
      for (int j = 0; j < nrhs; ++j) {
        const double* v = vals + 2 * ((vpos + ci) * nrhs + j);
        double2& e0 = ex[std::make_tuple(k, x, j)];
        e0.x += v[0]; e0.y += v[1];
        const int nb[4][2] = {{k - 1, x}, {k + 1, x}, {k, x - 1}, {k, x + 1}};
        for (auto& q : nb) {
          if (q[0] < 0 || q[0] >= n || q[1] < 0 || q[1] >= n || isd(q[0], q[1])) continue;
          double2& e1 = ex[std::make_tuple(q[0], q[1], j)];
          e1.x += ih2 * v[0]; e1.y += ih2 * v[1];
        }
      }
    }
    vpos += cells.size();
    if (sp.rank != c->plan.rank) continue;
    ExtraRHS er;
    TmpAllocs tmp(c);
    if (upload_extras(c, ex, er, tmp.p)) return -1;
    const long long nn = (long long)n * n;
    double2 *Y, *Bk, *G;
    CK(tmp.alloc(&Y, (size_t)nn * nrhs * sizeof(double2)));
    CK(tmp.alloc(&Bk, (size_t)n * nrhs * sizeof(double2)));
    CK(tmp.alloc(&G, (size_t)4 * n * nrhs * sizeof(double2)));
    // single class: pass its X and mask
    uint8_t* dm = nullptr;
    if (upload(c, &dm, oc.mask)) return -1;
    tmp.add(dm);
    CK(solve_boundary(*c, oc.X, 0, dm, 1, nrhs, 0, &er, Y, 0, Bk, 0, G, 0));
    std::vector<int> ft(4, -1);
    for (int q = 0; q < sp.k; ++q) ft[sp.face[q]] = sp.tgt_block[q] * n;
    int* dft = nullptr;
    if (upload(c, &dft, ft)) return -1;
    tmp.add(dft);
    launch_lift_b(*c, b, G, nrhs, 0, nrhs, dft, make_double2(coef.real(), coef.imag()));
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  }
  return finish_out(c, bout, b, LR, mem);
}

int hs_reconstruct(hs_ctx* c, const double* g, const double* lift_vals, double* field, int mem) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (int e = check_ready(c, 1)) return e;
  const int n = c->n;
  const long long L = c->plan.L;
  const long long F = (long long)c->n1 * c->n2 * n * n;
  const double2* dg;
  double2* df;
  if (int e = dev_in(c, g, L, mem, "rin", &dg)) return e;
  if (int e = dev_out(c, field, F, mem, "rout", &df)) return e;
  CK(cudaMemsetAsync(df, 0, F * sizeof(double2), c->stream));
  const double ih2 = 1.0 / (c->h * c->h);
  const std::complex<double> tau(c->tau_re, c->tau_im);
  const std::complex<double> d = 1.0 / c->h - tau / 2.0;
  const std::complex<double> rc = 1.0 / (c->h * c->h * d);  // rhs_coeff, discretization.py:141
  // lifting data of each Dirichlet subdomain, ordinal order (as hs_lifting_rhs)
  std::map<int, size_t> vstart;
  size_t vpos = 0;
  for (auto& kv : c->dcells) {
    vstart[kv.first] = vpos;
    vpos += kv.second.size();
  }
  for (size_t cl = 0; cl < c->classes.size(); ++cl) {
    const OpClass& oc = c->classes[cl];
    std::vector<int> face_off, col_ab, members;
    for (int s = 0; s < c->plan.nsub; ++s) {
      if (c->sub_class[s] != (int)cl || c->plan.subs[s].rank != c->plan.rank) continue;
      const SubPlan& sp = c->plan.subs[s];
      int fo[4] = {-1, -1, -1, -1};
      for (int q = 0; q < sp.k; ++q) fo[sp.face[q]] = (sp.first_block + q) * n;
      face_off.insert(face_off.end(), fo, fo + 4);
      col_ab.push_back(sp.i1);
      col_ab.push_back(sp.i2);
      members.push_back(s);
    }
    const int R = (int)members.size();
    if (R == 0) continue;
    // lifting: Dirichlet data at the scatterer cells and its coupling into the
    // free neighbours (eliminated form); Dirichlet cells on a face are not
    // supported here (the disk must clear the subdomain edge by half a cell)
    std::map<std::tuple<int, int, int>, double2> ex;
    for (int col = 0; col < R; ++col) {
      auto it = c->dcells.find(members[col]);
      if (it == c->dcells.end() || it->second.empty()) continue;
      for (int cell : it->second) {
        const int k = cell / n, x = cell % n;
        if (k == 0 || k == n - 1 || x == 0 || x == n - 1)
          return fail(c, 1, "reconstruction: scatterer cells on a subdomain face are not supported");
      }
      if (!lift_vals) continue;
      auto isd = [&](int k, int x) { return oc.mask[(size_t)k * n + x] != 0; };
      const size_t v0 = vstart[members[col]];
      for (size_t ci = 0; ci < it->second.size(); ++ci) {
        const int k = it->second[ci] / n, x = it->second[ci] % n;
        const double* v = lift_vals + 2 * (v0 + ci);
        double2& e0 = ex[std::make_tuple(k, x, col)];
        e0.x += v[0]; e0.y += v[1];
        const int nb[4][2] = {{k - 1, x}, {k + 1, x}, {k, x - 1}, {k, x + 1}};
        for (auto& q : nb) {
          if (isd(q[0], q[1])) continue;
          double2& e1 = ex[std::make_tuple(q[0], q[1], col)];
          e1.x += ih2 * v[0]; e1.y += ih2 * v[1];
        }
      }
    }
    ExtraRHS er;
    TmpAllocs tmp(c);
    if (upload_extras(c, ex, er, tmp.p)) return -1;
    int *dfo = nullptr, *dab = nullptr;
    uint8_t* dm = nullptr;
    const int up = upload(c, &dfo, face_off) || upload(c, &dab, col_ab) || upload(c, &dm, oc.mask);
    tmp.add(dfo); tmp.add(dab); tmp.add(dm);
    if (up) return -1;
    double2 *Y, *Bk;
    CK(tmp.alloc(&Y, (size_t)n * n * R * sizeof(double2)));
    CK(tmp.alloc(&Bk, (size_t)n * R * sizeof(double2)));
    CK(solve_fields(*c, oc.X, dm, R, dg, dfo, make_double2(rc.real(), rc.imag()), er, Y, Bk));
    launch_scatter_field(*c, df, c->n1 * n, Y, R, dab, 0);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(c->stream));
  }
  return finish_out(c, field, df, F, mem);
}

int hs_apply(hs_ctx* c, int mode, const double* g, double* out, int nrhs, int mem) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (int e = check_ready(c, nrhs)) return e;
  const long long LR = LRof(c, nrhs);
  const double2* dg;
  double2* dout;
  if (int e = dev_in(c, g, LR, mem, "in", &dg)) return e;
  if (int e = dev_out(c, out, LR, mem, "out", &dout)) return e;
  if (int e_ = do_apply(c, mode, dg, dout, nrhs)) return e_;
  return finish_out(c, out, dout, LR, mem);
}

int hs_restricted_apply(hs_ctx* c, const double* g, double* out, int nrhs, const int32_t* src,
                        int nsrc, const int32_t* tgt, int ntgt, int mem) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (int e = check_ready(c, nrhs)) return e;
  const long long LR = LRof(c, nrhs);
  const double2* dg;
  double2* dout;
  if (int e = dev_in(c, g, LR, mem, "in", &dg)) return e;
  if (int e = dev_out(c, out, LR, mem, "out", &dout)) return e;
  std::vector<int> S(src, src + std::max(nsrc, 0)), Tg(tgt, tgt + std::max(ntgt, 0));
  DevStep st;
  if (make_step(c, c->plan.restricted_step(S, Tg), st)) return -1;
  CK(cudaMemsetAsync(dout, 0, LR * sizeof(double2), c->stream));
  int rc = run_step(c, st, dg, dg, epi(EPI_SET, dout), nrhs);
  int rc2 = finish_out(c, out, dout, LR, mem);
  cudaStreamSynchronize(c->stream);
  free_step(c, st);
  return rc ? rc : rc2;
}

int hs_set_windows(hs_ctx* c, int kind, const int32_t* lo, const int32_t* hi, int nwin) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (kind != 0 && kind != 1) return fail(c, 1, "window kind must be 0 (lower) or 1 (upper)");
  std::vector<std::pair<int, int>> w;
  const int ng = c->plan.ng;
  for (int i = 0; i < nwin; ++i) {
    if (lo[i] < 2 || hi[i] > ng + 1 || lo[i] >= hi[i]) return fail(c, 1, "window out of range");
    w.push_back({lo[i], hi[i]});
  }
  (kind == 0 ? c->plan.win_lower : c->plan.win_upper) = w;
  c->steps_dirty = true;
  return 0;
}

int hs_set_precond_options(hs_ctx* c, int seam_mode, int inter) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (seam_mode != HS_SEAM_DEDUP && seam_mode != HS_SEAM_LITERAL) return fail(c, 1, "bad seam mode");
  c->seam = seam_mode;
  c->inter = inter ? 1 : 0;
  return 0;
}

int hs_precond(hs_ctx* c, int kind, const double* r, double* z, int nrhs, int mem) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (int e = check_ready(c, nrhs)) return e;
  const long long LR = LRof(c, nrhs);
  const double2* dr;
  double2* dz;
  if (int e = dev_in(c, r, LR, mem, "in", &dr)) return e;
  if (int e = dev_out(c, z, LR, mem, "out", &dz)) return e;
  if (int e_ = do_precond(c, kind, dr, dz, nrhs)) return e_;
  return finish_out(c, z, dz, LR, mem);
}

// A batch of independent host vectors through the preconditioner, pipelined
// over two copy streams and two device slots: vector i+1 lands (H2D) and
// vector i-1 drains (D2H) while vector i is applied, so each vector's copies
// hide behind a neighbour's apply.  Every vector still makes the full round
// trip host -> HBM -> host.
int hs_precond_batch(hs_ctx* c, int kind, const double* const* r, double* const* z, int nvec, int nrhs) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (nvec < 0 || (nvec > 0 && (!r || !z))) return fail(c, 1, "bad batch");
  if (int e = check_ready(c, nrhs)) return e;
  if (nvec == 0) return 0;
  const long long LR = LRof(c, nrhs);
  const size_t bytes = LR * sizeof(double2);
  if (!c->copy_in) {
    CK(cudaStreamCreateWithFlags(&c->copy_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->copy_out, cudaStreamNonBlocking));
    for (auto& e : c->bev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  double2 *din[2], *dout[2];
  if (ws_get(c, "bin0", LR, &din[0]) || ws_get(c, "bin1", LR, &din[1]) || ws_get(c, "bout0", LR, &dout[0]) ||
      ws_get(c, "bout1", LR, &dout[1]))
    return -1;
  cudaEvent_t* landed = c->bev;       // [2] input slot filled
  cudaEvent_t* applied = c->bev + 2;  // [2] apply done: input slot free, output ready
  cudaEvent_t* drained = c->bev + 4;  // [2] output copied out: output slot free
  for (int i = 0; i < nvec; ++i) {
    const int s = i & 1;
    if (i >= 2) CK(cudaStreamWaitEvent(c->copy_in, applied[s], 0));
    CK(cudaMemcpyAsync(din[s], r[i], bytes, cudaMemcpyHostToDevice, c->copy_in));
    CK(cudaEventRecord(landed[s], c->copy_in));
    CK(cudaStreamWaitEvent(c->stream, landed[s], 0));
    if (i >= 2) CK(cudaStreamWaitEvent(c->stream, drained[s], 0));
    if (int e_ = do_precond(c, kind, din[s], dout[s], nrhs)) {
      // no copy may still be in flight into the caller's buffers or the slots
      cudaStreamSynchronize(c->copy_in);
      cudaStreamSynchronize(c->copy_out);
      cudaStreamSynchronize(c->stream);
      return e_;
    }
    CK(cudaEventRecord(applied[s], c->stream));
    CK(cudaStreamWaitEvent(c->copy_out, applied[s], 0));
    CK(cudaMemcpyAsync(z[i], dout[s], bytes, cudaMemcpyDeviceToHost, c->copy_out));
    CK(cudaEventRecord(drained[s], c->copy_out));
  }
  CK(cudaStreamSynchronize(c->copy_out));
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int hs_half_apply(hs_ctx* c, int direction, const double* r, double* z, int nrhs, int mem) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (direction != 0 && direction != 1) return fail(c, 1, "direction must be 0 or 1");
  if (int e = check_ready(c, nrhs)) return e;
  const long long LR = LRof(c, nrhs);
  const double2* dr;
  double2* dz;
  if (int e = dev_in(c, r, LR, mem, "in", &dr)) return e;
  if (int e = dev_out(c, z, LR, mem, "out", &dz)) return e;
  if (int e_ = do_half(c, direction, dr, dz, nrhs)) return e_;
  return finish_out(c, z, dz, LR, mem);
}

int hs_gmres(hs_ctx* c, int pc, const double* b, double* x, int R, double tol, int maxit,
             int* iters, double* hist, int* converged, int mem) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (int e = check_ready(c, R)) return e;
  if (!(tol > 0) || maxit < 1) return fail(c, 1, "tol must be > 0 and maxit >= 1");
  if (pc < HS_PC_NONE || pc > HS_PC_BSP) return fail(c, 1, "unknown preconditioner kind");
  // Arnoldi: one cooperative kernel per iteration on one GPU; across row bands
  // (or when forced) the host-driven MGS over owned blocks + allreduce per dot
  // Row bands, one RHS, auto mode: CGS2 -- two all-reduces per iteration
  // instead of one per inner product (k + 1), which would dominate the sharded
  // iteration (54 small all-reduces per iteration on average at cfg5);
  // iterations within +-1 of MGS (tests).
  // One RHS, auto mode: CGS2 with the Gram correction -- ONE reduction per
  // iteration, two passes over V, no barrier chain -- on one GPU and across
  // row bands (HS_ARNOLDI_BANDS=cgs2: the two-reduction CGS2 across bands);
  // measured faster than the MGS kernels on every config (cfg1 1.9 vs 2.3 ms,
  // cfg2 5.4 vs 8.0, cfg3 23.3 vs 25.5, cfg5 0.240 vs 0.244 s GMRES) with the
  // same iterations and histories within 1e-10 of the oracle's MGS.  Mode 5
  // ("mgs") keeps the MGS kernels (the SPEC's literal Arnoldi).
  static const bool bands_cgs2 = getenv("HS_ARNOLDI_BANDS") && std::string(getenv("HS_ARNOLDI_BANDS")) == "cgs2";
  // (the coefficient kernel keeps ~8 (k + 1) complex values in shared memory
  // and the Gram matrix is (maxit + 1)^2: beyond 1500 iterations the MGS kernels)
  const bool auto1 = c->gmres_mode == 0 && R == 1 && maxit <= 1500;
  const bool cgs2 = c->gmres_mode == 3 || (auto1 && c->plan.nranks > 1 && bands_cgs2);
  const bool cgsg = c->gmres_mode == 4 || (auto1 && !(c->plan.nranks > 1 && bands_cgs2));
  const long long LR = LRof(c, R);
  // R right-hand sides on one rank: the same one-reduction Arnoldi, column by
  // column (auto mode, or forced "cgs2g"); HS_ARNOLDI_R=mgs keeps the
  // cooperative MGS kernel
  static const bool r_mgs = getenv("HS_ARNOLDI_R") && std::string(getenv("HS_ARNOLDI_R")) == "mgs";
  const bool cgsgR = R > 1 && c->plan.nranks == 1 && LR > 0 && ((c->gmres_mode == 0 && !r_mgs) || c->gmres_mode == 4) &&
                     gmres_cgsgR_ok(*c, LR, R, maxit);
  if (cgs2 && R != 1) return fail(c, 1, "CGS2 Arnoldi supports one right-hand side");
  if (cgsg && R != 1 && !cgsgR)
    return fail(c, 1, "the Gram-corrected CGS2 Arnoldi with several right-hand sides needs one rank, R <= 128 and maxit "
                      "small enough for the Gram matrices (2 GB)");
  if (cgsg && R == 1 && maxit > 1500) return fail(c, 1, "the Gram-corrected CGS2 Arnoldi supports maxit <= 1500");
  const bool dist = !cgsgR && (c->plan.nranks > 1 || c->gmres_mode == 1 || cgs2 || cgsg);
  if (LR == 0) {  // empty interface system (1 x 1 lattice): 0 iterations
    for (int r = 0; r < R; ++r) {
      if (iters) iters[r] = 0;
      if (converged) converged[r] = 1;
      if (hist) hist[r] = 1.0;
    }
    return 0;
  }
  const double2* db;
  double2* dx;
  if (int e = dev_in(c, b, LR, mem, "gin", &db)) return e;
  if (int e = dev_out(c, x, LR, mem, "gout", &dx)) return e;
  int chunk = 0;
  int grid = dist ? 2 * c->num_sms : gmres_coop_grid(*c, LR, R, &chunk);
  if (grid <= 0 && cgsgR) grid = 1;  // the cooperative kernel is not used
  if (grid <= 0) return fail(c, 3, "interface vector too large for the cooperative Arnoldi kernel");
  double2 *part2 = nullptr, *mgsout = nullptr, *part3 = nullptr, *hbuf = nullptr, *gram = nullptr;
  if (dist) {
    if (!c->d_owned) {
      std::vector<int> owned;
      for (int m = 0; m < c->plan.npairs; ++m)
        if (c->plan.subs[c->plan.block_sub[m]].rank == c->plan.rank) owned.push_back(m);
      if (upload(c, &c->d_owned, owned)) return -1;
      c->n_owned = (int)owned.size();
    }
    if (ws_get(c, "part2", (size_t)grid * 2 * R, &part2) || ws_get(c, "mgsout", (size_t)2 * R, &mgsout)) return -1;
    if (cgs2 && (ws_get(c, "part3", (size_t)grid * (maxit + 2), &part3) || ws_get(c, "hbuf", (size_t)maxit + 2, &hbuf)))
      return -1;
    if (cgsg && (ws_get(c, "part3", (size_t)grid * (2 * maxit + 3), &part3) ||
                 ws_get(c, "hbuf", (size_t)3 * maxit + 6, &hbuf) ||
                 ws_get(c, "gram", (size_t)(maxit + 1) * (maxit + 1), &gram)))
      return -1;
  }
  if (cgsgR) {
    const size_t g2 = 2 * (size_t)c->num_sms;
    if (ws_get(c, "part3", g2 * (2 * maxit + 3) * R, &part3) || ws_get(c, "hbuf", ((size_t)3 * maxit + 6) * R + 1, &hbuf) ||
        ws_get(c, "gram", (size_t)R * (maxit + 1) * (maxit + 1), &gram))
      return -1;
    // the coefficient kernels' active-count / ticket pair, past the buffer's data
    CK(cudaMemsetAsync(hbuf + ((size_t)3 * maxit + 6) * R, 0, sizeof(double2), c->stream));
  }
  GmresDev G;
  G.LR = LR; G.R = R; G.tol = tol;
  double2 *V, *Z;
  if (ws_get(c, "V", (size_t)(maxit + 1) * LR, &V) || ws_get(c, "Z", LR, &Z)) return -1;
  G.V = V;
  const long long hsz = (long long)R * ((long long)maxit * (maxit + 3) / 2 + 2);
  double2 *H, *sn, *g, *part, *y;
  double2* scal;
  if (ws_get(c, "H", hsz, &H) || ws_get(c, "sn", (size_t)maxit * R, &sn) ||
      ws_get(c, "g", (size_t)(maxit + 1) * R, &g) || ws_get(c, "part", (size_t)2 * (grid + 2 * c->num_sms) * R, &part) ||
      ws_get(c, "y", (size_t)maxit * R, &y) ||
      ws_get(c, "scal", (size_t)(maxit + 1) * R + 4 * R + (size_t)maxit * R, &scal))
    return -1;
  int* ints;
  double2* iw;
  if (ws_get(c, "gint", (size_t)(5 * R + 1) / 4 + 2, &iw)) return -1;
  ints = (int*)iw;
  G.H = H; G.sn = sn; G.g = g; G.partial = part; G.y = y;
  double* sd = (double*)scal;
  G.hist = sd;
  G.beta = sd + (size_t)(maxit + 1) * R;
  G.wnorm0 = G.beta + R;
  G.cs = G.wnorm0 + R;
  G.active = ints; G.iters = ints + R; G.conv = ints + 2 * R; G.brk = ints + 3 * R; G.nactive = ints + 4 * R;
  if (dist) CK(gmres_init_dist(*c, G, db, c->d_owned, c->n_owned, part2, mgsout, c->nccl));
  else CK(gmres_init(*c, G, db));
  int nact = 0;
  CK(cudaMemcpyAsync(&nact, G.nactive, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  // Convergence flags come back through pinned memory.  When an iteration is
  // short, iteration k+1 is enqueued before iteration k's flag is read (one
  // iteration of lookahead hides the round trip; a speculative iteration after
  // convergence is harmless: k_givens skips inactive right-hand sides and the
  // solution uses the device-side iteration counts).
  if (!c->h_flags) {
    CK(cudaHostAlloc((void**)&c->h_flags, 4 * sizeof(int), cudaHostAllocDefault));
    CK(cudaEventCreateWithFlags(&c->flag_ev[0], cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&c->flag_ev[1], cudaEventDisableTiming));
  }
  bool lookahead = c->map_mode == 1 || (double)c->T_elems * 16.0 < 2e9;
  if (const char* e = getenv("HS_GMRES_LOOKAHEAD")) lookahead = atoi(e) != 0;
  int c1chunk = 0, c1E = 0, c1bd = 0;
  const int c1cs = (dist || c->gmres_mode == 2) ? 0 : gmres_mgs1c_plan(LR, R, maxit, &c1chunk, &c1E, &c1bd);
  int cchunk = 0;
  const int ccs = (dist || c->gmres_mode == 2 || c1cs > 0) ? 0 : gmres_cluster_size(LR, R, &cchunk);
  int m1chunk = 0, m1E = 0, m1bd = 0;
  const int m1grid = (dist || c->gmres_mode == 2 || ccs > 0 || c1cs > 0) ? 0 : gmres_mgs1_plan(*c, LR, R, maxit, &m1chunk, &m1E, &m1bd);
  int kdone = 0;
  bool stop = nact == 0;
  for (int k = 0; k < maxit && !stop; ++k) {
    double2* vk = V + (long long)k * LR;
    double2* w = V + (long long)(k + 1) * LR;
    if (pc == HS_PC_BSP && fused_bsp_ok(c, R) && !c->timing) {
      if (int e_ = do_precond_ims(c, vk, Z, w)) return e_;  // A M v_k in one launch
    } else {
      const double2* zin = vk;
      if (pc != HS_PC_NONE) {
        if (int e_ = do_precond(c, pc, vk, Z, R)) return e_;
        zin = Z;
      }
      if (pc == HS_PC_BSP && map_once_steps(c) && !fused_bsp_ok(c, R) && !mma_fused_path(c, R)) {
        if (int e_ = do_ims_mo(c, vk, w, R)) return e_;  // (I - S) M v_k from the apply's own state
      } else {
        if (int e_ = do_apply(c, HS_APPLY_IMS, zin, w, R)) return e_;
      }
    }
    if (cgsgR) {
      CK(gmres_arnoldi_cgsgR(*c, G, k, part3, hbuf, gram, maxit + 1,
                             (int*)(hbuf + ((size_t)3 * maxit + 6) * R)));  // includes the Givens update
    } else if (cgsg) {
      // one rank owns every block, in order: identity element mapping
      CK(gmres_arnoldi_cgsg(*c, G, k, c->plan.nranks == 1 ? nullptr : c->d_owned, c->n_owned, part3, hbuf, gram,
                            maxit + 1, c->nccl));  // includes the Givens update
    } else if (cgs2) {
      CK(gmres_arnoldi_cgs2(*c, G, k, c->d_owned, c->n_owned, part3, hbuf, c->nccl));
      CK(gmres_givens(*c, G, k));
    } else if (dist) {
      CK(gmres_arnoldi_dist(*c, G, k, c->d_owned, c->n_owned, part2, mgsout, c->nccl));
      CK(gmres_givens(*c, G, k));
    } else if (c1cs > 0) {
      CK(gmres_arnoldi1c(*c, G, k, c1cs, c1chunk, c1E, c1bd));  // includes the Givens update
    } else if (ccs > 0) {
      CK(gmres_arnoldi_cluster(*c, G, k, ccs, cchunk));  // includes the Givens update
    } else if (m1grid > 0) {
      CK(gmres_arnoldi1(*c, G, k, m1grid, m1chunk, m1E, m1bd));  // includes the Givens update
    } else {
      CK(gmres_arnoldi(*c, G, k, grid, chunk));
      CK(gmres_givens(*c, G, k));
    }
    CK(cudaMemcpyAsync(&c->h_flags[k & 1], G.nactive, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaEventRecord(c->flag_ev[k & 1], c->stream));
    kdone = k + 1;
    const int chk = lookahead ? k - 1 : k;  // the iteration whose flag decides
    if (chk >= 0) {
      CK(cudaEventSynchronize(c->flag_ev[chk & 1]));
      if (c->h_flags[chk & 1] == 0) stop = true;
    }
  }
  if (kdone > 0) {
    double2* u;
    if (ws_get(c, "U", LR, &u)) return -1;
    CK(gmres_finish(*c, G, kdone, u));
    if (pc != HS_PC_NONE) {
      if (int e_ = do_precond(c, pc, u, dx, R)) return e_;
    } else {
      CK(cudaMemcpyAsync(dx, u, LR * sizeof(double2), cudaMemcpyDeviceToDevice, c->stream));
    }
  } else {
    CK(cudaMemsetAsync(dx, 0, LR * sizeof(double2), c->stream));
  }
  std::vector<int> hi(5 * R);
  CK(cudaMemcpyAsync(hi.data(), ints, 5 * R * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  if (hist) CK(cudaMemcpyAsync(hist, G.hist, (size_t)(kdone + 1) * R * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  if (int e = finish_out(c, x, dx, LR, mem)) return e;
  CK(cudaStreamSynchronize(c->stream));
  for (int r = 0; r < R; ++r) {
    if (iters) iters[r] = hi[R + r];
    if (converged) converged[r] = hi[2 * R + r];
  }
  int itmax = 0;  // the basis of the reported iterations (a look-ahead step may have built one more)
  for (int r = 0; r < R; ++r) itmax = std::max(itmax, hi[R + r]);
  c->gm_basis = itmax > 0 ? std::min(kdone, itmax) + 1 : 0;
  c->gm_LR = LR;
  return 0;
}

int hs_gmres_basis(hs_ctx* c, double* out, int ncols, int* avail) {
  if (!c || !avail) return fail(c, 1, "null argument");
  DEV_SCOPE(c);
  *avail = c->gm_basis;
  if (!out) return 0;
  if (ncols < 0 || ncols > c->gm_basis) return fail(c, 1, "ncols exceeds the basis of the last GMRES solve");
  auto it = c->ws.find("V");
  if (it == c->ws.end() || it->second.cap < (size_t)ncols * c->gm_LR) return fail(c, 1, "no GMRES basis");
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(out, it->second.p, (size_t)ncols * c->gm_LR * sizeof(double2), cudaMemcpyDeviceToHost));
  return 0;
}

// ---- introspection ---------------------------------------------------------
int hs_sizes(const hs_ctx* c, int64_t* L, int* nsub, int* ngroups, int* npairs) {
  if (!c) return 1;
  if (L) *L = c->plan.L;
  if (nsub) *nsub = c->plan.nsub;
  if (ngroups) *ngroups = c->plan.ng;
  if (npairs) *npairs = c->plan.npairs;
  return 0;
}

int hs_pairs(const hs_ctx* c, int32_t* pairs) {
  if (!c) return 1;
  const Plan& P = c->plan;
  for (int m = 0; m < P.npairs; ++m) {
    const SubPlan& o = P.subs[P.block_sub[m]];
    const int q = m - o.first_block;
    const SubPlan& nb = P.subs[o.nbr[q]];
    pairs[4 * m] = o.i1; pairs[4 * m + 1] = o.i2; pairs[4 * m + 2] = nb.i1; pairs[4 * m + 3] = nb.i2;
  }
  return 0;
}

int hs_block_owner(const hs_ctx* c, int32_t* owner) {
  if (!c) return 1;
  for (int m = 0; m < c->plan.npairs; ++m) owner[m] = c->plan.subs[c->plan.block_sub[m]].rank;
  return 0;
}

int hs_schedule(const hs_ctx* cc, int kind, int32_t* rec, int cap, int* count) {
  if (!cc) return 1;
  hs_ctx* c = const_cast<hs_ctx*>(cc);
  Plan P = c->plan;  // copy: full (unsharded) schedule
  P.nranks = 1; P.rank = 0;
  for (auto& s : P.subs) s.rank = 0;
  std::vector<int32_t> out;
  std::string bad;
  auto emit = [&](const std::vector<StepTable>& steps, int phase, int& step) {
    for (auto& st : steps) {
      ++step;
      if (bad.empty()) bad = P.check_step(st, true);
      std::set<int> seen;
      for (auto& it : st.items)
        if (seen.insert(it.s).second) { out.push_back(step); out.push_back(phase); out.push_back(it.s); }
    }
  };
  int step = 0;
  if (kind == HS_PC_SP) {
    P.win_lower.clear(); P.win_upper.clear();
    if (P.ng >= 2) { P.win_lower.push_back({2, P.ng + 1}); P.win_upper.push_back({2, P.ng + 1}); }
    emit(P.half_steps(0), 0, step);
    emit(P.half_steps(1), 2, step);
  } else if (kind == HS_PC_BSP) {
    emit(P.half_steps(0), 0, step);
    emit(P.half_steps(1), 2, step);
  } else if (kind != HS_PC_NONE) {
    return fail(c, 1, "unknown preconditioner kind");
  }
  if (!bad.empty()) return fail(c, 1, "windows give an unsafe sweep: " + bad);
  *count = (int)(out.size() / 3);
  if (rec) {
    if (cap < *count) return fail(c, 1, "schedule buffer too small");
    std::copy(out.begin(), out.end(), rec);
  }
  return 0;
}

int hs_exchange_plan(const hs_ctx* cc, int kind, int peer, int recv, int32_t* blocks, int cap,
                     int* count) {
  if (!cc) return 1;
  hs_ctx* c = const_cast<hs_ctx*>(cc);
  const Plan& P = c->plan;
  std::vector<StepTable> steps;
  if (kind == 0) steps = P.half_steps(0);
  else if (kind == 1) steps = P.half_steps(1);
  else if (kind == 2) steps.push_back(P.full_step());
  else if (kind >= 3 && kind <= 5) {  // map-once per-step tables: residual rows, (I - S) upper, late
    StepTable rs, up, late;
    std::vector<int> zero, rfill;
    map_once_tables(P, c->n, rs, up, late, zero, rfill);
    steps.push_back(P.localize(kind == 3 ? rs : kind == 4 ? up : late));
  } else return fail(c, 1, "kind must be 0..5");
  std::vector<int32_t> out;
  for (size_t t = 0; t < steps.size(); ++t) {
    if (recv) {
      for (auto& rs : steps[t].recv) {
        const int src = rs.dir == 0 ? P.rank - 1 : P.rank + 1;
        if (src != peer) continue;
        out.push_back((int32_t)t);
        out.push_back((int32_t)(rs.off / c->n));
        out.push_back(rs.slot);
      }
      continue;
    }
    for (auto& it : steps[t].items) {
      const SubPlan& sp = P.subs[it.s];
      for (int q = 0; q < sp.k; ++q) {
        const int sl = it.slot[q];
        if (sl == -1) continue;
        const int dst = sl >= 0 ? P.rank + 1 : P.rank - 1;
        if (dst != peer) continue;
        out.push_back((int32_t)t);
        out.push_back(sp.tgt_block[q]);
        out.push_back(sl >= 0 ? sl : -sl - 2);
      }
    }
  }
  *count = (int)(out.size() / 3);
  if (blocks) {
    if (cap < *count) return fail(c, 1, "buffer too small");
    std::copy(out.begin(), out.end(), blocks);
  }
  return 0;
}

int hs_get_schur(hs_ctx* c, int i1, int i2, double* T) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  NEED_GPU(c);
  if (!c->factored || (!c->T && !c->Tcls)) return fail(c, 1, "no maps (call hs_factor)");
  if (i1 < 1 || i1 > c->n1 || i2 < 1 || i2 > c->n2) return fail(c, 1, "subdomain out of range");
  const int s = c->plan.ordinal(i1, i2);
  const SubPlan& sp = c->plan.subs[s];
  const long long K = (long long)sp.k * c->n;
  const long long nt = (K + kRowTile - 1) / kRowTile;
  CK(cudaStreamSynchronize(c->stream));
  if (!c->T || sp.T_off < 0) {  // shared-map mode or another band's subdomain: compact sub-block of the class map
    const int n = c->n, n4 = 4 * n;
    std::vector<double2> t4((size_t)n4 * n4);
    CK(cudaMemcpy(t4.data(), c->classes[c->sub_class[s]].T4, t4.size() * sizeof(double2),
                  cudaMemcpyDeviceToHost));
    for (long long r = 0; r < K; ++r)
      for (long long col = 0; col < K; ++col) {
        const long long gr = sp.face[r / n] * n + r % n, gc = sp.face[col / n] * n + col % n;
        T[2 * (r * K + col)] = t4[(size_t)(gr * n4 + gc)].x;
        T[2 * (r * K + col) + 1] = t4[(size_t)(gr * n4 + gc)].y;
      }
    return 0;
  }
  std::vector<double2> tm((size_t)nt * kRowTile * K);
  CK(cudaMemcpy(tm.data(), c->T + sp.T_off, tm.size() * sizeof(double2), cudaMemcpyDeviceToHost));
  for (long long r = 0; r < K; ++r)
    for (long long col = 0; col < K; ++col) {
      const double2 v = tm[(size_t)((r / kRowTile) * K + col) * kRowTile + r % kRowTile];
      T[2 * (r * K + col)] = v.x;
      T[2 * (r * K + col) + 1] = v.y;
    }
  return 0;
}

int hs_set_schur(hs_ctx* c, int i1, int i2, const double* T) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  NEED_GPU(c);
  if (i1 < 1 || i1 > c->n1 || i2 < 1 || i2 > c->n2) return fail(c, 1, "subdomain out of range");
  if (!c->T) CK(dalloc(c, (void**)&c->T, c->T_elems * sizeof(double2)));
  const SubPlan& sp = c->plan.subs[c->plan.ordinal(i1, i2)];
  if (sp.T_off < 0) return fail(c, 1, "subdomain not in this rank's row band");
  const long long K = (long long)sp.k * c->n;
  const long long nt = (K + kRowTile - 1) / kRowTile;
  std::vector<double2> tm((size_t)nt * kRowTile * K, make_double2(0, 0));
  for (long long r = 0; r < K; ++r)
    for (long long col = 0; col < K; ++col)
      tm[(size_t)((r / kRowTile) * K + col) * kRowTile + r % kRowTile] =
          make_double2(T[2 * (r * K + col)], T[2 * (r * K + col) + 1]);
  CK(cudaMemcpyAsync(c->T + sp.T_off, tm.data(), tm.size() * sizeof(double2), cudaMemcpyHostToDevice,
                     c->stream));
  CK(cudaStreamSynchronize(c->stream));
  c->factored = true;  // bring-up: maps supplied by the caller
  return 0;
}

int hs_set_async(hs_ctx* c, int a) {
  if (!c) return 1;
  DEV_SCOPE(c);
  c->async_mode = a ? 1 : 0;
  return 0;
}

int hs_sync(hs_ctx* c) {
  if (!c) return 1;
  DEV_SCOPE(c);
  NEED_GPU(c);
  CK(cudaStreamSynchronize(c->stream));
  return 0;
}

int hs_stream(hs_ctx* c, uint64_t* s) {
  if (!c) return 1;
  NEED_GPU(c);
  *s = (uint64_t)(uintptr_t)c->stream;
  return 0;
}

int hs_set_fused(hs_ctx* c, int mask) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (mask < 0 || mask > 15) return fail(c, 1, "fused mask must be 0..15");
  if ((mask ^ c->fused_mode) & 4) {  // plan kind changed: rebuild the fused plans
    free_fused(c);
    free_emu(c);
    free_peer_plans(c);
  }
  c->fused_mode = mask;
  return 0;
}

int hs_set_trace(hs_ctx* c, int on) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (c->device < 0) return fail(c, 1, "plan-only context");
  c->trace_on = on != 0;
  if (c->trace_on && !c->trace) {
    size_t rows = 0;  // every strip of every map, up to 16 times (phases / RHS chunks / split-K ranks)
    for (const SubPlan& sp : c->plan.subs) rows += 16 * (size_t)((sp.k * c->n + kRowTile - 1) / kRowTile);
    CK(dalloc(c, (void**)&c->trace, rows * 6 * sizeof(unsigned long long)));
    c->trace_cap = rows;
  }
  c->trace_rows = 0;
  return 0;
}

int hs_get_trace(hs_ctx* c, uint64_t* out, int cap, int* rows) {
  if (!c || !rows) return fail(c, 1, "null argument");
  DEV_SCOPE(c);
  *rows = c->trace_rows;
  if (!out || c->trace_rows == 0) return 0;
  if (cap < c->trace_rows) return fail(c, 1, "trace buffer too small");
  CK(cudaStreamSynchronize(c->stream));
  CK(cudaMemcpy(out, c->trace, (size_t)c->trace_rows * 6 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  return 0;
}

// The reduction area at the tail of a rank's exported region (256-aligned).
static size_t peer_red_offset(const Ctx* c) {
  const size_t L = (size_t)c->plan.L;
  const size_t head = FV_N * L * sizeof(double2) + (size_t)(2 * c->plan.npairs + 2) * sizeof(int);
  return (head + 255) / 256 * 256;
}

int hs_peer_export(hs_ctx* c, uint8_t handle[64]) {
  if (!c || !handle) return fail(c, 1, "null argument");
  DEV_SCOPE(c);
  NEED_GPU(c);
  PeerRanks& p = c->peer;
  const size_t L = (size_t)c->plan.L;
  // FV_N vectors, npairs completion counters, the ticket, the inputs-posted
  // epoch flag, npairs wout-write counters
  const size_t need = peer_red_offset(c) + kPeerRedBytes;
  if (!p.own || p.bytes != need) {
    dfree(c, p.own, 0);
    p.own = nullptr;
    CK(dalloc(c, &p.own, need));
    CK(cudaMemset(p.own, 0, need));
    p.bytes = need;
  }
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, p.own));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle, &h, 64);
  return 0;
}

int hs_peer_open(hs_ctx* c, const uint8_t* handles, int nranks) {
  if (!c || !handles) return fail(c, 1, "null argument");
  DEV_SCOPE(c);
  NEED_GPU(c);
  PeerRanks& p = c->peer;
  if (nranks != c->plan.nranks) return fail(c, 1, "peer handles: nranks differs from the context's");
  if (nranks > kMaxRanks) return fail(c, 1, "peer ranks: at most 8");
  if (!p.own) return fail(c, 1, "hs_peer_export first");
  if (p.G > 0) return fail(c, 1, "peer ranks already open");
  if (nranks > 1 && !c->nccl) return fail(c, 1, "peer ranks need hs_comm_init (barriers)");
  const size_t L = (size_t)c->plan.L;
  for (int g = 0; g < nranks; ++g) {
    char* base;
    if (g == c->plan.rank) {
      base = (char*)p.own;
    } else {
      cudaIpcMemHandle_t h;
      memcpy(&h, handles + 64 * g, 64);
      void* q = nullptr;
      cudaError_t e = cudaIpcOpenMemHandle(&q, h, cudaIpcMemLazyEnablePeerAccess);
      if (e != cudaSuccess) {
        for (int k = 0; k < g; ++k)
          if (p.opened[k]) cudaIpcCloseMemHandle(p.opened[k]);
        for (int k = 0; k < kMaxRanks; ++k) p.opened[k] = nullptr;
        return fail(c, -1, std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e));
      }
      p.opened[g] = q;
      base = (char*)q;
    }
    p.vec[g] = (double2*)base;
    p.counters[g] = (int*)(base + FV_N * L * sizeof(double2));
    p.inflag[g] = p.counters[g] + c->plan.npairs + 1;
    p.wdone[g] = p.inflag[g] + 1;
    char* red = base + peer_red_offset(c);
    p.red_data[g] = (double*)red;
    p.red_flag[g] = (unsigned*)(red + 2 * kPeerRedCap * sizeof(double));
    p.red_consumed[g] = p.red_flag[g] + 2;
  }
  p.red_epoch = 0;
  p.red_on = !(getenv("HS_PEER_ALLREDUCE") && atoi(getenv("HS_PEER_ALLREDUCE")) == 0);
  std::vector<int> br(c->plan.npairs), own;
  for (int b = 0; b < c->plan.npairs; ++b) {
    br[b] = c->plan.subs[c->plan.block_sub[b]].rank;
    if (br[b] == c->plan.rank) own.push_back(b);
  }
  if (upload(c, &p.blk_rank, br)) return -1;
  if (upload(c, &p.own_blocks, own)) return -1;
  p.n_own = (int)own.size();
  p.epoch = 0;
  p.epochs = !(getenv("HS_PEER_BARRIERS") && atoi(getenv("HS_PEER_BARRIERS")) != 0);
  CK(dalloc(c, (void**)&p.bar, sizeof(double2)));
  CK(cudaMemset(p.bar, 0, sizeof(double2)));
  p.G = nranks;
  return 0;
}

int hs_map_once_plan(const hs_ctx* cc, int which, int32_t* out, int cap, int* count) {
  if (!cc) return 1;
  hs_ctx* c = const_cast<hs_ctx*>(cc);
  if (!count) return fail(c, 1, "null argument");
  if (which < 0 || which > 4) return fail(c, 1, "which must be 0..4");
  StepTable rs, up, late;
  std::vector<int> zero, rfill;
  map_once_tables(c->plan, c->n, rs, up, late, zero, rfill);
  std::vector<int32_t> v;
  if (which <= 2) {
    for (const Item& it : (which == 0 ? rs : which == 1 ? up : late).items) {
      const SubPlan& sp = c->plan.subs[it.s];
      v.insert(v.end(), {sp.i1, sp.i2, it.rlo, it.rhi});
    }
  } else {
    v.assign((which == 3 ? zero : rfill).begin(), (which == 3 ? zero : rfill).end());
  }
  *count = (int)v.size();
  if (!out) return 0;
  if (cap < (int)v.size()) return fail(c, 1, "buffer too small");
  std::copy(v.begin(), v.end(), out);
  return 0;
}

int hs_fused_plan(const hs_ctx* cc, int ims, int rank, int32_t* out, int cap, int* count) {
  if (!cc) return 1;
  hs_ctx* c = const_cast<hs_ctx*>(cc);
  if (!count) return fail(c, 1, "null argument");
  if (rank < 0 || rank >= c->plan.nranks) return fail(c, 1, "rank out of range");
  DevFused f;
  FusedHost H;
  if (int e = peer_plan_host(c, ims != 0, rank, f, H)) return e;
  std::vector<int32_t> v;
  for (const FusedTile& t : H.tiles) {
    const DevItem& it = H.items[t.item];
    const SubPlan& sp = c->plan.subs[it.s];
    const int32_t rec[12] = {sp.i1, sp.i2, it.rlo, it.rhi, it.c0, it.c1, it.alt, t.tile * kRowTile * f.rt,
                             t.phase, t.flags, t.rmask, t.ndep};
    v.insert(v.end(), rec, rec + 12);
    for (int d = 0; d < t.ndep; ++d) {
      v.push_back(H.deps[t.dep0 + d].block);
      v.push_back(H.deps[t.dep0 + d].count);
    }
  }
  *count = (int)v.size();
  if (!out) return 0;
  if (cap < (int)v.size()) return fail(c, 1, "plan buffer too small");
  std::copy(v.begin(), v.end(), out);
  return 0;
}

int hs_debug_check(hs_ctx* c, uint64_t* first, int* enabled) {
  if (!c || !first) return fail(c, 1, "null argument");
  DEV_SCOPE(c);
#ifdef HS_DEVICE_CHECKS
  if (enabled) *enabled = 1;
#else
  if (enabled) *enabled = 0;
#endif
  *first = 0;
  if (c->device < 0) return 0;
  CK(cudaStreamSynchronize(c->stream));
  unsigned long long (*take[4])() = {hs_dbg_take_apply, hs_dbg_take_zmma, hs_dbg_take_krylov, hs_dbg_take_schur};
  for (int u = 0; u < 4; ++u) {
    const unsigned long long v = take[u]();
    if (v && !*first) *first = (v & ((1ull << 48) - 1)) | ((unsigned long long)(u + 1) << 48);
  }
  return 0;
}

int hs_debug_selftest(hs_ctx* c) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  NEED_GPU(c);
  CK(launch_dbg_selftest(*c));
  return 0;
}

int hs_test_peer_allreduce(hs_ctx* c, int G, int count, int repeats, const double* in, double* out) {
  if (!c || !in || !out) return fail(c, 1, "null argument");
  DEV_SCOPE(c);
  NEED_GPU(c);
  if (G < 1 || G > kMaxRanks || count < 1 || count > kPeerRedCap || repeats < 1)
    return fail(c, 1, "peer all-reduce test: 1 <= G <= 8, 1 <= count <= 4096, repeats >= 1");
  // G emulated ranks' areas (zeroed: flags and counters start at epoch 0) and
  // per-epoch buffers, every reduction launched back to back on the stream
  const size_t area = kPeerRedBytes, nbuf = (size_t)repeats * G * count;
  char* d = nullptr;
  double* bufs = nullptr;
  cudaError_t ea = cudaMalloc((void**)&d, area * G);
  if (ea == cudaSuccess) ea = cudaMalloc((void**)&bufs, nbuf * sizeof(double));
  if (ea == cudaSuccess) ea = cudaMemsetAsync(d, 0, area * G, c->stream);
  if (ea == cudaSuccess) ea = cudaMemcpyAsync(bufs, in, nbuf * sizeof(double), cudaMemcpyHostToDevice, c->stream);
  if (ea != cudaSuccess) {
    if (d) cudaFree(d);
    if (bufs) cudaFree(bufs);
    CK(ea);
  }
  PeerRedArgs a;
  a.G = G;
  a.self = -1;
  a.count = count;
  for (int g = 0; g < G; ++g) {
    char* red = d + area * g;
    a.data[g] = (double*)red;
    a.flag[g] = (unsigned*)(red + 2 * kPeerRedCap * sizeof(double));
    a.consumed[g] = a.flag[g] + 2;
  }
  // one launch, every CTA running all the reductions: a fast rank races into
  // the next epoch while others still read this one (the parity / consumed
  // protocol is what keeps it correct)
  a.epoch = 1;
  a.repeats = repeats;
  a.stride = (long long)G * count;
  for (int g = 0; g < G; ++g) a.buf[g] = bufs + (size_t)g * count;
  cudaError_t e = launch_peer_allreduce(*c, a);
  if (e == cudaSuccess) e = cudaMemcpyAsync(out, bufs, nbuf * sizeof(double), cudaMemcpyDeviceToHost, c->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(c->stream);
  cudaFree(d);
  cudaFree(bufs);
  CK(e);
  return 0;
}

int hs_set_emulated_ranks(hs_ctx* c, int ranks) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (ranks < 1 || ranks > kMaxRanks || ranks > c->n2)
    return fail(c, 1, "emulated ranks must be in 1..min(8, N2)");
  if (c->plan.nranks != 1) return fail(c, 1, "emulated ranks need a single-rank context");
  free_emu(c);
  c->emu.G = ranks;
  return 0;
}

int hs_set_gmres_mode(hs_ctx* c, int mode) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (mode < 0 || mode > 5)
    return fail(c, 1, "gmres mode must be 0 (auto), 1 (host-driven MGS), 2 (grid-wide MGS), 3 (CGS2), 4 (CGS2, Gram-corrected, one reduction) or 5 (MGS kernels by size)");
  c->gmres_mode = mode;
  return 0;
}

int hs_set_map_mode(hs_ctx* c, int mode) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  if (mode < 0 || mode > 2)
    return fail(c, 1, "map mode must be 0 (per subdomain), 1 (shared class maps, DMMA) or 2 (per kind, aliased)");
  if (mode != c->map_mode) {
    c->map_mode = mode;
    c->factored = false;  // maps must be (re)built in the new layout
    c->steps_dirty = true;
  }
  return 0;
}

int hs_set_kernel_timing(hs_ctx* c, int on) {
  if (!c) return 1;
  DEV_SCOPE(c);
  c->timing = on != 0;
  return 0;
}

int hs_kernel_stats(hs_ctx* c, int64_t* launches, double* ms, double* bytes, double* flops, int reset) {
  if (!c) return 1;
  DEV_SCOPE(c);
  NEED_GPU(c);
  CK(cudaStreamSynchronize(c->stream));
  for (size_t i = 0; i < c->ev_pending.size(); ++i) {
    float t = 0;
    cudaEventElapsedTime(&t, c->ev_pending[i].first, c->ev_pending[i].second);
    c->k_ms += t;
    c->k_bytes += c->ev_bytes[i];
    c->k_flops += c->ev_flops[i];
    c->k_launches++;
    c->ev_pool.push_back(c->ev_pending[i].first);
    c->ev_pool.push_back(c->ev_pending[i].second);
  }
  c->ev_pending.clear();
  c->ev_bytes.clear();
  c->ev_flops.clear();
  if (launches) *launches = c->k_launches;
  if (ms) *ms = c->k_ms;
  if (bytes) *bytes = c->k_bytes;
  if (flops) *flops = c->k_flops;
  if (reset) { c->k_launches = 0; c->k_ms = 0; c->k_bytes = 0; c->k_flops = 0; }
  return 0;
}

int hs_launch_count(const hs_ctx* c, int64_t* n) {
  if (!c) return 1;
  *n = c->launches;
  return 0;
}

int hs_memory(const hs_ctx* c, int64_t* bytes) {
  if (!c) return 1;
  *bytes = c->dev_bytes;
  return 0;
}

int hs_nccl_unique_id(uint8_t id[128]) {
  Ctx* c = nullptr;
  ncclUniqueId u;
  NK(ncclGetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId size");
  std::memcpy(id, &u, 128);
  return 0;
}

int hs_comm_init(hs_ctx* c, const uint8_t id[128]) {
  if (!c) return fail(nullptr, 1, "null context");
  DEV_SCOPE(c);
  NEED_GPU(c);
  CK(cudaSetDevice(c->device));
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclComm_t comm;
  NK(ncclCommInitRank(&comm, c->plan.nranks, u, c->plan.rank));
  c->nccl = comm;
  return 0;
}

}  // extern "C"
