// Context of one GPU (or plan-only) instance and the device data structures
// shared by the kernels.  See include/hsb200.h for the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <map>
#include <string>
#include <vector>

#include "hs_plan.h"

namespace hs {

constexpr int kRowTile = 32;
constexpr int kZ2TicketSlots = 64;  // k_zmma2 persistent launches' ticket counters (a ring)  // rows per tile of the tile-major map layout
// Every 1-RHS step kernel (k_step1, k_bsp_fused, k_bsp_tma) splits a row's map
// columns the same way -- column c into partial sum (c % 32) / (32 / kSumWarps),
// accumulator c & 1, partials added in order -- so their results are bitwise
// identical.
constexpr int kSumWarps = 8;

// Per-subdomain record on the device.  Maps are stored tile-major:
// T_s[tile][col][lane] = T_s(tile*32 + lane, col), rows padded to a multiple of
// 32 with zeros, so a 32-row strip of a map is one contiguous K*512-byte run.
struct DevSub {
  long long T_off;  // element offset of the map
  int in_off;       // element offset of the incoming slab m(s, .) (block * n)
  int k;            // interface faces; K = k * n columns
  int nlow;         // leading W/S faces (map rows [0, nlow * n) feed the lower neighbours)
  int tgt[4];       // element offset (block * n) of the block written by each face
};

struct DevItem {
  int s, rlo, rhi, alt;
  int slot[4];
  int c0, c1;  // map columns used by the fused kernels (the rest of the slab reads as zero)
};

struct DevTile {
  int item, tile;
};

struct DevRecv {
  int dir, slot;
  long long off;
};

// Epilogue of a step: what to do with output row values y at element t.
enum EpiMode {
  EPI_SET = 0,    // o1[t] = y
  EPI_ACC = 1,    // o1[t] += y                       (sweep step, one state)
  EPI_IMS = 2,    // o1[t] = a[t] - y                 ((I - S) g)
  EPI_RESID = 3,  // v = a[t] - b[t] + y; o1 = v; o2 = v; o3 = b[t] + v   (BSP residual)
  EPI_ACC2 = 4,   // o1[t] += y; o2[t] += y           (BSP backward step)
  EPI_LATE = 5,   // o1[t] = (a[t] - b[t]) + (c[t] - y)  ((I - S) z on a backward window start's rows)
};

struct Epi {
  int mode;
  double2* o1;
  double2* o2;
  double2* o3;
  const double2* a;
  const double2* b;
  const double2* c;
  double2* send_up;
  double2* send_dn;
};

// DMMA contraction tasks (hs_zmma.cu): 32 map rows x up to 32 columns each.
struct MmaTask {
  long long a_off;  // element offset of the 32-row strip holding rows r0..r0+31
  int K;            // map columns
  int r0, rlo, rhi; // strip start; valid output rows [rlo, rhi)
  int col0, ncols;  // column descriptors [col0, col0 + ncols)
};

// One B column / output column: per face (map row block q), the element
// offset of position 0 in the input and output vectors (-1: face absent ->
// zero input, dropped output); consecutive positions are R apart.
struct MmaCol {
  long long in[4];
  long long out[4];
  int slot[4];
  int r;    // right-hand side index (exchange buffer layout)
  int alt;  // read srcB (the half's input) instead of srcA
};

struct DevMma {
  MmaTask* tasks = nullptr;
  MmaCol* cols = nullptr;
  int ntasks = 0, ncols = 0;
  int minK = 0;  // smallest K of the tasks (split-K decision)
  double flops = 0;
  int bn = 32;      // columns per task
  int kind = 0;     // 0: k_zmma (cp.async); 1: k_zmma2 k-major slab rows; 2: k_zmma2 n-major columns
};

// A step uploaded to the device: items + tiles + receive list.
struct DevStep {
  StepTable host;                 // kept to build contraction tasks lazily
  std::map<int, DevMma> mma;      // key: R (per-subdomain maps) or -R (shared maps)
  DevItem* items = nullptr;
  DevTile* tiles = nullptr;
  DevRecv* recv = nullptr;
  int nitems = 0, ntiles = 0, nrecv = 0;
  int nsend_up = 0, nsend_dn = 0, nrecv_up = 0, nrecv_dn = 0;
  int maxK = 0;
  double bytes_per_rhs_map = 0, bytes_per_rhs_vec = 0;  // algorithmic bytes: map part, per-RHS vector part
};

// Fused BSP apply (one persistent dataflow launch): a tile of some step, with
// the per-block completion counts it must wait for.
// Phases (what a tile multiplies and how its rows are finished; FT_* flags):
//   0 forward         y1 = T (r | zL):   zL += y1            [FT_ZERO: rp = w = 0, z = zL]
//   1 residual        y1 = T zL:         v = r - (zL - y1); rp = w = v; z = zL + v
//   2 backward        y1 = T (rp | w):   w += y1, z += y1    [FT_WOUT: wout = r; upper rows wout = r - y1]
//   3 (I - S) z       y1 = T z:          wout = z - y1
//   4 residual+bwd    y1 = T zL, y2 = T (rp | w): v = r - (zL - y1); rp = v; w = v + y2; z = (zL + v) + y2
//                                        [FT_WOUT: wout = r; upper rows wout = r - y2]
//   5 (I - S) late    y1 = T w (final):  lower rows wout = (r - rp) + (w - y1); upper rows wout = r - y1
// FT_DIFF (map-once, on a column range of the item): phase 1 multiplies
// zL - r and finishes with v = y1; phase 5 multiplies w - rp and finishes
// with wout = r - y1.
// Phases 0-3 in step order are the per-step arithmetic (bitwise); 0-2 + 4 + 5
// are the map-once plan of build_fused (each map row read ~once per apply).
enum FusedFlags { FT_ZERO = 1, FT_WOUT = 2, FT_DIFF = 4 };
struct FusedTile {
  int item;        // index into the fused item list
  int tile;        // tile index in units of rt strips
  int phase;       // see above
  int flags;       // FT_*
  int dep0, ndep;  // dependencies [dep0, dep0 + ndep) in the dep pool
  int rmask;       // bit q: slab face q of zL not yet written (read r); bit 4 + f: output face f likewise
  int c0, c1;      // map columns this tile streams (the item's range, or one half of it when split)
  int ks, pair;    // split-K: half 0 / 1 of pair `pair` (ks = -1: not split)
};

struct FusedDep {
  int block, count;  // wait until done[block] >= count
};

struct DevFused {
  DevItem* items = nullptr;
  FusedTile* tiles = nullptr;
  FusedDep* deps = nullptr;
  int nitems = 0, ntiles = 0, ndeps = 0, maxK = 0;
  std::vector<int> wtot;    // block -> completion signals per apply (all ranks' tiles)
  std::vector<int> wwtot;   // block -> wout-writing tile faces per apply (all ranks' tiles)
  int nv = 1;               // vectors per tile (2: the map-once plan's phase-4 tiles)
  bool map_once = false;    // map-once plan (else per-step order, bitwise = k_step1)
  int rt = 1;               // 32-row strips per tile
  int nw = 8;               // warps per CTA (consumer warps for the TMA kernel)
  bool tma = true;          // TMA-staged maps (k_bsp_tma), else register streaming (k_bsp_fused)
  int stages = 5;           // TMA ring depth: 5 (two CTAs per SM) or 12 (one CTA per SM)
  int direct_signal = 0;    // TMA kernel: consumers signal completions themselves (no signaller hop)
  int npairs_split = 0;     // split-K tile pairs (their partial sums meet in `split_buf`)
  double2* split_buf = nullptr;  // [pair][half][32 rows][2 vectors]
  int* split_cnt = nullptr;      // [pair] arrivals (never reset: the odd arrival combines)
  int* counters = nullptr;  // [npairs] block completion counters + [1] ticket
  double bytes = 0;         // algorithmic bytes of one apply
  bool built = false;
};

// Fused BSP apply on the DMMA contraction (R right-hand sides or shared maps).
struct FusedMmaTask {
  MmaTask task;
  int phase;       // 0 forward, 1 residual, 2 backward, 3 fill (rp = w = 0, z = zL on the counters' elements)
  int dep0, ndep;  // waits: counters[block * nchunk + chunk] >= count
  int inc0, ninc;  // counters this task completes
  int ks = -1;     // k_zmma2_df split-K: half 0 / 1 of pair `pair` (-1: whole K)
  int pair = -1;
};

struct DevFusedMma {
  FusedMmaTask* tasks = nullptr;
  MmaCol* cols = nullptr;
  FusedDep* deps = nullptr;
  int* incs = nullptr;
  int ntasks = 0, ncols = 0, ndeps = 0, nincs = 0;
  int ncounters = 0;        // npairs * ceil(R / 32)
  int* counters = nullptr;  // + 1 ticket
  int minK = 0;             // smallest task K (split-K decision)
  double flops = 0;
  int R = 0;
  int cw = 32;  // task / completion-counter width in right-hand sides (k_zmma2_df: 16 or 32)
  bool shared = false, built = false;
  int npairs_split = 0;          // split-K pairs (k_zmma2_df)
  double2* split_buf = nullptr;  // [pair][half][32 x 32] partial tiles
  int* split_cnt = nullptr;      // [pair] arrivals (never reset: the odd arrival combines)
};

struct FusedMmaArgs {
  const FusedMmaTask* tasks;
  const MmaCol* cols;
  const FusedDep* deps;
  const int* incs;
  const double2* A;
  const double2* r;
  double2* zL;
  double2* rp;
  double2* w;
  double2* z;
  int* done;
  int* ticket;
  int ntasks, n, R;
  unsigned long long* trace = nullptr;  // k_zmma2_df, per ticket: claimed, inputs met, first chunk, contracted, signalled, info
  double2* split_buf = nullptr;
  int* split_cnt = nullptr;
  const double2* zeros = nullptr;  // n-major form: the rows of absent faces and padding columns
  long long LR = 0;                // vector elements (bounds checks)
  // k_zmma2_df, k-major slabs: the vectors zL, r, w, rp as [L][2 R] FP64 tensors,
  // box (BN + 2 columns) x (32 positions): a chunk's slab rows in ONE tensor copy
  int use_tm = 0;
  alignas(64) CUtensorMap tm[4];
};

// Row-band ranks of the fused apply (multi-rank kernel instantiations): every
// block -- its vectors and its completion counter -- lives on its owner rank.
constexpr int kMaxRanks = 8;
enum FusedVec { FV_R = 0, FV_ZL, FV_RP, FV_W, FV_Z, FV_WOUT, FV_N };
struct MultiRankArgs {
  int G = 1, self = 0;                 // ranks; self >= 0: this GPU's rank, < 0: CTA c emulates rank c % G
  const int* blk_rank = nullptr;       // block -> owner rank
  double2* v[FV_N][kMaxRanks] = {};    // per rank: r, zL, rp, w, z, wout
  int* done[kMaxRanks] = {};
  int* ticket[kMaxRanks] = {};
  const FusedTile* tiles[kMaxRanks] = {};
  int ntiles[kMaxRanks] = {};
  // Epoch protocol (separate GPUs, epoch > 0): counters are never reset -- a
  // dependency (block, count) of apply `epoch` waits for count + (epoch - 1) *
  // wtot[block]; the consumers first wait until every rank has posted its
  // inputs for this epoch (inflag[g] >= epoch: its previous apply is over and
  // its r is in place), and before exiting drain this rank's own blocks
  // (counter == epoch * wtot): no barrier of any kind between applies.
  unsigned epoch = 0;
  const int* wtot = nullptr;           // block -> completion signals per apply
  const int* inflag[kMaxRanks] = {};   // per rank: last epoch whose inputs are posted
  const int* own_blocks = nullptr;     // this rank's blocks (drain)
  int n_own = 0;
  // wout (GMRES's (I - S) z) is written by tiles that signal nothing on done:
  // they count in wdone, drained to ims_epoch * wwtot for the A M v applies
  int* wdone[kMaxRanks] = {};
  const int* wwtot = nullptr;
  unsigned ims_epoch = 0;
};

// Emulated row bands on one GPU (hs_set_emulated_ranks): per-rank vectors,
// counters and tile lists of the fused plan, for testing the multi-rank
// kernels against the single-rank result.
struct EmuRanks {
  int G = 1;
  bool built = false;
  std::vector<int> sub_rank;             // subdomain -> rank
  int* blk_rank = nullptr;               // device: block -> rank
  FusedTile* tiles[kMaxRanks] = {};      // device: per-rank tile lists (plan order)
  int ntiles[kMaxRanks] = {};
  double2* buf = nullptr;                // device: G x (r, zL, rp, w, z) full-length vectors
  int* counters = nullptr;               // device: G x (npairs done + 1 ticket)
};

// Row-band ranks on separate GPUs running the fused apply over each other's
// buffers (hs_peer_export / hs_peer_open): every rank exports one region --
// FV_N full-length vectors + the completion counters of its blocks + a ticket
// -- through CUDA IPC and maps its peers' regions, so a tile writes its output
// blocks and signals their counters directly in the owner's HBM over NVLink.
struct PeerRanks {
  int G = 0;                          // 0: off
  void* own = nullptr;                // this rank's region (cudaMalloc, IPC-exported)
  size_t bytes = 0;
  double2* vec[kMaxRanks] = {};       // per rank: FV_N x L vectors
  int* counters[kMaxRanks] = {};      // per rank: npairs counters + 1 ticket
  void* opened[kMaxRanks] = {};       // IPC mappings (closed at destroy)
  int* inflag[kMaxRanks] = {};        // per rank: epoch whose inputs are posted (region tail)
  int* wdone[kMaxRanks] = {};         // per rank: wout-write counters of its blocks (region tail)
  int* wwtot = nullptr;               // block -> wout writes per A M v apply
  unsigned ims_epoch = 0;             // A M v applies run so far
  DevFused plan, plan_ims;            // global plans; tiles = this rank's only
  int* blk_rank = nullptr;            // block -> owner rank
  int* wtot = nullptr;                // block -> completion signals per apply (same for both plans)
  int* own_blocks = nullptr;          // this rank's blocks
  int n_own = 0;
  unsigned epoch = 0;                 // applies run so far (epoch protocol)
  bool epochs = true;                 // false: two NCCL barriers per apply (HS_PEER_BARRIERS=1)
  double2* bar = nullptr;             // one-element NCCL barrier buffer
  // GMRES inner-product all-reduce over the same mappings (region tail):
  // per rank [2 parities][kPeerRedCap] partials, 2 published-epoch flags and a
  // consumed-epoch counter; one kernel per reduction, no NCCL call
  double* red_data[kMaxRanks] = {};
  unsigned* red_flag[kMaxRanks] = {};
  unsigned* red_consumed[kMaxRanks] = {};
  unsigned red_epoch = 0;
  bool red_on = true;                 // HS_PEER_ALLREDUCE=0: NCCL all-reduce instead
};

constexpr int kPeerRedCap = 4096;     // doubles per parity (CGS2: 2 (k + 2) <= 4096)
// bytes of the reduction area at the tail of a rank's exported region
constexpr size_t kPeerRedBytes = 2 * kPeerRedCap * sizeof(double) + 64;

// The peer all-reduce (hs_krylov.cu): G ranks, every rank publishes its count
// partials in its own area and sums all ranks' in rank order (bitwise the
// same result on every rank).  self >= 0: this GPU's rank (one CTA); self < 0:
// CTA r emulates rank r on one GPU (buf[r] per rank, tests).
struct PeerRedArgs {
  int G = 1, self = 0, count = 0;
  unsigned epoch = 0;         // of the first reduction
  int repeats = 1;            // reductions in this launch (tests: ranks race across epochs)
  long long stride = 0;       // buffer offset between consecutive reductions
  double* data[kMaxRanks] = {};
  unsigned* flag[kMaxRanks] = {};
  unsigned* consumed[kMaxRanks] = {};
  double* buf[kMaxRanks] = {};
};

// One distinct subdomain operator (Dirichlet mask) and its factor.
struct OpClass {
  std::vector<uint8_t> mask;          // n*n, 1 = Dirichlet cell
  std::vector<int32_t> dcells;        // sorted Dirichlet cells
  double2* X = nullptr;               // n x (n x n) inverses of the block-LU pivots
  double2* T4 = nullptr;              // full 4n x 4n map (row-major)
  bool factored = false;
};

struct Workspace {
  double2* p = nullptr;
  size_t cap = 0;  // elements
};

struct Ctx {
  int device = -1;
  int n1 = 0, n2 = 0, n = 0;
  double h = 0, kappa = 0, tau_re = 0, tau_im = 0;
  Plan plan;
  std::string err;
  // per-subdomain Dirichlet cells (host) and classes
  std::map<int, std::vector<int32_t>> dcells;  // ordinal -> cells
  std::vector<OpClass> classes;
  std::vector<int> sub_class;
  bool factored = false;
  int map_mode = 0;               // 0: per-subdomain maps (HBM path), 1: shared class maps
  double2* Tcls = nullptr;        // class maps, strip-major, padded rows
  std::vector<long long> Tcls_off;
  size_t Tcls_elems = 0;
  // device state
  cudaStream_t stream = nullptr;
  cudaStream_t copy_in = nullptr, copy_out = nullptr;  // host-batch pipeline (hs_precond_batch)
  cudaStream_t aux = nullptr;                           // side work overlapping a step (map-once fills)
  cudaEvent_t aux_fork = nullptr, aux_join = nullptr;
  cudaEvent_t bev[6] = {};                              // per slot: input landed, applied, output drained
  double2* T = nullptr;
  size_t T_elems = 0;
  DevSub* dsubs = nullptr;
  // windows / precond options
  int seam = 0, inter = 1;
  bool steps_dirty = true;
  std::vector<DevStep> fwd, bwd, sp_fwd, sp_bwd;
  DevStep full;
  // map-once form of the per-step BSP (and of GMRES's A M v): the residual
  // step on the rows where r' can be nonzero, the upper rows of (I - S) z on
  // the final backward state, the window starts' late rows, and the blocks
  // filled without a map read (device lists of own blocks)
  DevStep mo_resid, mo_ims_up, mo_ims_late;
  int* mo_zero_blocks = nullptr;  int n_mo_zero = 0;   // rp = w = 0, z = zL
  std::vector<int> mo_zero_host;                      // the same blocks (dataflow plans)
  int* mo_r_blocks = nullptr;     int n_mo_r = 0;      // (I - S) z = r
  DevFused fused;        // BSP apply as one dataflow launch (1 RHS, per-subdomain maps, 1 rank)
  DevFused fused_ims;    // the same followed by (I - S) z: GMRES's A M v in one launch
  EmuRanks emu;          // emulated row-band ranks for the fused apply (tests)
  PeerRanks peer;        // row-band ranks on separate GPUs (fused apply over CUDA IPC)
  DevFusedMma fused_mma; // the same on the DMMA contraction (R RHS or shared maps)
  int fused_mode = 3;    // bit 0: 1-RHS dataflow apply, bit 1: R-RHS DMMA dataflow apply (hs_set_fused)
  std::vector<std::vector<int>> seam_blocks;  // [dir] blocks of seam groups (literal mode)
  int* d_seam[2] = {nullptr, nullptr};
  int n_seam[2] = {0, 0};
  // vectors (grown on demand): named work buffers
  std::map<std::string, Workspace> ws;
  // exchange buffers
  double2* send_up = nullptr; double2* send_dn = nullptr;
  double2* recv_up = nullptr; double2* recv_dn = nullptr;
  size_t xbuf_cap = 0;
  void* nccl = nullptr;  // ncclComm_t
  int gm_basis = 0;      // basis vectors built by the last hs_gmres (hs_gmres_basis)
  long long gm_LR = 0;   // their length
  int gmres_mode = 0;    // 0 auto (cooperative MGS on one rank), 1 host-driven MGS over owned blocks
  int* h_flags = nullptr;             // pinned: GMRES active counts (2 slots)
  cudaEvent_t flag_ev[2] = {nullptr, nullptr};
  double* mgs1_slots = nullptr;  // k_mgs1 partial sums [2][3][256] + grid barrier counter
  unsigned mgs1_bar = 0;         // barrier counter value after the last k_mgs1 launch
  int* d_owned = nullptr;  // this rank's blocks (host-driven MGS)
  int n_owned = 0;
  // execution control / timing
  int async_mode = 0;
  bool timing = false;
  // per-ticket timeline of the fused 1-RHS apply (hs_set_trace; diagnostics)
  bool trace_on = false;
  unsigned long long* trace = nullptr;
  size_t trace_cap = 0;   // rows of 5 words
  int trace_rows = 0;     // rows of the last traced launch
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending;
  std::vector<double> ev_bytes, ev_flops;
  std::vector<cudaEvent_t> ev_pool;
  int64_t k_launches = 0;
  int64_t launches = 0;  // every kernel this context launched
  double k_ms = 0, k_bytes = 0, k_flops = 0;
  int64_t dev_bytes = 0;
  std::map<void*, size_t> alloc_sz;  // live device allocations
  int num_sms = 148;
  int coop_ok = 0;
  double2* zeros = nullptr;  // 64 zero elements: the source of absent faces in bulk-copied operands
  unsigned* z2_tickets = nullptr;        // k_zmma2 persistent launches: a ring of ticket counters
  unsigned z2_base[64] = {};             // per slot: claims so far (the next launch's first ticket)
  unsigned long long z2_seq = 0;
};

}  // namespace hs
