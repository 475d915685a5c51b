/*
 * hsb200.h -- C ABI of the B200 hot path of the block Jacobi sweeping
 * preconditioner (arXiv 2209.10886) for the 2D Helmholtz interface problem
 * (I - S) g = b on an N1 x N2 checkerboard.
 *
 * The reference (`helmsweep`, pure Python over SciPy's SuperLU) has no FFI of
 * its own; its only language boundary is Python -> SuperLU's C code.  Each
 * entry point below replaces one reference interface (file:line relative to
 * /root/reference/pkg/src/helmsweep/ unless it names SPEC.md):
 *
 *   hs_create / hs_set_dirichlet / hs_factor
 *       InterfaceSystem.__init__            interface_system.py:73-89
 *       LocalOperator.__init__ + splu       discretization.py:126-174
 *   hs_lifting_rhs
 *       compute_liftings + assemble_rhs     interface_system.py:98-113
 *       solve_lifting                       discretization.py:315-332
 *   hs_apply (HS_APPLY_S / HS_APPLY_IMS)
 *       apply_scattering                    interface_system.py:135-142
 *       apply_interface_operator            interface_system.py:144-146
 *   hs_restricted_apply
 *       restricted_apply                    interface_system.py:148-162
 *   hs_set_windows / hs_precond / hs_half_apply
 *       forward_sweep, backward_sweep, sgs_apply, bj_half_apply, bsp_apply
 *                                           SPEC.md:306-348 (not shipped)
 *   hs_gmres
 *       gmres(apply_A, apply_M, b, opts)    SPEC.md:399-407 (not shipped)
 *   hs_get_schur
 *       the per-subdomain map solve_local + extract_outgoing_trace
 *                                           discretization.py:264-312
 *
 * Conventions
 *   - complex128 = two doubles (re, im) interleaved, i.e. numpy complex128.
 *   - interface vectors are in the reference m-order (interface_system.py:30-62):
 *     length L = 2*N_e*n, block m (1-based) = elements [(m-1)n, mn).  With
 *     nrhs > 1 a vector is [L][nrhs] row-major (right-hand side fastest).
 *   - `mem`: HS_MEM_HOST (caller host pointer; copied in/out inside the call)
 *     or HS_MEM_DEVICE (pointer on the context's device).
 *   - multi-GPU: one context per GPU/process; rank r owns a contiguous band of
 *     subdomain rows.  Vectors passed in/out are full length on
 *     every rank; a rank reads and writes only the blocks it owns.
 *   - return value: 0 = ok, > 0 = invalid argument (Python maps it to
 *     ValueError, like the reference's ValueError paths), < 0 = CUDA / NCCL /
 *     numerical failure (RuntimeError, like discretization.py:171-174).
 *     hs_last_error() gives the message.
 *   - a context is used by one host thread at a time.
 */
#ifndef HSB200_H
#define HSB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hs_ctx hs_ctx;

enum { HS_MEM_HOST = 0, HS_MEM_DEVICE = 1 };
enum { HS_APPLY_S = 0, HS_APPLY_IMS = 1 };
enum { HS_PC_NONE = 0, HS_PC_SP = 1, HS_PC_BSP = 2 };
enum { HS_SEAM_DEDUP = 0, HS_SEAM_LITERAL = 1 };
enum { HS_DIR_FORWARD = 0, HS_DIR_BACKWARD = 1 };

/* Library version and build flags ("hsb200 <ver> sm_100a ..."). */
const char* hs_version(void);

/* Message of the last failed call on this context (or of the last failed
 * hs_create when ctx is NULL).  Valid until the next call. */
const char* hs_last_error(const hs_ctx* ctx);

/* Create a context.  device = CUDA ordinal, or -1 for a plan-only context
 * (host tables only, no CUDA calls; used by CPU tests).  tau = tau_re + i tau_im
 * is the impedance coefficient (ImpedanceSpec, discretization.py:86-102).
 * rank/nranks: row-band sharding (nranks = 1 for a single GPU). */
int hs_create(hs_ctx** ctx, int device, int n1, int n2, int n, double h, double kappa,
              double tau_re, double tau_im, int rank, int nranks);
int hs_destroy(hs_ctx* ctx);

/* Scatterer cells (identity rows, discretization.py:187-200, 247-251) of
 * subdomain (i1, i2), 1-based lattice coordinates; cells index the n x n grid
 * row-major (y slow).  Must precede hs_factor. */
int hs_set_dirichlet(hs_ctx* ctx, int i1, int i2, const int32_t* cells, int ncells);

/* Map storage, before hs_factor: 0 = one compact map per subdomain streamed
 * from HBM by the step kernels (default); 1 = shared-operator mode: only the
 * distinct operators' 4n x 4n maps are kept (the reference matrix depends
 * only on the Dirichlet cells, discretization.py:224-229) and every step is a
 * DMMA contraction with the map L2-resident (needs n % 32 == 0). */
int hs_set_map_mode(hs_ctx* ctx, int mode);

/* Build every subdomain's interface Schur map on the GPU (block-tridiagonal
 * elimination of the Dirichlet-eliminated operator, one per distinct
 * operator, then scattered into per-subdomain compact maps). */
int hs_factor(hs_ctx* ctx);

/* Right-hand side b (interface_system.py:105-113) for nrhs liftings: vals holds
 * the Dirichlet data of the scatterer cells as [ncells][nrhs] complex (the
 * reference uses -u_inc, discretization.py:326-328).  b is [L][nrhs]. */
int hs_lifting_rhs(hs_ctx* ctx, const double* vals, int nrhs, double* b, int mem);

/* Field reconstruction (the driver's reconstruct_solution):
 * u_i = v_i + w_i for every subdomain this rank owns, where v_i solves the
 * subdomain with its incoming traces from g (solve_local,
 * discretization.py:264-293) and w_i is the lifting with Dirichlet data
 * lift_vals (as for hs_lifting_rhs; NULL -> no lifting), computed with the
 * stored block factors; stitched into field, (N2 n) x (N1 n) complex, y slow
 * (cells of other ranks' subdomains are zero). */
int hs_reconstruct(hs_ctx* ctx, const double* g, const double* lift_vals, double* field, int mem);

/* out = S g (mode HS_APPLY_S) or (I - S) g (HS_APPLY_IMS). */
int hs_apply(hs_ctx* ctx, int mode, const double* g, double* out, int nrhs, int mem);

/* out = V_T S V_Src^T g: solve subdomains of the source groups, write blocks
 * owned by the target groups, zero elsewhere. */
int hs_restricted_apply(hs_ctx* ctx, const double* g, double* out, int nrhs,
                        const int32_t* src_groups, int nsrc, const int32_t* tgt_groups, int ntgt,
                        int mem);

/* Window ranges [lo, hi] (group indices, inclusive) of the partial sweeps of
 * one direction (kind 0 = lower / forward, 1 = upper / backward).  Default
 * after hs_create: the reference rule (indexing.py:158-179). */
int hs_set_windows(hs_ctx* ctx, int kind, const int32_t* lo, const int32_t* hi, int nwin);

/* Preconditioner options: seam mode and the BSP intermediate residual
 * (SweepConfig). */
int hs_set_precond_options(hs_ctx* ctx, int seam_mode, int intermediate_residual);

/* z = M r for M in {identity, SP = S_U^-1 S_L^-1, BSP}. */
int hs_precond(hs_ctx* ctx, int kind, const double* r, double* z, int nrhs, int mem);
/* hs_precond on a batch of nvec independent HOST vectors (r[i] -> z[i], each
 * L x nrhs; pinned memory for full speed), pipelined: vector i+1 is copied in
 * and vector i-1 copied out on two copy streams while vector i is applied
 * (double-buffered device slots).  Returns when every z[i] is on the host.
 * The serving form of the SPEC.md:340-348 apply. */
int hs_precond_batch(hs_ctx* ctx, int kind, const double* const* r, double* const* z, int nvec, int nrhs);

/* One block-Jacobi half (bj_half_apply) with the configured
 * windows; with one window per direction it is forward_sweep / backward_sweep. */
int hs_half_apply(hs_ctx* ctx, int direction, const double* r, double* z, int nrhs, int mem);

/* Full right-preconditioned GMRES on the device (conventions in oracle/gmres.py):
 * b, x are [L][nrhs]; iters[nrhs], converged[nrhs]; hist (may be NULL) is
 * [maxit+1][nrhs] relative residual estimates (unused tail left untouched). */
int hs_gmres(hs_ctx* ctx, int pc_kind, const double* b, double* x, int nrhs, double tol,
             int maxit, int* iters, double* hist, int* converged, int mem);

/* Arnoldi implementation: 0 = auto (single GPU, one RHS: one MGS + Givens
 * kernel per iteration with w register-resident -- on one thread-block
 * cluster up to 32k elements (k_mgs1c), grid-wide beyond (k_mgs1); several
 * RHS: the cluster kernel k_mgs_cluster up to 32k elements, else the
 * grid-wide cooperative MGS kernel k_mgs + k_givens; across row bands:
 * host-driven MGS with one ncclAllReduce per inner product), 1 = force the
 * host-driven MGS (single-GPU test of the sharded algorithm), 2 = force the
 * generic grid-wide cooperative kernel (k_mgs + k_givens),
 * 3 = CGS2 (classical Gram-Schmidt + one reorthogonalisation; one RHS): two
 * reductions per iteration instead of k+1 -- one all-reduce each across row
 * bands; same iteration counts as MGS within +-1;
 * 4 = CGS2 with the reorthogonalisation done on the coefficients through the
 * device-kept Gram matrix V^H V: ONE reduction per iteration -- what mode 0
 * runs for one RHS, on one GPU and across row bands (HS_ARNOLDI_BANDS=cgs2:
 * mode 3 across bands); 5 = the MGS kernels for one RHS too (mode 0's choice
 * for several RHS: the cluster kernel up to 32k elements, k_mgs1 beyond). */
int hs_set_gmres_mode(hs_ctx* ctx, int mode);

/* Test hook for the multi-GPU path: run the fused 1-RHS BSP
 * apply of hs_precond as `ranks` row-band ranks emulated on this GPU -- every
 * rank with its own vectors, counters and tile list, reaching the other
 * ranks' blocks through their buffers (the peer-memory protocol of the
 * multi-GPU kernel) -- in one launch.  1 = off.  Results are bitwise those of
 * the single-rank apply. */
int hs_set_emulated_ranks(hs_ctx* ctx, int ranks);

/* Bit mask.  Bit 0 (default on): a BSP apply with one RHS on per-subdomain
 * maps runs as one persistent dataflow launch (per-block completion counters
 * instead of one launch per step).  Bit 2 (default off) selects the per-step
 * plan for it -- the step sequence's arithmetic, bitwise identical to bit 0
 * clear; otherwise the map-once plan computes the same z with every map row
 * read about once per apply (the intermediate residual vanishes inside the
 * forward windows and shares the backward steps' map reads),
 * equal to the step sequence to rounding.  Bit 1 (default on): R right-hand
 * sides on the per-subdomain maps run as one dataflow launch on the DMMA
 * contraction (k_zmma2_df: the step sequence's arithmetic, list-scheduled
 * tickets); bit 3 (default off) also the shared class maps (k_zmma_fused).
 * Default mask 3. */
int hs_set_fused(hs_ctx* ctx, int mask);

/* Row-band ranks on separate GPUs (one process per GPU, nranks > 1 and
 * hs_comm_init done), or nranks = 1 on one GPU: the fused 1-RHS apply (and
 * GMRES's A M v) runs over every rank's buffers through CUDA IPC -- a tile
 * writes its output blocks and signals their completion counters directly in
 * the owner's HBM (NVLink peer stores and system-scope atomics), with no
 * per-step exchange.  hs_peer_export allocates this rank's region and writes
 * its 64-byte IPC handle; after the host has all-gathered the handles (rank
 * order), hs_peer_open maps the peers' regions and enables the path.  Between
 * applies there is no barrier: counters carry epochs, each rank posts its
 * inputs' epoch and the kernel drains its own blocks (HS_PEER_BARRIERS=1: reset
 * + two NCCL barriers per apply instead).  Replaces the per-step NCCL
 * send/recv of hs_comm_init's path for the fused apply. */
int hs_peer_export(hs_ctx* ctx, uint8_t handle[64]);
int hs_peer_open(hs_ctx* ctx, const uint8_t* handles, int nranks);
/* The fused plan a rank runs on that path (plan-only contexts too), for
 * host-side emulation of the protocol: per tile (ticket order) 12 int32 --
 * subdomain i1, i2, item rows [rlo, rhi), columns [c0, c1), alt, first row of
 * the tile's 32-row strip, phase, flags, rmask, ndep -- then ndep (block,
 * count) pairs (wait until block's completion counter >= count).  *count =
 * int32 written (out = NULL: needed). */
int hs_fused_plan(const hs_ctx* ctx, int ims, int rank, int32_t* out, int cap, int* count);
/* The map-once per-step form's tables (plan-only contexts too): which = 0
 * residual rows, 1 (I - S) z upper rows, 2 the window starts' late rows -- 4
 * int32 per item (subdomain i1, i2, rows [rlo, rhi)), every rank's items; 3 /
 * 4: this rank's blocks filled without a map read (rp = w = 0, z = z_L /
 * (I - S) z = r).  hs_exchange_plan kinds 3..5 are the same three steps. */
int hs_map_once_plan(const hs_ctx* ctx, int which, int32_t* out, int cap, int* count);

/* Diagnostics: record a per-tile timeline of the fused 1-RHS apply (on = 1).
 * hs_get_trace copies the last traced launch: rows of 6 words per ticket --
 * claimed, work started, inputs ready, map streamed, completion signalled
 * (globaltimer ns), (SM id << 32) | (CTA << 8) | phase.  out = NULL returns
 * the row count only. */
int hs_set_trace(hs_ctx* ctx, int on);
int hs_get_trace(hs_ctx* ctx, uint64_t* out, int cap, int* rows);

/* Test hook of the peer-memory all-reduce that replaces ncclAllReduce for the
 * sharded Arnoldi's inner products once hs_peer_open has mapped the ranks'
 * regions (HS_PEER_ALLREDUCE=0 keeps NCCL): G ranks emulated by G co-resident
 * CTAs on this GPU run `repeats` back-to-back reductions of `count` doubles
 * (in/out: repeats x G x count, rank-major per reduction).  Every rank's
 * result must be the rank-order sum, bitwise. */
int hs_test_peer_allreduce(hs_ctx* ctx, int G, int count, int repeats, const double* in, double* out);

/* Device-side checks (the debug library libhsb200_debug.so, built with
 * -DHS_DEVICE_CHECKS; HS_LIB=debug loads it): bounds asserts on every table,
 * map and vector access of the dataflow kernels and a watchdog on every
 * cross-CTA spin-wait.  Synchronises the context's stream and returns in
 * *first the first failure since the last call -- (unit << 48) | (source line
 * << 8) | tag, unit 1 hs_apply.cu, 2 hs_zmma.cu, 3 hs_krylov.cu, 4
 * hs_schur.cu; tag = DbgTag (hs_common.cuh) -- or 0; *enabled = 1 in the
 * debug library, 0 in the release one (which checks nothing). */
int hs_debug_check(hs_ctx* ctx, uint64_t* first, int* enabled);
/* Launch one deliberately failing check (unit 1, tag 1): the debug library
 * then reports it through hs_debug_check; the release library reports 0. */
int hs_debug_selftest(hs_ctx* ctx);

/* ---- introspection (plan-only contexts too) ---------------------------- */
/* Sizes: L (= 2 N_e n), number of subdomains, number of groups, 2 N_e. */
int hs_sizes(const hs_ctx* ctx, int64_t* L, int* nsub, int* ngroups, int* npairs);
/* m-order pair table: pairs[4*k .. 4*k+3] = owner (i1,i2), neighbour (i1,i2). */
int hs_pairs(const hs_ctx* ctx, int32_t* pairs);
/* Rank that owns each subdomain block (owner's row band), length 2 N_e. */
int hs_block_owner(const hs_ctx* ctx, int32_t* owner_rank);
/* Step schedule of a preconditioner: rec[3*k] = step, rec[3*k+1] = phase
 * (0 forward, 1 residual, 2 backward), rec[3*k+2] = subdomain ordinal (index in
 * multi-index order).  Returns the number of entries in *count. */
int hs_schedule(const hs_ctx* ctx, int kind, int32_t* rec, int cap, int* count);
/* Trace-exchange plan of a step kind across row bands, for this rank: recv = 0
 * lists what it sends to `peer`, recv = 1 what it receives from `peer`, as
 * triples (step index, 0-based block m, buffer slot) in slot order, for the
 * steps of kind 0 (forward half), 1 (backward half), 2 (full apply) or the
 * map-once per-step form's 3 (residual rows), 4 ((I - S) z upper rows), 5
 * (window starts' late rows). */
int hs_exchange_plan(const hs_ctx* ctx, int kind, int peer, int recv, int32_t* triples, int cap,
                     int* count);

/* The Arnoldi basis of the last hs_gmres call on this context: the first
 * ncols basis vectors V[:, 0..ncols) as complex128, column after column, each
 * L x R ([L][R] layout); *avail = vectors built (max iterations + 1).  out =
 * NULL returns *avail only.  (max |V^H V - I| <= 1e-10; tests.) */
int hs_gmres_basis(hs_ctx* ctx, double* out, int ncols, int* avail);

/* Compact Schur map of subdomain (i1,i2) as a dense (k n) x (k n) complex
 * matrix, row-major (after hs_factor). */
int hs_get_schur(hs_ctx* ctx, int i1, int i2, double* T);
/* Replace the map of subdomain (i1,i2) (bring-up / tests only). */
int hs_set_schur(hs_ctx* ctx, int i1, int i2, const double* T);

/* ---- execution control / measurement ----------------------------------- */
/* 1 = calls with HS_MEM_DEVICE return without synchronising the stream. */
int hs_set_async(hs_ctx* ctx, int async_mode);
int hs_sync(hs_ctx* ctx);
/* The context's CUDA stream (cudaStream_t) as an integer. */
int hs_stream(hs_ctx* ctx, uint64_t* stream);
/* Kernel timing: when on, every step-apply launch is bracketed by CUDA events;
 * hs_kernel_stats reports launches, summed ms, algorithmic bytes (per-subdomain
 * map path) and algorithmic flops (8 per complex MAC) of the
 * step-apply kernels since the last reset. */
int hs_set_kernel_timing(hs_ctx* ctx, int on);
int hs_kernel_stats(hs_ctx* ctx, int64_t* launches, double* ms, double* bytes, double* flops,
                    int reset);
/* Number of kernels this context has launched (all kinds). */
int hs_launch_count(const hs_ctx* ctx, int64_t* n);
/* Bytes of device memory held by the context. */
int hs_memory(const hs_ctx* ctx, int64_t* bytes);

/* ---- multi-GPU ---------------------------------------------------------- */
/* Initialise the NCCL communicator of a sharded context from a 128-byte
 * ncclUniqueId produced by rank 0 (hs_nccl_unique_id). */
int hs_nccl_unique_id(uint8_t id[128]);
int hs_comm_init(hs_ctx* ctx, const uint8_t id[128]);

#ifdef __cplusplus
}
#endif
#endif /* HSB200_H */
