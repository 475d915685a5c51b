// Kernel launchers (host-callable), implemented in hs_apply.cu, hs_schur.cu, hs_krylov.cu.
#pragma once
#include <cuda_runtime.h>

#include <vector>

#include "hs_ctx.h"

namespace hs {

enum VecOp { VEC_ADD = 0, VEC_COPY2 = 1, VEC_INIT_BWD = 2 };

// Sparse right-hand-side additions of one operator class, grouped by grid row.
struct ExtraRHS {
  std::vector<int> row_ptr;  // n + 1 (empty = none)
  int* d_x = nullptr;
  int* d_col = nullptr;
  double2* d_val = nullptr;
};

// ---- step apply (hs_apply.cu)
void launch_step(Ctx& c, const DevStep& st, const double2* srcA, const double2* srcB, const Epi& e,
                 int R);
void launch_recv_epi(Ctx& c, const DevStep& st, const Epi& e, int R);
void launch_vec(Ctx& c, int op, long long len, double2* o1, double2* o2, const double2* a,
                const double2* b);
void launch_seam_add(Ctx& c, int dir, double2* z, const double2* r, int R);
void launch_block_fill(Ctx& c, const int* blocks, int nb, int mode, double2* o1, double2* o2, double2* o3,
                       const double2* a, int R, cudaStream_t st = nullptr);
cudaError_t set_step_smem_limit();
cudaError_t launch_bsp_fused_ranks(Ctx& c, const DevFused& f, const MultiRankArgs& mr);
void launch_gather_blocks(Ctx& c, double2* out, const double2* const* src, int G, const int* blk_rank, long long L);
// wout != null: the plan's phase-3 tiles write (I - S) z there (GMRES A M v in one launch)
cudaError_t launch_bsp_fused(Ctx& c, const DevFused& f, const double2* r, double2* zL, double2* rp,
                             double2* w, double2* z, double2* wout = nullptr);
void launch_zmma(Ctx& c, const DevMma& m, const double2* A, const double2* srcA, const double2* srcB,
                 const double2* zeros, const Epi& e, int R);
cudaError_t set_zmma_smem_limit();
cudaError_t launch_zmma_fused(Ctx& c, const DevFusedMma& f, FusedMmaArgs a);
void launch_pack_strips(Ctx& c, const double2* T4, double2* out, int rows, int cols);

// ---- factorisation (hs_schur.cu)
// Rp / Cp / Bk: two slices each (2 * ncls), one per elimination chain
cudaError_t factor_and_solve_boundary(Ctx& c, double2* X, long long xstride, const uint8_t* dmasks, int ncls,
                                      double2* Rp, double2* Cp, long long pstride, int* dbad, int R, int nunit,
                                      const ExtraRHS* extras, double2* Y, long long ystride, double2* Bk,
                                      long long bstride, double2* G, long long gstride);
cudaError_t solve_boundary(Ctx& c, const double2* X, long long xstride, const uint8_t* dmasks,
                           int ncls, int R, int nunit, const ExtraRHS* extras, double2* Y,
                           long long ystride, double2* Bk, long long bstride, double2* G,
                           long long gstride);
// DMMA path of zgemm (M, N, K multiples of 32); false when not applicable
bool zgemm_dmma(cudaStream_t st, int M, int N, int K, double2 alpha, const double2* A, int lda, long long sa,
                const double2* B, int ldb, long long sb, double2 beta, double2* C, int ldc, long long sc,
                int batch);
void zgemm(cudaStream_t st, int M, int N, int K, double2 alpha, const double2* A, int lda,
           long long sa, const double2* B, int ldb, long long sb, double2 beta, double2* C, int ldc,
           long long sc, int batch);
void launch_make_T4(Ctx& c, double2* T4, const double2* G, int R, double2 a, double2 b);
void launch_finite_check(Ctx& c, const double2* v, long long count, int* flag);
cudaError_t solve_fields(Ctx& c, const double2* X, const uint8_t* dmask, int R, const double2* g,
                         const int* face_off, double2 coeff, const ExtraRHS& extras, double2* Y, double2* Bk);
void launch_scatter_field(Ctx& c, double2* field, int nx_total, const double2* Y, int R, const int* col_ab,
                          int accumulate);
void launch_scatter_T(Ctx& c, const int2* tl, int ntiles, const int* sub_faces, const int* sub_cls,
                      double2* const* T4s);
void launch_lift_b(Ctx& c, double2* b, const double2* G, int Rtot, int col0, int nrhs,
                   const int* face_tgt, double2 coef);

// ---- GMRES (hs_krylov.cu)
struct GmresDev {
  double2* V;        // (maxit+1) x LR basis
  long long LR;      // L * R
  int R;
  double2* H;        // packed columns: column k at offset R * k(k+3)/2, length (k+2) x R
  double* cs;        // maxit x R
  double2* sn;       // maxit x R
  double2* g;        // (maxit+1) x R
  double* hist;      // (maxit+1) x R
  double* beta;      // R
  double* wnorm0;    // R
  int* active;       // R: 1 while iterating
  int* iters;        // R
  int* conv;         // R
  int* brk;          // R
  int* nactive;      // 1
  double2* partial;  // 2 x grid x R
  double2* y;        // maxit x R
  double tol;
};
cudaError_t gmres_init(Ctx& c, GmresDev& G, const double2* b);
cudaError_t gmres_arnoldi(Ctx& c, GmresDev& G, int k, int grid, int chunk);
cudaError_t gmres_givens(Ctx& c, GmresDev& G, int k);
cudaError_t gmres_finish(Ctx& c, GmresDev& G, int maxit, double2* u);
int gmres_coop_grid(Ctx& c, long long LR, int R, int* chunk);
// one right-hand side: register-resident w, cp.async-prefetched basis, Givens fused
// (grid > 0 when the vector and maxit fit; returns the grid)
int gmres_mgs1_plan(Ctx& c, long long LR, int R, int maxit, int* chunk, int* E, int* bd);
cudaError_t gmres_arnoldi1(Ctx& c, GmresDev& G, int k, int grid, int chunk, int E, int bd);
// the same on one thread-block cluster (returns the cluster size; 0 = not applicable)
int gmres_mgs1c_plan(long long LR, int R, int maxit, int* chunk, int* E, int* bd);
cudaError_t gmres_arnoldi1c(Ctx& c, GmresDev& G, int k, int cs, int chunk, int E, int bd);
// Arnoldi step + Givens on one thread-block cluster (small vectors)
int gmres_cluster_size(long long LR, int R, int* chunk);
cudaError_t gmres_arnoldi_cluster(Ctx& c, GmresDev& G, int k, int cs, int chunk);
// host-driven MGS over owned blocks (+ one ncclAllReduce per inner product when comm != null)
cudaError_t gmres_arnoldi_dist(Ctx& c, GmresDev& G, int k, const int* blocks, int nb, double2* part,
                               double2* out, void* nccl_comm);
cudaError_t gmres_init_dist(Ctx& c, GmresDev& G, const double2* b, const int* blocks, int nb,
                            double2* part, double2* out, void* nccl_comm);
// CGS2 Arnoldi (one RHS): two passes, one allreduce of k+1 values each across row bands
cudaError_t gmres_arnoldi_cgs2(Ctx& c, GmresDev& G, int k, const int* blocks, int nb, double2* part,
                               double2* hbuf, void* nccl_comm);
// in-place sum over ranks (implemented next to the NCCL calls in hs_api.cu)
cudaError_t gmres_arnoldi_cgsg(Ctx& c, GmresDev& G, int k, const int* blocks, int nb, double2* part,
                               double2* red, double2* Gm, int ldg, void* nccl_comm);
// the same for R right-hand sides on one rank (Givens included); ok: sizes fit
bool gmres_cgsgR_ok(Ctx& c, long long LR, int R, int maxit);
cudaError_t gmres_arnoldi_cgsgR(Ctx& c, GmresDev& G, int k, double2* part, double2* red, double2* Gm, int ldg,
                                int* sync);  // sync: two zeroed ints
cudaError_t allreduce_sum_doubles(Ctx& c, double* buf, size_t count, void* nccl_comm);
cudaError_t launch_peer_allreduce(Ctx& c, const PeerRedArgs& a);
// first device-check failure of each translation unit (0: none; debug library only)
unsigned long long hs_dbg_take_apply();
cudaError_t launch_dbg_selftest(Ctx& c);
unsigned long long hs_dbg_take_zmma();
unsigned long long hs_dbg_take_krylov();
unsigned long long hs_dbg_take_schur();

}  // namespace hs
