// Host-side plan: lattice numbering, windows, step records, device step tables
// and the row-band exchange plan.  No CUDA here: plan-only contexts (device -1)
// and the CPU tests use it without a GPU.
//
// Reference: indexing.py:79-179 (m-order, groups, windows),
// interface_system.py:115-162 (which blocks a solve reads / writes),
// SPEC.md:306-357 (sweep step records).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace hs {

enum Face { W = 0, S = 1, N = 2, E = 3 };

struct SubPlan {
  int i1 = 0, i2 = 0, group = 0;
  int k = 0;             // number of interface faces
  int face[4] = {0};     // compact face -> face id (W,S,N,E order)
  int nbr[4] = {0};      // compact face -> neighbour subdomain ordinal
  int first_block = 0;   // 0-based m of its first incoming block m(s, .)
  int tgt_block[4] = {0};  // 0-based m(nbr, s) per compact face (block written)
  int nlower = 0;        // # of W/S faces (leading compact faces)
  int rank = 0;          // owning rank (row band)
  int cls = 0;           // operator class (distinct Dirichlet mask)
  int64_t T_off = 0;     // element offset of its map (tile-major, see hs_device.h)
};

// One batched solve-application of subdomain s, producing rows [rlo, rhi) of T_s.
struct Item {
  int s = 0, rlo = 0, rhi = 0, alt = 0;
  int slot[4] = {-1, -1, -1, -1};  // per compact face: -1 local, >=0 slot in send-up
                                   // buffer, <= -2 slot (-slot-2) in send-down buffer
};

struct RecvSlot {
  int dir;      // 0 = from rank-1 (below), 1 = from rank+1 (above)
  int slot;     // slot in that peer's send buffer
  int64_t off;  // element offset (block * n) in the local vector
};

struct StepTable {
  std::vector<Item> items;
  int nsend_up = 0, nsend_dn = 0;    // slots sent to rank+1 / rank-1
  std::vector<RecvSlot> recv;        // slots received, in slot order per direction
  int nrecv_up = 0, nrecv_dn = 0;    // slots received from rank+1 / rank-1
};

struct Plan {
  int n1 = 0, n2 = 0, n = 0, ng = 0, npairs = 0, nsub = 0;
  int rank = 0, nranks = 1;
  int64_t L = 0;
  std::vector<SubPlan> subs;         // multi-index order (|i|_1, i1)
  std::vector<int> ord;              // (i1-1) + n1*(i2-1) -> ordinal
  std::vector<int> block_sub;        // block -> owner ordinal
  std::vector<int> block_group;      // block -> owner group
  std::vector<int> row_lo;           // rank -> first row (1-based), size nranks+1
  std::vector<std::pair<int, int>> win_lower, win_upper;

  std::string build(int n1, int n2, int n, int rank, int nranks);
  int ordinal(int i1, int i2) const { return ord[(i1 - 1) + n1 * (i2 - 1)]; }
  int rank_of_row(int i2) const;
  void reference_windows();
  std::vector<int> group_members(int g) const;

  // Step tables of the sweeps.  dir 0 = forward over win_lower, 1 = backward over win_upper.
  std::vector<StepTable> half_steps(int dir) const;
  // within a sweep step record the blocks the solves write are
  // pairwise distinct and disjoint from the blocks they read in z (the sweeps
  // update z in place, so an overlap would make the result depend on the order
  // of the step's solves; a window start reads the half's input r instead, the
  // dedup rule of SURVEY.md §8a11).  Empty string = OK, else the violation.
  std::string check_step(const StepTable& st, bool in_place) const;
  StepTable full_step() const;
  StepTable restricted_step(const std::vector<int>& src, const std::vector<int>& tgt) const;
  // Keep this rank's items; fill send slots / receive lists (row-band exchange).
  StepTable localize(const StepTable& global) const;
};

}  // namespace hs
