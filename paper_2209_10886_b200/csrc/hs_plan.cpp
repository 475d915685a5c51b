// Host plan construction.  See hs_plan.h.
#include "hs_plan.h"

#include <algorithm>
#include <cmath>
#include <set>

namespace hs {

static const int kStep[4][2] = {{-1, 0}, {0, -1}, {0, 1}, {1, 0}};  // W, S, N, E
static const int kOpposite[4] = {E, N, S, W};

std::string Plan::build(int n1_, int n2_, int n_, int rank_, int nranks_) {
  if (n1_ < 1 || n2_ < 1) return "partition dimensions must be positive";
  if (n_ < 4) return "cells_per_side must be >= 4";
  if (nranks_ < 1 || rank_ < 0 || rank_ >= nranks_) return "bad rank / nranks";
  if (nranks_ > n2_) return "more ranks than subdomain rows";
  n1 = n1_; n2 = n2_; n = n_; rank = rank_; nranks = nranks_;
  ng = n1 + n2 - 1;
  nsub = n1 * n2;
  // row bands: the first (n2 % nranks) ranks get one extra row
  row_lo.assign(nranks + 1, 1);
  int base = n2 / nranks, extra = n2 % nranks;
  for (int r = 0; r < nranks; ++r) row_lo[r + 1] = row_lo[r] + base + (r < extra ? 1 : 0);
  // subdomains in multi-index order (|i|_1, i1)   (indexing.py:100-102)
  subs.clear();
  for (int g = 2; g <= n1 + n2; ++g)
    for (int a = 1; a <= n1; ++a) {
      int b = g - a;
      if (b < 1 || b > n2) continue;
      SubPlan sp;
      sp.i1 = a; sp.i2 = b; sp.group = g;
      subs.push_back(sp);
    }
  ord.assign(nsub, -1);
  for (int s = 0; s < nsub; ++s) ord[(subs[s].i1 - 1) + n1 * (subs[s].i2 - 1)] = s;
  // interface faces in W,S,N,E order == neighbour-key order (indexing.py:104-117)
  int blk = 0;
  for (int s = 0; s < nsub; ++s) {
    SubPlan& sp = subs[s];
    sp.first_block = blk;
    sp.k = 0; sp.nlower = 0;
    for (int f = 0; f < 4; ++f) {
      int a = sp.i1 + kStep[f][0], b = sp.i2 + kStep[f][1];
      if (a < 1 || a > n1 || b < 1 || b > n2) continue;
      sp.face[sp.k] = f;
      sp.nbr[sp.k] = ordinal(a, b);
      if (f == W || f == S) sp.nlower++;
      sp.k++;
    }
    blk += sp.k;
    sp.rank = rank_of_row(sp.i2);
  }
  npairs = blk;
  if (npairs != 2 * (2 * n1 * n2 - n1 - n2)) return "internal: pair count mismatch";
  L = (int64_t)npairs * n;
  block_sub.assign(npairs, 0);
  block_group.assign(npairs, 0);
  for (int s = 0; s < nsub; ++s)
    for (int q = 0; q < subs[s].k; ++q) {
      block_sub[subs[s].first_block + q] = s;
      block_group[subs[s].first_block + q] = subs[s].group;
    }
  // written block of each face: m(nbr, s), the neighbour's face toward s
  for (int s = 0; s < nsub; ++s) {
    SubPlan& sp = subs[s];
    for (int q = 0; q < sp.k; ++q) {
      const SubPlan& nb = subs[sp.nbr[q]];
      int want = kOpposite[sp.face[q]], found = -1;
      for (int p = 0; p < nb.k; ++p)
        if (nb.face[p] == want) found = p;
      sp.tgt_block[q] = nb.first_block + found;
    }
  }
  reference_windows();
  return "";
}

int Plan::rank_of_row(int i2) const {
  for (int r = 0; r < nranks; ++r)
    if (i2 >= row_lo[r] && i2 < row_lo[r + 1]) return r;
  return nranks - 1;
}

std::vector<int> Plan::group_members(int g) const {
  std::vector<int> out;
  for (int s = 0; s < nsub; ++s)
    if (subs[s].group == g) out.push_back(s);
  return out;
}

// indexing.py:158-179: p = ceil((N_g - 1)/N1) windows of N1 group steps, clipped.
void Plan::reference_windows() {
  win_lower.clear();
  win_upper.clear();
  if (ng < 2) return;
  int p = (ng - 1 + n1 - 1) / n1;
  for (int b = 1; b <= p; ++b) {
    int lo = 2 + (b - 1) * n1, hi = 2 + b * n1;
    win_lower.push_back({std::max(lo, 2), std::min(hi, ng + 1)});
    lo = (1 + ng) - b * n1;
    hi = (1 + ng) - (b - 1) * n1;
    win_upper.push_back({std::max(lo, 2), std::min(hi, ng + 1)});
  }
}

// Forward step t of window [lo,hi] solves group lo+t-1 toward lo+t (upper faces);
// backward step t of [lo,hi] solves hi-t+1 toward hi-t (lower faces).  The
// window's first step reads the half's input ("alt"), later ones the state
// (dedup rule).  Tables are built for all ranks, then
// localized (localize()).
std::vector<StepTable> Plan::half_steps(int dir) const {
  const auto& wins = dir == 0 ? win_lower : win_upper;
  int depth = 0;
  for (auto& w : wins) depth = std::max(depth, w.second - w.first);
  std::vector<StepTable> out;
  for (int t = 1; t <= depth; ++t) {
    StepTable st;
    for (auto& w : wins) {
      if (t > w.second - w.first) continue;
      int g = dir == 0 ? w.first + t - 1 : w.second - t + 1;
      for (int s : group_members(g)) {
        const SubPlan& sp = subs[s];
        Item it;
        it.s = s;
        it.alt = (t == 1);
        if (dir == 0) { it.rlo = sp.nlower * n; it.rhi = sp.k * n; }
        else { it.rlo = 0; it.rhi = sp.nlower * n; }
        if (it.rhi > it.rlo) st.items.push_back(it);
      }
    }
    out.push_back(localize(st));
  }
  return out;
}

std::string Plan::check_step(const StepTable& st, bool in_place) const {
  std::set<int> reads, writes;
  for (const Item& it : st.items) {
    if (it.alt) continue;  // a window start reads the half's input r, not the z being written
    const SubPlan& sp = subs[it.s];
    for (int q = 0; q < sp.k; ++q) reads.insert(sp.first_block + q);  // its incoming slab m(s, .)
  }
  for (const Item& it : st.items) {
    const SubPlan& sp = subs[it.s];
    for (int q = it.rlo / n; q < (it.rhi + n - 1) / n; ++q) {
      const int b = sp.tgt_block[q];  // m(nbr, s): the block subdomain s writes toward face q
      if (!writes.insert(b).second)
        return "step record writes block " + std::to_string(b + 1) + " twice";
      if (in_place && reads.count(b))
        return "step record reads and writes block " + std::to_string(b + 1) + " (subdomain (" +
               std::to_string(sp.i1) + "," + std::to_string(sp.i2) + ") writes into a slab solved in the same step)";
    }
  }
  return "";
}

StepTable Plan::full_step() const {
  StepTable st;
  for (int s = 0; s < nsub; ++s) {
    Item it;
    it.s = s; it.rlo = 0; it.rhi = subs[s].k * n;
    st.items.push_back(it);
  }
  return localize(st);
}

StepTable Plan::restricted_step(const std::vector<int>& src, const std::vector<int>& tgt) const {
  std::set<int> S(src.begin(), src.end()), Tg(tgt.begin(), tgt.end());
  StepTable st;
  for (int s = 0; s < nsub; ++s) {
    const SubPlan& sp = subs[s];
    if (!S.count(sp.group)) continue;
    bool lower = Tg.count(sp.group - 1) > 0, upper = Tg.count(sp.group + 1) > 0;
    Item it;
    it.s = s;
    it.rlo = lower ? 0 : sp.nlower * n;
    it.rhi = upper ? sp.k * n : sp.nlower * n;
    if (it.rhi > it.rlo) st.items.push_back(it);
  }
  return localize(st);
}

// Keep this rank's items.  Faces whose written block m(j, s) is owned by
// another rank go through the send buffers as raw outputs; the owner applies
// the epilogue on receipt.  Slots are numbered in global item order per
// (sender, receiver) pair, so sender and receiver agree by construction.
StepTable Plan::localize(const StepTable& global) const {
  StepTable st;
  int up = 0, dn = 0, rup = 0, rdn = 0;
  for (const Item& g : global.items) {
    const SubPlan& sp = subs[g.s];
    Item it = g;
    for (int q = 0; q < 4; ++q) it.slot[q] = -1;
    for (int q = 0; q < sp.k; ++q) {
      int r0 = q * n, r1 = (q + 1) * n;
      if (r1 <= g.rlo || r0 >= g.rhi) continue;  // face not produced by this item
      int src = sp.rank, dst = subs[sp.nbr[q]].rank;
      if (src == dst) continue;
      if (src == rank) {
        if (dst == rank + 1) it.slot[q] = up++;
        else if (dst == rank - 1) it.slot[q] = -2 - dn++;
      } else if (dst == rank) {
        RecvSlot rs;
        rs.dir = (src == rank - 1) ? 0 : 1;
        rs.slot = rs.dir == 0 ? rdn++ : rup++;
        rs.off = (int64_t)sp.tgt_block[q] * n;
        st.recv.push_back(rs);
      }
    }
    if (sp.rank == rank) st.items.push_back(it);
  }
  st.nsend_up = up; st.nsend_dn = dn; st.nrecv_dn = rdn; st.nrecv_up = rup;
  return st;
}

}  // namespace hs
