// Partition of one RVE over a thread-block cluster (see cluster_schedule.hpp).
#include "host/cluster_schedule.hpp"

#include <algorithm>
#include <cstdint>
#include <numeric>

#include "fibra_cuda.h"

namespace fibra_b200 {
namespace {

// recursive coordinate bisection of nodes[lo, hi) into parts [part0, part0 + nparts),
// split along the longest extent at the weighted median (ties broken by node id, so the
// plan is deterministic)
void rcb(std::vector<int>& nodes, int lo, int hi, int part0, int nparts, const double* ref,
         const std::vector<double>& w, std::vector<int>& part_of) {
  if (nparts == 1) {
    for (int i = lo; i < hi; ++i) part_of[nodes[i]] = part0;
    return;
  }
  double mn[3] = {1e300, 1e300, 1e300}, mx[3] = {-1e300, -1e300, -1e300};
  for (int i = lo; i < hi; ++i)
    for (int k = 0; k < 3; ++k) {
      mn[k] = std::min(mn[k], ref[3 * nodes[i] + k]);
      mx[k] = std::max(mx[k], ref[3 * nodes[i] + k]);
    }
  int ax = 0;
  for (int k = 1; k < 3; ++k)
    if (mx[k] - mn[k] > mx[ax] - mn[ax]) ax = k;
  std::sort(nodes.begin() + lo, nodes.begin() + hi, [&](int x, int y) {
    const double cx = ref[3 * x + ax], cy = ref[3 * y + ax];
    return cx < cy || (cx == cy && x < y);
  });
  const int left = nparts / 2;
  double tot = 0;
  for (int i = lo; i < hi; ++i) tot += w[nodes[i]];
  const double target = tot * left / nparts;
  double acc = 0;
  int m = lo;
  while (m < hi - 1 && acc + 0.5 * w[nodes[m]] < target) acc += w[nodes[m++]];
  m = std::max(m, lo + 1);
  rcb(nodes, lo, m, part0, left, ref, w, part_of);
  rcb(nodes, m, hi, part0 + left, nparts - left, ref, w, part_of);
}

}  // namespace

void optimize_gather_banks(ClusterPlan& P, int c, int M, const int* a_pn, const int* b_pn,
                           int own_slots);

bool build_cluster_plan(int N, int NFN, int M, const int* a_pn, const int* b_pn,
                        const double* ref, int C, int T, int FPT, int NPT, bool mirror,
                        ClusterPlan& P) {
  P = ClusterPlan();
  P.mirror = mirror;
  P.C = C;
  P.T = T;
  P.FPT = FPT;
  P.NPT = NPT;
  if (C < 2 || N < C) return false;
  std::vector<double> w(N, 1.0);
  for (int f = 0; f < M; ++f) {
    w[a_pn[f]] += 1.0;
    w[b_pn[f]] += 1.0;
  }
  std::vector<int> nodes(N);
  std::iota(nodes.begin(), nodes.end(), 0);
  P.part_of_pn.assign(N, 0);
  rcb(nodes, 0, N, 0, C, ref, w, P.part_of_pn);

  // fiber ownership: internal fibers to their part; cross fibers to the lighter endpoint part
  std::vector<int> load(C, 0);
  P.owner_of_fiber.assign(M, -1);
  for (int f = 0; f < M; ++f)
    if (P.part_of_pn[a_pn[f]] == P.part_of_pn[b_pn[f]]) {
      P.owner_of_fiber[f] = P.part_of_pn[a_pn[f]];
      ++load[P.owner_of_fiber[f]];
    }
  for (int f = 0; f < M; ++f)
    if (P.owner_of_fiber[f] < 0) {
      const int pa = P.part_of_pn[a_pn[f]], pb = P.part_of_pn[b_pn[f]];
      const int o = load[pb] < load[pa] ? pb : pa;
      P.owner_of_fiber[f] = o;
      ++load[o];
    }

  P.parts.assign(C, ClusterPart());
  P.slot_of_pn.assign(N, -1);
  const int fiber_cap = FPT * (T - 32), slot_cap = NPT * T;
  for (int c = 0; c < C; ++c) {
    ClusterPart& Q = P.parts[c];
    std::vector<int> fr, fx;
    for (int pn = 0; pn < N; ++pn)
      if (P.part_of_pn[pn] == c) (pn < NFN ? fr : fx).push_back(pn);
    Q.n_free = static_cast<int>(fr.size());
    Q.n_fix = static_cast<int>(fx.size());
    Q.f0 = (Q.n_free + 31) / 32 * 32;
    Q.node_slots = (Q.f0 + Q.n_fix + 31) / 32 * 32;
    if (Q.node_slots > slot_cap) return false;
    // degree-sorted (descending, stable) so a warp's gather trip counts match
    auto by_degree = [&](int x, int y) { return w[x] > w[y]; };
    std::stable_sort(fr.begin(), fr.end(), by_degree);
    std::stable_sort(fx.begin(), fx.end(), by_degree);
    Q.pn_of_slot.assign(Q.node_slots, -1);
    for (int i = 0; i < Q.n_free; ++i) Q.pn_of_slot[i] = fr[i];
    for (int i = 0; i < Q.n_fix; ++i) Q.pn_of_slot[Q.f0 + i] = fx[i];
    for (int sl = 0; sl < Q.node_slots; ++sl)
      if (Q.pn_of_slot[sl] >= 0) P.slot_of_pn[Q.pn_of_slot[sl]] = sl;
  }
  for (int f = 0; f < M; ++f) {
    const int o = P.owner_of_fiber[f];
    ClusterPart& Q = P.parts[o];
    const bool a_here = P.part_of_pn[a_pn[f]] == o;
    const int tail = a_here ? a_pn[f] : b_pn[f];
    const int head = a_here ? b_pn[f] : a_pn[f];
    Q.fibers.push_back(f);
    Q.tail_pn.push_back(tail);
    Q.head_pn.push_back(head);
    const int ph = P.part_of_pn[head];
    if (ph != o) {
      Q.halo_pn.push_back(head);
      if (mirror) {  // the head's CTA evaluates it too (tail read from its halo)
        ClusterPart& R = P.parts[ph];
        R.fibers.push_back(f);
        R.tail_pn.push_back(tail);
        R.head_pn.push_back(head);
        R.halo_pn.push_back(tail);
      } else {
        P.parts[ph].h_fiber.push_back(f);
      }
    }
  }
  std::vector<int> copies(N, 0);
  std::vector<int> halo_of(N, -1);
  for (int c = 0; c < C; ++c) {
    ClusterPart& Q = P.parts[c];
    std::sort(Q.halo_pn.begin(), Q.halo_pn.end());
    Q.halo_pn.erase(std::unique(Q.halo_pn.begin(), Q.halo_pn.end()), Q.halo_pn.end());
    // Fiber slots: first-fit into half-warp groups of 16 whose tail x slots and head x slots
    // are distinct mod 16 (24-byte records: slot mod 16 selects the bank pair of every
    // component), flipping fibers with both ends here when that fits better.
    for (size_t h = 0; h < Q.halo_pn.size(); ++h) halo_of[Q.halo_pn[h]] = static_cast<int>(h);
    auto xbank = [&](int pn) {
      return P.part_of_pn[pn] == c ? P.slot_of_pn[pn] % 16 : (NPT * T + 2 + halo_of[pn]) % 16;
    };
    const int groups = fiber_cap / 16;
    std::vector<unsigned> tmask(groups, 0), hmask(groups, 0);
    std::vector<int> fill(groups, 0);
    Q.slot_fiber.assign(static_cast<size_t>(groups) * 16, -1);
    int open = 0;
    std::vector<int> leftovers;
    for (size_t i = 0; i < Q.fibers.size(); ++i) {
      const bool internal = mirror || P.part_of_pn[Q.head_pn[i]] == c;
      bool placed = false;
      for (int g = 0; g < open + 1 && g < groups && !placed; ++g) {
        if (fill[g] == 16) continue;
        for (int flip = 0; flip < (internal ? 2 : 1) && !placed; ++flip) {
          const int tl = flip ? Q.head_pn[i] : Q.tail_pn[i];
          const int hd = flip ? Q.tail_pn[i] : Q.head_pn[i];
          const unsigned tb = 1u << xbank(tl), hb = 1u << xbank(hd);
          if ((tmask[g] & tb) || (hmask[g] & hb)) continue;
          if (flip) std::swap(Q.tail_pn[i], Q.head_pn[i]);
          tmask[g] |= tb;
          hmask[g] |= hb;
          Q.slot_fiber[16 * g + fill[g]++] = static_cast<int>(i);
          open = std::max(open, g + 1);
          placed = true;
        }
      }
      if (!placed) leftovers.push_back(static_cast<int>(i));
    }
    for (int i : leftovers) {  // no conflict-free group left: any free slot
      int g = 0;
      while (g < groups && fill[g] == 16) ++g;
      if (g == groups) return false;
      Q.slot_fiber[16 * g + fill[g]++] = i;
    }
    for (int pn : Q.halo_pn) halo_of[pn] = -1;
    for (int pn : Q.halo_pn) P.max_push = std::max(P.max_push, ++copies[pn]);
    if (static_cast<int>(Q.fibers.size()) > fiber_cap) return false;
    P.max_halo = std::max(P.max_halo, static_cast<int>(Q.halo_pn.size()));
    P.max_records = std::max(P.max_records, static_cast<int>(Q.fibers.size() + Q.h_fiber.size()));
    P.max_fibers = std::max(P.max_fibers, static_cast<int>(Q.fibers.size()));
    P.max_node_slots = std::max(P.max_node_slots, Q.node_slots);
  }
  // Gather banks: a record's bank is its position mod 16, and the records a node half-warp
  // loads at one CSR step should sit in distinct banks.  Positions inside a fiber group are
  // free (the group's x loads stay conflict-free), and so are the positions of the copies of
  // remote fibers: local search over swaps that lower the sum over (half-warp, step) of the
  // largest bank multiplicity.
  for (int c = 0; c < C; ++c) optimize_gather_banks(P, c, M, a_pn, b_pn, fiber_cap);
  return true;
}

void optimize_gather_banks(ClusterPlan& P, int c, int M, const int* a_pn, const int* b_pn,
                           int own_slots) {
  ClusterPart& Q = P.parts[c];
  const int n_rec = own_slots + static_cast<int>(Q.h_fiber.size());
  // readers of every record: (half-warp, CSR entry index) of the local nodes gathering it;
  // the two entries of a step are separate load instructions, so the entry index is the cell
  std::vector<std::vector<std::pair<int, int>>> readers(n_rec);
  std::vector<int> rec_of_own(M, -1), rec_of_h(M, -1);  // this part's records
  for (int k = 0; k < static_cast<int>(Q.slot_fiber.size()); ++k)
    if (Q.slot_fiber[k] >= 0) rec_of_own[Q.fibers[Q.slot_fiber[k]]] = k;
  for (size_t h = 0; h < Q.h_fiber.size(); ++h) rec_of_h[Q.h_fiber[h]] = own_slots + static_cast<int>(h);
  std::vector<std::vector<int>> inc(Q.node_slots);
  std::vector<int> local_slot(P.slot_of_pn.size(), -1);
  for (int sl = 0; sl < Q.node_slots; ++sl)
    if (Q.pn_of_slot[sl] >= 0) local_slot[Q.pn_of_slot[sl]] = sl;
  for (int f = 0; f < M; ++f)
    for (int e : {a_pn[f], b_pn[f]})
      if (local_slot[e] >= 0 && (inc[local_slot[e]].empty() || inc[local_slot[e]].back() != f))
        inc[local_slot[e]].push_back(f);
  int max_steps = 0;
  for (int sl = 0; sl < Q.node_slots; ++sl) {
    for (size_t i = 0; i < inc[sl].size(); ++i) {
      const int f = inc[sl][i];
      const int r = rec_of_own[f] >= 0 ? rec_of_own[f] : rec_of_h[f];
      if (r >= 0) readers[r].push_back({sl / 16, static_cast<int>(i)});
    }
    max_steps = std::max(max_steps, static_cast<int>(inc[sl].size()));
  }
  const int hws = (Q.node_slots + 15) / 16;
  std::vector<int> cnt(static_cast<size_t>(hws) * max_steps * 16, 0);
  std::vector<int> pos(n_rec);  // record -> position (bank = pos % 16)
  for (int r = 0; r < n_rec; ++r) pos[r] = r;
  auto cell = [&](const std::pair<int, int>& hs) { return (hs.first * max_steps + hs.second) * 16; };
  for (int r = 0; r < n_rec; ++r)
    for (auto& hs : readers[r]) ++cnt[cell(hs) + pos[r] % 16];
  auto cell_cost = [&](int base) {
    int m = 0;
    for (int b = 0; b < 16; ++b) m = std::max(m, cnt[base + b]);
    return m;
  };
  // swap the banks of records r1 and r2 if that lowers the cost of the cells they touch
  auto try_swap = [&](int r1, int r2) {
    const int b1 = pos[r1] % 16, b2 = pos[r2] % 16;
    if (b1 == b2 || (readers[r1].empty() && readers[r2].empty())) return;
    std::vector<int> cells;
    for (auto& hs : readers[r1]) cells.push_back(cell(hs));
    for (auto& hs : readers[r2]) cells.push_back(cell(hs));
    std::sort(cells.begin(), cells.end());
    cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
    int before = 0, after = 0;
    for (int cb : cells) before += cell_cost(cb);
    for (auto& hs : readers[r1]) { --cnt[cell(hs) + b1]; ++cnt[cell(hs) + b2]; }
    for (auto& hs : readers[r2]) { --cnt[cell(hs) + b2]; ++cnt[cell(hs) + b1]; }
    for (int cb : cells) after += cell_cost(cb);
    if (after < before) {
      std::swap(pos[r1], pos[r2]);
    } else {  // undo
      for (auto& hs : readers[r1]) { ++cnt[cell(hs) + b1]; --cnt[cell(hs) + b2]; }
      for (auto& hs : readers[r2]) { ++cnt[cell(hs) + b2]; --cnt[cell(hs) + b1]; }
    }
  };
  const int n_h = n_rec - own_slots;
  for (int pass = 0; pass < 4; ++pass) {
    for (int g = 0; g < own_slots / 16; ++g)  // within a fiber group
      for (int i = 0; i < 16; ++i)
        for (int j = i + 1; j < 16; ++j) try_swap(16 * g + i, 16 * g + j);
    for (int i = 0; i < n_h; ++i)  // copies: against the next 15 in position order
      for (int d = 1; d < 16 && i + d < n_h; ++d) try_swap(own_slots + i, own_slots + i + d);
  }
  // apply: own records move inside their group, copies are reordered
  std::vector<int> slot_fiber(Q.slot_fiber.size(), -1);
  for (int k = 0; k < static_cast<int>(Q.slot_fiber.size()); ++k) slot_fiber[pos[k]] = Q.slot_fiber[k];
  Q.slot_fiber.swap(slot_fiber);
  std::vector<int> h_fiber(Q.h_fiber.size());
  for (int h = 0; h < n_h; ++h) h_fiber[pos[own_slots + h] - own_slots] = Q.h_fiber[h];
  Q.h_fiber.swap(h_fiber);
}

}  // namespace fibra_b200

// Diagnostics (C-ABI, no GPU needed): the cluster partition of one network.
extern "C" int fibra_cluster_report(const fibra_net_desc* d, int C, int T, int FPT, int NPT,
                                    int64_t* out) {
  const int N = d->n_nodes, M = d->n_fibers;
  std::vector<int> a(M), b(M);
  for (int f = 0; f < M; ++f) {
    a[f] = d->fiber_packed_dofs[6 * f] / 3;
    b[f] = d->fiber_packed_dofs[6 * f + 3] / 3;
  }
  fibra_b200::ClusterPlan plan;
  bool ok = fibra_b200::build_cluster_plan(N, d->n_free / 3, M, a.data(), b.data(),
                                           d->packed_ref, C, T, FPT, NPT, true, plan);
  if (!ok)
    ok = fibra_b200::build_cluster_plan(N, d->n_free / 3, M, a.data(), b.data(), d->packed_ref,
                                        C, T, FPT, NPT, false, plan);
  int min_fibers = M, cross = 0;
  for (const auto& q : plan.parts) min_fibers = std::min(min_fibers, static_cast<int>(q.fibers.size()));
  if (ok)
    for (int f = 0; f < M; ++f) cross += plan.part_of_pn[a[f]] != plan.part_of_pn[b[f]];
  out[0] = ok;
  out[1] = plan.max_fibers;
  out[2] = plan.parts.empty() ? 0 : min_fibers;
  out[3] = plan.max_node_slots;
  out[4] = plan.max_halo;
  out[5] = plan.max_records;
  out[6] = plan.max_push;
  out[7] = cross;
  return ok ? 0 : 21;
}
