// Bank-aware placement of an RVE topology onto the DR kernel's CTA (see schedule.hpp).
#include "schedule.hpp"

#include "fibra_cuda.h"

#include <algorithm>
#include <cmath>
#include <array>
#include <cstdint>
#include <numeric>
#include <random>
#include <vector>

namespace fibra_b200 {
namespace {

constexpr int kBanks = 16;

// Place one class (free or fixed) of nodes into consecutive 16-slot blocks starting at
// `first_slot`: nodes sorted by degree (descending), block rotation chosen greedily to keep
// the per-bank degree sums level.
void place_class(const std::vector<int>& nodes, const std::vector<int>& deg, int first_slot,
                 std::array<long, kBanks>& bank_deg, Schedule& s) {
  std::vector<int> order(nodes);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return deg[x] > deg[y]; });
  for (size_t b0 = 0; b0 < order.size(); b0 += kBanks) {
    const size_t cnt = std::min<size_t>(kBanks, order.size() - b0);
    int best_rot = 0;
    long best = -1;
    for (int rot = 0; rot < kBanks; ++rot) {
      std::array<long, kBanks> t = bank_deg;
      for (size_t i = 0; i < cnt; ++i) t[(i + rot) % kBanks] += deg[order[b0 + i]];
      long sq = 0;
      for (long v : t) sq += v * v;
      if (best < 0 || sq < best) {
        best = sq;
        best_rot = rot;
      }
    }
    const int block = first_slot + static_cast<int>(b0);
    for (size_t i = 0; i < cnt; ++i) {
      const int slot = block + static_cast<int>((i + best_rot) % kBanks);
      const int pn = order[b0 + i];
      s.slot_of_pn[pn] = slot;
      s.pn_of_slot[slot] = pn;
      bank_deg[slot % kBanks] += deg[pn];
    }
  }
}

}  // namespace

bool build_schedule(int N, int NFN, int M, const int* a_pn, const int* b_pn, int T, int FPT,
                    int NPT, Schedule& s) {
  s = Schedule{};
  s.T = T;
  s.FPT = FPT;
  s.NPT = NPT;
  s.n_free_nodes = NFN;
  s.n_fix_nodes = N - NFN;
  // class boundaries on warp multiples: the free/fixed branch of the node phase stays
  // warp-uniform
  s.f0 = (NFN + 31) / 32 * 32;
  s.node_slots = s.f0 + (s.n_fix_nodes + 31) / 32 * 32;
  s.fiber_slots = FPT * T;
  // the last warp reduces the convergence partials during the fiber phase and owns no
  // fibers (dr_kernel.cuh); its fiber groups stay empty
  const int reserved_warp = T / 32 - 1;
  auto usable = [&](int g) { return (g % (T / kBanks)) / 2 != reserved_warp; };
  if (s.node_slots > NPT * T || M > FPT * (T - 32)) return false;

  std::vector<int> deg(N, 0);
  for (int f = 0; f < M; ++f) {
    ++deg[a_pn[f]];
    ++deg[b_pn[f]];
  }
  s.slot_of_pn.assign(N, -1);
  s.pn_of_slot.assign(s.node_slots, -1);
  std::array<long, kBanks> bank_deg{};
  std::vector<int> free_nodes(NFN), fix_nodes(N - NFN);
  std::iota(free_nodes.begin(), free_nodes.end(), 0);
  std::iota(fix_nodes.begin(), fix_nodes.end(), NFN);
  place_class(free_nodes, deg, 0, bank_deg, s);
  place_class(fix_nodes, deg, s.f0, bank_deg, s);
  auto bank = [&](int pn) { return s.slot_of_pn[pn] % kBanks; };

  // ---- fiber groups: first fit under "bank degree <= 2 per group", best of a few orders
  const int n_groups = s.fiber_slots / kBanks;
  std::vector<std::vector<int>> best_groups;
  int best_leftover = -1;
  std::mt19937 rng(12345);
  std::vector<int> order(M);
  std::iota(order.begin(), order.end(), 0);
  for (int attempt = 0; attempt < 24 && best_leftover != 0; ++attempt) {
    if (attempt) std::shuffle(order.begin(), order.end(), rng);
    std::vector<std::vector<int>> groups(n_groups);
    std::vector<char> placed(M, 0);
    for (int g = 0; g < n_groups; ++g) {
      if (!usable(g)) continue;
      std::array<int, kBanks> d{};
      for (int f : order) {
        if (placed[f] || groups[g].size() == kBanks) continue;
        const int ra = bank(a_pn[f]), rb = bank(b_pn[f]);
        const bool ok = (ra == rb) ? d[ra] == 0 : (d[ra] < 2 && d[rb] < 2);
        if (!ok) continue;
        d[ra] += 1;
        d[rb] += 1;
        groups[g].push_back(f);
        placed[f] = 1;
      }
    }
    int left = 0;
    for (int f = 0; f < M; ++f) left += !placed[f];
    if (best_leftover < 0 || left < best_leftover) {
      best_leftover = left;
      // force leftovers into the emptiest groups (conflicting, but placed)
      for (int f = 0; f < M; ++f)
        if (!placed[f]) {
          int best = -1;
          for (int g = 0; g < n_groups; ++g)
            if (usable(g) && (best < 0 || groups[g].size() < groups[best].size())) best = g;
          groups[best].push_back(f);
        }
      best_groups = groups;
    }
  }
  bool ok_all = true;
  for (auto& g : best_groups) ok_all &= g.size() <= kBanks;
  if (!ok_all) return false;

  // ---- orientation: walk paths/cycles of each group's bank graph
  s.tail_pn.assign(M, -1);
  s.head_pn.assign(M, -1);
  s.fiber_of_fslot.assign(s.fiber_slots, -1);
  for (int g = 0; g < n_groups; ++g) {
    const auto& members = best_groups[g];
    std::array<std::vector<int>, kBanks> inc;
    for (int i = 0; i < static_cast<int>(members.size()); ++i) {
      const int f = members[i];
      inc[bank(a_pn[f])].push_back(i);
      if (bank(b_pn[f]) != bank(a_pn[f])) inc[bank(b_pn[f])].push_back(i);
    }
    std::vector<char> done(members.size(), 0);
    auto orient_from = [&](int r0) {  // one walk; false if r0 had no edge left
      int r = r0;
      for (bool first = true;; first = false) {
        int e = -1;
        for (int i : inc[r])
          if (!done[i]) { e = i; break; }
        if (e < 0) return !first;
        done[e] = 1;
        const int f = members[e];
        const int ra = bank(a_pn[f]);
        const bool a_tail = (ra == r);
        s.tail_pn[f] = a_tail ? a_pn[f] : b_pn[f];
        s.head_pn[f] = a_tail ? b_pn[f] : a_pn[f];
        r = bank(s.head_pn[f]);
      }
    };
    for (int r = 0; r < kBanks; ++r)
      if (inc[r].size() == 1) orient_from(r);  // path ends first
    // then cycles; a conflicting group (bank degree > 2) needs repeated walks per bank
    for (int r = 0; r < kBanks; ++r)
      while (orient_from(r)) {
      }
    std::array<int, kBanks> tails{}, heads{};
    bool conflict = false;
    for (int i = 0; i < static_cast<int>(members.size()); ++i) {
      const int f = members[i];
      if (s.tail_pn[f] < 0) return false;  // (every member is oriented above)
      conflict |= tails[bank(s.tail_pn[f])]++ > 0;
      conflict |= heads[bank(s.head_pn[f])]++ > 0;
      s.fiber_of_fslot[kBanks * g + i] = f;
    }
    s.groups_conflicting += conflict;
  }

  // ---- g*d records: each fiber writes a tail record (-g*d) and a head record (+g*d), each
  // read by exactly one gather step.  A record is an edge between its store group (the
  // half-warp STS instruction that writes it: fiber group x {tail, head}) and its gather
  // group (half-warp of the reading node x step in that node's list).  Both sides have
  // degree <= 16, so the bipartite multigraph is 16-edge-colourable (Koenig); colour c
  // becomes bank 3c mod 16 of the record and every store and gather is conflict-free.
  std::vector<int> group_of(M, 0);
  for (int g = 0; g < n_groups; ++g)
    for (int f : best_groups[g]) group_of[f] = g;
  std::vector<std::vector<int>> inc_fibers(N);
  for (int f = 0; f < M; ++f) {
    inc_fibers[a_pn[f]].push_back(f);
    inc_fibers[b_pn[f]].push_back(f);
  }
  int max_deg = 0;
  for (int pn = 0; pn < N; ++pn) max_deg = std::max<int>(max_deg, inc_fibers[pn].size());
  const int n_hw = s.node_slots / kBanks;
  // edges: 2f = tail record, 2f+1 = head record
  std::vector<int> eL(2 * M), eR(2 * M);
  for (int f = 0; f < M; ++f) {
    eL[2 * f] = 2 * group_of[f];
    eL[2 * f + 1] = 2 * group_of[f] + 1;
  }
  for (int pn = 0; pn < N; ++pn) {
    const int hw = s.slot_of_pn[pn] / kBanks;
    for (int k = 0; k < static_cast<int>(inc_fibers[pn].size()); ++k) {
      const int f = inc_fibers[pn][k];
      eR[2 * f + (pn == s.tail_pn[f] ? 0 : 1)] = hw * max_deg + k;
    }
  }
  const int nL = 2 * n_groups, nR = n_hw * max_deg;
  std::vector<std::array<int, kBanks>> atL(nL), atR(nR);  // edge holding colour c, or -1
  for (auto& x : atL) x.fill(-1);
  for (auto& x : atR) x.fill(-1);
  std::vector<int> colour(2 * M, -1);
  bool perfect = true;
  for (int e = 0; e < 2 * M; ++e) {
    const int u = eL[e], v = eR[e];
    int a = -1, b = -1;
    for (int c = 0; c < kBanks && a < 0; ++c)
      if (atL[u][c] < 0) a = c;
    for (int c = 0; c < kBanks && b < 0; ++c)
      if (atR[v][c] < 0) b = c;
    if (a < 0 || b < 0) {  // degree > 16 (cannot happen for <= 16-lane groups)
      perfect = false;
      colour[e] = 0;
      continue;
    }
    if (atR[v][a] >= 0) {
      // a is free at u, taken at v; b free at v.  Swap a<->b along the alternating path
      // that starts at v with colour a; it cannot reach u, after which a is free at v.
      std::vector<int> path;
      int node = v, side = 1, c = a;
      for (;;) {
        const int pe = side ? atR[node][c] : atL[node][c];
        if (pe < 0) break;
        path.push_back(pe);
        node = side ? eL[pe] : eR[pe];
        side ^= 1;
        c = (c == a) ? b : a;
      }
      for (int pe : path) {
        atL[eL[pe]][colour[pe]] = -1;
        atR[eR[pe]][colour[pe]] = -1;
      }
      for (int pe : path) {
        colour[pe] = (colour[pe] == a) ? b : a;
        atL[eL[pe]][colour[pe]] = pe;
        atR[eR[pe]][colour[pe]] = pe;
      }
    }
    colour[e] = a;
    atL[u][a] = e;
    atR[v][a] = e;
  }
  s.gather_steps = 0;
  for (int v = 0; v < nR; ++v) {
    bool any = false;
    for (int c = 0; c < kBanks; ++c) any |= atR[v][c] >= 0;
    s.gather_steps += any;
  }
  s.gather_excess = perfect ? 0 : -1;
  std::array<int, kBanks> used{};
  s.rec_tail.assign(M, -1);
  s.rec_head.assign(M, -1);
  for (int f = 0; f < M; ++f) {  // record index = colour + 16 * (running count of colour)
    const int ct = colour[2 * f], ch = colour[2 * f + 1];
    s.rec_tail[f] = ct + kBanks * used[ct]++;
    s.rec_head[f] = ch + kBanks * used[ch]++;
  }
  int mx = 0;
  for (int v : used) mx = std::max(mx, v);
  s.gd_slots = kBanks * std::max(mx, 1);
  return true;
}

}  // namespace fibra_b200

// Diagnostics (C-ABI, no GPU needed): schedule quality of one network for a kernel shape.
// Diagnostics: the node slot placement (packed node per slot, -1 empty) of that schedule.
extern "C" int fibra_schedule_slots(const fibra_net_desc* d, int T, int FPT, int NPT,
                                    int32_t* pn_of_slot, int32_t cap) {
  const int N = d->n_nodes, M = d->n_fibers;
  std::vector<int> a(M), b(M);
  for (int f = 0; f < M; ++f) {
    a[f] = d->fiber_packed_dofs[6 * f] / 3;
    b[f] = d->fiber_packed_dofs[6 * f + 3] / 3;
  }
  fibra_b200::Schedule s;
  if (!fibra_b200::build_schedule(N, d->n_free / 3, M, a.data(), b.data(), T, FPT, NPT, s))
    return 21;
  for (int i = 0; i < cap; ++i) pn_of_slot[i] = i < s.node_slots ? s.pn_of_slot[i] : -1;
  return 0;
}

extern "C" int fibra_schedule_report(const fibra_net_desc* d, int T, int FPT, int NPT,
                                     int64_t* out) {
  const int N = d->n_nodes, M = d->n_fibers;
  std::vector<int> a(M), b(M);
  for (int f = 0; f < M; ++f) {
    a[f] = d->fiber_packed_dofs[6 * f] / 3;
    b[f] = d->fiber_packed_dofs[6 * f + 3] / 3;
  }
  fibra_b200::Schedule s;
  const bool ok = fibra_b200::build_schedule(N, d->n_free / 3, M, a.data(), b.data(), T, FPT,
                                             NPT, s);
  out[0] = ok;
  out[1] = s.groups_conflicting;
  out[2] = s.gather_excess;
  out[3] = s.gather_steps;
  out[4] = s.gd_slots;
  out[5] = s.node_slots;
  return ok ? 0 : 21;
}
