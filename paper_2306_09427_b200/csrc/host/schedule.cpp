// Bank-aware placement of an RVE topology onto the DR kernel's CTA (see schedule.hpp).
#include "schedule.hpp"

#include <algorithm>
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
    auto orient_from = [&](int r0) {
      int r = r0;
      for (;;) {
        int e = -1;
        for (int i : inc[r])
          if (!done[i]) { e = i; break; }
        if (e < 0) return;
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
    for (int r = 0; r < kBanks; ++r) orient_from(r);  // then cycles (and any conflicts)
    std::array<int, kBanks> tails{}, heads{};
    bool conflict = false;
    for (int i = 0; i < static_cast<int>(members.size()); ++i) {
      const int f = members[i];
      conflict |= tails[bank(s.tail_pn[f])]++ > 0;
      conflict |= heads[bank(s.head_pn[f])]++ > 0;
      s.fiber_of_fslot[kBanks * g + i] = f;
    }
    s.groups_conflicting += conflict;
  }

  // ---- g*d banks: distinct inside each fiber group, min-conflict inside gather steps
  std::vector<int> beta(M, 0), group_of(M, 0);
  for (int g = 0; g < n_groups; ++g)
    for (int i = 0; i < static_cast<int>(best_groups[g].size()); ++i) {
      beta[best_groups[g][i]] = i;
      group_of[best_groups[g][i]] = g;
    }
  // incident fibers per node in ascending id -> gather step k of half-warp slot/16
  std::vector<std::vector<int>> inc_fibers(N);
  for (int f = 0; f < M; ++f) {
    inc_fibers[a_pn[f]].push_back(f);
    inc_fibers[b_pn[f]].push_back(f);
  }
  int max_deg = 0;
  for (int pn = 0; pn < N; ++pn) max_deg = std::max<int>(max_deg, inc_fibers[pn].size());
  const int n_hw = s.node_slots / kBanks;
  // gather group id = hw * max_deg + k ; each fiber sits in two of them
  std::vector<std::array<int, 2>> gg_of(M, {-1, -1});
  for (int pn = 0; pn < N; ++pn) {
    const int hw = s.slot_of_pn[pn] / kBanks;
    for (int k = 0; k < static_cast<int>(inc_fibers[pn].size()); ++k) {
      const int f = inc_fibers[pn][k];
      gg_of[f][gg_of[f][0] < 0 ? 0 : 1] = hw * max_deg + k;
    }
  }
  std::vector<std::array<int, kBanks>> cnt(static_cast<size_t>(n_hw) * max_deg);
  for (auto& c : cnt) c.fill(0);
  for (int f = 0; f < M; ++f)
    for (int gg : gg_of[f]) ++cnt[gg][beta[f]];
  auto move_delta = [&](int f, int to) {  // cost change of moving f's bank to `to`
    int d = 0;
    for (int gg : gg_of[f]) d += cnt[gg][to] - (cnt[gg][beta[f]] - 1);
    if (gg_of[f][0] == gg_of[f][1]) d += 0;  // both endpoints in one step: counted twice
    return d;
  };
  auto apply_move = [&](int f, int to) {
    for (int gg : gg_of[f]) {
      --cnt[gg][beta[f]];
      ++cnt[gg][to];
    }
    beta[f] = to;
  };
  for (int pass = 0; pass < 40; ++pass) {
    bool improved = false;
    for (int g = 0; g < n_groups; ++g) {
      auto& members = best_groups[g];
      std::array<int, kBanks> owner;
      owner.fill(-1);
      for (int f : members) owner[beta[f]] = f;
      for (int f : members) {
        int best_to = -1, best_d = 0;
        for (int to = 0; to < kBanks; ++to) {
          if (to == beta[f]) continue;
          int d;
          const int other = owner[to];
          if (other < 0) {
            d = move_delta(f, to);
          } else {  // swap banks with `other` (keeps the group bank-distinct)
            const int from = beta[f];
            d = move_delta(f, to);
            apply_move(f, to);
            d += move_delta(other, from);
            apply_move(f, from);
          }
          if (d < best_d) {
            best_d = d;
            best_to = to;
          }
        }
        if (best_to >= 0) {
          const int from = beta[f], other = owner[best_to];
          apply_move(f, best_to);
          owner[best_to] = f;
          owner[from] = other;
          if (other >= 0) apply_move(other, from);
          improved = true;
        }
      }
    }
    if (!improved) break;
  }
  for (const auto& c : cnt) {
    int mx = 0, tot = 0;
    for (int v : c) {
      mx = std::max(mx, v);
      tot += v;
    }
    if (tot) {
      s.gather_excess += mx - 1;
      ++s.gather_steps;
    }
  }
  std::array<int, kBanks> used{};
  s.gslot_of_fiber.assign(M, -1);
  for (int f = 0; f < M; ++f) s.gslot_of_fiber[f] = beta[f] + kBanks * used[beta[f]]++;
  int mx = 0;
  for (int v : used) mx = std::max(mx, v);
  s.gd_slots = kBanks * std::max(mx, 1);
  return true;
}

}  // namespace fibra_b200
