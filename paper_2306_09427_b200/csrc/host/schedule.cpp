// Bank-aware placement of an RVE topology onto the DR kernel's CTA (see schedule.hpp).
#include "schedule.hpp"

#include "fibra_cuda.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
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
  // every warp owns fibers; groups fill row by row (fiber slot j*T + tid), so the empty
  // slots gather in the last row of the last warps, which skip it (dr_kernel.cuh)
  auto usable = [&](int) { return true; };
  if (s.node_slots > NPT * T || M > FPT * T) return false;

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

  // ---- g*d records: one per fiber (+g*d), written by its fiber group's store and read by
  // two gather steps -- the tail's (negated) and the head's.  A record's colour c (bank
  // 3c mod 16) should be unique at each of those three "vertices": the store group, and
  // the (node half-warp, list position) of each reader.  Three vertices per record make
  // this a hypergraph colouring, so it is found by min-conflict search; a leftover
  // conflict costs one extra shared-memory wavefront, never a wrong result.
  std::vector<int> group_of(M, 0);
  for (int g = 0; g < n_groups; ++g)
    for (int f : best_groups[g]) group_of[f] = g;
  std::vector<std::vector<int>> inc_fibers(N);
  for (int f = 0; f < M; ++f) {
    inc_fibers[a_pn[f]].push_back(f);
    inc_fibers[b_pn[f]].push_back(f);
  }
  int max_deg = 0;
  for (int pn = 0; pn < N; ++pn) {
    std::sort(inc_fibers[pn].begin(), inc_fibers[pn].end());  // the gather's list order
    max_deg = std::max<int>(max_deg, inc_fibers[pn].size());
  }
  const int n_hw = s.node_slots / kBanks;
  // vertices: [0, n_groups) store groups, then n_hw * max_deg gather vertices
  std::vector<std::array<int, 3>> vert(M);
  for (int f = 0; f < M; ++f) vert[f] = {group_of[f], -1, -1};
  for (int pn = 0; pn < N; ++pn) {
    const int hw = s.slot_of_pn[pn] / kBanks;
    for (int k = 0; k < static_cast<int>(inc_fibers[pn].size()); ++k) {
      const int f = inc_fibers[pn][k];
      const int v = n_groups + hw * max_deg + k;
      if (vert[f][1] < 0) vert[f][1] = v;
      else if (vert[f][1] != v) vert[f][2] = v;  // same vertex: one broadcast read
    }
  }
  const int nV = n_groups + n_hw * max_deg;
  std::vector<std::array<int, kBanks>> cnt(nV);
  for (auto& x : cnt) x.fill(0);
  std::array<int, kBanks> used{};
  std::vector<int> colour(M, -1);
  auto weight = [&](int) { return 1; };  // a wavefront is a wavefront
  auto cost = [&](int f, int c) {  // conflicts f would add with colour c
    int w = 0;
    for (int i = 0; i < 3; ++i)
      if (vert[f][i] >= 0) w += weight(i) * cnt[vert[f][i]][c];
    return w;
  };
  auto place = [&](int f, int c, int d) {
    for (int i = 0; i < 3; ++i)
      if (vert[f][i] >= 0) cnt[vert[f][i]][c] += d;
    used[c] += d;
  };
  // greedy in order of descending gather degree of the readers (hardest first)
  std::vector<int> order_f(M);
  std::iota(order_f.begin(), order_f.end(), 0);
  std::stable_sort(order_f.begin(), order_f.end(), [&](int x, int y) {
    return deg[a_pn[x]] + deg[b_pn[x]] > deg[a_pn[y]] + deg[b_pn[y]];
  });
  for (int f : order_f) {
    int best = 0, bc = -1;
    for (int c = 0; c < kBanks; ++c) {
      const int w = cost(f, c);
      if (bc < 0 || w < bc || (w == bc && used[c] < used[best])) {
        bc = w;
        best = c;
      }
    }
    colour[f] = best;
    place(f, best, 1);
  }
  // Alternate (a) tabu search (TabuCol) over the colours -- the best non-tabu recolouring
  // of a conflicting record per step, a record may not return to a colour it just left --
  // and (b) store-group swaps: two fibers whose tail and head x slots lie in the same banks
  // may trade groups without disturbing the x loads; a swap is kept when it lowers the
  // conflicts of the two store groups (the gather vertices do not change).
  std::mt19937 crng(777);
  std::vector<std::vector<int>> at(nV);  // vertex -> records
  auto rebuild_at = [&]() {
    for (auto& x : at) x.clear();
    for (int f = 0; f < M; ++f)
      for (int i = 0; i < 3; ++i)
        if (vert[f][i] >= 0) at[vert[f][i]].push_back(f);
  };
  auto tabu = [&](long max_iter) {
    rebuild_at();
    std::vector<std::array<int, kBanks>> gam(M);  // weighted conflicts of f in colour c
    for (int f = 0; f < M; ++f) {
      place(f, colour[f], -1);
      for (int c = 0; c < kBanks; ++c) gam[f][c] = cost(f, c);
      place(f, colour[f], 1);
    }
    long conflicts = 0;
    for (int f = 0; f < M; ++f) conflicts += gam[f][colour[f]];
    conflicts /= 2;  // each conflicting pair is seen from both records
    std::vector<int> best_colour = colour;
    long best_conflicts = conflicts;
    std::vector<std::array<long, kBanks>> tabu_until(M);
    for (auto& x : tabu_until) x.fill(0);
    // the records in conflict, kept up to date as moves change their neighbours' counts
    std::vector<int> hot, where(M, -1);
    auto refresh = [&](int f) {
      const bool h = gam[f][colour[f]] > 0;
      if (h && where[f] < 0) {
        where[f] = static_cast<int>(hot.size());
        hot.push_back(f);
      } else if (!h && where[f] >= 0) {
        const int last = hot.back();
        hot[where[f]] = last;
        where[last] = where[f];
        hot.pop_back();
        where[f] = -1;
      }
    };
    for (int f = 0; f < M; ++f) refresh(f);
    long since_best = 0;
    for (long it = 1; it <= max_iter && conflicts > 0 && since_best < 4000; ++it, ++since_best) {
      int bf = -1, bcol = -1, bdelta = 0, ties = 0;
      for (int f : hot) {
        const int cur = gam[f][colour[f]];
        for (int c = 0; c < kBanks; ++c) {
          if (c == colour[f]) continue;
          const int delta = gam[f][c] - cur;
          if (!(tabu_until[f][c] < it || conflicts + delta < best_conflicts)) continue;
          if (bf < 0 || delta < bdelta) {
            bf = f; bcol = c; bdelta = delta; ties = 1;
          } else if (delta == bdelta && std::uniform_int_distribution<int>(0, ties++)(crng) == 0) {
            bf = f; bcol = c;
          }
        }
      }
      if (bf < 0) break;
      const int old = colour[bf];
      for (int i = 0; i < 3; ++i) {
        const int v = vert[bf][i];
        if (v < 0) continue;
        const int w = weight(i);  // the vertex's kind: store group or gather step
        for (int f2 : at[v]) {
          if (f2 == bf) continue;
          gam[f2][old] -= w;
          gam[f2][bcol] += w;
        }
      }
      place(bf, old, -1);
      colour[bf] = bcol;
      place(bf, bcol, 1);
      for (int i = 0; i < 3; ++i)
        if (vert[bf][i] >= 0)
          for (int f2 : at[vert[bf][i]]) refresh(f2);
      conflicts += bdelta;
      tabu_until[bf][old] = it + 10 + static_cast<long>(crng() % 10);
      if (conflicts < best_conflicts) {
        best_conflicts = conflicts;
        best_colour = colour;
        since_best = 0;
      }
    }
    if (best_conflicts < conflicts) {
      for (int f = 0; f < M; ++f) place(f, colour[f], -1);
      colour = best_colour;
      for (int f = 0; f < M; ++f) place(f, colour[f], 1);
    }
    return best_conflicts;
  };
  // swap partners: same (tail x bank, head x bank)
  auto xkey = [&](int f) {
    return (s.slot_of_pn[s.tail_pn[f]] % kBanks) * kBanks + s.slot_of_pn[s.head_pn[f]] % kBanks;
  };
  std::vector<std::vector<int>> by_key(kBanks * kBanks);
  for (int f = 0; f < M; ++f) by_key[xkey(f)].push_back(f);
  auto pairs = [&](int v) {
    int t = 0;
    for (int c = 0; c < kBanks; ++c) t += cnt[v][c] * (cnt[v][c] - 1) / 2;
    return t;
  };
  auto swap_pass = [&]() {
    bool any = false;
    for (int f = 0; f < M; ++f) {
      const int g1 = vert[f][0];
      if (cnt[g1][colour[f]] < 2) continue;  // f's store is not in conflict
      for (int f2 : by_key[xkey(f)]) {
        const int g2 = vert[f2][0];
        if (g2 == g1 || colour[f2] == colour[f]) continue;
        const int before = pairs(g1) + pairs(g2);
        --cnt[g1][colour[f]]; ++cnt[g2][colour[f]];
        --cnt[g2][colour[f2]]; ++cnt[g1][colour[f2]];
        if (pairs(g1) + pairs(g2) < before) {
          vert[f][0] = g2;
          vert[f2][0] = g1;
          auto& m1 = best_groups[g1];
          auto& m2 = best_groups[g2];
          *std::find(m1.begin(), m1.end(), f) = f2;
          *std::find(m2.begin(), m2.end(), f2) = f;
          any = true;
          break;
        }
        ++cnt[g1][colour[f]]; --cnt[g2][colour[f]];
        ++cnt[g2][colour[f2]]; --cnt[g1][colour[f2]];
      }
    }
    return any;
  };
  const char* rounds_env = getenv("FIBRA_SCHED_ROUNDS");  // diagnostics: search effort
  const int rounds = rounds_env ? atoi(rounds_env) : 2;
  const long iters = getenv("FIBRA_SCHED_ITERS") ? atol(getenv("FIBRA_SCHED_ITERS")) : 2000;
  long conflicts = tabu(2 * iters);
  for (int round = 0; round < rounds && conflicts > 0; ++round) {
    for (int sweep = 0; sweep < 10 && swap_pass(); ++sweep) {
    }
    conflicts = tabu(iters);
  }
  if (getenv("FIBRA_SCHED_DEBUG")) fprintf(stderr, "colouring: conflicts %ld\n", conflicts);
  for (int g = 0; g < n_groups; ++g)  // the store groups as finally composed
    for (int i = 0; i < static_cast<int>(best_groups[g].size()); ++i)
      s.fiber_of_fslot[kBanks * g + i] = best_groups[g][i];
  s.gather_steps = 0;
  for (int v = n_groups; v < nV; ++v) {
    int any = 0;
    for (int c = 0; c < kBanks; ++c) any |= cnt[v][c];
    s.gather_steps += any != 0;
  }
  s.gather_excess = 0;   // extra wavefronts: gather vertices
  s.store_excess = 0;    // and store groups
  for (int v = 0; v < nV; ++v) {
    int mx = 0;
    for (int c = 0; c < kBanks; ++c) mx = std::max(mx, cnt[v][c]);
    if (mx > 1) (v < n_groups ? s.store_excess : s.gather_excess) += mx - 1;
  }
  s.rec.assign(M, -1);
  std::array<int, kBanks> run{};
  for (int f = 0; f < M; ++f) s.rec[f] = colour[f] + kBanks * run[colour[f]]++;
  int mx = 0;
  for (int v : run) mx = std::max(mx, v);
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
  out[6] = s.store_excess;
  out[3] = s.gather_steps;
  out[4] = s.gd_slots;
  out[5] = s.node_slots;
  return ok ? 0 : 21;
}
