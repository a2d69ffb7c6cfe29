// Node placement for the node-centric DR kernel (see node_schedule.hpp).  Product code.
#include "node_schedule.hpp"

#include <algorithm>
#include <cstdint>
#include <numeric>

namespace fibra_b200 {

namespace {

struct Rng {  // splitmix64: deterministic placement for a given topology
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  int below(int n) { return static_cast<int>(next() % static_cast<uint64_t>(n)); }
};

}  // namespace

bool build_node_schedule(int N, int NFN, int M, const int* a, const int* b, int T, int NPT,
                         int search_moves, NodeSchedule& S) {
  S = NodeSchedule();
  S.T = T;
  S.NPT = NPT;
  const int NFIX = N - NFN;
  const int TS = T * NPT;
  S.f0 = (NFN + 31) / 32 * 32;
  S.node_slots = S.f0 + (NFIX + 31) / 32 * 32;
  if (S.node_slots > TS) return false;
  // incidence lists by packed node, ascending fiber id
  std::vector<std::vector<int>> fib(N), oth(N);
  for (int f = 0; f < M; ++f) {
    fib[a[f]].push_back(f);
    oth[a[f]].push_back(b[f]);
    fib[b[f]].push_back(f);
    oth[b[f]].push_back(a[f]);
  }
  std::vector<int> dg(N);
  for (int n = 0; n < N; ++n) dg[n] = static_cast<int>(fib[n].size());
  // degree-sorted placement (descending), free then fixed
  S.pn_of_slot.assign(TS, -1);
  S.slot_of_pn.assign(N, -1);
  auto place = [&](int lo, int hi, int slot0) {
    std::vector<int> ids(hi - lo);
    std::iota(ids.begin(), ids.end(), lo);
    std::stable_sort(ids.begin(), ids.end(), [&](int x, int y) { return dg[x] > dg[y]; });
    for (size_t i = 0; i < ids.size(); ++i) {
      S.pn_of_slot[slot0 + i] = ids[i];
      S.slot_of_pn[ids[i]] = static_cast<int>(slot0 + i);
    }
  };
  place(0, NFN, 0);
  place(NFN, N, S.f0);
  const int G = TS / 32;
  auto slot_deg = [&](int sl) { return S.pn_of_slot[sl] < 0 ? 0 : dg[S.pn_of_slot[sl]]; };

  // cost of one half-warp step: wavefronts beyond one per 64-bit load = the largest number
  // of distinct records sharing a bank pair, minus one
  auto cell_cost = [&](int g, int st, int h) {
    int load[16] = {0};
    int seen[16];
    int ns = 0;
    int worst = 0;
    for (int i = 0; i < 16; ++i) {
      const int pn = S.pn_of_slot[32 * g + 16 * h + i];
      if (pn < 0 || st >= dg[pn]) continue;
      const int o = S.slot_of_pn[oth[pn][st]];
      bool dup = false;
      for (int k = 0; k < ns; ++k) dup |= (seen[k] == o);
      if (dup) continue;
      seen[ns++] = o;
      worst = std::max(worst, ++load[o & 15]);
    }
    return worst > 0 ? worst - 1 : 0;
  };
  // the cells a node touches: its own steps, and the step at which each neighbour reads it
  auto cells_of = [&](int pn, std::vector<int64_t>& out) {
    const int sl = S.slot_of_pn[pn];
    for (int st = 0; st < dg[pn]; ++st)
      out.push_back((static_cast<int64_t>(sl / 32) << 32) | (st << 1) | ((sl & 31) >> 4));
    for (int k = 0; k < dg[pn]; ++k) {
      const int w = oth[pn][k];
      const int ws = S.slot_of_pn[w];
      const auto& lw = oth[w];
      for (int st = 0; st < dg[w]; ++st)
        if (lw[st] == pn)
          out.push_back((static_cast<int64_t>(ws / 32) << 32) | (st << 1) | ((ws & 31) >> 4));
    }
  };
  auto cost_of = [&](std::vector<int64_t>& cells) {
    std::sort(cells.begin(), cells.end());
    cells.erase(std::unique(cells.begin(), cells.end()), cells.end());
    long c = 0;
    for (int64_t k : cells)
      c += cell_cost(static_cast<int>(k >> 32), static_cast<int>((k & 0xffffffff) >> 1),
                     static_cast<int>(k & 1));
    return c;
  };
  auto total = [&]() {
    long c = 0, n = 0;
    for (int g = 0; g < G; ++g) {
      int mx = 0;
      for (int l = 0; l < 32; ++l) mx = std::max(mx, slot_deg(32 * g + l));
      for (int st = 0; st < mx; ++st)
        for (int h = 0; h < 2; ++h) {
          c += cell_cost(g, st, h);
          ++n;
        }
    }
    S.steps = n;
    return c;
  };
  S.excess_initial = total();
  // min-conflict search: swap two nodes of one class and equal degree (any warp), or two
  // slots of one warp (a node and a node or an empty slot); keep swaps that do not add
  // conflicts.  Swaps never change a warp's step count.
  Rng rng{static_cast<uint64_t>(N) * 1000003ull + static_cast<uint64_t>(M)};
  std::vector<int64_t> cells;
  long cur = S.excess_initial;
  for (int it = 0; it < search_moves && cur > 0; ++it) {
    const int pu = rng.below(N);
    const int su = S.slot_of_pn[pu];
    int sv;
    if (rng.next() & 1) {  // same warp, any lane of the same class region
      sv = (su & ~31) | rng.below(32);
    } else {  // same class, same degree, anywhere
      const int lo = pu < NFN ? 0 : NFN, hi = pu < NFN ? NFN : N;
      const int pv = lo + rng.below(hi - lo);
      if (dg[pv] != dg[pu]) continue;
      sv = S.slot_of_pn[pv];
    }
    if (sv == su) continue;
    const int pv = S.pn_of_slot[sv];
    if (pv >= 0 && ((pv < NFN) != (pu < NFN))) continue;
    if (pv < 0 && (sv < S.f0) != (su < S.f0)) continue;  // empty slot of the other class
    cells.clear();
    cells_of(pu, cells);
    if (pv >= 0) cells_of(pv, cells);
    const long before = cost_of(cells);
    auto swap_slots = [&]() {
      S.pn_of_slot[su] = pv;
      S.pn_of_slot[sv] = pu;
      S.slot_of_pn[pu] = sv;
      if (pv >= 0) S.slot_of_pn[pv] = su;
    };
    swap_slots();
    cells.clear();
    cells_of(pu, cells);
    if (pv >= 0) cells_of(pv, cells);
    const long after = cost_of(cells);
    if (after <= before) {
      cur += after - before;
    } else {  // undo
      S.pn_of_slot[su] = pu;
      S.pn_of_slot[sv] = pv;
      S.slot_of_pn[pu] = su;
      if (pv >= 0) S.slot_of_pn[pv] = sv;
    }
  }
  S.excess = total();
  // incidence rows per 32-slot group
  S.group_row0.assign(G + 1, 0);
  S.deg.assign(TS, 0);
  S.inc_fiber.assign(TS, {});
  S.inc_other.assign(TS, {});
  for (int g = 0; g < G; ++g) {
    int mx = 0;
    for (int l = 0; l < 32; ++l) {
      const int sl = 32 * g + l;
      const int pn = S.pn_of_slot[sl];
      if (pn < 0) continue;
      S.deg[sl] = dg[pn];
      S.inc_fiber[sl] = fib[pn];
      S.inc_other[sl] = oth[pn];
      mx = std::max(mx, dg[pn]);
    }
    S.group_row0[g + 1] = S.group_row0[g] + mx;
  }
  S.n_rows = S.group_row0[G];
  return true;
}

}  // namespace fibra_b200
