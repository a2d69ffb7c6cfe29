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

bool build_cluster_plan(int N, int NFN, int M, const int* a_pn, const int* b_pn,
                        const double* ref, int C, int T, int FPT, int NPT, ClusterPlan& P) {
  P = ClusterPlan();
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
      P.parts[ph].h_fiber.push_back(f);
    }
  }
  std::vector<int> copies(N, 0);
  for (int c = 0; c < C; ++c) {
    ClusterPart& Q = P.parts[c];
    std::sort(Q.halo_pn.begin(), Q.halo_pn.end());
    Q.halo_pn.erase(std::unique(Q.halo_pn.begin(), Q.halo_pn.end()), Q.halo_pn.end());
    for (int pn : Q.halo_pn) P.max_push = std::max(P.max_push, ++copies[pn]);
    if (static_cast<int>(Q.fibers.size()) > fiber_cap) return false;
    P.max_halo = std::max(P.max_halo, static_cast<int>(Q.halo_pn.size()));
    P.max_records = std::max(P.max_records, static_cast<int>(Q.fibers.size() + Q.h_fiber.size()));
    P.max_fibers = std::max(P.max_fibers, static_cast<int>(Q.fibers.size()));
    P.max_node_slots = std::max(P.max_node_slots, Q.node_slots);
  }
  return true;
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
  const bool ok = fibra_b200::build_cluster_plan(N, d->n_free / 3, M, a.data(), b.data(),
                                                 d->packed_ref, C, T, FPT, NPT, plan);
  int min_fibers = M, cross = 0;
  for (const auto& q : plan.parts) min_fibers = std::min(min_fibers, static_cast<int>(q.fibers.size()));
  for (const auto& q : plan.parts) cross += static_cast<int>(q.h_fiber.size());
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
