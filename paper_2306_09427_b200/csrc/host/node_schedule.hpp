// Host-side placement of one RVE topology for the node-centric DR kernel (dr_node.cuh).
//
// Every node slot walks its incident fibers in ascending reference fiber id (the
// accumulation order of network.cpp:298-303) and, at step s, gathers the x record of the
// other end.  The builder chooses:
//   * node slots: free nodes in [0, F0) (F0 a multiple of 32), fixed nodes after, each
//     sorted by degree so a warp's step count (its largest degree) wastes few lanes;
//   * the lane of every node inside its warp and, among nodes of equal degree, the warp:
//     a min-conflict local search over these placements makes the 16 x gathers of a
//     half-warp step hit distinct bank pairs (record o's components sit in bank pairs
//     3o + c mod 16, so a half-warp step is conflict-free iff its distinct records are
//     distinct mod 16).
// Nothing here changes an arithmetic operation or its order.
#pragma once

#include <cstdint>
#include <vector>

namespace fibra_b200 {

struct NodeSchedule {
  int T = 0, NPT = 0;
  int f0 = 0, node_slots = 0, n_rows = 0;
  std::vector<int> slot_of_pn, pn_of_slot;  // placement (-1 empty slot)
  std::vector<int> group_row0;              // per 32-slot group (+1): first incidence row
  std::vector<int> deg;                     // per slot
  // per slot: incident fibers in ascending id and the other end (packed node)
  std::vector<std::vector<int>> inc_fiber, inc_other;
  // quality report: half-warp gather steps, and their excess wavefronts over conflict-free
  long steps = 0, excess = 0, excess_initial = 0;
};

// a_pn/b_pn: fiber endpoints as packed node ids; nodes [0, n_free_nodes) are free.
// Returns false when the nodes do not fit NPT*T slots.
bool build_node_schedule(int n_nodes, int n_free_nodes, int n_fibers, const int* a_pn,
                         const int* b_pn, int T, int NPT, int search_moves, NodeSchedule& s);

}  // namespace fibra_b200
