// Host-side placement of one RVE topology onto a CTA (product code).
//
// The DR kernel exchanges positions x (node -> fiber) and fiber forces g*d (fiber -> node)
// through shared memory with random gathers.  64-bit shared loads of a half-warp are
// conflict-free when the 16 addresses fall in 16 distinct 8-byte bank pairs; records are
// 24-byte AoS (x,y,z), so record r's components sit in bank pairs 3r, 3r+1, 3r+2 (mod 16)
// and a half-warp is conflict-free iff its 16 record indices are distinct mod 16.
// This builder chooses, per entry:
//   * node slots: free nodes in [0, F0), fixed nodes in [F0, F0+...), each 16-slot block
//     holding nodes of similar degree (balanced gather trip counts), with a per-block
//     rotation that balances the bank degree;
//   * fiber groups (one half-warp of one fiber slot j): fibers whose endpoint banks form
//     paths/cycles, so after choosing each fiber's orientation the 16 "tail" loads and the
//     16 "head" loads are bank-distinct.  Swapping a fiber's endpoints is bitwise neutral:
//     x_a - x_b == -(x_b - x_a) and g*(-d) == -(g*d) in IEEE arithmetic;
//   * g*d record slots, one per fiber: bank-distinct inside every fiber group (stores) and
//     inside every gather step of every node half-warp (the tail's and the head's read),
//     by min-conflict search.
// Nothing here changes an arithmetic operation or its order: the reference accumulation
// order (ascending fiber id per node, network.cpp:298-303) is kept in each node's CSR list.
#pragma once

#include <cstdint>
#include <vector>

namespace fibra_b200 {

struct Schedule {
  int T = 0, FPT = 0, NPT = 0;
  int n_free_nodes = 0, f0 = 0, n_fix_nodes = 0;
  int node_slots = 0;    // slots in use (multiple of 16)
  int fiber_slots = 0;   // FPT * T
  int gd_slots = 0;      // multiple of 16
  std::vector<int> slot_of_pn, pn_of_slot;      // node placement (-1 empty)
  std::vector<int> fiber_of_fslot;              // fiber placement (-1 empty)
  std::vector<int> tail_pn, head_pn;            // stored orientation per fiber
  std::vector<int> rec;                         // g*d record per fiber (+g*d)
  // quality report
  int groups_conflicting = 0;       // fiber groups with a bank conflict on x loads
  long gather_excess = 0;           // extra wavefronts of the record colouring: gathers
  long store_excess = 0;            //   and g*d stores (0 and 0: perfect)
  long gather_steps = 0;
};

// a_pn/b_pn: fiber endpoints as packed node ids; nodes [0, n_free_nodes) are free.
bool build_schedule(int n_nodes, int n_free_nodes, int n_fibers, const int* a_pn,
                    const int* b_pn, int T, int FPT, int NPT, Schedule& s);

}  // namespace fibra_b200
