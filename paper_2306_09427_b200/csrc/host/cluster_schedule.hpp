// Host-side partition of one large RVE over a thread-block cluster (product code).
//
// An RVE whose fibers do not fit one CTA (the resident kernel holds ~1.3k fibers) is
// solved by a cluster of C CTAs (C = 2, 4, 8 or 16; DSMEM, barrier.cluster).  Each CTA
// owns a spatial part of the nodes (recursive coordinate bisection weighted by degree) and
// the fibers whose *tail* it owns; a cross-part fiber is oriented so that its tail lies in
// the lighter part.  Swapping a fiber's endpoints is bitwise neutral (x_a - x_b ==
// -(x_b - x_a), g*(-d) == -(g*d)), the same argument schedule.hpp uses.
//
// Data movement per DR iteration, all through shared memory of the cluster:
//   * x of a part's nodes that are heads of another part's fibers is pushed by the owner
//     into that part's halo slots (st.shared::cluster) right after the node update;
//   * a fiber stores +g*d once in its own CTA's record (the tail node gathers it negated
//     through the CSR sign bit) and, when the head node lives elsewhere, once more into
//     a record of the head's CTA.
// So every x load of the fiber phase and every record load of the CSR gather is local;
// only stores cross SMs.  Each node still accumulates its incident fibers in ascending
// fiber id (network.cpp:298-303).
//
// Mirror mode (when the parts have room): a cross fiber is evaluated by *both* CTAs that hold
// one of its ends (same halo x, same arithmetic, so the same bits), so every record a node
// gathers is written by its own CTA and the fiber -> node handoff needs only a CTA barrier;
// one cluster barrier per DR iteration remains (after the x push).
#pragma once

#include <vector>

namespace fibra_b200 {

struct ClusterPart {
  int n_free = 0, n_fix = 0;        // own nodes
  int f0 = 0, node_slots = 0;       // free slots [0, f0), fixed [f0, f0 + n_fix)
  std::vector<int> pn_of_slot;      // [node_slots] own packed node ids (-1 empty)
  std::vector<int> halo_pn;         // remote nodes whose x this part reads
  std::vector<int> fibers;          // owned fibers, in fiber-slot order
  std::vector<int> tail_pn, head_pn;  // per owned fiber (tail is owned here)
  std::vector<int> slot_fiber;      // compact fiber slot k -> index into `fibers` (-1 dummy);
                                    // half-warp groups of 16 slots have bank-distinct x loads
  std::vector<int> h_fiber;         // fibers owned elsewhere whose head lives here (copies)
};

struct ClusterPlan {
  int C = 0, T = 0, FPT = 0, NPT = 0;
  std::vector<int> part_of_pn;      // [N]
  std::vector<int> slot_of_pn;      // [N] slot in the owning part
  std::vector<int> owner_of_fiber;  // [M]
  std::vector<ClusterPart> parts;   // [C]
  int max_halo = 0, max_records = 0, max_fibers = 0, max_node_slots = 0;
  int max_push = 0;                 // most halo copies of one node
  bool mirror = false;              // cross fibers evaluated in both parts, no copies
};

// ref: packed reference coordinates (3N); nodes [0, NFN) are free.  Returns false when a
// part exceeds the per-CTA capacity of the kernel shape (T threads, FPT fibers and NPT
// nodes per thread; the last warp owns no fibers).
bool build_cluster_plan(int N, int NFN, int M, const int* a_pn, const int* b_pn,
                        const double* ref, int C, int T, int FPT, int NPT, bool mirror,
                        ClusterPlan& plan);

}  // namespace fibra_b200
