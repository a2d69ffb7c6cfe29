// Internal host-side types of the B200 solver library (not part of the C-ABI).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "fibra_cuda.h"

namespace fibra_b200 {

// Immutable RVE network with the reference's derived layout (network.cpp:67-157).
struct Network {
  int n_nodes = 0, n_fibers = 0, n_free = 0;  // n_free counts DOFs
  double box_half = 0.5, tol_bnd = 1e-6, max_ea = 0;
  std::vector<double> coords;             // 3N node order
  std::vector<int32_t> fiber_nodes;       // 2M
  std::vector<double> area, modulus;      // M
  std::vector<double> rest_length;        // M
  std::vector<int32_t> boundary_nodes;    // ascending
  std::vector<int32_t> packed_of_dof;     // 3N
  std::vector<double> packed_ref;         // 3N
  std::vector<int32_t> fiber_packed_dofs; // 6M
  std::vector<double> node_lump;          // N
};

extern thread_local std::string g_host_err;
int fail(int code, const std::string& what);

int build_network(std::vector<double> coords, std::vector<int32_t> fiber_nodes,
                  std::vector<double> area, std::vector<double> modulus, double box_half,
                  double tol_bnd, Network& net);
int read_network(const std::string& path, double box_half, double tol_bnd, Network& net);
int write_network(const Network& net, const std::string& path);
int generate_network(const fibra_netgen_spec& spec, uint64_t seed, Network& net);
int generate_lattice(int n, int fibers, double jitter, double area, double modulus,
                     double box_half, double tol_bnd, uint64_t seed, Network& net);
void describe(const Network& net, fibra_net_desc* d);

}  // namespace fibra_b200
