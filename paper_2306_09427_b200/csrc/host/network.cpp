// Host-side RVE network construction for the B200 solver (product code).
//
// Mirrors fibra::FiberNetwork (reference proj/include/fibra/network.hpp:55-101, ctor
// proj/src/network.cpp:67-157, file format network.cpp:164-230): validation, boundary
// classification, free-first DOF packing, rest lengths and lumping weights.  The solver
// consumes only the derived arrays (fibra_net_desc), so the reference's own object can
// feed the same C-ABI directly; this builder exists so the product can run without the
// reference library (bench inputs, Python API).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <unordered_set>
#include <vector>

#include "fibra_cuda.h"
#include "host_internal.hpp"

namespace fibra_b200 {

thread_local std::string g_host_err;

int fail(int code, const std::string& what) {
  g_host_err = what;
  return code;
}

int build_network(std::vector<double> coords, std::vector<int32_t> fiber_nodes,
                  std::vector<double> area, std::vector<double> modulus, double box_half,
                  double tol_bnd, Network& net) {
  const int nn = static_cast<int>(coords.size() / 3);
  const int nf = static_cast<int>(area.size());
  if (nn == 0) return fail(FIBRA_E_CONFIG, "network has no nodes");
  if (!(box_half > 0)) return fail(FIBRA_E_CONFIG, "RVE box half extent must be > 0");
  for (int i = 0; i < 3 * nn; ++i) {
    if (!std::isfinite(coords[i]))
      return fail(FIBRA_E_CONFIG, "non-finite coordinate at node " + std::to_string(i / 3));
    if (std::abs(coords[i]) > box_half + tol_bnd)
      return fail(FIBRA_E_CONFIG, "node " + std::to_string(i / 3) + " lies outside the RVE box");
  }
  net = Network{};
  net.n_nodes = nn;
  net.n_fibers = nf;
  net.box_half = box_half;
  net.tol_bnd = tol_bnd;
  net.rest_length.resize(nf);
  std::unordered_set<uint64_t> edges;
  edges.reserve(2 * static_cast<size_t>(nf) + 1);
  double max_ea = 0;
  for (int f = 0; f < nf; ++f) {
    const int32_t a = fiber_nodes[2 * f], b = fiber_nodes[2 * f + 1];
    const std::string fs = "fiber " + std::to_string(f);
    if (a < 0 || b < 0 || a >= nn || b >= nn) return fail(FIBRA_E_CONFIG, fs + " references a bad node index");
    if (a == b) return fail(FIBRA_E_CONFIG, fs + " connects a node to itself");
    if (!(area[f] > 0) || !(modulus[f] > 0)) return fail(FIBRA_E_CONFIG, fs + " needs positive area and modulus");
    const uint64_t key = (static_cast<uint64_t>(std::min(a, b)) << 32) | static_cast<uint32_t>(std::max(a, b));
    if (!edges.insert(key).second)
      return fail(FIBRA_E_CONFIG, "duplicate fiber between nodes " + std::to_string(a) + " and " + std::to_string(b));
    const double dx = coords[3 * b] - coords[3 * a];
    const double dy = coords[3 * b + 1] - coords[3 * a + 1];
    const double dz = coords[3 * b + 2] - coords[3 * a + 2];
    const double l0 = std::sqrt(dx * dx + dy * dy + dz * dz);
    if (!(l0 > 0)) return fail(FIBRA_E_CONFIG, fs + " has zero rest length");
    net.rest_length[f] = l0;
    const double ea = area[f] * modulus[f];
    max_ea = (max_ea < ea) ? ea : max_ea;
  }
  net.max_ea = max_ea;

  // boundary: any coordinate within tol of the face (network.cpp:109-117)
  std::vector<uint8_t> bnd(nn, 0);
  for (int i = 0; i < nn; ++i) {
    for (int k = 0; k < 3; ++k)
      if (std::abs(std::abs(coords[3 * i + k]) - box_half) <= tol_bnd) bnd[i] = 1;
    if (bnd[i]) net.boundary_nodes.push_back(i);
  }
  if (net.boundary_nodes.empty())
    return fail(FIBRA_E_CONFIG, "network has no boundary nodes; the RVE cannot carry load");

  // free-first packing: interior nodes ascending, then boundary nodes ascending
  net.packed_of_dof.assign(3 * nn, -1);
  int slot = 0;
  for (int pass = 0; pass < 2; ++pass) {
    for (int i = 0; i < nn; ++i) {
      if (bnd[i] != pass) continue;
      for (int k = 0; k < 3; ++k) net.packed_of_dof[3 * i + k] = slot++;
    }
    if (pass == 0) net.n_free = slot;
  }
  net.packed_ref.assign(3 * nn, 0.0);
  for (int d = 0; d < 3 * nn; ++d) net.packed_ref[net.packed_of_dof[d]] = coords[d];
  net.fiber_packed_dofs.resize(6 * static_cast<size_t>(nf));
  for (int f = 0; f < nf; ++f)
    for (int k = 0; k < 3; ++k) {
      net.fiber_packed_dofs[6 * f + k] = net.packed_of_dof[3 * fiber_nodes[2 * f] + k];
      net.fiber_packed_dofs[6 * f + 3 + k] = net.packed_of_dof[3 * fiber_nodes[2 * f + 1] + k];
    }
  // lumping weights: half rest length * area per incident fiber, fiber order
  net.node_lump.assign(nn, 0.0);
  for (int f = 0; f < nf; ++f) {
    const double half_seg = 0.5 * net.rest_length[f] * area[f];
    net.node_lump[fiber_nodes[2 * f]] += half_seg;
    net.node_lump[fiber_nodes[2 * f + 1]] += half_seg;
  }
  net.coords = std::move(coords);
  net.fiber_nodes = std::move(fiber_nodes);
  net.area = std::move(area);
  net.modulus = std::move(modulus);
  return FIBRA_OK;
}

int read_network(const std::string& path, double box_half, double tol_bnd, Network& net) {
  std::ifstream in(path);
  if (!in) return fail(FIBRA_E_IO, "cannot open network file " + path);
  std::vector<std::string> lines;
  std::string line;
  while (std::getline(in, line))
    if (line.find_first_not_of(" \t\r\n") != std::string::npos) lines.push_back(line);
  size_t li = 0;
  auto bad = [&](const std::string& what) {
    return fail(FIBRA_E_IO, "network file " + path + ": " + what);
  };
  long n = 0, m = 0;
  if (li >= lines.size()) return bad("unexpected end");
  {
    std::istringstream s(lines[li++]);
    if (!(s >> n >> m) || n <= 0 || m < 0) return bad("expected 'N M' header");
  }
  std::vector<double> coords(3 * n);
  for (long i = 0; i < n; ++i) {
    if (li >= lines.size()) return bad("unexpected end");
    std::istringstream s(lines[li++]);
    if (!(s >> coords[3 * i] >> coords[3 * i + 1] >> coords[3 * i + 2])) return bad("expected 'x y z'");
  }
  std::vector<int32_t> fn(2 * m);
  std::vector<double> area(m), modulus(m);
  for (long f = 0; f < m; ++f) {
    if (li >= lines.size()) return bad("unexpected end");
    std::istringstream s(lines[li++]);
    long a, b;
    if (!(s >> a >> b >> area[f] >> modulus[f])) return bad("expected 'i j area modulus'");
    if (a < 0 || b < 0 || a >= n || b >= n) return bad("node index out of range");
    if (!std::isfinite(area[f]) || !std::isfinite(modulus[f])) return bad("non-finite fiber data");
    fn[2 * f]= static_cast<int32_t>(a);
    fn[2 * f + 1] = static_cast<int32_t>(b);
  }
  const int rc = build_network(std::move(coords), std::move(fn), std::move(area),
                               std::move(modulus), box_half, tol_bnd, net);
  return rc == FIBRA_E_CONFIG ? FIBRA_E_IO : rc;
}

int write_network(const Network& net, const std::string& path) {
  FILE* fp = std::fopen(path.c_str(), "w");
  if (!fp) return fail(FIBRA_E_IO, "cannot write network file " + path);
  std::fprintf(fp, "%d %d\n", net.n_nodes, net.n_fibers);
  for (int i = 0; i < net.n_nodes; ++i)
    std::fprintf(fp, "%.17g %.17g %.17g\n", net.coords[3 * i], net.coords[3 * i + 1],
                 net.coords[3 * i + 2]);
  for (int f = 0; f < net.n_fibers; ++f)
    std::fprintf(fp, "%d %d %.17g %.17g\n", net.fiber_nodes[2 * f], net.fiber_nodes[2 * f + 1],
                 net.area[f], net.modulus[f]);
  const bool ok = std::fclose(fp) == 0;
  return ok ? FIBRA_OK : fail(FIBRA_E_IO, "failed writing network file " + path);
}

void describe(const Network& net, fibra_net_desc* d) {
  d->n_nodes = net.n_nodes;
  d->n_fibers = net.n_fibers;
  d->n_free = net.n_free;
  d->n_boundary = static_cast<int32_t>(net.boundary_nodes.size());
  d->coords = net.coords.data();
  d->fiber_nodes = net.fiber_nodes.data();
  d->fiber_area = net.area.data();
  d->fiber_modulus = net.modulus.data();
  d->packed_of_dof = net.packed_of_dof.data();
  d->packed_ref = net.packed_ref.data();
  d->fiber_packed_dofs = net.fiber_packed_dofs.data();
  d->rest_length = net.rest_length.data();
  d->node_lump = net.node_lump.data();
  d->boundary_nodes = net.boundary_nodes.data();
  d->box_half = net.box_half;
  d->max_ea = net.max_ea;
}

}  // namespace fibra_b200

using fibra_b200::Network;

struct fibra_network {
  Network net;
};

extern "C" {

const char* fibra_host_last_error(void) { return fibra_b200::g_host_err.c_str(); }

int fibra_network_create(const double* coords, int32_t n_nodes, const int32_t* fiber_nodes,
                         const double* area, const double* modulus, int32_t n_fibers,
                         double box_half, double tol_bnd, fibra_network** out) {
  if (!out || n_nodes < 0 || n_fibers < 0) return fibra_b200::fail(FIBRA_E_ARG, "bad arguments");
  auto* h = new fibra_network;
  std::vector<double> c(coords, coords + 3 * static_cast<size_t>(n_nodes));
  std::vector<int32_t> fn(fiber_nodes, fiber_nodes + 2 * static_cast<size_t>(n_fibers));
  std::vector<double> ar(area, area + n_fibers), mo(modulus, modulus + n_fibers);
  const int rc = fibra_b200::build_network(std::move(c), std::move(fn), std::move(ar),
                                           std::move(mo), box_half, tol_bnd, h->net);
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return FIBRA_OK;
}

int fibra_network_generate(const fibra_netgen_spec* spec, uint64_t seed, fibra_network** out) {
  if (!spec || !out) return fibra_b200::fail(FIBRA_E_ARG, "bad arguments");
  auto* h = new fibra_network;
  const int rc = fibra_b200::generate_network(*spec, seed, h->net);
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return FIBRA_OK;
}

int fibra_network_generate_lattice(int32_t n_side, int32_t fibers, double jitter, double area,
                                   double modulus, double box_half, double tol_bnd,
                                   uint64_t seed, fibra_network** out) {
  if (!out) return fibra_b200::fail(FIBRA_E_ARG, "bad arguments");
  auto* h = new fibra_network;
  const int rc = fibra_b200::generate_lattice(n_side, fibers, jitter, area, modulus, box_half,
                                              tol_bnd, seed, h->net);
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return FIBRA_OK;
}

int fibra_network_read(const char* path, double box_half, double tol_bnd, fibra_network** out) {
  auto* h = new fibra_network;
  const int rc = fibra_b200::read_network(path, box_half, tol_bnd, h->net);
  if (rc) {
    delete h;
    return rc;
  }
  *out = h;
  return FIBRA_OK;
}

int fibra_network_write(const fibra_network* net, const char* path) {
  return fibra_b200::write_network(net->net, path);
}

int fibra_network_describe(const fibra_network* net, fibra_net_desc* out) {
  if (!net || !out) return fibra_b200::fail(FIBRA_E_ARG, "bad arguments");
  fibra_b200::describe(net->net, out);
  return FIBRA_OK;
}

void fibra_network_free(fibra_network* net) { delete net; }

int fibra_assign_random(uint64_t seed, int32_t n_points, int32_t n_entries, int32_t* out) {
  if (n_entries < 1) return fibra_b200::fail(FIBRA_E_CONFIG, "RVE library is empty");
  std::mt19937_64 rng(seed);
  for (int32_t p = 0; p < n_points; ++p)
    out[p] = static_cast<int32_t>(rng() % static_cast<uint64_t>(n_entries));
  return FIBRA_OK;
}

}  // extern "C"
