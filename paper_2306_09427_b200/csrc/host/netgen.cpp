// Deterministic synthetic RVE networks for the B200 solver (product host code).
//
// Output-identical to the reference generator generate_network (proj/src/netgen.cpp:
// knn :162-274, segments :136-160, uniform01 :33-35, sample_direction :37-50) for every
// spec and seed -- same mt19937_64 draw order, same floating-point expressions -- but
// with the O(N^2) proximity scans replaced by a uniform grid that returns the same
// answer (existence test for point rejection, lowest index for endpoint merging), and
// the per-node full neighbour sort replaced by a partial sort of the same total order
// (metric, j).  This is the "network generation at scale" row: configs
// 3-4 need tens of thousands of networks.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <numeric>
#include <random>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "host_internal.hpp"

namespace fibra_b200 {
namespace {

struct V3 {
  double x[3];
  double& operator[](int k) { return x[k]; }
  double operator[](int k) const { return x[k]; }
};

inline double norm3(const V3& d) { return std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]); }
inline double dot3(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline V3 sub(const V3& a, const V3& b) { return {{a[0] - b[0], a[1] - b[1], a[2] - b[2]}}; }

inline double u01(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

// Uniform grid over the box; cells slightly wider than the query radius so a point within
// the radius is always in one of the 27 neighbouring cells despite rounding in floor().
class Grid {
 public:
  Grid(double half, double radius) : half_(half), active_(radius > 0) {
    if (!active_) return;
    cell_ = radius * (1.0 + 1e-9);
    dim_ = std::max<int64_t>(1, std::min<int64_t>(1 << 20, static_cast<int64_t>(2.0 * half / cell_) + 1));
  }
  bool active() const { return active_; }
  int64_t key(const V3& p) const {
    int64_t c[3];
    for (int k = 0; k < 3; ++k) c[k] = coord(p[k]);
    return (c[0] * (dim_ + 2) + c[1]) * (dim_ + 2) + c[2];
  }
  void insert(const V3& p, int32_t id) { cells_[key(p)].push_back(id); }
  template <class Fn>
  void visit(const V3& p, Fn&& fn) const {  // fn(id) over the 27 neighbouring cells
    int64_t c[3];
    for (int k = 0; k < 3; ++k) c[k] = coord(p[k]);
    for (int64_t i = c[0] - 1; i <= c[0] + 1; ++i)
      for (int64_t j = c[1] - 1; j <= c[1] + 1; ++j)
        for (int64_t k = c[2] - 1; k <= c[2] + 1; ++k) {
          auto it = cells_.find((i * (dim_ + 2) + j) * (dim_ + 2) + k);
          if (it == cells_.end()) continue;
          for (int32_t id : it->second) fn(id);
        }
  }

 private:
  int64_t coord(double v) const {
    int64_t c = static_cast<int64_t>(std::floor((v + half_) / cell_)) + 1;
    return std::clamp<int64_t>(c, 0, dim_ + 1);
  }
  double half_, cell_ = 1;
  bool active_;
  int64_t dim_ = 1;
  std::unordered_map<int64_t, std::vector<int32_t>> cells_;
};

int validate(const fibra_netgen_spec& s) {  // NetGenSpec::validate netgen.cpp:12-24
  if (s.fibers < 1) return fail(FIBRA_E_CONFIG, "netgen: fiber count must be >= 1");
  if (s.style == 1 && s.nodes < 2) return fail(FIBRA_E_CONFIG, "netgen: knn style needs >= 2 nodes");
  if (s.style == 0 && !(s.half_length > 0)) return fail(FIBRA_E_CONFIG, "netgen: half_length must be > 0");
  if (!(s.merge_radius >= 0)) return fail(FIBRA_E_CONFIG, "netgen: merge_radius must be >= 0");
  if (s.neighbors < 1) return fail(FIBRA_E_CONFIG, "netgen: neighbors must be >= 1");
  if (!(s.fiber_area > 0) || !(s.fiber_modulus > 0))
    return fail(FIBRA_E_CONFIG, "netgen: fiber section data must be > 0");
  if (s.align_bias < 0) return fail(FIBRA_E_CONFIG, "netgen: align_bias must be >= 0");
  const V3 ax{{s.align_axis[0], s.align_axis[1], s.align_axis[2]}};
  if (!(norm3(ax) > 0)) return fail(FIBRA_E_CONFIG, "netgen: align_axis is zero");
  return FIBRA_OK;
}

// direction with density ~ exp(bias (d.axis)^2), rejection sampled (netgen.cpp:37-50)
V3 direction(std::mt19937_64& rng, double bias, const V3& axis) {
  const double an = norm3(axis);
  const V3 ax{{axis[0] / an, axis[1] / an, axis[2] / an}};
  for (;;) {
    const double z = 2.0 * u01(rng) - 1.0;
    const double phi = 2.0 * 3.14159265358979323846 * u01(rng);
    const double r = std::sqrt(std::max(0.0, 1.0 - z * z));
    const V3 d{{r * std::cos(phi), r * std::sin(phi), z}};
    if (bias == 0.0) return d;
    const double c = dot3(d, ax);
    if (u01(rng) <= std::exp(bias * (c * c - 1.0))) return d;
  }
}

// segment clipping to the closed box with face snapping (netgen.cpp:88-134)
bool clip(V3& p0, V3& p1, double h) {
  double t0 = 0, t1 = 1;
  int face0 = -1, face1 = -1;
  for (int k = 0; k < 3; ++k) {
    const double d = p1[k] - p0[k];
    for (int sgn = -1; sgn <= 1; sgn += 2) {
      const double num = sgn * h - p0[k];
      if (d * sgn == 0.0) {
        if (p0[k] * sgn > h) return false;
        continue;
      }
      const double t = num / d;
      const int face = 2 * k + (sgn > 0 ? 1 : 0);
      if (d * sgn > 0) {
        if (t < t1) { t1 = t; face1 = face; }
      } else if (t > t0) {
        t0 = t;
        face0 = face;
      }
    }
  }
  if (t0 >= t1) return false;
  V3 q0, q1;
  for (int k = 0; k < 3; ++k) {
    q0[k] = p0[k] + t0 * (p1[k] - p0[k]);
    q1[k] = p0[k] + t1 * (p1[k] - p0[k]);
  }
  p0 = q0;
  p1 = q1;
  if (face0 >= 0) p0[face0 / 2] = (face0 % 2 ? h : -h);
  if (face1 >= 0) p1[face1 / 2] = (face1 % 2 ? h : -h);
  for (int k = 0; k < 3; ++k) {
    p0[k] = std::clamp(p0[k], -h, h);
    p1[k] = std::clamp(p1[k], -h, h);
  }
  return true;
}

inline uint64_t edge_key(int32_t a, int32_t b) {
  return (static_cast<uint64_t>(std::min(a, b)) << 32) | static_cast<uint32_t>(std::max(a, b));
}

int finish(std::vector<V3>& pts, std::vector<int32_t>& fn, const fibra_netgen_spec& s, Network& net) {
  std::vector<double> coords(3 * pts.size());
  for (size_t i = 0; i < pts.size(); ++i)
    for (int k = 0; k < 3; ++k) coords[3 * i + k] = pts[i][k];
  const size_t m = fn.size() / 2;
  return build_network(std::move(coords), std::move(fn), std::vector<double>(m, s.fiber_area),
                       std::vector<double>(m, s.fiber_modulus), s.box_half, s.tol_bnd, net);
}

int segments(const fibra_netgen_spec& s, uint64_t seed, Network& net) {
  std::mt19937_64 rng(seed);
  const double h = s.box_half;
  const V3 axis{{s.align_axis[0], s.align_axis[1], s.align_axis[2]}};
  std::vector<V3> pts;
  std::vector<int32_t> fn;
  std::unordered_set<uint64_t> edges;
  Grid grid(h, s.merge_radius);
  auto find_merge = [&](const V3& p) -> int32_t {  // lowest index within the radius
    int32_t best = -1;
    if (grid.active()) {
      grid.visit(p, [&](int32_t i) {
        if ((best < 0 || i < best) && norm3(sub(pts[i], p)) <= s.merge_radius) best = i;
      });
    } else {
      for (size_t i = 0; i < pts.size(); ++i)
        if (norm3(sub(pts[i], p)) <= s.merge_radius) return static_cast<int32_t>(i);
    }
    return best;
  };
  auto add_point = [&](const V3& p) {
    pts.push_back(p);
    if (grid.active()) grid.insert(p, static_cast<int32_t>(pts.size() - 1));
    return static_cast<int32_t>(pts.size() - 1);
  };
  int placed = 0;
  long attempts = 0;
  const long max_attempts = 10000L * s.fibers + 10000;
  while (placed < s.fibers) {
    if (++attempts > max_attempts)
      return fail(FIBRA_E_CONFIG, "netgen: segment placement stalled; relax the spec");
    V3 mid;
    for (int k = 0; k < 3; ++k) mid[k] = h * (2 * u01(rng) - 1);
    const V3 dir = direction(rng, s.align_bias, axis);
    V3 p0, p1;
    for (int k = 0; k < 3; ++k) {
      p0[k] = mid[k] - s.half_length * dir[k];
      p1[k] = mid[k] + s.half_length * dir[k];
    }
    if (!clip(p0, p1, h)) continue;
    if (norm3(sub(p1, p0)) <= 2.0 * s.merge_radius + 1e-12) continue;
    int32_t a = find_merge(p0), b = find_merge(p1);
    if (a >= 0 && a == b) continue;
    if (a >= 0 && b >= 0 && edges.count(edge_key(a, b))) continue;
    if (a < 0) a = add_point(p0);
    if (b < 0) b = add_point(p1);
    edges.insert(edge_key(a, b));
    fn.push_back(a);
    fn.push_back(b);
    ++placed;
  }
  return finish(pts, fn, s, net);
}

int knn(const fibra_netgen_spec& s, uint64_t seed, Network& net) {
  std::mt19937_64 rng(seed);
  const double h = s.box_half;
  const double snap = 0.12 * 2.0 * h;
  const int n = s.nodes;
  std::vector<V3> pts;
  pts.reserve(n);
  Grid grid(h, s.merge_radius);
  while (static_cast<int>(pts.size()) < n) {  // Poisson points with face snapping
    V3 p;
    for (int k = 0; k < 3; ++k) p[k] = h * (2 * u01(rng) - 1);
    for (int k = 0; k < 3; ++k) {
      if (p[k] > h - snap) p[k] = h;
      if (p[k] < -h + snap) p[k] = -h;
    }
    bool close = false;
    if (grid.active())
      grid.visit(p, [&](int32_t i) { close = close || norm3(sub(p, pts[i])) < s.merge_radius; });
    if (close) continue;
    pts.push_back(p);
    if (grid.active()) grid.insert(p, static_cast<int32_t>(pts.size() - 1));
  }

  const V3 axis{{s.align_axis[0], s.align_axis[1], s.align_axis[2]}};
  const double an = norm3(axis);
  const V3 ax{{axis[0] / an, axis[1] / an, axis[2] / an}};
  const double shrink = std::exp(-s.align_bias);
  auto metric = [&](int i, int j) {
    V3 d = sub(pts[j], pts[i]);
    const double axial = dot3(d, ax);
    for (int k = 0; k < 3; ++k) d[k] += (shrink - 1.0) * axial * ax[k];
    return norm3(d);
  };

  struct Cand {
    double len;
    int32_t a, b;
  };
  std::vector<Cand> cands;
  std::unordered_set<uint64_t> seen;
  const int kk = std::min(s.neighbors, n - 1);
  std::vector<std::pair<double, int>> near(n > 0 ? n - 1 : 0);
  for (int i = 0; i < n; ++i) {
    int c = 0;
    for (int j = 0; j < n; ++j)
      if (j != i) near[c++] = {metric(i, j), j};
    std::partial_sort(near.begin(), near.begin() + kk, near.end());
    for (int k = 0; k < kk; ++k) {
      const int j = near[k].second;
      if (seen.insert(edge_key(i, j)).second)
        cands.push_back({near[k].first, std::min(i, j), std::max(i, j)});
    }
  }
  std::sort(cands.begin(), cands.end(), [](const Cand& x, const Cand& y) {
    if (x.len != y.len) return x.len < y.len;
    if (x.a != y.a) return x.a < y.a;
    return x.b < y.b;
  });
  if (static_cast<int>(cands.size()) < s.fibers)
    return fail(FIBRA_E_CONFIG, "netgen: knn candidate pool too small; raise neighbors");

  // cover every node with its shortest unused candidate, then fill shortest-first
  std::vector<std::vector<int32_t>> touching(n);
  for (size_t c = 0; c < cands.size(); ++c) {
    touching[cands[c].a].push_back(static_cast<int32_t>(c));
    touching[cands[c].b].push_back(static_cast<int32_t>(c));
  }
  std::vector<int> degree(n, 0);
  std::vector<char> used(cands.size(), 0);
  std::vector<int32_t> chosen;
  for (int i = 0; i < n; ++i) {
    if (degree[i] > 0) continue;
    for (int32_t c : touching[i]) {
      if (used[c]) continue;
      used[c] = 1;
      chosen.push_back(c);
      ++degree[cands[c].a];
      ++degree[cands[c].b];
      break;
    }
  }
  if (static_cast<int>(chosen.size()) > s.fibers)
    return fail(FIBRA_E_CONFIG, "netgen: fiber budget below node-coverage minimum");
  for (size_t c = 0; c < cands.size() && static_cast<int>(chosen.size()) < s.fibers; ++c)
    if (!used[c]) {
      used[c] = 1;
      chosen.push_back(static_cast<int32_t>(c));
    }
  std::vector<int32_t> fn;
  fn.reserve(2 * chosen.size());
  for (int32_t c : chosen) {
    fn.push_back(cands[c].a);
    fn.push_back(cands[c].b);
  }
  int rc = finish(pts, fn, s, net);
  if (rc) return rc;

  // every connected component must touch the boundary (netgen.cpp:259-273)
  std::vector<int> root(n);
  std::iota(root.begin(), root.end(), 0);
  auto find = [&](int x) {
    while (root[x] != x) x = root[x] = root[root[x]];
    return x;
  };
  for (int f = 0; f < net.n_fibers; ++f)
    root[find(net.fiber_nodes[2 * f])] = find(net.fiber_nodes[2 * f + 1]);
  std::vector<char> attached(n, 0);
  for (int32_t bn : net.boundary_nodes) attached[find(bn)] = 1;
  for (int i = 0; i < n; ++i)
    if (!attached[find(i)])
      return fail(FIBRA_E_CONFIG, "netgen: component without boundary attachment (node " +
                                      std::to_string(i) + "); try another seed");
  return FIBRA_OK;
}

}  // namespace

// Builder-side jittered lattice for config-4 sized RVEs (the reference knn
// generator fails beyond ~6k nodes).  n^3 nodes on a cube lattice spanning the box; face
// nodes sit exactly on their face (so FiberNetwork's boundary test, network.cpp:110-117,
// finds them) and are jittered only tangentially; interior nodes are jittered by up to
// `jitter` lattice spacings per axis.  Fibers: every axis bond, then face diagonals drawn
// without replacement (mt19937_64(seed) shuffle) up to `fibers`.  The result goes through
// the same construction as a file read (build_network), so it can be written in the
// reference format and re-read there.
int generate_lattice(int n, int fibers, double jitter, double area, double modulus,
                     double box_half, double tol_bnd, uint64_t seed, Network& net) {
  if (n < 2 || !(jitter >= 0 && jitter < 0.5) || !(box_half > 0) || !(area > 0) ||
      !(modulus > 0))
    return fail(FIBRA_E_CONFIG, "lattice: need n >= 2, 0 <= jitter < 0.5, positive box/area/modulus");
  std::mt19937_64 rng(seed);
  const double a = 2.0 * box_half / (n - 1);
  auto id = [n](int i, int j, int k) { return (i * n + j) * n + k; };
  std::vector<double> coords(3 * static_cast<size_t>(n) * n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        const int idx[3] = {i, j, k};
        for (int ax = 0; ax < 3; ++ax) {
          double x = -box_half + idx[ax] * a;
          if (idx[ax] == 0) x = -box_half;
          else if (idx[ax] == n - 1) x = box_half;
          else x += jitter * a * (2.0 * u01(rng) - 1.0);
          coords[3 * static_cast<size_t>(id(i, j, k)) + ax] = x;
        }
      }
  std::vector<int32_t> fn;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        const int v = id(i, j, k);
        if (i + 1 < n) fn.insert(fn.end(), {v, id(i + 1, j, k)});
        if (j + 1 < n) fn.insert(fn.end(), {v, id(i, j + 1, k)});
        if (k + 1 < n) fn.insert(fn.end(), {v, id(i, j, k + 1)});
      }
  const int axis_bonds = static_cast<int>(fn.size() / 2);
  if (fibers < axis_bonds)
    return fail(FIBRA_E_CONFIG, "lattice: fibers below the " + std::to_string(axis_bonds) +
                                    " axis bonds of an n^3 lattice");
  std::vector<std::pair<int32_t, int32_t>> diag;  // both diagonals of every lattice square
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) {
        if (i + 1 < n && j + 1 < n) {
          diag.push_back({id(i, j, k), id(i + 1, j + 1, k)});
          diag.push_back({id(i + 1, j, k), id(i, j + 1, k)});
        }
        if (j + 1 < n && k + 1 < n) {
          diag.push_back({id(i, j, k), id(i, j + 1, k + 1)});
          diag.push_back({id(i, j + 1, k), id(i, j, k + 1)});
        }
        if (i + 1 < n && k + 1 < n) {
          diag.push_back({id(i, j, k), id(i + 1, j, k + 1)});
          diag.push_back({id(i + 1, j, k), id(i, j, k + 1)});
        }
      }
  const size_t extra = static_cast<size_t>(fibers - axis_bonds);
  if (extra > diag.size())
    return fail(FIBRA_E_CONFIG, "lattice: more fibers than axis bonds plus face diagonals");
  for (size_t i = 0; i < extra; ++i) {  // partial Fisher-Yates
    const size_t r = i + static_cast<size_t>(rng() % (diag.size() - i));
    std::swap(diag[i], diag[r]);
  }
  std::sort(diag.begin(), diag.begin() + static_cast<long>(extra));
  for (size_t i = 0; i < extra; ++i) fn.insert(fn.end(), {diag[i].first, diag[i].second});
  const size_t m = fn.size() / 2;
  return build_network(std::move(coords), std::move(fn), std::vector<double>(m, area),
                       std::vector<double>(m, modulus), box_half, tol_bnd, net);
}

int generate_network(const fibra_netgen_spec& spec, uint64_t seed, Network& net) {
  const int rc = validate(spec);
  if (rc) return rc;
  return spec.style == 0 ? segments(spec, seed, net) : knn(spec, seed, net);
}

}  // namespace fibra_b200
