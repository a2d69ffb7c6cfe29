// Drop-in check: the reference's own types and generator (compiled from /root/reference,
// oracle/_ref/obj) feed include/fibra_b200/batch_response.hpp, which runs on the B200
// through fibra_cuda.h; results are compared bit for bit with the oracle's batch_response.
#include <cstdio>
#include <cstring>
#include <random>
#include <span>
#include <vector>

#include "fibra/netgen.hpp"
#include "fibra_b200/batch_response.hpp"
#include "fibra_b200/network_batch_provider.hpp"
#include "fibra_oracle.h"

using namespace fibra;

static double u01(std::mt19937_64& r) { return static_cast<double>(r() >> 11) * 0x1.0p-53; }

static PackedStates fresh_states(const RveLibrary& lib, const BatchAssignment& assign) {
  const int n = static_cast<int>(assign.entry_of_point.size());
  PackedStates st;  // init_batch (batch.cpp:94-145) without the Eigen-dependent TU
  st.offsets.assign(n + 1, 0);
  for (int p = 0; p < n; ++p) {
    const FiberNetwork& net = lib.entries[assign.entry_of_point[p]];
    st.offsets[p + 1] = st.offsets[p] + net.n_dof();
    st.n_free.push_back(net.n_free());
  }
  const size_t tot = st.offsets.back();
  for (auto* v : {&st.u, &st.v, &st.a, &st.f_int, &st.f_damp, &st.mass, &st.inv_mass}) v->assign(tot, 0.0);
  st.t.assign(n, 0.0);
  st.iters.assign(n, 0);
  st.converged.assign(n, 0);
  return st;
}

static std::vector<Def3> batch_defs(int n) {
  std::vector<Def3> fs;
  std::mt19937_64 rng(55);  // test_batch.cpp:149-157
  for (int p = 0; p < n; ++p) {
    Def3 f = Def3::identity();
    f(0, 0) += 0.01 + 0.05 * u01(rng);
    f(1, 1) -= 0.0 + 0.02 * u01(rng);
    f(0, 1) += 0.0 + 0.02 * u01(rng);
    fs.push_back(f);
  }
  return fs;
}

// batch_response through the drop-in vs the oracle on `lib`: sigma, C, stats, PackedStates
static int run_case(RveLibrary& lib, uint64_t pick_seed) {
  const int n_entries = static_cast<int>(lib.entries.size());
  const int n = 8;
  BatchAssignment assign;
  std::mt19937_64 pick(pick_seed);
  for (int p = 0; p < n; ++p) assign.entry_of_point.push_back(static_cast<int32_t>(pick() % n_entries));
  PackedStates st = fresh_states(lib, assign);
  const size_t tot = st.offsets.back();
  const std::vector<Def3> fs = batch_defs(n);
  WorkerPool pool(1);
  const BatchResult br = fibra_b200::batch_response(lib, assign, st, FiberLaw{}, fs, RelaxConfig{},
                                                    StiffnessConfig{}, pool);
  // oracle
  std::vector<or_network> onets(n_entries);
  std::vector<const or_network*> optr;
  for (int e = 0; e < n_entries; ++e) {
    const FiberNetwork& net = lib.entries[e];
    std::vector<double> c(3 * net.n_nodes()), ar, mo;
    std::vector<int32_t> fa, fb;
    for (int i = 0; i < net.n_nodes(); ++i)
      for (int k = 0; k < 3; ++k) c[3 * i + k] = net.coords()[i][k];
    for (const Fiber& f : net.fibers()) {
      fa.push_back(f.a);
      fb.push_back(f.b);
      ar.push_back(f.area);
      mo.push_back(f.modulus);
    }
    if (or_network_build(c.data(), net.n_nodes(), fa.data(), fb.data(), ar.data(), mo.data(),
                         net.n_fibers(), 0.5, 1e-6, &onets[e])) return 2;
    optr.push_back(&onets[e]);
  }
  std::vector<double> u(tot, 0), v(tot, 0), a(tot, 0), fi(tot, 0), fd(tot, 0), m(tot, 0), im(tot, 0), t(n, 0);
  std::vector<int64_t> it(n, 0);
  std::vector<uint8_t> cv(n, 0);
  std::vector<double> F(9 * n);
  for (int p = 0; p < n; ++p)
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) F[9 * p + 3 * i + j] = fs[p](i, j);
  or_law law{0, 1.0, 1.2, 0};
  or_relax_cfg rc{2.0, 1e-6, 500000, 0.8, 1.0};
  std::vector<or_response> out(n);
  std::vector<int32_t> status(n);
  or_batch_response(optr.data(), assign.entry_of_point.data(), n, st.offsets.data(), u.data(), v.data(),
                    a.data(), fi.data(), fd.data(), m.data(), im.data(), t.data(), it.data(), cv.data(),
                    st.n_free.data(), &law, F.data(), &rc, 1e-5, 1, 1, 8, out.data(), status.data());
  int bad = 0;
  for (int p = 0; p < n; ++p) {
    const double s6[6] = {br.responses[p].sigma.xx, br.responses[p].sigma.yy, br.responses[p].sigma.zz,
                          br.responses[p].sigma.yz, br.responses[p].sigma.xz, br.responses[p].sigma.xy};
    bad += std::memcmp(s6, out[p].sigma, sizeof s6) != 0;
    bad += std::memcmp(&br.responses[p].spatial_c.m[0][0], out[p].spatial_c, sizeof out[p].spatial_c) != 0;
    bad += br.stats[p].solves != 7 || br.stats[p].relax_iterations != out[p].relax_iterations;
  }
  bad += !br.failed.empty();
  bad += std::memcmp(st.u.data(), u.data(), tot * 8) != 0;
  bad += std::memcmp(st.f_int.data(), fi.data(), tot * 8) != 0;
  for (auto& o : onets) or_network_free(&o);
  return bad;
}

static RveLibrary make_library(bool large) {
  RveLibrary lib;
  NetGenSpec spec;
  spec.style = NetGenSpec::Style::knn;
  spec.nodes = 14;
  spec.fibers = 38;
  spec.neighbors = 9;
  lib.entries.push_back(generate_network(spec, 101));
  spec.nodes = 12;
  spec.fibers = 32;
  lib.entries.push_back(generate_network(spec, 102));
  if (large) {  // a 1,900-fibre network: one CTA of a large resident shape
    spec.nodes = 712;
    spec.fibers = 1900;
    spec.neighbors = 10;
    lib.entries.push_back(generate_network(spec, 7));
  } else {
    spec.nodes = 20;
    spec.fibers = 56;
    spec.neighbors = 10;
    lib.entries.push_back(generate_network(spec, 31));
  }
  return lib;
}

int main() {
  int bad = 0;
  // 1. the drop-in against the oracle
  RveLibrary lib = make_library(true);
  int b = run_case(lib, 7);
  std::printf("batch_response: %d mismatches\n", b);
  bad += b;
  // 2. the same RveLibrary object edited in place: the content-keyed context re-uploads
  lib.entries = make_library(false).entries;
  b = run_case(lib, 9);
  std::printf("library edited in place: %d mismatches\n", b);
  bad += b;
  // 3. a PackedStates that does not match the library is a ConfigError, before any copy
  {
    BatchAssignment assign;
    assign.entry_of_point = {0, 1};
    PackedStates st = fresh_states(lib, assign);
    st.u.resize(st.u.size() - 3);
    const std::vector<Def3> fs = batch_defs(2);
    WorkerPool pool(1);
    bool threw = false;
    try {
      fibra_b200::batch_response(lib, assign, st, FiberLaw{}, fs, RelaxConfig{}, StiffnessConfig{}, pool);
    } catch (const ConfigError&) {
      threw = true;
    }
    std::printf("state layout mismatch throws ConfigError: %s\n", threw ? "yes" : "NO");
    bad += !threw;
  }
  // 4. device-resident provider over two Newton-like calls == batch_response on host states
  {
    BatchAssignment assign;
    assign.entry_of_point = {0, 1, 2, 0, 2, 1};
    const int n = 6;
    std::vector<Def3> f1 = batch_defs(n), f2 = f1;
    for (auto& f : f2) f(0, 0) += 0.002;
    fibra_b200::NetworkBatchProvider prov(lib, fresh_states(lib, assign), assign, FiberLaw{},
                                          RelaxConfig{}, StiffnessConfig{});
    PackedStates host = fresh_states(lib, assign);
    WorkerPool pool(1);
    int pb = 0;
    for (const auto* fs : {&f1, &f2}) {
      const ProviderResult pr = prov.respond(*fs);
      const BatchResult br = fibra_b200::batch_response(lib, assign, host, FiberLaw{}, *fs,
                                                        RelaxConfig{}, StiffnessConfig{}, pool);
      pb += pr.failed_points != br.failed;
      for (int p = 0; p < n; ++p) {
        pb += std::memcmp(&pr.responses[p].sigma, &br.responses[p].sigma, sizeof(SymTensor3)) != 0;
        pb += std::memcmp(&pr.responses[p].spatial_c, &br.responses[p].spatial_c, sizeof(Mandel66)) != 0;
      }
    }
    PackedStates& ps = prov.states();
    pb += std::memcmp(ps.u.data(), host.u.data(), host.u.size() * 8) != 0;
    pb += std::memcmp(ps.f_int.data(), host.f_int.data(), host.f_int.size() * 8) != 0;
    pb += ps.iters != host.iters;
    std::printf("device-resident provider (2 calls): %d mismatches, warm iterations %lld\n", pb,
                static_cast<long long>(ps.iters[0]));
    bad += pb;
  }
  // 5. several GPUs of this process (fibra_cuda_open_devices) == one GPU, bit for bit
  int ndev = 0;
  fibra_cuda_device_count(&ndev);
  if (ndev >= 2) {
    BatchAssignment assign;
    for (int p = 0; p < 10; ++p) assign.entry_of_point.push_back(p % 3);
    const std::vector<Def3> fs = batch_defs(10);
    PackedStates s1 = fresh_states(lib, assign), s2 = fresh_states(lib, assign);
    WorkerPool pool(1);
    const BatchResult b1 = fibra_b200::batch_response(lib, assign, s1, FiberLaw{}, fs,
                                                      RelaxConfig{}, StiffnessConfig{}, pool, 0);
    const BatchResult b2 = fibra_b200::batch_response(lib, assign, s2, FiberLaw{}, fs,
                                                      RelaxConfig{}, StiffnessConfig{}, pool,
                                                      std::vector<int32_t>{0, 1});
    int mb = b1.failed != b2.failed;
    for (int p = 0; p < 10; ++p) {
      mb += std::memcmp(&b1.responses[p], &b2.responses[p], sizeof(PointResponse)) != 0;
      mb += b1.stats[p].relax_iterations != b2.stats[p].relax_iterations;
    }
    mb += s1.u != s2.u || s1.f_int != s2.f_int || s1.iters != s2.iters;
    std::printf("two GPUs in one process vs one GPU: %d mismatches\n", mb);
    bad += mb;
  }
  std::printf("%s: %d mismatches (sigma, C, stats, PackedStates, provider)\n", bad ? "FAIL" : "OK", bad);
  return bad ? 1 : 0;
}
