// C++ drop-in for the reference's NetworkBatchProvider whose warm states live in HBM.
//
//   fibra_b200::NetworkBatchProvider provider(region_of_point, library, seed, law,
//                                             relax_cfg, stiff_cfg, workers);
//   fibra::newton_solve(mesh, numbering, bcs, provider, newton_cfg);
//
// Same constructors, interface and results as fibra::NetworkBatchProvider
// (/root/reference/proj/include/fibra/batch.hpp:103-129, src/batch.cpp:259-302), a
// fibra::ConstitutiveProvider (macrofem.hpp:62-70) that newton_solve (macrofem.cpp:342-370)
// calls once per Newton iteration.  The reference's provider hands its host PackedStates to
// batch_response every call, which through a device solver means uploading the warm u and
// downloading all seven state arrays each Newton iteration (1-2 GB at config 3).  This one
// uploads the library, the assignment and the initial states once; every respond() moves
// only F in and the 760-byte result records out.  states() downloads on demand and marks
// the host copy as possibly edited, so a caller that changes it gets its edit uploaded
// before the next respond().  The next respond() also starts the points that relaxed longest
// in this one first (fibra_cuda_set_schedule, FIBRA_SCHED_HINT); results do not depend on
// the order.  `workers` is accepted for signature compatibility: the GPU grid replaces the
// WorkerPool.  `devices` lists the GPUs (several: fibra_cuda_open_devices, points sharded
// across them, the warm states staying on the device that solves their point).
#pragma once

#include <cstdint>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "fibra/batch.hpp"
#include "fibra/macrofem.hpp"
#include "fibra_b200/batch_response.hpp"

namespace fibra_b200 {

class NetworkBatchProvider final : public fibra::ConstitutiveProvider {
 public:
  NetworkBatchProvider(std::span<const std::int32_t> region_of_point, fibra::RveLibrary library,
                       std::uint64_t seed, fibra::FiberLaw law, fibra::RelaxConfig relax_cfg,
                       fibra::StiffnessConfig stiff_cfg, int /*workers*/, std::vector<int32_t> devices = {0})
      : library_(std::move(library)), law_(law), relax_cfg_(relax_cfg), stiff_cfg_(stiff_cfg),
        devices_(std::move(devices)) {
    auto [states, assignment] = fibra::init_batch(region_of_point, library_, seed);
    states_ = std::move(states);
    assignment_ = std::move(assignment);
  }
  NetworkBatchProvider(const fibra::MacroMesh& mesh, fibra::RveLibrary library, std::uint64_t seed,
                       fibra::FiberLaw law, fibra::RelaxConfig relax_cfg,
                       fibra::StiffnessConfig stiff_cfg, int /*workers*/, std::vector<int32_t> devices = {0})
      : library_(std::move(library)), law_(law), relax_cfg_(relax_cfg), stiff_cfg_(stiff_cfg),
        devices_(std::move(devices)) {
    auto [states, assignment] = fibra::init_batch(mesh, library_, seed);
    states_ = std::move(states);
    assignment_ = std::move(assignment);
  }
  // States and assignment made by the caller (e.g. fibra::init_batch elsewhere).
  NetworkBatchProvider(fibra::RveLibrary library, fibra::PackedStates states,
                       fibra::BatchAssignment assignment, fibra::FiberLaw law,
                       fibra::RelaxConfig relax_cfg, fibra::StiffnessConfig stiff_cfg,
                       std::vector<int32_t> devices = {0})
      : library_(std::move(library)), states_(std::move(states)),
        assignment_(std::move(assignment)), law_(law), relax_cfg_(relax_cfg),
        stiff_cfg_(stiff_cfg), devices_(std::move(devices)) {}
  ~NetworkBatchProvider() override { fibra_cuda_close(ctx_); }
  NetworkBatchProvider(const NetworkBatchProvider&) = delete;
  NetworkBatchProvider& operator=(const NetworkBatchProvider&) = delete;

  fibra::ProviderResult respond(std::span<const fibra::Def3> deformation) override {
    const int n = states_.n_points();
    if (static_cast<int>(deformation.size()) != n)
      throw fibra::ConfigError("one deformation gradient per point is required");
    ensure_device();
    const std::vector<double> F = detail::flat_F(deformation);
    fibra_law L;
    fibra_relax_cfg R;
    fibra_stiff_cfg S;
    detail::to_cfg(law_, relax_cfg_, stiff_cfg_, L, R, S);
    std::vector<fibra_point_result> out(n);
    detail::check(fibra_cuda_solve(ctx_, F.data(), &L, &R, &S, 1, out.data()), ctx_);
    device_newer_ = true;
    // next call: longest relaxations first (failed ones ran to the cap)
    std::vector<double> cost(n);
    for (int p = 0; p < n; ++p)
      cost[p] = out[p].status == FIBRA_OK ? static_cast<double>(out[p].relax_iterations)
                : (out[p].status == FIBRA_E_NOT_CONVERGED || out[p].status == FIBRA_E_PROBE_FAILED)
                    ? 7.0 * static_cast<double>(relax_cfg_.max_iterations)
                    : 0.0;
    detail::check(fibra_cuda_set_schedule(ctx_, FIBRA_SCHED_HINT, cost.data()), ctx_);
    fibra::BatchResult br = detail::to_result(out);
    fibra::ProviderResult res;
    res.responses = std::move(br.responses);
    res.failed_points = std::move(br.failed);
    for (const fibra::ResponseStats& s : br.stats) {  // batch.cpp:286-291
      res.microscale_iterations += s.relax_iterations;
      total_solves_ += s.solves;
    }
    res.solves_per_point = br.stats.empty() ? 0 : br.stats.front().solves;
    return res;
  }

  // orientation_p2 of the point's current state (batch.cpp:296-302), on the device.
  std::optional<double> orientation(int point, const fibra::Vec3& ref_dir) const override {
    if (point < 0 || point >= states_.n_points()) return std::nullopt;
    auto& self = const_cast<NetworkBatchProvider&>(*this);
    if (!ctx_ || self.host_newer_) {  // the host copy is authoritative: reference path
      const auto& st = self.states_;  // PackedStates::view(point).u (batch.cpp:13-29)
      const std::int64_t lo = st.offsets[point], hi = st.offsets[point + 1];
      return fibra::orientation_p2(library_.entries[assignment_.entry_of_point[point]],
                                   std::span<const double>(st.u.data() + lo,
                                                           static_cast<size_t>(hi - lo)),
                                   ref_dir);
    }
    const int32_t pt = point;
    const double d[3] = {ref_dir[0], ref_dir[1], ref_dir[2]};
    double out = 0.0;
    detail::check(fibra_cuda_orientation(ctx_, &pt, 1, d, &out), ctx_);
    return out;
  }

  const fibra::BatchAssignment& assignment() const { return assignment_; }
  const fibra::RveLibrary& library() const { return library_; }
  // The warm states, downloaded from HBM when the device copy is newer.  The reference
  // returns a mutable reference, so an edit is assumed: it is uploaded before the next
  // respond().
  fibra::PackedStates& states() {
    if (ctx_ && device_newer_) {
      detail::check(fibra_cuda_download_states(ctx_, states_.u.data(), states_.v.data(),
                                               states_.a.data(), states_.f_int.data(),
                                               states_.f_damp.data(), states_.mass.data(),
                                               states_.inv_mass.data(), states_.t.data(),
                                               states_.iters.data(), states_.converged.data()),
                    ctx_);
      device_newer_ = false;
    }
    host_newer_ = true;
    return states_;
  }
  std::int64_t total_solves() const { return total_solves_; }

 private:
  void ensure_device() {
    if (!ctx_) {
      detail::Ctx c;  // owns the context until the library is on the device
      detail::check(detail::open_ctx(devices_, &c.ctx), nullptr);
      detail::upload(c, library_);
      detail::bind(c, library_, assignment_);
      detail::check_layout(c, states_);
      ctx_ = c.ctx;
      c.ctx = nullptr;
      host_newer_ = true;
    }
    if (host_newer_) {
      detail::check(fibra_cuda_upload_states(ctx_, states_.u.data(), states_.t.data(),
                                             states_.iters.data(), states_.converged.data()),
                    ctx_);
      host_newer_ = false;
    }
  }

  fibra::RveLibrary library_;
  fibra::PackedStates states_;
  fibra::BatchAssignment assignment_;
  fibra::FiberLaw law_;
  fibra::RelaxConfig relax_cfg_;
  fibra::StiffnessConfig stiff_cfg_;
  std::vector<int32_t> devices_;  // one GPU, or several of this process
  fibra_ctx* ctx_ = nullptr;
  bool device_newer_ = false;  // HBM holds states the host copy has not seen
  bool host_newer_ = true;     // the host copy may hold edits the device has not seen
  std::int64_t total_solves_ = 0;
};

}  // namespace fibra_b200
