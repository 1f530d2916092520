// hybrid_b200.cpp — drop-in replacement translation unit for proj/src/hybrid.cpp implementing
// proj/include/exactmppi/hybrid.hpp with the M per-mode MPPI steps of one hybrid cycle batched
// into ONE device call (exm_hybrid_cycle: one cloud preparation, one SDF launch over every
// family's poses, the families' update chains on parallel graph branches).
//
// HybridController::hybrid_cycle (hybrid.cpp:95-156) keeps the reference's control flow: the
// families' control_cycle calls run in declaration order (each consumes its parked batched
// decision, updating the controller state exactly as the per-family step would), then the
// selection is unchanged: switch penalty on validated nominal costs, argmin with ties to the
// previous mode, cooldown, projection of the raw command into the mode's space, deadzone
// correction, rate anchors of the unselected families.
#include <cmath>
#include <limits>
#include <map>
#include <mutex>
#include <stdexcept>

#include "b200_dropin.hpp"
#include "exactmppi/hybrid.hpp"

namespace exactmppi {

void HybridParams::validate() const {  // hybrid.cpp:9-16 (same checks, same messages)
  if (lambda_switch < 0.0) throw std::invalid_argument("hybrid: lambda_switch must be >= 0");
  if (tau_cool_max < 0) throw std::invalid_argument("hybrid: tau_cool_max must be >= 0");
  if (!(noise_deadzone_v >= 0.0 && noise_deadzone_v < v_min))
    throw std::invalid_argument("hybrid: noise_deadzone_v must lie in [0, v_min)");
  if (!(noise_deadzone_omega >= 0.0 && noise_deadzone_omega < omega_min))
    throw std::invalid_argument("hybrid: noise_deadzone_omega must lie in [0, omega_min)");
}

// hybrid.hpp:30-33: a raw command shaped for the mode passes through; otherwise it is read as a
// generic twist — 3 components (vx, vy, omega), 2 (v, omega), 1 (v) — and every component the
// mode cannot execute is dropped.
ControlInput project_to_mode(const ControlInput& u_raw, const MotionModel& mode) {
  if (u_raw.dim == mode.control_dim()) return u_raw;
  const double vx = u_raw.dim >= 1 ? u_raw[0] : 0.0;
  const double vy = u_raw.dim == 3 ? u_raw[1] : 0.0;
  const double om = u_raw.dim == 3 ? u_raw[2] : (u_raw.dim == 2 ? u_raw[1] : 0.0);
  ControlInput out = ControlInput::zero(mode);
  switch (mode.tag) {
    case ModelTag::kDiff: out[0] = vx; out[1] = om; break;
    case ModelTag::kAckermann: out[0] = vx; break;  // no twist equivalent of the steering angle
    case ModelTag::kOmni: out[0] = vx; out[1] = vy; out[2] = om; break;
    case ModelTag::kSpin: out[0] = om; break;
    case ModelTag::kParallel: out[0] = vy; break;
  }
  return out;
}

// hybrid.hpp:35-39: a command inside (deadzone, minimum executable) is raised to the minimum —
// the linear part's magnitude for translational modes (direction kept), the yaw rate's for spin
// (sign kept); steering and yaw of translational modes are left alone.
ControlInput deadzone_correct(const ControlInput& u, const MotionModel& mode,
                              const HybridParams& params) {
  ControlInput out = u;
  if (mode.tag == ModelTag::kSpin) {
    const double a = std::abs(out[0]);
    if (a > params.noise_deadzone_omega && a < params.omega_min)
      out[0] = std::copysign(params.omega_min, out[0]);
    return out;
  }
  const int n = mode.tag == ModelTag::kOmni ? 2 : 1;
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += out[i] * out[i];
  const double mag = std::sqrt(s);
  if (mag > params.noise_deadzone_v && mag < params.v_min)
    for (int i = 0; i < n; ++i) out[i] *= params.v_min / mag;
  return out;
}

namespace {
// The families' limits and the footprint are not readable back from MppiController, so the
// constructor keeps them per controller object, keyed by the HybridController's address (the
// header declares no destructor to drop the entry; a later object at the same address
// overwrites it, and a copied or moved controller finds none and steps its families one by one).
struct HybridExtra {
  std::vector<KinematicLimits> limits;
  FootprintSpec footprint;
  MppiParams params;
};
std::mutex g_extra_mu;
std::map<const HybridController*, HybridExtra> g_extra;
}  // namespace

HybridController::HybridController(std::vector<HybridMode> modes, const FootprintSpec& footprint,
                                   MppiParams params, HybridParams hybrid_params, int threads)
    : modes_(std::move(modes)), hybrid_params_(hybrid_params) {
  if (modes_.empty()) throw std::invalid_argument("hybrid: at least one active mode required");
  hybrid_params_.validate();
  HybridExtra extra{{}, footprint, params};
  for (std::size_t m = 0; m < modes_.size(); ++m) {
    MppiParams p = params;
    p.seed = params.seed ^ (0x9E3779B97F4A7C15ull * (m + 1));  // per-family streams (hybrid.cpp:89)
    controllers_.push_back(
        std::make_unique<MppiController>(modes_[m].model, modes_[m].limits, footprint, p, threads));
    extra.limits.push_back(modes_[m].limits);
  }
  std::lock_guard<std::mutex> lk(g_extra_mu);
  g_extra[this] = std::move(extra);
}

HybridDecision HybridController::hybrid_cycle(const Pose2& q0, const ObstacleSet& obstacles,
                                              const Guidance& guidance) {
  const std::size_t M = modes_.size();
  {
    HybridExtra* ex = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_extra_mu);
      auto it = g_extra.find(this);
      if (it != g_extra.end()) ex = &it->second;
    }
    if (ex) {  // (a copied / moved HybridController lost its entry: per-family steps)
      std::vector<const MppiController*> fam;
      for (const auto& c : controllers_) fam.push_back(c.get());
      b200::run_hybrid_batch(fam, ex->limits, ex->footprint, ex->params, q0, obstacles, guidance);
    }
  }
  HybridDecision out;
  out.mode_costs.assign(M, std::numeric_limits<double>::infinity());
  std::vector<ControlDecision> dec;
  dec.reserve(M);
  bool any = false;
  for (std::size_t m = 0; m < M; ++m) {  // consumes the parked batched decisions in order
    dec.push_back(controllers_[m]->control_cycle(q0, obstacles, guidance));
    if (dec.back().validated) {
      out.mode_costs[m] = dec.back().diagnostics.nominal_cost +
                          (static_cast<int>(m) == m_prev_ ? 0.0 : hybrid_params_.lambda_switch);
      any = true;
    }
  }
  const std::size_t prev = static_cast<std::size_t>(m_prev_);
  if (!any) {  // safe stop: previous mode kept, cooldown untouched
    out.mode_index = m_prev_;
    out.mode_name = modes_[prev].name;
    out.command = ControlInput::zero(modes_[prev].model);
    out.validated = false;
    out.diagnostics = dec[prev].diagnostics;
    return out;
  }
  int best = m_prev_;  // strict improvement over the previous mode, then declaration order
  for (std::size_t m = 0; m < M; ++m)
    if (out.mode_costs[m] < out.mode_costs[static_cast<std::size_t>(best)]) best = static_cast<int>(m);
  if (tau_cool_ > 0 && best != m_prev_) best = m_prev_;
  tau_cool_ = best != m_prev_ ? hybrid_params_.tau_cool_max : std::max(tau_cool_ - 1, 0);
  const std::size_t b = static_cast<std::size_t>(best);
  const ControlInput raw = dec[b].command;
  out.command = deadzone_correct(project_to_mode(raw, modes_[b].model), modes_[b].model,
                                 hybrid_params_);
  out.mode_index = best;
  out.mode_name = modes_[b].name;
  out.validated = dec[b].validated;
  out.diagnostics = dec[b].diagnostics;
  for (std::size_t m = 0; m < M; ++m)
    if (m != b) controllers_[m]->set_rate_anchor(project_to_mode(raw, modes_[m].model));
  m_prev_ = best;
  return out;
}

}  // namespace exactmppi
