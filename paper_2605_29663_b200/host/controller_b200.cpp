// controller_b200.cpp — drop-in replacement translation unit for the reference's
// proj/src/controller.cpp. It implements every declaration of
// proj/include/exactmppi/controller.hpp, with the hot path (sample_perturbations,
// evaluate_rollouts, validate_nominal, MppiController::control_cycle) marshalled into the
// B200 C ABI (include/exm_b200.h, libexm_b200.so). Link it with the reference's other
// sources (geometry, kinematics, hybrid, world, ...) in place of controller.cpp:
//
//   g++ -std=c++20 -O3 -I<ref>/proj/include -I<repo>/include controller_b200.cpp \
//       <ref>/proj/src/{geometry,kinematics,hybrid,world,...}.cpp -L<repo>/.../lib -lexm_b200
//
// The class layout of MppiController is fixed by the reference header (no slot for a device
// handle, no user destructor), so device handles live in a process-wide cache keyed by the
// controller configuration; the controller's own state (nominal_, u_prev_,
// cycle_) stays in the object and crosses the ABI per call.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "exactmppi/controller.hpp"
#include "exm_b200.h"

namespace exactmppi {
namespace {

// ---------------------------------------------------------------- ABI marshalling
void throw_status(exm_status st) {
  if (st == EXM_OK) return;
  if (st == EXM_ERR_INVALID_ARGUMENT) throw std::invalid_argument(exm_last_error());
  throw std::runtime_error(std::string("exm_b200: ") + exm_last_error());
}

struct Config {
  exm_footprint fp{};
  std::vector<double> x, y, hx, hy;
  exm_model model{};
  exm_limits limits{};
  exm_params params{};
  std::string key;
};

Config make_config(const PreparedFootprint& f, const MotionModel& m, const KinematicLimits& l,
                   const MppiParams& p) {
  Config c;
  if (f.kind == PreparedFootprint::Kind::kPolygon) {
    c.x = f.vx;  // prepare() keeps the (CCW) vertices as edge origins (geometry.cpp:241-242)
    c.y = f.vy;
    c.fp.kind = EXM_FOOTPRINT_POLYGON;
  } else {
    c.x = f.cx;
    c.y = f.cy;
    c.hx = f.hx;
    c.hy = f.hy;
    c.fp.kind = EXM_FOOTPRINT_RECT_COVER;
  }
  c.fp.count = static_cast<int32_t>(c.x.size());
  c.fp.x = c.x.data();
  c.fp.y = c.y.data();
  c.fp.hx = c.hx.empty() ? nullptr : c.hx.data();
  c.fp.hy = c.hy.empty() ? nullptr : c.hy.data();
  c.model.tag = static_cast<int32_t>(m.tag);
  c.model.wheelbase = m.wheelbase;
  for (int i = 0; i < 3; ++i) {
    c.limits.vel_min[i] = l.component[i].vel_min;
    c.limits.vel_max[i] = l.component[i].vel_max;
    c.limits.acc_min[i] = l.component[i].acc_min;
    c.limits.acc_max[i] = l.component[i].acc_max;
    c.params.sigma[i] = p.sigma[i];
  }
  c.limits.steer_max = l.steer_max;
  c.params.rollouts = p.rollouts;
  c.params.horizon = p.horizon;
  c.params.dt = p.dt;
  c.params.lambda = p.lambda;
  c.params.d_safe = p.d_safe;
  c.params.w_coll = p.w_coll;
  c.params.w_rep = p.w_rep;
  c.params.w_inf = p.w_inf;
  c.params.w_goal_pos = p.task.goal_pos;
  c.params.w_goal_head = p.task.goal_head;
  c.params.w_xtrack = p.task.xtrack;
  c.params.w_progress = p.task.progress;
  c.params.w_ctrl = p.w_ctrl;
  c.params.seed = p.seed;
  std::ostringstream k;
  k.precision(17);
  k << c.fp.kind << ':';
  for (std::size_t i = 0; i < c.x.size(); ++i)
    k << c.x[i] << ',' << c.y[i] << ',' << (c.hx.empty() ? 0.0 : c.hx[i]) << ','
      << (c.hy.empty() ? 0.0 : c.hy[i]) << ';';
  const unsigned char* raw[] = {reinterpret_cast<const unsigned char*>(&c.model),
                                reinterpret_cast<const unsigned char*>(&c.limits),
                                reinterpret_cast<const unsigned char*>(&c.params)};
  const std::size_t len[] = {sizeof c.model, sizeof c.limits, sizeof c.params};
  for (int b = 0; b < 3; ++b)
    for (std::size_t i = 0; i < len[b]; ++i) k << std::hex << static_cast<int>(raw[b][i]);
  c.key = k.str();
  return c;
}

struct Cached {
  exm_handle* h = nullptr;
  int n_cap = 0;
  int guide_cap = 0;
  ~Cached() {
    if (h) exm_destroy(h);
  }
};

std::mutex g_mu;
std::map<std::string, std::unique_ptr<Cached>> g_cache;

// Handle for this configuration with room for n points and g guidance vertices.
exm_handle* handle_for(const Config& c, int n, int g) {
  std::lock_guard<std::mutex> lock(g_mu);
  auto& slot = g_cache[c.key];
  if (!slot) slot = std::make_unique<Cached>();
  if (!slot->h || slot->n_cap < n || slot->guide_cap < g) {
    if (slot->h) exm_destroy(slot->h);
    slot->h = nullptr;
    const int ncap = std::max(n, std::max(1024, 2 * slot->n_cap));
    const int gcap = std::max(g, 64);
    throw_status(exm_create(&c.fp, &c.model, &c.limits, &c.params, ncap, gcap, -1, &slot->h));
    slot->n_cap = ncap;
    slot->guide_cap = gcap;
  }
  return slot->h;
}

// A unit-square footprint for the footprint-free entry points (sample_perturbations).
PreparedFootprint square_footprint() {
  PreparedFootprint f;
  f.kind = PreparedFootprint::Kind::kPolygon;
  f.vx = {0, 1, 1, 0};
  f.vy = {0, 0, 1, 1};
  return f;
}

struct Flat {
  std::vector<double> pts;
  std::vector<uint8_t> mask;
  std::vector<double> guide;
  double goal[3];
};

Flat flatten(const ObstacleSet& o, const Guidance& g) {
  Flat f;
  f.pts.resize(2 * o.points.size());
  for (std::size_t i = 0; i < o.points.size(); ++i) {
    f.pts[2 * i] = o.points[i].x;
    f.pts[2 * i + 1] = o.points[i].y;
  }
  f.mask = o.mask;
  if (g.path.empty()) throw std::invalid_argument("guidance polyline is empty");
  for (const auto& p : g.path) {
    f.guide.push_back(p.x);
    f.guide.push_back(p.y);
  }
  f.goal[0] = g.goal.x;
  f.goal[1] = g.goal.y;
  f.goal[2] = g.goal.theta;
  return f;
}

std::vector<double> flat_controls(const std::vector<ControlInput>& u, int dim) {
  std::vector<double> out(u.size() * dim);
  for (std::size_t i = 0; i < u.size(); ++i)
    for (int c = 0; c < dim; ++c) out[i * dim + c] = u[i][c];
  return out;
}

std::vector<ControlInput> unflat_controls(const double* v, std::size_t n, const MotionModel& m) {
  const int dim = m.control_dim();
  std::vector<ControlInput> out(n, ControlInput::zero(m));
  for (std::size_t i = 0; i < n; ++i)
    for (int c = 0; c < dim; ++c) out[i][c] = v[i * dim + c];
  return out;
}

struct PolyHit {
  double distance;
  double progress;
};

// Nearest point on the guidance polyline (first nearest segment wins; SPEC.md §controller).
PolyHit nearest_on_path(Point2 p, std::span<const Point2> path) {
  if (path.empty()) throw std::invalid_argument("guidance polyline is empty");
  if (path.size() == 1) return {norm(p - path[0]), 0.0};
  PolyHit best{std::numeric_limits<double>::infinity(), 0.0};
  double walked = 0.0;
  for (std::size_t i = 1; i < path.size(); ++i) {
    const Point2 a = path[i - 1], seg = path[i] - a;
    const double len = norm(seg);
    const double t = len > 0.0 ? std::clamp(dot(p - a, seg) / (len * len), 0.0, 1.0) : 0.0;
    const double d = norm(p - (a + t * seg));
    if (d < best.distance) best = {d, walked + t * len};
    walked += len;
  }
  return best;
}

}  // namespace

// ---------------------------------------------------------------- scalar API (host)
void MppiParams::validate() const {
  if (rollouts < 1) throw std::invalid_argument("mppi: rollouts must be >= 1");
  if (horizon < 1) throw std::invalid_argument("mppi: horizon must be >= 1");
  if (dt <= 0.0) throw std::invalid_argument("mppi: dt must be positive");
  if (lambda <= 0.0) throw std::invalid_argument("mppi: lambda must be positive");
  for (double s : sigma)
    if (s <= 0.0) throw std::invalid_argument("mppi: sigma components must be positive");
  if (d_safe < 0.0) throw std::invalid_argument("mppi: d_safe must be nonnegative");
  if (w_coll < 0.0 || w_rep < 0.0 || w_inf < 0.0)
    throw std::invalid_argument("mppi: penalty weights must be nonnegative");
}

NominalSequence NominalSequence::zero(const MotionModel& model, int horizon) {
  return constant(ControlInput::zero(model), horizon);
}

NominalSequence NominalSequence::constant(const ControlInput& u, int horizon) {
  NominalSequence s;
  s.controls.assign(static_cast<std::size_t>(horizon), u);
  return s;
}

double polyline_length(std::span<const Point2> path) {
  double total = 0.0;
  for (std::size_t i = 1; i < path.size(); ++i) total += norm(path[i] - path[i - 1]);
  return total;
}

double polyline_distance(Point2 p, std::span<const Point2> path) {
  return nearest_on_path(p, path).distance;
}

double polyline_progress(Point2 p, std::span<const Point2> path) {
  return nearest_on_path(p, path).progress;
}

double obstacle_cost(double d, const MppiParams& params) {
  const double m = std::max(params.d_safe - d, 0.0);
  return params.w_coll * (d < 0.0 ? 1.0 : 0.0) + params.w_rep * m * m;
}

double task_cost(const Pose2& q, const ControlInput&, const Guidance& guidance,
                 const TaskWeights& w, bool terminal) {
  const double gx = q.x - guidance.goal.x, gy = q.y - guidance.goal.y;
  double cost = w.goal_pos * (gx * gx + gy * gy);
  if (terminal) {
    const double e = wrap_angle(q.theta - guidance.goal.theta);
    cost += w.goal_head * e * e;
  }
  const PolyHit hit = nearest_on_path({q.x, q.y}, guidance.path);
  return cost + w.xtrack * hit.distance * hit.distance - w.progress * hit.progress;
}

double terminal_goal_cost(const Pose2& q, const Guidance& guidance, const TaskWeights& w) {
  const double gx = q.x - guidance.goal.x, gy = q.y - guidance.goal.y;
  const double e = wrap_angle(q.theta - guidance.goal.theta);
  return w.goal_pos * (gx * gx + gy * gy) + w.goal_head * e * e;
}

double control_cost(const ControlInput& u, const MppiParams& params) {
  double s = 0.0;
  for (int i = 0; i < u.dim; ++i) s += u[i] * u[i];
  return params.w_ctrl * s;
}

std::vector<double> weights_from_costs(std::span<const double> costs, double lambda) {
  if (costs.empty()) throw std::invalid_argument("weights need at least one cost");
  const double beta = *std::min_element(costs.begin(), costs.end());
  std::vector<double> w(costs.size());
  double total = 0.0;
  for (std::size_t r = 0; r < costs.size(); ++r) total += (w[r] = std::exp(-(costs[r] - beta) / lambda));
  for (double& x : w) x /= total;
  return w;
}

NominalSequence path_integral_update(const NominalSequence& nominal,
                                     std::span<const ControlInput> eps,
                                     std::span<const double> costs, double lambda) {
  const std::size_t K = costs.size(), T = nominal.controls.size();
  if (eps.size() != K * T) throw std::invalid_argument("perturbation array does not match K*T");
  const auto w = weights_from_costs(costs, lambda);
  NominalSequence out = nominal;
  for (std::size_t h = 0; h < T; ++h)
    for (std::size_t r = 0; r < K; ++r)
      for (int c = 0; c < out.controls[h].dim; ++c) out.controls[h][c] += w[r] * eps[r * T + h][c];
  return out;
}

// ---------------------------------------------------------------- hot path (B200)
std::vector<ControlInput> sample_perturbations(std::uint64_t seed, std::uint64_t cycle,
                                               const MotionModel& model, const MppiParams& params) {
  params.validate();
  const Config c = make_config(square_footprint(), model, KinematicLimits{}, params);
  exm_handle* h = handle_for(c, 1, 1);
  const std::size_t n = static_cast<std::size_t>(params.rollouts) * params.horizon;
  std::vector<double> flat(n * model.control_dim());
  throw_status(exm_sample_perturbations(h, seed, cycle, flat.data()));
  return unflat_controls(flat.data(), n, model);
}

RolloutBatch evaluate_rollouts(const Pose2& q0, const NominalSequence& nominal,
                               std::span<const ControlInput> perturbations,
                               const ObstacleSet& obstacles, const PreparedFootprint& footprint,
                               const MotionModel& model, const KinematicLimits& limits,
                               const MppiParams& params, const Guidance& guidance,
                               const ControlInput& u_prev, int /*threads*/) {
  params.validate();
  const int K = params.rollouts, T = params.horizon, D = model.control_dim();
  if (static_cast<int>(nominal.controls.size()) != T)
    throw std::invalid_argument("nominal length does not match horizon");
  if (perturbations.size() != static_cast<std::size_t>(K) * T)
    throw std::invalid_argument("perturbation array does not match K*T");
  const Config c = make_config(footprint, model, limits, params);
  const Flat f = flatten(obstacles, guidance);
  exm_handle* h = handle_for(c, static_cast<int>(obstacles.points.size()),
                             static_cast<int>(guidance.path.size()));
  const std::vector<double> eps = flat_controls({perturbations.begin(), perturbations.end()}, D);
  const std::vector<double> nom = flat_controls(nominal.controls, D);
  const double q[3] = {q0.x, q0.y, q0.theta};
  const double up[3] = {u_prev[0], u_prev[1], u_prev[2]};
  RolloutBatch b;
  b.rollouts = K;
  b.horizon = T;
  b.perturbations.assign(perturbations.begin(), perturbations.end());
  std::vector<double> controls(static_cast<std::size_t>(K) * T * D), states(static_cast<std::size_t>(K) * (T + 1) * 3);
  b.d_min.resize(static_cast<std::size_t>(K) * T);
  b.costs.resize(K);
  b.unsafe.resize(K);
  throw_status(exm_evaluate_rollouts(h, q, nom.data(), eps.data(), f.pts.data(), f.mask.data(),
                                     static_cast<int32_t>(obstacles.points.size()), f.guide.data(),
                                     static_cast<int32_t>(guidance.path.size()), f.goal, up,
                                     controls.data(), states.data(), b.d_min.data(),
                                     b.costs.data(), b.unsafe.data()));
  b.controls = unflat_controls(controls.data(), static_cast<std::size_t>(K) * T, model);
  b.states.resize(static_cast<std::size_t>(K) * (T + 1));
  for (std::size_t i = 0; i < b.states.size(); ++i) b.states[i] = {states[3 * i], states[3 * i + 1], states[3 * i + 2]};
  return b;
}

ValidationResult validate_nominal(const NominalSequence& nominal, const Pose2& q0,
                                  const ObstacleSet& obstacles, const PreparedFootprint& footprint,
                                  const MotionModel& model, const KinematicLimits& limits,
                                  const MppiParams& params, const Guidance& guidance,
                                  const ControlInput& u_prev) {
  MppiParams p = params;
  p.horizon = static_cast<int>(nominal.controls.size());
  const Config c = make_config(footprint, model, limits, p);
  const Flat f = flatten(obstacles, guidance);
  exm_handle* h = handle_for(c, static_cast<int>(obstacles.points.size()),
                             static_cast<int>(guidance.path.size()));
  const std::vector<double> nom = flat_controls(nominal.controls, model.control_dim());
  const double q[3] = {q0.x, q0.y, q0.theta};
  const double up[3] = {u_prev[0], u_prev[1], u_prev[2]};
  ValidationResult r;
  r.d_min.resize(nominal.controls.size());
  int32_t valid = 0;
  throw_status(exm_validate_nominal(h, nom.data(), q, f.pts.data(), f.mask.data(),
                                    static_cast<int32_t>(obstacles.points.size()), f.guide.data(),
                                    static_cast<int32_t>(guidance.path.size()), f.goal, up, &valid,
                                    r.d_min.data(), &r.cost));
  r.valid = valid != 0;
  return r;
}

MppiController::MppiController(MotionModel model, KinematicLimits limits,
                               const FootprintSpec& footprint, MppiParams params, int threads)
    : model_(model),
      limits_(limits),
      footprint_(prepare(footprint)),
      params_(params),
      threads_(std::max(threads, 1)),
      nominal_(NominalSequence::zero(model, params.horizon)),
      u_prev_(ControlInput::zero(model)) {
  params_.validate();
}

void MppiController::warm_start(const ControlInput& measured) {
  const ControlInput u = clamp_control(model_, measured, measured, limits_, params_.dt);
  nominal_ = NominalSequence::constant(u, params_.horizon);
  u_prev_ = u;
}

void MppiController::set_rate_anchor(const ControlInput& u) { u_prev_ = u; }

ControlDecision MppiController::control_cycle(const Pose2& q0, const ObstacleSet& obstacles,
                                              const Guidance& guidance) {
  const int T = params_.horizon, D = model_.control_dim();
  const Config c = make_config(footprint_, model_, limits_, params_);
  const Flat f = flatten(obstacles, guidance);
  exm_handle* h = handle_for(c, static_cast<int>(obstacles.points.size()),
                             static_cast<int>(guidance.path.size()));
  std::vector<double> nom = flat_controls(nominal_.controls, D);
  double up[3] = {u_prev_[0], u_prev_[1], u_prev_[2]};
  const double q[3] = {q0.x, q0.y, q0.theta};
  ControlDecision d;
  d.diagnostics.nominal_d_min.resize(static_cast<std::size_t>(T));
  exm_decision out{};
  out.nominal_dmin = d.diagnostics.nominal_d_min.data();
  throw_status(exm_control_cycle(h, q, f.pts.data(), f.mask.data(),
                                 static_cast<int32_t>(obstacles.points.size()), f.guide.data(),
                                 static_cast<int32_t>(guidance.path.size()), f.goal, nom.data(), up,
                                 cycle_, nullptr, &out));
  d.command = ControlInput::zero(model_);
  for (int k = 0; k < D; ++k) d.command[k] = out.command[k];
  d.validated = out.validated != 0;
  d.diagnostics.best_cost = out.best_cost;
  d.diagnostics.weight_entropy = out.weight_entropy;
  d.diagnostics.nominal_cost = out.nominal_cost;
  nominal_.controls = unflat_controls(nom.data(), static_cast<std::size_t>(T), model_);
  d.nominal = nominal_;
  u_prev_ = d.command;
  ++cycle_;
  return d;
}

}  // namespace exactmppi
