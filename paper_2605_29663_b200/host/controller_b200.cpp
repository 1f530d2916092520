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
#include <cstdlib>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "b200_dropin.hpp"
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
  // exact byte key (footprint arrays + the POD model / limits / params, zero-initialised so
  // padding is deterministic): equal keys <=> identical configurations
  auto put = [&c](const void* p, std::size_t n) {
    c.key.append(static_cast<const char*>(p), n);
  };
  put(&c.fp.kind, sizeof c.fp.kind);
  for (const auto* v : {&c.x, &c.y, &c.hx, &c.hy}) {
    const std::size_t n = v->size();
    put(&n, sizeof n);
    put(v->data(), n * sizeof(double));
  }
  put(&c.model, sizeof c.model);
  put(&c.limits, sizeof c.limits);
  put(&c.params, sizeof c.params);
  return c;
}

// One cached device handle. Shared: a caller keeps the handle it got alive even if another
// thread's larger cloud replaces the cache slot meanwhile; calls on one handle serialise on the
// handle's own lock inside the library (include/exm_b200.h, threading).
struct Cached {
  exm_handle* h = nullptr;
  int n_cap = 0;
  int guide_cap = 0;
  ~Cached() {
    if (h) exm_destroy(h);
  }
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<Cached>> g_cache;

// Handle for this configuration with room for n points and g guidance vertices.
std::shared_ptr<Cached> handle_for(const Config& c, int n, int g) {
  std::lock_guard<std::mutex> lock(g_mu);
  auto& slot = g_cache[c.key];
  if (!slot || slot->n_cap < n || slot->guide_cap < g) {
    auto fresh = std::make_shared<Cached>();
    const int ncap = std::max(n, std::max(1024, slot ? 2 * slot->n_cap : 0));
    const int gcap = std::max(g, 64);
    throw_status(exm_create(&c.fp, &c.model, &c.limits, &c.params, ncap, gcap, -1, &fresh->h));
    // evaluate_rollouts returns the reference's FP64 minima and costs (its callers check them
    // against scalar loops at 1e-9, acceptance_main.cpp:260-300); the control cycle keeps FP32
    throw_status(exm_set_option(fresh->h, EXM_OPT_SDF_FP64, 1));
    fresh->n_cap = ncap;
    fresh->guide_cap = gcap;
    slot = std::move(fresh);  // the previous handle lives on while a caller still holds it
  }
  return slot;
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
  const auto hc = handle_for(c, 1, 1);
  exm_handle* h = hc->h;
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
  const auto hc = handle_for(c, static_cast<int>(obstacles.points.size()),
                             static_cast<int>(guidance.path.size()));
  exm_handle* h = hc->h;
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
  const auto hc = handle_for(c, static_cast<int>(obstacles.points.size()),
                             static_cast<int>(guidance.path.size()));
  exm_handle* h = hc->h;
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

// ---------------------------------------------------------------- emulated rollout shards
// EXM_DROPIN_SHARDS=G (read once): controller steps run as G rollout shards on the one device
// (exm_set_shard + exm_sharded_cycle: the block partials exchanged as the ranks' all-gather
// would), for the episode determinism harness across shard counts (host/episode_main.cpp).
// Configurations whose K is not a multiple of 256*G run unsharded.
namespace {

int dropin_shards() {
  static const int g = [] {
    const char* e = std::getenv("EXM_DROPIN_SHARDS");
    return e ? std::max(1, std::atoi(e)) : 1;
  }();
  return g;
}

struct ShardSet {
  std::vector<exm_handle*> h;
  int n_cap = 0, guide_cap = 0;
  ~ShardSet() {
    for (auto* x : h)
      if (x) exm_destroy(x);
  }
};
std::mutex g_sh_mu;
std::map<std::string, std::shared_ptr<ShardSet>> g_sh_cache;

std::shared_ptr<ShardSet> shards_for(const Config& c, int G, int n, int g) {
  std::lock_guard<std::mutex> lock(g_sh_mu);
  auto& slot = g_sh_cache[c.key];
  if (!slot || slot->n_cap < n || slot->guide_cap < g) {
    auto fresh = std::make_shared<ShardSet>();
    fresh->n_cap = std::max(n, std::max(1024, slot ? 2 * slot->n_cap : 0));
    fresh->guide_cap = std::max(g, 64);
    fresh->h.assign(static_cast<std::size_t>(G), nullptr);
    for (int r = 0; r < G; ++r) {
      throw_status(exm_create(&c.fp, &c.model, &c.limits, &c.params, fresh->n_cap,
                              fresh->guide_cap, -1, &fresh->h[static_cast<std::size_t>(r)]));
      throw_status(exm_set_shard(fresh->h[static_cast<std::size_t>(r)], r, G));
    }
    slot = std::move(fresh);
  }
  return slot;
}

}  // namespace

// ---------------------------------------------------------------- batched hybrid families
namespace {

// A decision computed by a batched hybrid step for one family, waiting for that family's
// control_cycle call on the same inputs (same thread).
struct Parked {
  const MppiController* who = nullptr;
  const ObstacleSet* obstacles = nullptr;
  const Guidance* guidance = nullptr;
  Pose2 q0{};
  std::uint64_t cycle = 0;
  ControlDecision decision;
  std::vector<double> nominal;  // T x dim, after the step
};
thread_local std::vector<Parked> t_parked;

struct HybridCached {
  exm_hybrid* h = nullptr;
  int n_cap = 0, guide_cap = 0;
  ~HybridCached() {
    if (h) exm_hybrid_destroy(h);
  }
};
std::mutex g_hy_mu;
std::map<std::string, std::shared_ptr<HybridCached>> g_hy_cache;

}  // namespace

namespace b200 {

bool run_hybrid_batch(const std::vector<const MppiController*>& families,
                      const std::vector<KinematicLimits>& limits, const FootprintSpec& footprint,
                      const MppiParams& base_params, const Pose2& q0,
                      const ObstacleSet& obstacles, const Guidance& guidance) {
  t_parked.clear();
  const std::size_t M = families.size();
  if (M == 0 || limits.size() != M) return false;
  const std::uint64_t cycle = families[0]->cycle_index();
  for (const auto* f : families)
    if (f->cycle_index() != cycle || f->params().horizon != base_params.horizon ||
        f->params().rollouts != base_params.rollouts)
      return false;
  const int T = base_params.horizon;
  // configuration key: the footprint + every family's model and limits + the base params
  const Config c0 = make_config(prepare(footprint), families[0]->model(), limits[0], base_params);
  std::string key = c0.key;
  std::vector<exm_model> models(M);
  std::vector<exm_limits> lims(M);
  for (std::size_t m = 0; m < M; ++m) {
    const Config cm = make_config(prepare(footprint), families[m]->model(), limits[m], base_params);
    models[m] = cm.model;
    lims[m] = cm.limits;
    key.append(reinterpret_cast<const char*>(&models[m]), sizeof(exm_model));
    key.append(reinterpret_cast<const char*>(&lims[m]), sizeof(exm_limits));
  }
  const int n = static_cast<int>(obstacles.points.size());
  const int g = static_cast<int>(guidance.path.size());
  std::shared_ptr<HybridCached> hc;
  {
    std::lock_guard<std::mutex> lock(g_hy_mu);
    auto& slot = g_hy_cache[key];
    if (!slot || slot->n_cap < n || slot->guide_cap < g) {
      auto fresh = std::make_shared<HybridCached>();
      const int ncap = std::max(n, std::max(1024, slot ? 2 * slot->n_cap : 0));
      const int gcap = std::max(g, 64);
      throw_status(exm_hybrid_create(&c0.fp, models.data(), lims.data(), static_cast<int32_t>(M),
                                     &c0.params, ncap, gcap, -1, &fresh->h));
      fresh->n_cap = ncap;
      fresh->guide_cap = gcap;
      slot = std::move(fresh);
    }
    hc = slot;
  }
  const Flat f = flatten(obstacles, guidance);
  std::vector<double> noms(M * static_cast<std::size_t>(T) * 3, 0.0), ups(3 * M, 0.0);
  for (std::size_t m = 0; m < M; ++m) {
    const int D = families[m]->model().control_dim();
    const auto& u = families[m]->nominal().controls;
    for (int h = 0; h < T; ++h)
      for (int k = 0; k < D; ++k) noms[m * T * 3 + h * D + k] = u[static_cast<std::size_t>(h)][k];
    for (int k = 0; k < D; ++k) ups[3 * m + k] = families[m]->last_command()[k];
  }
  std::vector<exm_decision> out(M);
  std::vector<std::vector<double>> dmins(M, std::vector<double>(static_cast<std::size_t>(T)));
  for (std::size_t m = 0; m < M; ++m) out[m].nominal_dmin = dmins[m].data();
  const double q[3] = {q0.x, q0.y, q0.theta};
  throw_status(exm_hybrid_cycle(hc->h, q, f.pts.data(), f.mask.data(), n, f.guide.data(), g,
                                f.goal, noms.data(), ups.data(), cycle, out.data()));
  for (std::size_t m = 0; m < M; ++m) {
    const MotionModel& model = families[m]->model();
    const int D = model.control_dim();
    Parked p;
    p.who = families[m];
    p.obstacles = &obstacles;
    p.guidance = &guidance;
    p.q0 = q0;
    p.cycle = cycle;
    p.decision.command = ControlInput::zero(model);
    for (int k = 0; k < D; ++k) p.decision.command[k] = out[m].command[k];
    p.decision.validated = out[m].validated != 0;
    p.decision.diagnostics.best_cost = out[m].best_cost;
    p.decision.diagnostics.weight_entropy = out[m].weight_entropy;
    p.decision.diagnostics.nominal_cost = out[m].nominal_cost;
    p.decision.diagnostics.nominal_d_min = std::move(dmins[m]);
    p.nominal.assign(noms.begin() + static_cast<std::ptrdiff_t>(m * T * 3),
                     noms.begin() + static_cast<std::ptrdiff_t>(m * T * 3 + T * D));
    t_parked.push_back(std::move(p));
  }
  return true;
}

}  // namespace b200

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
  for (auto it = t_parked.begin(); it != t_parked.end(); ++it) {  // batched hybrid step
    if (it->who != this) continue;
    const bool same = it->obstacles == &obstacles && it->guidance == &guidance &&
                      it->q0.x == q0.x && it->q0.y == q0.y && it->q0.theta == q0.theta &&
                      it->cycle == cycle_;
    if (!same) {
      t_parked.erase(it);
      break;
    }
    ControlDecision d = std::move(it->decision);
    nominal_.controls = unflat_controls(it->nominal.data(), static_cast<std::size_t>(T), model_);
    t_parked.erase(it);
    d.nominal = nominal_;
    u_prev_ = d.command;
    ++cycle_;
    return d;
  }
  const Config c = make_config(footprint_, model_, limits_, params_);
  const Flat f = flatten(obstacles, guidance);
  const auto hc = handle_for(c, static_cast<int>(obstacles.points.size()),
                             static_cast<int>(guidance.path.size()));
  exm_handle* h = hc->h;
  std::vector<double> nom = flat_controls(nominal_.controls, D);
  double up[3] = {u_prev_[0], u_prev_[1], u_prev_[2]};
  const double q[3] = {q0.x, q0.y, q0.theta};
  ControlDecision d;
  d.diagnostics.nominal_d_min.resize(static_cast<std::size_t>(T));
  exm_decision out{};
  out.nominal_dmin = d.diagnostics.nominal_d_min.data();
  const int G = dropin_shards();
  if (G > 1 && params_.rollouts % (256 * G) == 0) {
    const auto set = shards_for(c, G, static_cast<int>(obstacles.points.size()),
                                static_cast<int>(guidance.path.size()));
    std::vector<double> noms, ups;
    for (int r = 0; r < G; ++r) {
      noms.insert(noms.end(), nom.begin(), nom.end());
      ups.insert(ups.end(), up, up + 3);
    }
    std::vector<exm_decision> outs(static_cast<std::size_t>(G), out);
    throw_status(exm_sharded_cycle(set->h.data(), G, q, f.pts.data(), f.mask.data(),
                                   static_cast<int32_t>(obstacles.points.size()), f.guide.data(),
                                   static_cast<int32_t>(guidance.path.size()), f.goal,
                                   noms.data(), ups.data(), cycle_, nullptr, outs.data()));
    out = outs[0];
    std::copy(noms.begin(), noms.begin() + static_cast<std::ptrdiff_t>(nom.size()), nom.begin());
  } else {
    throw_status(exm_control_cycle(h, q, f.pts.data(), f.mask.data(),
                                   static_cast<int32_t>(obstacles.points.size()), f.guide.data(),
                                   static_cast<int32_t>(guidance.path.size()), f.goal, nom.data(),
                                   up, cycle_, nullptr, &out));
  }
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
