// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. extern "C" entry points over the UNMODIFIED
// reference library, compiled from the reference's own sources into oracle/_ref/ by
// oracle/Makefile (nothing from the reference tree is copied into this repository).
//
// Used by tests (to pin oracle/exm_oracle.c bit-for-bit against the real reference) and by
// bench.py's cpu_baseline / --impl reference legs (the reference's own CPU path, timed on
// the host cores). Every call goes through the reference's public C++ API:
//   PolygonFootprint::make / RectangleCover::make / prepare   (geometry.hpp)
//   PreparedFootprint::sd, batch_signed_distance, min_signed_distance_at
//   sample_perturbations, evaluate_rollouts, weights_from_costs, validate_nominal
//   MppiController::control_cycle                              (controller.hpp)
//   sense                                                      (world.hpp)
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "exactmppi/controller.hpp"
#include "exactmppi/geometry.hpp"
#include "exactmppi/hybrid.hpp"
#include "exactmppi/kinematics.hpp"
#include "exactmppi/world.hpp"
#include "exm_b200.h"

using namespace exactmppi;

namespace {
thread_local std::string g_err;

struct RefCtx {
  FootprintSpec spec;
  PreparedFootprint prepared;
  MotionModel model;
  KinematicLimits limits;
  MppiParams params;
  int threads = 1;
  std::unique_ptr<MppiController> controller;
  ObstacleSet cloud;
};

FootprintSpec to_spec(const exm_footprint* fp) {
  FootprintSpec spec;
  spec.name = "abi";
  if (fp->kind == EXM_FOOTPRINT_POLYGON) {
    std::vector<Point2> v;
    for (int i = 0; i < fp->count; ++i) v.push_back({fp->x[i], fp->y[i]});
    spec.shape = PolygonFootprint::make(std::move(v));
  } else {
    std::vector<AxisRectangle> r;
    for (int i = 0; i < fp->count; ++i) r.push_back({{fp->x[i], fp->y[i]}, {fp->hx[i], fp->hy[i]}});
    spec.shape = RectangleCover::make(std::move(r));
  }
  return spec;
}

MotionModel to_model(const exm_model* m) {
  switch (m->tag) {
    case EXM_MODEL_DIFF: return MotionModel::diff();
    case EXM_MODEL_ACKERMANN: return MotionModel::ackermann(m->wheelbase);
    case EXM_MODEL_OMNI: return MotionModel::omni();
    case EXM_MODEL_SPIN: return MotionModel::spin();
    case EXM_MODEL_PARALLEL: return MotionModel::parallel();
  }
  throw std::invalid_argument("unknown motion model");
}

KinematicLimits to_limits(const exm_limits* l) {
  KinematicLimits k;
  for (int i = 0; i < 3; ++i) k.component[i] = {l->vel_min[i], l->vel_max[i], l->acc_min[i], l->acc_max[i]};
  k.steer_max = l->steer_max;
  return k;
}

MppiParams to_params(const exm_params* p) {
  MppiParams q;
  q.rollouts = p->rollouts;
  q.horizon = p->horizon;
  q.dt = p->dt;
  q.lambda = p->lambda;
  q.sigma = {p->sigma[0], p->sigma[1], p->sigma[2]};
  q.d_safe = p->d_safe;
  q.w_coll = p->w_coll;
  q.w_rep = p->w_rep;
  q.w_inf = p->w_inf;
  q.task = {p->w_goal_pos, p->w_goal_head, p->w_xtrack, p->w_progress};
  q.w_ctrl = p->w_ctrl;
  q.seed = p->seed;
  return q;
}

ObstacleSet to_cloud(const double* pts, const uint8_t* mask, int n) {
  ObstacleSet s;
  s.points.resize(static_cast<std::size_t>(n));
  s.mask.resize(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    s.points[i] = {pts[2 * i], pts[2 * i + 1]};
    s.mask[i] = mask ? mask[i] : 1;
  }
  return s;
}

Guidance to_guidance(const double* g, int n, const double goal[3]) {
  Guidance gd;
  for (int i = 0; i < n; ++i) gd.path.push_back({g[2 * i], g[2 * i + 1]});
  gd.goal = {goal[0], goal[1], goal[2]};
  return gd;
}

std::vector<ControlInput> to_controls(const double* u, std::size_t count, const MotionModel& m) {
  const int D = m.control_dim();
  std::vector<ControlInput> out(count, ControlInput::zero(m));
  for (std::size_t i = 0; i < count; ++i)
    for (int c = 0; c < D; ++c) out[i][c] = u[i * D + c];
  return out;
}

ControlInput to_control(const double* u, const MotionModel& m) {
  return to_controls(u, 1, m)[0];
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return EXM_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return EXM_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return EXM_ERR_INTERNAL;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void* ref_create(const exm_footprint* fp, const exm_model* m, const exm_limits* l,
                 const exm_params* p, int32_t threads) {
  RefCtx* c = nullptr;
  int st = guard([&] {
    auto ctx = std::make_unique<RefCtx>();
    ctx->spec = to_spec(fp);
    ctx->prepared = prepare(ctx->spec);
    ctx->model = to_model(m);
    ctx->limits = to_limits(l);
    ctx->params = to_params(p);
    ctx->params.validate();
    ctx->threads = threads < 1 ? 1 : threads;
    ctx->controller = std::make_unique<MppiController>(ctx->model, ctx->limits, ctx->spec,
                                                       ctx->params, ctx->threads);
    c = ctx.release();
  });
  return st == EXM_OK ? c : nullptr;
}

void ref_destroy(void* c) { delete static_cast<RefCtx*>(c); }

double ref_bounding_radius(void* c) { return static_cast<RefCtx*>(c)->prepared.bounding_radius; }

double ref_sd(void* c, double x, double y) { return static_cast<RefCtx*>(c)->prepared.sd({x, y}); }

int32_t ref_batch_signed_distance(void* cp, const double* q, int32_t n, double* out,
                                  int32_t threads) {
  auto* c = static_cast<RefCtx*>(cp);
  return guard([&] {
    std::vector<Point2> queries(static_cast<std::size_t>(n));
    for (int i = 0; i < n; ++i) queries[i] = {q[2 * i], q[2 * i + 1]};
    batch_signed_distance(queries, c->prepared, std::span<double>(out, static_cast<std::size_t>(n)),
                          threads);
  });
}

// Cloud kept in the context so repeated pose queries do not rebuild the ObstacleSet.
int32_t ref_set_cloud(void* cp, const double* pts, const uint8_t* mask, int32_t n) {
  auto* c = static_cast<RefCtx*>(cp);
  return guard([&] { c->cloud = to_cloud(pts, mask, n); });
}

int32_t ref_min_sd_at_batch(void* cp, const double* poses, int32_t n_poses, double* out) {
  auto* c = static_cast<RefCtx*>(cp);
  return guard([&] {
    for (int p = 0; p < n_poses; ++p)
      out[p] = min_signed_distance_at(c->prepared, {poses[3 * p], poses[3 * p + 1], poses[3 * p + 2]},
                                      c->cloud);
  });
}

int32_t ref_sample_perturbations(void* cp, uint64_t seed, uint64_t cycle, double* eps) {
  auto* c = static_cast<RefCtx*>(cp);
  return guard([&] {
    auto e = sample_perturbations(seed, cycle, c->model, c->params);
    const int D = c->model.control_dim();
    for (std::size_t i = 0; i < e.size(); ++i)
      for (int k = 0; k < D; ++k) eps[i * D + k] = e[i][k];
  });
}

int32_t ref_evaluate_rollouts(void* cp, const double q0[3], const double* nominal,
                              const double* eps, const double* pts, const uint8_t* mask,
                              int32_t n, const double* guide, int32_t n_guide,
                              const double goal[3], const double* u_prev, double* controls,
                              double* states, double* dmin, double* costs, uint8_t* unsafe) {
  auto* c = static_cast<RefCtx*>(cp);
  return guard([&] {
    const int K = c->params.rollouts, T = c->params.horizon, D = c->model.control_dim();
    NominalSequence nom;
    nom.controls = to_controls(nominal, static_cast<std::size_t>(T), c->model);
    auto e = to_controls(eps, static_cast<std::size_t>(K) * T, c->model);
    auto batch = evaluate_rollouts({q0[0], q0[1], q0[2]}, nom, e, to_cloud(pts, mask, n),
                                   c->prepared, c->model, c->limits, c->params,
                                   to_guidance(guide, n_guide, goal), to_control(u_prev, c->model),
                                   c->threads);
    for (std::size_t i = 0; i < batch.controls.size(); ++i) {
      if (controls)
        for (int k = 0; k < D; ++k) controls[i * D + k] = batch.controls[i][k];
      if (dmin) dmin[i] = batch.d_min[i];
    }
    if (states)
      for (std::size_t i = 0; i < batch.states.size(); ++i) {
        states[3 * i] = batch.states[i].x;
        states[3 * i + 1] = batch.states[i].y;
        states[3 * i + 2] = batch.states[i].theta;
      }
    for (int r = 0; r < K; ++r) {
      if (costs) costs[r] = batch.costs[r];
      if (unsafe) unsafe[r] = batch.unsafe[r];
    }
  });
}

int32_t ref_weights_from_costs(const double* costs, int32_t k, double lambda, double* w) {
  return guard([&] {
    auto v = weights_from_costs(std::span<const double>(costs, static_cast<std::size_t>(k)), lambda);
    std::memcpy(w, v.data(), sizeof(double) * v.size());
  });
}

int32_t ref_validate_nominal(void* cp, const double* nominal, const double q0[3],
                             const double* pts, const uint8_t* mask, int32_t n,
                             const double* guide, int32_t n_guide, const double goal[3],
                             const double* u_prev, int32_t* valid, double* dmin, double* cost) {
  auto* c = static_cast<RefCtx*>(cp);
  return guard([&] {
    NominalSequence nom;
    nom.controls = to_controls(nominal, static_cast<std::size_t>(c->params.horizon), c->model);
    auto res = validate_nominal(nom, {q0[0], q0[1], q0[2]}, to_cloud(pts, mask, n), c->prepared,
                                c->model, c->limits, c->params, to_guidance(guide, n_guide, goal),
                                to_control(u_prev, c->model));
    *valid = res.valid ? 1 : 0;
    if (dmin) std::memcpy(dmin, res.d_min.data(), sizeof(double) * res.d_min.size());
    *cost = res.cost;
  });
}

// MppiController::control_cycle on the context's own controller object (state lives in the
// object, exactly as in the reference). nominal_out / u_prev_out receive the state after
// the cycle; decision fields as in exm_decision (argmin is not exposed by the reference: -1).
int32_t ref_controller_cycle(void* cp, const double q0[3], int32_t use_stored_cloud,
                             const double* pts, const uint8_t* mask, int32_t n,
                             const double* guide, int32_t n_guide, const double goal[3],
                             double* nominal_out, double* u_prev_out, exm_decision* out) {
  auto* c = static_cast<RefCtx*>(cp);
  return guard([&] {
    ObstacleSet local;
    if (!use_stored_cloud) local = to_cloud(pts, mask, n);
    const ObstacleSet& cloud = use_stored_cloud ? c->cloud : local;
    auto d = c->controller->control_cycle({q0[0], q0[1], q0[2]}, cloud,
                                          to_guidance(guide, n_guide, goal));
    const int D = c->model.control_dim();
    if (nominal_out)
      for (std::size_t h = 0; h < d.nominal.controls.size(); ++h)
        for (int k = 0; k < D; ++k) nominal_out[h * D + k] = d.nominal.controls[h][k];
    if (u_prev_out)
      for (int k = 0; k < D; ++k) u_prev_out[k] = c->controller->last_command()[k];
    if (out) {
      for (int k = 0; k < 3; ++k) out->command[k] = k < D ? d.command[k] : 0.0;
      out->validated = d.validated ? 1 : 0;
      out->argmin = -1;
      out->best_cost = d.diagnostics.best_cost;
      out->weight_entropy = d.diagnostics.weight_entropy;
      out->nominal_cost = d.diagnostics.nominal_cost;
      if (out->nominal_dmin)
        std::memcpy(out->nominal_dmin, d.diagnostics.nominal_d_min.data(),
                    sizeof(double) * d.diagnostics.nominal_d_min.size());
    }
  });
}

// Reset the controller object (fresh MppiController: zero nominal, zero rate anchor, cycle 0).
int32_t ref_controller_reset(void* cp) {
  auto* c = static_cast<RefCtx*>(cp);
  return guard([&] {
    c->controller = std::make_unique<MppiController>(c->model, c->limits, c->spec, c->params,
                                                     c->threads);
  });
}

// ---- HybridController (hybrid.hpp:51-69) over the reference's own MppiControllers ----
struct RefHybrid {
  std::unique_ptr<HybridController> hc;
  std::vector<HybridMode> modes;
};

void* ref_hybrid_create(const exm_footprint* fp, const exm_model* models, const exm_limits* limits,
                        int32_t n_modes, const exm_params* p, const double hp[6], int32_t threads) {
  RefHybrid* out = nullptr;
  int st = guard([&] {
    auto h = std::make_unique<RefHybrid>();
    for (int m = 0; m < n_modes; ++m)
      h->modes.push_back({"m" + std::to_string(m), to_model(&models[m]), to_limits(&limits[m])});
    HybridParams hpar;
    hpar.lambda_switch = hp[0];
    hpar.tau_cool_max = static_cast<int>(hp[1]);
    hpar.v_min = hp[2];
    hpar.omega_min = hp[3];
    hpar.noise_deadzone_v = hp[4];
    hpar.noise_deadzone_omega = hp[5];
    h->hc = std::make_unique<HybridController>(h->modes, to_spec(fp), to_params(p), hpar,
                                               threads < 1 ? 1 : threads);
    out = h.release();
  });
  return st == EXM_OK ? out : nullptr;
}

void ref_hybrid_destroy(void* h) { delete static_cast<RefHybrid*>(h); }

// command[3], mode_index, validated, mode_costs[n_modes], and the selected mode's diagnostics.
int32_t ref_hybrid_cycle(void* hp, const double q0[3], const double* pts, const uint8_t* mask,
                         int32_t n, const double* guide, int32_t n_guide, const double goal[3],
                         double* command, int32_t* mode_index, int32_t* validated,
                         double* mode_costs, double* diag /* best, entropy, nominal_cost */) {
  auto* h = static_cast<RefHybrid*>(hp);
  return guard([&] {
    auto d = h->hc->hybrid_cycle({q0[0], q0[1], q0[2]}, to_cloud(pts, mask, n),
                                 to_guidance(guide, n_guide, goal));
    for (int k = 0; k < 3; ++k) command[k] = k < d.command.dim ? d.command[k] : 0.0;
    *mode_index = d.mode_index;
    *validated = d.validated ? 1 : 0;
    for (std::size_t m = 0; m < d.mode_costs.size(); ++m) mode_costs[m] = d.mode_costs[m];
    diag[0] = d.diagnostics.best_cost;
    diag[1] = d.diagnostics.weight_entropy;
    diag[2] = d.diagnostics.nominal_cost;
  });
}

}  // extern "C"

// sense(scenario, state, robot, key) with the given obstacles displaced by their offsets
// (geometry translated here, no trail motion: the reference then adds a zero offset).
extern "C" int ref_sense(const exm_world_obstacle* obs, int n, const double robot[3], double range,
                         int budget, uint64_t seed, uint64_t sample_key, double* pts_out,
                         uint8_t* mask_out, int* n_valid) {
  try {
    Scenario sc;
    sc.sensor.range = range;
    sc.sensor.budget = budget;
    sc.seed = seed;
    for (int i = 0; i < n; ++i) {
      const exm_world_obstacle& o = obs[i];
      Obstacle ob;
      if (o.kind == EXM_OBSTACLE_DISC) {
        ob.shape = Disc{{o.x[0] + o.offset[0], o.y[0] + o.offset[1]}, o.radius};
      } else {
        std::vector<Point2> v;
        for (int k = 0; k < o.count; ++k) v.push_back({o.x[k] + o.offset[0], o.y[k] + o.offset[1]});
        ob.shape = PolygonFootprint::make(v);
      }
      sc.obstacles.push_back(std::move(ob));
    }
    const WorldState st = WorldState::initial(sc);
    const ObstacleSet set = sense(sc, st, Pose2{robot[0], robot[1], robot[2]}, sample_key);
    int nv = 0;
    for (std::size_t i = 0; i < set.points.size(); ++i) {
      pts_out[2 * i] = set.points[i].x;
      pts_out[2 * i + 1] = set.points[i].y;
      mask_out[i] = set.mask[i];
      nv += set.mask[i] != 0;
    }
    *n_valid = nv;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// ---- world with trails (test infrastructure for exm_world_*): the reference's Scenario +
// WorldState, step_world and sense (world.hpp) ----
struct RefWorld {
  Scenario sc;
  WorldState st;
};

extern "C" void* ref_world_create(const exm_world_obstacle* obs, const int32_t* n_wp,
                                  const double* const* wp, const double* speed,
                                  const int32_t* ping_pong, int n, double range, int budget,
                                  uint64_t seed) {
  try {
    auto w = std::make_unique<RefWorld>();
    w->sc.sensor.range = range;
    w->sc.sensor.budget = budget;
    w->sc.seed = seed;
    for (int i = 0; i < n; ++i) {
      const exm_world_obstacle& o = obs[i];
      Obstacle ob;
      if (o.kind == EXM_OBSTACLE_DISC) {
        ob.shape = Disc{{o.x[0], o.y[0]}, o.radius};
      } else {
        std::vector<Point2> v;
        for (int k = 0; k < o.count; ++k) v.push_back({o.x[k], o.y[k]});
        ob.shape = PolygonFootprint::make(v);
      }
      if (n_wp[i] >= 2) {
        TrailMotion m;
        for (int k = 0; k < n_wp[i]; ++k) m.waypoints.push_back({wp[i][2 * k], wp[i][2 * k + 1]});
        m.speed = speed[i];
        m.ping_pong = ping_pong[i] != 0;
        ob.motion = m;
      }
      w->sc.obstacles.push_back(std::move(ob));
    }
    w->st = WorldState::initial(w->sc);
    return w.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

extern "C" void ref_world_destroy(void* w) { delete static_cast<RefWorld*>(w); }

extern "C" int ref_world_step(void* wp, double dt) {
  auto* w = static_cast<RefWorld*>(wp);
  try {
    w->st = step_world(w->sc, w->st, dt);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

extern "C" void ref_world_state(void* wp, double* arc, int32_t* dir, double* offsets) {
  auto* w = static_cast<RefWorld*>(wp);
  for (std::size_t i = 0; i < w->sc.obstacles.size(); ++i) {
    arc[i] = w->st.arc[i];
    dir[i] = w->st.direction[i];
    const Point2 o = obstacle_offset(w->sc, w->st, i);
    offsets[2 * i] = o.x;
    offsets[2 * i + 1] = o.y;
  }
}

extern "C" int ref_world_sense(void* wp, const double robot[3], uint64_t key, double* pts_out,
                               uint8_t* mask_out, int* n_valid) {
  auto* w = static_cast<RefWorld*>(wp);
  try {
    const ObstacleSet set = sense(w->sc, w->st, Pose2{robot[0], robot[1], robot[2]}, key);
    int nv = 0;
    for (std::size_t i = 0; i < set.points.size(); ++i) {
      pts_out[2 * i] = set.points[i].x;
      pts_out[2 * i + 1] = set.points[i].y;
      mask_out[i] = set.mask[i];
      nv += set.mask[i] != 0;
    }
    *n_valid = nv;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
