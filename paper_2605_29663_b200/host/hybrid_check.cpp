// hybrid_check.cpp — the reference's HybridController API (proj/include/exactmppi/hybrid.hpp)
// with hybrid_b200.cpp + controller_b200.cpp linked in place of hybrid.cpp / controller.cpp: the
// M mode families of every hybrid cycle run in ONE device call (exm_hybrid_cycle). The trap
// scenario comes from the reference's own generator (make_trap_scenario), the cloud from its
// sense(). It prints the inputs and one JSON line per cycle; tests/test_dropin.py replays the
// same inputs through the unmodified reference HybridController (oracle/_ref) and compares.
#include <cmath>
#include <cstdio>
#include <vector>

#include "exactmppi/hybrid.hpp"
#include "exactmppi/kinematics.hpp"
#include "exactmppi/scenario_gen.hpp"
#include "exactmppi/world.hpp"

using namespace exactmppi;

namespace {
void vec(const char* key, const std::vector<double>& v, bool last = false) {
  std::printf("\"%s\": [", key);
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
  std::printf("]%s", last ? "" : ", ");
}
}  // namespace

int main() {
  const Scenario sc = make_trap_scenario(1);
  const HybridSetup& hs = *sc.hybrid;
  // setup line: everything the Python side needs to build the same controller
  std::printf("{\"kind\": \"setup\", ");
  const auto& rc = std::get<RectangleCover>(sc.footprint.shape);
  std::vector<double> fx, fy, fhx, fhy;
  for (const auto& r : rc.rectangles) {
    fx.push_back(r.center.x);
    fy.push_back(r.center.y);
    fhx.push_back(r.half_extent.x);
    fhy.push_back(r.half_extent.y);
  }
  vec("rect_cx", fx);
  vec("rect_cy", fy);
  vec("rect_hx", fhx);
  vec("rect_hy", fhy);
  std::printf("\"modes\": [");
  for (std::size_t m = 0; m < hs.modes.size(); ++m) {
    const auto& md = hs.modes[m];
    std::printf("%s{\"tag\": %d, \"wheelbase\": %.17g, ", m ? ", " : "", static_cast<int>(md.model.tag),
                md.model.wheelbase);
    std::vector<double> l;
    for (int i = 0; i < 3; ++i) {
      const auto& c = md.limits.component[i];
      l.insert(l.end(), {c.vel_min, c.vel_max, c.acc_min, c.acc_max});
    }
    l.push_back(md.limits.steer_max);
    vec("limits", l, true);
    std::printf("}");
  }
  std::printf("], ");
  const MppiParams& p = sc.mppi;
  vec("params", {static_cast<double>(p.rollouts), static_cast<double>(p.horizon), p.dt, p.lambda,
                 p.sigma[0], p.sigma[1], p.sigma[2], p.d_safe, p.w_coll, p.w_rep, p.w_inf,
                 p.task.goal_pos, p.task.goal_head, p.task.xtrack, p.task.progress, p.w_ctrl,
                 static_cast<double>(p.seed)});
  const HybridParams& hp = hs.params;
  vec("hybrid", {hp.lambda_switch, static_cast<double>(hp.tau_cool_max), hp.v_min, hp.omega_min,
                 hp.noise_deadzone_v, hp.noise_deadzone_omega});
  const WorldState st = WorldState::initial(sc);
  const ObstacleSet cloud = sense(sc, st, sc.start, 0);
  std::vector<double> pts, mask;
  for (std::size_t i = 0; i < cloud.points.size(); ++i) {
    pts.push_back(cloud.points[i].x);
    pts.push_back(cloud.points[i].y);
    mask.push_back(cloud.mask[i]);
  }
  vec("points", pts);
  vec("mask", mask);
  std::vector<double> guide;
  for (const auto& g : sc.guidance) guide.insert(guide.end(), {g.x, g.y});
  vec("guide", guide);
  vec("goal", {sc.goal.x, sc.goal.y, sc.goal.theta});
  vec("start", {sc.start.x, sc.start.y, sc.start.theta}, true);
  std::printf("}\n");

  HybridController hc(hs.modes, sc.footprint, sc.mppi, hs.params, 1);
  Guidance gd{sc.guidance, sc.goal};
  Pose2 q = sc.start;
  for (int cyc = 0; cyc < 8; ++cyc) {
    const HybridDecision d = hc.hybrid_cycle(q, cloud, gd);
    std::printf("{\"kind\": \"cycle\", \"cycle\": %d, ", cyc);
    vec("q", {q.x, q.y, q.theta});
    std::vector<double> cmd;
    for (int i = 0; i < d.command.dim; ++i) cmd.push_back(d.command[i]);
    vec("command", cmd);
    std::vector<double> costs;
    for (double c : d.mode_costs) costs.push_back(std::isfinite(c) ? c : 1e300);
    vec("mode_costs", costs);
    std::printf("\"mode_index\": %d, \"validated\": %d, \"best_cost\": %.17g, \"entropy\": %.17g, "
                "\"nominal_cost\": %.17g}\n",
                d.mode_index, d.validated ? 1 : 0, d.diagnostics.best_cost,
                d.diagnostics.weight_entropy, d.diagnostics.nominal_cost);
    q = step(hs.modes[static_cast<std::size_t>(d.mode_index)].model, q, d.command, sc.mppi.dt);
  }
  return 0;
}
