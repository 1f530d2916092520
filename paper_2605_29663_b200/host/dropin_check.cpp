// dropin_check.cpp — exercises the reference's own C++ controller API
// (proj/include/exactmppi/controller.hpp) with controller_b200.cpp linked in place of
// proj/src/controller.cpp, i.e. exactly what a reference user gets after the link-time swap.
// It prints one JSON object per line; tests/test_dropin.py compares them with the CPU oracle.
#include <cmath>
#include <stdexcept>
#include <cstdio>
#include <numbers>
#include <string>
#include <vector>

#include "exactmppi/controller.hpp"
#include "exactmppi/geometry.hpp"
#include "exactmppi/kinematics.hpp"

using namespace exactmppi;

namespace {

FootprintSpec l_shape() {
  FootprintSpec s;
  s.name = "l_shape";
  s.shape = PolygonFootprint::make(
      {{-1.0, -1.0}, {1.0, -1.0}, {1.0, -0.6}, {-0.6, -0.6}, {-0.6, 1.0}, {-1.0, 1.0}});
  return s;
}

KinematicLimits diff_limits() {
  KinematicLimits l = KinematicLimits::unbounded();
  l.component[0] = {-2.0, 2.0, -2.5, 2.5};
  l.component[1] = {-0.9, 0.9, -6.0, 6.0};
  return l;
}

std::vector<Point2> ring_cloud() {
  std::vector<Point2> pts;
  for (int k = 0; k < 400; ++k) {
    const double a = 2.0 * std::numbers::pi * k / 400.0;
    pts.push_back({3.0 + 0.5 * std::cos(a), 0.4 + 0.5 * std::sin(a)});
    pts.push_back({5.0 * std::cos(a), 5.0 * std::sin(a)});
  }
  return pts;
}

void print_vec(const char* key, const std::vector<double>& v, bool last = false) {
  std::printf("\"%s\": [", key);
  for (std::size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
  std::printf("]%s", last ? "" : ", ");
}

}  // namespace

int main() {
  MppiParams p;
  p.rollouts = 512;
  p.horizon = 20;
  p.dt = 0.1;
  p.lambda = 0.8;
  p.sigma = {0.45, 0.6, 0.3};
  p.d_safe = 0.09;
  p.w_rep = 60.0;
  p.task = {0.25, 0.3, 1.6, 3.0};
  p.seed = 1;
  const auto cloud = ring_cloud();
  auto obstacles = ObstacleSet::padded(cloud, cloud.size() + 16);
  Guidance g;
  g.path = {{0.0, 0.0}, {6.0, 0.0}};
  g.goal = {6.0, 0.0, 0.0};

  // 1. MppiController::control_cycle, three cycles from a fresh controller.
  MppiController ctl(MotionModel::diff(), diff_limits(), l_shape(), p);
  Pose2 q{0.0, 0.0, 0.0};
  for (int c = 0; c < 3; ++c) {
    auto d = ctl.control_cycle(q, obstacles, g);
    std::vector<double> nom;
    for (const auto& u : d.nominal.controls) {
      nom.push_back(u[0]);
      nom.push_back(u[1]);
    }
    std::printf("{\"kind\": \"cycle\", \"cycle\": %d, \"validated\": %d, ", c, d.validated ? 1 : 0);
    print_vec("q", {q.x, q.y, q.theta});
    print_vec("command", {d.command[0], d.command[1]});
    print_vec("nominal", nom);
    print_vec("nominal_d_min", d.diagnostics.nominal_d_min);
    std::printf("\"best_cost\": %.17g, \"weight_entropy\": %.17g, \"nominal_cost\": %.17g}\n",
                d.diagnostics.best_cost, d.diagnostics.weight_entropy, d.diagnostics.nominal_cost);
    q = step(MotionModel::diff(), q, d.command, p.dt);
  }

  // 2. sample_perturbations + evaluate_rollouts through the reference signatures.
  MppiParams pr = p;
  pr.rollouts = 64;
  auto eps = sample_perturbations(7, 2, MotionModel::diff(), pr);
  NominalSequence nom0 = NominalSequence::constant(ControlInput{{0.5, 0.0, 0.0}, 2}, pr.horizon);
  auto batch = evaluate_rollouts({0.1, -0.2, 0.05}, nom0, eps, obstacles, prepare(l_shape()),
                                 MotionModel::diff(), diff_limits(), pr, g,
                                 ControlInput{{0.3, 0.0, 0.0}, 2});
  std::vector<double> e0, dmin(batch.d_min.begin(), batch.d_min.end()), costs(batch.costs);
  for (const auto& e : eps) {
    e0.push_back(e[0]);
    e0.push_back(e[1]);
  }
  std::printf("{\"kind\": \"rollouts\", ");
  print_vec("eps", e0);
  print_vec("d_min", dmin);
  print_vec("costs", costs, true);
  std::printf("}\n");

  // 3. Reference error behaviour crosses the boundary as std::invalid_argument.
  try {
    MppiParams bad = p;
    bad.lambda = 0.0;
    MppiController broken(MotionModel::diff(), diff_limits(), l_shape(), bad);
    std::printf("{\"kind\": \"error\", \"thrown\": 0}\n");
  } catch (const std::invalid_argument& e) {
    std::printf("{\"kind\": \"error\", \"thrown\": 1, \"what\": \"%s\"}\n", e.what());
  }
  return 0;
}
