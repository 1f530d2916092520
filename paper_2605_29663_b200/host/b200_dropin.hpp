// b200_dropin.hpp — internal interface between the drop-in translation units
// (controller_b200.cpp, hybrid_b200.cpp); not part of the reference API.
#pragma once

#include <cstdint>
#include <vector>

#include "exactmppi/controller.hpp"

namespace exactmppi::b200 {

// One hybrid step of M mode families batched into a single device call (exm_hybrid_cycle):
// run_hybrid_batch() takes every family's controller state through the public accessors
// (nominal(), last_command(), cycle_index()), runs all M MPPI steps in one CUDA graph, and parks
// each family's decision; the family's own MppiController::control_cycle then consumes its
// parked result (same inputs) instead of launching, which updates the controller's private
// state exactly as a per-family step would. Returns false (nothing parked) when the families
// cannot be batched (their cycle counters differ): the caller then steps them one by one.
bool run_hybrid_batch(const std::vector<const MppiController*>& families,
                      const std::vector<KinematicLimits>& limits, const FootprintSpec& footprint,
                      const MppiParams& base_params, const Pose2& q0,
                      const ObstacleSet& obstacles, const Guidance& guidance);

}  // namespace exactmppi::b200
