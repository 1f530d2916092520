// exm_exact64.cuh — the FP64 per-pose minimum of exm_evaluate_rollouts under EXM_OPT_SDF_FP64
// (the reference's own arithmetic: geometry.cpp:260-295 sd, :357-375 min_signed_distance_at).
#pragma once
#include "exm_common.cuh"

namespace exm {

// PreparedFootprint (geometry.hpp) in FP64, built on the host from the handle's footprint:
// polygon rows {vx, vy, ex, ey, inv_len2}, rectangle-cover rows {cx, cy, hx, hy, 0}.
struct FpDev64 {
  int kind;   // EXM_FOOTPRINT_*
  int count;
  double radius;  // FootprintSpec::bounding_radius (geometry.cpp:127-131)
  double v[kMaxEdges][5];
};

// out[r*T + h] = min_signed_distance_at(footprint, states[r][h], cloud) for h < T (the pre-step
// poses exm_launch_rollout writes, K x (T+1) x 3); mask == nullptr selects every point.
cudaError_t launch_sdf_exact64(const FpDev64& fp, const double* states, int K, int T,
                               const double* pts, const uint8_t* mask, int n, double* out,
                               cudaStream_t s);

// out[i] = PreparedFootprint::sd(q[i]) in FP64 (batch_signed_distance, geometry.cpp:298-318).
cudaError_t launch_sdf_points64(const FpDev64& fp, const double* q, int n, double* out,
                                cudaStream_t s);

// launch_rollout_costs with FP64 minima (the FP64 path of exm_evaluate_rollouts).
cudaError_t launch_rollout_costs_dmin64(const StepConst& sc, const double* task,
                                        const double* base_cost, const double* ctrl_cost,
                                        const double* dmin64, double* cost, uint8_t* unsafe,
                                        float* dstat, cudaStream_t s);

}  // namespace exm
