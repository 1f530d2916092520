// exm_device.cuh — device helpers shared by the two kernel translation units
// (exm_kernels.cu: cloud + signed distance, FP32; exm_dynamics.cu: rollouts, costs, softmax,
// FP64 compiled without FMA contraction). Internal linkage: each unit gets its own copy.
#pragma once

#include <cfloat>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>

#include "exm_common.cuh"

#define EXM_FOOTPRINT_RECT_COVER 0
#define EXM_FOOTPRINT_POLYGON 1
#define EXM_MODEL_DIFF 0
#define EXM_MODEL_ACKERMANN 1
#define EXM_MODEL_OMNI 2
#define EXM_MODEL_SPIN 3
#define EXM_MODEL_PARALLEL 4

namespace exm {
namespace {

// First statement of every kernel: with programmatic dependent launch (launch_k) wait for the
// predecessor grid's completion and memory flush; a no-op for a normally launched kernel.
// Then let the dependent grid launch right away: its CTAs take free SM slots and park in their
// own wait, so the launch latency overlaps this grid's execution.
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" :::);
}

constexpr double kPi = 3.14159265358979323846;
constexpr unsigned kFull = 0xffffffffu;

// ------------------------------------------------------------------ counter RNG (rng.hpp)
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__device__ __forceinline__ uint64_t hash_mix(uint64_t h, uint64_t v) {
  return splitmix64(h ^ (v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2)));
}
__device__ __forceinline__ double unit_oc(uint64_t h) {  // (0, 1]
  return static_cast<double>((h >> 11) + 1) * 0x1.0p-53;
}

// ------------------------------------------------------------------ FP64 scalar helpers
// std::min / std::max / std::clamp with libstdc++'s comparison order.
__device__ __forceinline__ double mn(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double mx(double a, double b) { return (a < b) ? b : a; }
__device__ __forceinline__ double clampd(double v, double lo, double hi) {
  return (v < lo) ? lo : (hi < v) ? hi : v;
}
__device__ __forceinline__ double wrap_angle(double a) {  // geometry.cpp:17-23
  const double tau = 2.0 * kPi;
  a = fmod(a, tau);
  if (a <= -kPi) a += tau;
  if (a > kPi) a -= tau;
  return a;
}

template <int TAG>
__host__ __device__ constexpr int model_dim() {  // kinematics.cpp:14-26
  return (TAG == EXM_MODEL_DIFF || TAG == EXM_MODEL_ACKERMANN) ? 2 : (TAG == EXM_MODEL_OMNI ? 3 : 1);
}

}  // namespace
}  // namespace exm
