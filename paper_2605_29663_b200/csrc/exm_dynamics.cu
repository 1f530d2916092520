// exm_dynamics.cu — sm_100a FP64 kernels of the EXACT-MPPI step: device noise, rollouts,
// rollout costs, softmax partials, update + validation rollout, finalize.
//
// Kernel map (reference function each one replaces, proj/...):
//   k_noise          sample_perturbations / gaussian_at      controller.cpp:78-96, rng.hpp:12-39
//   k_rollout        score_rollout minus the SDF and task    controller.cpp:138-174,
//                    cost (noise, clamp, Euler step)          kinematics.cpp:75-117
//   k_rollout_costs  task + control + obstacle cost, unsafe  controller.cpp:98-132, :151-171
//   k_block_partials augmented cost, min-shifted softmax     controller.cpp:222-233, :310-328
//                    partials
//   k_update         partial merge, weighted update,         controller.cpp:314-340
//                    sequential clamp, validation rollout     controller.cpp:254-282
//   k_finalize       validation cost, command, shift / hold  controller.cpp:342-364
//
// Compiled with -fmad=false: like the reference's x86-64 build, no multiply-add is fused, so
// every FP64 product and sum is rounded where the reference rounds it.
#include "exm_device.cuh"
#include "exm_exact64.cuh"

#ifdef EXM_TIMING  // phase timestamps of k_update (diagnostic builds only)
__device__ long long g_probe[16];
#define EXM_PROBE(i) \
  do {                \
    if (threadIdx.x == 0) g_probe[i] = clock64(); \
  } while (0)
extern "C" int exm_debug_probes(long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_probe, sizeof(g_probe)));
}
#else
#define EXM_PROBE(i) \
  do {               \
  } while (0)
#endif

namespace exm {
namespace {

// derivative + step (kinematics.cpp:75-97) are heading_rate / xy_rate below.

// project_on_polyline + task_cost, controller.cpp:50-66, :103-118
__device__ double task_cost(const StepConst& sc, const double q[3], const double* g, int ng,
                            const double* goal, bool terminal) {
  const double dx = q[0] - goal[0], dy = q[1] - goal[1];
  double cost = sc.w_goal_pos * (dx * dx + dy * dy);
  if (terminal) {
    const double e = wrap_angle(q[2] - goal[2]);
    cost += sc.w_goal_head * e * e;
  }
  double best_d, best_p = 0.0;
  if (ng == 1) {
    const double ax = q[0] - g[0], ay = q[1] - g[1];
    best_d = sqrt(ax * ax + ay * ay);
  } else {
    // Same values as the reference loop with fewer FP64 sqrt/div sequences: the quotient is
    // formed only when it is not clamped (num <= 0 -> t = 0, num >= len^2 -> t = 1 exactly, the
    // division being monotonic), and sqrt(e.e) only when e.e is below the best so far (sqrt is
    // monotonic, so e.e >= best_a implies d >= best_d and the reference keeps its best).
    best_d = HUGE_VAL;
    double best_a = HUGE_VAL, arc = 0.0;
    for (int i = 0; i + 1 < ng; ++i) {
      const double ax = g[2 * i], ay = g[2 * i + 1];
      const double sx = g[2 * i + 2] - ax, sy = g[2 * i + 3] - ay;
      const double len = sqrt(sx * sx + sy * sy);
      double t = 0.0;
      if (len > 0.0) {
        const double num = (q[0] - ax) * sx + (q[1] - ay) * sy, den = len * len;
        t = num <= 0.0 ? 0.0 : num >= den ? 1.0 : clampd(num / den, 0.0, 1.0);
      }
      const double ex = q[0] - (ax + t * sx), ey = q[1] - (ay + t * sy);
      const double a = ex * ex + ey * ey;
      if (a < best_a) {
        const double d = sqrt(a);
        if (d < best_d) {
          best_d = d;
          best_a = a;
          best_p = arc + t * len;
        }
      }
      arc += len;
    }
  }
  cost += sc.w_xtrack * best_d * best_d;
  cost -= sc.w_progress * best_p;
  return cost;
}

__device__ __forceinline__ double terminal_cost(const StepConst& sc, const double q[3],
                                                const double* goal) {  // controller.cpp:120-126
  const double dx = q[0] - goal[0], dy = q[1] - goal[1];
  const double e = wrap_angle(q[2] - goal[2]);
  return sc.w_goal_pos * (dx * dx + dy * dy) + sc.w_goal_head * e * e;
}

template <int TAG>
__device__ __forceinline__ double control_cost(const StepConst& sc, const double* u) {
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < model_dim<TAG>(); ++i) s += u[i] * u[i];
  return sc.w_ctrl * s;
}

__device__ __forceinline__ double obstacle_cost(const StepConst& sc, double d) {  // :98-101
  const double m = mx(sc.d_safe - d, 0.0);
  return sc.w_coll * (d < 0.0 ? 1.0 : 0.0) + sc.w_rep * m * m;
}

// FP64 dynamics with the reference's roundings: every product and sum below is rounded on its
// own (__dmul_rn / __dadd_rn: no FMA contraction), exactly as the reference's x86-64 build
// evaluates kinematics.cpp:75-117 and controller.cpp:151-167, so the clamped controls are
// bit-identical and the states differ only by the ulps of CUDA's vs glibc's sin/cos/tan.
//
// Heading rate of one clamped control (derivative, kinematics.cpp:75-92).
template <int TAG>
__device__ __forceinline__ double heading_rate(const StepConst& sc, const double* u) {
  if (TAG == EXM_MODEL_DIFF) return u[1];
  if (TAG == EXM_MODEL_ACKERMANN) return __dmul_rn(__ddiv_rn(u[0], sc.wheelbase), tan(u[1]));
  if (TAG == EXM_MODEL_OMNI) return u[2];
  if (TAG == EXM_MODEL_SPIN) return u[0];
  return 0.0;
}

template <int TAG>
__device__ __forceinline__ void xy_rate(const double* u, double ct, double st, double& fx,
                                        double& fy) {
  fx = 0.0;
  fy = 0.0;
  if (TAG == EXM_MODEL_DIFF || TAG == EXM_MODEL_ACKERMANN) {
    fx = __dmul_rn(u[0], ct);
    fy = __dmul_rn(u[0], st);
  }
  if (TAG == EXM_MODEL_OMNI) {
    fx = __dsub_rn(__dmul_rn(u[0], ct), __dmul_rn(u[1], st));
    fy = __dadd_rn(__dmul_rn(u[0], st), __dmul_rn(u[1], ct));
  }
  if (TAG == EXM_MODEL_PARALLEL) {
    fx = -__dmul_rn(u[0], st);
    fy = __dmul_rn(u[0], ct);
  }
}

// Device noise (sample_perturbations, controller.cpp:78-96 + rng.hpp:29-39) of one rollout:
// key of the (seed, cycle, r) row, then eps[h][c] for a (h, c) entry.
__device__ __forceinline__ uint64_t noise_row_key(const StepConst& sc, uint64_t cycle, int r) {
  return hash_mix(hash_mix(splitmix64(sc.seed), cycle), static_cast<uint64_t>(sc.r_offset + r));
}
__device__ __forceinline__ double noise_at(const StepConst& sc, uint64_t row_key, int h, int c) {
  const uint64_t kc = hash_mix(hash_mix(row_key, static_cast<uint64_t>(h)), static_cast<uint64_t>(c));
  const double u1 = unit_oc(hash_mix(kc, 0xD1B54A32D192ED03ull));
  const double u2 = unit_oc(hash_mix(kc, 0x8CB92BA72F3D8DD7ull));
  return sc.sigma[c] * (sqrt(-2.0 * log(u1)) * cos(2.0 * kPi * u2));
}

constexpr int kRolloutWarps = 4;  // rollouts (warps) per CTA in k_rollout
constexpr float kDstatClamp = 16.0f;       // d_min clamp in that mean (empty clouds: 1e6)
constexpr int kHstatEvery = 4;             // rollout blocks sampled for the per-step statistic
constexpr float kCapSigma = 3.0f;          // cap = mean + kCapSigma * std (+ kCapSlack * R)
constexpr float kCapSlack = 0.02f;

// The serial part of one rollout (score_rollout, controller.cpp:151-169, minus the SDF and the
// task cost, which k_rollout_costs computes in parallel over h), spread over one warp. Only
// true recurrences stay serial, each on its own lane and each a chain of single FP64 ops:
//   1. lanes stage u = nominal + eps (eps drawn on the fly when `draw`, else loaded)
//   2. lane c < D clamps component c over h (kinematics.cpp:99-117: the clamp of a component
//      depends on that component only); lanes then form the heading increments rate_h * dt
//   3. lane 0 sums the heading chain; lanes take sin/cos of every pre-step heading
//   4. lanes form the x/y increments; lane 0 sums the x chain while lane 1 sums the y chain
//   5. lanes write poses / positions / controls / states (coalesced)
// ctrl_out (optional): the control cost of every step (controller.cpp:128-132), summed later in
// the reference's order by k_rollout_costs / k_finalize. scratch: rollout_warp_scratch(T, D)
// doubles of shared memory per warp. Returns the terminal goal cost in every lane.
__host__ __device__ constexpr int rollout_warp_scratch(int T, int D) { return T * (D + 5); }

// xy_row (optional): pre-step positions; task_row (optional, with guide): the task cost of every
// pre-step state (controller.cpp:103-118), formed here off the step's critical path.
template <int TAG>
__device__ double rollout_warp(const StepConst& sc, const StepDyn& dyn, const double* nominal,
                               const double* eps_in, double* eps_out, uint64_t row_key,
                               float4* poses_row, double2* xy_row, double* controls_row,
                               double* states_row, double* ctrl_out, double* scratch,
                               double* task_row = nullptr, const double* guide = nullptr) {
  constexpr int D = model_dim<TAG>();
  const int T = sc.T, lane = threadIdx.x & 31;
  double* s_u = scratch;          // T*D controls (clamped in place)
  double* s_th = s_u + T * D;     // T heading increments, then pre-step headings
  double* s_c = s_th + T;         // T cos
  double* s_s = s_c + T;          // T sin
  double* s_x = s_s + T;          // T x increments, then pre-step x
  double* s_y = s_x + T;          // T y increments, then pre-step y
  for (int i = lane; i < T * D; i += 32) {
    double e = 0.0;
    if (eps_out) {
      e = noise_at(sc, row_key, i / D, i % D);
      eps_out[i] = e;
    } else if (eps_in) {
      e = eps_in[i];
    }
    // the velocity clamp of kinematics.cpp:105-112 does not depend on the previous control:
    // applied here in parallel, only the rate clamp (:113) stays in the serial chain
    const int c = i % D;
    double lo = sc.vel_min[c], hi = sc.vel_max[c];
    if (TAG == EXM_MODEL_ACKERMANN && c == 1) {
      lo = mx(lo, -sc.steer_max);
      hi = mn(hi, sc.steer_max);
    }
    s_u[i] = clampd(__dadd_rn(nominal[i], e), lo, hi);
  }
  __syncwarp();
  EXM_PROBE(4);
  if (lane < D) {
    const double amin = __dmul_rn(sc.acc_min[lane], sc.dt), amax = __dmul_rn(sc.acc_max[lane], sc.dt);
    double prev = dyn.u_prev[lane];
#pragma unroll 5
    for (int h = 0; h < T; ++h) {
      const double v = s_u[h * D + lane];
      prev = clampd(v, __dadd_rn(prev, amin), __dadd_rn(prev, amax));
      s_u[h * D + lane] = prev;
    }
  }
  __syncwarp();
  EXM_PROBE(5);
  for (int h = lane; h < T; h += 32) {
    double uc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < D; ++c) uc[c] = s_u[h * D + c];
    s_th[h] = __dmul_rn(heading_rate<TAG>(sc, uc), sc.dt);
    if (ctrl_out) ctrl_out[h] = control_cost<TAG>(sc, uc);
  }
  __syncwarp();
  if (lane == 0) {
    double th = dyn.q0[2];
#pragma unroll 5
    for (int h = 0; h < T; ++h) {
      const double inc = s_th[h];
      s_th[h] = th;
      th = __dadd_rn(th, inc);
    }
    s_c[0] = th;  // theta_T, parked until the sincos pass reads s_th
  }
  __syncwarp();
  EXM_PROBE(6);
  const double thT = s_c[0];
  __syncwarp();
  for (int h = lane; h < T; h += 32) {
    double st, ct;
    sincos(s_th[h], &st, &ct);
    s_s[h] = st;
    s_c[h] = ct;
    double uc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < D; ++c) uc[c] = s_u[h * D + c];
    double fx, fy;
    xy_rate<TAG>(uc, ct, st, fx, fy);
    s_x[h] = __dmul_rn(fx, sc.dt);
    s_y[h] = __dmul_rn(fy, sc.dt);
  }
  __syncwarp();
  EXM_PROBE(7);
  double endp = 0.0;
  if (lane < 2) {
    double* chain = lane == 0 ? s_x : s_y;
    double v = dyn.q0[lane];
#pragma unroll 5
    for (int h = 0; h < T; ++h) {
      const double inc = chain[h];
      chain[h] = v;
      v = __dadd_rn(v, inc);
    }
    endp = v;
  }
  EXM_PROBE(8);
  const double xT = __shfl_sync(kFull, endp, 0), yT = __shfl_sync(kFull, endp, 1);
  const double qT[3] = {xT, yT, thT};
  const double base = terminal_cost(sc, qT, dyn.goal);
  if (states_row && lane == 0) {
    states_row[3 * T] = xT;
    states_row[3 * T + 1] = yT;
    states_row[3 * T + 2] = thT;
  }
  __syncwarp();
  const double qx0 = dyn.q0[0], qy0 = dyn.q0[1];
  for (int h = lane; h < T; h += 32) {
    poses_row[h] = make_float4(static_cast<float>(s_x[h] - qx0), static_cast<float>(s_y[h] - qy0),
                               static_cast<float>(s_c[h]), static_cast<float>(s_s[h]));
    if (xy_row) xy_row[h] = make_double2(s_x[h], s_y[h]);
    if (task_row) {
      const double q[3] = {s_x[h], s_y[h], 0.0};
      task_row[h] = task_cost(sc, q, guide, dyn.n_guide, dyn.goal, false);
    }
    if (states_row) {
      states_row[3 * h] = s_x[h];
      states_row[3 * h + 1] = s_y[h];
      states_row[3 * h + 2] = s_th[h];
    }
  }
  if (controls_row)
    for (int i = lane; i < T * D; i += 32) controls_row[i] = s_u[i];
  __syncwarp();
  return base;
}


__global__ void k_noise(const StepConst sc, const StepDyn* __restrict__ dyn,
                        double* __restrict__ eps) {
  pdl_wait();
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;  // local (r, h)
  if (idx >= sc.k_local * sc.T) return;
  const int r = idx / sc.T, h = idx % sc.T;
  const uint64_t key = noise_row_key(sc, dyn->cycle, r);
  for (int c = 0; c < sc.D; ++c) eps[static_cast<size_t>(idx) * sc.D + c] = noise_at(sc, key, h, c);
}

// The next control step's device noise, generated in the idle tail of this step (after the
// softmax partials, the last reader of eps): cycle = the cycle this step's rollout drew + 1.
// The next rollout finds sc.nstate[1] == its cycle and reads eps instead of drawing (a
// different cycle, e.g. a caller restarting the sequence, simply draws). One thread per (r, h).
__global__ void k_noise_pregen(const StepConst sc, double* __restrict__ eps) {
  pdl_wait();
  const uint64_t cycle = sc.nstate[0] + 1;
  if (blockIdx.x == 0 && threadIdx.x == 0) sc.nstate[1] = cycle;  // read by the next graph
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= sc.k_local * sc.T) return;
  const int r = idx / sc.T, h = idx - r * sc.T;
  const uint64_t key = noise_row_key(sc, cycle, r);
  for (int c = 0; c < sc.D; ++c) eps[static_cast<size_t>(idx) * sc.D + c] = noise_at(sc, key, h, c);
}

template <int TAG>
__global__ void __launch_bounds__(kRolloutWarps * 32) k_rollout(
    const StepConst sc, const StepDyn* __restrict__ dynp, const double* __restrict__ nominal,
    double* __restrict__ eps, int draw, float4* __restrict__ poses, double* __restrict__ task,
    const double* __restrict__ guide, int guide_cap, double* __restrict__ base_cost,
    double* __restrict__ ctrl_cost, double* __restrict__ controls_out,
    double* __restrict__ states_out) {
  pdl_wait();
  // One warp per rollout (rollout_warp). draw: the perturbations are drawn here (device noise,
  // written to eps for the softmax update); else eps holds injected perturbations.
  extern __shared__ double sm[];
  const int TD = sc.T * sc.D;
  double* s_guide = sm;
  double* nom = sm + 2 * guide_cap;
  const int warp = threadIdx.x >> 5;
  double* scratch = nom + TD + warp * rollout_warp_scratch(sc.T, sc.D);
  for (int i = threadIdx.x; i < TD; i += blockDim.x) nom[i] = nominal[i];
  const StepDyn dyn = *dynp;
  for (int i = threadIdx.x; i < 2 * dyn.n_guide; i += blockDim.x) s_guide[i] = guide[i];
  const bool gen = draw && !(sc.nstate && sc.nstate[1] == dyn.cycle);  // else pregenerated
  if (draw && sc.nstate && blockIdx.x == 0 && threadIdx.x == 0) sc.nstate[0] = dyn.cycle;
  __syncthreads();
  const int r = blockIdx.x * kRolloutWarps + warp;
  if (r >= sc.k_local) return;  // warp-uniform
  const size_t row = static_cast<size_t>(r) * sc.T;
  double* eps_row = eps + row * sc.D;
  const double b = rollout_warp<TAG>(
      sc, dyn, nom, gen ? nullptr : eps_row, gen ? eps_row : nullptr,
      gen ? noise_row_key(sc, dyn.cycle, r) : 0ull, poses + row, nullptr,
      controls_out ? controls_out + row * sc.D : nullptr,
      states_out ? states_out + static_cast<size_t>(r) * (sc.T + 1) * 3 : nullptr, ctrl_cost + row,
      scratch, task + row, s_guide);
  if ((threadIdx.x & 31) == 0) base_cost[r] = b;
}

// The same rollouts as k_rollout with the recurrences on one LANE per rollout: a CTA of
// kLaneThreads threads takes R rollouts; the parallel work (noise, velocity clamp, heading
// rates, control costs, sin/cos, xy rates, stores) is spread over all (r, h, c) items, and each
// serial recurrence (rate clamp per component, heading, x, y) runs on R lanes side by side,
// so a chain instruction serves R rollouts instead of one. Every value is produced by the
// same single-rounded FP64 operations in the same order as rollout_warp (bit-identical).
// Shared memory ([item][R + 1] rows: conflict-free lanes over r):
//   u[T*D], a[T] (heading increments -> pre-step headings), x[T], y[T] doubles, cs[T] float2
constexpr int kLaneThreads = 256;
__host__ __device__ constexpr size_t rollout_lanes_smem(int T, int D, int R, int guide_cap) {
  return sizeof(double) * (static_cast<size_t>(T) * (D + 3) * (R + 1) + static_cast<size_t>(T) * D +
                           3 * R + 2 * static_cast<size_t>(guide_cap)) +
         sizeof(uint64_t) * R + sizeof(float2) * static_cast<size_t>(T) * (R + 1);
}

template <int TAG, int R>
__global__ void __launch_bounds__(1024) k_rollout_lanes(
    const StepConst sc, const StepDyn* __restrict__ dynp, const double* __restrict__ nominal,
    double* __restrict__ eps, int draw, float4* __restrict__ poses, double* __restrict__ task,
    const double* __restrict__ guide, int guide_cap, double* __restrict__ base_cost,
    double* __restrict__ ctrl_cost, double* __restrict__ controls_out,
    double* __restrict__ states_out) {
  pdl_wait();
  constexpr int D = model_dim<TAG>();
  constexpr int P = R + 1;
  const int T = sc.T, TD = T * D, tid = threadIdx.x, nthr = blockDim.x;
  extern __shared__ double smd[];
  double* s_u = smd;                          // [TD][P]
  double* s_a = s_u + static_cast<size_t>(TD) * P;  // [T][P]
  double* s_x = s_a + static_cast<size_t>(T) * P;
  double* s_y = s_x + static_cast<size_t>(T) * P;
  double* s_nom = s_y + static_cast<size_t>(T) * P;  // [TD]
  double* s_end = s_nom + TD;                 // [3][R]: x_T, y_T, theta_T
  double* s_guide = s_end + 3 * R;            // [2 * guide_cap]: the guidance polyline
  uint64_t* s_key = reinterpret_cast<uint64_t*>(s_guide + 2 * guide_cap);
  float2* s_cs = reinterpret_cast<float2*>(s_key + R);  // [T][P]
  const int r0 = blockIdx.x * R;
  const int nr = min(R, sc.k_local - r0);
  if (nr <= 0) return;
  const StepDyn dyn = *dynp;
  // eps already holds this cycle's noise when the previous step pregenerated it
  const bool gen = draw && !(sc.nstate && sc.nstate[1] == dyn.cycle);
  if (draw && sc.nstate && blockIdx.x == 0 && tid == 0) sc.nstate[0] = dyn.cycle;
  for (int i = tid; i < TD; i += nthr) s_nom[i] = nominal[i];
  for (int i = tid; i < 2 * dyn.n_guide; i += nthr) s_guide[i] = guide[i];
  if (gen && tid < R) s_key[tid] = noise_row_key(sc, dyn.cycle, r0 + tid);
  __syncthreads();
  // 1. u = clamp_velocity(nominal + eps); eps drawn here (device noise) or loaded, kPre
  //    loads per thread in flight together (the rows come from HBM)
  constexpr int kPre = 8;
  double* erow = eps + static_cast<size_t>(r0) * TD;
  const int n_items = nr * TD;
  for (int base = tid; base < n_items; base += nthr * kPre) {
    double ev[kPre];
#pragma unroll
    for (int k = 0; k < kPre; ++k) {
      const int idx = base + k * nthr;
      ev[k] = (!gen && idx < n_items) ? erow[idx] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < kPre; ++k) {
      const int idx = base + k * nthr;
      if (idx >= n_items) break;
      const int r = idx / TD, o = idx - r * TD, c = o % D;
      double e = ev[k];
      if (gen) {
        e = noise_at(sc, s_key[r], o / D, c);
        erow[idx] = e;
      }
      double lo = sc.vel_min[c], hi = sc.vel_max[c];
      if (TAG == EXM_MODEL_ACKERMANN && c == 1) {
        lo = mx(lo, -sc.steer_max);
        hi = mn(hi, sc.steer_max);
      }
      s_u[o * P + r] = clampd(__dadd_rn(s_nom[o], e), lo, hi);
    }
  }
  __syncthreads();
  // 2. rate clamp, one lane per (component, rollout) (kinematics.cpp:113)
  if (tid < D * R) {
    const int r = tid % R, c = tid / R;
    if (r < nr) {
      const double amin = __dmul_rn(sc.acc_min[c], sc.dt), amax = __dmul_rn(sc.acc_max[c], sc.dt);
      double prev = dyn.u_prev[c];
      double* col = s_u + c * P + r;
#pragma unroll 5
      for (int h = 0; h < T; ++h) {
        prev = clampd(col[h * D * P], __dadd_rn(prev, amin), __dadd_rn(prev, amax));
        col[h * D * P] = prev;
      }
    }
  }
  __syncthreads();
  // 3. heading increments and control costs
  for (int idx = tid; idx < nr * T; idx += nthr) {
    const int r = idx / T, h = idx - r * T;
    double uc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < D; ++c) uc[c] = s_u[(h * D + c) * P + r];
    s_a[h * P + r] = __dmul_rn(heading_rate<TAG>(sc, uc), sc.dt);
    ctrl_cost[static_cast<size_t>(r0) * T + idx] = control_cost<TAG>(sc, uc);
  }
  __syncthreads();
  // 4. heading chain
  if (tid < nr) {
    double th = dyn.q0[2];
#pragma unroll 5
    for (int h = 0; h < T; ++h) {
      const double inc = s_a[h * P + tid];
      s_a[h * P + tid] = th;
      th = __dadd_rn(th, inc);
    }
    s_end[2 * R + tid] = th;
  }
  __syncthreads();
  // 5. sin / cos of every pre-step heading, xy increments
  for (int idx = tid; idx < nr * T; idx += nthr) {
    const int r = idx / T, h = idx - r * T;
    double st, ct;
    sincos(s_a[h * P + r], &st, &ct);
    s_cs[h * P + r] = make_float2(static_cast<float>(ct), static_cast<float>(st));
    double uc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < D; ++c) uc[c] = s_u[(h * D + c) * P + r];
    double fx, fy;
    xy_rate<TAG>(uc, ct, st, fx, fy);
    s_x[h * P + r] = __dmul_rn(fx, sc.dt);
    s_y[h * P + r] = __dmul_rn(fy, sc.dt);
  }
  __syncthreads();
  // 6. x and y chains, one lane each per rollout
  if (tid < 2 * R) {
    const int r = tid % R, k = tid / R;
    if (r < nr) {
      double* chain = (k == 0 ? s_x : s_y) + r;
      double v = dyn.q0[k];
#pragma unroll 5
      for (int h = 0; h < T; ++h) {
        const double inc = chain[h * P];
        chain[h * P] = v;
        v = __dadd_rn(v, inc);
      }
      s_end[k * R + r] = v;
    }
  }
  __syncthreads();
  // 7. stores (rows of consecutive h: coalesced), the task cost of every pre-step state
  //    (controller.cpp:103-118: d_min-independent, so formed here, beside the cloud preparation,
  //    instead of in the step's serial tail) and the terminal cost
  const double qx0 = dyn.q0[0], qy0 = dyn.q0[1];
  for (int idx = tid; idx < nr * T; idx += nthr) {
    const int r = idx / T, h = idx - r * T;
    const double x = s_x[h * P + r], y = s_y[h * P + r];
    const float2 cs = s_cs[h * P + r];
    const size_t g = static_cast<size_t>(r0) * T + idx;
    poses[g] = make_float4(static_cast<float>(x - qx0), static_cast<float>(y - qy0), cs.x, cs.y);
    const double q[3] = {x, y, 0.0};
    task[g] = task_cost(sc, q, s_guide, dyn.n_guide, dyn.goal, false);
    if (states_out) {
      double* srow = states_out + static_cast<size_t>(r0 + r) * (T + 1) * 3;
      srow[3 * h] = x;
      srow[3 * h + 1] = y;
      srow[3 * h + 2] = s_a[h * P + r];
    }
  }
  if (controls_out)
    for (int idx = tid; idx < nr * TD; idx += nthr) {
      const int r = idx / TD, o = idx - r * TD;
      controls_out[static_cast<size_t>(r0) * TD + idx] = s_u[o * P + r];
    }
  if (tid < nr) {
    const double qT[3] = {s_end[tid], s_end[R + tid], s_end[2 * R + tid]};
    base_cost[r0 + tid] = terminal_cost(sc, qT, dyn.goal);
    if (states_out) {
      double* srow = states_out + static_cast<size_t>(r0 + tid) * (T + 1) * 3;
      srow[3 * T] = qT[0];
      srow[3 * T + 1] = qT[1];
      srow[3 * T + 2] = qT[2];
    }
  }
}

// Rollout cost J_r and unsafe flag chi_r (score_rollout, controller.cpp:151-171), one warp per
// rollout: lanes take the task and obstacle cost (controller.cpp:98-118) of the pre-step states
// h = lane, lane + 32, ... into shared memory; lane 0 then accumulates
//   cost += task_h; cost += ctrl_h; cost += obst_h   (h = 0 .. T-1), cost += terminal
// in exactly the reference's order (with k_rollout's control and terminal costs), so J_r is
// the reference's value for the same d_min. Also accumulates the search-radius statistic of
// the next step's cell size (k_cloud_prep).
template <int kCostWarps, bool kF64 = false>
__global__ void __launch_bounds__(kCostWarps * 32) k_rollout_costs(
    const StepConst sc, const double* __restrict__ task, const double* __restrict__ base_cost,
    const double* __restrict__ ctrl_cost, const float* __restrict__ dmin,
    double* __restrict__ cost, uint8_t* __restrict__ unsafe, float* __restrict__ dstat,
    float* __restrict__ hstat, const double* __restrict__ dmin64) {
  pdl_wait();
  extern __shared__ double g[];  // per warp: task[T], obst[T], ctrl[T]; then 2T floats
  __shared__ float red[2][kCostWarps];
  const int ng = 0, T = sc.T;
  float* sh = reinterpret_cast<float*>(g + 2 * ng + kCostWarps * 3 * T);
  // every kHstatEvery-th block samples the per-step d_min statistic (k_finalize -> caps)
  const bool sampled = hstat != nullptr && blockIdx.x % kHstatEvery == 0;
  if (sampled)
    for (int i = threadIdx.x; i < 2 * T; i += blockDim.x) sh[i] = 0.f;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* s_t = g + 2 * ng + warp * 3 * T;
  double* s_o = s_t + T;
  double* s_c = s_o + T;
  const int r = blockIdx.x * kCostWarps + warp;
  const bool live = r < sc.k_local;  // warp-uniform
  float dc = 0.f;
  bool bad = false;
  if (live) {
    const size_t row = static_cast<size_t>(r) * T;
    for (int h = lane; h < T; h += 32) {
      // kF64: the FP64 minima of exm_evaluate_rollouts under EXM_OPT_SDF_FP64 (a separate
      // instantiation: the control cycle's FP32 kernel carries no extra branch)
      const float df = kF64 ? static_cast<float>(dmin64[row + h]) : dmin[row + h];
      const double d = kF64 ? dmin64[row + h] : static_cast<double>(df);
      s_t[h] = task[row + h];  // formed by the rollout kernel
      s_o[h] = obstacle_cost(sc, d);
      s_c[h] = ctrl_cost[row + h];  // staged: the serial sum below reads shared memory only
      bad |= d < sc.d_safe;
      dc += fminf(fmaxf(df, 0.f), kDstatClamp);
      if (sampled) {
        const float dv = fminf(df, kDstatClamp);
        atomicAdd(&sh[h], dv);
        atomicAdd(&sh[T + h], dv * dv);
      }
    }
  }
  for (int o = 16; o; o >>= 1) dc += __shfl_xor_sync(kFull, dc, o);
  bad = __any_sync(kFull, bad);
  if (lane == 0) {
    if (live) unsafe[r] = bad ? 1 : 0;
    red[0][warp] = live ? dc : 0.f;
    red[1][warp] = live ? static_cast<float>(T) : 0.f;
  }
  __syncthreads();
  // J_r in the reference's order, one lane of warp 0 per rollout of the CTA (the serial sums of
  // the kCostWarps rollouts run side by side instead of on one lane of every warp)
  if (warp == 0 && lane < kCostWarps) {
    const int rr = blockIdx.x * kCostWarps + lane;
    if (rr < sc.k_local) {
      const double* t_ = g + 2 * ng + lane * 3 * T;
      const double jb = base_cost[rr];
      double J = 0.0;
#pragma unroll 10
      for (int h = 0; h < T; ++h) {
        J += t_[h];
        J += t_[2 * T + h];
        J += t_[T + h];
      }
      cost[rr] = J + jb;
    }
  }
  if (sampled) {
    for (int i = threadIdx.x; i < 2 * T; i += blockDim.x) atomicAdd(&hstat[i], sh[i]);
    if (threadIdx.x == 0) {
      int n = 0;
      for (int w = 0; w < kCostWarps; ++w) n += blockIdx.x * kCostWarps + w < sc.k_local;
      atomicAdd(&hstat[2 * T], static_cast<float>(n));
    }
  }
  if (threadIdx.x == 0) {  // one atomic pair per block
    float a = 0.f, c = 0.f;
    for (int w = 0; w < kCostWarps; ++w) {
      a += red[0][w];
      c += red[1][w];
    }
    if (c > 0.f) {
      atomicAdd(dstat, a);
      atomicAdd(dstat + 1, c);
    }
  }
}

// Augmented cost and the min-shifted softmax partial of one block of kBlockRollouts rollouts
// (fixed block size and fixed reduction trees: deterministic and independent of sharding).
//   Jt_r = J_r + w_inf * unsafe_r                       controller.cpp:310-312
//   {beta_b, S_b, A_b, argmin_b, U_b[T*D]}              controller.cpp:222-233, :316-328
// Grid (block, column group): every CTA recomputes the block's beta and weights (256 exps) and
// sums one group of kPartCols columns (h, c) of U_b, one column per lane, the 8 warps over
// interleaved rollouts, then the warp sums in warp order; column group 0 also writes the header.
// The eps rows are read by blocks x column groups CTAs instead of one CTA per block.
constexpr int kPartCols = 32;
__global__ void __launch_bounds__(kBlockRollouts) k_block_partials(
    const StepConst sc, const double* __restrict__ cost, const uint8_t* __restrict__ unsafe,
    const double* __restrict__ eps, double* __restrict__ partials) {
  pdl_wait();
  constexpr int kWarps = kBlockRollouts / 32;
  __shared__ double s_e[kBlockRollouts];
  __shared__ double s_v[kWarps];
  __shared__ double s_a[kWarps];
  __shared__ int s_i[kWarps];
  __shared__ double s_u[kWarps][kPartCols];
  __shared__ double s_beta;
  __shared__ int s_arg;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r0 = blockIdx.x * kBlockRollouts;
  const int r = r0 + tid;
  const bool valid = r < sc.k_local;
  const int TD = sc.T * sc.D;
  const int o = blockIdx.y * kPartCols + lane;
  const int nv = min(kBlockRollouts, sc.k_local - r0);
  // this lane's column of rows warp, warp + 8, ... fetched first: the loads do not depend on
  // the weights, so their latency overlaps the argmin / exp phase
  constexpr int kRows = kBlockRollouts / kWarps;
  double ev[kRows];
  {
    const double* col = eps + static_cast<size_t>(r0) * TD + o;
#pragma unroll
    for (int k = 0; k < kRows; ++k) {
      const int j = warp + k * kWarps;
      ev[k] = (o < TD && j < nv) ? col[static_cast<size_t>(j) * TD] : 0.0;
    }
  }
  double jt = HUGE_VAL;
  if (valid) jt = unsafe[r] ? cost[r] + sc.w_inf : cost[r];
  // argmin with first-index tie break (std::min_element)
  double v = jt;
  int vi = valid ? sc.r_offset + r : 0x7fffffff;
  for (int k = 16; k; k >>= 1) {
    const double ov = __shfl_xor_sync(kFull, v, k);
    const int oi = __shfl_xor_sync(kFull, vi, k);
    if (ov < v || (ov == v && oi < vi)) { v = ov; vi = oi; }
  }
  if (lane == 0) { s_v[warp] = v; s_i[warp] = vi; }
  __syncthreads();
  if (tid == 0) {
    double b = s_v[0];
    int bi = s_i[0];
    for (int w = 1; w < kWarps; ++w)
      if (s_v[w] < b || (s_v[w] == b && s_i[w] < bi)) { b = s_v[w]; bi = s_i[w]; }
    s_beta = b;
    s_arg = bi;
  }
  __syncthreads();
  const double beta = s_beta;
  const double z = valid ? (jt - beta) / sc.lambda : 0.0;
  const double e = valid ? exp(-z) : 0.0;
  s_e[tid] = e;
  const int stride = partial_stride(sc.T, sc.D);
  double* out = partials + static_cast<size_t>(sc.block_offset + blockIdx.x) * stride;
  if (blockIdx.y == 0) {
    const double a = valid ? e * z : 0.0;
    double se = e, sa = a;
    for (int k = 16; k; k >>= 1) {
      se += __shfl_xor_sync(kFull, se, k);
      sa += __shfl_xor_sync(kFull, sa, k);
    }
    __syncthreads();  // s_v reuse: the argmin values were consumed by thread 0 above
    if (lane == 0) { s_v[warp] = se; s_a[warp] = sa; }
    __syncthreads();
    if (tid == 0) {
      double S = 0.0, A = 0.0;
      for (int w = 0; w < kWarps; ++w) { S += s_v[w]; A += s_a[w]; }
      out[0] = beta;
      out[1] = S;
      out[2] = A;
      out[3] = static_cast<double>(s_arg);
    }
  } else {
    __syncthreads();
  }
  // U_b[o] = sum_r e_r eps[r][o]: warp w sums rollouts w, w + 8, ... (rows coalesced over the
  // lanes' columns), then the warp sums are added in warp order
  double acc = 0.0;
#pragma unroll
  for (int k = 0; k < kRows; ++k) acc += s_e[warp + k * kWarps] * ev[k];  // e = 0 past nv
  s_u[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && o < TD) {
    double u = 0.0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) u += s_u[w][lane];
    out[4 + o] = u;
  }
}

// Merge all block partials in block order (every rank does this identically), apply the
// weighted update u_h += U_h / S (controller.cpp:320-328), then one thread runs the sequential
// clamp + validation dynamics (controller.cpp:331-340, :254-282).
template <int TAG>
__global__ void __launch_bounds__(256) k_update(const StepConst sc,
                                                const double* __restrict__ partials,
                                                const double* __restrict__ nominal,
                                                const StepDyn* __restrict__ dynp,
                                                double* __restrict__ upd,
                                                float4* __restrict__ val_poses,
                                                double2* __restrict__ val_xy,
                                                double* __restrict__ val_base,
                                                DecisionDev* __restrict__ dec, int merge) {
  pdl_wait();
  extern __shared__ double sm_u[];  // T*D updated controls, nb factors, nb betas; then scratch
  __shared__ double s_beta, s_S;
  __shared__ StepDyn s_dyn;  // staged now: its load overlaps the merge instead of the rollout
  const int tid = threadIdx.x, lane = tid & 31;
  const int nb = sc.nblocks_total;
  const int stride = partial_stride(sc.T, sc.D);
  const int TD = sc.T * sc.D;
  static_assert(sizeof(StepDyn) % sizeof(uint64_t) == 0, "StepDyn copied as 8-byte words");
  constexpr int kDynWords = sizeof(StepDyn) / sizeof(uint64_t);
  if (tid >= blockDim.x - kDynWords)  // the last threads (idle in the U sums of every config)
    reinterpret_cast<uint64_t*>(&s_dyn)[tid - (blockDim.x - kDynWords)] =
        reinterpret_cast<const uint64_t*>(dynp)[tid - (blockDim.x - kDynWords)];
  const double nom0 = tid < TD ? nominal[tid] : 0.0;  // this thread's first nominal control
  double* s_upd = sm_u;
  double* sf = sm_u + TD;
  EXM_PROBE(0);
  if (merge) {
    double* sb = sf + nb;      // beta_b, then z_b = (beta_b - beta) / lambda
    double* sS = sb + nb;      // S_b
    double* sA = sS + nb;      // A_b
    double* sg = sA + nb;      // argmin_b
    for (int b = tid; b < nb; b += blockDim.x) {
      const double* p = partials + static_cast<size_t>(b) * stride;
      sb[b] = p[0];
      sS[b] = p[1];
      sA[b] = p[2];
      sg[b] = p[3];
    }
    __syncthreads();
    if (tid < 32) {  // beta = min_b beta_b, first block on ties (blocks are in rollout order)
      double v = HUGE_VAL;
      int vi = 0x7fffffff;
      for (int b = lane; b < nb; b += 32)
        if (sb[b] < v) { v = sb[b]; vi = b; }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(kFull, v, o);
        const int oi = __shfl_xor_sync(kFull, vi, o);
        if (ov < v || (ov == v && oi < vi)) { v = ov; vi = oi; }
      }
      if (tid == 0) {
        s_beta = v;
        dec->argmin = static_cast<int>(sg[vi]);
        dec->best_cost = v;
      }
    }
    __syncthreads();
    EXM_PROBE(1);
    for (int b = tid; b < nb; b += blockDim.x) {
      const double z = (sb[b] - s_beta) / sc.lambda;
      sb[b] = z;
      sf[b] = exp(-z);
    }
    __syncthreads();
    // block order: deterministic, independent of the GPU count. On the CTA's last thread, which
    // holds no U column when T * D < blockDim (every benchmark config), so warp 0's U sums do
    // not wait behind the serial S / A chains, the division and the log
    if (tid == blockDim.x - 1) {
      double S = 0.0, A = 0.0;
      for (int b = 0; b < nb; ++b) {
        S += sf[b] * sS[b];
        A += sf[b] * (sA[b] + sS[b] * sb[b]);
      }
      s_S = S;
      dec->entropy = A / S + log(S);
    }
    // U_o = sum_b f_b U_b[o] needs only the factors: overlaps thread 0's S / A sums
    double U[4] = {0.0, 0.0, 0.0, 0.0};
    for (int k = 0, o = tid; k < 4 && o < TD; ++k, o += blockDim.x) {
#pragma unroll 16
      for (int b = 0; b < nb; ++b) U[k] += sf[b] * partials[static_cast<size_t>(b) * stride + 4 + o];
    }
    __syncthreads();
    EXM_PROBE(2);
    for (int k = 0, o = tid; o < TD; ++k, o += blockDim.x) {
      double u = 0.0;
      if (k < 4) {
        u = U[k];
      } else {  // T * D > 4 * blockDim: the remaining outputs
#pragma unroll 16
        for (int b = 0; b < nb; ++b) u += sf[b] * partials[static_cast<size_t>(b) * stride + 4 + o];
      }
      s_upd[o] = (k == 0 ? nom0 : nominal[o]) + u / s_S;
    }
  } else {
    for (int o = tid; o < TD; o += blockDim.x) s_upd[o] = o == tid ? nom0 : nominal[o];
  }
  __syncthreads();
  EXM_PROBE(3);
  if (tid < 32) {
    // warp 0 clamps sequentially from u_prev and writes the clamped sequence back; the
    // reference's second clamp inside validate_nominal is idempotent on it.
    const double b = rollout_warp<TAG>(sc, s_dyn, s_upd, nullptr, nullptr, 0ull, val_poses, val_xy,
                                       upd, nullptr, val_base + 1,
                                       sf + (merge ? 5 * nb : 0));
    if (tid == 0) *val_base = b;
    EXM_PROBE(9);
  }
}

// Validation cost, validity, command and shift / zero-hold (controller.cpp:339-364).
__global__ void __launch_bounds__(64) k_finalize(
    const StepConst sc, const float* __restrict__ val_dmin, const double2* __restrict__ val_xy,
    const double* __restrict__ val_base, const double* __restrict__ upd,
    const double* __restrict__ guide, double* __restrict__ nominal, StepDyn* __restrict__ dyn,
    DecisionDev* __restrict__ dec, double* __restrict__ out_dmin,
    double* __restrict__ out_nominal, double* __restrict__ out_uprev, int commit,
    float* __restrict__ hstat, float* __restrict__ cap, float radius) {
  pdl_wait();
  extern __shared__ double sm2[];  // guide (2*ng) then per-step task (T) and obstacle (T) costs
  __shared__ int s_ok;
  const int tid = threadIdx.x;
  const int T = sc.T, D = sc.D;
  // every load of this thread's first step issued together with the header loads (one L2
  // round trip instead of one after the guide has been staged)
  const bool first = tid < T;
  const float dmin0 = first ? val_dmin[tid] : 0.f;
  const double2 xy0 = first ? val_xy[tid] : make_double2(0.0, 0.0);
  const double ctrl0 = first ? val_base[1 + tid] : 0.0;
  const double goal[3] = {dyn->goal[0], dyn->goal[1], dyn->goal[2]};
  const int ng = dyn->n_guide;
  double* g = sm2;
  double* c_t = sm2 + 2 * ng;
  double* c_o = c_t + T;
  double* c_c = c_o + T;  // val_base = {terminal, ctrl[T]}, staged
  for (int i = tid; i < 2 * ng; i += blockDim.x) g[i] = guide[i];
  if (tid == 0) s_ok = 1;
  __syncthreads();
  for (int h = tid; h < T; h += blockDim.x) {
    const bool f = h == tid;
    const double d = static_cast<double>(f ? dmin0 : val_dmin[h]);
    if (out_dmin) out_dmin[h] = d;
    if (d < sc.d_safe) atomicAnd(&s_ok, 0);
    const double2 xy = f ? xy0 : val_xy[h];
    const double q[3] = {xy.x, xy.y, 0.0};
    c_t[h] = task_cost(sc, q, g, ng, goal, false);
    c_o[h] = obstacle_cost(sc, d);
    c_c[h] = f ? ctrl0 : val_base[1 + h];
  }
  __syncthreads();
  const int ok = s_ok;
  if (tid == 0) {  // validate_nominal's order (controller.cpp:268-279)
    const double jb = val_base[0];
    double J = 0.0;
#pragma unroll 10
    for (int h = 0; h < T; ++h) {
      J += c_t[h];
      J += c_c[h];
      J += c_o[h];
    }
    dec->nominal_cost = J + jb;
    dec->validated = ok;
  }
  if (!commit) return;
  if (hstat != nullptr) {
    // next step's per-step caps for k_sdf_grid: that step's nominal is this one shifted by one,
    // so its step h looks like this step's h + 1 (a guess only: the SDF is exact for any cap)
    const float n = hstat[2 * T];
    for (int h = tid; h < T; h += blockDim.x) {
      const int src = h + 1 < T ? h + 1 : T - 1;
      float c = __int_as_float(0x7f800000);
      if (n > 0.f) {
        const float m = hstat[src] / n;
        const float v = fmaxf(hstat[T + src] / n - m * m, 0.f);
        c = m + kCapSigma * sqrtf(v) + kCapSlack * radius;
      }
      cap[h] = c;
    }
    __syncthreads();
    for (int i = tid; i <= 2 * T; i += blockDim.x) hstat[i] = 0.f;
  }
  for (int i = tid; i < T * D; i += blockDim.x) {
    const int h = i / D;
    const double v = ok ? upd[(h + 1 < T ? h + 1 : T - 1) * D + i % D] : 0.0;
    nominal[i] = v;
    if (out_nominal) out_nominal[i] = v;
  }
  if (tid < 3) {
    const double cmd = (ok && tid < D) ? upd[tid] : 0.0;
    dec->command[tid] = cmd;
    dyn->u_prev[tid] = cmd;
    if (out_uprev) out_uprev[tid] = cmd;
  }
  if (tid == 0) dyn->cycle += 1;
}

}  // namespace

// ------------------------------------------------------------------ launchers
cudaError_t launch_noise(const StepConst& sc, const StepDyn* dyn, double* eps, cudaStream_t s) {
  const int n = sc.k_local * sc.T;
  if (n <= 0) return cudaSuccess;
  { if (const cudaError_t le = launch_k(k_noise, (n + 255) / 256, 256, 0, s, sc, dyn, eps); le != cudaSuccess) return le; }
  return cudaGetLastError();
}

template <int TAG, int R>
cudaError_t rollout_lanes_launch(const StepConst& sc, const StepDyn* dyn, const double* nominal,
                                 double* eps, int draw, float4* poses, double* task,
                                 const double* guide, int guide_cap, double* base_cost,
                                 double* ctrl_cost, double* controls_out, double* states_out,
                                 size_t smem, cudaStream_t s) {
  // (per launch: the attribute is per device, and launches are captured into graphs)
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_rollout_lanes<TAG, R>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  if (const cudaError_t le = launch_k(k_rollout_lanes<TAG, R>, (sc.k_local + R - 1) / R,
                                      kLaneThreads, smem, s, sc, dyn, nominal, eps, draw, poses,
                                      task, guide, guide_cap, base_cost, ctrl_cost, controls_out,
                                      states_out);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

// Lanes per rollout (8 rollouts per CTA) when the CTA's shared memory fits, else 16, warp per
// rollout otherwise (very long horizons). -DEXM_ROLLOUT_WARP builds the warp kernel only (A/B).
#ifdef EXM_ROLLOUT_WARP
constexpr bool kRolloutWarpOnly = true;
#else
constexpr bool kRolloutWarpOnly = false;
#endif

cudaError_t launch_noise_pregen(const StepConst& sc, double* eps, cudaStream_t s) {
  const int n = sc.k_local * sc.T;
  if (n <= 0 || sc.nstate == nullptr) return cudaSuccess;
  { if (const cudaError_t le = launch_k(k_noise_pregen, (n + 255) / 256, 256, 0, s, sc, eps); le != cudaSuccess) return le; }
  return cudaGetLastError();
}

template <int TAG>
cudaError_t rollout_tag(const StepConst& sc, const StepDyn* dyn, const double* nominal,
                        double* eps, int draw, float4* poses, double* task, const double* guide,
                        int guide_cap, double* base_cost, double* ctrl_cost,
                        double* controls_out, double* states_out, cudaStream_t s) {
  if (!kRolloutWarpOnly) {
    constexpr int D = model_dim<TAG>();
    const size_t s16 = rollout_lanes_smem(sc.T, D, 16, guide_cap);
    // 8 rollouts per CTA: ~28 resident warps per SM hide the eps loads (cold L2) as well as
    // the warp-per-rollout kernel does, with a quarter of its instructions (16 / 32 measured
    // slower)
    const size_t s8 = rollout_lanes_smem(sc.T, D, 8, guide_cap);
    if (s8 <= 200 * 1024)
      return rollout_lanes_launch<TAG, 8>(sc, dyn, nominal, eps, draw, poses, task, guide,
                                          guide_cap, base_cost, ctrl_cost, controls_out,
                                          states_out, s8, s);
    if (s16 <= 200 * 1024)
      return rollout_lanes_launch<TAG, 16>(sc, dyn, nominal, eps, draw, poses, task, guide,
                                           guide_cap, base_cost, ctrl_cost, controls_out,
                                           states_out, s16, s);
  }
  const int threads = kRolloutWarps * 32;
  const size_t smem = sizeof(double) * (2 * static_cast<size_t>(guide_cap) +
                                        static_cast<size_t>(sc.T) * sc.D +
                                        kRolloutWarps * static_cast<size_t>(rollout_warp_scratch(sc.T, sc.D)));
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_rollout<TAG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  if (const cudaError_t le = launch_k(k_rollout<TAG>, (sc.k_local + kRolloutWarps - 1) / kRolloutWarps,
                                      threads, smem, s, sc, dyn, nominal, eps, draw, poses, task,
                                      guide, guide_cap, base_cost, ctrl_cost, controls_out,
                                      states_out);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

cudaError_t launch_rollout(const StepConst& sc, const StepDyn* dyn, const double* nominal,
                           double* eps, int draw, float4* poses, double* task,
                           const double* guide, int guide_cap, double* base_cost,
                           double* ctrl_cost, double* controls_out, double* states_out,
                           cudaStream_t s) {
  switch (sc.tag) {
    case EXM_MODEL_DIFF: return rollout_tag<EXM_MODEL_DIFF>(sc, dyn, nominal, eps, draw, poses, task, guide, guide_cap, base_cost, ctrl_cost, controls_out, states_out, s);
    case EXM_MODEL_ACKERMANN: return rollout_tag<EXM_MODEL_ACKERMANN>(sc, dyn, nominal, eps, draw, poses, task, guide, guide_cap, base_cost, ctrl_cost, controls_out, states_out, s);
    case EXM_MODEL_OMNI: return rollout_tag<EXM_MODEL_OMNI>(sc, dyn, nominal, eps, draw, poses, task, guide, guide_cap, base_cost, ctrl_cost, controls_out, states_out, s);
    case EXM_MODEL_SPIN: return rollout_tag<EXM_MODEL_SPIN>(sc, dyn, nominal, eps, draw, poses, task, guide, guide_cap, base_cost, ctrl_cost, controls_out, states_out, s);
    case EXM_MODEL_PARALLEL: return rollout_tag<EXM_MODEL_PARALLEL>(sc, dyn, nominal, eps, draw, poses, task, guide, guide_cap, base_cost, ctrl_cost, controls_out, states_out, s);
  }
  return cudaErrorInvalidValue;
}

template <int W, bool kF64 = false>
cudaError_t rollout_costs_launch(const StepConst& sc, const double* task, const double* base_cost,
                                 const double* ctrl_cost, const float* dmin, double* cost,
                                 uint8_t* unsafe, float* dstat, float* hstat, size_t smem,
                                 cudaStream_t s, const double* dmin64 = nullptr) {
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_rollout_costs<W, kF64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  if (const cudaError_t le = launch_k(k_rollout_costs<W, kF64>, (sc.k_local + W - 1) / W, W * 32, smem, s,
                                      sc, task, base_cost, ctrl_cost, dmin, cost, unsafe, dstat,
                                      hstat, dmin64);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

cudaError_t launch_rollout_costs(const StepConst& sc, const double* task, const double* base_cost,
                                 const double* ctrl_cost, const float* dmin, double* cost,
                                 uint8_t* unsafe, float* dstat, float* hstat, cudaStream_t s) {
  if (sc.k_local <= 0) return cudaSuccess;
  // 16 rollouts per CTA (8 and 4 measured slower on configs 2 and 3); long horizons (per-warp
  // stage arrays beyond ~200 KB) use fewer
  auto smem_for = [&](int w) {
    return sizeof(double) * (3 * static_cast<size_t>(w) * sc.T + sc.T);
  };
  if (smem_for(16) <= 200 * 1024)
    return rollout_costs_launch<16>(sc, task, base_cost, ctrl_cost, dmin, cost, unsafe, dstat, hstat,
                                    smem_for(16), s);
  if (smem_for(4) <= 200 * 1024)
    return rollout_costs_launch<4>(sc, task, base_cost, ctrl_cost, dmin, cost, unsafe, dstat, hstat,
                                   smem_for(4), s);
  return rollout_costs_launch<1>(sc, task, base_cost, ctrl_cost, dmin, cost, unsafe, dstat, hstat,
                                 smem_for(1), s);
}

cudaError_t launch_rollout_costs_dmin64(const StepConst& sc, const double* task,
                                        const double* base_cost, const double* ctrl_cost,
                                        const double* dmin64, double* cost, uint8_t* unsafe,
                                        float* dstat, cudaStream_t s) {
  if (sc.k_local <= 0) return cudaSuccess;
  auto smem_for = [&](int w) {
    return sizeof(double) * (3 * static_cast<size_t>(w) * sc.T + sc.T);
  };
  if (smem_for(16) <= 200 * 1024)
    return rollout_costs_launch<16, true>(sc, task, base_cost, ctrl_cost, nullptr, cost, unsafe, dstat,
                                    nullptr, smem_for(16), s, dmin64);
  if (smem_for(4) <= 200 * 1024)
    return rollout_costs_launch<4, true>(sc, task, base_cost, ctrl_cost, nullptr, cost, unsafe, dstat,
                                   nullptr, smem_for(4), s, dmin64);
  return rollout_costs_launch<1, true>(sc, task, base_cost, ctrl_cost, nullptr, cost, unsafe, dstat,
                                 nullptr, smem_for(1), s, dmin64);
}

cudaError_t launch_block_partials(const StepConst& sc, const double* cost, const uint8_t* unsafe,
                                  const double* eps, double* partials, cudaStream_t s) {
  if (sc.nblocks_local <= 0) return cudaSuccess;
  const dim3 grid(sc.nblocks_local, (sc.T * sc.D + kPartCols - 1) / kPartCols);
  { if (const cudaError_t le = launch_k(k_block_partials, grid, kBlockRollouts, 0, s, sc, cost, unsafe, eps, partials); le != cudaSuccess) return le; }
  return cudaGetLastError();
}

template <int TAG>
cudaError_t update_tag(const StepConst& sc, const double* partials, const double* nominal,
                       const StepDyn* dyn, double* upd, float4* val_poses, double2* val_xy,
                       double* val_base, DecisionDev* dec, int merge, cudaStream_t s) {
  const size_t smem = sizeof(double) * (static_cast<size_t>(sc.T) * sc.D +
                                        static_cast<size_t>(merge ? 5 * sc.nblocks_total : 0) +
                                        rollout_warp_scratch(sc.T, sc.D));
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_update<TAG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  { if (const cudaError_t le = launch_k(k_update<TAG>, 1, 256, smem, s, sc, partials, nominal, dyn, upd, val_poses, val_xy, val_base,
                                     dec, merge); le != cudaSuccess) return le; }
  return cudaGetLastError();
}

cudaError_t launch_update(const StepConst& sc, const double* partials, const double* nominal,
                          const StepDyn* dyn, double* upd, float4* val_poses, double2* val_xy,
                          double* val_base, DecisionDev* dec, int merge, cudaStream_t s) {
  switch (sc.tag) {
    case EXM_MODEL_DIFF: return update_tag<EXM_MODEL_DIFF>(sc, partials, nominal, dyn, upd, val_poses, val_xy, val_base, dec, merge, s);
    case EXM_MODEL_ACKERMANN: return update_tag<EXM_MODEL_ACKERMANN>(sc, partials, nominal, dyn, upd, val_poses, val_xy, val_base, dec, merge, s);
    case EXM_MODEL_OMNI: return update_tag<EXM_MODEL_OMNI>(sc, partials, nominal, dyn, upd, val_poses, val_xy, val_base, dec, merge, s);
    case EXM_MODEL_SPIN: return update_tag<EXM_MODEL_SPIN>(sc, partials, nominal, dyn, upd, val_poses, val_xy, val_base, dec, merge, s);
    case EXM_MODEL_PARALLEL: return update_tag<EXM_MODEL_PARALLEL>(sc, partials, nominal, dyn, upd, val_poses, val_xy, val_base, dec, merge, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_finalize(const StepConst& sc, const float* val_dmin, const double2* val_xy,
                            const double* val_base, const double* upd, const double* guide,
                            int guide_cap, double* nominal, StepDyn* dyn, DecisionDev* dec,
                            double* out_dmin, double* out_nominal, double* out_uprev, int commit,
                            float* hstat, float* cap, float radius, cudaStream_t s) {
  const size_t smem = sizeof(double) * (2 * static_cast<size_t>(guide_cap) + 3 * sc.T);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  { if (const cudaError_t le = launch_k(k_finalize, 1, 64, smem, s, sc, val_dmin, val_xy, val_base, upd, guide, nominal, dyn, dec,
                                 out_dmin, out_nominal, out_uprev, commit, hstat, cap, radius); le != cudaSuccess) return le; }
  return cudaGetLastError();
}

}  // namespace exm
