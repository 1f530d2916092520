// exm_common.cuh — structs shared by the host side (exm_abi.cu) and the kernels
// (exm_kernels.cu) of libexm_b200.so. Nothing here crosses the public C ABI.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <utility>

#include <cuda_runtime.h>

namespace exm {

constexpr int kMaxEdges = 64;        // polygon edges / cover boxes held in kernel parameters
constexpr int kMaxCover = 3;         // boxes of the polygon cull cover
constexpr int kBlockRollouts = 256;  // rollouts per softmax partial (fixed: G-invariant)
constexpr int kGridMax = 181;        // cloud grid cells per axis (<= 32761 cells, 131 KB smem histogram)
constexpr float kEmptyDistance = 1e6f;  // kEmptyMaskDistance (geometry.hpp:37)
constexpr float kCullMargin = 1e-4f;    // base slack on every lower-bound cull (m)
// cloud points per chunk (one bounding box each): 8 or 16, chosen per handle (GridMeta::chunk)
constexpr int kChunkMax = 16;
constexpr int kSubCells = 16;           // per-axis sub-cells of the in-cell Morton order

// FP32 footprint table, passed by value as a __grid_constant__ kernel parameter so the
// inner loops read it from the constant bank (uniform datapath), never from memory.
// Polygon edge b (prepare, geometry.cpp:236-247), recentring-free body frame:
//   e[b] = {vx, vy, ex, ey, ex/|e|^2, ey/|e|^2, -(v.e)/|e|^2, -ex}
// Box j (geometry.cpp:250-255): e[j] = {cx, cy, hx, hy, 0...}
struct FpDev {
  int kind;  // EXM_FOOTPRINT_*
  int count;
  float radius;  // PreparedFootprint::bounding_radius (max vertex norm, geometry.cpp:127-131)
  float reserved;
  float aabb[4];  // body-frame bounding box {xmin, xmax, ymin, ymax}
  // <= kMaxCover axis-aligned boxes {cx, cy, hx, hy} whose union contains the footprint
  // (polygons: exact for rectilinear shapes such as the L; rectangle covers of <= kMaxCover
  // boxes: the boxes themselves; otherwise the AABB): an exterior point's signed distance is
  // at least its distance to that union, a tighter cull bound than the AABB.
  int ncover;
  // polygons whose cover boxes tile them exactly (rectilinear: the L): outside the slackened
  // cover (every max(|b - c| - h) > cover_slack) the signed distance IS the distance to the
  // unslackened boxes cbox, so the exact value costs one box pass instead of the edge loop
  int cover_exact;
  float cover[kMaxCover][4];  // {cx, cy, hx + slack, hy + slack}
  float cbox[kMaxCover][4];   // {cx, cy, hx, hy} (cover_exact only)
  float cover_slack;
  float reserved3;
  float e[kMaxEdges][8];
  // polygon edges in pairs for the f32x2 path: ep[j][k] = {e[2j][k], e[2j+1][k]}; an odd
  // count is padded with the zero-length edge {v0x, v0y, 0...}
  alignas(8) float ep[kMaxEdges / 2][8][2];
};

// Uniform grid over the recentred valid cloud (written by the prep kernel).
struct GridMeta {
  float x0, y0, cs, inv_cs;
  int gx, gy, n_valid;
  float margin;  // cull slack (m): kCullMargin + rounding allowance for the cloud's extent
  int chunk;     // points per chunk (8 or 16)
  int reserved;
};

// Device cloud structure of one control step (HBM, rebuilt every cycle by launch_cloud_prep):
//   cloud[cell_start[c] .. cell_start[c+1])  cell c's points, Morton-ordered on a kSubCells^2
//       sub-grid, padded with NaN to a multiple of the chunk size C = GridMeta::chunk (NaN never
//       passes a distance test)
//   chunk[i]  bounding box {cx, cy, hx, hy} of cloud[C*i .. C*i + C)
// tmp / raw / raw_start are the prep kernels' scratch (compacted points, cell-sorted points).
struct CloudGrid {
  float2* tmp = nullptr;
  float2* raw = nullptr;
  int* raw_start = nullptr;
  float2* cloud = nullptr;
  float4* chunk = nullptr;
  int* cell_start = nullptr;
  GridMeta* gm = nullptr;
  // {sum of clamped per-pose minima, count} accumulated by the stage-cost kernel and consumed
  // (then reset) by the next step's prep kernel: sizes the cells for the searches to come
  float* dstat = nullptr;
  // {next pose, finished warps} of the persistent k_sdf_grid (zero between launches)
  unsigned* work = nullptr;
};
// Padded cloud capacity for n_cap points: every nonempty cell adds at most kChunkMax - 1 pads.
inline size_t cloud_capacity(int n_cap) {
  return static_cast<size_t>(n_cap) + static_cast<size_t>(kChunkMax - 1) * kGridMax * kGridMax + kChunkMax;
}

// Sensing (exm_world.cu): boundary-sample segments in the reference's sampling order and the
// obstacles for the line-of-sight test (world.cpp:39-65, :167-179), as base geometry: every
// obstacle's current trail offset comes from a device array (offsets[obs]), so the sample counts
// of displaced polygon edges (which depend on the offset through rounding) are formed on the
// device, as is the whole world state of the device world (exm_world_*).
struct SenseSeg {
  int kind;   // 0 polygon edge a -> b (base vertices), 1 disc (base centre a, radius r)
  int obs;    // obstacle index (offset)
  double ax, ay, bx, by, r;
};
struct SenseObs {
  int kind;  // 0 polygon (verts[first .. first + count)), 1 disc
  int count;
  int first;
  int reserved;
  double cx, cy, r;  // disc centre (base), radius
};
// Trail motion of one obstacle (world.hpp TrailMotion) and its state (WorldState).
struct TrailDev {
  int first, n;     // waypoints[first .. first + n) (n < 2: static)
  int ping_pong;
  int reserved;
  double speed;
};

// Per-step small inputs, uploaded with one copy (host API) or kept resident.
struct StepDyn {
  double q0[3];
  double goal[3];
  double u_prev[3];
  uint64_t cycle;
  int32_t n_points;
  int32_t n_guide;
  int32_t use_mask;
  int32_t reserved;
};

// Model, limits and MPPI parameters (kernel parameter).
struct StepConst {
  int K, T, D, tag;
  int k_local, r_offset;        // this rank's rollout shard [r_offset, r_offset + k_local)
  int nblocks_local, block_offset, nblocks_total;
  int reserved;
  double dt, lambda, d_safe, w_coll, w_rep, w_inf;
  double w_goal_pos, w_goal_head, w_xtrack, w_progress, w_ctrl, wheelbase;
  double sigma[3];
  double vel_min[3], vel_max[3], acc_min[3], acc_max[3];
  double steer_max;
  uint64_t seed;
  // device noise state {cycle of the last drawing rollout, cycle whose noise eps holds
  // (pregenerated by k_noise_pregen; ~0 = none)}; nullptr: always draw in the rollout
  uint64_t* nstate;
};

struct DecisionDev {
  double command[3];
  int32_t validated;
  int32_t argmin;
  double best_cost;
  double entropy;
  double nominal_cost;
  double reserved;
};

// Softmax partial of one block of kBlockRollouts rollouts:
//   {beta_b, S_b = sum e, A_b = sum e (J - beta_b)/lambda, argmin_b, U_b[T*D] = sum e eps}
inline __host__ __device__ int partial_stride(int T, int D) { return 4 + T * D; }

// Culling statistics of k_sdf_grid (statistics builds of the launch only, exm_sdf_cull_stats):
// per-lane counts of each kind of work, charged at its FP32 op count by the benchmark's
// executed-work roofline, plus warp-level iteration counts (lane efficiency).
enum {
  kCntRing = 0,       // ring steps (per warp)
  kCntCell = 1,       // nonempty-cell bound tests (per lane still searching)
  kCntChunk = 2,      // chunk box bound tests (per lane needing the cell)
  kCntPoint = 3,      // point circle tests (per lane needing the chunk)
  kCntPointWarp = 4,  // point-loop iterations (per warp)
  kCntTransform = 5,  // body-frame transforms (points inside the circle bound)
  kCntTile = 6,       // exact-cover tile tests
  kCntTileVal = 7,    // tile distances taken (exact value of an exterior point)
  kCntBound = 8,      // cover / AABB bound tests
  kCntEdges = 9,      // edge-loop (polygon) / box-loop (cover) signed distances
  kCntN = 10
};

// Signed-distance kernel selection. Production handles use kSdfAuto; the others exist for the
// exactness tests and A/B measurements (exm_set_sdf_mode): every bound disabled (brute), no
// chunk bound, a forced thread / warp / 8-warp-CTA per pose kernel, persistent warps at any
// size, caps ignored.
enum {
  kSdfAuto = 0, kSdfBrute = 1, kSdfNoChunk = 2, kSdfThread = 3, kSdfWarp = 4, kSdfCta = 5,
  kSdfPersist = 6, kSdfNoCap = 7
};
// What the last signed-distance launch of a step ran (exm_last_sdf_path).
struct SdfPath {
  int kernel;      // 0 thread per pose (k_sdf_grid), 1 warp per pose, 2 8-warp CTA per pose
  int chunk;       // points per cull chunk of the cloud layout (8 or 16)
  int persistent;  // 1: persistent warps with the work counter
  int ctas, threads;
  int hmajor;      // 1: lanes take consecutive rollouts at one step
};

// Kernel launch with programmatic dependent launch (PDL) allowed: the next kernel in the stream
// (or graph) may be scheduled while this one drains, and waits in pdl_wait() (griddepcontrol
// .wait, the first statement of every kernel) for the predecessor's completion and memory
// flush, so launch latency overlaps the previous kernel's tail. EXM_PDL=0 disables it.
#ifndef EXM_NO_PDL
constexpr bool kPdl = true;
#else
constexpr bool kPdl = false;  // A/B builds (-DEXM_NO_PDL)
#endif
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = kPdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---- kernel launchers (exm_kernels.cu) ---------------------------------------------------
cudaError_t launch_noise(const StepConst& sc, const StepDyn* dyn, double* eps, cudaStream_t s);
// The next cycle's device noise (cycle sc.nstate[0] + 1) into eps, marked in sc.nstate[1]
cudaError_t launch_noise_pregen(const StepConst& sc, double* eps, cudaStream_t s);
// chunk: points per cull chunk (8 for small clouds; 16 for clouds of >= 16k points, whose long
// walls make a chunk test per 8 points the larger cost)
cudaError_t launch_cloud_prep(const double* pts, const uint8_t* mask, const StepDyn* dyn,
                              float radius, const CloudGrid& g, int n_cap, cudaStream_t s);
int chunk_for_capacity(int n_cap);
// draw != 0: the rollout kernel draws the device noise into eps; else eps is read (injected).
// task: the task cost of every pre-step state (r, h) (guidance: guide_cap doubles x 2, n_guide
// and goal in dyn); base_cost: terminal goal cost per rollout; ctrl_cost: control cost per (r, h).
cudaError_t launch_rollout(const StepConst& sc, const StepDyn* dyn, const double* nominal,
                           double* eps, int draw, float4* poses, double* task,
                           const double* guide, int guide_cap, double* base_cost,
                           double* ctrl_cost, double* controls_out, double* states_out,
                           cudaStream_t s);
cudaError_t launch_sdf_grid(const FpDev& fp, const float4* poses, int n_poses, int T, bool hmajor,
                            const CloudGrid& g, const float* cap, int mode, float* out,
                            SdfPath* path, unsigned long long* stats, cudaStream_t s,
                            float thr = HUGE_VALF);  // results: min(exact minimum, thr)
cudaError_t launch_rollout_costs(const StepConst& sc, const double* task, const double* base_cost,
                                 const double* ctrl_cost, const float* dmin, double* cost,
                                 uint8_t* unsafe, float* dstat, float* hstat, cudaStream_t s);
cudaError_t launch_block_partials(const StepConst& sc, const double* cost, const uint8_t* unsafe,
                                  const double* eps, double* partials, cudaStream_t s);
// val_base: T + 1 doubles {terminal cost, control cost of every step} of the validation rollout
cudaError_t launch_update(const StepConst& sc, const double* partials, const double* nominal,
                          const StepDyn* dyn, double* upd, float4* val_poses, double2* val_xy,
                          double* val_base, DecisionDev* dec, int merge, cudaStream_t s);
// hstat ({sum d, sum d^2} per step + count, from k_rollout_costs) -> cap: the next step's
// per-step SDF caps (both optional; commit steps only).
cudaError_t launch_finalize(const StepConst& sc, const float* val_dmin, const double2* val_xy,
                            const double* val_base, const double* upd, const double* guide,
                            int guide_cap, double* nominal, StepDyn* dyn, DecisionDev* dec,
                            double* out_dmin, double* out_nominal, double* out_uprev, int commit,
                            float* hstat, float* cap, float radius, cudaStream_t s);
// Staged pose batches (exm_sdf_stage): center[2] = the poses' centroid (one CTA, fixed order),
// out = {x - cx, y - cy, cos theta, sin theta}; points recentred at the same device centre.
cudaError_t launch_pose_prep(const double* poses, int n, double* center, float4* out,
                             cudaStream_t s);
cudaError_t launch_recentre(const double* pts, int n, const double* center, float2* out,
                            cudaStream_t s);
// Body-frame queries -> signed distance (batch_signed_distance), FP32 in and out.
cudaError_t launch_sdf_points(const FpDev& fp, const float2* q, int n, float* out, cudaStream_t s);
cudaError_t launch_sdf_pairs(const FpDev& fp, const float4* poses, int n_poses,
                             const float2* pts, const uint8_t* mask, int n_points,
                             float* per_pair, unsigned* pose_min_key, cudaStream_t s);
// sense (world.cpp:182-243) over base geometry displaced by offsets[n_obs]; scratch: 2 ints per
// segment, a double and an int per sample (sample_cap samples; more fall back to recomputation),
// bin_state (sense_bin_state_bytes()).
cudaError_t launch_sense(const SenseSeg* seg, int nseg, const SenseObs* obs, int n_obs,
                         const double2* verts, const double2* offsets, double rx, double ry,
                         double range, int budget, uint64_t seed, uint64_t sample_key,
                         int* seg_scratch, double* d_scratch, int* bin_scratch, int sample_cap,
                         void* bin_state, double* pts_out, uint8_t* mask_out, int* n_out,
                         cudaStream_t s);
size_t sense_bin_state_bytes();
// step_world (world.cpp:127-157) + obstacle_offset (:159-164) for n_obs obstacles on the device:
// arc / direction advanced by dt (dt > 0) when `advance`, then offsets[i] = trail point - first
// waypoint.
cudaError_t launch_world_step(const TrailDev* trails, const double2* waypoints, int n_obs,
                              double dt, int advance, double* arc, int* dir, double2* offsets,
                              cudaStream_t s);
cudaError_t launch_min_keys_to_double(const unsigned* keys, int n, double* out, cudaStream_t s);
cudaError_t launch_fill_u32(unsigned* p, unsigned v, int n, cudaStream_t s);

}  // namespace exm
