/*
 * exm_b200.h — C ABI of the B200-native EXACT-MPPI rollout + exact-SDF hot path.
 *
 * Everything here is plain C: POD structs, host pointers and sizes, status codes.
 * No CUDA, torch or C++ types cross this boundary. The library (libexm_b200.so)
 * owns every device buffer, stream, CUDA graph and NCCL communicator behind an
 * opaque handle; the caller owns every host buffer it passes in.
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to the reference tree, proj/...). The reference is a C++20 CPU
 * library with no FFI; the drop-in is a replacement translation unit for
 * proj/src/controller.cpp that implements proj/include/exactmppi/controller.hpp on
 * top of these calls.
 *
 * Array layouts (all row-major, host memory):
 *   points        pts_xy[2*i + {0,1}]                   world frame, N entries
 *   mask          mask[i] != 0 marks a valid point     (ObstacleSet::mask, geometry.hpp:88-97)
 *   guidance      guide_xy[2*j + {0,1}]                 polyline, P >= 1 points
 *   controls      u[h*dim + c]                          NominalSequence, T x dim
 *   perturbations eps[(r*T + h)*dim + c]                 K x T x dim (RolloutBatch::at, controller.hpp:60-63)
 *   states        states[(r*(T+1) + h)*3 + {x,y,theta}]
 *   d_min         d_min[r*T + h]
 * dim is MotionModel::control_dim() (kinematics.cpp:14-26): diff/ackermann 2, omni 3,
 * spin/parallel 1.
 *
 * Threading: the reference's MppiController is "sendable between threads, not concurrently
 * shared" (controller.hpp:138-139). Here every call on a handle holds that handle's lock, so
 * concurrent calls on one handle are safe and serialise; distinct handles run concurrently.
 */
#ifndef EXM_B200_H
#define EXM_B200_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EXM_ABI_VERSION 2

typedef int32_t exm_status;
enum {
  EXM_OK = 0,
  EXM_ERR_INVALID_ARGUMENT = 1, /* reference: std::invalid_argument */
  EXM_ERR_CUDA = 2,
  EXM_ERR_NCCL = 3,
  EXM_ERR_UNSUPPORTED = 4,
  EXM_ERR_INTERNAL = 5
};

/* FootprintSpec::shape alternatives (geometry.hpp:41-85). */
enum { EXM_FOOTPRINT_RECT_COVER = 0, EXM_FOOTPRINT_POLYGON = 1 };

/* Polygon: count vertices (x[i], y[i]); CCW expected, CW is reversed with a warning
 * exactly like PolygonFootprint::make (geometry.cpp:79-110).
 * Rectangle cover: count boxes, centre (x[i], y[i]), half extents (hx[i], hy[i])
 * (RectangleCover::make, geometry.cpp:66-77). */
typedef struct exm_footprint {
  int32_t kind;
  int32_t count;
  const double* x;
  const double* y;
  const double* hx; /* rect cover only */
  const double* hy; /* rect cover only */
} exm_footprint;

/* ModelTag (kinematics.hpp:13). */
enum {
  EXM_MODEL_DIFF = 0,
  EXM_MODEL_ACKERMANN = 1,
  EXM_MODEL_OMNI = 2,
  EXM_MODEL_SPIN = 3,
  EXM_MODEL_PARALLEL = 4
};

/* MotionModel (kinematics.hpp:16-28). */
typedef struct exm_model {
  int32_t tag;
  int32_t reserved;
  double wheelbase;
} exm_model;

/* KinematicLimits / ComponentLimit (kinematics.hpp:51-63). */
typedef struct exm_limits {
  double vel_min[3];
  double vel_max[3];
  double acc_min[3];
  double acc_max[3];
  double steer_max;
} exm_limits;

/* MppiParams + TaskWeights (controller.hpp:13-35). */
typedef struct exm_params {
  int32_t rollouts; /* K */
  int32_t horizon;  /* T */
  double dt;
  double lambda;
  double sigma[3];
  double d_safe;
  double w_coll;
  double w_rep;
  double w_inf;
  double w_goal_pos;
  double w_goal_head;
  double w_xtrack;
  double w_progress;
  double w_ctrl;
  uint64_t seed;
} exm_params;

/* ControlDecision + CycleDiagnostics (controller.hpp:66-77), plus the argmin rollout
 * (index of beta) which the reference computes implicitly (controller.cpp:315). */
typedef struct exm_decision {
  double command[3];
  int32_t validated;
  int32_t argmin;
  double best_cost;      /* beta over augmented costs */
  double weight_entropy; /* -sum w log w */
  double nominal_cost;   /* cost of the validated sequence */
  double* nominal_dmin;  /* caller buffer of T doubles, or NULL */
} exm_decision;

typedef struct exm_handle exm_handle;

/* ---- library ----------------------------------------------------------------- */
int32_t exm_abi_version(void);
/* Thread-local message of the last failing call (reference exception text). */
const char* exm_last_error(void);

/* ---- lifetime ----------------------------------------------------------------
 * Replaces MppiController::MppiController (controller.hpp:141-142, controller.cpp:284-294):
 * validates the footprint (geometry.cpp:66-110), the model (kinematics.cpp:9-12) and the
 * params (MppiParams::validate, controller.cpp:13-23), prepares the footprint
 * (prepare, geometry.cpp:230-258) and sizes device buffers for (K, T, n_cap, guide_cap).
 * device < 0 selects the current CUDA device. */
exm_status exm_create(const exm_footprint* footprint, const exm_model* model,
                      const exm_limits* limits, const exm_params* params, int32_t n_cap,
                      int32_t guide_cap, int32_t device, exm_handle** out);
void exm_destroy(exm_handle* h);

/* ---- the MPPI step -------------------------------------------------------------
 * Replaces MppiController::control_cycle (controller.hpp:146-147, controller.cpp:304-365).
 * The controller state the reference keeps in the object (nominal_, u_prev_, cycle_;
 * controller.hpp:167-169) is passed in and out explicitly: nominal_inout (T x dim) and
 * u_prev_inout (dim) are read, then overwritten with the shifted/held nominal and the
 * command. cycle is the RNG key of sample_perturbations (controller.cpp:306).
 * eps_or_null: NULL draws perturbations on the device from (params.seed, cycle) exactly as
 * sample_perturbations keys them; non-NULL injects a K x T x dim array (parity mode).
 * Sharded handles (exm_attach_comm) process rollouts [rank*K/G, (rank+1)*K/G) and exchange
 * softmax partials with one NCCL all-gather; every rank returns the same decision. */
exm_status exm_control_cycle(exm_handle* h, const double q0[3], const double* pts_xy,
                             const uint8_t* mask, int32_t n_points, const double* guide_xy,
                             int32_t n_guide, const double goal[3], double* nominal_inout,
                             double* u_prev_inout, uint64_t cycle, const double* eps_or_null,
                             exm_decision* out);

/* Replaces evaluate_rollouts (controller.hpp:116-121, controller.cpp:178-220): rollouts,
 * clamped controls, states, per-step min signed distance, costs and unsafe flags for the
 * given perturbations (K x T x dim, required). Any output pointer may be NULL. */
exm_status exm_evaluate_rollouts(exm_handle* h, const double q0[3], const double* nominal,
                                 const double* eps, const double* pts_xy, const uint8_t* mask,
                                 int32_t n_points, const double* guide_xy, int32_t n_guide,
                                 const double goal[3], const double* u_prev,
                                 double* controls_out, double* states_out, double* dmin_out,
                                 double* costs_out, uint8_t* unsafe_out);

/* Replaces sample_perturbations (controller.hpp:107-108, controller.cpp:78-96), computed on
 * the device: eps_out[K*T*dim] = sigma_c * gaussian_at(seed, cycle, r, h, c). */
exm_status exm_sample_perturbations(exm_handle* h, uint64_t seed, uint64_t cycle,
                                    double* eps_out);

/* Replaces validate_nominal (controller.hpp:125-129, controller.cpp:254-282). */
exm_status exm_validate_nominal(exm_handle* h, const double* nominal, const double q0[3],
                                const double* pts_xy, const uint8_t* mask, int32_t n_points,
                                const double* guide_xy, int32_t n_guide, const double goal[3],
                                const double* u_prev, int32_t* valid_out, double* dmin_out,
                                double* cost_out);

/* ---- signed distance ------------------------------------------------------------
 * Replaces min_signed_distance_at (geometry.hpp:150-152, geometry.cpp:357-375) for a batch
 * of world poses (P x {x,y,theta}) against one cloud, and optionally emits every per-pair
 * signed distance (per_pair[p*N + i], body-frame sd of point i at pose p; masked points
 * report +inf). per_pose_min has the reference semantics: min over valid points, or
 * kEmptyMaskDistance (1e6) when the mask is empty. Either output may be NULL. */
exm_status exm_sdf_batch(exm_handle* h, const double* poses, int32_t n_poses,
                         const double* pts_xy, const uint8_t* mask, int32_t n_points,
                         float* per_pair, double* per_pose_min);

/* exm_sdf_batch in three phases for serving loops and benchmarks: stage the poses and the
 * cloud once (host -> device, recentred at the poses' centroid in FP64), run the kernel
 * n_steps times on the resident inputs (want_pairs: also write every per-pair value on the
 * device), read the last results back. */
exm_status exm_sdf_stage(exm_handle* h, const double* poses, int32_t n_poses,
                         const double* pts_xy, const uint8_t* mask, int32_t n_points);
exm_status exm_sdf_run_resident(exm_handle* h, int32_t n_steps, int32_t want_pairs);
exm_status exm_sdf_read(exm_handle* h, float* per_pair, double* per_pose_min);

/* Replaces batch_signed_distance (geometry.hpp:142-143, geometry.cpp:298-318): body-frame
 * queries, one signed distance each. */
exm_status exm_batch_signed_distance(exm_handle* h, const double* queries, int32_t n,
                                     double* out);

/* ---- hybrid mode families ---------------------------------------------
 * Replaces the per-mode loop of HybridController::hybrid_cycle (hybrid.cpp:103-111): n_modes
 * MPPI families that share the footprint, the cloud and the guidance, each with its own
 * model and limits (modes[m], limits[m]) and the seed params.seed ^ (0x9E3779B97F4A7C15*(m+1))
 * (hybrid.cpp:89). One call runs every family's MPPI step in one CUDA graph: one cloud
 * preparation, one SDF launch over all n_modes*K*T poses, per-family noise/rollout and
 * softmax/update/validation chains on parallel graph branches. Mode selection (switch
 * penalty, cooldown, projection, deadzone; hybrid.cpp:113-155) stays with the caller.
 * nominals_inout: n_modes blocks of T*3 doubles (family m uses its first T*dim_m);
 * u_prev_inout: n_modes*3; out: n_modes decisions. */
typedef struct exm_hybrid exm_hybrid;
exm_status exm_hybrid_create(const exm_footprint* footprint, const exm_model* models,
                             const exm_limits* limits, int32_t n_modes,
                             const exm_params* params, int32_t n_cap, int32_t guide_cap,
                             int32_t device, exm_hybrid** out);
void exm_hybrid_destroy(exm_hybrid* hy);
/* exm_set_option on every family handle (the hybrid step graph is re-captured). */
exm_status exm_hybrid_set_option(exm_hybrid* hy, int32_t option, int32_t value);
exm_status exm_hybrid_cycle(exm_hybrid* hy, const double q0[3], const double* pts_xy,
                            const uint8_t* mask, int32_t n_points, const double* guide_xy,
                            int32_t n_guide, const double goal[3], double* nominals_inout,
                            double* u_prev_inout, uint64_t cycle, exm_decision* out);

/* ---- multi-GPU (one process per GPU) ----------------------------------------------
 * The reference's only parallelism is a std::thread fork-join over rollouts
 * (controller.cpp:207-218). Here rollouts are sharded over ranks in fixed 256-rollout blocks
 * (rank g of G owns rollouts [g*K/G, (g+1)*K/G); K must be a multiple of 256*G); rank 0 creates
 * the id, the caller broadcasts it (e.g. torch.distributed), every rank attaches. With a
 * communicator attached (any world >= 1, a 1-rank one included) every control step issues one
 * in-place ncclAllGather of the softmax block partials inside its CUDA graph; every rank merges
 * them in block order and returns the same decision, bit-identical for every G.
 * exm_attach_comm(h, 0, 1, NULL) detaches (unsharded, no collective). */
exm_status exm_nccl_unique_id(uint8_t id_out[128]);
exm_status exm_attach_comm(exm_handle* h, int32_t rank, int32_t world, const uint8_t id[128]);

/* Sharding without a communicator, for several shard handles on ONE device (tests, and
 * emulating G ranks on one GPU): exm_set_shard(h, g, G) makes h own rank g's rollouts;
 * exm_sharded_cycle then runs one control step on all G shard handles (shards[g] of rank g,
 * same configuration, same device), exchanging the block partials between them with one
 * device-to-device copy per block where the ranks' all-gather would run. Per-shard state:
 * nominals_inout[g*T*dim ...], u_prevs_inout[3*g ...], out[g]. exm_set_shard(h, 0, 1) undoes. */
exm_status exm_set_shard(exm_handle* h, int32_t rank, int32_t world);
exm_status exm_sharded_cycle(exm_handle* const* shards, int32_t n_shards, const double q0[3],
                             const double* pts_xy, const uint8_t* mask, int32_t n_points,
                             const double* guide_xy, int32_t n_guide, const double goal[3],
                             double* nominals_inout, double* u_prevs_inout, uint64_t cycle,
                             const double* eps_or_null, exm_decision* out);

/* ---- resident-input stepping (benchmark / serving loop) -----------------------------
 * Stage the inputs of a control step once (host -> device), then run n_steps control
 * cycles on the resident inputs (receding horizon: the nominal and rate anchor evolve,
 * the cycle key advances). Timing is left to the caller, who records events on the
 * handle's stream (exm_stream). */
exm_status exm_stage_inputs(exm_handle* h, const double q0[3], const double* pts_xy,
                            const uint8_t* mask, int32_t n_points, const double* guide_xy,
                            int32_t n_guide, const double goal[3], const double* nominal,
                            const double* u_prev, uint64_t cycle);
exm_status exm_run_resident(exm_handle* h, int32_t n_steps);
exm_status exm_read_resident(exm_handle* h, double* nominal_out, double* u_prev_out,
                             exm_decision* out);
/* cudaStream_t of the handle, as an opaque pointer. */
void* exm_stream(exm_handle* h);
/* Kernel accounting: kernels launched per step, the SDF kernel's mean device time per step
 * (ms; CUDA events recorded around every SDF launch on the handle's stream) over all
 * exm_run_resident / exm_sdf_run_resident steps since the previous exm_step_stats call (or of
 * the last exm_control_cycle), and the point-pose pairs one SDF launch covers (poses x
 * points). Synchronises the stream and resets the accumulation. */
exm_status exm_step_stats(exm_handle* h, int32_t* launches_per_step, float* sdf_ms,
                          int64_t* sdf_pairs);

/* Culling statistics of the last resident step's pose set: re-runs the SDF kernel once with
 * counters (profiling only; not on the step path): point-pose pairs that reached a point test,
 * and pairs that reached the exact signed-distance evaluation. */
exm_status exm_sdf_cull_stats(exm_handle* h, int64_t* points_tested, int64_t* sdf_evaluated);

/* ---- options and diagnostics ------------------------------------------------------------ */
enum {
  EXM_OPT_SDF_MODE = 1,    /* EXM_SDF_* below (tests / A/B only; default EXM_SDF_AUTO) */
  EXM_OPT_AUTO_CAPS = 2,   /* 1: derive per-step SDF caps from each step's own d_min statistic */
  EXM_OPT_PREGEN = 3,      /* 0: no next-cycle noise pregeneration (default 1) */
  EXM_OPT_HOST_TIMING = 4, /* 1: accumulate exm_control_cycle host phases (exm_host_timing) */
  EXM_OPT_HOST_THREADS = 5, /* host threads converting batch_signed_distance queries (default:
                               min(8, hardware threads)); the reference's `threads` argument */
  EXM_OPT_SDF_MAP = 6,      /* lanes <-> poses of the thread-per-pose SDF: 0 tuned on the
                               handle's first steps (default), 1 a rollout's consecutive steps per
                               warp, 2 consecutive rollouts at one step per warp */
  EXM_OPT_SDF_THRESHOLD = 7, /* 1 (default): the rollout minima of exm_control_cycle /
                               exm_hybrid_cycle / exm_sharded_cycle are resolved exactly only below
                               d_safe (the obstacle cost is identically 0 and the rollout is not
                               unsafe at or above it, controller.cpp:98-101, :162, and no rollout
                               minimum is returned), so decisions are unchanged; 0: every rollout
                               minimum exact. exm_evaluate_rollouts is always exact. */
  EXM_OPT_SDF_FP64 = 8      /* 1: exm_batch_signed_distance evaluates PreparedFootprint::sd in
                               FP64 (16 B in / 8 B out per query on the link), and
                               exm_evaluate_rollouts computes its minima in FP64 with the
                               reference's own arithmetic (min_signed_distance_at over
                               PreparedFootprint::sd, geometry.cpp:260-295, :357-375; brute force,
                               one thread per pose) and its costs from them: minima and costs then
                               agree with the reference to the ulps of cos/sin (its 1e-9
                               batch-vs-scalar check, acceptance_main.cpp:260-300). 0 (default):
                               the FP32 culled kernels (within 1e-5 m). The control cycle is not
                               affected. */
};
/* Signed-distance kernel selection: automatic, or (tests) every bound disabled, no chunk
 * bound, a forced thread / warp / 8-warp-CTA per pose kernel, persistent warps, caps ignored. */
enum {
  EXM_SDF_AUTO = 0, EXM_SDF_BRUTE = 1, EXM_SDF_NOCHUNK = 2, EXM_SDF_THREAD = 3,
  EXM_SDF_WARP = 4, EXM_SDF_CTA = 5, EXM_SDF_PERSIST = 6, EXM_SDF_NOCAP = 7
};
/* Set a handle option. Captured step graphs are rebuilt on the next step. */
exm_status exm_set_option(exm_handle* h, int32_t option, int32_t value);
/* EXM_OPT_HOST_TIMING: mean host microseconds per exm_control_cycle call in each phase
 * {stage + H2D enqueue, graph launch + D2H enqueue, wait, unpack} and the call count. */
exm_status exm_host_timing(exm_handle* h, double us_per_call[4], int64_t* calls);

/* Which signed-distance kernel the last rollout / validation launch ran. */
typedef struct exm_sdf_path {
  int32_t kernel;     /* 0 thread per pose, 1 warp per pose, 2 8-warp CTA per pose */
  int32_t chunk;      /* points per cull chunk of the cloud layout (8 or 16) */
  int32_t persistent; /* 1: persistent warps with a work counter */
  int32_t ctas, threads;
  int32_t hmajor;     /* 1: a warp's lanes take consecutive rollouts at one horizon step */
} exm_sdf_path;
exm_status exm_last_sdf_path(exm_handle* h, exm_sdf_path* rollout, exm_sdf_path* validation);

/* Work counters of the rollout signed distance over the last step's poses (re-runs the kernel
 * once with counters; profiling only): counts[EXM_SDF_NCOUNT] = {ring steps (per warp),
 * cell bound tests, chunk bound tests, point circle tests, point-loop iterations (per warp),
 * body-frame transforms, exact-cover tile tests, tile distances taken, cover/AABB bound tests,
 * edge-loop (polygon) or box-loop (cover) signed distances}; per lane unless noted. */
#define EXM_SDF_NCOUNT 10
exm_status exm_sdf_work_stats(exm_handle* h, int64_t* counts);

/* ---- sensing (world.cpp:182-243) ---------------------------------------- */
enum { EXM_OBSTACLE_POLYGON = 0, EXM_OBSTACLE_DISC = 1 };
/* One scenario obstacle (world.hpp Obstacle): a polygon as PolygonFootprint stores it (CCW
 * vertices) or a disc {centre x[0], y[0]; radius}, displaced by its current trail offset
 * (obstacle_offset, world.cpp:159-164). */
typedef struct exm_world_obstacle {
  int32_t kind;
  int32_t count; /* polygon vertices (disc: 1) */
  const double* x;
  const double* y;
  double radius;
  double offset[2];
} exm_world_obstacle;

/* sense(scenario, state, robot, sample_key) (world.cpp:182-243) on the device: boundary
 * samples every 0.05 m, nearest sample per 720 angular bins within `range`, exact line of
 * sight, seeded partial Fisher-Yates downsample to `budget` (scenario seed), padded to
 * `budget` (ObstacleSet::padded: (1e9, 1e9), mask 0). Outputs pts_out[2*budget],
 * mask_out[budget], *n_valid. Errors: budget < 1 ("sensor budget must be >= 1"). */
exm_status exm_sense(exm_handle* h, const exm_world_obstacle* obstacles, int32_t n_obstacles,
                     const double robot[3], double range, int32_t budget, uint64_t seed,
                     uint64_t sample_key, double* pts_out, uint8_t* mask_out, int32_t* n_valid);

/* ---- device world: moving obstacles (step_world, world.cpp:127-157) + sense ----------------
 * A scenario's obstacles (shapes as exm_world_obstacle, whose `offset` is ignored here) with
 * their trail motion (world.hpp TrailMotion: >= 2 waypoints, the shape's coordinates at the first
 * one, speed >= 0, ping-pong or clamped), the sensor (range, budget) and the scenario seed, kept on
 * the device with the world state (WorldState: arc position and direction per obstacle, initially
 * 0 / +1). exm_world_step advances it by dt exactly as step_world; exm_world_sense is sense()
 * (world.cpp:182-243) with the current obstacle_offset of every obstacle (:159-164), computed on
 * the device. exm_world_state reads the state back (arc[n], dir[n], offsets[2n]; any may be NULL).
 * Errors: budget < 1 ("sensor budget must be >= 1"), dt <= 0 ("step_world requires dt > 0"). */
typedef struct exm_world exm_world;
typedef struct exm_world_trail {
  int32_t n_waypoints;     /* < 2: static obstacle */
  int32_t ping_pong;       /* 1: reflect at the ends, 0: clamp */
  const double* waypoints; /* 2 * n_waypoints */
  double speed;            /* m/s */
} exm_world_trail;
exm_status exm_world_create(exm_handle* h, const exm_world_obstacle* obstacles,
                            const exm_world_trail* trails_or_null, int32_t n_obstacles,
                            double range, int32_t budget, uint64_t seed, exm_world** out);
void exm_world_destroy(exm_world* w);
exm_status exm_world_step(exm_world* w, double dt);
exm_status exm_world_sense(exm_world* w, const double robot[3], uint64_t sample_key,
                           double* pts_out, uint8_t* mask_out, int32_t* n_valid);
exm_status exm_world_state(exm_world* w, double* arc_out, int32_t* dir_out, double* offsets_out);

/* Per-step hints for the culled signed distance (T floats, +inf = none): the rollout SDF first
 * prunes every point whose lower bound reaches cap[h], then re-runs without cap the poses it
 * left unresolved, so results are exact for any caps; good caps (a little above the step's
 * minima) only save work; caps below the minima cost a second pass. Caps persist in the handle
 * until set again (EXM_AUTO_CAPS=1: every committed step derives them from its own per-step
 * d_min mean + 3 sigma). No reference counterpart (an optimisation of min_signed_distance_at,
 * geometry.cpp:357-375). */
exm_status exm_set_sdf_caps(exm_handle* h, const float* caps);

/* Page-locked host memory (cudaHostAlloc, portable): input buffers (the cloud, the mask)
 * allocated here are uploaded by DMA without the driver's staging copy (cudaMemcpyAsync from
 * pageable memory copies through a bounce buffer on the calling thread). NULL on failure. */
void* exm_host_alloc(size_t bytes);
void exm_host_free(void* p);

/* Diagnostics (host only, no GPU needed): validates a footprint exactly as exm_create does and
 * returns the body-frame cull geometry the SDF kernels bound with: the bounding box
 * {xmin, xmax, ymin, ymax} (aabb_out[4]) and n_out <= 3 axis-aligned boxes
 * {cx, cy, hx, hy} whose union contains the footprint (boxes_out[12]). No reference
 * counterpart: PreparedFootprint (geometry.hpp:127-136) keeps only bounding_radius. */
exm_status exm_footprint_cull_boxes(const exm_footprint* fp, float* aabb_out, float* boxes_out,
                                    int32_t* n_out);

#ifdef __cplusplus
}
#endif

#endif /* EXM_B200_H */
