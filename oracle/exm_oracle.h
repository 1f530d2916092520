/*
 * exm_oracle.h — TEST INFRASTRUCTURE ONLY. CPU restatement of the reference's hot path.
 *
 * This is the checker, never the product: only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product path
 * (libexm_b200.so) never links or calls it.
 *
 * Each function restates one reference function (file:line under proj/ of the reference
 * tree) in plain C with the same operation order, so that built with the same compiler and
 * flags as the reference (-O3, no FMA contraction on baseline x86-64) it reproduces the
 * reference bit for bit; tests/test_oracle_ref.py checks exactly that against the real
 * reference compiled into oracle/_ref, and tests/test_oracle_kat.py against the reference
 * tests' known answers.
 *
 * The POD input types are the ones of the public C ABI (include/exm_b200.h), so oracle and
 * product are driven with identical arguments.
 */
#ifndef EXM_ORACLE_H
#define EXM_ORACLE_H

#include <stdint.h>

#include "../include/exm_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct exo_ctx exo_ctx;

const char* exo_last_error(void);

/* MppiController construction: validation + prepare (controller.cpp:284-294). */
exo_ctx* exo_create(const exm_footprint* fp, const exm_model* model, const exm_limits* limits,
                    const exm_params* params);
void exo_destroy(exo_ctx* c);
/* The prepared footprint after validation (CW input reversed): polygon vertices or boxes. */
int32_t exo_footprint_count(const exo_ctx* c);
double exo_bounding_radius(const exo_ctx* c);

/* rng.hpp:12-58 */
uint64_t exo_splitmix64(uint64_t x);
uint64_t exo_hash_combine(uint64_t h, uint64_t v);
double exo_gaussian_at(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d);
double exo_uniform_range(uint64_t seed, uint64_t a, uint64_t b, double lo, double hi);
uint64_t exo_uniform_index(uint64_t seed, uint64_t a, uint64_t b, uint64_t n);
/* geometry.cpp:17-23 */
double exo_wrap_angle(double a);

/* geometry.cpp:260-296 (PreparedFootprint::sd) */
double exo_sd(const exo_ctx* c, double px, double py);
/* geometry.cpp:298-318 */
void exo_batch_signed_distance(const exo_ctx* c, const double* q, int32_t n, double* out);
/* geometry.cpp:357-375 */
double exo_min_signed_distance_at(const exo_ctx* c, const double pose[3], const double* pts,
                                  const uint8_t* mask, int32_t n);
/* P poses: per-pose min_signed_distance_at, and (optional) every per-pair sd (masked: +inf). */
void exo_sdf_batch(const exo_ctx* c, const double* poses, int32_t n_poses, const double* pts,
                   const uint8_t* mask, int32_t n, double* per_pair, double* per_pose_min);

/* kinematics.cpp:75-117 (u, u_prev, out: dim doubles; q: 3 doubles) */
void exo_clamp_control(const exo_ctx* c, const double* u, const double* u_prev, double* out);
void exo_step(const exo_ctx* c, const double q[3], const double* u, double out[3]);

/* controller.cpp:98-132 */
double exo_obstacle_cost(const exo_ctx* c, double d);
double exo_task_cost(const exo_ctx* c, const double q[3], const double* guide, int32_t n_guide,
                     const double goal[3], int32_t terminal);
double exo_terminal_goal_cost(const exo_ctx* c, const double q[3], const double goal[3]);
double exo_control_cost(const exo_ctx* c, const double* u);

/* controller.cpp:78-96 */
void exo_sample_perturbations(const exo_ctx* c, uint64_t seed, uint64_t cycle, double* eps);
/* controller.cpp:178-220 (every output may be NULL) */
int32_t exo_evaluate_rollouts(const exo_ctx* c, const double q0[3], const double* nominal,
                              const double* eps, const double* pts, const uint8_t* mask,
                              int32_t n, const double* guide, int32_t n_guide,
                              const double goal[3], const double* u_prev, double* controls,
                              double* states, double* dmin, double* costs, uint8_t* unsafe);
/* controller.cpp:222-233 */
void exo_weights_from_costs(const double* costs, int32_t k, double lambda, double* w);
/* controller.cpp:254-282 */
int32_t exo_validate_nominal(const exo_ctx* c, const double* nominal, const double q0[3],
                             const double* pts, const uint8_t* mask, int32_t n,
                             const double* guide, int32_t n_guide, const double goal[3],
                             const double* u_prev, int32_t* valid, double* dmin, double* cost);
/* controller.cpp:304-365 with the controller state passed explicitly (as the C ABI does). */
int32_t exo_control_cycle(const exo_ctx* c, const double q0[3], const double* pts,
                          const uint8_t* mask, int32_t n, const double* guide, int32_t n_guide,
                          const double goal[3], double* nominal_inout, double* u_prev_inout,
                          uint64_t cycle, const double* eps_or_null, exm_decision* out);

#ifdef __cplusplus
}
#endif

#endif
