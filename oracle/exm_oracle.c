/*
 * exm_oracle.c — TEST INFRASTRUCTURE ONLY (see exm_oracle.h). CPU restatement of the
 * reference's rollout + exact signed-distance path, one function per reference function.
 *
 * Parity pinned: bit-for-bit against the reference compiled from its own sources
 * (oracle/_ref, tests/test_oracle_ref.py) and against the reference tests' known answers
 * (tests/test_oracle_kat.py).
 */
#include "exm_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define EXO_PI 3.14159265358979323846
#define EXO_EMPTY 1e6     /* kEmptyMaskDistance, geometry.hpp:37 */
#define EXO_BOUNDARY 1e-12 /* kBoundaryEpsilon, geometry.hpp:39 */

static __thread char g_err[256];
static void set_err(const char* m) { snprintf(g_err, sizeof g_err, "%s", m); }
const char* exo_last_error(void) { return g_err; }

struct exo_ctx {
  int kind; /* EXM_FOOTPRINT_* */
  int count;
  /* polygon edges, SoA (prepare, geometry.cpp:236-247) */
  double *vx, *vy, *ex, *ey, *inv_len2;
  /* boxes (geometry.cpp:250-255) */
  double *cx, *cy, *hx, *hy;
  double radius;
  exm_model model;
  exm_limits limits;
  exm_params params;
  int dim;
};

/* ---------------- rng.hpp:12-58 ---------------- */
uint64_t exo_splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
uint64_t exo_hash_combine(uint64_t h, uint64_t v) {
  return exo_splitmix64(h ^ (v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2)));
}
static double unit_open_closed(uint64_t h) { return (double)((h >> 11) + 1) * 0x1.0p-53; }
double exo_gaussian_at(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  uint64_t k = exo_hash_combine(
      exo_hash_combine(exo_hash_combine(exo_hash_combine(exo_splitmix64(seed), a), b), c), d);
  double u1 = unit_open_closed(exo_hash_combine(k, 0xD1B54A32D192ED03ull));
  double u2 = unit_open_closed(exo_hash_combine(k, 0x8CB92BA72F3D8DD7ull));
  return sqrt(-2.0 * log(u1)) * cos(2.0 * EXO_PI * u2);
}
static uint64_t key3(uint64_t seed, uint64_t a, uint64_t b) {
  return exo_hash_combine(exo_hash_combine(exo_splitmix64(seed), a), b);
}
double exo_uniform_range(uint64_t seed, uint64_t a, uint64_t b, double lo, double hi) {
  double u = (double)(key3(seed, a, b) >> 11) * 0x1.0p-53;
  return lo + u * (hi - lo);
}
uint64_t exo_uniform_index(uint64_t seed, uint64_t a, uint64_t b, uint64_t n) {
  uint64_t k = key3(seed, a, b);
  return n == 0 ? 0 : k % n;
}

/* ---------------- geometry.cpp ---------------- */
double exo_wrap_angle(double a) { /* geometry.cpp:17-23 */
  const double tau = 2.0 * EXO_PI;
  a = fmod(a, tau);
  if (a <= -EXO_PI) a += tau;
  if (a > EXO_PI) a -= tau;
  return a;
}
static double hyp(double x, double y) { return sqrt(x * x + y * y); }
/* std::min / std::max / std::clamp exactly as libstdc++ defines them */
static double mn(double a, double b) { return (b < a) ? b : a; }
static double mx(double a, double b) { return (a < b) ? b : a; }
static double clampd(double v, double lo, double hi) { return (v < lo) ? lo : (hi < v) ? hi : v; }

static int orient(double ax, double ay, double bx, double by, double cx, double cy) {
  double v = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
  return v > 0.0 ? 1 : (v < 0.0 ? -1 : 0);
}
static int on_seg(double ax, double ay, double bx, double by, double px, double py) {
  return mn(ax, bx) <= px && px <= mx(ax, bx) && mn(ay, by) <= py && py <= mx(ay, by);
}
/* segments_intersect, geometry.cpp:43-54 */
static int seg_hit(const double* x, const double* y, int i, int j, int n) {
  double ax = x[i], ay = y[i], bx = x[(i + 1) % n], by = y[(i + 1) % n];
  double cx = x[j], cy = y[j], dx = x[(j + 1) % n], dy = y[(j + 1) % n];
  int o1 = orient(ax, ay, bx, by, cx, cy), o2 = orient(ax, ay, bx, by, dx, dy);
  int o3 = orient(cx, cy, dx, dy, ax, ay), o4 = orient(cx, cy, dx, dy, bx, by);
  if (o1 != o2 && o3 != o4) return 1;
  if (o1 == 0 && on_seg(ax, ay, bx, by, cx, cy)) return 1;
  if (o2 == 0 && on_seg(ax, ay, bx, by, dx, dy)) return 1;
  if (o3 == 0 && on_seg(cx, cy, dx, dy, ax, ay)) return 1;
  if (o4 == 0 && on_seg(cx, cy, dx, dy, bx, by)) return 1;
  return 0;
}

static int model_dim(int tag) { /* kinematics.cpp:14-26 */
  switch (tag) {
    case EXM_MODEL_DIFF:
    case EXM_MODEL_ACKERMANN: return 2;
    case EXM_MODEL_OMNI: return 3;
    case EXM_MODEL_SPIN:
    case EXM_MODEL_PARALLEL: return 1;
  }
  return 0;
}

static double* dup_arr(int n) { return (double*)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

void exo_destroy(exo_ctx* c) {
  if (!c) return;
  free(c->vx); free(c->vy); free(c->ex); free(c->ey); free(c->inv_len2);
  free(c->cx); free(c->cy); free(c->hx); free(c->hy);
  free(c);
}

exo_ctx* exo_create(const exm_footprint* fp, const exm_model* model, const exm_limits* limits,
                    const exm_params* p) {
  if (!fp || !model || !limits || !p) { set_err("null argument"); return NULL; }
  /* MppiParams::validate, controller.cpp:13-23 */
  if (p->rollouts < 1) { set_err("mppi: rollouts must be >= 1"); return NULL; }
  if (p->horizon < 1) { set_err("mppi: horizon must be >= 1"); return NULL; }
  if (!(p->dt > 0.0)) { set_err("mppi: dt must be positive"); return NULL; }
  if (!(p->lambda > 0.0)) { set_err("mppi: lambda must be positive"); return NULL; }
  for (int i = 0; i < 3; ++i)
    if (p->sigma[i] <= 0.0) { set_err("mppi: sigma components must be positive"); return NULL; }
  if (p->d_safe < 0.0) { set_err("mppi: d_safe must be nonnegative"); return NULL; }
  if (p->w_coll < 0.0 || p->w_rep < 0.0 || p->w_inf < 0.0) {
    set_err("mppi: penalty weights must be nonnegative");
    return NULL;
  }
  if (model_dim(model->tag) == 0) { set_err("unknown motion model"); return NULL; }
  if (model->tag == EXM_MODEL_ACKERMANN && model->wheelbase <= 0.0) {
    set_err("ackermann wheelbase must be positive"); /* kinematics.cpp:9-12 */
    return NULL;
  }
  int n = fp->count;
  exo_ctx* c = (exo_ctx*)calloc(1, sizeof *c);
  c->kind = fp->kind;
  c->count = n;
  c->model = *model;
  c->limits = *limits;
  c->params = *p;
  c->dim = model_dim(model->tag);
  if (fp->kind == EXM_FOOTPRINT_POLYGON) {
    /* PolygonFootprint::make, geometry.cpp:79-110 */
    if (n < 3 || !fp->x || !fp->y) { set_err("polygon needs at least 3 vertices"); exo_destroy(c); return NULL; }
    double* x = dup_arr(n);
    double* y = dup_arr(n);
    for (int i = 0; i < n; ++i) {
      x[i] = fp->x[i];
      y[i] = fp->y[i];
      if (!isfinite(x[i]) || !isfinite(y[i])) {
        set_err("polygon has non-finite vertex");
        free(x); free(y); exo_destroy(c); return NULL;
      }
    }
    for (int i = 0; i < n; ++i) {
      if (hyp(x[(i + 1) % n] - x[i], y[(i + 1) % n] - y[i]) == 0.0) {
        set_err("polygon has a zero-length edge");
        free(x); free(y); exo_destroy(c); return NULL;
      }
    }
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) {
        if (j == i + 1 || (i == 0 && j == n - 1)) continue;
        if (seg_hit(x, y, i, j, n)) {
          set_err("polygon boundary self-intersects");
          free(x); free(y); exo_destroy(c); return NULL;
        }
      }
    double area2 = 0.0; /* signed_area2, geometry.cpp:56-64 */
    for (int i = 0; i < n; ++i) area2 += x[i] * y[(i + 1) % n] - y[i] * x[(i + 1) % n];
    if (area2 < 0.0) {
      fprintf(stderr, "[exactmppi] warning: polygon given clockwise, reversing to CCW\n");
      for (int i = 0, j = n - 1; i < j; ++i, --j) {
        double t = x[i]; x[i] = x[j]; x[j] = t;
        t = y[i]; y[i] = y[j]; y[j] = t;
      }
    }
    /* prepare, geometry.cpp:233-247 */
    c->vx = dup_arr(n); c->vy = dup_arr(n); c->ex = dup_arr(n); c->ey = dup_arr(n);
    c->inv_len2 = dup_arr(n);
    for (int i = 0; i < n; ++i) {
      double ax = x[i], ay = y[i], bx = x[(i + 1) % n], by = y[(i + 1) % n];
      c->vx[i] = ax;
      c->vy[i] = ay;
      c->ex[i] = bx - ax;
      c->ey[i] = by - ay;
      c->inv_len2[i] = 1.0 / ((bx - ax) * (bx - ax) + (by - ay) * (by - ay));
      c->radius = mx(c->radius, hyp(ax, ay)); /* bounding_radius, geometry.cpp:127-131 */
    }
    free(x);
    free(y);
  } else if (fp->kind == EXM_FOOTPRINT_RECT_COVER) {
    /* RectangleCover::make, geometry.cpp:66-77 */
    if (n < 1 || !fp->x || !fp->y || !fp->hx || !fp->hy) {
      set_err("rectangle cover must be nonempty"); exo_destroy(c); return NULL;
    }
    c->cx = dup_arr(n); c->cy = dup_arr(n); c->hx = dup_arr(n); c->hy = dup_arr(n);
    for (int i = 0; i < n; ++i) {
      double X = fp->x[i], Y = fp->y[i], HX = fp->hx[i], HY = fp->hy[i];
      if (!isfinite(X) || !isfinite(Y) || !isfinite(HX) || !isfinite(HY)) {
        set_err("rectangle cover has non-finite entries"); exo_destroy(c); return NULL;
      }
      if (HX <= 0.0 || HY <= 0.0) {
        set_err("rectangle half-extents must be strictly positive"); exo_destroy(c); return NULL;
      }
      c->cx[i] = X; c->cy[i] = Y; c->hx[i] = HX; c->hy[i] = HY;
    }
    /* all_vertices order: (-,-), (+,-), (+,+), (-,+) per box, geometry.cpp:117-122 */
    for (int i = 0; i < n; ++i) {
      const double sx[4] = {-1, 1, 1, -1}, sy[4] = {-1, -1, 1, 1};
      for (int k = 0; k < 4; ++k) {
        double vx = sx[k] < 0 ? c->cx[i] - c->hx[i] : c->cx[i] + c->hx[i];
        double vy = sy[k] < 0 ? c->cy[i] - c->hy[i] : c->cy[i] + c->hy[i];
        c->radius = mx(c->radius, hyp(vx, vy));
      }
    }
  } else {
    set_err("unknown footprint kind");
    exo_destroy(c);
    return NULL;
  }
  return c;
}

int32_t exo_footprint_count(const exo_ctx* c) { return c->count; }
double exo_bounding_radius(const exo_ctx* c) { return c->radius; }

double exo_sd(const exo_ctx* c, double px, double py) { /* geometry.cpp:260-296 */
  if (c->kind == EXM_FOOTPRINT_RECT_COVER) {
    double best = INFINITY;
    for (int j = 0; j < c->count; ++j) {
      double ax = fabs(px - c->cx[j]) - c->hx[j];
      double ay = fabs(py - c->cy[j]) - c->hy[j];
      double ox = ax > 0.0 ? ax : 0.0, oy = ay > 0.0 ? ay : 0.0;
      double in = mx(ax, ay);
      best = mn(best, sqrt(ox * ox + oy * oy) + (in < 0.0 ? in : 0.0));
    }
    return best;
  }
  double best2 = INFINITY;
  int parity = 0;
  for (int b = 0; b < c->count; ++b) {
    double rx = px - c->vx[b], ry = py - c->vy[b];
    double t = (rx * c->ex[b] + ry * c->ey[b]) * c->inv_len2[b];
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    double qx = rx - t * c->ex[b], qy = ry - t * c->ey[b];
    double q2 = qx * qx + qy * qy;
    if (q2 < best2) best2 = q2;
    double y0 = c->vy[b], y1 = c->vy[b] + c->ey[b];
    if ((y0 < py) != (y1 < py)) {
      if (c->vx[b] + (py - y0) * c->ex[b] / c->ey[b] > px) parity ^= 1;
    }
  }
  double d = sqrt(best2);
  if (d < EXO_BOUNDARY) return 0.0;
  return parity ? -d : d;
}

void exo_batch_signed_distance(const exo_ctx* c, const double* q, int32_t n, double* out) {
  for (int32_t i = 0; i < n; ++i) out[i] = exo_sd(c, q[2 * i], q[2 * i + 1]);
}

double exo_min_signed_distance_at(const exo_ctx* c, const double pose[3], const double* pts,
                                  const uint8_t* mask, int32_t n) { /* geometry.cpp:357-375 */
  const double co = cos(pose[2]), si = sin(pose[2]);
  double best = EXO_EMPTY;
  int seen = 0;
  for (int32_t i = 0; i < n; ++i) {
    if (mask && !mask[i]) continue;
    double dx = pts[2 * i] - pose[0], dy = pts[2 * i + 1] - pose[1];
    double lim = c->radius + (seen ? best : EXO_EMPTY);
    /* exact bounding-radius prune: sd >= |p - t| - R */
    if (seen && lim > 0.0 && dx * dx + dy * dy >= lim * lim) continue;
    double d = exo_sd(c, co * dx + si * dy, -si * dx + co * dy);
    if (!seen || d < best) best = d;
    seen = 1;
  }
  return seen ? best : EXO_EMPTY;
}

void exo_sdf_batch(const exo_ctx* c, const double* poses, int32_t n_poses, const double* pts,
                   const uint8_t* mask, int32_t n, double* per_pair, double* per_pose_min) {
  for (int32_t p = 0; p < n_poses; ++p) {
    const double* q = poses + 3 * p;
    if (per_pose_min) per_pose_min[p] = exo_min_signed_distance_at(c, q, pts, mask, n);
    if (per_pair) {
      const double co = cos(q[2]), si = sin(q[2]);
      for (int32_t i = 0; i < n; ++i) {
        if (mask && !mask[i]) { per_pair[(size_t)p * n + i] = INFINITY; continue; }
        double dx = pts[2 * i] - q[0], dy = pts[2 * i + 1] - q[1];
        per_pair[(size_t)p * n + i] = exo_sd(c, co * dx + si * dy, -si * dx + co * dy);
      }
    }
  }
}

/* ---------------- kinematics.cpp:75-117 ---------------- */
void exo_clamp_control(const exo_ctx* c, const double* u, const double* u_prev, double* out) {
  const double dt = c->params.dt;
  for (int i = 0; i < c->dim; ++i) {
    double lo = c->limits.vel_min[i], hi = c->limits.vel_max[i];
    if (c->model.tag == EXM_MODEL_ACKERMANN && i == 1) {
      lo = mx(lo, -c->limits.steer_max);
      hi = mn(hi, c->limits.steer_max);
    }
    double v = clampd(u[i], lo, hi);
    out[i] = clampd(v, u_prev[i] + c->limits.acc_min[i] * dt, u_prev[i] + c->limits.acc_max[i] * dt);
  }
}

void exo_step(const exo_ctx* c, const double q[3], const double* u, double out[3]) {
  const double ct = cos(q[2]), st = sin(q[2]), dt = c->params.dt;
  double fx = 0.0, fy = 0.0, fth = 0.0;
  switch (c->model.tag) {
    case EXM_MODEL_DIFF: fx = u[0] * ct; fy = u[0] * st; fth = u[1]; break;
    case EXM_MODEL_ACKERMANN:
      fx = u[0] * ct; fy = u[0] * st; fth = u[0] / c->model.wheelbase * tan(u[1]); break;
    case EXM_MODEL_OMNI:
      fx = u[0] * ct - u[1] * st; fy = u[0] * st + u[1] * ct; fth = u[2]; break;
    case EXM_MODEL_SPIN: fth = u[0]; break;
    case EXM_MODEL_PARALLEL: fx = -u[0] * st; fy = u[0] * ct; break;
  }
  out[0] = q[0] + fx * dt;
  out[1] = q[1] + fy * dt;
  out[2] = q[2] + fth * dt;
}

/* ---------------- controller.cpp:50-132 ---------------- */
static void polyline_hit(const double* g, int32_t n, double px, double py, double* dist,
                         double* prog) { /* project_on_polyline, controller.cpp:50-66 */
  if (n == 1) { *dist = hyp(px - g[0], py - g[1]); *prog = 0.0; return; }
  double bd = INFINITY, bp = 0.0, arc = 0.0;
  for (int32_t i = 0; i + 1 < n; ++i) {
    double ax = g[2 * i], ay = g[2 * i + 1], bx = g[2 * i + 2], by = g[2 * i + 3];
    double sx = bx - ax, sy = by - ay;
    double len = hyp(sx, sy);
    double t = 0.0;
    if (len > 0.0) t = clampd(((px - ax) * sx + (py - ay) * sy) / (len * len), 0.0, 1.0);
    double d = hyp(px - (ax + t * sx), py - (ay + t * sy));
    if (d < bd) { bd = d; bp = arc + t * len; }
    arc += len;
  }
  *dist = bd;
  *prog = bp;
}

double exo_obstacle_cost(const exo_ctx* c, double d) {
  double m = mx(c->params.d_safe - d, 0.0);
  return c->params.w_coll * (d < 0.0 ? 1.0 : 0.0) + c->params.w_rep * m * m;
}

double exo_task_cost(const exo_ctx* c, const double q[3], const double* guide, int32_t n_guide,
                     const double goal[3], int32_t terminal) {
  double dx = q[0] - goal[0], dy = q[1] - goal[1];
  double cost = c->params.w_goal_pos * (dx * dx + dy * dy);
  if (terminal) {
    double e = exo_wrap_angle(q[2] - goal[2]);
    cost += c->params.w_goal_head * e * e;
  }
  double dist, prog;
  polyline_hit(guide, n_guide, q[0], q[1], &dist, &prog);
  cost += c->params.w_xtrack * dist * dist;
  cost -= c->params.w_progress * prog;
  return cost;
}

double exo_terminal_goal_cost(const exo_ctx* c, const double q[3], const double goal[3]) {
  double dx = q[0] - goal[0], dy = q[1] - goal[1];
  double e = exo_wrap_angle(q[2] - goal[2]);
  return c->params.w_goal_pos * (dx * dx + dy * dy) + c->params.w_goal_head * e * e;
}

double exo_control_cost(const exo_ctx* c, const double* u) {
  double s = 0.0;
  for (int i = 0; i < c->dim; ++i) s += u[i] * u[i];
  return c->params.w_ctrl * s;
}

/* ---------------- controller.cpp:78-96 ---------------- */
void exo_sample_perturbations(const exo_ctx* c, uint64_t seed, uint64_t cycle, double* eps) {
  const int K = c->params.rollouts, T = c->params.horizon, D = c->dim;
  for (int r = 0; r < K; ++r)
    for (int h = 0; h < T; ++h)
      for (int k = 0; k < D; ++k)
        eps[((size_t)r * T + h) * D + k] =
            c->params.sigma[k] * exo_gaussian_at(seed, cycle, (uint64_t)r, (uint64_t)h, (uint64_t)k);
}

/* ---------------- controller.cpp:138-220 ---------------- */
int32_t exo_evaluate_rollouts(const exo_ctx* c, const double q0[3], const double* nominal,
                              const double* eps, const double* pts, const uint8_t* mask,
                              int32_t n, const double* guide, int32_t n_guide,
                              const double goal[3], const double* u_prev, double* controls,
                              double* states, double* dmin, double* costs, uint8_t* unsafe) {
  if (n_guide < 1) { set_err("guidance polyline is empty"); return EXM_ERR_INVALID_ARGUMENT; }
  const int K = c->params.rollouts, T = c->params.horizon, D = c->dim;
  for (int r = 0; r < K; ++r) { /* score_rollout, controller.cpp:138-174 */
    double prev[3] = {0, 0, 0}, u[3] = {0, 0, 0}, uc[3] = {0, 0, 0};
    for (int k = 0; k < D; ++k) prev[k] = u_prev[k];
    double q[3] = {q0[0], q0[1], q0[2]};
    if (states) memcpy(states + (size_t)r * (T + 1) * 3, q, sizeof q);
    double J = 0.0;
    int flag = 0;
    for (int h = 0; h < T; ++h) {
      const double* e = eps + ((size_t)r * T + h) * D;
      for (int k = 0; k < D; ++k) u[k] = nominal[h * D + k] + e[k];
      exo_clamp_control(c, u, prev, uc);
      for (int k = 0; k < D; ++k) prev[k] = uc[k];
      if (controls) memcpy(controls + ((size_t)r * T + h) * D, uc, sizeof(double) * D);
      double d = exo_min_signed_distance_at(c, q, pts, mask, n);
      if (dmin) dmin[(size_t)r * T + h] = d;
      flag = flag || (d < c->params.d_safe);
      J += exo_task_cost(c, q, guide, n_guide, goal, 0);
      J += exo_control_cost(c, uc);
      J += exo_obstacle_cost(c, d);
      double nq[3];
      exo_step(c, q, uc, nq);
      q[0] = nq[0]; q[1] = nq[1]; q[2] = nq[2];
      if (states) memcpy(states + ((size_t)r * (T + 1) + h + 1) * 3, q, sizeof q);
    }
    J += exo_terminal_goal_cost(c, q, goal);
    if (costs) costs[r] = J;
    if (unsafe) unsafe[r] = flag ? 1 : 0;
  }
  return EXM_OK;
}

/* controller.cpp:222-233 */
void exo_weights_from_costs(const double* costs, int32_t k, double lambda, double* w) {
  double beta = costs[0];
  for (int32_t r = 1; r < k; ++r)
    if (costs[r] < beta) beta = costs[r];
  double s = 0.0;
  for (int32_t r = 0; r < k; ++r) {
    w[r] = exp(-(costs[r] - beta) / lambda);
    s += w[r];
  }
  for (int32_t r = 0; r < k; ++r) w[r] /= s;
}

/* controller.cpp:254-282 */
int32_t exo_validate_nominal(const exo_ctx* c, const double* nominal, const double q0[3],
                             const double* pts, const uint8_t* mask, int32_t n,
                             const double* guide, int32_t n_guide, const double goal[3],
                             const double* u_prev, int32_t* valid, double* dmin, double* cost) {
  if (n_guide < 1) { set_err("guidance polyline is empty"); return EXM_ERR_INVALID_ARGUMENT; }
  const int T = c->params.horizon, D = c->dim;
  double q[3] = {q0[0], q0[1], q0[2]}, prev[3] = {0, 0, 0}, u[3] = {0, 0, 0};
  for (int k = 0; k < D; ++k) prev[k] = u_prev[k];
  int ok = 1;
  double J = 0.0;
  for (int h = 0; h < T; ++h) {
    exo_clamp_control(c, nominal + h * D, prev, u);
    for (int k = 0; k < D; ++k) prev[k] = u[k];
    double d = exo_min_signed_distance_at(c, q, pts, mask, n);
    if (dmin) dmin[h] = d;
    if (d < c->params.d_safe) ok = 0;
    J += exo_task_cost(c, q, guide, n_guide, goal, 0);
    J += exo_control_cost(c, u);
    J += exo_obstacle_cost(c, d);
    double nq[3];
    exo_step(c, q, u, nq);
    q[0] = nq[0]; q[1] = nq[1]; q[2] = nq[2];
  }
  J += exo_terminal_goal_cost(c, q, goal);
  if (valid) *valid = ok;
  if (cost) *cost = J;
  return EXM_OK;
}

/* controller.cpp:304-365 */
int32_t exo_control_cycle(const exo_ctx* c, const double q0[3], const double* pts,
                          const uint8_t* mask, int32_t n, const double* guide, int32_t n_guide,
                          const double goal[3], double* nominal_inout, double* u_prev_inout,
                          uint64_t cycle, const double* eps_or_null, exm_decision* out) {
  const int K = c->params.rollouts, T = c->params.horizon, D = c->dim;
  if (n_guide < 1) { set_err("guidance polyline is empty"); return EXM_ERR_INVALID_ARGUMENT; }
  double* eps = (double*)malloc(sizeof(double) * (size_t)K * T * D);
  if (eps_or_null) memcpy(eps, eps_or_null, sizeof(double) * (size_t)K * T * D);
  else exo_sample_perturbations(c, c->params.seed, cycle, eps);
  double* J = (double*)malloc(sizeof(double) * K);
  uint8_t* bad = (uint8_t*)malloc((size_t)K);
  exo_evaluate_rollouts(c, q0, nominal_inout, eps, pts, mask, n, guide, n_guide, goal,
                        u_prev_inout, NULL, NULL, NULL, J, bad);
  for (int r = 0; r < K; ++r)
    if (bad[r]) J[r] += c->params.w_inf;
  double* w = (double*)malloc(sizeof(double) * K);
  exo_weights_from_costs(J, K, c->params.lambda, w);
  int arg = 0;
  for (int r = 1; r < K; ++r)
    if (J[r] < J[arg]) arg = r;
  double H = 0.0;
  for (int r = 0; r < K; ++r)
    if (w[r] > 0.0) H -= w[r] * log(w[r]);

  double* upd = (double*)malloc(sizeof(double) * T * D);
  memcpy(upd, nominal_inout, sizeof(double) * T * D);
  for (int h = 0; h < T; ++h)
    for (int r = 0; r < K; ++r)
      for (int k = 0; k < D; ++k) upd[h * D + k] += w[r] * eps[((size_t)r * T + h) * D + k];
  double prev[3] = {0, 0, 0};
  for (int k = 0; k < D; ++k) prev[k] = u_prev_inout[k];
  for (int h = 0; h < T; ++h) { /* sequential clamp, controller.cpp:331-337 */
    double tmp[3];
    exo_clamp_control(c, upd + h * D, prev, tmp);
    for (int k = 0; k < D; ++k) upd[h * D + k] = prev[k] = tmp[k];
  }
  int32_t ok = 0;
  double vcost = 0.0;
  exo_validate_nominal(c, upd, q0, pts, mask, n, guide, n_guide, goal, u_prev_inout, &ok,
                       out ? out->nominal_dmin : NULL, &vcost);
  double cmd[3] = {0, 0, 0};
  if (ok) {
    for (int k = 0; k < D; ++k) cmd[k] = upd[k];
    for (int h = 0; h + 1 < T; ++h)
      for (int k = 0; k < D; ++k) nominal_inout[h * D + k] = upd[(h + 1) * D + k];
    for (int k = 0; k < D; ++k) nominal_inout[(T - 1) * D + k] = upd[(T - 1) * D + k];
  } else {
    for (int i = 0; i < T * D; ++i) nominal_inout[i] = 0.0;
  }
  for (int k = 0; k < D; ++k) u_prev_inout[k] = cmd[k];
  if (out) {
    for (int k = 0; k < 3; ++k) out->command[k] = cmd[k];
    out->validated = ok;
    out->argmin = arg;
    out->best_cost = J[arg];
    out->weight_entropy = H;
    out->nominal_cost = vcost;
  }
  free(eps); free(J); free(bad); free(w); free(upd);
  return EXM_OK;
}
