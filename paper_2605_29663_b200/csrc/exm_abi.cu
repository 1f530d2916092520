// exm_abi.cu — host side of libexm_b200.so: the C ABI of include/exm_b200.h.
//
// A handle owns: the prepared FP32 footprint table (kernel parameter), device buffers
// sized at create for (K, T, n_cap, guide_cap), one non-blocking stream, two captured CUDA
// graphs of the control step (device-drawn noise / injected noise), pinned staging buffers
// for the host<->device copies of one step, and optionally an NCCL communicator (loaded with
// dlopen so the process shares whatever libnccl torch already mapped).
//
// Every failure returns a status and sets a thread-local message; there is no CPU fallback.
#include <dlfcn.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <limits>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/exm_b200.h"
#include "exm_common.cuh"
#include "exm_exact64.cuh"

using namespace exm;

namespace {

thread_local std::string g_err;

exm_status fail(exm_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

#define EXM_CUDA(call)                                                                   \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(EXM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));     \
  } while (0)

// ---- minimal NCCL surface, resolved at attach time -------------------------------------
typedef struct {
  char internal[128];
} nccl_uid_t;
typedef void* nccl_comm_t;
typedef int (*fn_get_uid)(nccl_uid_t*);
typedef int (*fn_init_rank)(nccl_comm_t*, int, nccl_uid_t, int);
typedef int (*fn_allgather)(const void*, void*, size_t, int, nccl_comm_t, cudaStream_t);
typedef int (*fn_destroy)(nccl_comm_t);
typedef const char* (*fn_errstr)(int);
constexpr int kNcclDouble = 8;  // ncclFloat64

struct NcclApi {
  void* lib = nullptr;
  fn_get_uid get_uid = nullptr;
  fn_init_rank init_rank = nullptr;
  fn_allgather allgather = nullptr;
  fn_destroy destroy = nullptr;
  fn_errstr errstr = nullptr;
  bool load() {
    if (lib) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (lib) break;
    }
    if (!lib) return false;
    get_uid = reinterpret_cast<fn_get_uid>(dlsym(lib, "ncclGetUniqueId"));
    init_rank = reinterpret_cast<fn_init_rank>(dlsym(lib, "ncclCommInitRank"));
    allgather = reinterpret_cast<fn_allgather>(dlsym(lib, "ncclAllGather"));
    destroy = reinterpret_cast<fn_destroy>(dlsym(lib, "ncclCommDestroy"));
    errstr = reinterpret_cast<fn_errstr>(dlsym(lib, "ncclGetErrorString"));
    return get_uid && init_rank && allgather && destroy;
  }
};
NcclApi g_nccl;
constexpr double kPiHost = 3.14159265358979323846;  // std::numbers::pi

template <class T>
cudaError_t dalloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
}

template <class T>
cudaError_t halloc(T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  return cudaMallocHost(reinterpret_cast<void**>(p), count * sizeof(T));
}

// One device block for the cloud structure of a handle (CloudGrid views, 16-byte aligned).
cudaError_t alloc_cloud_grid(int n_cap, void** block, CloudGrid* g) {
  const size_t n = static_cast<size_t>(n_cap > 0 ? n_cap : 1), cap = cloud_capacity(n_cap);
  const size_t cells = static_cast<size_t>(kGridMax) * kGridMax + 1;
  auto up = [](size_t b) { return (b + 15) & ~static_cast<size_t>(15); };
  const size_t o_raw = up(n * sizeof(float2)), o_cloud = o_raw + up(n * sizeof(float2));
  const size_t o_chunk = o_cloud + up(cap * sizeof(float2));
  const size_t o_rs = o_chunk + up((cap / 4 + 1) * sizeof(float4));  // chunks of >= 4 points
  const size_t o_cs = o_rs + up(cells * sizeof(int)), o_gm = o_cs + up(cells * sizeof(int));
  const size_t o_ds = o_gm + up(sizeof(GridMeta));
  char* d = nullptr;
  const size_t o_wk = o_ds + up(2 * sizeof(float));
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&d), o_wk + 2 * sizeof(unsigned));
  if (e != cudaSuccess) return e;
  e = cudaMemset(d + o_ds, 0, o_wk + 2 * sizeof(unsigned) - o_ds);
  if (e != cudaSuccess) return e;
  *block = d;
  g->tmp = reinterpret_cast<float2*>(d);
  g->raw = reinterpret_cast<float2*>(d + o_raw);
  g->cloud = reinterpret_cast<float2*>(d + o_cloud);
  g->chunk = reinterpret_cast<float4*>(d + o_chunk);
  g->raw_start = reinterpret_cast<int*>(d + o_rs);
  g->cell_start = reinterpret_cast<int*>(d + o_cs);
  g->gm = reinterpret_cast<GridMeta*>(d + o_gm);
  g->dstat = reinterpret_cast<float*>(d + o_ds);
  g->work = reinterpret_cast<unsigned*>(d + o_wk);
  return cudaSuccess;
}

int model_dim(int tag) {  // kinematics.cpp:14-26
  switch (tag) {
    case EXM_MODEL_DIFF:
    case EXM_MODEL_ACKERMANN: return 2;
    case EXM_MODEL_OMNI: return 3;
    case EXM_MODEL_SPIN:
    case EXM_MODEL_PARALLEL: return 1;
  }
  return 0;
}

// ---- footprint validation + FP32 table (geometry.cpp:66-110, :127-131, :230-258) -------
int orientation(double ax, double ay, double bx, double by, double cx, double cy) {
  const double v = (bx - ax) * (cy - ay) - (by - ay) * (cx - ax);
  return v > 0.0 ? 1 : (v < 0.0 ? -1 : 0);
}
bool within(double ax, double ay, double bx, double by, double px, double py) {
  return std::min(ax, bx) <= px && px <= std::max(ax, bx) && std::min(ay, by) <= py &&
         py <= std::max(ay, by);
}
bool segments_cross(const std::vector<double>& x, const std::vector<double>& y, size_t i,
                    size_t j) {
  const size_t n = x.size();
  const double ax = x[i], ay = y[i], bx = x[(i + 1) % n], by = y[(i + 1) % n];
  const double cx = x[j], cy = y[j], dx = x[(j + 1) % n], dy = y[(j + 1) % n];
  const int o1 = orientation(ax, ay, bx, by, cx, cy), o2 = orientation(ax, ay, bx, by, dx, dy);
  const int o3 = orientation(cx, cy, dx, dy, ax, ay), o4 = orientation(cx, cy, dx, dy, bx, by);
  if (o1 != o2 && o3 != o4) return true;
  return (o1 == 0 && within(ax, ay, bx, by, cx, cy)) || (o2 == 0 && within(ax, ay, bx, by, dx, dy)) ||
         (o3 == 0 && within(cx, cy, dx, dy, ax, ay)) || (o4 == 0 && within(cx, cy, dx, dy, bx, by));
}

// Bounding box {x0, x1, y0, y1} of the part of polygon (x, y) inside the slab
// lo <= coord < hi along `axis` (Sutherland-Hodgman clip against two half-planes); empty ->
// x0 > x1.
std::array<double, 4> clipped_box(const std::vector<double>& x, const std::vector<double>& y,
                                  int axis, double lo, double hi) {
  std::vector<std::array<double, 2>> poly;
  for (size_t i = 0; i < x.size(); ++i) poly.push_back({x[i], y[i]});
  auto clip = [&](double bound, bool keep_above) {
    std::vector<std::array<double, 2>> out;
    const size_t n = poly.size();
    for (size_t i = 0; i < n; ++i) {
      const auto& a = poly[i];
      const auto& b = poly[(i + 1) % n];
      const bool ina = keep_above ? a[axis] >= bound : a[axis] <= bound;
      const bool inb = keep_above ? b[axis] >= bound : b[axis] <= bound;
      if (ina) out.push_back(a);
      if (ina != inb) {
        const double t = (bound - a[axis]) / (b[axis] - a[axis]);
        out.push_back({a[0] + t * (b[0] - a[0]), a[1] + t * (b[1] - a[1])});
      }
    }
    poly = out;
  };
  clip(lo, true);
  if (!poly.empty()) clip(hi, false);
  std::array<double, 4> bb = {1e300, -1e300, 1e300, -1e300};
  for (const auto& v : poly) {
    bb[0] = std::min(bb[0], v[0]);
    bb[1] = std::max(bb[1], v[0]);
    bb[2] = std::min(bb[2], v[1]);
    bb[3] = std::max(bb[3], v[1]);
  }
  return bb;
}

// Does the union of boxes {x0, x1, y0, y1} cover segment a-b? (Liang-Barsky parameter
// intervals of the segment inside each box, merged over [0, 1].)
bool segment_covered(double ax, double ay, double bx, double by,
                     const std::vector<std::array<double, 4>>& boxes) {
  std::vector<std::pair<double, double>> iv;
  for (const auto& q : boxes) {
    double t0 = 0.0, t1 = 1.0;
    const double d[2] = {bx - ax, by - ay}, p0[2] = {ax, ay};
    bool ok = true;
    for (int k = 0; k < 2 && ok; ++k) {
      const double lo = q[2 * k], hi = q[2 * k + 1];
      if (d[k] == 0.0) {
        ok = p0[k] >= lo && p0[k] <= hi;
      } else {
        double u = (lo - p0[k]) / d[k], v = (hi - p0[k]) / d[k];
        if (u > v) std::swap(u, v);
        t0 = std::max(t0, u);
        t1 = std::min(t1, v);
        ok = t0 <= t1;
      }
    }
    if (ok) iv.push_back({t0, t1});
  }
  std::sort(iv.begin(), iv.end());
  double reach = 0.0;
  for (const auto& [u, v] : iv) {
    if (u > reach + 1e-12) return false;
    reach = std::max(reach, v);
  }
  return reach >= 1.0 - 1e-12;
}

// Greedy cover of a polygon by <= max_boxes axis-aligned boxes: repeatedly split the largest
// box at the vertex coordinate (either axis) that minimises the summed area of the two halves,
// each half being the bounding box of the polygon strictly on its side of the cut (a boundary
// edge lying on the cut line would otherwise stretch both halves), extended back to the cut.
// Exact (zero slack) for rectilinear polygons such as the L. The result is checked: if some
// edge is not covered by the union the cover falls back to the bounding box.
std::vector<std::array<double, 4>> cover_boxes(const std::vector<double>& x,
                                               const std::vector<double>& y, int max_boxes) {
  auto area = [](const std::array<double, 4>& b) {
    return b[0] > b[1] ? 0.0 : (b[1] - b[0]) * (b[3] - b[2]);
  };
  const std::array<double, 4> whole = clipped_box(x, y, 0, -1e300, 1e300);
  const double eps = 1e-9 * (1.0 + std::max(whole[1] - whole[0], whole[3] - whole[2]));
  std::vector<std::array<double, 4>> boxes = {whole};
  while (static_cast<int>(boxes.size()) < max_boxes) {
    size_t big = 0;
    for (size_t j = 1; j < boxes.size(); ++j)
      if (area(boxes[j]) > area(boxes[big])) big = j;
    const auto b = boxes[big];
    double best_gain = 1e-6 * area(b);
    int best_axis = -1;
    std::array<double, 4> best_lo{}, best_hi{};
    for (int axis = 0; axis < 2; ++axis) {
      const std::vector<double>& c = axis == 0 ? x : y;
      const double lo0 = axis == 0 ? b[0] : b[2], hi1 = axis == 0 ? b[1] : b[3];
      for (double cut : c) {
        if (cut <= lo0 + 2 * eps || cut >= hi1 - 2 * eps) continue;
        auto lo = clipped_box(x, y, axis, lo0, cut - eps);
        auto hi = clipped_box(x, y, axis, cut + eps, hi1);
        if (lo[0] > lo[1] || hi[0] > hi[1]) continue;
        lo[2 * axis + 1] = cut;
        hi[2 * axis] = cut;
        // restrict to the current box on the other axis
        const int o = axis == 0 ? 2 : 0;
        for (auto* q : {&lo, &hi}) {
          (*q)[o] = std::max((*q)[o], b[o]);
          (*q)[o + 1] = std::min((*q)[o + 1], b[o + 1]);
        }
        const double gain = area(b) - area(lo) - area(hi);
        if (gain > best_gain) {
          best_gain = gain;
          best_axis = axis;
          best_lo = lo;
          best_hi = hi;
        }
      }
    }
    if (best_axis < 0) break;
    boxes[big] = best_lo;
    boxes.push_back(best_hi);
  }
  // safety net: every polygon edge must lie in the union (slack eps on each box)
  std::vector<std::array<double, 4>> grown = boxes;
  for (auto& q : grown) q = {q[0] - 4 * eps, q[1] + 4 * eps, q[2] - 4 * eps, q[3] + 4 * eps};
  const size_t n = x.size();
  for (size_t i = 0; i < n; ++i)
    if (!segment_covered(x[i], y[i], x[(i + 1) % n], y[(i + 1) % n], grown)) return {whole};
  return boxes;
}

// PreparedFootprint in FP64 (geometry.cpp:230-257) for the EXM_OPT_SDF_FP64 path, from a
// footprint build_footprint has validated (same counter-clockwise orientation as the FP32 table).
void build_footprint64(const exm_footprint* fp, FpDev64* out) {
  std::memset(out, 0, sizeof *out);
  const int n = fp->count;
  out->kind = fp->kind;
  out->count = n;
  double radius = 0.0;
  if (fp->kind == EXM_FOOTPRINT_POLYGON) {
    std::vector<double> x(fp->x, fp->x + n), y(fp->y, fp->y + n);
    double area2 = 0.0;
    for (int i = 0; i < n; ++i) area2 += x[i] * y[(i + 1) % n] - y[i] * x[(i + 1) % n];
    if (area2 < 0.0) {
      std::reverse(x.begin(), x.end());
      std::reverse(y.begin(), y.end());
    }
    for (int i = 0; i < n; ++i) {
      const double ax = x[i], ay = y[i], bx = x[(i + 1) % n], by = y[(i + 1) % n];
      double* v = out->v[i];
      v[0] = ax;
      v[1] = ay;
      v[2] = bx - ax;
      v[3] = by - ay;
      v[4] = 1.0 / ((bx - ax) * (bx - ax) + (by - ay) * (by - ay));
      radius = std::max(radius, std::sqrt(ax * ax + ay * ay));
    }
  } else {
    for (int i = 0; i < n; ++i) {
      const double cx = fp->x[i], cy = fp->y[i], hx = fp->hx[i], hy = fp->hy[i];
      double* v = out->v[i];
      v[0] = cx;
      v[1] = cy;
      v[2] = hx;
      v[3] = hy;
      // FootprintSpec::bounding_radius over the cover's outline corners (geometry.cpp:127-145)
      const double xs[2] = {cx - hx, cx + hx}, ys[2] = {cy - hy, cy + hy};
      for (double vx : xs)
        for (double vy : ys) radius = std::max(radius, std::sqrt(vx * vx + vy * vy));
    }
  }
  out->radius = radius;
}

exm_status build_footprint(const exm_footprint* fp, FpDev* out) {
  std::memset(out, 0, sizeof *out);
  if (!fp) return fail(EXM_ERR_INVALID_ARGUMENT, "footprint is null");
  const int n = fp->count;
  double radius = 0.0;
  if (fp->kind == EXM_FOOTPRINT_POLYGON) {
    if (n < 3 || !fp->x || !fp->y)
      return fail(EXM_ERR_INVALID_ARGUMENT, "polygon needs at least 3 vertices");
    std::vector<double> x(fp->x, fp->x + n), y(fp->y, fp->y + n);
    for (int i = 0; i < n; ++i)
      if (!std::isfinite(x[i]) || !std::isfinite(y[i]))
        return fail(EXM_ERR_INVALID_ARGUMENT, "polygon has non-finite vertex");
    for (int i = 0; i < n; ++i) {
      const double ex = x[(i + 1) % n] - x[i], ey = y[(i + 1) % n] - y[i];
      if (std::sqrt(ex * ex + ey * ey) == 0.0)
        return fail(EXM_ERR_INVALID_ARGUMENT, "polygon has a zero-length edge");
    }
    for (int i = 0; i < n; ++i)
      for (int j = i + 1; j < n; ++j) {
        if (j == i + 1 || (i == 0 && j == n - 1)) continue;
        if (segments_cross(x, y, i, j))
          return fail(EXM_ERR_INVALID_ARGUMENT, "polygon boundary self-intersects");
      }
    double area2 = 0.0;
    for (int i = 0; i < n; ++i) area2 += x[i] * y[(i + 1) % n] - y[i] * x[(i + 1) % n];
    if (area2 < 0.0) {
      std::fprintf(stderr, "[exactmppi] warning: polygon given clockwise, reversing to CCW\n");
      std::reverse(x.begin(), x.end());
      std::reverse(y.begin(), y.end());
    }
    if (n > kMaxEdges)
      return fail(EXM_ERR_UNSUPPORTED, "polygon has more than 64 edges (kernel-parameter table)");
    out->kind = EXM_FOOTPRINT_POLYGON;
    out->count = n;
    for (int i = 0; i < n; ++i) {
      const double vx = x[i], vy = y[i];
      const double ex = x[(i + 1) % n] - vx, ey = y[(i + 1) % n] - vy;
      const double inv = 1.0 / (ex * ex + ey * ey);
      float* e = out->e[i];
      e[0] = static_cast<float>(vx);
      e[1] = static_cast<float>(vy);
      e[2] = static_cast<float>(ex);
      e[3] = static_cast<float>(ey);
      e[4] = static_cast<float>(ex * inv);
      e[5] = static_cast<float>(ey * inv);
      e[6] = static_cast<float>(-(vx * ex + vy * ey) * inv);
      e[7] = static_cast<float>(-ex);
      radius = std::max(radius, std::sqrt(vx * vx + vy * vy));
    }
  } else if (fp->kind == EXM_FOOTPRINT_RECT_COVER) {
    if (n < 1 || !fp->x || !fp->y || !fp->hx || !fp->hy)
      return fail(EXM_ERR_INVALID_ARGUMENT, "rectangle cover must be nonempty");
    if (n > kMaxEdges)
      return fail(EXM_ERR_UNSUPPORTED, "rectangle cover has more than 64 boxes");
    out->kind = EXM_FOOTPRINT_RECT_COVER;
    out->count = n;
    for (int i = 0; i < n; ++i) {
      const double cx = fp->x[i], cy = fp->y[i], hx = fp->hx[i], hy = fp->hy[i];
      if (!std::isfinite(cx) || !std::isfinite(cy) || !std::isfinite(hx) || !std::isfinite(hy))
        return fail(EXM_ERR_INVALID_ARGUMENT, "rectangle cover has non-finite entries");
      if (hx <= 0.0 || hy <= 0.0)
        return fail(EXM_ERR_INVALID_ARGUMENT, "rectangle half-extents must be strictly positive");
      float* e = out->e[i];
      e[0] = static_cast<float>(cx);
      e[1] = static_cast<float>(cy);
      e[2] = static_cast<float>(hx);
      e[3] = static_cast<float>(hy);
      const double xs[2] = {cx - hx, cx + hx}, ys[2] = {cy - hy, cy + hy};
      for (double vx : xs)
        for (double vy : ys) radius = std::max(radius, std::sqrt(vx * vx + vy * vy));
    }
  } else {
    return fail(EXM_ERR_INVALID_ARGUMENT, "unknown footprint kind");
  }
  out->radius = static_cast<float>(radius);
  // body-frame AABB of all vertices (corners for a cover), widened by one FP32 ulp-ish margin
  double bx0 = 1e300, bx1 = -1e300, by0 = 1e300, by1 = -1e300;
  for (int i = 0; i < out->count; ++i) {
    const float* e = out->e[i];
    const double xs[2] = {out->kind == EXM_FOOTPRINT_POLYGON ? e[0] : e[0] - e[2],
                          out->kind == EXM_FOOTPRINT_POLYGON ? e[0] : e[0] + e[2]};
    const double ys[2] = {out->kind == EXM_FOOTPRINT_POLYGON ? e[1] : e[1] - e[3],
                          out->kind == EXM_FOOTPRINT_POLYGON ? e[1] : e[1] + e[3]};
    for (double v : xs) { bx0 = std::min(bx0, v); bx1 = std::max(bx1, v); }
    for (double v : ys) { by0 = std::min(by0, v); by1 = std::max(by1, v); }
  }
  const double m = 1e-4 * (1.0 + radius);
  out->aabb[0] = static_cast<float>(bx0 - m);
  out->aabb[1] = static_cast<float>(bx1 + m);
  out->aabb[2] = static_cast<float>(by0 - m);
  out->aabb[3] = static_cast<float>(by1 + m);
  if (out->kind == EXM_FOOTPRINT_RECT_COVER) {
    // the cover union is the footprint itself when it has <= kMaxCover boxes, else the AABB
    const bool own = out->count <= kMaxCover;
    out->ncover = own ? out->count : 1;
    for (int j = 0; j < kMaxCover; ++j) {  // unused slots repeat box 0 (the kernel unrolls)
      const float* e = out->e[own && j < out->count ? j : 0];
      if (own) {
        out->cover[j][0] = e[0];
        out->cover[j][1] = e[1];
        out->cover[j][2] = static_cast<float>(e[2] + m);
        out->cover[j][3] = static_cast<float>(e[3] + m);
      } else {
        out->cover[j][0] = 0.5f * (out->aabb[0] + out->aabb[1]);
        out->cover[j][1] = 0.5f * (out->aabb[2] + out->aabb[3]);
        out->cover[j][2] = 0.5f * (out->aabb[1] - out->aabb[0]);
        out->cover[j][3] = 0.5f * (out->aabb[3] - out->aabb[2]);
      }
    }
  }
  if (out->kind == EXM_FOOTPRINT_POLYGON) {
    for (int b = 0; b < out->count + (out->count & 1); ++b) {
      float z[8] = {out->e[0][0], out->e[0][1], 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      const float* e = b < out->count ? out->e[b] : z;
      for (int k = 0; k < 8; ++k) out->ep[b / 2][k][b & 1] = e[k];
    }
  }
  if (out->kind == EXM_FOOTPRINT_POLYGON) {
    std::vector<double> px(out->count), py(out->count);
    for (int i = 0; i < out->count; ++i) {
      px[i] = out->e[i][0];
      py[i] = out->e[i][1];
    }
    const auto boxes = cover_boxes(px, py, kMaxCover);
    out->ncover = static_cast<int>(boxes.size());
    // The cut-line boxes have disjoint interiors and contain the polygon, so they tile it
    // exactly iff their areas sum to the polygon's area (rectilinear shapes: the L).
    double box_area = 0.0, poly2 = 0.0;
    for (const auto& bj : boxes) box_area += (bj[1] - bj[0]) * (bj[3] - bj[2]);
    for (int i = 0; i < out->count; ++i) {
      const int k = (i + 1) % out->count;
      poly2 += px[i] * py[k] - py[i] * px[k];
    }
    const double poly_area = 0.5 * std::fabs(poly2);
    out->cover_exact = std::fabs(box_area - poly_area) <= 1e-9 * std::max(poly_area, 1e-12) ? 1 : 0;
    out->cover_slack = static_cast<float>(m);
    for (int j = 0; j < kMaxCover; ++j) {  // unused slots repeat box 0 (the kernel unrolls)
      const auto& bj = boxes[static_cast<size_t>(j) < boxes.size() ? j : 0];
      out->cover[j][0] = static_cast<float>(0.5 * (bj[0] + bj[1]));
      out->cover[j][1] = static_cast<float>(0.5 * (bj[2] + bj[3]));
      out->cover[j][2] = static_cast<float>(0.5 * (bj[1] - bj[0]) + m);
      out->cover[j][3] = static_cast<float>(0.5 * (bj[3] - bj[2]) + m);
      out->cbox[j][0] = out->cover[j][0];
      out->cbox[j][1] = out->cover[j][1];
      out->cbox[j][2] = static_cast<float>(0.5 * (bj[1] - bj[0]));
      out->cbox[j][3] = static_cast<float>(0.5 * (bj[3] - bj[2]));
    }
#ifdef EXM_NO_COVER_EXACT  // A/B builds: every polygon point through the edge loop
    out->cover_exact = 0;
#endif
  }
  return EXM_OK;
}

exm_status check_params(const exm_params* p) {  // MppiParams::validate, controller.cpp:13-23
  if (p->rollouts < 1) return fail(EXM_ERR_INVALID_ARGUMENT, "mppi: rollouts must be >= 1");
  if (p->horizon < 1) return fail(EXM_ERR_INVALID_ARGUMENT, "mppi: horizon must be >= 1");
  if (!(p->dt > 0.0)) return fail(EXM_ERR_INVALID_ARGUMENT, "mppi: dt must be positive");
  if (!(p->lambda > 0.0)) return fail(EXM_ERR_INVALID_ARGUMENT, "mppi: lambda must be positive");
  for (double s : p->sigma)
    if (s <= 0.0) return fail(EXM_ERR_INVALID_ARGUMENT, "mppi: sigma components must be positive");
  if (p->d_safe < 0.0) return fail(EXM_ERR_INVALID_ARGUMENT, "mppi: d_safe must be nonnegative");
  if (p->w_coll < 0.0 || p->w_rep < 0.0 || p->w_inf < 0.0)
    return fail(EXM_ERR_INVALID_ARGUMENT, "mppi: penalty weights must be nonnegative");
  return EXM_OK;
}

struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
};

// A small persistent host thread pool for the FP64 <-> FP32 staging of batch_signed_distance
// (the caller's `threads`, geometry.cpp:298-318). run(n, fn) calls fn(0..n-1) on the workers and
// the calling thread and returns when all are done. Workers spin briefly between jobs (queries
// arrive in bursts of pipelined chunks), then sleep.
class HostPool {
 public:
  explicit HostPool(int workers) {
    for (int i = 0; i < workers; ++i) th_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return static_cast<int>(th_.size()) + 1; }
  void run(int n, const std::function<void(int)>& fn) {
    if (n <= 0) return;
    if (th_.empty() || n == 1) {
      for (int i = 0; i < n; ++i) fn(i);
      return;
    }
    fn_ = &fn;
    n_ = n;
    next_.store(0);
    done_.store(0);
    {
      std::lock_guard<std::mutex> lk(mu_);
      gen_.fetch_add(1);
    }
    cv_.notify_all();
    work();
    while (done_.load(std::memory_order_acquire) < n) std::this_thread::yield();
  }

 private:
  void work() {
    for (;;) {
      const int i = next_.fetch_add(1);
      if (i >= n_) return;
      (*fn_)(i);
      done_.fetch_add(1, std::memory_order_release);
    }
  }
  void loop() {
    unsigned seen = gen_.load();
    for (;;) {
      // spin ~100 us for the next job of a pipelined burst, then sleep
      const auto t0 = std::chrono::steady_clock::now();
      while (gen_.load(std::memory_order_acquire) == seen &&
             std::chrono::steady_clock::now() - t0 < std::chrono::microseconds(100))
        std::this_thread::yield();
      if (gen_.load(std::memory_order_acquire) == seen) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_.load() != seen; });
      }
      seen = gen_.load();
      if (stop_) return;
      work();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::atomic<unsigned> gen_{0};
  std::atomic<int> next_{0}, done_{0};
  int n_ = 0;
  const std::function<void(int)>* fn_ = nullptr;
  bool stop_ = false;
};

void world_free(exm_world* w);  // sensing workspace (defined with the world API below)

constexpr int kRingMax = 512;  // SDF timing events kept before they are folded into a sum
constexpr int kBsdSlots = 3;   // batch_signed_distance pipeline depth (chunks in flight)

}  // namespace

struct exm_handle {
  // Every ABI call on a handle holds its mutex: calls on one handle serialise (the drop-in's
  // handle cache may hand one handle to controllers on several threads).
  std::mutex mu;
  int device = 0;
  // options (exm_set_option)
  int sdf_mode = kSdfAuto;
  bool auto_caps = false, pregen = true, host_timing = false;
  // EXM_OPT_SDF_THRESHOLD: the control cycle's rollout minima are resolved only below d_safe
  // (sdf_thr = the least float whose double value is >= d_safe; results min(exact, sdf_thr))
  bool sdf_threshold = true;
  float sdf_thr = HUGE_VALF;
  // EXM_OPT_SDF_FP64: exm_evaluate_rollouts takes its minima from the FP64 brute-force kernel
  // (the reference's arithmetic) instead of the FP32 culled one
  bool sdf_fp64 = false;
  FpDev64 fp64{};
  double* d_dmin64 = nullptr;
  // what the last rollout / validation signed-distance launch ran (exm_last_sdf_path)
  SdfPath roll_path{}, val_path{};
  // lane <-> pose mapping of the thread-per-pose SDF (EXM_OPT_SDF_MAP): 0 tuned per handle (the
  // first kTuneSteps steps alternate both mappings outside a graph, timed with events), 1 one
  // rollout's consecutive steps per warp, 2 consecutive rollouts at one step per warp
  int sdf_map = 0;
  bool hmajor = false;
  int tune_n = 0;
  double tune_ms[2] = {0.0, 0.0};
  exm_world* sense_ws = nullptr;  // exm_sense's reused workspace
  // sharding without a communicator (exm_set_shard: several shard handles on one device)
  bool emulated = false;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // parallel graph branch (cloud preparation, noise pregeneration)
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr, pg_fork = nullptr, pg_join = nullptr;
  uint64_t* d_nstate = nullptr;  // StepConst::nstate
  double host_us[4] = {0.0, 0.0, 0.0, 0.0};  // EXM_HOST_TIMING
  int64_t host_calls = 0;
  FpDev fp{};
  StepConst sc{};
  int K = 0, T = 0, D = 0, n_cap = 0, guide_cap = 0;
  // sharding
  int rank = 0, world = 1;
  nccl_comm_t comm = nullptr;
  // device buffers
  StepDyn* d_dyn = nullptr;
  double* d_nominal = nullptr;
  double* d_guide = nullptr;
  double* d_pts = nullptr;
  uint8_t* d_mask = nullptr;
  CloudGrid grid;                 // per-step cloud structure (views into d_grid_block)
  void* d_grid_block = nullptr;
  double* d_eps = nullptr;
  float4* d_poses = nullptr;
  double* d_task = nullptr;  // task cost per (r, h), formed by the rollout kernel
  double* d_ctrl = nullptr;       // control cost per (r, h)
  float* d_hstat = nullptr;       // per-step d_min statistic {sum[T], sum of squares[T], count}
  float* d_cap = nullptr;         // per-step SDF caps for the next step (T; +inf: none)
  double* d_base = nullptr;
  float* d_dmin = nullptr;
  double* d_partials = nullptr;
  double* d_upd = nullptr;
  float4* d_val_poses = nullptr;
  double2* d_val_xy = nullptr;
  double* d_val_base = nullptr;
  float* d_val_dmin = nullptr;
  // contiguous output block: DecisionDev | nominal_dmin[T] | nominal[T*D] | u_prev[3]
  unsigned char* d_out = nullptr;
  size_t out_bytes = 0;
  // evaluate_rollouts extras (lazy)
  double* d_controls = nullptr;
  double* d_states = nullptr;
  double* d_cost = nullptr;
  uint8_t* d_unsafe = nullptr;
  // pinned staging
  unsigned char* d_in_block = nullptr;  // d_dyn | d_nominal | d_guide | d_pts | d_mask
  unsigned char* h_in_block = nullptr;  // pinned mirror, same layout
  StepDyn* h_dyn = nullptr;
  double* h_nominal = nullptr;
  double* h_guide = nullptr;
  double* h_pts = nullptr;  // end of the pinned mirror (the cloud is copied from the caller)
  uint8_t* h_mask = nullptr;
  unsigned char* h_out = nullptr;
  // graphs: [0] device noise, [1] injected noise
  cudaGraphExec_t exec[2] = {};
  cudaGraph_t graph[2] = {};  // kept alive: exec node updates need its nodes
  cudaGraphNode_t ev_node[2][2] = {};
  EventPair graph_ev;
  // per-step SDF timing ring (resident runs)
  std::vector<EventPair> ring;
  int ring_used = 0;
  EventPair step_ev;
  EventPair ev_set[2];  // events the exec's SDF event nodes currently record
  int last_steps = 0;
  double ring_ms = 0.0;  // SDF times folded out of a full ring
  int ring_n = 0;
  // SDF batch workspace (grown on demand)
  int sb_poses_cap = 0, sb_points_cap = 0;
  size_t sb_pairs_cap = 0;
  double* sb_poses64 = nullptr;
  double* sb_center = nullptr;
  float4* sb_poses = nullptr;
  double* sb_pts64 = nullptr;
  float2* sb_pts = nullptr;
  uint8_t* sb_mask = nullptr;
  unsigned* sb_keys = nullptr;
  double* sb_min = nullptr;
  float* sb_pairs = nullptr;
  int sb_P = 0, sb_N = 0, sb_has_mask = 0, sb_last_pairs = 0;
  // batch_signed_distance pipeline: kBsdSlots chunks of bsd_chunk queries, pinned FP32 staging
  // on the host, device buffers, one completion event per slot; host conversion pool
  int bsd_chunk = 0;
  float2* bsd_hq = nullptr;  // pinned [slot][chunk]
  float* bsd_hd = nullptr;   // pinned [slot][chunk]
  float2* bsd_dq = nullptr;
  float* bsd_dd = nullptr;
  cudaEvent_t bsd_ev[kBsdSlots] = {};
  cudaStream_t bsd_st[kBsdSlots] = {};  // one stream per slot: chunk copies overlap both ways
  int host_threads = 0;  // 0: default
  HostPool* pool = nullptr;
  int launches_per_step = 0;
  int64_t last_pairs = 0;
  // hybrid families share the pose / d_min arrays and family 0's cloud grid
  bool borrowed_poses = false, borrowed_cloud = false;
};

namespace {

DecisionDev* out_dec(exm_handle* h) { return reinterpret_cast<DecisionDev*>(h->d_out); }
double* out_dmin(exm_handle* h) { return reinterpret_cast<double*>(h->d_out + sizeof(DecisionDev)); }
double* out_nominal(exm_handle* h) { return out_dmin(h) + h->T; }
double* out_uprev(exm_handle* h) { return out_nominal(h) + h->T * h->D; }

void set_shard(exm_handle* h) {
  StepConst& sc = h->sc;
  sc.k_local = h->K / h->world;
  sc.r_offset = h->rank * sc.k_local;
  sc.nblocks_local = (sc.k_local + kBlockRollouts - 1) / kBlockRollouts;
  sc.block_offset = h->rank * sc.nblocks_local;
  sc.nblocks_total = sc.nblocks_local * h->world;
}

void destroy_graphs(exm_handle* h) {
  for (auto& e : h->exec)
    if (e) {
      cudaGraphExecDestroy(e);
      e = nullptr;
    }
  for (auto& g : h->graph)
    if (g) {
      cudaGraphDestroy(g);
      g = nullptr;
    }
}

// Phases of one control step (all stream-ordered, capturable):
//   prep  : cloud preparation (mask, recentre, grid, in-cell sort, chunk boxes) -> grid
//   pre   : [noise] -> rollout                                       -> d_poses, d_task, d_base
//   sdf   : per-pose exact SDF over the step's K*T poses             -> d_dmin
//   post  : stage costs -> block partials -> [all-gather] -> merge/update/validation
//           dynamics -> validation SDF -> finalize                    -> d_out, state
exm_status enqueue_prep(exm_handle* h, cudaStream_t s) {  // k_cloud_prep + k_cell_sort
  EXM_CUDA(launch_cloud_prep(h->d_pts, h->d_mask, h->d_dyn, h->fp.radius, h->grid, h->n_cap, s));
  return EXM_OK;
}

exm_status enqueue_pre(exm_handle* h, bool draw_noise, cudaStream_t s, int* launches) {
  const StepConst& sc = h->sc;
  EXM_CUDA(launch_rollout(sc, h->d_dyn, h->d_nominal, h->d_eps, draw_noise ? 1 : 0, h->d_poses,
                          h->d_task, h->d_guide, h->guide_cap, h->d_base, h->d_ctrl, nullptr,
                          nullptr, s));
  ++*launches;
  return EXM_OK;
}

// post, first half: rollout costs, softmax block partials of this rank's blocks, and (when
// pregen) the next cycle's noise on the side branch (forked after the last reader of eps)
exm_status enqueue_post_a(exm_handle* h, cudaStream_t s, int* launches, bool pregen) {
  const StepConst& sc = h->sc;
  // automatic per-step caps (d_min statistic -> k_finalize) measured slower than none on the
  // benchmark configs (fallback passes): off unless EXM_OPT_AUTO_CAPS; exm_set_sdf_caps still works
  float* hstat = h->auto_caps ? h->d_hstat : nullptr;
  EXM_CUDA(launch_rollout_costs(sc, h->d_task, h->d_base, h->d_ctrl, h->d_dmin, h->d_cost,
                                h->d_unsafe, h->grid.dstat, hstat, s));
  EXM_CUDA(launch_block_partials(sc, h->d_cost, h->d_unsafe, h->d_eps, h->d_partials, s));
  *launches += 2;
  if (pregen) {
    EXM_CUDA(cudaEventRecord(h->pg_fork, s));
    EXM_CUDA(cudaStreamWaitEvent(h->side, h->pg_fork, 0));
    EXM_CUDA(launch_noise_pregen(sc, h->d_eps, h->side));
    EXM_CUDA(cudaEventRecord(h->pg_join, h->side));
    ++*launches;
  }
  return EXM_OK;
}

// post, second half: exchange of the block partials (one in-place NCCL all-gather whenever a
// communicator is attached, including a 1-rank one), merge + update + validation dynamics,
// validation SDF, finalize
exm_status enqueue_post_b(exm_handle* h, cudaStream_t s, int* launches) {
  const StepConst& sc = h->sc;
  float* hstat = h->auto_caps ? h->d_hstat : nullptr;
  if (h->comm) {
    const size_t count = static_cast<size_t>(sc.nblocks_local) * partial_stride(sc.T, sc.D);
    const int rc = g_nccl.allgather(h->d_partials + static_cast<size_t>(sc.block_offset) *
                                                        partial_stride(sc.T, sc.D),
                                    h->d_partials, count, kNcclDouble, h->comm, s);
    if (rc != 0)
      return fail(EXM_ERR_NCCL, std::string("ncclAllGather: ") + (g_nccl.errstr ? g_nccl.errstr(rc) : "error"));
  }
  EXM_CUDA(launch_update(sc, h->d_partials, h->d_nominal, h->d_dyn, h->d_upd, h->d_val_poses,
                         h->d_val_xy, h->d_val_base, out_dec(h), 1, s));
  EXM_CUDA(launch_sdf_grid(h->fp, h->d_val_poses, sc.T, 0, false, h->grid, nullptr, h->sdf_mode,
                           h->d_val_dmin, &h->val_path, nullptr, s));
  EXM_CUDA(launch_finalize(sc, h->d_val_dmin, h->d_val_xy, h->d_val_base, h->d_upd, h->d_guide,
                           h->guide_cap, h->d_nominal, h->d_dyn, out_dec(h), out_dmin(h),
                           out_nominal(h), out_uprev(h), 1, hstat, h->d_cap, h->fp.radius, s));
  *launches += 3;
  return EXM_OK;
}

exm_status enqueue_post(exm_handle* h, cudaStream_t s, int* launches, bool pregen = false) {
  exm_status st = enqueue_post_a(h, s, launches, pregen);
  if (st != EXM_OK) return st;
  return enqueue_post_b(h, s, launches);
}

exm_status record_ev(cudaEvent_t e, cudaStream_t s, bool capturing) {
  EXM_CUDA(capturing ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                     : cudaEventRecord(e, s));
  return EXM_OK;
}

// Threshold of the rollout SDF (EXM_OPT_SDF_THRESHOLD): a minimum at or above d_safe costs
// exactly 0 in obstacle_cost (w_coll [d < 0] + w_rep max(d_safe - d, 0)^2, controller.cpp:98-101)
// and leaves the rollout safe (d < d_safe, :162); the control cycle returns no rollout minimum.
// So the search of a pose stops once no point can come nearer than d_safe, and the pose reports
// the least float t with double(t) >= d_safe: every cost and flag is what the exact minimum gives.
float rollout_threshold(const exm_handle* h, bool exact) {
  return (exact || !h->sdf_threshold) ? HUGE_VALF : h->sdf_thr;
}
float least_float_at_or_above(double d) {
  float f = static_cast<float>(d);
  if (static_cast<double>(f) < d) f = std::nextafter(f, HUGE_VALF);
  return f;
}

// The rollout SDF of a step (capped by the previous step's per-step statistic when set).
exm_status enqueue_rollout_sdf(exm_handle* h, cudaStream_t s, bool exact = false) {
  const StepConst& sc = h->sc;
  EXM_CUDA(launch_sdf_grid(h->fp, h->d_poses, sc.k_local * sc.T, sc.T, h->hmajor, h->grid, h->d_cap,
                           h->sdf_mode, h->d_dmin, &h->roll_path, nullptr, s,
                           rollout_threshold(h, exact)));
  h->roll_path.chunk = chunk_for_capacity(h->n_cap);
  h->val_path.chunk = h->roll_path.chunk;
  return EXM_OK;
}

// Head of the control step: the cloud preparation (single CTA) runs on a side stream
// concurrently with the noise + rollout branch, joined before the rollout SDF.
exm_status enqueue_head(exm_handle* h, bool draw_noise, const EventPair* ev, cudaStream_t s,
                        bool capturing, int* launches) {
  exm_status st;
  EXM_CUDA(cudaEventRecord(h->fork_ev, s));
  EXM_CUDA(cudaStreamWaitEvent(h->side, h->fork_ev, 0));
  if ((st = enqueue_prep(h, h->side)) != EXM_OK) return st;
  *launches += 2;
  EXM_CUDA(cudaEventRecord(h->join_ev, h->side));
  if ((st = enqueue_pre(h, draw_noise, s, launches)) != EXM_OK) return st;
  EXM_CUDA(cudaStreamWaitEvent(s, h->join_ev, 0));
  if (ev && (st = record_ev(ev->a, s, capturing)) != EXM_OK) return st;
  if ((st = enqueue_rollout_sdf(h, s)) != EXM_OK) return st;
  ++*launches;
  if (ev && (st = record_ev(ev->b, s, capturing)) != EXM_OK) return st;
  return EXM_OK;
}

bool pregen_for(const exm_handle* h, bool draw_noise) {
  return draw_noise && h->sc.nstate != nullptr && h->pregen;
}

size_t head_bytes(const exm_handle* h) {  // dyn | nominal | guide of the pinned mirror
  return static_cast<size_t>(reinterpret_cast<const unsigned char*>(h->h_pts) -
                             reinterpret_cast<const unsigned char*>(h->h_dyn));
}

// The control step (captured into the handle's graphs).
exm_status enqueue_step(exm_handle* h, bool draw_noise, const EventPair* ev, cudaStream_t s,
                        bool capturing) {
  int launches = 0;
  exm_status st = enqueue_head(h, draw_noise, ev, s, capturing, &launches);
  if (st != EXM_OK) return st;
  const bool pregen = pregen_for(h, draw_noise);
  if ((st = enqueue_post(h, s, &launches, pregen)) != EXM_OK) return st;
  if (pregen) EXM_CUDA(cudaStreamWaitEvent(s, h->pg_join, 0));
  h->launches_per_step = launches;
  return EXM_OK;
}

// Mapping tuning: steps 0-1 (cold caches, first grid) run r-major unmeasured, then steps 2..5
// alternate r-major / h-major; the faster total wins and the graphs are captured with it. Only
// the thread-per-pose kernel has a mapping (small pose sets take the warp kernel: no tuning).
constexpr int kTuneSteps = 6;
bool tuning(const exm_handle* h) { return h->sdf_map == 0 && h->tune_n < kTuneSteps; }

exm_status tune_step(exm_handle* h, bool draw_noise, EventPair* ev) {
  const int t = h->tune_n;
  h->hmajor = t >= 2 && (t & 1);
  exm_status st = enqueue_step(h, draw_noise, ev, h->stream, false);
  if (st != EXM_OK) return st;
  EXM_CUDA(cudaEventSynchronize(ev->b));
  float ms = 0.0f;
  EXM_CUDA(cudaEventElapsedTime(&ms, ev->a, ev->b));
  if (t >= 2) h->tune_ms[h->hmajor ? 1 : 0] += ms;
  h->tune_n = h->roll_path.kernel == 0 ? t + 1 : kTuneSteps;
  if (h->tune_n == kTuneSteps) {
    h->hmajor = h->roll_path.kernel == 0 && h->tune_ms[1] < h->tune_ms[0];
    destroy_graphs(h);
  }
  return EXM_OK;
}

exm_status ensure_graph(exm_handle* h, int variant) {
  if (h->exec[variant]) return EXM_OK;
  cudaGraph_t g = nullptr;
  EXM_CUDA(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
  exm_status st = enqueue_step(h, variant == 0, &h->graph_ev, h->stream, true);
  cudaError_t ce = cudaStreamEndCapture(h->stream, &g);
  if (st != EXM_OK) {
    if (g) cudaGraphDestroy(g);
    return st;
  }
  if (ce != cudaSuccess) return fail(EXM_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(ce));
  size_t nn = 0;
  EXM_CUDA(cudaGraphGetNodes(g, nullptr, &nn));
  std::vector<cudaGraphNode_t> nodes(nn);
  EXM_CUDA(cudaGraphGetNodes(g, nodes.data(), &nn));
  cudaGraphExec_t exec = nullptr;
  EXM_CUDA(cudaGraphInstantiate(&exec, g, 0));
  for (auto n : nodes) {
    cudaGraphNodeType t;
    EXM_CUDA(cudaGraphNodeGetType(n, &t));
    if (t != cudaGraphNodeTypeEventRecord) continue;
    cudaEvent_t e;
    EXM_CUDA(cudaGraphEventRecordNodeGetEvent(n, &e));
    if (e == h->graph_ev.a) h->ev_node[variant][0] = n;
    if (e == h->graph_ev.b) h->ev_node[variant][1] = n;
  }
  h->graph[variant] = g;
  h->exec[variant] = exec;
  h->ev_set[variant] = h->graph_ev;  // as captured
  return EXM_OK;
}

exm_status launch_graph(exm_handle* h, int variant, const EventPair& ev) {
  exm_status st = ensure_graph(h, variant);
  if (st != EXM_OK) return st;
  // retarget the SDF-bracketing event nodes only when the events change (benchmark rings);
  // repeated exm_control_cycle calls reuse step_ev and skip the two exec-node updates
  if (h->ev_node[variant][0] && (h->ev_set[variant].a != ev.a || h->ev_set[variant].b != ev.b)) {
    EXM_CUDA(cudaGraphExecEventRecordNodeSetEvent(h->exec[variant], h->ev_node[variant][0], ev.a));
    EXM_CUDA(cudaGraphExecEventRecordNodeSetEvent(h->exec[variant], h->ev_node[variant][1], ev.b));
    h->ev_set[variant] = ev;
  }
  EXM_CUDA(cudaGraphLaunch(h->exec[variant], h->stream));
  return EXM_OK;
}

// Next SDF timing event pair of a resident run. The ring holds at most kRingMax pairs: a full
// ring is folded (stream synchronised, times summed into ring_ms) so it never grows unbounded.
exm_status next_ring_slot(exm_handle* h, EventPair** out) {
  if (h->ring_used >= kRingMax) {
    EXM_CUDA(cudaStreamSynchronize(h->stream));
    for (int i = 0; i < h->ring_used; ++i) {
      float ms = 0.0f;
      EXM_CUDA(cudaEventElapsedTime(&ms, h->ring[i].a, h->ring[i].b));
      h->ring_ms += ms;
      ++h->ring_n;
    }
    h->ring_used = 0;
  }
  if (static_cast<int>(h->ring.size()) <= h->ring_used) {
    EventPair p;
    EXM_CUDA(cudaEventCreate(&p.a));
    EXM_CUDA(cudaEventCreate(&p.b));
    h->ring.push_back(p);
  }
  *out = &h->ring[h->ring_used++];
  return EXM_OK;
}

// A one-shot call (exm_control_cycle, exm_sdf_batch, ...) times its SDF with step_ev and
// replaces any pending resident accumulation.
void reset_timing(exm_handle* h, int steps) {
  h->ring_used = 0;
  h->ring_ms = 0.0;
  h->ring_n = 0;
  h->last_steps = steps;
}

exm_status check_cloud(const exm_handle* h, const double* pts, int32_t n) {
  if (n < 0 || n > h->n_cap) return fail(EXM_ERR_INVALID_ARGUMENT, "point count exceeds obstacle-set capacity");
  if (n > 0 && !pts) return fail(EXM_ERR_INVALID_ARGUMENT, "points pointer is null");
  return EXM_OK;
}

exm_status check_guide(const exm_handle* h, const double* g, int32_t n) {
  if (n < 1 || !g) return fail(EXM_ERR_INVALID_ARGUMENT, "guidance polyline is empty");
  if (n > h->guide_cap) return fail(EXM_ERR_INVALID_ARGUMENT, "guidance polyline exceeds guide_cap");
  return EXM_OK;
}

// EXM_OPT_HOST_TIMING: per-phase host wall time of exm_control_cycle (stage+enqueue H2D,
// graph launch + D2H enqueue, wait, unpack), accumulated per handle (exm_host_timing).
struct HostTimer {
  exm_handle* h;
  std::chrono::steady_clock::time_point t0;
  explicit HostTimer(exm_handle* hh) : h(hh) {
    if (h->host_timing) t0 = std::chrono::steady_clock::now();
  }
  void mark(int phase);
};

void HostTimer::mark(int phase) {
  if (!h->host_timing) return;
  const auto t = std::chrono::steady_clock::now();
  h->host_us[phase] += std::chrono::duration<double, std::micro>(t - t0).count();
  t0 = t;
  if (phase == 3) ++h->host_calls;
}

int default_host_threads() {
  const unsigned hw = std::thread::hardware_concurrency();
  return static_cast<int>(std::max(1u, std::min(8u, hw ? hw : 1u)));
}

// The handle's host pool (EXM_OPT_HOST_THREADS threads, the caller's thread included).
HostPool* ensure_pool(exm_handle* h) {
  const int threads = h->host_threads > 0 ? h->host_threads : default_host_threads();
  if (!h->pool || h->pool->size() != threads) {
    delete h->pool;
    h->pool = new HostPool(threads - 1);
  }
  return h->pool;
}

// The per-step state of the pinned mirror (StepDyn, nominal, guidance).
exm_status fill_head(exm_handle* h, const double q0[3], const double* pts, const uint8_t* mask,
                     int32_t n, const double* guide, int32_t ng, const double goal[3],
                     const double* nominal, const double* u_prev, uint64_t cycle) {
  exm_status st = check_cloud(h, pts, n);
  if (st != EXM_OK) return st;
  st = check_guide(h, guide, ng);
  if (st != EXM_OK) return st;
  if (!q0 || !goal || !nominal || !u_prev) return fail(EXM_ERR_INVALID_ARGUMENT, "null input pointer");
  StepDyn& d = *h->h_dyn;
  for (int i = 0; i < 3; ++i) {
    d.q0[i] = q0[i];
    d.goal[i] = goal[i];
    d.u_prev[i] = i < h->D ? u_prev[i] : 0.0;
  }
  d.cycle = cycle;
  d.n_points = n;
  d.n_guide = ng;
  d.use_mask = mask ? 1 : 0;
  d.reserved = 0;
  std::memcpy(h->h_nominal, nominal, static_cast<size_t>(h->T) * h->D * sizeof(double));
  std::memcpy(h->h_guide, guide, 2 * static_cast<size_t>(ng) * sizeof(double));
  return EXM_OK;
}

// Stage the per-step inputs into pinned memory and enqueue their H2D copies.
exm_status upload_inputs(exm_handle* h, const double q0[3], const double* pts, const uint8_t* mask,
                         int32_t n, const double* guide, int32_t ng, const double goal[3],
                         const double* nominal, const double* u_prev, uint64_t cycle) {
  // a mask without a zero byte selects every point: no mask copy (memchr scans 10 kB in < 1 us)
  if (mask && n > 0 && !std::memchr(mask, 0, static_cast<size_t>(n))) mask = nullptr;
  exm_status st = fill_head(h, q0, pts, mask, n, guide, ng, goal, nominal, u_prev, cycle);
  if (st != EXM_OK) return st;
  cudaStream_t s = h->stream;
  // The small state (dyn | nominal | guide) goes in one pinned copy; the cloud goes straight from
  // the caller's buffers: pageable ones are staged by the driver on this thread (measured 10 us
  // per config-2 call faster than a host memcpy into a pinned mirror plus an async copy), and
  // page-locked ones (exm_host_alloc) are a plain DMA: 180 vs 187 us per config-2 call
  // (tools/host_timing.py, round 2; host staging 4.7 vs 12.2 us).
  EXM_CUDA(cudaMemcpyAsync(h->d_dyn, h->h_dyn, head_bytes(h), cudaMemcpyHostToDevice, s));
  if (n > 0)
    EXM_CUDA(cudaMemcpyAsync(h->d_pts, pts, 2 * static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice, s));
  if (mask && n > 0)
    EXM_CUDA(cudaMemcpyAsync(h->d_mask, mask, static_cast<size_t>(n), cudaMemcpyHostToDevice, s));
  return EXM_OK;
}

// eps is about to hold noise that is not the handle's pregenerated cycle: forget the mark
exm_status invalidate_pregen(exm_handle* h) {
  if (h->d_nstate) EXM_CUDA(cudaMemsetAsync(h->d_nstate + 1, 0xff, sizeof(uint64_t), h->stream));
  return EXM_OK;
}

exm_status upload_eps(exm_handle* h, const double* eps) {
  if (const exm_status st = invalidate_pregen(h); st != EXM_OK) return st;
  const size_t row = static_cast<size_t>(h->T) * h->D;
  EXM_CUDA(cudaMemcpyAsync(h->d_eps, eps + static_cast<size_t>(h->sc.r_offset) * row,
                           static_cast<size_t>(h->sc.k_local) * row * sizeof(double),
                           cudaMemcpyHostToDevice, h->stream));
  return EXM_OK;
}

void unpack_decision(exm_handle* h, exm_decision* out, double* nominal_out, double* u_prev_out) {
  const DecisionDev* d = reinterpret_cast<const DecisionDev*>(h->h_out);
  const double* dmin = reinterpret_cast<const double*>(h->h_out + sizeof(DecisionDev));
  const double* nom = dmin + h->T;
  const double* up = nom + h->T * h->D;
  if (out) {
    for (int i = 0; i < 3; ++i) out->command[i] = d->command[i];
    out->validated = d->validated;
    out->argmin = d->argmin;
    out->best_cost = d->best_cost;
    out->weight_entropy = d->entropy;
    out->nominal_cost = d->nominal_cost;
    if (out->nominal_dmin) std::memcpy(out->nominal_dmin, dmin, sizeof(double) * h->T);
  }
  if (nominal_out) std::memcpy(nominal_out, nom, sizeof(double) * h->T * h->D);
  if (u_prev_out)
    for (int i = 0; i < h->D; ++i) u_prev_out[i] = up[i];
}

exm_status ensure_sdf_workspace(exm_handle* h, int P, int N, bool pairs) {
  if (!h->sb_center) EXM_CUDA(dalloc(&h->sb_center, 2));
  if (P > h->sb_poses_cap) {
    cudaFree(h->sb_poses);
    cudaFree(h->sb_poses64);
    cudaFree(h->sb_keys);
    cudaFree(h->sb_min);
    h->sb_poses_cap = 0;
    EXM_CUDA(dalloc(&h->sb_poses64, 3 * static_cast<size_t>(P)));
    EXM_CUDA(dalloc(&h->sb_poses, P));
    EXM_CUDA(dalloc(&h->sb_keys, P));
    EXM_CUDA(dalloc(&h->sb_min, P));
    h->sb_poses_cap = P;
  }
  if (N > h->sb_points_cap) {
    cudaFree(h->sb_pts64);
    cudaFree(h->sb_pts);
    cudaFree(h->sb_mask);
    h->sb_points_cap = 0;
    EXM_CUDA(dalloc(&h->sb_pts64, 2 * static_cast<size_t>(N)));
    EXM_CUDA(dalloc(&h->sb_pts, N));
    EXM_CUDA(dalloc(&h->sb_mask, N));
    h->sb_points_cap = N;
  }
  const size_t np = static_cast<size_t>(P) * N;
  if (pairs && np > h->sb_pairs_cap) {
    cudaFree(h->sb_pairs);
    h->sb_pairs_cap = 0;
    EXM_CUDA(dalloc(&h->sb_pairs, np));
    h->sb_pairs_cap = np;
  }
  return EXM_OK;
}

exm_status sdf_enqueue(exm_handle* h, bool pairs, const EventPair* ev) {
  cudaStream_t s = h->stream;
  EXM_CUDA(launch_fill_u32(h->sb_keys, 0xffffffffu, h->sb_P, s));
  if (ev) EXM_CUDA(cudaEventRecord(ev->a, s));
  EXM_CUDA(launch_sdf_pairs(h->fp, h->sb_poses, h->sb_P, h->sb_pts,
                            h->sb_has_mask ? h->sb_mask : nullptr, h->sb_N,
                            pairs ? h->sb_pairs : nullptr, h->sb_keys, s));
  if (ev) EXM_CUDA(cudaEventRecord(ev->b, s));
  EXM_CUDA(launch_min_keys_to_double(h->sb_keys, h->sb_P, h->sb_min, s));
  return EXM_OK;
}

}  // namespace

// =========================================================================== C ABI
extern "C" {

int32_t exm_abi_version(void) { return EXM_ABI_VERSION; }

const char* exm_last_error(void) { return g_err.c_str(); }

exm_status exm_create(const exm_footprint* footprint, const exm_model* model,
                      const exm_limits* limits, const exm_params* params, int32_t n_cap,
                      int32_t guide_cap, int32_t device, exm_handle** out) {
  if (!out) return fail(EXM_ERR_INVALID_ARGUMENT, "out handle pointer is null");
  *out = nullptr;
  if (!model || !limits || !params) return fail(EXM_ERR_INVALID_ARGUMENT, "null argument");
  FpDev fp;
  exm_status st = build_footprint(footprint, &fp);
  if (st != EXM_OK) return st;
  const int D = model_dim(model->tag);
  if (D == 0) return fail(EXM_ERR_INVALID_ARGUMENT, "unknown motion model");
  if (model->tag == EXM_MODEL_ACKERMANN && model->wheelbase <= 0.0)
    return fail(EXM_ERR_INVALID_ARGUMENT, "ackermann wheelbase must be positive");
  st = check_params(params);
  if (st != EXM_OK) return st;
  if (n_cap < 0 || guide_cap < 1) return fail(EXM_ERR_INVALID_ARGUMENT, "bad capacity");

  int dev = device;
  if (dev < 0) EXM_CUDA(cudaGetDevice(&dev));
  EXM_CUDA(cudaSetDevice(dev));
  auto* h = new exm_handle();
  h->device = dev;
  h->fp = fp;
  build_footprint64(footprint, &h->fp64);
  h->K = params->rollouts;
  h->T = params->horizon;
  h->D = D;
  h->n_cap = n_cap;
  h->guide_cap = guide_cap;
  StepConst& sc = h->sc;
  std::memset(&sc, 0, sizeof sc);
  sc.K = h->K;
  sc.T = h->T;
  sc.D = D;
  sc.tag = model->tag;
  sc.dt = params->dt;
  sc.lambda = params->lambda;
  sc.d_safe = params->d_safe;
  h->sdf_thr = least_float_at_or_above(params->d_safe);
  sc.w_coll = params->w_coll;
  sc.w_rep = params->w_rep;
  sc.w_inf = params->w_inf;
  sc.w_goal_pos = params->w_goal_pos;
  sc.w_goal_head = params->w_goal_head;
  sc.w_xtrack = params->w_xtrack;
  sc.w_progress = params->w_progress;
  sc.w_ctrl = params->w_ctrl;
  sc.wheelbase = model->wheelbase;
  for (int i = 0; i < 3; ++i) {
    sc.sigma[i] = params->sigma[i];
    sc.vel_min[i] = limits->vel_min[i];
    sc.vel_max[i] = limits->vel_max[i];
    sc.acc_min[i] = limits->acc_min[i];
    sc.acc_max[i] = limits->acc_max[i];
  }
  sc.steer_max = limits->steer_max;
  sc.seed = params->seed;
  set_shard(h);

  auto cleanup_fail = [&](exm_status s) {
    exm_destroy(h);
    return s;
  };
#define EXM_CUDA_C(call)                                                                 \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return cleanup_fail(fail(EXM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_))); \
  } while (0)
  EXM_CUDA_C(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  EXM_CUDA_C(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
  EXM_CUDA_C(cudaEventCreateWithFlags(&h->fork_ev, cudaEventDisableTiming));
  EXM_CUDA_C(cudaEventCreateWithFlags(&h->join_ev, cudaEventDisableTiming));
  EXM_CUDA_C(cudaEventCreateWithFlags(&h->pg_fork, cudaEventDisableTiming));
  EXM_CUDA_C(cudaEventCreateWithFlags(&h->pg_join, cudaEventDisableTiming));
  const size_t KT = static_cast<size_t>(h->K) * h->T;
  const size_t TD = static_cast<size_t>(h->T) * D;
  {
    auto al = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
    const size_t o_nom = al(sizeof(StepDyn));
    const size_t o_guide = o_nom + al(TD * sizeof(double));
    const size_t o_pts = o_guide + al(2 * static_cast<size_t>(guide_cap) * sizeof(double));
    const size_t o_mask = o_pts + al(2 * static_cast<size_t>(n_cap) * sizeof(double));
    const size_t total = o_mask + al(static_cast<size_t>(n_cap) + 1);
    unsigned char* d = nullptr;
    unsigned char* hh = nullptr;
    EXM_CUDA_C(dalloc(&d, total));
    EXM_CUDA_C(halloc(&hh, o_pts));  // pinned mirror of the small state only
    h->d_in_block = d;
    h->h_in_block = hh;
    h->d_dyn = reinterpret_cast<StepDyn*>(d);
    h->d_nominal = reinterpret_cast<double*>(d + o_nom);
    h->d_guide = reinterpret_cast<double*>(d + o_guide);
    h->d_pts = reinterpret_cast<double*>(d + o_pts);
    h->d_mask = d + o_mask;
    h->h_dyn = reinterpret_cast<StepDyn*>(hh);
    h->h_nominal = reinterpret_cast<double*>(hh + o_nom);
    h->h_guide = reinterpret_cast<double*>(hh + o_guide);
    h->h_pts = reinterpret_cast<double*>(hh + o_pts);  // end of the pinned mirror (not dereferenced)
    h->h_mask = nullptr;
  }
  EXM_CUDA_C(alloc_cloud_grid(n_cap, &h->d_grid_block, &h->grid));
  EXM_CUDA_C(dalloc(&h->d_eps, KT * D));
  EXM_CUDA_C(dalloc(&h->d_nstate, 2));
  EXM_CUDA_C(cudaMemset(h->d_nstate, 0xff, 2 * sizeof(uint64_t)));
  h->sc.nstate = h->d_nstate;
  EXM_CUDA_C(dalloc(&h->d_poses, KT));
  EXM_CUDA_C(dalloc(&h->d_task, KT));
  EXM_CUDA_C(dalloc(&h->d_ctrl, KT));
  EXM_CUDA_C(dalloc(&h->d_hstat, 2 * static_cast<size_t>(h->T) + 1));
  EXM_CUDA_C(cudaMemset(h->d_hstat, 0, (2 * static_cast<size_t>(h->T) + 1) * sizeof(float)));
  EXM_CUDA_C(dalloc(&h->d_cap, static_cast<size_t>(h->T)));
  {
    const std::vector<float> inf(static_cast<size_t>(h->T), HUGE_VALF);
    EXM_CUDA_C(cudaMemcpy(h->d_cap, inf.data(), inf.size() * sizeof(float), cudaMemcpyHostToDevice));
  }
  EXM_CUDA_C(dalloc(&h->d_cost, static_cast<size_t>(h->K)));
  EXM_CUDA_C(dalloc(&h->d_unsafe, static_cast<size_t>(h->K)));
  EXM_CUDA_C(dalloc(&h->d_base, static_cast<size_t>(h->K)));
  EXM_CUDA_C(dalloc(&h->d_dmin, KT));
  const size_t nblocks_max = (static_cast<size_t>(h->K) + kBlockRollouts - 1) / kBlockRollouts + 8;
  EXM_CUDA_C(dalloc(&h->d_partials, nblocks_max * partial_stride(h->T, D)));
  EXM_CUDA_C(dalloc(&h->d_upd, TD));
  EXM_CUDA_C(dalloc(&h->d_val_poses, static_cast<size_t>(h->T)));
  EXM_CUDA_C(dalloc(&h->d_val_xy, static_cast<size_t>(h->T)));
  EXM_CUDA_C(dalloc(&h->d_val_base, static_cast<size_t>(h->T) + 1));
  EXM_CUDA_C(dalloc(&h->d_val_dmin, static_cast<size_t>(h->T)));
  h->out_bytes = sizeof(DecisionDev) + sizeof(double) * (h->T + TD + 3);
  EXM_CUDA_C(dalloc(&h->d_out, h->out_bytes));
  EXM_CUDA_C(cudaMemset(h->d_out, 0, h->out_bytes));
  EXM_CUDA_C(halloc(&h->h_out, h->out_bytes));
  EXM_CUDA_C(cudaEventCreate(&h->graph_ev.a));
  EXM_CUDA_C(cudaEventCreate(&h->graph_ev.b));
  EXM_CUDA_C(cudaEventCreate(&h->step_ev.a));
  EXM_CUDA_C(cudaEventCreate(&h->step_ev.b));
#undef EXM_CUDA_C
  *out = h;
  return EXM_OK;
}

void exm_destroy(exm_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  destroy_graphs(h);
  if (h->comm && g_nccl.destroy) g_nccl.destroy(h->comm);
  if (h->borrowed_poses) h->d_poses = nullptr, h->d_dmin = nullptr;
  void* dev[] = {h->d_in_block, h->d_grid_block, h->d_eps, h->d_poses, h->d_task, h->d_ctrl,
                 h->d_hstat, h->d_cap, h->d_val_xy, h->d_base, h->d_dmin,
                 h->d_partials, h->d_upd, h->d_val_poses, h->d_val_base, h->d_val_dmin, h->d_out,
                 h->d_controls, h->d_states, h->d_cost, h->d_unsafe, h->sb_poses, h->sb_pts64,
                 h->sb_pts, h->sb_mask, h->sb_keys, h->sb_min, h->sb_pairs, h->d_nstate,
                 h->sb_poses64, h->sb_center, h->bsd_dq, h->bsd_dd, h->d_dmin64};
  for (void* p : dev)
    if (p) cudaFree(p);
  delete h->pool;
  world_free(h->sense_ws);
  for (auto e : h->bsd_ev)
    if (e) cudaEventDestroy(e);
  for (auto st : h->bsd_st)
    if (st) cudaStreamDestroy(st);
  void* host[] = {h->h_in_block, h->h_out, h->bsd_hq, h->bsd_hd};
  for (void* p : host)
    if (p) cudaFreeHost(p);
  for (auto& p : h->ring) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  EventPair* evs[] = {&h->graph_ev, &h->step_ev};
  for (auto* p : evs) {
    if (p->a) cudaEventDestroy(p->a);
    if (p->b) cudaEventDestroy(p->b);
  }
  if (h->fork_ev) cudaEventDestroy(h->fork_ev);
  if (h->join_ev) cudaEventDestroy(h->join_ev);
  if (h->pg_fork) cudaEventDestroy(h->pg_fork);
  if (h->pg_join) cudaEventDestroy(h->pg_join);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

exm_status exm_control_cycle(exm_handle* h, const double q0[3], const double* pts_xy,
                             const uint8_t* mask, int32_t n_points, const double* guide_xy,
                             int32_t n_guide, const double goal[3], double* nominal_inout,
                             double* u_prev_inout, uint64_t cycle, const double* eps_or_null,
                             exm_decision* out) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  if (!nominal_inout || !u_prev_inout) return fail(EXM_ERR_INVALID_ARGUMENT, "null state pointer");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->emulated) return fail(EXM_ERR_INVALID_ARGUMENT, "shard handle without a communicator: use exm_sharded_cycle");
  HostTimer ht(h);
  EXM_CUDA(cudaSetDevice(h->device));
  exm_status st;
  // inputs: the small state via the pinned mirror, the cloud straight from the caller's pageable
  // buffers (the driver stages them while this call returns). Measured against rounding the cloud
  // to FP32 on the host into pinned memory (async copy, or H2D/D2H memcpy nodes in the graph):
  // those are 8 and 11 us per config-2 call slower end to end (round 2).
  st = upload_inputs(h, q0, pts_xy, mask, n_points, guide_xy, n_guide, goal, nominal_inout,
                     u_prev_inout, cycle);
  if (st == EXM_OK && eps_or_null) st = upload_eps(h, eps_or_null);
  if (st != EXM_OK) return st;
  ht.mark(0);
  // the handle's first steps run as plain launches, both lane mappings timed (tune_step)
  st = tuning(h) ? tune_step(h, eps_or_null == nullptr, &h->step_ev)
                 : launch_graph(h, eps_or_null ? 1 : 0, h->step_ev);
  if (st != EXM_OK) return st;
  EXM_CUDA(cudaMemcpyAsync(h->h_out, h->d_out, h->out_bytes, cudaMemcpyDeviceToHost, h->stream));
  ht.mark(1);
  EXM_CUDA(cudaStreamSynchronize(h->stream));
  ht.mark(2);
  reset_timing(h, 1);
  h->last_pairs = static_cast<int64_t>(h->sc.k_local) * h->T * n_points;
  unpack_decision(h, out, nominal_inout, u_prev_inout);
  ht.mark(3);
  return EXM_OK;
}

exm_status exm_evaluate_rollouts(exm_handle* h, const double q0[3], const double* nominal,
                                 const double* eps, const double* pts_xy, const uint8_t* mask,
                                 int32_t n_points, const double* guide_xy, int32_t n_guide,
                                 const double goal[3], const double* u_prev,
                                 double* controls_out, double* states_out, double* dmin_out,
                                 double* costs_out, uint8_t* unsafe_out) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->world > 1) return fail(EXM_ERR_UNSUPPORTED, "evaluate_rollouts on a sharded handle");
  if (!eps) return fail(EXM_ERR_INVALID_ARGUMENT, "perturbation array does not match K*T");
  EXM_CUDA(cudaSetDevice(h->device));
  exm_status st = upload_inputs(h, q0, pts_xy, mask, n_points, guide_xy, n_guide, goal, nominal,
                                u_prev, 0);
  if (st != EXM_OK) return st;
  st = upload_eps(h, eps);
  if (st != EXM_OK) return st;
  const size_t KT = static_cast<size_t>(h->K) * h->T;
  const bool fp64 = h->sdf_fp64;
  if (controls_out && !h->d_controls) EXM_CUDA(dalloc(&h->d_controls, KT * h->D));
  if ((states_out || fp64) && !h->d_states)
    EXM_CUDA(dalloc(&h->d_states, static_cast<size_t>(h->K) * (h->T + 1) * 3));
  if (fp64 && !h->d_dmin64) EXM_CUDA(dalloc(&h->d_dmin64, KT));
  cudaStream_t s = h->stream;
  const StepConst& sc = h->sc;
  if (!fp64)
    EXM_CUDA(launch_cloud_prep(h->d_pts, h->d_mask, h->d_dyn, h->fp.radius, h->grid, h->n_cap, s));
  EXM_CUDA(launch_rollout(sc, h->d_dyn, h->d_nominal, h->d_eps, 0, h->d_poses, h->d_task,
                          h->d_guide, h->guide_cap, h->d_base, h->d_ctrl,
                          controls_out ? h->d_controls : nullptr,
                          (states_out || fp64) ? h->d_states : nullptr, s));
  if (fp64) {
    // the mask upload_inputs skipped is all ones
    const bool use_mask = mask && n_points > 0 && std::memchr(mask, 0, static_cast<size_t>(n_points));
    EXM_CUDA(launch_sdf_exact64(h->fp64, h->d_states, h->K, h->T, h->d_pts,
                                use_mask ? h->d_mask : nullptr, n_points, h->d_dmin64, s));
    EXM_CUDA(launch_rollout_costs_dmin64(sc, h->d_task, h->d_base, h->d_ctrl, h->d_dmin64,
                                         h->d_cost, h->d_unsafe, h->grid.dstat, s));
  } else {
    if (const exm_status st2 = enqueue_rollout_sdf(h, s, true); st2 != EXM_OK) return st2;
    EXM_CUDA(launch_rollout_costs(sc, h->d_task, h->d_base, h->d_ctrl, h->d_dmin, h->d_cost,
                                  h->d_unsafe, h->grid.dstat, nullptr, s));
  }
  if (controls_out)
    EXM_CUDA(cudaMemcpyAsync(controls_out, h->d_controls, KT * h->D * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (states_out)
    EXM_CUDA(cudaMemcpyAsync(states_out, h->d_states, static_cast<size_t>(h->K) * (h->T + 1) * 3 * sizeof(double),
                             cudaMemcpyDeviceToHost, s));
  std::vector<float> dmin_f;
  if (dmin_out && fp64) {
    EXM_CUDA(cudaMemcpyAsync(dmin_out, h->d_dmin64, KT * sizeof(double), cudaMemcpyDeviceToHost, s));
  } else if (dmin_out) {
    dmin_f.resize(KT);
    EXM_CUDA(cudaMemcpyAsync(dmin_f.data(), h->d_dmin, KT * sizeof(float), cudaMemcpyDeviceToHost, s));
  }
  if (costs_out)
    EXM_CUDA(cudaMemcpyAsync(costs_out, h->d_cost, h->K * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (unsafe_out)
    EXM_CUDA(cudaMemcpyAsync(unsafe_out, h->d_unsafe, h->K, cudaMemcpyDeviceToHost, s));
  EXM_CUDA(cudaStreamSynchronize(s));
  if (dmin_out && !fp64)
    for (size_t i = 0; i < KT; ++i) dmin_out[i] = static_cast<double>(dmin_f[i]);
  return EXM_OK;
}

exm_status exm_sample_perturbations(exm_handle* h, uint64_t seed, uint64_t cycle, double* eps_out) {
  if (!h || !eps_out) return fail(EXM_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->world > 1) return fail(EXM_ERR_UNSUPPORTED, "sample_perturbations on a sharded handle");
  EXM_CUDA(cudaSetDevice(h->device));
  StepConst sc = h->sc;
  sc.seed = seed;
  h->h_dyn->cycle = cycle;
  EXM_CUDA(cudaMemcpyAsync(h->d_dyn, h->h_dyn, sizeof(StepDyn), cudaMemcpyHostToDevice, h->stream));
  if (const exm_status st = invalidate_pregen(h); st != EXM_OK) return st;
  EXM_CUDA(launch_noise(sc, h->d_dyn, h->d_eps, h->stream));
  const size_t n = static_cast<size_t>(h->K) * h->T * h->D;
  EXM_CUDA(cudaMemcpyAsync(eps_out, h->d_eps, n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  EXM_CUDA(cudaStreamSynchronize(h->stream));
  return EXM_OK;
}

exm_status exm_validate_nominal(exm_handle* h, const double* nominal, const double q0[3],
                                const double* pts_xy, const uint8_t* mask, int32_t n_points,
                                const double* guide_xy, int32_t n_guide, const double goal[3],
                                const double* u_prev, int32_t* valid_out, double* dmin_out,
                                double* cost_out) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  EXM_CUDA(cudaSetDevice(h->device));
  exm_status st = upload_inputs(h, q0, pts_xy, mask, n_points, guide_xy, n_guide, goal, nominal,
                                u_prev, 0);
  if (st != EXM_OK) return st;
  cudaStream_t s = h->stream;
  const StepConst& sc = h->sc;
  EXM_CUDA(launch_cloud_prep(h->d_pts, h->d_mask, h->d_dyn, h->fp.radius, h->grid, h->n_cap, s));
  EXM_CUDA(launch_update(sc, nullptr, h->d_nominal, h->d_dyn, h->d_upd, h->d_val_poses,
                         h->d_val_xy, h->d_val_base, out_dec(h), 0, s));
  EXM_CUDA(launch_sdf_grid(h->fp, h->d_val_poses, sc.T, 0, false, h->grid, nullptr, h->sdf_mode,
                           h->d_val_dmin, &h->val_path, nullptr, s));
  EXM_CUDA(launch_finalize(sc, h->d_val_dmin, h->d_val_xy, h->d_val_base, h->d_upd, h->d_guide,
                           h->guide_cap, h->d_nominal, h->d_dyn, out_dec(h), out_dmin(h), nullptr,
                           nullptr, 0, nullptr, nullptr, h->fp.radius, s));
  EXM_CUDA(cudaMemcpyAsync(h->h_out, h->d_out, h->out_bytes, cudaMemcpyDeviceToHost, s));
  EXM_CUDA(cudaStreamSynchronize(s));
  const DecisionDev* d = reinterpret_cast<const DecisionDev*>(h->h_out);
  if (valid_out) *valid_out = d->validated;
  if (cost_out) *cost_out = d->nominal_cost;
  if (dmin_out) std::memcpy(dmin_out, h->h_out + sizeof(DecisionDev), sizeof(double) * h->T);
  return EXM_OK;
}

}  // extern "C"

namespace {

// exm_sdf_stage without the lock: poses and points go to the device as the caller's FP64 arrays
// (pageable copies return once the driver has staged them), the device takes the poses'
// centroid, recentres both in FP64 and rounds once. No host loop, no sync.
exm_status sdf_stage(exm_handle* h, const double* poses, int32_t n_poses, const double* pts_xy,
                     const uint8_t* mask, int32_t n_points) {
  if (n_poses < 0 || n_points < 0 || (n_poses > 0 && !poses) || (n_points > 0 && !pts_xy))
    return fail(EXM_ERR_INVALID_ARGUMENT, "bad pose/point arrays");
  EXM_CUDA(cudaSetDevice(h->device));
  exm_status st = ensure_sdf_workspace(h, std::max(n_poses, 1), std::max(n_points, 1), false);
  if (st != EXM_OK) return st;
  cudaStream_t s = h->stream;
  if (n_poses > 0)
    EXM_CUDA(cudaMemcpyAsync(h->sb_poses64, poses, 3 * static_cast<size_t>(n_poses) * sizeof(double),
                             cudaMemcpyHostToDevice, s));
  if (n_points > 0)
    EXM_CUDA(cudaMemcpyAsync(h->sb_pts64, pts_xy, 2 * static_cast<size_t>(n_points) * sizeof(double),
                             cudaMemcpyHostToDevice, s));
  if (mask && n_points > 0)
    EXM_CUDA(cudaMemcpyAsync(h->sb_mask, mask, static_cast<size_t>(n_points), cudaMemcpyHostToDevice, s));
  EXM_CUDA(launch_pose_prep(h->sb_poses64, n_poses, h->sb_center, h->sb_poses, s));
  EXM_CUDA(launch_recentre(h->sb_pts64, n_points, h->sb_center, h->sb_pts, s));
  h->sb_P = n_poses;
  h->sb_N = n_points;
  h->sb_has_mask = mask ? 1 : 0;
  return EXM_OK;
}

exm_status sdf_run(exm_handle* h, int32_t n_steps, bool want_pairs, bool resident) {
  EXM_CUDA(cudaSetDevice(h->device));
  exm_status st = ensure_sdf_workspace(h, std::max(h->sb_P, 1), std::max(h->sb_N, 1), want_pairs);
  if (st != EXM_OK) return st;
  if (!resident) reset_timing(h, 1);
  for (int i = 0; i < n_steps; ++i) {
    EventPair* ev = &h->step_ev;
    if (resident && (st = next_ring_slot(h, &ev)) != EXM_OK) return st;
    if ((st = sdf_enqueue(h, want_pairs, ev)) != EXM_OK) return st;
  }
  if (resident) h->last_steps = n_steps;
  h->sb_last_pairs = want_pairs ? 1 : 0;
  h->launches_per_step = 3;
  h->last_pairs = static_cast<int64_t>(h->sb_P) * h->sb_N;
  return EXM_OK;
}

exm_status sdf_read(exm_handle* h, float* per_pair, double* per_pose_min) {
  EXM_CUDA(cudaSetDevice(h->device));
  cudaStream_t s = h->stream;
  if (per_pair) {
    if (!h->sb_last_pairs) return fail(EXM_ERR_INVALID_ARGUMENT, "per-pair output was not computed");
    EXM_CUDA(cudaMemcpyAsync(per_pair, h->sb_pairs, static_cast<size_t>(h->sb_P) * h->sb_N * sizeof(float),
                             cudaMemcpyDeviceToHost, s));
  }
  if (per_pose_min)
    EXM_CUDA(cudaMemcpyAsync(per_pose_min, h->sb_min, static_cast<size_t>(h->sb_P) * sizeof(double),
                             cudaMemcpyDeviceToHost, s));
  EXM_CUDA(cudaStreamSynchronize(s));
  return EXM_OK;
}

// Pipeline buffers of batch_signed_distance for chunks of `chunk` queries (grown on demand).
exm_status ensure_bsd(exm_handle* h, int chunk) {
  ensure_pool(h);
  if (chunk <= h->bsd_chunk) return EXM_OK;
  cudaFreeHost(h->bsd_hq);
  cudaFreeHost(h->bsd_hd);
  cudaFree(h->bsd_dq);
  cudaFree(h->bsd_dd);
  h->bsd_hq = nullptr;
  h->bsd_hd = nullptr;
  h->bsd_dq = nullptr;
  h->bsd_dd = nullptr;
  h->bsd_chunk = 0;
  const size_t n = static_cast<size_t>(chunk) * kBsdSlots;
  EXM_CUDA(halloc(&h->bsd_hq, n));
  EXM_CUDA(halloc(&h->bsd_hd, n));
  EXM_CUDA(dalloc(&h->bsd_dq, n));
  EXM_CUDA(dalloc(&h->bsd_dd, n));
  for (auto& e : h->bsd_ev)
    if (!e) EXM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& st : h->bsd_st)
    if (!st) EXM_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  h->bsd_chunk = chunk;
  return EXM_OK;
}

}  // namespace

extern "C" {

exm_status exm_sdf_stage(exm_handle* h, const double* poses, int32_t n_poses,
                         const double* pts_xy, const uint8_t* mask, int32_t n_points) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  return sdf_stage(h, poses, n_poses, pts_xy, mask, n_points);
}

exm_status exm_sdf_run_resident(exm_handle* h, int32_t n_steps, int32_t want_pairs) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  return sdf_run(h, n_steps, want_pairs != 0, true);
}

exm_status exm_sdf_read(exm_handle* h, float* per_pair, double* per_pose_min) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  return sdf_read(h, per_pair, per_pose_min);
}

exm_status exm_sdf_batch(exm_handle* h, const double* poses, int32_t n_poses,
                         const double* pts_xy, const uint8_t* mask, int32_t n_points,
                         float* per_pair, double* per_pose_min) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  exm_status st = sdf_stage(h, poses, n_poses, pts_xy, mask, n_points);
  if (st != EXM_OK) return st;
  st = sdf_run(h, 1, per_pair != nullptr, false);
  if (st != EXM_OK) return st;
  return sdf_read(h, per_pair, per_pose_min);
}

// batch_signed_distance as a host-to-host pipeline: chunks of queries are rounded to FP32 into
// pinned staging by the host pool while earlier chunks are copied, evaluated (k_sdf_points) and
// copied back, each slot on its own stream (so one chunk's upload overlaps another's download);
// results are widened to FP64 into the caller's array as their chunks complete.
// Host traffic per query: 16 B read + 8 B pinned write in, 4 B pinned read + 8 B write out; link
// traffic 8 B in + 4 B out. Chunks: up to 8 of at least 64k queries (fixed per-chunk costs:
// three async calls, one event, one pool dispatch); small chunks convert on the calling thread.
exm_status exm_batch_signed_distance(exm_handle* h, const double* queries, int32_t n, double* out) {
  if (!h || (n > 0 && (!queries || !out))) return fail(EXM_ERR_INVALID_ARGUMENT, "null argument");
  if (n < 0) return fail(EXM_ERR_INVALID_ARGUMENT, "negative query count");
  if (n == 0) return EXM_OK;
  std::lock_guard<std::mutex> lk(h->mu);
  EXM_CUDA(cudaSetDevice(h->device));
  const int nchunks = std::min(8, std::max(1, (n + 65535) / 65536));
  const int chunk = ((n + nchunks - 1) / nchunks + 1023) & ~1023;
  // EXM_OPT_SDF_FP64: FP64 queries and results (16 B / 8 B, two staging elements per query)
  // evaluated by the reference's arithmetic (k_sdf_points64); else rounded to FP32
  const bool f64 = h->sdf_fp64;
  const int cap = f64 ? 2 * chunk : chunk;  // staging elements per slot
  exm_status st = ensure_bsd(h, cap);
  if (st != EXM_OK) return st;
  // pieces per conversion: ~16k queries each, at most the pool's threads
  const int parts = std::max(1, std::min(h->pool->size(), chunk / 16384));
  auto to_f32 = [&](int c, int part) {  // queries of chunk c -> pinned slot, piece `part`
    const size_t c0 = static_cast<size_t>(c) * chunk;
    const size_t m = std::min<size_t>(chunk, static_cast<size_t>(n) - c0);
    const size_t a = m * part / parts, b = m * (part + 1) / parts;
    float2* dst = h->bsd_hq + static_cast<size_t>(c % kBsdSlots) * cap;
    const double* src = queries + 2 * c0;
    if (f64) {
      std::memcpy(reinterpret_cast<double*>(dst) + 2 * a, src + 2 * a, (b - a) * 2 * sizeof(double));
      return;
    }
    for (size_t i = a; i < b; ++i)
      dst[i] = make_float2(static_cast<float>(src[2 * i]), static_cast<float>(src[2 * i + 1]));
  };
  auto to_f64 = [&](int c, int part) {  // results of chunk c -> caller, piece `part`
    const size_t c0 = static_cast<size_t>(c) * chunk;
    const size_t m = std::min<size_t>(chunk, static_cast<size_t>(n) - c0);
    const size_t a = m * part / parts, b = m * (part + 1) / parts;
    const float* src = h->bsd_hd + static_cast<size_t>(c % kBsdSlots) * cap;
    if (f64) {
      std::memcpy(out + c0 + a, reinterpret_cast<const double*>(src) + a, (b - a) * sizeof(double));
      return;
    }
    for (size_t i = a; i < b; ++i) out[c0 + i] = static_cast<double>(src[i]);
  };
  for (int c = 0; c < nchunks; ++c) {
    // the slot chunk c reuses held chunk c - kBsdSlots: drain it (widen its results) first
    const int drain = c - kBsdSlots;
    if (drain >= 0) EXM_CUDA(cudaEventSynchronize(h->bsd_ev[drain % kBsdSlots]));
    h->pool->run(2 * parts, [&](int t) {
      if (t < parts) to_f32(c, t);
      else if (drain >= 0) to_f64(drain, t - parts);
    });
    const size_t c0 = static_cast<size_t>(c) * chunk;
    const int m = static_cast<int>(std::min<size_t>(chunk, static_cast<size_t>(n) - c0));
    const int slot = c % kBsdSlots;
    const size_t so = static_cast<size_t>(slot) * cap;
    cudaStream_t s = h->bsd_st[slot];
    const size_t qb = f64 ? 2 * sizeof(double) : sizeof(float2), rb = f64 ? sizeof(double) : sizeof(float);
    EXM_CUDA(cudaMemcpyAsync(h->bsd_dq + so, h->bsd_hq + so, m * qb, cudaMemcpyHostToDevice, s));
    if (f64)
      EXM_CUDA(launch_sdf_points64(h->fp64, reinterpret_cast<const double*>(h->bsd_dq + so), m,
                                   reinterpret_cast<double*>(h->bsd_dd + so), s));
    else
      EXM_CUDA(launch_sdf_points(h->fp, h->bsd_dq + so, m, h->bsd_dd + so, s));
    EXM_CUDA(cudaMemcpyAsync(h->bsd_hd + so, h->bsd_dd + so, m * rb, cudaMemcpyDeviceToHost, s));
    EXM_CUDA(cudaEventRecord(h->bsd_ev[slot], s));
  }
  // the last min(kBsdSlots, nchunks) chunks
  for (int c = std::max(0, nchunks - kBsdSlots); c < nchunks; ++c) {
    EXM_CUDA(cudaEventSynchronize(h->bsd_ev[c % kBsdSlots]));
    h->pool->run(parts, [&](int t) { to_f64(c, t); });
  }
  return EXM_OK;
}

exm_status exm_nccl_unique_id(uint8_t id_out[128]) {
  if (!id_out) return fail(EXM_ERR_INVALID_ARGUMENT, "null id buffer");
  if (!g_nccl.load()) return fail(EXM_ERR_NCCL, "libnccl.so.2 not loadable");
  nccl_uid_t id;
  const int rc = g_nccl.get_uid(&id);
  if (rc != 0) return fail(EXM_ERR_NCCL, "ncclGetUniqueId failed");
  std::memcpy(id_out, id.internal, 128);
  return EXM_OK;
}

exm_status exm_attach_comm(exm_handle* h, int32_t rank, int32_t world, const uint8_t id[128]) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  if (world < 1 || rank < 0 || rank >= world) return fail(EXM_ERR_INVALID_ARGUMENT, "bad rank/world");
  if (world > 1 && h->K % (world * kBlockRollouts) != 0)
    return fail(EXM_ERR_INVALID_ARGUMENT, "rollouts must be a multiple of 256 * world for sharding");
  if (world > 1 && !id) return fail(EXM_ERR_INVALID_ARGUMENT, "null id");
  EXM_CUDA(cudaSetDevice(h->device));
  EXM_CUDA(cudaStreamSynchronize(h->stream));
  destroy_graphs(h);
  if (h->comm && g_nccl.destroy) {
    g_nccl.destroy(h->comm);
    h->comm = nullptr;
  }
  h->rank = rank;
  h->world = world;
  h->emulated = false;
  if (id) {  // any world, a 1-rank communicator included: the step graph then holds the all-gather
    if (!g_nccl.load()) return fail(EXM_ERR_NCCL, "libnccl.so.2 not loadable");
    nccl_uid_t uid;
    std::memcpy(uid.internal, id, 128);
    const int rc = g_nccl.init_rank(&h->comm, world, uid, rank);
    if (rc != 0) {
      h->comm = nullptr;
      h->rank = 0;
      h->world = 1;
      set_shard(h);
      return fail(EXM_ERR_NCCL, std::string("ncclCommInitRank: ") + (g_nccl.errstr ? g_nccl.errstr(rc) : "failed"));
    }
  }
  set_shard(h);
  return invalidate_pregen(h);  // the shard (and so the noise rows eps holds) changed
}

exm_status exm_set_shard(exm_handle* h, int32_t rank, int32_t world) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  if (world < 1 || rank < 0 || rank >= world) return fail(EXM_ERR_INVALID_ARGUMENT, "bad rank/world");
  if (world > 1 && h->K % (world * kBlockRollouts) != 0)
    return fail(EXM_ERR_INVALID_ARGUMENT, "rollouts must be a multiple of 256 * world for sharding");
  if (h->comm) return fail(EXM_ERR_INVALID_ARGUMENT, "handle has a communicator attached");
  EXM_CUDA(cudaSetDevice(h->device));
  EXM_CUDA(cudaStreamSynchronize(h->stream));
  destroy_graphs(h);
  h->rank = rank;
  h->world = world;
  h->emulated = world > 1;
  set_shard(h);
  return invalidate_pregen(h);
}

exm_status exm_sharded_cycle(exm_handle* const* shards, int32_t n_shards, const double q0[3],
                             const double* pts_xy, const uint8_t* mask, int32_t n_points,
                             const double* guide_xy, int32_t n_guide, const double goal[3],
                             double* nominals_inout, double* u_prevs_inout, uint64_t cycle,
                             const double* eps_or_null, exm_decision* out) {
  if (!shards || n_shards < 1 || !nominals_inout || !u_prevs_inout)
    return fail(EXM_ERR_INVALID_ARGUMENT, "null argument");
  const int G = n_shards;
  for (int g = 0; g < G; ++g) {
    const exm_handle* h = shards[g];
    if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
    if (h->rank != g || h->world != G || h->comm)
      return fail(EXM_ERR_INVALID_ARGUMENT, "shard g must be set to rank g of n_shards (exm_set_shard)");
    if (h->device != shards[0]->device || h->K != shards[0]->K || h->T != shards[0]->T ||
        h->D != shards[0]->D)
      return fail(EXM_ERR_INVALID_ARGUMENT, "shards differ in device or configuration");
  }
  std::vector<std::unique_lock<std::mutex>> locks;
  for (int g = 0; g < G; ++g) locks.emplace_back(shards[g]->mu);
  EXM_CUDA(cudaSetDevice(shards[0]->device));
  const size_t TD = static_cast<size_t>(shards[0]->T) * shards[0]->D;
  const bool draw = eps_or_null == nullptr;
  // 1. each shard: inputs, head (prep || rollout -> SDF) and its block partials, on its stream
  for (int g = 0; g < G; ++g) {
    exm_handle* h = shards[g];
    exm_status st = upload_inputs(h, q0, pts_xy, mask, n_points, guide_xy, n_guide, goal,
                                  nominals_inout + g * TD, u_prevs_inout + 3 * g, cycle);
    if (st != EXM_OK) return st;
    if (eps_or_null && (st = upload_eps(h, eps_or_null)) != EXM_OK) return st;
    int launches = 0;
    if ((st = enqueue_head(h, draw, nullptr, h->stream, false, &launches)) != EXM_OK) return st;
    if ((st = enqueue_post_a(h, h->stream, &launches, pregen_for(h, draw))) != EXM_OK) return st;
    EXM_CUDA(cudaEventRecord(h->fork_ev, h->stream));
  }
  // 2. the exchange the ranks' all-gather performs: every shard receives every other shard's
  //    blocks, one device-to-device copy per 256-rollout block
  for (int g = 0; g < G; ++g) {
    exm_handle* h = shards[g];
    const size_t stride = static_cast<size_t>(partial_stride(h->T, h->D)) * sizeof(double);
    for (int o = 0; o < G; ++o) {
      if (o == g) continue;
      const exm_handle* src = shards[o];
      EXM_CUDA(cudaStreamWaitEvent(h->stream, src->fork_ev, 0));
      for (int b = 0; b < src->sc.nblocks_local; ++b) {
        const size_t blk = static_cast<size_t>(src->sc.block_offset + b);
        EXM_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(h->d_partials) + blk * stride,
                                 reinterpret_cast<const char*>(src->d_partials) + blk * stride,
                                 stride, cudaMemcpyDeviceToDevice, h->stream));
      }
    }
  }
  // 3. each shard: merge, update, validation, finalize; decision back
  for (int g = 0; g < G; ++g) {
    exm_handle* h = shards[g];
    int launches = 0;
    exm_status st = enqueue_post_b(h, h->stream, &launches);
    if (st != EXM_OK) return st;
    if (pregen_for(h, draw)) EXM_CUDA(cudaStreamWaitEvent(h->stream, h->pg_join, 0));
    EXM_CUDA(cudaMemcpyAsync(h->h_out, h->d_out, h->out_bytes, cudaMemcpyDeviceToHost, h->stream));
  }
  for (int g = 0; g < G; ++g) {
    exm_handle* h = shards[g];
    EXM_CUDA(cudaStreamSynchronize(h->stream));
    h->last_steps = 0;
    unpack_decision(h, out ? out + g : nullptr, nominals_inout + g * TD, u_prevs_inout + 3 * g);
  }
  return EXM_OK;
}

exm_status exm_stage_inputs(exm_handle* h, const double q0[3], const double* pts_xy,
                            const uint8_t* mask, int32_t n_points, const double* guide_xy,
                            int32_t n_guide, const double goal[3], const double* nominal,
                            const double* u_prev, uint64_t cycle) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  EXM_CUDA(cudaSetDevice(h->device));
  exm_status st = upload_inputs(h, q0, pts_xy, mask, n_points, guide_xy, n_guide, goal, nominal,
                                u_prev, cycle);
  if (st != EXM_OK) return st;
  EXM_CUDA(cudaStreamSynchronize(h->stream));
  return EXM_OK;
}

exm_status exm_run_resident(exm_handle* h, int32_t n_steps) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  if (h->emulated) return fail(EXM_ERR_INVALID_ARGUMENT, "shard handle without a communicator: use exm_sharded_cycle");
  EXM_CUDA(cudaSetDevice(h->device));
  for (int i = 0; i < n_steps; ++i) {
    EventPair* ev = nullptr;
    exm_status st = next_ring_slot(h, &ev);
    if (st != EXM_OK) return st;
    if ((st = tuning(h) ? tune_step(h, true, ev) : launch_graph(h, 0, *ev)) != EXM_OK) return st;
  }
  h->last_steps = n_steps;
  h->last_pairs = static_cast<int64_t>(h->sc.k_local) * h->T * h->h_dyn->n_points;
  return EXM_OK;
}

exm_status exm_read_resident(exm_handle* h, double* nominal_out, double* u_prev_out, exm_decision* out) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  EXM_CUDA(cudaSetDevice(h->device));
  EXM_CUDA(cudaMemcpyAsync(h->h_out, h->d_out, h->out_bytes, cudaMemcpyDeviceToHost, h->stream));
  EXM_CUDA(cudaStreamSynchronize(h->stream));
  unpack_decision(h, out, nominal_out, u_prev_out);
  return EXM_OK;
}

void* exm_stream(exm_handle* h) { return h ? static_cast<void*>(h->stream) : nullptr; }

}  // extern "C"

// ---------------------------------------------------------------------------- sensing / world
// The device world (exm_world_*) and one-shot sensing (exm_sense) share this layout: base
// geometry (segments in the reference's sampling order, world.cpp:39-65; obstacles and polygon
// vertices for the line of sight), trails, and the per-obstacle state and offsets, in one device
// block; outputs staged through pinned memory.
struct exm_world {
  exm_handle* h = nullptr;
  int nseg = 0, n_obs = 0, budget = 0, sample_cap = 0;
  // capacities of the device block (a handle's one-shot sensing workspace is reused)
  int cap_seg = 0, cap_obs = 0, cap_verts = 0, cap_wp = 0, cap_budget = 0;
  void* bins = nullptr;  // BinState of the three sensing launches
  double range = 0.0;
  uint64_t seed = 0;
  void* d_block = nullptr;
  SenseSeg* seg = nullptr;
  SenseObs* obs = nullptr;
  double2* verts = nullptr;
  TrailDev* trails = nullptr;
  double2* waypoints = nullptr;
  double* arc = nullptr;
  int* dir = nullptr;
  double2* offsets = nullptr;
  int* seg_scratch = nullptr;
  double* d_scratch = nullptr;
  int* bin_scratch = nullptr;
  double* out_pts = nullptr;  // budget x 2, then mask (budget bytes), then n (int)
  uint8_t* out_mask = nullptr;
  int* out_n = nullptr;
  unsigned char* h_out = nullptr;  // pinned mirror of the output block
  size_t out_bytes = 0;
};

namespace {

struct WorldHost {
  std::vector<SenseSeg> seg;
  std::vector<SenseObs> obs;
  std::vector<double2> verts, waypoints, offsets;
  std::vector<TrailDev> trails;
  int sample_bound = 0;  // samples at zero offsets + one per segment (offsets move counts by rounding)
};

exm_status build_world(const exm_world_obstacle* o_in, int n, const exm_world_trail* tr,
                       WorldHost* w) {
  constexpr double kSpacing = 0.05;  // kBoundarySpacing, world.cpp:15
  w->obs.assign(static_cast<size_t>(n), SenseObs{});
  w->trails.assign(static_cast<size_t>(n), TrailDev{});
  w->offsets.assign(static_cast<size_t>(n), make_double2(0.0, 0.0));
  long long bound = 0;
  for (int i = 0; i < n; ++i) {
    const exm_world_obstacle& o = o_in[i];
    SenseObs& so = w->obs[static_cast<size_t>(i)];
    w->offsets[static_cast<size_t>(i)] = make_double2(o.offset[0], o.offset[1]);
    if (o.kind == EXM_OBSTACLE_POLYGON) {
      if (o.count < 3 || !o.x || !o.y) return fail(EXM_ERR_INVALID_ARGUMENT, "obstacle polygon needs at least 3 vertices");
      so.kind = 0;
      so.count = o.count;
      so.first = static_cast<int>(w->verts.size());
      for (int v = 0; v < o.count; ++v) w->verts.push_back(make_double2(o.x[v], o.y[v]));
      for (int v = 0; v < o.count; ++v) {
        const int u = v + 1 == o.count ? 0 : v + 1;
        SenseSeg g = {};
        g.kind = 0;
        g.obs = i;
        g.ax = o.x[v];
        g.ay = o.y[v];
        g.bx = o.x[u];
        g.by = o.y[u];
        const double ex = g.bx - g.ax, ey = g.by - g.ay;
        bound += std::max(1, static_cast<int>(std::ceil(std::sqrt(ex * ex + ey * ey) / kSpacing))) + 1;
        w->seg.push_back(g);
      }
    } else if (o.kind == EXM_OBSTACLE_DISC) {
      if (!o.x || !o.y || !(o.radius >= 0.0)) return fail(EXM_ERR_INVALID_ARGUMENT, "bad disc obstacle");
      so.kind = 1;
      so.cx = o.x[0];
      so.cy = o.y[0];
      so.r = o.radius;
      SenseSeg g = {};
      g.kind = 1;
      g.obs = i;
      g.ax = o.x[0];
      g.ay = o.y[0];
      g.r = o.radius;
      bound += std::max(8, static_cast<int>(std::ceil(2.0 * kPiHost * o.radius / kSpacing))) + 1;
      w->seg.push_back(g);
    } else {
      return fail(EXM_ERR_INVALID_ARGUMENT, "unknown obstacle kind");
    }
    if (tr && tr[i].n_waypoints >= 2) {  // TrailMotion (world.hpp): waypoints >= 2, speed >= 0
      if (!tr[i].waypoints || !(tr[i].speed >= 0.0))
        return fail(EXM_ERR_INVALID_ARGUMENT, "bad obstacle trail");
      TrailDev& t = w->trails[static_cast<size_t>(i)];
      t.first = static_cast<int>(w->waypoints.size());
      t.n = tr[i].n_waypoints;
      t.ping_pong = tr[i].ping_pong ? 1 : 0;
      t.speed = tr[i].speed;
      for (int k = 0; k < t.n; ++k)
        w->waypoints.push_back(make_double2(tr[i].waypoints[2 * k], tr[i].waypoints[2 * k + 1]));
    }
  }
  w->sample_bound = static_cast<int>(std::min<long long>(bound + 64, 1 << 26));
  return EXM_OK;
}

void world_free(exm_world* w) {
  if (!w) return;
  if (w->d_block) cudaFree(w->d_block);
  if (w->h_out) cudaFreeHost(w->h_out);
  delete w;
}

// Device block of a world (geometry + state + scratch + outputs) with room for `wh`; reuses `w`
// when its capacities suffice (a handle's one-shot sensing workspace), else reallocates.
exm_status world_reserve(exm_handle* h, const WorldHost& wh, int budget, exm_world** io) {
  exm_world* w = *io;
  const int nseg = static_cast<int>(wh.seg.size()), n_obs = static_cast<int>(wh.obs.size());
  const int nv = static_cast<int>(wh.verts.size()), nw = static_cast<int>(wh.waypoints.size());
  if (w && w->cap_seg >= nseg && w->cap_obs >= n_obs && w->cap_verts >= nv && w->cap_wp >= nw &&
      w->cap_budget >= budget && w->sample_cap >= wh.sample_bound) {
    w->nseg = nseg;
    w->n_obs = n_obs;
    w->budget = budget;
    w->out_n = reinterpret_cast<int*>(
        (reinterpret_cast<uintptr_t>(w->out_mask + budget) + 3) & ~static_cast<uintptr_t>(3));
    return EXM_OK;
  }
  world_free(w);
  *io = nullptr;
  w = new exm_world();
  w->h = h;
  w->nseg = nseg;
  w->n_obs = n_obs;
  w->budget = budget;
  w->cap_seg = std::max(nseg, 1);
  w->cap_obs = std::max(n_obs, 1);
  w->cap_verts = std::max(nv, 1);
  w->cap_wp = std::max(nw, 1);
  w->cap_budget = budget;
  w->sample_cap = wh.sample_bound;
  auto up = [](size_t b) { return (b + 255) & ~static_cast<size_t>(255); };
  size_t off = 0;
  const size_t o_seg = off; off += up(w->cap_seg * sizeof(SenseSeg));
  const size_t o_obs = off; off += up(w->cap_obs * sizeof(SenseObs));
  const size_t o_ver = off; off += up(w->cap_verts * sizeof(double2));
  const size_t o_tr = off; off += up(w->cap_obs * sizeof(TrailDev));
  const size_t o_wp = off; off += up(w->cap_wp * sizeof(double2));
  const size_t o_off = off; off += up(w->cap_obs * sizeof(double2));
  const size_t o_arc = off; off += up(w->cap_obs * sizeof(double));
  const size_t o_dir = off; off += up(w->cap_obs * sizeof(int));
  const size_t o_ss = off; off += up(2 * static_cast<size_t>(w->cap_seg) * sizeof(int));
  const size_t o_ds = off; off += up(static_cast<size_t>(w->sample_cap) * sizeof(double));
  const size_t o_bs = off; off += up(static_cast<size_t>(w->sample_cap) * sizeof(int));
  const size_t o_bins = off; off += up(sense_bin_state_bytes());
  const size_t o_out = off;
  w->out_bytes = static_cast<size_t>(budget) * (2 * sizeof(double) + 1) + 16;
  off += up(w->out_bytes);
  cudaError_t e = cudaMalloc(&w->d_block, off);
  if (e == cudaSuccess) e = cudaMallocHost(reinterpret_cast<void**>(&w->h_out), w->out_bytes);
  if (e != cudaSuccess) {
    world_free(w);
    return fail(EXM_ERR_CUDA, std::string("world alloc: ") + cudaGetErrorString(e));
  }
  char* d = static_cast<char*>(w->d_block);
  w->seg = reinterpret_cast<SenseSeg*>(d + o_seg);
  w->obs = reinterpret_cast<SenseObs*>(d + o_obs);
  w->verts = reinterpret_cast<double2*>(d + o_ver);
  w->trails = reinterpret_cast<TrailDev*>(d + o_tr);
  w->waypoints = reinterpret_cast<double2*>(d + o_wp);
  w->offsets = reinterpret_cast<double2*>(d + o_off);
  w->arc = reinterpret_cast<double*>(d + o_arc);
  w->dir = reinterpret_cast<int*>(d + o_dir);
  w->seg_scratch = reinterpret_cast<int*>(d + o_ss);
  w->d_scratch = reinterpret_cast<double*>(d + o_ds);
  w->bin_scratch = reinterpret_cast<int*>(d + o_bs);
  w->bins = d + o_bins;
  w->out_pts = reinterpret_cast<double*>(d + o_out);
  w->out_mask = reinterpret_cast<uint8_t*>(w->out_pts + 2 * static_cast<size_t>(budget));
  // n after the mask, 4-byte aligned (out_bytes leaves room for it)
  w->out_n = reinterpret_cast<int*>(
      (reinterpret_cast<uintptr_t>(w->out_mask + budget) + 3) & ~static_cast<uintptr_t>(3));
  *io = w;
  return EXM_OK;
}

// Geometry, trails and the initial state (WorldState::initial: arc 0, direction +1) to the device.
exm_status world_upload(exm_world* w, const WorldHost& wh, double range, uint64_t seed) {
  w->range = range;
  w->seed = seed;
  cudaStream_t s = w->h->stream;
  // the geometry copies are small; pageable copies return once the driver has staged them
  auto h2d = [&](void* dst, const void* src, size_t bytes) {
    return bytes ? cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s) : cudaSuccess;
  };
  const size_t n_o = wh.obs.size();
  std::vector<double> arc0(n_o, 0.0);
  std::vector<int> dir0(n_o, 1);
  cudaError_t e;
  if ((e = h2d(w->seg, wh.seg.data(), wh.seg.size() * sizeof(SenseSeg))) != cudaSuccess ||
      (e = h2d(w->obs, wh.obs.data(), n_o * sizeof(SenseObs))) != cudaSuccess ||
      (e = h2d(w->verts, wh.verts.data(), wh.verts.size() * sizeof(double2))) != cudaSuccess ||
      (e = h2d(w->trails, wh.trails.data(), wh.trails.size() * sizeof(TrailDev))) != cudaSuccess ||
      (e = h2d(w->waypoints, wh.waypoints.data(), wh.waypoints.size() * sizeof(double2))) != cudaSuccess ||
      (e = h2d(w->offsets, wh.offsets.data(), n_o * sizeof(double2))) != cudaSuccess ||
      (e = h2d(w->arc, arc0.data(), n_o * sizeof(double))) != cudaSuccess ||
      (e = h2d(w->dir, dir0.data(), n_o * sizeof(int))) != cudaSuccess)
    return fail(EXM_ERR_CUDA, std::string("world upload: ") + cudaGetErrorString(e));
  return EXM_OK;
}

// sense() on the device with the world's current offsets; the padded ObstacleSet back to the host.
exm_status world_sense(exm_world* w, const double robot[3], uint64_t sample_key, double* pts_out,
                       uint8_t* mask_out, int32_t* n_valid) {
  cudaStream_t s = w->h->stream;
  EXM_CUDA(launch_sense(w->seg, w->nseg, w->obs, w->n_obs, w->verts, w->offsets, robot[0],
                        robot[1], w->range, w->budget, w->seed, sample_key, w->seg_scratch,
                        w->d_scratch, w->bin_scratch, w->sample_cap, w->bins, w->out_pts,
                        w->out_mask, w->out_n, s));
  EXM_CUDA(cudaMemcpyAsync(w->h_out, w->out_pts, w->out_bytes, cudaMemcpyDeviceToHost, s));
  EXM_CUDA(cudaStreamSynchronize(s));
  const size_t b = static_cast<size_t>(w->budget);
  std::memcpy(pts_out, w->h_out, 2 * b * sizeof(double));
  std::memcpy(mask_out, w->h_out + 2 * b * sizeof(double), b);
  if (n_valid)
    *n_valid = *reinterpret_cast<const int*>(
        w->h_out + (reinterpret_cast<const unsigned char*>(w->out_n) -
                    reinterpret_cast<const unsigned char*>(w->out_pts)));
  return EXM_OK;
}

}  // namespace

extern "C" {

// sense(scenario, state, robot, sample_key) (world.cpp:182-243) for obstacles displaced by the
// given offsets: a transient world (geometry built on the host, no trails), one device launch.
exm_status exm_sense(exm_handle* h, const exm_world_obstacle* obstacles, int32_t n_obstacles,
                     const double robot[3], double range, int32_t budget, uint64_t seed,
                     uint64_t sample_key, double* pts_out, uint8_t* mask_out, int32_t* n_valid) {
  if (!h || !robot || !pts_out || !mask_out || (n_obstacles > 0 && !obstacles))
    return fail(EXM_ERR_INVALID_ARGUMENT, "null argument");
  if (budget < 1) return fail(EXM_ERR_INVALID_ARGUMENT, "sensor budget must be >= 1");
  std::lock_guard<std::mutex> lk(h->mu);
  WorldHost wh;
  exm_status st = build_world(obstacles, n_obstacles, nullptr, &wh);
  if (st != EXM_OK) return st;
  EXM_CUDA(cudaSetDevice(h->device));
  if ((st = world_reserve(h, wh, budget, &h->sense_ws)) != EXM_OK) return st;
  if ((st = world_upload(h->sense_ws, wh, range, seed)) != EXM_OK) return st;
  return world_sense(h->sense_ws, robot, sample_key, pts_out, mask_out, n_valid);
}

exm_status exm_world_create(exm_handle* h, const exm_world_obstacle* obstacles,
                            const exm_world_trail* trails, int32_t n_obstacles, double range,
                            int32_t budget, uint64_t seed, exm_world** out) {
  if (!out) return fail(EXM_ERR_INVALID_ARGUMENT, "out world pointer is null");
  *out = nullptr;
  if (!h || (n_obstacles > 0 && !obstacles)) return fail(EXM_ERR_INVALID_ARGUMENT, "null argument");
  if (budget < 1) return fail(EXM_ERR_INVALID_ARGUMENT, "sensor budget must be >= 1");
  std::lock_guard<std::mutex> lk(h->mu);
  WorldHost wh;
  exm_status st = build_world(obstacles, n_obstacles, trails, &wh);
  if (st != EXM_OK) return st;
  EXM_CUDA(cudaSetDevice(h->device));
  exm_world* w = nullptr;
  if ((st = world_reserve(h, wh, budget, &w)) != EXM_OK) return st;
  if ((st = world_upload(w, wh, range, seed)) != EXM_OK) {
    world_free(w);
    return st;
  }
  // offsets of the initial state (arc 0: the shapes sit at their first waypoint)
  if (const cudaError_t e = launch_world_step(w->trails, w->waypoints, w->n_obs, 1.0, 0, w->arc,
                                              w->dir, w->offsets, h->stream);
      e != cudaSuccess) {
    world_free(w);
    return fail(EXM_ERR_CUDA, std::string("world init: ") + cudaGetErrorString(e));
  }
  *out = w;
  return EXM_OK;
}

void exm_world_destroy(exm_world* w) {
  if (!w) return;
  std::lock_guard<std::mutex> lk(w->h->mu);
  cudaSetDevice(w->h->device);
  cudaStreamSynchronize(w->h->stream);
  world_free(w);
}

exm_status exm_world_step(exm_world* w, double dt) {
  if (!w) return fail(EXM_ERR_INVALID_ARGUMENT, "world is null");
  if (!(dt > 0.0)) return fail(EXM_ERR_INVALID_ARGUMENT, "step_world requires dt > 0");
  std::lock_guard<std::mutex> lk(w->h->mu);
  EXM_CUDA(cudaSetDevice(w->h->device));
  EXM_CUDA(launch_world_step(w->trails, w->waypoints, w->n_obs, dt, 1, w->arc, w->dir, w->offsets,
                             w->h->stream));
  return EXM_OK;
}

exm_status exm_world_sense(exm_world* w, const double robot[3], uint64_t sample_key,
                           double* pts_out, uint8_t* mask_out, int32_t* n_valid) {
  if (!w || !robot || !pts_out || !mask_out) return fail(EXM_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lk(w->h->mu);
  EXM_CUDA(cudaSetDevice(w->h->device));
  return world_sense(w, robot, sample_key, pts_out, mask_out, n_valid);
}

exm_status exm_world_state(exm_world* w, double* arc_out, int32_t* dir_out, double* offsets_out) {
  if (!w) return fail(EXM_ERR_INVALID_ARGUMENT, "world is null");
  std::lock_guard<std::mutex> lk(w->h->mu);
  EXM_CUDA(cudaSetDevice(w->h->device));
  cudaStream_t s = w->h->stream;
  const size_t n = static_cast<size_t>(w->n_obs);
  if (arc_out && n) EXM_CUDA(cudaMemcpyAsync(arc_out, w->arc, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (dir_out && n) EXM_CUDA(cudaMemcpyAsync(dir_out, w->dir, n * sizeof(int), cudaMemcpyDeviceToHost, s));
  if (offsets_out && n)
    EXM_CUDA(cudaMemcpyAsync(offsets_out, w->offsets, n * sizeof(double2), cudaMemcpyDeviceToHost, s));
  EXM_CUDA(cudaStreamSynchronize(s));
  return EXM_OK;
}

exm_status exm_set_sdf_caps(exm_handle* h, const float* caps) {
  if (!h || !caps) return fail(EXM_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  EXM_CUDA(cudaSetDevice(h->device));
  EXM_CUDA(cudaMemcpyAsync(h->d_cap, caps, sizeof(float) * h->T, cudaMemcpyHostToDevice, h->stream));
  EXM_CUDA(cudaStreamSynchronize(h->stream));
  return EXM_OK;
}

void* exm_host_alloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0 || cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void exm_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

exm_status exm_footprint_cull_boxes(const exm_footprint* fp, float* aabb_out, float* boxes_out,
                                    int32_t* n_out) {
  FpDev d;
  const exm_status st = build_footprint(fp, &d);
  if (st != EXM_OK) return st;
  if (aabb_out)
    for (int k = 0; k < 4; ++k) aabb_out[k] = d.aabb[k];
  if (boxes_out)
    for (int j = 0; j < kMaxCover; ++j)
      for (int k = 0; k < 4; ++k) boxes_out[4 * j + k] = d.cover[j][k];
  if (n_out) *n_out = d.ncover;
  return EXM_OK;
}

exm_status exm_sdf_work_stats(exm_handle* h, int64_t* counts) {
  if (!h || !counts) return fail(EXM_ERR_INVALID_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lk(h->mu);
  EXM_CUDA(cudaSetDevice(h->device));
  unsigned long long* d = nullptr;
  EXM_CUDA(dalloc(&d, kCntN));
  unsigned long long hv[kCntN] = {};
  cudaStream_t s = h->stream;
  cudaError_t e = cudaMemsetAsync(d, 0, kCntN * sizeof(unsigned long long), s);
  if (e == cudaSuccess)
    e = launch_sdf_grid(h->fp, h->d_poses, h->sc.k_local * h->T, h->T, h->hmajor, h->grid, h->d_cap,
                        h->sdf_mode, h->d_dmin, nullptr, d, s, rollout_threshold(h, false));
  if (e == cudaSuccess) e = cudaMemcpyAsync(hv, d, sizeof hv, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d);
  if (e != cudaSuccess) return fail(EXM_ERR_CUDA, std::string("cull stats: ") + cudaGetErrorString(e));
  for (int k = 0; k < kCntN; ++k) counts[k] = static_cast<int64_t>(hv[k]);
  return EXM_OK;
}

exm_status exm_sdf_cull_stats(exm_handle* h, int64_t* points_tested, int64_t* sdf_evaluated) {
  int64_t c[kCntN];
  const exm_status st = exm_sdf_work_stats(h, c);
  if (st != EXM_OK) return st;
  if (points_tested) *points_tested = c[kCntPoint];
  if (sdf_evaluated) *sdf_evaluated = c[kCntTileVal] + c[kCntEdges];
  return EXM_OK;
}

exm_status exm_set_option(exm_handle* h, int32_t option, int32_t value) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  EXM_CUDA(cudaSetDevice(h->device));
  EXM_CUDA(cudaStreamSynchronize(h->stream));
  switch (option) {
    case EXM_OPT_SDF_MODE:
      if (value < kSdfAuto || value > kSdfNoCap) return fail(EXM_ERR_INVALID_ARGUMENT, "unknown SDF mode");
      h->sdf_mode = value;
      break;
    case EXM_OPT_AUTO_CAPS: h->auto_caps = value != 0; break;
    case EXM_OPT_SDF_THRESHOLD: h->sdf_threshold = value != 0; break;
    case EXM_OPT_SDF_FP64: h->sdf_fp64 = value != 0; return EXM_OK;  // not in the step graphs
    case EXM_OPT_SDF_MAP:
      if (value < 0 || value > 2) return fail(EXM_ERR_INVALID_ARGUMENT, "unknown SDF mapping");
      h->sdf_map = value;
      h->hmajor = value == 2;
      h->tune_n = 0;
      h->tune_ms[0] = h->tune_ms[1] = 0.0;
      break;
    case EXM_OPT_PREGEN: h->pregen = value != 0; break;
    case EXM_OPT_HOST_TIMING:
      h->host_timing = value != 0;
      for (double& u : h->host_us) u = 0.0;
      h->host_calls = 0;
      return EXM_OK;
    case EXM_OPT_HOST_THREADS:
      if (value < 0 || value > 256) return fail(EXM_ERR_INVALID_ARGUMENT, "host threads out of range");
      h->host_threads = value;
      return EXM_OK;
    default: return fail(EXM_ERR_INVALID_ARGUMENT, "unknown option");
  }
  destroy_graphs(h);  // the captured steps depend on the options
  return invalidate_pregen(h);
}

exm_status exm_host_timing(exm_handle* h, double us_per_call[4], int64_t* calls) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  for (int i = 0; i < 4; ++i)
    if (us_per_call) us_per_call[i] = h->host_calls ? h->host_us[i] / h->host_calls : 0.0;
  if (calls) *calls = h->host_calls;
  return EXM_OK;
}

exm_status exm_last_sdf_path(exm_handle* h, exm_sdf_path* rollout, exm_sdf_path* validation) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  auto put = [](const SdfPath& p, exm_sdf_path* o) {
    if (!o) return;
    o->kernel = p.kernel;
    o->chunk = p.chunk;
    o->persistent = p.persistent;
    o->ctas = p.ctas;
    o->threads = p.threads;
    o->hmajor = p.hmajor;
  };
  put(h->roll_path, rollout);
  put(h->val_path, validation);
  return EXM_OK;
}

exm_status exm_step_stats(exm_handle* h, int32_t* launches_per_step, float* sdf_ms,
                          int64_t* sdf_pairs) {
  if (!h) return fail(EXM_ERR_INVALID_ARGUMENT, "handle is null");
  std::lock_guard<std::mutex> lk(h->mu);
  EXM_CUDA(cudaSetDevice(h->device));
  EXM_CUDA(cudaStreamSynchronize(h->stream));
  double total = h->ring_ms;
  int n = h->ring_n;
  for (int i = 0; i < h->ring_used; ++i) {
    float ms = 0.0f;
    EXM_CUDA(cudaEventElapsedTime(&ms, h->ring[i].a, h->ring[i].b));
    total += ms;
    ++n;
  }
  if (n == 0 && h->last_steps > 0) {
    float ms = 0.0f;
    EXM_CUDA(cudaEventElapsedTime(&ms, h->step_ev.a, h->step_ev.b));
    total = ms;
    n = 1;
  }
  if (launches_per_step) *launches_per_step = h->launches_per_step;
  if (sdf_ms) *sdf_ms = n ? static_cast<float>(total / n) : 0.0f;
  reset_timing(h, 0);  // consumed: the next run starts a fresh accumulation
  if (sdf_pairs) *sdf_pairs = h->last_pairs;
  return EXM_OK;
}

}  // extern "C"

// =========================================================================== hybrid families
struct exm_hybrid {
  std::mutex mu;  // calls on one hybrid handle serialise
  int M = 0, K = 0, T = 0, device = 0;
  std::vector<exm_handle*> fam;
  float4* poses_all = nullptr;  // [m][r][h]
  float* dmin_all = nullptr;
  cudaEvent_t fork = nullptr, prep_done = nullptr, sdf_done = nullptr;
  std::vector<cudaEvent_t> pre_done, fin;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
};

namespace {

// One graph: cloud prep (family 0) || per-family noise+rollout -> one SDF over all families'
// poses -> per-family post chains in parallel -> join.
exm_status hybrid_enqueue(exm_hybrid* hy, cudaStream_t s0) {
  exm_handle* f0 = hy->fam[0];
  exm_status st;
  int launches = 0;
  EXM_CUDA(cudaEventRecord(hy->fork, s0));
  EXM_CUDA(cudaStreamWaitEvent(f0->side, hy->fork, 0));
  if ((st = enqueue_prep(f0, f0->side)) != EXM_OK) return st;
  EXM_CUDA(cudaEventRecord(hy->prep_done, f0->side));
  for (int m = 0; m < hy->M; ++m) {
    cudaStream_t sm = m == 0 ? s0 : hy->fam[m]->stream;
    if (m) EXM_CUDA(cudaStreamWaitEvent(sm, hy->fork, 0));
    if ((st = enqueue_pre(hy->fam[m], true, sm, &launches)) != EXM_OK) return st;
    EXM_CUDA(cudaEventRecord(hy->pre_done[m], sm));
  }
  for (int m = 1; m < hy->M; ++m) EXM_CUDA(cudaStreamWaitEvent(s0, hy->pre_done[m], 0));
  EXM_CUDA(cudaStreamWaitEvent(s0, hy->prep_done, 0));
  float thr = 0.f;  // the loosest family threshold keeps every family's minima below its own exact
  for (int m = 0; m < hy->M; ++m) thr = std::max(thr, rollout_threshold(hy->fam[m], false));
  EXM_CUDA(launch_sdf_grid(f0->fp, hy->poses_all, hy->M * hy->K * hy->T, hy->T, f0->hmajor, f0->grid,
                           nullptr, f0->sdf_mode, hy->dmin_all, &f0->roll_path, nullptr, s0, thr));
  EXM_CUDA(cudaEventRecord(hy->sdf_done, s0));
  for (int m = 0; m < hy->M; ++m) {
    cudaStream_t sm = m == 0 ? s0 : hy->fam[m]->stream;
    if (m) EXM_CUDA(cudaStreamWaitEvent(sm, hy->sdf_done, 0));
    if ((st = enqueue_post(hy->fam[m], sm, &launches)) != EXM_OK) return st;
    EXM_CUDA(cudaEventRecord(hy->fin[m], sm));
  }
  for (int m = 1; m < hy->M; ++m) EXM_CUDA(cudaStreamWaitEvent(s0, hy->fin[m], 0));
  return EXM_OK;
}

}  // namespace

extern "C" {

void exm_hybrid_destroy(exm_hybrid* hy) {
  if (!hy) return;
  cudaSetDevice(hy->device);
  if (!hy->fam.empty() && hy->fam[0]) cudaStreamSynchronize(hy->fam[0]->stream);
  if (hy->exec) cudaGraphExecDestroy(hy->exec);
  if (hy->graph) cudaGraphDestroy(hy->graph);
  cudaEvent_t evs[] = {hy->fork, hy->prep_done, hy->sdf_done};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  for (auto e : hy->pre_done) cudaEventDestroy(e);
  for (auto e : hy->fin) cudaEventDestroy(e);
  for (exm_handle* h : hy->fam) exm_destroy(h);  // families free only what they own
  if (hy->poses_all) cudaFree(hy->poses_all);
  if (hy->dmin_all) cudaFree(hy->dmin_all);
  delete hy;
}

exm_status exm_hybrid_set_option(exm_hybrid* hy, int32_t option, int32_t value) {
  if (!hy) return fail(EXM_ERR_INVALID_ARGUMENT, "hybrid handle is null");
  std::lock_guard<std::mutex> lk(hy->mu);
  for (exm_handle* h : hy->fam)
    if (const exm_status st = exm_set_option(h, option, value); st != EXM_OK) return st;
  cudaSetDevice(hy->device);
  if (hy->exec) cudaGraphExecDestroy(hy->exec);  // the hybrid step graph is re-captured
  if (hy->graph) cudaGraphDestroy(hy->graph);
  hy->exec = nullptr;
  hy->graph = nullptr;
  return EXM_OK;
}

exm_status exm_hybrid_create(const exm_footprint* footprint, const exm_model* models,
                             const exm_limits* limits, int32_t n_modes,
                             const exm_params* params, int32_t n_cap, int32_t guide_cap,
                             int32_t device, exm_hybrid** out) {
  if (!out) return fail(EXM_ERR_INVALID_ARGUMENT, "out handle pointer is null");
  *out = nullptr;
  if (n_modes < 1 || !models || !limits || !params)
    return fail(EXM_ERR_INVALID_ARGUMENT, "hybrid: at least one active mode required");
  auto* hy = new exm_hybrid();
  hy->M = n_modes;
  hy->K = params->rollouts;
  hy->T = params->horizon;
  for (int m = 0; m < n_modes; ++m) {
    exm_params p = *params;
    p.seed = params->seed ^ (0x9E3779B97F4A7C15ull * static_cast<uint64_t>(m + 1));  // hybrid.cpp:89
    exm_handle* h = nullptr;
    exm_status st = exm_create(footprint, &models[m], &limits[m], &p, m == 0 ? n_cap : 0,
                               guide_cap, device, &h);
    if (st != EXM_OK) {
      exm_hybrid_destroy(hy);
      return st;
    }
    hy->fam.push_back(h);
  }
  exm_handle* f0 = hy->fam[0];
  hy->device = f0->device;
  auto bail = [&](exm_status s) {
    exm_hybrid_destroy(hy);
    return s;
  };
  const size_t KT = static_cast<size_t>(hy->K) * hy->T;
  cudaError_t ce;
  if ((ce = dalloc(&hy->poses_all, KT * n_modes)) != cudaSuccess ||
      (ce = dalloc(&hy->dmin_all, KT * n_modes)) != cudaSuccess)
    return bail(fail(EXM_ERR_CUDA, std::string("hybrid alloc: ") + cudaGetErrorString(ce)));
  for (int m = 0; m < n_modes; ++m) {
    exm_handle* h = hy->fam[m];
    cudaFree(h->d_poses);
    cudaFree(h->d_dmin);
    h->d_poses = hy->poses_all + m * KT;
    h->d_dmin = hy->dmin_all + m * KT;
    h->borrowed_poses = true;
    if (m > 0) {
      cudaFree(h->d_grid_block);
      h->d_grid_block = nullptr;
      h->grid = f0->grid;
      h->borrowed_cloud = true;
    }
  }
  cudaEvent_t* evs[] = {&hy->fork, &hy->prep_done, &hy->sdf_done};
  for (auto e : evs)
    if ((ce = cudaEventCreateWithFlags(e, cudaEventDisableTiming)) != cudaSuccess)
      return bail(fail(EXM_ERR_CUDA, cudaGetErrorString(ce)));
  hy->pre_done.resize(n_modes);
  hy->fin.resize(n_modes);
  for (int m = 0; m < n_modes; ++m) {
    cudaEventCreateWithFlags(&hy->pre_done[m], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&hy->fin[m], cudaEventDisableTiming);
  }
  *out = hy;
  return EXM_OK;
}

exm_status exm_hybrid_cycle(exm_hybrid* hy, const double q0[3], const double* pts_xy,
                            const uint8_t* mask, int32_t n_points, const double* guide_xy,
                            int32_t n_guide, const double goal[3], double* nominals_inout,
                            double* u_prev_inout, uint64_t cycle, exm_decision* out) {
  if (!hy) return fail(EXM_ERR_INVALID_ARGUMENT, "hybrid handle is null");
  if (!nominals_inout || !u_prev_inout) return fail(EXM_ERR_INVALID_ARGUMENT, "null state pointer");
  std::lock_guard<std::mutex> lk(hy->mu);
  EXM_CUDA(cudaSetDevice(hy->device));
  exm_handle* f0 = hy->fam[0];
  cudaStream_t s0 = f0->stream;
  const size_t stride = static_cast<size_t>(hy->T) * 3;
  for (int m = 0; m < hy->M; ++m) {
    exm_handle* h = hy->fam[m];
    // only family 0 prepares the cloud; the others upload just their state and the guidance
    exm_status st = upload_inputs(h, q0, m == 0 ? pts_xy : nullptr, m == 0 ? mask : nullptr,
                                  m == 0 ? n_points : 0, guide_xy, n_guide, goal,
                                  nominals_inout + m * stride, u_prev_inout + 3 * m, cycle);
    if (st != EXM_OK) return st;
    if (m) {  // family m's copies were issued on its own stream: order them before the graph
      EXM_CUDA(cudaEventRecord(hy->pre_done[m], h->stream));
      EXM_CUDA(cudaStreamWaitEvent(s0, hy->pre_done[m], 0));
    }
  }
  if (!hy->exec) {
    cudaGraph_t g = nullptr;
    EXM_CUDA(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal));
    exm_status st = hybrid_enqueue(hy, s0);
    cudaError_t ce = cudaStreamEndCapture(s0, &g);
    if (st != EXM_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (ce != cudaSuccess) return fail(EXM_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(ce));
    EXM_CUDA(cudaGraphInstantiate(&hy->exec, g, 0));
    hy->graph = g;
  }
  EXM_CUDA(cudaGraphLaunch(hy->exec, s0));
  for (int m = 0; m < hy->M; ++m)
    EXM_CUDA(cudaMemcpyAsync(hy->fam[m]->h_out, hy->fam[m]->d_out, hy->fam[m]->out_bytes,
                             cudaMemcpyDeviceToHost, s0));
  EXM_CUDA(cudaStreamSynchronize(s0));
  for (int m = 0; m < hy->M; ++m) {
    exm_handle* h = hy->fam[m];
    reset_timing(h, 1);
    unpack_decision(h, out ? out + m : nullptr, nominals_inout + m * stride, u_prev_inout + 3 * m);
  }
  return EXM_OK;
}

}  // extern "C"
