// exm_world.cu — sm_100a device port of the reference's sensing step (world.cpp:182-243,
// SURVEY §8(f2)): boundary samples of every (moved) obstacle, nearest sample per 720-bin
// angular sector, exact line-of-sight, seeded partial Fisher-Yates downsample to the sensor
// budget, padded ObstacleSet (geometry.cpp:148-159). The output is the cloud the control step
// consumes, produced on the device next to it.
//
// Compiled with -fmad=false like exm_dynamics.cu: every FP64 product and sum rounds where the
// reference's x86-64 build rounds it, so samples, distances, bins and visibility are the
// reference's up to the last-bit differences of CUDA's vs glibc's cos / sin / atan2.
#include "exm_device.cuh"

namespace exm {
namespace {

constexpr int kOcclusionBins = 720;  // world.cpp:16
constexpr int kSenseThreads = 1024;

// rng.hpp: uniform_index(seed, a, b, n)
__device__ __forceinline__ uint64_t uniform_index(uint64_t seed, uint64_t a, uint64_t b,
                                                  uint64_t n) {
  uint64_t k = splitmix64(seed);
  k = hash_mix(k, a);
  k = hash_mix(k, b);
  return n == 0 ? 0 : k % n;
}

__device__ __forceinline__ double cross2(double ax, double ay, double bx, double by) {
  return __dsub_rn(__dmul_rn(ax, by), __dmul_rn(ay, bx));
}
// geometry.cpp:29-54
__device__ __forceinline__ int orientation_sign(double ax, double ay, double bx, double by,
                                                double cx, double cy) {
  const double v = cross2(__dsub_rn(bx, ax), __dsub_rn(by, ay), __dsub_rn(cx, ax), __dsub_rn(cy, ay));
  return v > 0.0 ? 1 : (v < 0.0 ? -1 : 0);
}
__device__ __forceinline__ bool on_segment(double ax, double ay, double bx, double by, double px,
                                           double py) {
  return mn(ax, bx) <= px && px <= mx(ax, bx) && mn(ay, by) <= py && py <= mx(ay, by);
}
__device__ bool segments_intersect(double ax, double ay, double bx, double by, double cx,
                                   double cy, double dx, double dy) {
  const int o1 = orientation_sign(ax, ay, bx, by, cx, cy);
  const int o2 = orientation_sign(ax, ay, bx, by, dx, dy);
  const int o3 = orientation_sign(cx, cy, dx, dy, ax, ay);
  const int o4 = orientation_sign(cx, cy, dx, dy, bx, by);
  if (o1 != o2 && o3 != o4) return true;
  if (o1 == 0 && on_segment(ax, ay, bx, by, cx, cy)) return true;
  if (o2 == 0 && on_segment(ax, ay, bx, by, dx, dy)) return true;
  if (o3 == 0 && on_segment(cx, cy, dx, dy, ax, ay)) return true;
  if (o4 == 0 && on_segment(cx, cy, dx, dy, bx, by)) return true;
  return false;
}
// geometry.cpp:185-194
__device__ double point_segment_distance(double px, double py, double ax, double ay, double bx,
                                         double by) {
  const double ex = __dsub_rn(bx, ax), ey = __dsub_rn(by, ay);
  const double len2 = __dadd_rn(__dmul_rn(ex, ex), __dmul_rn(ey, ey));
  double t = 0.0;
  if (len2 > 0.0)
    t = clampd(__ddiv_rn(__dadd_rn(__dmul_rn(__dsub_rn(px, ax), ex), __dmul_rn(__dsub_rn(py, ay), ey)),
                         len2),
               0.0, 1.0);
  const double dx = __dsub_rn(px, __dadd_rn(ax, __dmul_rn(t, ex)));
  const double dy = __dsub_rn(py, __dadd_rn(ay, __dmul_rn(t, ey)));
  return sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
}

// Boundary sample s (global index over all obstacles, in the reference's loop order;
// shape_boundary_samples, world.cpp:39-65).
__device__ void sample_point(const SenseSeg* __restrict__ seg, int nseg, int s, double& px,
                             double& py) {
  int lo = 0, hi = nseg - 1;  // last segment with start <= s
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg[mid].start <= s) lo = mid; else hi = mid - 1;
  }
  const SenseSeg& g = seg[lo];
  const int k = s - g.start;
  if (g.kind == 0) {  // polygon edge a -> b (vertices + offset), t = k / steps
    const double t = __ddiv_rn(static_cast<double>(k), static_cast<double>(g.steps));
    px = __dadd_rn(g.ax, __dmul_rn(t, __dsub_rn(g.bx, g.ax)));
    py = __dadd_rn(g.ay, __dmul_rn(t, __dsub_rn(g.by, g.ay)));
  } else {  // disc: centre + offset + r (cos, sin)(2 pi k / steps)
    const double ang = __ddiv_rn(__dmul_rn(2.0 * kPi, static_cast<double>(k)),
                                 static_cast<double>(g.steps));
    double sn, cs;
    sincos(ang, &sn, &cs);
    px = __dadd_rn(__dadd_rn(g.ax, g.bx), __dmul_rn(g.r, cs));
    py = __dadd_rn(__dadd_rn(g.ay, g.by), __dmul_rn(g.r, sn));
  }
}

// Distance and occlusion bin of a sample seen from the robot (world.cpp:193-200); -1: beyond
// the sensor range.
__device__ __forceinline__ int sample_bin(double px, double py, double rx, double ry,
                                          double range, double& d) {
  const double dx = __dsub_rn(px, rx), dy = __dsub_rn(py, ry);
  d = sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
  if (d > range) return -1;
  const double ang = atan2(dy, dx);
  const int bin = static_cast<int>(
      __dmul_rn(__ddiv_rn(__dadd_rn(ang, kPi), 2.0 * kPi), static_cast<double>(kOcclusionBins)));
  return min(max(bin, 0), kOcclusionBins - 1);
}

// The whole sensing step in one CTA (S samples, 720 bins, obstacles in shared memory).
__global__ void __launch_bounds__(kSenseThreads) k_sense(
    const SenseSeg* __restrict__ seg, int nseg, int n_samples,
    const SenseObs* __restrict__ obs, int n_obs, const double2* __restrict__ verts,
    double rx, double ry, double range, int budget, uint64_t seed, uint64_t sample_key,
    double* __restrict__ pts_out, uint8_t* __restrict__ mask_out, int* __restrict__ n_out) {
  pdl_wait();
  __shared__ unsigned long long s_d[kOcclusionBins];  // nearest distance bits per bin
  __shared__ int s_idx[kOcclusionBins];               // first sample at that distance
  __shared__ int s_vis[kOcclusionBins];               // visible-list position (-1: none)
  __shared__ int s_keep[kOcclusionBins];
  __shared__ int s_flag[kOcclusionBins];
  __shared__ int s_nkeep;
  const int tid = threadIdx.x;
  for (int b = tid; b < kOcclusionBins; b += blockDim.x) {
    s_d[b] = 0x7ff0000000000000ull;  // +inf
    s_idx[b] = 0x7fffffff;
  }
  __syncthreads();
  // nearest boundary sample per bin: strict '<' in sample order = min distance, then min index
  for (int s = tid; s < n_samples; s += blockDim.x) {
    double px, py, d;
    sample_point(seg, nseg, s, px, py);
    const int bin = sample_bin(px, py, rx, ry, range, d);
    if (bin >= 0) atomicMin(&s_d[bin], static_cast<unsigned long long>(__double_as_longlong(d)));
  }
  __syncthreads();
  for (int s = tid; s < n_samples; s += blockDim.x) {
    double px, py, d;
    sample_point(seg, nseg, s, px, py);
    const int bin = sample_bin(px, py, rx, ry, range, d);
    if (bin >= 0 && static_cast<unsigned long long>(__double_as_longlong(d)) == s_d[bin])
      atomicMin(&s_idx[bin], s);
  }
  __syncthreads();
  // exact line of sight (world.cpp:208-221): the ray to the sample, shortened by 1e-6 m
  for (int b = tid; b < kOcclusionBins; b += blockDim.x) {
    int vis = 0;
    if (s_idx[b] != 0x7fffffff) {
      double px, py;
      sample_point(seg, nseg, s_idx[b], px, py);
      const double d = __longlong_as_double(static_cast<long long>(s_d[b]));
      const double shrink = d > 1e-6 ? __ddiv_rn(__dsub_rn(d, 1e-6), d) : 0.0;
      const double tx = __dadd_rn(rx, __dmul_rn(shrink, __dsub_rn(px, rx)));
      const double ty = __dadd_rn(ry, __dmul_rn(shrink, __dsub_rn(py, ry)));
      bool blocked = false;
      for (int i = 0; i < n_obs && !blocked; ++i) {
        const SenseObs& o = obs[i];
        if (o.kind == 1) {
          blocked = point_segment_distance(__dadd_rn(o.cx, o.ox), __dadd_rn(o.cy, o.oy), rx, ry,
                                           tx, ty) < __dsub_rn(o.r, 1e-9);
        } else {
          for (int v = 0; v < o.count && !blocked; ++v) {
            const double2 a = verts[o.first + v];
            const double2 c = verts[o.first + (v + 1 == o.count ? 0 : v + 1)];
            blocked = segments_intersect(rx, ry, tx, ty, __dadd_rn(a.x, o.ox), __dadd_rn(a.y, o.oy),
                                         __dadd_rn(c.x, o.ox), __dadd_rn(c.y, o.oy));
          }
        }
      }
      vis = blocked ? 0 : 1;
    }
    s_vis[b] = vis;
  }
  __syncthreads();
  if (tid == 0) {  // visible list in bin (scan) order
    int n = 0;
    for (int b = 0; b < kOcclusionBins; ++b) s_vis[b] = s_vis[b] ? n++ : -1;
    int nk = n;
    if (n > budget) {
      // seeded partial Fisher-Yates over the visible list, then scan order (world.cpp:224-239)
      int* idx = s_keep;
      for (int i = 0; i < n; ++i) idx[i] = i;
      for (int i = 0; i < budget; ++i) {
        const int j = i + static_cast<int>(uniform_index(seed, sample_key, static_cast<uint64_t>(i),
                                                         static_cast<uint64_t>(n - i)));
        const int t = idx[i];
        idx[i] = idx[j];
        idx[j] = t;
      }
      for (int i = 0; i < n; ++i) s_flag[i] = 0;
      for (int i = 0; i < budget; ++i) s_flag[idx[i]] = 1;
      nk = budget;
    } else {
      for (int i = 0; i < n; ++i) s_flag[i] = 1;
    }
    // output slot of every kept bin, in scan order
    int w = 0;
    for (int b = 0; b < kOcclusionBins; ++b) {
      const int p = s_vis[b];
      s_vis[b] = (p >= 0 && s_flag[p]) ? w++ : -1;
    }
    s_nkeep = nk;
    *n_out = w;
  }
  __syncthreads();
  const int nk = s_nkeep;
  for (int b = tid; b < kOcclusionBins; b += blockDim.x) {
    const int w = s_vis[b];
    if (w < 0) continue;
    double px, py;
    sample_point(seg, nseg, s_idx[b], px, py);
    pts_out[2 * w] = px;
    pts_out[2 * w + 1] = py;
    mask_out[w] = 1;
  }
  for (int i = nk + tid; i < budget; i += blockDim.x) {  // ObstacleSet::padded, geometry.cpp:148-159
    pts_out[2 * i] = 1e9;
    pts_out[2 * i + 1] = 1e9;
    mask_out[i] = 0;
  }
}

}  // namespace

cudaError_t launch_sense(const SenseSeg* seg, int nseg, int n_samples, const SenseObs* obs,
                         int n_obs, const double2* verts, double rx, double ry, double range,
                         int budget, uint64_t seed, uint64_t sample_key, double* pts_out,
                         uint8_t* mask_out, int* n_out, cudaStream_t s) {
  if (const cudaError_t le = launch_k(k_sense, 1, kSenseThreads, 0, s, seg, nseg, n_samples, obs,
                                      n_obs, verts, rx, ry, range, budget, seed, sample_key,
                                      pts_out, mask_out, n_out);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

}  // namespace exm
