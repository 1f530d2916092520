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

constexpr double kSpacing = 0.05;  // kBoundarySpacing, world.cpp:15

// Boundary samples of segment g with its obstacle's offset (shape_boundary_samples,
// world.cpp:39-65): the displaced edge endpoints and the sample count the reference derives from
// them (max(1, ceil(|b - a| / 0.05)) per polygon edge, max(8, ceil(2 pi r / 0.05)) per disc).
__device__ __forceinline__ int segment_steps(const SenseSeg& g, double2 o) {
  if (g.kind == 0) {
    const double ax = __dadd_rn(g.ax, o.x), ay = __dadd_rn(g.ay, o.y);
    const double dx = __dsub_rn(__dadd_rn(g.bx, o.x), ax), dy = __dsub_rn(__dadd_rn(g.by, o.y), ay);
    const double len = sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
    return max(1, static_cast<int>(ceil(__ddiv_rn(len, kSpacing))));
  }
  const double circ = __dmul_rn(2.0 * kPi, g.r);
  return max(8, static_cast<int>(ceil(__ddiv_rn(circ, kSpacing))));
}

// Boundary sample s (global index over all obstacles, in the reference's loop order):
// seg_start[g] / seg_steps[g] from the kernel's prologue.
__device__ void sample_point(const SenseSeg* __restrict__ seg, const int* __restrict__ seg_start,
                             const int* __restrict__ seg_steps, const double2* __restrict__ off,
                             int nseg, int s, double& px, double& py) {
  int lo = 0, hi = nseg - 1;  // last segment with start <= s
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (seg_start[mid] <= s) lo = mid; else hi = mid - 1;
  }
  const SenseSeg& g = seg[lo];
  const double2 o = off[g.obs];
  const int k = s - seg_start[lo], steps = seg_steps[lo];
  if (g.kind == 0) {  // polygon edge a -> b (vertices + offset), t = k / steps
    const double ax = __dadd_rn(g.ax, o.x), ay = __dadd_rn(g.ay, o.y);
    const double bx = __dadd_rn(g.bx, o.x), by = __dadd_rn(g.by, o.y);
    const double t = __ddiv_rn(static_cast<double>(k), static_cast<double>(steps));
    px = __dadd_rn(ax, __dmul_rn(t, __dsub_rn(bx, ax)));
    py = __dadd_rn(ay, __dmul_rn(t, __dsub_rn(by, ay)));
  } else {  // disc: centre + offset + r (cos, sin)(2 pi k / steps)
    const double ang = __ddiv_rn(__dmul_rn(2.0 * kPi, static_cast<double>(k)),
                                 static_cast<double>(steps));
    double sn, cs;
    sincos(ang, &sn, &cs);
    px = __dadd_rn(__dadd_rn(g.ax, o.x), __dmul_rn(g.r, cs));
    py = __dadd_rn(__dadd_rn(g.ay, o.y), __dmul_rn(g.r, sn));
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

// Sensing in three launches: (1) one CTA forms the segment sample counts and starts from the
// current offsets and the nearest sample per bin (distances and bins kept from the first pass);
// (2) the exact line of sight of every (bin, obstacle) pair across the GPU; (3) one CTA builds the
// visible list, the seeded downsample and the padded output. BinState holds (1)'s result.
struct BinState {
  unsigned long long d[kOcclusionBins];  // nearest distance bits per bin (+inf: empty)
  int idx[kOcclusionBins];               // first sample at that distance
  int blocked[kOcclusionBins];           // line of sight blocked by some obstacle
};

__global__ void __launch_bounds__(kSenseThreads) k_sense_bins(
    const SenseSeg* __restrict__ seg, int nseg, const double2* __restrict__ off, double rx,
    double ry, double range, int* __restrict__ seg_start, double* __restrict__ dsc,
    int* __restrict__ bsc, int sample_cap, BinState* __restrict__ bins) {
  pdl_wait();
  __shared__ unsigned long long s_d[kOcclusionBins];
  __shared__ int s_idx[kOcclusionBins];
  __shared__ int s_warp[kSenseThreads / 32];
  __shared__ int s_total;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int* seg_steps = seg_start + nseg;
  for (int b = tid; b < kOcclusionBins; b += blockDim.x) {
    s_d[b] = 0x7ff0000000000000ull;  // +inf
    s_idx[b] = 0x7fffffff;
  }
  // sample counts per segment, then their exclusive scan (contiguous ranges per thread)
  for (int g = tid; g < nseg; g += blockDim.x) seg_steps[g] = segment_steps(seg[g], off[seg[g].obs]);
  __syncthreads();
  const int per = (nseg + blockDim.x - 1) / blockDim.x;
  const int g0 = min(nseg, tid * per), g1 = min(nseg, g0 + per);
  int local = 0;
  for (int g = g0; g < g1; ++g) local += seg_steps[g];
  int incl = local;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    const int v = lane < nw ? s_warp[lane] : 0;
    int sc = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(kFull, sc, o);
      if (lane >= o) sc += u;
    }
    if (lane < nw) s_warp[lane] = sc - v;
    if (lane == nw - 1) s_total = sc;
  }
  __syncthreads();
  int run = s_warp[warp] + incl - local;
  for (int g = g0; g < g1; ++g) {
    seg_start[g] = run;
    run += seg_steps[g];
  }
  const int n_samples = s_total;
  __syncthreads();
  // nearest boundary sample per bin: strict '<' in sample order = min distance, then min index
  for (int s = tid; s < n_samples; s += blockDim.x) {
    double px, py, d;
    sample_point(seg, seg_start, seg_steps, off, nseg, s, px, py);
    const int bin = sample_bin(px, py, rx, ry, range, d);
    if (s < sample_cap) {
      dsc[s] = d;
      bsc[s] = bin;
    }
    if (bin >= 0) atomicMin(&s_d[bin], static_cast<unsigned long long>(__double_as_longlong(d)));
  }
  __syncthreads();
  for (int s = tid; s < n_samples; s += blockDim.x) {
    double d;
    int bin;
    if (s < sample_cap) {
      d = dsc[s];
      bin = bsc[s];
    } else {
      double px, py;
      sample_point(seg, seg_start, seg_steps, off, nseg, s, px, py);
      bin = sample_bin(px, py, rx, ry, range, d);
    }
    if (bin >= 0 && static_cast<unsigned long long>(__double_as_longlong(d)) == s_d[bin])
      atomicMin(&s_idx[bin], s);
  }
  __syncthreads();
  for (int b = tid; b < kOcclusionBins; b += blockDim.x) {
    bins->d[b] = s_d[b];
    bins->idx[b] = s_idx[b];
    bins->blocked[b] = 0;
  }
}

// Exact line of sight (world.cpp:208-221), one thread per (bin, obstacle): the ray to the bin's
// sample, shortened by 1e-6 m, against the obstacle displaced by its offset.
constexpr int kLosThreads = 128;
__global__ void __launch_bounds__(kLosThreads) k_sense_los(
    const SenseSeg* __restrict__ seg, int nseg, const SenseObs* __restrict__ obs, int n_obs,
    const double2* __restrict__ verts, const double2* __restrict__ off, double rx, double ry,
    const int* __restrict__ seg_start, BinState* __restrict__ bins) {
  pdl_wait();
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= static_cast<int64_t>(kOcclusionBins) * n_obs) return;
  const int b = static_cast<int>(t % kOcclusionBins), i = static_cast<int>(t / kOcclusionBins);
  const int si = bins->idx[b];
  if (si == 0x7fffffff) return;
  double px, py;
  sample_point(seg, seg_start, seg_start + nseg, off, nseg, si, px, py);
  const double d = __longlong_as_double(static_cast<long long>(bins->d[b]));
  const double shrink = d > 1e-6 ? __ddiv_rn(__dsub_rn(d, 1e-6), d) : 0.0;
  const double tx = __dadd_rn(rx, __dmul_rn(shrink, __dsub_rn(px, rx)));
  const double ty = __dadd_rn(ry, __dmul_rn(shrink, __dsub_rn(py, ry)));
  const SenseObs& o = obs[i];
  const double2 oo = off[i];
  bool blocked = false;
  if (o.kind == 1) {
    blocked = point_segment_distance(__dadd_rn(o.cx, oo.x), __dadd_rn(o.cy, oo.y), rx, ry, tx,
                                     ty) < __dsub_rn(o.r, 1e-9);
  } else {
    for (int v = 0; v < o.count && !blocked; ++v) {
      const double2 a = verts[o.first + v];
      const double2 c = verts[o.first + (v + 1 == o.count ? 0 : v + 1)];
      blocked = segments_intersect(rx, ry, tx, ty, __dadd_rn(a.x, oo.x), __dadd_rn(a.y, oo.y),
                                   __dadd_rn(c.x, oo.x), __dadd_rn(c.y, oo.y));
    }
  }
  if (blocked) atomicOr(&bins->blocked[b], 1);
}

// Visible list in bin (scan) order, seeded partial Fisher-Yates when it exceeds the budget
// (world.cpp:224-239), padded ObstacleSet (geometry.cpp:148-159).
__global__ void __launch_bounds__(kSenseThreads) k_sense_out(
    const SenseSeg* __restrict__ seg, int nseg, const double2* __restrict__ off, int budget,
    uint64_t seed, uint64_t sample_key, const int* __restrict__ seg_start,
    const BinState* __restrict__ bins, double* __restrict__ pts_out, uint8_t* __restrict__ mask_out,
    int* __restrict__ n_out) {
  pdl_wait();
  __shared__ int s_vis[kOcclusionBins];  // visible-list position (-1: none)
  __shared__ int s_keep[kOcclusionBins];
  __shared__ int s_flag[kOcclusionBins];
  __shared__ int s_nkeep;
  const int tid = threadIdx.x;
  for (int b = tid; b < kOcclusionBins; b += blockDim.x)
    s_vis[b] = bins->idx[b] != 0x7fffffff && !bins->blocked[b];
  __syncthreads();
  if (tid == 0) {
    int n = 0;
    for (int b = 0; b < kOcclusionBins; ++b) s_vis[b] = s_vis[b] ? n++ : -1;
    int nk = n;
    if (n > budget) {
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
    int w = 0;  // output slot of every kept bin, in scan order
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
    sample_point(seg, seg_start, seg_start + nseg, off, nseg, bins->idx[b], px, py);
    pts_out[2 * w] = px;
    pts_out[2 * w + 1] = py;
    mask_out[w] = 1;
  }
  for (int i = nk + tid; i < budget; i += blockDim.x) {
    pts_out[2 * i] = 1e9;
    pts_out[2 * i + 1] = 1e9;
    mask_out[i] = 0;
  }
}

// step_world (world.cpp:127-157) and obstacle_offset (:159-164, trail_point :25-36), one thread
// per obstacle, FP64 in the reference's operation order.
__global__ void k_world_step(const TrailDev* __restrict__ trails, const double2* __restrict__ wp,
                             int n_obs, double dt, int advance, double* __restrict__ arc,
                             int* __restrict__ dir, double2* __restrict__ off) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_obs) return;
  const TrailDev t = trails[i];
  if (t.n < 2) {
    off[i] = make_double2(0.0, 0.0);
    return;
  }
  const double2* w = wp + t.first;
  auto seg_len = [&](int k) {
    const double dx = __dsub_rn(w[k + 1].x, w[k].x), dy = __dsub_rn(w[k + 1].y, w[k].y);
    return sqrt(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)));
  };
  double a = arc[i];
  if (advance && t.speed > 0.0) {
    double len = 0.0;
    for (int k = 0; k + 1 < t.n; ++k) len = __dadd_rn(len, seg_len(k));
    if (len > 0.0) {
      const double travel = __dmul_rn(t.speed, dt);
      int d = dir[i];
      if (t.ping_pong) {
        a = __dadd_rn(a, __dmul_rn(static_cast<double>(d), travel));
        while (a < 0.0 || a > len) {  // reflect until the arc lands inside [0, len]
          if (a > len) a = __dsub_rn(__dmul_rn(2.0, len), a);
          else a = -a;
          d = -d;
        }
      } else {
        a = clampd(__dadd_rn(a, __dmul_rn(static_cast<double>(d), travel)), 0.0, len);
      }
      arc[i] = a;
      dir[i] = d;
    }
  }
  // trail_point(a) - waypoints[0]
  double remaining = a;
  double2 at = w[0];
  for (int k = 0; k + 1 < t.n; ++k) {
    const double seg = seg_len(k);
    if (remaining <= seg || k + 2 == t.n) {
      const double tt = seg > 0.0 ? clampd(__ddiv_rn(remaining, seg), 0.0, 1.0) : 0.0;
      at = make_double2(__dadd_rn(w[k].x, __dmul_rn(tt, __dsub_rn(w[k + 1].x, w[k].x))),
                        __dadd_rn(w[k].y, __dmul_rn(tt, __dsub_rn(w[k + 1].y, w[k].y))));
      break;
    }
    remaining = __dsub_rn(remaining, seg);
  }
  off[i] = make_double2(__dsub_rn(at.x, w[0].x), __dsub_rn(at.y, w[0].y));
}

}  // namespace

cudaError_t launch_sense(const SenseSeg* seg, int nseg, const SenseObs* obs, int n_obs,
                         const double2* verts, const double2* offsets, double rx, double ry,
                         double range, int budget, uint64_t seed, uint64_t sample_key,
                         int* seg_scratch, double* d_scratch, int* bin_scratch, int sample_cap,
                         void* bin_state, double* pts_out, uint8_t* mask_out, int* n_out,
                         cudaStream_t s) {
  BinState* bins = static_cast<BinState*>(bin_state);
  if (const cudaError_t le = launch_k(k_sense_bins, 1, kSenseThreads, 0, s, seg, nseg, offsets, rx,
                                      ry, range, seg_scratch, d_scratch, bin_scratch, sample_cap,
                                      bins);
      le != cudaSuccess)
    return le;
  const int64_t pairs = static_cast<int64_t>(kOcclusionBins) * n_obs;
  if (pairs > 0)
    if (const cudaError_t le = launch_k(k_sense_los, static_cast<int>((pairs + kLosThreads - 1) / kLosThreads),
                                        kLosThreads, 0, s, seg, nseg, obs, n_obs, verts, offsets,
                                        rx, ry, static_cast<const int*>(seg_scratch), bins);
        le != cudaSuccess)
      return le;
  if (const cudaError_t le = launch_k(k_sense_out, 1, kSenseThreads, 0, s, seg, nseg, offsets,
                                      budget, seed, sample_key,
                                      static_cast<const int*>(seg_scratch),
                                      static_cast<const BinState*>(bins), pts_out, mask_out, n_out);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

size_t sense_bin_state_bytes() { return sizeof(BinState); }

cudaError_t launch_world_step(const TrailDev* trails, const double2* waypoints, int n_obs,
                              double dt, int advance, double* arc, int* dir, double2* offsets,
                              cudaStream_t s) {
  if (n_obs <= 0) return cudaSuccess;
  if (const cudaError_t le = launch_k(k_world_step, (n_obs + 127) / 128, 128, 0, s, trails,
                                      waypoints, n_obs, dt, advance, arc, dir, offsets);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

}  // namespace exm
