// exm_exact64.cu — FP64 per-pose signed-distance minima for exm_evaluate_rollouts under
// EXM_OPT_SDF_FP64: the reference's min_signed_distance_at (geometry.cpp:357-375) over
// PreparedFootprint::sd (geometry.cpp:260-295), one thread per pose, every point visited in
// cloud order with the reference's own radius skip. Compiled with -fmad=false like
// exm_dynamics.cu: every product and sum rounds where the reference's x86-64 build rounds it,
// so the minima equal the reference's up to the last-bit differences of CUDA's vs glibc's
// cos / sin of the heading. This is the opt-in path for callers that need the reference's
// 1e-9 batch-vs-scalar agreement (acceptance_main.cpp:260-300); the control cycle keeps the
// FP32 culled kernels (north-star tolerance 1e-5).
#include "exm_device.cuh"
#include "exm_exact64.cuh"

namespace exm {
namespace {

constexpr int kExactThreads = 128;

// PreparedFootprint::sd (geometry.cpp:260-295)
__device__ double sd64(const FpDev64& fp, double px, double py) {
  if (fp.kind == EXM_FOOTPRINT_RECT_COVER) {
    double d = HUGE_VAL;
    for (int j = 0; j < fp.count; ++j) {
      const double ax = fabs(px - fp.v[j][0]) - fp.v[j][2];
      const double ay = fabs(py - fp.v[j][1]) - fp.v[j][3];
      const double ox = ax > 0.0 ? ax : 0.0;
      const double oy = ay > 0.0 ? ay : 0.0;
      const double inner = ax < ay ? ay : ax;  // std::max(ax, ay)
      d = mn(d, sqrt(ox * ox + oy * oy) + (inner < 0.0 ? inner : 0.0));
    }
    return d;
  }
  double d2 = HUGE_VAL;
  bool inside = false;
  for (int b = 0; b < fp.count; ++b) {
    const double* e = fp.v[b];
    const double rx = px - e[0];
    const double ry = py - e[1];
    double t = (rx * e[2] + ry * e[3]) * e[4];
    t = t < 0.0 ? 0.0 : (t > 1.0 ? 1.0 : t);
    const double dx = rx - t * e[2];
    const double dy = ry - t * e[3];
    const double dist2 = dx * dx + dy * dy;
    if (dist2 < d2) d2 = dist2;
    const double ay = e[1];
    const double by = e[1] + e[3];
    if ((ay < py) != (by < py)) {
      const double x_cross = e[0] + (py - ay) * e[2] / e[3];
      if (x_cross > px) inside = !inside;
    }
  }
  const double d = sqrt(d2);
  if (d < 1e-12) return 0.0;  // kBoundaryEpsilon (geometry.hpp:39)
  return inside ? -d : d;
}

__global__ void __launch_bounds__(kExactThreads) k_sdf_exact64(
    const __grid_constant__ FpDev64 fp, const double* __restrict__ states, int K, int T,
    const double2* __restrict__ pts, const uint8_t* __restrict__ mask, int n,
    double* __restrict__ out) {
  pdl_wait();
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long long>(K) * T) return;
  const int r = static_cast<int>(i / T), h = static_cast<int>(i % T);
  const double* q = states + (static_cast<size_t>(r) * (T + 1) + h) * 3;
  const double qx = q[0], qy = q[1];
  double s, c;
  sincos(q[2], &s, &c);
  const double empty = 1e6;  // kEmptyMaskDistance (geometry.hpp:37)
  double best = empty;
  bool any = false;
  for (int j = 0; j < n; ++j) {
    if (mask && !mask[j]) continue;
    const double2 p = pts[j];
    const double dx = p.x - qx;
    const double dy = p.y - qy;
    const double thr = fp.radius + (any ? best : empty);
    if (any && thr > 0.0 && dx * dx + dy * dy >= thr * thr) continue;
    const double d = sd64(fp, c * dx + s * dy, -s * dx + c * dy);
    if (!any || d < best) best = d;
    any = true;
  }
  out[i] = any ? best : empty;
}

__global__ void __launch_bounds__(kExactThreads) k_sdf_points64(const __grid_constant__ FpDev64 fp,
                                                                const double2* __restrict__ q,
                                                                int n, double* __restrict__ out) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 p = q[i];
  out[i] = sd64(fp, p.x, p.y);
}

}  // namespace

cudaError_t launch_sdf_points64(const FpDev64& fp, const double* q, int n, double* out,
                                cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (const cudaError_t le = launch_k(k_sdf_points64, (n + kExactThreads - 1) / kExactThreads,
                                      kExactThreads, 0, s, fp, reinterpret_cast<const double2*>(q),
                                      n, out);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

cudaError_t launch_sdf_exact64(const FpDev64& fp, const double* states, int K, int T,
                               const double* pts, const uint8_t* mask, int n, double* out,
                               cudaStream_t s) {
  const long long np = static_cast<long long>(K) * T;
  if (np <= 0) return cudaSuccess;
  const int grid = static_cast<int>((np + kExactThreads - 1) / kExactThreads);
  if (const cudaError_t le = launch_k(k_sdf_exact64, grid, kExactThreads, 0, s, fp, states, K, T,
                                      reinterpret_cast<const double2*>(pts), mask, n, out);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

}  // namespace exm
