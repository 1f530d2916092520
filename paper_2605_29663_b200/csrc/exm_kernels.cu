// exm_kernels.cu — sm_100a kernels of the cloud preparation and the exact signed distance.
//
// Kernel map (reference function each one replaces, proj/...):
//   k_cloud_prep     ObstacleSet masking, recentring at q0,  geometry.cpp:357-375 (mask, layout)
//                    uniform-grid binning for exact culling
//   k_cell_sort      in-cell Morton order, chunk boxes       (cull structure, no counterpart)
//   k_sdf_grid       min_signed_distance_at over K*T poses   geometry.cpp:357-375, :260-296
//   k_sdf_grid_warp  the same, one warp per pose (few poses)
//   k_sdf_pairs      batch_signed_distance (every pair)      geometry.cpp:298-318
// The FP64 dynamics / cost / softmax kernels are in exm_dynamics.cu.
//
// Numerics: the signed distance inner loops are FP32 on coordinates recentred at q0 in FP64
// before rounding.
#include <algorithm>

#include "exm_device.cuh"

// The (footprint kind, edge count) instantiations of the signed-distance kernels are split over
// EXM_NPARTS translation units compiled in parallel from this file (build.py: -DEXM_PART=k
// -DEXM_NPARTS=P); part 0 also holds every non-templated kernel and the exported launchers,
// which route each footprint to the part that instantiated it. Without the macros: one unit.
#ifndef EXM_NPARTS
#define EXM_NPARTS 1
#endif
#ifndef EXM_PART
#define EXM_PART 0
#endif
#if EXM_NPARTS < 1 || EXM_NPARTS > 4 || EXM_PART < 0 || EXM_PART >= EXM_NPARTS
#error "EXM_PART / EXM_NPARTS out of range (at most 4 parts)"
#endif

#if defined(EXM_TIMING) && EXM_PART == 0  // phase timestamps of k_cloud_prep (diagnostic builds only)
__device__ long long g_probe_prep[16];
#define EXM_PROBE_P(i) \
  do {                 \
    if (threadIdx.x == 0) g_probe_prep[i] = clock64(); \
  } while (0)
extern "C" int exm_debug_probes_prep(long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_probe_prep, sizeof(g_probe_prep)));
}
#else
#define EXM_PROBE_P(i) \
  do {                 \
  } while (0)
#endif

namespace exm {
namespace {

// ---- TMA bulk copy (cp.async.bulk global -> shared, mbarrier completion) -------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, unsigned bytes,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ---- packed FP32x2 (sm_100 FFMA2/FADD2/FMUL2) helpers ---------------------------------
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo(u64 v) {
  return __uint_as_float(static_cast<unsigned>(v));
}
__device__ __forceinline__ float hi(u64 v) {
  return __uint_as_float(static_cast<unsigned>(v >> 32));
}
__device__ __forceinline__ u64 bc(float x) { return pk(x, x); }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ u64 mul2(u64 a, u64 b) {
  u64 r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ u64 sub2(u64 a, u64 b) {
  u64 r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned sgn_lo(u64 v) { return __float_as_uint(lo(v)); }
__device__ __forceinline__ unsigned sgn_hi(u64 v) { return __float_as_uint(hi(v)); }

__device__ __forceinline__ float min3f(float a, float b, float c) {
  float r;
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));  // FMNMX3
  return r;
}

// Cover-box loops run over fp.ncover boxes (uniform: the footprint table is a kernel parameter;
// the L takes 2 of the kMaxCover slots). -DEXM_COVER_ALL_SLOTS: all slots, unused ones repeating
// box 0 (round 1; A/B builds).
__device__ __forceinline__ bool cover_slot(const FpDev& fp, int j) {
#ifdef EXM_COVER_ALL_SLOTS
  return true;
#else
  return j == 0 || j < fp.ncover;
#endif
}

// ------------------------------------------------------------------ FP32 signed distance
// Polygon edge step (PreparedFootprint::sd polygon branch, geometry.cpp:273-292).
//   t  = sat(p.e/|e|^2 - v.e/|e|^2)           2 FFMA (second .SAT)
//   q  = v + t e - p;  d2 = |q|^2              2 FADD, 2 FFMA, FMUL, FFMA
//   crossing, division-free: with r = v - p, edge b counts iff (vy_b < py) != (vy_b+1 < py)
//   and x_cross - px = cross(v - p, e)/ey > 0, i.e. in sign bits
//   count = (sb(ry_b) ^ sb(ry_b+1)) & (sb(ry_b) ^ sb(rx ey - ry ex)).
//   Vertex signs are shared by the two edges that meet there, so the straddle count over a
//   closed polygon is always even (parity exact outside the footprint's y-range).
__device__ __forceinline__ void poly_edge(const float* e, float px, float py, float& ry,
                                          float ry_next, float& best2, unsigned& par) {
  const float t = __saturatef(fmaf(px, e[4], fmaf(py, e[5], e[6])));
  const float rx = e[0] - px;
  const float qx = fmaf(t, e[2], rx), qy = fmaf(t, e[3], ry);
  best2 = fminf(best2, fmaf(qx, qx, qy * qy));
  const float cr = fmaf(ry, e[7], rx * e[3]);  // e[7] = -ex
  par ^= (__float_as_uint(ry) ^ __float_as_uint(ry_next)) & (__float_as_uint(ry) ^ __float_as_uint(cr));
  ry = ry_next;
}

// The same polygon SDF with two edges per f32x2 operation (FFMA2/FADD2/FMUL2): edge pair j
// is fp.ep[j] (field k of edges 2j, 2j+1 adjacent; an odd count is padded with a zero-length
// edge at vertex 0, which neither straddles nor changes the minimum). Every lane performs the
// scalar poly_edge arithmetic in the same order, so the result is bit-identical.
__device__ __forceinline__ u64 ldp(const float (&a)[2]) { return *reinterpret_cast<const u64*>(a); }

template <int NB>
__device__ __forceinline__ float sd_polygon_x2(const FpDev& fp, float px, float py) {
  constexpr int NP = (NB + 1) / 2;
  const u64 PX = bc(px), PY = bc(py);
  const u64 RY0 = sub2(ldp(fp.ep[0][1]), PY);
  u64 RY = RY0;
  float best2 = __int_as_float(0x7f800000);
  unsigned par = 0u;
#pragma unroll
  for (int j = 0; j < NP; ++j) {
    const u64 RYn = j + 1 < NP ? sub2(ldp(fp.ep[j + 1][1]), PY) : RY0;
    const u64 TP = fma2(PY, ldp(fp.ep[j][5]), ldp(fp.ep[j][6]));
    const u64 T = pk(__saturatef(fmaf(px, fp.ep[j][4][0], lo(TP))),
                     __saturatef(fmaf(px, fp.ep[j][4][1], hi(TP))));
    const u64 RX = sub2(ldp(fp.ep[j][0]), PX);
    const u64 QX = fma2(T, ldp(fp.ep[j][2]), RX);
    const u64 QY = fma2(T, ldp(fp.ep[j][3]), RY);
    const u64 D2 = fma2(QX, QX, mul2(QY, QY));
    best2 = min3f(best2, lo(D2), hi(D2));
    const u64 CR = fma2(RY, ldp(fp.ep[j][7]), mul2(RX, ldp(fp.ep[j][3])));
    const unsigned a0 = sgn_lo(RY), a1 = sgn_hi(RY), a2 = sgn_lo(RYn);
    par ^= ((a0 ^ a1) & (a0 ^ sgn_lo(CR))) ^ ((a1 ^ a2) & (a1 ^ sgn_hi(CR)));
    RY = RYn;
  }
  if (best2 < 1e-24f) return 0.0f;  // kBoundaryEpsilon rule (d < 1e-12 -> 0)
  const float d = sqrtf(best2);
  return (par >> 31) ? -d : d;
}

template <int NB>
__device__ __forceinline__ float sd_polygon(const FpDev& fp, float px, float py) {
  float best2 = __int_as_float(0x7f800000);
  unsigned par = 0u;
  const float ry0 = fp.e[0][1] - py;
  float ry = ry0;
  if constexpr (NB > 0) {
#pragma unroll
    for (int b = 0; b < NB; ++b)
      poly_edge(fp.e[b], px, py, ry, b + 1 < NB ? fp.e[b + 1][1] - py : ry0, best2, par);
  } else {
    const int n = fp.count;
#pragma unroll 4
    for (int b = 0; b < n; ++b)
      poly_edge(fp.e[b], px, py, ry, b + 1 < n ? fp.e[b + 1][1] - py : ry0, best2, par);
  }
  if (best2 < 1e-24f) return 0.0f;  // kBoundaryEpsilon rule (d < 1e-12 -> 0)
  const float d = sqrtf(best2);
  return (par >> 31) ? -d : d;
}

// Rectangle cover (geometry.cpp:261-272): min_j [sqrt(|max(a,0)|^2) + min(max(ax,ay),0)]
// == (min_j max(ax,ay) <= 0) ? min_j max(ax,ay) : sqrt(min_j |max(a,0)|^2)  (sqrt monotone).
__device__ __forceinline__ void rect_box(const float* e, float px, float py, float& m_in,
                                         float& m_e2) {
  const float ax = fabsf(px - e[0]) - e[2];
  const float ay = fabsf(py - e[1]) - e[3];
  const float ox = fmaxf(ax, 0.0f), oy = fmaxf(ay, 0.0f);
  m_e2 = fminf(m_e2, fmaf(ox, ox, oy * oy));
  m_in = fminf(m_in, fmaxf(ax, ay));
}

template <int NB>
__device__ __forceinline__ float sd_rect(const FpDev& fp, float px, float py) {
  float m_in = __int_as_float(0x7f800000), m_e2 = __int_as_float(0x7f800000);
  if constexpr (NB > 0) {
#pragma unroll
    for (int j = 0; j < NB; ++j) rect_box(fp.e[j], px, py, m_in, m_e2);
  } else {
#pragma unroll 2
    for (int j = 0; j < fp.count; ++j) rect_box(fp.e[j], px, py, m_in, m_e2);
  }
  return m_in <= 0.0f ? m_in : sqrtf(m_e2);
}

template <int KIND, int NB>
__device__ __forceinline__ float sd_body(const FpDev& fp, float px, float py) {
  if constexpr (KIND == EXM_FOOTPRINT_POLYGON && NB > 0) return sd_polygon_x2<NB>(fp, px, py);
  else if constexpr (KIND == EXM_FOOTPRINT_POLYGON) return sd_polygon<NB>(fp, px, py);
  else return sd_rect<NB>(fp, px, py);
}

// Exact second-level cull on the body-frame point: the footprint lies inside its AABB, so an
// exterior point's signed distance is at least its distance to the AABB. Points inside the
// AABB (distance 0) may be inside the footprint and are always evaluated.
// Interior bound (p inside the AABB): the footprint lies inside its AABB, so p is no deeper
// in the footprint than in the AABB: sd(p) >= max(xmin - x, x - xmax, ymin - y, y - ymax).
// Culls interior points once a negative minimum is known (footprint overlapping obstacles).
__device__ __forceinline__ bool aabb_may_beat(const FpDev& fp, float bx, float by, float best,
                                              float mg) {
  const float dx = fmaxf(fp.aabb[0] - bx, bx - fp.aabb[1]);
  const float dy = fmaxf(fp.aabb[2] - by, by - fp.aabb[3]);
  const float ax = fmaxf(dx, 0.f), ay = fmaxf(dy, 0.f);
  const float a2 = fmaf(ax, ax, ay * ay);
  const float lim = best + mg;
  return a2 == 0.f ? fmaxf(dx, dy) < lim : (lim > 0.f && a2 < lim * lim);
}

// Polygon cover bound: the union of the kMaxCover cover boxes (unused slots repeat box 0)
// contains the polygon, so an exterior point's signed distance is at least its distance to the
// nearest box (0 inside a box: evaluate). Subsumes the AABB bound.
__device__ __forceinline__ bool cover_may_beat(const FpDev& fp, float bx, float by, float best,
                                               float mg) {
  float d2 = __int_as_float(0x7f800000);
#pragma unroll
  for (int j = 0; j < kMaxCover; ++j) {
    if (!cover_slot(fp, j)) break;
    const float ax = fmaxf(fabsf(bx - fp.cover[j][0]) - fp.cover[j][2], 0.f);
    const float ay = fmaxf(fabsf(by - fp.cover[j][1]) - fp.cover[j][3], 0.f);
    d2 = fminf(d2, fmaf(ax, ax, ay * ay));
  }
  const float lim = best + mg;
  if (d2 == 0.f)  // inside the cover: the AABB interior bound (aabb_may_beat)
    return fmaxf(fmaxf(fp.aabb[0] - bx, bx - fp.aabb[1]), fmaxf(fp.aabb[2] - by, by - fp.aabb[3])) < lim;
  return lim > 0.f && d2 < lim * lim;
}

// Exact-cover polygons (fp.cover_exact: rectilinear footprints tiled by their <= 3 cover boxes,
// the L): a point outside the slackened cover (every box: max(|b - c| - h) > slack, so it is
// exterior with a margin far above FP32 rounding) has signed distance = distance to the union
// of the unslackened tiles; returns that squared distance. Other points (inside or within the
// slack of the footprint) take the edge loop. Value function of the grid kernels:
//   v(p) = exterior ? sqrt(d2_tiles) : sd_polygon(p)
// (differs from the edge loop by FP32 rounding only; culled and brute-force modes share it).
__device__ __forceinline__ bool tiles_exterior_d2(const FpDev& fp, float bx, float by, float& d2) {
  float d2u = __int_as_float(0x7f800000), inm = __int_as_float(0x7f800000);
#pragma unroll
  for (int j = 0; j < kMaxCover; ++j) {
    if (!cover_slot(fp, j)) break;
    const float ax = fabsf(bx - fp.cbox[j][0]) - fp.cbox[j][2];
    const float ay = fabsf(by - fp.cbox[j][1]) - fp.cbox[j][3];
    const float ox = fmaxf(ax, 0.f), oy = fmaxf(ay, 0.f);
    d2u = fminf(d2u, fmaf(ox, ox, oy * oy));
    inm = fminf(inm, fmaxf(ax, ay));
  }
  d2 = d2u;
  return inm > fp.cover_slack;
}

// One body-frame candidate point of the grid kernels: lower-bound tests, then the value v(p);
// returns the new running minimum. BRUTE: no bound at all (every point valued, same arithmetic).
// `work` reports what ran (statistics builds charge each at its op count): kWorkTile (the
// exact-cover tile test), kWorkTileVal (tile distance taken), kWorkBound (cover / AABB bound
// test), kWorkEdges (edge loop / rectangle-cover SDF).
constexpr unsigned kWorkTile = 1u, kWorkTileVal = 2u, kWorkBound = 4u, kWorkEdges = 8u;
template <int KIND, int NB, bool BRUTE>
__device__ __forceinline__ float grid_point(const FpDev& fp, float bx, float by, float best,
                                            float mg, unsigned& work) {
  work = 0u;
  if constexpr (KIND == EXM_FOOTPRINT_POLYGON) {
    if (fp.cover_exact) {
      float d2;
      const float lim = best + mg;
      work = kWorkTile;
      if (tiles_exterior_d2(fp, bx, by, d2)) {
        if (BRUTE || (lim > 0.f && d2 < lim * lim)) {
          work |= kWorkTileVal;
          best = fminf(best, sqrtf(d2));
        }
        return best;
      }
      // inside (or at the rim of) the cover: the AABB interior bound, then the edge loop
      if (!BRUTE) work |= kWorkBound;
      if (BRUTE || fmaxf(fmaxf(fp.aabb[0] - bx, bx - fp.aabb[1]), fmaxf(fp.aabb[2] - by, by - fp.aabb[3])) < lim) {
        work |= kWorkEdges;
        best = fminf(best, sd_body<KIND, NB>(fp, bx, by));
      }
      return best;
    }
  }
  // polygons: the cover bound (exact for rectilinear shapes: the L's notch is culled);
  // rectangle covers of <= 3 boxes: the exact SDF is hardly dearer than a bound (skipping its
  // sqrt behind a squared-distance test measured slower: the branch diverges); larger
  // covers: the AABB pre-test
  constexpr bool kDirect = KIND != EXM_FOOTPRINT_POLYGON && NB > 0 && NB <= 3;
  if (!BRUTE && !kDirect) work = kWorkBound;
  if (BRUTE || kDirect ||
      (KIND == EXM_FOOTPRINT_POLYGON ? cover_may_beat(fp, bx, by, best, mg)
                                     : aabb_may_beat(fp, bx, by, best, mg))) {
    work |= kWorkEdges;
    best = fminf(best, sd_body<KIND, NB>(fp, bx, by));
  }
  return best;
}

// Chunk bound: the chunk's points lie in the world box {cx +- hx, cy +- hy}; in the body frame
// of pose q that box lies inside the box centred at R(theta)^T (c - t) with half extents
// (|cos| hx + |sin| hy, |sin| hx + |cos| hy). No point of the chunk is nearer to the footprint
// than that box is to the cover union (0 if they overlap: evaluate).
__device__ __forceinline__ bool chunk_may_beat(const FpDev& fp, float4 q, float4 b, float best,
                                               float mg) {
  const float dx = b.x - q.x, dy = b.y - q.y;
  const float bx = fmaf(q.z, dx, q.w * dy), by = fmaf(q.z, dy, -(q.w * dx));
  const float ac = fabsf(q.z), as = fabsf(q.w);
  const float ex = fmaf(ac, b.z, as * b.w), ey = fmaf(as, b.z, ac * b.w);
  float d2 = __int_as_float(0x7f800000);
#pragma unroll
  for (int j = 0; j < kMaxCover; ++j) {
    if (!cover_slot(fp, j)) break;
    const float ax = fmaxf(fabsf(bx - fp.cover[j][0]) - (fp.cover[j][2] + ex), 0.f);
    const float ay = fmaxf(fabsf(by - fp.cover[j][1]) - (fp.cover[j][3] + ey), 0.f);
    d2 = fminf(d2, fmaf(ax, ax, ay * ay));
  }
  const float lim = best + mg;
  if (d2 == 0.f) {  // touches the cover: every point is at least as shallow as the AABB allows
    const float lx = fmaxf(fp.aabb[0] - (bx + ex), (bx - ex) - fp.aabb[1]);
    const float ly = fmaxf(fp.aabb[2] - (by + ey), (by - ey) - fp.aabb[3]);
    return fmaxf(lx, ly) < lim;
  }
  return lim > 0.f && d2 < lim * lim;
}

// Order-preserving float -> u32 key (for min via integer reductions / atomics).
__device__ __forceinline__ unsigned fkey(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unkey(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// ------------------------------------------------------------------ kernels
#ifndef EXM_PTS_PER_CELL  // A/B builds override the cell-size constants below
#define EXM_PTS_PER_CELL 16.0f
#endif
#ifndef EXM_CELL_MIN_R
#define EXM_CELL_MIN_R 0.18f
#endif
#ifndef EXM_CELL_MAX_R
#define EXM_CELL_MAX_R 0.5f
#endif
#ifndef EXM_CELL_SEARCH_FRAC
#define EXM_CELL_SEARCH_FRAC 1.25f
#endif
constexpr float kPtsPerCell = EXM_PTS_PER_CELL;  // swept 8-64 (tools/cfg5_snapshots.py): cfg2/cfg3 flat over 16-32, cfg5 snapshots -3 % at 16
constexpr int kPrepCache = 12;  // cloud points per k_cloud_prep thread kept in registers
constexpr float kCellMinR = EXM_CELL_MIN_R;       // cell edge >= kCellMinR * R (swept 0.12-0.25: cfg3 1.99 -> 1.88 ms,
                                          // cfg5 snapshots -1 %, cfg1/cfg2 flat; cfg3 is alignment-sensitive)
constexpr float kCellMaxR = EXM_CELL_MAX_R;       // cell edge <= kCellMaxR * R ...
constexpr float kCellSearchFrac = EXM_CELL_SEARCH_FRAC;  // ... or <= this fraction of R + mean d_min
// (with the control cycle's d_safe threshold the mean d_min is the capped one, and the search
// disc radius <= R + d_safe; swept 0.25-2.0: cfg1 step 0.079 -> 0.058 ms and cfg2 0.145 ->
// 0.142 ms at 1.25 against the unthresholded 0.385; cfg3 / cfg5 flat: density-sized cells)
// Below this many poses one thread per pose leaves most SMs idle (< ~16 warps each): use one
// warp per pose instead.
// (measured on config 2's cloud: 25.6k poses warp 45 us / thread 64 us, 51.2k poses warp 76 us
// / thread 65 us; config 1's 30.7k poses warp 68 us / thread 114 us)
constexpr int kWarpPerPoseMax = 40000;
constexpr int kCtaPerPoseMax = 1024;  // ... and below this, a CTA of 8 warps per pose
// Grid of the recentred valid cloud: bounding box, cell edge from the point density and the
// previous step's search radius, cull margin (shared by both preparation kernels).
__device__ __forceinline__ GridMeta make_gridmeta(float mnx, float mxx, float mny, float mxy,
                                                  int cnt, float cs_lo, float cs_hi,
                                                  float pts_per_cell, float radius, float ds0,
                                                  float ds1, int chunk, float search_lo) {
  GridMeta g;
  g.n_valid = cnt;
  g.chunk = chunk;
  g.reserved = 0;
  g.margin = kCullMargin;
  if (cnt == 0) {
    g.x0 = g.y0 = 0.0f; g.cs = 1.0f; g.inv_cs = 1.0f; g.gx = g.gy = 1;
    return g;
  }
  // cull slack: covers the FP32 rounding of every bound (coordinates recentred at q0)
  g.margin += 5e-7f * fmaxf(fmaxf(fabsf(mnx), fabsf(mxx)), fmaxf(fabsf(mny), fabsf(mxy)));
  const float ex = mxx - mnx, ey = mxy - mny;
  // Cell edge: about pts_per_cell points per cell on average, within [cs_lo, cs_hi] (dense
  // boundary clouds get finer cells, sparse ones coarser), at most kGridMax per axis.
  const float dens = sqrtf(pts_per_cell * fmaxf(ex * ey, 1e-6f) / static_cast<float>(cnt));
  // upper bound: a fixed fraction of the expected search radius R + mean(d_min) of the
  // previous step when there is one (far obstacles: coarse cells, few rings), else cs_hi
  float hi = cs_hi;
  if (ds1 > 0.f) hi = fmaxf(cs_hi, kCellSearchFrac * (radius + ds0 / ds1));
  float cs = fminf(fmaxf(dens, cs_lo), hi);
  // far obstacles (large mean d_min): the search covers more rings; search_lo > 0 floors the
  // cell edge at that fraction of the expected search radius
  if (ds1 > 0.f && search_lo > 0.f) cs = fmaxf(cs, search_lo * (radius + ds0 / ds1));
  cs = fmaxf(cs, fmaxf(ex, ey) / static_cast<float>(kGridMax - 1) * 1.001f);
  cs = fmaxf(cs, 1e-4f);
  g.x0 = mnx; g.y0 = mny; g.cs = cs; g.inv_cs = 1.0f / cs;
  g.gx = min(kGridMax, static_cast<int>(ex * g.inv_cs) + 1);
  g.gy = min(kGridMax, static_cast<int>(ey * g.inv_cs) + 1);
  return g;
}

#if EXM_PART == 0
// Single-CTA cloud preparation: mask compaction, FP64 recentring at q0 then FP32 rounding,
// bounding box, uniform grid (cell >= cs_target, <= kGridMax per axis), counting sort.
__global__ void __launch_bounds__(1024) k_cloud_prep(const double* __restrict__ pts,
                                                     const uint8_t* __restrict__ mask,
                                                     const StepDyn* __restrict__ dyn,
                                                     float cs_lo, float cs_hi, float pts_per_cell,
                                                     float radius, int chunk, float search_lo,
                                                     int prefetch, float* __restrict__ dstat,
                                                     float2* __restrict__ tmp,
                                                     float2* __restrict__ raw,
                                                     int* __restrict__ raw_start,
                                                     int* __restrict__ cell_start,
                                                     GridMeta* __restrict__ gm_out) {
  pdl_wait();
  extern __shared__ int hist[];  // kGridMax * kGridMax
  __shared__ float red[4][32];
  __shared__ int redc[32];
  __shared__ long long scan_tot[32];
  __shared__ GridMeta gm;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = dyn->n_points;
  const bool use_mask = dyn->use_mask != 0;
  // One CTA cannot keep enough loads in flight to pull the cloud from HBM at speed: ask the L2
  // for it first, in 4 KB bulk prefetches spread over the L2 slices (a hint; no ordering).
  if (prefetch && tid < 64) {
    const size_t bytes = 16 * static_cast<size_t>(n);
    for (size_t off = static_cast<size_t>(tid) * 4096; off < bytes; off += 64 * 4096) {
      const unsigned sz = static_cast<unsigned>(bytes - off < 4096 ? bytes - off : 4096);
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const char*>(pts) + off), "r"(sz) : "memory");
    }
    const size_t mb = use_mask ? (static_cast<size_t>(n) & ~static_cast<size_t>(15)) : 0;
    if (tid == 63 && mb > 0)
      for (size_t off = 0; off < mb; off += 4096) {
        const unsigned sz = static_cast<unsigned>(mb - off < 4096 ? mb - off : 4096);
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(mask + off), "r"(sz) : "memory");
      }
  }
  const double qx = dyn->q0[0], qy = dyn->q0[1];
  const float nanf_ = __int_as_float(0x7fc00000);
  float mnx = FLT_MAX, mxx = -FLT_MAX, mny = FLT_MAX, mxy = -FLT_MAX;
  int cnt = 0;
  EXM_PROBE_P(0);
  // The first kPrepCache * blockDim points stay in registers across the three passes (bbox,
  // histogram, scatter); the rest (large clouds) go through `tmp`.
  const double2* p2 = reinterpret_cast<const double2*>(pts);
  float2 pc[kPrepCache];
  int pcell[kPrepCache];
  auto load = [&](int i) {
    const double2 w = p2[i];  // unconditional: independent of the mask load
    const bool v = !use_mask || mask[i] != 0;
    float2 p = make_float2(nanf_, nanf_);
    if (v) {
      p = make_float2(static_cast<float>(w.x - qx), static_cast<float>(w.y - qy));
      mnx = fminf(mnx, p.x); mxx = fmaxf(mxx, p.x);
      mny = fminf(mny, p.y); mxy = fmaxf(mxy, p.y);
      ++cnt;
    }
    return p;
  };
#pragma unroll
  for (int j = 0; j < kPrepCache; ++j) {
    const int i = tid + j * static_cast<int>(blockDim.x);
    pc[j] = i < n ? load(i) : make_float2(nanf_, nanf_);
  }
  const int n_cached = kPrepCache * static_cast<int>(blockDim.x);
#pragma unroll 4
  for (int i = n_cached + tid; i < n; i += blockDim.x) tmp[i] = load(i);
  for (int o = 16; o; o >>= 1) {
    mnx = fminf(mnx, __shfl_xor_sync(kFull, mnx, o));
    mxx = fmaxf(mxx, __shfl_xor_sync(kFull, mxx, o));
    mny = fminf(mny, __shfl_xor_sync(kFull, mny, o));
    mxy = fmaxf(mxy, __shfl_xor_sync(kFull, mxy, o));
    cnt += __shfl_xor_sync(kFull, cnt, o);
  }
  EXM_PROBE_P(1);
  if (lane == 0) { red[0][warp] = mnx; red[1][warp] = mxx; red[2][warp] = mny; red[3][warp] = mxy; redc[warp] = cnt; }
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    mnx = lane < nw ? red[0][lane] : FLT_MAX;
    mxx = lane < nw ? red[1][lane] : -FLT_MAX;
    mny = lane < nw ? red[2][lane] : FLT_MAX;
    mxy = lane < nw ? red[3][lane] : -FLT_MAX;
    cnt = lane < nw ? redc[lane] : 0;
    for (int o = 16; o; o >>= 1) {
      mnx = fminf(mnx, __shfl_xor_sync(kFull, mnx, o));
      mxx = fmaxf(mxx, __shfl_xor_sync(kFull, mxx, o));
      mny = fminf(mny, __shfl_xor_sync(kFull, mny, o));
      mxy = fmaxf(mxy, __shfl_xor_sync(kFull, mxy, o));
      cnt += __shfl_xor_sync(kFull, cnt, o);
    }
  }
  if (tid == 0) {
    const GridMeta g = make_gridmeta(mnx, mxx, mny, mxy, cnt, cs_lo, cs_hi, pts_per_cell, radius,
                                     dstat[0], dstat[1], chunk, search_lo);
    gm = g;
    *gm_out = g;
    dstat[0] = 0.f;  // consumed: the stage costs of this step accumulate the next statistic
    dstat[1] = 0.f;
  }
  __syncthreads();
  EXM_PROBE_P(2);
  const int cells = gm.gx * gm.gy;
  for (int c = tid; c < cells; c += blockDim.x) hist[c] = 0;
  __syncthreads();
  auto cell_of = [&](float2 p) {
    const int ix = min(gm.gx - 1, max(0, static_cast<int>((p.x - gm.x0) * gm.inv_cs)));
    const int iy = min(gm.gy - 1, max(0, static_cast<int>((p.y - gm.y0) * gm.inv_cs)));
    return iy * gm.gx + ix;
  };
  if (gm.n_valid > 0) {
#pragma unroll
    for (int j = 0; j < kPrepCache; ++j) {
      pcell[j] = pc[j].x == pc[j].x ? cell_of(pc[j]) : -1;
      if (pcell[j] >= 0) atomicAdd(&hist[pcell[j]], 1);
    }
#pragma unroll 4
    for (int i = n_cached + tid; i < n; i += blockDim.x) {
      const float2 p = tmp[i];
      if (p.x == p.x) atomicAdd(&hist[cell_of(p)], 1);
    }
  }
  __syncthreads();
  EXM_PROBE_P(3);
  // Exclusive scans of the cell counts (raw_start) and of the counts padded to whole chunks
  // (cell_start), as one 64-bit scan {padded:raw}; each thread owns a contiguous segment.
  const int seg = (cells + blockDim.x - 1) / blockDim.x;
  const int c0 = min(cells, tid * seg), c1 = min(cells, c0 + seg);
  auto both = [chunk](int h) {
    return (static_cast<long long>((h + chunk - 1) & ~(chunk - 1)) << 32) | static_cast<long long>(h);
  };
  long long local = 0;
  for (int c = c0; c < c1; ++c) local += both(hist[c]);
  long long incl = local;
  for (int o = 1; o < 32; o <<= 1) {
    const long long v = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) scan_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    const long long v = lane < nw ? scan_tot[lane] : 0;
    long long sc = v;
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = __shfl_up_sync(kFull, sc, o);
      if (lane >= o) sc += u;
    }
    if (lane < nw) scan_tot[lane] = sc - v;  // exclusive warp offsets
  }
  __syncthreads();
  long long run = scan_tot[warp] + incl - local;
  for (int c = c0; c < c1; ++c) {
    const int h = hist[c];
    raw_start[c] = static_cast<int>(run & 0xffffffffll);
    cell_start[c] = static_cast<int>(run >> 32);
    hist[c] = static_cast<int>(run & 0xffffffffll);  // becomes the scatter cursor
    run += both(h);
  }
  if (c0 < c1 && c1 == cells) {
    raw_start[cells] = static_cast<int>(run & 0xffffffffll);
    cell_start[cells] = static_cast<int>(run >> 32);
  }
  __syncthreads();
  EXM_PROBE_P(4);
  if (gm.n_valid > 0) {
#pragma unroll
    for (int j = 0; j < kPrepCache; ++j)
      if (pcell[j] >= 0) raw[atomicAdd(&hist[pcell[j]], 1)] = pc[j];
#pragma unroll 4
    for (int i = n_cached + tid; i < n; i += blockDim.x) {
      const float2 p = tmp[i];
      if (p.x == p.x) raw[atomicAdd(&hist[cell_of(p)], 1)] = p;
    }
  }
  __syncthreads();
  EXM_PROBE_P(5);
}

// Morton index of a point on the kSubCells x kSubCells sub-grid of its cell.
__device__ __forceinline__ int sub_key(float2 p, float ox, float oy, float sub) {
  const int sx = min(kSubCells - 1, max(0, static_cast<int>((p.x - ox) * sub)));
  const int sy = min(kSubCells - 1, max(0, static_cast<int>((p.y - oy) * sub)));
  auto spread = [](int v) {
    v = (v | (v << 2)) & 0x33;
    return (v | (v << 1)) & 0x55;
  };
  return spread(sx) | (spread(sy) << 1);
}

// One nonempty cell, one warp: counting sort of the cell's points by their sub-grid Morton index
// (so every chunk of consecutive points is compact), NaN pads up to a whole chunk, and the
// chunk bounding boxes. hist: kSubCells^2 ints of this warp's shared memory.
__device__ __forceinline__ void sort_cell(int c, int lane, int* hist, const float2* __restrict__ raw,
                                          const int* __restrict__ raw_start,
                                          const int* __restrict__ cell_start, const GridMeta& gm,
                                          float2* __restrict__ cloud, float4* __restrict__ chunk) {
  constexpr int kKeys = kSubCells * kSubCells;
  const float sub = gm.inv_cs * static_cast<float>(kSubCells);
  const float2 pad = make_float2(__int_as_float(0x7fc00000), __int_as_float(0x7fc00000));
  const int rs = raw_start[c], n = raw_start[c + 1] - rs;
  if (n == 0) return;  // warp-uniform
  const int ps = cell_start[c];
  const float ox = gm.x0 + static_cast<float>(c % gm.gx) * gm.cs;
  const float oy = gm.y0 + static_cast<float>(c / gm.gx) * gm.cs;
  for (int b = lane; b < kKeys; b += 32) hist[b] = 0;
  __syncwarp();
  for (int i = lane; i < n; i += 32) atomicAdd(&hist[sub_key(raw[rs + i], ox, oy, sub)], 1);
  __syncwarp();
  constexpr int kPer = kKeys / 32;
  int v[kPer], loc = 0;
#pragma unroll
  for (int k = 0; k < kPer; ++k) loc += (v[k] = hist[lane * kPer + k]);
  int incl = loc;
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += u;
  }
  int run = incl - loc;
#pragma unroll
  for (int k = 0; k < kPer; ++k) {
    hist[lane * kPer + k] = run;
    run += v[k];
  }
  __syncwarp();
  for (int i = lane; i < n; i += 32) {
    const float2 p = raw[rs + i];
    cloud[ps + atomicAdd(&hist[sub_key(p, ox, oy, sub)], 1)] = p;
  }
  const int C = gm.chunk;
  const int np = (n + C - 1) & ~(C - 1);
  if (n + lane < np) cloud[ps + n + lane] = pad;
  __syncwarp();  // orders the warp's global stores before the L2 reads below
  for (int j = lane; j < np / C; j += 32) {
    float x0 = FLT_MAX, x1 = -FLT_MAX, y0 = FLT_MAX, y1 = -FLT_MAX;
#pragma unroll 8
    for (int k = 0; k < C; ++k) {
      const float2 p = __ldcg(cloud + ps + j * C + k);
      if (p.x == p.x) {
        x0 = fminf(x0, p.x); x1 = fmaxf(x1, p.x);
        y0 = fminf(y0, p.y); y1 = fmaxf(y1, p.y);
      }
    }
    chunk[ps / C + j] =
        make_float4(0.5f * (x0 + x1), 0.5f * (y0 + y1), 0.5f * (x1 - x0), 0.5f * (y1 - y0));
  }
  __syncwarp();
}

// Second prep pass, one warp per nonempty cell: counting sort of the cell's points by their
// sub-grid Morton index (so every chunk of consecutive points is compact), NaN pads up
// to a whole chunk, and the chunk bounding boxes.
constexpr int kSortWarps = 8;
__global__ void __launch_bounds__(kSortWarps * 32) k_cell_sort(
    const float2* __restrict__ raw, const int* __restrict__ raw_start,
    const int* __restrict__ cell_start, const GridMeta* __restrict__ gmp,
    float2* __restrict__ cloud, float4* __restrict__ chunk) {
  pdl_wait();
  constexpr int kKeys = kSubCells * kSubCells;
  __shared__ int s_hist[kSortWarps][kKeys];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int* hist = s_hist[wid];
  const GridMeta gm = *gmp;
  const int cells = gm.n_valid > 0 ? gm.gx * gm.gy : 0;
  for (int c = blockIdx.x * kSortWarps + wid; c < cells; c += gridDim.x * kSortWarps)
    sort_cell(c, lane, hist, raw, raw_start, cell_start, gm, cloud, chunk);
}

#endif  // EXM_PART == 0

// Ring c (Chebyshev radius k >= 1) around (ci, cj): 8k cells, enumerated row/column-wise.
__device__ __forceinline__ void ring_cell(int k, int t, int ci, int cj, int& i, int& j) {
  if (k == 0) { i = ci; j = cj; return; }
  const int row = 2 * k + 1;
  if (t < row) { i = ci - k + t; j = cj + k; return; }
  t -= row;
  if (t < row) { i = ci - k + t; j = cj - k; return; }
  t -= row;
  const int col = 2 * k - 1;
  if (t < col) { i = ci - k; j = cj - k + 1 + t; return; }
  t -= col;
  i = ci + k; j = cj - k + 1 + t;
}

// World-frame AABB of the footprint at pose q: the body-frame AABB (fp.aabb) rotated by theta
// and re-boxed. Every footprint point lies inside it, so for any obstacle point o outside it
// sd(o) >= dist(o, W) — an exact lower bound that is much tighter than |o - t| - R for
// elongated or off-centre footprints (forklift, L).
struct WBox {
  float x0, x1, y0, y1;
};
__device__ __forceinline__ WBox world_box(const FpDev& fp, float4 q, float mg) {
  const float cx = 0.5f * (fp.aabb[0] + fp.aabb[1]), cy = 0.5f * (fp.aabb[2] + fp.aabb[3]);
  const float hx = 0.5f * (fp.aabb[1] - fp.aabb[0]), hy = 0.5f * (fp.aabb[3] - fp.aabb[2]);
  const float ac = fabsf(q.z), as = fabsf(q.w);
  const float wx = fmaf(ac, hx, as * hy) + mg, wy = fmaf(as, hx, ac * hy) + mg;
  const float ox = q.x + fmaf(q.z, cx, -(q.w * cy)), oy = q.y + fmaf(q.w, cx, q.z * cy);
  return {ox - wx, ox + wx, oy - wy, oy + wy};
}
// d2 = squared distance from W to the box [bx0,bx1]x[by0,by1] (0 if they overlap); may the box
// contain a point that beats `best`?
__device__ __forceinline__ bool box_may_beat(const WBox& w, float bx0, float bx1, float by0,
                                             float by1, float best, float mg) {
  const float gx = fmaxf(fmaxf(bx0 - w.x1, w.x0 - bx1), 0.f);
  const float gy = fmaxf(fmaxf(by0 - w.y1, w.y0 - by1), 0.f);
  const float d2 = fmaf(gx, gx, gy * gy);
  const float lim = best + mg;
  return d2 == 0.f || (lim > 0.f && d2 < lim * lim);
}

// Exact per-pose min signed distance with exact culling (min_signed_distance_at semantics).
// Thread <-> pose; a warp walks grid rings outward from its poses' centroid, nearest first, and
// stops once no lane's lower bound can beat that lane's running minimum. Lower bounds (all
// exact): ring and cell via the world box W of the footprint, then per point the
// distance to W and the distance to the body-frame AABB, then the exact polygon/cover SDF.
// STATS (profiling builds of the launch only): count the point tests and exact SDF
// evaluations the culls let through, for the executed-work roofline.
// MODE: kGridFull (every bound), kGridNoChunk (no chunk bound: A/B only), kGridBrute (no bound
// at all: every valid point is evaluated, the same arithmetic without culling — the reference
// the exactness tests compare the culled minimum with, bit for bit).
constexpr int kGridNoChunk = 0, kGridFull = 1, kGridBrute = 2;
// Read-only load of the cloud structure: from shared memory (SMEM: the CTA staged it by TMA) or
// through the read-only data path.
template <bool SMEM, typename V>
__device__ __forceinline__ V ldro(const V* p) {
  if constexpr (SMEM) return *p;
  else return __ldg(p);
}
template <int KIND, int NB, bool STATS, int MODE, bool SMEM = false>
__device__ __forceinline__ void sdf_grid_warp(const FpDev& fp, const float4* __restrict__ poses,
                                              int n_poses, const GridMeta& gm,
                                              const int* __restrict__ cell_start,
                                              const float2* __restrict__ cloud,
                                              const float4* __restrict__ chunk,
                                              const float* __restrict__ cap, float thr, int T,
                                              int rows, float* __restrict__ out, int i, int lane,
                                              unsigned long long* cnt) {
  const bool active = i < n_poses;
  // h-major lanes: the poses are stored [row][h] (row = rollout); with rows > 0 logical index
  // i = h * rows + row, so a warp takes 32 consecutive rollouts at the same step h (spatially
  // coherent: one set of ring cells serves all lanes) instead of one rollout's 32 steps
  int hh = 0, pi = i;
  if (rows > 0) {
    hh = i / rows;
    pi = (i - hh * rows) * T + hh;
  } else if (T > 0) {
    hh = i % T;
  }
  if (gm.n_valid == 0) {
    if (active) out[pi] = kEmptyDistance;
    return;
  }
  const float4 q = active ? poses[pi] : make_float4(0.f, 0.f, 1.f, 0.f);
  float sx = active ? q.x : 0.f, sy = active ? q.y : 0.f;
  int na = active ? 1 : 0;
  for (int o = 16; o; o >>= 1) {
    sx += __shfl_xor_sync(kFull, sx, o);
    sy += __shfl_xor_sync(kFull, sy, o);
    na += __shfl_xor_sync(kFull, na, o);
  }
  if (na == 0) return;
  const float cx = sx / na, cy = sy / na;
  const int ci = min(gm.gx - 1, max(0, static_cast<int>(floorf((cx - gm.x0) * gm.inv_cs))));
  const int cj = min(gm.gy - 1, max(0, static_cast<int>(floorf((cy - gm.y0) * gm.inv_cs))));
  const float mg = gm.margin;
  const WBox w = world_box(fp, q, mg);
  const float R = fp.radius + mg;
  const int kmax = max(max(ci, gm.gx - 1 - ci), max(cj, gm.gy - 1 - cj));
  // Capped first pass: cap[h] is a guess of step h's minimum (from the previous control step).
  // Bounds at or above the cap are pruned as if a point at distance cap had been evaluated, so a
  // pose whose true minimum m* lies below the cap still gets m* exactly (no point with sd = m*
  // is ever pruned: its bound is <= m* < best); poses left at the cap rerun uncapped (pass 1).
  const float kInf = __int_as_float(0x7f800000);
  // thr: results are min(exact minimum, thr) (+inf: exact everywhere); minima below thr are
  // exact, so thr acts as a cap that is never re-run
  const float capv = fminf((cap != nullptr && active && MODE != kGridBrute) ? cap[hh] : kInf, thr);
  float best = capv;
  bool todo = active;
  for (int pass = 0; pass < 2; ++pass) {
  if (pass == 1) {
    todo = active && !(best < capv) && capv < thr;
    if (!__any_sync(kFull, todo)) break;
    if (todo) best = thr;
  }
  for (int k = 0; k <= kmax; ++k) {
    if (k > 0) {
      // every point of ring k or beyond lies outside the inner square S_{k-1}
      const float bx0 = gm.x0 + static_cast<float>(ci - k + 1) * gm.cs;
      const float bx1 = gm.x0 + static_cast<float>(ci + k) * gm.cs;
      const float by0 = gm.y0 + static_cast<float>(cj - k + 1) * gm.cs;
      const float by1 = gm.y0 + static_cast<float>(cj + k) * gm.cs;
      // lbc: sd >= |o - t| - R holds inside the footprint too (|p| + depth <= R), so it bounds
      // negative minima; lbw (distance from W to the outside of S) only when W lies inside S
      const float lbw = fminf(fminf(w.x0 - bx0, bx1 - w.x1), fminf(w.y0 - by0, by1 - w.y1));
      const float lbc = fminf(fminf(q.x - bx0, bx1 - q.x), fminf(q.y - by0, by1 - q.y)) - R;
      const float lb = lbw > 0.f ? fmaxf(lbw, lbc) : lbc;
      const bool need = todo && (MODE == kGridBrute || lb < best + mg);
      if (!__any_sync(kFull, need)) break;
    }
    const int ncell = k == 0 ? 1 : 8 * k;
    if (STATS && lane == 0) ++cnt[kCntRing];
    // The warp enumerates the ring 32 cells at a time, one cell per lane (position, range,
    // CSR bounds: the cell_start loads of the 32 cells are in flight together), and then
    // visits only the in-range nonempty ones, in ring order, with the cell's data shuffled in.
    for (int t0 = 0; t0 < ncell; t0 += 32) {
      int c_i = 0, c_j = 0, c_s = 0, c_e = 0;
      if (t0 + lane < ncell) {
        ring_cell(k, t0 + lane, ci, cj, c_i, c_j);
        if (c_i >= 0 && c_j >= 0 && c_i < gm.gx && c_j < gm.gy) {
          const int c = c_j * gm.gx + c_i;
          c_s = ldro<SMEM>(cell_start + c);
          c_e = ldro<SMEM>(cell_start + c + 1);
        }
      }
      unsigned cells = __ballot_sync(kFull, c_s != c_e);
    while (cells) {
      const int src = __ffs(cells) - 1;
      cells &= cells - 1;
      const int ii = __shfl_sync(kFull, c_i, src), jj = __shfl_sync(kFull, c_j, src);
      const int s = __shfl_sync(kFull, c_s, src), e = __shfl_sync(kFull, c_e, src);
      const float bx0 = gm.x0 + static_cast<float>(ii) * gm.cs, bx1 = bx0 + gm.cs;
      const float by0 = gm.y0 + static_cast<float>(jj) * gm.cs, by1 = by0 + gm.cs;
      const float gx_ = fmaxf(fmaxf(bx0 - q.x, q.x - bx1), 0.f);
      const float gy_ = fmaxf(fmaxf(by0 - q.y, q.y - by1), 0.f);
      const float lim = R + best;
      const bool need = todo && (MODE == kGridBrute || ((gx_ * gx_ + gy_ * gy_ < lim * lim) &&
                                   box_may_beat(w, bx0, bx1, by0, by1, best, mg)));
      if (STATS && todo) ++cnt[kCntCell];
      if (!__any_sync(kFull, need)) continue;
      float l2 = lim * lim;
      // chunks of gm.chunk Morton-ordered points: one body-frame box bound per chunk, then the
      // per-point bounds and the exact SDF for the points of the chunks some lane still needs
      const int csh = gm.chunk == 16 ? 4 : (gm.chunk == 8 ? 3 : 2);
      for (int ch = s >> csh; ch < e >> csh; ++ch) {
        bool cneed = need;
        if (MODE == kGridFull) {
          cneed = need && chunk_may_beat(fp, q, ldro<SMEM>(chunk + ch), best, mg);
          if (STATS && need) ++cnt[kCntChunk];
          if (!__any_sync(kFull, cneed)) continue;
        }
        const float2* cp = cloud + (ch << csh);
#if defined(EXM_QUAD_POINTS)
        // A/B builds: four points per iteration (four independent chains)
#pragma unroll 1
        for (int p = 0; p < gm.chunk; p += 4) {
          const float4 oa = ldro<SMEM>(reinterpret_cast<const float4*>(cp + p));
          const float4 ob = ldro<SMEM>(reinterpret_cast<const float4*>(cp + p + 2));
          const float dx[4] = {oa.x - q.x, oa.z - q.x, ob.x - q.x, ob.z - q.x};
          const float dy[4] = {oa.y - q.y, oa.w - q.y, ob.y - q.y, ob.w - q.y};
          bool a[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            a[u] = cneed && (MODE == kGridBrute ? dx[u] == dx[u] : dx[u] * dx[u] + dy[u] * dy[u] < l2);
          if (a[0] || a[1] || a[2] || a[3]) {
            float nb = kInf;
            unsigned wa = 0u;
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              unsigned w;
              const float b = grid_point<KIND, NB, MODE == kGridBrute>(
                  fp, fmaf(q.z, dx[u], q.w * dy[u]), fmaf(q.z, dy[u], -(q.w * dx[u])), best, mg, w);
              nb = fminf(nb, a[u] ? b : kInf);
              wa |= a[u] ? w : 0u;
            }
            best = fminf(best, nb);
            if (wa & (kWorkTileVal | kWorkEdges)) {
              const float nl = R + best;
              l2 = nl * nl;
            }
          }
        }
#elif !defined(EXM_SINGLE_POINTS)
        // two points per iteration, both valued whenever either passes its circle test: two
        // independent dependency chains for the scheduler (measured -7% on cfg3, -2.3% on cfg5,
        // -1% on cfg2 against one point per iteration, which -DEXM_SINGLE_POINTS restores)
#pragma unroll 1
        for (int p = 0; p < gm.chunk; p += 2) {
          const float4 o2 = ldro<SMEM>(reinterpret_cast<const float4*>(cp + p));
          const float dx0 = o2.x - q.x, dy0 = o2.y - q.y, dx1 = o2.z - q.x, dy1 = o2.w - q.y;
          if (STATS && cneed) cnt[kCntPoint] += 2;
          if (STATS && lane == 0) cnt[kCntPointWarp] += 2;
          const bool a0 = cneed && (MODE == kGridBrute ? o2.x == o2.x : dx0 * dx0 + dy0 * dy0 < l2);
          const bool a1 = cneed && (MODE == kGridBrute ? o2.z == o2.z : dx1 * dx1 + dy1 * dy1 < l2);
          if (a0 || a1) {
            unsigned w0, w1;
            const float b0 = grid_point<KIND, NB, MODE == kGridBrute>(
                fp, fmaf(q.z, dx0, q.w * dy0), fmaf(q.z, dy0, -(q.w * dx0)), best, mg, w0);
            const float b1 = grid_point<KIND, NB, MODE == kGridBrute>(
                fp, fmaf(q.z, dx1, q.w * dy1), fmaf(q.z, dy1, -(q.w * dx1)), best, mg, w1);
            // only the passing points' values count: a NaN pad is not "never below best" (the
            // rectangle SDF's fmaxf(NaN, 0) reads 0), and a real point that failed its circle
            // test adds nothing the exact minimum needs
            best = fminf(best, fminf(a0 ? b0 : kInf, a1 ? b1 : kInf));
            if (STATS) {  // executed work: both points were transformed and valued
              cnt[kCntTransform] += 2;
              cnt[kCntTile] += ((w0 & kWorkTile) != 0u) + ((w1 & kWorkTile) != 0u);
              cnt[kCntTileVal] += ((w0 & kWorkTileVal) != 0u) + ((w1 & kWorkTileVal) != 0u);
              cnt[kCntBound] += ((w0 & kWorkBound) != 0u) + ((w1 & kWorkBound) != 0u);
              cnt[kCntEdges] += ((w0 & kWorkEdges) != 0u) + ((w1 & kWorkEdges) != 0u);
            }
            if (((a0 ? w0 : 0u) | (a1 ? w1 : 0u)) & (kWorkTileVal | kWorkEdges)) {
              const float nl = R + best;
              l2 = nl * nl;
            }
          }
        }
#else
#pragma unroll 1
        for (int p = 0; p < gm.chunk; ++p) {
          const float2 o = ldro<SMEM>(cp + p);
          const float dx = o.x - q.x, dy = o.y - q.y;
          if (STATS && cneed) ++cnt[kCntPoint];
          if (STATS && lane == 0) ++cnt[kCntPointWarp];
          if (cneed && (MODE == kGridBrute ? o.x == o.x : dx * dx + dy * dy < l2)) {  // NaN pads
            const float bx = fmaf(q.z, dx, q.w * dy);
            const float by = fmaf(q.z, dy, -(q.w * dx));
            unsigned wk;
            best = grid_point<KIND, NB, MODE == kGridBrute>(fp, bx, by, best, mg, wk);
            if (STATS) {
              ++cnt[kCntTransform];
              cnt[kCntTile] += (wk & kWorkTile) != 0u;
              cnt[kCntTileVal] += (wk & kWorkTileVal) != 0u;
              cnt[kCntBound] += (wk & kWorkBound) != 0u;
              cnt[kCntEdges] += (wk & kWorkEdges) != 0u;
            }
            if (wk & (kWorkTileVal | kWorkEdges)) {
              const float nl = R + best;
              l2 = nl * nl;
            }
          }
        }
#endif
      }
    }  // cells of this group
    }  // groups of 32 ring cells
  }
  }  // pass
  if (active) out[pi] = best;
}

// Persistent warps: the grid is sized to the resident capacity and every warp takes the next
// 32 poses from a work counter until none are left (the cost per pose varies by an order of
// magnitude between open space and clutter, so a static mapping ends in a long tail of a few
// busy SMs). The last warp to finish resets the counter pair for the next launch.
// work == nullptr: static mapping, warp <-> poses blockIdx.x * 128 + warp * 32 + lane.
#ifndef EXM_GRID_THREADS  // A/B builds: threads per CTA (32-128 measured within 1 %, round 1)
#define EXM_GRID_THREADS 128
#endif
// (-DEXM_GRID_MINB=n A/B builds: at least n resident CTAs per SM, capping registers; the product
// build leaves the register count to ptxas: 64, i.e. 8 CTAs of 128 threads per SM)
#ifdef EXM_GRID_MINB
#define EXM_GRID_BOUNDS __launch_bounds__(EXM_GRID_THREADS, EXM_GRID_MINB)
#else
#define EXM_GRID_BOUNDS __launch_bounds__(EXM_GRID_THREADS)
#endif
template <int KIND, int NB, bool STATS = false, int MODE = kGridFull>
__global__ void EXM_GRID_BOUNDS k_sdf_grid(const __grid_constant__ FpDev fp,
                                                  const float4* __restrict__ poses, int n_poses,
                                                  const GridMeta* __restrict__ gmp,
                                                  const int* __restrict__ cell_start,
                                                  const float2* __restrict__ cloud,
                                                  const float4* __restrict__ chunk,
                                                  const float* __restrict__ cap, float thr, int T,
                                                  int rows, float* __restrict__ out,
                                                  unsigned* __restrict__ work,
                                                  unsigned long long* __restrict__ stats = nullptr) {
  pdl_wait();
  unsigned long long cnt[kCntN];
#pragma unroll
  for (int k = 0; k < kCntN; ++k) cnt[k] = 0ull;
  const int lane = threadIdx.x & 31;
  const GridMeta gm = *gmp;
  if (work == nullptr) {
    sdf_grid_warp<KIND, NB, STATS, MODE>(fp, poses, n_poses, gm, cell_start, cloud, chunk, cap, thr,
                                         T, rows, out, blockIdx.x * blockDim.x + threadIdx.x, lane,
                                         cnt);
  } else {
    for (;;) {
      unsigned base = 0;
      if (lane == 0) base = atomicAdd(work, 32u);
      base = __shfl_sync(kFull, base, 0);
      if (base >= static_cast<unsigned>(n_poses)) break;
      sdf_grid_warp<KIND, NB, STATS, MODE>(fp, poses, n_poses, gm, cell_start, cloud, chunk, cap,
                                           thr, T, rows, out, static_cast<int>(base) + lane, lane, cnt);
    }
    if (lane == 0) {
      __threadfence();
      const unsigned warps = gridDim.x * (blockDim.x >> 5);
      if (atomicAdd(work + 1, 1u) == warps - 1) {  // every warp is past its last grab
        work[0] = 0u;
        work[1] = 0u;
        __threadfence();
      }
    }
  }
  if (STATS) {
#pragma unroll
    for (int k = 0; k < kCntN; ++k) {
      unsigned long long v = cnt[k];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
      if (lane == 0 && v) atomicAdd(stats + k, v);
    }
  }
}

// The cloud structure staged into shared memory by TMA bulk copies and shared by a persistent
// 1,024-thread CTA per SM (the north star's "point cloud staged into shared memory by TMA and
// broadcast across a CTA of poses"): cell table, chunk boxes and points (≤ smem_bytes; larger
// clouds fall back to the read-only data path in the same launch). Warps take 32 poses at a time
// from the work counter. A/B variant of k_sdf_grid (-DEXM_SDF_SMEM builds).
template <int KIND, int NB>
__global__ void __launch_bounds__(1024, 1) k_sdf_grid_smem(
    const __grid_constant__ FpDev fp, const float4* __restrict__ poses, int n_poses,
    const GridMeta* __restrict__ gmp, const int* __restrict__ cell_start,
    const float2* __restrict__ cloud, const float4* __restrict__ chunk,
    const float* __restrict__ cap, float thr, int T, int rows, float* __restrict__ out,
    unsigned* __restrict__ work, int smem_bytes) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char s_cloud_mem[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int s_fit;
  __shared__ unsigned s_off[3];
  const int lane = threadIdx.x & 31;
  const GridMeta gm = *gmp;
  if (threadIdx.x == 0) {
    const int cells = gm.n_valid > 0 ? gm.gx * gm.gy : 0;
    const int npad = cells ? cell_start[cells] : 0;
    auto r16 = [](unsigned b) { return (b + 15u) & ~15u; };
    const unsigned b_cell = r16(4u * static_cast<unsigned>(cells + 1));
    const unsigned b_chunk = 16u * static_cast<unsigned>(npad / (gm.chunk > 0 ? gm.chunk : 8));
    const unsigned b_cloud = r16(8u * static_cast<unsigned>(npad));
    s_off[0] = 0;
    s_off[1] = b_cell;
    s_off[2] = b_cell + b_chunk;
    const bool fit = cells > 0 && b_cell + b_chunk + b_cloud <= static_cast<unsigned>(smem_bytes);
    s_fit = fit;
    if (fit) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, b_cell + b_chunk + b_cloud);
      tma_bulk_g2s(s_cloud_mem, cell_start, b_cell, &bar);
      if (b_chunk) tma_bulk_g2s(s_cloud_mem + b_cell, chunk, b_chunk, &bar);
      if (b_cloud) tma_bulk_g2s(s_cloud_mem + b_cell + b_chunk, cloud, b_cloud, &bar);
    }
  }
  __syncthreads();
  const bool fit = s_fit != 0;
  if (fit) mbar_wait(&bar, 0);
  const int* cs = fit ? reinterpret_cast<const int*>(s_cloud_mem) : cell_start;
  const float4* ck = fit ? reinterpret_cast<const float4*>(s_cloud_mem + s_off[1]) : chunk;
  const float2* cl = fit ? reinterpret_cast<const float2*>(s_cloud_mem + s_off[2]) : cloud;
  unsigned long long cnt[kCntN];
  for (;;) {
    unsigned base = 0;
    if (lane == 0) base = atomicAdd(work, 32u);
    base = __shfl_sync(kFull, base, 0);
    if (base >= static_cast<unsigned>(n_poses)) break;
    if (fit)
      sdf_grid_warp<KIND, NB, false, kGridFull, true>(fp, poses, n_poses, gm, cs, cl, ck, cap, thr, T,
                                                      rows, out, static_cast<int>(base) + lane,
                                                      lane, cnt);
    else
      sdf_grid_warp<KIND, NB, false, kGridFull, false>(fp, poses, n_poses, gm, cs, cl, ck, cap, T,
                                                       rows, out, static_cast<int>(base) + lane,
                                                       lane, cnt);
  }
  if (lane == 0) {
    __threadfence();
    const unsigned warps = gridDim.x * (blockDim.x >> 5);
    if (atomicAdd(work + 1, 1u) == warps - 1) {
      work[0] = 0u;
      work[1] = 0u;
      __threadfence();
    }
  }
}

// Warp(s) <-> pose variant for few poses (the T validation poses, small rollout sets). Per ring,
// the lanes first claim cells that pass the box bound, then the W warps of the pose stride
// together over the concatenation of those cells' points (a shuffle search maps a flat index to
// its cell), so the loads coalesce and all lanes stay busy; the minimum over the pose's warps
// after every chunk drives the exact termination. W == 1: four poses per 128-thread CTA;
// W > 1: one pose per CTA of W warps.
template <int KIND, int NB, int W = 1>
__global__ void __launch_bounds__(W == 1 ? 128 : 32 * W) k_sdf_grid_warp(
    const __grid_constant__ FpDev fp, const float4* __restrict__ poses, int n_poses,
    const GridMeta* __restrict__ gmp, const int* __restrict__ cell_start,
    const float2* __restrict__ cloud, float thr, float* __restrict__ out) {
  pdl_wait();
  __shared__ float s_best[W];
  const int lane = threadIdx.x & 31;
  const int wid = W == 1 ? 0 : static_cast<int>(threadIdx.x >> 5);
  const int w = W == 1 ? static_cast<int>((blockIdx.x * blockDim.x + threadIdx.x) >> 5)
                       : static_cast<int>(blockIdx.x);
  if (w >= n_poses) return;  // uniform over the pose's warps
  const GridMeta gm = *gmp;
  if (gm.n_valid == 0) {
    if (lane == 0) out[w] = kEmptyDistance;
    return;
  }
  const float4 q = poses[w];
  const int ci = min(gm.gx - 1, max(0, static_cast<int>(floorf((q.x - gm.x0) * gm.inv_cs))));
  const int cj = min(gm.gy - 1, max(0, static_cast<int>(floorf((q.y - gm.y0) * gm.inv_cs))));
  const float mg = gm.margin;
  const float R = fp.radius + mg;
  float best = thr;  // min(exact minimum, thr)
  const int kmax = max(max(ci, gm.gx - 1 - ci), max(cj, gm.gy - 1 - cj));
  for (int k = 0; k <= kmax; ++k) {
    if (k > 0) {
      const float bx0 = gm.x0 + static_cast<float>(ci - k + 1) * gm.cs;
      const float bx1 = gm.x0 + static_cast<float>(ci + k) * gm.cs;
      const float by0 = gm.y0 + static_cast<float>(cj - k + 1) * gm.cs;
      const float by1 = gm.y0 + static_cast<float>(cj + k) * gm.cs;
      const float lb = fmaxf(fminf(fminf(q.x - bx0, bx1 - q.x), fminf(q.y - by0, by1 - q.y)), 0.f);
      if (!(lb < R + best)) break;  // best is warp-uniform here
    }
    const int ncell = k == 0 ? 1 : 8 * k;
    for (int t0 = 0; t0 < ncell; t0 += 32) {
      const int t = t0 + lane;
      int cnt = 0, st = 0;
      if (t < ncell) {
        int ii, jj;
        ring_cell(k, t, ci, cj, ii, jj);
        if (ii >= 0 && jj >= 0 && ii < gm.gx && jj < gm.gy) {
          const int c = jj * gm.gx + ii;
          const float bx0 = gm.x0 + static_cast<float>(ii) * gm.cs, bx1 = bx0 + gm.cs;
          const float by0 = gm.y0 + static_cast<float>(jj) * gm.cs, by1 = by0 + gm.cs;
          const float gx_ = fmaxf(fmaxf(bx0 - q.x, q.x - bx1), 0.f);
          const float gy_ = fmaxf(fmaxf(by0 - q.y, q.y - by1), 0.f);
          const float lim = R + best;
          if (gx_ * gx_ + gy_ * gy_ < lim * lim) {
            st = __ldg(cell_start + c);
            cnt = __ldg(cell_start + c + 1) - st;
          }
        }
      }
      int incl = cnt;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += v;
      }
      const int total = __shfl_sync(kFull, incl, 31);
      float mine = best;
      for (int b = wid * 32; b < total; b += 32 * W) {
        const int i = b + lane;
        // owner = first lane whose inclusive prefix exceeds i
        int lo = 0;
        for (int step = 16; step; step >>= 1) {
          const int probe = __shfl_sync(kFull, incl, lo + step - 1);
          if (probe <= i) lo += step;
        }
        const int o_incl = __shfl_sync(kFull, incl, lo);
        const int o_cnt = __shfl_sync(kFull, cnt, lo);
        const int o_st = __shfl_sync(kFull, st, lo);
        if (i < total) {
          const float2 o = __ldg(cloud + o_st + (i - (o_incl - o_cnt)));
          const float dx = o.x - q.x, dy = o.y - q.y;
          const float l2 = R + mine;
          if (dx * dx + dy * dy < l2 * l2) {
            const float bx = fmaf(q.z, dx, q.w * dy);
            const float by = fmaf(q.z, dy, -(q.w * dx));
            unsigned wk;
            mine = grid_point<KIND, NB, false>(fp, bx, by, mine, mg, wk);
          }
        }
      }
      for (int o = 16; o; o >>= 1) mine = fminf(mine, __shfl_xor_sync(kFull, mine, o));
      if constexpr (W == 1) {
        best = mine;
      } else {
        if (lane == 0) s_best[wid] = mine;
        __syncthreads();
        float m = s_best[0];
#pragma unroll
        for (int j = 1; j < W; ++j) m = fminf(m, s_best[j]);
        best = m;
        __syncthreads();
      }
    }
  }
  if (lane == 0 && wid == 0) out[w] = best;
}

// Recentring point of a staged pose batch: the poses' centroid, summed in a fixed order by one
// CTA (deterministic), then every pose / point is recentred in FP64 and rounded once.
#if EXM_PART == 0
__global__ void __launch_bounds__(1024) k_pose_center(const double* __restrict__ poses, int n,
                                                      double* __restrict__ center) {
  pdl_wait();
  __shared__ double sx[32], sy[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double x = 0.0, y = 0.0;
  for (int i = tid; i < n; i += blockDim.x) {
    x += poses[3 * static_cast<size_t>(i)];
    y += poses[3 * static_cast<size_t>(i) + 1];
  }
  for (int o = 16; o; o >>= 1) {
    x += __shfl_xor_sync(kFull, x, o);
    y += __shfl_xor_sync(kFull, y, o);
  }
  if (lane == 0) { sx[warp] = x; sy[warp] = y; }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, b = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) { a += sx[w]; b += sy[w]; }
    center[0] = n > 0 ? a / n : 0.0;
    center[1] = n > 0 ? b / n : 0.0;
  }
}

__global__ void k_pose_prep(const double* __restrict__ poses, int n,
                            const double* __restrict__ center, float4* __restrict__ out) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* q = poses + 3 * static_cast<size_t>(i);
  double sn, cs;
  sincos(q[2], &sn, &cs);
  out[i] = make_float4(static_cast<float>(q[0] - center[0]), static_cast<float>(q[1] - center[1]),
                       static_cast<float>(cs), static_cast<float>(sn));
}

__global__ void k_recentre(const double* __restrict__ pts, int n, const double* __restrict__ center,
                           float2* __restrict__ out) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double2 w = reinterpret_cast<const double2*>(pts)[i];
  out[i] = make_float2(static_cast<float>(w.x - center[0]), static_cast<float>(w.y - center[1]));
}
#endif  // EXM_PART == 0

// batch_signed_distance (geometry.cpp:298-318): one body-frame query per thread, FP32 queries
// rounded on the host while they are staged (the identity pose: no recentring).
template <int KIND, int NB>
__global__ void __launch_bounds__(256) k_sdf_points(const __grid_constant__ FpDev fp,
                                                    const float2* __restrict__ q, int n,
                                                    float* __restrict__ out) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float2 p = q[i];
  out[i] = sd_body<KIND, NB>(fp, p.x, p.y);
}

constexpr int kPairThreads = 256;
constexpr int kPairPts = 2;           // points per thread (registers)
constexpr int kPoseChunk = 1024;      // poses staged per TMA bulk copy (16 KB)

// Every point-pose pair (batch_signed_distance semantics per pose). Thread <-> 2 points in
// registers; pose tiles are staged into shared memory by one TMA bulk copy and broadcast.
// Per-pair output per_pair[p*N + i] (coalesced); per-pose min via REDUX + smem atomics.
template <int KIND, int NB>
__global__ void __launch_bounds__(kPairThreads) k_sdf_pairs(
    const __grid_constant__ FpDev fp, const float4* __restrict__ poses, int n_poses,
    const float2* __restrict__ pts, const uint8_t* __restrict__ mask, int n_points,
    float* __restrict__ per_pair, unsigned* __restrict__ pose_min_key) {
  pdl_wait();
  __shared__ __align__(128) float4 s_pose[kPoseChunk];
  __shared__ unsigned s_min[kPoseChunk];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int base = blockIdx.x * (kPairThreads * kPairPts);
  float px[kPairPts], py[kPairPts];
  bool ok[kPairPts];
#pragma unroll
  for (int k = 0; k < kPairPts; ++k) {
    const int i = base + k * kPairThreads + tid;
    ok[k] = i < n_points && (mask == nullptr || mask[i] != 0);
    const float2 p = i < n_points ? pts[i] : make_float2(0.f, 0.f);
    px[k] = p.x;
    py[k] = p.y;
  }
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  unsigned phase = 0;
  for (int p0 = 0; p0 < n_poses; p0 += kPoseChunk) {
    const int np = min(kPoseChunk, n_poses - p0);
    if (tid == 0) {
      const unsigned bytes = static_cast<unsigned>(np) * sizeof(float4);
      mbar_expect_tx(&bar, bytes);
      tma_bulk_g2s(s_pose, poses + p0, bytes, &bar);
    }
    for (int j = tid; j < np; j += kPairThreads) s_min[j] = 0xffffffffu;
    mbar_wait(&bar, phase);
    phase ^= 1u;
    __syncthreads();
    for (int j = 0; j < np; ++j) {
      const float4 q = s_pose[j];
      unsigned key = 0xffffffffu;
#pragma unroll
      for (int k = 0; k < kPairPts; ++k) {
        const float dx = px[k] - q.x, dy = py[k] - q.y;
        const float bx = fmaf(q.z, dx, q.w * dy);
        const float by = fmaf(q.z, dy, -(q.w * dx));
        float v = sd_body<KIND, NB>(fp, bx, by);
        v = ok[k] ? v : __int_as_float(0x7f800000);
        const int i = base + k * kPairThreads + tid;
        if (per_pair && i < n_points) per_pair[static_cast<size_t>(p0 + j) * n_points + i] = v;
        key = min(key, fkey(v));
      }
      if (pose_min_key) {
        key = __reduce_min_sync(kFull, key);
        if (lane == 0) atomicMin(&s_min[j], key);
      }
    }
    __syncthreads();
    if (pose_min_key)
      for (int j = tid; j < np; j += kPairThreads) atomicMin(&pose_min_key[p0 + j], s_min[j]);
    __syncthreads();
  }
}

// One polygon edge against two body-frame points packed in f32x2 lanes (same arithmetic as
// poly_edge, two pairs per FFMA2/FADD2/FMUL2). Per pair: 8 FP32 ops for the distance, 2 for
// the crossing product (CROSS), the clamp as scalar FFMA.SAT (no .sat form of FFMA2).
// Returns the packed squared distances; the caller folds two edges per FMNMX3.
template <bool CROSS>
__device__ __forceinline__ u64 poly_edge2(const float* e, float vy_next, u64 X, u64 Y, u64& RY,
                                          unsigned& pA, unsigned& pB) {
  const u64 TP = fma2(Y, bc(e[5]), bc(e[6]));
  const u64 Tt = pk(__saturatef(fmaf(lo(X), e[4], lo(TP))), __saturatef(fmaf(hi(X), e[4], hi(TP))));
  const u64 RX = sub2(bc(e[0]), X);
  const u64 QX = fma2(Tt, bc(e[2]), RX);
  const u64 QY = fma2(Tt, bc(e[3]), RY);
  const u64 D2 = fma2(QY, QY, mul2(QX, QX));
  const u64 RYN = sub2(bc(vy_next), Y);
  if constexpr (CROSS) {
    const u64 CR = fma2(RY, bc(e[7]), mul2(RX, bc(e[3])));
    pA ^= (sgn_lo(RY) ^ sgn_lo(RYN)) & (sgn_lo(RY) ^ sgn_lo(CR));
    pB ^= (sgn_hi(RY) ^ sgn_hi(RYN)) & (sgn_hi(RY) ^ sgn_hi(CR));
  }
  RY = RYN;
  return D2;
}

template <int NB, bool CROSS>
__device__ __forceinline__ void poly_pairs4(const FpDev& fp, u64 X01, u64 Y01, u64 X23, u64 Y23,
                                            float* b, unsigned* par) {
  // Edge groups of kEdgeGroup with a rolled outer loop: the per-edge constants stay uniform
  // (LDCU from the parameter bank at a uniform offset) while the code stays small enough for
  // the instruction cache at B = 64.
  // The distance-only pass (most pose-warps) is fully unrolled: every edge constant is an
  // immediate constant-bank/uniform operand. The rarer crossing pass keeps a rolled outer loop
  // so both together stay inside the instruction cache at B = 64.
  constexpr int G = CROSS ? (NB % 4 == 0 ? 4 : 2) : (NB / 2) * 2;
  const float vy0 = fp.e[0][1];
  u64 R01 = sub2(bc(vy0), Y01), R23 = sub2(bc(vy0), Y23);
  constexpr int NFULL = G > 0 ? (NB / G) * G : 0;
#pragma unroll 1
  for (int g = 0; g < NFULL; g += G) {
#pragma unroll
    for (int j = 0; j < G; j += 2) {
      const int e = g + j;
      const float vy1 = fp.e[e + 1][1];
      const float vy2 = e + 2 < NB ? fp.e[e + 2][1] : vy0;
      const u64 a01 = poly_edge2<CROSS>(fp.e[e], vy1, X01, Y01, R01, par[0], par[1]);
      const u64 a23 = poly_edge2<CROSS>(fp.e[e], vy1, X23, Y23, R23, par[2], par[3]);
      const u64 c01 = poly_edge2<CROSS>(fp.e[e + 1], vy2, X01, Y01, R01, par[0], par[1]);
      const u64 c23 = poly_edge2<CROSS>(fp.e[e + 1], vy2, X23, Y23, R23, par[2], par[3]);
      b[0] = min3f(b[0], lo(a01), lo(c01));
      b[1] = min3f(b[1], hi(a01), hi(c01));
      b[2] = min3f(b[2], lo(a23), lo(c23));
      b[3] = min3f(b[3], hi(a23), hi(c23));
    }
  }
#pragma unroll
  for (int e = NFULL; e < NB; ++e) {
    const float vyn = e + 1 < NB ? fp.e[e + 1][1] : vy0;
    const u64 a01 = poly_edge2<CROSS>(fp.e[e], vyn, X01, Y01, R01, par[0], par[1]);
    const u64 a23 = poly_edge2<CROSS>(fp.e[e], vyn, X23, Y23, R23, par[2], par[3]);
    b[0] = fminf(b[0], lo(a01));
    b[1] = fminf(b[1], hi(a01));
    b[2] = fminf(b[2], lo(a23));
    b[3] = fminf(b[3], hi(a23));
  }
}

constexpr int kPackPts = 4;  // points per thread (two f32x2 packs)

// Every point-pose pair for a polygon footprint, packed: thread <-> 4 points held in
// registers as two f32x2 packs, pose tiles staged into shared memory by one TMA bulk copy
// and broadcast. The crossing-number pass runs only for (pose, warp) tiles where some point
// lies inside the footprint's body-frame AABB: outside it no edge can count an odd number of
// crossings, so skipping is exact.
template <int NB>
__global__ void __launch_bounds__(kPairThreads, 2) k_sdf_pairs_poly(
    const __grid_constant__ FpDev fp, const float4* __restrict__ poses, int n_poses,
    const float2* __restrict__ pts, const uint8_t* __restrict__ mask, int n_points,
    float* __restrict__ per_pair, unsigned* __restrict__ pose_min_key) {
  pdl_wait();
  __shared__ __align__(128) float4 s_pose[kPoseChunk];
  __shared__ unsigned s_min[kPoseChunk];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid & 31;
  const int base = blockIdx.x * (kPairThreads * kPackPts);
  float px[kPackPts], py[kPackPts];
  bool ok[kPackPts];
#pragma unroll
  for (int k = 0; k < kPackPts; ++k) {
    const int i = base + k * kPairThreads + tid;
    ok[k] = i < n_points && (mask == nullptr || mask[i] != 0);
    const float2 p = i < n_points ? pts[i] : make_float2(0.f, 0.f);
    px[k] = p.x;
    py[k] = p.y;
  }
  const u64 PX01 = pk(px[0], px[1]), PY01 = pk(py[0], py[1]);
  const u64 PX23 = pk(px[2], px[3]), PY23 = pk(py[2], py[3]);
  const float ax0 = fp.aabb[0], ax1 = fp.aabb[1], ay0 = fp.aabb[2], ay1 = fp.aabb[3];
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  unsigned phase = 0;
  for (int p0 = 0; p0 < n_poses; p0 += kPoseChunk) {
    const int np = min(kPoseChunk, n_poses - p0);
    if (tid == 0) {
      const unsigned bytes = static_cast<unsigned>(np) * sizeof(float4);
      mbar_expect_tx(&bar, bytes);
      tma_bulk_g2s(s_pose, poses + p0, bytes, &bar);
    }
    for (int j = tid; j < np; j += kPairThreads) s_min[j] = 0xffffffffu;
    mbar_wait(&bar, phase);
    phase ^= 1u;
    __syncthreads();
    for (int j = 0; j < np; ++j) {
      const float4 q = s_pose[j];
      // body frame: b = R(theta)^T (o - t)
      const u64 DX01 = sub2(PX01, bc(q.x)), DY01 = sub2(PY01, bc(q.y));
      const u64 DX23 = sub2(PX23, bc(q.x)), DY23 = sub2(PY23, bc(q.y));
      const float ns = -q.w;
      const u64 X01 = fma2(DX01, bc(q.z), mul2(DY01, bc(q.w)));
      const u64 Y01 = fma2(DY01, bc(q.z), mul2(DX01, bc(ns)));
      const u64 X23 = fma2(DX23, bc(q.z), mul2(DY23, bc(q.w)));
      const u64 Y23 = fma2(DY23, bc(q.z), mul2(DX23, bc(ns)));
      const float bx[4] = {lo(X01), hi(X01), lo(X23), hi(X23)};
      const float by[4] = {lo(Y01), hi(Y01), lo(Y23), hi(Y23)};
      bool in = false;
#pragma unroll
      for (int k = 0; k < kPackPts; ++k)
        in |= bx[k] >= ax0 && bx[k] <= ax1 && by[k] >= ay0 && by[k] <= ay1;
      float b[4] = {__int_as_float(0x7f800000), __int_as_float(0x7f800000),
                    __int_as_float(0x7f800000), __int_as_float(0x7f800000)};
      unsigned par[4] = {0u, 0u, 0u, 0u};
      if (__any_sync(kFull, in)) poly_pairs4<NB, true>(fp, X01, Y01, X23, Y23, b, par);
      else poly_pairs4<NB, false>(fp, X01, Y01, X23, Y23, b, par);
      unsigned key = 0xffffffffu;
#pragma unroll
      for (int k = 0; k < kPackPts; ++k) {
        const float d2 = b[k] < 1e-24f ? 0.0f : b[k];
        const bool inside = (par[k] >> 31) != 0;
        if (per_pair) {
          const int i = base + k * kPairThreads + tid;
          float v = sqrtf(d2);
          v = inside ? -v : v;
          if (i < n_points) per_pair[static_cast<size_t>(p0 + j) * n_points + i] = ok[k] ? v : __int_as_float(0x7f800000);
        }
        // order by the signed square (same order as sd; one sqrt per pose below)
        const float s2 = ok[k] ? (inside ? -d2 : d2) : __int_as_float(0x7f800000);
        key = min(key, fkey(s2));
      }
      if (pose_min_key) {
        key = __reduce_min_sync(kFull, key);
        if (lane == 0) {
          const float s2 = unkey(key);
          const float d = isinf(s2) ? s2 : copysignf(sqrtf(fabsf(s2)), s2);
          atomicMin(&s_min[j], fkey(d));
        }
      }
    }
    __syncthreads();
    if (pose_min_key)
      for (int j = tid; j < np; j += kPairThreads) atomicMin(&pose_min_key[p0 + j], s_min[j]);
    __syncthreads();
  }
}

#if EXM_PART == 0
__global__ void k_keys_to_double(const unsigned* __restrict__ keys, int n,
                                 double* __restrict__ out) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const float v = unkey(keys[i]);
  out[i] = isinf(v) ? static_cast<double>(kEmptyDistance) : static_cast<double>(v);
}

__global__ void k_fill_u32(unsigned* p, unsigned v, int n) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}
#endif  // EXM_PART == 0

// ------------------------------------------------------------------ dispatch
// (kind, edge count) -> instantiation index; the part that instantiates it is index % EXM_NPARTS.
__host__ __device__ constexpr int combo_index(int kind, int count) {
  if (kind == EXM_FOOTPRINT_POLYGON) {
    switch (count) {
      case 3: return 0;
      case 4: return 1;
      case 5: return 2;
      case 6: return 3;
      case 7: return 4;
      case 8: return 5;
      case 10: return 6;
      case 12: return 7;
      case 16: return 8;
      case 32: return 9;
      case 64: return 10;
      default: return 11;
    }
  }
  switch (count) {
    case 1: return 12;
    case 2: return 13;
    case 3: return 14;
    case 4: return 15;
    default: return 16;
  }
}

template <template <int, int> class Launch, int KIND, int NB, typename... Args>
cudaError_t run_combo(const FpDev& fp, Args&&... args) {
  if constexpr (combo_index(KIND, NB) % EXM_NPARTS == EXM_PART)
    return Launch<KIND, NB>::run(fp, args...);
  else
    return cudaErrorInvalidValue;  // instantiated by another part: the launchers route there
}

template <template <int, int> class Launch, typename... Args>
cudaError_t dispatch_fp(const FpDev& fp, Args&&... args) {
  constexpr int P = EXM_FOOTPRINT_POLYGON, R = EXM_FOOTPRINT_RECT_COVER;
  if (fp.kind == EXM_FOOTPRINT_POLYGON) {
    switch (fp.count) {
      case 3: return run_combo<Launch, P, 3>(fp, args...);
      case 4: return run_combo<Launch, P, 4>(fp, args...);
      case 5: return run_combo<Launch, P, 5>(fp, args...);
      case 6: return run_combo<Launch, P, 6>(fp, args...);
      case 7: return run_combo<Launch, P, 7>(fp, args...);
      case 8: return run_combo<Launch, P, 8>(fp, args...);
      case 10: return run_combo<Launch, P, 10>(fp, args...);
      case 12: return run_combo<Launch, P, 12>(fp, args...);
      case 16: return run_combo<Launch, P, 16>(fp, args...);
      case 32: return run_combo<Launch, P, 32>(fp, args...);
      case 64: return run_combo<Launch, P, 64>(fp, args...);
      default: return run_combo<Launch, P, 0>(fp, args...);
    }
  }
  switch (fp.count) {
    case 1: return run_combo<Launch, R, 1>(fp, args...);
    case 2: return run_combo<Launch, R, 2>(fp, args...);
    case 3: return run_combo<Launch, R, 3>(fp, args...);
    case 4: return run_combo<Launch, R, 4>(fp, args...);
    default: return run_combo<Launch, R, 0>(fp, args...);
  }
}

// Persistent grid size of a k_sdf_grid instantiation on the current device: resident CTAs per
// SM x SMs (cached per device and instantiation).
template <typename K>
int persistent_blocks(K kernel, int threads) {
  constexpr int kMaxDev = 64;
  static int blocks[kMaxDev] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) dev = 0;
  if (blocks[dev] == 0) {
    int n_sm = 148, per_sm = 1;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, 0) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    blocks[dev] = n_sm * per_sm;
  }
  return blocks[dev];
}

#ifdef EXM_PERSIST_WAVES  // A/B builds
constexpr int kPersistentWaves = EXM_PERSIST_WAVES;
#else
constexpr int kPersistentWaves = 8;
#endif
constexpr int kGridThreads = EXM_GRID_THREADS;

template <int KIND, int NB, bool STATS, int MODE>
cudaError_t launch_grid_kernel(const FpDev& fp, const float4* poses, int n_poses, int T,
                               bool hmajor, const CloudGrid& g, const float* cap, float thr,
                               bool persist, float* out,
                               SdfPath* path, unsigned long long* stats, cudaStream_t s) {
  const int threads = kGridThreads;
  const int blocks = (n_poses + threads - 1) / threads;
  auto k = k_sdf_grid<KIND, NB, STATS, MODE>;
  // persistent only for many waves (cfg5: ~30): at one to three waves the hardware block
  // scheduler balances as well and the static mapping keeps neighbouring poses in one CTA
  // (measured: cfg2 / cfg3 slower persistent, cfg5 2.5 % faster)
  const int cap_blocks = persistent_blocks(k, threads);
  unsigned* work = (persist || blocks >= kPersistentWaves * cap_blocks) ? g.work : nullptr;
  const int grid = work ? cap_blocks : blocks;
  const int rows_used = (hmajor && T > 0 && n_poses % T == 0) ? n_poses / T : 0;
#ifdef EXM_SDF_SMEM
  if constexpr (!STATS && MODE == kGridFull) {
    constexpr int kSmem = 220 * 1024;
    auto ks = k_sdf_grid_smem<KIND, NB>;
    cudaError_t e = cudaFuncSetAttribute(ks, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem);
    if (e != cudaSuccess) return e;
    int dev = 0, n_sm = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (path) *path = SdfPath{0, 0, 1, n_sm, 1024, rows_used > 0 ? 1 : 0};
    if (const cudaError_t le = launch_k(ks, n_sm, 1024, kSmem, s, fp, poses, n_poses, g.gm,
                                        g.cell_start, g.cloud, g.chunk, cap, thr, T, rows_used, out,
                                        g.work, kSmem);
        le != cudaSuccess)
      return le;
    return cudaGetLastError();
  }
#endif
  if (path) *path = SdfPath{0, 0, work ? 1 : 0, grid, threads, rows_used > 0 ? 1 : 0};
  if (const cudaError_t le = launch_k(k, grid, threads, 0, s, fp, poses, n_poses, g.gm,
                                      g.cell_start, g.cloud, g.chunk, cap, thr, T, rows_used, out,
                                      work, stats);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

template <int KIND, int NB>
struct GridLaunch {
  static cudaError_t run(const FpDev& fp, const float4* poses, int n_poses, int T, bool hmajor,
                         const CloudGrid& g, const float* cap, float thr, int mode, float* out,
                         SdfPath* path, unsigned long long* stats, cudaStream_t s) {
    if (n_poses <= 0) return cudaSuccess;
    const bool persist = mode == kSdfPersist;
    if (mode == kSdfNoCap) cap = nullptr;
    if (stats) {
      if (mode == kSdfNoChunk)
        return launch_grid_kernel<KIND, NB, true, kGridNoChunk>(fp, poses, n_poses, T, hmajor, g, cap, thr, persist, out, path, stats, s);
      return launch_grid_kernel<KIND, NB, true, kGridFull>(fp, poses, n_poses, T, hmajor, g, cap, thr, persist, out, path, stats, s);
    }
    if (mode == kSdfBrute)
      return launch_grid_kernel<KIND, NB, false, kGridBrute>(fp, poses, n_poses, T, hmajor, g, cap, thr, persist, out, path, nullptr, s);
    if (mode == kSdfNoChunk)
      return launch_grid_kernel<KIND, NB, false, kGridNoChunk>(fp, poses, n_poses, T, hmajor, g, cap, thr, persist, out, path, nullptr, s);
    return launch_grid_kernel<KIND, NB, false, kGridFull>(fp, poses, n_poses, T, hmajor, g, cap, thr, persist, out, path, nullptr, s);
  }
};

template <int KIND, int NB>
struct GridWarpLaunch {
  static cudaError_t run(const FpDev& fp, const float4* poses, int n_poses, const CloudGrid& g,
                         bool cta, float thr, float* out, SdfPath* path, cudaStream_t s) {
    if (n_poses <= 0) return cudaSuccess;
    if (n_poses <= kCtaPerPoseMax || cta) {  // few poses: 8 warps each
      if (path) *path = SdfPath{2, 0, 0, n_poses, 256, 0};
      if (const cudaError_t le = launch_k(k_sdf_grid_warp<KIND, NB, 8>, n_poses, 256, 0, s, fp,
                                          poses, n_poses, g.gm, g.cell_start, g.cloud, thr, out);
          le != cudaSuccess)
        return le;
    } else {
      const int threads = 128, warps = threads / 32, grid = (n_poses + warps - 1) / warps;
      if (path) *path = SdfPath{1, 0, 0, grid, threads, 0};
      if (const cudaError_t le = launch_k(k_sdf_grid_warp<KIND, NB>, grid, threads, 0, s, fp,
                                          poses, n_poses, g.gm, g.cell_start, g.cloud, thr, out);
          le != cudaSuccess)
        return le;
    }
    return cudaGetLastError();
  }
};

template <int KIND, int NB>
struct PairsLaunch {
  static cudaError_t run(const FpDev& fp, const float4* poses, int n_poses, const float2* pts,
                         const uint8_t* mask, int n_points, float* per_pair, unsigned* keys,
                         cudaStream_t s) {
    if (n_poses <= 0 || n_points <= 0) return cudaSuccess;
    if constexpr (KIND == EXM_FOOTPRINT_POLYGON && NB > 0) {
      const int per_block = kPairThreads * kPackPts;
      { if (const cudaError_t le = launch_k(k_sdf_pairs_poly<NB>, (n_points + per_block - 1) / per_block, kPairThreads, 0, s, 
          fp, poses, n_poses, pts, mask, n_points, per_pair, keys); le != cudaSuccess) return le; }
    } else {
      const int per_block = kPairThreads * kPairPts;
      { if (const cudaError_t le = launch_k(k_sdf_pairs<KIND, NB>, (n_points + per_block - 1) / per_block, kPairThreads, 0, s, 
          fp, poses, n_poses, pts, mask, n_points, per_pair, keys); le != cudaSuccess) return le; }
    }
    return cudaGetLastError();
  }
};

}  // namespace

// ------------------------------------------------------------------ launchers
template <int KIND, int NB>
struct PointsLaunch {
  static cudaError_t run(const FpDev& fp, const float2* q, int n, float* out, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    if (const cudaError_t le = launch_k(k_sdf_points<KIND, NB>, (n + 255) / 256, 256, 0, s, fp,
                                        q, n, out);
        le != cudaSuccess)
      return le;
    return cudaGetLastError();
  }
};

// This part's share of the signed-distance launchers (named per part: sdf_*_p<k>).
#define EXM_PASTE2(a, b) a##b
#define EXM_PASTE(a, b) EXM_PASTE2(a, b)
#define EXM_PART_FNS(k)                                                                          \
  cudaError_t EXM_PASTE(sdf_grid_p, k)(const FpDev& fp, const float4* poses, int n_poses, int T,  \
                                       bool hmajor, const CloudGrid& g, const float* cap,         \
                                       float thr, int mode, bool warp, float* out, SdfPath* path, \
                                       unsigned long long* stats, cudaStream_t s);                \
  cudaError_t EXM_PASTE(sdf_points_p, k)(const FpDev& fp, const float2* q, int n, float* out,     \
                                         cudaStream_t s);                                         \
  cudaError_t EXM_PASTE(sdf_pairs_p, k)(const FpDev& fp, const float4* poses, int n_poses,        \
                                        const float2* pts, const uint8_t* mask, int n_points,     \
                                        float* per_pair, unsigned* pose_min_key, cudaStream_t s);
EXM_PART_FNS(EXM_PART)

cudaError_t EXM_PASTE(sdf_grid_p, EXM_PART)(const FpDev& fp, const float4* poses, int n_poses,
                                            int T, bool hmajor, const CloudGrid& g,
                                            const float* cap, float thr, int mode, bool warp,
                                            float* out, SdfPath* path, unsigned long long* stats,
                                            cudaStream_t s) {
  if (warp) return dispatch_fp<GridWarpLaunch>(fp, poses, n_poses, g, mode == kSdfCta, thr, out, path, s);
  return dispatch_fp<GridLaunch>(fp, poses, n_poses, T, hmajor, g, cap, thr, mode, out, path, stats, s);
}

cudaError_t EXM_PASTE(sdf_points_p, EXM_PART)(const FpDev& fp, const float2* q, int n, float* out,
                                              cudaStream_t s) {
  return dispatch_fp<PointsLaunch>(fp, q, n, out, s);
}

cudaError_t EXM_PASTE(sdf_pairs_p, EXM_PART)(const FpDev& fp, const float4* poses, int n_poses,
                                             const float2* pts, const uint8_t* mask, int n_points,
                                             float* per_pair, unsigned* pose_min_key,
                                             cudaStream_t s) {
  return dispatch_fp<PairsLaunch>(fp, poses, n_poses, pts, mask, n_points, per_pair,
                                  pose_min_key, s);
}

#if EXM_PART == 0
#if EXM_NPARTS > 1
EXM_PART_FNS(1)
#endif
#if EXM_NPARTS > 2
EXM_PART_FNS(2)
#endif
#if EXM_NPARTS > 3
EXM_PART_FNS(3)
#endif
// Route a footprint to the part that instantiated its kernels.
#if EXM_NPARTS > 3
#define EXM_ROUTE(fn, ...)                                                        \
  switch (combo_index(fp.kind, fp.count) % EXM_NPARTS) {                         \
    case 1: return EXM_PASTE(fn, 1)(__VA_ARGS__);                                \
    case 2: return EXM_PASTE(fn, 2)(__VA_ARGS__);                                \
    case 3: return EXM_PASTE(fn, 3)(__VA_ARGS__);                                \
    default: return EXM_PASTE(fn, 0)(__VA_ARGS__);                               \
  }
#elif EXM_NPARTS > 2
#define EXM_ROUTE(fn, ...)                                                        \
  switch (combo_index(fp.kind, fp.count) % EXM_NPARTS) {                         \
    case 1: return EXM_PASTE(fn, 1)(__VA_ARGS__);                                \
    case 2: return EXM_PASTE(fn, 2)(__VA_ARGS__);                                \
    default: return EXM_PASTE(fn, 0)(__VA_ARGS__);                               \
  }
#elif EXM_NPARTS > 1
#define EXM_ROUTE(fn, ...)                                                        \
  switch (combo_index(fp.kind, fp.count) % EXM_NPARTS) {                         \
    case 1: return EXM_PASTE(fn, 1)(__VA_ARGS__);                                \
    default: return EXM_PASTE(fn, 0)(__VA_ARGS__);                               \
  }
#else
#define EXM_ROUTE(fn, ...) return EXM_PASTE(fn, 0)(__VA_ARGS__);
#endif

// Chunk size per handle: 16-point chunks measured 10 % faster on the 20k / 50k-point aisle and
// moving-disc clouds (configs 3, 5), 6 % slower on config 2's 10k clutter points.
int chunk_for_capacity(int n_cap) {
#ifdef EXM_CHUNK
  return EXM_CHUNK;  // A/B builds
#else
  return n_cap >= 16384 ? 16 : 8;
#endif
}

cudaError_t launch_cloud_prep(const double* pts, const uint8_t* mask, const StepDyn* dyn,
                              float radius, const CloudGrid& g, int n_cap, cudaStream_t s) {
  // (A one-cluster version — 8 CTAs meeting through distributed shared memory, cell sort fused —
  // measured 20.9 us against 13.6 + 5.9 us for config 2: the cluster barriers cost what the
  // parallel load saves at 10k points. The single CTA stays.)
  const int smem = kGridMax * kGridMax * static_cast<int>(sizeof(int));
  // (cudaFuncSetAttribute applies to the current device: set it on every launch, it is cheap
  // and launches are captured into graphs anyway)
  cudaError_t e = cudaFuncSetAttribute(k_cloud_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  // Cells sized for about kPtsPerCell points, between kCellMinR * R and kCellMaxR * R: a cull
  // disc of radius R + d covers ~(2(R+d)/cs)^2 cells; the chunk bounds cull inside a cell.
  // The cloud is bulk-prefetched into L2 first (cfg2 0.193 -> 0.188 ms after an L2 flush).
  const float r = fmaxf(radius, 0.04f);
  if (const cudaError_t le = launch_k(k_cloud_prep, 1, 1024, smem, s, pts, mask, dyn, kCellMinR * r,
                                      kCellMaxR * r, kPtsPerCell, r, chunk_for_capacity(n_cap),
                                      0.0f, 1, g.dstat, g.tmp, g.raw, g.raw_start, g.cell_start,
                                      g.gm);
      le != cudaSuccess)
    return le;
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  int dev = 0, n_sm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess)
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
  if (const cudaError_t le = launch_k(k_cell_sort, 2 * n_sm, kSortWarps * 32, 0, s, g.raw,
                                      g.raw_start, g.cell_start, g.gm, g.cloud, g.chunk);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

cudaError_t launch_sdf_grid(const FpDev& fp, const float4* poses, int n_poses, int T, bool hmajor,
                            const CloudGrid& g, const float* cap, int mode, float* out,
                            SdfPath* path, unsigned long long* stats, cudaStream_t s, float thr) {
  // Few poses (validation rollout, single queries): one warp (or one 8-warp CTA) per pose keeps
  // all lanes busy; many poses: one thread per pose. Statistics builds exist for the latter.
  const bool warp = !stats && (mode == kSdfWarp || mode == kSdfCta ||
                               (n_poses <= kWarpPerPoseMax && mode != kSdfThread &&
                                mode != kSdfBrute && mode != kSdfPersist));
  EXM_ROUTE(sdf_grid_p, fp, poses, n_poses, T, hmajor, g, cap, thr, mode, warp, out, path, stats, s)
}

cudaError_t launch_pose_prep(const double* poses, int n, double* center, float4* out,
                             cudaStream_t s) {
  if (const cudaError_t le = launch_k(k_pose_center, 1, 1024, 0, s, poses, n, center);
      le != cudaSuccess)
    return le;
  if (n > 0)
    if (const cudaError_t le = launch_k(k_pose_prep, (n + 255) / 256, 256, 0, s, poses, n,
                                        static_cast<const double*>(center), out);
        le != cudaSuccess)
      return le;
  return cudaGetLastError();
}

cudaError_t launch_recentre(const double* pts, int n, const double* center, float2* out,
                            cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (const cudaError_t le = launch_k(k_recentre, (n + 255) / 256, 256, 0, s, pts, n, center, out);
      le != cudaSuccess)
    return le;
  return cudaGetLastError();
}

cudaError_t launch_sdf_points(const FpDev& fp, const float2* q, int n, float* out, cudaStream_t s) {
  EXM_ROUTE(sdf_points_p, fp, q, n, out, s)
}

cudaError_t launch_sdf_pairs(const FpDev& fp, const float4* poses, int n_poses,
                             const float2* pts, const uint8_t* mask, int n_points,
                             float* per_pair, unsigned* pose_min_key, cudaStream_t s) {
  EXM_ROUTE(sdf_pairs_p, fp, poses, n_poses, pts, mask, n_points, per_pair, pose_min_key, s)
}

cudaError_t launch_min_keys_to_double(const unsigned* keys, int n, double* out, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  { if (const cudaError_t le = launch_k(k_keys_to_double, (n + 255) / 256, 256, 0, s, keys, n, out); le != cudaSuccess) return le; }
  return cudaGetLastError();
}

cudaError_t launch_fill_u32(unsigned* p, unsigned v, int n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  { if (const cudaError_t le = launch_k(k_fill_u32, (n + 255) / 256, 256, 0, s, p, v, n); le != cudaSuccess) return le; }
  return cudaGetLastError();
}
#endif  // EXM_PART == 0

}  // namespace exm
