// geometry_sdf_b200.cpp — link-time drop-in for the reference's batch_signed_distance
// (proj/include/exactmppi/geometry.hpp:142-143, proj/src/geometry.cpp:298-318) on the B200.
//
// geometry.cpp holds the whole footprint library (validation, prepare, sd, transforms), so it
// stays linked as it is; only calls of batch_signed_distance from the OTHER translation units
// (scaling_benchmark, proj/src/bench.cpp:86 and :91; acceptance criterion 3,
// proj/tests/acceptance_main.cpp:134-174) are redirected here with the GNU linker's symbol
// wrapping:
//
//   g++ ... geometry_sdf_b200.cpp -Wl,--wrap=<mangled batch_signed_distance> -lexm_b200
//
// (the mangled name is EXM_BSD_MANGLED below; host/Makefile passes the same string).
//
// Semantics kept: the size check and its exception text (geometry.cpp:300), `threads` (here the
// host threads that stage FP64 queries to FP32 and widen the results back; <= 1: one thread),
// out[i] = signed distance of query i in the body frame. Values are FP64 in the reference's own
// arithmetic (EXM_OPT_SDF_FP64, csrc/exm_exact64.cu: the reference's 1e-12 batch-vs-scalar
// tests hold, proj/tests/test_geometry.cpp:307-320); EXM_DROPIN_SDF_FP32=1 selects the FP32
// kernel instead (within the north-star 1e-5 max(|d_ref|, 1 m); 8 B instead of 16 B per query
// on the link).
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "exactmppi/geometry.hpp"
#include "exm_b200.h"

#define EXM_BSD_MANGLED \
  "_ZN9exactmppi21batch_signed_distanceESt4spanIKNS_6Point2ELm18446744073709551615EERKNS_17PreparedFootprintES0_IdLm18446744073709551615EEi"

namespace exactmppi {

void b200_batch_signed_distance(std::span<const Point2> queries, const PreparedFootprint& footprint,
                                std::span<double> out, int threads)
    __asm__("__wrap_" EXM_BSD_MANGLED);

namespace {

struct SdfHandle {
  exm_handle* h = nullptr;
  int threads = -1;  // EXM_OPT_HOST_THREADS last set
  std::mutex mu;  // one call at a time per handle (the handle also locks; this guards options)
  ~SdfHandle() {
    if (h) exm_destroy(h);
  }
};

std::mutex g_mu;
std::map<std::string, std::unique_ptr<SdfHandle>> g_handles;

// Exact byte key of the prepared footprint's geometry (no formatting: no collisions).
std::string footprint_key(const PreparedFootprint& f) {
  std::string k(1, f.kind == PreparedFootprint::Kind::kPolygon ? 'P' : 'R');
  auto add = [&](const std::vector<double>& v) {
    const std::size_t n = v.size();
    k.append(reinterpret_cast<const char*>(&n), sizeof n);
    k.append(reinterpret_cast<const char*>(v.data()), n * sizeof(double));
  };
  if (f.kind == PreparedFootprint::Kind::kPolygon) {
    add(f.vx);
    add(f.vy);
  } else {
    add(f.cx);
    add(f.cy);
    add(f.hx);
    add(f.hy);
  }
  return k;
}

SdfHandle* handle_for(const PreparedFootprint& f) {
  const std::string key = footprint_key(f);
  std::lock_guard<std::mutex> lock(g_mu);
  auto& slot = g_handles[key];
  if (slot) return slot.get();
  auto s = std::make_unique<SdfHandle>();
  exm_footprint fp{};
  if (f.kind == PreparedFootprint::Kind::kPolygon) {
    fp.kind = EXM_FOOTPRINT_POLYGON;
    fp.count = static_cast<int32_t>(f.vx.size());
    fp.x = f.vx.data();  // prepare() keeps the CCW vertices as edge origins (geometry.cpp:241-242)
    fp.y = f.vy.data();
  } else {
    fp.kind = EXM_FOOTPRINT_RECT_COVER;
    fp.count = static_cast<int32_t>(f.cx.size());
    fp.x = f.cx.data();
    fp.y = f.cy.data();
    fp.hx = f.hx.data();
    fp.hy = f.hy.data();
  }
  // a signed-distance-only handle: the smallest rollout configuration
  exm_model m{};
  m.tag = EXM_MODEL_DIFF;
  exm_limits l{};
  for (int i = 0; i < 3; ++i) {
    l.vel_min[i] = -1.0;
    l.vel_max[i] = 1.0;
    l.acc_min[i] = -1e9;
    l.acc_max[i] = 1e9;
  }
  l.steer_max = 0.6;
  exm_params p{};
  p.rollouts = 1;
  p.horizon = 1;
  p.dt = 0.1;
  p.lambda = 1.0;
  p.sigma[0] = p.sigma[1] = p.sigma[2] = 0.3;
  exm_status st = exm_create(&fp, &m, &l, &p, 1, 1, -1, &s->h);
  if (st == EXM_OK) {
    const char* e = std::getenv("EXM_DROPIN_SDF_FP32");
    st = exm_set_option(s->h, EXM_OPT_SDF_FP64, (e && *e == '1') ? 0 : 1);
  }
  if (st != EXM_OK) {
    if (st == EXM_ERR_INVALID_ARGUMENT) throw std::invalid_argument(exm_last_error());
    throw std::runtime_error(std::string("exm_b200: ") + exm_last_error());
  }
  slot = std::move(s);
  return slot.get();
}

}  // namespace

void b200_batch_signed_distance(std::span<const Point2> queries, const PreparedFootprint& footprint,
                                std::span<double> out, int threads) {
  if (out.size() != queries.size()) throw std::invalid_argument("output span size mismatch");
  if (queries.empty()) return;
  SdfHandle* s = handle_for(footprint);
  std::lock_guard<std::mutex> lock(s->mu);
  static_assert(sizeof(Point2) == 2 * sizeof(double), "Point2 is {x, y} doubles");
  exm_status st = EXM_OK;
  if (s->threads != (threads < 1 ? 1 : threads)) {
    st = exm_set_option(s->h, EXM_OPT_HOST_THREADS, threads < 1 ? 1 : threads);
    s->threads = threads < 1 ? 1 : threads;
  }
  if (st == EXM_OK)
    st = exm_batch_signed_distance(s->h, reinterpret_cast<const double*>(queries.data()),
                                   static_cast<int32_t>(queries.size()), out.data());
  if (st == EXM_ERR_INVALID_ARGUMENT) throw std::invalid_argument(exm_last_error());
  if (st != EXM_OK) throw std::runtime_error(std::string("exm_b200: ") + exm_last_error());
}

}  // namespace exactmppi
