// scaling_main.cpp — the reference's evaluator benchmark (scaling_benchmark,
// proj/src/bench.cpp:55-113, compiled where it lies) with its batch_signed_distance calls
// redirected to the B200 by geometry_sdf_b200.cpp (linker symbol wrapping): the same protocol
// (3 warm-ups, steady_clock per call, benchmark_queries in a 50 m square), the same CSV
// (bench.cpp:57), every call host -> B200 -> host.
//
//   exm_scaling_b200 <fixtures_dir> <trials> <threads> <count> [<count> ...]
// Footprints: l_shape, l_shape_rect, t_shape, t_shape_rect, f_shape, f_shape_rect
// (<fixtures_dir>/footprints/<name>.json, loaded by the reference's scenario_io).
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "exactmppi/bench.hpp"
#include "exactmppi/scenario_io.hpp"

int main(int argc, char** argv) {
  using namespace exactmppi;
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s fixtures_dir trials threads count...\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  const int trials = std::atoi(argv[2]);
  const int threads = std::atoi(argv[3]);
  std::vector<std::size_t> counts;
  for (int i = 4; i < argc; ++i) counts.push_back(static_cast<std::size_t>(std::atoll(argv[i])));
  std::vector<FootprintSpec> specs;
  for (const char* n : {"l_shape", "l_shape_rect", "t_shape", "t_shape_rect", "f_shape", "f_shape_rect"})
    specs.push_back(load_footprint(dir + "/footprints/" + n + ".json"));
  const BenchReport r = scaling_benchmark(specs, counts, trials, 0, {threads});
  std::fputs(r.to_csv().c_str(), stdout);
  return 0;
}
