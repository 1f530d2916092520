// episode_main.cpp — whole-episode determinism harness through the drop-in (SURVEY §8(f)3,
// acceptance criterion 8, proj/tests/acceptance_main.cpp:400-448). The reference checks that its
// CLI `run` writes byte-identical trajectories for two thread counts; the CLI needs CLI11, which
// is absent, so this harness drives the same path the CLI's `run` takes
// (proj/tools/exact_mppi_main.cpp:33-76: generate the scenario from a template with the given
// seed, run_episode with the thread count and a diagnostics sink, trajectory_to_csv) directly,
// with every MPPI step on the B200 (controller_b200.cpp / hybrid_b200.cpp). With
// EXM_DROPIN_SHARDS=G in the environment the controller steps run as G rollout shards on the
// one GPU (exm_sharded_cycle), so traces can also be compared across G.
//
//   exm_episode_b200 <fixtures_dir> corridor|gap|trap <seed> <threads> <out_prefix>
// corridor: l_shape footprint, DoN 0.80 (corridor_don080); gap: l_shape, DoN 1.05 (the omni gap
// of omni_gap_don105); trap: the hybrid trap (trap_hybrid). Writes <out_prefix>_trajectory.csv
// and <out_prefix>_cycles.jsonl (one cycle_trace_to_json_line per control cycle).
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>

#include "exactmppi/scenario_gen.hpp"
#include "exactmppi/scenario_io.hpp"
#include "exactmppi/world.hpp"

int main(int argc, char** argv) {
  using namespace exactmppi;
  if (argc != 6) {
    std::fprintf(stderr, "usage: %s fixtures_dir corridor|gap|trap seed threads out_prefix\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1], kind = argv[2], out = argv[5];
  const std::uint64_t seed = std::strtoull(argv[3], nullptr, 10);
  const int threads = std::atoi(argv[4]);
  Scenario scenario;
  if (kind == "corridor") {
    scenario = make_corridor_scenario(load_footprint(dir + "/footprints/l_shape.json"), 0.80, seed);
  } else if (kind == "gap") {
    scenario = make_gap_scenario(load_footprint(dir + "/footprints/l_shape.json"), 1.05, seed);
  } else if (kind == "trap") {
    scenario = make_trap_scenario(seed);
  } else {
    std::fprintf(stderr, "unknown scenario kind %s\n", kind.c_str());
    return 2;
  }
  scenario.seed = seed;
  EpisodeOptions options;
  options.threads = threads;
  std::ostringstream diag;
  options.diagnostics_sink = [&diag](const CycleTrace& t) { diag << cycle_trace_to_json_line(t); };
  const EpisodeResult r = run_episode(scenario, options);
  write_text_file(out + "_trajectory.csv", trajectory_to_csv(r));
  write_text_file(out + "_cycles.jsonl", diag.str());
  std::printf("%s %s cycles=%zu nav_time=%.3f\n", kind.c_str(), r.success ? "success" : "failure",
              r.trajectory.size(), r.nav_time);
  return 0;
}
