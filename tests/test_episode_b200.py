"""Whole-episode determinism through the drop-in (the reference's acceptance
criterion 8, proj/tests/acceptance_main.cpp:400-448, which needs the CLI — absent here — so
lib/exm_episode_b200 drives the CLI `run` path, proj/tools/exact_mppi_main.cpp:33-76, directly).

Every MPPI step of run_episode (proj/src/world.cpp:354-499) runs on the B200: controller_b200.cpp
for MppiController, hybrid_b200.cpp (one batched device call per hybrid cycle) for the trap. The
trajectory CSV (trajectory_to_csv) and the per-cycle trace (cycle_trace_to_json_line) must be
byte-identical between two runs with different thread counts (the criterion), and between the
unsharded step and the step run as G = 2 rollout shards on the one GPU (EXM_DROPIN_SHARDS)."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2605_29663_b200", "lib", "exm_episode_b200")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(BIN), reason="episode binary not built")]


@pytest.fixture(scope="module")
def fixtures(tmp_path_factory):
    d = tmp_path_factory.mktemp("fixtures")
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "write_fixtures.py"), str(d)],
                   check=True, capture_output=True)
    return str(d)


def run(fixtures, kind, threads, out, shards=1):
    env = dict(os.environ, EXM_DROPIN_SHARDS=str(shards))
    r = subprocess.run([BIN, fixtures, kind, "42", str(threads), out], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr
    csv = open(out + "_trajectory.csv", "rb").read()
    jl = open(out + "_cycles.jsonl", "rb").read()
    assert csv and jl
    return r.stdout, csv, jl


@pytest.mark.parametrize("kind", ["corridor", "gap", "trap"])
def test_episode_bytes_identical_across_threads_and_shards(kind, fixtures, tmp_path):
    out_a, csv_a, jl_a = run(fixtures, kind, 2, str(tmp_path / "a"))
    out_b, csv_b, jl_b = run(fixtures, kind, 1, str(tmp_path / "b"))
    print(out_a.strip(), "| cycles:", jl_a.count(b"\n"))
    assert csv_a == csv_b and jl_a == jl_b
    if kind != "trap":  # K = 512: two shards of 256 rollouts (the trap's K = 384 does not split)
        _, csv_g, jl_g = run(fixtures, kind, 1, str(tmp_path / "g2"), shards=2)
        assert csv_g == csv_a and jl_g == jl_a
