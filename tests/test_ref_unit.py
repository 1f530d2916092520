"""The reference's own unit tests of the translation units the drop-ins replace
(proj/tests/test_controller.cpp for controller.cpp, test_hybrid.cpp for hybrid.cpp,
test_geometry.cpp and test_bench.cpp whose batch_signed_distance calls go to the B200 through
the linker wrap, test_world.cpp whose episodes run every MPPI step on the B200),
compiled where they lie with the doctest stand-in of tests/ref_unit/doctest.h; footprint fixtures
from tools/write_fixtures.py.

* CPU: the same files linked against the UNMODIFIED reference (oracle/_ref/ref_test_*, built by
  `make -C oracle refunit`) pass every case — this pins the stand-in.
* GPU: linked against the B200 drop-in (paper_2605_29663_b200/lib/exm_ref_test_*_b200, built by
  `make -C paper_2605_29663_b200/host refunit`): every MPPI cycle, rollout evaluation,
  validation and hybrid cycle these tests make runs on the device, and every case passes at the
  reference's own tolerances (1e-9 / 1e-12 batch-vs-scalar included, through EXM_OPT_SDF_FP64)."""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
UNITS = ["controller", "hybrid", "geometry", "world", "bench"]


def _run(path, tmp):
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "write_fixtures.py"), str(tmp)],
                   check=True, capture_output=True)
    env = dict(os.environ, EXM_FIXTURES_DIR=str(tmp))
    out = subprocess.run([path], capture_output=True, text=True, timeout=900, env=env)
    cases = re.findall(r"^\[(PASS|FAIL)\] (.*)$", out.stdout, re.M)
    return out.returncode, cases, out.stdout


@pytest.mark.parametrize("unit", UNITS)
def test_reference_unit_tests_on_reference(unit, tmp_path):
    path = os.path.join(ROOT, "oracle", "_ref", f"ref_test_{unit}")
    if not os.path.exists(path):
        pytest.skip("oracle/_ref unit tests not built")
    rc, cases, out = _run(path, tmp_path)
    assert cases, out
    assert rc == 0 and all(s == "PASS" for s, _ in cases), out


@pytest.mark.gpu
@pytest.mark.parametrize("unit", UNITS)
def test_reference_unit_tests_on_b200(unit, tmp_path):
    path = os.path.join(ROOT, "paper_2605_29663_b200", "lib", f"exm_ref_test_{unit}_b200")
    if not os.path.exists(path):
        pytest.skip("drop-in unit tests not built")
    rc, cases, out = _run(path, tmp_path)
    print(out)
    assert len(cases) >= 5, out
    assert rc == 0 and all(s == "PASS" for s, _ in cases), out
