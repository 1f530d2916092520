"""The reference's own acceptance suite (proj/tests/acceptance_main.cpp, compiled where it lies)
linked against the B200 drop-in (host/controller_b200.cpp replacing controller.cpp): whole
episodes through run_episode / HybridController with every MPPI step on the GPU.

Expected outcome: criteria 1-5, 7, 9 PASS with the reference's recorded behavioural numbers
(proj/test_output.txt). Criterion 6 contains a 1e-9 batch-vs-scalar d_min check that an FP32
signed distance cannot meet by design (north-star tolerance is 1e-5); criterion 8 needs the CLI,
which cannot be built here (CLI11 absent)."""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2605_29663_b200", "lib", "exm_acceptance_b200")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(BIN), reason="acceptance binary not built")]


def test_reference_acceptance_suite_on_b200(tmp_path):
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "write_fixtures.py"), str(tmp_path)],
                   check=True, capture_output=True)
    env = dict(os.environ, EXM_FIXTURES_DIR=str(tmp_path))
    out = subprocess.run([BIN], env=env, capture_output=True, text=True, timeout=1200).stdout
    res = {int(m.group(2)): (m.group(1), m.group(3))
           for m in re.finditer(r"\[(PASS|FAIL)\] criterion (\d+): (.*)", out)}
    for c in (1, 2, 3, 4, 5, 7, 9):
        assert res[c][0] == "PASS", (c, res[c][1])
    # behavioural numbers identical to the reference's recorded run (proj/test_output.txt:31-33)
    assert "hybrid 10/10" in res[7][1] and "median 8.2 s" in res[7][1]
    assert "DoN 1.05 exact 10/10" in res[4][1] and "hull 0/10" in res[4][1]
    assert "DoN 1: exact 10/10, hull 0/10" in res[5][1]
    assert res[6][0] == "FAIL" and "all hold" in res[6][1]  # only the 1e-9 d_min check trips
