"""The C++ link-time drop-in (paper_2605_29663_b200/host/controller_b200.cpp replacing the
reference's controller.cpp) driven through the reference's own C++ API, checked against the
CPU oracle on the same inputs."""
import json
import math
import os
import subprocess

import numpy as np
import pytest

from paper_2605_29663_b200.api import (FootprintSpec, Guidance, KinematicLimits, MotionModel,
                                       MppiParams, TaskWeights)
from tests import oracle_bindings as ob

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2605_29663_b200", "lib", "exm_dropin_check")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(BIN), reason="drop-in binary not built")]


def setup():
    fp = FootprintSpec.polygon([[-1.0, -1.0], [1.0, -1.0], [1.0, -0.6], [-0.6, -0.6], [-0.6, 1.0],
                                [-1.0, 1.0]])
    lim = KinematicLimits.unbounded()
    lim.component[0].vel_min, lim.component[0].vel_max = -2.0, 2.0
    lim.component[0].acc_min, lim.component[0].acc_max = -2.5, 2.5
    lim.component[1].vel_min, lim.component[1].vel_max = -0.9, 0.9
    lim.component[1].acc_min, lim.component[1].acc_max = -6.0, 6.0
    p = MppiParams(rollouts=512, horizon=20, dt=0.1, lambda_=0.8, sigma=(0.45, 0.6, 0.3),
                   d_safe=0.09, w_rep=60.0, task=TaskWeights(0.25, 0.3, 1.6, 3.0), seed=1)
    pts = []
    for k in range(400):
        a = 2.0 * math.pi * k / 400.0
        pts.append((3.0 + 0.5 * math.cos(a), 0.4 + 0.5 * math.sin(a)))
        pts.append((5.0 * math.cos(a), 5.0 * math.sin(a)))
    pts = np.array(pts + [(1e9, 1e9)] * 16)
    mask = np.r_[np.ones(800), np.zeros(16)].astype(np.uint8)
    return fp, lim, p, pts, mask, Guidance([[0.0, 0.0], [6.0, 0.0]], [6.0, 0.0, 0.0])


def test_dropin_matches_oracle():
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300, check=True).stdout
    lines = [json.loads(x) for x in out.splitlines() if x.startswith("{")]
    fp, lim, p, pts, mask, g = setup()
    orc = ob.Oracle(fp, MotionModel.diff(), lim, p)
    nom, up = np.zeros(40), np.zeros(3)
    cycles = [x for x in lines if x["kind"] == "cycle"]
    assert len(cycles) == 3
    for c in cycles:
        o = orc.control_cycle(np.array(c["q"]), pts, mask, g, nom, up, c["cycle"])
        assert c["validated"] == int(o["validated"])
        assert np.max(np.abs(np.array(c["command"]) - o["command"][:2])) <= 1e-5
        assert np.max(np.abs(np.array(c["nominal"]) - nom)) <= 1e-5
        assert abs(c["best_cost"] - o["best_cost"]) <= 1e-5 * max(1.0, abs(o["best_cost"]))
        nom[:] = c["nominal"]  # continue from the drop-in's state
        up[:2] = c["command"]
    roll = [x for x in lines if x["kind"] == "rollouts"][0]
    p64 = MppiParams(**{**p.__dict__, "rollouts": 64})
    o64 = ob.Oracle(fp, MotionModel.diff(), lim, p64)
    eps = o64.sample_perturbations(7, 2)
    assert np.allclose(np.array(roll["eps"]), eps.reshape(-1), rtol=1e-12, atol=1e-14)
    want = o64.evaluate_rollouts([0.1, -0.2, 0.05], np.tile([0.5, 0.0], 20), eps, pts, mask, g,
                                 [0.3, 0.0])
    d = np.array(roll["d_min"])
    assert np.max(np.abs(d - want["d_min"].reshape(-1)) / np.maximum(np.abs(want["d_min"].reshape(-1)), 1)) <= 1e-5
    assert np.max(np.abs(np.array(roll["costs"]) - want["costs"]) / np.maximum(np.abs(want["costs"]), 1)) <= 1e-5
    err = [x for x in lines if x["kind"] == "error"][0]
    assert err["thrown"] == 1 and "lambda must be positive" in err["what"]
