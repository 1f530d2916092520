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


HYBRID_BIN = os.path.join(ROOT, "paper_2605_29663_b200", "lib", "exm_hybrid_check")


@pytest.mark.skipif(not os.path.exists(HYBRID_BIN) or not ob.reference_available(),
                    reason="hybrid check binary or oracle/_ref not built")
def test_hybrid_dropin_matches_reference():
    """HybridController through hybrid_b200.cpp (all mode families of a cycle in one device
    call, exm_hybrid_cycle) vs the unmodified reference HybridController (hybrid.cpp:95-156, CPU,
    oracle/_ref) on the reference's trap scenario and sensed cloud: the same mode selection,
    commands and switch-penalised mode costs, cycle after cycle."""
    from paper_2605_29663_b200.api import ComponentLimit, HybridMode, HybridParams
    out = subprocess.run([HYBRID_BIN], capture_output=True, text=True, timeout=300, check=True).stdout
    lines = [json.loads(x) for x in out.splitlines() if x.startswith("{")]
    s = lines[0]
    fp = FootprintSpec.rect_cover(np.stack([s["rect_cx"], s["rect_cy"]], 1),
                                  np.stack([s["rect_hx"], s["rect_hy"]], 1))
    modes = []
    for m in s["modes"]:
        lim = KinematicLimits.unbounded()
        v = m["limits"]
        for i in range(3):
            lim.component[i] = ComponentLimit(*v[4 * i: 4 * i + 4])
        lim.steer_max = v[12]
        model = MotionModel(int(m["tag"]), float(m["wheelbase"]))
        modes.append(HybridMode(f"m{len(modes)}", model, lim))
    pv = s["params"]
    p = MppiParams(rollouts=int(pv[0]), horizon=int(pv[1]), dt=pv[2], lambda_=pv[3],
                   sigma=tuple(pv[4:7]), d_safe=pv[7], w_coll=pv[8], w_rep=pv[9], w_inf=pv[10],
                   task=TaskWeights(pv[11], pv[12], pv[13], pv[14]), w_ctrl=pv[15], seed=int(pv[16]))
    h = s["hybrid"]
    hp = HybridParams(lambda_switch=h[0], tau_cool_max=int(h[1]), v_min=h[2], omega_min=h[3],
                      noise_deadzone_v=h[4], noise_deadzone_omega=h[5])
    ref = ob.ReferenceHybrid(fp, modes, p, hp)
    pts = np.array(s["points"]).reshape(-1, 2)
    mask = np.array(s["mask"], np.uint8)
    g = Guidance(np.array(s["guide"]).reshape(-1, 2), s["goal"])
    cycles = [x for x in lines if x["kind"] == "cycle"]
    assert len(cycles) == 8
    for c in cycles:
        r = ref.hybrid_cycle(np.array(c["q"]), pts, mask, g)
        assert c["mode_index"] == r["mode_index"], c["cycle"]
        assert c["validated"] == int(r["validated"])
        cmd = np.array(c["command"])
        assert np.max(np.abs(cmd - r["command"][: cmd.size])) <= 1e-5
        rc = np.where(np.isfinite(r["mode_costs"]), r["mode_costs"], 1e300)
        assert np.allclose(c["mode_costs"], rc, rtol=1e-5, atol=1e-5)
        assert abs(c["nominal_cost"] - r["nominal_cost"]) <= 1e-5 * max(1.0, abs(r["nominal_cost"]))
