"""The control cycle's thresholded rollout SDF (EXM_OPT_SDF_THRESHOLD, GPU).

The reference's control_cycle uses a rollout's per-step minima only through obstacle_cost
(w_coll [d < 0] + w_rep max(d_safe - d, 0)^2, proj/src/controller.cpp:98-101) and the unsafe flag
(d < d_safe, :162), and returns none of them. So the library resolves each rollout minimum exactly
only below d_safe and reports the least float at or above d_safe otherwise. These tests check that
every decision field is bit-identical with the threshold on (default) and off, on every SDF kernel
path and footprint kind, through several warm-started cycles, for single handles and the hybrid
batch; and that the threshold actually removes work."""
import dataclasses

import numpy as np
import pytest

from paper_2605_29663_b200 import _abi
from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import Engine, HybridController, ObstacleSet

from tests.test_gpu_cull_exact import CASES

pytestmark = pytest.mark.gpu


def _cycles(wl, threshold, mode=None, n=4):
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    if mode:
        eng.set_sdf_mode(mode)
    eng.set_sdf_threshold(threshold)
    nom, up = wl.zero_state()
    out = []
    for cyc in range(n):
        d = eng.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, nom, up, cyc)
        out.append((d, nom.copy(), up.copy()))
    stats = eng.sdf_work_stats()
    eng.close()
    return out, stats


def _same(a, b):
    for (da, na, ua), (db, nb, ub) in zip(a, b):
        assert np.array_equal(da.command, db.command)
        assert da.argmin == db.argmin and da.validated == db.validated
        assert da.best_cost == db.best_cost and da.weight_entropy == db.weight_entropy
        assert da.nominal_cost == db.nominal_cost
        assert np.array_equal(da.nominal_d_min, db.nominal_d_min)
        assert np.array_equal(na, nb) and np.array_equal(ua, ub)


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("mode", [None, "thread", "warp", "persist"])
def test_threshold_keeps_decisions_bitwise(case, mode):
    wl = CASES[case]()
    on, s_on = _cycles(wl, True, mode)
    off, s_off = _cycles(wl, False, mode)
    _same(on, off)
    if mode in (None, "thread", "persist"):
        # the counters re-run the thread-per-pose kernel: never more work with the threshold
        assert s_on["point_tests"] <= s_off["point_tests"], (s_on, s_off)


def test_threshold_removes_work_on_cfg2():
    wl = W.cfg2()
    _, s_on = _cycles(wl, True, n=2)
    _, s_off = _cycles(wl, False, n=2)
    print("cfg2 point tests on/off:", s_on["point_tests"], s_off["point_tests"])
    assert s_on["point_tests"] < 0.8 * s_off["point_tests"]


@pytest.mark.parametrize("d_safe", [0.0, 0.1, 0.5])
def test_threshold_at_other_d_safe(d_safe):
    """d_safe = 0 (only the collision indicator remains), and a d_safe above most minima."""
    wl = W.cfg2(K=1024, T=30, N=10_000)
    wl = dataclasses.replace(wl, params=dataclasses.replace(wl.params, d_safe=d_safe))
    on, _ = _cycles(wl, True, n=3)
    off, _ = _cycles(wl, False, n=3)
    _same(on, off)


@pytest.mark.parametrize("which", ["trap", "cfg5"])
def test_threshold_hybrid_batch(which):
    """exm_hybrid_cycle (one SDF launch over every family's poses) with the threshold on / off."""
    if which == "trap":
        fp, modes, params, hp, q0, cloud, g = W.trap_hybrid()
    else:
        fp, modes, params, hp, q0, cloud, g = W.cfg5_hybrid(K=2048, T=40, N=20_000)
    obst = ObstacleSet(cloud, np.ones(cloud.shape[0], np.uint8))
    outs = []
    for thr in (1, 0):
        hc = HybridController(modes, fp, params, hp, n_cap=cloud.shape[0], guide_cap=8)
        hc.set_option(_abi.OPT_SDF_THRESHOLD, thr)
        outs.append([hc.family_cycles(q0, obst, g) for _ in range(3)])
        hc.close()
    for fa, fb in zip(*outs):
        for a, b in zip(fa, fb):
            assert np.array_equal(a.command, b.command) and a.argmin == b.argmin
            assert a.best_cost == b.best_cost and a.nominal_cost == b.nominal_cost
            assert np.array_equal(a.nominal.reshape(-1), b.nominal.reshape(-1))
