"""Pins the C restatement (oracle/exm_oracle.c) against the known answers of the reference's
own unit tests (proj/tests/test_geometry.cpp, test_controller.cpp, test_kinematics.cpp).
CPU only."""
import math

import numpy as np
import pytest

from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import (FootprintSpec, Guidance, KinematicLimits, MotionModel,
                                       MppiParams, TaskWeights)
from tests.oracle_bindings import Oracle, oracle_lib, oracle_weights


def mk(fp, model=None, params=None, limits=None):
    return Oracle(fp, model or MotionModel.diff(), limits or KinematicLimits.unbounded(),
                  params or MppiParams(rollouts=4, horizon=5))


def unit_square():
    return FootprintSpec.polygon([[0, 0], [1, 0], [1, 1], [0, 1]])


def approx(a, b, eps=1e-12):
    return abs(a - b) <= eps * max(1.0, abs(b))


def test_sd_box_examples():  # test_geometry.cpp:42-46
    o = mk(FootprintSpec.rect_cover([[0, 0]], [[1, 2]]))
    assert approx(o.sd(0, 0), -1.0) and approx(o.sd(3, 0), 2.0) and approx(o.sd(4, 6), 5.0)


def test_rect_cover_t():  # test_geometry.cpp:48-57
    o = mk(FootprintSpec.rect_cover([[0.0, 0.8], [0.0, 0.0]], [[1.0, 0.2], [0.2, 0.6]]))
    assert approx(o.sd(0, 2.0), 1.0)
    assert approx(o.sd(0, 0.8), -0.2)


def test_point_segment_examples():  # test_geometry.cpp:73-77 via a thin triangle's edge
    # distance to the closed segment [(-1,0),(1,0)] == sd of a degenerate-free triangle far below
    o = mk(FootprintSpec.polygon([[-1, 0], [1, 0], [0, -50]]))
    assert approx(o.sd(0, 1), 1.0) and approx(o.sd(3, 0), 2.0, 1e-9)


def test_polygon_examples():  # test_geometry.cpp:79-101
    sq = mk(unit_square())
    assert approx(sq.sd(0.5, 0.5), -0.5) and approx(sq.sd(2.0, 0.5), 1.0)
    L = mk(FootprintSpec.polygon([[0, 0], [2, 0], [2, 1], [1, 1], [1, 2], [0, 2]]))
    assert approx(L.sd(1.5, 1.5), 0.5)  # concave notch is outside
    assert L.sd(0.5, 0.5) < 0


def test_polygon_validation():  # test_geometry.cpp:103-113
    with pytest.raises(ValueError, match="at least 3"):
        mk(FootprintSpec.polygon([[0, 0], [1, 0]]))
    with pytest.raises(ValueError, match="zero-length"):
        mk(FootprintSpec.polygon([[0, 0], [1, 0], [1, 0], [0, 1]]))
    with pytest.raises(ValueError, match="self-intersects"):
        mk(FootprintSpec.polygon([[0, 0], [1, 1], [1, 0], [0, 1]]))
    cw = mk(FootprintSpec.polygon([[0, 0], [0, 1], [1, 1], [1, 0]]))  # reversed to CCW
    assert approx(cw.sd(0.5, 0.5), -0.5)


def test_rect_validation():  # test_geometry.cpp:66-71
    with pytest.raises(ValueError):
        mk(FootprintSpec.rect_cover([[0, 0]], [[0.0, 1.0]]))
    with pytest.raises(ValueError):
        mk(FootprintSpec.rect_cover([[0, 0]], [[1.0, -0.5]]))


def test_min_signed_distance_examples():  # test_geometry.cpp:136-146
    o = mk(unit_square())
    assert approx(o.min_signed_distance_at([0, 0, 0], [[2, 0], [0, 3]]), 1.0)
    assert approx(o.min_signed_distance_at([0, 0, 0], [[0.5, 0.5], [5, 5]]), -0.5)
    assert o.min_signed_distance_at([0, 0, 0], np.full((16, 2), 1e9), np.zeros(16)) == 1e6


def test_transform_examples():  # test_geometry.cpp:115-134, through min_signed_distance_at
    o = mk(FootprintSpec.rect_cover([[0, 0]], [[0.1, 0.1]]))
    # point (0,1) at pose (0,0,pi/2) lies on the body +x axis at distance 1
    d = o.min_signed_distance_at([0, 0, math.pi / 2], [[0, 1]])
    assert approx(d, 0.9, 1e-12)
    assert approx(o.min_signed_distance_at([1, 0, 0], [[2, 0]]), 0.9, 1e-12)


def test_gallery_vs_independent_oracle():  # test_geometry.cpp:230-253 (winding + dense samples)
    for name in W.GALLERY:
        fp = W.footprint(name)
        o = mk(fp)
        v = fp.a
        pts = np.stack([W.uniform_range(777, np.arange(300, dtype=np.uint64), 11, -4, 4),
                        W.uniform_range(777, np.arange(300, dtype=np.uint64), 13, -4, 4)], 1)
        d = o.batch_signed_distance(pts)
        n = len(v)
        for p, dp in zip(pts, d):
            seg = [(v[i], v[(i + 1) % n]) for i in range(n)]
            dist = min(_seg_dist(p, a, b) for a, b in seg)
            wind = sum(math.atan2(_cross(a - p, b - p), np.dot(a - p, b - p)) for a, b in seg)
            assert abs(abs(dp) - dist) <= 1e-12
            if abs(dp) > 1e-6:
                assert (dp < 0) == (abs(wind) / (2 * math.pi) > 0.5)


def _seg_dist(p, a, b):
    e = b - a
    t = np.clip(np.dot(p - a, e) / np.dot(e, e), 0.0, 1.0)
    return float(np.hypot(*(p - (a + t * e))))


def test_rect_polygon_agree():  # test_geometry.cpp:255-269
    for poly, rect in (("l_shape", "l_shape_rect"), ("t_shape", "t_shape_rect"),
                       ("f_shape", "f_shape_rect")):
        op, orr = mk(W.footprint(poly)), mk(W.footprint(rect))
        i = np.arange(2000, dtype=np.uint64)
        pts = np.stack([W.uniform_range(1234, i, 11, -3, 3), W.uniform_range(1234, i, 13, -3, 3)], 1)
        dp, dr = op.batch_signed_distance(pts), orr.batch_signed_distance(pts)
        ext = dr > 0
        assert np.max(np.abs(dp[ext] - dr[ext])) <= 1e-9
        both = (np.abs(dp) > 1e-9) & (np.abs(dr) > 1e-9)
        assert np.all((dp[both] < 0) == (dr[both] < 0))


def test_rng_matches_numpy_generator():  # rng.hpp:12-58 (two independent restatements)
    L = oracle_lib()
    for s in (0, 1, 7, 2 ** 63 + 5):
        for a in (0, 3, 1000):
            assert L.exo_uniform_range(s, a, 2, -1.0, 1.0) == float(W.uniform_range(s, a, 2, -1.0, 1.0))
    x = W.splitmix64(np.arange(10, dtype=np.uint64))
    assert [int(L.exo_splitmix64(i)) for i in range(10)] == [int(v) for v in x]


def test_perturbations_determinism_and_sigma():  # test_controller.cpp:58-76
    p = MppiParams(rollouts=16, horizon=8, seed=9)
    o = mk(unit_square(), params=p)
    a, b = o.sample_perturbations(42, 3), o.sample_perturbations(42, 3)
    assert np.array_equal(a, b)
    assert np.any(a[..., 0] != o.sample_perturbations(42, 4)[..., 0])
    tiny = mk(unit_square(), params=MppiParams(rollouts=16, horizon=8, sigma=(1e-12,) * 3))
    assert np.all(np.abs(tiny.sample_perturbations(1, 0)) < 1e-10)


def test_lln():  # test_controller.cpp:78-87
    o = mk(unit_square(), model=MotionModel.spin(),
           params=MppiParams(rollouts=10000, horizon=1, sigma=(0.5, 0.5, 0.5)))
    e = o.sample_perturbations(7, 0)
    assert abs(e.mean()) < 4.0 * 0.5 / math.sqrt(10000.0)


def test_obstacle_cost_examples():  # test_controller.cpp:89-97
    o = mk(unit_square(), params=MppiParams(d_safe=0.3, w_rep=10.0, w_coll=1e6))
    L = oracle_lib()
    assert approx(L.exo_obstacle_cost(o.ctx, 1.0), 0.0)
    assert approx(L.exo_obstacle_cost(o.ctx, 0.2), 0.1)
    assert approx(L.exo_obstacle_cost(o.ctx, -0.05), 1e6 + 10.0 * 0.35 * 0.35)


def test_task_cost_examples():  # test_controller.cpp:99-123
    L = oracle_lib()
    g = Guidance([[0, 0], [4, 0]], [4, 0, 0])

    def tc(w, q, terminal=False):
        o = mk(unit_square(), params=MppiParams(task=TaskWeights(*w)))
        q = np.asarray(q, np.float64)
        return L.exo_task_cost(o.ctx, q.ctypes.data_as(_dp()), g.path.ctypes.data_as(_dp()), 2,
                               g.goal.ctypes.data_as(_dp()), 1 if terminal else 0)

    assert approx(tc((0, 0, 0, 1.5), [4, 0, 0], True), -6.0)
    assert approx(tc((0, 0, 3, 0), [0, 0, 0]), 0.0)
    assert approx(tc((0, 0, 2, 0), [2, 1, 0]), 2.0)
    assert approx(tc((0, 1, 0, 0), [2, 0, 0.5]), 0.0)
    assert approx(tc((0, 1, 0, 0), [2, 0, 0.5], True), 0.25)


def _dp():
    import ctypes
    return ctypes.POINTER(ctypes.c_double)


def test_weights_examples():  # test_controller.cpp:125-151
    assert approx(oracle_weights([3.7], 1.0)[0], 1.0)
    assert np.allclose(oracle_weights([5.0, 5.0], 1.0), [0.5, 0.5])
    assert np.allclose(oracle_weights([0.0, math.log(3.0)], 1.0), [0.75, 0.25], rtol=1e-12)
    c = W.uniform_range(5, np.arange(200, dtype=np.uint64), 0, -10, 10)
    w = oracle_weights(c, 0.7)
    assert abs(w.sum() - 1.0) < 1e-12
    assert np.allclose(oracle_weights(c + 123.456, 0.7), w, rtol=1e-12)


def test_unsafe_mass():  # test_controller.cpp:153-168
    c = W.uniform_range(8, np.arange(500, dtype=np.uint64), 0, 0, 100)
    bad = np.arange(500) % 3 == 0
    w = oracle_weights(c + 1e9 * bad, 1e3)
    assert w[bad].sum() < 1e-6


def diff_limits():  # test_controller.cpp:41-46
    lim = KinematicLimits.unbounded()
    lim.component[0].vel_min, lim.component[0].vel_max = -1.5, 1.5
    lim.component[0].acc_min, lim.component[0].acc_max = -3.0, 3.0
    lim.component[1].vel_min, lim.component[1].vel_max = -1.0, 1.0
    lim.component[1].acc_min, lim.component[1].acc_max = -6.0, 6.0
    return lim


def square(h):
    return FootprintSpec.polygon([[-h, -h], [h, -h], [h, h], [-h, h]])


def test_trivial_rollouts():  # test_controller.cpp:170-204
    p = MppiParams(rollouts=1, horizon=10, d_safe=0.1, seed=9)
    o = mk(square(0.5), params=p, limits=diff_limits())
    g = Guidance([[0, 0], [3, 0]], [3, 0, 0])
    r = o.evaluate_rollouts([0, 0, 0], np.zeros(20), np.zeros((1, 10, 2)), np.full((8, 2), 1e9),
                            np.zeros(8), g, [0, 0])
    assert r["unsafe"][0] == 0 and np.allclose(r["states"][0, :, :2], 0.0)
    p3 = MppiParams(rollouts=3, horizon=10, d_safe=0.1, seed=9)
    o3 = mk(square(0.5), params=p3, limits=diff_limits())
    eps = o3.sample_perturbations(9, 0)
    r3 = o3.evaluate_rollouts([0, 0, 0], np.zeros(20), eps, [[0.1, 0.1]], None, g, [0, 0])
    assert np.all(r3["d_min"][:, 0] < 0) and np.all(r3["unsafe"] == 1)


def test_validate_nominal_examples():  # test_controller.cpp:292-319
    p = MppiParams(rollouts=4, horizon=10, d_safe=0.1, seed=9)
    o = mk(square(0.5), params=p, limits=diff_limits())
    g = Guidance([[0, 0], [3, 0]], [3, 0, 0])
    fwd = np.tile([1.0, 0.0], 10)
    ok, dmin, _ = o.validate_nominal(fwd, [0, 0, 0], np.full((8, 2), 1e9), np.zeros(8), g, [0, 0])
    assert ok and np.all(dmin == 1e6)
    bad, _, _ = o.validate_nominal(fwd, [0, 0, 0], [[0.6, 0.0]], None, g, [0, 0])
    assert not bad
    clear, _, _ = o.validate_nominal(fwd, [0, 0, 0], [[0.4, 0.5 + 0.1 + 1e-3]], None, g, [0, 0])
    assert clear


def test_safe_stop_when_enclosed():  # test_controller.cpp:338-355
    p = MppiParams(rollouts=64, horizon=10, d_safe=0.1, seed=9)
    o = mk(square(0.4), params=p, limits=diff_limits())
    a = 2 * math.pi * np.arange(32) / 32
    ring = np.stack([0.45 * np.cos(a), 0.45 * np.sin(a)], 1)
    nom, up = np.zeros(20), np.zeros(3)
    d = o.control_cycle([0, 0, 0], ring, None, Guidance([[0, 0], [3, 0]], [3, 0, 0]), nom, up, 0)
    assert not d["validated"] and np.all(d["command"] == 0) and np.all(nom == 0)


def test_kinematics_models():  # test_kinematics.cpp:28-131 (derivative/step/clamp)
    for model, u, expect in (
            (MotionModel.diff(), [1.0, 0.5], [0.1, 0.0, 0.05]),
            (MotionModel.omni(), [1.0, 2.0, 0.5], [0.1, 0.2, 0.05]),
            (MotionModel.spin(), [0.5], [0.0, 0.0, 0.05]),
            (MotionModel.parallel(), [1.0], [0.0, 0.1, 0.0]),
            (MotionModel.ackermann(0.5), [1.0, 0.0], [0.1, 0.0, 0.0])):
        o = mk(unit_square(), model=model, params=MppiParams(dt=0.1))
        assert np.allclose(o.step([0, 0, 0], u), expect, atol=1e-15)
    lim = diff_limits()
    o = mk(unit_square(), params=MppiParams(dt=0.1), limits=lim)
    assert np.allclose(o.clamp_control([5.0, -5.0], [0.0, 0.0]), [0.3, -0.6])
    once = o.clamp_control([5.0, -5.0], [1.4, 0.0])
    assert np.allclose(o.clamp_control(once, [1.4, 0.0]), once)  # idempotent


def _cross(a, b):
    return float(a[0] * b[1] - a[1] * b[0])
