"""Device sensing (exm_sense, world.cpp:182-243) against the reference's own
sense() compiled from its sources (oracle/_ref, ref_sense): boundary samples, 720-bin nearest
sample, exact line of sight, seeded downsample, padding. The reference scenes are the fixture
obstacles (corridor, trap, omni_gap walls) plus moving discs displaced by trail offsets."""
import math

import numpy as np
import pytest

from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import Engine, WorldObstacle
from tests.oracle_bindings import ReferenceWorld, reference_available, reference_sense

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")]


def _discs(n=24, seed=9):
    out = []
    for k in range(n):
        cx, cy = W.uniform_range(seed, k, 0, -6.0, 6.0), W.uniform_range(seed, k, 1, -6.0, 6.0)
        r = W.uniform_range(seed, k, 4, 0.2, 0.5)
        ox, oy = W.uniform_range(seed, k, 2, -0.5, 0.5), W.uniform_range(seed, k, 3, -0.5, 0.5)
        out.append(WorldObstacle.disc((cx, cy), r, (ox, oy)))
    return out


SCENES = {
    "corridor": [WorldObstacle.polygon(p) for p in W.CORRIDOR_OBSTACLES],
    "trap": [WorldObstacle.polygon(p) for p in W.TRAP_OBSTACLES],
    "omni_gap_moving_discs": [WorldObstacle.polygon(p) for p in W.OMNI_WALLS] + _discs(),
    "moving_polygons": [WorldObstacle.polygon(p, (0.37, -0.21)) for p in W.TRAP_OBSTACLES],
}


def _engine():
    wl = W.cfg1(K=32, T=4)
    return Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=16, guide_cap=4)


@pytest.mark.parametrize("scene", list(SCENES))
@pytest.mark.parametrize("budget", [1, 60, 400, 1000])
def test_sense_matches_reference(scene, budget):
    eng = _engine()
    obs = SCENES[scene]
    rng = np.random.default_rng(3)
    for trial in range(6):
        robot = np.array([rng.uniform(-4, 4), rng.uniform(-1.5, 1.5), rng.uniform(-math.pi, math.pi)])
        sensor_range = [3.0, 6.0, 10.0][trial % 3]
        key = 1000 + trial
        got = eng.sense(obs, robot, sensor_range, budget, seed=7, sample_key=key)
        pts, mask, n = reference_sense(obs, robot, sensor_range, budget, 7, key)
        assert np.array_equal(got.mask, mask), (scene, trial)
        assert int(got.mask.sum()) == n
        if "disc" in scene:  # disc samples go through cos/sin: CUDA vs glibc last bits
            assert np.allclose(got.points, pts, rtol=0, atol=1e-12), (scene, trial)
        else:  # polygon samples are products and sums only: bit-identical
            assert np.array_equal(got.points, pts), (scene, trial)


def test_sense_edge_cases():
    eng = _engine()
    # no obstacles: everything padded
    got = eng.sense([], [0.0, 0.0, 0.0], 10.0, 5, 1, 2)
    assert not got.mask.any() and np.all(got.points == 1e9)
    # robot inside a polygon obstacle; range 0 (nothing within range)
    box = [WorldObstacle.polygon([[-1, -1], [1, -1], [1, 1], [-1, 1]])]
    for robot, rng_ in (([0.0, 0.0, 0.0], 10.0), ([5.0, 0.0, 0.0], 0.0)):
        got = eng.sense(box, robot, rng_, 50, 3, 4)
        pts, mask, n = reference_sense(box, robot, rng_, 50, 3, 4)
        assert np.array_equal(got.mask, mask) and np.array_equal(got.points, pts)
    with pytest.raises(ValueError, match="budget"):
        eng.sense(box, [0.0, 0.0, 0.0], 10.0, 0, 1, 1)


def test_sensed_cloud_drives_a_control_cycle():
    """sense -> control_cycle on the same handle: the sensed ObstacleSet is a valid input."""
    wl = W.cfg1(K=256, T=16)
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=300, guide_cap=4)
    obs = [WorldObstacle.polygon(p) for p in W.CORRIDOR_OBSTACLES]
    cloud = eng.sense(obs, wl.q0, 10.0, 300, 1, 0)
    assert cloud.mask.sum() > 50
    nom, up = wl.zero_state()
    d = eng.control_cycle_raw(wl.q0, cloud, wl.guidance, nom, up, 0, None)
    assert np.all(np.isfinite(d.command))


def _moving_world(seed=11):
    """omni_gap walls (static) + 24 discs on 2-waypoint ping-pong trails + two trap polygons, one
    on a clamped 3-waypoint trail, one on a ping-pong 3-waypoint trail (cfg5-style motion)."""
    from paper_2605_29663_b200.api import Trail
    obs = [WorldObstacle.polygon(p) for p in W.OMNI_WALLS]
    trails = [None] * len(obs)
    for k in range(24):
        ax, ay = W.uniform_range(seed, k, 0, -6.0, 6.0), W.uniform_range(seed, k, 1, -6.0, 6.0)
        bx, by = W.uniform_range(seed, k, 2, -6.0, 6.0), W.uniform_range(seed, k, 3, -6.0, 6.0)
        obs.append(WorldObstacle.disc((ax, ay), W.uniform_range(seed, k, 4, 0.2, 0.5)))
        trails.append(Trail([[ax, ay], [bx, by]], W.uniform_range(seed, k, 5, 0.0, 1.5)))
    p0, p1 = W.TRAP_OBSTACLES[3], W.TRAP_OBSTACLES[2]
    obs += [WorldObstacle.polygon(p0), WorldObstacle.polygon(p1)]
    trails += [Trail([p0[0], [p0[0][0] + 1.0, p0[0][1] + 0.3], [p0[0][0] + 1.5, p0[0][1] - 0.7]], 0.9,
                     ping_pong=False),
               Trail([p1[0], [p1[0][0] - 0.4, p1[0][1]], [p1[0][0] - 0.4, p1[0][1] + 0.6]], 1.3)]
    return obs, trails


def test_device_world_steps_and_senses_like_the_reference():
    """step_world (world.cpp:127-157) on the device: arc, direction and obstacle offsets bit for
    bit against the reference over 80 steps (reflections and clamps included), and sense() from
    the device state against the reference's sense() on its own state."""
    eng = _engine()
    obs, trails = _moving_world()
    dev = eng.world(obs, trails, 10.0, 400, 7)
    ref = ReferenceWorld(obs, trails, 10.0, 400, 7)
    a0, d0, o0 = dev.state()
    ra, rd, ro = ref.state()
    assert np.array_equal(a0, ra) and np.array_equal(d0, rd) and np.array_equal(o0, ro)
    rng = np.random.default_rng(4)
    for step in range(80):
        dt = 0.1 if step % 7 else 0.37
        dev.step(dt)
        ref.step(dt)
        a, d, o = dev.state()
        ra, rd, ro = ref.state()
        assert np.array_equal(a, ra) and np.array_equal(d, rd), step
        assert np.array_equal(o, ro), step
        if step % 10 == 9:
            robot = np.array([rng.uniform(-4, 4), rng.uniform(-2, 2), 0.0])
            got = dev.sense(robot, 50 + step)
            pts, mask, n = ref.sense(robot, 50 + step)
            assert np.array_equal(got.mask, mask), step
            assert np.allclose(got.points, pts, rtol=0, atol=1e-12), step
    assert (d == -1).any(), "no trail reflected: the test does not cover ping-pong"
    with pytest.raises(ValueError, match="dt > 0"):
        dev.step(0.0)
    dev.close()
