"""Synthetic inputs of the five BASELINE.json configs, generated with the
reference's own counter RNG (rng.hpp:12-58, restated vectorised in numpy) so every run — and
the CPU reference — sees identical inputs. Fixture numbers are transcribed from
proj/fixtures/{footprints,scenarios}/*.json (cited per block); nothing is read from the
reference tree at run time.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .api import (ComponentLimit, FootprintSpec, Guidance, KinematicLimits, MotionModel,
                  MppiParams, ObstacleSet, TaskWeights)

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x):
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        x = x + _GOLD
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def hash_combine(h, v):
    h = np.asarray(h, dtype=np.uint64)
    v = np.asarray(v, dtype=np.uint64)
    with np.errstate(over="ignore"):
        return splitmix64(h ^ (v + _GOLD + (h << np.uint64(6)) + (h >> np.uint64(2))))


def uniform_range(seed, a, b, lo, hi):
    """rng.hpp:51-58, vectorised over any of seed/a/b."""
    k = hash_combine(hash_combine(splitmix64(seed), a), b)
    u = (k >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return lo + u * (hi - lo)


def gaussian_at(seed, a, b, c, d):
    """rng.hpp:29-39 (numpy: libm transcendental results may differ from glibc in the last bit)."""
    k = hash_combine(hash_combine(hash_combine(hash_combine(splitmix64(seed), a), b), c), d)
    u1 = ((hash_combine(k, np.uint64(0xD1B54A32D192ED03)) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    u2 = ((hash_combine(k, np.uint64(0x8CB92BA72F3D8DD7)) >> np.uint64(11)) + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


# ------------------------------------------------------------------------ fixture data
# proj/fixtures/footprints/*.json
FOOTPRINTS = {
    "t_shape": [[-0.2, -0.6], [0.2, -0.6], [0.2, 0.6], [0.6, 0.6], [0.6, 1.0], [-0.6, 1.0],
                [-0.6, 0.6], [-0.2, 0.6]],
    "f_shape": [[-0.5, -1.0], [-0.1, -1.0], [-0.1, -0.1], [0.3, -0.1], [0.3, 0.3], [-0.1, 0.3],
                [-0.1, 0.6], [0.7, 0.6], [0.7, 1.0], [-0.5, 1.0]],
    "l_shape": [[-1.0, -1.0], [1.0, -1.0], [1.0, -0.6], [-0.6, -0.6], [-0.6, 1.0], [-1.0, 1.0]],
    "star": [[0.0, 1.0], [-0.235114, 0.323607], [-0.951057, 0.309017], [-0.380423, -0.123607],
             [-0.587785, -0.809017], [0.0, -0.4], [0.587785, -0.809017], [0.380423, -0.123607],
             [0.951057, 0.309017], [0.235114, 0.323607]],
    "arrow": [[1.2, 0.0], [0.2, 0.7], [0.2, 0.3], [-1.0, 0.3], [-1.0, -0.3], [0.2, -0.3],
              [0.2, -0.7]],
    "diamond": [[1.0, 0.0], [0.0, 0.6], [-1.0, 0.0], [0.0, -0.6]],
    "trapezoid": [[-1.0, -0.5], [1.0, -0.5], [0.6, 0.5], [-0.6, 0.5]],
}
RECT_FOOTPRINTS = {
    "l_shape_rect": ([[0.0, -0.8], [-0.8, 0.0]], [[1.0, 0.2], [0.2, 1.0]]),
    "t_shape_rect": ([[0.0, 0.8], [0.0, 0.0]], [[0.6, 0.2], [0.2, 0.6]]),
    "f_shape_rect": ([[-0.3, 0.0], [0.1, 0.8], [-0.1, 0.1]], [[0.2, 1.0], [0.6, 0.2], [0.4, 0.2]]),
}
GALLERY = ["t_shape", "f_shape", "l_shape", "star", "arrow", "diamond", "trapezoid"]


def footprint(name: str) -> FootprintSpec:
    if name in FOOTPRINTS:
        return FootprintSpec.polygon(FOOTPRINTS[name], name)
    c, h = RECT_FOOTPRINTS[name]
    return FootprintSpec.rect_cover(c, h, name)


# corridor_don080.json (scenarios): limits :69-110 region, mppi block, obstacles, start.
CORRIDOR_LIMITS = {"acc_max": [2.5, 6.0], "acc_min": [-2.5, -6.0], "steer_max": 1e9,
                   "vel_max": [2.0, 0.9], "vel_min": [-2.0, -0.9]}
CORRIDOR_MPPI = {"d_safe": 0.09, "dt": 0.1, "horizon": 30, "lambda": 0.8, "rollouts": 512,
                 "sigma": [0.45, 0.6], "w_coll": 1e6, "w_ctrl": 0.02, "w_goal_head": 0.3,
                 "w_goal_pos": 0.25, "w_inf": 1e9, "w_progress": 3.0, "w_rep": 60.0,
                 "w_xtrack": 1.6}
CORRIDOR_OBSTACLES = [
    [[-7.5, 3.0], [7.5, 3.0], [7.5, 3.3], [-7.5, 3.3]],
    [[-7.5, -3.3], [7.5, -3.3], [7.5, -3.0], [-7.5, -3.0]],
    [[-0.4, 1.0], [0.4, 1.0], [0.4, 3.0], [-0.4, 3.0]],
    [[-0.4, -3.0], [0.4, -3.0], [0.4, -1.0], [-0.4, -1.0]],
]
# trap_hybrid.json: Ackermann mode limits and the mppi block.
TRAP_ACK_LIMITS = {"acc_max": [2.0, 3.0], "acc_min": [-2.0, -3.0], "steer_max": 0.45,
                   "vel_max": [1.0, 0.45], "vel_min": [-1.0, -0.45]}
TRAP_MPPI = {"d_safe": 0.05, "dt": 0.1, "horizon": 25, "lambda": 0.6, "rollouts": 384,
             "sigma": [0.3, 0.15], "w_coll": 1e6, "w_ctrl": 0.02, "w_goal_head": 0.2,
             "w_goal_pos": 0.8, "w_inf": 1e9, "w_progress": 2.0, "w_rep": 60.0, "w_xtrack": 3.0}
# omni_gap_don105.json
OMNI_LIMITS = {"acc_max": [2.0, 2.0, 2.0], "acc_min": [-2.0, -2.0, -2.0], "steer_max": 1e9,
               "vel_max": [1.0, 1.0, 1.0], "vel_min": [-1.0, -1.0, -1.0]}
OMNI_MPPI = {"d_safe": 0.12, "dt": 0.1, "horizon": 30, "lambda": 0.8, "rollouts": 512,
             "sigma": [0.4, 0.4, 0.5], "w_coll": 1e6, "w_ctrl": 0.02, "w_goal_head": 0.2,
             "w_goal_pos": 0.25, "w_inf": 1e9, "w_progress": 3.0, "w_rep": 60.0, "w_xtrack": 1.6}
OMNI_WALLS = [
    [[0.0, -10.0], [0.2, -10.0], [0.2, -0.7396144120134828], [0.0, -0.7396144120134828]],
    [[1.4, 0.7396144120134828], [1.5999999999999999, 0.7396144120134828],
     [1.5999999999999999, 10.0], [1.4, 10.0]],
]


def sample_boundaries(polys, n: int) -> np.ndarray:
    """n points at uniform arc length over the concatenated closed boundaries (arc carried
    across edges and polygons)."""
    segs = []
    for poly in polys:
        p = np.asarray(poly, np.float64)
        for i in range(len(p)):
            segs.append((p[i], p[(i + 1) % len(p)]))
    lens = np.array([np.hypot(*(b - a)) for a, b in segs])
    total = lens.sum()
    cum = np.concatenate([[0.0], np.cumsum(lens)])
    s = np.arange(n) * (total / n)
    idx = np.clip(np.searchsorted(cum, s, side="right") - 1, 0, len(segs) - 1)
    t = (s - cum[idx]) / lens[idx]
    a = np.array([segs[i][0] for i in idx])
    b = np.array([segs[i][1] for i in idx])
    return a + t[:, None] * (b - a)


@dataclass
class Workload:
    name: str
    footprint: FootprintSpec
    model: MotionModel
    limits: KinematicLimits
    params: MppiParams
    q0: np.ndarray
    cloud: np.ndarray  # (N, 2) world frame, all valid
    guidance: Guidance
    description: str

    @property
    def n_points(self) -> int:
        return int(self.cloud.shape[0])

    def obstacles(self) -> ObstacleSet:
        return ObstacleSet(self.cloud, np.ones(self.n_points, np.uint8))

    def zero_state(self):
        d = self.model.control_dim()
        return np.zeros(self.params.horizon * d), np.zeros(3)


def cfg1(K: int = 1024, T: int = 30) -> Workload:
    """Rectangle (trap_hybrid 'hybrid-box'), diff-drive, K=1024, T=30, 2,000 boundary samples of
    the corridor_don080 obstacles."""
    fp = FootprintSpec.rect_cover([[0.0, 0.0]], [[0.5, 0.25]], "hybrid-box")
    params = MppiParams.from_json(CORRIDOR_MPPI, rollouts=K, horizon=T, seed=1)
    cloud = sample_boundaries(CORRIDOR_OBSTACLES, 2000)
    return Workload("cfg1_rect_diff_K1024_T30_N2k", fp, MotionModel.diff(),
                    KinematicLimits.from_json(CORRIDOR_LIMITS), params,
                    np.array([-6.0, 0.0, 0.0]), cloud,
                    Guidance([[-6.5, 0.0], [6.5, 0.0]], [6.0, 0.0, 0.0]),
                    "rect R=1, diff, K=1024, T=30, N=2000 corridor boundary samples")


def l12_footprint() -> FootprintSpec:
    """l_shape.json with every edge midpoint inserted: 12 vertices, identical geometry."""
    v = np.asarray(FOOTPRINTS["l_shape"], np.float64)
    out = []
    for i in range(len(v)):
        out.append(v[i])
        out.append(0.5 * (v[i] + v[(i + 1) % len(v)]))
    return FootprintSpec.polygon(np.array(out), "l_shape_12")


def clutter_discs(n_points: int, seed: int = 5, half: float = 10.0, clear: float = 1.5,
                  spacing: float = 0.05) -> np.ndarray:
    """Dense static clutter (Appendix A.2): disc k has centre (U(-10,10), U(-10,10)) and radius
    U(0.1,0.4) from uniform_range(5, k, 0/1/2); rejected within 1.5 m + r of the origin; each
    disc contributes max(8, ceil(2 pi r / 0.05)) boundary samples until N is reached."""
    pts = []
    total = 0
    k = 0
    while total < n_points:
        cx = float(uniform_range(seed, k, 0, -half, half))
        cy = float(uniform_range(seed, k, 1, -half, half))
        r = float(uniform_range(seed, k, 2, 0.1, 0.4))
        k += 1
        if math.hypot(cx, cy) < clear + r:
            continue
        m = max(8, math.ceil(2.0 * math.pi * r / spacing))
        m = min(m, n_points - total)
        a = 2.0 * math.pi * np.arange(m) / max(8, math.ceil(2.0 * math.pi * r / spacing))
        pts.append(np.stack([cx + r * np.cos(a), cy + r * np.sin(a)], axis=1))
        total += m
    return np.concatenate(pts)[:n_points]


def cfg2(K: int = 4096, T: int = 50, N: int = 10_000) -> Workload:
    """Non-convex 12-vertex L, diff-drive, K=4096, T=50, N=10k dense clutter (Appendix A.2)."""
    params = MppiParams.from_json(CORRIDOR_MPPI, rollouts=K, horizon=T, seed=1)
    return Workload("cfg2_L12_diff_K4096_T50_N10k", l12_footprint(), MotionModel.diff(),
                    KinematicLimits.from_json(CORRIDOR_LIMITS), params, np.zeros(3),
                    clutter_discs(N), Guidance([[0.0, 0.0], [8.0, 0.0]], [8.0, 0.0, 0.0]),
                    "12-vertex L polygon, diff, K=4096, T=50, N=10000 clutter")


def forklift_footprint() -> FootprintSpec:
    """Appendix A.3: chassis, mast, forks + pallet (R=3 rectangle cover)."""
    return FootprintSpec.rect_cover([[0.0, 0.0], [0.65, 0.0], [1.25, 0.0]],
                                    [[0.60, 0.45], [0.05, 0.40], [0.60, 0.60]], "forklift")


def aisle_cloud(n_points: int) -> np.ndarray:
    """Rack faces y = +-0.75 over x in [-5, 25] plus 0.1 m square uprights every 2.7 m behind
    each face; uniform arc-length samples to exactly n_points."""
    polys = [[[-5.0, 0.75], [25.0, 0.75], [25.0, 0.85], [-5.0, 0.85]],
             [[-5.0, -0.85], [25.0, -0.85], [25.0, -0.75], [-5.0, -0.75]]]
    x = -5.0
    while x <= 25.0:
        for s in (1.0, -1.0):
            y0 = s * 0.85
            polys.append([[x, y0], [x + 0.1, y0], [x + 0.1, y0 + s * 0.1], [x, y0 + s * 0.1]])
        x += 2.7
    return sample_boundaries(polys, n_points)


def cfg3(K: int = 8192, T: int = 60, N: int = 20_000) -> Workload:
    """Forklift + pallet rectangle cover, Ackermann (L=1.2), K=8192, T=60, N=20k aisle."""
    params = MppiParams.from_json(TRAP_MPPI, rollouts=K, horizon=T, seed=1)
    return Workload("cfg3_forklift_ack_K8192_T60_N20k", forklift_footprint(),
                    MotionModel.ackermann(1.2), KinematicLimits.from_json(TRAP_ACK_LIMITS), params,
                    np.zeros(3), aisle_cloud(N), Guidance([[0.0, 0.0], [20.0, 0.0]], [20.0, 0.0, 0.0]),
                    "forklift R=3 cover, ackermann, K=8192, T=60, N=20000 narrow aisle")


def star64_footprint() -> FootprintSpec:
    """Appendix A.4: 32-point star, a_k = 2 pi k/64 + pi/2, r = 1.0 (even k) / 0.45 (odd k)."""
    k = np.arange(64)
    a = 2.0 * math.pi * k / 64 + math.pi / 2
    r = np.where(k % 2 == 0, 1.0, 0.45)
    return FootprintSpec.polygon(np.stack([r * np.cos(a), r * np.sin(a)], axis=1), "star64")


def benchmark_queries(count: int, region_side: float, seed: int) -> np.ndarray:
    """bench.cpp:46-53."""
    half = region_side / 2.0
    i = np.arange(count, dtype=np.uint64)
    return np.stack([uniform_range(seed, i, 0, -half, half),
                     uniform_range(seed, i, 1, -half, half)], axis=1)


def cfg4_poses(P: int = 1000) -> np.ndarray:
    p = np.arange(P, dtype=np.uint64)
    return np.stack([uniform_range(2, p, 0, -5.0, 5.0), uniform_range(2, p, 1, -5.0, 5.0),
                     uniform_range(2, p, 2, -math.pi, math.pi)], axis=1)


def cfg4(P: int = 1000, N: int = 1_000_000):
    """Distance-only: 64-vertex concave star vs P poses x N points (10^9 pairs at default)."""
    return star64_footprint(), cfg4_poses(P), benchmark_queries(N, 50.0, 1)


def cfg5(K: int = 65536, T: int = 80, N: int = 50_000, cycle: int = 0) -> Workload:
    """Omni L-shape, K=65536, T=80, N=50k: 64 discs (r in U[0.2,0.5]) on 2-waypoint ping-pong
    trails (speed U[0,0.2] m/s) plus the two omni_gap walls; boundary samples rescaled to
    exactly N, regenerated per cycle (quasi-static within the horizon)."""
    polys = [w for w in OMNI_WALLS]
    t = cycle * 0.1
    for k in range(64):
        ax, ay = uniform_range(9, k, 0, -8.0, 8.0), uniform_range(9, k, 1, -8.0, 8.0)
        bx, by = uniform_range(9, k, 2, -8.0, 8.0), uniform_range(9, k, 3, -8.0, 8.0)
        r = uniform_range(9, k, 4, 0.2, 0.5)
        v = uniform_range(9, k, 5, 0.0, 0.2)
        L = math.hypot(bx - ax, by - ay)
        s = (v * t) % (2 * L) if L > 0 else 0.0
        s = s if s <= L else 2 * L - s
        f = s / L if L > 0 else 0.0
        cx, cy = ax + f * (bx - ax), ay + f * (by - ay)
        if math.hypot(cx + 4.0, cy) < 1.5 + r:
            cx += 3.0
        ang = 2 * math.pi * np.arange(24) / 24
        polys.append(np.stack([cx + r * np.cos(ang), cy + r * np.sin(ang)], axis=1))
    params = MppiParams.from_json(OMNI_MPPI, rollouts=K, horizon=T, seed=1)
    guide = [[-4.5, 0.0], [-1.8, 0.5003855879865172], [1.2, 0.5003855879865172],
             [2.0, -0.5003855879865172], [3.2, -0.5003855879865172], [5.3, 0.0]]
    return Workload("cfg5_omni_L_K65536_T80_N50k", footprint("l_shape"), MotionModel.omni(),
                    KinematicLimits.from_json(OMNI_LIMITS), params, np.array([-4.0, 0.0, 0.0]),
                    sample_boundaries(polys, N), Guidance(guide, [4.8, 0.0, 0.0]),
                    "omni L (B=6), K=65536, T=80, N=50000, moving discs + gap walls")


# trap_hybrid.json: the three mode families, the obstacles and the hybrid block.
TRAP_OBSTACLES = [
    [[-5.0, 0.8], [5.0, 0.8], [5.0, 1.1], [-5.0, 1.1]],
    [[-5.0, -1.15], [2.0, -1.15], [2.0, -0.5], [-5.0, -0.5]],
    [[3.25, -1.15], [5.0, -1.15], [5.0, -0.5], [3.25, -0.5]],
    [[1.7, -1.45], [3.55, -1.45], [3.55, -1.15], [1.7, -1.15]],
]


def trap_hybrid(K: int = 384, T: int = 25, N: int = 400):
    """The trap_hybrid fixture as a hybrid workload: (footprint, modes, params, hybrid params,
    q0, cloud, guidance). Cloud: N boundary samples of the four trap obstacles."""
    from .api import HybridMode, HybridParams
    fp = FootprintSpec.rect_cover([[0.0, 0.0]], [[0.5, 0.25]], "hybrid-box")
    modes = [
        HybridMode("ackermann", MotionModel.ackermann(0.5), KinematicLimits.from_json(TRAP_ACK_LIMITS)),
        HybridMode("parallel", MotionModel.parallel(), KinematicLimits.from_json(
            {"acc_max": [1.5], "acc_min": [-1.5], "steer_max": 1e9, "vel_max": [0.5], "vel_min": [-0.5]})),
        HybridMode("spin", MotionModel.spin(), KinematicLimits.from_json(
            {"acc_max": [4.0], "acc_min": [-4.0], "steer_max": 1e9, "vel_max": [1.0], "vel_min": [-1.0]})),
    ]
    params = MppiParams.from_json(TRAP_MPPI, rollouts=K, horizon=T, seed=1)
    hp = HybridParams(lambda_switch=3.0, tau_cool_max=5, v_min=0.05, omega_min=0.05,
                      noise_deadzone_v=0.01, noise_deadzone_omega=0.01)
    return (fp, modes, params, hp, np.array([2.625, -0.825, 0.0]),
            sample_boundaries(TRAP_OBSTACLES, N),
            Guidance([[2.625, -0.825], [2.625, 0.15], [-3.0, 0.0]], [-3.0, 0.0, 0.0]))


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg5": cfg5}


def cfg5_hybrid(K: int = 65536, T: int = 80, N: int = 50_000, cycle: int = 0):
    """Config 5's hybrid variant: the trap_hybrid mode families
    (Ackermann / parallel / spin, M = 3) on config 5's L footprint, cloud and guidance, K rollouts
    per family. Returns (footprint, modes, params, hybrid params, q0, cloud, guidance)."""
    wl = cfg5(K=K, T=T, N=N, cycle=cycle)
    _, modes, _, hp, _, _, _ = trap_hybrid()
    return (wl.footprint, modes, wl.params, hp, wl.q0, wl.cloud, wl.guidance)
