"""Host-side mirror of the reference's controller API (proj/include/exactmppi/*.hpp), backed by
the B200 C ABI. Names, argument meaning and error behaviour follow the reference:

  reference (C++)                               here
  FootprintSpec / PolygonFootprint::make /      FootprintSpec.polygon / .rect_cover
    RectangleCover::make (geometry.hpp:41-85)   (validation in the library; ValueError)
  MotionModel (kinematics.hpp:16-28)            MotionModel
  KinematicLimits (kinematics.hpp:51-63)        KinematicLimits
  MppiParams / TaskWeights (controller.hpp:13-35) MppiParams / TaskWeights
  Guidance (controller.hpp:38-41)               Guidance
  ObstacleSet (geometry.hpp:88-97)              ObstacleSet
  MppiController (controller.hpp:140-170)       MppiController
  evaluate_rollouts (controller.hpp:116-121)    Controller handle .evaluate_rollouts
  sample_perturbations (controller.hpp:107)     .sample_perturbations
  validate_nominal (controller.hpp:125-129)     .validate_nominal
  batch_signed_distance (geometry.hpp:142)      .batch_signed_distance
  min_signed_distance_at (geometry.hpp:150)     .min_signed_distance_at

std::invalid_argument maps to ValueError. Arrays are numpy float64 (uint8 masks).
"""
from __future__ import annotations

import ctypes as C
import threading
import json
import math
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _abi
from ._abi import check, dptr, fptr, u8ptr

K_EMPTY_MASK_DISTANCE = 1e6  # geometry.hpp:37
K_PADDED_COORDINATE = 1e9    # geometry.hpp:35


# ------------------------------------------------------------------------------ types
@dataclass
class WorldObstacle:
    """A scenario obstacle for sensing (world.hpp Obstacle): a polygon (vertices, CCW as
    PolygonFootprint stores them; CW input is reversed like PolygonFootprint::make) or a disc
    (center, radius), displaced by its current trail offset (obstacle_offset, world.cpp:159-164)."""
    vertices: np.ndarray | None = None
    center: Sequence[float] | None = None
    radius: float = 0.0
    offset: Sequence[float] = (0.0, 0.0)

    @staticmethod
    def polygon(vertices, offset=(0.0, 0.0)) -> "WorldObstacle":
        v = np.ascontiguousarray(np.asarray(vertices, np.float64).reshape(-1, 2))
        area2 = float(np.sum(v[:, 0] * np.roll(v[:, 1], -1) - v[:, 1] * np.roll(v[:, 0], -1)))
        if area2 < 0.0:
            v = np.ascontiguousarray(v[::-1])
        return WorldObstacle(vertices=v, offset=tuple(offset))

    @staticmethod
    def disc(center, radius, offset=(0.0, 0.0)) -> "WorldObstacle":
        return WorldObstacle(center=tuple(center), radius=float(radius), offset=tuple(offset))

    def _c(self):
        if self.vertices is not None:
            x = np.ascontiguousarray(self.vertices[:, 0])
            y = np.ascontiguousarray(self.vertices[:, 1])
            o = _abi.ExmWorldObstacle(_abi.OBSTACLE_POLYGON, x.size, dptr(x), dptr(y), 0.0,
                                      (C.c_double * 2)(*self.offset))
        else:
            x = np.array([self.center[0]], np.float64)
            y = np.array([self.center[1]], np.float64)
            o = _abi.ExmWorldObstacle(_abi.OBSTACLE_DISC, 1, dptr(x), dptr(y), self.radius,
                                      (C.c_double * 2)(*self.offset))
        return o, (x, y)


@dataclass
class Trail:
    """TrailMotion (world.hpp): >= 2 waypoints (the shape's coordinates sit at the first), speed
    (m/s), ping-pong (reflect at the ends) or clamp."""
    waypoints: np.ndarray
    speed: float
    ping_pong: bool = True

    def __post_init__(self):
        self.waypoints = np.ascontiguousarray(np.asarray(self.waypoints, np.float64).reshape(-1, 2))


def world_trails_c(trails, n):
    """ctypes array of exm_world_trail (None entries: static) plus the buffers it points into."""
    arr = (_abi.ExmWorldTrail * max(n, 1))()
    keep = []
    for i, t in enumerate(trails or []):
        if t is None:
            continue
        wp = t.waypoints
        keep.append(wp)
        arr[i] = _abi.ExmWorldTrail(wp.shape[0], 1 if t.ping_pong else 0, dptr(wp), float(t.speed))
    return arr, keep


class DeviceWorld:
    """Moving obstacles kept on the device (exm_world_*): step_world (world.cpp:127-157) and
    sense() (:182-243) with the current obstacle offsets, no host round trip of the world state."""

    def __init__(self, engine, obstacles, trails, sensor_range: float, budget: int, seed: int):
        self.eng, self.budget, self.n = engine, int(budget), len(obstacles)
        self.lib = engine.lib
        arr, keep = world_obstacles_c(obstacles)
        tarr, tkeep = world_trails_c(trails, self.n)
        w = C.POINTER(_abi.ExmWorld)()
        check(self.lib.exm_world_create(engine.h, arr, tarr, self.n, float(sensor_range),
                                        self.budget, int(seed), C.byref(w)))
        del keep, tkeep
        self.w = w

    def step(self, dt: float):
        check(self.lib.exm_world_step(self.w, float(dt)))

    def sense(self, robot, sample_key: int) -> "ObstacleSet":
        pts = np.empty((self.budget, 2))
        mask = np.empty(self.budget, np.uint8)
        n = C.c_int32()
        r = np.ascontiguousarray(np.asarray(robot, np.float64).reshape(3))
        check(self.lib.exm_world_sense(self.w, dptr(r), int(sample_key), dptr(pts), u8ptr(mask),
                                       C.byref(n)))
        return ObstacleSet(pts, mask)

    def state(self):
        arc = np.empty(max(self.n, 1))
        d = np.empty(max(self.n, 1), np.int32)
        off = np.empty((max(self.n, 1), 2))
        check(self.lib.exm_world_state(self.w, dptr(arc), d.ctypes.data_as(C.POINTER(C.c_int32)),
                                       dptr(off)))
        return arc[: self.n], d[: self.n], off[: self.n]

    def close(self):
        if getattr(self, "w", None):
            self.lib.exm_world_destroy(self.w)
            self.w = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def world_obstacles_c(obstacles):
    """ctypes array of exm_world_obstacle plus the buffers it points into."""
    items = [o._c() for o in obstacles]
    arr = (_abi.ExmWorldObstacle * max(len(items), 1))(*[it[0] for it in items])
    return arr, [it[1] for it in items]


@dataclass
class FootprintSpec:
    """Exactly one of a simple polygon (CCW, validated by the library) or a rectangle cover."""
    kind: int
    a: np.ndarray  # polygon: vertices (n,2); cover: centres (n,2)
    b: np.ndarray | None = None  # cover: half extents (n,2)
    name: str = ""

    @staticmethod
    def polygon(vertices, name: str = "polygon") -> "FootprintSpec":
        v = np.ascontiguousarray(np.asarray(vertices, dtype=np.float64).reshape(-1, 2))
        return FootprintSpec(_abi.FOOTPRINT_POLYGON, v, None, name)

    @staticmethod
    def rect_cover(centers, half_extents, name: str = "cover") -> "FootprintSpec":
        c = np.ascontiguousarray(np.asarray(centers, dtype=np.float64).reshape(-1, 2))
        h = np.ascontiguousarray(np.asarray(half_extents, dtype=np.float64).reshape(-1, 2))
        return FootprintSpec(_abi.FOOTPRINT_RECT_COVER, c, h, name)

    @staticmethod
    def from_json(obj) -> "FootprintSpec":
        """Fixture schema of proj/fixtures/footprints/*.json (scenario_io.cpp footprint block)."""
        if isinstance(obj, str):
            with open(obj) as f:
                obj = json.load(f)
        if obj["kind"] == "polygon":
            return FootprintSpec.polygon(obj["vertices"], obj.get("name", ""))
        rects = obj["rectangles"]
        return FootprintSpec.rect_cover([r["center"] for r in rects],
                                        [r["half_extent"] for r in rects], obj.get("name", ""))

    def is_polygon(self) -> bool:
        return self.kind == _abi.FOOTPRINT_POLYGON

    def count(self) -> int:
        return int(self.a.shape[0])

    def all_vertices(self) -> np.ndarray:
        if self.is_polygon():
            return self.a.copy()
        out = []
        for (cx, cy), (hx, hy) in zip(self.a, self.b):
            out += [(cx - hx, cy - hy), (cx + hx, cy - hy), (cx + hx, cy + hy), (cx - hx, cy + hy)]
        return np.array(out)

    def bounding_radius(self) -> float:
        return float(np.max(np.hypot(*self.all_vertices().T)))

    def _c(self):
        """exm_footprint view; keeps the numpy buffers alive via the returned tuple."""
        cols = [np.ascontiguousarray(self.a[:, 0]), np.ascontiguousarray(self.a[:, 1])]
        if self.b is not None:
            cols += [np.ascontiguousarray(self.b[:, 0]), np.ascontiguousarray(self.b[:, 1])]
        else:
            cols += [None, None]
        fp = _abi.ExmFootprint(self.kind, self.count(), dptr(cols[0]), dptr(cols[1]),
                               dptr(cols[2]), dptr(cols[3]))
        return fp, cols

    def cull_boxes(self):
        """(aabb[4], boxes[n, 4] as {cx, cy, hx, hy}): the body-frame cull geometry of the SDF
        kernels (exm_footprint_cull_boxes; host-only, validates like exm_create)."""
        fp, keep = self._c()
        aabb = np.zeros(4, np.float32)
        boxes = np.zeros(12, np.float32)
        n = C.c_int32()
        check(_abi.load_library().exm_footprint_cull_boxes(C.byref(fp), fptr(aabb), fptr(boxes),
                                                           C.byref(n)))
        return aabb, boxes.reshape(3, 4)[: n.value]


@dataclass
class MotionModel:
    tag: int = _abi.MODEL_DIFF
    wheelbase: float = 0.0

    @staticmethod
    def diff():
        return MotionModel(_abi.MODEL_DIFF)

    @staticmethod
    def ackermann(wheelbase: float):
        if wheelbase <= 0.0:
            raise ValueError("ackermann wheelbase must be positive")
        return MotionModel(_abi.MODEL_ACKERMANN, wheelbase)

    @staticmethod
    def omni():
        return MotionModel(_abi.MODEL_OMNI)

    @staticmethod
    def spin():
        return MotionModel(_abi.MODEL_SPIN)

    @staticmethod
    def parallel():
        return MotionModel(_abi.MODEL_PARALLEL)

    @staticmethod
    def from_name(name: str, wheelbase: float = 0.0):
        table = {"diff": MotionModel.diff, "omni": MotionModel.omni, "spin": MotionModel.spin,
                 "parallel": MotionModel.parallel}
        if name == "ackermann":
            return MotionModel.ackermann(wheelbase)
        if name not in table:
            raise ValueError("unknown motion model: " + name)
        return table[name]()

    def control_dim(self) -> int:
        return {0: 2, 1: 2, 2: 3, 3: 1, 4: 1}[self.tag]

    def _c(self):
        return _abi.ExmModel(self.tag, 0, self.wheelbase)


@dataclass
class ComponentLimit:
    vel_min: float = -1.0
    vel_max: float = 1.0
    acc_min: float = -1e9
    acc_max: float = 1e9


@dataclass
class KinematicLimits:
    component: list = field(default_factory=lambda: [ComponentLimit() for _ in range(3)])
    steer_max: float = 0.6

    @staticmethod
    def unbounded():
        return KinematicLimits([ComponentLimit(-1e9, 1e9, -1e18, 1e18) for _ in range(3)], 1e9)

    @staticmethod
    def from_json(obj):
        lim = KinematicLimits()
        for key, attr in (("vel_min", "vel_min"), ("vel_max", "vel_max"), ("acc_min", "acc_min"),
                          ("acc_max", "acc_max")):
            for i, v in enumerate(obj.get(key, [])):
                setattr(lim.component[i], attr, float(v))
        lim.steer_max = float(obj.get("steer_max", lim.steer_max))
        return lim

    def _c(self):
        c = self.component
        return _abi.ExmLimits((C.c_double * 3)(*[x.vel_min for x in c]),
                              (C.c_double * 3)(*[x.vel_max for x in c]),
                              (C.c_double * 3)(*[x.acc_min for x in c]),
                              (C.c_double * 3)(*[x.acc_max for x in c]), self.steer_max)


@dataclass
class TaskWeights:
    goal_pos: float = 1.0
    goal_head: float = 0.5
    xtrack: float = 2.0
    progress: float = 2.0


@dataclass
class MppiParams:
    rollouts: int = 1000
    horizon: int = 50
    dt: float = 0.1
    lambda_: float = 1.0
    sigma: tuple = (0.3, 0.3, 0.3)
    d_safe: float = 0.1
    w_coll: float = 1e6
    w_rep: float = 50.0
    w_inf: float = 1e9
    task: TaskWeights = field(default_factory=TaskWeights)
    w_ctrl: float = 0.02
    seed: int = 0

    @staticmethod
    def from_json(obj, **override):
        p = MppiParams(rollouts=int(obj["rollouts"]), horizon=int(obj["horizon"]),
                       dt=float(obj["dt"]), lambda_=float(obj["lambda"]),
                       sigma=tuple(list(obj["sigma"]) + [0.3] * (3 - len(obj["sigma"]))),
                       d_safe=float(obj["d_safe"]), w_coll=float(obj["w_coll"]),
                       w_rep=float(obj["w_rep"]), w_inf=float(obj["w_inf"]),
                       task=TaskWeights(float(obj["w_goal_pos"]), float(obj["w_goal_head"]),
                                        float(obj["w_xtrack"]), float(obj["w_progress"])),
                       w_ctrl=float(obj["w_ctrl"]))
        for k, v in override.items():
            setattr(p, k, v)
        return p

    def _c(self):
        s = list(self.sigma) + [0.3] * (3 - len(self.sigma))
        return _abi.ExmParams(self.rollouts, self.horizon, self.dt, self.lambda_,
                              (C.c_double * 3)(*s[:3]), self.d_safe, self.w_coll, self.w_rep,
                              self.w_inf, self.task.goal_pos, self.task.goal_head,
                              self.task.xtrack, self.task.progress, self.w_ctrl,
                              int(self.seed) & 0xFFFFFFFFFFFFFFFF)


@dataclass
class Guidance:
    path: np.ndarray
    goal: np.ndarray

    def __post_init__(self):
        self.path = np.ascontiguousarray(np.asarray(self.path, dtype=np.float64).reshape(-1, 2))
        self.goal = np.ascontiguousarray(np.asarray(self.goal, dtype=np.float64).reshape(3))


class _PinnedBuffer:
    """exm_host_alloc'd bytes, freed with the object."""

    def __init__(self, nbytes: int):
        self.lib = _abi.load_library()
        self.n = max(int(nbytes), 1)
        self.p = self.lib.exm_host_alloc(self.n)
        if not self.p:
            raise MemoryError("exm_host_alloc failed")

    def view(self):
        v = (C.c_uint8 * self.n).from_address(self.p)
        v._owner = self  # numpy views hold the ctypes array, which holds the allocation
        return v

    def __del__(self):
        if getattr(self, "p", None):
            self.lib.exm_host_free(self.p)
            self.p = None


@dataclass
class ObstacleSet:
    points: np.ndarray
    mask: np.ndarray

    def __post_init__(self):
        self.points = np.ascontiguousarray(np.asarray(self.points, dtype=np.float64).reshape(-1, 2))
        self.mask = np.ascontiguousarray(np.asarray(self.mask, dtype=np.uint8).reshape(-1))
        if self.mask.size != self.points.shape[0]:
            raise ValueError("obstacle mask length must equal the number of points")

    @staticmethod
    def padded(valid_points, capacity: int) -> "ObstacleSet":
        v = np.asarray(valid_points, dtype=np.float64).reshape(-1, 2)
        if v.shape[0] > capacity:
            raise ValueError("more valid points than obstacle-set capacity")
        pts = np.full((capacity, 2), K_PADDED_COORDINATE)
        pts[: v.shape[0]] = v
        mask = np.zeros(capacity, np.uint8)
        mask[: v.shape[0]] = 1
        return ObstacleSet(pts, mask)

    @staticmethod
    def pinned(points, mask=None) -> "ObstacleSet":
        """The same set in page-locked host memory (exm_host_alloc): a sensor loop that writes
        its cloud into these arrays gets DMA uploads without the driver's staging copy."""
        src = ObstacleSet(points, np.ones(len(points), np.uint8) if mask is None else mask)
        n = src.points.shape[0]
        buf = _PinnedBuffer(16 * n + n)
        pts = np.frombuffer(buf.view(), dtype=np.float64, count=2 * n).reshape(n, 2)
        m = np.frombuffer(buf.view(), dtype=np.uint8, count=n, offset=16 * n)
        pts[:] = src.points
        m[:] = src.mask
        out = ObstacleSet(pts, m)
        out._pinned = buf  # keeps the allocation alive with the arrays
        return out

    @staticmethod
    def all_masked(capacity: int) -> "ObstacleSet":
        return ObstacleSet.padded(np.zeros((0, 2)), capacity)

    def capacity(self) -> int:
        return int(self.points.shape[0])

    def valid_count(self) -> int:
        return int(np.count_nonzero(self.mask))


@dataclass
class ControlDecision:
    command: np.ndarray
    validated: bool
    nominal: np.ndarray
    best_cost: float
    weight_entropy: float
    nominal_cost: float
    nominal_d_min: np.ndarray
    argmin: int


@dataclass
class RolloutBatch:
    rollouts: int
    horizon: int
    perturbations: np.ndarray  # (K, T, dim)
    controls: np.ndarray       # (K, T, dim)
    states: np.ndarray         # (K, T+1, 3)
    d_min: np.ndarray          # (K, T)
    costs: np.ndarray          # (K,)
    unsafe: np.ndarray         # (K,) uint8


# ------------------------------------------------------------------------------ engine
class _CallScratch:
    """Fixed-address host buffers of Engine.control_cycle_raw (one set per calling thread)."""

    def __init__(self, horizon: int):
        self.q0 = np.zeros(3)
        self.q0addr = self.q0.ctypes.data
        self.dmin = np.zeros(int(horizon))
        self.dec = _abi.ExmDecision()
        self.dec.nominal_dmin = dptr(self.dmin)
        self.decp = C.addressof(self.dec)


class Engine:
    """One device handle (libexm_b200.so). Sized at construction for (K, T, n_cap, guide_cap)."""

    def __init__(self, model: MotionModel, limits: KinematicLimits, footprint: FootprintSpec,
                 params: MppiParams, n_cap: int = 1024, guide_cap: int = 64, device: int = 0):
        self.lib = _abi.load_library()
        self.model, self.limits, self.footprint, self.params = model, limits, footprint, params
        self.dim = model.control_dim()
        self.n_cap, self.guide_cap = int(n_cap), int(guide_cap)
        fp, keep = footprint._c()
        self._keep = keep
        h = C.POINTER(_abi.ExmHandle)()
        m, l, p = model._c(), limits._c(), params._c()
        check(self.lib.exm_create(C.byref(fp), C.byref(m), C.byref(l), C.byref(p), self.n_cap,
                                  self.guide_cap, int(device), C.byref(h)))
        self.h = h
        # lean host path of control_cycle_raw: fixed-address scratch and cached addresses
        self._cc = _abi.fast_control_cycle(self.lib)
        self._hv = C.cast(h, C.c_void_p).value
        # per-thread call scratch (q0, decision, nominal d_min): the library serialises calls on
        # one handle, and each thread keeps its own host buffers
        self._tls = threading.local()
        self._addrs: dict = {}

    def _addr(self, a, dtype=np.float64, min_size: int = 0, size: int = -1):
        """Address of a C-contiguous array of `dtype`, cached per array object (the cache holds
        a reference, so an id cannot be reused while its entry lives and the array cannot be
        resized in place). Sizes are checked on a cache miss. Only long-lived arrays (state,
        guidance, obstacle buffers) go through here."""
        if a is None:
            return None
        ent = self._addrs.get(id(a))
        if ent is not None and ent[0] is a:
            return ent[1]
        if a.dtype != dtype or not a.flags.c_contiguous:
            raise ValueError("array must be C-contiguous " + np.dtype(dtype).name)
        if a.size < min_size or (size >= 0 and a.size != size):
            raise ValueError(f"array has {a.size} elements, expected "
                             f"{size if size >= 0 else f'at least {min_size}'}")
        if len(self._addrs) >= 16:
            self._addrs.clear()
        addr = a.ctypes.data
        self._addrs[id(a)] = (a, addr)
        return addr

    def close(self):
        if getattr(self, "h", None):
            self.lib.exm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- helpers
    def _cloud(self, obstacles: ObstacleSet | np.ndarray, mask=None):
        if isinstance(obstacles, ObstacleSet):
            pts, mask = obstacles.points, obstacles.mask
        else:
            pts = np.ascontiguousarray(np.asarray(obstacles, np.float64).reshape(-1, 2))
        if mask is not None:
            mask = np.ascontiguousarray(np.asarray(mask, np.uint8).reshape(-1))
        if pts.shape[0] > self.n_cap:
            raise ValueError("point count exceeds obstacle-set capacity")
        return pts, mask

    def _vec3(self, v):
        return np.ascontiguousarray(np.asarray(v, np.float64).reshape(3))

    def _u(self, u):
        out = np.zeros(3)
        u = np.asarray(u, np.float64).reshape(-1)
        out[: u.size] = u
        return out

    # -- reference free functions
    def sample_perturbations(self, seed: int, cycle: int) -> np.ndarray:
        P = self.params
        eps = np.empty((P.rollouts, P.horizon, self.dim))
        check(self.lib.exm_sample_perturbations(self.h, seed, cycle, dptr(eps)))
        return eps

    def evaluate_rollouts(self, q0, nominal, perturbations, obstacles, guidance: Guidance,
                          u_prev) -> RolloutBatch:
        P = self.params
        K, T, D = P.rollouts, P.horizon, self.dim
        eps = np.ascontiguousarray(np.asarray(perturbations, np.float64))
        if eps.size != K * T * D:
            raise ValueError("perturbation array does not match K*T")
        nom = np.ascontiguousarray(np.asarray(nominal, np.float64).reshape(-1))
        if nom.size != T * D:
            raise ValueError("nominal length does not match horizon")
        pts, mask = self._cloud(obstacles)
        controls = np.empty((K, T, D))
        states = np.empty((K, T + 1, 3))
        dmin = np.empty((K, T))
        costs = np.empty(K)
        unsafe = np.empty(K, np.uint8)
        check(self.lib.exm_evaluate_rollouts(
            self.h, dptr(self._vec3(q0)), dptr(nom), dptr(eps), dptr(pts), u8ptr(mask),
            pts.shape[0], dptr(guidance.path), guidance.path.shape[0], dptr(guidance.goal),
            dptr(self._u(u_prev)), dptr(controls), dptr(states), dptr(dmin), dptr(costs),
            u8ptr(unsafe)))
        return RolloutBatch(K, T, eps.reshape(K, T, D), controls, states, dmin, costs, unsafe)

    def validate_nominal(self, nominal, q0, obstacles, guidance: Guidance, u_prev):
        T, D = self.params.horizon, self.dim
        nom = np.ascontiguousarray(np.asarray(nominal, np.float64).reshape(-1))
        if nom.size != T * D:
            raise ValueError("nominal length does not match horizon")
        pts, mask = self._cloud(obstacles)
        valid = C.c_int32()
        dmin = np.empty(T)
        cost = C.c_double()
        check(self.lib.exm_validate_nominal(
            self.h, dptr(nom), dptr(self._vec3(q0)), dptr(pts), u8ptr(mask), pts.shape[0],
            dptr(guidance.path), guidance.path.shape[0], dptr(guidance.goal),
            dptr(self._u(u_prev)), C.byref(valid), dptr(dmin), C.byref(cost)))
        return bool(valid.value), dmin, float(cost.value)

    def control_cycle_raw(self, q0, obstacles, guidance: Guidance, nominal: np.ndarray,
                          u_prev: np.ndarray, cycle: int, eps=None) -> ControlDecision:
        """One MPPI step with explicit controller state (nominal and u_prev updated in place)."""
        if isinstance(obstacles, ObstacleSet) and obstacles.points.shape[0] <= self.n_cap:
            pts, mask = obstacles.points, obstacles.mask  # validated at ObstacleSet creation
        else:
            pts, mask = self._cloud(obstacles)
        sc = getattr(self._tls, "s", None)
        if sc is None:
            sc = self._tls.s = _CallScratch(self.params.horizon)
        q = sc.q0
        q[0], q[1], q[2] = q0[0], q0[1], q0[2]
        eps_addr = None
        if eps is not None:  # injected noise: not cached (a fresh array per call)
            eps_arr = np.ascontiguousarray(np.asarray(eps, np.float64))
            if eps_arr.size != self.params.rollouts * self.params.horizon * self.dim:
                raise ValueError("perturbation array does not match K*T")
            eps_addr = eps_arr.ctypes.data
        A = self._addr
        rc = self._cc(self._hv, sc.q0addr, A(pts), A(mask, np.uint8, size=pts.shape[0]),
                      pts.shape[0], A(guidance.path), guidance.path.shape[0], A(guidance.goal),
                      A(nominal, size=self.params.horizon * self.dim), A(u_prev, min_size=self.dim),
                      int(cycle), eps_addr, sc.decp)
        if rc:
            check(rc)
        dec = sc.dec
        D = self.dim
        cmd = np.empty(D)
        c = dec.command
        for i in range(D):
            cmd[i] = c[i]
        return ControlDecision(cmd, bool(dec.validated), nominal.reshape(-1, D).copy(),
                               dec.best_cost, dec.weight_entropy, dec.nominal_cost,
                               sc.dmin.copy(), dec.argmin)

    def batch_signed_distance(self, queries) -> np.ndarray:
        q = np.ascontiguousarray(np.asarray(queries, np.float64).reshape(-1, 2))
        out = np.empty(q.shape[0])
        check(self.lib.exm_batch_signed_distance(self.h, dptr(q), q.shape[0], dptr(out)))
        return out

    def sdf_batch(self, poses, points, mask=None, per_pair: bool = False):
        """Per-pose min_signed_distance_at (and optionally every per-pair value, float32)."""
        ps = np.ascontiguousarray(np.asarray(poses, np.float64).reshape(-1, 3))
        pts = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 2))
        m = None if mask is None else np.ascontiguousarray(np.asarray(mask, np.uint8))
        mins = np.empty(ps.shape[0])
        pairs = np.empty((ps.shape[0], pts.shape[0]), np.float32) if per_pair else None
        check(self.lib.exm_sdf_batch(self.h, dptr(ps), ps.shape[0], dptr(pts), u8ptr(m),
                                     pts.shape[0], fptr(pairs), dptr(mins)))
        return (mins, pairs) if per_pair else mins

    def min_signed_distance_at(self, pose, obstacles: ObstacleSet) -> float:
        return float(self.sdf_batch(np.asarray(pose).reshape(1, 3), obstacles.points,
                                    obstacles.mask)[0])

    # -- resident stepping (benchmarks / serving loops)
    def stage(self, q0, obstacles, guidance: Guidance, nominal, u_prev, cycle: int = 0):
        pts, mask = self._cloud(obstacles)
        nom = np.ascontiguousarray(np.asarray(nominal, np.float64).reshape(-1))
        check(self.lib.exm_stage_inputs(self.h, dptr(self._vec3(q0)), dptr(pts), u8ptr(mask),
                                        pts.shape[0], dptr(guidance.path),
                                        guidance.path.shape[0], dptr(guidance.goal), dptr(nom),
                                        dptr(self._u(u_prev)), int(cycle)))

    def run_resident(self, n_steps: int):
        check(self.lib.exm_run_resident(self.h, int(n_steps)))

    def read_resident(self):
        T, D = self.params.horizon, self.dim
        nom = np.empty(T * D)
        up = np.empty(3)
        dmin = np.empty(T)
        dec = _abi.ExmDecision()
        dec.nominal_dmin = dptr(dmin)
        check(self.lib.exm_read_resident(self.h, dptr(nom), dptr(up), C.byref(dec)))
        return ControlDecision(np.array(dec.command[:D]), bool(dec.validated), nom.reshape(T, D),
                               dec.best_cost, dec.weight_entropy, dec.nominal_cost, dmin,
                               dec.argmin)

    def sdf_stage(self, poses, points, mask=None):
        ps = np.ascontiguousarray(np.asarray(poses, np.float64).reshape(-1, 3))
        pts = np.ascontiguousarray(np.asarray(points, np.float64).reshape(-1, 2))
        m = None if mask is None else np.ascontiguousarray(np.asarray(mask, np.uint8))
        check(self.lib.exm_sdf_stage(self.h, dptr(ps), ps.shape[0], dptr(pts), u8ptr(m),
                                     pts.shape[0]))
        self._sdf_shape = (ps.shape[0], pts.shape[0])

    def sdf_run_resident(self, n_steps: int, want_pairs: bool):
        check(self.lib.exm_sdf_run_resident(self.h, int(n_steps), 1 if want_pairs else 0))

    def sdf_read(self, per_pair: bool = False):
        P, N = self._sdf_shape
        mins = np.empty(P)
        pairs = np.empty((P, N), np.float32) if per_pair else None
        check(self.lib.exm_sdf_read(self.h, fptr(pairs), dptr(mins)))
        return mins, pairs

    def sense(self, obstacles, robot, sensor_range: float, budget: int, seed: int,
              sample_key: int):
        """sense(scenario, state, robot, sample_key) on the device (exm_sense,
        world.cpp:182-243) -> ObstacleSet padded to `budget` (points (budget, 2), mask)."""
        arr, keep = world_obstacles_c(obstacles)
        pts = np.empty((budget, 2))
        mask = np.empty(budget, np.uint8)
        n = C.c_int32()
        check(self.lib.exm_sense(self.h, arr, len(obstacles), dptr(self._vec3(robot)),
                                 float(sensor_range), int(budget), int(seed), int(sample_key),
                                 dptr(pts), u8ptr(mask), C.byref(n)))
        del keep
        return ObstacleSet(pts, mask)

    def world(self, obstacles, trails, sensor_range: float, budget: int, seed: int) -> DeviceWorld:
        """A device world on this handle's device and stream (exm_world_create)."""
        return DeviceWorld(self, obstacles, trails, sensor_range, budget, seed)

    def set_sdf_caps(self, caps):
        """Per-step cap hints of the culled SDF (exm_set_sdf_caps; exact for any values)."""
        c = np.ascontiguousarray(np.broadcast_to(np.asarray(caps, np.float32),
                                                 (self.params.horizon,)))
        check(self.lib.exm_set_sdf_caps(self.h, fptr(c)))

    def cull_stats(self):
        """(pairs that reached a point test, pairs that reached the exact SDF) for the last
        resident step's poses (re-runs the SDF once with counters)."""
        a, b = C.c_int64(), C.c_int64()
        check(self.lib.exm_sdf_cull_stats(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def stream_ptr(self) -> int:
        return int(self.lib.exm_stream(self.h) or 0)

    def step_stats(self):
        n = C.c_int32()
        ms = C.c_float()
        pairs = C.c_int64()
        check(self.lib.exm_step_stats(self.h, C.byref(n), C.byref(ms), C.byref(pairs)))
        return {"launches_per_step": n.value, "sdf_ms": ms.value, "sdf_pairs": pairs.value}

    # -- multi-GPU
    @staticmethod
    def nccl_unique_id() -> bytes:
        lib = _abi.load_library()
        buf = (C.c_uint8 * 128)()
        check(lib.exm_nccl_unique_id(buf))
        return bytes(buf)

    def attach_comm(self, rank: int, world: int, uid: bytes | None):
        """Shard this handle as rank `rank` of `world` over an NCCL communicator built from `uid`
        (any world, a 1-rank communicator included); uid None with world 1 detaches."""
        buf = None if uid is None else (C.c_uint8 * 128)(*uid)
        check(self.lib.exm_attach_comm(self.h, int(rank), int(world), buf))

    def set_shard(self, rank: int, world: int):
        """Shard without a communicator (several shard handles on one device, sharded_cycle)."""
        check(self.lib.exm_set_shard(self.h, int(rank), int(world)))

    @staticmethod
    def sharded_cycle(shards, q0, obstacles, guidance: Guidance, nominals, u_prevs, cycle: int,
                      eps=None):
        """One control step on G shard engines (shards[g] set to rank g of G) on one device,
        the block partials exchanged between them as the ranks' all-gather would. nominals
        (G, T*dim) and u_prevs (G, 3) are updated in place; returns G decisions."""
        G = len(shards)
        e0 = shards[0]
        pts, mask = e0._cloud(obstacles) if not isinstance(obstacles, ObstacleSet) else (
            obstacles.points, obstacles.mask)
        hs = (C.POINTER(_abi.ExmHandle) * G)(*[e.h for e in shards])
        decs = (_abi.ExmDecision * G)()
        dmins = [np.zeros(e0.params.horizon) for _ in range(G)]
        for g in range(G):
            decs[g].nominal_dmin = dptr(dmins[g])
        assert nominals.dtype == np.float64 and nominals.flags.c_contiguous
        assert u_prevs.dtype == np.float64 and u_prevs.flags.c_contiguous and u_prevs.shape == (G, 3)
        eps_arr = None if eps is None else np.ascontiguousarray(np.asarray(eps, np.float64))
        check(e0.lib.exm_sharded_cycle(hs, G, dptr(e0._vec3(q0)), dptr(pts), u8ptr(mask),
                                       pts.shape[0], dptr(guidance.path), guidance.path.shape[0],
                                       dptr(guidance.goal), dptr(nominals), dptr(u_prevs),
                                       int(cycle), dptr(eps_arr), decs))
        D = e0.dim
        return [ControlDecision(np.array(decs[g].command[:D]), bool(decs[g].validated),
                                nominals[g].reshape(-1, D).copy(), decs[g].best_cost,
                                decs[g].weight_entropy, decs[g].nominal_cost, dmins[g],
                                decs[g].argmin) for g in range(G)]

    # -- options and diagnostics
    def set_option(self, option: int, value: int):
        check(self.lib.exm_set_option(self.h, int(option), int(value)))

    def set_sdf_mode(self, mode: str):
        """Signed-distance kernel selection (tests / A/B): auto, brute, nochunk, thread, warp,
        cta, persist, nocap."""
        self.set_option(_abi.OPT_SDF_MODE, _abi.SDF_MODES[mode])

    def set_sdf_map(self, mapping: str):
        """Lanes <-> poses of the thread-per-pose SDF: "tuned" (default: chosen on the first
        steps), "rmajor" (a rollout's consecutive steps per warp), "hmajor" (consecutive rollouts
        at one step per warp)."""
        self.set_option(_abi.OPT_SDF_MAP, {"tuned": 0, "rmajor": 1, "hmajor": 2}[mapping])

    def set_sdf_threshold(self, on: bool):
        """True (default): the control cycle resolves rollout minima exactly only below d_safe
        (the decision is unchanged: the obstacle cost is 0 and the rollout safe at or above it);
        False: every rollout minimum exact. evaluate_rollouts is always exact."""
        self.set_option(_abi.OPT_SDF_THRESHOLD, 1 if on else 0)

    def set_sdf_fp64(self, on: bool):
        """True: evaluate_rollouts computes its minima (and the costs built on them) in FP64 with
        the reference's own arithmetic (min_signed_distance_at over PreparedFootprint::sd,
        geometry.cpp:260-295, :357-375), brute force; False (default): the FP32 culled kernels.
        The control cycle is not affected."""
        self.set_option(_abi.OPT_SDF_FP64, 1 if on else 0)

    def last_sdf_path(self):
        """What the last rollout / validation SDF launches ran (kernel 0 thread, 1 warp, 2 CTA
        per pose; chunk; persistent; hmajor)."""
        r, v = _abi.ExmSdfPath(), _abi.ExmSdfPath()
        check(self.lib.exm_last_sdf_path(self.h, C.byref(r), C.byref(v)))
        as_dict = lambda x: {f: getattr(x, f) for f, _ in x._fields_}  # noqa: E731
        return as_dict(r), as_dict(v)

    def sdf_work_stats(self) -> dict:
        """Work counters of the rollout SDF over the last step's poses (re-runs it once)."""
        c = (C.c_int64 * _abi.SDF_NCOUNT)()
        check(self.lib.exm_sdf_work_stats(self.h, c))
        return dict(zip(_abi.SDF_COUNTERS, list(c)))

    def host_timing(self):
        us = np.zeros(4)
        n = C.c_int64()
        check(self.lib.exm_host_timing(self.h, dptr(us), C.byref(n)))
        return {"stage_h2d_us": us[0], "launch_us": us[1], "wait_us": us[2], "unpack_us": us[3],
                "calls": n.value}


class MppiController:
    """MppiController (controller.hpp:140-170): the object keeps nominal_, u_prev_ and cycle_
    (controller.hpp:167-169); each control_cycle runs one MPPI step on the B200."""

    def __init__(self, model: MotionModel, limits: KinematicLimits, footprint: FootprintSpec,
                 params: MppiParams, threads: int = 1, n_cap: int = 1024, guide_cap: int = 64,
                 device: int = 0):
        del threads  # the reference's std::thread count; the GPU path has no equivalent knob
        self.engine = Engine(model, limits, footprint, params, n_cap, guide_cap, device)
        self._model, self._params = model, params
        self.dim = model.control_dim()
        self._nominal = np.zeros(params.horizon * self.dim)
        self._u_prev = np.zeros(3)
        self._cycle = 0

    def warm_start(self, measured):  # controller.cpp:296-300
        lim = self.engine.limits
        m = np.zeros(3)
        m[: self.dim] = np.asarray(measured, np.float64).reshape(-1)[: self.dim]
        u = _clamp_control(self._model, lim, self._params.dt, m, m)
        self._nominal = np.tile(u[: self.dim], self._params.horizon).astype(np.float64)
        self._u_prev = u.copy()

    def set_rate_anchor(self, u):
        self._u_prev = np.zeros(3)
        self._u_prev[: self.dim] = np.asarray(u, np.float64).reshape(-1)[: self.dim]

    def control_cycle(self, q0, obstacles: ObstacleSet, guidance: Guidance,
                      eps=None) -> ControlDecision:
        d = self.engine.control_cycle_raw(q0, obstacles, guidance, self._nominal, self._u_prev,
                                          self._cycle, eps)
        self._cycle += 1
        return d

    def nominal(self) -> np.ndarray:
        return self._nominal.reshape(self._params.horizon, self.dim).copy()

    def last_command(self) -> np.ndarray:
        return self._u_prev[: self.dim].copy()

    def cycle_index(self) -> int:
        return self._cycle

    def params(self) -> MppiParams:
        return self._params

    def model(self) -> MotionModel:
        return self._model


def _clamp_control(model: MotionModel, lim: KinematicLimits, dt: float, u, prev):
    """clamp_control (kinematics.cpp:99-117) for the host-side warm start only."""
    out = np.zeros(3)
    for i in range(model.control_dim()):
        c = lim.component[i]
        lo, hi = c.vel_min, c.vel_max
        if model.tag == _abi.MODEL_ACKERMANN and i == 1:
            lo, hi = max(lo, -lim.steer_max), min(hi, lim.steer_max)
        v = lo if u[i] < lo else (hi if hi < u[i] else u[i])
        a, b = prev[i] + c.acc_min * dt, prev[i] + c.acc_max * dt
        out[i] = a if v < a else (b if b < v else v)
    return out


def pose_array(poses: Sequence) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(poses, np.float64).reshape(-1, 3))


def wrap_angle(a: float) -> float:  # geometry.cpp:17-23
    tau = 2.0 * math.pi
    a = math.fmod(a, tau)
    if a <= -math.pi:
        a += tau
    if a > math.pi:
        a -= tau
    return a


# ------------------------------------------------------------------------------ hybrid modes
@dataclass
class HybridParams:
    """HybridParams (hybrid.hpp:12-21)."""
    lambda_switch: float = 5.0
    tau_cool_max: int = 10
    v_min: float = 0.05
    omega_min: float = 0.05
    noise_deadzone_v: float = 0.01
    noise_deadzone_omega: float = 0.01

    def validate(self):  # hybrid.cpp:9-16
        if self.lambda_switch < 0.0:
            raise ValueError("hybrid: lambda_switch must be >= 0")
        if self.tau_cool_max < 0:
            raise ValueError("hybrid: tau_cool_max must be >= 0")
        if self.noise_deadzone_v < 0.0 or self.noise_deadzone_v >= self.v_min:
            raise ValueError("hybrid: noise_deadzone_v must lie in [0, v_min)")
        if self.noise_deadzone_omega < 0.0 or self.noise_deadzone_omega >= self.omega_min:
            raise ValueError("hybrid: noise_deadzone_omega must lie in [0, omega_min)")


@dataclass
class HybridMode:
    name: str
    model: MotionModel
    limits: KinematicLimits


@dataclass
class HybridDecision:
    command: np.ndarray
    mode_index: int
    mode_name: str
    validated: bool
    mode_costs: list
    diagnostics: ControlDecision


def project_to_mode(u_raw: np.ndarray, mode: MotionModel) -> np.ndarray:
    """hybrid.cpp:18-57: zero every inadmissible component; same-dim inputs pass through."""
    u_raw = np.asarray(u_raw, np.float64).reshape(-1)
    if u_raw.size == mode.control_dim():
        return u_raw.copy()
    vx = vy = om = 0.0
    if u_raw.size == 3:
        vx, vy, om = u_raw
    elif u_raw.size == 2:
        vx, om = u_raw
    elif u_raw.size == 1:
        vx = u_raw[0]
    out = np.zeros(mode.control_dim())
    if mode.tag == _abi.MODEL_DIFF:
        out[:] = (vx, om)
    elif mode.tag == _abi.MODEL_ACKERMANN:
        out[0] = vx
    elif mode.tag == _abi.MODEL_OMNI:
        out[:] = (vx, vy, om)
    elif mode.tag == _abi.MODEL_SPIN:
        out[0] = om
    else:
        out[0] = vy
    return out


def deadzone_correct(u: np.ndarray, mode: MotionModel, hp: HybridParams) -> np.ndarray:
    """hybrid.cpp:59-78."""
    out = np.asarray(u, np.float64).copy()
    if mode.tag == _abi.MODEL_SPIN:
        w = out[0]
        if hp.noise_deadzone_omega < abs(w) < hp.omega_min:
            out[0] = math.copysign(hp.omega_min, w)
        return out
    lin = 2 if mode.tag == _abi.MODEL_OMNI else 1
    mag = math.sqrt(sum(out[i] * out[i] for i in range(lin)))
    if hp.noise_deadzone_v < mag < hp.v_min:
        scale = hp.v_min / mag
        for i in range(lin):
            out[i] *= scale
    return out


class HybridController:
    """HybridController (hybrid.hpp:51-69, hybrid.cpp:80-156) with all mode families stepped in
    ONE device call (exm_hybrid_cycle: one cloud preparation, one SDF launch over every
    family's poses, parallel per-family chains). Selection logic stays on the host."""

    def __init__(self, modes, footprint: FootprintSpec, params: MppiParams,
                 hybrid_params: HybridParams, threads: int = 1, n_cap: int = 1024,
                 guide_cap: int = 64, device: int = 0):
        del threads
        if not modes:
            raise ValueError("hybrid: at least one active mode required")
        hybrid_params.validate()
        self.modes, self.hp, self.params = list(modes), hybrid_params, params
        self.M, self.T = len(self.modes), params.horizon
        self.lib = _abi.load_library()
        fp, keep = footprint._c()
        self._keep = keep
        models = (_abi.ExmModel * self.M)(*[m.model._c() for m in self.modes])
        limits = (_abi.ExmLimits * self.M)(*[m.limits._c() for m in self.modes])
        p = params._c()
        h = C.POINTER(_abi.ExmHybrid)()
        check(self.lib.exm_hybrid_create(C.byref(fp), models, limits, self.M, C.byref(p),
                                         int(n_cap), int(guide_cap), int(device), C.byref(h)))
        self.h = h
        self.n_cap = int(n_cap)
        self.nominals = np.zeros(self.M * self.T * 3)
        self.u_prev = np.zeros(self.M * 3)
        self.cycle = 0
        self.m_prev = 0
        self.tau_cool = 0

    def close(self):
        if getattr(self, "h", None):
            self.lib.exm_hybrid_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, option: int, value: int):
        """exm_set_option on every family (e.g. _abi.OPT_SDF_THRESHOLD)."""
        check(self.lib.exm_hybrid_set_option(self.h, int(option), int(value)))

    def family_cycles(self, q0, obstacles: ObstacleSet, guidance: Guidance):
        """One device call: every family's MppiController::control_cycle."""
        pts, mask = obstacles.points, obstacles.mask
        if pts.shape[0] > self.n_cap:
            raise ValueError("point count exceeds obstacle-set capacity")
        dm = [np.empty(self.T) for _ in range(self.M)]
        decs = (_abi.ExmDecision * self.M)()
        for m in range(self.M):
            decs[m].nominal_dmin = dptr(dm[m])
        q = np.ascontiguousarray(np.asarray(q0, np.float64).reshape(3))
        check(self.lib.exm_hybrid_cycle(self.h, dptr(q), dptr(pts), u8ptr(mask), pts.shape[0],
                                        dptr(guidance.path), guidance.path.shape[0],
                                        dptr(guidance.goal), dptr(self.nominals),
                                        dptr(self.u_prev), self.cycle, decs))
        self.cycle += 1
        out = []
        for m, mode in enumerate(self.modes):
            d, D = decs[m], mode.model.control_dim()
            nom = self.nominals[m * self.T * 3: m * self.T * 3 + self.T * D].reshape(self.T, D)
            out.append(ControlDecision(np.array(d.command[:D]), bool(d.validated), nom.copy(),
                                       d.best_cost, d.weight_entropy, d.nominal_cost, dm[m],
                                       d.argmin))
        return out

    def hybrid_cycle(self, q0, obstacles: ObstacleSet, guidance: Guidance) -> HybridDecision:
        decisions = self.family_cycles(q0, obstacles, guidance)
        costs = [math.inf] * self.M
        for m, d in enumerate(decisions):  # hybrid.cpp:103-111
            if d.validated:
                costs[m] = d.nominal_cost + (self.hp.lambda_switch if m != self.m_prev else 0.0)
        if not any(math.isfinite(c) for c in costs):  # safe stop, hybrid.cpp:113-123
            mp = self.modes[self.m_prev]
            return HybridDecision(np.zeros(mp.model.control_dim()), self.m_prev, mp.name, False,
                                  costs, decisions[self.m_prev])
        best, best_cost = self.m_prev, costs[self.m_prev]  # ties toward m_prev, then order
        for m in range(self.M):
            if costs[m] < best_cost:
                best, best_cost = m, costs[m]
        if self.tau_cool > 0 and best != self.m_prev:  # blocked switch
            best = self.m_prev
        self.tau_cool = self.hp.tau_cool_max if best != self.m_prev else max(self.tau_cool - 1, 0)
        sel = decisions[best]
        raw = sel.command
        cmd = deadzone_correct(project_to_mode(raw, self.modes[best].model),
                               self.modes[best].model, self.hp)
        for m in range(self.M):  # re-anchor the unselected families (hybrid.cpp:149-152)
            if m == best:
                continue
            a = project_to_mode(raw, self.modes[m].model)
            self.u_prev[3 * m: 3 * m + 3] = 0.0
            self.u_prev[3 * m: 3 * m + a.size] = a
        self.m_prev = best
        return HybridDecision(cmd, best, self.modes[best].name, sel.validated, costs, sel)
