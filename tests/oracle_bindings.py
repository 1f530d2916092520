"""TEST INFRASTRUCTURE: ctypes bindings of the checkers.

  Oracle     -> oracle/lib/libexm_oracle.so  (C restatement, oracle/exm_oracle.c)
  Reference  -> oracle/_ref/libexm_ref.so    (the unmodified reference sources + ref_shim.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs use this module.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from paper_2605_29663_b200 import _abi
from paper_2605_29663_b200._abi import ExmDecision, ExmFootprint, ExmLimits, ExmModel, ExmParams

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_LIB = os.path.join(ROOT, "oracle", "lib", "libexm_oracle.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libexm_ref.so")

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_d3 = C.c_double * 3


def _p(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _m(a):
    if a is None:
        return None
    a = np.ascontiguousarray(np.asarray(a, np.uint8))
    return a.ctypes.data_as(_u8p)


def _c(a):
    return np.ascontiguousarray(np.asarray(a, np.float64))


_olib = None
_rlib = None


def oracle_lib():
    global _olib
    if _olib is None:
        if not os.path.exists(ORACLE_LIB):
            raise RuntimeError(f"{ORACLE_LIB} missing: run `make -C oracle`")
        L = C.CDLL(ORACLE_LIB)
        sig = {
            "exo_last_error": (C.c_char_p, []),
            "exo_create": (C.c_void_p, [C.POINTER(ExmFootprint), C.POINTER(ExmModel),
                                        C.POINTER(ExmLimits), C.POINTER(ExmParams)]),
            "exo_destroy": (None, [C.c_void_p]),
            "exo_footprint_count": (C.c_int32, [C.c_void_p]),
            "exo_bounding_radius": (C.c_double, [C.c_void_p]),
            "exo_splitmix64": (C.c_uint64, [C.c_uint64]),
            "exo_hash_combine": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "exo_gaussian_at": (C.c_double, [C.c_uint64] * 5),
            "exo_uniform_range": (C.c_double, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double, C.c_double]),
            "exo_uniform_index": (C.c_uint64, [C.c_uint64] * 4),
            "exo_wrap_angle": (C.c_double, [C.c_double]),
            "exo_sd": (C.c_double, [C.c_void_p, C.c_double, C.c_double]),
            "exo_batch_signed_distance": (None, [C.c_void_p, _dp, C.c_int32, _dp]),
            "exo_min_signed_distance_at": (C.c_double, [C.c_void_p, _dp, _dp, _u8p, C.c_int32]),
            "exo_sdf_batch": (None, [C.c_void_p, _dp, C.c_int32, _dp, _u8p, C.c_int32, _dp, _dp]),
            "exo_clamp_control": (None, [C.c_void_p, _dp, _dp, _dp]),
            "exo_step": (None, [C.c_void_p, _dp, _dp, _dp]),
            "exo_obstacle_cost": (C.c_double, [C.c_void_p, C.c_double]),
            "exo_task_cost": (C.c_double, [C.c_void_p, _dp, _dp, C.c_int32, _dp, C.c_int32]),
            "exo_terminal_goal_cost": (C.c_double, [C.c_void_p, _dp, _dp]),
            "exo_control_cost": (C.c_double, [C.c_void_p, _dp]),
            "exo_sample_perturbations": (None, [C.c_void_p, C.c_uint64, C.c_uint64, _dp]),
            "exo_evaluate_rollouts": (C.c_int32, [C.c_void_p, _dp, _dp, _dp, _dp, _u8p, C.c_int32,
                                                  _dp, C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp, _u8p]),
            "exo_weights_from_costs": (None, [_dp, C.c_int32, C.c_double, _dp]),
            "exo_validate_nominal": (C.c_int32, [C.c_void_p, _dp, _dp, _dp, _u8p, C.c_int32, _dp,
                                                 C.c_int32, _dp, _dp, C.POINTER(C.c_int32), _dp, _dp]),
            "exo_control_cycle": (C.c_int32, [C.c_void_p, _dp, _dp, _u8p, C.c_int32, _dp, C.c_int32,
                                              _dp, _dp, _dp, C.c_uint64, _dp, C.POINTER(ExmDecision)]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _olib = L
    return _olib


def reference_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib():
    global _rlib
    if _rlib is None:
        if not os.path.exists(REF_LIB):
            raise RuntimeError(f"{REF_LIB} missing: run `make -C oracle ref` with the reference tree")
        L = C.CDLL(REF_LIB)
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_create": (C.c_void_p, [C.POINTER(ExmFootprint), C.POINTER(ExmModel),
                                        C.POINTER(ExmLimits), C.POINTER(ExmParams), C.c_int32]),
            "ref_destroy": (None, [C.c_void_p]),
            "ref_bounding_radius": (C.c_double, [C.c_void_p]),
            "ref_sd": (C.c_double, [C.c_void_p, C.c_double, C.c_double]),
            "ref_batch_signed_distance": (C.c_int32, [C.c_void_p, _dp, C.c_int32, _dp, C.c_int32]),
            "ref_set_cloud": (C.c_int32, [C.c_void_p, _dp, _u8p, C.c_int32]),
            "ref_min_sd_at_batch": (C.c_int32, [C.c_void_p, _dp, C.c_int32, _dp]),
            "ref_sample_perturbations": (C.c_int32, [C.c_void_p, C.c_uint64, C.c_uint64, _dp]),
            "ref_evaluate_rollouts": (C.c_int32, [C.c_void_p, _dp, _dp, _dp, _dp, _u8p, C.c_int32,
                                                  _dp, C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp, _u8p]),
            "ref_weights_from_costs": (C.c_int32, [_dp, C.c_int32, C.c_double, _dp]),
            "ref_validate_nominal": (C.c_int32, [C.c_void_p, _dp, _dp, _dp, _u8p, C.c_int32, _dp,
                                                 C.c_int32, _dp, _dp, C.POINTER(C.c_int32), _dp, _dp]),
            "ref_controller_cycle": (C.c_int32, [C.c_void_p, _dp, C.c_int32, _dp, _u8p, C.c_int32,
                                                 _dp, C.c_int32, _dp, _dp, _dp,
                                                 C.POINTER(ExmDecision)]),
            "ref_controller_reset": (C.c_int32, [C.c_void_p]),
        }
        for n, (r, a) in sig.items():
            f = getattr(L, n)
            f.restype, f.argtypes = r, a
        _rlib = L
    return _rlib


class _Base:
    prefix = ""

    def __init__(self, footprint, model, limits, params):
        self.footprint, self.model, self.limits, self.params = footprint, model, limits, params
        self.dim = model.control_dim()
        self.K, self.T = params.rollouts, params.horizon

    def _args(self):
        fp, keep = self.footprint._c()
        self._keep = keep
        self._cargs = (fp, self.model._c(), self.limits._c(), self.params._c())
        return [C.byref(x) for x in self._cargs]

    def _pad(self, u):
        out = np.zeros(3)
        u = np.asarray(u, np.float64).reshape(-1)
        out[: u.size] = u
        return out


class Oracle(_Base):
    """The C restatement (oracle/exm_oracle.c)."""

    def __init__(self, footprint, model, limits, params):
        super().__init__(footprint, model, limits, params)
        self.L = oracle_lib()
        self.ctx = self.L.exo_create(*self._args())
        if not self.ctx:
            raise ValueError(self.L.exo_last_error().decode())

    def __del__(self):
        try:
            self.L.exo_destroy(self.ctx)
        except Exception:
            pass

    def radius(self):
        return self.L.exo_bounding_radius(self.ctx)

    def sd(self, x, y):
        return self.L.exo_sd(self.ctx, x, y)

    def batch_signed_distance(self, q):
        q = _c(q).reshape(-1, 2)
        out = np.empty(q.shape[0])
        self.L.exo_batch_signed_distance(self.ctx, _p(q), q.shape[0], _p(out))
        return out

    def min_signed_distance_at(self, pose, pts, mask=None):
        pts = _c(pts).reshape(-1, 2)
        return self.L.exo_min_signed_distance_at(self.ctx, _p(_c(pose)), _p(pts), _m(mask), pts.shape[0])

    def sdf_batch(self, poses, pts, mask=None, per_pair=False):
        poses = _c(poses).reshape(-1, 3)
        pts = _c(pts).reshape(-1, 2)
        mins = np.empty(poses.shape[0])
        pairs = np.empty((poses.shape[0], pts.shape[0])) if per_pair else None
        self.L.exo_sdf_batch(self.ctx, _p(poses), poses.shape[0], _p(pts), _m(mask), pts.shape[0],
                             _p(pairs), _p(mins))
        return (mins, pairs) if per_pair else mins

    def sample_perturbations(self, seed, cycle):
        eps = np.empty((self.K, self.T, self.dim))
        self.L.exo_sample_perturbations(self.ctx, seed, cycle, _p(eps))
        return eps

    def clamp_control(self, u, prev):
        out = np.zeros(3)
        self.L.exo_clamp_control(self.ctx, _p(self._pad(u)), _p(self._pad(prev)), _p(out))
        return out[: self.dim]

    def step(self, q, u):
        out = np.zeros(3)
        self.L.exo_step(self.ctx, _p(_c(q)), _p(self._pad(u)), _p(out))
        return out

    def evaluate_rollouts(self, q0, nominal, eps, pts, mask, guidance, u_prev):
        pts = _c(pts).reshape(-1, 2)
        K, T, D = self.K, self.T, self.dim
        controls = np.empty((K, T, D))
        states = np.empty((K, T + 1, 3))
        dmin = np.empty((K, T))
        costs = np.empty(K)
        unsafe = np.empty(K, np.uint8)
        rc = self.L.exo_evaluate_rollouts(
            self.ctx, _p(_c(q0)), _p(_c(nominal).reshape(-1)), _p(_c(eps).reshape(-1)), _p(pts),
            _m(mask), pts.shape[0], _p(guidance.path), guidance.path.shape[0], _p(guidance.goal),
            _p(self._pad(u_prev)), _p(controls), _p(states), _p(dmin), _p(costs),
            unsafe.ctypes.data_as(_u8p))
        if rc:
            raise ValueError(self.L.exo_last_error().decode())
        return dict(controls=controls, states=states, d_min=dmin, costs=costs, unsafe=unsafe)

    def validate_nominal(self, nominal, q0, pts, mask, guidance, u_prev):
        pts = _c(pts).reshape(-1, 2)
        valid = C.c_int32()
        dmin = np.empty(self.T)
        cost = C.c_double()
        self.L.exo_validate_nominal(self.ctx, _p(_c(nominal).reshape(-1)), _p(_c(q0)), _p(pts),
                                    _m(mask), pts.shape[0], _p(guidance.path),
                                    guidance.path.shape[0], _p(guidance.goal),
                                    _p(self._pad(u_prev)), C.byref(valid), _p(dmin), C.byref(cost))
        return bool(valid.value), dmin, cost.value

    def control_cycle(self, q0, pts, mask, guidance, nominal, u_prev, cycle, eps=None):
        """nominal (T*dim) and u_prev (3) are updated in place, as exm_control_cycle does."""
        pts = _c(pts).reshape(-1, 2)
        dmin = np.empty(self.T)
        dec = ExmDecision()
        dec.nominal_dmin = _p(dmin)
        e = None if eps is None else _c(eps).reshape(-1)
        rc = self.L.exo_control_cycle(self.ctx, _p(_c(q0)), _p(pts), _m(mask), pts.shape[0],
                                      _p(guidance.path), guidance.path.shape[0], _p(guidance.goal),
                                      _p(nominal), _p(u_prev), cycle, _p(e), C.byref(dec))
        if rc:
            raise ValueError(self.L.exo_last_error().decode())
        return dict(command=np.array(dec.command[:]), validated=bool(dec.validated),
                    argmin=dec.argmin, best_cost=dec.best_cost, weight_entropy=dec.weight_entropy,
                    nominal_cost=dec.nominal_cost, nominal_d_min=dmin)


class Reference(_Base):
    """The unmodified reference, compiled from its own sources (oracle/_ref)."""

    def __init__(self, footprint, model, limits, params, threads=1):
        super().__init__(footprint, model, limits, params)
        self.L = ref_lib()
        args = self._args()
        self.ctx = self.L.ref_create(*args, int(threads))
        if not self.ctx:
            raise ValueError(self.L.ref_last_error().decode())

    def __del__(self):
        try:
            self.L.ref_destroy(self.ctx)
        except Exception:
            pass

    def radius(self):
        return self.L.ref_bounding_radius(self.ctx)

    def sd(self, x, y):
        return self.L.ref_sd(self.ctx, x, y)

    def batch_signed_distance(self, q, threads=1):
        q = _c(q).reshape(-1, 2)
        out = np.empty(q.shape[0])
        self.L.ref_batch_signed_distance(self.ctx, _p(q), q.shape[0], _p(out), threads)
        return out

    def set_cloud(self, pts, mask=None):
        pts = _c(pts).reshape(-1, 2)
        self.L.ref_set_cloud(self.ctx, _p(pts), _m(mask), pts.shape[0])

    def min_sd_at(self, poses):
        poses = _c(poses).reshape(-1, 3)
        out = np.empty(poses.shape[0])
        self.L.ref_min_sd_at_batch(self.ctx, _p(poses), poses.shape[0], _p(out))
        return out

    def sample_perturbations(self, seed, cycle):
        eps = np.empty((self.K, self.T, self.dim))
        self.L.ref_sample_perturbations(self.ctx, seed, cycle, _p(eps))
        return eps

    def evaluate_rollouts(self, q0, nominal, eps, pts, mask, guidance, u_prev):
        pts = _c(pts).reshape(-1, 2)
        K, T, D = self.K, self.T, self.dim
        controls = np.empty((K, T, D))
        states = np.empty((K, T + 1, 3))
        dmin = np.empty((K, T))
        costs = np.empty(K)
        unsafe = np.empty(K, np.uint8)
        rc = self.L.ref_evaluate_rollouts(
            self.ctx, _p(_c(q0)), _p(_c(nominal).reshape(-1)), _p(_c(eps).reshape(-1)), _p(pts),
            _m(mask), pts.shape[0], _p(guidance.path), guidance.path.shape[0], _p(guidance.goal),
            _p(self._pad(u_prev)), _p(controls), _p(states), _p(dmin), _p(costs),
            unsafe.ctypes.data_as(_u8p))
        if rc:
            raise ValueError(self.L.ref_last_error().decode())
        return dict(controls=controls, states=states, d_min=dmin, costs=costs, unsafe=unsafe)

    def weights_from_costs(self, costs, lam):
        costs = _c(costs)
        w = np.empty_like(costs)
        self.L.ref_weights_from_costs(_p(costs), costs.size, lam, _p(w))
        return w

    def validate_nominal(self, nominal, q0, pts, mask, guidance, u_prev):
        pts = _c(pts).reshape(-1, 2)
        valid = C.c_int32()
        dmin = np.empty(self.T)
        cost = C.c_double()
        self.L.ref_validate_nominal(self.ctx, _p(_c(nominal).reshape(-1)), _p(_c(q0)), _p(pts),
                                    _m(mask), pts.shape[0], _p(guidance.path),
                                    guidance.path.shape[0], _p(guidance.goal),
                                    _p(self._pad(u_prev)), C.byref(valid), _p(dmin), C.byref(cost))
        return bool(valid.value), dmin, cost.value

    def controller_cycle(self, q0, pts, mask, guidance, use_stored_cloud=False):
        """MppiController::control_cycle on the reference's own controller object."""
        pts = _c(pts).reshape(-1, 2) if pts is not None else np.zeros((0, 2))
        nom = np.empty(self.T * self.dim)
        up = np.zeros(3)
        dmin = np.empty(self.T)
        dec = ExmDecision()
        dec.nominal_dmin = _p(dmin)
        rc = self.L.ref_controller_cycle(self.ctx, _p(_c(q0)), 1 if use_stored_cloud else 0,
                                         _p(pts), _m(mask), pts.shape[0], _p(guidance.path),
                                         guidance.path.shape[0], _p(guidance.goal), _p(nom),
                                         _p(up), C.byref(dec))
        if rc:
            raise ValueError(self.L.ref_last_error().decode())
        return dict(command=np.array(dec.command[:]), validated=bool(dec.validated),
                    best_cost=dec.best_cost, weight_entropy=dec.weight_entropy,
                    nominal_cost=dec.nominal_cost, nominal_d_min=dmin, nominal=nom, u_prev=up)

    def reset(self):
        self.L.ref_controller_reset(self.ctx)


def oracle_weights(costs, lam):
    costs = _c(costs)
    w = np.empty_like(costs)
    oracle_lib().exo_weights_from_costs(_p(costs), costs.size, lam, _p(w))
    return w


class ReferenceHybrid:
    """The reference's HybridController (hybrid.cpp) over its own MppiControllers (oracle/_ref)."""

    def __init__(self, footprint, modes, params, hp, threads=1):
        L = ref_lib()
        if not hasattr(L, "_hy_ready"):
            L.ref_hybrid_create.restype = C.c_void_p
            L.ref_hybrid_create.argtypes = [C.POINTER(ExmFootprint), C.POINTER(ExmModel),
                                            C.POINTER(ExmLimits), C.c_int32, C.POINTER(ExmParams),
                                            _dp, C.c_int32]
            L.ref_hybrid_destroy.argtypes = [C.c_void_p]
            L.ref_hybrid_cycle.restype = C.c_int32
            L.ref_hybrid_cycle.argtypes = [C.c_void_p, _dp, _dp, _u8p, C.c_int32, _dp, C.c_int32,
                                           _dp, _dp, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                           _dp, _dp]
            L._hy_ready = True
        self.L, self.M = L, len(modes)
        fp, self._keep = footprint._c()
        models = (ExmModel * self.M)(*[m.model._c() for m in modes])
        limits = (ExmLimits * self.M)(*[m.limits._c() for m in modes])
        p = params._c()
        h = np.array([hp.lambda_switch, hp.tau_cool_max, hp.v_min, hp.omega_min,
                      hp.noise_deadzone_v, hp.noise_deadzone_omega], np.float64)
        self.ctx = L.ref_hybrid_create(C.byref(fp), models, limits, self.M, C.byref(p), _p(h),
                                       int(threads))
        if not self.ctx:
            raise ValueError(L.ref_last_error().decode())

    def __del__(self):
        try:
            self.L.ref_hybrid_destroy(self.ctx)
        except Exception:
            pass

    def hybrid_cycle(self, q0, pts, mask, guidance):
        pts = _c(pts).reshape(-1, 2)
        cmd = np.zeros(3)
        mi, val = C.c_int32(), C.c_int32()
        costs = np.zeros(self.M)
        diag = np.zeros(3)
        rc = self.L.ref_hybrid_cycle(self.ctx, _p(_c(q0)), _p(pts), _m(mask), pts.shape[0],
                                     _p(guidance.path), guidance.path.shape[0], _p(guidance.goal),
                                     _p(cmd), C.byref(mi), C.byref(val), _p(costs), _p(diag))
        if rc:
            raise ValueError(self.L.ref_last_error().decode())
        return dict(command=cmd, mode_index=mi.value, validated=bool(val.value), mode_costs=costs,
                    best_cost=diag[0], weight_entropy=diag[1], nominal_cost=diag[2])


def reference_sense(obstacles, robot, sensor_range, budget, seed, sample_key):
    """The reference's sense() (world.cpp:182-243) through oracle/_ref (ref_sense)."""
    from paper_2605_29663_b200.api import world_obstacles_c
    L = ref_lib()
    arr, keep = world_obstacles_c(obstacles)
    pts = np.empty((budget, 2))
    mask = np.empty(budget, np.uint8)
    n = C.c_int32()
    rc = L.ref_sense(arr, len(obstacles), _p(_c(robot)), C.c_double(sensor_range), budget,
                     C.c_uint64(seed), C.c_uint64(sample_key), _p(pts),
                     mask.ctypes.data_as(_u8p), C.byref(n))
    del keep
    if rc:
        raise ValueError(L.ref_last_error().decode())
    return pts, mask, n.value


class ReferenceWorld:
    """The reference's Scenario + WorldState with trail motion: step_world and sense
    (world.cpp:127-243) through oracle/_ref (ref_world_*)."""

    def __init__(self, obstacles, trails, sensor_range, budget, seed):
        from paper_2605_29663_b200.api import world_obstacles_c
        L = ref_lib()
        if not hasattr(L, "_world_ready"):
            L.ref_world_create.restype = C.c_void_p
            L.ref_world_create.argtypes = [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(_dp), _dp,
                                           C.POINTER(C.c_int32), C.c_int, C.c_double, C.c_int,
                                           C.c_uint64]
            L.ref_world_destroy.argtypes = [C.c_void_p]
            L.ref_world_step.restype = C.c_int
            L.ref_world_step.argtypes = [C.c_void_p, C.c_double]
            L.ref_world_state.argtypes = [C.c_void_p, _dp, C.POINTER(C.c_int32), _dp]
            L.ref_world_sense.restype = C.c_int
            L.ref_world_sense.argtypes = [C.c_void_p, _dp, C.c_uint64, _dp, _u8p,
                                          C.POINTER(C.c_int32)]
            L._world_ready = True
        self.L, self.n, self.budget = L, len(obstacles), int(budget)
        arr, self._keep = world_obstacles_c(obstacles)
        n = self.n
        nwp = (C.c_int32 * max(n, 1))()
        wps = (_dp * max(n, 1))()
        spd = np.zeros(max(n, 1))
        pp = (C.c_int32 * max(n, 1))()
        self._wp = []
        for i, t in enumerate(trails or []):
            if t is None:
                continue
            w = np.ascontiguousarray(t.waypoints)
            self._wp.append(w)
            nwp[i], wps[i], spd[i], pp[i] = w.shape[0], _p(w), t.speed, 1 if t.ping_pong else 0
        self._spd = spd
        self.ctx = L.ref_world_create(C.cast(arr, C.c_void_p), nwp, wps, _p(spd), pp, n,
                                      float(sensor_range), self.budget, int(seed))
        if not self.ctx:
            raise ValueError(L.ref_last_error().decode())

    def __del__(self):
        try:
            self.L.ref_world_destroy(self.ctx)
        except Exception:
            pass

    def step(self, dt):
        if self.L.ref_world_step(self.ctx, float(dt)):
            raise ValueError(self.L.ref_last_error().decode())

    def state(self):
        arc = np.empty(max(self.n, 1))
        d = np.empty(max(self.n, 1), np.int32)
        off = np.empty((max(self.n, 1), 2))
        self.L.ref_world_state(self.ctx, _p(arc), d.ctypes.data_as(C.POINTER(C.c_int32)), _p(off))
        return arc[: self.n], d[: self.n], off[: self.n]

    def sense(self, robot, key):
        pts = np.empty((self.budget, 2))
        mask = np.empty(self.budget, np.uint8)
        n = C.c_int32()
        if self.L.ref_world_sense(self.ctx, _p(_c(robot)), int(key), _p(pts),
                                  mask.ctypes.data_as(_u8p), C.byref(n)):
            raise ValueError(self.L.ref_last_error().decode())
        return pts, mask, n.value
