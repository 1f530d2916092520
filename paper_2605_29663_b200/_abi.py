"""ctypes binding of the C ABI in include/exm_b200.h (libexm_b200.so).

This is the reference-side binding a Python caller uses; the C++ drop-in
 binds the same symbols from C++. The library is REQUIRED: there is no
CPU fallback, and loading fails loudly when it has not been built.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EXM_LIB_PATH", os.path.join(HERE, "lib", "libexm_b200.so"))

EXM_OK = 0
EXM_ERR_INVALID_ARGUMENT = 1
EXM_ERR_CUDA = 2
EXM_ERR_NCCL = 3
EXM_ERR_UNSUPPORTED = 4
EXM_ERR_INTERNAL = 5

FOOTPRINT_RECT_COVER = 0
FOOTPRINT_POLYGON = 1

MODEL_DIFF, MODEL_ACKERMANN, MODEL_OMNI, MODEL_SPIN, MODEL_PARALLEL = range(5)

_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)
_fp = C.POINTER(C.c_float)


class ExmWorldObstacle(C.Structure):
    _fields_ = [("kind", C.c_int32), ("count", C.c_int32), ("x", C.POINTER(C.c_double)),
                ("y", C.POINTER(C.c_double)), ("radius", C.c_double), ("offset", C.c_double * 2)]


OBSTACLE_POLYGON, OBSTACLE_DISC = 0, 1


class ExmWorldTrail(C.Structure):
    _fields_ = [("n_waypoints", C.c_int32), ("ping_pong", C.c_int32),
                ("waypoints", C.POINTER(C.c_double)), ("speed", C.c_double)]


class ExmWorld(C.Structure):
    pass


_Wp = C.POINTER(ExmWorld)


class ExmFootprint(C.Structure):
    _fields_ = [("kind", C.c_int32), ("count", C.c_int32), ("x", _dp), ("y", _dp),
                ("hx", _dp), ("hy", _dp)]


class ExmModel(C.Structure):
    _fields_ = [("tag", C.c_int32), ("reserved", C.c_int32), ("wheelbase", C.c_double)]


class ExmLimits(C.Structure):
    _fields_ = [("vel_min", C.c_double * 3), ("vel_max", C.c_double * 3),
                ("acc_min", C.c_double * 3), ("acc_max", C.c_double * 3),
                ("steer_max", C.c_double)]


class ExmParams(C.Structure):
    _fields_ = [("rollouts", C.c_int32), ("horizon", C.c_int32), ("dt", C.c_double),
                ("lambda_", C.c_double), ("sigma", C.c_double * 3), ("d_safe", C.c_double),
                ("w_coll", C.c_double), ("w_rep", C.c_double), ("w_inf", C.c_double),
                ("w_goal_pos", C.c_double), ("w_goal_head", C.c_double),
                ("w_xtrack", C.c_double), ("w_progress", C.c_double), ("w_ctrl", C.c_double),
                ("seed", C.c_uint64)]


class ExmDecision(C.Structure):
    _fields_ = [("command", C.c_double * 3), ("validated", C.c_int32), ("argmin", C.c_int32),
                ("best_cost", C.c_double), ("weight_entropy", C.c_double),
                ("nominal_cost", C.c_double), ("nominal_dmin", _dp)]


class ExmSdfPath(C.Structure):
    _fields_ = [("kernel", C.c_int32), ("chunk", C.c_int32), ("persistent", C.c_int32),
                ("ctas", C.c_int32), ("threads", C.c_int32), ("hmajor", C.c_int32)]


# exm_set_option options and EXM_SDF_* modes (include/exm_b200.h)
OPT_SDF_MODE, OPT_AUTO_CAPS, OPT_PREGEN, OPT_HOST_TIMING, OPT_HOST_THREADS, OPT_SDF_MAP = 1, 2, 3, 4, 5, 6
OPT_SDF_THRESHOLD = 7
OPT_SDF_FP64 = 8
SDF_MODES = {"auto": 0, "brute": 1, "nochunk": 2, "thread": 3, "warp": 4, "cta": 5,
             "persist": 6, "nocap": 7}
SDF_NCOUNT = 10
SDF_COUNTERS = ("ring_steps", "cell_tests", "chunk_tests", "point_tests", "point_iters_warp",
                "transforms", "tile_tests", "tile_values", "bound_tests", "edge_loops")


class ExmHandle(C.Structure):
    pass


_Hp = C.POINTER(ExmHandle)


class ExmHybrid(C.Structure):
    pass


_HYp = C.POINTER(ExmHybrid)

# name -> (restype, argtypes); every entry point declared in include/exm_b200.h
SIGNATURES = {
    "exm_abi_version": (C.c_int32, []),
    "exm_last_error": (C.c_char_p, []),
    "exm_create": (C.c_int32, [C.POINTER(ExmFootprint), C.POINTER(ExmModel),
                               C.POINTER(ExmLimits), C.POINTER(ExmParams), C.c_int32, C.c_int32,
                               C.c_int32, C.POINTER(_Hp)]),
    "exm_destroy": (None, [_Hp]),
    "exm_control_cycle": (C.c_int32, [_Hp, _dp, _dp, _u8p, C.c_int32, _dp, C.c_int32, _dp, _dp,
                                      _dp, C.c_uint64, _dp, C.POINTER(ExmDecision)]),
    "exm_evaluate_rollouts": (C.c_int32, [_Hp, _dp, _dp, _dp, _dp, _u8p, C.c_int32, _dp,
                                          C.c_int32, _dp, _dp, _dp, _dp, _dp, _dp, _u8p]),
    "exm_sample_perturbations": (C.c_int32, [_Hp, C.c_uint64, C.c_uint64, _dp]),
    "exm_validate_nominal": (C.c_int32, [_Hp, _dp, _dp, _dp, _u8p, C.c_int32, _dp, C.c_int32,
                                         _dp, _dp, C.POINTER(C.c_int32), _dp, _dp]),
    "exm_sdf_batch": (C.c_int32, [_Hp, _dp, C.c_int32, _dp, _u8p, C.c_int32, _fp, _dp]),
    "exm_sdf_stage": (C.c_int32, [_Hp, _dp, C.c_int32, _dp, _u8p, C.c_int32]),
    "exm_sdf_run_resident": (C.c_int32, [_Hp, C.c_int32, C.c_int32]),
    "exm_sdf_read": (C.c_int32, [_Hp, _fp, _dp]),
    "exm_batch_signed_distance": (C.c_int32, [_Hp, _dp, C.c_int32, _dp]),
    "exm_hybrid_create": (C.c_int32, [C.POINTER(ExmFootprint), C.POINTER(ExmModel),
                                      C.POINTER(ExmLimits), C.c_int32, C.POINTER(ExmParams),
                                      C.c_int32, C.c_int32, C.c_int32, C.POINTER(_HYp)]),
    "exm_hybrid_destroy": (None, [_HYp]),
    "exm_hybrid_set_option": (C.c_int32, [_HYp, C.c_int32, C.c_int32]),
    "exm_hybrid_cycle": (C.c_int32, [_HYp, _dp, _dp, _u8p, C.c_int32, _dp, C.c_int32, _dp, _dp,
                                     _dp, C.c_uint64, C.POINTER(ExmDecision)]),
    "exm_nccl_unique_id": (C.c_int32, [C.POINTER(C.c_uint8)]),
    "exm_attach_comm": (C.c_int32, [_Hp, C.c_int32, C.c_int32, C.POINTER(C.c_uint8)]),
    "exm_stage_inputs": (C.c_int32, [_Hp, _dp, _dp, _u8p, C.c_int32, _dp, C.c_int32, _dp, _dp,
                                     _dp, C.c_uint64]),
    "exm_run_resident": (C.c_int32, [_Hp, C.c_int32]),
    "exm_read_resident": (C.c_int32, [_Hp, _dp, _dp, C.POINTER(ExmDecision)]),
    "exm_stream": (C.c_void_p, [_Hp]),
    "exm_sdf_cull_stats": (C.c_int32, [_Hp, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "exm_set_sdf_caps": (C.c_int32, [_Hp, C.POINTER(C.c_float)]),
    "exm_sense": (C.c_int32, [_Hp, C.POINTER(ExmWorldObstacle), C.c_int32, _dp, C.c_double,
                              C.c_int32, C.c_uint64, C.c_uint64, _dp, _u8p,
                              C.POINTER(C.c_int32)]),
    "exm_host_alloc": (C.c_void_p, [C.c_size_t]),
    "exm_host_free": (None, [C.c_void_p]),
    "exm_footprint_cull_boxes": (C.c_int32, [C.POINTER(ExmFootprint), C.POINTER(C.c_float),
                                             C.POINTER(C.c_float), C.POINTER(C.c_int32)]),
    "exm_step_stats": (C.c_int32, [_Hp, C.POINTER(C.c_int32), C.POINTER(C.c_float),
                                   C.POINTER(C.c_int64)]),
    "exm_set_shard": (C.c_int32, [_Hp, C.c_int32, C.c_int32]),
    "exm_sharded_cycle": (C.c_int32, [C.POINTER(_Hp), C.c_int32, _dp, _dp, _u8p, C.c_int32, _dp,
                                      C.c_int32, _dp, _dp, _dp, C.c_uint64, _dp,
                                      C.POINTER(ExmDecision)]),
    "exm_set_option": (C.c_int32, [_Hp, C.c_int32, C.c_int32]),
    "exm_host_timing": (C.c_int32, [_Hp, _dp, C.POINTER(C.c_int64)]),
    "exm_last_sdf_path": (C.c_int32, [_Hp, C.POINTER(ExmSdfPath), C.POINTER(ExmSdfPath)]),
    "exm_sdf_work_stats": (C.c_int32, [_Hp, C.POINTER(C.c_int64)]),
    "exm_world_create": (C.c_int32, [_Hp, C.POINTER(ExmWorldObstacle), C.POINTER(ExmWorldTrail),
                                     C.c_int32, C.c_double, C.c_int32, C.c_uint64,
                                     C.POINTER(_Wp)]),
    "exm_world_destroy": (None, [_Wp]),
    "exm_world_step": (C.c_int32, [_Wp, C.c_double]),
    "exm_world_sense": (C.c_int32, [_Wp, _dp, C.c_uint64, _dp, _u8p, C.POINTER(C.c_int32)]),
    "exm_world_state": (C.c_int32, [_Wp, _dp, C.POINTER(C.c_int32), _dp]),
}

_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load libexm_b200.so (raises if it has not been built: no fallback path exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} is missing: the CUDA library is required (build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'`)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class ExmError(RuntimeError):
    pass


def check(status: int) -> None:
    if status == EXM_OK:
        return
    msg = (load_library().exm_last_error() or b"").decode()
    if status == EXM_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)  # the reference throws std::invalid_argument
    raise ExmError(f"exm status {status}: {msg}")


def dptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def fptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(_fp)


def u8ptr(a: np.ndarray | None):
    if a is None:
        return None
    assert a.dtype == np.uint8 and a.flags.c_contiguous
    return a.ctypes.data_as(_u8p)


def fast_control_cycle(lib):
    """exm_control_cycle bound a second time with void* pointer arguments: callers pass cached
    integer addresses (Engine.control_cycle_raw), which skips ctypes' per-call pointer-object
    construction (several microseconds per argument on the host)."""
    fn = C.CDLL(lib._name)["exm_control_cycle"]
    v = C.c_void_p
    fn.restype = C.c_int32
    fn.argtypes = [v, v, v, v, C.c_int32, v, C.c_int32, v, v, v, C.c_uint64, v, v]
    return fn

