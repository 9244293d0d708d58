"""ctypes binding of the in-tree C ABI (``include/kinoptik_b200.h``).

The shared library is built by ``paper_2505_03728_b200._build`` (or
``__graft_entry__.build()``) into this package directory.  There is no CPU
fallback: if the library is missing, importing anything that computes raises.
"""

from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# KOP_LIB selects another in-tree build of the same library (A/B timing of kernel variants)
LIB_PATH = os.environ.get("KOP_LIB") or os.path.join(_HERE, "libkinoptik_b200.so")

KOP_OK, KOP_EINVAL, KOP_EUNSUPPORTED, KOP_ECUDA = 0, -1, -2, -3
KOP_FP32, KOP_FP64 = 0, 1
KOP_BASE_NONE, KOP_BASE_SE2, KOP_BASE_SE3 = 0, 1, 2
KOP_TERM_LIMIT, KOP_TERM_REST, KOP_TERM_SMOOTHNESS, KOP_TERM_VELOCITY, KOP_TERM_STENCIL = 0, 1, 2, 3, 4
KOP_TERM_WORLD, KOP_TERM_SELF, KOP_TERM_SWEPT = 5, 6, 7

_p = C.c_void_p
_i32, _i64, _u64, _f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double


class KopModelDesc(C.Structure):
    _fields_ = [
        ("num_links", _i32), ("num_joints", _i32), ("num_actuated", _i32),
        ("parent_link", _p), ("child_link", _p), ("kind", _p), ("qcol", _p),
        ("mult", _p), ("offset", _p), ("origin_wxyz", _p), ("origin_xyz", _p), ("axis", _p),
        ("lower", _p), ("upper", _p), ("rest", _p),
        ("num_spheres", _i32), ("sphere_link", _p), ("sphere_center", _p), ("sphere_radius", _p),
        ("num_self_pairs", _i32), ("self_pair_links", _p),
    ]


class KopIkParams(C.Structure):
    _fields_ = [
        ("w_position", _f64), ("w_orientation", _f64), ("w_limit", _f64), ("w_rest", _f64),
        ("seeds", _i32), ("total_steps", _i32), ("prune_after", _i32), ("keep", _i32),
        ("success_pos_tol", _f64), ("success_rot_tol", _f64), ("precision", _i32),
        ("optimize_base", _i32), ("w_base", _f64),
    ]


class KopObstacle(C.Structure):
    _fields_ = [("kind", _i32), ("a", _f64 * 3), ("b", _f64 * 3), ("radius", _f64)]


class KopCollisionCosts(C.Structure):
    _fields_ = [(f, _f64) for f in ("w_position", "w_orientation", "w_limit", "w_rest", "w_world", "eta_world",
                                    "w_self", "eta_self", "sharpness")] + \
               [("hard_min", _i32), ("num_obstacles", _i32), ("obstacles", C.POINTER(KopObstacle))]


class KopLmOptions(C.Structure):
    _fields_ = [("max_iterations", _i32), ("initial_damping", _f64), ("damping_increase", _f64),
                ("damping_decrease", _f64), ("gradient_tolerance", _f64), ("step_tolerance", _f64),
                ("max_rejections", _i32), ("precision", _i32)]


class KopTrajCosts(C.Structure):
    _fields_ = [("timesteps", _i32), ("dt", _f64)] + \
               [(f, _f64) for f in ("w_anchor", "w_smoothness", "w_velocity", "w_acceleration", "w_jerk", "w_limit",
                                    "w_rest", "w_self", "eta_self", "w_world", "eta_world", "sharpness")] + \
               [("hard_min", _i32), ("velocity_limits", C.POINTER(_f64)), ("rest", C.POINTER(_f64))]


class KopPoseCosts(C.Structure):
    _fields_ = [("num_poses", _i32), ("links", _p), ("w_position", _p), ("w_orientation", _p),
                ("w_limit", _f64), ("w_rest", _f64), ("rest", _p)]


# name -> (restype, argtypes); must match include/kinoptik_b200.h exactly
SIGNATURES = {
    "kop_model_create": (C.c_int, [C.POINTER(KopModelDesc), C.POINTER(_p)]),
    "kop_model_destroy": (None, [_p]),
    "kop_model_chain_length": (C.c_int, [_p, _i32]),
    "kop_model_chain_export": (C.c_int, [_p, _i32, _p, _p, _p, _p, _p, _p, _p]),
    "kop_last_error": (C.c_char_p, []),
    "kop_build_info": (C.c_char_p, []),
    "kop_fk": (C.c_int, [_p, _i32, _p, _i64, _p, _p, _p, _p, _p]),
    "kop_lane_residuals_jacobian": (C.c_int, [_p, _i32, _i32, _p, _p, _p, _p, _p, _i64, _p, _p, _p]),
    "kop_lane_start": (C.c_int, [_p, _i32, _i32, _p, _p, _p, _p, _p, _i64, _p, _p, _p]),
    "kop_lane_run": (C.c_int, [_p, _i32, _i32, _p, _p, _p, _i64, _i32, _p, _p, _p, _p, _p, _p]),
    "kop_ik_beam_workspace_bytes": (_i64, [_p, _i32, C.POINTER(KopIkParams), _i64]),
    "kop_ik_beam": (C.c_int, [_p, _i32, C.POINTER(KopIkParams), _p, _i64, _p, _p, _i64,
                              _p, _p, _p, _p, _p, _p, _p, _p]),
    "kop_ik_beam_stage": (C.c_int, [_p, _i32, C.POINTER(KopIkParams), _i32, _p, _i64, _p, _p, _i64,
                                    _p, _p, _p, _p, _p, _p, _p, _p]),
    "kop_collision_rows": (C.c_int, [_p, _i32, C.POINTER(KopCollisionCosts)]),
    "kop_collision_residuals_jacobian": (C.c_int, [_p, _i32, _i32, C.POINTER(KopCollisionCosts), _p, _p, _p, _i64,
                                                   _p, _p, _p]),
    "kop_ik_beam_collision_workspace_bytes": (_i64, [_p, _i32, C.POINTER(KopIkParams),
                                                     C.POINTER(KopCollisionCosts), _i64]),
    "kop_ik_beam_collision": (C.c_int, [_p, _i32, C.POINTER(KopIkParams), C.POINTER(KopCollisionCosts), _p, _i64,
                                        _p, _p, _i64, _p, _p, _p, _p, _p, _p, _p]),
    "kop_lm_solve": (C.c_int, [_p, _i32, C.POINTER(KopCollisionCosts), C.POINTER(KopLmOptions), _p, _p, _i64,
                               _p, _p, _p, _p, _p, _p, _p]),
    "kop_multi_pose_solve": (C.c_int, [_p, C.POINTER(KopPoseCosts), C.POINTER(KopLmOptions), _p, _p, _i64,
                                       _p, _p, _p, _p, _p, _p, _p]),
    "kop_multi_pose_solve_base": (C.c_int, [_p, C.POINTER(KopPoseCosts), C.POINTER(KopLmOptions), _i32, _p, _p, _p,
                                            _i64, _p, _p, _p, _p, _p, _p, _p, _p]),
    "kop_ik_beam_host": (C.c_int, [_p, _i32, C.POINTER(KopIkParams), _p, _i64, _p, _p, _p, _p, _p, _p, _p, _p,
                                   _i64, _i32, _p]),
    "kop_traj_solve": (C.c_int, [_p, _i32, C.POINTER(KopTrajCosts), C.POINTER(KopLmOptions), _p, _p, _p, _i32,
                                 _i64, _p, _p, _p, _p, _p, _p, _p]),
    "kop_traj_normal_equations": (C.c_int, [_p, _i32, C.POINTER(KopTrajCosts), _i32, _p, _p, _p, _i32, _i64, _p,
                                            _p, _p, _p]),
    "kop_traj_report": (C.c_int, [_p, _i32, _i32, _p, _p, _i32, _p, _i64, _p, _p, _p, _p, _p, _p, _p]),
    "kop_multi_pose_beam_workspace_bytes": (C.c_int64, [_p, C.POINTER(KopPoseCosts), C.POINTER(KopIkParams), _i64]),
    "kop_multi_pose_beam": (C.c_int, [_p, C.POINTER(KopPoseCosts), C.POINTER(KopIkParams), _p, _i64, _p, _p, _i64,
                                      _p, _p, _p, _p, _p, _p, _p]),
    "kop_sample_uniform": (C.c_int, [_u64, _u64, _i64, _i32, _p, _p, _p, _p, _p]),
    "kop_jacobian": (C.c_int, [_p, _i32, _p, _i64, _i32, _p, _i32, _p, _p]),
    "kop_link_poses": (C.c_int, [_p, _i32, _p, _i64, _p, _p]),
    "kop_fma_peak_kernel": (C.c_int, [_i32, _i32, _i32, _p, C.POINTER(_f64), _p]),
    "kop_dfma_peak_kernel": (C.c_int, [_i32, _i32, _i32, _p, C.POINTER(_f64), _p]),
    "kop_check_probe": (C.c_int, [_p, _i32, _p]),
    "kop_term_pose": (C.c_int, [_p, _i32, _p, _i32, _p, _p, _i64, _p, _p, _p, _p]),
    "kop_term_joint": (C.c_int, [_p, _i32, _p, _p, _f64, _p, _p, _i64, _p, _p, _p]),
    "kop_term_collision": (C.c_int, [_p, _i32, C.POINTER(KopObstacle), _i32, _f64, _f64, _i32, _p, _p, _i64, _p, _p,
                                     _p, _p]),
    "kop_term_rows": (C.c_int, [_p, _i32, _i32]),
    "kop_term_manipulability": (C.c_int, [_p, _i32, _f64, _p, _i64, _p, _p, _p, _p, _p]),
}

_lib = None


def lib():
    """Load (once) and return the CDLL; raise loudly if it is not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        dll = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(dll, name)
            fn.restype = res
            fn.argtypes = args
        _lib = dll
    return _lib


def check(status: int, what: str) -> None:
    """Map a KOP_* status to the reference's exception types."""
    if status == KOP_OK:
        return
    msg = lib().kop_last_error().decode(errors="replace")
    if status == KOP_EINVAL:
        raise ValueError(f"{what}: {msg}")
    if status == KOP_EUNSUPPORTED:
        from .errors import UnsupportedFeatureError
        raise UnsupportedFeatureError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")
