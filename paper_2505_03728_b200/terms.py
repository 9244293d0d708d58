"""Device evaluation of single cost terms (the C ABI ``kop_term_*``, FP64).

The reference's cost builders return CostTerms whose ``evaluator`` /
``jacobian`` closures compute one term's raw rows and per-variable Jacobian
blocks in NumPy (costs.py:98-619); ``CostTerm.raw_residual`` and
``solver.assemble`` call them (solver.py:142-152, 289-324).  Here those
closures launch ``csrc/kop_terms.cu`` on the device for a batch of evaluation
points: the same rows, the same order, no CPU fallback.  ``*_batch``
functions take (B, ...) arrays; ``term_closures`` builds the single-point
evaluator / jacobian pair a typed CostTerm carries.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _device as dv
from ._lib import (KOP_BASE_NONE, KOP_BASE_SE2, KOP_BASE_SE3, KOP_TERM_LIMIT, KOP_TERM_REST, KOP_TERM_SELF,
                   KOP_TERM_SMOOTHNESS, KOP_TERM_STENCIL, KOP_TERM_SWEPT, KOP_TERM_VELOCITY, KOP_TERM_WORLD, check, lib)
from .errors import UnsupportedFeatureError
from .liegroups import Transform2, Transform3

_JOINT_KINDS = {"limit": KOP_TERM_LIMIT, "rest": KOP_TERM_REST, "smoothness": KOP_TERM_SMOOTHNESS,
                "velocity": KOP_TERM_VELOCITY, "acceleration": KOP_TERM_STENCIL, "jerk": KOP_TERM_STENCIL}
_COLLISION_KINDS = {"world_collision": KOP_TERM_WORLD, "self_collision": KOP_TERM_SELF,
                    "swept_collision": KOP_TERM_SWEPT}


def _base_arrays(bases):
    """Base values (Transform2 | Transform3) -> (kind, (B, 7) wxyz xyz, tangent dim)."""
    if isinstance(bases[0], Transform2):
        if not all(isinstance(b, Transform2) for b in bases):
            raise TypeError("mixed base variable types")
        return KOP_BASE_SE2, np.stack([b.to_transform3().as_array() for b in bases]), 3
    if isinstance(bases[0], Transform3):
        if not all(isinstance(b, Transform3) for b in bases):
            raise TypeError("mixed base variable types")
        return KOP_BASE_SE3, np.stack([b.as_array() for b in bases]), 6
    raise TypeError(f"base variable must be a Transform2 or Transform3, got {type(bases[0]).__name__}")


def pose_rows_batch(model, link: str, target: Transform3, q, bases=None, jacobian: bool = True):
    """pose_cost rows (costs.py:98-166) at (B, n) configurations: r (B, 6), J_q (B, 6, n) and,
    with a base per point (Transform2 / Transform3 list), J_base (B, 6, 3 | 6)."""
    q = np.ascontiguousarray(np.asarray(q, dtype=float).reshape(-1, model.actuated_count))
    b, n = q.shape
    kind, base, db = KOP_BASE_NONE, None, 0
    if bases is not None:
        kind, base, db = _base_arrays(list(bases))
    tgt = np.ascontiguousarray(target.as_array(), dtype=float)
    qd = dv.to_dev(q)
    bd = dv.to_dev(base) if base is not None else None
    r = dv.empty((b, 6))
    jq = dv.empty((b, 6, n)) if jacobian else None
    jb = dv.empty((b, 6, db)) if jacobian and db else None
    check(lib().kop_term_pose(model._handle, model.link_index(link), tgt.ctypes.data, kind, dv.ptr(qd), dv.ptr(bd), b,
                              dv.ptr(r), dv.ptr(jq), dv.ptr(jb), dv.stream_handle()), "kop_term_pose")
    out = [r.cpu().numpy()]
    if jacobian:
        out.append(jq.cpu().numpy())
        out.append(jb.cpu().numpy() if jb is not None else None)
    return tuple(out)


def joint_rows_batch(model, kind: str, qs, rest=None, velocity_limits=None, dt: float = 0.0, coeffs=None,
                     jacobian: bool = True):
    """Joint-space rows (limit / rest / smoothness / velocity / stencils, costs.py:174-341) at
    qs (B, nvars, n): r (B, n) and the Jacobian blocks (B, nvars, n, n) (diagonal)."""
    code = _JOINT_KINDS[kind]
    n = model.actuated_count
    qs = np.ascontiguousarray(np.asarray(qs, dtype=float))
    b, nv = qs.shape[0], qs.shape[1]
    keep = []

    def host(x):
        if x is None:
            return None
        a = np.ascontiguousarray(np.asarray(x, dtype=float).reshape(-1))
        keep.append(a)
        return a.ctypes.data
    qd = dv.to_dev(qs)
    r = dv.empty((b, n))
    jd = dv.empty((b, nv, n)) if jacobian else None
    check(lib().kop_term_joint(model._handle, code, host(rest), host(velocity_limits), float(dt), host(coeffs),
                               dv.ptr(qd), b, dv.ptr(r), dv.ptr(jd), dv.stream_handle()), f"kop_term_joint({kind})")
    if not jacobian:
        return (r.cpu().numpy(),)
    d = jd.cpu().numpy()
    blocks = np.zeros((b, nv, n, n))
    idx = np.arange(n)
    blocks[:, :, idx, idx] = d
    return r.cpu().numpy(), blocks


def collision_rows_batch(model, kind: str, q0, q1=None, world=None, eta: float = 0.05, sharpness: float = 100.0,
                         hard_min: bool = False, jacobian: bool = True):
    """Collision rows (world / self / swept, costs.py:423-619) at (B, n) configurations (q1: the
    second timestep of swept rows): r (B, rows), J0 (B, rows, n) (and J1 for swept)."""
    from .solver import _obstacles

    code = _COLLISION_KINDS[kind]
    n = model.actuated_count
    q0 = np.ascontiguousarray(np.asarray(q0, dtype=float).reshape(-1, n))
    b = q0.shape[0]
    nobs = len(world.obstacles) if world is not None else 0
    obs = _obstacles(world) if nobs else None
    rows = lib().kop_term_rows(model._handle, code, nobs)
    if rows < 0:
        check(rows, "kop_term_rows")
    q0d = dv.to_dev(q0)
    q1d = dv.to_dev(np.ascontiguousarray(np.asarray(q1, dtype=float).reshape(-1, n))) if q1 is not None else None
    r = dv.empty((b, rows))
    j0 = dv.empty((b, rows, n)) if jacobian else None
    j1 = dv.empty((b, rows, n)) if jacobian and code == KOP_TERM_SWEPT else None
    check(lib().kop_term_collision(model._handle, code, obs, nobs, float(eta), float(sharpness), int(hard_min),
                                   dv.ptr(q0d), dv.ptr(q1d), b, dv.ptr(r), dv.ptr(j0), dv.ptr(j1),
                                   dv.stream_handle()), f"kop_term_collision({kind})")
    out = [r.cpu().numpy()]
    if jacobian:
        out.append(j0.cpu().numpy())
        if j1 is not None:
            out.append(j1.cpu().numpy())
    return tuple(out)


def manipulability_batch(model, link: str, q, eps: float = 1e-6, jacobian: bool = True, derivative: bool = False):
    """manipulability_cost rows (costs.py:349-401) at (B, n): r (B, 1), gradient rows (B, 1, n);
    derivative=True also returns the translational Jacobian (B, 3, n) and dJ/dq (B, n, 3, n)."""
    n = model.actuated_count
    q = np.ascontiguousarray(np.asarray(q, dtype=float).reshape(-1, n))
    b = q.shape[0]
    qd = dv.to_dev(q)
    r, jr = dv.empty((b, 1)), dv.empty((b, 1, n)) if jacobian else None
    jac = dv.empty((b, 3, n)) if derivative else None
    djac = dv.empty((b, n, 3, n)) if derivative else None
    check(lib().kop_term_manipulability(model._handle, model.link_index(link), float(eps), dv.ptr(qd), b, dv.ptr(r),
                                        dv.ptr(jr), dv.ptr(jac), dv.ptr(djac), dv.stream_handle()),
          "kop_term_manipulability")
    out = [r.cpu().numpy()]
    if jacobian:
        out.append(jr.cpu().numpy())
    if derivative:
        out += [jac.cpu().numpy(), djac.cpu().numpy()]
    return tuple(out)


def term_closures(kind: str, params: dict, nvars: int):
    """(evaluator(*values), jacobian(*values)) for one typed CostTerm, evaluated on the device
    at a single point -- the closures the reference's builders return."""
    p = params
    if kind == "pose":
        def ev(q, *base):
            return pose_rows_batch(p["model"], p["link"], p["target"], q, [base[0]] if base else None,
                                   jacobian=False)[0][0]

        def jac(q, *base):
            r, jq, jb = pose_rows_batch(p["model"], p["link"], p["target"], q, [base[0]] if base else None)
            return [jq[0]] + ([jb[0]] if base else [])
        return ev, jac
    if kind in _JOINT_KINDS:
        model = p["model"] if "model" in p else None
        kw = {}
        if kind == "rest":
            kw["rest"] = p["q_rest"]
        if kind == "velocity":
            kw.update(velocity_limits=p["model"].velocity_limits, dt=p["dt"])
        if kind in ("acceleration", "jerk"):
            kw["coeffs"] = p["coeffs"]

        def run(values, jacobian):
            m = model or p.get("model") or _RestModel(len(values[0]))
            qs = np.stack([np.asarray(v, dtype=float).reshape(-1) for v in values])[None]
            return joint_rows_batch(m, kind, qs, jacobian=jacobian, **kw)

        def ev(*values):
            return run(values, False)[0][0]

        def jac(*values):
            return list(run(values, True)[1][0])
        return ev, jac
    if kind == "velocity_direct":  # |qd - 0| - limit * 1: the velocity rows' second block
        def run_direct(qd, jacobian):
            n = p["model"].actuated_count
            qs = np.stack([np.zeros(n), np.asarray(qd, dtype=float).reshape(-1)])[None]
            return joint_rows_batch(p["model"], "velocity", qs, velocity_limits=p["model"].velocity_limits, dt=1.0,
                                    jacobian=jacobian)

        def ev(qd):
            return run_direct(qd, False)[0][0]

        def jac(qd):
            return [run_direct(qd, True)[1][0][1]]
        return ev, jac
    if kind in _COLLISION_KINDS:
        kw = dict(world=p.get("world"), eta=p["eta"], sharpness=p["sharpness"], hard_min=p["hard_min"])

        def ev(*values):
            return collision_rows_batch(p["model"], kind, values[0], values[1] if len(values) > 1 else None,
                                        jacobian=False, **kw)[0][0]

        def jac(*values):
            out = collision_rows_batch(p["model"], kind, values[0], values[1] if len(values) > 1 else None, **kw)
            return [b[0] for b in out[1:]]
        return ev, jac

    if kind == "manipulability":
        def ev(q):
            return manipulability_batch(p["model"], p["link"], q, p["eps"], jacobian=False)[0][0]

        def jac(q):
            return [manipulability_batch(p["model"], p["link"], q, p["eps"])[1][0]]
        return ev, jac

    def unsupported(*values):
        raise UnsupportedFeatureError(f"cost kind '{kind}' has no device evaluation kernel (no CPU fallback)")
    return unsupported, unsupported


class _RestModel:
    """rest_cost binds no model (costs.py:259-271): the joint kernel only needs n; it runs on a
    private one-column-per-joint model handle of the right width."""

    _cache: dict = {}

    def __new__(cls, n: int):
        if n not in cls._cache:
            from .robot import Joint, RobotModel

            links = [f"l{i}" for i in range(n + 1)]
            joints = [Joint(f"j{i}", "prismatic", links[i], links[i + 1], Transform3.identity(),
                            np.array([1.0, 0.0, 0.0])) for i in range(n)]
            cls._cache[n] = RobotModel(links, joints)
        return cls._cache[n]
