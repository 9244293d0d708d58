"""Nonlinear least squares on the device: CostTerm / Problem / solve (solver.py).

The reference's generic LM (solver.py:364-429: dense Cholesky, per-iteration
rejection loop with damping x10, gradient / step / numerical-failure
terminations) runs here as one GPU thread per problem (csrc/kop_collision.cu,
``kop_lm_solve``) for problems built from the typed cost builders of
``costs.py``: one configuration variable and the pose / limit / rest /
world-collision / self-collision families (the viewer's stack,
server.py:60-97, and config 4), several pose costs on a tree (config 3,
one warp per problem), and plan_trajectory-shaped problems over T
configuration variables (config 5, one CTA per problem, banded normal
equations).  ``solve_batch`` launches every compatible problem of a batch
together.  Costs built from Python callables cannot run on
the device and raise UnsupportedFeatureError -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np

from .errors import CostEvaluationError, UnsupportedFeatureError
from .liegroups import Rotation3, Transform2, Transform3

DENSE_TANGENT_LIMIT = 200
DAMPING_MAX = 1e10
DAMPING_MIN = 1e-12
DIAG_CLAMP = 1e-8
TERMINATIONS = {0: ("max_iterations", ""), 1: ("gradient_converged", ""), 2: ("step_converged", ""),
                3: ("numerical_failure", "no acceptable step below damping 1e10"),
                4: ("step_converged", "rejection budget exhausted without descent"),
                5: ("numerical_failure", "cost evaluation returned a non-finite residual"),
                6: ("step_converged", "no cost decrease resolvable in FP32 (model decrease below 2^-17 of the cost)")}


def _tangent_dim(x) -> int:
    if isinstance(x, Transform3):
        return 6
    if isinstance(x, (Transform2, Rotation3)):
        return 3
    return int(np.asarray(x).size)


class VariableSet:
    """Ordered, typed variables (solver.py:36-108; value access)."""

    def __init__(self):
        self._ids, self._values, self._index = [], [], {}
        self.tangent_offsets = [0]

    @staticmethod
    def of(**variables) -> "VariableSet":
        vs = VariableSet()
        for k, v in variables.items():
            vs.add(k, v)
        return vs

    def add(self, var_id: str, value) -> "VariableSet":
        if var_id in self._index:
            raise ValueError(f"duplicate variable id '{var_id}'")
        if isinstance(value, (list, tuple)) or np.isscalar(value):
            value = np.atleast_1d(np.asarray(value, dtype=float))
        if isinstance(value, np.ndarray):
            value = value.astype(float).reshape(-1)
        elif not isinstance(value, (Transform3, Transform2, Rotation3)):
            raise TypeError(f"unsupported variable type {type(value).__name__}")
        self._index[var_id] = len(self._ids)
        self._ids.append(var_id)
        self._values.append(value)
        self.tangent_offsets.append(self.tangent_offsets[-1] + _tangent_dim(value))
        return self

    @property
    def ids(self):
        return list(self._ids)

    @property
    def tangent_dim(self) -> int:
        return self.tangent_offsets[-1]

    def index(self, var_id: str) -> int:
        try:
            return self._index[var_id]
        except KeyError:
            raise ValueError(f"unknown variable '{var_id}'") from None

    def value(self, var_id: str):
        return self._values[self.index(var_id)]

    def values(self, var_ids) -> list:
        return [self._values[self.index(v)] for v in var_ids]

    def tangent_slice(self, var_id: str) -> slice:
        i = self.index(var_id)
        return slice(self.tangent_offsets[i], self.tangent_offsets[i + 1])

    def updated(self, delta) -> "VariableSet":
        """A copy with the stacked tangent step applied through each variable's
        retraction (solver.py:91-102)."""
        from .liegroups import local_update

        delta = np.asarray(delta, dtype=float)
        if delta.shape != (self.tangent_dim,):
            raise ValueError(f"tangent step has shape {delta.shape}, expected ({self.tangent_dim},)")
        out = VariableSet()
        for i, (vid, value) in enumerate(zip(self._ids, self._values)):
            out.add(vid, local_update(value, delta[self.tangent_offsets[i]:self.tangent_offsets[i + 1]]))
        return out

    def copy(self) -> "VariableSet":
        out = VariableSet()
        for vid, v in zip(self._ids, self._values):
            out.add(vid, v.copy() if isinstance(v, np.ndarray) else v)
        return out


@dataclass
class CostTerm:
    """Weighted residual block (solver.py:111-152).  ``kind``/``params`` describe a
    device cost family; ``evaluator``/``jacobian`` callables are accepted for API
    compatibility but cannot be evaluated on the device."""

    name: str
    residual_dim: int
    variable_refs: list
    weight: np.ndarray
    evaluator: object = None
    jacobian: object = None
    kind: str | None = None
    params: dict = field(default_factory=dict)

    def __post_init__(self):
        w = np.asarray(self.weight, dtype=float)
        if w.ndim == 0:
            w = np.full(self.residual_dim, float(w))
        if w.shape != (self.residual_dim,):
            raise ValueError(f"cost '{self.name}': weight shape {w.shape} does not match residual_dim "
                             f"{self.residual_dim}")
        if np.any(w < 0.0):
            raise ValueError(f"cost '{self.name}': weights must be nonnegative")
        self.weight = w

    def raw_residual(self, values) -> np.ndarray:
        """The unweighted residual at the referenced variables' values (solver.py:142-152);
        typed terms evaluate on the device (terms.py)."""
        if self.evaluator is None:
            raise UnsupportedFeatureError(f"cost '{self.name}' has no evaluator")
        r = np.asarray(self.evaluator(*values), dtype=float).reshape(-1)
        if r.shape != (self.residual_dim,):
            raise CostEvaluationError(self.name, f"evaluator returned shape {r.shape}, declared residual_dim "
                                                 f"{self.residual_dim}")
        if not np.all(np.isfinite(r)):
            raise CostEvaluationError(self.name, "evaluator returned non-finite residual")
        return r


@dataclass
class Problem:
    variables: VariableSet
    costs: list

    def __post_init__(self):
        for cost in self.costs:
            for ref in cost.variable_refs:
                self.variables.index(ref)

    @property
    def residual_dim(self) -> int:
        return sum(c.residual_dim for c in self.costs)

    @property
    def sparsity(self) -> list:
        """Structurally nonzero (cost index, variable index) blocks (solver.py:166-172)."""
        return [(ci, self.variables.index(ref)) for ci, cost in enumerate(self.costs) for ref in cost.variable_refs]


@dataclass
class SolveOptions:
    max_iterations: int = 100
    initial_damping: float = 1e-4
    damping_increase: float = 10.0
    damping_decrease: float = 1.0 / 3.0
    gradient_tolerance: float = 1e-8
    step_tolerance: float = 1e-10
    linear_solver: str | None = None
    max_rejections: int = 20
    precision: str = "fp64"

    def __post_init__(self):
        if self.max_iterations <= 0 or self.initial_damping <= 0:
            raise ValueError("max_iterations and initial_damping must be positive")
        if self.damping_increase <= 1.0:
            raise ValueError("damping_increase must exceed 1")
        if not 0.0 < self.damping_decrease < 1.0:
            raise ValueError("damping_decrease must be in (0, 1)")
        if self.linear_solver not in (None, "dense_cholesky", "sparse_cholesky"):
            raise ValueError(f"unknown linear_solver '{self.linear_solver}'")


@dataclass
class SolveReport:
    final_values: VariableSet
    initial_cost: float
    final_cost: float
    iterations_run: int
    termination: str  # max_iterations | gradient_converged | step_converged | numerical_failure
    cost_history: list = field(default_factory=list)
    solve_time_s: float = 0.0
    message: str = ""

    def to_json(self, include_timing: bool = False) -> dict:
        out = {"initial_cost": self.initial_cost, "final_cost": self.final_cost,
               "iterations_run": self.iterations_run, "termination": self.termination,
               "cost_history": list(self.cost_history)}
        if self.message:
            out["message"] = self.message
        if include_timing:
            out["solve_time_s"] = self.solve_time_s
        return out


# ---------------------------------------------------------------------------
# assembly of the weighted stack (solver.py:216-324): per-term evaluations
# (device kernels for typed terms, terms.py) stacked into r and a block Jacobian
# ---------------------------------------------------------------------------

class BlockJacobian:
    """Weighted Jacobian as per-(cost, variable) dense blocks (solver.py:216-257)."""

    def __init__(self, problem: "Problem", row_offsets: list, blocks: dict):
        self.problem = problem
        self.row_offsets = row_offsets
        self.blocks = blocks  # (cost index, variable index) -> (m, td)
        self.shape = (row_offsets[-1], problem.variables.tangent_dim)

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.shape)
        offsets = self.problem.variables.tangent_offsets
        for (ci, vi), block in self.blocks.items():
            r0 = self.row_offsets[ci]
            out[r0:r0 + block.shape[0], offsets[vi]:offsets[vi] + block.shape[1]] = block
        return out

    def to_csr(self):
        import scipy.sparse

        offsets = self.problem.variables.tangent_offsets
        rows, cols, vals = [], [], []
        for (ci, vi), block in self.blocks.items():
            m, td = block.shape
            rr, cc = np.meshgrid(np.arange(m), np.arange(td), indexing="ij")
            rows.append((rr + self.row_offsets[ci]).ravel())
            cols.append((cc + offsets[vi]).ravel())
            vals.append(block.ravel())
        if not rows:
            return scipy.sparse.csr_matrix(self.shape)
        return scipy.sparse.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                       shape=self.shape)


def numeric_jacobian(cost: CostTerm, values, step: float = 1e-6) -> list:
    """Central differences of the raw residual in tangent space (solver.py:260-279)."""
    from .liegroups import local_update

    blocks = []
    for k, value in enumerate(values):
        td = _tangent_dim(value)
        block = np.empty((cost.residual_dim, td))
        for j in range(td):
            d = np.zeros(td)
            d[j] = step
            plus, minus = list(values), list(values)
            plus[k] = local_update(value, d)
            minus[k] = local_update(value, -d)
            block[:, j] = (cost.raw_residual(plus) - cost.raw_residual(minus)) / (2 * step)
        if not np.all(np.isfinite(block)):
            raise CostEvaluationError(cost.name, "non-finite numeric Jacobian")
        blocks.append(block)
    return blocks


def _residual_vector(problem: "Problem", at: VariableSet) -> np.ndarray:
    parts = [c.weight * c.raw_residual(at.values(c.variable_refs)) for c in problem.costs]
    return np.concatenate(parts) if parts else np.zeros(0)


def assemble(problem: "Problem", at: VariableSet):
    """Stacked weighted residual and block Jacobian at ``at`` (solver.py:289-324)."""
    residuals, row_offsets, blocks = [], [0], {}
    for ci, cost in enumerate(problem.costs):
        values = at.values(cost.variable_refs)
        r = cost.raw_residual(values)
        residuals.append(cost.weight * r)
        row_offsets.append(row_offsets[-1] + cost.residual_dim)
        raw = cost.jacobian(*values) if cost.jacobian is not None else numeric_jacobian(cost, values)
        if len(raw) != len(cost.variable_refs):
            raise CostEvaluationError(cost.name, f"jacobian returned {len(raw)} blocks for "
                                                 f"{len(cost.variable_refs)} variables")
        for ref, block in zip(cost.variable_refs, raw):
            vi = problem.variables.index(ref)
            block = np.asarray(block, dtype=float)
            expected = (cost.residual_dim, at.tangent_offsets[vi + 1] - at.tangent_offsets[vi])
            if block.shape != expected:
                raise CostEvaluationError(cost.name, f"jacobian block shape {block.shape}, expected {expected}")
            weighted = cost.weight[:, None] * block
            blocks[(ci, vi)] = blocks[(ci, vi)] + weighted if (ci, vi) in blocks else weighted
    r = np.concatenate(residuals) if residuals else np.zeros(0)
    return r, BlockJacobian(problem, row_offsets, blocks)


# ---------------------------------------------------------------------------
# mapping typed problems onto the device stack
# ---------------------------------------------------------------------------

_DEVICE_KINDS = ("pose", "limit", "rest", "world_collision", "self_collision")


@dataclass
class _Plan:
    model: object
    link: str
    var: str
    target: Transform3
    costs: object  # KopCollisionCosts (path "chain") or KopPoseCosts (path "tree")
    keep: list     # ctypes / numpy arrays kept alive
    key: tuple
    path: str = "chain"
    targets: list = field(default_factory=list)  # tree path: one Transform3 per pose cost
    traj: dict = field(default_factory=dict)     # traj path: var ids, anchors, obstacle table
    base: str | None = None                      # tree path: the pose costs' base variable (SE(2) / SE(3))
    base_kind: int = 0


def _obstacles(world):
    from . import _lib as L
    from .collision import Capsule, HalfSpace, Sphere

    arr = (L.KopObstacle * max(1, len(world.obstacles)))()
    for i, ob in enumerate(world.obstacles):
        if isinstance(ob, Sphere):
            arr[i].kind, arr[i].a[:], arr[i].radius = 0, list(ob.center), ob.radius
        elif isinstance(ob, Capsule):
            arr[i].kind, arr[i].a[:], arr[i].b[:], arr[i].radius = 1, list(ob.endpoint_a), list(ob.endpoint_b), \
                ob.radius
        elif isinstance(ob, HalfSpace):
            arr[i].kind, arr[i].a[:], arr[i].radius = 2, list(ob.normal), ob.offset
        else:
            raise UnsupportedFeatureError(f"unsupported obstacle kind {type(ob).__name__}")
    return arr


def _uniform(w, name):
    w = np.asarray(w, dtype=float)
    if w.size and not np.all(w == w[0]):
        raise UnsupportedFeatureError(f"cost '{name}': per-row weights are not supported on the device")
    return float(w[0]) if w.size else 0.0


def plan(problem: Problem) -> _Plan:
    """Typed device plan of a problem, or UnsupportedFeatureError.

    path "chain": one pose cost (+ limit / rest / world / self collision) on a
    root->link chain of <= 8 moving joints -- one thread per problem
    (kop_lm_solve).  path "tree": several pose costs (multi end effector) and
    limit / rest on trees of <= 32 actuated joints -- one warp per problem
    (kop_multi_pose_solve, config 3)."""
    from . import _lib as L

    if not problem.costs or problem.residual_dim < 1:
        raise ValueError("problem must declare at least one cost with residual rows")
    base_vars = {c.params.get("base_var") for c in problem.costs if c.kind == "pose"}
    base_var = None
    if base_vars - {None}:
        if len(base_vars) != 1:
            raise UnsupportedFeatureError("pose costs must all use the same base variable (or none)")
        base_var = base_vars.pop()
        if len(problem.variables.ids) != 2:
            raise UnsupportedFeatureError("a base-variable device solve takes one configuration and one base variable")
    elif len(problem.variables.ids) > 1:
        return _plan_trajectory(problem)
    var = [v for v in problem.variables.ids if v != base_var][0]
    by, poses = {}, []
    for c in problem.costs:
        if c.kind not in _DEVICE_KINDS:
            raise UnsupportedFeatureError(
                f"cost '{c.name}' has no device kernel (custom Python costs cannot run on the GPU; "
                "there is no CPU fallback)")
        if c.kind == "pose":
            poses.append(c)
            continue
        if c.kind in by:
            raise UnsupportedFeatureError(f"more than one '{c.kind}' cost in a device problem")
        by[c.kind] = c
    if not poses:
        raise UnsupportedFeatureError("device solve needs a pose cost")
    model = poses[0].params["model"]
    value = problem.variables.value(var)
    if not isinstance(value, np.ndarray) or value.size != model.actuated_count:
        raise ValueError(f"variable '{var}' must be a configuration of {model.actuated_count} values")
    for c in poses + list(by.values()):
        if c.params.get("model", model) is not model:
            raise UnsupportedFeatureError("all costs of a device problem must use the same RobotModel")
    collision = "world_collision" in by or "self_collision" in by
    link = poses[0].params["link"]
    if base_var is not None:
        from ._lib import KOP_BASE_SE2, KOP_BASE_SE3

        bval = problem.variables.value(base_var)
        if isinstance(bval, Transform2):
            base_kind = KOP_BASE_SE2
        elif isinstance(bval, Transform3):
            base_kind = KOP_BASE_SE3
        else:
            raise UnsupportedFeatureError(f"base variable '{base_var}' must be a Transform2 or Transform3")
        if collision:
            raise UnsupportedFeatureError("collision costs with a base variable are not supported by the device solve")
        if any(base_var in c.variable_refs for c in by.values()):
            raise UnsupportedFeatureError("only pose costs may reference the base variable")
    chain_ok = model.actuated_count <= 8 and model.chain_length(link) >= 0 and base_var is None
    w_lim = _uniform(by["limit"].weight, "limit") if "limit" in by else 0.0
    w_rest = _uniform(by["rest"].weight, "rest") if "rest" in by else 0.0
    if len(poses) == 1 and (chain_ok or collision):
        pose = poses[0]
        if "rest" in by and not np.array_equal(by["rest"].params["q_rest"], model.rest_pose):
            raise UnsupportedFeatureError("rest costs must use the model's rest pose on the chain solve")
        cc = L.KopCollisionCosts()
        cc.w_position, cc.w_orientation = _uniform(pose.weight[:3], pose.name), _uniform(pose.weight[3:], pose.name)
        cc.w_limit, cc.w_rest = w_lim, w_rest
        keep, world_key = [], ()
        cc.sharpness, cc.hard_min = 100.0, 0
        cc.eta_world = cc.eta_self = 1.0
        if "world_collision" in by:
            wcp = by["world_collision"].params
            arr = _obstacles(wcp["world"])
            keep.append(arr)
            cc.w_world, cc.eta_world = _uniform(by["world_collision"].weight, "world_collision"), wcp["eta"]
            cc.num_obstacles, cc.obstacles = len(wcp["world"].obstacles), arr
            cc.sharpness, cc.hard_min = wcp["sharpness"], int(wcp["hard_min"])
            world_key = (id(wcp["world"]), wcp["eta"], wcp["sharpness"], wcp["hard_min"])
        if "self_collision" in by:
            scp = by["self_collision"].params
            cc.w_self, cc.eta_self = _uniform(by["self_collision"].weight, "self_collision"), scp["eta"]
            if "world_collision" in by and (scp["sharpness"] != cc.sharpness or int(scp["hard_min"]) != cc.hard_min):
                raise UnsupportedFeatureError("world and self collision costs must share sharpness / hard_min")
            cc.sharpness, cc.hard_min = scp["sharpness"], int(scp["hard_min"])
        key = ("chain", id(model), link, cc.w_position, cc.w_orientation, cc.w_limit, cc.w_rest, cc.w_world,
               cc.w_self, cc.eta_self, world_key)
        return _Plan(model, link, var, pose.params["target"], cc, keep, key, "chain")
    if collision:
        raise UnsupportedFeatureError("collision costs need a single pose cost on a chain of <= 8 moving joints")
    if model.actuated_count > 32 or len(model.joints) > 64 or len(poses) > 8:
        raise UnsupportedFeatureError("tree solve supports <= 32 actuated joints, 64 joints and 8 pose costs")
    links = np.ascontiguousarray([model.link_index(p.params["link"]) for p in poses], dtype=np.int32)
    wpos = np.ascontiguousarray([_uniform(p.weight[:3], p.name) for p in poses])
    wori = np.ascontiguousarray([_uniform(p.weight[3:], p.name) for p in poses])
    rest = np.ascontiguousarray(by["rest"].params["q_rest"] if "rest" in by else model.rest_pose, dtype=float)
    pc = L.KopPoseCosts(len(poses), links.ctypes.data, wpos.ctypes.data, wori.ctypes.data, w_lim, w_rest,
                        rest.ctypes.data)
    key = ("tree", id(model), tuple(links), tuple(wpos), tuple(wori), w_lim, w_rest, rest.tobytes(),
           base_kind if base_var else 0)
    return _Plan(model, poses[0].params["link"], var, poses[0].params["target"], pc, [links, wpos, wori, rest],
                 key, "tree", [p.params["target"] for p in poses], base=base_var,
                 base_kind=base_kind if base_var else 0)


_TRAJ_KINDS = ("rest", "limit", "smoothness", "velocity", "acceleration", "jerk", "self_collision",
               "world_collision", "swept_collision")


def _plan_trajectory(problem: Problem) -> _Plan:
    """Path "traj": variables q_0..q_{T-1} (VariableSet order) under the
    plan_trajectory cost families (tasks.py:347-403) -- anchors (rest costs on
    q_0 / q_{T-1}), per-pair smoothness / velocity / swept collision, stencils
    on every 5-window, per-timestep limit / rest / self / world -- each family
    present everywhere it applies with one weight, or absent.  Solved by
    kop_traj_solve (CTA per trajectory, banded normal equations)."""
    from . import _lib as L
    from .trajectory import MAX_OBSTACLES, MAX_STEPS, _obstacle_table

    ids = problem.variables.ids
    T = len(ids)
    pos = {v: i for i, v in enumerate(ids)}
    model = None
    fam = {k: [] for k in _TRAJ_KINDS}
    for c in problem.costs:
        if c.kind not in _TRAJ_KINDS:
            raise UnsupportedFeatureError(
                f"cost '{c.name}' ({c.kind}) is not a trajectory family the device solve supports")
        m = c.params.get("model")
        if m is not None:
            if model is not None and m is not model:
                raise UnsupportedFeatureError("all costs of a device problem must use the same RobotModel")
            model = model or m
        fam[c.kind].append(c)
    if model is None:
        raise UnsupportedFeatureError("trajectory problem needs at least one model-bound cost")
    n = model.actuated_count
    for v in ids:
        val = problem.variables.value(v)
        if not isinstance(val, np.ndarray) or val.size != n:
            raise UnsupportedFeatureError(f"variable '{v}' is not a configuration of {n} values")
    if not 5 <= T <= MAX_STEPS:
        raise UnsupportedFeatureError(f"trajectory device solve needs 5..{MAX_STEPS} timesteps, got {T}")

    def steps(c):
        return [pos[r] for r in c.variable_refs]

    def uniform_family(kind, expect, what):
        """One cost per expected variable tuple, all with one weight (and params); returns the weight or 0."""
        cs = fam[kind]
        if not cs:
            return 0.0, None
        got = sorted(tuple(steps(c)) for c in cs)
        if got != sorted(expect):
            raise UnsupportedFeatureError(f"'{kind}' costs must cover {what}")
        w = {_uniform(c.weight, c.name) for c in cs}
        if len(w) != 1:
            raise UnsupportedFeatureError(f"'{kind}' costs must share one weight")
        return w.pop(), cs[0]

    pairs = [(t - 1, t) for t in range(1, T)]
    w_smooth, _ = uniform_family("smoothness", pairs, "every consecutive pair")
    w_vel, vc = uniform_family("velocity", pairs, "every consecutive pair")
    win = [tuple(range(t - 2, t + 3)) for t in range(2, T - 2)]
    w_acc, ac = uniform_family("acceleration", win, "every 5-window t-2..t+2, t = 2..T-3")
    w_jerk, jc = uniform_family("jerk", win, "every 5-window t-2..t+2, t = 2..T-3")
    each = [(t,) for t in range(T)]
    w_lim, _ = uniform_family("limit", each, "every timestep")
    w_self, sc = uniform_family("self_collision", each, "every timestep")
    w_world, wc = uniform_family("world_collision", each, "every timestep")
    w_swept, swc = uniform_family("swept_collision", pairs, "every consecutive pair")
    dts = {c.params["dt"] for c in fam["velocity"] + fam["acceleration"] + fam["jerk"]}
    if len(dts) > 1:
        raise UnsupportedFeatureError("velocity / stencil costs must share one dt")
    dt = dts.pop() if dts else 0.1
    if w_world or w_swept:
        if not (wc and swc) or w_world != w_swept:
            raise UnsupportedFeatureError("world and swept collision costs must both be present with one weight")
        worlds = {id(c.params["world"]) for c in fam["world_collision"] + fam["swept_collision"]}
        keyset = {(c.params["eta"], c.params["sharpness"], c.params["hard_min"])
                  for c in fam["world_collision"] + fam["swept_collision"]}
        if len(worlds) != 1 or len(keyset) != 1:
            raise UnsupportedFeatureError("world / swept collision costs must share one world, eta and softmin")
    if sc is not None and wc is not None and (sc.params["sharpness"], sc.params["hard_min"]) != (
            wc.params["sharpness"], wc.params["hard_min"]):
        raise UnsupportedFeatureError("world and self collision costs must share sharpness / hard_min")
    # rest costs: anchors on q_0 / q_{T-1}, optionally one rest family on every timestep
    rests = {t: [c for c in fam["rest"] if steps(c) == [t]] for t in range(T)}
    if any(len(c.variable_refs) != 1 for c in fam["rest"]):
        raise UnsupportedFeatureError("rest costs must bind one variable")
    inner = [rests[t] for t in range(1, T - 1)]
    w_rest, rest = 0.0, model.rest_pose
    if any(inner):
        if any(len(r) != 1 for r in inner):
            raise UnsupportedFeatureError("rest costs must be on every timestep or only on the endpoints")
        w_rest = _uniform(inner[0][0].weight, inner[0][0].name)
        rest = inner[0][0].params["q_rest"]
        for r in inner:
            if _uniform(r[0].weight, r[0].name) != w_rest or not np.array_equal(r[0].params["q_rest"], rest):
                raise UnsupportedFeatureError("per-timestep rest costs must share weight and rest pose")
    anchors = []
    for t in (0, T - 1):
        cand = list(rests[t])
        if w_rest:
            fam_c = [c for c in cand if _uniform(c.weight, c.name) == w_rest and np.array_equal(c.params["q_rest"], rest)]
            if not fam_c:
                raise UnsupportedFeatureError("the per-timestep rest cost is missing on an endpoint")
            cand.remove(fam_c[0])
        if len(cand) != 1:
            raise UnsupportedFeatureError("each endpoint needs exactly one anchor (rest) cost")
        anchors.append(cand[0])
    w_anchor = {_uniform(c.weight, c.name) for c in anchors}
    if len(w_anchor) != 1:
        raise UnsupportedFeatureError("the two anchor costs must share one weight")
    w_anchor = w_anchor.pop()
    vlim = np.ascontiguousarray(model.velocity_limits, dtype=float)
    rest = np.ascontiguousarray(rest, dtype=float)
    cp = (wc or sc).params if (wc or sc) else {"eta": 0.05, "sharpness": SOFTMIN_DEFAULT, "hard_min": False}
    tc = L.KopTrajCosts(T, dt, w_anchor, w_smooth, w_vel, w_acc, w_jerk, w_lim, w_rest, w_self,
                        sc.params["eta"] if sc is not None else 0.01, w_world,
                        wc.params["eta"] if wc is not None else 0.05, cp["sharpness"], int(cp["hard_min"]),
                        vlim.ctypes.data_as(C.POINTER(C.c_double)), rest.ctypes.data_as(C.POINTER(C.c_double)))
    world = wc.params["world"] if wc is not None else None
    if world is not None and len(world.obstacles) > MAX_OBSTACLES:
        raise UnsupportedFeatureError(f"more than {MAX_OBSTACLES} obstacles are not compiled in")
    table, n_obs = _obstacle_table([world] if world is not None else [], 1)
    link = model.link_names[-1]
    key = ("traj", id(model), T, dt, w_anchor, w_smooth, w_vel, w_acc, w_jerk, w_lim, w_rest, rest.tobytes(),
           w_self, w_world, n_obs, tc.eta_self, tc.eta_world, tc.sharpness, tc.hard_min)
    traj = {"vars": ids, "anchors": np.stack([anchors[0].params["q_rest"], anchors[1].params["q_rest"]]),
            "obstacles": table[0] if n_obs else None, "n_obs": n_obs}
    return _Plan(model, link, ids[0], Transform3.identity(), tc, [vlim, rest], key, "traj", traj=traj)


SOFTMIN_DEFAULT = 100.0


def _options(options: SolveOptions):
    from . import _lib as L
    from .robot import _precision

    o = L.KopLmOptions()
    o.max_iterations, o.initial_damping = options.max_iterations, options.initial_damping
    o.damping_increase, o.damping_decrease = options.damping_increase, options.damping_decrease
    o.gradient_tolerance, o.step_tolerance = options.gradient_tolerance, options.step_tolerance
    # range(max_rejections) in solver.py:389: a negative budget allows no trial, like 0
    o.max_rejections, o.precision = max(0, int(options.max_rejections)), _precision(options.precision)
    return o


def _base_state(value) -> np.ndarray:
    """Base variable -> the kernel's state: SE(2) (angle, x, y), SE(3) (wxyz, xyz)."""
    if isinstance(value, Transform2):
        return np.array([value.angle, value.translation[0], value.translation[1]])
    return value.as_array()


def _base_value(kind: int, state):
    from ._lib import KOP_BASE_SE2

    if kind == KOP_BASE_SE2:
        return Transform2(float(state[0]), np.array(state[1:3]))
    return Transform3.from_parts(state[:4], state[4:7])


def _run(plans, problems, options: SolveOptions) -> list:
    """One kop_lm_solve launch for problems sharing a plan key."""
    from . import _device as dv
    from ._lib import check, lib

    p0 = plans[0]
    b = len(plans)
    if p0.path == "traj":
        return _run_traj(plans, problems, options)
    if p0.path == "tree":
        tg = dv.to_dev(np.stack([np.stack([t.as_array() for t in p.targets]) for p in plans]))
    else:
        tg = dv.to_dev(np.stack([p.target.as_array() for p in plans]))
    q0 = dv.to_dev(np.stack([pr.variables.value(p.var) for p, pr in zip(plans, problems)]))
    n = p0.model.actuated_count
    t = dv.require_cuda()
    q, cost, init = dv.empty((b, n)), dv.empty(b), dv.empty(b)
    hist = dv.empty((b, options.max_iterations + 1))
    iters = t.empty(b, dtype=t.int32, device="cuda")
    term = t.empty(b, dtype=t.int32, device="cuda")
    opts = _options(options)
    t0 = time.perf_counter()
    base_out = None
    if p0.path == "tree" and p0.base is not None:
        b0 = np.stack([_base_state(pr.variables.value(p.base)) for p, pr in zip(plans, problems)])
        base0, base_out = dv.to_dev(b0), dv.empty(b0.shape)
        check(lib().kop_multi_pose_solve_base(p0.model._handle, C.byref(p0.costs), C.byref(opts), p0.base_kind,
                                              dv.ptr(tg), dv.ptr(q0), dv.ptr(base0), b, dv.ptr(q), dv.ptr(base_out),
                                              dv.ptr(cost), dv.ptr(init), dv.ptr(hist), dv.ptr(iters), dv.ptr(term),
                                              dv.stream_handle()), "kop_multi_pose_solve_base")
    elif p0.path == "tree":
        check(lib().kop_multi_pose_solve(p0.model._handle, C.byref(p0.costs), C.byref(opts), dv.ptr(tg), dv.ptr(q0),
                                         b, dv.ptr(q), dv.ptr(cost), dv.ptr(init), dv.ptr(hist), dv.ptr(iters),
                                         dv.ptr(term), dv.stream_handle()), "kop_multi_pose_solve")
    else:
        check(lib().kop_lm_solve(p0.model._handle, p0.model.link_index(p0.link), C.byref(p0.costs), C.byref(opts),
                                 dv.ptr(tg), dv.ptr(q0), b, dv.ptr(q), dv.ptr(cost), dv.ptr(init), dv.ptr(hist),
                                 dv.ptr(iters), dv.ptr(term), dv.stream_handle()), "kop_lm_solve")
    qh, ch, ih, hh = q.cpu().numpy(), cost.cpu().numpy(), init.cpu().numpy(), hist.cpu().numpy()
    ith, th = iters.cpu().numpy(), term.cpu().numpy()
    dt = (time.perf_counter() - t0) / b
    out = []
    bh = base_out.cpu().numpy() if base_out is not None else None
    for i, (p, pr) in enumerate(zip(plans, problems)):
        termination, message = TERMINATIONS[int(th[i])]
        h = hh[i, : int(ith[i]) + 1]
        if p.base is not None:  # both variables, in the problem's order
            vals = {p.var: qh[i], p.base: _base_value(p.base_kind, bh[i])}
            final = VariableSet()
            for vid in pr.variables.ids:
                final.add(vid, vals[vid])
        else:
            final = VariableSet.of(**{p.var: qh[i]})
        out.append(SolveReport(final_values=final, initial_cost=float(ih[i]),
                               final_cost=float(ch[i]), iterations_run=int(ith[i]), termination=termination,
                               cost_history=[float(x) for x in h], solve_time_s=dt, message=message))
    return out


def _run_traj(plans, problems, options: SolveOptions) -> list:
    """One kop_traj_solve launch for trajectory problems sharing a plan key."""
    from . import _device as dv
    from ._lib import check, lib

    p0 = plans[0]
    t = dv.require_cuda()
    b, T, n = len(plans), p0.costs.timesteps, p0.model.actuated_count
    qi = dv.to_dev(np.stack([np.stack([pr.variables.value(v) for v in p.traj["vars"]])
                             for p, pr in zip(plans, problems)]))
    anchors = dv.to_dev(np.stack([p.traj["anchors"] for p in plans]))
    n_obs = p0.traj["n_obs"]
    obs = dv.to_dev(np.stack([p.traj["obstacles"] for p in plans])) if n_obs else None
    q, cost, init = dv.empty((b, T, n)), dv.empty(b), dv.empty(b)
    hist = dv.empty((b, options.max_iterations + 1))
    iters = t.empty(b, dtype=t.int32, device="cuda")
    term = t.empty(b, dtype=t.int32, device="cuda")
    opts = _options(options)
    t0 = time.perf_counter()
    check(lib().kop_traj_solve(p0.model._handle, p0.model.link_index(p0.link), C.byref(p0.costs), C.byref(opts),
                               dv.ptr(qi), dv.ptr(anchors), dv.ptr(obs), n_obs, b, dv.ptr(q), dv.ptr(cost),
                               dv.ptr(init), dv.ptr(hist), dv.ptr(iters), dv.ptr(term), dv.stream_handle()),
          "kop_traj_solve")
    qh, ch, ih, hh = q.cpu().numpy(), cost.cpu().numpy(), init.cpu().numpy(), hist.cpu().numpy()
    ith, th = iters.cpu().numpy(), term.cpu().numpy()
    dt = (time.perf_counter() - t0) / b
    out = []
    for i, p in enumerate(plans):
        termination, message = TERMINATIONS[int(th[i])]
        values = VariableSet()
        for k, v in enumerate(p.traj["vars"]):
            values.add(v, qh[i, k])
        out.append(SolveReport(final_values=values, initial_cost=float(ih[i]), final_cost=float(ch[i]),
                               iterations_run=int(ith[i]), termination=termination,
                               cost_history=[float(x) for x in hh[i, : int(ith[i]) + 1]], solve_time_s=dt,
                               message=message))
    return out


def _raise_non_finite(problem: Problem, rep: SolveReport):
    """Device termination code 5 (a non-finite residual at the start or at a candidate) is where the
    reference's raw_residual raises CostEvaluationError (solver.py:142-152) out of solve()."""
    if rep.termination == "numerical_failure" and rep.message == TERMINATIONS[5][1]:
        raise CostEvaluationError(problem.costs[0].name, "evaluator returned non-finite residual")


def solve(problem: Problem, options: SolveOptions | None = None) -> SolveReport:
    """Minimise the sum of squared weighted residuals by LM on the device."""
    options = options or SolveOptions()
    rep = _run([plan(problem)], [problem], options)[0]
    _raise_non_finite(problem, rep)
    return rep


def solve_batch(problems: list, options: SolveOptions | None = None, workers: int = 1) -> list:
    """Solve independent problems; compatible ones share one device launch.
    Per-problem failures are isolated into that problem's report (solver.py:432-460)."""
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    options = options or SolveOptions()
    reports = [None] * len(problems)
    groups = {}
    for i, pr in enumerate(problems):
        try:
            p = plan(pr)
        except Exception as exc:  # isolate per-problem failures
            reports[i] = SolveReport(final_values=pr.variables, initial_cost=float("nan"), final_cost=float("nan"),
                                     iterations_run=0, termination="numerical_failure", message=str(exc))
            continue
        groups.setdefault(p.key, []).append((i, p))
    for members in groups.values():
        idx = [i for i, _ in members]
        for i, rep in zip(idx, _run([p for _, p in members], [problems[i] for i in idx], options)):
            try:
                _raise_non_finite(problems[i], rep)
                reports[i] = rep
            except CostEvaluationError as exc:  # the reference's isolated-failure report (solver.py:446-455)
                reports[i] = SolveReport(final_values=problems[i].variables, initial_cost=float("nan"),
                                         final_cost=float("nan"), iterations_run=0, termination="numerical_failure",
                                         message=str(exc))
    return reports
