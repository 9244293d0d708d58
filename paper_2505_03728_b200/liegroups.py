"""Host-side SO(3)/SE(3)/SE(2) value types for the public API.

These are the reference's value classes (liegroups.py:317-454) -- plain
float64 NumPy on the host, used to pass targets in and results out.  None of
the batched math runs here: the device kernels in ``csrc/kop_lie.cuh`` carry
the hot-path Lie algebra.

Conventions (liegroups.py:1-13): quaternions (w, x, y, z) with canonical sign
w >= 0 (at w == 0 the largest-magnitude vector component is positive),
translation-first twists, right-multiplicative retraction.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SMALL_ANGLE = 1e-7
_TWO_PI = 2.0 * math.pi


def quat_normalize_canonical(q) -> np.ndarray:
    q = np.asarray(q, dtype=float)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    s = np.where(q[..., :1] < 0.0, -1.0, 1.0)
    zw = q[..., 0] == 0.0
    if np.any(zw):
        v = q[..., 1:]
        lead = np.take_along_axis(v, np.argmax(np.abs(v), axis=-1)[..., None], axis=-1)
        s = np.where(zw[..., None], np.where(lead < 0.0, -1.0, 1.0), s)
    return q * s


def quat_mul(a, b) -> np.ndarray:
    a, b = np.asarray(a, dtype=float), np.asarray(b, dtype=float)
    w = a[..., :1] * b[..., :1] - np.sum(a[..., 1:] * b[..., 1:], axis=-1, keepdims=True)
    v = a[..., :1] * b[..., 1:] + b[..., :1] * a[..., 1:] + np.cross(a[..., 1:], b[..., 1:])
    return np.concatenate([w, v], axis=-1)


def quat_conj(q) -> np.ndarray:
    q = np.array(q, dtype=float, copy=True)
    q[..., 1:] *= -1.0
    return q


def quat_rotate(q, p) -> np.ndarray:
    q, p = np.asarray(q, dtype=float), np.asarray(p, dtype=float)
    t = 2.0 * np.cross(q[..., 1:], p)
    return p + q[..., :1] * t + np.cross(q[..., 1:], t)


def quat_to_matrix(q) -> np.ndarray:
    w, x, y, z = np.moveaxis(np.asarray(q, dtype=float), -1, 0)
    return np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], -2)


def quat_exp(omega) -> np.ndarray:
    omega = np.asarray(omega, dtype=float)
    th = np.linalg.norm(omega, axis=-1, keepdims=True)
    k = np.where(th < SMALL_ANGLE, 0.5 - th * th / 48.0, np.sin(0.5 * th) / np.where(th == 0.0, 1.0, th))
    return quat_normalize_canonical(np.concatenate([np.cos(0.5 * th), k * omega], axis=-1))


def quat_log(q) -> np.ndarray:
    q = np.asarray(q, dtype=float)
    q = q * np.where(q[..., :1] < 0.0, -1.0, 1.0)
    s = np.linalg.norm(q[..., 1:], axis=-1, keepdims=True)
    ang = 2.0 * np.arctan2(s, q[..., :1])
    scale = np.where(s < SMALL_ANGLE, 2.0 / np.maximum(q[..., :1], 0.5) * (1.0 - s * s / 3.0),
                     ang / np.where(s == 0.0, 1.0, s))
    return scale * q[..., 1:]


def _hat(v):
    v = np.asarray(v, dtype=float)
    return np.array([[0.0, -v[2], v[1]], [v[2], 0.0, -v[0]], [-v[1], v[0], 0.0]])


def skew(v) -> np.ndarray:
    """[v]x over the last axis: (..., 3) -> (..., 3, 3)."""
    v = np.asarray(v, dtype=float)
    z = np.zeros(v.shape[:-1])
    return np.stack([np.stack([z, -v[..., 2], v[..., 1]], -1), np.stack([v[..., 2], z, -v[..., 0]], -1),
                     np.stack([-v[..., 1], v[..., 0], z], -1)], -2)


def quat_from_matrix(m) -> np.ndarray:
    """Rotation matrix (..., 3, 3) -> canonical quaternion (..., 4) (Shepperd's
    method: the largest of w, x, y, z is recovered from the trace first)."""
    m = np.asarray(m, dtype=float)
    tr = m[..., 0, 0] + m[..., 1, 1] + m[..., 2, 2]
    cand = np.stack([tr, m[..., 0, 0], m[..., 1, 1], m[..., 2, 2]], -1)
    k = np.argmax(cand, axis=-1)
    out = np.empty(m.shape[:-2] + (4,))
    r = lambda i, j: m[..., i, j]
    s0 = np.sqrt(np.maximum(1.0 + tr, 0.0)) * 2.0
    s1 = np.sqrt(np.maximum(1.0 + r(0, 0) - r(1, 1) - r(2, 2), 0.0)) * 2.0
    s2 = np.sqrt(np.maximum(1.0 - r(0, 0) + r(1, 1) - r(2, 2), 0.0)) * 2.0
    s3 = np.sqrt(np.maximum(1.0 - r(0, 0) - r(1, 1) + r(2, 2), 0.0)) * 2.0
    safe = lambda x: np.where(x == 0.0, 1.0, x)
    q0 = np.stack([0.25 * s0, (r(2, 1) - r(1, 2)) / safe(s0), (r(0, 2) - r(2, 0)) / safe(s0),
                   (r(1, 0) - r(0, 1)) / safe(s0)], -1)
    q1 = np.stack([(r(2, 1) - r(1, 2)) / safe(s1), 0.25 * s1, (r(0, 1) + r(1, 0)) / safe(s1),
                   (r(0, 2) + r(2, 0)) / safe(s1)], -1)
    q2 = np.stack([(r(0, 2) - r(2, 0)) / safe(s2), (r(0, 1) + r(1, 0)) / safe(s2), 0.25 * s2,
                   (r(1, 2) + r(2, 1)) / safe(s2)], -1)
    q3 = np.stack([(r(1, 0) - r(0, 1)) / safe(s3), (r(0, 2) + r(2, 0)) / safe(s3), (r(1, 2) + r(2, 1)) / safe(s3),
                   0.25 * s3], -1)
    out = np.where((k == 0)[..., None], q0, np.where((k == 1)[..., None], q1, np.where((k == 2)[..., None], q2, q3)))
    return quat_normalize_canonical(out)


def _jl_coeffs(th):
    """(1 - cos th) / th^2, (th - sin th) / th^3 with series below 1e-3 rad."""
    small = th < 1e-3
    t = np.where(small, 1.0, th)
    t2 = th * th
    a = np.where(small, 0.5 - t2 / 24.0 + t2 * t2 / 720.0, (1.0 - np.cos(t)) / (t * t))
    b = np.where(small, 1.0 / 6.0 - t2 / 120.0 + t2 * t2 / 5040.0, (t - np.sin(t)) / t ** 3)
    return a, b


def so3_left_jacobian(omega) -> np.ndarray:
    """Jl(omega) = I + a [w]x + b [w]x^2, (..., 3) -> (..., 3, 3)."""
    omega = np.asarray(omega, dtype=float)
    th = np.linalg.norm(omega, axis=-1)[..., None, None]
    k = skew(omega)
    a, b = _jl_coeffs(th)
    return np.eye(3) + a * k + b * (k @ k)


def so3_left_jacobian_inv(omega) -> np.ndarray:
    """Jl(omega)^-1 = I - [w]x / 2 + c [w]x^2, c = (1 - (th/2) cot(th/2)) / th^2."""
    omega = np.asarray(omega, dtype=float)
    th = np.linalg.norm(omega, axis=-1)[..., None, None]
    k = skew(omega)
    small = th < 1e-3
    t = np.where(small, 1.0, th)
    h = 0.5 * t
    c = np.where(small, 1.0 / 12.0 + th * th / 720.0, (1.0 - h * np.cos(h) / np.sin(h)) / (t * t))
    return np.eye(3) - 0.5 * k + c * (k @ k)


def se3_exp_arrays(xi):
    """Translation-first twist (..., 6) -> (quaternion (..., 4), translation (..., 3))."""
    xi = np.asarray(xi, dtype=float)
    return quat_exp(xi[..., 3:]), np.einsum("...ij,...j->...i", so3_left_jacobian(xi[..., 3:]), xi[..., :3])


def se3_log_arrays(q, t) -> np.ndarray:
    """(quaternion, translation) -> translation-first twist (..., 6)."""
    phi = quat_log(q)
    rho = np.einsum("...ij,...j->...i", so3_left_jacobian_inv(phi), np.asarray(t, dtype=float))
    return np.concatenate([rho, phi], axis=-1)


def _se3_q(rho, phi):
    """Barfoot's Q(rho, phi) block of the SE(3) left Jacobian, series below 1e-2 rad."""
    th = np.linalg.norm(phi, axis=-1)[..., None, None]
    P, R = skew(phi), skew(rho)
    small = th < 1e-2
    t = np.where(small, 1.0, th)
    t2 = th * th
    c1 = np.where(small, 1 / 6 - t2 / 120 + t2 * t2 / 5040, (t - np.sin(t)) / t ** 3)
    c2 = np.where(small, 1 / 24 - t2 / 720 + t2 * t2 / 40320, (0.5 * t * t + np.cos(t) - 1.0) / t ** 4)
    c3 = np.where(small, 1 / 120 - t2 / 2520 + t2 * t2 / 120960, (2 * t - 3 * np.sin(t) + t * np.cos(t)) / (2 * t ** 5))
    PR, RP, PRP = P @ R, R @ P, P @ R @ P
    return 0.5 * R + c1 * (PR + RP + PRP) + c2 * (P @ P @ R + R @ P @ P - 3.0 * PRP) + c3 * (PRP @ P + P @ PRP)


def se3_left_jacobian_inv(xi) -> np.ndarray:
    """SE(3) left Jacobian inverse [[A, -A Q A], [0, A]], A = Jl^-1(phi) (..., 6, 6)."""
    xi = np.asarray(xi, dtype=float)
    a = so3_left_jacobian_inv(xi[..., 3:])
    out = np.zeros(xi.shape[:-1] + (6, 6))
    out[..., :3, :3] = a
    out[..., 3:, 3:] = a
    out[..., :3, 3:] = -a @ _se3_q(xi[..., :3], xi[..., 3:]) @ a
    return out


def se3_right_jacobian_inv(xi) -> np.ndarray:
    """Jr^-1(xi) = Jl^-1(-xi)."""
    return se3_left_jacobian_inv(-np.asarray(xi, dtype=float))


def se3_adjoint(q, t) -> np.ndarray:
    """Adjoint of (q, t) on translation-first twists: [[R, [t]x R], [0, R]]."""
    r = quat_to_matrix(q)
    out = np.zeros(r.shape[:-2] + (6, 6))
    out[..., :3, :3] = r
    out[..., 3:, 3:] = r
    out[..., :3, 3:] = skew(t) @ r
    return out


def se2_exp_arrays(delta):
    """SE(2) tangent (vx, vy, w) (..., 3) -> (angle (...), translation (..., 2))."""
    delta = np.asarray(delta, dtype=float)
    w = delta[..., 2]
    small = np.abs(w) < 1e-7
    ws = np.where(small, 1.0, w)
    s = np.where(small, 1.0 - w * w / 6.0, np.sin(ws) / ws)
    c = np.where(small, 0.5 * w, (1.0 - np.cos(ws)) / ws)
    vx, vy = delta[..., 0], delta[..., 1]
    return w, np.stack([s * vx - c * vy, c * vx + s * vy], -1)


def se2_log_arrays(angle, t) -> np.ndarray:
    """Inverse of se2_exp_arrays: (angle, translation) -> (vx, vy, w)."""
    w = np.asarray(angle, dtype=float)
    t = np.asarray(t, dtype=float)
    small = np.abs(w) < 1e-7
    ws = np.where(small, 1.0, w)
    s = np.where(small, 1.0 - w * w / 6.0, np.sin(ws) / ws)
    c = np.where(small, 0.5 * w, (1.0 - np.cos(ws)) / ws)
    det = s * s + c * c
    vx = (s * t[..., 0] + c * t[..., 1]) / det
    vy = (-c * t[..., 0] + s * t[..., 1]) / det
    return np.stack([vx, vy, w], -1)


def _jl(omega):
    th = float(np.linalg.norm(omega))
    k = _hat(omega)
    if th < SMALL_ANGLE:
        a, b = 0.5 - th * th / 24.0, 1.0 / 6.0 - th * th / 120.0
    else:
        a, b = (1.0 - math.cos(th)) / th ** 2, (th - math.sin(th)) / th ** 3
    return np.eye(3) + a * k + b * (k @ k)


def _jl_inv(omega):
    th = float(np.linalg.norm(omega))
    k = _hat(omega)
    if th < SMALL_ANGLE:
        b = 1.0 / 12.0 + th * th / 720.0
    else:
        h = 0.5 * th
        b = (1.0 - h * math.cos(h) / math.sin(h)) / (th * th)
    return np.eye(3) - 0.5 * k + b * (k @ k)


def wrap_angle(a):
    w = np.mod(np.asarray(a, dtype=float) + math.pi, _TWO_PI) - math.pi
    return np.where(w == -math.pi, math.pi, w)


def rot2(angle):
    c, s = np.cos(angle), np.sin(angle)
    return np.array([[c, -s], [s, c]])


@dataclass(frozen=True)
class Rotation3:
    """SO(3) element stored as a canonical unit quaternion (w, x, y, z)."""

    wxyz: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "wxyz", quat_normalize_canonical(np.asarray(self.wxyz, float).reshape(4)))

    @staticmethod
    def identity() -> "Rotation3":
        return Rotation3(np.array([1.0, 0.0, 0.0, 0.0]))

    @staticmethod
    def exp(omega) -> "Rotation3":
        return Rotation3(quat_exp(np.asarray(omega, float).reshape(3)))

    @staticmethod
    def from_matrix(m) -> "Rotation3":
        return Rotation3(quat_from_matrix(m))

    def log(self) -> np.ndarray:
        return quat_log(self.wxyz)

    def matrix(self) -> np.ndarray:
        return quat_to_matrix(self.wxyz)

    def compose(self, other: "Rotation3") -> "Rotation3":
        return Rotation3(quat_mul(self.wxyz, other.wxyz))

    def inverse(self) -> "Rotation3":
        return Rotation3(quat_conj(self.wxyz))

    def apply(self, p) -> np.ndarray:
        return quat_rotate(self.wxyz, p)

    def angle_to(self, other: "Rotation3") -> float:
        return float(np.linalg.norm(self.inverse().compose(other).log()))


@dataclass(frozen=True)
class Transform3:
    """SE(3) element: rotation plus translation (meters)."""

    rotation: Rotation3
    translation: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "translation", np.asarray(self.translation, float).reshape(3))

    @staticmethod
    def identity() -> "Transform3":
        return Transform3(Rotation3.identity(), np.zeros(3))

    @staticmethod
    def from_parts(wxyz, pos) -> "Transform3":
        return Transform3(Rotation3(wxyz), pos)

    @staticmethod
    def exp(xi) -> "Transform3":
        xi = np.asarray(xi, float).reshape(6)
        return Transform3(Rotation3.exp(xi[3:]), _jl(xi[3:]) @ xi[:3])

    def log(self) -> np.ndarray:
        om = self.rotation.log()
        return np.concatenate([_jl_inv(om) @ self.translation, om])

    def compose(self, other: "Transform3") -> "Transform3":
        return Transform3(self.rotation.compose(other.rotation),
                          self.translation + self.rotation.apply(other.translation))

    def inverse(self) -> "Transform3":
        ri = self.rotation.inverse()
        return Transform3(ri, -ri.apply(self.translation))

    def apply(self, p) -> np.ndarray:
        return self.rotation.apply(p) + self.translation

    def matrix(self) -> np.ndarray:
        m = np.eye(4)
        m[:3, :3], m[:3, 3] = self.rotation.matrix(), self.translation
        return m

    def as_array(self) -> np.ndarray:
        """(w, x, y, z, px, py, pz) -- the C ABI pose layout."""
        return np.concatenate([self.rotation.wxyz, self.translation])

    def to_json(self) -> dict:
        return {"wxyz": self.rotation.wxyz.tolist(), "pos": self.translation.tolist()}

    @staticmethod
    def from_json(data: dict) -> "Transform3":
        return Transform3.from_parts(data["wxyz"], data["pos"])


@dataclass(frozen=True)
class Transform2:
    """SE(2) element; angle wrapped to (-pi, pi]."""

    angle: float
    translation: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "angle", float(wrap_angle(self.angle)))
        object.__setattr__(self, "translation", np.asarray(self.translation, float).reshape(2))

    @staticmethod
    def identity() -> "Transform2":
        return Transform2(0.0, np.zeros(2))

    def compose(self, other: "Transform2") -> "Transform2":
        return Transform2(self.angle + other.angle, self.translation + rot2(self.angle) @ other.translation)

    def inverse(self) -> "Transform2":
        return Transform2(-self.angle, -(rot2(-self.angle) @ self.translation))

    def apply(self, p) -> np.ndarray:
        return rot2(self.angle) @ np.asarray(p, float) + self.translation

    @staticmethod
    def exp(delta) -> "Transform2":
        ang, t = se2_exp_arrays(np.asarray(delta, dtype=float).reshape(3))
        return Transform2(float(ang), t)

    def log(self) -> np.ndarray:
        return se2_log_arrays(self.angle, self.translation)

    def to_transform3(self) -> Transform3:
        return Transform3(Rotation3.exp([0.0, 0.0, self.angle]),
                          np.array([self.translation[0], self.translation[1], 0.0]))


def compose(a, b):
    return a.compose(b)


def inverse(a):
    return a.inverse()


def se3_log(t: Transform3) -> np.ndarray:
    return t.log()


def se3_exp(xi) -> Transform3:
    return Transform3.exp(xi)


def so3_log(r: Rotation3) -> np.ndarray:
    return r.log()


def so3_exp(omega) -> Rotation3:
    return Rotation3.exp(omega)


def apply(a, p) -> np.ndarray:
    return a.apply(p)


def interpolate(a: Transform3, b: Transform3, alpha: float) -> Transform3:
    """a * exp(alpha * log(a^-1 b)): the constant-twist path from a to b (liegroups.py:490-494)."""
    if not 0.0 <= alpha <= 1.0:
        raise ValueError(f"interpolation parameter must be in [0, 1], got {alpha}")
    return a.compose(Transform3.exp(float(alpha) * a.inverse().compose(b).log()))


def tangent_dim(x) -> int:
    if isinstance(x, Transform3):
        return 6
    if isinstance(x, (Transform2, Rotation3)):
        return 3
    return int(np.asarray(x).size)


def local_update(x, delta):
    """Right-multiplicative retraction x * exp(delta) (vector spaces: x + delta)."""
    if isinstance(x, (Transform3, Transform2, Rotation3)):
        return x.compose(type(x).exp(delta))
    return np.asarray(x, dtype=float) + np.asarray(delta, dtype=float)
