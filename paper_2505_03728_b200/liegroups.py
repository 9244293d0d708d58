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
