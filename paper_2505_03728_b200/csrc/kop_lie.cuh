// Device Lie-group kernels (SO(3)/SE(3)), templated on float / double.
//
// Conventions follow liegroups.py:1-13: quaternions (w,x,y,z), twists
// translation-first, right-multiplicative retraction.  The functions are
// register-only __device__ code meant to be inlined into the fused LM kernel.
//
// FP32 hazard: the reference's closed forms for the SO(3)/SE(3)
// Jacobian coefficients (liegroups.py:176-191, :210-235) cancel
// catastrophically in float well above its 1e-7 series threshold.  In float
// every coefficient is a Taylor polynomial (exact rational coefficients,
// derived independently of the reference's -- whose c2/c3 series carry a sign
// slip) over the whole [0, pi], relative error <= 1.4e-7; double
// uses the series below 0.03 rad and the closed forms above.
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "kop_check.cuh"

namespace kop {

template <typename T>
struct quat {
  T w, x, y, z;
};
template <typename T>
struct vec3 {
  T x, y, z;
};

// ---- scalar helpers ------------------------------------------------------
// float sin/cos of a joint half-angle: Cody-Waite reduction by pi/2 (two
// constants, exact for |x| < 2^12) and Cephes minimax polynomials on
// [-pi/4, pi/4] (<= 2 ulp), quadrant fixed up with selects.  Branch-free, no
// Payne-Hanek slow path: 20 instructions instead of sincosf's ~40 + branch.
// Valid for |x| < 4096 rad (LM iterates never leave that range; NaN/inf
// propagate to a non-finite cost, which the LM step rejects).
__device__ __forceinline__ void sincos_t(float x, float* sp, float* cp) {
  const float k = rintf(x * 0.63661977236758134f);
  const int q = (int)k;
  float y = fmaf(k, -1.57079637050628662109375f, x);
  y = fmaf(k, 4.37113900018624283e-8f, y);
  const float z = y * y;
  const float sy = fmaf(y * z, fmaf(z, fmaf(z, -1.9515295891e-4f, 8.3321608736e-3f), -1.6666654611e-1f), y);
  const float cy = fmaf(z * z, fmaf(z, fmaf(z, 2.443315711809948e-5f, -1.388731625493765e-3f),
                                   4.166664568298827e-2f), fmaf(z, -0.5f, 1.0f));
  const float s0 = (q & 1) ? cy : sy;
  const float c0 = (q & 1) ? sy : cy;
  *sp = (q & 2) ? -s0 : s0;
  *cp = ((q + 1) & 2) ? -c0 : c0;
}
__device__ __forceinline__ void sincos_t(double a, double* s, double* c) { sincos(a, s, c); }
__device__ __forceinline__ float sqrt_t(float a) { return sqrtf(a); }
__device__ __forceinline__ double sqrt_t(double a) { return sqrt(a); }
__device__ __forceinline__ float rsqrt_t(float a) { return rsqrtf(a); }
__device__ __forceinline__ double rsqrt_t(double a) { return ::rsqrt(a); }
__device__ __forceinline__ float atan2_t(float y, float x) { return atan2f(y, x); }
__device__ __forceinline__ double atan2_t(double y, double x) { return atan2(y, x); }
__device__ __forceinline__ float tan_t(float a) { return tanf(a); }
__device__ __forceinline__ double tan_t(double a) { return tan(a); }
__device__ __forceinline__ bool finite_t(float a) { return isfinite(a); }
// float: MUFU.RCP-based quotient (<= 2 ulp); double: IEEE division
__device__ __forceinline__ float div_t(float a, float b) { return __fdividef(a, b); }
__device__ __forceinline__ double div_t(double a, double b) { return a / b; }
__device__ __forceinline__ bool finite_t(double a) { return isfinite(a); }
// |v| and 1/|v| from dd = v.v (0 and +inf at dd = 0).  float: one MUFU.RSQ
// (<= 2 ulp) instead of an IEEE sqrt plus an IEEE division; double: exact.
__device__ __forceinline__ void norm_inv_t(float dd, float& n, float& inv) {
  inv = rsqrtf(dd);
  n = dd > 0.f ? dd * inv : 0.f;
}
__device__ __forceinline__ void norm_inv_t(double dd, double& n, double& inv) {
  n = sqrt(dd);
  inv = 1.0 / n;
}
__device__ __forceinline__ float norm_t(float dd) { return dd > 0.f ? dd * rsqrtf(dd) : 0.f; }
__device__ __forceinline__ double norm_t(double dd) { return sqrt(dd); }

template <typename T>
__device__ __forceinline__ T tmax(T a, T b) { return a > b ? a : b; }
template <typename T>
__device__ __forceinline__ T tmin(T a, T b) { return a < b ? a : b; }

// Series thresholds (double Jacobian coefficients; so(3) log in both types).
template <typename T>
struct LieConst;
template <>
struct LieConst<float> {
  static constexpr float series_below = 1.0f;
  static constexpr float log_series_below = 1e-7f;  // liegroups.py:23,139-140
};
template <>
struct LieConst<double> {
  static constexpr double series_below = 0.03;
  static constexpr double log_series_below = 1e-7;
};

// ---- quaternion kernels (liegroups.py:48-85) ------------------------------
template <typename T>
__device__ __forceinline__ vec3<T> cross(const vec3<T>& a, const vec3<T>& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
template <typename T>
__device__ __forceinline__ T dot(const vec3<T>& a, const vec3<T>& b) {
  return a.x * b.x + a.y * b.y + a.z * b.z;
}

// Hamilton product a*b.
template <typename T>
__device__ __forceinline__ quat<T> qmul(const quat<T>& a, const quat<T>& b) {
  return {a.w * b.w - (a.x * b.x + a.y * b.y + a.z * b.z),
          a.w * b.x + b.w * a.x + (a.y * b.z - a.z * b.y),
          a.w * b.y + b.w * a.y + (a.z * b.x - a.x * b.z),
          a.w * b.z + b.w * a.z + (a.x * b.y - a.y * b.x)};
}

// a * (c, 0, 0, s): composition with a rotation about the local z axis.
template <typename T>
__device__ __forceinline__ quat<T> qmul_z(const quat<T>& a, T c, T s) {
  return {a.w * c - a.z * s, a.x * c + a.y * s, a.y * c - a.x * s, a.z * c + a.w * s};
}

// Rotate p by unit q: p + w t + v x t with t = 2 v x p.
template <typename T>
__device__ __forceinline__ vec3<T> qrot(const quat<T>& q, const vec3<T>& p) {
  const vec3<T> v{q.x, q.y, q.z};
  vec3<T> t = cross(v, p);
  t = {T(2) * t.x, T(2) * t.y, T(2) * t.z};
  const vec3<T> u = cross(v, t);
  return {p.x + q.w * t.x + u.x, p.y + q.w * t.y + u.y, p.z + q.w * t.z + u.z};
}

// Third column of R(q) = q * e_z (the world direction of a local z axis).
template <typename T>
__device__ __forceinline__ vec3<T> qzaxis(const quat<T>& q) {
  return {T(2) * (q.x * q.z + q.w * q.y), T(2) * (q.y * q.z - q.w * q.x),
          T(1) - T(2) * (q.x * q.x + q.y * q.y)};
}

template <typename T>
struct mat3 {
  T m[3][3];
};

template <typename T>
__device__ __forceinline__ mat3<T> qmat(const quat<T>& q) {
  const T xx = q.x * q.x, yy = q.y * q.y, zz = q.z * q.z;
  const T xy = q.x * q.y, xz = q.x * q.z, yz = q.y * q.z;
  const T wx = q.w * q.x, wy = q.w * q.y, wz = q.w * q.z;
  mat3<T> r;
  r.m[0][0] = T(1) - T(2) * (yy + zz);
  r.m[0][1] = T(2) * (xy - wz);
  r.m[0][2] = T(2) * (xz + wy);
  r.m[1][0] = T(2) * (xy + wz);
  r.m[1][1] = T(1) - T(2) * (xx + zz);
  r.m[1][2] = T(2) * (yz - wx);
  r.m[2][0] = T(2) * (xz - wy);
  r.m[2][1] = T(2) * (yz + wx);
  r.m[2][2] = T(1) - T(2) * (xx + yy);
  return r;
}

template <typename T>
__device__ __forceinline__ vec3<T> mulT(const mat3<T>& r, const vec3<T>& v) {  // R^T v
  return {r.m[0][0] * v.x + r.m[1][0] * v.y + r.m[2][0] * v.z,
          r.m[0][1] * v.x + r.m[1][1] * v.y + r.m[2][1] * v.z,
          r.m[0][2] * v.x + r.m[1][2] * v.y + r.m[2][2] * v.z};
}
template <typename T>
__device__ __forceinline__ vec3<T> mul(const mat3<T>& r, const vec3<T>& v) {  // R v
  return {r.m[0][0] * v.x + r.m[0][1] * v.y + r.m[0][2] * v.z,
          r.m[1][0] * v.x + r.m[1][1] * v.y + r.m[1][2] * v.z,
          r.m[2][0] * v.x + r.m[2][1] * v.y + r.m[2][2] * v.z};
}

// ---- so(3) log (liegroups.py:130-141) -------------------------------------
// float: angle/|v| = 2 atan2(s, w)/s with w >= 0 after the sign flip, so only
// the first quadrant is needed: atan(r) = r P(r^2) on r = min/max in [0, 1]
// (polynomial below) and the pi/2 - atan(1/r) reflection by select.
// The s < 1e-7 series branch of the reference is kept (selected, not
// branched).
__device__ __forceinline__ vec3<float> qlog(quat<float> q) {
  if (q.w < 0.f) q = {-q.w, -q.x, -q.y, -q.z};
  const float s2 = q.x * q.x + q.y * q.y + q.z * q.z;
  const float rs = rsqrtf(s2);
  const float s = s2 * rs;
  const float w = q.w;
  const float mx = fmaxf(s, w), mn = fminf(s, w);
  const float r = __fdividef(mn, mx);
  const float r2 = r * r;
  // atan(r)/r as a degree-8 polynomial in r^2 on [0, 1] (weighted least-squares
  // near-minimax fit, |atan error| <= 1e-7 evaluated in float)
  float p = fmaf(r2, 2.9151442264e-03f, -1.6329356575e-02f);
  p = fmaf(p, r2, 4.3114652315e-02f);
  p = fmaf(p, r2, -7.5400433873e-02f);
  p = fmaf(p, r2, 1.0657660650e-01f);
  p = fmaf(p, r2, -1.4207892660e-01f);
  p = fmaf(p, r2, 1.9993148939e-01f);
  p = fmaf(p, r2, -3.3333098471e-01f);
  p = fmaf(p, r2, 9.9999998672e-01f);
  const float a = r * p;
  const float half = s > w ? 1.57079632679489662f - a : a;
  const float series = 2.f / fmaxf(w, 0.5f) * (1.f - s2 * (1.f / 3.f));
  const float scale = s < LieConst<float>::log_series_below ? series : 2.f * half * rs;
  return {scale * q.x, scale * q.y, scale * q.z};
}

template <typename T>
__device__ __forceinline__ vec3<T> qlog(quat<T> q) {
  if (q.w < T(0)) q = {-q.w, -q.x, -q.y, -q.z};
  const T s = sqrt_t(q.x * q.x + q.y * q.y + q.z * q.z);
  T scale;
  if (s < LieConst<T>::log_series_below) {
    scale = T(2) / tmax(q.w, T(0.5)) * (T(1) - s * s / T(3));
  } else {
    scale = div_t(T(2) * atan2_t(s, q.w), s);
  }
  return {scale * q.x, scale * q.y, scale * q.z};
}

// ---- Jacobian coefficients, Horner in t = theta^2 -------------------------
// c1 = (th - sin th)/th^3;  k2 = (th^2/2 + cos th - 1)/th^4;
// k3 = (2 th - 3 sin th + th cos th)/(2 th^5);  b = (1 - (th/2)cot(th/2))/th^2.
template <typename T>
struct JacCoef {
  T c1, k2, k3, b;
};

// float: one branch-free Horner polynomial per coefficient in t = theta^2,
// valid on the whole range theta in [0, pi] that qlog produces (truncation
// < 1.4e-7 relative at theta = pi, checked against 40-digit arithmetic);
// no divisions, no sin/cos, and no warp divergence between small- and
// large-angle lanes.  b has radius of convergence 2 pi, hence 13 terms.
__device__ __forceinline__ JacCoef<float> jac_coefs_t(float t) {
  JacCoef<float> k;
  k.c1 = 0.16666666666666666f + t * (-0.0083333333333333332f + t * (0.00019841269841269841f +
         t * (-2.7557319223985893e-06f + t * (2.505210838544172e-08f + t * (-1.6059043836821613e-10f +
         t * (7.6471637318198164e-13f + t * (-2.8114572543455206e-15f + t * 8.2206352466243295e-18f)))))));
  k.k2 = 0.041666666666666664f + t * (-0.0013888888888888889f + t * (2.4801587301587302e-05f +
         t * (-2.7557319223985888e-07f + t * (2.08767569878681e-09f + t * (-1.1470745597729725e-11f +
         t * (4.7794773323873853e-14f + t * (-1.5619206968586225e-16f + t * 4.1103176233121648e-19f)))))));
  k.k3 = 0.0083333333333333332f + t * (-0.00039682539682539683f + t * (8.2671957671957678e-06f +
         t * (-1.0020843354176688e-07f + t * (8.0295219184108074e-10f + t * (-4.5882982390918896e-12f +
         t * (1.9680200780418645e-14f + t * (-6.5765081972994636e-17f + t * 1.7615646957052136e-19f)))))));
  k.b = 0.083333333333333329f + t * (0.0013888888888888889f + t * (3.3068783068783071e-05f +
        t * (8.2671957671957675e-07f + t * (2.08767569878681e-08f + t * (5.2841901386874932e-10f +
        t * (1.3382536530684679e-11f + t * (3.3896802963225827e-13f + t * (8.5860620562778452e-15f +
        t * (2.1748686985580619e-16f + t * (5.5090028283602295e-18f + t * (1.3954464685812522e-19f +
        t * 3.5347070396294673e-21f)))))))))));
  return k;
}

// double: 6-term series below 0.03 rad (truncation < 1e-20), closed forms above.
__device__ __forceinline__ JacCoef<double> jac_coefs_t(double t) {
  const double th = sqrt(t);
  JacCoef<double> k;
  if (th < LieConst<double>::series_below) {
    k.c1 = 1.0 / 6.0 + t * (-1.0 / 120.0 + t * (1.0 / 5040.0 + t * (-1.0 / 362880.0 +
           t * (1.0 / 39916800.0 + t * (-1.0 / 6227020800.0)))));
    k.k2 = 1.0 / 24.0 + t * (-1.0 / 720.0 + t * (1.0 / 40320.0 + t * (-1.0 / 3628800.0 +
           t * (1.0 / 479001600.0 + t * (-1.0 / 87178291200.0)))));
    k.k3 = 1.0 / 120.0 + t * (-1.0 / 2520.0 + t * (1.0 / 120960.0 + t * (-1.0 / 9979200.0 +
           t * (1.0 / 1245404160.0 + t * (-1.0 / 217945728000.0)))));
    k.b = 1.0 / 12.0 + t * (1.0 / 720.0 + t * (1.0 / 30240.0 + t * (1.0 / 1209600.0 +
          t * (1.0 / 47900160.0 + t * (691.0 / 1307674368000.0)))));
  } else {
    double sn, cs;
    sincos(th, &sn, &cs);
    const double t2 = t * t;
    k.c1 = (th - sn) / (t * th);
    k.k2 = (0.5 * t + cs - 1.0) / t2;
    k.k3 = (2.0 * th - 3.0 * sn + th * cs) / (2.0 * t2 * th);
    const double h = 0.5 * th;
    k.b = (1.0 - h / tan(h)) / t;
  }
  return k;
}

// ---- SE(3) log as a translation-first twist (liegroups.py:203-207) -------
// v = Jl^-1(phi) t = t - phi x t / 2 + b phi x (phi x t).
template <typename T>
struct Twist {
  vec3<T> v, phi;
  T theta2;  // |phi|^2
  JacCoef<T> k;
};

template <typename T>
__device__ __forceinline__ Twist<T> se3_log(const quat<T>& q, const vec3<T>& t) {
  Twist<T> xi;
  xi.phi = qlog(q);
  xi.theta2 = dot(xi.phi, xi.phi);
  xi.k = jac_coefs_t(xi.theta2);
  const vec3<T> a = cross(xi.phi, t);
  const vec3<T> b2 = cross(xi.phi, a);
  xi.v = {t.x - T(0.5) * a.x + xi.k.b * b2.x, t.y - T(0.5) * a.y + xi.k.b * b2.y,
          t.z - T(0.5) * a.z + xi.k.b * b2.z};
  return xi;
}

// ---- Jr^-1(xi) = Jl^-1(-xi) = [[A, Bm], [0, A]] (liegroups.py:238-252) ----
// With rho = -v, ph = -phi, d = ph.rho:
//   A  = (1 - b th^2) I - [ph]x / 2 + b ph ph^T           (so3 Jl^-1)
//   Q  = [s]x + c1 (rho ph^T + ph rho^T) - 2 k3 d ph ph^T + (2 k3 d th^2 - 2 c1 d) I,
//        s = (1/2 - k2 th^2) rho + (2 k2 - c1) d ph        (Barfoot's Q, expanded
//        with [a]x[b]x = b a^T - (a.b) I; equals liegroups.py:230-235)
//   Bm = -A Q A.
template <typename T>
struct JrInv {
  mat3<T> A, B;
};

template <typename T>
__device__ __forceinline__ JrInv<T> se3_jr_inv(const Twist<T>& xi) {
  const vec3<T> rho{-xi.v.x, -xi.v.y, -xi.v.z};
  const vec3<T> ph{-xi.phi.x, -xi.phi.y, -xi.phi.z};
  const T t = xi.theta2;
  const T b = xi.k.b, c1 = xi.k.c1, k2 = xi.k.k2, k3 = xi.k.k3;
  const T d = dot(ph, rho);
  JrInv<T> J;
  const T diag = T(1) - b * t;
  const T px[3] = {ph.x, ph.y, ph.z};
  const T rx[3] = {rho.x, rho.y, rho.z};
  // A
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) J.A.m[i][j] = b * px[i] * px[j] + (i == j ? diag : T(0));
  J.A.m[0][1] += T(0.5) * ph.z;
  J.A.m[0][2] -= T(0.5) * ph.y;
  J.A.m[1][0] -= T(0.5) * ph.z;
  J.A.m[1][2] += T(0.5) * ph.x;
  J.A.m[2][0] += T(0.5) * ph.y;
  J.A.m[2][1] -= T(0.5) * ph.x;
  // Q
  const T a1 = T(0.5) - k2 * t, a2 = (T(2) * k2 - c1) * d;
  const vec3<T> s{a1 * rho.x + a2 * ph.x, a1 * rho.y + a2 * ph.y, a1 * rho.z + a2 * ph.z};
  const T e = T(-2) * k3 * d;
  const T qd = T(2) * k3 * d * t - T(2) * c1 * d;
  mat3<T> Q;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      Q.m[i][j] = c1 * (rx[i] * px[j] + px[i] * rx[j]) + e * px[i] * px[j] + (i == j ? qd : T(0));
  Q.m[0][1] -= s.z;
  Q.m[0][2] += s.y;
  Q.m[1][0] += s.z;
  Q.m[1][2] -= s.x;
  Q.m[2][0] -= s.y;
  Q.m[2][1] += s.x;
  // B = -A Q A
  mat3<T> QA;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      QA.m[i][j] = Q.m[i][0] * J.A.m[0][j] + Q.m[i][1] * J.A.m[1][j] + Q.m[i][2] * J.A.m[2][j];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      J.B.m[i][j] = -(J.A.m[i][0] * QA.m[0][j] + J.A.m[i][1] * QA.m[1][j] + J.A.m[i][2] * QA.m[2][j]);
  return J;
}

}  // namespace kop
