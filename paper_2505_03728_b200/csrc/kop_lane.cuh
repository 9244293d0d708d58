// One IK lane, entirely in registers: FK over the compiled chain, weighted
// residual stack, analytic Jacobian, normal equations, damped Cholesky solve
// and the per-lane LM accept/reject -- the body of beam.py:114-240 for a
// single lane, with the lane batch mapped onto CUDA threads.
//
// Residual stack per lane (beam.py:95-100, 114-131), weighted:
//   rows 0-2  w_pos * v      rows 3-5  w_ori * phi     (xi = log(T_t^-1 FK(q)))
//   rows 6..  w_lim * (max(0, q-u) + max(0, l-q))      rows 6+n..  w_rest * (q - rest)
// The limit and rest rows are diagonal in the Jacobian (beam.py:158-166), so
// only the 6 pose rows are dense: J^T J = Jp^T Jp + diag(...), which is what
// the code forms (168 FMAs for n = 7 instead of a dense 20x7 product).
#pragma once

#include "kop_chain.h"
#include "kop_lie.cuh"

namespace kop {

template <int N>
struct Tri {
  static constexpr int size = N * (N + 1) / 2;
  __host__ __device__ static constexpr int at(int i, int j) { return i * (i + 1) / 2 + j; }  // i >= j
};

template <typename T>
struct TargetInv {
  quat<T> q;
  vec3<T> t;
};

// Inverse of a canonical target pose (Transform3.inverse, liegroups.py:388-390),
// evaluated in double and canonicalised like Rotation3 (liegroups.py:33-45).
__device__ __forceinline__ void target_inverse(const double* __restrict__ pose, double out[7]) {
  double w = pose[0], x = -pose[1], y = -pose[2], z = -pose[3];
  const double nrm = sqrt(w * w + x * x + y * y + z * z);
  w /= nrm; x /= nrm; y /= nrm; z /= nrm;
  double sign = w < 0.0 ? -1.0 : 1.0;
  if (w == 0.0) {
    const double ax = fabs(x), ay = fabs(y), az = fabs(z);
    const double lead = (ax >= ay && ax >= az) ? x : (ay >= az ? y : z);
    sign = lead < 0.0 ? -1.0 : 1.0;
  }
  const quat<double> q{w * sign, x * sign, y * sign, z * sign};
  const vec3<double> t = qrot(q, vec3<double>{pose[4], pose[5], pose[6]});
  out[0] = q.w; out[1] = q.x; out[2] = q.y; out[3] = q.z;
  out[4] = -t.x; out[5] = -t.y; out[6] = -t.z;
}

// Per-lane target inverse.  double: the exact canonical inverse above.
// float: q^-1 = conj(q) renormalised with rsqrtf and t^-1 = -R(q^-1) t, all in
// float (the target is already canonical, so the canonical sign flip is the
// identity except at w == 0, handled by the same lead-component rule).
template <typename T>
__device__ __forceinline__ TargetInv<T> target_inverse_t(const double* __restrict__ pose);

template <>
__device__ __forceinline__ TargetInv<double> target_inverse_t<double>(const double* __restrict__ pose) {
  double v[7];
  target_inverse(pose, v);
  return {{v[0], v[1], v[2], v[3]}, {v[4], v[5], v[6]}};
}

template <>
__device__ __forceinline__ TargetInv<float> target_inverse_t<float>(const double* __restrict__ pose) {
  float w = float(pose[0]), x = -float(pose[1]), y = -float(pose[2]), z = -float(pose[3]);
  const float rn = rsqrtf(w * w + x * x + y * y + z * z);
  w *= rn; x *= rn; y *= rn; z *= rn;
  float sign = w < 0.f ? -1.f : 1.f;
  if (w == 0.f) {
    const float ax = fabsf(x), ay = fabsf(y), az = fabsf(z);
    const float lead = (ax >= ay && ax >= az) ? x : (ay >= az ? y : z);
    sign = lead < 0.f ? -1.f : 1.f;
  }
  const quat<float> q{w * sign, x * sign, y * sign, z * sign};
  const vec3<float> t = qrot(q, vec3<float>{float(pose[4]), float(pose[5]), float(pose[6])});
  return {q, {-t.x, -t.y, -t.z}};
}

template <typename T>
__device__ __forceinline__ TargetInv<T> to_target(const double v[7]) {
  return {{T(v[0]), T(v[1]), T(v[2]), T(v[3])}, {T(v[4]), T(v[5]), T(v[6])}};
}

template <typename T>
__device__ __forceinline__ TargetInv<T> load_target_inv(const double* __restrict__ p) {
  return {{T(p[0]), T(p[1]), T(p[2]), T(p[3])}, {T(p[4]), T(p[5]), T(p[6])}};
}

// q[idx] for a runtime idx without dynamic register indexing (select chain).
template <typename T, int NQ>
__device__ __forceinline__ T pick(const T (&q)[NQ], int idx) {
  T v = q[0];
#pragma unroll
  for (int c = 1; c < NQ; ++c) v = (idx == c) ? q[c] : v;
  return v;
}

// Compile-time lane configuration: scalar type, actuated joints NQ, chain
// joints K, identity column map, and the optional SE(2) mobile base (three
// extra tangent dimensions after the joints, beam.py:98-102).
template <typename T_, int NQ_, int K_, bool ID_, bool BASE_>
struct Cfg {
  using T = T_;
  static constexpr int NQ = NQ_, K = K_, ND = NQ_ + (BASE_ ? 3 : 0);
  static constexpr bool ID = ID_, BASE = BASE_;
};

// ---------------------------------------------------------------------------
// Pose residual (6 weighted rows) and, if JAC, its weighted Jacobian rows
// over the ND tangent columns.
// ID: the chain's moving joints are exactly the actuated joints in order with
// unit multipliers (qcol[k] == k), so columns need no scatter.
//
// Backward pass (kop_chain.h): S = child_k -> EE starts at the EE offset and
// is pre-multiplied by M_k = Rz(theta_k) (or Tz) and the joint frame O_k for
// k = K-1 .. 0, ending at the world EE pose.  Before composing joint k, S is
// child_k -> EE, where joint k's axis is +z through the origin, so its body
// (EE-frame) Jacobian column is  ang = R_S^T z = row 2 of R_S,
// lin = R_S^T (z x p_S) = -p_y row0 + p_x row1  -- the same columns as
// beam.py:142-146 (R^T J_geom) without any per-joint world state.
//
// Mobile base (beam.py:104-112, 167-179): the SE(2) base B = (Rz(a), (x,y,0))
// left-multiplies the arm; its right-multiplicative tangent (vx, vy, w) acts
// like a prismatic-x, prismatic-y and revolute-z joint at the arm root, so its
// columns Jr^-1 Ad(FK^-1) E_se2 are read off S_0 exactly like joint columns.
// ---------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ quat<T> zmul_left(T c, T s, const quat<T>& b) {  // (c,0,0,s) * b
  return {c * b.w - s * b.z, c * b.x - s * b.y, c * b.y + s * b.x, c * b.z + s * b.w};
}

// body columns of S = (sq, sp) for a revolute-z / prismatic-z joint at S's origin
template <typename T>
__device__ __forceinline__ void s_columns(const quat<T>& sq, const vec3<T>& sp, T (&rev)[6], T (&px)[3],
                                          T (&py)[3], T (&pz)[3]) {
  const T x2 = sq.x + sq.x, y2 = sq.y + sq.y, z2 = sq.z + sq.z;
  const T r00 = T(1) - (sq.y * y2 + sq.z * z2), r01 = sq.x * y2 - sq.w * z2, r02 = sq.x * z2 + sq.w * y2;
  const T r10 = sq.x * y2 + sq.w * z2, r11 = T(1) - (sq.x * x2 + sq.z * z2), r12 = sq.y * z2 - sq.w * x2;
  const T r20 = sq.x * z2 - sq.w * y2, r21 = sq.y * z2 + sq.w * x2, r22 = T(1) - (sq.x * x2 + sq.y * y2);
  rev[0] = sp.x * r10 - sp.y * r00;
  rev[1] = sp.x * r11 - sp.y * r01;
  rev[2] = sp.x * r12 - sp.y * r02;
  rev[3] = r20; rev[4] = r21; rev[5] = r22;
  px[0] = r00; px[1] = r01; px[2] = r02;
  py[0] = r10; py[1] = r11; py[2] = r12;
  pz[0] = r20; pz[1] = r21; pz[2] = r22;
}

// Pose residual of the (base-composed) world EE pose (sq, sp) and, if JAC,
// the weighted pose Jacobian J = diag(w) Jr^-1(xi) [lin; ang] from the
// body-frame columns `col` (chain joints, then the 3 base columns).
template <class G, bool JAC>
__device__ __forceinline__ void pose_finish(const ChainParams<typename G::T, G::K>& C,
                                            const CostParams<typename G::T, G::NQ>& W,
                                            const TargetInv<typename G::T>& tg, const quat<typename G::T>& sq,
                                            const vec3<typename G::T>& sp,
                                            const typename G::T (&col)[G::K + (G::BASE ? 3 : 0)][6],
                                            typename G::T (&r)[6], typename G::T (&J)[6][G::ND]) {
  using T = typename G::T;
  constexpr int K = G::K, NQ = G::NQ;
  constexpr bool ID = G::ID;
  // pose error T_t^-1 * (B) * FK  (beam.py:119-121)
  const quat<T> e_q = qmul(tg.q, sq);
  const vec3<T> et = qrot(tg.q, sp);
  const vec3<T> e_t{tg.t.x + et.x, tg.t.y + et.y, tg.t.z + et.z};
  const Twist<T> xi = se3_log(e_q, e_t);
  r[0] = W.w_pos * xi.v.x;
  r[1] = W.w_pos * xi.v.y;
  r[2] = W.w_pos * xi.v.z;
  r[3] = W.w_ori * xi.phi.x;
  r[4] = W.w_ori * xi.phi.y;
  r[5] = W.w_ori * xi.phi.z;
  if (!JAC) return;

  // J_pose = diag(w) Jr^-1(xi) [lin; ang]   (beam.py:142-156, 170)
  const JrInv<T> jr = se3_jr_inv(xi);
  mat3<T> At, Bt, Ab;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      At.m[i][j] = W.w_pos * jr.A.m[i][j];
      Bt.m[i][j] = W.w_pos * jr.B.m[i][j];
      Ab.m[i][j] = W.w_ori * jr.A.m[i][j];
    }
  if (!ID) {
#pragma unroll
    for (int m = 0; m < 6; ++m)
#pragma unroll
      for (int c = 0; c < NQ; ++c) J[m][c] = T(0);
  }
#pragma unroll
  for (int k = 0; k < K + (G::BASE ? 3 : 0); ++k) {
    if (ID || k >= K || k < C.k) {
      const vec3<T> lin{col[k][0], col[k][1], col[k][2]}, ang{col[k][3], col[k][4], col[k][5]};
      const vec3<T> t1 = mul(At, lin), t2 = mul(Bt, ang), b1 = mul(Ab, ang);
      const T cj[6] = {t1.x + t2.x, t1.y + t2.y, t1.z + t2.z, b1.x, b1.y, b1.z};
      if (ID || k >= K) {
        const int c = k >= K ? NQ + (k - K) : k;
#pragma unroll
        for (int m = 0; m < 6; ++m) J[m][c] = cj[m];
      } else {
        const int qc = C.qcol[k];
        const T mu = C.mult[k];
#pragma unroll
        for (int c = 0; c < NQ; ++c)
          if (qc == c) {
#pragma unroll
            for (int m = 0; m < 6; ++m) J[m][c] += mu * cj[m];
          }
      }
    }
  }
}

// Target-independent part of a lane evaluation: the backward pass over the
// compiled chain at q, giving the arm's EE pose S_0 = (sq, sp) and (JAC) the
// body-frame Jacobian columns.  A function of q alone -- IK-Beam evaluates it
// once per seed for the start state (k_seed_frames).
template <class G, bool JAC>
__device__ __forceinline__ void pose_backward(const ChainParams<typename G::T, G::K>& C,
                                              const typename G::T (&q)[G::NQ], quat<typename G::T>& sq_out,
                                              vec3<typename G::T>& sp_out,
                                              typename G::T (&col)[G::K + (G::BASE ? 3 : 0)][6]) {
  using T = typename G::T;
  constexpr int K = G::K, NQ = G::NQ, ND = G::ND;
  constexpr bool ID = G::ID;
  quat<T> sq{C.eq[0], C.eq[1], C.eq[2], C.eq[3]};
  vec3<T> sp{C.ep[0], C.ep[1], C.ep[2]};
#pragma unroll
  for (int k = K - 1; k >= 0; --k) {
    if (ID || k < C.k) {
      const bool pri = !ID && C.prismatic[k];
      if (JAC) {
        T rev[6], px[3], py[3], pz[3];
        s_columns(sq, sp, rev, px, py, pz);
        if (pri) {
          col[k][0] = pz[0]; col[k][1] = pz[1]; col[k][2] = pz[2];
          col[k][3] = T(0); col[k][4] = T(0); col[k][5] = T(0);
        } else {
#pragma unroll
          for (int m = 0; m < 6; ++m) col[k][m] = rev[m];
        }
      }
      const T th = ID ? q[k] : pick(q, C.qcol[k]) * C.mult[k] + C.offset[k];
      if (pri) {
        sp.z += th;
      } else {
        T s, c;
        sincos_t(T(0.5) * th, &s, &c);
        sq = zmul_left(c, s, sq);
        const T c2 = c * c - s * s, s2 = T(2) * c * s;
        sp = {c2 * sp.x - s2 * sp.y, s2 * sp.x + c2 * sp.y, sp.z};
      }
      sq = qmul(quat<T>{C.tq[k][0], C.tq[k][1], C.tq[k][2], C.tq[k][3]}, sq);
      sp = {C.tp[k][0] + (C.tr[k][0][0] * sp.x + C.tr[k][0][1] * sp.y + C.tr[k][0][2] * sp.z),
            C.tp[k][1] + (C.tr[k][1][0] * sp.x + C.tr[k][1][1] * sp.y + C.tr[k][1][2] * sp.z),
            C.tp[k][2] + (C.tr[k][2][0] * sp.x + C.tr[k][2][1] * sp.y + C.tr[k][2][2] * sp.z)};
    }
  }
  sq_out = sq;
  sp_out = sp;
}

template <class G, bool JAC>
__device__ __forceinline__ void pose_rows(const ChainParams<typename G::T, G::K>& C,
                                          const CostParams<typename G::T, G::NQ>& W,
                                          const TargetInv<typename G::T>& tg, const typename G::T (&q)[G::NQ],
                                          const typename G::T (&base)[3], typename G::T (&r)[6],
                                          typename G::T (&J)[6][G::ND]) {
  using T = typename G::T;
  constexpr int K = G::K;
  quat<T> sq;
  vec3<T> sp;
  T col[K + (G::BASE ? 3 : 0)][6];
  pose_backward<G, JAC>(C, q, sq, sp, col);
  if (G::BASE) {
    if (JAC) {  // base tangent (vx, vy, w): prismatic x, prismatic y, revolute z at the arm root
      T rev[6], px[3], py[3], pz[3];
      s_columns(sq, sp, rev, px, py, pz);
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        col[K][m] = px[m]; col[K][3 + m] = T(0);
        col[K + 1][m] = py[m]; col[K + 1][3 + m] = T(0);
      }
#pragma unroll
      for (int m = 0; m < 6; ++m) col[K + 2][m] = rev[m];
    }
    T s, c;  // compose the base: B * S_0 (beam.py:104-112)
    sincos_t(T(0.5) * base[2], &s, &c);
    sq = zmul_left(c, s, sq);
    const T c2 = c * c - s * s, s2 = T(2) * c * s;
    sp = {c2 * sp.x - s2 * sp.y + base[0], s2 * sp.x + c2 * sp.y + base[1], sp.z};
  }
  pose_finish<G, JAC>(C, W, tg, sq, sp, col, r, J);
}

// Diagonal limit / rest rows (beam.py:122-125, 158-166): residuals, J diag.
template <typename T, int NQ>
__device__ __forceinline__ void diag_rows(const CostParams<T, NQ>& W, const T (&q)[NQ], T (&rl)[NQ],
                                          T (&gl)[NQ], T (&rr)[NQ]) {
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    const T above = q[i] - W.upper[i], below = W.lower[i] - q[i];
    rl[i] = W.w_lim * (tmax(T(0), above) + tmax(T(0), below));
    gl[i] = W.w_lim * ((q[i] > W.upper[i] ? T(1) : T(0)) + (q[i] < W.lower[i] ? T(-1) : T(0)));
    rr[i] = W.w_rest * (q[i] - W.rest[i]);
  }
}

// Weighted residual stack, its cost and (JAC) the normal equations
// A = J^T J (packed lower, ND x ND), g = J^T r.  Rows: pose (6, dense), limit
// and rest (diagonal), base regularisation (x, y, a) * w_base whose Jacobian
// [[R(a), 0], [0, 1]] (beam.py:171-178) is orthogonal, so it adds w_base^2 I
// to A and w_base R^T-rotated residuals to g.
template <class G, bool JAC>
__device__ __forceinline__ typename G::T assemble_rows(const CostParams<typename G::T, G::NQ>& W,
                                                       const typename G::T (&q)[G::NQ],
                                                       const typename G::T (&base)[3], const typename G::T (&r)[6],
                                                       const typename G::T (&J)[6][G::ND],
                                                       typename G::T (&A)[Tri<G::ND>::size],
                                                       typename G::T (&g)[G::ND]) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, ND = G::ND;
  T rl[NQ], gl[NQ], rr[NQ];
  diag_rows(W, q, rl, gl, rr);
  T rb[3] = {T(0), T(0), T(0)};
  if (G::BASE) {
    rb[0] = W.w_base * base[0];
    rb[1] = W.w_base * base[1];
    rb[2] = W.w_base * base[2];
  }
  T c = T(0);
#pragma unroll
  for (int m = 0; m < 6; ++m) c += r[m] * r[m];
#pragma unroll
  for (int i = 0; i < NQ; ++i) c += rl[i] * rl[i];
#pragma unroll
  for (int i = 0; i < NQ; ++i) c += rr[i] * rr[i];
  if (G::BASE) c += rb[0] * rb[0] + rb[1] * rb[1] + rb[2] * rb[2];
  if (!JAC) return c;
#pragma unroll
  for (int i = 0; i < ND; ++i) {
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      if (j <= i) {
        T a = T(0);
#pragma unroll
        for (int m = 0; m < 6; ++m) a += J[m][i] * J[m][j];
        A[Tri<ND>::at(i, j)] = a;
      }
    }
    T s = T(0);
#pragma unroll
    for (int m = 0; m < 6; ++m) s += J[m][i] * r[m];
    g[i] = s;
  }
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    A[Tri<ND>::at(i, i)] += gl[i] * gl[i] + W.w_rest * W.w_rest;
    g[i] += gl[i] * rl[i] + W.w_rest * rr[i];
  }
  if (G::BASE) {
    const T wb2 = W.w_base * W.w_base;
    T sa, ca;
    sincos_t(T(0.5) * base[2], &sa, &ca);
    const T cs = ca * ca - sa * sa, sn = T(2) * ca * sa;  // cos a, sin a
#pragma unroll
    for (int i = NQ; i < ND; ++i) A[Tri<ND>::at(i, i)] += wb2;
    g[NQ] += W.w_base * (cs * rb[0] + sn * rb[1]);
    g[NQ + 1] += W.w_base * (-sn * rb[0] + cs * rb[1]);
    g[NQ + 2] += W.w_base * rb[2];
  }
  return c;
}

template <class G, bool JAC>
__device__ __forceinline__ typename G::T lane_eval(const ChainParams<typename G::T, G::K>& C,
                                                   const CostParams<typename G::T, G::NQ>& W,
                                                   const TargetInv<typename G::T>& tg,
                                                   const typename G::T (&q)[G::NQ], const typename G::T (&base)[3],
                                                   typename G::T (&A)[Tri<G::ND>::size],
                                                   typename G::T (&g)[G::ND]) {
  using T = typename G::T;
  T r[6], J[6][G::ND];
  pose_rows<G, JAC>(C, W, tg, q, base, r, J);
  return assemble_rows<G, JAC>(W, q, base, r, J, A, g);
}

// delta = -(A + lam diag(max(diag A, 1e-8)))^-1 g by an in-register Cholesky.
// Returns false if a pivot is not positive / finite (the reference's
// LinAlgError, beam.py:207-213, handled per lane -- see DESIGN.md).
template <typename T, int NQ>
__device__ __forceinline__ bool damped_solve(const T (&A)[Tri<NQ>::size], const T (&g)[NQ], T lam,
                                             T (&delta)[NQ]) {
  // All loops have constant trip counts with the triangular bounds as
  // predicates, so they unroll completely and L stays in registers (nested
  // loops with j-dependent bounds were left rolled and put L in local memory).
  T L[Tri<NQ>::size];
  T dinv[NQ];
  bool ok = true;
#pragma unroll
  for (int i = 0; i < Tri<NQ>::size; ++i) L[i] = A[i];
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    const T d = L[Tri<NQ>::at(i, i)];
    L[Tri<NQ>::at(i, i)] = d + lam * tmax(d, T(BeamConsts::diag_clamp));
  }
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    T s = L[Tri<NQ>::at(j, j)];
#pragma unroll
    for (int k = 0; k < NQ; ++k)
      if (k < j) s -= L[Tri<NQ>::at(j, k)] * L[Tri<NQ>::at(j, k)];
    ok = ok && (s > T(0)) && finite_t(s);
    const T inv = rsqrt_t(s);
    dinv[j] = inv;
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      if (i > j) {
        T v = L[Tri<NQ>::at(i, j)];
#pragma unroll
        for (int k = 0; k < NQ; ++k)
          if (k < j) v -= L[Tri<NQ>::at(i, k)] * L[Tri<NQ>::at(j, k)];
        L[Tri<NQ>::at(i, j)] = v * inv;
      }
    }
  }
  T y[NQ];
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    T v = -g[i];
#pragma unroll
    for (int k = 0; k < NQ; ++k)
      if (k < i) v -= L[Tri<NQ>::at(i, k)] * y[k];
    y[i] = v * dinv[i];
  }
#pragma unroll
  for (int ii = 0; ii < NQ; ++ii) {
    const int i = NQ - 1 - ii;
    T v = y[i];
#pragma unroll
    for (int k = 0; k < NQ; ++k)
      if (k > i) v -= L[Tri<NQ>::at(k, i)] * delta[k];
    delta[i] = v * dinv[i];
  }
  return ok;
}

// Per-lane LM state.  The normal equations AT the current iterate (packed
// lower A, then g) live in shared memory, element e of this lane at
// Ag[e * stride]: the fused step keeps them from the accepted candidate's
// evaluation instead of recomputing FK, and holding them outside the register
// file keeps the lane at <= 128 registers (2 CTAs of 256 threads per SM).
template <class G>
struct LaneState {
  typename G::T q[G::NQ];
  typename G::T base[3];  // (x, y, angle) of the SE(2) base when G::BASE
  typename G::T lam, cost;
  typename G::T* Ag;
  int stride;
};

// STRIDE: the block size when it is a compile-time constant (then every
// shared-memory access is base + immediate), 0 = use s.stride.
template <int STRIDE, class G>
__device__ __forceinline__ void store_normal(const LaneState<G>& s, const typename G::T (&A)[Tri<G::ND>::size],
                                             const typename G::T (&g)[G::ND]) {
  const int st = STRIDE ? STRIDE : s.stride;
#pragma unroll
  for (int i = 0; i < Tri<G::ND>::size; ++i) s.Ag[i * st] = A[i];
#pragma unroll
  for (int i = 0; i < G::ND; ++i) s.Ag[(Tri<G::ND>::size + i) * st] = g[i];
}

template <int STRIDE, class G>
__device__ __forceinline__ void load_normal(const LaneState<G>& s, typename G::T (&A)[Tri<G::ND>::size],
                                            typename G::T (&g)[G::ND]) {
  const int st = STRIDE ? STRIDE : s.stride;
#pragma unroll
  for (int i = 0; i < Tri<G::ND>::size; ++i) A[i] = s.Ag[i * st];
#pragma unroll
  for (int i = 0; i < G::ND; ++i) g[i] = s.Ag[(Tri<G::ND>::size + i) * st];
}

template <typename T>
__device__ __forceinline__ T inf_t() { return T(INFINITY); }

// wrap to (-pi, pi] (liegroups.py:270-273, np.mod semantics)
template <typename T>
__device__ __forceinline__ T wrap_angle_t(T a) {
  const T two_pi = T(6.283185307179586476925286766559);
  const T x = a + T(3.1415926535897932384626433832795);
  T w = x - two_pi * floor(x / two_pi) - T(3.1415926535897932384626433832795);
  return w == -T(3.1415926535897932384626433832795) ? T(3.1415926535897932384626433832795) : w;
}

// SE(2) retraction of the base (beam.py:216-221, liegroups.py:276-287):
// angle' = wrap(a + wrap(w)); xy' = xy + R(a) V(w) v.  float evaluates
// (1 - cos w)/w as 2 sin^2(w/2)/w (the reference form cancels in float).
template <typename T>
__device__ __forceinline__ void base_retract(const T (&b)[3], T vx, T vy, T w, T (&out)[3]) {
  T s, c;
  if (fabs(w) < T(1e-7)) {
    s = T(1) - w * w / T(6);
    c = T(0.5) * w - w * w * w / T(24);
  } else {
    T sw, cw;
    sincos_t(w, &sw, &cw);
    s = sw / w;
    if (sizeof(T) == 4) {
      T sh, ch;
      sincos_t(T(0.5) * w, &sh, &ch);
      c = T(2) * sh * sh / w;
    } else {
      c = (T(1) - cw) / w;
    }
  }
  const T tx = s * vx - c * vy, ty = c * vx + s * vy;
  T sa, ca;
  sincos_t(T(0.5) * b[2], &sa, &ca);
  const T cs = ca * ca - sa * sa, sn = T(2) * ca * sa;
  out[0] = b[0] + (cs * tx - sn * ty);
  out[1] = b[1] + (sn * tx + cs * ty);
  out[2] = wrap_angle_t(b[2] + wrap_angle_t(w));
}

// One LM iteration of a lane, or its start (beam.py:182-196) when mode != 0.
//   mode 0  one proposal (beam.py:201-239), fused form: the candidate's
//           evaluation also produces its normal equations, so an accepted step
//           needs no second FK at the start of the next step.  Same accept /
//           reject semantics: accept iff finite and cost' < cost; lam /3
//           (>= 1e-12) or x10 (<= 1e10).
//   mode 1  start at q: cost and normal equations from one evaluation.
//   mode 2  restart at q keeping the carried cost (survivors after the prune:
//           LaneState.select keeps cost, beam.py:60-68, while r and J are
//           re-derived at q, beam.py:202).
// A single inlined evaluation serves all three (one copy of the ~2K-instruction
// body per kernel keeps the hot loop inside the instruction cache).
// The residual model of a lane: pose + limit + rest (+ base) rows.  Other
// models (collision rows, kop_collision.cuh) provide the same eval().
template <class G>
struct PoseModel {
  using T = typename G::T;
  const ChainParams<T, G::K>& C;
  const CostParams<T, G::NQ>& W;
  TargetInv<T> tg;
  template <bool JAC>
  __device__ __forceinline__ T eval(const T (&q)[G::NQ], const T (&base)[3], T (&A)[Tri<G::ND>::size],
                                    T (&g)[G::ND]) const {
    return lane_eval<G, JAC>(C, W, tg, q, base, A, g);
  }
  // the start evaluation at seed s from its precomputed frame (k_seed_frames,
  // field-major table tab[f * S + s]): only the target-dependent part remains
  __device__ __forceinline__ T eval_seed(const T* __restrict__ tab, int S, int s, const T (&q)[G::NQ],
                                         const T (&base)[3], T (&A)[Tri<G::ND>::size], T (&g)[G::ND]) const {
    static_assert(!G::BASE, "seed frames exclude the mobile base");
    const quat<T> sq{tab[0 * S + s], tab[1 * S + s], tab[2 * S + s], tab[3 * S + s]};
    const vec3<T> sp{tab[4 * S + s], tab[5 * S + s], tab[6 * S + s]};
    T col[G::K][6];
#pragma unroll
    for (int k = 0; k < G::K; ++k)
#pragma unroll
      for (int m = 0; m < 6; ++m) col[k][m] = tab[(7 + 6 * k + m) * S + s];
    T r[6], J[6][G::ND];
    pose_finish<G, true>(C, W, tg, sq, sp, col, r, J);
    return assemble_rows<G, true>(W, q, base, r, J, A, g);
  }
};

// seed frame table size in elements (per seed: EE quaternion, position, 6 K columns)
template <class G>
__host__ __device__ constexpr int seed_frame_fields() { return 7 + 6 * G::K; }

template <class G, int STRIDE, class M>
__device__ __forceinline__ void lm_iter(const M& model, LaneState<G>& s, int mode) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, ND = G::ND;
  // A failed pivot (<= 0, or NaN input) poisons the step with inf / NaN, so the
  // candidate's cost is non-finite and the step is rejected with damping x10
  // -- the outcome of the reference's LinAlgError branch (beam.py:209-213) --
  // without tracking a flag through the factorisation.
  T d[ND];
  if (mode == 0) {
    T A[Tri<ND>::size], g[ND];
    load_normal<STRIDE>(s, A, g);
    (void)damped_solve<T, ND>(A, g, s.lam, d);
  } else {
#pragma unroll
    for (int i = 0; i < ND; ++i) d[i] = T(0);
  }
  T qn[NQ], bn[3];
#pragma unroll
  for (int i = 0; i < NQ; ++i) qn[i] = s.q[i] + d[i];
  if (G::BASE) {
    if (mode == 0) {
      base_retract(s.base, d[NQ], d[NQ + 1], d[NQ + 2], bn);
    } else {
      bn[0] = s.base[0]; bn[1] = s.base[1]; bn[2] = s.base[2];
    }
  }
  T An[Tri<ND>::size], gn[ND];
  const T raw = model.template eval<true>(qn, bn, An, gn);
  const T cn = finite_t(raw) ? raw : inf_t<T>();
  const bool acc = mode != 0 || cn < s.cost;
  if (acc) store_normal<STRIDE>(s, An, gn);  // one store site for start and accept
  if (mode != 0) {
    if (mode == 1) s.cost = raw;  // start_state keeps a non-finite cost as is
    return;
  }
  if (acc) {
#pragma unroll
    for (int i = 0; i < NQ; ++i) s.q[i] = qn[i];
    if (G::BASE) {
      s.base[0] = bn[0]; s.base[1] = bn[1]; s.base[2] = bn[2];
    }
    s.cost = cn;
    s.lam = tmax(s.lam * T(BeamConsts::damping_down), T(BeamConsts::damping_min));
  } else {
    s.lam = tmin(s.lam * T(BeamConsts::damping_up), T(BeamConsts::damping_max));
  }
}

// Sort key of a lane for the stable top-k prune: (cost bits, lane index) as
// one uint64.  Costs are sums of squares, so their IEEE bits (sign cleared)
// order like the values, +inf above every finite cost and NaN (0x7fffffff)
// above +inf -- np.argsort(kind="stable") order with NaN last.
__device__ __forceinline__ unsigned long long prune_key(float c, int idx) {
  uint32_t b = __float_as_uint(c) & 0x7fffffffu;
  if (c != c) b = 0x7fffffffu;
  return ((unsigned long long)b << 32) | (uint32_t)idx;
}
// (cost, index) ordering of np.argsort(kind="stable") with NaN last.
template <typename T>
__device__ __forceinline__ bool rank_less(T a, int ia, T b, int ib) {
  const bool na = !(a == a), nb = !(b == b);
  if (na || nb) return (!na && nb) || (na && nb && ia < ib);
  return a < b || (a == b && ia < ib);
}

}  // namespace kop
