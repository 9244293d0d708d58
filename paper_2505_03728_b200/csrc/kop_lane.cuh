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

// ---------------------------------------------------------------------------
// Pose residual (6 weighted rows) and, if JAC, its weighted Jacobian rows.
// ID: the chain's moving joints are exactly the actuated joints in order with
// unit multipliers (qcol[k] == k), so columns need no scatter.
// ---------------------------------------------------------------------------
template <typename T, int NQ, int K, bool ID, bool JAC>
__device__ __forceinline__ void pose_rows(const ChainParams<T, K>& C, const CostParams<T, NQ>& W,
                                          const TargetInv<T>& tg, const T (&q)[NQ], T (&r)[6],
                                          T (&J)[6][NQ]) {
  quat<T> pq{T(1), T(0), T(0), T(0)};
  vec3<T> pp{T(0), T(0), T(0)};
  vec3<T> anc[K], ax[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (ID || k < C.k) {
      const quat<T> tq{C.tq[k][0], C.tq[k][1], C.tq[k][2], C.tq[k][3]};
      const vec3<T> tp{C.tp[k][0], C.tp[k][1], C.tp[k][2]};
      quat<T> fq;
      vec3<T> fp;
      if (k == 0) {  // the root frame is the identity (robot.py:418-419)
        fq = tq;
        fp = tp;
      } else {
        fq = qmul(pq, tq);
        const vec3<T> o = qrot(pq, tp);
        fp = {pp.x + o.x, pp.y + o.y, pp.z + o.z};
      }
      const vec3<T> z = qzaxis(fq);
      if (JAC) {
        anc[k] = fp;
        ax[k] = z;
      }
      const T th = ID ? q[k] : pick(q, C.qcol[k]) * C.mult[k] + C.offset[k];
      if (C.prismatic[k]) {
        pq = fq;
        pp = {fp.x + th * z.x, fp.y + th * z.y, fp.z + th * z.z};
      } else {
        T s, c;
        sincos_t(T(0.5) * th, &s, &c);
        pq = qmul_z(fq, c, s);
        pp = fp;
      }
    }
  }
  // end-effector frame
  const quat<T> eq = qmul(pq, quat<T>{C.eq[0], C.eq[1], C.eq[2], C.eq[3]});
  const vec3<T> eo = qrot(pq, vec3<T>{C.ep[0], C.ep[1], C.ep[2]});
  const vec3<T> ep{pp.x + eo.x, pp.y + eo.y, pp.z + eo.z};
  // pose error T_t^-1 * FK  (beam.py:119-121)
  const quat<T> e_q = qmul(tg.q, eq);
  const vec3<T> et = qrot(tg.q, ep);
  const vec3<T> e_t{tg.t.x + et.x, tg.t.y + et.y, tg.t.z + et.z};
  const Twist<T> xi = se3_log(e_q, e_t);
  r[0] = W.w_pos * xi.v.x;
  r[1] = W.w_pos * xi.v.y;
  r[2] = W.w_pos * xi.v.z;
  r[3] = W.w_ori * xi.phi.x;
  r[4] = W.w_ori * xi.phi.y;
  r[5] = W.w_ori * xi.phi.z;
  if (!JAC) return;

  // J_pose = diag(w) Jr^-1(xi) [R^T J_lin; R^T J_ang]   (beam.py:142-156)
  JrInv<T> jr = se3_jr_inv(xi);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      jr.B.m[i][j] *= W.w_pos;
    }
  mat3<T> At, Ab;
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      At.m[i][j] = W.w_pos * jr.A.m[i][j];
      Ab.m[i][j] = W.w_ori * jr.A.m[i][j];
    }
  const mat3<T> R = qmat(eq);
  if (!ID) {
#pragma unroll
    for (int m = 0; m < 6; ++m)
#pragma unroll
      for (int c = 0; c < NQ; ++c) J[m][c] = T(0);
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (ID || k < C.k) {
      const vec3<T> ab = mulT(R, ax[k]);
      vec3<T> lin, ang;
      if (C.prismatic[k]) {
        lin = ab;
        ang = {T(0), T(0), T(0)};
      } else {
        const vec3<T> db = mulT(R, vec3<T>{ep.x - anc[k].x, ep.y - anc[k].y, ep.z - anc[k].z});
        lin = cross(ab, db);
        ang = ab;
      }
      const vec3<T> t1 = mul(At, lin), t2 = mul(jr.B, ang), b1 = mul(Ab, ang);
      const T col[6] = {t1.x + t2.x, t1.y + t2.y, t1.z + t2.z, b1.x, b1.y, b1.z};
      if (ID) {
#pragma unroll
        for (int m = 0; m < 6; ++m) J[m][k] = col[m];
      } else {
        const int qc = C.qcol[k];
        const T mu = C.mult[k];
#pragma unroll
        for (int c = 0; c < NQ; ++c)
          if (qc == c) {
#pragma unroll
            for (int m = 0; m < 6; ++m) J[m][c] += mu * col[m];
          }
      }
    }
  }
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

// Cost only (candidate evaluation in the reference-structured step).
template <typename T, int NQ, int K, bool ID>
__device__ __forceinline__ T lane_cost(const ChainParams<T, K>& C, const CostParams<T, NQ>& W,
                                       const TargetInv<T>& tg, const T (&q)[NQ]) {
  T r[6], J[6][NQ];
  pose_rows<T, NQ, K, ID, false>(C, W, tg, q, r, J);
  T rl[NQ], gl[NQ], rr[NQ];
  diag_rows(W, q, rl, gl, rr);
  T c = T(0);
#pragma unroll
  for (int m = 0; m < 6; ++m) c += r[m] * r[m];
#pragma unroll
  for (int i = 0; i < NQ; ++i) c += rl[i] * rl[i];
#pragma unroll
  for (int i = 0; i < NQ; ++i) c += rr[i] * rr[i];
  return c;
}

// Cost plus normal equations A = J^T J (packed lower), g = J^T r.
template <typename T, int NQ, int K, bool ID>
__device__ __forceinline__ T lane_normal(const ChainParams<T, K>& C, const CostParams<T, NQ>& W,
                                         const TargetInv<T>& tg, const T (&q)[NQ],
                                         T (&A)[Tri<NQ>::size], T (&g)[NQ]) {
  T r[6], J[6][NQ];
  pose_rows<T, NQ, K, ID, true>(C, W, tg, q, r, J);
  T rl[NQ], gl[NQ], rr[NQ];
  diag_rows(W, q, rl, gl, rr);
  T c = T(0);
#pragma unroll
  for (int m = 0; m < 6; ++m) c += r[m] * r[m];
#pragma unroll
  for (int i = 0; i < NQ; ++i) c += rl[i] * rl[i];
#pragma unroll
  for (int i = 0; i < NQ; ++i) c += rr[i] * rr[i];
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
#pragma unroll
    for (int j = 0; j <= i; ++j) {
      T a = T(0);
#pragma unroll
      for (int m = 0; m < 6; ++m) a += J[m][i] * J[m][j];
      A[Tri<NQ>::at(i, j)] = a;
    }
    A[Tri<NQ>::at(i, i)] += gl[i] * gl[i] + W.w_rest * W.w_rest;
    T s = T(0);
#pragma unroll
    for (int m = 0; m < 6; ++m) s += J[m][i] * r[m];
    g[i] = s + gl[i] * rl[i] + W.w_rest * rr[i];
  }
  return c;
}

// delta = -(A + lam diag(max(diag A, 1e-8)))^-1 g by an in-register Cholesky.
// Returns false if a pivot is not positive / finite (the reference's
// LinAlgError, beam.py:207-213, handled per lane -- see DESIGN.md).
template <typename T, int NQ>
__device__ __forceinline__ bool damped_solve(const T (&A)[Tri<NQ>::size], const T (&g)[NQ], T lam,
                                             T (&delta)[NQ]) {
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
    for (int k = 0; k < j; ++k) s -= L[Tri<NQ>::at(j, k)] * L[Tri<NQ>::at(j, k)];
    ok = ok && (s > T(0)) && finite_t(s);
    const T inv = rsqrt_t(s);
    dinv[j] = inv;
#pragma unroll
    for (int i = j + 1; i < NQ; ++i) {
      T v = L[Tri<NQ>::at(i, j)];
#pragma unroll
      for (int k = 0; k < j; ++k) v -= L[Tri<NQ>::at(i, k)] * L[Tri<NQ>::at(j, k)];
      L[Tri<NQ>::at(i, j)] = v * inv;
    }
  }
  T y[NQ];
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    T v = -g[i];
#pragma unroll
    for (int k = 0; k < i; ++k) v -= L[Tri<NQ>::at(i, k)] * y[k];
    y[i] = v * dinv[i];
  }
#pragma unroll
  for (int i = NQ - 1; i >= 0; --i) {
    T v = y[i];
#pragma unroll
    for (int k = i + 1; k < NQ; ++k) v -= L[Tri<NQ>::at(k, i)] * delta[k];
    delta[i] = v * dinv[i];
  }
  return ok;
}

// Per-lane LM state.  A/g are the normal equations AT q (fused mode keeps
// them from the accepted candidate's evaluation instead of recomputing FK).
template <typename T, int NQ>
struct LaneState {
  T q[NQ];
  T A[Tri<NQ>::size];
  T g[NQ];
  T lam, cost;
};

template <typename T>
__device__ __forceinline__ T inf_t() { return T(INFINITY); }

// One LM proposal (beam.py:201-239), fused form: the candidate's evaluation
// also produces its normal equations, so an accepted step needs no second FK
// at the start of the next step.  Identical accept/reject semantics:
// accept iff finite and cost' < cost; lam /3 (>= 1e-12) or x10 (<= 1e10).
template <typename T, int NQ, int K, bool ID>
__device__ __forceinline__ void lm_step(const ChainParams<T, K>& C, const CostParams<T, NQ>& W,
                                        const TargetInv<T>& tg, LaneState<T, NQ>& s) {
  T d[NQ];
  const bool ok = damped_solve<T, NQ>(s.A, s.g, s.lam, d);
  T qn[NQ];
#pragma unroll
  for (int i = 0; i < NQ; ++i) qn[i] = s.q[i] + (ok ? d[i] : T(0));
  T An[Tri<NQ>::size], gn[NQ];
  T cn = lane_normal<T, NQ, K, ID>(C, W, tg, qn, An, gn);
  if (!finite_t(cn)) cn = inf_t<T>();
  const bool acc = ok && (cn < s.cost);
  if (acc) {
#pragma unroll
    for (int i = 0; i < NQ; ++i) s.q[i] = qn[i];
#pragma unroll
    for (int i = 0; i < Tri<NQ>::size; ++i) s.A[i] = An[i];
#pragma unroll
    for (int i = 0; i < NQ; ++i) s.g[i] = gn[i];
    s.cost = cn;
    s.lam = tmax(s.lam * T(BeamConsts::damping_down), T(BeamConsts::damping_min));
  } else {
    s.lam = tmin(s.lam * T(BeamConsts::damping_up), T(BeamConsts::damping_max));
  }
}

// Reference-structured step (two FK per step, beam.py:202 + :224): kept for
// A/B measurement of the fused form.
template <typename T, int NQ, int K, bool ID>
__device__ __forceinline__ void lm_step_twopass(const ChainParams<T, K>& C,
                                                const CostParams<T, NQ>& W,
                                                const TargetInv<T>& tg, LaneState<T, NQ>& s) {
  T A[Tri<NQ>::size], g[NQ];
  lane_normal<T, NQ, K, ID>(C, W, tg, s.q, A, g);
  T d[NQ];
  const bool ok = damped_solve<T, NQ>(A, g, s.lam, d);
  T qn[NQ];
#pragma unroll
  for (int i = 0; i < NQ; ++i) qn[i] = s.q[i] + (ok ? d[i] : T(0));
  T cn = lane_cost<T, NQ, K, ID>(C, W, tg, qn);
  if (!finite_t(cn)) cn = inf_t<T>();
  const bool acc = ok && (cn < s.cost);
  if (acc) {
#pragma unroll
    for (int i = 0; i < NQ; ++i) s.q[i] = qn[i];
    s.cost = cn;
    s.lam = tmax(s.lam * T(BeamConsts::damping_down), T(BeamConsts::damping_min));
  } else {
    s.lam = tmin(s.lam * T(BeamConsts::damping_up), T(BeamConsts::damping_max));
  }
}

// (cost, index) ordering of np.argsort(kind="stable") with NaN last.
template <typename T>
__device__ __forceinline__ bool rank_less(T a, int ia, T b, int ib) {
  const bool na = !(a == a), nb = !(b == b);
  if (na || nb) return (!na && nb) || (na && nb && ia < ib);
  return a < b || (a == b && ia < ib);
}

}  // namespace kop
