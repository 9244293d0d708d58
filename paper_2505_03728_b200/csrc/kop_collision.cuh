// Collision rows of a lane (config 4): world (sphere link x obstacle) and
// self (link pair) activation rows with their analytic Jacobians, appended to
// the pose / limit / rest stack -- costs.py:423-551 with collision.py:115-269.
//
// Evaluation is a FORWARD pass over the compiled chain (kop_chain.h) that
// leaves, per lane in shared memory, the Pluecker coordinates (a_k, m_k =
// a_k x o_k) of every moving joint axis and the world centres of every
// collision sphere.  With them a collision row needs no per-sphere point
// Jacobian:  for aggregated weights w_s and unit gradients n_s,
//   sum_s w_s n_s . J_point(c_s)[k] = a_k . M - m_k . G,
//   M = sum_s w_s c_s x n_s,  G = sum_s w_s n_s          (revolute k)
//   = a_k . G                                            (prismatic k)
// over the joints k upstream of the sphere's link, i.e. 6 FMAs per joint per
// row instead of a 3 x n Jacobian per sphere.  The pose rows reuse the same
// Pluecker data: body column k = R_ee^T [a_k x p_ee - m_k ; a_k].
#pragma once

#include "kop_lane.cuh"

namespace kop {

constexpr int kMaxSpheres = 32;
constexpr int kMaxObstacles = 16;
constexpr int kMaxSphereLinks = 16;
constexpr int kMaxSelfPairs = 64;
constexpr int kMaxSlots = 10;  // chain slots -1 .. 8

enum ObstacleKind : int32_t { kObSphere = 0, kObCapsule = 1, kObHalfSpace = 2 };

template <typename T>
struct CollisionParams {
  int32_t ns;                   // spheres, sorted by chain slot then model link order
  T sc[kMaxSpheres][3];         // centre in the aligned child frame of its slot (world for slot -1)
  T sr[kMaxSpheres];
  int32_t slot_first[kMaxSlots + 1];  // spheres of slot k: [slot_first[k+1], slot_first[k+2])
  int32_t nl;                   // sphere-bearing links (model order)
  int32_t lfirst[kMaxSphereLinks], lcount[kMaxSphereLinks], lslot[kMaxSphereLinks];
  int32_t no;                   // obstacles
  int32_t okind[kMaxObstacles];
  T oa[kMaxObstacles][3];       // sphere centre | capsule endpoint a | half-space normal
  T ob[kMaxObstacles][3];       // capsule endpoint b
  T orad[kMaxObstacles];        // radius | half-space offset
  int32_t np;                   // self pairs (sphere-link indices)
  int32_t pa[kMaxSelfPairs], pb[kMaxSelfPairs];
  T w_world, eta_world, w_self, eta_self, beta;
  int32_t hard;                 // hard minimum instead of the softmin
  // soft-minimum reach log(count)/beta (0 for the hard minimum) per sphere link
  // and per self pair: the aggregate never lies below dmin - reach, so a row
  // whose dmin - reach clears eta has activation exactly 0 and is skipped
  T lreach[kMaxSphereLinks], preach[kMaxSelfPairs];
};

// scratch layout per lane (stride = block size): a_k, m_k [6 * K] | centres [3 * ns]
template <class G>
__host__ __device__ constexpr int col_scratch_fixed() { return 6 * G::K; }

__device__ __forceinline__ float exp_t(float x) { return __expf(x); }
__device__ __forceinline__ double exp_t(double x) { return exp(x); }
__device__ __forceinline__ float log_t(float x) { return __logf(x); }
__device__ __forceinline__ double log_t(double x) { return log(x); }

// Eq. 1 activation and derivative (collision.py:245-269)
template <typename T>
__device__ __forceinline__ void activation_t(T d, T eta, T& a, T& da) {
  if (d < T(0)) {
    a = -d + T(0.5) * eta;
    da = T(-1);
  } else if (d < eta) {
    const T ie = div_t(T(1), eta);
    a = (T(0.5) * ie) * (eta - d) * (eta - d);
    da = -(eta - d) * ie;
  } else {
    a = T(0);
    da = T(0);
  }
}

// Soft minimum over candidate distances (costs.py:409-420) accumulated in ONE
// pass: the weights z = exp(-beta (d - dmin)) and the NV weighted gradient sums
// are rescaled whenever the running minimum drops, which gives the reference's
// two-pass value.  hard: argmin (first on ties) with weight 1.
template <typename T, int NV>
struct SoftMin {
  T dmin, sumz;
  vec3<T> acc[NV];
  __device__ __forceinline__ SoftMin() : dmin(inf_t<T>()), sumz(T(0)) {
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = {T(0), T(0), T(0)};
  }
  // weight of a candidate at distance d (0: not part of the hard minimum)
  __device__ __forceinline__ T weight(T d, T beta, bool hard) {
    if (hard) {
      if (!(d < dmin)) return T(0);
      dmin = d;
      sumz = T(0);
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] = {T(0), T(0), T(0)};
      return T(1);
    }
    if (d < dmin) {
      const T sc = exp_t(-beta * (dmin - d));  // 0 for the first candidate
      sumz *= sc;
#pragma unroll
      for (int v = 0; v < NV; ++v) acc[v] = {acc[v].x * sc, acc[v].y * sc, acc[v].z * sc};
      dmin = d;
    }
    return exp_t(-beta * (d - dmin));
  }
  __device__ __forceinline__ void add(T z, int v, const vec3<T>& x) {
    acc[v] = {acc[v].x + z * x.x, acc[v].y + z * x.y, acc[v].z + z * x.z};
  }
  __device__ __forceinline__ T aggregate(T beta, bool hard) const { return hard ? dmin : dmin - log_t(sumz) / beta; }
  // the weight-normalised sums (the soft-min gradient weights z / sum z)
  __device__ __forceinline__ void normalise() {
    const T inv = div_t(T(1), sumz);
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = {acc[v].x * inv, acc[v].y * inv, acc[v].z * inv};
  }
};

// Obstacle tables: CollisionParams (kernel parameter) or a per-problem copy in
// shared memory (trajectories) -- any type with okind/oa/ob/orad members.
template <typename T>
struct ObstacleTable {
  int32_t no;
  int32_t okind[kMaxObstacles];
  T oa[kMaxObstacles][3], ob[kMaxObstacles][3], orad[kMaxObstacles];
};

// sphere (centre c, radius r) vs obstacle o: distance and unit gradient (collision.py:192-204)
template <typename T, class OB>
__device__ __forceinline__ T sphere_obstacle_t(const OB& P, int o, const vec3<T>& c, T r, vec3<T>& n) {
  const int kind = P.okind[o];
  const vec3<T> a{P.oa[o][0], P.oa[o][1], P.oa[o][2]};
  if (kind == kObHalfSpace) {
    n = a;
    return dot(a, c) - P.orad[o] - r;
  }
  vec3<T> p = a;
  if (kind == kObCapsule) {  // closest point on the segment (collision.py:115-121)
    const vec3<T> d{P.ob[o][0] - a.x, P.ob[o][1] - a.y, P.ob[o][2] - a.z};
    const T dd = dot(d, d);
    T u = T(0);
    if (!(dd < T(1e-16))) {
      u = div_t(dot(vec3<T>{c.x - a.x, c.y - a.y, c.z - a.z}, d), dd);
      u = tmin(tmax(u, T(0)), T(1));
    }
    p = {a.x + u * d.x, a.y + u * d.y, a.z + u * d.z};
  }
  const vec3<T> v{c.x - p.x, c.y - p.y, c.z - p.z};
  T nn, inv;
  norm_inv_t(dot(v, v), nn, inv);
  if (nn < T(1e-12)) {
    n = {T(0), T(0), T(0)};
    return T(0) - r - P.orad[o];
  }
  n = {v.x * inv, v.y * inv, v.z * inv};
  return nn - r - P.orad[o];
}

// capsule (endpoints c0, c1, radius r) vs obstacle o: distance and the
// gradients at both endpoints (collision.py:207-237 with :115-152)
template <typename T, class OB>
__device__ __forceinline__ T capsule_obstacle_t(const OB& O, int o, const vec3<T>& c0, const vec3<T>& c1, T r,
                                                vec3<T>& ga, vec3<T>& gb) {
  const int kind = O.okind[o];
  const vec3<T> a{O.oa[o][0], O.oa[o][1], O.oa[o][2]};
  if (kind == kObHalfSpace) {
    const T da = dot(a, c0), db = dot(a, c1);
    const vec3<T> z{T(0), T(0), T(0)};
    if (da <= db) {
      ga = a;
      gb = z;
    } else {
      ga = z;
      gb = a;
    }
    return tmin(da, db) - O.orad[o] - r;
  }
  const vec3<T> d1{c1.x - c0.x, c1.y - c0.y, c1.z - c0.z};
  T s = T(0);
  vec3<T> qpt = a;
  if (kind == kObSphere) {
    const T dd = dot(d1, d1);
    if (!(dd < T(1e-16))) s = tmin(tmax(dot(vec3<T>{a.x - c0.x, a.y - c0.y, a.z - c0.z}, d1) / dd, T(0)), T(1));
  } else {  // capsule-capsule: Ericson's clamped quadratic (collision.py:124-152)
    const vec3<T> b{O.ob[o][0], O.ob[o][1], O.ob[o][2]};
    const vec3<T> d2{b.x - a.x, b.y - a.y, b.z - a.z};
    const vec3<T> rr{c0.x - a.x, c0.y - a.y, c0.z - a.z};
    const T aa = dot(d1, d1), e = dot(d2, d2), f = dot(d2, rr);
    T t = T(0);
    if (aa < T(1e-16) && e < T(1e-16)) {
      s = t = T(0);
    } else if (aa < T(1e-16)) {
      s = T(0);
      t = tmin(tmax(f / e, T(0)), T(1));
    } else {
      const T c = dot(d1, rr);
      if (e < T(1e-16)) {
        s = tmin(tmax(-c / aa, T(0)), T(1));
        t = T(0);
      } else {
        const T bb = dot(d1, d2);
        const T den = aa * e - bb * bb;
        s = den > T(1e-16) ? tmin(tmax((bb * f - c * e) / den, T(0)), T(1)) : T(0);
        t = (bb * s + f) / e;
        if (t < T(0)) {
          t = T(0);
          s = tmin(tmax(-c / aa, T(0)), T(1));
        } else if (t > T(1)) {
          t = T(1);
          s = tmin(tmax((bb - c) / aa, T(0)), T(1));
        }
      }
    }
    qpt = {a.x + t * d2.x, a.y + t * d2.y, a.z + t * d2.z};
  }
  const vec3<T> p{c0.x + s * d1.x, c0.y + s * d1.y, c0.z + s * d1.z};
  const vec3<T> v{p.x - qpt.x, p.y - qpt.y, p.z - qpt.z};
  const T nn = sqrt_t(dot(v, v));
  vec3<T> dir{T(0), T(0), T(0)};
  if (!(nn < T(1e-12))) {
    const T inv = T(1) / nn;
    dir = {v.x * inv, v.y * inv, v.z * inv};
  }
  ga = {(T(1) - s) * dir.x, (T(1) - s) * dir.y, (T(1) - s) * dir.z};
  gb = {s * dir.x, s * dir.y, s * dir.z};
  return (nn < T(1e-12) ? T(0) : nn) - r - O.orad[o];
}

// distance only (no gradient): the screening pass of a collision row
template <typename T, class OB>
__device__ __forceinline__ T sphere_obstacle_dist_t(const OB& P, int o, const vec3<T>& c, T r) {
  const int kind = P.okind[o];
  const vec3<T> a{P.oa[o][0], P.oa[o][1], P.oa[o][2]};
  if (kind == kObHalfSpace) return dot(a, c) - P.orad[o] - r;
  vec3<T> p = a;
  if (kind == kObCapsule) {
    const vec3<T> d{P.ob[o][0] - a.x, P.ob[o][1] - a.y, P.ob[o][2] - a.z};
    const T dd = dot(d, d);
    T u = T(0);
    if (!(dd < T(1e-16))) u = tmin(tmax(div_t(dot(vec3<T>{c.x - a.x, c.y - a.y, c.z - a.z}, d), dd), T(0)), T(1));
    p = {a.x + u * d.x, a.y + u * d.y, a.z + u * d.z};
  }
  const vec3<T> v{c.x - p.x, c.y - p.y, c.z - p.z};
  const T nn = norm_t(dot(v, v));
  return (nn < T(1e-12) ? T(0) : nn) - r - P.orad[o];
}

template <class G>
struct ColLane {  // per-lane scratch accessors
  typename G::T* s;
  int stride;
  __device__ __forceinline__ typename G::T& am(int k, int i) const { return s[(6 * k + i) * stride]; }
  __device__ __forceinline__ typename G::T& cen(int sph, int i) const {
    return s[(col_scratch_fixed<G>() + 3 * sph + i) * stride];
  }
};

// rank-1 update of the normal equations by one weighted row over the chain
// joints k <= kmax (and optionally minus those <= kmin2), row entries
// e_k = a_k . M - m_k . G (revolute) or a_k . G (prismatic), scaled by s.
template <class G>
__device__ __forceinline__ void col_row_accumulate(const ChainParams<typename G::T, G::K>& C, const ColLane<G>& L,
                                                   int slot_a, const vec3<typename G::T>& Ma, int slot_b,
                                                   const vec3<typename G::T>& Mb, const vec3<typename G::T>& Gv,
                                                   typename G::T scale, typename G::T res,
                                                   typename G::T (&A)[Tri<G::ND>::size], typename G::T (&g)[G::ND]) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, ND = G::ND;
  T jr[NQ];
#pragma unroll
  for (int c = 0; c < NQ; ++c) jr[c] = T(0);
#pragma unroll
  for (int k = 0; k < G::K; ++k) {
    if ((G::ID || k < C.k) && (k <= slot_a || k <= slot_b)) {
      const vec3<T> a{L.am(k, 0), L.am(k, 1), L.am(k, 2)};
      const vec3<T> m{L.am(k, 3), L.am(k, 4), L.am(k, 5)};
      const bool pri = !G::ID && C.prismatic[k];
      T e = T(0);
      if (k <= slot_a) e += pri ? T(0) : dot(a, Ma);
      if (k <= slot_b) e -= pri ? T(0) : dot(a, Mb);
      // G terms: + for side a, - for side b (self rows); world rows pass slot_b = -1
      const T gsign = (k <= slot_a ? T(1) : T(0)) - (k <= slot_b ? T(1) : T(0));
      e += gsign * (pri ? dot(a, Gv) : -dot(m, Gv));
      e *= scale;
      if (G::ID) {
        jr[k] += e;
      } else {
        const int qc = C.qcol[k];
        const T mu = C.mult[k];
#pragma unroll
        for (int c = 0; c < NQ; ++c)
          if (qc == c) jr[c] += mu * e;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
#pragma unroll
    for (int j = 0; j < NQ; ++j)
      if (j <= i) A[Tri<ND>::at(i, j)] += jr[i] * jr[j];
    g[i] += jr[i] * res;
  }
}

// Forward pass over the compiled chain: Pluecker axes of the moving joints and
// world sphere centres into the lane scratch; returns the EE world pose.
template <class G>
__device__ __forceinline__ void col_forward(const ChainParams<typename G::T, G::K>& C,
                                            const CollisionParams<typename G::T>& P, const ColLane<G>& L,
                                            const typename G::T (&q)[G::NQ], quat<typename G::T>& eq_out,
                                            vec3<typename G::T>& ep_out) {
  using T = typename G::T;
  constexpr int K = G::K;
  for (int s = P.slot_first[0]; s < P.slot_first[1]; ++s)
#pragma unroll
    for (int i = 0; i < 3; ++i) L.cen(s, i) = P.sc[s][i];
  quat<T> pq{T(1), T(0), T(0), T(0)};
  vec3<T> pp{T(0), T(0), T(0)};
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (G::ID || k < C.k) {
      const quat<T> tq{C.tq[k][0], C.tq[k][1], C.tq[k][2], C.tq[k][3]};
      quat<T> fq;
      vec3<T> fp;
      if (k == 0) {
        fq = tq;
        fp = {C.tp[0][0], C.tp[0][1], C.tp[0][2]};
      } else {
        fq = qmul(pq, tq);
        const vec3<T> o = qrot(pq, vec3<T>{C.tp[k][0], C.tp[k][1], C.tp[k][2]});
        fp = {pp.x + o.x, pp.y + o.y, pp.z + o.z};
      }
      const vec3<T> a = qzaxis(fq);
      const vec3<T> m = cross(a, fp);
      L.am(k, 0) = a.x; L.am(k, 1) = a.y; L.am(k, 2) = a.z;
      L.am(k, 3) = m.x; L.am(k, 4) = m.y; L.am(k, 5) = m.z;
      const T th = G::ID ? q[k] : pick(q, C.qcol[k]) * C.mult[k] + C.offset[k];
      if (!G::ID && C.prismatic[k]) {
        pq = fq;
        pp = {fp.x + th * a.x, fp.y + th * a.y, fp.z + th * a.z};
      } else {
        T sn, cs;
        sincos_t(T(0.5) * th, &sn, &cs);
        pq = qmul_z(fq, cs, sn);
        pp = fp;
      }
      const int s0 = P.slot_first[k + 1], s1 = P.slot_first[k + 2];
      if (s1 > s0) {
        const mat3<T> R = qmat(pq);
        for (int s = s0; s < s1; ++s) {
          const vec3<T> c = mul(R, vec3<T>{P.sc[s][0], P.sc[s][1], P.sc[s][2]});
          L.cen(s, 0) = c.x + pp.x;
          L.cen(s, 1) = c.y + pp.y;
          L.cen(s, 2) = c.z + pp.z;
        }
      }
    }
  }
  eq_out = qmul(pq, quat<T>{C.eq[0], C.eq[1], C.eq[2], C.eq[3]});
  const vec3<T> eo = qrot(pq, vec3<T>{C.ep[0], C.ep[1], C.ep[2]});
  ep_out = {pp.x + eo.x, pp.y + eo.y, pp.z + eo.z};

}

// World (sphere link x obstacle) and self (link pair) activation rows from the
// lane scratch filled by col_forward: adds their squares to the returned cost
// and, if JAC, their rank-1 terms to A, g.  row/row_out/jac_out: parity output.
// SCREEN: a first distance-only pass skips rows that are inactive on every
// lane of the warp (pays off when most rows are far from every obstacle, as in
// trajectories; in IK-Beam the seeds of a warp rarely agree, so it is off).
// PART: bit 0 world rows, bit 1 self rows (trajectories split them over two threads).
template <class G, bool JAC, class OB = CollisionParams<typename G::T>, bool SCREEN = false, int PART = 3>
__device__ __forceinline__ typename G::T col_rows(const ChainParams<typename G::T, G::K>& C,
                                                  const CollisionParams<typename G::T>& P, const ColLane<G>& L,
                                                  typename G::T (&A)[Tri<G::ND>::size], typename G::T (&g)[G::ND],
                                                  int row = 0, double* row_out = nullptr,
                                                  double* jac_out = nullptr, const OB* obs = nullptr,
                                                  int pair0 = 0, int pair1 = 1 << 30) {
  using T = typename G::T;
  constexpr int NQ = G::NQ;
  const OB& O = obs ? *obs : reinterpret_cast<const OB&>(P);
  T cost = T(0);
  // ---- world rows: (sphere link, obstacle), costs.py:499-551 ---------------
  if ((PART & 1) && P.w_world > T(0)) {
    for (int li = 0; li < P.nl; ++li) {
      const int f = P.lfirst[li], nsph = P.lcount[li];
      for (int o = 0; o < O.no; ++o, ++row) {
        if (SCREEN) {  // an inactive row (activation exactly 0) needs no gradient work
          T dscr = inf_t<T>();
          for (int s = 0; s < nsph; ++s)
            dscr = tmin(dscr, sphere_obstacle_dist_t<T>(O, o, vec3<T>{L.cen(f + s, 0), L.cen(f + s, 1),
                                                                     L.cen(f + s, 2)}, P.sr[f + s]));
          // warp-uniform: lanes that skip would otherwise idle beside active ones
          if (__all_sync(__activemask(), dscr - P.lreach[li] > P.eta_world * T(1.00001))) {
            if (row_out) row_out[row] = 0.0;
            continue;
          }
        }
        const bool hard = P.hard || nsph == 1;
        SoftMin<T, 2> sm;  // acc[0] = sum z c x n, acc[1] = sum z n
        for (int s = 0; s < nsph; ++s) {
          const vec3<T> c{L.cen(f + s, 0), L.cen(f + s, 1), L.cen(f + s, 2)};
          vec3<T> n;
          const T d = sphere_obstacle_t<T>(O, o, c, P.sr[f + s], n);
          const T z = sm.weight(d, P.beta, hard);
          if (z == T(0)) continue;  // zero weights add nothing (the reference skips them, costs.py:541)
          sm.sumz += z;
          if (JAC) {
            sm.add(z, 0, cross(c, n));
            sm.add(z, 1, n);
          }
        }
        T act, dact;
        activation_t(sm.aggregate(P.beta, hard), P.eta_world, act, dact);
        const T res = P.w_world * act;
        cost += res * res;
        if (row_out) row_out[row] = double(res);
        if (JAC && dact != T(0)) {
          sm.normalise();
          const vec3<T> M = sm.acc[0], Gv = sm.acc[1];
          col_row_accumulate<G>(C, L, P.lslot[li], M, -1, M, Gv, P.w_world * dact, res, A, g);
          if (jac_out) {  // parity output: recompute the row entries
            T Az[Tri<NQ>::size], gz[NQ];
#pragma unroll
            for (int i = 0; i < Tri<NQ>::size; ++i) Az[i] = T(0);
#pragma unroll
            for (int i = 0; i < NQ; ++i) gz[i] = T(0);
            col_row_accumulate<G>(C, L, P.lslot[li], M, -1, M, Gv, P.w_world * dact, T(1), Az, gz);
#pragma unroll
            for (int c = 0; c < NQ; ++c) jac_out[row * NQ + c] = double(gz[c]);
          }
        }
      }
    }
  }

  // ---- self rows: link pairs, costs.py:435-496 ------------------------------
  if ((PART & 2) && P.w_self > T(0)) {
    const int pend = P.np < pair1 ? P.np : pair1;  // self pairs [pair0, pend) (split across threads: trajectories)
    for (int pi = pair0; pi < pend; ++pi, ++row) {
      const int la = P.pa[pi], lb = P.pb[pi];
      const int fa = P.lfirst[la], na = P.lcount[la], fb = P.lfirst[lb], nb = P.lcount[lb];
      if (SCREEN) {
        T dscr = inf_t<T>();
        for (int i = 0; i < na; ++i)
          for (int j = 0; j < nb; ++j) {
            const vec3<T> v{L.cen(fa + i, 0) - L.cen(fb + j, 0), L.cen(fa + i, 1) - L.cen(fb + j, 1),
                            L.cen(fa + i, 2) - L.cen(fb + j, 2)};
            dscr = tmin(dscr, norm_t(dot(v, v)) - P.sr[fa + i] - P.sr[fb + j]);
          }
        if (__all_sync(__activemask(), dscr - P.preach[pi] > P.eta_self * T(1.00001))) {
          if (row_out) row_out[row] = 0.0;
          continue;
        }
      }
      const bool hard = P.hard || na * nb == 1;
      SoftMin<T, 3> sm;  // acc[0] = sum z ca x n, acc[1] = sum z cb x n, acc[2] = sum z n
      for (int i = 0; i < na; ++i)
        for (int j = 0; j < nb; ++j) {
          const vec3<T> ca{L.cen(fa + i, 0), L.cen(fa + i, 1), L.cen(fa + i, 2)};
          const vec3<T> cb{L.cen(fb + j, 0), L.cen(fb + j, 1), L.cen(fb + j, 2)};
          const vec3<T> v{ca.x - cb.x, ca.y - cb.y, ca.z - cb.z};
          T dist, inv;
          norm_inv_t(dot(v, v), dist, inv);
          const T z = sm.weight(dist - P.sr[fa + i] - P.sr[fb + j], P.beta, hard);
          if (z == T(0)) continue;
          sm.sumz += z;
          if (JAC && dist > T(1e-12)) {
            const vec3<T> n{v.x * inv, v.y * inv, v.z * inv};
            sm.add(z, 0, cross(ca, n));
            sm.add(z, 1, cross(cb, n));
            sm.add(z, 2, n);
          }
        }
      T act, dact;
      activation_t(sm.aggregate(P.beta, hard), P.eta_self, act, dact);
      const T res = P.w_self * act;
      cost += res * res;
      if (row_out) row_out[row] = double(res);
      if (JAC && dact != T(0)) {
        sm.normalise();
        const vec3<T> Ma = sm.acc[0], Mb = sm.acc[1], Gv = sm.acc[2];
        col_row_accumulate<G>(C, L, P.lslot[la], Ma, P.lslot[lb], Mb, Gv, P.w_self * dact, res, A, g);
        if (jac_out) {
          T Az[Tri<NQ>::size], gz[NQ];
#pragma unroll
          for (int i = 0; i < Tri<NQ>::size; ++i) Az[i] = T(0);
#pragma unroll
          for (int i = 0; i < NQ; ++i) gz[i] = T(0);
          col_row_accumulate<G>(C, L, P.lslot[la], Ma, P.lslot[lb], Mb, Gv, P.w_self * dact, T(1), Az, gz);
#pragma unroll
          for (int c = 0; c < NQ; ++c) jac_out[row * NQ + c] = double(gz[c]);
        }
      }
    }
  }
  return cost;
}

// Weighted residual stack [pose 6 | limit n | rest n | world nl*no | self np]
// of a collision lane: returns the cost; JAC also forms A = J^T J, g = J^T r.
// row_out (optional, for the parity API) receives every weighted residual and
// jac_out its Jacobian rows (rows x NQ).
template <class G, bool JAC>
__device__ __forceinline__ typename G::T col_eval(const ChainParams<typename G::T, G::K>& C,
                                                  const CostParams<typename G::T, G::NQ>& W,
                                                  const CollisionParams<typename G::T>& P,
                                                  const TargetInv<typename G::T>& tg, const ColLane<G>& L,
                                                  const typename G::T (&q)[G::NQ],
                                                  typename G::T (&A)[Tri<G::ND>::size], typename G::T (&g)[G::ND],
                                                  double* row_out = nullptr, double* jac_out = nullptr) {
  using T = typename G::T;
  constexpr int K = G::K, NQ = G::NQ;
  static_assert(!G::BASE, "collision lanes have a fixed base");
  quat<T> eq;
  vec3<T> ep;
  col_forward<G>(C, P, L, q, eq, ep);
  // ---- pose rows: body columns from the Pluecker axes -----------------------
  T col[K][6];
  if (JAC) {
    const mat3<T> R = qmat(eq);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (G::ID || k < C.k) {
        const vec3<T> a{L.am(k, 0), L.am(k, 1), L.am(k, 2)};
        const vec3<T> ang = mulT(R, a);
        if (!G::ID && C.prismatic[k]) {
          col[k][0] = ang.x; col[k][1] = ang.y; col[k][2] = ang.z;
          col[k][3] = T(0); col[k][4] = T(0); col[k][5] = T(0);
        } else {
          const vec3<T> m{L.am(k, 3), L.am(k, 4), L.am(k, 5)};
          const vec3<T> x = cross(a, ep);
          const vec3<T> lin = mulT(R, vec3<T>{x.x - m.x, x.y - m.y, x.z - m.z});
          col[k][0] = lin.x; col[k][1] = lin.y; col[k][2] = lin.z;
          col[k][3] = ang.x; col[k][4] = ang.y; col[k][5] = ang.z;
        }
      }
    }
  }
  T r[6], J[6][NQ];
  const T zb[3] = {T(0), T(0), T(0)};
  pose_finish<G, JAC>(C, W, tg, eq, ep, col, r, J);
  T cost = assemble_rows<G, JAC>(W, q, zb, r, J, A, g);
  if (row_out) {
#pragma unroll
    for (int m = 0; m < 6; ++m) {
      row_out[m] = double(r[m]);
      if (jac_out)
#pragma unroll
        for (int c = 0; c < NQ; ++c) jac_out[m * NQ + c] = double(J[m][c]);
    }
  }
  int row = 6 + 2 * NQ;  // next row index (parity output)

  return cost + col_rows<G, JAC>(C, P, L, A, g, row, row_out, jac_out);
}


template <class G>
struct CollisionModel {
  using T = typename G::T;
  const ChainParams<T, G::K>& C;
  const CostParams<T, G::NQ>& W;
  const CollisionParams<T>& P;
  TargetInv<T> tg;
  ColLane<G> L;
  template <bool JAC>
  __device__ __forceinline__ T eval(const T (&q)[G::NQ], const T (&)[3], T (&A)[Tri<G::ND>::size],
                                    T (&g)[G::ND]) const {
    return col_eval<G, JAC>(C, W, P, tg, L, q, A, g);
  }
};

}  // namespace kop
