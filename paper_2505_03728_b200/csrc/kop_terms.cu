// Per-term evaluation of the typed cost families: the raw (unweighted)
// residual rows of ONE CostTerm and its Jacobian block per referenced
// variable, at a batch of variable values -- the device side of
// CostTerm.raw_residual / CostTerm.jacobian / solver.assemble
// (solver.py:142-152, 289-324) for the builders of costs.py:98-619.
//
// These kernels are the inspection / assembly API, not the solve hot path:
// FP64, one thread per evaluation point, a plain full-tree FK (reference op
// order, robot.py:404-448) with world joint anchors and axes, point
// Jacobians over the link's ancestor joints (robot.py:486-506) -- the
// reference's formulation of each row, independent of the fused solve
// kernels (which tests/test_gpu_terms.py checks them against).
#include <cuda_runtime.h>
#include <stdint.h>

#include "kop_collision.cuh"
#include "kop_kernels.cuh"
#include "kop_terms.cuh"

namespace kop {

namespace {

struct Frames {
  quat<double> lq[kMaxLinks];
  vec3<double> lp[kMaxLinks];
  vec3<double> jp[kMaxTreeJoints], ja[kMaxTreeJoints];  // world anchor / axis before the motion
};

// fk_arrays (robot.py:404-448): link frames, joint anchors and world axes
__device__ void tree_fk(const TreeParams& P, const double* __restrict__ q, Frames& F) {
  F.lq[0] = {1.0, 0.0, 0.0, 0.0};
  F.lp[0] = {0.0, 0.0, 0.0};
  for (int j = 0; j < P.nj; ++j) {
    const quat<double> pq = F.lq[P.parent[j]];
    const vec3<double> pp = F.lp[P.parent[j]];
    const quat<double> fq = qmul(pq, quat<double>{P.oq[j][0], P.oq[j][1], P.oq[j][2], P.oq[j][3]});
    const vec3<double> o = qrot(pq, vec3<double>{P.op[j][0], P.op[j][1], P.op[j][2]});
    const vec3<double> fp{pp.x + o.x, pp.y + o.y, pp.z + o.z};
    const vec3<double> axis{P.axis[j][0], P.axis[j][1], P.axis[j][2]};
    const vec3<double> wa = qrot(fq, axis);
    F.jp[j] = fp;
    F.ja[j] = wa;
    const int c = P.child[j];
    if (P.kind[j] == 0) {
      F.lq[c] = fq;
      F.lp[c] = fp;
      continue;
    }
    const double th = q[P.qcol[j]] * P.mult[j] + P.offset[j];
    if (P.kind[j] == 1) {
      double s, co;
      sincos(0.5 * th, &s, &co);
      F.lq[c] = qmul(fq, quat<double>{co, s * axis.x, s * axis.y, s * axis.z});
      F.lp[c] = fp;
    } else {
      F.lq[c] = fq;
      F.lp[c] = {fp.x + th * wa.x, fp.y + th * wa.y, fp.z + th * wa.z};
    }
  }
}

// row += s * (g . J_point(p)) over the ancestor joints of `link` (robot.py:486-506,
// rotational=False): revolute mult * (a x (p - anchor)), prismatic mult * a
__device__ void point_row(const TreeParams& P, const LinkMap& link_pj, const Frames& F, int link,
                          const vec3<double>& p, const vec3<double>& g, double s, double* row) {
  for (int j = link_pj.pj[link]; j >= 0; j = link_pj.pj[P.parent[j]]) {
    if (P.kind[j] == 0) continue;
    const vec3<double> a = F.ja[j];
    vec3<double> col = a;
    if (P.kind[j] == 1) col = cross(a, vec3<double>{p.x - F.jp[j].x, p.y - F.jp[j].y, p.z - F.jp[j].z});
    row[P.qcol[j]] += s * P.mult[j] * dot(g, col);
  }
}

__device__ __forceinline__ vec3<double> sphere_centre(const TermGeom& G, const Frames& F, int s) {
  const int l = G.s_link[s];
  const vec3<double> c = qrot(F.lq[l], vec3<double>{G.s_c[s][0], G.s_c[s][1], G.s_c[s][2]});
  return {c.x + F.lp[l].x, c.y + F.lp[l].y, c.z + F.lp[l].z};
}

// _softmin (costs.py:409-420) weights, hard minimum = first argmin
__device__ double softmin_weights(const double* d, int n, double beta, bool hard, double* w) {
  if (hard || n == 1) {
    int k = 0;
    for (int i = 1; i < n; ++i)
      if (d[i] < d[k]) k = i;
    for (int i = 0; i < n; ++i) w[i] = i == k ? 1.0 : 0.0;
    return d[k];
  }
  double dmin = d[0];
  for (int i = 1; i < n; ++i) dmin = fmin(dmin, d[i]);
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    w[i] = exp(-beta * (d[i] - dmin));
    s += w[i];
  }
  for (int i = 0; i < n; ++i) w[i] /= s;
  return dmin - log(s) / beta;
}

}  // namespace

// ---- pose_cost (costs.py:98-166), optional SE(2) / SE(3) base ---------------
__global__ void __launch_bounds__(64)
k_term_pose(const TreeParams P, const LinkMap link_pj, int link, TermPose T,
            const double* __restrict__ q, const double* __restrict__ base, int64_t B, double* __restrict__ r_out,
            double* __restrict__ jq_out, double* __restrict__ jb_out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  Frames F;
  tree_fk(P, q + b * P.n, F);
  const quat<double> fq = F.lq[link];
  const vec3<double> fp = F.lp[link];
  quat<double> cq = fq;
  vec3<double> cp = fp;
  if (T.base_kind != 0) {  // B * FK (costs.py:114-119): base as (wxyz, xyz)
    const double* bb = base + b * 7;
    const quat<double> bq{bb[0], bb[1], bb[2], bb[3]};
    const vec3<double> t = qrot(bq, fp);
    cq = qmul(bq, fq);
    cp = {t.x + bb[4], t.y + bb[5], t.z + bb[6]};
  }
  const quat<double> tq{T.tinv[0], T.tinv[1], T.tinv[2], T.tinv[3]};
  const quat<double> eq = qmul(tq, cq);
  const vec3<double> et0 = qrot(tq, cp);
  const vec3<double> et{T.tinv[4] + et0.x, T.tinv[5] + et0.y, T.tinv[6] + et0.z};
  const Twist<double> xi = se3_log(eq, et);
  double* r = r_out + b * 6;
  r[0] = xi.v.x; r[1] = xi.v.y; r[2] = xi.v.z;
  r[3] = xi.phi.x; r[4] = xi.phi.y; r[5] = xi.phi.z;
  if (!jq_out && !jb_out) return;
  const JrInv<double> jr = se3_jr_inv(xi);
  const mat3<double> R = qmat(fq);
  auto apply = [&](const vec3<double>& lin, const vec3<double>& ang, double* col, int stride) {
    // Jr^-1 [lin; ang] into column col[m * stride]
    const vec3<double> t1 = mul(jr.A, lin), t2 = mul(jr.B, ang), a1 = mul(jr.A, ang);
    col[0] += t1.x + t2.x; col[stride] += t1.y + t2.y; col[2 * stride] += t1.z + t2.z;
    col[3 * stride] += a1.x; col[4 * stride] += a1.y; col[5 * stride] += a1.z;
  };
  if (jq_out) {  // Jr^-1 [R^T J_lin; R^T J_ang] (costs.py:123-136)
    const int n = P.n;
    double* J = jq_out + b * 6 * n;
    for (int i = 0; i < 6 * n; ++i) J[i] = 0.0;
    for (int j = link_pj.pj[link]; j >= 0; j = link_pj.pj[P.parent[j]]) {
      if (P.kind[j] == 0) continue;
      const vec3<double> a = F.ja[j];
      vec3<double> lin = a, ang{0.0, 0.0, 0.0};
      if (P.kind[j] == 1) {
        lin = cross(a, vec3<double>{fp.x - F.jp[j].x, fp.y - F.jp[j].y, fp.z - F.jp[j].z});
        ang = a;
      }
      const double mu = P.mult[j];
      const vec3<double> lb = mulT(R, lin), ab = mulT(R, ang);
      apply({mu * lb.x, mu * lb.y, mu * lb.z}, {mu * ab.x, mu * ab.y, mu * ab.z}, J + P.qcol[j], n);
    }
  }
  if (jb_out && T.base_kind != 0) {  // Jr^-1 Ad(FK^-1) [E_se2] (costs.py:140-146)
    // Ad(FK^-1) e_i: translation i -> [R^T e_i; 0]; rotation i -> [R^T (e_i x p); R^T e_i]
    const int db = T.base_kind == 1 ? 3 : 6;
    double* J = jb_out + b * 6 * db;
    for (int i = 0; i < 6 * db; ++i) J[i] = 0.0;
    for (int c = 0; c < db; ++c) {
      // tangent component of column c: SE(2) (vx, vy, w) = se(3) (0, 1, 5); SE(3) all six
      const int comp = T.base_kind == 1 ? (c == 2 ? 5 : c) : c;
      vec3<double> e{comp % 3 == 0 ? 1.0 : 0.0, comp % 3 == 1 ? 1.0 : 0.0, comp % 3 == 2 ? 1.0 : 0.0};
      vec3<double> lin, ang{0.0, 0.0, 0.0};
      if (comp < 3) {
        lin = mulT(R, e);
      } else {
        lin = mulT(R, cross(e, fp));
        ang = mulT(R, e);
      }
      apply(lin, ang, J + c, db);
    }
  }
}

// ---- joint-space families (costs.py:174-341) ---------------------------------
__global__ void __launch_bounds__(128)
k_term_joint(TermJoint T, int n, const double* __restrict__ qs, int64_t B, double* __restrict__ r_out,
             double* __restrict__ jd_out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const double* x = qs + b * T.nvars * n;
  double* r = r_out + b * n;
  double* jd = jd_out ? jd_out + b * T.nvars * n : nullptr;  // diagonal of each variable's block
  for (int i = 0; i < n; ++i) {
    double v = 0.0;
    double d[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    switch (T.kind) {
      case KOP_TERM_LIMIT: {  // max(0, q - u) + max(0, l - q), subgradient 0 at the boundary
        const double qi = x[i];
        v = fmax(0.0, qi - T.upper[i]) + fmax(0.0, T.lower[i] - qi);
        d[0] = (qi > T.upper[i] ? 1.0 : 0.0) + (qi < T.lower[i] ? -1.0 : 0.0);
        break;
      }
      case KOP_TERM_REST:
        v = x[i] - T.rest[i];
        d[0] = 1.0;
        break;
      case KOP_TERM_SMOOTHNESS:
        v = x[n + i] - x[i];
        d[0] = -1.0;
        d[1] = 1.0;
        break;
      case KOP_TERM_VELOCITY: {  // max(0, |dq| - v dt); unlimited joints 0 (costs.py:198-231)
        const double dq = x[n + i] - x[i], lim = T.vlim[i] * T.dt;
        if (isfinite(T.vlim[i]) && fabs(dq) - lim > 0.0) {
          v = fabs(dq) - lim;
          const double sg = dq > 0.0 ? 1.0 : (dq < 0.0 ? -1.0 : 0.0);
          d[0] = -sg;
          d[1] = sg;
        }
        break;
      }
      case KOP_TERM_STENCIL:  // sum(c_k q_k) in numpy's order, no FMA contraction (costs.py:309-310)
        for (int k = 0; k < 5; ++k) {
          v = __dadd_rn(v, __dmul_rn(T.coeffs[k], x[k * n + i]));
          d[k] = T.coeffs[k];
        }
        break;
    }
    r[i] = v;
    if (jd)
      for (int k = 0; k < T.nvars; ++k) jd[k * n + i] = d[k];
  }
}

// ---- collision families (costs.py:423-619) -----------------------------------
__global__ void __launch_bounds__(64)
k_term_collision(const TreeParams P, const LinkMap link_pj, const TermGeom G, int kind,
                 const double* __restrict__ q0, const double* __restrict__ q1, int64_t B, double* __restrict__ r_out,
                 double* __restrict__ j0_out, double* __restrict__ j1_out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int n = P.n;
  Frames F0;
  tree_fk(P, q0 + b * n, F0);
  Frames* F1 = nullptr;
  Frames F1s;
  if (kind == KOP_TERM_SWEPT) {
    tree_fk(P, q1 + b * n, F1s);
    F1 = &F1s;
  }
  const int rows = kind == KOP_TERM_SELF ? G.np : G.nl * G.O.no;
  double* r = r_out + b * rows;
  double* J0 = j0_out ? j0_out + b * rows * n : nullptr;
  double* J1 = j1_out ? j1_out + b * rows * n : nullptr;
  if (J0)
    for (int i = 0; i < rows * n; ++i) J0[i] = 0.0;
  if (J1)
    for (int i = 0; i < rows * n; ++i) J1[i] = 0.0;
  double d[kMaxSpheres * kMaxSpheres > 64 ? 64 : kMaxSpheres * kMaxSpheres], w[64];
  vec3<double> ga[64], gb[64];
  for (int row = 0; row < rows; ++row) {
    int cnt = 0;
    if (kind == KOP_TERM_SELF) {  // sphere pairs of the two links (costs.py:449-465)
      const int la = G.pa[row], lb = G.pb[row];
      for (int sa = 0; sa < G.ns; ++sa) {
        if (G.s_link[sa] != la) continue;
        const vec3<double> ca = sphere_centre(G, F0, sa);
        for (int sb = 0; sb < G.ns; ++sb) {
          if (G.s_link[sb] != lb || cnt >= 64) continue;
          const vec3<double> cb = sphere_centre(G, F0, sb);
          const vec3<double> v{ca.x - cb.x, ca.y - cb.y, ca.z - cb.z};
          const double dist = sqrt(dot(v, v));
          d[cnt] = dist - G.s_r[sa] - G.s_r[sb];
          ga[cnt] = dist > 1e-12 ? vec3<double>{v.x / dist, v.y / dist, v.z / dist} : vec3<double>{0.0, 0.0, 0.0};
          cnt++;
        }
      }
    } else {  // (sphere link, obstacle) rows in link-major order (costs.py:520-522, 581-583)
      const int li = G.links[row / G.O.no], o = row % G.O.no;
      for (int s = 0; s < G.ns; ++s) {
        if (G.s_link[s] != li || cnt >= 64) continue;
        const vec3<double> c0 = sphere_centre(G, F0, s);
        if (kind == KOP_TERM_WORLD) {
          d[cnt] = sphere_obstacle_t<double>(G.O, o, c0, G.s_r[s], ga[cnt]);
        } else {
          const vec3<double> c1 = sphere_centre(G, *F1, s);
          d[cnt] = capsule_obstacle_t<double>(G.O, o, c0, c1, G.s_r[s], ga[cnt], gb[cnt]);
        }
        cnt++;
      }
    }
    const double agg = softmin_weights(d, cnt, G.beta, G.hard != 0, w);
    double act, dact;
    activation_t(agg, G.eta, act, dact);
    r[row] = act;
    if (!J0 || dact == 0.0) continue;
    double* row0 = J0 + row * n;
    double* row1 = J1 ? J1 + row * n : nullptr;
    int k = 0;
    if (kind == KOP_TERM_SELF) {  // w_k n_k . (J_a(c_a) - J_b(c_b)) (costs.py:467-476)
      const int la = G.pa[row], lb = G.pb[row];
      for (int sa = 0; sa < G.ns; ++sa) {
        if (G.s_link[sa] != la) continue;
        const vec3<double> ca = sphere_centre(G, F0, sa);
        for (int sb = 0; sb < G.ns; ++sb) {
          if (G.s_link[sb] != lb || k >= 64) continue;
          if (w[k] != 0.0) {
            const vec3<double> cb = sphere_centre(G, F0, sb);
            point_row(P, link_pj, F0, la, ca, ga[k], dact * w[k], row0);
            point_row(P, link_pj, F0, lb, cb, ga[k], -dact * w[k], row0);
          }
          k++;
        }
      }
    } else {
      const int li = G.links[row / G.O.no];
      for (int s = 0; s < G.ns; ++s) {
        if (G.s_link[s] != li || k >= 64) continue;
        if (w[k] != 0.0) {
          point_row(P, link_pj, F0, li, sphere_centre(G, F0, s), ga[k], dact * w[k], row0);
          if (kind == KOP_TERM_SWEPT && row1)
            point_row(P, link_pj, *F1, li, sphere_centre(G, *F1, s), gb[k], dact * w[k], row1);
        }
        k++;
      }
    }
  }
}

// ---- manipulability_cost (costs.py:349-401) with translational_jacobian_with_derivative
// (robot.py:509-566): J (3 x n) of `link`'s origin and dJ/dq_a, differentiating the geometric
// column formulas joint by joint (mimic multipliers folded into both axes); measure
// m = sqrt(det(J J^T)) (n >= 3) or sqrt(det(J^T J)) (n < 3); r = 1 / (m + eps), gradient
// -0.5 m tr(G^-1 dG_a) / (m + eps)^2, zero at singularities (det <= 1e-18).
__global__ void __launch_bounds__(32)
k_term_manip(const TreeParams P, const LinkMap link_pj, int link, double eps, const double* __restrict__ q,
             int64_t B, double* __restrict__ r_out, double* __restrict__ jrow_out, double* __restrict__ jac_out,
             double* __restrict__ djac_out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  const int n = P.n;
  Frames F;
  tree_fk(P, q + b * n, F);
  const vec3<double> pe = F.lp[link];
  int mv[kMaxTreeJoints], nm = 0;  // moving joints on the root -> link path
  for (int j = link_pj.pj[link]; j >= 0; j = link_pj.pj[P.parent[j]])
    if (P.kind[j] != 0) mv[nm++] = j;
  vec3<double> raw[kMaxTreeJoints];
  for (int k = 0; k < nm; ++k) {
    const int j = mv[k];
    raw[j] = P.kind[j] == 1 ? cross(F.ja[j], vec3<double>{pe.x - F.jp[j].x, pe.y - F.jp[j].y, pe.z - F.jp[j].z})
                            : F.ja[j];
  }
  double* J = jac_out ? jac_out + b * 3 * n : nullptr;
  double* dJ = djac_out ? djac_out + b * 3 * n * n : nullptr;
  double Jl[3 * kTreeMaxDofsTerms];
  for (int i = 0; i < 3 * n; ++i) Jl[i] = 0.0;
  for (int k = 0; k < nm; ++k) {
    const int j = mv[k], c = P.qcol[j];
    Jl[0 * n + c] += P.mult[j] * raw[j].x;
    Jl[1 * n + c] += P.mult[j] * raw[j].y;
    Jl[2 * n + c] += P.mult[j] * raw[j].z;
  }
  if (J)
    for (int i = 0; i < 3 * n; ++i) J[i] = Jl[i];
  // s is an ancestor of joint i's frame: walking up from i's parent link meets s
  auto upstream = [&](int s, int i) {
    for (int j = link_pj.pj[P.parent[i]]; j >= 0; j = link_pj.pj[P.parent[j]])
      if (j == s) return true;
    return false;
  };
  // dJ[a][row][col], a = qcol of the differentiated joint s
  double gram[9], ginv[9];
  const bool wide = n >= 3;  // J J^T (3 x 3) or J^T J (n x n, n < 3)
  const int gdim = wide ? 3 : n;
  for (int u = 0; u < gdim; ++u)
    for (int v = 0; v < gdim; ++v) {
      double acc = 0.0;
      if (wide)
        for (int c = 0; c < n; ++c) acc += Jl[u * n + c] * Jl[v * n + c];
      else
        for (int rr = 0; rr < 3; ++rr) acc += Jl[rr * n + u] * Jl[rr * n + v];
      gram[u * gdim + v] = acc;
    }
  double det;
  if (gdim == 3) {
    const double* g = gram;
    det = g[0] * (g[4] * g[8] - g[5] * g[7]) - g[1] * (g[3] * g[8] - g[5] * g[6]) + g[2] * (g[3] * g[7] - g[4] * g[6]);
    ginv[0] = (g[4] * g[8] - g[5] * g[7]) / det; ginv[1] = (g[2] * g[7] - g[1] * g[8]) / det;
    ginv[2] = (g[1] * g[5] - g[2] * g[4]) / det; ginv[3] = (g[5] * g[6] - g[3] * g[8]) / det;
    ginv[4] = (g[0] * g[8] - g[2] * g[6]) / det; ginv[5] = (g[2] * g[3] - g[0] * g[5]) / det;
    ginv[6] = (g[3] * g[7] - g[4] * g[6]) / det; ginv[7] = (g[1] * g[6] - g[0] * g[7]) / det;
    ginv[8] = (g[0] * g[4] - g[1] * g[3]) / det;
  } else if (gdim == 2) {
    det = gram[0] * gram[3] - gram[1] * gram[2];
    ginv[0] = gram[3] / det; ginv[1] = -gram[1] / det; ginv[2] = -gram[2] / det; ginv[3] = gram[0] / det;
  } else {
    det = gram[0];
    ginv[0] = 1.0 / det;
  }
  const bool singular = !(det > 1e-18);
  const double m = singular ? 0.0 : sqrt(det);
  if (r_out) r_out[b] = 1.0 / (m + eps);
  double grad[kTreeMaxDofsTerms];
  for (int a = 0; a < n; ++a) grad[a] = 0.0;
  if (dJ)
    for (int i = 0; i < 3 * n * n; ++i) dJ[i] = 0.0;
  // d_col of column i w.r.t. theta_s (robot.py:544-565); dJa = dJ/dq_a accumulated per a
  for (int a = 0; a < n; ++a) {
    double dJa[3 * kTreeMaxDofsTerms];
    for (int i = 0; i < 3 * n; ++i) dJa[i] = 0.0;
    bool any = false;
    for (int ks = 0; ks < nm; ++ks) {
      const int s = mv[ks];
      if (P.qcol[s] != a) continue;
      any = true;
      for (int ki = 0; ki < nm; ++ki) {
        const int i = mv[ki];
        const bool rev_i = P.kind[i] == 1;
        vec3<double> dcol{0.0, 0.0, 0.0};
        if (upstream(s, i)) {
          vec3<double> dw{0.0, 0.0, 0.0}, dp;
          if (P.kind[s] == 1) {
            dw = cross(F.ja[s], F.ja[i]);
            dp = cross(F.ja[s], vec3<double>{F.jp[i].x - F.jp[s].x, F.jp[i].y - F.jp[s].y, F.jp[i].z - F.jp[s].z});
          } else {
            dp = F.ja[s];
          }
          if (rev_i) {
            const vec3<double> t1 = cross(dw, vec3<double>{pe.x - F.jp[i].x, pe.y - F.jp[i].y, pe.z - F.jp[i].z});
            const vec3<double> t2 = cross(F.ja[i], vec3<double>{raw[s].x - dp.x, raw[s].y - dp.y, raw[s].z - dp.z});
            dcol = {t1.x + t2.x, t1.y + t2.y, t1.z + t2.z};
          } else {
            dcol = dw;
          }
        } else if (rev_i) {
          dcol = cross(F.ja[i], raw[s]);
        }
        const double mm = P.mult[i] * P.mult[s];
        const int c = P.qcol[i];
        dJa[0 * n + c] += mm * dcol.x;
        dJa[1 * n + c] += mm * dcol.y;
        dJa[2 * n + c] += mm * dcol.z;
      }
    }
    if (!any) continue;
    if (dJ)
      for (int i = 0; i < 3 * n; ++i) dJ[a * 3 * n + i] = dJa[i];
    if (singular) continue;
    // tr(G^-1 dG), dG = dJa J^T + J dJa^T (wide) or dJa^T J + J^T dJa
    double tr = 0.0;
    for (int u = 0; u < gdim; ++u)
      for (int v = 0; v < gdim; ++v) {
        double dg = 0.0;
        if (wide)
          for (int c = 0; c < n; ++c) dg += dJa[u * n + c] * Jl[v * n + c] + Jl[u * n + c] * dJa[v * n + c];
        else
          for (int rr = 0; rr < 3; ++rr) dg += dJa[rr * n + u] * Jl[rr * n + v] + Jl[rr * n + u] * dJa[rr * n + v];
        tr += ginv[v * gdim + u] * dg;
      }
    grad[a] = 0.5 * m * tr;
  }
  if (jrow_out)
    for (int a = 0; a < n; ++a) jrow_out[b * n + a] = -grad[a] / ((m + eps) * (m + eps));
}

cudaError_t launch_term_manip(const TreeParams& P, const LinkMap& L, int link, double eps, const double* q,
                              int64_t B, double* r, double* jrow, double* jac, double* djac, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  k_term_manip<<<(unsigned)((B + 31) / 32), 32, 0, st>>>(P, L, link, eps, q, B, r, jrow, jac, djac);
  return cudaGetLastError();
}

cudaError_t launch_term_pose(const TreeParams& P, const LinkMap& link_pj, int link, const TermPose& T,
                             const double* q, const double* base, int64_t B, double* r, double* jq, double* jb,
                             cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  k_term_pose<<<(unsigned)((B + 63) / 64), 64, 0, st>>>(P, link_pj, link, T, q, base, B, r, jq, jb);
  return cudaGetLastError();
}

cudaError_t launch_term_joint(const TermJoint& T, int n, const double* qs, int64_t B, double* r, double* jd,
                              cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  k_term_joint<<<(unsigned)((B + 127) / 128), 128, 0, st>>>(T, n, qs, B, r, jd);
  return cudaGetLastError();
}

cudaError_t launch_term_collision(const TreeParams& P, const LinkMap& link_pj, const TermGeom& G, int kind,
                                  const double* q0, const double* q1, int64_t B, double* r, double* j0, double* j1,
                                  cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  k_term_collision<<<(unsigned)((B + 63) / 64), 64, 0, st>>>(P, link_pj, G, kind, q0, q1, B, r, j0, j1);
  return cudaGetLastError();
}

}  // namespace kop
