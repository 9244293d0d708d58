// Multi-end-effector IK on a kinematic TREE through the generic LM (config 3:
// humanoid, n <= 32 actuated joints): one warp per problem.
//
// Reference path: one pose_cost per end effector (costs.py:98-166) +
// limit_cost + rest_cost, solved by solver.solve (solver.py:364-429).
//
// Warp mapping (a problem is too large for one thread's registers -- a 24x29
// Jacobian, a 29x29 normal matrix):
//   * FK:  every joint's local transform at once, then log2(depth) pointer-
//         jumping composition rounds over the tree (fixed joints folded into
//         their children on the host), the Pluecker axis (a, m = a x o) of
//         each moving joint; lanes e < E read the end-effector frames, then
//         form the pose residual xi_e and the weighted Jr^-1(xi_e) blocks.
//   * J:   lane c owns Jacobian column c (its joint(s) via qcol), 6E entries
//         in registers, mirrored to shared memory.
//   * A:   lane i forms row i of J^T J (its lower part) from its own column and broadcast reads.
//   * LM:  right-looking Cholesky of A + lam D with lane i holding row i of L
//         in registers (pivot columns travel by shuffles), triangular solves
//         as warp-wide axpys, the rejection loop and terminations of
//         solver.solve, warp-uniform control flow.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kop_kernels.cuh"
#include "kop_tree.cuh"

namespace kop {

// Per-warp shared memory for NE end-effector slots (ne <= NE; the unused
// slots are zero).  The FK frames, Pluecker axes and the Jacobian mirror live
// only inside an evaluation (in that order, each pair overlapping once the
// first is dead), L only inside a solve, so they share storage.
// A(i, j), i >= j: column j holds rows j .. 31 (lane i reads column j at
// consecutive addresses: conflict-free)
constexpr int kTreePacked = 32 * 33 / 2;
__host__ __device__ constexpr int tree_pa(int i, int j) { return j * 32 - j * (j - 1) / 2 + (i - j); }
template <typename T, int NE>
struct TreeScratch {
  T q[32], qn[32];
  T bs[8], bn[8];            // base variable: current / candidate (SE(2): angle, x, y; SE(3): wxyz, xyz)
  T cb[2][32];               // Cholesky pivot column, double-buffered (16-byte aligned rows)
  T dg[32];                  // undamped diagonal of A (A's diagonal holds the damped one during a solve)
  T ee[NE][48];              // per EE: r[6], R^T[9], p[3], At[9], Bt[9], Ab[9]
  T A[kTreePacked];          // lower triangle of J^T J, packed by columns (tree_pa)
  union {
    struct {
      union {
        T fb[kTreeMaxJoints][7];  // FK ping-pong buffer, then
        T am[kTreeMaxJoints][6];  // the Pluecker axis of each moving tree joint
      };
      union {
        T wf[kTreeMaxJoints][7];  // world frame after each joint's motion (wxyz, xyz), then
        T J[6 * NE][32];          // the Jacobian (formed after the end-effector frames are read)
      };
    };
    T L[32 * 33];
  };
};

// Per-joint / per-column tables staged in shared memory once per CTA: lanes
// index them by different joints, which the constant bank would serialise.
template <typename T>
struct TreeTable {
  T oq[kTreeMaxJoints][4], op[kTreeMaxJoints][3], axis[kTreeMaxJoints][3];
  T mult[kTreeMaxJoints], offset[kTreeMaxJoints];
  T lower[kTreeMaxDofs], upper[kTreeMaxDofs], rest[kTreeMaxDofs];
  int32_t parent[kTreeMaxJoints], kind[kTreeMaxJoints], qcol[kTreeMaxJoints];
  int32_t col_nj[kTreeMaxDofs];
  int8_t lev_joint[kTreeMaxJoints];
  int8_t anc[6][kTreeMaxJoints];  // ancestor joint 2^r levels up (-1: past the root)
  int8_t col_joint[kTreeMaxDofs][kTreeMaxPerCol];
};

template <typename T>
__device__ __forceinline__ void stage_tree_table(const TreeLmParams<T>& P, TreeTable<T>& Q) {
  for (int j = threadIdx.x; j < P.nj; j += blockDim.x) {
    for (int i = 0; i < 4; ++i) Q.oq[j][i] = P.oq[j][i];
    for (int i = 0; i < 3; ++i) {
      Q.op[j][i] = P.op[j][i];
      Q.axis[j][i] = P.axis[j][i];
    }
    Q.mult[j] = P.mult[j];
    Q.offset[j] = P.offset[j];
    Q.parent[j] = P.parent_joint[j];
    Q.kind[j] = P.kind[j];
    Q.qcol[j] = P.qcol[j];
    Q.lev_joint[j] = P.lev_joint[j];
    int a = j;
    for (int r = 0; r < 6; ++r) {  // a: 2^(r-1) levels up -> 2^r levels up
      for (int st = 0; st < (r ? 1 << (r - 1) : 1) && a >= 0; ++st) a = P.parent_joint[a];
      Q.anc[r][j] = (int8_t)a;
    }
  }
  for (int c = threadIdx.x; c < P.n; c += blockDim.x) {
    Q.lower[c] = P.lower[c];
    Q.upper[c] = P.upper[c];
    Q.rest[c] = P.rest[c];
    Q.col_nj[c] = P.col_nj[c];
    for (int i = 0; i < kTreeMaxPerCol; ++i) Q.col_joint[c][i] = P.col_joint[c][i];
  }
}

__device__ __forceinline__ float shfl_t(float v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ double shfl_t(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = tmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// four consecutive shared-memory values (16-byte aligned for float, 32 for
// double): one LDS.128 (two for double) instead of four scalar loads
__device__ __forceinline__ void ld4(const float* p, float (&v)[4]) {
  const float4 t = *reinterpret_cast<const float4*>(p);
  v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
}
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  const double2 a = reinterpret_cast<const double2*>(p)[0], b = reinterpret_cast<const double2*>(p)[1];
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// Evaluate the stack at S.q (or S.qn when cand): returns the cost (all lanes);
// JAC also forms A (S.A, packed lower triangle) and g (register, lane i = g_i).
// root frame of the tree: the base variable's pose (Transform2.to_transform3 for
// SE(2), liegroups.py:450-454) or the identity
template <typename T>
__device__ __forceinline__ void base_frame(int kind, const T* base, quat<T>& bq, vec3<T>& bp) {
  if (kind == 1) {
    T s, c;
    sincos_t(T(0.5) * base[0], &s, &c);
    bq = {c, T(0), T(0), s};
    bp = {base[1], base[2], T(0)};
  } else if (kind == 2) {
    bq = {base[0], base[1], base[2], base[3]};
    bp = {base[4], base[5], base[6]};
  } else {
    bq = {T(1), T(0), T(0), T(0)};
    bp = {T(0), T(0), T(0)};
  }
}

// JAC (warp-uniform) selects the Jacobian / normal-equation part at run time, so
// a caller with one evaluation site carries one inlined copy of the code
template <typename T, int NE>
__device__ __forceinline__ T tree_eval(const TreeLmParams<T>& P, const TreeTable<T>& Q,
                                       const double* __restrict__ targets, TreeScratch<T, NE>& S, const T* q,
                                       const T* base, int lane, T& g_out, const bool JAC) {
  const int n = P.n, ne = P.ne, nd = n + base_dim(P.base_kind);
  quat<T> bq;
  vec3<T> bp;
  base_frame(P.base_kind, base, bq, bp);
#ifndef KOP_TREE_FK_LEVELS
  // ---- FK by pointer jumping over the tree: world frame after every joint ------
  // after(j) = after(parent) * O_j * Mot_j (robot.py:404-448).  Every joint's
  // local transform X_j = O_j Mot_j at once (lanes j, j + 32); round r then
  // composes each partial product with the one 2^r levels up the tree, so
  // after ceil(log2(depth)) rounds joint j holds root -> after(j): log2(depth)
  // warp-wide rounds instead of depth-many levels of a few lanes each.  (The
  // products associate differently from a root-to-leaf walk: rounding only.)
  {
    const int nj = P.nj;
    const int R = P.nlev > 1 ? 32 - __clz(P.nlev - 1) : 0;
    T* const fbuf[2] = {&S.wf[0][0], &S.fb[0][0]};
    int cur = R & 1;  // the last round writes wf
    for (int j = lane; j < nj; j += 32) {
      const quat<T> oq{Q.oq[j][0], Q.oq[j][1], Q.oq[j][2], Q.oq[j][3]};
      quat<T> xq = oq;
      vec3<T> xp{Q.op[j][0], Q.op[j][1], Q.op[j][2]};
      if (Q.kind[j] != 0) {
        const vec3<T> ax{Q.axis[j][0], Q.axis[j][1], Q.axis[j][2]};
        const T th = q[Q.qcol[j]] * Q.mult[j] + Q.offset[j];
        if (Q.kind[j] == 1) {
          T sn, cs;
          sincos_t(T(0.5) * th, &sn, &cs);
          xq = qmul(oq, quat<T>{cs, sn * ax.x, sn * ax.y, sn * ax.z});
        } else {
          const vec3<T> t = qrot(oq, ax);
          xp = {xp.x + th * t.x, xp.y + th * t.y, xp.z + th * t.z};
        }
      }
      T* d = fbuf[cur] + 7 * j;
      d[0] = xq.w; d[1] = xq.x; d[2] = xq.y; d[3] = xq.z;
      d[4] = xp.x; d[5] = xp.y; d[6] = xp.z;
    }
    __syncwarp();
    for (int r = 0; r < R; ++r) {
      const T* src = fbuf[cur];
      T* dst = fbuf[cur ^ 1];
      for (int j = lane; j < nj; j += 32) {
        const T* o = src + 7 * j;
        quat<T> wq{o[0], o[1], o[2], o[3]};
        vec3<T> wp{o[4], o[5], o[6]};
        const int a = Q.anc[r][j];
        if (a >= 0) {  // (A_a) o (A_j)
          const T* u = src + 7 * a;
          const quat<T> uq{u[0], u[1], u[2], u[3]};
          const vec3<T> t = qrot(uq, wp);
          wp = {u[4] + t.x, u[5] + t.y, u[6] + t.z};
          wq = qmul(uq, wq);
        }
        T* d = dst + 7 * j;
        d[0] = wq.w; d[1] = wq.x; d[2] = wq.y; d[3] = wq.z;
        d[4] = wp.x; d[5] = wp.y; d[6] = wp.z;
      }
      cur ^= 1;
      __syncwarp();
    }
    // the base pose, then the Pluecker axis (a, m = a x o) of each moving joint:
    // its axis is invariant under its own motion and a x (th a) = 0, so both come
    // from the frame after the motion
    for (int j = lane; j < nj; j += 32) {
      T* w = &S.wf[j][0];
      quat<T> wq{w[0], w[1], w[2], w[3]};
      vec3<T> wp{w[4], w[5], w[6]};
      if (P.base_kind != 0) {
        const vec3<T> t = qrot(bq, wp);
        wp = {bp.x + t.x, bp.y + t.y, bp.z + t.z};
        wq = qmul(bq, wq);
        w[0] = wq.w; w[1] = wq.x; w[2] = wq.y; w[3] = wq.z;
        w[4] = wp.x; w[5] = wp.y; w[6] = wp.z;
      }
      if (JAC && Q.kind[j] != 0) {
        const vec3<T> a = qrot(wq, vec3<T>{Q.axis[j][0], Q.axis[j][1], Q.axis[j][2]});
        const vec3<T> m = cross(a, wp);
        S.am[j][0] = a.x; S.am[j][1] = a.y; S.am[j][2] = a.z;
        S.am[j][3] = m.x; S.am[j][4] = m.y; S.am[j][5] = m.z;
      }
    }
    __syncwarp();
  }
#else
  // ---- FK, level by level: world frame after every joint, Pluecker axes -------
  // after(j) = after(parent) * O_j * Mot_j (robot.py:404-448 composition)
  for (int d = 0; d < P.nlev; ++d) {
    for (int idx = P.lev_start[d] + lane; idx < P.lev_start[d + 1]; idx += 32) {
      const int j = Q.lev_joint[idx], pj = Q.parent[j];
      quat<T> wq = bq;
      vec3<T> wp = bp;
      if (pj >= 0) {
        wq = {S.wf[pj][0], S.wf[pj][1], S.wf[pj][2], S.wf[pj][3]};
        wp = {S.wf[pj][4], S.wf[pj][5], S.wf[pj][6]};
      }
      const vec3<T> t = qrot(wq, vec3<T>{Q.op[j][0], Q.op[j][1], Q.op[j][2]});
      wp = {wp.x + t.x, wp.y + t.y, wp.z + t.z};
      wq = qmul(wq, quat<T>{Q.oq[j][0], Q.oq[j][1], Q.oq[j][2], Q.oq[j][3]});
      if (Q.kind[j] != 0) {
        const vec3<T> ax{Q.axis[j][0], Q.axis[j][1], Q.axis[j][2]};
        const vec3<T> a = qrot(wq, ax);
        if (JAC) {
          const vec3<T> m = cross(a, wp);
          S.am[j][0] = a.x; S.am[j][1] = a.y; S.am[j][2] = a.z;
          S.am[j][3] = m.x; S.am[j][4] = m.y; S.am[j][5] = m.z;
        }
        const T th = q[Q.qcol[j]] * Q.mult[j] + Q.offset[j];
        if (Q.kind[j] == 1) {
          T sn, cs;
          sincos_t(T(0.5) * th, &sn, &cs);
          wq = qmul(wq, quat<T>{cs, sn * ax.x, sn * ax.y, sn * ax.z});
        } else {
          wp = {wp.x + th * a.x, wp.y + th * a.y, wp.z + th * a.z};
        }
      }
      S.wf[j][0] = wq.w; S.wf[j][1] = wq.x; S.wf[j][2] = wq.y; S.wf[j][3] = wq.z;
      S.wf[j][4] = wp.x; S.wf[j][5] = wp.y; S.wf[j][6] = wp.z;
    }
    __syncwarp();
  }
#endif
  // ---- EE frames, pose residuals, Jr^-1 blocks ----------------------------------
  T cost_part = T(0);
  if (lane < ne) {
    quat<T> wq = bq;
    vec3<T> wp = bp;
    const int ej = P.ee_joint[lane];
    if (ej >= 0) {
      wq = {S.wf[ej][0], S.wf[ej][1], S.wf[ej][2], S.wf[ej][3]};
      wp = {S.wf[ej][4], S.wf[ej][5], S.wf[ej][6]};
    }
    {  // folded fixed joints between that frame and the link (identity: exact no-op)
      const vec3<T> t = qrot(wq, vec3<T>{P.ee_op[lane][0], P.ee_op[lane][1], P.ee_op[lane][2]});
      wp = {wp.x + t.x, wp.y + t.y, wp.z + t.z};
      wq = qmul(wq, quat<T>{P.ee_oq[lane][0], P.ee_oq[lane][1], P.ee_oq[lane][2], P.ee_oq[lane][3]});
    }
    const double* tp = targets + 7 * lane;
    const TargetInv<T> tg = target_inverse_t<T>(tp);
    const quat<T> e_q = qmul(tg.q, wq);
    const vec3<T> et = qrot(tg.q, wp);
    const Twist<T> xi = se3_log(e_q, vec3<T>{tg.t.x + et.x, tg.t.y + et.y, tg.t.z + et.z});
    const T wpos = P.w_pos[lane], wori = P.w_ori[lane];
    T* E = S.ee[lane];
    E[0] = wpos * xi.v.x; E[1] = wpos * xi.v.y; E[2] = wpos * xi.v.z;
    E[3] = wori * xi.phi.x; E[4] = wori * xi.phi.y; E[5] = wori * xi.phi.z;
    for (int m = 0; m < 6; ++m) cost_part += E[m] * E[m];
    if (JAC) {
      const mat3<T> R = qmat(wq);
      for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) E[6 + 3 * i + k] = R.m[k][i];  // R^T
      E[15] = wp.x; E[16] = wp.y; E[17] = wp.z;
      const JrInv<T> jr = se3_jr_inv(xi);
      for (int i = 0; i < 3; ++i)
        for (int k = 0; k < 3; ++k) {
          E[18 + 3 * i + k] = wpos * jr.A.m[i][k];
          E[27 + 3 * i + k] = wpos * jr.B.m[i][k];
          E[36 + 3 * i + k] = wori * jr.A.m[i][k];
        }
    }
  }
  // ---- limit / rest rows (lane i owns joint i) ----------------------------------
  T rl = T(0), gl = T(0), rr = T(0);
  if (lane < n) {
    const T qi = q[lane];
    rl = P.w_lim * (tmax(T(0), qi - Q.upper[lane]) + tmax(T(0), Q.lower[lane] - qi));
    gl = P.w_lim * ((qi > Q.upper[lane] ? T(1) : T(0)) + (qi < Q.lower[lane] ? T(-1) : T(0)));
    rr = P.w_rest * (qi - Q.rest[lane]);
    cost_part += rl * rl + rr * rr;
  }
  const T cost = warp_sum(cost_part);
  if (!JAC) return cost;
  __syncwarp();
  // ---- Jacobian column `lane` -----------------------------------------------------
  T col[6 * NE];
#pragma unroll
  for (int m = 0; m < 6 * NE; ++m) col[m] = T(0);
  // columns: lane c < n owns actuated column c (its moving joints via col_joint); lanes n .. nd-1
  // the base tangent, which acts like virtual joints at the root frame B -- prismatic along B's
  // axes (translation components), revolute about B's axes through B's origin (rotation
  // components): the body column Ad(FK^-1) e_i of costs.py:140-146 (SE(2): x, y, and z-rotation)
  const int nvirt = lane >= n && lane < nd ? 1 : 0;
  const int ncj = lane < n ? Q.col_nj[lane] : nvirt;
  for (int cj = 0; cj < ncj; ++cj) {
    int j = -1, vk = 0;
    vec3<T> a, mm;
    T mu = T(1);
    if (lane < n) {
      j = Q.col_joint[lane][cj];
      a = {S.am[j][0], S.am[j][1], S.am[j][2]};
      mm = {S.am[j][3], S.am[j][4], S.am[j][5]};
      mu = Q.mult[j];
      vk = Q.kind[j];
    } else {
      const int c = lane - n;
      const int comp = P.base_kind == 1 ? (c == 2 ? 5 : c) : c;  // se(3) component of the tangent column
      const vec3<T> ei{comp % 3 == 0 ? T(1) : T(0), comp % 3 == 1 ? T(1) : T(0), comp % 3 == 2 ? T(1) : T(0)};
      a = qrot(bq, ei);
      mm = cross(a, bp);
      vk = comp < 3 ? 2 : 1;
    }
    {
#pragma unroll
      for (int e = 0; e < NE; ++e) {
        if (e >= ne || (j >= 0 && !((P.anc_ee[e] >> j) & 1ull))) continue;
        const T* E = S.ee[e];
        vec3<T> lw, aw;
        if (vk == 1) {
          const vec3<T> pe{E[15], E[16], E[17]};
          const vec3<T> x = cross(a, pe);
          lw = {x.x - mm.x, x.y - mm.y, x.z - mm.z};
          aw = a;
        } else {
          lw = a;
          aw = {T(0), T(0), T(0)};
        }
        // body column = R^T [lw; aw]
        const vec3<T> lb{E[6] * lw.x + E[7] * lw.y + E[8] * lw.z, E[9] * lw.x + E[10] * lw.y + E[11] * lw.z,
                         E[12] * lw.x + E[13] * lw.y + E[14] * lw.z};
        const vec3<T> ab{E[6] * aw.x + E[7] * aw.y + E[8] * aw.z, E[9] * aw.x + E[10] * aw.y + E[11] * aw.z,
                         E[12] * aw.x + E[13] * aw.y + E[14] * aw.z};
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          col[6 * e + i] += mu * (E[18 + 3 * i] * lb.x + E[19 + 3 * i] * lb.y + E[20 + 3 * i] * lb.z +
                                  E[27 + 3 * i] * ab.x + E[28 + 3 * i] * ab.y + E[29 + 3 * i] * ab.z);
          col[6 * e + 3 + i] += mu * (E[36 + 3 * i] * ab.x + E[37 + 3 * i] * ab.y + E[38 + 3 * i] * ab.z);
        }
      }
    }
  }
#pragma unroll
  for (int m = 0; m < 6 * NE; ++m) S.J[m][lane] = col[m];
  __syncwarp();
  // ---- normal equations: lane i forms row i ----------------------------------------
  T g = T(0);
  if (lane < nd) {
    for (int j4 = 0; j4 < nd; j4 += 4) {  // four columns of J per vector load; unused slots are zero
      T a[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int m = 0; m < 6 * NE; ++m) {
        T v[4];
        ld4(&S.J[m][j4], v);
#pragma unroll
        for (int t = 0; t < 4; ++t) a[t] += col[m] * v[t];
      }
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (j4 + t <= lane) S.A[tree_pa(lane, j4 + t)] = a[t];  // rows >= n: zero, unread
    }
    if (lane < n) S.A[tree_pa(lane, lane)] += gl * gl + P.w_rest * P.w_rest;
    S.dg[lane] = S.A[tree_pa(lane, lane)];
#pragma unroll
    for (int m = 0; m < 6 * NE; ++m) g += col[m] * S.ee[m / 6][m % 6];
    g += gl * rl + P.w_rest * rr;  // zero on base lanes
  }
  g_out = g;
  __syncwarp();
  return cost;
}

// delta (lane i -> d_i) = -(A + lam diag(max(diag A, 1e-8)))^-1 g; false if a pivot fails
template <typename T, int NE>
__device__ __forceinline__ bool tree_damped_solve(const TreeLmParams<T>& P, TreeScratch<T, NE>& S, T g, T lam,
                                                  int lane, T& delta) {
  // right-looking Cholesky with lane i holding row i of L in registers; the
  // scaled pivot column is published once per step in shared memory and read
  // back as vector broadcasts.  Lanes update their whole row: the entries
  // right of the diagonal are never read, so no per-entry lane test.
  const int n = P.n + base_dim(P.base_kind);  // the tangent: actuated columns, then the base's
  if (lane < n) S.A[tree_pa(lane, lane)] = S.dg[lane] + lam * tmax(S.dg[lane], T(BeamConsts::diag_clamp));
  __syncwarp();
  T row[kTreeMaxDofs];  // entries right of the diagonal start at zero (never read)
#pragma unroll
  for (int j = 0; j < kTreeMaxDofs; ++j) row[j] = (lane < n && j < n && j <= lane) ? S.A[tree_pa(lane, j)] : T(0);
  bool ok = true;
  T dinv_mine = T(0);
  // forward substitution y = L^-1 (-g) carried along: lane k's y is final
  // when column k is factored
  T y = -g;
#pragma unroll
  for (int k = 0; k < kTreeMaxDofs; ++k) {
    if (k < n) {  // warp-uniform
      const T dk = shfl_t(row[k], k);
      const T yr = shfl_t(y, k);
      ok = ok && (dk > T(0)) && finite_t(dk);
      const T inv = rsqrt_t(dk);
      row[k] *= inv;  // lane k: dk * inv = L(k, k); lanes > k: L(lane, k)
      if (lane == k) dinv_mine = inv;
      const T yk = yr * inv;
      if (lane == k) y = yk;
      if (lane > k && lane < n) y -= row[k] * yk;
      T* cb = S.cb[k & 1];  // the buffer of step k - 2 is free: every lane passed step k - 1's sync
      cb[lane] = row[k];    // rows / lanes >= n are zero
      __syncwarp();
#pragma unroll
      for (int j4 = (k + 1) & ~3; j4 < kTreeMaxDofs; j4 += 4) {
        T l[4];
        ld4(cb + j4, l);
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (j4 + t > k) row[j4 + t] -= row[k] * l[t];
      }
    }
  }
  if (lane < n) {  // L(lane, j) for the backward sweep
#pragma unroll
    for (int j = 0; j < kTreeMaxDofs; ++j)
      if (j < lane && j < n) S.L[j * 33 + lane] = row[j];
    S.L[lane * 33 + lane] = dinv_mine;  // the diagonal slot carries 1 / L(lane, lane)
  }
  __syncwarp();
  // backward: x = L^-T y, two rows per step: every lane forms x_k and x_{k-1}
  // from lanes k, k-1 (the same operations as row-by-row), so the serial
  // chain is one shuffle round per two rows
  T x = y;
  int k = n - 1;
  for (; k >= 1; k -= 2) {
    const T lkk = S.L[(k - 1) * 33 + k], dk1 = S.L[(k - 1) * 33 + k - 1];  // L(k, k-1), 1 / L(k-1, k-1)
    const T lk = lane < k ? S.L[lane * 33 + k] : T(0), lk1 = lane < k - 1 ? S.L[lane * 33 + k - 1] : T(0);
    const T xk = shfl_t(x * dinv_mine, k), xr = shfl_t(x, k - 1);
    const T xk1 = (xr - lkk * xk) * dk1;
    if (lane == k) x = xk;
    if (lane == k - 1) x = xk1;
    if (lane < k - 1) x = x - lk * xk - lk1 * xk1;  // L[k][lane], L[k-1][lane]
  }
  if (k == 0) {
    const T x0 = shfl_t(x * dinv_mine, 0);
    if (lane == 0) x = x0;
  }
  delta = lane < n ? x : T(0);
  return ok;
}

// warps per CTA: FP32 runs one-warp CTAs (a finished problem frees its slot at
// once); FP64 keeps four (measured faster: register-limited residency)
#ifndef KOP_TREE_WARPS32
#define KOP_TREE_WARPS32 1
#endif
#ifndef KOP_TREE_WARPS64
#define KOP_TREE_WARPS64 4
#endif
template <typename T>
constexpr int tree_warps() { return sizeof(T) == 4 ? KOP_TREE_WARPS32 : KOP_TREE_WARPS64; }

// IK-Beam stage 1 runs a fixed step count (no early exit), so its warps finish
// together and share one staged table per CTA: 8 warps (FP32) / 6 (FP64) per
// CTA fill the SM's shared memory with 24 / 12 resident warps (measured +10% /
// +7% over 4-warp CTAs at 100K humanoid targets)
#ifndef KOP_TREE_BEAM_WARPS32
#define KOP_TREE_BEAM_WARPS32 8
#endif
#ifndef KOP_TREE_BEAM_WARPS64
#define KOP_TREE_BEAM_WARPS64 6
#endif
#ifndef KOP_TREE_S2_TARGETS32
#define KOP_TREE_S2_TARGETS32 2
#endif
template <typename T>
constexpr int tree_beam_warps() { return sizeof(T) == 4 ? KOP_TREE_BEAM_WARPS32 : KOP_TREE_BEAM_WARPS64; }

// canonical unit quaternion (quat_normalize_canonical, liegroups.py:33-46)
template <typename T>
__device__ __forceinline__ quat<T> canon_t(quat<T> q) {
  const T inv = T(1) / sqrt_t(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  q = {q.w * inv, q.x * inv, q.y * inv, q.z * inv};
  T sign = q.w < T(0) ? T(-1) : T(1);
  if (q.w == T(0)) {
    const T ax = fabs(q.x), ay = fabs(q.y), az = fabs(q.z);
    const T lead = (ax >= ay && ax >= az) ? q.x : (ay >= az ? q.y : q.z);
    sign = lead < T(0) ? T(-1) : T(1);
  }
  return {q.w * sign, q.x * sign, q.y * sign, q.z * sign};
}

// base <- base * exp(delta): Transform2.compose(Transform2.exp) (liegroups.py:431-445; the SE(2) state
// is (angle, x, y)) or Transform3.compose(Transform3.exp) (liegroups.py:379-390, se3_exp_arrays :194-200;
// state (wxyz, xyz)), i.e. local_update (liegroups.py:505-519) of the base variable
template <typename T>
__device__ __forceinline__ void tree_base_retract(int kind, const T* b, const T (&d)[6], T* out) {
  if (kind == 1) {
    const T cur[3] = {b[1], b[2], b[0]};
    T nxt[3];
    base_retract(cur, d[0], d[1], d[2], nxt);
    out[0] = nxt[2];
    out[1] = nxt[0];
    out[2] = nxt[1];
    return;
  }
  const vec3<T> rho{d[0], d[1], d[2]}, phi{d[3], d[4], d[5]};
  const T t2 = dot(phi, phi), th = sqrt_t(t2);
  const bool small = th < T(1e-7);
  T sh, ch, s1, c1;
  sincos_t(T(0.5) * th, &sh, &ch);
  sincos_t(th, &s1, &c1);
  const T k = small ? T(0.5) - t2 / T(48) : sh / th;
  const quat<T> qe = canon_t(quat<T>{ch, k * phi.x, k * phi.y, k * phi.z});
  const T a = small ? T(0.5) - t2 / T(24) : (T(1) - c1) / t2;
  const T bb = small ? T(1) / T(6) - t2 / T(120) : (th - s1) / (t2 * th);
  const vec3<T> pr = cross(phi, rho), ppr = cross(phi, pr);
  const vec3<T> v{rho.x + a * pr.x + bb * ppr.x, rho.y + a * pr.y + bb * ppr.y, rho.z + a * pr.z + bb * ppr.z};
  const quat<T> qb{b[0], b[1], b[2], b[3]};
  const quat<T> qn = canon_t(qmul(qb, qe));
  const vec3<T> tv = qrot(qb, v);
  out[0] = qn.w; out[1] = qn.x; out[2] = qn.y; out[3] = qn.z;
  out[4] = b[4] + tv.x; out[5] = b[5] + tv.y; out[6] = b[6] + tv.z;
}

template <typename T, int NE>
__global__ void __launch_bounds__(32 * tree_warps<T>())
k_tree_solve(const TreeLmParams<T> P, const double* __restrict__ targets, const double* __restrict__ q0, int64_t B,
             const LmOptions O, double* __restrict__ q_out, double* __restrict__ cost_out,
             double* __restrict__ init_cost_out, double* __restrict__ hist_out, int32_t* __restrict__ iters_out,
             int32_t* __restrict__ term_out, const double* __restrict__ base0, double* __restrict__ base_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  TreeTable<T>& Q = *reinterpret_cast<TreeTable<T>*>(smem_raw);
  TreeScratch<T, NE>& S =
      reinterpret_cast<TreeScratch<T, NE>*>(smem_raw + (sizeof(TreeTable<T>) + 15) / 16 * 16)[wib];
  stage_tree_table(P, Q);
  __syncthreads();      // the only CTA-wide barrier: warps are independent from here on
  if (b >= B) return;  // whole warp exits together
  const int n = P.n, nd = n + base_dim(P.base_kind), bsz = base_state(P.base_kind);
  for (int i = lane; i < NE * 48; i += 32) (&S.ee[0][0])[i] = T(0);  // unused slots stay zero
  const double* tg = targets + b * 7 * P.ne;
  S.q[lane] = lane < n ? T(q0[b * n + lane]) : T(0);
  if (lane < 8) S.bs[lane] = lane < bsz ? T(base0[b * bsz + lane]) : T(0);
  __syncwarp();
  T g, cost = T(0);
  const int hstride = O.max_iterations + 1;
  int term = 0;
  int iters = 0;
  T damping = T(O.damping0);
  // ONE evaluation site for both kinds -- J at the iterate (the start evaluation
  // and each accepted iterate) or the candidate's cost in the rejection loop --
  // selected at run time: a single inlined copy keeps the kernel's hot code
  // inside the instruction cache.  The control flow is solver.solve's
  // (solver.py:381-419): per iteration a gradient test, then damped trials
  // until one decreases the cost (x down) or the damping / rejection budget
  // runs out (x up per rejected or failed trial).
  bool jac = true;  // next evaluation: J at the iterate
  int it = 0, rj = 0;
  T dg = T(0), d = T(0);
  for (;;) {
    if (!jac) {  // a damped trial from the iterate
      bool ok = tree_damped_solve(P, S, g, damping, lane, d);
      ok = __all_sync(0xffffffffu, ok && finite_t(d));
      if (ok) {
        S.qn[lane] = S.q[lane] + d;
        if (bsz) {  // the base moves by its own retraction (local_update)
          T db[6];
#pragma unroll
          for (int c = 0; c < 6; ++c) db[c] = shfl_t(d, n + c < 32 ? n + c : 31);
          if (lane == 0) tree_base_retract(P.base_kind, S.bs, db, S.bn);
        }
        __syncwarp();
      } else {  // a failed factorisation is a rejected trial without an evaluation
        damping *= T(O.up);
        if (damping > T(BeamConsts::damping_max) || ++rj >= O.max_rejections) {
          term = damping > T(BeamConsts::damping_max) ? 3 : 4;
          break;
        }
        continue;
      }
    }
    T gd;
    const T c = tree_eval<T, NE>(P, Q, tg, S, jac ? S.q : S.qn, jac ? S.bs : S.bn, lane, jac ? g : gd, jac);
    if (jac) {
      if (it == 0) {
        cost = c;
        if (lane == 0) {
          if (hist_out) hist_out[b * hstride] = double(cost);
          init_cost_out[b] = double(cost);
        }
        term = finite_t(cost) ? 0 : 5;
      }
      if (term != 0 || it >= O.max_iterations) break;
      if (warp_max(lane < nd ? fabs(g) : T(0)) < T(O.grad_tol)) {
        term = 1;
        break;
      }
      // diag of J^T J at the iterate (lane i), for the FP32 rule's model decrease
      dg = lane < nd ? tmax(S.dg[lane], T(BeamConsts::diag_clamp)) : T(0);
      if (O.max_rejections <= 0) {  // no trial allowed
        term = damping > T(BeamConsts::damping_max) ? 3 : 4;
        break;
      }
      rj = 0;
      jac = false;
      continue;
    }
    if (!finite_t(c)) {
      term = 5;
      break;
    }
    if (c < cost) {  // accepted
      S.q[lane] = S.qn[lane];
      if (lane < bsz) S.bs[lane] = S.bn[lane];
      cost = c;
      damping = tmax(damping * T(O.down), T(BeamConsts::damping_min));
      __syncwarp();
      ++iters;
      if (lane == 0 && hist_out) hist_out[b * hstride + iters] = double(cost);
      if (warp_max(fabs(d)) < T(O.step_tol)) {
        term = 2;
        break;
      }
      ++it;
      jac = true;
      continue;
    }
    // FP32 rule (kop_collision.cu kFp32Tau): a rejected trial whose quadratic-model decrease
    // -g.d + lam d^T D d is below 2^-17 of the cost is not resolvable in float32
    if (sizeof(T) == 4 && warp_sum(lane < nd ? damping * dg * d * d - g * d : T(0)) <=
                              T(7.62939453125e-6f) * cost) {
      term = 6;
      break;
    }
    damping *= T(O.up);
    if (damping > T(BeamConsts::damping_max) || ++rj >= O.max_rejections) {
      term = damping > T(BeamConsts::damping_max) ? 3 : 4;
      break;
    }
  }
  if (hist_out)
    for (int i = iters + 1 + lane; i < hstride; i += 32) hist_out[b * hstride + i] = NAN;
  if (lane < n) q_out[b * n + lane] = double(S.q[lane]);
  if (lane < bsz && base_out) base_out[b * bsz + lane] = double(S.bs[lane]);
  if (lane == 0) {
    cost_out[b] = double(cost);
    iters_out[b] = iters;
    term_out[b] = term;
  }
}

template <typename T, int NE>
cudaError_t launch_tree_ne(const TreeLmParams<T>& P, const TreeLaunch& L, cudaStream_t st) {
  constexpr int warps = tree_warps<T>();
  const size_t smem = (sizeof(TreeTable<T>) + 15) / 16 * 16 + sizeof(TreeScratch<T, NE>) * warps;
  cudaFuncSetAttribute(k_tree_solve<T, NE>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_tree_solve<T, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tree_solve<T, NE><<<(unsigned)((L.B + warps - 1) / warps), 32 * warps, smem, st>>>(
      P, L.targets, L.q0, L.B, L.opts, L.q_out, L.cost_out, L.init_cost, L.hist_out, L.iters, L.term, L.base0,
      L.base_out);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_tree_solve(const TreeLmParams<T>& P, const TreeLaunch& L, cudaStream_t st) {
  if (L.B == 0) return cudaSuccess;
  if (P.ne <= 1) return launch_tree_ne<T, 1>(P, L, st);
  if (P.ne <= 2) return launch_tree_ne<T, 2>(P, L, st);
  if (P.ne <= 4) return launch_tree_ne<T, 4>(P, L, st);
  return launch_tree_ne<T, kTreeMaxPoses>(P, L, st);
}

template cudaError_t launch_tree_solve<float>(const TreeLmParams<float>&, const TreeLaunch&, cudaStream_t);
template cudaError_t launch_tree_solve<double>(const TreeLmParams<double>&, const TreeLaunch&, cudaStream_t);

// ---------------------------------------------------------------------------
// Multi-end-effector IK-Beam ("beam-style lanes
// generalised to K pose blocks"): the lane LM of beam.py:198-240 (one proposal
// per step, per-lane accept / damping x1/3 | x10) and the tasks.py:119-161
// beam control flow, over the tree residual [pose_1..pose_K | limit | rest].
// One warp per lane, as in the tree solve.
// ---------------------------------------------------------------------------

// `steps` beam.py proposals from S.q (beam.py:198-240).  One J-evaluation
// site: the start evaluation (cost = start_state's when `start`, else the
// carried `cost`) and, after an accepted step that is not the last, J at the
// accepted iterate (beam.py:202) -- one inlined copy of the evaluation keeps
// the kernel inside the instruction cache.  Lane h0 + it keeps the cost after
// step it in hv (and lane 0 the start cost when `start`).
template <typename T, int NE>
__device__ __forceinline__ T tree_beam_run(const TreeLmParams<T>& P, const TreeTable<T>& Q,
                                           const double* __restrict__ tg, TreeScratch<T, NE>& S, int lane,
                                           int steps, bool start, T cost, T& lam, int h0, T& hv) {
  // one evaluation site for both kinds (J at the iterate, cost at the candidate):
  // a single inlined copy of the evaluation keeps the kernel's hot code smaller
  T g = T(0);
  bool need = true;  // J-evaluation at S.q pending
  for (int it = 0;;) {
    if (!need && it == steps) break;
    T cn = inf_t<T>();
    bool eval = true;
    if (!need) {
      T d;
      bool ok = tree_damped_solve(P, S, g, lam, lane, d);
      ok = __all_sync(0xffffffffu, ok && finite_t(d));
      if (ok) {  // a failed factorisation rejects the step (beam.py:209-213, per lane)
        S.qn[lane] = S.q[lane] + d;
        __syncwarp();
      }
      eval = ok;
    }
    if (eval) {
      const T c = tree_eval<T, NE>(P, Q, tg, S, need ? S.q : S.qn, nullptr, lane, g, need);
      if (need) {
        if (start && it == 0) {
          cost = c;
          if (lane == 0) hv = c;
        }
        need = false;
        continue;
      }
      cn = finite_t(c) ? c : inf_t<T>();
    }
    if (cn < cost) {
      S.q[lane] = S.qn[lane];
      __syncwarp();
      lam = tmax(lam * T(BeamConsts::damping_down), T(BeamConsts::damping_min));
      cost = cn;
      need = it + 1 < steps;
    } else {
      lam = tmin(lam * T(BeamConsts::damping_up), T(BeamConsts::damping_max));
    }
    if (lane == h0 + it) hv = cost;
    ++it;
  }
  return cost;
}

template <typename T, int NE>
__global__ void __launch_bounds__(32 * tree_beam_warps<T>())
k_tree_beam_stage1(const TreeLmParams<T> P, const double* __restrict__ targets, int64_t B,
                   const double* __restrict__ seeds, int S, int steps1, T* __restrict__ recs) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t L = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;  // lane = target * S + seed
  TreeTable<T>& Q = *reinterpret_cast<TreeTable<T>*>(smem_raw);
  TreeScratch<T, NE>& Sc =
      reinterpret_cast<TreeScratch<T, NE>*>(smem_raw + (sizeof(TreeTable<T>) + 15) / 16 * 16)[wib];
  stage_tree_table(P, Q);
  __syncthreads();
  if (L >= B * S) return;
  const int64_t b = L / S;
  const int s = (int)(L % S), n = P.n;
  for (int i = lane; i < NE * 48; i += 32) (&Sc.ee[0][0])[i] = T(0);
  Sc.q[lane] = lane < n ? T(seeds[(size_t)s * n + lane]) : T(0);
  __syncwarp();
  const double* tg = targets + b * 7 * P.ne;
  T lam = T(BeamConsts::damping_init);
  T hv = T(0);  // lane h keeps hist[h]; start_state (beam.py:182-196) inside
  const T cost = tree_beam_run(P, Q, tg, Sc, lane, steps1, true, T(0), lam, 1, hv);
  const int rec = tree_beam_rec(n, steps1);
  T* out = recs + L * rec;  // records in the solve precision: FP64 q / damping / cost are carried exactly
  if (lane < n) out[lane] = Sc.q[lane];
  if (lane == 0) {
    out[n] = lam;
    out[n + 1] = cost;
  }
  if (lane <= steps1) out[n + 2 + lane] = hv;
}

// stable top-`keep` seeds of each target by (final stage-1 cost, seed index),
// NaN last (np.argsort(kind="stable"), tasks.py:135): one warp per target
template <typename T>
__global__ void __launch_bounds__(128)
k_tree_beam_prune(const T* __restrict__ recs, int rec, int n, int64_t B, int S, int keep,
                  int32_t* __restrict__ surv) {
  const int lane = threadIdx.x & 31;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;
  const T* base = recs + b * S * rec + n + 1;
  for (int s = lane; s < S; s += 32) {
    const T c = base[(size_t)s * rec];
    int rank = 0;
    for (int j = 0; j < S; ++j) rank += rank_less(base[(size_t)j * rec], j, c, s) ? 1 : 0;
    if (rank < keep) surv[b * keep + rank] = s;
  }
}

// FP64 world frame after tree joint j (identity for j < 0), walking up the tree
__device__ __forceinline__ void tree_frame_f64(const TreeLmParams<double>& P, const double* q, int j,
                                               quat<double>& wq, vec3<double>& wp) {
  wq = {1.0, 0.0, 0.0, 0.0};
  wp = {0.0, 0.0, 0.0};
  for (int a = j; a >= 0; a = P.parent_joint[a]) {  // (wq, wp) <- O_a Mot_a (wq, wp)
    if (P.kind[a] != 0) {
      const double th = q[P.qcol[a]] * P.mult[a] + P.offset[a];
      const vec3<double> ax{P.axis[a][0], P.axis[a][1], P.axis[a][2]};
      if (P.kind[a] == 1) {
        double sn, cs;
        sincos(0.5 * th, &sn, &cs);
        const quat<double> r{cs, sn * ax.x, sn * ax.y, sn * ax.z};
        wp = qrot(r, wp);
        wq = qmul(r, wq);
      } else {
        wp = {wp.x + th * ax.x, wp.y + th * ax.y, wp.z + th * ax.z};
      }
    }
    const quat<double> mq{P.oq[a][0], P.oq[a][1], P.oq[a][2], P.oq[a][3]};
    const vec3<double> t = qrot(mq, wp);
    wp = {t.x + P.op[a][0], t.y + P.op[a][1], t.z + P.op[a][2]};
    wq = qmul(mq, wq);
  }
}

// survivors of one target: one warp each, 10 more steps, winner = argmin
// (ties -> better stage-1 rank, tasks.py:139), outputs and FP64 pose errors
template <typename T, int NE>
__global__ void __launch_bounds__(256)
k_tree_beam_stage2(const TreeLmParams<T> P, const TreeLmParams<double> Pd, const double* __restrict__ targets,
                   int64_t B, const T* __restrict__ recs, int S, const int32_t* __restrict__ surv, int steps1,
                   int steps2, int keep, double pos_tol, double rot_tol, double* __restrict__ q_out,
                   double* __restrict__ cost_out, double* __restrict__ hist_out, double* __restrict__ pos_err,
                   double* __restrict__ rot_err, uint8_t* __restrict__ success, int tpc) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  // tpc targets per CTA (one staged table for all), `keep` warps each: warp r of
  // group grp = survivor of stage-1 rank r of target b
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, grp = w / keep, r = w - grp * keep;
  const int64_t b = (int64_t)blockIdx.x * tpc + grp;
  const bool live = b < B;
  TreeTable<T>& Q = *reinterpret_cast<TreeTable<T>*>(smem_raw);
  const size_t tab = (sizeof(TreeTable<T>) + 15) / 16 * 16;
  TreeScratch<T, NE>& Sc = reinterpret_cast<TreeScratch<T, NE>*>(smem_raw + tab)[w];
  T* wcost = reinterpret_cast<T*>(smem_raw + tab + sizeof(TreeScratch<T, NE>) * keep * tpc);
  int* wsel = reinterpret_cast<int*>(wcost + keep * tpc);
  stage_tree_table(P, Q);
  __syncthreads();
  const int n = P.n, rec = tree_beam_rec(n, steps1);
  const T* in = recs + (live ? (b * S + surv[b * keep + r]) * rec : 0);
  const double* tg = targets + (live ? b : 0) * 7 * P.ne;
  T cost = T(0), hv = T(0);  // lane h keeps stage-2 hist[h]; J re-derived, the carried cost is stage 1's
  if (live) {
    for (int i = lane; i < NE * 48; i += 32) (&Sc.ee[0][0])[i] = T(0);
    Sc.q[lane] = lane < n ? in[lane] : T(0);
    __syncwarp();
    T lam = in[n];
    cost = tree_beam_run(P, Q, tg, Sc, lane, steps2, false, in[n + 1], lam, 0, hv);
    if (lane == 0) wcost[w] = cost;
  }
  __syncthreads();
  if (live && lane == 0 && r == 0) {
    const T* wc = wcost + grp * keep;
    int best = 0;
    for (int k = 1; k < keep; ++k)
      if (wc[k] < wc[best] || (wc[best] != wc[best] && wc[k] == wc[k])) best = k;
    wsel[grp] = best;
  }
  __syncthreads();
  if (!live || r != wsel[grp]) return;
  if (lane < n) q_out[b * n + lane] = double(Sc.q[lane]);
  if (lane == 0) cost_out[b] = double(cost);
  if (hist_out) {
    double* h = hist_out + b * (steps1 + 1 + steps2);
    if (lane <= steps1) h[lane] = double(in[n + 2 + lane]);
    if (lane < steps2) h[steps1 + 1 + lane] = double(hv);
  }
  // FP64 pose errors of every end effector (tasks.py:109-116); success = all in tolerance
  double qd[kTreeMaxDofs];
  for (int i = 0; i < n; ++i) qd[i] = double(Sc.q[i]);
  bool ok = true;
  if (lane < P.ne) {
    quat<double> wq;
    vec3<double> wp;
    tree_frame_f64(Pd, qd, Pd.ee_joint[lane], wq, wp);
    const double nq = sqrt(wq.w * wq.w + wq.x * wq.x + wq.y * wq.y + wq.z * wq.z);
    wq = {wq.w / nq, wq.x / nq, wq.y / nq, wq.z / nq};
    double ti[7];
    target_inverse(tg + 7 * lane, ti);
    const quat<double> iq{ti[0], ti[1], ti[2], ti[3]};
    const quat<double> rq = qmul(iq, wq);
    const vec3<double> rt0 = qrot(iq, wp);
    const vec3<double> rt{ti[4] + rt0.x, ti[5] + rt0.y, ti[6] + rt0.z};
    const double pe = sqrt(rt.x * rt.x + rt.y * rt.y + rt.z * rt.z);
    const vec3<double> w = qlog(rq);
    const double re = sqrt(w.x * w.x + w.y * w.y + w.z * w.z);
    pos_err[b * P.ne + lane] = pe;
    rot_err[b * P.ne + lane] = re;
    ok = pe < pos_tol && re < rot_tol;
  }
  const bool all_ok = __all_sync(0xffffffffu, ok);
  if (lane == 0) success[b] = all_ok ? 1 : 0;
}

template <typename T, int NE>
cudaError_t launch_tree_beam_ne(const TreeLmParams<T>& P, const TreeLmParams<double>& Pd, const TreeBeamLaunch& L,
                                cudaStream_t st) {
  constexpr int warps = tree_beam_warps<T>();
  const size_t tab = (sizeof(TreeTable<T>) + 15) / 16 * 16;
  const int rec = tree_beam_rec(P.n, L.steps1);
  T* recs = static_cast<T*>(L.workspace);
  int32_t* surv = reinterpret_cast<int32_t*>(static_cast<char*>(L.workspace) +
                                             ((size_t)L.B * L.S * rec * sizeof(T) + 255) / 256 * 256);
  const size_t smem1 = tab + sizeof(TreeScratch<T, NE>) * warps;
  cudaFuncSetAttribute(k_tree_beam_stage1<T, NE>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (smem1 > 48 * 1024)
    cudaFuncSetAttribute(k_tree_beam_stage1<T, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  const int64_t lanes = L.B * L.S;
  k_tree_beam_stage1<T, NE><<<(unsigned)((lanes + warps - 1) / warps), 32 * warps, smem1, st>>>(
      P, L.targets, L.B, L.seeds, L.S, L.steps1, recs);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_tree_beam_prune<T><<<(unsigned)((L.B + 3) / 4), 128, 0, st>>>(recs, rec, P.n, L.B, L.S, L.keep, surv);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  // FP32: two targets per CTA (2 x keep warps share the staged table: 24 resident warps per SM
  // instead of 20 for keep = 4); FP64 scratch fills the SM either way
  const int tpc = (sizeof(T) == 4 && 2 * L.keep <= 8) ? KOP_TREE_S2_TARGETS32 : 1;
  const size_t smem2 =
      tab + sizeof(TreeScratch<T, NE>) * L.keep * tpc + (sizeof(T) + sizeof(int)) * 32 + 16;
  cudaFuncSetAttribute(k_tree_beam_stage2<T, NE>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (smem2 > 48 * 1024)
    cudaFuncSetAttribute(k_tree_beam_stage2<T, NE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  k_tree_beam_stage2<T, NE><<<(unsigned)((L.B + tpc - 1) / tpc), 32 * L.keep * tpc, smem2, st>>>(
      P, Pd, L.targets, L.B, recs, L.S, surv, L.steps1, L.steps2, L.keep, L.pos_tol, L.rot_tol, L.q_out, L.cost_out,
      L.hist_out, L.pos_err, L.rot_err, L.success, tpc);
  return cudaGetLastError();
}

template <typename T>
cudaError_t launch_tree_beam(const TreeLmParams<T>& P, const TreeLmParams<double>& Pd, const TreeBeamLaunch& L,
                             cudaStream_t st) {
  if (L.B == 0) return cudaSuccess;
  if (P.ne <= 1) return launch_tree_beam_ne<T, 1>(P, Pd, L, st);
  if (P.ne <= 2) return launch_tree_beam_ne<T, 2>(P, Pd, L, st);
  if (P.ne <= 4) return launch_tree_beam_ne<T, 4>(P, Pd, L, st);
  return launch_tree_beam_ne<T, kTreeMaxPoses>(P, Pd, L, st);
}

template cudaError_t launch_tree_beam<float>(const TreeLmParams<float>&, const TreeLmParams<double>&,
                                             const TreeBeamLaunch&, cudaStream_t);
template cudaError_t launch_tree_beam<double>(const TreeLmParams<double>&, const TreeLmParams<double>&,
                                              const TreeBeamLaunch&, cudaStream_t);

}  // namespace kop
