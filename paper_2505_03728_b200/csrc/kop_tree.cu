// Multi-end-effector IK on a kinematic TREE through the generic LM (config 3:
// humanoid, n <= 32 actuated joints): one warp per problem.
//
// Reference path: one pose_cost per end effector (costs.py:98-166) +
// limit_cost + rest_cost, solved by solver.solve (solver.py:364-429).
//
// Warp mapping (a problem is too large for one thread's registers -- a 24x29
// Jacobian, a 29x29 normal matrix):
//   * FK:  lane l computes the world frame of tree joints l and l+32 by
//         walking UP the tree (T = O_a Mot_a T for each ancestor a -- no
//         stack), leaving its Pluecker axis (a, m = a x o) in shared memory;
//         lanes e < E compute the end-effector frames the same way, then the
//         pose residual xi_e and the weighted Jr^-1(xi_e) blocks.
//   * J:   lane c owns Jacobian column c (its joint(s) via qcol), 6E entries
//         in registers, mirrored to shared memory.
//   * A:   lane i forms row i of J^T J from its own column and broadcast reads.
//   * LM:  right-looking Cholesky of A + lam D in shared memory (row stride 33,
//         conflict-free), triangular solves as warp-wide axpys, the rejection
//         loop and terminations of solver.solve, warp-uniform control flow.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kop_kernels.cuh"
#include "kop_tree.cuh"

namespace kop {

template <typename T>
struct TreeScratch {  // per-warp shared memory
  T q[32], qn[32], d[32];
  T am[kTreeMaxJoints][6];   // Pluecker axis of each moving tree joint
  T ee[kTreeMaxPoses][48];   // per EE: r[6], R^T[9], p[3], At[9], Bt[9], Ab[9]
  T J[6 * kTreeMaxPoses][32];
  T A[32 * 33];
  T L[32 * 33];
  T red[32];
};

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

// world frame AFTER the motion of tree joint j (identity for j < 0), walking up
template <typename T>
__device__ __forceinline__ void frame_after(const TreeLmParams<T>& P, const T* q, int j, quat<T>& wq, vec3<T>& wp) {
  wq = {T(1), T(0), T(0), T(0)};
  wp = {T(0), T(0), T(0)};
  for (int a = j; a >= 0; a = P.parent_joint[a]) {
    // M = O_a * Mot_a ; (wq, wp) <- M * (wq, wp)
    quat<T> mq{T(P.oq[a][0]), T(P.oq[a][1]), T(P.oq[a][2]), T(P.oq[a][3])};
    vec3<T> mp{P.op[a][0], P.op[a][1], P.op[a][2]};
    if (P.kind[a] != 0) {
      const T th = q[P.qcol[a]] * P.mult[a] + P.offset[a];
      const vec3<T> ax{P.axis[a][0], P.axis[a][1], P.axis[a][2]};
      if (P.kind[a] == 1) {
        T s, c;
        sincos_t(T(0.5) * th, &s, &c);
        // Mot * (wq, wp): rotate by (c, s ax)
        const quat<T> r{c, s * ax.x, s * ax.y, s * ax.z};
        wp = qrot(r, wp);
        wq = qmul(r, wq);
      } else {
        wp = {wp.x + th * ax.x, wp.y + th * ax.y, wp.z + th * ax.z};
      }
    }
    const vec3<T> t = qrot(mq, wp);
    wp = {t.x + mp.x, t.y + mp.y, t.z + mp.z};
    wq = qmul(mq, wq);
  }
}

// world frame BEFORE the motion of joint j (its joint frame): parent-after * O_j
template <typename T>
__device__ __forceinline__ void frame_before(const TreeLmParams<T>& P, const T* q, int j, quat<T>& wq, vec3<T>& wp) {
  frame_after(P, q, P.parent_joint[j], wq, wp);
  const vec3<T> t = qrot(wq, vec3<T>{P.op[j][0], P.op[j][1], P.op[j][2]});
  wp = {wp.x + t.x, wp.y + t.y, wp.z + t.z};
  wq = qmul(wq, quat<T>{T(P.oq[j][0]), T(P.oq[j][1]), T(P.oq[j][2]), T(P.oq[j][3])});
}

// Evaluate the stack at S.q (or S.qn when cand): returns the cost (all lanes);
// JAC also forms A (S.A, stride 33) and g (register, lane i = g_i).
template <typename T, bool JAC>
__device__ __forceinline__ T tree_eval(const TreeLmParams<T>& P, const double* __restrict__ targets,
                                       TreeScratch<T>& S, const T* q, int lane, T& g_out) {
  const int n = P.n, ne = P.ne;
  // ---- FK: Pluecker axes of the moving joints --------------------------------
  if (JAC) {
    for (int j = lane; j < P.nj; j += 32) {
      if (P.kind[j] == 0) continue;
      quat<T> wq;
      vec3<T> wp;
      frame_before(P, q, j, wq, wp);
      const vec3<T> a = qrot(wq, vec3<T>{P.axis[j][0], P.axis[j][1], P.axis[j][2]});
      const vec3<T> m = cross(a, wp);
      S.am[j][0] = a.x; S.am[j][1] = a.y; S.am[j][2] = a.z;
      S.am[j][3] = m.x; S.am[j][4] = m.y; S.am[j][5] = m.z;
    }
  }
  // ---- EE frames, pose residuals, Jr^-1 blocks ----------------------------------
  T cost_part = T(0);
  if (lane < ne) {
    quat<T> wq;
    vec3<T> wp;
    frame_after(P, q, P.ee_joint[lane], wq, wp);
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
    rl = P.w_lim * (tmax(T(0), qi - P.upper[lane]) + tmax(T(0), P.lower[lane] - qi));
    gl = P.w_lim * ((qi > P.upper[lane] ? T(1) : T(0)) + (qi < P.lower[lane] ? T(-1) : T(0)));
    rr = P.w_rest * (qi - P.rest[lane]);
    cost_part += rl * rl + rr * rr;
  }
  const T cost = warp_sum(cost_part);
  if (!JAC) return cost;
  __syncwarp();
  // ---- Jacobian column `lane` -----------------------------------------------------
  T col[6 * kTreeMaxPoses];
#pragma unroll
  for (int m = 0; m < 6 * kTreeMaxPoses; ++m) col[m] = T(0);
  if (lane < n) {
    for (int j = 0; j < P.nj; ++j) {
      if (P.kind[j] == 0 || P.qcol[j] != lane) continue;
      const vec3<T> a{S.am[j][0], S.am[j][1], S.am[j][2]};
      const vec3<T> mm{S.am[j][3], S.am[j][4], S.am[j][5]};
      const T mu = P.mult[j];
#pragma unroll
      for (int e = 0; e < kTreeMaxPoses; ++e) {
        if (e >= ne || !((P.anc_ee[e] >> j) & 1ull)) continue;
        const T* E = S.ee[e];
        vec3<T> lw, aw;
        if (P.kind[j] == 1) {
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
  for (int m = 0; m < 6 * kTreeMaxPoses; ++m) S.J[m][lane] = col[m];
  __syncwarp();
  // ---- normal equations: lane i forms row i ----------------------------------------
  T g = T(0);
  if (lane < n) {
    for (int j = 0; j < n; ++j) {
      T a = T(0);
#pragma unroll
      for (int m = 0; m < 6 * kTreeMaxPoses; ++m)
        if (m < 6 * ne) a += col[m] * S.J[m][j];
      S.A[j * 33 + lane] = a;
    }
    S.A[lane * 33 + lane] += gl * gl + P.w_rest * P.w_rest;
#pragma unroll
    for (int m = 0; m < 6 * kTreeMaxPoses; ++m)
      if (m < 6 * ne) g += col[m] * S.ee[m / 6][m % 6];
    g += gl * rl + P.w_rest * rr;
  }
  g_out = g;
  __syncwarp();
  return cost;
}

// delta (lane i -> d_i) = -(A + lam diag(max(diag A, 1e-8)))^-1 g; false if a pivot fails
template <typename T>
__device__ __forceinline__ bool tree_damped_solve(const TreeLmParams<T>& P, TreeScratch<T>& S, T g, T lam,
                                                  int lane, T& delta) {
  const int n = P.n;
  if (lane < n)
    for (int j = 0; j < n; ++j) S.L[j * 33 + lane] = S.A[j * 33 + lane];
  __syncwarp();
  if (lane < n) {
    const T dd = S.A[lane * 33 + lane];
    S.L[lane * 33 + lane] = dd + lam * tmax(dd, T(BeamConsts::diag_clamp));
  }
  __syncwarp();
  bool ok = true;
  T dinv_mine = T(0);
  for (int k = 0; k < n; ++k) {
    const T dk = S.L[k * 33 + k];
    ok = ok && (dk > T(0)) && finite_t(dk);
    const T inv = rsqrt_t(dk);
    if (lane == k) dinv_mine = inv;
    __syncwarp();
    if (lane > k && lane < n) S.L[k * 33 + lane] *= inv;  // L[lane][k]
    __syncwarp();
    if (lane > k && lane < n) {
      const T lik = S.L[k * 33 + lane];
      for (int j = k + 1; j <= lane; ++j) S.L[j * 33 + lane] -= lik * S.L[k * 33 + j];
    }
    __syncwarp();
  }
  // forward: y = L^-1 (-g)
  T y = -g;
  for (int k = 0; k < n; ++k) {
    T yk = shfl_t(y * dinv_mine, k);
    if (lane == k) y = yk;
    if (lane > k && lane < n) y -= S.L[k * 33 + lane] * yk;
  }
  // backward: x = L^-T y
  T x = y;
  for (int k = n - 1; k >= 0; --k) {
    const T xk = shfl_t(x * dinv_mine, k);
    if (lane == k) x = xk;
    if (lane < k) x -= S.L[lane * 33 + k] * xk;  // L[k][lane]
  }
  delta = lane < n ? x : T(0);
  return ok;
}

template <typename T>
__global__ void __launch_bounds__(128)
k_tree_solve(const TreeLmParams<T> P, const double* __restrict__ targets, const double* __restrict__ q0, int64_t B,
             const LmOptions O, double* __restrict__ q_out, double* __restrict__ cost_out,
             double* __restrict__ init_cost_out, double* __restrict__ hist_out, int32_t* __restrict__ iters_out,
             int32_t* __restrict__ term_out) {
  extern __shared__ unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  if (b >= B) return;  // whole warp exits together
  TreeScratch<T>& S = reinterpret_cast<TreeScratch<T>*>(smem_raw)[wib];
  const int n = P.n;
  const double* tg = targets + b * 7 * P.ne;
  S.q[lane] = lane < n ? T(q0[b * n + lane]) : T(0);
  __syncwarp();
  T g;
  T cost = tree_eval<T, true>(P, tg, S, S.q, lane, g);
  const int hstride = O.max_iterations + 1;
  if (lane == 0) {
    if (hist_out) hist_out[b * hstride] = double(cost);
    init_cost_out[b] = double(cost);
  }
  int term = finite_t(cost) ? 0 : 5;
  int iters = 0;
  T damping = T(O.damping0);
  for (int it = 0; it < O.max_iterations && term == 0; ++it) {
    if (warp_max(lane < n ? fabs(g) : T(0)) < T(O.grad_tol)) {
      term = 1;
      break;
    }
    bool accepted = false;
    T step = T(0);
    for (int rj = 0; rj < O.max_rejections; ++rj) {
      T d;
      bool ok = tree_damped_solve(P, S, g, damping, lane, d);
      ok = __all_sync(0xffffffffu, ok && finite_t(d));
      if (ok) {
        S.qn[lane] = S.q[lane] + d;
        __syncwarp();
        T gd;
        const T cn = tree_eval<T, false>(P, tg, S, S.qn, lane, gd);
        if (!finite_t(cn)) {
          term = 5;
          break;
        }
        if (cn < cost) {
          S.q[lane] = S.qn[lane];
          step = d;
          cost = cn;
          damping = tmax(damping * T(O.down), T(BeamConsts::damping_min));
          accepted = true;
          __syncwarp();
          break;
        }
      }
      damping *= T(O.up);
      if (damping > T(BeamConsts::damping_max)) break;
    }
    if (term != 0) break;
    if (!accepted) {
      term = damping > T(BeamConsts::damping_max) ? 3 : 4;
      break;
    }
    ++iters;
    if (lane == 0 && hist_out) hist_out[b * hstride + iters] = double(cost);
    if (warp_max(fabs(step)) < T(O.step_tol)) {
      term = 2;
      break;
    }
    tree_eval<T, true>(P, tg, S, S.q, lane, g);
  }
  if (hist_out)
    for (int i = iters + 1 + lane; i < hstride; i += 32) hist_out[b * hstride + i] = NAN;
  if (lane < n) q_out[b * n + lane] = double(S.q[lane]);
  if (lane == 0) {
    cost_out[b] = double(cost);
    iters_out[b] = iters;
    term_out[b] = term;
  }
}

template <typename T>
cudaError_t launch_tree_solve(const TreeLmParams<T>& P, const TreeLaunch& L, cudaStream_t st) {
  if (L.B == 0) return cudaSuccess;
  const int warps = 4;
  const size_t smem = sizeof(TreeScratch<T>) * warps;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_tree_solve<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_tree_solve<T><<<(unsigned)((L.B + warps - 1) / warps), 32 * warps, smem, st>>>(
      P, L.targets, L.q0, L.B, L.opts, L.q_out, L.cost_out, L.init_cost, L.hist_out, L.iters, L.term);
  return cudaGetLastError();
}

template cudaError_t launch_tree_solve<float>(const TreeLmParams<float>&, const TreeLaunch&, cudaStream_t);
template cudaError_t launch_tree_solve<double>(const TreeLmParams<double>&, const TreeLaunch&, cudaStream_t);

}  // namespace kop
