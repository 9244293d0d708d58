// Batched trajectory optimisation (config 5): the plan_trajectory cost set
// (tasks.py:347-403) solved by solver.solve's LM (solver.py:364-429), one CTA
// (128 threads) per trajectory of T <= 64 timesteps.
//
// Variables q_0..q_{T-1} (NQ each) are one vector of N = T*NQ unknowns.  The
// costs couple timestep t with t-1 (smoothness, velocity limit: diagonal;
// swept capsules: full NQ x NQ blocks) and, through the 5-point acceleration /
// jerk stencils over t-2..t+2, with t-2, t-3, t-4 (diagonal blocks).  So J^T J
// is a band matrix of half-bandwidth 4*NQ whose block row t holds a full
// lower-triangular diagonal block, a full (t, t-1) block and three diagonal
// blocks; H is stored in that compact form (NT + NQ^2 + 3 NQ per timestep),
// its Cholesky factor -- which fills the band -- as a band (the reference
// switches to SuperLU above 200 unknowns, solver.py:327-354; a banded
// Cholesky is the same linear solve).
//
// Per evaluation:
//   A  thread t: FK forward pass of q_t (Pluecker axes + sphere centres in
//      shared memory), the timestep-local rows (limit, rest, anchors, world,
//      self), smoothness / velocity rows of the pair (t-1, t) and the stencil
//      rows: it owns block row t of the band (rows t*NQ .. t*NQ+NQ-1).
//   B  thread t: swept-capsule rows of the pair (t-1, t) (costs.py:554-619):
//      cross block H[t][t-1] written directly, the H[t-1][t-1] part handed to
//      thread t-1 through a per-pair buffer.
//   C  thread t adds the handed-over part; block reduction of the cost.
// LM: gradient test, banded Cholesky of H + lam diag(max(diag H, 1e-8)) with
// two barriers per timestep block, triangular solves by warp 0, rejection loop,
// terminations -- the semantics of solver.solve.
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "kop_beam.cuh"
#include "kop_collision.cuh"
#include "kop_kernels.cuh"
#include "kop_traj.cuh"

namespace kop {

// Threads per trajectory CTA: 128 (4 warps) for FP32, whose CTAs (89 KB of
// shared memory at T = 64) run two per SM; 256 (8 warps, the two-sided
// factorisation) for FP64, whose 175 KB CTAs run one per SM.
// Trailing-update pairs per thread: FP32 holds its table entries in registers
// for the whole sweep and issues 4 dot products together; FP64, at the
// register cap, reads one entry of the shared table per dot product (measured
// at T = 64: both +30% / +0% over the other choice in FP64 / FP32).
#ifndef KOP_TRAJ_CH32
#define KOP_TRAJ_CH32 4
#endif
#ifndef KOP_TRAJ_CH64
#define KOP_TRAJ_CH64 1
#endif
#ifndef KOP_TRAJ_FP32_THREADS
#define KOP_TRAJ_FP32_THREADS 128
#endif
template <class G>
constexpr int traj_threads() {
  return std::is_same<typename G::T, double>::value ? 256 : KOP_TRAJ_FP32_THREADS;
}

#ifdef KOP_TRAJ_TIMELINE
// debug timeline of the first damped solve of CTA 0: [role][block][event] clock64 stamps
__device__ long long g_traj_tl[4][72][6];
__device__ int g_traj_tl_on = 1;
__device__ __forceinline__ long long tl_clock() {
  long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t)::"memory");
  return t;
}
#define KOP_TL(role, blk, ev) \
  if (blockIdx.x == 0 && g_traj_tl_on && (threadIdx.x & 31) == 0 && (role) < 4 && (blk) < 72) g_traj_tl[role][blk][ev] = tl_clock()
#else
#define KOP_TL(role, blk, ev)
#endif

#ifdef KOP_TRAJ_PROFILE
// debug instrumentation (tools/build_variant.py NAME -DKOP_TRAJ_PROFILE): clock64
// cycles of thread 0 per phase, summed over CTAs:
//   0 eval+J, 1 eval, 2 solve setup, 3 factor loop, 4 back substitution, 5 #solves, 6 #evals+J, 7 #evals,
//   per block of a sweep (main lane 0): 8.. top sweep, 12.. bottom sweep, 16.. separator sweep:
//   +0 rows, +1 barrier 1, +2 diagonal pairs + factor, +3 barrier 2
__device__ unsigned long long g_traj_prof[20];
#define KOP_PROF_T(v) long long v = clock64()
#define KOP_PROF_SET(v) v = clock64()
#define KOP_PROF_ADD(slot, cycles) \
  if (threadIdx.x == 0) atomicAdd(&g_traj_prof[slot], (unsigned long long)(cycles))
#else
#define KOP_PROF_T(v)
#define KOP_PROF_SET(v)
#define KOP_PROF_ADD(slot, cycles)
#endif

// Shared-memory layout, sized by the trajectory length at launch:
//   obstacle table | trailing-update pair table | reduction buffer | q, qn, g, y, 1/diag(L)  [N each]
//   H compact [T x HB]: per timestep D (lower NT) | X = H(t, t-1) (NQ^2, row-major) | E2, E3, E4 (NQ each)
//   union { L band [N x LW], L(i, i-d) at [i][d]  |  FK scratch [(6K + 3 ns) x T] + pair buffers }
// The union is safe: L lives from the factorisation to the end of the
// triangular solves, the scratch and pair buffers only inside an evaluation.
template <class G>
struct TrajView {
  using T = typename G::T;
  static constexpr int NQ = G::NQ, BW = 4 * NQ, NT = Tri<NQ>::size, HB = NT + NQ * NQ + 3 * NQ;
  // trailing-update pairs (ri, ci), NQ <= ri < BW, 0 <= ci <= ri, taken by warps 1..3
  static constexpr int NPAIR = BW * (BW + 1) / 2 - NT;
  // band row stride: BW + 1 entries and one pad, so that rows r, r + 1 of one
  // block column (stride LW + 1) fall in different banks
  static constexpr int LW = BW + 2;
  static constexpr int TH = traj_threads<G>();
  static constexpr bool TWIST = TH == 256;  // two-sided factorisation
  static constexpr size_t kHead = (sizeof(ObstacleTable<T>) + 15) / 16 * 16 + (NPAIR * 2 + 15) / 16 * 16;
  ObstacleTable<T>* obs;
  uint16_t* pairs;  // ri | ci << 8
  T *red, *anc, *q, *qn, *g, *y, *dinv, *H, *L, *scratch, *pbufA, *pbufg, *sbuf, *dbuf, *sbuf2;
  // 256-thread CTAs (FP64): the self-collision pairs of timestep t are split
  // between threads t + 64 and t + 128 (idle in the evaluation otherwise)
  static constexpr bool SPLIT = TH >= 192;
  int steps;
  __host__ __device__ static size_t bytes(int steps, int ns) {
    const size_t N = (size_t)steps * NQ;
    const size_t band = N * LW;
    const size_t uni_b = (size_t)(6 * G::K + 3 * ns) * steps + (size_t)steps * ((NT + NQ) * (SPLIT ? 3 : 2) + 2 * NQ);
    return kHead + sizeof(T) * (TH + 2 * NQ + 5 * N + (size_t)steps * HB + (band > uni_b ? band : uni_b));
  }
  __device__ TrajView(unsigned char* base, int steps_, int ns) : steps(steps_) {
    const int N = steps * NQ;
    obs = reinterpret_cast<ObstacleTable<T>*>(base);
    pairs = reinterpret_cast<uint16_t*>(base + (sizeof(ObstacleTable<T>) + 15) / 16 * 16);
    T* p = reinterpret_cast<T*>(base + kHead);
    red = p; p += TH;
    anc = p; p += 2 * NQ;
    q = p; p += N;
    qn = p; p += N;
    g = p; p += N;
    y = p; p += N;
    dinv = p; p += N;
    H = p; p += steps * HB;
    L = p;
    scratch = p; p += (6 * G::K + 3 * ns) * steps;
    pbufA = p; p += steps * NT;
    pbufg = p; p += steps * NQ;
    sbuf = p; p += steps * (NT + NQ);  // block t parts of thread t + 64's rows (self, swept)
    dbuf = p; p += steps * 2 * NQ;  // diagonal block t-1 parts of the smoothness / velocity rows of pair (t-1, t)
    sbuf2 = p;  // (SPLIT) block t parts of thread t + 128's self pairs
  }
  // pair q of the trailing update, in the order (ri = NQ, ci = 0..ri), (ri = NQ + 1, ...), ...
  __device__ void build_pairs() const {
    for (int q = threadIdx.x; q < NPAIR; q += blockDim.x) {
      int ri = NQ, base = 0;
      while (q >= base + ri + 1) {
        base += ri + 1;
        ++ri;
      }
      pairs[q] = uint16_t(ri | (q - base) << 8);
    }
  }
  __device__ __forceinline__ T* hd(int t) const { return H + t * HB; }            // D_t
  __device__ __forceinline__ T* hx(int t) const { return H + t * HB + NT; }       // X_t
  __device__ __forceinline__ T* he(int t) const { return H + t * HB + NT + NQ * NQ; }  // E2..E4
  // H(i, i - d) of the band from the compact blocks
  __device__ __forceinline__ T h(int i, int d) const {
    const int t = i / NQ, a = i % NQ;
    if (d <= a) return hd(t)[Tri<NQ>::at(a, a - d)];
    if (d <= a + NQ) return t >= 1 ? hx(t)[a * NQ + NQ + a - d] : T(0);
    const int m = d / NQ;
    return (d % NQ == 0 && t >= m) ? he(t)[(m - 2) * NQ + a] : T(0);
  }
  __device__ __forceinline__ T& l(int i, int d) const { return L[i * LW + d]; }
  __device__ __forceinline__ ColLane<G> lane(int t) const { return ColLane<G>{scratch + t, steps}; }
};

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const T r = red[0];
  __syncthreads();
  return r;
}

template <typename T>
__device__ __forceinline__ T block_max(T v, T* red) {
  red[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] = tmax(red[threadIdx.x], red[threadIdx.x + o]);
    __syncthreads();
  }
  const T r = red[0];
  __syncthreads();
  return r;
}

template <typename T>
__device__ __forceinline__ void load_obstacles(ObstacleTable<T>& O, const double* __restrict__ obstacles, int64_t b,
                                               int n_obs) {
  if (threadIdx.x == 0) O.no = n_obs;
  for (int o = threadIdx.x; o < n_obs; o += blockDim.x) {
    const double* src = obstacles + (b * n_obs + o) * 8;
    O.okind[o] = int(src[0]);
    for (int i = 0; i < 3; ++i) {
      O.oa[o][i] = T(src[1 + i]);
      O.ob[o][i] = T(src[4 + i]);
    }
    O.orad[o] = T(src[7]);
  }
}

// Jacobian row over the chain joints k <= slot of sum_s w_s g_s . J(c_s):
// e_k = a_k . M - m_k . G (revolute), a_k . G (prismatic)
template <class G>
__device__ __forceinline__ void col_row_entries(const ChainParams<typename G::T, G::K>& C, const ColLane<G>& L,
                                                int slot, const vec3<typename G::T>& M,
                                                const vec3<typename G::T>& Gv, typename G::T scale,
                                                typename G::T (&jr)[G::NQ]) {
  using T = typename G::T;
#pragma unroll
  for (int c = 0; c < G::NQ; ++c) jr[c] = T(0);
#pragma unroll
  for (int k = 0; k < G::K; ++k) {
    if ((G::ID || k < C.k) && k <= slot) {
      const vec3<T> a{L.am(k, 0), L.am(k, 1), L.am(k, 2)};
      const vec3<T> m{L.am(k, 3), L.am(k, 4), L.am(k, 5)};
      const T e = scale * ((!G::ID && C.prismatic[k]) ? dot(a, Gv) : dot(a, M) - dot(m, Gv));
      if (G::ID) {
        jr[k] += e;
      } else {
#pragma unroll
        for (int c = 0; c < G::NQ; ++c)
          if (C.qcol[k] == c) jr[c] += C.mult[k] * e;
      }
    }
  }
}

// Swept-capsule rows of the pair (t-1, t) (costs.py:554-619): cost, the block
// t-1 part (pA, pg), the block t part (Ad, gd) and the cross block H(t, t-1)
// written into t's own compact rows.
template <class G, bool JAC>
__device__ __forceinline__ typename G::T traj_swept_rows(const ChainParams<typename G::T, G::K>& C,
                                                         const CollisionParams<typename G::T>& P,
                                                         const TrajCosts<typename G::T>& W, const TrajView<G>& S,
                                                         int t, typename G::T (&pA)[Tri<G::NQ>::size],
                                                         typename G::T (&pg)[G::NQ],
                                                         typename G::T (&Ad)[Tri<G::NQ>::size],
                                                         typename G::T (&gd)[G::NQ]) {
  using T = typename G::T;
  constexpr int NQ = G::NQ;
  T cost = T(0);
  const ColLane<G> L0 = S.lane(t - 1), L1 = S.lane(t);
  for (int li = 0; li < P.nl; ++li) {
    const int f = P.lfirst[li], nsph = P.lcount[li];
    for (int o = 0; o < S.obs->no; ++o) {
      {  // screening, as in col_rows: skip rows inactive on every lane of the warp
        T dscr = inf_t<T>();
        for (int s = 0; s < nsph; ++s) {
          vec3<T> ga, gb;
          dscr = tmin(dscr, capsule_obstacle_t<T>(
                                *S.obs, o, vec3<T>{L0.cen(f + s, 0), L0.cen(f + s, 1), L0.cen(f + s, 2)},
                                vec3<T>{L1.cen(f + s, 0), L1.cen(f + s, 1), L1.cen(f + s, 2)}, P.sr[f + s], ga, gb));
        }
        if (__all_sync(__activemask(), dscr - P.lreach[li] > W.eta_world * T(1.00001))) continue;
      }
      const bool hard = P.hard || nsph == 1;
      SoftMin<T, 4> sm;  // sum z c0 x ga, sum z ga, sum z c1 x gb, sum z gb
      for (int s = 0; s < nsph; ++s) {
        const vec3<T> c0{L0.cen(f + s, 0), L0.cen(f + s, 1), L0.cen(f + s, 2)};
        const vec3<T> c1{L1.cen(f + s, 0), L1.cen(f + s, 1), L1.cen(f + s, 2)};
        vec3<T> ga, gb;
        const T d = capsule_obstacle_t<T>(*S.obs, o, c0, c1, P.sr[f + s], ga, gb);
        const T z = sm.weight(d, P.beta, hard);
        if (z == T(0)) continue;  // zero weights add nothing (the reference skips them, costs.py:541)
        sm.sumz += z;
        if (JAC) {
          sm.add(z, 0, cross(c0, ga));
          sm.add(z, 1, ga);
          sm.add(z, 2, cross(c1, gb));
          sm.add(z, 3, gb);
        }
      }
      T act, dact;
      activation_t(sm.aggregate(P.beta, hard), W.eta_world, act, dact);
      const T res = W.w_world * act;
      cost += res * res;
      if (JAC && dact != T(0)) {
        sm.normalise();
        const vec3<T> M0 = sm.acc[0], G0 = sm.acc[1], M1 = sm.acc[2], G1 = sm.acc[3];
        T j0[NQ], j1[NQ];
        col_row_entries<G>(C, L0, P.lslot[li], M0, G0, W.w_world * dact, j0);
        col_row_entries<G>(C, L1, P.lslot[li], M1, G1, W.w_world * dact, j1);
#pragma unroll
        for (int a = 0; a < NQ; ++a) {
#pragma unroll
          for (int b = 0; b < NQ; ++b) {
            if (b <= a) {
              pA[Tri<NQ>::at(a, b)] += j0[a] * j0[b];
              Ad[Tri<NQ>::at(a, b)] += j1[a] * j1[b];
            }
            S.hx(t)[a * NQ + b] += j1[a] * j0[b];  // H(t, t-1) block, own rows
          }
          pg[a] += j0[a] * res;
          gd[a] += j1[a] * res;
        }
      }
    }
  }
  return cost;
}

// Evaluate the trajectory stack at x (S.q or S.qn); JAC also forms the band
// H and g.  Returns the cost on every thread.
template <class G, bool JAC>
__device__ typename G::T traj_eval(const ChainParams<typename G::T, G::K>& C, const CollisionParams<typename G::T>& P,
                                   const TrajCosts<typename G::T>& W, const TrajView<G>& S, const typename G::T* x) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, NT = Tri<NQ>::size;
  const int tid = threadIdx.x, Tn = W.T_steps;
  T cost = T(0);
  // ---- A: FK + timestep-local rows + smoothness / velocity / stencils --------
  T Ad[NT], gd[NQ];
#pragma unroll
  for (int i = 0; i < NT; ++i) Ad[i] = T(0);
#pragma unroll
  for (int i = 0; i < NQ; ++i) gd[i] = T(0);
  T cross_diag[NQ], off_diag[3][NQ];  // diagonal entries of H(t, t-1) and H(t, t-2..t-4) from diagonal rows
#pragma unroll
  for (int i = 0; i < NQ; ++i) cross_diag[i] = off_diag[0][i] = off_diag[1][i] = off_diag[2][i] = T(0);
  T prevA_diag[NQ], prev_g[NQ];  // diagonal-row contributions to block t-1 (pair (t-1, t))
#pragma unroll
  for (int i = 0; i < NQ; ++i) prevA_diag[i] = prev_g[i] = T(0);
  const int t = tid;
  if (t < Tn) {  // FK of timestep t: Pluecker axes and sphere centres into the lane scratch
    T q[NQ];
#pragma unroll
    for (int i = 0; i < NQ; ++i) q[i] = x[t * NQ + i];
    quat<T> eq;
    vec3<T> ep;
    col_forward<G>(C, P, S.lane(t), q, eq, ep);
    if (JAC)  // the (t, t-1) block is accumulated by thread t + 64 (swept rows) and t (diagonal rows)
      for (int i = 0; i < NQ * NQ; ++i) S.hx(t)[i] = T(0);
  }
  __syncthreads();
  // thread t + 64: the self rows of timestep t and the swept rows of the pair
  // (t-1, t), beside thread t's local / world / smoothness / stencil rows
  const bool self_rows = P.np > 0 && P.w_self > T(0);
  const bool swept_rows = W.w_world > T(0) && S.obs->no > 0;
  if (tid >= 64 && tid - 64 < Tn && (self_rows || swept_rows)) {
    const int u = tid - 64;
    T As[NT], gs[NQ];
#pragma unroll
    for (int i = 0; i < NT; ++i) As[i] = T(0);
#pragma unroll
    for (int i = 0; i < NQ; ++i) gs[i] = T(0);
    if (self_rows)
      cost += col_rows<G, JAC, ObstacleTable<T>, true, 2>(C, P, S.lane(u), As, gs, 0, nullptr, nullptr, S.obs, 0,
                                                          TrajView<G>::SPLIT ? P.np / 2 : P.np);
    if (swept_rows && u >= 1) {
      T pA[NT], pg[NQ];  // block u-1 part
#pragma unroll
      for (int i = 0; i < NT; ++i) pA[i] = T(0);
#pragma unroll
      for (int i = 0; i < NQ; ++i) pg[i] = T(0);
      cost += traj_swept_rows<G, JAC>(C, P, W, S, u, pA, pg, As, gs);
      if (JAC) {
#pragma unroll
        for (int i = 0; i < NT; ++i) S.pbufA[u * NT + i] = pA[i];
#pragma unroll
        for (int i = 0; i < NQ; ++i) S.pbufg[u * NQ + i] = pg[i];
      }
    }
    if (JAC) {
#pragma unroll
      for (int i = 0; i < NT; ++i) S.sbuf[u * (NT + NQ) + i] = As[i];
#pragma unroll
      for (int i = 0; i < NQ; ++i) S.sbuf[u * (NT + NQ) + NT + i] = gs[i];
    }
  }
  if constexpr (TrajView<G>::SPLIT) {  // thread t + 128: the second half of timestep t's self pairs
    if (tid >= 128 && tid - 128 < Tn && self_rows && P.np / 2 < P.np) {
      const int u = tid - 128;
      T As2[NT], gs2[NQ];
#pragma unroll
      for (int i = 0; i < NT; ++i) As2[i] = T(0);
#pragma unroll
      for (int i = 0; i < NQ; ++i) gs2[i] = T(0);
      cost += col_rows<G, JAC, ObstacleTable<T>, true, 2>(C, P, S.lane(u), As2, gs2, 0, nullptr, nullptr, S.obs,
                                                          P.np / 2, P.np);
      if (JAC) {
#pragma unroll
        for (int i = 0; i < NT; ++i) S.sbuf2[u * (NT + NQ) + i] = As2[i];
#pragma unroll
        for (int i = 0; i < NQ; ++i) S.sbuf2[u * (NT + NQ) + NT + i] = gs2[i];
      }
    }
  }
  if (t < Tn) {
    T q[NQ];
#pragma unroll
    for (int i = 0; i < NQ; ++i) q[i] = x[t * NQ + i];
    const ColLane<G> L = S.lane(t);
    // limit (costs.py:174-195), rest (tasks.py:386-389), anchors (tasks.py:352-355)
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      const T above = q[i] - W.upper[i], below = W.lower[i] - q[i];
      const T rl = W.w_lim * (tmax(T(0), above) + tmax(T(0), below));
      const T gl = W.w_lim * ((q[i] > W.upper[i] ? T(1) : T(0)) + (q[i] < W.lower[i] ? T(-1) : T(0)));
      const T rr = W.w_rest * (q[i] - W.rest[i]);
      cost += rl * rl + rr * rr;
      Ad[Tri<NQ>::at(i, i)] += gl * gl + W.w_rest * W.w_rest;
      gd[i] += gl * rl + W.w_rest * rr;
      if (t == 0 || t == Tn - 1) {
        const T ra = W.anchor * (q[i] - S.anc[(t == 0 ? 0 : NQ) + i]);
        cost += ra * ra;
        Ad[Tri<NQ>::at(i, i)] += W.anchor * W.anchor;
        gd[i] += W.anchor * ra;
      }
    }
    // world rows (per-problem obstacle table); the self rows run on thread t + 64
    cost += col_rows<G, JAC, ObstacleTable<T>, true, 1>(C, P, L, Ad, gd, 0, nullptr, nullptr, S.obs);
    // smoothness + velocity of the pair (t-1, t) (costs.py:198-231, 274-290)
    if (t >= 1) {
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const T dq = q[i] - x[(t - 1) * NQ + i];
        const T rs = W.w_smooth * dq;
        cost += rs * rs;
        T jv = T(0), rv = T(0);
        if (W.w_vel > T(0) && finite_t(W.vbudget[i]) && fabs(dq) > W.vbudget[i]) {
          rv = W.w_vel * (fabs(dq) - W.vbudget[i]);
          jv = W.w_vel * (dq > T(0) ? T(1) : (dq < T(0) ? T(-1) : T(0)));
        }
        cost += rv * rv;
        const T h = W.w_smooth * W.w_smooth + jv * jv;
        Ad[Tri<NQ>::at(i, i)] += h;
        prevA_diag[i] += h;
        cross_diag[i] -= h;
        gd[i] += W.w_smooth * rs + jv * rv;
        prev_g[i] -= W.w_smooth * rs + jv * rv;
      }
    }
    // 5-point stencils (costs.py:293-341): this thread owns block row t and
    // adds every stencil centred at s = t-2 .. t+2 that touches it; the cost
    // of stencil s is added by thread s
    for (int s = t - 2; s <= t + 2; ++s) {
      if (s < 2 || s > Tn - 3) continue;
      const int j = t - s + 2;  // this row's coefficient index
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        T ra = T(0), rj = T(0);
#pragma unroll
        for (int kk = 0; kk < 5; ++kk) {
          const T xv = x[(s + kk - 2) * NQ + i];
          ra += W.acc_c[kk] * xv;
          rj += W.jerk_c[kk] * xv;
        }
        ra *= W.w_acc;
        rj *= W.w_jerk;
        if (s == t) cost += ra * ra + rj * rj;
        const T ca = W.w_acc * W.acc_c[j], cj = W.w_jerk * W.jerk_c[j];
        Ad[Tri<NQ>::at(i, i)] += ca * ca + cj * cj;
        gd[i] += ca * ra + cj * rj;
        if (j >= 1) cross_diag[i] += ca * W.w_acc * W.acc_c[j - 1] + cj * W.w_jerk * W.jerk_c[j - 1];
#pragma unroll
        for (int m = 2; m <= 4; ++m)
          if (j >= m) off_diag[m - 2][i] += ca * W.w_acc * W.acc_c[j - m] + cj * W.w_jerk * W.jerk_c[j - m];
      }
    }
  }
  if (JAC && t >= 1 && t < Tn) {  // diagonal rows' block t-1 part of the pair (t-1, t)
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      S.dbuf[t * 2 * NQ + i] = prevA_diag[i];
      S.dbuf[t * 2 * NQ + NQ + i] = prev_g[i];
    }
  }
  __syncthreads();
  // ---- C: assemble own block row -------------------------------------------------
  if (JAC && t < Tn) {
    if (t + 1 < Tn) {
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        Ad[Tri<NQ>::at(i, i)] += S.dbuf[(t + 1) * 2 * NQ + i];
        gd[i] += S.dbuf[(t + 1) * 2 * NQ + NQ + i];
      }
      if (swept_rows) {
#pragma unroll
        for (int i = 0; i < NT; ++i) Ad[i] += S.pbufA[(t + 1) * NT + i];
#pragma unroll
        for (int i = 0; i < NQ; ++i) gd[i] += S.pbufg[(t + 1) * NQ + i];
      }
    }
    if (self_rows || swept_rows) {
#pragma unroll
      for (int i = 0; i < NT; ++i) Ad[i] += S.sbuf[t * (NT + NQ) + i];
#pragma unroll
      for (int i = 0; i < NQ; ++i) gd[i] += S.sbuf[t * (NT + NQ) + NT + i];
    }
    if (TrajView<G>::SPLIT && self_rows && P.np / 2 < P.np) {
#pragma unroll
      for (int i = 0; i < NT; ++i) Ad[i] += S.sbuf2[t * (NT + NQ) + i];
#pragma unroll
      for (int i = 0; i < NQ; ++i) gd[i] += S.sbuf2[t * (NT + NQ) + NT + i];
    }
#pragma unroll
    for (int a = 0; a < NQ; ++a) {
#pragma unroll
      for (int b = 0; b < NQ; ++b)
        if (b <= a) S.hd(t)[Tri<NQ>::at(a, b)] = Ad[Tri<NQ>::at(a, b)];
      if (t >= 1) S.hx(t)[a * NQ + a] += cross_diag[a];
#pragma unroll
      for (int m = 0; m < 3; ++m) S.he(t)[m * NQ + a] = off_diag[m][a];
      S.g[t * NQ + a] = gd[a];
    }
  }
  return block_sum(cost, S.red);
}

// Banded damped Cholesky solve: y <- -(H + lam diag(max(diag H, 1e-8)))^-1 g.
//
// Two-sided ("twisted") blocked factorisation over timestep blocks of NQ
// columns.  The N unknowns are ordered [top | bottom (reversed) | separator]:
// the separator is the 4 blocks (= the half-bandwidth BW) that decouple the
// top blocks 0..nbA-1 from the bottom blocks nbA+4..nblk-1, so both halves
// are eliminated at the same time, the top one downwards by warps 0 + 2 and
// the bottom one upwards (the same code on the index-reversed band) by warps
// 1 + 3, each pair synchronised by its own named barrier.  Their Schur
// complements meet on the separator (the bottom one is added afterwards from
// its stored factor columns, so no entry has two writers), which all four
// warps then factor; the back substitution solves the separator, then both
// halves outwards concurrently.  The serial chain -- one diagonal-block
// factorisation per timestep -- is half as long as a one-sided sweep.
//
// Per eliminated block jb of a sweep:
//   rows   main warp lanes 0..BW-1: the BW rows below block jb solve
//          x D^T = a (their NQ-wide slice of the block column), y_r -= x . z;
//   trail  the main warp updates the NEXT diagonal block and its lane 0
//          factors it in registers (carrying the forward substitution) while
//          the trailing warp(s) apply L(r, c) -= x_r . x_c to the rest of the
//          BW x BW lower triangle below block jb (pairs from the smem table).
// Two barriers per block.  Entries of the band beyond half-width BW are
// structural zeros of the factor (the profile of row t*NQ+a starts at
// (t-4)*NQ+a) and are never stored.
//
// Each routine below is inlined once per view direction (the sweeps and the
// back substitutions are loops over phases with per-warp parameters): the
// kernel is large, and more copies of the sweep thrash the instruction cache.

// The band seen in forward or index-reversed (REV) order, as an affine map: view
// entry (i, i - d) of the lower band of P A P, P the reversal, is
// A(N-1-i+d, N-1-i) = storage (N-1-i+d, d); along a block column the view's
// entries are sd apart in storage, down it 1 (reversed) or LW + 1 apart.
template <class G, bool REV>
struct BandView {
  using T = typename G::T;
  static constexpr int BW = 4 * G::NQ, LW = TrajView<G>::LW;
  static constexpr int si = REV ? -LW : LW, sd = REV ? LW + 1 : 1, ys = REV ? -1 : 1;
  T *L, *y, *dinv;
  int o, yo;
  __device__ BandView(const TrajView<G>& S, int N)
      : L(S.L), y(S.y), dinv(S.dinv), o(REV ? (N - 1) * LW : 0), yo(REV ? N - 1 : 0) {}
  __device__ __forceinline__ T& l(int i, int d) const { return L[(REV ? o : 0) + si * i + sd * d]; }
  // p with p[-b * sd] = view L(r, c0 + b)
  __device__ __forceinline__ T* rowp(int r, int c0) const { return L + (REV ? o : 0) + si * r + sd * (r - c0); }
  __device__ __forceinline__ T& yv(int i) const { return y[(REV ? yo : 0) + ys * i]; }
  __device__ __forceinline__ T& dv(int i) const { return dinv[(REV ? yo : 0) + ys * i]; }
};

// barrier `id` over `nthreads` (whole warps); the warp reconverges first so
// that it arrives once (lane 0 may still be factoring when lanes 1..31 get here)
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  __syncwarp();
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
  KOP_JITTER_POINT();
}

template <class G, class V_>
__device__ __forceinline__ bool traj_factor_diag(const V_& V, int c0) {
  using T = typename G::T;
  constexpr int NQ = G::NQ;
  T Lb[Tri<NQ>::size], yv[NQ];
  bool ok = true;
#pragma unroll
  for (int a = 0; a < NQ; ++a) {
#pragma unroll
    for (int b = 0; b <= a; ++b) Lb[Tri<NQ>::at(a, b)] = V.l(c0 + a, a - b);
    yv[a] = V.yv(c0 + a);
  }
#pragma unroll
  for (int k = 0; k < NQ; ++k) {
    const T dk = Lb[Tri<NQ>::at(k, k)];
    ok = ok && dk > T(0) && finite_t(dk);
    const T inv = rsqrt_t(dk);
    Lb[Tri<NQ>::at(k, k)] = dk * inv;
    V.dv(c0 + k) = inv;
    const T yk = yv[k] * inv;
    yv[k] = yk;
#pragma unroll
    for (int i = k + 1; i < NQ; ++i) {
      const T lik = Lb[Tri<NQ>::at(i, k)] * inv;
      Lb[Tri<NQ>::at(i, k)] = lik;
      yv[i] -= lik * yk;
    }
#pragma unroll
    for (int i = k + 1; i < NQ; ++i)
#pragma unroll
      for (int j = k + 1; j <= i; ++j) Lb[Tri<NQ>::at(i, j)] -= Lb[Tri<NQ>::at(i, k)] * Lb[Tri<NQ>::at(j, k)];
  }
#pragma unroll
  for (int a = 0; a < NQ; ++a) {
#pragma unroll
    for (int b = 0; b <= a; ++b) V.l(c0 + a, a - b) = Lb[Tri<NQ>::at(a, b)];
    V.yv(c0 + a) = yv[a];
  }
  return ok;
}

// sum_b L(r, c0 + b) L(c, c0 + b) for view rows r = c0+NQ+ri >= c = c0+NQ+ci
template <class G, class V_>
__device__ __forceinline__ typename G::T traj_trailing_dot(const V_& V, int c0, int ri, int ci) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, BW = 4 * NQ;
  const T* lr = V.rowp(c0 + NQ + ri, c0);
  const T* lc = V.rowp(c0 + NQ + ci, c0);
  const int blo = NQ + ri - BW;  // both vanish for b < blo (band edge of row r)
  T acc = T(0);
#pragma unroll
  for (int b = 0; b < NQ; ++b) {  // branch-free; the index is clamped into the band (row N-1 ends the smem)
    const int bb = (b >= blo ? b : blo) * V.sd;
    acc += (b >= blo ? lr[-bb] : T(0)) * lc[-bb];
  }
  return acc;
}

// One sweep: eliminate view blocks jb0 .. jb0+nb-1 with rows up to nlim.
// Main warp (`main`; its lane 0 factors), nwt trailing threads (index tt >= 0),
// barrier (bar, nbar).  defer: leave the separator x separator entries (view
// columns >= sepv) and the separator right-hand side alone (the bottom sweep;
// traj_bottom_schur adds them later).
template <class G, class V_>
__device__ __forceinline__ bool traj_sweep(const TrajView<G>& S, const V_& V, int jb0, int nb, int nlim,
                                           int sepv, bool defer, bool main, int tt, int nwt, int bar, int nbar) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, BW = 4 * NQ, NT = Tri<NQ>::size, NPAIR = TrajView<G>::NPAIR, CH = std::is_same<typename G::T, double>::value ? KOP_TRAJ_CH64 : KOP_TRAJ_CH32;
  const int lane = threadIdx.x & 31;
  int dri[2] = {BW, BW}, dci[2] = {0, 0};  // main warp: diagonal-block pairs lane, lane + 32
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    int rem = lane + 32 * h, ri = 0;
    if (!main || rem >= NT) continue;
    while (rem > ri) {
      rem -= ri + 1;
      ++ri;
    }
    dri[h] = ri;
    dci[h] = rem;
  }
  bool ok = true;
  if (nb <= 0) return ok;
  // FP32: this thread's table entries q = tt + p * nwt, held for the whole sweep (nwt >= 96)
  constexpr bool PREG = !std::is_same<T, double>::value;
  constexpr int PPT = PREG ? (NPAIR + 95) / 96 : 1;
  int pcode[PPT];
#pragma unroll
  for (int p = 0; p < PPT; ++p) {
    const int q = tt + p * nwt;
    pcode[p] = (PREG && tt >= 0 && q < NPAIR) ? S.pairs[q] : -1;
  }
  if (main && lane == 0) ok = traj_factor_diag<G, V_>(V, jb0 * NQ);
  named_bar(bar, nbar);
#ifdef KOP_TRAJ_PROFILE
  long long ph[4] = {0, 0, 0, 0}, tq = clock64(), tn;
#define KOP_PHASE(i) tn = clock64(), ph[i] += tn - tq, tq = tn
#else
#define KOP_PHASE(i)
#endif
  const int role = threadIdx.x >> 5;
  for (int jb = jb0; jb < jb0 + nb; ++jb) {
    const int c0 = jb * NQ;
    KOP_TL(role, jb, 0);
    if (main && lane < BW && c0 + NQ + lane < nlim) {  // rows below the block
      const int r = c0 + NQ + lane;
      const int blo = NQ + lane - BW;  // L(r, c0 + b) = 0 below the band for b < blo
      const T* lr = V.rowp(r, c0);     // L(r, c0 + b) = lr[-b * sd]
      T x[NQ];
      T yu = T(0);
#pragma unroll
      for (int b = 0; b < NQ; ++b) {
        T v = b >= blo ? lr[-(b >= blo ? b : blo) * V.sd] : T(0);  // clamped: never read past the band
#pragma unroll
        for (int m = 0; m < NQ; ++m)
          if (m < b) v -= x[m] * V.l(c0 + b, b - m);
        x[b] = v * V.dv(c0 + b);
        yu += x[b] * V.yv(c0 + b);
      }
#pragma unroll
      for (int b = 0; b < NQ; ++b)
        if (b >= blo) V.l(r, r - (c0 + b)) = x[b];
      if (!defer || r < sepv) V.yv(r) -= yu;
    }
    KOP_PHASE(0);
    KOP_TL(role, jb, 1);
    named_bar(bar, nbar);
    KOP_TL(role, jb, 2);
    KOP_PHASE(1);
    if (c0 + NQ < nlim) {  // trailing update (and look-ahead factor) of the rows below
      const bool next_own = jb + 1 < jb0 + nb;
      if (main) {
        if (!defer || next_own) {
#pragma unroll
          for (int h = 0; h < 2; ++h)
            if (dri[h] < BW) V.l(c0 + NQ + dri[h], dri[h] - dci[h]) -= traj_trailing_dot<G, V_>(V, c0, dri[h], dci[h]);
        }
        __syncwarp();
        if (lane == 0 && next_own) ok = traj_factor_diag<G, V_>(V, c0 + NQ) && ok;
      } else if (tt >= 0) {
        // pairs q = tt + p * nwt (ri >= NQ) of the table, CH dot products issued
        // together (an unused slot reads row c0 + NQ and is dropped)
        for (int p0 = 0; PREG ? p0 < PPT : tt + p0 * nwt < NPAIR; p0 += CH) {
          T acc[CH];
          int code[CH];
          bool use[CH];
#pragma unroll
          for (int p = 0; p < CH; ++p) {
            bool has;
            if constexpr (PREG) {
              has = p0 + p < PPT && pcode[p0 + p] >= 0;
              code[p] = has ? pcode[p0 + p] : 0;
            } else {
              const int q = tt + (p0 + p) * nwt;
              has = q < NPAIR;
              code[p] = has ? S.pairs[q] : 0;
            }
            const int ri = code[p] & 0xff, ci = code[p] >> 8;
            use[p] = has && c0 + NQ + ri < nlim && (!defer || c0 + NQ + ci < sepv);
            acc[p] = traj_trailing_dot<G, V_>(V, c0, use[p] ? ri : 0, use[p] ? ci : 0);
          }
#pragma unroll
          for (int p = 0; p < CH; ++p)
            if (use[p]) {
              const int ri = code[p] & 0xff, ci = code[p] >> 8;
              V.l(c0 + NQ + ri, ri - ci) -= acc[p];
            }
        }
      }
    }
    KOP_PHASE(2);
    KOP_TL(role, jb, 3);
    named_bar(bar, nbar);
    KOP_TL(role, jb, 4);
    KOP_PHASE(3);
  }
#ifdef KOP_TRAJ_PROFILE
  if (main && lane == 0)
    for (int i = 0; i < 4; ++i)
      atomicAdd(&g_traj_prof[(jb0 > 0 ? 16 : defer ? 12 : 8) + i], (unsigned long long)ph[i]);
#endif
#undef KOP_PHASE
  return ok;
}

// The bottom sweep's deferred part of the separator Schur complement:
// view (reversed) rows i >= j >= sepv: L(i, j) -= sum_{c < sepv} L(i, c) L(j, c),
// y_i -= sum_{c < sepv} L(i, c) z_c.  All threads; deterministic order.
template <class G>
__device__ __forceinline__ void traj_bottom_schur(const BandView<G, true>& V, int sepv, int nsep) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, BW = 4 * NQ;
  const int ns = nsep * NQ, ntri = ns * (ns + 1) / 2;
  for (int k = threadIdx.x; k < ntri + ns; k += blockDim.x) {
    int i, j;
    if (k < ntri) {
      i = 0;
      int rem = k;
      while (rem > i) {
        rem -= i + 1;
        ++i;
      }
      j = rem + sepv;
    } else {
      i = k - ntri;
      j = -1;  // right-hand side
    }
    i += sepv;
    const int lo = max(i - BW, 0);
    T acc = T(0);
    if (j < 0) {
      for (int c = lo; c < sepv; ++c) acc += V.l(i, i - c) * V.yv(c);
      V.yv(i) -= acc;
    } else if (i - j <= BW) {
      for (int c = lo; c < sepv; ++c) acc += V.l(i, i - c) * V.l(j, j - c);  // j - c <= i - c <= BW
      V.l(i, i - j) -= acc;
    }
  }
}

// Back substitution L^T x = z over view blocks hi..lo by one warp.  Every lane
// solves the block's triangular system in registers (blocks >= known already
// hold x; lane 0 stores the solution), so x needs no broadcast, and lanes < BW
// remove its contribution from the rows above.  All of a block's loads (its
// right-hand sides, factor entries and this lane's row-update entries) are
// issued together at the top of the block, so the serial chain sees one
// shared-memory latency per block.  Same operations in the same order as a
// one-lane solve.
template <class G, class V_>
__device__ __forceinline__ void traj_back(const V_& V, int hi, int lo, int known) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, BW = 4 * NQ;
  const int lane = threadIdx.x & 31;
  for (int jb = hi; jb >= lo; --jb) {
    const int c0 = jb * NQ, c = c0 - 1 - lane;
    const bool upd = lane < BW && c >= 0 && (jb < known || c < known * NQ);  // solved rows of a known block stay
    T x[NQ], lu[NQ];
#pragma unroll
    for (int b = 0; b < NQ; ++b) {
      x[b] = V.yv(c0 + b);
      const bool in = upd && c0 + b - c <= BW;
      const T v = V.l(c0 + b, in ? c0 + b - c : 0);  // clamped: a valid entry, dropped
      lu[b] = in ? v : T(0);
    }
    if (jb < known) {
#pragma unroll
      for (int bb = 0; bb < NQ; ++bb) {
        const int b = NQ - 1 - bb;
        T v = x[b];
#pragma unroll
        for (int m = NQ - 1; m > b; --m) v -= V.l(c0 + m, m - b) * x[m];  // newest x last
        x[b] = v * V.dv(c0 + b);
      }
      if (lane == 0)
#pragma unroll
        for (int b = 0; b < NQ; ++b) V.yv(c0 + b) = x[b];
    }
    if (upd) {
      T acc = T(0);
#pragma unroll
      for (int b = 0; b < NQ; ++b)
        if (c0 + b - c <= BW) acc += lu[b] * x[b];
      V.yv(c) -= acc;
    }
    __syncwarp();
  }
}

template <class G>
__device__ bool traj_damped_solve(const TrajView<G>& S, int N, typename G::T lam) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, BW = TrajView<G>::BW, NT = Tri<NQ>::size, TH = TrajView<G>::TH;
  static_assert(BW <= 32 && NT <= 64, "band wider than a warp");
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  KOP_PROF_T(pt0);
  for (int i = tid; i < N; i += TH) {
    for (int d = 0; d <= BW; ++d) S.l(i, d) = S.h(i, d);  // zero outside the compact blocks
    S.l(i, 0) += lam * tmax(S.h(i, 0), T(BeamConsts::diag_clamp));
    S.y[i] = -S.g[i];
  }
  const int nblk = N / NQ;
  __syncthreads();
  KOP_PROF_T(pt1);
  KOP_PROF_ADD(2, pt1 - pt0);
  bool ok = true;
  KOP_PROF_T(pt2);
  if constexpr (TrajView<G>::TWIST) {
    // phase 0: both halves at once -- top on the even warps (warp 0 main),
    // bottom on the odd warps (warp 1 main) -- then the bottom half's share of
    // the separator; phase 1: the separator on all warps (warp 0 main)
    const int nsep = min(4, nblk), nbA = (nblk - nsep + 1) / 2, nbB = nblk - nsep - nbA;
    const bool bottom = (warp & 1) != 0;
    const BandView<G, false> A(S, N);
    const BandView<G, true> Bv(S, N);
    for (int ph = 0; ph < 2; ++ph) {
      const bool sep = ph == 1;
      const int tt = sep ? tid - 32 : warp >= 2 ? ((warp >> 1) - 1) * 32 + lane : -1;
      if (!sep && bottom)
        ok = traj_sweep<G>(S, Bv, 0, nbB, (nbB + nsep) * NQ, nbB * NQ, true, warp == 1, tt, TH / 2 - 32, 2, TH / 2);
      else
        ok = traj_sweep<G>(S, A, sep ? nbA : 0, sep ? nsep : nbA, (nbA + nsep) * NQ, N, false,
                           sep ? warp == 0 : warp == 0, tt, sep ? TH - 32 : TH / 2 - 32, sep ? 0 : 1, sep ? TH : TH / 2) &&
             ok;
      __syncthreads();
      if (ph == 0 && nbB > 0) {
        traj_bottom_schur<G>(Bv, nbB * NQ, nsep);
        __syncthreads();
      }
    }
    ok = __syncthreads_and(ok);
    KOP_PROF_SET(pt2);
    KOP_PROF_ADD(3, pt2 - pt1);
    // back substitution: phase 0 the separator (warp 0), phase 1 the top
    // (warp 0) and the bottom (warp 1, starting with the separator's
    // contributions to it) outwards
    for (int ph = 0; ph < 2; ++ph) {
      if (warp == 0) traj_back<G>(A, ph == 0 ? nbA + nsep - 1 : nbA - 1, ph == 0 ? nbA : 0, nblk);
      if (ph == 0 && warp < 2) named_bar(3, 64);
    }
    if (warp == 1) traj_back<G>(Bv, nbB + nsep - 1, 0, nbB);
  } else {
    // one-sided: warp 0 main, warps 1..3 trailing, back substitution on warp 0
    const BandView<G, false> V(S, N);
    ok = traj_sweep<G>(S, V, 0, nblk, N, N, false, warp == 0, tid - 32, TH - 32, 0, TH);
    ok = __syncthreads_and(ok);
    KOP_PROF_SET(pt2);
    KOP_PROF_ADD(3, pt2 - pt1);
    if (warp == 0) traj_back<G>(V, nblk - 1, 0, nblk);
  }
#ifdef KOP_TRAJ_TIMELINE
  __syncthreads();
  if (blockIdx.x == 0 && threadIdx.x == 0) g_traj_tl_on = 0;
#endif
  __syncthreads();
  KOP_PROF_T(pt3);
  KOP_PROF_ADD(4, pt3 - pt2);
  KOP_PROF_ADD(5, 1);
  return ok;
}

// FP32 stopping rule, as in k_col_solve (kop_collision.cu): a rejected trial whose
// quadratic-model decrease is below 2^-17 of the cost is not resolvable in FP32
constexpr float kTrajFp32Tau = 7.62939453125e-6f;

template <class G>
__global__ void __launch_bounds__(traj_threads<G>())
k_traj_solve(const ChainParams<typename G::T, G::K> C, const CollisionParams<typename G::T> P,
             const TrajCosts<typename G::T> W, const double* __restrict__ q_init, const double* __restrict__ anchors,
             const double* __restrict__ obstacles, int n_obs, int64_t B, const LmOptions O,
             double* __restrict__ q_out, double* __restrict__ cost_out, double* __restrict__ init_cost_out,
             double* __restrict__ hist_out, int32_t* __restrict__ iters_out, int32_t* __restrict__ term_out) {
  using T = typename G::T;
  constexpr int NQ = G::NQ;
  extern __shared__ unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  const TrajView<G> S(smem_raw, W.T_steps, P.ns);
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, Tn = W.T_steps, N = Tn * NQ, n = W.n;
  for (int i = tid; i < 2 * NQ; i += traj_threads<G>()) {
    const int c = i % NQ;
    S.anc[i] = c < n ? T(anchors[(b * 2 + i / NQ) * n + c]) : T(0);
  }
  load_obstacles(*S.obs, obstacles, b, n_obs);
  S.build_pairs();
  for (int i = tid; i < N; i += traj_threads<G>()) {
    const int tt = i / NQ, c = i % NQ;
    if (q_init) {
      S.q[i] = c < n ? T(q_init[(b * Tn + tt) * n + c]) : T(0);
    } else {  // straight line between the anchors (tasks.py:344-345, np.linspace)
      const double alpha = tt == Tn - 1 ? 1.0 : double(tt) * (1.0 / double(Tn - 1));
      const double qa = c < n ? anchors[(b * 2) * n + c] : 0.0, qb = c < n ? anchors[(b * 2 + 1) * n + c] : 0.0;
      S.q[i] = T(__dadd_rn(__dmul_rn(qa, 1.0 - alpha), __dmul_rn(qb, alpha)));  // no FMA: numpy's rounding
    }
  }
  __syncthreads();
  T cost = traj_eval<G, true>(C, P, W, S, S.q);
  const int hstride = O.max_iterations + 1;
  if (tid == 0) {
    if (hist_out) hist_out[b * hstride] = double(cost);
    init_cost_out[b] = double(cost);
  }
  int term = finite_t(cost) ? 0 : 5, iters = 0;
  T damping = T(O.damping0);
  for (int it = 0; it < O.max_iterations && term == 0; ++it) {
    T gm = T(0);
    for (int i = tid; i < N; i += traj_threads<G>()) gm = tmax(gm, fabs(S.g[i]));
    if (block_max(gm, S.red) < T(O.grad_tol)) {
      term = 1;
      break;
    }
    bool accepted = false;
    T smax = T(0);
    for (int rj = 0; rj < O.max_rejections; ++rj) {
      const bool ok = traj_damped_solve<G>(S, N, damping);
      T fin = T(1), pp = T(0);
      for (int i = tid; i < N; i += traj_threads<G>()) {
        S.qn[i] = S.q[i] + S.y[i];
        if (!finite_t(S.y[i])) fin = T(0);
        if (sizeof(T) == 4)  // quadratic-model decrease -g.d + lam d^T D d (the FP32 rule below)
          pp += damping * tmax(S.h(i, 0), T(BeamConsts::diag_clamp)) * S.y[i] * S.y[i] - S.g[i] * S.y[i];
      }
      __syncthreads();
      const bool finite_ok = __syncthreads_and(fin > T(0));
      const T pred = sizeof(T) == 4 ? block_sum(pp, S.red) : T(0);
      if (ok && finite_ok) {
        KOP_PROF_T(pe0);
        const T cn = traj_eval<G, false>(C, P, W, S, S.qn);
        KOP_PROF_T(pe1);
        KOP_PROF_ADD(1, pe1 - pe0);
        KOP_PROF_ADD(7, 1);
        if (!finite_t(cn)) {
          term = 5;
          break;
        }
        if (cn < cost) {
          T sm = T(0);
          for (int i = tid; i < N; i += traj_threads<G>()) {
            sm = tmax(sm, fabs(S.y[i]));
            S.q[i] = S.qn[i];
          }
          smax = block_max(sm, S.red);
          cost = cn;
          damping = tmax(damping * T(O.down), T(BeamConsts::damping_min));
          accepted = true;
          break;
        }
        if (sizeof(T) == 4 && pred <= T(kTrajFp32Tau) * cost) {  // FP32 rule (kop_collision.cu kFp32Tau)
          term = 6;
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
    if (tid == 0 && hist_out) hist_out[b * hstride + iters] = double(cost);
    if (smax < T(O.step_tol)) {
      term = 2;
      break;
    }
    KOP_PROF_T(pj0);
    traj_eval<G, true>(C, P, W, S, S.q);
    KOP_PROF_T(pj1);
    KOP_PROF_ADD(0, pj1 - pj0);
    KOP_PROF_ADD(6, 1);
  }
  // outputs + hard-minimum static / swept signed distances (tasks.py:251-275)
  if (hist_out)
    for (int i = iters + 1 + tid; i < hstride; i += traj_threads<G>()) hist_out[b * hstride + i] = NAN;
  for (int i = tid; i < N; i += traj_threads<G>()) {
    const int tt = i / NQ, c = i % NQ;
    if (c < n) q_out[(b * Tn + tt) * n + c] = double(S.q[i]);
  }
  if (tid == 0) {
    cost_out[b] = double(cost);
    iters_out[b] = iters;
    term_out[b] = term;
  }
}

// Normal equations of the trajectory problem at given trajectories (parity
// hook): cost, gradient J^T r and the band of J^T J, unpadded to T*n dense.
template <class G>
__global__ void __launch_bounds__(traj_threads<G>())
k_traj_normal(const ChainParams<typename G::T, G::K> C, const CollisionParams<typename G::T> P,
              const TrajCosts<typename G::T> W, const double* __restrict__ qs, const double* __restrict__ anchors,
              const double* __restrict__ obstacles, int n_obs, int64_t B, double* __restrict__ cost_out,
              double* __restrict__ grad_out, double* __restrict__ hess_out) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, BW = TrajView<G>::BW;
  extern __shared__ unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  const TrajView<G> S(smem_raw, W.T_steps, P.ns);
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x, Tn = W.T_steps, N = Tn * NQ, n = W.n, Nr = Tn * n;
  for (int i = tid; i < 2 * NQ; i += traj_threads<G>()) {
    const int c = i % NQ;
    S.anc[i] = c < n ? T(anchors[(b * 2 + i / NQ) * n + c]) : T(0);
  }
  load_obstacles(*S.obs, obstacles, b, n_obs);
  for (int i = tid; i < N; i += traj_threads<G>()) {
    const int tt = i / NQ, c = i % NQ;
    S.q[i] = c < n ? T(qs[(b * Tn + tt) * n + c]) : T(0);
  }
  __syncthreads();
  const T cost = traj_eval<G, true>(C, P, W, S, S.q);
  if (tid == 0) cost_out[b] = double(cost);
  for (int i = tid; i < N; i += traj_threads<G>()) {
    const int a = i % NQ;
    if (a >= n) continue;
    const int r1 = (i / NQ) * n + a;
    grad_out[b * Nr + r1] = double(S.g[i]);
    for (int d = 0; d <= BW; ++d) {
      const int pc = i - d;
      if (pc < 0 || pc % NQ >= n) continue;
      const int r2 = (pc / NQ) * n + pc % NQ;
      hess_out[(b * Nr + r1) * Nr + r2] = double(S.h(i, d));
      hess_out[(b * Nr + r2) * Nr + r1] = double(S.h(i, d));
    }
  }
}

// trajectory_signed_distances (tasks.py:251-275) and the endpoint pose errors
// of plan_trajectory (tasks.py:412-415) for B finished trajectories, FP64:
// thread t runs the forward pass of q_t, then the static distances of
// timestep t and the swept distances of the pair (t-1, t).
template <class G>
__global__ void __launch_bounds__(traj_threads<G>())
k_traj_report(const ChainParams<double, G::K> C, const CollisionParams<double> P, int steps, int n,
              const double* __restrict__ qs, const double* __restrict__ obstacles, int n_obs,
              const double* __restrict__ targets, int64_t B, double* __restrict__ static_out,
              double* __restrict__ swept_out, double* __restrict__ min_static, double* __restrict__ min_swept,
              double* __restrict__ pos_err, double* __restrict__ rot_err) {
  static_assert(sizeof(typename G::T) == 8, "reports run in FP64");
  constexpr int NQ = G::NQ;
  extern __shared__ unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  const TrajView<G> S(smem_raw, steps, P.ns);
  const int64_t b = blockIdx.x;
  const int tid = threadIdx.x;
  load_obstacles(*S.obs, obstacles, b, n_obs);
  __syncthreads();
  double q[NQ];
  if (tid < steps) {
#pragma unroll
    for (int i = 0; i < NQ; ++i) q[i] = i < n ? qs[(b * steps + tid) * n + i] : 0.0;
    quat<double> eq;
    vec3<double> ep;
    col_forward<G>(C, P, S.lane(tid), q, eq, ep);
  }
  __syncthreads();
  double ds = INFINITY, dw = INFINITY;
  if (tid < steps) {
    const ColLane<G> L1 = S.lane(tid);
    for (int s = 0; s < P.ns; ++s) {
      const vec3<double> c1{L1.cen(s, 0), L1.cen(s, 1), L1.cen(s, 2)};
      for (int o = 0; o < S.obs->no; ++o) {
        vec3<double> nrm;
        ds = fmin(ds, sphere_obstacle_t<double>(*S.obs, o, c1, P.sr[s], nrm));
        if (tid >= 1) {
          const ColLane<G> L0 = S.lane(tid - 1);
          vec3<double> ga, gb;
          dw = fmin(dw, capsule_obstacle_t<double>(*S.obs, o, vec3<double>{L0.cen(s, 0), L0.cen(s, 1), L0.cen(s, 2)},
                                                   c1, P.sr[s], ga, gb));
        }
      }
    }
    if (static_out) static_out[b * steps + tid] = ds;
    if (swept_out && tid >= 1) swept_out[b * (steps - 1) + tid - 1] = dw;
    if (targets && (tid == 0 || tid == steps - 1)) {
      const int e = tid == 0 ? 0 : 1;
      double ti[7], pe, re;
      target_inverse(targets + (b * 2 + e) * 7, ti);
      pose_errors_f64<G::K>(C, q, nullptr, ti, pe, re);
      pos_err[b * 2 + e] = pe;
      rot_err[b * 2 + e] = re;
    }
  }
  ds = -block_max(-ds, S.red);
  dw = -block_max(-dw, S.red);
  if (tid == 0) {
    if (min_static) min_static[b] = ds;
    if (min_swept) min_swept[b] = dw;
  }
}

template <class G>
cudaError_t launch_traj(const ChainParams<typename G::T, G::K>& C, const CollisionParams<typename G::T>& P,
                        const TrajCosts<typename G::T>& W, const TrajLaunch& L, cudaStream_t st) {
  if (L.B == 0) return cudaSuccess;
  const size_t smem = TrajView<G>::bytes(W.T_steps, P.ns);
  cudaFuncSetAttribute(k_traj_solve<G>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaError_t e = cudaFuncSetAttribute(k_traj_solve<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_traj_solve<G><<<(unsigned)L.B, traj_threads<G>(), smem, st>>>(C, P, W, L.q_init, L.anchors, L.obstacles, L.n_obs,
                                                             L.B, L.opts, L.q_out, L.cost_out, L.init_cost,
                                                             L.hist_out, L.iters, L.term);
  return cudaGetLastError();
}

template <class G>
cudaError_t launch_traj_normal(const ChainParams<typename G::T, G::K>& C, const CollisionParams<typename G::T>& P,
                               const TrajCosts<typename G::T>& W, const TrajLaunch& L, cudaStream_t st) {
  if (L.B == 0) return cudaSuccess;
  const size_t smem = TrajView<G>::bytes(W.T_steps, P.ns);
  cudaFuncSetAttribute(k_traj_normal<G>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaError_t e = cudaFuncSetAttribute(k_traj_normal<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_traj_normal<G><<<(unsigned)L.B, traj_threads<G>(), smem, st>>>(C, P, W, L.q_init, L.anchors, L.obstacles, L.n_obs,
                                                              L.B, L.cost_out, L.grad_out, L.hess_out);
  return cudaGetLastError();
}

template <class G>
cudaError_t launch_traj_report(const ChainParams<double, G::K>& C, const CollisionParams<double>& P,
                               const TrajReportLaunch& L, cudaStream_t st) {
  if (L.B == 0) return cudaSuccess;
  const size_t smem = TrajView<G>::bytes(L.steps, P.ns);
  cudaFuncSetAttribute(k_traj_report<G>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  cudaError_t e = cudaFuncSetAttribute(k_traj_report<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_traj_report<G><<<(unsigned)L.B, traj_threads<G>(), smem, st>>>(C, P, L.steps, L.n, L.qs, L.obstacles, L.n_obs,
                                                              L.targets, L.B, L.static_out, L.swept_out,
                                                              L.min_static, L.min_swept, L.pos_err, L.rot_err);
  return cudaGetLastError();
}

template cudaError_t launch_traj_report<Cfg<double, 7, 7, true, false>>(const ChainParams<double, 7>&,
                                                                        const CollisionParams<double>&,
                                                                        const TrajReportLaunch&, cudaStream_t);
template cudaError_t launch_traj_report<Cfg<double, 8, 8, false, false>>(const ChainParams<double, 8>&,
                                                                         const CollisionParams<double>&,
                                                                         const TrajReportLaunch&, cudaStream_t);

#define KOP_TRAJ_INSTANTIATE(T, NQ, K, ID)                                                                   \
  template cudaError_t launch_traj_normal<Cfg<T, NQ, K, ID, false>>(                                        \
      const ChainParams<T, K>&, const CollisionParams<T>&, const TrajCosts<T>&, const TrajLaunch&, cudaStream_t); \
  template cudaError_t launch_traj<Cfg<T, NQ, K, ID, false>>(const ChainParams<T, K>&,                      \
                                                             const CollisionParams<T>&, const TrajCosts<T>&, \
                                                             const TrajLaunch&, cudaStream_t);

KOP_FOR_EACH_COLLISION_SHAPE(KOP_TRAJ_INSTANTIATE)

}  // namespace kop

#ifdef KOP_TRAJ_TIMELINE
extern "C" int kop_debug_traj_timeline(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, kop::g_traj_tl, sizeof(kop::g_traj_tl));
}
#endif
#ifdef KOP_TRAJ_PROFILE
extern "C" int kop_debug_traj_profile(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, kop::g_traj_prof, sizeof(kop::g_traj_prof));
  if (reset) {
    unsigned long long z[20] = {};
    cudaMemcpyToSymbol(kop::g_traj_prof, z, sizeof(z));
  }
  return 0;
}
#endif
