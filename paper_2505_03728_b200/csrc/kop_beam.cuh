// IK-Beam control flow (tasks.py:119-161) as device bodies shared by every
// residual model: the plain pose/limit/rest(/base) lanes (kop_kernels.cu) and
// the collision lanes (kop_collision.cu).  A model factory `mf(tg, scratch)`
// builds the lane's residual model from its target inverse and a per-lane
// shared-memory scratch pointer (stride = block size).
#pragma once

#include "kop_lane.cuh"

namespace kop {

template <class G>
struct Rec {  // survivor record layout: q[NQ], base[3] (BASE), lam, cost, hist[steps1 + 1]
  static constexpr int base = G::NQ;
  static constexpr int lam = G::NQ + (G::BASE ? 3 : 0);
  static constexpr int cost = lam + 1;
  static constexpr int hist = lam + 2;
  static int size(int steps1) { return hist + steps1 + 1; }
};

// ---------------------------------------------------------------------------
// seed frames: the target-independent start evaluation, once per seed
// ---------------------------------------------------------------------------
template <class G>
__global__ void __launch_bounds__(64)
k_seed_frames(const ChainParams<typename G::T, G::K> C, const double* __restrict__ seeds, int S,
              typename G::T* __restrict__ tab) {
  using T = typename G::T;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  T q[G::NQ];
#pragma unroll
  for (int i = 0; i < G::NQ; ++i) q[i] = T(seeds[(size_t)s * G::NQ + i]);
  quat<T> sq;
  vec3<T> sp;
  T col[G::K + (G::BASE ? 3 : 0)][6];
  pose_backward<G, true>(C, q, sq, sp, col);
  tab[0 * S + s] = sq.w; tab[1 * S + s] = sq.x; tab[2 * S + s] = sq.y; tab[3 * S + s] = sq.z;
  tab[4 * S + s] = sp.x; tab[5 * S + s] = sp.y; tab[6 * S + s] = sp.z;
#pragma unroll
  for (int k = 0; k < G::K; ++k)
#pragma unroll
    for (int m = 0; m < 6; ++m) tab[(7 + 6 * k + m) * S + s] = col[k][m];
}

// ---------------------------------------------------------------------------
// IK-Beam stage 1
// ---------------------------------------------------------------------------
// shared memory of stage 1, in elements of T plus 8-byte keys:
// hist [(steps1+1) * TPB] | keys [TPB] (8 B) | Ag [(Tri + ND) * TPB] | scratch [extra * TPB]
template <class G>
__host__ __device__ inline size_t beam_stage1_smem(int tpb, int steps1, int extra) {
  return sizeof(typename G::T) * ((size_t)(steps1 + 1) * tpb + (size_t)(Tri<G::ND>::size + G::ND + extra) * tpb) +
         8 * (size_t)tpb;
}

// SEED_TAB: the start state comes from the seeds' precomputed frames
// (k_seed_frames) and the LM loop holds only the proposal step.
template <class G, int TPB, bool SEED_TAB = false, class MF>
__device__ __forceinline__ void beam_stage1_body(const MF& mf, const double* __restrict__ targets, int64_t B,
                                                 const double* __restrict__ seeds, int S, int P, int steps1,
                                                 int keep, typename G::T* __restrict__ surv, int rec,
                                                 const typename G::T* __restrict__ seed_tab = nullptr) {
  using T = typename G::T;
  constexpr int NQ = G::NQ;
  extern __shared__ unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  T* hist = reinterpret_cast<T*>(smem_raw);  // [(steps1+1) * TPB]
  unsigned long long* keys =                  // [TPB] 8-byte prune keys (or double costs)
      reinterpret_cast<unsigned long long*>(hist + (size_t)(steps1 + 1) * TPB);
  T* Ag = reinterpret_cast<T*>(keys + TPB);  // [(Tri + ND) * TPB]
  T* scratch = Ag + (size_t)(Tri<G::ND>::size + G::ND) * TPB;
  const int tid = threadIdx.x;
  const int64_t tgt = (int64_t)blockIdx.x * (TPB / P) + tid / P;
  const int s = tid % P;
  const bool active = (tgt < B) && (s < S);
  const int64_t tc = tgt < B ? tgt : B - 1;
  const TargetInv<T> tg = target_inverse_t<T>(targets + tc * 7);

  LaneState<G> st;
  st.Ag = Ag + tid;
  st.stride = TPB;
  const double* sd = seeds + (size_t)(s < S ? s : 0) * NQ;
#pragma unroll
  for (int i = 0; i < NQ; ++i) st.q[i] = T(sd[i]);
  st.base[0] = st.base[1] = st.base[2] = T(0);  // every seed starts with the base at identity
  st.lam = T(BeamConsts::damping_init);
  const auto model = mf(tg, scratch + tid);
  if constexpr (SEED_TAB) {  // start_state (beam.py:182-196) from the seed's frame
    T A[Tri<G::ND>::size], g[G::ND];
    const T raw = model.eval_seed(seed_tab, S, s < S ? s : 0, st.q, st.base, A, g);
    store_normal<TPB>(st, A, g);
    st.cost = raw;
    hist[tid] = st.cost;
    for (int it = 1; it <= steps1; ++it) {
      lm_iter<G, TPB>(model, st, 0);
      hist[(size_t)it * TPB + tid] = st.cost;
    }
  } else {
    for (int it = 0; it <= steps1; ++it) {  // it == 0: start_state
      lm_iter<G, TPB>(model, st, it == 0 ? 1 : 0);
      hist[(size_t)it * TPB + tid] = st.cost;
    }
  }
  // stable top-`keep` of the target's S lanes (tasks.py:135): rank = number of
  // lanes ordered before this one by (cost, seed index), NaN last
  const int basel = tid - s;
  int rank = 0;
  if constexpr (sizeof(T) == 4) {
    keys[tid] = active ? prune_key(st.cost, s) : ~0ull;  // padding lanes sort last
    __syncthreads();
    if (!active) return;
    const unsigned long long me = keys[tid];
    if (P >= 2) {
      const ulonglong2* kv = reinterpret_cast<const ulonglong2*>(keys + basel);
#pragma unroll 8
      for (int j = 0; j < P / 2; ++j) {
        const ulonglong2 v = kv[j];
        rank += (v.x < me ? 1 : 0) + (v.y < me ? 1 : 0);
      }
    }
  } else {
    T* costs = reinterpret_cast<T*>(keys);
    costs[tid] = active ? st.cost : T(NAN);
    __syncthreads();
    if (!active) return;
    for (int j = 0; j < S; ++j) rank += rank_less(costs[basel + j], j, st.cost, s) ? 1 : 0;
  }
  if (rank >= keep) return;
  T* out = surv + (size_t)(tgt * keep + rank) * rec;
#pragma unroll
  for (int i = 0; i < NQ; ++i) out[i] = st.q[i];
  if (G::BASE) {
    out[Rec<G>::base] = st.base[0];
    out[Rec<G>::base + 1] = st.base[1];
    out[Rec<G>::base + 2] = st.base[2];
  }
  out[Rec<G>::lam] = st.lam;
  out[Rec<G>::cost] = st.cost;
  for (int h = 0; h <= steps1; ++h) out[Rec<G>::hist + h] = hist[(size_t)h * TPB + tid];
}

// ---------------------------------------------------------------------------
// IK-Beam stage 2 + winner + pose errors
// ---------------------------------------------------------------------------
template <int K>
__device__ __forceinline__ void chain_pose_f64(const ChainParams<double, K>& C, const double* q,
                                               quat<double>& eq, vec3<double>& ep) {
  quat<double> pq{1.0, 0.0, 0.0, 0.0};
  vec3<double> pp{0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (k < C.k) {
      const quat<double> tq{C.tq[k][0], C.tq[k][1], C.tq[k][2], C.tq[k][3]};
      const vec3<double> tp{C.tp[k][0], C.tp[k][1], C.tp[k][2]};
      const quat<double> fq = qmul(pq, tq);
      const vec3<double> o = qrot(pq, tp);
      const vec3<double> fp{pp.x + o.x, pp.y + o.y, pp.z + o.z};
      const double th = q[C.qcol[k]] * C.mult[k] + C.offset[k];
      if (C.prismatic[k]) {
        const vec3<double> z = qzaxis(fq);
        pq = fq;
        pp = {fp.x + th * z.x, fp.y + th * z.y, fp.z + th * z.z};
      } else {
        double sn, cs;
        sincos(0.5 * th, &sn, &cs);
        pq = qmul_z(fq, cs, sn);
        pp = fp;
      }
    }
  }
  eq = qmul(pq, quat<double>{C.eq[0], C.eq[1], C.eq[2], C.eq[3]});
  const vec3<double> eo = qrot(pq, vec3<double>{C.ep[0], C.ep[1], C.ep[2]});
  ep = {pp.x + eo.x, pp.y + eo.y, pp.z + eo.z};
}

// tasks.py:109-116: |t(T_t^-1 (B) T)| and |log R(T_t^-1 (B) T)| in double;
// base = (x, y, angle) or NULL.
template <int K>
__device__ __forceinline__ void pose_errors_f64(const ChainParams<double, K>& C, const double* q,
                                                const double* base, const double tinv[7], double& pe,
                                                double& re) {
  quat<double> eq;
  vec3<double> ep;
  chain_pose_f64<K>(C, q, eq, ep);
  const double n = sqrt(eq.w * eq.w + eq.x * eq.x + eq.y * eq.y + eq.z * eq.z);
  eq = {eq.w / n, eq.x / n, eq.y / n, eq.z / n};
  if (base) {  // Transform2.to_transform3().compose(current) (liegroups.py:449-453)
    double sh, ch;
    sincos(0.5 * base[2], &sh, &ch);
    const quat<double> bq{ch, 0.0, 0.0, sh};
    const vec3<double> r = qrot(bq, ep);
    eq = qmul(bq, eq);
    ep = {base[0] + r.x, base[1] + r.y, r.z};
  }
  const quat<double> iq{tinv[0], tinv[1], tinv[2], tinv[3]};
  const quat<double> rq = qmul(iq, eq);
  const vec3<double> rt = qrot(iq, ep);
  const vec3<double> t{tinv[4] + rt.x, tinv[5] + rt.y, tinv[6] + rt.z};
  pe = sqrt(t.x * t.x + t.y * t.y + t.z * t.z);
  const vec3<double> w = qlog(rq);
  re = sqrt(w.x * w.x + w.y * w.y + w.z * w.z);
}

// shared memory of stage 2 (BD threads): hist [steps2 * BD] | Ag | scratch
template <class G, int BD = 128>
__host__ __device__ inline size_t beam_stage2_smem(int steps2, int extra) {
  return sizeof(typename G::T) * ((size_t)(steps2 > 0 ? steps2 : 1) * BD +
                                  (size_t)(Tri<G::ND>::size + G::ND + extra) * BD);
}

template <class G, int BD = 128, class MF>
__device__ __forceinline__ void beam_stage2_body(const MF& mf, const ChainParams<double, G::K>& Cd,
                                                 const double* __restrict__ targets, int64_t B,
                                                 const typename G::T* __restrict__ surv, int rec, int steps1,
                                                 int steps2, int keep, int G2, double pos_tol, double rot_tol,
                                                 double* __restrict__ q_out, double* __restrict__ base_out,
                                                 double* __restrict__ cost_out, double* __restrict__ hist_out,
                                                 double* __restrict__ pos_err, double* __restrict__ rot_err,
                                                 uint8_t* __restrict__ success) {
  using T = typename G::T;
  constexpr int NQ = G::NQ;
  constexpr int bd = BD;
  extern __shared__ unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  T* hist = reinterpret_cast<T*>(smem_raw);  // [steps2 * bd]
  T* Ag = hist + (size_t)(steps2 > 0 ? steps2 : 1) * bd;  // [(Tri + ND) * bd]
  T* scratch = Ag + (size_t)(Tri<G::ND>::size + G::ND) * bd;
  const int tid = threadIdx.x;
  const int64_t lane = (int64_t)blockIdx.x * bd + tid;
  const int64_t tgt = lane / G2;
  const int r = (int)(lane % G2);
  const bool active = (tgt < B) && (r < keep);
  const int64_t tc = tgt < B ? tgt : B - 1;
  const int rc = r < keep ? r : 0;
  const TargetInv<T> tg = target_inverse_t<T>(targets + tc * 7);
  const T* rin = surv + (size_t)(tc * keep + rc) * rec;

  LaneState<G> st;
  st.Ag = Ag + tid;
  st.stride = bd;
#pragma unroll
  for (int i = 0; i < NQ; ++i) st.q[i] = rin[i];
  st.base[0] = st.base[1] = st.base[2] = T(0);
  if (G::BASE) {
    st.base[0] = rin[Rec<G>::base];
    st.base[1] = rin[Rec<G>::base + 1];
    st.base[2] = rin[Rec<G>::base + 2];
  }
  st.lam = rin[Rec<G>::lam];
  // the carried cost is the stage-1 state cost (LaneState.select, beam.py:60-68);
  // A/g are re-derived at q, as the reference re-derives r and J (beam.py:202)
  st.cost = rin[Rec<G>::cost];
  const auto model = mf(tg, scratch + tid);
  for (int it = -1; it < steps2; ++it) {  // it == -1: re-derive A, g at the survivor
    lm_iter<G, BD>(model, st, it < 0 ? 2 : 0);
    if (it >= 0) hist[(size_t)it * bd + tid] = st.cost;
  }
  // winner = argmin over the keep survivors, ties -> lower stage-1 rank (tasks.py:139)
  T best = active ? st.cost : T(NAN);
  int bidx = active ? r : (1 << 30);
  for (int off = G2 >> 1; off > 0; off >>= 1) {
    const T oc = __shfl_xor_sync(0xffffffffu, best, off);
    const int oi = __shfl_xor_sync(0xffffffffu, bidx, off);
    if (rank_less(oc, oi, best, bidx)) {
      best = oc;
      bidx = oi;
    }
  }
  if (!active || bidx != r) return;
  double qd[NQ], bd3[3] = {0.0, 0.0, 0.0};
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    qd[i] = double(st.q[i]);
    q_out[tgt * NQ + i] = qd[i];
  }
  if (G::BASE) {
    for (int i = 0; i < 3; ++i) bd3[i] = double(st.base[i]);
    if (base_out)
      for (int i = 0; i < 3; ++i) base_out[tgt * 3 + i] = bd3[i];
  }
  cost_out[tgt] = double(st.cost);
  if (hist_out) {
    double* h = hist_out + tgt * (steps1 + 1 + steps2);
    for (int i = 0; i <= steps1; ++i) h[i] = double(rin[Rec<G>::hist + i]);
    for (int i = 0; i < steps2; ++i) h[steps1 + 1 + i] = double(hist[(size_t)i * bd + tid]);
  }
  if (G::BASE) {  // mobile lanes: errors here (the base may not be written out)
    double tinv[7];
    target_inverse(targets + tgt * 7, tinv);
    double pe, re;
    pose_errors_f64<G::K>(Cd, qd, bd3, tinv, pe, re);
    pos_err[tgt] = pe;
    rot_err[tgt] = re;
    success[tgt] = (pe < pos_tol && re < rot_tol) ? 1 : 0;
  }
}

// FP64 pose errors and success of the winners (tasks.py:109-116, 147), one
// thread per target after stage 2 (fixed-base shapes).  Kept out of stage 2 so
// its LM loop is not diluted by FP64 code run by one lane in four.
template <int K, int NQ>
__global__ void __launch_bounds__(128)
k_beam_errors(const ChainParams<double, K> Cd, const double* __restrict__ targets, int64_t B,
              const double* __restrict__ q_out, double pos_tol, double rot_tol, double* __restrict__ pos_err,
              double* __restrict__ rot_err, uint8_t* __restrict__ success) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= B) return;
  double qd[NQ];
#pragma unroll
  for (int i = 0; i < NQ; ++i) qd[i] = q_out[t * NQ + i];
  double tinv[7];
  target_inverse(targets + t * 7, tinv);
  double pe, re;
  pose_errors_f64<K>(Cd, qd, nullptr, tinv, pe, re);
  pos_err[t] = pe;
  rot_err[t] = re;
  success[t] = (pe < pos_tol && re < rot_tol) ? 1 : 0;
}

template <class G>
cudaError_t launch_beam_errors(const ChainParams<double, G::K>& Cd, const double* targets, int64_t B,
                               const double* q_out, double pos_tol, double rot_tol, double* pos_err,
                               double* rot_err, uint8_t* success, cudaStream_t st) {
  if (G::BASE || B == 0) return cudaSuccess;
  k_beam_errors<G::K, G::NQ><<<(unsigned)((B + 127) / 128), 128, 0, st>>>(Cd, targets, B, q_out, pos_tol, rot_tol,
                                                                         pos_err, rot_err, success);
  return cudaGetLastError();
}

}  // namespace kop
