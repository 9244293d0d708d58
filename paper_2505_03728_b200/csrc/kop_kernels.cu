// sm_100a kernels of the batched LM-IK engine.
//
//   k_beam_stage1  one thread per (target, seed) lane: start + prune_after LM
//                  steps + in-CTA stable top-`keep` prune (tasks.py:131-136)
//   k_beam_stage2  one thread per survivor: remaining LM steps, segmented
//                  warp-shuffle argmin, FP64 pose errors (tasks.py:137-161)
//   k_lane_*       the IkLaneProblem API (beam.py:133-240), one thread/lane
//
// Mapping: the workload is compute/latency bound (FP32 FMA + MUFU), so lanes
// map to threads with the whole LM state in registers; model constants are
// kernel parameters (constant bank).  Blocks are 256 threads (4 targets x 64
// seeds) in stage 1; shared memory holds the per-lane normal equations, the
// cost history and the prune keys.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kop_kernels.cuh"

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
// IK-Beam stage 1
// ---------------------------------------------------------------------------
template <class G, int TPB>
__global__ void __launch_bounds__(TPB, (TPB <= 256 ? 2 : 1))
k_beam_stage1(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
              const double* __restrict__ targets, int64_t B, const double* __restrict__ seeds, int S, int P,
              int steps1, int keep, typename G::T* __restrict__ surv, int rec) {
  using T = typename G::T;
  constexpr int NQ = G::NQ;
  extern __shared__ unsigned char smem_raw[];
  T* hist = reinterpret_cast<T*>(smem_raw);  // [(steps1+1) * TPB]
  unsigned long long* keys =                  // [TPB] 8-byte prune keys (or double costs)
      reinterpret_cast<unsigned long long*>(hist + (size_t)(steps1 + 1) * TPB);
  T* Ag = reinterpret_cast<T*>(keys + TPB);  // [(Tri + ND) * TPB]
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
  for (int it = 0; it <= steps1; ++it) {  // it == 0: start_state
    lm_iter<G, TPB>(C, W, tg, st, it == 0 ? 1 : 0);
    hist[(size_t)it * TPB + tid] = st.cost;
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

template <class G>
__global__ void __launch_bounds__(128, 4)
k_beam_stage2(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
              const ChainParams<double, G::K> Cd, const double* __restrict__ targets, int64_t B,
              const typename G::T* __restrict__ surv, int rec, int steps1, int steps2, int keep, int G2,
              double pos_tol, double rot_tol, double* __restrict__ q_out, double* __restrict__ base_out,
              double* __restrict__ cost_out, double* __restrict__ hist_out, double* __restrict__ pos_err,
              double* __restrict__ rot_err, uint8_t* __restrict__ success) {
  using T = typename G::T;
  constexpr int NQ = G::NQ;
  constexpr int bd = 128;  // launch_beam launches stage 2 with 128 threads
  extern __shared__ unsigned char smem_raw[];
  T* hist = reinterpret_cast<T*>(smem_raw);  // [steps2 * bd]
  T* Ag = hist + (size_t)(steps2 > 0 ? steps2 : 1) * bd;  // [(Tri + ND) * bd]
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
  for (int it = -1; it < steps2; ++it) {  // it == -1: re-derive A, g at the survivor
    lm_iter<G, 128>(C, W, tg, st, it < 0 ? 2 : 0);
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
  double tinv[7];
  target_inverse(targets + tgt * 7, tinv);
  double pe, re;
  pose_errors_f64<G::K>(Cd, qd, G::BASE ? bd3 : nullptr, tinv, pe, re);
  pos_err[tgt] = pe;
  rot_err[tgt] = re;
  success[tgt] = (pe < pos_tol && re < rot_tol) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// Lane API kernels (IkLaneProblem with one target per lane); the base state
// (x, y, angle) per lane is read/written when G::BASE.
// ---------------------------------------------------------------------------
template <class G>
__device__ __forceinline__ void load_lane(const double* q_in, const double* base_in, int64_t l,
                                          typename G::T (&q)[G::NQ], typename G::T (&b)[3]) {
  using T = typename G::T;
#pragma unroll
  for (int i = 0; i < G::NQ; ++i) q[i] = T(q_in[l * G::NQ + i]);
  b[0] = b[1] = b[2] = T(0);
  if (G::BASE)
    for (int i = 0; i < 3; ++i) b[i] = T(base_in[l * 3 + i]);
}

template <class G>
__global__ void __launch_bounds__(128)
k_lane_resjac(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
              const double* __restrict__ tinv, const int32_t* __restrict__ lane_target,
              const double* __restrict__ q_in, const double* __restrict__ base_in, int64_t lanes,
              double* __restrict__ res, double* __restrict__ jac) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, ND = G::ND;
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= lanes) return;
  const TargetInv<T> tg = load_target_inv<T>(tinv + (int64_t)lane_target[l] * 7);
  T q[NQ], b[3];
  load_lane<G>(q_in, base_in, l, q, b);
  T r[6], J[6][ND];
  pose_rows<G, true>(C, W, tg, q, b, r, J);
  T rl[NQ], gl[NQ], rr[NQ];
  diag_rows(W, q, rl, gl, rr);
  constexpr int M = 6 + 2 * NQ + (G::BASE ? 3 : 0);
  double* ro = res + l * M;
  double* jo = jac + l * M * ND;
  for (int i = 0; i < M * ND; ++i) jo[i] = 0.0;
#pragma unroll
  for (int m = 0; m < 6; ++m) {
    ro[m] = double(r[m]);
#pragma unroll
    for (int c = 0; c < ND; ++c) jo[m * ND + c] = double(J[m][c]);
  }
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    ro[6 + i] = double(rl[i]);
    ro[6 + NQ + i] = double(rr[i]);
    jo[(6 + i) * ND + i] = double(gl[i]);
    jo[(6 + NQ + i) * ND + i] = double(W.w_rest);
  }
  if (G::BASE) {  // beam.py:127-130, 171-178
    const int rb = 6 + 2 * NQ;
    const T ca = cos(b[2]), sa = sin(b[2]);
    for (int i = 0; i < 3; ++i) ro[rb + i] = double(W.w_base * b[i]);
    jo[rb * ND + NQ] = double(W.w_base * ca);
    jo[rb * ND + NQ + 1] = double(-W.w_base * sa);
    jo[(rb + 1) * ND + NQ] = double(W.w_base * sa);
    jo[(rb + 1) * ND + NQ + 1] = double(W.w_base * ca);
    jo[(rb + 2) * ND + NQ + 2] = double(W.w_base);
  }
}

template <class G>
__global__ void __launch_bounds__(128)
k_lane_start(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
             const double* __restrict__ tinv, const int32_t* __restrict__ lane_target,
             const double* __restrict__ q_in, const double* __restrict__ base_in, int64_t lanes,
             double* __restrict__ lam, double* __restrict__ cost) {
  using T = typename G::T;
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= lanes) return;
  const TargetInv<T> tg = load_target_inv<T>(tinv + (int64_t)lane_target[l] * 7);
  T q[G::NQ], b[3], A[Tri<G::ND>::size], g[G::ND];
  load_lane<G>(q_in, base_in, l, q, b);
  cost[l] = double(lane_eval<G, false>(C, W, tg, q, b, A, g));
  lam[l] = BeamConsts::damping_init;
}

template <class G>
__global__ void __launch_bounds__(128, 4)
k_lane_run(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
           const double* __restrict__ tinv, const int32_t* __restrict__ lane_target, int64_t lanes, int steps,
           double* __restrict__ q_io, double* __restrict__ base_io, double* __restrict__ lam_io,
           double* __restrict__ cost_io, double* __restrict__ hist) {
  using T = typename G::T;
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= lanes) return;
  extern __shared__ unsigned char smem_raw[];
  const TargetInv<T> tg = load_target_inv<T>(tinv + (int64_t)lane_target[l] * 7);
  LaneState<G> st;
  st.Ag = reinterpret_cast<T*>(smem_raw) + threadIdx.x;
  st.stride = 128;
  load_lane<G>(q_io, base_io, l, st.q, st.base);
  st.lam = T(lam_io[l]);
  st.cost = T(cost_io[l]);
  for (int it = -1; it < steps; ++it) {
    lm_iter<G, 128>(C, W, tg, st, it < 0 ? 2 : 0);
    if (hist && it >= 0) hist[l * steps + it] = double(st.cost);
  }
#pragma unroll
  for (int i = 0; i < G::NQ; ++i) q_io[l * G::NQ + i] = double(st.q[i]);
  if (G::BASE)
    for (int i = 0; i < 3; ++i) base_io[l * 3 + i] = double(st.base[i]);
  lam_io[l] = double(st.lam);
  cost_io[l] = double(st.cost);
}

// ---------------------------------------------------------------------------
// Launchers (instantiated per supported shape)
// ---------------------------------------------------------------------------
template <class G>
cudaError_t launch_beam(const ChainParams<typename G::T, G::K>& C, const CostParams<typename G::T, G::NQ>& W,
                        const ChainParams<double, G::K>& Cd, const BeamLaunch& L, cudaStream_t st) {
  using T = typename G::T;
  const int rec = Rec<G>::size(L.steps1);
  T* surv = reinterpret_cast<T*>(L.workspace);
  constexpr int kAg = Tri<G::ND>::size + G::ND;
  cudaError_t e = cudaSuccess;
  if (L.stages & 1) {
    // stage 1: P lanes per target (power of two >= S)
    const int tpb = L.P <= 256 ? 256 : 1024;  // P <= 1024 (seeds <= 1024)
    const int per_block = tpb / L.P;
    const int64_t blocks1 = (L.B + per_block - 1) / per_block;
    const size_t smem1 = sizeof(T) * ((size_t)(L.steps1 + 1) * tpb + (size_t)kAg * tpb) + 8 * (size_t)tpb;
    if (tpb == 256) {
      if (smem1 > 48 * 1024)
        cudaFuncSetAttribute(k_beam_stage1<G, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
      k_beam_stage1<G, 256><<<(unsigned)blocks1, 256, smem1, st>>>(C, W, L.targets, L.B, L.seeds, L.S, L.P,
                                                                   L.steps1, L.keep, surv, rec);
    } else {
      if (smem1 > 48 * 1024)
        cudaFuncSetAttribute(k_beam_stage1<G, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
      k_beam_stage1<G, 1024><<<(unsigned)blocks1, 1024, smem1, st>>>(C, W, L.targets, L.B, L.seeds, L.S, L.P,
                                                                     L.steps1, L.keep, surv, rec);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (!(L.stages & 2)) return cudaSuccess;
  const int tpb2 = 128;
  const int64_t lanes2 = L.B * L.G;
  const int64_t blocks2 = (lanes2 + tpb2 - 1) / tpb2;
  const size_t smem2 = sizeof(T) * ((size_t)(L.steps2 > 0 ? L.steps2 : 1) * tpb2 + (size_t)kAg * tpb2);
  if (smem2 > 48 * 1024)
    cudaFuncSetAttribute(k_beam_stage2<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  k_beam_stage2<G><<<(unsigned)blocks2, tpb2, smem2, st>>>(
      C, W, Cd, L.targets, L.B, surv, rec, L.steps1, L.steps2, L.keep, L.G, L.pos_tol, L.rot_tol, L.q_out,
      L.base_out, L.cost_out, L.hist_out, L.pos_err, L.rot_err, L.success);
  return cudaGetLastError();
}

template <class G>
cudaError_t launch_lane(const ChainParams<typename G::T, G::K>& C, const CostParams<typename G::T, G::NQ>& W,
                        const LaneLaunch& L, cudaStream_t st) {
  using T = typename G::T;
  const int tpb = 128;
  const unsigned blocks = (unsigned)((L.lanes + tpb - 1) / tpb);
  if (L.lanes == 0) return cudaSuccess;
  switch (L.op) {
    case LaneOp::kResJac:
      k_lane_resjac<G><<<blocks, tpb, 0, st>>>(C, W, L.tinv, L.lane_target, L.q_in, L.base_in, L.lanes, L.res,
                                               L.jac);
      break;
    case LaneOp::kStart:
      k_lane_start<G><<<blocks, tpb, 0, st>>>(C, W, L.tinv, L.lane_target, L.q_in, L.base_in, L.lanes, L.lam,
                                              L.cost);
      break;
    case LaneOp::kRun: {
      const size_t smem = sizeof(T) * (Tri<G::ND>::size + G::ND) * tpb;
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_lane_run<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      k_lane_run<G><<<blocks, tpb, smem, st>>>(C, W, L.tinv, L.lane_target, L.lanes, L.steps, L.q_io, L.base_io,
                                               L.lam, L.cost, L.hist);
      break;
    }
  }
  return cudaGetLastError();
}

#define KOP_INSTANTIATE(T, NQ, K, ID, BASE)                                                                 \
  template cudaError_t launch_beam<Cfg<T, NQ, K, ID, BASE>>(const ChainParams<T, K>&, const CostParams<T, NQ>&, \
                                                            const ChainParams<double, K>&, const BeamLaunch&,   \
                                                            cudaStream_t);                                      \
  template cudaError_t launch_lane<Cfg<T, NQ, K, ID, BASE>>(const ChainParams<T, K>&, const CostParams<T, NQ>&, \
                                                            const LaneLaunch&, cudaStream_t);

KOP_FOR_EACH_SHAPE(KOP_INSTANTIATE)

}  // namespace kop
