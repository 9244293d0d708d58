// sm_100a kernels of the batched LM-IK engine.
//
//   k_beam_stage1  one thread per (target, seed) lane: start + prune_after LM
//                  steps + in-CTA stable top-`keep` prune (tasks.py:131-136)
//   k_beam_stage2  one thread per survivor: remaining LM steps, segmented
//                  warp-shuffle argmin (tasks.py:137-161)
//   k_beam_errors  one thread per target: FP64 pose errors / success of the
//                  winner (tasks.py:109-116, 147)
//   k_lane_*       the IkLaneProblem API (beam.py:133-240), one thread/lane
//
// Mapping: the workload is compute/latency bound (FP32 FMA + MUFU), so lanes
// map to threads with the whole LM state in registers; model constants are
// kernel parameters (constant bank).  Blocks are 256 threads (4 targets x 64
// seeds) in stage 1; shared memory holds the per-lane normal equations, the
// cost history and the prune keys.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kop_beam.cuh"
#include "kop_kernels.cuh"

namespace kop {

// Residual-model factory for the plain IK lanes.
template <class G>
struct PoseModelFactory {
  const ChainParams<typename G::T, G::K>& C;
  const CostParams<typename G::T, G::NQ>& W;
  __device__ __forceinline__ PoseModel<G> operator()(const TargetInv<typename G::T>& tg,
                                                     typename G::T* /*scratch*/) const {
    return PoseModel<G>{C, W, tg};
  }
};

// resident 256-thread CTAs per SM the register allocation targets: FP32 2 (128 registers,
// 16 warps); FP64 KOP_STAGE1_MINB64 (A/B-measured)
#ifndef KOP_STAGE1_MINB64
#define KOP_STAGE1_MINB64 2
#endif
#ifndef KOP_STAGE2_MINB64
#define KOP_STAGE2_MINB64 4
#endif
template <class G>
constexpr int stage1_min_blocks(int tpb) {
  return tpb > 256 ? 1 : (sizeof(typename G::T) == 8 ? KOP_STAGE1_MINB64 : 2);
}

template <class G, int TPB>
__global__ void __launch_bounds__(TPB, stage1_min_blocks<G>(TPB))
k_beam_stage1(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
              const double* __restrict__ targets, int64_t B, const double* __restrict__ seeds, int S, int P,
              int steps1, int keep, typename G::T* __restrict__ surv, int rec,
              const typename G::T* __restrict__ seed_tab) {
  // fixed-base lanes start from the seed frames (k_seed_frames); mobile lanes evaluate in place
  beam_stage1_body<G, TPB, !G::BASE>(PoseModelFactory<G>{C, W}, targets, B, seeds, S, P, steps1, keep, surv,
                                     rec, seed_tab);
}

constexpr int kStage2Threads = 128;

template <class G>
__global__ void __launch_bounds__(kStage2Threads, sizeof(typename G::T) == 8 ? KOP_STAGE2_MINB64 : 4)
k_beam_stage2(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
              const ChainParams<double, G::K> Cd, const double* __restrict__ targets, int64_t B,
              const typename G::T* __restrict__ surv, int rec, int steps1, int steps2, int keep, int G2,
              double pos_tol, double rot_tol, double* __restrict__ q_out, double* __restrict__ base_out,
              double* __restrict__ cost_out, double* __restrict__ hist_out, double* __restrict__ pos_err,
              double* __restrict__ rot_err, uint8_t* __restrict__ success) {
  beam_stage2_body<G, kStage2Threads>(PoseModelFactory<G>{C, W}, Cd, targets, B, surv, rec, steps1, steps2, keep,
                                      G2, pos_tol,
                      rot_tol, q_out, base_out, cost_out, hist_out, pos_err, rot_err, success);
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
  extern __shared__ unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  if (l >= lanes) return;
  const TargetInv<T> tg = load_target_inv<T>(tinv + (int64_t)lane_target[l] * 7);
  LaneState<G> st;
  st.Ag = reinterpret_cast<T*>(smem_raw) + threadIdx.x;
  st.stride = 128;
  load_lane<G>(q_io, base_io, l, st.q, st.base);
  st.lam = T(lam_io[l]);
  st.cost = T(cost_io[l]);
  const PoseModel<G> model{C, W, tg};
  for (int it = -1; it < steps; ++it) {
    lm_iter<G, 128>(model, st, it < 0 ? 2 : 0);
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
  // seed frame table after the survivor records (kop_ik_beam_workspace_bytes)
  T* seed_tab = reinterpret_cast<T*>(static_cast<char*>(L.workspace) +
                                     ((size_t)L.B * L.keep * rec * sizeof(T) + 255) / 256 * 256);
  if (L.stages & 1) {
    if (!G::BASE) {
      k_seed_frames<G><<<(L.S + 63) / 64, 64, 0, st>>>(C, L.seeds, L.S, seed_tab);
      e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    // stage 1: P lanes per target (power of two >= S)
    const int tpb = L.P <= 256 ? 256 : 1024;  // P <= 1024 (seeds <= 1024)
    const int per_block = tpb / L.P;
    const int64_t blocks1 = (L.B + per_block - 1) / per_block;
    const size_t smem1 = beam_stage1_smem<G>(tpb, L.steps1, 0);
    // FP64 with > 256 seeds needs ~350 KB per 1024-thread CTA: refuse instead of a generic launch failure
    int dev = 0, optin = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess ||
        (e = cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev)) != cudaSuccess)
      return e;
    if (smem1 > (size_t)optin) return cudaErrorNotSupported;
    if (tpb == 256) {
      if (smem1 > 48 * 1024 &&
          (e = cudaFuncSetAttribute(k_beam_stage1<G, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem1)) != cudaSuccess)
        return e;
      k_beam_stage1<G, 256><<<(unsigned)blocks1, 256, smem1, st>>>(C, W, L.targets, L.B, L.seeds, L.S, L.P,
                                                                   L.steps1, L.keep, surv, rec, seed_tab);
    } else {
      if (smem1 > 48 * 1024 &&
          (e = cudaFuncSetAttribute(k_beam_stage1<G, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem1)) != cudaSuccess)
        return e;
      k_beam_stage1<G, 1024><<<(unsigned)blocks1, 1024, smem1, st>>>(C, W, L.targets, L.B, L.seeds, L.S, L.P,
                                                                     L.steps1, L.keep, surv, rec, seed_tab);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (!(L.stages & 2)) return cudaSuccess;
  const int tpb2 = kStage2Threads;
  const int64_t lanes2 = L.B * L.G;
  const int64_t blocks2 = (lanes2 + tpb2 - 1) / tpb2;
  const size_t smem2 = beam_stage2_smem<G, kStage2Threads>(L.steps2, 0);
  if (smem2 > 48 * 1024)
    cudaFuncSetAttribute(k_beam_stage2<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  k_beam_stage2<G><<<(unsigned)blocks2, tpb2, smem2, st>>>(
      C, W, Cd, L.targets, L.B, surv, rec, L.steps1, L.steps2, L.keep, L.G, L.pos_tol, L.rot_tol, L.q_out,
      L.base_out, L.cost_out, L.hist_out, L.pos_err, L.rot_err, L.success);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_beam_errors<G>(Cd, L.targets, L.B, L.q_out, L.pos_tol, L.rot_tol, L.pos_err, L.rot_err, L.success,
                               st);
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
