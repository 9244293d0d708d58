// Collision IK kernels (config 4) and the generic classic-LM solve.
//
//   k_col_resjac       weighted residual stack + Jacobian rows per lane (parity API)
//   k_col_beam_stage1  IK-Beam (tasks.py:119-161) over the collision stack
//   k_col_beam_stage2
//   k_col_solve        solver.solve (solver.py:364-429): classic LM with the
//                      rejection loop, gradient / step / numerical-failure
//                      terminations, one problem per thread
//
// The per-lane scratch (Pluecker axes + sphere centres, kop_collision.cuh)
// lives in shared memory; blocks are 128 threads.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "kop_beam.cuh"
#include "kop_collision.cuh"
#include "kop_kernels.cuh"

namespace kop {

template <class G>
struct CollisionModelFactory {
  using T = typename G::T;
  const ChainParams<T, G::K>& C;
  const CostParams<T, G::NQ>& W;
  const CollisionParams<T>& P;
  int stride;
  __device__ __forceinline__ CollisionModel<G> operator()(const TargetInv<T>& tg, T* scratch) const {
    return CollisionModel<G>{C, W, P, tg, ColLane<G>{scratch, stride}};
  }
};

// resident 128-thread CTAs per SM the register allocation targets: FP32 3 (168 registers);
// FP64 2 (255 registers, 268 B spill instead of 168 registers with 1.6 KB / 3.6 KB spill stores /
// loads: 204 -> 174 ms on 100K config-4 targets, A/B via KOP_COL_BEAM_MINB64)
#ifndef KOP_COL_BEAM_MINB64
#define KOP_COL_BEAM_MINB64 2
#endif
template <class G>
constexpr int col_beam_min_blocks() { return sizeof(typename G::T) == 8 ? KOP_COL_BEAM_MINB64 : 3; }

template <class G>
__global__ void __launch_bounds__(128, col_beam_min_blocks<G>())
k_col_beam_stage1(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
                  const CollisionParams<typename G::T> P, const double* __restrict__ targets, int64_t B,
                  const double* __restrict__ seeds, int S, int Pw, int steps1, int keep,
                  typename G::T* __restrict__ surv, int rec) {
  beam_stage1_body<G, 128>(CollisionModelFactory<G>{C, W, P, 128}, targets, B, seeds, S, Pw, steps1, keep, surv,
                           rec);
}

template <class G>
__global__ void __launch_bounds__(128, col_beam_min_blocks<G>())
k_col_beam_stage2(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
                  const CollisionParams<typename G::T> P, const ChainParams<double, G::K> Cd,
                  const double* __restrict__ targets, int64_t B, const typename G::T* __restrict__ surv, int rec,
                  int steps1, int steps2, int keep, int G2, double pos_tol, double rot_tol,
                  double* __restrict__ q_out, double* __restrict__ cost_out, double* __restrict__ hist_out,
                  double* __restrict__ pos_err, double* __restrict__ rot_err, uint8_t* __restrict__ success) {
  beam_stage2_body<G>(CollisionModelFactory<G>{C, W, P, 128}, Cd, targets, B, surv, rec, steps1, steps2, keep, G2,
                      pos_tol, rot_tol, q_out, nullptr, cost_out, hist_out, pos_err, rot_err, success);
}

template <class G>
__global__ void __launch_bounds__(128)
k_col_resjac(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
             const CollisionParams<typename G::T> P, const double* __restrict__ tinv,
             const int32_t* __restrict__ lane_target, const double* __restrict__ q_in, int64_t lanes, int rows,
             double* __restrict__ res, double* __restrict__ jac) {
  using T = typename G::T;
  constexpr int NQ = G::NQ;
  extern __shared__ unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= lanes) return;
  const TargetInv<T> tg = load_target_inv<T>(tinv + (int64_t)lane_target[l] * 7);
  T q[NQ];
#pragma unroll
  for (int i = 0; i < NQ; ++i) q[i] = T(q_in[l * NQ + i]);
  const ColLane<G> L{reinterpret_cast<T*>(smem_raw) + threadIdx.x, 128};
  double* ro = res + l * rows;
  double* jo = jac + l * rows * NQ;
  for (int i = 0; i < rows * NQ; ++i) jo[i] = 0.0;
  T A[Tri<NQ>::size], g[NQ];
  col_eval<G, true>(C, W, P, tg, L, q, A, g, ro, jo);
  T rl[NQ], gl[NQ], rr[NQ];  // diagonal rows (beam.py:158-166)
  diag_rows(W, q, rl, gl, rr);
#pragma unroll
  for (int i = 0; i < NQ; ++i) {
    ro[6 + i] = double(rl[i]);
    ro[6 + NQ + i] = double(rr[i]);
    jo[(6 + i) * NQ + i] = double(gl[i]);
    jo[(6 + NQ + i) * NQ + i] = double(W.w_rest);
  }
}

// termination codes (SolveReport.termination + message, solver.py:381-426)
enum Termination : int32_t {
  kMaxIterations = 0,
  kGradientConverged = 1,
  kStepConverged = 2,         // max |step| < step_tolerance
  kNumericalFailure = 3,      // damping above 1e10 ("no acceptable step below damping 1e10")
  kRejectionsExhausted = 4,   // step_converged, "rejection budget exhausted without descent"
  kNonFiniteCost = 5,         // numerical_failure: CostEvaluationError isolated by solve_batch
  kFp32Resolution = 6,        // FP32 only: step_converged, no cost decrease resolvable in FP32
};

// FP32 stopping rule: a rejected trial whose quadratic-model
// decrease -g.d + lam d^T D d is below kFp32Tau * cost cannot be resolved by a
// float32 cost, so further damping increases only walk lambda up to 1e10 (the
// FP64 run would stop by its gradient / step tolerance there instead).
constexpr float kFp32Tau = 7.62939453125e-6f;  // 2^-17 = 64 float32 ulps of 1

// solver.solve (solver.py:364-429), one problem per thread, written as a
// UNIFORM TRIAL MACHINE: every pass of the loop is "solve the damped normal
// equations held in shared memory, evaluate the candidate WITH its Jacobian";
// the start evaluation is the trial with a zero step and an accepted
// candidate's normal equations are the next iterate's (the assemble at the
// new values, solver.py:419).  The rejection loop (:389-409) is a run of
// rejected trials, so all 32 lanes of a warp execute the same instruction
// stream whatever their accept / reject / iteration state, and a lane whose
// problem terminates takes the next problem from a global queue (counter)
// instead of idling until the warp's slowest problem finishes.
template <class G>
__global__ void __launch_bounds__(128)
k_col_solve(const ChainParams<typename G::T, G::K> C, const CostParams<typename G::T, G::NQ> W,
            const CollisionParams<typename G::T> P, const double* __restrict__ targets,
            const double* __restrict__ q0, int64_t B, const LmOptions O, double* __restrict__ q_out,
            double* __restrict__ cost_out, double* __restrict__ init_cost_out, double* __restrict__ hist_out,
            int32_t* __restrict__ iters_out, int32_t* __restrict__ term_out, unsigned long long* __restrict__ queue) {
  using T = typename G::T;
  constexpr int NQ = G::NQ, NT = Tri<NQ>::size;
  constexpr bool F32 = sizeof(T) == 4;
  extern __shared__ unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  T* Ag = reinterpret_cast<T*>(smem_raw) + threadIdx.x;  // [(NT + NQ) * 128]
  T* scratch = reinterpret_cast<T*>(smem_raw) + (NT + NQ) * 128 + threadIdx.x;
  const int64_t first_wave = (int64_t)gridDim.x * blockDim.x;
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int hstride = O.max_iterations + 1;
  const T zb[3] = {T(0), T(0), T(0)};
  T q[NQ], d[NQ];
  T cost = T(0), damping = T(0), pred = T(0);
  int iters = 0, rej = 0;
  bool start = true;
  TargetInv<T> tg{};
  auto begin = [&](int64_t bb) {
    tg = target_inverse_t<T>(targets + bb * 7);
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      q[i] = T(q0[bb * NQ + i]);
      d[i] = T(0);
    }
    damping = T(O.damping0);
    iters = rej = 0;
    start = true;
  };
  if (b < B) begin(b);
  while (b < B) {
    // ---- the one evaluation site: candidate q + d (the start: d = 0) ----
    T qc[NQ], A[NT], g[NQ];
#pragma unroll
    for (int i = 0; i < NQ; ++i) qc[i] = q[i] + d[i];
    const CollisionModel<G> model{C, W, P, tg, ColLane<G>{scratch, 128}};
    const T cn = model.template eval<true>(qc, zb, A, g);
    int term = -1;
    bool fresh = false;  // normal equations of a new iterate: iteration-start checks
    if (start) {
      start = false;
      cost = cn;
      init_cost_out[b] = double(cn);
      if (hist_out) hist_out[b * hstride] = double(cn);
      fresh = true;
      if (!finite_t(cn)) term = kNonFiniteCost;  // raw_residual raises on non-finite
    } else if (!finite_t(cn)) {
      term = kNonFiniteCost;  // CostEvaluationError -> solve_batch's numerical_failure
    } else if (cn < cost) {
      T smax = T(0);
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        q[i] = qc[i];
        smax = tmax(smax, fabs(d[i]));
      }
      cost = cn;
      damping = tmax(damping * T(O.down), T(BeamConsts::damping_min));
      rej = 0;
      ++iters;
      if (hist_out) hist_out[b * hstride + iters] = double(cost);
      fresh = true;
      if (smax < T(O.step_tol)) term = kStepConverged;
    } else if (F32 && pred <= T(kFp32Tau) * cost) {
      term = kFp32Resolution;
    } else {
      damping *= T(O.up);
      ++rej;
      if (damping > T(BeamConsts::damping_max)) term = kNumericalFailure;
      else if (rej >= O.max_rejections) term = kRejectionsExhausted;
    }
    if (fresh) {
#pragma unroll
      for (int i = 0; i < NT; ++i) Ag[i * 128] = A[i];
#pragma unroll
      for (int i = 0; i < NQ; ++i) Ag[(NT + i) * 128] = g[i];
      if (term < 0) {
        if (iters >= O.max_iterations) {
          term = kMaxIterations;
        } else {
          T gmax = T(0);
#pragma unroll
          for (int i = 0; i < NQ; ++i) gmax = tmax(gmax, fabs(g[i]));
          if (gmax < T(O.grad_tol)) term = kGradientConverged;
          else if (O.max_rejections <= 0) term = kRejectionsExhausted;  // no trial allowed (solver.py:389)
        }
      }
    }
    // ---- the next trial's step (a failed factorisation is a rejected trial) ----
    while (term < 0) {
#pragma unroll
      for (int i = 0; i < NT; ++i) A[i] = Ag[i * 128];
#pragma unroll
      for (int i = 0; i < NQ; ++i) g[i] = Ag[(NT + i) * 128];
      bool ok = damped_solve<T, NQ>(A, g, damping, d);
      T gd = T(0), dd = T(0);
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        ok = ok && finite_t(d[i]);
        gd += g[i] * d[i];
        dd += tmax(A[Tri<NQ>::at(i, i)], T(BeamConsts::diag_clamp)) * d[i] * d[i];
      }
      if (ok) {
        pred = damping * dd - gd;  // quadratic-model decrease of the trial
        break;
      }
      damping *= T(O.up);
      ++rej;
      if (damping > T(BeamConsts::damping_max)) term = kNumericalFailure;
      else if (rej >= O.max_rejections) term = kRejectionsExhausted;
    }
    if (term >= 0) {
      if (hist_out)
        for (int i = iters + 1; i < hstride; ++i) hist_out[b * hstride + i] = NAN;
#pragma unroll
      for (int i = 0; i < NQ; ++i) q_out[b * NQ + i] = double(q[i]);
      cost_out[b] = double(cost);
      iters_out[b] = iters;
      term_out[b] = term;
      b = first_wave + (int64_t)atomicAdd(queue, 1ull);
      if (b < B) begin(b);
    }
  }
}

// ---------------------------------------------------------------------------
// launchers
// ---------------------------------------------------------------------------
template <class G>
size_t col_scratch_bytes(const CollisionParams<typename G::T>& P) {
  return sizeof(typename G::T) * (size_t)(col_scratch_fixed<G>() + 3 * P.ns) * 128;
}

template <class G>
cudaError_t launch_col(const ChainParams<typename G::T, G::K>& C, const CostParams<typename G::T, G::NQ>& W,
                       const CollisionParams<typename G::T>& P, const ChainParams<double, G::K>& Cd,
                       const ColLaunch& L, cudaStream_t st) {
  using T = typename G::T;
  const int extra = col_scratch_fixed<G>() + 3 * P.ns;
  if (L.op == ColOp::kResJac) {
    if (L.lanes == 0) return cudaSuccess;
    const size_t smem = col_scratch_bytes<G>(P);
    cudaFuncSetAttribute(k_col_resjac<G>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(k_col_resjac<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_col_resjac<G><<<(unsigned)((L.lanes + 127) / 128), 128, smem, st>>>(C, W, P, L.tinv, L.lane_target, L.q_in,
                                                                           L.lanes, L.rows, L.res, L.jac);
    return cudaGetLastError();
  }
  if (L.op == ColOp::kSolve) {
    if (L.B == 0) return cudaSuccess;
    const size_t smem = sizeof(T) * (Tri<G::NQ>::size + G::NQ) * 128 + col_scratch_bytes<G>(P);
    cudaError_t e;
    cudaFuncSetAttribute(k_col_solve<G>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (smem > 48 * 1024 &&
        (e = cudaFuncSetAttribute(k_col_solve<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
            cudaSuccess)
      return e;
    // persistent grid: every resident CTA, lanes pull further problems from the queue
    int dev = 0, sms = 0, per_sm = 0;
    if ((e = cudaGetDevice(&dev)) != cudaSuccess ||
        (e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess ||
        (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_col_solve<G>, 128, smem)) != cudaSuccess)
      return e;
    const int64_t need = (L.B + 127) / 128;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sms * std::max(per_sm, 1)));
    unsigned long long* queue = nullptr;
    if ((e = cudaMallocAsync(reinterpret_cast<void**>(&queue), sizeof(unsigned long long), st)) != cudaSuccess)
      return e;
    cudaMemsetAsync(queue, 0, sizeof(unsigned long long), st);
    k_col_solve<G><<<(unsigned)grid, 128, smem, st>>>(C, W, P, L.targets, L.q_in, L.B, L.opts, L.q_out, L.cost_out,
                                                      L.init_cost, L.hist_out, L.iters, L.term, queue);
    e = cudaGetLastError();
    cudaFreeAsync(queue, st);
    return e;
  }
  // IK-Beam over the collision stack
  const BeamLaunch& Bm = L.beam;
  const int rec = Rec<G>::size(Bm.steps1);
  T* surv = reinterpret_cast<T*>(Bm.workspace);
  if (Bm.P > 128) return cudaErrorInvalidValue;  // collision beams keep 64-lane (<= 128) targets per block
  const int per_block = 128 / Bm.P;
  const int64_t blocks1 = (Bm.B + per_block - 1) / per_block;
  const size_t smem1 = beam_stage1_smem<G>(128, Bm.steps1, extra);
  cudaFuncSetAttribute(k_col_beam_stage1<G>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (smem1 > 48 * 1024)
    cudaFuncSetAttribute(k_col_beam_stage1<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1);
  if (Bm.stages & 1) {
    k_col_beam_stage1<G><<<(unsigned)blocks1, 128, smem1, st>>>(C, W, P, Bm.targets, Bm.B, Bm.seeds, Bm.S, Bm.P,
                                                                 Bm.steps1, Bm.keep, surv, rec);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (!(Bm.stages & 2)) return cudaSuccess;
  const int64_t blocks2 = (Bm.B * Bm.G + 127) / 128;
  const size_t smem2 = beam_stage2_smem<G>(Bm.steps2, extra);
  cudaFuncSetAttribute(k_col_beam_stage2<G>, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  if (smem2 > 48 * 1024)
    cudaFuncSetAttribute(k_col_beam_stage2<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  k_col_beam_stage2<G><<<(unsigned)blocks2, 128, smem2, st>>>(C, W, P, Cd, Bm.targets, Bm.B, surv, rec, Bm.steps1,
                                                               Bm.steps2, Bm.keep, Bm.G, Bm.pos_tol, Bm.rot_tol,
                                                               Bm.q_out, Bm.cost_out, Bm.hist_out, Bm.pos_err,
                                                               Bm.rot_err, Bm.success);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return launch_beam_errors<G>(Cd, Bm.targets, Bm.B, Bm.q_out, Bm.pos_tol, Bm.rot_tol, Bm.pos_err, Bm.rot_err,
                               Bm.success, st);
}

#define KOP_COL_INSTANTIATE(T, NQ, K, ID)                                                                     \
  template cudaError_t launch_col<Cfg<T, NQ, K, ID, false>>(const ChainParams<T, K>&, const CostParams<T, NQ>&, \
                                                            const CollisionParams<T>&,                          \
                                                            const ChainParams<double, K>&, const ColLaunch&,    \
                                                            cudaStream_t);

KOP_FOR_EACH_COLLISION_SHAPE(KOP_COL_INSTANTIATE)

}  // namespace kop
