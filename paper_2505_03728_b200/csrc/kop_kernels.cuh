// Internal launch interface between the C ABI (kop_capi.cu) and the kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kop_chain.h"
#include "kop_collision.cuh"
#include "kop_lane.cuh"

namespace kop {

// Compiled (T, NQ actuated, K chain joints, identity column map, SE(2) base)
// shapes.  ID shapes serve serial chains whose moving joints are exactly the
// actuated joints (Panda, planar 2R, UR-class); the generic shape serves
// trees, mimic joints and sub-chains with K <= NQ <= 8 (smaller robots are
// padded to NQ = 8 exactly, see kop_capi.cu:make_costs).
#define KOP_FOR_EACH_SHAPE(X)   \
  X(float, 2, 2, true, false)   \
  X(double, 2, 2, true, false)  \
  X(float, 6, 6, true, false)   \
  X(double, 6, 6, true, false)  \
  X(float, 7, 7, true, false)   \
  X(double, 7, 7, true, false)  \
  X(float, 8, 8, false, false)  \
  X(double, 8, 8, false, false) \
  X(float, 7, 7, true, true)    \
  X(double, 7, 7, true, true)   \
  X(float, 8, 8, false, true)   \
  X(double, 8, 8, false, true)

struct BeamLaunch {
  const double* targets;
  int64_t B;
  const double* seeds;
  int S, P, G;  // seeds, lanes per target (pow2 >= S), survivor group (pow2 >= keep)
  int steps1, steps2, keep;
  double pos_tol, rot_tol;
  void* workspace;
  double *q_out, *base_out, *cost_out, *hist_out, *pos_err, *rot_err;
  uint8_t* success;
  int stages;  // bit 0: stage 1 (seeds + prune), bit 1: stage 2 (survivors + winner)
};

enum class LaneOp { kResJac, kStart, kRun };

struct LaneLaunch {
  LaneOp op;
  const double* tinv;
  const int32_t* lane_target;
  const double* q_in;
  const double* base_in;  // [lanes*3] (x, y, angle) when the base is optimised
  int64_t lanes;
  int steps;
  double *q_io, *base_io, *lam, *cost, *hist, *res, *jac;
};

// collision-stack shapes (fixed base): the Panda identity chain and the
// generic padded 8-joint shape
#define KOP_FOR_EACH_COLLISION_SHAPE(X) \
  X(float, 7, 7, true)                 \
  X(double, 7, 7, true)                \
  X(float, 8, 8, false)                \
  X(double, 8, 8, false)

// solver.SolveOptions (solver.py:179-198) as the device sees them
struct LmOptions {
  int max_iterations, max_rejections;
  double damping0, up, down, grad_tol, step_tol;
};

enum class ColOp { kResJac, kBeam, kSolve };

struct ColLaunch {
  ColOp op;
  // kResJac
  const double* tinv;
  const int32_t* lane_target;
  const double* q_in;  // also q0 for kSolve
  int64_t lanes;
  int rows;
  double *res, *jac;
  // kSolve
  const double* targets;
  int64_t B;
  double *q_out, *cost_out, *init_cost, *hist_out;
  int32_t *iters, *term;
  LmOptions opts;
  // kBeam
  BeamLaunch beam;
};

template <class G>
cudaError_t launch_col(const ChainParams<typename G::T, G::K>& C, const CostParams<typename G::T, G::NQ>& W,
                       const CollisionParams<typename G::T>& P, const ChainParams<double, G::K>& Cd,
                       const ColLaunch& L, cudaStream_t st);

template <class G>
cudaError_t launch_beam(const ChainParams<typename G::T, G::K>& C, const CostParams<typename G::T, G::NQ>& W,
                        const ChainParams<double, G::K>& Cd, const BeamLaunch& L, cudaStream_t st);

template <class G>
cudaError_t launch_lane(const ChainParams<typename G::T, G::K>& C, const CostParams<typename G::T, G::NQ>& W,
                        const LaneLaunch& L, cudaStream_t st);

// kop_aux.cu
cudaError_t launch_fk_tree(const TreeParams& P, int precision, const double* q, int64_t B,
                           double* lq, double* lp, double* jp, double* ja, cudaStream_t st);
cudaError_t launch_link_pose(const TreeParams& path, const double* q, int64_t B, double* poses,
                             cudaStream_t st);
cudaError_t launch_philox(uint64_t key0, uint64_t key1_base, int64_t count, int n, const double* lo,
                          const double* range, const uint8_t* negate, double* out, cudaStream_t st);
cudaError_t launch_jacobian_tree(const TreeParams& P, int precision, const double* q, int64_t B, int link,
                                 unsigned long long anc, const double* points, int rotational, double* jac,
                                 cudaStream_t st);
cudaError_t launch_fma_peak(int blocks, int threads, int iters, float* sink, cudaStream_t st);
cudaError_t launch_dfma_peak(int blocks, int threads, int iters, double* sink, cudaStream_t st);
cudaError_t launch_check_probe(uint32_t* out, int words, cudaStream_t st);

}  // namespace kop
