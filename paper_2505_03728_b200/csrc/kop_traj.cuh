// Trajectory optimisation (config 5) -- parameters and launcher declaration.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kop_chain.h"
#include "kop_collision.cuh"
#include "kop_kernels.cuh"

namespace kop {

constexpr int kTrajMaxSteps = 64;

// plan_trajectory's cost set (tasks.py:347-403) with the weights already
// folded in; the anchors q_start / q_goal are per problem (TrajLaunch).
template <typename T>
struct TrajCosts {
  int32_t T_steps;  // timesteps
  int32_t n;        // actuated joints (<= NQ, the rest are padding)
  T lower[8], upper[8], rest[8];
  T vbudget[8];     // velocity_limit * dt, +inf for unlimited joints
  T w_lim, w_rest, anchor, w_smooth, w_vel, w_acc, w_jerk;
  T acc_c[5], jerk_c[5];  // five-point stencils / dt^2, dt^3 (costs.py:295-296)
  T w_world, eta_world;   // swept-capsule rows (costs.py:554-619)
};

struct TrajLaunch {
  const double* q_init;     // [B, T, n], or null: straight line between the anchors
  const double* anchors;    // [B, 2, n]  q_start, q_goal
  const double* obstacles;  // [B, n_obs, 8]  kind, a[3], b[3], radius|offset (robot base frame)
  int n_obs;
  int64_t B;
  LmOptions opts;
  double *q_out, *cost_out, *init_cost, *hist_out;
  int32_t *iters, *term;
  double *grad_out, *hess_out;  // kop_traj_normal_equations
};

struct TrajReportLaunch {
  int steps, n;
  const double* qs;         // [B, T, n]
  const double* obstacles;  // [B, n_obs, 8]
  int n_obs;
  const double* targets;    // [B, 2, 7] start / goal poses, or null
  int64_t B;
  double *static_out, *swept_out, *min_static, *min_swept, *pos_err, *rot_err;
};

template <class G>
cudaError_t launch_traj_report(const ChainParams<double, G::K>& C, const CollisionParams<double>& P,
                               const TrajReportLaunch& L, cudaStream_t st);

template <class G>
cudaError_t launch_traj_normal(const ChainParams<typename G::T, G::K>& C, const CollisionParams<typename G::T>& P,
                               const TrajCosts<typename G::T>& W, const TrajLaunch& L, cudaStream_t st);

template <class G>
cudaError_t launch_traj(const ChainParams<typename G::T, G::K>& C, const CollisionParams<typename G::T>& P,
                        const TrajCosts<typename G::T>& W, const TrajLaunch& L, cudaStream_t st);

}  // namespace kop
