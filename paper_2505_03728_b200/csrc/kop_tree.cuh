// Kernel parameters of the tree (multi-end-effector) LM solve, kop_tree.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kop_kernels.cuh"

namespace kop {

constexpr int kTreeMaxJoints = 64;
constexpr int kTreeMaxPoses = 8;
constexpr int kTreeMaxDofs = 32;  // one warp lane per actuated joint

template <typename T>
struct TreeLmParams {
  int32_t nj, n, ne;
  int32_t parent_joint[kTreeMaxJoints];  // joint owning the parent link (-1: root link)
  int32_t kind[kTreeMaxJoints], qcol[kTreeMaxJoints];
  T oq[kTreeMaxJoints][4], op[kTreeMaxJoints][3], axis[kTreeMaxJoints][3];
  T mult[kTreeMaxJoints], offset[kTreeMaxJoints];
  int32_t ee_joint[kTreeMaxPoses];          // joint owning each end-effector link (-1: root)
  unsigned long long anc_ee[kTreeMaxPoses]; // ancestor-joint mask of each end effector
  T w_pos[kTreeMaxPoses], w_ori[kTreeMaxPoses];
  T lower[kTreeMaxDofs], upper[kTreeMaxDofs], rest[kTreeMaxDofs];
  T w_lim, w_rest;
};

struct TreeLaunch {
  const double* targets;  // [B * ne * 7]
  const double* q0;       // [B * n]
  int64_t B;
  LmOptions opts;
  double *q_out, *cost_out, *init_cost, *hist_out;
  int32_t *iters, *term;
};

template <typename T>
cudaError_t launch_tree_solve(const TreeLmParams<T>& P, const TreeLaunch& L, cudaStream_t st);

}  // namespace kop
