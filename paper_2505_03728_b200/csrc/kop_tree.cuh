// Kernel parameters of the tree (multi-end-effector) LM solve, kop_tree.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "kop_kernels.cuh"

namespace kop {

constexpr int kTreeMaxJoints = 64;
constexpr int kTreeMaxPoses = 8;
constexpr int kTreeMaxDofs = 32;  // one warp lane per actuated joint
constexpr int kTreeMaxPerCol = 4;  // moving joints driven by one column (leader + mimics)

template <typename T>
struct TreeLmParams {
  int32_t nj, n, ne;
  int32_t parent_joint[kTreeMaxJoints];  // joint owning the parent link (-1: root link)
  int32_t kind[kTreeMaxJoints], qcol[kTreeMaxJoints];
  T oq[kTreeMaxJoints][4], op[kTreeMaxJoints][3], axis[kTreeMaxJoints][3];
  T mult[kTreeMaxJoints], offset[kTreeMaxJoints];
  int32_t ee_joint[kTreeMaxPoses];          // joint owning each end-effector link (-1: root)
  T ee_oq[kTreeMaxPoses][4], ee_op[kTreeMaxPoses][3];  // fixed offset of the link from that joint's frame
  unsigned long long anc_ee[kTreeMaxPoses]; // ancestor-joint mask of each end effector
  T w_pos[kTreeMaxPoses], w_ori[kTreeMaxPoses];
  T lower[kTreeMaxDofs], upper[kTreeMaxDofs], rest[kTreeMaxDofs];
  T w_lim, w_rest;
  // joints grouped by depth (parents in earlier levels): level d = lev_joint[lev_start[d] .. lev_start[d+1])
  int32_t nlev;
  int32_t lev_start[kTreeMaxJoints + 1];
  int8_t lev_joint[kTreeMaxJoints];
  // moving joints of each actuated column
  int8_t col_nj[kTreeMaxDofs];
  int8_t col_joint[kTreeMaxDofs][kTreeMaxPerCol];
  // optional base variable of the pose costs (costs.py:98-166, base_var): 0 none, 1 SE(2), 2 SE(3);
  // its tangent is columns n .. n + db - 1
  int32_t base_kind;
};

__host__ __device__ inline int base_dim(int base_kind) { return base_kind == 1 ? 3 : (base_kind == 2 ? 6 : 0); }
__host__ __device__ inline int base_state(int base_kind) { return base_kind == 1 ? 3 : (base_kind == 2 ? 7 : 0); }

struct TreeLaunch {
  const double* targets;  // [B * ne * 7]
  const double* q0;       // [B * n]
  const double* base0;    // [B * 3] (angle, x, y) for SE(2) | [B * 7] (wxyz, xyz) for SE(3) | null
  double* base_out;       // same layout
  int64_t B;
  LmOptions opts;
  double *q_out, *cost_out, *init_cost, *hist_out;
  int32_t *iters, *term;
};

template <typename T>
cudaError_t launch_tree_solve(const TreeLmParams<T>& P, const TreeLaunch& L, cudaStream_t st);

// multi-end-effector IK-Beam (config 3 as SURVEY.md section 8 H6 states it)
struct TreeBeamLaunch {
  const double* targets;  // [B * ne * 7]
  int64_t B;
  const double* seeds;    // [S * n]
  int S, steps1, steps2, keep;
  double pos_tol, rot_tol;
  void* workspace;        // lane records [B * S * rec] | survivor seeds [B * keep] int32
  double *q_out, *cost_out, *hist_out, *pos_err, *rot_err;
  uint8_t* success;
};

__host__ __device__ inline int tree_beam_rec(int n, int steps1) { return n + 2 + steps1 + 1; }  // q | lam | cost | hist

template <typename T>
cudaError_t launch_tree_beam(const TreeLmParams<T>& P, const TreeLmParams<double>& Pd, const TreeBeamLaunch& L,
                             cudaStream_t st);

}  // namespace kop
