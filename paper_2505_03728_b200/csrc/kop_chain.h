// Compiled kinematic chain + cost parameters, passed BY VALUE as kernel
// parameters so every model constant is a constant-bank operand of the FMA
// that uses it (no register or shared-memory cost, broadcast to all lanes).
//
// The host compiles the reference's joint tables (robot.py:74-112) for one
// end-effector link into the moving joints of its root->link path:
//  * fixed joints are folded into the next moving joint's origin (or into the
//    end-effector offset), robot.py:433-436;
//  * each moving joint's frame is post-rotated so its axis is the local +z
//    (the next origin is pre-rotated back), so a revolute motion is the
//    8-FMA product q * (cos, 0, 0, sin) and the world axis is one column of
//    R(q) -- the same transform as robot.py:437-447, fewer flops.
// Mathematically identical to fk_arrays; differences are rounding only.
//
// The device evaluates the chain BACKWARD (end effector -> root): with
// S_k = child_k -> EE, the body-frame Jacobian column of joint k is read off
// S_k directly (axis = +z there), so no per-joint world anchors/axes are kept
// live and the pass ends with the world EE pose S_0 for the residual.
#pragma once

#include <stdint.h>

namespace kop {

constexpr int kMaxTreeJoints = 64;  // full-tree FK kernel limit
constexpr int kMaxLinks = kMaxTreeJoints + 1;

template <typename T, int K>
struct ChainParams {
  T tq[K][4];    // joint-frame rotation relative to the previous moving child frame
  T tp[K][3];    // joint anchor translation relative to the previous moving child frame
  T tr[K][3][3]; // R(tq): the backward pass rotates positions with 9 constant-operand FMAs
  T mult[K];     // mimic multiplier (robot.py:93-97)
  T offset[K];   // mimic offset
  int32_t qcol[K];
  int32_t prismatic[K];
  T eq[4];       // end-effector link offset after the last moving joint
  T ep[3];
  int32_t k;     // moving joints actually on the chain (<= K)
};

template <typename T, int NQ>
struct CostParams {
  T lower[NQ], upper[NQ], rest[NQ];
  T w_pos, w_ori, w_lim, w_rest;  // beam.py:95-100 row weights
  T w_base;                       // base regularisation rows (beam.py:98-99)
};

// Full-tree tables for the generic FK kernel (robot.py:404-448 semantics,
// reference operation order).
struct TreeParams {
  int32_t nl, nj, n;
  int32_t parent[kMaxTreeJoints], child[kMaxTreeJoints], kind[kMaxTreeJoints], qcol[kMaxTreeJoints];
  double mult[kMaxTreeJoints], offset[kMaxTreeJoints];
  double oq[kMaxTreeJoints][4], op[kMaxTreeJoints][3], axis[kMaxTreeJoints][3];
};

// LM / beam constants, beam.py:37-42 and tasks.py:47-52.
struct BeamConsts {
  static constexpr double damping_init = 1e-4;
  static constexpr double damping_up = 10.0;
  static constexpr double damping_down = 1.0 / 3.0;
  static constexpr double damping_min = 1e-12;
  static constexpr double damping_max = 1e10;
  static constexpr double diag_clamp = 1e-8;
};

}  // namespace kop
