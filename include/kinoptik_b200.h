/*
 * kinoptik_b200 -- C ABI of the B200 (sm_100a) batched LM-IK engine.
 *
 * Plain pointers, sizes and an opaque model handle; no torch or CUDA C++
 * types cross this boundary (streams are passed as `void*` = cudaStream_t).
 * Every array argument marked "device" must point to device memory on the
 * current CUDA device; "host" arrays are read synchronously before return.
 *
 * Each entry point names the reference interface it replaces.  The reference
 * (`kinoptik`, /root/reference/pkg/src/kinoptik) is pure NumPy and has no FFI
 * of its own; INTEGRATION.md shows the ctypes stub a kinoptik maintainer
 * would add at each of these seams.
 *
 * Conventions (liegroups.py:1-13): quaternions (w,x,y,z), twists
 * translation-first, right-multiplicative retraction; a pose is 7 doubles
 * (w,x,y,z,px,py,pz).  Configurations are the actuated joints in the
 * topological (BFS) order of robot.py:325-340.
 *
 * Status codes: 0 ok; KOP_EINVAL invalid argument (the reference raises
 * ValueError); KOP_EUNSUPPORTED kinematic shape not compiled in (the
 * reference would run it -- the caller must raise UnsupportedFeatureError,
 * never fall back to the CPU); KOP_ECUDA a CUDA launch/runtime error.
 * kop_last_error() returns a thread-local message for the last failure.
 *
 * Thread safety: a KopModel is immutable after creation and holds no device
 * state, so one model may be used concurrently from one host thread per GPU
 * (robot.py:8-12 purity contract).  All launches are asynchronous on the
 * given stream; results are bitwise reproducible run to run and independent
 * of batch size and GPU count (no atomics, fixed reduction orders).
 */
#ifndef KINOPTIK_B200_H
#define KINOPTIK_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KOP_OK 0
#define KOP_EINVAL (-1)
#define KOP_EUNSUPPORTED (-2)
#define KOP_ECUDA (-3)

#define KOP_FP32 0 /* measured mode: float arithmetic on the device       */
#define KOP_FP64 1 /* parity-debug mode: double arithmetic, same algorithm */

#define KOP_JOINT_FIXED 0     /* robot.py:27-36 kind codes */
#define KOP_JOINT_REVOLUTE 1  /* revolute and continuous  */
#define KOP_JOINT_PRISMATIC 2

typedef struct KopModel KopModel;

/* Kinematic tree in the reference's SoA layout, robot.py:74-112 (host). */
typedef struct {
  int32_t num_links;            /* L; link 0 is the root (robot.py:418-419)   */
  int32_t num_joints;           /* J, topological order                        */
  int32_t num_actuated;         /* n                                           */
  const int32_t* parent_link;   /* [J]                                         */
  const int32_t* child_link;    /* [J]                                         */
  const int32_t* kind;          /* [J] KOP_JOINT_*                             */
  const int32_t* qcol;          /* [J] actuated column, -1 for fixed           */
  const double* mult;           /* [J] mimic multiplier (1 otherwise)          */
  const double* offset;         /* [J] mimic offset (0 otherwise)              */
  const double* origin_wxyz;    /* [J*4] joint origin rotation                 */
  const double* origin_xyz;     /* [J*3] joint origin translation              */
  const double* axis;           /* [J*3] unit joint axis in the joint frame    */
  const double* lower;          /* [n] (-inf where absent, robot.py:114-126)   */
  const double* upper;          /* [n] (+inf where absent)                     */
  const double* rest;           /* [n] rest pose (robot.py:128-141)            */
  /* collision spheres (URDF <collision><sphere> or sidecar, robot.py:209-218,
   * 355-361) in model link order, and self-collision link pairs
   * (RobotModel.self_collision_pairs, robot.py:174-190); counts may be 0 */
  int32_t num_spheres;          /* S <= 32                                     */
  const int32_t* sphere_link;   /* [S] link index                              */
  const double* sphere_center;  /* [S*3] centre in the link frame              */
  const double* sphere_radius;  /* [S]                                         */
  int32_t num_self_pairs;       /* P <= 64                                     */
  const int32_t* self_pair_links; /* [P*2] link index pairs                    */
} KopModelDesc;

/* IK-Beam request scalars: IkRequest (tasks.py:40-60) + CostWeights
 * (costs.py:52-62).  Defaults: 50, 10, 100, 0.01; 64/16/6/4; 5 mm, 0.05. */
typedef struct {
  double w_position, w_orientation, w_limit, w_rest;
  int32_t seeds, total_steps, prune_after, keep;
  double success_pos_tol, success_rot_tol;
  int32_t precision;     /* KOP_FP32 | KOP_FP64 */
  int32_t optimize_base; /* 1: SE(2) mobile base as 3 extra variables (beam.py:98-112) */
  double w_base;         /* base regularisation weight (IkRequest.base_reg_weight) */
} KopIkParams;

/* --- model ----------------------------------------------------------------
 * replaces: robot.RobotModel.__init__ tables (robot.py:55-144); the URDF /
 * sidecar parse itself stays on the host (robot.py:221-387). */
int kop_model_create(const KopModelDesc* desc, KopModel** out);
void kop_model_destroy(KopModel* model);
/* Moving joints on the root->link chain (fixed joints folded); -1 on error. */
int kop_model_chain_length(const KopModel* model, int32_t link);
/* The compiled root->link chain the IK kernels evaluate (kop_chain.h): per
 * moving joint k < K (K = return value, <= 8) the joint frame relative to the
 * previous moving child frame with its axis rotated onto +z: tq [K*4],
 * tp [K*3]; qcol/mult/offset/prismatic [K]; ee [7] the link offset after the
 * last moving joint.  Host arrays, any may be NULL.  For tests and tooling. */
int kop_model_chain_export(const KopModel* model, int32_t link, double* tq, double* tp, int32_t* qcol,
                           double* mult, double* offset, int32_t* prismatic, double* ee);
const char* kop_last_error(void);
const char* kop_build_info(void);

/* --- forward kinematics ---------------------------------------------------
 * replaces: robot.fk_arrays(model, q[B,n]) (robot.py:404-448).
 * q: device [B*n] double.  Outputs (device, double, any may be NULL):
 * link_wxyz [B*L*4] raw (non-canonical) quaternions, link_xyz [B*L*3],
 * joint_xyz [B*J*3] joint anchors, joint_axis [B*J*3] world axes. */
int kop_fk(const KopModel* model, int32_t precision, const double* q, int64_t batch,
           double* link_wxyz, double* link_xyz, double* joint_xyz, double* joint_axis,
           void* stream);

/* replaces: robot.link_jacobian / point_jacobian (robot.py:461-506): the
 * geometric Jacobian of `link` at q [B*n] (device).  points: device [B*3]
 * world points rigidly attached to the link, or NULL for the link origin;
 * rotational != 0 adds the angular rows.  jac: device [B*rows*n] double,
 * rows = 6 (rotational) or 3, mimic joints folded into their source column. */
int kop_jacobian(const KopModel* model, int32_t precision, const double* q, int64_t batch, int32_t link,
                 const double* points, int32_t rotational, double* jac, void* stream);

/* --- lane engine ----------------------------------------------------------
 * replaces: beam.IkLaneProblem(model, link, target, weights..., use_base,
 * base_reg_weight) with .residuals_and_jacobian (beam.py:133-180),
 * .start_state (beam.py:182-196) and .run(state, steps) (beam.py:198-240),
 * generalised to one target per lane.  target_inv: device [T*7] double, the
 * INVERSE target pose per target (beam.py:89-91); lane_target: device [B]
 * int32 target index per lane.  State arrays (device, double): q [B*n]
 * in/out, base_state [B*3] (x, y, angle) in/out or NULL for a fixed base
 * (NULL = use_base False), damping [B] in/out, cost [B] in/out; history:
 * device [B*steps] double (may be NULL).  weights: host [5] (position,
 * orientation, limit, rest, base).  Residual rows: 6 pose, n limit, n rest,
 * (3 base); Jacobian columns: n joints (+3 base tangent vx, vy, w). */
int kop_lane_residuals_jacobian(const KopModel* model, int32_t link, int32_t precision,
                                const double* weights, const double* target_inv,
                                const int32_t* lane_target, const double* q, const double* base_state,
                                int64_t lanes, double* residual, double* jacobian, void* stream);
int kop_lane_start(const KopModel* model, int32_t link, int32_t precision, const double* weights,
                   const double* target_inv, const int32_t* lane_target, const double* q,
                   const double* base_state, int64_t lanes, double* damping, double* cost, void* stream);
int kop_lane_run(const KopModel* model, int32_t link, int32_t precision, const double* weights,
                 const double* target_inv, const int32_t* lane_target, int64_t lanes,
                 int32_t steps, double* q, double* base_state, double* damping, double* cost,
                 double* history, void* stream);

/* --- IK-Beam ----------------------------------------------------------------
 * replaces: tasks.solve_ik_beam / solve_ik_mobile(IkRequest) -> IkResult
 * (tasks.py:119-180),
 * batched over B independent targets (the reference loops targets one by one,
 * benchmark.py:136-151).  targets: device [B*7] double (w,x,y,z,px,py,pz);
 * seeds: device [S*n] double, shared by every target (tasks.py:131).
 * Outputs (device): q [B*n] double, base [B*3] (x, y, angle; NULL ok, only
 * written with optimize_base), cost [B] double, history [B*(total_steps+1)]
 * double (NULL ok), pos_err [B], rot_err [B] double (tasks.py:109-116,
 * evaluated in double, base included), success [B] uint8.
 * workspace: device scratch of kop_ik_beam_workspace_bytes() bytes. */
int64_t kop_ik_beam_workspace_bytes(const KopModel* model, int32_t link, const KopIkParams* params,
                                    int64_t batch);
int kop_ik_beam(const KopModel* model, int32_t link, const KopIkParams* params,
                const double* targets, int64_t batch, const double* seeds, void* workspace,
                int64_t workspace_bytes, double* q_out, double* base_out, double* cost_out,
                double* history_out, double* pos_err, double* rot_err, uint8_t* success, void* stream);

/* The two launches of kop_ik_beam issued separately (stages: 1 = seeds +
 * prune into the workspace, 2 = survivors + winner + errors, 3 = both), so a
 * caller can bracket each kernel with CUDA events.  Same arguments. */
int kop_ik_beam_stage(const KopModel* model, int32_t link, const KopIkParams* params, int32_t stages,
                      const double* targets, int64_t batch, const double* seeds, void* workspace,
                      int64_t workspace_bytes, double* q_out, double* base_out, double* cost_out,
                      double* history_out, double* pos_err, double* rot_err, uint8_t* success,
                      void* stream);

/* replaces: tasks.solve_ik_beam over B targets with HOST arrays end to end
 * (the binding a NumPy caller uses, INTEGRATION.md seam 3b): targets host
 * [B*7], seeds host [S*n]; outputs host, shapes as kop_ik_beam (base_out,
 * history_out NULL ok).  The batch streams through `n_streams` (1..8, 0 = 8)
 * internal CUDA streams in chunks of `chunk` targets (0 = 16384), overlapping
 * host->device copies, kernels and device->host copies; pinned host memory
 * gives full overlap.  Enqueued behind `stream` and joined back into it:
 * host buffers must stay valid until `stream` completes.  Internal device
 * buffers are cached per host thread and device (grow-only). */
int kop_ik_beam_host(const KopModel* model, int32_t link, const KopIkParams* params, const double* targets,
                     int64_t batch, const double* seeds, double* q_out, double* base_out, double* cost_out,
                     double* history_out, double* pos_err, double* rot_err, uint8_t* success, int64_t chunk,
                     int32_t n_streams, void* stream);

/* --- collision IK (config 4) and the generic LM solve -------------------
 * Cost stack (the viewer's, server.py:60-97): pose (w_position,
 * w_orientation) | limit (w_limit) | rest (w_rest) | world collision, one
 * row per (sphere link, obstacle) (costs.py:499-551; w_world, eta_world) |
 * self collision, one row per model self pair (costs.py:435-496; w_self,
 * eta_self); soft minimum with `sharpness` (1/m) unless hard_min.
 * Spheres must lie on links of the root->link chain. */
#define KOP_OBSTACLE_SPHERE 0    /* a = centre, radius                  */
#define KOP_OBSTACLE_CAPSULE 1   /* a, b = endpoints, radius            */
#define KOP_OBSTACLE_HALFSPACE 2 /* a = normal, radius = offset         */

typedef struct {
  int32_t kind;
  double a[3], b[3];
  double radius;
} KopObstacle;

typedef struct {
  double w_position, w_orientation, w_limit, w_rest;
  double w_world, eta_world, w_self, eta_self, sharpness;
  int32_t hard_min;
  int32_t num_obstacles;        /* <= 16 */
  const KopObstacle* obstacles; /* host */
} KopCollisionCosts;

/* solver.SolveOptions (solver.py:179-198) */
typedef struct {
  int32_t max_iterations;
  double initial_damping, damping_increase, damping_decrease;
  double gradient_tolerance, step_tolerance;
  int32_t max_rejections;
  int32_t precision;
} KopLmOptions;

/* Residual rows of the stack for `link` (6 + 2n + links*obstacles + pairs), or < 0. */
int kop_collision_rows(const KopModel* model, int32_t link, const KopCollisionCosts* costs);
/* replaces: the costs' raw_residual * weight and jacobian (solver.py:289-324)
 * for one target per lane: residual [lanes*R], jacobian [lanes*R*n] (device). */
int kop_collision_residuals_jacobian(const KopModel* model, int32_t link, int32_t precision,
                                     const KopCollisionCosts* costs, const double* target_inv,
                                     const int32_t* lane_target, const double* q, int64_t lanes,
                                     double* residual, double* jacobian, void* stream);
/* IK-Beam (tasks.py:119-161) over the collision stack; same outputs as kop_ik_beam. */
int64_t kop_ik_beam_collision_workspace_bytes(const KopModel* model, int32_t link, const KopIkParams* params,
                                              const KopCollisionCosts* costs, int64_t batch);
int kop_ik_beam_collision(const KopModel* model, int32_t link, const KopIkParams* params,
                          const KopCollisionCosts* costs, const double* targets, int64_t batch,
                          const double* seeds, void* workspace, int64_t workspace_bytes, double* q_out,
                          double* cost_out, double* history_out, double* pos_err, double* rot_err,
                          uint8_t* success, void* stream);
/* replaces: solver.solve / solve_batch (solver.py:364-460) for problems of
 * this cost stack: one problem per target, q0 [B*n] start configurations.
 * Outputs (device): q [B*n], cost [B], initial cost [B], history
 * [B*(max_iterations+1)] (NaN-padded, NULL ok), iterations [B] int32,
 * termination [B] int32: 0 max_iterations, 1 gradient_converged,
 * 2 step_converged (step tolerance), 3 numerical_failure (damping > 1e10),
 * 4 step_converged (rejection budget exhausted), 5 numerical_failure
 * (non-finite residual, the CostEvaluationError solve_batch isolates). */
int kop_lm_solve(const KopModel* model, int32_t link, const KopCollisionCosts* costs, const KopLmOptions* options,
                 const double* targets, const double* q0, int64_t batch, double* q_out, double* cost_out,
                 double* init_cost_out, double* history_out, int32_t* iterations_out,
                 int32_t* termination_out, void* stream);

/* --- multi-end-effector IK on a tree (config 3) ----------------------------
 * replaces: solver.solve over [pose_cost(link_e) for each e] + limit_cost +
 * rest_cost (costs.py:98-271, solver.py:364-429) on robots with up to 32
 * actuated / 64 total joints (humanoids): one warp per problem.
 * targets: device [B*E*7] (pose of end effector e of problem b); q0 [B*n].
 * Outputs and termination codes as kop_lm_solve. */
typedef struct {
  int32_t num_poses;           /* E <= 8 */
  const int32_t* links;        /* host [E] end-effector link indices */
  const double* w_position;    /* host [E] */
  const double* w_orientation; /* host [E] */
  double w_limit, w_rest;
  const double* rest;          /* host [n] rest configuration, NULL = the model's */
} KopPoseCosts;

int kop_multi_pose_solve(const KopModel* model, const KopPoseCosts* costs, const KopLmOptions* options,
                         const double* targets, const double* q0, int64_t batch, double* q_out,
                         double* cost_out, double* init_cost_out, double* history_out,
                         int32_t* iterations_out, int32_t* termination_out, void* stream);
/* the same tree LM with a BASE VARIABLE shared by the pose costs (costs.py:98-166
 * base_var; solver.py:36-108 typed variables): the tangent is [q | base],
 * base_kind KOP_BASE_SE2 (state (angle, x, y), tangent (vx, vy, w)) or
 * KOP_BASE_SE3 (state (wxyz, xyz), tangent (v, w)), retracted by local_update
 * (liegroups.py:505-519).  base0 / base_out: device [batch * 3 | 7]. */
int kop_multi_pose_solve_base(const KopModel* model, const KopPoseCosts* costs, const KopLmOptions* options,
                              int32_t base_kind, const double* targets, const double* q0, const double* base0,
                              int64_t batch, double* q_out, double* base_out, double* cost_out, double* init_cost_out,
                              double* history_out, int32_t* iterations_out, int32_t* termination_out, void* stream);

/* --- trajectory optimisation (config 5) -----------------------------------
 * replaces: the solve(...) call of plan_trajectory (tasks.py:347-403) over
 * its cost set -- anchors at q_0 / q_{T-1} (w_anchor), per-pair smoothness
 * and velocity limit, five-point acceleration / jerk stencils over
 * t = 2..T-3, per-timestep limit, rest (w_rest), self (w_self, eta_self)
 * and world (w_world, eta_world) collision, and swept-capsule world rows for
 * every consecutive pair -- solved by solver.solve (solver.py:364-429), plus
 * trajectory_signed_distances (tasks.py:251-275) at the solution.
 * `link` is the chain link (the trajectory's target link) whose root->link
 * chain carries every collision sphere.  One CTA per trajectory, 5 <= T <= 64.
 * Device arrays: q_init [B*T*n] (initial trajectories) or NULL,
 * anchors [B*2*n] (q_start, q_goal), obstacles [B*num_obstacles*8] =
 * (kind, a[3], b[3], radius|offset) in the robot base frame, unit normals.
 * q_init NULL = the straight line between the anchors (tasks.py:344-345).
 * Outputs: q [B*T*n], cost / initial cost [B], history
 * [B*(max_iterations+1)] (NULL ok), iterations / termination [B] (codes of
 * kop_lm_solve). */
typedef struct {
  int32_t timesteps;
  double dt;
  double w_anchor, w_smoothness, w_velocity, w_acceleration, w_jerk, w_limit, w_rest;
  double w_self, eta_self, w_world, eta_world, sharpness;
  int32_t hard_min;
  const double* velocity_limits; /* host [n], +inf where unlimited; NULL = all unlimited */
  const double* rest;            /* host [n], NULL = the model's rest pose */
} KopTrajCosts;

int kop_traj_solve(const KopModel* model, int32_t link, const KopTrajCosts* costs, const KopLmOptions* options,
                   const double* q_init, const double* anchors, const double* obstacles, int32_t num_obstacles,
                   int64_t batch, double* q_out, double* cost_out, double* init_cost_out, double* history_out,
                   int32_t* iterations_out, int32_t* termination_out, void* stream);
/* replaces: solver.assemble + _normal_equation_parts (solver.py:287-343) on
 * the plan_trajectory Problem: cost r.r [B], gradient J^T r [B*T*n] and
 * J^T J [B*(T*n)^2] (dense, zero outside the band) at trajectories qs
 * [B*T*n] -- the parity hook of kop_traj_solve (device arrays). */
int kop_traj_normal_equations(const KopModel* model, int32_t link, const KopTrajCosts* costs, int32_t precision,
                              const double* qs, const double* anchors, const double* obstacles,
                              int32_t num_obstacles, int64_t batch, double* cost_out, double* grad_out,
                              double* hess_out, void* stream);
/* replaces: trajectory_signed_distances (tasks.py:251-275) and the endpoint
 * _pose_errors of plan_trajectory (tasks.py:412-415), FP64, for B
 * trajectories qs [B*T*n] (device): static [B*T], swept [B*(T-1)], and
 * their minima [B] (+inf without obstacles); with targets [B*2*7] (start,
 * goal poses; NULL skips) pos_err / rot_err [B*2].  Output pointers may be
 * NULL except pos_err / rot_err when targets is given. */
int kop_traj_report(const KopModel* model, int32_t link, int32_t timesteps, const double* qs,
                    const double* obstacles, int32_t num_obstacles, const double* targets, int64_t batch,
                    double* static_out, double* swept_out, double* min_static, double* min_swept,
                    double* pos_err, double* rot_err, void* stream);

/* Multi-end-effector IK-Beam on a tree (config 3 as SURVEY.md section 8 H6
 * states it): IK-Beam (tasks.py:119-161) with the lane LM of beam.py:198-240
 * over [pose_1..pose_E | limit | rest] (KopPoseCosts weights and rest; the
 * params' w_* are ignored).  targets device [B*E*7]; seeds device [S*n].
 * Outputs (device): q [B*n], cost [B], history [B*(total_steps+1)] (NULL ok),
 * pos_err / rot_err [B*E] (FP64, tasks.py:109-116 per end effector),
 * success [B] (every end effector within tolerance).  One warp per lane;
 * keep <= 8, prune_after <= 31, total_steps - prune_after <= 32. */
int64_t kop_multi_pose_beam_workspace_bytes(const KopModel* model, const KopPoseCosts* costs,
                                            const KopIkParams* params, int64_t batch);
int kop_multi_pose_beam(const KopModel* model, const KopPoseCosts* costs, const KopIkParams* params,
                        const double* targets, int64_t batch, const double* seeds, void* workspace,
                        int64_t workspace_bytes, double* q_out, double* cost_out, double* history_out,
                        double* pos_err, double* rot_err, uint8_t* success, void* stream);

/* --- counter-based sampling ---------------------------------------------
 * replaces: tasks.sample_seed_configurations (tasks.py:88-106) and the draws
 * of benchmark.generate_reachable_targets (benchmark.py:83-93): row i is
 * numpy Generator(Philox(key=[key0, key1_base+i])).uniform(lo, hi), bit-exact;
 * negate[j] != 0 flips column j (continuous joints, tasks.py:105).
 * lo, hi, negate: host [n]; out: device [count*n] double. */
int kop_sample_uniform(uint64_t key0, uint64_t key1_base, int64_t count, int32_t n,
                       const double* lo, const double* hi, const uint8_t* negate, double* out,
                       void* stream);
/* FK (double) of `link` at configurations q[count*n] -> canonical poses
 * [count*7] (Transform3.from_parts canonicalisation, liegroups.py:323-325). */
int kop_link_poses(const KopModel* model, int32_t link, const double* q, int64_t count,
                   double* poses, void* stream);

/* --- measurement helper ---------------------------------------------------
 * FP32 FMA-pipe microbenchmark used for the roofline denominator (no FP32
 * entry exists in MEASURED_PEAKS.json).  Writes flops executed to *flops. */
int kop_fma_peak_kernel(int32_t blocks, int32_t threads, int32_t iters, float* sink, double* flops,
                        void* stream);
/* FP64 twin (8 independent DFMA chains per thread) for the FP64 roofline of
 * the parity-mode / widened kernels. */
int kop_dfma_peak_kernel(int32_t blocks, int32_t threads, int32_t iters, double* sink, double* flops,
                         void* stream);

/* --- per-term evaluation (FP64) ---------------------------------------------
 * replaces: the evaluator / jacobian closures of the typed cost builders
 * (costs.py:98-619) behind CostTerm.raw_residual (solver.py:142-152),
 * CostTerm.jacobian and solver.assemble (solver.py:289-324): the RAW
 * (unweighted) rows of one term at `count` evaluation points and the Jacobian
 * block of each referenced variable, in the reference's row order.
 * All arrays are device arrays; jacobian outputs may be null. */
#define KOP_BASE_NONE 0
#define KOP_BASE_SE2 1 /* base tangent (vx, vy, w)              */
#define KOP_BASE_SE3 2 /* base tangent (vx, vy, vz, wx, wy, wz) */
/* pose_cost (costs.py:98-166): r [count*6] = log(T_t^-1 (B) FK_link(q));
 * jq [count*6*n], jb [count*6*db] (db = 3 | 6); base [count*7] (wxyz, xyz),
 * SE(2) bases as their Transform3 (liegroups.py:450-454); target: host [7]. */
int kop_term_pose(const KopModel* model, int32_t link, const double* target, int32_t base_kind, const double* q,
                  const double* base, int64_t count, double* r, double* jq, double* jb, void* stream);
#define KOP_TERM_LIMIT 0      /* q               (costs.py:174-195) */
#define KOP_TERM_REST 1       /* q               (costs.py:259-271) */
#define KOP_TERM_SMOOTHNESS 2 /* q_prev, q_curr  (costs.py:274-290) */
#define KOP_TERM_VELOCITY 3   /* q_prev, q_curr  (costs.py:198-231) */
#define KOP_TERM_STENCIL 4    /* q_0..q_4, coeffs = stencil / dt^k (costs.py:293-341) */
/* joint-space rows: qs [count*nvars*n] (variable-major per point), r
 * [count*n], jdiag [count*nvars*n] = the diagonal of each variable's block
 * (every joint-space block is diagonal); rest, velocity_limits (+inf where
 * unlimited): host [n]; coeffs: host [5]. */
int kop_term_joint(const KopModel* model, int32_t kind, const double* rest, const double* velocity_limits, double dt,
                   const double* coeffs, const double* qs, int64_t count, double* r, double* jdiag, void* stream);
#define KOP_TERM_WORLD 5 /* q: one row per (sphere link, obstacle), link-major (costs.py:499-551) */
#define KOP_TERM_SELF 6  /* q: one row per model self pair (costs.py:435-496)                     */
#define KOP_TERM_SWEPT 7 /* q_prev, q_curr: capsules swept by every sphere (costs.py:554-619)     */
/* activation rows of a collision family: r [count*rows], j0 / j1 [count*rows*n]
 * (j1 for SWEPT only); obstacles: host, <= 16; returns the row count via
 * kop_term_rows. */
int kop_term_collision(const KopModel* model, int32_t kind, const KopObstacle* obstacles, int32_t num_obstacles,
                       double eta, double sharpness, int32_t hard_min, const double* q0, const double* q1,
                       int64_t count, double* r, double* j0, double* j1, void* stream);
/* manipulability_cost (costs.py:349-401): r [count] = 1 / (m + eps) with m the
 * Yoshikawa measure of `link`'s translational Jacobian, jrow [count*n] its
 * gradient row; jac [count*3*n] / djac [count*n*3*n] (nullable) = J and dJ/dq_a
 * (robot.translational_jacobian_with_derivative, robot.py:509-566).  n <= 32. */
int kop_term_manipulability(const KopModel* model, int32_t link, double eps, const double* q, int64_t count,
                            double* r, double* jrow, double* jac, double* djac, void* stream);
/* rows of a collision family for this model (negative status on error) */
int kop_term_rows(const KopModel* model, int32_t kind, int32_t num_obstacles);

/* --- checking builds ----------------------------------------------------
 * Copies `words` 32-bit words of a probe kernel's never-written dynamic
 * shared memory to device `out` (<= 12288 words).  In the shared-memory
 * poison build (kop_build_info() names it) every word is 0xFFFFFFFF. */
int kop_check_probe(uint32_t* out, int32_t words, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* KINOPTIK_B200_H */
