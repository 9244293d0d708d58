// Per-term evaluation (kop_terms.cu): kernel parameter blocks and launchers.
#pragma once

#include "kop_chain.h"
#include "kop_collision.cuh"
#include "kinoptik_b200.h"

namespace kop {

constexpr int kTreeMaxDofsTerms = 32;  // manipulability: actuated columns held per thread

struct LinkMap {  // parent joint of every link (-1 for the root)
  int32_t pj[kMaxLinks];
};

struct TermPose {
  double tinv[7];   // canonical inverse of the target (wxyz, xyz)
  int32_t base_kind;  // KOP_BASE_NONE / SE2 / SE3
};

struct TermJoint {
  int32_t kind, nvars;
  double lower[kMaxTreeJoints], upper[kMaxTreeJoints], rest[kMaxTreeJoints], vlim[kMaxTreeJoints];
  double dt, coeffs[5];
};

struct TermGeom {
  int32_t ns;                  // spheres, grouped by link in model order
  int32_t s_link[kMaxSpheres];
  double s_c[kMaxSpheres][3], s_r[kMaxSpheres];
  int32_t nl, links[kMaxSphereLinks];  // sphere-bearing links, model order
  int32_t np, pa[kMaxSelfPairs], pb[kMaxSelfPairs];  // self pairs (link indices)
  ObstacleTable<double> O;
  double eta, beta;
  int32_t hard;
};

cudaError_t launch_term_pose(const TreeParams& P, const LinkMap& L, int link, const TermPose& T, const double* q,
                             const double* base, int64_t B, double* r, double* jq, double* jb, cudaStream_t st);
cudaError_t launch_term_manip(const TreeParams& P, const LinkMap& L, int link, double eps, const double* q,
                              int64_t B, double* r, double* jrow, double* jac, double* djac, cudaStream_t st);
cudaError_t launch_term_joint(const TermJoint& T, int n, const double* qs, int64_t B, double* r, double* jd,
                              cudaStream_t st);
cudaError_t launch_term_collision(const TreeParams& P, const LinkMap& L, const TermGeom& G, int kind,
                                  const double* q0, const double* q1, int64_t B, double* r, double* j0, double* j1,
                                  cudaStream_t st);

}  // namespace kop
