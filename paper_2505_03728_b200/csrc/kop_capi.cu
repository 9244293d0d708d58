// C ABI (include/kinoptik_b200.h): model compilation, argument validation,
// shape dispatch.  Host code only; every compute path launches a kernel.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <future>

#include <string>
#include <vector>

#include "../../include/kinoptik_b200.h"
#include "kop_collision.cuh"
#include "kop_kernels.cuh"
#include "kop_traj.cuh"
#include "kop_terms.cuh"
#include "kop_tree.cuh"

using namespace kop;

struct KopModel {
  TreeParams tree;
  std::vector<double> lower, upper, rest;
  std::vector<int32_t> parent_joint;  // per link, -1 for the root
  // collision spheres (robot.py:66, sidecar) and default self pairs (robot.py:174-190)
  std::vector<int32_t> sphere_link;
  std::vector<double> sphere_center, sphere_radius;
  std::vector<int32_t> pair_links;  // [P*2]
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return KOP_OK;
  if (e == cudaErrorNotSupported)  // launchers return it for request shapes over a per-block limit
    return fail(KOP_EUNSUPPORTED, "request shape needs more shared memory per block than the device has "
                                  "(e.g. FP64 IK-Beam with more than 256 seeds)");
  return fail(KOP_ECUDA, std::string("CUDA error: ") + cudaGetErrorString(e));
}

// ---- quaternion helpers (host, double) -------------------------------------
struct HQ {
  double w, x, y, z;
};
HQ hmul(const HQ& a, const HQ& b) {
  return {a.w * b.w - (a.x * b.x + a.y * b.y + a.z * b.z),
          a.w * b.x + b.w * a.x + (a.y * b.z - a.z * b.y),
          a.w * b.y + b.w * a.y + (a.z * b.x - a.x * b.z),
          a.w * b.z + b.w * a.z + (a.x * b.y - a.y * b.x)};
}
void hrot(const HQ& q, const double p[3], double out[3]) {
  const double t0 = 2 * (q.y * p[2] - q.z * p[1]), t1 = 2 * (q.z * p[0] - q.x * p[2]),
               t2 = 2 * (q.x * p[1] - q.y * p[0]);
  out[0] = p[0] + q.w * t0 + (q.y * t2 - q.z * t1);
  out[1] = p[1] + q.w * t1 + (q.z * t0 - q.x * t2);
  out[2] = p[2] + q.w * t2 + (q.x * t1 - q.y * t0);
}
void hmat(const HQ& q, double r[3][3]) {
  const double xx = q.x * q.x, yy = q.y * q.y, zz = q.z * q.z, xy = q.x * q.y, xz = q.x * q.z,
               yz = q.y * q.z, wx = q.w * q.x, wy = q.w * q.y, wz = q.w * q.z;
  r[0][0] = 1 - 2 * (yy + zz); r[0][1] = 2 * (xy - wz); r[0][2] = 2 * (xz + wy);
  r[1][0] = 2 * (xy + wz); r[1][1] = 1 - 2 * (xx + zz); r[1][2] = 2 * (yz - wx);
  r[2][0] = 2 * (xz - wy); r[2][1] = 2 * (yz + wx); r[2][2] = 1 - 2 * (xx + yy);
}
// Rotation taking +z onto the unit vector a.
HQ align_z(const double a[3]) {
  if (a[2] < -1.0 + 1e-12) return {0.0, 1.0, 0.0, 0.0};
  HQ q{1.0 + a[2], -a[1], a[0], 0.0};
  const double n = sqrt(q.w * q.w + q.x * q.x + q.y * q.y + q.z * q.z);
  return {q.w / n, q.x / n, q.y / n, q.z / n};
}

constexpr int kChainMax = 8;

// Root->link moving-joint chain with fixed joints folded and axes aligned to
// +z (kop_chain.h).  Returns the number of moving joints or a negative status.
// frame of a link on the compiled path: aligned child frame of moving joint
// `slot` (-1: the root) composed with (q, p)
struct LinkFrame {
  int link, slot;
  HQ q;
  double p[3];
};

int compile_chain(const KopModel& m, int link, ChainParams<double, kChainMax>& C, bool& identity,
                  std::vector<LinkFrame>* frames = nullptr) {
  const TreeParams& P = m.tree;
  if (link < 0 || link >= P.nl) return fail(KOP_EINVAL, "unknown link index " + std::to_string(link));
  std::vector<int> path;
  for (int j = m.parent_joint[link]; j >= 0; j = m.parent_joint[P.parent[j]]) path.push_back(j);
  HQ pend{1, 0, 0, 0};
  double pend_p[3] = {0, 0, 0};
  int k = 0;
  memset(&C, 0, sizeof(C));
  if (frames) {
    frames->clear();
    frames->push_back({0, -1, {1, 0, 0, 0}, {0, 0, 0}});
  }
  for (auto it = path.rbegin(); it != path.rend(); ++it) {
    const int j = *it;
    const HQ oq{P.oq[j][0], P.oq[j][1], P.oq[j][2], P.oq[j][3]};
    double o[3];
    hrot(pend, P.op[j], o);
    const double tp[3] = {pend_p[0] + o[0], pend_p[1] + o[1], pend_p[2] + o[2]};
    if (P.kind[j] == KOP_JOINT_FIXED) {
      pend = hmul(pend, oq);
      memcpy(pend_p, tp, sizeof(tp));
      if (frames) frames->push_back({P.child[j], k - 1, pend, {pend_p[0], pend_p[1], pend_p[2]}});
      continue;
    }
    if (k >= kChainMax)
      return fail(KOP_EUNSUPPORTED, "chain has more than 8 moving joints (not compiled in)");
    const HQ al = align_z(P.axis[j]);
    const HQ tq = hmul(hmul(pend, oq), al);
    C.tq[k][0] = tq.w; C.tq[k][1] = tq.x; C.tq[k][2] = tq.y; C.tq[k][3] = tq.z;
    memcpy(C.tp[k], tp, sizeof(tp));
    hmat(tq, C.tr[k]);
    C.mult[k] = P.mult[j];
    C.offset[k] = P.offset[j];
    C.qcol[k] = P.qcol[j];
    C.prismatic[k] = P.kind[j] == KOP_JOINT_PRISMATIC ? 1 : 0;
    ++k;
    pend = {al.w, -al.x, -al.y, -al.z};
    pend_p[0] = pend_p[1] = pend_p[2] = 0.0;
    if (frames) frames->push_back({P.child[j], k - 1, pend, {0, 0, 0}});
  }
  C.eq[0] = pend.w; C.eq[1] = pend.x; C.eq[2] = pend.y; C.eq[3] = pend.z;
  memcpy(C.ep, pend_p, sizeof(pend_p));
  C.k = k;
  identity = (k == P.n);
  for (int i = 0; i < k && identity; ++i)
    identity = C.qcol[i] == i && C.mult[i] == 1.0 && C.offset[i] == 0.0 && !C.prismatic[i];
  return k;
}

template <typename T, int K>
ChainParams<T, K> cast_chain(const ChainParams<double, kChainMax>& D) {
  ChainParams<T, K> C;
  memset(&C, 0, sizeof(C));
  for (int k = 0; k < K && k < kChainMax; ++k) {
    for (int i = 0; i < 4; ++i) C.tq[k][i] = T(D.tq[k][i]);
    for (int i = 0; i < 3; ++i) C.tp[k][i] = T(D.tp[k][i]);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) C.tr[k][i][j] = T(D.tr[k][i][j]);
    C.mult[k] = T(D.mult[k]);
    C.offset[k] = T(D.offset[k]);
    C.qcol[k] = D.qcol[k];
    C.prismatic[k] = D.prismatic[k];
  }
  for (int i = 0; i < 4; ++i) C.eq[i] = T(D.eq[i]);
  for (int i = 0; i < 3; ++i) C.ep[i] = T(D.ep[i]);
  C.k = D.k;
  return C;
}

// Cost parameters; dimensions beyond the robot's n are padded with an
// unlimited, zero-rest, Jacobian-free joint: its normal-equation row is
// decoupled (A_ii = w_rest^2, g_i = 0), so the padded solve is exact.
// w: (position, orientation, limit, rest, base) row weights.
template <typename T, int NQ>
CostParams<T, NQ> make_costs(const KopModel& m, const double w[5]) {
  CostParams<T, NQ> W;
  const int n = m.tree.n;
  for (int i = 0; i < NQ; ++i) {
    W.lower[i] = i < n ? T(m.lower[i]) : T(-INFINITY);
    W.upper[i] = i < n ? T(m.upper[i]) : T(INFINITY);
    W.rest[i] = i < n ? T(m.rest[i]) : T(0);
  }
  W.w_pos = T(w[0]);
  W.w_ori = T(w[1]);
  W.w_lim = T(w[2]);
  W.w_rest = T(w[3]);
  W.w_base = T(w[4]);
  return W;
}

int next_pow2(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

// Shape selection shared by every chain-based entry point.
enum class Shape { kId2, kId6, kId7, kGen8, kNone };

Shape pick_shape(int n, int k, bool identity, bool base) {
  if (identity && n == 7) return Shape::kId7;
  if (!base && identity && n == 2) return Shape::kId2;
  if (!base && identity && n == 6) return Shape::kId6;
  if (n <= 8 && k <= 8) return Shape::kGen8;
  return Shape::kNone;
}

// Padded-configuration helpers: the generic shape works on NQ = 8 internally;
// the API arrays have stride n, so for n < 8 the host pads through device
// scratch allocated here (not on the Panda path, which is an ID shape).
struct PadBuf {
  double* ptr = nullptr;
  ~PadBuf() {
    if (ptr) cudaFree(ptr);
  }
};

int kernel_nq(Shape sh, int n) { return sh == Shape::kGen8 ? 8 : n; }

// Collision parameters for IK on `link` (kop_collision.cuh): every
// sphere-bearing link must lie on the compiled root->link chain.
int compile_collision(const KopModel& m, const std::vector<LinkFrame>& frames, const KopCollisionCosts* cc,
                      CollisionParams<double>& P) {
  memset(&P, 0, sizeof(P));
  if (!cc) return fail(KOP_EINVAL, "null collision costs");
  if (cc->num_obstacles < 0 || cc->num_obstacles > kMaxObstacles)
    return fail(KOP_EUNSUPPORTED, "more than 16 obstacles (not compiled in)");
  if ((cc->w_world > 0 && !(cc->eta_world > 0)) || (cc->w_self > 0 && !(cc->eta_self > 0)))
    return fail(KOP_EINVAL, "buffer distance must be positive");
  // sphere links in model order (spheres arrive grouped by link)
  std::vector<int> links, first, count, slot;
  for (size_t s = 0; s < m.sphere_link.size(); ++s) {
    const int l = m.sphere_link[s];
    if (links.empty() || links.back() != l) {
      int fi = -1;
      for (size_t f = 0; f < frames.size(); ++f)
        if (frames[f].link == l) fi = (int)f;
      if (fi < 0)
        return fail(KOP_EUNSUPPORTED, "collision spheres on link " + std::to_string(l) +
                                          ", which is not on the root->IK-link chain (not compiled in)");
      links.push_back(l);
      first.push_back((int)s);
      count.push_back(0);
      slot.push_back(frames[fi].slot);
    }
    count.back()++;
  }
  if ((int)links.size() > kMaxSphereLinks) return fail(KOP_EUNSUPPORTED, "more than 16 sphere links");
  for (size_t i = 1; i < slot.size(); ++i)
    if (slot[i] < slot[i - 1]) return fail(KOP_EUNSUPPORTED, "sphere links out of chain order");
  P.ns = (int)m.sphere_link.size();
  int slot_count[kMaxSlots] = {0};
  for (size_t li = 0; li < links.size(); ++li) {
    const LinkFrame* fr = nullptr;
    for (const auto& f : frames)
      if (f.link == links[li]) fr = &f;
    P.lfirst[li] = first[li];
    P.lcount[li] = count[li];
    P.lslot[li] = slot[li];
    slot_count[slot[li] + 1] += count[li];
    for (int s = first[li]; s < first[li] + count[li]; ++s) {
      double c[3];
      hrot(fr->q, &m.sphere_center[3 * s], c);
      for (int i = 0; i < 3; ++i) P.sc[s][i] = c[i] + fr->p[i];
      P.sr[s] = m.sphere_radius[s];
    }
  }
  P.slot_first[0] = 0;
  for (int k = 0; k < kMaxSlots; ++k) P.slot_first[k + 1] = P.slot_first[k] + slot_count[k];
  P.nl = (int)links.size();
  P.no = cc->w_world > 0 ? cc->num_obstacles : 0;
  for (int o = 0; o < P.no; ++o) {
    const KopObstacle& ob = cc->obstacles[o];
    if (ob.kind < 0 || ob.kind > 2) return fail(KOP_EINVAL, "unknown obstacle kind");
    P.okind[o] = ob.kind;
    double n = 1.0;
    if (ob.kind == KOP_OBSTACLE_HALFSPACE) {
      n = sqrt(ob.a[0] * ob.a[0] + ob.a[1] * ob.a[1] + ob.a[2] * ob.a[2]);
      if (n < 1e-12) return fail(KOP_EINVAL, "half-space normal must be nonzero");
    }
    for (int i = 0; i < 3; ++i) {
      P.oa[o][i] = ob.a[i] / n;
      P.ob[o][i] = ob.b[i];
    }
    P.orad[o] = ob.radius;
  }
  P.np = 0;
  if (cc->w_self > 0) {
    for (size_t p = 0; p + 1 < m.pair_links.size(); p += 2) {
      int a = -1, b = -1;
      for (size_t li = 0; li < links.size(); ++li) {
        if (links[li] == m.pair_links[p]) a = (int)li;
        if (links[li] == m.pair_links[p + 1]) b = (int)li;
      }
      if (a < 0 || b < 0) return fail(KOP_EUNSUPPORTED, "self pair link without spheres on the chain");
      P.pa[P.np] = a;
      P.pb[P.np] = b;
      P.np++;
    }
  }
  P.w_world = cc->w_world;
  P.eta_world = cc->eta_world > 0 ? cc->eta_world : 1.0;
  P.w_self = cc->w_self;
  P.eta_self = cc->eta_self > 0 ? cc->eta_self : 1.0;
  P.beta = cc->sharpness > 0 ? cc->sharpness : 100.0;
  P.hard = cc->hard_min;
  for (int li = 0; li < P.nl; ++li)
    P.lreach[li] = (P.hard || P.lcount[li] <= 1) ? 0.0 : log((double)P.lcount[li]) / P.beta;
  for (int p = 0; p < P.np; ++p) {
    const int c = P.lcount[P.pa[p]] * P.lcount[P.pb[p]];
    P.preach[p] = (P.hard || c <= 1) ? 0.0 : log((double)c) / P.beta;
  }
  return KOP_OK;
}

template <typename T>
CollisionParams<T> cast_collision(const CollisionParams<double>& D) {
  CollisionParams<T> P;
  memset(&P, 0, sizeof(P));
  P.ns = D.ns;
  for (int s = 0; s < kMaxSpheres; ++s) {
    for (int i = 0; i < 3; ++i) P.sc[s][i] = T(D.sc[s][i]);
    P.sr[s] = T(D.sr[s]);
  }
  for (int k = 0; k <= kMaxSlots; ++k) P.slot_first[k] = D.slot_first[k];
  P.nl = D.nl;
  for (int l = 0; l < kMaxSphereLinks; ++l) {
    P.lfirst[l] = D.lfirst[l];
    P.lcount[l] = D.lcount[l];
    P.lslot[l] = D.lslot[l];
  }
  P.no = D.no;
  for (int o = 0; o < kMaxObstacles; ++o) {
    P.okind[o] = D.okind[o];
    for (int i = 0; i < 3; ++i) {
      P.oa[o][i] = T(D.oa[o][i]);
      P.ob[o][i] = T(D.ob[o][i]);
    }
    P.orad[o] = T(D.orad[o]);
  }
  P.np = D.np;
  for (int p = 0; p < kMaxSelfPairs; ++p) {
    P.pa[p] = D.pa[p];
    P.pb[p] = D.pb[p];
  }
  P.w_world = T(D.w_world);
  P.eta_world = T(D.eta_world);
  P.w_self = T(D.w_self);
  P.eta_self = T(D.eta_self);
  P.beta = T(D.beta);
  P.hard = D.hard;
  for (int l = 0; l < kMaxSphereLinks; ++l) P.lreach[l] = T(D.lreach[l]);
  for (int p = 0; p < kMaxSelfPairs; ++p) P.preach[p] = T(D.preach[p]);
  return P;
}

int collision_rows(const KopModel& m, const CollisionParams<double>& P) {
  return 6 + 2 * m.tree.n + P.nl * P.no + P.np;
}

}  // namespace

extern "C" {

const char* kop_last_error(void) { return g_err.c_str(); }

#if defined(KOP_SMEM_POISON)
#define KOP_CHECK_MODE "; checking build: shared-memory poison"
#elif defined(KOP_JITTER)
#define KOP_CHECK_MODE "; checking build: barrier jitter"
#else
#define KOP_CHECK_MODE ""
#endif

const char* kop_build_info(void) {
  return "kinoptik_b200 sm_100a; fp32/fp64; IK lanes {id2, id6, id7, gen8} + SE(2) base {id7, gen8}; "
         "collision lanes / LM / trajectories {id7, gen8}; tree LM (n <= 32, 1..8 poses)" KOP_CHECK_MODE;
}

int kop_model_create(const KopModelDesc* d, KopModel** out) {
  if (!d || !out) return fail(KOP_EINVAL, "null argument");
  if (d->num_joints < 0 || d->num_joints > kMaxTreeJoints)
    return fail(KOP_EUNSUPPORTED, "more than 64 joints (not compiled in)");
  if (d->num_links != d->num_joints + 1)
    return fail(KOP_EINVAL, "a kinematic tree has num_links == num_joints + 1");
  if (d->num_actuated < 0 || d->num_actuated > d->num_joints)
    return fail(KOP_EINVAL, "bad actuated joint count");
  KopModel* m = new KopModel();
  memset(&m->tree, 0, sizeof(m->tree));
  TreeParams& P = m->tree;
  P.nl = d->num_links;
  P.nj = d->num_joints;
  P.n = d->num_actuated;
  m->parent_joint.assign(P.nl, -1);
  std::vector<char> placed(P.nl, 0);
  placed[0] = 1;
  for (int j = 0; j < P.nj; ++j) {
    const int pl = d->parent_link[j], cl = d->child_link[j];
    if (pl < 0 || pl >= P.nl || cl <= 0 || cl >= P.nl || !placed[pl] || placed[cl]) {
      delete m;
      return fail(KOP_EINVAL, "joints must be in topological order over links rooted at link 0");
    }
    placed[cl] = 1;
    const int kind = d->kind[j];
    if (kind < 0 || kind > 2) {
      delete m;
      return fail(KOP_EINVAL, "unknown joint kind");
    }
    const int qc = d->qcol[j];
    if ((kind == KOP_JOINT_FIXED) != (qc < 0) || qc >= P.n) {
      delete m;
      return fail(KOP_EINVAL, "qcol must be -1 exactly for fixed joints and < num_actuated");
    }
    P.parent[j] = pl;
    P.child[j] = cl;
    P.kind[j] = kind;
    P.qcol[j] = qc;
    P.mult[j] = d->mult[j];
    P.offset[j] = d->offset[j];
    for (int i = 0; i < 4; ++i) P.oq[j][i] = d->origin_wxyz[j * 4 + i];
    for (int i = 0; i < 3; ++i) {
      P.op[j][i] = d->origin_xyz[j * 3 + i];
      P.axis[j][i] = d->axis[j * 3 + i];
    }
    m->parent_joint[cl] = j;
  }
  if (d->num_spheres < 0 || d->num_spheres > kMaxSpheres || d->num_self_pairs < 0 ||
      d->num_self_pairs > kMaxSelfPairs) {
    delete m;
    return fail(KOP_EUNSUPPORTED, "more than 32 collision spheres or 64 self pairs (not compiled in)");
  }
  for (int s = 0; s < d->num_spheres; ++s) {
    const int l = d->sphere_link[s];
    if (l < 0 || l >= P.nl || !(d->sphere_radius[s] > 0.0)) {
      delete m;
      return fail(KOP_EINVAL, "bad collision sphere");
    }
    m->sphere_link.push_back(l);
    for (int i = 0; i < 3; ++i) m->sphere_center.push_back(d->sphere_center[3 * s + i]);
    m->sphere_radius.push_back(d->sphere_radius[s]);
  }
  for (int p = 0; p < 2 * d->num_self_pairs; ++p) {
    if (d->self_pair_links[p] < 0 || d->self_pair_links[p] >= P.nl) {
      delete m;
      return fail(KOP_EINVAL, "bad self-collision pair");
    }
    m->pair_links.push_back(d->self_pair_links[p]);
  }
  m->lower.assign(d->lower, d->lower + P.n);
  m->upper.assign(d->upper, d->upper + P.n);
  m->rest.assign(d->rest, d->rest + P.n);
  *out = m;
  return KOP_OK;
}

void kop_model_destroy(KopModel* m) { delete m; }

int kop_model_chain_length(const KopModel* m, int32_t link) {
  if (!m) return fail(KOP_EINVAL, "null model");
  ChainParams<double, kChainMax> C;
  bool id;
  const int k = compile_chain(*m, link, C, id);
  return k;
}

int kop_model_chain_export(const KopModel* m, int32_t link, double* tq, double* tp, int32_t* qcol, double* mult,
                           double* offset, int32_t* prismatic, double* ee) {
  if (!m) return fail(KOP_EINVAL, "null model");
  ChainParams<double, kChainMax> C;
  bool id;
  const int k = compile_chain(*m, link, C, id);
  if (k < 0) return k;
  for (int i = 0; i < k; ++i) {
    if (tq) memcpy(tq + 4 * i, C.tq[i], sizeof(C.tq[i]));
    if (tp) memcpy(tp + 3 * i, C.tp[i], sizeof(C.tp[i]));
    if (qcol) qcol[i] = C.qcol[i];
    if (mult) mult[i] = C.mult[i];
    if (offset) offset[i] = C.offset[i];
    if (prismatic) prismatic[i] = C.prismatic[i];
  }
  if (ee) {
    memcpy(ee, C.eq, sizeof(C.eq));
    memcpy(ee + 4, C.ep, sizeof(C.ep));
  }
  return k;
}

int kop_fk(const KopModel* m, int32_t precision, const double* q, int64_t batch, double* lq, double* lp,
           double* jp, double* ja, void* stream) {
  if (!m || batch < 0 || (batch > 0 && !q)) return fail(KOP_EINVAL, "invalid FK arguments");
  if (precision != KOP_FP32 && precision != KOP_FP64) return fail(KOP_EINVAL, "bad precision");
  return cuda_status(launch_fk_tree(m->tree, precision, q, batch, lq, lp, jp, ja, (cudaStream_t)stream));
}

int kop_jacobian(const KopModel* m, int32_t precision, const double* q, int64_t batch, int32_t link,
                 const double* points, int32_t rotational, double* jac, void* stream) {
  if (!m || batch < 0 || (batch > 0 && (!q || !jac))) return fail(KOP_EINVAL, "invalid Jacobian arguments");
  if (precision != KOP_FP32 && precision != KOP_FP64) return fail(KOP_EINVAL, "bad precision");
  if (link < 0 || link >= m->tree.nl) return fail(KOP_EINVAL, "unknown link index");
  unsigned long long anc = 0;  // joints on the root -> link path
  for (int j = m->parent_joint[link]; j >= 0; j = m->parent_joint[m->tree.parent[j]]) anc |= 1ull << j;
  return cuda_status(launch_jacobian_tree(m->tree, precision, q, batch, link, anc, points, rotational ? 1 : 0, jac,
                                          (cudaStream_t)stream));
}

int kop_link_poses(const KopModel* m, int32_t link, const double* q, int64_t count, double* poses,
                   void* stream) {
  if (!m || count < 0 || link < 0 || link >= m->tree.nl) return fail(KOP_EINVAL, "invalid arguments");
  TreeParams path;
  memset(&path, 0, sizeof(path));
  std::vector<int> js;
  for (int j = m->parent_joint[link]; j >= 0; j = m->parent_joint[m->tree.parent[j]]) js.push_back(j);
  path.n = m->tree.n;
  path.nj = (int)js.size();
  path.nl = path.nj + 1;
  for (int i = 0; i < path.nj; ++i) {
    const int j = js[js.size() - 1 - i];
    path.kind[i] = m->tree.kind[j];
    path.qcol[i] = m->tree.qcol[j];
    path.mult[i] = m->tree.mult[j];
    path.offset[i] = m->tree.offset[j];
    memcpy(path.oq[i], m->tree.oq[j], sizeof(path.oq[i]));
    memcpy(path.op[i], m->tree.op[j], sizeof(path.op[i]));
    memcpy(path.axis[i], m->tree.axis[j], sizeof(path.axis[i]));
  }
  return cuda_status(launch_link_pose(path, q, count, poses, (cudaStream_t)stream));
}

int kop_sample_uniform(uint64_t key0, uint64_t key1_base, int64_t count, int32_t n, const double* lo,
                       const double* hi, const uint8_t* negate, double* out, void* stream) {
  if (count < 0 || n < 0 || n > 64 || (count > 0 && !out)) return fail(KOP_EINVAL, "invalid arguments");
  // the per-column constants live in a small device buffer
  double* dev = nullptr;
  const size_t bytes = sizeof(double) * 2 * n + n;
  if (cudaMalloc(&dev, bytes + 16) != cudaSuccess) return cuda_status(cudaGetLastError());
  std::vector<double> host(2 * n);
  std::vector<uint8_t> neg(n);
  for (int j = 0; j < n; ++j) {
    host[j] = lo[j];
    host[n + j] = hi[j] - lo[j];  // numpy: arange = np.subtract(high, low)
    neg[j] = negate ? negate[j] : 0;
  }
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyAsync(dev, host.data(), sizeof(double) * 2 * n, cudaMemcpyHostToDevice, st);
  uint8_t* dneg = reinterpret_cast<uint8_t*>(dev + 2 * n);
  cudaMemcpyAsync(dneg, neg.data(), n, cudaMemcpyHostToDevice, st);
  cudaError_t e = launch_philox(key0, key1_base, count, n, dev, dev + n, dneg, out, st);
  cudaStreamSynchronize(st);  // host staging vectors die at return
  cudaFree(dev);
  return cuda_status(e != cudaSuccess ? e : cudaGetLastError());
}

int64_t kop_ik_beam_workspace_bytes(const KopModel* m, int32_t link, const KopIkParams* p, int64_t batch) {
  if (!m || !p || batch < 0) return fail(KOP_EINVAL, "invalid arguments");
  ChainParams<double, kChainMax> C;
  bool id;
  const int k = compile_chain(*m, link, C, id);
  if (k < 0) return k;
  const Shape sh = pick_shape(m->tree.n, k, id, p->optimize_base != 0);
  if (sh == Shape::kNone) return fail(KOP_EUNSUPPORTED, "robot shape not compiled in");
  const int nq = kernel_nq(sh, m->tree.n);
  const size_t el = p->precision == KOP_FP64 ? 8 : 4;
  const int64_t rec = nq + (p->optimize_base ? 3 : 0) + 2 + p->prune_after + 1;
  // survivor records, then (fixed base) the seed frame table: (7 + 6 K) x seeds, K <= 8
  const int64_t surv = (batch * (int64_t)p->keep * rec * (int64_t)el + 255) / 256 * 256;
  return surv + (int64_t)(7 + 6 * 8) * p->seeds * (int64_t)el + 256;
}

}  // extern "C"

namespace {

template <class G>
cudaError_t run_beam(const KopModel& m, const ChainParams<double, kChainMax>& D, const double w[5],
                     const BeamLaunch& L, cudaStream_t st) {
  return launch_beam<G>(cast_chain<typename G::T, G::K>(D), make_costs<typename G::T, G::NQ>(m, w),
                        cast_chain<double, G::K>(D), L, st);
}

template <typename T, bool BASE>
cudaError_t dispatch_beam(Shape sh, const KopModel& m, const ChainParams<double, kChainMax>& D,
                          const double w[5], const BeamLaunch& L, cudaStream_t st) {
  if constexpr (BASE) {
    switch (sh) {
      case Shape::kId7: return run_beam<Cfg<T, 7, 7, true, true>>(m, D, w, L, st);
      case Shape::kGen8: return run_beam<Cfg<T, 8, 8, false, true>>(m, D, w, L, st);
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (sh) {
      case Shape::kId7: return run_beam<Cfg<T, 7, 7, true, false>>(m, D, w, L, st);
      case Shape::kId2: return run_beam<Cfg<T, 2, 2, true, false>>(m, D, w, L, st);
      case Shape::kId6: return run_beam<Cfg<T, 6, 6, true, false>>(m, D, w, L, st);
      case Shape::kGen8: return run_beam<Cfg<T, 8, 8, false, false>>(m, D, w, L, st);
      default: return cudaErrorInvalidValue;
    }
  }
}

template <class G>
cudaError_t run_lane(const KopModel& m, const ChainParams<double, kChainMax>& D, const double w[5],
                     const LaneLaunch& L, cudaStream_t st) {
  return launch_lane<G>(cast_chain<typename G::T, G::K>(D), make_costs<typename G::T, G::NQ>(m, w), L, st);
}

template <typename T, bool BASE>
cudaError_t dispatch_lane(Shape sh, const KopModel& m, const ChainParams<double, kChainMax>& D,
                          const double w[5], const LaneLaunch& L, cudaStream_t st) {
  if constexpr (BASE) {
    switch (sh) {
      case Shape::kId7: return run_lane<Cfg<T, 7, 7, true, true>>(m, D, w, L, st);
      case Shape::kGen8: return run_lane<Cfg<T, 8, 8, false, true>>(m, D, w, L, st);
      default: return cudaErrorInvalidValue;
    }
  } else {
    switch (sh) {
      case Shape::kId7: return run_lane<Cfg<T, 7, 7, true, false>>(m, D, w, L, st);
      case Shape::kId2: return run_lane<Cfg<T, 2, 2, true, false>>(m, D, w, L, st);
      case Shape::kId6: return run_lane<Cfg<T, 6, 6, true, false>>(m, D, w, L, st);
      case Shape::kGen8: return run_lane<Cfg<T, 8, 8, false, false>>(m, D, w, L, st);
      default: return cudaErrorInvalidValue;
    }
  }
}

// Resolve the chain + shape for a lane / beam call.
int prepare(const KopModel* m, int link, int precision, bool base, ChainParams<double, kChainMax>& C, Shape& sh) {
  if (!m) return fail(KOP_EINVAL, "null model");
  if (precision != KOP_FP32 && precision != KOP_FP64) return fail(KOP_EINVAL, "bad precision");
  bool id = false;
  const int k = compile_chain(*m, link, C, id);
  if (k < 0) return k;
  sh = pick_shape(m->tree.n, k, id, base);
  if (sh == Shape::kNone)
    return fail(KOP_EUNSUPPORTED, "robot with " + std::to_string(m->tree.n) +
                                      " actuated joints is not compiled in (max 8)");
  return KOP_OK;
}

// Stride-n <-> stride-8 copies for the generic shape (kernels use stride NQ).
__global__ void k_restride(const double* __restrict__ src, int64_t rows, int sn, int dn, double pad,
                           double* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * dn) return;
  const int64_t r = i / dn;
  const int c = (int)(i % dn);
  dst[i] = c < sn ? src[r * sn + c] : pad;
}

cudaError_t restride(const double* src, int64_t rows, int sn, int dn, double* dst, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  const int64_t total = rows * dn;
  k_restride<<<(unsigned)((total + 127) / 128), 128, 0, st>>>(src, rows, sn, dn, 0.0, dst);
  return cudaGetLastError();
}

}  // namespace

extern "C" {

int kop_ik_beam_stage(const KopModel* m, int32_t link, const KopIkParams* p, int32_t stages, const double* targets,
                      int64_t batch, const double* seeds, void* workspace, int64_t workspace_bytes, double* q_out,
                      double* base_out, double* cost_out, double* history_out, double* pos_err, double* rot_err,
                      uint8_t* success, void* stream) {
  if (stages < 1 || stages > 3) return fail(KOP_EINVAL, "stages must be 1, 2 or 3");
  if (!p) return fail(KOP_EINVAL, "null params");
  const bool base = p->optimize_base != 0;
  ChainParams<double, kChainMax> C;
  Shape sh;
  int rc = prepare(m, link, p->precision, base, C, sh);
  if (rc != KOP_OK) return rc;
  // IkRequest.__post_init__ (tasks.py:56-60)
  if (!(0 < p->prune_after && p->prune_after < p->total_steps))
    return fail(KOP_EINVAL, "need 0 < prune_after < total_steps");
  if (!(1 <= p->keep && p->keep <= p->seeds)) return fail(KOP_EINVAL, "need 1 <= keep <= seeds");
  if (p->seeds > 1024 || p->keep > 32)
    return fail(KOP_EUNSUPPORTED, "seeds <= 1024 and keep <= 32 are compiled in");
  if (batch < 0) return fail(KOP_EINVAL, "negative batch");
  if (batch == 0) return KOP_OK;
  if (!targets || !seeds || !workspace || !q_out || !cost_out || !pos_err || !rot_err || !success)
    return fail(KOP_EINVAL, "null array argument");
  const int64_t need = kop_ik_beam_workspace_bytes(m, link, p, batch);
  if (workspace_bytes < need) return fail(KOP_EINVAL, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int n = m->tree.n;
  const int nq = kernel_nq(sh, n);
  if (nq != n && stages != 3)
    return fail(KOP_EUNSUPPORTED, "split-stage launches need n == 8 or an identity-chain shape");
  PadBuf seeds_pad, q_pad;
  const double* seeds_k = seeds;
  double* q_k = q_out;
  if (nq != n) {
    if (cudaMalloc(&seeds_pad.ptr, sizeof(double) * nq * p->seeds) != cudaSuccess ||
        cudaMalloc(&q_pad.ptr, sizeof(double) * nq * batch) != cudaSuccess)
      return cuda_status(cudaGetLastError());
    rc = cuda_status(restride(seeds, p->seeds, n, nq, seeds_pad.ptr, st));
    if (rc) return rc;
    seeds_k = seeds_pad.ptr;
    q_k = q_pad.ptr;
  }
  BeamLaunch L;
  L.targets = targets;
  L.B = batch;
  L.seeds = seeds_k;
  L.S = p->seeds;
  L.P = next_pow2(p->seeds);
  L.G = next_pow2(p->keep);
  L.steps1 = p->prune_after;
  L.steps2 = p->total_steps - p->prune_after;
  L.keep = p->keep;
  L.pos_tol = p->success_pos_tol;
  L.rot_tol = p->success_rot_tol;
  L.workspace = workspace;
  L.q_out = q_k;
  L.base_out = base_out;
  L.cost_out = cost_out;
  L.hist_out = history_out;
  L.pos_err = pos_err;
  L.rot_err = rot_err;
  L.success = success;
  L.stages = stages;
  const double w[5] = {p->w_position, p->w_orientation, p->w_limit, p->w_rest, p->w_base};
  cudaError_t e;
  if (p->precision == KOP_FP32)
    e = base ? dispatch_beam<float, true>(sh, *m, C, w, L, st) : dispatch_beam<float, false>(sh, *m, C, w, L, st);
  else
    e = base ? dispatch_beam<double, true>(sh, *m, C, w, L, st) : dispatch_beam<double, false>(sh, *m, C, w, L, st);
  if (e == cudaSuccess && q_k != q_out) e = restride(q_k, batch, nq, n, q_out, st);
  if (seeds_pad.ptr) cudaStreamSynchronize(st);  // scratch freed at return
  return cuda_status(e);
}

int kop_ik_beam(const KopModel* m, int32_t link, const KopIkParams* p, const double* targets, int64_t batch,
                const double* seeds, void* workspace, int64_t workspace_bytes, double* q_out, double* base_out,
                double* cost_out, double* history_out, double* pos_err, double* rot_err, uint8_t* success,
                void* stream) {
  return kop_ik_beam_stage(m, link, p, 3, targets, batch, seeds, workspace, workspace_bytes, q_out, base_out,
                           cost_out, history_out, pos_err, rot_err, success, stream);
}

static int lane_call(const KopModel* m, int32_t link, int32_t precision, const double* weights, LaneLaunch L,
                     int64_t lanes, void* stream) {
  const bool base = L.base_in != nullptr || L.base_io != nullptr;
  ChainParams<double, kChainMax> C;
  Shape sh;
  int rc = prepare(m, link, precision, base, C, sh);
  if (rc != KOP_OK) return rc;
  if (!weights) return fail(KOP_EINVAL, "null weights");
  if (lanes < 0) return fail(KOP_EINVAL, "negative lane count");
  if (lanes == 0) return KOP_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int n = m->tree.n;
  const int nq = kernel_nq(sh, n);
  const int nd = nq + (base ? 3 : 0), ndu = n + (base ? 3 : 0);
  L.lanes = lanes;
  PadBuf qin, qio, res, jac;
  double* user_qio = L.q_io;
  double* user_res = L.res;
  double* user_jac = L.jac;
  if (nq != n) {  // pad to the kernel stride
    if (L.q_in) {
      if (cudaMalloc(&qin.ptr, sizeof(double) * nq * lanes) != cudaSuccess) return cuda_status(cudaGetLastError());
      if ((rc = cuda_status(restride(L.q_in, lanes, n, nq, qin.ptr, st)))) return rc;
      L.q_in = qin.ptr;
    }
    if (L.q_io) {
      if (cudaMalloc(&qio.ptr, sizeof(double) * nq * lanes) != cudaSuccess) return cuda_status(cudaGetLastError());
      if ((rc = cuda_status(restride(L.q_io, lanes, n, nq, qio.ptr, st)))) return rc;
      L.q_io = qio.ptr;
    }
    if (L.res) {
      const int M = 6 + 2 * nq + (base ? 3 : 0);
      if (cudaMalloc(&res.ptr, sizeof(double) * M * lanes) != cudaSuccess ||
          cudaMalloc(&jac.ptr, sizeof(double) * M * nd * lanes) != cudaSuccess)
        return cuda_status(cudaGetLastError());
      L.res = res.ptr;
      L.jac = jac.ptr;
    }
  }
  cudaError_t e;
  if (precision == KOP_FP32)
    e = base ? dispatch_lane<float, true>(sh, *m, C, weights, L, st)
             : dispatch_lane<float, false>(sh, *m, C, weights, L, st);
  else
    e = base ? dispatch_lane<double, true>(sh, *m, C, weights, L, st)
             : dispatch_lane<double, false>(sh, *m, C, weights, L, st);
  if (e == cudaSuccess && nq != n) {
    if (user_qio) e = restride(L.q_io, lanes, nq, n, user_qio, st);
    if (e == cudaSuccess && user_res) {
      // rows: pose 6 | limit nq | rest nq | base 3  ->  pose 6 | limit n | rest n | base 3;
      // cols: q nq | base 3  ->  q n | base 3
      const int Mk = 6 + 2 * nq + (base ? 3 : 0), Mu = 6 + 2 * n + (base ? 3 : 0);
      std::vector<int> rowmap;
      for (int r = 0; r < 6; ++r) rowmap.push_back(r);
      for (int r = 0; r < n; ++r) rowmap.push_back(6 + r);
      for (int r = 0; r < n; ++r) rowmap.push_back(6 + nq + r);
      if (base)
        for (int r = 0; r < 3; ++r) rowmap.push_back(6 + 2 * nq + r);
      for (int r = 0; r < Mu && e == cudaSuccess; ++r) {
        e = cudaMemcpy2DAsync(user_res + r, sizeof(double) * Mu, L.res + rowmap[r], sizeof(double) * Mk,
                              sizeof(double), lanes, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess)
          e = cudaMemcpy2DAsync(user_jac + (size_t)r * ndu, sizeof(double) * Mu * ndu,
                                L.jac + (size_t)rowmap[r] * nd, sizeof(double) * Mk * nd, sizeof(double) * n,
                                lanes, cudaMemcpyDeviceToDevice, st);
        if (e == cudaSuccess && base)
          e = cudaMemcpy2DAsync(user_jac + (size_t)r * ndu + n, sizeof(double) * Mu * ndu,
                                L.jac + (size_t)rowmap[r] * nd + nq, sizeof(double) * Mk * nd, sizeof(double) * 3,
                                lanes, cudaMemcpyDeviceToDevice, st);
      }
    }
    cudaStreamSynchronize(st);  // scratch freed at return
  }
  return cuda_status(e);
}

int kop_lane_residuals_jacobian(const KopModel* m, int32_t link, int32_t precision, const double* weights,
                                const double* tinv, const int32_t* lane_target, const double* q,
                                const double* base_state, int64_t lanes, double* residual, double* jacobian,
                                void* stream) {
  if (lanes > 0 && (!tinv || !lane_target || !q || !residual || !jacobian))
    return fail(KOP_EINVAL, "null array argument");
  LaneLaunch L{};
  L.op = LaneOp::kResJac;
  L.tinv = tinv;
  L.lane_target = lane_target;
  L.q_in = q;
  L.base_in = base_state;
  L.res = residual;
  L.jac = jacobian;
  return lane_call(m, link, precision, weights, L, lanes, stream);
}

int kop_lane_start(const KopModel* m, int32_t link, int32_t precision, const double* weights,
                   const double* tinv, const int32_t* lane_target, const double* q, const double* base_state,
                   int64_t lanes, double* damping, double* cost, void* stream) {
  if (lanes > 0 && (!tinv || !lane_target || !q || !damping || !cost))
    return fail(KOP_EINVAL, "null array argument");
  LaneLaunch L{};
  L.op = LaneOp::kStart;
  L.tinv = tinv;
  L.lane_target = lane_target;
  L.q_in = q;
  L.base_in = base_state;
  L.lam = damping;
  L.cost = cost;
  return lane_call(m, link, precision, weights, L, lanes, stream);
}

int kop_lane_run(const KopModel* m, int32_t link, int32_t precision, const double* weights, const double* tinv,
                 const int32_t* lane_target, int64_t lanes, int32_t steps, double* q, double* base_state,
                 double* damping, double* cost, double* history, void* stream) {
  if (steps < 0) return fail(KOP_EINVAL, "negative step count");
  if (lanes > 0 && (!tinv || !lane_target || !q || !damping || !cost))
    return fail(KOP_EINVAL, "null array argument");
  LaneLaunch L{};
  L.op = LaneOp::kRun;
  L.tinv = tinv;
  L.lane_target = lane_target;
  L.steps = steps;
  L.q_io = q;
  L.base_io = base_state;
  L.lam = damping;
  L.cost = cost;
  L.hist = history;
  return lane_call(m, link, precision, weights, L, lanes, stream);
}

}  // extern "C"

namespace {

template <class G>
cudaError_t run_col(const KopModel& m, const ChainParams<double, kChainMax>& D, const CollisionParams<double>& PD,
                    const double w[5], const ColLaunch& L, cudaStream_t st) {
  return launch_col<G>(cast_chain<typename G::T, G::K>(D), make_costs<typename G::T, G::NQ>(m, w),
                       cast_collision<typename G::T>(PD), cast_chain<double, G::K>(D), L, st);
}

template <typename T>
cudaError_t dispatch_col(Shape sh, const KopModel& m, const ChainParams<double, kChainMax>& D,
                         const CollisionParams<double>& PD, const double w[5], const ColLaunch& L, cudaStream_t st) {
  switch (sh) {
    case Shape::kId7: return run_col<Cfg<T, 7, 7, true, false>>(m, D, PD, w, L, st);
    case Shape::kGen8: return run_col<Cfg<T, 8, 8, false, false>>(m, D, PD, w, L, st);
    default: return cudaErrorInvalidValue;
  }
}

// chain + collision params + collision shape (id7 or the padded generic shape)
int prepare_col(const KopModel* m, int link, int precision, const KopCollisionCosts* cc,
                ChainParams<double, kChainMax>& C, CollisionParams<double>& PD, Shape& sh) {
  if (!m) return fail(KOP_EINVAL, "null model");
  if (precision != KOP_FP32 && precision != KOP_FP64) return fail(KOP_EINVAL, "bad precision");
  bool id = false;
  std::vector<LinkFrame> frames;
  const int k = compile_chain(*m, link, C, id, &frames);
  if (k < 0) return k;
  sh = (id && m->tree.n == 7) ? Shape::kId7 : (m->tree.n <= 8 ? Shape::kGen8 : Shape::kNone);
  if (sh == Shape::kNone) return fail(KOP_EUNSUPPORTED, "collision IK supports up to 8 actuated joints");
  return compile_collision(*m, frames, cc, PD);
}

void col_weights(const KopCollisionCosts* cc, double w[5]) {
  w[0] = cc->w_position;
  w[1] = cc->w_orientation;
  w[2] = cc->w_limit;
  w[3] = cc->w_rest;
  w[4] = 0.0;
}

}  // namespace

extern "C" {

int kop_collision_rows(const KopModel* m, int32_t link, const KopCollisionCosts* cc) {
  ChainParams<double, kChainMax> C;
  CollisionParams<double> PD;
  Shape sh;
  const int rc = prepare_col(m, link, KOP_FP64, cc, C, PD, sh);
  return rc != KOP_OK ? rc : collision_rows(*m, PD);
}

int kop_collision_residuals_jacobian(const KopModel* m, int32_t link, int32_t precision, const KopCollisionCosts* cc,
                                     const double* tinv, const int32_t* lane_target, const double* q,
                                     int64_t lanes, double* residual, double* jacobian, void* stream) {
  ChainParams<double, kChainMax> C;
  CollisionParams<double> PD;
  Shape sh;
  int rc = prepare_col(m, link, precision, cc, C, PD, sh);
  if (rc != KOP_OK) return rc;
  if (lanes < 0) return fail(KOP_EINVAL, "negative lane count");
  if (lanes == 0) return KOP_OK;
  if (!tinv || !lane_target || !q || !residual || !jacobian) return fail(KOP_EINVAL, "null array argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int n = m->tree.n, nq = kernel_nq(sh, n);
  const int R = collision_rows(*m, PD), Rk = R + 2 * (nq - n);
  PadBuf qin, res, jac;
  ColLaunch L{};
  L.op = ColOp::kResJac;
  L.tinv = tinv;
  L.lane_target = lane_target;
  L.q_in = q;
  L.lanes = lanes;
  L.rows = Rk;
  L.res = residual;
  L.jac = jacobian;
  if (nq != n) {
    if (cudaMalloc(&qin.ptr, sizeof(double) * nq * lanes) != cudaSuccess ||
        cudaMalloc(&res.ptr, sizeof(double) * Rk * lanes) != cudaSuccess ||
        cudaMalloc(&jac.ptr, sizeof(double) * Rk * nq * lanes) != cudaSuccess)
      return cuda_status(cudaGetLastError());
    if ((rc = cuda_status(restride(q, lanes, n, nq, qin.ptr, st)))) return rc;
    L.q_in = qin.ptr;
    L.res = res.ptr;
    L.jac = jac.ptr;
  }
  double w[5];
  col_weights(cc, w);
  cudaError_t e = precision == KOP_FP32 ? dispatch_col<float>(sh, *m, C, PD, w, L, st)
                                        : dispatch_col<double>(sh, *m, C, PD, w, L, st);
  if (e == cudaSuccess && nq != n) {
    std::vector<int> rowmap;
    for (int r = 0; r < 6; ++r) rowmap.push_back(r);
    for (int r = 0; r < n; ++r) rowmap.push_back(6 + r);
    for (int r = 0; r < n; ++r) rowmap.push_back(6 + nq + r);
    for (int r = 6 + 2 * n; r < R; ++r) rowmap.push_back(r + 2 * (nq - n));
    for (int r = 0; r < R && e == cudaSuccess; ++r) {
      e = cudaMemcpy2DAsync(residual + r, sizeof(double) * R, L.res + rowmap[r], sizeof(double) * Rk,
                            sizeof(double), lanes, cudaMemcpyDeviceToDevice, st);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(jacobian + (size_t)r * n, sizeof(double) * R * n, L.jac + (size_t)rowmap[r] * nq,
                              sizeof(double) * Rk * nq, sizeof(double) * n, lanes, cudaMemcpyDeviceToDevice, st);
    }
    cudaStreamSynchronize(st);
  }
  return cuda_status(e);
}

int64_t kop_ik_beam_collision_workspace_bytes(const KopModel* m, int32_t link, const KopIkParams* p,
                                              const KopCollisionCosts* cc, int64_t batch) {
  if (!p || batch < 0) return fail(KOP_EINVAL, "invalid arguments");
  ChainParams<double, kChainMax> C;
  CollisionParams<double> PD;
  Shape sh;
  const int rc = prepare_col(m, link, p->precision, cc, C, PD, sh);
  if (rc != KOP_OK) return rc;
  const int64_t rec = kernel_nq(sh, m->tree.n) + 2 + p->prune_after + 1;
  return batch * (int64_t)p->keep * rec * (p->precision == KOP_FP64 ? 8 : 4) + 256;
}

int kop_ik_beam_collision(const KopModel* m, int32_t link, const KopIkParams* p, const KopCollisionCosts* cc,
                          const double* targets, int64_t batch, const double* seeds, void* workspace,
                          int64_t workspace_bytes, double* q_out, double* cost_out, double* history_out,
                          double* pos_err, double* rot_err, uint8_t* success, void* stream) {
  if (!p) return fail(KOP_EINVAL, "null params");
  ChainParams<double, kChainMax> C;
  CollisionParams<double> PD;
  Shape sh;
  int rc = prepare_col(m, link, p->precision, cc, C, PD, sh);
  if (rc != KOP_OK) return rc;
  if (!(0 < p->prune_after && p->prune_after < p->total_steps))
    return fail(KOP_EINVAL, "need 0 < prune_after < total_steps");
  if (!(1 <= p->keep && p->keep <= p->seeds)) return fail(KOP_EINVAL, "need 1 <= keep <= seeds");
  if (p->seeds > 128 || p->keep > 32)
    return fail(KOP_EUNSUPPORTED, "collision IK-Beam supports seeds <= 128 and keep <= 32");
  if (batch < 0) return fail(KOP_EINVAL, "negative batch");
  if (batch == 0) return KOP_OK;
  if (!targets || !seeds || !workspace || !q_out || !cost_out || !pos_err || !rot_err || !success)
    return fail(KOP_EINVAL, "null array argument");
  if (workspace_bytes < kop_ik_beam_collision_workspace_bytes(m, link, p, cc, batch))
    return fail(KOP_EINVAL, "workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  const int n = m->tree.n, nq = kernel_nq(sh, n);
  PadBuf seeds_pad, q_pad;
  const double* seeds_k = seeds;
  double* q_k = q_out;
  if (nq != n) {
    if (cudaMalloc(&seeds_pad.ptr, sizeof(double) * nq * p->seeds) != cudaSuccess ||
        cudaMalloc(&q_pad.ptr, sizeof(double) * nq * batch) != cudaSuccess)
      return cuda_status(cudaGetLastError());
    if ((rc = cuda_status(restride(seeds, p->seeds, n, nq, seeds_pad.ptr, st)))) return rc;
    seeds_k = seeds_pad.ptr;
    q_k = q_pad.ptr;
  }
  ColLaunch L{};
  L.op = ColOp::kBeam;
  BeamLaunch& Bm = L.beam;
  Bm.targets = targets;
  Bm.B = batch;
  Bm.seeds = seeds_k;
  Bm.S = p->seeds;
  Bm.P = next_pow2(p->seeds);
  Bm.G = next_pow2(p->keep);
  Bm.steps1 = p->prune_after;
  Bm.steps2 = p->total_steps - p->prune_after;
  Bm.keep = p->keep;
  Bm.pos_tol = p->success_pos_tol;
  Bm.rot_tol = p->success_rot_tol;
  Bm.workspace = workspace;
  Bm.q_out = q_k;
  Bm.base_out = nullptr;
  Bm.cost_out = cost_out;
  Bm.hist_out = history_out;
  Bm.pos_err = pos_err;
  Bm.rot_err = rot_err;
  Bm.success = success;
  Bm.stages = 3;
  double w[5];
  col_weights(cc, w);
  cudaError_t e = p->precision == KOP_FP32 ? dispatch_col<float>(sh, *m, C, PD, w, L, st)
                                           : dispatch_col<double>(sh, *m, C, PD, w, L, st);
  if (e == cudaSuccess && q_k != q_out) e = restride(q_k, batch, nq, n, q_out, st);
  if (seeds_pad.ptr) cudaStreamSynchronize(st);
  return cuda_status(e);
}

int kop_lm_solve(const KopModel* m, int32_t link, const KopCollisionCosts* cc, const KopLmOptions* o,
                 const double* targets, const double* q0, int64_t batch, double* q_out, double* cost_out,
                 double* init_cost_out, double* history_out, int32_t* iterations_out, int32_t* termination_out,
                 void* stream) {
  if (!o) return fail(KOP_EINVAL, "null options");
  ChainParams<double, kChainMax> C;
  CollisionParams<double> PD;
  Shape sh;
  int rc = prepare_col(m, link, o->precision, cc, C, PD, sh);
  if (rc != KOP_OK) return rc;
  // SolveOptions.__post_init__ (solver.py:190-198)
  if (o->max_iterations <= 0 || !(o->initial_damping > 0)) return fail(KOP_EINVAL, "max_iterations and initial_damping must be positive");
  if (!(o->damping_increase > 1.0)) return fail(KOP_EINVAL, "damping_increase must exceed 1");
  if (!(o->damping_decrease > 0.0 && o->damping_decrease < 1.0)) return fail(KOP_EINVAL, "damping_decrease must be in (0, 1)");
  if (o->max_rejections < 0) return fail(KOP_EINVAL, "max_rejections must be nonnegative");
  if (batch < 0) return fail(KOP_EINVAL, "negative batch");
  if (batch == 0) return KOP_OK;
  if (!targets || !q0 || !q_out || !cost_out || !init_cost_out || !iterations_out || !termination_out)
    return fail(KOP_EINVAL, "null array argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int n = m->tree.n, nq = kernel_nq(sh, n);
  PadBuf q0p, qop;
  ColLaunch L{};
  L.op = ColOp::kSolve;
  L.targets = targets;
  L.q_in = q0;
  L.B = batch;
  L.q_out = q_out;
  L.cost_out = cost_out;
  L.init_cost = init_cost_out;
  L.hist_out = history_out;
  L.iters = iterations_out;
  L.term = termination_out;
  L.opts = {o->max_iterations, o->max_rejections, o->initial_damping, o->damping_increase, o->damping_decrease,
            o->gradient_tolerance, o->step_tolerance};
  if (nq != n) {
    if (cudaMalloc(&q0p.ptr, sizeof(double) * nq * batch) != cudaSuccess ||
        cudaMalloc(&qop.ptr, sizeof(double) * nq * batch) != cudaSuccess)
      return cuda_status(cudaGetLastError());
    if ((rc = cuda_status(restride(q0, batch, n, nq, q0p.ptr, st)))) return rc;
    L.q_in = q0p.ptr;
    L.q_out = qop.ptr;
  }
  double w[5];
  col_weights(cc, w);
  cudaError_t e = o->precision == KOP_FP32 ? dispatch_col<float>(sh, *m, C, PD, w, L, st)
                                           : dispatch_col<double>(sh, *m, C, PD, w, L, st);
  if (e == cudaSuccess && nq != n) {
    e = restride(qop.ptr, batch, nq, n, q_out, st);
    cudaStreamSynchronize(st);
  }
  return cuda_status(e);
}

}  // extern "C"

namespace {

// double-precision pose (wxyz, xyz) composition a o b
struct HostPose {
  double q[4] = {1, 0, 0, 0}, p[3] = {0, 0, 0};
};
HostPose host_compose(const HostPose& a, const HostPose& b) {
  HostPose r;
  const double *x = a.q, *y = b.q;
  r.q[0] = x[0] * y[0] - x[1] * y[1] - x[2] * y[2] - x[3] * y[3];
  r.q[1] = x[0] * y[1] + x[1] * y[0] + x[2] * y[3] - x[3] * y[2];
  r.q[2] = x[0] * y[2] - x[1] * y[3] + x[2] * y[0] + x[3] * y[1];
  r.q[3] = x[0] * y[3] + x[1] * y[2] - x[2] * y[1] + x[3] * y[0];
  // p_a + R(q_a) p_b
  const double w = x[0], vx = x[1], vy = x[2], vz = x[3], *v = b.p;
  const double tx = 2 * (vy * v[2] - vz * v[1]), ty = 2 * (vz * v[0] - vx * v[2]), tz = 2 * (vx * v[1] - vy * v[0]);
  r.p[0] = a.p[0] + v[0] + w * tx + (vy * tz - vz * ty);
  r.p[1] = a.p[1] + v[1] + w * ty + (vz * tx - vx * tz);
  r.p[2] = a.p[2] + v[2] + w * tz + (vx * ty - vy * tx);
  return r;
}

// Kernel view of the tree.  fold: fixed joints are folded into their children's
// origin transforms (and into the end-effector offsets) in double, so the
// kernel's FK runs over the moving joints only -- the humanoid's 34 joints
// become 29, one warp pass; the composed transforms are exact up to the final
// rounding.  Unfolded (fold = false) for the FP64 pose errors, which follow
// the reference's joint-by-joint walk.
template <typename T>
TreeLmParams<T> tree_params(const KopModel& m, const KopPoseCosts* pc, bool fold = true) {
  TreeLmParams<T> P;
  memset(&P, 0, sizeof(P));
  const TreeParams& t = m.tree;
  const int nj0 = t.nj;
  std::vector<int> pj(nj0), nid(nj0, -1), eff(nj0, -1);
  std::vector<HostPose> acc(nj0);  // fixed joint j: after(j) = after(eff[j]) o acc[j]
  int nj = 0;
  for (int j = 0; j < nj0; ++j) {
    pj[j] = m.parent_joint[t.parent[j]];
    HostPose o;
    for (int i = 0; i < 4; ++i) o.q[i] = t.oq[j][i];
    for (int i = 0; i < 3; ++i) o.p[i] = t.op[j][i];
    const bool pfix = fold && pj[j] >= 0 && nid[pj[j]] < 0;  // parent folded away
    const HostPose pre = pfix ? acc[pj[j]] : HostPose();
    const int par = pj[j] < 0 ? -1 : (pfix ? eff[pj[j]] : pj[j]);
    if (fold && t.kind[j] == 0) {
      eff[j] = par;
      acc[j] = pfix ? host_compose(pre, o) : o;
      continue;
    }
    const int k = nj++;
    nid[j] = k;
    const HostPose oj = pfix ? host_compose(pre, o) : o;
    P.parent_joint[k] = par < 0 ? -1 : nid[par];
    P.kind[k] = t.kind[j];
    P.qcol[k] = t.qcol[j];
    for (int i = 0; i < 4; ++i) P.oq[k][i] = T(oj.q[i]);
    for (int i = 0; i < 3; ++i) {
      P.op[k][i] = T(oj.p[i]);
      P.axis[k][i] = T(t.axis[j][i]);
    }
    P.mult[k] = T(t.mult[j]);
    P.offset[k] = T(t.offset[j]);
  }
  P.nj = nj;
  P.n = t.n;
  P.ne = pc->num_poses;
  for (int e = 0; e < pc->num_poses; ++e) {
    const int ej = m.parent_joint[pc->links[e]];
    HostPose off;
    int k = -1;
    if (ej >= 0 && nid[ej] >= 0) {
      k = nid[ej];
    } else if (ej >= 0) {
      k = eff[ej] < 0 ? -1 : nid[eff[ej]];
      off = acc[ej];
    }
    P.ee_joint[e] = k;
    for (int i = 0; i < 4; ++i) P.ee_oq[e][i] = T(off.q[i]);
    for (int i = 0; i < 3; ++i) P.ee_op[e][i] = T(off.p[i]);
    unsigned long long mask = 0;
    for (int a = k; a >= 0; a = P.parent_joint[a]) mask |= 1ull << a;
    P.anc_ee[e] = mask;
    P.w_pos[e] = T(pc->w_position[e]);
    P.w_ori[e] = T(pc->w_orientation[e]);
  }
  for (int i = 0; i < t.n; ++i) {
    P.lower[i] = T(m.lower[i]);
    P.upper[i] = T(m.upper[i]);
    P.rest[i] = T(pc->rest ? pc->rest[i] : m.rest[i]);
  }
  P.w_lim = T(pc->w_limit);
  P.w_rest = T(pc->w_rest);
  // depth levels (joint order is topological: parents come first, robot.py:325-340)
  std::vector<int> depth(nj, 0);
  int maxd = 0;
  for (int j = 0; j < nj; ++j) {
    const int p = P.parent_joint[j];
    depth[j] = p >= 0 ? depth[p] + 1 : 0;
    if (depth[j] > maxd) maxd = depth[j];
  }
  P.nlev = nj ? maxd + 1 : 0;
  int at = 0;
  for (int d = 0; d < P.nlev; ++d) {
    P.lev_start[d] = at;
    for (int j = 0; j < nj; ++j)
      if (depth[j] == d) P.lev_joint[at++] = (int8_t)j;
  }
  P.lev_start[P.nlev] = at;
  for (int j = 0; j < nj; ++j) {
    if (P.kind[j] == 0 || P.qcol[j] < 0) continue;
    const int c = P.qcol[j];
    P.col_joint[c][P.col_nj[c]++] = (int8_t)j;  // bounded by tree_params_ok
  }
  return P;
}

// shape limits of the tree kernel beyond the joint / dof counts
bool tree_params_ok(const KopModel& m) {
  int per[kTreeMaxDofs] = {0};
  for (int j = 0; j < m.tree.nj; ++j) {
    if (m.tree.kind[j] == 0 || m.tree.qcol[j] < 0) continue;
    if (++per[m.tree.qcol[j]] > kTreeMaxPerCol) return false;
  }
  return true;
}

}  // namespace

extern "C" {

int kop_multi_pose_solve(const KopModel* m, const KopPoseCosts* pc, const KopLmOptions* o, const double* targets,
                         const double* q0, int64_t batch, double* q_out, double* cost_out, double* init_cost_out,
                         double* history_out, int32_t* iterations_out, int32_t* termination_out, void* stream) {
  return kop_multi_pose_solve_base(m, pc, o, KOP_BASE_NONE, targets, q0, nullptr, batch, q_out, nullptr, cost_out,
                                   init_cost_out, history_out, iterations_out, termination_out, stream);
}

int kop_multi_pose_solve_base(const KopModel* m, const KopPoseCosts* pc, const KopLmOptions* o, int32_t base_kind,
                              const double* targets, const double* q0, const double* base0, int64_t batch,
                              double* q_out, double* base_out, double* cost_out, double* init_cost_out,
                              double* history_out, int32_t* iterations_out, int32_t* termination_out, void* stream) {
  if (!m || !pc || !o) return fail(KOP_EINVAL, "null argument");
  if (base_kind < KOP_BASE_NONE || base_kind > KOP_BASE_SE3) return fail(KOP_EINVAL, "bad base kind");
  if (m->tree.n + base_dim(base_kind) > kTreeMaxDofs)
    return fail(KOP_EUNSUPPORTED, "actuated joints plus base tangent dimensions exceed 32");
  if (base_kind != KOP_BASE_NONE && batch > 0 && (!base0 || !base_out))
    return fail(KOP_EINVAL, "a base variable needs base0 and base_out");
  if (o->precision != KOP_FP32 && o->precision != KOP_FP64) return fail(KOP_EINVAL, "bad precision");
  if (m->tree.n > kTreeMaxDofs || m->tree.nj > kTreeMaxJoints || !tree_params_ok(*m))
    return fail(KOP_EUNSUPPORTED, "tree solve supports up to 32 actuated and 64 total joints");
  if (pc->num_poses < 1 || pc->num_poses > kTreeMaxPoses)
    return fail(KOP_EUNSUPPORTED, "tree solve supports 1..8 pose costs");
  for (int e = 0; e < pc->num_poses; ++e)
    if (pc->links[e] < 0 || pc->links[e] >= m->tree.nl) return fail(KOP_EINVAL, "unknown link index");
  if (o->max_iterations <= 0 || !(o->initial_damping > 0)) return fail(KOP_EINVAL, "max_iterations and initial_damping must be positive");
  if (!(o->damping_increase > 1.0)) return fail(KOP_EINVAL, "damping_increase must exceed 1");
  if (!(o->damping_decrease > 0.0 && o->damping_decrease < 1.0)) return fail(KOP_EINVAL, "damping_decrease must be in (0, 1)");
  if (o->max_rejections < 0) return fail(KOP_EINVAL, "max_rejections must be nonnegative");
  if (batch < 0) return fail(KOP_EINVAL, "negative batch");
  if (batch == 0) return KOP_OK;
  if (!targets || !q0 || !q_out || !cost_out || !init_cost_out || !iterations_out || !termination_out)
    return fail(KOP_EINVAL, "null array argument");
  TreeLaunch L;
  L.targets = targets;
  L.q0 = q0;
  L.B = batch;
  L.opts = {o->max_iterations, o->max_rejections, o->initial_damping, o->damping_increase, o->damping_decrease,
            o->gradient_tolerance, o->step_tolerance};
  L.q_out = q_out;
  L.cost_out = cost_out;
  L.init_cost = init_cost_out;
  L.hist_out = history_out;
  L.iters = iterations_out;
  L.term = termination_out;
  L.base0 = base0;
  L.base_out = base_out;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (o->precision == KOP_FP32) {
    TreeLmParams<float> P = tree_params<float>(*m, pc);
    P.base_kind = base_kind;
    e = launch_tree_solve<float>(P, L, st);
  } else {
    TreeLmParams<double> P = tree_params<double>(*m, pc);
    P.base_kind = base_kind;
    e = launch_tree_solve<double>(P, L, st);
  }
  return cuda_status(e);
}

}  // extern "C"

namespace {

// plan_trajectory's weights and stencils (tasks.py:347-403, costs.py:198-341)
template <class G>
TrajCosts<typename G::T> make_traj_costs(const KopModel& m, const KopTrajCosts* c) {
  using T = typename G::T;
  TrajCosts<T> W;
  memset(&W, 0, sizeof(W));
  const int n = m.tree.n;
  W.T_steps = c->timesteps;
  W.n = n;
  for (int i = 0; i < 8; ++i) {
    W.lower[i] = i < n ? T(m.lower[i]) : T(-INFINITY);
    W.upper[i] = i < n ? T(m.upper[i]) : T(INFINITY);
    W.rest[i] = i < n ? T(c->rest ? c->rest[i] : m.rest[i]) : T(0);
    W.vbudget[i] = (i < n && c->velocity_limits) ? T(c->velocity_limits[i] * c->dt) : T(INFINITY);
  }
  W.w_lim = T(c->w_limit);
  W.w_rest = T(c->w_rest);
  W.anchor = T(c->w_anchor);
  W.w_smooth = T(c->w_smoothness);
  W.w_vel = T(c->w_velocity);
  W.w_acc = T(c->w_acceleration);
  W.w_jerk = T(c->w_jerk);
  const double acc[5] = {-1.0, 16.0, -30.0, 16.0, -1.0}, jerk[5] = {-1.0, 2.0, 0.0, -2.0, 1.0};
  const double dt2 = c->dt * c->dt, dt3 = c->dt * c->dt * c->dt;
  for (int k = 0; k < 5; ++k) {
    W.acc_c[k] = T((acc[k] / 12.0) / dt2);
    W.jerk_c[k] = T((jerk[k] / 2.0) / dt3);
  }
  W.w_world = T(c->w_world);
  W.eta_world = T(c->eta_world > 0 ? c->eta_world : 1.0);
  return W;
}

template <class G>
cudaError_t run_traj(const KopModel& m, const ChainParams<double, kChainMax>& D, const CollisionParams<double>& PD,
                     const KopTrajCosts* c, const TrajLaunch& L, cudaStream_t st) {
  return launch_traj<G>(cast_chain<typename G::T, G::K>(D), cast_collision<typename G::T>(PD),
                        make_traj_costs<G>(m, c), L, st);
}

template <class G>
cudaError_t run_traj_normal(const KopModel& m, const ChainParams<double, kChainMax>& D,
                            const CollisionParams<double>& PD, const KopTrajCosts* c, const TrajLaunch& L,
                            cudaStream_t st) {
  return launch_traj_normal<G>(cast_chain<typename G::T, G::K>(D), cast_collision<typename G::T>(PD),
                               make_traj_costs<G>(m, c), L, st);
}

template <typename T>
cudaError_t dispatch_traj(Shape sh, const KopModel& m, const ChainParams<double, kChainMax>& D,
                          const CollisionParams<double>& PD, const KopTrajCosts* c, const TrajLaunch& L,
                          cudaStream_t st, bool normal = false) {
  switch (sh) {
    case Shape::kId7:
      return normal ? run_traj_normal<Cfg<T, 7, 7, true, false>>(m, D, PD, c, L, st)
                    : run_traj<Cfg<T, 7, 7, true, false>>(m, D, PD, c, L, st);
    case Shape::kGen8:
      return normal ? run_traj_normal<Cfg<T, 8, 8, false, false>>(m, D, PD, c, L, st)
                    : run_traj<Cfg<T, 8, 8, false, false>>(m, D, PD, c, L, st);
    default: return cudaErrorInvalidValue;
  }
}

int prepare_traj(const KopModel* m, int link, const KopTrajCosts* c, int precision, int num_obstacles,
                 ChainParams<double, kChainMax>& C, CollisionParams<double>& PD, Shape& sh) {
  if (!m || !c) return fail(KOP_EINVAL, "null argument");
  // TrajRequest.__post_init__ (tasks.py:208-213)
  if (c->timesteps < 5) return fail(KOP_EINVAL, "trajectory needs at least 5 timesteps for the stencils");
  if (c->timesteps > kTrajMaxSteps) return fail(KOP_EUNSUPPORTED, "more than 64 timesteps (not compiled in)");
  if (!(c->dt > 0)) return fail(KOP_EINVAL, "dt must be positive");
  const double ws[] = {c->w_anchor, c->w_smoothness, c->w_velocity, c->w_acceleration, c->w_jerk,
                       c->w_limit,  c->w_rest,       c->w_self,     c->w_world};
  for (double w : ws)
    if (!(w >= 0)) return fail(KOP_EINVAL, "weights must be nonnegative");
  if (num_obstacles < 0 || num_obstacles > kMaxObstacles)
    return fail(KOP_EUNSUPPORTED, "more than 16 obstacles (not compiled in)");
  KopCollisionCosts cc{};
  cc.w_self = c->w_self;
  cc.eta_self = c->eta_self;
  cc.w_world = c->w_world;
  cc.eta_world = c->eta_world;
  cc.sharpness = c->sharpness;
  cc.hard_min = c->hard_min;
  cc.num_obstacles = 0;  // per-problem obstacles travel separately
  return prepare_col(m, link, precision, &cc, C, PD, sh);
}

}  // namespace

extern "C" {

int kop_traj_solve(const KopModel* m, int32_t link, const KopTrajCosts* c, const KopLmOptions* o,
                   const double* q_init, const double* anchors, const double* obstacles, int32_t num_obstacles,
                   int64_t batch, double* q_out, double* cost_out, double* init_cost_out, double* history_out,
                   int32_t* iterations_out, int32_t* termination_out, void* stream) {
  if (!o) return fail(KOP_EINVAL, "null argument");
  ChainParams<double, kChainMax> C;
  CollisionParams<double> PD;
  Shape sh;
  int rc = prepare_traj(m, link, c, o->precision, num_obstacles, C, PD, sh);
  if (rc != KOP_OK) return rc;
  if (o->max_iterations <= 0 || !(o->initial_damping > 0)) return fail(KOP_EINVAL, "max_iterations and initial_damping must be positive");
  if (!(o->damping_increase > 1.0)) return fail(KOP_EINVAL, "damping_increase must exceed 1");
  if (!(o->damping_decrease > 0.0 && o->damping_decrease < 1.0)) return fail(KOP_EINVAL, "damping_decrease must be in (0, 1)");
  if (o->max_rejections < 0) return fail(KOP_EINVAL, "max_rejections must be nonnegative");
  if (batch < 0) return fail(KOP_EINVAL, "negative batch");
  if (batch == 0) return KOP_OK;
  if (!anchors || (num_obstacles > 0 && !obstacles) || !q_out || !cost_out || !init_cost_out ||
      !iterations_out || !termination_out)
    return fail(KOP_EINVAL, "null array argument");
  TrajLaunch L{};
  L.q_init = q_init;
  L.anchors = anchors;
  L.obstacles = obstacles;
  L.n_obs = c->w_world > 0 ? num_obstacles : 0;
  L.B = batch;
  L.opts = {o->max_iterations, o->max_rejections, o->initial_damping, o->damping_increase, o->damping_decrease,
            o->gradient_tolerance, o->step_tolerance};
  L.q_out = q_out;
  L.cost_out = cost_out;
  L.init_cost = init_cost_out;
  L.hist_out = history_out;
  L.iters = iterations_out;
  L.term = termination_out;
  cudaStream_t st = (cudaStream_t)stream;
  const cudaError_t e = o->precision == KOP_FP32 ? dispatch_traj<float>(sh, *m, C, PD, c, L, st)
                                                 : dispatch_traj<double>(sh, *m, C, PD, c, L, st);
  return cuda_status(e);
}

int kop_traj_normal_equations(const KopModel* m, int32_t link, const KopTrajCosts* c, int32_t precision,
                              const double* qs, const double* anchors, const double* obstacles,
                              int32_t num_obstacles, int64_t batch, double* cost_out, double* grad_out,
                              double* hess_out, void* stream) {
  ChainParams<double, kChainMax> C;
  CollisionParams<double> PD;
  Shape sh;
  int rc = prepare_traj(m, link, c, precision, num_obstacles, C, PD, sh);
  if (rc != KOP_OK) return rc;
  if (precision != KOP_FP32 && precision != KOP_FP64) return fail(KOP_EINVAL, "bad precision");
  if (batch < 0) return fail(KOP_EINVAL, "negative batch");
  if (batch == 0) return KOP_OK;
  if (!qs || !anchors || (num_obstacles > 0 && !obstacles) || !cost_out || !grad_out || !hess_out)
    return fail(KOP_EINVAL, "null array argument");
  const int64_t nr = (int64_t)c->timesteps * m->tree.n;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(hess_out, 0, sizeof(double) * batch * nr * nr, st);
  if (e != cudaSuccess) return cuda_status(e);
  TrajLaunch L{};
  L.q_init = qs;
  L.anchors = anchors;
  L.obstacles = obstacles;
  L.n_obs = c->w_world > 0 ? num_obstacles : 0;
  L.B = batch;
  L.cost_out = cost_out;
  L.grad_out = grad_out;
  L.hess_out = hess_out;
  e = precision == KOP_FP32 ? dispatch_traj<float>(sh, *m, C, PD, c, L, st, true)
                            : dispatch_traj<double>(sh, *m, C, PD, c, L, st, true);
  return cuda_status(e);
}

int kop_traj_report(const KopModel* m, int32_t link, int32_t timesteps, const double* qs, const double* obstacles,
                    int32_t num_obstacles, const double* targets, int64_t batch, double* static_out,
                    double* swept_out, double* min_static, double* min_swept, double* pos_err, double* rot_err,
                    void* stream) {
  if (timesteps < 1) return fail(KOP_EINVAL, "need at least one timestep");
  if (timesteps > kTrajMaxSteps) return fail(KOP_EUNSUPPORTED, "more than 64 timesteps (not compiled in)");
  if (num_obstacles < 0 || num_obstacles > kMaxObstacles)
    return fail(KOP_EUNSUPPORTED, "more than 16 obstacles (not compiled in)");
  if (batch < 0) return fail(KOP_EINVAL, "negative batch");
  KopCollisionCosts cc{};
  ChainParams<double, kChainMax> C;
  CollisionParams<double> PD;
  Shape sh;
  int rc = prepare_col(m, link, KOP_FP64, &cc, C, PD, sh);
  if (rc != KOP_OK) return rc;
  if (batch == 0) return KOP_OK;
  if (!qs || (num_obstacles > 0 && !obstacles) || (targets && (!pos_err || !rot_err)))
    return fail(KOP_EINVAL, "null array argument");
  TrajReportLaunch L{};
  L.steps = timesteps;
  L.n = m->tree.n;
  L.qs = qs;
  L.obstacles = obstacles;
  L.n_obs = num_obstacles;
  L.targets = targets;
  L.B = batch;
  L.static_out = static_out;
  L.swept_out = swept_out;
  L.min_static = min_static;
  L.min_swept = min_swept;
  L.pos_err = pos_err;
  L.rot_err = rot_err;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  if (sh == Shape::kId7)
    e = launch_traj_report<Cfg<double, 7, 7, true, false>>(cast_chain<double, 7>(C), PD, L, st);
  else
    e = launch_traj_report<Cfg<double, 8, 8, false, false>>(cast_chain<double, 8>(C), PD, L, st);
  return cuda_status(e);
}

int64_t kop_multi_pose_beam_workspace_bytes(const KopModel* m, const KopPoseCosts* pc, const KopIkParams* p,
                                             int64_t batch) {
  if (!m || !pc || !p || batch < 0) return fail(KOP_EINVAL, "invalid arguments");
  const int rec = tree_beam_rec(m->tree.n, p->prune_after);
  const int64_t elem = p->precision == KOP_FP64 ? 8 : 4;  // stage-1 records are stored in the solve precision
  return ((int64_t)batch * p->seeds * rec * elem + 255) / 256 * 256 + (int64_t)batch * p->keep * 4 + 256;
}

int kop_multi_pose_beam(const KopModel* m, const KopPoseCosts* pc, const KopIkParams* p, const double* targets,
                        int64_t batch, const double* seeds, void* workspace, int64_t workspace_bytes, double* q_out,
                        double* cost_out, double* history_out, double* pos_err, double* rot_err, uint8_t* success,
                        void* stream) {
  if (!m || !pc || !p) return fail(KOP_EINVAL, "null argument");
  if (p->precision != KOP_FP32 && p->precision != KOP_FP64) return fail(KOP_EINVAL, "bad precision");
  if (m->tree.n > kTreeMaxDofs || m->tree.nj > kTreeMaxJoints || !tree_params_ok(*m))
    return fail(KOP_EUNSUPPORTED, "tree IK-Beam supports up to 32 actuated and 64 total joints");
  if (pc->num_poses < 1 || pc->num_poses > kTreeMaxPoses)
    return fail(KOP_EUNSUPPORTED, "tree IK-Beam supports 1..8 end effectors");
  for (int e = 0; e < pc->num_poses; ++e)
    if (pc->links[e] < 0 || pc->links[e] >= m->tree.nl) return fail(KOP_EINVAL, "unknown link index");
  // IkRequest.__post_init__ (tasks.py:56-60)
  if (!(0 < p->prune_after && p->prune_after < p->total_steps))
    return fail(KOP_EINVAL, "need 0 < prune_after < total_steps");
  if (!(1 <= p->keep && p->keep <= p->seeds)) return fail(KOP_EINVAL, "need 1 <= keep <= seeds");
  if (p->keep > 8 || p->prune_after > 31 || p->total_steps - p->prune_after > 32)
    return fail(KOP_EUNSUPPORTED, "tree IK-Beam compiled for keep <= 8 and <= 31 + 32 steps");
  if (batch < 0) return fail(KOP_EINVAL, "negative batch");
  if (batch == 0) return KOP_OK;
  if (!targets || !seeds || !workspace || !q_out || !cost_out || !pos_err || !rot_err || !success)
    return fail(KOP_EINVAL, "null array argument");
  if (workspace_bytes < kop_multi_pose_beam_workspace_bytes(m, pc, p, batch))
    return fail(KOP_EINVAL, "workspace too small");
  TreeBeamLaunch L{};
  L.targets = targets;
  L.B = batch;
  L.seeds = seeds;
  L.S = p->seeds;
  L.steps1 = p->prune_after;
  L.steps2 = p->total_steps - p->prune_after;
  L.keep = p->keep;
  L.pos_tol = p->success_pos_tol;
  L.rot_tol = p->success_rot_tol;
  L.workspace = workspace;
  L.q_out = q_out;
  L.cost_out = cost_out;
  L.hist_out = history_out;
  L.pos_err = pos_err;
  L.rot_err = rot_err;
  L.success = success;
  cudaStream_t st = (cudaStream_t)stream;
  const TreeLmParams<double> Pd = tree_params<double>(*m, pc, false);  // FP64 pose errors: the joint-by-joint walk
  const cudaError_t e = p->precision == KOP_FP32 ? launch_tree_beam<float>(tree_params<float>(*m, pc), Pd, L, st)
                                                 : launch_tree_beam<double>(tree_params<double>(*m, pc), Pd, L, st);
  return cuda_status(e);
}

int kop_dfma_peak_kernel(int32_t blocks, int32_t threads, int32_t iters, double* sink, double* flops,
                         void* stream) {
  if (blocks <= 0 || threads <= 0 || iters <= 0 || !sink) return fail(KOP_EINVAL, "invalid arguments");
  if (flops) *flops = 2.0 * 8.0 * (double)blocks * threads * (double)iters;
  return cuda_status(launch_dfma_peak(blocks, threads, iters, sink, (cudaStream_t)stream));
}

namespace {
LinkMap link_map(const KopModel& m) {
  LinkMap L;
  for (int l = 0; l < kMaxLinks; ++l) L.pj[l] = l < (int)m.parent_joint.size() ? m.parent_joint[l] : -1;
  return L;
}

// sphere-bearing links in model order (spheres arrive grouped by link)
std::vector<int> sphere_links(const KopModel& m) {
  std::vector<int> links;
  for (int l : m.sphere_link)
    if (links.empty() || links.back() != l) links.push_back(l);
  return links;
}
}  // namespace

int kop_term_pose(const KopModel* m, int32_t link, const double* target, int32_t base_kind, const double* q,
                  const double* base, int64_t count, double* r, double* jq, double* jb, void* stream) {
  if (!m || !target || count < 0) return fail(KOP_EINVAL, "invalid arguments");
  if (link < 0 || link >= m->tree.nl) return fail(KOP_EINVAL, "unknown link index");
  if (base_kind < KOP_BASE_NONE || base_kind > KOP_BASE_SE3) return fail(KOP_EINVAL, "bad base kind");
  if (count == 0) return KOP_OK;
  if (!q || !r || (base_kind != KOP_BASE_NONE && !base)) return fail(KOP_EINVAL, "null array argument");
  TermPose T{};
  double tv[7];
  HQ tq{target[0], -target[1], -target[2], -target[3]};  // Transform3.inverse, canonical (liegroups.py:388-390)
  const double nq = sqrt(tq.w * tq.w + tq.x * tq.x + tq.y * tq.y + tq.z * tq.z);
  tq = {tq.w / nq, tq.x / nq, tq.y / nq, tq.z / nq};
  if (tq.w < 0.0) tq = {-tq.w, -tq.x, -tq.y, -tq.z};
  double t[3];
  hrot(tq, target + 4, t);
  tv[0] = tq.w; tv[1] = tq.x; tv[2] = tq.y; tv[3] = tq.z;
  tv[4] = -t[0]; tv[5] = -t[1]; tv[6] = -t[2];
  memcpy(T.tinv, tv, sizeof(tv));
  T.base_kind = base_kind;
  return cuda_status(launch_term_pose(m->tree, link_map(*m), link, T, q, base, count, r, jq, jb,
                                      (cudaStream_t)stream));
}

int kop_term_joint(const KopModel* m, int32_t kind, const double* rest, const double* velocity_limits, double dt,
                   const double* coeffs, const double* qs, int64_t count, double* r, double* jdiag, void* stream) {
  if (!m || count < 0) return fail(KOP_EINVAL, "invalid arguments");
  TermJoint T{};
  T.kind = kind;
  const int n = m->tree.n;
  switch (kind) {
    case KOP_TERM_LIMIT: T.nvars = 1; break;
    case KOP_TERM_REST:
      if (!rest) return fail(KOP_EINVAL, "rest cost needs q_rest");
      T.nvars = 1;
      break;
    case KOP_TERM_SMOOTHNESS: T.nvars = 2; break;
    case KOP_TERM_VELOCITY:
      if (!(dt > 0.0)) return fail(KOP_EINVAL, "dt must be positive");
      if (!velocity_limits) return fail(KOP_EINVAL, "velocity cost needs the velocity limits");
      T.nvars = 2;
      break;
    case KOP_TERM_STENCIL:
      if (!coeffs) return fail(KOP_EINVAL, "stencil needs coefficients");
      T.nvars = 5;
      break;
    default: return fail(KOP_EINVAL, "unknown joint-space term kind");
  }
  for (int i = 0; i < n; ++i) {
    T.lower[i] = m->lower[i];
    T.upper[i] = m->upper[i];
    T.rest[i] = rest ? rest[i] : 0.0;
    T.vlim[i] = velocity_limits ? velocity_limits[i] : INFINITY;
  }
  T.dt = dt;
  for (int k = 0; k < 5; ++k) T.coeffs[k] = coeffs ? coeffs[k] : 0.0;
  if (count == 0) return KOP_OK;
  if (!qs || !r) return fail(KOP_EINVAL, "null array argument");
  return cuda_status(launch_term_joint(T, n, qs, count, r, jdiag, (cudaStream_t)stream));
}

int kop_term_manipulability(const KopModel* m, int32_t link, double eps, const double* q, int64_t count,
                            double* r, double* jrow, double* jac, double* djac, void* stream) {
  if (!m || count < 0) return fail(KOP_EINVAL, "invalid arguments");
  if (link < 0 || link >= m->tree.nl) return fail(KOP_EINVAL, "unknown link index");
  if (m->tree.n > kTreeMaxDofsTerms) return fail(KOP_EUNSUPPORTED, "manipulability supports <= 32 actuated joints");
  if (count == 0) return KOP_OK;
  if (!q) return fail(KOP_EINVAL, "null array argument");
  return cuda_status(launch_term_manip(m->tree, link_map(*m), link, eps, q, count, r, jrow, jac, djac,
                                       (cudaStream_t)stream));
}

int kop_term_rows(const KopModel* m, int32_t kind, int32_t num_obstacles) {
  if (!m) return fail(KOP_EINVAL, "null model");
  if (kind == KOP_TERM_SELF) return (int)(m->pair_links.size() / 2);
  if (kind == KOP_TERM_WORLD || kind == KOP_TERM_SWEPT) return (int)sphere_links(*m).size() * num_obstacles;
  return fail(KOP_EINVAL, "not a collision term kind");
}

int kop_term_collision(const KopModel* m, int32_t kind, const KopObstacle* obstacles, int32_t num_obstacles,
                       double eta, double sharpness, int32_t hard_min, const double* q0, const double* q1,
                       int64_t count, double* r, double* j0, double* j1, void* stream) {
  if (!m || count < 0) return fail(KOP_EINVAL, "invalid arguments");
  if (kind != KOP_TERM_WORLD && kind != KOP_TERM_SELF && kind != KOP_TERM_SWEPT)
    return fail(KOP_EINVAL, "not a collision term kind");
  if (!(eta > 0.0)) return fail(KOP_EINVAL, "buffer distance must be positive");
  if (kind != KOP_TERM_SELF && (num_obstacles < 1 || !obstacles))
    return fail(KOP_EINVAL, "no (link, obstacle) pairs: empty world");
  if (num_obstacles > kMaxObstacles) return fail(KOP_EUNSUPPORTED, "more than 16 obstacles (not compiled in)");
  const std::vector<int> links = sphere_links(*m);
  if ((int)m->sphere_link.size() > kMaxSpheres || (int)links.size() > kMaxSphereLinks ||
      (int)m->pair_links.size() / 2 > kMaxSelfPairs)
    return fail(KOP_EUNSUPPORTED, "more than 32 spheres / 16 sphere links / 64 self pairs (not compiled in)");
  TermGeom G{};
  G.ns = (int)m->sphere_link.size();
  for (int s = 0; s < G.ns; ++s) {
    G.s_link[s] = m->sphere_link[s];
    for (int i = 0; i < 3; ++i) G.s_c[s][i] = m->sphere_center[3 * s + i];
    G.s_r[s] = m->sphere_radius[s];
  }
  G.nl = (int)links.size();
  for (int i = 0; i < G.nl; ++i) G.links[i] = links[i];
  G.np = (int)m->pair_links.size() / 2;
  for (int p = 0; p < G.np; ++p) {
    G.pa[p] = m->pair_links[2 * p];
    G.pb[p] = m->pair_links[2 * p + 1];
  }
  if (kind == KOP_TERM_SELF && G.np == 0) return fail(KOP_EINVAL, "model declares no self-collision pairs");
  G.O.no = kind == KOP_TERM_SELF ? 0 : num_obstacles;
  for (int o = 0; o < G.O.no; ++o) {
    const KopObstacle& ob = obstacles[o];
    if (ob.kind < 0 || ob.kind > 2) return fail(KOP_EINVAL, "unknown obstacle kind");
    G.O.okind[o] = ob.kind;
    double nrm = 1.0;
    if (ob.kind == KOP_OBSTACLE_HALFSPACE) {
      nrm = sqrt(ob.a[0] * ob.a[0] + ob.a[1] * ob.a[1] + ob.a[2] * ob.a[2]);
      if (nrm < 1e-12) return fail(KOP_EINVAL, "half-space normal must be nonzero");
    }
    for (int i = 0; i < 3; ++i) {
      G.O.oa[o][i] = ob.a[i] / nrm;
      G.O.ob[o][i] = ob.b[i];
    }
    G.O.orad[o] = ob.radius;
  }
  G.eta = eta;
  G.beta = sharpness > 0.0 ? sharpness : 100.0;
  G.hard = hard_min;
  if (count == 0) return KOP_OK;
  if (!q0 || !r || (kind == KOP_TERM_SWEPT && !q1)) return fail(KOP_EINVAL, "null array argument");
  return cuda_status(launch_term_collision(m->tree, link_map(*m), G, kind, q0, q1, count, r, j0,
                                           kind == KOP_TERM_SWEPT ? j1 : nullptr, (cudaStream_t)stream));
}

int kop_check_probe(uint32_t* out, int32_t words, void* stream) {
  if (!out || words <= 0 || words > 12 * 1024) return fail(KOP_EINVAL, "invalid arguments");
  return cuda_status(launch_check_probe(out, words, (cudaStream_t)stream));
}

int kop_fma_peak_kernel(int32_t blocks, int32_t threads, int32_t iters, float* sink, double* flops,
                        void* stream) {
  if (blocks <= 0 || threads <= 0 || iters <= 0 || !sink) return fail(KOP_EINVAL, "invalid arguments");
  if (flops) *flops = 2.0 * 16.0 * (double)blocks * threads * (double)iters;
  return cuda_status(launch_fma_peak(blocks, threads, iters, sink, (cudaStream_t)stream));
}

}  // extern "C"

// ---------------------------------------------------------------------------
// IK-Beam with host buffers end to end (the binding a NumPy caller uses)
// ---------------------------------------------------------------------------
namespace {

// Per host thread and device: grow-only device buffers and streams of the
// host pipeline.  Buffer set i is only ever used on stream i, so successive
// calls are ordered by the streams themselves.
struct HostPipe {
  int device = -1;
  int nstreams = 0;
  int64_t chunk = 0, ws_bytes = 0, seeds_len = 0;
  cudaStream_t st[8] = {};
  cudaEvent_t done[8] = {};
  void* buf[8] = {};
  // pinned staging of one buffer set's host side (pageable callers), allocated on first use
  void* stage[8] = {};
  cudaEvent_t chunk_done[8] = {};
  size_t stage_bytes = 0;
  double* seeds = nullptr;
  ~HostPipe() { release(); }
  void release() {
    for (int i = 0; i < 8; ++i) {
      if (buf[i]) cudaFree(buf[i]);
      if (stage[i]) cudaFreeHost(stage[i]);
      if (st[i]) cudaStreamDestroy(st[i]);
      if (done[i]) cudaEventDestroy(done[i]);
      if (chunk_done[i]) cudaEventDestroy(chunk_done[i]);
      buf[i] = nullptr;
      stage[i] = nullptr;
      st[i] = nullptr;
      done[i] = nullptr;
      chunk_done[i] = nullptr;
    }
    stage_bytes = 0;
    if (seeds) cudaFree(seeds);
    seeds = nullptr;
    nstreams = 0;
    chunk = ws_bytes = seeds_len = 0;
  }
};
thread_local HostPipe g_pipe;

struct ChunkLayout {  // byte offsets of one buffer set
  size_t tg, q, base, cost, hist, pe, re, ok, ws, total;
};
ChunkLayout chunk_layout(int64_t chunk, int n, int hist_len, int64_t ws_bytes) {
  auto al = [](size_t v) { return (v + 255) / 256 * 256; };
  ChunkLayout L{};
  size_t at = 0;
  L.tg = at; at = al(at + sizeof(double) * 7 * chunk);
  L.q = at; at = al(at + sizeof(double) * n * chunk);
  L.base = at; at = al(at + sizeof(double) * 3 * chunk);
  L.cost = at; at = al(at + sizeof(double) * chunk);
  L.hist = at; at = al(at + sizeof(double) * hist_len * chunk);
  L.pe = at; at = al(at + sizeof(double) * chunk);
  L.re = at; at = al(at + sizeof(double) * chunk);
  L.ok = at; at = al(at + chunk);
  L.ws = at; at = al(at + (size_t)ws_bytes);
  L.total = at;
  return L;
}

}  // namespace

extern "C" {

int kop_ik_beam_host(const KopModel* m, int32_t link, const KopIkParams* p, const double* targets, int64_t batch,
                     const double* seeds, double* q_out, double* base_out, double* cost_out, double* history_out,
                     double* pos_err, double* rot_err, uint8_t* success, int64_t chunk, int32_t n_streams,
                     void* stream) {
  if (!m || !p) return fail(KOP_EINVAL, "null argument");
  if (batch < 0) return fail(KOP_EINVAL, "negative batch");
  if (n_streams < 0 || n_streams > 8) return fail(KOP_EINVAL, "n_streams must be in 0..8");
  if (chunk < 0) return fail(KOP_EINVAL, "negative chunk");
  // validates the request (and the shape) without touching the device
  const int64_t ws1 = kop_ik_beam_workspace_bytes(m, link, p, 1);
  if (ws1 < 0) return (int)ws1;
  if (batch == 0) return KOP_OK;
  if (!targets || !seeds || !q_out || !cost_out || !pos_err || !rot_err || !success)
    return fail(KOP_EINVAL, "null array argument");
  const int n = m->tree.n, hist_len = p->total_steps + 1;
  if (hist_len > 64 || n > 8) return fail(KOP_EUNSUPPORTED, "host pipeline compiled for <= 63 steps, <= 8 joints");
  // defaults from a chunk x stream sweep at 1M targets (tools/e2e_host_sweep.py): 16K-target chunks over
  // 8 streams overlap the small kernels' tails and the copies best (31.9M vs 30.5M solves/s at 64K x 4)
  const int ns = n_streams ? n_streams : 8;
  const int64_t ck = chunk ? (chunk < batch ? chunk : batch) : (batch < 16384 ? batch : 16384);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e);
  HostPipe& P = g_pipe;
  const int64_t ws = kop_ik_beam_workspace_bytes(m, link, p, ck);
  if (P.device != dev || P.nstreams < ns || P.chunk < ck || P.ws_bytes < ws) {
    const int64_t keep_chunk = P.device == dev && P.chunk > ck ? P.chunk : ck;
    const int64_t keep_ws = P.device == dev && P.ws_bytes > ws ? P.ws_bytes : ws;
    const int keep_ns = P.device == dev && P.nstreams > ns ? P.nstreams : ns;
    if (P.device >= 0) cudaDeviceSynchronize();
    P.release();
    P.device = dev;
    P.chunk = keep_chunk;
    P.ws_bytes = keep_ws;
    P.nstreams = keep_ns;
    const ChunkLayout Lk = chunk_layout(P.chunk, 8, 64, P.ws_bytes);
    for (int i = 0; i < P.nstreams; ++i) {
      if ((e = cudaStreamCreateWithFlags(&P.st[i], cudaStreamNonBlocking)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&P.done[i], cudaEventDisableTiming)) != cudaSuccess ||
          (e = cudaMalloc(&P.buf[i], Lk.total)) != cudaSuccess) {
        P.release();
        P.device = -1;
        return cuda_status(e);
      }
    }
  }
  const ChunkLayout L = chunk_layout(P.chunk, 8, 64, P.ws_bytes);
  const int64_t seeds_len = (int64_t)p->seeds * n;
  if (P.seeds_len < seeds_len) {
    if (P.seeds) cudaFree(P.seeds);
    P.seeds = nullptr;
    if ((e = cudaMalloc(&P.seeds, sizeof(double) * seeds_len)) != cudaSuccess) return cuda_status(e);
    P.seeds_len = seeds_len;
  }
  cudaStream_t caller = (cudaStream_t)stream;
  // seeds: copied on stream 0 after the caller's prior work; the other streams wait for them
  cudaEvent_t start;
  if ((e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming)) != cudaSuccess) return cuda_status(e);
  cudaEventRecord(start, caller);
  cudaStreamWaitEvent(P.st[0], start, 0);
  // the seed buffer is shared by every buffer set: kernels of the previous call may still read it on
  // any pipeline stream, so the overwrite waits for all of them (never-recorded events are no-ops)
  for (int i = 1; i < P.nstreams; ++i) cudaStreamWaitEvent(P.st[0], P.done[i], 0);
  cudaMemcpyAsync(P.seeds, seeds, sizeof(double) * seeds_len, cudaMemcpyHostToDevice, P.st[0]);
  cudaEventRecord(start, P.st[0]);
  for (int i = 1; i < ns; ++i) cudaStreamWaitEvent(P.st[i], start, 0);
  // Pageable (not page-locked) host arrays -- the NumPy drop-in path: copies from pageable memory
  // would serialise the pipeline, so each buffer set gets a pinned host staging area; this thread
  // copies a chunk's targets into it before the H2D and the chunk's results out of it once its D2H
  // completed (when the set comes round again), overlapping those CPU copies with the kernels and
  // copies of the other sets.  The call then returns with the outputs written (synchronous).
  auto pageable = [](const void* ptr) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
      cudaGetLastError();
      return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
  };
  const bool staged = pageable(targets) || pageable(q_out);
  const ChunkLayout H = chunk_layout(P.chunk, 8, 64, 0);
  if (staged && P.stage_bytes < H.total) {
    for (int i = 0; i < P.nstreams; ++i) {
      if (P.stage[i]) cudaFreeHost(P.stage[i]);
      P.stage[i] = nullptr;
    }
    for (int i = 0; i < P.nstreams; ++i) {
      if ((e = cudaHostAlloc(&P.stage[i], H.total, cudaHostAllocDefault)) != cudaSuccess ||
          (!P.chunk_done[i] && (e = cudaEventCreateWithFlags(&P.chunk_done[i], cudaEventDisableTiming)) != cudaSuccess)) {
        cudaEventDestroy(start);
        return cuda_status(e);
      }
    }
    P.stage_bytes = H.total;
  }
  // results of the chunk staged in set i -> the caller's arrays, on a helper thread per in-flight set
  // (it waits for the chunk's D2H, then copies; first-touch page faults of fresh NumPy outputs make
  // these copies the slow part, so several run at once, overlapped with the GPU work)
  std::future<void> drains[8];
  auto drain_async = [&](int i, int64_t lo, int64_t cnt) {
    const char* h = static_cast<const char*>(P.stage[i]);
    cudaEvent_t ev = P.chunk_done[i];
    const bool with_base = base_out && p->optimize_base;
    drains[i] = std::async(std::launch::async, [=]() {
      cudaEventSynchronize(ev);
      memcpy(q_out + lo * n, h + H.q, sizeof(double) * n * cnt);
      if (with_base) memcpy(base_out + lo * 3, h + H.base, sizeof(double) * 3 * cnt);
      memcpy(cost_out + lo, h + H.cost, sizeof(double) * cnt);
      if (history_out) memcpy(history_out + lo * hist_len, h + H.hist, sizeof(double) * hist_len * cnt);
      memcpy(pos_err + lo, h + H.pe, sizeof(double) * cnt);
      memcpy(rot_err + lo, h + H.re, sizeof(double) * cnt);
      memcpy(success + lo, h + H.ok, cnt);
    });
  };
  auto drain = [&](int i) {  // set i's previous results copied out: its staging area is free again
    if (drains[i].valid()) drains[i].get();
  };
  int rc = KOP_OK;
  for (int64_t lo = 0, c = 0; lo < batch && rc == KOP_OK; lo += ck, ++c) {
    const int64_t cnt = (batch - lo) < ck ? (batch - lo) : ck;
    const int i = (int)(c % ns);
    cudaStream_t s = P.st[i];
    char* b = static_cast<char*>(P.buf[i]);
    if (staged) {
      drain(i);
      char* h = static_cast<char*>(P.stage[i]);
      memcpy(h + H.tg, targets + lo * 7, sizeof(double) * 7 * cnt);
      double* dtg = reinterpret_cast<double*>(b + L.tg);
      cudaMemcpyAsync(dtg, h + H.tg, sizeof(double) * 7 * cnt, cudaMemcpyHostToDevice, s);
      rc = kop_ik_beam_stage(m, link, p, 3, dtg, cnt, P.seeds, b + L.ws, P.ws_bytes,
                             reinterpret_cast<double*>(b + L.q),
                             p->optimize_base ? reinterpret_cast<double*>(b + L.base) : nullptr,
                             reinterpret_cast<double*>(b + L.cost),
                             history_out ? reinterpret_cast<double*>(b + L.hist) : nullptr,
                             reinterpret_cast<double*>(b + L.pe), reinterpret_cast<double*>(b + L.re),
                             reinterpret_cast<uint8_t*>(b + L.ok), s);
      if (rc != KOP_OK) break;
      cudaMemcpyAsync(h + H.q, b + L.q, sizeof(double) * n * cnt, cudaMemcpyDeviceToHost, s);
      if (base_out && p->optimize_base)
        cudaMemcpyAsync(h + H.base, b + L.base, sizeof(double) * 3 * cnt, cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(h + H.cost, b + L.cost, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s);
      if (history_out)
        cudaMemcpyAsync(h + H.hist, b + L.hist, sizeof(double) * hist_len * cnt, cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(h + H.pe, b + L.pe, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(h + H.re, b + L.re, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(h + H.ok, b + L.ok, cnt, cudaMemcpyDeviceToHost, s);
      cudaEventRecord(P.chunk_done[i], s);
      drain_async(i, lo, cnt);
      continue;
    }
    double* dtg = reinterpret_cast<double*>(b + L.tg);
    double* dq = reinterpret_cast<double*>(b + L.q);
    double* dbase = reinterpret_cast<double*>(b + L.base);
    double* dcost = reinterpret_cast<double*>(b + L.cost);
    double* dhist = reinterpret_cast<double*>(b + L.hist);
    double* dpe = reinterpret_cast<double*>(b + L.pe);
    double* dre = reinterpret_cast<double*>(b + L.re);
    uint8_t* dok = reinterpret_cast<uint8_t*>(b + L.ok);
    cudaMemcpyAsync(dtg, targets + lo * 7, sizeof(double) * 7 * cnt, cudaMemcpyHostToDevice, s);
    rc = kop_ik_beam_stage(m, link, p, 3, dtg, cnt, P.seeds, b + L.ws, P.ws_bytes, dq,
                           p->optimize_base ? dbase : nullptr, dcost, history_out ? dhist : nullptr, dpe, dre, dok, s);
    if (rc != KOP_OK) break;
    cudaMemcpyAsync(q_out + lo * n, dq, sizeof(double) * n * cnt, cudaMemcpyDeviceToHost, s);
    if (base_out && p->optimize_base)
      cudaMemcpyAsync(base_out + lo * 3, dbase, sizeof(double) * 3 * cnt, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(cost_out + lo, dcost, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s);
    if (history_out)
      cudaMemcpyAsync(history_out + lo * hist_len, dhist, sizeof(double) * hist_len * cnt, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(pos_err + lo, dpe, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(rot_err + lo, dre, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(success + lo, dok, cnt, cudaMemcpyDeviceToHost, s);
  }
  if (staged)
    for (int i = 0; i < ns; ++i) drain(i);
  // join: the caller's stream waits for every pipeline stream
  for (int i = 0; i < ns; ++i) {
    cudaEventRecord(P.done[i], P.st[i]);
    cudaStreamWaitEvent(caller, P.done[i], 0);
  }
  cudaEventDestroy(start);
  if (rc != KOP_OK) return rc;
  return cuda_status(cudaGetLastError());
}

}  // extern "C"
