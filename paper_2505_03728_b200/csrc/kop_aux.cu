// Non-hot-path kernels: full-tree FK (the forward_kinematics / fk_arrays
// API), single-link FK for benchmark targets, numpy-exact Philox sampling,
// and the FP32 FMA-pipe microbenchmark that gives the roofline denominator.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kop_kernels.cuh"

namespace kop {

// ---------------------------------------------------------------------------
// Full-tree FK in the reference's operation order (robot.py:404-448):
// for each joint in topological order: fq = q_parent * q_origin,
// fp = p_parent + R_parent p_origin; anchor = fp, world axis = R(fq) axis;
// revolute: child = fq * (cos th/2, sin th/2 axis); prismatic: fp + th axis_w.
//
// HBM-write-bound (per configuration n doubles in, L * 7 + J * 6 doubles
// out): every thread builds its frames in SHARED memory (thread-major,
// [link][wxyz xyz] then [joint][anchor axis]), then the CTA writes its rows
// of each output array as one contiguous, coalesced stream -- instead of each
// thread storing its own L * 4 / L * 3 / J * 3 segments at a stride of a
// whole row (round 1: per-thread local arrays, uncoalesced AoS stores).
// ---------------------------------------------------------------------------
template <typename T, bool KOP_FK_STAGE_JOINTS>
__global__ void __launch_bounds__(256)
k_fk_tree(const TreeParams P, const double* __restrict__ q, int64_t B, double* __restrict__ lq_out,
          double* __restrict__ lp_out, double* __restrict__ jp_out, double* __restrict__ ja_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int nl = P.nl, nj = P.nj, per = 7 * nl + (KOP_FK_STAGE_JOINTS ? 6 * nj : 0);  // T words per configuration
  T* my = reinterpret_cast<T*>(smem_raw) + (size_t)threadIdx.x * per;
  const int64_t b0 = (int64_t)blockIdx.x * blockDim.x;
  const int64_t b = b0 + threadIdx.x;
  const int rows = (int)(B - b0 < (int64_t)blockDim.x ? B - b0 : (int64_t)blockDim.x);
  if (b < B) {
    T* F = my;            // link frames [nl][7]
    T* A = my + 7 * nl;   // joint anchor / axis [nj][6]
    F[0] = T(1); F[1] = T(0); F[2] = T(0); F[3] = T(0); F[4] = T(0); F[5] = T(0); F[6] = T(0);
    const double* qb = q + b * P.n;
    for (int j = 0; j < nj; ++j) {
      const T* pf = F + 7 * P.parent[j];
      const quat<T> pq{pf[0], pf[1], pf[2], pf[3]};
      const vec3<T> pp{pf[4], pf[5], pf[6]};
      const quat<T> fq = qmul(pq, quat<T>{T(P.oq[j][0]), T(P.oq[j][1]), T(P.oq[j][2]), T(P.oq[j][3])});
      const vec3<T> o = qrot(pq, vec3<T>{T(P.op[j][0]), T(P.op[j][1]), T(P.op[j][2])});
      const vec3<T> fp{pp.x + o.x, pp.y + o.y, pp.z + o.z};
      const vec3<T> axis{T(P.axis[j][0]), T(P.axis[j][1]), T(P.axis[j][2])};
      const vec3<T> wa = qrot(fq, axis);
      if (KOP_FK_STAGE_JOINTS) {
        T* aj = A + 6 * j;
        aj[0] = fp.x; aj[1] = fp.y; aj[2] = fp.z;
        aj[3] = wa.x; aj[4] = wa.y; aj[5] = wa.z;
      } else {  // anchors / axes straight to global (3 consecutive doubles each)
        if (jp_out) {
          double* d = jp_out + (b * nj + j) * 3;
          d[0] = fp.x; d[1] = fp.y; d[2] = fp.z;
        }
        if (ja_out) {
          double* d = ja_out + (b * nj + j) * 3;
          d[0] = wa.x; d[1] = wa.y; d[2] = wa.z;
        }
      }
      quat<T> cq = fq;
      vec3<T> cp = fp;
      if (P.kind[j] != 0) {
        const T th = T(qb[P.qcol[j]]) * T(P.mult[j]) + T(P.offset[j]);
        if (P.kind[j] == 1) {
          T s, co;
          sincos_t(T(0.5) * th, &s, &co);
          cq = qmul(fq, quat<T>{co, s * axis.x, s * axis.y, s * axis.z});
        } else {
          cp = {fp.x + th * wa.x, fp.y + th * wa.y, fp.z + th * wa.z};
        }
      }
      T* cf = F + 7 * P.child[j];
      cf[0] = cq.w; cf[1] = cq.x; cf[2] = cq.y; cf[3] = cq.z;
      cf[4] = cp.x; cf[5] = cp.y; cf[6] = cp.z;
    }
  }
  __syncthreads();
  // coalesced write-out of this CTA's `rows` consecutive output rows of each array
  const T* base = reinterpret_cast<const T*>(smem_raw);
  auto stream = [&](double* out, int width, int stride_in_row, int off, int comps) {
    if (!out) return;
    const int64_t n_out = (int64_t)rows * width * comps;
    double* dst = out + b0 * width * comps;
    for (int64_t i = threadIdx.x; i < n_out; i += blockDim.x) {
      const int r = (int)(i / (width * comps)), rem = (int)(i % (width * comps));
      const int e = rem / comps, c = rem % comps;
      dst[i] = double(base[(size_t)r * per + off + e * stride_in_row + c]);
    }
  };
  stream(lq_out, nl, 7, 0, 4);
  stream(lp_out, nl, 7, 4, 3);
  if (KOP_FK_STAGE_JOINTS) {
    stream(jp_out, nj, 6, 7 * nl, 3);
    stream(ja_out, nj, 6, 7 * nl + 3, 3);
  }
}

cudaError_t launch_fk_tree(const TreeParams& P, int precision, const double* q, int64_t B,
                           double* lq, double* lp, double* jp, double* ja, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const size_t word = precision == 0 ? sizeof(float) : sizeof(double);
  // as many 32-thread groups as fit in ~96 KB of shared memory (2 CTAs per SM), <= 256 threads; the joint
  // anchors / axes are staged too when that still leaves >= 128 threads per CTA, else stored directly
  // (A/B, tools/fk_time.py: staging everything wins for the Panda in FP32, direct joint stores for the
  // Panda in FP64 and for the humanoid, whose footprint would leave too few warps)
  auto tpb_for = [&](size_t per) {
    const int t = (int)((96 * 1024) / (per * 32)) * 32;
    return t < 32 ? 32 : (t > 256 ? 256 : t);
  };
  const size_t per_all = word * (size_t)(7 * P.nl + 6 * P.nj), per_frames = word * (size_t)(7 * P.nl);
  const bool stage = tpb_for(per_all) >= 128;
  const size_t per = stage ? per_all : per_frames;
  const int tpb = tpb_for(per);
  const size_t smem = per * tpb;
  const unsigned blocks = (unsigned)((B + tpb - 1) / tpb);
  cudaError_t e = cudaSuccess;
  auto go = [&](auto kern) {
    if (smem > 48 * 1024 &&
        (e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
      return;
    kern<<<blocks, tpb, smem, st>>>(P, q, B, lq, lp, jp, ja);
    e = cudaGetLastError();
  };
  if (precision == 0)
    stage ? go(k_fk_tree<float, true>) : go(k_fk_tree<float, false>);
  else
    stage ? go(k_fk_tree<double, true>) : go(k_fk_tree<double, false>);
  return e;
}

// Geometric Jacobian (robot.py:461-506): rows 0-2 the world linear velocity of
// a point rigidly attached to `link` (its origin when points == null), rows
// 3-5 (rotational) the angular velocity; mimic joints fold into their source
// column.  FK as k_fk_tree, then one pass over the link's ancestor joints.
template <typename T>
__global__ void __launch_bounds__(128)
k_jacobian_tree(const TreeParams P, const double* __restrict__ q, int64_t B, int link,
                unsigned long long anc, const double* __restrict__ points, int rotational,
                double* __restrict__ jac) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  quat<T> lq[kMaxLinks];
  vec3<T> lp[kMaxLinks], jp[kMaxTreeJoints], ja[kMaxTreeJoints];
  lq[0] = {T(1), T(0), T(0), T(0)};
  lp[0] = {T(0), T(0), T(0)};
  const double* qb = q + b * P.n;
  for (int j = 0; j < P.nj; ++j) {
    const quat<T> pq = lq[P.parent[j]];
    const vec3<T> pp = lp[P.parent[j]];
    const quat<T> fq = qmul(pq, quat<T>{T(P.oq[j][0]), T(P.oq[j][1]), T(P.oq[j][2]), T(P.oq[j][3])});
    const vec3<T> o = qrot(pq, vec3<T>{T(P.op[j][0]), T(P.op[j][1]), T(P.op[j][2])});
    const vec3<T> fp{pp.x + o.x, pp.y + o.y, pp.z + o.z};
    const vec3<T> axis{T(P.axis[j][0]), T(P.axis[j][1]), T(P.axis[j][2])};
    const vec3<T> wa = qrot(fq, axis);
    jp[j] = fp;
    ja[j] = wa;
    const int c = P.child[j];
    if (P.kind[j] == 0) {
      lq[c] = fq;
      lp[c] = fp;
      continue;
    }
    const T th = T(qb[P.qcol[j]]) * T(P.mult[j]) + T(P.offset[j]);
    if (P.kind[j] == 1) {
      T s, co;
      sincos_t(T(0.5) * th, &s, &co);
      lq[c] = qmul(fq, quat<T>{co, s * axis.x, s * axis.y, s * axis.z});
      lp[c] = fp;
    } else {
      lq[c] = fq;
      lp[c] = {fp.x + th * wa.x, fp.y + th * wa.y, fp.z + th * wa.z};
    }
  }
  const vec3<T> pt = points ? vec3<T>{T(points[b * 3]), T(points[b * 3 + 1]), T(points[b * 3 + 2])} : lp[link];
  const int rows = rotational ? 6 : 3;
  double* J = jac + b * rows * P.n;
  for (int i = 0; i < rows * P.n; ++i) J[i] = 0.0;
  for (int j = 0; j < P.nj; ++j) {
    if (!((anc >> j) & 1ull) || P.kind[j] == 0) continue;
    const int col = P.qcol[j];
    const T mu = T(P.mult[j]);
    const vec3<T> a = ja[j];
    if (P.kind[j] == 1) {
      const vec3<T> lever{pt.x - jp[j].x, pt.y - jp[j].y, pt.z - jp[j].z};
      const vec3<T> v = cross(a, lever);
      J[0 * P.n + col] += double(mu * v.x);
      J[1 * P.n + col] += double(mu * v.y);
      J[2 * P.n + col] += double(mu * v.z);
      if (rotational) {
        J[3 * P.n + col] += double(mu * a.x);
        J[4 * P.n + col] += double(mu * a.y);
        J[5 * P.n + col] += double(mu * a.z);
      }
    } else {
      J[0 * P.n + col] += double(mu * a.x);
      J[1 * P.n + col] += double(mu * a.y);
      J[2 * P.n + col] += double(mu * a.z);
    }
  }
}

cudaError_t launch_jacobian_tree(const TreeParams& P, int precision, const double* q, int64_t B, int link,
                                 unsigned long long anc, const double* points, int rotational, double* jac,
                                 cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const int tpb = 128;
  const unsigned blocks = (unsigned)((B + tpb - 1) / tpb);
  if (precision == 0)
    k_jacobian_tree<float><<<blocks, tpb, 0, st>>>(P, q, B, link, anc, points, rotational, jac);
  else
    k_jacobian_tree<double><<<blocks, tpb, 0, st>>>(P, q, B, link, anc, points, rotational, jac);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// FK of one link along its root path (joints of `path` are consecutive:
// each joint's parent is the previous joint's child), canonicalised like
// Transform3.from_parts (liegroups.py:33-45, 372-374).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128)
k_link_pose(const TreeParams P, const double* __restrict__ q, int64_t B, double* __restrict__ out) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= B) return;
  quat<double> pq{1.0, 0.0, 0.0, 0.0};
  vec3<double> pp{0.0, 0.0, 0.0};
  const double* qb = q + b * P.n;
  for (int j = 0; j < P.nj; ++j) {
    const quat<double> fq = qmul(pq, quat<double>{P.oq[j][0], P.oq[j][1], P.oq[j][2], P.oq[j][3]});
    const vec3<double> o = qrot(pq, vec3<double>{P.op[j][0], P.op[j][1], P.op[j][2]});
    const vec3<double> fp{pp.x + o.x, pp.y + o.y, pp.z + o.z};
    const vec3<double> axis{P.axis[j][0], P.axis[j][1], P.axis[j][2]};
    if (P.kind[j] == 0) {
      pq = fq;
      pp = fp;
      continue;
    }
    const double th = qb[P.qcol[j]] * P.mult[j] + P.offset[j];
    if (P.kind[j] == 1) {
      double s, c;
      sincos(0.5 * th, &s, &c);
      pq = qmul(fq, quat<double>{c, s * axis.x, s * axis.y, s * axis.z});
      pp = fp;
    } else {
      const vec3<double> wa = qrot(fq, axis);
      pq = fq;
      pp = {fp.x + th * wa.x, fp.y + th * wa.y, fp.z + th * wa.z};
    }
  }
  const double n = sqrt(pq.w * pq.w + pq.x * pq.x + pq.y * pq.y + pq.z * pq.z);
  double w = pq.w / n, x = pq.x / n, y = pq.y / n, z = pq.z / n;
  double sign = w < 0.0 ? -1.0 : 1.0;
  if (w == 0.0) {
    const double ax = fabs(x), ay = fabs(y), az = fabs(z);
    const double lead = (ax >= ay && ax >= az) ? x : (ay >= az ? y : z);
    sign = lead < 0.0 ? -1.0 : 1.0;
  }
  double* d = out + b * 7;
  d[0] = w * sign; d[1] = x * sign; d[2] = y * sign; d[3] = z * sign;
  d[4] = pp.x; d[5] = pp.y; d[6] = pp.z;
}

cudaError_t launch_link_pose(const TreeParams& path, const double* q, int64_t B, double* poses,
                             cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  const int tpb = 128;
  k_link_pose<<<(unsigned)((B + tpb - 1) / tpb), tpb, 0, st>>>(path, q, B, poses);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// numpy.random.Philox (Philox4x64-10, Random123 constants): the counter is
// incremented BEFORE each 4-word block (numpy philox_next), key = (k0, k1),
// counter starts at 0.  next_double = (u >> 11) * 2^-53; Generator.uniform
// is low + (high - low) * u (numpy random_uniform), evaluated without FMA
// contraction so the draws are bit-identical to numpy's.
// ---------------------------------------------------------------------------
struct Philox {
  uint64_t ctr[4];
  uint64_t key[2];
  uint64_t buf[4];
  int pos;
};

__device__ __forceinline__ void philox_block(const uint64_t in[4], const uint64_t key_in[2], uint64_t out[4]) {
  uint64_t c0 = in[0], c1 = in[1], c2 = in[2], c3 = in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B97F4A7C15ull;
      k1 += 0xBB67AE8584CAA73Bull;
    }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ull * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ull, c0);
    const uint64_t lo1 = 0xCA5A826395121157ull * c2, hi1 = __umul64hi(0xCA5A826395121157ull, c2);
    const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

__device__ __forceinline__ uint64_t philox_next(Philox& s) {
  if (s.pos < 4) return s.buf[s.pos++];
  s.ctr[0]++;
  if (s.ctr[0] == 0) {
    s.ctr[1]++;
    if (s.ctr[1] == 0) {
      s.ctr[2]++;
      if (s.ctr[2] == 0) s.ctr[3]++;
    }
  }
  philox_block(s.ctr, s.key, s.buf);
  s.pos = 1;
  return s.buf[0];
}

__global__ void __launch_bounds__(128)
k_philox(uint64_t key0, uint64_t key1_base, int64_t count, int n, const double* __restrict__ lo,
         const double* __restrict__ range, const uint8_t* __restrict__ negate, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  Philox s;
  s.ctr[0] = s.ctr[1] = s.ctr[2] = s.ctr[3] = 0;
  s.key[0] = key0;
  s.key[1] = key1_base + (uint64_t)i;
  s.pos = 4;
  for (int j = 0; j < n; ++j) {
    const uint64_t u = philox_next(s);
    const double x = __dmul_rn((double)(u >> 11), 1.0 / 9007199254740992.0);
    double v = __dadd_rn(lo[j], __dmul_rn(range[j], x));
    if (negate[j]) v = -v;
    out[i * n + j] = v;
  }
}

cudaError_t launch_philox(uint64_t key0, uint64_t key1_base, int64_t count, int n, const double* lo,
                          const double* range, const uint8_t* negate, double* out, cudaStream_t st) {
  if (count == 0) return cudaSuccess;
  const int tpb = 128;
  k_philox<<<(unsigned)((count + tpb - 1) / tpb), tpb, 0, st>>>(key0, key1_base, count, n, lo, range,
                                                                negate, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// FP32 FMA-pipe peak: 16 independent immediate-operand FFMA chains/thread.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_fma_peak(float* sink, int iters) {
  float a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = (float)(threadIdx.x + k) * 1e-3f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) a[k] = fmaf(a[k], 0.9999f, 0.0001f);
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += a[k];
  if (s == 12345.678f) sink[blockIdx.x] = s;  // never true; defeats DCE
}

cudaError_t launch_fma_peak(int blocks, int threads, int iters, float* sink, cudaStream_t st) {
  k_fma_peak<<<blocks, threads, 0, st>>>(sink, iters);
  return cudaGetLastError();
}

// FP64 twin: 8 independent DFMA chains per thread
__global__ void __launch_bounds__(256) k_dfma_peak(double* sink, int iters) {
  double a[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = (double)(threadIdx.x + k) * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], 0.9999, 0.0001);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.678) sink[blockIdx.x] = s;  // never true; defeats DCE
}

cudaError_t launch_dfma_peak(int blocks, int threads, int iters, double* sink, cudaStream_t st) {
  k_dfma_peak<<<blocks, threads, 0, st>>>(sink, iters);
  return cudaGetLastError();
}

// Checking-build probe: copies its (never written) dynamic shared memory out.
// In the poison build every word is 0xFFFFFFFF (the positive control of
// tests/test_gpu_checks.py); in the normal build the values are undefined.
__global__ void __launch_bounds__(128) k_check_probe(uint32_t* out, int words) {
  extern __shared__ unsigned char smem_raw[];
  KOP_SMEM_ENTRY(smem_raw);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(smem_raw);
  for (int i = threadIdx.x; i < words; i += blockDim.x) out[i] = w[i];
}

cudaError_t launch_check_probe(uint32_t* out, int words, cudaStream_t st) {
  k_check_probe<<<1, 128, (size_t)words * 4, st>>>(out, words);
  return cudaGetLastError();
}

}  // namespace kop
