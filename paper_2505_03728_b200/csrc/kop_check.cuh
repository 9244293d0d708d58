// Checking builds (compute-sanitizer is closed on this GPU pool, DESIGN.md
// section 5): compile-time switches that leave the normal build untouched.
//
//   KOP_SMEM_POISON  every kernel first fills its dynamic shared memory with
//                    0xFF bytes (a NaN in float and double) -- a read of shared
//                    memory that was never written then poisons the result,
//                    which tests/test_gpu_checks.py compares bitwise with the
//                    normal build (the initcheck of shared memory).
//   KOP_JITTER       every __syncthreads / __syncwarp / named barrier is
//                    preceded and followed by a pseudo-random __nanosleep per
//                    thread, so threads reach and leave barriers in a different
//                    order on every run: a missing barrier (a race) shows up as
//                    results that differ from the normal build's (racecheck by
//                    schedule perturbation).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#if defined(KOP_JITTER) && defined(__CUDA_ARCH__)
__device__ __forceinline__ void kop_jitter() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  unsigned h = (unsigned)t ^ (threadIdx.x * 2654435761u) ^ (blockIdx.x * 40503u);
  h ^= h >> 13;
  h *= 0x5bd1e995u;
  __nanosleep(h & 2047u);
}
__device__ __forceinline__ void kop_syncthreads_jittered() {
  kop_jitter();
  __syncthreads();
  kop_jitter();
}
__device__ __forceinline__ void kop_syncwarp_jittered(unsigned mask = 0xffffffffu) {
  kop_jitter();
  __syncwarp(mask);
  kop_jitter();
}
#define __syncthreads() kop_syncthreads_jittered()
#define __syncwarp(...) kop_syncwarp_jittered(__VA_ARGS__)
#define KOP_JITTER_POINT() kop_jitter()
#else
#define KOP_JITTER_POINT() ((void)0)
#endif

#if defined(KOP_SMEM_POISON) && defined(__CUDA_ARCH__)
// must run before any thread of the block can return (it ends with a barrier)
#define KOP_SMEM_ENTRY(base)                                                      \
  do {                                                                             \
    unsigned kop_dyn_;                                                             \
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(kop_dyn_));            \
    uint32_t* kop_w_ = reinterpret_cast<uint32_t*>(base);                          \
    for (unsigned i = threadIdx.x; i < kop_dyn_ / 4; i += blockDim.x) kop_w_[i] = 0xFFFFFFFFu; \
    __syncthreads();                                                               \
  } while (0)
#else
#define KOP_SMEM_ENTRY(base) ((void)0)
#endif
