// Shared device helpers for the QMCUR sm_100a kernels.
//
// Device layout: a quaternion matrix X (m x n) is stored
// *interleaved*, row-major: element (i, j) occupies the 32 bytes
// X[(i*ld + j)*4 + {0,1,2,3}] = (a0, a1, a2, a3).  Viewed as reals it is the
// row-major m x 4n matrix the FP64 DMMA tiles consume directly.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

namespace qcur {

// True the first time it is called on the current device for this flag: kernel
// attributes (cudaFuncSetAttribute) are per device, so a process driving several
// GPUs sets them once on each.
inline bool first_on_device(std::atomic<unsigned>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned bit = 1u << (dev & 31);
  return !(done.fetch_or(bit) & bit);
}


struct __align__(32) Quat {
  double w, x, y, z;
};

__device__ __forceinline__ Quat qzero() { return Quat{0.0, 0.0, 0.0, 0.0}; }

// Hamilton product (quat.py:67-76 convention: ij = k, jk = i, ki = j).
__device__ __forceinline__ Quat qmul(const Quat& a, const Quat& b) {
  Quat r;
  r.w = a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z;
  r.x = a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y;
  r.y = a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x;
  r.z = a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w;
  return r;
}
__device__ __forceinline__ Quat qconj(const Quat& a) { return Quat{a.w, -a.x, -a.y, -a.z}; }
__device__ __forceinline__ Quat qadd(const Quat& a, const Quat& b) {
  return Quat{a.w + b.w, a.x + b.x, a.y + b.y, a.z + b.z};
}
__device__ __forceinline__ Quat qsub(const Quat& a, const Quat& b) {
  return Quat{a.w - b.w, a.x - b.x, a.y - b.y, a.z - b.z};
}
__device__ __forceinline__ Quat qscale(const Quat& a, double s) { return Quat{a.w * s, a.x * s, a.y * s, a.z * s}; }
__device__ __forceinline__ double qnorm2(const Quat& a) { return a.w * a.w + a.x * a.x + a.y * a.y + a.z * a.z; }
// acc += conj(a) * b
__device__ __forceinline__ void qfma_conj(Quat& acc, const Quat& a, const Quat& b) {
  acc.w += a.w * b.w + a.x * b.x + a.y * b.y + a.z * b.z;
  acc.x += a.w * b.x - a.x * b.w - a.y * b.z + a.z * b.y;
  acc.y += a.w * b.y + a.x * b.z - a.y * b.w - a.z * b.x;
  acc.z += a.w * b.z - a.x * b.y + a.y * b.x - a.z * b.w;
}
// acc += a * b
__device__ __forceinline__ void qfma(Quat& acc, const Quat& a, const Quat& b) {
  acc.w += a.w * b.w - a.x * b.x - a.y * b.y - a.z * b.z;
  acc.x += a.w * b.x + a.x * b.w + a.y * b.z - a.z * b.y;
  acc.y += a.w * b.y - a.x * b.z + a.y * b.w + a.z * b.x;
  acc.z += a.w * b.z + a.x * b.y - a.y * b.x + a.z * b.w;
}

// 256-bit global load of one interleaved quaternion (LDG.E.ENL2.256 on sm_100).
__device__ __forceinline__ Quat ldq(const double* p) {
  Quat q;
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(q.w), "=d"(q.x), "=d"(q.y), "=d"(q.z)
               : "l"(p));
  return q;
}
__device__ __forceinline__ Quat ldq_nc(const double* p) {
  Quat q;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
               : "=d"(q.w), "=d"(q.x), "=d"(q.y), "=d"(q.z)
               : "l"(p));
  return q;
}
__device__ __forceinline__ void stq(double* p, const Quat& q) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(q.w), "d"(q.x), "d"(q.y), "d"(q.z)
               : "memory");
}

// Warp reductions in a fixed butterfly order (deterministic).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ Quat warp_sum(Quat q) {
  q.w = warp_sum(q.w);
  q.x = warp_sum(q.x);
  q.y = warp_sum(q.y);
  q.z = warp_sum(q.z);
  return q;
}

// Device-side status word bits, read back by the host after a pipeline.
enum StatusBits : unsigned {
  ST_SAMPLING = 1u,        // SamplingError (cur.py:223-227, 233-234)
  ST_DEGENERATE = 2u,      // DegenerateDistributionError (cur.py:145-146)
  ST_CHOL_FAIL_C = 4u,     // CholeskyQR2 broke down on C   -> robust path
  ST_CHOL_FAIL_R = 8u,     // CholeskyQR2 broke down on R^H -> robust path
  ST_DRAW_FALLBACK = 16u,  // a draw needed the exact sequential cumsum (info only)
  ST_SHAPE = 32u,
};

}  // namespace qcur

namespace qcur {
// number of kernels this library has launched (bench.py reports it as gpu_launches)
extern unsigned long long g_launches;
}  // namespace qcur
