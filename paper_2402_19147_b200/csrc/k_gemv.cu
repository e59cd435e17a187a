// Quaternion matrix-vector products for the Krylov spectral norm (linalg.py:365-367,
// spectral_norm = the largest singular value; used by the CLI `approx` metrics,
// cli.py:169-189).  HBM-bound: one pass over A per product, fixed reduction orders
// (bitwise reproducible).
//   N: y = A x   (A m x n, row-major interleaved; one warp per row)
//   H: y = A^H x (32 columns per CTA, 8 row slices reduced in slice order)
#include "common.cuh"
#include "kernels.h"

namespace qcur {

namespace {

__global__ void __launch_bounds__(256) k_qgemv_n(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                                 const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (row >= m) return;
  const double* a = A + row * lda * 4;
  Quat acc = qzero();
  for (int64_t j = lane; j < n; j += 32) acc = qadd(acc, qmul(ldq_nc(a + j * 4), ldq_nc(x + j * 4)));
  acc = warp_sum(acc);
  if (lane == 0) stq(y + row * 4, acc);
}

__global__ void __launch_bounds__(256) k_qgemv_h(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                                 const double* __restrict__ x, double* __restrict__ y) {
  __shared__ Quat part[8][32];
  const int lane = threadIdx.x & 31, slice = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const int64_t rows_per = (m + 7) / 8, r0 = slice * rows_per, r1 = r0 + rows_per < m ? r0 + rows_per : m;
  Quat acc = qzero();
  if (j < n)
    for (int64_t i = r0; i < r1; ++i) acc = qadd(acc, qmul(qconj(ldq_nc(A + (i * lda + j) * 4)), ldq_nc(x + i * 4)));
  part[slice][lane] = acc;
  __syncthreads();
  if (slice == 0 && j < n) {
    Quat s = part[0][lane];
    for (int k = 1; k < 8; ++k) s = qadd(s, part[k][lane]);
    stq(y + j * 4, s);
  }
}

}  // namespace

void launch_qgemv(int op, const double* A, int64_t m, int64_t n, int64_t lda, const double* x, double* y,
                  cudaStream_t st) {
  ++::qcur::g_launches;
  if (op == 0) k_qgemv_n<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(A, m, n, lda, x, y);
  else k_qgemv_h<<<(unsigned)((n + 31) / 32), 256, 0, st>>>(A, m, n, lda, x, y);
}

}  // namespace qcur
