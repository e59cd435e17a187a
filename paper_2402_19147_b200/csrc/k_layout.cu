// K0 / K3 — layout conversion and the bit-exact C / R gathers.
//
// K0 converts the reference's storage (four planar float64 planes,
// pkg/src/qcur/quat.py:129-143) to the device's interleaved 32-byte
// quaternions and back.  K3 replaces QMatrix.take_cols / take_rows
// (quat.py:215-225): C = X[:, J] and R = X[I, :] are pure copies, so they are
// bit-identical to the reference by construction.
#include "common.cuh"
#include "kernels.h"

namespace qcur {

static int grid_for(int64_t work, int threads, int cap = 148 * 16) {
  int64_t b = (work + threads - 1) / threads;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

__global__ void k0_planar_to_interleaved(const double* __restrict__ a0, const double* __restrict__ a1,
                                         const double* __restrict__ a2, const double* __restrict__ a3, int64_t N,
                                         double* __restrict__ X) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    Quat q{a0[t], a1[t], a2[t], a3[t]};
    stq(X + t * 4, q);
  }
}

__global__ void k0_interleaved_to_planar(const double* __restrict__ X, int64_t m, int64_t n, int64_t ldx,
                                         double* __restrict__ a0, double* __restrict__ a1, double* __restrict__ a2,
                                         double* __restrict__ a3) {
  const int64_t N = m * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t - i * n;
    Quat q = ldq_nc(X + (i * ldx + j) * 4);
    a0[t] = q.w;
    a1[t] = q.x;
    a2[t] = q.y;
    a3[t] = q.z;
  }
}

// C[i, jj] = X[i, J[jj]]: lanes run along jj so each warp writes one contiguous
// 1 KB segment of C and reads 32 independent 32-byte sectors of X.
__global__ void k3_gather_cols(const double* __restrict__ X, int64_t m, int64_t ldx, const int64_t* __restrict__ J,
                               int64_t c, double* __restrict__ C) {
  const int64_t N = m * c;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / c, jj = t - i * c;
    stq(C + t * 4, ldq_nc(X + (i * ldx + J[jj]) * 4));
  }
}

__global__ void k3_gather_rows(const double* __restrict__ X, int64_t n, int64_t ldx, const int64_t* __restrict__ I,
                               int64_t r, double* __restrict__ R) {
  const int64_t N = r * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t ii = t / n, j = t - ii * n;
    stq(R + t * 4, ldq_nc(X + (I[ii] * ldx + j) * 4));
  }
}

// out = mask ? Y : X per quaternion (project_observed, completion.py:101-111)
__global__ void k_project_observed(const double* __restrict__ X, const double* __restrict__ Y,
                                   const unsigned char* __restrict__ mask, int64_t N, double* __restrict__ out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N; t += (int64_t)gridDim.x * blockDim.x)
    stq(out + t * 4, ldq_nc((mask[t] ? Y : X) + t * 4));
}

// AH (n x m) = A^H (quat.py:299-302), tiled through shared memory.
__global__ void k_conj_transpose(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda,
                                 double* __restrict__ AH, int64_t ldah) {
  __shared__ Quat tile[32][33];
  const int64_t i0 = (int64_t)blockIdx.y * 32, j0 = (int64_t)blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t i = i0 + r, j = j0 + threadIdx.x;
    if (i < m && j < n) tile[r][threadIdx.x] = ldq(A + (i * lda + j) * 4);
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const int64_t j = j0 + r, i = i0 + threadIdx.x;
    if (i < m && j < n) stq(AH + (j * ldah + i) * 4, qconj(tile[threadIdx.x][r]));
  }
}

// status words of a batch's lane contexts OR-ed into the caller's, then cleared
struct StatusSrc {
  unsigned* p[16];
  int n;
};
__global__ void k_status_or(unsigned* dst, StatusSrc src) {
  if (threadIdx.x == 0) {
    unsigned v = 0;
    for (int k = 0; k < src.n; ++k) {
      v |= *src.p[k];
      *src.p[k] = 0u;
    }
    *dst |= v;
  }
}

void launch_status_or(unsigned* dst, unsigned* const* srcs, int n, cudaStream_t st) {
  StatusSrc s{};
  s.n = n < 16 ? n : 16;
  for (int k = 0; k < s.n; ++k) s.p[k] = srcs[k];
  ++::qcur::g_launches;
  k_status_or<<<1, 32, 0, st>>>(dst, s);
}

// Deterministic fixed-order reduction of (a, b) pairs: out2 = (sum a, sum b).
__global__ void k_reduce_pairs(const double* __restrict__ parts, int64_t nparts, double* __restrict__ out2) {
  __shared__ double sa[1024], sb[1024];
  double a = 0.0, b = 0.0;
  for (int64_t t = threadIdx.x; t < nparts; t += blockDim.x) {
    a += parts[2 * t];
    b += parts[2 * t + 1];
  }
  sa[threadIdx.x] = a;
  sb[threadIdx.x] = b;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      sa[threadIdx.x] += sa[threadIdx.x + s];
      sb[threadIdx.x] += sb[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out2[0] = sa[0];
    out2[1] = sb[0];
  }
}

// Deterministic fixed-order column sums of a [nrows][width] table (width <= 8).
__global__ void k_reduce_rows(const double* __restrict__ parts, int64_t nrows, int width, double* __restrict__ out) {
  __shared__ double sh[8][256];
  for (int c = 0; c < width; ++c) {
    double a = 0.0;
    for (int64_t t = threadIdx.x; t < nrows; t += blockDim.x) a += parts[t * width + c];
    sh[c][threadIdx.x] = a;
  }
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int c = 0; c < width; ++c) sh[c][threadIdx.x] += sh[c][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < width) out[threadIdx.x] = sh[threadIdx.x][0];
}

void launch_reduce_rows(const double* parts, int64_t nrows, int width, double* out, cudaStream_t st) {
  ++::qcur::g_launches;
  k_reduce_rows<<<1, 256, 0, st>>>(parts, nrows, width, out);
}

void launch_planar_to_interleaved(const double* a0, const double* a1, const double* a2, const double* a3, int64_t m,
                                  int64_t n, double* X, cudaStream_t st) {
  ++::qcur::g_launches;
  k0_planar_to_interleaved<<<grid_for(m * n, 256), 256, 0, st>>>(a0, a1, a2, a3, m * n, X);
}
void launch_interleaved_to_planar(const double* X, int64_t m, int64_t n, int64_t ldx, double* a0, double* a1,
                                  double* a2, double* a3, cudaStream_t st) {
  ++::qcur::g_launches;
  k0_interleaved_to_planar<<<grid_for(m * n, 256), 256, 0, st>>>(X, m, n, ldx, a0, a1, a2, a3);
}
void launch_gather_cols(const double* X, int64_t m, int64_t ldx, const int64_t* J, int64_t c, double* C,
                        cudaStream_t st) {
  ++::qcur::g_launches;
  k3_gather_cols<<<grid_for(m * c, 256), 256, 0, st>>>(X, m, ldx, J, c, C);
}
void launch_gather_rows(const double* X, int64_t n, int64_t ldx, const int64_t* I, int64_t r, double* R,
                        cudaStream_t st) {
  ++::qcur::g_launches;
  k3_gather_rows<<<grid_for(r * n, 256), 256, 0, st>>>(X, n, ldx, I, r, R);
}
void launch_project_observed(const double* X, const double* Y, const unsigned char* mask, int64_t m, int64_t n,
                             double* out, cudaStream_t st) {
  ++::qcur::g_launches;
  k_project_observed<<<grid_for(m * n, 256), 256, 0, st>>>(X, Y, mask, m * n, out);
}
// chi(A) (linalg.py:151-164): the 2m x 2n complex adjoint, row-major complex128 (re, im pairs):
// [[A_a, A_b], [-conj(A_b), conj(A_a)]] with A_a = a0 + i a1, A_b = a2 + i a3.  Sign flips only.
__global__ void k_complex_adjoint(const double* __restrict__ X, int64_t m, int64_t n, double* __restrict__ chi) {
  const int64_t ld = 4 * n;  // doubles per row of chi (2n complex)
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t - i * n;
    const Quat q = ldq_nc(X + t * 4);
    double* top = chi + i * ld;
    double* bot = chi + (m + i) * ld;
    *reinterpret_cast<double2*>(top + 2 * j) = make_double2(q.w, q.x);
    *reinterpret_cast<double2*>(top + 2 * (n + j)) = make_double2(q.y, q.z);
    *reinterpret_cast<double2*>(bot + 2 * j) = make_double2(-q.y, q.z);
    *reinterpret_cast<double2*>(bot + 2 * (n + j)) = make_double2(q.w, -q.x);
  }
}

void launch_complex_adjoint(const double* X, int64_t m, int64_t n, double* chi, cudaStream_t st) {
  ++::qcur::g_launches;
  k_complex_adjoint<<<grid_for(m * n, 256), 256, 0, st>>>(X, m, n, chi);
}

void launch_conj_transpose(const double* A, int64_t m, int64_t n, int64_t lda, double* AH, int64_t ldah,
                           cudaStream_t st) {
  dim3 grid((unsigned)((n + 31) / 32), (unsigned)((m + 31) / 32));
  ++::qcur::g_launches;
  k_conj_transpose<<<grid, dim3(32, 8), 0, st>>>(A, m, n, lda, AH, ldah);
}
void launch_reduce_pairs(const double* parts, int64_t nparts, double* out2, cudaStream_t st) {
  ++::qcur::g_launches;
  k_reduce_pairs<<<1, 1024, 0, st>>>(parts, nparts, out2);
}

}  // namespace qcur
