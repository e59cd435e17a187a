// Quaternion singular value decomposition on the GPU: one-sided (Hestenes) Jacobi directly in
// quaternion arithmetic, all pairs of a round in parallel.
//
// Replaces qsvd (pkg/src/qcur/linalg.py:226-310), which takes the complex adjoint chi(A)
// (2m x 2n), runs LAPACK zgesdd, keeps one singular value per pair and pulls the singular
// vectors back with pivoted Gram-Schmidt, and its users numerical_rank (linalg.py:370-378),
// lowrank_truncate (:381-383) and the perturbation bounds (cur.py:306-388).  Working on the
// quaternion columns themselves avoids the pairing: every rotation is a quaternion Givens
// rotation of two columns (a, b) that zeroes their inner product a^H b, so the singular values
// come out once each and ties need no special treatment.  One-sided Jacobi is also the most
// accurate dense SVD (small singular values to high relative accuracy).
//
// Layout: A (m x n, m >= n) column-major, each column m contiguous quaternions; V (n x n)
// column-major.  A round pairs all n columns by the round-robin (circle) schedule; one warp
// rotates one pair (A columns and V columns).  A sweep is n-1 rounds; the host stops after the
// first sweep without a rotation (flag) or after 60 sweeps.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace qcur {

namespace {

__device__ __forceinline__ Quat ldQ(const double* p) { return *reinterpret_cast<const Quat*>(p); }
__device__ __forceinline__ void stQ(double* p, const Quat& q) { *reinterpret_cast<Quat*>(p) = q; }

__global__ void __launch_bounds__(256) k_jac_round(double* __restrict__ A, int64_t m, int64_t n, double* __restrict__ V,
                                                  int64_t rnd, unsigned* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t pk = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  const int64_t nn = n + (n & 1), npairs = nn / 2;
  if (pk >= npairs) return;
  int64_t a, b;
  if (pk == 0) {
    a = rnd;
    b = nn - 1;
  } else {
    a = (rnd + pk) % (nn - 1);
    b = (rnd - pk + (nn - 1)) % (nn - 1);
  }
  if (a >= n || b >= n) return;
  double* ca = A + a * m * 4;
  double* cb = A + b * m * 4;
  double al = 0.0, be = 0.0;
  Quat g = qzero();
  for (int64_t i = lane; i < m; i += 32) {
    const Quat xa = ldQ(ca + i * 4), xb = ldQ(cb + i * 4);
    al += qnorm2(xa);
    be += qnorm2(xb);
    qfma_conj(g, xa, xb);  // g += conj(xa) xb
  }
  al = warp_sum(al);
  be = warp_sum(be);
  g = warp_sum(g);
  const double gn = sqrt(qnorm2(g));
  // rotate unless the pair is already orthogonal to working precision
  if (!(gn > 4.0 * DBL_EPSILON * sqrt(al) * sqrt(be)) || !(al > 0.0) || !(be > 0.0)) return;
  if (lane == 0) *flag = 1u;
  // with mu = g / |g|: [a b mu^-1] rotated by the real angle that zeroes the 2 x 2 Gram's off-diagonal
  const Quat mu_bar = qconj(qscale(g, 1.0 / gn));
  const double zeta = (be - al) / (2.0 * gn);
  const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
  for (int64_t i = lane; i < m; i += 32) {
    const Quat xa = ldQ(ca + i * 4), xb = qmul(ldQ(cb + i * 4), mu_bar);
    stQ(ca + i * 4, qsub(qscale(xa, c), qscale(xb, s)));
    stQ(cb + i * 4, qadd(qscale(xa, s), qscale(xb, c)));
  }
  if (V) {
    double* va = V + a * n * 4;
    double* vb = V + b * n * 4;
    for (int64_t i = lane; i < n; i += 32) {
      const Quat ya = ldQ(va + i * 4), yb = qmul(ldQ(vb + i * 4), mu_bar);
      stQ(va + i * 4, qsub(qscale(ya, c), qscale(yb, s)));
      stQ(vb + i * 4, qadd(qscale(ya, s), qscale(yb, c)));
    }
  }
}

// sigma_j = ||a_j|| (one warp per column)
__global__ void k_col_norms(const double* __restrict__ A, int64_t m, int64_t n, double* __restrict__ sigma) {
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= n) return;
  const double* cj = A + j * m * 4;
  double s = 0.0;
  for (int64_t i = lane; i < m; i += 32) s += qnorm2(ldQ(cj + i * 4));
  s = warp_sum(s);
  if (lane == 0) sigma[j] = sqrt(s);
}

__global__ void k_to_colmajor(const double* __restrict__ A, int64_t m, int64_t n, int64_t lda, double* __restrict__ Acm) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / m, i = t - j * m;
    stQ(Acm + t * 4, ldQ(A + (i * lda + j) * 4));
  }
}

__global__ void k_identity_cm(double* __restrict__ V, int64_t n) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / n, i = t - j * n;
    stQ(V + t * 4, Quat{i == j ? 1.0 : 0.0, 0.0, 0.0, 0.0});
  }
}

}  // namespace

void launch_jacobi_round(double* Acm, int64_t m, int64_t n, double* Vcm, int64_t rnd, unsigned* flag, cudaStream_t st) {
  const int64_t npairs = (n + (n & 1)) / 2;
  ++::qcur::g_launches;
  k_jac_round<<<(unsigned)((npairs + 7) / 8), 256, 0, st>>>(Acm, m, n, Vcm, rnd, flag);
}

void launch_col_norms(const double* Acm, int64_t m, int64_t n, double* sigma, cudaStream_t st) {
  ++::qcur::g_launches;
  k_col_norms<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(Acm, m, n, sigma);
}

void launch_to_colmajor(const double* A, int64_t m, int64_t n, int64_t lda, double* Acm, cudaStream_t st) {
  int blocks = (int)((m * n + 255) / 256);
  if (blocks > 4736) blocks = 4736;
  if (blocks < 1) blocks = 1;
  ++::qcur::g_launches;
  k_to_colmajor<<<blocks, 256, 0, st>>>(A, m, n, lda, Acm);
}

void launch_identity_cm(double* Vcm, int64_t n, cudaStream_t st) {
  int blocks = (int)((n * n + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  if (blocks < 1) blocks = 1;
  ++::qcur::g_launches;
  k_identity_cm<<<blocks, 256, 0, st>>>(Vcm, n);
}

}  // namespace qcur
