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
// column-major.  A round pairs all n columns by the round-robin (circle) schedule; one CTA
// rotates one pair (A columns and V columns).  A sweep is n-1 rounds; the host stops after the
// first sweep without a rotation (flag) or after 60 sweeps.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace qcur {

namespace {

__device__ __forceinline__ Quat ldQ(const double* p) { return *reinterpret_cast<const Quat*>(p); }
__device__ __forceinline__ void stQ(double* p, const Quat& q) { *reinterpret_cast<Quat*>(p) = q; }

// The (a, b) pair of round rnd of the round-robin schedule over nn = n + (n & 1) slots.
__device__ __forceinline__ void round_pair(int64_t pk, int64_t nn, int64_t rnd, int64_t& a, int64_t& b) {
  if (pk == 0) {
    a = rnd;
    b = nn - 1;
  } else {
    a = (rnd + pk) % (nn - 1);
    b = (rnd - pk + (nn - 1)) % (nn - 1);
  }
}

// One CTA of T threads rotates one pair.  With R > 0 each thread keeps its R rows of both columns
// in registers between the inner products and the rotation (R * T >= m), so A is read once and
// written once per round; R == 0 streams the columns twice (m > 4 * 512).
template <int T, int R>
__global__ void __launch_bounds__(T) k_jac_pair(double* __restrict__ A, int64_t m, int64_t n, double* __restrict__ V,
                                               int64_t rnd, unsigned* __restrict__ flag) {
  constexpr int W = T / 32;
  __shared__ double red[W][6];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  int64_t a, b;
  round_pair(blockIdx.x, n + (n & 1), rnd, a, b);
  if (a >= n || b >= n) return;
  double* ca = A + a * m * 4;
  double* cb = A + b * m * 4;
  double al = 0.0, be = 0.0;
  Quat g = qzero();
  Quat xa[R > 0 ? R : 1], xb[R > 0 ? R : 1];
  if constexpr (R > 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = tid + (int64_t)r * T;
      if (i < m) {
        xa[r] = ldQ(ca + i * 4);
        xb[r] = ldQ(cb + i * 4);
      } else {
        xa[r] = qzero();
        xb[r] = qzero();
      }
      al += qnorm2(xa[r]);
      be += qnorm2(xb[r]);
      qfma_conj(g, xa[r], xb[r]);
    }
  } else {
    for (int64_t i = tid; i < m; i += T) {
      const Quat pa = ldQ(ca + i * 4), pb = ldQ(cb + i * 4);
      al += qnorm2(pa);
      be += qnorm2(pb);
      qfma_conj(g, pa, pb);
    }
  }
  al = warp_sum(al);
  be = warp_sum(be);
  g = warp_sum(g);
  if (lane == 0) {
    red[wid][0] = al;
    red[wid][1] = be;
    red[wid][2] = g.w;
    red[wid][3] = g.x;
    red[wid][4] = g.y;
    red[wid][5] = g.z;
  }
  __syncthreads();
  al = red[0][0];
  be = red[0][1];
  g = Quat{red[0][2], red[0][3], red[0][4], red[0][5]};
#pragma unroll
  for (int w = 1; w < W; ++w) {
    al += red[w][0];
    be += red[w][1];
    g = qadd(g, Quat{red[w][2], red[w][3], red[w][4], red[w][5]});
  }
  const double gn = sqrt(qnorm2(g));
  // rotate unless the pair is already orthogonal to working precision (uniform over the CTA)
  if (!(gn > 4.0 * DBL_EPSILON * sqrt(al) * sqrt(be)) || !(al > 0.0) || !(be > 0.0)) return;
  if (tid == 0) *flag = 1u;
  // with mu = g / |g|: [a b mu^-1] rotated by the real angle that zeroes the 2 x 2 Gram's off-diagonal
  const Quat mu_bar = qconj(qscale(g, 1.0 / gn));
  const double zeta = (be - al) / (2.0 * gn);
  const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
  if constexpr (R > 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = tid + (int64_t)r * T;
      if (i < m) {
        const Quat pb = qmul(xb[r], mu_bar);
        stQ(ca + i * 4, qsub(qscale(xa[r], c), qscale(pb, s)));
        stQ(cb + i * 4, qadd(qscale(xa[r], s), qscale(pb, c)));
      }
    }
  } else {
    for (int64_t i = tid; i < m; i += T) {
      const Quat pa = ldQ(ca + i * 4), pb = qmul(ldQ(cb + i * 4), mu_bar);
      stQ(ca + i * 4, qsub(qscale(pa, c), qscale(pb, s)));
      stQ(cb + i * 4, qadd(qscale(pa, s), qscale(pb, c)));
    }
  }
  if (V) {
    double* va = V + a * n * 4;
    double* vb = V + b * n * 4;
    for (int64_t i = tid; i < n; i += T) {
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

// Certificate for the truncated SVD: flag = 1 if any column j is not orthogonal to one of the k
// columns top[0..k), |a_i^H a_j| > max(4, sqrt(m)) eps ||a_i|| ||a_j|| (one warp per column j).
// sqrt(m) eps is the rounding level of the inner product itself (LAPACK's one-sided Jacobi uses the
// same stopping threshold); the rotation kernels keep the stricter 4 eps.
__global__ void __launch_bounds__(256) k_jac_cert(const double* __restrict__ A, int64_t m, int64_t n,
                                                 const int* __restrict__ top, int k, const double* __restrict__ sigma,
                                                 unsigned* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (j >= n) return;
  const double* cj = A + j * m * 4;
  const double tol = fmax(4.0, sqrt((double)m)) * DBL_EPSILON;
  for (int t = 0; t < k; ++t) {
    const int64_t i = top[t];
    if (i == j) continue;
    const double* ci = A + i * m * 4;
    Quat g = qzero();
    for (int64_t r = lane; r < m; r += 32) qfma_conj(g, ldQ(ci + r * 4), ldQ(cj + r * 4));
    g = warp_sum(g);
    if (sqrt(qnorm2(g)) > tol * sigma[i] * sigma[j]) {
      if (lane == 0) *flag = 1u;
      return;
    }
  }
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

int64_t jacobi_sweep_rounds(int64_t, int64_t n) { return n + (n & 1) - 1; }

void launch_jacobi_round(double* Acm, int64_t m, int64_t n, double* Vcm, int64_t rnd, unsigned* flag, cudaStream_t st) {
  ++::qcur::g_launches;
  const unsigned npairs = (unsigned)((n + (n & 1)) / 2);
  // threads per pair: enough for 4 register rows each, 64..512
  if (m <= 64 * 4) {
    if (m <= 64) k_jac_pair<64, 1><<<npairs, 64, 0, st>>>(Acm, m, n, Vcm, rnd, flag);
    else if (m <= 128) k_jac_pair<64, 2><<<npairs, 64, 0, st>>>(Acm, m, n, Vcm, rnd, flag);
    else k_jac_pair<64, 4><<<npairs, 64, 0, st>>>(Acm, m, n, Vcm, rnd, flag);
  } else if (m <= 128 * 4) {
    k_jac_pair<128, 4><<<npairs, 128, 0, st>>>(Acm, m, n, Vcm, rnd, flag);
  } else if (m <= 256 * 4) {
    k_jac_pair<256, 4><<<npairs, 256, 0, st>>>(Acm, m, n, Vcm, rnd, flag);
  } else if (m <= 512 * 4) {
    k_jac_pair<512, 4><<<npairs, 512, 0, st>>>(Acm, m, n, Vcm, rnd, flag);
  } else {
    k_jac_pair<512, 0><<<npairs, 512, 0, st>>>(Acm, m, n, Vcm, rnd, flag);
  }
}

void launch_col_norms(const double* Acm, int64_t m, int64_t n, double* sigma, cudaStream_t st) {
  ++::qcur::g_launches;
  k_col_norms<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(Acm, m, n, sigma);
}

void launch_jacobi_cert(const double* Acm, int64_t m, int64_t n, const int* top, int k, const double* sigma,
                        unsigned* flag, cudaStream_t st) {
  ++::qcur::g_launches;
  k_jac_cert<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(Acm, m, n, top, k, sigma, flag);
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
