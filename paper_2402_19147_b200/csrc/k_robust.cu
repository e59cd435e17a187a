// Robust factorization of a tall block Z (p x q) for pinv (the path rank-deficient or
// ill-conditioned C and R take; replacement of linalg.py:346-362 with the reference's cutoff):
// one-sided (Hestenes) Jacobi on Z itself, on one 16-CTA thread-block cluster.
//
//   Z V = A (columns a_j, ||a_j|| = sigma_j),  Z = W Sigma V^H,  pinv(Z) = V Sigma^+ W^H = F Q^H
//   with Q = W (a_j / sigma_j) and F = V Sigma^+, sigma_j <= cutoff dropped
//   (cutoff = eps max(p, q) sigma_max as linalg.py:338-339, or the caller's absolute tol).
//
// Round 1 ran a single-CTA Householder QR followed by a single-CTA Jacobi SVD of the q x q
// factor: 340 ms per side at cfg2 (p = 4000, q = 200; measured round 2, tools/robust_time.py).
// Here every round of the circle schedule rotates its q/2 disjoint column pairs on 16 CTAs
// (1024 threads each, a thread keeps its rows of the pair in registers), with one cluster
// barrier per round; a sweep ends with a cluster-wide "any rotation" vote read through
// distributed shared memory.  Launched unconditionally, it returns at once unless the fast
// path raised the problem's failure bit (no host synchronisation).
#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace qcur {

namespace {

constexpr int kRCl = 16;
constexpr int kRThreads = 1024;
constexpr int kRWarps = kRThreads / 32;
constexpr int kMaxSweeps = 60;

__device__ __forceinline__ Quat ldQr(const double* p) { return *reinterpret_cast<const Quat*>(p); }
__device__ __forceinline__ void stQr(double* p, const Quat& q) { *reinterpret_cast<Quat*>(p) = q; }

__device__ __forceinline__ void pair_of(int64_t pk, int64_t nn, int64_t rnd, int64_t& a, int64_t& b) {
  if (pk == 0) {
    a = rnd;
    b = nn - 1;
  } else {
    a = (rnd + pk) % (nn - 1);
    b = (rnd - pk + (nn - 1)) % (nn - 1);
  }
}

// rotate columns a, b of A (p rows, column-major) and of V (q rows) so that a^H b = 0; returns
// whether a rotation happened (uniform over the CTA).  R > 0: R rows per thread in registers.
template <int R>
__device__ bool rotate_pair(double* A, int64_t p, double* V, int64_t q, int64_t a, int64_t b, double (*red)[6]) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double* ca = A + a * p * 4;
  double* cb = A + b * p * 4;
  double al = 0.0, be = 0.0;
  Quat g = qzero();
  Quat xa[R > 0 ? R : 1], xb[R > 0 ? R : 1];
  if constexpr (R > 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = tid + (int64_t)r * kRThreads;
      xa[r] = i < p ? ldQr(ca + i * 4) : qzero();
      xb[r] = i < p ? ldQr(cb + i * 4) : qzero();
      al += qnorm2(xa[r]);
      be += qnorm2(xb[r]);
      qfma_conj(g, xa[r], xb[r]);
    }
  } else {
    for (int64_t i = tid; i < p; i += kRThreads) {
      const Quat pa = ldQr(ca + i * 4), pb = ldQr(cb + i * 4);
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
#pragma unroll 4
  for (int w = 1; w < kRWarps; ++w) {
    al += red[w][0];
    be += red[w][1];
    g = qadd(g, Quat{red[w][2], red[w][3], red[w][4], red[w][5]});
  }
  __syncthreads();  // red is reused by the next pair
  const double gn = sqrt(qnorm2(g));
  // rotation threshold: a few ulps of the pair's norms, growing like sqrt(p) with the rounding of the
  // p-term inner product (a fixed 4 eps kept some pairs rotating on their own rounding noise)
  const double tol = fmax(4.0, sqrt((double)p)) * DBL_EPSILON;
  if (!(gn > tol * sqrt(al) * sqrt(be)) || !(al > 0.0) || !(be > 0.0)) return false;
  const Quat mu_bar = qconj(qscale(g, 1.0 / gn));
  const double zeta = (be - al) / (2.0 * gn);
  const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
  const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
  if constexpr (R > 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int64_t i = tid + (int64_t)r * kRThreads;
      if (i < p) {
        const Quat pb = qmul(xb[r], mu_bar);
        stQr(ca + i * 4, qsub(qscale(xa[r], c), qscale(pb, s)));
        stQr(cb + i * 4, qadd(qscale(xa[r], s), qscale(pb, c)));
      }
    }
  } else {
    for (int64_t i = tid; i < p; i += kRThreads) {
      const Quat pa = ldQr(ca + i * 4), pb = qmul(ldQr(cb + i * 4), mu_bar);
      stQr(ca + i * 4, qsub(qscale(pa, c), qscale(pb, s)));
      stQr(cb + i * 4, qadd(qscale(pa, s), qscale(pb, c)));
    }
  }
  double* va = V + a * q * 4;
  double* vb = V + b * q * 4;
  for (int64_t i = tid; i < q; i += kRThreads) {
    const Quat ya = ldQr(va + i * 4), yb = qmul(ldQr(vb + i * 4), mu_bar);
    stQr(va + i * 4, qsub(qscale(ya, c), qscale(yb, s)));
    stQr(vb + i * 4, qadd(qscale(ya, s), qscale(yb, c)));
  }
  __syncthreads();
  return true;
}

template <int R>
__global__ void __cluster_dims__(kRCl, 1, 1) __launch_bounds__(kRThreads, 1)
    k_robust_jacobi(double* A, int64_t p, int64_t q, double* V, double* Q, int64_t ldq, double* F, int64_t ldf,
                    double cutoff_scale, double cutoff_abs, const unsigned* status, unsigned gate_bit) {
  if (!(*status & gate_bit)) return;  // the fast path held (same word in all 16 CTAs)
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  const int tid = threadIdx.x;
  __shared__ double red[kRWarps][6];
  __shared__ int s_rot;
  __shared__ double s_max;
  // V = I, columns c, c + 16, ...
  for (int64_t j = c; j < q; j += kRCl)
    for (int64_t i = tid; i < q; i += kRThreads) stQr(V + (j * q + i) * 4, Quat{i == j ? 1.0 : 0.0, 0.0, 0.0, 0.0});
  const int64_t nn = q + (q & 1), npairs = nn / 2;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    if (tid == 0) s_rot = 0;
    cl.sync();
    int rot = 0;
    for (int64_t rnd = 0; rnd < nn - 1; ++rnd) {
      for (int64_t pk = c; pk < npairs; pk += kRCl) {
        int64_t a, b;
        pair_of(pk, nn, rnd, a, b);
        if (a >= q || b >= q) continue;
        rot |= rotate_pair<R>(A, p, V, q, a, b, red) ? 1 : 0;
      }
      cl.sync();  // the next round pairs columns this round's CTAs rotated (global memory)
    }
    if (tid == 0 && rot) s_rot = 1;
    cl.sync();
    int any = 0;
    for (int r = 0; r < kRCl; ++r) any |= *cl.map_shared_rank(&s_rot, r);
    cl.sync();  // every CTA has read the votes before the next sweep resets them
    if (!any) break;
  }
  // singular values of the own columns, then sigma_max over the cluster
  double mx = 0.0;
  for (int64_t j = c; j < q; j += kRCl) {
    const double* cj = A + j * p * 4;
    double s2 = 0.0;
    for (int64_t i = tid; i < p; i += kRThreads) s2 += qnorm2(ldQr(cj + i * 4));
    s2 = warp_sum(s2);
    if ((tid & 31) == 0) red[tid >> 5][0] = s2;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < kRWarps; ++w) tot += red[w][0];
    __syncthreads();
    mx = fmax(mx, sqrt(tot));
  }
  if (tid == 0) s_max = mx;
  cl.sync();
  double smax = 0.0;
  for (int r = 0; r < kRCl; ++r) smax = fmax(smax, *cl.map_shared_rank(&s_max, r));
  cl.sync();
  const double cutoff = cutoff_abs >= 0.0 ? cutoff_abs : cutoff_scale * smax;
  // Q = W (row-major p x q) and F = V Sigma^+ (row-major q x q), own columns
  for (int64_t j = c; j < q; j += kRCl) {
    const double* cj = A + j * p * 4;
    double s2 = 0.0;
    for (int64_t i = tid; i < p; i += kRThreads) s2 += qnorm2(ldQr(cj + i * 4));
    s2 = warp_sum(s2);
    if ((tid & 31) == 0) red[tid >> 5][0] = s2;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < kRWarps; ++w) tot += red[w][0];
    __syncthreads();
    const double sig = sqrt(tot);
    const bool keep = smax > 0.0 && sig > cutoff;
    const double inv = keep ? 1.0 / sig : 0.0;
    for (int64_t i = tid; i < p; i += kRThreads) stQr(Q + (i * ldq + j) * 4, qscale(ldQr(cj + i * 4), inv));
    const double* vj = V + j * q * 4;
    for (int64_t i = tid; i < q; i += kRThreads) stQr(F + (i * ldf + j) * 4, qscale(ldQr(vj + i * 4), inv));
  }
  cl.sync();  // no CTA leaves while a peer may still read its shared memory
}

template <int R>
void launch_rj(double* A, int64_t p, int64_t q, double* V, double* Q, int64_t ldq, double* F, int64_t ldf,
               double cutoff_scale, double cutoff_abs, const unsigned* status, unsigned gate_bit, cudaStream_t st) {
  static std::atomic<unsigned> attr{0};
  if (first_on_device(attr)) cudaFuncSetAttribute(k_robust_jacobi<R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  ++::qcur::g_launches;
  k_robust_jacobi<R><<<kRCl, kRThreads, 0, st>>>(A, p, q, V, Q, ldq, F, ldf, cutoff_scale, cutoff_abs, status,
                                                 gate_bit);
}

}  // namespace

void launch_robust_jacobi(double* Zcm, int64_t p, int64_t q, double* Vcm, double* Q, int64_t ldq, double* F,
                          int64_t ldf, double cutoff_scale, double cutoff_abs, const unsigned* status, unsigned gate_bit,
                          cudaStream_t st) {
  // R = 1 keeps a thread's rows of the pair in registers; larger R spills at 1024 threads (64 registers), so
  // taller blocks stream their rows twice (measured: cfg2 p = 4000 streaming 520 ms, R = 4 slower)
  if (p <= kRThreads)
    launch_rj<1>(Zcm, p, q, Vcm, Q, ldq, F, ldf, cutoff_scale, cutoff_abs, status, gate_bit, st);
  else
    launch_rj<0>(Zcm, p, q, Vcm, Q, ldq, F, ldf, cutoff_scale, cutoff_abs, status, gate_bit, st);
}

}  // namespace qcur
