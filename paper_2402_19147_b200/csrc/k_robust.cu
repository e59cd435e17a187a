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

#include <atomic>
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

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

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


// ---------------------------------------------------------------------------
// Householder QR of Z (p x q, column-major, p >= q) on one 16-CTA cluster, then the explicit
// Q = H_0 ... H_{q-1} [I; 0].  CTA c owns the contiguous rows [c P, (c+1) P) of every column.
// Step k: the column norm below the diagonal (cluster sum of the CTAs' partial sums, read through
// distributed shared memory in rank order: every CTA gets the same bits), the reflector
// H = I - beta v v^H with v = x - alpha e1, alpha = -(x1/|x1|) ||x|| (every CTA forms alpha and
// beta itself from the shared x1), the products w_j = beta v^H z_j of the trailing columns
// (per-CTA partials, reduced by their owner CTA j % 16 and gathered back), and the update
// z_j -= v w_j of the CTA's own rows.  T (upper triangular, column-major) collects alpha and
// the updated row k.  The same reflectors, applied backwards to [I; 0], give Q.
// ---------------------------------------------------------------------------
constexpr int kHThreads = 512, kHWarps = kHThreads / 32;

struct HqrArgs {
  double* Zcm;  // p x q column-major; overwritten with the reflectors v (column k from row k down)
  int64_t p, q;
  double* betas;  // [q]
  double* Ycm;    // p x q column-major workspace (Q before the row-major copy)
  double* Q;      // p x q row-major, leading dimension ldq
  int64_t ldq;
  double* Tcm;  // q x q column-major: the triangular factor
  const unsigned* status;
  unsigned gate_bit;
};

// both blocks of a factorization step in one launch: cluster b = blockIdx.x / kRCl takes A.a[b]
struct HqrPair {
  HqrArgs a[2];
};

__global__ void __cluster_dims__(kRCl, 1, 1) __launch_bounds__(kHThreads, 1) k_robust_hqr(const __grid_constant__ HqrPair P) {
  const HqrArgs& A = P.a[blockIdx.x / kRCl];
  if (!(*A.status & A.gate_bit)) return;
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t p = A.p, q = A.q;
  const int64_t rows_per = (p + kRCl - 1) / kRCl;
  const int64_t r0 = (int64_t)c * rows_per < p ? (int64_t)c * rows_per : p;
  const int64_t r1 = r0 + rows_per < p ? r0 + rows_per : p;
  double* Z = A.Zcm;
  double* Y = A.Ycm;
  extern __shared__ __align__(32) double hs[];
  double* part = hs;            // [q] quaternions: this CTA's partial products
  double* red = part + 4 * q;   // [q]: the cluster sums of the entries this CTA owns (j % 16 == c)
  double* wv = red + 4 * q;     // [q]: every cluster sum, times beta
  __shared__ double s_warp[kHWarps];
  __shared__ double s_part;

  // sum over the cluster of one double per CTA (the same bits everywhere)
  auto cluster_sum = [&](double v) -> double {
    v = warp_sum(v);
    if (lane == 0) s_warp[warp] = v;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int w = 0; w < kHWarps; ++w) t += s_warp[w];
      s_part = t;
    }
    cl.sync();
    double tot = 0.0;
    for (int r = 0; r < kRCl; ++r) tot += *cl.map_shared_rank(&s_part, r);
    return tot;
  };
  // wv[j] = beta * (sum over the cluster of part[j]) for j in [j0, q)
  auto cluster_vec = [&](int64_t j0, double beta) {
    cl.sync();  // every CTA's partials are written
    for (int64_t j = j0 + ((c - j0 % kRCl) + kRCl) % kRCl + (int64_t)tid * kRCl; j < q; j += (int64_t)kHThreads * kRCl) {
      Quat t = qzero();
      for (int r = 0; r < kRCl; ++r) t = qadd(t, ldQr(cl.map_shared_rank(part, r) + j * 4));
      stQr(red + j * 4, t);
    }
    cl.sync();  // the owners' sums are written
    for (int64_t j = j0 + tid; j < q; j += kHThreads)
      stQr(wv + j * 4, qscale(ldQr(cl.map_shared_rank(red, (int)(j % kRCl)) + j * 4), beta));
    __syncthreads();
  };

  for (int64_t t = (int64_t)c * kHThreads + tid; t < q * q; t += (int64_t)kRCl * kHThreads) stQr(A.Tcm + t * 4, qzero());
  for (int64_t k = 0; k < q; ++k) {
    const int64_t i0 = r0 > k ? r0 : k;  // own rows at or below the diagonal
    double pn = 0.0;
    for (int64_t i = i0 + tid; i < r1; i += kHThreads) pn += qnorm2(ldQr(Z + (k * p + i) * 4));
    const double norm2 = cluster_sum(pn);  // includes a cluster barrier: row k of the last step is written
    const Quat x1 = ldQr(Z + (k * p + k) * 4);
    Quat alpha = qzero(), vk = qzero();
    double beta = 0.0;
    if (norm2 > 0.0) {
      const double nrm = sqrt(norm2), a1 = sqrt(qnorm2(x1));
      alpha = a1 > 0.0 ? qscale(x1, -nrm / a1) : Quat{-nrm, 0.0, 0.0, 0.0};
      vk = qsub(x1, alpha);
      beta = 1.0 / (norm2 + nrm * a1);
    }
    const bool own_k = k >= r0 && k < r1;
    if (c == 0 && tid == 0) {
      A.betas[k] = beta;
      stQr(A.Tcm + (k * q + k) * 4, alpha);
    }
    if (beta != 0.0 && k + 1 < q) {
      for (int64_t j = k + 1 + warp; j < q; j += kHWarps) {
        Quat w = qzero();
        for (int64_t i = i0 + lane; i < r1; i += 32) qfma_conj(w, i == k ? vk : ldQr(Z + (k * p + i) * 4), ldQr(Z + (j * p + i) * 4));
        w = warp_sum(w);
        if (lane == 0) stQr(part + j * 4, w);
      }
      cluster_vec(k + 1, beta);
      for (int64_t j = k + 1 + warp; j < q; j += kHWarps) {
        const Quat wj = ldQr(wv + j * 4);
        for (int64_t i = i0 + lane; i < r1; i += 32) {
          double* zij = Z + (j * p + i) * 4;
          stQr(zij, qsub(ldQr(zij), qmul(i == k ? vk : ldQr(Z + (k * p + i) * 4), wj)));
        }
      }
      __syncthreads();
    } else {
      cl.sync();  // keep the barrier count uniform with the other branch's reduction
      cl.sync();
    }
    if (own_k) {
      for (int64_t j = k + 1 + tid; j < q; j += kHThreads) stQr(A.Tcm + (j * q + k) * 4, ldQr(Z + (j * p + k) * 4));
      __syncthreads();
      if (tid == 0) stQr(Z + (k * p + k) * 4, vk);  // every CTA has read x1 (two barriers ago)
    }
  }
  // Q = H_0 ... H_{q-1} [I; 0], backwards
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = r0 + tid; i < r1; i += kHThreads) stQr(Y + (j * p + i) * 4, Quat{i == j ? 1.0 : 0.0, 0.0, 0.0, 0.0});
  cl.sync();  // every v_k and beta_k is written
  for (int64_t k = q - 1; k >= 0; --k) {
    const double beta = A.betas[k];
    if (beta == 0.0) continue;  // the same in every CTA
    const int64_t i0 = r0 > k ? r0 : k;
    for (int64_t j = k + warp; j < q; j += kHWarps) {
      Quat w = qzero();
      for (int64_t i = i0 + lane; i < r1; i += 32) qfma_conj(w, ldQr(Z + (k * p + i) * 4), ldQr(Y + (j * p + i) * 4));
      w = warp_sum(w);
      if (lane == 0) stQr(part + j * 4, w);
    }
    cluster_vec(k, beta);
    for (int64_t j = k + warp; j < q; j += kHWarps) {
      const Quat wj = ldQr(wv + j * 4);
      for (int64_t i = i0 + lane; i < r1; i += 32) {
        double* yij = Y + (j * p + i) * 4;
        stQr(yij, qsub(ldQr(yij), qmul(ldQr(Z + (k * p + i) * 4), wj)));
      }
    }
    __syncthreads();
  }
  // row-major copy of the own rows
  for (int64_t t = tid; t < (r1 - r0) * q; t += kHThreads) {
    const int64_t i = r0 + t / q, j = t % q;
    stQr(A.Q + (i * A.ldq + j) * 4, ldQr(Y + (j * p + i) * 4));
  }
  cl.sync();  // no CTA leaves while a peer may still read its shared memory
}

// ---------------------------------------------------------------------------
// pinv of the q x q triangular factor, F = T^+ (row-major), by one-sided Jacobi on T's columns with
// one WARP per column pair (q <= kSmallQ: a lane keeps <= 8 rows of each column in registers), all
// pairs of a round at once on the 16-CTA cluster (256 threads each), one cluster barrier per round.
// Then sigma_j = ||t_j||, the reference's cutoff, and F = sum_{sigma_j > cutoff} v_j t_j^H / sigma_j^2.
// ---------------------------------------------------------------------------
constexpr int kSmallQ = 256, kSThreads = 256, kSWarps = kSThreads / 32, kSR = kSmallQ / 32;

struct TpinvArgs {
  double* Tcm;
  int64_t q;
  double* Vcm;
  double* F;
  int64_t ldf;
  double cutoff_scale, cutoff_abs;
  const unsigned* status;
  unsigned gate_bit;
};
struct TpinvPair {
  TpinvArgs a[2];
};

__global__ void __cluster_dims__(kRCl, 1, 1) __launch_bounds__(kSThreads, 1)
    k_robust_tpinv(const __grid_constant__ TpinvPair P) {
  const TpinvArgs& A = P.a[blockIdx.x / kRCl];
  double* Tcm = A.Tcm;
  const int64_t q = A.q;
  double* Vcm = A.Vcm;
  double* F = A.F;
  const int64_t ldf = A.ldf;
  const double cutoff_scale = A.cutoff_scale, cutoff_abs = A.cutoff_abs;
  const unsigned* status = A.status;
  const unsigned gate_bit = A.gate_bit;
  if (!(*status & gate_bit)) return;
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gw = c * kSWarps + warp;  // this warp's pair index in a round
  __shared__ int s_rot;
  __shared__ double s_max;
  double* sig = Vcm + q * q * 4;  // [q] sigma_j
  for (int64_t t = (int64_t)c * kSThreads + tid; t < q * q; t += (int64_t)kRCl * kSThreads) {
    const int64_t j = t / q, i = t - j * q;
    stQr(Vcm + t * 4, Quat{i == j ? 1.0 : 0.0, 0.0, 0.0, 0.0});
  }
  const int64_t nn = q + (q & 1), npairs = nn / 2;
  const double tol = fmax(4.0, sqrt((double)q)) * DBL_EPSILON;
  for (int sweep = 0; sweep < kMaxSweeps && q > 1; ++sweep) {
    if (tid == 0) s_rot = 0;
    cl.sync();
    int rot = 0;
    for (int64_t rnd = 0; rnd < nn - 1; ++rnd) {
      int64_t a = 0, b = 0;
      if (gw < npairs) pair_of(gw, nn, rnd, a, b);
      if (gw < npairs && a < q && b < q) {
        double* ca = Tcm + a * q * 4;
        double* cb = Tcm + b * q * 4;
        Quat xa[kSR], xb[kSR];
        double al = 0.0, be = 0.0;
        Quat g = qzero();
#pragma unroll
        for (int r = 0; r < kSR; ++r) {
          const int64_t i = lane + 32 * r;
          xa[r] = i < q ? ldQr(ca + i * 4) : qzero();
          xb[r] = i < q ? ldQr(cb + i * 4) : qzero();
          al += qnorm2(xa[r]);
          be += qnorm2(xb[r]);
          qfma_conj(g, xa[r], xb[r]);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        g = warp_sum(g);
        const double gn = sqrt(qnorm2(g));
        if (gn > tol * sqrt(al) * sqrt(be) && al > 0.0 && be > 0.0) {
          rot = 1;
          const Quat mu_bar = qconj(qscale(g, 1.0 / gn));
          const double zeta = (be - al) / (2.0 * gn);
          const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
#pragma unroll
          for (int r = 0; r < kSR; ++r) {
            const int64_t i = lane + 32 * r;
            if (i < q) {
              const Quat pb = qmul(xb[r], mu_bar);
              stQr(ca + i * 4, qsub(qscale(xa[r], cs), qscale(pb, sn)));
              stQr(cb + i * 4, qadd(qscale(xa[r], sn), qscale(pb, cs)));
            }
          }
          double* va = Vcm + a * q * 4;
          double* vb = Vcm + b * q * 4;
#pragma unroll
          for (int r = 0; r < kSR; ++r) {
            const int64_t i = lane + 32 * r;
            if (i < q) {
              const Quat ya = ldQr(va + i * 4), yb = qmul(ldQr(vb + i * 4), mu_bar);
              stQr(va + i * 4, qsub(qscale(ya, cs), qscale(yb, sn)));
              stQr(vb + i * 4, qadd(qscale(ya, sn), qscale(yb, cs)));
            }
          }
        }
      }
      cl.sync();  // the next round pairs columns this round rotated (global memory, cluster scope)
    }
    if (rot && lane == 0) atomicOr(&s_rot, 1);
    cl.sync();
    int any = 0;
    for (int r = 0; r < kRCl; ++r) any |= *cl.map_shared_rank(&s_rot, r);
    cl.sync();  // every CTA has read the votes before the next sweep resets them
    if (!any) break;
  }
  // sigma_j, sigma_max (one warp per column), the cutoff
  double mx = 0.0;
  for (int64_t j = gw; j < q; j += (int64_t)kRCl * kSWarps) {
    double s2 = 0.0;
    for (int64_t i = lane; i < q; i += 32) s2 += qnorm2(ldQr(Tcm + (j * q + i) * 4));
    s2 = warp_sum(s2);
    if (lane == 0) sig[j] = sqrt(s2);
    mx = fmax(mx, sqrt(s2));
  }
  mx = warp_max(mx);
  if (tid == 0) s_max = 0.0;
  __syncthreads();
  if (lane == 0) atomicMax(reinterpret_cast<unsigned long long*>(&s_max), (unsigned long long)__double_as_longlong(mx));
  cl.sync();  // sigma of every column and each CTA's maximum are written
  double smax = 0.0;
  for (int r = 0; r < kRCl; ++r) smax = fmax(smax, *cl.map_shared_rank(&s_max, r));
  const double cutoff = cutoff_abs >= 0.0 ? cutoff_abs : cutoff_scale * smax;
  // F[i][k] = sum_j v_ij conj(t_kj) / sigma_j^2 over the kept j; CTA c takes rows i = c, c + 16, ...
  for (int64_t e = (int64_t)c * kSThreads + tid; e < q * q; e += (int64_t)kRCl * kSThreads) {
    const int64_t i = e / q, kk = e - i * q;
    Quat acc = qzero();
    for (int64_t j = 0; j < q; ++j) {
      const double sj = sig[j];
      if (!(smax > 0.0 && sj > cutoff)) continue;
      acc = qadd(acc, qscale(qmul(ldQr(Vcm + (j * q + i) * 4), qconj(ldQr(Tcm + (j * q + kk) * 4))), 1.0 / (sj * sj)));
    }
    stQr(F + (i * ldf + kk) * 4, acc);
  }
  cl.sync();  // no CTA leaves while a peer may still read its shared memory
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

namespace qcur {

size_t robust_hqr_smem(int64_t q) { return (size_t)3 * 4 * q * sizeof(double); }

bool robust_qr_supported(int64_t p, int64_t q) {
  return q <= kSmallQ && p >= q && robust_hqr_smem(q) <= 200 * 1024;
}

void launch_robust_qr_pinv_multi(const RobustQrJob* J, int nj, cudaStream_t st) {
  static std::atomic<unsigned> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_robust_hqr, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_robust_hqr, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(k_robust_tpinv, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  }
  HqrPair H{};
  TpinvPair T{};
  size_t smem = 0;
  for (int k = 0; k < nj; ++k) {
    const RobustQrJob& a = J[k];
    H.a[k] = HqrArgs{a.Zcm, a.p, a.q, a.betas, a.Ycm, a.Q, a.ldq, a.Tcm, a.status, a.gate_bit};
    T.a[k] = TpinvArgs{a.Tcm, a.q, a.Vcm, a.F, a.ldf, a.cutoff_scale, a.cutoff_abs, a.status, a.gate_bit};
    const size_t b = robust_hqr_smem(a.q);
    smem = b > smem ? b : smem;
  }
  ++::qcur::g_launches;
  k_robust_hqr<<<kRCl * nj, kHThreads, smem, st>>>(H);
  ++::qcur::g_launches;
  k_robust_tpinv<<<kRCl * nj, kSThreads, 0, st>>>(T);
}

void launch_robust_qr_pinv(double* Zcm, int64_t p, int64_t q, double* betas, double* Ycm, double* Q, int64_t ldq,
                           double* Tcm, double* Vcm, double* F, int64_t ldf, double cutoff_scale, double cutoff_abs,
                           const unsigned* status, unsigned gate_bit, cudaStream_t st) {
  RobustQrJob j{Zcm, p, q, betas, Ycm, Q, ldq, Tcm, Vcm, F, ldf, cutoff_scale, cutoff_abs, status, gate_bit};
  launch_robust_qr_pinv_multi(&j, 1, st);
}

}  // namespace qcur
