// Cholesky-factor inverse X = L^{-1} of small Hermitian quaternion Gram
// matrices G = L L^H on one 16-CTA thread-block cluster (distributed shared
// memory), for the CholeskyQR2 fast path of pseudoinverse (replacement of
// linalg.py:346-362; see k_dense.cu).
//
// Everything lives on chip.  CTA c owns Gram ROWS i = c, c+16, ... (Cholesky,
// right-looking) and inverse COLUMNS k = c, c+16, ... (W -> X).  Step j:
//   1. every CTA holds a replicated running diagonal and forms l_jj itself;
//      owners scale their column-j Gram entries (L_ij, i > j) and store them
//      into every CTA's column buffer (DSMEM);
//   2. the column arrives by st.async with mbarrier complete_tx (plus one remote
//      arrive per producer), so each CTA waits only on its own mbarrier — no
//      cluster-wide barrier or GPU-scope fence per step (both cost ~2 us/step
//      when profiled);
//   3. Cholesky: own rows i > j:  G_ik -= L_ij conj(L_kj),  j < k <= i;
//      inverse: own columns k <= j: X_jk = W_jk / l_jj, then W_ik -= L_ij X_jk
//      for i > j.
// Column j of L is the only data exchanged: the column-cyclic inverse needs no
// row broadcast (profiled: the earlier row-cyclic inverse spent 40% of its
// time waiting on DSMEM pulls of X rows).  The two problems of a QMCUR step
// (C and R^H) run as two clusters of one launch.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace qcur {

namespace {
constexpr int kCl = 16;  // CTAs per cluster (non-portable size, supported on B200)
constexpr int kThreads = 512;
constexpr int kClusterQMax = 304;  // compact triangles + 3 column buffers within 227 KB of smem

__device__ __forceinline__ Quat ldQ(const double* p) { return *reinterpret_cast<const Quat*>(p); }
__device__ __forceinline__ void stQ(double* p, const Quat& q) { *reinterpret_cast<Quat*>(p) = q; }

struct CholProblems {
  CholJob p[2];
  int64_t q;
  unsigned* status;
};

__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t mapa(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_init(uint64_t* mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, unsigned parity) {
  const uint32_t a = smem_u32(mb);
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t remote_mb) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_mb) : "memory");
}
// 32-byte quaternion into a peer's shared memory, completing 32 tx bytes on its mbarrier
__device__ __forceinline__ void st_async_quat(uint32_t remote, const Quat& v, uint32_t remote_mb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(remote),
               "d"(v.w), "d"(v.x), "r"(remote_mb)
               : "memory");
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(remote + 16),
               "d"(v.y), "d"(v.z), "r"(remote_mb)
               : "memory");
}
}  // namespace

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kThreads, 1) k_chol_inv_cluster(CholProblems P) {
  const int c = (int)cg::this_cluster().block_rank();
  const CholJob pr = P.p[blockIdx.x / kCl];
  const int q = (int)P.q;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kWarps = kThreads / 32;
  const int nown = (q - c + kCl - 1) / kCl;  // own rows i = c + 16 s  and own columns k = c + 16 u
  const int nmax = (q + kCl - 1) / kCl;      // identical layout in every CTA: DSMEM offsets must agree
  // Fixed-offset region first (identical in every CTA: DSMEM targets), then the
  // CTA's own triangles stored compactly: Gram row i = c + 16 s keeps k <= i
  // (rowbase(s) + k), inverse column k = c + 16 u keeps i >= k (colbase(u) + i - k).
  extern __shared__ __align__(32) double sm[];
  double* colbuf = sm;                           // [3][q] quaternions: columns of L in flight
  double* diag = colbuf + 3 * (size_t)q * 4;     // [q] replicated running diagonal
  uint64_t* mbar = reinterpret_cast<uint64_t*>(diag + q + (q & 1));  // [3] one per column buffer
  double* rows = reinterpret_cast<double*>(mbar + 4);
  auto rowbase = [&](int s) -> size_t { return (size_t)s * (c + 1) + (size_t)8 * s * (s - 1); };
  auto colbase = [&](int u) -> size_t { return (size_t)u * (q - c) - (size_t)8 * u * (u - 1); };
  double* wcol = rows + rowbase(nown) * 4;
  (void)nmax;

  for (int s = 0; s < nown; ++s) {
    const int i = c + kCl * s;
    double* row = rows + rowbase(s) * 4;
    for (int k = tid; k <= i; k += kThreads) stQ(row + (size_t)k * 4, ldQ(pr.G + ((size_t)i * q + k) * 4));
    double* col = wcol + colbase(s) * 4;  // own column k = i
    for (int r = i + tid; r < q; r += kThreads) stQ(col + (size_t)(r - i) * 4, Quat{r == i ? 1.0 : 0.0, 0.0, 0.0, 0.0});
  }
  for (int i = tid; i < q; i += kThreads) diag[i] = pr.G[((size_t)i * q + i) * 4];
  if (tid == 0) {
    for (int k = 0; k < 3; ++k) mbar_init(&mbar[k], kCl + 1);  // 16 producer arrives + local expect_tx
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_barrier();

  // Send column j of L (entries of own rows i > j, already updated through step
  // j-1) to every CTA; returns false (in every CTA alike) if l_jj breaks down.
  auto produce = [&](int j) -> bool {
    const double d = diag[j];
    if (!(d > 0.0) || !isfinite(d)) return false;
    const double inv = 1.0 / sqrt(d);
    const int b = j % 3;
    if (tid == 0) mbar_expect_tx(&mbar[b], 32u * (unsigned)(q - 1 - j));
    const uint32_t cb_u = smem_u32(colbuf + (size_t)b * q * 4), mb_u = smem_u32(&mbar[b]);
    for (int t = tid; t < nown * kCl; t += kThreads) {
      const int s = t / kCl, dst = t - s * kCl;
      const int i = c + kCl * s;
      if (i <= j) continue;
      st_async_quat(mapa(cb_u + 32u * (unsigned)i, dst), qscale(ldQ(rows + (rowbase(s) + j) * 4), inv),
                    mapa(mb_u, dst));
    }
    if (tid < kCl) mbar_arrive_remote(mapa(mb_u, tid));
    return true;
  };

  bool ok = produce(0);
  for (int j = 0; ok && j < q; ++j) {
    const int b = j % 3;
    double* cb = colbuf + (size_t)b * q * 4;
    mbar_wait(&mbar[b], (unsigned)(j / 3) & 1u);
    const double inv = 1.0 / sqrt(diag[j]);
    // look-ahead: finish column j+1 first and send it, so its transfer overlaps
    // the bulk of this step's update
    if (j + 1 < q) {
      const Quat lj1 = ldQ(cb + (size_t)(j + 1) * 4);
      for (int s = tid; s < nown; s += kThreads) {
        const int i = c + kCl * s;
        if (i <= j + 1) continue;
        double* e = rows + (rowbase(s) + j + 1) * 4;
        stQ(e, qsub(ldQ(e), qmul(ldQ(cb + (size_t)i * 4), qconj(lj1))));
      }
      if (tid == 0) diag[j + 1] = diag[j + 1] - qnorm2(lj1);
      __syncthreads();
      ok = produce(j + 1);
    }
    // bulk Cholesky update (k = j+1 done above): one warp per own row
    for (int s = warp; s < nown; s += kWarps) {
      const int i = c + kCl * s;
      if (i <= j + 1) continue;
      const Quat lij = ldQ(cb + (size_t)i * 4);
      double* row = rows + rowbase(s) * 4;
      int k = j + 2 + lane;
      for (; k + 32 <= i; k += 64) {  // two independent updates in flight
        const Quat a0 = ldQ(row + (size_t)k * 4), b0 = ldQ(cb + (size_t)k * 4);
        const Quat a1 = ldQ(row + (size_t)(k + 32) * 4), b1 = ldQ(cb + (size_t)(k + 32) * 4);
        stQ(row + (size_t)k * 4, qsub(a0, qmul(lij, qconj(b0))));
        stQ(row + (size_t)(k + 32) * 4, qsub(a1, qmul(lij, qconj(b1))));
      }
      if (k <= i) stQ(row + (size_t)k * 4, qsub(ldQ(row + (size_t)k * 4), qmul(lij, qconj(ldQ(cb + (size_t)k * 4)))));
    }
    // inverse, own columns k <= j: X_jk = W_jk / l_jj;  W_ik -= L_ij X_jk (i > j)
    for (int u = warp; u < nown; u += kWarps) {
      const int k = c + kCl * u;
      if (k > j) continue;
      double* w = wcol + colbase(u) * 4 - (size_t)k * 4;  // w + i*4 addresses W_ik (i >= k)
      const Quat xjk = qscale(ldQ(w + (size_t)j * 4), inv);
      if (lane == 0) stQ(w + (size_t)j * 4, xjk);
      int i = j + 1 + lane;
      for (; i + 32 < q; i += 64) {
        const Quat a0 = ldQ(w + (size_t)i * 4), b0 = ldQ(cb + (size_t)i * 4);
        const Quat a1 = ldQ(w + (size_t)(i + 32) * 4), b1 = ldQ(cb + (size_t)(i + 32) * 4);
        stQ(w + (size_t)i * 4, qsub(a0, qmul(b0, xjk)));
        stQ(w + (size_t)(i + 32) * 4, qsub(a1, qmul(b1, xjk)));
      }
      if (i < q) stQ(w + (size_t)i * 4, qsub(ldQ(w + (size_t)i * 4), qmul(ldQ(cb + (size_t)i * 4), xjk)));
    }
    for (int i = j + 2 + tid; i < q; i += kThreads) diag[i] = diag[i] - qnorm2(ldQ(cb + (size_t)i * 4));
    __syncthreads();
  }
  if (!ok) {  // identical in every CTA (replicated diagonal): no transfer is left in flight
    if (c == 0 && tid == 0) atomicOr(P.status, pr.fail_bit);
    cluster_barrier();
    return;
  }
  // X_ik for own columns k (i >= k), zero above the diagonal
  for (int u = 0; u < nown; ++u) {
    const int k = c + kCl * u;
    const double* w = wcol + colbase(u) * 4;
    for (int i = tid; i < q; i += kThreads) stQ(pr.X + ((size_t)i * q + k) * 4, i >= k ? ldQ(w + (size_t)(i - k) * 4) : qzero());
  }
  cluster_barrier();
}

int chol_cluster_qmax() { return kClusterQMax; }

// dynamic shared memory of the CTA with the largest triangles (rank 0)
static size_t chol_cluster_smem(int64_t q) {
  size_t best = 0;
  for (int c = 0; c < kCl; ++c) {
    const int64_t nown = (q - c + kCl - 1) / kCl;
    const int64_t rows = nown * (c + 1) + 8 * nown * (nown - 1);
    const int64_t cols = nown * (q - c) - 8 * nown * (nown - 1);
    const size_t b = (size_t)(3 * q * 4 + q + (q & 1) + 4 + 4 * (rows + cols)) * sizeof(double);
    best = b > best ? b : best;
  }
  return best;
}

void launch_chol_inv_cluster(const CholJob* jobs, int njobs, int64_t q, unsigned* status, cudaStream_t st) {
  CholProblems P{};
  for (int k = 0; k < njobs && k < 2; ++k) P.p[k] = jobs[k];
  P.q = q;
  P.status = status;
  const size_t smem = chol_cluster_smem(q);
  static std::atomic<unsigned> set{0};
  if (first_on_device(set)) {
    cudaFuncSetAttribute(k_chol_inv_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_chol_inv_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  ++::qcur::g_launches;
  k_chol_inv_cluster<<<kCl * njobs, kThreads, smem, st>>>(P);
}

}  // namespace qcur
