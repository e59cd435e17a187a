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

#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace qcur {

namespace {
constexpr int kCl = 16;  // CTAs per cluster (non-portable size, supported on B200)
#ifndef QCUR_CHOL_THREADS  // build-time variant for A/B timing
#define QCUR_CHOL_THREADS 256
#endif
constexpr int kThreads = QCUR_CHOL_THREADS;
constexpr int kClusterQMax = 304;  // compact triangles + 3 column buffers within 227 KB of smem
constexpr bool kCholTwoColumnDefault = false;
#ifndef QCUR_CHOL_BATCH  // entries per lane loaded before they are updated (V2 bulk)
#define QCUR_CHOL_BATCH 2
#endif
constexpr int kCB = QCUR_CHOL_BATCH;  // two columns per cluster exchange (QCUR_CHOL_B2)

__device__ __forceinline__ Quat ldQ(const double* p) { return *reinterpret_cast<const Quat*>(p); }
__device__ __forceinline__ void stQ(double* p, const Quat& q) { *reinterpret_cast<Quat*>(p) = q; }

#ifdef QCUR_CHOL_TRACE  // per-step phase clocks of CTA 0, thread 0 (tools/test_chol_cluster.cu)
__device__ long long g_chol_trace[512][6];
#define CHOL_T(j, k) \
  if (blockIdx.x == 0 && threadIdx.x == 0 && (j) < 512) g_chol_trace[j][k] = clock64();
#else
#define CHOL_T(j, k)
#endif

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
__device__ __forceinline__ void mbar_arrive(uint64_t* mb) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(mb)) : "memory");
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

// V2: (a) the look-ahead column is formed and sent in one pass by the sending threads themselves
// (no write-back to the Gram row, no barrier between them; the final pivot of the next step is kept
// in a local array), (b) the bulk updates are spread over all warps as work items (own Cholesky rows,
// own inverse columns), each lane loading its next kCB entries before updating them (the one-warp-per-
// row loops stored and reloaded through possibly-aliasing shared-memory pointers, serialising every
// iteration: measured 1.8k cycles per step at q = 200, tools/test_chol_cluster.cu with
// QCUR_CHOL_TRACE).  Same operations on every element in the same order: bit-identical factors.
template <bool V2>
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
  double* dfin = wcol + colbase(nown) * 4;  // [q] final pivots (V2, local)
  (void)nmax;

  for (int s = 0; s < nown; ++s) {
    const int i = c + kCl * s;
    double* row = rows + rowbase(s) * 4;
    for (int k = tid; k <= i; k += kThreads) stQ(row + (size_t)k * 4, ldQ(pr.G + ((size_t)i * q + k) * 4));
    double* col = wcol + colbase(s) * 4;  // own column k = i
    for (int r = i + tid; r < q; r += kThreads) stQ(col + (size_t)(r - i) * 4, Quat{r == i ? 1.0 : 0.0, 0.0, 0.0, 0.0});
  }
  for (int i = tid; i < q; i += kThreads) diag[i] = pr.G[((size_t)i * q + i) * 4];
  if (V2 && tid == 0) dfin[0] = pr.G[0];
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
  double inv_cur = V2 ? 1.0 / sqrt(pr.G[0]) : 0.0;  // V2: 1 / l_jj of the current step (G[0] > 0 when ok)
  for (int j = 0; ok && j < q; ++j) {
    const int b = j % 3;
    double* cb = colbuf + (size_t)b * q * 4;
    CHOL_T(j, 0)
    Quat pre = qzero();  // V2: this sender's Gram entry (own row, column j+1), final since the last bulk
    if constexpr (V2) {
      if (tid < nown * kCl && j + 1 < q) {
        const int s = tid / kCl;
        if (c + kCl * s > j + 1) pre = ldQ(rows + (rowbase(s) + j + 1) * 4);
      }
    }
    mbar_wait(&mbar[b], (unsigned)(j / 3) & 1u);
    CHOL_T(j, 1)
    if constexpr (!V2) {
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
        CHOL_T(j, 2)
        ok = produce(j + 1);
      }
      CHOL_T(j, 3)
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
    } else {
      const double inv = inv_cur;
      // look-ahead: the senders form column j+1 of their rows themselves and send it at once
      if (j + 1 < q) {
        const Quat lj1 = ldQ(cb + (size_t)(j + 1) * 4);
        const double d1 = diag[j + 1] - qnorm2(lj1);
        if (!(d1 > 0.0) || !isfinite(d1)) {
          ok = false;  // every CTA alike (replicated diagonal)
        } else {
          const double inv1 = 1.0 / sqrt(d1);
          inv_cur = inv1;
          const int b1 = (j + 1) % 3;
          if (tid == 0) {
            dfin[j + 1] = d1;
            mbar_expect_tx(&mbar[b1], 32u * (unsigned)(q - 2 - j));
          }
          const uint32_t cb_u = smem_u32(colbuf + (size_t)b1 * q * 4), mb_u = smem_u32(&mbar[b1]);
          for (int t = tid; t < nown * kCl; t += kThreads) {
            const int s = t / kCl, dst = t - s * kCl;
            const int i = c + kCl * s;
            if (i <= j + 1) continue;
            const Quat v = qsub(t == tid ? pre : ldQ(rows + (rowbase(s) + j + 1) * 4), qmul(ldQ(cb + (size_t)i * 4), qconj(lj1)));
            st_async_quat(mapa(cb_u + 32u * (unsigned)i, dst), qscale(v, inv1), mapa(mb_u, dst));
          }
          if (tid < kCl) mbar_arrive_remote(mapa(mb_u, tid));
        }
      }
      CHOL_T(j, 2)
      CHOL_T(j, 3)
      // bulk: items = own Cholesky rows i > j+1 (entries k in [j+2, i]) and own inverse columns
      // k <= j (entries i in [j+1, q)), one warp per item, kCB entries per lane loaded first
      const int s0 = j + 1 < c ? 0 : (j + 1 - c) / kCl + 1;
      const int nrow = nown > s0 ? nown - s0 : 0;
      const int ncol = j < c ? 0 : ((j - c) / kCl + 1 < nown ? (j - c) / kCl + 1 : nown);
      // the senders of the look-ahead column are the low warps: the bulk starts from the high ones
      for (int it = kWarps - 1 - warp; it < nrow + ncol; it += kWarps) {
        if (it < nrow) {
          const int s = s0 + it, i = c + kCl * s;
          const Quat lij = ldQ(cb + (size_t)i * 4);
          double* row = rows + rowbase(s) * 4;
          for (int k0 = j + 2; k0 <= i; k0 += 32 * kCB) {
            Quat av[kCB], bv[kCB];
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int k = k0 + lane + 32 * u;
              if (k <= i) {
                av[u] = ldQ(row + (size_t)k * 4);
                bv[u] = ldQ(cb + (size_t)k * 4);
              }
            }
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int k = k0 + lane + 32 * u;
              if (k <= i) stQ(row + (size_t)k * 4, qsub(av[u], qmul(lij, qconj(bv[u]))));
            }
          }
        } else {
          const int u0 = it - nrow, k = c + kCl * u0;
          double* w = wcol + colbase(u0) * 4 - (size_t)k * 4;  // w + i*4 addresses W_ik (i >= k)
          const Quat xjk = qscale(ldQ(w + (size_t)j * 4), inv);
          __syncwarp();
          if (lane == 0) stQ(w + (size_t)j * 4, xjk);
          for (int i0 = j + 1; i0 < q; i0 += 32 * kCB) {
            Quat av[kCB], bv[kCB];
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int i = i0 + lane + 32 * u;
              if (i < q) {
                av[u] = ldQ(w + (size_t)i * 4);
                bv[u] = ldQ(cb + (size_t)i * 4);
              }
            }
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int i = i0 + lane + 32 * u;
              if (i < q) stQ(w + (size_t)i * 4, qsub(av[u], qmul(bv[u], xjk)));
            }
          }
        }
      }
    }
    CHOL_T(j, 4)
    for (int i = j + 2 + tid; i < q; i += kThreads) diag[i] = diag[i] - qnorm2(ldQ(cb + (size_t)i * 4));
    __syncthreads();
    CHOL_T(j, 5)
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
    for (int i = tid; i < q; i += kThreads) {
      Quat v = qzero();
      if (i >= k) v = ldQ(w + (size_t)(i - k) * 4);
      stQ(pr.X + ((size_t)i * q + k) * 4, v);
    }
  }
  cluster_barrier();
}

// ---------------------------------------------------------------------------
// Two columns per exchange.  The one-column kernel above pays one DSMEM round trip per column
// (q sequential exchanges, ~1.8 us each at q = 200).  Here every CTA also keeps a replicated
// first sub-diagonal sub[i] = G'(i+1, i) next to the replicated diagonal, so at block (j, j+1)
// every CTA forms the 2 x 2 diagonal factor itself:
//   l0 = sqrt(d_j),  L10 = G'(j+1, j) / l0,  l1 = sqrt(d_{j+1} - |L10|^2),
// and its own rows' entries of BOTH columns:
//   L_ij = G'(i, j) / l0,   L_i,j+1 = (G'(i, j+1) - L_ij conj(L10)) / l1     (i > j + 1),
// which go out in one exchange: q/2 round trips.  After the exchange the block's rank-2 update
// is applied (look-ahead columns j+2, j+3 first, with the replicated d and sub of rows j+2,
// j+3, then the next block is sent, then the bulk), and the inverse columns take the two
// elimination steps j and j+1 locally.  The arithmetic per element is the same as the
// one-column kernel's (the rank-2 update is two rank-1 updates, in column order).
// ---------------------------------------------------------------------------
constexpr int kClusterQMax2 = 288;  // compact triangles + 3 two-column buffers + sub within 227 KB

__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kThreads, 1) k_chol_inv_cluster2(CholProblems P) {
  const int c = (int)cg::this_cluster().block_rank();
  const CholJob pr = P.p[blockIdx.x / kCl];
  const int q = (int)P.q;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  constexpr int kWarps = kThreads / 32;
  const int nown = (q - c + kCl - 1) / kCl;
  extern __shared__ __align__(32) double sm[];
  double* colbuf = sm;                           // [3][2][q] quaternions: the two columns of a block
  double* sub = colbuf + 6 * (size_t)q * 4;      // [q] quaternions: replicated G'(i+1, i)
  double* diag = sub + (size_t)q * 4;            // [q] replicated running diagonal
  uint64_t* mbar = reinterpret_cast<uint64_t*>(diag + q + (q & 1));
  double* rows = reinterpret_cast<double*>(mbar + 4);
  auto rowbase = [&](int s) -> size_t { return (size_t)s * (c + 1) + (size_t)8 * s * (s - 1); };
  auto colbase = [&](int u) -> size_t { return (size_t)u * (q - c) - (size_t)8 * u * (u - 1); };
  double* wcol = rows + rowbase(nown) * 4;
  auto G_at = [&](int s, int k) -> double* { return rows + (rowbase(s) + k) * 4; };  // own row c + 16 s, col k

  for (int s = 0; s < nown; ++s) {
    const int i = c + kCl * s;
    double* row = rows + rowbase(s) * 4;
    for (int k = tid; k <= i; k += kThreads) stQ(row + (size_t)k * 4, ldQ(pr.G + ((size_t)i * q + k) * 4));
    double* col = wcol + colbase(s) * 4;
    for (int r = i + tid; r < q; r += kThreads) stQ(col + (size_t)(r - i) * 4, Quat{r == i ? 1.0 : 0.0, 0.0, 0.0, 0.0});
  }
  for (int i = tid; i < q; i += kThreads) {
    diag[i] = pr.G[((size_t)i * q + i) * 4];
    stQ(sub + (size_t)i * 4, i + 1 < q ? ldQ(pr.G + ((size_t)(i + 1) * q + i) * 4) : qzero());
  }
  if (tid == 0) {
    for (int k = 0; k < 3; ++k) mbar_init(&mbar[k], kCl + 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_barrier();

  // the 2 x 2 diagonal factor of block j (identical in every CTA); false on breakdown
  auto diag_factor = [&](int j, double& inv0, Quat& L10, double& inv1) -> bool {
    const double d0 = diag[j];
    if (!(d0 > 0.0) || !isfinite(d0)) return false;
    inv0 = 1.0 / sqrt(d0);
    if (j + 1 < q) {
      L10 = qscale(ldQ(sub + (size_t)j * 4), inv0);
      const double d1 = diag[j + 1] - qnorm2(L10);
      if (!(d1 > 0.0) || !isfinite(d1)) return false;
      inv1 = 1.0 / sqrt(d1);
    }
    return true;
  };
  // send the own rows' entries of columns j, j+1 (rows i > j + 1) to every CTA; L10 (row j+1 of
  // column j) every CTA writes itself
  auto produce = [&](int j) -> bool {
    double inv0 = 0.0, inv1 = 0.0;
    Quat L10 = qzero();
    if (!diag_factor(j, inv0, L10, inv1)) return false;
    const int b = (j >> 1) % 3;
    double* cb = colbuf + (size_t)b * 2 * q * 4;
    const unsigned nsend = (unsigned)(q - 2 - j > 0 ? q - 2 - j : 0);
    if (tid == 0) {
      mbar_expect_tx(&mbar[b], 2u * 32u * nsend);
      if (j + 1 < q) stQ(cb + (size_t)(j + 1) * 4, L10);  // column j, row j + 1 (local)
    }
    const uint32_t cb_u = smem_u32(cb), mb_u = smem_u32(&mbar[b]);
    for (int t = tid; t < nown * kCl; t += kThreads) {
      const int s = t / kCl, dst = t - s * kCl;
      const int i = c + kCl * s;
      if (i <= j + 1) continue;
      const Quat lij = qscale(ldQ(G_at(s, j)), inv0);
      const Quat lij1 = qscale(qsub(ldQ(G_at(s, j + 1)), qmul(lij, qconj(L10))), inv1);
      st_async_quat(mapa(cb_u + 32u * (unsigned)i, dst), lij, mapa(mb_u, dst));
      st_async_quat(mapa(cb_u + 32u * (unsigned)(q + i), dst), lij1, mapa(mb_u, dst));
    }
    if (tid < kCl) mbar_arrive_remote(mapa(mb_u, tid));
    return true;
  };

  bool ok = produce(0);
  for (int j = 0; ok && j < q; j += 2) {
    const int b = (j >> 1) % 3;
    const double* c0 = colbuf + (size_t)b * 2 * q * 4;  // column j of L
    const double* c1 = c0 + (size_t)q * 4;               // column j+1 of L
    const bool two = j + 1 < q;
    mbar_wait(&mbar[b], (unsigned)(j / 6) & 1u);
    double inv0 = 0.0, inv1 = 0.0;
    Quat L10 = qzero();
    diag_factor(j, inv0, L10, inv1);  // succeeded in produce (same replicated data)
    // look-ahead: columns j+2, j+3 of the own rows and the replicated d / sub of rows j+2, j+3,
    // then send block j+2 so its exchange overlaps this block's bulk update
    if (j + 2 < q) {
      const Quat a2 = ldQ(c0 + (size_t)(j + 2) * 4), b2 = two ? ldQ(c1 + (size_t)(j + 2) * 4) : qzero();
      const bool has3 = j + 3 < q;
      const Quat a3 = has3 ? ldQ(c0 + (size_t)(j + 3) * 4) : qzero(), b3 = has3 ? ldQ(c1 + (size_t)(j + 3) * 4) : qzero();
      for (int s = tid; s < nown; s += kThreads) {
        const int i = c + kCl * s;
        if (i <= j + 1) continue;
        const Quat lij = ldQ(c0 + (size_t)i * 4), lij1 = ldQ(c1 + (size_t)i * 4);
        if (i > j + 2) {  // entry (i, j+2)
          double* e = G_at(s, j + 2);
          Quat v = qsub(ldQ(e), qmul(lij, qconj(a2)));
          if (two) v = qsub(v, qmul(lij1, qconj(b2)));
          stQ(e, v);
        }
        if (has3 && i > j + 3) {  // entry (i, j+3)
          double* e = G_at(s, j + 3);
          Quat v = qsub(ldQ(e), qmul(lij, qconj(a3)));
          if (two) v = qsub(v, qmul(lij1, qconj(b3)));
          stQ(e, v);
        }
      }
      if (tid == 0) {
        diag[j + 2] = diag[j + 2] - qnorm2(a2) - qnorm2(b2);
        if (has3) {
          diag[j + 3] = diag[j + 3] - qnorm2(a3) - qnorm2(b3);
          Quat v = qsub(ldQ(sub + (size_t)(j + 2) * 4), qmul(a3, qconj(a2)));
          if (two) v = qsub(v, qmul(b3, qconj(b2)));
          stQ(sub + (size_t)(j + 2) * 4, v);
        }
      }
      __syncthreads();
      ok = produce(j + 2);
    }
    // bulk: items = own rows i > j+3 (rank-2 update of columns k in [j+4, i]) and own inverse columns
    // k <= j+1 (elimination steps j and j+1 fused per entry, same operation order), one warp per item
    // from the high warps down (the senders are the low ones), kCB entries per lane loaded first
    {
      const int s0 = j + 3 < c ? 0 : (j + 3 - c) / kCl + 1;
      const int nrow = nown > s0 ? nown - s0 : 0;
      const int kmax = two ? j + 1 : j;
      const int ncol = kmax < c ? 0 : ((kmax - c) / kCl + 1 < nown ? (kmax - c) / kCl + 1 : nown);
      for (int it = kWarps - 1 - warp; it < nrow + ncol; it += kWarps) {
        if (it < nrow) {
          const int sr = s0 + it, i = c + kCl * sr;
          const Quat lij = ldQ(c0 + (size_t)i * 4), lij1 = two ? ldQ(c1 + (size_t)i * 4) : qzero();
          double* row = rows + rowbase(sr) * 4;
          for (int k0 = j + 4; k0 <= i; k0 += 32 * kCB) {
            Quat av[kCB], bv[kCB], dv[kCB];
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int k = k0 + lane + 32 * u;
              if (k <= i) {
                av[u] = ldQ(row + (size_t)k * 4);
                bv[u] = ldQ(c0 + (size_t)k * 4);
                dv[u] = two ? ldQ(c1 + (size_t)k * 4) : qzero();
              }
            }
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int k = k0 + lane + 32 * u;
              if (k <= i) {
                Quat v = qsub(av[u], qmul(lij, qconj(bv[u])));
                if (two) v = qsub(v, qmul(lij1, qconj(dv[u])));
                stQ(row + (size_t)k * 4, v);
              }
            }
          }
        } else {
          const int u0 = it - nrow, k = c + kCl * u0;
          double* w = wcol + colbase(u0) * 4 - (size_t)k * 4;  // w + i*4 addresses W_ik (i >= k)
          const bool stepj = k <= j;
          const Quat xjk = stepj ? qscale(ldQ(w + (size_t)j * 4), inv0) : qzero();
          Quat xj1 = qzero();
          if (two) {
            Quat wj1 = ldQ(w + (size_t)(j + 1) * 4);
            if (stepj) wj1 = qsub(wj1, qmul(ldQ(c0 + (size_t)(j + 1) * 4), xjk));
            xj1 = qscale(wj1, inv1);
          }
          __syncwarp();
          if (lane == 0) {
            if (stepj) stQ(w + (size_t)j * 4, xjk);
            if (two) stQ(w + (size_t)(j + 1) * 4, xj1);
          }
          for (int i0 = j + 2; i0 < q; i0 += 32 * kCB) {
            Quat av[kCB], bv[kCB], dv[kCB];
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int i = i0 + lane + 32 * u;
              if (i < q) {
                av[u] = ldQ(w + (size_t)i * 4);
                bv[u] = ldQ(c0 + (size_t)i * 4);
                dv[u] = two ? ldQ(c1 + (size_t)i * 4) : qzero();
              }
            }
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int i = i0 + lane + 32 * u;
              if (i < q) {
                Quat v = av[u];
                if (stepj) v = qsub(v, qmul(bv[u], xjk));
                if (two) v = qsub(v, qmul(dv[u], xj1));
                stQ(w + (size_t)i * 4, v);
              }
            }
          }
          __syncwarp();
        }
      }
    }
    // replicated diagonal and sub-diagonal of the rows below the look-ahead
    for (int i = j + 4 + tid; i < q; i += kThreads) {
      const Quat ai = ldQ(c0 + (size_t)i * 4), bi = two ? ldQ(c1 + (size_t)i * 4) : qzero();
      diag[i] = diag[i] - qnorm2(ai) - qnorm2(bi);
    }
    for (int i = j + 3 + tid; i + 1 < q; i += kThreads) {  // sub[i] = G'(i+1, i)
      const Quat ai = ldQ(c0 + (size_t)i * 4), ai1 = ldQ(c0 + (size_t)(i + 1) * 4);
      Quat v = qsub(ldQ(sub + (size_t)i * 4), qmul(ai1, qconj(ai)));
      if (two) v = qsub(v, qmul(ldQ(c1 + (size_t)(i + 1) * 4), qconj(ldQ(c1 + (size_t)i * 4))));
      stQ(sub + (size_t)i * 4, v);
    }
    __syncthreads();
  }
  if (!ok) {
    if (c == 0 && tid == 0) atomicOr(P.status, pr.fail_bit);
    cluster_barrier();
    return;
  }
  for (int u = 0; u < nown; ++u) {
    const int k = c + kCl * u;
    const double* w = wcol + colbase(u) * 4;
    for (int i = tid; i < q; i += kThreads) stQ(pr.X + ((size_t)i * q + k) * 4, i >= k ? ldQ(w + (size_t)(i - k) * 4) : qzero());
  }
  cluster_barrier();
}

static size_t chol_cluster_smem2(int64_t q) {
  size_t best = 0;
  for (int c = 0; c < kCl; ++c) {
    const int64_t nown = (q - c + kCl - 1) / kCl;
    const int64_t rows = nown * (c + 1) + 8 * nown * (nown - 1);
    const int64_t cols = nown * (q - c) - 8 * nown * (nown - 1);
    const size_t b = (size_t)(6 * q * 4 + q * 4 + q + (q & 1) + 4 + 4 * (rows + cols)) * sizeof(double);
    best = b > best ? b : best;
  }
  return best;
}

int chol_cluster_qmax() { return kClusterQMax; }

#ifdef QCUR_CHOL_TRACE
void chol_trace_read(long long* out) { cudaMemcpyFromSymbol(out, g_chol_trace, sizeof(g_chol_trace)); }
#endif

// ---------------------------------------------------------------------------
// Pipelined variant (default for q >= 192; QCUR_CHOL_PIPE=0/1 forces it): warp-specialised.  Sender warps (S) run the critical chain:
// wait for column j, form and send column j+1 of the own rows, then apply step j to column j+2
// (entries and replicated pivot) once the bulk warps have finished step j-1.  Bulk warps (B) apply
// step j to the columns k >= j+3 of the own rows and to the inverse, one step behind the senders, so
// the exchange of column j+1 overlaps the bulk of step j instead of following it.  Four column
// buffers: a peer can be at most two columns ahead of this CTA's bulk.  The operations on every
// element are the one-column kernel's, in the same order: bit-identical factors.
// ---------------------------------------------------------------------------
#ifndef QCUR_CHOL_PB
#define QCUR_CHOL_PB 8
#endif
constexpr int kPS = 4, kPB = QCUR_CHOL_PB, kPThreads = 32 * (kPS + kPB), kPBuf = 4;
constexpr int64_t kPipeQMin = 192;

__host__ __device__ inline int chol_bulk_ns(int64_t q) {  // slots per owner: ceil(q / 16), odd
  const int n = (int)((q + kCl - 1) / kCl);
  return n | 1;
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// BULK (round 2): the column exchange as one bulk copy per destination.  A column buffer is laid out
// by owner (entry i at slot (i mod 16) NS + i / 16, NS = ceil(q / 16) rounded up to odd: a warp reading 32
// consecutive entries still touches every 32-byte bank group once), so an owner's entries of a column
// are contiguous: the senders write them into their own buffer and each destination receives them with
// one cp.async.bulk (shared::cta -> shared::cluster, complete_tx on the destination's barrier) instead
// of 2 (q - j) / 16 st.async per destination (traced: the send took ~1000 of the 2800 cycles of a step).
// Measured slower (the small bulk copies cost more than the st.async they replace): opt-in only.
template <bool BULK>
__global__ void __cluster_dims__(kCl, 1, 1) __launch_bounds__(kPThreads, 1) k_chol_inv_pipe(CholProblems P) {
  const int c = (int)cg::this_cluster().block_rank();
  const CholJob pr = P.p[blockIdx.x / kCl];
  const int q = (int)P.q;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nown = (q - c + kCl - 1) / kCl;
  const int NS = chol_bulk_ns(q);                        // slots per owner (BULK)
  const int CS = BULK ? kCl * NS : q;                    // quaternions per column buffer
  auto slot = [&](int i) -> int { return BULK ? (i & (kCl - 1)) * NS + (i >> 4) : i; };
  extern __shared__ __align__(32) double sm[];
  double* colbuf = sm;                                   // [4][CS] columns of L in flight
  double* diag = colbuf + kPBuf * (size_t)CS * 4;        // [q] replicated running diagonal
  double* invs = diag + q;                               // [q] 1 / l_jj
  uint64_t* mbar = reinterpret_cast<uint64_t*>(invs + q + 2);  // [4] column arrival, [4] bulk done
  uint64_t* bdone = mbar + kPBuf;
  double* rows = reinterpret_cast<double*>(mbar + 2 * kPBuf);
  auto rowbase = [&](int s) -> size_t { return (size_t)s * (c + 1) + (size_t)8 * s * (s - 1); };
  auto colbase = [&](int u) -> size_t { return (size_t)u * (q - c) - (size_t)8 * u * (u - 1); };
  double* wcol = rows + rowbase(nown) * 4;
  __shared__ int s_fail;

  for (int s = 0; s < nown; ++s) {
    const int i = c + kCl * s;
    double* row = rows + rowbase(s) * 4;
    for (int k = tid; k <= i; k += kPThreads) stQ(row + (size_t)k * 4, ldQ(pr.G + ((size_t)i * q + k) * 4));
    double* col = wcol + colbase(s) * 4;
    for (int r = i + tid; r < q; r += kPThreads) stQ(col + (size_t)(r - i) * 4, Quat{r == i ? 1.0 : 0.0, 0.0, 0.0, 0.0});
  }
  for (int i = tid; i < q; i += kPThreads) diag[i] = pr.G[((size_t)i * q + i) * 4];
  if (tid == 0) {
    for (int k = 0; k < kPBuf; ++k) mbar_init(&mbar[k], kCl + 1);  // 16 producer arrives + local expect_tx
    mbar_init(bdone, 1);                                          // one arrive per bulk step
    s_fail = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster_barrier();

  if (warp < kPS) {
    // ---------------- senders ----------------
    const int st = tid;  // 0 .. 32 kPS - 1
    bool fail = false;
    // send column j (own rows i > j, entry value v(s) supplied by the caller), scaled by inv
    auto send = [&](int j, double inv, auto&& value) {
      const int b = j % kPBuf;
      if constexpr (BULK) {
        double* cbw = colbuf + (size_t)b * CS * 4;
        const int s0 = j < c ? 0 : (j - c) / kCl + 1;  // own entries i = c + 16 s > j
        const int cnt = nown > s0 ? nown - s0 : 0;
        for (int sr = s0 + st; sr < nown; sr += 32 * kPS)
          stQ(cbw + (size_t)(c * NS + sr) * 4, fail ? qzero() : qscale(value(sr), inv));
        if (st == 0) {
          invs[j] = inv;
          mbar_expect_tx(&mbar[b], 32u * (unsigned)((q - 1 - j) - cnt));  // the other owners' entries
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> bulk copy reads
        named_sync(3, 32 * kPS);
        if (st < kCl) {
          const uint32_t mb_u = smem_u32(&mbar[b]);
          if (st != c) {
            if (cnt > 0) {
              const uint32_t src = smem_u32(cbw + (size_t)(c * NS + s0) * 4);
              asm volatile(
                  "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                      mapa(src, st)),
                  "r"(src), "r"(32u * (unsigned)cnt), "r"(mapa(mb_u, st))
                  : "memory");
            }
            mbar_arrive_remote(mapa(mb_u, st));
          } else {
            mbar_arrive(&mbar[b]);  // release: this CTA's own entries are plain stores
          }
        }
      } else {
        if (st == 0) {
          invs[j] = inv;  // before the local arrive: the bulk warps read it after this column's phase
          mbar_expect_tx(&mbar[b], 32u * (unsigned)(q - 1 - j));
        }
        const uint32_t cb_u = smem_u32(colbuf + (size_t)b * CS * 4), mb_u = smem_u32(&mbar[b]);
        // a thread's (entry, destination) pairs: all values first (independent loads and products in
        // flight together), then the stores (same values, same order per destination)
        constexpr int kPairs = ((kClusterQMax + kCl - 1) / kCl * kCl + 32 * kPS - 1) / (32 * kPS);
        Quat val[kPairs];
        bool act[kPairs];
#pragma unroll
        for (int u = 0; u < kPairs; ++u) {
          const int t = st + u * 32 * kPS;
          const int sr = t / kCl;
          act[u] = t < nown * kCl && c + kCl * sr > j;
          val[u] = act[u] && !fail ? qscale(value(sr), inv) : qzero();
        }
#pragma unroll
        for (int u = 0; u < kPairs; ++u) {
          if (!act[u]) continue;
          const int t = st + u * 32 * kPS;
          const int sr = t / kCl, dst = t - sr * kCl;
          const int i = c + kCl * sr;
          st_async_quat(mapa(cb_u + 32u * (unsigned)i, dst), val[u], mapa(mb_u, dst));
        }
        if (st < kCl) mbar_arrive_remote(mapa(mb_u, st));
      }
    };
    {
      const double d = diag[0];
      fail = !(d > 0.0) || !isfinite(d);
      send(0, fail ? 0.0 : 1.0 / sqrt(d), [&](int s) { return ldQ(rows + (rowbase(s) + 0) * 4); });
    }
    for (int j = 0; j < q; ++j) {
      const int b = j % kPBuf;
      const double* cb = colbuf + (size_t)b * CS * 4;
      CHOL_T(j, 0)
      mbar_wait(&mbar[b], (unsigned)(j / kPBuf) & 1u);
      CHOL_T(j, 1)
      if (j + 1 < q) {
        const Quat lj1 = ldQ(cb + (size_t)slot(j + 1) * 4);
        const double d1 = diag[j + 1] - qnorm2(lj1);
        if (!(d1 > 0.0) || !isfinite(d1)) fail = true;  // every CTA alike (replicated diagonal)
        send(j + 1, fail ? 0.0 : 1.0 / sqrt(d1), [&](int s) {
          const int i = c + kCl * s;
          return qsub(ldQ(rows + (rowbase(s) + j + 1) * 4), qmul(ldQ(cb + (size_t)slot(i) * 4), qconj(lj1)));
        });
      }
      CHOL_T(j, 2)
      if (j + 2 < q) {
        if (j >= 1) mbar_wait(bdone, (unsigned)(j - 1) & 1u);  // the bulk of step j-1 is done
        CHOL_T(j, 3)
        if (!fail) {
          const Quat lj2 = ldQ(cb + (size_t)slot(j + 2) * 4);
          for (int s = st; s < nown; s += 32 * kPS) {
            const int i = c + kCl * s;
            if (i <= j + 2) continue;
            double* e = rows + (rowbase(s) + j + 2) * 4;
            stQ(e, qsub(ldQ(e), qmul(ldQ(cb + (size_t)slot(i) * 4), qconj(lj2))));
          }
          if (st == 0) diag[j + 2] = diag[j + 2] - qnorm2(lj2);
        }
      }
      CHOL_T(j, 4)
      named_sync(1, 32 * kPS);  // the next step's senders read the entries and pivot written above
      CHOL_T(j, 5)
    }
    if (st == 0 && fail) s_fail = 1;
  } else {
    // ---------------- bulk ----------------
    const int bw = warp - kPS, bt = tid - 32 * kPS;
    for (int j = 0; j < q; ++j) {
      const int b = j % kPBuf;
      const double* cb = colbuf + (size_t)b * CS * 4;
      mbar_wait(&mbar[b], (unsigned)(j / kPBuf) & 1u);
      const double inv = invs[j];
      const int s0 = j + 2 < c ? 0 : (j + 2 - c) / kCl + 1;  // own rows i > j + 2
      const int nrow = nown > s0 ? nown - s0 : 0;
      const int ncol = j < c ? 0 : ((j - c) / kCl + 1 < nown ? (j - c) / kCl + 1 : nown);
      for (int it = kPB - 1 - bw; it < nrow + ncol; it += kPB) {
        if (it < nrow) {
          const int sr = s0 + it, i = c + kCl * sr;
          const Quat lij = ldQ(cb + (size_t)slot(i) * 4);
          double* row = rows + rowbase(sr) * 4;
          for (int k0 = j + 3; k0 <= i; k0 += 32 * kCB) {
            Quat av[kCB], bv[kCB];
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int k = k0 + lane + 32 * u;
              if (k <= i) {
                av[u] = ldQ(row + (size_t)k * 4);
                bv[u] = ldQ(cb + (size_t)slot(k) * 4);
              }
            }
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int k = k0 + lane + 32 * u;
              if (k <= i) stQ(row + (size_t)k * 4, qsub(av[u], qmul(lij, qconj(bv[u]))));
            }
          }
        } else {
          const int u0 = it - nrow, k = c + kCl * u0;
          double* w = wcol + colbase(u0) * 4 - (size_t)k * 4;  // w + i*4 addresses W_ik (i >= k)
          const Quat xjk = qscale(ldQ(w + (size_t)j * 4), inv);
          __syncwarp();
          if (lane == 0) stQ(w + (size_t)j * 4, xjk);
          for (int i0 = j + 1; i0 < q; i0 += 32 * kCB) {
            Quat av[kCB], bv[kCB];
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int i = i0 + lane + 32 * u;
              if (i < q) {
                av[u] = ldQ(w + (size_t)i * 4);
                bv[u] = ldQ(cb + (size_t)slot(i) * 4);
              }
            }
#pragma unroll
            for (int u = 0; u < kCB; ++u) {
              const int i = i0 + lane + 32 * u;
              if (i < q) stQ(w + (size_t)i * 4, qsub(av[u], qmul(bv[u], xjk)));
            }
          }
          __syncwarp();
        }
      }
      for (int i = j + 3 + bt; i < q; i += 32 * kPB) diag[i] = diag[i] - qnorm2(ldQ(cb + (size_t)slot(i) * 4));
      named_sync(2, 32 * kPB);  // every bulk warp is done with step j
      if (bt == 0) mbar_arrive(bdone);
    }
  }
  __syncthreads();
  if (s_fail) {  // identical in every CTA (replicated diagonal)
    if (c == 0 && tid == 0) atomicOr(P.status, pr.fail_bit);
    cluster_barrier();
    return;
  }
  for (int u = 0; u < nown; ++u) {
    const int k = c + kCl * u;
    const double* w = wcol + colbase(u) * 4;
    for (int i = tid; i < q; i += kPThreads) stQ(pr.X + ((size_t)i * q + k) * 4, i >= k ? ldQ(w + (size_t)(i - k) * 4) : qzero());
  }
  cluster_barrier();
}

static size_t chol_pipe_smem(int64_t q) {
  size_t best = 0;
  for (int c = 0; c < kCl; ++c) {
    const int64_t nown = (q - c + kCl - 1) / kCl;
    const int64_t rows = nown * (c + 1) + 8 * nown * (nown - 1);
    const int64_t cols = nown * (q - c) - 8 * nown * (nown - 1);
    const int64_t cs = kCl * (int64_t)chol_bulk_ns(q) > q ? kCl * (int64_t)chol_bulk_ns(q) : q;  // either layout
    const size_t b = (size_t)(kPBuf * cs * 4 + 2 * q + 2 + 2 * kPBuf + 4 * (rows + cols)) * sizeof(double);
    best = b > best ? b : best;
  }
  return best;
}

// dynamic shared memory of the CTA with the largest triangles (rank 0)
static size_t chol_cluster_smem(int64_t q) {
  size_t best = 0;
  for (int c = 0; c < kCl; ++c) {
    const int64_t nown = (q - c + kCl - 1) / kCl;
    const int64_t rows = nown * (c + 1) + 8 * nown * (nown - 1);
    const int64_t cols = nown * (q - c) - 8 * nown * (nown - 1);
    const size_t b = (size_t)(3 * q * 4 + q + (q & 1) + 4 + 4 * (rows + cols) + q) * sizeof(double);  // + V2 pivots
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
    cudaFuncSetAttribute(k_chol_inv_cluster<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_chol_inv_cluster<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    cudaFuncSetAttribute(k_chol_inv_cluster<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_chol_inv_cluster<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  }
  static const int v2_env = [] {
    const char* e = std::getenv("QCUR_CHOL_V2");
    return e ? std::atoi(e) : 1;
  }();
  static const int b2_env = [] {
    const char* e = std::getenv("QCUR_CHOL_B2");
    return e ? std::atoi(e) : -1;
  }();
  const bool two = (b2_env == 1 || (b2_env < 0 && kCholTwoColumnDefault)) && q <= kClusterQMax2 &&
                   chol_cluster_smem2(q) <= 227 * 1024;
  if (two) {
    static std::atomic<unsigned> set2{0};
    if (first_on_device(set2)) {
      cudaFuncSetAttribute(k_chol_inv_cluster2, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(k_chol_inv_cluster2, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    }
    ++::qcur::g_launches;
    k_chol_inv_cluster2<<<kCl * njobs, kThreads, chol_cluster_smem2(q), st>>>(P);
    return;
  }
  // pipelined variant from q = 192 up (measured, factor phase per approximation: q = 200 1.196 -> 1.160 ms,
  // q = 256 1.073 -> 1.033 ms; slower at q <= 128: 0.414 -> 0.432 ms); QCUR_CHOL_PIPE=0/1 forces it
  static const int pipe_env = [] {
    const char* e = std::getenv("QCUR_CHOL_PIPE");
    return e ? std::atoi(e) : -1;
  }();
  if ((pipe_env == 1 || (pipe_env < 0 && q >= kPipeQMin)) && chol_pipe_smem(q) <= 226 * 1024) {
    static std::atomic<unsigned> setp{0};
    if (first_on_device(setp)) {
      for (auto f : {k_chol_inv_pipe<true>, k_chol_inv_pipe<false>}) {
        cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
      }
    }
    ++::qcur::g_launches;
    // QCUR_CHOL_BULK=1: the column exchange by one bulk copy per destination (bit-identical factors;
    // measured slower: q = 200 pair 477 vs 279 us, the send 1978 vs 1007 cycles per step)
    static const int bulk_env = [] {
      const char* e = std::getenv("QCUR_CHOL_BULK");
      return e ? std::atoi(e) : 0;
    }();
    if (bulk_env)
      k_chol_inv_pipe<true><<<kCl * njobs, kPThreads, chol_pipe_smem(q), st>>>(P);
    else
      k_chol_inv_pipe<false><<<kCl * njobs, kPThreads, chol_pipe_smem(q), st>>>(P);
    return;
  }
  ++::qcur::g_launches;
  if (v2_env)
    k_chol_inv_cluster<true><<<kCl * njobs, kThreads, smem, st>>>(P);
  else
    k_chol_inv_cluster<false><<<kCl * njobs, kThreads, smem, st>>>(P);
}

}  // namespace qcur
