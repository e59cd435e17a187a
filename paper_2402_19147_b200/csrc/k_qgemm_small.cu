// Small quaternion products C = alpha op(A) op(B) + beta C with N, K <= kSmallMax and M <= kSmallMax or
// little total work (the q x q products of a factorization step and of the core: S += E E,
// F = L1^{-H} S, U = F_C M F_R^H; at the small configurations also Q_1 = Z L_1^{-H} and P = C U;
// linalg.py:346-362 / cur.py:268 on the device).
//
// The persistent DMMA GEMM (k_qgemm.cu) is built for tall products: at q = 200 a q x q x q product is
// 20 of its 64 x 160 tiles, split into k ranges that meet on tickets, and it ran at 33-54 us with half
// of the SMs idle for half of the launch (ncu sm__cycles_active.avg 58k of 107k elapsed cycles).
// Here a thread-block CLUSTER of kKS (4) CTAs owns one 32 x 32 output tile: CTA r sums the k range
// [r K / kKS, (r + 1) K / kKS) with FP64 FMAs (a thread keeps 2 x 4 quaternions of the tile in
// registers: 128 FMAs per 6 quaternions read from shared memory), writes its partial tile to its
// shared memory, and after a cluster barrier CTA r adds rows [8 r, 8 r + 8) of all kKS partials in
// rank order through distributed shared memory.  No workspace, no tickets, one launch for one or
// two problems.  The k split depends on K only, so an element's value does not depend on M, N or on
// the pairing: two problems in one launch give the bits of two separate launches.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace qcur {

namespace {
#ifndef QCUR_SMALL_KS  // build-time variant for A/B timing
#define QCUR_SMALL_KS 4
#endif
constexpr int kKS = QCUR_SMALL_KS;
static_assert(kKS == 1 || kKS == 2 || kKS == 4 || kKS == 8, "the cluster's ranks split the 32-row reduction evenly");  // CTAs per cluster (k ranges): 4-CTA clusters pack the GPCs in one wave
                                   // at q = 200 (8-CTA clusters: 784 CTAs in ~3 waves, 49 us for the pair)
constexpr int kT = 32;        // output tile edge (quaternions)
constexpr int kKC = 16;       // quaternions of K staged per step
constexpr int kThreadsS = 128;
constexpr int64_t kSmallMax = 256;

struct SmallProb {
  const double* A;
  const double* B;
  double* C;
  int64_t M, N, K, lda, ldb, ldc;
  double alpha, beta;
  int opA, opB;  // 0: as stored, 1: conjugate transpose
  int tn;        // tile columns
  int tiles;     // tile count
};
struct SmallProbs {
  SmallProb p[2];
  int clusters0;  // clusters of problem 0
};

__device__ __forceinline__ Quat ldq(const double* p) { return *reinterpret_cast<const Quat*>(p); }

// acc += op(a) op(b) with explicit FMA chains (16 FMAs); CA / CB: conjugate a / b
template <bool CA, bool CB>
__device__ __forceinline__ void qmac(Quat& c, const Quat& a, const Quat& b) {
  const double ax = CA ? -a.x : a.x, ay = CA ? -a.y : a.y, az = CA ? -a.z : a.z;
  const double bx = CB ? -b.x : b.x, by = CB ? -b.y : b.y, bz = CB ? -b.z : b.z;
  c.w = fma(a.w, b.w, c.w);
  c.w = fma(-ax, bx, c.w);
  c.w = fma(-ay, by, c.w);
  c.w = fma(-az, bz, c.w);
  c.x = fma(a.w, bx, c.x);
  c.x = fma(ax, b.w, c.x);
  c.x = fma(ay, bz, c.x);
  c.x = fma(-az, by, c.x);
  c.y = fma(a.w, by, c.y);
  c.y = fma(-ax, bz, c.y);
  c.y = fma(ay, b.w, c.y);
  c.y = fma(az, bx, c.y);
  c.z = fma(a.w, bz, c.z);
  c.z = fma(ax, by, c.z);
  c.z = fma(-ay, bx, c.z);
  c.z = fma(az, b.w, c.z);
}

// the eight products acc[u][v] += op(a_u) op(b_v), issued step by step across all 32 accumulators
// (four rounds of 32 independent FMAs instead of 32 chains of four dependent ones: at one or two
// warps per scheduler the chains stalled on the FMA latency).  Each accumulator sees the same
// operations in the same order as qmac: identical bits.
template <bool CA, bool CB>
__device__ __forceinline__ void qmac8(Quat (&acc)[2][4], const Quat (&a)[2], const Quat (&b)[4]) {
  double A[2][4], B[4][4];
#pragma unroll
  for (int u = 0; u < 2; ++u) {
    A[u][0] = a[u].w;
    A[u][1] = CA ? -a[u].x : a[u].x;
    A[u][2] = CA ? -a[u].y : a[u].y;
    A[u][3] = CA ? -a[u].z : a[u].z;
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) {
    B[v][0] = b[v].w;
    B[v][1] = CB ? -b[v].x : b[v].x;
    B[v][2] = CB ? -b[v].y : b[v].y;
    B[v][3] = CB ? -b[v].z : b[v].z;
  }
  // component t, step s: c_t += sg * A[ia] * B[ib]   (the Hamilton table of qmac, row by row)
  constexpr int kIa[4][4] = {{0, 1, 2, 3}, {0, 1, 2, 3}, {0, 1, 2, 3}, {0, 1, 2, 3}};
  constexpr int kIb[4][4] = {{0, 1, 2, 3}, {1, 0, 3, 2}, {2, 3, 0, 1}, {3, 2, 1, 0}};
  constexpr int kSg[4][4] = {{1, -1, -1, -1}, {1, 1, 1, -1}, {1, -1, 1, 1}, {1, 1, -1, 1}};
#pragma unroll
  for (int st = 0; st < 4; ++st)
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        Quat& c = acc[u][v];
        c.w = fma(kSg[0][st] * A[u][kIa[0][st]], B[v][kIb[0][st]], c.w);
        c.x = fma(kSg[1][st] * A[u][kIa[1][st]], B[v][kIb[1][st]], c.x);
        c.y = fma(kSg[2][st] * A[u][kIa[2][st]], B[v][kIb[2][st]], c.y);
        c.z = fma(kSg[3][st] * A[u][kIa[3][st]], B[v][kIb[3][st]], c.z);
      }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Operand staging.  Both operands are copied as stored (raw rows, cp.async, zero fill outside the
// matrix or the CTA's k range) and conjugated when used:
//   op(A) = A   : rows i (kT) of kKC quaternions   -> X[i][kk]    op(A) = A^H : rows kk of kT -> X[kk][i]
//   op(B) = B   : rows kk (kKC) of kT quaternions  -> X[kk][j]    op(B) = B^H : rows j of kKC -> X[j][kk]
// A buffer row holds L quaternions at a stride of L + 1 (bank spread for the 32-byte reads).
constexpr int kStageQ = (kT * (kKC + 1) > kKC * (kT + 1) ? kT * (kKC + 1) : kKC * (kT + 1));  // quaternions
constexpr int kStageD = 2 * kStageQ * 4;                                                   // doubles (A | B)
constexpr size_t kSmallSmem = (size_t)2 * kStageD * sizeof(double);

// rows x L quaternions from src rows (row r: global row g0 + r, columns c0 ..) into X (stride L + 1)
template <int ROWS, int L>
__device__ __forceinline__ void stage(double* X, const double* src, int64_t ld, int64_t g0, int64_t gmax, int64_t c0,
                                      int64_t cmax) {
  // 16-byte pieces: ROWS * L * 2 of them, kThreadsS per pass
#pragma unroll
  for (int s = 0; s < ROWS * L * 2 / kThreadsS; ++s) {
    const int idx = threadIdx.x + kThreadsS * s;
    const int r = idx / (2 * L), rem = idx - r * 2 * L, c = rem >> 1, h = rem & 1;
    const int64_t g = g0 + r, cc = c0 + c;
    const bool ok = g < gmax && cc < cmax;
    const double* sp = ok ? src + (g * ld + cc) * 4 + 2 * h : src;
    cp_async16(X + ((size_t)r * (L + 1) + c) * 4 + 2 * h, sp, ok);
  }
}

template <int OPA, int OPB>
__global__ void __launch_bounds__(kThreadsS) k_qgemm_small(const __grid_constant__ SmallProbs P) {
  const int cl = (int)blockIdx.x / kKS;
  const int pi = cl < P.clusters0 ? 0 : 1;
  const SmallProb& pr = P.p[pi];
  const int tile = pi == 0 ? cl : cl - P.clusters0;
  const int rank = (int)cg::this_cluster().block_rank();
  const int i0 = (tile / pr.tn) * kT, j0 = (tile % pr.tn) * kT;
  const int64_t kb = (int64_t)rank * pr.K / kKS, ke = (int64_t)(rank + 1) * pr.K / kKS;
  extern __shared__ __align__(128) double sm[];  // two stages of (A | B); then the partial tile (stage 0)
  const int tid = threadIdx.x;
  const int ti = tid >> 3, tj = tid & 7;  // rows 2 ti, 2 ti + 1; columns tj + 8 v
  Quat acc[2][4];
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = qzero();
  auto load = [&](int buf, int64_t k0) {
    double* As = sm + buf * kStageD;
    double* Bs = As + kStageQ * 4;
    if (OPA == 0) stage<kT, kKC>(As, pr.A, pr.lda, i0, pr.M, k0, ke);
    else stage<kKC, kT>(As, pr.A, pr.lda, k0, ke, i0, pr.M);
    if (OPB == 0) stage<kKC, kT>(Bs, pr.B, pr.ldb, k0, ke, j0, pr.N);
    else stage<kT, kKC>(Bs, pr.B, pr.ldb, j0, pr.N, k0, ke);
    cp_async_commit();
  };
  int buf = 0;
  if (kb < ke) load(0, kb);
  for (int64_t k0 = kb; k0 < ke; k0 += kKC) {
    const bool more = k0 + kKC < ke;
    if (more) load(buf ^ 1, k0 + kKC);
    if (more) cp_async_wait<1>();
    else cp_async_wait<0>();
    __syncthreads();
    const double* As = sm + buf * kStageD;
    const double* Bs = As + kStageQ * 4;
    const int kn = (int)(ke - k0 < kKC ? ke - k0 : kKC);
#pragma unroll 2
    for (int kk = 0; kk < kn; ++kk) {
      Quat a[2], b[4];
#pragma unroll
      for (int u = 0; u < 2; ++u)
        a[u] = OPA == 0 ? ldq(As + ((2 * ti + u) * (kKC + 1) + kk) * 4) : ldq(As + (kk * (kT + 1) + 2 * ti + u) * 4);
#pragma unroll
      for (int v = 0; v < 4; ++v)
        b[v] = OPB == 0 ? ldq(Bs + (kk * (kT + 1) + tj + 8 * v) * 4) : ldq(Bs + ((tj + 8 * v) * (kKC + 1) + kk) * 4);
      qmac8<OPA != 0, OPB != 0>(acc, a, b);
    }
    __syncthreads();  // the buffer is refilled by the next iteration's prefetch
    buf ^= 1;
  }
  double* part = sm;  // [kT][kT] quaternions (fits one stage)
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) *reinterpret_cast<Quat*>(part + ((2 * ti + u) * kT + tj + 8 * v) * 4) = acc[u][v];
  cg::this_cluster().sync();
  // rows [R rank, R rank + R) of the tile (R = kT / kKS): the kKS partials added in rank order
  constexpr int kRows = kT / kKS;
#pragma unroll
  for (int o = tid; o < kRows * kT; o += kThreadsS) {
    const int r = o >> 5, j = o & 31;
    const int li = kRows * rank + r;
    const int64_t gi = i0 + li, gj = j0 + j;
    Quat s = qzero();
#pragma unroll
    for (int q = 0; q < kKS; ++q) {
      const double* src = cg::this_cluster().map_shared_rank(part, q);
      const Quat v = ldq(src + (li * kT + j) * 4);
      s = q == 0 ? v : qadd(s, v);
    }
    if (gi < pr.M && gj < pr.N) {
      double* c = pr.C + (gi * pr.ldc + gj) * 4;
      Quat out = qscale(s, pr.alpha);
      if (pr.beta != 0.0) out = qadd(out, qscale(ldq(c), pr.beta));
      *reinterpret_cast<Quat*>(c) = out;
    }
  }
  cg::this_cluster().sync();  // no CTA leaves while a peer still reads its partial tile
}
static_assert(kT * kT * 4 <= kStageD, "the partial tile fits one stage");

SmallProb small_prob(const GemmArgs& g) {
  SmallProb p{};
  p.A = g.A;
  p.B = g.B;
  p.C = g.C;
  p.M = g.Mq;
  p.N = g.Nq;
  p.K = g.Kq;
  p.lda = g.lda;
  p.ldb = g.ldb;
  p.ldc = g.ldc;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.opA = g.opA;
  p.opB = g.opB;
  p.tn = (int)((g.Nq + kT - 1) / kT);
  p.tiles = (int)((g.Mq + kT - 1) / kT) * p.tn;
  return p;
}

bool small_env_on() {
  static const int v = [] {
    const char* e = getenv("QCUR_SMALL_GEMM");  // 0: every product on the DMMA GEMM (A/B timing)
    return e ? atoi(e) : 1;
  }();
  return v != 0;
}
}  // namespace

// q x q products, and tall products with small N and K while their total work is small (the
// triangular Q_1 = Z L_1^-H and P = C U of cfg1 / cfg4: 1000-1024 rows, q = 40-80, where the persistent
// DMMA GEMM spends ~24 us on ~1e6-7e6 quaternion MACs); QCUR_SMALL_MNK overrides the work bound
bool qgemm_small_ok(const GemmArgs& g) {
  static const double mnk_max = [] {
    const char* e = getenv("QCUR_SMALL_MNK");
    return e ? atof(e) : 1.2e7;
  }();
  const bool shape = g.Nq <= kSmallMax && g.Kq <= kSmallMax &&
                     (g.Mq <= kSmallMax || (double)g.Mq * (double)g.Nq * (double)g.Kq <= mnk_max);
  return small_env_on() && !g.whole_tiles && g.Mq >= 1 && g.Nq >= 1 && g.Kq >= 1 && shape &&
         (g.opA == 0 || g.opA == 1) && (g.opB == 0 || g.opB == 1);
}

void launch_qgemm_small(const GemmArgs* g, int np, cudaStream_t st) {
  SmallProbs P{};
  int clusters = 0;
  for (int k = 0; k < np; ++k) {
    P.p[k] = small_prob(g[k]);
    clusters += P.p[k].tiles;
  }
  P.clusters0 = P.p[0].tiles;
  void (*fn)(SmallProbs) = g[0].opA == 0 ? (g[0].opB == 0 ? k_qgemm_small<0, 0> : k_qgemm_small<0, 1>)
                                         : (g[0].opB == 0 ? k_qgemm_small<1, 0> : k_qgemm_small<1, 1>);
  static std::atomic<unsigned> set{0};
  if (first_on_device(set)) {
    for (auto f : {k_qgemm_small<0, 0>, k_qgemm_small<0, 1>, k_qgemm_small<1, 0>, k_qgemm_small<1, 1>}) {
      cudaFuncSetAttribute(f, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmallSmem);
    }
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(clusters * kKS));
  cfg.blockDim = dim3(kThreadsS);
  cfg.dynamicSmemBytes = kSmallSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = kKS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++::qcur::g_launches;
  cudaLaunchKernelEx(&cfg, fn, P);
}

}  // namespace qcur
