// Quaternion GEMM on the FP64 tensor path (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4),
// fed by TMA through an mbarrier pipeline.
//
// Replaces qmat_matmul (pkg/src/qcur/quat.py:274-296), the reference's
// "16 real GEMMs with the Hamilton sign pattern", which cur.py:268 and
// cur.py:274 use for U = pinv(C) @ X @ pinv(R) and C @ U @ R.
//
// Formulation: with X interleaved, row i of a quaternion matrix A is a real
// row of 4K doubles, and  row(a*b) = row(a) * E(b)  where E(b) is the 4x4 real
// block  E[t][s] = sign(t,s) * b[t ^ s].  So C = A*B is the real GEMM
// C_r (M x 4N) = A_r (M x 4K) * E(B) (4K x 4N).  The k4 step of one DMMA is
// exactly one quaternion of A's row; the B fragment element each lane needs is
// one component of one compact quaternion of B with a per-lane sign, so E(B) is
// never materialised (4x less shared memory and L2 traffic than expanding).
// op(A)=H / op(B)=H read k-major / j-major tiles with the conjugate sign table.
//
// CTA = 8 DMMA warps (2 x 4, warp tile WM x WN) + 1 TMA producer warpgroup (one
// issuing thread; setmaxnreg hands its registers to the DMMA warps), one CTA per SM.
// The producer streams (A, B) k-block stages into a 5-8 deep ring of
// shared-memory buffers with cp.async.bulk.tensor (A of op N through the
// 128-byte swizzle, so the fragment loads are bank-conflict free); full/empty
// mbarriers hand stages between the roles.  The DMMA warps do no address
// arithmetic at all in the main loop.
//
// Schedule: the work is the list of (tile, k-block) iterations of every output
// tile (row-major tiles; tiles above the diagonal of a Hermitian output are
// absent; an upper-triangular op(B) shortens each tile's k range).
//  * stream-K (many tiles): CTA c takes one contiguous span of the list, so
//    every SM gets the same number of k-blocks whatever the tile count.  A
//    tile cut between CTAs is finished by its last contributor (ticket), which
//    adds the parts in CTA (= k) order.
//  * split (fewer tiles than SMs/2, equal depth): each tile is cut into S equal
//    k ranges; the last of the S CTAs to finish (ticket) adds the parts in split order.
// Both orders are fixed, so results are bitwise deterministic run to run
// (test_cur.py:243-250).
//
// EPI_ERR fuses the error of the reference's caller (cli.py:173-175,
// imaging.py:170-177): CTAs take whole tiles, the tile of (P R) is subtracted
// from the matching tile of X in registers and only per-tile sums leave the
// CTA, so CUR is never written to HBM.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "kernels.h"

namespace qcur {

namespace {

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// named barrier among the DMMA warps only (the producer warp never joins)
template <int N>
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double flip(double v, unsigned long long m) {
  return __longlong_as_double(__double_as_longlong(v) ^ m);
}

// negative-entry masks of E(b) (bit t*4+s) for op N and for conj(b) (op H)
constexpr unsigned kSignN = 0x3950u;
constexpr unsigned kSignH = 0x428Eu;

enum { EPI_STORE = 0, EPI_ERR = 1, EPI_COMPLETE = 2 };
enum { MODE_STREAMK = 0, MODE_SPLIT = 1, MODE_TILES = 2 };

constexpr int kBKQ = 8;  // quaternions of K per stage
constexpr int kSmemBudget = 220 * 1024;

template <int BM, int BN, int EPI = 0>
struct Cfg {
  static constexpr int WARPS_M = 2, WARPS_N = 4;
  static constexpr int WM = BM / WARPS_M, WN = BN / WARPS_N;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int CONSUMERS = WARPS_M * WARPS_N * 32;
  // + one producer warpgroup (one thread issues TMA; the group exists so setmaxnreg can
  // move its registers to the two DMMA warpgroups: 8 x 232 + 4 x 40 per SM sub-partition set)
  static constexpr int THREADS = CONSUMERS + 128;
  static constexpr int PRODUCER_REGS = 40, CONSUMER_REGS = 232;
  static constexpr int A_BYTES = BM * kBKQ * 32;
  static constexpr int B_BYTES = kBKQ * BN * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // EPI_ERR: the epilogue's X tile is staged by TMA too (one BM x BN buffer)
  static constexpr int X_BYTES = EPI != 0 ? BM * BN * 8 : 0;
  static constexpr int STAGES =
      (kSmemBudget - X_BYTES) / STAGE_BYTES > 8 ? 8 : (kSmemBudget - X_BYTES) / STAGE_BYTES;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + X_BYTES + 1024 + (2 * STAGES + 2) * 8;
  static_assert(BM % 64 == 0 && (BN / 4) % kBKQ == 0 && WN % 8 == 0, "tile shape");
  static_assert(STAGE_BYTES % 1024 == 0, "stage buffers must keep the 1024-byte swizzle alignment");
};

struct KParams {
  int64_t Mq, Nq, Kq;
  double* C;
  int64_t ldc;
  double alpha, beta;
  const double* X;     // EPI_ERR: reference matrix
  int64_t ldx;
  double* partials;    // EPI_ERR: [tiles][4]
  double psnr_scale;   // EPI_ERR: > 0 -> also the u8 image statistic at this scale (255)
  const double* Y;              // EPI_COMPLETE: observed values
  const unsigned char* mask;    // EPI_COMPLETE: m x n, nonzero = observed
  unsigned* counters;  // per-tile tickets (zero between launches); [65536] + done counters
  double* slots;       // partial tiles [grid][2][BM*BN]
  int b_upper;         // op(B) is upper triangular: tile column j only needs k <= j
  int herm_lower;      // output is Hermitian and only its lower triangle is consumed
  int gx, gy;          // tile grid (columns of BN reals, rows of BM quaternion rows)
  int nkb_full;        // k-blocks of a full-depth tile (>= 1)
  int total;           // iterations (sum of k-blocks over tiles, < 2^31)
  int mode;
  int splits;          // MODE_SPLIT: CTAs per tile (the first split_extra tiles get one more)
  int split_extra;
  int waves;           // MODE_STREAMK: rounds of whole tiles before the stream-K tail
  int cta_G, cta_c;    // device side only: this problem's CTA count and this CTA's index
};

// Iteration space bookkeeping (closed form).
template <int BM, int BN>
struct Space {
  static constexpr int W = BN / 4;     // quaternion columns per tile
  static constexpr int w = W / kBKQ;   // k-blocks per tile column step (triangular op(B))
  const KParams& p;
  __device__ explicit Space(const KParams& kp) : p(kp) {}
  __device__ int last_col(int ty) const {
    if (!p.herm_lower) return p.gx - 1;
    const int L = (ty * BM + BM - 1) / W;
    return L < p.gx - 1 ? L : p.gx - 1;
  }
  __device__ int nkb_col(int tx) const {
    if (!p.b_upper) return p.nkb_full;
    const int v = (tx + 1) * w;
    return v < p.nkb_full ? v : p.nkb_full;
  }
  __device__ int prefix_cols(int L) const {  // sum of nkb_col over tile columns 0..L
    if (L < 0) return 0;
    if (!p.b_upper) return (L + 1) * p.nkb_full;
    const int tcap = (p.nkb_full + w - 1) / w - 1;  // first column at full depth
    if (L < tcap) return w * (L + 1) * (L + 2) / 2;
    return w * tcap * (tcap + 1) / 2 + (L - tcap + 1) * p.nkb_full;
  }
  __device__ int row_iters(int ty) const { return prefix_cols(last_col(ty)); }
  __device__ int tile_nkb(int t) const {
    const int ty = t / p.gx, tx = t - ty * p.gx;
    return tx > last_col(ty) ? 0 : nkb_col(tx);
  }
  __device__ void locate(int i, int& t, int& kb) const {  // (tile, k-block) of iteration i
    int ty = 0, base = 0;
    if (!p.herm_lower) {
      const int S = row_iters(0);
      ty = i / S;
      base = ty * S;
    } else {
      for (;; ++ty) {
        const int S = row_iters(ty);
        if (i < base + S) break;
        base += S;
      }
    }
    int rem = i - base, tx = 0;
    for (;; ++tx) {
      const int n = nkb_col(tx);
      if (rem < n) break;
      rem -= n;
    }
    t = ty * p.gx + tx;
    kb = rem;
  }
  __device__ void advance(int& t, int& kb, int& nkb) const {
    if (++kb == nkb) {
      kb = 0;
      const int ntiles = p.gx * p.gy;
      do {
        ++t;
        nkb = t < ntiles ? tile_nkb(t) : 1;
      } while (nkb == 0);
    }
  }
};

// Span s of this CTA: [sb, se) in the iteration list; false past the last span.
//  * whole tiles: one contiguous run of tiles (the error kernel);
//  * split: one equal k range of one tile;
//  * stream-K: `waves` rounds of whole tiles (tile w*G + c: CTAs in lock step work on
//    neighbouring tiles, so each A row block is fetched from HBM once and the other
//    column tiles hit L2), then one contiguous span of the remaining tiles' iterations.
// MODE_SPLIT: tile ordinal o, split z of S for CTA c, and the tile's first CTA
__device__ __forceinline__ void split_of(const KParams& p, int c, int& o, int& z, int& S, int& first) {
  const int big = p.split_extra * (p.splits + 1);
  if (c < big) {
    S = p.splits + 1;
    o = c / S;
    first = o * S;
  } else {
    S = p.splits;
    o = p.split_extra + (c - big) / S;
    first = big + (o - p.split_extra) * S;
  }
  z = c - first;
}

__device__ __forceinline__ bool cta_span(const KParams& p, int G, int c, int s, int& sb, int& se) {
  if (s < p.waves) {
    const int t = c + s * G;
    sb = t * p.nkb_full;
    se = sb + p.nkb_full;
    return true;
  }
  if (s > p.waves) return false;
  if (p.mode == MODE_TILES) {
    const int ntiles = p.gx * p.gy;
    sb = (int)((int64_t)c * ntiles / G) * p.nkb_full;
    se = (int)((int64_t)(c + 1) * ntiles / G) * p.nkb_full;
    return true;
  }
  if (p.mode == MODE_SPLIT) {
    int o, z, S, first;
    split_of(p, c, o, z, S, first);
    sb = o * p.nkb_full + (int)((int64_t)z * p.nkb_full / S);
    se = o * p.nkb_full + (int)((int64_t)(z + 1) * p.nkb_full / S);
    return true;
  }
  const int base = p.waves * G * p.nkb_full;
  const int64_t tail = (int64_t)p.total - base;
  sb = base + (int)((int64_t)c * tail / G);
  se = base + (int)((int64_t)(c + 1) * tail / G);
  return true;
}

// A launch carries one or two independent problems of the same shape class (the C and R^H
// sides of a CholeskyQR2 step): CTAs [0, grid0) run problem 0, the rest problem 1.
struct KPair {
  KParams p[2];
  int grid0;
};

template <int BM, int BN, int OPA, int OPB, int EPI>
__global__ void __launch_bounds__(Cfg<BM, BN, EPI>::THREADS, 1)
    qgemm_kernel(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                 const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                 const __grid_constant__ CUtensorMap tmX, const __grid_constant__ KPair pp) {
  using CF = Cfg<BM, BN, EPI>;
  const bool second = (int)blockIdx.x >= pp.grid0;
  // this CTA's problem, copied to shared memory once (uniform LDS instead of generic
  // loads from the parameter window)
  __shared__ KParams s_kp;
  if (threadIdx.x == 0) {
    s_kp = pp.p[second ? 1 : 0];
    s_kp.cta_G = second ? (int)gridDim.x - pp.grid0 : pp.grid0;
    s_kp.cta_c = second ? (int)blockIdx.x - pp.grid0 : (int)blockIdx.x;
  }
  __syncthreads();
  const KParams& p = s_kp;
  const CUtensorMap& tmA = second ? tmA1 : tmA0;
  const CUtensorMap& tmB = second ? tmB1 : tmB0;
  // (G, c) are read from shared memory where needed: keeping them live across the DMMA
  // loop costs accumulator registers
#define G (p.cta_G)
#define c (p.cta_c)
  constexpr int S = CF::STAGES;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // 1024-byte aligned stage ring (swizzle atoms); offsetting the shared array keeps
  // the fragment loads in the shared window (LDS, not generic LD)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  double* xs = reinterpret_cast<double*>(smem + (size_t)S * CF::STAGE_BYTES);  // EPI_ERR X tile
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * CF::STAGE_BYTES + CF::X_BYTES);
  uint64_t* empty = full + S;
  uint64_t* xfull = empty + S;
  uint64_t* xempty = xfull + 1;
  __shared__ unsigned s_flag;
  __shared__ double red[4][CF::CONSUMERS / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const Space<BM, BN> sp(p);
  {
    int sb, se;
    if (!cta_span(p, G, c, 0, sb, se) || sb >= se) return;
  }

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CF::CONSUMERS / 32);
    }
    mbar_init(xfull, 1);
    mbar_init(xempty, CF::CONSUMERS / 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp >= CF::CONSUMERS / 32) {
    // ------------------------------ TMA producer ------------------------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(CF::PRODUCER_REGS));
    if (warp == CF::CONSUMERS / 32 && lane == 0) {
      int stage = 0;
      unsigned phase = 0, xphase = 0;
      int sb, se;
      for (int sidx = 0; cta_span(p, G, c, sidx, sb, se); ++sidx) {
      int t, kb, nkb;
      sp.locate(sb, t, kb);
      nkb = sp.tile_nkb(t);
      for (int it = sb; it < se; ++it) {
        mbar_wait(&empty[stage], phase ^ 1u);
        unsigned char* As = smem + (size_t)stage * CF::STAGE_BYTES;
        unsigned char* Bs = As + CF::A_BYTES;
        mbar_expect_tx(&full[stage], CF::STAGE_BYTES);
        const int ty = t / p.gx, tx = t - ty * p.gx;
        const int i0 = ty * BM, jq0 = tx * (BN / 4), k0 = kb * kBKQ;
        if (OPA == 0) {  // two swizzled boxes [BM rows][4 quaternions]
          tma_load_2d(As, &tmA, k0 * 4, i0, &full[stage]);
          tma_load_2d(As + BM * 128, &tmA, k0 * 4 + 16, i0, &full[stage]);
        } else {  // k-major [8 k][64 quaternions] boxes
#pragma unroll
          for (int b = 0; b < BM / 64; ++b) tma_load_2d(As + b * 8 * 256 * 8, &tmA, (i0 + 64 * b) * 4, k0, &full[stage]);
        }
        if (OPB == 0) tma_load_2d(Bs, &tmB, jq0 * 4, k0, &full[stage]);  // [8 k][BN reals]
        else tma_load_2d(Bs, &tmB, k0 * 4, jq0, &full[stage]);           // [BN/4 j][8 quaternions]
        if (EPI != EPI_STORE && kb + 1 == nkb) {  // the tile's X block for the fused epilogue
          mbar_wait(xempty, xphase ^ 1u);
          mbar_expect_tx(xfull, CF::X_BYTES);
          tma_load_2d(xs, &tmX, tx * BN, i0, xfull);
          xphase ^= 1u;
        }
        sp.advance(t, kb, nkb);
        if (++stage == S) {
          stage = 0;
          phase ^= 1u;
        }
      }
      }
    }
    return;
  }

  // ------------------------------ DMMA warps ------------------------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(CF::CONSUMER_REGS));
  const int wm0 = (warp / CF::WARPS_N) * CF::WM;
  const int wn0 = (warp % CF::WARPS_N) * CF::WN;
  double acc[CF::FM][CF::FN][2];
#pragma unroll
  for (int a = 0; a < CF::FM; ++a)
#pragma unroll
    for (int b = 0; b < CF::FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  const int t4 = lane & 3, s4 = (lane >> 2) & 3, jl = lane >> 4;
  const unsigned long long bsign =
      (((OPB == 0 ? kSignN : kSignH) >> (t4 * 4 + s4)) & 1u) ? 0x8000000000000000ull : 0ull;
  const unsigned long long asign = (OPA == 1 && t4 != 0) ? 0x8000000000000000ull : 0ull;
  const int arow = lane >> 2;
  const int tcomp = t4 ^ s4;

  int stage = 0;
  unsigned phase = 0;
  unsigned xphase = 0;
  int ib, ie;
  // the fused-epilogue kernels run one contiguous span: a constant trip count keeps their
  // loop as simple as a single-span kernel's
  constexpr int kMaxSpans = EPI == EPI_STORE ? (1 << 30) : 1;
  for (int sidx = 0; sidx < kMaxSpans && cta_span(p, G, c, sidx, ib, ie); ++sidx) {
  int ct, ckb, cnkb;
  sp.locate(ib, ct, ckb);
  cnkb = sp.tile_nkb(ct);
  int seg_begin = ib;
  for (int it = ib; it < ie; ++it) {
    mbar_wait(&full[stage], phase);
    const double* As = reinterpret_cast<const double*>(smem + (size_t)stage * CF::STAGE_BYTES);
    const double* Bs = reinterpret_cast<const double*>(smem + (size_t)stage * CF::STAGE_BYTES + CF::A_BYTES);
#pragma unroll
    for (int kk = 0; kk < kBKQ; ++kk) {
      double af[CF::FM], bf[CF::FN];
#pragma unroll
      for (int a = 0; a < CF::FM; ++a) {
        const int i = wm0 + 8 * a + arow;
        double v;
        if (OPA == 0) {
          const int chunk = ((kk & 3) * 2 + (t4 >> 1)) ^ (i & 7);
          v = As[(kk >> 2) * BM * 16 + i * 16 + chunk * 2 + (t4 & 1)];
        } else {
          v = As[(i >> 6) * 2048 + kk * 256 + (i & 63) * 4 + t4];
        }
        af[a] = OPA == 1 ? flip(v, asign) : v;
      }
#pragma unroll
      for (int b = 0; b < CF::FN; ++b) {
        double v;
        if (OPB == 0) v = Bs[kk * BN + wn0 + 8 * b + jl * 4 + tcomp];
        else v = Bs[((wn0 + 8 * b) / 4 + jl) * 32 + kk * 4 + tcomp];
        bf[b] = flip(v, bsign);
      }
#pragma unroll
      for (int a = 0; a < CF::FM; ++a)
#pragma unroll
        for (int b = 0; b < CF::FN; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[stage]);
    if (++stage == S) {
      stage = 0;
      phase ^= 1u;
    }

    const bool tile_done = ckb + 1 == cnkb;
    if (tile_done || it + 1 == ie) {
      // ---------------- epilogue of tile ct ----------------
      const int ty = ct / p.gx, tx = ct - ty * p.gx;
      const int64_t i0 = (int64_t)ty * BM, jr0 = (int64_t)tx * BN;
      const int64_t Nr = 4 * p.Nq;
      const int tile_first = it - ckb;  // iteration of the tile's k-block 0
      const bool whole = tile_done && seg_begin == tile_first;
      if (EPI == EPI_STORE) {
        if (whole) {
#pragma unroll
          for (int a = 0; a < CF::FM; ++a) {
            const int64_t gi = i0 + wm0 + 8 * a + arow;
            if (gi >= p.Mq) continue;
#pragma unroll
            for (int b = 0; b < CF::FN; ++b) {
              const int64_t gj = jr0 + wn0 + 8 * b + 2 * t4;
              if (gj >= Nr) continue;
              double* cp = p.C + gi * p.ldc * 4 + gj;
              double2 v = make_double2(p.alpha * acc[a][b][0], p.alpha * acc[a][b][1]);
              if (p.beta != 0.0) {
                const double2 o = *reinterpret_cast<const double2*>(cp);
                v.x += p.beta * o.x;
                v.y += p.beta * o.y;
              }
              *reinterpret_cast<double2*>(cp) = v;
            }
          }
        } else {
          // park the partial tile: slot 0 if this is the CTA's first tile, else slot 1
          const int slot = (p.mode == MODE_SPLIT || seg_begin == ib) ? 0 : 1;
          double* sl = p.slots + (int64_t)(c * 2 + slot) * (BM * BN);
#pragma unroll
          for (int a = 0; a < CF::FM; ++a)
#pragma unroll
            for (int b = 0; b < CF::FN; ++b)
              __stcg(reinterpret_cast<double2*>(sl + (wm0 + 8 * a + arow) * BN + wn0 + 8 * b + 2 * t4),
                     make_double2(acc[a][b][0], acc[a][b][1]));
          __threadfence();
          consumer_sync<CF::CONSUMERS>();
          if (p.mode == MODE_SPLIT) {
            // the last of the tile's S parts to arrive adds all S in split order (no CTA
            // ever waits for another, so no co-residency assumption)
            int o, z_, nsp, first;
            split_of(p, c, o, z_, nsp, first);
            if (tid == 0) s_flag = (atomicAdd(&p.counters[ct], 1u) == (unsigned)nsp - 1) ? 1u : 0u;
            consumer_sync<CF::CONSUMERS>();
            if (s_flag) {
              __threadfence();
              for (int idx = tid; idx < BM * (BN / 2); idx += CF::CONSUMERS) {
                const int r = idx / (BN / 2), cc = 2 * (idx % (BN / 2));
                const int64_t gi = i0 + r, gj = jr0 + cc;
                if (gi >= p.Mq || gj >= Nr) continue;
                const double* base = p.slots + (int64_t)first * 2 * (BM * BN) + r * BN + cc;
                double sx = 0.0, sy = 0.0;
                for (int k = 0; k < nsp; k += 8) {
                  double2 v[8];
#pragma unroll
                  for (int u = 0; u < 8; ++u)
                    if (k + u < nsp)
                      v[u] = __ldcg(reinterpret_cast<const double2*>(base + (int64_t)(k + u) * 2 * (BM * BN)));
#pragma unroll
                  for (int u = 0; u < 8; ++u)
                    if (k + u < nsp) {
                      sx += v[u].x;
                      sy += v[u].y;
                    }
                }
                double* cp = p.C + gi * p.ldc * 4 + gj;
                double2 ov = make_double2(p.alpha * sx, p.alpha * sy);
                if (p.beta != 0.0) {
                  const double2 old = *reinterpret_cast<const double2*>(cp);
                  ov.x += p.beta * old.x;
                  ov.y += p.beta * old.y;
                }
                *reinterpret_cast<double2*>(cp) = ov;
              }
              if (tid == 0) p.counters[ct] = 0u;
            }
            // s_flag is rewritten at this CTA's next partial tile, which a fast warp can
            // reach while others still read it here (short tiles fit in the stage ring)
            consumer_sync<CF::CONSUMERS>();
          } else {
            if (tid == 0) {
              const unsigned mine = (unsigned)(it + 1 - seg_begin);
              s_flag = (atomicAdd(&p.counters[ct], mine) + mine == (unsigned)cnkb) ? 1u : 0u;
            }
            consumer_sync<CF::CONSUMERS>();
            if (s_flag) {
              __threadfence();
              // contributors (stream-K tail, iterations counted from its base): CTAs k0..k1 in
              // k order; CTA k's part sits in slot 0 when its span starts inside this tile,
              // else in slot 1
              const int base = p.waves * G * p.nkb_full;
              const int64_t T = (int64_t)p.total - base;
              const int64_t tf = tile_first - base, tile_end = tf + cnkb;
              const int k0 = (int)(((tf + 1) * G - 1) / T), k1 = (int)((tile_end * G - 1) / T);
              for (int idx = tid; idx < BM * (BN / 2); idx += CF::CONSUMERS) {
                const int r = idx / (BN / 2), cc = 2 * (idx % (BN / 2));
                const int64_t gi = i0 + r, gj = jr0 + cc;
                if (gi >= p.Mq || gj >= Nr) continue;
                double sx = 0.0, sy = 0.0;
                for (int k = k0; k <= k1; k += 4) {
                  double2 v[4];
#pragma unroll
                  for (int u = 0; u < 4; ++u)
                    if (k + u <= k1) {
                      const int64_t ks = (int64_t)(k + u) * T / G;
                      const int sl2 = ks >= tf ? 0 : 1;
                      v[u] = __ldcg(reinterpret_cast<const double2*>(p.slots + (int64_t)((k + u) * 2 + sl2) * (BM * BN) +
                                                                     r * BN + cc));
                    }
#pragma unroll
                  for (int u = 0; u < 4; ++u)
                    if (k + u <= k1) {
                      sx += v[u].x;
                      sy += v[u].y;
                    }
                }
                double* cp = p.C + gi * p.ldc * 4 + gj;
                double2 ov = make_double2(p.alpha * sx, p.alpha * sy);
                if (p.beta != 0.0) {
                  const double2 old = *reinterpret_cast<const double2*>(cp);
                  ov.x += p.beta * old.x;
                  ov.y += p.beta * old.y;
                }
                *reinterpret_cast<double2*>(cp) = ov;
              }
              if (tid == 0) p.counters[ct] = 0u;
            }
            // s_flag is rewritten at this CTA's next partial tile, which a fast warp can
            // reach while others still read it here (short tiles fit in the stage ring)
            consumer_sync<CF::CONSUMERS>();
          }
        }
      } else if (EPI == EPI_COMPLETE) {
        // completion sweep (completion.py:214-219): out = observed ? Y : (P R) written
        // back, per tile [0] sum (out - X)^2 (the step), [1] sum X^2 (the scale), X being
        // the current iterate (TMA-staged like the error kernel's X block)
        double v[2] = {0.0, 0.0};
        mbar_wait(xfull, xphase);
        xphase ^= 1u;
#pragma unroll
        for (int a = 0; a < CF::FM; ++a) {
          const int64_t gi = i0 + wm0 + 8 * a + arow;
#pragma unroll
          for (int b = 0; b < CF::FN; ++b) {
            const int64_t gj = jr0 + wn0 + 8 * b + 2 * t4;
            if (gi < p.Mq && gj < Nr) {
              const double2 x =
                  *reinterpret_cast<const double2*>(xs + (wm0 + 8 * a + arow) * BN + wn0 + 8 * b + 2 * t4);
              double2 o = make_double2(p.alpha * acc[a][b][0], p.alpha * acc[a][b][1]);
              if (p.mask[gi * p.Nq + (gj >> 2)]) o = __ldg(reinterpret_cast<const double2*>(p.Y + gi * p.ldx * 4 + gj));
              *reinterpret_cast<double2*>(p.C + gi * p.ldc * 4 + gj) = o;
              const double d0 = o.x - x.x, d1 = o.y - x.y;
              v[0] += d0 * d0;
              v[0] += d1 * d1;
              v[1] += x.x * x.x;
              v[1] += x.y * x.y;
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(xempty);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          v[k] = warp_sum(v[k]);
          if (lane == 0) red[k][warp] = v[k];
        }
        consumer_sync<CF::CONSUMERS>();
        if (tid < 4) {
          double acc4 = 0.0;
          if (tid < 2)
            for (int w2 = 0; w2 < CF::CONSUMERS / 32; ++w2) acc4 += red[tid][w2];
          p.partials[4 * ct + tid] = acc4;
        }
        consumer_sync<CF::CONSUMERS>();
      } else {
        // per tile: [0] sum (X - PR)^2, [1] sum X^2, [2] sum over the imaginary
        // components of (X - PR)^2 (float PSNR), [3] sum of squared differences of
        // the u8 images rint(clip(s X, 0, 255)) vs rint(clip(s PR, 0, 255)) over the
        // imaginary components (imaging.py:90-124 semantics; integers, exact in fp64)
        const double sc = p.psnr_scale;
        double v[4] = {0.0, 0.0, 0.0, 0.0};
        mbar_wait(xfull, xphase);
        xphase ^= 1u;
#pragma unroll
        for (int a = 0; a < CF::FM; ++a) {
          const int64_t gi = i0 + wm0 + 8 * a + arow;
#pragma unroll
          for (int b = 0; b < CF::FN; ++b) {
            const int64_t gj = jr0 + wn0 + 8 * b + 2 * t4;
            if (gi < p.Mq && gj < Nr) {
              const double2 x =
                  *reinterpret_cast<const double2*>(xs + (wm0 + 8 * a + arow) * BN + wn0 + 8 * b + 2 * t4);
              const double r0 = p.alpha * acc[a][b][0], r1 = p.alpha * acc[a][b][1];
              const double d0 = x.x - r0, d1 = x.y - r1;
              v[0] += d0 * d0;
              v[0] += d1 * d1;
              v[1] += x.x * x.x;
              v[1] += x.y * x.y;
              const bool first_real = (gj & 3) == 0;  // (gj, gj+1) = components (0,1) or (2,3)
              if (!first_real) v[2] += d0 * d0;
              v[2] += d1 * d1;
              if (sc > 0.0) {
                auto u8 = [&](double z) { return rint(fmin(fmax(sc * z, 0.0), 255.0)); };
                const double q1 = u8(x.y) - u8(r1);
                v[3] += q1 * q1;
                if (!first_real) {
                  const double q0 = u8(x.x) - u8(r0);
                  v[3] += q0 * q0;
                }
              }
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(xempty);  // X block consumed
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          v[k] = warp_sum(v[k]);
          if (lane == 0) red[k][warp] = v[k];
        }
        consumer_sync<CF::CONSUMERS>();
        if (tid < 4) {
          double acc4 = 0.0;
          for (int w2 = 0; w2 < CF::CONSUMERS / 32; ++w2) acc4 += red[tid][w2];
          p.partials[4 * ct + tid] = acc4;
        }
        consumer_sync<CF::CONSUMERS>();  // red[] is reused by the next tile
      }
#pragma unroll
      for (int a = 0; a < CF::FM; ++a)
#pragma unroll
        for (int b = 0; b < CF::FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
      seg_begin = it + 1;
    }
    sp.advance(ct, ckb, cnkb);
  }
  }
}

#undef G
#undef c

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      f = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  }();
  return fn;
}

// 2-D float64 tensor map: inner extent `w` doubles, `h` rows, row pitch `pitch_q`
// quaternions, box (bw, bh)
bool make_map(CUtensorMap* m, const double* base, int64_t w, int64_t h, int64_t pitch_q, int bw, int bh, bool swz) {
  auto enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)(w > 0 ? w : 1), (cuuint64_t)(h > 0 ? h : 1)};
  cuuint64_t strides[1] = {(cuuint64_t)(pitch_q * 32)};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BM, int BN>
bool make_maps(const double* A, int64_t lda, int opA, const double* B, int64_t ldb, int opB, int64_t Mq, int64_t Nq,
               int64_t Kq, CUtensorMap* ta, CUtensorMap* tb) {
  bool ok;
  if (opA == 0) ok = make_map(ta, A, 4 * Kq, Mq, lda, 16, BM, true);  // A: Mq x Kq
  else ok = make_map(ta, A, 4 * Mq, Kq, lda, 256, kBKQ, false);     // A stored Kq x Mq
  if (opB == 0) ok = ok && make_map(tb, B, 4 * Nq, Kq, ldb, BN, kBKQ, false);       // B: Kq x Nq
  else ok = ok && make_map(tb, B, 4 * Kq, Nq, ldb, 4 * kBKQ, BN / 4, false);        // B stored Nq x Kq
  return ok;
}

int num_sms() {
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  return sms;
}

struct TileCfg {
  int bm, bn;
};
// 0: 64 x 128, 1: 64 x 160 (9 warps at one CTA per SM leave 168 registers per thread:
// the 32 x 40 warp tile's 80 accumulator registers fit without spills)
constexpr TileCfg kCfgs[2] = {{64, 128}, {64, 160}};

int pick_cfg(int64_t Mq, int64_t Nq) {
  static const int forced = [] {
    const char* e = getenv("QCUR_GEMM_CFG");  // experiments only: force one tile configuration
    return e ? atoi(e) : -1;
  }();
  if (forced >= 0 && forced < 2) return forced;
  (void)Mq;
  const int64_t Nr = 4 * Nq;
  const int64_t pad128 = (Nr + 127) / 128 * 128, pad160 = (Nr + 159) / 160 * 160;
  return pad160 < pad128 ? 1 : 0;
}

int64_t host_total(const TileCfg& c, int64_t gx, int64_t gy, int64_t nkb_full, int b_upper, int herm) {
  const int64_t W = c.bn / 4, w = W / kBKQ;
  auto nkb_col = [&](int64_t tx) {
    if (!b_upper) return nkb_full;
    const int64_t v = (tx + 1) * w;
    return v < nkb_full ? v : nkb_full;
  };
  if (!herm && !b_upper) return gy * gx * nkb_full;
  int64_t total = 0;
  for (int64_t ty = 0; ty < gy; ++ty) {
    int64_t L = gx - 1;
    if (herm) {
      const int64_t l = (ty * c.bm + c.bm - 1) / W;
      L = l < L ? l : L;
    }
    int64_t row = 0;
    for (int64_t tx = 0; tx <= L; ++tx) row += nkb_col(tx);
    if (!herm) return row * gy;  // identical rows
    total += row;
  }
  return total;
}

int64_t host_active_tiles(const TileCfg& c, int64_t gx, int64_t gy, int herm) {
  if (!herm) return gx * gy;
  int64_t n = 0;
  for (int64_t ty = 0; ty < gy; ++ty) {
    const int64_t l = (ty * c.bm + c.bm - 1) / (c.bn / 4);
    n += (l < gx - 1 ? l : gx - 1) + 1;
  }
  return n;
}

bool no_split() {
  static const bool v = getenv("QCUR_NO_SPLIT") != nullptr;  // experiments only
  return v;
}

struct Plan {
  int cfg;
  KParams kp;
  int grid;
  size_t slot_bytes;
};

Plan make_plan(const GemmArgs& g, int64_t gmax = 0) {
  Plan pl{};
  pl.cfg = pick_cfg(g.Mq, g.Nq);
  const TileCfg& c = kCfgs[pl.cfg];
  KParams& kp = pl.kp;
  kp.Mq = g.Mq;
  kp.Nq = g.Nq;
  kp.Kq = g.Kq;
  kp.C = g.C;
  kp.ldc = g.ldc;
  kp.alpha = g.alpha;
  kp.beta = g.beta;
  kp.b_upper = g.b_upper;
  kp.herm_lower = g.herm_lower;
  kp.gx = (int)((4 * g.Nq + c.bn - 1) / c.bn);
  kp.gy = (int)((g.Mq + c.bm - 1) / c.bm);
  kp.nkb_full = g.Kq > 0 ? (int)((g.Kq + kBKQ - 1) / kBKQ) : 1;
  kp.total = (int)host_total(c, kp.gx, kp.gy, kp.nkb_full, g.b_upper, g.herm_lower);
  const int64_t G = gmax > 0 ? gmax : num_sms();
  const int64_t ntiles = (int64_t)kp.gx * kp.gy;
  const int64_t active = host_active_tiles(c, kp.gx, kp.gy, g.herm_lower);
  int64_t grid;
  if (ntiles > 65536 || (g.whole_tiles && !g.b_upper && !g.herm_lower)) {
    // beyond the ticket array, or asked for: whole tiles per CTA (uniform tiles only)
    kp.mode = MODE_TILES;
    grid = (!g.b_upper && !g.herm_lower) ? (ntiles < G ? ntiles : G) : 1;
  } else if (!no_split() && 2 * active <= G && kp.nkb_full >= 2) {
    // few tiles: cut each into equal k ranges.  A triangular op(B) runs at full depth
    // here (its zero triangle is stored as zeros, so the extra products add exact zeros)
    kp.mode = MODE_SPLIT;
    kp.b_upper = 0;
    kp.total = (int)host_total(c, kp.gx, kp.gy, kp.nkb_full, 0, g.herm_lower);
    // S_t = G / active splits, one more on the first G % active tiles: every SM busy
    int64_t sp = G / active, extra = G % active;
    if (sp >= kp.nkb_full) {
      sp = kp.nkb_full;
      extra = 0;
    }
    kp.splits = (int)sp;
    kp.split_extra = (int)extra;
    grid = active * sp + extra;
  } else {
    kp.mode = MODE_STREAMK;
    grid = (kp.total + 3) / 4;  // >= 4 k-blocks per CTA
    if (grid > G) grid = G;
    // deep uniform GEMMs (X Q_R): whole-tile rounds first so the X row blocks are read
    // from HBM about once; stream-K only over the remainder
    if (!g.b_upper && !g.herm_lower && grid == G && kp.nkb_full >= 64) kp.waves = (int)(ntiles / G);
  }
  if (grid < 1) grid = 1;
  pl.grid = (int)grid;
  pl.slot_bytes = kp.mode == MODE_TILES ? 0 : (size_t)grid * 2 * c.bm * c.bn * sizeof(double);
  return pl;
}

template <int BM, int BN, int OPA, int OPB, int EPI>
void launch_k2(const CUtensorMap* ta, const CUtensorMap* tb, const CUtensorMap& tx, const KPair& kp, int grid,
               cudaStream_t st) {
  using CF = Cfg<BM, BN, EPI>;
  auto fn = qgemm_kernel<BM, BN, OPA, OPB, EPI>;
  static std::atomic<unsigned> set{0};
  if (first_on_device(set)) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
  }
  ++::qcur::g_launches;
  fn<<<grid, CF::THREADS, CF::SMEM, st>>>(ta[0], tb[0], ta[1], tb[1], tx, kp);
}

template <int BM, int BN, int OPA, int OPB, int EPI>
void launch_k(const CUtensorMap& ta, const CUtensorMap& tb, const CUtensorMap& tx, const KParams& kp, int grid,
              cudaStream_t st) {
  const CUtensorMap a[2] = {ta, ta}, b[2] = {tb, tb};
  KPair pr;
  pr.p[0] = pr.p[1] = kp;
  pr.grid0 = grid;
  launch_k2<BM, BN, OPA, OPB, EPI>(a, b, tx, pr, grid, st);
}

// one or two problems (same ops and tile configuration) in one launch
template <int BM, int BN>
void launch_cfg(const GemmArgs* g, const KParams* kp, const int* grid, int np, cudaStream_t st) {
  CUtensorMap ta[2], tb[2];
  for (int k = 0; k < np; ++k)
    if (!make_maps<BM, BN>(g[k].A, g[k].lda, g[k].opA, g[k].B, g[k].ldb, g[k].opB, g[k].Mq, g[k].Nq, g[k].Kq,
                           &ta[k], &tb[k])) {
      // surfaces through the caller's launch check as a CUDA error
      cudaLaunchKernel((const void*)nullptr, dim3(1), dim3(1), nullptr, 0, st);
      return;
    }
  if (np == 1) {
    ta[1] = ta[0];
    tb[1] = tb[0];
  }
  KPair pr;
  pr.p[0] = kp[0];
  pr.p[1] = kp[np - 1];
  pr.grid0 = grid[0];
  const int total = np == 1 ? grid[0] : grid[0] + grid[1];
  const int opA = g[0].opA, opB = g[0].opB;
  if (opA == 0 && opB == 0) launch_k2<BM, BN, 0, 0, EPI_STORE>(ta, tb, tb[0], pr, total, st);
  else if (opA == 0) launch_k2<BM, BN, 0, 1, EPI_STORE>(ta, tb, tb[0], pr, total, st);
  else if (opB == 0) launch_k2<BM, BN, 1, 0, EPI_STORE>(ta, tb, tb[0], pr, total, st);
  else launch_k2<BM, BN, 1, 1, EPI_STORE>(ta, tb, tb[0], pr, total, st);
}

}  // namespace

size_t qgemm_workspace_bytes(const GemmArgs& g) { return make_plan(g).slot_bytes; }

void launch_qgemm(const GemmArgs& g, double* workspace, unsigned* counters, cudaStream_t st) {
  if (g.Mq <= 0 || g.Nq <= 0) return;
  if (g.Kq > 0 && qgemm_small_ok(g)) {  // q x q products: one cluster per 32 x 32 tile (k_qgemm_small.cu)
    launch_qgemm_small(&g, 1, st);
    return;
  }
  Plan pl = make_plan(g);
  pl.kp.counters = counters;
  pl.kp.slots = workspace;
  if (pl.kp.mode != MODE_TILES && pl.grid > 1 && (!workspace || !counters)) {  // no workspace: one span
    pl.kp.mode = MODE_STREAMK;
    pl.grid = 1;
  }
  if (pl.cfg == 1) launch_cfg<64, 160>(&g, &pl.kp, &pl.grid, 1, st);
  else launch_cfg<64, 128>(&g, &pl.kp, &pl.grid, 1, st);
}

void launch_qgemm_pair(const GemmArgs& g0, double* ws0, const GemmArgs& g1, double* ws1, unsigned* counters,
                       cudaStream_t st) {
  if (qgemm_small_ok(g0) && qgemm_small_ok(g1) && g0.Kq > 0 && g1.Kq > 0 && g0.opA == g1.opA && g0.opB == g1.opB) {
    const GemmArgs g[2] = {g0, g1};
    launch_qgemm_small(g, 2, st);
    return;
  }
  static const bool no_pair = getenv("QCUR_NO_PAIR") != nullptr;  // experiments only
  const bool same = !no_pair && g0.opA == g1.opA && g0.opB == g1.opB && pick_cfg(g0.Mq, g0.Nq) == pick_cfg(g1.Mq, g1.Nq) &&
                    g0.Mq > 0 && g0.Nq > 0 && g1.Mq > 0 && g1.Nq > 0 && ws0 && ws1 && counters;
  if (!same) {
    launch_qgemm(g0, ws0, counters, st);
    launch_qgemm(g1, ws1, counters, st);
    return;
  }
  // split the SMs in proportion to the two problems' k-block counts
  const int64_t G = num_sms();
  const int64_t t0 = make_plan(g0).kp.total, t1 = make_plan(g1).kp.total;
  int64_t G0 = (G * t0 + (t0 + t1) / 2) / (t0 + t1 > 0 ? t0 + t1 : 1);
  if (G0 < 1) G0 = 1;
  if (G0 > G - 1) G0 = G - 1;
  Plan pl[2] = {make_plan(g0, G0), make_plan(g1, G - G0)};
  if (pl[0].kp.mode == MODE_TILES || pl[1].kp.mode == MODE_TILES) {
    launch_qgemm(g0, ws0, counters, st);
    launch_qgemm(g1, ws1, counters, st);
    return;
  }
  pl[0].kp.counters = counters;
  pl[1].kp.counters = counters + 32768;  // tickets 32768.., done counters 98304..
  pl[0].kp.slots = ws0;
  pl[1].kp.slots = ws1;
  const GemmArgs g[2] = {g0, g1};
  const KParams kp[2] = {pl[0].kp, pl[1].kp};
  const int grid[2] = {pl[0].grid, pl[1].grid};
  if (pl[0].cfg == 1) launch_cfg<64, 160>(g, kp, grid, 2, st);
  else launch_cfg<64, 128>(g, kp, grid, 2, st);
}

// error kernel: 64 x 160 tiles when 4n is a multiple of 160, else 64 x 128
namespace {
int err_bn(int64_t n) { return (4 * n) % 160 == 0 ? 160 : 128; }
}  // namespace

int64_t err_partials_count(int64_t m, int64_t n) {
  const int bn = err_bn(n);
  return ((4 * n + bn - 1) / bn) * ((m + 64 - 1) / 64);
}

void launch_cur_error(const double* X, int64_t ldx, const double* P, int64_t ldp, const double* R, int64_t ldr,
                      int64_t m, int64_t n, int64_t r, double psnr_scale, double* partials, double* out4,
                      cudaStream_t st) {
  const int bn = err_bn(n);
  KParams kp{};
  kp.Mq = m;
  kp.Nq = n;
  kp.Kq = r;
  kp.alpha = 1.0;
  kp.X = X;
  kp.ldx = ldx;
  kp.partials = partials;
  kp.psnr_scale = psnr_scale;
  kp.gx = (int)((4 * n + bn - 1) / bn);
  kp.gy = (int)((m + 64 - 1) / 64);
  kp.nkb_full = r > 0 ? (int)((r + kBKQ - 1) / kBKQ) : 1;
  kp.total = (int)((int64_t)kp.gx * kp.gy * kp.nkb_full);
  kp.mode = MODE_TILES;
  const int64_t ntiles = (int64_t)kp.gx * kp.gy, G = num_sms();
  const int grid = (int)(ntiles < G ? ntiles : G);
  CUtensorMap ta, tb, tx;
  bool ok;
  if (bn == 160) {
    ok = make_maps<64, 160>(P, ldp, 0, R, ldr, 0, m, n, r, &ta, &tb) &&
         make_map(&tx, X, 4 * n, m, ldx, 160, 64, false);
    if (ok) launch_k<64, 160, 0, 0, EPI_ERR>(ta, tb, tx, kp, grid, st);
  } else {
    ok = make_maps<64, 128>(P, ldp, 0, R, ldr, 0, m, n, r, &ta, &tb) &&
         make_map(&tx, X, 4 * n, m, ldx, 128, 64, false);
    if (ok) launch_k<64, 128, 0, 0, EPI_ERR>(ta, tb, tx, kp, grid, st);
  }
  if (!ok) cudaLaunchKernel((const void*)nullptr, dim3(1), dim3(1), nullptr, 0, st);
  launch_reduce_rows(partials, ntiles, 4, out4, st);
}

void launch_complete_step(const double* X, const double* Y, const unsigned char* mask, int64_t ld, const double* P,
                          int64_t ldp, const double* R, int64_t ldr, int64_t m, int64_t n, int64_t r, double* out,
                          double* partials, double* out4, cudaStream_t st) {
  const int bn = err_bn(n);
  KParams kp{};
  kp.Mq = m;
  kp.Nq = n;
  kp.Kq = r;
  kp.alpha = 1.0;
  kp.X = X;
  kp.ldx = ld;
  kp.Y = Y;
  kp.mask = mask;
  kp.C = out;
  kp.ldc = ld;
  kp.partials = partials;
  kp.gx = (int)((4 * n + bn - 1) / bn);
  kp.gy = (int)((m + 64 - 1) / 64);
  kp.nkb_full = r > 0 ? (int)((r + kBKQ - 1) / kBKQ) : 1;
  kp.total = (int)((int64_t)kp.gx * kp.gy * kp.nkb_full);
  kp.mode = MODE_TILES;
  const int64_t ntiles = (int64_t)kp.gx * kp.gy, G = num_sms();
  const int grid = (int)(ntiles < G ? ntiles : G);
  CUtensorMap ta, tb, tx;
  bool ok;
  if (bn == 160) {
    ok = make_maps<64, 160>(P, ldp, 0, R, ldr, 0, m, n, r, &ta, &tb) && make_map(&tx, X, 4 * n, m, ld, 160, 64, false);
    if (ok) launch_k<64, 160, 0, 0, EPI_COMPLETE>(ta, tb, tx, kp, grid, st);
  } else {
    ok = make_maps<64, 128>(P, ldp, 0, R, ldr, 0, m, n, r, &ta, &tb) && make_map(&tx, X, 4 * n, m, ld, 128, 64, false);
    if (ok) launch_k<64, 128, 0, 0, EPI_COMPLETE>(ta, tb, tx, kp, grid, st);
  }
  if (!ok) cudaLaunchKernel((const void*)nullptr, dim3(1), dim3(1), nullptr, 0, st);
  launch_reduce_rows(partials, ntiles, 4, out4, st);
}

}  // namespace qcur
