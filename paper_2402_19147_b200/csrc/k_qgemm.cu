// Quaternion GEMM on the FP64 tensor path (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4).
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
// op(A)=H / op(B)=H are the same loads with a transposed placement and the
// conjugate sign table.
//
// Tiles: BM x BN reals per CTA, WM x WN per warp, BKQ quaternions of K per
// cp.async stage (zero-filled at the edges), STAGES-deep pipeline.  Split-K
// writes fixed partial slabs reduced in a fixed order, so every result is
// bitwise deterministic run to run (test_cur.py:243-250).
//
// EPI_ERR fuses the error of the reference's caller (cli.py:173-175,
// imaging.py:170-177): the tile of (P R) is subtracted from the matching tile
// of X in registers and only sum((X - PR)^2) and sum(X^2) leave the CTA, so
// CUR is never written to HBM.
#include "common.cuh"
#include "kernels.h"

namespace qcur {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
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

enum { EPI_STORE = 0, EPI_ERR = 1 };

template <int BM, int BN, int WM, int WN, int BKQ, int STAGES, int OPA, int OPB, int EPI>
struct Cfg {
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int THREADS = WARPS_M * WARPS_N * 32;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int AS = 4 * BKQ + 4;  // padded row stride (doubles): conflict-free A fragments
  static constexpr int A_ELEMS = BM * AS;
  static constexpr int B_ELEMS = BKQ * BN;
  static constexpr int STAGE_ELEMS = A_ELEMS + B_ELEMS;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_ELEMS * sizeof(double);
};

struct KParams {
  int64_t Mq, Nq, Kq;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  double alpha, beta;
  double* work;        // split-K slabs [splits][Mq][4Nq], or null
  int64_t kchunk;      // quaternions of K per split
  const double* X;     // EPI_ERR: reference matrix
  int64_t ldx;
  double* partials;    // EPI_ERR: [tiles][2]
};

template <int BM, int BN, int WM, int WN, int BKQ, int STAGES, int OPA, int OPB, int EPI>
__global__ void __launch_bounds__(Cfg<BM, BN, WM, WN, BKQ, STAGES, OPA, OPB, EPI>::THREADS, 2)
    qgemm_kernel(KParams p) {
  using CF = Cfg<BM, BN, WM, WN, BKQ, STAGES, OPA, OPB, EPI>;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm0 = (warp / CF::WARPS_N) * WM;
  const int wn0 = (warp % CF::WARPS_N) * WN;
  const int64_t i0 = (int64_t)blockIdx.y * BM;   // quaternion rows
  const int64_t jr0 = (int64_t)blockIdx.x * BN;  // real columns
  const int64_t jq0 = jr0 / 4;
  const int64_t kbeg = (int64_t)blockIdx.z * p.kchunk;
  int64_t kend = kbeg + p.kchunk;
  if (kend > p.Kq) kend = p.Kq;
  const int nkb = (int)((kend - kbeg + BKQ - 1) / BKQ);

  auto load_stage = [&](int buf, int64_t k0) {
    double* As = smem + buf * CF::STAGE_ELEMS;
    double* Bs = As + CF::A_ELEMS;
    // A tile: BM rows x BKQ quaternions = BM*BKQ*2 16-byte chunks
    constexpr int ACH = BM * BKQ * 2;
    for (int id = tid; id < ACH; id += CF::THREADS) {
      int row, kq, half;
      if (OPA == 0) {
        row = id / (2 * BKQ);
        int cc = id % (2 * BKQ);
        kq = cc >> 1;
        half = cc & 1;
      } else {
        kq = id / (2 * BM);
        int rem = id % (2 * BM);
        row = rem >> 1;
        half = rem & 1;
      }
      const int64_t gi = i0 + row, gk = k0 + kq;
      const bool v = gi < p.Mq && gk < kend;
      const double* src = p.A;
      if (v) src = (OPA == 0) ? p.A + (gi * p.lda + gk) * 4 + half * 2 : p.A + (gk * p.lda + gi) * 4 + half * 2;
      cp_async16(As + row * CF::AS + kq * 4 + half * 2, src, v);
    }
    // B tile: BKQ x (BN/4) quaternions
    constexpr int BCH = BKQ * (BN / 4) * 2;
    for (int id = tid; id < BCH; id += CF::THREADS) {
      int kq, jq, half;
      if (OPB == 0) {
        kq = id / (BN / 2);
        int cc = id % (BN / 2);
        jq = cc >> 1;
        half = cc & 1;
      } else {
        jq = id / (2 * BKQ);
        int rem = id % (2 * BKQ);
        kq = rem >> 1;
        half = rem & 1;
      }
      const int64_t gk = k0 + kq, gj = jq0 + jq;
      const bool v = gk < kend && gj < p.Nq;
      const double* src = p.B;
      if (v) src = (OPB == 0) ? p.B + (gk * p.ldb + gj) * 4 + half * 2 : p.B + (gj * p.ldb + gk) * 4 + half * 2;
      cp_async16(Bs + kq * BN + jq * 4 + half * 2, src, v);
    }
  };

  double acc[CF::FM][CF::FN][2];
#pragma unroll
  for (int a = 0; a < CF::FM; ++a)
#pragma unroll
    for (int b = 0; b < CF::FN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  // per-lane fragment constants
  const int t = lane & 3, s = (lane >> 2) & 3, jl = lane >> 4;
  const unsigned smask = OPB == 0 ? kSignN : kSignH;
  const unsigned long long bsign = ((smask >> (t * 4 + s)) & 1u) ? 0x8000000000000000ull : 0ull;
  const int boff = jl * 4 + (t ^ s);
  const unsigned long long asign = (OPA == 1 && t != 0) ? 0x8000000000000000ull : 0ull;
  const int arow = lane >> 2;

#pragma unroll
  for (int st = 0; st < STAGES - 1; ++st) {
    if (st < nkb) load_stage(st, kbeg + (int64_t)st * BKQ);
    cp_async_commit();
  }
  for (int kb = 0; kb < nkb; ++kb) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kb + STAGES - 1;
      if (nk < nkb) load_stage(nk % STAGES, kbeg + (int64_t)nk * BKQ);
      cp_async_commit();
    }
    const double* As = smem + (kb % STAGES) * CF::STAGE_ELEMS;
    const double* Bs = As + CF::A_ELEMS;
#pragma unroll
    for (int kk = 0; kk < BKQ; ++kk) {
      double af[CF::FM], bf[CF::FN];
#pragma unroll
      for (int a = 0; a < CF::FM; ++a) {
        double v = As[(wm0 + 8 * a + arow) * CF::AS + kk * 4 + t];
        af[a] = OPA == 1 ? flip(v, asign) : v;
      }
#pragma unroll
      for (int b = 0; b < CF::FN; ++b) bf[b] = flip(Bs[kk * BN + wn0 + 8 * b + boff], bsign);
#pragma unroll
      for (int a = 0; a < CF::FM; ++a)
#pragma unroll
        for (int b = 0; b < CF::FN; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
  }
  cp_async_wait<0>();

  if (EPI == EPI_STORE) {
    const int64_t Nr = 4 * p.Nq;
#pragma unroll
    for (int a = 0; a < CF::FM; ++a) {
      const int64_t gi = i0 + wm0 + 8 * a + arow;
      if (gi >= p.Mq) continue;
#pragma unroll
      for (int b = 0; b < CF::FN; ++b) {
        const int64_t gj = jr0 + wn0 + 8 * b + 2 * t;
        if (gj >= Nr) continue;
        if (p.work) {
          double* w = p.work + ((int64_t)blockIdx.z * p.Mq + gi) * Nr + gj;
          *reinterpret_cast<double2*>(w) = make_double2(acc[a][b][0], acc[a][b][1]);
        } else {
          double* c = p.C + gi * p.ldc * 4 + gj;
          double2 v = make_double2(p.alpha * acc[a][b][0], p.alpha * acc[a][b][1]);
          if (p.beta != 0.0) {
            double2 o = *reinterpret_cast<const double2*>(c);
            v.x += p.beta * o.x;
            v.y += p.beta * o.y;
          }
          *reinterpret_cast<double2*>(c) = v;
        }
      }
    }
  } else {
    __shared__ double red[2][CF::THREADS / 32];
    const int64_t Nr = 4 * p.Nq;
    double e = 0.0, xs = 0.0;
#pragma unroll
    for (int a = 0; a < CF::FM; ++a) {
      const int64_t gi = i0 + wm0 + 8 * a + arow;
#pragma unroll
      for (int b = 0; b < CF::FN; ++b) {
        const int64_t gj = jr0 + wn0 + 8 * b + 2 * t;
        if (gi < p.Mq && gj < Nr) {
          const double2 x = __ldg(reinterpret_cast<const double2*>(p.X + gi * p.ldx * 4 + gj));
          const double d0 = x.x - p.alpha * acc[a][b][0], d1 = x.y - p.alpha * acc[a][b][1];
          e += d0 * d0;
          e += d1 * d1;
          xs += x.x * x.x;
          xs += x.y * x.y;
        }
      }
    }
    e = warp_sum(e);
    xs = warp_sum(xs);
    if (lane == 0) {
      red[0][warp] = e;
      red[1][warp] = xs;
    }
    __syncthreads();
    if (tid == 0) {
      double se = 0.0, sx = 0.0;
      for (int w = 0; w < CF::THREADS / 32; ++w) {
        se += red[0][w];
        sx += red[1][w];
      }
      const int64_t tile = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
      p.partials[2 * tile] = se;
      p.partials[2 * tile + 1] = sx;
    }
  }
}

__global__ void splitk_reduce(const double* __restrict__ work, int splits, int64_t Mq, int64_t Nr,
                              double* __restrict__ C, int64_t ldc, double alpha, double beta) {
  const int64_t total = Mq * Nr;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / Nr, j = t - i * Nr;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += work[(int64_t)z * total + t];
    double* c = C + i * ldc * 4 + j;
    double v = alpha * s;
    if (beta != 0.0) v += beta * *c;
    *c = v;
  }
}

// Tile configuration used for every product (tuned for the FP64 DMMA pipe:
// 2 CTAs x 8 warps per SM, 32x32 warp tiles, 3-stage cp.async pipeline).
constexpr int G_BM = 64, G_BN = 128, G_WM = 32, G_WN = 32, G_BKQ = 8, G_ST = 3;

template <int OPA, int OPB, int EPI>
void launch_cfg(const KParams& kp, dim3 grid, cudaStream_t st) {
  using CF = Cfg<G_BM, G_BN, G_WM, G_WN, G_BKQ, G_ST, OPA, OPB, EPI>;
  auto kern = qgemm_kernel<G_BM, G_BN, G_WM, G_WN, G_BKQ, G_ST, OPA, OPB, EPI>;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CF::SMEM);
    set = true;
  }
  ++::qcur::g_launches;
  kern<<<grid, CF::THREADS, CF::SMEM, st>>>(kp);
}

int choose_splits(int64_t tiles, int64_t Kq) {
  const int64_t slots = 148 * 2;
  if (tiles >= 2 * slots) return 1;
  int64_t sp = (3 * slots + tiles - 1) / tiles;
  int64_t maxsp = Kq / (4 * G_BKQ);  // keep >= 32 quaternions of K per split
  if (sp > maxsp) sp = maxsp;
  if (sp < 1) sp = 1;
  if (sp > 64) sp = 64;
  return (int)sp;
}

}  // namespace

size_t qgemm_workspace_bytes(const GemmArgs& g) {
  const int64_t tiles = ((4 * g.Nq + G_BN - 1) / G_BN) * ((g.Mq + G_BM - 1) / G_BM);
  const int sp = choose_splits(tiles, g.Kq);
  return sp > 1 ? (size_t)sp * g.Mq * 4 * g.Nq * sizeof(double) : 0;
}

void launch_qgemm(const GemmArgs& g, double* workspace, cudaStream_t st) {
  if (g.Mq <= 0 || g.Nq <= 0) return;
  KParams kp{};
  kp.Mq = g.Mq;
  kp.Nq = g.Nq;
  kp.Kq = g.Kq;
  kp.A = g.A;
  kp.lda = g.lda;
  kp.B = g.B;
  kp.ldb = g.ldb;
  kp.C = g.C;
  kp.ldc = g.ldc;
  kp.alpha = g.alpha;
  kp.beta = g.beta;
  const int64_t gx = (4 * g.Nq + G_BN - 1) / G_BN, gy = (g.Mq + G_BM - 1) / G_BM;
  const int sp = g.Kq > 0 ? choose_splits(gx * gy, g.Kq) : 1;
  int64_t kchunk = (g.Kq + sp - 1) / sp;
  kchunk = ((kchunk + G_BKQ - 1) / G_BKQ) * G_BKQ;
  const int spz = kchunk > 0 ? (int)((g.Kq + kchunk - 1) / kchunk) : 1;
  kp.kchunk = kchunk > 0 ? kchunk : G_BKQ;
  kp.work = spz > 1 ? workspace : nullptr;
  dim3 grid((unsigned)gx, (unsigned)gy, (unsigned)spz);
  if (g.opA == 0 && g.opB == 0) launch_cfg<0, 0, EPI_STORE>(kp, grid, st);
  else if (g.opA == 0 && g.opB == 1) launch_cfg<0, 1, EPI_STORE>(kp, grid, st);
  else if (g.opA == 1 && g.opB == 0) launch_cfg<1, 0, EPI_STORE>(kp, grid, st);
  else launch_cfg<1, 1, EPI_STORE>(kp, grid, st);
  if (spz > 1) {
    const int64_t total = g.Mq * 4 * g.Nq;
    int blocks = (int)((total + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    ++::qcur::g_launches;
    splitk_reduce<<<blocks, 256, 0, st>>>(workspace, spz, g.Mq, 4 * g.Nq, g.C, g.ldc, g.alpha, g.beta);
  }
}

int64_t err_partials_count(int64_t m, int64_t n) { return ((4 * n + G_BN - 1) / G_BN) * ((m + G_BM - 1) / G_BM); }

void launch_cur_error(const double* X, int64_t ldx, const double* P, int64_t ldp, const double* R, int64_t ldr,
                      int64_t m, int64_t n, int64_t r, double* partials, double* out2, cudaStream_t st) {
  KParams kp{};
  kp.Mq = m;
  kp.Nq = n;
  kp.Kq = r;
  kp.A = P;
  kp.lda = ldp;
  kp.B = R;
  kp.ldb = ldr;
  kp.alpha = 1.0;
  kp.kchunk = ((r + G_BKQ - 1) / G_BKQ) * G_BKQ;
  kp.X = X;
  kp.ldx = ldx;
  kp.partials = partials;
  const int64_t gx = (4 * n + G_BN - 1) / G_BN, gy = (m + G_BM - 1) / G_BM;
  launch_cfg<0, 0, EPI_ERR>(kp, dim3((unsigned)gx, (unsigned)gy, 1), st);
  launch_reduce_pairs(partials, gx * gy, out2, st);
}

}  // namespace qcur
