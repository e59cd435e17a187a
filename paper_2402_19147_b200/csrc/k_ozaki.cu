// Y = X * B for quaternion matrices on the INT8 tensor cores (tcgen05.mma kind::i8),
// by exact modular arithmetic (Ozaki scheme II).
//
// This is the big contraction of the projection core, Y = X Q_R (cur.py:268 via
// qmat_matmul, quat.py:274-296): X is m x n, B is n x r, 32 m n r flop.  The FP64
// tensor path (mma.sync DMMA, k_qgemm.cu) tops out near 37 TFLOP/s on B200; the
// INT8 tcgen05 path runs at ~4.5 POP/s, so the product is computed exactly in
// integers instead:
//
//  1. Scale each row i of X (as reals, m x 4n) by 2^ex_i and each quaternion
//     column j of B by 2^fx_j and round to integers X', B' with |X'|, |B'| <= 2^bits.
//     This is the only rounding of the scheme: relative to the row (column) maximum it is
//     2^-(bits+1), below the FP64 accumulation error of a K = 4n dot product.
//  2. The real product Z = X' E(B') (E = the 4x4 Hamilton expansion, E[4k+s][4j+t] =
//     sign(s,t) b_kj[s^t]) is an integer with |Z| <= 4n 2^(2 bits) < M/2,
//     M = p_1 ... p_L for L pairwise coprime moduli p_l <= 256.  For every l the
//     residues X' mod p_l, E(B') mod p_l are signed bytes and Z mod p_l follows from
//     one int8 GEMM with exact int32 accumulation (|sum| <= 4n 2^14 < 2^31).
//  3. Z is recovered from its L residues by the Chinese remainder theorem in 128-bit
//     integer arithmetic and scaled back: Y = 2^-(ex_i + fx_j) Z (one rounding).
//
// Kernels: k_oz_xres (row max + residues of X, HBM-bound), k_oz_bmax/k_oz_bres (B,
// small), k_oz_gemm (tcgen05, TMA, TMEM; persistent, one CTA per SM), k_oz_crt.
// The GEMM kernel: warp 0 issues TMA loads of 128x128-byte A tiles and BNx128-byte B
// tiles (128-byte swizzle, K-major) into a 4-stage mbarrier ring; warp 1 (one thread)
// issues tcgen05.mma.cta_group::1.kind::i8 (M=128, N=BN, K=32) into a double-buffered
// TMEM accumulator (2 x 256 columns) and commits stage/accumulator barriers; warps 2-5
// drain the accumulator with tcgen05.ld, reduce it mod p_l and store residue bytes.
// Work units are (modulus, 128-row block, BN-column block) with the whole K range, so
// every result is a fixed integer: bitwise deterministic.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace qcur {

namespace {

using namespace tc;

constexpr int kOzMaxMod = 20;
constexpr int kOzMaxModDefault = 15;
// pairwise coprime, largest first
constexpr int kOzModuli[kOzMaxMod] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227,
                                      223, 217, 211, 199, 197, 193, 191, 181, 179, 173};
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52: x + kMagic rounds x to an integer

struct OzMods {
  int L;
  int p[kOzMaxMod];
  double pd[kOzMaxMod];
  double pinv[kOzMaxMod];
};

__device__ __forceinline__ int lo_int(double t) { return __double2loint(t); }

// v: integer-valued double, |v| < 2^51.  Returns r = v mod p as a byte in [-128, 127].
__device__ __forceinline__ unsigned residue_byte(double v, int l, const OzMods& md) {
  if (l == 0) return (unsigned)lo_int(v + kMagic) & 0xffu;  // p = 256: the low byte
  const double q = fma(v, md.pinv[l], kMagic) - kMagic;    // round(v / p), maybe off by one
  int r = lo_int(fma(-q, md.pd[l], v) + kMagic);           // exact, |r| <= p/2 + 1
  const int p = md.p[l];
  r = r > 127 ? r - p : r;
  r = r < -128 ? r + p : r;
  return (unsigned)r & 0xffu;
}

// x * 2^e, exact for every finite x whose result is representable (two steps keep 2^e finite)
__device__ __forceinline__ double scale2(double x, int e) {
  const int e1 = e / 2;
  return x * ldexp(1.0, e1) * ldexp(1.0, e - e1);
}

// ---------------------------------------------------------------------------
// residues of X: one CTA per row (K = 4n reals), |X'| <= 2^bits.
// X' = rint(x 2^e) is split into four signed 13-bit limbs (as exact floats), and for every
// odd modulus r = sum_i limb_i (2^(13 i) mod p) (exact in fp32, |.| < 2^22) is reduced with
// one rounded quotient; p = 256 takes the low byte of X'.  All moduli are compile-time
// constants (template L), so the modulus loop is straight-line FP32 code.
// ---------------------------------------------------------------------------
constexpr float kMagicF = 12582912.0f;  // 1.5 * 2^23

__host__ __device__ constexpr int cmod(long long v, int p) {
  long long r = v % p;
  if (r < 0) r += p;
  return (int)(r > p / 2 ? r - p : r);  // centered
}


// residue of the limb sum modulo P; the low byte of the result is r mod 256 (two's complement)
// Packed FP32 pairs (sm_100 FFMA2 / FADD2): two values per instruction.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pk(float lo, float hi) {
  return (f32x2)__float_as_uint(lo) | ((f32x2)__float_as_uint(hi) << 32);
}
__device__ __forceinline__ f32x2 ffma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 fadd2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 fmul2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// per odd modulus (index l >= 1): 2^13, 2^26, 2^39 mod p (centred), 1/p and -p, each duplicated
struct OzPairConsts {
  f32x2 c1[kOzMaxMod], c2[kOzMaxMod], c3[kOzMaxMod], pinv[kOzMaxMod], negp[kOzMaxMod];
};
constexpr unsigned f2u(float f) { return __builtin_bit_cast(unsigned, f); }
constexpr f32x2 dup(float f) { return (f32x2)f2u(f) | ((f32x2)f2u(f) << 32); }
constexpr OzPairConsts make_pair_consts() {
  OzPairConsts k{};
  for (int l = 0; l < kOzMaxMod; ++l) {
    const int p = kOzModuli[l];
    k.c1[l] = dup((float)cmod(1ll << 13, p));
    k.c2[l] = dup((float)cmod(1ll << 26, p));
    k.c3[l] = dup((float)cmod(1ll << 39, p));
    k.pinv[l] = dup(1.0f / (float)p);
    k.negp[l] = dup(-(float)p);
  }
  return k;
}
__constant__ OzPairConsts c_pair = make_pair_consts();

// residues of a pair of values (limbs f0..f3 as pairs) modulo kOzModuli[l]; the low byte of
// each 32-bit half is r mod 256 (two's complement)
template <int l>
__device__ __forceinline__ f32x2 pair_residue(f32x2 f0, f32x2 f1, f32x2 f2, f32x2 f3, f32x2 mag, f32x2 nmag) {
  const f32x2 t = ffma2(f3, c_pair.c3[l], ffma2(f2, c_pair.c2[l], ffma2(f1, c_pair.c1[l], f0)));
  const f32x2 q = fadd2(ffma2(t, c_pair.pinv[l], mag), nmag);  // round(t / p)
  f32x2 r = ffma2(q, c_pair.negp[l], t);                       // exact, |r| <= p/2 + 1
  constexpr int P = kOzModuli[l];
  if constexpr (P > 253) {  // p = 255: r = 128 -> r - p
    float lo = __uint_as_float((unsigned)r), hi = __uint_as_float((unsigned)(r >> 32));
    lo = lo > 127.0f ? lo - (float)P : lo;
    hi = hi > 127.0f ? hi - (float)P : hi;
    r = pk(lo, hi);
  }
  return fadd2(r, mag);
}
// low bytes of the four halves of two pairs -> one word
__device__ __forceinline__ unsigned pack_pairs(f32x2 a, f32x2 b) {
  return __byte_perm(__byte_perm((unsigned)a, (unsigned)(a >> 32), 0x0040),
                     __byte_perm((unsigned)b, (unsigned)(b >> 32), 0x0040), 0x5410);
}

__device__ __forceinline__ double amax4(const double4& v) {
  return fmax(fmax(fabs(v.x), fabs(v.y)), fmax(fabs(v.z), fabs(v.w)));
}

// VPT: values of X per thread and pass (16: uint4 residue stores; 8: uint2 stores, half the limb
// registers: no spills under the two-CTAs-per-SM register cap)
// Rows are taken grid-stride (row = blockIdx.x, += gridDim.x up to M): with QCUR_XRES_RESERVE=n the
// side-stream launch uses one 512-thread CTA per SM on all but n SMs, so the latency-bound main-stream
// kernels beside it (the draws, the cluster Cholesky) find whole SMs free (measured: no net gain).
template <int L, int NT, int VPT = 16, int MINB = 2>
__global__ void __launch_bounds__(NT, MINB) k_oz_xres(const double* __restrict__ X, int64_t K, int64_t ldx, int bits,
                                                      uint8_t* __restrict__ res, int64_t pitch, int64_t plane,
                                                      int* __restrict__ ex, int64_t M) {
  static_assert(VPT == 16 || VPT == 8, "values per thread");
  constexpr int NQ = VPT / 4;  // 32-byte loads per pass
  __shared__ double sh[NT / 32];
  for (int64_t row = blockIdx.x; row < M; row += gridDim.x) {
  const double* x = X + row * ldx;
  double mx = 0.0;
  int64_t k = threadIdx.x * 4;
  for (; k + 3 * NT * 4 < K; k += 4 * NT * 4) {  // four independent 32-byte loads in flight
    const double4 v0 = *reinterpret_cast<const double4*>(x + k);
    const double4 v1 = *reinterpret_cast<const double4*>(x + k + NT * 4);
    const double4 v2 = *reinterpret_cast<const double4*>(x + k + 2 * NT * 4);
    const double4 v3 = *reinterpret_cast<const double4*>(x + k + 3 * NT * 4);
    mx = fmax(mx, fmax(fmax(amax4(v0), amax4(v1)), fmax(amax4(v2), amax4(v3))));
  }
  for (; k < K; k += NT * 4) mx = fmax(mx, amax4(*reinterpret_cast<const double4*>(x + k)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) mx = fmax(mx, sh[w]);
  int e = 0;
  if (mx > 0.0) {
    int E;
    frexp(mx, &E);  // mx = f 2^E, f in [0.5, 1)
    e = bits - E;
  }
  if (threadIdx.x == 0) ex[row] = e;
  const double s1 = ldexp(1.0, e / 2), s2 = ldexp(1.0, e - e / 2);
  const long long magic_bits = __double_as_longlong(kMagic);
  const f32x2 mag = dup(kMagicF), nmag = dup(-kMagicF), lmag = dup(-8388608.0f);
  uint8_t* out = res + row * pitch;
  for (int64_t k0 = threadIdx.x * VPT; k0 < pitch; k0 += NT * VPT) {
    f32x2 f[VPT / 2][4];  // pair h holds values 2h, 2h+1; limbs 0..3
    unsigned low[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double4 t = make_double4(0.0, 0.0, 0.0, 0.0);
      if (k0 + 4 * q < K) t = *reinterpret_cast<const double4*>(x + k0 + 4 * q);
      const double vv[4] = {t.x, t.y, t.z, t.w};
      unsigned lb[4], lm[4][4];
      float sg[4];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const long long iv = __double_as_longlong(vv[h] * s1 * s2 + kMagic) - magic_bits;  // rint(x 2^e)
        lb[h] = (unsigned)iv;                                                              // mod 2^32
        const unsigned long long u = (unsigned long long)(iv < 0 ? -iv : iv);
        sg[h] = iv < 0 ? -1.0f : 1.0f;
        lm[h][0] = 0x4B000000u | ((unsigned)u & 0x1fffu);  // limb + 2^23 as a float
        lm[h][1] = 0x4B000000u | ((unsigned)(u >> 13) & 0x1fffu);
        lm[h][2] = 0x4B000000u | ((unsigned)(u >> 26) & 0x1fffu);
        lm[h][3] = 0x4B000000u | (unsigned)(u >> 39);
      }
      low[q] = __byte_perm(__byte_perm(lb[0], lb[1], 0x0040), __byte_perm(lb[2], lb[3], 0x0040), 0x5410);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const f32x2 sgn = pk(sg[2 * h], sg[2 * h + 1]);
#pragma unroll
        for (int i = 0; i < 4; ++i)
          f[2 * q + h][i] = fmul2(fadd2(((f32x2)lm[2 * h][i]) | ((f32x2)lm[2 * h + 1][i] << 32), lmag), sgn);
      }
    }
    if constexpr (VPT == 16) *reinterpret_cast<uint4*>(out + k0) = make_uint4(low[0], low[1], low[2], low[3]);  // p = 256
    else *reinterpret_cast<uint2*>(out + k0) = make_uint2(low[0], low[1]);
#define OZ_PLANE(l)                                                                                     \
    if constexpr (l < L) {                                                                              \
      unsigned w[NQ];                                                                                   \
      _Pragma("unroll") for (int q = 0; q < NQ; ++q) w[q] = pack_pairs(                                 \
          pair_residue<l>(f[2 * q][0], f[2 * q][1], f[2 * q][2], f[2 * q][3], mag, nmag),               \
          pair_residue<l>(f[2 * q + 1][0], f[2 * q + 1][1], f[2 * q + 1][2], f[2 * q + 1][3], mag, nmag)); \
      if constexpr (VPT == 16)                                                                          \
        *reinterpret_cast<uint4*>(out + (l) * plane + k0) = make_uint4(w[0], w[1], w[2], w[3]);         \
      else                                                                                              \
        *reinterpret_cast<uint2*>(out + (l) * plane + k0) = make_uint2(w[0], w[1]);                     \
    }
    OZ_PLANE(1) OZ_PLANE(2) OZ_PLANE(3) OZ_PLANE(4) OZ_PLANE(5) OZ_PLANE(6) OZ_PLANE(7) OZ_PLANE(8)
    OZ_PLANE(9) OZ_PLANE(10) OZ_PLANE(11) OZ_PLANE(12) OZ_PLANE(13) OZ_PLANE(14) OZ_PLANE(15)
    OZ_PLANE(16) OZ_PLANE(17) OZ_PLANE(18) OZ_PLANE(19)
#undef OZ_PLANE
  }
  __syncthreads();  // sh is rewritten by the next row's maximum
  }
}

// column maxima of B (Kq x Nq quaternions): 32 columns x a slab of rows per CTA (coalesced rows,
// 8 warps striding the slab), one atomicMax per column and CTA on the bits of the non-negative max
__global__ void k_oz_bmax(const double* __restrict__ B, int64_t Kq, int64_t Nq, int64_t ldb, int64_t rows_per,
                          unsigned long long* __restrict__ colmax) {
  __shared__ double sh[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const int64_t k0 = (int64_t)blockIdx.y * rows_per, k1 = k0 + rows_per < Kq ? k0 + rows_per : Kq;
  double mx = 0.0;
  if (j < Nq)
    for (int64_t k = k0 + w; k < k1; k += 8) {
      const Quat q = ldq_nc(B + (k * ldb + j) * 4);
      mx = fmax(mx, fmax(fmax(fabs(q.w), fabs(q.x)), fmax(fabs(q.y), fabs(q.z))));
    }
  sh[w][lane] = mx;
  __syncthreads();
  if (w == 0 && j < Nq) {
    for (int k = 1; k < 8; ++k) mx = fmax(mx, sh[k][lane]);
    atomicMax(colmax + j, (unsigned long long)__double_as_longlong(mx));
  }
}

__global__ void k_oz_bexp(const unsigned long long* __restrict__ colmax, int64_t Nq, int bits, int* __restrict__ fx) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= Nq) return;
  const double mx = __longlong_as_double((long long)colmax[j]);
  int e = 0;
  if (mx > 0.0) {
    int E;
    frexp(mx, &E);
    e = bits - E;
  }
  fx[j] = e;
}

// residues of E(B') stored K-major: row 4j+t, byte 4k+s = sign(s,t) b'_kj[s^t] mod p
__global__ void k_oz_bres(const double* __restrict__ B, int64_t Kq, int64_t Nq, int64_t ldb,
                          const __grid_constant__ OzMods md, const int* __restrict__ fx, uint8_t* __restrict__ res,
                          int64_t pitch, int64_t plane) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t kq_pad = pitch / 4;
  if (id >= Nq * kq_pad) return;
  const int64_t j = id / kq_pad, k = id - j * kq_pad;
  double b[4] = {0.0, 0.0, 0.0, 0.0};
  if (k < Kq) {
    const Quat q = ldq_nc(B + (k * ldb + j) * 4);
    const int e = fx[j];
    b[0] = (scale2(q.w, e) + kMagic) - kMagic;
    b[1] = (scale2(q.x, e) + kMagic) - kMagic;
    b[2] = (scale2(q.y, e) + kMagic) - kMagic;
    b[3] = (scale2(q.z, e) + kMagic) - kMagic;
  }
  // negative entries of E: (s,t) = (1,0) (2,0) (3,0) (3,1) (1,2) (2,3)
  for (int l = 0; l < md.L; ++l) {
    unsigned r[4], n[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      r[u] = residue_byte(b[u], l, md);
      n[u] = (0u - r[u]) & 0xffu;  // -r: for p = 256, -(-128) wraps to -128 (same residue)
    }
    uint8_t* o = res + l * plane + (4 * j) * pitch + 4 * k;
    // t = 0: s0 +b0, s1 -b1, s2 -b2, s3 -b3
    *reinterpret_cast<unsigned*>(o) = r[0] | (n[1] << 8) | (n[2] << 16) | (n[3] << 24);
    // t = 1: s0 +b1, s1 +b0, s2 +b3, s3 -b2
    *reinterpret_cast<unsigned*>(o + pitch) = r[1] | (r[0] << 8) | (r[3] << 16) | (n[2] << 24);
    // t = 2: s0 +b2, s1 -b3, s2 +b0, s3 +b1
    *reinterpret_cast<unsigned*>(o + 2 * pitch) = r[2] | (n[3] << 8) | (r[0] << 16) | (r[1] << 24);
    // t = 3: s0 +b3, s1 +b2, s2 -b1, s3 +b0
    *reinterpret_cast<unsigned*>(o + 3 * pitch) = r[3] | (r[2] << 8) | (n[1] << 16) | (r[0] << 24);
  }
}

// k_oz_bres with the moduli as compile-time constants and the FP32 limb reduction of k_oz_xres
// (pair_residue) instead of FP64 quotients per modulus and value: the FP64 pipe bounded k_oz_bres
// (cfg2 Q_R: 48 us for 74 MB).  Same layout and signs.  An odd modulus' byte may be the other centred
// representative of the same residue (r vs r - p); every consumer reduces the int32 sums modulo p,
// so the products are bit-identical (tests compare the factors).
// residues of one quaternion b (already loaded; zero for padding) of column j, row k of E(B') with
// column exponent e: the layout and signs of k_oz_bres, for the L compile-time moduli
template <int L>
__device__ __forceinline__ void bres_quat_fast(const double (&b)[4], int e, uint8_t* o0, int64_t pitch, int64_t plane) {
  const double s1 = ldexp(1.0, e / 2), s2 = ldexp(1.0, e - e / 2);  // scale2's two steps
  const long long magic_bits = __double_as_longlong(kMagic);
  const f32x2 mag = dup(kMagicF), nmag = dup(-kMagicF), lmag = dup(-8388608.0f);
  unsigned lb[4], lm[4][4];
  float sg[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const long long iv = __double_as_longlong(b[h] * s1 * s2 + kMagic) - magic_bits;  // rint(b 2^e)
    lb[h] = (unsigned)iv & 0xffu;
    const unsigned long long u = (unsigned long long)(iv < 0 ? -iv : iv);
    sg[h] = iv < 0 ? -1.0f : 1.0f;
    lm[h][0] = 0x4B000000u | ((unsigned)u & 0x1fffu);
    lm[h][1] = 0x4B000000u | ((unsigned)(u >> 13) & 0x1fffu);
    lm[h][2] = 0x4B000000u | ((unsigned)(u >> 26) & 0x1fffu);
    lm[h][3] = 0x4B000000u | (unsigned)(u >> 39);
  }
  f32x2 f[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const f32x2 sgn = pk(sg[2 * h], sg[2 * h + 1]);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      f[h][i] = fmul2(fadd2(((f32x2)lm[2 * h][i]) | ((f32x2)lm[2 * h + 1][i] << 32), lmag), sgn);
  }
  auto store = [&](uint8_t* o, const unsigned* r) {
    unsigned n[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) n[u] = (0u - r[u]) & 0xffu;
    *reinterpret_cast<unsigned*>(o) = r[0] | (n[1] << 8) | (n[2] << 16) | (n[3] << 24);
    *reinterpret_cast<unsigned*>(o + pitch) = r[1] | (r[0] << 8) | (r[3] << 16) | (n[2] << 24);
    *reinterpret_cast<unsigned*>(o + 2 * pitch) = r[2] | (n[3] << 8) | (r[0] << 16) | (r[1] << 24);
    *reinterpret_cast<unsigned*>(o + 3 * pitch) = r[3] | (r[2] << 8) | (n[1] << 16) | (r[0] << 24);
  };
  store(o0, lb);
#define OZ_BPLANE(l)                                                                        \
  if constexpr (l < L) {                                                                    \
    const f32x2 a = pair_residue<l>(f[0][0], f[0][1], f[0][2], f[0][3], mag, nmag);         \
    const f32x2 c = pair_residue<l>(f[1][0], f[1][1], f[1][2], f[1][3], mag, nmag);         \
    const unsigned r[4] = {(unsigned)a & 0xffu, (unsigned)(a >> 32) & 0xffu, (unsigned)c & 0xffu, \
                           (unsigned)(c >> 32) & 0xffu};                                    \
    store(o0 + (l) * plane, r);                                                             \
  }
  OZ_BPLANE(1) OZ_BPLANE(2) OZ_BPLANE(3) OZ_BPLANE(4) OZ_BPLANE(5) OZ_BPLANE(6) OZ_BPLANE(7) OZ_BPLANE(8)
  OZ_BPLANE(9) OZ_BPLANE(10) OZ_BPLANE(11) OZ_BPLANE(12) OZ_BPLANE(13) OZ_BPLANE(14) OZ_BPLANE(15)
  OZ_BPLANE(16) OZ_BPLANE(17) OZ_BPLANE(18) OZ_BPLANE(19)
#undef OZ_BPLANE
}

// k_oz_bres_fast with coalesced reads: a CTA takes 32 rows k x 8 columns j of B (each warp reads four
// 256-byte row segments instead of 32 quaternions a row apart), forms the residues of one plane at a
// time and stages its 4 x 8 output rows of 32 words in shared memory, so every warp store is 128
// contiguous bytes of one output row.  Same bytes as k_oz_bres_fast.  Measured slower at cfg2 (61.9 vs
// 39 us: 30 barriers per 256 quaternions), kept opt-in (QCUR_BRES_FAST=3).
template <int L>
__global__ void __launch_bounds__(256) k_oz_bres_tile(const double* __restrict__ B, int64_t Kq, int64_t Nq, int64_t ldb,
                                                      const int* __restrict__ fx, uint8_t* __restrict__ res,
                                                      int64_t pitch, int64_t plane) {
  __shared__ unsigned st[32][33];  // [4 jj + t][k]
  const int jj = threadIdx.x & 7, kk = threadIdx.x >> 3;
  const int64_t kq_pad = pitch / 4;
  const int64_t k = (int64_t)blockIdx.x * 32 + kk, j = (int64_t)blockIdx.y * 8 + jj;
  double b[4] = {0.0, 0.0, 0.0, 0.0};
  if (j < Nq && k < Kq) {
    const Quat q = ldq_nc(B + (k * ldb + j) * 4);
    b[0] = q.w;
    b[1] = q.x;
    b[2] = q.y;
    b[3] = q.z;
  }
  const int e = j < Nq ? fx[j] : 0;
  const double s1 = ldexp(1.0, e / 2), s2 = ldexp(1.0, e - e / 2);
  const long long magic_bits = __double_as_longlong(kMagic);
  const f32x2 mag = dup(kMagicF), nmag = dup(-kMagicF), lmag = dup(-8388608.0f);
  unsigned lb[4], lm[4][4];
  float sg[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const long long iv = __double_as_longlong(b[h] * s1 * s2 + kMagic) - magic_bits;
    lb[h] = (unsigned)iv & 0xffu;
    const unsigned long long u = (unsigned long long)(iv < 0 ? -iv : iv);
    sg[h] = iv < 0 ? -1.0f : 1.0f;
    lm[h][0] = 0x4B000000u | ((unsigned)u & 0x1fffu);
    lm[h][1] = 0x4B000000u | ((unsigned)(u >> 13) & 0x1fffu);
    lm[h][2] = 0x4B000000u | ((unsigned)(u >> 26) & 0x1fffu);
    lm[h][3] = 0x4B000000u | (unsigned)(u >> 39);
  }
  f32x2 f[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const f32x2 sgn = pk(sg[2 * h], sg[2 * h + 1]);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      f[h][i] = fmul2(fadd2(((f32x2)lm[2 * h][i]) | ((f32x2)lm[2 * h + 1][i] << 32), lmag), sgn);
  }
  // writer: word w of the tile (4 per thread): output row 4 (j0 + w / 128) + (w / 32) % 4, column k0 + w % 32
  const int64_t k0 = (int64_t)blockIdx.x * 32, j0 = (int64_t)blockIdx.y * 8;
  auto stage_and_write = [&](int l, const unsigned* r) {
    unsigned n[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) n[u] = (0u - r[u]) & 0xffu;
    st[4 * jj + 0][kk] = r[0] | (n[1] << 8) | (n[2] << 16) | (n[3] << 24);
    st[4 * jj + 1][kk] = r[1] | (r[0] << 8) | (r[3] << 16) | (n[2] << 24);
    st[4 * jj + 2][kk] = r[2] | (n[3] << 8) | (r[0] << 16) | (r[1] << 24);
    st[4 * jj + 3][kk] = r[3] | (r[2] << 8) | (n[1] << 16) | (r[0] << 24);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int w = threadIdx.x + 256 * i, row = w >> 5, kc = w & 31;
      const int64_t jo = j0 + (row >> 2), ko = k0 + kc;
      if (jo < Nq && ko < kq_pad)
        *reinterpret_cast<unsigned*>(res + l * plane + (4 * jo + (row & 3)) * pitch + 4 * ko) = st[row][kc];
    }
    __syncthreads();
  };
  stage_and_write(0, lb);
#define OZ_TPLANE(l)                                                                        \
  if constexpr (l < L) {                                                                    \
    const f32x2 a = pair_residue<l>(f[0][0], f[0][1], f[0][2], f[0][3], mag, nmag);         \
    const f32x2 c = pair_residue<l>(f[1][0], f[1][1], f[1][2], f[1][3], mag, nmag);         \
    const unsigned r[4] = {(unsigned)a & 0xffu, (unsigned)(a >> 32) & 0xffu, (unsigned)c & 0xffu, \
                           (unsigned)(c >> 32) & 0xffu};                                    \
    stage_and_write(l, r);                                                                  \
  }
  OZ_TPLANE(1) OZ_TPLANE(2) OZ_TPLANE(3) OZ_TPLANE(4) OZ_TPLANE(5) OZ_TPLANE(6) OZ_TPLANE(7) OZ_TPLANE(8)
  OZ_TPLANE(9) OZ_TPLANE(10) OZ_TPLANE(11) OZ_TPLANE(12) OZ_TPLANE(13) OZ_TPLANE(14) OZ_TPLANE(15)
  OZ_TPLANE(16) OZ_TPLANE(17) OZ_TPLANE(18) OZ_TPLANE(19)
#undef OZ_TPLANE
}

// QCUR_BRES_FAST=0: the FP64-quotient residue kernels; 3: k_oz_bres_tile (A/B: 61.9 vs 39 us at cfg2; default 1)
static int bres_fast_on() {
  static const int v = [] {
    const char* e = std::getenv("QCUR_BRES_FAST");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

template <int L>
__global__ void __launch_bounds__(256) k_oz_bres_fast(const double* __restrict__ B, int64_t Kq, int64_t Nq, int64_t ldb,
                                                      const int* __restrict__ fx, uint8_t* __restrict__ res,
                                                      int64_t pitch, int64_t plane) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t kq_pad = pitch / 4;
  if (id >= Nq * kq_pad) return;
  const int64_t j = id / kq_pad, k = id - j * kq_pad;
  double b[4] = {0.0, 0.0, 0.0, 0.0};
  if (k < Kq) {
    const Quat q = ldq_nc(B + (k * ldb + j) * 4);
    b[0] = q.w;
    b[1] = q.x;
    b[2] = q.y;
    b[3] = q.z;
  }
  bres_quat_fast<L>(b, fx[j], res + (4 * j) * pitch + 4 * k, pitch, plane);
}

// The small right operand of a factorization product (Q_1 = Z L_1^{-H}: B = L_1^{-H}, q x q) for up to
// two problems in one launch: one CTA per quaternion column j of B reduces the column maximum, stores
// the exponent and writes the residues of E(B') for that column (k_oz_bmax + k_oz_bexp + k_oz_bres
// without the atomics and the two extra launches).  conjT: B = A^H, read from A's row j (contiguous).
struct OzBColJob {
  const double* B;
  int64_t Kq, Nq, ldb, pitch, plane;
  int conjT, bits;
  int* fx;
  uint8_t* res;
};
struct OzBColJobs {
  OzBColJob j[2];
};

template <int NT, int L = 0>
__global__ void __launch_bounds__(NT) k_oz_bcol(const __grid_constant__ OzBColJobs J, const __grid_constant__ OzMods md) {
  const OzBColJob& jb = J.j[blockIdx.y];
  const int64_t j = blockIdx.x;
  if (j >= jb.Nq) return;
  auto ld = [&](int64_t k) -> Quat {
    if (jb.conjT) {
      const Quat a = ldq_nc(jb.B + (j * jb.ldb + k) * 4);
      return Quat{a.w, -a.x, -a.y, -a.z};
    }
    return ldq_nc(jb.B + (k * jb.ldb + j) * 4);
  };
  __shared__ double sh[NT / 32];
  double mx = 0.0;
  for (int64_t k = threadIdx.x; k < jb.Kq; k += NT) {
    const Quat q = ld(k);
    mx = fmax(mx, fmax(fmax(fabs(q.w), fabs(q.x)), fmax(fabs(q.y), fabs(q.z))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) mx = fmax(mx, sh[w]);
  int e = 0;
  if (mx > 0.0) {
    int E;
    frexp(mx, &E);
    e = jb.bits - E;
  }
  if (threadIdx.x == 0) jb.fx[j] = e;
  const int64_t kq_pad = jb.pitch / 4;
  for (int64_t k = threadIdx.x; k < kq_pad; k += NT) {
    double b[4] = {0.0, 0.0, 0.0, 0.0};
    if constexpr (L > 0) {  // the FP32 limb reduction of k_oz_bres_fast
      if (k < jb.Kq) {
        const Quat q = ld(k);
        b[0] = q.w;
        b[1] = q.x;
        b[2] = q.y;
        b[3] = q.z;
      }
      bres_quat_fast<L>(b, e, jb.res + (4 * j) * jb.pitch + 4 * k, jb.pitch, jb.plane);
      continue;
    }
    if (k < jb.Kq) {
      const Quat q = ld(k);
      b[0] = (scale2(q.w, e) + kMagic) - kMagic;
      b[1] = (scale2(q.x, e) + kMagic) - kMagic;
      b[2] = (scale2(q.y, e) + kMagic) - kMagic;
      b[3] = (scale2(q.z, e) + kMagic) - kMagic;
    }
    for (int l = 0; l < md.L; ++l) {  // the layout and signs of k_oz_bres
      unsigned r[4], n[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        r[u] = residue_byte(b[u], l, md);
        n[u] = (0u - r[u]) & 0xffu;
      }
      uint8_t* o = jb.res + l * jb.plane + (4 * j) * jb.pitch + 4 * k;
      *reinterpret_cast<unsigned*>(o) = r[0] | (n[1] << 8) | (n[2] << 16) | (n[3] << 24);
      *reinterpret_cast<unsigned*>(o + jb.pitch) = r[1] | (r[0] << 8) | (r[3] << 16) | (n[2] << 24);
      *reinterpret_cast<unsigned*>(o + 2 * jb.pitch) = r[2] | (n[3] << 8) | (r[0] << 16) | (r[1] << 24);
      *reinterpret_cast<unsigned*>(o + 3 * jb.pitch) = r[3] | (r[2] << 8) | (n[1] << 16) | (r[0] << 24);
    }
  }
}

// ---------------------------------------------------------------------------
// tcgen05 int8 GEMM:  res[l][i][j] = (A_l[i,:] . B_l[j,:]) mod p_l  (bytes in [0, p_l))
// ---------------------------------------------------------------------------
// a unit is 256 rows (two M = 128 accumulators sharing every B tile) x BN <= 256 columns
#ifndef QCUR_OZ_EPI_WARPS  // epilogue warps: 8 (one per TMEM lane quarter and accumulator) or 16 (columns split)
#define QCUR_OZ_EPI_WARPS 16
#endif
constexpr int OZ_EPI = QCUR_OZ_EPI_WARPS;
constexpr int OZ_BM = 256, OZ_BK = 128, OZ_STAGES = 3, OZ_THREADS = 64 + 32 * OZ_EPI;
constexpr int kOzCluster = 1;  // CTAs per cluster sharing the A tile by TMA multicast (QCUR_OZ_CLUSTER)
constexpr int OZ_A_BYTES = OZ_BM * OZ_BK, OZ_B_SLOT = 256 * OZ_BK;
constexpr int OZ_SMEM = 1024 + OZ_STAGES * (OZ_A_BYTES + OZ_B_SLOT) + 256;

struct OzProb {
  int64_t m, N;  // rows of the A operand; columns (reals) of the product
  int kblocks, mblocks, nblocks, BN, units;
  // lower: a symmetric product (A = B, the plane Grams of CholeskyQR2): only the tiles meeting the
  // lower triangle are computed (the CRT reads the mirror entry of the others).  tiles per modulus,
  // of which the first `fulls` have both 128-row halves (the last row block's may be all-padding
  // in its second half and costs half).
  int lower, tiles, fulls;
  uint32_t idesc;
  uint8_t* res;
  int64_t res_pitch, res_plane;
};

// up to two independent products in one launch (the SMs split by work units)
struct OzGemm {
  int L, total;
  int nfull;  // units of full cost (both problems), scheduled before the half-cost ones
  int exp;  // timing experiments only (QCUR_OZ_EXP=1: the epilogue releases TMEM without reading it)
  OzProb pr[2];
  int p[kOzMaxMod];
  int bm[kOzMaxMod];  // floor(2^32 / p) for the Barrett reduction of the epilogue
  double pinv[kOzMaxMod];
};

// unit u of the launch -> (problem, modulus l, row block mb, column block nb).  With clusters of CL
// CTAs a unit is a group of CL adjacent column blocks (this CTA's is nb = group * CL + rank).
// tiles of row block mb (lower products: those meeting the lower triangle)
__host__ __device__ __forceinline__ int oz_row_tiles(const OzProb& q, int mb) {
  if (!q.lower) return q.nblocks;
  const int t = (mb * OZ_BM + OZ_BM - 1) / q.BN + 1;
  return t < q.nblocks ? t : q.nblocks;
}

// CL = 1: units sorted by cost (every full-cost unit of both problems first, then the half-cost
// ones), within a class by modulus then tile (row block, column block) so that concurrently running
// CTAs share A tiles in L2; round-robin over the CTAs then leaves at most one half unit of imbalance.
template <int CL>
__device__ __forceinline__ int unit_coords(const OzGemm& P, int u, int& l, int& mb, int& nb, int crank) {
  if constexpr (CL == 1) {
    const int L = P.L;
    int k, tile;
    if (u < P.nfull) {
      const int f0 = L * P.pr[0].fulls;
      k = u < f0 ? 0 : 1;
      const int tl = u - (k ? f0 : 0), F = P.pr[k].fulls;
      l = tl / F;
      tile = tl - l * F;
    } else {
      const int v = u - P.nfull, h0 = L * (P.pr[0].tiles - P.pr[0].fulls);
      k = v < h0 ? 0 : 1;
      const int tl = v - (k ? h0 : 0), H = P.pr[k].tiles - P.pr[k].fulls;
      l = tl / H;
      tile = P.pr[k].fulls + (tl - l * H);
    }
    const OzProb& q = P.pr[k];
    if (!q.lower) {
      mb = tile / q.nblocks;
      nb = tile - mb * q.nblocks;
    } else {
      mb = 0;
      for (int c = oz_row_tiles(q, 0); tile >= c; c = oz_row_tiles(q, mb)) {
        tile -= c;
        ++mb;
      }
      nb = tile;
    }
    (void)crank;
    return k;
  }
  const int k = u < P.pr[0].units ? 0 : 1;
  const OzProb& q = P.pr[k];
  u -= k ? P.pr[0].units : 0;
  const int ngroups = (q.nblocks + CL - 1) / CL;
  nb = (u % ngroups) * CL + crank;
  const int t = u / ngroups;
  mb = t % q.mblocks;
  l = t / q.mblocks;
  return k;
}

// CL = 2: the two CTAs of a cluster take the same (modulus, row block) and two adjacent column
// blocks; each loads one 128-row half of the shared A tile and multicasts it to both, and loads
// its own B tile; a stage is released by a multicast commit to both CTAs' "empty" barriers.
template <int CL>
__global__ void __launch_bounds__(OZ_THREADS, 1)
    k_oz_gemm(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
              const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
              const __grid_constant__ OzGemm P) {
  extern __shared__ uint8_t smem_raw[];
  const unsigned pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sA = smem;
  uint8_t* sB = smem + OZ_STAGES * OZ_A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + OZ_STAGES * OZ_B_SLOT);
  uint64_t* empty = full + OZ_STAGES;
  uint64_t* tfull = empty + OZ_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  const int cid = CL > 1 ? (int)cluster_id_x() : (int)blockIdx.x;
  const int ncl = CL > 1 ? (int)ncluster_x() : (int)gridDim.x;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);  // one commit from each CTA of the cluster
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, OZ_EPI);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  if constexpr (CL > 1)
    cluster_sync_all();  // every CTA's barriers initialised before any multicast reaches them
  else
    __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA0)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB0)) : "memory");
      int stage = 0;
      unsigned phase = 0;
      for (int u = cid; u < P.total; u += ncl) {
        int l, mb, nb;
        const int k = unit_coords<CL>(P, u, l, mb, nb, crank);
        const OzProb& q = P.pr[k];
        const CUtensorMap* ta = k ? &tmA1 : &tmA0;
        const CUtensorMap* tb = k ? &tmB1 : &tmB0;
        const unsigned bytes = OZ_A_BYTES + q.BN * OZ_BK;
        for (int kb = 0; kb < q.kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_expect_tx(&full[stage], bytes);
          // A tile = two 128-row boxes (with CL = 2: this CTA's half, multicast to both CTAs)
          if constexpr (CL == 1) {
            tma_load_3d(sA + stage * OZ_A_BYTES, ta, kb * OZ_BK, mb * OZ_BM, l, &full[stage]);
            tma_load_3d(sA + stage * OZ_A_BYTES + OZ_A_BYTES / 2, ta, kb * OZ_BK, mb * OZ_BM + OZ_BM / 2, l,
                        &full[stage]);
          } else {
            tma_load_3d_mc(sA + stage * OZ_A_BYTES + crank * (OZ_A_BYTES / 2), ta, kb * OZ_BK,
                           mb * OZ_BM + crank * (OZ_BM / 2), l, &full[stage], kMask);
          }
          tma_load_3d(sB + stage * OZ_B_SLOT, tb, kb * OZ_BK, nb * q.BN, l, &full[stage]);
          if (++stage == OZ_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the issue loop (uniform registers, no per-MMA election loops); one
    // elected lane issues each k-block's MMAs and commits
    const uint64_t adesc0 = umma_desc(smem_u32(sA)), bdesc0 = umma_desc(smem_u32(sB));
    int stage = 0;
    unsigned phase = 0;
    int t = 0;
    for (int u = cid; u < P.total; u += ncl, ++t) {
      int l, mb, nb;
      const OzProb& q = P.pr[unit_coords<CL>(P, u, l, mb, nb, crank)];
      const bool second_half = (int64_t)mb * OZ_BM + OZ_BM / 2 < q.m;
      mbar_wait(tempty, ((unsigned)t & 1u) ^ 1u);  // the epilogue has drained the previous unit
      tc_fence_after();
      for (int kb = 0; kb < q.kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = adesc0 + (uint64_t)((stage * OZ_A_BYTES) >> 4);
        const uint64_t bd0 = bdesc0 + (uint64_t)((stage * OZ_B_SLOT) >> 4);
        if (elect_one_sync()) {
#pragma unroll
          for (int k = 0; k < OZ_BK / 32; ++k) {
            const uint64_t bd = bd0 + (uint64_t)(k * 2);  // +32 bytes along K
            mma_i8(tbase, ad + (uint64_t)(k * 2), bd, q.idesc, (kb | k) != 0);  // rows 0..127
            // rows 128..255 only when the block has any (the 800-row outputs of the Hermitian
            // products end 32 rows into their fourth block: its second half is all padding)
            if (second_half)
              mma_i8(tbase + 256, ad + (uint64_t)((128 * OZ_BK + k * 32) >> 4), bd, q.idesc, (kb | k) != 0);
          }
          if constexpr (CL == 1)
            mma_commit(&empty[stage]);
          else
            mma_commit_mc(&empty[stage], kMask);  // the stage is free in both CTAs' rings
        }
        __syncwarp();
        if (++stage == OZ_STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
      if (elect_one_sync()) mma_commit(tfull);
      __syncwarp();
    }
  } else {
    // epilogue warps: warp w drains TMEM lanes 32 (w % 4) .. +31 of accumulator ((w - 2) / 4) % 2,
    // with 16 warps the column chunks split in two parts ((w - 2) / 8)
    const int quarter = warp & 3, half = ((warp - 2) >> 2) & 1, cpart = OZ_EPI == 16 ? (warp - 2) >> 3 : 0;
    const int rloc = half * 128 + quarter * 32 + lane;
    int t = 0;
    for (int u = cid; u < P.total; u += ncl, ++t) {
      int l, mb, nb;
      const OzProb& q = P.pr[unit_coords<CL>(P, u, l, mb, nb, crank)];
      mbar_wait(tfull, (unsigned)t & 1u);
      tc_fence_after();
      if (P.exp) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
        continue;
      }
      const int64_t row = (int64_t)mb * OZ_BM + rloc;
      if ((int64_t)mb * OZ_BM + half * (OZ_BM / 2) >= q.m) {  // an all-padding half (no MMA was issued)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
        continue;
      }
      const int p = P.p[l];
      const int bm = P.bm[l];  // floor(2^32 / p)
      uint8_t* out = q.res + l * q.res_plane + row * q.res_pitch + (int64_t)nb * q.BN;
      const bool store = row < q.m && nb < q.nblocks;
      // residues of 32 accumulator columns: p = 256 the low byte; odd p by Barrett reduction with
      // the 32-bit high product (q = floor(z floor(2^32/p) / 2^32) is floor(z/p) or one off either
      // way for |z| < 2^31, so r = z - q p needs one correction each way; integer pipes only)
      auto emit = [&](const uint32_t(&v)[32], int c0) {
        uint32_t w[8];
#pragma unroll
        for (int z = 0; z < 8; ++z) w[z] = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          uint32_t r;
          if (l == 0) {
            r = v[i] & 255u;
          } else {
            const int z = (int)v[i];
            int rr = (int)(v[i] - (uint32_t)__mulhi(z, bm) * (uint32_t)p);
            rr += rr < 0 ? p : 0;
            rr -= rr >= p ? p : 0;
            r = (uint32_t)rr;
          }
          w[i >> 2] |= r << (8 * (i & 3));
        }
        if (store) {
          *reinterpret_cast<uint4*>(out + c0) = make_uint4(w[0], w[1], w[2], w[3]);
          if (c0 + 32 <= q.BN) *reinterpret_cast<uint4*>(out + c0 + 16) = make_uint4(w[4], w[5], w[6], w[7]);
        }
      };
      // TMEM loads one chunk ahead of the arithmetic (two register buffers)
      const uint32_t taddr = tbase + (uint32_t)(half * 256) + ((uint32_t)(quarter * 32) << 16);
      const int nall = (q.BN + 31) / 32, nfirst = OZ_EPI == 16 ? (nall + 1) / 2 : nall;
      const int ch0 = cpart ? nfirst : 0, nch = cpart ? nall : nfirst;
      if (ch0 < nch) {
        uint32_t va[32], vb[32];
        tmem_ld32_async(taddr + (uint32_t)(ch0 * 32), va);
        tmem_wait_ld();
        for (int ch = ch0; ch < nch; ch += 2) {
          if (ch + 1 < nch) tmem_ld32_async(taddr + (uint32_t)((ch + 1) * 32), vb);
          emit(va, ch * 32);
          tmem_wait_ld();
          if (ch + 1 < nch) {
            if (ch + 2 < nch) tmem_ld32_async(taddr + (uint32_t)((ch + 2) * 32), va);
            emit(vb, (ch + 1) * 32);
            tmem_wait_ld();
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
  // no CTA may leave while its peer can still multicast into its shared memory or barriers
  if constexpr (CL > 1) cluster_sync_all();
}

// ---------------------------------------------------------------------------
// Round 2: the modular GEMM on CTA pairs sharing B, with double-buffered accumulators.
// The two CTAs of a cluster take the two 128-row halves of one 256-row unit; each loads its own
// 128 A rows and one half of the B tile (BN / 2 rows), multicast to both, so the L2 -> SM bytes per
// MAC equal the single-CTA kernel's (its 256-row unit reads both A halves itself).  A CTA's
// accumulator is one M = 128 x BN block, so two of them fit TMEM (2 x 256 columns): the MMAs of
// unit t + 1 run while the epilogue drains unit t (the single-CTA kernel's two 128-row halves fill
// TMEM and its MMAs wait for every drain: ncu with the epilogue skipped, Gram 84 -> 58 us, X Q_R
// 560 -> 511 us).  A stage is 16 KB of A + up to 32 KB of B: four stages.  Measured: bit-identical
// results, no faster (Gram 82-85 us, X Q_R 588 us against 563): the drain was not what the skipped
// epilogue saved.  Off by default (QCUR_OZ_BMC=1).
// ---------------------------------------------------------------------------
constexpr int OZB_STAGES = 4, OZB_A = 128 * OZ_BK, OZB_B = 256 * OZ_BK;
constexpr int OZB_SMEM = 1024 + OZB_STAGES * (OZB_A + OZB_B) + 256;
static_assert(OZB_SMEM <= OZ_SMEM + 4096, "B-multicast stages");

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(OZ_THREADS, 1)
    k_oz_gemm_bmc(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
                  const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
                  const __grid_constant__ OzGemm P) {
  extern __shared__ uint8_t smem_raw[];
  const unsigned pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint8_t* sA = smem;
  uint8_t* sB = smem + OZB_STAGES * OZB_A;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + OZB_STAGES * OZB_B);
  uint64_t* empty = full + OZB_STAGES;
  uint64_t* tfull = empty + OZB_STAGES;  // [2]
  uint64_t* tempty = tfull + 2;          // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = (int)cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)ncluster_x();
  constexpr uint16_t kMask = 3;
  if (threadIdx.x == 0) {
    for (int s = 0; s < OZB_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 2);  // one commit from each CTA: both have consumed their copy of B
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], OZ_EPI);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();  // every CTA's barriers initialised before any multicast reaches them
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA0)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB0)) : "memory");
      int stage = 0;
      unsigned phase = 0;
      for (int u = cid; u < P.total; u += ncl) {
        int l, mb, nb;
        const int k = unit_coords<1>(P, u, l, mb, nb, 0);
        const OzProb& q = P.pr[k];
        const CUtensorMap* ta = k ? &tmA1 : &tmA0;
        const CUtensorMap* tb = k ? &tmB1 : &tmB0;  // boxes of BN / 2 rows
        const int hb = q.BN / 2;
        const unsigned bytes = OZB_A + q.BN * OZ_BK;  // own A + both halves of B
        for (int kb = 0; kb < q.kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_expect_tx(&full[stage], bytes);
          tma_load_3d(sA + stage * OZB_A, ta, kb * OZ_BK, mb * OZ_BM + crank * (OZ_BM / 2), l, &full[stage]);
          tma_load_3d_mc(sB + stage * OZB_B + crank * hb * OZ_BK, tb, kb * OZ_BK, nb * q.BN + crank * hb, l,
                         &full[stage], kMask);
          if (++stage == OZB_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    const uint64_t adesc0 = umma_desc(smem_u32(sA)), bdesc0 = umma_desc(smem_u32(sB));
    int stage = 0;
    unsigned phase = 0;
    int t = 0;
    for (int u = cid; u < P.total; u += ncl, ++t) {
      int l, mb, nb;
      const OzProb& q = P.pr[unit_coords<1>(P, u, l, mb, nb, 0)];
      const bool mine = (int64_t)mb * OZ_BM + crank * (OZ_BM / 2) < q.m;  // any valid row in this CTA's half
      const int buf = t & 1;
      mbar_wait(&tempty[buf], (((unsigned)t >> 1) & 1u) ^ 1u);  // the epilogue has drained unit t - 2
      tc_fence_after();
      const uint32_t d = tbase + (uint32_t)(buf * 256);
      for (int kb = 0; kb < q.kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = adesc0 + (uint64_t)((stage * OZB_A) >> 4);
        const uint64_t bd0 = bdesc0 + (uint64_t)((stage * OZB_B) >> 4);
        if (elect_one_sync()) {
          if (mine) {
#pragma unroll
            for (int kk = 0; kk < OZ_BK / 32; ++kk)
              mma_i8(d, ad + (uint64_t)(kk * 2), bd0 + (uint64_t)(kk * 2), q.idesc, (kb | kk) != 0);
          }
          mma_commit_mc(&empty[stage], kMask);  // this CTA's copy of the stage is consumed
        }
        __syncwarp();
        if (++stage == OZB_STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
      if (elect_one_sync()) mma_commit(&tfull[buf]);
      __syncwarp();
    }
  } else {
    // epilogue: warp w drains TMEM lanes 32 (w % 4) .. +31 and column part (w - 2) / 4 of OZ_EPI / 4
    constexpr int kParts = OZ_EPI / 4;
    const int quarter = warp & 3, cpart = (warp - 2) >> 2;
    const int rloc = crank * (OZ_BM / 2) + quarter * 32 + lane;
    int t = 0;
    for (int u = cid; u < P.total; u += ncl, ++t) {
      int l, mb, nb;
      const OzProb& q = P.pr[unit_coords<1>(P, u, l, mb, nb, 0)];
      const int buf = t & 1;
      mbar_wait(&tfull[buf], ((unsigned)t >> 1) & 1u);
      tc_fence_after();
      const bool mine = (int64_t)mb * OZ_BM + crank * (OZ_BM / 2) < q.m;
      if (P.exp || !mine) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[buf]);
        continue;
      }
      const int64_t row = (int64_t)mb * OZ_BM + rloc;
      const int p = P.p[l];
      const int bm = P.bm[l];
      uint8_t* out = q.res + l * q.res_plane + row * q.res_pitch + (int64_t)nb * q.BN;
      const bool store = row < q.m && nb < q.nblocks;
      auto emit = [&](const uint32_t(&v)[32], int c0) {  // as k_oz_gemm's epilogue
        uint32_t w[8];
#pragma unroll
        for (int z = 0; z < 8; ++z) w[z] = 0;
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          uint32_t r;
          if (l == 0) {
            r = v[i] & 255u;
          } else {
            const int z = (int)v[i];
            int rr = (int)(v[i] - (uint32_t)__mulhi(z, bm) * (uint32_t)p);
            rr += rr < 0 ? p : 0;
            rr -= rr >= p ? p : 0;
            r = (uint32_t)rr;
          }
          w[i >> 2] |= r << (8 * (i & 3));
        }
        if (store) {
          *reinterpret_cast<uint4*>(out + c0) = make_uint4(w[0], w[1], w[2], w[3]);
          if (c0 + 32 <= q.BN) *reinterpret_cast<uint4*>(out + c0 + 16) = make_uint4(w[4], w[5], w[6], w[7]);
        }
      };
      const uint32_t taddr = tbase + (uint32_t)(buf * 256) + ((uint32_t)(quarter * 32) << 16);
      const int nall = (q.BN + 31) / 32;
      const int ch0 = cpart * nall / kParts, nch = (cpart + 1) * nall / kParts;
      if (ch0 < nch) {
        uint32_t va[32], vb[32];
        tmem_ld32_async(taddr + (uint32_t)(ch0 * 32), va);
        tmem_wait_ld();
        for (int ch = ch0; ch < nch; ch += 2) {
          if (ch + 1 < nch) tmem_ld32_async(taddr + (uint32_t)((ch + 1) * 32), vb);
          emit(va, ch * 32);
          tmem_wait_ld();
          if (ch + 1 < nch) {
            if (ch + 2 < nch) tmem_ld32_async(taddr + (uint32_t)((ch + 2) * 32), va);
            emit(vb, (ch + 1) * 32);
            tmem_wait_ld();
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[buf]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
  cluster_sync_all();  // no CTA leaves while its peer can still multicast into it
}

// ---------------------------------------------------------------------------
// CRT: Z from its residues, Y = 2^-(ex_i + fx_j) Z.  S = sum_l ((r_l w_l) mod p_l) (M / p_l)
// in 128-bit integers (S < L M), Z = S mod M centred; four outputs per thread.
// ---------------------------------------------------------------------------
struct OzCrt {
  int L;
  float w[kOzMaxMod];  // (M / p_l)^-1 mod p_l
  float P[kOzMaxMod], pinv[kOzMaxMod];
  unsigned mi[kOzMaxMod][4];  // M / p_l as four 32-bit limbs, least significant first
  unsigned long long M_lo, M_hi;
  double Md;
  double Mr;  // 1 / Md: the quotient estimate by one multiply (corrected both ways below)
};

// Exact small-integer <-> float conversions on the FMA / integer pipes instead of the conversion
// unit (I2F / F2I run at a quarter of the FMA rate or less; the CRT kernels issued 120 of them per
// thread, ncu: 40 % of k_oz_crt's time).
__device__ __forceinline__ float byte_to_float(unsigned word, int h) {  // byte h of word, exact
  return __uint_as_float(__byte_perm(word, 0x4B000000u, 0x7650u | (unsigned)h)) - 8388608.0f;
}
__device__ __forceinline__ unsigned small_float_to_uint(float t) {  // t integer-valued in [0, 2^23)
  return __float_as_uint(t + 8388608.0f) - 0x4B000000u;
}
__device__ __forceinline__ float small_int_to_float(int v) {  // |v| < 2^22, exact
  return __int_as_float(0x4B400000 + v) - 12582912.0f;
}

// S = sum_l t_l (M / p_l) with t_l = (r_l w_l) mod p_l < 256: the limb products t * mi[k] < 2^40
// accumulate in four 64-bit columns without overflow (L <= 16), carries are resolved once.
template <int L>
__global__ void __launch_bounds__(256) k_oz_crt(const uint8_t* __restrict__ res, int64_t m, int64_t N, int64_t pitch,
                                                int64_t plane, const int* __restrict__ ex,
                                                const int* __restrict__ fx, const __grid_constant__ OzCrt c,
                                                double* __restrict__ Y, int64_t ldy) {
  const int64_t nq = N >> 2;  // N = 4 r: one quaternion (4 outputs) per thread
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= m * nq) return;
  const int64_t i = id / nq, jq = id - i * nq;
  const uint8_t* rp = res + i * pitch + 4 * jq;
  unsigned long long col[4][4] = {};
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const unsigned r4 = __ldg(reinterpret_cast<const unsigned*>(rp + l * plane));
    const float P = c.P[l], pinv = c.pinv[l];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const float rw = byte_to_float(r4, h) * c.w[l];  // < 2^16, exact
      float t = fmaf(-(fmaf(rw, pinv, kMagicF) - kMagicF), P, rw);
      t = t < 0.0f ? t + P : t;
      const unsigned tt = small_float_to_uint(t);
#pragma unroll
      for (int k = 0; k < 4; ++k) col[h][k] += (unsigned long long)tt * c.mi[l][k];
    }
  }
  const unsigned __int128 M = ((unsigned __int128)c.M_hi << 64) | c.M_lo;
  const int e = -(ex[i] + fx[jq]);
  const double s1 = ldexp(1.0, e / 2), s2 = ldexp(1.0, e - e / 2);
  double out[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    // resolve the column carries: S = col0 + col1 2^32 + col2 2^64 + col3 2^96
    const unsigned long long w0 = col[h][0];
    const unsigned long long c1 = col[h][1] + (w0 >> 32);
    const unsigned long long c2 = col[h][2] + (c1 >> 32);
    const unsigned long long c3 = col[h][3] + (c2 >> 32);
    const unsigned long long lo = (w0 & 0xffffffffull) | (c1 << 32);
    const unsigned long long hi = (c2 & 0xffffffffull) | (c3 << 32);
    unsigned __int128 S = ((unsigned __int128)hi << 64) | lo;
    const double sd = (double)hi * 18446744073709551616.0 + (double)lo;
    long long q = (long long)floor(sd * c.Mr);
    q = q < 0 ? 0 : q;
    S -= M * (unsigned long long)q;
    if ((__int128)S < 0) S += M;  // the estimate was one too large
    if (S >= M) S -= M;
    __int128 Z = (__int128)S;
    if (S > (M >> 1)) Z -= (__int128)M;
    const double z = (double)(long long)(Z >> 64) * 18446744073709551616.0 + (double)(unsigned long long)Z;
    out[h] = z * s1 * s2;
  }
  double* y = Y + i * ldy + 4 * jq;
  *reinterpret_cast<double4*>(y) = make_double4(out[0], out[1], out[2], out[3]);
}

// ---------------------------------------------------------------------------
// Hermitian products C = A^H B (A: p x qa, B: p x qb quaternions) by real plane products:
// C_t[i][j] = sum_{a,b} sign_t(a,b) (A_a^T B_b)[i][j], the 16 plane products forming one real
// GEMM of W_A (4qa x p) by W_B (4qb x p), both K-major stacks of the scaled planes.  No 4x
// Hamilton expansion of either operand; the signed combination is exact (128-bit integers).
// ---------------------------------------------------------------------------
// the plane residues of rows k0..k0+3 of column i of Z (scaled by 2^e)
template <int L>
__device__ __forceinline__ void oz_wres_body(const double* __restrict__ Z, int64_t p, int64_t q, int64_t ldz, int e,
                                             uint8_t* __restrict__ res, int64_t pitch, int64_t plane, int64_t i,
                                             int64_t k0) {
  const double s1 = ldexp(1.0, e / 2), s2 = ldexp(1.0, e - e / 2);
  const long long magic_bits = __double_as_longlong(kMagic);
  const f32x2 mag = dup(kMagicF), nmag = dup(-kMagicF), lmag = dup(-8388608.0f);
  // per plane a: limbs of the four values k0..k0+3 as two FP32 pairs, and their low bytes (p = 256)
  f32x2 f[4][2][4];
  unsigned low[4];
  double v[4][4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    Quat z = qzero();
    if (k0 + h < p) z = ldq_nc(Z + ((k0 + h) * ldz + i) * 4);
    v[0][h] = z.w;
    v[1][h] = z.x;
    v[2][h] = z.y;
    v[3][h] = z.z;
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    unsigned lb[4], lm[4][4];
    float sg[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const long long iv = __double_as_longlong(v[a][h] * s1 * s2 + kMagic) - magic_bits;  // rint(x 2^e)
      lb[h] = (unsigned)iv;
      const unsigned long long u = (unsigned long long)(iv < 0 ? -iv : iv);
      sg[h] = iv < 0 ? -1.0f : 1.0f;
      lm[h][0] = 0x4B000000u | ((unsigned)u & 0x1fffu);
      lm[h][1] = 0x4B000000u | ((unsigned)(u >> 13) & 0x1fffu);
      lm[h][2] = 0x4B000000u | ((unsigned)(u >> 26) & 0x1fffu);
      lm[h][3] = 0x4B000000u | (unsigned)(u >> 39);
    }
    low[a] = __byte_perm(__byte_perm(lb[0], lb[1], 0x0040), __byte_perm(lb[2], lb[3], 0x0040), 0x5410);
#pragma unroll
    for (int hp = 0; hp < 2; ++hp) {
      const f32x2 sgn = pk(sg[2 * hp], sg[2 * hp + 1]);
#pragma unroll
      for (int t = 0; t < 4; ++t)
        f[a][hp][t] = fmul2(fadd2(((f32x2)lm[2 * hp][t]) | ((f32x2)lm[2 * hp + 1][t] << 32), lmag), sgn);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) *reinterpret_cast<unsigned*>(res + (a * q + i) * pitch + k0) = low[a];  // p = 256
#define OZ_WPLANE(l)                                                                                      \
  if constexpr (l < L) {                                                                                  \
    _Pragma("unroll") for (int a = 0; a < 4; ++a) {                                                       \
      const unsigned w = pack_pairs(pair_residue<l>(f[a][0][0], f[a][0][1], f[a][0][2], f[a][0][3], mag, nmag), \
                                    pair_residue<l>(f[a][1][0], f[a][1][1], f[a][1][2], f[a][1][3], mag, nmag)); \
      *reinterpret_cast<unsigned*>(res + (l) * plane + (a * q + i) * pitch + k0) = w;                     \
    }                                                                                                     \
  }
  OZ_WPLANE(1) OZ_WPLANE(2) OZ_WPLANE(3) OZ_WPLANE(4) OZ_WPLANE(5) OZ_WPLANE(6) OZ_WPLANE(7) OZ_WPLANE(8)
  OZ_WPLANE(9) OZ_WPLANE(10) OZ_WPLANE(11) OZ_WPLANE(12) OZ_WPLANE(13) OZ_WPLANE(14) OZ_WPLANE(15)
#undef OZ_WPLANE
}

// Up to four operands' plane residues in two launches (the Hermitian products of one factorization
// step: C and R^H, or A and B): column maxima (k_oz_pmax, one atomicMax per column and slab), then
// exponents and residues (k_oz_pres: the thread of row block 0 also stores the column's exponent).
struct OzPlaneJob {
  const double* Z;
  int64_t p, q, ldz, rows_per, pitch, plane;
  int slabs, bits;
  unsigned long long* cmax;
  int* ex;
  uint8_t* w;
};
struct OzPlaneJobs {
  OzPlaneJob j[4];
};

__global__ void k_oz_pmax(const __grid_constant__ OzPlaneJobs J) {
  const OzPlaneJob& jb = J.j[blockIdx.z];
  if ((int64_t)blockIdx.x * 32 >= jb.q || (int)blockIdx.y >= jb.slabs) return;
  __shared__ double sh[8][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t j = (int64_t)blockIdx.x * 32 + lane;
  const int64_t k0 = (int64_t)blockIdx.y * jb.rows_per, k1 = k0 + jb.rows_per < jb.p ? k0 + jb.rows_per : jb.p;
  double mx = 0.0;
  if (j < jb.q)
    for (int64_t k = k0 + w; k < k1; k += 8) {
      const Quat z = ldq_nc(jb.Z + (k * jb.ldz + j) * 4);
      mx = fmax(mx, fmax(fmax(fabs(z.w), fabs(z.x)), fmax(fabs(z.y), fabs(z.z))));
    }
  sh[w][lane] = mx;
  __syncthreads();
  if (w == 0 && j < jb.q) {
    for (int k = 1; k < 8; ++k) mx = fmax(mx, sh[k][lane]);
    atomicMax(jb.cmax + j, (unsigned long long)__double_as_longlong(mx));
  }
}

template <int L>
__global__ void __launch_bounds__(256) k_oz_pres(const __grid_constant__ OzPlaneJobs J) {
  const OzPlaneJob& jb = J.j[blockIdx.y];
  const int64_t k4n = jb.pitch / 4;
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= jb.q * k4n) return;
  const int64_t i = id / k4n, k0 = 4 * (id - i * k4n);
  const double mx = __longlong_as_double((long long)jb.cmax[i]);
  int e = 0;
  if (mx > 0.0) {
    int E;
    frexp(mx, &E);
    e = jb.bits - E;
  }
  if (k0 == 0) jb.ex[i] = e;
  oz_wres_body<L>(jb.Z, jb.p, jb.q, jb.ldz, e, jb.w, jb.pitch, jb.plane, i, k0);
}

// one product value from its L residue bytes (stride `plane`), centred in (-M/2, M/2]
template <int L>
__device__ __forceinline__ __int128 crt_one(const uint8_t* rp, int64_t plane, const OzCrt& c) {
  unsigned long long col[4] = {0, 0, 0, 0};
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const float rw = small_int_to_float((int)rp[l * plane]) * c.w[l];
    float t = fmaf(-(fmaf(rw, c.pinv[l], kMagicF) - kMagicF), c.P[l], rw);
    t = t < 0.0f ? t + c.P[l] : t;
    const unsigned tt = small_float_to_uint(t);
#pragma unroll
    for (int k = 0; k < 4; ++k) col[k] += (unsigned long long)tt * c.mi[l][k];
  }
  const unsigned long long c1 = col[1] + (col[0] >> 32);
  const unsigned long long c2 = col[2] + (c1 >> 32);
  const unsigned long long c3 = col[3] + (c2 >> 32);
  const unsigned long long lo = (col[0] & 0xffffffffull) | (c1 << 32);
  const unsigned long long hi = (c2 & 0xffffffffull) | (c3 << 32);
  unsigned __int128 S = ((unsigned __int128)hi << 64) | lo;
  const unsigned __int128 M = ((unsigned __int128)c.M_hi << 64) | c.M_lo;
  long long q = (long long)floor(((double)hi * 18446744073709551616.0 + (double)lo) * c.Mr);
  q = q < 0 ? 0 : q;
  S -= M * (unsigned long long)q;
  if ((__int128)S < 0) S += M;
  if (S >= M) S -= M;
  __int128 Z = (__int128)S;
  if (S > (M >> 1)) Z -= (__int128)M;
  return Z;
}

// C[i][j] from the 16 plane products: conj(x) y = (x0y0 + x1y1 + x2y2 + x3y3) + (x0y1 - x1y0 - x2y3 + x3y2) i
//   + (x0y2 + x1y3 - x2y0 - x3y1) j + (x0y3 - x1y2 + x2y1 - x3y0) k.
// One CTA per 16 x 16 block of (i, j) and component t, a thread per output.  One thread TMA-loads,
// for each of t's four plane products, the residue block of every modulus (a 3-D box, 32 columns from
// the 16-byte aligned start: a TMA box must begin on a 16-byte boundary, tools/tma3d_probe.cu), and
// for lower products (lower_bn = BN of the GEMM: the plane Grams of CholeskyQR2 computed only the
// tiles meeting the lower triangle) also the mirror block; each thread then takes its element from
// the direct block, or from the mirror when its tile was not computed, forms the signed residue sum
// and accumulates one CRT (CRT is linear, and the exact integer sum obeys |sum| <= 4 p 2^(2 bits)
// < M / 2).
constexpr int kHB = 16;  // output block edge

__device__ __forceinline__ bool oz_tile_computed(int row, int col, int lower_bn) {  // 32-bit: cheap divisions
  return !lower_bn || (unsigned)col / (unsigned)lower_bn * (unsigned)lower_bn <= ((unsigned)row & ~(unsigned)(OZ_BM - 1)) + OZ_BM - 1;
}

// a TMA box starts on a 16-byte column boundary: boxes are 32 columns wide from the aligned start
constexpr int kHBW = 32;
constexpr int kOzHcrtSmem = 8 * kOzMaxModDefault * kHB * kHBW + 64;  // [u | mirror u + 4][modulus][row][32]

// Both problems of a factorization step in one launch (blockIdx.z); a problem whose consumers read
// only the lower triangle of its Hermitian output (the CholeskyQR2 Grams: the Cholesky, the series
// and the kappa guard read k <= i) enumerates only the 16 x 16 blocks on or below the diagonal.
struct OzHcrtProb {
  CUtensorMap tm;
  int64_t qa, qb, ldc;
  const int* exa;
  const int* exb;
  double* C;
  int lower_bn, tri, nbx, nblk;
};
struct OzHcrtJobs {
  OzHcrtProb p[2];
};

template <int L>
__global__ void __launch_bounds__(kHB * kHB) k_oz_hcrt(const __grid_constant__ OzHcrtJobs H,
                                                       const __grid_constant__ OzCrt c) {
  const OzHcrtProb& hp = H.p[blockIdx.z];
  if ((int)blockIdx.x >= hp.nblk) return;
  int bi, bj;
  if (hp.tri) {  // linear index -> (bi, bj), bj <= bi
    const int b = (int)blockIdx.x;
    bi = (int)((sqrtf(8.0f * (float)b + 1.0f) - 1.0f) * 0.5f);
    while ((bi + 1) * (bi + 2) / 2 <= b) ++bi;
    while (bi * (bi + 1) / 2 > b) --bi;
    bj = b - bi * (bi + 1) / 2;
  } else {
    bi = (int)blockIdx.x / hp.nbx;
    bj = (int)blockIdx.x - bi * hp.nbx;
  }
  const CUtensorMap& tm = hp.tm;
  const int64_t qa = hp.qa, qb = hp.qb, ldc = hp.ldc;
  const int* __restrict__ exa = hp.exa;
  const int* __restrict__ exb = hp.exb;
  double* __restrict__ C = hp.C;
  const int lower_bn = hp.lower_bn;
  extern __shared__ __align__(128) uint8_t hsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(hsm + 8 * L * kHB * kHBW);
  auto blk = [&](int box, int l, int row, int col) -> uint8_t {
    return hsm[((box * L + l) * kHB + row) * kHBW + col];
  };
  const int tx = threadIdx.x % kHB, ty = threadIdx.x / kHB;
  const int t = (int)blockIdx.y;
  const int i0 = bi * kHB, j0 = bj * kHB;
  // plane product u of component t is A_u^T B_(u^t) with sign -1 where bit u of nibble t of 0xAC60 is set:
  // t = 0: + + + +,  t = 1: + - - +,  t = 2: + + - -,  t = 3: + - + -  (no runtime-indexed local table)
  const unsigned neg = (0xAC60u >> (4 * t)) & 0xFu;
  const int iqa = (int)qa, iqb = (int)qb;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int nb = lower_bn ? 8 : 4;
    mbar_expect_tx(bar, (unsigned)(nb * L * kHB * kHBW));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int a = u, b = u ^ t;
      const int xd = b * iqb + j0, xm = a * iqa + i0;  // first column of the direct / mirror block
      tma_load_3d(hsm + u * L * kHB * kHBW, &tm, xd & ~15, a * iqa + i0, 0, bar);  // x = column, y = row
      if (lower_bn) tma_load_3d(hsm + (4 + u) * L * kHB * kHBW, &tm, xm & ~15, b * iqb + j0, 0, bar);
    }
  }
  const int i = i0 + ty, j = j0 + tx;
  int sg[4], cd[4], cm[4];
  bool dir[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int a = u, b = u ^ t;
    sg[u] = (neg >> u) & 1u ? -1 : 1;
    dir[u] = oz_tile_computed(a * iqa + i, b * iqb + j, lower_bn);
    cd[u] = ((b * iqb + j0) & 15) + tx;  // column of the element in the direct block (row ty)
    cm[u] = ((a * iqa + i0) & 15) + ty;  // column of the element in the mirror block (row tx)
  }
  mbar_wait(bar, 0);
  unsigned long long col[4] = {};
#pragma unroll
  for (int l = 0; l < L; ++l) {
    int sum = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) sum += sg[u] * (int)(dir[u] ? blk(u, l, ty, cd[u]) : blk(4 + u, l, tx, cm[u]));
    const float P = c.P[l], pinv = c.pinv[l];
    // (sum mod p) w mod p, exact in FP32: |sum| < 1024, (sum mod p) w < 2^16
    const float sf = small_int_to_float(sum);
    float sm = fmaf(-(fmaf(sf, pinv, kMagicF) - kMagicF), P, sf);
    sm = sm < 0.0f ? sm + P : sm;
    sm = sm >= P ? sm - P : sm;
    const float rw = sm * c.w[l];
    float tq = fmaf(-(fmaf(rw, pinv, kMagicF) - kMagicF), P, rw);
    tq = tq < 0.0f ? tq + P : tq;
    const unsigned tt = small_float_to_uint(tq);
#pragma unroll
    for (int k = 0; k < 4; ++k) col[k] += (unsigned long long)tt * c.mi[l][k];
  }
  if (i >= iqa || j >= iqb) return;
  const unsigned __int128 M = ((unsigned __int128)c.M_hi << 64) | c.M_lo;
  const unsigned long long w0 = col[0];
  const unsigned long long c1 = col[1] + (w0 >> 32);
  const unsigned long long c2 = col[2] + (c1 >> 32);
  const unsigned long long c3 = col[3] + (c2 >> 32);
  const unsigned long long lo = (w0 & 0xffffffffull) | (c1 << 32);
  const unsigned long long hi = (c2 & 0xffffffffull) | (c3 << 32);
  unsigned __int128 S = ((unsigned __int128)hi << 64) | lo;
  long long q = (long long)floor(((double)hi * 18446744073709551616.0 + (double)lo) * c.Mr);
  q = q < 0 ? 0 : q;
  S -= M * (unsigned long long)q;
  if ((__int128)S < 0) S += M;
  if (S >= M) S -= M;
  __int128 Z = (__int128)S;
  if (S > (M >> 1)) Z -= (__int128)M;
  const int e = -(exa[i] + exb[j]);
  const double s1 = ldexp(1.0, e / 2), s2 = ldexp(1.0, e - e / 2);
  C[(int64_t)i * ldc + 4 * j + t] =
      ((double)(long long)(Z >> 64) * 18446744073709551616.0 + (double)(unsigned long long)Z) * s1 * s2;
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 oz_encode() {
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

bool oz_map(CUtensorMap* map, const uint8_t* base, int64_t K, int64_t rows, int64_t pitch, int64_t L, int box_rows) {
  auto enc = oz_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)L};
  cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)(pitch * rows)};
  cuuint32_t box[3] = {(cuuint32_t)OZ_BK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// as oz_map with an explicit row stride and plane stride (bytes)
bool oz_map_strided(CUtensorMap* map, const uint8_t* base, int64_t K, int64_t rows, int64_t row_stride,
                    int64_t plane_stride, int64_t L, int box_rows) {
  auto enc = oz_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)L};
  cuuint64_t strides[2] = {(cuuint64_t)row_stride, (cuuint64_t)plane_stride};
  cuuint32_t box[3] = {(cuuint32_t)OZ_BK, (cuuint32_t)box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<uint8_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int oz_sms() {
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  return sms;
}

struct OzPlan {
  int L, bits;
  int64_t K, Kpitch, N, Npitch, BN, nblocks;
  size_t off_ares, off_bres, off_res, off_ex, off_fx, off_cmax, total;
};

OzPlan oz_plan(int64_t m, int64_t n, int64_t r, int L) {
  OzPlan p{};
  p.L = L;
  p.K = 4 * n;
  p.Kpitch = (p.K + 15) / 16 * 16;
  p.N = 4 * r;
  p.nblocks = (p.N + 255) / 256;
  p.BN = 16 * ((p.N + 16 * p.nblocks - 1) / (16 * p.nblocks));
  p.Npitch = p.nblocks * p.BN;
  double log2M = 0.0;
  for (int l = 0; l < L; ++l) log2M += std::log2((double)kOzModuli[l]);
  // |Z| <= K 2^(2 bits) < M / 2
  int bits = (int)std::floor((log2M - 1.0 - std::log2((double)p.K) - 1e-6) / 2.0);
  p.bits = bits > 51 ? 51 : bits;
  auto al = [](size_t v) { return (v + 255) / 256 * 256; };
  size_t o = 0;
  p.off_ares = o;
  o = al(o + (size_t)L * m * p.Kpitch);
  p.off_bres = o;
  o = al(o + (size_t)L * p.N * p.Kpitch);
  p.off_res = o;
  o = al(o + (size_t)L * m * p.Npitch);
  p.off_ex = o;
  o = al(o + (size_t)m * 4);
  p.off_fx = o;
  o = al(o + (size_t)r * 4);
  p.off_cmax = o;
  o = al(o + (size_t)r * 8);
  p.total = o;
  return p;
}

OzMods oz_mods(int L) {
  OzMods md{};
  md.L = L;
  for (int l = 0; l < L; ++l) {
    md.p[l] = kOzModuli[l];
    md.pd[l] = (double)kOzModuli[l];
    md.pinv[l] = 1.0 / (double)kOzModuli[l];
  }
  return md;
}

OzCrt oz_crt(int L) {
  OzCrt c{};
  c.L = L;
  unsigned __int128 M = 1;
  for (int l = 0; l < L; ++l) M *= (unsigned)kOzModuli[l];
  c.M_lo = (unsigned long long)M;
  c.M_hi = (unsigned long long)(M >> 64);
  c.Md = (double)c.M_hi * 18446744073709551616.0 + (double)c.M_lo;
  c.Mr = 1.0 / c.Md;
  for (int l = 0; l < L; ++l) {
    const int p = kOzModuli[l];
    const unsigned __int128 mi = M / (unsigned)p;
    for (int k = 0; k < 4; ++k) c.mi[l][k] = (unsigned)(mi >> (32 * k));
    const int mr = (int)(mi % (unsigned)p);
    int w = 1;
    while ((mr * w) % p != 1) ++w;
    c.w[l] = (float)w;
    c.P[l] = (float)p;
    c.pinv[l] = 1.0f / (float)p;
  }
  return c;
}

// INT8 tensor-core peak probe (roofline denominator): back-to-back tcgen05.mma kind::i8
// M = 128, N = 256, K = 32 from one pair of shared-memory tiles, one CTA per SM.
__global__ void __launch_bounds__(128, 1) k_i8_probe(int iters, int* sink) {
  __shared__ __align__(1024) uint8_t tiles[128 * 128 + 128 * 128];  // B rows 128..255 alias A (values are immaterial)
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (int)sizeof(tiles) / 4; i += blockDim.x) reinterpret_cast<int*>(tiles)[i] = 0x01010101;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(256 >> 3) << 17) | (8u << 24);
    const uint32_t a0 = smem_u32(tiles), b0 = a0;  // N = 256 rows read from the 32 KB block
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        mma_i8(tb + (uint32_t)((it & 1) * 256), umma_desc(a0 + k * 32), umma_desc(b0 + k * 32), idesc, 1u);
    mma_commit(&done);
    mbar_wait(&done, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    uint32_t v[32];
    if (threadIdx.x < 32) tmem_ld32(tb, v);
    if (threadIdx.x == 0 && v[0] == 0x7fffffffu) *sink = 1;  // keep the result live
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
  }
}

// plan of C = A^H B: K = p; A operand 4qa rows, B operand 4qb rows (N = 4qb)
struct OzHPlan {
  OzPlan g;  // K, Kpitch, N, Npitch, BN, nblocks, bits of the GEMM
  size_t off_wa, off_wb, off_res, off_exa, off_exb, off_ca, off_cb, total;
};

OzHPlan oz_hplan(int64_t p, int64_t qa, int64_t qb, int L, bool same) {
  OzHPlan h{};
  OzPlan& g = h.g;
  g.L = L;
  g.K = p;
  g.Kpitch = (p + 15) / 16 * 16;
  g.N = 4 * qb;
  g.nblocks = (g.N + 255) / 256;
  g.BN = 16 * ((g.N + 16 * g.nblocks - 1) / (16 * g.nblocks));
  g.Npitch = g.nblocks * g.BN;
  double log2M = 0.0;
  for (int l = 0; l < L; ++l) log2M += std::log2((double)kOzModuli[l]);
  // |P_ab| <= p 2^(2 bits), and the signed sum of four of them (one quaternion component, recovered
  // by a single CRT) stays below M / 2
  const int bits = (int)std::floor((log2M - 3.0 - std::log2((double)p) - 1e-6) / 2.0);
  g.bits = bits > 51 ? 51 : bits;
  auto al = [](size_t v) { return (v + 255) / 256 * 256; };
  size_t o = 0;
  h.off_wa = o;
  o = al(o + (size_t)L * 4 * qa * g.Kpitch);
  h.off_wb = o;
  if (!same) o = al(o + (size_t)L * 4 * qb * g.Kpitch);
  h.off_res = o;
  o = al(o + (size_t)L * 4 * qa * g.Npitch);
  h.off_exa = o;
  o = al(o + (size_t)qa * 4);
  h.off_exb = o;
  o = al(o + (size_t)qb * 4);
  h.off_ca = o;
  o = al(o + (size_t)qa * 8);
  h.off_cb = o;
  o = al(o + (size_t)qb * 8);
  h.total = o;
  return h;
}

// exponents (column maxima) and residues of the planes of Z (p x q) for the Hermitian products
OzPlaneJob oz_plane_job(const double* Z, int64_t p, int64_t q, int64_t ldz, int bits, unsigned long long* cmax,
                        int* ex, uint8_t* w, int64_t pitch) {
  OzPlaneJob j{};
  j.Z = Z;
  j.p = p;
  j.q = q;
  j.ldz = ldz;
  j.slabs = (int)((p + 63) / 64 < 64 ? (p + 63) / 64 : 64);
  j.rows_per = (p + j.slabs - 1) / j.slabs;
  j.pitch = pitch;
  j.plane = 4 * q * pitch;
  j.bits = bits;
  j.cmax = cmax;
  j.ex = ex;
  j.w = w;
  return j;
}

void oz_planes_launch(const OzPlaneJob* jobs, int n, int L, cudaStream_t st) {
  OzPlaneJobs J{};
  unsigned cb = 1, sl = 1, rb = 1;
  for (int k = 0; k < n; ++k) {
    J.j[k] = jobs[k];
    cudaMemsetAsync(jobs[k].cmax, 0, (size_t)jobs[k].q * 8, st);
    cb = std::max(cb, (unsigned)((jobs[k].q + 31) / 32));
    sl = std::max(sl, (unsigned)jobs[k].slabs);
    rb = std::max(rb, (unsigned)((jobs[k].q * (jobs[k].pitch / 4) + 255) / 256));
  }
  ++::qcur::g_launches;
  k_oz_pmax<<<dim3(cb, sl, (unsigned)n), 256, 0, st>>>(J);
  ++::qcur::g_launches;
  if (L == 14)
    k_oz_pres<14><<<dim3(rb, (unsigned)n), 256, 0, st>>>(J);
  else
    k_oz_pres<15><<<dim3(rb, (unsigned)n), 256, 0, st>>>(J);
}

}  // namespace

int ozaki_max_moduli() { return kOzMaxMod; }

// the residues of X run on the context's low-priority side stream: a captured graph gives their nodes
// the low priority explicitly (graph replays otherwise run every node at the launch stream's priority)
bool ozaki_side_kernel(const void* f) {
  return f == (const void*)k_oz_xres<15, 256, 8, 2> || f == (const void*)k_oz_xres<15, 256, 16, 2> ||
         f == (const void*)k_oz_xres<14, 256, 16, 2> || f == (const void*)k_oz_xres<15, 512, 8, 1>;
}

size_t ozaki_herm_workspace_bytes(int64_t p, int64_t qa, int64_t qb, int same) {
  return oz_hplan(p, qa, qb, kOzMaxModDefault, same != 0).total + 1024;
}

bool ozaki_herm_supported(int64_t p, int64_t qa, int64_t qb) {
  // odd-moduli residues in [-127, 127]: p 127^2 < 2^31; workspace cap as the other products
  return p >= 1 && qa >= 1 && qb >= 1 && p <= 133140 &&
         (double)oz_hplan(p, qa, qb, kOzMaxModDefault, false).total <= 4e9;
}



// dense INT8 tensor-core rate of this GPU in TOP/s (2 ops per multiply-add)
double run_i8_peak(int sms, cudaStream_t st) {
  int* sink = nullptr;
  if (cudaMalloc(&sink, 64) != cudaSuccess) return 0.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 2000;
  ++::qcur::g_launches;
  k_i8_probe<<<sms, 128, 0, st>>>(100, sink);
  float ms = 0.f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0, st);
    ++::qcur::g_launches;
    k_i8_probe<<<sms, 128, 0, st>>>(iters, sink);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < 20.f) iters = (int)(iters * (40.f / (ms > 0.01f ? ms : 0.01f)));
    else break;
  }
  const double ops = 2.0 * 128.0 * 256.0 * 32.0 * 4.0 * (double)iters * (double)sms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  return ms > 0.f ? ops / ((double)ms * 1e-3) / 1e12 : 0.0;
}

size_t ozaki_workspace_bytes(int64_t m, int64_t n, int64_t r, int L) { return oz_plan(m, n, r, L).total + 1024; }

// Rows per chunk for a product whose whole-matrix workspace exceeds the cap: the residues of X
// are produced and consumed one chunk of rows at a time (rows are independent: each row's
// scale comes from its own maximum), E(B)'s residues once.  0 when no chunk of 256 rows fits.
int64_t ozaki_chunk_rows(int64_t m, int64_t n, int64_t r, double cap_bytes) {
  if (m < 1 || n < 1 || r < 1 || 4 * n > 133140) return 0;
  const double fixed = (double)oz_plan(0, n, r, kOzMaxModDefault).total;
  const double per_row = (double)oz_plan(256, n, r, kOzMaxModDefault).total / 256.0 - fixed / 256.0;
  if (!(per_row > 0.0) || fixed + 256.0 * per_row > cap_bytes) return 0;
  int64_t rows = (int64_t)((cap_bytes - fixed) / per_row) / 256 * 256;
  if (rows > m) rows = m;
  return rows;
}

bool ozaki_supported(int64_t m, int64_t n, int64_t r) {
  // int32 accumulation: the odd moduli have residues in [-127, 127], so 4n 127^2 < 2^31; for
  // p = 256 the accumulator may wrap, which leaves it exact mod 2^32 and hence mod 256.
  // Residues of X take 15 bytes per real of X (and E(B) 15 bytes per real of E(B)).
  // workspace cap of the one-shot product (else row chunks or the FP64 engine); QCUR_OZ_ONESHOT_CAP
  // lowers it for tests of the chunked path
  const char* cap_env = std::getenv("QCUR_OZ_ONESHOT_CAP");
  const double cap = cap_env ? std::atof(cap_env) : 4e9;
  return m >= 1 && n >= 1 && r >= 1 && 4 * n <= 133140 && (double)oz_plan(m, n, r, kOzMaxModDefault).total <= cap;
}

// SMs the side-stream residues of X leave free for the main stream (QCUR_XRES_RESERVE=n; default 0: one
// 256-thread CTA per row, two per SM, on every SM).  Measured at cfg2 with n = 28: the graph's draw phase
// 191 -> 121 us, but the residues then stretch over the factorization (1.09 -> 1.17 ms): one at a time
// 298 -> 293 approx/s, cfg1 in flight 6066 -> 5645, cfg4 4534 -> 4276; so off.
int xres_reserve() {
  static const int v = [] {
    const char* e = std::getenv("QCUR_XRES_RESERVE");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

// values per thread of k_oz_xres: 8 (no spills; cfg2 385.6 -> 367.5 us, ncu); QCUR_XRES_VPT=16 for A/B timing
int xres_vpt() {
  static const int v = [] {
    const char* e = std::getenv("QCUR_XRES_VPT");
    return e && std::atoi(e) == 16 ? 16 : 8;
  }();
  return v;
}

// Phase 1 (depends on X only; may run on a side stream): row exponents and residues of X.
int launch_ozaki_prepare(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t r, int L, void* workspace,
                         cudaStream_t st) {
  if (L < 14 || L > 15) return 1;
  const OzPlan pl = oz_plan(m, n, r, L);
  uint8_t* ws = reinterpret_cast<uint8_t*>(((uintptr_t)workspace + 255) / 256 * 256);
  uint8_t* ares = ws + pl.off_ares;
  int* ex = reinterpret_cast<int*>(ws + pl.off_ex);
  const int64_t aplane = m * pl.Kpitch;
  ++::qcur::g_launches;
  switch (L) {
    case 14: k_oz_xres<14, 256><<<(unsigned)m, 256, 0, st>>>(X, pl.K, ldx * 4, pl.bits, ares, pl.Kpitch, aplane, ex, m); break;
    case 15: {
      const int reserve = xres_reserve();
      if (reserve > 0 && m > oz_sms() - reserve) {
        const int grid = oz_sms() - reserve;
        k_oz_xres<15, 512, 8, 1><<<(unsigned)grid, 512, 0, st>>>(X, pl.K, ldx * 4, pl.bits, ares, pl.Kpitch, aplane, ex, m);
      } else if (xres_vpt() == 8) {
        k_oz_xres<15, 256, 8><<<(unsigned)m, 256, 0, st>>>(X, pl.K, ldx * 4, pl.bits, ares, pl.Kpitch, aplane, ex, m);
      } else {
        k_oz_xres<15, 256><<<(unsigned)m, 256, 0, st>>>(X, pl.K, ldx * 4, pl.bits, ares, pl.Kpitch, aplane, ex, m);
      }
      break;
    }
    default: return 1;
  }
  return 0;
}

// Phase 1 for rows [row0, row0 + rows) of an m-row X (the chunk at X_rows): the same residues and
// exponents launch_ozaki_prepare writes for those rows (used while X is uploaded chunk by chunk)
int launch_ozaki_prepare_rows(const double* X_rows, int64_t rows, int64_t row0, int64_t m, int64_t n, int64_t ldx,
                              int64_t r, int L, void* workspace, cudaStream_t st) {
  if (L != 15 || rows < 1) return 1;
  const OzPlan pl = oz_plan(m, n, r, L);
  uint8_t* ws = reinterpret_cast<uint8_t*>(((uintptr_t)workspace + 255) / 256 * 256);
  uint8_t* ares = ws + pl.off_ares + row0 * pl.Kpitch;
  int* ex = reinterpret_cast<int*>(ws + pl.off_ex) + row0;
  ++::qcur::g_launches;
  k_oz_xres<15, 256, 8><<<(unsigned)rows, 256, 0, st>>>(X_rows, pl.K, ldx * 4, pl.bits, ares, pl.Kpitch,
                                                         m * pl.Kpitch, ex, rows);
  return 0;
}

// Phase 2a: column exponents and residues of E(B).
int launch_ozaki_prep_b(int64_t m, int64_t n, const double* B, int64_t r, int64_t ldb, int L, void* workspace,
                        cudaStream_t st) {
  if (L < 14 || L > 15) return 1;
  const OzPlan pl = oz_plan(m, n, r, L);
  uint8_t* ws = reinterpret_cast<uint8_t*>(((uintptr_t)workspace + 255) / 256 * 256);
  uint8_t* bres = ws + pl.off_bres;
  int* fx = reinterpret_cast<int*>(ws + pl.off_fx);
  const OzMods md = oz_mods(L);
  const int64_t bplane = pl.N * pl.Kpitch;
  // one launch (a 1024-thread CTA per quaternion column of B: maximum, exponent, residues) for small B:
  // measured per approximation cfg1 22.6 -> 16.9 us, cfg4 23.1 -> 16.9, cfg3 c = 128 31.2 -> 25.9, but at
  // cfg2 (n r = 8e5, 200 CTAs) 66 -> 82 us; bit-identical.  QCUR_PREPB_BCOL=0/1 forces either way.
  static const int bcol_env = [] {
    const char* e = std::getenv("QCUR_PREPB_BCOL");
    return e ? std::atoi(e) : -1;
  }();
  if (bcol_env == 1 || (bcol_env < 0 && (double)n * (double)r <= 4e5)) {
    OzBColJobs bj{};
    bj.j[0] = OzBColJob{B, n, r, ldb, pl.Kpitch, bplane, 0, pl.bits, fx, bres};
    ++::qcur::g_launches;
    if (bres_fast_on() && md.L == 15) k_oz_bcol<1024, 15><<<dim3((unsigned)r, 1), 1024, 0, st>>>(bj, md);
    else if (bres_fast_on() && md.L == 14) k_oz_bcol<1024, 14><<<dim3((unsigned)r, 1), 1024, 0, st>>>(bj, md);
    else k_oz_bcol<1024><<<dim3((unsigned)r, 1), 1024, 0, st>>>(bj, md);
    return 0;
  }
  unsigned long long* cmax = reinterpret_cast<unsigned long long*>(ws + pl.off_cmax);
  cudaMemsetAsync(cmax, 0, (size_t)r * 8, st);
  const int64_t slabs = (n + 63) / 64 < 64 ? (n + 63) / 64 : 64, rows_per = (n + slabs - 1) / slabs;
  ++::qcur::g_launches;
  k_oz_bmax<<<dim3((unsigned)((r + 31) / 32), (unsigned)slabs), 256, 0, st>>>(B, n, r, ldb, rows_per, cmax);
  ++::qcur::g_launches;
  k_oz_bexp<<<(unsigned)((r + 255) / 256), 256, 0, st>>>(cmax, r, pl.bits, fx);
  const int64_t nb_threads = r * (pl.Kpitch / 4);
  ++::qcur::g_launches;
  const int bres_env = bres_fast_on();
  const unsigned nblk = (unsigned)((nb_threads + 255) / 256);
  const dim3 tgrid((unsigned)((pl.Kpitch / 4 + 31) / 32), (unsigned)((r + 7) / 8));
  if (bres_env == 3 && md.L == 15)
    k_oz_bres_tile<15><<<tgrid, 256, 0, st>>>(B, n, r, ldb, fx, bres, pl.Kpitch, bplane);
  else if (bres_env == 3 && md.L == 14)
    k_oz_bres_tile<14><<<tgrid, 256, 0, st>>>(B, n, r, ldb, fx, bres, pl.Kpitch, bplane);
  else if (bres_env && md.L == 15)
    k_oz_bres_fast<15><<<nblk, 256, 0, st>>>(B, n, r, ldb, fx, bres, pl.Kpitch, bplane);
  else if (bres_env && md.L == 14)
    k_oz_bres_fast<14><<<nblk, 256, 0, st>>>(B, n, r, ldb, fx, bres, pl.Kpitch, bplane);
  else
    k_oz_bres<<<nblk, 256, 0, st>>>(B, n, r, ldb, md, fx, bres, pl.Kpitch, bplane);
  return 0;
}

// one product of a launch: A residues (tensor map over `ares`, rows `arow_stride` bytes apart),
// B residues, and where the residue bytes of the product go
struct OzJob {
  CUtensorMap ta, tb;
  CUtensorMap tbh;  // B in boxes of BN / 2 rows (k_oz_gemm_bmc: each CTA of a pair loads one half)
  OzProb pr;
};

// a symmetric product (A = B): keep only the tiles meeting the lower triangle
void oz_job_lower(OzJob& j, int L) {
  OzProb& q = j.pr;
  q.lower = 1;
  q.tiles = 0;
  for (int mb = 0; mb < q.mblocks; ++mb) q.tiles += oz_row_tiles(q, mb);
  const bool last_half = !((int64_t)(q.mblocks - 1) * OZ_BM + OZ_BM / 2 < q.m);
  q.fulls = last_half ? q.tiles - oz_row_tiles(q, q.mblocks - 1) : q.tiles;
  q.units = L * q.tiles;
}

bool oz_job(OzJob& j, const OzPlan& pl, int64_t m, const uint8_t* ares, int64_t arow_stride, const uint8_t* bres,
            int L, uint8_t* res) {
  // A planes are m rows of arow_stride bytes (Kpitch for X, 4 Kpitch for the rows 4j of E(A))
  if (!oz_map_strided(&j.ta, ares, pl.K, m, arow_stride, arow_stride * m, L, OZ_BM / 2) ||
      !oz_map(&j.tb, bres, pl.K, pl.N, pl.Kpitch, L, (int)pl.BN) ||
      !oz_map(&j.tbh, bres, pl.K, pl.N, pl.Kpitch, L, (int)pl.BN / 2))
    return false;
  OzProb& q = j.pr;
  q.m = m;
  q.N = pl.N;
  q.kblocks = (int)((pl.K + OZ_BK - 1) / OZ_BK);
  q.mblocks = (int)((m + OZ_BM - 1) / OZ_BM);
  q.nblocks = (int)pl.nblocks;
  q.BN = (int)pl.BN;
  q.lower = 0;
  q.tiles = q.mblocks * q.nblocks;
  q.fulls = (int64_t)(q.mblocks - 1) * OZ_BM + OZ_BM / 2 < m ? q.tiles : q.tiles - q.nblocks;
  q.units = L * q.tiles;
  // kind::i8: D = s32 (bits 4-5 = 2), A/B signed (bits 7-9, 10-12 = 1), K-major, N>>3 at 17, M>>4 at 24 (M = 128)
  q.idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(q.BN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  q.res = res;
  q.res_pitch = pl.Npitch;
  q.res_plane = m * pl.Npitch;
  return true;
}

void oz_launch_gemm(const OzJob* jobs, int nj, int L, cudaStream_t st) {
  OzGemm P{};
  P.L = L;
  P.pr[0] = jobs[0].pr;
  P.pr[1] = nj > 1 ? jobs[1].pr : jobs[0].pr;
  P.total = jobs[0].pr.units + (nj > 1 ? jobs[1].pr.units : 0);
  P.nfull = L * (jobs[0].pr.fulls + (nj > 1 ? jobs[1].pr.fulls : 0));
  for (int l = 0; l < L; ++l) {
    P.p[l] = kOzModuli[l];
    P.bm[l] = (int)((1ull << 32) / (unsigned long long)kOzModuli[l]);  // < 2^31 for p >= 3 (p = 256 unused)
    P.pinv[l] = 1.0 / (double)kOzModuli[l];
  }
  static std::atomic<unsigned> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_oz_gemm<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM);
    cudaFuncSetAttribute(k_oz_gemm<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, OZ_SMEM);
  }
  static const int exp_env = [] {
    const char* e = std::getenv("QCUR_OZ_EXP");
    return e ? std::atoi(e) : 0;
  }();
  P.exp = exp_env;
  static const int cl_env = [] {
    const char* e = std::getenv("QCUR_OZ_CLUSTER");
    return e ? std::atoi(e) : 0;
  }();
  const bool any_lower = jobs[0].pr.lower || (nj > 1 && jobs[1].pr.lower);
  const int CL = any_lower ? 1 : cl_env == 1 || cl_env == 2 ? cl_env : kOzCluster;
  const OzJob& j1 = nj > 1 ? jobs[1] : jobs[0];
  static const int bmc_env = [] {  // QCUR_OZ_BMC=1: the B-multicast pair kernel (correct, bit-identical; measured
    const char* e = std::getenv("QCUR_OZ_BMC");  // no faster: Gram 84 -> 82-85 us, X Q_R 563 -> 588 us)
    return e ? std::atoi(e) : 0;
  }();
  if (bmc_env && cl_env == 0) {
    static std::atomic<unsigned> battr{0};
    static int max_clusters = 0;
    cudaLaunchConfig_t cfg{};
    cfg.blockDim = dim3(OZ_THREADS);
    cfg.dynamicSmemBytes = OZB_SMEM;
    cfg.stream = st;
    if (first_on_device(battr)) {
      cudaFuncSetAttribute(k_oz_gemm_bmc, cudaFuncAttributeMaxDynamicSharedMemorySize, OZB_SMEM);
      int nc = 0;
      cfg.gridDim = dim3((unsigned)(oz_sms() / 2 * 2));
      max_clusters = (cudaOccupancyMaxActiveClusters(&nc, k_oz_gemm_bmc, &cfg) == cudaSuccess && nc > 0) ? nc
                                                                                                         : oz_sms() / 2;
      (void)cudaGetLastError();
    }
    const int ncl = P.total < max_clusters ? P.total : max_clusters;
    cfg.gridDim = dim3((unsigned)(2 * ncl));
    ++::qcur::g_launches;
    cudaLaunchKernelEx(&cfg, k_oz_gemm_bmc, jobs[0].ta, jobs[0].tbh, j1.ta, j1.tbh, P);
    return;
  }
  ++::qcur::g_launches;
  if (CL == 1) {
    const int grid = P.total < oz_sms() ? P.total : oz_sms();
    k_oz_gemm<1><<<grid, OZ_THREADS, OZ_SMEM, st>>>(jobs[0].ta, jobs[0].tb, j1.ta, j1.tb, P);
    return;
  }
  // clusters of two CTAs over pairs of column blocks: units count the pairs
  for (int k = 0; k < 2; ++k) P.pr[k].units = L * P.pr[k].mblocks * ((P.pr[k].nblocks + 1) / 2);
  P.total = P.pr[0].units + (nj > 1 ? P.pr[1].units : 0);
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(OZ_THREADS);
  cfg.dynamicSmemBytes = OZ_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static int max_active = 0;
  if (!max_active) {
    int nc = 0;
    cfg.gridDim = dim3((unsigned)(oz_sms() / 2 * 2));
    max_active = (cudaOccupancyMaxActiveClusters(&nc, k_oz_gemm<2>, &cfg) == cudaSuccess && nc > 0) ? nc : oz_sms() / 2;
    (void)cudaGetLastError();
  }
  const int nclusters = P.total < max_active ? P.total : max_active;
  cfg.gridDim = dim3((unsigned)(2 * nclusters));
  cudaLaunchKernelEx(&cfg, k_oz_gemm<2>, jobs[0].ta, jobs[0].tb, j1.ta, j1.tb, P);
}

int oz_launch_crt(const uint8_t* res, int64_t m, const OzPlan& pl, const int* ex, const int* fx, double* Y,
                  int64_t ldy, int L, cudaStream_t st) {
  const OzCrt cc = oz_crt(L);
  const unsigned cblocks = (unsigned)((m * (pl.N / 4) + 255) / 256);
  const int64_t rplane = m * pl.Npitch;
  ++::qcur::g_launches;
  switch (L) {
    case 14: k_oz_crt<14><<<cblocks, 256, 0, st>>>(res, m, pl.N, pl.Npitch, rplane, ex, fx, cc, Y, ldy * 4); break;
    case 15: k_oz_crt<15><<<cblocks, 256, 0, st>>>(res, m, pl.N, pl.Npitch, rplane, ex, fx, cc, Y, ldy * 4); break;
    default: return 1;
  }
  return 0;
}

// Phase 2b: the L int8 GEMMs on tcgen05 and the CRT into Y (m x r).
int launch_ozaki_multiply(int64_t m, int64_t n, int64_t r, double* Y, int64_t ldy, int L, void* workspace,
                          cudaStream_t st) {
  if (L < 14 || L > 15) return 1;
  const OzPlan pl = oz_plan(m, n, r, L);
  uint8_t* ws = reinterpret_cast<uint8_t*>(((uintptr_t)workspace + 255) / 256 * 256);
  OzJob j;
  if (!oz_job(j, pl, m, ws + pl.off_ares, pl.Kpitch, ws + pl.off_bres, L, ws + pl.off_res)) return 2;
  oz_launch_gemm(&j, 1, L, st);
  return oz_launch_crt(ws + pl.off_res, m, pl, reinterpret_cast<int*>(ws + pl.off_ex),
                       reinterpret_cast<int*>(ws + pl.off_fx), Y, ldy, L, st);
}


int launch_ozaki_finish(int64_t m, int64_t n, const double* B, int64_t r, int64_t ldb, double* Y, int64_t ldy, int L,
                        void* workspace, cudaStream_t st) {
  int rc = launch_ozaki_prep_b(m, n, B, r, ldb, L, workspace, st);
  return rc ? rc : launch_ozaki_multiply(m, n, r, Y, ldy, L, workspace, st);
}

// Y (m x r) = X (m x n) * B (n x r), interleaved quaternions (ld in quaternions)
int launch_ozaki_gemm(const double* X, int64_t m, int64_t n, int64_t ldx, const double* B, int64_t r, int64_t ldb,
                      double* Y, int64_t ldy, int L, void* workspace, cudaStream_t st) {
  int rc = launch_ozaki_prepare(X, m, n, ldx, r, L, workspace, st);
  return rc ? rc : launch_ozaki_finish(m, n, B, r, ldb, Y, ldy, L, workspace, st);
}

// Y_k (m_k x r_k) = X_k (m_k x n_k) op(B_k) for np <= 2 problems with small right operands (the
// triangular products Q_1 = Z L_1^{-H} of a factorization step): residues of each X_k (one CTA per
// row), of every op(B_k) in one k_oz_bcol launch, one tcgen05 launch for all products, one CRT each.
// conjT[k]: op(B_k) = B_k^H (B_k is r_k x n_k).  workspace[k]: ozaki_workspace_bytes(m_k, n_k, r_k, L).
int launch_ozaki_pair(const double* const* X, const int64_t* m, const int64_t* n, const int64_t* ldx,
                      const double* const* B, const int64_t* r, const int64_t* ldb, const int* conjT, double* const* Y,
                      const int64_t* ldy, int np, int L, void* const* workspace, cudaStream_t st) {
  if (L < 14 || L > 15 || np < 1 || np > 2) return 1;
  OzJob jobs[2];
  OzPlan pl[2];
  uint8_t* ws[2];
  OzBColJobs bj{};
  int64_t rmax = 0;
  for (int k = 0; k < np; ++k) {
    pl[k] = oz_plan(m[k], n[k], r[k], L);
    ws[k] = reinterpret_cast<uint8_t*>(((uintptr_t)workspace[k] + 255) / 256 * 256);
    uint8_t* ares = ws[k] + pl[k].off_ares;
    int* ex = reinterpret_cast<int*>(ws[k] + pl[k].off_ex);
    ++::qcur::g_launches;
    if (L == 14)
      k_oz_xres<14, 256><<<(unsigned)m[k], 256, 0, st>>>(X[k], pl[k].K, ldx[k] * 4, pl[k].bits, ares, pl[k].Kpitch,
                                                         m[k] * pl[k].Kpitch, ex, m[k]);
    else
      k_oz_xres<15, 256><<<(unsigned)m[k], 256, 0, st>>>(X[k], pl[k].K, ldx[k] * 4, pl[k].bits, ares, pl[k].Kpitch,
                                                         m[k] * pl[k].Kpitch, ex, m[k]);
    bj.j[k] = OzBColJob{B[k], n[k], r[k], ldb[k], pl[k].Kpitch, pl[k].N * pl[k].Kpitch, conjT[k], pl[k].bits,
                        reinterpret_cast<int*>(ws[k] + pl[k].off_fx), ws[k] + pl[k].off_bres};
    rmax = r[k] > rmax ? r[k] : rmax;
    if (!oz_job(jobs[k], pl[k], m[k], ares, pl[k].Kpitch, ws[k] + pl[k].off_bres, L, ws[k] + pl[k].off_res)) return 2;
  }
  ++::qcur::g_launches;
  if (bres_fast_on() && L == 15) k_oz_bcol<256, 15><<<dim3((unsigned)rmax, (unsigned)np), 256, 0, st>>>(bj, oz_mods(L));
  else if (bres_fast_on() && L == 14) k_oz_bcol<256, 14><<<dim3((unsigned)rmax, (unsigned)np), 256, 0, st>>>(bj, oz_mods(L));
  else k_oz_bcol<256><<<dim3((unsigned)rmax, (unsigned)np), 256, 0, st>>>(bj, oz_mods(L));
  oz_launch_gemm(jobs, np, L, st);
  for (int k = 0; k < np; ++k) {
    const int rc = oz_launch_crt(ws[k] + pl[k].off_res, m[k], pl[k], reinterpret_cast<int*>(ws[k] + pl[k].off_ex),
                                 reinterpret_cast<int*>(ws[k] + pl[k].off_fx), Y[k], ldy[k], L, st);
    if (rc) return rc;
  }
  return 0;
}

// C_k (qa_k x qb_k) = A_k^H B_k for np <= 2 problems (A_k: p_k x qa_k, B_k: p_k x qb_k, B_k == A_k
// allowed: its planes are formed once); one INT8 GEMM launch for all of them
int launch_ozaki_herm(const double* const* A, const double* const* B, const int64_t* p, const int64_t* qa,
                      const int64_t* qb, const int64_t* lda, const int64_t* ldb, double* const* C,
                      const int64_t* ldc, int np, int L, void* const* workspace, cudaStream_t st, int lower_only) {
  if (L < 14 || L > 15 || np < 1 || np > 2) return 1;
  static const int lower_env = [] {  // QCUR_OZ_LOWER=0: full plane Grams (A/B timing)
    const char* e = std::getenv("QCUR_OZ_LOWER");
    return e ? std::atoi(e) : 1;
  }();
  OzJob jobs[2];
  OzHPlan hp[2];
  uint8_t* ws[2];
  OzPlaneJob pj[4];
  int npj = 0;
  for (int k = 0; k < np; ++k) {
    const bool same = A[k] == B[k] && qa[k] == qb[k] && lda[k] == ldb[k];
    hp[k] = oz_hplan(p[k], qa[k], qb[k], L, same);
    ws[k] = reinterpret_cast<uint8_t*>(((uintptr_t)workspace[k] + 255) / 256 * 256);
    const OzHPlan& h = hp[k];
    uint8_t* wa = ws[k] + h.off_wa;
    uint8_t* wb = same ? wa : ws[k] + h.off_wb;
    int* exa = reinterpret_cast<int*>(ws[k] + h.off_exa);
    int* exb = same ? exa : reinterpret_cast<int*>(ws[k] + h.off_exb);
    pj[npj++] = oz_plane_job(A[k], p[k], qa[k], lda[k], h.g.bits,
                             reinterpret_cast<unsigned long long*>(ws[k] + h.off_ca), exa, wa, h.g.Kpitch);
    if (!same)
      pj[npj++] = oz_plane_job(B[k], p[k], qb[k], ldb[k], h.g.bits,
                               reinterpret_cast<unsigned long long*>(ws[k] + h.off_cb), exb, wb, h.g.Kpitch);
    if (!oz_job(jobs[k], h.g, 4 * qa[k], wa, h.g.Kpitch, wb, L, ws[k] + h.off_res)) return 2;
    if (same && lower_env) oz_job_lower(jobs[k], L);
  }
  oz_planes_launch(pj, npj, L, st);
  oz_launch_gemm(jobs, np, L, st);
  const OzCrt cc = oz_crt(L);
  OzHcrtJobs H{};
  int gx = 0;
  for (int k = 0; k < np; ++k) {
    const OzHPlan& h = hp[k];
    const bool same = A[k] == B[k] && qa[k] == qb[k] && lda[k] == ldb[k];
    OzHcrtProb& P = H.p[k];
    P.exa = reinterpret_cast<int*>(ws[k] + h.off_exa);
    P.exb = same ? P.exa : reinterpret_cast<int*>(ws[k] + h.off_exb);
    P.qa = qa[k];
    P.qb = qb[k];
    P.ldc = ldc[k] * 4;
    P.C = C[k];
    P.lower_bn = jobs[k].pr.lower ? jobs[k].pr.BN : 0;
    const int nba = (int)((qa[k] + kHB - 1) / kHB), nbb = (int)((qb[k] + kHB - 1) / kHB);
    P.tri = same && lower_only ? 1 : 0;
    P.nbx = nbb;
    P.nblk = P.tri ? nba * (nba + 1) / 2 : nba * nbb;
    gx = P.nblk > gx ? P.nblk : gx;
    // residue planes as a 3-D tensor: columns (Npitch bytes), rows (4 qa), moduli; 16 x 16 x L boxes
    auto enc = oz_encode();
    cuuint64_t dims[3] = {(cuuint64_t)h.g.Npitch, (cuuint64_t)(4 * qa[k]), (cuuint64_t)L};
    cuuint64_t strides[2] = {(cuuint64_t)h.g.Npitch, (cuuint64_t)(4 * qa[k] * h.g.Npitch)};
    cuuint32_t box[3] = {(cuuint32_t)kHBW, (cuuint32_t)kHB, (cuuint32_t)L};
    cuuint32_t estr[3] = {1, 1, 1};
    if (!enc || enc(&P.tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, ws[k] + h.off_res, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return 2;
  }
  static std::atomic<unsigned> hattr{0};
  if (first_on_device(hattr)) {
    cudaFuncSetAttribute(k_oz_hcrt<14>, cudaFuncAttributeMaxDynamicSharedMemorySize, kOzHcrtSmem);
    cudaFuncSetAttribute(k_oz_hcrt<15>, cudaFuncAttributeMaxDynamicSharedMemorySize, kOzHcrtSmem);
  }
  const dim3 grid((unsigned)gx, 4, (unsigned)np);
  ++::qcur::g_launches;
  if (L == 14)
    k_oz_hcrt<14><<<grid, kHB * kHB, kOzHcrtSmem, st>>>(H, cc);
  else
    k_oz_hcrt<15><<<grid, kHB * kHB, kOzHcrtSmem, st>>>(H, cc);
  return 0;
}

}  // namespace qcur
