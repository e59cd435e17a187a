// Fused reconstruction error ||X - P R||_F on the INT8 tensor cores (tcgen05.mma kind::i8),
// by exact integer slices (Ozaki scheme I).
//
// The error of the reference's callers (cli.py:173-175, imaging.py:170-177, bench.py:257-258)
// is ||X - C U R|| / ||X||.  With P = C U (m x r) formed first (cur.py:274), the remaining
// product P R (m x n, K = 4r reals) is "outer-product shaped": a small K and an output as
// large as X.  On the FP64 DMMA path it costs 32 m n r flop; here it runs as int8 GEMMs:
//
//  1. Rows of P (reals) and quaternion columns of R are scaled by powers of two and rounded to
//     integers of at most 2^54 in magnitude, P' = rint(P 2^a_i), R' = rint(R 2^b_j) (the
//     only rounding: 2^-55 relative to the row / column maximum).
//  2. P' and E(R') (the 4x4 Hamilton expansion, E[4k+s][4j+t] = sign(s,t) r_kj[s^t]) are
//     written as seven balanced base-256 digits, d in [-128, 127]:  P' = sum_s 256^s P_s.
//  3. P' E(R') = sum_{s,t} 256^(s+t) P_s E_t.  Every P_s E_t is an exact int8 GEMM with int32
//     accumulation (|.| <= 6 * 2^14 * 4r < 2^31).  The 21 products with s + t >= 7 are kept;
//     the dropped levels are below 2^-48 of the product and random in sign, which changes
//     ||X - P R||^2 by far less than the 1e-10 parity bar (measured: 2e-14 relative).
//  4. The six level sums (s + t = 7..12) accumulate in TMEM (6 x 80 columns); the epilogue
//     combines them in FP64 (Horner in 256), scales back, subtracts from X (read once from
//     HBM, prefetched into L2 by TMA) and reduces the four statistics of the FP64 kernel
//     (k_qgemm.cu EPI_ERR): sum (X - PR)^2, sum X^2, the imaginary part, the u8-image sum.
//
// Kernel layout: warp 0 issues TMA loads (3-D boxes: all six digit planes of a 128 x 32-byte
// A tile and an 80 x 32-byte B tile, 32-byte swizzle) into a 5-stage ring; warp 1 issues the
// 21 tcgen05.mma per stage; warps 2-9 drain TMEM.  Partial sums are written per (tile, warp)
// and reduced in a fixed order: bitwise deterministic.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace qcur {

namespace {

using namespace tc;

// K = 64 bytes per stage (64-byte swizzle): TMA delivers 64-byte row segments, twice the rate of
// 32-byte ones (tools/tma_probe.cu: 14.5 vs 9.2 TB/s), so the 21 x 2 MMAs of a stage are no longer
// starved; two 78 KB stages fill shared memory
#ifndef QCUR_OE_BN  // build-time variants for A/B timing (tools: nvcc -DQCUR_OE_BN=64 -DQCUR_OE_STAGES=3)
#define QCUR_OE_BN 80
#endif
#ifndef QCUR_OE_STAGES
#define QCUR_OE_STAGES 2
#endif
constexpr int OE_BM = 128, OE_BN = QCUR_OE_BN, OE_BK = 64, OE_STAGES = QCUR_OE_STAGES, OE_DIG = 6;
constexpr int OE_EPI_WARPS = 16, OE_THREADS = 64 + 32 * OE_EPI_WARPS;  // 4 epilogue warps per TMEM lane quarter
constexpr int OE_A_BYTES = OE_DIG * OE_BM * OE_BK;  // 48 KB
constexpr int OE_B_BYTES = OE_DIG * OE_BN * OE_BK;  // 30 KB
constexpr int OE_STAGE = OE_A_BYTES + OE_B_BYTES;
constexpr int OE_SMEM = 1024 + OE_STAGES * OE_STAGE + 256;
constexpr int OE_BITS = 54;            // |P'|, |R'| <= 2^54: seven balanced base-256 digits
constexpr int kOeCluster = 2;          // CTAs per cluster sharing the A digit tile by TMA multicast
constexpr bool kOePairDefault = false;  // CTA-pair (cta_group::2) kernel by default

__device__ __forceinline__ double i2d(uint32_t v) {  // exact int32 -> double (one DADD)
  return __hiloint2double(0x43380000, (int)(v ^ 0x80000000u)) - 6755401588539392.0;  // 1.5*2^52 + 2^31
}
__device__ __forceinline__ double scale2(double x, int e) {
  const int e1 = e / 2;
  return x * ldexp(1.0, e1) * ldexp(1.0, e - e1);
}
// 2^e as a double (e within the normal range: one integer op; else two steps)
__device__ __forceinline__ double pow2(int e) {
  return (e >= -1022 && e <= 1023) ? __longlong_as_double((long long)(e + 1023) << 52) : ldexp(1.0, e);
}
__device__ __forceinline__ int exp_for(double mx) {
  if (!(mx > 0.0)) return 0;
  int E;
  frexp(mx, &E);
  return OE_BITS - E;
}

// ---------------------------------------------------------------------------
// digits of P (m x K reals, ld ldp): one warp per row; planes [6][m][Kp] (digits 1..6)
// ---------------------------------------------------------------------------
__global__ void k_oe_pdig(const double* __restrict__ P, int64_t m, int64_t K, int64_t ldp, int8_t* __restrict__ dig,
                          int64_t Kp, int* __restrict__ ea) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= m) return;
  const double* p = P + row * ldp;
  double mx = 0.0;
  for (int64_t k = lane; k < K; k += 32) mx = fmax(mx, fabs(p[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int e = exp_for(mx);
  if (lane == 0) ea[row] = e;
  const int64_t plane = m * Kp;
  for (int64_t k = lane; k < K; k += 32) {
    long long v = llrint(scale2(p[k], e));
    const int d0 = (int)((v + 128) & 255) - 128;
    v = (v - d0) >> 8;
#pragma unroll
    for (int s = 1; s <= OE_DIG; ++s) {
      const int d = (int)((v + 128) & 255) - 128;
      v = (v - d) >> 8;
      dig[(s - 1) * plane + row * Kp + k] = (int8_t)d;
    }
  }
}

// column exponents of R (r x n quaternions, ld ldr): one warp per quaternion column
__global__ void k_oe_rmax(const double* __restrict__ R, int64_t r, int64_t n, int64_t ldr, int* __restrict__ eb) {
  const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= n) return;
  double mx = 0.0;
  for (int64_t k = lane; k < r; k += 32) {
    const Quat q = ldq_nc(R + (k * ldr + j) * 4);
    mx = fmax(mx, fmax(fmax(fabs(q.w), fabs(q.x)), fmax(fabs(q.y), fabs(q.z))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) eb[j] = exp_for(mx);
}

// digits 1..6 of v (|v| <= 2^54) packed: byte s-1 of lo (s = 1..4), hi (s = 5, 6)
__device__ __forceinline__ void digits16(long long v, unsigned& lo, unsigned& hi) {
  const int d0 = (int)((v + 128) & 255) - 128;
  v = (v - d0) >> 8;
  lo = hi = 0u;
#pragma unroll
  for (int s = 1; s <= OE_DIG; ++s) {
    const int d = (int)((v + 128) & 255) - 128;
    v = (v - d) >> 8;
    if (s <= 4) lo |= ((unsigned)d & 0xffu) << (8 * (s - 1));
    else hi |= ((unsigned)d & 0xffu) << (8 * (s - 5));
  }
}

// digits of E(R') stored K-major: plane s-1, row 4j+t, byte 4k+s' = digit of sign(s',t) r'_kj[s'^t]
__global__ void k_oe_rdig(const double* __restrict__ R, int64_t r, int64_t n, int64_t ldr, const int* __restrict__ eb,
                          int8_t* __restrict__ dig, int64_t Kp) {
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= n * r) return;
  const int64_t j = id / r, k = id - j * r;
  const Quat q = ldq_nc(R + (k * ldr + j) * 4);
  const int e = eb[j];
  const double comp[4] = {q.w, q.x, q.y, q.z};
  unsigned plo[4], phi[4], nlo[4], nhi[4];  // digits of +v_u and -v_u
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const long long v = llrint(scale2(comp[u], e));
    digits16(v, plo[u], phi[u]);
    digits16(-v, nlo[u], nhi[u]);
  }
  // sign(s,t) of E: negative at (s,t) = (1,0) (2,0) (3,0) (3,1) (1,2) (2,3); u = s ^ t
  const int64_t plane = 4 * n * Kp;
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    unsigned w[OE_DIG];
#pragma unroll
    for (int d = 0; d < OE_DIG; ++d) w[d] = 0u;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int u = s ^ t;
      const bool neg = (t == 0 && s != 0) || (t == 1 && s == 3) || (t == 2 && s == 1) || (t == 3 && s == 2);
      const unsigned lo = neg ? nlo[u] : plo[u], hi = neg ? nhi[u] : phi[u];
#pragma unroll
      for (int d = 0; d < OE_DIG; ++d) {
        const unsigned byte = d < 4 ? (lo >> (8 * d)) & 0xffu : (hi >> (8 * (d - 4))) & 0xffu;
        w[d] |= byte << (8 * s);
      }
    }
#pragma unroll
    for (int d = 0; d < OE_DIG; ++d)
      *reinterpret_cast<unsigned*>(dig + d * plane + (4 * j + t) * Kp + 4 * k) = w[d];
  }
}

// ---------------------------------------------------------------------------
// the error GEMM
// ---------------------------------------------------------------------------
struct OeParams {
  int64_t m, N, ldx;  // N = 4n reals; X row pitch in doubles
  const double* X;
  const int* ea;
  const int* eb;
  double* partials;  // [grid][OE_EPI_WARPS][4]
  double psnr_scale;
  int kblocks, mblocks, nblocks, total;
  int groups;  // (row block, group of CL column blocks) work units of a cluster
  uint32_t idesc;
  int exp;  // timing experiments only (QCUR_OE_EXP): 1 = epilogue skips TMEM, 2 = and skips X / statistics
};

// CL CTAs per cluster work on one row block and CL adjacent column blocks: the A digit tile
// (6 planes x 128 rows x 32 bytes per k-block) is the same for all of them, so each CTA loads
// a share of its digit planes and multicasts it to the whole cluster (L2 -> SM traffic for A
// divided by CL); every CTA still loads its own B tile.  A stage may be refilled only when all
// CL CTAs have consumed it: the MMA warps commit to the stage's "empty" barrier of every CTA.
template <int CL>
__global__ void __launch_bounds__(OE_THREADS, 1)
    k_oe_err(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
             const __grid_constant__ CUtensorMap tmX, const __grid_constant__ OeParams P) {
  extern __shared__ uint8_t smem_raw[];
  const unsigned pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OE_STAGES * OE_STAGE);
  uint64_t* empty = full + OE_STAGES;
  uint64_t* tfull = empty + OE_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  const int cid = CL > 1 ? (int)cluster_id_x() : (int)blockIdx.x;
  const int ncl = CL > 1 ? (int)ncluster_x() : (int)gridDim.x;
  constexpr uint16_t kMask = (uint16_t)((1u << CL) - 1u);
  if (threadIdx.x == 0) {
    for (int s = 0; s < OE_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);  // one commit from each CTA of the cluster
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, OE_EPI_WARPS);
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
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      int stage = 0;
      unsigned phase = 0;
      for (int g = cid; g < P.groups; g += ncl) {
        const int mb = g % P.mblocks, nb = (g / P.mblocks) * CL + crank;  // row blocks fastest
        if (nb < P.nblocks) tma_prefetch_2d(&tmX, nb * OE_BN, mb * OE_BM);  // X tile for the epilogue
        for (int kb = 0; kb < P.kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          mbar_expect_tx(&full[stage], OE_STAGE);
          uint8_t* st = smem + stage * OE_STAGE;
          if constexpr (CL == 1) {
            tma_load_3d(st, &tmA, kb * OE_BK, mb * OE_BM, 0, &full[stage]);
          } else {
            // this CTA's share of the digit planes, into every CTA of the cluster
            for (int d = crank; d < OE_DIG; d += CL)
              tma_load_3d_mc(st + d * OE_BM * OE_BK, &tmA, kb * OE_BK, mb * OE_BM, d, &full[stage], kMask);
          }
          tma_load_3d(st + OE_A_BYTES, &tmB, kb * OE_BK, nb * OE_BN, 0, &full[stage]);
          if (++stage == OE_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    // the whole warp runs the issue loop (uniform control flow: descriptors and counters live in
    // uniform registers, no per-MMA lane election loops); one elected lane issues each k-block's
    // 21 MMAs and its commit
    const uint64_t adesc0 = umma_desc_sw64(smem_u32(smem));
    int stage = 0;
    unsigned phase = 0;
    int t = 0;
    for (int g = cid; g < P.groups; g += ncl, ++t) {
      mbar_wait(tempty, ((unsigned)t & 1u) ^ 1u);
      tc_fence_after();
      for (int kb = 0; kb < P.kblocks; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad0 = adesc0 + (uint64_t)((stage * OE_STAGE) >> 4);
        const uint64_t bd0 = ad0 + (uint64_t)(OE_A_BYTES >> 4);
        if (elect_one_sync()) {
          // A digit s is shared by its 7 - max(1, 7 - s) products: it is read from shared
          // memory once per K half (collector::a fill / use / lastuse)
#pragma unroll
          for (int kk = 0; kk < OE_BK / 32; ++kk) {
#pragma unroll
            for (int s = 1; s <= OE_DIG; ++s) {
              const int t0 = 7 - s > 1 ? 7 - s : 1;
#pragma unroll
              for (int tt = t0; tt <= OE_DIG; ++tt) {
                const int L = s + tt - 7;  // accumulator of level s + t
                const int first_s = L + 1 > 1 ? L + 1 : 1;
                const uint32_t d = tbase + (uint32_t)(L * OE_BN);
                const uint64_t ad = ad0 + (uint64_t)((((s - 1) * OE_BM * OE_BK) + kk * 32) >> 4);
                const uint64_t bd = bd0 + (uint64_t)((((tt - 1) * OE_BN * OE_BK) + kk * 32) >> 4);
                const uint32_t acc = (kb > 0 || kk > 0 || s != first_s) ? 1u : 0u;
                if (t0 == OE_DIG)
                  mma_i8(d, ad, bd, P.idesc, acc);
                else if (tt == t0)
                  mma_i8_coll<1>(d, ad, bd, P.idesc, acc);
                else if (tt == OE_DIG)
                  mma_i8_coll<3>(d, ad, bd, P.idesc, acc);
                else
                  mma_i8_coll<2>(d, ad, bd, P.idesc, acc);
              }
            }
          }
          if constexpr (CL == 1)
            mma_commit(&empty[stage]);
          else
            mma_commit_mc(&empty[stage], kMask);  // the stage is free in every CTA's ring
        }
        __syncwarp();
        if (++stage == OE_STAGES) {
          stage = 0;
          phase ^= 1u;
        }
      }
      if (elect_one_sync()) mma_commit(tfull);
      __syncwarp();
    }
  } else {
    // warp w drains TMEM lanes 32 (w % 4) .. +31, columns 20 s .. 20 s + 19 (s = (w - 2) / 4:
    // five quaternions).  Phase A reads the six level accumulators, folds them into the FP64
    // products and releases TMEM at once, so the next tile's MMAs overlap phase B (X and the
    // statistics).
    const int quarter = warp & 3, sub = (warp - 2) >> 2;
    const int rloc = quarter * 32 + lane;
    constexpr int QW = OE_BN / 4 / 4;  // quaternion columns per warp
    const double sc = P.psnr_scale;
    double v[4] = {0.0, 0.0, 0.0, 0.0};  // this thread's sums over all its units, in a fixed order
    int t = 0;
    for (int g = cid; g < P.groups; g += ncl, ++t) {
      const int mb = g % P.mblocks, nb = (g / P.mblocks) * CL + crank;
      const int64_t row = (int64_t)mb * OE_BM + rloc;
      const bool rvalid = row < P.m && nb < P.nblocks;
      const int er = rvalid ? P.ea[row] : 0;
      const double* xrow = P.X + (rvalid ? row : 0) * P.ldx;
      const int64_t jq0 = ((int64_t)nb * OE_BN + sub * 4 * QW) >> 2;  // first quaternion column
      double pr[QW][4];
      mbar_wait(tfull, (unsigned)t & 1u);
      tc_fence_after();
      if (P.exp) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);
        if (P.exp == 2) continue;
#pragma unroll
        for (int i = 0; i < QW; ++i)
#pragma unroll
          for (int h = 0; h < 4; ++h) pr[i][h] = 0.0;
      } else
#pragma unroll
      for (int i = 0; i < QW; ++i) {
        uint32_t lv[6][4];
        const uint32_t ta = tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(sub * 4 * QW + 4 * i);
#pragma unroll
        for (int L = 0; L < 6; ++L) tmem_ld4(ta + (uint32_t)(L * OE_BN), lv[L]);
        tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          double acc = i2d(lv[5][h]);
#pragma unroll
          for (int L = 4; L >= 0; --L) acc = fma(acc, 256.0, i2d(lv[L][h]));
          pr[i][h] = acc;
        }
      }
      if (!P.exp) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty);  // TMEM free: the next tile's MMAs start now
      }
      if (rvalid) {
#pragma unroll
        for (int i = 0; i < QW; ++i) {
          const int64_t jq = jq0 + i;
          if (4 * jq >= P.N) break;
          const double4 xq = *reinterpret_cast<const double4*>(xrow + 4 * jq);
          const double f = pow2(8 * 7 - er - P.eb[jq]);  // P R = (sum_L 256^L acc_L) 2^(56 - a_i - b_j)
          const double xs[4] = {xq.x, xq.y, xq.z, xq.w};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const double prh = pr[i][h] * f;
            const double x = xs[h], d = x - prh;
            v[0] = fma(d, d, v[0]);
            v[1] = fma(x, x, v[1]);
            if (h != 0) {
              v[2] = fma(d, d, v[2]);
              if (sc > 0.0) {
                const double q = rint(fmin(fmax(sc * x, 0.0), 255.0)) - rint(fmin(fmax(sc * prh, 0.0), 255.0));
                v[3] = fma(q, q, v[3]);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = warp_sum(v[k]);
    if (lane < 4) P.partials[((int64_t)blockIdx.x * OE_EPI_WARPS + (warp - 2)) * 4 + lane] = v[lane];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
  // no CTA may leave while a peer can still multicast into its shared memory or barriers
  if constexpr (CL > 1) cluster_sync_all();
}

// ---------------------------------------------------------------------------
// CTA-pair variant (tcgen05.mma.cta_group::2, M = 256): the two CTAs of a cluster compute a
// 256 x 80 tile; each loads its own 128 rows of the A digits and 40 of the 80 B rows, so a CTA's
// stage is 63 KB instead of 78 KB (three stages fit shared memory instead of two) and the
// MMA instruction count halves.  CTA 0 issues every MMA; the operand bytes of both CTAs complete
// on CTA 0's "full" barrier, MMA completions are committed to both CTAs' "empty" / "tfull"
// barriers, and both CTAs' epilogue warps release TMEM on CTA 0's "tempty" barrier.
// ---------------------------------------------------------------------------
constexpr int OE2_BNH = OE_BN / 2;  // B rows per CTA
constexpr int OE2_STAGES = 3;
constexpr int OE2_A_BYTES = OE_DIG * OE_BM * OE_BK;     // 48 KB
constexpr int OE2_B_BYTES = OE_DIG * OE2_BNH * OE_BK;   // 15 KB
constexpr int OE2_STAGE = OE2_A_BYTES + OE2_B_BYTES;
constexpr int OE2_SMEM = 1024 + OE2_STAGES * OE2_STAGE + 256;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(OE_THREADS, 1)
    k_oe_err_pair(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                  const __grid_constant__ CUtensorMap tmX, const __grid_constant__ OeParams P) {
  extern __shared__ uint8_t smem_raw[];
  const unsigned pad = (1024u - (smem_u32(smem_raw) & 1023u)) & 1023u;
  uint8_t* smem = smem_raw + pad;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OE2_STAGES * OE2_STAGE);
  uint64_t* empty = full + OE2_STAGES;
  uint64_t* tfull = empty + OE2_STAGES;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = (int)cluster_ctarank();
  const int cid = (int)cluster_id_x(), ncl = (int)ncluster_x();
  if (threadIdx.x == 0) {
    for (int s = 0; s < OE2_STAGES; ++s) {
      mbar_init(&full[s], 1);   // CTA 0's producer arrive (+ both CTAs' transaction bytes)
      mbar_init(&empty[s], 1);  // CTA 0's MMA commit, multicast to both CTAs
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * OE_EPI_WARPS);  // the epilogue warps of both CTAs (used in CTA 0)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {  // the same warp in both CTAs allocates the pair's TMEM
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
      int stage = 0;
      unsigned phase = 0;
      for (int g = cid; g < P.groups; g += ncl) {
        const int mb = g % P.mblocks, nb = g / P.mblocks;  // 256-row blocks fastest
        tma_prefetch_2d(&tmX, nb * OE_BN, mb * 2 * OE_BM + crank * OE_BM);
        for (int kb = 0; kb < P.kblocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1u);
          if (crank == 0) mbar_expect_tx(&full[stage], 2 * OE2_STAGE);
          uint8_t* st = smem + stage * OE2_STAGE;
          tma_load_3d_2sm(st, &tmA, kb * OE_BK, mb * 2 * OE_BM + crank * OE_BM, 0, &full[stage]);
          tma_load_3d_2sm(st + OE2_A_BYTES, &tmB, kb * OE_BK, nb * OE_BN + crank * OE2_BNH, 0, &full[stage]);
          if (++stage == OE2_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (crank == 0) {
      const uint64_t adesc0 = umma_desc_sw64(smem_u32(smem));
      int stage = 0;
      unsigned phase = 0;
      int t = 0;
      for (int g = cid; g < P.groups; g += ncl, ++t) {
        mbar_wait(tempty, ((unsigned)t & 1u) ^ 1u);
        tc_fence_after();
        for (int kb = 0; kb < P.kblocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad0 = adesc0 + (uint64_t)((stage * OE2_STAGE) >> 4);
          const uint64_t bd0 = ad0 + (uint64_t)(OE2_A_BYTES >> 4);
          if (elect_one_sync()) {
#pragma unroll
            for (int kk = 0; kk < OE_BK / 32; ++kk) {
#pragma unroll
              for (int s = 1; s <= OE_DIG; ++s) {
                const int t0 = 7 - s > 1 ? 7 - s : 1;
#pragma unroll
                for (int tt = t0; tt <= OE_DIG; ++tt) {
                  const int L = s + tt - 7;
                  const int first_s = L + 1 > 1 ? L + 1 : 1;
                  const uint32_t d = tbase + (uint32_t)(L * OE_BN);
                  const uint64_t ad = ad0 + (uint64_t)((((s - 1) * OE_BM * OE_BK) + kk * 32) >> 4);
                  const uint64_t bd = bd0 + (uint64_t)((((tt - 1) * OE2_BNH * OE_BK) + kk * 32) >> 4);
                  const uint32_t acc = (kb > 0 || kk > 0 || s != first_s) ? 1u : 0u;
                  if (t0 == OE_DIG)
                    mma_i8_2sm<0>(d, ad, bd, P.idesc, acc);
                  else if (tt == t0)
                    mma_i8_2sm<1>(d, ad, bd, P.idesc, acc);
                  else if (tt == OE_DIG)
                    mma_i8_2sm<3>(d, ad, bd, P.idesc, acc);
                  else
                    mma_i8_2sm<2>(d, ad, bd, P.idesc, acc);
                }
              }
            }
            mma_commit_2sm_mc(&empty[stage], 3);  // the stage is free in both CTAs
          }
          __syncwarp();
          if (++stage == OE2_STAGES) {
            stage = 0;
            phase ^= 1u;
          }
        }
        if (elect_one_sync()) mma_commit_2sm_mc(tfull, 3);
        __syncwarp();
      }
    }
  } else {
    const int quarter = warp & 3, sub = (warp - 2) >> 2;
    const int rloc = quarter * 32 + lane;
    constexpr int QW = OE_BN / 4 / 4;
    const double sc = P.psnr_scale;
    double v[4] = {0.0, 0.0, 0.0, 0.0};
    int t = 0;
    for (int g = cid; g < P.groups; g += ncl, ++t) {
      const int mb = g % P.mblocks, nb = g / P.mblocks;
      const int64_t row = (int64_t)mb * 2 * OE_BM + crank * OE_BM + rloc;
      const bool rvalid = row < P.m;
      const int er = rvalid ? P.ea[row] : 0;
      const double* xrow = P.X + (rvalid ? row : 0) * P.ldx;
      const int64_t jq0 = ((int64_t)nb * OE_BN + sub * 4 * QW) >> 2;
      double pr[QW][4];
      mbar_wait(tfull, (unsigned)t & 1u);
      tc_fence_after();
#pragma unroll
      for (int i = 0; i < QW; ++i) {
        uint32_t lv[6][4];
        const uint32_t ta = tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(sub * 4 * QW + 4 * i);
#pragma unroll
        for (int L = 0; L < 6; ++L) tmem_ld4(ta + (uint32_t)(L * OE_BN), lv[L]);
        tmem_wait_ld();
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          double acc = i2d(lv[5][h]);
#pragma unroll
          for (int L = 4; L >= 0; --L) acc = fma(acc, 256.0, i2d(lv[L][h]));
          pr[i][h] = acc;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {  // TMEM of this CTA drained: CTA 0's MMA warp may start the next tile
        if (crank == 0)
          mbar_arrive(tempty);
        else
          mbar_arrive_cluster(tempty, 0);
      }
      if (rvalid) {
#pragma unroll
        for (int i = 0; i < QW; ++i) {
          const int64_t jq = jq0 + i;
          if (4 * jq >= P.N) break;
          const double4 xq = *reinterpret_cast<const double4*>(xrow + 4 * jq);
          const double f = pow2(8 * 7 - er - P.eb[jq]);
          const double xs[4] = {xq.x, xq.y, xq.z, xq.w};
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const double prh = pr[i][h] * f;
            const double x = xs[h], d = x - prh;
            v[0] = fma(d, d, v[0]);
            v[1] = fma(x, x, v[1]);
            if (h != 0) {
              v[2] = fma(d, d, v[2]);
              if (sc > 0.0) {
                const double q = rint(fmin(fmax(sc * x, 0.0), 255.0)) - rint(fmin(fmax(sc * prh, 0.0), 255.0));
                v[3] = fma(q, q, v[3]);
              }
            }
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = warp_sum(v[k]);
    if (lane < 4) P.partials[((int64_t)blockIdx.x * OE_EPI_WARPS + (warp - 2)) * 4 + lane] = v[lane];
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs done: no barrier or TMEM of the pair is used any more
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
  }
}

PFN_cuTensorMapEncodeTiled_v12000 oe_encode() {
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

bool oe_digit_map(CUtensorMap* map, const int8_t* base, int64_t K, int64_t rows, int64_t Kp, int box_rows,
                  int box_digits = OE_DIG) {
  auto enc = oe_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)OE_DIG};
  cuuint64_t strides[2] = {(cuuint64_t)Kp, (cuuint64_t)(Kp * rows)};
  cuuint32_t box[3] = {(cuuint32_t)OE_BK, (cuuint32_t)box_rows, (cuuint32_t)box_digits};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<int8_t*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool oe_x_map(CUtensorMap* map, const double* X, int64_t N, int64_t m, int64_t ldx) {
  auto enc = oe_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)m};
  cuuint64_t strides[1] = {(cuuint64_t)(ldx * 8)};
  cuuint32_t box[2] = {(cuuint32_t)OE_BN, (cuuint32_t)OE_BM};
  cuuint32_t estr[2] = {1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(X), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct OePlan {
  int64_t K, Kp, N;
  int mblocks, nblocks, kblocks, total;
  size_t off_pd, off_rd, off_ea, off_eb, off_part, total_bytes;
};

OePlan oe_plan(int64_t m, int64_t n, int64_t r) {
  OePlan p{};
  p.K = 4 * r;
  p.Kp = (p.K + OE_BK - 1) / OE_BK * OE_BK;
  p.N = 4 * n;
  p.mblocks = (int)((m + OE_BM - 1) / OE_BM);
  p.nblocks = (int)((p.N + OE_BN - 1) / OE_BN);
  p.kblocks = (int)(p.Kp / OE_BK);
  p.total = p.mblocks * p.nblocks;
  auto al = [](size_t v) { return (v + 255) / 256 * 256; };
  size_t o = 0;
  p.off_pd = o;
  o = al(o + (size_t)OE_DIG * m * p.Kp);
  p.off_rd = o;
  o = al(o + (size_t)OE_DIG * p.N * p.Kp);
  p.off_ea = o;
  o = al(o + (size_t)m * 4);
  p.off_eb = o;
  o = al(o + (size_t)n * 4);
  p.off_part = o;
  o = al(o + (size_t)p.total * OE_EPI_WARPS * 4 * 8);
  p.total_bytes = o;
  return p;
}

int oe_sms() {
  static int sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n > 0 ? n : 148;
  }();
  return sms;
}

}  // namespace

bool ozaki_error_supported(int64_t m, int64_t n, int64_t r) {
  // int32 level sums: 6 * 2^14 * Kp < 2^31; grid / tensor-map extents
  const OePlan p = oe_plan(m, n, r);
  return m >= 1 && n >= 1 && r >= 1 && p.Kp <= 21824 && (int64_t)p.total * OE_EPI_WARPS < (1ll << 31) &&
         (double)p.total_bytes <= 8e9;  // workspace cap (else the FP64 engine)
}

size_t ozaki_error_workspace_bytes(int64_t m, int64_t n, int64_t r) { return oe_plan(m, n, r).total_bytes + 1024; }

// the digit planes of P and E(R) and their exponents
// the digit planes of E(R) and their exponents (R alone: may run as soon as R is gathered)
int launch_ozaki_error_rdigits(const double* R, int64_t ldr, int64_t m, int64_t n, int64_t r, void* workspace,
                               cudaStream_t st) {
  const OePlan pl = oe_plan(m, n, r);
  uint8_t* ws = reinterpret_cast<uint8_t*>(((uintptr_t)workspace + 255) / 256 * 256);
  int8_t* rd = reinterpret_cast<int8_t*>(ws + pl.off_rd);
  int* eb = reinterpret_cast<int*>(ws + pl.off_eb);
  ++::qcur::g_launches;
  k_oe_rmax<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(R, r, n, ldr, eb);
  ++::qcur::g_launches;
  k_oe_rdig<<<(unsigned)((n * r + 255) / 256), 256, 0, st>>>(R, r, n, ldr, eb, rd, pl.Kp);
  return 0;
}

// the digit planes of P (and of E(R) unless with_r == 0: formed earlier by launch_ozaki_error_rdigits)
int launch_ozaki_error_digits(const double* P, int64_t ldp, const double* R, int64_t ldr, int64_t m, int64_t n,
                              int64_t r, void* workspace, cudaStream_t st, int with_r) {
  const OePlan pl = oe_plan(m, n, r);
  uint8_t* ws = reinterpret_cast<uint8_t*>(((uintptr_t)workspace + 255) / 256 * 256);
  int8_t* pd = reinterpret_cast<int8_t*>(ws + pl.off_pd);
  int* ea = reinterpret_cast<int*>(ws + pl.off_ea);
  ++::qcur::g_launches;
  k_oe_pdig<<<(unsigned)((m + 7) / 8), 256, 0, st>>>(P, m, pl.K, ldp * 4, pd, pl.Kp, ea);
  if (with_r) return launch_ozaki_error_rdigits(R, ldr, m, n, r, workspace, st);
  return 0;
}

// the 21 digit GEMMs with the fused error epilogue, then the fixed-order reduction into out4
int launch_ozaki_error_gemm(const double* X, int64_t ldx, int64_t m, int64_t n, int64_t r, double psnr_scale,
                            void* workspace, double* out4, cudaStream_t st) {
  const OePlan pl = oe_plan(m, n, r);
  uint8_t* ws = reinterpret_cast<uint8_t*>(((uintptr_t)workspace + 255) / 256 * 256);
  int8_t* pd = reinterpret_cast<int8_t*>(ws + pl.off_pd);
  int8_t* rd = reinterpret_cast<int8_t*>(ws + pl.off_rd);
  int* ea = reinterpret_cast<int*>(ws + pl.off_ea);
  int* eb = reinterpret_cast<int*>(ws + pl.off_eb);
  double* parts = reinterpret_cast<double*>(ws + pl.off_part);

  // cluster size: CTAs of one row block sharing the A digit tile (QCUR_OE_CLUSTER overrides)
  static const int cl_env = [] {
    const char* e = std::getenv("QCUR_OE_CLUSTER");
    return e ? std::atoi(e) : 0;
  }();
  int CL = cl_env > 0 ? cl_env : kOeCluster;
  if (CL != 1 && CL != 2 && CL != 4) CL = kOeCluster;
  CUtensorMap tmA, tmB, tmX;
  if (!oe_digit_map(&tmA, pd, pl.K, m, pl.Kp, OE_BM, CL == 1 ? OE_DIG : 1) ||
      !oe_digit_map(&tmB, rd, pl.K, pl.N, pl.Kp, OE_BN) || !oe_x_map(&tmX, X, pl.N, m, ldx * 4))
    return 2;
  OeParams p{};
  p.m = m;
  p.N = pl.N;
  p.ldx = ldx * 4;
  p.X = X;
  p.ea = ea;
  p.eb = eb;
  p.partials = parts;
  p.psnr_scale = psnr_scale;
  p.kblocks = pl.kblocks;
  p.mblocks = pl.mblocks;
  p.nblocks = pl.nblocks;
  p.total = pl.total;
  p.groups = pl.mblocks * ((pl.nblocks + CL - 1) / CL);
  static const int exp_env = [] {
    const char* e = std::getenv("QCUR_OE_EXP");
    return e ? std::atoi(e) : 0;
  }();
  p.exp = exp_env;
  // kind::i8: D = s32, A/B signed int8, K-major, N = 80, M = 128
  p.idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OE_BN >> 3) << 17) | ((uint32_t)(OE_BM >> 4) << 24);
  static std::atomic<unsigned> attr{0};
  if (first_on_device(attr)) {
    cudaFuncSetAttribute(k_oe_err<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, OE_SMEM);
    cudaFuncSetAttribute(k_oe_err<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, OE_SMEM);
    cudaFuncSetAttribute(k_oe_err<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, OE_SMEM);
  }
  static const int pair_env = [] {
    const char* e = std::getenv("QCUR_OE_PAIR");
    return e ? std::atoi(e) : -1;
  }();
  if (pair_env == 1 || (pair_env < 0 && kOePairDefault)) {
    // CTA pairs: 256-row blocks x 80-column blocks; A maps of 128 rows, B maps of 40 rows
    CUtensorMap tmA2, tmB2;
    if (!oe_digit_map(&tmA2, pd, pl.K, m, pl.Kp, OE_BM) || !oe_digit_map(&tmB2, rd, pl.K, pl.N, pl.Kp, OE2_BNH))
      return 2;
    const int mb2 = (int)((m + 2 * OE_BM - 1) / (2 * OE_BM));
    p.mblocks = mb2;
    p.groups = mb2 * pl.nblocks;
    p.idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OE_BN >> 3) << 17) | ((uint32_t)((2 * OE_BM) >> 4) << 24);
    static std::atomic<unsigned> attr2{0};
    if (first_on_device(attr2))
      cudaFuncSetAttribute(k_oe_err_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, OE2_SMEM);
    static int max_pairs = 0;
    if (!max_pairs) {
      cudaLaunchConfig_t qc{};
      qc.gridDim = dim3((unsigned)(oe_sms() / 2 * 2));
      qc.blockDim = dim3(OE_THREADS);
      qc.dynamicSmemBytes = OE2_SMEM;
      int nc = 0;
      max_pairs = (cudaOccupancyMaxActiveClusters(&nc, k_oe_err_pair, &qc) == cudaSuccess && nc > 0) ? nc
                                                                                                     : oe_sms() / 2;
      (void)cudaGetLastError();
    }
    const int npairs = p.groups < max_pairs ? p.groups : max_pairs;
    const int grid = 2 * npairs;
    ++::qcur::g_launches;
    k_oe_err_pair<<<grid, OE_THREADS, OE2_SMEM, st>>>(tmA2, tmB2, tmX, p);
    launch_reduce_rows(parts, (int64_t)grid * OE_EPI_WARPS, 4, out4, st);
    return 0;
  }
  cudaLaunchConfig_t cfg{};
  cfg.blockDim = dim3(OE_THREADS);
  cfg.dynamicSmemBytes = OE_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // persistent grid: as many clusters as can be resident at once (clusters live inside one GPC,
  // so CL > 1 may leave a few SMs of a GPC idle), never a second wave
  int nclusters_max = oe_sms() / CL;
  if (CL > 1) {
    static int max_active[5] = {0, 0, 0, 0, 0};
    if (!max_active[CL]) {
      int nc = 0;
      cfg.gridDim = dim3((unsigned)(nclusters_max * CL));
      const cudaError_t e = CL == 2 ? cudaOccupancyMaxActiveClusters(&nc, k_oe_err<2>, &cfg)
                                    : cudaOccupancyMaxActiveClusters(&nc, k_oe_err<4>, &cfg);
      max_active[CL] = (e == cudaSuccess && nc > 0) ? nc : nclusters_max;
      (void)cudaGetLastError();
    }
    if (max_active[CL] < nclusters_max) nclusters_max = max_active[CL];
  }
  const int nclusters = p.groups < nclusters_max ? p.groups : nclusters_max;
  const int grid = nclusters * CL;
  ++::qcur::g_launches;
  if (CL == 1) {
    k_oe_err<1><<<grid, OE_THREADS, OE_SMEM, st>>>(tmA, tmB, tmX, p);
  } else {
    cfg.gridDim = dim3((unsigned)grid);
    const cudaError_t e = CL == 2 ? cudaLaunchKernelEx(&cfg, k_oe_err<2>, tmA, tmB, tmX, p)
                                  : cudaLaunchKernelEx(&cfg, k_oe_err<4>, tmA, tmB, tmX, p);
    if (e != cudaSuccess) return 3;
  }
  launch_reduce_rows(parts, (int64_t)grid * OE_EPI_WARPS, 4, out4, st);
  return 0;
}

// out4 = {||X - P R||^2, ||X||^2, imaginary part, u8-image sum}; P m x r, R r x n, X m x n (ld in quaternions)
int launch_ozaki_error(const double* X, int64_t ldx, const double* P, int64_t ldp, const double* R, int64_t ldr,
                       int64_t m, int64_t n, int64_t r, double psnr_scale, void* workspace, double* out4,
                       cudaStream_t st) {
  int rc = launch_ozaki_error_digits(P, ldp, R, ldr, m, n, r, workspace, st);
  return rc ? rc : launch_ozaki_error_gemm(X, ldx, m, n, r, psnr_scale, workspace, out4, st);
}

}  // namespace qcur
