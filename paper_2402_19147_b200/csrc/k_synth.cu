// Synthetic workloads for the BASELINE configs, generated on the device.
//
// BASELINE.json configs are "rank-k product of Gaussian quaternion factors
// plus Gaussian noise".  Factors and noise are drawn with a counter-based
// Philox4x32-10 generator (keyed by seed, addressed by (stream, element)), so
// any element or row block is reproducible independently of launch shape; the
// product S = P Q^H runs on the DMMA quaternion GEMM.  The host never
// generates the large matrices (cfg5 is 34 GB).  Also hosts the FP64 DMMA
// peak probe used as the roofline denominator (MEASURED_PEAKS.json has none).
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace qcur {

__host__ __device__ inline void philox4x32_10(uint32_t ctr[4], uint32_t k0, uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)M0 * ctr[0];
    const uint64_t p1 = (uint64_t)M1 * ctr[2];
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    const uint32_t n0 = hi1 ^ ctr[1] ^ k0, n1 = lo1, n2 = hi0 ^ ctr[3] ^ k1, n3 = lo0;
    ctr[0] = n0;
    ctr[1] = n1;
    ctr[2] = n2;
    ctr[3] = n3;
    k0 += W0;
    k1 += W1;
  }
}

// Two standard normals for counter `idx` of `stream` (Box-Muller on 53-bit uniforms).
__device__ inline void normal_pair(uint64_t seed, uint64_t stream, uint64_t idx, double& z0, double& z1) {
  uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), (uint32_t)stream, (uint32_t)(stream >> 32)};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  const uint64_t a = ((uint64_t)c[0] << 21) ^ (uint64_t)c[1];
  const uint64_t b = ((uint64_t)c[2] << 21) ^ (uint64_t)c[3];
  const double u1 = ((double)(a & ((1ull << 53) - 1)) + 1.0) * (1.0 / 9007199254740992.0);  // (0, 1]
  const double u2 = (double)(b & ((1ull << 53) - 1)) * (1.0 / 9007199254740992.0);          // [0, 1)
  const double rad = sqrt(-2.0 * log(u1));
  double s, co;
  sincospi(2.0 * u2, &s, &co);
  z0 = rad * co;
  z1 = rad * s;
}

// `pair0` = first Philox counter (element offset / 2): any row block of a larger
// matrix draws exactly the values the whole-matrix generation would.
__global__ void k_normal_fill(double* __restrict__ out, int64_t count, uint64_t seed, uint64_t stream, double scale,
                              uint64_t pair0) {
  const int64_t pairs = (count + 1) / 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < pairs; t += (int64_t)gridDim.x * blockDim.x) {
    double z0, z1;
    normal_pair(seed, stream, pair0 + (uint64_t)t, z0, z1);
    out[2 * t] = scale * z0;
    if (2 * t + 1 < count) out[2 * t + 1] = scale * z1;
  }
}

// X += sigma * z, sigma = rel * sqrt(ssq / total) if ssq else rel (absolute std)
__global__ void k_add_noise(double* __restrict__ X, int64_t count, uint64_t seed, uint64_t stream,
                            const double* __restrict__ ssq, double rel, uint64_t pair0, double total) {
  const double sigma = ssq ? rel * sqrt(*ssq / total) : rel;
  const int64_t pairs = (count + 1) / 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < pairs; t += (int64_t)gridDim.x * blockDim.x) {
    double z0, z1;
    normal_pair(seed, stream, pair0 + (uint64_t)t, z0, z1);
    X[2 * t] += sigma * z0;
    if (2 * t + 1 < count) X[2 * t + 1] += sigma * z1;
  }
}

__global__ void k_sumsq_parts(const double* __restrict__ X, int64_t count, double* __restrict__ parts) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    s += X[t] * X[t];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r += sh[w];
    parts[2 * blockIdx.x] = r;
    parts[2 * blockIdx.x + 1] = 0.0;
  }
}

void launch_normal_fill(double* out, int64_t count, uint64_t seed, uint64_t stream, double scale, cudaStream_t st,
                        int64_t offset) {
  ++::qcur::g_launches;
  k_normal_fill<<<148 * 8, 256, 0, st>>>(out, count, seed, stream, scale, (uint64_t)(offset / 2));
}
void launch_add_scaled_noise(double* X, int64_t count, uint64_t seed, uint64_t stream, const double* ssq, double rel,
                             cudaStream_t st, int64_t offset, int64_t total) {
  ++::qcur::g_launches;
  k_add_noise<<<148 * 8, 256, 0, st>>>(X, count, seed, stream, ssq, rel, (uint64_t)(offset / 2),
                                       (double)(total > 0 ? total : count));
}
void launch_sumsq(const double* X, int64_t count, double* partials, int64_t nparts, double* out, cudaStream_t st) {
  ++::qcur::g_launches;
  k_sumsq_parts<<<(unsigned)nparts, 256, 0, st>>>(X, count, partials);
  launch_reduce_pairs(partials, nparts, out, st);
}

// ---------------------------------------------------------------------------
// cfg3: synthetic colour-image-like pure quaternion matrix (BASELINE.json
// configs[2]).  Plane p in {i, j, k} = sum_{l < L} f_{p,l}(y) g_{p,l}(x) with
// random cosine series f(y) = sum_{t<3} a_t cos(2 pi w_t y / H + phi_t),
// a_t ~ N(0,1)/(t+1), w_t ~ U[0, 8], phi_t ~ U[0, 2 pi) (same for g over x),
// min-max mapped to [0, 1], quantised to multiples of 1/255, plus N(0, noise^2).
// The real part is zero.  All randomness is Philox (seed, stream, counter).
// ---------------------------------------------------------------------------
constexpr int kImgTerms = 3;

__device__ inline void uniform_pair(uint64_t seed, uint64_t stream, uint64_t idx, double& u0, double& u1) {
  uint32_t c[4] = {(uint32_t)idx, (uint32_t)(idx >> 32), (uint32_t)stream, (uint32_t)(stream >> 32)};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  u0 = (double)((((uint64_t)c[0] << 21) ^ c[1]) & ((1ull << 53) - 1)) * (1.0 / 9007199254740992.0);
  u1 = (double)((((uint64_t)c[2] << 21) ^ c[3]) & ((1ull << 53) - 1)) * (1.0 / 9007199254740992.0);
}

// F[(p * L + l) * 2 + side][pos]: side 0 = f over rows (len m), side 1 = g over columns (len n)
__global__ void k_img_series(double* __restrict__ F, int64_t m, int64_t n, int L, uint64_t seed) {
  const int64_t maxlen = m > n ? m : n;
  const int64_t total = 3LL * L * 2 * maxlen;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t fn = t / maxlen, pos = t - fn * maxlen;
    const int side = (int)(fn & 1);
    const int64_t len = side ? n : m;
    if (pos >= len) continue;
    double v = 0.0;
    for (int k = 0; k < kImgTerms; ++k) {
      double z0, z1, u0, u1;
      normal_pair(seed, 100, (uint64_t)(fn * kImgTerms + k), z0, z1);
      uniform_pair(seed, 101, (uint64_t)(fn * kImgTerms + k), u0, u1);
      const double amp = z0 / (double)(k + 1), w = 8.0 * u0, phi = 2.0 * u1;  // phase in units of pi
      v += amp * cospi(2.0 * w * (double)pos / (double)len + phi);
    }
    F[fn * maxlen + pos] = v;
  }
}

// X(i, j) = (0, V_1, V_2, V_3), V_p = sum_l f_{p,l}(i) g_{p,l}(j)
__global__ void k_img_compose(const double* __restrict__ F, int64_t m, int64_t n, int L, double* __restrict__ X) {
  const int64_t maxlen = m > n ? m : n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m * n; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / n, j = t - i * n;
    double v[3];
    for (int p = 0; p < 3; ++p) {
      double s = 0.0;
      for (int l = 0; l < L; ++l) {
        const int64_t fn = (int64_t)(p * L + l) * 2;
        s += F[fn * maxlen + i] * F[(fn + 1) * maxlen + j];
      }
      v[p] = s;
    }
    stq(X + t * 4, Quat{0.0, v[0], v[1], v[2]});
  }
}

// per-block min / max of the three imaginary planes -> part[block][6]
__global__ void k_img_minmax(const double* __restrict__ X, int64_t count, double* __restrict__ part) {
  __shared__ double sh[6][256];
  double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x)
    for (int p = 0; p < 3; ++p) {
      const double v = X[t * 4 + 1 + p];
      mn[p] = fmin(mn[p], v);
      mx[p] = fmax(mx[p], v);
    }
  for (int p = 0; p < 3; ++p) {
    sh[p][threadIdx.x] = mn[p];
    sh[3 + p][threadIdx.x] = mx[p];
  }
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s)
      for (int p = 0; p < 3; ++p) {
        sh[p][threadIdx.x] = fmin(sh[p][threadIdx.x], sh[p][threadIdx.x + s]);
        sh[3 + p][threadIdx.x] = fmax(sh[3 + p][threadIdx.x], sh[3 + p][threadIdx.x + s]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 6) part[blockIdx.x * 6 + threadIdx.x] = sh[threadIdx.x][0];
}

// v <- rint(255 (v - min) / (max - min)) / 255 + noise N(0, sigma^2)
__global__ void k_img_finish(double* __restrict__ X, int64_t count, const double* __restrict__ part, int nparts,
                             uint64_t seed, double sigma) {
  double mn[3], mx[3];
  for (int p = 0; p < 3; ++p) {
    mn[p] = INFINITY;
    mx[p] = -INFINITY;
    for (int b = 0; b < nparts; ++b) {
      mn[p] = fmin(mn[p], part[b * 6 + p]);
      mx[p] = fmax(mx[p], part[b * 6 + 3 + p]);
    }
  }
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count; t += (int64_t)gridDim.x * blockDim.x) {
    double z[4];
    normal_pair(seed, 102, (uint64_t)(2 * t), z[0], z[1]);
    normal_pair(seed, 102, (uint64_t)(2 * t + 1), z[2], z[3]);
    for (int p = 0; p < 3; ++p) {
      const double span = mx[p] > mn[p] ? mx[p] - mn[p] : 1.0;
      const double v = (X[t * 4 + 1 + p] - mn[p]) / span;
      X[t * 4 + 1 + p] = rint(255.0 * v) / 255.0 + sigma * z[p];
    }
  }
}

void launch_synth_image(int64_t m, int64_t n, int L, uint64_t seed, double sigma, double* F, double* part,
                        double* X, cudaStream_t st) {
  const int nparts = 296;
  ++::qcur::g_launches;
  k_img_series<<<148 * 8, 256, 0, st>>>(F, m, n, L, seed);
  ++::qcur::g_launches;
  k_img_compose<<<148 * 8, 256, 0, st>>>(F, m, n, L, X);
  ++::qcur::g_launches;
  k_img_minmax<<<nparts, 256, 0, st>>>(X, m * n, part);
  ++::qcur::g_launches;
  k_img_finish<<<148 * 8, 256, 0, st>>>(X, m * n, part, nparts, seed, sigma);
}

// ---------------------------------------------------------------------------
// FP64 DMMA peak probe (same instruction mix as the GEMM inner loop)
// ---------------------------------------------------------------------------
__global__ void k_dmma_probe(double* out, int iters) {
  double c[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) c[t] = 0.0;
  const double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[2 * q]), "+d"(c[2 * q + 1])
                     : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 16; ++t) s += c[t];
  if (s == 1234.5) out[0] = s;
}

double run_dmma_peak(int sms, cudaStream_t st) {
  double* out = nullptr;
  if (cudaMalloc(&out, 64) != cudaSuccess) return 0.0;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 2;
  int iters = 200;
  ++::qcur::g_launches;
  k_dmma_probe<<<blocks, threads, 0, st>>>(out, 20);
  float ms = 0.f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0, st);
    ++::qcur::g_launches;
    k_dmma_probe<<<blocks, threads, 0, st>>>(out, iters);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < 20.f) iters = (int)(iters * (40.f / (ms > 0.01f ? ms : 0.01f)));
    else break;
  }
  const double flop = 2.0 * 256.0 * 64.0 * (double)iters * (double)blocks * (threads / 32);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return flop / ((double)ms * 1e-3) / 1e12;
}

}  // namespace qcur
