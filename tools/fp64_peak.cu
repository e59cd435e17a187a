// FP64 peak microbenchmark for B200 (sm_100a): DFMA pipe, DMMA (mma.sync f64) and
// a 256-bit-load HBM read stream.  Prints one JSON line per test.  Used to
// measure the FP64 roofline denominator that MEASURED_PEAKS.json lacks.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double b, double c) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  double a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  double s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678) out[0] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters, double a, double b) {
  double c[16];
#pragma unroll
  for (int t = 0; t < 16; ++t) c[t] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      dmma(c[0], c[1], a, b); dmma(c[2], c[3], a, b); dmma(c[4], c[5], a, b); dmma(c[6], c[7], a, b);
      dmma(c[8], c[9], a, b); dmma(c[10], c[11], a, b); dmma(c[12], c[13], a, b); dmma(c[14], c[15], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 16; ++t) s += c[t];
  if (s == 12345.678) out[0] = s;
}

__global__ void read256_kernel(const double4* __restrict__ in, size_t n, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    double4 v;
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(in + i));
    acc += v.x + v.y + v.z + v.w;
  }
  if (acc == 12345.678) out[0] = acc;
}

int main(int argc, char** argv) {
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* out; CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  double secs = argc > 1 ? atof(argv[1]) : 0.5;  // target duration per timed run
  for (int blocks_per_sm : {2, 4, 8}) {
    int threads = 256, iters = 1000;
    dim3 grid(sms * blocks_per_sm);
    dfma_kernel<<<grid, threads>>>(out, 10, 1.0000001, 1e-9);
    CK(cudaEventRecord(e0)); dfma_kernel<<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    iters = (int)(iters * secs * 1e3 / ms) + 1;
    CK(cudaEventRecord(e0)); dfma_kernel<<<grid, threads>>>(out, iters, 1.0000001, 1e-9);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double flop = 2.0 * 64.0 * iters * (double)grid.x * threads;
    printf("{\"test\": \"dfma\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n", blocks_per_sm, ms,
           flop / ms / 1e9);
  }
  for (int warps_per_sm : {4, 8, 16}) {
    int threads = 128, iters = 1000;
    dim3 grid(sms * warps_per_sm / 4);
    dmma_kernel<<<grid, threads>>>(out, 10, 1.0, 1.0);
    CK(cudaEventRecord(e0)); dmma_kernel<<<grid, threads>>>(out, iters, 1.0, 1.0);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    iters = (int)(iters * secs * 1e3 / ms) + 1;
    CK(cudaEventRecord(e0)); dmma_kernel<<<grid, threads>>>(out, iters, 1.0, 1.0);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
    double flop = 2.0 * 256.0 * 64.0 * iters * (double)(grid.x * threads / 32);
    printf("{\"test\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"ms\": %.3f, \"tflops\": %.3f}\n", warps_per_sm, ms,
           flop / ms / 1e9);
  }
  {
    size_t bytes = (size_t)4 << 30;
    double4* buf; CK(cudaMalloc(&buf, bytes)); CK(cudaMemset(buf, 0, bytes));
    size_t n = bytes / sizeof(double4);
    for (int bps : {4, 8}) {
      float best = 1e30f;
      for (int rep = 0; rep < 5; ++rep) {
        CK(cudaEventRecord(e0)); read256_kernel<<<sms * bps, 512>>>(buf, n, out);
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < best) best = ms;
      }
      printf("{\"test\": \"read256\", \"blocks_per_sm\": %d, \"ms\": %.3f, \"gbs\": %.1f}\n", bps, best,
             bytes / best / 1e6);
    }
    CK(cudaFree(buf));
  }
  return 0;
}
