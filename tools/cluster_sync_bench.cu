// Microbenchmark: latency of cluster.sync() and DSMEM round trips vs cluster size (debug aid).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
template <int CL>
__global__ void __cluster_dims__(CL, 1, 1) k_sync(int iters, double* out, int mode) {
  __shared__ double buf[64];
  cg::cluster_group cl = cg::this_cluster();
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (mode == 1 && threadIdx.x < 32) {
      double* r = cl.map_shared_rank(buf, (cl.block_rank() + 1) % CL);
      r[threadIdx.x] = i;
    }
    if (mode == 2) { __syncthreads(); continue; }
    cl.sync();
    acc += buf[threadIdx.x & 31];
  }
  if (acc == -1) out[0] = acc;
}
template <int CL>
void run(int threads, int mode) {
  cudaFuncSetAttribute(k_sync<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_sync<CL><<<CL, threads>>>(10, out, mode);
  int iters = 20000;
  cudaEventRecord(a); k_sync<CL><<<CL, threads>>>(iters, out, mode); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  printf("cluster=%2d threads=%4d mode=%d  %.3f us/iter  (%s)\n", CL, threads, mode, ms * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int t : {128, 512, 1024}) { run<2>(t, 0); run<4>(t, 0); run<8>(t, 0); run<16>(t, 0); }
  run<16>(512, 1); run<8>(512, 1); run<16>(512, 2);
}
