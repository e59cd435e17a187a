// Achievable tcgen05.mma kind::i8 rate (cta_group::1, M = 128, K = 32 per MMA, operands in shared
// memory) for the N and operand pattern of the error kernel (k_ozaki_err.cu): back-to-back MMAs
// into 6 accumulators of N columns, 21 per "k-block" as (A digit s, B digit t) with s + t >= 7.
// Prints TOP/s per configuration.  Build: make -C tools i8_shape_probe
#include <cstdio>
#include <cstdint>
#include "../paper_2402_19147_b200/csrc/tc_ptx.cuh"
using namespace qcur::tc;

template <int N, int PATTERN>  // PATTERN 0: 21-MMA digit pattern, sw32 operands; 1: plain sw128 N x K128
__global__ void __launch_bounds__(128, 1) probe(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* tiles = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t done;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < (6 * 128 * 32 + 6 * 256 * 32) / 4; i += blockDim.x) reinterpret_cast<int*>(tiles)[i] = 0x01010101;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (warp == 0) {
    const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
    const uint64_t ad0 = umma_desc_sw32(smem_u32(tiles)), bd0 = umma_desc_sw32(smem_u32(tiles + 6 * 128 * 32));
    for (int it = 0; it < iters; ++it) {
      if (elect_one_sync()) {
#pragma unroll
        for (int s = 1; s <= 6; ++s) {
          const int t0 = 7 - s > 1 ? 7 - s : 1;
#pragma unroll
          for (int t = t0; t <= 6; ++t) {
            const int L = s + t - 7;
            const uint32_t d = tb + (uint32_t)(N <= 80 ? L * N : (N == 128 ? (L % 4) * 128 : (L & 1) * 256));
            const uint64_t ad = ad0 + (uint64_t)(((s - 1) * 128 * 32) >> 4);
            const uint64_t bd = bd0 + (uint64_t)(((t - 1) * N * 32) >> 4);
            if (PATTERN == 0) {
              if (t0 == 6) mma_i8(d, ad, bd, idesc, 1u);
              else if (t == t0) mma_i8_coll<1>(d, ad, bd, idesc, 1u);
              else if (t == 6) mma_i8_coll<3>(d, ad, bd, idesc, 1u);
              else mma_i8_coll<2>(d, ad, bd, idesc, 1u);
            } else {
              mma_i8(d, ad, bd, idesc, 1u);
            }
          }
        }
      }
      __syncwarp();
    }
    if (elect_one_sync()) mma_commit(&done);
    __syncwarp();
    mbar_wait(&done, 0);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    uint32_t v[32];
    tmem_ld32(tb, v);
    if (threadIdx.x == 0 && v[0] == 0x7fffffffu) *sink = 1;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
  }
}

template <int N, int PATTERN>
void run(const char* name) {
  int* sink;
  cudaMalloc(&sink, 64);
  const int smem = 1024 + 6 * 128 * 32 + 6 * 256 * 32;
  cudaFuncSetAttribute(probe<N, PATTERN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int iters = 2000;
  probe<N, PATTERN><<<148, 128, smem>>>(100, sink);
  float ms = 0;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    probe<N, PATTERN><<<148, 128, smem>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < 30.f) iters = (int)(iters * 60.f / (ms > 0.01f ? ms : 0.01f)); else break;
  }
  const double ops = 2.0 * 128.0 * N * 32.0 * 21.0 * iters * 148.0;
  printf("{\"probe\": \"%s\", \"N\": %d, \"TOPs\": %.1f, \"ms\": %.2f, \"err\": \"%s\"}\n", name, N, ops / (ms * 1e-3) / 1e12, ms,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(sink);
}

int main() {
  run<80, 0>("digit21_collector");
  run<80, 1>("digit21_plain");
  run<64, 0>("digit21_collector");
  run<128, 1>("21mma_plain_N128_shared_acc");
  run<256, 1>("21mma_plain_N256_shared_acc");
  return 0;
}
