// L2 -> shared-memory throughput of TMA loads by box shape (all SMs, 4-stage ring, no compute):
// does a 32-byte inner box row (the INT8 error kernel's digit tiles) cost delivery rate against
// 64- or 128-byte rows?  Source: a 96 MB int8 buffer (L2-resident after the first pass).
// Build: make -C tools tma_probe
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2402_19147_b200/csrc/tc_ptx.cuh"
using namespace qcur::tc;

constexpr int STAGES = 4;

__global__ void __launch_bounds__(64, 1) k_tma(const __grid_constant__ CUtensorMap tm, int box_bytes, int iters, int nx,
                                               int ny, int nz, int bx, int by, int bz, int* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t full[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned phase = 0;
    int stage = 0;
    const int tiles_x = nx / bx, tiles_y = ny / by, tiles_z = nz / bz;
    const int ntiles = tiles_x * tiles_y * tiles_z;
    int t = blockIdx.x * 7;
    for (int s = 0; s < STAGES; ++s) {  // prologue
      mbar_expect_tx(&full[s], box_bytes);
      const int tt = (t++) % ntiles;
      tma_load_3d(sm + s * box_bytes, &tm, (tt % tiles_x) * bx, ((tt / tiles_x) % tiles_y) * by,
                  (tt / (tiles_x * tiles_y)) * bz, &full[s]);
    }
    for (int it = 0; it < iters; ++it) {
      mbar_wait(&full[stage], phase);
      mbar_expect_tx(&full[stage], box_bytes);
      const int tt = (t++) % ntiles;
      tma_load_3d(sm + stage * box_bytes, &tm, (tt % tiles_x) * bx, ((tt / tiles_x) % tiles_y) * by,
                  (tt / (tiles_x * tiles_y)) * bz, &full[stage]);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_wait(&full[stage], phase);
      if (++stage == STAGES) {
        stage = 0;
        phase ^= 1u;
      }
    }
    if (sm[5] == 123) *sink = 1;
  }
}

int main() {
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const size_t bytes = (size_t)96 << 20;
  uint8_t* buf;
  int* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 64);
  cudaMemset(buf, 1, bytes);
  struct Shape { int row_bytes, rows, planes; CUtensorMapSwizzle sw; const char* name; };
  const Shape shapes[] = {{32, 128, 6, CU_TENSOR_MAP_SWIZZLE_32B, "A digits 32Bx128x6"},
                          {32, 80, 6, CU_TENSOR_MAP_SWIZZLE_32B, "B digits 32Bx80x6"},
                          {64, 128, 3, CU_TENSOR_MAP_SWIZZLE_64B, "64Bx128x3"},
                          {128, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B, "128Bx128"},
                          {128, 192, 1, CU_TENSOR_MAP_SWIZZLE_128B, "128Bx192"},
                          {32, 128, 1, CU_TENSOR_MAP_SWIZZLE_32B, "32Bx128x1"}};
  for (const Shape& s : shapes) {
    // tensor: dim0 = K bytes (row pitch 800, like Kp at cfg2), dim1 = rows, dim2 = planes
    const int K = 800, rows = 4096;
    const int planes = (int)(bytes / ((size_t)K * rows));
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)planes};
    cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)K * rows};
    cuuint32_t box[3] = {(cuuint32_t)s.row_bytes, (cuuint32_t)s.rows, (cuuint32_t)s.planes};
    cuuint32_t es[3] = {1, 1, 1};
    CUtensorMap tm;
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     s.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int box_bytes = s.row_bytes * s.rows * s.planes;
    const int smem = STAGES * box_bytes + 1024;
    cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 4000;
    k_tma<<<148, 64, smem>>>(tm, box_bytes, 200, K, rows, planes, s.row_bytes, s.rows, s.planes, sink);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_tma<<<148, 64, smem>>>(tm, box_bytes, iters, K, rows, planes, s.row_bytes, s.rows, s.planes, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double tot = (double)box_bytes * (iters + STAGES) * 148;
    printf("{\"shape\": \"%s\", \"box_bytes\": %d, \"encode\": %d, \"TBps\": %.2f, \"B_per_clk_per_SM_at_1965\": %.1f, \"err\": \"%s\"}\n",
           s.name, box_bytes, (int)r, tot / (ms * 1e-3) / 1e12, tot / (ms * 1e-3) / 148 / 1.965e9,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
