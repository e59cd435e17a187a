// Probe: 3-D TMA boxes of a byte tensor [L][rows][pitch] into static shared memory (16 x 16 x L),
// as the Hermitian CRT kernel stages its residue blocks.  Variant 0: one 3-D box; 1: L 2-D boxes.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include "../paper_2402_19147_b200/csrc/tc_ptx.cuh"
using namespace qcur::tc;
constexpr int L = 15;
__global__ void k_probe(const __grid_constant__ CUtensorMap tm, int variant, int x0, int y0, uint8_t* out, int bx) {
  __shared__ __align__(1024) uint8_t blk[L][16][32];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, L * 16 * bx);
    if (variant == 0)
      tma_load_3d(&blk[0][0][0], &tm, x0, y0, 0, &bar);
    else
      for (int l = 0; l < L; ++l) tma_load_3d(&blk[0][0][0] + l * 16 * bx, &tm, x0, y0, l, &bar);
  }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < L * 16 * bx; i += blockDim.x) out[i] = (&blk[0][0][0])[i];
}
int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int bx = argc > 2 ? atoi(argv[2]) : 16;
  const int swz = argc > 3 ? atoi(argv[3]) : 0;
  const int x0a = argc > 4 ? atoi(argv[4]) : 37;
  const int rows = 800, pitch = 832;
  uint8_t* d;
  cudaMalloc(&d, (size_t)L * rows * pitch);
  uint8_t* h = (uint8_t*)malloc((size_t)L * rows * pitch);
  for (size_t i = 0; i < (size_t)L * rows * pitch; ++i) h[i] = (uint8_t)(i * 2654435761u >> 24);
  cudaMemcpy(d, h, (size_t)L * rows * pitch, cudaMemcpyHostToDevice);
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  for (int variant = 0; variant < 2; ++variant) {
    if (only >= 0 && variant != only) continue;
    CUtensorMap tm;
    cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)rows, (cuuint64_t)L};
    cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)rows * pitch};
    cuuint32_t box[3] = {(cuuint32_t)bx, 16, variant == 0 ? (cuuint32_t)L : 1u};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     swz == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    uint8_t* o;
    cudaMalloc(&o, L * 512);
    k_probe<<<1, 256>>>(tm, variant, x0a, 211, o, bx);
    cudaError_t e = cudaDeviceSynchronize();
    uint8_t ho[L * 512];
    int bad = -1;
    if (e == cudaSuccess) {
      cudaMemcpy(ho, o, L * 16 * bx, cudaMemcpyDeviceToHost);
      bad = 0;
      for (int l = 0; l < L; ++l)
        for (int y = 0; y < 16; ++y)
          for (int x = 0; x < 16; ++x)
            bad += swz == 0 && ho[(l * 16 + y) * bx + x] != h[((size_t)l * rows + 211 + y) * pitch + x0a + x];
    }
    printf("variant %d bx %d swz %d encode %d launch %s mismatches %d\n", variant, bx, swz, (int)r, cudaGetErrorString(e), bad);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
