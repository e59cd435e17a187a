// Per-draw clock trace of k2_draw (debug aid, not part of the library): cfg2-sized axes (4000 weights,
// 200 draws), clocks of CTA 0 lane 0 at the loop top, after the descent, after the removal.
// nvcc -DQCUR_DRAW_TRACE -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr
//      tools/test_draw_trace.cu paper_2402_19147_b200/csrc/k_draw.cu -o tools/test_draw_trace
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2402_19147_b200/csrc/common.cuh"
#include "../paper_2402_19147_b200/csrc/kernels.h"
unsigned long long qcur::g_launches = 0;
namespace qcur { void draw_trace_read(long long* out); }
int main() {
  const int64_t len = 4000, count = 200;
  std::vector<double> p(len);
  srand(7);
  double s = 0;
  for (auto& v : p) { v = rand() / (double)RAND_MAX + 0.01; s += v; }
  for (auto& v : p) v /= s;
  double *dp, *w; int64_t* out; unsigned* st;
  cudaMalloc(&dp, len * 8); cudaMalloc(&w, qcur::draw_work_doubles(len) * 8); cudaMalloc(&out, count * 8);
  cudaMalloc(&st, 4); cudaMemset(st, 0, 4);
  cudaMemcpy(dp, p.data(), len * 8, cudaMemcpyHostToDevice);
  qcur::DrawJob j{dp, len, count, 1, 2, 3, 5, out, w};
  for (int rep = 0; rep < 3; ++rep) qcur::launch_draw(&j, 1, st, 0);
  cudaDeviceSynchronize();
  std::vector<long long> tr(1026 * 3);
  qcur::draw_trace_read(tr.data());
  auto T = [&](int t, int k) { return tr[t * 3 + k]; };
  printf("init to tree start %lld, tree build %lld, tree end to first draw %lld, draws total %lld cycles\n",
         T(1024, 1) - T(1024, 0), T(1024, 2) - T(1024, 1), T(0, 0) - T(1024, 2), T(1025, 0) - T(0, 0));
  double d = 0, r = 0, l = 0;
  for (int t = 1; t < count; ++t) { d += T(t, 1) - T(t, 0); r += T(t, 2) - T(t, 1); l += T(t, 0) - T(t - 1, 2); }
  printf("per draw: descent+proof %.0f, removal+store %.0f, loop gap %.0f cycles\n", d / (count - 1), r / (count - 1), l / (count - 1));
  return 0;
}
