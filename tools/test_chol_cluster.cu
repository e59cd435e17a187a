// Standalone harness for k_chol_inv_cluster (debug aid, not part of the library).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "../paper_2402_19147_b200/csrc/common.cuh"
#include "../paper_2402_19147_b200/csrc/kernels.h"
unsigned long long qcur::g_launches = 0;
#ifdef QCUR_CHOL_TRACE
namespace qcur { void chol_trace_read(long long* out); }
#endif
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)
struct Q { double w, x, y, z; };
static Q mul(Q a, Q b) { return {a.w*b.w-a.x*b.x-a.y*b.y-a.z*b.z, a.w*b.x+a.x*b.w+a.y*b.z-a.z*b.y, a.w*b.y-a.x*b.z+a.y*b.w+a.z*b.x, a.w*b.z+a.x*b.y-a.y*b.x+a.z*b.w}; }
static Q cj(Q a) { return {a.w, -a.x, -a.y, -a.z}; }
int main() {
  for (int q : {4, 17, 40, 200, 256, 300}) {
    int p = q + 30;
    std::vector<Q> Z(p * q), G(q * q);
    srand(q);
    for (auto& v : Z) v = {rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5};
    for (int i = 0; i < q; ++i) for (int j = 0; j < q; ++j) { Q s{0,0,0,0}; for (int k = 0; k < p; ++k) { Q t = mul(cj(Z[k*q+i]), Z[k*q+j]); s.w+=t.w; s.x+=t.x; s.y+=t.y; s.z+=t.z; } G[i*q+j] = s; }
    double *dG, *dL, *dX; unsigned* st;
    CK(cudaMalloc(&dG, q*q*32)); CK(cudaMalloc(&dL, q*q*32)); CK(cudaMalloc(&dX, q*q*32)); CK(cudaMalloc(&st, 4)); CK(cudaMemset(st, 0, 4));
    CK(cudaMemcpy(dG, G.data(), q*q*32, cudaMemcpyHostToDevice));
    qcur::CholJob jobs[2] = {{dG, dL, dX, 4u}, {dG, dL, dX, 8u}};
    qcur::launch_chol_inv_cluster(jobs, 1, q, st, 0);
    CK(cudaGetLastError()); CK(cudaDeviceSynchronize());
    std::vector<Q> L(q*q), X(q*q); unsigned hs;
    CK(cudaMemcpy(L.data(), dL, q*q*32, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(X.data(), dX, q*q*32, cudaMemcpyDeviceToHost)); CK(cudaMemcpy(&hs, st, 4, cudaMemcpyDeviceToHost));
    // X = L^{-1}  =>  X G X^H = I
    std::vector<Q> XG(q*q);
    for (int i = 0; i < q; ++i) for (int j = 0; j < q; ++j) { Q s{0,0,0,0}; for (int k = 0; k < q; ++k) { Q a = mul(X[i*q+k], G[k*q+j]); s.w+=a.w; s.x+=a.x; s.y+=a.y; s.z+=a.z; } XG[i*q+j] = s; }
    double e1 = 0, e2 = 0;
    for (int i = 0; i < q; ++i) for (int j = 0; j < q; ++j) {
      Q s{0,0,0,0}; for (int k = 0; k < q; ++k) { Q a = mul(XG[i*q+k], cj(X[j*q+k])); s.w+=a.w; s.x+=a.x; s.y+=a.y; s.z+=a.z; }
      e1 = fmax(e1, fabs(s.w-(i==j))+fabs(s.x)+fabs(s.y)+fabs(s.z));
      if (j > i) e2 = fmax(e2, fabs(X[i*q+j].w)+fabs(X[i*q+j].x)+fabs(X[i*q+j].y)+fabs(X[i*q+j].z));
    }
    double gn = 1.0;
    float ms; cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a); for (int r = 0; r < 10; ++r) qcur::launch_chol_inv_cluster(jobs, 2, q, st, 0); cudaEventRecord(b); CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
#ifdef QCUR_CHOL_TRACE
    {
      long long tr[512][6];
      qcur::chol_trace_read(&tr[0][0]);
      double acc[6] = {0};
      int steps = q - 1 < 511 ? q - 1 : 511;
      for (int j = 1; j < steps; ++j) {
        for (int k = 1; k < 6; ++k) acc[k] += (double)(tr[j][k] - tr[j][k - 1]);
        acc[0] += (double)(tr[j + 1][0] - tr[j][5]);
      }
      printf("q=%d per-step cycles: wait %.0f lookahead %.0f produce %.0f bulk %.0f diag+sync %.0f loop %.0f  total/step %.0f\n", q,
             acc[1] / steps, acc[2] / steps, acc[3] / steps, acc[4] / steps, acc[5] / steps, acc[0] / steps,
             (double)(tr[steps][5] - tr[1][0]) / (steps - 1));
    }
#endif
    printf("q=%d status=%u |XGX^H-I|=%.2e upper(X)=%.2e  time(2 problems)=%.1f us\n", q, hs, e1/gn, e2, ms*100);
  }
  return 0;
}
