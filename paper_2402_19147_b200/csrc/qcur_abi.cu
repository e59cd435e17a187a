// C-ABI implementation and host orchestration of the QMCUR device pipeline.
// See include/qcur_b200.h for the contract of every entry point and the
// reference function it replaces.
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/qcur_b200.h"
#include "common.cuh"
#include "kernels.h"
#include "pairwise.h"
#include "pcg64.h"

using namespace qcur;

namespace {

constexpr double kEps = 2.220446049250313e-16;

struct DevProgram {
  DevPairwise d{};
  void* buf = nullptr;
  int64_t scratch_len = 0;  // doubles per segment for the top tree
};

// bump allocator over one device block; reset per API call
struct Arena {
  char* base = nullptr;
  size_t cap = 0, used = 0;
  void* take(size_t bytes) {
    size_t off = (used + 255) & ~(size_t)255;
    if (off + bytes > cap) return nullptr;
    used = off + bytes;
    return base + off;
  }
};

}  // namespace

struct qcur_ctx {
  int device = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  unsigned* status_dev = nullptr;
  unsigned* status_host = nullptr;  // pinned
  unsigned last_info = 0;
  double kappa_limit = 1e7;
  bool force_robust = false;
  Arena arena;
  std::map<int64_t, DevProgram> programs;
  std::string err;

  int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    err = buf;
    return code;
  }
  int cuda_fail(cudaError_t e, const char* where) {
    return fail(QCUR_E_CUDA, "CUDA error in %s: %s", where, cudaGetErrorString(e));
  }
  // Grow the workspace to hold `bytes`; invalidates earlier arena pointers.
  int reserve(size_t bytes) {
    arena.used = 0;
    if (arena.cap >= bytes) return QCUR_OK;
    cudaError_t e = cudaStreamSynchronize(stream);
    if (e != cudaSuccess) return cuda_fail(e, "reserve/sync");
    if (arena.base) cudaFree(arena.base);
    arena.base = nullptr;
    arena.cap = 0;
    size_t want = bytes + bytes / 4 + (64u << 20);
    e = cudaMalloc((void**)&arena.base, want);
    if (e != cudaSuccess) return cuda_fail(e, "workspace cudaMalloc");
    arena.cap = want;
    return QCUR_OK;
  }
  template <class T>
  T* take(size_t count) {
    return (T*)arena.take(count * sizeof(T));
  }
  const DevProgram* program(int64_t length);
};

const DevProgram* qcur_ctx::program(int64_t length) {
  auto it = programs.find(length);
  if (it != programs.end()) return &it->second;
  PairwiseProgram pp = compile_pairwise(length);
  std::vector<int32_t> plan_len, leaf_ptr{0}, prog_ptr{0}, leaf_off, leaf_len, prog;
  int32_t maxc = 0;
  for (const ChunkPlan& cp : pp.plans) {
    plan_len.push_back(cp.len);
    maxc = cp.len > maxc ? cp.len : maxc;
    leaf_off.insert(leaf_off.end(), cp.leaf_off.begin(), cp.leaf_off.end());
    leaf_len.insert(leaf_len.end(), cp.leaf_len.begin(), cp.leaf_len.end());
    prog.insert(prog.end(), cp.prog.begin(), cp.prog.end());
    leaf_ptr.push_back((int32_t)leaf_off.size());
    prog_ptr.push_back((int32_t)prog.size());
  }
  // pack: int64 chunk_off first, then the int32 arrays
  std::vector<const std::vector<int32_t>*> arrs = {&pp.chunk_plan, &plan_len, &leaf_ptr, &prog_ptr, &leaf_off,
                                                   &leaf_len,      &prog,     &pp.node_l, &pp.node_r, &pp.level_ptr};
  size_t bytes = pp.chunk_off.size() * 8;
  std::vector<size_t> offs;
  for (auto* a : arrs) {
    bytes = (bytes + 15) & ~(size_t)15;
    offs.push_back(bytes);
    bytes += a->size() * 4 + 4;
  }
  std::vector<char> host(bytes, 0);
  memcpy(host.data(), pp.chunk_off.data(), pp.chunk_off.size() * 8);
  for (size_t k = 0; k < arrs.size(); ++k)
    if (!arrs[k]->empty()) memcpy(host.data() + offs[k], arrs[k]->data(), arrs[k]->size() * 4);
  DevProgram dp;
  if (cudaMalloc(&dp.buf, bytes) != cudaSuccess) return nullptr;
  cudaMemcpy(dp.buf, host.data(), bytes, cudaMemcpyHostToDevice);
  char* b = (char*)dp.buf;
  dp.d.length = length;
  dp.d.nchunks = (int32_t)pp.chunk_off.size();
  dp.d.nnodes = (int32_t)pp.node_l.size();
  dp.d.maxh = (int32_t)pp.level_ptr.size() - 2;
  if (dp.d.nnodes == 0) dp.d.maxh = 0;
  dp.d.max_chunk_len = maxc;
  dp.d.chunk_off = (const int64_t*)b;
  const int32_t** dst[] = {&dp.d.chunk_plan, &dp.d.plan_len, &dp.d.plan_leaf_ptr, &dp.d.plan_prog_ptr,
                           &dp.d.leaf_off,   &dp.d.leaf_len, &dp.d.prog,          &dp.d.node_l,
                           &dp.d.node_r,     &dp.d.level_ptr};
  for (size_t k = 0; k < arrs.size(); ++k) *dst[k] = (const int32_t*)(b + offs[k]);
  dp.scratch_len = (int64_t)dp.d.nchunks + dp.d.nnodes;
  return &(programs[length] = dp);
}

namespace {

inline int64_t qbytes(int64_t rows, int64_t cols) { return rows * cols * 4 * (int64_t)sizeof(double); }

#define CK_LAUNCH(ctx, where)                                   \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return (ctx)->cuda_fail(_e, where);  \
  } while (0)

// pairwise sums of nseg segments (each `length` doubles, stride `stride`) -> out[nseg]
int pairwise_sum(qcur_ctx* ctx, const double* data, int64_t nseg, int64_t stride, int64_t length, double* out) {
  const DevProgram* dp = ctx->program(length);
  if (!dp) return ctx->fail(QCUR_E_CUDA, "pairwise program allocation failed");
  double* scratch = nullptr;
  if (dp->d.nnodes > 0) {
    scratch = ctx->take<double>((size_t)(nseg * dp->scratch_len));
    if (!scratch) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (pairwise)");
  }
  launch_pairwise(data, nseg, stride, dp->d, scratch, out, ctx->stream);
  CK_LAUNCH(ctx, "pairwise");
  return QCUR_OK;
}

size_t pairwise_scratch_bytes(qcur_ctx* ctx, int64_t nseg, int64_t length) {
  const DevProgram* dp = ctx->program(length);
  return dp ? (size_t)(nseg * dp->scratch_len) * 8 + 256 : 0;
}

size_t length_ws_bytes(qcur_ctx* ctx, int64_t m, int64_t n) {
  size_t b = (size_t)(m * n) * 8 + 256;                  // sq
  b += (size_t)(n + m) * 8 * 2 + 2048;                   // colsum, rowsum, scaled copies, scalars
  b += pairwise_scratch_bytes(ctx, m, n);                // row trees
  b += pairwise_scratch_bytes(ctx, 1, m * n);            // flat tree
  b += pairwise_scratch_bytes(ctx, 1, n) + pairwise_scratch_bytes(ctx, 1, m);
  return b;
}

// length_distributions on the device (cur.py:132-150); arena must be reserved.
int length_distributions_impl(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, double* col, double* row) {
  cudaStream_t st = ctx->stream;
  double* sq = ctx->take<double>((size_t)(m * n));
  double* colsum = ctx->take<double>((size_t)n);
  double* rowsum = ctx->take<double>((size_t)m);
  double* scal = ctx->take<double>(8);  // total, colnorm, rownorm
  if (!sq || !colsum || !rowsum || !scal) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (length)");
  launch_colstrip(X, m, n, n, sq, colsum, st);
  CK_LAUNCH(ctx, "colstrip");
  int rc;
  if ((rc = pairwise_sum(ctx, sq, m, n, n, rowsum)) != QCUR_OK) return rc;
  if ((rc = pairwise_sum(ctx, sq, 1, 0, m * n, scal)) != QCUR_OK) return rc;
  // col = colsum / total ; row = rowsum / total   (cur.py:147-148); total <= 0 -> degenerate
  launch_scale(colsum, n, scal, col, ctx->status_dev, ST_DEGENERATE, st);
  launch_scale(rowsum, m, scal, row, ctx->status_dev, 0, st);
  // col / col.sum(), row / row.sum()   (cur.py:150)
  if ((rc = pairwise_sum(ctx, col, 1, 0, n, scal + 1)) != QCUR_OK) return rc;
  if ((rc = pairwise_sum(ctx, row, 1, 0, m, scal + 2)) != QCUR_OK) return rc;
  launch_scale(col, n, scal + 1, col, ctx->status_dev, 0, st);
  launch_scale(row, m, scal + 2, row, ctx->status_dev, 0, st);
  CK_LAUNCH(ctx, "length scale");
  return QCUR_OK;
}

// ---------------------------------------------------------------------------
// pinv factorization of a tall p x q block Z (p >= q):  pinv(Z) = F Q^H.
// Z is given as `src` with `zh`: 0 -> Z = src (p x q, row-major),
//                                1 -> Z = src^H where src is q x p row-major.
// ---------------------------------------------------------------------------
struct FactorOut {
  double* Q;  // p x q
  double* F;  // q x q
};

size_t factor_ws_bytes(int64_t p, int64_t q) {
  size_t b = 0;
  b += qbytes(p, q) * 3;        // Q1, Zcm, Qcm
  b += qbytes(q, q) * 10;       // G1, L1inv, G2, L2inv, T, Tcm, Vcm, ...
  b += (size_t)(q + 8) * 8 * 4;  // betas, sigma
  GemmArgs g{};
  g.Mq = p;
  g.Nq = q;
  g.Kq = q;
  size_t w1 = qgemm_workspace_bytes(g);
  g.Mq = q;
  g.Nq = q;
  g.Kq = p;
  size_t w2 = qgemm_workspace_bytes(g);
  b += (w1 > w2 ? w1 : w2) + 4096;
  return b + 16 * 256;
}

int gemm(qcur_ctx* ctx, const GemmArgs& g, double* ws) {
  launch_qgemm(g, ws, ctx->stream);
  CK_LAUNCH(ctx, "qgemm");
  return QCUR_OK;
}

GemmArgs gargs(int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, int opA, const double* B, int64_t ldb,
               int opB, double* C, int64_t ldc, double alpha = 1.0, double beta = 0.0) {
  GemmArgs g;
  g.Mq = M;
  g.Nq = N;
  g.Kq = K;
  g.A = A;
  g.lda = lda;
  g.opA = opA;
  g.B = B;
  g.ldb = ldb;
  g.opB = opB;
  g.C = C;
  g.ldc = ldc;
  g.alpha = alpha;
  g.beta = beta;
  return g;
}

int factor_tall(qcur_ctx* ctx, const double* src, int zh, int64_t p, int64_t q, unsigned fail_bit, double cutoff_abs,
                FactorOut out) {
  cudaStream_t st = ctx->stream;
  unsigned* status = ctx->status_dev;
  double* G1 = ctx->take<double>((size_t)(q * q * 4));
  double* L1i = ctx->take<double>((size_t)(q * q * 4));
  double* Q1 = ctx->take<double>((size_t)(p * q * 4));
  double* G2 = ctx->take<double>((size_t)(q * q * 4));
  double* L2i = ctx->take<double>((size_t)(q * q * 4));
  double* T = ctx->take<double>((size_t)(q * q * 4));
  double* betas = ctx->take<double>((size_t)q + 8);
  double* Zcm = ctx->take<double>((size_t)(p * q * 4));
  double* Qcm = ctx->take<double>((size_t)(p * q * 4));
  double* Tcm = ctx->take<double>((size_t)(q * q * 4));
  double* Vcm = ctx->take<double>((size_t)(q * q * 4 + q + 8));
  GemmArgs probe = gargs(p, q, q, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  GemmArgs probe2 = gargs(q, q, p, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  size_t wsb = qgemm_workspace_bytes(probe);
  size_t wsb2 = qgemm_workspace_bytes(probe2);
  double* gws = ctx->take<double>((wsb > wsb2 ? wsb : wsb2) / 8 + 16);
  if (!G1 || !L1i || !Q1 || !G2 || !L2i || !T || !betas || !Zcm || !Qcm || !Tcm || !Vcm || !gws)
    return ctx->fail(QCUR_E_CUDA, "workspace exhausted (factor)");
  int rc;
  const bool robust_only = ctx->force_robust || cutoff_abs >= 0.0;
  if (robust_only) {
    launch_set_status(status, fail_bit, st);
    CK_LAUNCH(ctx, "force robust");
  } else {
    // G1 = Z^H Z
    if (!zh) rc = gemm(ctx, gargs(q, q, p, src, q, 1, src, q, 0, G1, q), gws);
    else rc = gemm(ctx, gargs(q, q, p, src, p, 0, src, p, 1, G1, q), gws);
    if (rc) return rc;
    launch_cholesky(G1, q, q, status, fail_bit, st);
    launch_tri_inverse_lower(G1, q, q, L1i, q, st);
    CK_LAUNCH(ctx, "chol1");
    // Q1 = Z L1^{-H}
    if (!zh) rc = gemm(ctx, gargs(p, q, q, src, q, 0, L1i, q, 1, Q1, q), gws);
    else rc = gemm(ctx, gargs(p, q, q, src, p, 1, L1i, q, 1, Q1, q), gws);
    if (rc) return rc;
    // G2 = Q1^H Q1
    if ((rc = gemm(ctx, gargs(q, q, p, Q1, q, 1, Q1, q, 0, G2, q), gws))) return rc;
    launch_cholesky(G2, q, q, status, fail_bit, st);
    launch_tri_inverse_lower(G2, q, q, L2i, q, st);
    CK_LAUNCH(ctx, "chol2");
    // Q = Q1 L2^{-H};  F = T^{-1} = L1^{-H} L2^{-H};  T = L2^H L1^H
    if ((rc = gemm(ctx, gargs(p, q, q, Q1, q, 0, L2i, q, 1, out.Q, q), gws))) return rc;
    if ((rc = gemm(ctx, gargs(q, q, q, L1i, q, 1, L2i, q, 1, out.F, q), gws))) return rc;
    if ((rc = gemm(ctx, gargs(q, q, q, G2, q, 1, G1, q, 1, T, q), gws))) return rc;
    launch_kappa_check(T, out.F, q, ctx->kappa_limit, status, fail_bit, st);
    CK_LAUNCH(ctx, "kappa");
  }
  // robust path, gated on fail_bit
  if (!zh) launch_rowmajor_to_colmajor(src, p, q, q, Zcm, status, fail_bit, st);
  else launch_conj_copy(src, p * q, Zcm, status, fail_bit, st);
  launch_householder_qr(Zcm, p, q, betas, Qcm, T, q, status, fail_bit, st);
  launch_colmajor_to_rowmajor(Qcm, p, q, out.Q, q, status, fail_bit, 0, st);
  launch_rowmajor_to_colmajor(T, q, q, q, Tcm, status, fail_bit, st);
  launch_jacobi_pinv_factor(Tcm, Vcm, q, kEps * (double)(p > q ? p : q), cutoff_abs, out.F, q, status, fail_bit,
                            st);
  CK_LAUNCH(ctx, "robust factor");
  return QCUR_OK;
}

// explicit pinv (any shape) into out (n x m), arena reserved by caller
int pinv_impl(qcur_ctx* ctx, const double* A, int64_t m, int64_t n, double cutoff_abs, double* out, unsigned bit) {
  const bool tall = m >= n;
  const int64_t p = tall ? m : n, q = tall ? n : m;
  double* Q = ctx->take<double>((size_t)(p * q * 4));
  double* F = ctx->take<double>((size_t)(q * q * 4));
  if (!Q || !F) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (pinv)");
  int rc = factor_tall(ctx, A, tall ? 0 : 1, p, q, bit, cutoff_abs, FactorOut{Q, F});
  if (rc) return rc;
  GemmArgs probe = gargs(q, p, q, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  double* gws = ctx->take<double>(qgemm_workspace_bytes(probe) / 8 + 16);
  if (tall) return gemm(ctx, gargs(q, p, q, F, q, 0, Q, q, 1, out, p), gws);  // F Q^H  (n x m)
  return gemm(ctx, gargs(p, q, q, Q, q, 0, F, q, 1, out, q), gws);            // Q F^H  (n x m)
}

size_t pinv_ws_bytes(int64_t m, int64_t n) {
  const int64_t p = m > n ? m : n, q = m > n ? n : m;
  GemmArgs probe = gargs(q, p, q, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  return factor_ws_bytes(p, q) + qbytes(p, q) + qbytes(q, q) + qgemm_workspace_bytes(probe) + 4096;
}

size_t qmcur_ws_bytes(int64_t m, int64_t n, int64_t c, int64_t r) {
  size_t b = 0;
  b += (size_t)(draw_work_doubles(n) + draw_work_doubles(m)) * 8 + 1024;
  const bool std_shape = m >= c && n >= r;
  if (std_shape) {
    b += factor_ws_bytes(m, c) + factor_ws_bytes(n, r);
    b += qbytes(m, c) + qbytes(c, c) + qbytes(n, r) + qbytes(r, r);  // Q_C F_C Q_R F_R
    b += qbytes(m, r) + qbytes(c, r) * 2;                            // Y, M, W
    GemmArgs g1 = gargs(m, r, n, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    GemmArgs g2 = gargs(c, r, m, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    size_t a = qgemm_workspace_bytes(g1), d = qgemm_workspace_bytes(g2);
    b += (a > d ? a : d) + 4096;
  } else {
    b += pinv_ws_bytes(m, c) + pinv_ws_bytes(r, n) + qbytes(c, m) + qbytes(n, r) + qbytes(m, r);
    GemmArgs g1 = gargs(m, r, n, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    GemmArgs g2 = gargs(c, r, m, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    size_t a = qgemm_workspace_bytes(g1), d = qgemm_workspace_bytes(g2);
    b += (a > d ? a : d) + 4096;
  }
  return b + 64 * 256;
}

// draw + gather + pinv + U.  Arena reserved by the caller.
int qmcur_impl(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, const double* colp, const double* rowp,
               int64_t c, int64_t r, const uint64_t state[4], int64_t* J, int64_t* I, double* C, double* U,
               double* R) {
  cudaStream_t st = ctx->stream;
  // 1. draws: columns first, then rows, one stream (cur.py:251-253)
  Pcg64 g;
  g.state = u128{state[0], state[1]};
  g.inc = u128{state[2], state[3]};
  Pcg64 g2 = g;
  g2.advance((uint64_t)c);
  DrawJob jobs[2];
  jobs[0] = DrawJob{colp, n, c, g.state.hi, g.state.lo, g.inc.hi, g.inc.lo, J,
                    ctx->take<double>((size_t)draw_work_doubles(n))};
  jobs[1] = DrawJob{rowp, m, r, g2.state.hi, g2.state.lo, g2.inc.hi, g2.inc.lo, I,
                    ctx->take<double>((size_t)draw_work_doubles(m))};
  if (!jobs[0].work || !jobs[1].work) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (draw)");
  launch_draw(jobs, 2, ctx->status_dev, st);
  CK_LAUNCH(ctx, "draw");
  // 2. gathers (quat.py:215-225)
  launch_gather_cols(X, m, n, J, c, C, st);
  launch_gather_rows(X, n, n, I, r, R, st);
  CK_LAUNCH(ctx, "gather");
  int rc;
  if (m >= c && n >= r) {
    double* QC = ctx->take<double>((size_t)(m * c * 4));
    double* FC = ctx->take<double>((size_t)(c * c * 4));
    double* QR = ctx->take<double>((size_t)(n * r * 4));
    double* FR = ctx->take<double>((size_t)(r * r * 4));
    double* Y = ctx->take<double>((size_t)(m * r * 4));
    double* M = ctx->take<double>((size_t)(c * r * 4));
    double* W = ctx->take<double>((size_t)(c * r * 4));
    if (!QC || !FC || !QR || !FR || !Y || !M || !W) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (qmcur)");
    // 3. pinv(C) = F_C Q_C^H ; pinv(R) = Q_R F_R^H  (R^H = Q_R T_R)
    if ((rc = factor_tall(ctx, C, 0, m, c, ST_CHOL_FAIL_C, -1.0, FactorOut{QC, FC}))) return rc;
    if ((rc = factor_tall(ctx, R, 1, n, r, ST_CHOL_FAIL_R, -1.0, FactorOut{QR, FR}))) return rc;
    GemmArgs g1 = gargs(m, r, n, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    GemmArgs g2a = gargs(c, r, m, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    size_t a = qgemm_workspace_bytes(g1), d = qgemm_workspace_bytes(g2a);
    double* gws = ctx->take<double>((a > d ? a : d) / 8 + 16);
    if (!gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (qmcur gemm)");
    // 4. Y = X Q_R (m x r) — the big contraction (cur.py:268)
    if ((rc = gemm(ctx, gargs(m, r, n, X, n, 0, QR, r, 0, Y, r), gws))) return rc;
    // 5. M = Q_C^H Y (c x r)
    if ((rc = gemm(ctx, gargs(c, r, m, QC, c, 1, Y, r, 0, M, r), gws))) return rc;
    // 6. U = F_C M F_R^H
    if ((rc = gemm(ctx, gargs(c, r, c, FC, c, 0, M, r, 0, W, r), gws))) return rc;
    if ((rc = gemm(ctx, gargs(c, r, r, W, r, 0, FR, r, 1, U, r), gws))) return rc;
  } else {
    // non-standard shapes (c > m or r > n): explicit pseudoinverses
    double* PC = ctx->take<double>((size_t)(c * m * 4));
    double* PR = ctx->take<double>((size_t)(n * r * 4));
    double* Y = ctx->take<double>((size_t)(m * r * 4));
    if (!PC || !PR || !Y) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (qmcur general)");
    if ((rc = pinv_impl(ctx, C, m, c, -1.0, PC, ST_CHOL_FAIL_C))) return rc;
    if ((rc = pinv_impl(ctx, R, r, n, -1.0, PR, ST_CHOL_FAIL_R))) return rc;
    GemmArgs g1 = gargs(m, r, n, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    GemmArgs g2a = gargs(c, r, m, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    size_t a = qgemm_workspace_bytes(g1), d = qgemm_workspace_bytes(g2a);
    double* gws = ctx->take<double>((a > d ? a : d) / 8 + 16);
    if (!gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (qmcur general gemm)");
    if ((rc = gemm(ctx, gargs(m, r, n, X, n, 0, PR, r, 0, Y, r), gws))) return rc;
    if ((rc = gemm(ctx, gargs(c, r, m, PC, m, 0, Y, r, 0, U, r), gws))) return rc;
  }
  return QCUR_OK;
}

size_t error_ws_bytes(int64_t m, int64_t n, int64_t c, int64_t r) {
  (void)c;
  GemmArgs g = gargs(m, r, c, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  return qbytes(m, r) + (size_t)err_partials_count(m, n) * 16 + qgemm_workspace_bytes(g) + 4096;
}

int error_impl(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, const double* C, int64_t c, const double* U,
               const double* R, int64_t r, double* out2) {
  double* P = ctx->take<double>((size_t)(m * r * 4));
  double* parts = ctx->take<double>((size_t)err_partials_count(m, n) * 2);
  GemmArgs g = gargs(m, r, c, C, c, 0, U, r, 0, P, r);
  double* gws = ctx->take<double>(qgemm_workspace_bytes(g) / 8 + 16);
  if (!P || !parts || !gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (error)");
  int rc;
  // P = C U (m x r) (cur.py:274 left product), then the fused ||X - P R|| pass
  if ((rc = gemm(ctx, g, gws))) return rc;
  launch_cur_error(X, n, P, r, R, n, m, n, r, parts, out2, ctx->stream);
  CK_LAUNCH(ctx, "cur_error");
  return QCUR_OK;
}

int map_status(qcur_ctx* ctx, unsigned bits) {
  ctx->last_info = bits & (ST_CHOL_FAIL_C | ST_CHOL_FAIL_R | ST_DRAW_FALLBACK);
  if (bits & ST_SAMPLING) return ctx->fail(QCUR_E_SAMPLING, "index draw failed: not enough positive weights");
  if (bits & ST_DEGENERATE) return ctx->fail(QCUR_E_DEGENERATE_DISTRIBUTION, "all sampling weights vanish (zero matrix)");
  return QCUR_OK;
}

int sync_status(qcur_ctx* ctx) {
  cudaError_t e = cudaMemcpyAsync(ctx->status_host, ctx->status_dev, sizeof(unsigned), cudaMemcpyDeviceToHost,
                                  ctx->stream);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "status readback");
  e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "stream sync");
  unsigned bits = *ctx->status_host;
  cudaMemsetAsync(ctx->status_dev, 0, sizeof(unsigned), ctx->stream);
  return map_status(ctx, bits);
}

int reset_status(qcur_ctx* ctx) {
  cudaError_t e = cudaMemsetAsync(ctx->status_dev, 0, sizeof(unsigned), ctx->stream);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "status reset");
  return QCUR_OK;
}

}  // namespace

// ===========================================================================
// extern "C"
// ===========================================================================
extern "C" {

int qcur_abi_version(void) { return 1; }

int qcur_create(int device, qcur_ctx** out) {
  if (!out) return QCUR_E_PARAMETER;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) return QCUR_E_CUDA;
  if (device < 0 || device >= ndev) return QCUR_E_PARAMETER;
  if (cudaSetDevice(device) != cudaSuccess) return QCUR_E_CUDA;
  qcur_ctx* ctx = new qcur_ctx();
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&ctx->status_dev, 64) != cudaSuccess || cudaMallocHost(&ctx->status_host, 64) != cudaSuccess) {
    delete ctx;
    return QCUR_E_CUDA;
  }
  cudaMemset(ctx->status_dev, 0, 64);
  *out = ctx;
  return QCUR_OK;
}

void qcur_destroy(qcur_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (auto& kv : ctx->programs) cudaFree(kv.second.buf);
  if (ctx->arena.base) cudaFree(ctx->arena.base);
  cudaFree(ctx->status_dev);
  cudaFreeHost(ctx->status_host);
  delete ctx;
}

const char* qcur_last_error(const qcur_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }
unsigned qcur_last_info(const qcur_ctx* ctx) {
  if (!ctx) return 0;
  unsigned r = 0;
  if (ctx->last_info & ST_CHOL_FAIL_C) r |= QCUR_INFO_ROBUST_C;
  if (ctx->last_info & ST_CHOL_FAIL_R) r |= QCUR_INFO_ROBUST_R;
  if (ctx->last_info & ST_DRAW_FALLBACK) r |= QCUR_INFO_DRAW_EXACT;
  return r;
}

int qcur_set_stream(qcur_ctx* ctx, void* s) {
  if (!ctx) return QCUR_E_PARAMETER;
  ctx->stream = (cudaStream_t)s;
  return QCUR_OK;
}

int qcur_synchronize(qcur_ctx* ctx) {
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  return e == cudaSuccess ? QCUR_OK : ctx->cuda_fail(e, "synchronize");
}

int qcur_set_kappa_limit(qcur_ctx* ctx, double limit) {
  if (!ctx || !(limit > 0.0)) return QCUR_E_PARAMETER;
  ctx->kappa_limit = limit;
  return QCUR_OK;
}
int qcur_force_robust(qcur_ctx* ctx, int on) {
  if (!ctx) return QCUR_E_PARAMETER;
  ctx->force_robust = on != 0;
  return QCUR_OK;
}

int qcur_rng_seed(const uint32_t* words, int nwords, uint64_t state[4]) {
  if (!words || nwords < 1 || !state) return QCUR_E_PARAMETER;
  Pcg64 g = pcg64_from_entropy(words, nwords);
  state[0] = g.state.hi;
  state[1] = g.state.lo;
  state[2] = g.inc.hi;
  state[3] = g.inc.lo;
  return QCUR_OK;
}
int qcur_rng_advance(uint64_t state[4], uint64_t delta) {
  Pcg64 g;
  g.state = u128{state[0], state[1]};
  g.inc = u128{state[2], state[3]};
  g.advance(delta);
  state[0] = g.state.hi;
  state[1] = g.state.lo;
  return QCUR_OK;
}
int qcur_rng_random(uint64_t state[4], int64_t count, double* out) {
  Pcg64 g;
  g.state = u128{state[0], state[1]};
  g.inc = u128{state[2], state[3]};
  for (int64_t t = 0; t < count; ++t) out[t] = g.next_double();
  state[0] = g.state.hi;
  state[1] = g.state.lo;
  return QCUR_OK;
}

int qcur_memcpy(qcur_ctx* ctx, void* dst, const void* src, size_t bytes, int kind) {
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, (cudaMemcpyKind)kind, ctx->stream);
  return e == cudaSuccess ? QCUR_OK : ctx->cuda_fail(e, "memcpy");
}

int qcur_upload_planar(qcur_ctx* ctx, const double* a0, const double* a1, const double* a2, const double* a3,
                       int64_t m, int64_t n, double* x_dev) {
  if (m < 1 || n < 1) return ctx->fail(QCUR_E_SHAPE, "degenerate matrix shape (%lld, %lld)", (long long)m, (long long)n);
  const size_t pb = (size_t)(m * n) * sizeof(double);
  int rc = ctx->reserve(4 * pb + 1024);
  if (rc) return rc;
  double* planes[4];
  const double* src[4] = {a0, a1, a2, a3};
  for (int k = 0; k < 4; ++k) {
    planes[k] = ctx->take<double>((size_t)(m * n));
    cudaError_t e = cudaMemcpyAsync(planes[k], src[k], pb, cudaMemcpyHostToDevice, ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "upload H2D");
  }
  launch_planar_to_interleaved(planes[0], planes[1], planes[2], planes[3], m, n, x_dev, ctx->stream);
  CK_LAUNCH(ctx, "planar_to_interleaved");
  return QCUR_OK;
}

int qcur_download_planar(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, int64_t ld, double* a0,
                         double* a1, double* a2, double* a3) {
  const size_t pb = (size_t)(m * n) * sizeof(double);
  int rc = ctx->reserve(4 * pb + 1024);
  if (rc) return rc;
  double* planes[4];
  for (int k = 0; k < 4; ++k) planes[k] = ctx->take<double>((size_t)(m * n));
  launch_interleaved_to_planar(x_dev, m, n, ld, planes[0], planes[1], planes[2], planes[3], ctx->stream);
  CK_LAUNCH(ctx, "interleaved_to_planar");
  double* dst[4] = {a0, a1, a2, a3};
  for (int k = 0; k < 4; ++k) {
    cudaError_t e = cudaMemcpyAsync(dst[k], planes[k], pb, cudaMemcpyDeviceToHost, ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "download D2H");
  }
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  return e == cudaSuccess ? QCUR_OK : ctx->cuda_fail(e, "download sync");
}

int qcur_length_distributions(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, double* col, double* row) {
  if (m < 1 || n < 1) return ctx->fail(QCUR_E_SHAPE, "degenerate matrix shape");
  int rc = ctx->reserve(length_ws_bytes(ctx, m, n));
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  if ((rc = length_distributions_impl(ctx, x_dev, m, n, col, row))) return rc;
  return sync_status(ctx);
}

int qcur_uniform_distributions(qcur_ctx* ctx, int64_t m, int64_t n, double* col, double* row) {
  if (m < 1 || n < 1) return ctx->fail(QCUR_E_PARAMETER, "dimensions must be positive, got (%lld, %lld)",
                                       (long long)m, (long long)n);
  launch_fill(col, n, 1.0 / (double)n, ctx->stream);
  launch_fill(row, m, 1.0 / (double)m, ctx->stream);
  CK_LAUNCH(ctx, "uniform");
  return QCUR_OK;
}

int qcur_draw_indices(qcur_ctx* ctx, const double* probs, int64_t size, int64_t count, uint64_t state[4],
                      int64_t* out) {
  if (size < 1) return ctx->fail(QCUR_E_SHAPE, "probs must be a non-empty 1-D array");
  if (count < 1) return ctx->fail(QCUR_E_PARAMETER, "count must be positive, got %lld", (long long)count);
  int rc = ctx->reserve((size_t)draw_work_doubles(size) * 8 + 4096);
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  DrawJob job{probs, size, count, state[0], state[1], state[2], state[3], out,
              ctx->take<double>((size_t)draw_work_doubles(size))};
  launch_draw(&job, 1, ctx->status_dev, ctx->stream);
  CK_LAUNCH(ctx, "draw");
  qcur_rng_advance(state, (uint64_t)count);
  return sync_status(ctx);
}

int qcur_qmcur(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* colp, const double* rowp,
               int64_t c, int64_t r, const uint64_t state[4], int64_t* J, int64_t* I, double* C, double* U,
               double* R) {
  if (m < 1 || n < 1 || c < 1 || r < 1 || c > n || r > m)
    return ctx->fail(QCUR_E_SHAPE, "qmcur: bad sizes m=%lld n=%lld c=%lld r=%lld", (long long)m, (long long)n,
                     (long long)c, (long long)r);
  int rc = ctx->reserve(qmcur_ws_bytes(m, n, c, r));
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  if ((rc = qmcur_impl(ctx, x_dev, m, n, colp, rowp, c, r, state, J, I, C, U, R))) return rc;
  return sync_status(ctx);
}

int qcur_cur_error(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* C, int64_t c,
                   const double* U, const double* R, int64_t r, double* out2) {
  int rc = ctx->reserve(error_ws_bytes(m, n, c, r));
  if (rc) return rc;
  return error_impl(ctx, x_dev, m, n, C, c, U, R, r, out2);
}

int qcur_approx(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, int strategy, const uint64_t state[4],
                int64_t c, int64_t r, int64_t* J, int64_t* I, double* C, double* U, double* R, double* err2) {
  if (m < 1 || n < 1 || c < 1 || r < 1 || c > n || r > m) return ctx->fail(QCUR_E_SHAPE, "qcur_approx: bad sizes");
  if (strategy != QCUR_STRATEGY_LENGTH && strategy != QCUR_STRATEGY_UNIFORM)
    return ctx->fail(QCUR_E_PARAMETER, "unknown strategy %d", strategy);
  size_t need = (size_t)(m + n) * 8 + 1024 + qmcur_ws_bytes(m, n, c, r) + error_ws_bytes(m, n, c, r);
  if (strategy == QCUR_STRATEGY_LENGTH) need += length_ws_bytes(ctx, m, n);
  int rc = ctx->reserve(need);
  if (rc) return rc;
  double* colp = ctx->take<double>((size_t)n);
  double* rowp = ctx->take<double>((size_t)m);
  if (strategy == QCUR_STRATEGY_LENGTH) {
    if ((rc = length_distributions_impl(ctx, x_dev, m, n, colp, rowp))) return rc;
  } else {
    launch_fill(colp, n, 1.0 / (double)n, ctx->stream);
    launch_fill(rowp, m, 1.0 / (double)m, ctx->stream);
  }
  if ((rc = qmcur_impl(ctx, x_dev, m, n, colp, rowp, c, r, state, J, I, C, U, R))) return rc;
  return error_impl(ctx, x_dev, m, n, C, c, U, R, r, err2);
}

int qcur_check(qcur_ctx* ctx) { return sync_status(ctx); }

int qcur_qgemm(qcur_ctx* ctx, int opA, int opB, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
               int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  if (M < 0 || N < 0 || K < 0) return ctx->fail(QCUR_E_SHAPE, "negative gemm size");
  GemmArgs g = gargs(M, N, K, A, lda, opA, B, ldb, opB, C, ldc, alpha, beta);
  int rc = ctx->reserve(qgemm_workspace_bytes(g) + 4096);
  if (rc) return rc;
  double* ws = ctx->take<double>(qgemm_workspace_bytes(g) / 8 + 16);
  if (K == 0) {
    // C = beta C
    GemmArgs z = g;
    z.Kq = 0;
    launch_qgemm(z, ws, ctx->stream);
  } else {
    launch_qgemm(g, ws, ctx->stream);
  }
  CK_LAUNCH(ctx, "qgemm");
  return QCUR_OK;
}

int qcur_pseudoinverse(qcur_ctx* ctx, const double* a_dev, int64_t m, int64_t n, double tol, double* out_dev) {
  if (m < 1 || n < 1) return ctx->fail(QCUR_E_SHAPE, "degenerate matrix shape");
  int rc = ctx->reserve(pinv_ws_bytes(m, n) + 4096);
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  if ((rc = pinv_impl(ctx, a_dev, m, n, tol >= 0.0 ? tol : -1.0, out_dev, ST_CHOL_FAIL_C))) return rc;
  return sync_status(ctx);
}

int qcur_frobenius_sq(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, double* out_host) {
  const int64_t nparts = 296;
  int rc = ctx->reserve((size_t)nparts * 16 + 1024);
  if (rc) return rc;
  double* parts = ctx->take<double>((size_t)nparts * 2);
  double* out2 = ctx->take<double>(4);
  launch_sumsq(x_dev, m * n * 4, parts, nparts, out2, ctx->stream);
  CK_LAUNCH(ctx, "sumsq");
  cudaError_t e = cudaMemcpyAsync(out_host, out2, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  return e == cudaSuccess ? QCUR_OK : ctx->cuda_fail(e, "frobenius");
}

int qcur_synth_lowrank(qcur_ctx* ctx, int64_t m, int64_t n, int64_t k, uint64_t seed, double noise,
                       int noise_relative, double* x_dev) {
  if (m < 1 || n < 1 || k < 1) return ctx->fail(QCUR_E_PARAMETER, "synth: bad sizes");
  const int64_t nparts = 296;
  GemmArgs gprobe = gargs(m, n, k, nullptr, 0, 0, nullptr, 0, 1, nullptr, 0);
  int rc = ctx->reserve((size_t)qbytes(m, k) + qbytes(n, k) + nparts * 16 + qgemm_workspace_bytes(gprobe) + 8192);
  if (rc) return rc;
  double* P = ctx->take<double>((size_t)(m * k * 4));
  double* Q = ctx->take<double>((size_t)(n * k * 4));
  double* parts = ctx->take<double>((size_t)nparts * 2);
  double* ssq = ctx->take<double>(4);
  launch_normal_fill(P, m * k * 4, seed, 1, 1.0, ctx->stream);
  launch_normal_fill(Q, n * k * 4, seed, 2, 1.0, ctx->stream);
  GemmArgs g = gargs(m, n, k, P, k, 0, Q, k, 1, x_dev, n);  // S = P Q^H
  double* gws = ctx->take<double>(qgemm_workspace_bytes(g) / 8 + 16);
  if (!P || !Q || !parts || !ssq || !gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (synth)");
  launch_qgemm(g, gws, ctx->stream);
  CK_LAUNCH(ctx, "synth gemm");
  if (noise > 0.0) {
    if (noise_relative) {
      launch_sumsq(x_dev, m * n * 4, parts, nparts, ssq, ctx->stream);
      launch_add_scaled_noise(x_dev, m * n * 4, seed, 3, ssq, noise, ctx->stream);
    } else {
      launch_add_scaled_noise(x_dev, m * n * 4, seed, 3, nullptr, noise, ctx->stream);
    }
  }
  CK_LAUNCH(ctx, "synth noise");
  return QCUR_OK;
}

double qcur_fp64_peak_tflops(qcur_ctx* ctx) { return run_dmma_peak(ctx->sms, ctx->stream); }

}  // extern "C"
