// C-ABI implementation and host orchestration of the QMCUR device pipeline.
// See include/qcur_b200.h for the contract of every entry point and the
// reference function it replaces.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <algorithm>
#include <vector>

#include "../../include/qcur_b200.h"
#include "common.cuh"
#include "kernels.h"
#include "pairwise.h"
#include "pcg64.h"

using namespace qcur;

unsigned long long qcur::g_launches = 0;

namespace {

constexpr double kEps = 2.220446049250313e-16;
constexpr int kOzakiModuli = 15;  // default modulus count of the INT8 (Ozaki II) GEMM
constexpr size_t kSeriesTickets = 2 * 65536, kCounterWords = 2 * 65536 + 64;  // ctx->counters layout

// Optional phase timing: CUDA events recorded on the launching stream between
// pipeline phases; harvested (after a sync) by qcur_profile_read.
struct Profiler {
  bool on = false;
  bool keep = false;  // qcur_profile(ctx, 2): marks captured into a CUDA graph persist across harvests
                      // (each replay re-records the same events; harvest after every replay)
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<std::string, cudaEvent_t>> marks;  // phase name ends at this event
  cudaEvent_t start = nullptr;
  std::map<std::string, std::pair<double, long>> acc;       // name -> (total ms, count)
  cudaEvent_t next() {
    if (used == pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      pool.push_back(e);
    }
    return pool[used++];
  }
};

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
  cudaStream_t copy_stream = nullptr;  // D2H of finished factors, overlapped with the rest of the pipeline
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaStream_t side_stream = nullptr;  // residues of X for the INT8 GEMM, overlapped with the factorizations
  cudaEvent_t ev_sfork = nullptr, ev_sjoin = nullptr;
  cudaEvent_t ev_rjoin = nullptr;  // E(R)'s error digits, formed on the side stream after the gathers
  int gemm_mode = 0;                   // Y = X Q_R: 0 auto, 1 FP64 DMMA, 2 INT8 tcgen05 (Ozaki II)
  int xq_moduli = 15;                  // moduli of the INT8 X Q_R product (14 or 15; env QCUR_XQ_MODULI)
  int herm_moduli = 15;                // moduli of the INT8 Hermitian products (Grams, Q_C^H Y; QCUR_HERM_MODULI)
  // qcur_approx runs its pipeline on a high-priority stream forked from the caller's, so that
  // the low-priority side stream (residues of X) only fills SMs the pipeline leaves idle
  cudaStream_t hi_stream = nullptr;
  cudaEvent_t ev_hfork = nullptr, ev_hjoin = nullptr;
  bool prio = true;
  unsigned* status_dev = nullptr;
  unsigned* status_host = nullptr;  // pinned
  unsigned* counters = nullptr;     // split-K tickets for launch_qgemm (kept zero between launches)
                                    // [2 * 65536, + 2): tickets of launch_series_kappa
  unsigned last_info = 0;
  double kappa_limit = 1e7;
  bool force_robust = false;
  Arena arena;
  std::map<int64_t, DevProgram> programs;
  std::map<std::pair<int64_t, int64_t>, int32_t*> rf_sched;  // rows + flat chunk job lists (length tail)
  std::string err;
  Profiler prof;
  // qcur_approx_batched: child contexts (own streams, workspace, status), one per concurrent lane
  std::vector<qcur_ctx*> lanes;
  std::vector<cudaEvent_t> lane_ev;
  cudaEvent_t ev_bfork = nullptr;

  // mark the end of a named phase (no-op unless profiling).  Inside a stream capture the record
  // becomes an external event node of the graph, so replays time the phases as the graph runs them.
  void record(cudaEvent_t e) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(stream, &cs);
    if (cs == cudaStreamCaptureStatusActive) cudaEventRecordWithFlags(e, stream, cudaEventRecordExternal);
    else cudaEventRecord(e, stream);
  }
  void mark(const char* name) {
    if (!prof.on) return;
    if (!prof.start) {
      prof.start = prof.next();
      record(prof.start);
    }
    cudaEvent_t e = prof.next();
    record(e);
    prof.marks.emplace_back(name, e);
  }
  void mark_begin() {
    if (!prof.on) return;
    if (!prof.start) {
      prof.start = prof.next();
      record(prof.start);
    }
  }
  void harvest() {
    cudaEvent_t prev = prof.start;
    for (auto& mk : prof.marks) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, prev, mk.second);
      auto& a = prof.acc[mk.first];
      a.first += ms;
      a.second += 1;
      prev = mk.second;
    }
    if (prof.keep) return;
    prof.marks.clear();
    prof.start = nullptr;
    prof.used = 0;
  }

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
  std::vector<int32_t> node_ptr{0}, lvl_ptr{0}, cnode_l, cnode_r, clvl;
  int32_t maxc = 0;
  for (const ChunkPlan& cp : pp.plans) {
    plan_len.push_back(cp.len);
    maxc = cp.len > maxc ? cp.len : maxc;
    leaf_off.insert(leaf_off.end(), cp.leaf_off.begin(), cp.leaf_off.end());
    leaf_len.insert(leaf_len.end(), cp.leaf_len.begin(), cp.leaf_len.end());
    prog.insert(prog.end(), cp.prog.begin(), cp.prog.end());
    leaf_ptr.push_back((int32_t)leaf_off.size());
    prog_ptr.push_back((int32_t)prog.size());
    cnode_l.insert(cnode_l.end(), cp.node_l.begin(), cp.node_l.end());
    cnode_r.insert(cnode_r.end(), cp.node_r.begin(), cp.node_r.end());
    clvl.insert(clvl.end(), cp.lvl.begin(), cp.lvl.end());
    node_ptr.push_back((int32_t)cnode_l.size());
    lvl_ptr.push_back((int32_t)clvl.size());
  }
  // pack: int64 chunk_off first, then the int32 arrays
  std::vector<const std::vector<int32_t>*> arrs = {
      &pp.chunk_plan, &plan_len, &leaf_ptr, &prog_ptr, &leaf_off, &leaf_len, &prog,    &pp.node_l,
      &pp.node_r,     &pp.level_ptr, &node_ptr, &lvl_ptr, &cnode_l,  &cnode_r,  &clvl};
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
  const int32_t** dst[] = {&dp.d.chunk_plan,    &dp.d.plan_len,     &dp.d.plan_leaf_ptr, &dp.d.plan_prog_ptr,
                           &dp.d.leaf_off,      &dp.d.leaf_len,     &dp.d.prog,          &dp.d.node_l,
                           &dp.d.node_r,        &dp.d.level_ptr,    &dp.d.plan_node_ptr, &dp.d.plan_lvl_ptr,
                           &dp.d.cnode_l,       &dp.d.cnode_r,      &dp.d.clvl};
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
// K1 after the column pass: row / flat pairwise trees and the normalisations (cur.py:144-150)
// Job list of pairwise_rows_flat: row i, then the flat chunks of sq.ravel() starting in row i.
const int32_t* rows_flat_schedule(qcur_ctx* ctx, int64_t m, int64_t n) {
  auto key = std::make_pair(m, n);
  auto it = ctx->rf_sched.find(key);
  if (it != ctx->rf_sched.end()) return it->second;
  const PairwiseProgram pp = compile_pairwise(m * n);
  std::vector<int32_t> jobs;
  jobs.reserve((size_t)m + pp.chunk_off.size());
  size_t k = 0;
  for (int64_t i = 0; i < m; ++i) {
    jobs.push_back((int32_t)i);
    while (k < pp.chunk_off.size() && pp.chunk_off[k] < (i + 1) * n) jobs.push_back(-(int32_t)(k++) - 1);
  }
  int32_t* d = nullptr;
  if (cudaMalloc(&d, jobs.size() * sizeof(int32_t)) != cudaSuccess) return nullptr;
  cudaMemcpy(d, jobs.data(), jobs.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
  ctx->rf_sched[key] = d;
  return d;
}

int length_tail(qcur_ctx* ctx, const double* sq, const double* colsum, int64_t m, int64_t n, double* col,
                double* row) {
  cudaStream_t st = ctx->stream;
  double* rowsum = ctx->take<double>((size_t)m);
  double* scal = ctx->take<double>(8);  // total, colnorm, rownorm
  if (!rowsum || !scal) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (length)");
  int rc;
  const DevProgram* pc = ctx->program(n);
  const DevProgram* pr = ctx->program(m);
  const DevProgram* pf = ctx->program(m * n);
  if (!pc || !pr || !pf) return ctx->fail(QCUR_E_CUDA, "pairwise program allocation failed");
  if (finalize_supported(pf->d, pc->d, pr->d)) {
    // rows and flat chunks in one launch, interleaved by position and bottom-up (L2 reuse of sq),
    // then one fused tail
    double* flat = scal;
    if (pf->d.nnodes > 0) {
      flat = ctx->take<double>((size_t)pf->scratch_len);
      if (!flat) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (length)");
    }
    const int32_t* sched = rows_flat_schedule(ctx, m, n);
    if (!sched) return ctx->fail(QCUR_E_CUDA, "length schedule allocation failed");
    launch_rows_flat(sq, m, n, pc->d, pf->d, sched, rowsum, flat, st);
    launch_finalize(flat, pf->d, colsum, pc->d, col, rowsum, pr->d, row, ctx->status_dev, st);
    CK_LAUNCH(ctx, "length tail");
    ctx->mark("length");
    return QCUR_OK;
  }
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
  ctx->mark("length");
  return QCUR_OK;
}

int length_distributions_impl(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, double* col, double* row) {
  double* sq = ctx->take<double>((size_t)(m * n));
  double* colsum = ctx->take<double>((size_t)n);
  if (!sq || !colsum) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (length)");
  launch_colstrip(X, m, n, n, sq, colsum, ctx->stream);
  CK_LAUNCH(ctx, "colstrip");
  return length_tail(ctx, sq, colsum, m, n, col, row);
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

bool int8_q1_fits(int64_t p, int64_t q);

size_t factor_ws_bytes(int64_t p, int64_t q) {
  size_t b = 0;
  b += qbytes(p, q) * 2;        // Zcm, Qcm
  b += qbytes(q, q) * 12;       // G1, L1, L1inv, G2, L2, L2inv, T, Tcm, Vcm, ...
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
  if (q > 304)  // blocked Cholesky scratch (chol_inv_blocked): A, L, blocks, T and its GEMM slabs
    b += 2 * qbytes(q, q) + 2 * qbytes(256, 256) + qbytes(256, q) + (size_t)16 * q * q * 8 + 8192;
  if (ozaki_herm_supported(p, q, q)) b += ozaki_herm_workspace_bytes(p, q, q, 1) + 4096;  // INT8 Grams
  if (int8_q1_fits(p, q)) b += ozaki_workspace_bytes(p, q, q, 15) + 4096;                   // INT8 Q1
  return b + 16 * 256;
}

int gemm(qcur_ctx* ctx, const GemmArgs& g, double* ws) {
  launch_qgemm(g, ws, ctx->counters, ctx->stream);
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

// Y = X Q_R on the INT8 tensor cores?  auto: when the product is large enough to pay for the residues
// Thresholds (round 2, measured for throughput): the INT8 engine wins from cfg1's size up
// (1000^2, r = 40: 1708 -> 1875 approx/s one at a time; cfg4's 64 x 1024^2: 2910 -> 3920 matrices/s).
constexpr double kInt8MinMNRDefault = 3e7, kInt8MinGramDefault = 1e6;
// QCUR_INT8_MIN_MNR / QCUR_INT8_MIN_GRAM override the thresholds (A/B timing)
double env_or(const char* name, double v) {
  const char* e = std::getenv(name);
  return e ? std::atof(e) : v;
}
const double kInt8MinMNR = env_or("QCUR_INT8_MIN_MNR", kInt8MinMNRDefault);
const double kInt8MinGram = env_or("QCUR_INT8_MIN_GRAM", kInt8MinGramDefault);
bool use_int8(const qcur_ctx* ctx, int64_t m, int64_t n, int64_t r) {
  if (ctx->gemm_mode == 1 || !ozaki_supported(m, n, r)) return false;
  return ctx->gemm_mode == 2 || (double)m * (double)n * (double)r >= kInt8MinMNR;
}

// Y = X Q_R on the INT8 tensor cores one chunk of rows at a time (a product whose residues
// exceed the one-shot workspace cap, e.g. cfg5's 32768^2 X: 64 GB of residue planes)?
// bytes of INT8 workspace for the chunked product (QCUR_OZ_CHUNK_CAP lowers it for tests)
double oz_chunk_cap() {
  const char* e = std::getenv("QCUR_OZ_CHUNK_CAP");
  return e ? std::atof(e) : 24e9;
}
int64_t int8_chunk_rows(const qcur_ctx* ctx, int64_t m, int64_t n, int64_t r) {
  if (ctx->gemm_mode == 1 || ozaki_supported(m, n, r)) return 0;
  if (!(ctx->gemm_mode == 2 || (double)m * (double)n * (double)r >= 2e8)) return 0;
  return ozaki_chunk_rows(m, n, r, oz_chunk_cap());
}

// the Grams Z^H Z (Z: p x q) of CholeskyQR2 on the INT8 tensor cores?
bool use_int8_gram(const qcur_ctx* ctx, int64_t p, int64_t q) {
  if (ctx->gemm_mode == 1 || !ozaki_herm_supported(p, q, q)) return false;
  return ctx->gemm_mode == 2 || (double)p * (double)q * (double)q >= kInt8MinGram;
}

// the triangular product Q1 = Z L1^{-H} (Z: p x q) of CholeskyQR2 on the INT8 tensor cores?  Off by
// default: measured slower than the FP64 DMMA GEMM at every BASELINE size (cfg2 pair: residues 2 x 59,
// GEMM 155, CRT 2 x 52 = 386 us against 230 us on DMMA; factor phase 1.162 -> 1.327 ms).
// QCUR_INT8_MIN_Q1 (a p q^2 threshold) turns it on for A/B timing and tests.
const double kInt8MinQ1 = env_or("QCUR_INT8_MIN_Q1", 1e300);
constexpr double kInt8Q1WorkspaceCap = 2e9;  // bytes per block (cfg5's q = 1000 stays on DMMA)
bool int8_q1_fits(int64_t p, int64_t q) {
  return ozaki_supported(p, q, q) && (double)ozaki_workspace_bytes(p, q, q, 15) <= kInt8Q1WorkspaceCap;
}
bool use_int8_q1(const qcur_ctx* ctx, int64_t p, int64_t q) {
  if (ctx->gemm_mode == 1 || !int8_q1_fits(p, q)) return false;
  return ctx->gemm_mode == 2 || (double)p * (double)q * (double)q >= kInt8MinQ1;
}

// the fused error ||X - P R|| on the INT8 tensor cores?  (same policy, its own shape limits)
bool use_int8_err(const qcur_ctx* ctx, int64_t m, int64_t n, int64_t r) {
  if (ctx->gemm_mode == 1 || !ozaki_error_supported(m, n, r)) return false;
  return ctx->gemm_mode == 2 || (double)m * (double)n * (double)r >= kInt8MinMNR;
}

// structure hints: op(B) upper triangular; Hermitian output with only its lower triangle consumed
GemmArgs with_flags(GemmArgs g, int b_upper, int herm_lower) {
  g.b_upper = b_upper;
  g.herm_lower = herm_lower;
  return g;
}

// Blocked Cholesky + inverse for Grams larger than one cluster holds (q > 304,
// e.g. cfg5's c = r = 1000).  Diagonal blocks of kBlk run on the 16-CTA cluster
// kernel; panels L_ik = A_ik X_kk^H and trailing updates A -= L_p L_p^H run on
// the DMMA GEMM; X = L^{-1} follows by block forward substitution
// X_i,0:i = -X_ii (L_i,0:i X_0:i,0:i).  G is read only; X (q x q) receives L^{-1}.
constexpr int64_t kBlk = 256;

size_t chol_blocked_ws_bytes(int64_t q) {
  GemmArgs g = gargs(q, q, kBlk, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  GemmArgs g2 = gargs(kBlk, q, q, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  size_t w1 = qgemm_workspace_bytes(g), w2 = qgemm_workspace_bytes(g2);
  return 2 * qbytes(q, q) + 2 * qbytes(kBlk, kBlk) + qbytes(kBlk, q) + (w1 > w2 ? w1 : w2) + 8 * 256;
}

int chol_inv_blocked(qcur_ctx* ctx, const double* G, int64_t q, double* X, unsigned fail_bit) {
  cudaStream_t st = ctx->stream;
  double* A = ctx->take<double>((size_t)(q * q * 4));
  double* L = ctx->take<double>((size_t)(q * q * 4));
  double* D = ctx->take<double>((size_t)(kBlk * kBlk * 4));
  double* Xb = ctx->take<double>((size_t)(kBlk * kBlk * 4));
  double* T = ctx->take<double>((size_t)(kBlk * q * 4));
  GemmArgs g = gargs(q, q, kBlk, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  GemmArgs g2 = gargs(kBlk, q, q, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  size_t w1 = qgemm_workspace_bytes(g), w2 = qgemm_workspace_bytes(g2);
  double* gws = ctx->take<double>((w1 > w2 ? w1 : w2) / 8 + 16);
  if (!A || !L || !D || !Xb || !T || !gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (blocked cholesky)");
  const size_t row = (size_t)q * 32, qb = 32;
  cudaMemcpyAsync(A, G, (size_t)qbytes(q, q), cudaMemcpyDeviceToDevice, st);
  cudaMemsetAsync(X, 0, (size_t)qbytes(q, q), st);
  cudaMemsetAsync(L, 0, (size_t)qbytes(q, q), st);
  int rc;
  const int64_t nb = (q + kBlk - 1) / kBlk;
  for (int64_t k = 0; k < nb; ++k) {
    const int64_t kb = k * kBlk, bs = (q - kb) < kBlk ? (q - kb) : kBlk, rem = q - kb - bs;
    cudaMemcpy2DAsync(D, bs * qb, A + (kb * q + kb) * 4, row, bs * qb, bs, cudaMemcpyDeviceToDevice, st);
    CholJob job{D, nullptr, Xb, fail_bit};
    launch_chol_inv_cluster(&job, 1, bs, ctx->status_dev, st);
    cudaMemcpy2DAsync(X + (kb * q + kb) * 4, row, Xb, bs * qb, bs * qb, bs, cudaMemcpyDeviceToDevice, st);
    CK_LAUNCH(ctx, "blocked cholesky diag");
    if (rem == 0) break;
    double* Lp = L + ((kb + bs) * q + kb) * 4;
    // panel L_ik = A_ik X_kk^H  (op(B) upper triangular)
    if ((rc = gemm(ctx, with_flags(gargs(rem, bs, bs, A + ((kb + bs) * q + kb) * 4, q, 0, Xb, bs, 1, Lp, q), 1, 0),
                   gws)))
      return rc;
    // trailing A_jj -= L_p L_p^H (lower triangle only)
    if ((rc = gemm(ctx,
                   with_flags(gargs(rem, rem, bs, Lp, q, 0, Lp, q, 1, A + ((kb + bs) * q + kb + bs) * 4, q, -1.0, 1.0),
                              0, 1),
                   gws)))
      return rc;
  }
  for (int64_t i = 1; i < nb; ++i) {
    const int64_t ib = i * kBlk, bs = (q - ib) < kBlk ? (q - ib) : kBlk;
    // T = L_i,0:i X_0:i,0:i   (bs x ib)
    if ((rc = gemm(ctx, gargs(bs, ib, ib, L + ib * q * 4, q, 0, X, q, 0, T, ib), gws))) return rc;
    // X_i,0:i = -X_ii T
    if ((rc = gemm(ctx, gargs(bs, ib, bs, X + (ib * q + ib) * 4, q, 0, T, ib, 0, X + ib * q * 4, q, -1.0, 0.0), gws)))
      return rc;
  }
  (void)row;
  return QCUR_OK;
}

struct FactorSpec {
  const double* src;  // Z = src (zh = 0, p x q) or Z = src^H (zh = 1, src is q x p)
  int zh;
  int64_t p, q;
  unsigned fail_bit;
  double cutoff_abs;  // >= 0: explicit pinv tolerance (forces the robust path)
  FactorOut out;
};

// Factor up to two tall blocks together (C and R^H of one QMCUR step) so the
// latency-bound small kernels (cluster Cholesky) serve both in one launch.
int factor_multi(qcur_ctx* ctx, const FactorSpec* specs_in, int ns) {
  cudaStream_t st = ctx->stream;
  unsigned* status = ctx->status_dev;
  FactorSpec specs[2];
  for (int k = 0; k < ns; ++k) specs[k] = specs_in[k];
  // Two blocks factor in lock step with paired GEMM launches (one launch, the SMs split
  // between the C and R^H problems).  The pair needs identical ops, so a block given as
  // src^H (R) is materialised as Z = R^H first (one 32-byte-per-element transpose).
  if (ns == 2) {
    for (int k = 0; k < 2; ++k) {
      if (!specs[k].zh) continue;
      double* ZH = ctx->take<double>((size_t)(specs[k].p * specs[k].q * 4));
      if (!ZH) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (factor transpose)");
      launch_conj_transpose(specs[k].src, specs[k].q, specs[k].p, specs[k].p, ZH, specs[k].q, st);
      CK_LAUNCH(ctx, "factor transpose");
      specs[k].src = ZH;
      specs[k].zh = 0;
    }
  }
  struct Bufs {
    double *G1, *L1, *L1i, *G2, *L2, *L2i, *T, *betas, *Zcm, *Qcm, *Tcm, *Vcm, *gws;
  } B[2];
  for (int k = 0; k < ns; ++k) {
    const int64_t p = specs[k].p, q = specs[k].q;
    Bufs& b = B[k];
    b.G1 = ctx->take<double>((size_t)(q * q * 4));
    b.L1 = ctx->take<double>((size_t)(q * q * 4));
    b.L1i = ctx->take<double>((size_t)(q * q * 4));
    b.G2 = ctx->take<double>((size_t)(q * q * 4));
    b.L2 = ctx->take<double>((size_t)(q * q * 4));
    b.L2i = ctx->take<double>((size_t)(q * q * 4));
    b.T = ctx->take<double>((size_t)(q * q * 4));
    b.betas = ctx->take<double>((size_t)q + 8);
    b.Zcm = ctx->take<double>((size_t)(p * q * 4));
    b.Qcm = ctx->take<double>((size_t)(p * q * 4));
    b.Tcm = ctx->take<double>((size_t)(q * q * 4));
    b.Vcm = ctx->take<double>((size_t)(q * q * 4 + q + 8));
    GemmArgs probe = gargs(p, q, q, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    GemmArgs probe2 = gargs(q, q, p, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    size_t w1 = qgemm_workspace_bytes(probe), w2 = qgemm_workspace_bytes(probe2);
    b.gws = ctx->take<double>((w1 > w2 ? w1 : w2) / 8 + 16);
    if (!b.G1 || !b.L1 || !b.L1i || !b.G2 || !b.L2 || !b.L2i || !b.T || !b.betas || !b.Zcm || !b.Qcm ||
        !b.Tcm || !b.Vcm || !b.gws)
      return ctx->fail(QCUR_E_CUDA, "workspace exhausted (factor)");
  }
  int rc;
  bool fast[2] = {false, false};
  for (int k = 0; k < ns; ++k) fast[k] = !(ctx->force_robust || specs[k].cutoff_abs >= 0.0);
  // Grams on the INT8 tensor cores (Ozaki II, k_ozaki.cu) when every fast block qualifies
  bool i8gram = true;
  void* gws8[2] = {nullptr, nullptr};
  for (int k = 0; k < ns; ++k)
    if (fast[k] && (specs[k].zh || !use_int8_gram(ctx, specs[k].p, specs[k].q))) i8gram = false;
  if (i8gram)
    for (int k = 0; k < ns; ++k) {
      if (!fast[k]) continue;
      gws8[k] = ctx->take<uint8_t>(ozaki_herm_workspace_bytes(specs[k].p, specs[k].q, specs[k].q, 1));
      if (!gws8[k]) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (int8 gram)");
    }
  // G = Z^H Z for every fast block (second: Z = Q1), INT8 or FP64 (paired launches either way)
  auto gram_each = [&](bool second) -> int {
    if (i8gram) {
      const double* A[2];
      int64_t pp[2], qq[2], lda[2], ldg[2];
      double* G[2];
      void* w[2];
      int np = 0;
      for (int k = 0; k < ns; ++k) {
        if (!fast[k]) continue;
        A[np] = second ? specs[k].out.Q : specs[k].src;
        pp[np] = specs[k].p;
        qq[np] = specs[k].q;
        lda[np] = specs[k].q;
        ldg[np] = specs[k].q;
        G[np] = second ? B[k].G2 : B[k].G1;
        w[np] = gws8[k];
        ++np;
      }
      if (np == 0) return QCUR_OK;
      if (launch_ozaki_herm(A, A, pp, qq, qq, lda, lda, G, ldg, np, ctx->herm_moduli, w, st, 1))
        return ctx->fail(QCUR_E_CUDA, "int8 gram: tensor map encode failed");
      CK_LAUNCH(ctx, "int8 gram");
      return QCUR_OK;
    }
    return QCUR_E_CUDA + 100;  // caller falls back to the FP64 GEMMs
  };
  // one GEMM per fast block: paired into one launch when both blocks are on the fast path
  auto gemm_each = [&](auto&& args_of) -> int {
    if (ns == 2 && fast[0] && fast[1]) {
      launch_qgemm_pair(args_of(0), B[0].gws, args_of(1), B[1].gws, ctx->counters, st);
      CK_LAUNCH(ctx, "qgemm pair");
      return QCUR_OK;
    }
    for (int k = 0; k < ns; ++k) {
      if (!fast[k]) continue;
      const int r2 = gemm(ctx, args_of(k), B[k].gws);
      if (r2) return r2;
    }
    return QCUR_OK;
  };
  // Cholesky + inverse of each Gram: one cluster launch when both fit, else per problem
  auto chol_inv = [&](bool second) -> int {  // (second pass uses the series below)
    CholJob jobs[2];
    int nj = 0;
    int64_t qj = -1;
    bool together = true;
    for (int k = 0; k < ns; ++k) {
      if (!fast[k]) continue;
      Bufs& b = B[k];
      jobs[nj++] = CholJob{second ? b.G2 : b.G1, second ? b.L2 : b.L1, second ? b.L2i : b.L1i, specs[k].fail_bit};
      if (qj >= 0 && qj != specs[k].q) together = false;
      qj = specs[k].q;
    }
    if (nj == 0) return QCUR_OK;
    if (together && qj <= chol_cluster_qmax()) {
      launch_chol_inv_cluster(jobs, nj, qj, status, st);
    } else {
      for (int k = 0; k < ns; ++k) {
        if (!fast[k]) continue;
        Bufs& b = B[k];
        const int64_t q = specs[k].q;
        double* G = second ? b.G2 : b.G1;
        double* L = second ? b.L2 : b.L1;
        double* Li = second ? b.L2i : b.L1i;
        if (q <= chol_cluster_qmax()) {
          CholJob j1{G, L, Li, specs[k].fail_bit};
          launch_chol_inv_cluster(&j1, 1, q, status, st);
        } else {
          (void)L;
          const int rcb = chol_inv_blocked(ctx, G, q, Li, specs[k].fail_bit);
          if (rcb) return rcb;
        }
      }
    }
    CK_LAUNCH(ctx, "cholesky");
    return QCUR_OK;
  };
  for (int k = 0; k < ns; ++k) {
    if (fast[k]) continue;
    launch_set_status(status, specs[k].fail_bit, st);
    CK_LAUNCH(ctx, "force robust");
  }
  auto zsrc = [&](int k) { return specs[k]; };
  // G1 = Z^H Z
  if (i8gram) {
    if ((rc = gram_each(false))) return rc;
  } else if ((rc = gemm_each([&](int k) {
         const FactorSpec f = zsrc(k);
         const int64_t p = f.p, q = f.q;
         return f.zh ? with_flags(gargs(q, q, p, f.src, p, 0, f.src, p, 1, B[k].G1, q), 0, 1)
                     : with_flags(gargs(q, q, p, f.src, q, 1, f.src, q, 0, B[k].G1, q), 0, 1);
       })))
    return rc;
  if ((rc = chol_inv(false))) return rc;
  // Q1 = Z L1^{-H} (written straight into the output Q);  G2 = Q1^H Q1
  // Q1 on the INT8 tensor cores (Ozaki II, both blocks in shared launches) next to INT8 Grams
  bool i8q1 = i8gram;
  for (int k = 0; k < ns; ++k)
    if (fast[k] && !use_int8_q1(ctx, specs[k].p, specs[k].q)) i8q1 = false;
  if (i8q1) {
    const double* X[2];
    const double* Bm[2];
    int64_t mm[2], nn[2], ld[2];
    int cj[2];
    double* Y[2];
    void* w[2];
    int np = 0;
    for (int k = 0; k < ns; ++k) {
      if (!fast[k]) continue;
      X[np] = specs[k].src;
      Bm[np] = B[k].L1i;
      mm[np] = specs[k].p;
      nn[np] = specs[k].q;
      ld[np] = specs[k].q;
      cj[np] = 1;
      Y[np] = specs[k].out.Q;
      w[np] = ctx->take<uint8_t>(ozaki_workspace_bytes(specs[k].p, specs[k].q, specs[k].q, ctx->herm_moduli));
      if (!w[np]) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (int8 Q1)");
      ++np;
    }
    if (np && launch_ozaki_pair(X, mm, nn, ld, Bm, nn, ld, cj, Y, ld, np, ctx->herm_moduli, w, st))
      return ctx->fail(QCUR_E_CUDA, "int8 Q1: tensor map encode failed");
    CK_LAUNCH(ctx, "int8 Q1");
  } else if ((rc = gemm_each([&](int k) {
         const FactorSpec f = zsrc(k);
         const int64_t p = f.p, q = f.q;
         return f.zh ? with_flags(gargs(p, q, q, f.src, p, 1, B[k].L1i, q, 1, f.out.Q, q), 1, 0)
                     : with_flags(gargs(p, q, q, f.src, q, 0, B[k].L1i, q, 1, f.out.Q, q), 1, 0);
       })))
    return rc;
  if (i8gram) {
    if ((rc = gram_each(true))) return rc;
  } else if ((rc = gemm_each([&](int k) {
               const int64_t p = specs[k].p, q = specs[k].q;
               return with_flags(gargs(q, q, p, specs[k].out.Q, q, 1, specs[k].out.Q, q, 0, B[k].G2, q), 0, 1);
             }))) {
    return rc;
  }
  // second pass, round 2: Z = Q T with Q = Q1 L2^{-H}, T = L2^H L1^H and G2 = L2 L2^H, so
  // pinv(Z) = T^{-1} Q^H = L1^{-H} L2^{-H} L2^{-1} Q1^H = (L1^{-H} G2^{-1}) Q1^H: the factor is
  // F = L1^{-H} (I - E + E^2) with E = G2 - I ~ kappa^2 u (gate max|E| <= 1e-5, dropped term
  // |E|^3 <= 1e-15), two small GEMMs instead of the series for L2^{-1}, T and T L2^{-1} (four).
  // The kappa_F guard uses ||L1^{-1}||_F (= ||T^{-1}||_F up to 1 + |E|).
  static const int series_env = [] {
    const char* e = std::getenv("QCUR_SERIES_INV");
    return e ? std::atoi(e) : -1;
  }();
  if (series_env != 0) {
    // E, S = I - E and the kappa_F guard of both blocks in one launch
    SeriesKappaJobs sj{};
    int nsj = 0;
    for (int k = 0; k < ns; ++k) {
      if (!fast[k]) continue;
      double* part = ctx->take<double>((size_t)2 * series_kappa_blocks(specs[k].q) + 8);
      if (!part) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (series)");
      sj.j[nsj++] = SeriesKappaJob{B[k].G2, B[k].G1, B[k].L1i, B[k].Tcm, B[k].Vcm, part, specs[k].q, specs[k].fail_bit};
    }
    if (nsj) launch_series_kappa(sj, nsj, status, ctx->counters + kSeriesTickets, 1e-5, ctx->kappa_limit, st);
    CK_LAUNCH(ctx, "series prep");
    if ((rc = gemm_each([&](int k) {  // S += E E  (S = I - E + E^2)
           const int64_t q = specs[k].q;
           return gargs(q, q, q, B[k].Tcm, q, 0, B[k].Tcm, q, 0, B[k].Vcm, q, 1.0, 1.0);
         })))
      return rc;
    if ((rc = gemm_each([&](int k) {  // F = L1^{-H} S
           const int64_t q = specs[k].q;
           return gargs(q, q, q, B[k].L1i, q, 1, B[k].Vcm, q, 0, specs[k].out.F, q);
         })))
      return rc;
  } else {
  // second pass: G2 = I + E with E ~ kappa^2 u; L2^{-1} by a second-order series
  // (no sequential Cholesky; blocks with max|E| > 1e-5 take the robust path)
  // M0 = lh(E) in b.L2, P = M0 M0^H in b.T, M1 in b.Tcm, P2 = M1 M1 in b.Vcm
  for (int k = 0; k < ns; ++k)
    if (fast[k]) launch_series_lh(B[k].G2, nullptr, specs[k].q, B[k].L2, status, specs[k].fail_bit, 1e-5, st);
  if ((rc = gemm_each([&](int k) {
         const int64_t q = specs[k].q;
         return with_flags(gargs(q, q, q, B[k].L2, q, 0, B[k].L2, q, 1, B[k].T, q), 1, 1);
       })))
    return rc;
  for (int k = 0; k < ns; ++k)
    if (fast[k]) launch_series_lh(B[k].G2, B[k].T, specs[k].q, B[k].Tcm, status, specs[k].fail_bit, 1e-5, st);
  if ((rc = gemm_each([&](int k) {
         const int64_t q = specs[k].q;
         return gargs(q, q, q, B[k].Tcm, q, 0, B[k].Tcm, q, 0, B[k].Vcm, q);
       })))
    return rc;
  for (int k = 0; k < ns; ++k)
    if (fast[k]) launch_series_final(B[k].Tcm, B[k].Vcm, specs[k].q, B[k].L2i, st);
  CK_LAUNCH(ctx, "series");
  // Z = Q T with Q = Q1 L2^{-H}, T = L2^H L1^H.  The tall product Q1 L2^{-H} is never
  // formed: pinv(Z) = T^{-1} Q^H = (T^{-1} L2^{-1}) Q1^H, so the factor pair is
  // (Q1, F = T^{-1} L2^{-1}) and every consumer (X Q_R, Q_C^H Y, F Q^H) applies the
  // well-conditioned L2^{-1} (kappa ~ 1 + kappa(Z)^2 u) on the small side instead.
  // kappa_F(T) = ||Z||_F ||T^{-1}||_F = sqrt(tr G1) ||T^{-1}||_F guards the fast path.
  // (T^{-1} lives in b.T, free again after the series.)
  if ((rc = gemm_each([&](int k) {
         const int64_t q = specs[k].q;
         return with_flags(gargs(q, q, q, B[k].L1i, q, 1, B[k].L2i, q, 1, B[k].T, q), 1, 0);
       })))
    return rc;
  for (int k = 0; k < ns; ++k)
    if (fast[k]) launch_kappa_check(B[k].G1, B[k].T, specs[k].q, ctx->kappa_limit, status, specs[k].fail_bit, st);
  CK_LAUNCH(ctx, "kappa");
  if ((rc = gemm_each([&](int k) {
         const int64_t q = specs[k].q;
         return gargs(q, q, q, B[k].T, q, 0, B[k].L2i, q, 0, specs[k].out.F, q);
       })))
    return rc;
  }
  // robust path, gated on each fail_bit (no-op launches when the fast path held)
  static const int mode_env = [] {
    const char* e = std::getenv("QCUR_ROBUST");
    if (!e) return 0;
    return std::string(e) == "jacobi" ? 1 : std::string(e) == "hh" ? 2 : 0;
  }();
  bool merged = mode_env == 0;
  for (int k = 0; k < ns; ++k)
    if (specs[k].zh || !robust_qr_supported(specs[k].p, specs[k].q)) merged = false;
  if (merged) {  // both blocks' gated copies, Householder QRs and triangular pinvs in three launches
    const double* Z[2];
    double* Zc[2];
    int64_t pp[2], qq[2];
    unsigned bits[2];
    RobustQrJob rj[2];
    for (int k = 0; k < ns; ++k) {
      const FactorSpec& f = specs[k];
      Bufs& b = B[k];
      Z[k] = f.src;
      Zc[k] = b.Zcm;
      pp[k] = f.p;
      qq[k] = f.q;
      bits[k] = f.fail_bit;
      rj[k] = RobustQrJob{b.Zcm, f.p, f.q, b.betas, b.Qcm, f.out.Q, f.q, b.Tcm, b.Vcm, f.out.F, f.q,
                          kEps * (double)(f.p > f.q ? f.p : f.q), f.cutoff_abs, status, f.fail_bit};
    }
    launch_rowmajor_to_colmajor2(Z, pp, qq, qq, Zc, ns, status, bits, st);
    launch_robust_qr_pinv_multi(rj, ns, st);
    CK_LAUNCH(ctx, "robust factor");
    return QCUR_OK;
  }
  for (int k = 0; k < ns; ++k) {
    const FactorSpec& f = specs[k];
    const int64_t p = f.p, q = f.q;
    Bufs& b = B[k];
    if (!f.zh) launch_rowmajor_to_colmajor(f.src, p, q, q, b.Zcm, status, f.fail_bit, st);
    else launch_conj_copy(f.src, p * q, b.Zcm, status, f.fail_bit, st);
    // round 2: Householder QR and the one-sided Jacobi pinv of its triangular factor, each on a
    // 16-CTA cluster (k_robust.cu).  QCUR_ROBUST=jacobi: one-sided Jacobi on Z itself (cluster);
    // QCUR_ROBUST=hh: round 1's single-CTA Householder QR + Jacobi (340 ms per side at cfg2).
    const double cutoff_scale = kEps * (double)(p > q ? p : q);
    if (mode_env == 2) {
      launch_householder_qr(b.Zcm, p, q, b.betas, b.Qcm, b.T, q, status, f.fail_bit, st);
      launch_colmajor_to_rowmajor(b.Qcm, p, q, f.out.Q, q, status, f.fail_bit, 0, st);
      launch_rowmajor_to_colmajor(b.T, q, q, q, b.Tcm, status, f.fail_bit, st);
      launch_jacobi_pinv_factor(b.Tcm, b.Vcm, q, cutoff_scale, f.cutoff_abs, f.out.F, q, status, f.fail_bit, st);
    } else if (mode_env == 0 && robust_qr_supported(p, q)) {
      launch_robust_qr_pinv(b.Zcm, p, q, b.betas, b.Qcm, f.out.Q, q, b.Tcm, b.Vcm, f.out.F, q, cutoff_scale,
                            f.cutoff_abs, status, f.fail_bit, st);
    } else {
      launch_robust_jacobi(b.Zcm, p, q, b.Vcm, f.out.Q, q, f.out.F, q, cutoff_scale, f.cutoff_abs, status, f.fail_bit,
                           st);
    }
    CK_LAUNCH(ctx, "robust factor");
  }
  return QCUR_OK;
}

int factor_tall(qcur_ctx* ctx, const double* src, int zh, int64_t p, int64_t q, unsigned fail_bit, double cutoff_abs,
                FactorOut out) {
  FactorSpec f{src, zh, p, q, fail_bit, cutoff_abs, out};
  return factor_multi(ctx, &f, 1);
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
    b += factor_ws_bytes(m, c) + factor_ws_bytes(n, r) + qbytes(n, r);  // + R^H for the paired factor
    b += qbytes(m, c) + qbytes(c, c) + qbytes(n, r) + qbytes(r, r);  // Q_C F_C Q_R F_R
    b += qbytes(m, r) + qbytes(c, r) * 2;                            // Y, M, W
    GemmArgs g1 = gargs(m, r, n, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    GemmArgs g2 = gargs(c, r, m, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    size_t a = qgemm_workspace_bytes(g1), d = qgemm_workspace_bytes(g2);
    b += (a > d ? a : d) + 4096;
    if (ozaki_supported(m, n, r)) b += ozaki_workspace_bytes(m, n, r, kOzakiModuli) + 4096;
    else if (int64_t mc = ozaki_chunk_rows(m, n, r, oz_chunk_cap())) b += ozaki_workspace_bytes(mc, n, r, kOzakiModuli) + 4096;
    if (ozaki_herm_supported(m, c, r)) b += ozaki_herm_workspace_bytes(m, c, r, 0) + 4096;  // Q_C^H Y
  } else {
    b += pinv_ws_bytes(m, c) + pinv_ws_bytes(r, n) + qbytes(c, m) + qbytes(n, r) + qbytes(m, r);
    GemmArgs g1 = gargs(m, r, n, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    GemmArgs g2 = gargs(c, r, m, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    size_t a = qgemm_workspace_bytes(g1), d = qgemm_workspace_bytes(g2);
    b += (a > d ? a : d) + 4096;
  }
  return b + 64 * 256;
}

int qmcur_core(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, int64_t c, int64_t r, const int64_t* J,
               const double* C, double* U, const double* R, int core, void* oz_ready = nullptr);

// Start the X-only half of the INT8 contraction (residues of X) on the side stream, so that it
// overlaps the draws and factorizations; the main stream joins before the GEMM.  Returns the
// workspace holding the residues, or nullptr when the FP64 path will be used.
void* int8_fork_prepare(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, int64_t r, int* rc);
// qcur_approx forms E(R)'s error digits on the side stream right after the gathers (QCUR_RDIG_EARLY=0: with
// the digits of P, just before the error kernel)
bool rdigits_early() {
  static const bool v = [] {
    const char* e = std::getenv("QCUR_RDIG_EARLY");
    return !(e && std::string(e) == "0");
  }();
  return v;
}
// QCUR_XRES_FORK=draw: the residues of X fork after the draws instead of after the length pass
bool xres_fork_after_draw() {
  static const bool v = [] {
    const char* e = std::getenv("QCUR_XRES_FORK");
    return e && std::string(e) == "draw";
  }();
  return v;
}

// Host destinations for qcur_qmcur_host (planar, the reference's QMatrix layout).
struct HostOut {
  int64_t* J;
  int64_t* I;
  double* C[4];
  double* U[4];
  double* R[4];
};

size_t host_out_ws_bytes(int64_t m, int64_t n, int64_t c, int64_t r) {
  return qbytes(m, c) + qbytes(r, n) + qbytes(c, r) + 1024;
}

// Fork the copy stream off the main stream at this point and queue there the
// planar conversion + D2H of a finished p x q interleaved factor (and optional
// index vectors).  The main stream carries on with the pipeline.
int copy_out(qcur_ctx* ctx, const double* A, int64_t p, int64_t q, double* const dst[4], const int64_t* idx_a,
             int64_t na, int64_t* host_a, const int64_t* idx_b, int64_t nb, int64_t* host_b) {
  cudaStream_t cs = ctx->copy_stream;
  cudaError_t e = cudaEventRecord(ctx->ev_fork, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ctx->ev_fork, 0);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "copy fork");
  const size_t pb = (size_t)(p * q) * sizeof(double);
  double* planes[4];
  for (int k = 0; k < 4; ++k) planes[k] = ctx->take<double>((size_t)(p * q));
  if (!planes[3]) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (host copy)");
  launch_interleaved_to_planar(A, p, q, q, planes[0], planes[1], planes[2], planes[3], cs);
  CK_LAUNCH(ctx, "copy-out planar");
  for (int k = 0; k < 4 && e == cudaSuccess; ++k) e = cudaMemcpyAsync(dst[k], planes[k], pb, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess && host_a) e = cudaMemcpyAsync(host_a, idx_a, (size_t)na * 8, cudaMemcpyDeviceToHost, cs);
  if (e == cudaSuccess && host_b) e = cudaMemcpyAsync(host_b, idx_b, (size_t)nb * 8, cudaMemcpyDeviceToHost, cs);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "copy-out D2H");
  return QCUR_OK;
}

// Join: the main stream waits for every queued copy-out.
int copy_join(qcur_ctx* ctx) {
  cudaError_t e = cudaEventRecord(ctx->ev_join, ctx->copy_stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->stream, ctx->ev_join, 0);
  return e == cudaSuccess ? QCUR_OK : ctx->cuda_fail(e, "copy join");
}

// draw + gather + pinv + U.  Arena reserved by the caller.  With `ho`, C, R
// and the indices stream to the host while the factorizations and the X Q_R
// contraction run; U follows at the end.
int qmcur_impl(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, const double* colp, const double* rowp,
               int64_t c, int64_t r, const uint64_t state[4], int64_t* J, int64_t* I, double* C, double* U,
               double* R, int core = QCUR_CORE_PROJECTION, const HostOut* ho = nullptr, void* oz_pre = nullptr,
               void* rdig_ws = nullptr) {
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
  int rc = QCUR_OK;
  void* oz = oz_pre;
  const bool fork_late = xres_fork_after_draw();
  if (!oz && !fork_late && core == QCUR_CORE_PROJECTION && m >= c && n >= r) {
    oz = int8_fork_prepare(ctx, X, m, n, r, &rc);
    if (rc) return rc;
  }
  if (!launch_draw(jobs, 2, ctx->status_dev, st))
    return ctx->fail(QCUR_E_PARAMETER, "draw: axis longer than 2^30 entries");
  if (!oz && fork_late && core == QCUR_CORE_PROJECTION && m >= c && n >= r) {
    oz = int8_fork_prepare(ctx, X, m, n, r, &rc);  // the draws' two CTAs get their SMs first
    if (rc) return rc;
  }
  ctx->mark("draw");
  CK_LAUNCH(ctx, "draw");
  // 2. gathers (quat.py:215-225)
  launch_gather_cols(X, m, n, J, c, C, st);
  launch_gather_rows(X, n, n, I, r, R, st);
  CK_LAUNCH(ctx, "gather");
  ctx->mark("gather");
  if (rdig_ws) {  // E(R)'s digits for the error kernel depend on R alone: side stream, joined by error_impl
    cudaError_t e = cudaEventRecord(ctx->ev_sfork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->side_stream, ctx->ev_sfork, 0);
    if (e == cudaSuccess) launch_ozaki_error_rdigits(R, n, m, n, r, rdig_ws, ctx->side_stream);
    if (e == cudaSuccess) e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_rjoin, ctx->side_stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "error digits fork");
  }
  if (ho) {
    if ((rc = copy_out(ctx, C, m, c, ho->C, J, c, ho->J, I, r, ho->I))) return rc;
    if ((rc = copy_out(ctx, R, r, n, ho->R, nullptr, 0, nullptr, nullptr, 0, nullptr))) return rc;
  }
  if ((rc = qmcur_core(ctx, X, m, n, c, r, J, C, U, R, core, oz))) return rc;
  if (ho) {
    if ((rc = copy_out(ctx, U, c, r, ho->U, nullptr, 0, nullptr, nullptr, 0, nullptr))) return rc;
    if ((rc = copy_join(ctx))) return rc;
  }
  return QCUR_OK;
}

// U from the gathered C, R (projection: pinv(C) X pinv(R); intersection: pinv(R[:, J]))
void* int8_fork_prepare(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, int64_t r, int* rc) {
  *rc = QCUR_OK;
  if (!use_int8(ctx, m, n, r)) return nullptr;
  void* ozws = ctx->take<uint8_t>(ozaki_workspace_bytes(m, n, r, kOzakiModuli));
  if (!ozws) {
    *rc = ctx->fail(QCUR_E_CUDA, "workspace exhausted (int8 gemm)");
    return nullptr;
  }
  cudaError_t e = cudaEventRecord(ctx->ev_sfork, ctx->stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->side_stream, ctx->ev_sfork, 0);
  if (e == cudaSuccess && launch_ozaki_prepare(X, m, n, n, r, ctx->xq_moduli, ozws, ctx->side_stream)) {
    *rc = ctx->fail(QCUR_E_CUDA, "int8 gemm: bad modulus count");
    return nullptr;
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_sjoin, ctx->side_stream);
  if (e != cudaSuccess) {
    *rc = ctx->cuda_fail(e, "int8 fork");
    return nullptr;
  }
  return ozws;
}

// Y = X Q_R (m x r) with the engine policy of qmcur when no residues were forked: INT8 in
// one shot, INT8 in row chunks, or the FP64 DMMA GEMM (gws: its workspace, or nullptr to take it).
int xq_product(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, int64_t ldx, const double* QR, int64_t r,
               double* Y, double* gws) {
  cudaStream_t st = ctx->stream;
  const int64_t mc = int8_chunk_rows(ctx, m, n, r);
  if (use_int8(ctx, m, n, r) || mc > 0) {
    const int64_t rows = mc > 0 ? mc : m;
    void* ws = ctx->take<uint8_t>(ozaki_workspace_bytes(rows, n, r, kOzakiModuli));
    if (!ws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (int8 X Q_R)");
    if (launch_ozaki_prep_b(rows, n, QR, r, r, ctx->xq_moduli, ws, st))
      return ctx->fail(QCUR_E_CUDA, "int8 gemm: bad modulus count");
    // chunks of `rows` rows; the last one ends at row m and may overlap its predecessor (rows are
    // independent, so the overlap is recomputed to the same bits)
    for (int64_t i0 = 0; i0 < m; i0 += rows) {
      const int64_t a = i0 + rows <= m ? i0 : m - rows;
      if (launch_ozaki_prepare(X + a * ldx * 4, rows, n, ldx, r, ctx->xq_moduli, ws, st) ||
          launch_ozaki_multiply(rows, n, r, Y + a * r * 4, r, ctx->xq_moduli, ws, st))
        return ctx->fail(QCUR_E_CUDA, "int8 gemm: tensor map encode failed");
    }
    CK_LAUNCH(ctx, "int8 X Q_R");
    return QCUR_OK;
  }
  GemmArgs g = gargs(m, r, n, X, ldx, 0, QR, r, 0, Y, r);
  if (!gws) {
    gws = ctx->take<double>(qgemm_workspace_bytes(g) / 8 + 16);
    if (!gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (X Q_R)");
  }
  return gemm(ctx, g, gws);
}

int qmcur_core(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, int64_t c, int64_t r, const int64_t* J,
               const double* C, double* U, const double* R, int core, void* oz_ready) {
  cudaStream_t st = ctx->stream;
  int rc;
  if (core == QCUR_CORE_INTERSECTION) {
    // U = pinv(W), W = X[I, J] = R[:, J] (r x c): the north star's intersection core,
    // oracle pseudoinverse(x.take_rows(I).take_cols(J)) (linalg.py:346-362, quat.py:215-225)
    double* W = ctx->take<double>((size_t)(r * c * 4));
    if (!W) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (intersection)");
    launch_gather_cols(R, r, n, J, c, W, st);
    CK_LAUNCH(ctx, "gather W");
    if ((rc = pinv_impl(ctx, W, r, c, -1.0, U, ST_CHOL_FAIL_C))) return rc;
    ctx->mark("core_u");
    return QCUR_OK;
  }
  if (m >= c && n >= r) {
    double* QC = ctx->take<double>((size_t)(m * c * 4));
    double* FC = ctx->take<double>((size_t)(c * c * 4));
    double* QR = ctx->take<double>((size_t)(n * r * 4));
    double* FR = ctx->take<double>((size_t)(r * r * 4));
    double* Y = ctx->take<double>((size_t)(m * r * 4));
    double* M = ctx->take<double>((size_t)(c * r * 4));
    double* W = ctx->take<double>((size_t)(c * r * 4));
    if (!QC || !FC || !QR || !FR || !Y || !M || !W) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (qmcur)");
    // INT8 path: the residues of X depend on X alone, so they are computed on the side
    // stream while the (latency-bound) factorizations run on the main stream
    void* ozws = oz_ready;
    if (!ozws) {
      ozws = int8_fork_prepare(ctx, X, m, n, r, &rc);
      if (rc) return rc;
    }
    const bool i8 = ozws != nullptr;
    // 3. pinv(C) = F_C Q_C^H ; pinv(R) = Q_R F_R^H  (R^H = Q_R T_R)
    FactorSpec specs[2] = {FactorSpec{C, 0, m, c, ST_CHOL_FAIL_C, -1.0, FactorOut{QC, FC}},
                           FactorSpec{R, 1, n, r, ST_CHOL_FAIL_R, -1.0, FactorOut{QR, FR}}};
    if ((rc = factor_multi(ctx, specs, 2))) return rc;
    GemmArgs g1 = gargs(m, r, n, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    GemmArgs g2a = gargs(c, r, m, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
    size_t a = qgemm_workspace_bytes(g1), d = qgemm_workspace_bytes(g2a);
    double* gws = ctx->take<double>((a > d ? a : d) / 8 + 16);
    if (!gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (qmcur gemm)");
    ctx->mark("factor");
    // 4. Y = X Q_R (m x r) — the big contraction (cur.py:268)
    if (i8) {
      cudaError_t e = cudaStreamWaitEvent(st, ctx->ev_sjoin, 0);
      if (e != cudaSuccess) return ctx->cuda_fail(e, "int8 join");
      if (launch_ozaki_prep_b(m, n, QR, r, r, ctx->xq_moduli, ozws, st))
        return ctx->fail(QCUR_E_CUDA, "int8 gemm: bad modulus count");
      ctx->mark("xq_residues");  // includes the wait for the residues of X (side stream)
      if (launch_ozaki_multiply(m, n, r, Y, r, ctx->xq_moduli, ozws, st))
        return ctx->fail(QCUR_E_CUDA, "int8 gemm: tensor map encode failed");
      CK_LAUNCH(ctx, "int8 gemm");
    } else if ((rc = xq_product(ctx, X, m, n, n, QR, r, Y, gws))) {
      return rc;
    }
    ctx->mark("gemm_xq");
    // 5. M = Q_C^H Y (c x r): INT8 Hermitian product (plane products) when the engine is on
    if (i8 && use_int8_gram(ctx, m, c) && ozaki_herm_supported(m, c, r)) {
      void* ws2 = ctx->take<uint8_t>(ozaki_herm_workspace_bytes(m, c, r, 0));
      if (!ws2) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (int8 Q_C^H Y)");
      const double* A1 = QC;
      const double* B1 = Y;
      double* C1 = M;
      const int64_t p1 = m, qa1 = c, qb1 = r, lda1 = c, ldb1 = r, ldc1 = r;
      if (launch_ozaki_herm(&A1, &B1, &p1, &qa1, &qb1, &lda1, &ldb1, &C1, &ldc1, 1, ctx->herm_moduli, &ws2, st))
        return ctx->fail(QCUR_E_CUDA, "int8 Q_C^H Y: tensor map encode failed");
      CK_LAUNCH(ctx, "int8 Q_C^H Y");
    } else if ((rc = gemm(ctx, gargs(c, r, m, QC, c, 1, Y, r, 0, M, r), gws))) {
      return rc;
    }
    // 6. U = F_C M F_R^H
    if ((rc = gemm(ctx, gargs(c, r, c, FC, c, 0, M, r, 0, W, r), gws))) return rc;
    if ((rc = gemm(ctx, gargs(c, r, r, W, r, 0, FR, r, 1, U, r), gws))) return rc;
    ctx->mark("core_u");
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
    ctx->mark("core_u");
  }
  return QCUR_OK;
}

size_t error_ws_bytes(int64_t m, int64_t n, int64_t c, int64_t r) {
  (void)c;
  GemmArgs g = gargs(m, r, c, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  size_t b = qbytes(m, r) + (size_t)err_partials_count(m, n) * 32 + qgemm_workspace_bytes(g) + 4096;
  if (ozaki_error_supported(m, n, r)) b += ozaki_error_workspace_bytes(m, n, r) + 4096;
  return b;
}

int error_impl(qcur_ctx* ctx, const double* X, int64_t m, int64_t n, const double* C, int64_t c, const double* U,
               const double* R, int64_t r, double psnr_scale, double* out4, void* rdig_ws = nullptr) {
  double* P = ctx->take<double>((size_t)(m * r * 4));
  double* parts = ctx->take<double>((size_t)err_partials_count(m, n) * 4);
  GemmArgs g = gargs(m, r, c, C, c, 0, U, r, 0, P, r);
  double* gws = ctx->take<double>(qgemm_workspace_bytes(g) / 8 + 16);
  if (!P || !parts || !gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (error)");
  int rc;
  // P = C U (m x r) (cur.py:274 left product), then the fused ||X - P R|| pass
  if ((rc = gemm(ctx, g, gws))) return rc;
  ctx->mark("cu");
  if (use_int8_err(ctx, m, n, r)) {
    void* ws = rdig_ws ? rdig_ws : ctx->take<uint8_t>(ozaki_error_workspace_bytes(m, n, r));
    if (!ws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (int8 error)");
    launch_ozaki_error_digits(P, r, R, n, m, n, r, ws, ctx->stream, rdig_ws ? 0 : 1);
    if (rdig_ws) {  // E(R)'s digits were formed on the side stream after the gathers
      cudaError_t e = cudaStreamWaitEvent(ctx->stream, ctx->ev_rjoin, 0);
      if (e != cudaSuccess) return ctx->cuda_fail(e, "error digits join");
    }
    ctx->mark("error_digits");
    if (launch_ozaki_error_gemm(X, n, m, n, r, psnr_scale, ws, out4, ctx->stream))
      return ctx->fail(QCUR_E_CUDA, "int8 error: tensor map encode failed");
  } else {
    launch_cur_error(X, n, P, r, R, n, m, n, r, psnr_scale, parts, out4, ctx->stream);
  }
  ctx->mark("error");
  CK_LAUNCH(ctx, "cur_error");
  return QCUR_OK;
}

int map_status(qcur_ctx* ctx, unsigned bits) {
  ctx->last_info = bits & (ST_CHOL_FAIL_C | ST_CHOL_FAIL_R | ST_DRAW_FALLBACK);
  // K1's degenerate distribution precedes (and causes) any failed draw (cur.py:145-146 raises first)
  if (bits & ST_DEGENERATE) return ctx->fail(QCUR_E_DEGENERATE_DISTRIBUTION, "all sampling weights vanish (zero matrix)");
  if (bits & ST_SAMPLING) return ctx->fail(QCUR_E_SAMPLING, "index draw failed: not enough positive weights");
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

// Every entry point runs on its context's device and leaves the caller's current
// device as it found it (a process may drive several GPUs from one thread).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const qcur_ctx* ctx) {
    if (!ctx) return;
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != ctx->device) cudaSetDevice(ctx->device);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

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
  int prev_device = 0;
  cudaGetDevice(&prev_device);
  if (cudaSetDevice(device) != cudaSuccess) return QCUR_E_CUDA;
  // restore the caller's device however this function returns
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{prev_device};
  qcur_ctx* ctx = new qcur_ctx();
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&ctx->status_dev, 64) != cudaSuccess || cudaMallocHost(&ctx->status_host, 64) != cudaSuccess) {
    delete ctx;
    return QCUR_E_CUDA;
  }
  cudaMemset(ctx->status_dev, 0, 64);
  if (cudaMalloc(&ctx->counters, (size_t)kCounterWords * sizeof(unsigned)) != cudaSuccess) {
    delete ctx;
    return QCUR_E_CUDA;
  }
  cudaMemset(ctx->counters, 0, (size_t)kCounterWords * sizeof(unsigned));
  if (const char* xm = std::getenv("QCUR_XQ_MODULI")) ctx->xq_moduli = std::atoi(xm) == 14 ? 14 : 15;
  if (const char* hm = std::getenv("QCUR_HERM_MODULI")) ctx->herm_moduli = std::atoi(hm) == 14 ? 14 : 15;
  if (const char* gm = std::getenv("QCUR_GEMM"))
    ctx->gemm_mode = std::strcmp(gm, "dmma") == 0 ? 1 : std::strcmp(gm, "int8") == 0 ? 2 : 0;
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (const char* pe = std::getenv("QCUR_PRIO")) ctx->prio = std::strcmp(pe, "0") != 0;
  if (cudaStreamCreateWithPriority(&ctx->hi_stream, cudaStreamNonBlocking, prio_hi) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_hfork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_hjoin, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithPriority(&ctx->side_stream, cudaStreamNonBlocking, prio_lo) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_sfork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_sjoin, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_rjoin, cudaEventDisableTiming) != cudaSuccess ||
      cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming) != cudaSuccess) {
    delete ctx;
    return QCUR_E_CUDA;
  }
  *out = ctx;
  return QCUR_OK;
}

void qcur_destroy(qcur_ctx* ctx) {
  DeviceGuard device_guard_(ctx);
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  for (size_t k = 0; k < ctx->lanes.size(); ++k) {
    cudaStream_t ls = ctx->lanes[k]->stream;
    qcur_destroy(ctx->lanes[k]);
    cudaStreamDestroy(ls);
    cudaEventDestroy(ctx->lane_ev[k]);
  }
  if (ctx->ev_bfork) cudaEventDestroy(ctx->ev_bfork);
  for (auto& kv : ctx->programs) cudaFree(kv.second.buf);
  for (auto& kv : ctx->rf_sched) cudaFree(kv.second);
  if (ctx->arena.base) cudaFree(ctx->arena.base);
  cudaFree(ctx->status_dev);
  cudaFree(ctx->counters);
  cudaFreeHost(ctx->status_host);
  cudaStreamSynchronize(ctx->copy_stream);
  cudaStreamDestroy(ctx->copy_stream);
  cudaStreamSynchronize(ctx->side_stream);
  cudaStreamDestroy(ctx->side_stream);
  cudaStreamSynchronize(ctx->hi_stream);
  cudaStreamDestroy(ctx->hi_stream);
  cudaEventDestroy(ctx->ev_hfork);
  cudaEventDestroy(ctx->ev_hjoin);
  cudaEventDestroy(ctx->ev_sfork);
  cudaEventDestroy(ctx->ev_sjoin);
  cudaEventDestroy(ctx->ev_rjoin);
  cudaEventDestroy(ctx->ev_fork);
  cudaEventDestroy(ctx->ev_join);
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
  DeviceGuard device_guard_(ctx);
  if (!ctx) return QCUR_E_PARAMETER;
  ctx->stream = (cudaStream_t)s;
  return QCUR_OK;
}

// Native CUDA graphs of a captured ABI call (bench / DeviceApprox graph replays).  Replays of a graph
// run every kernel at the priority of the stream they are launched into unless the graph is
// instantiated with node priorities: the capture is closed here, every kernel node gets the
// context's high priority except the side stream's residues of X (low), and the graph is
// instantiated with cudaGraphInstantiateFlagUseNodePriority, so the latency-bound main chain (the
// draws, the cluster Cholesky) is scheduled ahead of the residue CTAs as in direct launches.
int qcur_graph_begin(qcur_ctx* ctx) {
  DeviceGuard device_guard_(ctx);
  if (!ctx) return QCUR_E_PARAMETER;
  cudaError_t e = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal);
  return e == cudaSuccess ? QCUR_OK : ctx->cuda_fail(e, "graph capture begin");
}

int qcur_graph_end(qcur_ctx* ctx, void** exec_out) {
  DeviceGuard device_guard_(ctx);
  if (!ctx || !exec_out) return QCUR_E_PARAMETER;
  *exec_out = nullptr;
  cudaGraph_t g = nullptr;
  cudaError_t e = cudaStreamEndCapture(ctx->stream, &g);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "graph capture end");
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  size_t n = 0;
  cudaGraphGetNodes(g, nullptr, &n);
  std::vector<cudaGraphNode_t> nodes(n);
  if (n) cudaGraphGetNodes(g, nodes.data(), &n);
  for (cudaGraphNode_t node : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(node, &t) != cudaSuccess || t != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp{};
    if (cudaGraphKernelNodeGetParams(node, &kp) != cudaSuccess) continue;
    cudaLaunchAttributeValue v{};
    v.priority = ozaki_side_kernel(kp.func) ? lo : hi;
    cudaGraphKernelNodeSetAttribute(node, cudaLaunchAttributePriority, &v);
  }
  (void)cudaGetLastError();
  cudaGraphExec_t ex = nullptr;
  e = cudaGraphInstantiateWithFlags(&ex, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "graph instantiate");
  *exec_out = ex;
  return QCUR_OK;
}

int qcur_graph_launch(qcur_ctx* ctx, void* exec) {
  DeviceGuard device_guard_(ctx);
  if (!ctx || !exec) return QCUR_E_PARAMETER;
  cudaError_t e = cudaGraphLaunch((cudaGraphExec_t)exec, ctx->stream);
  return e == cudaSuccess ? QCUR_OK : ctx->cuda_fail(e, "graph launch");
}

int qcur_graph_destroy(void* exec) {
  if (!exec) return QCUR_E_PARAMETER;
  return cudaGraphExecDestroy((cudaGraphExec_t)exec) == cudaSuccess ? QCUR_OK : QCUR_E_CUDA;
}

int qcur_synchronize(qcur_ctx* ctx) {
  DeviceGuard device_guard_(ctx);
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  return e == cudaSuccess ? QCUR_OK : ctx->cuda_fail(e, "synchronize");
}

int qcur_set_kappa_limit(qcur_ctx* ctx, double limit) {
  DeviceGuard device_guard_(ctx);
  if (!ctx || !(limit > 0.0)) return QCUR_E_PARAMETER;
  ctx->kappa_limit = limit;
  return QCUR_OK;
}
int qcur_force_robust(qcur_ctx* ctx, int on) {
  DeviceGuard device_guard_(ctx);
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
  DeviceGuard device_guard_(ctx);
  cudaError_t e = cudaMemcpyAsync(dst, src, bytes, (cudaMemcpyKind)kind, ctx->stream);
  return e == cudaSuccess ? QCUR_OK : ctx->cuda_fail(e, "memcpy");
}

int qcur_upload_planar(qcur_ctx* ctx, const double* a0, const double* a1, const double* a2, const double* a3,
                       int64_t m, int64_t n, double* x_dev) {
  DeviceGuard device_guard_(ctx);
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

namespace {
int upload_length_impl(qcur_ctx* ctx, const double* a0, const double* a1, const double* a2, const double* a3,
                       int64_t m, int64_t n, double* x_dev, double* col_dev, double* row_dev, int64_t xq_r,
                       void* xq_ws);
}  // namespace

int qcur_upload_length(qcur_ctx* ctx, const double* a0, const double* a1, const double* a2, const double* a3,
                       int64_t m, int64_t n, double* x_dev, double* col_dev, double* row_dev) {
  DeviceGuard device_guard_(ctx);
  return upload_length_impl(ctx, a0, a1, a2, a3, m, n, x_dev, col_dev, row_dev, 0, nullptr);
}

size_t qcur_xq_workspace_bytes(qcur_ctx* ctx, int64_t m, int64_t n, int64_t r) {
  DeviceGuard device_guard_(ctx);
  if (!ctx || m < 1 || n < 1 || r < 1 || r > m || ctx->xq_moduli != 15 || !use_int8(ctx, m, n, r)) return 0;
  return ozaki_workspace_bytes(m, n, r, 15) + 256;
}

int qcur_upload_length_xq(qcur_ctx* ctx, const double* a0, const double* a1, const double* a2, const double* a3,
                          int64_t m, int64_t n, int64_t r, double* x_dev, double* col_dev, double* row_dev,
                          void* xq_ws) {
  DeviceGuard device_guard_(ctx);
  return upload_length_impl(ctx, a0, a1, a2, a3, m, n, x_dev, col_dev, row_dev, r, xq_ws);
}

namespace {
int upload_length_impl(qcur_ctx* ctx, const double* a0, const double* a1, const double* a2, const double* a3,
                       int64_t m, int64_t n, double* x_dev, double* col_dev, double* row_dev, int64_t xq_r,
                       void* xq_ws) {
  if (m < 1 || n < 1) return ctx->fail(QCUR_E_SHAPE, "degenerate matrix shape (%lld, %lld)", (long long)m, (long long)n);
  // row chunks of ~32 MB per plane: the copy engine streams chunk k+1 while the SMs convert
  // chunk k and carry numpy's sequential column sums through it (colstrip with acc_in)
  int64_t rows = (int64_t)((32u << 20) / ((size_t)n * 8));
  if (rows < 64) rows = 64;
  if (rows > m) rows = m;
  const int64_t nchunks = (m + rows - 1) / rows;
  const size_t stage = (size_t)(rows * n);  // doubles per plane per chunk
  int rc = ctx->reserve(2 * 4 * stage * 8 + length_ws_bytes(ctx, m, n) + 4096);
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  double* buf[2][4];
  for (int b = 0; b < 2; ++b)
    for (int k = 0; k < 4; ++k) buf[b][k] = ctx->take<double>(stage);
  double* sq = ctx->take<double>((size_t)(m * n));
  double* colsum2[2] = {ctx->take<double>((size_t)n), ctx->take<double>((size_t)n)};  // ping-pong running sums
  if (!buf[1][3] || !sq || !colsum2[1]) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (upload_length)");
  cudaStream_t st = ctx->stream, cs = ctx->copy_stream;
  cudaEvent_t ev_in[2], ev_used[2];
  for (int b = 0; b < 2; ++b) {
    cudaEventCreateWithFlags(&ev_in[b], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_used[b], cudaEventDisableTiming);
  }
  // the copy stream starts after everything already queued on the main stream
  cudaEventRecord(ctx->ev_fork, st);
  cudaStreamWaitEvent(cs, ctx->ev_fork, 0);
  const double* src[4] = {a0, a1, a2, a3};
  cudaError_t e = cudaSuccess;
  for (int64_t c = 0; c < nchunks && e == cudaSuccess; ++c) {
    const int b = (int)(c & 1);
    const int64_t r0 = c * rows, nr = (m - r0) < rows ? (m - r0) : rows;
    if (c >= 2) e = cudaStreamWaitEvent(cs, ev_used[b], 0);  // staging buffer b free again
    for (int k = 0; k < 4 && e == cudaSuccess; ++k)
      e = cudaMemcpyAsync(buf[b][k], src[k] + r0 * n, (size_t)(nr * n) * 8, cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(ev_in[b], cs);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, ev_in[b], 0);
    if (e != cudaSuccess) break;
    launch_planar_to_interleaved(buf[b][0], buf[b][1], buf[b][2], buf[b][3], nr, n, x_dev + r0 * n * 4, st);
    cudaEventRecord(ev_used[b], st);
    launch_colstrip(x_dev + r0 * n * 4, nr, n, n, sq + r0 * n, colsum2[b], st, c == 0 ? nullptr : colsum2[b ^ 1]);
    // the residues of X for the INT8 X Q_R of a later qmcur on this matrix: the SMs and HBM are idle
    // while the link streams the next chunk (rows are scaled independently: chunking changes nothing)
    if (xq_ws && launch_ozaki_prepare_rows(x_dev + r0 * n * 4, nr, r0, m, n, n, xq_r, 15, xq_ws, st))
      return ctx->fail(QCUR_E_PARAMETER, "upload residues: unsupported modulus count");
  }
  double* colsum = colsum2[(nchunks - 1) & 1];
  for (int b = 0; b < 2; ++b) {
    cudaEventDestroy(ev_in[b]);
    cudaEventDestroy(ev_used[b]);
  }
  if (e != cudaSuccess) return ctx->cuda_fail(e, "upload_length H2D");
  CK_LAUNCH(ctx, "upload_length");
  if ((rc = length_tail(ctx, sq, colsum, m, n, col_dev, row_dev))) return rc;
  return sync_status(ctx);
}
}  // namespace

int qcur_download_planar(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, int64_t ld, double* a0,
                         double* a1, double* a2, double* a3) {
  DeviceGuard device_guard_(ctx);
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
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1) return ctx->fail(QCUR_E_SHAPE, "degenerate matrix shape");
  int rc = ctx->reserve(length_ws_bytes(ctx, m, n));
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  if ((rc = length_distributions_impl(ctx, x_dev, m, n, col, row))) return rc;
  return sync_status(ctx);
}

int qcur_uniform_distributions(qcur_ctx* ctx, int64_t m, int64_t n, double* col, double* row) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1) return ctx->fail(QCUR_E_PARAMETER, "dimensions must be positive, got (%lld, %lld)",
                                       (long long)m, (long long)n);
  launch_fill(col, n, 1.0 / (double)n, ctx->stream);
  launch_fill(row, m, 1.0 / (double)m, ctx->stream);
  CK_LAUNCH(ctx, "uniform");
  return QCUR_OK;
}

int qcur_draw_indices(qcur_ctx* ctx, const double* probs, int64_t size, int64_t count, uint64_t state[4],
                      int64_t* out) {
  DeviceGuard device_guard_(ctx);
  if (size < 1) return ctx->fail(QCUR_E_SHAPE, "probs must be a non-empty 1-D array");
  if (count < 1) return ctx->fail(QCUR_E_PARAMETER, "count must be positive, got %lld", (long long)count);
  int rc = ctx->reserve((size_t)draw_work_doubles(size) * 8 + 4096);
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  DrawJob job{probs, size, count, state[0], state[1], state[2], state[3], out,
              ctx->take<double>((size_t)draw_work_doubles(size))};
  if (!launch_draw(&job, 1, ctx->status_dev, ctx->stream))
    return ctx->fail(QCUR_E_PARAMETER, "draw: axis longer than 2^30 entries");
  CK_LAUNCH(ctx, "draw");
  qcur_rng_advance(state, (uint64_t)count);
  return sync_status(ctx);
}

int qcur_qmcur(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* colp, const double* rowp,
               int64_t c, int64_t r, const uint64_t state[4], int64_t* J, int64_t* I, double* C, double* U,
               double* R) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1 || c < 1 || r < 1 || c > n || r > m)
    return ctx->fail(QCUR_E_SHAPE, "qmcur: bad sizes m=%lld n=%lld c=%lld r=%lld", (long long)m, (long long)n,
                     (long long)c, (long long)r);
  int rc = ctx->reserve(qmcur_ws_bytes(m, n, c, r));
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  if ((rc = qmcur_impl(ctx, x_dev, m, n, colp, rowp, c, r, state, J, I, C, U, R))) return rc;
  return sync_status(ctx);
}

int qcur_qmcur_ex(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* colp, const double* rowp,
                  int64_t c, int64_t r, const uint64_t state[4], int core, int64_t* J, int64_t* I, double* C,
                  double* U, double* R) {
  DeviceGuard device_guard_(ctx);
  if (core != QCUR_CORE_PROJECTION && core != QCUR_CORE_INTERSECTION)
    return ctx->fail(QCUR_E_PARAMETER, "unknown core mode %d", core);
  if (m < 1 || n < 1 || c < 1 || r < 1 || c > n || r > m) return ctx->fail(QCUR_E_SHAPE, "qmcur: bad sizes");
  int rc = ctx->reserve(qmcur_ws_bytes(m, n, c, r) + qbytes(r, c) + pinv_ws_bytes(r, c));
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  if ((rc = qmcur_impl(ctx, x_dev, m, n, colp, rowp, c, r, state, J, I, C, U, R, core))) return rc;
  return sync_status(ctx);
}

int qcur_qmcur_host(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* colp,
                    const double* rowp, int64_t c, int64_t r, const uint64_t state[4], int core, int64_t* J,
                    int64_t* I, double* C, double* U, double* R, int64_t* J_host, int64_t* I_host,
                    double* const C_host[4], double* const U_host[4], double* const R_host[4]) {
  DeviceGuard device_guard_(ctx);
  if (core != QCUR_CORE_PROJECTION && core != QCUR_CORE_INTERSECTION)
    return ctx->fail(QCUR_E_PARAMETER, "unknown core mode %d", core);
  if (m < 1 || n < 1 || c < 1 || r < 1 || c > n || r > m) return ctx->fail(QCUR_E_SHAPE, "qmcur: bad sizes");
  if (!J_host || !I_host || !C_host || !U_host || !R_host) return ctx->fail(QCUR_E_PARAMETER, "null host output");
  HostOut ho{J_host, I_host, {}, {}, {}};
  for (int k = 0; k < 4; ++k) {
    ho.C[k] = C_host[k];
    ho.U[k] = U_host[k];
    ho.R[k] = R_host[k];
    if (!ho.C[k] || !ho.U[k] || !ho.R[k]) return ctx->fail(QCUR_E_PARAMETER, "null host plane");
  }
  int rc = ctx->reserve(qmcur_ws_bytes(m, n, c, r) + qbytes(r, c) + pinv_ws_bytes(r, c) + host_out_ws_bytes(m, n, c, r));
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  if ((rc = qmcur_impl(ctx, x_dev, m, n, colp, rowp, c, r, state, J, I, C, U, R, core, &ho))) {
    cudaStreamSynchronize(ctx->copy_stream);
    return rc;
  }
  return sync_status(ctx);
}

// qcur_qmcur_host whose X residues were formed at upload (qcur_upload_length_xq into xq_ws, for the same r)
int qcur_qmcur_host_xq(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* colp,
                       const double* rowp, int64_t c, int64_t r, const uint64_t state[4], int core, int64_t* J,
                       int64_t* I, double* C, double* U, double* R, int64_t* J_host, int64_t* I_host,
                       double* const C_host[4], double* const U_host[4], double* const R_host[4], void* xq_ws) {
  DeviceGuard device_guard_(ctx);
  if (core != QCUR_CORE_PROJECTION && core != QCUR_CORE_INTERSECTION)
    return ctx->fail(QCUR_E_PARAMETER, "unknown core mode %d", core);
  if (m < 1 || n < 1 || c < 1 || r < 1 || c > n || r > m) return ctx->fail(QCUR_E_SHAPE, "qmcur: bad sizes");
  if (!J_host || !I_host || !C_host || !U_host || !R_host) return ctx->fail(QCUR_E_PARAMETER, "null host output");
  HostOut ho{J_host, I_host, {}, {}, {}};
  for (int k = 0; k < 4; ++k) {
    ho.C[k] = C_host[k];
    ho.U[k] = U_host[k];
    ho.R[k] = R_host[k];
    if (!ho.C[k] || !ho.U[k] || !ho.R[k]) return ctx->fail(QCUR_E_PARAMETER, "null host plane");
  }
  // the residues are used only on the path whose policy formed them (INT8 X Q_R at this shape)
  void* oz = (xq_ws && core == QCUR_CORE_PROJECTION && ctx->xq_moduli == 15 && use_int8(ctx, m, n, r) && m >= c &&
              n >= r)
                 ? xq_ws
                 : nullptr;
  int rc = ctx->reserve(qmcur_ws_bytes(m, n, c, r) + qbytes(r, c) + pinv_ws_bytes(r, c) + host_out_ws_bytes(m, n, c, r));
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  // qmcur joins the side stream's residues through ev_sjoin: here they were formed on this stream at
  // upload, so the join event is recorded here (its previous record may belong to a graph capture)
  if (oz) {
    cudaError_t e = cudaEventRecord(ctx->ev_sjoin, ctx->stream);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "residues join");
  }
  if ((rc = qmcur_impl(ctx, x_dev, m, n, colp, rowp, c, r, state, J, I, C, U, R, core, &ho, oz))) {
    cudaStreamSynchronize(ctx->copy_stream);
    return rc;
  }
  return sync_status(ctx);
}

int qcur_cur_error(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* C, int64_t c,
                   const double* U, const double* R, int64_t r, double psnr_scale, double* out4) {
  DeviceGuard device_guard_(ctx);
  int rc = ctx->reserve(error_ws_bytes(m, n, c, r));
  if (rc) return rc;
  return error_impl(ctx, x_dev, m, n, C, c, U, R, r, psnr_scale, out4);
}

int qcur_cur_given(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const int64_t* J, int64_t c,
                   const int64_t* I, int64_t r, double* C, double* U, double* R) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1 || c < 1 || r < 1 || c > n || r > m) return ctx->fail(QCUR_E_SHAPE, "cur_given: bad sizes");
  int rc = ctx->reserve(qmcur_ws_bytes(m, n, c, r) + 4096);
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  launch_gather_cols(x_dev, m, n, J, c, C, ctx->stream);
  launch_gather_rows(x_dev, n, n, I, r, R, ctx->stream);
  CK_LAUNCH(ctx, "cur_given gather");
  if ((rc = qmcur_core(ctx, x_dev, m, n, c, r, J, C, U, R, QCUR_CORE_PROJECTION))) return rc;
  return sync_status(ctx);
}

int qcur_complex_adjoint(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, double* chi_dev) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1) return ctx->fail(QCUR_E_SHAPE, "complex_adjoint: bad sizes");
  launch_complex_adjoint(x_dev, m, n, chi_dev, ctx->stream);
  CK_LAUNCH(ctx, "complex_adjoint");
  return QCUR_OK;
}

int qcur_qgemv(qcur_ctx* ctx, int op, int64_t m, int64_t n, const double* a_dev, int64_t lda, const double* x_dev,
               double* y_dev) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1 || lda < n) return ctx->fail(QCUR_E_SHAPE, "qgemv: bad sizes");
  if (op != QCUR_OP_N && op != QCUR_OP_H) return ctx->fail(QCUR_E_PARAMETER, "qgemv: op must be N or H");
  launch_qgemv(op, a_dev, m, n, lda, x_dev, y_dev, ctx->stream);
  CK_LAUNCH(ctx, "qgemv");
  return QCUR_OK;
}

int qcur_project_observed(qcur_ctx* ctx, const double* x_dev, const double* y_dev, const unsigned char* mask_dev,
                          int64_t m, int64_t n, double* out_dev) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1) return ctx->fail(QCUR_E_SHAPE, "degenerate matrix shape");
  launch_project_observed(x_dev, y_dev, mask_dev, m, n, out_dev, ctx->stream);
  CK_LAUNCH(ctx, "project_observed");
  return QCUR_OK;
}

int qcur_complete_sweep(qcur_ctx* ctx, const double* cur_dev, const double* y_dev, const unsigned char* mask_dev,
                        int64_t m, int64_t n, int strategy, const uint64_t state[4], int64_t count,
                        const int64_t* fixed_J, const int64_t* fixed_I, int64_t* J_out, int64_t* I_out,
                        double* out_dev, double* stats4_dev) {
  DeviceGuard device_guard_(ctx);
  const int64_t c = count, r = count;
  if (m < 1 || n < 1 || c < 1 || c > n || r > m) return ctx->fail(QCUR_E_SHAPE, "complete_sweep: bad sizes");
  if ((fixed_J == nullptr) != (fixed_I == nullptr))
    return ctx->fail(QCUR_E_PARAMETER, "fixed_J and fixed_I go together");
  if (!fixed_J && strategy != QCUR_STRATEGY_LENGTH && strategy != QCUR_STRATEGY_UNIFORM)
    return ctx->fail(QCUR_E_PARAMETER, "unknown strategy %d", strategy);
  size_t need = (size_t)(m + n) * 8 + 4096 + qmcur_ws_bytes(m, n, c, r) + error_ws_bytes(m, n, c, r) +
                qbytes(m, c) + qbytes(c, r) + qbytes(r, n) + (size_t)(c + r) * 8;
  if (!fixed_J && strategy == QCUR_STRATEGY_LENGTH) need += length_ws_bytes(ctx, m, n);
  int rc = ctx->reserve(need);
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  double* C = ctx->take<double>((size_t)(m * c * 4));
  double* U = ctx->take<double>((size_t)(c * r * 4));
  double* R = ctx->take<double>((size_t)(r * n * 4));
  int64_t* J = J_out ? J_out : ctx->take<int64_t>((size_t)c);
  int64_t* I = I_out ? I_out : ctx->take<int64_t>((size_t)r);
  if (!C || !U || !R || !J || !I) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (complete)");
  cudaStream_t st = ctx->stream;
  ctx->mark_begin();
  if (fixed_J) {
    // stabilized_reconstruct (cur.py:277-286): the same projection core on given index sets
    if (J != fixed_J) cudaMemcpyAsync(J, fixed_J, (size_t)c * 8, cudaMemcpyDeviceToDevice, st);
    if (I != fixed_I) cudaMemcpyAsync(I, fixed_I, (size_t)r * 8, cudaMemcpyDeviceToDevice, st);
    launch_gather_cols(cur_dev, m, n, J, c, C, st);
    launch_gather_rows(cur_dev, n, n, I, r, R, st);
    CK_LAUNCH(ctx, "complete gather");
    if ((rc = qmcur_core(ctx, cur_dev, m, n, c, r, J, C, U, R, QCUR_CORE_PROJECTION))) return rc;
  } else {
    // make_plan(current, strategy, rank, seed, count, count) + qmcur (completion.py:207-216)
    double* colp = ctx->take<double>((size_t)n);
    double* rowp = ctx->take<double>((size_t)m);
    if (strategy == QCUR_STRATEGY_LENGTH) {
      if ((rc = length_distributions_impl(ctx, cur_dev, m, n, colp, rowp))) return rc;
    } else {
      launch_fill(colp, n, 1.0 / (double)n, st);
      launch_fill(rowp, m, 1.0 / (double)m, st);
    }
    if ((rc = qmcur_impl(ctx, cur_dev, m, n, colp, rowp, c, r, state, J, I, C, U, R))) return rc;
  }
  // approx = C U R with the observed entries restored, and the step / scale sums (completion.py:214-219)
  double* P = ctx->take<double>((size_t)(m * r * 4));
  double* parts = ctx->take<double>((size_t)err_partials_count(m, n) * 4);
  GemmArgs g = gargs(m, r, c, C, c, 0, U, r, 0, P, r);
  double* gws = ctx->take<double>(qgemm_workspace_bytes(g) / 8 + 16);
  if (!P || !parts || !gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (complete step)");
  if ((rc = gemm(ctx, g, gws))) return rc;
  launch_complete_step(cur_dev, y_dev, mask_dev, n, P, r, R, n, m, n, r, out_dev, parts, stats4_dev, st);
  CK_LAUNCH(ctx, "complete step");
  ctx->mark("complete");
  return sync_status(ctx);
}

int qcur_approx(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, int strategy, const uint64_t state[4],
                int64_t c, int64_t r, int64_t* J, int64_t* I, double* C, double* U, double* R, double psnr_scale,
                int core, double* err4) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1 || c < 1 || r < 1 || c > n || r > m) return ctx->fail(QCUR_E_SHAPE, "qcur_approx: bad sizes");
  if (strategy != QCUR_STRATEGY_LENGTH && strategy != QCUR_STRATEGY_UNIFORM)
    return ctx->fail(QCUR_E_PARAMETER, "unknown strategy %d", strategy);
  if (core != QCUR_CORE_PROJECTION && core != QCUR_CORE_INTERSECTION)
    return ctx->fail(QCUR_E_PARAMETER, "unknown core mode %d", core);
  size_t need = (size_t)(m + n) * 8 + 1024 + qmcur_ws_bytes(m, n, c, r) + error_ws_bytes(m, n, c, r) +
                qbytes(r, c) + pinv_ws_bytes(r, c);
  if (strategy == QCUR_STRATEGY_LENGTH) need += length_ws_bytes(ctx, m, n);
  int rc = ctx->reserve(need);
  if (rc) return rc;
  double* colp = ctx->take<double>((size_t)n);
  double* rowp = ctx->take<double>((size_t)m);
  // the pipeline runs on the context's high-priority stream, forked from (and joined back
  // to) the caller's stream; the residues of X start after the length pass on the low-priority side stream
  cudaStream_t user = ctx->stream;
  if (ctx->prio) {
    cudaError_t e = cudaEventRecord(ctx->ev_hfork, user);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->hi_stream, ctx->ev_hfork, 0);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "priority fork");
    ctx->stream = ctx->hi_stream;
  }
  ctx->mark_begin();
  void* oz = nullptr;
  if (!rc) {
    if (strategy == QCUR_STRATEGY_LENGTH) {
      rc = length_distributions_impl(ctx, x_dev, m, n, colp, rowp);
    } else {
      launch_fill(colp, n, 1.0 / (double)n, ctx->stream);
      launch_fill(rowp, m, 1.0 / (double)m, ctx->stream);
      ctx->mark("dists");
    }
  }
  // the residues of X fork after the length pass: overlapping it (both HBM-bound) gained nothing,
  // overlapping the latency-bound draws and factorizations does
  if (!rc && !xres_fork_after_draw() && core == QCUR_CORE_PROJECTION && m >= c && n >= r)
    oz = int8_fork_prepare(ctx, x_dev, m, n, r, &rc);
  void* rdig = nullptr;
  if (!rc && use_int8_err(ctx, m, n, r) && rdigits_early()) {
    rdig = ctx->take<uint8_t>(ozaki_error_workspace_bytes(m, n, r));
    if (!rdig) rc = ctx->fail(QCUR_E_CUDA, "workspace exhausted (int8 error)");
  }
  if (!rc) rc = qmcur_impl(ctx, x_dev, m, n, colp, rowp, c, r, state, J, I, C, U, R, core, nullptr, oz, rdig);
  if (!rc) rc = error_impl(ctx, x_dev, m, n, C, c, U, R, r, psnr_scale, err4, rdig);
  if (ctx->prio) {
    cudaError_t e = cudaEventRecord(ctx->ev_hjoin, ctx->hi_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(user, ctx->ev_hjoin, 0);
    ctx->stream = user;
    if (!rc && e != cudaSuccess) rc = ctx->cuda_fail(e, "priority join");
  }
  return rc;
}

// Batched approximations (cfg4; caller shape /root/reference/pkg/src/qcur/bench.py:346-351, one
// make_plan + qmcur per matrix): `batch` independent m x n matrices through the whole pipeline of
// qcur_approx.  Matrix b runs on lane b % L (L child contexts with their own stream, workspace and
// status word), forked from and joined back to the caller's stream, so one matrix's
// latency-bound phases (draws, Cholesky, small products) overlap the others' tensor-bound ones.
// Capturable into one CUDA graph (event fork / join only).  Lane status words are OR-ed into the
// context's own, so qcur_check reports the batch.
int qcur_approx_batched(qcur_ctx* ctx, int64_t batch, const double* const* x_devs, int64_t m, int64_t n, int strategy,
                        const uint64_t* states, int64_t c, int64_t r, int64_t* J, int64_t* I, double* C, double* U,
                        double* R, double psnr_scale, int core, double* err4, int lanes) {
  DeviceGuard device_guard_(ctx);
  if (batch < 1 || !x_devs || !states) return ctx->fail(QCUR_E_PARAMETER, "approx_batched: empty batch");
  if (lanes < 1) lanes = 4;
  if (lanes > 16) lanes = 16;
  if (lanes > batch) lanes = (int)batch;
  cudaError_t e = cudaSuccess;
  if (!ctx->ev_bfork) e = cudaEventCreateWithFlags(&ctx->ev_bfork, cudaEventDisableTiming);
  while (e == cudaSuccess && (int)ctx->lanes.size() < lanes) {
    qcur_ctx* child = nullptr;
    const int rc = qcur_create(ctx->device, &child);
    if (rc) return ctx->fail(rc, "approx_batched: lane context creation failed");
    cudaStream_t ls = nullptr;
    cudaEvent_t ev = nullptr;
    e = cudaStreamCreateWithFlags(&ls, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    child->stream = ls;
    child->gemm_mode = ctx->gemm_mode;
    child->prio = ctx->prio;
    child->kappa_limit = ctx->kappa_limit;
    child->force_robust = ctx->force_robust;
    ctx->lanes.push_back(child);
    ctx->lane_ev.push_back(ev);
  }
  if (e != cudaSuccess) return ctx->cuda_fail(e, "approx_batched lanes");
  if ((e = cudaEventRecord(ctx->ev_bfork, ctx->stream)) != cudaSuccess) return ctx->cuda_fail(e, "batch fork");
  for (int k = 0; k < lanes; ++k) {
    qcur_ctx* L = ctx->lanes[k];
    L->gemm_mode = ctx->gemm_mode;
    L->force_robust = ctx->force_robust;
    L->kappa_limit = ctx->kappa_limit;
    if ((e = cudaStreamWaitEvent(L->stream, ctx->ev_bfork, 0)) != cudaSuccess) return ctx->cuda_fail(e, "batch fork");
  }
  for (int64_t b = 0; b < batch; ++b) {
    qcur_ctx* L = ctx->lanes[b % lanes];
    const int rc = qcur_approx(L, x_devs[b], m, n, strategy, states + 4 * b, c, r, J + b * c, I + b * r,
                               C + b * m * c * 4, U + b * c * r * 4, R + b * r * n * 4, psnr_scale, core, err4 + 4 * b);
    if (rc) return ctx->fail(rc, "approx_batched: matrix %lld: %s", (long long)b, L->err.c_str());
  }
  unsigned* st[16] = {};
  for (int k = 0; k < lanes; ++k) {
    qcur_ctx* L = ctx->lanes[k];
    if ((e = cudaEventRecord(ctx->lane_ev[k], L->stream)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(ctx->stream, ctx->lane_ev[k], 0)) != cudaSuccess)
      return ctx->cuda_fail(e, "batch join");
    st[k] = L->status_dev;
  }
  launch_status_or(ctx->status_dev, st, lanes, ctx->stream);
  CK_LAUNCH(ctx, "batch status");
  return QCUR_OK;
}

int qcur_check(qcur_ctx* ctx) {
  DeviceGuard device_guard_(ctx); return sync_status(ctx); }

int qcur_status_async(qcur_ctx* ctx, unsigned* host_dst) {
  DeviceGuard device_guard_(ctx);
  cudaError_t e = cudaMemcpyAsync(host_dst, ctx->status_dev, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream);
  if (e == cudaSuccess) e = cudaMemsetAsync(ctx->status_dev, 0, sizeof(unsigned), ctx->stream);
  return e == cudaSuccess ? QCUR_OK : ctx->cuda_fail(e, "status_async");
}

int qcur_status_map(qcur_ctx* ctx, unsigned bits) {
  DeviceGuard device_guard_(ctx); return map_status(ctx, bits); }

int qcur_profile(qcur_ctx* ctx, int on) {
  DeviceGuard device_guard_(ctx);
  if (!ctx) return QCUR_E_PARAMETER;
  cudaStreamSynchronize(ctx->stream);
  ctx->prof.marks.clear();
  ctx->prof.start = nullptr;
  ctx->prof.used = 0;
  ctx->prof.acc.clear();
  ctx->prof.on = on != 0;
  ctx->prof.keep = on == 2;
  return QCUR_OK;
}

int qcur_profile_read(qcur_ctx* ctx, char* buf, size_t len) {
  DeviceGuard device_guard_(ctx);
  if (!ctx || !buf || len == 0) return QCUR_E_PARAMETER;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return ctx->cuda_fail(e, "profile sync");
  ctx->harvest();
  std::string out;
  char tmp[160];
  for (auto& kv : ctx->prof.acc) {
    snprintf(tmp, sizeof tmp, "%s:%.6f:%ld;", kv.first.c_str(), kv.second.first, kv.second.second);
    out += tmp;
  }
  snprintf(buf, len, "%s", out.c_str());
  return QCUR_OK;
}

unsigned long long qcur_launch_count(void) { return qcur::g_launches; }

// Host evaluation of the compiled pairwise program (the exact tree the K1
// kernels execute), so the plan compiler is testable without a GPU.
int qcur_pairwise_host(const double* data, int64_t n, double* out) {
  if (!data || !out || n < 0) return QCUR_E_PARAMETER;
  PairwiseProgram pp = compile_pairwise(n);
  std::vector<double> vals(pp.chunk_off.size() + pp.node_l.size());
  for (size_t ch = 0; ch < pp.chunk_off.size(); ++ch) {
    const ChunkPlan& cp = pp.plans[pp.chunk_plan[ch]];
    const double* src = data + pp.chunk_off[ch];
    std::vector<double> leaf(cp.leaf_off.size());
    for (size_t l = 0; l < cp.leaf_off.size(); ++l) {
      const double* a = src + cp.leaf_off[l];
      const int len = cp.leaf_len[l];
      double res;
      if (len < 8) {
        res = 0.0;
        for (int i = 0; i < len; ++i) res += a[i];
      } else {
        double r[8];
        for (int k = 0; k < 8; ++k) r[k] = a[k];
        int i = 8;
        for (; i < len - (len % 8); i += 8)
          for (int k = 0; k < 8; ++k) r[k] += a[i + k];
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < len; ++i) res += a[i];
      }
      leaf[l] = res;
    }
    // the level-by-level node form the device kernel executes
    const size_t nl = leaf.size();
    leaf.resize(nl + cp.node_l.size());
    for (size_t k = 0; k < cp.node_l.size(); ++k) leaf[nl + k] = leaf[cp.node_l[k]] + leaf[cp.node_r[k]];
    vals[ch] = cp.node_l.empty() ? (nl ? leaf[0] : 0.0) : leaf.back();
  }
  const size_t nch = pp.chunk_off.size();
  for (size_t k = 0; k < pp.node_l.size(); ++k) vals[nch + k] = vals[pp.node_l[k]] + vals[pp.node_r[k]];
  *out = pp.node_l.empty() ? (nch ? vals[0] : 0.0) : vals.back();
  return QCUR_OK;
}

int qcur_qgemm(qcur_ctx* ctx, int opA, int opB, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
               int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  DeviceGuard device_guard_(ctx);
  if (M < 0 || N < 0 || K < 0) return ctx->fail(QCUR_E_SHAPE, "negative gemm size");
  GemmArgs g = gargs(M, N, K, A, lda, opA, B, ldb, opB, C, ldc, alpha, beta);
  int rc = ctx->reserve(qgemm_workspace_bytes(g) + 4096);
  if (rc) return rc;
  double* ws = ctx->take<double>(qgemm_workspace_bytes(g) / 8 + 16);
  if (K == 0) {
    // C = beta C
    GemmArgs z = g;
    z.Kq = 0;
    launch_qgemm(z, ws, ctx->counters, ctx->stream);
  } else {
    launch_qgemm(g, ws, ctx->counters, ctx->stream);
  }
  CK_LAUNCH(ctx, "qgemm");
  return QCUR_OK;
}

int qcur_pseudoinverse(qcur_ctx* ctx, const double* a_dev, int64_t m, int64_t n, double tol, double* out_dev) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1) return ctx->fail(QCUR_E_SHAPE, "degenerate matrix shape");
  int rc = ctx->reserve(pinv_ws_bytes(m, n) + 4096);
  if (rc) return rc;
  if ((rc = reset_status(ctx))) return rc;
  if ((rc = pinv_impl(ctx, a_dev, m, n, tol >= 0.0 ? tol : -1.0, out_dev, ST_CHOL_FAIL_C))) return rc;
  return sync_status(ctx);
}

int qcur_frobenius_sq(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, double* out_host) {
  DeviceGuard device_guard_(ctx);
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
  DeviceGuard device_guard_(ctx);
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
  g.whole_tiles = 1;  // S(i, j) independent of the launch shape (same bits as any row block)
  double* gws = ctx->take<double>(qgemm_workspace_bytes(g) / 8 + 16);
  if (!P || !Q || !parts || !ssq || !gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (synth)");
  launch_qgemm(g, gws, ctx->counters, ctx->stream);
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

double qcur_fp64_peak_tflops(qcur_ctx* ctx) {
  DeviceGuard device_guard_(ctx); return run_dmma_peak(ctx->sms, ctx->stream); }
double qcur_int8_peak_tops(qcur_ctx* ctx) {
  DeviceGuard device_guard_(ctx); return run_i8_peak(ctx->sms, ctx->stream); }

int qcur_synth_normals(qcur_ctx* ctx, uint64_t seed, uint64_t stream, int64_t offset, int64_t count, double scale,
                       double* out_dev) {
  DeviceGuard device_guard_(ctx);
  if (offset < 0 || (offset & 1) || count < 1 || !out_dev)
    return ctx->fail(QCUR_E_PARAMETER, "synth_normals: offset must be even and non-negative, count positive");
  launch_normal_fill(out_dev, count, seed, stream, scale, ctx->stream, offset);
  CK_LAUNCH(ctx, "synth normals");
  return QCUR_OK;
}

int qcur_synth_lowrank_rows(qcur_ctx* ctx, int64_t m, int64_t n, int64_t k, uint64_t seed, double noise,
                            int64_t row0, int64_t rows, double* x_dev) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1 || k < 1 || row0 < 0 || rows < 1 || row0 + rows > m)
    return ctx->fail(QCUR_E_PARAMETER, "synth_lowrank_rows: bad sizes");
  GemmArgs gprobe = gargs(rows, n, k, nullptr, 0, 0, nullptr, 0, 1, nullptr, 0);
  int rc = ctx->reserve((size_t)qbytes(rows, k) + qbytes(n, k) + qgemm_workspace_bytes(gprobe) + 8192);
  if (rc) return rc;
  double* P = ctx->take<double>((size_t)(rows * k * 4));
  double* Q = ctx->take<double>((size_t)(n * k * 4));
  GemmArgs g = gargs(rows, n, k, P, k, 0, Q, k, 1, x_dev, n);  // S rows = P rows Q^H
  g.whole_tiles = 1;  // every row block of S has the bits of the whole-matrix generation
  double* gws = ctx->take<double>(qgemm_workspace_bytes(g) / 8 + 16);
  if (!P || !Q || !gws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (synth rows)");
  launch_normal_fill(P, rows * k * 4, seed, 1, 1.0, ctx->stream, row0 * k * 4);
  launch_normal_fill(Q, n * k * 4, seed, 2, 1.0, ctx->stream);
  launch_qgemm(g, gws, ctx->counters, ctx->stream);
  // noise relative to the analytic E||S||_F^2 = 16 k m n: sigma = noise * sqrt(4 k)
  if (noise > 0.0)
    launch_add_scaled_noise(x_dev, rows * n * 4, seed, 3, nullptr, noise * sqrt(4.0 * (double)k), ctx->stream,
                            row0 * n * 4);
  CK_LAUNCH(ctx, "synth rows");
  return QCUR_OK;
}

// ---- phase-level entry points (row-block sharded QMCUR, paper_2402_19147_b200/rowshard.py) ----
int qcur_colsums_seq(qcur_ctx* ctx, const double* x_dev, int64_t rows, int64_t n, const double* acc_in,
                     double* colsum_out, double* sq_out) {
  DeviceGuard device_guard_(ctx);
  if (rows < 1 || n < 1) return ctx->fail(QCUR_E_SHAPE, "colsums_seq: bad sizes");
  launch_colstrip(x_dev, rows, n, n, sq_out, colsum_out, ctx->stream, acc_in);
  CK_LAUNCH(ctx, "colsums_seq");
  return QCUR_OK;
}

int qcur_colsums_seq_ex(qcur_ctx* ctx, const double* x_dev, int64_t rows, int64_t ncols, int64_t ldx,
                        const double* acc_in, double* colsum_out, double* sq_out, int64_t ldsq) {
  DeviceGuard device_guard_(ctx);
  if (rows < 1 || ncols < 1 || ldx < ncols || ldsq < ncols) return ctx->fail(QCUR_E_SHAPE, "colsums_seq_ex: bad sizes");
  launch_colstrip(x_dev, rows, ncols, ldx, sq_out, colsum_out, ctx->stream, acc_in, ldsq);
  CK_LAUNCH(ctx, "colsums_seq_ex");
  return QCUR_OK;
}

int qcur_pairwise_sums(qcur_ctx* ctx, const double* data, int64_t nseg, int64_t stride, int64_t length,
                       double* out) {
  DeviceGuard device_guard_(ctx);
  if (nseg < 1 || length < 0) return ctx->fail(QCUR_E_SHAPE, "pairwise_sums: bad sizes");
  int rc = ctx->reserve(pairwise_scratch_bytes(ctx, nseg, length) + 4096);
  if (rc) return rc;
  return pairwise_sum(ctx, data, nseg, stride, length, out);
}

int qcur_vec_div(qcur_ctx* ctx, const double* in, int64_t len, const double* denom, double* out) {
  DeviceGuard device_guard_(ctx);
  launch_scale(in, len, denom, out, ctx->status_dev, ST_DEGENERATE, ctx->stream);
  CK_LAUNCH(ctx, "vec_div");
  return QCUR_OK;
}

int qcur_gather_cols(qcur_ctx* ctx, const double* x_dev, int64_t rows, int64_t n, const int64_t* J, int64_t c,
                     double* out) {
  DeviceGuard device_guard_(ctx);
  launch_gather_cols(x_dev, rows, n, J, c, out, ctx->stream);
  CK_LAUNCH(ctx, "gather_cols");
  return QCUR_OK;
}

int qcur_gather_rows(qcur_ctx* ctx, const double* x_dev, int64_t n, const int64_t* I, int64_t r, double* out) {
  DeviceGuard device_guard_(ctx);
  launch_gather_rows(x_dev, n, n, I, r, out, ctx->stream);
  CK_LAUNCH(ctx, "gather_rows");
  return QCUR_OK;
}

int qcur_qgemm_ex(qcur_ctx* ctx, int opA, int opB, int64_t M, int64_t N, int64_t K, double alpha, const double* A,
                  int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc, int flags) {
  DeviceGuard device_guard_(ctx);
  GemmArgs g = with_flags(gargs(M, N, K, A, lda, opA, B, ldb, opB, C, ldc, alpha, beta), flags & 1, (flags >> 1) & 1);
  int rc = ctx->reserve(qgemm_workspace_bytes(g) + 4096);
  if (rc) return rc;
  return gemm(ctx, g, ctx->take<double>(qgemm_workspace_bytes(g) / 8 + 16));
}

// Quaternion SVD by one-sided Jacobi (qsvd, linalg.py:226-310): A (m x n, m >= n, row pitch lda)
// is copied column-major into acm and rotated until its columns are orthogonal; then
// A V = acm (columns a_j with ||a_j|| = sigma_j), V (n x n column-major, nullable) orthonormal.
//
// Truncated (0 < k < n): the sweeps may stop before the whole matrix has converged, once the k
// columns of largest norm are certified: every one of them is orthogonal, to the rounding level
// of an inner product (sqrt(m) eps, relative), to every other column (measured directly, k_jac_cert), and the other columns'
// Frobenius norm is at most half the k-th largest column norm, so the remaining block cannot
// hold a singular value that belongs in the top k.  Those k columns then are singular triplets
// to the same accuracy as after full convergence (qsvd(x, k) returns only them).
int qcur_qsvd_jacobi_top(qcur_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda, double* acm,
                         double* vcm, double* sigma, int64_t k, int* sweeps_out) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1 || m < n) return ctx->fail(QCUR_E_SHAPE, "qsvd_jacobi: need m >= n >= 1");
  if (k < 0 || k > n) return ctx->fail(QCUR_E_PARAMETER, "qsvd_jacobi: need 0 <= k <= n");
  const bool trunc = k > 0 && k < n;
  int rc = ctx->reserve(4096 + (trunc ? (size_t)k * sizeof(int) : 0));
  if (rc) return rc;
  unsigned* flag = ctx->take<unsigned>(16);
  int* top_dev = trunc ? ctx->take<int>(k) : nullptr;
  if (!flag || (trunc && !top_dev)) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (qsvd)");
  cudaStream_t st = ctx->stream;
  launch_to_colmajor(a, m, n, lda, acm, st);
  if (vcm) launch_identity_cm(vcm, n, st);
  CK_LAUNCH(ctx, "qsvd setup");
  const int64_t rounds = jacobi_sweep_rounds(m, n);
  std::vector<double> norms(trunc ? n : 0);
  std::vector<int> order(trunc ? n : 0);
  int sweep = 0;
  for (; sweep < 60 && n > 1; ++sweep) {
    cudaMemsetAsync(flag, 0, sizeof(unsigned), st);
    for (int64_t rnd = 0; rnd < rounds; ++rnd) launch_jacobi_round(acm, m, n, vcm, rnd, flag, st);
    CK_LAUNCH(ctx, "jacobi round");
    unsigned h = 0;
    cudaError_t e = cudaMemcpyAsync(&h, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess && trunc) {
      launch_col_norms(acm, m, n, sigma, st);
      e = cudaMemcpyAsync(norms.data(), sigma, n * sizeof(double), cudaMemcpyDeviceToHost, st);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "qsvd sweep");
    if (!h) break;
    if (!trunc) continue;
    for (int64_t j = 0; j < n; ++j) order[j] = (int)j;
    std::partial_sort(order.begin(), order.begin() + k, order.end(),
                      [&](int x, int y) { return norms[x] > norms[y] || (norms[x] == norms[y] && x < y); });
    const double kth = norms[order[k - 1]];
    double rest = 0.0;
    for (int64_t j = k; j < n; ++j) rest += norms[order[j]] * norms[order[j]];
    if (!(kth > 0.0) || !(rest <= 0.25 * kth * kth)) continue;
    e = cudaMemcpyAsync(top_dev, order.data(), k * sizeof(int), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemsetAsync(flag, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "qsvd certificate");
    launch_jacobi_cert(acm, m, n, top_dev, (int)k, sigma, flag, st);
    CK_LAUNCH(ctx, "qsvd certificate");
    e = cudaMemcpyAsync(&h, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return ctx->cuda_fail(e, "qsvd certificate");
    if (!h) break;
  }
  launch_col_norms(acm, m, n, sigma, st);
  CK_LAUNCH(ctx, "qsvd norms");
  if (sweeps_out) *sweeps_out = sweep + 1;
  return QCUR_OK;
}

int qcur_qsvd_jacobi(qcur_ctx* ctx, const double* a, int64_t m, int64_t n, int64_t lda, double* acm, double* vcm,
                     double* sigma, int* sweeps_out) {
  DeviceGuard device_guard_(ctx);
  return qcur_qsvd_jacobi_top(ctx, a, m, n, lda, acm, vcm, sigma, 0, sweeps_out);
}

int qcur_set_gemm_mode(qcur_ctx* ctx, int mode) {
  DeviceGuard device_guard_(ctx);
  if (mode < 0 || mode > 2) return ctx->fail(QCUR_E_PARAMETER, "gemm mode must be 0 (auto), 1 (fp64) or 2 (int8)");
  ctx->gemm_mode = mode;
  return QCUR_OK;
}

int qcur_qgemm_herm_int8(qcur_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda,
                         const double* B, int64_t ldb, double* C, int64_t ldc) {
  DeviceGuard device_guard_(ctx);
  if (M < 1 || N < 1 || K < 1 || !ozaki_herm_supported(K, M, N))
    return ctx->fail(QCUR_E_SHAPE, "qgemm_herm_int8: bad shape");
  const int same = A == B && M == N && lda == ldb;
  const size_t wsb = ozaki_herm_workspace_bytes(K, M, N, same);
  int rc = ctx->reserve(wsb + 4096);
  if (rc) return rc;
  void* ws = ctx->take<uint8_t>(wsb);
  if (!ws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (qgemm_herm_int8)");
  if (launch_ozaki_herm(&A, &B, &K, &M, &N, &lda, &ldb, &C, &ldc, 1, kOzakiModuli, &ws, ctx->stream))
    return ctx->fail(QCUR_E_CUDA, "qgemm_herm_int8: tensor map encode failed");
  CK_LAUNCH(ctx, "qgemm_herm_int8");
  return QCUR_OK;
}

int qcur_xq(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, int64_t ldx, const double* qr_dev, int64_t r,
            double* y_dev) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1 || r < 1 || ldx < n) return ctx->fail(QCUR_E_SHAPE, "xq: bad sizes");
  const int64_t mc = int8_chunk_rows(ctx, m, n, r);
  const int64_t rows = mc > 0 ? mc : m;
  GemmArgs g = gargs(m, r, n, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  size_t b = qgemm_workspace_bytes(g) + 4096;
  if (use_int8(ctx, m, n, r) || mc > 0) b += ozaki_workspace_bytes(rows, n, r, kOzakiModuli) + 4096;
  int rc = ctx->reserve(b);
  if (rc) return rc;
  return xq_product(ctx, x_dev, m, n, ldx, qr_dev, r, y_dev, nullptr);
}

int qcur_qgemm_int8(qcur_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* A, int64_t lda, const double* B,
                    int64_t ldb, double* C, int64_t ldc, int nmod) {
  DeviceGuard device_guard_(ctx);
  if (nmod == 0) nmod = kOzakiModuli;
  if (M < 1 || N < 1 || K < 1 || !ozaki_supported(M, K, N)) return ctx->fail(QCUR_E_SHAPE, "qgemm_int8: bad shape");
  if (nmod < 14 || nmod > 15) return ctx->fail(QCUR_E_PARAMETER, "qgemm_int8: modulus count must be 14 or 15");
  const size_t wsb = ozaki_workspace_bytes(M, K, N, nmod);
  int rc = ctx->reserve(wsb + 4096);
  if (rc) return rc;
  void* ws = ctx->take<uint8_t>(wsb);
  if (!ws) return ctx->fail(QCUR_E_CUDA, "workspace exhausted (qgemm_int8)");
  if (launch_ozaki_gemm(A, M, K, lda, B, N, ldb, C, ldc, nmod, ws, ctx->stream))
    return ctx->fail(QCUR_E_CUDA, "qgemm_int8: tensor map encode failed");
  CK_LAUNCH(ctx, "qgemm_int8");
  return QCUR_OK;
}

int qcur_chol_inv(qcur_ctx* ctx, const double* G, int64_t q, double* X) {
  DeviceGuard device_guard_(ctx);
  if (q < 1) return ctx->fail(QCUR_E_SHAPE, "chol_inv: bad size");
  if (q <= chol_cluster_qmax()) {
    CholJob j{G, nullptr, X, ST_CHOL_FAIL_C};
    launch_chol_inv_cluster(&j, 1, q, ctx->status_dev, ctx->stream);
    CK_LAUNCH(ctx, "chol_inv");
    return QCUR_OK;
  }
  int rc = ctx->reserve(chol_blocked_ws_bytes(q) + 4096);
  if (rc) return rc;
  return chol_inv_blocked(ctx, G, q, X, ST_CHOL_FAIL_C);
}

int qcur_series_l2inv(qcur_ctx* ctx, const double* G2, int64_t q, double* L2inv) {
  DeviceGuard device_guard_(ctx);
  GemmArgs probe = gargs(q, q, q, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  int rc = ctx->reserve(4 * qbytes(q, q) + qgemm_workspace_bytes(probe) + 8192);
  if (rc) return rc;
  double *M0 = ctx->take<double>((size_t)(q * q * 4)), *P = ctx->take<double>((size_t)(q * q * 4));
  double *M1 = ctx->take<double>((size_t)(q * q * 4)), *P2 = ctx->take<double>((size_t)(q * q * 4));
  double* gws = ctx->take<double>(qgemm_workspace_bytes(probe) / 8 + 16);
  launch_series_lh(G2, nullptr, q, M0, ctx->status_dev, ST_CHOL_FAIL_C, 1e-5, ctx->stream);
  if ((rc = gemm(ctx, with_flags(gargs(q, q, q, M0, q, 0, M0, q, 1, P, q), 1, 1), gws))) return rc;
  launch_series_lh(G2, P, q, M1, ctx->status_dev, ST_CHOL_FAIL_C, 1e-5, ctx->stream);
  if ((rc = gemm(ctx, gargs(q, q, q, M1, q, 0, M1, q, 0, P2, q), gws))) return rc;
  launch_series_final(M1, P2, q, L2inv, ctx->stream);
  CK_LAUNCH(ctx, "series");
  return QCUR_OK;
}

// G2^{-1} ~ S = I - E + E^2, E = G2 - I (the second CholeskyQR pass of factor_multi: the factor is
// F = L1^{-H} S); raises the fast-path failure bit when max|E| > 1e-5
int qcur_series_inv(qcur_ctx* ctx, const double* G2, int64_t q, double* S) {
  DeviceGuard device_guard_(ctx);
  GemmArgs probe = gargs(q, q, q, nullptr, 0, 0, nullptr, 0, 0, nullptr, 0);
  int rc = ctx->reserve(qbytes(q, q) + qgemm_workspace_bytes(probe) + 8192);
  if (rc) return rc;
  double* E = ctx->take<double>((size_t)(q * q * 4));
  double* gws = ctx->take<double>(qgemm_workspace_bytes(probe) / 8 + 16);
  launch_series_inv_prep(G2, q, E, S, ctx->status_dev, ST_CHOL_FAIL_C, 1e-5, ctx->stream);
  CK_LAUNCH(ctx, "series prep");
  return gemm(ctx, gargs(q, q, q, E, q, 0, E, q, 0, S, q, 1.0, 1.0), gws);
}

int qcur_kappa_check(qcur_ctx* ctx, const double* G1, const double* F, int64_t q) {
  DeviceGuard device_guard_(ctx);
  launch_kappa_check(G1, F, q, ctx->kappa_limit, ctx->status_dev, ST_CHOL_FAIL_C, ctx->stream);
  CK_LAUNCH(ctx, "kappa");
  return QCUR_OK;
}

int qcur_factor(qcur_ctx* ctx, const double* src, int zh, int64_t p, int64_t q, double* Q, double* F) {
  DeviceGuard device_guard_(ctx);
  if (p < q || q < 1) return ctx->fail(QCUR_E_SHAPE, "factor: needs a tall block (p >= q)");
  int rc = ctx->reserve(factor_ws_bytes(p, q) + 4096);
  if (rc) return rc;
  return factor_tall(ctx, src, zh, p, q, ST_CHOL_FAIL_C, -1.0, FactorOut{Q, F});
}

int qcur_synth_image(qcur_ctx* ctx, int64_t m, int64_t n, int nterms, uint64_t seed, double noise_std,
                     double* x_dev) {
  DeviceGuard device_guard_(ctx);
  if (m < 1 || n < 1 || nterms < 1) return ctx->fail(QCUR_E_PARAMETER, "synth_image: bad sizes");
  const int64_t maxlen = m > n ? m : n;
  int rc = ctx->reserve((size_t)(6 * nterms * maxlen + 296 * 6) * 8 + 4096);
  if (rc) return rc;
  double* F = ctx->take<double>((size_t)(6 * nterms * maxlen));
  double* part = ctx->take<double>(296 * 6);
  launch_synth_image(m, n, nterms, seed, noise_std, F, part, x_dev, ctx->stream);
  CK_LAUNCH(ctx, "synth_image");
  return QCUR_OK;
}

}  // extern "C"
