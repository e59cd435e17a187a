/*
 * qcur_b200 — C ABI of the B200-native QMCUR hot path.
 *
 * The reference (arxiv 2402.19147, package `qcur`, pure Python) has no FFI
 * layer: its boundary is the Python functions of pkg/src/qcur/cur.py and
 * linalg.py.  Each entry point below replaces one of them; the Python mirror
 * (paper_2402_19147_b200/) binds these with ctypes and keeps the reference's
 * names, argument meaning and exceptions.  Plain pointers and sizes only.
 *
 * Conventions
 *  - Quaternion matrices on the device are INTERLEAVED, row-major: element
 *    (i, j) of an m x n matrix with leading dimension ld (in quaternions) is the
 *    four doubles at x[(i*ld + j)*4 + 0..3] = (a0, a1, a2, a3).  Host buffers
 *    use the reference's PLANAR layout (four m x n float64 planes,
 *    pkg/src/qcur/quat.py:110-143).
 *  - All calls are asynchronous on the context's stream unless they return a
 *    value that needs the device (then they synchronise that stream).
 *  - Status codes map 1:1 onto the reference exceptions (errors.py:4-29).
 *  - One context per host thread / stream; the caller owns every buffer
 *    passed in; the library owns only its workspace.
 */
#ifndef QCUR_B200_H
#define QCUR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct qcur_ctx qcur_ctx;

enum qcur_status {
  QCUR_OK = 0,
  QCUR_E_SHAPE = 1,                  /* ShapeError                  errors.py:8  */
  QCUR_E_PARAMETER = 2,              /* ParameterError              errors.py:12 */
  QCUR_E_DEGENERATE_DISTRIBUTION = 3,/* DegenerateDistributionError errors.py:20 */
  QCUR_E_SAMPLING = 4,               /* SamplingError               errors.py:24 */
  QCUR_E_CUDA = 5                    /* CUDA runtime failure / no device          */
};

enum qcur_strategy { QCUR_STRATEGY_LENGTH = 0, QCUR_STRATEGY_UNIFORM = 1 }; /* cur.py:56 STRATEGIES */
enum qcur_op { QCUR_OP_N = 0, QCUR_OP_H = 1 };                             /* op(A) = A or A^H      */
/* middle factor: the reference's U = pinv(C) X pinv(R) (cur.py:268), or the
 * north star's opt-in intersection core U = pinv(X[I, J]) */
enum qcur_core { QCUR_CORE_PROJECTION = 0, QCUR_CORE_INTERSECTION = 1 };

/* informational bits returned by qcur_last_info() */
enum qcur_info {
  QCUR_INFO_ROBUST_C = 4,     /* pinv(C) took the Householder + Jacobi path */
  QCUR_INFO_ROBUST_R = 8,     /* pinv(R) took the Householder + Jacobi path */
  QCUR_INFO_DRAW_EXACT = 16   /* a draw needed the exact sequential cumsum  */
};

/* ---- context ------------------------------------------------------------ */
int qcur_abi_version(void);
int qcur_create(int device, qcur_ctx** out);
void qcur_destroy(qcur_ctx* ctx);
const char* qcur_last_error(const qcur_ctx* ctx);
unsigned qcur_last_info(const qcur_ctx* ctx);
int qcur_set_stream(qcur_ctx* ctx, void* cuda_stream); /* cudaStream_t; NULL = legacy default */
int qcur_synchronize(qcur_ctx* ctx);
/* kappa_F limit for the CholeskyQR2 fast path of pinv (default 1e7) */
int qcur_set_kappa_limit(qcur_ctx* ctx, double limit);
int qcur_force_robust(qcur_ctx* ctx, int on); /* testing: always use Householder + Jacobi */

/* ---- numpy-compatible random stream --------------------------------------
 * np.random.default_rng(seed) (cur.py:228, 251): PCG64 seeded by SeedSequence.
 * seed is given as little-endian 32-bit words (seed 0 -> {0}).  state[4] =
 * {state_hi, state_lo, inc_hi, inc_lo}.  Host-only, no device needed. */
int qcur_rng_seed(const uint32_t* words, int nwords, uint64_t state[4]);
int qcur_rng_advance(uint64_t state[4], uint64_t delta);
int qcur_rng_random(uint64_t state[4], int64_t count, double* out);

/* qcur_upload_planar fused with qcur_length_distributions for a host matrix (make_plan's
 * first use of x, cur.py:132-150): row chunks stream in on a copy stream while the SMs
 * interleave them and carry numpy's sequential column sums through each chunk; the
 * pairwise row / flat trees follow.  Same outputs as the two calls; synchronizes. */
int qcur_upload_length(qcur_ctx* ctx, const double* a0, const double* a1, const double* a2, const double* a3,
                       int64_t m, int64_t n, double* x_dev, double* col_probs_dev, double* row_probs_dev);
/* ---- host <-> device (the e2e boundary: reference planar host buffers) --- */
int qcur_upload_planar(qcur_ctx* ctx, const double* a0, const double* a1, const double* a2, const double* a3,
                       int64_t m, int64_t n, double* x_dev);
int qcur_download_planar(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, int64_t ld, double* a0,
                         double* a1, double* a2, double* a3);
int qcur_memcpy(qcur_ctx* ctx, void* dst, const void* src, size_t bytes, int kind /* cudaMemcpyKind */);

/* ---- the QMCUR path ---------------------------------------------------- */
/* length_distributions (cur.py:132-150): bit-identical to numpy. */
int qcur_length_distributions(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, double* col_probs_dev,
                              double* row_probs_dev);
/* uniform_distributions (cur.py:153-157) */
int qcur_uniform_distributions(qcur_ctx* ctx, int64_t m, int64_t n, double* col_probs_dev, double* row_probs_dev);
/* draw_indices (cur.py:202-242): `count` distinct indices, index-exact vs numpy,
 * consuming `count` doubles of the stream `state` (advanced on return).
 * QCUR_E_PARAMETER for size > 2^30 (the 64-ary draw tree's capacity). */
int qcur_draw_indices(qcur_ctx* ctx, const double* probs_dev, int64_t size, int64_t count, uint64_t state[4],
                      int64_t* out_dev);
/* qmcur (cur.py:257-269) + plan_indices (cur.py:245-254):
 * J (num_cols) then I (num_rows) from one stream; C = X[:,J] (m x c),
 * R = X[I,:] (r x n), U = pinv(C) X pinv(R) (c x r). */
int qcur_qmcur(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* col_probs_dev,
               const double* row_probs_dev, int64_t num_cols, int64_t num_rows, const uint64_t state[4],
               int64_t* col_idx_dev, int64_t* row_idx_dev, double* c_dev, double* u_dev, double* r_dev);
/* qcur_qmcur with a choice of middle factor (enum qcur_core): projection
 * U = pinv(C) X pinv(R) (the reference) or intersection U = pinv(X[I, J]). */
int qcur_qmcur_ex(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* col_probs_dev,
                  const double* row_probs_dev, int64_t num_cols, int64_t num_rows, const uint64_t state[4], int core,
                  int64_t* col_idx_dev, int64_t* row_idx_dev, double* c_dev, double* u_dev, double* r_dev);
/* qcur_qmcur_ex that also delivers the factors to host memory in the reference's
 * planar layout (four float64 planes per matrix, quat.py:110-143): C, R and the
 * indices stream out on a copy stream while the factorizations and the X Q_R
 * contraction run; U follows.  Host buffers should be pinned for the overlap.
 * The device outputs are written as in qcur_qmcur_ex.  Returns after the copies. */
int qcur_qmcur_host(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* col_probs_dev,
                    const double* row_probs_dev, int64_t num_cols, int64_t num_rows, const uint64_t state[4],
                    int core, int64_t* col_idx_dev, int64_t* row_idx_dev, double* c_dev, double* u_dev,
                    double* r_dev, int64_t* col_idx_host, int64_t* row_idx_host, double* const c_host[4],
                    double* const u_host[4], double* const r_host[4]);
/* C = X[:, J], R = X[I, :], U = pinv(C) X pinv(R) for given index sets: the factors of
 * stabilized_reconstruct (cur.py:277-286).  J, I: device int64. */
int qcur_cur_given(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const int64_t* col_idx_dev,
                   int64_t num_cols, const int64_t* row_idx_dev, int64_t num_rows, double* c_dev, double* u_dev,
                   double* r_dev);
/* y = op(A) x for a quaternion m x n matrix and quaternion vectors (op: QCUR_OP_N -> y in H^m,
 * QCUR_OP_H -> y in H^n): the products of the Krylov spectral norm (spectral_norm,
 * linalg.py:365-367).  HBM-bound, fixed reduction order. */
int qcur_qgemv(qcur_ctx* ctx, int op, int64_t m, int64_t n, const double* a_dev, int64_t lda, const double* x_dev,
               double* y_dev);
/* ---- low-rank completion (Algorithm 2; completion.py) ---- */
/* out = mask ? y : x elementwise (project_observed, completion.py:101-111); mask: m x n bytes,
 * nonzero = observed. */
int qcur_project_observed(qcur_ctx* ctx, const double* x_dev, const double* y_dev, const unsigned char* mask_dev,
                          int64_t m, int64_t n, double* out_dev);
/* One completion sweep on the device iterate cur (completion.py:204-219): sample count rows and
 * columns (make_plan with `strategy` and the PCG64 `state`, or the given fixed index sets for
 * index_policy "fixed" = stabilized_reconstruct), reconstruct C U R, restore the observed entries
 * into out_dev and return stats4_dev = {||out - cur||_F^2, ||cur||_F^2, 0, 0}.  J_out / I_out
 * (nullable, device) receive the index sets.  Synchronizes; maps degenerate draws to status codes. */
int qcur_complete_sweep(qcur_ctx* ctx, const double* cur_dev, const double* y_dev, const unsigned char* mask_dev,
                        int64_t m, int64_t n, int strategy, const uint64_t state[4], int64_t count,
                        const int64_t* fixed_J, const int64_t* fixed_I, int64_t* J_out, int64_t* I_out,
                        double* out_dev, double* stats4_dev);
/* Error statistics of X - C U R without forming CUR (callers: cli.py:173-175,
 * bench.py:257-258, imaging.py:170-177).  out4_dev (4 doubles, device):
 *   [0] ||X - CUR||_F^2   [1] ||X||_F^2   [2] imaginary-part ||X - CUR||^2 (float PSNR)
 *   [3] sum of squared differences of the u8 images qmat_to_image(s X) and
 *       qmat_to_image(s CUR) (imaging.py:90-124; exact integers) when psnr_scale s > 0 */
int qcur_cur_error(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* c_dev, int64_t c,
                   const double* u_dev, const double* r_dev, int64_t r, double psnr_scale, double* out4_dev);
/* One whole approximation, device resident, no host synchronisation:
 * distributions (strategy) + draw + gather + pinv + U + fused error. */
int qcur_approx(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, int strategy, const uint64_t state[4],
                int64_t num_cols, int64_t num_rows, int64_t* col_idx_dev, int64_t* row_idx_dev, double* c_dev,
                double* u_dev, double* r_dev, double psnr_scale, int core, double* err4_dev);
/* Batched: `batch` independent m x n matrices x_devs[b] (device pointers, host array) through the
 * pipeline of qcur_approx, matrix b with PCG64 state states[4b..4b+3]; outputs packed per matrix
 * (col_idx batch x num_cols, c batch x m x num_cols, ..., err4 batch x 4).  Matrices run on `lanes`
 * (1..16; 0 = 4) internal lane contexts overlapping one another; fork/join on the context stream,
 * capturable into one CUDA graph.  The caller's shape: the per-matrix make_plan + qmcur loop of
 * the reference's scaling experiment (pkg/src/qcur/bench.py:346-351). */
int qcur_approx_batched(qcur_ctx* ctx, int64_t batch, const double* const* x_devs, int64_t m, int64_t n, int strategy,
                        const uint64_t* states, int64_t num_cols, int64_t num_rows, int64_t* col_idx_dev,
                        int64_t* row_idx_dev, double* c_dev, double* u_dev, double* r_dev, double psnr_scale,
                        int core, double* err4_dev, int lanes);
/* read back and clear the device status word; returns the mapped status code */
int qcur_check(qcur_ctx* ctx);
/* Asynchronous status: queue a copy of the context's status word to host_dst (pinned) and
 * clear it, both on the context stream (no synchronisation); after the stream reached that
 * point, qcur_status_map turns the word into the status code qcur_check would have returned. */
int qcur_status_async(qcur_ctx* ctx, unsigned* host_dst);
int qcur_status_map(qcur_ctx* ctx, unsigned bits);

/* ---- linear algebra used by the path -------------------------------------- */
/* qmat_matmul (quat.py:274-296): C = alpha op(A) op(B) + beta C, sizes in quaternions */
int qcur_qgemm(qcur_ctx* ctx, int opA, int opB, int64_t M, int64_t N, int64_t K, double alpha, const double* a_dev,
               int64_t lda, const double* b_dev, int64_t ldb, double beta, double* c_dev, int64_t ldc);
/* pseudoinverse (linalg.py:346-362); tol < 0 -> default eps*max(m,n)*sigma_max */
int qcur_pseudoinverse(qcur_ctx* ctx, const double* a_dev, int64_t m, int64_t n, double tol, double* out_dev);
/* qmat_frobenius_norm^2 (quat.py:305-307) */
int qcur_frobenius_sq(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, double* out_host);

/* ---- synthetic BASELINE workloads and the FP64 roofline probe ------------ */
/* X = P Q^H + N, P (m x k), Q (n x k), components i.i.d. N(0,1) (Philox).
 * noise_relative != 0: noise std = noise * ||S||_F / sqrt(4mn); else std = noise. */
int qcur_synth_lowrank(qcur_ctx* ctx, int64_t m, int64_t n, int64_t k, uint64_t seed, double noise,
                       int noise_relative, double* x_dev);
double qcur_fp64_peak_tflops(qcur_ctx* ctx);
double qcur_int8_peak_tops(qcur_ctx* ctx); /* dense tcgen05 kind::i8 rate, TOP/s (roofline of the INT8 kernels) */
/* Rows [row0, row0+rows) of the m x n matrix P Q^H + N with noise std
 * noise * sqrt(4k) (relative to the analytic E||S||_F^2 = 16 k m n), so every
 * rank of a row-sharded run generates exactly its block of the same matrix. */
int qcur_synth_lowrank_rows(qcur_ctx* ctx, int64_t m, int64_t n, int64_t k, uint64_t seed, double noise,
                            int64_t row0, int64_t rows, double* x_dev);
/* The generator stream itself: out[t] = scale * z(offset + t), z the standard normals of
 * Philox4x32-10 keyed by `seed`, counter (pair index, stream) and Box-Muller on 53-bit
 * uniforms (`offset` even).  Streams: 1 = P, 2 = Q, 3 = noise, in element order.  For
 * host restatements / spot checks of any block of a generated matrix. */
int qcur_synth_normals(qcur_ctx* ctx, uint64_t seed, uint64_t stream, int64_t offset, int64_t count, double scale,
                       double* out_dev);
/* cfg3 image-like pure quaternion matrix: each imaginary plane = sum of `nterms`
 * separable products of random cosine series (frequencies U[0,8]), min-max to
 * [0,1], quantised to 1/255, plus N(0, noise_std^2); real part 0. */
int qcur_synth_image(qcur_ctx* ctx, int64_t m, int64_t n, int nterms, uint64_t seed, double noise_std,
                     double* x_dev);

/* ---- phase-level entry points for the row-block sharded path ------------------
 * Used by paper_2402_19147_b200/rowshard.py, which interleaves them with NCCL
 * collectives.  All asynchronous on the context stream; failures
 * of the fast factorisation raise the status bit read back by qcur_check() /
 * qcur_last_info() (QCUR_INFO_ROBUST_C). */
/* sq of a row block and numpy's sequential column sums continued from acc_in (nullable) */
int qcur_colsums_seq(qcur_ctx* ctx, const double* x_dev, int64_t rows, int64_t n, const double* acc_in_dev,
                     double* colsum_out_dev, double* sq_out_dev);
/* The same over a slice of columns: x_dev points at the slice's first column (row pitch ldx
 * quaternions), sq_out at its first column in the full sq rows (pitch ldsq): the row-sharded
 * path pipelines numpy's sequential column chain across ranks chunk by chunk. */
int qcur_colsums_seq_ex(qcur_ctx* ctx, const double* x_dev, int64_t rows, int64_t ncols, int64_t ldx,
                        const double* acc_in, double* colsum_out, double* sq_out, int64_t ldsq);
/* numpy pairwise sums of nseg segments of `length` doubles (stride apart) */
int qcur_pairwise_sums(qcur_ctx* ctx, const double* data_dev, int64_t nseg, int64_t stride, int64_t length,
                       double* out_dev);
int qcur_vec_div(qcur_ctx* ctx, const double* in_dev, int64_t len, const double* denom_dev, double* out_dev);
int qcur_gather_cols(qcur_ctx* ctx, const double* x_dev, int64_t rows, int64_t n, const int64_t* J_dev, int64_t c,
                     double* out_dev);
int qcur_gather_rows(qcur_ctx* ctx, const double* x_dev, int64_t n, const int64_t* I_dev, int64_t r, double* out_dev);
/* qgemm with structure flags: 1 = op(B) upper triangular, 2 = Hermitian output (lower triangle only) */
int qcur_qgemm_ex(qcur_ctx* ctx, int opA, int opB, int64_t M, int64_t N, int64_t K, double alpha, const double* a_dev,
                  int64_t lda, const double* b_dev, int64_t ldb, double beta, double* c_dev, int64_t ldc, int flags);
/* X = L^{-1} for G = L L^H (cluster kernel, or blocked for q > 304) */
/* Quaternion SVD core (qsvd, linalg.py:226-310; numerical_rank :370-378): one-sided Jacobi on
   A (m x n, m >= n, row pitch lda, interleaved).  acm_dev (m x n column-major) receives A V, whose
   column norms are the singular values (sigma_dev, unsorted); vcm_dev (n x n column-major,
   nullable) receives V.  sweeps_out (nullable): Jacobi sweeps used. */
int qcur_qsvd_jacobi(qcur_ctx* ctx, const double* a_dev, int64_t m, int64_t n, int64_t lda, double* acm_dev,
                     double* vcm_dev, double* sigma_dev, int* sweeps_out);
/* Truncated variant for qsvd(x, k) (linalg.py:226-310): same outputs, but with 0 < k < n the sweeps
   stop as soon as the k largest columns of A V are certified to be singular triplets (each orthogonal
   to every other column to max(4, sqrt(m)) eps relative; the rest's Frobenius norm at most half the k-th
   largest).  k = 0 or k = n: full convergence, as qcur_qsvd_jacobi. */
int qcur_qsvd_jacobi_top(qcur_ctx* ctx, const double* a_dev, int64_t m, int64_t n, int64_t lda, double* acm_dev,
                         double* vcm_dev, double* sigma_dev, int64_t k, int* sweeps_out);
/* Engine of the X Q_R contraction inside qmcur: 0 auto (INT8 when large), 1 FP64 DMMA, 2 INT8 (Ozaki II).
   The environment variable QCUR_GEMM=dmma|int8 sets the initial mode of new contexts. */
int qcur_set_gemm_mode(qcur_ctx* ctx, int mode);
/* C (M x N) = A^H B with A (K x M), B (K x N): the Hermitian products of CholeskyQR2 and the core
   (Z^H Z, Q_C^H Y) on the INT8 tensor cores as 16 real plane products (exact modular arithmetic). */
int qcur_qgemm_herm_int8(qcur_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* a_dev, int64_t lda,
                         const double* b_dev, int64_t ldb, double* c_dev, int64_t ldc);
/* C (M x N) = A (M x K) * B (K x N), op N, on the INT8 tensor cores by exact modular arithmetic
   (Ozaki scheme II, nmod moduli; 0 = default).  Same contract as qcur_qgemm with alpha = 1, beta = 0. */
int qcur_qgemm_int8(qcur_ctx* ctx, int64_t M, int64_t N, int64_t K, const double* a_dev, int64_t lda,
                    const double* b_dev, int64_t ldb, double* c_dev, int64_t ldc, int nmod);
/* Y (m x r) = X (m x n, row pitch ldx) Q_R (n x r): the big contraction of qmcur (cur.py:268) with
   qmcur's engine policy: INT8 in one shot, INT8 one chunk of rows at a time when the residue planes
   exceed the one-shot workspace (cfg5), else the FP64 DMMA GEMM.  Used by the row-sharded path. */
int qcur_xq(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, int64_t ldx, const double* qr_dev, int64_t r,
            double* y_dev);
/* to_complex_adjoint (linalg.py:151-164): chi(A), 2m x 2n complex128 row-major (re, im interleaved) */
int qcur_complex_adjoint(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, double* chi_dev);
int qcur_chol_inv(qcur_ctx* ctx, const double* g_dev, int64_t q, double* x_dev);
/* second CholeskyQR pass: L2^{-1} of G2 = I + E by series */
int qcur_series_l2inv(qcur_ctx* ctx, const double* g2_dev, int64_t q, double* l2inv_dev);
/* S = I - E + E^2 ~ G2^{-1} with E = G2 - I (the second CholeskyQR pass: F = L1^{-H} S) */
int qcur_series_inv(qcur_ctx* ctx, const double* g2_dev, int64_t q, double* s_dev);
int qcur_kappa_check(qcur_ctx* ctx, const double* g1_dev, const double* f_dev, int64_t q);
/* local factorisation of a tall block Z = src (zh=0) or src^H (zh=1): pinv(Z) = F Q^H */
int qcur_factor(qcur_ctx* ctx, const double* src_dev, int zh, int64_t p, int64_t q, double* q_dev, double* f_dev);

/* ---- measurement hooks (bench.py) ------------------------------------------
 * qcur_profile(ctx, 1) records CUDA events on the context stream at the end of
 * every pipeline phase (length, draw, gather, factor_c, factor_r, gemm_xq,
 * core_u, cu, error); qcur_profile_read synchronises and writes
 * "phase:total_ms:count;..." into buf.  qcur_profile(ctx, 2): the same, for a
 * call captured into a CUDA graph (the phase events become external event
 * nodes); the marks persist, so call qcur_profile_read after every replay.
 * qcur_launch_count is the number of kernels this library has launched in the
 * process. */
/* CUDA graphs of captured calls with node priorities (the main chain high, the side stream's
 * residues of X low), instantiated with cudaGraphInstantiateFlagUseNodePriority:
 * qcur_graph_begin starts capturing the context stream (not the legacy default stream), the
 * captured ABI calls follow, qcur_graph_end closes the capture and returns the executable graph,
 * qcur_graph_launch replays it on the context stream, qcur_graph_destroy frees it. */
/* The drop-in path with the INT8 X Q_R's residues of X formed while X uploads (make_plan on a host
 * matrix, then qmcur with the same r): qcur_xq_workspace_bytes gives the device workspace the residues
 * live in (0: the shape does not take the INT8 X Q_R), qcur_upload_length_xq is qcur_upload_length that
 * also fills it, and qcur_qmcur_host_xq is qcur_qmcur_host that consumes it instead of forming the
 * residues itself.  Same results as the plain calls (identical residues). */
size_t qcur_xq_workspace_bytes(qcur_ctx* ctx, int64_t m, int64_t n, int64_t r);
int qcur_upload_length_xq(qcur_ctx* ctx, const double* a0, const double* a1, const double* a2, const double* a3,
                          int64_t m, int64_t n, int64_t r, double* x_dev, double* col_dev, double* row_dev,
                          void* xq_ws);
int qcur_qmcur_host_xq(qcur_ctx* ctx, const double* x_dev, int64_t m, int64_t n, const double* col_probs_dev,
                       const double* row_probs_dev, int64_t num_cols, int64_t num_rows, const uint64_t state[4],
                       int core, int64_t* col_idx_dev, int64_t* row_idx_dev, double* c_dev, double* u_dev,
                       double* r_dev, int64_t* col_idx_host, int64_t* row_idx_host, double* const c_host[4],
                       double* const u_host[4], double* const r_host[4], void* xq_ws);
int qcur_graph_begin(qcur_ctx* ctx);
int qcur_graph_end(qcur_ctx* ctx, void** exec_out);
int qcur_graph_launch(qcur_ctx* ctx, void* exec);
int qcur_graph_destroy(void* exec);
int qcur_profile(qcur_ctx* ctx, int on);
int qcur_profile_read(qcur_ctx* ctx, char* buf, size_t len);
unsigned long long qcur_launch_count(void);
/* Host evaluation of the numpy pairwise-summation program the K1 kernels run
 * (cur.py:144, 148, 150 orders); test hook, no device needed. */
int qcur_pairwise_host(const double* data, int64_t n, double* out);

#ifdef __cplusplus
}
#endif
#endif /* QCUR_B200_H */
