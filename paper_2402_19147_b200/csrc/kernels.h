// Internal launcher interface between the C-ABI orchestration (qcur_abi.cu)
// and the kernel translation units.  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace qcur {

struct DevPairwise {
  int64_t length;
  int32_t nchunks, nnodes, maxh, max_chunk_len;
  const int64_t* chunk_off;
  const int32_t* chunk_plan;
  const int32_t* plan_len;
  const int32_t* plan_leaf_ptr;
  const int32_t* plan_prog_ptr;
  const int32_t* leaf_off;
  const int32_t* leaf_len;
  const int32_t* prog;
  const int32_t* node_l;
  const int32_t* node_r;
  const int32_t* level_ptr;
  // chunk trees level by level (ChunkPlan::node_l/node_r/lvl, concatenated over plans)
  const int32_t* plan_node_ptr;
  const int32_t* plan_lvl_ptr;
  const int32_t* cnode_l;
  const int32_t* cnode_r;
  const int32_t* clvl;
};

// k_norms.cu
// ldsq: row pitch of sq (0 = n): a column slice of X writes its slice of the full sq rows
void launch_colstrip(const double* X, int64_t m, int64_t n, int64_t ldx, double* sq, double* colsum, cudaStream_t st,
                     const double* acc_in = nullptr, int64_t ldsq = 0);
void launch_pairwise(const double* data, int64_t nseg, int64_t seg_stride, const DevPairwise& pw, double* scratch,
                     double* out, cudaStream_t st, bool with_top = true, bool reverse = false);
// fused tail of the length distributions (axes of one pairwise chunk; see k_norms.cu)
void launch_rows_flat(const double* sq, int64_t m, int64_t n, const DevPairwise& rpw, const DevPairwise& fpw,
                      const int32_t* sched, double* rowsum, double* flat, cudaStream_t st);
bool finalize_supported(const DevPairwise& fpw, const DevPairwise& cpw, const DevPairwise& rpw);
void launch_finalize(const double* flat, const DevPairwise& fpw, const double* colsum, const DevPairwise& cpw,
                     double* col, const double* rowsum, const DevPairwise& rpw, double* row, unsigned* status,
                     cudaStream_t st);
void launch_scale(const double* in, int64_t len, const double* denom, double* out, unsigned* status,
                  unsigned check_bit, cudaStream_t st);
void launch_fill(double* out, int64_t len, double v, cudaStream_t st);

// k_draw.cu
struct DrawJob {
  const double* probs;  // [len]
  int64_t len;
  int64_t count;
  uint64_t st_hi, st_lo, inc_hi, inc_lo;  // PCG64 state at the first uniform of this job
  int64_t* out;                           // [count]
  double* work;                           // >= draw_work_doubles(len)
};
int64_t draw_work_doubles(int64_t len);
// njobs <= 2; false (nothing launched) for an axis longer than the draw tree holds (64^5 entries)
bool launch_draw(const DrawJob* jobs_host, int njobs, unsigned* status, cudaStream_t st);

// k_layout.cu
void launch_planar_to_interleaved(const double* a0, const double* a1, const double* a2, const double* a3, int64_t m,
                                  int64_t n, double* X, cudaStream_t st);
void launch_interleaved_to_planar(const double* X, int64_t m, int64_t n, int64_t ldx, double* a0, double* a1,
                                  double* a2, double* a3, cudaStream_t st);
void launch_gather_cols(const double* X, int64_t m, int64_t ldx, const int64_t* J, int64_t c, double* C,
                        cudaStream_t st);
void launch_gather_rows(const double* X, int64_t n, int64_t ldx, const int64_t* I, int64_t r, double* R,
                        cudaStream_t st);
void launch_status_or(unsigned* dst, unsigned* const* srcs, int n, cudaStream_t st);
void launch_complex_adjoint(const double* X, int64_t m, int64_t n, double* chi, cudaStream_t st);
void launch_conj_transpose(const double* A, int64_t m, int64_t n, int64_t lda, double* AH, int64_t ldah,
                           cudaStream_t st);
void launch_reduce_pairs(const double* parts, int64_t nparts, double* out2, cudaStream_t st);
void launch_reduce_rows(const double* parts, int64_t nrows, int width, double* out, cudaStream_t st);  // width <= 8

// k_qgemm.cu : C(Mq x Nq) = alpha * op(A) * op(B) + beta * C, quaternion, interleaved.
// op: 0 = N, 1 = H (conjugate transpose).  lda/ldb/ldc in quaternions.
struct GemmArgs {
  int64_t Mq, Nq, Kq;
  const double* A;
  int64_t lda;
  int opA;
  const double* B;
  int64_t ldb;
  int opB;
  double* C;
  int64_t ldc;
  double alpha, beta;
  int b_upper = 0;     // op(B) upper triangular (skip k > j)
  int herm_lower = 0;  // Hermitian output, only the lower triangle is produced / consumed
  int whole_tiles = 0;  // every output tile summed by one CTA over k in order: an element's value does not
                        // depend on M (row blocks of a generated matrix concatenate bit for bit)
};
size_t qgemm_workspace_bytes(const GemmArgs& g);
// small products (N, K <= 256 and M <= 256 or M N K <= 1.2e7 quaternion MACs, not whole_tiles):
// launch_qgemm / launch_qgemm_pair route them to k_qgemm_small (no workspace or counters used)
bool qgemm_small_ok(const GemmArgs& g);
void launch_qgemm_small(const GemmArgs* g, int np, cudaStream_t st);
// counters: >= 65536 zero-initialised uints owned by the caller (split-K tickets)
void launch_qgemm(const GemmArgs& g, double* workspace, unsigned* counters, cudaStream_t st);
// two independent products in one launch (SMs split by work); falls back to two launches
// when their ops or tile configurations differ.  Tile counts < 32768 each.
void launch_qgemm_pair(const GemmArgs& g0, double* ws0, const GemmArgs& g1, double* ws1, unsigned* counters,
                       cudaStream_t st);
// Fused error of X - P R (P: m x r, R: r x n, X: m x n, all interleaved).  out4 =
// {||X-PR||^2, ||X||^2, imaginary part of ||X-PR||^2, u8-image squared-diff sum at psnr_scale}
int64_t err_partials_count(int64_t m, int64_t n);  // tiles; the partial buffer needs 4 doubles per tile
void launch_cur_error(const double* X, int64_t ldx, const double* P, int64_t ldp, const double* R, int64_t ldr,
                      int64_t m, int64_t n, int64_t r, double psnr_scale, double* partials, double* out4,
                      cudaStream_t st);

// Completion sweep (completion.py:214-219): out = mask ? Y : P R (m x n), out4 = {sum (out - X)^2, sum X^2, 0, 0};
// X, Y, out share the row pitch ld (quaternions); mask is m x n bytes.  partials: err_partials_count(m, n) * 4.
void launch_complete_step(const double* X, const double* Y, const unsigned char* mask, int64_t ld, const double* P,
                          int64_t ldp, const double* R, int64_t ldr, int64_t m, int64_t n, int64_t r, double* out,
                          double* partials, double* out4, cudaStream_t st);
// out = mask ? Y : X elementwise (project_observed, completion.py:101-111)
void launch_project_observed(const double* X, const double* Y, const unsigned char* mask, int64_t m, int64_t n,
                             double* out, cudaStream_t st);

// k_gemv.cu : y = op(A) x for quaternion vectors (op 0 = N, 1 = H), HBM-bound, deterministic
void launch_qgemv(int op, const double* A, int64_t m, int64_t n, int64_t lda, const double* x, double* y,
                  cudaStream_t st);

// k_dense.cu : small (q x q) dense factorizations, one CTA each.
void launch_cholesky(double* G, int64_t q, int64_t ldg, unsigned* status, unsigned fail_bit, cudaStream_t st);
void launch_tri_inverse_lower(const double* L, int64_t q, int64_t ldl, double* Linv, int64_t ldi, cudaStream_t st);
void launch_set_identity(double* A, int64_t q, int64_t lda, cudaStream_t st);
void launch_set_status(unsigned* status, unsigned bits, cudaStream_t st);
void launch_kappa_check(const double* G1, const double* Tinv, int64_t q, double limit, unsigned* status,
                        unsigned fail_bit, cudaStream_t st);

// k_chol_cluster.cu : Cholesky + inverse of up to two q x q Grams on 16-CTA clusters
struct CholJob {
  const double* G;  // q x q Hermitian (lower read)
  double* L;        // out: Cholesky factor (upper zeroed)
  double* X;        // out: L^{-1} (upper zeroed)
  unsigned fail_bit;
};
int chol_cluster_qmax();
// second CholeskyQR pass by series (k_dense.cu): M = lh(G2 - I - P) (P may be null; then also
// checks max|G2 - I| <= thresh), L2inv = I - M1 + P2
void launch_series_lh(const double* G2, const double* P, int64_t q, double* M, unsigned* status, unsigned fail_bit,
                      double thresh, cudaStream_t st);
void launch_series_final(const double* M1, const double* P2, int64_t q, double* L2inv, cudaStream_t st);
// E = G2 - I and S = I - E, both full (from G2's lower triangle); fail_bit when max|E| > thresh
struct SeriesKappaJob {
  const double* G2;   // second Gram (lower triangle read)
  const double* G1;   // first Gram (diagonal read: trace)
  const double* L1i;  // L1^{-1} (kappa guard)
  double* E;
  double* S;
  double* partials;  // [2 * series_kappa_blocks(q)]
  int64_t q;
  unsigned fail_bit;
};
struct SeriesKappaJobs {
  SeriesKappaJob j[2];
};
int series_kappa_blocks(int64_t q);
// k_series_inv_prep + k_kappa_check of up to two blocks in one launch; tickets[0..nj) zero between launches
void launch_series_kappa(const SeriesKappaJobs& J, int nj, unsigned* status, unsigned* tickets, double thresh,
                         double limit, cudaStream_t st);
void launch_series_inv_prep(const double* G2, int64_t q, double* E, double* S, unsigned* status, unsigned fail_bit,
                            double thresh, cudaStream_t st);
void launch_chol_inv_cluster(const CholJob* jobs, int njobs, int64_t q, unsigned* status, cudaStream_t st);
// robust path (runs only when `status & gate_bit`, otherwise returns immediately)
// robust factor on a 16-CTA cluster (k_robust.cu): one-sided Jacobi on Zcm (p x q, column-major, overwritten),
// Q = W (row-major, ld ldq), F = V Sigma^+ (row-major, ld ldf); gated on `status & gate_bit`
// robust factorization by Householder QR + one-sided Jacobi pinv of the triangular factor, both on
// 16-CTA clusters (k_robust.cu): Q (p x q row-major), F = T^+ (q x q row-major); gated on gate_bit
bool robust_qr_supported(int64_t p, int64_t q);
struct RobustQrJob {
  double* Zcm;
  int64_t p, q;
  double* betas;
  double* Ycm;
  double* Q;
  int64_t ldq;
  double* Tcm;
  double* Vcm;
  double* F;
  int64_t ldf;
  double cutoff_scale, cutoff_abs;
  const unsigned* status;
  unsigned gate_bit;
};
// launch_robust_qr_pinv for up to two blocks (each gated on its own bit) in two launches
void launch_robust_qr_pinv_multi(const RobustQrJob* J, int nj, cudaStream_t st);
// row-major -> column-major copies of up to two blocks in one launch (each gated on its bit)
void launch_rowmajor_to_colmajor2(const double* const* Z, const int64_t* p, const int64_t* q, const int64_t* ldz,
                                  double* const* Zcm, int nj, const unsigned* status, const unsigned* gate_bit,
                                  cudaStream_t st);

void launch_robust_qr_pinv(double* Zcm, int64_t p, int64_t q, double* betas, double* Ycm, double* Q, int64_t ldq,
                           double* Tcm, double* Vcm, double* F, int64_t ldf, double cutoff_scale, double cutoff_abs,
                           const unsigned* status, unsigned gate_bit, cudaStream_t st);
void launch_robust_jacobi(double* Zcm, int64_t p, int64_t q, double* Vcm, double* Q, int64_t ldq, double* F,
                          int64_t ldf, double cutoff_scale, double cutoff_abs, const unsigned* status, unsigned gate_bit,
                          cudaStream_t st);
void launch_householder_qr(double* Zcm, int64_t p, int64_t q, double* alpha, double* Qcm, double* T, int64_t ldt,
                           const unsigned* status, unsigned gate_bit, cudaStream_t st);
// cutoff = cutoff_abs if cutoff_abs >= 0 else cutoff_scale * sigma_max; Vcm needs q*q*4 + q doubles
void launch_jacobi_pinv_factor(double* Tcm, double* Vcm, int64_t q, double cutoff_scale, double cutoff_abs, double* F,
                               int64_t ldf, const unsigned* status, unsigned gate_bit, cudaStream_t st);
void launch_conj_copy(const double* src, int64_t count_q, double* dst, const unsigned* status, unsigned gate_bit,
                      cudaStream_t st);
void launch_colmajor_to_rowmajor(const double* Zcm, int64_t p, int64_t q, double* Z, int64_t ldz,
                                 const unsigned* status, unsigned gate_bit, int gate_invert, cudaStream_t st);
void launch_rowmajor_to_colmajor(const double* Z, int64_t p, int64_t q, int64_t ldz, double* Zcm,
                                 const unsigned* status, unsigned gate_bit, cudaStream_t st);

// k_qsvd.cu : quaternion one-sided Jacobi SVD (column-major A m x n with m >= n, V n x n)
void launch_to_colmajor(const double* A, int64_t m, int64_t n, int64_t lda, double* Acm, cudaStream_t st);
void launch_identity_cm(double* Vcm, int64_t n, cudaStream_t st);
int64_t jacobi_sweep_rounds(int64_t m, int64_t n);
void launch_jacobi_round(double* Acm, int64_t m, int64_t n, double* Vcm, int64_t rnd, unsigned* flag, cudaStream_t st);
void launch_col_norms(const double* Acm, int64_t m, int64_t n, double* sigma, cudaStream_t st);
void launch_jacobi_cert(const double* Acm, int64_t m, int64_t n, const int* top, int k, const double* sigma,
                        unsigned* flag, cudaStream_t st);

// k_synth.cu : synthetic workloads (Philox normal generator)
// offset: element offset (even) of this block within the whole generated array
void launch_normal_fill(double* out, int64_t count, uint64_t seed, uint64_t stream, double scale, cudaStream_t st,
                        int64_t offset = 0);
// sigma = rel * sqrt(*ssq / total) (total = element count of the whole matrix; 0 -> count)
void launch_add_scaled_noise(double* X, int64_t count, uint64_t seed, uint64_t stream, const double* ssq,
                             double rel, cudaStream_t st, int64_t offset = 0, int64_t total = 0);
void launch_sumsq(const double* X, int64_t count, double* partials, int64_t nparts, double* out, cudaStream_t st);
// cfg3 image-like input; F: 6 L max(m,n) doubles, part: 296*6 doubles scratch
void launch_synth_image(int64_t m, int64_t n, int L, uint64_t seed, double sigma, double* F, double* part,
                        double* X, cudaStream_t st);

// k_ozaki.cu : Y (m x r) = X (m x n) * B (n x r) on the INT8 tensor cores (tcgen05 kind::i8) by exact
// modular arithmetic over L moduli (Ozaki scheme II); interleaved quaternions, ld in quaternions.
int ozaki_max_moduli();
bool ozaki_supported(int64_t m, int64_t n, int64_t r);
size_t ozaki_workspace_bytes(int64_t m, int64_t n, int64_t r, int L);
int64_t ozaki_chunk_rows(int64_t m, int64_t n, int64_t r, double cap_bytes);
int launch_ozaki_gemm(const double* X, int64_t m, int64_t n, int64_t ldx, const double* B, int64_t r, int64_t ldb,
                      double* Y, int64_t ldy, int L, void* workspace, cudaStream_t st);
// the same in two phases: prepare (residues of X; depends on X only) and finish (B, GEMMs, CRT)
int launch_ozaki_prepare_rows(const double* X_rows, int64_t rows, int64_t row0, int64_t m, int64_t n, int64_t ldx,
                              int64_t r, int L, void* workspace, cudaStream_t st);
int launch_ozaki_prepare(const double* X, int64_t m, int64_t n, int64_t ldx, int64_t r, int L, void* workspace,
                         cudaStream_t st);
int launch_ozaki_finish(int64_t m, int64_t n, const double* B, int64_t r, int64_t ldb, double* Y, int64_t ldy, int L,
                        void* workspace, cudaStream_t st);
// finish = prep_b (exponents and residues of E(B)) + multiply (the L GEMMs and the CRT)
int launch_ozaki_prep_b(int64_t m, int64_t n, const double* B, int64_t r, int64_t ldb, int L, void* workspace,
                        cudaStream_t st);
int launch_ozaki_multiply(int64_t m, int64_t n, int64_t r, double* Y, int64_t ldy, int L, void* workspace,
                          cudaStream_t st);
// C_k = A_k^H B_k (A_k p_k x qa_k, B_k p_k x qb_k; B_k == A_k allowed) for up to two problems in one
// INT8 GEMM launch, by the 16 real plane products (no Hamilton expansion); ldc in quaternions
size_t ozaki_herm_workspace_bytes(int64_t p, int64_t qa, int64_t qb, int same);
bool ozaki_herm_supported(int64_t p, int64_t qa, int64_t qb);
bool ozaki_side_kernel(const void* f);  // kernels of the low-priority side stream (graph node priorities)
int launch_ozaki_pair(const double* const* X, const int64_t* m, const int64_t* n, const int64_t* ldx,
                      const double* const* B, const int64_t* r, const int64_t* ldb, const int* conjT, double* const* Y,
                      const int64_t* ldy, int np, int L, void* const* workspace, cudaStream_t st);
int launch_ozaki_herm(const double* const* A, const double* const* B, const int64_t* p, const int64_t* qa,
                      const int64_t* qb, const int64_t* lda, const int64_t* ldb, double* const* C,
                      const int64_t* ldc, int np, int L, void* const* workspace, cudaStream_t st,
                      int lower_only = 0);  // 1: same-operand products write only blocks on/below the diagonal

// k_ozaki_err.cu : the fused error ||X - P R|| (out4 as launch_cur_error) with P R on the INT8
// tensor cores by exact base-256 digit slices (Ozaki scheme I, 21 digit products).
bool ozaki_error_supported(int64_t m, int64_t n, int64_t r);
size_t ozaki_error_workspace_bytes(int64_t m, int64_t n, int64_t r);
int launch_ozaki_error(const double* X, int64_t ldx, const double* P, int64_t ldp, const double* R, int64_t ldr,
                       int64_t m, int64_t n, int64_t r, double psnr_scale, void* workspace, double* out4,
                       cudaStream_t st);
// the same in two steps: digit planes, then the GEMMs with the fused epilogue
int launch_ozaki_error_digits(const double* P, int64_t ldp, const double* R, int64_t ldr, int64_t m, int64_t n,
                              int64_t r, void* workspace, cudaStream_t st, int with_r = 1);
int launch_ozaki_error_rdigits(const double* R, int64_t ldr, int64_t m, int64_t n, int64_t r, void* workspace,
                               cudaStream_t st);
int launch_ozaki_error_gemm(const double* X, int64_t ldx, int64_t m, int64_t n, int64_t r, double psnr_scale,
                            void* workspace, double* out4, cudaStream_t st);

// INT8 tensor-core peak probe (TOP/s; bench roofline denominator of the INT8 kernels)
double run_i8_peak(int sms, cudaStream_t st);
// fp64 peak probe (bench roofline denominator)
double run_dmma_peak(int sms, cudaStream_t st);

}  // namespace qcur
