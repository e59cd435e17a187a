// K1 — length-squared sampling distributions, bit-identical to numpy.
//
// Replaces length_distributions (pkg/src/qcur/cur.py:132-150):
//   sq    = ((a0^2 + a1^2) + a2^2) + a3^2        per entry, no FMA   (cur.py:143)
//   total = pairwise(sq.ravel())                                     (cur.py:144)
//   col   = sequential sum down the rows                             (cur.py:147)
//   row   = pairwise sum along each row                              (cur.py:148)
//   col/total, row/total, then divided by their own pairwise sums    (cur.py:150)
//
// Pass A (k1_colstrip): one CTA per 16-column strip streams its strip of X
// top to bottom (coalesced 512-byte row segments, register double-buffered),
// computes sq, writes it row-major for pass B and keeps the exact sequential
// column accumulator in one lane per column.
// Pass B (pairwise_chunks / pairwise_top): numpy's pairwise tree over each row
// and over the flat array, evaluated from the sq buffer chunk by chunk.
#include "common.cuh"
#include "kernels.h"
#include "pairwise.h"

namespace qcur {

// ---------------------------------------------------------------------------
// Pass A: sq + exact sequential column sums.
// ---------------------------------------------------------------------------
constexpr int kStripW = 16;    // quaternion columns per CTA (half a warp per row: 512-byte segments)
constexpr int kStripRB = 128;  // rows per pipeline stage (8 quaternions in flight per thread)
constexpr int kStripThreads = 256;

// acc_in (nullable): running column sums of the rows above this block, so a
// row-sharded matrix continues numpy's sequential axis-0 order across ranks.
// 16-column strips: n / 16 CTAs (250 at n = 4000) cover every SM, where 32-column
// strips left 23 of 148 idle.
__global__ void __launch_bounds__(kStripThreads) k1_colstrip(const double* __restrict__ X, int64_t m, int64_t n,
                                                             int64_t ldx, double* __restrict__ sq,
                                                             double* __restrict__ colsum,
                                                             const double* __restrict__ acc_in, int64_t ldsq) {
  __shared__ double sqs[2][kStripRB][kStripW];
  const int tid = threadIdx.x;
  const int lane = tid & 31, col = lane & (kStripW - 1);
  const int prow = (tid >> 5) * 2 + (lane >> 4);  // 0..15: row within a 16-row pass
  const int64_t j = (int64_t)blockIdx.x * kStripW + col;
  const bool jok = j < n;
  constexpr int kPer = kStripRB / 16;  // rows per thread per stage
  Quat buf[kPer];
  auto load_stage = [&](int64_t r0) {
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      int64_t i = r0 + prow + 16 * k;
      if (jok && i < m)
        buf[k] = ldq_nc(X + (i * ldx + j) * 4);
      else
        buf[k] = qzero();
    }
  };
  // numpy starts from the first row; 0 + sq[0] == sq[0] exactly (sq >= 0)
  double acc = (acc_in != nullptr && jok) ? acc_in[j] : 0.0;
  const int64_t nstages = (m + kStripRB - 1) / kStripRB;
  load_stage(0);
  for (int64_t s = 0; s < nstages; ++s) {
    const int64_t r0 = s * kStripRB;
    const int b = (int)(s & 1);
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const Quat q = buf[k];
      double v = __dmul_rn(q.w, q.w);
      v = __dadd_rn(v, __dmul_rn(q.x, q.x));
      v = __dadd_rn(v, __dmul_rn(q.y, q.y));
      v = __dadd_rn(v, __dmul_rn(q.z, q.z));
      const int rr = prow + 16 * k;
      sqs[b][rr][col] = v;
      const int64_t i = r0 + rr;
      if (jok && i < m) sq[i * ldsq + j] = v;
    }
    if (s + 1 < nstages) load_stage(r0 + kStripRB);
    __syncthreads();
    if (tid < kStripW) {
      const int rows = (int)((m - r0) < kStripRB ? (m - r0) : kStripRB);
      for (int rr = 0; rr < rows; ++rr) acc = __dadd_rn(acc, sqs[b][rr][col]);
    }
    // the double buffer lets the next stage's sq writes proceed while warp 0
    // accumulates; a second barrier is only needed before a buffer is reused,
    // which the barrier of the following stage provides.
  }
  if (tid < kStripW && jok) colsum[j] = acc;
}

// ---------------------------------------------------------------------------
// Pass B: numpy pairwise trees.
// ---------------------------------------------------------------------------
constexpr int kChunkThreads = 256;
constexpr int kFinThreads = 1024;

// All threads of a CTA evaluate chunk `chunk` of numpy's pairwise tree over
// `vals` (the segment's data: HBM or shared memory), using `leafv` (shared,
// nleaves + chunk nodes) for the leaf sums and inner nodes.  Returns the chunk
// sum in every thread.
__device__ __forceinline__ double chunk_eval(const double* __restrict__ vals, const DevPairwise& pw, int chunk,
                                             double* leafv) {
  const int pid = pw.chunk_plan[chunk];
  const int leaf0 = pw.plan_leaf_ptr[pid], nleaves = pw.plan_leaf_ptr[pid + 1] - leaf0;
  vals += pw.chunk_off[chunk];
  const int q = threadIdx.x & 7;
  for (int base = 0; base < nleaves; base += (int)blockDim.x / 8) {
    const int leaf = base + ((int)threadIdx.x >> 3);
    const bool active = leaf < nleaves;
    int off = 0, ln = 0;
    if (active) {
      off = pw.leaf_off[leaf0 + leaf];
      ln = pw.leaf_len[leaf0 + leaf];
    }
    double r = 0.0;
    const int body = ln - (ln & 7);
    if (active && ln >= 8) {
      // a numpy leaf holds at most 128 values (PW_BLOCKSIZE), so this lane's <= 16 are loaded
      // first (independent loads in flight) and then added in numpy's order
      double buf[16];
#pragma unroll
      for (int t = 0; t < 16; ++t) buf[t] = 8 * t < body ? vals[off + 8 * t + q] : 0.0;
      r = buf[0];
#pragma unroll
      for (int t = 1; t < 16; ++t)
        if (8 * t < body) r = __dadd_rn(r, buf[t]);
    }
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) in lane group order
    double t1 = __shfl_xor_sync(0xffffffffu, r, 1);
    double a = __dadd_rn(r, t1);
    double t2 = __shfl_xor_sync(0xffffffffu, a, 2);
    double bsum = __dadd_rn(a, t2);
    double t4 = __shfl_xor_sync(0xffffffffu, bsum, 4);
    double res = __dadd_rn(bsum, t4);
    if (active && q == 0) {
      if (ln < 8) {
        res = 0.0;
        for (int i = 0; i < ln; ++i) res = __dadd_rn(res, vals[off + i]);
      } else {
        for (int i = body; i < ln; ++i) res = __dadd_rn(res, vals[off + i]);
      }
      leafv[leaf] = res;
    }
  }
  __syncthreads();
  // combine the chunk's tree one level at a time (all threads), numpy's order
  const int n0 = pw.plan_node_ptr[pid], l0 = pw.plan_lvl_ptr[pid], nl = pw.plan_lvl_ptr[pid + 1] - l0;
  int prev = 0;
  for (int h = 0; h < nl; ++h) {
    const int end = pw.clvl[l0 + h];
    for (int k = prev + threadIdx.x; k < end; k += blockDim.x)
      leafv[nleaves + k] = __dadd_rn(leafv[pw.cnode_l[n0 + k]], leafv[pw.cnode_r[n0 + k]]);
    prev = end;
    __syncthreads();
  }
  const double sum = nl > 0 ? leafv[nleaves + prev - 1] : leafv[0];
  __syncthreads();  // leafv may be reused by the caller
  return sum;
}

// One CTA evaluates one chunk (<= kChunkMax elements) of one segment.
// out[seg * out_stride + chunk].  reverse: segments in descending order (the
// row pass right after the column strips finds the last-written rows of sq in L2).
__global__ void __launch_bounds__(kChunkThreads) pairwise_chunks(const double* __restrict__ data, int64_t seg_stride,
                                                                 DevPairwise pw, double* __restrict__ out,
                                                                 int64_t out_stride, int reverse) {
  extern __shared__ double sm[];
  const int chunk = blockIdx.x;
  const int64_t seg = reverse ? (int64_t)gridDim.y - 1 - blockIdx.y : (int64_t)blockIdx.y;
  const double v = chunk_eval(data + seg * seg_stride, pw, chunk, sm);  // leaves read from HBM
  if (threadIdx.x == 0) out[seg * out_stride + chunk] = v;
}

// The row pass and the flat pass in one launch, scheduled by position: job list entries
// >= 0 are rows (rowsum[i] = pairwise(sq[i, :])), entries < 0 are flat chunks -(k+1)
// (chunk sums of sq.ravel()); each row is followed by the flat chunks that start inside it,
// so the second reader of every stretch of sq finds it in L2.  Jobs run bottom-up (the
// column strips wrote the bottom rows last).
__global__ void __launch_bounds__(kChunkThreads) pairwise_rows_flat(const double* __restrict__ sq, int64_t n,
                                                                    DevPairwise rpw, DevPairwise fpw,
                                                                    const int32_t* __restrict__ sched,
                                                                    double* __restrict__ rowsum,
                                                                    double* __restrict__ flat) {
  extern __shared__ double sm[];
  const int job = sched[gridDim.x - 1 - blockIdx.x];
  if (job >= 0) {
    const double v = chunk_eval(sq + (int64_t)job * n, rpw, 0, sm);
    if (threadIdx.x == 0) rowsum[job] = v;
  } else {
    const int chunk = -job - 1;
    const double v = chunk_eval(sq, fpw, chunk, sm);
    if (threadIdx.x == 0) flat[chunk] = v;
  }
}

// Fused tail of length_distributions (cur.py:144-150) for axes of at most one
// pairwise chunk: CTA 0 handles the columns, CTA 1 the rows.  Each CTA
//   1. evaluates the flat top tree over the chunk sums of sq.ravel() in shared
//      memory -> total (both CTAs alike, bit-identical);
//   2. sc = axis_sum / total  (col = sq.sum(axis=0) / total), kept in shared memory;
//   3. s = pairwise(sc)  (col.sum()), numpy's tree;
//   4. out = sc / s.
// Same divisions in the same order as the unfused launches, so the same bits.
struct FinalizeAxis {
  const double* sum;  // colsum or rowsum
  double* out;        // col or row
  DevPairwise pw;     // the axis length's program (a single chunk)
};

__global__ void __launch_bounds__(kFinThreads) k1_finalize(const double* __restrict__ flat, DevPairwise fpw,
                                                           FinalizeAxis ax0, FinalizeAxis ax1, unsigned* status) {
  extern __shared__ double sm[];
  const FinalizeAxis& ax = blockIdx.x == 0 ? ax0 : ax1;
  double total;
  if (fpw.nnodes == 0) {
    total = flat[0];
  } else {
    // the tree program is staged in shared memory with the chunk sums (one round trip
    // instead of one per level)
    double* v = sm;
    int32_t* nl = reinterpret_cast<int32_t*>(v + fpw.nchunks + fpw.nnodes);
    int32_t* nr = nl + fpw.nnodes;
    int32_t* lp = nr + fpw.nnodes;
    for (int k = threadIdx.x; k < fpw.nchunks; k += blockDim.x) v[k] = flat[k];
    for (int k = threadIdx.x; k < fpw.nnodes; k += blockDim.x) {
      nl[k] = fpw.node_l[k];
      nr[k] = fpw.node_r[k];
    }
    for (int k = threadIdx.x; k < fpw.maxh + 2; k += blockDim.x) lp[k] = fpw.level_ptr[k];
    __syncthreads();
    for (int h = 1; h <= fpw.maxh; ++h) {
      const int a = lp[h], b = lp[h + 1];
      for (int k = a + threadIdx.x; k < b; k += blockDim.x) v[fpw.nchunks + k] = __dadd_rn(v[nl[k]], v[nr[k]]);
      __syncthreads();
    }
    total = v[fpw.nchunks + fpw.nnodes - 1];
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && !(total > 0.0)) atomicOr(status, (unsigned)ST_DEGENERATE);
  const int64_t len = ax.pw.length;
  double* sc = sm;
  double* leafv = sm + ((len + 31) & ~(int64_t)31);
  for (int64_t t = threadIdx.x; t < len; t += blockDim.x) sc[t] = __ddiv_rn(ax.sum[t], total);
  __syncthreads();
  const double s = chunk_eval(sc, ax.pw, 0, leafv);
  for (int64_t t = threadIdx.x; t < len; t += blockDim.x) ax.out[t] = __ddiv_rn(sc[t], s);
}

// Top tree over chunk sums; one CTA per segment.  vals: [nseg][nchunks+nnodes]
__global__ void pairwise_top(double* __restrict__ vals, DevPairwise pw, double* __restrict__ out) {
  const int64_t seg = blockIdx.x;
  const int64_t w = (int64_t)pw.nchunks + pw.nnodes;
  double* v = vals + seg * w;
  for (int h = 1; h <= pw.maxh; ++h) {
    const int a = pw.level_ptr[h], b = pw.level_ptr[h + 1];
    for (int k = a + threadIdx.x; k < b; k += blockDim.x)
      v[pw.nchunks + k] = __dadd_rn(v[pw.node_l[k]], v[pw.node_r[k]]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[seg] = pw.nnodes > 0 ? v[w - 1] : v[0];
}

__global__ void k1_scale(const double* __restrict__ in, int64_t len, const double* __restrict__ denom,
                         double* __restrict__ out, unsigned* status, unsigned check_bit) {
  const double d = *denom;
  if (check_bit && blockIdx.x == 0 && threadIdx.x == 0 && !(d > 0.0)) atomicOr(status, check_bit);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < len; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = __ddiv_rn(in[t], d);
}

__global__ void k_fill(double* __restrict__ out, int64_t len, double v) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < len; t += (int64_t)gridDim.x * blockDim.x)
    out[t] = v;
}

// ---------------------------------------------------------------------------
// host launchers
// ---------------------------------------------------------------------------
void launch_colstrip(const double* X, int64_t m, int64_t n, int64_t ldx, double* sq, double* colsum,
                     cudaStream_t st, const double* acc_in, int64_t ldsq) {
  dim3 grid((unsigned)((n + kStripW - 1) / kStripW));
  ++::qcur::g_launches;
  k1_colstrip<<<grid, kStripThreads, 0, st>>>(X, m, n, ldx, sq, colsum, acc_in, ldsq > 0 ? ldsq : n);
}

void launch_pairwise(const double* data, int64_t nseg, int64_t seg_stride, const DevPairwise& pw, double* scratch,
                     double* out, cudaStream_t st, bool with_top, bool reverse) {
  size_t smem = (size_t)(kChunkMax + kChunkMax / 8 + 8) * sizeof(double);
  static std::atomic<unsigned> attr_set{0};
  if (first_on_device(attr_set)) {
    cudaFuncSetAttribute(pairwise_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  }
  // dynamic smem: leaf sums and the chunk's tree nodes only (the data streams from HBM)
  size_t need = (size_t)(pw.max_chunk_len / 4 + 16) * sizeof(double);
  if (pw.nnodes == 0) {
    // single chunk per segment: write straight to out
    dim3 grid(1, (unsigned)nseg);
    ++::qcur::g_launches;
    pairwise_chunks<<<grid, kChunkThreads, need, st>>>(data, seg_stride, pw, out, 1, reverse ? 1 : 0);
    return;
  }
  const int64_t w = (int64_t)pw.nchunks + pw.nnodes;
  dim3 grid((unsigned)pw.nchunks, (unsigned)nseg);
  ++::qcur::g_launches;
  pairwise_chunks<<<grid, kChunkThreads, need, st>>>(data, seg_stride, pw, scratch, w, reverse ? 1 : 0);
  if (!with_top) return;
  ++::qcur::g_launches;
  pairwise_top<<<(unsigned)nseg, 256, 0, st>>>(scratch, pw, out);
}

static size_t finalize_smem(const DevPairwise& fpw, int64_t n, int64_t m) {
  // chunk sums and nodes (doubles) + node_l, node_r, level_ptr (int32)
  const int64_t top = fpw.nnodes == 0 ? 0 : (int64_t)fpw.nchunks + fpw.nnodes + (2 * (int64_t)fpw.nnodes + fpw.maxh + 3) / 2;
  const int64_t len = n > m ? n : m;
  const int64_t axis = ((len + 31) & ~(int64_t)31) + len / 4 + 64;
  return (size_t)(top > axis ? top : axis) * sizeof(double);
}

void launch_rows_flat(const double* sq, int64_t m, int64_t n, const DevPairwise& rpw, const DevPairwise& fpw,
                      const int32_t* sched, double* rowsum, double* flat, cudaStream_t st) {
  const int64_t mc = rpw.max_chunk_len > fpw.max_chunk_len ? rpw.max_chunk_len : fpw.max_chunk_len;
  const size_t need = (size_t)(mc / 4 + 16) * sizeof(double);
  ++::qcur::g_launches;
  pairwise_rows_flat<<<(unsigned)(m + fpw.nchunks), kChunkThreads, need, st>>>(sq, n, rpw, fpw, sched, rowsum, flat);
}

bool finalize_supported(const DevPairwise& fpw, const DevPairwise& cpw, const DevPairwise& rpw) {
  return cpw.nnodes == 0 && cpw.nchunks == 1 && rpw.nnodes == 0 && rpw.nchunks == 1 &&
         finalize_smem(fpw, cpw.length, rpw.length) <= (size_t)200 * 1024;
}

void launch_finalize(const double* flat, const DevPairwise& fpw, const double* colsum, const DevPairwise& cpw,
                     double* col, const double* rowsum, const DevPairwise& rpw, double* row, unsigned* status,
                     cudaStream_t st) {
  static std::atomic<unsigned> attr_set{0};
  if (first_on_device(attr_set)) {
    cudaFuncSetAttribute(k1_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  }
  ++::qcur::g_launches;
  k1_finalize<<<2, kFinThreads, finalize_smem(fpw, cpw.length, rpw.length), st>>>(
      flat, fpw, FinalizeAxis{colsum, col, cpw}, FinalizeAxis{rowsum, row, rpw}, status);
}

void launch_scale(const double* in, int64_t len, const double* denom, double* out, unsigned* status,
                  unsigned check_bit, cudaStream_t st) {
  int blocks = (int)((len + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  if (blocks < 1) blocks = 1;
  ++::qcur::g_launches;
  k1_scale<<<blocks, 256, 0, st>>>(in, len, denom, out, status, check_bit);
}

void launch_fill(double* out, int64_t len, double v, cudaStream_t st) {
  int blocks = (int)((len + 255) / 256);
  if (blocks > 1184) blocks = 1184;
  if (blocks < 1) blocks = 1;
  ++::qcur::g_launches;
  k_fill<<<blocks, 256, 0, st>>>(out, len, v);
}

}  // namespace qcur
