// K2 — iterated weighted draw without replacement, index-exact vs numpy.
//
// Replaces draw_indices / plan_indices (pkg/src/qcur/cur.py:202-254).  Per
// draw the reference forms cum = np.cumsum(p) (sequential), scales one
// Generator.random() by cum[-1], takes searchsorted(cum, u, 'right'), clamps,
// walks back over zero weights, records the index and zeroes its weight.
//
// Device design: one CTA per axis (columns and rows run concurrently).  The
// CTA copies p and builds a 32-ary sum tree over it; one warp then performs
// the `count` draws, each a root-to-leaf descent of warp scans (O(log32 n)
// per draw instead of an O(n) cumsum).  The descent's prefix values differ
// from numpy's sequential cumsum only by rounding, bounded by
// (n + 70) * 2^-53 * total; a draw is accepted only when the uniform sits
// farther than twice that bound from both neighbouring prefix values, which
// proves the numpy index.  Drawn weights leave the tree by subtraction along the
// path (the margin grows by the per-draw rounding).  Otherwise (probability ~1e-12 per draw) the lane
// recomputes the exact sequential cumsum — numpy's own order — for that draw.
// The PCG64 stream is advanced on device (pcg64.h), one double per draw.
#include "common.cuh"
#include "kernels.h"
#include "pcg64.h"

namespace qcur {

constexpr int kMaxLevels = 8;
constexpr int64_t kDrawSmemMaxLen = 24576;  // p (+ its tree) fits the 224 KB dynamic shared memory cap

struct Levels {
  double* lev[kMaxLevels];
  int64_t sz[kMaxLevels];
  int top;  // index of the top level (sz[top] <= 32)
};

__host__ __device__ inline Levels make_levels(double* work, int64_t len) {
  Levels L;
  int64_t off = 0;
  int64_t s = len;
  int h = 0;
  L.lev[0] = work;
  L.sz[0] = len;
  off = len;
  while (s > 32 && h + 1 < kMaxLevels) {
    s = (s + 31) / 32;
    ++h;
    L.lev[h] = work + off;
    L.sz[h] = s;
    off += s;
  }
  L.top = h;
  return L;
}

// work buffer: p (len) | tree levels | 64 slack | uniforms (count <= len)
__host__ __device__ inline int64_t draw_uniform_offset(int64_t len) {
  int64_t total = len, s = len;
  while (s > 32) {
    s = (s + 31) / 32;
    total += s;
  }
  return total + 64;
}

int64_t draw_work_doubles(int64_t len) { return draw_uniform_offset(len) + len; }

// recompute node `node` of level h (h >= 1) from its 32 children; called by a full warp
__device__ __forceinline__ void refresh_node(const Levels& L, int h, int64_t node, int lane) {
  const int64_t c = node * 32 + lane;
  double v = c < L.sz[h - 1] ? L.lev[h - 1][c] : 0.0;
  v = warp_sum(v);
  if (lane == 0) L.lev[h][node] = v;
  __syncwarp();
}

struct DrawJobs {
  DrawJob j[2];
};

__global__ void __launch_bounds__(1024) k2_draw(DrawJobs jobs, unsigned* status) {
  const DrawJob job = jobs.j[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int64_t len = job.len;
  // The weights and the sum tree live in shared memory (a draw is a chain of
  // dependent probes: ~30-cycle smem latency instead of ~600-cycle L2); for
  // very long axes only the tree does and p stays in the global work buffer.
  extern __shared__ double sm_draw[];
  Levels L = make_levels(job.work, len);
  {
    const bool p_in_smem = len <= kDrawSmemMaxLen;
    double* base = p_in_smem ? sm_draw : sm_draw - len;  // tree always follows p's slot in smem
    Levels S = make_levels(base, len);
    if (!p_in_smem) S.lev[0] = job.work;
    L = S;
  }
  // copy p and count positives
  __shared__ int s_pos[32];
  int pos = 0;
  for (int64_t t = tid; t < len; t += blockDim.x) {
    double v = job.probs[t];
    L.lev[0][t] = v;
    pos += v > 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, o);
  if (lane == 0) s_pos[warp] = pos;
  __syncthreads();
  // build the sum tree (all warps)
  for (int h = 1; h <= L.top; ++h) {
    for (int64_t node = warp; node < L.sz[h]; node += nw) refresh_node(L, h, node, lane);
    __syncthreads();
  }
  // the draw's uniforms: uniform t is the stream advanced by t (numpy draws one
  // double per draw, columns first), computed in parallel instead of in the chain
  double* uni = job.work + draw_uniform_offset(len);
  for (int64_t t = tid; t < job.count; t += blockDim.x) {
    Pcg64 g;
    g.state = u128{job.st_hi, job.st_lo};
    g.inc = u128{job.inc_hi, job.inc_lo};
    g.advance((uint64_t)t);
    uni[t] = g.next_double();
  }
  __syncthreads();
  if (warp != 0) return;
  int positive = 0;
  for (int w = 0; w < nw; ++w) positive += s_pos[w];
  if (job.count > positive) {
    // "cannot draw {count} distinct indices from {positive} positive weights"
    if (lane == 0) atomicOr(status, (unsigned)ST_SAMPLING);
    for (int64_t t = lane; t < job.count; t += 32) job.out[t] = 0;
    return;
  }
  const double u53 = 1.0 / 9007199254740992.0;
  const int count = (int)job.count;
  double u_next = uni[0];
  for (int t = 0; t < count; ++t) {
    const double u = u_next;  // identical on every lane
    if (t + 1 < count) u_next = uni[t + 1];
    // descend; the top level's inclusive scan also yields the total
    double base = 0.0, lower = 0.0, upper = 0.0, total = 0.0, target = 0.0;
    int g = 0;
    bool ok = true;
    for (int h = L.top; h >= 0; --h) {
      const int c = g * 32 + lane;
      const bool valid = c < (int)L.sz[h];
      double s = valid ? L.lev[h][c] : 0.0;
      // inclusive Hillis-Steele scan (fixed order)
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        double y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      if (h == L.top) {
        total = __shfl_sync(0xffffffffu, s, 31);
        if (!(total > 0.0)) break;
        target = u * total;
      }
      const double posv = base + s;
      const unsigned hit = __ballot_sync(0xffffffffu, valid && posv > target);
      if (hit == 0u) {
        ok = false;
        break;
      }
      const int k = __ffs(hit) - 1;
      const double s_prev = __shfl_sync(0xffffffffu, s, (k + 31) & 31);
      const double s_k = __shfl_sync(0xffffffffu, s, k);
      const double nb = k > 0 ? base + s_prev : base;
      if (h == 0) {
        lower = nb;
        upper = base + s_k;
      }
      base = nb;
      g = g * 32 + k;
    }
    if (!(total > 0.0)) {
      if (lane == 0) atomicOr(status, (unsigned)ST_SAMPLING);
      for (int q = t + lane; q < count; q += 32) job.out[q] = 0;
      return;
    }
    int64_t idx = g;
    if (ok) {
      const double tot_est = total * (1.0 + 1e-12);
      // 2 (n + 70 + 2 count) 2^-53 T: the fresh tree's prefix error plus one rounding per
      // level for every earlier removal
      const double delta = 2.0 * ((double)len + 70.0 + 2.0 * (double)count) * u53 * tot_est;
      ok = (lower <= target - delta) && (upper > target + delta) && (L.lev[0][idx] > 0.0);
    }
    if (!ok) {
      // exact numpy order: sequential cumsum, searchsorted(side='right'), clamp, zero walk
      if (lane == 0) {
        atomicOr(status, (unsigned)ST_DRAW_FALLBACK);
        const double* p = L.lev[0];
        double acc = 0.0;
        for (int64_t i = 0; i < len; ++i) acc = (i == 0) ? p[0] : acc + p[i];
        const double tot = acc;
        const double tgt = u * tot;
        acc = 0.0;
        int64_t found = len;
        for (int64_t i = 0; i < len; ++i) {
          acc = (i == 0) ? p[0] : acc + p[i];
          if (acc > tgt) {
            found = i;
            break;
          }
        }
        if (found > len - 1) found = len - 1;
        while (found > 0 && p[found] == 0.0) --found;
        idx = found;
      }
      idx = __shfl_sync(0xffffffffu, idx, 0);
    }
    if (lane == 0) {
      // remove the drawn weight: zero the leaf, subtract it along the path (one rounding per
      // level and draw; the acceptance margin above covers the accumulated error)
      const double wgt = L.lev[0][idx];
      job.out[t] = idx;
      L.lev[0][idx] = 0.0;
      int node = (int)idx;
      for (int h = 1; h <= L.top; ++h) {
        node >>= 5;
        L.lev[h][node] -= wgt;
      }
    }
    __syncwarp();
  }
}

void launch_draw(const DrawJob* jobs, int njobs, unsigned* status, cudaStream_t st) {
  DrawJobs j{};
  size_t smem = 0;
  for (int k = 0; k < njobs && k < 2; ++k) {
    j.j[k] = jobs[k];
    const int64_t len = jobs[k].len;
    const int64_t tree = draw_uniform_offset(len) - len;  // levels >= 1 (+ slack)
    const int64_t need = (len <= kDrawSmemMaxLen ? len : 0) + tree;
    if ((size_t)need * sizeof(double) > smem) smem = (size_t)need * sizeof(double);
  }
  static bool attr = false;
  if (!attr) {
    // 227 KB minus the kernel's static shared memory (a failing attribute call
    // would otherwise surface as the launch's error)
    cudaFuncSetAttribute(k2_draw, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
    attr = true;
  }
  ++::qcur::g_launches;
  k2_draw<<<njobs, 1024, smem, st>>>(j, status);
}

}  // namespace qcur
