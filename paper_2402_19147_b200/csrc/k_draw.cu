// K2 — iterated weighted draw without replacement, index-exact vs numpy.
//
// Replaces draw_indices / plan_indices (pkg/src/qcur/cur.py:202-254).  Per
// draw the reference forms cum = np.cumsum(p) (sequential), scales one
// Generator.random() by cum[-1], takes searchsorted(cum, u, 'right'), clamps,
// walks back over zero weights, records the index and zeroes its weight.
//
// Device design: one CTA per axis (columns and rows run concurrently).  The
// CTA builds a 64-ary PREFIX tree over p: node k of level h holds, for its 64
// children, the inclusive prefix sums of their totals (every level padded with
// zeros to a multiple of 64, so a node is one aligned 512-byte run).  One warp
// then performs the `count` draws; each is a root-to-leaf descent in which
// every lane loads two adjacent prefix values (one 16-byte load) and a pair of
// ballots finds the first prefix above the uniform: no scan on the dependent
// chain, and a 4000-long axis is two levels deep.  A drawn weight leaves the
// tree by subtracting it from the prefix entries at and after its position in
// each node of its path, using the values the descent already holds (stores
// only, all levels independent).  The level pointers and sizes are
// compile-time-indexed registers (fully unrolled level loops).
// The descent's prefix values differ from numpy's sequential cumsum only by
// rounding.  numpy's own cumsum is within (n + 2) * 2^-53 * total of the exact
// prefix; the tree's entries carry their build rounding (relative to the total
// the tree was BUILT at) plus one rounding per level for every earlier removal
// (relative to the total at THAT removal, which can be far above today's total
// when a dominant weight was drawn).  The kernel keeps that running bound and
// accepts a draw only when the uniform sits farther than twice the sum from
// both neighbouring prefix values, which proves the numpy index.  When the
// tree's accumulated bound outgrows numpy's own term the tree is rebuilt from
// the exact remaining weights (drawn entries exactly zero), so a dominant
// weight costs one rebuild, not a run of fallbacks.  A draw that cannot be
// proved (probability ~1e-12 for ordinary weights) is made by lane 0 with the
// exact sequential cumsum — numpy's own order — over the exact weights.
// The PCG64 stream is advanced on device (pcg64.h), one double per draw.
#include "common.cuh"
#include "kernels.h"
#include "pcg64.h"

namespace qcur {

constexpr int kFan = 64;                    // children per node: two per lane
constexpr int kMaxL = 5;                    // 64^5 leaves: any axis length up to 2^30
constexpr int64_t kDrawSmemMaxLen = 24576;         // leaf prefixes (+ upper levels) fit the 224 KB smem cap
constexpr int64_t kMaxDrawLen = (int64_t)1 << 30;  // 64^5: the deepest tree kMaxL levels hold

__host__ __device__ inline int64_t rup64(int64_t x) { return (x + kFan - 1) / kFan * kFan; }

struct Tree {
  int top;             // index of the top level (sz[top] <= 64)
  int64_t sz[kMaxL];   // entries per level
  int64_t off[kMaxL];  // offsets of levels >= 1 in the upper-level buffer (each padded to 64)
  int64_t upper;       // doubles of the upper-level buffer
  int64_t root;        // offset of the top level in the upper-level buffer (top >= 1)
};

__host__ __device__ inline Tree make_tree(int64_t len) {
  Tree T;
  int64_t s = len, off = 0;
  T.top = 0;
  T.sz[0] = len;
  T.off[0] = 0;
  // fully unrolled (static indices keep the tree in registers)
#pragma unroll
  for (int k = 1; k < kMaxL; ++k) {
    T.off[k] = off;
    if (s > kFan) {
      s = (s + kFan - 1) / kFan;
      T.top = k;
      T.sz[k] = s;
      off += rup64(s);
    } else {
      T.sz[k] = 0;
    }
  }
  T.upper = off;
  T.root = T.top >= 1 ? off - kFan : 0;  // the top level is one node, allocated last
  return T;
}

// global work buffer: exact weights p (zeroed as drawn; the fallback's cumsum) | the
// level-0 prefix entries when they do not fit shared memory | uniforms | the upper
// levels and node-total buffers when even those do not fit shared memory
static int64_t draw_upper_doubles(int64_t len) {
  const Tree T = make_tree(len);
  return T.upper + 2 * rup64((len + kFan - 1) / kFan);
}
int64_t draw_work_doubles(int64_t len) { return 3 * rup64(len) + draw_upper_doubles(len) + 64; }

static constexpr size_t kDrawSmemCap = 224 * 1024;

// shared memory: level-0 prefixes (when they fit) | levels >= 1 | two node-total buffers
static int64_t draw_smem_doubles(int64_t len) {
  const int64_t need = (len <= kDrawSmemMaxLen ? rup64(len) : 0) + draw_upper_doubles(len);
  return (size_t)need * 8 <= kDrawSmemCap ? need : 0;  // 0: everything in global memory
}

struct DrawJobs {
  DrawJob j[2];
};

#ifdef QCUR_DRAW_TRACE  // per-draw clocks of CTA 0, lane 0 (tools/test_draw_trace.cu)
__device__ long long g_draw_trace[1026][3];
#define DRAW_T(t, k) \
  if (blockIdx.x == 0 && threadIdx.x == 0 && (t) < 1026) g_draw_trace[t][k] = clock64();
void draw_trace_read(long long* out) { cudaMemcpyFromSymbol(out, g_draw_trace, sizeof(g_draw_trace)); }
#else
#define DRAW_T(t, k)
#endif

// The prefix tree over the exact weights pw, level by level: a warp per node scans its 64
// children (pair sums, then a fixed-order Hillis-Steele scan); the node's total feeds the
// level above.  Run by the whole block (block = true) or, for a rebuild, by warp 0 alone.
template <bool kBlock>
__device__ __forceinline__ void build_tree(const Tree& T, double* const* P, double* const* Sb, const double* pw,
                                           int warp, int nw, int lane) {
#pragma unroll
  for (int h = 0; h < kMaxL; ++h) {
    if (h > T.top) continue;  // (continue, not break: keeps the loop unrolled, P[h] in registers)
    const double* in = h == 0 ? pw : Sb[(h - 1) & 1];
    double* tot = Sb[h & 1];
    const int64_t nnode = rup64(T.sz[h]) / kFan;
    for (int64_t node = warp; node < nnode; node += nw) {
      const int64_t c = node * kFan + 2 * lane;
      const double a = c < T.sz[h] ? in[c] : 0.0;
      const double b = c + 1 < T.sz[h] ? in[c + 1] : 0.0;
      double s = __dadd_rn(a, b);
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s = __dadd_rn(s, y);
      }
      double ex = __shfl_up_sync(0xffffffffu, s, 1);
      if (lane == 0) ex = 0.0;
      *reinterpret_cast<double2*>(P[h] + c) = make_double2(__dadd_rn(ex, a), s);
      if (lane == 31 && h < T.top) tot[node] = s;
    }
    if (kBlock)
      __syncthreads();
    else
      __syncwarp();
  }
}

// kLeafSmem: the level-0 prefixes live in shared memory (every job's axis is at most
// kDrawSmemMaxLen long), so all tree accesses compile to shared-memory loads.
// up_global: the upper levels do not fit shared memory either (axes beyond ~1.7M entries).
template <bool kLeafSmem>
__global__ void __launch_bounds__(512, 1) k2_draw(DrawJobs jobs, unsigned* status, int up_global) {
  const DrawJob job = jobs.j[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int64_t len = job.len;
  DRAW_T(1024, 0)
  const Tree T = make_tree(len);
  extern __shared__ __align__(16) double sm_draw[];
  constexpr bool p_in_smem = kLeafSmem;
  double* P[kMaxL];
  P[0] = p_in_smem ? sm_draw : job.work + rup64(len);
  double* up = p_in_smem ? sm_draw + rup64(len) : (up_global ? job.work + 3 * rup64(len) : sm_draw);
#pragma unroll
  for (int h = 1; h < kMaxL; ++h) P[h] = up + T.off[h];
  const int64_t nodes0 = rup64((len + kFan - 1) / kFan);
  double* Sb[2] = {up + T.upper, up + T.upper + nodes0};
  double* pw = job.work;  // exact weights
  double* uni = job.work + 2 * rup64(len);
  // exact weights (zero padded) and the count of positives
  __shared__ int s_pos[32];
  int pos = 0;
  for (int64_t t = tid; t < rup64(len); t += blockDim.x) {
    const double v = t < len ? job.probs[t] : 0.0;
    pw[t] = v;
    pos += v > 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) pos += __shfl_xor_sync(0xffffffffu, pos, o);
  if (lane == 0) s_pos[warp] = pos;
  // the draw's uniforms: uniform t is the stream advanced by t (numpy draws one
  // double per draw, columns first), computed in parallel instead of in the chain.
  // count > len always fails the positives check below, so len uniforms suffice.
  const int64_t nuni = job.count < len ? job.count : len;
  for (int64_t t = tid; t < nuni; t += blockDim.x) {
    Pcg64 g;
    g.state = u128{job.st_hi, job.st_lo};
    g.inc = u128{job.inc_hi, job.inc_lo};
    g.advance((uint64_t)t);
    uni[t] = g.next_double();
  }
  __syncthreads();
  DRAW_T(1024, 1)
  build_tree<true>(T, P, Sb, pw, warp, nw, lane);
  DRAW_T(1024, 2)
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
  const double* rootp = (T.top == 0 ? P[0] : up + T.root) + (kFan - 1);  // the root's last inclusive prefix
  // Error bookkeeping, in units of 2^-53 (module header).  Let E bound |tree prefix - exact
  // prefix| over every position.  The build leaves at most 7 roundings per stored prefix per
  // level, inherited upward: E0 = c_build * total0 (total0 = the total the tree was built at).
  // A removal subtracts the leaf's prefix difference wl from the entries after it on every
  // level: the drawn leaf's own build error (two adjacent within-node prefixes, <= 14 * total0)
  // leaves with it, and every level adds one rounding of entries no larger than the current
  // total (plus wl's own): E += 14 * total0 + c_rem * total.  numpy's sequential cumsum is within
  // (len + 2) * total of the exact prefix and the descent adds one rounding per level (c_np).
  // A draw is proved when the uniform is 2 (c_np * total + E) away from both neighbours.
  const double c_build = 4.0 * (T.top + 1) * (T.top + 2) + 16.0;
  const double c_rem = (double)(T.top + 3);
  const double c_np = (double)len + 2.0 + (double)(T.top + 2);
  double total0 = *rootp, err_acc = c_build * total0;
  // uniforms in registers, 32 draws per block (lane l holds draw 32 b + l), the next block
  // prefetched a whole block ahead: an L2 round trip per draw would otherwise be the chain's
  // longest link
  double ublk = lane < count ? uni[lane] : 0.0;
  double unext = 32 + lane < count ? uni[32 + lane] : 0.0;
  for (int t = 0; t < count; ++t) {
    DRAW_T(t, 0)
    if ((t & 31) == 0 && t > 0) {
      ublk = unext;
      unext = t + 32 + lane < count ? uni[t + 32 + lane] : 0.0;
    }
    const double u = __shfl_sync(0xffffffffu, ublk, t & 31);  // identical on every lane
    double total = *rootp;
    if (err_acc > c_np * total && total > 0.0) {
      // the tree's rounding (from heavier, already drawn weights) outweighs numpy's own:
      // rebuild it from the exact remaining weights
      build_tree<false>(T, P, Sb, pw, 0, 1, lane);
      total = *rootp;
      total0 = total;
      err_acc = c_build * total0;
    }
    if (!(total > 0.0)) {
      if (lane == 0) atomicOr(status, (unsigned)ST_SAMPLING);
      for (int q = t + lane; q < count; q += 32) job.out[q] = 0;
      return;
    }
    const double target = u * total;
    double q0[kMaxL], q1[kMaxL];
    int e_at[kMaxL];
    double base = 0.0, lower = 0.0, upper = 0.0, wl = 0.0;
    int64_t g = 0;
    bool ok = true;
#pragma unroll
    for (int h = kMaxL - 1; h >= 0; --h) {
      q0[h] = q1[h] = 0.0;
      e_at[h] = 0;
      if (h > T.top || !ok) continue;
      const double2 v = *reinterpret_cast<const double2*>(P[h] + g * kFan + 2 * lane);
      q0[h] = v.x;
      q1[h] = v.y;
      const double a0 = base + v.x, a1 = base + v.y;
      const unsigned b0 = __ballot_sync(0xffffffffu, a0 > target);
      const unsigned b1 = __ballot_sync(0xffffffffu, a1 > target);
      if ((b0 | b1) == 0u) {
        ok = false;
        continue;
      }
      const int k = __ffs(b0 | b1) - 1;
      const bool first = (b0 >> k) & 1u;
      const double a0k = __shfl_sync(0xffffffffu, a0, k), a1k = __shfl_sync(0xffffffffu, a1, k);
      const double a1p = __shfl_sync(0xffffffffu, a1, (k + 31) & 31);
      const double lo = first ? (k > 0 ? a1p : base) : a0k;
      if (h == 0) {
        // the leaf's weight as the tree sees it (within-node prefix difference)
        const double v0k = __shfl_sync(0xffffffffu, v.x, k), v1k = __shfl_sync(0xffffffffu, v.y, k);
        const double v1p = __shfl_sync(0xffffffffu, v.y, (k + 31) & 31);
        wl = first ? (k > 0 ? __dsub_rn(v0k, v1p) : v0k) : __dsub_rn(v1k, v0k);
        lower = lo;
        upper = first ? a0k : a1k;
      }
      const int e = 2 * k + (first ? 0 : 1);
      e_at[h] = e;
      base = lo;
      g = g * kFan + e;
    }
    DRAW_T(t, 1)
    int64_t idx = g;
    if (ok) {
      const double delta = 2.0 * u53 * (c_np * total + err_acc) * (1.0 + 1e-9);
      ok = (lower <= target - delta) && (upper > target + delta) && (wl > 0.0);
    }
    err_acc += (14.0 * total0 + c_rem * total) * (1.0 + 1e-9);
    if (ok) {
      // remove: entries at and after the path position of every node on the path
#pragma unroll
      for (int h = 0; h < kMaxL; ++h) {
        if (h > T.top) continue;
        const int e = e_at[h];
        if (2 * lane + 1 >= e) {
          const int64_t node = idx >> (6 * (h + 1));
          const double n0 = 2 * lane >= e ? __dsub_rn(q0[h], wl) : q0[h];
          *reinterpret_cast<double2*>(P[h] + node * kFan + 2 * lane) = make_double2(n0, __dsub_rn(q1[h], wl));
        }
      }
    } else {
      // exact numpy order: sequential cumsum, searchsorted(side='right'), clamp, zero walk
      if (lane == 0) {
        atomicOr(status, (unsigned)ST_DRAW_FALLBACK);
        double acc = 0.0;
        for (int64_t i = 0; i < len; ++i) acc = (i == 0) ? pw[0] : acc + pw[i];
        const double tgt = u * acc;
        acc = 0.0;
        int64_t found = len;
        for (int64_t i = 0; i < len; ++i) {
          acc = (i == 0) ? pw[0] : acc + pw[i];
          if (acc > tgt) {
            found = i;
            break;
          }
        }
        if (found > len - 1) found = len - 1;
        while (found > 0 && pw[found] == 0.0) --found;
        idx = found;
      }
      idx = __shfl_sync(0xffffffffu, idx, 0);
      const double w = pw[idx];
      // remove the exact weight along idx's path (reload: the descent may have left it)
#pragma unroll
      for (int h = 0; h < kMaxL; ++h) {
        if (h > T.top) continue;
        const int e = (int)((idx >> (6 * h)) & (kFan - 1));
        const int64_t node = idx >> (6 * (h + 1));
        double2* at = reinterpret_cast<double2*>(P[h] + node * kFan + 2 * lane);
        const double2 v = *at;
        if (2 * lane + 1 >= e) *at = make_double2(2 * lane >= e ? __dsub_rn(v.x, w) : v.x, __dsub_rn(v.y, w));
      }
    }
    if (lane == 0) {
      job.out[t] = idx;
      pw[idx] = 0.0;
    }
    __syncwarp();
    DRAW_T(t, 2)
  }
  DRAW_T(1025, 0)
}

bool launch_draw(const DrawJob* jobs, int njobs, unsigned* status, cudaStream_t st) {
  for (int k = 0; k < njobs && k < 2; ++k)
    if (jobs[k].len > kMaxDrawLen) return false;
  DrawJobs j{};
  size_t smem = 0;
  bool leaf_smem = true, up_global = false;
  for (int k = 0; k < njobs && k < 2; ++k) {
    j.j[k] = jobs[k];
    const int64_t len = jobs[k].len;
    const int64_t need = draw_smem_doubles(len);
    if (need == 0) up_global = true;
    if ((size_t)need * sizeof(double) > smem) smem = (size_t)need * sizeof(double);
    leaf_smem = leaf_smem && len <= kDrawSmemMaxLen;
  }
  if (up_global) smem = 0;  // one launch, one layout: both jobs keep their tree in global memory
  // the large-shared-memory attribute, once per device (cudaFuncSetAttribute is per device)
  static std::atomic<unsigned> attr_done{0};
  if (first_on_device(attr_done)) {
    // 227 KB minus the kernel's static shared memory (a failing attribute call
    // would otherwise surface as the launch's error)
    cudaFuncSetAttribute(k2_draw<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDrawSmemCap);
    cudaFuncSetAttribute(k2_draw<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDrawSmemCap);
  }
  ++::qcur::g_launches;
  if (leaf_smem && !up_global)
    k2_draw<true><<<njobs, 512, smem, st>>>(j, status, 0);
  else
    k2_draw<false><<<njobs, 512, smem, st>>>(j, status, up_global ? 1 : 0);
  return true;
}

}  // namespace qcur
