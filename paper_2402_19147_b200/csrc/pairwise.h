// Host-side compiler for numpy's pairwise-summation tree.
//
// numpy sums a contiguous run of n doubles as
//   n < 8        : sequential from 0.0
//   8 <= n <= 128: eight strided accumulators, combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
//                  then the n % 8 tail sequentially
//   n > 128      : split at n2 = n/2 - (n/2 % 8) and add the two halves.
// The reference relies on it for sq.sum() and sq.sum(axis=1) and the two
// normalisers (pkg/src/qcur/cur.py:144, 148, 150).  To reproduce those sums
// bit for bit on the GPU the tree is cut into "chunks" (subtrees of at most
// kChunkMax elements, evaluated by one CTA each from shared memory) and a
// "top" tree over chunk results (evaluated level by level).  Chunk trees are
// encoded as leaves + a postfix program; the top tree as (left,right) node
// pairs grouped by height.  oracle/numpy_order.c is the independent checker.
#pragma once
#include <stdint.h>
#include <map>
#include <vector>

namespace qcur {

constexpr int64_t kChunkMax = 8192;

struct ChunkPlan {
  int32_t len = 0;
  std::vector<int32_t> leaf_off, leaf_len;
  std::vector<int32_t> prog;  // >= 0: push leaf value; -1: pop b, pop a, push a + b
  // the same tree level by level: value slots [0, nleaves) are leaves, slot
  // nleaves + k is node k; nodes of height h are [lvl[h-1], lvl[h]) (h >= 1)
  std::vector<int32_t> node_l, node_r, lvl;
};

// Re-express a postfix program as (left, right) node pairs grouped by height,
// so a CTA can combine one whole level in parallel.
inline void levelize(ChunkPlan& p) {
  const int32_t nleaves = (int32_t)p.leaf_off.size();
  std::vector<int32_t> tl, tr, th;
  std::vector<std::pair<int32_t, int32_t>> st;  // (slot: leaf >= 0, node -(k+1)), height
  for (int32_t op : p.prog) {
    if (op >= 0) {
      st.push_back({op, 0});
    } else {
      auto b = st.back();
      st.pop_back();
      auto a = st.back();
      st.pop_back();
      const int32_t h = (a.second > b.second ? a.second : b.second) + 1;
      tl.push_back(a.first);
      tr.push_back(b.first);
      th.push_back(h);
      st.push_back({-(int32_t)tl.size(), h});
    }
  }
  int32_t maxh = 0;
  for (int32_t h : th) maxh = h > maxh ? h : maxh;
  std::vector<int32_t> order, newpos(tl.size());
  p.lvl.clear();
  for (int32_t h = 1; h <= maxh; ++h) {
    for (size_t k = 0; k < tl.size(); ++k)
      if (th[k] == h) order.push_back((int32_t)k);
    p.lvl.push_back((int32_t)order.size());
  }
  for (size_t q = 0; q < order.size(); ++q) newpos[order[q]] = (int32_t)q;
  auto remap = [&](int32_t s) { return s >= 0 ? s : nleaves + newpos[-s - 1]; };
  p.node_l.resize(order.size());
  p.node_r.resize(order.size());
  for (size_t q = 0; q < order.size(); ++q) {
    p.node_l[q] = remap(tl[order[q]]);
    p.node_r[q] = remap(tr[order[q]]);
  }
}

struct PairwiseProgram {
  int64_t length = 0;
  std::vector<int64_t> chunk_off;  // chunk start within the segment, in order
  std::vector<int32_t> chunk_plan;
  std::vector<ChunkPlan> plans;
  // top tree: value slots [0, nchunks) are chunk sums, slot nchunks + k is node k.
  std::vector<int32_t> node_l, node_r;
  std::vector<int32_t> level_ptr;  // nodes of height h: [level_ptr[h], level_ptr[h+1])
};

namespace detail {
inline void chunk_tree(int64_t off, int64_t n, ChunkPlan& p) {
  if (n <= 128) {
    p.prog.push_back((int32_t)p.leaf_off.size());
    p.leaf_off.push_back((int32_t)off);
    p.leaf_len.push_back((int32_t)n);
    return;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  chunk_tree(off, n2, p);
  chunk_tree(off + n2, n - n2, p);
  p.prog.push_back(-1);
}

struct TopBuilder {
  PairwiseProgram* pp;
  std::map<int64_t, int32_t> plan_of_len;
  std::vector<int32_t> tl, tr, th;  // unsorted internal nodes with heights
  // returns (slot, height); slots < 0 encode internal node -(k+1)
  std::pair<int64_t, int> build(int64_t off, int64_t n) {
    if (n <= kChunkMax) {
      auto it = plan_of_len.find(n);
      int32_t pid;
      if (it == plan_of_len.end()) {
        ChunkPlan cp;
        cp.len = (int32_t)n;
        chunk_tree(0, n, cp);
        levelize(cp);
        pid = (int32_t)pp->plans.size();
        pp->plans.push_back(std::move(cp));
        plan_of_len[n] = pid;
      } else {
        pid = it->second;
      }
      int64_t slot = (int64_t)pp->chunk_off.size();
      pp->chunk_off.push_back(off);
      pp->chunk_plan.push_back(pid);
      return {slot, 0};
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    auto a = build(off, n2);
    auto b = build(off + n2, n - n2);
    int h = (a.second > b.second ? a.second : b.second) + 1;
    int32_t k = (int32_t)tl.size();
    tl.push_back((int32_t)a.first);
    tr.push_back((int32_t)b.first);
    th.push_back(h);
    return {-(int64_t)k - 1, h};
  }
};
}  // namespace detail

inline PairwiseProgram compile_pairwise(int64_t n) {
  PairwiseProgram pp;
  pp.length = n;
  detail::TopBuilder tb;
  tb.pp = &pp;
  tb.build(0, n);
  int64_t nch = (int64_t)pp.chunk_off.size();
  int64_t nn = (int64_t)tb.tl.size();
  int maxh = 0;
  for (int h : tb.th) maxh = h > maxh ? h : maxh;
  // order nodes by height; remap slot ids
  std::vector<int32_t> order;
  order.reserve(nn);
  pp.level_ptr.assign(maxh + 2, 0);
  for (int h = 1; h <= maxh; ++h) {
    pp.level_ptr[h] = (int32_t)order.size();
    for (int64_t k = 0; k < nn; ++k)
      if (tb.th[k] == h) order.push_back((int32_t)k);
  }
  pp.level_ptr[maxh + 1] = (int32_t)order.size();
  std::vector<int32_t> newpos(nn);
  for (int64_t p = 0; p < nn; ++p) newpos[order[p]] = (int32_t)p;
  auto remap = [&](int32_t s) -> int32_t { return s >= 0 ? s : (int32_t)(nch + newpos[-(int64_t)s - 1]); };
  pp.node_l.resize(nn);
  pp.node_r.resize(nn);
  for (int64_t p = 0; p < nn; ++p) {
    pp.node_l[p] = remap(tb.tl[order[p]]);
    pp.node_r[p] = remap(tb.tr[order[p]]);
  }
  if (maxh == 0) pp.level_ptr.assign(2, 0);
  return pp;
}

}  // namespace qcur
