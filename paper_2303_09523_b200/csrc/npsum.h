// Host builder of numpy's pairwise-summation tree (DOUBLE_pairwise_sum in
// numpy/_core/src/umath/loops_utils.h.src): an array of n float64 is summed as
// sum(a, n2) + sum(a + n2, n - n2) with n2 = n/2 rounded down to a multiple of
// 8 while n > 128; a leaf of <= 128 elements uses eight strided accumulators
// combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then its n % 8 tail in order.
// Header-only so the CPU tests can check it against numpy (tests/native).
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

namespace vk {

struct NpSumTreeHost {
  std::vector<int32_t> leaf_off;     // [nleaf + 1]
  std::vector<int32_t> node_lr;      // [nnode][2] flat children (leaf i -> i, node j -> nleaf + j)
  std::vector<int32_t> level;        // [nlevel + 1] node ranges by height
};

inline NpSumTreeHost build_npsum_tree(int64_t m) {
  NpSumTreeHost t;
  std::vector<int> height;                 // per internal node
  std::vector<int32_t> lr;
  // returns node id: < 0 -> leaf -(id+1), >= 0 -> internal node
  struct Rec {
    static int64_t go(int64_t off, int64_t n, std::vector<int32_t>& leaf_off, std::vector<int32_t>& lr,
                      std::vector<int>& height, int* h_out) {
      if (n <= 128) {
        leaf_off.push_back((int32_t)off);
        *h_out = 0;
        return -(int64_t)leaf_off.size();          // -(leaf index + 1)
      }
      int64_t n2 = n / 2;
      n2 -= n2 % 8;
      int hl = 0, hr = 0;
      const int64_t l = go(off, n2, leaf_off, lr, height, &hl);
      const int64_t r = go(off + n2, n - n2, leaf_off, lr, height, &hr);
      lr.push_back((int32_t)l);
      lr.push_back((int32_t)r);
      height.push_back(std::max(hl, hr) + 1);
      *h_out = height.back();
      return (int64_t)height.size() - 1;
    }
  };
  int h = 0;
  Rec::go(0, m, t.leaf_off, lr, height, &h);
  const int nleaf = (int)t.leaf_off.size();
  t.leaf_off.push_back((int32_t)m);
  const int nnode = (int)height.size();
  // children as flat indices: leaf i -> i, internal node j -> nleaf + j;
  // internal nodes renumbered by height so that a level's nodes are contiguous
  const int H = nnode ? *std::max_element(height.begin(), height.end()) : 0;
  std::vector<int> order;
  order.reserve(nnode);
  t.level.assign(1, 0);
  for (int lev = 1; lev <= H; ++lev) {
    for (int j = 0; j < nnode; ++j)
      if (height[j] == lev) order.push_back(j);
    t.level.push_back((int32_t)order.size());
  }
  std::vector<int32_t> newid(nnode);
  for (int i = 0; i < nnode; ++i) newid[order[i]] = i;
  auto flat = [&](int32_t c) { return c < 0 ? (-c - 1) : nleaf + newid[c]; };
  t.node_lr.resize((size_t)nnode * 2);
  for (int i = 0; i < nnode; ++i) {
    t.node_lr[2 * i + 0] = flat(lr[2 * order[i] + 0]);
    t.node_lr[2 * i + 1] = flat(lr[2 * order[i] + 1]);
  }
  return t;
}


// Warp decomposition of the same tree for the device: maximal subtrees of at
// most 32 leaves ("warp roots", contiguous leaf ranges in left-to-right order)
// are summed by one warp each -- lane i sums leaf i, then the subtree's
// internal nodes are added in height order -- and only the tree above the
// warp roots is left to the level-by-level kernel.  Same additions, same
// order: bit-identical to build_npsum_tree's evaluation.
struct NpSumWarpHost {
  std::vector<int32_t> leaf_off;     // [nleaf + 1] element offsets of the true leaves
  std::vector<int32_t> wr_leaf;      // [nwr + 1] first leaf of each warp root
  std::vector<int16_t> prog;         // [nwr][31]: children (lo byte, hi byte) of the
                                     // root's internal nodes in height order; local
                                     // ids: leaf i -> i, internal node j -> 32 + j
  std::vector<int8_t> nint;          // [nwr] internal nodes per warp root
  NpSumTreeHost top;                 // the tree above: its leaf i is warp root i
};

inline NpSumWarpHost build_npsum_warp(int64_t m) {
  struct Node { int64_t l = -1, r = -1; int leaf = -1; int nleaf = 0; int height = 0; };
  std::vector<Node> nodes;
  NpSumWarpHost w;
  struct Rec {
    static int go(int64_t off, int64_t n, std::vector<Node>& nodes, std::vector<int32_t>& leaf_off) {
      Node nd;
      if (n <= 128) {
        nd.leaf = (int)leaf_off.size();
        leaf_off.push_back((int32_t)off);
        nd.nleaf = 1;
        nodes.push_back(nd);
        return (int)nodes.size() - 1;
      }
      int64_t n2 = n / 2;
      n2 -= n2 % 8;
      const int l = go(off, n2, nodes, leaf_off);
      const int r = go(off + n2, n - n2, nodes, leaf_off);
      nd.l = l;
      nd.r = r;
      nd.nleaf = nodes[l].nleaf + nodes[r].nleaf;
      nd.height = std::max(nodes[l].height, nodes[r].height) + 1;
      nodes.push_back(nd);
      return (int)nodes.size() - 1;
    }
  };
  const int root = Rec::go(0, m, nodes, w.leaf_off);
  w.leaf_off.push_back((int32_t)m);
  // warp roots in left-to-right order; top-tree nodes recorded on the way
  std::vector<int> wr_node;
  std::vector<int> top_l, top_r, top_h;     // top internal nodes (child: < 0 -> warp root -(id+1))
  struct Top {
    static int go(int v, std::vector<Node>& nodes, std::vector<int>& wr_node, std::vector<int>& tl,
                  std::vector<int>& tr, std::vector<int>& th, int* h) {
      if (nodes[v].nleaf <= 32) {
        wr_node.push_back(v);
        *h = 0;
        return -(int)wr_node.size();
      }
      int hl = 0, hr = 0;
      const int a = go((int)nodes[v].l, nodes, wr_node, tl, tr, th, &hl);
      const int b = go((int)nodes[v].r, nodes, wr_node, tl, tr, th, &hr);
      tl.push_back(a);
      tr.push_back(b);
      th.push_back(std::max(hl, hr) + 1);
      *h = th.back();
      return (int)th.size() - 1;
    }
  };
  int htop = 0;
  Top::go(root, nodes, wr_node, top_l, top_r, top_h, &htop);
  const int nwr = (int)wr_node.size();
  // each warp root: its leaves and internal nodes (height order)
  for (int i = 0; i < nwr; ++i) {
    const int v = wr_node[i];
    std::vector<int> inner;                  // internal nodes of the subtree
    std::vector<int> stack{v};
    int first_leaf = 1 << 30;
    while (!stack.empty()) {
      const int u = stack.back();
      stack.pop_back();
      if (nodes[u].leaf >= 0) { first_leaf = std::min(first_leaf, nodes[u].leaf); continue; }
      inner.push_back(u);
      stack.push_back((int)nodes[u].l);
      stack.push_back((int)nodes[u].r);
    }
    std::stable_sort(inner.begin(), inner.end(),
                     [&](int a, int b) { return nodes[a].height < nodes[b].height; });
    std::vector<int> local(nodes.size(), -1);
    for (size_t j = 0; j < inner.size(); ++j) local[inner[j]] = 32 + (int)j;
    auto lid = [&](int u) { return nodes[u].leaf >= 0 ? nodes[u].leaf - first_leaf : local[u]; };
    w.wr_leaf.push_back(first_leaf);
    w.nint.push_back((int8_t)inner.size());
    for (int j = 0; j < 31; ++j) {
      int16_t code = 0;
      if (j < (int)inner.size())
        code = (int16_t)(lid((int)nodes[inner[j]].l) | (lid((int)nodes[inner[j]].r) << 8));
      w.prog.push_back(code);
    }
  }
  w.wr_leaf.push_back((int32_t)w.leaf_off.size() - 1);
  // the top tree in NpSumTreeHost form (leaf i = warp root i)
  const int nnode = (int)top_h.size();
  NpSumTreeHost& t = w.top;
  t.leaf_off.assign((size_t)nwr + 1, 0);
  const int H = nnode ? *std::max_element(top_h.begin(), top_h.end()) : 0;
  std::vector<int> order;
  t.level.assign(1, 0);
  for (int lev = 1; lev <= H; ++lev) {
    for (int j = 0; j < nnode; ++j)
      if (top_h[j] == lev) order.push_back(j);
    t.level.push_back((int32_t)order.size());
  }
  std::vector<int32_t> newid(nnode);
  for (int i = 0; i < nnode; ++i) newid[order[i]] = i;
  auto flat = [&](int c) { return c < 0 ? (-c - 1) : nwr + newid[c]; };
  t.node_lr.resize((size_t)nnode * 2);
  for (int i = 0; i < nnode; ++i) {
    t.node_lr[2 * i + 0] = flat(top_l[order[i]]);
    t.node_lr[2 * i + 1] = flat(top_r[order[i]]);
  }
  return w;
}

}  // namespace vk
