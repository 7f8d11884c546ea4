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

}  // namespace vk
