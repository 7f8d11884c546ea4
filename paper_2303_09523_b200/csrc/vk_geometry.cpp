// Host geometry of the plane-structured kriging path (see vk_geometry.h).
#include "vk_geometry.h"

#include <algorithm>
#include <cmath>
#include <map>

namespace vk {

namespace {

// _window_bounds (kriging.py:334-342): half-open [c-(e/2-1), c+e/2] clamped.
void window(int c, int extent, int size, int* lo, int* hi) {
  *lo = std::max(0, c - (extent / 2 - 1));
  *hi = std::min(size, c + extent / 2 + 1);
}

// _choose_plane_window (kriging.py:444-455) on local coordinates.
bool choose_planes(int z, const std::vector<int>& kz, int depth, std::vector<int>* out) {
  static const int schedule[3] = {4, 8, 16};
  bool found = false;
  for (int ext : schedule) {
    int lo, hi;
    window(z, ext, depth, &lo, &hi);
    std::vector<int> sel;
    for (size_t i = 0; i < kz.size(); ++i)
      if (kz[i] >= lo && kz[i] < hi) sel.push_back((int)i);
    if (sel.empty()) continue;
    *out = sel;
    found = true;
    bool below = false, above = false;
    for (int i : sel) {
      below |= kz[i] < z;
      above |= kz[i] > z;
    }
    if (below && above) break;
  }
  return found;
}

// Rank of small integer-valued column sets (the _independent_columns test of
// kriging.py:145-156 is exact on integer offsets: dependent columns leave a
// ~1e-15 residual, independent ones >= O(1e-2) >> 1e-9).
int rank_of(const std::vector<std::vector<double>>& cols) {
  if (cols.empty()) return 0;
  const size_t n = cols[0].size();
  std::vector<std::vector<double>> a = cols;
  int rank = 0;
  std::vector<bool> used(n, false);
  for (size_t c = 0; c < a.size(); ++c) {
    size_t piv = n;
    double best = 1e-7;
    for (size_t r = 0; r < n; ++r)
      if (!used[r] && std::fabs(a[c][r]) > best) { best = std::fabs(a[c][r]); piv = r; }
    if (piv == n) continue;
    used[piv] = true;
    ++rank;
    for (size_t c2 = c + 1; c2 < a.size(); ++c2) {
      const double f = a[c2][piv] / a[c][piv];
      for (size_t r = 0; r < n; ++r) a[c2][r] -= f * a[c][r];
    }
  }
  return rank;
}

}  // namespace

std::string build_geometry(int H, int W, int T, const int* known_z, int K, int S,
                           int part_len, int drift, Geometry* g) {
  if (H < 1 || W < 1 || T < 1) return "Invalid: empty grid";
  if (K < 1) return "NoKnownNeighbors: grid has no known voxels at all";
  if (S < 1) return "Invalid: n_subparts must be >= 1";
  for (int i = 0; i < K; ++i) {
    if (known_z[i] < 0 || known_z[i] >= T) return "Invalid: known plane outside the grid";
    if (i > 0 && known_z[i] <= known_z[i - 1]) return "Invalid: known planes must increase";
  }
  g->H = H; g->W = W; g->T = T; g->K = K; g->S = S;
  g->known_z.assign(known_z, known_z + K);
  const int q = part_len > 0 ? part_len : K / S;
  if (q < 1) return "Invalid: more sub-parts than known slices";
  if ((int64_t)(S - 1) * q > K - 1) return "Invalid: part_len too large for the stack";
  std::vector<char> is_known(T, 0);
  for (int i = 0; i < K; ++i) is_known[known_z[i]] = 1;

  std::map<std::vector<int>, int> pattern_id;
  std::map<std::pair<int64_t, std::vector<int>>, int> class_id;
  g->parts.clear();
  for (int s = 0; s < S; ++s) {
    PartInfo p;
    p.b = s * q;
    p.e = (s < S - 1) ? (s + 1) * q : K - 1;
    p.zlo = (s == 0) ? 0 : known_z[p.b];
    p.zhi = (s == S - 1) ? T - 1 : known_z[p.e];
    p.m = (int64_t)(p.e - p.b + 1) * H * W;
    std::vector<int> zloc;
    for (int k = p.b; k <= p.e; ++k) zloc.push_back(known_z[k] - known_z[p.b]);
    auto key = std::make_pair(p.m, zloc);
    auto it = class_id.find(key);
    if (it == class_id.end()) {
      it = class_id.emplace(key, (int)g->pair_classes.size()).first;
      g->pair_classes.push_back(PairClass{p.m, zloc});
    }
    p.pair_class = it->second;
    g->parts.push_back(p);

    std::vector<int> kz;   // local z of the part's known planes
    for (int k = p.b; k <= p.e; ++k) kz.push_back(known_z[k] - p.zlo);
    const int depth = p.zhi - p.zlo + 1;
    for (int z = p.zlo; z <= p.zhi; ++z) {
      if (is_known[z]) continue;
      std::vector<int> sel;
      if (!choose_planes(z - p.zlo, kz, depth, &sel))
        return "NoKnownNeighbors: no known plane within reach of z=" + std::to_string(z);
      if ((int)sel.size() > NPMAX)
        return "Unsupported: a missing plane reads more than 8 known planes";
      std::vector<int> offs;
      for (int i : sel) offs.push_back(kz[i] - (z - p.zlo));
      auto pit = pattern_id.find(offs);
      if (pit == pattern_id.end()) {
        pit = pattern_id.emplace(offs, (int)g->patterns.size()).first;
        g->patterns.push_back(offs);
      }
      g->miss_z.push_back(z);
      g->miss_part.push_back(s);
      g->miss_pattern.push_back(pit->second);
      for (int i = 0; i < NPMAX; ++i)
        g->miss_planes.push_back(i < (int)sel.size() ? p.b + sel[i] : -1);
    }
  }

  // axis kinds actually present
  for (int i = 0; i < NKIND1; ++i) { g->kx_map[i] = g->ky_map[i] = -1; }
  g->nkx = g->nky = 0;
  for (int x = 0; x < W; ++x) {
    const int k = axis_kind(x, W);
    if (g->kx_map[k] < 0) { g->kx_map[k] = g->nkx; g->kx_list[g->nkx++] = k; }
  }
  for (int y = 0; y < H; ++y) {
    const int k = axis_kind(y, H);
    if (g->ky_map[k] < 0) { g->ky_map[k] = g->nky; g->ky_list[g->nky++] = k; }
  }

  // stencils for every (pattern, kind) and their drift column sets
  const int NK = g->n_kinds();
  g->stencils.clear();
  for (size_t p = 0; p < g->patterns.size(); ++p) {
    const std::vector<int>& offs = g->patterns[p];
    for (int yc = 0; yc < g->nky; ++yc) {
      for (int xc = 0; xc < g->nkx; ++xc) {
        StencilGeom sg;
        sg.pattern = (int)p;
        sg.ky = g->ky_list[yc];
        sg.kx = g->kx_list[xc];
        std::vector<double> cx, cy, cz;
        for (int pl = 0; pl < (int)offs.size(); ++pl)
          for (int oy = kind_lo(sg.ky); oy < kind_hi(sg.ky); ++oy)
            for (int ox = kind_lo(sg.kx); ox < kind_hi(sg.kx); ++ox) {
              sg.taps.push_back((int8_t)ox);
              sg.taps.push_back((int8_t)oy);
              sg.taps.push_back((int8_t)pl);
              sg.pad.push_back((int16_t)(pl * 16 + (oy + 1) * 4 + (ox + 1)));
              cx.push_back(ox); cy.push_back(oy); cz.push_back(offs[pl]);
            }
        sg.n = (int)sg.pad.size();
        sg.drift_cols = 1;
        if (drift == DRIFT_LINEAR) {
          std::vector<std::vector<double>> kept = {std::vector<double>(sg.n, 1.0)};
          const std::vector<double>* cand[3] = {&cx, &cy, &cz};
          for (int j = 0; j < 3; ++j) {
            std::vector<std::vector<double>> trial = kept;
            trial.push_back(*cand[j]);
            if (rank_of(trial) > (int)kept.size()) {
              kept.push_back(*cand[j]);
              sg.drift_cols |= 1 << (j + 1);
            }
          }
        }
        g->stencils.push_back(sg);
      }
    }
  }
  // systems: for every part, every pattern it uses, every kind
  g->sys_part.clear();
  g->sys_stencil.clear();
  std::vector<std::vector<char>> used(S, std::vector<char>(g->patterns.size(), 0));
  for (size_t i = 0; i < g->miss_z.size(); ++i) used[g->miss_part[i]][g->miss_pattern[i]] = 1;
  for (int s = 0; s < S; ++s)
    for (size_t p = 0; p < g->patterns.size(); ++p)
      if (used[s][p])
        for (int k = 0; k < NK; ++k) {
          g->sys_part.push_back(s);
          g->sys_stencil.push_back((int)p * NK + k);
        }

  // fast streaming path eligibility
  g->fast = false;
  g->G = 0;
  g->gap_part.clear();
  g->gap_pattern.clear();
  g->why_generic.clear();
  if (g->miss_z.empty()) { g->why_generic = "no missing planes"; return ""; }
  if (W % 4 != 0 || W < 8 || H < 4) { g->why_generic = "in-plane dims (need W%4==0, W>=8, H>=4)"; return ""; }
  if (K < 2) { g->why_generic = "fewer than 2 known planes"; return ""; }
  const int G = known_z[1] - known_z[0] - 1;
  for (int k = 0; k + 1 < K; ++k)
    if (known_z[k + 1] - known_z[k] - 1 != G) { g->why_generic = "irregular gaps"; return ""; }
  if (G < 1 || G > 8) { g->why_generic = "gap size outside 1..8"; return ""; }
  if ((int64_t)g->miss_z.size() != (int64_t)(K - 1) * G) { g->why_generic = "missing planes outside the known range"; return ""; }
  g->gap_part.assign(K - 1, -1);
  g->gap_pattern.assign((size_t)(K - 1) * G, -1);
  for (size_t i = 0; i < g->miss_z.size(); ++i) {
    const int z = g->miss_z[i];
    const int k = (z - known_z[0]) / (G + 1);
    const int j = z - known_z[k] - 1;
    const int* pl = &g->miss_planes[i * NPMAX];
    if (pl[0] != k || pl[1] != k + 1 || pl[2] != -1) {
      g->why_generic = "a missing plane reads planes other than its two brackets";
      g->gap_part.clear();
      g->gap_pattern.clear();
      return "";
    }
    g->gap_part[k] = g->miss_part[i];
    g->gap_pattern[(size_t)k * G + j] = g->miss_pattern[i];
  }
  g->fast = true;
  g->G = G;
  return "";
}

// Systems that are exact images of another system of the same part:
// the z-mirror of a plane pattern (offsets negated and reversed; the
// covariance is isotropic and the drift span {1, x, y, z} closed under
// z -> -z) and the x<->y transpose of a window kind.  Their weights are the
// solved system's with the planes reversed and / or the in-plane taps
// transposed (bit-identical variance), so only one system per orbit is
// solved (C4: 40 of 112 per part).  The reference solves each separately;
// the two solutions agree to solver rounding.  Within each part the solved
// systems come first.
void canonical_systems(Geometry* gp, std::vector<int>* sys_canon, std::vector<int32_t>* der_src,
                       std::vector<int32_t>* der_flags, int* n_derived) {
  Geometry& g = *gp;
  *n_derived = 0;
  {
    const int NPq = (int)g.patterns.size(), NKq = g.n_kinds();
    std::map<std::vector<int>, int> pat_index;
    for (int q = 0; q < NPq; ++q) pat_index[g.patterns[q]] = q;
    std::vector<int> pmir(NPq, -1), ktr(std::max(1, NKq), -1);
    for (int q = 0; q < NPq; ++q) {
      std::vector<int> m(g.patterns[q].rbegin(), g.patterns[q].rend());
      for (int& v : m) v = -v;
      auto it = pat_index.find(m);
      if (it != pat_index.end()) pmir[q] = it->second;
    }
    for (int yc = 0; yc < g.nky; ++yc)
      for (int xc = 0; xc < g.nkx; ++xc) {
        const int y2 = g.ky_map[g.kx_list[xc]], x2 = g.kx_map[g.ky_list[yc]];
        if (y2 >= 0 && x2 >= 0) ktr[yc * g.nkx + xc] = y2 * g.nkx + x2;
      }
    auto swapxy = [](int dc) { return (dc & 9) | ((dc & 2) << 1) | ((dc & 4) >> 1); };
    const int n = (int)g.sys_part.size();
    std::vector<int> order, src_of(n, -1), flag_of(n, 0);
    std::vector<int> new_part, new_stencil;
    sys_canon->assign(g.S, -1);                  // -1: part without systems (the caller fixes)
    int i0 = 0;
    while (i0 < n) {
      const int s = g.sys_part[i0];
      int i1 = i0;
      while (i1 < n && g.sys_part[i1] == s) ++i1;
      std::map<int, int> by_stc;                  // stencil -> system index in this part
      for (int i = i0; i < i1; ++i) by_stc[g.sys_stencil[i]] = i;
      for (int i = i0; i < i1; ++i) {
        const int stc = g.sys_stencil[i], pq = stc / std::max(1, NKq), kq = stc % std::max(1, NKq);
        const int dc = g.stencils[stc].drift_cols;
        int best = stc, bflag = 0;
        for (int fl = 1; fl < 4; ++fl) {
          const int p2 = (fl & 1) ? pmir[pq] : pq, k2 = (fl & 2) ? ktr[kq] : kq;
          if (p2 < 0 || k2 < 0) continue;
          const int stc2 = p2 * NKq + k2;
          if (!by_stc.count(stc2)) continue;
          if (g.patterns[p2].size() != g.patterns[pq].size()) continue;
          if (g.stencils[stc2].drift_cols != ((fl & 2) ? swapxy(dc) : dc)) continue;
          if (stc2 < best) { best = stc2; bflag = fl; }
        }
        if (best != stc) { src_of[i] = by_stc[best]; flag_of[i] = bflag | ((int)g.patterns[pq].size() << 8); }
      }
      // a system whose representative is itself derived solves itself (the
      // orbit minimum is always solved, so this only guards odd orbits)
      for (int i = i0; i < i1; ++i)
        if (src_of[i] >= 0 && src_of[src_of[i]] >= 0) { src_of[i] = -1; flag_of[i] = 0; }
      for (int i = i0; i < i1; ++i) if (src_of[i] < 0) order.push_back(i);
      (*sys_canon)[s] = (int)order.size();
      for (int i = i0; i < i1; ++i) if (src_of[i] >= 0) order.push_back(i);
      i0 = i1;
    }
    std::vector<int> new_index(n);
    for (int j = 0; j < n; ++j) new_index[order[j]] = j;
    der_src->assign(n, -1);
    der_flags->assign(n, 0);
    for (int j = 0; j < n; ++j) {
      const int i = order[j];
      new_part.push_back(g.sys_part[i]);
      new_stencil.push_back(g.sys_stencil[i]);
      if (src_of[i] >= 0) { (*der_src)[j] = new_index[src_of[i]]; (*der_flags)[j] = flag_of[i]; ++*n_derived; }
    }
    g.sys_part.swap(new_part);
    g.sys_stencil.swap(new_stencil);
  }
}

}  // namespace vk
