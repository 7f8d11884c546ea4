// Host-side geometry of the plane-structured kriging path: which known
// planes each missing plane reads (kriging.py:444-455), the in-plane window
// kinds at the borders (kriging.py:334-342, 531-557), the distinct stencil
// systems to solve per Z sub-part (kriging.py:364-381), and the gap table the
// streaming prediction kernel walks.  All integer work, done once per plan.
#pragma once
#include <cstdint>
#include <map>
#include <string>
#include <vector>
#include "vk_common.h"

namespace vk {

struct PartInfo {
  int b, e;             // known-slice index range [b, e] (inclusive, trailing halo)
  int zlo, zhi;         // local grid z range [zlo, zhi] in output coordinates
  int64_t m;            // known voxels = samples for the variogram
  int pair_class;       // index into Geometry::pair_classes
};

struct PairClass {
  int64_t m;
  std::vector<int> zloc;   // local z of each known plane (sample coordinates)
};

struct StencilGeom {    // one (pattern, y-kind, x-kind) stencil
  int pattern, ky, kx;
  int n;                // neighbours
  std::vector<int8_t> taps;   // n x (ox, oy, oz_index) in reference order
  std::vector<int16_t> pad;   // n padded slots in [0, WPAD)
  int drift_cols;             // bitmask of kept drift columns (bit0 = 1, x, y, z)
};

struct Geometry {
  int H = 0, W = 0, T = 0, K = 0, S = 0;
  std::vector<int> known_z;            // [K]
  std::vector<PartInfo> parts;         // [S]
  std::vector<PairClass> pair_classes;
  // patterns: distinct tuples of plane offsets dz (target-relative)
  std::vector<std::vector<int>> patterns;
  // missing planes (output z not known): owner part, pattern, known indices
  std::vector<int> miss_z, miss_part, miss_pattern;
  std::vector<int> miss_planes;        // [n_miss * NPMAX] known-slice indices (-1 pad)
  // per-axis kind compaction: used axis kinds -> compact index
  int nkx = 0, nky = 0;
  int kx_map[NKIND1], ky_map[NKIND1];  // -1 if unused
  int kx_list[NKIND1], ky_list[NKIND1];
  int n_kinds() const { return nkx * nky; }
  // stencils (pattern x kind) and systems (part x stencil actually used)
  std::vector<StencilGeom> stencils;   // index = pattern * n_kinds + ky_c * nkx + kx_c
  std::vector<int> sys_part, sys_stencil;    // systems to solve
  // fast path: every gap k reads exactly planes (k, k+1) with G missing planes
  bool fast = false;
  int G = 0;
  std::vector<int> gap_part;           // [K-1]
  std::vector<int> gap_pattern;        // [(K-1) * G]
  std::string why_generic;             // reason the fast path is off
  int64_t n_missing_voxels() const { return (int64_t)miss_z.size() * H * W; }
};

// Builds the geometry; returns "" on success or an error message.
// Error prefixes: "NoKnownNeighbors:", "Unsupported:", "Invalid:".
std::string build_geometry(int H, int W, int T, const int* known_z, int K, int S,
                           int part_len, int drift, Geometry* g);

// Orders each part's systems so that the solved ones come first and marks
// the z-mirror / x<->y-transpose images of a solved system of the same part:
// der_src[i] = index of the solved system (-1: solved), der_flags[i] = bit 0
// mirror (planes reversed), bit 1 transpose (in-plane taps), bits 8.. planes
// of the pattern; sys_canon[s] = end of part s's solved systems (-1 for a
// part without systems).  Reorders g->sys_part / g->sys_stencil.
void canonical_systems(Geometry* g, std::vector<int>* sys_canon, std::vector<int32_t>* der_src,
                       std::vector<int32_t>* der_flags, int* n_derived);

}  // namespace vk
