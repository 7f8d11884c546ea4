// Shared definitions for the volkrig-b200 kriging path (host + device).
#pragma once
#include <cstdint>
#include <cmath>

#if defined(__CUDACC__)
#define VK_HD __host__ __device__ __forceinline__
#else
#define VK_HD inline
#endif
// Out-of-line helpers of the serial fit chain: one copy per translation unit
// keeps the fit kernel's hot loop inside the instruction caches (the fully
// inlined form was 1.5 MB of SASS for one warp per SM).
// VK_HDC marks cold paths (never inlined); VK_HDN the mid-level routines of
// the fit and VK_DN their warp forms, inlined unless VK_FIT_OUTLINE is
// defined (out of line they are 22 % slower: call overhead and spills, not
// instruction-cache misses, dominate -- measured on C4).
#if defined(__CUDACC__)
#define VK_HDC static __host__ __device__ __noinline__
#if !defined(VK_FIT_OUTLINE)
#define VK_HDN VK_HD
#define VK_DN __device__ __forceinline__
#else
#define VK_HDN static __host__ __device__ __noinline__
#define VK_DN static __device__ __noinline__
#endif
#else
#define VK_HDC static __attribute__((noinline))
#define VK_HDN static __attribute__((noinline))
#endif

namespace vk {

constexpr int NPMAX = 8;              // max known planes read by one missing plane
constexpr int WPAD = NPMAX * 16;      // padded weights per system: [plane][oy+1][ox+1]
constexpr int MAX_BINS = 32;          // n_bins upper bound (reference default 15)
constexpr int NKIND1 = 6;             // (lo_off, hi_off) window kinds per axis

enum Kind { KIND_EXPONENTIAL = 0, KIND_GAUSSIAN = 1, KIND_SPHERICAL = 2 };
enum Drift { DRIFT_LINEAR = 0, DRIFT_CONSTANT = 1 };

// Per-part status codes written by kernels (mapped to vk_status on the host).
enum PartStatus : int32_t {
  PS_OK = 0,
  PS_SINGULAR = 1,
  PS_INSUFFICIENT = 2,
  PS_DEGENERATE = 3,
  PS_FIT_FAILED = 4,
  PS_PAIRS_SHORT = 5,
  PS_NEED_SCALAR_FIT = 6,   // internal: handed to the scalar TRF kernel
  PS_NONFINITE = 7,         // a known value of the part is NaN / inf
};

// Variogram model parameters as the reference's VariogramModel
// (kriging.py:44-57): nugget, sill, range_len.
struct Model {
  double nugget, sill, range_len;
};

// gamma(h) -- kriging.py:59-72.  h == 0 -> 0.
VK_HD double semivariance(int kind, const Model& m, double h) {
  if (h == 0.0) return 0.0;
  const double psill = m.sill - m.nugget;
  const double r = m.range_len;
  double shape;
  if (kind == KIND_EXPONENTIAL) {
    shape = 1.0 - exp((-3.0 * h) / r);
  } else if (kind == KIND_GAUSSIAN) {
    const double t = h / r;
    shape = 1.0 - exp(-3.0 * (t * t));
  } else {
    const double t = fmin(h / r, 1.0);
    shape = 1.5 * t - 0.5 * pow(t, 3.0);
  }
  return m.nugget + psill * shape;
}

// gamma(h) for a compile-time kind, without the h == 0 branch folded into
// control flow (same arithmetic as semivariance): straight-line code the
// device fit can interleave across independent evaluations.
template <int KIND>
VK_HD double semivariance_k(const Model& m, double h) {
  const double psill = m.sill - m.nugget;
  const double r = m.range_len;
  double shape;
  if constexpr (KIND == KIND_EXPONENTIAL) {
    shape = 1.0 - exp((-3.0 * h) / r);
  } else if constexpr (KIND == KIND_GAUSSIAN) {
    const double t = h / r;
    shape = 1.0 - exp(-3.0 * (t * t));
  } else {
    const double t = fmin(h / r, 1.0);
    shape = 1.5 * t - 0.5 * pow(t, 3.0);
  }
  return h == 0.0 ? 0.0 : m.nugget + psill * shape;
}

// C(h) = sill - gamma(h); unit white noise when sill <= 0 -- kriging.py:74-84.
VK_HD double covariance(int kind, const Model& m, double h) {
  if (m.sill <= 0.0) return h == 0.0 ? 1.0 : 0.0;
  return m.sill - semivariance(kind, m, h);
}

// In-plane window kind of coordinate c on an axis of length n: the clamped
// window [max(0,c-1), min(n,c+3)) of kriging.py:334-342 with extent 4,
// encoded by (lo - c in {-1,0}, hi - c in {1,2,3}) -> 0..5.  Interior = 2.
VK_HD int axis_kind(int c, int n) {
  const int lo = (c > 0) ? -1 : 0;
  const int hi = (n - c < 3) ? (n - c) : 3;
  return (lo + 1) * 3 + (hi - 1);
}
VK_HD int kind_lo(int k) { return k / 3 - 1; }
VK_HD int kind_hi(int k) { return k % 3 + 1; }
constexpr int AXIS_INTERIOR = 2;

}  // namespace vk
