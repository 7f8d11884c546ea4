// Prediction kernels of the plane-structured fill (kriging.py:499-557).
//
// predict_fast   : the production layout -- every missing plane reads its two
//                  bracketing known planes (k, k+1).  Persistent CTAs walk
//                  (in-plane tile, run of gaps) units; known-plane tiles are
//                  streamed into a 4-deep shared-memory ring by TMA
//                  (cp.async.bulk.tensor, OOB zero fill supplies the volume
//                  halo) so each known plane is read from HBM once per run.
//                  Units come from a guided dynamic schedule (FtSched: unit
//                  lengths halving from ~70 interpolated planes to single
//                  gaps, claimed from a global counter) and the ring runs
//                  across units, so all CTAs end within one short unit.
//                  The G missing planes of a gap come in z-mirror pairs
//                  (j, G-1-j) whose interior stencils are mirror images, so
//                  each pair is computed from S = A+B and D = A-B (exact in
//                  fp64) with one symmetric and one antisymmetric 16-tap
//                  stencil -- 16 instead of 32 DFMA per voxel.  Each thread
//                  keeps one 7-wide row of S and D in registers and
//                  accumulates 4 columns x G planes; results are clamped to
//                  the part's known range and stored as 128-bit streaming
//                  stores; the known planes are copied through from the
//                  same tiles.  Border rows (y in {0, H-2, H-1}) use their
//                  clamped-window kind's stencils (zero taps outside the
//                  window); the three border columns are computed by one
//                  thread per (row, column) with their own kinds.
// predict_generic: any plane pattern (up to 8 planes, any dims); one thread
//                  per missing voxel, reading the known planes through L1/L2.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdlib>
#include <cstdio>
#include <algorithm>
#include <type_traits>
#include "vk_kernels.h"
#include "vk_tma.cuh"

namespace vk {

namespace {

__device__ __forceinline__ int compact_kind(const int32_t* kmap, int nkx, int x, int y, int W, int H) {
  return kmap[NKIND1 + axis_kind(y, H)] * nkx + kmap[axis_kind(x, W)];
}

template <typename Acc>
__device__ __forceinline__ Acc tap_fma(double w, float v, Acc acc);
template <>
__device__ __forceinline__ double tap_fma<double>(double w, float v, double acc) {
  return fma(w, (double)v, acc);
}
template <>
__device__ __forceinline__ float tap_fma<float>(double w, float v, float acc) {
  return fmaf((float)w, v, acc);
}

// --------------------------------------------------------------------------
// generic path
// --------------------------------------------------------------------------
template <typename Acc>
__global__ void __launch_bounds__(256) predict_generic_kernel(PredictArgs a) {
  const int i = blockIdx.y;
  const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= a.P) return;
  const int y = (int)(pix / a.W), x = (int)(pix - (int64_t)y * a.W);
  const int z = a.miss_z[i], s = a.miss_part[i], p = a.miss_pattern[i];
  const int kind = compact_kind(a.kmap, a.nkx, x, y, a.W, a.H);
  const int64_t slot = ((int64_t)s * a.NP + p) * a.NK + kind;
  const double* w = a.weights + slot * WPAD;
  const int kx = axis_kind(x, a.W), ky = axis_kind(y, a.H);
  const int x0 = kind_lo(kx), x1 = kind_hi(kx), y0 = kind_lo(ky), y1 = kind_hi(ky);
  Acc acc = (Acc)0;
  for (int pl = 0; pl < NPMAX; ++pl) {
    const int k = a.miss_planes[i * NPMAX + pl];
    if (k < 0) break;
    const float* plane = a.known + (int64_t)k * a.P;
    for (int oy = y0; oy < y1; ++oy)
      for (int ox = x0; ox < x1; ++ox)
        acc = tap_fma<Acc>(w[pl * 16 + (oy + 1) * 4 + (ox + 1)],
                           __ldg(plane + (int64_t)(y + oy) * a.W + (x + ox)), acc);
  }
  const Acc lo = (Acc)a.lohi[2 * s], hi = (Acc)a.lohi[2 * s + 1];
  acc = acc < lo ? lo : acc;
  acc = acc > hi ? hi : acc;
  a.out[(int64_t)z * a.P + pix] = (float)acc;
  if (a.var) a.var[(int64_t)z * a.P + pix] = a.svar[slot];
}

__global__ void __launch_bounds__(256) copy_known_kernel(PredictArgs a) {
  const int k = blockIdx.y;
  const int64_t z = a.known_z[k];
  const int64_t n4 = a.P / 4;
  const float4* src = reinterpret_cast<const float4*>(a.known + (int64_t)k * a.P);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.P; i += (int64_t)gridDim.x * blockDim.x) {
    if ((a.P & 3) == 0) {
      if (i < n4) {
        reinterpret_cast<float4*>(a.out + z * a.P)[i] = src[i];
        if (a.var) {
          double2 zz = make_double2(0.0, 0.0);
          reinterpret_cast<double2*>(a.var + z * a.P)[2 * i] = zz;
          reinterpret_cast<double2*>(a.var + z * a.P)[2 * i + 1] = zz;
        }
      }
    } else {
      a.out[z * a.P + i] = a.known[(int64_t)k * a.P + i];
      if (a.var) a.var[z * a.P + i] = 0.0;
    }
  }
}

// --------------------------------------------------------------------------
// fast streaming path
// --------------------------------------------------------------------------
#ifndef VK_FT_WARPS
#define VK_FT_WARPS 8
#define VK_FT_TY 32
#define VK_FT_MINB 2
#endif
constexpr int FT_WARPS = VK_FT_WARPS;
constexpr int FT_THREADS = FT_WARPS * 32;
constexpr int FT_TY = VK_FT_TY;            // tile rows (warps x row steps)
constexpr int FT_SY = FT_TY + 3;           // smem rows: y0-1 .. y0+33
constexpr int FT_BUF_FLOATS = ((FT_SX * FT_SY * 4 + 127) / 128) * 128 / 4;
// Occupancy by gap size: with G <= 4 missing planes the accumulators fit 80
// registers, so three CTAs share an SM (3-deep ring); larger G keeps 128
// registers, two CTAs and a 4-deep ring (C5 fp32: 58.9 -> 60.6 % of the HBM
// roofline; C4 (G = 7) spills at 80 registers and stays at two CTAs).
#ifndef VK_FT_F32_MINB3
#define VK_FT_F32_MINB3 0                // fp32 kernel: three CTAs per SM at every G
#endif
#ifndef VK_FT_NSTAGE
#define VK_FT_NSTAGE 4                   // ring depth at two CTAs per SM
#endif
__host__ __device__ constexpr int ft_stages(int G, bool f32 = false) {
  return (G <= 4 || (f32 && VK_FT_F32_MINB3)) ? 3 : VK_FT_NSTAGE;
}
__host__ __device__ constexpr int ft_minb(int G, bool f32 = false) {
  return (G <= 4 || (f32 && VK_FT_F32_MINB3)) ? 3 : VK_FT_MINB;
}
constexpr int FT_WPARTS = 4;             // parts whose stencils a unit stages ...
constexpr int FT_WSLOTS = 12;            // ... in (part, row kind) slots: four parts unless one tile
                                         // holds all three border rows (H <= FT_TY: three parts)
constexpr int FT_MAXU = 32;              // gaps per unit (per-gap metadata staged in shared memory)

template <typename Acc>
struct AccVec;
template <>
struct AccVec<double> {
  static __device__ __forceinline__ double cvt(float v) { return (double)v; }
};
template <>
struct AccVec<float> {
  static __device__ __forceinline__ float cvt(float v) { return v; }
};

__device__ __forceinline__ void st_cs_f4(float* p, float4 v) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
               "f"(v.w)
               : "memory");
}

// predicated streaming stores (one instruction each, no branch)
__device__ __forceinline__ void st_cs_f4_if(float* p, const float* v, bool c) {
  asm volatile("{.reg .pred q; setp.ne.u32 q, %5, 0; @q st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};}"
               ::"l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "r"((unsigned)c) : "memory");
}
__device__ __forceinline__ void st_cs_f2_if(float* p, float x, float y, bool c) {
  asm volatile("{.reg .pred q; setp.ne.u32 q, %3, 0; @q st.global.cs.v2.f32 [%0], {%1, %2};}"
               ::"l"(p), "f"(x), "f"(y), "r"((unsigned)c) : "memory");
}
__device__ __forceinline__ void st_cs_f1_if(float* p, float x, bool c) {
  asm volatile("{.reg .pred q; setp.ne.u32 q, %2, 0; @q st.global.cs.f32 [%0], %1;}"
               ::"l"(p), "f"(x), "r"((unsigned)c) : "memory");
}

// predicated 128-bit streaming stores of two doubles (the variance volume)
__device__ __forceinline__ void st_cs_d2_if(double* p, double x, double y, bool c) {
  asm volatile("{.reg .pred q; setp.ne.u32 q, %3, 0; @q st.global.cs.v2.f64 [%0], {%1, %2};}"
               ::"l"(p), "d"(x), "d"(y), "r"((unsigned)c) : "memory");
}
__device__ __forceinline__ void st_cs_d1_if(double* p, double x, bool c) {
  asm volatile("{.reg .pred q; setp.ne.u32 q, %2, 0; @q st.global.cs.f64 [%0], %1;}"
               ::"l"(p), "d"(x), "r"((unsigned)c) : "memory");
}

template <int COLS>
__device__ __forceinline__ void st_cs_cols(float* p, const float* v) {
  if constexpr (COLS == 4) {
    st_cs_f4(p, make_float4(v[0], v[1], v[2], v[3]));
  } else {
    asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" ::"l"(p), "f"(v[0]), "f"(v[1]) : "memory");
  }
}

#ifndef VK_FT_COLS
#define VK_FT_COLS 4
#endif
#ifndef VK_FT_SYM32
#define VK_FT_SYM32 1                    // x<->y symmetric interior rows in the fp32 kernel
#endif
#ifndef VK_FT_SPLIT
#define VK_FT_SPLIT 1                    // fp64 kernel: exact-split FFMA2 symmetric rows (integer planes)
#endif
#ifndef VK_FT_L2PF
#define VK_FT_L2PF 0                     // planes ahead of a ring load to prefetch into L2 (0: none;
                                         // C4: 1 or 2 planes ahead 0.627 vs 0.626 ms, no effect)
#endif
#ifndef VK_FT_MIDF64
#define VK_FT_MIDF64 0                   // exact-split rows: the middle plane's stencil on the FP64 pipe
                                         // (C4: 0.645 vs 0.601 ms -- the 40 F2F conversions per row
                                         // step cost more than the 80 FMA-pipe cycles they free)
#endif
#ifndef VK_FT_ROWROT
#define VK_FT_ROWROT 0                   // rows rotate over the warps with the gap (C4: 0.626 vs 0.619 ms)
#endif
#ifndef VK_FT_SYM32_MAXG
#define VK_FT_SYM32_MAXG 4               // ... for gaps of up to this many missing planes
#endif

// Mirror-pair stencil table for the streaming kernel (one thread per
// (part, kind, tap)).  Missing planes j and G-1-j are z-mirrors: their
// stencils satisfy wA_j = wB_{G-1-j}, wB_j = wA_{G-1-j} (isotropic covariance;
// drift span closed under z -> -z).  With a, b the mirror-averaged plane-A /
// plane-B stencils of j, out_j = a*A + b*B = K+*(A+B) + K-*(A-B) and
// out_{G-1-j} = K+*(A+B) - K-*(A-B) with K+- = (a +- b)/2: one symmetric and
// one antisymmetric 16-tap stencil per pair instead of four.  Layout
// [s][kind][tap][K+_0, K-_0, ..., K_mid, pad] so one 128-bit load fetches a
// pair.  Taps outside a clamped border window are 0 in the solved weights.
// Per-tap layout of the mirror-pair stencils.  fp64 (DFMA, one stencil per
// instruction): [K+_0, K-_0, K+_1, K-_1, ..., K_mid, pad].  fp32 (FFMA2, two
// stencils per instruction against one broadcast S or D value): the symmetric
// stencils together, then the antisymmetric ones, each run padded to a pair:
// [K+_0, K+_1, ..., K+_{n-1}, K_mid, (pad) | K-_0, ..., K-_{n-1}, (pad)].
template <int G, typename Acc>
struct StLayout {
  static constexpr int NPAIR = G / 2;
  static constexpr bool MID = (G & 1) != 0;
  static constexpr bool PAIRED = std::is_same<Acc, float>::value;
  static constexpr int NPP = (NPAIR + (MID ? 1 : 0) + 1) & ~1;   // paired: symmetric run
  static constexpr int NMP = (NPAIR + 1) & ~1;                   // paired: antisymmetric run
  static constexpr int NSTP = PAIRED ? NPP + NMP : ((2 * NPAIR + (MID ? 1 : 0) + 1) & ~1);
  static __host__ __device__ constexpr int plus(int p) { return PAIRED ? p : 2 * p; }
  static __host__ __device__ constexpr int minus(int p) { return PAIRED ? NPP + p : 2 * p + 1; }
  static __host__ __device__ constexpr int mid() { return PAIRED ? NPAIR : 2 * NPAIR; }
};

template <int G, typename Acc>
__global__ void __launch_bounds__(256) fast_stencil_kernel(PredictArgs a) {
  using L = StLayout<G, Acc>;
  constexpr int NPAIR = L::NPAIR, NSTP = L::NSTP;
  constexpr bool MID = L::MID;
  const int per_part = a.NK * 16;
  const int n = (a.part1 - a.part0) * per_part;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int s = a.part0 + i / per_part, r = i - (i / per_part) * per_part;
    const int kind = r >> 4, t = r & 15;
    Acc* dst = reinterpret_cast<Acc*>(a.kpm) + (((size_t)s * a.NK + kind) * 16 + t) * NSTP;
    for (int q = 0; q < NSTP; ++q) dst[q] = (Acc)0;
    // interior kind: stencils are x<->y symmetric up to solver rounding
    // (isotropic covariance, drift span closed under x <-> y); the table
    // holds the transposition average so the streaming kernel may pair taps
    const int kin = a.kmap[NKIND1 + AXIS_INTERIOR] * a.nkx + a.kmap[AXIS_INTERIOR];
    const bool symm = kind == kin && a.kmap[AXIS_INTERIOR] >= 0 && a.kmap[NKIND1 + AXIS_INTERIOR] >= 0;
    const int tt = (t & 3) * 4 + (t >> 2);                 // transposed tap
    // patterns are identical for every gap on the fast path (each missing
    // plane reads exactly its two bracketing known planes)
    for (int pr = 0; pr < NPAIR + (MID ? 1 : 0); ++pr) {
      const int pj = a.gap_pattern[pr], pm = a.gap_pattern[G - 1 - pr];
      const double* wj = a.weights + (((int64_t)s * a.NP + pj) * a.NK + kind) * WPAD;
      const double* wm = a.weights + (((int64_t)s * a.NP + pm) * a.NK + kind) * WPAD;
      double av = 0.5 * (wj[t] + wm[16 + t]);
      double bv = 0.5 * (wj[16 + t] + wm[t]);
      if (symm && tt != t) {
        av = 0.5 * (av + 0.5 * (wj[tt] + wm[16 + tt]));
        bv = 0.5 * (bv + 0.5 * (wj[16 + tt] + wm[tt]));
      }
      if (pr < NPAIR) {
        dst[L::plus(pr)] = (Acc)(0.5 * (av + bv));
        dst[L::minus(pr)] = (Acc)(0.5 * (av - bv));
      } else {
        dst[L::mid()] = (Acc)(0.5 * (av + bv));
      }
    }
  }
}

// Exact-split stencils for the fp64 symmetric rows (integer planes).  For
// each mirror pair j of part s (interior kind) the stencils K+_j, K-_j are
// split as K = Kh + Kl with Kh = round(K 2^e) 2^-e on a grid 2^-e shared by
// the pair, e chosen so that 2 Vmax (sum|K+_j| + sum|K-_j|) 2^e <= 2^23
// (Vmax = max |known| of the part).  For integer pair sums v, every product
// Kh v and every partial sum of the Kh parts -- and Sh +- Dh -- is then a
// multiple of 2^-e below 2^24 2^-e: exact in fp32.  Kl = fl32(K - Kh)
// (|Kl| <= 2^-e-1) carries the rest with an fp32 rounding error below
// ~1e-8 of the range for |known| < 2^17, so one FFMA2 per (tap, stencil,
// column) on the FMA pipe replaces a DFMA plus the fp32 -> fp64 conversion
// of its operand (F2F, a quarter-rate MIO instruction: 22 % of the fp64
// kernel's stall samples).  Layout per (part, tap): the run layout of
// StLayout<G, float> with (hi, lo) float pairs -- [K+_0 .. K+_{n-1}, K_mid,
// (pad) | K-_0 .. K-_{n-1}, (pad)] -- after the part's [NK][16][8] fp64
// table block of kpm.
template <int G>
__global__ void __launch_bounds__(128) split_stencil_kernel(PredictArgs a) {
  using L = StLayout<G, double>;
  using LR = StLayout<G, float>;
  constexpr int NPAIR = L::NPAIR;
  constexpr bool MID = L::MID;
  constexpr int NJ = NPAIR + (MID ? 1 : 0);
  const int n = (a.part1 - a.part0) * NJ;
  const int kin = a.kmap[NKIND1 + AXIS_INTERIOR] * a.nkx + a.kmap[AXIS_INTERIOR];
  if (a.kmap[AXIS_INTERIOR] < 0 || a.kmap[NKIND1 + AXIS_INTERIOR] < 0) return;
  const double* kpm = reinterpret_cast<const double*>(a.kpm);
  float2* spl = reinterpret_cast<float2*>(const_cast<double*>(kpm) + split_table_offset(a.S, a.NK));
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int s = a.part0 + i / NJ, j = i % NJ;
    const double* w = kpm + ((size_t)s * a.NK + kin) * 16 * L::NSTP;
    const bool pair = j < NPAIR;
    const int ip = pair ? L::plus(j) : L::mid(), im = L::minus(j);
    const double vmax = fmax(fabs(a.lohi[2 * s]), fabs(a.lohi[2 * s + 1]));
    double bsum = 0.0;
    for (int t = 0; t < 16; ++t) bsum += fabs(w[t * L::NSTP + ip]) + (pair ? fabs(w[t * L::NSTP + im]) : 0.0);
    const double bound = 2.0 * vmax * bsum;
    int e = 0;
    if (bound > 0.0) {
      int x;
      frexp(bound, &x);                                    // bound < 2^x
      e = 23 - x;
    }
    const double sc = ldexp(1.0, e), isc = ldexp(1.0, -e);
    float2* dst = spl + (size_t)s * 16 * LR::NSTP;
    for (int t = 0; t < 16; ++t) {
      const double kp = w[t * L::NSTP + ip];
      const double hp = rint(kp * sc) * isc;
      dst[t * LR::NSTP + (pair ? LR::plus(j) : LR::mid())] = make_float2((float)hp, (float)(kp - hp));
      if (pair) {
        const double km = w[t * L::NSTP + im];
        const double hm = rint(km * sc) * isc;
        dst[t * LR::NSTP + LR::minus(j)] = make_float2((float)hm, (float)(km - hm));
      }
    }
    if (j == 0)                                            // padding entries
      for (int t = 0; t < 16; ++t)
        for (int q = 0; q < LR::NSTP; ++q) {
          const bool used = (q < NJ) || (q >= LR::NPP && q < LR::NPP + NPAIR);
          if (!used) dst[t * LR::NSTP + q] = make_float2(0.f, 0.f);
        }
  }
}

// packed fp32x2 FMA (FFMA2) on 64-bit register pairs; a pair built from one
// value twice becomes the instruction's broadcast operand
__device__ __forceinline__ uint64_t f2pack(float x, float y) {
  return (uint64_t)__float_as_uint(x) | ((uint64_t)__float_as_uint(y) << 32);
}
__device__ __forceinline__ float f2lo(uint64_t v) { return __uint_as_float((uint32_t)v); }
__device__ __forceinline__ float f2hi(uint64_t v) { return __uint_as_float((uint32_t)(v >> 32)); }
__device__ __forceinline__ uint64_t f2fma(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}


// L2 policy of a known-plane tile load (plane k of a run ending at plane ke).
// Evict-first everywhere (VK_FT_EF_MODE 1, default) keeps the concurrent
// fits' lines in L2: C4 fp64 step 2.33 -> 2.19 ms, fp32 2.28 -> 2.15 ms; the
// kernel alone loses its halo / run-boundary re-reads from L2 (fp64 0.814 ->
// 0.818 ms, fp32 0.622 -> 0.658 ms); sparing the run's last plane (mode 2)
// measured the same as mode 1.  Mode 0: the default policy everywhere.
#ifndef VK_FT_EF_MODE
#define VK_FT_EF_MODE 1
#endif
__device__ __forceinline__ bool ft_evict_first(int k, int ke) {
  (void)k; (void)ke;
  return VK_FT_EF_MODE != 0;
}

// Guided unit schedule of one launch.  Units are (tile, run of gaps); every
// tile's gap range is cut into levels of decreasing unit length and the units
// are handed out level by level (tile fastest) from a global counter: the
// first gridDim.x units statically, the rest to whichever CTA asks next, so
// all CTAs -- and both CTAs of an SM -- stay busy until the pool is empty and
// the end-time spread is one short unit.  (A static equal split left CTAs
// running 333-644 us of a 644 us launch on C4: whichever CTA of an SM the
// warp schedulers favour finishes early and its sibling, alone on the SM, is
// latency-bound; SMs were idle 8 % of the launch.)
constexpr int FT_NLV = 6;
struct FtSched {
  int n_lv;
  int len[FT_NLV];          // gaps per unit of the level
  int off[FT_NLV + 1];      // the level's first gap within a tile's range (off[n_lv] = gaps)
  int base[FT_NLV + 1];     // the level's first unit index (base[n_lv] = units in all)
};
__device__ __forceinline__ bool ft_unit(const FtSched& sc, int u, int n_tiles, int gap0, int& tile, int& kb,
                                        int& ke) {
  if (u >= sc.base[sc.n_lv]) return false;
  int l = 0;
  while (l + 1 < sc.n_lv && u >= sc.base[l + 1]) ++l;
  const int idx = u - sc.base[l];
  tile = idx % n_tiles;
  kb = gap0 + sc.off[l] + (idx / n_tiles) * sc.len[l];
  ke = min(kb + sc.len[l], gap0 + sc.off[l + 1]);
  return true;
}

#ifdef VK_FT_DIAG
// development diagnostic (tools/cta_times.py, variant builds only): per CTA
// {smid, first tile, start, end} of the last streaming launch (globaltimer ns)
__device__ unsigned long long g_cta_diag[4 * 1024];
#endif

// Streaming kernel.  No CTA-wide barrier inside a unit: each warp waits only
// for the TMA of the two planes its gap reads and, when done with plane k,
// releases it; the last warp to release a ring slot refills it with plane
// k + FT_STAGES.  Warps therefore drift apart by up to a few gaps, so the
// FP64 pipe of an SM sub-partition sees a mix of DFMA-heavy and
// load/convert/store phases instead of all warps in lock step.
template <int G, typename Acc, bool VAR, int COLS = VK_FT_COLS>
__global__ void __launch_bounds__(FT_THREADS, ft_minb(G, std::is_same<Acc, float>::value))
    predict_fast_kernel(const __grid_constant__ CUtensorMap tmap, PredictArgs a, int n_tiles_x,
                        int n_tiles, const FtSched sch) {
  using L = StLayout<G, Acc>;
  constexpr int NPAIR = L::NPAIR;
  constexpr bool MID = L::MID;
  constexpr int NSTP = L::NSTP;                            // padded: 16-byte aligned taps
  // staged stencils use the run layout of StLayout<G, float> for both
  // accumulators ([K+_0 .. K+_{n-1}, K_mid, pad | K-_0 .. K-_{n-1}, pad]): the
  // fp64 table in global memory is interleaved and is permuted while staging
  using LR = StLayout<G, float>;
  constexpr int NPP = LR::NPP, NMP = LR::NMP;
  constexpr int NSTP_S = NSTP > LR::NSTP ? NSTP : LR::NSTP;
  constexpr bool F64 = std::is_same<Acc, double>::value;
  constexpr int FT_STAGES = ft_stages(G, std::is_same<Acc, float>::value);
  extern __shared__ __align__(128) float ring[];           // FT_STAGES x FT_BUF_FLOATS
  __shared__ __align__(8) uint64_t full[FT_STAGES];
  __shared__ int released[FT_STAGES];                      // warps done with the slot's plane
  // mirror-pair stencils of the unit's parts (<= FT_WPARTS) x row kinds of the
  // tile (interior x kind), double-buffered by unit so staging the next
  // unit's needs no barrier beyond the unit-start one
  __shared__ __align__(16) Acc s_w[2][FT_WSLOTS * 16 * NSTP_S];
  // exact-split interior stencils ((hi, lo) float pairs, run layout) of the
  // unit's parts for the fp64 symmetric rows (split_stencil_kernel)
  constexpr bool SPLIT = F64 && VK_FT_SPLIT;
  __shared__ __align__(16) uint64_t s_ws[SPLIT ? 2 : 1][SPLIT ? FT_WPARTS * 16 * LR::NSTP : 2];
  // per-gap metadata of the unit (part, output plane, exact-S/D flag) and the
  // clamp range of its parts, staged with the stencils: read per gap from
  // global memory they were a chain of dependent loads (gap -> part -> range)
  // on every warp's critical path (5 % of the kernel's stall samples)
  __shared__ int s_gpart[2][FT_MAXU], s_gz[2][FT_MAXU], s_gflag[2][FT_MAXU];
  __shared__ float2 s_plohi[2][FT_WPARTS];
  __shared__ int s_unit[2][4];                             // unit of iteration uc + 1: tile, kb, ke, valid
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int H = a.H, W = a.W;
  const int64_t P = a.P;
#ifdef VK_FT_DIAG
  unsigned long long diag_t0 = 0;
  if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(diag_t0));
#endif
  if (tid == 0) {
    for (int i = 0; i < FT_STAGES; ++i) {
      mbar_init(&full[i], 1);
      released[i] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t tile_bytes = FT_SX * FT_SY * 4;
  uint32_t load_seq = 0;                                   // loads issued so far
  const int n_gaps = a.K - 1;
  const Acc* kpm = reinterpret_cast<const Acc*>(a.kpm);
  const int kint = a.kmap[AXIS_INTERIOR];                  // compact interior x-kind
  // warp layout: WX column groups x WY rows per row step
  constexpr int WX = (FT_TX / COLS) / 32;
  constexpr int WY = FT_WARPS / WX;
  const int wx = warp % WX, wy = warp / WX;
  const int lc = lane + 32 * wx;                           // column group in the tile

  // Units come from the guided schedule (FtSched): the first is unit
  // blockIdx.x; while a unit is staged, thread 0 claims the next one, so its
  // first planes can be loaded as the current unit's ring slots drain.
  int tile = 0, kb = 0, ke = 0, n_prev = 0;
  bool have = ft_unit(sch, blockIdx.x, n_tiles, a.gap0, tile, kb, ke);
  for (int uc = 0; have; ++uc) {
    if (tid == 0) {
      int t2 = 0, kb2 = 0, ke2 = 0;
      const bool v = ft_unit(sch, (int)gridDim.x + atomicAdd(a.work, 1), n_tiles, a.gap0, t2, kb2, ke2);
      s_unit[(uc + 1) & 1][0] = t2;
      s_unit[(uc + 1) & 1][1] = kb2;
      s_unit[(uc + 1) & 1][2] = ke2;
      s_unit[(uc + 1) & 1][3] = v;
    }
    const int tx = tile % n_tiles_x, ty = tile / n_tiles_x;
    const int x0 = tx * FT_TX, y0 = ty * FT_TY;
    const int ty1 = min(H, y0 + FT_TY), tx1 = min(W, x0 + FT_TX);
    int nbc = 0, bcol[3] = {0, 0, 0};                      // border columns in this tile
    int nky = 1, kyl[4] = {AXIS_INTERIOR, 0, 0, 0};        // row kinds: interior first
    {
      const int cc[3] = {0, W - 2, W - 1};
      for (int q = 0; q < 3; ++q)
        if (cc[q] >= x0 && cc[q] < tx1) bcol[nbc++] = cc[q];
      const int rc[3] = {0, H - 2, H - 1};
      for (int q = 0; q < 3; ++q)
        if (rc[q] >= y0 && rc[q] < ty1) kyl[nky++] = axis_kind(rc[q], H);
    }
    const int s_first = a.gap_part[kb];
    const int npu = a.gap_part[ke - 1] - s_first + 1;       // <= FT_WPARTS (host caps chunk)
    if (npu > FT_WPARTS || npu * nky > FT_WSLOTS) __trap();
    Acc* sw = s_w[uc & 1];
    {
      const int per_k = 16 * NSTP_S, n = npu * nky * per_k;
      for (int i = tid; i < n; i += FT_THREADS) {
        const int e = i % per_k, q = i / per_k;
        const int t = e / NSTP_S, d = e - t * NSTP_S;
        const int iy = q % nky, pi = q / nky;
        const int kind = a.kmap[NKIND1 + kyl[iy]] * a.nkx + kint;
        int src = d;                                       // fp32: already the run layout
        if constexpr (F64) {
          if (d < NPP) src = d < NPAIR ? L::plus(d) : ((MID && d == NPAIR) ? L::mid() : -1);
          else src = (d - NPP < NPAIR) ? L::minus(d - NPP) : -1;
        }
        sw[i] = src >= 0 ? kpm[(((size_t)(s_first + pi) * a.NK + kind) * 16 + t) * NSTP + src] : (Acc)0;
      }
      if constexpr (SPLIT) {
        const uint64_t* spl = reinterpret_cast<const uint64_t*>(a.kpm) + split_table_offset(a.S, a.NK) +
                              (size_t)s_first * 16 * LR::NSTP;
        uint64_t* sws = s_ws[uc & 1];
        for (int i = tid; i < npu * 16 * LR::NSTP; i += FT_THREADS) sws[i] = spl[i];
      }
      if (ke - kb > FT_MAXU) __trap();
      for (int i = tid; i < ke - kb; i += FT_THREADS) {
        s_gpart[uc & 1][i] = a.gap_part[kb + i];
        s_gz[uc & 1][i] = a.known_z[kb + i];
        s_gflag[uc & 1][i] =
            a.sd_inexact != nullptr && (a.sd_inexact[kb + i] | a.sd_inexact[kb + i + 1]) == 0;
      }
      if (tid >= FT_THREADS - FT_WPARTS && tid - (FT_THREADS - FT_WPARTS) < npu) {
        const int pi = tid - (FT_THREADS - FT_WPARTS);
        s_plohi[uc & 1][pi] = make_float2((float)a.lohi[2 * (s_first + pi)], (float)a.lohi[2 * (s_first + pi) + 1]);
      }
    }
    const uint32_t seq0 = load_seq;
    const int n_planes = ke - kb + 1;
    // load `sq` of the CTA's plane sequence: plane kp of the tile at (xt, yt)
    // (evict-first: the tiles must not displace the concurrent fits'
    // instruction and stack lines from L2)
    auto issue = [&](uint32_t sq, int xt, int yt, int kp) {
      float* buf = ring + (sq % FT_STAGES) * FT_BUF_FLOATS;
      fence_proxy_async();
      mbar_expect_tx(&full[sq % FT_STAGES], tile_bytes);
      if (ft_evict_first(kp, kp))
        tma_load_3d_ef(buf, &tmap, &full[sq % FT_STAGES], xt, yt, kp, l2_evict_first_policy());
      else
        tma_load_3d(buf, &tmap, &full[sq % FT_STAGES], xt, yt, kp);
    };
    __syncthreads();                                       // stencils staged, next unit known
    // The ring runs across units: the last warp to release load q issues load
    // q + FT_STAGES, of this unit or -- past its end -- of the next one.  What
    // is left for the unit start are the loads whose slot was last used
    // before the previous unit (all of them for the CTA's first unit).
    if (tid == 0)
      for (int i = 0; i < min(FT_STAGES - n_prev, n_planes); ++i) issue(seq0 + i, x0 - 4, y0 - 1, kb + i);
    load_seq += n_planes;
    const int gx = x0 + COLS * lc;
    const bool col_ok = gx < W;
    const bool xb0 = (gx == 0), xb1 = (gx + COLS > W - 2);  // group holds border columns
    for (int k = kb; k < ke; ++k) {
      const uint32_t sq_a = seq0 + (k - kb), sq_b = sq_a + 1;
      const int s = s_gpart[uc & 1][k - kb];
      const Acc* wpart = kpm + (size_t)s * a.NK * 16 * NSTP;
      // the clamp commutes with the f32 rounding (lo, hi are f32 values and
      // rounding is monotone), so it is applied after the conversion
      const float2 plh = s_plohi[uc & 1][s - s_first];
      const float lo = plh.x, hi = plh.y;
      const int64_t zk = s_gz[uc & 1][k - kb];
      const bool copy_b = (k == n_gaps - 1);
      mbar_wait(&full[sq_a % FT_STAGES], (sq_a / FT_STAGES) & 1);
      mbar_wait(&full[sq_b % FT_STAGES], (sq_b / FT_STAGES) & 1);
      const float* bufA = ring + (sq_a % FT_STAGES) * FT_BUF_FLOATS;
      const float* bufB = ring + (sq_b % FT_STAGES) * FT_BUF_FLOATS;
      const bool sd_exact = s_gflag[uc & 1][k - kb] != 0;
      // x<->y symmetric interior rows (fp64, integer planes): pair sums of S
      // and D are exact in fp32 when |known| < 2^22 (|S1 + S2| <= 2^24)
      const bool sym_ok = F64 && sd_exact && fmaxf(fabsf(lo), fabsf(hi)) < 4194304.f;
      // one 7-wide row of the two planes' tiles (columns x-1 .. x+COLS+1)
      auto load_rows = [&](int rr, float* fa, float* fb) {
        const float* ra = bufA + rr * FT_SX + COLS * lc;
        const float* rb = bufB + rr * FT_SX + COLS * lc;
        if constexpr (COLS == 4) {
          const float4 a0 = *reinterpret_cast<const float4*>(ra);
          const float4 a1 = *reinterpret_cast<const float4*>(ra + 4);
          const float2 a2 = *reinterpret_cast<const float2*>(ra + 8);
          const float4 b0 = *reinterpret_cast<const float4*>(rb);
          const float4 b1 = *reinterpret_cast<const float4*>(rb + 4);
          const float2 b2 = *reinterpret_cast<const float2*>(rb + 8);
          fa[0] = a0.w; fa[1] = a1.x; fa[2] = a1.y; fa[3] = a1.z; fa[4] = a1.w; fa[5] = a2.x; fa[6] = a2.y;
          fb[0] = b0.w; fb[1] = b1.x; fb[2] = b1.y; fb[3] = b1.z; fb[4] = b1.w; fb[5] = b2.x; fb[6] = b2.y;
        } else {
          const float a0 = ra[3];
          const float2 a1 = *reinterpret_cast<const float2*>(ra + 4);
          const float2 a2 = *reinterpret_cast<const float2*>(ra + 6);
          const float b0 = rb[3];
          const float2 b1 = *reinterpret_cast<const float2*>(rb + 4);
          const float2 b2 = *reinterpret_cast<const float2*>(rb + 6);
          fa[0] = a0; fa[1] = a1.x; fa[2] = a1.y; fa[3] = a2.x; fa[4] = a2.y;
          fb[0] = b0; fb[1] = b1.x; fb[2] = b1.y; fb[3] = b2.x; fb[4] = b2.y;
        }
      };
      // stores of one row step: known planes through, G predictions clamped
      auto emit = [&](int gy, int kyr, const float* selfA, const float* selfB, auto out_of) {
        const int64_t pix = (int64_t)gy * W + gx;
        // known planes pass through bit-exactly (kriging.py:481)
        st_cs_cols<COLS>(a.out + zk * P + pix, selfA);
        if (copy_b) st_cs_cols<COLS>(a.out + (zk + G + 1) * P + pix, selfB);
        if (VAR) {
          // known planes: zero variance, 128-bit streaming stores (32-byte
          // aligned: gx % 4 == 0 and W % 4 == 0 on the streaming path)
          if constexpr (COLS == 4) {
            double* v0 = a.var + zk * P + pix;
            st_cs_d2_if(v0, 0.0, 0.0, true);
            st_cs_d2_if(v0 + 2, 0.0, 0.0, true);
            double* v1 = a.var + (zk + G + 1) * P + pix;
            st_cs_d2_if(v1, 0.0, 0.0, copy_b);
            st_cs_d2_if(v1 + 2, 0.0, 0.0, copy_b);
          } else {
            for (int c = 0; c < COLS; ++c) a.var[zk * P + pix + c] = 0.0;
            if (copy_b)
              for (int c = 0; c < COLS; ++c) a.var[(zk + G + 1) * P + pix + c] = 0.0;
          }
        }
        float* dst = a.out + (zk + 1) * P + pix;
#pragma unroll
        for (int j = 0; j < G; ++j, dst += P) {
          float o[COLS];
#pragma unroll
          for (int c = 0; c < COLS; ++c) o[c] = fminf(fmaxf(out_of(j, c), lo), hi);
          if constexpr (COLS == 4) {
            // border columns (x = 0, W-2, W-1) belong to the border pass:
            // predicated stores, no divergent branch (groups at x = 0 and
            // x = W-4 hold them; W % 4 == 0 on the streaming path).  (A
            // CTA-uniform branch to one plain store for tiles without border
            // columns measured slower: C4 0.632 vs 0.619 ms.)
            st_cs_f4_if(dst, o, !xb0 && !xb1);
            st_cs_f1_if(dst + 1, o[1], xb0);
            st_cs_f2_if(dst + 2, o[2], o[3], xb0);
            st_cs_f2_if(dst, o[0], o[1], xb1 && !xb0);
            if constexpr (VAR) {
              const double vj = a.svar[((int64_t)s * a.NP + a.gap_pattern[k * G + j]) * a.NK +
                                       a.kmap[NKIND1 + kyr] * a.nkx + kint];
              double* vdst = a.var + (zk + 1 + j) * P + pix;
              st_cs_d2_if(vdst, vj, vj, !xb0);                 // columns 0, 1 (not at x = 0)
              st_cs_d2_if(vdst + 2, vj, vj, !xb1);             // columns 2, 3 (not at x = W-2)
              st_cs_d1_if(vdst + 1, vj, xb0);                  // x = 1 of the first group
            }
          } else {
            double* vdst = VAR ? a.var + (zk + 1 + j) * P + pix : nullptr;
            const double vj =
                VAR ? a.svar[((int64_t)s * a.NP + a.gap_pattern[k * G + j]) * a.NK +
                               a.kmap[NKIND1 + kyr] * a.nkx + kint]
                    : 0.0;
            if (!xb0 && !xb1) {
              st_cs_cols<COLS>(dst, o);
              if (VAR)
                for (int c = 0; c < COLS; ++c) vdst[c] = vj;
            } else {
#pragma unroll
              for (int c = 0; c < COLS; ++c) {
                const int xx = gx + c;
                if (xx >= 1 && xx <= W - 3) {
                  dst[c] = o[c];
                  if (VAR) vdst[c] = vj;
                }
              }
            }
          }
        }
      };
      // general row step: 16 taps, one window row at a time
      auto row_general = [&](auto exact_c, int r, int gy, int kyr) {
        constexpr bool EXACT = decltype(exact_c)::value;
        int iy = 0;                                        // row kind (border rows of edge tiles)
        for (int q = 1; q < nky; ++q)
          if (kyl[q] == kyr) iy = q;
        const Acc* wk = sw + (size_t)((s - s_first) * nky + iy) * 16 * NSTP_S;
        constexpr bool PAIRED = L::PAIRED;
        constexpr int QP = PAIRED ? NPP / 2 : 1, QM = (PAIRED && NMP > 0) ? NMP / 2 : 1;
        Acc accS[NPAIR > 0 ? NPAIR : 1][COLS], accD[NPAIR > 0 ? NPAIR : 1][COLS], accC[COLS];
        uint64_t aP[QP][COLS], aM[QM][COLS];               // fp32: stencil pairs (FFMA2)
#pragma unroll
        for (int c = 0; c < COLS; ++c) {
          accC[c] = (Acc)0;
#pragma unroll
          for (int p = 0; p < NPAIR; ++p) { accS[p][c] = (Acc)0; accD[p][c] = (Acc)0; }
#pragma unroll
          for (int q = 0; q < QP; ++q) aP[q][c] = 0;
#pragma unroll
          for (int q = 0; q < QM; ++q) aM[q][c] = 0;
        }
        float selfA[COLS], selfB[COLS];
#pragma unroll
        for (int oy = -1; oy <= 2; ++oy) {
          float fa[COLS + 3], fb[COLS + 3];
          load_rows(r + 1 + oy, fa, fb);
          if (oy == 0) {
#pragma unroll
            for (int c = 0; c < COLS; ++c) { selfA[c] = fa[c + 1]; selfB[c] = fb[c + 1]; }
          }
          Acc S[COLS + 3], D[COLS + 3];                    // exact in fp64
#pragma unroll
          for (int i = 0; i < COLS + 3; ++i) {
            if constexpr (EXACT) {
              // integer data below 2^23: fa +- fb is exact in fp32, so the two
              // DADDs leave the FP64 pipe (same S, D bits)
              S[i] = (Acc)(fa[i] + fb[i]);
              D[i] = (Acc)(fa[i] - fb[i]);
            } else {
              const Acc x = AccVec<Acc>::cvt(fa[i]), y = AccVec<Acc>::cvt(fb[i]);
              S[i] = x + y;
              D[i] = x - y;
            }
          }
#pragma unroll
          for (int ox = -1; ox <= 2; ++ox) {
            const int t = (oy + 1) * 4 + (ox + 1);
            const Acc* wt = wk + t * NSTP_S;
            if constexpr (PAIRED) {
              // two stencils per FFMA2 against the broadcast S (or D) value
#pragma unroll
              for (int q = 0; q < NPP / 2; ++q) {
                const uint64_t w2 = reinterpret_cast<const uint64_t*>(wt)[q];
#pragma unroll
                for (int c = 0; c < COLS; ++c)
                  aP[q][c] = f2fma(w2, f2pack(S[c + ox + 1], S[c + ox + 1]), aP[q][c]);
              }
#pragma unroll
              for (int q = 0; q < NMP / 2; ++q) {
                const uint64_t w2 = reinterpret_cast<const uint64_t*>(wt + NPP)[q];
#pragma unroll
                for (int c = 0; c < COLS; ++c)
                  aM[q][c] = f2fma(w2, f2pack(D[c + ox + 1], D[c + ox + 1]), aM[q][c]);
              }
            } else {
              double kp[NPP > 0 ? NPP : 2], km[NMP > 0 ? NMP : 2];
#pragma unroll
              for (int q = 0; q < NPP / 2; ++q) {
                const double2 v = reinterpret_cast<const double2*>(wt)[q];
                kp[2 * q] = v.x;
                kp[2 * q + 1] = v.y;
              }
#pragma unroll
              for (int q = 0; q < NMP / 2; ++q) {
                const double2 v = reinterpret_cast<const double2*>(wt + NPP)[q];
                km[2 * q] = v.x;
                km[2 * q + 1] = v.y;
              }
#pragma unroll
              for (int p = 0; p < NPAIR; ++p) {
#pragma unroll
                for (int c = 0; c < COLS; ++c) {
                  accS[p][c] = fma(kp[p], S[c + ox + 1], accS[p][c]);
                  accD[p][c] = fma(km[p], D[c + ox + 1], accD[p][c]);
                }
              }
              if (MID) {
#pragma unroll
                for (int c = 0; c < COLS; ++c) accC[c] = fma(kp[NPAIR], S[c + ox + 1], accC[c]);
              }
            }
          }
        }
        emit(gy, kyr, selfA, selfB, [&](int j, int c) -> float {
          Acc t;
          if constexpr (PAIRED) {
            auto pv = [&](int i) { return (i & 1) ? f2hi(aP[i >> 1][c]) : f2lo(aP[i >> 1][c]); };
            auto mv = [&](int i) { return (i & 1) ? f2hi(aM[i >> 1][c]) : f2lo(aM[i >> 1][c]); };
            if (MID && j == NPAIR) t = pv(NPAIR);
            else if (j < NPAIR) t = pv(j) + mv(j);
            else t = pv(G - 1 - j) - mv(G - 1 - j);
          } else {
            if (MID && j == NPAIR) t = accC[c];
            else if (j < NPAIR) t = accS[j][c] + accD[j][c];
            else t = accS[G - 1 - j][c] - accD[G - 1 - j][c];
          }
          return (float)t;
        });
      };
      // x<->y symmetric interior row step (fp64, integer planes).  Interior
      // stencils satisfy K(ox, oy) = K(oy, ox) (isotropic covariance; the
      // drift span is closed under x <-> y; the table is symmetrised), so
      // sum_t K_t v_t = sum_diag K v + sum_{ox<oy} K (v(ox,oy) + v(oy,ox)):
      // 10 DFMA per stencil instead of 16.  The 4 x (COLS+3) windows of S
      // and then D are held in fp32 registers (exact integers) so the
      // transposed partner of each tap is a register, and each pair sum is
      // exact in fp32 (|known| < 2^22) before its one conversion.
      auto row_sym = [&](int r, int gy) {
        const Acc* wk = sw + (size_t)((s - s_first) * nky + 0) * 16 * NSTP_S;   // interior rows: iy = 0
        constexpr int QP = NPP / 2, QM = NMP > 0 ? NMP / 2 : 1;
        double accS[F64 && NPAIR > 0 ? NPAIR : 1][COLS], accD[F64 && NPAIR > 0 ? NPAIR : 1][COLS];
        double accC[F64 ? COLS : 1];
        uint64_t aP[F64 ? 1 : QP][COLS], aM[F64 ? 1 : QM][COLS];   // fp32: stencil pairs (FFMA2)
        float selfA[COLS], selfB[COLS];
        float Wv[4][COLS + 3];
#pragma unroll
        for (int c = 0; c < COLS; ++c) {
          if constexpr (F64) {
            accC[c] = 0.0;
#pragma unroll
            for (int p = 0; p < NPAIR; ++p) { accS[p][c] = 0.0; accD[p][c] = 0.0; }
          } else {
#pragma unroll
            for (int q = 0; q < QP; ++q) aP[q][c] = 0;
#pragma unroll
            for (int q = 0; q < QM; ++q) aM[q][c] = 0;
          }
        }
#pragma unroll
        for (int ph = 0; ph < 2; ++ph) {                   // 0: S = A + B, 1: D = A - B
#pragma unroll
          for (int oy = -1; oy <= 2; ++oy) {
            float fa[COLS + 3], fb[COLS + 3];
            load_rows(r + 1 + oy, fa, fb);
            if (ph == 0 && oy == 0) {
#pragma unroll
              for (int c = 0; c < COLS; ++c) { selfA[c] = fa[c + 1]; selfB[c] = fb[c + 1]; }
            }
#pragma unroll
            for (int i = 0; i < COLS + 3; ++i) Wv[oy + 1][i] = ph == 0 ? fa[i] + fb[i] : fa[i] - fb[i];
          }
#pragma unroll
          for (int by = 0; by < 4; ++by) {
#pragma unroll
            for (int bx = 0; bx <= by; ++bx) {              // tap (ox, oy) = (bx - 1, by - 1)
              const Acc* wt = wk + (by * 4 + bx) * NSTP_S + (ph == 0 ? 0 : NPP);
              if constexpr (F64) {
                constexpr int NW = NPP > NMP ? NPP : NMP;
                double kw[NW > 0 ? NW : 2];
#pragma unroll
                for (int q = 0; q < (ph == 0 ? NPP : NMP) / 2; ++q) {
                  const double2 v = reinterpret_cast<const double2*>(wt)[q];
                  kw[2 * q] = v.x;
                  kw[2 * q + 1] = v.y;
                }
#pragma unroll
                for (int c = 0; c < COLS; ++c) {
                  const float v = bx == by ? Wv[by][c + bx] : Wv[by][c + bx] + Wv[bx][c + by];
                  const double pd = (double)v;
                  if (ph == 0) {
#pragma unroll
                    for (int p = 0; p < NPAIR; ++p) accS[p][c] = fma(kw[p], pd, accS[p][c]);
                    if (MID) accC[c] = fma(kw[NPAIR], pd, accC[c]);
                  } else {
#pragma unroll
                    for (int p = 0; p < NPAIR; ++p) accD[p][c] = fma(kw[p], pd, accD[p][c]);
                  }
                }
              } else {
                uint64_t kw[QP > QM ? QP : QM];
#pragma unroll
                for (int q = 0; q < (ph == 0 ? QP : (NMP > 0 ? QM : 0)); ++q)
                  kw[q] = reinterpret_cast<const uint64_t*>(wt)[q];
#pragma unroll
                for (int c = 0; c < COLS; ++c) {
                  const float v = bx == by ? Wv[by][c + bx] : Wv[by][c + bx] + Wv[bx][c + by];
                  const uint64_t vv = f2pack(v, v);
                  if (ph == 0) {
#pragma unroll
                    for (int q = 0; q < QP; ++q) aP[q][c] = f2fma(kw[q], vv, aP[q][c]);
                  } else if (NMP > 0) {
#pragma unroll
                    for (int q = 0; q < QM; ++q) aM[q][c] = f2fma(kw[q], vv, aM[q][c]);
                  }
                }
              }
            }
          }
        }
        emit(gy, AXIS_INTERIOR, selfA, selfB, [&](int j, int c) -> float {
          if constexpr (F64) {
            double t;
            if (MID && j == NPAIR) t = accC[c];
            else if (j < NPAIR) t = accS[j][c] + accD[j][c];
            else t = accS[G - 1 - j][c] - accD[G - 1 - j][c];
            return (float)t;
          } else {
            auto pv = [&](int i) { return (i & 1) ? f2hi(aP[i >> 1][c]) : f2lo(aP[i >> 1][c]); };
            auto mv = [&](int i) { return (i & 1) ? f2hi(aM[i >> 1][c]) : f2lo(aM[i >> 1][c]); };
            if (MID && j == NPAIR) return pv(NPAIR);
            if (j < NPAIR) return pv(j) + mv(j);
            return pv(G - 1 - j) - mv(G - 1 - j);
          }
        });
      };
      // exact-split symmetric row step (fp64 gate, integer planes): the same
      // 10-tap x<->y symmetric form, each stencil as (hi, lo) fp32 parts on
      // one FFMA2 against the broadcast pair sum (split_stencil_kernel: the
      // hi sums are exact, the lo sums carry < ~1e-8 of the range), so no
      // operand is converted to fp64 and no DFMA is issued
      auto row_split = [&](int r, int gy) {
        const uint64_t* wk = s_ws[uc & 1] + (size_t)(s - s_first) * 16 * LR::NSTP;
        // VK_FT_MIDF64 (off: measured slower): the middle plane (odd G) has
        // no antisymmetric part; its stencil as DFMA on the otherwise idle
        // FP64 pipe, from the fp64 table's symmetrised K_mid, with the pair
        // sums converted once (F2F), takes 80 of a row step's ~740 FMA-pipe
        // cycles off the binding pipe.
        constexpr bool MF = MID && VK_FT_MIDF64;
        constexpr int NJ = NPAIR + (MID && !MF ? 1 : 0);
        const Acc* wkd = sw + (size_t)((s - s_first) * nky + 0) * 16 * NSTP_S + NPAIR;   // K_mid, interior rows
        uint64_t aS[NJ > 0 ? NJ : 1][COLS], aD[NPAIR > 0 ? NPAIR : 1][COLS];
        double accC[MF ? COLS : 1];
        float selfA[COLS], selfB[COLS];
        float Wv[4][COLS + 3];
#pragma unroll
        for (int c = 0; c < COLS; ++c) {
#pragma unroll
          for (int q = 0; q < NJ; ++q) aS[q][c] = 0;
#pragma unroll
          for (int q = 0; q < NPAIR; ++q) aD[q][c] = 0;
          if (MF) accC[c] = 0.0;
        }
#pragma unroll
        for (int ph = 0; ph < 2; ++ph) {                   // 0: S = A + B, 1: D = A - B
#pragma unroll
          for (int oy = -1; oy <= 2; ++oy) {
            float fa[COLS + 3], fb[COLS + 3];
            load_rows(r + 1 + oy, fa, fb);
            if (ph == 0 && oy == 0) {
#pragma unroll
              for (int c = 0; c < COLS; ++c) { selfA[c] = fa[c + 1]; selfB[c] = fb[c + 1]; }
            }
#pragma unroll
            for (int i = 0; i < COLS + 3; ++i) Wv[oy + 1][i] = ph == 0 ? fa[i] + fb[i] : fa[i] - fb[i];
          }
#pragma unroll
          for (int by = 0; by < 4; ++by) {
#pragma unroll
            for (int bx = 0; bx <= by; ++bx) {
              const uint64_t* wt = wk + (by * 4 + bx) * LR::NSTP + (ph == 0 ? 0 : NPP);
              constexpr int NW = NJ > NPAIR ? NJ : NPAIR;
              uint64_t kw[NW > 0 ? NW : 1];
#pragma unroll
              for (int q = 0; q < (ph == 0 ? NJ : NPAIR); ++q) kw[q] = wt[q];
              double kmid = 0.0;
              if (MF && ph == 0) kmid = (double)wkd[(by * 4 + bx) * NSTP_S];
#pragma unroll
              for (int c = 0; c < COLS; ++c) {
                const float v = bx == by ? Wv[by][c + bx] : Wv[by][c + bx] + Wv[bx][c + by];
                const uint64_t vv = f2pack(v, v);
                if (ph == 0) {
#pragma unroll
                  for (int q = 0; q < NJ; ++q) aS[q][c] = f2fma(kw[q], vv, aS[q][c]);
                  if (MF) accC[c] = fma(kmid, (double)v, accC[c]);
                } else {
#pragma unroll
                  for (int q = 0; q < NPAIR; ++q) aD[q][c] = f2fma(kw[q], vv, aD[q][c]);
                }
              }
            }
          }
        }
        emit(gy, AXIS_INTERIOR, selfA, selfB, [&](int j, int c) -> float {
          if (MID && j == NPAIR) {
            if constexpr (MF) return (float)accC[c];
            else return f2lo(aS[NJ - 1][c]) + f2hi(aS[NJ - 1][c]);
          }
          const int q = j < NPAIR ? j : G - 1 - j;
          // hi parts: exact (common 2^-e grid of the pair); then one rounding
          const float h = j < NPAIR ? f2lo(aS[q][c]) + f2lo(aD[q][c]) : f2lo(aS[q][c]) - f2lo(aD[q][c]);
          const float l = j < NPAIR ? f2hi(aS[q][c]) + f2hi(aD[q][c]) : f2hi(aS[q][c]) - f2hi(aD[q][c]);
          return h + l;
        });
      };
      auto row_steps = [&](auto exact_c, auto sym_c, auto split_c) {
        constexpr bool SYM = decltype(sym_c)::value;
        constexpr bool SPL = decltype(split_c)::value;
#pragma unroll 1
        for (int rs = 0; rs < FT_TY / WY; ++rs) {
          // tile row (warp-uniform); the rows rotate over the warps with the
          // gap so a tile's border rows (general 16-tap form) are not always
          // the same warps'
          const int r = (VK_FT_ROWROT ? (wy + k) % WY : wy) + rs * WY;
          const int gy = y0 + r;
          if (gy >= H || !col_ok) continue;
          const int kyr = axis_kind(gy, H);
          if (SPL && kyr == AXIS_INTERIOR) row_split(r, gy);
          else if (SYM && kyr == AXIS_INTERIOR) row_sym(r, gy);
          else row_general(exact_c, r, gy, kyr);
        }
      };
      // exact split (row_split): integer planes with |known| < 2^17, and the
      // final fp32 rounding (<= 1 ulp of |known| from the reference's) well
      // inside 1e-6 of the range: max |known| <= 4 (hi - lo)
      const float vmx = fmaxf(fabsf(lo), fabsf(hi));
      const bool split_ok = SPLIT && sym_ok && vmx < 131072.f && vmx <= 4.f * (hi - lo);
      if constexpr (F64) {
        if (split_ok) row_steps(std::true_type{}, std::true_type{}, std::true_type{});
        else if (sym_ok) row_steps(std::true_type{}, std::true_type{}, std::false_type{});
        else if (sd_exact) row_steps(std::true_type{}, std::false_type{}, std::false_type{});
        else row_steps(std::false_type{}, std::false_type{}, std::false_type{});
      } else {
        // fp32: pair sums round like every other fp32 operation (1e-3 gate)
        // (measured: C5 (G = 3) 2.757 -> 2.654 ms; C4 (G = 7) 0.628 -> 0.635 ms,
        // so the 16-tap form stays for G > 4)
        if (VK_FT_SYM32 && G <= VK_FT_SYM32_MAXG) row_steps(std::false_type{}, std::true_type{}, std::false_type{});
        else row_steps(std::false_type{}, std::false_type{}, std::false_type{});
      }
      // ---- border columns x in {0, W-2, W-1}: one thread per (row, column),
      // all G planes with the column's window kind, same mirror-pair form
      if (nbc > 0) {
        const int rows_in = ty1 - y0;
        // the (row, column) items fill at most three warps; which warps take
        // them rotates with the gap (the ring lets warps drift by two gaps),
        // so no warp is the CTA's slowest on every gap: with fixed warps a
        // border tile's CTA ran ~1.25 x longer than an interior tile's
        const int vt = (tid + FT_THREADS - 32 * ((3 * k) % FT_WARPS)) % FT_THREADS;
        for (int idx = vt; idx < rows_in * nbc; idx += FT_THREADS) {
          const int ic = idx % nbc, r = idx / nbc;
          const int gy = y0 + r, xb = bcol[ic];
          const int kind = a.kmap[NKIND1 + axis_kind(gy, H)] * a.nkx + a.kmap[axis_kind(xb, W)];
          const Acc* wk = wpart + (size_t)kind * 16 * NSTP;
          Acc aS[NPAIR > 0 ? NPAIR : 1], aD[NPAIR > 0 ? NPAIR : 1], aC = (Acc)0;
          for (int p = 0; p < NPAIR; ++p) { aS[p] = (Acc)0; aD[p] = (Acc)0; }
          const int cx = xb - x0 + 4;
#pragma unroll
          for (int oy = -1; oy <= 2; ++oy) {
#pragma unroll
            for (int ox = -1; ox <= 2; ++ox) {
              const int t = (oy + 1) * 4 + (ox + 1);
              const Acc x = AccVec<Acc>::cvt(bufA[(r + 1 + oy) * FT_SX + cx + ox]);
              const Acc y = AccVec<Acc>::cvt(bufB[(r + 1 + oy) * FT_SX + cx + ox]);
              const Acc Sv = x + y, Dv = x - y;
#pragma unroll
              for (int p = 0; p < NPAIR; ++p) {
                aS[p] = fma(wk[t * NSTP + L::plus(p)], Sv, aS[p]);
                aD[p] = fma(wk[t * NSTP + L::minus(p)], Dv, aD[p]);
              }
              if (MID) aC = fma(wk[t * NSTP + L::mid()], Sv, aC);
            }
          }
          const int64_t pix = (int64_t)gy * W + xb;
#pragma unroll
          for (int j = 0; j < G; ++j) {
            Acc t;
            if (MID && j == NPAIR) t = aC;
            else if (j < NPAIR) t = aS[j] + aD[j];
            else t = aS[G - 1 - j] - aD[G - 1 - j];
            a.out[(zk + 1 + j) * P + pix] = fminf(fmaxf((float)t, lo), hi);
            if (VAR)
              a.var[(zk + 1 + j) * P + pix] =
                  a.svar[((int64_t)s * a.NP + a.gap_pattern[k * G + j]) * a.NK + kind];
          }
        }
      }
      // ---- release plane k (and the unit's last plane with its last gap);
      // the last warp out refills the slot
      __syncwarp();
      if (lane == 0) {
        for (uint32_t q = sq_a; q <= (k == ke - 1 ? sq_b : sq_a); ++q) {
          const int slot = q % FT_STAGES;
          __threadfence_block();
          const int c = atomicAdd(&released[slot], 1);
          if (c == FT_WARPS - 1) {
            __threadfence_block();
            released[slot] = 0;
            const int j = (int)(q + FT_STAGES - seq0);     // plane of load q + FT_STAGES
            if (j < n_planes) {
              issue(q + FT_STAGES, x0 - 4, y0 - 1, kb + j);
              if (VK_FT_L2PF > 0 && j + VK_FT_L2PF < n_planes) tma_prefetch_3d(&tmap, x0 - 4, y0 - 1, kb + j + VK_FT_L2PF);
            } else if (s_unit[(uc + 1) & 1][3] && j - n_planes <= s_unit[(uc + 1) & 1][2] - s_unit[(uc + 1) & 1][1]) {
              const int t2 = s_unit[(uc + 1) & 1][0];
              issue(q + FT_STAGES, (t2 % n_tiles_x) * FT_TX - 4, (t2 / n_tiles_x) * FT_TY - 1,
                    s_unit[(uc + 1) & 1][1] + j - n_planes);
            }
          }
        }
      }
    }
    n_prev = min(n_planes, FT_STAGES);
    tile = s_unit[(uc + 1) & 1][0];
    kb = s_unit[(uc + 1) & 1][1];
    ke = s_unit[(uc + 1) & 1][2];
    have = s_unit[(uc + 1) & 1][3] != 0;
  }
  // the last CTA out rewinds the unit counter for the next launch
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(a.work + 1, 1) == (int)gridDim.x - 1) {
      a.work[0] = 0;
      a.work[1] = 0;
      __threadfence();
    }
  }
#ifdef VK_FT_DIAG
  __syncthreads();
  if (tid == 0 && blockIdx.x < 1024) {
    unsigned long long t1;
    unsigned smid;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_cta_diag[4 * blockIdx.x + 0] = smid;
    g_cta_diag[4 * blockIdx.x + 1] = 0;
    g_cta_diag[4 * blockIdx.x + 2] = diag_t0;
    g_cta_diag[4 * blockIdx.x + 3] = t1;
  }
#endif
}

}  // namespace

#ifdef VK_FT_DIAG
extern "C" int vk_debug_cta_times(unsigned long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, g_cta_diag, sizeof(unsigned long long) * 4 * (n < 1024 ? n : 1024));
}
#endif

cudaError_t launch_copy_known(const PredictArgs& a, cudaStream_t st) {
  const int64_t per = (a.P & 3) == 0 ? a.P / 4 : a.P;
  dim3 grid((unsigned)std::min<int64_t>(1024, (per + 255) / 256), a.K);
  copy_known_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_predict_generic(const PredictArgs& a, cudaStream_t st) {
  if (a.n_miss == 0) return cudaSuccess;
  dim3 grid((unsigned)((a.P + 255) / 256), a.n_miss);
  if (a.accum == 1) predict_generic_kernel<float><<<grid, 256, 0, st>>>(a);
  else predict_generic_kernel<double><<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// ---- TMA descriptor (driver entry point, no -lcuda needed) ----------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

int predict_fast_supported(int G, int accum) {
  (void)accum;
  return G >= 1 && G <= 8;
}

static size_t fast_smem(int G, bool f32) { return (size_t)ft_stages(G, f32) * FT_BUF_FLOATS * sizeof(float); }

template <int G, typename Acc>
static cudaError_t occupancy_t(int* occ) {
  const size_t smem = fast_smem(G, std::is_same<Acc, float>::value);
  cudaError_t e = cudaFuncSetAttribute(predict_fast_kernel<G, Acc, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(predict_fast_kernel<G, Acc, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, predict_fast_kernel<G, Acc, false>, FT_THREADS, smem);
  *occ = std::max(1, *occ);
  return e;
}

cudaError_t fast_stencil_table(int G, const PredictArgs& a, cudaStream_t st) {
  const int n_st = (a.part1 - a.part0) * a.NK * 16;
  if (n_st <= 0) return cudaSuccess;
  const int blocks = (n_st + 255) / 256;
  switch (G) {
#define VK_CASE(g) \
  case g: fast_stencil_kernel<g, double><<<blocks, 256, 0, st>>>(a); break;
    VK_CASE(1) VK_CASE(2) VK_CASE(3) VK_CASE(4) VK_CASE(5) VK_CASE(6) VK_CASE(7) VK_CASE(8)
#undef VK_CASE
    default: return cudaErrorNotSupported;
  }
  return cudaGetLastError();
}

// Guided schedule of a launch over n_gaps gaps of every tile.  `fixed` (the
// per-part chains: units of half a part's gaps) gives one level; otherwise the
// unit length starts at `cap` (<= FT_WPARTS parts, <= FT_MAXU gaps, and no more
// than a resident CTA's equal share) and halves level by level down to single
// gaps; the levels after the first take 15 / 9 / 6 / 4 % of a tile's gaps
// (VK_FT_GUIDE="15,9,6,4" overrides; development only).  The single-gap tail
// is what levels the CTAs' end times: C4 with 15/7/3/1-gap units 0.622 ms,
// with 22/11/5/2-gap units (no single gaps) 0.647 ms.
static FtSched make_sched(int n_gaps, int n_tiles, int cap, bool fixed) {
  FtSched sc{};
  static const char* env = std::getenv("VK_FT_GUIDE");
  int pct[4] = {15, 9, 6, 4};
  if (env) std::sscanf(env, "%d,%d,%d,%d", &pct[0], &pct[1], &pct[2], &pct[3]);
  int len[FT_NLV] = {cap}, gaps[FT_NLV] = {n_gaps}, nl = 1;
  if (!fixed) {
    int tail = 0;
    for (int l = 1; l <= 4 && (cap >> l) >= 1; ++l) {
      const int ln = cap >> l;
      len[nl] = ln;
      gaps[nl] = (pct[l - 1] * n_gaps + 50 * ln) / (100 * ln) * ln;
      tail += gaps[nl++];
      if (ln == 1) break;
    }
    if (tail > n_gaps / 2) nl = 1;         // a handful of gaps: one level
    else gaps[0] = n_gaps - tail;
  }
  int off = 0, base = 0, k = 0;
  for (int l = 0; l < nl; ++l) {
    if (gaps[l] <= 0) continue;
    sc.len[k] = len[l];
    sc.off[k] = off;
    sc.base[k] = base;
    off += gaps[l];
    base += (gaps[l] + len[l] - 1) / len[l] * n_tiles;
    ++k;
  }
  sc.n_lv = k;
  sc.off[k] = n_gaps;
  sc.base[k] = base;
  return sc;
}

// mirror-pair stencil table (and, fp64, the exact-split table) of parts
// [a.part0, a.part1) from the solved weights
template <int G, typename Acc>
static cudaError_t launch_tables_t(const PredictArgs& a, cudaStream_t st) {
  const int n_st = (a.part1 - a.part0) * a.NK * 16;
  if (n_st > 0) fast_stencil_kernel<G, Acc><<<(n_st + 255) / 256, 256, 0, st>>>(a);
  if (std::is_same<Acc, double>::value && VK_FT_SPLIT && a.part1 > a.part0) {
    const int n_sp = (a.part1 - a.part0) * (G / 2 + (G & 1));
    split_stencil_kernel<G><<<(n_sp + 127) / 128, 128, 0, st>>>(a);
  }
  return cudaGetLastError();
}

template <int G, typename Acc>
static cudaError_t launch_fast_t(const FastLaunch& fl, const PredictArgs& a, cudaStream_t st) {
  const size_t smem = fast_smem(G, std::is_same<Acc, float>::value);
  const int ntx = (a.W + FT_TX - 1) / FT_TX, nty = (a.H + FT_TY - 1) / FT_TY;
  const int n_tiles = ntx * nty, n_gaps = a.gap1 - a.gap0;
  if (n_gaps <= 0) return cudaSuccess;
  if (!a.work) return cudaErrorInvalidValue;
  const int resident = a.num_sms * fl.occ;
  // unit length: <= max_chunk keeps a unit within FT_WPARTS parts and FT_MAXU
  // bounds the staged per-gap metadata.  An explicit a.chunk (per-part chains:
  // half a part's gaps, so CTAs retire often) is taken as is; otherwise the
  // first level's units are at most a resident CTA's equal share, at least 4
  // gaps (the extra plane per run).
  const int64_t n_items = (int64_t)n_tiles * n_gaps;
  int hard = std::min(n_gaps, FT_MAXU);                    // what the staged tables hold
  if (a.max_chunk > 0) {
    // max_chunk = 2 * (shortest part run) + 1 bounds a unit to three parts;
    // four parts fit the staged (part, row kind) slots when H > FT_TY
    const int min_len = (a.max_chunk - 1) / 2, parts = a.H > FT_TY ? FT_WPARTS : FT_WPARTS - 1;
    hard = std::min(hard, (parts - 1) * min_len + 1);
  }
  const bool fixed = a.chunk > 0;
  int cap = hard;
  if (fixed) cap = std::min(cap, a.chunk);
  else cap = (int)std::min<int64_t>(hard, std::max<int64_t>(std::min(4, n_gaps), n_items / std::max(1, resident)));
  // Longer units are not better: warps drift apart inside a unit until the
  // ring stops the leaders, and the unit-start barrier realigns them.  C4
  // (G = 7): 6 / 10 / 15 / 22 gaps 0.626 / 0.620 / 0.629 / 0.650 ms; C5 (G = 3):
  // 8 / 16 / 24 / 32 gaps 3.370 / 3.334 / 3.325 / 3.325 ms (a unit's extra
  // plane weighs more at small G) -> about 70 interpolated planes per unit.
  static const int env_cap = std::getenv("VK_FT_CAP") ? std::atoi(std::getenv("VK_FT_CAP")) : 0;   // development
  if (!fixed) cap = std::min(cap, env_cap > 0 ? env_cap : std::max(4, 70 / G));
  const FtSched sc = make_sched(n_gaps, n_tiles, cap, fixed);
  const int grid = std::max(1, std::min(resident, sc.base[sc.n_lv]));
  if (!a.tables_done) {
    cudaError_t e = launch_tables_t<G, Acc>(a, st);
    if (e != cudaSuccess) return e;
  }
  const CUtensorMap& map = *reinterpret_cast<const CUtensorMap*>(fl.tmap);
  if (a.var)
    predict_fast_kernel<G, Acc, true><<<grid, FT_THREADS, smem, st>>>(map, a, ntx, n_tiles, sc);
  else
    predict_fast_kernel<G, Acc, false><<<grid, FT_THREADS, smem, st>>>(map, a, ntx, n_tiles, sc);
  return cudaGetLastError();
}

cudaError_t prepare_predict_fast(const PredictArgs& a, FastLaunch* fl) {
  if (fl->known == a.known && fl->G == a.G && fl->accum == a.accum) return cudaSuccess;
  EncodeTiledFn enc = get_encode();
  if (!enc) return cudaErrorNotSupported;
  const cuuint64_t dims[3] = {(cuuint64_t)a.W, (cuuint64_t)a.H, (cuuint64_t)a.K};
  const cuuint64_t strides[2] = {(cuuint64_t)a.W * 4, (cuuint64_t)a.P * 4};
  const cuuint32_t box[3] = {FT_SX, FT_SY, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(reinterpret_cast<CUtensorMap*>(fl->tmap), CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                   (void*)a.known, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return cudaErrorInvalidValue;
  cudaError_t e = cudaErrorNotSupported;
  const bool f32 = a.accum == 1;
  if (a.accum == 2) e = occupancy_fixed(a.G, &fl->occ);
  else switch (a.G) {
#define VK_CASE(g) \
  case g: e = f32 ? occupancy_t<g, float>(&fl->occ) : occupancy_t<g, double>(&fl->occ); break;
    VK_CASE(1) VK_CASE(2) VK_CASE(3) VK_CASE(4) VK_CASE(5) VK_CASE(6) VK_CASE(7) VK_CASE(8)
#undef VK_CASE
    default: break;
  }
  if (e != cudaSuccess) return e;
  fl->known = a.known;
  fl->G = a.G;
  fl->accum = a.accum;
  return cudaSuccess;
}

cudaError_t launch_predict_fast_prepared(const FastLaunch& fl, const PredictArgs& a, cudaStream_t st) {
  if (a.accum == 2) return launch_predict_fixed(fl.tmap, fl.occ, a, st);
  const bool f32 = a.accum == 1;
  switch (a.G) {
#define VK_CASE(g) \
  case g: return f32 ? launch_fast_t<g, float>(fl, a, st) : launch_fast_t<g, double>(fl, a, st);
    VK_CASE(1) VK_CASE(2) VK_CASE(3) VK_CASE(4) VK_CASE(5) VK_CASE(6) VK_CASE(7) VK_CASE(8)
#undef VK_CASE
    default:
      return cudaErrorNotSupported;
  }
}

cudaError_t launch_predict_fast_tables(const PredictArgs& a, cudaStream_t st) {
  if (a.accum == 2) return cudaErrorNotSupported;          // the fixed path builds its own tables
  const bool f32 = a.accum == 1;
  switch (a.G) {
#define VK_CASE(g) \
  case g: return f32 ? launch_tables_t<g, float>(a, st) : launch_tables_t<g, double>(a, st);
    VK_CASE(1) VK_CASE(2) VK_CASE(3) VK_CASE(4) VK_CASE(5) VK_CASE(6) VK_CASE(7) VK_CASE(8)
#undef VK_CASE
    default:
      return cudaErrorNotSupported;
  }
}

cudaError_t launch_predict_fast(const PredictArgs& a, cudaStream_t st) {
  FastLaunch fl;
  cudaError_t e = prepare_predict_fast(a, &fl);
  if (e != cudaSuccess) return e;
  return launch_predict_fast_prepared(fl, a, st);
}

}  // namespace vk
