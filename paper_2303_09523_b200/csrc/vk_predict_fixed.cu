// Fixed-point streaming prediction on the integer tensor cores
// (accum = VK_ACCUM_FIXED).  Same work as predict_fast (kriging.py:523-557 on
// the plane-structured layout: every missing plane of a gap reads the 4x4
// windows of its two bracketing known planes), arranged as one small integer
// GEMM per tile row:
//
//   out[x, j] = c0_j + step * 2^-P * sum_k q[x, k] * W[k, j]
//
//   x : 16 consecutive voxels of a row          (MMA M = 16)
//   k : 32 taps = 2 planes x 4 columns x 4 rows (MMA K = 32)
//   j : the G <= 8 missing planes of the gap    (MMA N = 8)
//
// q   = known values quantised to 24-bit fixed point over the volume's range,
//       v = L + q * step + e, |e| <= step (step = range / (2^24 - 1));
// W   = round(w * 2^P), the kriging weights in 32-bit fixed point (P = 30 when
//       max|w| < 2, one bit less per doubling);
// c0_j = L * sum_k w_jk in fp64 (kept as a float pair).
//
// q and W are split into unsigned bytes (the top weight byte signed):
// q = q0 + 2^8 q1 + 2^16 q2, W = W0 + 2^8 W1 + 2^16 W2 + 2^24 W3.  The nine
// byte products with a + b >= 2 run as mma.sync m16n8k32 (u8 x u8 / u8 x s8,
// s32 accumulate -- exact) into four accumulators grouped by a + b; the three
// dropped products are bounded by 32*255*255*513 * 2^-P * step ~ step.  The
// accumulators are recombined in fp32 (exact integers up to 2^24 scale).
// Error against the exact fp64 sum: <= sum|w| * step (quantisation)
// + 32 * 2^-P-1 * range (weights) + ~2 step (dropped products, fp32 recombine)
// ~ 2e-7 of the range -- inside the 1e-6 fp64 gate.
//
// Data layout in shared memory: known-plane f32 tiles arrive by TMA (the same
// 136 x 35 box as predict_fast), are quantised once per unit into three byte
// images stored column-major (x-major, 4 rows per 32-bit word) so that the
// A-fragment register for (voxel x, tap column ox) is the 4 bytes of rows
// y-1..y+2 of column x+ox: a byte_perm of two words, which slide down the
// column as the warp walks the tile rows.  B fragments (weights) stay in
// registers for a whole gap.  Border columns x in {0, W-2, W-1} (a different
// window kind per voxel of the MMA row) are computed per voxel in fp64 from
// the mirror-pair stencil table.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cfloat>
#include <cstdint>
#include "vk_kernels.h"
#include "vk_tma.cuh"

namespace vk {

namespace {

constexpr int FX_WARPS = 8;
constexpr int FX_THREADS = FX_WARPS * 32;
constexpr int FX_TY = 32;                        // tile rows
constexpr int FX_SY = FX_TY + 3;                 // staged rows y0-1 .. y0+33
constexpr int FX_BUF_FLOATS = ((FT_SX * FX_SY * 4 + 127) / 128) * 128 / 4;
constexpr int FX_STAGES = 3;                     // f32 TMA ring
constexpr int FX_CW = 9;                         // words per byte-image column (36 rows)
constexpr int FX_IMG_WORDS = FT_SX * FX_CW;      // one byte image
constexpr int FX_PLANE_WORDS = 3 * FX_IMG_WORDS; // three byte images of a plane
constexpr int FX_SLOTS = 3;                      // quantised-plane ring
constexpr float FX_QMAX = 16777215.0f;           // 2^24 - 1

__device__ __forceinline__ void mma_u8u8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_u8s8(int (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// volume-wide quantisation range from the per-part known ranges
}  // namespace

// ---- tables: one warp per (part, kind) -----------------------------------
// fxb [s][kind][lane][8] u32 : B fragments, reg 2*b + r = weight byte b,
//                              k-half r (plane A / plane B)
// fxc [s][kind][8] float4    : (c0 hi, c0 lo, cG, cH) per missing plane j
// fxq float4                 : (L, 1/step, step, 0), then double2 (L, step)
template <int G>
__global__ void __launch_bounds__(32) fixed_table_kernel(PredictArgs a) {
  const int s = a.part0 + blockIdx.x / a.NK, kind = blockIdx.x % a.NK;
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  const double2 Ls = reinterpret_cast<const double2*>(a.fxq)[1];
  const double L = Ls.x, step = Ls.y;
  // weights of missing plane g (patterns are identical for every gap here)
  const double* w = nullptr;
  if (g < G) w = a.weights + (((int64_t)s * a.NP + a.gap_pattern[g]) * a.NK + kind) * WPAD;
  // fixed-point exponent from the largest weight of this (part, kind)
  double mx = 0.0;
  if (w)
    for (int i = t; i < 32; i += 4) mx = fmax(mx, fabs(w[i]));
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int P = 30;
  if (mx >= 2.0) P = 30 - ilogb(mx);
  uint32_t frag[8];
  for (int r = 0; r < 2; ++r) {              // k-half: plane A (r = 0), plane B (r = 1)
    int64_t Wq[4];
    for (int i = 0; i < 4; ++i)              // k = 16 r + 4 t + i <-> (ox = t - 1, oy = i - 1)
      Wq[i] = w ? llrint(ldexp(w[16 * r + 4 * i + t], P)) : 0;
    for (int b = 0; b < 4; ++b) {
      uint32_t word = 0;
      for (int i = 0; i < 4; ++i) word |= (uint32_t)((Wq[i] >> (8 * b)) & 0xff) << (8 * i);
      frag[2 * b + r] = word;
    }
  }
  uint4* dst = reinterpret_cast<uint4*>(a.fxb) + (((size_t)s * a.NK + kind) * 32 + lane) * 2;
  dst[0] = make_uint4(frag[0], frag[1], frag[2], frag[3]);
  dst[1] = make_uint4(frag[4], frag[5], frag[6], frag[7]);
  if (lane < 8) {
    double sw = 0.0;
    if (lane < G) {
      const double* wj = a.weights + (((int64_t)s * a.NP + a.gap_pattern[lane]) * a.NK + kind) * WPAD;
      for (int i = 0; i < 32; ++i) sw += wj[i];
    }
    const double c0 = L * sw;
    const float hi = (float)c0;
    reinterpret_cast<float4*>(a.fxc)[((size_t)s * a.NK + kind) * 8 + lane] =
        make_float4(hi, (float)(c0 - (double)hi), (float)ldexp(step, 32 - P), (float)ldexp(step, 16 - P));
  }
}

// The quantisation range is the volume's known range: the union of every
// part's clamp range (min/max of the non-empty statistics chunks, as the fit
// kernel reduces them per part), computed once from the statistics pass so a
// part's tables never depend on other parts' fits (chained schedule).
__global__ void __launch_bounds__(256) quant_range_kernel(const ChunkStat* __restrict__ stats, int n, void* fxq) {
  double mn = DBL_MAX, mx = -DBL_MAX;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const ChunkStat cs = stats[i];
    if (cs.n <= 0) continue;
    mn = fmin(mn, cs.mn);
    mx = fmax(mx, cs.mx);
  }
  for (int o = 16; o; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __shared__ double sh[2][8];
  if ((threadIdx.x & 31) == 0) {
    sh[0][threadIdx.x >> 5] = mn;
    sh[1][threadIdx.x >> 5] = mx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < 8; ++w) {
      mn = fmin(mn, sh[0][w]);
      mx = fmax(mx, sh[1][w]);
    }
    if (mn > mx) mn = mx = 0.0;                    // no finite known value: the fit reports it
    const double L = mn, R = mx - mn;
    const double step = R > 0 ? R / 16777215.0 : 0.0;
    reinterpret_cast<float4*>(fxq)[0] = make_float4((float)L, step > 0 ? (float)(1.0 / step) : 0.f, (float)step, 0.f);
    reinterpret_cast<double2*>(fxq)[1] = make_double2(L, step);
  }
}

template <int G, bool VAR>
__global__ void __launch_bounds__(FX_THREADS, 2)
    predict_fixed_kernel(const __grid_constant__ CUtensorMap tmap, PredictArgs a, int n_tiles_x, int n_tiles,
                         int chunk, int n_units) {
  constexpr int NPAIR = G / 2;
  constexpr bool MID = (G & 1) != 0;
  constexpr int NST = 2 * NPAIR + (MID ? 1 : 0);
  constexpr int NSTP = (NST + 1) & ~1;
  extern __shared__ __align__(128) float ring[];          // FX_STAGES f32 tiles, then byte images
  uint32_t* img = reinterpret_cast<uint32_t*>(ring + FX_STAGES * FX_BUF_FLOATS);
  __shared__ __align__(8) uint64_t full[FX_STAGES];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int H = a.H, W = a.W;
  const int64_t P = a.P;
  if (tid == 0) {
    for (int i = 0; i < FX_STAGES; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const float4 qp = *reinterpret_cast<const float4*>(a.fxq);
  const float qL = qp.x, qinv = qp.y;
  const double qstep = (double)qp.z;
  const uint32_t tile_bytes = FT_SX * FX_SY * 4;
  const int n_gaps = a.K - 1;
  const int kint = a.kmap[AXIS_INTERIOR];
  const double* kpm = reinterpret_cast<const double*>(a.kpm);
  uint32_t load_seq = 0;

  for (int u = blockIdx.x; u < n_units; u += gridDim.x) {
    const int chunk_id = u / n_tiles, tile = u - chunk_id * n_tiles;
    const int tx = tile % n_tiles_x, ty = tile / n_tiles_x;
    const int x0 = tx * FT_TX, y0 = ty * FX_TY;
    const int kb = a.gap0 + chunk_id * chunk, ke = min(a.gap1, kb + chunk);   // gaps [kb, ke)
    const int ty1 = min(H, y0 + FX_TY), tx1 = min(W, x0 + FT_TX);
    int nbc = 0, bcol[3] = {0, 0, 0};
    {
      const int cc[3] = {0, W - 2, W - 1};
      for (int q = 0; q < 3; ++q)
        if (cc[q] >= x0 && cc[q] < tx1) bcol[nbc++] = cc[q];
    }
    const uint32_t seq0 = load_seq;
    load_seq += ke - kb + 1;
    __syncthreads();                                       // previous unit done with the rings
    if (tid == 0) {
      fence_proxy_async();
      for (int i = 0; i < 2 && kb + i <= ke; ++i) {
        const uint32_t sq = seq0 + i;
        mbar_expect_tx(&full[sq % FX_STAGES], tile_bytes);
        tma_load_3d(ring + (sq % FX_STAGES) * FX_BUF_FLOATS, &tmap, &full[sq % FX_STAGES], x0 - 4, y0 - 1,
                    kb + i);
      }
    }
    for (int pk = kb; pk <= ke; ++pk) {
      const uint32_t sq = seq0 + (pk - kb);
      // ---- quantise known plane pk into its byte images; pass it through to
      // the output (kriging.py:481) if this unit owns it
      {
        mbar_wait(&full[sq % FX_STAGES], (sq / FX_STAGES) & 1);
        const float* fb = ring + (sq % FX_STAGES) * FX_BUF_FLOATS;
        uint32_t* im = img + (sq % FX_SLOTS) * FX_PLANE_WORDS;
        const bool copy = pk < ke || pk == n_gaps;
        const int64_t zk = a.known_z[pk];
        for (int i = tid; i < FX_IMG_WORDS; i += FX_THREADS) {
          const int yq = i / FT_SX, cx = i - yq * FT_SX;   // lanes walk columns
          uint32_t w0 = 0, w1 = 0, w2 = 0;
#pragma unroll
          for (int r = 0; r < 4; ++r) {
            const int row = 4 * yq + r;
            const float v = row < FX_SY ? fb[row * FT_SX + cx] : qL;
            const uint32_t q = __float2uint_rn(fminf(fmaxf((v - qL) * qinv, 0.f), FX_QMAX));
            w0 |= (q & 0xffu) << (8 * r);
            w1 |= ((q >> 8) & 0xffu) << (8 * r);
            w2 |= (q >> 16) << (8 * r);
            if (copy) {
              const int y = y0 + row - 1, x = x0 + cx - 4;
              if (row >= 1 && row <= FX_TY && cx >= 4 && cx < 4 + FT_TX && y < H && x < W) {
                st_cs_f32(a.out + zk * P + (int64_t)y * W + x, v);
                if (VAR) a.var[zk * P + (int64_t)y * W + x] = 0.0;
              }
            }
          }
          im[cx * FX_CW + yq] = w0;
          im[FX_IMG_WORDS + cx * FX_CW + yq] = w1;
          im[2 * FX_IMG_WORDS + cx * FX_CW + yq] = w2;
        }
      }
      __syncthreads();                                     // images of pk visible; f32 tile of pk consumed
      if (tid == 0 && pk + 2 <= ke) {
        const uint32_t sn = sq + 2;                        // slot of plane pk - 1: quantised last step
        fence_proxy_async();
        mbar_expect_tx(&full[sn % FX_STAGES], tile_bytes);
        tma_load_3d(ring + (sn % FX_STAGES) * FX_BUF_FLOATS, &tmap, &full[sn % FX_STAGES], x0 - 4, y0 - 1,
                    pk + 2);
      }
      if (pk == kb) continue;
      // ---- gap k = pk - 1 between known planes k (A) and pk (B)
      const int k = pk - 1;
      const uint32_t* imA = img + ((sq - 1) % FX_SLOTS) * FX_PLANE_WORDS;
      const uint32_t* imB = img + (sq % FX_SLOTS) * FX_PLANE_WORDS;
      const int s = a.gap_part[k];
      const float lo = (float)a.lohi[2 * s], hi = (float)a.lohi[2 * s + 1];
      const int64_t zk = a.known_z[k];
      const int xs = x0 + 16 * warp;                       // this warp's 16 columns
      if (xs < W) {
        const uint4* bsrc = reinterpret_cast<const uint4*>(a.fxb);
        const float4* csrc = reinterpret_cast<const float4*>(a.fxc);
        const int kin = a.kmap[NKIND1 + AXIS_INTERIOR] * a.nkx + kint;   // interior kind
        const int j0 = 2 * t, j1 = 2 * t + 1;              // C columns of this lane
        uint32_t bf[8];
        float chi0, chi1, clo0, clo1, cg, ch;              // constants of planes 2t, 2t+1
        double vj0 = 0.0, vj1 = 0.0;
        auto load_kind = [&](int kind) {
          const size_t sk = (size_t)s * a.NK + kind;
          const uint4 b01 = bsrc[(sk * 32 + lane) * 2];
          const uint4 b23 = bsrc[(sk * 32 + lane) * 2 + 1];
          bf[0] = b01.x; bf[1] = b01.y; bf[2] = b01.z; bf[3] = b01.w;
          bf[4] = b23.x; bf[5] = b23.y; bf[6] = b23.z; bf[7] = b23.w;
          const float4 e0 = csrc[sk * 8 + j0], e1 = csrc[sk * 8 + j1];
          chi0 = e0.x; chi1 = e1.x;
          clo0 = e0.y; clo1 = e1.y;
          cg = e0.z;
          ch = e0.w;
          if (VAR) {
            if (j0 < G) vj0 = a.svar[((int64_t)s * a.NP + a.gap_pattern[k * G + j0]) * a.NK + kind];
            if (j1 < G) vj1 = a.svar[((int64_t)s * a.NP + a.gap_pattern[k * G + j1]) * a.NK + kind];
          }
        };
        load_kind(kin);
        int kcur = kin;
        // rows that need attention: border rows (own window kind), the row
        // after the top border row (back to interior), rows past the volume
        uint32_t special = 0;
        for (int r = 0; r < FX_TY; ++r) {
          const int y = y0 + r;
          if (y >= H || y == 0 || y == 1 || y >= H - 2) special |= 1u << r;
        }
        // byte-image columns of this lane's A registers: (x, plane A), (x+8, A),
        // (x, B), (x+8, B) with x = xs + g and tap column ox = t - 1
        const int cx = xs - x0 + g + t + 3;
        const uint32_t* col[4] = {imA + cx * FX_CW, imA + (cx + 8) * FX_CW, imB + cx * FX_CW,
                                  imB + (cx + 8) * FX_CW};
        const int xv0 = xs + g, xv1 = xs + g + 8;          // voxels of C rows g, g + 8
        const bool okx0 = xv0 >= 1 && xv0 <= W - 3, okx1 = xv1 >= 1 && xv1 <= W - 3;
        const bool m0 = j0 < G && okx0, m1 = j1 < G && okx0, m2 = j0 < G && okx1, m3 = j1 < G && okx1;
        // output pointers of (plane 2t, voxel xv0) and (plane 2t+1, voxel xv0);
        // voxel xv1 = xv0 + 8 is an immediate offset
        float* p0 = a.out + (zk + 1 + j0) * P + (int64_t)y0 * W + xv0;
        float* p1 = p0 + P;
        double* q0 = VAR ? a.var + (zk + 1 + j0) * P + (int64_t)y0 * W + xv0 : nullptr;
        double* q1 = VAR ? q0 + P : nullptr;
        bool done = false;
        // one row: A fragments from the sliding byte words, 9 MMAs, epilogue
        auto row = [&](const uint32_t (&wl)[3][4], const uint32_t (&wh)[3][4], const int r, const int sh) {
          if (special & (1u << r)) {                       // warp-uniform
            const int y = y0 + r;
            if (y >= H) { done = true; return; }
            const int kind_y = a.kmap[NKIND1 + axis_kind(y, H)] * a.nkx + kint;
            if (kind_y != kcur) {
              kcur = kind_y;
              load_kind(kcur);
            }
          }
          uint32_t A[3][4];
#pragma unroll
          for (int sl = 0; sl < 3; ++sl)
#pragma unroll
            for (int m = 0; m < 4; ++m)
              A[sl][m] = sh == 0 ? wl[sl][m] : __byte_perm(wl[sl][m], wh[sl][m], 0x3210 + 0x1111 * sh);
          int acc[4][4];
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int c = 0; c < 4; ++c) acc[q][c] = 0;
          // group a + b = 2 .. 5 -> acc[a + b - 2]
          mma_u8u8(acc[0], A[0], bf[4], bf[5]);            // (0, 2)
          mma_u8u8(acc[0], A[1], bf[2], bf[3]);            // (1, 1)
          mma_u8u8(acc[0], A[2], bf[0], bf[1]);            // (2, 0)
          mma_u8s8(acc[1], A[0], bf[6], bf[7]);            // (0, 3)
          mma_u8u8(acc[1], A[1], bf[4], bf[5]);            // (1, 2)
          mma_u8u8(acc[1], A[2], bf[2], bf[3]);            // (2, 1)
          mma_u8s8(acc[2], A[1], bf[6], bf[7]);            // (1, 3)
          mma_u8u8(acc[2], A[2], bf[4], bf[5]);            // (2, 2)
          mma_u8s8(acc[3], A[2], bf[6], bf[7]);            // (2, 3)
          // C fragment: (c0, c1) -> voxel xv0, planes (2t, 2t+1); (c2, c3) -> xv1.
          // T = 2^32 (256 P5 + P4) + 2^16 (256 P3 + P2); out = c0 + step 2^-P T
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int ga = acc[3][2 * h] * 256 + acc[2][2 * h], gb = acc[3][2 * h + 1] * 256 + acc[2][2 * h + 1];
            const int ha = acc[1][2 * h] * 256 + acc[0][2 * h], hb = acc[1][2 * h + 1] * 256 + acc[0][2 * h + 1];
            const float vx = fminf(fmaxf(fmaf((float)ga, cg, fmaf((float)ha, ch, clo0)) + chi0, lo), hi);
            const float vy = fminf(fmaxf(fmaf((float)gb, cg, fmaf((float)hb, ch, clo1)) + chi1, lo), hi);
            const bool ma = h ? m2 : m0, mb = h ? m3 : m1;
            if (ma) st_cs_f32(p0 + 8 * h, vx);
            if (mb) st_cs_f32(p1 + 8 * h, vy);
            if (VAR) {
              if (ma) q0[8 * h] = vj0;
              if (mb) q1[8 * h] = vj1;
            }
          }
          p0 += W;
          p1 += W;
          if (VAR) { q0 += W; q1 += W; }
        };
        // words (rows 4i .. 4i+3) of the four columns in the three byte images;
        // ping-pong between wa and wb so no register copies are needed
        uint32_t wa[3][4], wb[3][4];
#pragma unroll
        for (int sl = 0; sl < 3; ++sl)
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            wa[sl][m] = col[m][sl * FX_IMG_WORDS];
            wb[sl][m] = col[m][sl * FX_IMG_WORDS + 1];
          }
#pragma unroll 1
        for (int r8 = 0; r8 < FX_TY / 8 && !done; ++r8) {
#pragma unroll
          for (int sh = 0; sh < 4 && !done; ++sh) row(wa, wb, 8 * r8 + sh, sh);
#pragma unroll
          for (int sl = 0; sl < 3; ++sl)
#pragma unroll
            for (int m = 0; m < 4; ++m) wa[sl][m] = col[m][sl * FX_IMG_WORDS + 2 * r8 + 2];
#pragma unroll
          for (int sh = 0; sh < 4 && !done; ++sh) row(wb, wa, 8 * r8 + 4 + sh, sh);
          if (r8 + 1 < FX_TY / 8) {
#pragma unroll
            for (int sl = 0; sl < 3; ++sl)
#pragma unroll
              for (int m = 0; m < 4; ++m) wb[sl][m] = col[m][sl * FX_IMG_WORDS + 2 * r8 + 3];
          }
        }
      }
      // ---- border columns: per voxel, fp64, mirror-pair stencils of the
      // column's kind, values dequantised from the byte images
      if (nbc > 0) {
        const int rows_in = ty1 - y0;
        for (int idx = tid; idx < rows_in * nbc; idx += FX_THREADS) {
          const int ic = idx % nbc, r = idx / nbc;
          const int gy = y0 + r, xb = bcol[ic];
          const int kind = a.kmap[NKIND1 + axis_kind(gy, H)] * a.nkx + a.kmap[axis_kind(xb, W)];
          const double* wk = kpm + ((size_t)s * a.NK + kind) * 16 * NSTP;
          double aS[NPAIR > 0 ? NPAIR : 1], aD[NPAIR > 0 ? NPAIR : 1], aC = 0.0;
          for (int p = 0; p < NPAIR; ++p) { aS[p] = 0.0; aD[p] = 0.0; }
          const int cxb = xb - x0 + 4;
          for (int oy = -1; oy <= 2; ++oy) {
            const int row = r + 1 + oy;
            for (int ox = -1; ox <= 2; ++ox) {
              const int tap = (oy + 1) * 4 + (ox + 1);
              const int wi = (cxb + ox) * FX_CW + (row >> 2), sh = 8 * (row & 3);
              const uint32_t qa = ((imA[wi] >> sh) & 0xffu) | (((imA[FX_IMG_WORDS + wi] >> sh) & 0xffu) << 8) |
                                  (((imA[2 * FX_IMG_WORDS + wi] >> sh) & 0xffu) << 16);
              const uint32_t qb = ((imB[wi] >> sh) & 0xffu) | (((imB[FX_IMG_WORDS + wi] >> sh) & 0xffu) << 8) |
                                  (((imB[2 * FX_IMG_WORDS + wi] >> sh) & 0xffu) << 16);
              // sum of the two planes' values minus 2L, difference exact in fp64
              const double Sv = (double)(qa + qb) * qstep, Dv = ((double)qa - (double)qb) * qstep;
              for (int p = 0; p < NPAIR; ++p) {
                aS[p] = fma(wk[tap * NSTP + 2 * p], Sv, aS[p]);
                aD[p] = fma(wk[tap * NSTP + 2 * p + 1], Dv, aD[p]);
              }
              if (MID) aC = fma(wk[tap * NSTP + 2 * NPAIR], Sv, aC);
            }
          }
          const int64_t pix = (int64_t)gy * W + xb;
          const float4* csrc = reinterpret_cast<const float4*>(a.fxc);
          for (int j = 0; j < G; ++j) {
            double v;
            if (MID && j == NPAIR) v = aC;
            else if (j < NPAIR) v = aS[j] + aD[j];
            else v = aS[G - 1 - j] - aD[G - 1 - j];
            const float4 cc = csrc[((size_t)s * a.NK + kind) * 8 + j];
            v += (double)cc.x + (double)cc.y;              // + L * sum(w)
            a.out[(zk + 1 + j) * P + pix] = fminf(fmaxf((float)v, lo), hi);
            if (VAR) a.var[(zk + 1 + j) * P + pix] = a.svar[((int64_t)s * a.NP + a.gap_pattern[k * G + j]) * a.NK + kind];
          }
        }
      }
    }
  }
}

static size_t fixed_smem() {
  return (size_t)FX_STAGES * FX_BUF_FLOATS * sizeof(float) + (size_t)FX_SLOTS * FX_PLANE_WORDS * 4;
}

template <int G>
static cudaError_t occupancy_fixed_t(int* occ) {
  const size_t smem = fixed_smem();
  cudaError_t e = cudaFuncSetAttribute(predict_fixed_kernel<G, true>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(predict_fixed_kernel<G, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, predict_fixed_kernel<G, false>, FX_THREADS, smem);
  *occ = *occ < 1 ? 1 : *occ;
  return e;
}

template <int G>
static cudaError_t launch_fixed_t(const void* tmap, int occ, const PredictArgs& a, cudaStream_t st) {
  const int ntx = (a.W + FT_TX - 1) / FT_TX, nty = (a.H + FX_TY - 1) / FX_TY;
  const int n_tiles = ntx * nty, n_gaps = a.gap1 - a.gap0;
  if (n_gaps <= 0) return cudaSuccess;
  const int n_tab = (a.part1 - a.part0) * a.NK;
  if (n_tab > 0) {
    fast_stencil_table(G, a, st);                          // fp64 mirror pairs for the border columns
    fixed_table_kernel<G><<<n_tab, 32, 0, st>>>(a);
  }
  const int resident = a.num_sms * occ;
  int chunk = (int)((int64_t)n_tiles * n_gaps / ((int64_t)resident * 6));
  chunk = chunk < 1 ? 1 : chunk;
  const int lo4 = n_gaps < 4 ? n_gaps : 4;
  chunk = chunk < lo4 ? lo4 : chunk;
  chunk = chunk > n_gaps ? n_gaps : chunk;
  if (a.chunk > 0) chunk = a.chunk < n_gaps ? a.chunk : n_gaps;
  const int n_chunks = (n_gaps + chunk - 1) / chunk;
  const int n_units = n_tiles * n_chunks;
  const int grid = n_units < resident ? n_units : resident;
  const CUtensorMap& map = *reinterpret_cast<const CUtensorMap*>(tmap);
  if (a.var)
    predict_fixed_kernel<G, true><<<grid, FX_THREADS, fixed_smem(), st>>>(map, a, ntx, n_tiles, chunk, n_units);
  else
    predict_fixed_kernel<G, false><<<grid, FX_THREADS, fixed_smem(), st>>>(map, a, ntx, n_tiles, chunk, n_units);
  return cudaGetLastError();
}

cudaError_t occupancy_fixed(int G, int* occ) {
  switch (G) {
#define VK_CASE(g) \
  case g: return occupancy_fixed_t<g>(occ);
    VK_CASE(1) VK_CASE(2) VK_CASE(3) VK_CASE(4) VK_CASE(5) VK_CASE(6) VK_CASE(7) VK_CASE(8)
#undef VK_CASE
    default: return cudaErrorNotSupported;
  }
}

cudaError_t launch_quant_range(const ChunkStat* stats, int n, void* fxq, cudaStream_t st) {
  quant_range_kernel<<<1, 256, 0, st>>>(stats, n, fxq);
  return cudaGetLastError();
}

cudaError_t launch_predict_fixed(const void* tmap, int occ, const PredictArgs& a, cudaStream_t st) {
  switch (a.G) {
#define VK_CASE(g) \
  case g: return launch_fixed_t<g>(tmap, occ, a, st);
    VK_CASE(1) VK_CASE(2) VK_CASE(3) VK_CASE(4) VK_CASE(5) VK_CASE(6) VK_CASE(7) VK_CASE(8)
#undef VK_CASE
    default: return cudaErrorNotSupported;
  }
}

}  // namespace vk
