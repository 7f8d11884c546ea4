// Empirical semivariogram + bounded fit per Z sub-part (fit_variogram,
// kriging.py:264-328), and the per-part clamp range (kriging.py:475-479).
//
//   plane_stats  : one pass over the known planes -> per-chunk count / mean /
//                  M2 / min / max (deterministic block trees; merged per part
//                  in a fixed order with Chan's update) -> svar, lo, hi.
//   pair_table   : numpy-identical pair draw (PCG64 + Lemire, see pcg64.h)
//                  with LCG jump-ahead and a grid-wide stream compaction
//                  (count / scan / scatter), then lags, hmax, bin index per
//                  pair and bin counts.  Lags
//                  and bins depend only on geometry, so one table serves every
//                  part with the same sample layout.
//   bins         : per part, sum of 0.5*(v_i - v_j)^2 per bin; per-thread
//                  shared-memory accumulators reduced in a fixed order.
//   fit          : per part, the TRF fit on the non-empty bins: one warp per
//                  part, residual rows on lanes (trf_warp.cuh, trf.h); svar
//                  and the bin sums come numpy-exact from vk_npstats.cu.
#include <cuda_runtime.h>
#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include "pcg64.h"
#include "trf.h"
#include "trf_warp.cuh"
#include "vk_kernels.h"
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

namespace vk {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// statistics of chunk c of plane k (one CTA)
template <typename T>
__device__ __forceinline__ void stats_chunk(const T* __restrict__ data, int64_t P, int nchunk, int k, int c,
                                            ChunkStat* __restrict__ out, int* __restrict__ inexact) {
  const int64_t beg = (int64_t)c * STATS_CHUNK;
  const int64_t end = min(P, beg + (int64_t)STATS_CHUNK);
  const T* p = data + (int64_t)k * P;
  const double shift = (beg < end) ? (double)p[beg] : 0.0;
  double s1 = 0.0, s2 = 0.0, mn = DBL_MAX, mx = -DBL_MAX, bad = 0.0;
  auto take = [&](double v) {
    if (!(v - v == 0.0)) { bad += 1.0; return; }
    const double d = v - shift;
    s1 += d;
    s2 = fma(d, d, s2);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  };
  bool notint = false;
  const bool vec = sizeof(T) == 4 && ((P & 3) == 0) && ((end - beg) & 3) == 0;
  if (vec) {
    // 128-bit loads, 4 in flight per thread.  Fast form: no per-element
    // finiteness test (a non-finite value poisons s1 / s2 and the thread
    // redoes its elements with `take` below), min / max and the integer test
    // in fp32 (exact on f32 data); the fp64 shifted sums are unchanged, so
    // the chunk statistics are bit-identical to the careful form.
    const float4* q = reinterpret_cast<const float4*>(p + beg);
    const int64_t n4 = (end - beg) >> 2;
    float fmn = FLT_MAX, fmx = -FLT_MAX;
    auto fast = [&](float x) {
      const double d = (double)x - shift;
      s1 += d;
      s2 = fma(d, d, s2);
      fmn = fminf(fmn, x);
      fmx = fmaxf(fmx, x);
      notint |= x != rintf(x);
    };
    for (int64_t i = threadIdx.x; i < n4; i += 4 * (int64_t)blockDim.x) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t k = i + (int64_t)u * blockDim.x;
        v[u] = k < n4 ? __ldg(q + k) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i + (int64_t)u * blockDim.x >= n4) continue;
        fast(v[u].x); fast(v[u].y); fast(v[u].z); fast(v[u].w);
      }
    }
    // integer-valued with |v| < 2^23: A +- B of two such values is exact in
    // fp32 (the streaming kernel's fp64 path then forms S, D in fp32)
    notint |= fmaxf(fabsf(fmn), fabsf(fmx)) >= 8388608.0f;
    if (s1 - s1 == 0.0 && s2 - s2 == 0.0) {
      if (fmn <= fmx) {
        mn = (double)fmn;
        mx = (double)fmx;
      }
    } else {                                        // non-finite values: careful form
      s1 = 0.0; s2 = 0.0; mn = DBL_MAX; mx = -DBL_MAX; bad = 0.0;
      for (int64_t i = threadIdx.x; i < n4; i += 4 * (int64_t)blockDim.x)
        for (int u = 0; u < 4; ++u) {
          const int64_t k = i + (int64_t)u * blockDim.x;
          if (k >= n4) continue;
          const float4 w = __ldg(q + k);
          take(w.x); take(w.y); take(w.z); take(w.w);
        }
    }
  } else {
    for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
      const double dv = (double)p[i];
      take(dv);
      notint |= (dv != rint(dv)) | (fabs(dv) >= 8388608.0);
    }
  }
  if (inexact && __syncthreads_or(notint) && threadIdx.x == 0) atomicOr(inexact + k, 1);
  __shared__ double sh[5][8];
  s1 = warp_sum(s1); s2 = warp_sum(s2); bad = warp_sum(bad);
  mn = warp_min(mn); mx = warp_max(mx);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) { sh[0][w] = s1; sh[1][w] = s2; sh[2][w] = mn; sh[3][w] = mx; sh[4][w] = bad; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a1 = 0, a2 = 0, amn = DBL_MAX, amx = -DBL_MAX, ab = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      a1 += sh[0][i]; a2 += sh[1][i]; amn = fmin(amn, sh[2][i]); amx = fmax(amx, sh[3][i]); ab += sh[4][i];
    }
    ChunkStat cs;
    cs.n = (double)(end - beg) - ab;
    cs.mean = cs.n > 0 ? shift + a1 / cs.n : 0.0;
    cs.m2 = cs.n > 0 ? fmax(a2 - a1 * a1 / cs.n, 0.0) : 0.0;
    cs.mn = amn; cs.mx = amx; cs.bad = ab;
    // integer-valued chunk: every partial of a1 is an exact integer, and so
    // is shift * n (< 2^38), hence the raw sum is exact
    cs.sum = a1 + shift * (double)(end - beg);
    out[(int64_t)k * nchunk + c] = cs;
  }
}

// CTAs walk the (plane, chunk) items of planes [k0, k0 + n_items / nchunk)
// with a grid stride (one item per CTA unless the grid is persistent).
template <typename T>
__global__ void __launch_bounds__(256) plane_stats_kernel(const T* __restrict__ data, int64_t P, int nchunk,
                                                          int k0, int n_items, ChunkStat* __restrict__ out,
                                                          int* __restrict__ inexact) {
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    stats_chunk<T>(data, P, nchunk, k0 + it / nchunk, it % nchunk, out, inexact);
    __syncthreads();                          // thread 0 has read the shared partials
  }
}

__device__ __forceinline__ double sample_lag(const SampleGeom& g, int64_t i, int64_t j) {
  if (g.coords) {
    // d = c_i - c_j; sum over the last axis in order, no FMA contraction
    const double d0 = __dsub_rn(g.coords[i * 3 + 0], g.coords[j * 3 + 0]);
    const double d1 = __dsub_rn(g.coords[i * 3 + 1], g.coords[j * 3 + 1]);
    const double d2 = __dsub_rn(g.coords[i * 3 + 2], g.coords[j * 3 + 2]);
    return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
  }
  // structured samples: indices and plane sizes are below 2^32 (the plan
  // rejects parts with more samples), so 32-bit divisions give the same
  // quotients at a fraction of the 64-bit emulation's cost
  const uint32_t ui = (uint32_t)i, uj = (uint32_t)j, uP = (uint32_t)g.P, uW = (uint32_t)g.W;
  const uint32_t qi = ui / uP, ri = ui - qi * uP, qj = uj / uP, rj = uj - qj * uP;
  const uint32_t yi = ri / uW, xi = ri - yi * uW, yj = rj / uW, xj = rj - yj * uW;
  const int64_t dx = (int64_t)xi - xj, dy = (int64_t)yi - yj, dz = (int64_t)g.zloc[qi] - g.zloc[qj];
  return sqrt((double)(dx * dx + dy * dy + dz * dz));
}

// ---- pair draw: numpy default_rng(seed).integers(0, m, max_pairs) x 2 ------
// Raw PCG64 outputs are split into chunks of PT_RAW per thread; each thread
// jumps its LCG to the chunk start (pcg_advance), counts accepted Lemire
// halves, a single block scans the counts, and the same threads regenerate
// and scatter accepted draws to their stream positions (ii = first
// max_pairs draws, jj = the next max_pairs).  All pair classes of a plan are
// drawn by the same launches (blockIdx.y = class).
constexpr int PT_RAW = 16;
constexpr int PT_BLOCK = 256;

__global__ void __launch_bounds__(PT_BLOCK) pair_count_kernel(const PairJob* jobs) {
  const PairJob& J = jobs[blockIdx.y];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g == 0) {                                   // per-class accumulators start at zero
    *J.t.hbits = 0ull;
    for (int b = 0; b < MAX_BINS; ++b) J.t.counts[b] = 0;
  }
  if (J.triu) return;
  const int64_t r0 = g * PT_RAW;
  if (r0 >= J.n_raw) return;
  const int64_t r1 = min(J.n_raw, r0 + PT_RAW);
  const u128 inc = ((u128)J.inc_hi << 64) | J.inc_lo;
  u128 s = pcg_advance(((u128)J.st_hi << 64) | J.st_lo, inc, (uint64_t)r0);
  const u128 mul = pcg_mult();
  int c = 0;
  for (int64_t r = r0; r < r1; ++r) {
    s = s * mul + inc;
    const uint64_t raw = pcg_output(s);
    c += ((uint32_t)((uint64_t)(uint32_t)raw * J.m) >= J.thr);
    c += ((uint32_t)((uint64_t)(uint32_t)(raw >> 32) * J.m) >= J.thr);
  }
  J.t.cnt[g] = c;
}

// exclusive scan of the per-thread counts in one block per class; off[n] = total
__global__ void __launch_bounds__(1024) pair_scan_kernel(const PairJob* jobs) {
  const PairJob& J = jobs[blockIdx.x];
  if (J.triu) return;
  __shared__ int64_t part[1024];
  const int tid = threadIdx.x;
  const int64_t n = J.n_thr;
  const int64_t per = (n + 1023) / 1024;
  const int64_t b = min(n, tid * per), e = min(n, b + per);
  int64_t acc = 0;
  for (int64_t i = b; i < e; ++i) acc += J.t.cnt[i];
  part[tid] = acc;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t v = tid >= o ? part[tid - o] : 0;
    __syncthreads();
    part[tid] += v;
    __syncthreads();
  }
  int64_t run = part[tid] - acc;
  for (int64_t i = b; i < e; ++i) {
    J.t.off[i] = run;
    run += J.t.cnt[i];
  }
  if (tid == 1023) J.t.off[n] = part[1023];
}

__global__ void __launch_bounds__(PT_BLOCK) pair_scatter_kernel(const PairJob* jobs) {
  const PairJob& J = jobs[blockIdx.y];
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (J.triu) {
    // np.triu_indices(m, 1): row-major upper triangle (all pairs fit)
    const int64_t m = J.m;
    for (int64_t i = g; i < m - 1; i += (int64_t)gridDim.x * blockDim.x) {
      const int64_t o = i * (m - 1) - i * (i - 1) / 2;
      for (int64_t j = i + 1; j < m; ++j) {
        J.t.ii[o + (j - i - 1)] = (int32_t)i;
        J.t.jj[o + (j - i - 1)] = (int32_t)j;
      }
    }
    return;
  }
  const int64_t r0 = g * PT_RAW;
  if (r0 >= J.n_raw) return;
  int64_t pos = J.t.off[g];
  if (pos >= J.need) return;
  const int64_t r1 = min(J.n_raw, r0 + PT_RAW);
  const u128 inc = ((u128)J.inc_hi << 64) | J.inc_lo;
  u128 s = pcg_advance(((u128)J.st_hi << 64) | J.st_lo, inc, (uint64_t)r0);
  const u128 mul = pcg_mult();
  for (int64_t r = r0; r < r1 && pos < J.need; ++r) {
    s = s * mul + inc;
    const uint64_t raw = pcg_output(s);
    for (int h = 0; h < 2 && pos < J.need; ++h) {
      const uint64_t prod = (uint64_t)(uint32_t)(h ? (raw >> 32) : raw) * J.m;
      if ((uint32_t)prod >= J.thr) {
        const int32_t v = (int32_t)(prod >> 32);
        if (pos < J.max_pairs) J.t.ii[pos] = v; else J.t.jj[pos - J.max_pairs] = v;
        ++pos;
      }
    }
  }
}

// hmax reduced as the bit pattern of a non-negative double (order-preserving
// as uint64), so the max is exact and order independent
__global__ void __launch_bounds__(PT_BLOCK) pair_lag_kernel(const PairJob* jobs) {
  const PairJob& J = jobs[blockIdx.y];
  double lmax = 0.0;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < J.npairs; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = J.t.ii[p], j = J.t.jj[p];
    if (i == j) continue;
    lmax = fmax(lmax, sample_lag(J.geom, i, j));
  }
  lmax = warp_max(lmax);
  if ((threadIdx.x & 31) == 0 && lmax > 0.0) atomicMax(J.t.hbits, (unsigned long long)__double_as_longlong(lmax));
}

// scal: [0] hmax [1] lag_max [2] npairs [3] status
__global__ void __launch_bounds__(PT_BLOCK) pair_bin_kernel(const PairJob* jobs) {
  const PairJob& J = jobs[blockIdx.y];
  __shared__ unsigned long long h[MAX_BINS];
  if (threadIdx.x < MAX_BINS) h[threadIdx.x] = 0ull;
  __syncthreads();
  const int n_bins = J.n_bins;
  const double hmax = __longlong_as_double((long long)*J.t.hbits);
  const double step = hmax / (double)n_bins;   // np.linspace(0, hmax, n_bins + 1)
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < J.npairs; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = J.t.ii[p], j = J.t.jj[p];
    uint8_t b = 255;
    if (i != j) {
      const double lag = sample_lag(J.geom, i, j);
      if (lag > 0.0) {
        int c = 0;                                 // digitize: #edges <= lag
        for (int e = 0; e < n_bins; ++e) c += (__dmul_rn((double)e, step) <= lag);
        c += (hmax <= lag);
        c = min(max(c - 1, 0), n_bins - 1);
        b = (uint8_t)c;
        atomicAdd(&h[c], 1ull);
      }
    }
    J.t.bin[p] = b;
  }
  __syncthreads();
  if (threadIdx.x < n_bins && h[threadIdx.x])
    atomicAdd((unsigned long long*)&J.t.counts[threadIdx.x], h[threadIdx.x]);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    J.t.scal[0] = hmax;
    J.t.scal[1] = hmax;                              // lag_max == hmax when any lag > 0
    J.t.scal[2] = (double)J.npairs;
    J.t.scal[3] = (!J.triu && J.t.off[J.n_thr] < J.need) ? (double)PS_PAIRS_SHORT : 0.0;
  }
}

__global__ void __launch_bounds__(256) bins_kernel(BinsArgs a) {
  extern __shared__ double acc[];          // [n_bins][blockDim]
  // parts in reverse: the statistics pass streams the planes in order just
  // before, so the last parts' planes are still in L2 when their random
  // gathers start
  const int n_parts = a.n_parts > 0 ? a.n_parts : a.S;
  const int s = a.part0 + n_parts - 1 - (int)blockIdx.y, blk = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const PairTable t = a.tables[a.part_class[s]];
  const int64_t npairs = (int64_t)t.scal[2];
  const int64_t per = (npairs + a.nblk - 1) / a.nblk;
  const int64_t p0 = (int64_t)blk * per, p1 = min(npairs, p0 + per);
  for (int b = 0; b < a.n_bins; ++b) acc[b * nt + tid] = 0.0;
  const int64_t base = a.part_base[s];
  constexpr int U = 8;                       // gathers in flight per thread
  for (int64_t p = p0 + tid; p < p1; p += (int64_t)nt * U) {
    int32_t ii[U], jj[U];
    uint8_t bb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = p + (int64_t)u * nt;
      const bool ok = q < p1;
      bb[u] = ok ? t.bin[q] : (uint8_t)255;
      ii[u] = ok ? t.ii[q] : 0;
      jj[u] = ok ? t.jj[q] : 0;
    }
    double vi[U], vj[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (a.values) { vi[u] = a.values[base + ii[u]]; vj[u] = a.values[base + jj[u]]; }
      else { vi[u] = (double)__ldg(a.known + base + ii[u]); vj[u] = (double)__ldg(a.known + base + jj[u]); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (bb[u] == 255) continue;
      const double d = __dsub_rn(vi[u], vj[u]);
      acc[bb[u] * nt + tid] += __dmul_rn(0.5, __dmul_rn(d, d));
    }
  }
  __syncthreads();
  if (tid < a.n_bins) {
    double sum = 0.0;
    for (int i = 0; i < nt; ++i) sum += acc[tid * nt + i];
    a.partial[((int64_t)s * a.nblk + blk) * a.n_bins + tid] = sum;
  }
}

__global__ void __launch_bounds__(FIT_THREADS) fit_kernel(FitArgs a) {
  // One CTA of FIT_WARPS warps per sub-part.  Statistics are merged
  // redundantly by every warp (same order -> same bits); bins are reduced
  // lane-per-bin; the TRF runs redundantly on every thread with residual
  // rows, Jacobian columns and the SVD's independent stages spread over the
  // threads (trf_warp.cuh).
  if ((int)threadIdx.x >= FIT_THREADS) return;
  const int s = a.part0 + blockIdx.x, lane = threadIdx.x & 31;
  const bool lead = threadIdx.x == 0;
  __shared__ TrfProblem P;
  // Chan merge of the part's chunk statistics: lanes merge strided chunks,
  // then a butterfly merges lanes in a canonical (lower, upper) order so every
  // lane ends with the same bits -- deterministic across runs.
  double n = 0.0, mean = 0.0, m2 = 0.0, mn = DBL_MAX, mx = -DBL_MAX, bad = 0.0;
  const int kb = a.part_b ? a.part_b[s] : 0, ke = a.part_e ? a.part_e[s] : 0;
  const int n_items = (ke - kb + 1) * a.nchunk;
  auto merge = [](double& na, double& ma, double& qa, double nb, double mb, double qb) {
    if (nb <= 0) return;
    if (na <= 0) { na = nb; ma = mb; qa = qb; return; }
    const double nn = na + nb, d = mb - ma;
    ma = ma + d * (nb / nn);
    qa = qa + qb + d * d * (na * nb / nn);
    na = nn;
  };
  for (int it = lane; it < n_items; it += 32) {
    const ChunkStat cs = a.stats[(int64_t)kb * a.nchunk + it];
    bad += cs.bad;
    if (cs.n <= 0) continue;
    mn = fmin(mn, cs.mn);
    mx = fmax(mx, cs.mx);
    merge(n, mean, m2, cs.n, cs.mean, cs.m2);
  }
  for (int o = 1; o < 32; o <<= 1) {
    const double on = __shfl_xor_sync(0xffffffffu, n, o), om = __shfl_xor_sync(0xffffffffu, mean, o),
                 oq = __shfl_xor_sync(0xffffffffu, m2, o);
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if (lane & o) {                       // (other, self): lower lane first
      double nn = on, mm = om, qq = oq;
      merge(nn, mm, qq, n, mean, m2);
      n = nn; mean = mm; m2 = qq;
    } else {
      merge(n, mean, m2, on, om, oq);
    }
  }
  if (lead) {
    a.lohi[2 * s + 0] = mn;
    a.lohi[2 * s + 1] = mx;
  }
  int status = PS_OK;
  if (bad > 0) status = PS_NONFINITE;
  else if (n <= 0) status = PS_FIT_FAILED;
  if (!a.fit) { if (lead) a.status[s] = status; return; }
  const double svar = a.svar ? a.svar[s] : m2 / n;
  const int64_t m = a.part_m[s];
  if (m * (m - 1) / 2 < 30) { if (lead) a.status[s] = PS_INSUFFICIENT; return; }
  const PairTable t = a.tables[a.part_class[s]];
  if (t.scal[3] != 0.0) { if (lead) a.status[s] = PS_PAIRS_SHORT; return; }
  const double hmax = t.scal[0];
  if (!(hmax > 0.0)) { if (lead) a.status[s] = PS_DEGENERATE; return; }
  double* model = a.models + 3 * s;
  if (svar == 0.0) {                    // kriging.py:294-297
    if (lead) {
      model[0] = 0.0; model[1] = 0.0; model[2] = fmax(t.scal[1], 1.0);
      a.status[s] = status;
    }
    return;
  }
  // non-empty bins -> residual rows, in bin order
  const double step = hmax / (double)a.n_bins;
  const int64_t cnt = lane < a.n_bins ? t.counts[lane] : 0;
  const unsigned nzmask = __ballot_sync(0xffffffffu, cnt > 0);
  if (cnt > 0) {
    double sum = 0.0;
    if (a.bsum) sum = a.bsum[(int64_t)s * a.n_bins + lane];
    else
      for (int blk = 0; blk < a.nblk; ++blk) sum += a.partial[((int64_t)s * a.nblk + blk) * a.n_bins + lane];
    const int r = __popc(nzmask & ((1u << lane) - 1u));
    // 0.5 * (edges[:-1] + edges[1:]) without contraction (numpy rounding)
    const double e0 = __dmul_rn((double)lane, step);
    const double e1 = (lane + 1 == a.n_bins) ? hmax : __dmul_rn((double)(lane + 1), step);
    P.h[r] = __dmul_rn(0.5, __dadd_rn(e0, e1));
    P.gemp[r] = sum / (double)cnt;
    P.w[r] = sqrt((double)cnt);
  }
  if (lane == 0) { P.kind = a.kind; P.nb = __popc(nzmask); }   // identical from both warps
  __syncthreads();
  const double x0[3] = {0.0, svar, hmax / 3.0};
  const double lb[3] = {0.0, 0.0, 1e-6};
  const double ub[3] = {2.0 * svar + 1e-12, 4.0 * svar + 1e-12, 10.0 * hmax};
  if (!(ub[2] > lb[2])) { if (lead) a.status[s] = PS_FIT_FAILED; return; }
  __shared__ FitShared fsh;
  TrfResult r;
  r = trf_fit_t(WarpEval(P, fsh, threadIdx.x), x0, lb, ub);
  if (!lead) return;
  if (r.status < 0) { a.status[s] = PS_FIT_FAILED; return; }
  const double nug = pymax(r.x[0], 0.0);
  model[0] = nug;
  model[1] = nug + pymax(r.x[1], 0.0);
  model[2] = pymax(r.x[2], 1e-6);
  a.status[s] = status;
}

}  // namespace


cudaError_t launch_plane_stats(const float* known, int k0, int k1, int64_t P, ChunkStat* out, int nchunk,
                               cudaStream_t st, int* inexact) {
  if (k1 <= k0) return cudaSuccess;
  if (inexact) {
    cudaError_t e = cudaMemsetAsync(inexact + k0, 0, sizeof(int) * (size_t)(k1 - k0), st);
    if (e != cudaSuccess) return e;
  }
  // one CTA per (plane, chunk) item by default: persistent CTAs (one wave,
  // VK_STATS_PERSISTENT=1) shorten the pass alone but hold every SM slot, so
  // the concurrent high-priority pair draw starts later -- C4 step 1.304-1.308
  // ms one CTA per item vs 1.313-1.319 ms persistent (same box, alternating)
  static int slots = 0;
  if (!slots) {
    slots = 1 << 30;
    if (const char* e = std::getenv("VK_STATS_PERSISTENT"); e && std::atoi(e) != 0) {
      int dev = 0, sms = 0, per = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, plane_stats_kernel<float>, 256, 0);
      slots = std::max(1, sms * std::max(1, per));
    }
  }
  const int n_items = (k1 - k0) * nchunk;
  plane_stats_kernel<float><<<std::min(n_items, slots), 256, 0, st>>>(known, P, nchunk, k0, n_items, out, inexact);
  return cudaGetLastError();
}

cudaError_t launch_plane_stats_f64(const double* values, int64_t m, ChunkStat* out, int nchunk,
                                   cudaStream_t st) {
  plane_stats_kernel<double><<<nchunk, 256, 0, st>>>(values, m, nchunk, 0, nchunk, out, nullptr);
  return cudaGetLastError();
}

PairJob make_pair_job(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t m,
                      int64_t max_pairs, int n_bins, SampleGeom geom, PairTable t) {
  PairJob J{};
  J.st_hi = st_hi; J.st_lo = st_lo; J.inc_hi = inc_hi; J.inc_lo = inc_lo;
  J.t = t;
  J.geom = geom;
  J.n_bins = n_bins;
  J.max_pairs = max_pairs;
  const int64_t total = m * (m - 1) / 2;
  J.triu = total <= max_pairs;
  J.npairs = J.triu ? total : max_pairs;
  J.m = (uint32_t)m;
  if (!J.triu) {
    J.thr = lemire_threshold(J.m);
    J.need = 2 * max_pairs;
    const double prej = (double)J.thr / 4294967296.0;
    J.n_raw = (int64_t)((double)J.need * (1.0 + 4.0 * prej) / 2.0) + 4096;
    J.n_thr = (J.n_raw + PT_RAW - 1) / PT_RAW;
  }
  return J;
}

int64_t pair_scratch_elems(int64_t m, int64_t max_pairs) {
  if (m * (m - 1) / 2 <= max_pairs) return 1;
  const uint32_t thr = lemire_threshold((uint32_t)m);
  const double prej = (double)thr / 4294967296.0;
  const int64_t n_raw = (int64_t)((double)(2 * max_pairs) * (1.0 + 4.0 * prej) / 2.0) + 4096;
  return (n_raw + PT_RAW - 1) / PT_RAW;
}

// The whole draw in one cooperative launch (blockIdx.y = class): count the
// accepted Lemire halves of each thread's PT_RAW raw outputs (the LCG state
// at the chunk start is kept in registers), block scan, grid sync, block
// offsets from the per-block totals, scatter by regenerating the chunk,
// grid sync, lag maximum, grid sync, digitize.  Same arithmetic and outputs
// as the five-kernel form above, without four launch gaps and tails.
__global__ void __launch_bounds__(PT_BLOCK) pair_draw_kernel(const PairJob* jobs) {
  cg::grid_group grid = cg::this_grid();
  const PairJob& J = jobs[blockIdx.y];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t g = (int64_t)blockIdx.x * PT_BLOCK + tid;
  const int64_t nb_gen = J.triu ? 0 : (J.n_thr + PT_BLOCK - 1) / PT_BLOCK;
  if (blockIdx.x == 0 && tid == 0) {
    *J.t.hbits = 0ull;
    for (int b = 0; b < MAX_BINS; ++b) J.t.counts[b] = 0;
  }
  const u128 inc = ((u128)J.inc_hi << 64) | J.inc_lo;
  const u128 mul = pcg_mult();
  const int64_t r0 = g * PT_RAW;
  const bool gen = !J.triu && r0 < J.n_raw;
  const int64_t r1 = gen ? min(J.n_raw, r0 + PT_RAW) : r0;
  u128 s0 = 0;
  int c = 0;
  if (gen) {
    s0 = pcg_advance(((u128)J.st_hi << 64) | J.st_lo, inc, (uint64_t)r0);
    u128 s = s0;
    for (int64_t r = r0; r < r1; ++r) {
      s = s * mul + inc;
      const uint64_t raw = pcg_output(s);
      c += ((uint32_t)((uint64_t)(uint32_t)raw * J.m) >= J.thr);
      c += ((uint32_t)((uint64_t)(uint32_t)(raw >> 32) * J.m) >= J.thr);
    }
  }
  // block-exclusive scan of the counts
  __shared__ int wsum[PT_BLOCK / 32];
  __shared__ int64_t boff, total;
  int incl = c;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  int before = 0, btot = 0;
  for (int w = 0; w < PT_BLOCK / 32; ++w) {
    before += w < warp ? wsum[w] : 0;
    btot += wsum[w];
  }
  const int excl = before + incl - c;
  if (tid == 0 && blockIdx.x < nb_gen) J.t.cnt[blockIdx.x] = btot;
  grid.sync();
  if (warp == 0) {
    int64_t a = 0, t = 0;
    for (int64_t b = lane; b < nb_gen; b += 32) {
      const int64_t v = J.t.cnt[b];
      a += b < (int64_t)blockIdx.x ? v : 0;
      t += v;
    }
    for (int o = 16; o; o >>= 1) {
      a += __shfl_xor_sync(0xffffffffu, a, o);
      t += __shfl_xor_sync(0xffffffffu, t, o);
    }
    if (lane == 0) {
      boff = a;
      total = t;
    }
  }
  __syncthreads();
  if (blockIdx.x == 0 && tid == 0 && !J.triu) J.t.off[J.n_thr] = total;
  if (J.triu) {
    // np.triu_indices(m, 1): row-major upper triangle (all pairs fit)
    const int64_t m = J.m;
    for (int64_t i = g; i < m - 1; i += (int64_t)gridDim.x * PT_BLOCK) {
      const int64_t o = i * (m - 1) - i * (i - 1) / 2;
      for (int64_t j = i + 1; j < m; ++j) {
        J.t.ii[o + (j - i - 1)] = (int32_t)i;
        J.t.jj[o + (j - i - 1)] = (int32_t)j;
      }
    }
  } else if (gen) {
    int64_t pos = boff + excl;
    u128 s = s0;
    for (int64_t r = r0; r < r1 && pos < J.need; ++r) {
      s = s * mul + inc;
      const uint64_t raw = pcg_output(s);
      for (int h = 0; h < 2 && pos < J.need; ++h) {
        const uint64_t prod = (uint64_t)(uint32_t)(h ? (raw >> 32) : raw) * J.m;
        if ((uint32_t)prod >= J.thr) {
          const int32_t v = (int32_t)(prod >> 32);
          if (pos < J.max_pairs) J.t.ii[pos] = v; else J.t.jj[pos - J.max_pairs] = v;
          ++pos;
        }
      }
    }
  }
  grid.sync();
  double lmax = 0.0;
  for (int64_t p = g; p < J.npairs; p += (int64_t)gridDim.x * PT_BLOCK) {
    const int64_t i = J.t.ii[p], j = J.t.jj[p];
    if (i == j) continue;
    lmax = fmax(lmax, sample_lag(J.geom, i, j));
  }
  lmax = warp_max(lmax);
  if (lane == 0 && lmax > 0.0) atomicMax(J.t.hbits, (unsigned long long)__double_as_longlong(lmax));
  grid.sync();
  __shared__ unsigned long long h[MAX_BINS];
  if (tid < MAX_BINS) h[tid] = 0ull;
  __syncthreads();
  const int n_bins = J.n_bins;
  const double hmax = __longlong_as_double((long long)*J.t.hbits);
  const double step = hmax / (double)n_bins;   // np.linspace(0, hmax, n_bins + 1)
  for (int64_t p = g; p < J.npairs; p += (int64_t)gridDim.x * PT_BLOCK) {
    const int64_t i = J.t.ii[p], j = J.t.jj[p];
    uint8_t b = 255;
    if (i != j) {
      const double lag = sample_lag(J.geom, i, j);
      if (lag > 0.0) {
        int cb = 0;                                // digitize: #edges <= lag
        for (int e = 0; e < n_bins; ++e) cb += (__dmul_rn((double)e, step) <= lag);
        cb += (hmax <= lag);
        cb = min(max(cb - 1, 0), n_bins - 1);
        b = (uint8_t)cb;
        atomicAdd(&h[cb], 1ull);
      }
    }
    J.t.bin[p] = b;
  }
  __syncthreads();
  if (tid < n_bins && h[tid]) atomicAdd((unsigned long long*)&J.t.counts[tid], h[tid]);
  if (blockIdx.x == 0 && tid == 0) {
    J.t.scal[0] = hmax;
    J.t.scal[1] = hmax;                              // lag_max == hmax when any lag > 0
    J.t.scal[2] = (double)J.npairs;
    J.t.scal[3] = (!J.triu && total < J.need) ? (double)PS_PAIRS_SHORT : 0.0;
  }
}

static cudaError_t launch_pair_draw(const PairJob* d_jobs, const PairJob* h_jobs, int n_jobs, cudaStream_t st,
                                    int* launches) {
  int64_t max_thr = 1, max_pairs = 1, max_m = 1;
  for (int c = 0; c < n_jobs; ++c) {
    max_thr = std::max(max_thr, h_jobs[c].n_thr);
    max_pairs = std::max(max_pairs, h_jobs[c].npairs);
    if (h_jobs[c].triu) max_m = std::max<int64_t>(max_m, h_jobs[c].m);
  }
  const unsigned nb = (unsigned)std::max<int64_t>((max_thr + PT_BLOCK - 1) / PT_BLOCK,
                                                  std::min<int64_t>(1024, (max_m + PT_BLOCK - 1) / PT_BLOCK));
  // one cooperative launch when the grid fits on the device at once; the
  // five-kernel form otherwise (or with VK_PAIR_DRAW_SPLIT=1)
  static int coop_slots = -1;
  if (coop_slots < 0) {
    int dev = 0, sms = 0, per = 0, coop = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, pair_draw_kernel, PT_BLOCK, 0);
    const char* e = std::getenv("VK_PAIR_DRAW_SPLIT");
    coop_slots = (coop && !(e && std::atoi(e) != 0)) ? sms * per : 0;
  }
  {
    // enough blocks for the lag / digitize passes too (4 pairs per thread)
    const int64_t want = std::max<int64_t>(nb, (max_pairs + 4 * PT_BLOCK - 1) / (4 * PT_BLOCK));
    const int64_t cap = coop_slots / std::max(1, n_jobs);
    if (cap >= nb) {
      dim3 grid((unsigned)std::min(want, cap), n_jobs);
      void* args[] = {(void*)&d_jobs};
      if (launches) *launches = 1;
      return cudaLaunchCooperativeKernel((void*)pair_draw_kernel, grid, dim3(PT_BLOCK), args, 0, st);
    }
  }
  if (launches) *launches = 5;
  pair_count_kernel<<<dim3(nb, n_jobs), PT_BLOCK, 0, st>>>(d_jobs);
  pair_scan_kernel<<<n_jobs, 1024, 0, st>>>(d_jobs);
  pair_scatter_kernel<<<dim3(nb, n_jobs), PT_BLOCK, 0, st>>>(d_jobs);
  const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(1184, (max_pairs + PT_BLOCK - 1) / PT_BLOCK));
  pair_lag_kernel<<<dim3(gb, n_jobs), PT_BLOCK, 0, st>>>(d_jobs);
  pair_bin_kernel<<<dim3(gb, n_jobs), PT_BLOCK, 0, st>>>(d_jobs);
  return cudaGetLastError();
}

// draw, then the stable bin order of the pairs (tables that keep one)
cudaError_t launch_pair_tables(const PairJob* d_jobs, const PairJob* h_jobs, int n_jobs, cudaStream_t st,
                               int* launches) {
  cudaError_t e = launch_pair_draw(d_jobs, h_jobs, n_jobs, st, launches);
  if (e != cudaSuccess) return e;
  bool order = false;
  for (int c = 0; c < n_jobs; ++c) order |= h_jobs[c].t.order != nullptr;
  if (!order) return cudaSuccess;
  if (launches) *launches += 1;
  return launch_pair_order(d_jobs, h_jobs, n_jobs, st);
}

cudaError_t launch_bins(const BinsArgs& a, cudaStream_t st) {
  dim3 grid(a.nblk, a.n_parts > 0 ? a.n_parts : a.S);
  const size_t smem = (size_t)a.n_bins * 256 * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(bins_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  bins_kernel<<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

#ifdef VK_FIT_PROFILE
extern "C" int vk_debug_fit_profile(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, vk::g_fit_prof, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(vk::g_fit_prof, z, sizeof(z));
  }
  return 0;
}
#endif

cudaError_t launch_fit(const FitArgs& a, cudaStream_t st) {
  if (a.n_parts <= 0) return cudaSuccess;
  if (a.reserve_smem > 48 * 1024) {
    static int set_to = 0;
    if (set_to < a.reserve_smem) {
      cudaError_t e = cudaFuncSetAttribute(fit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           a.reserve_smem);
      if (e != cudaSuccess) return e;
      set_to = a.reserve_smem;
    }
  }
  fit_kernel<<<a.n_parts, FIT_THREADS, a.reserve_smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace vk
