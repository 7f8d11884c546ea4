// Empirical semivariogram + bounded fit per Z sub-part (fit_variogram,
// kriging.py:264-328), and the per-part clamp range (kriging.py:475-479).
//
//   plane_stats  : one pass over the known planes -> per-chunk count / mean /
//                  M2 / min / max (deterministic block trees; merged per part
//                  in a fixed order with Chan's update) -> svar, lo, hi.
//   pair_table   : numpy-identical pair draw (PCG64 + Lemire, see pcg64.h)
//                  with LCG jump-ahead and a block-wide stream compaction,
//                  then lags, hmax, bin index per pair and bin counts.  Lags
//                  and bins depend only on geometry, so one table serves every
//                  part with the same sample layout.
//   bins         : per part, sum of 0.5*(v_i - v_j)^2 per bin; per-thread
//                  shared-memory accumulators reduced in a fixed order.
//   fit          : per part, the TRF fit (trf.h) on the non-empty bins.
#include <cuda_runtime.h>
#include <cfloat>
#include "pcg64.h"
#include "trf.h"
#include "vk_kernels.h"

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

template <typename T>
__global__ void __launch_bounds__(256) plane_stats_kernel(const T* __restrict__ data, int64_t P,
                                                          int nchunk, ChunkStat* __restrict__ out) {
  const int k = blockIdx.y, c = blockIdx.x;
  const int64_t beg = (int64_t)c * STATS_CHUNK;
  const int64_t end = min(P, beg + (int64_t)STATS_CHUNK);
  const T* p = data + (int64_t)k * P;
  const double shift = (beg < end) ? (double)p[beg] : 0.0;
  double s1 = 0.0, s2 = 0.0, mn = DBL_MAX, mx = -DBL_MAX, bad = 0.0;
  for (int64_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const double v = (double)p[i];
    if (!(v - v == 0.0)) { bad += 1.0; continue; }
    const double d = v - shift;
    s1 += d;
    s2 = fma(d, d, s2);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
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
    out[(int64_t)k * nchunk + c] = cs;
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
  const int64_t qi = i / g.P, ri = i - qi * g.P, qj = j / g.P, rj = j - qj * g.P;
  const int64_t yi = ri / g.W, xi = ri - yi * g.W, yj = rj / g.W, xj = rj - yj * g.W;
  const int64_t dx = xi - xj, dy = yi - yj, dz = (int64_t)g.zloc[qi] - g.zloc[qj];
  return sqrt((double)(dx * dx + dy * dy + dz * dz));
}

constexpr int PT_THREADS = 1024;

__global__ void __launch_bounds__(PT_THREADS) pair_table_kernel(
    uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t m,
    int64_t max_pairs, int n_bins, SampleGeom geom, PairTable t) {
  __shared__ int64_t s_cnt[PT_THREADS];
  __shared__ double s_red[2][32];
  __shared__ unsigned long long s_counts[MAX_BINS];
  __shared__ int64_t s_total;
  const int tid = threadIdx.x;
  const int64_t total_pairs = m * (m - 1) / 2;
  int64_t npairs;
  int status = 0;
  if (total_pairs <= max_pairs) {
    // np.triu_indices(m, 1): row-major upper triangle
    npairs = total_pairs;
    for (int64_t i = tid; i < m - 1; i += PT_THREADS) {
      const int64_t off = i * (m - 1) - i * (i - 1) / 2;
      for (int64_t j = i + 1; j < m; ++j) {
        t.ii[off + (j - i - 1)] = (int32_t)i;
        t.jj[off + (j - i - 1)] = (int32_t)j;
      }
    }
  } else {
    npairs = max_pairs;
    const u128 state = ((u128)st_hi << 64) | st_lo;
    const u128 inc = ((u128)inc_hi << 64) | inc_lo;
    const uint32_t mm = (uint32_t)m;
    const uint32_t thr = lemire_threshold(mm);
    const int64_t need = 2 * max_pairs;
    const double prej = (double)thr / 4294967296.0;
    int64_t R = (int64_t)((double)need * (1.0 + 4.0 * prej) / 2.0) + 4096;
    for (int attempt = 0; attempt < 8; ++attempt) {
      const int64_t B = (R + PT_THREADS - 1) / PT_THREADS;
      const int64_t r0 = min(R, (int64_t)tid * B), r1 = min(R, r0 + B);
      int64_t cnt = 0;
      u128 s = pcg_advance(state, inc, (uint64_t)r0);
      const u128 mul = pcg_mult();
      for (int64_t r = r0; r < r1; ++r) {
        s = s * mul + inc;
        const uint64_t raw = pcg_output(s);
        cnt += ((uint32_t)((uint64_t)(uint32_t)raw * mm) >= thr);
        cnt += ((uint32_t)((uint64_t)(uint32_t)(raw >> 32) * mm) >= thr);
      }
      s_cnt[tid] = cnt;
      __syncthreads();
      // inclusive Hillis-Steele scan over 1024 counts
      for (int o = 1; o < PT_THREADS; o <<= 1) {
        const int64_t v = (tid >= o) ? s_cnt[tid - o] : 0;
        __syncthreads();
        s_cnt[tid] += v;
        __syncthreads();
      }
      const int64_t accepted = s_cnt[PT_THREADS - 1];
      int64_t pos = s_cnt[tid] - cnt;
      __syncthreads();
      if (accepted < need) { R *= 2; continue; }
      s = pcg_advance(state, inc, (uint64_t)r0);
      for (int64_t r = r0; r < r1 && pos < need; ++r) {
        s = s * mul + inc;
        const uint64_t raw = pcg_output(s);
        for (int h = 0; h < 2 && pos < need; ++h) {
          const uint64_t prod = (uint64_t)(uint32_t)(h ? (raw >> 32) : raw) * mm;
          if ((uint32_t)prod >= thr) {
            const int32_t v = (int32_t)(prod >> 32);
            if (pos < max_pairs) t.ii[pos] = v; else t.jj[pos - max_pairs] = v;
            ++pos;
          }
        }
      }
      status = 0;
      break;
    }
    if (s_cnt[PT_THREADS - 1] < need) status = PS_PAIRS_SHORT;
  }
  __syncthreads();   // pair arrays visible block-wide
  // lags: lag_max over kept pairs, hmax over lag > 0
  double lmax = 0.0;
  for (int64_t p = tid; p < npairs; p += PT_THREADS) {
    const int64_t i = t.ii[p], j = t.jj[p];
    if (i == j) continue;
    lmax = fmax(lmax, sample_lag(geom, i, j));
  }
  lmax = warp_max(lmax);
  if ((tid & 31) == 0) s_red[0][tid >> 5] = lmax;
  if (tid < MAX_BINS) s_counts[tid] = 0ull;
  __syncthreads();
  if (tid == 0) {
    double a = 0.0;
    for (int w = 0; w < PT_THREADS / 32; ++w) a = fmax(a, s_red[0][w]);
    s_red[1][0] = a;
  }
  __syncthreads();
  const double hmax = s_red[1][0];
  // edges = np.linspace(0, hmax, n_bins + 1); bin = clip(digitize - 1)
  const double step = hmax / (double)n_bins;
  for (int64_t p = tid; p < npairs; p += PT_THREADS) {
    const int64_t i = t.ii[p], j = t.jj[p];
    uint8_t b = 255;
    if (i != j) {
      const double lag = sample_lag(geom, i, j);
      if (lag > 0.0) {
        int c = 0;
        for (int e = 0; e < n_bins; ++e) c += ((double)e * step <= lag);
        c += (hmax <= lag);
        c = min(max(c - 1, 0), n_bins - 1);
        b = (uint8_t)c;
        atomicAdd(&s_counts[c], 1ull);
      }
    }
    t.bin[p] = b;
  }
  __syncthreads();
  if (tid < n_bins) t.counts[tid] = (int64_t)s_counts[tid];
  if (tid == 0) {
    t.scal[0] = hmax;
    t.scal[1] = hmax;      // lag_max == hmax whenever any lag > 0
    t.scal[2] = (double)npairs;
    t.scal[3] = (double)status;
  }
}

__global__ void __launch_bounds__(256) bins_kernel(BinsArgs a) {
  extern __shared__ double acc[];          // [n_bins][blockDim]
  const int s = blockIdx.y, blk = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const PairTable t = a.tables[a.part_class[s]];
  const int64_t npairs = (int64_t)t.scal[2];
  const int64_t per = (npairs + a.nblk - 1) / a.nblk;
  const int64_t p0 = (int64_t)blk * per, p1 = min(npairs, p0 + per);
  for (int b = 0; b < a.n_bins; ++b) acc[b * nt + tid] = 0.0;
  const int64_t base = a.part_base[s];
  for (int64_t p = p0 + tid; p < p1; p += nt) {
    const uint8_t b = t.bin[p];
    if (b == 255) continue;
    double vi, vj;
    if (a.values) { vi = a.values[base + t.ii[p]]; vj = a.values[base + t.jj[p]]; }
    else { vi = (double)__ldg(a.known + base + t.ii[p]); vj = (double)__ldg(a.known + base + t.jj[p]); }
    const double d = __dsub_rn(vi, vj);
    acc[b * nt + tid] += __dmul_rn(0.5, __dmul_rn(d, d));
  }
  __syncthreads();
  if (tid < a.n_bins) {
    double sum = 0.0;
    for (int i = 0; i < nt; ++i) sum += acc[tid * nt + i];
    a.partial[((int64_t)s * a.nblk + blk) * a.n_bins + tid] = sum;
  }
}

__global__ void __launch_bounds__(32) fit_kernel(FitArgs a) {
  const int s = blockIdx.x;
  if (threadIdx.x != 0) return;
  // --- merge chunk statistics of the part's planes in a fixed order
  double n = 0.0, mean = 0.0, m2 = 0.0, mn = DBL_MAX, mx = -DBL_MAX, bad = 0.0;
  const int kb = a.part_b ? a.part_b[s] : 0, ke = a.part_e ? a.part_e[s] : 0;
  for (int k = kb; k <= ke; ++k) {
    for (int c = 0; c < a.nchunk; ++c) {
      const ChunkStat cs = a.stats[(int64_t)k * a.nchunk + c];
      bad += cs.bad;
      if (cs.n <= 0) continue;
      mn = fmin(mn, cs.mn);
      mx = fmax(mx, cs.mx);
      const double nn = n + cs.n, d = cs.mean - mean;
      mean = mean + d * (cs.n / nn);
      m2 = m2 + cs.m2 + d * d * (n * cs.n / nn);
      n = nn;
    }
  }
  a.lohi[2 * s + 0] = mn;
  a.lohi[2 * s + 1] = mx;
  int status = PS_OK;
  if (bad > 0 || n <= 0) status = PS_FIT_FAILED;
  if (!a.fit) { a.status[s] = status; return; }
  const double svar = m2 / n;
  const int64_t m = a.part_m[s];
  if (m * (m - 1) / 2 < 30) { a.status[s] = PS_INSUFFICIENT; return; }
  const PairTable t = a.tables[a.part_class[s]];
  if (t.scal[3] != 0.0) { a.status[s] = PS_PAIRS_SHORT; return; }
  const double hmax = t.scal[0];
  if (!(hmax > 0.0)) { a.status[s] = PS_DEGENERATE; return; }
  double* model = a.models + 3 * s;
  if (svar == 0.0) {                    // kriging.py:294-297
    model[0] = 0.0; model[1] = 0.0; model[2] = fmax(t.scal[1], 1.0);
    a.status[s] = status;
    return;
  }
  TrfProblem P;
  P.kind = a.kind;
  P.nb = 0;
  const double step = hmax / (double)a.n_bins;
  for (int b = 0; b < a.n_bins; ++b) {
    const int64_t cnt = t.counts[b];
    if (cnt <= 0) continue;
    double sum = 0.0;
    for (int blk = 0; blk < a.nblk; ++blk) sum += a.partial[((int64_t)s * a.nblk + blk) * a.n_bins + b];
    const double e0 = (double)b * step;
    const double e1 = (b + 1 == a.n_bins) ? hmax : (double)(b + 1) * step;
    P.h[P.nb] = 0.5 * (e0 + e1);
    P.gemp[P.nb] = sum / (double)cnt;
    P.w[P.nb] = sqrt((double)cnt);
    P.nb++;
  }
  const double x0[3] = {0.0, svar, hmax / 3.0};
  const double lb[3] = {0.0, 0.0, 1e-6};
  const double ub[3] = {2.0 * svar + 1e-12, 4.0 * svar + 1e-12, 10.0 * hmax};
  if (!(ub[2] > lb[2])) { a.status[s] = PS_FIT_FAILED; return; }
  const TrfResult r = trf_fit(P, x0, lb, ub);
  if (r.status < 0) { a.status[s] = PS_FIT_FAILED; return; }
  const double nug = pymax(r.x[0], 0.0);
  model[0] = nug;
  model[1] = nug + pymax(r.x[1], 0.0);
  model[2] = pymax(r.x[2], 1e-6);
  a.status[s] = status;
}

}  // namespace

cudaError_t launch_plane_stats(const float* known, int K, int64_t P, ChunkStat* out, int nchunk,
                               cudaStream_t st) {
  dim3 grid(nchunk, K);
  plane_stats_kernel<float><<<grid, 256, 0, st>>>(known, P, nchunk, out);
  return cudaGetLastError();
}

cudaError_t launch_plane_stats_f64(const double* values, int64_t m, ChunkStat* out, int nchunk,
                                   cudaStream_t st) {
  dim3 grid(nchunk, 1);
  plane_stats_kernel<double><<<grid, 256, 0, st>>>(values, m, nchunk, out);
  return cudaGetLastError();
}

cudaError_t launch_pair_table(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo,
                              int64_t m, int64_t max_pairs, int n_bins, SampleGeom geom,
                              PairTable t, cudaStream_t st) {
  pair_table_kernel<<<1, PT_THREADS, 0, st>>>(st_hi, st_lo, inc_hi, inc_lo, m, max_pairs, n_bins,
                                              geom, t);
  return cudaGetLastError();
}

cudaError_t launch_bins(const BinsArgs& a, cudaStream_t st) {
  dim3 grid(a.nblk, a.S);
  const size_t smem = (size_t)a.n_bins * 256 * sizeof(double);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(bins_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  bins_kernel<<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_fit(const FitArgs& a, cudaStream_t st) {
  fit_kernel<<<a.S, 32, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace vk
