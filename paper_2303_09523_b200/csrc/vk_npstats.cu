// numpy-exact statistics of fit_variogram (kriging.py:288-309) on the device.
//
// The fit's starting point and bounds come from svar = values.var() and its
// residuals from bin_gamma = np.bincount(which, weights=sq) / counts; the TRF
// amplifies ulp-level differences in either, so both are reproduced bit for
// bit here:
//
//   npvar  : numpy's float64 sum is a pairwise summation (DOUBLE_pairwise_sum:
//            leaves of <= 128 elements with eight strided accumulators, split
//            at n/2 rounded down to a multiple of 8).  The tree depends only on
//            the sample count m, so the host builds it once per pair class
//            (build_npsum_warp); the device sums every subtree of <= 32
//            leaves with one warp (a lane per leaf, numpy's combination order)
//            and then adds the nodes above level by level in one CTA per part.  Two
//            rounds: mean = sum(v) / m, then svar = sum((v - mean)^2) / m.
//   bins   : np.bincount accumulates each bin's weights sequentially in pair
//            order.  pair_order_kernel sorts the pairs of a class by bin
//            (stable counting sort, once per draw); binsq_kernel forms
//            0.5 * (v_i - v_j)^2 for every pair at its sorted slot (random
//            gathers, fully parallel); binsum_kernel adds each bin's slots in
//            order, one lane per bin.
#include <cuda_runtime.h>
#include <algorithm>
#include <vector>
#include "vk_kernels.h"
#include "npsum.h"

namespace vk {

namespace {

// ---- pairwise sums ----------------------------------------------------------
// value of sample i: MODE 0 v, MODE 1 (v - mean)^2 -- numpy forms arr - mean
// and x * x as separate float64 arrays (one rounding each)
template <int MODE>
__device__ __forceinline__ double npv(const float* __restrict__ known, const double* __restrict__ values,
                                      int64_t i, double mean) {
  const double v = values ? values[i] : (double)__ldg(known + i);
  if (MODE == 0) return v;
  const double t = __dsub_rn(v, mean);
  return __dmul_rn(t, t);
}

// part s is integer-valued (every known plane flagged exact by the
// statistics pass, |v| < 2^23, m < 2^30): each pairwise partial sum of the
// values is an exact integer below 2^53, so numpy's sum equals the exact sum
__device__ __forceinline__ bool int_part(const NpVarArgs& a, int s) {
  if (!a.inexact || !a.stats || a.values || a.part_m[s] >= (int64_t(1) << 30)) return false;
  for (int k = a.part_b[s]; k <= a.part_e[s]; ++k)
    if (__ldg(a.inexact + k)) return false;
  return true;
}

// numpy's leaf sum of n <= 128 elements starting at absolute sample g: eight
// strided accumulators r[k] (initialised with the first eight values), combined
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the n % 8 tail in order
template <int MODE>
__device__ __forceinline__ double np_leaf_sum(const NpVarArgs& a, int64_t g, int n, double mean) {
  auto f = [&](double v) -> double {
    if (MODE == 0) return v;
    const double t = __dsub_rn(v, mean);
    return __dmul_rn(t, t);
  };
  auto at = [&](int i) -> double { return f(a.values ? a.values[g + i] : (double)__ldg(a.known + g + i)); };
  if (n < 8) {
    double res = -0.0;
    for (int i = 0; i < n; ++i) res = __dadd_rn(res, at(i));
    return res;
  }
  const int n8 = n - n % 8;
  double r[8];
  if (!a.values && ((g & 3) == 0)) {
    const float4* p = reinterpret_cast<const float4*>(a.known + g);
    {
      const float4 x0 = __ldg(p), x1 = __ldg(p + 1);
      r[0] = f(x0.x); r[1] = f(x0.y); r[2] = f(x0.z); r[3] = f(x0.w);
      r[4] = f(x1.x); r[5] = f(x1.y); r[6] = f(x1.z); r[7] = f(x1.w);
    }
#pragma unroll 4
    for (int q = 2; q < n8 / 4; q += 2) {
      const float4 x0 = __ldg(p + q), x1 = __ldg(p + q + 1);
      r[0] = __dadd_rn(r[0], f(x0.x)); r[1] = __dadd_rn(r[1], f(x0.y));
      r[2] = __dadd_rn(r[2], f(x0.z)); r[3] = __dadd_rn(r[3], f(x0.w));
      r[4] = __dadd_rn(r[4], f(x1.x)); r[5] = __dadd_rn(r[5], f(x1.y));
      r[6] = __dadd_rn(r[6], f(x1.z)); r[7] = __dadd_rn(r[7], f(x1.w));
    }
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) r[k] = at(k);
    for (int i = 8; i < n8; i += 8)
#pragma unroll
      for (int k = 0; k < 8; ++k) r[k] = __dadd_rn(r[k], at(i + k));
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (int i = n8; i < n; ++i) res = __dadd_rn(res, at(i));
  return res;
}

// One warp per warp root (a subtree of <= 32 leaves, npsum.h): lane i sums
// leaf i straight from global memory (16-byte loads, each lane walking its own
// leaf), then lane 0 adds the subtree's internal nodes in height order from
// shared memory; the root's value goes to a.leaf for the top-tree kernel.
constexpr int NPW_WARPS = 8;
#ifndef VK_NPW_PAIR
#define VK_NPW_PAIR 1
#endif

template <int MODE>
__global__ void __launch_bounds__(32 * NPW_WARPS) npsum_warp_kernel(NpVarArgs a) {
  // the second pass walks the parts last to first: the statistics pass (and
  // the first pass) ended on the last parts' planes, which are still in L2
  const int s = a.part0 + (MODE == 1 ? (int)(gridDim.y - 1 - blockIdx.y) : (int)blockIdx.y);
  if (MODE == 0 && int_part(a, s)) return;              // the mean comes from the chunk sums
  const NpSumTree T = a.trees[a.part_class[s]];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * NPW_WARPS + warp;
  if (r >= T.nleaf) return;
  const int l0 = T.wr_leaf[r], nl = T.wr_leaf[r + 1] - l0;
  const double mean = MODE ? a.mean[s] : 0.0;
  __shared__ double val[NPW_WARPS][64];
#if VK_NPW_PAIR
  // two lanes per leaf, sixteen leaves per round: lane h of a leaf holds
  // numpy's accumulators r[4h .. 4h+3] and reads their four columns of every
  // eight-element row with one 16-byte load, so a load instruction touches
  // sixteen 32-byte sectors (a lane per leaf touched 32 lines per
  // instruction and was bound by L1 tag throughput at ~3 TB/s)
  {
    const int h = lane & 1;
    auto f = [&](float x) -> double {
      const double v = (double)x;
      if (MODE == 0) return v;
      const double t = __dsub_rn(v, mean);
      return __dmul_rn(t, t);
    };
    const int64_t base = a.part_base[s];
    for (int l = lane >> 1; l < ((nl + 15) & ~15); l += 16) {
      const bool act = l < nl;
      int o = 0, n = 0;
      if (act) {
        o = T.leaf_off[l0 + l];
        n = T.leaf_off[l0 + l + 1] - o;
      }
      const int64_t g = base + o;
      const int n8 = n - n % 8;
      const bool vec = act && !a.values && (g & 3) == 0 && n >= 8;
      double part = 0.0;
      if (vec) {
        const float4* p = reinterpret_cast<const float4*>(a.known + g) + h;
        float4 x = __ldg(p);
        double r0 = f(x.x), r1 = f(x.y), r2 = f(x.z), r3 = f(x.w);
#pragma unroll 4
        for (int q = 1; q < n8 / 8; ++q) {
          x = __ldg(p + 2 * q);
          r0 = __dadd_rn(r0, f(x.x)); r1 = __dadd_rn(r1, f(x.y));
          r2 = __dadd_rn(r2, f(x.z)); r3 = __dadd_rn(r3, f(x.w));
        }
        part = __dadd_rn(__dadd_rn(r0, r1), __dadd_rn(r2, r3));   // (r0+r1)+(r2+r3) / (r4+r5)+(r6+r7)
      }
      const double other = __shfl_down_sync(0xffffffffu, part, 1);
      if (act && h == 0) {
        double res;
        if (vec) {
          res = __dadd_rn(part, other);
          for (int i = n8; i < n; ++i) res = __dadd_rn(res, f(__ldg(a.known + g + i)));
        } else {
          res = np_leaf_sum<MODE>(a, g, n, mean);          // explicit samples / unaligned / n < 8
        }
        val[warp][l] = res;
      }
    }
  }
#else
  {
    double v = 0.0;
    if (lane < nl) {
      const int o = T.leaf_off[l0 + lane];
      v = np_leaf_sum<MODE>(a, a.part_base[s] + o, T.leaf_off[l0 + lane + 1] - o, mean);
    }
    val[warp][lane] = v;
  }
#endif
  __syncwarp();
  if (lane == 0) {
    const int ni = T.wr_nint[r];
    const int16_t* prog = T.wr_prog + (int64_t)r * 31;
    double* vv = val[warp];
    for (int j = 0; j < ni; ++j) {
      const int code = (uint16_t)prog[j];
      vv[32 + j] = __dadd_rn(vv[code & 0xff], vv[code >> 8]);
    }
    a.leaf[(int64_t)s * a.leaf_stride + r] = ni ? vv[32 + ni - 1] : vv[0];
  }
}

// internal nodes level by level; MODE 0 -> mean, MODE 1 -> svar
template <int MODE>
__global__ void __launch_bounds__(1024) npsum_tree_kernel(NpVarArgs a) {
  const int s = a.part0 + blockIdx.x;
  if (MODE == 0 && int_part(a, s)) {
    // exact sum of the part's chunk sums (any order), one warp
    if (threadIdx.x >= 32) return;
    const int64_t i0 = (int64_t)a.part_b[s] * a.nchunk, i1 = (int64_t)(a.part_e[s] + 1) * a.nchunk;
    double t = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += 32) t += a.stats[i].sum;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) a.mean[s] = __ddiv_rn(t, (double)a.part_m[s]);
    return;
  }
  const NpSumTree T = a.trees[a.part_class[s]];
  const double* leaf = a.leaf + (int64_t)s * a.leaf_stride;
  double* node = a.node + (int64_t)s * a.node_stride;
  for (int lev = 0; lev < T.nlevel; ++lev) {
    for (int j = T.level[lev] + threadIdx.x; j < T.level[lev + 1]; j += blockDim.x) {
      const int l = T.node_lr[2 * j], r = T.node_lr[2 * j + 1];
      const double vl = l < T.nleaf ? leaf[l] : node[l - T.nleaf];
      const double vr = r < T.nleaf ? leaf[r] : node[r - T.nleaf];
      node[j] = __dadd_rn(vl, vr);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double total = T.nnode ? node[T.nnode - 1] : leaf[0];
    const double q = __ddiv_rn(total, (double)a.part_m[s]);
    if (MODE == 0) a.mean[s] = q;
    else a.svar[s] = q;
  }
}

// ---- bins -------------------------------------------------------------------
// stable counting sort of a class's pairs by bin: order[boff[b] + rank] = k.
// Chunks of ORD_CHUNK consecutive pairs per CTA: pass 1 counts each chunk's
// bins, pass 2 offsets every chunk by boff (from the draw's bin counts) plus
// the earlier chunks' counts and ranks its pairs in order -- inside a warp
// with __match_any_sync, across the chunk's warps and rounds by running
// per-bin counters.
constexpr int ORD_CHUNK = 2048;

__global__ void __launch_bounds__(256) pair_order_count_kernel(const PairJob* jobs) {
  const PairJob& J = jobs[blockIdx.y];
  if (!J.t.order) return;
  const int64_t c0 = (int64_t)blockIdx.x * ORD_CHUNK;
  if (c0 >= J.npairs) return;
  __shared__ int cnt[MAX_BINS];
  if (threadIdx.x < MAX_BINS) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t c1 = min(J.npairs, c0 + ORD_CHUNK);
  for (int64_t k = c0 + threadIdx.x; k < c1; k += blockDim.x) {
    const int bb = J.t.bin[k];
    if (bb != 255) atomicAdd(&cnt[bb], 1);
  }
  __syncthreads();
  if (threadIdx.x < J.n_bins) J.t.ocnt[blockIdx.x * MAX_BINS + threadIdx.x] = cnt[threadIdx.x];
}

__global__ void __launch_bounds__(256) pair_order_kernel(const PairJob* jobs) {
  const PairJob& J = jobs[blockIdx.y];
  if (!J.t.order) return;
  const int64_t c0 = (int64_t)blockIdx.x * ORD_CHUNK;
  if (c0 >= J.npairs) return;
  __shared__ int base[MAX_BINS];
  __shared__ int wcnt[8][MAX_BINS + 1];
  const int nb = J.n_bins, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < nb) {
    int acc = 0;                                          // boff[tid] + earlier chunks
    for (int b = 0; b < tid; ++b) acc += (int)J.t.counts[b];
    for (int c = 0; c < (int)blockIdx.x; ++c) acc += J.t.ocnt[c * MAX_BINS + tid];
    base[tid] = acc;
    if (blockIdx.x == 0) {
      J.t.boff[tid] = acc;
      if (tid == nb - 1) J.t.boff[nb] = acc + (int)J.t.counts[tid];
    }
  }
  const int64_t c1 = min(J.npairs, c0 + ORD_CHUNK);
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t r0 = c0; r0 < c1; r0 += 256) {
    for (int t = tid; t < 8 * (MAX_BINS + 1); t += 256) (&wcnt[0][0])[t] = 0;
    __syncthreads();
    const int64_t k = r0 + tid;
    const int bb = k < c1 ? (int)J.t.bin[k] : 255;
    const unsigned same = __match_any_sync(0xffffffffu, bb);
    const int wrank = __popc(same & lt);
    if (bb != 255 && wrank == 0) wcnt[warp][bb] = __popc(same);
    __syncthreads();
    if (bb != 255) {
      int before = base[bb] + wrank;
      for (int w = 0; w < warp; ++w) before += wcnt[w][bb];
      J.t.order[before] = (int32_t)k;
    }
    __syncthreads();
    if (tid < nb) {
      int c = 0;
      for (int w = 0; w < 8; ++w) c += wcnt[w][tid];
      base[tid] += c;
    }
    __syncthreads();
  }
}

// 0.5 * (v_i - v_j)^2 of every pair at its bin-sorted slot
__global__ void __launch_bounds__(256) binsq_kernel(BinSumArgs a) {
  const int s = a.part0 + blockIdx.y;
  const PairTable t = a.tables[a.part_class[s]];
  const int nvalid = t.boff[a.n_bins];
  const int64_t base = a.part_base[s];
  double* out = a.sq + (int64_t)s * a.max_pairs;
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < nvalid; q += gridDim.x * blockDim.x) {
    const int k = t.order[q];
    const int64_t i = t.ii[k], j = t.jj[k];
    double vi, vj;
    if (a.values) { vi = a.values[base + i]; vj = a.values[base + j]; }
    else { vi = (double)__ldg(a.known + base + i); vj = (double)__ldg(a.known + base + j); }
    const double d = __dsub_rn(vi, vj);
    out[q] = __dmul_rn(0.5, __dmul_rn(d, d));
  }
}

// bin sums in pair order (np.bincount: out[b] += w in order): one CTA per
// (part, bin).  Integer-valued data first: all eight warps test and sum the
// bin's weights in any order (exact, see below); otherwise warp 0 streams the
// bin's slots in coalesced chunks of 256 into registers, parks them in shared
// memory, and lane 0 adds them in order while the next chunk's loads are in
// flight.
constexpr int BINSUM_THREADS = 256;

__global__ void __launch_bounds__(BINSUM_THREADS) binsum_kernel(BinSumArgs a) {
  const int s = a.part0 + blockIdx.y, b = blockIdx.x, lane = threadIdx.x & 31;
  const PairTable t = a.tables[a.part_class[s]];
  const int q0 = t.boff[b], q1 = t.boff[b + 1];
  const double* x = a.sq + (int64_t)s * a.max_pairs;
  // integer-valued data: every weight is a half-integer, and while the total
  // stays below 2^51 every partial sum in any order is exact -- the
  // CTA-parallel sum then equals the sequential one bit for bit
  {
    double ps = 0.0;
    bool ok = true;
    for (int c = q0 + (int)threadIdx.x; c < q1; c += 4 * BINSUM_THREADS) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = c + u * BINSUM_THREADS;
        v[u] = q < q1 ? x[q] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double t2 = 2.0 * v[u];
        ok &= (t2 == rint(t2));
        ps += v[u];
      }
    }
    ok = __syncthreads_and(ok);
    if (ok) {
      __shared__ double red[BINSUM_THREADS / 32];
      for (int o = 16; o > 0; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
      if (lane == 0) red[threadIdx.x >> 5] = ps;
      __syncthreads();
      if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int w = 0; w < BINSUM_THREADS / 32; ++w) tot += red[w];
        if (tot < 0x1p51) {
          a.bsum[(int64_t)s * a.n_bins + b] = tot;
          red[0] = -1.0;                              // done
        } else {
          red[0] = 0.0;
        }
      }
      __syncthreads();
      if (red[0] < 0.0) return;
    }
    if (threadIdx.x >= 32) return;                    // the ordered sum is one warp's
  }
  __shared__ double buf[2][256];
  double v[8];
  auto fetch = [&](int q) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = q + lane + 32 * u;
      v[u] = i < q1 ? x[i] : 0.0;
    }
  };
  auto park = [&](int slot) {
#pragma unroll
    for (int u = 0; u < 8; ++u) buf[slot][lane + 32 * u] = v[u];
  };
  double sum = 0.0;
  int cur = 0;
  if (q0 < q1) {
    fetch(q0);
    park(0);
  }
  __syncwarp();
  for (int q = q0; q < q1; q += 256) {
    const bool more = q + 256 < q1;
    if (more) fetch(q + 256);                 // in flight while lane 0 adds
    if (lane == 0) {
      const int n = min(256, q1 - q);
      const double* c = buf[cur];
      int k = 0;
      for (; k + 8 <= n; k += 8) {
        double w[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = c[k + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) sum = __dadd_rn(sum, w[u]);
      }
      for (; k < n; ++k) sum = __dadd_rn(sum, c[k]);
    }
    __syncwarp();
    if (more) park(cur ^ 1);
    __syncwarp();
    cur ^= 1;
  }
  if (lane == 0) a.bsum[(int64_t)s * a.n_bins + b] = sum;
}

}  // namespace

cudaError_t launch_npvar(const NpVarArgs& a, cudaStream_t st) {
  if (a.n_parts <= 0) return cudaSuccess;
  // a.max_leaf: most warp roots of a class in the launch
  const dim3 lgrid((unsigned)((a.max_leaf + NPW_WARPS - 1) / NPW_WARPS), (unsigned)a.n_parts);
  npsum_warp_kernel<0><<<lgrid, 32 * NPW_WARPS, 0, st>>>(a);
  npsum_tree_kernel<0><<<a.n_parts, 1024, 0, st>>>(a);
  npsum_warp_kernel<1><<<lgrid, 32 * NPW_WARPS, 0, st>>>(a);
  npsum_tree_kernel<1><<<a.n_parts, 1024, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pair_order(const PairJob* d_jobs, const PairJob* h_jobs, int n_jobs, cudaStream_t st) {
  bool any = false;
  int64_t mp = 1;
  for (int c = 0; c < n_jobs; ++c) {
    any |= h_jobs[c].t.order != nullptr;
    mp = std::max(mp, h_jobs[c].npairs);
  }
  if (!any) return cudaSuccess;
  const dim3 grid((unsigned)((mp + ORD_CHUNK - 1) / ORD_CHUNK), (unsigned)n_jobs);
  pair_order_count_kernel<<<grid, 256, 0, st>>>(d_jobs);
  pair_order_kernel<<<grid, 256, 0, st>>>(d_jobs);
  return cudaGetLastError();
}

cudaError_t launch_binsums(const BinSumArgs& a, cudaStream_t st) {
  if (a.n_parts <= 0) return cudaSuccess;
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(64, (a.max_pairs + 1023) / 1024));
  binsq_kernel<<<dim3(gx, a.n_parts), 256, 0, st>>>(a);
  binsum_kernel<<<dim3(a.n_bins, a.n_parts), BINSUM_THREADS, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace vk
