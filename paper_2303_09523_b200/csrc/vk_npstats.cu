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
//            (build_npsum_tree); the device sums every leaf in parallel
//            (eight lanes per leaf, numpy's combination order) and then adds
//            the internal nodes level by level in one CTA per part.  Two
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

// eight lanes per leaf (lane k holds numpy's accumulator r[k]), four leaves
// per warp
template <int MODE>
__global__ void __launch_bounds__(256) npsum_leaf_kernel(NpVarArgs a) {
  const int s = a.part0 + blockIdx.y;
  const NpSumTree T = a.trees[a.part_class[s]];
  const int leaf = (blockIdx.x * blockDim.x + threadIdx.x) >> 3;
  const int k = threadIdx.x & 7;
  const bool act = leaf < T.nleaf;
  const int64_t base = a.part_base[s];
  const double mean = MODE ? a.mean[s] : 0.0;
  double r = 0.0;
  int64_t o = 0, n = 0, n8 = 0;
  if (act) {
    o = T.leaf_off[leaf];
    n = T.leaf_off[leaf + 1] - o;
    n8 = n - n % 8;
    if (n >= 8) {
      r = npv<MODE>(a.known, a.values, base + o + k, mean);
#pragma unroll 4
      for (int64_t i = 8; i < n8; i += 8) r = __dadd_rn(r, npv<MODE>(a.known, a.values, base + o + i + k, mean));
    }
  }
  // res = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7))
  const unsigned full = 0xffffffffu;
  double t = __shfl_down_sync(full, r, 1);
  r = __dadd_rn(r, t);
  t = __shfl_down_sync(full, r, 2);
  r = __dadd_rn(r, t);
  t = __shfl_down_sync(full, r, 4);
  r = __dadd_rn(r, t);
  if (act && k == 0) {
    double res = r;
    if (n < 8) {                                    // whole array below 8 (not reached: m >= 9)
      res = -0.0;
      n8 = 0;
    }
    for (int64_t i = n8; i < n; ++i) res = __dadd_rn(res, npv<MODE>(a.known, a.values, base + o + i, mean));
    a.leaf[(int64_t)s * a.leaf_stride + leaf] = res;
  }
}

// internal nodes level by level; MODE 0 -> mean, MODE 1 -> svar
template <int MODE>
__global__ void __launch_bounds__(1024) npsum_tree_kernel(NpVarArgs a) {
  const int s = a.part0 + blockIdx.x;
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
// stable counting sort of a class's pairs by bin: order[boff[b] + rank] = k
__global__ void __launch_bounds__(1024) pair_order_kernel(const PairJob* jobs) {
  const PairJob& J = jobs[blockIdx.x];
  if (!J.t.order) return;
  extern __shared__ int cnt[];                      // [n_bins][1024]
  __shared__ int tot[MAX_BINS + 1];
  const int nb = J.n_bins, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t np_ = J.npairs;
  const int64_t per = (np_ + 1023) / 1024;
  const int64_t b0 = min(np_, (int64_t)tid * per), b1 = min(np_, b0 + per);
  for (int b = 0; b < nb; ++b) cnt[b * 1024 + tid] = 0;
  for (int64_t k = b0; k < b1; ++k) {
    const int bb = J.t.bin[k];
    if (bb != 255) cnt[bb * 1024 + tid] += 1;
  }
  __syncthreads();
  // per-bin exclusive scan over the 1024 threads: warp w scans bin w
  for (int b = warp; b < nb; b += 32) {
    int run = 0;
    for (int c = 0; c < 1024; c += 32) {
      const int v = cnt[b * 1024 + c + lane];
      int incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      cnt[b * 1024 + c + lane] = run + incl - v;
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) tot[b] = run;
  }
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int b = 0; b < nb; ++b) {
      J.t.boff[b] = acc;
      const int t = tot[b];
      tot[b] = acc;
      acc += t;
    }
    J.t.boff[nb] = acc;
  }
  __syncthreads();
  for (int64_t k = b0; k < b1; ++k) {
    const int bb = J.t.bin[k];
    if (bb == 255) continue;
    const int slot = tot[bb] + cnt[bb * 1024 + tid];
    cnt[bb * 1024 + tid] += 1;
    J.t.order[slot] = (int32_t)k;
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

// bin sums in pair order (np.bincount: out[b] += w in order): one warp per
// (part, bin).  The warp streams the bin's slots in coalesced chunks of 256
// into registers, parks them in shared memory, and lane 0 adds them in order
// while the next chunk's loads are in flight.
__global__ void __launch_bounds__(32) binsum_kernel(BinSumArgs a) {
  const int s = a.part0 + blockIdx.y, b = blockIdx.x, lane = threadIdx.x;
  const PairTable t = a.tables[a.part_class[s]];
  const int q0 = t.boff[b], q1 = t.boff[b + 1];
  const double* x = a.sq + (int64_t)s * a.max_pairs;
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
  const dim3 lgrid((unsigned)((a.max_leaf * 8 + 255) / 256), (unsigned)a.n_parts);
  npsum_leaf_kernel<0><<<lgrid, 256, 0, st>>>(a);
  npsum_tree_kernel<0><<<a.n_parts, 1024, 0, st>>>(a);
  npsum_leaf_kernel<1><<<lgrid, 256, 0, st>>>(a);
  npsum_tree_kernel<1><<<a.n_parts, 1024, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_pair_order(const PairJob* d_jobs, const PairJob* h_jobs, int n_jobs, cudaStream_t st) {
  int nb = 1;
  bool any = false;
  for (int c = 0; c < n_jobs; ++c) {
    nb = std::max(nb, h_jobs[c].n_bins);
    any |= h_jobs[c].t.order != nullptr;
  }
  if (!any) return cudaSuccess;
  const size_t smem = (size_t)nb * 1024 * sizeof(int);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(pair_order_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  pair_order_kernel<<<n_jobs, 1024, smem, st>>>(d_jobs);
  return cudaGetLastError();
}

cudaError_t launch_binsums(const BinSumArgs& a, cudaStream_t st) {
  if (a.n_parts <= 0) return cudaSuccess;
  const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(64, (a.max_pairs + 1023) / 1024));
  binsq_kernel<<<dim3(gx, a.n_parts), 256, 0, st>>>(a);
  binsum_kernel<<<dim3(a.n_bins, a.n_parts), 32, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace vk
