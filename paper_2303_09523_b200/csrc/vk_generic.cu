// Generic per-voxel fill for masks that are not whole known / missing planes
// (the reference's fallback, kriging.py:408-431 with _gather_window
// kriging.py:345-357, the window schedule kriging.py:37-40 and the weight
// cache kriging.py:364-381).
//
//   1. missing voxels are compacted (atomic append; order is irrelevant to
//      the values, and the first failing voxel is tracked by atomicMin over
//      raster indices, as the reference raises on the first one it meets);
//   2. one thread per missing voxel walks the schedule (4,4) (4,8) (4,16)
//      (8,16) (16,16): the first window whose known voxels bracket z, or at
//      z extent 16 the first window with any known voxel; it hashes the
//      window's known pattern (bounds relative to the target + occupancy
//      bits in np.nonzero (z, y, x) order) to 128 bits;
//   3. the host deduplicates the hashes (the reference's cache key is the
//      relative-offset list, which the pattern determines exactly); every
//      voxel's pattern is then compared word by word with its
//      representative's on the device, so a hash collision fails loudly;
//   4. one CTA per distinct pattern assembles [[C, Q], [Q^T, 0]] in global
//      scratch (drift columns dropped by the reference's numerical rank
//      test, kriging.py:145-156), LU with partial pivoting, residual check
//      1e-8, one ridge retry, variance (kriging.py:200-245);
//   5. one thread per missing voxel computes w . values in fp64 over the
//      window's known voxels in the same order, clamps, writes f32 (+ var).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>
#include "vk_common.h"
#include "vk_kernels.h"

namespace vk {

namespace {

constexpr int GEN_NWIN = 5;
__constant__ int c_sched[GEN_NWIN][2] = {{4, 4}, {4, 8}, {4, 16}, {8, 16}, {16, 16}};
constexpr int GEN_MAX_N = 1024;            // neighbours per system on the device

struct Win {
  int x0, x1, y0, y1, z0, z1;
};

__device__ __forceinline__ int wlo(int c, int extent) { return max(0, c - (extent / 2 - 1)); }
__device__ __forceinline__ int whi(int c, int extent, int n) { return min(n, c + extent / 2 + 1); }

__device__ __forceinline__ Win window_of(int e, int x, int y, int z, int T, int H, int W) {
  const int ip = c_sched[e][0], ze = c_sched[e][1];
  return {wlo(x, ip), whi(x, ip, W), wlo(y, ip), whi(y, ip, H), wlo(z, ze), whi(z, ze, T)};
}

__device__ __forceinline__ uint64_t mix64(uint64_t h, uint64_t v, uint64_t k) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= k;
  return h ^ (h >> 31);
}

struct Sel {
  int32_t win;        // schedule index, -1: no neighbours
  int32_t n;          // known voxels in the window
  uint64_t h1, h2;
};

__global__ void compact_missing_kernel(const uint8_t* __restrict__ mask, int64_t N, int64_t* list,
                                       unsigned long long* count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    if (mask[i]) {
      const unsigned long long k = atomicAdd(count, 1ull);
      if (list) list[k] = i;                          // null list: count only
    }
}

__global__ void select_kernel(const uint8_t* __restrict__ mask, int T, int H, int W, const int64_t* miss,
                              int64_t n_miss, Sel* sel, unsigned long long* first_fail) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_miss) return;
  const int64_t v = miss[i], P = (int64_t)H * W;
  const int z = (int)(v / P), y = (int)((v % P) / W), x = (int)(v % W);
  Sel s{-1, 0, 0, 0};
  for (int e = 0; e < GEN_NWIN && s.win < 0; ++e) {
    const Win w = window_of(e, x, y, z, T, H, W);
    int cnt = 0;
    bool below = false, above = false;
    for (int zz = w.z0; zz < w.z1; ++zz)
      for (int yy = w.y0; yy < w.y1; ++yy) {
        const uint8_t* row = mask + (int64_t)zz * P + (int64_t)yy * W;
        for (int xx = w.x0; xx < w.x1; ++xx)
          if (!row[xx]) {
            ++cnt;
            below |= zz < z;
            above |= zz > z;
          }
      }
    if (cnt == 0) continue;
    if ((below && above) || c_sched[e][1] == 16) {
      s.win = e;
      s.n = cnt;
      // pattern hash: relative bounds + occupancy bits in (z, y, x) order
      uint64_t h1 = 0x243f6a8885a308d3ull, h2 = 0x13198a2e03707344ull;
      const uint64_t b = (uint64_t)(w.x0 - x + 64) | ((uint64_t)(w.x1 - x + 64) << 8) |
                         ((uint64_t)(w.y0 - y + 64) << 16) | ((uint64_t)(w.y1 - y + 64) << 24) |
                         ((uint64_t)(w.z0 - z + 64) << 32) | ((uint64_t)(w.z1 - z + 64) << 40) |
                         ((uint64_t)e << 48);
      h1 = mix64(h1, b, 0xff51afd7ed558ccdull);
      h2 = mix64(h2, b, 0xc4ceb9fe1a85ec53ull);
      uint64_t word = 0;
      int nb = 0;
      for (int zz = w.z0; zz < w.z1; ++zz)
        for (int yy = w.y0; yy < w.y1; ++yy) {
          const uint8_t* row = mask + (int64_t)zz * P + (int64_t)yy * W;
          for (int xx = w.x0; xx < w.x1; ++xx) {
            word |= (uint64_t)(row[xx] == 0) << nb;
            if (++nb == 64) {
              h1 = mix64(h1, word, 0xff51afd7ed558ccdull);
              h2 = mix64(h2, word, 0xc4ceb9fe1a85ec53ull);
              word = 0;
              nb = 0;
            }
          }
        }
      h1 = mix64(h1, word ^ ((uint64_t)nb << 56), 0xff51afd7ed558ccdull);
      h2 = mix64(h2, word ^ ((uint64_t)nb << 56), 0xc4ceb9fe1a85ec53ull);
      s.h1 = h1;
      s.h2 = h2;
    }
  }
  sel[i] = s;
  if (s.win < 0) atomicMin(first_fail, (unsigned long long)v);
}

// exact pattern check of every voxel against its representative
__global__ void verify_kernel(const uint8_t* __restrict__ mask, int T, int H, int W, const int64_t* miss,
                              int64_t n_miss, const Sel* sel, const int32_t* uid, const int64_t* rep,
                              int* mismatch) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_miss) return;
  const int64_t P = (int64_t)H * W;
  const int64_t v = miss[i], r = miss[rep[uid[i]]];
  const int z = (int)(v / P), y = (int)((v % P) / W), x = (int)(v % W);
  const int zr = (int)(r / P), yr = (int)((r % P) / W), xr = (int)(r % W);
  const int e = sel[i].win;
  const Win a = window_of(e, x, y, z, T, H, W), b = window_of(e, xr, yr, zr, T, H, W);
  if (e != sel[rep[uid[i]]].win || a.x0 - x != b.x0 - xr || a.x1 - x != b.x1 - xr || a.y0 - y != b.y0 - yr ||
      a.y1 - y != b.y1 - yr || a.z0 - z != b.z0 - zr || a.z1 - z != b.z1 - zr) {
    atomicExch(mismatch, 1);
    return;
  }
  for (int dz = 0; dz < a.z1 - a.z0; ++dz)
    for (int dy = 0; dy < a.y1 - a.y0; ++dy) {
      const uint8_t* ra = mask + (int64_t)(a.z0 + dz) * P + (int64_t)(a.y0 + dy) * W + a.x0;
      const uint8_t* rb = mask + (int64_t)(b.z0 + dz) * P + (int64_t)(b.y0 + dy) * W + b.x0;
      for (int dx = 0; dx < a.x1 - a.x0; ++dx)
        if ((ra[dx] == 0) != (rb[dx] == 0)) {
          atomicExch(mismatch, 1);
          return;
        }
    }
}

// relative offsets of a representative's window, np.nonzero order
__global__ void rel_kernel(const uint8_t* __restrict__ mask, int T, int H, int W, const int64_t* miss,
                           const Sel* sel, const int64_t* rep, const int64_t* rel_off, int u0, int nu,
                           int16_t* rel) {
  const int u = u0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= u0 + nu) return;
  const int64_t P = (int64_t)H * W, v = miss[rep[u]];
  const int z = (int)(v / P), y = (int)((v % P) / W), x = (int)(v % W);
  const Win w = window_of(sel[rep[u]].win, x, y, z, T, H, W);
  int16_t* out = rel + 3 * rel_off[u];
  int c = 0;
  for (int zz = w.z0; zz < w.z1; ++zz)
    for (int yy = w.y0; yy < w.y1; ++yy)
      for (int xx = w.x0; xx < w.x1; ++xx)
        if (!mask[(int64_t)zz * P + (int64_t)yy * W + xx]) {
          out[3 * c + 0] = (int16_t)(xx - x);
          out[3 * c + 1] = (int16_t)(yy - y);
          out[3 * c + 2] = (int16_t)(zz - z);
          ++c;
        }
}

__device__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < nw; ++k) t += red[k];
  return t;
}

struct SolveCtx {
  int kind, drift;
  Model m;
};

// One CTA per system.  Matrix in global scratch (N x N row-major), rhs /
// solution in shared memory.  Returns per-system status.
__global__ void __launch_bounds__(256) generic_solve_kernel(SolveCtx ctx, const int16_t* rel,
                                                            const int64_t* rel_off, const int32_t* n_of,
                                                            const int64_t* mat_off, int u0, double* scratch,
                                                            double* weights, double* var, int32_t* status) {
  const int u = u0 + blockIdx.x;
  const int n = n_of[u];
  const int16_t* r = rel + 3 * rel_off[u];
  double* A = scratch + mat_off[u] - mat_off[u0];
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double red[32];
  __shared__ double x[GEN_MAX_N + 4], bvec[GEN_MAX_N + 4];
  __shared__ int piv_s;
  __shared__ double pval_s;
  __shared__ int keep[4];
  // ---- drift columns, kept by the reference's rank test (kriging.py:145-156):
  // column j stays if its residual after projection on the kept columns
  // exceeds 1e-9 (||col|| + 1).  Gram-Schmidt on the (n x 4) integer design.
  const int ncols = ctx.drift == DRIFT_LINEAR ? 4 : 1;
  // modified Gram-Schmidt with block reductions; the orthonormal basis of
  // the kept columns lives in the (not yet assembled) scratch matrix
  double* Bw = A;                                   // [4][n] basis workspace
  int nk = 0;
  for (int j = 0; j < ncols; ++j) {
    // column j values for row i: 1, x, y, z
    for (int i = tid; i < n; i += nt) Bw[nk * n + i] = j == 0 ? 1.0 : (double)r[3 * i + (j - 1)];
    __syncthreads();
    double nrm0 = 0.0;
    for (int i = tid; i < n; i += nt) nrm0 += Bw[nk * n + i] * Bw[nk * n + i];
    nrm0 = sqrt(block_sum(nrm0, red));
    for (int k = 0; k < nk; ++k) {                   // project out kept (orthonormal) columns
      double d = 0.0;
      for (int i = tid; i < n; i += nt) d += Bw[k * n + i] * Bw[nk * n + i];
      d = block_sum(d, red);
      for (int i = tid; i < n; i += nt) Bw[nk * n + i] -= d * Bw[k * n + i];
      __syncthreads();
    }
    double rn = 0.0;
    for (int i = tid; i < n; i += nt) rn += Bw[nk * n + i] * Bw[nk * n + i];
    rn = sqrt(block_sum(rn, red));
    if (j == 0 || rn > 1e-9 * (nrm0 + 1.0)) {
      for (int i = tid; i < n; i += nt) Bw[nk * n + i] /= rn;
      if (tid == 0) keep[nk] = j;
      ++nk;
    }
    __syncthreads();
  }
  const int p = nk, N = n + p;
  const double c00 = covariance(ctx.kind, ctx.m, 0.0);
  auto qcol = [&](int i, int k) -> double {          // kept drift column k at row i
    const int j = keep[k];
    return j == 0 ? 1.0 : (double)r[3 * i + (j - 1)];
  };
  int st = PS_OK;
  for (int attempt = 0; attempt < 2; ++attempt) {
    // ---- assemble [[C + ridge I, Q], [Q^T, 0]] and rhs [c0, q0]
    double ridge = 0.0;
    if (attempt == 1) ridge = fmax(1e-10 * (c00 * n) / n, 1e-12);   // tr(C) = n C(0)
    for (int idx = tid; idx < N * N; idx += nt) {
      const int i = idx / N, j = idx - i * N;
      double a;
      if (i < n && j < n) {
        const double dx = r[3 * i] - r[3 * j], dy = r[3 * i + 1] - r[3 * j + 1], dz = r[3 * i + 2] - r[3 * j + 2];
        a = covariance(ctx.kind, ctx.m, sqrt(dx * dx + dy * dy + dz * dz)) + (i == j ? ridge : 0.0);
      } else if (i < n) {
        a = qcol(i, j - n);
      } else if (j < n) {
        a = qcol(j, i - n);
      } else {
        a = 0.0;
      }
      A[idx] = a;
    }
    for (int i = tid; i < N; i += nt) {
      if (i < n) {
        const double dx = r[3 * i], dy = r[3 * i + 1], dz = r[3 * i + 2];
        bvec[i] = covariance(ctx.kind, ctx.m, sqrt(dx * dx + dy * dy + dz * dz));
      } else {
        bvec[i] = keep[i - n] == 0 ? 1.0 : 0.0;      // q0 = drift at the target (origin)
      }
      x[i] = bvec[i];
    }
    __syncthreads();
    // ---- LU with partial pivoting (LAPACK getf2 order), applied to x
    bool singular = false;
    for (int k = 0; k < N; ++k) {
      // pivot: first index of the max |A[i][k]|, i >= k (idamax)
      double best = -1.0;
      int bi = k;
      for (int i = k + tid; i < N; i += nt) {
        const double a = fabs(A[(int64_t)i * N + k]);
        if (a > best) { best = a; bi = i; }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      __shared__ double wb[8];
      __shared__ int wi[8];
      if ((tid & 31) == 0) { wb[tid >> 5] = best; wi[tid >> 5] = bi; }
      __syncthreads();
      if (tid == 0) {
        double b0 = wb[0];
        int i0 = wi[0];
        for (int w = 1; w < (nt >> 5); ++w)
          if (wb[w] > b0 || (wb[w] == b0 && wi[w] < i0)) { b0 = wb[w]; i0 = wi[w]; }
        piv_s = i0;
        pval_s = A[(int64_t)i0 * N + k];
      }
      __syncthreads();
      const int pi = piv_s;
      const double pv = pval_s;
      if (pv == 0.0) { singular = true; break; }
      if (pi != k) {
        for (int j = tid; j < N; j += nt) {
          const double t = A[(int64_t)k * N + j];
          A[(int64_t)k * N + j] = A[(int64_t)pi * N + j];
          A[(int64_t)pi * N + j] = t;
        }
        if (tid == 0) { const double t = x[k]; x[k] = x[pi]; x[pi] = t; }
      }
      __syncthreads();
      const double rp = __drcp_rn(pv);                 // = 1.0 / pv, correctly rounded
      for (int i = k + 1 + tid; i < N; i += nt) A[(int64_t)i * N + k] *= rp;
      __syncthreads();
      const int rem = N - k - 1;
      for (int idx = tid; idx < rem * rem; idx += nt) {
        const int i = k + 1 + idx / rem, j = k + 1 + idx % rem;
        A[(int64_t)i * N + j] -= A[(int64_t)i * N + k] * A[(int64_t)k * N + j];
      }
      if (tid == 0) {
        const double xk = x[k];
        for (int i = k + 1; i < N; ++i) x[i] -= A[(int64_t)i * N + k] * xk;   // forward (L unit)
      }
      __syncthreads();
    }
    if (!singular) {
      if (tid == 0) {
        for (int i = N - 1; i >= 0; --i) {              // back substitution (U)
          double s = x[i];
          for (int j = i + 1; j < N; ++j) s -= A[(int64_t)i * N + j] * x[j];
          x[i] = s / A[(int64_t)i * N + i];
        }
      }
      __syncthreads();
    }
    // ---- unbiasedness residual Q^T w - q0 (kriging.py:219-229)
    bool bad = singular;
    if (!bad) {
      double worst = 0.0;
      bool finite = true;
      for (int k = 0; k < p; ++k) {
        double s = 0.0;
        for (int i = tid; i < n; i += nt) s += qcol(i, k) * x[i];
        s = block_sum(s, red);
        const double q0 = keep[k] == 0 ? 1.0 : 0.0;
        worst = fmax(worst, fabs(s - q0));
      }
      for (int i = 0; i < N; ++i) finite &= (x[i] - x[i] == 0.0);
      bad = !finite || worst > 1e-8;
    }
    if (!bad) {
      st = PS_OK;
      break;
    }
    st = PS_SINGULAR;
    __syncthreads();
  }
  if (tid == 0) status[u] = st;
  if (st != PS_OK) return;
  for (int i = tid; i < n; i += nt) weights[rel_off[u] + i] = x[i];
  // variance = C(0) - w . c0 - lambda . q0 (kriging.py:239-244)
  double s = 0.0;
  for (int i = tid; i < n; i += nt) s += x[i] * bvec[i];
  s = block_sum(s, red);
  if (tid == 0) {
    double lq = 0.0;
    for (int k = 0; k < p; ++k) lq += x[n + k] * bvec[n + k];
    var[u] = c00 - s - lq;
  }
}

__global__ void generic_predict_kernel(const float* __restrict__ data, const uint8_t* __restrict__ mask, int T,
                                       int H, int W, const int64_t* miss, int64_t n_miss, const Sel* sel,
                                       const int32_t* uid, const int64_t* rel_off, const double* weights,
                                       const double* svar, double lo, double hi, float* out, double* var) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_miss) return;
  const int64_t P = (int64_t)H * W, v = miss[i];
  const int z = (int)(v / P), y = (int)((v % P) / W), x = (int)(v % W);
  const Win w = window_of(sel[i].win, x, y, z, T, H, W);
  const double* wt = weights + rel_off[uid[i]];
  double acc = 0.0;
  int c = 0;
  for (int zz = w.z0; zz < w.z1; ++zz)
    for (int yy = w.y0; yy < w.y1; ++yy) {
      const int64_t rowb = (int64_t)zz * P + (int64_t)yy * W;
      for (int xx = w.x0; xx < w.x1; ++xx)
        if (!mask[rowb + xx]) acc = fma(wt[c++], (double)data[rowb + xx], acc);
    }
  acc = fmin(fmax(acc, lo), hi);
  out[v] = (float)acc;
  if (var) var[v] = svar[uid[i]];
}

__global__ void zero_known_var_kernel(const uint8_t* __restrict__ mask, int64_t N, double* var) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    if (!mask[i]) var[i] = 0.0;
}

template <typename T>
struct DevBuf {
  T* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  cudaError_t alloc(size_t n) { return cudaMalloc((void**)&p, std::max<size_t>(n, 1) * sizeof(T)); }
};

struct Key {
  uint64_t h1, h2;
  int32_t win, n;
  bool operator==(const Key& o) const { return h1 == o.h1 && h2 == o.h2 && win == o.win && n == o.n; }
};
struct KeyHash {
  size_t operator()(const Key& k) const { return (size_t)(k.h1 ^ (k.h2 * 0x9e3779b97f4a7c15ull) ^ k.n); }
};

}  // namespace

cudaError_t solve_systems_device(const int16_t* rel_dev, const std::vector<int64_t>& rel_off, int kind, int drift,
                                 const double* model, double* w_dev, double* var_dev, int32_t* status_dev,
                                 cudaStream_t st) {
  const int nu = (int)rel_off.size() - 1;
  if (nu <= 0) return cudaSuccess;
  std::vector<int32_t> n_of(nu);
  std::vector<int64_t> mat_off(nu + 1, 0);
  int64_t biggest = 0;
  for (int u = 0; u < nu; ++u) {
    n_of[u] = (int32_t)(rel_off[u + 1] - rel_off[u]);
    const int64_t NN = n_of[u] + 4;
    mat_off[u + 1] = mat_off[u] + NN * NN;
    biggest = std::max(biggest, NN * NN);
  }
  DevBuf<int32_t> d_n;
  DevBuf<int64_t> d_rel_off, d_mat_off;
  DevBuf<double> scratch;
  const int64_t max_scratch = (int64_t)256 << 20;   // doubles per batch (2 GB)
  cudaError_t e = d_n.alloc(nu);
  if (e == cudaSuccess) e = d_rel_off.alloc(nu + 1);
  if (e == cudaSuccess) e = d_mat_off.alloc(nu + 1);
  if (e == cudaSuccess) e = scratch.alloc((size_t)std::min(mat_off[nu], std::max(max_scratch, biggest)));
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_n.p, n_of.data(), nu * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_rel_off.p, rel_off.data(), (nu + 1) * 8, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_mat_off.p, mat_off.data(), (nu + 1) * 8, cudaMemcpyHostToDevice, st);
  SolveCtx ctx{kind, drift, Model{model[0], model[1], model[2]}};
  for (int u0 = 0; e == cudaSuccess && u0 < nu;) {
    int u1 = u0 + 1;
    while (u1 < nu && mat_off[u1 + 1] - mat_off[u0] <= max_scratch && u1 - u0 < 65535) ++u1;
    generic_solve_kernel<<<u1 - u0, 256, 0, st>>>(ctx, rel_dev, d_rel_off.p, d_n.p, d_mat_off.p, u0, scratch.p,
                                                  w_dev, var_dev, status_dev);
    e = cudaGetLastError();
    u0 = u1;
  }
  // the buffers above are freed when this returns: finish the work first
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e;
}

GenericResult fill_generic(const float* data, const uint8_t* mask, int T, int H, int W, const double* model,
                           int kind, int drift, double lo, double hi, float* out, double* var,
                           cudaStream_t st) {
  GenericResult res;
  const int64_t N = (int64_t)T * H * W;
  auto cuda_fail = [&](cudaError_t e, const char* what) {
    res.status = 7;
    res.msg = std::string(what) + ": " + cudaGetErrorString(e);
    return res;
  };
#define GEN_TRY(call)                                 \
  do {                                                \
    cudaError_t e_ = (call);                          \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)
  // known voxels pass through bit-exactly (kriging.py:481)
  GEN_TRY(cudaMemcpyAsync(out, data, N * sizeof(float), cudaMemcpyDeviceToDevice, st));
  if (var) zero_known_var_kernel<<<1024, 256, 0, st>>>(mask, N, var);
  DevBuf<unsigned long long> cnt;
  GEN_TRY(cnt.alloc(2));
  GEN_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
  const unsigned long long init_fail = ~0ull;
  GEN_TRY(cudaMemcpyAsync(cnt.p + 1, &init_fail, sizeof(init_fail), cudaMemcpyHostToDevice, st));
  // count, then compact, the missing voxels
  DevBuf<int64_t> miss;
  compact_missing_kernel<<<1024, 256, 0, st>>>(mask, N, nullptr, cnt.p);
  unsigned long long n_miss_u = 0;
  GEN_TRY(cudaMemcpyAsync(&n_miss_u, cnt.p, sizeof(n_miss_u), cudaMemcpyDeviceToHost, st));
  GEN_TRY(cudaStreamSynchronize(st));
  const int64_t n_miss = (int64_t)n_miss_u;
  if (n_miss == 0) return res;
  GEN_TRY(miss.alloc(n_miss));
  GEN_TRY(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long), st));
  compact_missing_kernel<<<1024, 256, 0, st>>>(mask, N, miss.p, cnt.p);
  DevBuf<Sel> sel;
  GEN_TRY(sel.alloc(n_miss));
  const unsigned nb = (unsigned)((n_miss + 127) / 128);
  select_kernel<<<nb, 128, 0, st>>>(mask, T, H, W, miss.p, n_miss, sel.p, cnt.p + 1);
  GEN_TRY(cudaGetLastError());
  std::vector<Sel> hs(n_miss);
  unsigned long long first_fail = 0;
  GEN_TRY(cudaMemcpyAsync(hs.data(), sel.p, n_miss * sizeof(Sel), cudaMemcpyDeviceToHost, st));
  GEN_TRY(cudaMemcpyAsync(&first_fail, cnt.p + 1, sizeof(first_fail), cudaMemcpyDeviceToHost, st));
  GEN_TRY(cudaStreamSynchronize(st));
  if (first_fail != ~0ull) {
    const int64_t P = (int64_t)H * W, v = (int64_t)first_fail;
    res.status = 2;
    res.failed = v;
    res.msg = "no known voxel near (" + std::to_string(v % W) + ", " + std::to_string((v % P) / W) + ", " +
              std::to_string(v / P) + ")";
    return res;
  }
  // ---- distinct patterns (host), representative = first occurrence
  std::unordered_map<Key, int32_t, KeyHash> ids;
  ids.reserve((size_t)std::min<int64_t>(n_miss, 1 << 20));
  std::vector<int32_t> uid(n_miss);
  std::vector<int64_t> rep;
  std::vector<int32_t> n_of;
  for (int64_t i = 0; i < n_miss; ++i) {
    const Key k{hs[i].h1, hs[i].h2, hs[i].win, hs[i].n};
    auto it = ids.find(k);
    if (it == ids.end()) {
      if (hs[i].n > GEN_MAX_N) {
        res.status = 6;
        res.msg = "generic path: a window with " + std::to_string(hs[i].n) +
                  " known voxels exceeds the device solver's " + std::to_string(GEN_MAX_N);
        return res;
      }
      it = ids.emplace(k, (int32_t)rep.size()).first;
      rep.push_back(i);
      n_of.push_back(hs[i].n);
    }
    uid[i] = it->second;
  }
  const int nu = (int)rep.size();
  std::vector<int64_t> rel_off(nu + 1, 0);
  for (int u = 0; u < nu; ++u) rel_off[u + 1] = rel_off[u] + n_of[u];
  DevBuf<int32_t> d_uid, d_status;
  DevBuf<int64_t> d_rep, d_rel_off;
  DevBuf<int16_t> d_rel;
  DevBuf<double> d_w, d_var;
  DevBuf<int> d_mis;
  GEN_TRY(d_uid.alloc(n_miss));
  GEN_TRY(d_status.alloc(nu));
  GEN_TRY(d_rep.alloc(nu));
  GEN_TRY(d_rel_off.alloc(nu + 1));
  GEN_TRY(d_rel.alloc(3 * rel_off[nu]));
  GEN_TRY(d_w.alloc(rel_off[nu]));
  GEN_TRY(d_var.alloc(nu));
  GEN_TRY(d_mis.alloc(1));
  GEN_TRY(cudaMemcpyAsync(d_uid.p, uid.data(), n_miss * 4, cudaMemcpyHostToDevice, st));
  GEN_TRY(cudaMemcpyAsync(d_rep.p, rep.data(), nu * 8, cudaMemcpyHostToDevice, st));
  GEN_TRY(cudaMemcpyAsync(d_rel_off.p, rel_off.data(), (nu + 1) * 8, cudaMemcpyHostToDevice, st));
  GEN_TRY(cudaMemsetAsync(d_mis.p, 0, sizeof(int), st));
  verify_kernel<<<nb, 128, 0, st>>>(mask, T, H, W, miss.p, n_miss, sel.p, d_uid.p, d_rep.p, d_mis.p);
  rel_kernel<<<(nu + 127) / 128, 128, 0, st>>>(mask, T, H, W, miss.p, sel.p, d_rep.p, d_rel_off.p, 0, nu,
                                              d_rel.p);
  GEN_TRY(cudaGetLastError());
  // ---- solve the distinct systems (batched, bounded scratch)
  {
    cudaError_t e = solve_systems_device(d_rel.p, rel_off, kind, drift, model, d_w.p, d_var.p, d_status.p, st);
    if (e != cudaSuccess) return cuda_fail(e, "solve_systems_device");
  }
  std::vector<int32_t> status(nu);
  int mismatch = 0;
  GEN_TRY(cudaMemcpyAsync(status.data(), d_status.p, nu * 4, cudaMemcpyDeviceToHost, st));
  GEN_TRY(cudaMemcpyAsync(&mismatch, d_mis.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  GEN_TRY(cudaStreamSynchronize(st));
  if (mismatch) {
    res.status = 7;
    res.msg = "generic path: pattern hash collision (fail loudly; please report)";
    return res;
  }
  for (int u = 0; u < nu; ++u)
    if (status[u] != PS_OK) {
      res.status = 3;
      res.msg = "extended kriging matrix is singular (generic window)";
      return res;
    }
  generic_predict_kernel<<<nb, 128, 0, st>>>(data, mask, T, H, W, miss.p, n_miss, sel.p, d_uid.p, d_rel_off.p,
                                             d_w.p, d_var.p, lo, hi, out, var);
  GEN_TRY(cudaGetLastError());
  GEN_TRY(cudaStreamSynchronize(st));
  res.n_systems = nu;
  res.n_missing = n_miss;
#undef GEN_TRY
  return res;
}

}  // namespace vk
