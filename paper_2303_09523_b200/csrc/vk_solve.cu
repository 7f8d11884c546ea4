// Batched universal-kriging stencil solves: one warp per (sub-part, stencil).
//
// Restates build_system + solve_ked (kriging.py:159-245) for the stencil
// families of the plane-structured fill (kriging.py:516-557): the extended
// matrix [[C, Q], [Q^T, 0]] on target-relative integer offsets is assembled
// in shared memory in fp64, factorised by LU with partial pivoting (the
// algorithm of LAPACK dgesv behind np.linalg.solve), checked for finiteness
// and the unbiasedness residual (<= 1e-8), retried once with the ridge
// max(1e-10 tr(C)/n, 1e-12) on the covariance block, and the kriging
// variance C(0) - w.c0 - lambda.q0 is formed.  Weights are written into the
// zero-padded [plane][oy+1][ox+1] layout the prediction kernels read.
// Drift columns kept by _independent_columns (kriging.py:145-156) are decided
// exactly on the host (integer offsets) and passed as a bitmask.
#include <cuda_runtime.h>
#include <algorithm>
#include "vk_kernels.h"

namespace vk {

namespace {

constexpr int SOLVE_WARPS_MAX = 4;

// One warp per system; `ws` systems per CTA, each with its own shared-memory
// slice [A | b] (N x (N+1)), solution and relative offsets.
// UPD_SLOTS: 8-column slots of the LU update (ld <= 8 UPD_SLOTS); YS: 32-row
// slots of the back substitution (N <= 32 YS)
template <int UPD_SLOTS, int YS>
__global__ void __launch_bounds__(32 * SOLVE_WARPS_MAX) solve_kernel(SolveArgs a, int ws, size_t slice) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int sys = a.sys0 + blockIdx.x * ws + wid;
  if (wid >= ws || sys >= a.sys0 + a.n_sys) return;
  if (a.der_src && a.der_src[sys] >= 0) return;   // filled by derive_kernel
  const int s = a.sys_part[sys], stc = a.sys_stencil[sys];
  const int n = a.st_n[stc], off = a.st_off[stc], dcols = a.st_drift[stc];
  const int pat = a.st_pattern[stc];
  const int kind_idx = stc % a.NK;
  Model mdl;
  mdl.nugget = a.models[3 * s + 0];
  mdl.sill = a.models[3 * s + 1];
  mdl.range_len = a.models[3 * s + 2];
  int cols[4], pq = 0;
  for (int c = 0; c < 4; ++c)
    if (dcols & (1 << c)) cols[pq++] = c;
  const int N = n + pq, ld = (N + 1) | 1;     // odd: row-strided lane accesses are bank-conflict free
  double* A = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + (size_t)wid * slice);
  double* xsol = A + (size_t)N * ld;
  double* rinv = xsol + N;
  int* rel = reinterpret_cast<int*>(rinv + N);
  for (int i = lane; i < n; i += 32) {
    const int pl = a.taps[3 * (off + i) + 2];
    rel[3 * i + 0] = a.taps[3 * (off + i) + 0];
    rel[3 * i + 1] = a.taps[3 * (off + i) + 1];
    rel[3 * i + 2] = a.pat_dz[pat * NPMAX + pl];
  }
  // covariance by integer squared lag: every lag in the system is
  // sqrt(dx^2 + dy^2 + dz^2) of small integers, so the distinct values are
  // tabulated once (kriging.py:185-188 evaluates C element by element)
  int maxdz = 0;
  for (int p1 = 0; p1 < NPMAX; ++p1) {
    const int z1 = a.pat_dz[pat * NPMAX + p1];
    maxdz = max(maxdz, abs(z1));
    for (int p2 = 0; p2 < NPMAX; ++p2) maxdz = max(maxdz, abs(z1 - a.pat_dz[pat * NPMAX + p2]));
  }
  const int maxd2 = 18 + maxdz * maxdz;
  double* ctab = reinterpret_cast<double*>(reinterpret_cast<char*>(rel) +
                                           ((3 * a.max_n * sizeof(int) + 7) & ~(size_t)7));   // [maxd2 + 1]
  for (int d2 = lane; d2 <= maxd2; d2 += 32) ctab[d2] = covariance(a.kind, mdl, sqrt((double)d2));
  __syncwarp();
  const double cov0 = ctab[0];
  double trace = 0.0;
  for (int i = 0; i < n; ++i) trace += cov0;     // np.trace of C
  const double ridge = fmax(1e-10 * trace / n, 1e-12);
  bool done = false;
  for (int attempt = 0; attempt < 2 && !done; ++attempt) {
    // ---- assemble [A | b]: rows of [C Q | c0] then [Q^T 0 | q0]
    for (int i = 0; i < n; ++i) {
      const int xi = rel[3 * i], yi = rel[3 * i + 1], zi = rel[3 * i + 2];
      for (int j = lane; j < ld; j += 32) {
        double v;
        if (j < n) {
          const int dx = xi - rel[3 * j], dy = yi - rel[3 * j + 1], dz = zi - rel[3 * j + 2];
          v = ctab[dx * dx + dy * dy + dz * dz];
          if (attempt == 1 && i == j) v += ridge;
        } else if (j < N) {
          const int c = cols[j - n];
          v = (c == 0) ? 1.0 : (double)rel[3 * i + c - 1];
        } else {
          v = ctab[xi * xi + yi * yi + zi * zi];   // c0
        }
        A[i * ld + j] = v;
      }
    }
    for (int i = n; i < N; ++i) {
      const int c = cols[i - n];
      for (int j = lane; j < ld; j += 32) {
        double v;
        if (j < n) v = (c == 0) ? 1.0 : (double)rel[3 * j + c - 1];
        else if (j < N) v = 0.0;
        else v = (c == 0) ? 1.0 : 0.0;             // q0 = drift at the target
        A[i * ld + j] = v;
      }
    }
    __syncwarp();
    // ---- LU with partial pivoting (first maximal |pivot|, as idamax), rhs
    // carried as column N
    bool fail = false;
    for (int k = 0; k < N; ++k) {
      double best = -1.0;
      int bi = N;
      for (int r = k + lane; r < N; r += 32) {
        const double v = fabs(A[r * ld + k]);
        if (v > best) { best = v; bi = r; }        // NaN never wins, as in idamax
      }
      // first maximal |pivot| across lanes with integer warp reductions on
      // the bit pattern of the non-negative double (order preserving), then
      // the smallest row among the lanes holding the maximum
      {
        const unsigned long long key = best > 0.0 ? (unsigned long long)__double_as_longlong(best) : 0ull;
        const unsigned hi = (unsigned)(key >> 32), lo = (unsigned)key;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, hi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, hi == mhi ? lo : 0u);
        const bool win = hi == mhi && lo == mlo;
        bi = (int)__reduce_min_sync(0xffffffffu, win ? (unsigned)bi : 0xffffffffu);
        best = __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
      }
      if (!(best > 0.0)) { fail = true; break; }   // exact zero pivot: dgesv info > 0
      if (bi != k) {
        for (int j = lane; j < ld; j += 32) {
          const double t = A[k * ld + j];
          A[k * ld + j] = A[bi * ld + j];
          A[bi * ld + j] = t;
        }
        __syncwarp();
      }
      // column scale and rank-1 update, lanes over rows: each lane keeps its
      // row's multiplier in a register and streams the pivot row (broadcast
      // loads) in batches of 8 columns, loads before stores (dgetf2's
      // arithmetic: l = a_rk * (1 / a_kk), a_rj -= l * a_kj)
      const double inv = __drcp_rn(A[k * ld + k]);   // = 1.0 / a_kk (both correctly rounded), no division call
      const double* Ak = A + (size_t)k * ld;
      for (int r = k + 1 + lane; r < N; r += 32) {
        double* Ar = A + (size_t)r * ld;
        const double l = Ar[k] * inv;
        Ar[k] = l;
        int j = k + 1;
        for (; j + 8 <= ld; j += 8) {
          double u[8], v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) u[t] = Ak[j + t];
#pragma unroll
          for (int t = 0; t < 8; ++t) v[t] = Ar[j + t];
#pragma unroll
          for (int t = 0; t < 8; ++t) Ar[j + t] = fma(-l, u[t], v[t]);
        }
        if (j < ld) {                                 // tail: one predicated batch
          double u[8], v[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) u[t] = j + t < ld ? Ak[j + t] : 0.0;
#pragma unroll
          for (int t = 0; t < 8; ++t) v[t] = j + t < ld ? Ar[j + t] : 0.0;
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (j + t < ld) Ar[j + t] = fma(-l, u[t], v[t]);
        }
      }
      __syncwarp();
    }
    if (!fail) {
      // back substitution U x = y, column oriented as dtrsm (Left, Upper,
      // NoTrans): x_i = y_i / u_ii, then y_r -= x_i u_ri for r < i.  y lives
      // in registers (lane r holds rows r and r + 32); the reciprocals of the
      // diagonal are formed off the dependent chain, which is then one
      // multiply, one shuffle and one FMA per row
      bool finite = true;
      for (int r = lane; r < N; r += 32) rinv[r] = __drcp_rn(A[(size_t)r * ld + r]);
      double y[YS];
#pragma unroll
      for (int t = 0; t < YS; ++t) {
        const int r = lane + 32 * t;
        y[t] = r < N ? A[(size_t)r * ld + N] : 0.0;
      }
      __syncwarp();
      for (int i = N - 1; i >= 0; --i) {
        const int ti = i >> 5;
        double src = y[0];
#pragma unroll
        for (int t = 1; t < YS; ++t) src = ti == t ? y[t] : src;
        const double xi = __shfl_sync(0xffffffffu, src, i & 31) * rinv[i];
        finite = finite && (xi - xi == 0.0);
#pragma unroll
        for (int t = 0; t < YS; ++t) {
          const int r = lane + 32 * t;
          if (r < i) y[t] = fma(-xi, A[(size_t)r * ld + i], y[t]);
          else if (r == i) y[t] = xi;
        }
      }
#pragma unroll
      for (int t = 0; t < YS; ++t)
        if (lane + 32 * t < N) xsol[lane + 32 * t] = y[t];
      __syncwarp();
      // unbiasedness residual max_c |sum_i Q_ic w_i - q0_c|  (kriging.py:223)
      double resid = 0.0;
      for (int c = 0; c < pq; ++c) {
        double part = 0.0;
        for (int i = lane; i < n; i += 32) {
          const double q = (cols[c] == 0) ? 1.0 : (double)rel[3 * i + cols[c] - 1];
          part += q * xsol[i];
        }
        for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        resid = fmax(resid, fabs(part - ((cols[c] == 0) ? 1.0 : 0.0)));
      }
      done = finite && (resid <= 1e-8);
    }
  }
  // ---- outputs
  const int64_t slot = ((int64_t)s * a.NP + pat) * a.NK + kind_idx;
  double* w = a.weights + slot * WPAD;
  for (int i = lane; i < WPAD; i += 32) w[i] = 0.0;
  __syncwarp();
  if (done) {
    for (int i = lane; i < n; i += 32) w[a.pad[off + i]] = xsol[i];
    // variance = C(0) - w.c0 - lambda.q0  (kriging.py:239-244)
    double part = 0.0;
    for (int i = lane; i < n; i += 32) {
      const int dx = rel[3 * i], dy = rel[3 * i + 1], dz = rel[3 * i + 2];
      part += xsol[i] * ctab[dx * dx + dy * dy + dz * dz];
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) {
      double lq = 0.0;
      for (int c = 0; c < pq; ++c) lq += xsol[n + c] * ((cols[c] == 0) ? 1.0 : 0.0);
      a.var[slot] = cov0 - part - lq;
    }
  } else if (lane == 0) {
    a.var[slot] = 0.0;
  }
  if (lane == 0) a.sys_status[sys] = done ? PS_OK : PS_SINGULAR;
}

// Derived systems: weights of the source system with the planes reversed
// (z-mirror) and / or the in-plane taps transposed (x<->y), variance and
// status copied.  One thread per (system, padded weight slot).
__global__ void __launch_bounds__(256) derive_kernel(SolveArgs a) {
  const int64_t total = (int64_t)a.n_sys * WPAD;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int sys = a.sys0 + (int)(i / WPAD), e = (int)(i % WPAD);
    const int src = a.der_src[sys];
    if (src < 0) continue;
    const int fl = a.der_flags[sys], np = fl >> 8;
    const int64_t dslot = (int64_t)a.sys_part[sys] * a.NP * a.NK + a.sys_stencil[sys];
    const int64_t sslot = (int64_t)a.sys_part[src] * a.NP * a.NK + a.sys_stencil[src];
    const int pl = e >> 4, t = e & 15;
    const int spl = (fl & 1) ? np - 1 - pl : pl;
    const int stp = (fl & 2) ? (t & 3) * 4 + (t >> 2) : t;
    a.weights[dslot * WPAD + e] = pl < np ? a.weights[sslot * WPAD + spl * 16 + stp] : 0.0;
    if (e == 0) {
      a.var[dslot] = a.var[sslot];
      a.sys_status[sys] = a.sys_status[src];
    }
  }
}

}  // namespace

cudaError_t launch_derive(const SolveArgs& a, cudaStream_t st) {
  if (a.n_sys <= 0 || !a.der_src) return cudaSuccess;
  const int64_t total = (int64_t)a.n_sys * WPAD;
  derive_kernel<<<(unsigned)std::min<int64_t>(1024, (total + 255) / 256), 256, 0, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_solve(const SolveArgs& a, cudaStream_t st) {
  if (a.n_sys == 0) return cudaSuccess;
  const int N = a.max_n + 4;
  const int maxd2 = 18 + a.max_dz * a.max_dz;
  const size_t slice = (((size_t)N * (N + 2) + 2 * N) * sizeof(double) + (size_t)a.max_n * 3 * sizeof(int) +
                        (size_t)(maxd2 + 3) * sizeof(double) + 127) / 128 * 128;
  int ws = (int)std::max<size_t>(1, std::min<size_t>(SOLVE_WARPS_MAX, (size_t)(96 * 1024) / slice));
  const size_t smem = slice * ws;
  // plane stencils of the streaming path (2 planes x 16 taps + drift) take
  // the small instance; windows of up to NPMAX planes the general one
  const bool small = N + 2 <= 48 && N <= 64;
  const void* fn = small ? (const void*)solve_kernel<6, 2> : (const void*)solve_kernel<(NPMAX * 16 + 4 + 2 + 7) / 8, (NPMAX * 16 + 4 + 31) / 32>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (small)
    solve_kernel<6, 2><<<(a.n_sys + ws - 1) / ws, 32 * ws, smem, st>>>(a, ws, slice);
  else
    solve_kernel<(NPMAX * 16 + 4 + 2 + 7) / 8, (NPMAX * 16 + 4 + 31) / 32><<<(a.n_sys + ws - 1) / ws, 32 * ws, smem, st>>>(a, ws, slice);
  return cudaGetLastError();
}

}  // namespace vk
