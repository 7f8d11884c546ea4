// Batched universal-kriging stencil solves: one CTA per (sub-part, stencil).
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
#include "vk_kernels.h"

namespace vk {

namespace {

constexpr int SOLVE_THREADS = 128;

__global__ void __launch_bounds__(SOLVE_THREADS) solve_kernel(SolveArgs a) {
  extern __shared__ double sm[];
  const int sys = blockIdx.x, tid = threadIdx.x;
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
  const int N = n + pq, ld = N + 1;
  double* A = sm;                                  // [N][ld]
  double* xsol = sm + (size_t)N * ld;              // [N]
  int* rel = (int*)(xsol + N);                     // [n][3]
  __shared__ int s_piv, s_fail, s_done;
  __shared__ double s_red[SOLVE_THREADS / 32];
  __shared__ int s_redi[SOLVE_THREADS / 32];
  for (int i = tid; i < n; i += SOLVE_THREADS) {
    const int pl = a.taps[3 * (off + i) + 2];
    rel[3 * i + 0] = a.taps[3 * (off + i) + 0];
    rel[3 * i + 1] = a.taps[3 * (off + i) + 1];
    rel[3 * i + 2] = a.pat_dz[pat * NPMAX + pl];
  }
  if (tid == 0) { s_fail = 0; s_done = 0; }
  __syncthreads();
  const double cov0 = covariance(a.kind, mdl, 0.0);
  double trace = 0.0;
  for (int i = 0; i < n; ++i) trace += cov0;     // np.trace of C: sum of C(0)
  const double ridge = fmax(1e-10 * trace / n, 1e-12);

  int status = PS_SINGULAR;
  for (int attempt = 0; attempt < 2 && !s_done; ++attempt) {
    // ---- assemble [A | b]
    for (int idx = tid; idx < N * ld; idx += SOLVE_THREADS) {
      const int i = idx / ld, j = idx - i * ld;
      double v;
      if (j == N) {                                // rhs
        if (i < n) {
          const int dx = rel[3 * i], dy = rel[3 * i + 1], dz = rel[3 * i + 2];
          v = covariance(a.kind, mdl, sqrt((double)(dx * dx + dy * dy + dz * dz)));
        } else {
          v = (cols[i - n] == 0) ? 1.0 : 0.0;      // q0 = drift at the target
        }
      } else if (i < n && j < n) {
        const int dx = rel[3 * i] - rel[3 * j], dy = rel[3 * i + 1] - rel[3 * j + 1],
                  dz = rel[3 * i + 2] - rel[3 * j + 2];
        v = covariance(a.kind, mdl, sqrt((double)(dx * dx + dy * dy + dz * dz)));
        if (attempt == 1 && i == j) v += ridge;
      } else if (i < n) {
        const int c = cols[j - n];
        v = (c == 0) ? 1.0 : (double)rel[3 * i + c - 1];
      } else if (j < n) {
        const int c = cols[i - n];
        v = (c == 0) ? 1.0 : (double)rel[3 * j + c - 1];
      } else {
        v = 0.0;
      }
      A[i * ld + j] = v;
    }
    if (tid == 0) s_fail = 0;
    __syncthreads();
    // ---- LU with partial pivoting, rhs carried as column N
    for (int k = 0; k < N; ++k) {
      if (tid < 32) {
        double best = -1.0;
        int bi = N;
        for (int r = k + tid; r < N; r += 32) {
          const double v = fabs(A[r * ld + k]);
          if (v > best) { best = v; bi = r; }
        }
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_down_sync(0xffffffffu, best, o);
          const int oi = __shfl_down_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (tid == 0) {
          s_piv = bi;
          if (!(best > 0.0)) s_fail = 1;           // exact zero pivot: dgesv info > 0
        }
      }
      __syncthreads();
      if (s_fail) break;
      const int piv = s_piv;
      if (piv != k)
        for (int j = tid; j < ld; j += SOLVE_THREADS) {
          const double t = A[k * ld + j];
          A[k * ld + j] = A[piv * ld + j];
          A[piv * ld + j] = t;
        }
      __syncthreads();
      const double inv = 1.0 / A[k * ld + k];
      for (int r = k + 1 + tid; r < N; r += SOLVE_THREADS) A[r * ld + k] *= inv;
      __syncthreads();
      const int rows = N - k - 1, colsn = ld - k - 1;
      for (int idx = tid; idx < rows * colsn; idx += SOLVE_THREADS) {
        const int r = k + 1 + idx / colsn, j = k + 1 + idx % colsn;
        A[r * ld + j] -= A[r * ld + k] * A[k * ld + j];
      }
      __syncthreads();
    }
    if (tid == 0 && !s_fail) {
      // back substitution U x = y
      bool finite = true;
      for (int i = N - 1; i >= 0; --i) {
        double acc = A[i * ld + N];
        for (int j = i + 1; j < N; ++j) acc -= A[i * ld + j] * xsol[j];
        xsol[i] = acc / A[i * ld + i];
        finite = finite && (xsol[i] - xsol[i] == 0.0);
      }
      // unbiasedness residual max_c |sum_i Q_ic w_i - q0_c|
      double resid = 0.0;
      for (int c = 0; c < pq; ++c) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) {
          const double q = (cols[c] == 0) ? 1.0 : (double)rel[3 * i + cols[c] - 1];
          acc += q * xsol[i];
        }
        resid = fmax(resid, fabs(acc - ((cols[c] == 0) ? 1.0 : 0.0)));
      }
      if (!finite || !(resid <= 1e-8)) s_fail = 1;
      else s_done = 1;
    }
    __syncthreads();
  }
  if (s_done) status = PS_OK;
  // ---- outputs
  const int64_t slot = ((int64_t)s * a.NP + pat) * a.NK + kind_idx;
  double* w = a.weights + slot * WPAD;
  for (int i = tid; i < WPAD; i += SOLVE_THREADS) w[i] = 0.0;
  __syncthreads();
  if (status == PS_OK) {
    for (int i = tid; i < n; i += SOLVE_THREADS) w[a.pad[off + i]] = xsol[i];
    // variance = C(0) - w.c0 - lambda.q0  (kriging.py:239-244)
    double part = 0.0;
    for (int i = tid; i < n; i += SOLVE_THREADS) {
      const int dx = rel[3 * i], dy = rel[3 * i + 1], dz = rel[3 * i + 2];
      part += xsol[i] * covariance(a.kind, mdl, sqrt((double)(dx * dx + dy * dy + dz * dz)));
    }
    for (int o = 16; o > 0; o >>= 1) part += __shfl_down_sync(0xffffffffu, part, o);
    if ((tid & 31) == 0) s_red[tid >> 5] = part;
    __syncthreads();
    if (tid == 0) {
      double wc = 0.0;
      for (int i = 0; i < SOLVE_THREADS / 32; ++i) wc += s_red[i];
      double lq = 0.0;
      for (int c = 0; c < pq; ++c) lq += xsol[n + c] * ((cols[c] == 0) ? 1.0 : 0.0);
      a.var[slot] = cov0 - wc - lq;
    }
  } else if (tid == 0) {
    a.var[slot] = 0.0;
  }
  if (tid == 0) a.sys_status[sys] = status;
  (void)s_redi;
}

}  // namespace

cudaError_t launch_solve(const SolveArgs& a, cudaStream_t st) {
  if (a.n_sys == 0) return cudaSuccess;
  const int N = a.max_n + 4;
  const size_t smem = (size_t)N * (N + 1) * sizeof(double) + N * sizeof(double) +
                      (size_t)a.max_n * 3 * sizeof(int) + 16;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
  }
  solve_kernel<<<a.n_sys, SOLVE_THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace vk
