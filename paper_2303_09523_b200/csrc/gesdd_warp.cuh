// Warp-cooperative form of gesdd.h's svd_m3 for the device fit (one warp per
// sub-part).  Same operations in the same order -- every value is
// bit-identical to svd_m3 -- but the M-row work is spread over the lanes:
//   * dnrm2: the squares on all lanes, the four x87 accumulator chains on
//     lanes 0-3 (lane 0 also takes the n % 8 tail), the combination and the
//     fsqrt emulation redundantly on every lane;
//   * dlarfg's dscal and dlarf's dger: one element per lane;
//   * dlarf's dgemv_t: one kernel accumulator chain per lane (two per column
//     in dgemv_kernel_4x2, four in dgemv_kernel_4x1), combined in the
//     kernel's order on every lane;
//   * dorg2r likewise; dgemm(Q, U_B): one output element per lane.
// The 3 x 3 stages (dgebd2, dbdsqr, the two dormbr) are a few hundred scalar
// operations and run redundantly on every lane from registers.
// The matrix lives in shared memory; only designated lanes write, and every
// phase ends with __syncwarp().
#pragma once
#include "gesdd.h"
#include "trf.h"

namespace vk {
namespace lapack {

// svd_m3_2w: the 3 x 3 stages' results, from warp 1 to both warps
struct SvdXchg {
  double d[3], Ub[9], VTb[9];
  int info;
};

struct SvdWarpSmem {
  double A[GMAXM * 3];        // column-major, lda = M
  double U[GMAXM * 3];        // row-major result
  uint64_t em[GMAXM];         // dnrm2 squares (extended significand, exponent)
  int ee[GMAXM];
};

__device__ __forceinline__ Ext shfl_ext(Ext v, int src) {
  Ext r;
  r.m = (uint64_t)__shfl_sync(0xffffffffu, (long long)v.m, src);
  r.e = __shfl_sync(0xffffffffu, v.e, src);
  return r;
}

// Fast form of the x87 dnrm2 below (see dnrm2_decide): the exact sum of
// squares as a double-double over a warp tree; about 1 % of the calls fall
// back to the exact emulation.  Lanes may associate the tree differently, so
// the fallback is taken warp-uniformly (__any_sync); a lane's fast result,
// when taken, is provably the x87 result.
__device__ __forceinline__ bool dnrm2_fast(int n, const double* x, int lane, double* res) {
  double h = 0.0, l = 0.0;
  if (lane < n) {
    const double v = x[lane];
    h = mul(v, v);
    l = fma_(v, v, -h);                        // exact square h + l
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double bh = __shfl_xor_sync(0xffffffffu, h, o), bl = __shfl_xor_sync(0xffffffffu, l, o);
    dd_add(h, l, bh, bl);
  }
  const bool ok = dnrm2_decide(h, l, res);
  return !__any_sync(0xffffffffu, !ok);
}

// dnrm2(n, x, 1), x in shared memory; every lane returns the same value
VK_DN double dnrm2_warp(int n, const double* x, SvdWarpSmem& sm, int lane) {
  if (n <= 0) return 0.0;
  if (n == 1) return fabs(x[0]);
  if (n <= 32) {
    double r;
    if (dnrm2_fast(n, x, lane, &r)) return r;
  }
  for (int j = lane; j < n; j += 32) {
    const Ext q = ext_sq(x[j]);
    sm.em[j] = q.m;
    sm.ee[j] = q.e;
  }
  __syncwarp();
  const int n8 = n & ~7;
  Ext acc{0, 0};
  if (lane < 4) {
    for (int j = lane; j < n8; j += 4) acc = ext_add(acc, Ext{sm.em[j], sm.ee[j]});
    if (lane == 0)
      for (int j = n8; j < n; ++j) acc = ext_add(acc, Ext{sm.em[j], sm.ee[j]});
  }
  const Ext a0 = shfl_ext(acc, 0), a1 = shfl_ext(acc, 1), a2 = shfl_ext(acc, 2), a3 = shfl_ext(acc, 3);
  __syncwarp();
  return ext_sqrt_to_double(ext_add(ext_add(ext_add(a2, a0), a1), a3));
}

__device__ void dscal_warp(int n, double a, double* x, int lane) {
  for (int i = lane; i < n; i += 32) x[i] = mul(x[i], a);
  __syncwarp();
}

// dlarfg(n, alpha, x, 1, tau) with alpha and x in shared memory
VK_DN void dlarfg_warp(int n, double* alpha, double* x, double* tau, SvdWarpSmem& sm, int lane) {
  if (n <= 1) { *tau = 0.0; return; }
  VK_TP(tn);
  double xnorm = dnrm2_warp(n - 1, x, sm, lane);
  VK_TACC(14, tn);
  if (xnorm == 0.0) { *tau = 0.0; return; }
  double a = *alpha;
  double beta = -fsign(dlapy2(a, xnorm), a);
  const double safmin = DL_SFMIN / DL_EPS;
  const double rsafmn = 1.0 / safmin;
  int knt = 0;
  if (fabs(beta) < safmin) {
    do {
      ++knt;
      dscal_warp(n - 1, rsafmn, x, lane);
      beta = mul(beta, rsafmn);
      a = mul(a, rsafmn);
    } while (fabs(beta) < safmin && knt < 20);
    xnorm = dnrm2_warp(n - 1, x, sm, lane);
    beta = -fsign(dlapy2(a, xnorm), a);
  }
  *tau = div(sub(beta, a), beta);
  dscal_warp(n - 1, div(1.0, sub(a, beta)), x, lane);
  for (int j = 0; j < knt; ++j) beta = mul(beta, safmin);
  if (lane == 0) *alpha = beta;
  __syncwarp();
}

// dlarf('L', m, n, v, 1, tau, C, ldc) with n <= 2 columns, v and C in shared memory
VK_DN void dlarf_left_warp(int m, int n, const double* v, double tau, double* C, int ldc, int lane) {
  int lastv = 0, lastc = 0;
  if (tau != 0.0) {
    lastv = m;
    while (lastv > 0 && v[lastv - 1] == 0.0) --lastv;
    lastc = n;
    if (n > 0 && C[0 + (n - 1) * ldc] == 0.0 && C[(lastv - 1) + (n - 1) * ldc] == 0.0) {
      lastc = 0;
      for (int j = n - 1; j >= 0 && lastc == 0; --j)
        for (int r = 0; r < lastv; ++r)
          if (C[r + j * ldc] != 0.0) { lastc = j + 1; break; }
    }
  }
  if (lastv <= 0 || lastc <= 0) return;
  // dgemv_t(lastv, lastc): kernel chains over the first nb rows, then the tail
  const int m3 = lastv & 3, nb = lastv - m3;
  const bool k4x1 = (lastc & 1) != 0;               // n2 & 1: the last column via the 4x1 kernel
  // chain q of column c: 4x2 columns take q in {0 (even rows), 1 (odd rows)},
  // the 4x1 column q in {0..3} (rows = q mod 4)
  double part = 0.0;
  {
    int c = -1, q = 0, step = 0;
    if (k4x1) {
      if (lastc == 1 && lane < 4) { c = 0; q = lane; step = 4; }
      // lastc == 3 does not occur (n <= 2)
    } else if (lane < 2 * lastc) {
      c = lane >> 1; q = lane & 1; step = 2;
    }
    if (c >= 0)
      for (int i = q; i < nb; i += step) part = add(part, mul(C[i + c * ldc], v[i]));
  }
  double w[2];
  for (int c = 0; c < lastc; ++c) {
    double acc = 0.0;
    if (nb > 0) {
      if (k4x1) {
        const double l0 = __shfl_sync(0xffffffffu, part, 0), l1 = __shfl_sync(0xffffffffu, part, 1),
                     l2 = __shfl_sync(0xffffffffu, part, 2), l3 = __shfl_sync(0xffffffffu, part, 3);
        acc = add(add(l0, l2), add(l1, l3));
      } else {
        const double e = __shfl_sync(0xffffffffu, part, 2 * c), o = __shfl_sync(0xffffffffu, part, 2 * c + 1);
        acc = add(e, o);
      }
    }
    const double* at = C + c * ldc + nb;
    const double* xt = v + nb;
    if (m3 == 3) acc = add(acc, fma_(at[2], xt[2], fma_(at[0], xt[0], mul(at[1], xt[1]))));
    if (m3 == 2) acc = add(acc, fma_(at[0], xt[0], mul(at[1], xt[1])));
    if (m3 == 1) acc = fma_(at[0], xt[0], acc);
    w[c] = acc;
  }
  __syncwarp();
  // dger(lastv, lastc, -tau, v, w, C): one element per lane
  const double y0[2] = {mul(-tau, w[0]), lastc > 1 ? mul(-tau, w[1]) : 0.0};
  for (int t = lane; t < lastv * lastc; t += 32) {
    const int c = t / lastv, r = t - c * lastv;
    C[r + c * ldc] = fma_(y0[c], v[r], C[r + c * ldc]);
  }
  __syncwarp();
}

// numpy.linalg.svd(A, full_matrices=False) of the row-major (M x 3) A (the
// same on every lane); outputs on every lane as svd_m3.
VK_DN int svd_m3_warp(const double* A_rm, int M, double* U_rm, double* s, double* VT_rm,
                           SvdWarpSmem& sm, int lane) {
  const int N = 3;
  double* A = sm.A;
  VK_TP(t0);
  for (int t = lane; t < M * N; t += 32) {
    const int r = t / N, c = t - r * N;
    A[r + c * M] = A_rm[t];
  }
  __syncwarp();
  double tau[3];
  // dgeqr2
  for (int i = 0; i < N; ++i) {
    dlarfg_warp(M - i, &A[i + i * M], &A[(i + 1 < M ? i + 1 : M - 1) + i * M], &tau[i], sm, lane);
    if (i < N - 1) {
      const double aii = A[i + i * M];
      __syncwarp();
      if (lane == 0) A[i + i * M] = 1.0;
      __syncwarp();
      VK_TP(tl);
      dlarf_left_warp(M - i, N - i - 1, &A[i + i * M], tau[i], &A[i + (i + 1) * M], M, lane);
      VK_TACC(15, tl);
      if (lane == 0) A[i + i * M] = aii;
      __syncwarp();
    }
  }
  VK_TACC(8, t0);
  VK_TP(t1);
  double R[9];
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < N; ++i) R[i + j * N] = (i <= j) ? A[i + j * M] : 0.0;
  __syncwarp();
  // dorg2r(M, 3, 3)
  for (int i = N - 1; i >= 0; --i) {
    if (i < N - 1) {
      if (lane == 0) A[i + i * M] = 1.0;
      __syncwarp();
      dlarf_left_warp(M - i, N - i - 1, &A[i + i * M], tau[i], &A[i + (i + 1) * M], M, lane);
    }
    if (i < M - 1) dscal_warp(M - i - 1, -tau[i], &A[i + 1 + i * M], lane);
    if (lane == 0) A[i + i * M] = sub(1.0, tau[i]);
    if (lane < i) A[lane + i * M] = 0.0;
    __syncwarp();
  }
  VK_TACC(9, t1);
  VK_TP(t2);
  // the 3 x 3 stages, redundantly on every lane
  double d[3], e[3], tauq[3], taup[3];
  dgebd2(N, N, R, N, d, e, tauq, taup);
  VK_TACC(12, t2);
  VK_TP(t3);
  double Ub[9], VTb[9];
  const int info = dbdsdc(N, d, e, Ub, N, VTb, N);
  if (info) return info;
  VK_TACC(13, t3);
  VK_TP(t4);
  dorm2r_ln(N, N, N, R, N, tauq, Ub, N);
  dorml2_rn(N, N - 1, N - 1, &R[0 + 1 * N], N, taup, &VTb[0 + 1 * N], N);
  VK_TACC(10, t4);
  VK_TP(t5);
  // dgemm('N','N', M, 3, 3, 1, Q, Ub, 0, U)
  for (int t = lane; t < M * N; t += 32) {
    const int i = t / N, j = t - i * N;
    double c = mul(A[i + 0 * M], Ub[0 + j * N]);
    c = fma_(A[i + 1 * M], Ub[1 + j * N], c);
    c = fma_(A[i + 2 * M], Ub[2 + j * N], c);
    sm.U[t] = c;
  }
  __syncwarp();
  for (int t = 0; t < M * N; ++t) U_rm[t] = sm.U[t];
  for (int i = 0; i < N; ++i) {
    s[i] = d[i];
    for (int j = 0; j < N; ++j) VT_rm[i * N + j] = VTb[i + j * N];
  }
  __syncwarp();
  VK_TACC(11, t5);
  return 0;
}

// Two-warp form of svd_m3_warp (same operations, same bits): both warps run
// the Householder QR on their own copy of the matrix, then warp 0 forms Q
// (dorg2r) while warp 1 runs the 3 x 3 stages (dgebd2, dbdsdc, dormbr x 2);
// after one CTA barrier each warp forms U = Q U_B from warp 0's Q and warp
// 1's U_B.  Called by both warps of the fit CTA with their own `sm` (`other`
// is the other warp's).  A warp rewrites its Q / the exchange only in its
// next call, after the caller's next CTA barrier (trf_warp.cuh).
VK_DN int svd_m3_2w(const double* A_rm, int M, double* U_rm, double* s, double* VT_rm, SvdWarpSmem& sm,
                    const SvdWarpSmem& other, SvdXchg& xc, int lane, int wid) {
  const int N = 3;
  double* A = sm.A;
  VK_TP(t0);
  for (int t = lane; t < M * N; t += 32) {
    const int r = t / N, c = t - r * N;
    A[r + c * M] = A_rm[t];
  }
  __syncwarp();
  double tau[3];
  // dgeqr2
  for (int i = 0; i < N; ++i) {
    dlarfg_warp(M - i, &A[i + i * M], &A[(i + 1 < M ? i + 1 : M - 1) + i * M], &tau[i], sm, lane);
    if (i < N - 1) {
      const double aii = A[i + i * M];
      __syncwarp();
      if (lane == 0) A[i + i * M] = 1.0;
      __syncwarp();
      VK_TP(tl);
      dlarf_left_warp(M - i, N - i - 1, &A[i + i * M], tau[i], &A[i + (i + 1) * M], M, lane);
      VK_TACC(15, tl);
      if (lane == 0) A[i + i * M] = aii;
      __syncwarp();
    }
  }
  VK_TACC(8, t0);
  VK_TP(t1);
  double R[9];
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < N; ++i) R[i + j * N] = (i <= j) ? A[i + j * M] : 0.0;
  __syncwarp();
  if (wid == 0) {
    // dorg2r(M, 3, 3)
    for (int i = N - 1; i >= 0; --i) {
      if (i < N - 1) {
        if (lane == 0) A[i + i * M] = 1.0;
        __syncwarp();
        dlarf_left_warp(M - i, N - i - 1, &A[i + i * M], tau[i], &A[i + (i + 1) * M], M, lane);
      }
      if (i < M - 1) dscal_warp(M - i - 1, -tau[i], &A[i + 1 + i * M], lane);
      if (lane == 0) A[i + i * M] = sub(1.0, tau[i]);
      if (lane < i) A[lane + i * M] = 0.0;
      __syncwarp();
    }
    VK_TACC(9, t1);
  } else {
    // the 3 x 3 stages, redundantly on every lane of warp 1
    double d[3], e[3], tauq[3], taup[3];
    dgebd2(N, N, R, N, d, e, tauq, taup);
    double Ub[9], VTb[9];
    const int info = dbdsdc(N, d, e, Ub, N, VTb, N);
    if (!info) {
      dorm2r_ln(N, N, N, R, N, tauq, Ub, N);
      dorml2_rn(N, N - 1, N - 1, &R[0 + 1 * N], N, taup, &VTb[0 + 1 * N], N);
    }
    if (lane == 0) {
      xc.info = info;
      for (int i = 0; i < 3; ++i) xc.d[i] = d[i];
      for (int i = 0; i < 9; ++i) { xc.Ub[i] = Ub[i]; xc.VTb[i] = VTb[i]; }
    }
  }
  __syncthreads();                                   // Q and the 3 x 3 results visible to both warps
  if (xc.info) return xc.info;
  VK_TP(t5);
  // dgemm('N','N', M, 3, 3, 1, Q, Ub, 0, U)
  const double* Q = wid == 0 ? A : other.A;
  for (int t = lane; t < M * N; t += 32) {
    const int i = t / N, j = t - i * N;
    double c = mul(Q[i + 0 * M], xc.Ub[0 + j * N]);
    c = fma_(Q[i + 1 * M], xc.Ub[1 + j * N], c);
    c = fma_(Q[i + 2 * M], xc.Ub[2 + j * N], c);
    sm.U[t] = c;
  }
  __syncwarp();
  for (int t = 0; t < M * N; ++t) U_rm[t] = sm.U[t];
  for (int i = 0; i < N; ++i) {
    s[i] = xc.d[i];
    for (int j = 0; j < N; ++j) VT_rm[i * N + j] = xc.VTb[i + j * N];
  }
  __syncwarp();
  VK_TACC(11, t5);
  return 0;
}

}  // namespace lapack
}  // namespace vk
