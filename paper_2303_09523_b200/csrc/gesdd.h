// numpy.linalg.svd(J_augmented, full_matrices=False) for the (M x 3)
// augmented Jacobian of the variogram fit, restated so the device TRF
// (trf.h) gets the reference's factors bit for bit.
//
// numpy 2.3.5 calls LAPACK dgesdd(jobz='S') in its bundled OpenBLAS 0.3.30
// (LAPACK reference Fortran, built without FMA; BLAS kernels for SKYLAKEX on
// the hosts the reference was pinned on).  For M >= 5 rows and N = 3 columns
// dgesdd takes its "M much larger than N" path 3:
//   dgeqrf -> dgeqr2          A = Q R (Householder, dlarfg / dlarf)
//   dorgqr -> dorg2r          Q explicitly
//   dgebrd -> dgebd2          R = Q_B B P^T (B upper bidiagonal)
//   dbdsdc('U','I') -> dlasdq -> dbdsqr   B = U_B S V_B^T (implicit QR)
//   dormbr('Q','L','N'), dormbr('P','R','T')   U_R = Q_B U_B, V^T = V_B^T P^T
//   dgemm                     U = Q U_R
// (checked here: composing those exported routines reproduces numpy.linalg.svd
// bit for bit).  Each routine below follows the published LAPACK algorithm;
// the BLAS calls inside them follow the SKYLAKEX kernels' operation order:
// dnrm2 accumulates squares in x87 80-bit registers (four accumulators, then
// fsqrt and one rounding to double) -- emulated exactly with 64-bit integer
// significands; dgemv_t / dgemv_n / daxpy (dger) / drot / dgemm as noted at
// each function.  Storage is column-major (Fortran), 0-based.
#pragma once
#include <cstdint>
#include <cmath>
#include <type_traits>
#include "vk_common.h"
#include "npref.h"

namespace vk {
namespace lapack {

using np::add;
using np::sub;
using np::mul;
using np::div;
using np::fma_;
using np::sqrt_;

constexpr int GMAXM = MAX_BINS + 3;
constexpr double DL_EPS = 1.1102230246251565e-16;      // dlamch('E') = 2^-53
constexpr double DL_SFMIN = 2.2250738585072014e-308;   // dlamch('S')
constexpr double DL_HUGE = 1.7976931348623157e308;     // dlamch('O')

VK_HD double fsign(double a, double b) { return copysign(fabs(a), b); }   // Fortran SIGN (gfortran: IEEE sign of b)

// ---------------------------------------------------------------- dnrm2 (x87)
struct Ext {            // value = m * 2^e, bit 63 of m set (m == 0: zero)
  uint64_t m;
  int e;
};

VK_HD int clz64(uint64_t x) {
#if defined(__CUDA_ARCH__)
  return __clzll((long long)x);
#else
  return __builtin_clzll(x);
#endif
}

VK_HD double u128_to_double(unsigned __int128 v) {
  return (double)(uint64_t)(v >> 64) * 18446744073709551616.0 + (double)(uint64_t)v;
}

VK_HD int top_bit128(unsigned __int128 v) {
  const uint64_t hi = (uint64_t)(v >> 64);
  return hi ? 127 - clz64(hi) : 63 - clz64((uint64_t)v);
}

VK_HD uint64_t umulhi64(uint64_t a, uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

VK_HD uint64_t dbits(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  uint64_t b;
  __builtin_memcpy(&b, &x, 8);
  return b;
#endif
}

// round-to-nearest-even increment of a 64-bit significand m whose discarded
// fraction is frac (bit 63 = one half, bit 0 sticky)
VK_HD Ext ext_round_frac(uint64_t m, uint64_t frac, int e) {
  const uint64_t half = 1ull << 63;
  if (frac > half || (frac == half && (m & 1))) {
    m += 1;
    if (m == 0) return Ext{half, e + 1};
  }
  return Ext{m, e};
}

// fmul st(0), st(0) of a double loaded with fldl: x*x in extended precision
VK_HD Ext ext_sq(double x) {
  const uint64_t bits = dbits(x) & 0x7fffffffffffffffull;
  if (bits == 0) return Ext{0, 0};
  int ex = (int)(bits >> 52);
  uint64_t mx = bits & 0xfffffffffffffull;
  if (ex == 0) {                                        // subnormal: normalise
    const int sh = clz64(mx) - 11;
    mx <<= sh;
    ex = 1 - sh;
  } else {
    mx |= 1ull << 52;
  }
  // x = mx * 2^(ex - 1075); x^2 = mx^2 * 2^(2ex - 2150), mx^2 in [2^104, 2^106)
  const uint64_t lo = mx * mx, hi = umulhi64(mx, mx);
  const int e2 = 2 * ex - 2150;
  if (hi >> 41) {                                       // top bit 105: drop 42 bits
    const uint64_t m = (hi << 22) | (lo >> 42);
    const uint64_t rest = lo << 22;                     // the 42 dropped bits, left-aligned
    return ext_round_frac(m, rest, e2 + 42);
  }
  const uint64_t m = (hi << 23) | (lo >> 41);           // top bit 104: drop 41 bits
  const uint64_t rest = lo << 23;
  return ext_round_frac(m, rest, e2 + 41);
}

// faddp of two non-negative extended values (round to nearest even, 64 bits)
VK_HD Ext ext_add(Ext a, Ext b) {
  if (a.m == 0) return b;
  if (b.m == 0) return a;
  if (b.e > a.e || (b.e == a.e && b.m > a.m)) { const Ext t = a; a = b; b = t; }
  const int d = a.e - b.e;
  if (d >= 66) return a;                                // b < a quarter ulp of a: no change
  uint64_t bh, frac;
  if (d == 0) { bh = b.m; frac = 0; }
  else if (d < 64) { bh = b.m >> d; frac = b.m << (64 - d); }
  else { bh = 0; frac = (b.m >> (d - 64)) | ((b.m << (128 - d)) != 0 ? 1ull : 0ull); }
  const uint64_t sum = a.m + bh;
  if (sum >= a.m) return ext_round_frac(sum, frac, a.e);   // no carry
  // carry: true significand is 2^64 + sum; shift right one (keep sticky)
  const uint64_t m = (1ull << 63) | (sum >> 1);
  const uint64_t f2 = ((sum & 1) << 63) | (frac >> 1) | (frac & 1);
  return ext_round_frac(m, f2, a.e + 1);
}

// fsqrt (correctly rounded to 64 bits) then fstpl (rounded to double), by
// exact integer square root -- the reference form, and the fallback of
// ext_sqrt_to_double near a rounding boundary
VK_HDC double ext_sqrt_exact(Ext a) {
  if (a.m == 0) return 0.0;
  unsigned __int128 M;
  int re;
  if (((a.e % 2) + 2) % 2 == 0) { M = ((unsigned __int128)a.m) << 64; re = (a.e - 64) / 2; }
  else { M = ((unsigned __int128)a.m) << 63; re = (a.e - 63) / 2; }
  // r = floor(sqrt(M)) from a double estimate plus exact integer correction
  uint64_t r = (uint64_t)sqrt(u128_to_double(M));
  for (int it = 0; it < 4; ++it) {
    const unsigned __int128 r2 = (unsigned __int128)r * r;
    if (r2 > M) {
      const double err = u128_to_double(r2 - M) / (2.0 * (double)r);
      const uint64_t dr = (uint64_t)err + 1;
      r -= dr;
    } else {
      const unsigned __int128 r12 = (unsigned __int128)(r + 1) * (r + 1);
      if (r12 <= M) {
        const double err = u128_to_double(M - r12) / (2.0 * (double)r);
        r += (uint64_t)err + 1;
      } else {
        break;
      }
    }
  }
  while ((unsigned __int128)r * r > M) --r;
  while ((unsigned __int128)(r + 1) * (r + 1) <= M) ++r;
  const unsigned __int128 R = M - (unsigned __int128)r * r;
  if (R > r) {                                           // sqrt(M) > r + 1/2
    r += 1;
    if (r == 0) { r = 1ull << 63; re += 1; }
  }
  // round the 64-bit significand to 53 bits, nearest even
  uint64_t q = r >> 11;
  const uint64_t rem = r & 0x7ff;
  if (rem > 0x400 || (rem == 0x400 && (q & 1))) q += 1;
  return ldexp((double)q, re + 11);
}

// fsqrt then fstpl, fast form: S = F 2^E with F in [1, 4) (E even) as an
// exact double pair Fh + Fl; y = sqrt(Fh) rounded, one Newton correction
// d = (Fh - y^2 + Fl) / 2y (Fh - y^2 exact by FMA) gives sqrt(S) to ~2^-103
// absolute, i.e. the offset t = d / 2^-63 from y on the 64-bit grid to ~2^-40;
// t rounds to the 64-bit result unless it lies within 2^-30 of a half (then
// the exact integer form decides), and the 64-bit result rounds to 53 bits by
// integer arithmetic on t (ties to even).
VK_HD double ext_sqrt_to_double(Ext a) {
  if (a.m == 0) return 0.0;
  int E = a.e + 63;
  double Fh = (double)(a.m & ~0x7ffull) * 0x1p-63;       // exact: 53 significant bits
  double Fl = (double)(a.m & 0x7ffull) * 0x1p-63;        // exact: 11 bits
  if (E & 1) { Fh *= 2.0; Fl *= 2.0; E -= 1; }
  const double y = sqrt_(Fh);                            // in [1, 2]
  if (!(y < 2.0)) return ext_sqrt_exact(a);
  const double e1 = fma_(-y, y, Fh);                     // exact residual
  const double R = add(e1, Fl);
#if defined(__CUDA_ARCH__)
  const double half_inv = 0.5 * __drcp_rn(y);
#else
  const double half_inv = 0.5 / y;
#endif
  const double t = mul(R, half_inv) * 0x1p63;             // offset in units of 2^-63
  const double n = rint(t);
  if (fabs(fabs(t - n) - 0.5) < 0x1p-30) return ext_sqrt_exact(a);
  // 53-bit rounding of y + n 2^-63: y's ulp is 2^-52 = 2^11 units
  const long long ni = (long long)n;
  long long q0 = ni >> 11;                               // floor(n / 2048)
  const long long r = ni - (q0 << 11);                   // 0 .. 2047
  const long long ymant = (long long)(dbits(y) & 0xfffffffffffffull);
  long long q = q0;
  if (r > 1024 || (r == 1024 && ((ymant + q0) & 1))) q = q0 + 1;
  const double res = y + (double)q * 0x1p-52;            // exact: a few ulps of y
  return scalbn(res, E / 2);
}

// (h, l) += (bh, bl) for non-negative double-doubles: two-sum of the high
// parts, low parts added to its error, renormalised
VK_HD void dd_add(double& h, double& l, double bh, double bl) {
  const double s = add(h, bh), bb = sub(s, h);
  const double e = add(add(sub(h, sub(s, bb)), sub(bh, bb)), add(l, bl));
  h = add(s, e);
  l = sub(e, sub(h, s));
}

// Fast decision of the x87 dnrm2 from the exact sum of squares S = h + l (a
// double-double, relative error < 2^-100).  The x87 chain rounds each square
// and each partial sum to 64 bits: n <= 32 terms give |X - S| <= n 2^-64 S,
// so round64(sqrt X) lies within 2^-59 y of y = sqrt(S).  If y is farther
// than that from every midpoint between two doubles, round53(round64(sqrt X))
// = round53(y) = yh (the correctly rounded sqrt(h), corrected by yl < ulp/2).
// Returns false (the caller runs the exact emulation) near a midpoint (about
// 1 % of inputs), when yh is a power of two, or outside [2^-900, 2^900].
VK_HD bool dnrm2_decide(double h, double l, double* res) {
  if (!(h > 0x1p-900 && h < 0x1p+900)) return false;
  const double yh = sqrt_(h);
  const double r = add(fma_(-yh, yh, h), l);             // S - yh^2 (first term exact)
  const double yl = mul(r, div(0.5, yh));
  const uint64_t b = dbits(yh);
  if ((b & 0xfffffffffffffull) == 0) return false;
  const double ulp = np::from_bits(((b >> 52) - 52) << 52);
  if (!(fabs(yl) < sub(mul(0.5, ulp), mul(yh, 0x1p-58)))) return false;
  *res = yh;
  return true;
}

// double-double accumulation of squares (error-free products, two-sum; every
// operation rounded separately -- no contraction)
VK_HD void dd_add_sq(double v, double& h, double& l) {
  const double p = mul(v, v);
  const double pe = fma_(v, v, -p);
  dd_add(h, l, p, pe);
}

// OpenBLAS dnrm2 (interface: n == 1 -> |x|; kernel dnrm2_k SKYLAKEX, x87)
VK_HDN double dnrm2(int n, const double* x, int incx) {
  if (n <= 0) return 0.0;
  if (n == 1) return fabs(x[0]);
  if (n <= 32) {
    double h = 0.0, l = 0.0, r;
    for (int i = 0; i < n; ++i) dd_add_sq(x[i * incx], h, l);
    if (dnrm2_decide(h, l, &r)) return r;
  }
  Ext acc[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  int i = 0;
  const int n8 = n & ~7;
  for (; i < n8; ++i) acc[i & 3] = ext_add(acc[i & 3], ext_sq(x[i * incx]));
  for (; i < n; ++i) acc[0] = ext_add(acc[0], ext_sq(x[i * incx]));
  const Ext t = ext_add(ext_add(ext_add(acc[2], acc[0]), acc[1]), acc[3]);
  return ext_sqrt_to_double(t);
}

// ------------------------------------------------------------------ BLAS 1/2
VK_HD void dscal(int n, double a, double* x, int incx) {
  for (int i = 0; i < n; ++i) x[i * incx] = mul(x[i * incx], a);
}

// y := A^T x for an (m x n) column-major A (dgemv_t SKYLAKEX, alpha 1, beta 0)
VK_HD void dgemv_t(int m, int n, const double* A, int lda, const double* x, double* y) {
  const int m3 = m & 3, nb = m - m3;
  for (int j = 0; j < n; ++j) {
    const double* a = A + j * lda;
    double acc = 0.0;
    if (nb > 0) {
      const int n4 = (n >> 2) << 2;   // columns through the 4x4 kernel (n >= 4 only)
      const bool k4x1 = (j >= n4) && ((n & 3) & 1) && (j == n - 1);
      if (!k4x1) {                                       // dgemv_kernel_4x2 (and 4x4)
        double e = 0.0, o = 0.0;
        for (int i = 0; i < nb; i += 2) {
          e = add(e, mul(a[i], x[i]));
          o = add(o, mul(a[i + 1], x[i + 1]));
        }
        acc = add(e, o);
      } else {                                           // dgemv_kernel_4x1
        double l0 = 0.0, l1 = 0.0, l2 = 0.0, l3 = 0.0;
        for (int i = 0; i < nb; i += 4) {
          l0 = add(l0, mul(a[i], x[i]));
          l1 = add(l1, mul(a[i + 1], x[i + 1]));
          l2 = add(l2, mul(a[i + 2], x[i + 2]));
          l3 = add(l3, mul(a[i + 3], x[i + 3]));
        }
        acc = add(add(l0, l2), add(l1, l3));
      }
    }
    const double* at = a + nb;
    const double* xt = x + nb;
    if (m3 == 3) acc = add(acc, fma_(at[2], xt[2], fma_(at[0], xt[0], mul(at[1], xt[1]))));
    if (m3 == 2) acc = add(acc, fma_(at[0], xt[0], mul(at[1], xt[1])));
    if (m3 == 1) acc = fma_(at[0], xt[0], acc);
    y[j] = acc;
  }
}

// y := A x for an (m x n) column-major A, m <= 3 rows (dgemv_n SKYLAKEX
// row-tail paths, alpha 1, beta 0): the unrolled pair form when lda == 3 and
// incx == 1, else one FMA per column.
VK_HD void dgemv_n(int m, int n, const double* A, int lda, const double* x, int incx, double* y) {
  for (int i = 0; i < m; ++i) {
    double acc = 0.0;
    if (m == 3 && lda == 3 && incx == 1) {
      int k = 0;
      for (; k + 4 <= n; k += 4) {
        acc = add(acc, fma_(A[i + k * lda], x[k], mul(A[i + (k + 1) * lda], x[k + 1])));
        acc = add(acc, fma_(A[i + (k + 2) * lda], x[k + 2], mul(A[i + (k + 3) * lda], x[k + 3])));
      }
      for (; k < n; ++k) acc = fma_(A[i + k * lda], x[k], acc);
    } else {
      for (int k = 0; k < n; ++k) acc = fma_(A[i + k * lda], x[k * incx], acc);
    }
    y[i] = acc;
  }
}

// A += alpha x y^T (dger: per column daxpy with y0 = alpha*y[j], FMA update)
VK_HD void dger(int m, int n, double alpha, const double* x, const double* y, int incy,
                double* A, int lda) {
  for (int j = 0; j < n; ++j) {
    const double y0 = mul(alpha, y[j * incy]);
    for (int i = 0; i < m; ++i) A[i + j * lda] = fma_(y0, x[i], A[i + j * lda]);
  }
}

// drot SKYLAKEX: x' = c x + s y, y' = c y - s x
VK_HD void drot(int n, double* x, int incx, double* y, int incy, double c, double s) {
  for (int i = 0; i < n; ++i) {
    const double xi = x[i * incx], yi = y[i * incy];
    x[i * incx] = fma_(c, xi, mul(s, yi));
    y[i * incy] = fma_(c, yi, -mul(s, xi));
  }
}

VK_HD void dswap(int n, double* x, int incx, double* y, int incy) {
  for (int i = 0; i < n; ++i) {
    const double t = x[i * incx];
    x[i * incx] = y[i * incy];
    y[i * incy] = t;
  }
}

// ------------------------------------------------------------------- LAPACK
VK_HDN double dlapy2(double x, double y) {
  if (x != x) return x;
  if (y != y) return y;
  const double xa = fabs(x), ya = fabs(y);
  const double w = fmax(xa, ya), z = fmin(xa, ya);
  if (z == 0.0 || w > DL_HUGE) return w;
  const double q = div(z, w);
  return mul(w, sqrt_(add(1.0, mul(q, q))));
}

// dlarfg(n, alpha, x, incx, tau)
VK_HDN void dlarfg(int n, double* alpha, double* x, int incx, double* tau) {
  if (n <= 1) { *tau = 0.0; return; }
  double xnorm = dnrm2(n - 1, x, incx);
  if (xnorm == 0.0) { *tau = 0.0; return; }
  double beta = -fsign(dlapy2(*alpha, xnorm), *alpha);
  const double safmin = DL_SFMIN / DL_EPS;
  const double rsafmn = 1.0 / safmin;
  int knt = 0;
  if (fabs(beta) < safmin) {
    do {
      ++knt;
      dscal(n - 1, rsafmn, x, incx);
      beta = mul(beta, rsafmn);
      *alpha = mul(*alpha, rsafmn);
    } while (fabs(beta) < safmin && knt < 20);
    xnorm = dnrm2(n - 1, x, incx);
    beta = -fsign(dlapy2(*alpha, xnorm), *alpha);
  }
  *tau = div(sub(beta, *alpha), beta);
  dscal(n - 1, div(1.0, sub(*alpha, beta)), x, incx);
  for (int j = 0; j < knt; ++j) beta = mul(beta, safmin);
  *alpha = beta;
}

// dlarf(side, m, n, v, incv, tau, C, ldc)
VK_HDN void dlarf(bool left, int m, int n, const double* v, int incv, double tau, double* C, int ldc) {
  int lastv = 0, lastc = 0;
  if (tau != 0.0) {
    lastv = left ? m : n;
    int i = (incv > 0) ? (lastv - 1) * incv : 0;
    while (lastv > 0 && v[i] == 0.0) { --lastv; i -= incv; }
    if (left) {                                           // iladlc(lastv, n, C, ldc)
      lastc = n;
      if (n > 0 && C[0 + (n - 1) * ldc] == 0.0 && C[(lastv - 1) + (n - 1) * ldc] == 0.0) {
        lastc = 0;
        for (int j = n - 1; j >= 0 && lastc == 0; --j)
          for (int r = 0; r < lastv; ++r)
            if (C[r + j * ldc] != 0.0) { lastc = j + 1; break; }
      }
    } else {                                              // iladlr(m, lastv, C, ldc)
      lastc = m;
      if (m > 0 && C[(m - 1) + 0] == 0.0 && C[(m - 1) + (lastv - 1) * ldc] == 0.0) {
        lastc = 0;
        for (int j = 0; j < lastv; ++j) {
          int r = m;
          while (r >= 1 && C[(r - 1) + j * ldc] == 0.0) --r;
          if (r > lastc) lastc = r;
        }
      }
    }
  }
  if (lastv <= 0 || lastc <= 0) return;
  double w[GMAXM];
  double vv[GMAXM];
  for (int k = 0; k < lastv; ++k) vv[k] = v[k * incv];
  if (left) {
    dgemv_t(lastv, lastc, C, ldc, vv, w);
    dger(lastv, lastc, -tau, vv, w, 1, C, ldc);
  } else {
    dgemv_n(lastc, lastv, C, ldc, v, incv, w);
    dger(lastc, lastv, -tau, w, vv, 1, C, ldc);
  }
}

// dgeqr2(m, n, A, lda, tau), n = 3
VK_HDN void dgeqr2(int m, int n, double* A, int lda, double* tau) {
  const int k = m < n ? m : n;
  for (int i = 0; i < k; ++i) {
    dlarfg(m - i, &A[i + i * lda], &A[(i + 1 < m ? i + 1 : m - 1) + i * lda], 1, &tau[i]);
    if (i < n - 1) {
      const double aii = A[i + i * lda];
      A[i + i * lda] = 1.0;
      dlarf(true, m - i, n - i - 1, &A[i + i * lda], 1, tau[i], &A[i + (i + 1) * lda], lda);
      A[i + i * lda] = aii;
    }
  }
}

// dorg2r(m, n, k, A, lda, tau), k = n
VK_HDN void dorg2r(int m, int n, int k, double* A, int lda, const double* tau) {
  for (int i = k - 1; i >= 0; --i) {
    if (i < n - 1) {
      A[i + i * lda] = 1.0;
      dlarf(true, m - i, n - i - 1, &A[i + i * lda], 1, tau[i], &A[i + (i + 1) * lda], lda);
    }
    if (i < m - 1) dscal(m - i - 1, -tau[i], &A[i + 1 + i * lda], 1);
    A[i + i * lda] = sub(1.0, tau[i]);
    for (int l = 0; l < i; ++l) A[l + i * lda] = 0.0;
  }
}

// dgebd2(m, n, A, lda, d, e, tauq, taup), m >= n
VK_HDN void dgebd2(int m, int n, double* A, int lda, double* d, double* e, double* tauq, double* taup) {
  for (int i = 0; i < n; ++i) {
    dlarfg(m - i, &A[i + i * lda], &A[(i + 1 < m ? i + 1 : m - 1) + i * lda], 1, &tauq[i]);
    d[i] = A[i + i * lda];
    A[i + i * lda] = 1.0;
    if (i < n - 1) dlarf(true, m - i, n - i - 1, &A[i + i * lda], 1, tauq[i], &A[i + (i + 1) * lda], lda);
    A[i + i * lda] = d[i];
    if (i < n - 1) {
      dlarfg(n - i - 1, &A[i + (i + 1) * lda], &A[i + (i + 2 < n ? i + 2 : n - 1) * lda], lda, &taup[i]);
      e[i] = A[i + (i + 1) * lda];
      A[i + (i + 1) * lda] = 1.0;
      dlarf(false, m - i - 1, n - i - 1, &A[i + (i + 1) * lda], lda, taup[i], &A[(i + 1) + (i + 1) * lda], lda);
      A[i + (i + 1) * lda] = e[i];
    } else {
      taup[i] = 0.0;
    }
  }
}

// dlartg (LAPACK 3.10+ form)
VK_HDN void dlartg(double f, double g, double* c, double* s, double* r) {
  const double safmin = 2.2250738585072014e-308;         // 2^-1022
  const double safmax = 4.49423283715579e+307;           // 2^1022
  const double rtmin = 1.4916681462400413e-154;          // sqrt(safmin)
  const double rtmax = sqrt(safmax / 2);
  const double f1 = fabs(f), g1 = fabs(g);
  if (g == 0.0) {
    *c = 1.0; *s = 0.0; *r = f;
  } else if (f == 0.0) {
    *c = 0.0; *s = fsign(1.0, g); *r = g1;
  } else if (f1 > rtmin && f1 < rtmax && g1 > rtmin && g1 < rtmax) {
    const double d = sqrt_(add(mul(f, f), mul(g, g)));
    *c = div(f1, d);
    *r = fsign(d, f);
    *s = div(g, *r);
  } else {
    const double u = fmin(safmax, fmax(safmin, fmax(f1, g1)));
    const double fs = div(f, u), gs = div(g, u);
    const double d = sqrt_(add(mul(fs, fs), mul(gs, gs)));
    *c = div(fabs(fs), d);
    *r = fsign(d, f);
    *s = div(gs, *r);
    *r = mul(*r, u);
  }
}

// dlas2: singular values of [[f, g], [0, h]]
VK_HDN void dlas2(double f, double g, double h, double* ssmin, double* ssmax) {
  const double fa = fabs(f), ga = fabs(g), ha = fabs(h);
  const double fhmn = fmin(fa, ha), fhmx = fmax(fa, ha);
  if (fhmn == 0.0) {
    *ssmin = 0.0;
    if (fhmx == 0.0) {
      *ssmax = ga;
    } else {
      const double q = div(fmin(fhmx, ga), fmax(fhmx, ga));
      *ssmax = mul(fmax(fhmx, ga), sqrt_(add(1.0, mul(q, q))));
    }
  } else {
    if (ga < fhmx) {
      const double as = add(1.0, div(fhmn, fhmx));
      const double at = div(sub(fhmx, fhmn), fhmx);
      const double q = div(ga, fhmx);
      const double au = mul(q, q);
      const double c = div(2.0, add(sqrt_(add(mul(as, as), au)), sqrt_(add(mul(at, at), au))));
      *ssmin = mul(fhmn, c);
      *ssmax = div(fhmx, c);
    } else {
      const double au = div(fhmx, ga);
      if (au == 0.0) {
        *ssmin = div(mul(fhmn, fhmx), ga);
        *ssmax = ga;
      } else {
        const double as = add(1.0, div(fhmn, fhmx));
        const double at = div(sub(fhmx, fhmn), fhmx);
        const double p1 = mul(as, au), p2 = mul(at, au);
        const double c = div(1.0, add(sqrt_(add(1.0, mul(p1, p1))), sqrt_(add(1.0, mul(p2, p2)))));
        double smin = mul(mul(fhmn, c), au);
        smin = add(smin, smin);
        *ssmin = smin;
        *ssmax = div(ga, add(c, c));
      }
    }
  }
}

// dlasv2: SVD of [[f, g], [0, h]]
VK_HDN void dlasv2(double f, double g, double h, double* ssmin, double* ssmax, double* snr,
                  double* csr, double* snl, double* csl) {
  double ft = f, fa = fabs(ft), ht = h, ha = fabs(h);
  int pmax = 1;
  const bool swap = ha > fa;
  if (swap) {
    pmax = 3;
    double t = ft; ft = ht; ht = t;
    t = fa; fa = ha; ha = t;
  }
  const double gt = g, ga = fabs(gt);
  double clt, crt, slt, srt, smin, smax;
  if (ga == 0.0) {
    smin = ha; smax = fa;
    clt = 1.0; crt = 1.0; slt = 0.0; srt = 0.0;
  } else {
    bool gasmal = true;
    if (ga > fa) {
      pmax = 2;
      if (div(fa, ga) < DL_EPS) {
        gasmal = false;
        smax = ga;
        if (ha > 1.0) smin = div(fa, div(ga, ha));
        else smin = mul(div(fa, ga), ha);
        clt = 1.0;
        slt = div(ht, gt);
        srt = 1.0;
        crt = div(ft, gt);
      }
    }
    if (gasmal) {
      const double d = sub(fa, ha);
      double l = (d == fa) ? 1.0 : div(d, fa);
      const double m = div(gt, ft);
      double t = sub(2.0, l);
      const double mm = mul(m, m), tt = mul(t, t);
      const double s = sqrt_(add(tt, mm));
      const double r = (l == 0.0) ? fabs(m) : sqrt_(add(mul(l, l), mm));
      const double a = mul(0.5, add(s, r));
      smin = div(ha, a);
      smax = mul(fa, a);
      if (mm == 0.0) {
        if (l == 0.0) t = mul(fsign(2.0, ft), fsign(1.0, gt));
        else t = add(div(gt, fsign(d, ft)), div(m, t));
      } else {
        t = mul(add(div(m, add(s, t)), div(m, add(r, l))), add(1.0, a));
      }
      l = sqrt_(add(mul(t, t), 4.0));
      crt = div(2.0, l);
      srt = div(t, l);
      clt = div(add(crt, mul(srt, m)), a);
      slt = div(mul(div(ht, ft), srt), a);
    }
  }
  if (swap) { *csl = srt; *snl = crt; *csr = slt; *snr = clt; }
  else { *csl = clt; *snl = slt; *csr = crt; *snr = srt; }
  double tsign = 1.0;
  if (pmax == 1) tsign = mul(mul(fsign(1.0, *csr), fsign(1.0, *csl)), fsign(1.0, f));
  if (pmax == 2) tsign = mul(mul(fsign(1.0, *snr), fsign(1.0, *csl)), fsign(1.0, g));
  if (pmax == 3) tsign = mul(mul(fsign(1.0, *snr), fsign(1.0, *snl)), fsign(1.0, h));
  *ssmax = fsign(smax, tsign);
  *ssmin = fsign(smin, mul(mul(tsign, fsign(1.0, f)), fsign(1.0, h)));
}

// dlasr(side, 'V', direct, m, n, c, s, A, lda)
VK_HDN void dlasr(bool left, bool forward, int m, int n, const double* c, const double* s, double* A, int lda) {
  if (left) {
    for (int jj = 0; jj < m - 1; ++jj) {
      const int j = forward ? jj : m - 2 - jj;
      const double ct = c[j], st = s[j];
      if (ct != 1.0 || st != 0.0) {
        for (int i = 0; i < n; ++i) {
          const double temp = A[(j + 1) + i * lda];
          A[(j + 1) + i * lda] = sub(mul(ct, temp), mul(st, A[j + i * lda]));
          A[j + i * lda] = add(mul(st, temp), mul(ct, A[j + i * lda]));
        }
      }
    }
  } else {
    for (int jj = 0; jj < n - 1; ++jj) {
      const int j = forward ? jj : n - 2 - jj;
      const double ct = c[j], st = s[j];
      if (ct != 1.0 || st != 0.0) {
        for (int i = 0; i < m; ++i) {
          const double temp = A[i + (j + 1) * lda];
          A[i + (j + 1) * lda] = sub(mul(ct, temp), mul(st, A[i + j * lda]));
          A[i + j * lda] = add(mul(st, temp), mul(ct, A[i + j * lda]));
        }
      }
    }
  }
}

// dbdsqr('U', n, ncvt = n, nru = n, ncc = 0, d, e, VT, ldvt, U, ldu); n <= 3.
// Returns info (0 on convergence).
VK_HDN int dbdsqr(int n, double* d, double* e, double* VT, int ldvt, double* U, int ldu) {
  const int ncvt = n, nru = n;
  const double eps = DL_EPS, unfl = DL_SFMIN;
  const int maxitr = 6;
  if (n == 0) return 0;
  if (n > 1) {
    const int nm1 = n - 1, nm12 = nm1 + nm1, nm13 = nm12 + nm1;
    double work[4 * 3];
    int idir = 0;
    const double tolmul = 0x1.8ace5422aa0dbp+6;           // max(10, min(100, eps**(-1/8))), glibc pow
    const double tol = mul(tolmul, eps);
    double smax = 0.0;
    for (int i = 0; i < n; ++i) smax = fmax(smax, fabs(d[i]));
    for (int i = 0; i < n - 1; ++i) smax = fmax(smax, fabs(e[i]));
    double smin = 0.0, thresh;
    {
      double sminoa = fabs(d[0]);
      if (sminoa != 0.0) {
        double mu = sminoa;
        for (int i = 1; i < n; ++i) {
          mu = mul(fabs(d[i]), div(mu, add(mu, fabs(e[i - 1]))));
          sminoa = fmin(sminoa, mu);
          if (sminoa == 0.0) break;
        }
      }
      sminoa = div(sminoa, sqrt_((double)n));
      thresh = fmax(mul(tol, sminoa), mul((double)maxitr, mul((double)n, mul((double)n, unfl))));
    }
    const int maxitdivn = maxitr * n;
    int iterdivn = 0, iter = -1, oldll = -1, oldm = -1;
    int M = n;                                             // 1-based index of last unconverged
    // 1-based accessors
#define D_(i) d[(i) - 1]
#define E_(i) e[(i) - 1]
    while (true) {
      if (M <= 1) break;
      if (iter >= n) {
        iter -= n;
        ++iterdivn;
        if (iterdivn >= maxitdivn) return 1;
      }
      // find diagonal block to work on
      smax = fabs(D_(M));
      int ll = 0;
      bool split = false;
      for (int lll = 1; lll <= M - 1; ++lll) {
        ll = M - lll;
        const double abss = fabs(D_(ll)), abse = fabs(E_(ll));
        if (abse <= thresh) { split = true; break; }
        smax = fmax(smax, fmax(abss, abse));
      }
      if (split) {
        E_(ll) = 0.0;
        if (ll == M - 1) { M -= 1; continue; }
      } else {
        ll = 0;
      }
      ll += 1;
      if (ll == M - 1) {
        double sigmn, sigmx, sinr, cosr, sinl, cosl;
        dlasv2(D_(M - 1), E_(M - 1), D_(M), &sigmn, &sigmx, &sinr, &cosr, &sinl, &cosl);
        D_(M - 1) = sigmx;
        E_(M - 1) = 0.0;
        D_(M) = sigmn;
        drot(ncvt, &VT[(M - 2)], ldvt, &VT[(M - 1)], ldvt, cosr, sinr);
        drot(nru, &U[(M - 2) * ldu], 1, &U[(M - 1) * ldu], 1, cosl, sinl);
        M -= 2;
        continue;
      }
      if (ll > oldm || M < oldll) {
        if (fabs(D_(ll)) >= fabs(D_(M))) idir = 1;
        else idir = 2;
      }
      bool restart = false;
      if (idir == 1) {
        if (fabs(E_(M - 1)) <= mul(fabs(tol), fabs(D_(M)))) { E_(M - 1) = 0.0; continue; }
        double mu = fabs(D_(ll));
        smin = mu;
        for (int lll = ll; lll <= M - 1; ++lll) {
          if (fabs(E_(lll)) <= mul(tol, mu)) { E_(lll) = 0.0; restart = true; break; }
          mu = mul(fabs(D_(lll + 1)), div(mu, add(mu, fabs(E_(lll)))));
          smin = fmin(smin, mu);
        }
      } else {
        if (fabs(E_(ll)) <= mul(fabs(tol), fabs(D_(ll)))) { E_(ll) = 0.0; continue; }
        double mu = fabs(D_(M));
        smin = mu;
        for (int lll = M - 1; lll >= ll; --lll) {
          if (fabs(E_(lll)) <= mul(tol, mu)) { E_(lll) = 0.0; restart = true; break; }
          mu = mul(fabs(D_(lll)), div(mu, add(mu, fabs(E_(lll)))));
          smin = fmin(smin, mu);
        }
      }
      if (restart) continue;
      oldll = ll;
      oldm = M;
      double shift, r;
      if (mul(mul((double)n, tol), div(smin, smax)) <= fmax(eps, mul(0.01, tol))) {
        shift = 0.0;
      } else {
        double sll;
        if (idir == 1) {
          sll = fabs(D_(ll));
          dlas2(D_(M - 1), E_(M - 1), D_(M), &shift, &r);
        } else {
          sll = fabs(D_(M));
          dlas2(D_(ll), E_(ll), D_(ll + 1), &shift, &r);
        }
        if (sll > 0.0) {
          const double q = div(shift, sll);
          if (mul(q, q) < eps) shift = 0.0;
        }
      }
      iter += M - ll;
      if (shift == 0.0) {
        if (idir == 1) {
          double cs = 1.0, oldcs = 1.0, sn = 0.0, oldsn = 0.0;
          for (int i = ll; i <= M - 1; ++i) {
            dlartg(mul(D_(i), cs), E_(i), &cs, &sn, &r);
            if (i > ll) E_(i - 1) = mul(oldsn, r);
            dlartg(mul(oldcs, r), mul(D_(i + 1), sn), &oldcs, &oldsn, &D_(i));
            work[i - ll] = cs;
            work[i - ll + nm1] = sn;
            work[i - ll + nm12] = oldcs;
            work[i - ll + nm13] = oldsn;
          }
          const double hh = mul(D_(M), cs);
          D_(M) = mul(hh, oldcs);
          E_(M - 1) = mul(hh, oldsn);
          dlasr(true, true, M - ll + 1, ncvt, &work[0], &work[n - 1], &VT[(ll - 1)], ldvt);
          dlasr(false, true, nru, M - ll + 1, &work[nm12], &work[nm13], &U[(ll - 1) * ldu], ldu);
          if (fabs(E_(M - 1)) <= thresh) E_(M - 1) = 0.0;
        } else {
          double cs = 1.0, oldcs = 1.0, sn = 0.0, oldsn = 0.0;
          for (int i = M; i >= ll + 1; --i) {
            dlartg(mul(D_(i), cs), E_(i - 1), &cs, &sn, &r);
            if (i < M) E_(i) = mul(oldsn, r);
            dlartg(mul(oldcs, r), mul(D_(i - 1), sn), &oldcs, &oldsn, &D_(i));
            work[i - ll - 1] = cs;
            work[i - ll - 1 + nm1] = -sn;
            work[i - ll - 1 + nm12] = oldcs;
            work[i - ll - 1 + nm13] = -oldsn;
          }
          const double hh = mul(D_(ll), cs);
          D_(ll) = mul(hh, oldcs);
          E_(ll) = mul(hh, oldsn);
          dlasr(true, false, M - ll + 1, ncvt, &work[nm12], &work[nm13], &VT[(ll - 1)], ldvt);
          dlasr(false, false, nru, M - ll + 1, &work[0], &work[n - 1], &U[(ll - 1) * ldu], ldu);
          if (fabs(E_(ll)) <= thresh) E_(ll) = 0.0;
        }
      } else {
        if (idir == 1) {
          double f = mul(sub(fabs(D_(ll)), shift), add(fsign(1.0, D_(ll)), div(shift, D_(ll))));
          double g = E_(ll);
          double cosr, sinr, cosl, sinl;
          for (int i = ll; i <= M - 1; ++i) {
            dlartg(f, g, &cosr, &sinr, &r);
            if (i > ll) E_(i - 1) = r;
            f = add(mul(cosr, D_(i)), mul(sinr, E_(i)));
            E_(i) = sub(mul(cosr, E_(i)), mul(sinr, D_(i)));
            g = mul(sinr, D_(i + 1));
            D_(i + 1) = mul(cosr, D_(i + 1));
            dlartg(f, g, &cosl, &sinl, &r);
            D_(i) = r;
            f = add(mul(cosl, E_(i)), mul(sinl, D_(i + 1)));
            D_(i + 1) = sub(mul(cosl, D_(i + 1)), mul(sinl, E_(i)));
            if (i < M - 1) {
              g = mul(sinl, E_(i + 1));
              E_(i + 1) = mul(cosl, E_(i + 1));
            }
            work[i - ll] = cosr;
            work[i - ll + nm1] = sinr;
            work[i - ll + nm12] = cosl;
            work[i - ll + nm13] = sinl;
          }
          E_(M - 1) = f;
          dlasr(true, true, M - ll + 1, ncvt, &work[0], &work[n - 1], &VT[(ll - 1)], ldvt);
          dlasr(false, true, nru, M - ll + 1, &work[nm12], &work[nm13], &U[(ll - 1) * ldu], ldu);
          if (fabs(E_(M - 1)) <= thresh) E_(M - 1) = 0.0;
        } else {
          double f = mul(sub(fabs(D_(M)), shift), add(fsign(1.0, D_(M)), div(shift, D_(M))));
          double g = E_(M - 1);
          double cosr, sinr, cosl, sinl;
          for (int i = M; i >= ll + 1; --i) {
            dlartg(f, g, &cosr, &sinr, &r);
            if (i < M) E_(i) = r;
            f = add(mul(cosr, D_(i)), mul(sinr, E_(i - 1)));
            E_(i - 1) = sub(mul(cosr, E_(i - 1)), mul(sinr, D_(i)));
            g = mul(sinr, D_(i - 1));
            D_(i - 1) = mul(cosr, D_(i - 1));
            dlartg(f, g, &cosl, &sinl, &r);
            D_(i) = r;
            f = add(mul(cosl, E_(i - 1)), mul(sinl, D_(i - 1)));
            D_(i - 1) = sub(mul(cosl, D_(i - 1)), mul(sinl, E_(i - 1)));
            if (i > ll + 1) {
              g = mul(sinl, E_(i - 2));
              E_(i - 2) = mul(cosl, E_(i - 2));
            }
            work[i - ll - 1] = cosr;
            work[i - ll - 1 + nm1] = -sinr;
            work[i - ll - 1 + nm12] = cosl;
            work[i - ll - 1 + nm13] = -sinl;
          }
          E_(ll) = f;
          if (fabs(E_(ll)) <= thresh) E_(ll) = 0.0;
          dlasr(true, false, M - ll + 1, ncvt, &work[nm12], &work[nm13], &VT[(ll - 1)], ldvt);
          dlasr(false, false, nru, M - ll + 1, &work[0], &work[n - 1], &U[(ll - 1) * ldu], ldu);
        }
      }
    }
#undef D_
#undef E_
  }
  // make singular values positive
  for (int i = 0; i < n; ++i) {
    if (d[i] < 0.0) {
      d[i] = -d[i];
      dscal(ncvt, -1.0, &VT[i], ldvt);
    }
  }
  // sort into decreasing order
  for (int i = 1; i <= n - 1; ++i) {
    int isub = 1;
    double smin = d[0];
    for (int j = 2; j <= n + 1 - i; ++j) {
      if (d[j - 1] <= smin) { isub = j; smin = d[j - 1]; }
    }
    if (isub != n + 1 - i) {
      d[isub - 1] = d[n - i];
      d[n - i] = smin;
      dswap(ncvt, &VT[isub - 1], ldvt, &VT[n - i], ldvt);
      dswap(nru, &U[(isub - 1) * ldu], 1, &U[(n - i) * ldu], 1);
    }
  }
  return 0;
}

// dbdsdc('U', 'I', n): identity U, VT, then dlasdq -> dbdsqr, then the
// selection sort of dlasdq / dbdsdc (no-ops on dbdsqr's sorted output unless
// values tie, which the same code then resolves identically).
// ---- n = 3, every array in registers ---------------------------------------
// dbdsqr / dbdsdc above specialised for the fit's 3 x 3 bidiagonal: for n = 3
// the only QR sweep is over the whole matrix (ll = 1, M = 3 -- a 2 x 2 block
// goes to dlasv2), so every index is a compile-time constant and d, e, U, VT
// stay in registers instead of local memory.  Same operations in the same
// order as the generic code (tests/test_fit_parity.py checks both against
// OpenBLAS).  U, VT column-major, ld = 3.

// dlasr('L', 'V', direct, 3, 3, c, s, A, 3): rotations j = 0, 1 on rows (j, j+1)
template <bool FORWARD>
VK_HD void dlasr3_left(const double* c, const double* s, double* A) {
#pragma unroll
  for (int jj = 0; jj < 2; ++jj) {
    const int j = FORWARD ? jj : 1 - jj;
    const double ct = c[j], st = s[j];
    if (ct != 1.0 || st != 0.0) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double temp = A[(j + 1) + i * 3];
        A[(j + 1) + i * 3] = sub(mul(ct, temp), mul(st, A[j + i * 3]));
        A[j + i * 3] = add(mul(st, temp), mul(ct, A[j + i * 3]));
      }
    }
  }
}

// dlasr('R', 'V', direct, 3, 3, c, s, A, 3): rotations j = 0, 1 on columns (j, j+1)
template <bool FORWARD>
VK_HD void dlasr3_right(const double* c, const double* s, double* A) {
#pragma unroll
  for (int jj = 0; jj < 2; ++jj) {
    const int j = FORWARD ? jj : 1 - jj;
    const double ct = c[j], st = s[j];
    if (ct != 1.0 || st != 0.0) {
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double temp = A[i + (j + 1) * 3];
        A[i + (j + 1) * 3] = sub(mul(ct, temp), mul(st, A[i + j * 3]));
        A[i + j * 3] = add(mul(st, temp), mul(ct, A[i + j * 3]));
      }
    }
  }
}

// rows a, b of VT (drot over the 3 columns) and columns a, b of U
template <int A_, int B_>
VK_HD void rot3_rows(double* VT, double c, double s) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double xi = VT[A_ + i * 3], yi = VT[B_ + i * 3];
    VT[A_ + i * 3] = fma_(c, xi, mul(s, yi));
    VT[B_ + i * 3] = fma_(c, yi, -mul(s, xi));
  }
}
template <int A_, int B_>
VK_HD void rot3_cols(double* U, double c, double s) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const double xi = U[i + A_ * 3], yi = U[i + B_ * 3];
    U[i + A_ * 3] = fma_(c, xi, mul(s, yi));
    U[i + B_ * 3] = fma_(c, yi, -mul(s, xi));
  }
}
template <int A_, int B_>
VK_HD void swap3_rows(double* VT) {
#pragma unroll
  for (int i = 0; i < 3; ++i) { const double t = VT[A_ + i * 3]; VT[A_ + i * 3] = VT[B_ + i * 3]; VT[B_ + i * 3] = t; }
}
template <int A_, int B_>
VK_HD void swap3_cols(double* U) {
#pragma unroll
  for (int i = 0; i < 3; ++i) { const double t = U[i + A_ * 3]; U[i + A_ * 3] = U[i + B_ * 3]; U[i + B_ * 3] = t; }
}

// swap d[a], d[b] (a < b), rows a, b of VT and columns a, b of U; a, b runtime
// in {0, 1, 2}, dispatched to constant indices
VK_HD void sv3_swap(int a, int b, double* d, double* VT, double* U, bool vt_first) {
  auto sw = [&](auto ca, auto cb) {
    constexpr int A_ = decltype(ca)::value, B_ = decltype(cb)::value;
    if (vt_first) { swap3_rows<A_, B_>(VT); swap3_cols<A_, B_>(U); }
    else { swap3_cols<A_, B_>(U); swap3_rows<A_, B_>(VT); }
  };
  if (a == 0 && b == 1) sw(std::integral_constant<int, 0>{}, std::integral_constant<int, 1>{});
  else if (a == 0 && b == 2) sw(std::integral_constant<int, 0>{}, std::integral_constant<int, 2>{});
  else sw(std::integral_constant<int, 1>{}, std::integral_constant<int, 2>{});
  (void)d;
}

VK_HD double sel3(const double* d, int i) { return i == 0 ? d[0] : (i == 1 ? d[1] : d[2]); }
VK_HD void put3(double* d, int i, double v) {
  if (i == 0) d[0] = v;
  else if (i == 1) d[1] = v;
  else d[2] = v;
}

VK_HD int dbdsdc3(double* dio, double* eio, double* Uo, double* VTo) {
  double d[3] = {dio[0], dio[1], dio[2]};
  double e[2] = {eio[0], eio[1]};
  double U[9], VT[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) { U[i] = (i % 4 == 0) ? 1.0 : 0.0; VT[i] = U[i]; }
  const int n = 3;
  const double eps = DL_EPS, unfl = DL_SFMIN;
  const int maxitr = 6;
  const double tolmul = 0x1.8ace5422aa0dbp+6;
  const double tol = mul(tolmul, eps);
  double smax = 0.0;
  for (int i = 0; i < 3; ++i) smax = fmax(smax, fabs(d[i]));
  for (int i = 0; i < 2; ++i) smax = fmax(smax, fabs(e[i]));
  double smin = 0.0, thresh;
  {
    double sminoa = fabs(d[0]);
    if (sminoa != 0.0) {
      double mu = sminoa;
#pragma unroll
      for (int i = 1; i < 3; ++i) {
        mu = mul(fabs(d[i]), div(mu, add(mu, fabs(e[i - 1]))));
        sminoa = fmin(sminoa, mu);
        if (sminoa == 0.0) break;
      }
    }
    sminoa = div(sminoa, sqrt_((double)n));
    thresh = fmax(mul(tol, sminoa), mul((double)maxitr, mul((double)n, mul((double)n, unfl))));
  }
  const int maxitdivn = maxitr * n;
  int iterdivn = 0, iter = -1, oldll = -1, oldm = -1, idir = 0;
  int M = 3;
  while (true) {
    if (M <= 1) break;
    if (iter >= n) {
      iter -= n;
      ++iterdivn;
      if (iterdivn >= maxitdivn) return 1;
    }
    // find the diagonal block: M in {2, 3}
    int ll = 0;
    bool split = false;
    if (M == 3) {
      smax = fabs(d[2]);
      if (fabs(e[1]) <= thresh) { ll = 2; split = true; }
      else {
        smax = fmax(smax, fmax(fabs(d[1]), fabs(e[1])));
        if (fabs(e[0]) <= thresh) { ll = 1; split = true; }
        else smax = fmax(smax, fmax(fabs(d[0]), fabs(e[0])));
      }
    } else {
      smax = fabs(d[1]);
      if (fabs(e[0]) <= thresh) { ll = 1; split = true; }
      else smax = fmax(smax, fmax(fabs(d[0]), fabs(e[0])));
    }
    if (split) {
      if (ll == 1) e[0] = 0.0; else e[1] = 0.0;
      if (ll == M - 1) { M -= 1; continue; }
    } else {
      ll = 0;
    }
    ll += 1;
    if (ll == M - 1) {
      double sigmn, sigmx, sinr, cosr, sinl, cosl;
      if (M == 3) {
        dlasv2(d[1], e[1], d[2], &sigmn, &sigmx, &sinr, &cosr, &sinl, &cosl);
        d[1] = sigmx; e[1] = 0.0; d[2] = sigmn;
        rot3_rows<1, 2>(VT, cosr, sinr);
        rot3_cols<1, 2>(U, cosl, sinl);
      } else {
        dlasv2(d[0], e[0], d[1], &sigmn, &sigmx, &sinr, &cosr, &sinl, &cosl);
        d[0] = sigmx; e[0] = 0.0; d[1] = sigmn;
        rot3_rows<0, 1>(VT, cosr, sinr);
        rot3_cols<0, 1>(U, cosl, sinl);
      }
      M -= 2;
      continue;
    }
    // here ll = 1, M = 3: the whole matrix
    if (ll > oldm || M < oldll) {
      if (fabs(d[0]) >= fabs(d[2])) idir = 1;
      else idir = 2;
    }
    bool restart = false;
    if (idir == 1) {
      if (fabs(e[1]) <= mul(fabs(tol), fabs(d[2]))) { e[1] = 0.0; continue; }
      double mu = fabs(d[0]);
      smin = mu;
      if (fabs(e[0]) <= mul(tol, mu)) { e[0] = 0.0; restart = true; }
      else {
        mu = mul(fabs(d[1]), div(mu, add(mu, fabs(e[0]))));
        smin = fmin(smin, mu);
        if (fabs(e[1]) <= mul(tol, mu)) { e[1] = 0.0; restart = true; }
        else {
          mu = mul(fabs(d[2]), div(mu, add(mu, fabs(e[1]))));
          smin = fmin(smin, mu);
        }
      }
    } else {
      if (fabs(e[0]) <= mul(fabs(tol), fabs(d[0]))) { e[0] = 0.0; continue; }
      double mu = fabs(d[2]);
      smin = mu;
      if (fabs(e[1]) <= mul(tol, mu)) { e[1] = 0.0; restart = true; }
      else {
        mu = mul(fabs(d[1]), div(mu, add(mu, fabs(e[1]))));
        smin = fmin(smin, mu);
        if (fabs(e[0]) <= mul(tol, mu)) { e[0] = 0.0; restart = true; }
        else {
          mu = mul(fabs(d[0]), div(mu, add(mu, fabs(e[0]))));
          smin = fmin(smin, mu);
        }
      }
    }
    if (restart) continue;
    oldll = ll;
    oldm = M;
    double shift, r;
    if (mul(mul((double)n, tol), div(smin, smax)) <= fmax(eps, mul(0.01, tol))) {
      shift = 0.0;
    } else {
      double sll;
      if (idir == 1) {
        sll = fabs(d[0]);
        dlas2(d[1], e[1], d[2], &shift, &r);
      } else {
        sll = fabs(d[2]);
        dlas2(d[0], e[0], d[1], &shift, &r);
      }
      if (sll > 0.0) {
        const double q = div(shift, sll);
        if (mul(q, q) < eps) shift = 0.0;
      }
    }
    iter += M - ll;
    double work[8];                                   // [cs 0..1 | sn | oldcs | oldsn], n - 1 = 2 each
    if (shift == 0.0) {
      if (idir == 1) {
        double cs = 1.0, oldcs = 1.0, sn = 0.0, oldsn = 0.0;
        dlartg(mul(d[0], cs), e[0], &cs, &sn, &r);
        dlartg(mul(oldcs, r), mul(d[1], sn), &oldcs, &oldsn, &d[0]);
        work[0] = cs; work[2] = sn; work[4] = oldcs; work[6] = oldsn;
        dlartg(mul(d[1], cs), e[1], &cs, &sn, &r);
        e[0] = mul(oldsn, r);
        dlartg(mul(oldcs, r), mul(d[2], sn), &oldcs, &oldsn, &d[1]);
        work[1] = cs; work[3] = sn; work[5] = oldcs; work[7] = oldsn;
        const double hh = mul(d[2], cs);
        d[2] = mul(hh, oldcs);
        e[1] = mul(hh, oldsn);
        dlasr3_left<true>(&work[0], &work[2], VT);
        dlasr3_right<true>(&work[4], &work[6], U);
        if (fabs(e[1]) <= thresh) e[1] = 0.0;
      } else {
        double cs = 1.0, oldcs = 1.0, sn = 0.0, oldsn = 0.0;
        dlartg(mul(d[2], cs), e[1], &cs, &sn, &r);
        dlartg(mul(oldcs, r), mul(d[1], sn), &oldcs, &oldsn, &d[2]);
        work[1] = cs; work[3] = -sn; work[5] = oldcs; work[7] = -oldsn;
        dlartg(mul(d[1], cs), e[0], &cs, &sn, &r);
        e[1] = mul(oldsn, r);
        dlartg(mul(oldcs, r), mul(d[0], sn), &oldcs, &oldsn, &d[1]);
        work[0] = cs; work[2] = -sn; work[4] = oldcs; work[6] = -oldsn;
        const double hh = mul(d[0], cs);
        d[0] = mul(hh, oldcs);
        e[0] = mul(hh, oldsn);
        dlasr3_left<false>(&work[4], &work[6], VT);
        dlasr3_right<false>(&work[0], &work[2], U);
        if (fabs(e[0]) <= thresh) e[0] = 0.0;
      }
    } else {
      if (idir == 1) {
        double f = mul(sub(fabs(d[0]), shift), add(fsign(1.0, d[0]), div(shift, d[0])));
        double g = e[0];
        double cosr, sinr, cosl, sinl;
        // i = 1
        dlartg(f, g, &cosr, &sinr, &r);
        f = add(mul(cosr, d[0]), mul(sinr, e[0]));
        e[0] = sub(mul(cosr, e[0]), mul(sinr, d[0]));
        g = mul(sinr, d[1]);
        d[1] = mul(cosr, d[1]);
        dlartg(f, g, &cosl, &sinl, &r);
        d[0] = r;
        f = add(mul(cosl, e[0]), mul(sinl, d[1]));
        d[1] = sub(mul(cosl, d[1]), mul(sinl, e[0]));
        g = mul(sinl, e[1]);
        e[1] = mul(cosl, e[1]);
        work[0] = cosr; work[2] = sinr; work[4] = cosl; work[6] = sinl;
        // i = 2
        dlartg(f, g, &cosr, &sinr, &r);
        e[0] = r;
        f = add(mul(cosr, d[1]), mul(sinr, e[1]));
        e[1] = sub(mul(cosr, e[1]), mul(sinr, d[1]));
        g = mul(sinr, d[2]);
        d[2] = mul(cosr, d[2]);
        dlartg(f, g, &cosl, &sinl, &r);
        d[1] = r;
        f = add(mul(cosl, e[1]), mul(sinl, d[2]));
        d[2] = sub(mul(cosl, d[2]), mul(sinl, e[1]));
        work[1] = cosr; work[3] = sinr; work[5] = cosl; work[7] = sinl;
        e[1] = f;
        dlasr3_left<true>(&work[0], &work[2], VT);
        dlasr3_right<true>(&work[4], &work[6], U);
        if (fabs(e[1]) <= thresh) e[1] = 0.0;
      } else {
        double f = mul(sub(fabs(d[2]), shift), add(fsign(1.0, d[2]), div(shift, d[2])));
        double g = e[1];
        double cosr, sinr, cosl, sinl;
        // i = 3
        dlartg(f, g, &cosr, &sinr, &r);
        f = add(mul(cosr, d[2]), mul(sinr, e[1]));
        e[1] = sub(mul(cosr, e[1]), mul(sinr, d[2]));
        g = mul(sinr, d[1]);
        d[1] = mul(cosr, d[1]);
        dlartg(f, g, &cosl, &sinl, &r);
        d[2] = r;
        f = add(mul(cosl, e[1]), mul(sinl, d[1]));
        d[1] = sub(mul(cosl, d[1]), mul(sinl, e[1]));
        g = mul(sinl, e[0]);
        e[0] = mul(cosl, e[0]);
        work[1] = cosr; work[3] = -sinr; work[5] = cosl; work[7] = -sinl;
        // i = 2
        dlartg(f, g, &cosr, &sinr, &r);
        e[1] = r;
        f = add(mul(cosr, d[1]), mul(sinr, e[0]));
        e[0] = sub(mul(cosr, e[0]), mul(sinr, d[1]));
        g = mul(sinr, d[0]);
        d[0] = mul(cosr, d[0]);
        dlartg(f, g, &cosl, &sinl, &r);
        d[1] = r;
        f = add(mul(cosl, e[0]), mul(sinl, d[0]));
        d[0] = sub(mul(cosl, d[0]), mul(sinl, e[0]));
        work[0] = cosr; work[2] = -sinr; work[4] = cosl; work[6] = -sinl;
        e[0] = f;
        if (fabs(e[0]) <= thresh) e[0] = 0.0;
        dlasr3_left<false>(&work[4], &work[6], VT);
        dlasr3_right<false>(&work[0], &work[2], U);
      }
    }
  }
  // make singular values positive
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (d[i] < 0.0) {
      d[i] = -d[i];
#pragma unroll
      for (int c = 0; c < 3; ++c) VT[i + c * 3] = mul(VT[i + c * 3], -1.0);
    }
  }
  // dbdsqr: sort into decreasing order (insertion of the minimum at the end)
  for (int i = 1; i <= 2; ++i) {
    int isub = 1;
    double smn = d[0];
    for (int j = 2; j <= 4 - i; ++j) {
      const double dj = sel3(d, j - 1);
      if (dj <= smn) { isub = j; smn = dj; }
    }
    if (isub != 4 - i) {
      put3(d, isub - 1, sel3(d, 3 - i));
      put3(d, 3 - i, smn);
      sv3_swap(isub - 1, 3 - i, d, VT, U, true);
    }
  }
  // dbdsdc: dlasdq sort (ascending scan, swap to the end)
  for (int i = 1; i <= 3; ++i) {
    int isub = i;
    double smn = sel3(d, i - 1);
    for (int j = i + 1; j <= 3; ++j) {
      const double dj = sel3(d, j - 1);
      if (dj < smn) { isub = j; smn = dj; }
    }
    if (isub != 4 - i) {
      put3(d, isub - 1, sel3(d, 3 - i));
      put3(d, 3 - i, smn);
      const int a = isub - 1 < 3 - i ? isub - 1 : 3 - i, b = isub - 1 < 3 - i ? 3 - i : isub - 1;
      sv3_swap(a, b, d, VT, U, true);
    }
  }
  // dbdsdc: selection sort into decreasing order
  for (int ii = 2; ii <= 3; ++ii) {
    const int i = ii - 1;
    int kk = i;
    double p = sel3(d, i - 1);
    for (int j = ii; j <= 3; ++j) {
      const double dj = sel3(d, j - 1);
      if (dj > p) { kk = j; p = dj; }
    }
    if (kk != i) {
      put3(d, kk - 1, sel3(d, i - 1));
      put3(d, i - 1, p);
      sv3_swap(i - 1, kk - 1, d, VT, U, false);
    }
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) dio[i] = d[i];
  eio[0] = e[0];
  eio[1] = e[1];
#pragma unroll
  for (int i = 0; i < 9; ++i) { Uo[i] = U[i]; VTo[i] = VT[i]; }
  return 0;
}

VK_HDN int dbdsdc(int n, double* d, double* e, double* U, int ldu, double* VT, int ldvt) {
  if (n == 3 && ldu == 3 && ldvt == 3) return dbdsdc3(d, e, U, VT);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      U[i + j * ldu] = (i == j) ? 1.0 : 0.0;
      VT[i + j * ldvt] = (i == j) ? 1.0 : 0.0;
    }
  const int info = dbdsqr(n, d, e, VT, ldvt, U, ldu);
  if (info) return info;
  // dlasdq sort (ascending scan, swap to the end)
  for (int i = 1; i <= n; ++i) {
    int isub = i;
    double smin = d[i - 1];
    for (int j = i + 1; j <= n; ++j)
      if (d[j - 1] < smin) { isub = j; smin = d[j - 1]; }
    if (isub != n + 1 - i) {
      d[isub - 1] = d[n - i];
      d[n - i] = smin;
      dswap(n, &VT[isub - 1], ldvt, &VT[n - i], ldvt);
      dswap(n, &U[(isub - 1) * ldu], 1, &U[(n - i) * ldu], 1);
    }
  }
  // dbdsdc selection sort into decreasing order
  for (int ii = 2; ii <= n; ++ii) {
    const int i = ii - 1;
    int kk = i;
    double p = d[i - 1];
    for (int j = ii; j <= n; ++j)
      if (d[j - 1] > p) { kk = j; p = d[j - 1]; }
    if (kk != i) {
      d[kk - 1] = d[i - 1];
      d[i - 1] = p;
      dswap(n, &U[(i - 1) * ldu], 1, &U[(kk - 1) * ldu], 1);
      dswap(n, &VT[i - 1], ldvt, &VT[kk - 1], ldvt);
    }
  }
  return 0;
}

// dorm2r('L', 'N', m, n, k, A, lda, tau, C, ldc): C := Q C
VK_HDN void dorm2r_ln(int m, int n, int k, double* A, int lda, const double* tau, double* C, int ldc) {
  for (int i = k - 1; i >= 0; --i) {
    const double aii = A[i + i * lda];
    A[i + i * lda] = 1.0;
    dlarf(true, m - i, n, &A[i + i * lda], 1, tau[i], &C[i], ldc);
    A[i + i * lda] = aii;
  }
}

// dorml2('R', 'N', m, n, k, A, lda, tau, C, ldc): C := C Q (Q from dgelqf rows)
VK_HDN void dorml2_rn(int m, int n, int k, double* A, int lda, const double* tau, double* C, int ldc) {
  for (int i = k - 1; i >= 0; --i) {
    const double aii = A[i + i * lda];
    A[i + i * lda] = 1.0;
    dlarf(false, m, n - i, &A[i + i * lda], lda, tau[i], &C[i * ldc], ldc);
    A[i + i * lda] = aii;
  }
}

// numpy.linalg.svd(A, full_matrices=False) for a row-major (M x 3) A, M >= 5.
// Outputs U row-major (M x 3), s (3), VT row-major (3 x 3).  Returns 0 on
// success, nonzero if dbdsqr did not converge (numpy raises LinAlgError).
VK_HDN int svd_m3(const double* A_rm, int M, double* U_rm, double* s, double* VT_rm) {
  const int N = 3;
  double A[GMAXM * 3];                                   // column-major, lda = M
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < N; ++c) A[r + c * M] = A_rm[r * N + c];
  double tau[3];
  dgeqr2(M, N, A, M, tau);
  double R[9];                                           // upper triangle, lda = 3
  for (int j = 0; j < N; ++j)
    for (int i = 0; i < N; ++i) R[i + j * N] = (i <= j) ? A[i + j * M] : 0.0;
  dorg2r(M, N, N, A, M, tau);
  double d[3], e[3], tauq[3], taup[3];
  dgebd2(N, N, R, N, d, e, tauq, taup);
  double Ub[9], VTb[9];
  const int info = dbdsdc(N, d, e, Ub, N, VTb, N);
  if (info) return info;
  dorm2r_ln(N, N, N, R, N, tauq, Ub, N);                 // dormbr('Q','L','N')
  dorml2_rn(N, N - 1, N - 1, &R[0 + 1 * N], N, taup, &VTb[0 + 1 * N], N);  // dormbr('P','R','T')
  // dgemm('N','N', M, 3, 3, 1, Q, Ub, 0, U): one FMA chain over k per element
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      double c = mul(A[i + 0 * M], Ub[0 + j * N]);
      c = fma_(A[i + 1 * M], Ub[1 + j * N], c);
      c = fma_(A[i + 2 * M], Ub[2 + j * N], c);
      U_rm[i * N + j] = c;
    }
  for (int i = 0; i < N; ++i) {
    s[i] = d[i];
    for (int j = 0; j < N; ++j) VT_rm[i * N + j] = VTb[i + j * N];
  }
  return 0;
}

}  // namespace lapack
}  // namespace vk
