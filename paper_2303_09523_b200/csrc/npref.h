// Floating-point primitives of the reference's fit, restated operation by
// operation so the device TRF (trf.h) reproduces scipy's iterates bit for bit.
//
// fit_variogram (kriging.py:311-324) runs numpy 2.3.5 + scipy 1.18.1 on
// OpenBLAS 0.3.30.  On the x86 hosts the reference was pinned on (AVX512_SKX)
// the arithmetic behind its lines is:
//   * np.exp on float64 arrays        -> Intel SVML __svml_exp8_ha (numpy
//     dispatches DOUBLE_exp to it on AVX512_SKX): 2^(j/16) table, 6-term
//     polynomial, reduction by a round-toward-zero fused multiply-add;
//   * np.dot(a, b), 1-D, n < 16       -> OpenBLAS ddot: sequential FMA chain;
//   * J.dot(s), J C-order (m, 3)      -> dgemv_t "m3 == 3" tail: per row
//     fma(a2, x2, fma(a0, x0, a1 * x1));
//   * J.T.dot(f), J F-order (m, 3)    -> dgemv_t SKYLAKEX: columns 0/1 through
//     dgemv_kernel_4x2 (two SSE lanes, even / odd rows, no FMA), column 2
//     through dgemv_kernel_4x1 (four lanes), then the m & 3 tail rows;
//   * A.dot(x), A F-order (3, M)      -> dgemv_n SKYLAKEX 3-row path: column
//     pairs fma(a_k, x_k, a_k+1 * x_k+1) added in order, tail columns by FMA;
//   * numpy elementwise ops           -> one IEEE rounding each (no FMA).
// Each model was derived from the shipped binaries and checked bit-exact on
// random inputs against numpy (tools/fit_parity.py, tests/test_fit_parity.py).
// On the device every product/sum that numpy rounds separately uses the
// explicit _rn intrinsics, so nvcc cannot contract it into an FMA.
#pragma once
#include <cstdint>
#include <cmath>
#include "vk_common.h"

namespace vk {
namespace np {

#if defined(__CUDA_ARCH__)
VK_HD double mul(double a, double b) { return __dmul_rn(a, b); }
VK_HD double add(double a, double b) { return __dadd_rn(a, b); }
VK_HD double sub(double a, double b) { return __dsub_rn(a, b); }
VK_HD double div(double a, double b) { return __ddiv_rn(a, b); }
VK_HD double sqrt_(double a) { return __dsqrt_rn(a); }
VK_HD double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }
#else
VK_HD double mul(double a, double b) { return a * b; }
VK_HD double add(double a, double b) { return a + b; }
VK_HD double sub(double a, double b) { return a - b; }
VK_HD double div(double a, double b) { return a / b; }
VK_HD double fma_(double a, double b, double c) { return std::fma(a, b, c); }
VK_HD double sqrt_(double a) { return std::sqrt(a); }
#endif

VK_HD double from_bits(uint64_t b) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)b);
#else
  double d;
  __builtin_memcpy(&d, &b, 8);
  return d;
#endif
}

// 2^(j/16) = T_HI[j] * (1 + T_LO[j]): T_HI the nearest double, T_LO the
// nearest double of the relative remainder (generated from exact powers).
static const double EXP_T_HI[16] = {
    0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
    0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0,
    0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
    0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0};
static const double EXP_T_LO[16] = {
    0x0.0p+0, 0x1.79aa65d837b6dp-54, -0x1.01b15eaa59348p-55, 0x1.68efde3a8a894p-54,
    0x1.34d754db0abb6p-55, 0x1.59f48a72a4c6dp-55, 0x1.690cebb7aafb0p-56, 0x1.063e1e21c5409p-54,
    -0x1.3b3efbf5e2228p-54, -0x1.b32dcb94da51dp-56, 0x1.db72fc1f0eab4p-55, 0x1.1affc2b91ce27p-56,
    0x1.c1a7792cb3387p-55, 0x1.36eae30af0cb3p-56, 0x1.4a385a63d07a7p-56, -0x1.ff7128fd391f0p-55};
#if defined(__CUDACC__)
__device__ __constant__ double EXP_T_HI_D[16] = {
    0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
    0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0,
    0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
    0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0};
__device__ __constant__ double EXP_T_LO_D[16] = {
    0x0.0p+0, 0x1.79aa65d837b6dp-54, -0x1.01b15eaa59348p-55, 0x1.68efde3a8a894p-54,
    0x1.34d754db0abb6p-55, 0x1.59f48a72a4c6dp-55, 0x1.690cebb7aafb0p-56, 0x1.063e1e21c5409p-54,
    -0x1.3b3efbf5e2228p-54, -0x1.b32dcb94da51dp-56, 0x1.db72fc1f0eab4p-55, 0x1.1affc2b91ce27p-56,
    0x1.c1a7792cb3387p-55, 0x1.36eae30af0cb3p-56, 0x1.4a385a63d07a7p-56, -0x1.ff7128fd391f0p-55};
#endif

// np.exp(x) for float64 as SVML exp8_ha computes it on the main path.
// out of line: called from the lane-parallel residual rows (measured on C4:
// fit 1.730 -> 1.705 ms; an out-of-line division measured 1.843 ms)
VK_HDC double exp_(double x) {
  const double L2E = 0x1.71547652b82fep+0;              // 1 / ln 2
  const double C1 = 0x1.62e42fefa39efp-1;               // ln 2, high part
  const double C2 = 0x1.abc9e3b39803fp-56;              // ln 2, low part
  const double P0 = 0x1.7411836940c04p-10, P1 = 0x1.1101cbbc265c0p-7,
               P2 = 0x1.55557242d68fep-5, P3 = 0x1.5555553939732p-3,
               P4 = 0x1.000000000d008p-1, P5 = 0x1.fffffffffff70p-1;
  if (!(fabs(x) < 0x1.61da04cbafe44p+9)) return exp(x);  // rare path: |x| >= 707.7
  // SVML rounds x*L2E + 1.5*2^48 toward zero: on that grid (2^-4) this is the
  // floor of 16 * (x*L2E), formed here from the exact product hi + lo
  const double hi = mul(x, L2E);
  const double lo = fma_(x, L2E, -hi);
  const double h16 = hi * 16.0;                         // exact (power of two)
  double f = floor(h16);
  if (f == h16 && lo < 0.0) f -= 1.0;
  const long long fi = (long long)f;
  const double N = f * 0.0625;                          // exact
  double R = fma_(-N, C1, x);
  R = fma_(-N, C2, R);
  const double R2 = mul(R, R);
  double a = fma_(R, P0, P1);
  const double b = fma_(R, P2, P3);
  const double c = fma_(R, P4, P5);
  a = fma_(R2, a, b);
  a = fma_(R2, a, c);
  const int j = (int)(fi & 15);
#if defined(__CUDA_ARCH__)
  const double th = EXP_T_HI_D[j], tl = EXP_T_LO_D[j];
#else
  const double th = EXP_T_HI[j], tl = EXP_T_LO[j];
#endif
  double res = fma_(a, R, tl);
  res = fma_(th, res, th);
  return scalbn(res, (int)(fi >> 4));                   // vscalefpd: 2^floor(N)
}

// x**3 (np.power; SVML pow8_ha is within half an ulp of the exact cube
// except near ties): the correctly rounded cube from an exact x*x split.
VK_HD double cube(double x) {
  const double h2 = mul(x, x);
  const double l2 = fma_(x, x, -h2);
  const double p1 = mul(h2, x);
  const double e1 = fma_(h2, x, -p1);
  return add(p1, fma_(l2, x, e1));
}

// np.dot(a, b) for 1-D float64, n < 16 (OpenBLAS ddot tail loop).
VK_HD double dot(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s = fma_(a[i], b[i], s);
  return s;
}

// numpy.linalg.norm(x) = sqrt(x.dot(x)).
VK_HD double norm(const double* a, int n) { return sqrt_(dot(a, a, n)); }

// J.dot(s) row r for a C-contiguous (m, 3) J.
VK_HD double row3(const double* a, const double* x) {
  return fma_(a[2], x[2], fma_(a[0], x[0], mul(a[1], x[1])));
}

// Column `col` of J.T.dot(f) for an F-contiguous (M, 3) J: a = J[:, col].
VK_HD double colT(const double* a, const double* x, int M, int col) {
  const int m3 = M & 3, nb = M - m3;
  double y = 0.0;
  if (nb > 0) {
    if (col < 2) {                                      // dgemv_kernel_4x2
      double e = 0.0, o = 0.0;
      for (int i = 0; i < nb; i += 2) {
        e = add(e, mul(a[i], x[i]));
        o = add(o, mul(a[i + 1], x[i + 1]));
      }
      y = add(e, o);
    } else {                                            // dgemv_kernel_4x1
      double l0 = 0.0, l1 = 0.0, l2 = 0.0, l3 = 0.0;
      for (int i = 0; i < nb; i += 4) {
        l0 = add(l0, mul(a[i], x[i]));
        l1 = add(l1, mul(a[i + 1], x[i + 1]));
        l2 = add(l2, mul(a[i + 2], x[i + 2]));
        l3 = add(l3, mul(a[i + 3], x[i + 3]));
      }
      y = add(add(l0, l2), add(l1, l3));
    }
  }
  const double* at = a + nb;
  const double* xt = x + nb;
  if (m3 == 3) y = add(y, fma_(at[2], xt[2], fma_(at[0], xt[0], mul(at[1], xt[1]))));
  if (m3 == 2) y = add(y, fma_(at[0], xt[0], mul(at[1], xt[1])));
  if (m3 == 1) y = fma_(at[0], xt[0], y);
  return y;
}

// Row i of A.dot(x) for an F-contiguous (3, M) A given as its row a[k*sa].
VK_HD double rowN(const double* a, int sa, const double* x, int M) {
  double y = 0.0;
  int r = 0;
  for (; r + 4 <= M; r += 4) {
    y = add(y, fma_(a[r * sa], x[r], mul(a[(r + 1) * sa], x[r + 1])));
    y = add(y, fma_(a[(r + 2) * sa], x[r + 2], mul(a[(r + 3) * sa], x[r + 3])));
  }
  for (; r < M; ++r) y = fma_(a[r * sa], x[r], y);
  return y;
}

}  // namespace np
}  // namespace vk
