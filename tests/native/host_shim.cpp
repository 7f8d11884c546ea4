// TEST-ONLY host build of the header-only pieces of the device code (PCG64
// pair sampling, TRF fit) so tests/ can check them against numpy/scipy on a
// machine without a GPU.  Never linked into the product library.
#include <cstdint>
#include <vector>
#include "pcg64.h"
#include "trf.h"
#include <cstdio>
#include <string>

using namespace vk;

extern "C" {

void vkh_pcg_state(uint64_t seed, uint64_t* out4) {
  Pcg64 g = pcg64_from_seed(seed);
  out4[0] = (uint64_t)(g.state >> 64); out4[1] = (uint64_t)g.state;
  out4[2] = (uint64_t)(g.inc >> 64);   out4[3] = (uint64_t)g.inc;
}

uint64_t vkh_raw(uint64_t seed, uint64_t r) { return pcg_raw_at(pcg64_from_seed(seed), r); }

// Draw 2*n Lemire-bounded integers in [0, m) as the compaction of accepted
// 32-bit halves (what the device kernel computes in parallel).
int vkh_draws(uint64_t seed, uint32_t m, int64_t n, int64_t* out) {
  Pcg64 g = pcg64_from_seed(seed);
  const uint32_t thr = lemire_threshold(m);
  int64_t k = 0;
  u128 st = g.state;
  while (k < 2 * n) {
    st = st * pcg_mult() + g.inc;
    const uint64_t raw = pcg_output(st);
    const uint32_t halves[2] = {(uint32_t)raw, (uint32_t)(raw >> 32)};
    for (int h = 0; h < 2 && k < 2 * n; ++h) {
      const uint64_t prod = (uint64_t)halves[h] * m;
      if ((uint32_t)prod >= thr) out[k++] = (int64_t)(prod >> 32);
    }
  }
  return 0;
}

int vkh_trf(int kind, int nb, const double* h, const double* gemp, const double* w,
            const double* x0, const double* lb, const double* ub, double* x_out,
            int32_t* info) {
  TrfProblem P;
  P.kind = kind; P.nb = nb;
  for (int i = 0; i < nb; ++i) { P.h[i] = h[i]; P.gemp[i] = gemp[i]; P.w[i] = w[i]; }
  TrfResult r = trf_fit(P, x0, lb, ub);
  for (int i = 0; i < 3; ++i) x_out[i] = r.x[i];
  info[0] = r.status; info[1] = r.nfev; info[2] = r.iterations;
  return r.status;
}

}

// ---- geometry (vk_geometry.cpp compiled into this test shim) --------------
#include "vk_geometry.h"

extern "C" {

// Returns 0 on success, 1 on error (message copied to err).  Outputs:
// info[0..5] = n_miss, n_patterns, n_stencils, fast, G, n_systems
// miss_z[n_miss], miss_planes[n_miss*8], pat_off[n_patterns*8] (pad 99),
// pat_n[n_patterns], st[n_stencils*5] = (pattern, ky, kx, n, drift_cols)
int vkh_geometry(int H, int W, int T, const int* known_z, int K, int S, int drift,
                 int32_t* info, int32_t* miss_z, int32_t* miss_planes, int32_t* pat_off,
                 int32_t* pat_n, int32_t* st, char* err, int errlen) {
  vk::Geometry g;
  std::string e = vk::build_geometry(H, W, T, known_z, K, S, 0, drift, &g);
  if (!e.empty()) {
    snprintf(err, errlen, "%s", e.c_str());
    return 1;
  }
  info[0] = (int)g.miss_z.size();
  info[1] = (int)g.patterns.size();
  info[2] = (int)g.stencils.size();
  info[3] = g.fast ? 1 : 0;
  info[4] = g.G;
  info[5] = (int)g.sys_part.size();
  for (size_t i = 0; i < g.miss_z.size(); ++i) {
    miss_z[i] = g.miss_z[i];
    for (int k = 0; k < vk::NPMAX; ++k) miss_planes[i * 8 + k] = g.miss_planes[i * vk::NPMAX + k];
  }
  for (size_t p = 0; p < g.patterns.size(); ++p) {
    pat_n[p] = (int)g.patterns[p].size();
    for (int k = 0; k < 8; ++k) pat_off[p * 8 + k] = k < (int)g.patterns[p].size() ? g.patterns[p][k] : 99;
  }
  for (size_t i = 0; i < g.stencils.size(); ++i) {
    st[i * 5 + 0] = g.stencils[i].pattern;
    st[i * 5 + 1] = g.stencils[i].ky;
    st[i * 5 + 2] = g.stencils[i].kx;
    st[i * 5 + 3] = g.stencils[i].n;
    st[i * 5 + 4] = g.stencils[i].drift_cols;
  }
  return 0;
}

}

extern "C" {

// Orbit reduction of the stencil systems (vk_geometry.cpp canonical_systems).
// n_out[0] = systems, n_out[1] = derived; sys[n*4] = (part, pattern, ky, kx)
// in the reordered list; src[n], flags[n]; canon[S]; pat_off[NP*8] (pad 99).
int vkh_orbits(int H, int W, int T, const int* known_z, int K, int S, int drift, int32_t* n_out,
               int32_t* sys, int32_t* src, int32_t* flags, int32_t* canon, int32_t* pat_off) {
  vk::Geometry g;
  if (!vk::build_geometry(H, W, T, known_z, K, S, 0, drift, &g).empty()) return 1;
  std::vector<int> sc;
  std::vector<int32_t> ds, df;
  int nd = 0;
  vk::canonical_systems(&g, &sc, &ds, &df, &nd);
  const int n = (int)g.sys_part.size();
  n_out[0] = n;
  n_out[1] = nd;
  for (int i = 0; i < n; ++i) {
    const vk::StencilGeom& sg = g.stencils[g.sys_stencil[i]];
    sys[i * 4 + 0] = g.sys_part[i];
    sys[i * 4 + 1] = sg.pattern;
    sys[i * 4 + 2] = sg.ky;
    sys[i * 4 + 3] = sg.kx;
    src[i] = ds[i];
    flags[i] = df[i];
  }
  for (int s2 = 0; s2 < g.S; ++s2) canon[s2] = sc[s2];
  for (size_t p = 0; p < g.patterns.size(); ++p)
    for (int k = 0; k < 8; ++k) pat_off[p * 8 + k] = k < (int)g.patterns[p].size() ? g.patterns[p][k] : 99;
  return 0;
}

}

// ---- TRF pieces exposed for the fit-parity tests --------------------------
extern "C" {

// svd_aug of an (M x 3) row-major matrix: U (M x 3), s (3), VT (3 x 3) as numpy.linalg.svd returns them
void vkh_svd_aug(const double* A, int M, double* U, double* s, double* VT) {
  double V[9];
  vk::svd_aug(A, M, U, s, V);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) VT[k * 3 + i] = V[i * 3 + k];
}

void vkh_np_exp(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) y[i] = vk::np::exp_(x[i]);
}

}
extern "C" void vkh_cube(const double* x, double* y, long n) {
  for (long i = 0; i < n; ++i) y[i] = vk::np::cube(x[i]);
}

// ---- LAPACK / BLAS restatements of gesdd.h (checked against the shipped OpenBLAS) ----
#include "gesdd.h"
extern "C" {
double vkl_dnrm2(int n, const double* x, int incx) { return vk::lapack::dnrm2(n, x, incx); }
void vkl_dlarfg(int n, double* alpha, double* x, int incx, double* tau) { vk::lapack::dlarfg(n, alpha, x, incx, tau); }
void vkl_dlarf(int left, int m, int n, const double* v, int incv, double tau, double* C, int ldc) { vk::lapack::dlarf(left != 0, m, n, v, incv, tau, C, ldc); }
void vkl_dgeqr2(int m, int n, double* A, int lda, double* tau) { vk::lapack::dgeqr2(m, n, A, lda, tau); }
void vkl_dorg2r(int m, int n, int k, double* A, int lda, const double* tau) { vk::lapack::dorg2r(m, n, k, A, lda, tau); }
void vkl_dgebd2(int m, int n, double* A, int lda, double* d, double* e, double* tq, double* tp) { vk::lapack::dgebd2(m, n, A, lda, d, e, tq, tp); }
void vkl_dlartg(double f, double g, double* c, double* s, double* r) { vk::lapack::dlartg(f, g, c, s, r); }
void vkl_dlas2(double f, double g, double h, double* a, double* b) { vk::lapack::dlas2(f, g, h, a, b); }
void vkl_dlasv2(double f, double g, double h, double* o) { vk::lapack::dlasv2(f, g, h, o, o + 1, o + 2, o + 3, o + 4, o + 5); }
int vkl_dbdsqr(int n, double* d, double* e, double* VT, int ldvt, double* U, int ldu) { return vk::lapack::dbdsqr(n, d, e, VT, ldvt, U, ldu); }
int vkl_dbdsdc(int n, double* d, double* e, double* U, int ldu, double* VT, int ldvt) { return vk::lapack::dbdsdc(n, d, e, U, ldu, VT, ldvt); }
int vkl_svd_m3(const double* A, int M, double* U, double* s, double* VT) { return vk::lapack::svd_m3(A, M, U, s, VT); }
void vkl_drot(int n, double* x, int incx, double* y, int incy, double c, double s) { vk::lapack::drot(n, x, incx, y, incy, c, s); }
void vkl_dger(int m, int n, double alpha, const double* x, const double* y, int incy, double* A, int lda) { vk::lapack::dger(m, n, alpha, x, y, incy, A, lda); }
void vkl_dgemv_t(int m, int n, const double* A, int lda, const double* x, double* y) { vk::lapack::dgemv_t(m, n, A, lda, x, y); }
void vkl_dgemv_n(int m, int n, const double* A, int lda, const double* x, int incx, double* y) { vk::lapack::dgemv_n(m, n, A, lda, x, incx, y); }
}

// ---- numpy pairwise-summation tree (npsum.h) ----
#include "npsum.h"
extern "C" {
// numpy's sum of a[0:n] evaluated over the host-built tree; returns nleaf
double vkh_npsum_tree(const double* a, int64_t n, int32_t* nleaf_out) {
  const vk::NpSumTreeHost t = vk::build_npsum_tree(n);
  const int nleaf = (int)t.leaf_off.size() - 1;
  const int nnode = (int)t.node_lr.size() / 2;
  std::vector<double> v(nleaf + nnode);
  for (int l = 0; l < nleaf; ++l) {
    const int64_t o = t.leaf_off[l], m = t.leaf_off[l + 1] - o;
    const double* x = a + o;
    double res;
    if (m < 8) {
      res = -0.0;
      for (int64_t i = 0; i < m; ++i) res += x[i];
    } else {
      double r[8];
      for (int k = 0; k < 8; ++k) r[k] = x[k];
      int64_t i = 8;
      for (; i < m - m % 8; i += 8)
        for (int k = 0; k < 8; ++k) r[k] += x[i + k];
      res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
      for (; i < m; ++i) res += x[i];
    }
    v[l] = res;
  }
  for (int lev = 0; lev + 1 < (int)t.level.size(); ++lev)
    for (int j = t.level[lev]; j < t.level[lev + 1]; ++j)
      v[nleaf + j] = v[t.node_lr[2 * j]] + v[t.node_lr[2 * j + 1]];
  if (nleaf_out) *nleaf_out = nleaf;
  return nnode ? v[nleaf + nnode - 1] : v[0];
}
// the device's warp decomposition (build_npsum_warp) evaluated on the host:
// true leaves, then each warp root's program, then the top tree; returns the
// number of warp roots in *nwr_out
static double npsum_leaf(const double* x, int64_t m) {
  if (m < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < m; ++i) res += x[i];
    return res;
  }
  double r[8];
  for (int k = 0; k < 8; ++k) r[k] = x[k];
  int64_t i = 8;
  for (; i < m - m % 8; i += 8)
    for (int k = 0; k < 8; ++k) r[k] += x[i + k];
  double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < m; ++i) res += x[i];
  return res;
}
double vkh_npsum_warp(const double* a, int64_t n, int32_t* nwr_out) {
  const vk::NpSumWarpHost w = vk::build_npsum_warp(n);
  const int nwr = (int)w.wr_leaf.size() - 1;
  std::vector<double> root(nwr);
  for (int r = 0; r < nwr; ++r) {
    double val[64];
    const int l0 = w.wr_leaf[r], nl = w.wr_leaf[r + 1] - l0;
    if (nl > 32 || w.nint[r] != nl - 1) return NAN;
    for (int i = 0; i < nl; ++i) {
      const int64_t o = w.leaf_off[l0 + i];
      val[i] = npsum_leaf(a + o, w.leaf_off[l0 + i + 1] - o);
    }
    for (int j = 0; j < w.nint[r]; ++j) {
      const int code = (uint16_t)w.prog[(size_t)r * 31 + j];
      val[32 + j] = val[code & 0xff] + val[code >> 8];
    }
    root[r] = w.nint[r] ? val[32 + w.nint[r] - 1] : val[0];
  }
  const vk::NpSumTreeHost& t = w.top;
  const int nnode = (int)t.node_lr.size() / 2;
  std::vector<double> v(nwr + nnode);
  for (int r = 0; r < nwr; ++r) v[r] = root[r];
  for (int lev = 0; lev + 1 < (int)t.level.size(); ++lev)
    for (int j = t.level[lev]; j < t.level[lev + 1]; ++j)
      v[nwr + j] = v[t.node_lr[2 * j]] + v[t.node_lr[2 * j + 1]];
  if (nwr_out) *nwr_out = nwr;
  return nnode ? v[nwr + nnode - 1] : v[0];
}
}
