// Bounded Trust Region Reflective least squares for the 3-parameter
// variogram fit of fit_variogram (kriging.py:311-328), restated so that the
// device reproduces the reference's iterates.
//
// The reference calls scipy.optimize.least_squares(resid, x0, bounds,
// method="trf") with scipy's defaults: jac="2-point" (one-sided steps adjusted
// to the bounds), x_scale=1, tr_solver="exact", ftol=xtol=gtol=1e-8,
// max_nfev=100*n.  This header restates that published algorithm (Branch,
// Coleman & Li 1999 as implemented in scipy 1.18 optimize/_lsq/trf.py
// trf_bounds/select_step, _lsq/common.py and _numdiff.py) for n = 3 unknowns
// and at most MAX_BINS residuals, statement by statement, with every numpy
// reduction and BLAS call in the order the reference's numpy/OpenBLAS compute
// it (npref.h).
// numpy.linalg.svd of the augmented Jacobian is LAPACK dgesdd, restated with
// its BLAS kernels in gesdd.h (svd_aug, a one-sided Jacobi SVD, only serves
// the degenerate M < 5 case that takes another dgesdd path).
//
// trf_fit_t is templated on an evaluator that supplies the residuals and the
// finite-difference Jacobian, so the host (one thread, TrfScalarEval) and the
// device (one warp, residual rows on lanes; trf_warp.cuh) run the same code.
#pragma once
#include <cstdint>
#include <cmath>
#include "vk_common.h"
#include "npref.h"
#include "gesdd.h"

namespace vk {

struct TrfProblem {
  int kind;
  int nb;                    // residuals = non-empty bins
  double h[MAX_BINS];        // bin centres
  double gemp[MAX_BINS];     // empirical semivariance per bin
  double w[MAX_BINS];        // sqrt(count)
};

struct TrfResult {
  double x[3];
  int status;                // scipy status: 0 max_nfev, 1 gtol, 2 ftol, 3 xtol, 4 both; <0 error
  int nfev;
  int iterations;
};

constexpr double TRF_EPS = 2.220446049250313e-16;   // np.finfo(float).eps
constexpr int TRF_MAXM = MAX_BINS + 3;              // rows of the augmented Jacobian

// The TRF's row-length arrays.  The evaluator owns them: the host evaluator
// as a member, the device warp in shared memory -- every lane stores the same
// bits, so each lane reads back its own store or an identical one, and the
// 32 lanes share one copy instead of 32 copies of local memory (~100 KB per
// warp, more than the L1 left beside a fit's shared-memory reservation).
struct TrfWork {
  double f[MAX_BINS], J[MAX_BINS * 3], Ja[TRF_MAXM * 3], U[TRF_MAXM * 3];
  double f_new[MAX_BINS], fa[TRF_MAXM];
  double q1[MAX_BINS], q2[MAX_BINS];   // evaluate_quadratic / build_quadratic_1d rows
  double J_new[MAX_BINS * 3];          // Jacobian at the trial point (speculative)
};

VK_HD bool finite_d(double v) { return v - v == 0.0; }

VK_HD double pymax(double a, double b) { return (b > a) ? b : a; }  // Python max(a, b)

// One residual of kriging.py:311-319 in numpy's arithmetic:
//   mdl = VariogramModel(kind, max(nug,0), max(nug,0) + max(psill,0), max(r,1e-6))
//   gamma = nugget + (sill - nugget) * shape(h)        (kriging.py:59-72)
//   resid = bin_w * (gamma - bin_gamma)
// x -> (nugget, sill, range) is resolved once per evaluation by the caller.
struct FitModel {
  double nugget, psill, range_len;
};

VK_HD FitModel fit_model(const double* x) {
  FitModel m;
  m.nugget = pymax(x[0], 0.0);
  const double sill = np::add(m.nugget, pymax(x[1], 0.0));
  m.psill = np::sub(sill, m.nugget);
  m.range_len = pymax(x[2], 1e-6);
  return m;
}

template <int KIND>
VK_HD double fit_residual(const FitModel& m, double h, double gemp, double w) {
  double shape;
  if constexpr (KIND == KIND_EXPONENTIAL) {
    shape = np::sub(1.0, np::exp_(np::div(np::mul(-3.0, h), m.range_len)));
  } else if constexpr (KIND == KIND_GAUSSIAN) {
    const double t = np::div(h, m.range_len);
    shape = np::sub(1.0, np::exp_(np::mul(-3.0, np::mul(t, t))));
  } else {
    const double t = fmin(np::div(h, m.range_len), 1.0);
    shape = np::sub(np::mul(1.5, t), np::mul(0.5, np::cube(t)));
  }
  const double g = (h == 0.0) ? 0.0 : np::add(m.nugget, np::mul(m.psill, shape));
  return np::mul(w, np::sub(g, gemp));
}

VK_HD double fit_residual_kind(int kind, const FitModel& m, double h, double gemp, double w) {
  if (kind == KIND_GAUSSIAN) return fit_residual<KIND_GAUSSIAN>(m, h, gemp, w);
  if (kind == KIND_SPHERICAL) return fit_residual<KIND_SPHERICAL>(m, h, gemp, w);
  return fit_residual<KIND_EXPONENTIAL>(m, h, gemp, w);
}

// _numdiff.py _compute_absolute_step + _adjust_scheme_to_bounds('1-sided')
// for the 2-point scheme: the step of parameter i.
VK_HD double fd_step(const double* x, const double* lb, const double* ub, int i) {
  const double rstep = 1.4901161193847656e-08;   // EPS ** 0.5
  const double sign = (x[i] >= 0.0) ? 1.0 : -1.0;
  double h = np::mul(rstep * sign, fmax(1.0, fabs(x[i])));
  const double lower_dist = np::sub(x[i], lb[i]), upper_dist = np::sub(ub[i], x[i]);
  const double xt = np::add(x[i], h);
  const bool violated = (xt < lb[i]) || (xt > ub[i]);
  const bool fitting = fabs(h) <= fmax(lower_dist, upper_dist);
  if (violated && fitting) h = -h;
  if (!fitting) h = (upper_dist >= lower_dist) ? upper_dist : -lower_dist;
  return h;
}

// Host evaluator: residual rows and the 2-point Jacobian in a loop.
// J is stored column-major (J[c * m + r]): scipy's approx_derivative returns
// J_transposed.T, an F-contiguous (m, 3) array.
struct TrfScalarEval {
  const TrfProblem& P;
  mutable TrfWork wk;
  VK_HD explicit TrfScalarEval(const TrfProblem& p) : P(p) {}
  VK_HD TrfWork& work() const { return wk; }
  VK_HD int m() const { return P.nb; }
  VK_HD void resid(const double* x, double* f) const {
    const FitModel md = fit_model(x);
    for (int r = 0; r < P.nb; ++r) f[r] = fit_residual_kind(P.kind, md, P.h[r], P.gemp[r], P.w[r]);
  }
  // numpy.linalg.svd of the augmented Jacobian (gesdd.h)
  VK_HD int svd(const double* A, int M, double* U, double* s, double* VT) const {
    return lapack::svd_m3(A, M, U, s, VT);
  }
  // the residuals at a trial point and, speculatively, the Jacobian there
  // (used only if the step is accepted: then it is jac(x_new, f_new))
  VK_HD void resid_spec(const double* x, const double* lb, const double* ub, double* f, double* J) const {
    resid(x, f);
    jac(x, f, lb, ub, J);
  }
  VK_HD void jac(const double* x, const double* f0, const double* lb, const double* ub, double* J) const {
    double f1[MAX_BINS];
    for (int i = 0; i < 3; ++i) {
      const double h = fd_step(x, lb, ub, i);
      double x1[3] = {x[0], x[1], x[2]};
      x1[i] = np::add(x[i], h);
      resid(x1, f1);
      const double dx = np::sub(np::add(x[i], h), x[i]);
      for (int r = 0; r < P.nb; ++r) J[i * P.nb + r] = np::div(np::sub(f1[r], f0[r]), dx);
    }
  }
};

// Thin SVD of the (M x 3) augmented Jacobian A (row-major): A = U diag(s) V^T,
// s descending, U (M x 3, row-major), V (3 x 3, row-major: V[i*3+k] = V_ik).
// One-sided Jacobi on the columns of A (rotations until every pair is
// orthogonal to working precision), then normalised columns.
VK_HDC void svd_aug(const double* A, int M, double* U, double* s, double* V) {
  double B[TRF_MAXM * 3];
  for (int i = 0; i < M * 3; ++i) B[i] = A[i];
  for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < 2; ++p) {
      for (int q = p + 1; q < 3; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int r = 0; r < M; ++r) {
          const double a = B[r * 3 + p], b = B[r * 3 + q];
          alpha = np::fma_(a, a, alpha);
          beta = np::fma_(b, b, beta);
          gamma = np::fma_(a, b, gamma);
        }
        if (gamma == 0.0 || fabs(gamma) <= TRF_EPS * sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int r = 0; r < M; ++r) {
          const double a = B[r * 3 + p], b = B[r * 3 + q];
          B[r * 3 + p] = c * a - sn * b;
          B[r * 3 + q] = sn * a + c * b;
        }
        for (int r = 0; r < 3; ++r) {
          const double a = V[r * 3 + p], b = V[r * 3 + q];
          V[r * 3 + p] = c * a - sn * b;
          V[r * 3 + q] = sn * a + c * b;
        }
      }
    }
    if (!rotated) break;
  }
  double sv[3];
  for (int j = 0; j < 3; ++j) {
    double acc = 0.0;
    for (int r = 0; r < M; ++r) acc = np::fma_(B[r * 3 + j], B[r * 3 + j], acc);
    sv[j] = sqrt(acc);
  }
  int order[3] = {0, 1, 2};
  for (int a = 0; a < 3; ++a)
    for (int b = a + 1; b < 3; ++b)
      if (sv[order[b]] > sv[order[a]]) { const int t = order[a]; order[a] = order[b]; order[b] = t; }
  double Vs[9];
  for (int k = 0; k < 3; ++k) {
    const int j = order[k];
    s[k] = sv[j];
    for (int r = 0; r < 3; ++r) Vs[r * 3 + k] = V[r * 3 + j];
    for (int r = 0; r < M; ++r) U[r * 3 + k] = sv[j] > 0.0 ? B[r * 3 + j] / sv[j] : 0.0;
  }
  for (int i = 0; i < 9; ++i) V[i] = Vs[i];
}

// V.dot(x) for V = VT.T (F-contiguous 3x3): seq. FMA over k per row.
VK_HD void v_dot(const double* V, const double* x, double* y) {
  for (int i = 0; i < 3; ++i) y[i] = np::rowN(V + i * 3, 1, x, 3);
}

// common.py solve_lsq_trust_region (More's method on one SVD).
VK_HDN void lsq_trust_region(int m, const double* uf, const double* s, const double* V,
                            double Delta, double initial_alpha, double* p, double* alpha_out) {
  const int n = 3;
  double suf[3];
  for (int i = 0; i < 3; ++i) suf[i] = np::mul(s[i], uf[i]);
  bool full_rank = false;
  if (m >= n) full_rank = s[n - 1] > np::mul(TRF_EPS * m, s[0]);
  if (full_rank) {
    double t[3];
    for (int i = 0; i < 3; ++i) t[i] = np::div(uf[i], s[i]);
    v_dot(V, t, p);
    for (int i = 0; i < 3; ++i) p[i] = -p[i];
    if (np::norm(p, 3) <= Delta) { *alpha_out = 0.0; return; }
  }
  // phi_and_derivative
  auto phi_d = [&](double a, double& phi, double& dphi) {
    double q[3], r[3];
    for (int i = 0; i < 3; ++i) {
      const double den = np::add(np::mul(s[i], s[i]), a);
      q[i] = np::div(suf[i], den);
      r[i] = np::div(np::mul(suf[i], suf[i]), np::cube(den));
    }
    const double pn = np::norm(q, 3);
    phi = np::sub(pn, Delta);
    double sum = -0.0;                                   // np.sum, n < 8
    for (int i = 0; i < 3; ++i) sum = np::add(sum, r[i]);
    dphi = np::div(-sum, pn);
  };
  double alpha_upper = np::div(np::norm(suf, 3), Delta);
  double alpha_lower = 0.0;
  if (full_rank) {
    double phi, dphi;
    phi_d(0.0, phi, dphi);
    alpha_lower = np::div(-phi, dphi);
  }
  double alpha;
  if (!full_rank && initial_alpha == 0.0)
    alpha = pymax(np::mul(0.001, alpha_upper), np::sqrt_(np::mul(alpha_lower, alpha_upper)));
  else
    alpha = initial_alpha;
  for (int it = 0; it < 10; ++it) {
    if (alpha < alpha_lower || alpha > alpha_upper)
      alpha = pymax(np::mul(0.001, alpha_upper), np::sqrt_(np::mul(alpha_lower, alpha_upper)));
    double phi, dphi;
    phi_d(alpha, phi, dphi);
    if (phi < 0) alpha_upper = alpha;
    const double ratio = np::div(phi, dphi);
    alpha_lower = pymax(alpha_lower, np::sub(alpha, ratio));
    alpha = np::sub(alpha, np::div(np::mul(np::add(phi, Delta), ratio), Delta));
    if (fabs(phi) < np::mul(0.01, Delta)) break;
  }
  double t[3];
  for (int i = 0; i < 3; ++i) t[i] = np::div(suf[i], np::add(np::mul(s[i], s[i]), alpha));
  v_dot(V, t, p);
  for (int i = 0; i < 3; ++i) p[i] = -p[i];
  const double sc = np::div(Delta, np::norm(p, 3));
  for (int i = 0; i < 3; ++i) p[i] = np::mul(p[i], sc);
  *alpha_out = alpha;
}

VK_HD bool in_bounds3(const double* x, const double* lb, const double* ub) {
  for (int i = 0; i < 3; ++i)
    if (!(x[i] >= lb[i] && x[i] <= ub[i])) return false;
  return true;
}

// common.py step_size_to_bound
VK_HDN double step_to_bound(const double* x, const double* s, const double* lb,
                           const double* ub, int* hits) {
  double steps[3];
  double mn = INFINITY;
  for (int i = 0; i < 3; ++i) {
    steps[i] = INFINITY;
    if (s[i] != 0.0) {
      const double a = np::div(np::sub(lb[i], x[i]), s[i]);
      const double b = np::div(np::sub(ub[i], x[i]), s[i]);
      steps[i] = (a != a || b != b) ? NAN : (b > a ? b : a);   // np.maximum
    }
    mn = (i == 0) ? steps[0] : ((steps[i] < mn || steps[i] != steps[i]) ? steps[i] : mn);
  }
  for (int i = 0; i < 3; ++i)
    hits[i] = (steps[i] == mn) ? (s[i] > 0 ? 1 : (s[i] < 0 ? -1 : 0)) : 0;
  return mn;
}

// common.py intersect_trust_region: roots t of ||x + s t|| = Delta
VK_HDN bool intersect_tr(const double* x, const double* s, double Delta, double* t_neg, double* t_pos) {
  const double a = np::dot(s, s, 3);
  if (a == 0.0) return false;
  const double b = np::dot(x, s, 3);
  const double c = np::sub(np::dot(x, x, 3), np::mul(Delta, Delta));
  if (c > 0.0) return false;
  const double d = np::sqrt_(np::sub(np::mul(b, b), np::mul(a, c)));
  const double q = -np::add(b, copysign(d, b));
  const double t1 = np::div(q, a), t2 = np::div(c, q);
  if (t1 < t2) { *t_neg = t1; *t_pos = t2; } else { *t_neg = t2; *t_pos = t1; }
  return true;
}

// J_h.dot(s) for the C-contiguous (m, 3) J_h = J_augmented[:m]
VK_HD void jh_dot(const double* Jh, int m, const double* s, double* out) {
  for (int r = 0; r < m; ++r) out[r] = np::row3(Jh + r * 3, s);
}

// common.py evaluate_quadratic (1-D s)
VK_HDN double eval_quad(const double* Jh, int m, const double* g, const double* s, const double* diag,
                        double* Js) {
  jh_dot(Jh, m, s, Js);
  double q = np::dot(Js, Js, m);
  double sd[3];
  for (int i = 0; i < 3; ++i) sd[i] = np::mul(s[i], diag[i]);
  q = np::add(q, np::dot(sd, s, 3));
  const double l = np::dot(s, g, 3);
  return np::add(np::mul(0.5, q), l);
}

// common.py build_quadratic_1d (with s0 when given)
VK_HDN void build_quad_1d(const double* Jh, int m, const double* g, const double* s,
                         const double* diag, const double* s0, double* a, double* b, double* c,
                         double* v, double* u) {
  jh_dot(Jh, m, s, v);
  double aa = np::dot(v, v, m);
  double sd[3];
  for (int i = 0; i < 3; ++i) sd[i] = np::mul(s[i], diag[i]);
  aa = np::add(aa, np::dot(sd, s, 3));
  aa = np::mul(aa, 0.5);
  double bb = np::dot(g, s, 3);
  double cc = 0.0;
  if (s0) {
    jh_dot(Jh, m, s0, u);
    bb = np::add(bb, np::dot(u, v, m));
    cc = np::add(np::mul(0.5, np::dot(u, u, m)), np::dot(g, s0, 3));
    double s0d[3];
    for (int i = 0; i < 3; ++i) s0d[i] = np::mul(s0[i], diag[i]);
    bb = np::add(bb, np::dot(s0d, s, 3));
    cc = np::add(cc, np::mul(0.5, np::dot(s0d, s0, 3)));
  }
  *a = aa; *b = bb; *c = cc;
}

// common.py minimize_quadratic_1d: y = t * (a * t + b) + c at lb, ub (and the
// interior extremum), first minimum as np.argmin
VK_HD void min_quad_1d(double a, double b, double lb, double ub, double c, double* t_out, double* y_out) {
  double t[3] = {lb, ub, 0.0};
  int nt = 2;
  if (a != 0.0) {
    const double ext = np::div(np::mul(-0.5, b), a);
    if (lb < ext && ext < ub) t[nt++] = ext;
  }
  int best = 0;
  double yb = np::add(np::mul(t[0], np::add(np::mul(a, t[0]), b)), c);
  for (int i = 1; i < nt; ++i) {
    const double y = np::add(np::mul(t[i], np::add(np::mul(a, t[i]), b)), c);
    if (y < yb) { yb = y; best = i; }
  }
  *t_out = t[best];
  *y_out = yb;
}

// trf.py select_step.  step/step_h out; returns predicted reduction; false on error.
VK_HDN bool select_step(const double* x, const double* Jh, int m, const double* diag_h,
                       const double* g_h, double* p, double* p_h, const double* d,
                       double Delta, const double* lb, const double* ub, double theta,
                       double* step, double* step_h, double* pred, TrfWork& w) {
  double xp[3];
  for (int i = 0; i < 3; ++i) xp[i] = np::add(x[i], p[i]);
  if (in_bounds3(xp, lb, ub)) {
    const double pv = eval_quad(Jh, m, g_h, p_h, diag_h, w.q1);
    for (int i = 0; i < 3; ++i) { step[i] = p[i]; step_h[i] = p_h[i]; }
    *pred = -pv;
    return true;
  }
  int hits[3];
  const double p_stride = step_to_bound(x, p, lb, ub, hits);
  double r_h[3], r[3];
  for (int i = 0; i < 3; ++i) {
    r_h[i] = p_h[i];
    if (hits[i] != 0) r_h[i] = -r_h[i];
    r[i] = np::mul(d[i], r_h[i]);
  }
  for (int i = 0; i < 3; ++i) { p[i] = np::mul(p[i], p_stride); p_h[i] = np::mul(p_h[i], p_stride); }
  double x_on_bound[3];
  for (int i = 0; i < 3; ++i) x_on_bound[i] = np::add(x[i], p[i]);
  double t_neg, to_tr;
  if (!intersect_tr(p_h, r_h, Delta, &t_neg, &to_tr)) return false;
  int hits2[3];
  const double to_bound = step_to_bound(x_on_bound, r, lb, ub, hits2);
  double r_stride = (to_tr < to_bound) ? to_tr : to_bound;          // min(to_bound, to_tr)
  double r_stride_l, r_stride_u;
  if (r_stride > 0) {
    r_stride_l = np::div(np::mul(np::sub(1.0, theta), p_stride), r_stride);
    if (r_stride == to_bound) r_stride_u = np::mul(theta, to_bound);
    else r_stride_u = to_tr;
  } else {
    r_stride_l = 0;
    r_stride_u = -1;
  }
  double r_value;
  if (r_stride_l <= r_stride_u) {
    double a, b, c;
    build_quad_1d(Jh, m, g_h, r_h, diag_h, p_h, &a, &b, &c, w.q1, w.q2);
    min_quad_1d(a, b, r_stride_l, r_stride_u, c, &r_stride, &r_value);
    for (int i = 0; i < 3; ++i) {
      r_h[i] = np::mul(r_h[i], r_stride);
      r_h[i] = np::add(r_h[i], p_h[i]);
      r[i] = np::mul(r_h[i], d[i]);
    }
  } else {
    r_value = INFINITY;
  }
  for (int i = 0; i < 3; ++i) { p[i] = np::mul(p[i], theta); p_h[i] = np::mul(p_h[i], theta); }
  const double p_value = eval_quad(Jh, m, g_h, p_h, diag_h, w.q1);
  double ag_h[3], ag[3];
  for (int i = 0; i < 3; ++i) { ag_h[i] = -g_h[i]; ag[i] = np::mul(d[i], ag_h[i]); }
  const double to_tr2 = np::div(Delta, np::norm(ag_h, 3));
  int hits3[3];
  const double to_bound2 = step_to_bound(x, ag, lb, ub, hits3);
  double ag_stride = (to_bound2 < to_tr2) ? np::mul(theta, to_bound2) : to_tr2;
  double a2, b2, c2;
  build_quad_1d(Jh, m, g_h, ag_h, diag_h, nullptr, &a2, &b2, &c2, w.q1, w.q2);
  double ag_value;
  min_quad_1d(a2, b2, 0.0, ag_stride, 0.0, &ag_stride, &ag_value);
  for (int i = 0; i < 3; ++i) { ag_h[i] = np::mul(ag_h[i], ag_stride); ag[i] = np::mul(ag[i], ag_stride); }
  if (p_value < r_value && p_value < ag_value) {
    for (int i = 0; i < 3; ++i) { step[i] = p[i]; step_h[i] = p_h[i]; }
    *pred = -p_value;
  } else if (r_value < p_value && r_value < ag_value) {
    for (int i = 0; i < 3; ++i) { step[i] = r[i]; step_h[i] = r_h[i]; }
    *pred = -r_value;
  } else {
    for (int i = 0; i < 3; ++i) { step[i] = ag[i]; step_h[i] = ag_h[i]; }
    *pred = -ag_value;
  }
  return true;
}

VK_HD double next_toward(double from, double to) {
#if defined(__CUDA_ARCH__)
  return ::nextafter(from, to);
#else
  return std::nextafter(from, to);
#endif
}

// common.py make_strictly_feasible (rstep > 0 uses the relative rule,
// rstep == 0 uses nextafter).
VK_HDN void make_strictly_feasible(double* x, const double* lb, const double* ub, double rstep) {
  for (int i = 0; i < 3; ++i) {
    int active = 0;
    if (rstep == 0.0) {
      if (x[i] <= lb[i]) active = -1;
      if (x[i] >= ub[i]) active = 1;
    } else {
      const double ld = np::sub(x[i], lb[i]), ud = np::sub(ub[i], x[i]);
      const double lt = np::mul(rstep, fmax(1.0, fabs(lb[i]))), ut = np::mul(rstep, fmax(1.0, fabs(ub[i])));
      if (ld <= fmin(ud, lt)) active = -1;
      if (ud <= fmin(ld, ut)) active = 1;
    }
    double xn = x[i];
    if (active == -1) xn = (rstep == 0.0) ? next_toward(lb[i], ub[i]) : np::add(lb[i], np::mul(rstep, fmax(1.0, fabs(lb[i]))));
    if (active == 1) xn = (rstep == 0.0) ? next_toward(ub[i], lb[i]) : np::sub(ub[i], np::mul(rstep, fmax(1.0, fabs(ub[i]))));
    if (xn < lb[i] || xn > ub[i]) xn = np::mul(0.5, np::add(lb[i], ub[i]));
    x[i] = xn;
  }
}

// compute_grad: J.T.dot(f) for the F-contiguous (m, 3) J (column-major here)
VK_HDN void trf_grad(const double* J, const double* f, int m, double* g) {
  for (int i = 0; i < 3; ++i) g[i] = np::colT(J + i * m, f, m, i);
}

// optional per-phase cycle counters of the device fit (-DVK_FIT_PROFILE,
// tools/fit_phase_profile.py): 0 resid, 1 jac+grad, 2 svd, 3 lsq, 4 select,
// 5 total, 6 iterations, 7 nfev
#if defined(VK_FIT_PROFILE) && defined(__CUDACC__)
__device__ unsigned long long g_fit_prof[16];
#endif
#if defined(VK_FIT_PROFILE) && defined(__CUDA_ARCH__)
#define VK_TP(v) const long long v = clock64()
#define VK_TACC(slot, a) if (threadIdx.x == 0) atomicAdd(&g_fit_prof[slot], (unsigned long long)(clock64() - (a)))
#define VK_TADD(slot, n) if (threadIdx.x == 0) atomicAdd(&g_fit_prof[slot], (unsigned long long)(n))
#else
#define VK_TP(v)
#define VK_TACC(slot, a)
#define VK_TADD(slot, n)
#endif

// trf.py trf_bounds with loss='linear', x_scale=1, tr_solver='exact'.
template <class Eval>
VK_HD TrfResult trf_fit_t(const Eval& ev, const double* x0_in, const double* lb, const double* ub) {
  VK_TP(t_all);
  const int m = ev.m();
  const double ftol = 1e-8, xtol = 1e-8, gtol = 1e-8;
  const int max_nfev = 300;
  TrfResult res;
  double x[3] = {x0_in[0], x0_in[1], x0_in[2]};
  make_strictly_feasible(x, lb, ub, 1e-10);      // least_squares.py: x0 strictly feasible
  TrfWork& w = ev.work();
  double* const f = w.f;
  double* const J = w.J;
  ev.resid(x, f);
  ev.jac(x, f, lb, ub, J);
  int nfev = 1;
  double cost = np::mul(0.5, np::dot(f, f, m));
  double g[3];
  trf_grad(J, f, m, g);
  double v[3], dv[3];
  auto cl_scaling = [&]() {
    for (int i = 0; i < 3; ++i) {
      v[i] = 1.0; dv[i] = 0.0;
      if (g[i] < 0 && finite_d(ub[i])) { v[i] = np::sub(ub[i], x[i]); dv[i] = -1.0; }
      if (g[i] > 0 && finite_d(lb[i])) { v[i] = np::sub(x[i], lb[i]); dv[i] = 1.0; }
    }
  };
  cl_scaling();
  double Delta;
  {
    double t[3];   // norm(x0 * scale_inv / v**0.5), x0 already strictly feasible
    for (int i = 0; i < 3; ++i) t[i] = np::div(x[i], np::sqrt_(v[i]));
    Delta = np::norm(t, 3);
    if (Delta == 0) Delta = 1.0;
  }
  double alpha = 0.0;
  int status = -100;       // None
  int iteration = 0;
  double* const Ja = w.Ja;
  double* const U = w.U;
  double* const f_new = w.f_new;
  double* const fa = w.fa;
  double sv[3], V[9];
  double x_new[3];
  double cost_new = 0.0;
  double g_norm = 0.0;
  const int M = m + 3;
  while (true) {
#ifdef TRF_DEBUG
    printf("it %d nfev %d cost %.17g x %.17g %.17g %.17g Delta %.17g alpha %.17g\n", iteration, nfev,
           cost, x[0], x[1], x[2], Delta, alpha);
#endif
    cl_scaling();
    g_norm = 0.0;
    for (int i = 0; i < 3; ++i) g_norm = pymax(g_norm, fabs(np::mul(g[i], v[i])));
    if (g_norm < gtol) status = 1;
    if (status != -100 || nfev == max_nfev) break;
    double d[3], diag_h[3], g_h[3];
    for (int i = 0; i < 3; ++i) {
      d[i] = np::sqrt_(v[i]);
      diag_h[i] = np::mul(g[i], dv[i]);
      g_h[i] = np::mul(d[i], g[i]);
    }
    // J_augmented = [J * d; diag(diag_h ** 0.5)], C-contiguous; J_h its first m rows
    for (int r = 0; r < m; ++r)
      for (int c = 0; c < 3; ++c) Ja[r * 3 + c] = np::mul(J[c * m + r], d[c]);
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) Ja[(m + r) * 3 + c] = (r == c) ? np::sqrt_(diag_h[r]) : 0.0;
    {
      double VT[9];
      VK_TP(t_svd);
      if (M < 5 || ev.svd(Ja, M, U, sv, VT) != 0) svd_aug(Ja, M, U, sv, V);
      else
        for (int i = 0; i < 3; ++i)
          for (int k = 0; k < 3; ++k) V[i * 3 + k] = VT[k * 3 + i];
      VK_TACC(2, t_svd);
    }
    for (int r = 0; r < M; ++r) fa[r] = r < m ? f[r] : 0.0;
    double uf[3];
    for (int c = 0; c < 3; ++c) uf[c] = np::rowN(U + c, 3, fa, M);   // U.T.dot(f_augmented)
    const double theta = pymax(0.995, np::sub(1.0, g_norm));
    double actual_reduction = -1;
    double step_norm = 0.0;
    while (actual_reduction <= 0 && nfev < max_nfev) {
      double p_h[3], p[3];
      VK_TP(t_lsq);
      lsq_trust_region(m, uf, sv, V, Delta, alpha, p_h, &alpha);
      VK_TACC(3, t_lsq);
      VK_TP(t_sel);
      for (int i = 0; i < 3; ++i) p[i] = np::mul(d[i], p_h[i]);
      double step[3], step_h[3], pred;
      const bool sel_ok = select_step(x, Ja, m, diag_h, g_h, p, p_h, d, Delta, lb, ub, theta, step, step_h, &pred, w);
      VK_TACC(4, t_sel);
      if (!sel_ok) {
        res.status = -1;
        res.nfev = nfev;
        res.iterations = iteration;
        for (int i = 0; i < 3; ++i) res.x[i] = x[i];
        return res;
      }
      for (int i = 0; i < 3; ++i) x_new[i] = np::add(x[i], step[i]);
      make_strictly_feasible(x_new, lb, ub, 0.0);
      VK_TP(t_res);
      // residuals at the trial point together with the Jacobian there: an
      // evaluator with spare lanes computes both in one round, and an
      // accepted step (most of them) then needs no Jacobian evaluation
      ev.resid_spec(x_new, lb, ub, f_new, w.J_new);
      VK_TACC(0, t_res);
      nfev += 1;
      const double step_h_norm = np::norm(step_h, 3);
      bool finite = true;
      for (int r = 0; r < m; ++r) finite = finite && finite_d(f_new[r]);
      if (!finite) { Delta = np::mul(0.25, step_h_norm); continue; }
      cost_new = np::mul(0.5, np::dot(f_new, f_new, m));
      actual_reduction = np::sub(cost, cost_new);
      // update_tr_radius
      double ratio;
      if (pred > 0) ratio = np::div(actual_reduction, pred);
      else if (pred == actual_reduction && pred == 0) ratio = 1;
      else ratio = 0;
      double Delta_new = Delta;
      if (ratio < 0.25) Delta_new = np::mul(0.25, step_h_norm);
      else if (ratio > 0.75 && step_h_norm > np::mul(0.95, Delta)) Delta_new = np::mul(Delta, 2.0);
      step_norm = np::norm(step, 3);
      // check_termination
      const bool ftol_ok = actual_reduction < np::mul(ftol, cost) && ratio > 0.25;
      const bool xtol_ok = step_norm < np::mul(xtol, np::add(xtol, np::norm(x, 3)));
      if (ftol_ok && xtol_ok) status = 4;
      else if (ftol_ok) status = 2;
      else if (xtol_ok) status = 3;
      if (status != -100) break;
      alpha = np::mul(alpha, np::div(Delta, Delta_new));
      Delta = Delta_new;
    }
    if (actual_reduction > 0) {
      for (int i = 0; i < 3; ++i) x[i] = x_new[i];
      for (int r = 0; r < m; ++r) f[r] = f_new[r];
      cost = cost_new;
      VK_TP(t_jac);
      for (int k = 0; k < 3 * m; ++k) J[k] = w.J_new[k];    // jac(x, f): evaluated with the step
      trf_grad(J, f, m, g);
      VK_TACC(1, t_jac);
    }
    iteration += 1;
  }
  if (status == -100) status = 0;
  for (int i = 0; i < 3; ++i) res.x[i] = x[i];
  res.status = status;
  res.nfev = nfev;
  res.iterations = iteration;
  VK_TACC(5, t_all);
  VK_TADD(6, iteration);
  VK_TADD(7, nfev);
  return res;
}

VK_HD TrfResult trf_fit(const TrfProblem& P, const double* x0_in, const double* lb, const double* ub) {
  TrfScalarEval ev(P);
  return trf_fit_t(ev, x0_in, lb, ub);
}

}  // namespace vk
