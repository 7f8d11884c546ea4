// Bounded Trust Region Reflective least squares for the 3-parameter
// variogram fit of fit_variogram (kriging.py:311-328).
//
// The reference calls scipy.optimize.least_squares(resid, x0, bounds,
// method="trf") with scipy's defaults: jac="2-point" (one-sided steps
// adjusted to the bounds), x_scale=1, tr_solver="exact", ftol=xtol=gtol=1e-8,
// max_nfev=100*n.  This header restates that published algorithm (Branch,
// Coleman & Li 1999 as implemented in scipy 1.18 optimize/_lsq/trf.py
// trf_bounds/select_step and _lsq/common.py helpers) for n = 3 unknowns and
// at most MAX_BINS residuals, so one thread can run it on the device and the
// same code can be checked on the host against scipy.  The SVD of the
// augmented Jacobian is a one-sided Jacobi SVD (scipy uses LAPACK gesdd); the
// trust-region step only depends on basis-independent products, so the two
// agree to rounding.
#pragma once
#include <cstdint>
#include <cmath>
#include "vk_common.h"

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

VK_HD bool finite_d(double v) { return v - v == 0.0; }

VK_HD double pymax(double a, double b) { return (b > a) ? b : a; }  // Python max(a, b)

// resid(params) of kriging.py:311-319: bin_w * (gamma_of(params, bin_h) - bin_gamma)
VK_HD void trf_residual(const TrfProblem& P, const double* x, double* f) {
  Model m;
  m.nugget = pymax(x[0], 0.0);
  m.sill = m.nugget + pymax(x[1], 0.0);
  m.range_len = pymax(x[2], 1e-6);
  for (int i = 0; i < P.nb; ++i)
    f[i] = P.w[i] * (semivariance(P.kind, m, P.h[i]) - P.gemp[i]);
}

VK_HD double vdot(const double* a, const double* b, int n) {
  double s = 0.0;
  for (int i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
VK_HD double vnorm(const double* a, int n) { return sqrt(vdot(a, a, n)); }

// J (m x 3, row-major) by '2-point' differences at x with f0 = f(x)
// (scipy _numdiff approx_derivative + _adjust_scheme_to_bounds '1-sided').
VK_HD void trf_jacobian(const TrfProblem& P, const double* x, const double* f0,
                        const double* lb, const double* ub, double* J) {
  const double rstep = 1.4901161193847656e-08;   // EPS ** 0.5
  double f1[MAX_BINS];
  for (int i = 0; i < 3; ++i) {
    const double sign = (x[i] >= 0.0) ? 1.0 : -1.0;
    double h = rstep * sign * fmax(1.0, fabs(x[i]));
    const double lower_dist = x[i] - lb[i], upper_dist = ub[i] - x[i];
    const double xt = x[i] + h;
    const bool violated = (xt < lb[i]) || (xt > ub[i]);
    const bool fitting = fabs(h) <= fmax(lower_dist, upper_dist);
    if (violated && fitting) h = -h;
    if (!fitting) h = (upper_dist >= lower_dist) ? upper_dist : -lower_dist;
    double x1[3] = {x[0], x[1], x[2]};
    x1[i] = x[i] + h;
    trf_residual(P, x1, f1);
    const double dx = (x[i] + h) - x[i];
    for (int r = 0; r < P.nb; ++r) J[r * 3 + i] = (f1[r] - f0[r]) / dx;
  }
}

// Thin SVD of an (mr x 3) row-major matrix: A = U diag(s) V^T, s descending.
VK_HD void svd3(const double* A, int mr, double* U, double* s, double* V) {
  double B[(MAX_BINS + 3) * 3];
  for (int i = 0; i < mr * 3; ++i) B[i] = A[i];
  for (int i = 0; i < 9; ++i) V[i] = (i % 4 == 0) ? 1.0 : 0.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < 2; ++p) {
      for (int q = p + 1; q < 3; ++q) {
        double alpha = 0.0, beta = 0.0, gamma = 0.0;
        for (int r = 0; r < mr; ++r) {
          const double a = B[r * 3 + p], b = B[r * 3 + q];
          alpha += a * a;
          beta += b * b;
          gamma += a * b;
        }
        if (gamma == 0.0 || fabs(gamma) <= TRF_EPS * sqrt(alpha * beta)) continue;
        rotated = true;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), sn = c * t;
        for (int r = 0; r < mr; ++r) {
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
    for (int r = 0; r < mr; ++r) acc += B[r * 3 + j] * B[r * 3 + j];
    sv[j] = sqrt(acc);
  }
  int order[3] = {0, 1, 2};
  for (int a = 0; a < 3; ++a)
    for (int b = a + 1; b < 3; ++b)
      if (sv[order[b]] > sv[order[a]]) { int t = order[a]; order[a] = order[b]; order[b] = t; }
  double Vs[9];
  for (int k = 0; k < 3; ++k) {
    const int j = order[k];
    s[k] = sv[j];
    for (int r = 0; r < 3; ++r) Vs[r * 3 + k] = V[r * 3 + j];
    for (int r = 0; r < mr; ++r) U[r * 3 + k] = sv[j] > 0.0 ? B[r * 3 + j] / sv[j] : 0.0;
  }
  for (int i = 0; i < 9; ++i) V[i] = Vs[i];
}

// common.py solve_lsq_trust_region (More's method on one SVD).
VK_HD void lsq_trust_region(int m, const double* uf, const double* s, const double* V,
                            double Delta, double initial_alpha, double* p, double* alpha_out) {
  const int n = 3;
  double suf[3];
  for (int i = 0; i < 3; ++i) suf[i] = s[i] * uf[i];
  bool full_rank = false;
  if (m >= n) full_rank = s[n - 1] > TRF_EPS * m * s[0];
  if (full_rank) {
    double t[3];
    for (int i = 0; i < 3; ++i) t[i] = uf[i] / s[i];
    for (int r = 0; r < 3; ++r) p[r] = -(V[r * 3 + 0] * t[0] + V[r * 3 + 1] * t[1] + V[r * 3 + 2] * t[2]);
    if (vnorm(p, 3) <= Delta) { *alpha_out = 0.0; return; }
  }
  auto phi_d = [&](double a, double& phi, double& dphi) {
    double q[3], s3 = 0.0;
    for (int i = 0; i < 3; ++i) {
      const double rden = 1.0 / (s[i] * s[i] + a);
      q[i] = suf[i] * rden;
      s3 += q[i] * q[i] * rden;                 // suf^2 / den^3
    }
    const double pn = vnorm(q, 3);
    phi = pn - Delta;
    dphi = -s3 / pn;
  };
  double alpha_upper = vnorm(suf, 3) / Delta;
  double alpha_lower = 0.0;
  if (full_rank) {
    double phi, dphi;
    phi_d(0.0, phi, dphi);
    alpha_lower = -phi / dphi;
  }
  double alpha;
  if (!full_rank && initial_alpha == 0.0)
    alpha = fmax(0.001 * alpha_upper, sqrt(alpha_lower * alpha_upper));
  else
    alpha = initial_alpha;
  for (int it = 0; it < 10; ++it) {
    if (alpha < alpha_lower || alpha > alpha_upper)
      alpha = fmax(0.001 * alpha_upper, sqrt(alpha_lower * alpha_upper));
    double phi, dphi;
    phi_d(alpha, phi, dphi);
    if (phi < 0) alpha_upper = alpha;
    const double ratio = phi / dphi;
    alpha_lower = fmax(alpha_lower, alpha - ratio);
    alpha -= (phi + Delta) * ratio / Delta;
    if (fabs(phi) < 0.01 * Delta) break;
  }
  double t[3];
  for (int i = 0; i < 3; ++i) t[i] = suf[i] / (s[i] * s[i] + alpha);
  for (int r = 0; r < 3; ++r) p[r] = -(V[r * 3 + 0] * t[0] + V[r * 3 + 1] * t[1] + V[r * 3 + 2] * t[2]);
  const double sc = Delta / vnorm(p, 3);
  for (int r = 0; r < 3; ++r) p[r] *= sc;
  *alpha_out = alpha;
}

VK_HD bool in_bounds3(const double* x, const double* lb, const double* ub) {
  for (int i = 0; i < 3; ++i)
    if (!(x[i] >= lb[i] && x[i] <= ub[i])) return false;
  return true;
}

// common.py step_size_to_bound
VK_HD double step_to_bound(const double* x, const double* s, const double* lb,
                           const double* ub, int* hits) {
  double steps[3];
  double mn = INFINITY;
  for (int i = 0; i < 3; ++i) {
    steps[i] = INFINITY;
    if (s[i] != 0.0) steps[i] = fmax((lb[i] - x[i]) / s[i], (ub[i] - x[i]) / s[i]);
    mn = fmin(mn, steps[i]);
  }
  for (int i = 0; i < 3; ++i)
    hits[i] = (steps[i] == mn) ? (s[i] > 0 ? 1 : (s[i] < 0 ? -1 : 0)) : 0;
  return mn;
}

// common.py intersect_trust_region: roots t of ||x + s t|| = Delta
VK_HD bool intersect_tr(const double* x, const double* s, double Delta, double* t_neg, double* t_pos) {
  const double a = vdot(s, s, 3);
  if (a == 0.0) return false;
  const double b = vdot(x, s, 3);
  const double c = vdot(x, x, 3) - Delta * Delta;
  if (c > 0.0) return false;
  const double d = sqrt(b * b - a * c);
  const double q = -(b + copysign(d, b));
  const double t1 = q / a, t2 = c / q;
  if (t1 < t2) { *t_neg = t1; *t_pos = t2; } else { *t_neg = t2; *t_pos = t1; }
  return true;
}

// J_h s for J_h = J * d (m x 3)
VK_HD void jh_dot(const double* Jh, int m, const double* s, double* out) {
  for (int r = 0; r < m; ++r)
    out[r] = Jh[r * 3 + 0] * s[0] + Jh[r * 3 + 1] * s[1] + Jh[r * 3 + 2] * s[2];
}

// common.py evaluate_quadratic
VK_HD double eval_quad(const double* Jh, int m, const double* g, const double* s, const double* diag) {
  double Js[MAX_BINS];
  jh_dot(Jh, m, s, Js);
  double q = vdot(Js, Js, m);
  double sd[3] = {s[0] * diag[0], s[1] * diag[1], s[2] * diag[2]};
  q += vdot(sd, s, 3);
  return 0.5 * q + vdot(s, g, 3);
}

// common.py build_quadratic_1d (with s0 when given)
VK_HD void build_quad_1d(const double* Jh, int m, const double* g, const double* s,
                         const double* diag, const double* s0, double* a, double* b, double* c) {
  double v[MAX_BINS];
  jh_dot(Jh, m, s, v);
  double aa = vdot(v, v, m);
  double sd[3] = {s[0] * diag[0], s[1] * diag[1], s[2] * diag[2]};
  aa += vdot(sd, s, 3);
  aa *= 0.5;
  double bb = vdot(g, s, 3);
  double cc = 0.0;
  if (s0) {
    double u[MAX_BINS];
    jh_dot(Jh, m, s0, u);
    bb += vdot(u, v, m);
    cc = 0.5 * vdot(u, u, m) + vdot(g, s0, 3);
    double s0d[3] = {s0[0] * diag[0], s0[1] * diag[1], s0[2] * diag[2]};
    bb += vdot(s0d, s, 3);
    cc += 0.5 * vdot(s0d, s0, 3);
  }
  *a = aa; *b = bb; *c = cc;
}

// common.py minimize_quadratic_1d
VK_HD void min_quad_1d(double a, double b, double lb, double ub, double c, double* t_out, double* y_out) {
  double t[3] = {lb, ub, 0.0};
  int nt = 2;
  if (a != 0.0) {
    const double ext = -0.5 * b / a;
    if (lb < ext && ext < ub) t[nt++] = ext;
  }
  int best = 0;
  double yb = t[0] * (a * t[0] + b) + c;
  for (int i = 1; i < nt; ++i) {
    const double y = t[i] * (a * t[i] + b) + c;
    if (y < yb) { yb = y; best = i; }
  }
  *t_out = t[best];
  *y_out = yb;
}

// trf.py select_step.  step/step_h out; returns predicted reduction; false on error.
VK_HD bool select_step(const double* x, const double* Jh, int m, const double* diag_h,
                       const double* g_h, double* p, double* p_h, const double* d,
                       double Delta, const double* lb, const double* ub, double theta,
                       double* step, double* step_h, double* pred) {
  double xp[3] = {x[0] + p[0], x[1] + p[1], x[2] + p[2]};
  if (in_bounds3(xp, lb, ub)) {
    const double pv = eval_quad(Jh, m, g_h, p_h, diag_h);
    for (int i = 0; i < 3; ++i) { step[i] = p[i]; step_h[i] = p_h[i]; }
    *pred = -pv;
    return true;
  }
  int hits[3];
  const double p_stride = step_to_bound(x, p, lb, ub, hits);
  double r_h[3], r[3];
  for (int i = 0; i < 3; ++i) {
    r_h[i] = p_h[i];
    if (hits[i] != 0) r_h[i] *= -1.0;
    r[i] = d[i] * r_h[i];
  }
  for (int i = 0; i < 3; ++i) { p[i] *= p_stride; p_h[i] *= p_stride; }
  double x_on_bound[3] = {x[0] + p[0], x[1] + p[1], x[2] + p[2]};
  double t_neg, to_tr;
  if (!intersect_tr(p_h, r_h, Delta, &t_neg, &to_tr)) return false;
  int hits2[3];
  const double to_bound = step_to_bound(x_on_bound, r, lb, ub, hits2);
  double r_stride = fmin(to_bound, to_tr);
  double r_stride_l, r_stride_u;
  if (r_stride > 0) {
    r_stride_l = (1 - theta) * p_stride / r_stride;
    if (r_stride == to_bound) r_stride_u = theta * to_bound;
    else r_stride_u = to_tr;
  } else {
    r_stride_l = 0;
    r_stride_u = -1;
  }
  double r_value;
  if (r_stride_l <= r_stride_u) {
    double a, b, c;
    build_quad_1d(Jh, m, g_h, r_h, diag_h, p_h, &a, &b, &c);
    min_quad_1d(a, b, r_stride_l, r_stride_u, c, &r_stride, &r_value);
    for (int i = 0; i < 3; ++i) {
      r_h[i] *= r_stride;
      r_h[i] += p_h[i];
      r[i] = r_h[i] * d[i];
    }
  } else {
    r_value = INFINITY;
  }
  for (int i = 0; i < 3; ++i) { p[i] *= theta; p_h[i] *= theta; }
  const double p_value = eval_quad(Jh, m, g_h, p_h, diag_h);
  double ag_h[3], ag[3];
  for (int i = 0; i < 3; ++i) { ag_h[i] = -g_h[i]; ag[i] = d[i] * ag_h[i]; }
  const double to_tr2 = Delta / vnorm(ag_h, 3);
  int hits3[3];
  const double to_bound2 = step_to_bound(x, ag, lb, ub, hits3);
  double ag_stride = (to_bound2 < to_tr2) ? theta * to_bound2 : to_tr2;
  double a2, b2, c2;
  build_quad_1d(Jh, m, g_h, ag_h, diag_h, nullptr, &a2, &b2, &c2);
  double ag_value;
  min_quad_1d(a2, b2, 0.0, ag_stride, 0.0, &ag_stride, &ag_value);
  for (int i = 0; i < 3; ++i) { ag_h[i] *= ag_stride; ag[i] *= ag_stride; }
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
VK_HD void make_strictly_feasible(double* x, const double* lb, const double* ub, double rstep) {
  for (int i = 0; i < 3; ++i) {
    int active = 0;
    if (rstep == 0.0) {
      if (x[i] <= lb[i]) active = -1;
      if (x[i] >= ub[i]) active = 1;
    } else {
      const double ld = x[i] - lb[i], ud = ub[i] - x[i];
      const double lt = rstep * fmax(1.0, fabs(lb[i])), ut = rstep * fmax(1.0, fabs(ub[i]));
      if (ld <= fmin(ud, lt)) active = -1;
      if (ud <= fmin(ld, ut)) active = 1;
    }
    double xn = x[i];
    if (active == -1) xn = (rstep == 0.0) ? next_toward(lb[i], ub[i]) : lb[i] + rstep * fmax(1.0, fabs(lb[i]));
    if (active == 1) xn = (rstep == 0.0) ? next_toward(ub[i], lb[i]) : ub[i] - rstep * fmax(1.0, fabs(ub[i]));
    if (xn < lb[i] || xn > ub[i]) xn = 0.5 * (lb[i] + ub[i]);
    x[i] = xn;
  }
}

// trf.py trf_bounds with loss='linear', x_scale=1, tr_solver='exact'.
VK_HD TrfResult trf_fit(const TrfProblem& P, const double* x0_in, const double* lb, const double* ub) {
  const int m = P.nb;
  const double ftol = 1e-8, xtol = 1e-8, gtol = 1e-8;
  const int max_nfev = 300;
  TrfResult res;
  double x[3] = {x0_in[0], x0_in[1], x0_in[2]};
  make_strictly_feasible(x, lb, ub, 1e-10);      // least_squares.py: x0 strictly feasible
  double f[MAX_BINS], J[MAX_BINS * 3];
  trf_residual(P, x, f);
  trf_jacobian(P, x, f, lb, ub, J);
  int nfev = 1;
  double cost = 0.5 * vdot(f, f, m);
  double g[3];
  for (int i = 0; i < 3; ++i) {
    double acc = 0.0;
    for (int r = 0; r < m; ++r) acc += J[r * 3 + i] * f[r];
    g[i] = acc;
  }
  double v[3], dv[3];
  auto cl_scaling = [&]() {
    for (int i = 0; i < 3; ++i) {
      v[i] = 1.0; dv[i] = 0.0;
      if (g[i] < 0 && finite_d(ub[i])) { v[i] = ub[i] - x[i]; dv[i] = -1.0; }
      if (g[i] > 0 && finite_d(lb[i])) { v[i] = x[i] - lb[i]; dv[i] = 1.0; }
    }
  };
  cl_scaling();
  double Delta;
  {
    double t[3];   // norm(x0 * scale_inv / v**0.5), x0 already strictly feasible
    for (int i = 0; i < 3; ++i) t[i] = x[i] * 1.0 / sqrt(v[i]);
    Delta = vnorm(t, 3);
    if (Delta == 0) Delta = 1.0;
  }
  double alpha = 0.0;
  int status = -100;       // None
  int iteration = 0;
  double Jh[MAX_BINS * 3], Ja[(MAX_BINS + 3) * 3], U[(MAX_BINS + 3) * 3], sv[3], V[9];
  double x_new[3], f_new[MAX_BINS];
  double cost_new = 0.0;
  double g_norm = 0.0;
  while (true) {
#ifdef TRF_DEBUG
    printf("it %d nfev %d cost %.10e x %.17g %.17g %.17g\n", iteration, nfev, cost, x[0], x[1], x[2]);
#endif
    cl_scaling();
    g_norm = 0.0;
    for (int i = 0; i < 3; ++i) g_norm = fmax(g_norm, fabs(g[i] * v[i]));
    if (g_norm < gtol) status = 1;
    if (status != -100 || nfev == max_nfev) break;
    double d[3], diag_h[3], g_h[3];
    for (int i = 0; i < 3; ++i) {
      d[i] = sqrt(v[i]);
      diag_h[i] = g[i] * dv[i];
      g_h[i] = d[i] * g[i];
    }
    for (int r = 0; r < m; ++r)
      for (int c = 0; c < 3; ++c) {
        Jh[r * 3 + c] = J[r * 3 + c] * d[c];
        Ja[r * 3 + c] = Jh[r * 3 + c];
      }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) Ja[(m + r) * 3 + c] = (r == c) ? sqrt(diag_h[r]) : 0.0;
    svd3(Ja, m + 3, U, sv, V);
    double uf[3];
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;
      for (int r = 0; r < m; ++r) acc += U[r * 3 + c] * f[r];
      uf[c] = acc;
    }
    const double theta = fmax(0.995, 1 - g_norm);
    double actual_reduction = -1;
    double step_norm = 0.0;
    while (actual_reduction <= 0 && nfev < max_nfev) {
      double p_h[3], p[3];
      lsq_trust_region(m, uf, sv, V, Delta, alpha, p_h, &alpha);
      for (int i = 0; i < 3; ++i) p[i] = d[i] * p_h[i];
      double step[3], step_h[3], pred;
      if (!select_step(x, Jh, m, diag_h, g_h, p, p_h, d, Delta, lb, ub, theta, step, step_h, &pred)) {
        res.status = -1;
        res.nfev = nfev;
        res.iterations = iteration;
        for (int i = 0; i < 3; ++i) res.x[i] = x[i];
        return res;
      }
      for (int i = 0; i < 3; ++i) x_new[i] = x[i] + step[i];
      make_strictly_feasible(x_new, lb, ub, 0.0);
      trf_residual(P, x_new, f_new);
      nfev += 1;
      const double step_h_norm = vnorm(step_h, 3);
      bool finite = true;
      for (int r = 0; r < m; ++r) finite = finite && finite_d(f_new[r]);
      if (!finite) { Delta = 0.25 * step_h_norm; continue; }
      cost_new = 0.5 * vdot(f_new, f_new, m);
      actual_reduction = cost - cost_new;
      // update_tr_radius
      double ratio;
      if (pred > 0) ratio = actual_reduction / pred;
      else if (pred == actual_reduction && pred == 0) ratio = 1;
      else ratio = 0;
      double Delta_new = Delta;
      if (ratio < 0.25) Delta_new = 0.25 * step_h_norm;
      else if (ratio > 0.75 && step_h_norm > 0.95 * Delta) Delta_new = Delta * 2.0;
      step_norm = vnorm(step, 3);
      // check_termination
      const bool ftol_ok = actual_reduction < ftol * cost && ratio > 0.25;
      const bool xtol_ok = step_norm < xtol * (xtol + vnorm(x, 3));
      if (ftol_ok && xtol_ok) status = 4;
      else if (ftol_ok) status = 2;
      else if (xtol_ok) status = 3;
      if (status != -100) break;
      alpha *= Delta / Delta_new;
      Delta = Delta_new;
    }
    if (actual_reduction > 0) {
      for (int i = 0; i < 3; ++i) x[i] = x_new[i];
      for (int r = 0; r < m; ++r) f[r] = f_new[r];
      cost = cost_new;
      trf_jacobian(P, x, f, lb, ub, J);
      for (int i = 0; i < 3; ++i) {
        double acc = 0.0;
        for (int r = 0; r < m; ++r) acc += J[r * 3 + i] * f[r];
        g[i] = acc;
      }
    }
    iteration += 1;
  }
  if (status == -100) status = 0;
  for (int i = 0; i < 3; ++i) res.x[i] = x[i];
  res.status = status;
  res.nfev = nfev;
  res.iterations = iteration;
  return res;
}

}  // namespace vk
