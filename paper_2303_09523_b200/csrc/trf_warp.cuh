// Warp-parallel form of trf.h for the device fit: one warp per sub-part,
// lane r owns residual / Jacobian row r (bins), lanes m..m+2 own the three
// diagonal rows of the augmented matrix.  The SVD of the augmented Jacobian
// (scipy: LAPACK gesdd) is a lane-parallel Householder QR followed by a
// Jacobi SVD of the 3x3 R factor; the trust-region step only uses s, V and
// U^T f, which both routes produce to rounding.  Every scalar decision (trust
// region, reflections, termination) is evaluated redundantly on all lanes
// from all-reduced values, so the lanes never diverge.  The algorithm and its
// order of operations follow trf.h (scipy 1.18 trf_bounds) step by step; only
// the sums over residual rows become butterfly reductions.
#pragma once
#include "trf.h"

namespace vk {

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

#ifdef VK_FIT_PROFILE
__device__ unsigned long long g_fit_prof[12];  // cycles: jac, svd, trsolve, select, resid, total, nfev, iters, svd-qr, svd-jacobi, sweeps
#define VK_PT(v) const long long v = clock64()
#define VK_PACC(slot, a, b) if (lane == 0) atomicAdd(&g_fit_prof[slot], (unsigned long long)((b) - (a)))
#else
#define VK_PT(v)
#define VK_PACC(slot, a, b)
#endif

template <int KIND>
struct WarpTrf {
  const TrfProblem& P;
  int lane, m;
  bool row;          // lane holds a residual row
  double h, gemp, w; // this lane's bin

  __device__ WarpTrf(const TrfProblem& p, int l) : P(p), lane(l), m(p.nb), row(l < p.nb) {
    h = row ? P.h[l] : 0.0;
    gemp = row ? P.gemp[l] : 0.0;
    w = row ? P.w[l] : 0.0;
  }

  // branch-free (lanes without a row evaluate h = 0 and are masked): the
  // kind is a template parameter, so independent evaluations interleave
  __device__ double resid(const double* x) const {
    Model md;
    md.nugget = pymax(x[0], 0.0);
    md.sill = md.nugget + pymax(x[1], 0.0);
    md.range_len = pymax(x[2], 1e-6);
    const double f = w * (semivariance_k<KIND>(md, h) - gemp);
    return row ? f : 0.0;
  }

  // 2-point Jacobian (scipy approx_derivative with bounds): the three steps
  // first, then the three perturbed residuals, then the quotients
  __device__ void jac(const double* x, double f0, const double* lb, const double* ub, double* J) const {
    const double rstep = 1.4901161193847656e-08;
    double hh[3], f1[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double sign = (x[i] >= 0.0) ? 1.0 : -1.0;
      double hi = rstep * sign * fmax(1.0, fabs(x[i]));
      const double ld = x[i] - lb[i], ud = ub[i] - x[i];
      const double xt = x[i] + hi;
      const bool violated = (xt < lb[i]) || (xt > ub[i]);
      const bool fitting = fabs(hi) <= fmax(ld, ud);
      if (violated && fitting) hi = -hi;
      if (!fitting) hi = (ud >= ld) ? ud : -ld;
      hh[i] = hi;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      double x1[3] = {x[0], x[1], x[2]};
      x1[i] = x[i] + hh[i];
      f1[i] = resid(x1);
    }
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const double dx = (x[i] + hh[i]) - x[i];
      J[i] = row ? (f1[i] - f0) / dx : 0.0;
    }
  }

  // SVD of the augmented matrix [J_h; diag(sqrt(diag_h))] (this lane's row in
  // a[3]) as Householder QR across the lanes (two reduction rounds per
  // column), then a one-sided Jacobi SVD of the 3x3 R in registers.  Returns
  // s (descending), V, and uf = U^T f_aug directly (U = Q U_R).
  __device__ void svd_uf(double* a, double fl, double* s, double* V, double* uf) const {
    VK_PT(t_q0);
    double R[9];
    for (int k = 0; k < 3; ++k) {
      const bool act = lane >= k;
      const double xk = act ? a[k] : 0.0;
      const double nrm2 = wsum(xk * xk);
      const double x_kk = __shfl_sync(0xffffffffu, a[k], k);
      const double nrm = sqrt(nrm2);
      const double alpha = (x_kk > 0.0) ? -nrm : nrm;
      const double vv = 2.0 * (nrm2 - x_kk * alpha);     // ||v||^2
      double v = act ? a[k] : 0.0;
      if (lane == k) v = x_kk - alpha;
      // project the remaining columns and f onto v in one reduction round
      double d1 = 0.0, d2 = 0.0, df = 0.0;
      if (k + 1 < 3) d1 = wsum(v * a[k + 1]);
      if (k + 2 < 3) d2 = wsum(v * a[k + 2]);
      df = wsum(v * fl);
      if (vv > 0.0) {
        const double sc = 2.0 / vv;
        if (k + 1 < 3) a[k + 1] -= sc * d1 * v;
        if (k + 2 < 3) a[k + 2] -= sc * d2 * v;
        fl -= sc * df * v;
        if (lane == k) a[k] = alpha;
        else if (act) a[k] = 0.0;
      }
    }
    double qf[3];
    for (int r = 0; r < 3; ++r) {
      for (int c = 0; c < 3; ++c) R[r * 3 + c] = __shfl_sync(0xffffffffu, a[c], r);
      qf[r] = __shfl_sync(0xffffffffu, fl, r);
    }
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < r; ++c) R[r * 3 + c] = 0.0;
    VK_PT(t_q1);
    VK_PACC(8, t_q0, t_q1);
    // one-sided Jacobi on the columns of R (3x3, no cross-lane traffic),
    // warm-started from the caller's V (the previous iteration's right singular
    // vectors: J moves little between TRF iterations, so R V is already nearly
    // column-orthogonal and one or two sweeps finish it).  V enters orthogonal;
    // the result is the SVD of R up to column order and signs, as from a cold
    // start.
    {
      double RV[9];
      for (int r = 0; r < 3; ++r)
        for (int c = 0; c < 3; ++c)
          RV[r * 3 + c] = R[r * 3 + 0] * V[0 + c] + R[r * 3 + 1] * V[3 + c] + R[r * 3 + 2] * V[6 + c];
      for (int i = 0; i < 9; ++i) R[i] = RV[i];
    }
    for (int sweep = 0; sweep < 60; ++sweep) {
      bool rotated = false;
      for (int p = 0; p < 2; ++p)
        for (int q = p + 1; q < 3; ++q) {
          double alpha = 0.0, beta = 0.0, gamma = 0.0;
          for (int r = 0; r < 3; ++r) {
            alpha += R[r * 3 + p] * R[r * 3 + p];
            beta += R[r * 3 + q] * R[r * 3 + q];
            gamma += R[r * 3 + p] * R[r * 3 + q];
          }
          // converged pair: |gamma| <= 1e-15 sqrt(alpha beta) (orthogonal to
          // working precision; the trust-region step uses s, V to ~1e-14)
          if (gamma == 0.0 || gamma * gamma <= 1e-30 * (alpha * beta)) continue;
          rotated = true;
          // the smaller Jacobi angle (|theta| <= pi/4) from its double angle:
          // cos 2t = |b-a| / h, sin 2t = 2 gamma sign(b-a) / h, h = sqrt((b-a)^2 + 4 gamma^2);
          // c = sqrt((1 + cos 2t) / 2), s = sin 2t / (2 c) -- two rsqrt, no
          // division or sqrt on the dependent chain (x in [1/2, 1])
          const double bma = beta - alpha;
          const double sg = (bma >= 0.0) ? 1.0 : -1.0;
          const double ih = rsqrt(bma * bma + 4.0 * gamma * gamma);
          const double xh = 0.5 + 0.5 * (fabs(bma) * ih);
          const double rx = rsqrt(xh);
          const double c = xh * rx, sn = (gamma * sg) * ih * rx;
          for (int r = 0; r < 3; ++r) {
            const double rp = R[r * 3 + p], rq = R[r * 3 + q];
            R[r * 3 + p] = c * rp - sn * rq;
            R[r * 3 + q] = sn * rp + c * rq;
            const double vp = V[r * 3 + p], vq = V[r * 3 + q];
            V[r * 3 + p] = c * vp - sn * vq;
            V[r * 3 + q] = sn * vp + c * vq;
          }
        }
#ifdef VK_FIT_PROFILE
      if (lane == 0) atomicAdd(&g_fit_prof[10], 1ull);
#endif
      if (!rotated) break;
    }
    VK_PT(t_q2);
    VK_PACC(9, t_q1, t_q2);
    double sv[3], uq[3];
    for (int j = 0; j < 3; ++j) {
      const double n2 = R[0 + j] * R[0 + j] + R[3 + j] * R[3 + j] + R[6 + j] * R[6 + j];
      const double rn = n2 > 0.0 ? rsqrt(n2) : 0.0;
      sv[j] = n2 * rn;
      uq[j] = (R[0 + j] * qf[0] + R[3 + j] * qf[1] + R[6 + j] * qf[2]) * rn;
    }
    int order[3] = {0, 1, 2};
    for (int x = 0; x < 3; ++x)
      for (int y = x + 1; y < 3; ++y)
        if (sv[order[y]] > sv[order[x]]) { const int t = order[x]; order[x] = order[y]; order[y] = t; }
    double Vs[9];
    for (int k = 0; k < 3; ++k) {
      const int j = order[k];
      s[k] = sv[j];
      uf[k] = uq[j];
      for (int r = 0; r < 3; ++r) Vs[r * 3 + k] = V[r * 3 + j];
    }
    for (int i = 0; i < 9; ++i) V[i] = Vs[i];
  }

  __device__ double jh_row(const double* Jh, const double* s) const {
    return row ? Jh[0] * s[0] + Jh[1] * s[1] + Jh[2] * s[2] : 0.0;
  }

  __device__ double eval_quad(const double* Jh, const double* g, const double* s, const double* diag) const {
    const double js = jh_row(Jh, s);
    double q = wsum(js * js);
    double sd[3] = {s[0] * diag[0], s[1] * diag[1], s[2] * diag[2]};
    q += vdot(sd, s, 3);
    return 0.5 * q + vdot(s, g, 3);
  }

  __device__ void build_quad(const double* Jh, const double* g, const double* s, const double* diag,
                             const double* s0, double* a, double* b, double* c) const {
    const double v = jh_row(Jh, s);
    double aa = wsum(v * v);
    double sd[3] = {s[0] * diag[0], s[1] * diag[1], s[2] * diag[2]};
    aa += vdot(sd, s, 3);
    aa *= 0.5;
    double bb = vdot(g, s, 3);
    double cc = 0.0;
    if (s0) {
      const double u = jh_row(Jh, s0);
      bb += wsum(u * v);
      cc = 0.5 * wsum(u * u) + vdot(g, s0, 3);
      double s0d[3] = {s0[0] * diag[0], s0[1] * diag[1], s0[2] * diag[2]};
      bb += vdot(s0d, s, 3);
      cc += 0.5 * vdot(s0d, s0, 3);
    }
    *a = aa; *b = bb; *c = cc;
  }

  __device__ bool select(const double* x, const double* Jh, const double* diag_h, const double* g_h,
                         double* p, double* p_h, const double* d, double Delta, const double* lb,
                         const double* ub, double theta, double* step, double* step_h, double* pred) const {
    double xp[3] = {x[0] + p[0], x[1] + p[1], x[2] + p[2]};
    if (in_bounds3(xp, lb, ub)) {
      const double pv = eval_quad(Jh, g_h, p_h, diag_h);
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
    double xb[3] = {x[0] + p[0], x[1] + p[1], x[2] + p[2]};
    double t_neg, to_tr;
    if (!intersect_tr(p_h, r_h, Delta, &t_neg, &to_tr)) return false;
    int h2[3];
    const double to_bound = step_to_bound(xb, r, lb, ub, h2);
    double r_stride = fmin(to_bound, to_tr);
    double rl, ru;
    if (r_stride > 0) {
      rl = (1 - theta) * p_stride / r_stride;
      ru = (r_stride == to_bound) ? theta * to_bound : to_tr;
    } else {
      rl = 0;
      ru = -1;
    }
    double r_value;
    if (rl <= ru) {
      double a, b, c;
      build_quad(Jh, g_h, r_h, diag_h, p_h, &a, &b, &c);
      min_quad_1d(a, b, rl, ru, c, &r_stride, &r_value);
      for (int i = 0; i < 3; ++i) {
        r_h[i] *= r_stride;
        r_h[i] += p_h[i];
        r[i] = r_h[i] * d[i];
      }
    } else {
      r_value = INFINITY;
    }
    for (int i = 0; i < 3; ++i) { p[i] *= theta; p_h[i] *= theta; }
    const double p_value = eval_quad(Jh, g_h, p_h, diag_h);
    double ag_h[3], ag[3];
    for (int i = 0; i < 3; ++i) { ag_h[i] = -g_h[i]; ag[i] = d[i] * ag_h[i]; }
    const double to_tr2 = Delta / vnorm(ag_h, 3);
    int h3[3];
    const double to_bound2 = step_to_bound(x, ag, lb, ub, h3);
    double ag_stride = (to_bound2 < to_tr2) ? theta * to_bound2 : to_tr2;
    double a2, b2, c2;
    build_quad(Jh, g_h, ag_h, diag_h, nullptr, &a2, &b2, &c2);
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

  __device__ TrfResult fit(const double* x0_in, const double* lb, const double* ub) const {
    const double ftol = 1e-8, xtol = 1e-8, gtol = 1e-8;
    const int max_nfev = 300;
    TrfResult res;
    double x[3] = {x0_in[0], x0_in[1], x0_in[2]};
    make_strictly_feasible(x, lb, ub, 1e-10);
    double f = resid(x);
    double J[3];
    jac(x, f, lb, ub, J);
    int nfev = 1;
    double cost = 0.5 * wsum(f * f);
    double g[3];
    for (int i = 0; i < 3; ++i) g[i] = wsum(J[i] * f);
    double v[3], dv[3];
    auto cl = [&]() {
      for (int i = 0; i < 3; ++i) {
        v[i] = 1.0; dv[i] = 0.0;
        if (g[i] < 0 && finite_d(ub[i])) { v[i] = ub[i] - x[i]; dv[i] = -1.0; }
        if (g[i] > 0 && finite_d(lb[i])) { v[i] = x[i] - lb[i]; dv[i] = 1.0; }
      }
    };
    cl();
    double Delta;
    {
      double t[3];
      for (int i = 0; i < 3; ++i) t[i] = x[i] * 1.0 / sqrt(v[i]);
      Delta = vnorm(t, 3);
      if (Delta == 0) Delta = 1.0;
    }
    double alpha = 0.0;
    double V[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};   // right singular vectors, carried across iterations
    int status = -100;
    int iteration = 0;
    double x_new[3], f_new = 0.0, cost_new = 0.0, g_norm = 0.0;
    while (true) {
      cl();
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
      double Jh[3], a[3];
      for (int c = 0; c < 3; ++c) Jh[c] = J[c] * d[c];
      if (row) {
        for (int c = 0; c < 3; ++c) a[c] = Jh[c];
      } else {
        const int dr = lane - m;   // diagonal rows m..m+2
        for (int c = 0; c < 3; ++c) a[c] = (dr >= 0 && dr < 3 && dr == c) ? sqrt(diag_h[c]) : 0.0;
      }
      double sv[3], uf[3];
      VK_PT(t_s0);
      svd_uf(a, row ? f : 0.0, sv, V, uf);
      VK_PT(t_s1);
      VK_PACC(1, t_s0, t_s1);
      const double theta = fmax(0.995, 1 - g_norm);
      double actual_reduction = -1;
      double step_norm = 0.0;
      while (actual_reduction <= 0 && nfev < max_nfev) {
        double p_h[3], p[3];
        VK_PT(t_t0);
        lsq_trust_region(m, uf, sv, V, Delta, alpha, p_h, &alpha);
        VK_PT(t_t1);
        VK_PACC(2, t_t0, t_t1);
        for (int i = 0; i < 3; ++i) p[i] = d[i] * p_h[i];
        double step[3], step_h[3], pred;
        const bool sel_ok = select(x, Jh, diag_h, g_h, p, p_h, d, Delta, lb, ub, theta, step, step_h, &pred);
        VK_PT(t_t2);
        VK_PACC(3, t_t1, t_t2);
        if (!sel_ok) {
          res.status = -1;
          res.nfev = nfev;
          res.iterations = iteration;
          for (int i = 0; i < 3; ++i) res.x[i] = x[i];
          return res;
        }
        for (int i = 0; i < 3; ++i) x_new[i] = x[i] + step[i];
        make_strictly_feasible(x_new, lb, ub, 0.0);
        VK_PT(t_r0);
        f_new = resid(x_new);
        VK_PT(t_r1);
        VK_PACC(4, t_r0, t_r1);
        nfev += 1;
        const double step_h_norm = vnorm(step_h, 3);
        const bool finite = __all_sync(0xffffffffu, finite_d(f_new));
        if (!finite) { Delta = 0.25 * step_h_norm; continue; }
        cost_new = 0.5 * wsum(f_new * f_new);
        actual_reduction = cost - cost_new;
        double ratio;
        if (pred > 0) ratio = actual_reduction / pred;
        else if (pred == actual_reduction && pred == 0) ratio = 1;
        else ratio = 0;
        double Delta_new = Delta;
        if (ratio < 0.25) Delta_new = 0.25 * step_h_norm;
        else if (ratio > 0.75 && step_h_norm > 0.95 * Delta) Delta_new = Delta * 2.0;
        step_norm = vnorm(step, 3);
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
        f = f_new;
        cost = cost_new;
        VK_PT(t_j0);
        jac(x, f, lb, ub, J);
        for (int i = 0; i < 3; ++i) g[i] = wsum(J[i] * f);
        VK_PT(t_j1);
        VK_PACC(0, t_j0, t_j1);
      }
      iteration += 1;
    }
    if (status == -100) status = 0;
    for (int i = 0; i < 3; ++i) res.x[i] = x[i];
    res.status = status;
    res.nfev = nfev;
    res.iterations = iteration;
#ifdef VK_FIT_PROFILE
    if (lane == 0) {
      atomicAdd(&g_fit_prof[6], (unsigned long long)nfev);
      atomicAdd(&g_fit_prof[7], (unsigned long long)iteration);
    }
#endif
    return res;
  }
};

}  // namespace vk
