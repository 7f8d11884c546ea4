// Warp evaluator for the device fit: one warp per sub-part runs trf.h's
// trf_fit_t (scipy 1.18 trf_bounds restated with numpy/OpenBLAS arithmetic)
// redundantly on all 32 lanes -- every lane holds the same iterate, bit for
// bit, so lanes never diverge -- while the residual rows (one bin per lane)
// and the three finite-difference columns of the Jacobian are evaluated
// lane-parallel and shared through a per-warp shared-memory row buffer, and
// the SVD's row work is spread over the lanes (gesdd_warp.cuh).
// The residual is the only part of an iteration whose cost grows with the
// bins, and its SVML exp is the most expensive scalar operation of the fit.
#pragma once
#include "trf.h"
#include "gesdd_warp.cuh"

namespace vk {

struct WarpEval {
  const TrfProblem& P;      // shared memory
  double* row;              // shared memory, >= 3 * MAX_BINS doubles
  lapack::SvdWarpSmem& sv;  // shared memory
  TrfWork& wk;              // shared memory (identical stores from every lane)
  int lane;

  __device__ WarpEval(const TrfProblem& p, double* buf, lapack::SvdWarpSmem& s, TrfWork& w, int l)
      : P(p), row(buf), sv(s), wk(w), lane(l) {}
  __device__ int m() const { return P.nb; }
  __device__ TrfWork& work() const { return wk; }

  __device__ int svd(const double* A, int M, double* U, double* s, double* VT) const {
    return lapack::svd_m3_warp(A, M, U, s, VT, sv, lane);
  }

  __device__ void resid(const double* x, double* f) const {
    const FitModel md = fit_model(x);
    if (lane < P.nb) row[lane] = fit_residual_kind(P.kind, md, P.h[lane], P.gemp[lane], P.w[lane]);
    __syncwarp();
    for (int r = 0; r < P.nb; ++r) f[r] = row[r];
    __syncwarp();
  }

  // _numdiff.py 2-point: column i = (f(x + h_i e_i) - f0) / dx_i
  __device__ void jac(const double* x, const double* f0, const double* lb, const double* ub, double* J) const {
    const int m = P.nb;
    if (lane < m) {
      const double fr = f0[lane];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const double h = fd_step(x, lb, ub, i);
        double x1[3] = {x[0], x[1], x[2]};
        x1[i] = np::add(x[i], h);
        const FitModel md = fit_model(x1);
        const double f1 = fit_residual_kind(P.kind, md, P.h[lane], P.gemp[lane], P.w[lane]);
        const double dx = np::sub(np::add(x[i], h), x[i]);
        row[i * m + lane] = np::div(np::sub(f1, fr), dx);
      }
    }
    __syncwarp();
    for (int k = 0; k < 3 * m; ++k) J[k] = row[k];
    __syncwarp();
  }
};

}  // namespace vk
