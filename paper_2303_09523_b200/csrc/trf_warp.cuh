// Evaluator for the device fit: a CTA of FIT_WARPS (2) warps per sub-part runs
// trf.h's trf_fit_t (scipy 1.18 trf_bounds restated with numpy/OpenBLAS
// arithmetic) redundantly on every thread -- every thread holds the same
// iterate, bit for bit, so threads never diverge and reach every barrier
// together.  Each warp keeps its own copies of the TRF's row arrays and of
// the SVD workspace (the warps are not in lock step), and the threads
// cooperate where the chain has independent work:
//   * residual rows and Jacobian columns: one (bin, column) item per thread;
//     at a trial point the residuals and the Jacobian there are evaluated in
//     the same round (resid_spec), so an accepted step needs no separate
//     Jacobian round;
//   * the SVD (gesdd_warp.cuh svd_m3_2w): after each warp's Householder QR,
//     warp 0 forms Q (dorg2r) while warp 1 runs the 3 x 3 stages (dgebd2,
//     dbdsqr, the two dormbr); the warps exchange Q and (d, U_B, V_B^T)
//     through shared memory.
// Every value is the one the single-thread restatement computes.
#pragma once
#include "trf.h"
#include "gesdd_warp.cuh"

namespace vk {

constexpr int FIT_WARPS = 2;
constexpr int FIT_THREADS = 32 * FIT_WARPS;

struct FitShared {
  double row[4 * MAX_BINS];                 // item exchange (residuals, Jacobian columns)
  lapack::SvdWarpSmem sv[FIT_WARPS];        // per-warp SVD workspace
  lapack::SvdXchg xchg;                     // warp 1 -> both: the 3 x 3 stages' results
  TrfWork wk[FIT_WARPS];                    // per-warp TRF row arrays
};

struct WarpEval {
  const TrfProblem& P;
  FitShared& S;
  int tid, lane, wid;

  __device__ WarpEval(const TrfProblem& p, FitShared& s, int t)
      : P(p), S(s), tid(t), lane(t & 31), wid(t >> 5) {}
  __device__ int m() const { return P.nb; }
  __device__ TrfWork& work() const { return S.wk[wid]; }

  __device__ int svd(const double* A, int M, double* U, double* s, double* VT) const {
    return lapack::svd_m3_2w(A, M, U, s, VT, S.sv[wid], S.sv[wid ^ 1], S.xchg, lane, wid);
  }

  // item k < m: residual row k at x; then item m + i*m + r: Jacobian column
  // i, row r (_numdiff.py 2-point: (f(x + h_i e_i) - f(x)) / dx_i), whose f(x)
  // row is recomputed inside the item (the same bits as item r)
  __device__ double item(const double* x, const double* lb, const double* ub, int k, bool with_f) const {
    const int mm = P.nb;
    const FitModel md = fit_model(x);
    if (with_f) {
      if (k < mm) return fit_residual_kind(P.kind, md, P.h[k], P.gemp[k], P.w[k]);
      k -= mm;
    }
    const int i = k / mm, r = k - i * mm;
    const double h = fd_step(x, lb, ub, i);
    double x1[3] = {x[0], x[1], x[2]};
    x1[i] = np::add(x[i], h);
    const FitModel m1 = fit_model(x1);
    const double f1 = fit_residual_kind(P.kind, m1, P.h[r], P.gemp[r], P.w[r]);
    const double f0 = fit_residual_kind(P.kind, md, P.h[r], P.gemp[r], P.w[r]);
    const double dx = np::sub(np::add(x[i], h), x[i]);
    return np::div(np::sub(f1, f0), dx);
  }

  __device__ void resid(const double* x, double* f) const {
    const FitModel md = fit_model(x);
    for (int k = tid; k < P.nb; k += FIT_THREADS)
      S.row[k] = fit_residual_kind(P.kind, md, P.h[k], P.gemp[k], P.w[k]);
    __syncthreads();
    for (int r = 0; r < P.nb; ++r) f[r] = S.row[r];
    __syncthreads();
  }

  __device__ void jac(const double* x, const double* f0, const double* lb, const double* ub, double* J) const {
    (void)f0;                                   // recomputed per item (same bits)
    const int n = 3 * P.nb;
    for (int k = tid; k < n; k += FIT_THREADS) S.row[k] = item(x, lb, ub, k, false);
    __syncthreads();
    for (int k = 0; k < n; ++k) J[k] = S.row[k];
    __syncthreads();
  }

  __device__ void resid_spec(const double* x, const double* lb, const double* ub, double* f, double* J) const {
    const int mm = P.nb, n = 4 * mm;
    for (int k = tid; k < n; k += FIT_THREADS) S.row[k] = item(x, lb, ub, k, true);
    __syncthreads();
    for (int r = 0; r < mm; ++r) f[r] = S.row[r];
    for (int k = 0; k < 3 * mm; ++k) J[k] = S.row[mm + k];
    __syncthreads();
  }
};

}  // namespace vk
