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
