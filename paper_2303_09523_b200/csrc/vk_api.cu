// C ABI of the volkrig-b200 kriging path (include/volkrig_b200.h): plan
// creation (host geometry + device tables), stream-ordered execution of
// stats -> pairs -> bins -> fit -> solve -> predict, and status mapping.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <string>
#include <mutex>
#include <vector>
#include <thread>
#include <memory>

#include "../../include/volkrig_b200.h"
#include "pcg64.h"
#include "vk_geometry.h"
#include "vk_kernels.h"

namespace vk {
cudaError_t launch_plane_stats_f64(const double* values, int64_t m, ChunkStat* out, int nchunk,
                                   cudaStream_t st);
}

using namespace vk;

namespace {

thread_local std::string g_last_error;

int set_err(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define VK_CUDA(call)                                                             \
  do {                                                                            \
    cudaError_t e_ = (call);                                                      \
    if (e_ != cudaSuccess)                                                        \
      return set_err(VK_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

template <typename T>
cudaError_t upload(T** dst, const std::vector<T>& src) {
  *dst = nullptr;
  if (src.empty()) return cudaSuccess;
  cudaError_t e = cudaMalloc((void**)dst, src.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
}

int status_from_part(int ps) {
  switch (ps) {
    case PS_OK: return VK_OK;
    case PS_SINGULAR: return VK_E_SINGULAR_SYSTEM;
    case PS_INSUFFICIENT: return VK_E_INSUFFICIENT_SAMPLES;
    case PS_DEGENERATE: return VK_E_DEGENERATE_LAGS;
    case PS_FIT_FAILED: return VK_E_FIT_FAILED;
    case PS_NONFINITE: return VK_E_INVALID_GRID;
    default: return VK_E_CUDA;
  }
}

}  // namespace

namespace vk {
// error reporting for the other translation units of the C ABI (vk_comm.cpp)
int comm_set_err(int status, const std::string& msg) { return set_err(status, msg); }
}  // namespace vk

struct vk_plan {
  vk_plan_desc desc;
  Geometry geo;
  int num_sms = 0;
  int NP = 0, NK = 0, n_sys = 0, max_n = 0, max_dz = 0;
  int nchunk = 0, nblk = 0;
  std::vector<void*> allocs;
  // device tables
  int32_t *d_known_z = nullptr, *d_miss_z = nullptr, *d_miss_part = nullptr, *d_miss_pattern = nullptr,
          *d_miss_planes = nullptr, *d_sys_part = nullptr, *d_sys_stencil = nullptr, *d_st_off = nullptr,
          *d_st_n = nullptr, *d_st_drift = nullptr, *d_st_pattern = nullptr, *d_pat_dz = nullptr,
          *d_gap_part = nullptr, *d_gap_pattern = nullptr, *d_kmap = nullptr, *d_part_b = nullptr,
          *d_part_e = nullptr, *d_part_class = nullptr, *d_zloc = nullptr;
  int8_t* d_taps = nullptr;
  int16_t* d_pad = nullptr;
  int64_t *d_part_base = nullptr, *d_part_m = nullptr;
  // workspace
  ChunkStat* d_stats = nullptr;
  double *d_partial = nullptr, *d_models = nullptr, *d_lohi = nullptr, *d_weights = nullptr, *d_var = nullptr;
  double* d_kpm = nullptr;
  int* d_inexact = nullptr;           // stats pass: any known value not an integer below 2^23
  int* d_work = nullptr;              // [S + 1][2] unit counters of the streaming launches (part s; S: serial)
  uint32_t* d_fxb = nullptr;           // fixed path tables
  float *d_fxc = nullptr, *d_fxq = nullptr;
  int max_chunk = 0;                  // fast path: a run of this many gaps spans <= 3 parts
  int fit_reserve = 160 * 1024;       // overlapped schedule: smem a fit CTA reserves on its SM
  int32_t *d_part_status = nullptr, *d_sys_status = nullptr;
  std::vector<PairTable> tables;
  PairTable* d_tables = nullptr;
  std::vector<PairJob> jobs;          // one per pair class
  PairJob* d_jobs = nullptr;
  // numpy-exact svar and bin sums (vk_npstats.cu)
  std::vector<NpSumTree> trees;       // one per pair class
  NpSumTree* d_trees = nullptr;
  int max_leaf = 0;
  int64_t leaf_stride = 0, node_stride = 0;
  double *d_npleaf = nullptr, *d_npnode = nullptr, *d_mean = nullptr, *d_svar = nullptr;
  double *d_sq = nullptr, *d_bsum = nullptr;
  bool pairs_ready = false;
  // pinned staging of caller models ([S][3] each): a ring, so an execute
  // queued behind another on a busy stream never overwrites models whose
  // host-to-device copy has not run yet (each slot's copy is fenced by an event)
  static constexpr int NMODEL_RING = 4;
  double* h_models[NMODEL_RING] = {};
  cudaEvent_t ev_models[NMODEL_RING] = {};
  int models_slot = 0;
  int kernels = 0;
  cudaStream_t side = nullptr;        // pair draw runs here, concurrent with stats
  cudaStream_t io = nullptr;          // vk_plan_download: host-side known planes
  cudaEvent_t ev_io_fork = nullptr, ev_io_join = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // per-part chains (fit -> solve -> predict): one stream per part (up to
  // NCH), so every part's latency-bound fit starts at once
  static constexpr int NCH = 64;
  cudaStream_t chain[NCH] = {};        // fit -> solve (high priority)
  cudaStream_t pchain[NCH] = {};       // predict (low priority), after its part's solve
  cudaEvent_t ev_kfork = nullptr, ev_kjoin[NCH] = {}, ev_solved[NCH] = {}, ev_pjoin[NCH] = {};
  // head parts (chained schedule): statistics and bins of the first parts go
  // first, so their chains start before the rest of the volume is reduced
  cudaEvent_t ev_hstats = nullptr, ev_hbins = nullptr;
  int head_parts = 0;
  std::vector<int> sys_begin;         // [S + 1] system range of each part
  std::vector<int> sys_canon;         // [S] end of each part's solved (canonical) systems
  int n_derived = 0;
  int32_t *d_der_src = nullptr, *d_der_flags = nullptr;
  std::vector<int> gap_begin;         // [S + 1] gap range of each part (fast path)
  FastLaunch fast_launch;             // cached TMA descriptor + occupancy
  int ring = 0;                       // timing ring size (0 = off)
  int64_t n_exec = 0;                 // executes recorded so far
  int64_t n_runs = 0;                 // executes issued (diagnostics)
  std::vector<cudaEvent_t> ev;        // [ring][VK_N_STAGES + 1]

  template <typename T>
  cudaError_t alloc(T** p, size_t n) {
    cudaError_t e = cudaMalloc((void**)p, std::max<size_t>(n, 1) * sizeof(T));
    if (e == cudaSuccess) allocs.push_back(*p);
    return e;
  }
  template <typename T>
  cudaError_t put(T** p, const std::vector<T>& v) {
    cudaError_t e = upload(p, v);
    if (e == cudaSuccess && *p) allocs.push_back(*p);
    return e;
  }
  ~vk_plan() {
    for (cudaEvent_t e : ev) cudaEventDestroy(e);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (side) cudaStreamDestroy(side);
    if (io) cudaStreamDestroy(io);
    if (ev_io_fork) cudaEventDestroy(ev_io_fork);
    if (ev_io_join) cudaEventDestroy(ev_io_join);
    if (ev_kfork) cudaEventDestroy(ev_kfork);
    if (ev_hstats) cudaEventDestroy(ev_hstats);
    if (ev_hbins) cudaEventDestroy(ev_hbins);
    for (int i = 0; i < NCH; ++i) {
      if (ev_kjoin[i]) cudaEventDestroy(ev_kjoin[i]);
      if (ev_solved[i]) cudaEventDestroy(ev_solved[i]);
      if (ev_pjoin[i]) cudaEventDestroy(ev_pjoin[i]);
      if (chain[i]) cudaStreamDestroy(chain[i]);
      if (pchain[i]) cudaStreamDestroy(pchain[i]);
    }
    for (void* p : allocs) cudaFree(p);
    for (int i = 0; i < NMODEL_RING; ++i) {
      if (h_models[i]) cudaFreeHost(h_models[i]);
      if (ev_models[i]) cudaEventDestroy(ev_models[i]);
    }
  }
};

extern "C" {

int vk_abi_version(void) { return VK_ABI_VERSION; }

const char* vk_status_string(int s) {
  switch (s) {
    case VK_OK: return "ok";
    case VK_E_INVALID_ARGUMENT: return "invalid argument";
    case VK_E_NO_KNOWN_NEIGHBORS: return "no known neighbors";
    case VK_E_SINGULAR_SYSTEM: return "singular kriging system";
    case VK_E_INSUFFICIENT_SAMPLES: return "insufficient samples";
    case VK_E_DEGENERATE_LAGS: return "degenerate lags";
    case VK_E_UNSUPPORTED: return "unsupported layout";
    case VK_E_CUDA: return "cuda error";
    case VK_E_INVALID_GRID: return "invalid grid";
    case VK_E_FIT_FAILED: return "variogram fit failed";
    default: return "unknown";
  }
}

const char* vk_last_error(void) { return g_last_error.c_str(); }

int vk_plan_create(const vk_plan_desc* d, vk_plan** out) {
  if (!d || !out) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  if (d->kind < 0 || d->kind > 2) return set_err(VK_E_INVALID_ARGUMENT, "kind");
  if (d->drift < 0 || d->drift > 1) return set_err(VK_E_INVALID_ARGUMENT, "drift");
  if (d->accum < 0 || d->accum > 2) return set_err(VK_E_INVALID_ARGUMENT, "accum");
  if (d->n_bins < 1 || d->n_bins > MAX_BINS) return set_err(VK_E_INVALID_ARGUMENT, "n_bins must be in 1..32");
  if (d->max_pairs < 1 || d->max_pairs > (1ll << 30)) return set_err(VK_E_INVALID_ARGUMENT, "max_pairs");
  if (!d->known_z && d->n_known > 0) return set_err(VK_E_INVALID_ARGUMENT, "known_z");
  vk_plan* p = new vk_plan();
  p->desc = *d;
  p->desc.known_z = nullptr;
  std::string err = build_geometry(d->height, d->width, d->depth, d->known_z, d->n_known, d->n_subparts,
                                   d->part_len, d->drift, &p->geo);
  if (!err.empty()) {
    delete p;
    if (err.rfind("NoKnownNeighbors", 0) == 0) return set_err(VK_E_NO_KNOWN_NEIGHBORS, err);
    if (err.rfind("Unsupported", 0) == 0) return set_err(VK_E_UNSUPPORTED, err);
    return set_err(VK_E_INVALID_ARGUMENT, err);
  }
  Geometry& g = p->geo;
  if (d->flags & VK_FLAG_FORCE_GENERIC) g.fast = false;
  // systems that are z-mirror / x<->y-transpose images of another system of
  // the same part are derived, not solved (vk_geometry.cpp canonical_systems)
  std::vector<int32_t> der_src, der_flags;
  canonical_systems(&g, &p->sys_canon, &der_src, &der_flags, &p->n_derived);
  const int64_t P = (int64_t)g.H * g.W;
  if (d->fit_variogram) {
    for (const PartInfo& pi : g.parts)
      if (pi.m > 0xffffffffll)
        return delete p, set_err(VK_E_UNSUPPORTED, "more than 2^32 samples in one sub-part");
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev);
  p->NP = (int)g.patterns.size();
  p->NK = g.n_kinds();
  p->n_sys = (int)g.sys_part.size();
  p->nchunk = (int)((P + STATS_CHUNK - 1) / STATS_CHUNK);
  p->nblk = (int)std::max<int64_t>(1, (std::min<int64_t>(d->max_pairs, (int64_t)1 << 30) + 4095) / 4096);

  // ---- host tables
  std::vector<int32_t> st_off, st_n, st_drift, st_pattern, pat_dz((size_t)std::max(1, p->NP) * NPMAX, 0);
  std::vector<int8_t> taps;
  std::vector<int16_t> pad;
  for (const StencilGeom& sg : g.stencils) {
    st_off.push_back((int32_t)pad.size());
    st_n.push_back(sg.n);
    st_drift.push_back(sg.drift_cols);
    st_pattern.push_back(sg.pattern);
    taps.insert(taps.end(), sg.taps.begin(), sg.taps.end());
    pad.insert(pad.end(), sg.pad.begin(), sg.pad.end());
    p->max_n = std::max(p->max_n, sg.n);
  }
  for (int q = 0; q < p->NP; ++q)
    for (size_t i = 0; i < g.patterns[q].size(); ++i) {
      pat_dz[(size_t)q * NPMAX + i] = g.patterns[q][i];
      for (size_t i2 = 0; i2 < g.patterns[q].size(); ++i2)
        p->max_dz = std::max(p->max_dz, std::abs(g.patterns[q][i] - g.patterns[q][i2]));
      p->max_dz = std::max(p->max_dz, std::abs(g.patterns[q][i]));
    }
  std::vector<int32_t> kmap(2 * NKIND1, 0);
  for (int i = 0; i < NKIND1; ++i) {
    kmap[i] = std::max(0, g.kx_map[i]);
    kmap[NKIND1 + i] = std::max(0, g.ky_map[i]);
  }
  std::vector<int32_t> part_b, part_e, part_class, zloc_all;
  std::vector<int64_t> part_base, part_m;
  std::vector<int32_t> class_zoff;
  for (const PairClass& pc : g.pair_classes) {
    class_zoff.push_back((int32_t)zloc_all.size());
    zloc_all.insert(zloc_all.end(), pc.zloc.begin(), pc.zloc.end());
  }
  for (const PartInfo& pi : g.parts) {
    part_b.push_back(pi.b);
    part_e.push_back(pi.e);
    part_class.push_back(pi.pair_class);
    part_base.push_back((int64_t)pi.b * P);
    part_m.push_back(pi.m);
  }
  std::vector<int32_t> known_z(g.known_z.begin(), g.known_z.end());
  const int S = g.S;
  cudaError_t e = cudaSuccess;
#define VK_TRY(x)                                                           \
  if ((e = (x)) != cudaSuccess) {                                           \
    delete p;                                                               \
    return set_err(VK_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e)); \
  }
  VK_TRY(p->put(&p->d_known_z, known_z));
  VK_TRY(p->put(&p->d_miss_z, g.miss_z));
  VK_TRY(p->put(&p->d_miss_part, g.miss_part));
  VK_TRY(p->put(&p->d_miss_pattern, g.miss_pattern));
  VK_TRY(p->put(&p->d_miss_planes, g.miss_planes));
  VK_TRY(p->put(&p->d_sys_part, g.sys_part));
  VK_TRY(p->put(&p->d_sys_stencil, g.sys_stencil));
  if (!der_src.empty()) {
    VK_TRY(p->put(&p->d_der_src, der_src));
    VK_TRY(p->put(&p->d_der_flags, der_flags));
  }
  VK_TRY(p->put(&p->d_st_off, st_off));
  VK_TRY(p->put(&p->d_st_n, st_n));
  VK_TRY(p->put(&p->d_st_drift, st_drift));
  VK_TRY(p->put(&p->d_st_pattern, st_pattern));
  VK_TRY(p->put(&p->d_pat_dz, pat_dz));
  VK_TRY(p->put(&p->d_taps, taps));
  VK_TRY(p->put(&p->d_pad, pad));
  VK_TRY(p->put(&p->d_kmap, kmap));
  VK_TRY(p->put(&p->d_gap_part, g.gap_part));
  VK_TRY(p->put(&p->d_gap_pattern, g.gap_pattern));
  VK_TRY(p->put(&p->d_part_b, part_b));
  VK_TRY(p->put(&p->d_part_e, part_e));
  VK_TRY(p->put(&p->d_part_class, part_class));
  VK_TRY(p->put(&p->d_part_base, part_base));
  VK_TRY(p->put(&p->d_part_m, part_m));
  VK_TRY(p->put(&p->d_zloc, zloc_all));
  VK_TRY(p->alloc(&p->d_stats, (size_t)g.K * p->nchunk));
  VK_TRY(p->alloc(&p->d_models, (size_t)S * 3));
  VK_TRY(p->alloc(&p->d_lohi, (size_t)S * 2));
  VK_TRY(p->alloc(&p->d_part_status, (size_t)S));
  VK_TRY(p->alloc(&p->d_sys_status, (size_t)std::max(1, p->n_sys)));
  VK_TRY(p->alloc(&p->d_weights, (size_t)S * std::max(1, p->NP) * std::max(1, p->NK) * WPAD));
  VK_TRY(p->alloc(&p->d_var, (size_t)S * std::max(1, p->NP) * std::max(1, p->NK)));
  if (g.fast) VK_TRY(p->alloc(&p->d_kpm, kpm_elems(S, std::max(1, p->NK))));
  VK_TRY(p->alloc(&p->d_inexact, (size_t)g.K));
  VK_TRY(p->alloc(&p->d_work, (size_t)(S + 1) * 2));
  VK_TRY(cudaMemset(p->d_work, 0, (size_t)(S + 1) * 2 * sizeof(int)));
  if (g.fast && d->accum == VK_ACCUM_FIXED) {
    VK_TRY(p->alloc(&p->d_fxb, fxb_words(S, std::max(1, p->NK))));
    VK_TRY(p->alloc(&p->d_fxc, fxc_floats(S, std::max(1, p->NK))));
    VK_TRY(p->alloc(&p->d_fxq, (size_t)8));
  }
  for (int i = 0; i < vk_plan::NMODEL_RING; ++i) {
    VK_TRY(cudaMallocHost((void**)&p->h_models[i], (size_t)S * 3 * sizeof(double)));
    VK_TRY(cudaEventCreateWithFlags(&p->ev_models[i], cudaEventDisableTiming));
  }
  if (d->fit_variogram) {
    VK_TRY(p->alloc(&p->d_partial, (size_t)S * p->nblk * d->n_bins));
    for (size_t c = 0; c < g.pair_classes.size(); ++c) {
      PairTable t;
      VK_TRY(p->alloc(&t.ii, (size_t)d->max_pairs));
      VK_TRY(p->alloc(&t.jj, (size_t)d->max_pairs));
      VK_TRY(p->alloc(&t.bin, (size_t)d->max_pairs));
      VK_TRY(p->alloc(&t.counts, (size_t)MAX_BINS));
      VK_TRY(p->alloc(&t.scal, (size_t)4));
      const int64_t ns = pair_scratch_elems(g.pair_classes[c].m, d->max_pairs);
      VK_TRY(p->alloc(&t.cnt, (size_t)ns));
      VK_TRY(p->alloc(&t.off, (size_t)ns + 1));
      VK_TRY(p->alloc(&t.hbits, (size_t)1));
      VK_TRY(p->alloc(&t.order, (size_t)d->max_pairs));
      VK_TRY(p->alloc(&t.boff, (size_t)MAX_BINS + 1));
      VK_TRY(p->alloc(&t.ocnt, (size_t)order_chunks(d->max_pairs) * MAX_BINS));
      p->tables.push_back(t);
      // numpy's pairwise-summation tree for this class's sample count
      const NpSumWarpHost wh = build_npsum_warp(g.pair_classes[c].m);
      const NpSumTreeHost& th = wh.top;
      NpSumTree tr;
      tr.nleaf = (int32_t)wh.wr_leaf.size() - 1;
      tr.nnode = (int32_t)th.node_lr.size() / 2;
      tr.nlevel = (int32_t)th.level.size() - 1;
      int32_t *lo = nullptr, *lr = nullptr, *lv = nullptr, *wl = nullptr;
      int16_t* wp = nullptr;
      int8_t* wn = nullptr;
      VK_TRY(p->put(&lo, wh.leaf_off));
      VK_TRY(p->put(&lr, th.node_lr.empty() ? std::vector<int32_t>{0, 0} : th.node_lr));
      VK_TRY(p->put(&lv, th.level));
      VK_TRY(p->put(&wl, wh.wr_leaf));
      VK_TRY(p->put(&wp, wh.prog));
      VK_TRY(p->put(&wn, wh.nint));
      tr.leaf_off = lo;
      tr.node_lr = lr;
      tr.level = lv;
      tr.wr_leaf = wl;
      tr.wr_prog = wp;
      tr.wr_nint = wn;
      p->trees.push_back(tr);
      p->max_leaf = std::max(p->max_leaf, tr.nleaf);
      p->leaf_stride = std::max<int64_t>(p->leaf_stride, tr.nleaf);
      p->node_stride = std::max<int64_t>(p->node_stride, std::max(1, tr.nnode));
    }
    VK_TRY(p->put(&p->d_tables, p->tables));
    VK_TRY(p->put(&p->d_trees, p->trees));
    VK_TRY(p->alloc(&p->d_npleaf, (size_t)S * p->leaf_stride));
    VK_TRY(p->alloc(&p->d_npnode, (size_t)S * p->node_stride));
    VK_TRY(p->alloc(&p->d_mean, (size_t)S));
    VK_TRY(p->alloc(&p->d_svar, (size_t)S));
    VK_TRY(p->alloc(&p->d_sq, (size_t)S * d->max_pairs));
    VK_TRY(p->alloc(&p->d_bsum, (size_t)S * d->n_bins));
    {
      const Pcg64 gen = pcg64_from_seed(d->seed);
      int32_t zoff = 0;
      for (size_t c = 0; c < g.pair_classes.size(); ++c) {
        SampleGeom sg;
        sg.coords = nullptr;
        sg.zloc = p->d_zloc + zoff;
        sg.P = P;
        sg.W = g.W;
        zoff += (int32_t)g.pair_classes[c].zloc.size();
        p->jobs.push_back(make_pair_job((uint64_t)(gen.state >> 64), (uint64_t)gen.state,
                                        (uint64_t)(gen.inc >> 64), (uint64_t)gen.inc,
                                        g.pair_classes[c].m, d->max_pairs, d->n_bins, sg, p->tables[c]));
      }
      VK_TRY(p->put(&p->d_jobs, p->jobs));
    }
    {
      int lo_prio = 0, hi_prio = 0;
      VK_TRY(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
      VK_TRY(cudaStreamCreateWithPriority(&p->side, cudaStreamNonBlocking, hi_prio));
    }
    VK_TRY(cudaEventCreateWithFlags(&p->ev_fork, cudaEventDisableTiming));
    VK_TRY(cudaEventCreateWithFlags(&p->ev_join, cudaEventDisableTiming));
  }
  // per-part ranges for the overlapped schedule
  p->sys_begin.assign(S + 1, 0);
  for (int i = 0; i < p->n_sys; ++i) p->sys_begin[g.sys_part[i] + 1]++;
  for (int s = 0; s < S; ++s) p->sys_begin[s + 1] += p->sys_begin[s];
  for (int s = 0; s < S; ++s)
    if (p->sys_canon[s] < 0) p->sys_canon[s] = p->sys_begin[s];
  p->gap_begin.assign(S + 1, 0);
  if (g.fast) {
    for (int s = 0; s <= S; ++s) p->gap_begin[s] = (s < S) ? g.parts[s].b : g.K - 1;
    for (int s = 0; s < S; ++s) p->gap_begin[s] = std::min(p->gap_begin[s], g.K - 1);
    // shortest non-empty run of gaps owned by one part: a run of c gaps that
    // touches 4 parts holds 2 of them whole, so c <= 2 * min_len + 1 keeps
    // every unit within the kernel's 3 staged parts (FT_WPARTS)
    int min_len = g.K;
    for (int k = 0, run = 0; k < g.K - 1; ++k) {
      ++run;
      if (k == g.K - 2 || g.gap_part[k + 1] != g.gap_part[k]) { min_len = std::min(min_len, run); run = 0; }
    }
    p->max_chunk = 2 * std::max(1, min_len) + 1;
  }
  if (const char* e = std::getenv("VK_FIT_RESERVE")) p->fit_reserve = std::atoi(e);   // tuning
  // per-part chains are the default schedule whenever there is more than one
  // part on the streaming path; VK_FLAG_SERIAL keeps one stream (per-stage
  // timing, debugging)
  if (!(d->flags & VK_FLAG_SERIAL) && S > 1 && g.fast) {
    VK_TRY(cudaEventCreateWithFlags(&p->ev_kfork, cudaEventDisableTiming));
    VK_TRY(cudaEventCreateWithFlags(&p->ev_hstats, cudaEventDisableTiming));
    VK_TRY(cudaEventCreateWithFlags(&p->ev_hbins, cudaEventDisableTiming));
    // off by default: C4 measured 1.325 / 1.334 / 1.325 / 1.334 ms per step
    // with 0 / 2 / 4 / 8 head parts -- the head fits themselves (~0.1-0.2 ms
    // of TRF latency) and not the statistics gate the first predictions
    const char* hp = std::getenv("VK_HEAD_PARTS");
    p->head_parts = std::min(S - 1, std::max(0, hp ? std::atoi(hp) : 0));
    // fits and solves are latency chains: their streams get the highest
    // priority so a part's solve CTAs are placed ahead of the streaming CTAs
    // of parts already predicting; predicts run at the lowest priority
    int prio_lo = 0, prio_hi = 0;
    VK_TRY(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    for (int i = 0; i < std::min(S, vk_plan::NCH); ++i) {
      VK_TRY(cudaStreamCreateWithPriority(&p->chain[i], cudaStreamNonBlocking, prio_hi));
      VK_TRY(cudaStreamCreateWithPriority(&p->pchain[i], cudaStreamNonBlocking, prio_lo));
      VK_TRY(cudaEventCreateWithFlags(&p->ev_solved[i], cudaEventDisableTiming));
      VK_TRY(cudaEventCreateWithFlags(&p->ev_pjoin[i], cudaEventDisableTiming));
      VK_TRY(cudaEventCreateWithFlags(&p->ev_kjoin[i], cudaEventDisableTiming));
    }
  }
#undef VK_TRY
  (void)class_zoff;
  *out = p;
  return VK_OK;
}

void vk_plan_destroy(vk_plan* p) { delete p; }

int vk_plan_get_info(const vk_plan* p, vk_plan_info* info) {
  if (!p || !info) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  const Geometry& g = p->geo;
  info->fast_path = g.fast ? 1 : 0;
  info->gap_planes = g.G;
  info->n_patterns = p->NP;
  info->n_kinds = p->NK;
  info->n_systems = p->n_sys;
  info->n_missing_planes = (int32_t)g.miss_z.size();
  info->n_pair_classes = (int32_t)g.pair_classes.size();
  info->kernels_per_execute = p->kernels;
  info->interpolated_voxels = g.n_missing_voxels();
  return VK_OK;
}

int vk_plan_execute(vk_plan* p, const float* known, const double* models, float* out, double* var,
                    void* stream) {
  if (!p || !known || !out) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const Geometry& g = p->geo;
  const vk_plan_desc& d = p->desc;
  const int64_t P = (int64_t)g.H * g.W;
  const int S = g.S;
  int kernels = 0;
  const int slot = p->ring ? (int)(p->n_exec % p->ring) : 0;
  auto mark = [&](int stage) -> cudaError_t {
    if (!p->ring) return cudaSuccess;
    return cudaEventRecord(p->ev[(size_t)slot * (VK_N_STAGES + 1) + stage], st);
  };
  VK_CUDA(mark(0));
  // VK_CHAIN_TRACE (debug): per-part fit / solve / predict completion times
  static const bool trace = std::getenv("VK_CHAIN_TRACE") != nullptr;
  cudaEvent_t t_start = nullptr, t_pre[5] = {};     // draw, head bins, bins, head stats, stats
  if (trace) {
    cudaEventCreate(&t_start);
    cudaEventRecord(t_start, st);
    for (auto& e : t_pre) cudaEventCreate(&e);
  }
  if (!d.fit_variogram) {
    if (!models) return set_err(VK_E_INVALID_ARGUMENT, "models required when fit_variogram == 0");
    const int slot = p->models_slot;
    p->models_slot = (slot + 1) % vk_plan::NMODEL_RING;
    VK_CUDA(cudaEventSynchronize(p->ev_models[slot]));     // that slot's earlier copy has run
    std::memcpy(p->h_models[slot], models, (size_t)S * 3 * sizeof(double));
    VK_CUDA(cudaMemcpyAsync(p->d_models, p->h_models[slot], (size_t)S * 3 * sizeof(double),
                            cudaMemcpyHostToDevice, st));
    VK_CUDA(cudaEventRecord(p->ev_models[slot], st));
  }
  // the pair draw depends only on geometry and seed: fork it onto the side
  // stream so it overlaps the plane statistics
  const bool draw = d.fit_variogram && (!p->pairs_ready || (d.flags & VK_FLAG_REDRAW_PAIRS));
  // chained schedule: the binned semivariogram needs the pair tables and the
  // data, not the statistics, so it follows the draw on the side stream
  // (highest priority: the draw's small grids are placed first and the
  // statistics pass fills the remaining SMs)
  const bool side_bins = d.fit_variogram && p->chain[0] != nullptr;
  const bool fast = g.fast && predict_fast_supported(g.G, d.accum);
  const bool chained = p->chain[0] != nullptr && fast;
  // head parts: statistics of their planes and their bins are issued first
  // and signalled separately, so the first chains' fits start while the rest
  // of the volume is still being reduced
  const int H = chained ? p->head_parts : 0;
  const int kh = H > 0 ? g.parts[H - 1].e + 1 : 0;   // head planes [0, kh)
  BinSumArgs ba;
  ba.known = known;
  ba.values = nullptr;
  ba.part_base = p->d_part_base;
  ba.part_class = p->d_part_class;
  ba.tables = p->d_tables;
  ba.max_pairs = d.max_pairs;
  ba.n_bins = d.n_bins;
  ba.sq = p->d_sq;
  ba.bsum = p->d_bsum;
  ba.part0 = 0;
  ba.n_parts = S;
  NpVarArgs va;
  va.known = known;
  va.values = nullptr;
  va.part_base = p->d_part_base;
  va.part_m = p->d_part_m;
  va.part_class = p->d_part_class;
  va.trees = p->d_trees;
  va.max_leaf = p->max_leaf;
  va.leaf_stride = p->leaf_stride;
  va.node_stride = p->node_stride;
  va.leaf = p->d_npleaf;
  va.node = p->d_npnode;
  va.mean = p->d_mean;
  va.svar = p->d_svar;
  va.stats = p->d_stats;
  va.inexact = p->d_inexact;
  va.part_b = p->d_part_b;
  va.part_e = p->d_part_e;
  va.nchunk = p->nchunk;
  if (draw || side_bins) {
    VK_CUDA(cudaEventRecord(p->ev_fork, st));
    VK_CUDA(cudaStreamWaitEvent(p->side, p->ev_fork, 0));
    if (draw) {
      int nl = 0;
      VK_CUDA(launch_pair_tables(p->d_jobs, p->jobs.data(), (int)p->jobs.size(), p->side, &nl));
      kernels += nl;
      p->pairs_ready = true;
    }
    if (trace) cudaEventRecord(t_pre[0], p->side);
    if (side_bins && H > 0) {
      BinSumArgs b1 = ba;
      b1.part0 = 0;
      b1.n_parts = H;
      VK_CUDA(launch_binsums(b1, p->side));
      VK_CUDA(cudaEventRecord(p->ev_hbins, p->side));
      if (trace) cudaEventRecord(t_pre[1], p->side);
      b1.part0 = H;
      b1.n_parts = S - H;
      VK_CUDA(launch_binsums(b1, p->side));
      kernels += 4;
    } else if (side_bins) {
      VK_CUDA(launch_binsums(ba, p->side));
      kernels += 2;
    }
    if (trace) cudaEventRecord(t_pre[2], p->side);
    VK_CUDA(cudaEventRecord(p->ev_join, p->side));
  }
  if (H > 0) {
    VK_CUDA(launch_plane_stats(known, 0, kh, P, p->d_stats, p->nchunk, st, p->d_inexact));
    ++kernels;
    if (d.fit_variogram) {
      NpVarArgs v1 = va;
      v1.part0 = 0;
      v1.n_parts = H;
      VK_CUDA(launch_npvar(v1, st));
      kernels += 4;
    }
    VK_CUDA(cudaEventRecord(p->ev_hstats, st));
  }
  if (trace) cudaEventRecord(t_pre[3], st);
  VK_CUDA(launch_plane_stats(known, kh, g.K, P, p->d_stats, p->nchunk, st, p->d_inexact));
  ++kernels;
  if (d.fit_variogram) {
    NpVarArgs v1 = va;
    v1.part0 = H;
    v1.n_parts = S - H;
    VK_CUDA(launch_npvar(v1, st));
    kernels += 4;
  }
  if (trace) cudaEventRecord(t_pre[4], st);
  if (fast && d.accum == VK_ACCUM_FIXED) {
    VK_CUDA(launch_quant_range(p->d_stats, g.K * p->nchunk, p->d_fxq, st));
    ++kernels;
  }
  VK_CUDA(mark(1));
  if (draw || side_bins) VK_CUDA(cudaStreamWaitEvent(st, p->ev_join, 0));   // "pairs" = residual wait
  if (d.fit_variogram && !side_bins) {
    VK_CUDA(mark(2));
    VK_CUDA(launch_binsums(ba, st));
    kernels += 2;
  }
  if (!d.fit_variogram || side_bins) VK_CUDA(mark(2));
  VK_CUDA(mark(3));
  FitArgs fa;
  fa.S = S;
  fa.n_bins = d.n_bins;
  fa.nblk = p->nblk;
  fa.kind = d.kind;
  fa.fit = d.fit_variogram;
  fa.nchunk = p->nchunk;
  fa.stats = p->d_stats;
  fa.part_b = p->d_part_b;
  fa.part_e = p->d_part_e;
  fa.part_class = p->d_part_class;
  fa.part_m = p->d_part_m;
  fa.tables = p->d_tables;
  fa.partial = p->d_partial;
  fa.svar = p->d_svar;
  fa.bsum = p->d_bsum;
  fa.models = p->d_models;
  fa.lohi = p->d_lohi;
  fa.status = p->d_part_status;
  fa.part0 = 0;
  fa.n_parts = S;
  fa.reserve_smem = 0;
  SolveArgs sa;
  sa.n_sys = p->n_sys;
  sa.sys0 = 0;
  sa.kind = d.kind;
  sa.drift = d.drift;
  sa.NP = p->NP;
  sa.NK = p->NK;
  sa.sys_part = p->d_sys_part;
  sa.sys_stencil = p->d_sys_stencil;
  sa.st_off = p->d_st_off;
  sa.st_n = p->d_st_n;
  sa.st_drift = p->d_st_drift;
  sa.st_pattern = p->d_st_pattern;
  sa.taps = p->d_taps;
  sa.pad = p->d_pad;
  sa.pat_dz = p->d_pat_dz;
  sa.models = p->d_models;
  sa.weights = p->d_weights;
  sa.var = p->d_var;
  sa.sys_status = p->d_sys_status;
  sa.max_n = p->max_n;
  sa.max_dz = p->max_dz;
  sa.der_src = p->d_der_src;
  sa.der_flags = p->d_der_flags;
  PredictArgs pa;
  pa.known = known;
  pa.out = out;
  pa.var = var;
  pa.H = g.H;
  pa.W = g.W;
  pa.K = g.K;
  pa.NP = p->NP;
  pa.NK = p->NK;
  pa.accum = d.accum;
  pa.P = P;
  pa.known_z = p->d_known_z;
  pa.weights = p->d_weights;
  pa.svar = p->d_var;
  pa.lohi = p->d_lohi;
  pa.kmap = p->d_kmap;
  pa.nkx = g.nkx;
  pa.n_miss = (int)g.miss_z.size();
  pa.miss_z = p->d_miss_z;
  pa.miss_part = p->d_miss_part;
  pa.miss_pattern = p->d_miss_pattern;
  pa.miss_planes = p->d_miss_planes;
  pa.G = g.G;
  pa.gap0 = 0;
  pa.gap1 = g.K - 1;
  pa.chunk = 0;
  pa.gap_part = p->d_gap_part;
  pa.gap_pattern = p->d_gap_pattern;
  pa.part0 = 0;
  pa.part1 = S;
  pa.max_chunk = p->max_chunk;
  pa.kpm = p->d_kpm;
  pa.sd_inexact = p->d_inexact;
  pa.S = S;
  pa.fxb = p->d_fxb;
  pa.fxc = p->d_fxc;
  pa.fxq = p->d_fxq;
  pa.num_sms = p->num_sms;
  pa.work = p->d_work + 2 * S;
  if (fast) VK_CUDA(prepare_predict_fast(pa, &p->fast_launch));
  if (chained) {
    // ---- overlapped schedule: part s runs fit -> solve -> predict on chain
    // stream s % NCH; a part whose variogram fit converges early streams its
    // planes while slower fits are still iterating.
    VK_CUDA(cudaEventRecord(p->ev_kfork, st));
    const int nch = std::min(S, vk_plan::NCH);
    // head chains start from their own statistics and bins; every other
    // chain (and a head chain's later parts when S > NCH) from the fork
    for (int c = 0; c < nch; ++c) {
      if (c < H) {
        VK_CUDA(cudaStreamWaitEvent(p->chain[c], p->ev_hstats, 0));
        if (side_bins) VK_CUDA(cudaStreamWaitEvent(p->chain[c], p->ev_hbins, 0));
        // fixed path: the quantisation range covers the whole volume
        if (d.accum == VK_ACCUM_FIXED) VK_CUDA(cudaStreamWaitEvent(p->pchain[c], p->ev_kfork, 0));
      } else {
        VK_CUDA(cudaStreamWaitEvent(p->chain[c], p->ev_kfork, 0));
      }
    }
    std::vector<cudaEvent_t> tev;
    if (trace) {
      tev.resize(1 + 3 * S);
      for (auto& e : tev) cudaEventCreate(&e);
      cudaEventRecord(tev[0], st);
    }
    // breadth-first launch order (all fits, then all solves, then all
    // predicts): a chain's solve waits on its fit, and a waiting kernel at
    // the head of a hardware work queue would block the fits queued behind it
    for (int s = 0; s < S; ++s) {
      if (s >= nch && s % nch < H && s < nch + H) VK_CUDA(cudaStreamWaitEvent(p->chain[s % nch], p->ev_kfork, 0));
      FitArgs f1 = fa;
      f1.part0 = s;
      f1.n_parts = 1;
      f1.reserve_smem = p->fit_reserve;
      // VK_DIAG_SKIP (diagnostics only: results reuse the previous execute's
      // models / weights): bit 1 skips fits, bit 2 skips solves after the first execute
      static const int diag_skip = std::getenv("VK_DIAG_SKIP") ? std::atoi(std::getenv("VK_DIAG_SKIP")) : 0;
      if (!(diag_skip & 1) || p->n_runs == 0) VK_CUDA(launch_fit(f1, p->chain[s % nch]));
      ++kernels;
      if (trace) cudaEventRecord(tev[1 + 3 * s], p->chain[s % nch]);
    }
    for (int s = 0; s < S; ++s) {
      SolveArgs s1 = sa;
      s1.sys0 = p->sys_begin[s];
      s1.n_sys = p->sys_canon[s] - p->sys_begin[s];          // solved systems of the part
      SolveArgs d1 = sa;
      d1.sys0 = p->sys_canon[s];
      d1.n_sys = p->sys_begin[s + 1] - p->sys_canon[s];      // its mirror / transpose images
      static const int diag_skip2 = std::getenv("VK_DIAG_SKIP") ? std::atoi(std::getenv("VK_DIAG_SKIP")) : 0;
      if (!(diag_skip2 & 2) || p->n_runs == 0) {
        VK_CUDA(launch_solve(s1, p->chain[s % nch]));
        VK_CUDA(launch_derive(d1, p->chain[s % nch]));
      }
      kernels += (s1.n_sys > 0) + (d1.n_sys > 0 && d1.der_src);
      if (trace) cudaEventRecord(tev[2 + 3 * s], p->chain[s % nch]);
    }
    for (int s = 0; s < S; ++s) {
      PredictArgs p1 = pa;
      p1.gap0 = p->gap_begin[s];
      p1.gap1 = p->gap_begin[s + 1];
      // units of half a part's gaps: streaming CTAs retire often enough that
      // a late part's solve finds a free slot soon (they hold all of an SM's
      // registers), at the cost of one extra known-plane load per unit
      // (C4: 8-gap units 1.351 ms, 4-gap 1.329 ms, 2-gap 1.342 ms with the
      // round-1 fit).  With the exact fit the step ends with the slowest
      // part's prediction alone on the GPU, where shorter units spread its
      // gaps over more CTAs: a quarter of the part's gaps when a gap is seven
      // or more interpolated planes (C4: 2 / 3 / 4 / 8-gap units 2.051 / 2.062
      // / 2.069 / 2.097 ms); at smaller G the unit's extra known plane weighs
      // more and the step is bandwidth-bound (C5), so half a part stays
      static const int chain_chunk = std::getenv("VK_CHAIN_CHUNK") ? std::atoi(std::getenv("VK_CHAIN_CHUNK")) : 0;
      const int part_gaps = p1.gap1 - p1.gap0;
      const int div = g.G >= 7 ? 4 : 2;
      p1.chunk = part_gaps > 4 ? std::max(2, (part_gaps + div - 1) / div) : part_gaps;
      if (chain_chunk > 0) p1.chunk = std::min(part_gaps, chain_chunk);
      p1.part0 = s;
      p1.part1 = s + 1;
      p1.work = p->d_work + 2 * s;
      // the part's solve finished on its high-priority chain (a part reuses
      // a chain slot only when S > NCH, in launch order, so the event
      // recorded last on the slot covers this part)
      VK_CUDA(cudaEventRecord(p->ev_solved[s % nch], p->chain[s % nch]));
      VK_CUDA(cudaStreamWaitEvent(p->pchain[s % nch], p->ev_solved[s % nch], 0));
      // VK_DIAG_SKIP bit 4 (diagnostics only): no prediction launches
      static const int diag_skip4 = std::getenv("VK_DIAG_SKIP") ? std::atoi(std::getenv("VK_DIAG_SKIP")) : 0;
      if (!(diag_skip4 & 4)) VK_CUDA(launch_predict_fast_prepared(p->fast_launch, p1, p->pchain[s % nch]));
      kernels += 2;
      if (trace) cudaEventRecord(tev[3 + 3 * s], p->pchain[s % nch]);
    }
    for (int c = 0; c < nch; ++c) {
      VK_CUDA(cudaEventRecord(p->ev_kjoin[c], p->chain[c]));
      VK_CUDA(cudaStreamWaitEvent(st, p->ev_kjoin[c], 0));
      VK_CUDA(cudaEventRecord(p->ev_pjoin[c], p->pchain[c]));
      VK_CUDA(cudaStreamWaitEvent(st, p->ev_pjoin[c], 0));
    }
    if (trace) {
      cudaStreamSynchronize(st);
      float f0 = 0;
      cudaEventElapsedTime(&f0, t_start, tev[0]);
      std::fprintf(stderr, "fork at %.3f ms after the step start\n", f0);
      const char* names[5] = {"draw", "head bins", "bins", "head stats", "stats"};
      for (int i = 0; i < 5; ++i) {
        float t = -1;
        if (cudaEventElapsedTime(&t, t_start, t_pre[i]) != cudaSuccess) t = -1;
        std::fprintf(stderr, "  %s done at %.3f ms\n", names[i], t);
      }
      for (auto& e : t_pre) cudaEventDestroy(e);
      for (int s2 = 0; s2 < S; ++s2) {
        float f = 0, v = 0, q = 0;
        cudaEventElapsedTime(&f, tev[0], tev[1 + 3 * s2]);
        cudaEventElapsedTime(&v, tev[0], tev[2 + 3 * s2]);
        cudaEventElapsedTime(&q, tev[0], tev[3 + 3 * s2]);
        std::fprintf(stderr, "chain %2d fit %.3f solve %.3f predict %.3f ms\n", s2, f, v, q);
      }
      for (auto& e : tev) cudaEventDestroy(e);
      cudaEventDestroy(t_start);
      (void)cudaGetLastError();                  // elapsed-time queries on unrecorded events
    }
    VK_CUDA(mark(4));
    VK_CUDA(mark(5));
  } else {
    VK_CUDA(launch_fit(fa, st));
    ++kernels;
    VK_CUDA(mark(4));
    VK_CUDA(launch_solve(sa, st));
    VK_CUDA(launch_derive(sa, st));
    if (p->n_sys) kernels += 1 + (p->n_derived > 0);
    // the stencil tables derive from the solved weights: they close the
    // solve stage, so the prediction stage times the streaming kernel alone
    if (fast && d.accum != VK_ACCUM_FIXED) {
      VK_CUDA(launch_predict_fast_tables(pa, st));
      pa.tables_done = 1;
    }
    VK_CUDA(mark(5));
    if (fast) {
      VK_CUDA(launch_predict_fast_prepared(p->fast_launch, pa, st));
      kernels += 2;                             // stencil table + streaming kernel
    } else {
      VK_CUDA(launch_copy_known(pa, st));
      VK_CUDA(launch_predict_generic(pa, st));
      kernels += 1 + (pa.n_miss > 0);
    }
  }
  VK_CUDA(mark(6));
  if (p->ring) ++p->n_exec;
  ++p->n_runs;
  p->kernels = kernels;
  return VK_OK;
}

int vk_fill_generic(const float* data, const uint8_t* mask, int32_t depth, int32_t height, int32_t width,
                    int32_t kind, int32_t drift, const double* model, double lo, double hi, float* out,
                    double* var, int64_t* info, void* stream) {
  if (!data || !mask || !model || !out) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  if (depth < 1 || height < 1 || width < 1) return set_err(VK_E_INVALID_ARGUMENT, "dims");
  if (kind < 0 || kind > 2) return set_err(VK_E_INVALID_ARGUMENT, "kind");
  if (drift < 0 || drift > 1) return set_err(VK_E_INVALID_ARGUMENT, "drift");
  const GenericResult r = fill_generic(data, mask, depth, height, width, model, kind, drift, lo, hi, out, var,
                                       (cudaStream_t)stream);
  if (info) {
    info[0] = r.failed;
    info[1] = r.n_systems;
    info[2] = r.n_missing;
  }
  switch (r.status) {
    case 0: return VK_OK;
    case 2: return set_err(VK_E_NO_KNOWN_NEIGHBORS, r.msg);
    case 3: return set_err(VK_E_SINGULAR_SYSTEM, r.msg);
    case 6: return set_err(VK_E_UNSUPPORTED, r.msg);
    default: return set_err(VK_E_CUDA, r.msg);
  }
}

int vk_solve_systems(const int16_t* rel, const int64_t* offsets, int32_t n_systems, int32_t kind, int32_t drift,
                     const double* model, double* weights, double* variance, int32_t* status, void* stream) {
  if (!rel || !offsets || !model || !weights || !variance || n_systems < 1)
    return set_err(VK_E_INVALID_ARGUMENT, "null argument or no systems");
  if (kind < 0 || kind > 2) return set_err(VK_E_INVALID_ARGUMENT, "kind");
  if (drift < 0 || drift > 1) return set_err(VK_E_INVALID_ARGUMENT, "drift");
  std::vector<int64_t> off(offsets, offsets + n_systems + 1);
  for (int i = 0; i < n_systems; ++i) {
    const int64_t n = off[i + 1] - off[i];
    if (n <= 0) return set_err(VK_E_NO_KNOWN_NEIGHBORS, "cannot build a system with zero neighbors");
    if (n > 1024) return set_err(VK_E_UNSUPPORTED, "a system with more than 1024 neighbours");
  }
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* d_status = nullptr;
  VK_CUDA(cudaMallocAsync((void**)&d_status, n_systems * sizeof(int32_t), st));
  cudaError_t e = solve_systems_device(rel, off, kind, drift, model, weights, variance, d_status, st);
  std::vector<int32_t> hs(n_systems, 0);
  if (e == cudaSuccess) e = cudaMemcpyAsync(hs.data(), d_status, n_systems * 4, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d_status, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return set_err(VK_E_CUDA, std::string("vk_solve_systems: ") + cudaGetErrorString(e));
  bool bad = false;
  for (int i = 0; i < n_systems; ++i) {
    if (status) status[i] = hs[i] == PS_OK ? 0 : 1;
    bad |= hs[i] != PS_OK;
  }
  return bad ? set_err(VK_E_SINGULAR_SYSTEM, "extended kriging matrix is singular") : VK_OK;
}

int vk_crc32(const void* data, int64_t n_bytes, uint32_t crc_in, uint32_t* crc_out, void* stream) {
  if ((!data && n_bytes > 0) || !crc_out || n_bytes < 0) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  VK_CUDA(crc32_device(data, n_bytes, crc_in, crc_out, (cudaStream_t)stream));
  return VK_OK;
}

int vk_packbits(const uint8_t* mask, int64_t n, uint8_t* bits, void* stream) {
  if ((!mask || !bits) && n > 0) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  VK_CUDA(packbits_device(mask, n, bits, (cudaStream_t)stream));
  return VK_OK;
}

int vk_unpackbits(const uint8_t* bits, int64_t n, uint8_t* mask, void* stream) {
  if ((!mask || !bits) && n > 0) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  VK_CUDA(unpackbits_device(bits, n, mask, (cudaStream_t)stream));
  return VK_OK;
}

int vk_decode_samples(const void* raw, int32_t sample_type, int64_t n, float* out, void* stream) {
  if (sample_type < VK_SAMPLE_U8 || sample_type > VK_SAMPLE_F32 || n < 0)
    return set_err(VK_E_INVALID_ARGUMENT, "bad sample type / count");
  if ((!raw || !out) && n > 0) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  VK_CUDA(decode_samples_device(raw, sample_type, n, out, (cudaStream_t)stream));
  return VK_OK;
}

int vk_normalize_stack(const void* raw, int32_t sample_type, int64_t n, float* out, int32_t* minmax,
                       void* stream) {
  if (sample_type < VK_SAMPLE_U8 || sample_type > VK_SAMPLE_F32 || n < 0)
    return set_err(VK_E_INVALID_ARGUMENT, "bad sample type / count");
  if ((!raw || !out) && n > 0) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  if (out == raw && sample_type != VK_SAMPLE_F32 && n > 0)
    return set_err(VK_E_INVALID_ARGUMENT, "in-place normalisation needs f32 samples");
  cudaStream_t st = (cudaStream_t)stream;
  int* keys = minmax;
  if (!keys) VK_CUDA(cudaMallocAsync((void**)&keys, 2 * sizeof(int), st));
  const cudaError_t e = normalize_stack_device(raw, sample_type, n, out, keys, st);
  if (!minmax) cudaFreeAsync(keys, st);
  VK_CUDA(e);
  return VK_OK;
}

int vk_plan_set_timing(vk_plan* p, int ring) {
  if (!p || ring < 0) return set_err(VK_E_INVALID_ARGUMENT, "bad plan / ring");
  for (cudaEvent_t e : p->ev) cudaEventDestroy(e);
  p->ev.clear();
  p->ring = 0;
  p->n_exec = 0;
  for (int i = 0; i < ring * (VK_N_STAGES + 1); ++i) {
    cudaEvent_t e;
    VK_CUDA(cudaEventCreate(&e));
    p->ev.push_back(e);
  }
  p->ring = ring;
  return VK_OK;
}

int vk_plan_stage_ms(vk_plan* p, int back, float* ms) {
  if (!p || !ms) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  if (!p->ring) return set_err(VK_E_INVALID_ARGUMENT, "timing not enabled");
  if (back < 0 || back >= p->ring || back >= p->n_exec) return set_err(VK_E_INVALID_ARGUMENT, "no such execute");
  const int slot = (int)((p->n_exec - 1 - back) % p->ring);
  cudaEvent_t* e = &p->ev[(size_t)slot * (VK_N_STAGES + 1)];
  VK_CUDA(cudaEventSynchronize(e[VK_N_STAGES]));
  for (int i = 0; i < VK_N_STAGES; ++i) {
    float t = 0.f;
    VK_CUDA(cudaEventElapsedTime(&t, e[i], e[i + 1]));
    ms[i] = t;
  }
  return VK_OK;
}

namespace {
// known planes of a downloaded volume, copied by host threads
struct HostPlaneCopy {
  char* dst;
  const char* src;
  size_t plane;
  std::vector<int> z;     // destination plane of known slice k
};
void CUDART_CB host_plane_copy(void* arg) {
  std::unique_ptr<HostPlaneCopy> j(static_cast<HostPlaneCopy*>(arg));
  static const int env_threads = std::getenv("VK_HOST_COPY_THREADS") ? std::atoi(std::getenv("VK_HOST_COPY_THREADS")) : 0;
  const int K = (int)j->z.size();
  const int hw = (int)std::max(1u, std::thread::hardware_concurrency());
  // 4 threads: the copy shares host memory bandwidth with the concurrent
  // device-to-host DMA (C4 e2e 39.3 / 37.9 / 38.0 / 39.3 ms per step with
  // 8 / 4 / 2 / 16 threads on a 16-core host)
  const int nt = std::max(1, std::min({K, env_threads > 0 ? env_threads : std::min(4, hw)}));
  auto work = [&](int t) {
    for (int k = t; k < K; k += nt) std::memcpy(j->dst + (size_t)j->z[k] * j->plane, j->src + (size_t)k * j->plane, j->plane);
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
}
}  // namespace

int vk_plan_download(vk_plan* p, const float* out_dev, const float* known_host, float* out_host, void* stream) {
  if (!p || !out_dev || !known_host || !out_host) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  cudaStream_t st = (cudaStream_t)stream;
  const Geometry& g = p->geo;
  const size_t plane = (size_t)g.H * g.W * sizeof(float);
  if (!p->io) {
    VK_CUDA(cudaStreamCreateWithFlags(&p->io, cudaStreamNonBlocking));
    VK_CUDA(cudaEventCreateWithFlags(&p->ev_io_fork, cudaEventDisableTiming));
    VK_CUDA(cudaEventCreateWithFlags(&p->ev_io_join, cudaEventDisableTiming));
  }
  const int K = g.K;
  bool regular = K >= 2 && g.known_z[0] == 0 && g.known_z[K - 1] == g.T - 1;
  const int f = K >= 2 ? g.known_z[1] - g.known_z[0] : 1;
  for (int k = 1; regular && k < K; ++k) regular = g.known_z[k] - g.known_z[k - 1] == f;
  char* oh = reinterpret_cast<char*>(out_host);
  const char* od = reinterpret_cast<const char*>(out_dev);
  // known planes: copied on the host from the caller's input (the device
  // holds bit-identical copies, kriging.py:481) by a host function on the
  // plan's io stream -- worker threads, concurrent with the DMA below, and
  // ordered after everything the caller queued before this call (the fork
  // is recorded before the download is queued, so the two overlap)
  VK_CUDA(cudaEventRecord(p->ev_io_fork, st));
  VK_CUDA(cudaStreamWaitEvent(p->io, p->ev_io_fork, 0));
  auto* job = new HostPlaneCopy{oh, reinterpret_cast<const char*>(known_host), plane, g.known_z};
  const cudaError_t ce = cudaLaunchHostFunc(p->io, host_plane_copy, job);
  if (ce != cudaSuccess) {
    delete job;
    VK_CUDA(ce);
  }
  // interpolated planes: device to host on the caller's stream
  if (regular) {
    if (f > 1)     // every gap's f - 1 interpolated planes: one strided copy
      VK_CUDA(cudaMemcpy2DAsync(oh + plane, f * plane, od + plane, f * plane, (f - 1) * plane, K - 1,
                                cudaMemcpyDeviceToHost, st));
  } else {
    int z = 0;
    for (int k = 0; k <= K; ++k) {                 // runs of missing planes between known ones
      const int z1 = k < K ? g.known_z[k] : g.T;
      if (z1 > z)
        VK_CUDA(cudaMemcpyAsync(oh + (size_t)z * plane, od + (size_t)z * plane, (size_t)(z1 - z) * plane,
                                cudaMemcpyDeviceToHost, st));
      z = z1 + 1;
    }
  }
  VK_CUDA(cudaEventRecord(p->ev_io_join, p->io));
  VK_CUDA(cudaStreamWaitEvent(st, p->ev_io_join, 0));
  return VK_OK;
}

int vk_plan_finish(vk_plan* p, void* stream, int32_t* failed_part, double* models_out, double* lohi_out) {
  if (!p) return set_err(VK_E_INVALID_ARGUMENT, "null plan");
  cudaStream_t st = (cudaStream_t)stream;
  VK_CUDA(cudaStreamSynchronize(st));
  const int S = p->geo.S;
  std::vector<int32_t> ps(S), ss(std::max(1, p->n_sys));
  VK_CUDA(cudaMemcpy(ps.data(), p->d_part_status, S * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (p->n_sys)
    VK_CUDA(cudaMemcpy(ss.data(), p->d_sys_status, p->n_sys * sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (models_out)
    VK_CUDA(cudaMemcpy(models_out, p->d_models, (size_t)S * 3 * sizeof(double), cudaMemcpyDeviceToHost));
  if (lohi_out)
    VK_CUDA(cudaMemcpy(lohi_out, p->d_lohi, (size_t)S * 2 * sizeof(double), cudaMemcpyDeviceToHost));
  if (failed_part) *failed_part = -1;
  for (int s = 0; s < S; ++s) {
    if (ps[s] != PS_OK) {
      if (failed_part) *failed_part = s;
      const char* why = ps[s] == PS_NONFINITE      ? "known voxels must be finite"
                        : ps[s] == PS_INSUFFICIENT ? "too few samples: need >= 30 pairs"
                        : ps[s] == PS_DEGENERATE   ? "all sample pairs are co-located"
                        : ps[s] == PS_FIT_FAILED   ? "variogram fit failed"
                        : ps[s] == PS_SINGULAR     ? "extended kriging matrix is singular"
                                                   : "device status";
      return set_err(status_from_part(ps[s]), "sub-part " + std::to_string(s) + ": " + why + " (status " +
                                                  std::to_string(ps[s]) + ")");
    }
  }
  for (int i = 0; i < p->n_sys; ++i) {
    if (ss[i] != PS_OK) {
      if (failed_part) *failed_part = p->geo.sys_part[i];
      return set_err(VK_E_SINGULAR_SYSTEM, "extended kriging matrix is singular");
    }
  }
  return VK_OK;
}

int vk_plan_get_systems(vk_plan* p, double* weights, double* variance, int32_t* ids) {
  if (!p) return set_err(VK_E_INVALID_ARGUMENT, "null plan");
  const Geometry& g = p->geo;
  const size_t nslot = (size_t)g.S * std::max(1, p->NP) * std::max(1, p->NK);
  std::vector<double> w(nslot * WPAD), v(nslot);
  VK_CUDA(cudaDeviceSynchronize());
  VK_CUDA(cudaMemcpy(w.data(), p->d_weights, w.size() * sizeof(double), cudaMemcpyDeviceToHost));
  VK_CUDA(cudaMemcpy(v.data(), p->d_var, v.size() * sizeof(double), cudaMemcpyDeviceToHost));
  for (int i = 0; i < p->n_sys; ++i) {
    const int s = g.sys_part[i], stc = g.sys_stencil[i];
    const StencilGeom& sg = g.stencils[stc];
    const size_t slot = ((size_t)s * p->NP + sg.pattern) * p->NK + (stc % p->NK);
    if (weights) std::memcpy(weights + (size_t)i * WPAD, &w[slot * WPAD], WPAD * sizeof(double));
    if (variance) variance[i] = v[slot];
    if (ids) {
      ids[4 * i + 0] = s;
      ids[4 * i + 1] = sg.pattern;
      ids[4 * i + 2] = sg.ky;
      ids[4 * i + 3] = sg.kx;
    }
  }
  return VK_OK;
}

int vk_sample_pairs(int64_t m, int64_t max_pairs, uint64_t seed, int32_t* ii, int32_t* jj, int64_t* n_out,
                    void* stream) {
  if (m < 2 || m > 0xffffffffll || max_pairs < 1) return set_err(VK_E_INVALID_ARGUMENT, "m / max_pairs");
  cudaStream_t st = (cudaStream_t)stream;
  PairTable t;
  t.ii = ii;
  t.jj = jj;
  VK_CUDA(cudaMalloc((void**)&t.bin, (size_t)max_pairs));
  VK_CUDA(cudaMalloc((void**)&t.counts, MAX_BINS * sizeof(int64_t)));
  VK_CUDA(cudaMalloc((void**)&t.scal, 4 * sizeof(double)));
  const int64_t ns = pair_scratch_elems(m, max_pairs);
  VK_CUDA(cudaMalloc((void**)&t.cnt, ns * sizeof(int32_t)));
  VK_CUDA(cudaMalloc((void**)&t.off, (ns + 1) * sizeof(int64_t)));
  VK_CUDA(cudaMalloc((void**)&t.hbits, sizeof(unsigned long long)));
  int32_t* zl = nullptr;
  VK_CUDA(cudaMalloc((void**)&zl, sizeof(int32_t)));
  VK_CUDA(cudaMemsetAsync(zl, 0, sizeof(int32_t), st));
  const Pcg64 gen = pcg64_from_seed(seed);
  SampleGeom sg;
  sg.coords = nullptr;
  sg.zloc = zl;
  sg.P = m;            // one "plane" holding every sample: lags unused here
  sg.W = (int32_t)std::min<int64_t>(m, 1 << 30);
  const PairJob job = make_pair_job((uint64_t)(gen.state >> 64), (uint64_t)gen.state,
                                    (uint64_t)(gen.inc >> 64), (uint64_t)gen.inc, m, max_pairs, 15, sg, t);
  PairJob* d_job = nullptr;
  cudaError_t e = cudaMalloc((void**)&d_job, sizeof(PairJob));
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_job, &job, sizeof(PairJob), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = launch_pair_tables(d_job, &job, 1, st);
  double scal[4] = {0, 0, 0, 0};
  if (e == cudaSuccess) e = cudaMemcpyAsync(scal, t.scal, sizeof(scal), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFree(d_job);
  cudaFree(t.bin);
  cudaFree(t.counts);
  cudaFree(t.scal);
  cudaFree(t.cnt);
  cudaFree(t.off);
  cudaFree(t.hbits);
  cudaFree(zl);
  if (e != cudaSuccess) return set_err(VK_E_CUDA, cudaGetErrorString(e));
  if (n_out) *n_out = (int64_t)scal[2];
  return scal[3] == 0.0 ? VK_OK : set_err(VK_E_CUDA, "pair draw ran short");
}

int vk_fit_variogram_samples(const double* coords, const double* values, int64_t m, int32_t kind,
                             int32_t n_bins, int64_t max_pairs, uint64_t seed, double* model_out,
                             void* stream) {
  if (!coords || !values || !model_out) return set_err(VK_E_INVALID_ARGUMENT, "null argument");
  if (kind < 0 || kind > 2 || n_bins < 1 || n_bins > MAX_BINS || max_pairs < 1)
    return set_err(VK_E_INVALID_ARGUMENT, "kind / n_bins / max_pairs");
  if (m * (m - 1) / 2 < 30)
    return set_err(VK_E_INSUFFICIENT_SAMPLES, std::to_string(m) + " samples give " +
                                                  std::to_string(m * (m - 1) / 2) + " pairs; need >= 30");
  if (m > 0xffffffffll) return set_err(VK_E_UNSUPPORTED, "more than 2^32 samples");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t npmax = std::min<int64_t>(max_pairs, m * (m - 1) / 2);
  const int nchunk = (int)((m + STATS_CHUNK - 1) / STATS_CHUNK);
  const int nblk = (int)std::max<int64_t>(1, (npmax + 4095) / 4096);
  // device scratch: the blocks of the previous call are reused in allocation
  // order (grown when too small), so repeated drop-in calls do no cudaMalloc /
  // cudaFree (each a device synchronisation); calls are serialised, and each
  // call synchronises its stream before it returns
  static std::mutex scratch_mu;
  static std::vector<std::pair<void*, size_t>> scratch;
  std::lock_guard<std::mutex> scratch_lock(scratch_mu);
  std::vector<void*> mem;
  size_t n_get = 0;
  auto get = [&](size_t bytes) -> void* {
    bytes = (std::max<size_t>(bytes, 8) + 255) & ~(size_t)255;
    if (n_get == scratch.size()) scratch.push_back({nullptr, 0});
    auto& blk = scratch[n_get++];
    if (blk.second < bytes) {
      if (blk.first) cudaFree(blk.first);
      blk = {nullptr, 0};
      void* q = nullptr;
      if (cudaMalloc(&q, bytes) == cudaSuccess) blk = {q, bytes};
    }
    mem.push_back(blk.first);
    return blk.first;
  };
  PairTable t;
  t.ii = (int32_t*)get(npmax * 4);
  t.jj = (int32_t*)get(npmax * 4);
  t.bin = (uint8_t*)get(npmax);
  t.counts = (int64_t*)get(MAX_BINS * 8);
  t.scal = (double*)get(4 * 8);
  const int64_t ns = pair_scratch_elems(m, max_pairs);
  t.cnt = (int32_t*)get((size_t)ns * 4);
  t.off = (int64_t*)get((size_t)(ns + 1) * 8);
  t.hbits = (unsigned long long*)get(8);
  t.order = (int32_t*)get((size_t)npmax * 4);
  t.boff = (int32_t*)get((MAX_BINS + 1) * 4);
  t.ocnt = (int32_t*)get((size_t)order_chunks(npmax) * MAX_BINS * 4);
  PairTable* d_t = (PairTable*)get(sizeof(PairTable));
  ChunkStat* stats = (ChunkStat*)get((size_t)nchunk * sizeof(ChunkStat));
  double* partial = (double*)get((size_t)nblk * n_bins * 8);
  // numpy's pairwise-sum decomposition depends only on m: built once per m
  // (2 ms on the host for a C4 sub-part's 786 k samples, 13 ms for 2.4 M)
  static std::vector<std::pair<int64_t, std::shared_ptr<const NpSumWarpHost>>> np_cache;
  std::shared_ptr<const NpSumWarpHost> whp;
  for (auto& c : np_cache)
    if (c.first == m) whp = c.second;
  if (!whp) {
    whp = std::make_shared<const NpSumWarpHost>(build_npsum_warp(m));
    if (np_cache.size() >= 8) np_cache.erase(np_cache.begin());
    np_cache.push_back({m, whp});
  }
  const NpSumWarpHost& wh = *whp;
  const NpSumTreeHost& th = wh.top;
  NpSumTree tr;
  tr.nleaf = (int32_t)wh.wr_leaf.size() - 1;
  tr.nnode = (int32_t)th.node_lr.size() / 2;
  tr.nlevel = (int32_t)th.level.size() - 1;
  int32_t* t_lo = (int32_t*)get(wh.leaf_off.size() * 4);
  int32_t* t_lr = (int32_t*)get(std::max<size_t>(2, th.node_lr.size()) * 4);
  int32_t* t_lv = (int32_t*)get(th.level.size() * 4);
  int32_t* t_wl = (int32_t*)get(wh.wr_leaf.size() * 4);
  int16_t* t_wp = (int16_t*)get(wh.prog.size() * 2);
  int8_t* t_wn = (int8_t*)get(wh.nint.size());
  tr.leaf_off = t_lo;
  tr.node_lr = t_lr;
  tr.level = t_lv;
  tr.wr_leaf = t_wl;
  tr.wr_prog = t_wp;
  tr.wr_nint = t_wn;
  NpSumTree* d_tr = (NpSumTree*)get(sizeof(NpSumTree));
  double* npleaf = (double*)get((size_t)std::max(1, tr.nleaf) * 8);
  double* npnode = (double*)get((size_t)std::max(1, tr.nnode) * 8);
  double* npstat = (double*)get(2 * 8);
  double* sq = (double*)get((size_t)npmax * 8);
  double* bsum = (double*)get((size_t)n_bins * 8);
  double* models = (double*)get(3 * 8);
  double* lohi = (double*)get(2 * 8);
  int32_t* status = (int32_t*)get(4);
  int32_t* zero32 = (int32_t*)get(8);
  int64_t* zero64 = (int64_t*)get(8);
  int64_t* mm = (int64_t*)get(8);
  auto cleanup = [&]() {};                     // scratch stays cached for the next call
  for (void* q : mem)
    if (!q) { cleanup(); return set_err(VK_E_CUDA, "cudaMalloc failed"); }
  cudaError_t e = cudaMemcpyAsync(d_t, &t, sizeof(PairTable), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t_lo, wh.leaf_off.data(), wh.leaf_off.size() * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t_wl, wh.wr_leaf.data(), wh.wr_leaf.size() * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t_wp, wh.prog.data(), wh.prog.size() * 2, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t_wn, wh.nint.data(), wh.nint.size(), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess && !th.node_lr.empty())
    e = cudaMemcpyAsync(t_lr, th.node_lr.data(), th.node_lr.size() * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(t_lv, th.level.data(), th.level.size() * 4, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_tr, &tr, sizeof(NpSumTree), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(zero32, 0, 8, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(zero64, 0, 8, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(mm, &m, 8, cudaMemcpyHostToDevice, st);
  const Pcg64 gen = pcg64_from_seed(seed);
  SampleGeom sg;
  sg.coords = coords;
  sg.zloc = nullptr;
  sg.P = m;
  sg.W = 1;
  const PairJob job = make_pair_job((uint64_t)(gen.state >> 64), (uint64_t)gen.state,
                                    (uint64_t)(gen.inc >> 64), (uint64_t)gen.inc, m, max_pairs, n_bins, sg, t);
  PairJob* d_job = (PairJob*)get(sizeof(PairJob));
  if (!d_job) { cleanup(); return set_err(VK_E_CUDA, "cudaMalloc failed"); }
  if (e == cudaSuccess) e = cudaMemcpyAsync(d_job, &job, sizeof(PairJob), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = launch_pair_tables(d_job, &job, 1, st);
  if (e == cudaSuccess) e = launch_plane_stats_f64(values, m, stats, nchunk, st);
  NpVarArgs va;
  va.known = nullptr;
  va.values = values;
  va.part_base = zero64;
  va.part_m = mm;
  va.part_class = zero32;
  va.trees = d_tr;
  va.part0 = 0;
  va.n_parts = 1;
  va.max_leaf = tr.nleaf;
  va.leaf_stride = tr.nleaf;
  va.node_stride = std::max(1, tr.nnode);
  va.leaf = npleaf;
  va.node = npnode;
  va.mean = npstat;
  va.svar = npstat + 1;
  if (e == cudaSuccess) e = launch_npvar(va, st);
  BinSumArgs ba;
  ba.known = nullptr;
  ba.values = values;
  ba.part_base = zero64;
  ba.part_class = zero32;
  ba.tables = d_t;
  ba.max_pairs = npmax;
  ba.n_bins = n_bins;
  ba.sq = sq;
  ba.bsum = bsum;
  ba.part0 = 0;
  ba.n_parts = 1;
  if (e == cudaSuccess) e = launch_binsums(ba, st);
  FitArgs fa;
  fa.S = 1;
  fa.n_bins = n_bins;
  fa.nblk = nblk;
  fa.kind = kind;
  fa.fit = 1;
  fa.nchunk = nchunk;
  fa.stats = stats;
  fa.part_b = zero32;
  fa.part_e = zero32;
  fa.part_class = zero32;
  fa.part_m = mm;
  fa.tables = d_t;
  fa.partial = partial;
  fa.svar = npstat + 1;
  fa.bsum = bsum;
  fa.models = models;
  fa.lohi = lohi;
  fa.status = status;
  fa.part0 = 0;
  fa.n_parts = 1;
  fa.reserve_smem = 0;
  if (e == cudaSuccess) e = launch_fit(fa, st);
  double mo[3] = {0, 0, 0};
  int32_t s = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(mo, models, sizeof(mo), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&s, status, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cleanup();
  if (e != cudaSuccess) return set_err(VK_E_CUDA, cudaGetErrorString(e));
  if (s != PS_OK) {
    if (s == PS_DEGENERATE) return set_err(VK_E_DEGENERATE_LAGS, "all sample pairs are co-located");
    return set_err(status_from_part(s), "fit failed with status " + std::to_string(s));
  }
  std::memcpy(model_out, mo, sizeof(mo));
  return VK_OK;
}

// ---- drop-in helpers for fill_missing(grid): validation + plane compaction
namespace {
__global__ void grid_scan_kernel(const float* __restrict__ data, const uint8_t* __restrict__ mask,
                                 int64_t PE, int32_t* counts) {
  const int64_t z = blockIdx.y;
  int c_miss = 0, c_nan = 0, c_bad = 0, c_inf = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < PE; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = data[z * PE + i];
    const bool m = mask[z * PE + i] != 0;
    const bool isn = v != v;
    c_miss += m;
    c_nan += isn;
    c_bad += (isn != m);
    c_inf += (!m && !isn && isinf(v));
  }
  for (int o = 16; o > 0; o >>= 1) {
    c_miss += __shfl_down_sync(0xffffffffu, c_miss, o);
    c_nan += __shfl_down_sync(0xffffffffu, c_nan, o);
    c_bad += __shfl_down_sync(0xffffffffu, c_bad, o);
    c_inf += __shfl_down_sync(0xffffffffu, c_inf, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&counts[z * 4 + 0], c_miss);
    atomicAdd(&counts[z * 4 + 1], c_nan);
    atomicAdd(&counts[z * 4 + 2], c_bad);
    atomicAdd(&counts[z * 4 + 3], c_inf);
  }
}

__global__ void gather_planes_kernel(const float* __restrict__ src, const int32_t* __restrict__ kz, int64_t PE,
                                     float* __restrict__ dst) {
  const int k = blockIdx.y;
  const int64_t z = kz[k];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < PE; i += (int64_t)gridDim.x * blockDim.x)
    dst[(int64_t)k * PE + i] = src[z * PE + i];
}
}  // namespace

int vk_grid_scan(const float* data, const uint8_t* mask, int64_t planes, int64_t plane_elems, int32_t* counts,
                 void* stream) {
  if (!data || !mask || !counts || planes < 1 || plane_elems < 1) return set_err(VK_E_INVALID_ARGUMENT, "scan args");
  cudaStream_t st = (cudaStream_t)stream;
  VK_CUDA(cudaMemsetAsync(counts, 0, (size_t)planes * 4 * sizeof(int32_t), st));
  dim3 grid((unsigned)std::min<int64_t>(64, (plane_elems + 255) / 256), (unsigned)planes);
  grid_scan_kernel<<<grid, 256, 0, st>>>(data, mask, plane_elems, counts);
  VK_CUDA(cudaGetLastError());
  return VK_OK;
}

int vk_gather_planes(const float* src, const int32_t* known_z, int32_t K, int64_t plane_elems, float* dst,
                     void* stream) {
  if (!src || !known_z || !dst || K < 1) return set_err(VK_E_INVALID_ARGUMENT, "gather args");
  cudaStream_t st = (cudaStream_t)stream;
  int32_t* dkz = nullptr;
  VK_CUDA(cudaMallocAsync((void**)&dkz, K * sizeof(int32_t), st));
  VK_CUDA(cudaMemcpyAsync(dkz, known_z, K * sizeof(int32_t), cudaMemcpyHostToDevice, st));
  dim3 grid((unsigned)std::min<int64_t>(256, (plane_elems + 255) / 256), (unsigned)K);
  gather_planes_kernel<<<grid, 256, 0, st>>>(src, dkz, plane_elems, dst);
  VK_CUDA(cudaGetLastError());
  VK_CUDA(cudaFreeAsync(dkz, st));
  return VK_OK;
}

}  // extern "C"
