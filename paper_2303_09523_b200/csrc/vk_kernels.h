// Internal launcher interface between the plan (vk_api.cu) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>
#include <vector>
#include "vk_common.h"
#include "npsum.h"

namespace vk {

// Per-chunk plane statistics (count, mean, M2, min, max, non-finite).
struct ChunkStat {
  double n, mean, m2, mn, mx, bad;
  double sum;                        // raw sum: exact when the chunk is integer-valued (< 2^23)
};
constexpr int STATS_CHUNK = 32768;   // elements per stats block

struct PairTable {                   // one per pair class (device pointers)
  int32_t* ii;
  int32_t* jj;
  uint8_t* bin;                      // 255 = skipped (i == j or lag == 0)
  int64_t* counts;                   // [n_bins]
  double* scal;                      // [0] hmax, [1] lag_max, [2] n_drawn, [3] status
  // scratch of the parallel draw (sized by pair_scratch_elems)
  int32_t* cnt;                      // [n_thr]
  int64_t* off;                      // [n_thr + 1]
  unsigned long long* hbits;         // [1]
  // pairs sorted by bin, stable (launch_pair_order; nullptr: not kept)
  int32_t* order = nullptr;          // [npairs]
  int32_t* boff = nullptr;           // [n_bins + 1]
  int32_t* ocnt = nullptr;           // [order_chunks(npairs) * MAX_BINS] scratch of the sort
};
// number of draw threads (= scratch entries) for a pair class
int64_t pair_scratch_elems(int64_t m, int64_t max_pairs);

// Coordinates of sample i of a structured sub-part: plane i / P at local z
// zloc[i / P], pixel (i % P) -> (x, y).  Explicit: coords[i*3 + {0,1,2}].
struct SampleGeom {
  const double* coords;              // explicit coords or nullptr
  const int32_t* zloc;               // structured: local z per known plane
  int64_t P;
  int32_t W;
};

cudaError_t launch_plane_stats(const float* known, int k0, int k1, int64_t P, ChunkStat* out, int nchunk,
                               cudaStream_t st, int* inexact = nullptr);
// One pair class to draw (numpy-identical PCG64 + Lemire; triu when all
// pairs fit), with its table and the sample geometry for the lags.
struct PairJob {
  uint64_t st_hi, st_lo, inc_hi, inc_lo;
  uint32_t m, thr;
  int64_t n_raw, need, max_pairs, npairs, n_thr;
  int triu, n_bins;
  PairTable t;
  SampleGeom geom;
};
PairJob make_pair_job(uint64_t st_hi, uint64_t st_lo, uint64_t inc_hi, uint64_t inc_lo, int64_t m,
                      int64_t max_pairs, int n_bins, SampleGeom geom, PairTable t);
// all classes in one cooperative launch, or 5 launches (blockIdx.y = class);
// h_jobs mirrors d_jobs; *launches (optional) = kernels launched
cudaError_t launch_pair_tables(const PairJob* d_jobs, const PairJob* h_jobs, int n_jobs, cudaStream_t st,
                               int* launches = nullptr);
struct BinsArgs {
  const float* known;      // structured: known planes; sample i of part s = known[base_s + i]
  const double* values;    // explicit samples (fit_variogram API) or nullptr
  const int64_t* part_base;// [S] element offset of each part's first sample
  const int32_t* part_class;
  const PairTable* tables;  // device array [n_classes]
  int64_t max_pairs;
  int n_bins, nblk, S;
  double* partial;          // [S][nblk][n_bins]
  int part0 = 0, n_parts = 0;   // parts [part0, part0 + n_parts) of this launch (n_parts <= 0: all S)
};
cudaError_t launch_bins(const BinsArgs& a, cudaStream_t st);

// ---- numpy-exact statistics (vk_npstats.cu) ----
// numpy's pairwise-summation tree for an array of m float64 (leaves of <= 128
// elements, internal nodes grouped by height)
struct NpSumTree {                   // device view of one class's tree (npsum.h build_npsum_warp)
  int32_t nleaf, nnode, nlevel;      // the tree above the warp roots: leaf i = warp root i
  const int32_t* leaf_off;           // [n true leaves + 1] element offsets
  const int32_t* node_lr;
  const int32_t* level;
  const int32_t* wr_leaf;            // [nleaf + 1] first true leaf of each warp root
  const int16_t* wr_prog;            // [nleaf][31] children of the root's internal nodes
  const int8_t* wr_nint;             // [nleaf] internal nodes per warp root
};
// svar[s] = values.var() of part s exactly as numpy computes it
struct NpVarArgs {
  const float* known;                // structured samples (known planes) or nullptr
  const double* values;              // explicit samples or nullptr
  const int64_t* part_base;          // [S]
  const int64_t* part_m;             // [S]
  const int32_t* part_class;         // [S]
  const NpSumTree* trees;            // [n_classes]
  int part0 = 0, n_parts = 0;
  int max_leaf = 0;                  // max nleaf over the classes of the launch
  int64_t leaf_stride = 0, node_stride = 0;
  double* leaf;                      // [S][leaf_stride]
  double* node;                      // [S][node_stride]
  double* mean;                      // [S]
  double* svar;                      // [S]
  // integer-valued parts: the mean's pairwise sum is the exact sum, read from
  // the statistics pass's chunk sums (nullptr: always the pairwise pass)
  const ChunkStat* stats = nullptr;  // [K][nchunk]
  const int* inexact = nullptr;      // [K] per known plane
  const int32_t* part_b = nullptr;   // [S] first / last known plane of the part
  const int32_t* part_e = nullptr;
  int nchunk = 0;
};
cudaError_t launch_npvar(const NpVarArgs& a, cudaStream_t st);
// stable sort of each class's pairs by bin (tables with order != nullptr)
inline int64_t order_chunks(int64_t npairs) { return (npairs + 2047) / 2048; }
cudaError_t launch_pair_order(const PairJob* d_jobs, const PairJob* h_jobs, int n_jobs, cudaStream_t st);
// bsum[s][b] = np.bincount(which, weights=0.5*(v_i - v_j)^2)[b] of part s
struct BinSumArgs {
  const float* known;
  const double* values;
  const int64_t* part_base;
  const int32_t* part_class;
  const PairTable* tables;
  int part0 = 0, n_parts = 0, n_bins = 0;
  int64_t max_pairs = 0;
  double* sq;                        // [S][max_pairs] scratch
  double* bsum;                      // [S][n_bins]
};
cudaError_t launch_binsums(const BinSumArgs& a, cudaStream_t st);

struct FitArgs {
  int S, n_bins, nblk, kind, fit, nchunk;
  int part0, n_parts;       // parts [part0, part0 + n_parts) of this launch
  int reserve_smem;         // dynamic smem to request (keeps co-resident CTAs off the SM)
  const ChunkStat* stats;   // [K][nchunk] (structured) or [1][nchunk] (explicit)
  const int32_t* part_b;    // [S]
  const int32_t* part_e;    // [S]
  const int32_t* part_class;
  const int64_t* part_m;    // [S]
  const PairTable* tables;
  const double* partial;    // bins partials (used when bsum == nullptr)
  const double* svar = nullptr;   // [S] numpy-exact values.var() (else the Chan merge of the stats)
  const double* bsum = nullptr;   // [S][n_bins] numpy-exact bin sums (else the partials)
  double* models;           // [S][3] in/out
  double* lohi;             // [S][2]
  int32_t* status;          // [S]
};
cudaError_t launch_fit(const FitArgs& a, cudaStream_t st);

struct SolveArgs {
  int n_sys, kind, drift, NP, NK;
  int sys0;                  // systems [sys0, sys0 + n_sys) of this launch
  const int32_t* sys_part;
  const int32_t* sys_stencil;
  const int32_t* st_off;     // [n_stencils] offset into taps/pad
  const int32_t* st_n;       // [n_stencils]
  const int32_t* st_drift;   // [n_stencils]
  const int32_t* st_pattern; // [n_stencils]
  const int8_t* taps;        // [.. * 3] (ox, oy, plane)
  const int16_t* pad;
  const int32_t* pat_dz;     // [NP][NPMAX]
  const double* models;      // [S][3]
  double* weights;           // [S][NP][NK][WPAD]
  double* var;               // [S][NP][NK]
  int32_t* sys_status;       // [n_sys]
  int max_n;                 // max neighbours over stencils (smem sizing)
  int max_dz;                // max |plane offset| or offset difference over patterns
  // derived systems (z-mirror / x<->y transpose images of a solved system of
  // the same part): source system or -1, flags bit 0 mirror, bit 1 transpose,
  // bits 8.. planes of the pattern.  launch_solve skips them; launch_derive
  // fills their weights, variance and status from the source.
  const int32_t* der_src = nullptr;
  const int32_t* der_flags = nullptr;
};
cudaError_t launch_solve(const SolveArgs& a, cudaStream_t st);
cudaError_t launch_derive(const SolveArgs& a, cudaStream_t st);

struct PredictArgs {
  const float* known;        // [K][H][W]
  float* out;                // [T][H][W]
  double* var;               // [T][H][W] or nullptr
  int H, W, K, NP, NK, accum;
  int64_t P;
  const int32_t* known_z;    // [K]
  const double* weights;     // [S][NP][NK][WPAD]
  const double* svar;        // [S][NP][NK]
  const double* lohi;        // [S][2]
  const int32_t* kmap;       // [2][NKIND1] compact kind maps (x then y)
  int nkx;
  // generic path
  int n_miss;
  const int32_t* miss_z, *miss_part, *miss_pattern, *miss_planes;
  // fast path: gaps [gap0, gap1) of this launch
  int G, gap0, gap1;
  int chunk;                   // gaps per unit (0: automatic)
  const int32_t* gap_part;     // [K-1]
  const int32_t* gap_pattern;  // [(K-1) * G]
  int part0, part1;            // parts whose mirror-pair stencils this launch prepares
  int S;                       // parts in the plan
  void* fxb;                   // fixed path: [S][NK][32][8] u32 B fragments
  void* fxc;                   // fixed path: [S][NK][8] float4 epilogue constants
  void* fxq;                   // fixed path: float4 (L, 1/step, step, 0) + double2 (L, step),
                               // written by launch_quant_range from the statistics pass
  int max_chunk;               // gaps per unit so that a unit spans <= 4 parts (0: none)
  void* kpm;                   // [S][NK][16][NSTP] Acc mirror-pair stencils (fast path)
  const int* sd_inexact;       // [K] per-plane flags from the stats pass: 0 -> every value of the
                               // plane is an integer below 2^23, so A +- B is exact in fp32
  int num_sms;
  int tables_done = 0;         // fast path: the stencil tables of [part0, part1) were already built
                               // (launch_predict_fast_tables) -- the launch is the streaming kernel alone
  int* work = nullptr;         // fast path: {next unit, CTAs done} of this launch (zero between
                               // launches; concurrent launches need their own pair)
};
// doubles the K+- table needs (fast path)
// (the fp64 table [S][NK][16][8], then the exact-split interior stencils
// [S][16][8] of (hi, lo) float pairs, vk_predict.cu split_stencil_kernel)
VK_HD size_t split_table_offset(int S, int NK) { return (size_t)S * (size_t)NK * 16 * 8; }
VK_HD size_t kpm_elems(int S, int NK) { return split_table_offset(S, NK) + (size_t)S * 16 * 8; }
// Launch state of the streaming kernel prepared once per known-plane buffer:
// TMA descriptor, occupancy-derived grid size.
struct FastLaunch {
  alignas(64) unsigned char tmap[128];   // CUtensorMap
  const float* known = nullptr;
  int G = 0, accum = -1, occ = 0;
};
cudaError_t prepare_predict_fast(const PredictArgs& a, FastLaunch* fl);
cudaError_t launch_predict_fast_prepared(const FastLaunch& fl, const PredictArgs& a, cudaStream_t st);
// the stencil-table kernels of the streaming launch on their own (fp64 / fp32 accumulation)
cudaError_t launch_predict_fast_tables(const PredictArgs& a, cudaStream_t st);
cudaError_t launch_copy_known(const PredictArgs& a, cudaStream_t st);
cudaError_t launch_predict_generic(const PredictArgs& a, cudaStream_t st);
cudaError_t launch_predict_fast(const PredictArgs& a, cudaStream_t st);
int predict_fast_supported(int G, int accum);
// fp64 mirror-pair stencil table (a.kpm) for parts [a.part0, a.part1)
cudaError_t fast_stencil_table(int G, const PredictArgs& a, cudaStream_t st);
// fixed-point tensor-core path (vk_predict_fixed.cu)
cudaError_t occupancy_fixed(int G, int* occ);
cudaError_t launch_quant_range(const ChunkStat* stats, int n, void* fxq, cudaStream_t st);
cudaError_t launch_predict_fixed(const void* tmap, int occ, const PredictArgs& a, cudaStream_t st);
// generic per-voxel fill (vk_generic.cu); synchronous on `st`
struct GenericResult {
  int status = 0;          // 0 ok, 2 no neighbours, 3 singular, 6 unsupported, 7 CUDA
  std::string msg;
  int64_t failed = -1;     // first voxel (raster index) without neighbours
  int n_systems = 0;       // distinct window patterns solved
  int64_t n_missing = 0;
};
// batched extended-system solves for arbitrary neighbour sets (vk_generic.cu):
// rel_dev int16 [total][3] target-relative offsets, rel_off host [n + 1];
// writes weights [total], variances [n], PartStatus [n] (device); synchronous
cudaError_t solve_systems_device(const int16_t* rel_dev, const std::vector<int64_t>& rel_off, int kind, int drift,
                                 const double* model, double* w_dev, double* var_dev, int32_t* status_dev,
                                 cudaStream_t st);
GenericResult fill_generic(const float* data, const uint8_t* mask, int T, int H, int W, const double* model,
                           int kind, int drift, double lo, double hi, float* out, double* var, cudaStream_t st);
// binary volume format helpers (vk_volio.cu)
cudaError_t crc32_device(const void* data, int64_t n, uint32_t crc_in, uint32_t* crc_out, cudaStream_t st);
cudaError_t packbits_device(const uint8_t* mask, int64_t n, uint8_t* bits, cudaStream_t st);
cudaError_t unpackbits_device(const uint8_t* bits, int64_t n, uint8_t* mask, cudaStream_t st);
cudaError_t decode_samples_device(const void* raw, int sample_type, int64_t n, float* out, cudaStream_t st);
cudaError_t normalize_stack_device(const void* raw, int sample_type, int64_t n, float* out, int* keys,
                                   cudaStream_t st);
inline size_t fxb_words(int S, int NK) { return (size_t)S * (size_t)NK * 32 * 8; }
inline size_t fxc_floats(int S, int NK) { return (size_t)S * (size_t)NK * 8 * 4; }

}  // namespace vk
