/*
 * volkrig-b200 -- C ABI of the B200-native kriging interpolation path.
 *
 * Drop-in boundary for the reference's Python entry points (paths relative to
 * /root/reference/pkg/src/volkrig):
 *
 *   fill_missing(grid, model, drift="linear", return_variance=False)
 *       kriging.py:458-496 (plane-structured branch kriging.py:499-557)
 *       -> vk_grid_scan + vk_plan_create(fit_variogram = 0)
 *          + vk_plan_execute(models = the caller's model) + vk_plan_finish
 *   fit_variogram(samples, kind="exponential", n_bins=15,
 *                 max_pairs=100_000, seed=0)
 *       kriging.py:264-328
 *       -> vk_fit_variogram_samples
 *   reconstruct_block's kriging half over Z sub-parts (the
 *   absent block_pipeline): per-part fit_variogram then
 *   fill_missing, merged by dropping each part's trailing halo plane
 *       -> vk_plan_create(fit_variogram = 1, n_subparts = S)
 *          + vk_plan_execute(models = NULL) + vk_plan_finish
 *
 * Conventions: plain pointers and sizes, no torch types.  Volumes are float32
 * [z][y][x] C-order (model.py:5-9); device pointers are CUDA global memory of
 * the current device; every call that takes a stream is stream-ordered and
 * asynchronous; errors detected on the device surface at vk_plan_finish.
 * The library never frees caller memory; a plan owns its own workspace.
 * Plans are not thread-safe; use one plan per thread/stream.
 */
#ifndef VOLKRIG_B200_H
#define VOLKRIG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VK_ABI_VERSION 1

/* Status codes; the Python layer maps them to the reference's exception
 * classes (errors.py:54-67). */
typedef enum {
  VK_OK = 0,
  VK_E_INVALID_ARGUMENT = 1,    /* ValueError                        */
  VK_E_NO_KNOWN_NEIGHBORS = 2,  /* NoKnownNeighbors  kriging.py:477,513 */
  VK_E_SINGULAR_SYSTEM = 3,     /* SingularSystem    kriging.py:232,236 */
  VK_E_INSUFFICIENT_SAMPLES = 4,/* InsufficientSamples kriging.py:275   */
  VK_E_DEGENERATE_LAGS = 5,     /* DegenerateLags    kriging.py:291     */
  VK_E_UNSUPPORTED = 6,         /* layout outside the device path      */
  VK_E_CUDA = 7,                /* CUDA runtime failure                */
  VK_E_INVALID_GRID = 8,        /* validate(): mask/NaN out of sync (model.py:111-117) */
  VK_E_FIT_FAILED = 9           /* least_squares raised (scipy ValueError) */
} vk_status;

enum { VK_KIND_EXPONENTIAL = 0, VK_KIND_GAUSSIAN = 1, VK_KIND_SPHERICAL = 2 };
enum { VK_DRIFT_LINEAR = 0, VK_DRIFT_CONSTANT = 1 };
/* prediction arithmetic: fp64 / fp32 DFMA-FFMA stencils, or FIXED: 24-bit
 * fixed-point known values x 32-bit fixed-point weights on the int8 tensor
 * cores with exact s32 accumulation (error <= ~2e-7 of the data range;
 * plane-structured fast layout only, fp64 elsewhere) */
enum { VK_ACCUM_FP64 = 0, VK_ACCUM_FP32 = 1, VK_ACCUM_FIXED = 2 };

typedef struct vk_plan vk_plan;

typedef struct {
  int32_t height;          /* dy                                          */
  int32_t width;           /* dx                                          */
  int32_t depth;           /* dz of the output grid                       */
  int32_t n_known;         /* K known planes                              */
  const int32_t* known_z;  /* host [K], strictly increasing, in [0,depth) */
  int32_t n_subparts;      /* S >= 1 Z sub-parts (1: whole grid)          */
  int32_t kind;            /* VK_KIND_*                                   */
  int32_t drift;           /* VK_DRIFT_*                                  */
  int32_t accum;           /* VK_ACCUM_* prediction accumulation          */
  int32_t n_bins;          /* 15 (kriging.py:264)                         */
  int64_t max_pairs;       /* 100000                                      */
  uint64_t seed;           /* 0                                           */
  int32_t fit_variogram;   /* 1: per-part device fit; 0: models supplied  */
  int32_t flags;           /* VK_FLAG_*                                   */
  int32_t part_len;        /* known slices per part q (0: K / S); part s =
                              [s*q, (s+1)*q], the last part takes the rest  */
} vk_plan_desc;

#define VK_FLAG_FORCE_GENERIC 1   /* disable the streaming fast kernel (testing) */
#define VK_FLAG_REDRAW_PAIRS 2    /* redraw the pair tables on every execute
                                     (default: drawn once per plan, they depend
                                     only on geometry and seed)               */
#define VK_FLAG_OVERLAP 4         /* accepted for compatibility: the per-part
                                     chain schedule is now the default        */
#define VK_FLAG_SERIAL 8          /* one launch per stage on the caller's
                                     stream (per-stage timing).  Default with
                                     S > 1 on the streaming path: per-part
                                     fit -> solve -> predict chains on side
                                     streams, launched breadth-first (all
                                     fits, then solves, then predicts), so a
                                     part whose variogram fit converges early
                                     streams its planes while slower fits are
                                     still iterating.  Set
                                     CUDA_DEVICE_MAX_CONNECTIONS >= 32 before
                                     the CUDA context is created for one
                                     hardware queue per chain.                */

/* Replaces: the window/stencil setup of fill_missing (kriging.py:485-515)
 * and the partition of SPEC.md:392-400.  Host-side, O(K + H + W). */
int vk_plan_create(const vk_plan_desc* desc, vk_plan** out);

void vk_plan_destroy(vk_plan* plan);

/* Replaces: fill_missing / the per-part reconstruct_block kriging chain.
 *   known   device f32 [K][H][W]  (the known planes, in known_z order)
 *   models  host f64 [S][3] (nugget, sill, range_len) when fit_variogram==0,
 *           else NULL
 *   out     device f32 [depth][H][W]  (known planes copied bit-exactly)
 *   var     device f64 [depth][H][W] kriging variance or NULL
 *           (return_variance, kriging.py:482, 492-496)
 *   stream  cudaStream_t (NULL = legacy default stream)                   */
int vk_plan_execute(vk_plan* plan, const float* known, const double* models,
                    float* out, double* var, void* stream);

/* Copies a reconstructed volume to host memory, as the reference's
 * fill_missing returns it (kriging.py:481-496): the interpolated planes come
 * from the device volume `out_dev` (one strided device-to-host copy on a
 * regular layout), the known planes from the caller's host input
 * `known_host` ([n_known][H][W], the device holds bit-identical copies of
 * them), copied host to host on a plan-owned stream concurrently with the
 * download.  Stream-ordered on `stream`; pinned `out_host` / `known_host`
 * make it asynchronous.  Device-to-host bytes: the interpolated planes only. */
int vk_plan_download(vk_plan* plan, const float* out_dev, const float* known_host, float* out_host,
                     void* stream);

/* Synchronises the stream, maps device-side statuses to a vk_status.
 * failed_part: first failing sub-part or -1.  models_out: host f64 [S][3]
 * fitted (or supplied) models, may be NULL.  lohi_out: host f64 [S][2] clamp
 * range per part, may be NULL. */
int vk_plan_finish(vk_plan* plan, void* stream, int32_t* failed_part,
                   double* models_out, double* lohi_out);

/* Introspection for tests / benchmarks. */
typedef struct {
  int32_t fast_path;        /* 1 if the streaming kernel handles all gaps  */
  int32_t gap_planes;       /* G missing planes per gap on the fast path   */
  int32_t n_patterns;
  int32_t n_kinds;
  int32_t n_systems;
  int32_t n_missing_planes;
  int32_t n_pair_classes;
  int32_t kernels_per_execute;
  int64_t interpolated_voxels;
} vk_plan_info;
int vk_plan_get_info(const vk_plan* plan, vk_plan_info* info);

/* Stage timing with CUDA events recorded on the execute stream:
 * stats, pairs, bins, fit, solve, predict (ms; 0 for skipped stages).
 * On the serial schedule "solve" ends with the stencil-table kernels built
 * from the solved weights and "predict" is the streaming kernel alone.
 * set_timing(ring): keep events of the last `ring` executes (0 disables).
 * stage_ms(back): times of the execute `back` calls ago (0 = latest);
 * synchronises on that execute's last event. */
#define VK_N_STAGES 6
int vk_plan_set_timing(vk_plan* plan, int ring);
int vk_plan_stage_ms(vk_plan* plan, int back, float* ms);

/* Copies solved stencils to host: weights f64 [n_systems][128] padded
 * ([plane][oy+1][ox+1]), variance f64 [n_systems], and per system (part,
 * pattern, ky, kx) int32 [n_systems][4].  Call after vk_plan_finish. */
int vk_plan_get_systems(vk_plan* plan, double* weights, double* variance,
                        int32_t* ids);

/* Replaces: fit_variogram(samples, ...) (kriging.py:264-328) for explicit
 * samples.  coords device f64 [m][3] (x,y,z), values device f64 [m].
 * Synchronous; writes the model (nugget, sill, range_len) to model_out. */
int vk_fit_variogram_samples(const double* coords, const double* values,
                             int64_t m, int32_t kind, int32_t n_bins,
                             int64_t max_pairs, uint64_t seed,
                             double* model_out, void* stream);

/* The pair draw of kriging.py:278-286 on the device: ii/jj device int32
 * [max_pairs] (triu order when m(m-1)/2 <= max_pairs).  Returns the number of
 * pairs written in *n_out (before dropping ii == jj).  Synchronous. */
int vk_sample_pairs(int64_t m, int64_t max_pairs, uint64_t seed, int32_t* ii,
                    int32_t* jj, int64_t* n_out, void* stream);

/* Replaces: VolumeGrid.validate + _plane_structured (model.py:111-117,
 * kriging.py:434-441).  data device f32 [T][P], mask device u8 [T][P];
 * counts device int32 [T][4] = (#missing, #nan, #nan!=mask, #known
 * non-finite) per plane. */
int vk_grid_scan(const float* data, const uint8_t* mask, int64_t planes,
                 int64_t plane_elems, int32_t* counts, void* stream);

/* Gathers known planes: dst[k] = src[known_z[k]] (device f32, [*][P]),
 * known_z host int32 [K]. */
int vk_gather_planes(const float* src, const int32_t* known_z, int32_t K,
                     int64_t plane_elems, float* dst, void* stream);

/* Host -> device copy of a caller-owned (pageable) host buffer through a
 * ring of page-locked staging chunks filled by host threads while the DMA of
 * the previous chunk runs (replaces the driver's ~11 GB/s pageable copy for
 * the drop-in entry points, whose inputs are numpy arrays: fit_variogram
 * samples, kriging.py:264; fill_missing grids, kriging.py:458).  Enqueued on
 * `stream`; returns once `src` may be reused. */
int vk_copy_h2d(void* dst, const void* src, int64_t bytes, void* stream);

/* Generic per-voxel fill for masks that are not whole known / missing
 * planes: the reference's fallback _predict_generic (kriging.py:408-431,
 * window schedule kriging.py:37-40, _gather_window kriging.py:345-357,
 * weight cache kriging.py:364-381).  data f32 [depth][height][width] (NaN at
 * missing voxels), mask u8 same shape (1 = missing), model = (nugget, sill,
 * range_len), lo/hi = known-value clamp range (kriging.py:475-479).  Writes
 * out (known voxels copied bit-exactly) and, if var != NULL, the kriging
 * variance (0 at known voxels).  info[3] (host, may be NULL): first voxel
 * without neighbours (raster index, -1 if none), distinct window patterns
 * solved, missing voxels.  Synchronous on `stream`.  Status
 * VK_E_NO_KNOWN_NEIGHBORS, VK_E_SINGULAR_SYSTEM, or VK_E_UNSUPPORTED when a
 * window holds more than 1024 known voxels. */
int vk_fill_generic(const float* data, const uint8_t* mask, int32_t depth, int32_t height,
                    int32_t width, int32_t kind, int32_t drift, const double* model, double lo,
                    double hi, float* out, double* var, int64_t* info, void* stream);

/* Batched extended kriging systems for arbitrary neighbour sets -- the
 * reference's build_system + solve_ked (kriging.py:159-245) for each entry of
 * a weight cache (kriging.py:364-381): rel = device int16 [total][3]
 * target-relative (x, y, z) offsets of every system's neighbours, offsets =
 * host int64 [n_systems + 1] (system i owns rel rows offsets[i] ..
 * offsets[i+1]-1, 1..1024 rows), model = host (nugget, sill, range_len).
 * Drift columns are kept by the reference's rank test; LU with partial
 * pivoting, residual check 1e-8, one ridge retry.  Writes weights (device
 * f64 [total]) and variance (device f64 [n_systems]); status (host int32
 * [n_systems], may be NULL): 0 ok, 1 singular.  Synchronous on `stream`. */
int vk_solve_systems(const int16_t* rel, const int64_t* offsets, int32_t n_systems, int32_t kind,
                     int32_t drift, const double* model, double* weights, double* variance,
                     int32_t* status, void* stream);

/* Binary volume format (io.py:146-200, VOLKRIG\0 v1): CRC-32 of device
 * bytes continuing from `crc_in` exactly as zlib.crc32(data, crc_in) (so a
 * host header, a device payload and a device mask chain into the file's
 * single CRC), and the mask bit packing of np.packbits / np.unpackbits
 * (big-endian bits, zero-padded last byte).  vk_crc32 is synchronous on
 * `stream`; the packers are asynchronous. */
int vk_crc32(const void* data, int64_t n_bytes, uint32_t crc_in, uint32_t* crc_out, void* stream);
int vk_packbits(const uint8_t* mask, int64_t n, uint8_t* bits, void* stream);
int vk_unpackbits(const uint8_t* bits, int64_t n, uint8_t* mask, void* stream);

/* Slice stack decode and normalisation -- _decode_slice + normalize_stack
 * (io.py:108-125, model.py:189-202).  `raw` holds n device samples of one
 * type: VK_SAMPLE_U8 (PIL "L"/"P"/"1" after convert("L"), / 255),
 * VK_SAMPLE_U16 ("I;16", / 65535), VK_SAMPLE_I32 ("I", f32(v) / 65535) or
 * VK_SAMPLE_F32 (already decoded).  vk_decode_samples writes the decoded f32
 * values; vk_normalize_stack decodes, reduces the global min/max and writes
 * (v - lo) / f32(hi - lo) in f32 (all zeros when hi == lo), bit-identical to
 * numpy.  `minmax` is a device int[2] scratch (ordered-integer keys of lo and
 * hi on return); it may be NULL (the library then allocates stream-ordered
 * scratch).  `out` may alias `raw` for VK_SAMPLE_F32 only.  Asynchronous. */
enum { VK_SAMPLE_U8 = 0, VK_SAMPLE_U16 = 1, VK_SAMPLE_I32 = 2, VK_SAMPLE_F32 = 3 };
int vk_decode_samples(const void* raw, int32_t sample_type, int64_t n, float* out, void* stream);
int vk_normalize_stack(const void* raw, int32_t sample_type, int64_t n, float* out, int32_t* minmax,
                       void* stream);

/* Multi-GPU Z-sub-part sharding: an NCCL communicator per rank
 * (NCCL is loaded at run time; VK_E_UNSUPPORTED when it is absent), the
 * one-known-plane halo exchange -- rank r sends `first_plane` (n floats) to
 * r - 1 and receives rank r + 1's first plane into `halo` (ranks below the
 * last) -- and the gather of every rank's core planes on rank 0 (`out`
 * holds sum(counts) floats there; counts[r] floats from rank r, in rank
 * order).  Grouped point-to-point transfers on `stream`, asynchronous.
 * `id` is 128 bytes (vk_comm_unique_id on one rank, broadcast by the host). */
int vk_comm_unique_id(unsigned char* id);
int vk_comm_create(const unsigned char* id, int32_t world, int32_t rank, void** comm);
int vk_comm_destroy(void* comm);
int vk_halo_exchange(void* comm, const float* first_plane, float* halo, int64_t n, void* stream);
int vk_gather_core(void* comm, const float* core, const int64_t* counts, float* out, void* stream);

const char* vk_status_string(int status);
/* Message of the last failing call on this thread (for exceptions). */
const char* vk_last_error(void);
int vk_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VOLKRIG_B200_H */
