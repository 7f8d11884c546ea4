// Device side of the reference's binary volume format (io.py:146-200):
// CRC-32 of the payload (zlib's CRC: reflected polynomial 0xEDB88320, init
// and final xor 0xFFFFFFFF) and the missing-mask bit packing of
// np.packbits / np.unpackbits (big-endian bit order, zero-padded last byte).
//
// Slice decode + normalisation of load_stack (io.py:108-143, model.py:189-202)
// on the device: raw PNG samples (u8 "L", u16 "I;16", i32 "I") or already
// decoded f32 are converted exactly as numpy does it (f32(sample) / 255 or
// / 65535, IEEE division in f32), the global min/max are reduced as ordered
// integer keys, and out = (v - lo) / f32(double(hi) - double(lo)) in f32, or
// 0 for a constant stack.  Two passes over the raw samples, no host sync.
//
// CRC over n bytes at HBM speed: one thread per 16 KB chunk computes the raw
// CRC of its chunk (register starting at 0) with slicing-by-16 tables in
// shared memory; chunk CRCs are merged pairwise, bottom-up, by
//   raw(A || B) = raw(B) ^ shift(raw(A), |B|),   shift(v, n) = v * x^(8n) mod P
// (GF(2) arithmetic in the reflected representation, the combine algorithm
// zlib publishes as crc32_combine).  Continuing from a previous CRC c:
//   crc32(data, c) = ~(raw(data) ^ shift(~c, |data|)).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>
#include <vector>
#include "../../include/volkrig_b200.h"
#include "vk_kernels.h"

namespace vk {

namespace {

constexpr uint32_t CRC_POLY = 0xEDB88320u;
constexpr int64_t CRC_CHUNK = 16384;

__host__ __device__ uint32_t multmodp(uint32_t a, uint32_t b) {
  // a * b mod P, reflected: bit 31 is x^0
  uint32_t m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ CRC_POLY : b >> 1;
  }
  return p;
}

// x^(2^k) mod P for k = 0..63 (x^1 is 1 << 30 in the reflected form)
struct X2n {
  uint32_t v[64];
};
X2n make_x2n() {
  X2n t;
  uint32_t p = 1u << 30;
  t.v[0] = p;
  for (int k = 1; k < 64; ++k) t.v[k] = p = multmodp(p, p);
  return t;
}

__host__ __device__ uint32_t x8nmodp(int64_t n, const uint32_t* x2n) {
  // x^(8 n) mod P
  uint32_t p = 1u << 31;                             // x^0
  int k = 3;
  while (n) {
    if (n & 1) p = multmodp(x2n[k & 63], p);
    n >>= 1;
    ++k;
  }
  return p;
}

struct Tables {
  uint32_t t[16][256];
};
Tables make_tables() {
  Tables T;
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ CRC_POLY : c >> 1;
    T.t[0][i] = c;
  }
  for (int s = 1; s < 16; ++s)
    for (int i = 0; i < 256; ++i) T.t[s][i] = (T.t[s - 1][i] >> 8) ^ T.t[0][T.t[s - 1][i] & 0xff];
  return T;
}

__global__ void __launch_bounds__(256) crc_chunks_kernel(const uint8_t* __restrict__ data, int64_t n,
                                                         const Tables* __restrict__ gt, uint32_t* crc,
                                                         int64_t* len, int64_t n_chunks) {
  __shared__ uint32_t t[16][256];
  for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) t[i >> 8][i & 255] = gt->t[i >> 8][i & 255];
  __syncthreads();
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_chunks) return;
  const int64_t b = c * CRC_CHUNK, e = min(n, b + CRC_CHUNK);
  const uint8_t* p = data + b;
  int64_t m = e - b;
  uint32_t r = 0;
  // bytes up to 16-byte alignment, then slicing-by-16
  while (m > 0 && (reinterpret_cast<uintptr_t>(p) & 15)) {
    r = t[0][(r ^ *p++) & 0xff] ^ (r >> 8);
    --m;
  }
  for (; m >= 16; m -= 16, p += 16) {
    const uint4 q = *reinterpret_cast<const uint4*>(p);
    const uint32_t a = q.x ^ r;
    r = t[15][a & 0xff] ^ t[14][(a >> 8) & 0xff] ^ t[13][(a >> 16) & 0xff] ^ t[12][a >> 24] ^
        t[11][q.y & 0xff] ^ t[10][(q.y >> 8) & 0xff] ^ t[9][(q.y >> 16) & 0xff] ^ t[8][q.y >> 24] ^
        t[7][q.z & 0xff] ^ t[6][(q.z >> 8) & 0xff] ^ t[5][(q.z >> 16) & 0xff] ^ t[4][q.z >> 24] ^
        t[3][q.w & 0xff] ^ t[2][(q.w >> 8) & 0xff] ^ t[1][(q.w >> 16) & 0xff] ^ t[0][q.w >> 24];
  }
  for (; m > 0; --m) r = t[0][(r ^ *p++) & 0xff] ^ (r >> 8);
  crc[c] = r;
  len[c] = e - b;
}

// pairwise merge, one level: segment i of the next level = (2i, 2i+1)
__global__ void crc_merge_kernel(const uint32_t* crc_in, const int64_t* len_in, int64_t n_in, uint32_t* crc_out,
                                 int64_t* len_out, X2n x2n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n_out = (n_in + 1) / 2;
  if (i >= n_out) return;
  const int64_t a = 2 * i, b = a + 1;
  if (b >= n_in) {
    crc_out[i] = crc_in[a];
    len_out[i] = len_in[a];
    return;
  }
  crc_out[i] = crc_in[b] ^ multmodp(x8nmodp(len_in[b], x2n.v), crc_in[a]);
  len_out[i] = len_in[a] + len_in[b];
}

__global__ void packbits_kernel(const uint8_t* __restrict__ mask, int64_t n, uint8_t* bits) {
  const int64_t nb = (n + 7) / 8;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t v = 0;
    const int64_t b = 8 * j;
    for (int k = 0; k < 8; ++k) v |= (uint32_t)(b + k < n && mask[b + k] != 0) << (7 - k);
    bits[j] = (uint8_t)v;
  }
}

__global__ void unpackbits_kernel(const uint8_t* __restrict__ bits, int64_t n, uint8_t* mask) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    mask[i] = (bits[i >> 3] >> (7 - (i & 7))) & 1;
}

// monotone float <-> signed int key (total order of non-NaN floats)
__device__ __forceinline__ int f2key(float f) {
  const int i = __float_as_int(f);
  return i >= 0 ? i : i ^ 0x7fffffff;
}
__device__ __forceinline__ float key2f(int k) { return __int_as_float(k >= 0 ? k : k ^ 0x7fffffff); }

// Sample traits: raw type, samples per 16-byte vector, decode, and an integer
// order key.  Decoding is monotone in the raw value (int -> f32 and a
// correctly rounded division by a positive constant both are), so the min/max
// pass reduces raw integers and decodes only the two extremes.
template <int T> struct Samp;
template <> struct Samp<VK_SAMPLE_U8> {
  using raw_t = uint8_t;
  static __device__ __forceinline__ float decode(raw_t v) { return __fdiv_rn((float)v, 255.0f); }
  static __device__ __forceinline__ int key(raw_t v) { return v; }
  static __device__ __forceinline__ float value(int k) { return __fdiv_rn((float)k, 255.0f); }
};
template <> struct Samp<VK_SAMPLE_U16> {
  using raw_t = uint16_t;
  static __device__ __forceinline__ float decode(raw_t v) { return __fdiv_rn((float)v, 65535.0f); }
  static __device__ __forceinline__ int key(raw_t v) { return v; }
  static __device__ __forceinline__ float value(int k) { return __fdiv_rn((float)k, 65535.0f); }
};
template <> struct Samp<VK_SAMPLE_I32> {
  using raw_t = int32_t;
  static __device__ __forceinline__ float decode(raw_t v) { return __fdiv_rn(__int2float_rn(v), 65535.0f); }
  static __device__ __forceinline__ int key(raw_t v) { return v; }
  static __device__ __forceinline__ float value(int k) { return __fdiv_rn(__int2float_rn(k), 65535.0f); }
};
template <> struct Samp<VK_SAMPLE_F32> {
  using raw_t = float;
  static __device__ __forceinline__ float decode(raw_t v) { return v; }
  static __device__ __forceinline__ int key(raw_t v) { return f2key(v); }
  static __device__ __forceinline__ float value(int k) { return key2f(k); }
};

constexpr int EW_THREADS = 256;
constexpr int EW_UNROLL = 4;    // 16-byte vectors in flight per thread

template <int T>
union Vec16 {
  uint4 q;
  typename Samp<T>::raw_t s[16 / sizeof(typename Samp<T>::raw_t)];
};

__global__ void init_keys_kernel(int* keys) {
  if (threadIdx.x == 0) {
    keys[0] = 0x7fffffff;
    keys[1] = (int)0x80000000;
  }
}

// Pass 1: min/max order keys.  nvec 16-byte vectors (0 when the buffer is
// not 16-byte aligned), then the scalar tail [nvec * V, n).
template <int T>
__global__ void __launch_bounds__(EW_THREADS) minmax_kernel(const void* __restrict__ raw, int64_t n, int64_t nvec,
                                                            int* __restrict__ keys) {
  using S = Samp<T>;
  using raw_t = typename S::raw_t;
  constexpr int V = 16 / sizeof(raw_t);
  int lo = 0x7fffffff, hi = (int)0x80000000;
  const uint4* vec = reinterpret_cast<const uint4*>(raw);
  const int64_t step = (int64_t)gridDim.x * EW_THREADS * EW_UNROLL;
  for (int64_t base = (int64_t)blockIdx.x * EW_THREADS * EW_UNROLL + threadIdx.x; base < nvec; base += step) {
    Vec16<T> v[EW_UNROLL];
#pragma unroll
    for (int u = 0; u < EW_UNROLL; ++u) {
      const int64_t i = base + (int64_t)u * EW_THREADS;
      v[u].q = __ldcs(vec + (i < nvec ? i : base));   // out-of-range lanes re-read `base`: harmless for min/max
    }
#pragma unroll
    for (int u = 0; u < EW_UNROLL; ++u)
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const raw_t x = v[u].s[j];
        if (T == VK_SAMPLE_F32 && !(x == x)) continue;
        lo = min(lo, S::key(x));
        hi = max(hi, S::key(x));
      }
  }
  const raw_t* r = reinterpret_cast<const raw_t*>(raw);
  for (int64_t i = nvec * V + (int64_t)blockIdx.x * EW_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * EW_THREADS) {
    const raw_t x = r[i];
    if (T == VK_SAMPLE_F32 && !(x == x)) continue;
    lo = min(lo, S::key(x));
    hi = max(hi, S::key(x));
  }
  for (int o = 16; o; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  __shared__ int s[2][EW_THREADS / 32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s[0][w] = lo;
    s[1][w] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < EW_THREADS / 32; ++k) {
      lo = min(lo, s[0][k]);
      hi = max(hi, s[1][k]);
    }
    if (lo <= hi) {                           // decoded keys of this block's extremes
      atomicMin(keys, f2key(S::value(lo)));
      atomicMax(keys + 1, f2key(S::value(hi)));
    }
  }
}

// Pass 2 (RESCALE) or plain decode: out = decode(raw) or
// (decode(raw) - lo) / f32(double(hi) - double(lo)), 0 for a flat stack.
// Each thread loads EW_UNROLL vectors before storing any, so out may alias
// raw (f32 in place: every element is read and written by one thread).
template <int T, bool RESCALE>
__global__ void __launch_bounds__(EW_THREADS) map_kernel(const void* raw, int64_t n, int64_t nvec,
                                                         const int* __restrict__ keys, float* out) {
  using S = Samp<T>;
  using raw_t = typename S::raw_t;
  constexpr int V = 16 / sizeof(raw_t);
  float lo = 0.0f, range = 1.0f;
  bool flat = false;
  if (RESCALE) {
    lo = key2f(keys[0]);
    const float hi = key2f(keys[1]);
    flat = !(hi > lo);
    range = (float)((double)hi - (double)lo);   // a Python float, cast to f32 by numpy
  }
  auto f = [&](raw_t x) {
    const float d = S::decode(x);
    return RESCALE ? (flat ? 0.0f : __fdiv_rn(__fsub_rn(d, lo), range)) : d;
  };
  const uint4* vec = reinterpret_cast<const uint4*>(raw);
  float4* o4 = reinterpret_cast<float4*>(out);
  const int64_t step = (int64_t)gridDim.x * EW_THREADS * EW_UNROLL;
  for (int64_t base = (int64_t)blockIdx.x * EW_THREADS * EW_UNROLL + threadIdx.x; base < nvec; base += step) {
    Vec16<T> v[EW_UNROLL];
#pragma unroll
    for (int u = 0; u < EW_UNROLL; ++u) {
      const int64_t i = base + (int64_t)u * EW_THREADS;
      if (i < nvec) v[u].q = __ldcs(vec + i);
    }
#pragma unroll
    for (int u = 0; u < EW_UNROLL; ++u) {
      const int64_t i = base + (int64_t)u * EW_THREADS;
      if (i >= nvec) break;
#pragma unroll
      for (int j = 0; j < V; j += 4)
        __stcs(o4 + i * (V / 4) + j / 4,
               make_float4(f(v[u].s[j]), f(v[u].s[j + 1]), f(v[u].s[j + 2]), f(v[u].s[j + 3])));
    }
  }
  const raw_t* r = reinterpret_cast<const raw_t*>(raw);
  for (int64_t i = nvec * V + (int64_t)blockIdx.x * EW_THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * EW_THREADS)
    out[i] = f(r[i]);
}

int sm_count() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

// grid: enough CTAs for every vector once, capped at 8 resident CTAs per SM
int map_grid(int64_t nvec, int64_t n) {
  const int64_t per = (int64_t)EW_THREADS * EW_UNROLL;
  const int64_t need = nvec > 0 ? (nvec + per - 1) / per : (n + EW_THREADS - 1) / EW_THREADS;
  return (int)std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)sm_count() * 8));
}

template <int T>
int64_t n_vectors(const void* raw, const float* out, int64_t n) {
  const bool aligned = ((reinterpret_cast<uintptr_t>(raw) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  return aligned ? n / (16 / (int64_t)sizeof(typename Samp<T>::raw_t)) : 0;
}

template <int T>
void launch_decode(const void* raw, int64_t n, float* out, cudaStream_t st) {
  const int64_t nv = n_vectors<T>(raw, out, n);
  map_kernel<T, false><<<map_grid(nv, n), EW_THREADS, 0, st>>>(raw, n, nv, nullptr, out);
}

template <int T>
void launch_normalize(const void* raw, int64_t n, float* out, int* keys, cudaStream_t st) {
  const int64_t nv = n_vectors<T>(raw, out, n);
  const int g = map_grid(nv, n);
  minmax_kernel<T><<<g, EW_THREADS, 0, st>>>(raw, n, nv, keys);
  map_kernel<T, true><<<g, EW_THREADS, 0, st>>>(raw, n, nv, keys, out);
}

}  // namespace

cudaError_t decode_samples_device(const void* raw, int sample_type, int64_t n, float* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  switch (sample_type) {
    case VK_SAMPLE_U8: launch_decode<VK_SAMPLE_U8>(raw, n, out, st); break;
    case VK_SAMPLE_U16: launch_decode<VK_SAMPLE_U16>(raw, n, out, st); break;
    case VK_SAMPLE_I32: launch_decode<VK_SAMPLE_I32>(raw, n, out, st); break;
    case VK_SAMPLE_F32: launch_decode<VK_SAMPLE_F32>(raw, n, out, st); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t normalize_stack_device(const void* raw, int sample_type, int64_t n, float* out, int* keys,
                                   cudaStream_t st) {
  init_keys_kernel<<<1, 32, 0, st>>>(keys);
  if (n <= 0) return cudaGetLastError();
  switch (sample_type) {
    case VK_SAMPLE_U8: launch_normalize<VK_SAMPLE_U8>(raw, n, out, keys, st); break;
    case VK_SAMPLE_U16: launch_normalize<VK_SAMPLE_U16>(raw, n, out, keys, st); break;
    case VK_SAMPLE_I32: launch_normalize<VK_SAMPLE_I32>(raw, n, out, keys, st); break;
    case VK_SAMPLE_F32: launch_normalize<VK_SAMPLE_F32>(raw, n, out, keys, st); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t crc32_device(const void* data, int64_t n, uint32_t crc_in, uint32_t* crc_out, cudaStream_t st) {
  static const Tables host_tables = make_tables();
  static const X2n x2n = make_x2n();
  if (n <= 0) {
    *crc_out = crc_in;
    return cudaSuccess;
  }
  const int64_t n_chunks = (n + CRC_CHUNK - 1) / CRC_CHUNK;
  Tables* dt = nullptr;
  uint32_t* c[2] = {nullptr, nullptr};
  int64_t* l[2] = {nullptr, nullptr};
  cudaError_t e = cudaMallocAsync((void**)&dt, sizeof(Tables), st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&c[0], n_chunks * 4, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&c[1], n_chunks * 4, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&l[0], n_chunks * 8, st);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&l[1], n_chunks * 8, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(dt, &host_tables, sizeof(Tables), cudaMemcpyHostToDevice, st);
  uint32_t raw = 0;
  if (e == cudaSuccess) {
    crc_chunks_kernel<<<(unsigned)((n_chunks + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const uint8_t*>(data), n, dt, c[0], l[0], n_chunks);
    e = cudaGetLastError();
  }
  int cur = 0;
  for (int64_t m = n_chunks; e == cudaSuccess && m > 1; m = (m + 1) / 2) {
    const int64_t mo = (m + 1) / 2;
    crc_merge_kernel<<<(unsigned)((mo + 255) / 256), 256, 0, st>>>(c[cur], l[cur], m, c[cur ^ 1], l[cur ^ 1], x2n);
    e = cudaGetLastError();
    cur ^= 1;
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(&raw, c[cur], 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  for (int k = 0; k < 2; ++k) {
    if (c[k]) cudaFreeAsync(c[k], st);
    if (l[k]) cudaFreeAsync(l[k], st);
  }
  if (dt) cudaFreeAsync(dt, st);
  if (e != cudaSuccess) return e;
  *crc_out = ~(raw ^ multmodp(x8nmodp(n, x2n.v), ~crc_in));
  return cudaSuccess;
}

cudaError_t packbits_device(const uint8_t* mask, int64_t n, uint8_t* bits, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  packbits_kernel<<<1024, 256, 0, st>>>(mask, n, bits);
  return cudaGetLastError();
}

cudaError_t unpackbits_device(const uint8_t* bits, int64_t n, uint8_t* mask, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  unpackbits_kernel<<<1024, 256, 0, st>>>(bits, n, mask);
  return cudaGetLastError();
}

}  // namespace vk
