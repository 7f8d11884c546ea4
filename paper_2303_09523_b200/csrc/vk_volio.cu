// Device side of the reference's binary volume format (io.py:146-200):
// CRC-32 of the payload (zlib's CRC: reflected polynomial 0xEDB88320, init
// and final xor 0xFFFFFFFF) and the missing-mask bit packing of
// np.packbits / np.unpackbits (big-endian bit order, zero-padded last byte).
//
// CRC over n bytes at HBM speed: one thread per 16 KB chunk computes the raw
// CRC of its chunk (register starting at 0) with slicing-by-16 tables in
// shared memory; chunk CRCs are merged pairwise, bottom-up, by
//   raw(A || B) = raw(B) ^ shift(raw(A), |B|),   shift(v, n) = v * x^(8n) mod P
// (GF(2) arithmetic in the reflected representation, the combine algorithm
// zlib publishes as crc32_combine).  Continuing from a previous CRC c:
//   crc32(data, c) = ~(raw(data) ^ shift(~c, |data|)).
#include <cuda_runtime.h>
#include <cstdint>
#include <vector>
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

}  // namespace

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
