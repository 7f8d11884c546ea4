// Streaming-write bandwidth of a B200 for the prediction kernel's traffic
// shape (C4: 1 known plane read per 7 interpolated planes + 1 known plane
// written): what a kernel with no arithmetic achieves when it writes like
// predict_fast_kernel does.
//   write_only : 128-bit streaming stores (st.global.cs.v4) over the buffer
//   rw_1_8     : per (tile, gap) read one plane tile, write 8 plane tiles
//                (the known plane + 7 predictions), 128-bit loads / stores
//   memset     : cudaMemsetAsync of the buffer
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/write_bw_microbench tools/write_bw_microbench.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

__global__ void write_only(float4* __restrict__ out, size_t n4) {
  const float4 v = make_float4(1.f, 2.f, 3.f, 4.f);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(out + i), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

// planes of P floats; gap k reads known plane k and writes output planes
// 8k .. 8k+7 (known copy + 7 predictions = known * (j+1))
__global__ void rw_1_8(const float4* __restrict__ known, float4* __restrict__ out, int K, size_t P4) {
  const size_t items = (size_t)(K - 1) * P4;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < items; i += (size_t)gridDim.x * blockDim.x) {
    const size_t k = i / P4, p = i - k * P4;
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(known + k * P4 + p));
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float s = (float)(j + 1);
      asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(out + (k * 8 + j) * P4 + p), "f"(v.x * s),
                   "f"(v.y * s), "f"(v.z * s), "f"(v.w * s)
                   : "memory");
    }
  }
}

int main() {
  const int K = 256;
  const size_t P = 512 * 512, P4 = P / 4;
  const size_t out_floats = (size_t)((K - 1) * 8 + 1) * P;       // C4 output volume
  float *known = nullptr, *out = nullptr;
  cudaMalloc(&known, (size_t)K * P * 4);
  cudaMalloc(&out, out_floats * 4);
  cudaMemset(known, 0, (size_t)K * P * 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](const char* name, double bytes, auto fn) {
    for (int w = 0; w < 3; ++w) fn();
    float best = 1e9f;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(a);
      fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("{\"kernel\": \"%s\", \"ms\": %.4f, \"GB\": %.4f, \"GBps\": %.1f}\n", name, best, bytes / 1e9,
           bytes / (best * 1e-3) / 1e9);
  };
  const double wbytes = (double)(K - 1) * 8 * P * 4;
  for (int per_sm : {2, 4, 8, 16}) {
    char nm[64];
    snprintf(nm, sizeof nm, "write_only_%dctaPerSM", per_sm);
    timeit(nm, wbytes, [&] { write_only<<<sms * per_sm, 256>>>((float4*)out, (size_t)(K - 1) * 8 * P4); });
  }
  for (int per_sm : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, sizeof nm, "rw_1_8_%dctaPerSM", per_sm);
    timeit(nm, wbytes + (double)(K - 1) * P * 4,
           [&] { rw_1_8<<<sms * per_sm, 256>>>((const float4*)known, (float4*)out, K, P4); });
  }
  timeit("memset", wbytes, [&] { cudaMemsetAsync(out, 0, (size_t)wbytes); });
  return 0;
}
