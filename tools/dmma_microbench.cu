// Microbenchmark: FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput on
// the GPU box, next to DFMA in the same harness.  Decides whether the
// prediction contraction (voxels x taps) x (taps x stencils) should run on
// DMMA instead of DFMA.  Prints JSON lines.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_kernel(double* out, int iters, double a0, double b0) {
  double acc[CH][2];
  double a = a0 + threadIdx.x * 1e-12, b = b0 - threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < CH; ++i) { acc[i][0] = 0; acc[i][1] = i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
          : "+d"(acc[i][0]), "+d"(acc[i][1])
          : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

// DMMA and DFMA interleaved on independent chains: do they share a pipe?
__global__ void mixed_kernel(double* out, int iters, double a0, double b0) {
  double acc[4][2], x[8];
  double a = a0 + threadIdx.x * 1e-12, b = b0 - threadIdx.x * 1e-12;
#pragma unroll
  for (int i = 0; i < 4; ++i) { acc[i][0] = 0; acc[i][1] = i; }
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-9 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
          : "+d"(acc[i][0]), "+d"(acc[i][1])
          : "d"(a), "d"(b));
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.678) out[0] = s;
}

// int8 warp MMA (m16n8k32, s32 accumulate)
template <int CH>
__global__ void imma_kernel(int* out, int iters, int a0, int b0) {
  int acc[CH][4];
  const int a = a0 ^ threadIdx.x, b = b0 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < CH; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = i + j;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
          "{%0, %1, %2, %3};"
          : "+r"(acc[i][0]), "+r"(acc[i][1]), "+r"(acc[i][2]), "+r"(acc[i][3])
          : "r"(a), "r"(a + 1), "r"(a + 2), "r"(a + 3), "r"(b), "r"(b + 1));
    }
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
  if (s == 12345) out[0] = s;
}

static int clk_khz() {
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  return clk;
}

template <int CH>
void run_dmma(int blocks, int threads, int iters, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dmma_kernel<CH><<<blocks, threads>>>(d, 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  dmma_kernel<CH><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32;
  const double fma = 256.0 * CH * iters * warps;      // 8x8x4 per warp instruction
  printf("{\"test\":\"dmma\",\"chains\":%d,\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f,"
         "\"fma_per_clk_per_sm_at_max\":%.2f,\"err\":\"%s\"}\n",
         CH, blocks, threads, ms, 2 * fma / ms / 1e9, fma / (ms * 1e-3) / (148 * (clk_khz() * 1e3)),
         cudaGetErrorString(cudaGetLastError()));
}

template <int CH>
void run_dfma(int blocks, int threads, int iters, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<CH><<<blocks, threads>>>(d, 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  dfma_kernel<CH><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double fma = (double)CH * iters * blocks * threads;
  printf("{\"test\":\"dfma\",\"chains\":%d,\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f,"
         "\"fma_per_clk_per_sm_at_max\":%.2f}\n",
         CH, blocks, threads, ms, 2 * fma / ms / 1e9, fma / (ms * 1e-3) / (148 * (clk_khz() * 1e3)));
}

template <int CH>
void run_imma(int blocks, int threads, int iters, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  imma_kernel<CH><<<blocks, threads>>>((int*)d, 10, 3, 5);
  cudaEventRecord(e0);
  imma_kernel<CH><<<blocks, threads>>>((int*)d, iters, 3, 5);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32;
  const double mac = 4096.0 * CH * iters * warps;
  printf("{\"test\":\"imma_m16n8k32\",\"chains\":%d,\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"tops\":%.1f,"
         "\"mac_per_clk_per_sm_at_max\":%.1f,\"err\":\"%s\"}\n",
         CH, blocks, threads, ms, 2 * mac / ms / 1e9, mac / (ms * 1e-3) / (148 * (clk_khz() * 1e3)),
         cudaGetErrorString(cudaGetLastError()));
}

void run_mixed(int blocks, int threads, int iters, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mixed_kernel<<<blocks, threads>>>(d, 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  mixed_kernel<<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = (double)blocks * threads / 32;
  const double fma = (256.0 * 4 + 32.0 * 32) * iters * warps;   // 4 DMMA + 32 DFMA per warp-iter
  printf("{\"test\":\"dmma+dfma\",\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f,"
         "\"fma_per_clk_per_sm_at_max\":%.2f}\n",
         blocks, threads, ms, 2 * fma / ms / 1e9, fma / (ms * 1e-3) / (148 * (clk_khz() * 1e3)));
}

int main() {
  double* d;
  cudaMalloc(&d, 64);
  const int iters = 4000;
  run_dfma<8>(148 * 2, 256, iters * 8, d);
  run_dmma<1>(148 * 2, 256, iters, d);
  run_dmma<2>(148 * 2, 256, iters, d);
  run_dmma<4>(148 * 2, 256, iters, d);
  run_dmma<8>(148 * 2, 256, iters, d);
  run_dmma<4>(148 * 4, 256, iters, d);
  run_dmma<8>(148 * 4, 256, iters, d);
  run_dmma<4>(148 * 1, 128, iters, d);
  run_dmma<8>(148 * 1, 128, iters, d);
  run_mixed(148 * 2, 256, iters, d);
  run_imma<4>(148 * 2, 256, iters * 4, d);
  run_imma<8>(148 * 2, 256, iters * 4, d);
  run_imma<8>(148 * 4, 256, iters * 4, d);
  return 0;
}
