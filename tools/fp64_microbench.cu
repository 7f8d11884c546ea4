// Microbenchmark: DFMA throughput / latency and F2F.F64.F32 throughput on the
// GPU box (MEASURED_PEAKS.json has no fp64 figure).  Prints JSON.
#include <cstdio>
#include <cuda_runtime.h>

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

__global__ void f2f_kernel(double* out, int iters, float a) {
  float v = threadIdx.x * 1e-3f;
  double s = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { s += (double)(v + (float)i); }
    v += a;
  }
  if (s == 12345.678) out[0] = s;
}

template <int CH>
void run(int blocks, int threads, int iters, double* d) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  dfma_kernel<CH><<<blocks, threads>>>(d, 10, 1.0000001, 1e-9);
  cudaEventRecord(e0);
  dfma_kernel<CH><<<blocks, threads>>>(d, iters, 1.0000001, 1e-9);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double flops = 2.0 * CH * (double)iters * blocks * threads;
  printf("{\"test\":\"dfma\",\"chains\":%d,\"blocks\":%d,\"threads\":%d,\"ms\":%.4f,\"tflops\":%.3f,\"dfma_per_clk_per_sm_at_max\":%.2f}\n",
         CH, blocks, threads, ms, flops / ms / 1e9, flops / 2 / (ms * 1e-3) / (148 * (clk * 1e3)));
}

int main() {
  double* d; cudaMalloc(&d, 64);
  int iters = 20000;
  for (int t : {128, 256, 512, 1024}) run<8>(148 * 2, t, iters, d);
  run<1>(148 * 8, 256, iters, d);
  run<2>(148 * 8, 256, iters, d);
  run<4>(148 * 4, 256, iters, d);
  run<4>(148 * 8, 256, iters, d);
  run<16>(148 * 2, 256, iters / 2, d);
  run<4>(148 * 2, 256, iters, d);   // 16 warps/SM, 4 chains
  run<8>(148 * 2, 256, iters, d);   // 16 warps/SM, 8 chains
  run<16>(148 * 2, 256, iters / 2, d);
  run<32>(148 * 2, 128, iters / 4, d);
  // F2F throughput
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  f2f_kernel<<<148 * 8, 256>>>(d, 10, 1e-3f);
  cudaEventRecord(e0);
  f2f_kernel<<<148 * 8, 256>>>(d, iters, 1e-3f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double n = 8.0 * iters * 148 * 8 * 256;
  printf("{\"test\":\"f2f+dadd\",\"ms\":%.4f,\"ops_per_clk_per_sm_at_max\":%.2f}\n", ms, n / (ms * 1e-3) / (148 * (clk * 1e3)));
  return 0;
}
