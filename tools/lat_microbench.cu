// Dependent-chain latency of the FP64 operations the serial fit is made of
// (one thread, clock64 around 256 chained operations), sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lat tools/lat_microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 256;

__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

template <int OP>
__global__ void chain(double a, double b, double* out, long long* cyc) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < N; ++i) {
    if (OP == 0) x = __fma_rn(x, b, a);             // DFMA
    if (OP == 1) x = __dadd_rn(x, b);               // DADD
    if (OP == 2) x = __ddiv_rn(a, x);               // div.rn.f64
    if (OP == 3) x = __dsqrt_rn(x + b);             // sqrt.rn.f64 (+ DADD)
    if (OP == 4) x = rcp_approx(x);                 // MUFU.RCP64H path
    if (OP == 5) x = __drcp_rn(x);                  // rcp.rn.f64
    if (OP == 6) x = (double)(float)x;              // F2F pair
    if (OP == 7) x = __dmul_rn(x, b);               // DMUL
  }
  long long t1 = clock64();
  out[0] = x;
  cyc[0] = t1 - t0;
}

int main() {
  double* d_out; long long* d_cyc;
  cudaMalloc(&d_out, 8); cudaMalloc(&d_cyc, 8);
  const char* names[] = {"dfma", "dadd", "ddiv_rn", "dsqrt_rn+dadd", "rcp.approx.f64", "drcp_rn", "f2f f64->f32->f64", "dmul"};
  for (int op = 0; op < 8; ++op) {
    long long c = 0;
    for (int rep = 0; rep < 3; ++rep) {
      switch (op) {
        case 0: chain<0><<<1, 1>>>(1.0000001, 0.9999999, d_out, d_cyc); break;
        case 1: chain<1><<<1, 1>>>(1.0, 1e-300, d_out, d_cyc); break;
        case 2: chain<2><<<1, 1>>>(1.5, 1.0, d_out, d_cyc); break;
        case 3: chain<3><<<1, 1>>>(2.0, 1.0, d_out, d_cyc); break;
        case 4: chain<4><<<1, 1>>>(1.5, 1.0, d_out, d_cyc); break;
        case 5: chain<5><<<1, 1>>>(1.5, 1.0, d_out, d_cyc); break;
        case 6: chain<6><<<1, 1>>>(1.5, 1.0, d_out, d_cyc); break;
        case 7: chain<7><<<1, 1>>>(1.5, 1.0, d_out, d_cyc); break;
      }
      cudaMemcpy(&c, d_cyc, 8, cudaMemcpyDeviceToHost);
    }
    printf("{\"op\": \"%s\", \"cycles_per_op\": %.1f}\n", names[op], (double)c / N);
  }
  return 0;
}
