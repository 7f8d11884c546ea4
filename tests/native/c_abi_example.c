/* Plain-C caller of the C ABI (the INTEGRATION.md section 3 flow): a smooth
 * known stack is uploaded, one plan fits a variogram per Z sub-part and fills
 * the missing planes on the device, and the result is checked on the host
 * (known planes bit-exact, a linear field reproduced, values in range).
 * Exit code 0 on success; prints one summary line. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include "volkrig_b200.h"

#define CK(x)                                                             \
  do {                                                                    \
    int s_ = (x);                                                         \
    if (s_ != 0) {                                                        \
      fprintf(stderr, "%s -> %d (%s)\n", #x, s_, vk_last_error());        \
      return 1;                                                           \
    }                                                                     \
  } while (0)

int main(void) {
  const int H = 64, W = 64, K = 9, f = 4, S = 2;
  const int T = (K - 1) * f + 1;
  const size_t P = (size_t)H * W;
  int32_t kz[9];
  float* host = (float*)malloc(sizeof(float) * K * P);
  float* out_h = (float*)malloc(sizeof(float) * T * P);
  if (!host || !out_h) return 1;
  for (int k = 0; k < K; ++k) {
    kz[k] = k * f;
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x)   /* linear field: reproduced exactly by universal kriging */
        host[k * P + y * W + x] = 0.25f * x + 0.5f * y + 0.125f * (float)(k * f) + 3.0f;
  }
  if (vk_abi_version() < 1) return 1;
  float *known_d = NULL, *out_d = NULL;
  if (cudaMalloc((void**)&known_d, sizeof(float) * K * P) != cudaSuccess) return 1;
  if (cudaMalloc((void**)&out_d, sizeof(float) * T * P) != cudaSuccess) return 1;
  cudaMemcpy(known_d, host, sizeof(float) * K * P, cudaMemcpyHostToDevice);

  vk_plan_desc d = {0};
  d.height = H; d.width = W; d.depth = T; d.n_known = K; d.known_z = kz; d.n_subparts = S;
  d.kind = VK_KIND_EXPONENTIAL; d.drift = VK_DRIFT_LINEAR; d.accum = VK_ACCUM_FP64;
  d.n_bins = 15; d.max_pairs = 100000; d.seed = 0; d.fit_variogram = 1;
  vk_plan* plan = NULL;
  CK(vk_plan_create(&d, &plan));
  vk_plan_info info;
  CK(vk_plan_get_info(plan, &info));
  CK(vk_plan_execute(plan, known_d, NULL, out_d, NULL, NULL));
  int32_t failed = -1;
  double models[2 * 3], lohi[2 * 2];
  CK(vk_plan_finish(plan, NULL, &failed, models, lohi));
  cudaMemcpy(out_h, out_d, sizeof(float) * T * P, cudaMemcpyDeviceToHost);
  vk_plan_destroy(plan);

  double err = 0.0;
  int known_ok = 1;
  for (int z = 0; z < T; ++z)
    for (int y = 0; y < H; ++y)
      for (int x = 0; x < W; ++x) {
        const double exact = 0.25 * x + 0.5 * y + 0.125 * z + 3.0;
        const float v = out_h[z * P + y * W + x];
        if (z % f == 0 && v != host[(z / f) * P + y * W + x]) known_ok = 0;
        err = fmax(err, fabs((double)v - exact));
      }
  const double range = 0.25 * (W - 1) + 0.5 * (H - 1) + 0.125 * (T - 1);
  printf("c_abi_example fast_path=%d kernels=%d failed_part=%d known_exact=%d max_err/range=%.3e "
         "sill0=%.4g\n", info.fast_path, info.kernels_per_execute, failed, known_ok, err / range, models[1]);
  cudaFree(known_d);
  cudaFree(out_d);
  free(host);
  free(out_h);
  return (known_ok && err <= 1e-6 * range && failed == -1) ? 0 : 2;
}
