/* c_api_demo.c — the C ABI used directly from C (no Python, no torch):
 * one replica (M = 1) of a 2-fragment Streaming DiLoCo calendar, with the
 * fragment state in plain cudaMalloc'd buffers.
 *
 *   gcc -std=c99 -I include examples/c_api_demo.c -L paper_2501_18512_b200 -lsd \
 *       -Wl,-rpath,$PWD/paper_2501_18512_b200 -I /usr/local/cuda/include \
 *       -L /usr/local/cuda/lib64 -lcudart -o c_api_demo && ./c_api_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "sd.h"

#define CHECK(call)                                                                         \
  do {                                                                                      \
    sd_status st_ = (call);                                                                 \
    if (st_ != SD_OK) {                                                                     \
      fprintf(stderr, "%s failed (%d): %s\n", #call, (int)st_, sd_last_error(ctx));         \
      return 1;                                                                             \
    }                                                                                       \
  } while (0)

int main(void) {
  sd_ctx* ctx = NULL;
  sd_config cfg;
  const int64_t n = 1 << 20;  /* elements per fragment */
  int32_t P = 0, send[8], recv[8], ns = 0, nr = 0;
  float *theta[2], *anchor[2], *mom[2];
  void* gather[2];
  float* host = (float*)malloc(sizeof(float) * (size_t)n);
  int devices = 0;

  CHECK(sd_config_default(&cfg, 2, 1, 10)); /* L = 2 blocks, |p| = 1, H = 10, tau = 1 */
  cfg.T = 40;
  CHECK(sd_fragment_count(&cfg, &P));
  if (cudaGetDeviceCount(&devices) != cudaSuccess || devices == 0) {
    printf("c_api_demo: %d fragments, payload %zu bytes; no CUDA device, stopping after the host-only calls\n", P,
           sd_payload_bytes(&cfg, n));
    return 0;
  }
  CHECK(sd_init(&ctx, &cfg, 0, 1, NULL, 0));
  for (int p = 0; p < P; ++p) {
    for (int64_t i = 0; i < n; ++i) host[i] = 0.01f * sinf((float)(i + p * 7));
    cudaMalloc((void**)&theta[p], sizeof(float) * (size_t)n);
    cudaMalloc((void**)&anchor[p], sizeof(float) * (size_t)n);
    cudaMalloc((void**)&mom[p], sizeof(float) * (size_t)n);
    cudaMemcpy(theta[p], host, sizeof(float) * (size_t)n, cudaMemcpyHostToDevice);
    CHECK(sd_outer_state_init(ctx, theta[p], anchor[p], mom[p], n, NULL));
    CHECK(sd_gather_alloc(ctx, n, &gather[p]));
  }
  for (int64_t t = 1; t <= cfg.T; ++t) {
    /* (the inner step would update theta here) */
    CHECK(sd_fragment_schedule(&cfg, t, send, &ns, recv, &nr, 8));
    for (int k = 0; k < ns; ++k) {
      CHECK(sd_outer_grad_quantize(ctx, send[k], t, theta[send[k]], anchor[send[k]], n, gather[send[k]], NULL));
      CHECK(sd_fragment_sync(ctx, send[k], t, gather[send[k]], n, NULL));
    }
    for (int k = 0; k < nr; ++k)
      CHECK(sd_merge(ctx, recv[k], t, gather[recv[k]], theta[recv[k]], anchor[recv[k]], mom[recv[k]], n, NULL));
  }
  {
    int64_t first_bad = -1;
    CHECK(sd_check(ctx, &first_bad));
  }
  printf("c_api_demo: %d fragments x %lld elements through %lld steps, %llu libsd kernels, status OK\n", P,
         (long long)n, (long long)cfg.T, (unsigned long long)sd_kernel_launch_count());
  for (int p = 0; p < P; ++p) {
    cudaFree(theta[p]);
    cudaFree(anchor[p]);
    cudaFree(mom[p]);
  }
  CHECK(sd_finalize(ctx));
  free(host);
  return 0;
}
