// mb_read.cu — what DRAM mix can B200 stream fastest?  Ceiling for
// k_quantize's mix (read theta + A, write 1/16 of that) against a pure read
// and a 1:1 copy, all with k_quantize's access pattern (256-bit loads, one
// thread per 8 elements, one CTA per 2048 elements).  Not part of the product.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_read scripts/mb_read.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

struct f8 { float v[8]; };
__device__ __forceinline__ f8 ld8(const float* p) {
  f8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]),
                 "=f"(r.v[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st8(float* p, const f8& r) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]),
               "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7])
               : "memory");
}

// MODE 0: read a, b (8 B/elem); MODE 1: + write 0.5 B/elem; MODE 2: copy a -> c (4 + 4 B/elem)
template <int MODE>
__global__ void __launch_bounds__(256) k(const float* a, const float* b, float* c, uint32_t* w, int64_t n8) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  const f8 x = ld8(a + 8 * i);
  if (MODE == 2) {
    st8(c + 8 * i, x);
    return;
  }
  const f8 y = ld8(b + 8 * i);
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x.v[j] - y.v[j];
  if (MODE == 1) w[i] = __float_as_uint(s);
  else if (s == 1234.5f) w[0] = 1;  // keep the loads alive
}

int main() {
  const int64_t n = 151007616, n8 = n / 8;
  float *a, *b, *c;
  uint32_t* w;
  cudaMalloc(&a, 4 * n);
  cudaMalloc(&b, 4 * n);
  cudaMalloc(&c, 4 * n);
  cudaMalloc(&w, 4 * n8);
  cudaMemset(a, 0, 4 * n);
  cudaMemset(b, 0, 4 * n);
  const int grid = (int)((n8 + 255) / 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* name[3] = {"read 2 arrays (8 B/elem)", "read 8 + write 0.5 B/elem (quantize mix)", "copy 4 + 4 B/elem"};
  const double bytes[3] = {8.0 * n, 8.5 * n, 8.0 * n};
  for (int mode = 0; mode < 3; ++mode) {
    float best = 1e9f;
    for (int it = 0; it < 12; ++it) {
      cudaEventRecord(e0);
      if (mode == 0) k<0><<<grid, 256>>>(a, b, c, w, n8);
      if (mode == 1) k<1><<<grid, 256>>>(a, b, c, w, n8);
      if (mode == 2) k<2><<<grid, 256>>>(a, b, c, w, n8);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 2 && ms < best) best = ms;
    }
    printf("%-44s %.1f us  %.0f GB/s\n", name[mode], best * 1e3, bytes[mode] / (best * 1e-3) / 1e9);
  }
  cudaError_t err = cudaGetLastError();
  printf("%s\n", err == cudaSuccess ? "ok" : cudaGetErrorString(err));
  return 0;
}
