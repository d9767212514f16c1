// mb_apply.cu — microbenchmark of memory-access variants for k_apply's
// streaming pattern (read A, v, theta + M code words, write A, v, theta).
// Not part of the product; used to pick the access pattern of sd_kernels.cu.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_apply scripts/mb_apply.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct f8 { float v[8]; };

template <int HINT>
__device__ __forceinline__ f8 ld8(const float* p) {
  f8 r;
  if (HINT == 0)
    asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p));
  else if (HINT == 1)
    asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p));
  else
    asm volatile("ld.global.L1::evict_first.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]), "=f"(r.v[6]), "=f"(r.v[7]) : "l"(p));
  return r;
}
template <int HINT>
__device__ __forceinline__ void st8(float* p, const f8& r) {
  if (HINT == 0)
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7]) : "memory");
  else if (HINT == 1)
    asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7]) : "memory");
  else
    asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]), "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7]) : "memory");
}

// U groups of 8 per thread per iteration; LH/SH load/store hints
template <int U, int LH, int SH, int M>
__global__ void __launch_bounds__(256) k8(float* A, float* v, float* th, const uint32_t* codes, size_t cstride, int64_t n) {
  const int64_t n8 = n >> 3;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n8; i0 += U * nthr) {
    f8 a[U], w[U], t[U];
    uint32_t c[U][M];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * nthr;
      if (i < n8) {
        a[u] = ld8<LH>(A + 8 * i); w[u] = ld8<LH>(v + 8 * i); t[u] = ld8<LH>(th + 8 * i);
#pragma unroll
        for (int m = 0; m < M; ++m) c[u][m] = __ldg(codes + m * cstride + i);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * nthr;
      if (i < n8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float S = 0.f;
#pragma unroll
          for (int m = 0; m < M; ++m) S = __fadd_rn(S, __uint_as_float(((c[u][m] >> (4 * j)) & 7u) << 23));
          w[u].v[j] = __fadd_rn(__fmul_rn(0.9f, w[u].v[j]), S);
          a[u].v[j] = __fsub_rn(a[u].v[j], __fmul_rn(0.4f, __fadd_rn(S, __fmul_rn(0.9f, w[u].v[j]))));
          t[u].v[j] = __fadd_rn(__fmul_rn(0.5f, t[u].v[j]), __fmul_rn(0.5f, a[u].v[j]));
        }
        st8<SH>(A + 8 * i, a[u]); st8<SH>(v + 8 * i, w[u]); st8<SH>(th + 8 * i, t[u]);
      }
    }
  }
}

// float4 variant (v1 layout): thread handles float4 i and i + nthr
template <int M>
__global__ void __launch_bounds__(256) k4(float4* A, float4* v, float4* th, const uint16_t* codes, size_t cstride, int64_t n) {
  const int64_t n4 = n >> 2;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n4; i0 += 2 * nthr) {
    float4 a[2], w[2], t[2]; uint32_t c[2][M];
#pragma unroll
    for (int u = 0; u < 2; ++u) { const int64_t i = i0 + u * nthr; if (i < n4) { a[u] = A[i]; w[u] = v[i]; t[u] = __ldcs(th + i);
#pragma unroll
      for (int m = 0; m < M; ++m) c[u][m] = __ldg(codes + 2 * m * cstride + i); } }
#pragma unroll
    for (int u = 0; u < 2; ++u) { const int64_t i = i0 + u * nthr; if (i < n4) {
      float* pa = &a[u].x; float* pw = &w[u].x; float* pt = &t[u].x;
#pragma unroll
      for (int j = 0; j < 4; ++j) { float S = 0.f;
#pragma unroll
        for (int m = 0; m < M; ++m) S = __fadd_rn(S, __uint_as_float(((c[u][m] >> (4 * j)) & 7u) << 23));
        pw[j] = __fadd_rn(__fmul_rn(0.9f, pw[j]), S);
        pa[j] = __fsub_rn(pa[j], __fmul_rn(0.4f, __fadd_rn(S, __fmul_rn(0.9f, pw[j]))));
        pt[j] = __fadd_rn(__fmul_rn(0.5f, pt[j]), __fmul_rn(0.5f, pa[j])); }
      A[i] = a[u]; v[i] = w[u]; __stcs(th + i, t[u]); } }
  }
}

__global__ void kcopy(const float4* a, float4* b, int64_t n4) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <typename K, typename... Args>
float timeit(K k, int blocks_per_sm, Args... args) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, 0);
  int bps = blocks_per_sm > 0 ? blocks_per_sm : occ;
  int grid = 148 * bps;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int i = 0; i < 3; ++i) k<<<grid, 256>>>(args...);
  cudaEventRecord(e0);
  const int R = 20;
  for (int i = 0; i < R; ++i) k<<<grid, 256>>>(args...);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / R;
}

int main() {
  const int64_t n = 151007616;
  float *A, *v, *th; uint32_t* codes;
  cudaMalloc(&A, n * 4); cudaMalloc(&v, n * 4); cudaMalloc(&th, n * 4);
  const size_t cstride = n / 8 + 64;
  cudaMalloc(&codes, 8 * cstride * 4);
  cudaMemset(A, 0, n * 4); cudaMemset(v, 0, n * 4); cudaMemset(th, 0, n * 4); cudaMemset(codes, 0x11, 8 * cstride * 4);
  auto rep = [&](const char* name, float ms, int M) {
    double bytes = 24.0 * n + M * 0.5 * n;
    printf("%-40s M=%d %8.3f ms %8.1f GB/s\n", name, M, ms, bytes / ms / 1e6);
  };
  float* cp; cudaMalloc(&cp, n * 4 * 2);
  float ms = timeit(kcopy, 0, (const float4*)cp, (float4*)(cp + n), n / 4);
  printf("%-40s %8.3f ms %8.1f GB/s\n", "copy float4", ms, 8.0 * n / ms / 1e6);
#define RUN(M)                                                                                      \
  rep("k8 U1 plain/plain", timeit(k8<1, 0, 0, M>, 0, A, v, th, codes, cstride, n), M);            \
  rep("k8 U1 noalloc/noalloc", timeit(k8<1, 1, 1, M>, 0, A, v, th, codes, cstride, n), M);        \
  rep("k8 U1 evictfirst/cs", timeit(k8<1, 2, 2, M>, 0, A, v, th, codes, cstride, n), M);          \
  rep("k8 U2 plain/plain", timeit(k8<2, 0, 0, M>, 0, A, v, th, codes, cstride, n), M);            \
  rep("k8 U2 noalloc/noalloc", timeit(k8<2, 1, 1, M>, 0, A, v, th, codes, cstride, n), M);        \
  rep("k8 U1 plain/plain 2blk", timeit(k8<1, 0, 0, M>, 2, A, v, th, codes, cstride, n), M);       \
  rep("k8 U1 plain/plain 8blk", timeit(k8<1, 0, 0, M>, 8, A, v, th, codes, cstride, n), M);       \
  rep("k4 U2 (v1)", timeit(k4<M>, 0, (float4*)A, (float4*)v, (float4*)th, (const uint16_t*)codes, cstride, n), M);
  RUN(1) RUN(2) RUN(4) RUN(8)
  cudaError_t e = cudaGetLastError();
  printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
