// synth_cuda.cu — device twin of synth_cpu.c (harness only: tests and bench.py
// create their inputs with it; it is never part of the timed hot path).
// Bit-identical to the host generator: same synth.h, each float op rounded once.
#include <cuda_runtime.h>
#include <stdint.h>
#include "synth.h"

namespace {

enum Op { FILL_INIT = 0, APPLY_WINDOW = 1, APPLY_DRIFT = 2 };

__global__ void k_synth_seg(float* __restrict__ x, synth_segment seg, uint64_t seed, int32_t p,
                            int32_t m, int32_t r, int64_t lo, int64_t hi, int64_t i0, int op) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi; i += stride) {
    float* px = x + (i - i0);
    if (op == FILL_INIT) *px = syn_init_value(&seg, seed, p, i);
    else if (op == APPLY_WINDOW) *px = __fsub_rn(*px, syn_window_value(&seg, seed, p, m, r, i));
    else *px = __fsub_rn(*px, syn_drift_value(&seg, seed, p, m, r, i));
  }
}

__global__ void k_synth_toy(float* __restrict__ x, uint64_t seed, int32_t m, int64_t t, int64_t i0,
                            int64_t i1) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < i1; i += stride)
    x[i - i0] = __fsub_rn(x[i - i0], syn_toy_value(seed, m, t, i));
}

// AdamW-shaped synthetic inner step (the overlap load of bench.py; a stand-in
// for Alg. 2 L3-5, not the method): gradient from a counter
// hash, m/v moments, bias-corrected update.  Reads theta, m, v and writes them
// back: 24 B per parameter, like a fused optimizer pass.
__global__ void k_inner_adamw(float* __restrict__ th, float* __restrict__ m1, float* __restrict__ m2,
                              int64_t n, uint64_t key, float lr, float bc1, float bc2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float g = 1e-3f * syn_U(key, (uint64_t)i);
    const float a = 0.9f * m1[i] + 0.1f * g;
    const float b = 0.99f * m2[i] + 0.01f * g * g;
    m1[i] = a;
    m2[i] = b;
    th[i] -= lr * ((a / bc1) / (sqrtf(b / bc2) + 1e-8f));
  }
}

int grid_for(int64_t n) {
  int64_t g = (n + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : (int)g;
}

int run_segments(float* x, const synth_segment* segs, int nseg, uint64_t seed, int32_t p,
                 int32_t m, int32_t r, int64_t i0, int64_t i1, int op, cudaStream_t st) {
  for (int s = 0; s < nseg; ++s) {
    int64_t lo = segs[s].start > i0 ? segs[s].start : i0;
    int64_t hi = segs[s].start + segs[s].len < i1 ? segs[s].start + segs[s].len : i1;
    if (lo >= hi) continue;
    k_synth_seg<<<grid_for(hi - lo), 256, 0, st>>>(x, segs[s], seed, p, m, r, lo, hi, i0, op);
  }
  return (int)cudaGetLastError();
}

}  // namespace

extern "C" {

// segs: HOST array of segments; x: DEVICE pointer to element i0.  Returns cudaError_t.
int synth_cuda_fill_init(float* x, const synth_segment* segs, int nseg, uint64_t seed, int32_t p,
                         int64_t i0, int64_t i1, cudaStream_t st) {
  return run_segments(x, segs, nseg, seed, p, 0, 0, i0, i1, FILL_INIT, st);
}
int synth_cuda_apply_window(float* x, const synth_segment* segs, int nseg, uint64_t seed,
                            int32_t p, int32_t m, int32_t r, int64_t i0, int64_t i1,
                            cudaStream_t st) {
  return run_segments(x, segs, nseg, seed, p, m, r, i0, i1, APPLY_WINDOW, st);
}
int synth_cuda_apply_drift(float* x, const synth_segment* segs, int nseg, uint64_t seed,
                           int32_t p, int32_t m, int32_t r, int64_t i0, int64_t i1,
                           cudaStream_t st) {
  return run_segments(x, segs, nseg, seed, p, m, r, i0, i1, APPLY_DRIFT, st);
}
int synth_cuda_apply_toy(float* x, uint64_t seed, int32_t m, int64_t t, int64_t i0, int64_t i1,
                         cudaStream_t st) {
  if (i1 <= i0) return 0;
  k_synth_toy<<<grid_for(i1 - i0), 256, 0, st>>>(x, seed, m, t, i0, i1);
  return (int)cudaGetLastError();
}

int synth_cuda_inner_adamw(float* th, float* m1, float* m2, int64_t n, uint64_t seed, int32_t m, int64_t t,
                           cudaStream_t st) {
  if (n <= 0) return 0;
  const float bc1 = 1.0f - powf(0.9f, (float)t), bc2 = 1.0f - powf(0.99f, (float)t);
  k_inner_adamw<<<148 * 8, 256, 0, st>>>(th, m1, m2, n, syn_key(seed, 9, 0, (uint64_t)m, (uint64_t)t), 1e-4f,
                                         bc1, bc2);
  return (int)cudaGetLastError();
}

}  // extern "C"
