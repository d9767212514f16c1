/* synth.h — seeded, counter-based synthetic inputs for Streaming DiLoCo's
 * per-fragment outer sync.
 *
 * This is the ONE module both the CPU oracle (oracle/) and the CUDA path's
 * harness (tests/, bench.py) use.  It holds none of the method's arithmetic:
 * no outer gradient, no E3M0, no averaging, no Nesterov, no merge.  It only
 * produces the inputs the method consumes — initial parameters, the lumped
 * inner-step window updates, the tau-step drift and the toy per-step updates
 * (stand-ins for Alg. 2 L3-5, which need a model and data).
 *
 * Recipe: SURVEY.md §8(d) "Synthetic data", restated in DESIGN.md §3.
 *   H(x)      = splitmix64
 *   key(a,p,m,r) = H(H(H(H(seed ^ a) ^ p) ^ m) ^ r)   (m = 255: shared by replicas)
 *   U(key,i)  = ((H(key ^ i) >> 40) - 2^23) * 2^-23    exact fp32 in [-1, 1)
 * Every value is a pure function of (seed, purpose, p, m, r/t, i), so the
 * host (synth_cpu.c) and the device (synth_cuda.cu) produce identical bits
 * as long as each float op rounds once: SYN_MUL / SYN_ADD / SYN_SUB are
 * __fmul_rn/__fadd_rn/__fsub_rn on the device and plain ops compiled with
 * -ffp-contract=off on the host.
 */
#ifndef SYNTH_H_
#define SYNTH_H_

#include <stdint.h>

#ifdef __CUDACC__
#define SYN_FN static __host__ __device__ __forceinline__
#if defined(__CUDA_ARCH__)
#define SYN_MUL(a, b) __fmul_rn((a), (b))
#define SYN_ADD(a, b) __fadd_rn((a), (b))
#define SYN_SUB(a, b) __fsub_rn((a), (b))
#else
#define SYN_MUL(a, b) ((a) * (b))
#define SYN_ADD(a, b) ((a) + (b))
#define SYN_SUB(a, b) ((a) - (b))
#endif
#else
#define SYN_FN static inline
#define SYN_MUL(a, b) ((a) * (b))
#define SYN_ADD(a, b) ((a) + (b))
#define SYN_SUB(a, b) ((a) - (b))
#endif

#define SYNTH_SEED 250118512ULL

/* purpose codes */
enum {
  SYN_INIT = 1,      /* theta_init                (1, p, 255, 0) */
  SYN_SHARED = 2,    /* shared window component   (2, p, 255, r) */
  SYN_PRIVATE = 3,   /* private window component  (3, p, m,   r) */
  SYN_DRIFT = 4,     /* tau-step drift            (4, p, m,   r) */
  SYN_OUTLIER = 5,   /* outlier mask              (5, p, m,   r) */
  SYN_EMBROW = 6,    /* embedding-row mask        (6, p, 255, r) */
  SYN_TOY_SH = 7,    /* toy per-step shared       (7, 0, 255, t) */
  SYN_TOY_PR = 8     /* toy per-step private      (8, 0, m,   t) */
};

/* tensor kinds inside a fragment slab */
enum { SYN_MATRIX = 0, SYN_NORM = 1, SYN_EMBED = 2 };

typedef struct {
  int64_t start;       /* first element of the segment inside the fragment slab */
  int64_t len;         /* elements */
  int32_t kind;        /* SYN_MATRIX / SYN_NORM / SYN_EMBED */
  int32_t first_block; /* 1: tensor of transformer block 0 (higher cosine) */
  int32_t row;         /* d_model: embedding row length (row mask granularity) */
  int32_t pad_;
} synth_segment;

SYN_FN uint64_t syn_H(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

SYN_FN uint64_t syn_key(uint64_t seed, uint64_t purpose, uint64_t p, uint64_t m, uint64_t r) {
  return syn_H(syn_H(syn_H(syn_H(seed ^ purpose) ^ p) ^ m) ^ r);
}

/* exact fp32 in [-1, 1): a 24-bit integer times 2^-23 */
SYN_FN float syn_U(uint64_t key, uint64_t i) {
  int32_t k = (int32_t)(syn_H(key ^ i) >> 40) - (1 << 23);
  return (float)k * (1.0f / 8388608.0f);
}

/* sigma_c: 2^-9 for matrices and embedding, 2^-7 for norm gains */
SYN_FN float syn_sigma(int32_t kind) { return kind == SYN_NORM ? 0.0078125f : 0.001953125f; }

/* theta_init: 2^-6 * U1 (matrices, embedding); 1 + 2^-8 * U1 (norm gains) */
SYN_FN float syn_init_value(const synth_segment* s, uint64_t seed, int32_t p, int64_t i) {
  float u = syn_U(syn_key(seed, SYN_INIT, (uint64_t)p, 255, 0), (uint64_t)i);
  if (s->kind == SYN_NORM) return SYN_ADD(1.0f, SYN_MUL(0.00390625f, u));
  return SYN_MUL(0.015625f, u);
}

/* lumped H - tau inner steps of round r on replica m:
 *   D = sigma * ((w * U2) + U3), w = fl(1/3) (fl(2/3) in block 0);
 *   x 2^5 with probability 2^-12 (outliers); 0 on masked embedding rows. */
SYN_FN float syn_window_value(const synth_segment* s, uint64_t seed, int32_t p, int32_t m,
                              int32_t r, int64_t i) {
  if (s->kind == SYN_EMBED) {
    uint64_t row = (uint64_t)((i - s->start) / s->row);
    if ((syn_H(syn_key(seed, SYN_EMBROW, (uint64_t)p, 255, (uint64_t)r) ^ row) & 1ULL) == 0ULL)
      return 0.0f;
  }
  const float w = s->first_block ? (2.0f / 3.0f) : (1.0f / 3.0f);
  float u2 = syn_U(syn_key(seed, SYN_SHARED, (uint64_t)p, 255, (uint64_t)r), (uint64_t)i);
  float u3 = syn_U(syn_key(seed, SYN_PRIVATE, (uint64_t)p, (uint64_t)m, (uint64_t)r), (uint64_t)i);
  float d = SYN_MUL(syn_sigma(s->kind), SYN_ADD(SYN_MUL(w, u2), u3));
  if ((syn_H(syn_key(seed, SYN_OUTLIER, (uint64_t)p, (uint64_t)m, (uint64_t)r) ^ (uint64_t)i) &
       0xFFFULL) == 0ULL)
    d = SYN_MUL(d, 32.0f);
  return d;
}

/* tau overlapped inner steps: 2^-3 * sigma * U4 */
SYN_FN float syn_drift_value(const synth_segment* s, uint64_t seed, int32_t p, int32_t m,
                             int32_t r, int64_t i) {
  float u4 = syn_U(syn_key(seed, SYN_DRIFT, (uint64_t)p, (uint64_t)m, (uint64_t)r), (uint64_t)i);
  return SYN_MUL(SYN_MUL(0.125f, syn_sigma(s->kind)), u4);
}

/* toy config, one inner step t on replica m: 2^-12 * ((w * U7) + U8), w = fl(1/3) */
SYN_FN float syn_toy_value(uint64_t seed, int32_t m, int64_t t, int64_t i) {
  float u7 = syn_U(syn_key(seed, SYN_TOY_SH, 0, 255, (uint64_t)t), (uint64_t)i);
  float u8 = syn_U(syn_key(seed, SYN_TOY_PR, 0, (uint64_t)m, (uint64_t)t), (uint64_t)i);
  return SYN_MUL(0.000244140625f, SYN_ADD(SYN_MUL(1.0f / 3.0f, u7), u8));
}

#endif /* SYNTH_H_ */
