/* synth_cpu.c — host implementation of synth.h's generators over arrays.
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -shared -fPIC.
 * All functions work on the element range [i0, i1) of a fragment slab; `x`
 * points at element i0.  No method arithmetic lives here (see synth.h). */
#include <stddef.h>
#include "synth.h"

/* segment holding element i (segments are sorted and cover the slab) */
static const synth_segment* seg_of(const synth_segment* segs, int nseg, int64_t i) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {
    int mid = (lo + hi + 1) / 2;
    if (segs[mid].start <= i) lo = mid; else hi = mid - 1;
  }
  return &segs[lo];
}

void synth_fill_init(float* x, const synth_segment* segs, int nseg, uint64_t seed, int32_t p,
                     int64_t i0, int64_t i1) {
  for (int64_t i = i0; i < i1; ++i) x[i - i0] = syn_init_value(seg_of(segs, nseg, i), seed, p, i);
}

/* theta <- theta - D (the lumped window of round r) */
void synth_apply_window(float* x, const synth_segment* segs, int nseg, uint64_t seed, int32_t p,
                        int32_t m, int32_t r, int64_t i0, int64_t i1) {
  for (int64_t i = i0; i < i1; ++i)
    x[i - i0] = SYN_SUB(x[i - i0], syn_window_value(seg_of(segs, nseg, i), seed, p, m, r, i));
}

/* theta <- theta - drift (the tau overlapped steps of round r) */
void synth_apply_drift(float* x, const synth_segment* segs, int nseg, uint64_t seed, int32_t p,
                       int32_t m, int32_t r, int64_t i0, int64_t i1) {
  for (int64_t i = i0; i < i1; ++i)
    x[i - i0] = SYN_SUB(x[i - i0], syn_drift_value(seg_of(segs, nseg, i), seed, p, m, r, i));
}

/* toy config: theta <- theta - u(m, t) for one inner step t */
void synth_apply_toy(float* x, uint64_t seed, int32_t m, int64_t t, int64_t i0, int64_t i1) {
  for (int64_t i = i0; i < i1; ++i) x[i - i0] = SYN_SUB(x[i - i0], syn_toy_value(seed, m, t, i));
}

/* raw draws, for tests of the generator itself */
void synth_fill_U(float* x, uint64_t key, int64_t i0, int64_t i1) {
  for (int64_t i = i0; i < i1; ++i) x[i - i0] = syn_U(key, (uint64_t)i);
}
uint64_t synth_key(uint64_t seed, uint64_t purpose, uint64_t p, uint64_t m, uint64_t r) {
  return syn_key(seed, purpose, p, m, r);
}
uint64_t synth_H(uint64_t x) { return syn_H(x); }
