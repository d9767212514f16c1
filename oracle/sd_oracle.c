/* sd_oracle.c — plain single-threaded CPU oracle of Streaming DiLoCo's
 * per-fragment outer synchronization.  TEST INFRASTRUCTURE ONLY (see
 * sd_oracle.h for who may call it).  Citations: "P:n" = PAPER.md line n,
 * "S:n" = SPEC.md line n; readings AMB-k are listed in DESIGN.md §2.
 *
 * Build: gcc -std=c99 -O2 -fno-fast-math -ffp-contract=off -shared -fPIC
 *        sd_oracle.c ../synth/synth_cpu.c -lm                 -> liboracle.so (1 thread)
 * and the same source with -fopenmp                           -> liboracle_omp.so
 * The `omp` pragmas below only split loops whose iterations are independent
 * (one element, one byte of codes, one scale block); every float operation,
 * and the ascending-m fold of each element, is the same in both builds, so
 * the N-thread oracle equals the 1-thread oracle bit for bit (SPEC.md:437,
 * :614 "determinism under parallelism"; pinned in tests/test_oracle_omp.py).
 * A max over |Delta| is exact and order-free; the first non-finite index is
 * a min over indices.
 */
#include "sd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "../synth/synth.h"

#define OR_MAGIC 0x31304453u /* "SD01" little-endian */

/* ===================================================================== */
/* Schedule                                                              */
/* ===================================================================== */

/* P = L / |p| block fragments, plus one embedding fragment when
 * embed_policy = 1 (AMB-4: reproduces "every 11, 5, 2 steps"). */
int32_t or_num_fragments(const or_config* c) {
  return c->L / c->fs + (c->embed_policy == 1 ? 1 : 0);
}

/* Blocks of fragment p: sequential p*|p| .. (p+1)*|p|-1, strided
 * p, p+P, p+2P, ... (P = number of block fragments).  The embedding fragment
 * of embed_policy 1 holds no blocks.  Returns the count written to out. */
int32_t or_fragment_blocks(const or_config* c, int32_t p, int32_t* out) {
  const int32_t Pb = c->L / c->fs;
  if (p >= Pb) return 0;
  for (int32_t k = 0; k < c->fs; ++k) out[k] = c->pattern == 0 ? p * c->fs + k : p + k * Pb;
  return c->fs;
}

/* t_p = floor(p * H / P). */
int32_t or_offset(const or_config* c, int32_t p) {
  const int64_t P = or_num_fragments(c);
  return (int32_t)(((int64_t)p * c->H) / P);
}

/* Brute-force calendar scan, t = 1..T (Alg. 2):
 *   send p at t   iff  t >= H and (t - t_p) mod H == 0      (L6; first send S:73)
 *   receive p     at  send + tau                              (L10)
 *   flush: a send whose receive would fall after T is received at T.
 * Within a step: inner step, then sends, then receives (Alg. 2 order, AMB-6);
 * ascending p inside each kind.  Returns the number of events (<= cap written). */
int64_t or_calendar(const or_config* c, or_event* out, int64_t cap) {
  const int32_t P = or_num_fragments(c);
  int64_t* pending = (int64_t*)malloc(sizeof(int64_t) * (size_t)P); /* send step in flight, or 0 */
  int64_t k = 0;
  for (int32_t p = 0; p < P; ++p) pending[p] = 0;
  for (int64_t t = 1; t <= c->T; ++t) {
    for (int32_t p = 0; p < P; ++p) {
      const int64_t tp = or_offset(c, p);
      if (t >= c->H && (t - tp) % c->H == 0) {
        if (k < cap) { out[k].t = t; out[k].kind = 0; out[k].p = p; out[k].send_step = t; }
        ++k;
        pending[p] = t;
      }
    }
    for (int32_t p = 0; p < P; ++p) {
      if (pending[p] == 0) continue;
      if (pending[p] + c->tau == t || t == c->T) {
        if (k < cap) { out[k].t = t; out[k].kind = 1; out[k].p = p; out[k].send_step = pending[p]; }
        ++k;
        pending[p] = 0;
      }
    }
  }
  free(pending);
  return k;
}

/* ===================================================================== */
/* E3M0 codec                                                            */
/* ===================================================================== */

/* scale = max |d| over the block (AMB-7); -0 counts as 0. */
float or_block_scale(const float* d, int64_t len) {
  float s = 0.0f;
#pragma omp parallel for reduction(max : s) if (len >= (1 << 16))
  for (int64_t i = 0; i < len; ++i) {
    float a = fabsf(d[i]);
    if (a > s) s = a;
  }
  return s;
}

/* E3M0 (AMB-8/9/10): code = sign<<3 | e, e in 1..7 meaning
 * sign * 2^(e-7) * s, chosen as the nearest grid point in log2; below
 * 2^-6.5 * s it underflows to code 0.  Written as exact threshold counts:
 *   e = #{ j in 0..6 : d^2 >= s^2 * 2^(-2j-1) }
 * i.e. |d| >= s * 2^(-j-1/2), the midpoint in log2 between 2^-j and
 * 2^-(j+1).  d^2 and s^2 of binary32 values are exact in binary64 and the
 * power-of-two scaling is exact, so every comparison is exact. */
uint8_t or_e3m0_code(float d, float s) {
  if (s == 0.0f) return 0;
  const double d2 = (double)d * (double)d;
  const double s2 = (double)s * (double)s;
  int e = 0;
  for (int j = 0; j <= 6; ++j)
    if (d2 >= ldexp(s2, -2 * j - 1)) ++e;
  if (e == 0) return 0; /* encoders emit s=0 with e=0 */
  return (uint8_t)((signbit(d) ? 8 : 0) | e);
}

/* decode: LUT[e] = 2^(e-7), LUT[8|e] = -2^(e-7), LUT[0] = LUT[8] = +0;
 * value = LUT[code] * s in binary32. */
float or_e3m0_decode(uint8_t code, float s) {
  static const float LUT[16] = {
      0.0f,     0.015625f,  0.03125f,  0.0625f,  0.125f,  0.25f,  0.5f,  1.0f,
      0.0f,    -0.015625f, -0.03125f, -0.0625f, -0.125f, -0.25f, -0.5f, -1.0f};
  return LUT[code & 15] * s;
}

/* number of scale blocks: B = 0 -> one per fragment; else ceil(n/B) */
int64_t or_num_scale_blocks(int64_t n, int32_t B) {
  if (n == 0) return 0;
  return B == 0 ? 1 : (n + B - 1) / B;
}

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

/* Payload layout (AMB-7/8; wire size S:261):
 *   [0, ceil(n/2))            codes, element 2k in the low nibble of byte k
 *   zero pad to 256           -> scales_offset
 *   nb fp32 scales (LE)
 *   zero pad to 16            -> trailer: u32 magic "SD01", u32 nb,
 *                                         u64 first non-finite index (2^64-1: clean)
 *   zero pad to 256 */
size_t or_scales_offset(int64_t n) { return (size_t)align_up((n + 1) / 2, 256); }

size_t or_payload_bytes(int64_t n, int32_t B) {
  const int64_t nb = or_num_scale_blocks(n, B);
  return or_scales_offset(n) + (size_t)align_up(align_up(4 * nb, 16) + 16, 256);
}

/* Alg. 2 L7 + E3M0 encode of one replica's fragment into one payload.
 *   Delta_i = A_i - theta_i        (anchor reading AMB-1; sign of S:183)
 *   per block b: s_b = max |Delta|, codes per or_e3m0_code, packed.
 * A non-finite Delta poisons the payload: its index goes into the trailer
 * ("non-finite input -> encode error with index"); codes and scales
 * of a poisoned payload are unspecified.  Returns 1 if poisoned, else 0. */
int or_quantize(const float* theta, const float* anchor, int64_t n, int32_t B, uint8_t* payload) {
  const size_t bytes = or_payload_bytes(n, B);
  const size_t soff = or_scales_offset(n);
  const int64_t nb = or_num_scale_blocks(n, B);
  const int64_t blen = B == 0 ? n : B;
  float* delta = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  uint64_t first_bad = UINT64_MAX;
  memset(payload, 0, bytes);

#pragma omp parallel for reduction(min : first_bad)
  for (int64_t i = 0; i < n; ++i) {
    delta[i] = anchor[i] - theta[i];
    if (!isfinite(delta[i]) && (uint64_t)i < first_bad) first_bad = (uint64_t)i;
  }
  /* B is even (a power of two >= 256) or the block is the whole fragment,
   * so no byte of codes straddles two blocks */
#pragma omp parallel for if (nb > 1)
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t lo = b * blen;
    const int64_t len = (lo + blen <= n) ? blen : n - lo;
    const float s = or_block_scale(delta + lo, len);
    memcpy(payload + soff + 4 * (size_t)b, &s, 4);
    /* byte k = code(2k) | code(2k+1) << 4; an odd tail leaves 0 in the high nibble */
#pragma omp parallel for if (nb == 1 && len >= (1 << 16))
    for (int64_t k = lo / 2; k < (lo + len + 1) / 2; ++k) {
      const uint8_t c0 = or_e3m0_code(delta[2 * k], s);
      const uint8_t c1 = (2 * k + 1 < lo + len) ? or_e3m0_code(delta[2 * k + 1], s) : 0;
      payload[k] = (uint8_t)(c0 | (c1 << 4));
    }
  }
  {
    const size_t toff = soff + (size_t)align_up(4 * nb, 16);
    const uint32_t magic = OR_MAGIC, nb32 = (uint32_t)nb;
    memcpy(payload + toff, &magic, 4);
    memcpy(payload + toff + 4, &nb32, 4);
    memcpy(payload + toff + 8, &first_bad, 8);
  }
  free(delta);
  return first_bad != UINT64_MAX;
}

/* reads the trailer: returns 1 if poisoned (first_bad set), -1 if the magic is wrong */
int or_payload_poisoned(const uint8_t* payload, int64_t n, int32_t B, uint64_t* first_bad) {
  const size_t toff = or_scales_offset(n) + (size_t)align_up(4 * or_num_scale_blocks(n, B), 16);
  uint32_t magic;
  uint64_t fb;
  memcpy(&magic, payload + toff, 4);
  memcpy(&fb, payload + toff + 8, 8);
  if (first_bad) *first_bad = fb;
  if (magic != OR_MAGIC) return -1;
  return fb != UINT64_MAX;
}

/* ===================================================================== */
/* Accumulation, OuterOpt, merge                                         */
/* ===================================================================== */

/* Alg. 2 L8 receive side ("1/M sum", "accumulation is done in
 * FP32"; S:385 ascending replica order, then divide by M; AMB-11/12):
 *   S_i = q_{0,i};  S_i = S_i + q_{m,i} for m = 1..M-1;  g_i = S_i / M
 * with q_{m,i} = decode(code_{m,i}, s_{m,b(i)}).  Every replica, including
 * the local one, contributes its decoded value. */
void or_decode_mean(const uint8_t* gather, int32_t M, int64_t n, int32_t B, float* g) {
  const size_t pb = or_payload_bytes(n, B);
  const size_t soff = or_scales_offset(n);
  const int64_t blen = B == 0 ? n : B;
#pragma omp parallel for
  for (int64_t i = 0; i < n; ++i) {
    float S = 0.0f;
    for (int32_t m = 0; m < M; ++m) {
      const uint8_t* slot = gather + (size_t)m * pb;
      const uint8_t byte = slot[i / 2];
      const uint8_t code = (uint8_t)((i % 2 == 0) ? (byte & 15) : (byte >> 4));
      float s;
      memcpy(&s, slot + soff + 4 * (size_t)(i / blen), 4);
      const float q = or_e3m0_decode(code, s);
      S = (m == 0) ? q : S + q;
    }
    g[i] = S / (float)M;
  }
}

/* OuterOpt = SGD with Nesterov momentum (Alg. 2 L12), the
 * "momentum-then-lookahead" form of S:184 (AMB-13):
 *   v <- mu*v + g ;  A <- A - lr*(g + mu*v)   (v already updated) */
void or_nesterov(float* A, float* v, const float* g, int64_t n, float lr, float mu) {
#pragma omp parallel for
  for (int64_t i = 0; i < n; ++i) {
    v[i] = mu * v[i] + g[i];
    A[i] = A[i] - lr * (g[i] + mu * v[i]);
  }
}

/* Outer-state store init ("outer global
 * parameters" + "outer Nesterov state"): the anchor starts as
 * the initial parameters, A_p <- theta_init,p (bit copy, AMB-2), and the
 * outer momentum at zero, v_p <- 0. */
void or_outer_state_init(const float* theta, float* A, float* v, int64_t n) {
  memcpy(A, theta, sizeof(float) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) v[i] = 0.0f;
}

/* alpha-merge (Alg. 2 L13): theta <- alpha*theta + (1-alpha)*A,
 * with beta = 1 - alpha rounded once (AMB-14). */
void or_merge(float* theta, const float* A, int64_t n, float alpha) {
  const float beta = 1.0f - alpha;
#pragma omp parallel for
  for (int64_t i = 0; i < n; ++i) theta[i] = alpha * theta[i] + beta * A[i];
}

/* One replica's receive (Alg. 2 L11-13): block-receive done by the caller;
 * if any of the M payloads is poisoned nothing changes (DESIGN.md §5:
 * rank-consistent skip); else mean, Nesterov on the anchor, merge.
 * Returns 1 if skipped because of poison, -1 on a bad magic, 0 otherwise. */
int or_apply(const uint8_t* gather, int32_t M, int64_t n, int32_t B, float lr, float mu,
             float alpha, float* A, float* v, float* theta) {
  const size_t pb = or_payload_bytes(n, B);
  for (int32_t m = 0; m < M; ++m) {
    const int r = or_payload_poisoned(gather + (size_t)m * pb, n, B, NULL);
    if (r != 0) return r;
  }
  float* g = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  or_decode_mean(gather, M, n, B, g);
  or_nesterov(A, v, g, n, lr, mu);
  or_merge(theta, A, n, alpha);
  free(g);
  return 0;
}

/* One full round for one fragment on all M replicas (Alg. 2 L6-13):
 * quantize each theta_send[m] against A into gather slot m, then (as every
 * replica would after the all-gather) mean + Nesterov once on the shared
 * anchor/momentum, and merge into every theta_merge[m] (live parameters
 * after the tau overlapped steps).  gather: M * or_payload_bytes(n, B). */
int or_round(int32_t M, int64_t n, int32_t B, float lr, float mu, float alpha,
             float* const* theta_send, float* const* theta_merge_inout, float* A, float* v,
             uint8_t* gather) {
  const size_t pb = or_payload_bytes(n, B);
  int poisoned = 0;
  for (int32_t m = 0; m < M; ++m)
    poisoned |= or_quantize(theta_send[m], A, n, B, gather + (size_t)m * pb);
  if (poisoned) return 1;
  {
    float* g = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
    or_decode_mean(gather, M, n, B, g);
    or_nesterov(A, v, g, n, lr, mu);
    for (int32_t m = 0; m < M; ++m) or_merge(theta_merge_inout[m], A, n, alpha);
    free(g);
  }
  return 0;
}

/* ===================================================================== */
/* The toy configuration, Alg. 2 end to end                              */
/* ===================================================================== */

/* Runs Alg. 2 for t = 1..T on M replicas of a flat vector of
 * L blocks of block_len elements, fragment-contiguous (AMB-18):
 *   theta[m*Ntot + p*n_p + i], A[p*n_p + i], v[p*n_p + i],  n_p = |p|*block_len.
 * Init: A_p = theta_init (2^-6 * U1, synth.h), v_p = 0, theta_m = A (AMB-2).
 * Step t: L3-5 inner step = synthetic update theta_m <- theta_m - u(m,t)
 *         (synth.h, global index p*n_p + i); L6-8 sends (quantize every
 *         replica into the fragment's gather buffer); L10-13 receives
 *         (or_apply per replica on the shared anchor, momentum once).
 * The calendar is or_calendar (brute force).  bytes_sent accumulates
 * M * payload per send.  Returns 0, or 1 if a round was poisoned. */
int or_toy_run(const or_config* c, int32_t M, int64_t block_len, uint64_t seed, float* theta,
               float* A, float* v, int64_t* bytes_sent) {
  const int32_t P = or_num_fragments(c);
  const int64_t n = (int64_t)c->fs * block_len;
  const int64_t Ntot = (int64_t)P * n;
  const size_t pb = or_payload_bytes(n, c->B);
  uint8_t* gather = (uint8_t*)calloc((size_t)P * (size_t)M, pb);
  int64_t nev = or_calendar(c, NULL, 0);
  or_event* ev = (or_event*)malloc(sizeof(or_event) * (size_t)(nev > 0 ? nev : 1));
  int any_poison = 0;
  synth_segment seg;
  or_calendar(c, ev, nev);
  *bytes_sent = 0;

  for (int32_t p = 0; p < P; ++p) {
    seg.start = 0; seg.len = n; seg.kind = SYN_MATRIX; seg.first_block = 0; seg.row = 1; seg.pad_ = 0;
    for (int64_t i = 0; i < n; ++i) A[p * n + i] = syn_init_value(&seg, seed, p, i);
    for (int64_t i = 0; i < n; ++i) v[p * n + i] = 0.0f;
  }
  for (int32_t m = 0; m < M; ++m) memcpy(theta + m * Ntot, A, sizeof(float) * (size_t)Ntot);

  int64_t e = 0;
  for (int64_t t = 1; t <= c->T; ++t) {
    for (int32_t m = 0; m < M; ++m) /* L3-5 */
      for (int64_t gi = 0; gi < Ntot; ++gi)
        theta[m * Ntot + gi] = theta[m * Ntot + gi] - syn_toy_value(seed, m, t, gi);
    for (; e < nev && ev[e].t == t; ++e) {
      const int32_t p = ev[e].p;
      uint8_t* gp = gather + (size_t)p * (size_t)M * pb;
      if (ev[e].kind == 0) { /* L6-8: Delta, E3M0, (all-)gather */
        for (int32_t m = 0; m < M; ++m)
          or_quantize(theta + m * Ntot + p * n, A + p * n, n, c->B, gp + (size_t)m * pb);
        *bytes_sent += (int64_t)M * (int64_t)pb;
      } else { /* L10-13: mean, OuterOpt on the anchor (once), merge each replica */
        float* g = (float*)malloc(sizeof(float) * (size_t)n);
        int skip = 0;
        for (int32_t m = 0; m < M; ++m) skip |= or_payload_poisoned(gp + (size_t)m * pb, n, c->B, NULL) != 0;
        if (skip) { any_poison = 1; free(g); continue; }
        or_decode_mean(gp, M, n, c->B, g);
        or_nesterov(A + p * n, v + p * n, g, n, c->lr, c->mu);
        for (int32_t m = 0; m < M; ++m) or_merge(theta + m * Ntot + p * n, A + p * n, n, c->alpha);
        free(g);
      }
    }
  }
  free(ev);
  free(gather);
  return any_poison;
}

/* Per-replica overlap delay tau_m (Sec. 3.3.2 "Overlapping
 * with some slack between workers": all replicas send at the same step, each
 * receives tau_m steps later).  Same as or_toy_run but every
 * replica keeps its own copy of the (replicated) anchor and momentum, applies
 * OuterOpt at its own receive step and merges its own parameters then.
 * A_m[m*Ntot + ...], v_m likewise.  Returns 0, or 1 if a round was poisoned. */
int or_toy_run_taus(const or_config* c, int32_t M, int64_t block_len, uint64_t seed, const int32_t* taus,
                    float* theta, float* A_m, float* v_m, int64_t* bytes_sent) {
  const int32_t P = or_num_fragments(c);
  const int64_t n = (int64_t)c->fs * block_len;
  const int64_t Ntot = (int64_t)P * n;
  const size_t pb = or_payload_bytes(n, c->B);
  uint8_t* gather = (uint8_t*)calloc((size_t)P * (size_t)M, pb);
  or_event** ev = (or_event**)malloc(sizeof(or_event*) * (size_t)M);
  int64_t* nev = (int64_t*)malloc(sizeof(int64_t) * (size_t)M);
  int64_t* e = (int64_t*)calloc((size_t)M, sizeof(int64_t));
  float* g = (float*)malloc(sizeof(float) * (size_t)(n > 0 ? n : 1));
  int any_poison = 0;
  synth_segment seg;
  *bytes_sent = 0;
  for (int32_t m = 0; m < M; ++m) { /* each replica's own calendar: same sends, receives at s + tau_m */
    or_config cm = *c;
    cm.tau = taus[m];
    nev[m] = or_calendar(&cm, NULL, 0);
    ev[m] = (or_event*)malloc(sizeof(or_event) * (size_t)(nev[m] > 0 ? nev[m] : 1));
    or_calendar(&cm, ev[m], nev[m]);
  }
  for (int32_t p = 0; p < P; ++p) {
    seg.start = 0; seg.len = n; seg.kind = SYN_MATRIX; seg.first_block = 0; seg.row = 1; seg.pad_ = 0;
    for (int64_t i = 0; i < n; ++i) A_m[p * n + i] = syn_init_value(&seg, seed, p, i);
    for (int64_t i = 0; i < n; ++i) v_m[p * n + i] = 0.0f;
  }
  for (int32_t m = 1; m < M; ++m) {
    memcpy(A_m + m * Ntot, A_m, sizeof(float) * (size_t)Ntot);
    memcpy(v_m + m * Ntot, v_m, sizeof(float) * (size_t)Ntot);
  }
  for (int32_t m = 0; m < M; ++m) memcpy(theta + m * Ntot, A_m, sizeof(float) * (size_t)Ntot);

  for (int64_t t = 1; t <= c->T; ++t) {
    for (int32_t m = 0; m < M; ++m) /* L3-5 */
      for (int64_t gi = 0; gi < Ntot; ++gi)
        theta[m * Ntot + gi] = theta[m * Ntot + gi] - syn_toy_value(seed, m, t, gi);
    /* L6-8: sends are common to all replicas (replica 0's calendar lists them) */
    for (int64_t k = e[0]; k < nev[0] && ev[0][k].t == t; ++k) {
      if (ev[0][k].kind != 0) continue;
      const int32_t p = ev[0][k].p;
      uint8_t* gp = gather + (size_t)p * (size_t)M * pb;
      for (int32_t m = 0; m < M; ++m)
        or_quantize(theta + m * Ntot + p * n, A_m + m * Ntot + p * n, n, c->B, gp + (size_t)m * pb);
      *bytes_sent += (int64_t)M * (int64_t)pb;
    }
    /* L10-13 per replica at its own receive steps */
    for (int32_t m = 0; m < M; ++m) {
      for (; e[m] < nev[m] && ev[m][e[m]].t == t; ++e[m]) {
        if (ev[m][e[m]].kind != 1) continue;
        const int32_t p = ev[m][e[m]].p;
        uint8_t* gp = gather + (size_t)p * (size_t)M * pb;
        int skip = 0;
        for (int32_t q = 0; q < M; ++q) skip |= or_payload_poisoned(gp + (size_t)q * pb, n, c->B, NULL) != 0;
        if (skip) { any_poison = 1; continue; }
        or_decode_mean(gp, M, n, c->B, g);
        or_nesterov(A_m + m * Ntot + p * n, v_m + m * Ntot + p * n, g, n, c->lr, c->mu);
        or_merge(theta + m * Ntot + p * n, A_m + m * Ntot + p * n, n, c->alpha);
      }
    }
  }
  for (int32_t m = 0; m < M; ++m) free(ev[m]);
  free(ev); free(nev); free(e); free(g); free(gather);
  return any_poison;
}

/* ===================================================================== */
/* InnerOpt = AdamW (NEXT-1)                                             */
/* ===================================================================== */

/* One AdamW inner step (Alg. 2 L5; InnerOpt = Adam, P:77;
 * SPEC.md:171-179 adamw_step, decoupled weight decay), step index k >= 1.
 * Operation order (DESIGN.md §2 AMB-20), each op rounded once:
 *   m <- b1*m + (1-b1)*g ;  v <- b2*v + (1-b2)*(g*g)
 *   denom = sqrt(v) / sqrt(bc2) + eps
 *   theta <- theta*(1 - lr*wd) - (lr/bc1) * (m / denom)
 * with bc1 = 1 - b1^k, bc2 = 1 - b2^k (evaluated in binary64, rounded to
 * binary32 once), and 1-b1, 1-b2, 1-lr*wd, lr/bc1, sqrt(bc2) rounded once. */
void or_adamw(float* theta, const float* g, float* m, float* v, int64_t n, int64_t k, float lr, float b1,
              float b2, float eps, float wd) {
  const float bc1 = (float)(1.0 - pow((double)b1, (double)k));
  const float bc2 = (float)(1.0 - pow((double)b2, (double)k));
  const float c1 = 1.0f - b1, c2 = 1.0f - b2;
  const float decay = 1.0f - lr * wd;
  const float step = lr / bc1;
  const float sbc2 = sqrtf(bc2);
#pragma omp parallel for
  for (int64_t i = 0; i < n; ++i) {
    m[i] = b1 * m[i] + c1 * g[i];
    v[i] = b2 * v[i] + c2 * (g[i] * g[i]);
    const float denom = sqrtf(v[i]) / sbc2 + eps;
    theta[i] = theta[i] * decay - step * (m[i] / denom);
  }
}
