/* sd_oracle.h — the CPU oracle for Streaming DiLoCo's per-fragment outer sync.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load, call or execute
 * anything under oracle/.  The product path (paper_2501_18512_b200/) never
 * does; the two share no code, header, table or helper.  The one shared
 * module is synth/ (seeded inputs, no method arithmetic).
 *
 * Plain C99 (liboracle.so: single-threaded; liboracle_omp.so: the same
 * source built with -fopenmp, bit-identical results) that follows PAPER.md Alg. 2 (lines 103-134)
 * step by step in the paper's order, with SPEC.md's codec and optimizer
 * definitions, under the readings listed in DESIGN.md §2.  Built with
 * -O2 -fno-fast-math -ffp-contract=off: every float operation below rounds
 * once (IEEE binary32, round-to-nearest-even), nothing is fused.
 *
 * Parity status: every function here is pinned by a
 * `-m "not gpu"` test against something other than itself (paper worked
 * examples, SPEC examples, closed forms, exact-rational brute force,
 * torch.optim.SGD, textbook reductions).  None is "parity unpinned".
 */
#ifndef SD_ORACLE_H_
#define SD_ORACLE_H_
#include <stddef.h>
#include <stdint.h>

typedef struct {
  int32_t L;            /* number of synchronizable blocks (layers)            */
  int32_t fs;           /* fragment size |p| in blocks                          */
  int32_t pattern;      /* 0 sequential, 1 strided                              */
  int32_t embed_policy; /* 0: non-block params in the last fragment; 1: own   */
  int32_t H;            /* inner steps per round                                */
  int32_t tau;          /* overlap delay, 0 <= tau < H                          */
  int64_t T;            /* last step (flush), > 0 for the oracle's calendar     */
  float alpha, lr, mu;  /* merge mix, outer lr, outer momentum                  */
  int32_t B;            /* elements per scale block, 0 = one per fragment       */
} or_config;

typedef struct {
  int64_t t;         /* step (1-based)                         */
  int32_t kind;      /* 0 = send (Alg.2 L6-8), 1 = receive (L10-13) */
  int32_t p;         /* fragment                               */
  int64_t send_step; /* for receives: the matching send step   */
} or_event;

/* ---- schedule (Alg. 2 L6/L10) ---- */
int32_t or_num_fragments(const or_config* c);
int32_t or_fragment_blocks(const or_config* c, int32_t p, int32_t* out);
int32_t or_offset(const or_config* c, int32_t p);
int64_t or_calendar(const or_config* c, or_event* out, int64_t cap);

/* ---- codec ---- */
float or_block_scale(const float* d, int64_t len);
uint8_t or_e3m0_code(float d, float s);
float or_e3m0_decode(uint8_t code, float s);
int64_t or_num_scale_blocks(int64_t n, int32_t B);
size_t or_payload_bytes(int64_t n, int32_t B);
size_t or_scales_offset(int64_t n);
int or_quantize(const float* theta, const float* anchor, int64_t n, int32_t B, uint8_t* payload);
int or_payload_poisoned(const uint8_t* payload, int64_t n, int32_t B, uint64_t* first_bad);

/* ---- accumulation, OuterOpt, merge ---- */
void or_decode_mean(const uint8_t* gather, int32_t M, int64_t n, int32_t B, float* g);
void or_nesterov(float* A, float* v, const float* g, int64_t n, float lr, float mu);
void or_merge(float* theta, const float* A, int64_t n, float alpha);
void or_outer_state_init(const float* theta, float* A, float* v, int64_t n);
int or_apply(const uint8_t* gather, int32_t M, int64_t n, int32_t B, float lr, float mu,
             float alpha, float* A, float* v, float* theta);
int or_round(int32_t M, int64_t n, int32_t B, float lr, float mu, float alpha,
             float* const* theta_send, float* const* theta_merge_inout, float* A, float* v,
             uint8_t* gather);

/* ---- the toy configuration run end to end (Alg. 2 for t = 1..T) ---- */
int or_toy_run(const or_config* c, int32_t M, int64_t block_len, uint64_t seed, float* theta,
               float* A, float* v, int64_t* bytes_sent);

int or_toy_run_taus(const or_config* c, int32_t M, int64_t block_len, uint64_t seed, const int32_t* taus,
                    float* theta, float* A_m, float* v_m, int64_t* bytes_sent);

/* ---- InnerOpt = AdamW (NEXT-1) ---- */
void or_adamw(float* theta, const float* g, float* m, float* v, int64_t n, int64_t k, float lr, float b1,
              float b2, float eps, float wd);

#endif /* SD_ORACLE_H_ */
