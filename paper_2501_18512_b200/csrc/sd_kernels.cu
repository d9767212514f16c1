// sd_kernels.cu — the hot path of Streaming DiLoCo's per-fragment outer sync
// on B200 (sm_100a).  Two HBM-bound kernels (no tensor-core work: every step
// is elementwise or a per-block max):
//
//   k_quantize  Alg. 2 L7 + E3M0
//               Delta = A - theta, per-block absmax (warp REDUX), exact
//               E3M0 code, nibble pack, payload trailer.
//   k_apply     Alg. 2 L8 receive side + L12 + L13
//               decode, M-way fp32 sum in ascending replica order, /M,
//               Nesterov, anchor update, alpha-merge.
//   k_absmax + k_encode_staged (k_encode without a workspace): the two-pass
//               variant for B = 0 (one scale per fragment) and
//               B > 1024 -- pass 1 keeps 16-bit summaries of the Deltas in
//               the caller's workspace, pass 2 encodes from them.
// Around them: the fused all-gather protocol (push: NVLink stores from the
// quantize; pull: NVLink loads in the apply; round flags signalled by the
// payload kernel's last CTA or a one-thread kernel, k_round_wait for the
// block-receive) and the AdamW inner step fused with
// the quantize or its first pass (k_adamw_quantize, k_adamw_absmax) and with
// the apply (k_apply<M, true>) -- SURVEY.md §8(f) NEXT-1/NEXT-2.
//
// Memory: every lane moves 8 consecutive fp32 with one 256-bit access
// (sm_100 LDG.256 / STG.256), so a warp instruction covers 1 KB and a lane's
// 8 codes are one 32-bit word of the payload.
//
// Arithmetic: every float op is an explicit round-to-nearest intrinsic and the
// file is compiled with -fmad=false: nothing is contracted into an FMA
// (DESIGN.md §2 AMB-15), so the results equal the oracle's bit for bit.
//
// Exact E3M0: code e = #{j in 0..6 : |d| >= T_j}, T_j the
// smallest binary32 with T_j^2 >= s^2 2^(-2j-1) (checked in exact binary64).
// While T_6 is a normal number, T_j = T_0 / 2^j exactly, i.e. bits(T_j) =
// bits(T_0) - j 2^23, and since |d| <= s < 2 T_0 the count is the integer
//   e = max(0, 7 - ((bits(T_0) + 2^23 - 1 - bits(|d|)) >> 23)).
// Blocks whose T_6 would be subnormal (s < ~2^-119.5) take the 7-compare path.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <float.h>
#include <math_constants.h>
#include <stdint.h>
#include <stdlib.h>

#include "sd_kernels.h"

namespace sdk {
namespace {

constexpr uint32_t kMagic = 0x31304453u;  // "SD01"
constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;
constexpr uint32_t kInfBits = 0x7f800000u;

struct f8 {
  float v[8];
};

// 256-bit global accesses (sm_100): read-once streams bypass L1.
__device__ __forceinline__ f8 ld8_stream(const float* p) {
  f8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                 "=f"(r.v[6]), "=f"(r.v[7])
               : "l"(p));
  return r;
}
// the same, evict-first in L2 (data this pass reads once and nobody re-reads soon)
__device__ __forceinline__ f8 ld8_stream_ef(const float* p) {
  f8 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                 "=f"(r.v[6]), "=f"(r.v[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ f8 ld8(const float* p) {
  f8 r;
  asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                 "=f"(r.v[6]), "=f"(r.v[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_global_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st8(float* p, const f8& r) {
  asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(r.v[0]),
               "f"(r.v[1]), "f"(r.v[2]), "f"(r.v[3]), "f"(r.v[4]), "f"(r.v[5]), "f"(r.v[6]), "f"(r.v[7])
               : "memory");
}
__device__ __forceinline__ uint32_t ld_code_word(const uint32_t* p) {
  uint32_t w;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(w) : "l"(p));
  return w;
}

__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7fffffffu; }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Smallest binary32 x >= 0 with (double)x * x >= s^2 * 2^(-2j-1): |d| >= T_j
// <=> d^2 >= s^2 2^(-2j-1) exactly, i.e. |d|/s >= 2^(-j-1/2), the log2
// midpoint between grid points 2^-j and 2^-(j+1).  s = 0 -> +inf (all codes 0).
__device__ __noinline__ float e3m0_threshold(float s, int j) {
  if (!(s > 0.0f) || !(s <= FLT_MAX)) return CUDART_INF_F;
  const double pw = __longlong_as_double((long long)(1023 - 2 * j - 1) << 52);   // 2^(-2j-1)
  const double b = __dmul_rn(__dmul_rn((double)s, (double)s), pw);              // exact
  const double k = __dmul_rn(0.70710678118654757, __longlong_as_double((long long)(1023 - j) << 52));
  float c = __double2float_rn(__dmul_rn((double)s, k));                          // ~ s 2^(-j-1/2)
  while (__dmul_rn((double)c, (double)c) < b) c = __uint_as_float(__float_as_uint(c) + 1u);
  while (c > 0.0f) {
    const float pc = __uint_as_float(__float_as_uint(c) - 1u);
    if (__dmul_rn((double)pc, (double)pc) >= b) c = pc; else break;
  }
  return c;
}

// Fast-path encode (T_0..T_6 normal): c0 = bits(T_0) + 2^23 - 1.
__device__ __forceinline__ uint32_t encode_fast(float d, uint32_t c0) {
  const uint32_t db = __float_as_uint(d);
  const int k = (int)((c0 - (db & 0x7fffffffu)) >> 23);
  const uint32_t e = (uint32_t)max(7 - k, 0);
  return e | ((e + 7u) & (db >> 28) & 8u);  // sign bit only when e > 0 (never code 8)
}

// General encode: e = #{j : |d| >= T_j} against explicit thresholds.
__device__ __forceinline__ uint32_t encode_slow(float d, const float (&T)[7]) {
  const float a = fabsf(d);
  uint32_t e = 0;
#pragma unroll
  for (int j = 0; j < 7; ++j) e += (uint32_t)(a >= T[j]);
  return e | ((e + 7u) & (__float_as_uint(d) >> 28) & 8u);
}

__device__ __forceinline__ bool fast_ok(float s, float t0) {
  // all seven thresholds normal (bits(T_6) >= 2^23) and s finite, nonzero
  return s > 0.0f && s <= FLT_MAX && __float_as_uint(t0) >= 0x03800000u;
}

struct QArgs {
  const float* theta;
  const float* anchor;
  int64_t n;        // elements
  int64_t nb;       // scale blocks
  int32_t lgB;      // log2(B), or -1 for one block per fragment
  uint8_t* slot;    // payload base
  size_t scales_off, trailer_off, bytes;
  // fused all-gather (push mode): every payload word is also stored into the
  // same offset of this rank's slot in each peer's gather buffer (NVLink,
  // NCCL symmetric window, LSA pointers)
  int push;
  ncclWindow_t win;
  size_t win_off;   // window offset of this rank's slot (same on every rank)
  int rank, M;
  // round signal (push and pull modes) fused into the kernel's last CTA:
  // {round id, first_bad} release-stored into entry `rank` of every peer's
  // flag array (window offset flags_off); `counter` elects the last CTA
  int sig;
  size_t flags_off;
  unsigned long long seq;
  unsigned int* counter;
  // staged two-pass quantize (B = 0 or B > 1024, caller workspace): pass 1
  // also writes a 16-bit summary of every Delta (2 per word; chunk c, row k,
  // lane l at word c*512 + 128k + 4l) and each row's max |Delta| bits
  // (stg_max[4c + k]); pass 2 encodes from them.  Null: pass 2 re-reads theta, A.
  uint32_t* stg;
  uint32_t* stg_max;
  int stg_hints;    // bit 0: pass 1 reads theta, A (and g) L2 evict-first; bit 1: pass 2 discards consumed lines
  int64_t stg_keep_from;  // pass 1 stores the summaries of chunks >= this L2 evict-last (pass 2 reads them first)
};

__device__ __forceinline__ void push_u32(const QArgs& a, size_t off, uint32_t v) {
  for (int q = 0; q < a.M; ++q)
    if (q != a.rank) *reinterpret_cast<uint32_t*>(ncclGetLsaPointer(a.win, a.win_off + off, q)) = v;
}
__device__ __forceinline__ void push_u8(const QArgs& a, size_t off, uint8_t v) {
  for (int q = 0; q < a.M; ++q)
    if (q != a.rank) *reinterpret_cast<uint8_t*>(ncclGetLsaPointer(a.win, a.win_off + off, q)) = v;
}

// Round signal, fused into the end of the kernel that finishes the payload
// (DESIGN.md §7): every CTA, after its last store (bar.sync), takes a ticket
// with an acquire-release atomic; the CTA that takes the last one has
// observed every other CTA's payload writes (release/acquire chain through
// the counter, cumulative over each CTA's barrier), so after a system-scope fence
// its release-stores of {round id, first non-finite index} into each peer's
// flag entry publish the whole payload to the peers' acquire loads.  In push
// mode it also copies the first non-finite index into the peers' copies of
// this rank's trailer.  The counter is reset for the next round (stream order).
__device__ __forceinline__ void signal_round(const QArgs& a) {
  __syncthreads();
  if (threadIdx.x != 0) return;
  unsigned int ticket;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(ticket) : "l"(a.counter) : "memory");
  if (ticket != gridDim.x - 1) return;
  const unsigned long long fb = *reinterpret_cast<volatile unsigned long long*>(a.slot + a.trailer_off + 8);
  *a.counter = 0u;
  if (a.push)
    for (int q = 0; q < a.M; ++q)
      if (q != a.rank)
        *reinterpret_cast<unsigned long long*>(ncclGetLsaPointer(a.win, a.win_off + a.trailer_off + 8, q)) = fb;
  __threadfence_system();
  for (int q = 0; q < a.M; ++q) {
    if (q == a.rank) continue;
    unsigned long long* e =
        reinterpret_cast<unsigned long long*>(ncclGetLsaPointer(a.win, a.flags_off + 16 * (size_t)a.rank, q));
    e[1] = fb;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(e), "l"(a.seq) : "memory");
  }
}

// Chunk = 1024 elements = 4 rows of 256; lane `lane` owns elements
// c*1024 + k*256 + 8*lane .. +7 of row k (one LDG.256 per array and row).
// Elements past n of the ragged last chunk read as Delta = +0.
template <bool kFullChunk, bool kEvictFirst = false>
__device__ __forceinline__ void load_chunk(const QArgs& a, int64_t c, int lane, f8 (&d)[4]) {
  const int64_t e0 = c * 1024 + 8 * lane;
  if (kFullChunk) {
    f8 th[4], an[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      th[k] = kEvictFirst ? ld8_stream_ef(a.theta + e0 + 256 * k) : ld8_stream(a.theta + e0 + 256 * k);
      an[k] = kEvictFirst ? ld8_stream_ef(a.anchor + e0 + 256 * k) : ld8_stream(a.anchor + e0 + 256 * k);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) d[k].v[i] = __fsub_rn(an[k].v[i], th[k].v[i]);  // Alg. 2 L7
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int64_t e = e0 + 256 * k + i;
        d[k].v[i] = (e < a.n) ? __fsub_rn(a.anchor[e], a.theta[e]) : 0.0f;
      }
  }
}

__device__ __forceinline__ uint32_t row_max_bits(const f8& r) {
  uint32_t m = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) m = max(m, abs_bits(r.v[i]));
  return m;
}

// Index of the first non-finite Delta of the chunk -> atomicMin into the trailer.
__device__ __forceinline__ void record_first_bad(const QArgs& a, int64_t c, int lane, const f8 (&d)[4]) {
  uint32_t best = 0xffffffffu;
#pragma unroll
  for (int k = 3; k >= 0; --k)
#pragma unroll
    for (int i = 7; i >= 0; --i)
      if (abs_bits(d[k].v[i]) >= kInfBits) best = (uint32_t)(256 * k + 8 * lane + i);
  best = __reduce_min_sync(kFull, best);
  if (lane == 0 && best != 0xffffffffu)
    atomicMin(reinterpret_cast<unsigned long long*>(a.slot + a.trailer_off + 8),
              (unsigned long long)(c * 1024 + best));
}

// Stores one row's 8 codes (element 8*lane + i -> nibble i) as a word;
// the ragged last chunk only writes words inside the codes region (those
// past n hold zero codes = the zero padding up to the scales).
__device__ __forceinline__ void store_row_codes(const QArgs& a, int64_t c, int k, int lane, uint32_t w,
                                                bool guard) {
  const int64_t word = (c * 1024 + 256 * k + 8 * lane) >> 3;
  if (!guard || 4 * (size_t)word < a.scales_off) {
    reinterpret_cast<uint32_t*>(a.slot)[word] = w;
    if (a.push) push_u32(a, 4 * (size_t)word, w);
  }
}

// Encodes the 4 rows of a chunk; s[q] = scale of block q of the chunk
// (row k belongs to block k / (4 / NB)).
template <int NB, bool kFullChunk>
__device__ __forceinline__ void encode_chunk_rows(const QArgs& a, int64_t c, int lane, const f8 (&d)[4],
                                                  const float (&s)[NB]) {
  float sl = s[0];
#pragma unroll
  for (int q = 1; q < NB; ++q) sl = (lane == q) ? s[q] : sl;
  const float t0_l = (lane < NB) ? e3m0_threshold(sl, 0) : 0.0f;  // T_0 of block `lane`
  float t0[NB];
  bool all_fast = true;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    t0[q] = __shfl_sync(kFull, t0_l, q);
    all_fast &= fast_ok(s[q], t0[q]);
  }
  if (all_fast) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t c0 = __float_as_uint(t0[k / (4 / NB)]) + 0x7fffffu;
      uint32_t w = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) w |= encode_fast(d[k].v[i], c0) << (4 * i);
      store_row_codes(a, c, k, lane, w, !kFullChunk);
    }
  } else {  // tiny, zero or non-finite scale somewhere in the chunk: explicit thresholds
    float tl = CUDART_INF_F;
    {
      const int q = lane >> 3, j = lane & 7;
      float sq = s[0];
#pragma unroll
      for (int r = 1; r < NB; ++r) sq = (q == r) ? s[r] : sq;
      if (q < NB && j < 7) tl = e3m0_threshold(sq, j);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int q = k / (4 / NB);
      float T[7];
#pragma unroll
      for (int j = 0; j < 7; ++j) T[j] = __shfl_sync(kFull, tl, q * 8 + j);
      uint32_t w = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) w |= encode_slow(d[k].v[i], T) << (4 * i);
      store_row_codes(a, c, k, lane, w, !kFullChunk);
    }
  }
}

// Writes the payload bytes after the scales: zero pad, trailer magic + nb,
// zero pad to the payload end (first_bad is left to the memset + atomics).
__device__ void write_tail(const QArgs& a) {
  const size_t lo = a.scales_off + 4 * (size_t)a.nb;
  for (size_t o = lo + threadIdx.x; o < a.bytes; o += blockDim.x) {
    if (o >= a.trailer_off && o < a.trailer_off + 16) continue;
    a.slot[o] = 0;
    if (a.push) push_u8(a, o, 0);
  }
  if (threadIdx.x == 0) {
    *reinterpret_cast<uint32_t*>(a.slot + a.trailer_off) = kMagic;
    *reinterpret_cast<uint32_t*>(a.slot + a.trailer_off + 4) = (uint32_t)a.nb;
    if (a.push) {
      push_u32(a, a.trailer_off, kMagic);
      push_u32(a, a.trailer_off + 4, (uint32_t)a.nb);
    }
  }
}

// ---------------------------------------------------------------------------
// k_quantize: single pass, B in {256, 512, 1024} (NB = 1024 / B blocks per
// warp chunk).  One warp per 1024-element chunk, grid-stride over chunks.
// ---------------------------------------------------------------------------
// Block maxima, poison check, codes and scales of a chunk whose Deltas are in d.
template <int NB, bool kFullChunk>
__device__ __forceinline__ void encode_block_rows(const QArgs& a, int64_t c, int lane, const f8 (&d)[4]) {
  constexpr int KB = 4 / NB;  // rows per scale block
  float s[NB];
  bool bad = false;
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    uint32_t m = 0;
#pragma unroll
    for (int k = q * KB; k < (q + 1) * KB; ++k) m = max(m, row_max_bits(d[k]));
    m = __reduce_max_sync(kFull, m);  // exact max |Delta| of the block (as bits)
    bad |= m >= kInfBits;
    s[q] = __uint_as_float(m);
  }
  if (bad) record_first_bad(a, c, lane, d);
  encode_chunk_rows<NB, kFullChunk>(a, c, lane, d, s);
  if (lane < NB) {
    const int64_t blk = c * NB + lane;
    float sv = s[0];
#pragma unroll
    for (int q = 1; q < NB; ++q) sv = (lane == q) ? s[q] : sv;
    if (blk < a.nb) {
      reinterpret_cast<float*>(a.slot + a.scales_off)[blk] = sv;
      if (a.push) push_u32(a, a.scales_off + 4 * (size_t)blk, __float_as_uint(sv));
    }
  }
}

template <int NB, bool kFullChunk>
__device__ __forceinline__ void quantize_chunk(const QArgs& a, int64_t c, int lane) {
  f8 d[4];
  load_chunk<kFullChunk>(a, c, lane, d);
  encode_block_rows<NB, kFullChunk>(a, c, lane, d);
}

template <int NB>
// 3 resident CTAs per SM (<= 85 registers, no spills): 24 warps with 8 KB of
// loads in flight each; measured 211 vs 222 us per 1B fragment at 2 CTAs/SM.
__global__ void __launch_bounds__(kThreads, 3) k_quantize(QArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nfull = a.n >> 10;
  for (int64_t c = warp; c < nfull; c += nwarps) quantize_chunk<NB, true>(a, c, lane);
  if ((nfull << 10) < a.n && warp == nfull % nwarps) quantize_chunk<NB, false>(a, nfull, lane);
  if (blockIdx.x == 0) write_tail(a);
  if (a.sig) signal_round(a);
}

// ---------------------------------------------------------------------------
// Two-pass variant: B = 0 (whole fragment) or B a power of two >= 2048.
// Pass 1: per-block max |Delta| by atomicMax on the bit patterns (valid for
// non-negative floats; NaN/inf sort above every finite value).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t block_of_chunk(const QArgs& a, int64_t c) {
  return a.lgB < 0 ? 0 : ((c << 10) >> a.lgB);
}

// Staged two-pass: pass 1 keeps, per element, a 16-bit
// summary of |Delta| relative to its row's max m_r (256 elements):
//   base = bits(2^(exp(m_r) - 7)) (0 if that is subnormal),
//   o = clamp(bits|Delta| - base, 0, 2^26 - 1), summary = (o >> 11) | sign << 15,
// i.e. |Delta|'s bit pattern to within a bucket of 2^11 ulps (12 mantissa
// bits) over the 8 octaves below m_r.  Any scale s >= m_r puts T_6(s) >=
// m_r 2^-6.5 above the bucket of everything below base, so those code 0.
// Pass 2 evaluates the (monotone) fast-path code at both ends of the bucket;
// if they agree that is the code, else (about 1 element in 4000) it re-reads
// theta and A for that element and encodes it exactly.
__device__ __forceinline__ uint32_t stage_base(uint32_t mbits) {
  const uint32_t E = mbits & kInfBits;
  return E >= (7u << 23) ? E - (7u << 23) : 0u;
}
__device__ __forceinline__ uint32_t stage16(float d, uint32_t base) {
  const uint32_t b = abs_bits(d);
  const uint32_t o = b > base ? min(b - base, 0x3ffffffu) : 0u;
  return (o >> 11) | ((__float_as_uint(d) >> 16) & 0x8000u);
}
__device__ __forceinline__ void stage_row(const QArgs& a, int64_t c, int k, int lane, const float* d, uint32_t mbits) {
  const uint32_t base = stage_base(mbits);
  uint32_t w[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) w[i] = stage16(d[2 * i], base) | (stage16(d[2 * i + 1], base) << 16);
  if (c >= a.stg_keep_from) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(a.stg + c * 512 + 128 * k + 4 * lane),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "l"(pol)
                 : "memory");
  } else {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(a.stg + c * 512 + 128 * k + 4 * lane), "r"(w[0]),
                 "r"(w[1]), "r"(w[2]), "r"(w[3])
                 : "memory");
  }
}

template <bool kFullChunk, bool kStage, bool kEF>
__device__ __forceinline__ void absmax_chunk(const QArgs& a, int64_t c, int lane, int64_t& cur, uint32_t& run) {
  f8 d[4];
  load_chunk<kFullChunk, kEF>(a, c, lane, d);
  uint32_t m = 0;
  if (kStage) {
    uint32_t mr[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      mr[k] = __reduce_max_sync(kFull, row_max_bits(d[k]));
      m = max(m, mr[k]);
      stage_row(a, c, k, lane, d[k].v, mr[k]);
    }
    if (lane == 0)
      asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(a.stg_max + 4 * c), "r"(mr[0]), "r"(mr[1]),
                   "r"(mr[2]), "r"(mr[3])
                   : "memory");
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) m = max(m, row_max_bits(d[k]));
    m = __reduce_max_sync(kFull, m);
  }
  if (m >= kInfBits) record_first_bad(a, c, lane, d);
  const int64_t blk = block_of_chunk(a, c);
  if (blk != cur) {
    if (cur >= 0 && lane == 0) atomicMax(reinterpret_cast<unsigned int*>(a.slot + a.scales_off) + cur, run);
    cur = blk;
    run = 0;
  }
  run = max(run, m);
}

__device__ __forceinline__ void flush_block_max(const QArgs& a, int lane, int64_t cur, uint32_t run);

// staged: 3 CTAs/SM (<= 85 registers) as k_quantize
template <bool kStage, bool kEF>
__global__ void __launch_bounds__(kThreads, kStage ? 3 : 1) k_absmax(QArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nfull = a.n >> 10;
  int64_t cur = -1;
  uint32_t run = 0;
  for (int64_t c = warp; c < nfull; c += nwarps) absmax_chunk<true, kStage, kEF>(a, c, lane, cur, run);
  if ((nfull << 10) < a.n && warp == nfull % nwarps) absmax_chunk<false, kStage, kEF>(a, nfull, lane, cur, run);
  flush_block_max(a, lane, cur, run);
}

// Merges the CTA's warps that ended in the same block: one atomic per distinct
// block per CTA (B = 0: one per CTA instead of one per warp).
__device__ __forceinline__ void flush_block_max(const QArgs& a, int lane, int64_t cur, uint32_t run) {
  __shared__ int64_t s_blk[kThreads / 32];
  __shared__ uint32_t s_run[kThreads / 32];
  if (lane == 0) {
    s_blk[threadIdx.x >> 5] = cur;
    s_run[threadIdx.x >> 5] = run;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t b = -1;
    uint32_t r = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      if (s_blk[w] < 0) continue;
      if (s_blk[w] != b) {
        if (b >= 0) atomicMax(reinterpret_cast<unsigned int*>(a.slot + a.scales_off) + b, r);
        b = s_blk[w];
        r = 0;
      }
      r = max(r, s_run[w]);
    }
    if (b >= 0) atomicMax(reinterpret_cast<unsigned int*>(a.slot + a.scales_off) + b, r);
  }
}

template <bool kFullChunk>
__device__ __forceinline__ void encode_chunk(const QArgs& a, int64_t c, int lane) {
  f8 d[4];
  load_chunk<kFullChunk>(a, c, lane, d);
  const float s[1] = {reinterpret_cast<const float*>(a.slot + a.scales_off)[block_of_chunk(a, c)]};
  encode_chunk_rows<1, kFullChunk>(a, c, lane, d, s);
}

// Pass 2 from the staged summaries (fast path only: the block's thresholds
// T_j = T_0 / 2^j are normal; zero and non-finite scales give all-zero codes,
// as e3m0_threshold's +inf thresholds do).  In bucket units of a row
// (u = (bits|Delta| - base) / 2^11, summary u = floor of it): a_0 = bits(T_0)
// - base = 2^11 q_0 + r_0 and a_j = a_0 - j 2^23, so the bucket lies at or
// above T_j iff u >= q_0 + (r_0 != 0) - 4096 j, i.e. with
// D = q_0 + (r_0 != 0) + 4095 and K = 32767 - D the code magnitude is
//   e = max(floor((u + K) / 4096), 0)      (<= 7: u <= D since |Delta| <= s < 2 T_0),
// and the bucket straddles a threshold iff r_0 != 0 and u == q_0 (mod 4096)
// -- those elements re-read theta and A and encode exactly.  Everything
// below base was stored as u = 0, whose e is 0 (a_0 >= 6.41 octaves).
// SIMD form per 32-bit word (two summaries): v = (word & 0x7fff7fff) +
// (K + 2^15) per half (K clamped to >= -2^15, so each half stays in
// [0, 2^16): no carry between halves); the high nibble of each half is
// n = e_raw + 8, i.e. e > 0 iff n >= 9, and then the code is (n & 7) | sign << 3.
// Straddling (r_0 != 0): u - q_0 == 0 (mod 4096) iff the low 12 bits of the
// half of v are all ones (q_0 + K + 2^15 == -1 mod 4096), i.e. iff adding 1
// carries into bit 12.  The 8 high nibbles and 8 sign bits of a lane's row
// are gathered with PRMT into the row's code word (nibble i = element i).
__device__ __forceinline__ uint32_t gather_hi_nibbles(const uint32_t (&v)[4]) {
  const uint32_t A = __byte_perm(__byte_perm(v[0], v[1], 0x0051), __byte_perm(v[2], v[3], 0x0051), 0x5410);  // bytes 1
  const uint32_t B = __byte_perm(__byte_perm(v[0], v[1], 0x0073), __byte_perm(v[2], v[3], 0x0073), 0x5410);  // bytes 3
  return ((A >> 4) & 0x0f0f0f0fu) | (B & 0xf0f0f0f0u);  // nibble 2k: low half of word k, 2k+1: high half
}

// The code word of one row of one lane; *straddle = some element needs the exact re-read.
// Row parameters (depend on the row max and T_0 only): Kpair = (K + 2^15)
// in both halves, rho = (r_0 != 0).
__device__ __forceinline__ uint32_t staged_row_kpair(uint32_t t0bits, uint32_t row_max, uint32_t* rho) {
  const uint32_t a0 = t0bits - stage_base(row_max);
  *rho = (a0 & 2047u) != 0u ? 1u : 0u;
  const int K = max(32767 - (int)((a0 >> 11) + *rho + 4095u), -32768);
  return (uint32_t)(K + 32768) * 0x10001u;
}

__device__ __forceinline__ uint32_t staged_row_codes(uint32_t Kpair, bool rho, const uint4& qv, bool* straddle) {
  const uint32_t qw[4] = {qv.x, qv.y, qv.z, qv.w};
  uint32_t v[4], acc = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[i] = (qw[i] & 0x7fff7fffu) + Kpair;
    acc |= v[i] ^ (v[i] + 0x00010001u);  // bit 12 / 28 flips iff the half's low 12 bits are all ones
  }
  *straddle = rho && (acc & 0x10001000u);
  const uint32_t n = gather_hi_nibbles(v);
  const uint32_t sg = gather_hi_nibbles(qw) & 0x88888888u;                        // sign -> bit 3 of each nibble
  const uint32_t keep3 = ((n & 0x77777777u) + 0x77777777u) & n & 0x88888888u;  // bit 3 set iff n >= 9
  const uint32_t M = keep3 | (keep3 - (keep3 >> 3));                          // 0xF per kept nibble
  return (n ^ sg ^ 0x88888888u) & M;                                            // (n & 7) | sign << 3
}


// Pass 2 without a workspace: re-reads theta and A (k_encode), last chunk
// first (pass 1 streamed the fragment forward, so its tail is what the L2
// still holds).
__global__ void __launch_bounds__(kThreads, 3) k_encode(QArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nfull = a.n >> 10;
  const int64_t nchunks = nfull + ((nfull << 10) < a.n ? 1 : 0);
  for (int64_t k = warp; k < nchunks; k += nwarps) {
    const int64_t c = nchunks - 1 - k;
    if (c < nfull) encode_chunk<true>(a, c, lane);
    else encode_chunk<false>(a, c, lane);
  }
  if (blockIdx.x == 0) write_tail(a);
  if (a.sig) signal_round(a);
}

// T_0(s) = smallest binary32 c with c^2 >= s^2 / 2 (e3m0_threshold(s, 0)),
// for a normal s >= 2^-100 (the fast path's range): fl(s * fl(1/sqrt 2)) is
// within 2 ulps of it, then exact binary64 checks step to it.  Inline, so
// every lane of a warp computes it without a call or a shuffle.
__device__ __forceinline__ float e3m0_t0_normal(float s) {
  const double b = __dmul_rn(__dmul_rn((double)s, (double)s), 0.5);  // exact
  float c = __fmul_rn(s, 0.70710678f);
#pragma unroll 1
  while (__dmul_rn((double)c, (double)c) < b) c = __uint_as_float(__float_as_uint(c) + 1u);
#pragma unroll 1
  for (;;) {
    const float pc = __uint_as_float(__float_as_uint(c) - 1u);
    if (__dmul_rn((double)pc, (double)pc) >= b) c = pc; else break;
  }
  return c;
}

// Pass 2 from the summaries (k_encode_staged): one CTA per tile of
// 8 kStagedCpw chunks, tiles walked last to first (pass 1 streamed the
// fragment forward, so its tail is what the L2 still holds).  Each warp
// issues the loads of all its chunks' summaries (2 KB + 16 B each) before it
// encodes any, and the code is kept small (the straddle fix-up and the
// re-reading fallback are off the straight path): a persistent 2-CTA/SM form with a 3-deep
// software pipeline ran at 1.8 TB/s, stalled on instruction fetch
// (profiles/r2_b0_staged.txt).  Codes are stored locally (the two-pass paths
// push the finished slot separately).
__device__ __forceinline__ void encode_chunk_call(const QArgs& a, int64_t c, int lane, bool full) {
  if (full) encode_chunk<true>(a, c, lane);
  else encode_chunk<false>(a, c, lane);
}

struct Staged {
  uint4 mr;
  uint4 q[4];
};

__device__ __forceinline__ void load_staged(const QArgs& a, int64_t c, int lane, Staged& st) {
  st.mr = __ldg(reinterpret_cast<const uint4*>(a.stg_max + 4 * c));
  const uint4* p = reinterpret_cast<const uint4*>(a.stg + c * 512 + 4 * lane);
#pragma unroll
  for (int k = 0; k < 4; ++k) st.q[k] = __ldg(p + 32 * k);
}

// The fast path of one chunk (s, t0b: its block scale and bits(T_0(s)), t0b
// = 0 off the fast path).  Stores the codes read off the summaries and
// returns the work left for after the chunk loop, so that nothing is live
// across it: bit k = row k of this lane straddles a threshold (re-encode it
// exactly), bit 4 = the block's thresholds are below the normal range
// (re-read the chunk, explicit compares).
__device__ __forceinline__ uint32_t encode_staged(const QArgs& a, int64_t c, int lane, float s, uint32_t t0b,
                                                  const Staged& st, int64_t nfull) {
  uint32_t todo = 0u;
  if (t0b) {
    // the 4 rows' parameters: lane k (mod 4) computes row k's, then broadcast
    const int r = lane & 3;
    const uint32_t mrl = r == 0 ? st.mr.x : r == 1 ? st.mr.y : r == 2 ? st.mr.z : st.mr.w;
    uint32_t rho;
    const uint32_t kp = staged_row_kpair(t0b, mrl, &rho);
    const uint32_t rhos = __ballot_sync(kFull, rho != 0u);  // bit k: row k
    uint32_t* wp = reinterpret_cast<uint32_t*>(a.slot) + (c * 128 + lane);  // row k's word: wp + 32 k
    const bool full = c < nfull;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      bool straddle;
      const uint32_t w = staged_row_codes(__shfl_sync(kFull, kp, k), (rhos >> k) & 1u, st.q[k], &straddle);
      todo |= straddle ? 1u << k : 0u;
      if (full) st_global_u32(wp + 32 * k, w);
      else store_row_codes(a, c, k, lane, w, true);
    }
  } else if (!(s > 0.0f) || !(s <= FLT_MAX)) {  // zero or non-finite scale: every code 0
#pragma unroll
    for (int k = 0; k < 4; ++k) store_row_codes(a, c, k, lane, 0u, c >= nfull);
  } else {
    todo = 16u;
  }
  if (a.stg_hints & 2) {  // the chunk's 2 KB of summaries are dead: drop them from L2 without a write-back
    __syncwarp();
    if (lane < 16) asm volatile("discard.global.L2 [%0], 128;" ::"l"(a.stg + c * 512 + 32 * lane) : "memory");
  }
  return todo;
}

// Exact codes of one row of 8 elements from theta and A (the fast-path
// encode is exact given Delta), overwriting the word pass 2 stored.
__device__ __forceinline__ void fix_row(const QArgs& a, int64_t r, uint32_t t0b) {
  const int64_t e0 = 8 * r;
  uint32_t w = 0u;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t idx = e0 + i;
    const uint32_t code = idx < a.n ? encode_fast(__fsub_rn(a.anchor[idx], a.theta[idx]), t0b + 0x7fffffu) : 0u;
    w |= code << (4 * i);
  }
  if (4 * (size_t)r < a.scales_off) reinterpret_cast<uint32_t*>(a.slot)[r] = w;  // past n: padding words hold 0
}

// After the chunk loop (nothing else live): bit 4 (warp-uniform) re-reads
// the whole chunk; the straddling rows (bits 0-3 of each lane) are
// re-encoded in place.  (Deferring them to a fix-up kernel through a list
// measured the same: the kernel's 6-8 us ate what pass 2 saved.)
__device__ __forceinline__ void finish_staged(const QArgs& a, int64_t c, int lane, uint32_t t0b, uint32_t todo,
                                              int64_t nfull) {
  if (__any_sync(kFull, todo & 16u)) {
    encode_chunk_call(a, c, lane, c < nfull);
    return;
  }
#pragma unroll 1
  for (int k = 0; k < 4; ++k)
    if ((todo >> k) & 1u) fix_row(a, (c * 1024 + 256 * k + 8 * lane) >> 3, t0b);
}

// The chunk's block scale s and bits(T_0(s)) for the fast path: normal
// s >= 2^-100 (T_0 inline, e3m0_t0_normal; its T_6 is then normal); any other
// s gets t0b = 0 and encode_staged's other branches.  Cached per block.
__device__ __forceinline__ void staged_scale(const QArgs& a, int64_t c, int64_t& blk, float& s, uint32_t& t0b) {
  const int64_t b = block_of_chunk(a, c);
  if (b == blk) return;
  blk = b;
  s = reinterpret_cast<const float*>(a.slot + a.scales_off)[b];
  uint32_t t = 0u;
  if (s >= 0x1p-100f && s <= FLT_MAX) {
    const float t0 = e3m0_t0_normal(s);
    t = fast_ok(s, t0) ? __float_as_uint(t0) : 0u;
  }
  t0b = t;
}

// kStagedCpw chunks per warp, 4 resident CTAs per SM (<= 64 registers; measured against 1 chunk at 6
// CTAs/SM, 4 at 2, a TMA-staged tile and a persistent grid: profiles/r2_b0_staged.txt)
constexpr int kStagedCpw = 2;

__global__ void __launch_bounds__(kThreads, 4) k_encode_staged(QArgs a) {
  const int lane = threadIdx.x & 31;
  constexpr int kWpb = kThreads / 32;
  const int64_t nfull = a.n >> 10;
  const int64_t nchunks = nfull + ((nfull << 10) < a.n ? 1 : 0);
  // tile b = chunks [top - 8 kStagedCpw, top), top = nchunks - b * 8 kStagedCpw; chunk j of warp w: top - 1 - w - 8 j
  const int64_t top = nchunks - (int64_t)blockIdx.x * (kWpb * kStagedCpw) - 1 - (threadIdx.x >> 5);
  // every load first, then per chunk its block's T_0 (inline, cached per block) and the codes,
  // then the rare exact re-encodes (nothing else live)
  Staged x[kStagedCpw];
#pragma unroll
  for (int j = 0; j < kStagedCpw; ++j)
    if (top - kWpb * j >= 0) load_staged(a, top - kWpb * j, lane, x[j]);
  int64_t blk = -1;
  float s = 0.0f;
  uint32_t t0b = 0u, t0s[kStagedCpw], todo[kStagedCpw];
#pragma unroll
  for (int j = 0; j < kStagedCpw; ++j) {
    const int64_t c = top - kWpb * j;
    todo[j] = 0u;
    t0s[j] = 0u;
    if (c < 0) continue;
    staged_scale(a, c, blk, s, t0b);
    t0s[j] = t0b;
    todo[j] = encode_staged(a, c, lane, s, t0b, x[j], nfull);
  }
#pragma unroll
  for (int j = 0; j < kStagedCpw; ++j)
    if (__any_sync(kFull, todo[j] != 0u)) finish_staged(a, top - kWpb * j, lane, t0s[j], todo[j], nfull);
  if (blockIdx.x == 0) write_tail(a);
  if (a.sig) signal_round(a);
}

// ---------------------------------------------------------------------------
// Fused all-gather protocol (push and pull modes).
// k_push_copy: the two-pass quantize paths push the finished local slot
//   (scales written by atomics) to every peer, then signal the round.
// k_round_wait: the block-receive (Alg. 2 L11).  One CTA decides the round
//   once -- every peer's flag entry holds the round id (acquire, system
//   scope), or, with a timeout configured (SD_WAIT_TIMEOUT_MS), a peer missed
//   it -- and writes the verdict {first_bad, code} that the apply's CTAs read
//   as plain stream-ordered data.  (Waiting in every apply CTA instead was
//   measured slower: a system-scope acquire per CTA cost the apply 5% in push
//   and 18% in pull mode at N = 2, profiles/r2_fused_wait_ab.txt.)
// Verdict codes (also status[1]): 0 apply, 1 non-finite Delta somewhere,
// 2 malformed own payload, 3 a peer missed the block-receive deadline (or
// this context already had a timeout: sticky, status[2] = 1).
// ---------------------------------------------------------------------------
// k_signal: the round signal as its own one-thread kernel after the payload
// kernel (push mode; see signal_kernel()): same stores as signal_round's last
// CTA, ordered by the kernel boundary instead of the ticket counter.
__global__ void k_signal(QArgs a) {
  if (threadIdx.x != 0) return;
  const unsigned long long fb = *reinterpret_cast<volatile unsigned long long*>(a.slot + a.trailer_off + 8);
  if (a.push)
    for (int q = 0; q < a.M; ++q)
      if (q != a.rank)
        *reinterpret_cast<unsigned long long*>(ncclGetLsaPointer(a.win, a.win_off + a.trailer_off + 8, q)) = fb;
  __threadfence_system();
  for (int q = 0; q < a.M; ++q) {
    if (q == a.rank) continue;
    unsigned long long* e =
        reinterpret_cast<unsigned long long*>(ncclGetLsaPointer(a.win, a.flags_off + 16 * (size_t)a.rank, q));
    e[1] = fb;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(e), "l"(a.seq) : "memory");
  }
}

constexpr unsigned long long kPeerTimedOut = 0xFFFFFFFFFFFFFFFEull;  // first_bad value a timed-out rank publishes

__global__ void __launch_bounds__(kThreads) k_push_copy(QArgs a) {
  const size_t n16 = a.bytes / 16;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(a.slot)[i];
    for (int q = 0; q < a.M; ++q)
      if (q != a.rank) *reinterpret_cast<uint4*>(ncclGetLsaPointer(a.win, a.win_off + 16 * i, q)) = v;
  }
  if (a.sig) signal_round(a);
}

struct WArgs {
  const unsigned long long* flags;  // this half's flag entries {round id, first_bad} x M (local)
  const uint8_t* own;               // this rank's own slot (local)
  size_t trailer_off;
  unsigned long long* verdict;      // {first_bad, code} (local)
  int M, rank;
  unsigned long long seq, timeout_ns;
  volatile unsigned long long* status;  // host-mapped {first_bad, code, dead}
  ncclWindow_t win;
  size_t flags_off;                 // window offset of this half's flag array
  int pull;                         // pull mode: check the slot addressing of the apply
  size_t half_off, pb;
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// The own slot's trailer: its magic and first non-finite index (written by this
// rank's own quantize earlier in stream order).
__device__ __forceinline__ unsigned long long own_trailer_fb(const uint8_t* own, size_t trailer_off, int* bad) {
  if (*reinterpret_cast<const uint32_t*>(own + trailer_off) != kMagic) *bad = 1;
  return *reinterpret_cast<const unsigned long long*>(own + trailer_off + 8);
}

__global__ void k_round_wait(WArgs w) {
  __shared__ unsigned long long s_fb;
  __shared__ int s_code;
  if (threadIdx.x == 0) {
    s_fb = ~0ull;
    s_code = w.status[2] ? 3 : 0;  // sticky: an earlier timeout on this context
  }
  __syncthreads();
  const int q = threadIdx.x;
  if (q < w.M && s_code != 3) {
    unsigned long long fb;
    int code = 0;
    if (w.pull && w.M > 1) {  // the apply addresses slot m as LSA(half, 0) + m (LSA stride + pb): check it
      const uint8_t* b0 = static_cast<const uint8_t*>(ncclGetLsaPointer(w.win, w.half_off, 0));
      const uint8_t* b1 = static_cast<const uint8_t*>(ncclGetLsaPointer(w.win, w.half_off, 1));
      const uint8_t* bq = static_cast<const uint8_t*>(ncclGetLsaPointer(w.win, w.half_off + (size_t)q * w.pb, q));
      if (bq != b0 + (size_t)q * ((size_t)(b1 - b0) + w.pb)) atomicMax(&s_code, 2);
    }
    if (q == w.rank) {
      int bad = 0;
      fb = own_trailer_fb(w.own, w.trailer_off, &bad);
      if (bad) code = 2;
    } else {
      const unsigned long long t0 = globaltimer_ns();
      bool ok = false;
      while (true) {
        if (ld_acquire_sys(w.flags + 2 * q) == w.seq) {
          ok = true;
          break;
        }
        if (w.timeout_ns && globaltimer_ns() - t0 > w.timeout_ns) break;
        __nanosleep(128);
      }
      fb = ok ? w.flags[2 * q + 1] : ~0ull;
      if (!ok || fb == kPeerTimedOut) code = 3;
    }
    if (code == 3 || fb == kPeerTimedOut) atomicMax(&s_code, 3);
    else if (code) atomicMax(&s_code, code);
    if (fb != kPeerTimedOut) atomicMin(&s_fb, fb);
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int code = s_code;
  if (code == 0 && s_fb != ~0ull) code = 1;
  w.verdict[0] = s_fb;
  w.verdict[1] = (unsigned long long)code;
  if (code == 0) return;
  w.status[0] = s_fb;
  w.status[1] = (unsigned long long)code;
  if (code == 3 && !w.status[2]) {
    // first timeout on this context: sticky from now on, and tell the peers
    // (best effort) so that a peer that has not yet passed its own wait for
    // this round skips it too
    w.status[2] = 1ull;
    __threadfence_system();
    for (int p = 0; p < w.M; ++p) {
      if (p == w.rank) continue;
      unsigned long long* e =
          reinterpret_cast<unsigned long long*>(ncclGetLsaPointer(w.win, w.flags_off + 16 * (size_t)w.rank, p));
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(e + 1), "l"(kPeerTimedOut) : "memory");
    }
  }
}

// ---------------------------------------------------------------------------
// InnerOpt = AdamW (NEXT-1; Alg. 2 L5), with
// the op order of the oracle's or_adamw (DESIGN.md AMB-20):
//   m = b1 m + (1-b1) g ; v = b2 v + (1-b2) g^2
//   theta = theta (1 - lr wd) - (lr/bc1) (m / (sqrt(v)/sqrt(bc2) + eps))
// k_adamw: one thread per 8 elements (256-bit accesses).  k_adamw_quantize:
// the inner step that precedes a send, fused with Alg. 2 L7 + E3M0 -- the
// updated theta stays in registers, so the quantize costs 4.5 B/param of
// extra traffic (A read + codes) instead of 8.5.
// ---------------------------------------------------------------------------
struct AdamArgs {
  float* theta;
  const float* grad;
  float* m;
  float* v;
  int64_t n;
  float b1, b2, c1, c2, decay, step, sbc2, eps;
};

__device__ __forceinline__ void adamw_one(float& th, float g, float& m, float& v, const AdamArgs& h) {
  m = __fadd_rn(__fmul_rn(h.b1, m), __fmul_rn(h.c1, g));
  v = __fadd_rn(__fmul_rn(h.b2, v), __fmul_rn(h.c2, __fmul_rn(g, g)));
  const float denom = __fadd_rn(__fdiv_rn(__fsqrt_rn(v), h.sbc2), h.eps);
  th = __fsub_rn(__fmul_rn(th, h.decay), __fmul_rn(h.step, __fdiv_rn(m, denom)));
}

__global__ void __launch_bounds__(kThreads) k_adamw(AdamArgs h) {
  const int64_t n8 = h.n >> 3;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += nthr) {
    f8 t = ld8(h.theta + 8 * i), g = ld8_stream(h.grad + 8 * i), m = ld8(h.m + 8 * i), v = ld8(h.v + 8 * i);
#pragma unroll
    for (int j = 0; j < 8; ++j) adamw_one(t.v[j], g.v[j], m.v[j], v.v[j], h);
    st8(h.theta + 8 * i, t);
    st8(h.m + 8 * i, m);
    st8(h.v + 8 * i, v);
  }
  if (blockIdx.x == 0 && threadIdx.x < (h.n & 7)) {
    const int64_t e = (n8 << 3) + threadIdx.x;
    float t = h.theta[e], m = h.m[e], v = h.v[e];
    adamw_one(t, h.grad[e], m, v, h);
    h.theta[e] = t;
    h.m[e] = m;
    h.v[e] = v;
  }
}

// AdamW on the chunk's 4 rows, write back theta, m, v; d = A - theta'.
template <bool kFullChunk>
__device__ __forceinline__ void adamw_chunk(const QArgs& a, const AdamArgs& h, int64_t c, int lane, f8 (&d)[4]) {
  const int64_t e0 = c * 1024 + 8 * lane;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t e = e0 + 256 * k;
    if (kFullChunk) {
      f8 t = ld8(h.theta + e), g = ld8_stream(h.grad + e), m = ld8(h.m + e), v = ld8(h.v + e);
      const f8 an = ld8_stream(a.anchor + e);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        adamw_one(t.v[j], g.v[j], m.v[j], v.v[j], h);
        d[k].v[j] = __fsub_rn(an.v[j], t.v[j]);  // Alg. 2 L7 on the updated theta
      }
      st8(h.theta + e, t);
      st8(h.m + e, m);
      st8(h.v + e, v);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        d[k].v[j] = 0.0f;
        if (e + j < a.n) {
          float t = h.theta[e + j], m = h.m[e + j], v = h.v[e + j];
          adamw_one(t, h.grad[e + j], m, v, h);
          h.theta[e + j] = t;
          h.m[e + j] = m;
          h.v[e + j] = v;
          d[k].v[j] = __fsub_rn(a.anchor[e + j], t);
        }
      }
    }
  }
}

// 3 CTAs/SM (<= 85 registers; ptxas spills ~50 B): 0.770 vs 0.792 ms per 1B fragment at
// 2 CTAs/SM and 124 registers (profiles/r2_kernel_ab.txt)
template <int NB>
__global__ void __launch_bounds__(kThreads, 3) k_adamw_quantize(QArgs a, AdamArgs h) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nfull = a.n >> 10;
  for (int64_t c = warp; c < nfull; c += nwarps) {
    f8 d[4];
    adamw_chunk<true>(a, h, c, lane, d);
    encode_block_rows<NB, true>(a, c, lane, d);
  }
  if ((nfull << 10) < a.n && warp == nfull % nwarps) {
    f8 d[4];
    adamw_chunk<false>(a, h, nfull, lane, d);
    encode_block_rows<NB, false>(a, nfull, lane, d);
  }
  if (blockIdx.x == 0) write_tail(a);
  if (a.sig) signal_round(a);
}

// AdamW on a chunk fused with the first pass of the two-pass quantize (B = 0,
// SPEC.md:266, or B > 1024): the updated theta is written and its Delta's
// block max accumulated in the same pass, so the inner step before a send
// costs 32 + 8.5 B/param (k_encode re-reads theta and A) instead of
// 28 + 16.5 with a separate absmax pass.
template <bool kFullChunk, bool kStage, bool kEF>
__device__ __forceinline__ void adamw_absmax_chunk(const QArgs& a, const AdamArgs& h, int64_t c, int lane,
                                                   int64_t& cur, uint32_t& run) {
  // row by row (no Delta kept past its row): the block max and the first
  // non-finite index only need a running max and a running min
  const int64_t e0 = c * 1024 + 8 * lane;
  uint32_t mx = 0, bad = 0xffffffffu;
#pragma unroll 1
  for (int k = 0; k < 4; ++k) {
    const int64_t e = e0 + 256 * k;
    float d[8];
    if (kFullChunk) {
      f8 t = ld8(h.theta + e), g = kEF ? ld8_stream_ef(h.grad + e) : ld8_stream(h.grad + e), m = ld8(h.m + e),
         v = ld8(h.v + e);
      const f8 an = kEF ? ld8_stream_ef(a.anchor + e) : ld8_stream(a.anchor + e);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        adamw_one(t.v[j], g.v[j], m.v[j], v.v[j], h);
        d[j] = __fsub_rn(an.v[j], t.v[j]);  // Alg. 2 L7 on the updated theta
      }
      st8(h.theta + e, t);
      st8(h.m + e, m);
      st8(h.v + e, v);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        d[j] = 0.0f;
        if (e + j < a.n) {
          float t = h.theta[e + j], m = h.m[e + j], v = h.v[e + j];
          adamw_one(t, h.grad[e + j], m, v, h);
          h.theta[e + j] = t;
          h.m[e + j] = m;
          h.v[e + j] = v;
          d[j] = __fsub_rn(a.anchor[e + j], t);
        }
      }
    }
    uint32_t rm = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {  // rows ascending, then j ascending: the lane's first bad index
      const uint32_t ab = abs_bits(d[j]);
      rm = max(rm, ab);
      if (ab >= kInfBits && bad == 0xffffffffu) bad = (uint32_t)(256 * k + 8 * lane + j);
    }
    if (kStage) {
      rm = __reduce_max_sync(kFull, rm);
      stage_row(a, c, k, lane, d, rm);
      if (lane == k) a.stg_max[4 * c + k] = rm;
    }
    mx = max(mx, rm);
  }
  const uint32_t m = kStage ? mx : __reduce_max_sync(kFull, mx);
  if (m >= kInfBits) {  // index of the first non-finite Delta of the chunk (as record_first_bad)
    const uint32_t b = __reduce_min_sync(kFull, bad);
    if (lane == 0 && b != 0xffffffffu)
      atomicMin(reinterpret_cast<unsigned long long*>(a.slot + a.trailer_off + 8), (unsigned long long)(c * 1024 + b));
  }
  const int64_t blk = block_of_chunk(a, c);
  if (blk != cur) {
    if (cur >= 0 && lane == 0) atomicMax(reinterpret_cast<unsigned int*>(a.slot + a.scales_off) + cur, run);
    cur = blk;
    run = 0;
  }
  run = max(run, m);
}

template <bool kStage, bool kEF>
__global__ void __launch_bounds__(kThreads, 3) k_adamw_absmax(QArgs a, AdamArgs h) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nfull = a.n >> 10;
  int64_t cur = -1;
  uint32_t run = 0;
  for (int64_t c = warp; c < nfull; c += nwarps) adamw_absmax_chunk<true, kStage, kEF>(a, h, c, lane, cur, run);
  if ((nfull << 10) < a.n && warp == nfull % nwarps)
    adamw_absmax_chunk<false, kStage, kEF>(a, h, nfull, lane, cur, run);
  flush_block_max(a, lane, cur, run);
}

// ---------------------------------------------------------------------------
// k_apply: fused receive side.  Thread i owns elements 8i..8i+7: one LDG.256
// of A, v, theta each, one 32-bit code word and one scale per slot.
// ---------------------------------------------------------------------------
struct AArgs {
  const uint8_t* gather;
  size_t pb;             // payload bytes (slot stride)
  int M;
  int64_t n;
  int32_t lgB;           // log2(B) or -1
  size_t scales_off, trailer_off;
  float* A;
  float* v;
  float* theta;
  float lr, mu, alpha, beta, invM;
  int pow2M;
  unsigned long long* status;
  // push and pull modes: k_round_wait's verdict {first_bad, code} for this
  // round; null in copy-engine mode (the CTAs read the local trailers)
  const unsigned long long* verdict;
  int rank;
  // pull mode: slot m != rank is read from rank m's own buffer over NVLink
  // (symmetric window; M <= 32, enforced by the host)
  int pull;
  ncclWindow_t win;
  size_t half_off;
};

// The round check every CTA makes before touching A, v, theta, by thread 0:
// copy-engine mode reads the M trailers (local, L2-resident after the first
// CTAs); push and pull modes read k_round_wait's verdict.  -> code (0 apply,
// 1 non-finite, 2 malformed, 3 timeout) and the smallest first_bad.
__device__ __forceinline__ int round_check(const AArgs& p, int M, unsigned long long& fb) {
  if (p.verdict) {
    fb = p.verdict[0];
    return (int)p.verdict[1];
  }
  int bad = 0;
  fb = ~0ull;
  for (int q = 0; q < M; ++q) {
    const unsigned long long f = own_trailer_fb(p.gather + (size_t)q * p.pb, p.trailer_off, &bad);
    fb = f < fb ? f : fb;
  }
  return bad ? 2 : (fb != ~0ull ? 1 : 0);
}

// Decodes 8 codes (nibble i = element i) into LUT values +-2^(e-7) (codes 0
// and 8 -> +0) times s.  The LUT value's top 16 bits are the
// bf16 pattern sign<<15 | (e+120)<<7: byte tables via PRMT build two bf16
// per 32-bit word, the valid signs are PRMT-moved to bits 15/31, and each
// bf16 widens to fp32 by a shift or a mask.  q = LUT * s rounds like the
// oracle's LUT[c] * s (exact unless it underflows).
__device__ __forceinline__ void decode8(uint32_t w, float s, float (&q)[8]) {
  const uint32_t ctrl = w & 0x77777777u;                                  // e of each nibble
  const uint32_t sg = w & ((ctrl + 0x77777777u) & 0x88888888u);           // sign bits of codes with e > 0
  const uint32_t z = sg << 4;
  const uint32_t hi_a = __byte_perm(0x3D3D3C00u, 0x3F3F3E3Eu, ctrl);       // (e+120)>>1, e = 0 -> 0
  const uint32_t lo_a = __byte_perm(0x80008000u, 0x80008000u, ctrl);       // ((e+120)&1)<<7, e = 0 -> 0
  const uint32_t hi_b = __byte_perm(0x3D3D3C00u, 0x3F3F3E3Eu, ctrl >> 16);
  const uint32_t lo_b = __byte_perm(0x80008000u, 0x80008000u, ctrl >> 16);
  uint32_t pr[4];
  pr[0] = __byte_perm(lo_a, hi_a, 0x5140) | (__byte_perm(z, sg, 0x4400) & 0x80008000u);
  pr[1] = __byte_perm(lo_a, hi_a, 0x7362) | (__byte_perm(z, sg, 0x5511) & 0x80008000u);
  pr[2] = __byte_perm(lo_b, hi_b, 0x5140) | (__byte_perm(z, sg, 0x6622) & 0x80008000u);
  pr[3] = __byte_perm(lo_b, hi_b, 0x7362) | (__byte_perm(z, sg, 0x7733) & 0x80008000u);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    q[2 * k] = __fmul_rn(__uint_as_float(pr[k] << 16), s);
    q[2 * k + 1] = __fmul_rn(__uint_as_float(pr[k] & 0xffff0000u), s);
  }
}

__device__ __forceinline__ void outer_step(float S, float& a, float& w, float& t, const AArgs& p) {
  const float g = p.pow2M ? __fmul_rn(S, p.invM) : __fdiv_rn(S, (float)p.M);     // (1/M) sum
  w = __fadd_rn(__fmul_rn(p.mu, w), g);                                            // v = mu v + g
  a = __fsub_rn(a, __fmul_rn(p.lr, __fadd_rn(g, __fmul_rn(p.mu, w))));            // A -= lr (g + mu v)
  t = __fadd_rn(__fmul_rn(p.alpha, t), __fmul_rn(p.beta, a));                      // alpha merge
}

template <int kM, bool kAdam>
#ifndef SD_APPLY_MINB
#define SD_APPLY_MINB 4  // <= 64 registers, no spills: M = 8 apply 1.03 vs 0.975 at 3 CTAs/SM (B200 A/B)
#endif
#ifndef SD_APPLY_MINB_ADAM8
#define SD_APPLY_MINB_ADAM8 3  // AdamW-fused M = 8 apply: spill-free at 80 registers, 1.060 vs 1.076 ms at 4 (profiles/fused_merge_r1.txt)
#endif
__global__ void __launch_bounds__(kThreads, (kAdam && kM == 8) ? SD_APPLY_MINB_ADAM8 : SD_APPLY_MINB)
    k_apply(AArgs p, AdamArgs h) {
  __shared__ int s_skip;
  const int M = kM > 0 ? kM : p.M;
  // one barrier (each CTA is short-lived: a second one measured 2.5% slower)
  if (threadIdx.x == 0) {
    unsigned long long fb;
    const int code = round_check(p, M, fb);
    s_skip = code != 0;
    if (code && blockIdx.x == 0 && p.status && !p.verdict) {
      volatile unsigned long long* st = p.status;
      st[0] = fb;
      st[1] = (unsigned long long)code;
    }
  }
  __syncthreads();
  const bool skip = s_skip;
  if (skip && !kAdam) return;  // skipped round: nothing changes (with kAdam the inner step still runs)
  // slot m's base address.  Pull mode: slot m of rank m's buffer through the
  // window's NVLink (LSA) mapping, ncclGetLsaPointer(win, half_off + m pb, m)
  // = LSA(half_off, 0) + m (LSA stride + pb) -- the flat per-peer layout of
  // the LSA window; k_round_wait checks that identity for every peer of
  // every round before the apply may run.  Kept in registers: reading the M
  // addresses from shared memory instead measured 4% slower
  // (profiles/r2_pull_ab.txt).
  const uint8_t* gb = p.gather;
  size_t gs = p.pb;
  if (p.pull) {
    const uint8_t* b0 = static_cast<const uint8_t*>(ncclGetLsaPointer(p.win, p.half_off, 0));
    gb = b0;
    if (M > 1) gs = (size_t)(static_cast<const uint8_t*>(ncclGetLsaPointer(p.win, p.half_off, 1)) - b0) + p.pb;
  }
  auto slot_of = [&](int m) -> const uint8_t* { return gb + (size_t)m * gs; };

  const int64_t n8 = p.n >> 3;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += nthr) {
    // payload words first: in pull mode M-1 of them come over NVLink (longest latency)
    constexpr int kMr = kM > 0 ? kM : 1;
    uint32_t code[kMr];
    float scl[kMr];
    const int64_t blk = p.lgB < 0 ? 0 : ((8 * i) >> p.lgB);
    if (kM > 0 && !(kAdam && skip)) {
#pragma unroll
      for (int m = 0; m < kMr; ++m) {
        const uint8_t* slot = slot_of(m);
        code[m] = ld_code_word(reinterpret_cast<const uint32_t*>(slot) + i);
        scl[m] = __ldg(reinterpret_cast<const float*>(slot + p.scales_off) + blk);
      }
    }
    f8 t = ld8(p.theta + 8 * i);  // coherent load: this kernel writes theta
    if (kAdam) {  // the inner step of this step first (Alg. 2 L5 precedes L10-13)
      const f8 g = ld8_stream(h.grad + 8 * i);
      f8 m1 = ld8(h.m + 8 * i), m2 = ld8(h.v + 8 * i);
#pragma unroll
      for (int j = 0; j < 8; ++j) adamw_one(t.v[j], g.v[j], m1.v[j], m2.v[j], h);
      st8(h.m + 8 * i, m1);
      st8(h.v + 8 * i, m2);
      if (skip) {
        st8(p.theta + 8 * i, t);
        continue;
      }
    }
    f8 a = ld8(p.A + 8 * i);
    f8 w = ld8(p.v + 8 * i);
    float S[8];
#pragma unroll 8
    for (int m = 0; m < M; ++m) {
      uint32_t cw;
      float s;
      if (kM > 0) {
        cw = code[m];
        s = scl[m];
      } else {
        const uint8_t* slot = slot_of(m);
        cw = ld_code_word(reinterpret_cast<const uint32_t*>(slot) + i);
        s = __ldg(reinterpret_cast<const float*>(slot + p.scales_off) + blk);
      }
      float q[8];
      decode8(cw, s, q);
#pragma unroll
      for (int j = 0; j < 8; ++j) S[j] = (m == 0) ? q[j] : __fadd_rn(S[j], q[j]);  // ascending m
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) outer_step(S[j], a.v[j], w.v[j], t.v[j], p);
    st8(p.A + 8 * i, a);
    st8(p.v + 8 * i, w);
    st8(p.theta + 8 * i, t);
  }
  // ragged tail: the last n % 8 elements, one thread each
  if (blockIdx.x == 0 && threadIdx.x < (p.n & 7)) {
    const int64_t e = (n8 << 3) + threadIdx.x;
    float t = p.theta[e];
    if (kAdam) {
      float m1 = h.m[e], m2 = h.v[e];
      adamw_one(t, h.grad[e], m1, m2, h);
      h.m[e] = m1;
      h.v[e] = m2;
      if (skip) {
        p.theta[e] = t;
        return;
      }
    }
    const int64_t blk = p.lgB < 0 ? 0 : (e >> p.lgB);
    float S = 0.0f;
    for (int m = 0; m < M; ++m) {
      const uint8_t* slot = slot_of(m);
      const uint32_t c = (slot[e >> 1] >> ((e & 1) * 4)) & 15u;
      float q[8];
      decode8(c, reinterpret_cast<const float*>(slot + p.scales_off)[blk], q);
      S = (m == 0) ? q[0] : __fadd_rn(S, q[0]);
    }
    float a = p.A[e], w = p.v[e];
    outer_step(S, a, w, t, p);
    p.A[e] = a;
    p.v[e] = w;
    p.theta[e] = t;
  }
}

int ilog2_or_neg(int32_t B) {
  if (B <= 0) return -1;
  int l = 0;
  while ((1 << l) < B) ++l;
  return l;
}

// Grid sizing.  Measured on B200 (scripts/gpu_grid_sweep.sh, 1B fragments):
// one CTA per tile of work (no grid-stride iterations) beats a persistent
// SMs x occupancy grid by ~8% (apply) / ~10% (quantize) -- the resident CTAs
// then cover a compact, advancing address window, which keeps DRAM pages
// open.  SD_BLOCKS_PER_SM=<k> caps the grid at k CTAs per SM (experiments).
int blocks_per_sm_cap() {
  static int cap = -1;
  if (cap < 0) {
    const char* e = getenv("SD_BLOCKS_PER_SM");
    cap = e ? atoi(e) : 0;
  }
  return cap;
}

template <typename K>
int grid_for(K kernel, int num_sms, int64_t work_items, int items_per_block) {
  (void)kernel;
  int64_t g = (work_items + items_per_block - 1) / items_per_block;
  if (blocks_per_sm_cap() > 0 && g > (int64_t)num_sms * blocks_per_sm_cap()) g = (int64_t)num_sms * blocks_per_sm_cap();
  if (g > 0x7fffffffLL) g = 0x7fffffffLL;
  return g < 1 ? 1 : (int)g;
}


}  // namespace

namespace {
// Round-signal form: fused into the payload kernel's last CTA, or a separate
// one-thread kernel after it.  Measured at N = 2 and 4 (profiles/r2_pull_ab.txt):
// equal for pull; for push the fused form costs the quantize ~6% (its CTAs
// linger on the release ticket until their NVLink stores complete), so push
// signals from its own kernel.  SD_SIGNAL_KERNEL=0|1 forces one form.
bool signal_kernel(bool push) {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("SD_SIGNAL_KERNEL");
    v = e ? (atoi(e) == 1 ? 1 : 0) : -1;
  }
  return v >= 0 ? v == 1 : push;
}

QArgs make_qargs(const float* theta, const float* anchor, const Payload& pl, uint8_t* slot, const Round& rd) {
  QArgs a;
  a.theta = theta;
  a.anchor = anchor;
  a.n = pl.n;
  a.nb = pl.nb;
  a.lgB = ilog2_or_neg(pl.B);
  a.slot = slot;
  a.scales_off = pl.scales_off;
  a.trailer_off = pl.trailer_off;
  a.bytes = pl.bytes;
  a.push = rd.win != nullptr && rd.push;
  a.win = rd.win;
  a.win_off = rd.win_off;
  a.rank = rd.rank;
  a.M = rd.M;
  a.sig = rd.win != nullptr && !signal_kernel(rd.push);
  a.flags_off = rd.flags_off;
  a.seq = (unsigned long long)rd.seq;
  a.counter = rd.counter;
  a.stg = nullptr;
  a.stg_max = nullptr;
  a.stg_hints = 0;
  a.stg_keep_from = INT64_MAX;
  return a;
}

bool single_pass(int32_t B) { return B == 256 || B == 512 || B == 1024; }

// the separate-kernel form of the round signal (SD_SIGNAL_KERNEL=1)
int maybe_signal(const Round& rd, const QArgs& a, cudaStream_t st) {
  if (!rd.win || !signal_kernel(rd.push)) return 0;
  QArgs s = a;
  s.push = rd.push;
  k_signal<<<1, 32, 0, st>>>(s);
  return 1;
}

}  // namespace

namespace {
// Two passes (B = 0 or B > 1024): the scales come from atomics, so the slot
// is built locally; in push mode the finished slot is then pushed (and the
// round signalled) by k_push_copy.  Pass 1 is k_absmax, or k_adamw_absmax
// when an AdamW step is fused in (h != nullptr).
// Staging hints (SD_STAGE_HINTS, measurement switch; default both): bit 0
// pass 1 reads theta, A (and g) evict-first in L2, so the summaries it
// writes stay there for pass 2; bit 1 pass 2 discards the summaries it has
// consumed (no write-back of dead lines).
int stage_hints() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SD_STAGE_HINTS");
    v = e ? (atoi(e) & 3) : 3;
  }
  return v;
}

// MB of summaries kept in L2 between the passes (SD_STAGE_L2_MB, measurement switch; default 40)
int stage_keep_mb() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SD_STAGE_L2_MB");
    v = e ? atoi(e) : 40;
    if (v < 0) v = 0;
  }
  return v;
}

template <bool kStage, bool kEF>
void launch_pass1(const QArgs& a, const AdamArgs* h, int g, cudaStream_t st) {
  if (h)
    k_adamw_absmax<kStage, kEF><<<g, kThreads, 0, st>>>(a, *h);
  else
    k_absmax<kStage, kEF><<<g, kThreads, 0, st>>>(a);
}

int two_pass(const QArgs& a, const Round& rd, const Payload& pl, uint8_t* slot, int num_sms, cudaStream_t st,
             const AdamArgs* h, const Workspace& ws) {
  const int64_t chunks = (pl.n + 1023) >> 10;
  const int wpb = kThreads / 32;
  QArgs loc = a;
  loc.push = 0;
  loc.sig = a.sig && !a.push;
  if (ws.ptr && ws.bytes >= stage_bytes(pl.n) && chunks > 0) {
    loc.stg = reinterpret_cast<uint32_t*>(ws.ptr);
    loc.stg_max = reinterpret_cast<uint32_t*>(ws.ptr + 2048 * (size_t)chunks);
    loc.stg_hints = stage_hints();
    // the last stage_keep_mb() MB of summaries pass 1 writes stay in L2 for pass 2 (which starts there and
    // discards them: no write-back) -- only with the discard hint, or they would linger as evict-last lines
    if (loc.stg_hints & 2) loc.stg_keep_from = chunks - (int64_t)stage_keep_mb() * (1 << 20) / 2048;
  }
  if (pl.nb > 0 && cudaMemsetAsync(slot + pl.scales_off, 0, 4 * (size_t)pl.nb, st) != cudaSuccess) return -1;
  QArgs pass1 = loc;
  pass1.sig = 0;
  const int g1 = grid_for(k_absmax<false, false>, num_sms, chunks, wpb);
  if (!loc.stg)
    launch_pass1<false, false>(pass1, h, g1, st);
  else if (loc.stg_hints & 1)
    launch_pass1<true, true>(pass1, h, g1, st);
  else
    launch_pass1<true, false>(pass1, h, g1, st);
  if (loc.stg) {
    const int64_t g = (chunks + wpb * kStagedCpw - 1) / (wpb * kStagedCpw);  // one CTA per tile (>= 1: write_tail)
    k_encode_staged<<<g < 1 ? 1 : (int)g, kThreads, 0, st>>>(loc);
  } else {
    k_encode<<<grid_for(k_encode, num_sms, chunks, wpb), kThreads, 0, st>>>(loc);
  }
  int launched = 2;
  if (a.push) {
    k_push_copy<<<grid_for(k_push_copy, num_sms, (int64_t)(pl.bytes / 16), kThreads), kThreads, 0, st>>>(a);
    ++launched;
  }
  launched += maybe_signal(rd, a, st);
  return cudaGetLastError() == cudaSuccess ? launched : -1;
}
}  // namespace

// [chunks x 2 KB summaries][chunks x 16 B row maxima]
size_t stage_bytes(int64_t n) {
  const int64_t chunks = n > 0 ? (n + 1023) >> 10 : 0;
  return (size_t)chunks * (2048 + 16);
}

int launch_quantize(const float* theta, const float* anchor, const Payload& pl, uint8_t* slot, const Round& rd,
                    int num_sms, cudaStream_t st, const Workspace& ws) {
  const QArgs a = make_qargs(theta, anchor, pl, slot, rd);
  const int64_t chunks = (pl.n + 1023) >> 10;
  const int wpb = kThreads / 32;
  if (single_pass(pl.B)) {
    const int g = grid_for(k_quantize<1>, num_sms, chunks > 0 ? chunks : 1, wpb);  // >= 1 CTA: write_tail
    if (pl.B == 1024) k_quantize<1><<<g, kThreads, 0, st>>>(a);
    else if (pl.B == 512) k_quantize<2><<<g, kThreads, 0, st>>>(a);
    else k_quantize<4><<<g, kThreads, 0, st>>>(a);
    const int ks = maybe_signal(rd, a, st);
    return cudaGetLastError() == cudaSuccess ? 1 + ks : -1;
  }
  return two_pass(a, rd, pl, slot, num_sms, st, nullptr, ws);
}

int launch_round_wait(const RoundRecv& rr, const Payload& pl, int M, uint64_t timeout_ns, unsigned long long* status,
                      cudaStream_t st) {
  WArgs w;
  w.flags = rr.flags;
  w.own = rr.own;
  w.trailer_off = pl.trailer_off;
  w.verdict = rr.verdict;
  w.M = M;
  w.rank = rr.rank;
  w.seq = (unsigned long long)rr.seq;
  w.timeout_ns = (unsigned long long)timeout_ns;
  w.status = status;
  w.win = rr.win;
  w.flags_off = rr.flags_off;
  w.pull = rr.pull;
  w.half_off = rr.half_off;
  w.pb = pl.bytes;
  const int threads = 32 * ((M + 31) / 32);
  k_round_wait<<<1, threads, 0, st>>>(w);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

namespace {
AdamArgs make_adam(float* theta, const float* grad, float* m, float* v, int64_t n, const AdamHyper& hp) {
  AdamArgs h;
  h.theta = theta;
  h.grad = grad;
  h.m = m;
  h.v = v;
  h.n = n;
  h.b1 = hp.b1;
  h.b2 = hp.b2;
  h.c1 = hp.c1;
  h.c2 = hp.c2;
  h.decay = hp.decay;
  h.step = hp.step;
  h.sbc2 = hp.sbc2;
  h.eps = hp.eps;
  return h;
}
}  // namespace

int launch_adamw(float* theta, const float* grad, float* m, float* v, int64_t n, const AdamHyper& hp, int num_sms,
                 cudaStream_t st) {
  const AdamArgs h = make_adam(theta, grad, m, v, n, hp);
  const int64_t items = (n >> 3) > 0 ? (n >> 3) : 1;
  k_adamw<<<grid_for(k_adamw, num_sms, items, kThreads), kThreads, 0, st>>>(h);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

int launch_adamw_quantize(float* theta, const float* grad, float* m, float* v, const float* anchor, const Payload& pl,
                          uint8_t* slot, const AdamHyper& hp, const Round& rd, int num_sms, cudaStream_t st,
                          const Workspace& ws) {
  const QArgs a = make_qargs(theta, anchor, pl, slot, rd);
  const AdamArgs h = make_adam(theta, grad, m, v, pl.n, hp);
  if (!single_pass(pl.B)) return two_pass(a, rd, pl, slot, num_sms, st, &h, ws);  // AdamW + block max, then encode
  const int64_t chunks = (pl.n + 1023) >> 10;
  const int g = grid_for(k_adamw_quantize<1>, num_sms, chunks > 0 ? chunks : 1, kThreads / 32);
  if (pl.B == 1024)
    k_adamw_quantize<1><<<g, kThreads, 0, st>>>(a, h);
  else if (pl.B == 512)
    k_adamw_quantize<2><<<g, kThreads, 0, st>>>(a, h);
  else
    k_adamw_quantize<4><<<g, kThreads, 0, st>>>(a, h);
  const int ks = maybe_signal(rd, a, st);
  return cudaGetLastError() == cudaSuccess ? 1 + ks : -1;
}

int launch_apply(const uint8_t* gather, const Payload& pl, int M, float* theta, float* anchor, float* momentum,
                 float lr, float mu, float alpha, unsigned long long* status, int num_sms, cudaStream_t st,
                 const AdamInner* inner, const RoundRecv* rr) {
  AArgs p;
  p.gather = gather;
  p.pb = pl.bytes;
  p.M = M;
  p.n = pl.n;
  p.lgB = ilog2_or_neg(pl.B);
  p.scales_off = pl.scales_off;
  p.trailer_off = pl.trailer_off;
  p.A = anchor;
  p.v = momentum;
  p.theta = theta;
  p.lr = lr;
  p.mu = mu;
  p.alpha = alpha;
  p.beta = 1.0f - alpha;  // rounded once (AMB-14), host fp32 subtraction
  p.pow2M = (M & (M - 1)) == 0;
  p.invM = 1.0f / (float)M;  // exact when M is a power of two
  p.status = status;
  p.verdict = rr ? rr->verdict : nullptr;
  p.rank = rr ? rr->rank : 0;
  p.pull = rr != nullptr && rr->pull;
  p.win = rr ? rr->win : nullptr;
  p.half_off = rr ? rr->half_off : 0;
  AdamArgs h{};
  if (inner) h = make_adam(theta, inner->grad, inner->m, inner->v, pl.n, inner->hp);
  const int64_t items = (p.n >> 3) > 0 ? (p.n >> 3) : 1;
  const int g = grid_for(k_apply<1, false>, num_sms, items, kThreads);
#define SD_APPLY_CASE(KM)                                     \
  if (inner)                                                  \
    k_apply<KM, true><<<g, kThreads, 0, st>>>(p, h);          \
  else                                                        \
    k_apply<KM, false><<<g, kThreads, 0, st>>>(p, h);
  switch (M) {
    case 1: SD_APPLY_CASE(1) break;
    case 2: SD_APPLY_CASE(2) break;
    case 4: SD_APPLY_CASE(4) break;
    case 8: SD_APPLY_CASE(8) break;
    default: SD_APPLY_CASE(0) break;
  }
#undef SD_APPLY_CASE
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace sdk
