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
//   k_absmax + k_encode: the two-pass variant for B = 0 (one scale per
//               fragment) and B > 1024.
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
__device__ __forceinline__ f8 ld8(const float* p) {
  f8 r;
  asm volatile("ld.global.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]), "=f"(r.v[4]), "=f"(r.v[5]),
                 "=f"(r.v[6]), "=f"(r.v[7])
               : "l"(p));
  return r;
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
  int64_t c_begin;  // first 1024-element chunk this launch handles (k_quantize tail after the TMA kernel)
  // fused all-gather (push mode): every payload word is also stored into the
  // same offset of this rank's slot in each peer's gather buffer (NVLink,
  // NCCL symmetric window, LSA pointers)
  int push;
  ncclWindow_t win;
  size_t win_off;   // window offset of this rank's slot (same on every rank)
  int rank, M;
};

__device__ __forceinline__ void push_u32(const QArgs& a, size_t off, uint32_t v) {
  for (int q = 0; q < a.M; ++q)
    if (q != a.rank) *reinterpret_cast<uint32_t*>(ncclGetLsaPointer(a.win, a.win_off + off, q)) = v;
}
__device__ __forceinline__ void push_u8(const QArgs& a, size_t off, uint8_t v) {
  for (int q = 0; q < a.M; ++q)
    if (q != a.rank) *reinterpret_cast<uint8_t*>(ncclGetLsaPointer(a.win, a.win_off + off, q)) = v;
}

// Chunk = 1024 elements = 4 rows of 256; lane `lane` owns elements
// c*1024 + k*256 + 8*lane .. +7 of row k (one LDG.256 per array and row).
// Elements past n of the ragged last chunk read as Delta = +0.
template <bool kFullChunk>
__device__ __forceinline__ void load_chunk(const QArgs& a, int64_t c, int lane, f8 (&d)[4]) {
  const int64_t e0 = c * 1024 + 8 * lane;
  if (kFullChunk) {
    f8 th[4], an[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      th[k] = ld8_stream(a.theta + e0 + 256 * k);
      an[k] = ld8_stream(a.anchor + e0 + 256 * k);
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
  for (int64_t c = a.c_begin + warp; c < nfull; c += nwarps) quantize_chunk<NB, true>(a, c, lane);
  if ((nfull << 10) < a.n && warp == (nfull - a.c_begin) % nwarps) quantize_chunk<NB, false>(a, nfull, lane);
  if (blockIdx.x == 0) write_tail(a);
}

// ---------------------------------------------------------------------------
// k_quantize_tma: the same quantize with its input streams staged through
// shared memory by the bulk-copy engine (cp.async.bulk, 1-D TMA) in a
// kStages-deep mbarrier pipeline.  One producer warp per CTA issues the bulk
// copies of a tile (kCW chunks of theta and of A, 2 x 32 KB); kCW consumer
// warps each take one 1024-element chunk of the stage from shared memory and
// run the unchanged block-max / encode / store path.  Persistent grid (one
// CTA per SM); whole tiles only -- the remainder goes to k_quantize.
// ---------------------------------------------------------------------------
constexpr int kCW = 8;                       // consumer warps = chunks per tile
constexpr int kStages = 3;
constexpr int kTileBytes = kCW * 1024 * 4;   // per array
constexpr int kTmaThreads = 32 * (kCW + 1);
constexpr int kTmaSmem = kStages * 2 * kTileBytes + 2 * kStages * 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int NB>
__global__ void __launch_bounds__(kTmaThreads, 1) k_quantize_tma(QArgs a, int64_t ntiles) {
  extern __shared__ __align__(128) uint8_t smem[];
  float* sth = reinterpret_cast<float*>(smem);                      // [kStages][kCW*1024]
  float* san = reinterpret_cast<float*>(smem + kStages * kTileBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * kStages * kTileBytes);
  uint64_t* empty = full + kStages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {  // producer
    if (lane == 0) {
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % kStages;
        const uint32_t ph = (uint32_t)(it / kStages) & 1u;
        mbar_wait(&empty[st], ph ^ 1u);  // slot free (first pass: passes at once)
        mbar_expect_tx(&full[st], 2 * kTileBytes);
        const int64_t e0 = tile * (kCW * 1024);
        bulk_g2s(sth + st * (kCW * 1024), a.theta + e0, kTileBytes, &full[st]);
        bulk_g2s(san + st * (kCW * 1024), a.anchor + e0, kTileBytes, &full[st]);
      }
    }
    return;
  }
  const int cw = warp - 1;  // consumer index = chunk within the tile
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % kStages;
    const uint32_t ph = (uint32_t)(it / kStages) & 1u;
    mbar_wait(&full[st], ph);
    const float* th = sth + st * (kCW * 1024) + cw * 1024 + 8 * lane;
    const float* an = san + st * (kCW * 1024) + cw * 1024 + 8 * lane;
    f8 d[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 t0 = *reinterpret_cast<const float4*>(th + 256 * k);
      const float4 t1 = *reinterpret_cast<const float4*>(th + 256 * k + 4);
      const float4 a0 = *reinterpret_cast<const float4*>(an + 256 * k);
      const float4 a1 = *reinterpret_cast<const float4*>(an + 256 * k + 4);
      d[k].v[0] = __fsub_rn(a0.x, t0.x);
      d[k].v[1] = __fsub_rn(a0.y, t0.y);
      d[k].v[2] = __fsub_rn(a0.z, t0.z);
      d[k].v[3] = __fsub_rn(a0.w, t0.w);
      d[k].v[4] = __fsub_rn(a1.x, t1.x);
      d[k].v[5] = __fsub_rn(a1.y, t1.y);
      d[k].v[6] = __fsub_rn(a1.z, t1.z);
      d[k].v[7] = __fsub_rn(a1.w, t1.w);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // the stage's smem may be refilled
    encode_block_rows<NB, true>(a, tile * kCW + cw, lane, d);
  }
}

// ---------------------------------------------------------------------------
// Two-pass variant: B = 0 (whole fragment) or B a power of two >= 2048.
// Pass 1: per-block max |Delta| by atomicMax on the bit patterns (valid for
// non-negative floats; NaN/inf sort above every finite value).
// ---------------------------------------------------------------------------
__device__ __forceinline__ int64_t block_of_chunk(const QArgs& a, int64_t c) {
  return a.lgB < 0 ? 0 : ((c << 10) >> a.lgB);
}

template <bool kFullChunk>
__device__ __forceinline__ void absmax_chunk(const QArgs& a, int64_t c, int lane, int64_t& cur, uint32_t& run) {
  f8 d[4];
  load_chunk<kFullChunk>(a, c, lane, d);
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) m = max(m, row_max_bits(d[k]));
  m = __reduce_max_sync(kFull, m);
  if (m >= kInfBits) record_first_bad(a, c, lane, d);
  const int64_t blk = block_of_chunk(a, c);
  if (blk != cur) {
    if (cur >= 0 && lane == 0) atomicMax(reinterpret_cast<unsigned int*>(a.slot + a.scales_off) + cur, run);
    cur = blk;
    run = 0;
  }
  run = max(run, m);
}

__global__ void __launch_bounds__(kThreads) k_absmax(QArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nfull = a.n >> 10;
  int64_t cur = -1;
  uint32_t run = 0;
  for (int64_t c = warp; c < nfull; c += nwarps) absmax_chunk<true>(a, c, lane, cur, run);
  if ((nfull << 10) < a.n && warp == nfull % nwarps) absmax_chunk<false>(a, nfull, lane, cur, run);
  // merge the CTA's warps that ended in the same block: one atomic per distinct
  // block per CTA (B = 0: one per CTA instead of one per warp)
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

__global__ void __launch_bounds__(kThreads, 3) k_encode(QArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t nfull = a.n >> 10;
  const int64_t nchunks = nfull + ((nfull << 10) < a.n ? 1 : 0);
  // last chunk first: k_absmax streamed the fragment forward, so its tail is
  // what the L2 still holds when this second pass starts
  for (int64_t k = warp; k < nchunks; k += nwarps) {
    const int64_t c = nchunks - 1 - k;
    if (c < nfull) encode_chunk<true>(a, c, lane);
    else encode_chunk<false>(a, c, lane);
  }
  if (blockIdx.x == 0) write_tail(a);
}

// ---------------------------------------------------------------------------
// Push-mode all-gather completion (fused into the quantize).
// k_push_copy: two-pass quantize paths push the finished local slot (scales
//   written by atomics) to every peer.
// k_push_signal: after the pushing kernel, publish this rank's first
//   non-finite index, fence at system scope, then release-store the round id
//   (count of sends of the fragment, same on every rank) into flags[rank] of
//   every peer.
// k_push_wait: block-receive -- acquire-spin until every peer's flag holds it
//   (bounded: on a timeout the missing peer's slot is marked invalid, the
//   apply then skips the round and sd_check reports it).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_push_copy(QArgs a) {
  const size_t n16 = a.bytes / 16;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = reinterpret_cast<const uint4*>(a.slot)[i];
    for (int q = 0; q < a.M; ++q)
      if (q != a.rank) *reinterpret_cast<uint4*>(ncclGetLsaPointer(a.win, a.win_off + 16 * i, q)) = v;
  }
}

__global__ void k_push_signal(QArgs a, size_t flags_off, unsigned long long t) {
  if (threadIdx.x != 0) return;
  const unsigned long long fb = *reinterpret_cast<volatile unsigned long long*>(a.slot + a.trailer_off + 8);
  for (int q = 0; q < a.M; ++q)
    if (q != a.rank)
      *reinterpret_cast<unsigned long long*>(ncclGetLsaPointer(a.win, a.win_off + a.trailer_off + 8, q)) = fb;
  __threadfence_system();
  for (int q = 0; q < a.M; ++q) {
    if (q == a.rank) continue;
    unsigned long long* f =
        reinterpret_cast<unsigned long long*>(ncclGetLsaPointer(a.win, flags_off + 8 * (size_t)a.rank, q));
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(t) : "memory");
  }
}

__global__ void k_push_wait(const unsigned long long* flags, uint8_t* half, size_t pb, size_t trailer_off, int M,
                            int rank, unsigned long long t, unsigned long long timeout_ns,
                            unsigned long long* status) {
  const int q = threadIdx.x;
  if (q >= M || q == rank) return;
  const unsigned long long t0 = globaltimer_ns();
  unsigned long long v = 0;
  while (true) {
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flags + q) : "memory");
    if (v == t) return;
    if (globaltimer_ns() - t0 > timeout_ns) break;
    __nanosleep(256);
  }
  // invalidate the missing peer's local slot and this rank's own slot: the
  // apply reads its own slot locally in every mode (the peers' slots are
  // remote in pull mode), so a bad magic there makes it skip the round
  *reinterpret_cast<volatile uint32_t*>(half + (size_t)q * pb + trailer_off) = 0u;
  *reinterpret_cast<volatile uint32_t*>(half + (size_t)rank * pb + trailer_off) = 0u;
  if (status) {
    volatile unsigned long long* st = status;
    st[1] = 2ull;
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

template <int NB>
__global__ void __launch_bounds__(kThreads) k_adamw_quantize(QArgs a, AdamArgs h) {
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
  // pull mode: slot m lives in rank m's own buffer (symmetric window); the
  // LSA mapping makes slot m = base0 + m * (peer stride + payload)
  int pull;
  ncclWindow_t win;
  size_t half_off;
};

__device__ __forceinline__ void slot_geometry(const AArgs& p, const uint8_t*& base, size_t& stride) {
  if (p.pull) {
    const uint8_t* b0 = static_cast<const uint8_t*>(ncclGetLsaPointer(p.win, p.half_off, 0));
    const uint8_t* b1 = static_cast<const uint8_t*>(ncclGetLsaPointer(p.win, p.half_off, 1));
    base = b0;
    stride = (size_t)(b1 - b0) + p.pb;
  } else {
    base = p.gather;
    stride = p.pb;
  }
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
  __shared__ int skip;
  const int M = kM > 0 ? kM : p.M;
  const uint8_t* gbase;
  size_t gstride;
  slot_geometry(p, gbase, gstride);
  if (threadIdx.x == 0) {
    unsigned long long fb = ~0ull;
    int badmagic = 0;
    for (int m = 0; m < M; ++m) {
      const uint8_t* tr = gbase + (size_t)m * gstride + p.trailer_off;
      if (*reinterpret_cast<const uint32_t*>(tr) != kMagic) badmagic = 1;
      const unsigned long long f = *reinterpret_cast<const unsigned long long*>(tr + 8);
      fb = f < fb ? f : fb;
    }
    skip = badmagic || fb != ~0ull;
    if (skip && blockIdx.x == 0 && p.status) {
      volatile unsigned long long* st = p.status;
      st[0] = fb;
      st[1] = badmagic ? 2ull : 1ull;
    }
  }
  __syncthreads();
  if (skip && !kAdam) return;  // poisoned round: nothing changes (with kAdam the inner step still runs)

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
        const uint8_t* slot = gbase + (size_t)m * gstride;
        code[m] = ld_code_word(reinterpret_cast<const uint32_t*>(slot) + i);
        scl[m] = __ldg(reinterpret_cast<const float*>(slot + p.scales_off) + blk);
      }
    }
    f8 t = kAdam ? ld8(p.theta + 8 * i) : ld8_stream(p.theta + 8 * i);
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
        const uint8_t* slot = gbase + (size_t)m * gstride;
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
      const uint8_t* slot = gbase + (size_t)m * gstride;
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

// ---------------------------------------------------------------------------
// k_apply_tma: k_apply with a tile's A, v, theta and M code chunks staged
// through shared memory by 1-D bulk copies (cp.async.bulk) in a
// kAStages-deep mbarrier ring: one producer warp, kAW consumer warps (two
// 256-element rows each), results stored directly with 256-bit stores.
// Persistent grid (one CTA per SM), whole tiles only -- launch_apply hands
// the rest to k_apply.  The north star's "staged through shared memory/TMA"
// design, kept as a measured alternative (SD_APPLY_TMA=1); same arithmetic
// (decode8 + ascending-m sum + outer_step), so bit-identical to k_apply.
// ---------------------------------------------------------------------------
#ifndef SD_ATMA_STAGES
#define SD_ATMA_STAGES 2  // best of the measured configurations (profiles/atma_ab_r1.txt)
#endif
#ifndef SD_ATMA_CTAS
#define SD_ATMA_CTAS 1  // CTAs per SM
#endif
constexpr int kAW = 8;                  // consumer warps
constexpr int kATile = kAW * 512;       // elements per tile
constexpr int kAStages = SD_ATMA_STAGES;
constexpr int kATmaThreads = 32 * (kAW + 1);
template <int kM>
struct ApplyTmaLayout {
  static constexpr int kArr = 4 * kATile;                      // bytes of A (or v, theta) per stage
  static constexpr int kCodes = kATile / 2;                    // code bytes per slot per stage
  static constexpr int kStage = 3 * kArr + kM * kCodes;
  static constexpr int kSmem = kAStages * kStage + 2 * kAStages * 8;
};

template <int kM>
__global__ void __launch_bounds__(kATmaThreads, SD_ATMA_CTAS) k_apply_tma(AArgs p, int64_t ntiles) {
  using L = ApplyTmaLayout<kM>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kAStages * L::kStage);
  uint64_t* empty = full + kAStages;
  __shared__ int skip;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint8_t* gbase = p.gather;
  const size_t gstride = p.pb;
  if (threadIdx.x == 0) {
    unsigned long long fb = ~0ull;
    int badmagic = 0;
    for (int m = 0; m < kM; ++m) {
      const uint8_t* tr = gbase + (size_t)m * gstride + p.trailer_off;
      if (*reinterpret_cast<const uint32_t*>(tr) != kMagic) badmagic = 1;
      const unsigned long long f = *reinterpret_cast<const unsigned long long*>(tr + 8);
      fb = f < fb ? f : fb;
    }
    skip = badmagic || fb != ~0ull;
    if (skip && blockIdx.x == 0 && p.status) {
      volatile unsigned long long* st = p.status;
      st[0] = fb;
      st[1] = badmagic ? 2ull : 1ull;
    }
    for (int s = 0; s < kAStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kAW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (skip) return;
  if (warp == 0) {  // producer
    if (lane == 0) {
      int it = 0;
      for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int st = it % kAStages;
        const uint32_t ph = (uint32_t)(it / kAStages) & 1u;
        mbar_wait(&empty[st], ph ^ 1u);
        mbar_expect_tx(&full[st], L::kStage);
        uint8_t* sb = smem + st * L::kStage;
        const int64_t e0 = tile * kATile;
        bulk_g2s(sb, p.A + e0, L::kArr, &full[st]);
        bulk_g2s(sb + L::kArr, p.v + e0, L::kArr, &full[st]);
        bulk_g2s(sb + 2 * L::kArr, p.theta + e0, L::kArr, &full[st]);
#pragma unroll
        for (int m = 0; m < kM; ++m)
          bulk_g2s(sb + 3 * L::kArr + m * L::kCodes, gbase + (size_t)m * gstride + e0 / 2, L::kCodes, &full[st]);
      }
    }
    return;
  }
  const int cw = warp - 1;
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    const int st = it % kAStages;
    const uint32_t ph = (uint32_t)(it / kAStages) & 1u;
    mbar_wait(&full[st], ph);
    const uint8_t* sb = smem + st * L::kStage;
#pragma unroll 1
    for (int r = 0; r < 2; ++r) {  // one 256-element row at a time: 24 floats + M code words live
      const int le = cw * 512 + r * 256 + 8 * lane;
      const float* sa = reinterpret_cast<const float*>(sb) + le;
      const float* sv = reinterpret_cast<const float*>(sb + L::kArr) + le;
      const float* stt = reinterpret_cast<const float*>(sb + 2 * L::kArr) + le;
      f8 a, w, t;
#pragma unroll
      for (int j = 0; j < 8; j += 4) {
        const float4 x = *reinterpret_cast<const float4*>(sa + j);
        const float4 y = *reinterpret_cast<const float4*>(sv + j);
        const float4 z = *reinterpret_cast<const float4*>(stt + j);
        a.v[j] = x.x; a.v[j + 1] = x.y; a.v[j + 2] = x.z; a.v[j + 3] = x.w;
        w.v[j] = y.x; w.v[j + 1] = y.y; w.v[j + 2] = y.z; w.v[j + 3] = y.w;
        t.v[j] = z.x; t.v[j + 1] = z.y; t.v[j + 2] = z.z; t.v[j + 3] = z.w;
      }
      uint32_t code[kM];
#pragma unroll
      for (int m = 0; m < kM; ++m) code[m] = *reinterpret_cast<const uint32_t*>(sb + 3 * L::kArr + m * L::kCodes + le / 2);
      const int64_t e = tile * kATile + le;
      const int64_t blk = p.lgB < 0 ? 0 : (e >> p.lgB);
      float S[8];
#pragma unroll
      for (int m = 0; m < kM; ++m) {
        const float sc = __ldg(reinterpret_cast<const float*>(gbase + (size_t)m * gstride + p.scales_off) + blk);
        float q[8];
        decode8(code[m], sc, q);
#pragma unroll
        for (int j = 0; j < 8; ++j) S[j] = (m == 0) ? q[j] : __fadd_rn(S[j], q[j]);  // ascending m
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) outer_step(S[j], a.v[j], w.v[j], t.v[j], p);
      st8(p.A + e, a);
      st8(p.v + e, w);
      st8(p.theta + e, t);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);  // the stage may be refilled
  }
}

bool use_tma_apply() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SD_APPLY_TMA");
    v = (e && atoi(e) == 1) ? 1 : 0;
  }
  return v == 1;
}

template <int kM>
void launch_apply_tma(const AArgs& p, int64_t ntiles, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_apply_tma<kM>, cudaFuncAttributeMaxDynamicSharedMemorySize, ApplyTmaLayout<kM>::kSmem);
    attr = true;
  }
  k_apply_tma<kM><<<grid, kATmaThreads, ApplyTmaLayout<kM>::kSmem, st>>>(p, ntiles);
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
QArgs make_qargs(const float* theta, const float* anchor, const Payload& pl, uint8_t* slot, const Push& push) {
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
  a.c_begin = 0;
  a.push = push.win != nullptr;
  a.win = push.win;
  a.win_off = push.win_off;
  a.rank = push.rank;
  a.M = push.M;
  return a;
}

bool single_pass(int32_t B) { return B == 256 || B == 512 || B == 1024; }

// SD_QUANTIZE_TMA=1 stages the quantize's input streams through shared memory
// with bulk copies (k_quantize_tma); default: direct 256-bit loads.
bool use_tma_quantize() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SD_QUANTIZE_TMA");
    v = (e && atoi(e) == 1) ? 1 : 0;
  }
  return v == 1;
}

template <int NB>
void launch_tma(const QArgs& a, int64_t ntiles, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_quantize_tma<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem);
    attr = true;
  }
  k_quantize_tma<NB><<<grid, kTmaThreads, kTmaSmem, st>>>(a, ntiles);
}
}  // namespace

int launch_quantize(const float* theta, const float* anchor, const Payload& pl, uint8_t* slot, const Push& push,
                    int num_sms, cudaStream_t st) {
  const QArgs a = make_qargs(theta, anchor, pl, slot, push);
  const int64_t chunks = (pl.n + 1023) >> 10;
  const int wpb = kThreads / 32;
  int launched = 0;
  if (single_pass(pl.B)) {
    QArgs t = a;
    const int64_t ntiles = use_tma_quantize() ? (pl.n >> 10) / kCW : 0;
    if (ntiles > 0) {  // whole tiles through the bulk-copy pipeline, the rest below
      const int g = (int)(ntiles < num_sms ? ntiles : num_sms);
      if (pl.B == 1024) launch_tma<1>(a, ntiles, g, st);
      else if (pl.B == 512) launch_tma<2>(a, ntiles, g, st);
      else launch_tma<4>(a, ntiles, g, st);
      t.c_begin = ntiles * kCW;
      ++launched;
    }
    const int64_t rest = chunks - t.c_begin > 0 ? chunks - t.c_begin : 1;  // >= 1 CTA: write_tail
    if (pl.B == 1024) k_quantize<1><<<grid_for(k_quantize<1>, num_sms, rest, wpb), kThreads, 0, st>>>(t);
    else if (pl.B == 512) k_quantize<2><<<grid_for(k_quantize<2>, num_sms, rest, wpb), kThreads, 0, st>>>(t);
    else k_quantize<4><<<grid_for(k_quantize<4>, num_sms, rest, wpb), kThreads, 0, st>>>(t);
    ++launched;
  } else {
    QArgs loc = a;
    loc.push = 0;  // scales come from atomics: build locally, then push the finished slot
    if (pl.nb > 0 && cudaMemsetAsync(slot + pl.scales_off, 0, 4 * (size_t)pl.nb, st) != cudaSuccess) return -1;
    k_absmax<<<grid_for(k_absmax, num_sms, chunks, wpb), kThreads, 0, st>>>(loc);
    k_encode<<<grid_for(k_encode, num_sms, chunks, wpb), kThreads, 0, st>>>(loc);
    launched = 2;
    if (a.push) {
      k_push_copy<<<grid_for(k_push_copy, num_sms, (int64_t)(pl.bytes / 16), kThreads), kThreads, 0, st>>>(a);
      launched = 3;
    }
  }
  return cudaGetLastError() == cudaSuccess ? launched : -1;
}

int launch_push_signal(const Payload& pl, uint8_t* slot, const Push& push, size_t flags_off, uint64_t t,
                       cudaStream_t st) {
  const QArgs a = make_qargs(nullptr, nullptr, pl, slot, push);
  k_push_signal<<<1, 32, 0, st>>>(a, flags_off, (unsigned long long)t);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

// ---------------------------------------------------------------------------
// Multicast gather support (NVLS through the NCCL device API).
// ---------------------------------------------------------------------------
struct McState {
  ncclDevComm_t dc;
  void** host_ptr = nullptr;  // mapped pinned word for mc_base
};

namespace {
__global__ void k_mc_base(ncclWindow_t w, ncclMultimemHandle mm, void** out) {
  *out = ncclGetMultimemPointer(w, 0, mm);
}
__global__ void k_flag_signal(ncclWindow_t w, size_t flags_off, int rank, int M, unsigned long long t) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int q = 0; q < M; ++q) {
    if (q == rank) continue;
    unsigned long long* f = reinterpret_cast<unsigned long long*>(ncclGetLsaPointer(w, flags_off + 8 * (size_t)rank, q));
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f), "l"(t) : "memory");
  }
}
}  // namespace

int mc_create(ncclComm_t comm, McState** out) {
  *out = nullptr;
  McState* s = new McState();
  ncclDevCommRequirements_t req = {};
  req.lsaMultimem = true;
  if (ncclDevCommCreate(comm, &req, &s->dc) != ncclSuccess) {
    delete s;
    return -1;
  }
  if (s->dc.lsaMultimem.mcBasePtr == nullptr ||
      cudaHostAlloc(reinterpret_cast<void**>(&s->host_ptr), sizeof(void*), cudaHostAllocMapped) != cudaSuccess) {
    ncclDevCommDestroy(comm, &s->dc);
    delete s;
    return 0;
  }
  *out = s;
  return 1;
}

void mc_destroy(ncclComm_t comm, McState* s) {
  if (!s) return;
  ncclDevCommDestroy(comm, &s->dc);
  if (s->host_ptr) cudaFreeHost(s->host_ptr);
  delete s;
}

int mc_base(McState* s, ncclWindow_t win, uint8_t** out, cudaStream_t st) {
  void** dev = nullptr;
  if (cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), s->host_ptr, 0) != cudaSuccess) return -1;
  k_mc_base<<<1, 1, 0, st>>>(win, s->dc.lsaMultimem, dev);
  if (cudaGetLastError() != cudaSuccess || cudaStreamSynchronize(st) != cudaSuccess) return -1;
  *out = static_cast<uint8_t*>(*reinterpret_cast<void* volatile*>(s->host_ptr));
  return *out ? 1 : -1;
}

int launch_flag_signal(ncclWindow_t win, size_t flags_off, int rank, int M, uint64_t t, cudaStream_t st) {
  k_flag_signal<<<1, 32, 0, st>>>(win, flags_off, rank, M, (unsigned long long)t);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

int launch_push_wait(const unsigned long long* flags, uint8_t* half, const Payload& pl, int M, int rank, uint64_t t,
                     uint64_t timeout_ns, unsigned long long* status, cudaStream_t st) {
  k_push_wait<<<1, 32, 0, st>>>(flags, half, pl.bytes, pl.trailer_off, M, rank, (unsigned long long)t,
                                (unsigned long long)timeout_ns, status);
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
                          uint8_t* slot, const AdamHyper& hp, const Push& push, int num_sms, cudaStream_t st) {
  if (!single_pass(pl.B)) {  // two-pass scales: AdamW, then quantize
    const int k1 = launch_adamw(theta, grad, m, v, pl.n, hp, num_sms, st);
    if (k1 < 0) return -1;
    const int k2 = launch_quantize(theta, anchor, pl, slot, push, num_sms, st);
    return k2 < 0 ? -1 : k1 + k2;
  }
  const QArgs a = make_qargs(theta, anchor, pl, slot, push);
  const AdamArgs h = make_adam(theta, grad, m, v, pl.n, hp);
  const int64_t chunks = (pl.n + 1023) >> 10;
  const int wpb = kThreads / 32;
  if (pl.B == 1024)
    k_adamw_quantize<1><<<grid_for(k_adamw_quantize<1>, num_sms, chunks, wpb), kThreads, 0, st>>>(a, h);
  else if (pl.B == 512)
    k_adamw_quantize<2><<<grid_for(k_adamw_quantize<2>, num_sms, chunks, wpb), kThreads, 0, st>>>(a, h);
  else
    k_adamw_quantize<4><<<grid_for(k_adamw_quantize<4>, num_sms, chunks, wpb), kThreads, 0, st>>>(a, h);
  return cudaGetLastError() == cudaSuccess ? 1 : -1;
}

int launch_apply(const uint8_t* gather, const Payload& pl, int M, float* theta, float* anchor, float* momentum,
                 float lr, float mu, float alpha, unsigned long long* status, int num_sms, cudaStream_t st,
                 const AdamInner* inner, const Pull* pull) {
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
  p.pull = pull != nullptr && pull->win != nullptr;
  p.win = p.pull ? pull->win : nullptr;
  p.half_off = p.pull ? pull->half_off : 0;
  AdamArgs h{};
  if (inner) h = make_adam(theta, inner->grad, inner->m, inner->v, pl.n, inner->hp);
  int launched = 0;
  // SD_APPLY_TMA=1: whole tiles through the bulk-copy pipeline (local slots,
  // no inner step, B a divisor of the tile), the rest through k_apply below
  const int64_t ntiles = (use_tma_apply() && !inner && !p.pull && (M == 1 || M == 2 || M == 4 || M == 8) &&
                          (pl.B == 0 || (pl.B >= 256 && pl.B <= kATile)))
                             ? pl.n / kATile
                             : 0;
  if (ntiles > 0) {
#ifdef SD_ATMA_ONESHOT
    const int64_t cap = ntiles;  // one CTA per tile
#else
    const int64_t cap = (int64_t)num_sms * SD_ATMA_CTAS;
#endif
    const int g = (int)(ntiles < cap ? ntiles : cap);
    switch (M) {
      case 1: launch_apply_tma<1>(p, ntiles, g, st); break;
      case 2: launch_apply_tma<2>(p, ntiles, g, st); break;
      case 4: launch_apply_tma<4>(p, ntiles, g, st); break;
      default: launch_apply_tma<8>(p, ntiles, g, st); break;
    }
    ++launched;
    const int64_t off = ntiles * kATile;  // a multiple of B: shift every stream to the rest
    p.A += off;
    p.v += off;
    p.theta += off;
    p.n -= off;
    p.gather += off / 2;
    p.scales_off = p.scales_off - (size_t)(off / 2) + (p.lgB < 0 ? 0 : 4 * (size_t)(off >> p.lgB));
    p.trailer_off -= (size_t)(off / 2);
    if (p.n == 0) return cudaGetLastError() == cudaSuccess ? launched : -1;
  }
  const int64_t items = (p.n >> 3) > 0 ? (p.n >> 3) : 1;
#define SD_APPLY_CASE(KM)                                                                                         \
  if (inner)                                                                                                      \
    k_apply<KM, true><<<grid_for(k_apply<KM, true>, num_sms, items, kThreads), kThreads, 0, st>>>(p, h);          \
  else                                                                                                            \
    k_apply<KM, false><<<grid_for(k_apply<KM, false>, num_sms, items, kThreads), kThreads, 0, st>>>(p, h);
  switch (M) {
    case 1: SD_APPLY_CASE(1) break;
    case 2: SD_APPLY_CASE(2) break;
    case 4: SD_APPLY_CASE(4) break;
    case 8: SD_APPLY_CASE(8) break;
    default: SD_APPLY_CASE(0) break;
  }
#undef SD_APPLY_CASE
  return cudaGetLastError() == cudaSuccess ? launched + 1 : -1;
}

}  // namespace sdk
