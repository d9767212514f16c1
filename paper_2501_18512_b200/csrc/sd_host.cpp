// sd_host.cpp — libsd host side: config validation, the closed-form fragment
// scheduler, the per-replica context (NCCL communicator, comm stream, events,
// in-flight table) and the C ABI of include/sd.h.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>  // ncclTeamLsa (host side of the NCCL 2.28 device API)

#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "sd.h"
#include "sd_kernels.h"

namespace {

thread_local char g_err[512] = "";
std::atomic<uint64_t> g_launches{0};

sd_status fail(char* buf, sd_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, 512, fmt, ap);
  va_end(ap);
  return st;
}

int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }

// Full validation (config is validated before any work).  Messages
// name the offending values.
sd_status validate(const sd_config* c, char* msg, size_t cap) {
  char tmp[512];
  sd_status st = SD_OK;
  if (!c) {
    st = fail(tmp, SD_ERR_ARG, "config pointer is NULL");
  } else if (c->abi_version != SD_ABI_VERSION) {
    st = fail(tmp, SD_ERR_CONFIG, "abi_version %u != SD_ABI_VERSION %u", c->abi_version, SD_ABI_VERSION);
  } else if (c->num_blocks < 1 || c->fragment_size < 1) {
    st = fail(tmp, SD_ERR_CONFIG, "num_blocks %d and fragment_size %d must both be >= 1", c->num_blocks,
              c->fragment_size);
  } else if (c->num_blocks % c->fragment_size != 0) {
    st = fail(tmp, SD_ERR_CONFIG, "fragment_size %d does not divide num_blocks %d", c->fragment_size,
              c->num_blocks);
  } else if (c->pattern != 0 && c->pattern != 1) {
    st = fail(tmp, SD_ERR_CONFIG, "pattern %d is neither 0 (sequential) nor 1 (strided)", c->pattern);
  } else if (c->embed_policy != 0 && c->embed_policy != 1) {
    st = fail(tmp, SD_ERR_CONFIG, "embed_policy %d is neither 0 nor 1", c->embed_policy);
  } else {
    const int32_t P = c->num_blocks / c->fragment_size + (c->embed_policy == 1 ? 1 : 0);
    if (c->H < 1 || c->H < P) {
      st = fail(tmp, SD_ERR_CONFIG, "H %d must be >= 1 and >= the number of fragments P %d", c->H, P);
    } else if (c->tau < 0 || c->tau >= c->H) {
      st = fail(tmp, SD_ERR_CONFIG, "tau %d violates 0 <= tau < H (H = %d)", c->tau, c->H);
    } else if (c->T < 0) {
      st = fail(tmp, SD_ERR_CONFIG, "T %lld must be >= 0 (0 = unbounded)", (long long)c->T);
    } else if (!(c->alpha >= 0.0f && c->alpha <= 1.0f)) {
      st = fail(tmp, SD_ERR_CONFIG, "alpha %g is not in [0, 1]", (double)c->alpha);
    } else if (!(c->outer_lr == c->outer_lr) || c->outer_lr > 3.4e38f || c->outer_lr < -3.4e38f) {
      st = fail(tmp, SD_ERR_CONFIG, "outer_lr %g is not finite", (double)c->outer_lr);
    } else if (!(c->outer_momentum >= 0.0f && c->outer_momentum < 1.0f)) {
      st = fail(tmp, SD_ERR_CONFIG, "outer_momentum %g is not in [0, 1)", (double)c->outer_momentum);
    } else if (c->scale_block != 0 &&
               (!is_pow2(c->scale_block) || c->scale_block < 256 || c->scale_block > (1 << 20))) {
      st = fail(tmp, SD_ERR_CONFIG, "scale_block %d is neither 0 nor a power of two in [256, 1048576]",
                c->scale_block);
    }
  }
  if (st != SD_OK) {
    snprintf(g_err, sizeof g_err, "%s", tmp);
    if (msg && cap) snprintf(msg, cap, "%s", tmp);
  }
  return st;
}

int32_t num_fragments(const sd_config* c) {
  return c->num_blocks / c->fragment_size + (c->embed_policy == 1 ? 1 : 0);
}

int32_t offset_of(const sd_config* c, int32_t p) {  // t_p = floor(p H / P)
  return (int32_t)(((int64_t)p * c->H) / num_fragments(c));
}

// (t - t_p) mod H == 0 with t >= H  (Alg. 2 L6; first send S:73)
bool sends_at(const sd_config* c, int32_t p, int64_t t) {
  return t >= c->H && (t - offset_of(c, p)) % c->H == 0;
}

// the send step s whose receive falls at t, or 0 (Alg. 2 L10; flush S:322)
int64_t receive_send_step(const sd_config* c, int32_t p, int64_t t) {
  if (c->T > 0 && t > c->T) return 0;
  const int64_t s = t - c->tau;
  if (s >= 1 && sends_at(c, p, s)) return s;
  if (c->T > 0 && t == c->T) {  // flush: the send of p in (T - tau, T], if any
    for (int64_t q = c->T - c->tau + 1; q <= c->T; ++q)
      if (q >= 1 && sends_at(c, p, q)) return q;
  }
  return 0;
}

sdk::Payload payload_of(const sd_config* c, int64_t n) {
  sdk::Payload pl;
  pl.n = n;
  pl.B = c->scale_block;
  pl.nb = n == 0 ? 0 : (c->scale_block == 0 ? 1 : (n + c->scale_block - 1) / c->scale_block);
  pl.scales_off = (size_t)align_up((n + 1) / 2, 256);
  pl.trailer_off = pl.scales_off + (size_t)align_up(4 * pl.nb, 16);
  pl.bytes = pl.scales_off + (size_t)align_up(align_up(4 * pl.nb, 16) + 16, 256);
  return pl;
}

enum FragState { IDLE = 0, QUANTIZED = 1, SYNCED = 2 };

struct Inflight {
  FragState state = IDLE;
  int64_t send_step = 0;
  int64_t n = 0;
  const void* slot = nullptr;
  const void* gather = nullptr;
  bool push = false;      // two-round symmetric buffer with round flags (PUSH or PULL mode)
  bool pull = false;      // PULL: the apply reads the peers' slots over NVLink
  bool waited = false;    // bounded wait: k_round_wait was issued for this round
  size_t half_off = 0;    // push / pull: byte offset of this round's half
  uint64_t seq = 0;       // push / pull: round id published in the peers' flags
};

}  // namespace

struct GatherBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  ncclWindow_t win = nullptr;
  bool nccl = false;
  bool push = false;   // two-round layout: halves (round parity) of M payloads + round flags (PUSH/PULL)
  bool pull = false;   // PULL mode: peers' payloads stay in the peers' buffers, read by the apply
  size_t half = 0;     // bytes per half
  size_t pb = 0;       // payload bytes
  // layout of a half (push / pull): [M payloads][M flag entries {round id, first_bad}]
  //                                 [verdict {first_bad, code}][last-CTA counter]
  size_t flags_rel(int M) const { return (size_t)M * pb; }
  size_t verdict_rel(int M) const { return flags_rel(M) + 16 * (size_t)M; }
  size_t counter_rel(int M) const { return verdict_rel(M) + 16; }
};

struct sd_ctx {
  sd_config cfg;
  std::vector<GatherBuf> bufs;
  int32_t gather_mode = SD_GATHER_AUTO;
  std::vector<uint64_t> round_seq;  // push mode: sends of each fragment so far (round id, same on every rank)
  int32_t rank = 0, M = 1, device = 0, P = 0, num_sms = 148;
  ncclComm_t comm = nullptr;
  bool lsa_all = false;        // every rank is in this rank's NVLink (LSA) team: PUSH / PULL possible
  bool dead = false;           // a bounded block-receive timed out: every later device call fails (sticky)
  cudaStream_t comm_stream = nullptr;
  cudaStream_t copy_stream = nullptr;               // outer-state offload (NEXT-3): host -> device
  cudaStream_t wb_stream = nullptr;                 // outer-state offload: device -> host (full duplex)
  std::vector<cudaEvent_t> ready, done;
  std::vector<cudaEvent_t> staged;                   // prefetch of fragment p landed
  std::vector<char> prefetch_pending;                // quantize must wait on staged[p]
  cudaEvent_t copy_gate = nullptr;
  // last writeback out of each device staging buffer (by anchor address): a
  // prefetch into that buffer waits for it; other copies run concurrently
  struct Drain {
    const void* staging;
    cudaEvent_t ev;
  };
  std::vector<Drain> drains;
  std::vector<Inflight> fl;
  sdk::Workspace ws;                          // caller-owned scratch of the two-pass quantize (sd_set_workspace)
  unsigned long long* status_host = nullptr;  // {first_bad, code, dead}: pinned, mapped
  unsigned long long* status_dev = nullptr;
  char err[512] = "";
};

namespace {

GatherBuf* find_buf(sd_ctx* c, const void* p) {
  for (GatherBuf& b : c->bufs)
    if (static_cast<const char*>(p) >= static_cast<const char*>(b.ptr) &&
        static_cast<const char*>(p) < static_cast<const char*>(b.ptr) + b.bytes)
      return &b;
  return nullptr;
}

sd_status cuda_fail(sd_ctx* c, cudaError_t e, const char* what) {
  snprintf(g_err, sizeof g_err, "%s: CUDA error %d (%s)", what, (int)e, cudaGetErrorString(e));
  if (c) snprintf(c->err, sizeof c->err, "%s", g_err);
  return SD_ERR_CUDA;
}

sd_status ctx_fail(sd_ctx* c, sd_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(c->err, sizeof c->err, fmt, ap);
  va_end(ap);
  snprintf(g_err, sizeof g_err, "%s", c->err);
  return st;
}

#define SD_CUDA(ctx, call)                              \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #call); \
  } while (0)

sd_status check_ptr(sd_ctx* c, const void* ptr, size_t align, const char* name) {
  if (!ptr) return ctx_fail(c, SD_ERR_ARG, "%s is NULL", name);
  if (reinterpret_cast<uintptr_t>(ptr) % align != 0)
    return ctx_fail(c, SD_ERR_ARG, "%s = %p is not %zu-byte aligned", name, ptr, align);
  return SD_OK;
}

sd_status check_fragment(sd_ctx* c, int32_t p, int64_t t, int64_t n) {
  if (p < 0 || p >= c->P) return ctx_fail(c, SD_ERR_ARG, "fragment %d out of range [0, %d)", p, c->P);
  if (t < 1) return ctx_fail(c, SD_ERR_ARG, "step t = %lld must be >= 1 (1-based, S:323)", (long long)t);
  if (n < 0) return ctx_fail(c, SD_ERR_ARG, "n = %lld is negative", (long long)n);
  return SD_OK;
}

}  // namespace

extern "C" {

sd_status sd_config_default(sd_config* c, int32_t num_blocks, int32_t fragment_size, int32_t H) {
  if (!c) return fail(g_err, SD_ERR_ARG, "config pointer is NULL");
  c->abi_version = SD_ABI_VERSION;
  c->num_blocks = num_blocks;
  c->fragment_size = fragment_size;
  c->pattern = 1;
  c->embed_policy = 0;
  c->H = H;
  c->tau = 1;
  c->T = 0;
  c->alpha = 0.5f;
  c->outer_lr = 0.4f;
  c->outer_momentum = 0.9f;
  c->scale_block = 1024;
  return SD_OK;
}

sd_status sd_config_validate(const sd_config* cfg, char* msg, size_t cap) {
  if (msg && cap) msg[0] = 0;
  return validate(cfg, msg, cap);
}

sd_status sd_fragment_count(const sd_config* cfg, int32_t* P) {
  sd_status st = validate(cfg, nullptr, 0);
  if (st != SD_OK) return st;
  if (!P) return fail(g_err, SD_ERR_ARG, "P pointer is NULL");
  *P = num_fragments(cfg);
  return SD_OK;
}

sd_status sd_fragment_layout(const sd_config* cfg, int32_t p, int32_t* blocks, int32_t cap,
                             int32_t* n_blocks, int32_t* t_p, int32_t* holds_embed) {
  sd_status st = validate(cfg, nullptr, 0);
  if (st != SD_OK) return st;
  const int32_t P = num_fragments(cfg);
  const int32_t Pb = cfg->num_blocks / cfg->fragment_size;
  if (p < 0 || p >= P) return fail(g_err, SD_ERR_ARG, "fragment %d out of range [0, %d)", p, P);
  const int32_t nbk = p < Pb ? cfg->fragment_size : 0;
  if (blocks && cap < nbk) return fail(g_err, SD_ERR_ARG, "cap %d < %d blocks of fragment %d", cap, nbk, p);
  if (blocks)
    for (int32_t k = 0; k < nbk; ++k) blocks[k] = cfg->pattern == 0 ? p * cfg->fragment_size + k : p + k * Pb;
  if (n_blocks) *n_blocks = nbk;
  if (t_p) *t_p = offset_of(cfg, p);
  if (holds_embed) *holds_embed = (cfg->embed_policy == 0) ? (p == Pb - 1) : (p == Pb);
  return SD_OK;
}

sd_status sd_fragment_schedule(const sd_config* cfg, int64_t t, int32_t* send, int32_t* n_send,
                               int32_t* recv, int32_t* n_recv, int32_t cap) {
  sd_status st = validate(cfg, nullptr, 0);
  if (st != SD_OK) return st;
  if (t < 1) return fail(g_err, SD_ERR_ARG, "step t = %lld must be >= 1 (1-based, S:323)", (long long)t);
  if (!n_send || !n_recv) return fail(g_err, SD_ERR_ARG, "n_send / n_recv pointer is NULL");
  const int32_t P = num_fragments(cfg);
  int32_t ns = 0, nr = 0;
  for (int32_t p = 0; p < P; ++p) {
    if ((cfg->T == 0 || t <= cfg->T) && sends_at(cfg, p, t)) {
      if (ns >= cap || !send) return fail(g_err, SD_ERR_ARG, "send list capacity %d too small", cap);
      send[ns++] = p;
    }
  }
  for (int32_t p = 0; p < P; ++p) {
    if (receive_send_step(cfg, p, t) != 0) {
      if (nr >= cap || !recv) return fail(g_err, SD_ERR_ARG, "receive list capacity %d too small", cap);
      recv[nr++] = p;
    }
  }
  *n_send = ns;
  *n_recv = nr;
  return SD_OK;
}

int64_t sd_num_scale_blocks(const sd_config* cfg, int64_t n) {
  if (validate(cfg, nullptr, 0) != SD_OK || n < 0) return 0;
  return payload_of(cfg, n).nb;
}

size_t sd_payload_bytes(const sd_config* cfg, int64_t n) {
  if (validate(cfg, nullptr, 0) != SD_OK || n < 0) return 0;
  return payload_of(cfg, n).bytes;
}

size_t sd_payload_scales_offset(int64_t n) { return n < 0 ? 0 : (size_t)align_up((n + 1) / 2, 256); }

size_t sd_payload_trailer_offset(const sd_config* cfg, int64_t n) {
  if (validate(cfg, nullptr, 0) != SD_OK || n < 0) return 0;
  return payload_of(cfg, n).trailer_off;
}

sd_status sd_get_unique_id(uint8_t id[SD_UNIQUE_ID_BYTES]) {
  if (!id) return fail(g_err, SD_ERR_ARG, "id pointer is NULL");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return fail(g_err, SD_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  static_assert(sizeof(u.internal) == SD_UNIQUE_ID_BYTES, "NCCL unique id size");
  memcpy(id, u.internal, SD_UNIQUE_ID_BYTES);
  return SD_OK;
}

sd_status sd_init(sd_ctx** out, const sd_config* cfg, int32_t rank, int32_t M, const uint8_t* id,
                  int32_t device) {
  if (!out) return fail(g_err, SD_ERR_ARG, "out pointer is NULL");
  *out = nullptr;
  sd_status st = validate(cfg, nullptr, 0);
  if (st != SD_OK) return st;
  if (M < 1 || rank < 0 || rank >= M) return fail(g_err, SD_ERR_ARG, "rank %d / M %d: need 0 <= rank < M", rank, M);
  sd_ctx* c = new (std::nothrow) sd_ctx();
  if (!c) return fail(g_err, SD_ERR_ARG, "out of host memory");
  c->cfg = *cfg;
  c->rank = rank;
  c->M = M;
  c->device = device;
  c->P = num_fragments(cfg);
  c->fl.resize((size_t)c->P);
  c->round_seq.assign((size_t)c->P, 0);
  auto bail = [&](sd_status s) {
    sd_finalize(c);
    return s;
  };
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "cudaSetDevice"));
  e = cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "cudaDeviceGetAttribute"));
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  e = cudaStreamCreateWithPriority(&c->comm_stream, cudaStreamNonBlocking, hi);
  if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "cudaStreamCreateWithPriority"));
  e = cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "cudaStreamCreate(copy)"));
  e = cudaStreamCreateWithFlags(&c->wb_stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "cudaStreamCreate(writeback)"));
  e = cudaEventCreateWithFlags(&c->copy_gate, cudaEventDisableTiming);
  if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "cudaEventCreate(copy_gate)"));
  c->staged.assign((size_t)c->P, nullptr);
  c->prefetch_pending.assign((size_t)c->P, 0);
  for (int32_t p = 0; p < c->P; ++p) {
    e = cudaEventCreateWithFlags(&c->staged[p], cudaEventDisableTiming);
    if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "cudaEventCreate(staged)"));
  }
  c->ready.assign((size_t)c->P, nullptr);
  c->done.assign((size_t)c->P, nullptr);
  for (int32_t p = 0; p < c->P; ++p) {
    e = cudaEventCreateWithFlags(&c->ready[p], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->done[p], cudaEventDisableTiming);
    if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "cudaEventCreate"));
  }
  e = cudaHostAlloc(reinterpret_cast<void**>(&c->status_host), 3 * sizeof(unsigned long long), cudaHostAllocMapped);
  if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "cudaHostAlloc(status)"));
  c->status_host[0] = ~0ull;
  c->status_host[1] = 0;
  c->status_host[2] = 0;
  e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->status_dev), c->status_host, 0);
  if (e != cudaSuccess) return bail(cuda_fail(nullptr, e, "cudaHostGetDevicePointer"));
  if (id) {  // M = 1 too: a one-rank communicator runs the same paths (tests)
    ncclUniqueId u;
    memcpy(u.internal, id, SD_UNIQUE_ID_BYTES);
    // copy-engine collectives on symmetric windows: the gather takes no SMs
    ncclConfig_t ncfg = NCCL_CONFIG_INITIALIZER;
    ncfg.CTAPolicy = NCCL_CTA_POLICY_ZERO;
    ncclResult_t r = ncclCommInitRankConfig(&c->comm, M, u, rank, &ncfg);
    if (r != ncclSuccess) {
      c->comm = nullptr;
      fail(g_err, SD_ERR_NCCL, "ncclCommInitRank(M=%d, rank=%d): %s", M, rank, ncclGetErrorString(r));
      return bail(SD_ERR_NCCL);
    }
    // the fused gathers address every peer through NVLink (LSA) pointers indexed by rank
    const ncclTeam_t lsa = ncclTeamLsa(c->comm);
    c->lsa_all = lsa.nRanks == M && lsa.rank == rank && M <= 32;
    if (getenv("SD_LOG_INIT"))
      fprintf(stderr, "[libsd] rank %d/%d: NCCL communicator up on device %d (LSA team %d ranks, fused gathers %s)\n",
              rank, M, device, lsa.nRanks, c->lsa_all ? "available" : "off");
  }
  *out = c;
  return SD_OK;
}

namespace {
void release(sd_ctx* c, GatherBuf& b) {
  if (b.nccl) {
    if (b.win) ncclCommWindowDeregister(c->comm, b.win);
    ncclMemFree(b.ptr);
  } else if (b.ptr) {
    cudaFree(b.ptr);
  }
  b = GatherBuf();
}
}  // namespace

sd_status sd_gather_alloc(sd_ctx* c, int64_t n, void** out) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  if (!out) return ctx_fail(c, SD_ERR_ARG, "out pointer is NULL");
  *out = nullptr;
  if (n < 0) return ctx_fail(c, SD_ERR_ARG, "n = %lld is negative", (long long)n);
  SD_CUDA(c, cudaSetDevice(c->device));
  GatherBuf b;
  b.pb = payload_of(&c->cfg, n).bytes;
  // AUTO, from B200 measurements: with tau >= 1 the copy-engine
  // gather hides behind the next kernels; with tau = 0 it is on the critical
  // path and a fused variant wins -- the push at M = 2, the pull at M = 4, 8.
  // The fused modes need every rank in this rank's NVLink (LSA) team and
  // M <= 32 (one flag entry and, in pull mode, one slot pointer per peer);
  // otherwise the copy engines carry the gather.
  int mode = c->gather_mode;
  if (mode == SD_GATHER_AUTO)
    mode = c->cfg.tau > 0 ? SD_GATHER_COPY_ENGINE : ((c->M == 4 || c->M == 8) ? SD_GATHER_PULL : SD_GATHER_PUSH);
  if ((mode == SD_GATHER_PUSH || mode == SD_GATHER_PULL) && !c->lsa_all) mode = SD_GATHER_COPY_ENGINE;
  b.push = c->comm && (mode == SD_GATHER_PUSH || mode == SD_GATHER_PULL);
  b.pull = b.push && mode == SD_GATHER_PULL;
  if (b.push) {
    b.half = (size_t)align_up((int64_t)(b.pb * (size_t)c->M + 16 * (size_t)c->M + 64), 256);
    b.bytes = (size_t)align_up((int64_t)(2 * b.half), 2 << 20);
  } else {
    b.bytes = (size_t)align_up((int64_t)(b.pb * (size_t)c->M), 2 << 20);
  }
  if (c->comm) {
    ncclResult_t r = ncclMemAlloc(&b.ptr, b.bytes);
    if (r != ncclSuccess) return ctx_fail(c, SD_ERR_NCCL, "ncclMemAlloc(%zu): %s", b.bytes, ncclGetErrorString(r));
    if (b.push) {
      // round flags and counters start at 0 (never a round id).  Zeroed BEFORE the
      // collective registration: once any rank returns from it, every rank
      // has finished its memset, so no peer's first push can be overwritten
      cudaError_t e = cudaMemset(b.ptr, 0, b.bytes);
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        ncclMemFree(b.ptr);
        return cuda_fail(c, e, "cudaMemset(gather flags)");
      }
    }
    r = ncclCommWindowRegister(c->comm, b.ptr, b.bytes, &b.win, NCCL_WIN_COLL_SYMMETRIC);
    if (r != ncclSuccess) {
      ncclMemFree(b.ptr);
      return ctx_fail(c, SD_ERR_NCCL, "ncclCommWindowRegister(%zu): %s", b.bytes, ncclGetErrorString(r));
    }
    b.nccl = true;
  } else {
    SD_CUDA(c, cudaMalloc(&b.ptr, b.bytes));
  }
  if (!b.push && c->comm) {
    // one full-size all-gather now: NCCL sets up the symmetric-window
    // copy-engine collective lazily (~0.4 s on the first call), which would
    // otherwise stall the host inside the first sd_fragment_sync
    ncclResult_t r = ncclAllGather(static_cast<char*>(b.ptr) + (size_t)c->rank * b.pb, b.ptr, b.pb, ncclUint8,
                                   c->comm, c->comm_stream);
    if (r != ncclSuccess) {
      release(c, b);
      return ctx_fail(c, SD_ERR_NCCL, "warm-up ncclAllGather: %s", ncclGetErrorString(r));
    }
    const cudaError_t e = cudaStreamSynchronize(c->comm_stream);
    if (e != cudaSuccess) {
      release(c, b);
      return cuda_fail(c, e, "warm-up ncclAllGather");
    }
  }
  c->bufs.push_back(b);
  *out = b.ptr;
  return SD_OK;
}

sd_status sd_gather_payloads(sd_ctx* c, int32_t p, const void* gather_buf, const void** out) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  if (!out) return ctx_fail(c, SD_ERR_ARG, "out pointer is NULL");
  if (p < 0 || p >= c->P) return ctx_fail(c, SD_ERR_ARG, "fragment %d out of range [0, %d)", p, c->P);
  *out = gather_buf;
  GatherBuf* b = find_buf(c, gather_buf);
  if (b && b->push) *out = static_cast<const char*>(b->ptr) + (size_t)(c->round_seq[p] & 1) * b->half;
  return SD_OK;
}

sd_status sd_set_gather_mode(sd_ctx* c, int32_t mode) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  if (mode != SD_GATHER_COPY_ENGINE && mode != SD_GATHER_PUSH && mode != SD_GATHER_AUTO && mode != SD_GATHER_PULL)
    return ctx_fail(c, SD_ERR_ARG, "gather mode %d is not SD_GATHER_COPY_ENGINE, _PUSH, _PULL or _AUTO", mode);
  for (const Inflight& f : c->fl)
    if (f.state != IDLE) return ctx_fail(c, SD_ERR_STATE, "gather mode changed while a fragment is in flight");
  c->gather_mode = mode;
  return SD_OK;
}

sd_status sd_gather_free(sd_ctx* c, void* gather_buf) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  for (size_t i = 0; i < c->bufs.size(); ++i) {
    if (c->bufs[i].ptr == gather_buf) {
      SD_CUDA(c, cudaSetDevice(c->device));
      SD_CUDA(c, cudaDeviceSynchronize());
      release(c, c->bufs[i]);
      c->bufs.erase(c->bufs.begin() + (long)i);
      return SD_OK;
    }
  }
  return ctx_fail(c, SD_ERR_ARG, "gather_buf %p was not allocated by sd_gather_alloc on this ctx", gather_buf);
}

sd_status sd_state_prefetch(sd_ctx* c, int32_t p, const float* anchor_host, const float* momentum_host,
                            float* anchor, float* momentum, int64_t n, sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  sd_status st;
  if ((st = check_fragment(c, p, 1, n))) return st;
  if (c->fl[p].state != IDLE)
    return ctx_fail(c, SD_ERR_STATE, "fragment %d is in flight: its outer state is in use", p);
  if (n == 0) return SD_OK;
  if ((st = check_ptr(c, anchor_host, 4, "anchor_host")) || (st = check_ptr(c, momentum_host, 4, "momentum_host")) ||
      (st = check_ptr(c, anchor, 32, "anchor")) || (st = check_ptr(c, momentum, 32, "momentum")))
    return st;
  SD_CUDA(c, cudaSetDevice(c->device));
  // the staging slot is free once `stream`'s prior work (the last user of the slot) is done
  // and the last writeback out of it has finished
  SD_CUDA(c, cudaEventRecord(c->copy_gate, static_cast<cudaStream_t>(stream)));
  SD_CUDA(c, cudaStreamWaitEvent(c->copy_stream, c->copy_gate, 0));
  for (const sd_ctx::Drain& d : c->drains)
    if (d.staging == anchor || d.staging == momentum) SD_CUDA(c, cudaStreamWaitEvent(c->copy_stream, d.ev, 0));
  SD_CUDA(c, cudaMemcpyAsync(anchor, anchor_host, 4 * (size_t)n, cudaMemcpyHostToDevice, c->copy_stream));
  SD_CUDA(c, cudaMemcpyAsync(momentum, momentum_host, 4 * (size_t)n, cudaMemcpyHostToDevice, c->copy_stream));
  SD_CUDA(c, cudaEventRecord(c->staged[p], c->copy_stream));
  c->prefetch_pending[p] = 1;
  return SD_OK;
}

sd_status sd_state_writeback(sd_ctx* c, int32_t p, const float* anchor, const float* momentum, float* anchor_host,
                             float* momentum_host, int64_t n, sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  sd_status st;
  if ((st = check_fragment(c, p, 1, n))) return st;
  if (c->fl[p].state != IDLE)
    return ctx_fail(c, SD_ERR_STATE, "fragment %d is in flight: merge it before writing its state back", p);
  if (n == 0) return SD_OK;
  if ((st = check_ptr(c, anchor_host, 4, "anchor_host")) || (st = check_ptr(c, momentum_host, 4, "momentum_host")) ||
      (st = check_ptr(c, anchor, 32, "anchor")) || (st = check_ptr(c, momentum, 32, "momentum")))
    return st;
  SD_CUDA(c, cudaSetDevice(c->device));
  SD_CUDA(c, cudaEventRecord(c->copy_gate, static_cast<cudaStream_t>(stream)));  // after the merge
  SD_CUDA(c, cudaStreamWaitEvent(c->wb_stream, c->copy_gate, 0));
  // a writeback of host buffers that a prefetch is still reading must not overtake it
  SD_CUDA(c, cudaEventRecord(c->copy_gate, c->copy_stream));
  SD_CUDA(c, cudaStreamWaitEvent(c->wb_stream, c->copy_gate, 0));
  SD_CUDA(c, cudaMemcpyAsync(anchor_host, anchor, 4 * (size_t)n, cudaMemcpyDeviceToHost, c->wb_stream));
  SD_CUDA(c, cudaMemcpyAsync(momentum_host, momentum, 4 * (size_t)n, cudaMemcpyDeviceToHost, c->wb_stream));
  sd_ctx::Drain* d = nullptr;
  for (sd_ctx::Drain& x : c->drains)
    if (x.staging == anchor) d = &x;
  if (!d) {
    c->drains.push_back({anchor, nullptr});
    d = &c->drains.back();
    SD_CUDA(c, cudaEventCreateWithFlags(&d->ev, cudaEventDisableTiming));
  }
  SD_CUDA(c, cudaEventRecord(d->ev, c->wb_stream));
  return SD_OK;
}

sd_status sd_state_sync(sd_ctx* c, sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  SD_CUDA(c, cudaSetDevice(c->device));
  SD_CUDA(c, cudaEventRecord(c->copy_gate, c->copy_stream));
  SD_CUDA(c, cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), c->copy_gate, 0));
  SD_CUDA(c, cudaEventRecord(c->copy_gate, c->wb_stream));
  SD_CUDA(c, cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), c->copy_gate, 0));
  return SD_OK;
}

sd_status sd_comm_stream(sd_ctx* c, sd_stream* out) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  if (!out) return ctx_fail(c, SD_ERR_ARG, "out pointer is NULL");
  *out = static_cast<sd_stream>(c->comm_stream);
  return SD_OK;
}

sd_status sd_outer_state_init(sd_ctx* c, const float* theta, float* anchor, float* momentum, int64_t n,
                              sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  if (n < 0) return ctx_fail(c, SD_ERR_ARG, "n = %lld is negative", (long long)n);
  if (n == 0) return SD_OK;
  sd_status st;
  if ((st = check_ptr(c, theta, 32, "theta")) || (st = check_ptr(c, anchor, 32, "anchor")) ||
      (st = check_ptr(c, momentum, 32, "momentum")))
    return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SD_CUDA(c, cudaSetDevice(c->device));
  if (anchor != theta) SD_CUDA(c, cudaMemcpyAsync(anchor, theta, 4 * (size_t)n, cudaMemcpyDeviceToDevice, s));
  SD_CUDA(c, cudaMemsetAsync(momentum, 0, 4 * (size_t)n, s));
  return SD_OK;
}

namespace {

// Push / pull modes: where this round's payloads live and the send side of the protocol.
struct PushRound {
  GatherBuf* buf = nullptr;
  size_t half_off = 0;
  uint64_t seq = 0;
  bool pull = false;
  sdk::Round round;
};

sd_status push_round(sd_ctx* c, int32_t p, void* slot_out, const sdk::Payload& pl, PushRound* r) {
  GatherBuf* b = find_buf(c, slot_out);
  if (!b || !b->push) return SD_OK;
  if (b->pb != pl.bytes) return ctx_fail(c, SD_ERR_ARG, "gather buffer was allocated for payloads of %zu bytes, not %zu", b->pb, pl.bytes);
  if (static_cast<char*>(slot_out) != static_cast<char*>(b->ptr) + (size_t)c->rank * pl.bytes)
    return ctx_fail(c, SD_ERR_ARG, "slot_out must be gather_buf + rank * payload");
  r->seq = c->round_seq[p] + 1;  // this send's round id (identical on every rank: same call sequence)
  r->buf = b;
  r->half_off = (size_t)(r->seq & 1) * b->half;
  r->pull = b->pull;
  r->round.win = b->win;
  r->round.win_off = r->half_off + (size_t)c->rank * pl.bytes;
  r->round.flags_off = r->half_off + b->flags_rel(c->M);
  r->round.counter = reinterpret_cast<unsigned int*>(static_cast<char*>(b->ptr) + r->half_off + b->counter_rel(c->M));
  r->round.seq = r->seq;
  r->round.rank = c->rank;
  r->round.M = c->M;
  r->round.push = !b->pull;
  return SD_OK;
}

// The payload's local slot: this round's half in push / pull modes.
uint8_t* local_slot(sd_ctx* c, void* slot_out, const PushRound& pr, const sdk::Payload& pl) {
  if (!pr.buf) return static_cast<uint8_t*>(slot_out);
  return static_cast<uint8_t*>(pr.buf->ptr) + pr.half_off + (size_t)c->rank * pl.bytes;
}

// A bounded block-receive timed out earlier (sticky): the replicas' outer
// state may have diverged, so every later device call is refused.
sd_status check_alive(sd_ctx* c) {
  if (!c->dead && c->status_host && *reinterpret_cast<volatile unsigned long long*>(c->status_host + 2) != 0)
    c->dead = true;
  if (c->dead)
    return ctx_fail(c, SD_ERR_STATE,
                    "a block-receive timed out on this context: the replicas' outer state may differ; "
                    "re-initialize every replica from a common state (sd_finalize + sd_init)");
  return SD_OK;
}

sd_status begin_send(sd_ctx* c, int32_t p, int64_t t, const float* theta, const float* anchor, int64_t n,
                     void* slot_out, cudaStream_t s, sdk::Payload* pl, PushRound* pr) {
  sd_status st;
  if ((st = check_fragment(c, p, t, n))) return st;
  if ((st = check_alive(c))) return st;
  if ((c->cfg.T == 0 || t <= c->cfg.T) ? !sends_at(&c->cfg, p, t) : true)
    return ctx_fail(c, SD_ERR_SCHEDULE, "fragment %d is not scheduled to send at step %lld (t_p = %d, H = %d)", p,
                    (long long)t, offset_of(&c->cfg, p), c->cfg.H);
  if (c->fl[p].state != IDLE)
    return ctx_fail(c, SD_ERR_STATE, "fragment %d is still in flight (sent at step %lld)", p,
                    (long long)c->fl[p].send_step);
  if ((st = check_ptr(c, slot_out, 256, "slot_out"))) return st;
  if (n > 0 && ((st = check_ptr(c, theta, 32, "theta")) || (st = check_ptr(c, anchor, 32, "anchor")))) return st;
  *pl = payload_of(&c->cfg, n);
  if ((st = push_round(c, p, slot_out, *pl, pr))) return st;
  SD_CUDA(c, cudaSetDevice(c->device));
  if (c->prefetch_pending[p]) {  // offloaded outer state: the anchor must have landed
    SD_CUDA(c, cudaStreamWaitEvent(s, c->staged[p], 0));
    c->prefetch_pending[p] = 0;
  }
  SD_CUDA(c, cudaMemsetAsync(local_slot(c, slot_out, *pr, *pl) + pl->trailer_off + 8, 0xFF, 8, s));  // first_bad = 2^64-1
  return SD_OK;
}

sd_status end_send(sd_ctx* c, int32_t p, int64_t t, int64_t n, void* slot_out, const PushRound& pr) {
  if (pr.buf) c->round_seq[p] = pr.seq;  // the kernel's last CTA has signalled the peers
  c->fl[p].state = QUANTIZED;
  c->fl[p].send_step = t;
  c->fl[p].n = n;
  c->fl[p].slot = slot_out;
  c->fl[p].push = pr.buf != nullptr;
  c->fl[p].pull = pr.pull;
  c->fl[p].waited = false;
  c->fl[p].half_off = pr.half_off;
  c->fl[p].seq = pr.seq;
  return SD_OK;
}

sd_status adam_hyper(sd_ctx* c, int64_t k, const sd_adamw* hp, sdk::AdamHyper* h) {
  if (!hp) return ctx_fail(c, SD_ERR_ARG, "adamw hyper-parameter pointer is NULL");
  if (k < 1) return ctx_fail(c, SD_ERR_ARG, "AdamW step k = %lld must be >= 1", (long long)k);
  if (!(hp->beta1 >= 0.0f && hp->beta1 < 1.0f) || !(hp->beta2 >= 0.0f && hp->beta2 < 1.0f))
    return ctx_fail(c, SD_ERR_CONFIG, "beta1 %g / beta2 %g not in [0, 1)", (double)hp->beta1, (double)hp->beta2);
  if (!(hp->eps > 0.0f) || !(hp->lr == hp->lr) || !(hp->weight_decay == hp->weight_decay))
    return ctx_fail(c, SD_ERR_CONFIG, "eps %g must be > 0, lr %g and weight_decay %g finite", (double)hp->eps,
                    (double)hp->lr, (double)hp->weight_decay);
  // constants of the op order (oracle or_adamw): bias corrections in binary64, rounded once
  const float bc1 = (float)(1.0 - pow((double)hp->beta1, (double)k));
  const float bc2 = (float)(1.0 - pow((double)hp->beta2, (double)k));
  volatile float lw = hp->lr * hp->weight_decay;  // no contraction into 1 - lr*wd
  h->b1 = hp->beta1;
  h->b2 = hp->beta2;
  h->c1 = 1.0f - hp->beta1;
  h->c2 = 1.0f - hp->beta2;
  h->decay = 1.0f - lw;
  h->step = hp->lr / bc1;
  h->sbc2 = sqrtf(bc2);
  h->eps = hp->eps;
  return SD_OK;
}

}  // namespace

size_t sd_quantize_workspace_bytes(const sd_config* cfg, int64_t n) {
  if (!cfg || validate(cfg, nullptr, 0) != SD_OK || n <= 0) return 0;
  const int32_t B = cfg->scale_block;
  if (B == 256 || B == 512 || B == 1024) return 0;  // single pass: no scratch
  return sdk::stage_bytes(n);
}

sd_status sd_set_workspace(sd_ctx* c, void* ws, size_t bytes) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  if (ws == nullptr || bytes == 0) {
    c->ws = sdk::Workspace();
    return SD_OK;
  }
  sd_status st;
  if ((st = check_ptr(c, ws, 256, "workspace"))) return st;
  c->ws.ptr = static_cast<uint8_t*>(ws);
  c->ws.bytes = bytes;
  return SD_OK;
}

sd_status sd_outer_grad_quantize(sd_ctx* c, int32_t p, int64_t t, const float* theta, const float* anchor,
                                 int64_t n, void* slot_out, sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  sdk::Payload pl;
  PushRound pr;
  sd_status st = begin_send(c, p, t, theta, anchor, n, slot_out, s, &pl, &pr);
  if (st != SD_OK) return st;
  const int k =
      sdk::launch_quantize(theta, anchor, pl, local_slot(c, slot_out, pr, pl), pr.round, c->num_sms, s, c->ws);
  if (k < 0) return cuda_fail(c, cudaGetLastError(), "k_quantize launch");
  g_launches += (uint64_t)k;
  return end_send(c, p, t, n, slot_out, pr);
}

sd_status sd_inner_adamw(sd_ctx* c, int64_t k, float* theta, const float* grad, float* m, float* v, int64_t n,
                         const sd_adamw* hp, sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  if (n < 0) return ctx_fail(c, SD_ERR_ARG, "n = %lld is negative", (long long)n);
  sdk::AdamHyper h;
  sd_status st = adam_hyper(c, k, hp, &h);
  if (st != SD_OK) return st;
  if (n == 0) return SD_OK;
  if ((st = check_ptr(c, theta, 32, "theta")) || (st = check_ptr(c, grad, 32, "grad")) ||
      (st = check_ptr(c, m, 32, "m")) || (st = check_ptr(c, v, 32, "v")))
    return st;
  SD_CUDA(c, cudaSetDevice(c->device));
  const int kl = sdk::launch_adamw(theta, grad, m, v, n, h, c->num_sms, static_cast<cudaStream_t>(stream));
  if (kl < 0) return cuda_fail(c, cudaGetLastError(), "k_adamw launch");
  g_launches += (uint64_t)kl;
  return SD_OK;
}

sd_status sd_inner_adamw_quantize(sd_ctx* c, int32_t p, int64_t t, int64_t k, float* theta, const float* grad,
                                  float* m, float* v, const float* anchor, int64_t n, void* slot_out,
                                  const sd_adamw* hp, sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  sdk::AdamHyper h;
  sd_status st = adam_hyper(c, k, hp, &h);
  if (st != SD_OK) return st;
  if (n > 0 && ((st = check_ptr(c, grad, 32, "grad")) || (st = check_ptr(c, m, 32, "m")) ||
                (st = check_ptr(c, v, 32, "v"))))
    return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  sdk::Payload pl;
  PushRound pr;
  st = begin_send(c, p, t, theta, anchor, n, slot_out, s, &pl, &pr);
  if (st != SD_OK) return st;
  const int kl = sdk::launch_adamw_quantize(theta, grad, m, v, anchor, pl, local_slot(c, slot_out, pr, pl), h,
                                            pr.round, c->num_sms, s, c->ws);
  if (kl < 0) return cuda_fail(c, cudaGetLastError(), "k_adamw_quantize launch");
  g_launches += (uint64_t)kl;
  return end_send(c, p, t, n, slot_out, pr);
}

sd_status sd_fragment_sync(sd_ctx* c, int32_t p, int64_t t, void* gather_buf, int64_t n, sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  sd_status st;
  if ((st = check_fragment(c, p, t, n))) return st;
  Inflight& f = c->fl[p];
  if (f.state != QUANTIZED || f.send_step != t)
    return ctx_fail(c, SD_ERR_STATE, "fragment %d: sync at step %lld without a quantize at that step", p, (long long)t);
  if (f.n != n) return ctx_fail(c, SD_ERR_ARG, "fragment %d: n = %lld but quantized n = %lld", p, (long long)n, (long long)f.n);
  if ((st = check_ptr(c, gather_buf, 256, "gather_buf"))) return st;
  const sdk::Payload pl = payload_of(&c->cfg, n);
  uint8_t* g = static_cast<uint8_t*>(gather_buf);
  if (f.slot != g + (size_t)c->rank * pl.bytes)
    return ctx_fail(c, SD_ERR_ARG, "slot_out %p != gather_buf + rank * payload (%p + %d * %zu)", f.slot, gather_buf,
                    c->rank, pl.bytes);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  SD_CUDA(c, cudaSetDevice(c->device));
  if ((st = check_alive(c))) return st;
  if (f.push) {  // push: the quantize stored the payload into the peers; pull: the apply reads it
    SD_CUDA(c, cudaEventRecord(c->done[p], s));
  } else if (c->comm) {
    SD_CUDA(c, cudaEventRecord(c->ready[p], s));
    SD_CUDA(c, cudaStreamWaitEvent(c->comm_stream, c->ready[p], 0));
    ncclResult_t r = ncclAllGather(g + (size_t)c->rank * pl.bytes, g, pl.bytes, ncclUint8, c->comm, c->comm_stream);
    if (r != ncclSuccess) return ctx_fail(c, SD_ERR_NCCL, "ncclAllGather(fragment %d): %s", p, ncclGetErrorString(r));
    SD_CUDA(c, cudaEventRecord(c->done[p], c->comm_stream));
  } else {
    SD_CUDA(c, cudaEventRecord(c->done[p], s));
  }
  f.state = SYNCED;
  f.gather = gather_buf;
  return SD_OK;
}

namespace {
// Bound of the block-receive wait on the peers' round flags (push / pull
// modes): SD_WAIT_TIMEOUT_MS (read once per process), 0 or unset = no bound.
uint64_t wait_timeout_ns() {
  static int64_t ns = -1;
  if (ns < 0) {
    const char* e = getenv("SD_WAIT_TIMEOUT_MS");
    const long long ms = e ? atoll(e) : 0;
    ns = ms > 0 ? (int64_t)ms * 1000000ll : 0;
  }
  return (uint64_t)ns;
}

// The receive side of this round (push / pull modes).
sdk::RoundRecv round_recv(sd_ctx* c, const Inflight& f, GatherBuf* b) {
  sdk::RoundRecv rr;
  const sdk::Payload pl = payload_of(&c->cfg, f.n);
  uint8_t* half = static_cast<uint8_t*>(b->ptr) + f.half_off;
  rr.flags = reinterpret_cast<const unsigned long long*>(half + b->flags_rel(c->M));
  rr.own = half + (size_t)c->rank * pl.bytes;
  rr.verdict = reinterpret_cast<unsigned long long*>(half + b->verdict_rel(c->M));
  rr.seq = f.seq;
  rr.rank = c->rank;
  rr.pull = f.pull;
  rr.win = b->win;
  rr.half_off = f.half_off;
  rr.flags_off = f.half_off + b->flags_rel(c->M);
  return rr;
}

// block-receive of the fused gathers: one k_round_wait per round
sd_status issue_round_wait(sd_ctx* c, int32_t p, cudaStream_t s) {
  Inflight& f = c->fl[p];
  if (!f.push || f.waited) return SD_OK;
  GatherBuf* b = find_buf(c, f.gather);
  if (!b) return ctx_fail(c, SD_ERR_STATE, "fragment %d: push/pull-mode gather buffer not found", p);
  const sdk::RoundRecv rr = round_recv(c, f, b);
  const int k = sdk::launch_round_wait(rr, payload_of(&c->cfg, f.n), c->M, wait_timeout_ns(), c->status_dev, s);
  if (k < 0) return cuda_fail(c, cudaGetLastError(), "k_round_wait launch");
  g_launches += (uint64_t)k;
  f.waited = true;
  return SD_OK;
}
}  // namespace

sd_status sd_fragment_wait(sd_ctx* c, int32_t p, int64_t t, sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  sd_status st;
  if ((st = check_fragment(c, p, t, 0))) return st;
  const int64_t s_step = receive_send_step(&c->cfg, p, t);
  if (s_step == 0)
    return ctx_fail(c, SD_ERR_SCHEDULE, "fragment %d is not scheduled to be received at step %lld (tau = %d)", p,
                    (long long)t, c->cfg.tau);
  if (c->fl[p].state != SYNCED || c->fl[p].send_step != s_step)
    return ctx_fail(c, SD_ERR_STATE, "fragment %d: wait at step %lld needs the sync of step %lld first", p,
                    (long long)t, (long long)s_step);
  if ((st = check_alive(c))) return st;
  SD_CUDA(c, cudaSetDevice(c->device));
  SD_CUDA(c, cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), c->done[p], 0));
  return issue_round_wait(c, p, static_cast<cudaStream_t>(stream));
}

namespace {
sd_status do_merge(sd_ctx* c, int32_t p, int64_t t, const void* gather_buf, float* theta, float* anchor,
                   float* momentum, int64_t n, cudaStream_t s, const sdk::AdamInner* inner) {
  sd_status st;
  if ((st = check_fragment(c, p, t, n))) return st;
  const int64_t s_step = receive_send_step(&c->cfg, p, t);
  if (s_step == 0)
    return ctx_fail(c, SD_ERR_SCHEDULE, "fragment %d is not scheduled to be received at step %lld (tau = %d)", p,
                    (long long)t, c->cfg.tau);
  Inflight& f = c->fl[p];
  if (f.state != SYNCED || f.send_step != s_step)
    return ctx_fail(c, SD_ERR_STATE, "fragment %d: merge at step %lld needs the sync of step %lld first", p,
                    (long long)t, (long long)s_step);
  if (f.n != n) return ctx_fail(c, SD_ERR_ARG, "fragment %d: n = %lld but synced n = %lld", p, (long long)n, (long long)f.n);
  if (f.gather != gather_buf)
    return ctx_fail(c, SD_ERR_ARG, "fragment %d: gather_buf %p is not the synced buffer %p", p, gather_buf, f.gather);
  if ((st = check_alive(c))) return st;
  if (n > 0 && ((st = check_ptr(c, theta, 32, "theta")) || (st = check_ptr(c, anchor, 32, "anchor")) ||
                (st = check_ptr(c, momentum, 32, "momentum"))))
    return st;
  if (c->comm && !f.push) {  // a failed gather must not be merged (polled here and in sd_check)
    ncclResult_t ar = ncclSuccess;
    const ncclResult_t r = ncclCommGetAsyncError(c->comm, &ar);
    if (r != ncclSuccess || ar != ncclSuccess)
      return ctx_fail(c, SD_ERR_NCCL, "fragment %d: NCCL async error before the merge: %s", p,
                      ncclGetErrorString(r != ncclSuccess ? r : ar));
  }
  const sdk::Payload pl = payload_of(&c->cfg, n);
  SD_CUDA(c, cudaSetDevice(c->device));
  SD_CUDA(c, cudaStreamWaitEvent(s, c->done[p], 0));  // block-receive (Alg. 2 L11)
  if ((st = issue_round_wait(c, p, s))) return st;
  const uint8_t* payloads = static_cast<const uint8_t*>(gather_buf) + (f.push ? f.half_off : 0);
  sdk::RoundRecv rr;
  if (f.push) {
    GatherBuf* b = find_buf(c, gather_buf);
    if (!b) return ctx_fail(c, SD_ERR_STATE, "fragment %d: push/pull-mode gather buffer not found", p);
    rr = round_recv(c, f, b);
  }
  const int k = sdk::launch_apply(payloads, pl, c->M, theta, anchor, momentum, c->cfg.outer_lr,
                                  c->cfg.outer_momentum, c->cfg.alpha, c->status_dev, c->num_sms, s, inner,
                                  f.push ? &rr : nullptr);
  if (k < 0) return cuda_fail(c, cudaGetLastError(), "k_apply launch");
  g_launches += (uint64_t)k;
  f = Inflight();
  return SD_OK;
}
}  // namespace

sd_status sd_merge(sd_ctx* c, int32_t p, int64_t t, const void* gather_buf, float* theta, float* anchor,
                   float* momentum, int64_t n, sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  return do_merge(c, p, t, gather_buf, theta, anchor, momentum, n, static_cast<cudaStream_t>(stream), nullptr);
}

sd_status sd_inner_adamw_merge(sd_ctx* c, int32_t p, int64_t t, int64_t k, float* theta, const float* grad,
                               float* m, float* v, const void* gather_buf, float* anchor, float* momentum,
                               int64_t n, const sd_adamw* hp, sd_stream stream) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  sdk::AdamInner in;
  sd_status st = adam_hyper(c, k, hp, &in.hp);
  if (st != SD_OK) return st;
  if (n > 0 && ((st = check_ptr(c, grad, 32, "grad")) || (st = check_ptr(c, m, 32, "m")) ||
                (st = check_ptr(c, v, 32, "v"))))
    return st;
  in.grad = grad;
  in.m = m;
  in.v = v;
  return do_merge(c, p, t, gather_buf, theta, anchor, momentum, n, static_cast<cudaStream_t>(stream), &in);
}

sd_status sd_check(sd_ctx* c, int64_t* first_bad_index) {
  if (!c) return fail(g_err, SD_ERR_ARG, "ctx is NULL");
  if (first_bad_index) *first_bad_index = -1;
  SD_CUDA(c, cudaSetDevice(c->device));
  SD_CUDA(c, cudaDeviceSynchronize());
  if (c->comm) {
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(c->comm, &ar);
    if (r != ncclSuccess || ar != ncclSuccess)
      return ctx_fail(c, SD_ERR_NCCL, "NCCL async error: %s", ncclGetErrorString(r != ncclSuccess ? r : ar));
  }
  volatile unsigned long long* h = c->status_host;
  const unsigned long long code = h[1], fb = h[0];
  if (h[2] != 0) c->dead = true;
  if (code != 0) {
    if (code != 3) {  // a timeout stays reported (sticky)
      h[0] = ~0ull;
      h[1] = 0;
    }
    if (first_bad_index) *first_bad_index = fb == ~0ull ? -1 : (int64_t)fb;
    if (code == 3)
      return ctx_fail(c, SD_ERR_STATE,
                      "a block-receive timed out (a peer missed its round flag for SD_WAIT_TIMEOUT_MS); the round "
                      "was skipped here and this context refuses further device calls");
    if (code == 2) return ctx_fail(c, SD_ERR_STATE, "a gather slot had no valid payload trailer; round skipped");
    return ctx_fail(c, SD_ERR_NONFINITE, "non-finite outer gradient at fragment index %llu; round skipped", fb);
  }
  return SD_OK;
}

const char* sd_last_error(const sd_ctx* c) { return c ? c->err : g_err; }

sd_status sd_finalize(sd_ctx* c) {
  if (!c) return SD_OK;
  cudaSetDevice(c->device);
  if (!c->bufs.empty() || c->ws.ptr) cudaDeviceSynchronize();  // before the caller may free the workspace
  for (GatherBuf& b : c->bufs) release(c, b);
  c->bufs.clear();
  if (c->comm) {
    ncclCommDestroy(c->comm);
    c->comm = nullptr;
  }
  for (cudaEvent_t e : c->ready)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->done)
    if (e) cudaEventDestroy(e);
  if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->wb_stream) cudaStreamDestroy(c->wb_stream);
  for (sd_ctx::Drain& d : c->drains)
    if (d.ev) cudaEventDestroy(d.ev);
  for (cudaEvent_t e : c->staged)
    if (e) cudaEventDestroy(e);
  if (c->copy_gate) cudaEventDestroy(c->copy_gate);
  if (c->status_host) cudaFreeHost(c->status_host);
  delete c;
  return SD_OK;
}

uint64_t sd_kernel_launch_count(void) { return g_launches.load(); }

}  // extern "C"
