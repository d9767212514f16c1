// sd_kernels.h — launchers of libsd's sm_100a kernels (internal to libsd).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

namespace sdk {

struct Payload {          // byte offsets inside one replica payload (sd.h)
  int64_t n;              // fragment elements
  int64_t nb;             // scale blocks
  int32_t B;              // elements per scale block (0 = whole fragment)
  size_t scales_off;      // align256(ceil(n/2))
  size_t trailer_off;     // scales_off + align16(4 nb)
  size_t bytes;           // total payload bytes
};

// Push mode (fused all-gather): the quantize also stores every payload word
// into this rank's slot of each peer's gather buffer through the NCCL
// symmetric window `win` (window offset win_off).  win == nullptr: local only.
struct Push {
  ncclWindow_t win = nullptr;
  size_t win_off = 0;
  int rank = 0, M = 1;
};

// Delta = anchor - theta, per-block absmax, exact E3M0, nibble pack, trailer.
// slot: one payload (256-aligned).  The trailer's first_bad word must hold
// 2^64-1 before the launch (sd_outer_grad_quantize memsets it).
// Returns the number of kernels launched, or -1 on a launch error.
int launch_quantize(const float* theta, const float* anchor, const Payload& pl, uint8_t* slot,
                    const Push& push, int num_sms, cudaStream_t st);

// Push mode completion: publish first_bad to the peers, fence, release-store
// the round id into flags[rank] of every peer (window offset flags_off).
int launch_push_signal(const Payload& pl, uint8_t* slot, const Push& push, size_t flags_off, uint64_t t,
                       cudaStream_t st);

// Push mode block-receive: acquire-wait until every peer's flag == the round id t (at most
// timeout_ns, then the peer's slot is invalidated and status[1] = 2).
int launch_push_wait(const unsigned long long* flags, uint8_t* half, const Payload& pl, int M, int rank, uint64_t t,
                     uint64_t timeout_ns, unsigned long long* status, cudaStream_t st);

// Multicast gather (SD_GATHER_MULTICAST): the copy engine writes this rank's
// payload once through the window's NVLS multicast alias and NVSwitch
// delivers it to every rank's slot.  McState wraps the NCCL device
// communicator that owns the LSA-team multimem handle.
struct McState;
// Collective (all ranks, same order).  Returns 1 and *out on success, 0 if the
// system has no multicast (no NVLS), -1 on an NCCL error.
int mc_create(ncclComm_t comm, McState** out);
void mc_destroy(ncclComm_t comm, McState* s);
// Device address of byte 0 of window `win` in the multicast space (the
// alias is linear in the window offset).  Synchronizes `st`.
int mc_base(McState* s, ncclWindow_t win, uint8_t** out, cudaStream_t st);
// Release-store the round id t into flags[rank] of every peer (window offset
// flags_off) after a system-scope fence: ordered after the stream's prior
// work, i.e. after the multicast copy has landed everywhere.
int launch_flag_signal(ncclWindow_t win, size_t flags_off, int rank, int M, uint64_t t, cudaStream_t st);

// AdamW hyper-parameters with the host-side constants of the op order
// (bias corrections in binary64 rounded once, DESIGN.md AMB-20).
struct AdamHyper {
  float b1, b2, c1, c2;  // beta1, beta2, 1 - beta1, 1 - beta2
  float decay;           // 1 - lr * wd
  float step;            // lr / bc1
  float sbc2;            // sqrt(bc2)
  float eps;
};

// One AdamW inner step over n elements (theta, m, v in place).
int launch_adamw(float* theta, const float* grad, float* m, float* v, int64_t n, const AdamHyper& hp, int num_sms,
                 cudaStream_t st);

// AdamW step fused with Delta + E3M0 of the updated theta into one payload
// (single pass for B in {256, 512, 1024}; AdamW + two-pass quantize otherwise).
int launch_adamw_quantize(float* theta, const float* grad, float* m, float* v, const float* anchor, const Payload& pl,
                          uint8_t* slot, const AdamHyper& hp, const Push& push, int num_sms, cudaStream_t st);

// Fused decode + M-way fp32 mean + Nesterov + anchor update + alpha-merge.
// status: host-mapped pinned word pair {first_bad, flags} written when the
// round is skipped.  Returns kernels launched or -1.
// inner: optional AdamW step applied to theta first (the step's inner update
// fused with the receive; theta is read and written once).
struct AdamInner {
  const float* grad;
  float* m;
  float* v;
  AdamHyper hp;
};
// Pull mode: slot m != rank is read from rank m's own buffer over NVLink
// (symmetric window, LSA pointers) at window offset half_off + m * payload.
struct Pull {
  ncclWindow_t win = nullptr;
  size_t half_off = 0;
  int rank = 0;
};
int launch_apply(const uint8_t* gather, const Payload& pl, int M, float* theta, float* anchor,
                 float* momentum, float lr, float mu, float alpha, unsigned long long* status,
                 int num_sms, cudaStream_t st, const AdamInner* inner = nullptr, const Pull* pull = nullptr);

}  // namespace sdk
