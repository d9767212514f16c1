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

// Send side of the fused all-gather (push and pull modes; win == nullptr:
// copy-engine mode or no communicator -- the payload is only written locally).
// The kernel that finishes the payload also signals the round from its last
// CTA: {round id seq, first non-finite index} release-stored into entry
// `rank` of every peer's flag array (window offset flags_off).  push: every
// payload word is also stored into this rank's slot of each peer's buffer
// (window offset win_off) as it is produced.
struct Round {
  ncclWindow_t win = nullptr;
  size_t win_off = 0;
  size_t flags_off = 0;
  unsigned int* counter = nullptr;  // last-CTA ticket, 0 between launches
  uint64_t seq = 0;
  int rank = 0, M = 1;
  bool push = false;
};

// Caller workspace of the two-pass quantize (B = 0 or B > 1024): with at
// least stage_bytes(n) bytes (256-aligned) pass 1 leaves 16-bit summaries of
// the Deltas there and pass 2 encodes from them instead of re-reading theta
// and A.  Empty: pass 2 re-reads.
struct Workspace {
  uint8_t* ptr = nullptr;
  size_t bytes = 0;
};
size_t stage_bytes(int64_t n);

// Delta = anchor - theta, per-block absmax, exact E3M0, nibble pack, trailer
// (+ the round signal).  slot: one payload (256-aligned).  The trailer's
// first_bad word must hold 2^64-1 before the launch (sd_outer_grad_quantize
// memsets it).  Returns the number of kernels launched, or -1.
int launch_quantize(const float* theta, const float* anchor, const Payload& pl, uint8_t* slot, const Round& rd,
                    int num_sms, cudaStream_t st, const Workspace& ws = Workspace());

// Receive side of the fused all-gather: this half's flag entries (local),
// this rank's own slot, and in pull mode the window to reach the peers'
// slots (slot m at window offset half_off + m * payload of rank m).
// verdict: where k_round_wait writes its decision for the round (local).
struct RoundRecv {
  const unsigned long long* flags = nullptr;
  const uint8_t* own = nullptr;
  unsigned long long* verdict = nullptr;
  uint64_t seq = 0;
  int rank = 0;
  bool pull = false;
  ncclWindow_t win = nullptr;
  size_t half_off = 0;
  size_t flags_off = 0;
};

// Block-receive of the fused gathers: waits for every peer's flag entry
// (at most timeout_ns; 0 = no bound), writes rr.verdict {first_bad, code}; on
// a timeout status[1] = 3, status[2] = 1 (sticky) and the peers are told.
int launch_round_wait(const RoundRecv& rr, const Payload& pl, int M, uint64_t timeout_ns, unsigned long long* status,
                      cudaStream_t st);

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
// (single pass for B in {256, 512, 1024}; otherwise AdamW fused with the first
// pass -- the block max -- then k_encode).
int launch_adamw_quantize(float* theta, const float* grad, float* m, float* v, const float* anchor, const Payload& pl,
                          uint8_t* slot, const AdamHyper& hp, const Round& rd, int num_sms, cudaStream_t st,
                          const Workspace& ws = Workspace());

// Fused decode + M-way fp32 mean + Nesterov + anchor update + alpha-merge.
// status: host-mapped pinned words {first_bad, code, dead} (code written
// when the round is skipped).  rr: push / pull modes (null: copy-engine or
// local slots at gather + m * payload).  Returns kernels launched or -1.
// inner: optional AdamW step applied to theta first (the step's inner update
// fused with the receive; theta is read and written once).
struct AdamInner {
  const float* grad;
  float* m;
  float* v;
  AdamHyper hp;
};
int launch_apply(const uint8_t* gather, const Payload& pl, int M, float* theta, float* anchor,
                 float* momentum, float lr, float mu, float alpha, unsigned long long* status,
                 int num_sms, cudaStream_t st, const AdamInner* inner = nullptr, const RoundRecv* rr = nullptr);

}  // namespace sdk
