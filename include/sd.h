/* sd.h — C ABI of libsd, the B200-native per-fragment outer synchronization of
 * Streaming DiLoCo (arXiv 2501.18512).  ABI version 1.
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n (the reference
 * paper text and the CPU-program spec written from it); AMB-k = a reading of
 * the paper recorded in DESIGN.md §2.
 *
 * The method (Alg. 2) on one replica m, for one fragment p:
 *   send step s   (t - t_p) mod H == 0, t >= H        Alg. 2 L6
 *     Delta_m = A_p - theta_m                           L7  (anchor reading AMB-1)
 *     4-bit E3M0 codes + fp32 per-block scales
 *     all-gather of the packed payloads over NVLink     L8
 *   receive step s + tau                                L10
 *     wait for the gather                               L11
 *     g = (1/M) sum_m decode(payload_m), fp32
 *     v = mu v + g ; A = A - lr (g + mu v)              L12
 *     theta_m = alpha theta_m + (1 - alpha) A           L13
 *
 * Conventions
 *  - Every function returns sd_status; nothing throws, exits or prints.
 *    A failing call leaves a message in sd_last_error(ctx) (thread-local
 *    when ctx == NULL) naming the offending values.
 *  - Device pointers are CUDA device addresses of the ctx's device, 32-byte
 *    aligned (256 recommended; gather buffers MUST be 256-byte aligned).
 *    The caller owns theta, anchor and momentum and must keep them alive
 *    until the stream work using them is done.  Gather buffers are either
 *    caller-owned device memory or (recommended) allocated by
 *    sd_gather_alloc in NCCL symmetric memory, which lets the all-gather run
 *    on the copy engines with zero SMs.  Apart from those and NCCL
 *    internals the library allocates no device memory, and it writes only
 *    slot_out, gather_buf, anchor, momentum, theta and the caller's
 *    quantize workspace (sd_set_workspace).
 *  - sd_stream is a cudaStream_t (NULL = legacy default stream).  Every
 *    device call is stream-ordered and asynchronous; errors raised on the
 *    device (non-finite outer gradients, NCCL async errors) surface at
 *    sd_check().
 *  - One sd_ctx per replica (= per GPU process), used from one host thread
 *    in program order.  The schedule functions are pure and thread-safe.
 *  - Layout: a fragment is one contiguous fp32 slab of n elements (AMB-18).
 *  - Environment (read once per process): SD_BLOCKS_PER_SM=k caps the grids
 *    at k CTAs per SM (measurement switch, results bit-identical);
 *    SD_WAIT_TIMEOUT_MS bounds the fused gathers' block-receive (below);
 *    SD_LOG_INIT=1 prints one line per communicator set up (stderr);
 *    measurement switches of the staged two-pass quantize (results
 *    bit-identical): SD_STAGE_HINTS (bit 0: pass 1 reads evict-first, bit 1:
 *    pass 2 discards consumed summaries; default 3), SD_STAGE_L2_MB (MB of
 *    summaries kept in L2 between the passes, default 40); SD_SIGNAL_KERNEL=0|1
 *    forces the fused gathers' round signal into the payload kernel's last
 *    CTA or a one-thread kernel after it (default: the kernel for push, the
 *    last CTA for pull).
 */
#ifndef SD_H_
#define SD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SD_ABI_VERSION 1u
#define SD_UNIQUE_ID_BYTES 128
#define SD_PAYLOAD_MAGIC 0x31304453u /* "SD01" little-endian */

typedef struct sd_ctx sd_ctx;
typedef void* sd_stream; /* cudaStream_t */

typedef enum {
  SD_OK = 0,
  SD_ERR_ARG = 1,       /* null / misaligned pointer, n mismatch, wrong slot  */
  SD_ERR_CONFIG = 2,    /* invalid sd_config (see sd_config_validate)         */
  SD_ERR_SCHEDULE = 3,  /* fragment p is not scheduled to send/receive at t   */
  SD_ERR_STATE = 4,     /* call order: merge without sync, p still in flight  */
  SD_ERR_NONFINITE = 5, /* a replica sent a non-finite outer gradient */
  SD_ERR_CUDA = 6,
  SD_ERR_NCCL = 7
} sd_status;

/* Method configuration.  Defaults (sd_config_default): strided pattern,
 * embed_policy 0, tau 1, alpha 0.5, outer lr 0.4, momentum 0.9, B 1024. */
typedef struct {
  uint32_t abi_version;   /* must be SD_ABI_VERSION                                       */
  int32_t num_blocks;     /* L: synchronizable blocks (transformer layers), >= 1          */
  int32_t fragment_size;  /* |p|: blocks per fragment, divides L                 */
  int32_t pattern;        /* 0 sequential, 1 strided (default)                 */
  int32_t embed_policy;   /* 0: non-block params join the last fragment             */
                          /* 1: they form their own extra fragment (reproduces P:501)      */
  int32_t H;              /* inner steps per round; H >= P                          */
  int32_t tau;            /* overlap delay, 0 <= tau < H                    */
  int64_t T;              /* last step: receives due after T are flushed at T;     */
                          /* 0 = unbounded                                                 */
  float alpha;            /* merge mix in [0, 1] (default 0.5)        */
  float outer_lr;         /* Nesterov outer learning rate (0.4), finite             */
  float outer_momentum;   /* mu in [0, 1) (0.9)                                     */
  int32_t scale_block;    /* B: elements per fp32 scale; 0 = one scale per fragment        */
                          /* (SPEC-exact); else a power of two in [256, 2^20]       */
                          /* (AMB-7; default 1024)                                         */
} sd_config;

/* ------------------------------------------------------------------------
 * Host-only, pure: configuration and the fragment scheduler (§8(a) a1).
 * ---------------------------------------------------------------------- */

/* Fills the defaults listed above for L = num_blocks, |p| = fragment_size, H. */
sd_status sd_config_default(sd_config* cfg, int32_t num_blocks, int32_t fragment_size, int32_t H);

/* Validates cfg before any work.  On error writes a message naming
 * the offending values into msg (if msg != NULL, truncated to cap bytes). */
sd_status sd_config_validate(const sd_config* cfg, char* msg, size_t cap);

/* P: number of fragments = L/|p| (+1 with embed_policy 1). */
sd_status sd_fragment_count(const sd_config* cfg, int32_t* P);

/* Fragment p: its block indices in ascending order (strided: p, p+P, p+2P, ...;
 * sequential: p|p| .. (p+1)|p|-1), t_p = floor(p*H/P), and
 * whether it also holds the non-block (embedding) parameters.
 * blocks may be NULL (cap 0) to query n_blocks only. */
sd_status sd_fragment_layout(const sd_config* cfg, int32_t p, int32_t* blocks, int32_t cap,
                             int32_t* n_blocks, int32_t* t_p, int32_t* holds_embed);

/* The calendar at 1-based step t (Alg. 2 L6 and L10):
 *   send    = { p : t >= H and (t - t_p) mod H == 0 }
 *   receive = { p : t - tau >= H and (t - tau - t_p) mod H == 0 }
 *             plus, at t == T > 0, every p whose send s satisfies T - tau < s <= T.
 * Both lists ascending, at most cap entries each (cap >= P always suffices). */
sd_status sd_fragment_schedule(const sd_config* cfg, int64_t t, int32_t* send, int32_t* n_send,
                               int32_t* recv, int32_t* n_recv, int32_t cap);

/* Scale blocks of a fragment of n elements: 0 if n == 0, 1 if B == 0, else ceil(n/B). */
int64_t sd_num_scale_blocks(const sd_config* cfg, int64_t n);

/* Bytes of one replica's payload for a fragment of n elements:
 *   [codes: ceil(n/2) bytes, element 2k in the low nibble of byte k]
 *   [zero pad to 256]  -> scales offset
 *   [nb fp32 scales, little endian][zero pad to 16]
 *   [trailer: u32 magic SD_PAYLOAD_MAGIC, u32 nb, u64 first non-finite index or 2^64-1]
 *   [zero pad to 256]
 * Returns 0 on an invalid cfg.  A gather buffer holds M consecutive payloads. */
size_t sd_payload_bytes(const sd_config* cfg, int64_t n);
size_t sd_payload_scales_offset(int64_t n);
size_t sd_payload_trailer_offset(const sd_config* cfg, int64_t n);

/* ------------------------------------------------------------------------
 * Device context: one per replica = one per GPU.
 * ---------------------------------------------------------------------- */

/* NCCL unique id for sd_init; rank 0 calls it, the caller broadcasts the
 * SD_UNIQUE_ID_BYTES bytes (e.g. with torch.distributed). */
sd_status sd_get_unique_id(uint8_t id[SD_UNIQUE_ID_BYTES]);

/* Creates the context of replica `rank` of M on CUDA device `device`.
 * id == NULL: no communicator.  Valid for M == 1, and as the single-GPU
 * emulation seam for M > 1: the caller then fills every slot of the gather
 * buffer itself (one ctx per emulated replica) and sd_fragment_sync only
 * orders streams.  id != NULL: collective over the M processes (blocking
 * NCCL communicator init; M == 1 included: a one-rank communicator runs the
 * same gather paths, every one trivially).  Creates a highest-priority comm
 * stream.  */
sd_status sd_init(sd_ctx** out, const sd_config* cfg, int32_t rank, int32_t M, const uint8_t* id,
                  int32_t device);

/* Allocates a gather buffer for a fragment of n elements: M payloads,
 * 256-byte aligned.  With a communicator: NCCL symmetric memory
 * (ncclMemAlloc) registered as a symmetric window of the ctx's communicator
 * -- COLLECTIVE: every rank calls it in the same order with the same n --
 * so sd_fragment_sync's all-gather runs on the copy engines
 * (NCCL_CTA_POLICY_ZERO), leaving every SM to the compute stream.  Without a
 * communicator: plain device memory.  Freed by sd_gather_free (collective
 * with a communicator) or sd_finalize. */
sd_status sd_gather_alloc(sd_ctx* ctx, int64_t n, void** out);
sd_status sd_gather_free(sd_ctx* ctx, void* gather_buf);

/* How the all-gather of Alg. 2 L8 is carried out for buffers from
 * sd_gather_alloc (set before allocating; default SD_GATHER_AUTO):
 *  SD_GATHER_COPY_ENGINE  sd_fragment_sync issues NCCL's in-place all-gather
 *                         on the comm stream (copy engines, zero SMs); it
 *                         overlaps whatever the compute stream does next.
 *  SD_GATHER_PUSH         fused: the quantize kernel stores every payload
 *                         word into this rank's slot of each peer's buffer
 *                         over NVLink as it produces it (NCCL symmetric-window
 *                         LSA pointers), then release-signals a per-round
 *                         flag with the round id (the count of sends of
 *                         this fragment, the same on every rank); the
 *                         block-receive is an acquire-wait on the peers'
 *                         flags.  Buffers hold two rounds (alternating by
 *                         round id), so no rendezvous is needed.
 * SD_GATHER_PULL is the same protocol with the transfer fused into the merge
 * instead (the apply reads the peers' slots from their buffers over NVLink).
 * In both, the round signal is fused into the end of the kernel that
 * finishes the payload (its last CTA release-stores {round id, first
 * non-finite index} into each peer's flag entry); the block-receive is one
 * single-CTA kernel per round that acquire-waits on the local flag entries
 * and leaves its verdict for the apply's CTAs.
 * The fused modes need every rank in this rank's NVLink (LSA) team and
 * M <= 32; otherwise (or without a communicator) the copy engines carry the
 * gather.
 * Block-receive timeout (PUSH, PULL): none by default -- the wait kernel
 * waits for every peer's flag.  SD_WAIT_TIMEOUT_MS=<ms> bounds it; on a timeout the round is skipped on this rank (A, v,
 * theta untouched), this rank tells its peers (a peer that has not passed its
 * own wait for the round skips it too), and the context becomes unusable:
 * sd_check and every later device call return SD_ERR_STATE, because the
 * replicas' outer state may no longer be identical -- re-initialize every
 * replica from a common state.
 * With caller-owned buffers or without a communicator the mode is ignored.
 * In PUSH and PULL modes a gather buffer must serve a single fragment (its
 * round ids count that fragment's sends). */
#define SD_GATHER_COPY_ENGINE 0
#define SD_GATHER_PUSH 1
#define SD_GATHER_AUTO 2 /* default: COPY_ENGINE when tau >= 1 (hidden behind later work); with tau == 0
                            (nothing to overlap with) PULL for M in {4, 8}, else PUSH -- measured on B200 */
#define SD_GATHER_PULL 3 /* fused into the apply: the quantize writes locally and signals; the merge
                            kernel reads the peers' payloads from their buffers over NVLink (no HBM
                            staging of the M payloads) */
sd_status sd_set_gather_mode(sd_ctx* ctx, int32_t mode);

/* Address of the M payloads of fragment p's most recent round inside
 * gather_buf (the buffer itself, or that round's half in push mode). */
sd_status sd_gather_payloads(sd_ctx* ctx, int32_t p, const void* gather_buf, const void** out);

/* Outer-state store init (§8(a) a2; AMB-2): anchor <- theta, momentum <- 0. */
sd_status sd_outer_state_init(sd_ctx* ctx, const float* theta, float* anchor, float* momentum,
                              int64_t n, sd_stream stream);

/* Host-offloaded outer-state store (PAPER.md:145-149:
 * "only a subset of the outer parameters and outer optimizer state is needed
 * at a given time ... we can start the transfer from RAM to HBM of a fragment
 * ... while finishing the previous (inner) gradients passes").  A_p and v_p
 * live in (pinned) host memory; `anchor`/`momentum` are device staging
 * buffers of n floats (HBM holds 2 x |p| instead of 2 x the model).
 *  sd_state_prefetch: after `stream`'s prior work (the staging buffers' last
 *    user), H2D copies on the ctx's copy stream; the next
 *    sd_outer_grad_quantize of p waits for them.  p must not be in flight.
 *  sd_state_writeback: after `stream`'s prior work (the merge of p), D2H
 *    copies on the copy stream.  p must not be in flight.
 *  sd_state_sync: `stream` waits for every copy issued so far (e.g. before
 *    reading the host store or reusing the host buffers).
 * Prefetches run on one copy stream (host -> device), writebacks on another
 * (device -> host), so the two directions overlap (PCIe is full duplex); a
 * prefetch into a staging buffer waits for the last writeback out of that
 * buffer, and a writeback waits for the prefetches issued before it (so it
 * never overwrites host data a prefetch is still reading). */
sd_status sd_state_prefetch(sd_ctx* ctx, int32_t p, const float* anchor_host, const float* momentum_host,
                            float* anchor, float* momentum, int64_t n, sd_stream stream);
sd_status sd_state_writeback(sd_ctx* ctx, int32_t p, const float* anchor, const float* momentum,
                             float* anchor_host, float* momentum_host, int64_t n, sd_stream stream);
sd_status sd_state_sync(sd_ctx* ctx, sd_stream stream);

/* The ctx's communication stream (highest priority; the copy-engine
 * all-gather of sd_fragment_sync runs on it), for tracing and timelines:
 * an event recorded on it after sd_fragment_sync completes with the gather.
 * Owned by the ctx; do not enqueue work on it. */
sd_status sd_comm_stream(sd_ctx* ctx, sd_stream* out);

/* InnerOpt = AdamW (NEXT-1; Alg. 2 L5; Adam as InnerOpt, P:77;
 * SPEC.md:171-179 adamw_step with decoupled weight decay). */
typedef struct {
  float lr, beta1, beta2, eps, weight_decay;
} sd_adamw;

/* One AdamW inner step (AdamW step index k >= 1, for the bias corrections):
 *   m = b1 m + (1-b1) g ; v = b2 v + (1-b2) g^2
 *   theta = theta (1 - lr wd) - (lr / bc1) (m / (sqrt(v) / sqrt(bc2) + eps))
 * bc_i = 1 - b_i^k evaluated in binary64 and rounded once; every other op
 * rounds once (DESIGN.md AMB-20).  theta, m, v updated in place; grad read. */
sd_status sd_inner_adamw(sd_ctx* ctx, int64_t k, float* theta, const float* grad, float* m, float* v, int64_t n,
                         const sd_adamw* hp, sd_stream stream);

/* The inner step that precedes a send, fused with Alg. 2 L7 + E3M0: same
 * AdamW update, then fragment p's payload from the updated theta in the same
 * pass (theta is not re-read), with sd_outer_grad_quantize's schedule and
 * state rules (p sends at step t). */
sd_status sd_inner_adamw_quantize(sd_ctx* ctx, int32_t p, int64_t t, int64_t k, float* theta, const float* grad,
                                  float* m, float* v, const float* anchor, int64_t n, void* slot_out,
                                  const sd_adamw* hp, sd_stream stream);

/* Scratch of the two-pass quantize.  With B = 0 (one scale per fragment,
 * S:266) or B >= 2048 every code depends on a block maximum over more data
 * than one pass keeps on chip, so the quantize makes two passes (block max,
 * then encode).  Without a workspace the second pass re-reads theta and A
 * (16.5 B/param moved for 8.5 needed).  With one, the first pass also writes
 * a 16-bit summary of every Delta there and the second pass encodes from it,
 * re-reading theta and A only for the rare elements whose summary straddles
 * a code threshold (about 1 in 4000) -- same codes, bit for bit.
 *  sd_quantize_workspace_bytes: bytes needed for a fragment of n elements
 *    (0 when the single pass applies: B in {256, 512, 1024}, or n == 0, or an
 *    invalid cfg).
 *  sd_set_workspace: caller-owned device memory, 256-byte aligned (NULL or 0
 *    bytes detaches).  Used by sd_outer_grad_quantize and
 *    sd_inner_adamw_quantize for every fragment whose need fits in `bytes`
 *    (others take the re-reading pass).  Its contents between calls are
 *    meaningless; the calls that use it must be ordered with each other (one
 *    stream, as Alg. 2's sends are), and it must stay alive until that
 *    stream's work using it is done. */
size_t sd_quantize_workspace_bytes(const sd_config* cfg, int64_t n);
sd_status sd_set_workspace(sd_ctx* ctx, void* ws, size_t bytes);

/* Alg. 2 L7 + E3M0 (§8(a) a3).  p must be scheduled to send at t and not be
 * in flight.  Reads theta[n], anchor[n]; writes one payload
 * (sd_payload_bytes) at slot_out, which must be gather_buf + rank * payload
 * of the buffer later passed to sd_fragment_sync.  A non-finite Delta is
 * recorded in the payload trailer (index of the first one); the round is
 * then skipped on every replica and sd_check reports SD_ERR_NONFINITE. */
sd_status sd_outer_grad_quantize(sd_ctx* ctx, int32_t p, int64_t t, const float* theta,
                                 const float* anchor, int64_t n, void* slot_out, sd_stream stream);

/* Alg. 2 L8 transport (§8(a) a4): after `stream`'s prior work (the
 * quantize), an in-place all-gather of the M payloads of gather_buf on the
 * ctx's comm stream; returns immediately (async-send).  No communicator:
 * only orders streams. */
sd_status sd_fragment_sync(sd_ctx* ctx, int32_t p, int64_t t, void* gather_buf, int64_t n,
                           sd_stream stream);

/* Alg. 2 L11 block-receive on its own (§8(a) a5): `stream` waits for the
 * all-gather of p, whose receive falls at t.  Optional: sd_merge performs
 * the same wait; splitting it out lets a caller time the merge kernel
 * apart from any exposed gather time. */
sd_status sd_fragment_wait(sd_ctx* ctx, int32_t p, int64_t t, sd_stream stream);

/* Alg. 2 L11-13 (§8(a) a5 + a6): `stream` waits for the gather of p
 * (block-receive), then one fused kernel: decode + M-way fp32 mean in
 * ascending replica order, Nesterov on (anchor, momentum), alpha-merge into
 * theta (the live parameters after tau inner steps).  p must be received at
 * t (send step + tau, or the flush at T).  If any payload is poisoned or
 * malformed, nothing is written (identically on every replica).  An NCCL
 * async error already reported by the communicator fails the call with
 * SD_ERR_NCCL before anything is enqueued. */
sd_status sd_merge(sd_ctx* ctx, int32_t p, int64_t t, const void* gather_buf, float* theta,
                   float* anchor, float* momentum, int64_t n, sd_stream stream);

/* The inner step of the receive step fused with its receive (Alg. 2 L5 then
 * L11-13 at t = send + tau): AdamW on theta (as sd_inner_adamw, step k),
 * then the same block-receive, mean, Nesterov and alpha-merge as sd_merge
 * on the updated theta -- theta is read and written once.  On a poisoned
 * round the AdamW step still happens and the merge is skipped. */
sd_status sd_inner_adamw_merge(sd_ctx* ctx, int32_t p, int64_t t, int64_t k, float* theta, const float* grad,
                               float* m, float* v, const void* gather_buf, float* anchor, float* momentum,
                               int64_t n, const sd_adamw* hp, sd_stream stream);

/* Synchronizes the device and reports deferred errors: CUDA errors, NCCL
 * async errors, and a skipped round -- SD_ERR_NONFINITE with
 * *first_bad_index (if non-NULL) = index of the first non-finite Delta for
 * a poisoned round; SD_ERR_STATE for a malformed payload, or (sticky) for a
 * block-receive timeout (SD_WAIT_TIMEOUT_MS). */
sd_status sd_check(sd_ctx* ctx, int64_t* first_bad_index);

/* Message of the last failing call on ctx (thread-local one if ctx == NULL). */
const char* sd_last_error(const sd_ctx* ctx);

/* Destroys the communicator, streams and events and frees the gather buffers
 * of sd_gather_alloc; with gather buffers or a workspace attached it first
 * synchronizes the device, so the caller may free the workspace afterwards.
 * NULL is a no-op. */
sd_status sd_finalize(sd_ctx* ctx);

/* Number of kernels libsd has launched in this process (for bench.py's
 * gpu_launches accounting). */
uint64_t sd_kernel_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SD_H_ */
