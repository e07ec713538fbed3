/*
 * tarragon.h — C ABI of the B200-native Tarragon MoE-layer round trip.
 *
 * One call of tg_moe_layer() is one pass of the attention-worker (AW) ->
 * expert-worker (EW) -> AW round trip of one MoE layer, as in
 * PAPER.md §2.2.1 ("every data-parallel AW ... selects a subset of
 * experts, sends token embeddings to the corresponding EWs, and waits until
 * all selected experts return their outputs") through the Reconfigurable
 * Forwarding Engine's expert_io path (§4.2):
 *   gate (fp32 top-k)  ->  ERT resolve (masked EW -> shadow)  ->  permute
 *   ->  dispatch exchange  ->  grouped SwiGLU expert FFN  ->  combine
 *   exchange  ->  weighted unpermute.
 * The operation computed is out[t] = sum_{e in TopK(t)} w_{t,e} FFN_e(x_t)
 * (+ FFN_shared(x_t)) (§2.1); DESIGN.md §3 lists every reading
 * of a point the paper leaves open.
 *
 * Processes and devices.  One process ("rank") per GPU; every rank is an AW
 * shard (it owns a contiguous block of the global tokens, "each AW
 * serving a disjoint subset of requests") and hosts zero or more logical EWs
 * ("EWs ... partition expert FFNs across GPUs").  Dispatch and combine
 * are one-sided stores into peer-mapped buffers over NVLink (P:739, P:865-867:
 * point-to-point, no collective group membership per call).
 *
 * Conventions.
 *   - All tensors are row-major and contiguous.  bf16 = IEEE bfloat16 bits.
 *   - "device" pointers are CUDA device pointers on the ctx's device.
 *   - Every call returns tg_status; on failure tg_last_error() describes it.
 *   - Validation errors are synchronous and leave the ctx unchanged.
 *   - CUDA errors are sticky: once TG_ERR_CUDA is returned the ctx must be
 *     finalised.  A ctx is not thread-safe.
 *   - There is no CPU fallback: with no usable sm_100a device tg_init()
 *     returns TG_ERR_CUDA / TG_ERR_UNSUPPORTED (a host-only ctx, device = -1,
 *     exists for validating tables and masks; its tg_moe_layer() returns
 *     TG_ERR_UNSUPPORTED).
 */
#ifndef TARRAGON_H_
#define TARRAGON_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct tg_ctx tg_ctx; /* opaque; one per (rank, MoE layer) */

typedef enum {
  TG_OK = 0,
  TG_ERR_INVALID = -1,        /* bad argument, shape or capacity */
  TG_ERR_NO_ROUTE = -2,       /* some expert has no unmasked candidate */
  TG_ERR_NOT_LOADED = -3,     /* a candidate (ew, slot) does not hold that expert */
  TG_ERR_STALE_VERSION = -4,  /* route-table version <= current */
  TG_ERR_CUDA = -5,           /* CUDA runtime/driver error or device timeout (sticky) */
  TG_ERR_PEER = -6,           /* peer mapping / exchange error */
  TG_ERR_OOM = -7,            /* device allocation failed */
  TG_ERR_UNSUPPORTED = -8     /* host-only ctx, or a shape outside the supported set */
} tg_status;

/* Layer shape and placement.  Copied by tg_init; the caller may free it.
 *   d_model, n_experts, top_k, d_ffn : d, E, k, F  (north_star SwiGLU)
 *     d % 64 == 0, F % 64 == 0, 1 <= k <= min(E, 8), E <= 256.
 *   d_ffn_shared  : merged shared-expert width (0 = none), % 64 == 0.
 *   n_ews, ew_rank: W logical EWs; EW w lives on rank ew_rank[w] (W may
 *                   exceed world: several EWs per GPU).  EWs of one rank get
 *                   consecutive bank slots in ew order.
 *   slots_per_ew  : expert slots per EW (primaries + shadows).
 *   max_tokens_per_rank : capacity of x/out per call on each rank.       */
typedef struct {
  int d_model, n_experts, top_k, d_ffn;
  int d_ffn_shared;
  int n_ews;
  const int32_t *ew_rank; /* [n_ews] */
  int slots_per_ew;
  int max_tokens_per_rank;
  /* Gating variant (R#2 / R#17, SURVEY NEXT-3b):
   *   gate_mode 0: w = softmax over the k selected logits (renormalised top-k; default);
   *   gate_mode 1: w = softmax over all E logits, the k selected kept un-renormalised
   *                (the public DS-V2-Lite / Qwen1.5-MoE routers, norm_topk_prob = false).
   *   shared_gate 1: the shared expert's output is scaled by sigmoid(x . wsg) per token
   *                (Qwen1.5-MoE shared_expert_gate; load wsg with tg_load_shared_gate). */
  int gate_mode;
  int shared_gate;
} tg_config;

/* Create a ctx on `cuda_device` (-1: host-only ctx for table/mask logic).
 * Allocates the expert bank, receive/combine buffers and flags in HBM.
 * Collective in the sense that every rank must create its ctx with the same
 * config before tg_connect_peers().                                      */
tg_status tg_init(const tg_config *cfg, int rank, int world, int cuda_device, tg_ctx **out);

/* Peer bootstrap (world > 1; point-to-point, no collective
 * group per call).  tg_peer_handle_size() bytes per rank: the caller gathers
 * every rank's handle (e.g. torch.distributed.all_gather) and passes them
 * concatenated in rank order to tg_connect_peers(), which maps each peer's
 * buffers for direct NVLink loads/stores.  A handle carries the layout
 * signature of the rank's peer-visible region (one-sided stores land at the
 * sender's offsets): every rank must use the same tg_config, including
 * max_tokens_per_rank, else TG_ERR_PEER and nothing is mapped.  world == 1
 * needs no connect call.                                                   */
size_t tg_peer_handle_size(void);
tg_status tg_get_peer_handle(tg_ctx *ctx, void *out);
tg_status tg_connect_peers(tg_ctx *ctx, const void *all_handles);

/* Virtual ranks on one GPU (tests, and a GPU shared by several AW/EW
 * shards): ctxs[q] (q < world <= 4) are the ctxs of ranks 0..world-1, created
 * in this process on the SAME device; tg_connect_local(ctx, ctxs) maps them
 * as ctx's peers by device pointer (the data plane is the same code as over
 * NVLink: stores into peer regions, epoch flags).  Layout signatures must
 * match (TG_ERR_PEER).  The ranks of a call wait on one another's flags, so
 * they run as ONE cooperative launch, each rank on SM count / world CTAs:
 * tg_moe_layer_multi(ctxs, world, x[], out[], n_tokens[], stream) is one
 * tg_moe_layer call of every rank (n_tokens[r] < 0: rank r does not take part,
 * as a rank that died before the call), and tg_failover_multi(ctxs, world,
 * x[], out[], n_tokens[], stream, failed[]) is tg_failover of every rank that
 * saw a failure (failed[r] = its failed-rank mask), in one launch.  Errors as
 * tg_moe_layer / tg_failover; TG_ERR_INVALID if the ctxs are not ranks
 * 0..world-1 of one device, TG_ERR_PEER if not connected by tg_connect_local. */
tg_status tg_connect_local(tg_ctx *ctx, tg_ctx *const *ctxs);
tg_status tg_moe_layer_multi(tg_ctx *const *ctxs, int world, const void *const *x, void *const *out,
                             const int *n_tokens, void *stream);
tg_status tg_failover_multi(tg_ctx *const *ctxs, int world, const void *const *x, void *const *out,
                            const int *n_tokens, void *stream, uint32_t *failed);

/* Router weights Wg [E][d] bf16 (host or device source; copied).  SPMD.
 * The gating network of P:265 §2.1 ("a gating network ... selects the top-k
 * experts"): a linear router without bias (R#1).                 */
tg_status tg_load_gate(tg_ctx *ctx, const void *wg, int src_on_device);

/* Load expert `expert_id` into slot `slot` of EW `ew` (P:954 shadow experts:
 * loading the same expert into another (ew, slot) creates a bit-identical
 * shadow replica).  w1, w3: [F][d] bf16; w2: [d][F] bf16.  Only the rank
 * hosting `ew` reads the weights (others may pass NULL); every rank records
 * slot -> expert.  Synchronous.  SPMD.                                     */
tg_status tg_load_experts(tg_ctx *ctx, int ew, int slot, int expert_id, const void *w1,
                          const void *w3, const void *w2, int src_on_device);

/* Merged shared expert (F_sh = d_ffn_shared): w1, w3 [F_sh][d]; w2 [d][F_sh].
 * Replicated on every rank; added to the routed sum with weight 1.  Not in
 * the paper: BASELINE.json configs[3] (DeepSeek-V2-Lite shape, "+ 2 shared");
 * DESIGN.md R#16.                                                          */
tg_status tg_load_shared(tg_ctx *ctx, const void *w1, const void *w3, const void *w2,
                         int src_on_device);

/* Shared-expert gate vector wsg [d] bf16 (config shared_gate = 1).  SPMD.
 * Not in the paper: the public Qwen1.5-MoE shared_expert_gate, R#17. */
tg_status tg_load_shared_gate(tg_ctx *ctx, const void *wsg, int src_on_device);

/* Expert Routing Table (§4.2): cand[e][c] = (ew, slot) for
 * c < max_cands, primaries then shadows, (-1, -1) padding.  Accepted only
 * if version > current version (else TG_ERR_STALE_VERSION, table ignored),
 * every candidate (ew, slot) holds expert e (else TG_ERR_NOT_LOADED), and
 * every expert has an unmasked candidate (else TG_ERR_NO_ROUTE).  Host-only;
 * takes effect at the NEXT tg_moe_layer call, without re-initialisation.  */
tg_status tg_set_route_table(tg_ctx *ctx, uint64_t version, const int32_t *cand, int max_cands);

/* Fail-stop an EW (masked = 1) or let it rejoin (0) (§3.3,
 * P:914-916 §5.1).  Always applied.  From the next tg_moe_layer on, the
 * masked EW receives no rows and none of its memory is read; its experts are
 * served by the first unmasked candidate (a shadow).  Returns TG_ERR_NO_ROUTE
 * as a warning if some expert lost its last candidate; tg_moe_layer then
 * fails with TG_ERR_NO_ROUTE (nothing launched) until the table or mask is
 * fixed.  Host-only, O(E * max_cands).                                     */
tg_status tg_mask_worker(tg_ctx *ctx, int ew, int masked);

/* Fail-stop a whole rank (masked = 1): its AW shard and every EW it hosts
 * (§3.3; §5.2 "EWs tolerate AW failures": the surviving
 * ranks proceed without the failed AW's tokens).  Every surviving rank makes
 * the same call (SPMD); from the next tg_moe_layer on, the masked rank is
 * never awaited, written or read, its counts are taken as zero, and its
 * experts are served by shadows (TG_ERR_NO_ROUTE as for tg_mask_worker if
 * some expert has none).  The masked rank must not call tg_moe_layer again;
 * rejoining needs re-provisioning (new ctxs, out of scope):
 * masked = 0 on a masked rank returns TG_ERR_UNSUPPORTED.  Host-only.      */
tg_status tg_mask_rank(tg_ctx *ctx, int rank, int masked);

/* In-call EW failover (§5.1 "the AW re-dispatches the affected
 * tokens to a shadow").  During a call, this rank's waits on a
 * PEER's data-ready and combine flags give up after the failure timeout
 * (default 200 ms; tg_set_failure_timeout, (0, 4000] ms) and record the peer as
 * failed instead of trapping; the call completes with the outputs of the pairs
 * that peer held undefined.  tg_failover(ctx, x, out, n_tokens, stream, &failed)
 * then synchronises `stream` and, if the last tg_moe_layer saw a failure:
 * fail-stops the failed ranks (as tg_mask_rank), re-routes the pairs this rank
 * had sent them to the next live candidate of each expert (ERT order) and
 * recomputes them and `out` for every token, all within the same call's inputs
 * (x, n_tokens must be the failed call's; outputs of pairs other EWs served are
 * kept) — bitwise the output an unfailed call gives.  *failed = bit mask of the
 * failed ranks (0: nothing to do, out untouched).
 * Detection: within a call every live rank waits for every other live rank's
 * count flag (timeout 10 x the failure timeout, <= 4 s: host threads may be
 * late) and combine flag, so all survivors see a rank that fails at any point
 * of the call in that same call; a rank silent in the count exchange is taken
 * as failed with zero rows (EWs proceed with the tokens they have, §5.2
 * P:927-941) and nothing is dispatched to it.
 * Replay: tg_failover is collective among the survivors (every surviving rank
 * calls it after every call; it returns at once when nothing failed).  The
 * re-routed pairs go to the next live candidate of their expert on WHICHEVER
 * rank it lives (a replay run with its own flags: the replay rows are the
 * whole work list of the EWs that serve them, "replayed requests are
 * prioritized").  Returns TG_OK; TG_ERR_NO_ROUTE when some pair has no live
 * candidate left (not recomputed); TG_ERR_PEER when another rank failed
 * during the replay itself (call tg_failover again).  No device wait on a
 * peer traps: a silent peer is always recorded as failed.                   */
tg_status tg_set_failure_timeout(tg_ctx *ctx, double ms);
tg_status tg_failover(tg_ctx *ctx, const void *x, void *out, int n_tokens, void *stream, uint32_t *failed);

/* Fault injection (tests): the next tg_moe_layer on this ctx runs its front
 * and dispatch and then stops, as a process that crashes mid-call (peers hold
 * its rows and wait for its expert outputs).  The ctx is dead afterwards:
 * only tg_finalize may follow.                                               */
tg_status tg_inject_failure(tg_ctx *ctx);

/* KV-cache checkpointing in the AW-EW idle gaps (§6.1; segment
 * size C = 2 H_kv (d / H_attn) S_elem, App. C: 4 KB per token and
 * layer for Mixtral).  The checkpoint store of this AW is a pinned host bucket
 * written by the copy engines (no SM time, no NVLink: the layer's traffic is
 * untouched).  tg_kv_store_init(ctx, bytes) allocates it.
 * tg_kv_checkpoint(ctx, seg, bytes, offset, seq, stream) enqueues, ordered
 * after the work already on `stream` (the layer call that produced the
 * segment), a copy of `bytes` from DEVICE `seg` to bucket + offset on a
 * lowest-priority stream, then a commit record: seq becomes the committed
 * sequence number once that copy (and every earlier one) has landed ("async
 * log + commit record").  Non-blocking; seq must increase.
 * tg_kv_committed(ctx, &seq): last committed seq (0: none yet).
 * tg_kv_restore(ctx, dst, bytes, offset, stream): waits for the pending
 * checkpoints, then copies bucket + offset back to DEVICE `dst` on `stream`
 * (request-level restoration).  `seg` must stay allocated and
 * unmodified until tg_kv_committed() reaches seq (the copy runs later, on
 * the checkpoint stream; the Python binding keeps a reference until then).
 * Errors: TG_ERR_NOT_LOADED (no
 * store), TG_ERR_INVALID (range), TG_ERR_STALE_VERSION (seq not increasing),
 * TG_ERR_UNSUPPORTED (host-only ctx), TG_ERR_OOM.                          */
tg_status tg_kv_store_init(tg_ctx *ctx, size_t bytes);
tg_status tg_kv_checkpoint(tg_ctx *ctx, const void *seg, size_t bytes, size_t offset, uint64_t seq, void *stream);
tg_status tg_kv_committed(tg_ctx *ctx, uint64_t *seq);
tg_status tg_kv_restore(tg_ctx *ctx, void *dst, size_t bytes, size_t offset, void *stream);

/* One MoE layer round trip (collective: every live rank calls it, same order).
 * x: device bf16 [n_tokens][d] (this rank's tokens); out: device bf16
 * [n_tokens][d], must not alias x.  n_tokens <= max_tokens_per_rank (may be
 * 0).  Enqueued on `stream` (cudaStream_t; NULL = legacy default stream);
 * returns without synchronising.  x must stay valid until the stream passes
 * the call.  One kernel launch (programmatic dependent launch): consecutive
 * calls on one stream overlap — the next call's CTAs start on the SMs the
 * previous call frees and, for decode-sized calls, begin their expert GEMM
 * before the previous call has completed (alternate calls use alternate
 * internal buffer sets).  Stream order still holds for the caller: work
 * enqueued after a call sees its output.  The launch keeps one CTA per SM
 * and never waits on a later call, so every CTA becomes resident; do not run
 * a kernel beside it on the same GPU that waits for the layer.           */
tg_status tg_moe_layer(tg_ctx *ctx, const void *x, void *out, int n_tokens, void *stream);

/* End-to-end form: x_host/out_host are pinned HOST buffers.  The H2D copy of
 * x and the D2H copy of out run on the ctx's own copy streams, pipelined over
 * two staging buffers so that they overlap the layers of the neighbouring
 * calls on `stream`.  The outputs (and the right to reuse x_host) are
 * guaranteed once `stream` passes a later tg_host_sync(ctx, stream), which
 * makes `stream` wait for every pending host-path copy and orders the next
 * host-path copies after the work already on `stream`.  The copy streams are
 * ordered against the layer launches by device words (cuStreamWaitValue32 /
 * cuStreamWriteValue32 on the copy streams, polled by the kernel), so nothing
 * is enqueued on `stream` between two consecutive layer launches and they
 * overlap as tg_moe_layer calls do; where stream memory operations are not
 * available, event ordering is used instead (the launches then serialise).  */
tg_status tg_host_sync(tg_ctx *ctx, void *stream);
tg_status tg_moe_layer_host(tg_ctx *ctx, const void *x_host, void *out_host, int n_tokens,
                            void *stream);

/* Routing of the LAST call, for parity tests (device destination buffers,
 * any may be NULL):  idx int32 [n][k] (ascending expert id), w fp32 [n][k],
 * dst_rank / dst_slot (bank slot on that rank) / dst_pos (row in that rank's
 * receive buffer; -1 for a pair whose destination failed in the count
 * exchange) int32 [n][k], counts int32 [world][S_max] = rows per (rank, bank
 * slot) summed over ALL source ranks.  n_tokens must equal the last call's
 * (TG_ERR_INVALID otherwise: the buffers are sized by it).  Enqueued on
 * stream.                                                                  */
tg_status tg_get_routing(tg_ctx *ctx, int n_tokens, int32_t *idx, float *w, int32_t *dst_rank,
                         int32_t *dst_slot, int32_t *dst_pos, int32_t *counts, void *stream);

/* Stage values of the LAST call on this rank, for per-storage-point parity
 * tests: each is what the next stage of the path read.
 *   TG_STAGE_LOGITS fp32 [n][E (+1 shared-gate row)]  router logits O1 (only
 *                   written while tg_set_stage_export(ctx, 1) is on)
 *   TG_STAGE_RECV   bf16 [R][d]   token rows this EW received (R = rows of all
 *                   its slots, slots in ascending bank slot, P:385 batches)
 *   TG_STAGE_META   int32 [R][2]  origin of each row: (source rank, t * k + j)
 *   TG_STAGE_H      bf16 [R][F]   SwiGLU activations h = silu(a1) * a3 (O6a)
 *   TG_STAGE_Y      bf16 [n][k][d] expert outputs returned to this AW (O6b)
 *   TG_STAGE_HSH / TG_STAGE_YSH  bf16 [n][F_sh] / [n][d]  shared expert (O7)
 *   TG_STAGE_SGATE  fp32 [n]      sigmoid shared-expert gate (O7')
 * tg_get_stage(ctx, stage, dst, cap, &bytes) synchronises the device and
 * copies `bytes` to dst (host or device; dst = NULL: size query only).
 * TG_ERR_INVALID if cap < bytes or the stage is unknown.                    */
enum { TG_STAGE_LOGITS = 0, TG_STAGE_RECV = 1, TG_STAGE_META = 2, TG_STAGE_H = 3, TG_STAGE_Y = 4,
       TG_STAGE_HSH = 5, TG_STAGE_YSH = 6, TG_STAGE_SGATE = 7 };
tg_status tg_set_stage_export(tg_ctx *ctx, int on);
tg_status tg_get_stage(tg_ctx *ctx, int stage, void *dst, size_t cap, size_t *bytes);

/* S_max = max bank slots on any rank; bank slot of (ew, slot) on its rank. */
int tg_max_slots(const tg_ctx *ctx);
int tg_bank_slot(const tg_ctx *ctx, int ew, int slot);

/* Cumulative rows routed to each (rank, bank slot) since tg_init, from this
 * rank's tokens: int64 [world][S_max] host array.  Synchronises the device.
 * The per-EW load the paper's shadow-inactivity and failover experiments
 * observe (App. D: shadows receive no traffic until activated;
 * §5.1: a masked EW receives none after the reroute).            */
tg_status tg_get_stats(tg_ctx *ctx, int64_t *rows);

/* Per-kernel CUDA-event timing (events on the call's stream around each
 * launch, no host synchronisation per call).  tg_set_profiling(ctx, 1) starts
 * a new record; tg_get_kernel_times(ctx, ms, &n) synchronises and writes n
 * (= 1) MEAN durations in ms over the recorded calls (at most the last 512):
 * the one launch of a call, k_layer (gate, rank, count exchange, dispatch ||
 * grouped expert FFN, fused combine exchange, combine).                   */
tg_status tg_set_profiling(tg_ctx *ctx, int on);
tg_status tg_get_kernel_times(tg_ctx *ctx, float *ms, int *n);

/* Diagnostics (performance analysis of k_layer).
 * tg_set_trace(ctx, 1): subsequent calls record, per GEMM work unit, its
 * completion (globaltimer ns << 16 | unit kind << 12 | SM id), per CTA the
 * start time of its GEMM phase, and phase timestamps of the front phases.
 * tg_get_trace(ctx, trace, cap, &n_units, &n_ctas) synchronises and copies
 * the last call's records to the HOST array trace (uint64, cap entries):
 * [0, n_units) unit records, then 148 CTA start stamps, then 64 phase stamps. */
tg_status tg_set_trace(tg_ctx *ctx, int on);
tg_status tg_get_trace(tg_ctx *ctx, uint64_t *trace, int cap, int *n_units, int *n_ctas);

/* Kernel launches enqueued by the last tg_moe_layer call. */
int tg_last_launch_count(const tg_ctx *ctx);

/* Human-readable description of the last error on ctx (or of the last
 * failed tg_init if ctx == NULL).  Never NULL.                             */
const char *tg_last_error(const tg_ctx *ctx);

/* Free everything (collective with world > 1: peers must not be inside a
 * tg_moe_layer call).                                                      */
tg_status tg_finalize(tg_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* TARRAGON_H_ */
