/*
 * moe.h -- C ABI of libmoe, the B200 (sm_100a) expert-parallel MoE-layer hot
 * path of MoETuner (arXiv 2502.06643).
 *
 * Citation key: P:Lnnn = PAPER.md line nnn (§ named), S:Lnnn = SPEC.md line nnn,
 * Gnn = a reading of the paper listed in DESIGN.md §3.
 *
 * The layer (Fig. background-ep(b)):
 *   moe_route        top-k gating
 *   moe_route_stats  load P and co-activation R counts
 *   moe_dispatch     placement-aware permute + all-to-all
 *   moe_expert_ffn   grouped SwiGLU expert FFN
 *   moe_combine      all-to-all back + weighted unpermute
 *
 * Conventions that hold for every call:
 *   - Every tensor argument is a DEVICE pointer owned by the caller unless the
 *     comment says "host".  Layouts are dense row-major, no padding.
 *   - bf16 tensors are passed as raw 16-bit patterns (moe_bf16).
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  All device
 *     work is enqueued on it; calls return before it completes unless stated.
 *   - Argument validation is synchronous: on MOE_ERR_INVALID_ARG nothing was
 *     enqueued.  moe_last_error(ctx) holds a message for the last failure.
 *   - The library never aborts and never prints.
 *   - A context is bound to one device and is not thread-safe.  Calls run on
 *     the context's device and leave the caller's current device unchanged.
 *
 * Ranks.  An EP group has G ranks.  G = config.world real processes (one per
 * GPU, NCCL between them), or G = config.virtual_ranks ranks emulated inside
 * one process on one GPU (world must then be 1): the kernels, slot, count and
 * receive layouts are exactly those of G real ranks, and the all-to-all
 * becomes device-local row copies (SURVEY §4 "virtual ranks").
 * Token ownership (G7): source rank s owns a contiguous block of
 * floor(T/G) + [s < T mod G] tokens.  In virtual mode the T passed to a call
 * covers all G ranks' tokens concatenated in rank order; in real mode T is
 * this rank's own token count (may differ per rank, may be 0).
 *
 * Tensor parallelism inside the experts (config.tp > 1; the paper's "4EP-2TP",
 * P:L77-79; reading G20): the G ranks form G/tp EP groups of tp
 * consecutive ranks (rank r = TP index r % tp of group r / tp).  Every rank owns
 * a token block and is a source; the placement maps experts to EP GROUPS; every
 * rank of group g receives all rows routed to g's experts (the TP all-gather is
 * part of the dispatch) and computes the slice of the FFN dimension its TP index
 * owns; the bf16 partial outputs go back to the source, which sums the tp
 * partials (fp32, TP index ascending) before the gate-weighted combine (the TP
 * reduce-scatter is part of the combine).
 */
#ifndef MOE_H
#define MOE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct moe_ctx* moe_ctx_t;
typedef uint16_t moe_bf16;     /* raw bf16 bits, binary compatible with __nv_bfloat16 */
typedef void* moe_stream_t;    /* cudaStream_t */

typedef enum {
  MOE_OK = 0,
  MOE_ERR_INVALID_ARG = 1,   /* bad argument; nothing enqueued */
  MOE_ERR_CUDA = 2,          /* a CUDA runtime/driver call failed */
  MOE_ERR_NCCL = 3,          /* an NCCL call failed */
  MOE_ERR_CAPACITY = 4,      /* size exceeds what the context was created for */
  MOE_ERR_UNSUPPORTED = 5,   /* shape/mode not implemented (e.g. H % 64 != 0) */
  MOE_ERR_DEVICE = 6,        /* latched device-side error (bad expert id ...) */
  MOE_ERR_TIMEOUT = 7
} moe_status;

typedef enum { MOE_A2A_NCCL = 0, MOE_A2A_P2P = 1 } moe_a2a_mode;

typedef struct {
  int32_t max_tokens;     /* upper bound on T of any call (per process) */
  int32_t hidden;         /* H; multiple of 64 */
  int32_t ffn;            /* F; multiple of 64 */
  int32_t num_experts;    /* E; 1..256 */
  int32_t max_k;          /* upper bound on k; 1..E, <= 16 */
  int32_t world;          /* real EP ranks (processes); 1 => no NCCL */
  int32_t rank;           /* this process's rank in [0, world) */
  int32_t device;         /* CUDA device ordinal */
  int32_t virtual_ranks;  /* >1 => emulate that many EP ranks (world must be 1) */
  int32_t a2a_mode;       /* moe_a2a_mode (real ranks only; tp > 1 needs MOE_A2A_P2P):
                           * MOE_A2A_NCCL: count all-gather + one host sync to read the
                           *   G x E count matrix + grouped ncclSend/ncclRecv per (peer, expert);
                           * MOE_A2A_P2P: receive / expert-output buffers and a signal block
                           *   are mapped into every peer with CUDA IPC at creation; the
                           *   count exchange, the dispatch (NVLink stores straight into the
                           *   hosting rank's receive rows) and the combine (NVLink loads of
                           *   the hosting rank's output rows) run inside the kernels with
                           *   epoch-valued release/acquire flags; no host synchronisation. */
  int32_t tp;             /* tensor-parallel ranks per expert (0 or 1: none).  G % tp == 0,
                           * tp <= 8, (F / tp) % 64 == 0; real ranks need MOE_A2A_P2P. */
} moe_config;

/* Host-side summary of the last dispatch (optional output of moe_dispatch). */
typedef struct {
  int32_t world;                 /* G */
  int32_t num_local_experts;     /* experts hosted by this process (virtual: E) */
  int64_t recv_rows;             /* routed rows this process computes */
  int32_t send_counts[64];       /* rows this rank sends to rank g (real mode) */
  int32_t recv_counts[64];       /* rows rank g receives (all ranks) */
} moe_dispatch_info;

/* ---- lifecycle ------------------------------------------------------------ */

/* Create an NCCL unique id (rank 0 only); the caller broadcasts the 128 bytes
 * (e.g. with torch.distributed).  out: host, 128 bytes. */
moe_status moe_get_unique_id(uint8_t out[128]);

/* Create a context (collective over the EP group when world > 1).  Allocates
 * every workspace for the worst case of dropless routing (G6): per process
 * max_tokens * min(k, E_local) routed rows plus per-expert padding to the GEMM
 * M tile (256 rows; 128 rows for decode-sized contexts whose worst case averages
 * <= 256 routed rows per expert -- they run the GEMM on 128-row tiles).
 * uid: host, 128 bytes from moe_get_unique_id, or NULL when world == 1. */
moe_status moe_ctx_create(const moe_config* cfg, const uint8_t* uid, moe_ctx_t* out);
/* Single-process group: create the n contexts of an n-rank EP group inside this
 * process (out: host array of n handles; rank r = out[r]).  Same semantics as n
 * processes calling moe_ctx_create with world = n, rank = r and a2a_mode =
 * MOE_A2A_P2P, except that the peer tables hold the other contexts' device
 * pointers directly -- no CUDA IPC, no NCCL (moe_stats_allreduce* return
 * MOE_ERR_UNSUPPORTED).  devices: host int32 [n], the device of each rank, or
 * NULL = cfg->device for all; ranks on different devices use peer access.
 * Several ranks may share one device (e.g. an EP group emulated with the real
 * multi-rank data plane on one GPU): each then runs its persistent GEMM grids on
 * (SMs - 16) / (ranks on the device) SMs, so every rank's kernels co-reside;
 * s ranks on one device need CUDA_DEVICE_MAX_CONNECTIONS >= 2s hardware queues
 * (default 8: up to 4 ranks), else MOE_ERR_UNSUPPORTED.
 * cfg->world and cfg->rank are ignored; cfg->virtual_ranks must be <= 1.  Every
 * rank's calls are issued on its own stream(s); a rank's collective calls may be
 * issued from one host thread in rank order (no call blocks on a peer) -- except
 * moe_dispatch with info != NULL, moe_ctx_sync and the debug / timing reads,
 * which synchronise and so must come after every rank's calls they depend on.
 * Copy-engine mode (environment MOE_A2A_CE=1, P2P, tp 1): moe_dispatch of a
 * multi-process rank blocks until this dispatch's count matrix is known (it
 * queues the peer copies); a group rank's moe_expert_ffn does, so every rank's
 * moe_dispatch must precede any rank's moe_expert_ffn.  Not used while the stream
 * is being captured into a CUDA graph. */
moe_status moe_ctx_create_group(const moe_config* cfg, int32_t n, const int32_t* devices, moe_ctx_t* out);
/* Collective when world > 1 (starts with a barrier over the group, so no peer
 * still reads this rank's mapped buffers).  A single-process group's context
 * synchronises every device of the group first. */
moe_status moe_ctx_destroy(moe_ctx_t ctx);
moe_status moe_ctx_sync(moe_ctx_t ctx);                   /* sync the last stream; surfaces MOE_ERR_DEVICE */
const char* moe_status_str(moe_status s);
const char* moe_last_error(moe_ctx_t ctx);                /* "" if none; ctx may be NULL */
int32_t moe_abi_version(void);                            /* MOE_ABI_VERSION */
#define MOE_ABI_VERSION 3   /* 2: moe_config.tp; 3: device expert_to_rank, moe_expert_ffn n_w, groups */

/* ---- a1: gating (G1, G2, G3) -------------------------------------
 * For each token t: idx[t][0..k-1] = the k largest logits[t][.] in descending
 * order, ties to the lower expert id, -0.0 == +0.0; w[t][j] = softmax over the
 * k selected logits = exp(l_j - l_0) / sum_j' exp(l_j' - l_0) (fp32).
 * logits: float [T][E]; idx: int32 [T][k]; w: float [T][k].  Rank-local.
 * A NaN logit latches MOE_ERR_DEVICE (reading G3: logits are finite). */
moe_status moe_route(moe_ctx_t ctx, const float* logits, int32_t T, int32_t E, int32_t k,
                     int32_t* idx, float* w, moe_stream_t stream);

/* ---- a2: routing statistics (P:L581 P_{e,l}; P:L654 R_{e1,e2,l}; G10) ----------
 * load[e]        += #{(t,j)      : idx_l[t][j] == e}
 * coact[e1][e2]  += #{(t,j1,j2)  : idx_l[t][j1] == e1 && idx_l1[t][j2] == e2}
 * idx_l, idx_l1: int32 [T][k], the same token rows at layers l and l+1
 * (idx_l1 may be NULL: then coact is not touched).  load: int64 [E],
 * coact: int64 [E][E] e1-major; both ACCUMULATE (caller zeroes them).
 * Out-of-range ids latch MOE_ERR_DEVICE.  Rank-local; see moe_stats_allreduce. */
moe_status moe_route_stats(moe_ctx_t ctx, const int32_t* idx_l, const int32_t* idx_l1,
                           int32_t T, int32_t E, int32_t k, int64_t* load, int64_t* coact,
                           moe_stream_t stream);

/* Sum load [E] and coact [E][E] (int64, in place) over the EP group (NCCL
 * all-reduce).  No-op when world == 1.  coact may be NULL. */
moe_status moe_stats_allreduce(moe_ctx_t ctx, int64_t* load, int64_t* coact, int32_t E,
                               moe_stream_t stream);

/* The same for a whole profiling pass in one collective: load int64 [L][E] and
 * coact int64 [L-1][E][E] (coact may be NULL; L >= 1), e.g. the per-layer
 * statistics of moe_route_stats over L layers (P:L581 P_{e,l}, P:L654 R_{e1,e2,l}). */
moe_status moe_stats_allreduce_layers(moe_ctx_t ctx, int64_t* load, int64_t* coact, int32_t E, int32_t L,
                                      moe_stream_t stream);

/* ---- a3-a5: dispatch (G7, G8, G9, G13, G14) ---
 * x: bf16 [T][H] (this process's tokens); idx: int32 [T][k] from moe_route.
 * expert_to_rank: DEVICE int32 [E], values in [0, G/tp) (the placement input --
 * "the custom expert-to-GPU mapping is loaded and applied", P:L515-519 -- the EP
 * rank, with tp > 1 the EP group, hosting each expert; a rank may host 0
 * experts).  It is read by the kernels this call enqueues (stream order), so a
 * per-layer placement is just another device array: no host synchronisation,
 * and a multi-layer chain with per-layer placements can be captured in one CUDA
 * graph.  Its values are validated on the device: one outside [0, G/tp) latches
 * MOE_ERR_DEVICE (and is treated as 0); MOE_A2A_NCCL, which reads the placement
 * on the host anyway, returns MOE_ERR_INVALID_ARG from this call instead.
 * Builds the stable send order (key P[e], e, t), the
 * expert-major receive layout (e ascending on g, then source s, then t; each
 * expert segment padded to the GEMM M tile) and moves every routed row to the rank
 * hosting its expert.  Collective when world > 1 (NCCL mode synchronises the
 * stream once to read the G x E count matrix).  The plan stays in the context
 * until the next moe_dispatch.  info: host, optional; if non-NULL the call
 * synchronises `stream` and fills it.  A hash of expert_to_rank travels with the
 * counts and every rank checks that all ranks dispatched with the same placement:
 * MOE_A2A_P2P latches MOE_ERR_DEVICE on the device (reported by the next
 * synchronising call); MOE_A2A_NCCL all-gathers the maps themselves and returns
 * MOE_ERR_DEVICE from this call.
 * CUDA graphs: a whole layer (moe_route .. moe_combine) may be captured and
 * replayed on a stream (not in MOE_A2A_NCCL mode, whose dispatch reads the
 * counts on the host).  In MOE_A2A_P2P mode the flag epoch lives on the device
 * and advances once per dispatch, so every rank must replay its graph the same
 * number of times, in the same order as its other collective calls; the
 * captured placement array is read at replay time. */
moe_status moe_dispatch(moe_ctx_t ctx, const moe_bf16* x, const int32_t* idx, int32_t T, int32_t k,
                        const int32_t* expert_to_rank, moe_dispatch_info* info,
                        moe_stream_t stream);

/* ---- NEXT-4: direct layer l -> l+1 dispatch (Eq. 8; reading G11) -------
 * Eq. 8 models token traffic from the GPU hosting a token's layer-l expert to the
 * GPU hosting its layer-(l+1) expert.  Home-rank EP (moe_combine, then the next
 * moe_dispatch from the token's home) never puts that traffic on the wire; this
 * pair of calls does.  moe_set_output_mode(prev, MOE_OUT_STAY) before layer l's
 * moe_expert_ffn keeps layer l's expert outputs on the hosting ranks (no
 * moe_combine for that layer).  moe_dispatch_from(ctx, prev, w_prev, idx, T, k,
 * expert_to_rank) then dispatches layer l+1 (ctx, another context of the same
 * rank and EP group; idx and expert_to_rank as in moe_dispatch) without a
 * hidden-state row: every rank hosting a layer-(l+1) expert of token t forms its
 * receive row itself as
 *     x_{l+1}[t] = bf16( sum_{j ascending} w_prev[t][j] * Y_l[item (t, j)] )
 * (G4: fp32 FMA, one bf16 rounding -- bit-identical to the home-rank combine),
 * reading Y_l where layer l computed it: locally when both experts share a GPU
 * (what ILP 2 arranges), over NVLink otherwise.  The source sends only 12 bytes
 * per routed row and layer-l item (slot, row, weight).  w_prev: float [T][k_l]
 * (layer l's gate weights, device).  T must equal layer l's T on this rank.
 * Collective like moe_dispatch; P2P, virtual ranks or one rank; tp == 1.  The
 * last layer of a chain returns home with moe_combine (MOE_OUT_HOME, default). */
typedef enum { MOE_OUT_HOME = 0, MOE_OUT_STAY = 1 } moe_output_mode;
moe_status moe_set_output_mode(moe_ctx_t ctx, int32_t mode);
moe_status moe_dispatch_from(moe_ctx_t ctx, moe_ctx_t prev, const float* w_prev, const int32_t* idx, int32_t T,
                             int32_t k, const int32_t* expert_to_rank, moe_stream_t stream);

/* ---- a6: grouped SwiGLU expert FFN (G5) ---------------------------------
 * For every hosted expert e and its received rows X_e:
 *   h = bf16( silu(X_e W1_e^T) * (X_e W3_e^T) ),  Y_e = bf16( h W2_e^T )
 * with fp32 accumulation on tcgen05 tensor cores.  w13: bf16 packed
 * [n_w][2F][H] (see moe_pack_w13), w2: bf16 [n_w][H][F]; n_w experts in
 * ascending global id: the experts the last dispatch's placement hosts here
 * (real mode; 0 allowed, w13/w2 may then be NULL) or all E (virtual: n_w must
 * be E).  Since the placement is a device array, n_w is checked on the device:
 * a count that differs from the hosted experts latches MOE_ERR_DEVICE (weight
 * rows past n_w read as zeros, no out-of-bounds access).
 * tp > 1, real ranks: this rank's slice q = rank % tp only, F_q = F / tp:
 *   w13 = moe_pack_w13(W1[:, qF_q:(q+1)F_q, :], W3[same rows], n_w, F_q, H) [n_w][2F_q][H],
 *   w2  = W2[:, :, qF_q:(q+1)F_q] made contiguous                          [n_w][H][F_q];
 * Y is then this slice's bf16 partial output.  tp > 1, virtual ranks: the full
 * w13 / w2 as above; every slice's partial output is computed separately.
 * Decode-sized contexts may split the down projection over F (fp32 partials in
 * a context-owned workspace, summed in a fixed order before the bf16 rounding),
 * so Y can differ from an unsplit run in the last bf16 bit; the result is
 * deterministic for a given context.
 * Collective in MOE_A2A_P2P mode: every rank calls it after moe_dispatch, also
 * a rank hosting no expert (w13/w2 may then be NULL) -- it raises the flag the
 * peers' moe_combine waits for. */
moe_status moe_expert_ffn(moe_ctx_t ctx, const moe_bf16* w13, const moe_bf16* w2, int32_t n_w,
                          moe_stream_t stream);

/* ---- a7-a8: combine (G4) -------------------------------------------------
 * Returns every expert output row to its source rank and writes
 * out[t] = bf16( sum_{j ascending} w[t][j] * Y[item (t,j)] ) in fp32; with
 * tp > 1, Y[item] = sum_{q ascending} (partial output of TP slice q) in fp32.
 * w: float [T][k] (from moe_route); out: bf16 [T][H].  Uses the plan of the
 * last moe_dispatch (same T, k).  Collective when world > 1. */
moe_status moe_combine(moe_ctx_t ctx, const float* w, moe_bf16* out, moe_stream_t stream);

/* ---- helpers ---------------------------------------------------------------------- */

/* Pack per-expert W1, W3 ([n][F][H] each) into w13 [n][2F][H]: for every
 * 128-row block b of F (64 if F % 128 != 0), rows [2b*B, 2b*B+B) = W1 block b and
 * rows [2b*B+B, 2b*B+2B) = W3 block b, B = block size, so one GEMM N-tile holds
 * matching gate and up columns.  Device pointers, async on `stream`. */
moe_status moe_pack_w13(const moe_bf16* w1, const moe_bf16* w3, int32_t n, int32_t F, int32_t H,
                        moe_bf16* w13, moe_stream_t stream);

/* Megatron's contiguous placement: out[e] = e / (E/G).  out: host
 * int32 [E].  E % G != 0 => MOE_ERR_INVALID_ARG. */
moe_status moe_placement_contiguous(int32_t E, int32_t G, int32_t* out);

/* Host-side dispatch layout (the arithmetic NCCL mode uses to post its
 * send/recv segments; exported for CPU tests).  Inputs host: P [E], cnt [G][E].
 * Outputs host (any may be NULL):
 *   seg_start [E]  padded start row of expert e's segment on rank P[e]
 *   recv_base [G][E] receive row of the first item of (source s, expert e)
 *   recv_rows [G]  unpadded routed rows received by rank g
 *   send_base [G][E] position of the first item of (s, e) in s's send order */
moe_status moe_layout_host(int32_t E, int32_t G, const int32_t* P, const int32_t* cnt,
                           int32_t* seg_start, int32_t* recv_base, int32_t* recv_rows,
                           int32_t* send_base);

/* ---- debug / test views (synchronise the context's last stream) ------------------- */

/* Copies the plan of the last moe_dispatch to host arrays sized for the T and k
 * of that call (any pointer may be NULL):
 *   dest_rank [T][k]  rank (EP group when tp > 1) hosting item (t, j)'s expert
 *   recv_pos  [T][k]  unpadded position of the item in that rank's receive order
 *   send_slot [T][k]  position of the item in its source's send order (C3 slot), as
 *                     computed by the device (the fused combine's return slot)
 *   cnt       [G][E]  count matrix of all ranks. */
moe_status moe_debug_plan(moe_ctx_t ctx, int32_t* dest_rank, int32_t* recv_pos,
                          int32_t* send_slot, int32_t* cnt);

/* Expert FFN replaced by the identity (Y = received rows; with tp > 1 TP slice 0
 * returns the rows and the other slices zeros), for bit-exact dispatch/combine
 * tests (out must equal x). */
moe_status moe_debug_identity_ffn(moe_ctx_t ctx, moe_stream_t stream);

/* MOE_A2A_NCCL mode: copies the compact send buffer of the last dispatch -- this
 * rank's rows for remote experts, in the C3 send order (key P[e], e, t; G9) -- to
 * host bf16 [rows][H] (rows_host may be NULL to query *rows_out).  Copy-engine
 * mode (MOE_A2A_CE, P2P): the staging buffer, indexed by the full C3 send-order
 * slot (rows = this rank's routed items; the slots of its own experts' items are
 * not staged); single-process groups: after the rank's moe_expert_ffn.  Other
 * modes have no send buffer (MOE_ERR_UNSUPPORTED): P2P stores rows straight into
 * the peers' receive buffers, virtual ranks into the shared receive buffer. */
moe_status moe_debug_send(moe_ctx_t ctx, moe_bf16* rows_host, int64_t max_rows, int64_t* rows_out);

/* Copies the received rows of the last dispatch, in unpadded receive order of
 * this process (virtual: rank 0's rows first, ...), to host bf16 [rows][H].
 * P2P: waits for every source's rows first (a latched flag timeout is returned);
 * copy-engine mode in a single-process group: after every rank's moe_expert_ffn
 * (which queues that rank's copies). */
moe_status moe_debug_recv(moe_ctx_t ctx, moe_bf16* rows_host, int64_t max_rows, int64_t* rows_out);

/* Number of kernels this context has launched since creation (for the bench's
 * gpu_launches count). */
int64_t moe_kernel_launches(moe_ctx_t ctx);

/* Per-kernel timing of moe_expert_ffn.  moe_ffn_timing_enable(ctx, n) arms n
 * records (0 disarms): each of the next n moe_expert_ffn calls records CUDA
 * events on its stream around the K5 (gate/up + SwiGLU) and K6 (down) GEMM
 * launches -- no host synchronisation.  moe_ffn_timing_read synchronises on
 * the recorded events, writes ms[i][0] = K5 and ms[i][1] = K6 durations in
 * milliseconds for every record i < *n_out (host float [max_records][2]) and
 * re-arms the records. */
moe_status moe_ffn_timing_enable(moe_ctx_t ctx, int32_t max_records);
moe_status moe_ffn_timing_read(moe_ctx_t ctx, float* ms, int32_t max_records, int32_t* n_out);

/* Layer timeline (profiling).  moe_timeline_enable(ctx, n) arms n records (0
 * disarms); each of the next n moe_dispatch -> moe_expert_ffn -> moe_combine
 * sequences records 8 CUDA events: 0 dispatch entry, 1 after the plan/layout
 * kernels (P2P: includes the count all-gather), 2 after the scatter on `stream`
 * (P2P: this rank's own rows), 3 after the scatter of the peers' rows (P2P side
 * stream; else = 2), 4 expert_ffn entry, 5 after K5, 6 after K6, 7 after the
 * combine kernel.  moe_timeline_read synchronises the device and writes
 * ms[i][j] = event j - event 0 of record i in milliseconds (host float
 * [max_records][8]; -1 for an event that was not recorded), then re-arms. */
moe_status moe_timeline_enable(moe_ctx_t ctx, int32_t max_records);
moe_status moe_timeline_read(moe_ctx_t ctx, float* ms, int32_t max_records, int32_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* MOE_H */
