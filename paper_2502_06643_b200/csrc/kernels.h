// kernels.h -- host-side launch entry points of the libmoe kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace moe {

// K1 / K9 (route.cu)
void launch_route(const float* logits, int T, int E, int k, int32_t* idx, float* w, int* err, cudaStream_t s);
void launch_route_stats(const int32_t* idx_l, const int32_t* idx_l1, int T, int E, int k, int64_t* load,
                        int64_t* coact, int* err, int num_sms, cudaStream_t s);

// Shared signal block of one rank (P2P mode), exported to its peers through
// CUDA IPC.  Peers write their count rows and raise epoch-valued flags here.
struct SigBlock {
  int cnt[64 * 256];          // [G][E] count matrix (row s written by source s)
  unsigned flag_cnt[64];      // flag_cnt[s] = epoch once source s's count row landed
  unsigned flag_data[64];     // flag_data[s] = epoch once every row s sends here landed
  unsigned flag_y[64];        // flag_y[g] = epoch once rank g's expert outputs are ready
  unsigned phash[64];         // phash[s] = hash of the placement source s dispatched with
  unsigned flag_exp[64];      // gather dispatch: flag_exp[s] = epoch once this rank expanded source
                              // s's token rows into its receive layout (local flag; [me] too)
  unsigned flag_se[64 * 256]; // copy-engine dispatch: flag_se[s][e] = epoch once source s's rows
                              // for expert e landed here (a stream memory write after the copy)
};

// Dispatch plan arguments shared by K2/K3/K8 (dispatch.cu).
struct PlanArgs {
  int T;        // tokens of this process in this call
  int k;
  int E;
  int H;
  int V;        // sources handled by this process (1 real, G virtual)
  int G;        // ranks (sources): the EP group size, or EP groups x tp
  int me;       // real rank (0 in virtual mode)
  int tp;       // tensor-parallel ranks per EP group (1: none); P[e] is an EP group id
  int grp;      // this rank's EP group (me / tp)
  int virt;     // 1 = virtual ranks (every expert hosted by this process)
  int p2p;      // 1 = in-kernel NVLink peer stores/loads (real ranks)
  const unsigned* epoch_ptr;  // P2P: device word holding this dispatch's flag value
                             // (k_layout increments it, so captured CUDA graphs replay correctly)
  int n_tiles;  // sum over sources of ceil(T_s / kTileTokens)
  int col_split;  // K3/K8: CTAs per token tile, each copying a slice of the hidden dim
  int plan_done;  // the plan arrays of this dispatch were written already (mode 3): mode 1 skips them
  int seg_align;  // expert segments are padded to this many rows (= the GEMM M tile, 128 or 256)
  int fused;      // K8 reads the local return buffer at the C3 slot (fused-combine mode)
  int gather;     // P2P gather dispatch: token rows reach the peers by copy engine, rows are
                  // expanded into the expert-major layout on the receiver (k_expand)
  unsigned long long timeout_ns;  // bound on every P2P flag wait (latches MOE_ERR_TIMEOUT)
  int direct;     // direct layer l -> l+1 dispatch (moe_dispatch_from): the receive rows are
                  // combined on the hosting rank from layer l's expert outputs (k_expand_direct)
  int ce;         // copy-engine data plane (P2P): K3 stages the peers' rows in the send buffer
                  // (send order) for the copy engines; K8 reads the peers' returned rows from the
                  // return buffer and this rank's own rows from its expert-output buffer
};

// Device-side plan state (allocated by the context).
struct PlanBuffers {
  const int32_t* P_in;   // [E] the caller's expert_to_rank of this dispatch (device)
  int32_t* P;            // [E] context copy, validated by k_layout (read by the later kernels)
  int32_t* tile_hist;    // [n_tiles][E]
  int32_t* tile_base;    // [n_tiles][E]  within-source exclusive prefix
  int32_t* cnt_local;    // [V][E]
  const int32_t* cnt_all;  // [G][E] (NCCL/virtual); P2P reads SigBlock::cnt of this rank
  int32_t* base_row;     // [V][E] destination row of the first item of (s, e)
  int32_t* seg_meta;     // [1 + 3E + 4]: nseg, seg_row0[E], seg_rows[E], seg_w[E], totals
  int32_t* row_of_item;  // [T*k] destination row (-1: invalid expert id)
  uint8_t* slot_of_item; // [T*k] index into dst_table / src_table
  uint4* const* dst_table;        // scatter destinations by slot
  const uint4* const* src_table;  // combine sources by slot
  SigBlock* const* peer_sig;      // [G] (P2P) every rank's signal block, own included
  SigBlock* my_sig;               // (P2P) this rank's signal block
  unsigned* done_counter;         // last-CTA detection in k_scatter
  int* err;
  // fused combine (P2P): K6 stores each expert-output row straight into the
  // source rank's return buffer at the item's send-order slot (C3 slot)
  uint4* sendbuf;                 // copy-engine mode: the staged peers' rows, in send order
  int32_t* seg_src;               // [E][G][3]: per hosted segment and source: first row, rows, first slot
  int32_t* cslot_base;            // [V][E] send-order slot of local source s's first item for expert e
  int32_t* cslot_of_item;         // [T*k] send-order slot (C3) of every item (within its source)
  const uint4* ret_local;         // this rank's return buffer
  // tp > 1: the tp partial outputs of one item live part_stride uint4 apart (virtual
  // mode: the expert-output buffers of the slices; fused combine: the return buffers)
  long long part_stride;
  // gather dispatch (P2P): every token row lands once in tok [G][tok_rows][H] of every peer
  // hosting one of its experts; the source writes, for each of its rows a peer receives, the
  // token-buffer row into that peer's xmap [cap_rows]; the peer's k_expand copies the rows
  uint4* recv_local;              // this rank's receive buffer
  const uint4* tok_local;         // this rank's token buffer
  const int32_t* xmap_local;      // this rank's row -> token-buffer row map
  int32_t* const* xmap_table;     // [G] every rank's xmap
  uint4* const* tok_table;        // [G] every rank's token buffer
  unsigned* exp_counter;          // [G] k_expand last-CTA detection per source
  long long tok_rows;             // token-buffer rows per source (max_tokens)
  const int32_t* seg_meta_c;      // segment table (nseg at [0]) for k_expand
  // direct layer l -> l+1 dispatch: per receive row, prev_k descriptors {slot, row, w} of
  // the layer-l expert-output rows it combines (desc [cap_rows][desc_k][3] int32 per rank)
  int32_t* const* desc_table;     // [G] every rank's descriptor buffer (virtual: [0] = own)
  const int32_t* desc_local;
  int desc_k;                     // descriptor slots per row (the context's max_k)
  const int32_t* prev_row;        // layer l's row_of_item [T*prev_k] (this rank)
  const uint8_t* prev_slot;       // layer l's slot_of_item (hosting rank / buffer slot)
  const float* prev_w;            // layer l's gate weights [T][prev_k]
  int prev_k;
  const uint4* const* prev_src;   // layer l's expert-output buffers by slot (this rank's table)
  const unsigned* prev_flag_y;    // layer l's flag_y in this rank's layer-l signal block (P2P)
  const unsigned* prev_epoch;     // layer l's flag epoch
  int32_t* seg_e;                 // [E] global expert id of hosted segment i (k_layout)
};

// K5 per-tile arrival waits (P2P overlap): the producer waits only for the source
// ranks whose rows a tile reads; tiles holding only this rank's own rows run first.
struct SrcWait {
  const unsigned* flags;          // SigBlock::flag_data [G] of this rank; nullptr = no waits
  // copy-engine dispatch: wait per (source, segment) on flags_se[s * E + seg_e[seg]]
  // instead (nullptr: per source on flags)
  const unsigned* flags_se;
  const int32_t* seg_e;
  int E;
  const int32_t* seg_src;         // see PlanBuffers::seg_src
  int G;
  int me;
  const unsigned* epoch_ptr;      // see PlanArgs::epoch_ptr
  unsigned long long timeout_ns;  // see PlanArgs::timeout_ns
};

// K6 epilogue redirection (fused combine, P2P mode); enabled == 0 -> plain stores.
struct FusedRet {
  uint16_t* const* ret_table;     // [G] every rank's return buffer
  const int32_t* seg_src;         // see PlanBuffers::seg_src
  int G;
  int enabled;
  // copy-engine combine (plain stores): every epilogue warp adds 1 to segdone[segment]
  // once its stores of a tile have completed, so the copy engines' stream (waiting on
  // the value with cuStreamWaitValue32) returns a segment's rows as soon as it is done
  unsigned* segdone;
};

// Load every kernel of the library onto the current device now (CUDA 12 loads
// modules lazily, at a function's first launch; a first launch may wait for the
// device's running kernels -- and in a single-process EP group a running kernel
// can be spinning on a flag that only a later launch of this thread raises).
void preload_route_kernels();
void preload_dispatch_kernels();
void preload_gemm_kernels();

int plan_tiles(int T, int V);
void launch_count(const PlanArgs& a, const int32_t* idx, const PlanBuffers& b, cudaStream_t s);
void launch_scan(const PlanArgs& a, const PlanBuffers& b, cudaStream_t s);
void launch_layout(const PlanArgs& a, const PlanBuffers& b, int64_t cap_rows, cudaStream_t s);
// mode 0: all rows; P2P: 3 = the plan arrays only (before the TMA push of the peers' rows),
// 1 = rows hosted here,
// 5 = gather dispatch: only the row -> token-buffer map entries of the peers' rows,
// 6 = direct dispatch: the combine descriptors of every row (all destinations, own included)
void launch_scatter(const PlanArgs& a, const uint16_t* x, const int32_t* idx, const PlanBuffers& b, int mode,
                    cudaStream_t s, int max_ctas = 0);  // max_ctas > 0: persistent grid of that size
void launch_combine(const PlanArgs& a, const float* w, const PlanBuffers& b, uint16_t* out, cudaStream_t s);
// Direct dispatch: every receive row = bf16(sum_j w_j * Y_l[slot_j][row_j]) (fp32 FMA, j
// ascending -- the home-rank combine's arithmetic); P2P: after every source's descriptors
// (flag_data) and every rank's layer-l outputs (layer-l flag_y) arrived; raises flag_exp.
void launch_expand_direct(const PlanArgs& a, const PlanBuffers& b, int max_ctas, cudaStream_t s);
// P2P dispatch of the peers' rows on the TMA engines: one warp per CTA bulk-copies each
// token row (in 4 KB pieces) from x into shared memory once and from there into every
// remote receive row of its items; reads the plan arrays (mode 3); raises flag_data.
void launch_push_tma(const PlanArgs& a, const uint16_t* x, const PlanBuffers& b, int ctas, cudaStream_t s);
// Gather dispatch: expand every peer's token rows (token buffer -> receive layout),
// source by source as each source's flag_data arrives; raises flag_exp per source.
void launch_expand(const PlanArgs& a, const PlanBuffers& b, int max_ctas, cudaStream_t s);
// P2P: raise flag `which` (0 cnt, 1 data, 2 y) = epoch on every rank, after a system fence.
void launch_signal(const PlanArgs& a, const PlanBuffers& b, int which, cudaStream_t s);
// P2P: wait until flags[0..n) >= epoch (system-scope acquire).
void launch_wait(const unsigned* flags, int n, const unsigned* epoch_ptr, int* err, unsigned long long timeout_ns,
                 cudaStream_t s);
// Latch kErrWeights unless the last layout hosts exactly n expert segments here.
void launch_expect_nseg(const int32_t* seg_meta, int n, int* err, cudaStream_t s);
void launch_pack_w13(const uint16_t* w1, const uint16_t* w3, int n, int F, int H, uint16_t* w13,
                     cudaStream_t s);

// K5/K6 grouped GEMM (gemm.cu).
int gemm_block_n(int N, bool swiglu);
int gemm_b_box_rows(int N, bool swiglu, int cg);  // TMA box rows of the B (weight) operand per CTA
int pack_block(int F);
// Launch the persistent grouped GEMM: D[rows][ldd] for every hosted expert segment.
// tmA / tmB are CUtensorMap (128 bytes each) built by make_tmap_2d.  If wait_flags is
// non-NULL the kernel first waits until wait_flags[0..wait_n) >= epoch (P2P arrivals).
// cg = CTAs per MMA (2: tcgen05 cta_group::2, 256-row tiles; 1: 128-row tiles for
// small token counts); must match the segment padding of the dispatch layout.
cudaError_t launch_grouped_gemm(const void* tmA, const void* tmB, uint16_t* D, int ldd, const int32_t* seg_meta,
                                int E, int n_w, int N, int K, bool swiglu, int cg, int num_sms, const SrcWait& sw, int* err,
                                unsigned* sched, const FusedRet& fr, cudaStream_t s, int ksplit = 1,
                                float* part = nullptr, long long part_stride = 0, const void* tmD = nullptr);
// tmD: TMA-store map of D (make_tmap_store_2d) for the plain / SwiGLU epilogues.
// ksplit > 1 (plain GEMMs, no fused combine): fp32 partials of the K slices go to
// part[slice][row][N]; launch_splitk_reduce then writes D = bf16(sum over slices).
cudaError_t launch_splitk_reduce(const float* part, long long part_stride, int S, const int32_t* seg_meta, int E,
                                 int N, int cg, uint16_t* D, int ldd, int num_sms, cudaStream_t s);
// sched: 2 zero-initialised device counters (tile counter, exit counter) owned by the
// caller; the kernel resets them to 0 when it completes.
// Encode a 2D bf16 K-major tensor map [rows][cols] with box {64, box_rows}, 128B swizzle.
bool make_tmap_2d(void* tmap_out, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows);
// Same with a row pitch of ld elements (a column slice of a wider matrix).
bool make_tmap_2d_ld(void* tmap_out, const void* base, uint64_t rows, uint64_t cols, uint64_t ld,
                     uint32_t box_rows);
// Store map for the GEMM epilogue: bf16 [rows][cols] with pitch ld, box {32, 32}, no swizzle.
bool make_tmap_store_2d(void* tmap_out, const void* base, uint64_t rows, uint64_t cols, uint64_t ld);

}  // namespace moe
