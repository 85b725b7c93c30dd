// moe_api.cu -- the C ABI of libmoe (include/moe.h): context, validation,
// workspace ownership, NCCL orchestration of the all-to-all, launches.
#include <nccl.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/moe.h"
#include "common.cuh"
#include "kernels.h"

using namespace moe;

struct moe_ctx {
  moe_config cfg{};
  int G = 1, V = 1, me = 0, virt = 0;
  // tensor parallelism inside the experts (G20): EP group grp = me / tp, TP index
  // tpi = me % tp; Fl = the FFN width this process computes per GEMM (F / tp for
  // real TP ranks; F in virtual mode, whose K6 runs once per slice)
  int tp = 1, grp = 0, tpi = 0, Fl = 0;
  int num_sms = 148;
  int E = 0, H = 0, F = 0;
  cudaStream_t last_stream = nullptr;
  ncclComm_t comm = nullptr;
  std::string err;
  int64_t launches = 0;

  // placement of the last dispatch: the caller passes it as a device array; k_layout
  // validates it and copies it here (NCCL mode also all-gathers every rank's copy
  // into P_all and reads it on the host with the counts)
  int32_t* P_dev = nullptr;
  int32_t* P_all = nullptr;         // NCCL mode: [G][E]
  int32_t* P_all_pinned = nullptr;  // [G][E] host staging
  std::vector<int32_t> P_host;      // NCCL mode: this rank's row of P_all after the sync

  // plan workspaces
  int max_tiles = 0;
  int32_t* tile_hist = nullptr;
  int32_t* tile_base = nullptr;
  int32_t* cnt_local = nullptr;
  int32_t* cnt_all = nullptr;
  int32_t* base_row = nullptr;
  int32_t* seg_meta = nullptr;
  int32_t* row_of_item = nullptr;
  int* err_dev = nullptr;
  int32_t* cnt_pinned = nullptr;  // host copy of cnt_all (NCCL mode / debug)

  // payload buffers
  int64_t cap_rows = 0;      // receive-layout rows (padded)
  int64_t send_rows = 0;     // remote send rows (NCCL mode)
  uint16_t* recv = nullptr;  // [cap_rows][H]
  uint16_t* hbuf = nullptr;  // [cap_rows][F]
  uint16_t* ybuf = nullptr;  // [cap_rows][H]
  uint16_t* sendbuf = nullptr;  // [send_rows][H]
  uint16_t* retbuf = nullptr;   // [send_rows][H]
  alignas(64) uint8_t tmA1[128];  // A of GEMM1: recv [cap][H]
  alignas(64) uint8_t tmA2[128];  // A of GEMM2: hbuf [cap][F]
  alignas(64) uint8_t tmB1[128];
  alignas(64) uint8_t tmB2[128];
  alignas(64) uint8_t tmA2s[kMaxTP][128];  // virtual TP: h column slice q
  alignas(64) uint8_t tmDh[128];           // epilogue TMA-store maps: h [cap][Fl]
  alignas(64) uint8_t tmDy[128];           //   y [cap][H]
  alignas(64) uint8_t tmDys[kMaxTP][128];  //   virtual TP: partial-output buffer q
  alignas(64) uint8_t tmB2s[kMaxTP][128];  // virtual TP: W2 column slice q
  const void* tmB1_ptr = nullptr;
  const void* tmB2_ptr = nullptr;
  int tmB_nw = -1;
  // split-K workspace for K6 in decode-sized contexts (fp32 partials [S][cap][H])
  float* splitk_ws = nullptr;
  size_t splitk_bytes = 0;

  // optional K5/K6 timing event records (3 events per moe_expert_ffn call)
  std::vector<cudaEvent_t> ev;
  int timing_used = 0;
  // optional layer timeline: kTimeline events per dispatch -> expert_ffn -> combine
  std::vector<cudaEvent_t> tl;
  std::vector<uint8_t> tl_mask;  // [record] bit j = event j recorded
  int tl_used = 0, tl_cur = -1;

  // per-item destination slot, pointer tables (slot -> buffer), P2P state
  uint8_t* slot_of_item = nullptr;
  uint4** dst_table = nullptr;          // device [max(G,2)]
  const uint4** src_table = nullptr;    // device [max(G,2)]
  SigBlock** peer_sig = nullptr;        // device [G]
  SigBlock* sig = nullptr;              // this rank's signal block (IPC-exported)
  unsigned* done_counter = nullptr;
  bool p2p = false;
  unsigned* epoch_dev = nullptr;        // P2P flag value, advanced on the device by k_layout
  // GEMM M tile / segment padding: 256 rows (CTA pair) or, when the context's worst
  // case averages <= 256 routed rows per expert (decode-sized batches), 128 rows on
  // one CTA -- halving the MMA work spent on padding rows.  Fixed per context so
  // every rank derives the same receive layout.
  int seg_align = kSegAlign;
  int gemm_cg = kGemmCG;
  std::vector<void*> ipc_opened;        // peer mappings to close
  // fused combine (P2P): K6 stores expert outputs into the sources' return buffers
  int32_t* seg_src = nullptr;           // [E][G][3]
  int32_t* cslot_base = nullptr;        // [E]
  int32_t* cslot_of_item = nullptr;     // [max_tokens * k]
  uint16_t** ret_table = nullptr;       // device [G]
  bool ffn_fused = false;               // the last expert FFN already returned its rows
  // P2P overlap: rows for peers are pushed on a side stream while K5 starts on
  // this rank's own rows (fork after the layout kernel, join in combine).  (A
  // send-order push with per-(source, expert) arrival flags measured slower at E64
  // 4EP -- 6.87 vs 6.64 ms, round 1 -- and was removed.)
  cudaStream_t side = nullptr;
  // CTAs of the peers'-rows scatter that overlaps K5 (persistent grid; 0 = one per
  // tile x column slice).  32 CTAs still fill NVLink and leave the other SMs to
  // K5: D5 4EP step 6.24 ms vs 6.73 (one CTA per tile), 6.53 (16), 6.28 (64),
  // 6.59 (128) in one run (profiles/r1_v13_timeline_ctas_*); Mixtral 4EP unchanged.
  // MOE_SCATTER_CTAS overrides.
  int remote_ctas = 32;
  // gather dispatch (P2P): with top-k >= G/tp a token usually has
  // several experts on one rank, so each token row crosses NVLink once per
  // destination rank (not once per routed row), with a 4-byte row -> token index
  // per routed row, and the receiver expands its rows locally (k_expand).  Opt-in
  // (MOE_DISPATCH=gather): at E64 top-8 on 4 GPUs it halves the NVLink bytes, but
  // the receiver's expansion costs more SM time next to K5 than the push saves
  // (DESIGN.md §11).  (Copy-engine block
  // copies were tried first: one peer cudaMemcpyAsync moves ~90 GB/s on this
  // machine, profiles/r2_ce_probe.json -- far below the SMs' NVLink stores.)
  uint16_t* tokbuf = nullptr;           // [G][max_tokens][H]: every source's token block
  int32_t* xmap = nullptr;              // [cap_rows]: receive row -> token-buffer row
  int32_t** xmap_table = nullptr;       // device [G]
  void** tok_table = nullptr;           // device [G]
  unsigned* exp_counter = nullptr;      // [G]
  std::vector<void*> tok_peer;          // host [G]: every rank's token buffer (peer pointers)
  bool last_gather = false;             // the last dispatch used the gather path
  // direct layer l -> l+1 dispatch (NEXT-4): combine descriptors [cap_rows][max_k][3]
  // of this rank's receive rows (written by the sources), peers' tables
  int32_t* desc = nullptr;
  int32_t** desc_table = nullptr;       // device [max(G, 1)]
  bool last_direct = false;             // the last dispatch was moe_dispatch_from
  // copy-engine data plane (MOE_A2A_CE, P2P): the dispatch stages the peers' rows in
  // the send buffer; moe_expert_ffn reads the count matrix on the host and queues, on
  // the side stream, one peer copy per (destination, expert) run plus a flag write per
  // destination, and for the combine, per hosted segment, a wait on K6's segment
  // counter and one copy per source run, then flag_y on every rank.  The copy engines
  // move the rows, so no SM shares its TMA unit or issue slots with the GEMMs.
  bool last_ce = false;
  cudaEvent_t ev_cnt = nullptr, ev_staged = nullptr, ev_k6 = nullptr, ev_side2 = nullptr;
  cudaStream_t side2 = nullptr;         // second copy-engine stream (the combine's runs alternate)
  int32_t* ce_pinned = nullptr;         // host: count matrix [G][E], placement [E], epoch, error word
  unsigned* segdone = nullptr;          // [E] K6 per-segment completion counters
  std::vector<void*> recv_h, sig_h, ret_h;  // host copies of the peer tables (P2P)
  bool ce_dispatched = false;           // this dispatch's copies are queued
  int32_t* seg_e = nullptr;             // [E] global expert of hosted segment i (device)
  unsigned ce_epoch = 0;
  std::vector<int32_t> ce_recv_base, ce_send_base;  // layout of the last dispatch (host)
  bool out_stay = false;                // MOE_OUT_STAY: outputs stay for moe_dispatch_from
  bool ffn_done = false;                // moe_expert_ffn ran after the last dispatch
  unsigned long long flag_timeout_ns = kFlagTimeoutNs;  // MOE_FLAG_TIMEOUT_MS overrides
  // single-process group (moe_ctx_create_group): every rank's context lives in this
  // process; the peer tables hold the other contexts' device pointers directly (no
  // IPC, no NCCL).  shared_dev: another rank of the group runs on the same device --
  // the persistent grids are capped so every rank's kernels co-reside, and no kernel
  // with more than one CTA spins on a peer flag.
  bool local_group = false;
  bool shared_dev = false;
  int share = 1;                        // ranks of this process's group on this device
  std::shared_ptr<std::vector<int>> group_devices;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // the same pair for layers captured into a CUDA graph (an event recorded inside a
  // capture must not be waited on by eager work afterwards); cur_join = the join
  // event of the last dispatch
  cudaEvent_t ev_fork_cap = nullptr, ev_join_cap = nullptr, cur_join = nullptr;

  // last dispatch
  bool have_plan = false;
  int last_T = 0, last_k = 0, last_tiles = 0;
  std::vector<int32_t> cnt_host;  // [G][E] (NCCL mode)
};

static thread_local std::string g_err;

static moe_status fail(moe_ctx_t c, moe_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  g_err = buf;
  return s;
}

#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) return fail(ctx, MOE_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
  } while (0)
#define NC(call)                                                                          \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess) return fail(ctx, MOE_ERR_NCCL, "%s: %s", #call, ncclGetErrorString(r_)); \
  } while (0)
#define LAUNCHED(ctx, n)                                                                  \
  do {                                                                                    \
    cudaError_t e_ = cudaGetLastError();                                                  \
    if (e_ != cudaSuccess) return fail(ctx, MOE_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e_)); \
    (ctx)->launches += (n);                                                               \
  } while (0)

static constexpr int kTimeline = 8;
static void tl_rec(moe_ctx_t c, int j, cudaStream_t s) {
  if (c->tl_cur < 0) return;
  if (cudaEventRecord(c->tl[(size_t)c->tl_cur * kTimeline + j], s) == cudaSuccess) c->tl_mask[c->tl_cur] |= 1u << j;
}

static PlanBuffers plan_buffers(moe_ctx_t c) {
  PlanBuffers b;
  b.P_in = nullptr;  // set by moe_dispatch
  b.P = c->P_dev;
  b.tile_hist = c->tile_hist;
  b.tile_base = c->tile_base;
  b.cnt_local = c->cnt_local;
  // count matrix [G][E]: the local rows (virtual / G=1), the NCCL all-gather
  // result, or (P2P) the rows peers wrote into this rank's signal block
  b.cnt_all = c->virt || c->G == 1 ? c->cnt_local : (c->p2p ? reinterpret_cast<int32_t*>(c->sig) : c->cnt_all);
  b.base_row = c->base_row;
  b.seg_meta = c->seg_meta;
  b.row_of_item = c->row_of_item;
  b.slot_of_item = c->slot_of_item;
  b.dst_table = c->dst_table;
  b.src_table = c->src_table;
  b.peer_sig = c->peer_sig;
  b.my_sig = c->sig;
  b.done_counter = c->done_counter;
  b.err = c->err_dev;
  b.seg_src = c->seg_src;
  b.cslot_base = c->cslot_base;
  b.cslot_of_item = c->cslot_of_item;
  b.sendbuf = reinterpret_cast<uint4*>(c->sendbuf);
  b.seg_e = c->seg_e;
  b.ret_local = reinterpret_cast<const uint4*>(c->retbuf);
  b.part_stride = c->virt ? c->cap_rows * c->H / 8 : c->send_rows * c->H / 8;
  b.recv_local = reinterpret_cast<uint4*>(c->recv);
  b.tok_local = reinterpret_cast<const uint4*>(c->tokbuf);
  b.xmap_local = c->xmap;
  b.xmap_table = c->xmap_table;
  b.tok_table = reinterpret_cast<uint4* const*>(c->tok_table);
  b.exp_counter = c->exp_counter;
  b.tok_rows = c->cfg.max_tokens;
  b.seg_meta_c = c->seg_meta;
  b.desc_table = c->desc_table;
  b.desc_local = c->desc;
  b.desc_k = c->cfg.max_k;
  return b;
}

static PlanArgs plan_args(moe_ctx_t c, int T, int k) {
  PlanArgs a;
  a.T = T;
  a.k = k;
  a.E = c->E;
  a.H = c->H;
  a.V = c->V;
  a.G = c->G;
  a.me = c->me;
  a.tp = c->tp;
  a.grp = c->grp;
  a.virt = c->virt;
  a.p2p = c->p2p;
  a.epoch_ptr = c->epoch_dev;
  a.n_tiles = plan_tiles(T, c->V);
  a.seg_align = c->seg_align;
  a.fused = c->p2p && c->ffn_fused;
  a.gather = 0;
  a.direct = 0;
  a.ce = c->p2p && c->last_ce && !c->ffn_fused;  // K8: the copy engines returned the peers' rows
  a.plan_done = 0;
  a.timeout_ns = c->flag_timeout_ns;
  // enough CTAs for the HBM/NVLink-bound row copies, but no partial second wave:
  // K3/K8 CTAs (512 threads) fit twice per SM, so aim at <= 2 x num_sms CTAs
  const int chunks = c->H / 8;
  int split = a.n_tiles > 0 ? (2 * c->num_sms) / a.n_tiles : 1;
  // (at most 32 slices of >= 16 16-byte chunks each: decode-sized batches have one
  // or two token tiles, and every slice is another CTA pulling/pushing rows)
  static const int cap = getenv("MOE_COL_SPLIT_MAX") ? std::max(1, atoi(getenv("MOE_COL_SPLIT_MAX"))) : 32;
  split = std::max(1, std::min(split, std::min(cap, chunks / 16 > 0 ? chunks / 16 : 1)));
  a.col_split = split;
  return a;
}

extern "C" {

int32_t moe_abi_version(void) { return MOE_ABI_VERSION; }

const char* moe_status_str(moe_status s) {
  switch (s) {
    case MOE_OK: return "MOE_OK";
    case MOE_ERR_INVALID_ARG: return "MOE_ERR_INVALID_ARG";
    case MOE_ERR_CUDA: return "MOE_ERR_CUDA";
    case MOE_ERR_NCCL: return "MOE_ERR_NCCL";
    case MOE_ERR_CAPACITY: return "MOE_ERR_CAPACITY";
    case MOE_ERR_UNSUPPORTED: return "MOE_ERR_UNSUPPORTED";
    case MOE_ERR_DEVICE: return "MOE_ERR_DEVICE";
    case MOE_ERR_TIMEOUT: return "MOE_ERR_TIMEOUT";
  }
  return "MOE_ERR_UNKNOWN";
}

const char* moe_last_error(moe_ctx_t ctx) { return ctx ? ctx->err.c_str() : g_err.c_str(); }

int64_t moe_kernel_launches(moe_ctx_t ctx) { return ctx ? ctx->launches : 0; }

moe_status moe_get_unique_id(uint8_t out[128]) {
  moe_ctx_t ctx = nullptr;
  if (!out) return fail(ctx, MOE_ERR_INVALID_ARG, "out is NULL");
  ncclUniqueId id;
  NC(ncclGetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "nccl unique id size");
  memcpy(out, &id, 128);
  return MOE_OK;
}

moe_status moe_placement_contiguous(int32_t E, int32_t G, int32_t* out) {
  moe_ctx_t ctx = nullptr;
  if (!out || E <= 0 || G <= 0) return fail(ctx, MOE_ERR_INVALID_ARG, "bad arguments");
  if (E % G != 0) return fail(ctx, MOE_ERR_INVALID_ARG, "E %% G != 0 (E=%d, G=%d)", E, G);
  const int per = E / G;
  for (int e = 0; e < E; ++e) out[e] = e / per;
  return MOE_OK;
}

static moe_status layout_host_impl(int32_t E, int32_t G, const int32_t* P, const int32_t* cnt, int align,
                                   int32_t* seg_start, int32_t* recv_base, int32_t* recv_rows, int32_t* send_base);

moe_status moe_layout_host(int32_t E, int32_t G, const int32_t* P, const int32_t* cnt, int32_t* seg_start,
                           int32_t* recv_base, int32_t* recv_rows, int32_t* send_base) {
  return layout_host_impl(E, G, P, cnt, kSegAlign, seg_start, recv_base, recv_rows, send_base);
}

static moe_status layout_host_impl(int32_t E, int32_t G, const int32_t* P, const int32_t* cnt, int align,
                                   int32_t* seg_start, int32_t* recv_base, int32_t* recv_rows, int32_t* send_base) {
  moe_ctx_t ctx = nullptr;
  if (E <= 0 || G <= 0 || !P || !cnt) return fail(ctx, MOE_ERR_INVALID_ARG, "bad arguments");
  for (int e = 0; e < E; ++e)
    if (P[e] < 0 || P[e] >= G) return fail(ctx, MOE_ERR_INVALID_ARG, "placement value out of range");
  std::vector<int64_t> start(E, 0);
  for (int g = 0; g < G; ++g) {
    int64_t acc = 0, unp = 0;
    for (int e = 0; e < E; ++e) {
      if (P[e] != g) continue;
      int64_t rows = 0;
      for (int s = 0; s < G; ++s) rows += cnt[s * E + e];
      start[e] = acc;
      acc += (rows + align - 1) / align * align;
      unp += rows;
    }
    if (recv_rows) recv_rows[g] = (int32_t)unp;
  }
  for (int e = 0; e < E; ++e) {
    if (seg_start) seg_start[e] = (int32_t)start[e];
    int64_t acc = start[e];
    for (int s = 0; s < G; ++s) {
      if (recv_base) recv_base[s * E + e] = (int32_t)acc;
      acc += cnt[s * E + e];
    }
  }
  if (send_base) {
    // full send order of source s: key (P[e], e)
    for (int s = 0; s < G; ++s) {
      int64_t acc = 0;
      for (int g = 0; g < G; ++g)
        for (int e = 0; e < E; ++e)
          if (P[e] == g) {
            send_base[s * E + e] = (int32_t)acc;
            acc += cnt[s * E + e];
          }
    }
  }
  return MOE_OK;
}

// Every API call that selects the context's device restores the caller's current
// device on return (a single-process group drives several devices from one thread).
struct DeviceGuard {
  int prev = -1;
  DeviceGuard() {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

// Configuration checks shared by moe_ctx_create and moe_ctx_create_group.
static moe_status check_cfg(const moe_config& c) {
  moe_ctx_t ctx = nullptr;
  if (c.hidden <= 0 || c.hidden % 64) return fail(ctx, MOE_ERR_UNSUPPORTED, "hidden must be a positive multiple of 64");
  if (c.ffn <= 0 || c.ffn % 64) return fail(ctx, MOE_ERR_UNSUPPORTED, "ffn must be a positive multiple of 64");
  if (c.num_experts < 1 || c.num_experts > kMaxExperts)
    return fail(ctx, MOE_ERR_INVALID_ARG, "num_experts must be in [1, %d]", kMaxExperts);
  if (c.max_k < 1 || c.max_k > c.num_experts || c.max_k > kMaxK)
    return fail(ctx, MOE_ERR_INVALID_ARG, "max_k must be in [1, min(E, %d)]", kMaxK);
  if (c.max_tokens < 0) return fail(ctx, MOE_ERR_INVALID_ARG, "max_tokens < 0");
  if (c.world < 1 || c.world > kMaxWorld || c.rank < 0 || c.rank >= c.world)
    return fail(ctx, MOE_ERR_INVALID_ARG, "bad world/rank");
  if (c.virtual_ranks > 1 && c.world != 1) return fail(ctx, MOE_ERR_INVALID_ARG, "virtual_ranks needs world == 1");
  if (c.virtual_ranks > kMaxWorld) return fail(ctx, MOE_ERR_INVALID_ARG, "virtual_ranks > %d", kMaxWorld);
  if (c.a2a_mode != MOE_A2A_NCCL && c.a2a_mode != MOE_A2A_P2P)
    return fail(ctx, MOE_ERR_INVALID_ARG, "unknown a2a_mode %d", c.a2a_mode);
  const int tp = c.tp <= 1 ? 1 : c.tp;
  const int ranks = c.virtual_ranks > 1 ? c.virtual_ranks : c.world;
  if (tp > kMaxTP) return fail(ctx, MOE_ERR_INVALID_ARG, "tp=%d > %d", tp, kMaxTP);
  if (ranks % tp) return fail(ctx, MOE_ERR_INVALID_ARG, "tp=%d does not divide the %d ranks", tp, ranks);
  if (c.ffn % (64 * tp)) return fail(ctx, MOE_ERR_UNSUPPORTED, "ffn / tp must be a multiple of 64");
  if (tp > 1 && c.virtual_ranks <= 1 && c.a2a_mode != MOE_A2A_P2P)
    return fail(ctx, MOE_ERR_UNSUPPORTED, "tp > 1 on real ranks needs MOE_A2A_P2P");
  return MOE_OK;
}

// Allocate one rank's context: every workspace, the activation tensor maps.  No
// communicator, no peer tables (moe_ctx_create / moe_ctx_create_group add those).
// share = ranks of a single-process group on this device (1 otherwise).
static moe_status ctx_alloc(const moe_config& c, int share, moe_ctx_t* out) {
  moe_ctx_t ctx = new moe_ctx();
  *out = ctx;
  ctx->cfg = c;
  ctx->E = c.num_experts;
  ctx->H = c.hidden;
  ctx->F = c.ffn;
  ctx->virt = c.virtual_ranks > 1;
  ctx->G = ctx->virt ? c.virtual_ranks : c.world;
  ctx->V = ctx->virt ? c.virtual_ranks : 1;
  ctx->me = ctx->virt ? 0 : c.rank;
  const int tp = c.tp <= 1 ? 1 : c.tp;
  ctx->tp = tp;
  ctx->grp = ctx->me / tp;
  ctx->tpi = ctx->me % tp;
  ctx->Fl = ctx->virt ? c.ffn : c.ffn / tp;
  if (cudaSetDevice(c.device) != cudaSuccess) return fail(ctx, MOE_ERR_CUDA, "cudaSetDevice(%d) failed", c.device);
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, c.device);
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, c.device);
  if (major != 10)
    return fail(ctx, MOE_ERR_UNSUPPORTED, "libmoe needs an sm_100 (B200) device, got compute capability %d.x", major);
  static unsigned long long preloaded = 0;  // per device
  if (first_time_on_device(preloaded)) {
    preload_route_kernels();
    preload_dispatch_kernels();
    preload_gemm_kernels();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ctx, MOE_ERR_CUDA, "loading the kernels: %s", cudaGetErrorString(e));
  }
  if (const char* ft = getenv("MOE_FLAG_TIMEOUT_MS"))
    ctx->flag_timeout_ns = std::max(1ull, (unsigned long long)atoll(ft)) * 1000000ull;
  if (share > 1) {
    // ranks sharing one device: each gets an equal slice of the SMs for its persistent
    // grids, 16 SMs stay free for the peers' row copies, so a GEMM CTA waiting for a
    // peer's rows never blocks the kernel that delivers them
    ctx->shared_dev = true;
    ctx->share = share;
    ctx->num_sms = std::max(2, ((ctx->num_sms - 16) / share) & ~1);
    ctx->remote_ctas = std::max(1, std::min(ctx->remote_ctas, ctx->num_sms / 2));
  }
  const int E = ctx->E, G = ctx->G, k = c.max_k;
  const int64_t Tm = c.max_tokens;
  // receive layout capacity (dropless, reading G6)
  int64_t rows;
  if (ctx->virt || G == 1) rows = Tm * k;
  else rows = (int64_t)G * Tm * k;  // every source may send all its items here
  if (rows <= (int64_t)256 * E) {   // decode-sized worst case: 128-row tiles on one CTA
    ctx->seg_align = 128;
    ctx->gemm_cg = 1;
  }
  if (getenv("MOE_GEMM_CG")) {      // tuning / testing override: 1 or 2
    ctx->gemm_cg = atoi(getenv("MOE_GEMM_CG")) == 1 ? 1 : 2;
    ctx->seg_align = 128 * ctx->gemm_cg;
  }
  ctx->cap_rows = rows + (int64_t)E * ctx->seg_align;
  ctx->send_rows = (!ctx->virt && G > 1) ? Tm * k : 0;
  ctx->max_tiles = plan_tiles((int)Tm, ctx->V) + ctx->V;

  auto A = [&](void** p, size_t bytes) -> bool {
    if (bytes == 0) bytes = 16;
    if (cudaMalloc(p, bytes) != cudaSuccess) {
      fail(ctx, MOE_ERR_CUDA, "cudaMalloc(%zu) failed", bytes);
      return false;
    }
    return true;
  };
  bool ok = A((void**)&ctx->P_dev, sizeof(int32_t) * E) &&
            A((void**)&ctx->P_all, sizeof(int32_t) * (size_t)G * E) &&
            A((void**)&ctx->tile_hist, sizeof(int32_t) * (size_t)ctx->max_tiles * E) &&
            A((void**)&ctx->tile_base, sizeof(int32_t) * (size_t)ctx->max_tiles * E) &&
            A((void**)&ctx->cnt_local, sizeof(int32_t) * (size_t)ctx->V * E) &&
            A((void**)&ctx->cnt_all, sizeof(int32_t) * (size_t)G * E) &&
            A((void**)&ctx->base_row, sizeof(int32_t) * (size_t)ctx->V * E) &&
            A((void**)&ctx->seg_meta, sizeof(int32_t) * (size_t)(1 + 3 * E + 4)) &&
            A((void**)&ctx->row_of_item, sizeof(int32_t) * (size_t)std::max<int64_t>(Tm * k, 1)) &&
            A((void**)&ctx->err_dev, sizeof(int)) &&
            A((void**)&ctx->recv, (size_t)ctx->cap_rows * c.hidden * 2) &&
            A((void**)&ctx->hbuf, (size_t)ctx->cap_rows * ctx->Fl * 2) &&
            A((void**)&ctx->ybuf, (size_t)ctx->cap_rows * c.hidden * 2 * (ctx->virt ? tp : 1)) &&
            A((void**)&ctx->sendbuf, (size_t)ctx->send_rows * c.hidden * 2) &&
            A((void**)&ctx->retbuf, (size_t)ctx->send_rows * c.hidden * 2 * tp) &&
            A((void**)&ctx->slot_of_item, (size_t)std::max<int64_t>(Tm * k, 1)) &&
            A((void**)&ctx->dst_table, sizeof(void*) * (size_t)std::max(G, 2)) &&
            A((void**)&ctx->src_table, sizeof(void*) * (size_t)std::max(G, 2)) &&
            A((void**)&ctx->peer_sig, sizeof(void*) * (size_t)G) &&
            A((void**)&ctx->sig, sizeof(SigBlock)) && A((void**)&ctx->done_counter, 4 * sizeof(unsigned)) &&
            A((void**)&ctx->seg_src, sizeof(int32_t) * 3 * (size_t)E * G) &&
            A((void**)&ctx->cslot_base, sizeof(int32_t) * (size_t)ctx->V * E) &&
            A((void**)&ctx->cslot_of_item, sizeof(int32_t) * (size_t)std::max<int64_t>(Tm * k, 1)) &&
            A((void**)&ctx->seg_e, sizeof(int32_t) * (size_t)E) &&
            A((void**)&ctx->ret_table, sizeof(void*) * (size_t)G) &&
            A((void**)&ctx->epoch_dev, sizeof(unsigned)) &&
            A((void**)&ctx->desc, sizeof(int32_t) * 3 * (size_t)k * ctx->cap_rows) &&
            A((void**)&ctx->desc_table, sizeof(void*) * (size_t)std::max(G, 1));
  if (!ok) return MOE_ERR_CUDA;
  cudaMemset(ctx->sig, 0, sizeof(SigBlock));
  cudaMemset(ctx->done_counter, 0, 4 * sizeof(unsigned));  // [0] scatter last-CTA, [2..3] GEMM scheduler
  cudaMemset(ctx->err_dev, 0, sizeof(int));
  cudaMemset(ctx->epoch_dev, 0, sizeof(unsigned));
  cudaMemset(ctx->seg_meta, 0, sizeof(int32_t) * (1 + 3 * E + 4));
  if (cudaMallocHost((void**)&ctx->P_all_pinned, sizeof(int32_t) * (size_t)G * E) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->cnt_pinned, sizeof(int32_t) * (size_t)G * E) != cudaSuccess ||
      cudaMallocHost((void**)&ctx->ce_pinned, sizeof(int32_t) * ((size_t)G * E + E + 2)) != cudaSuccess ||
      cudaMalloc((void**)&ctx->segdone, sizeof(unsigned) * (size_t)E) != cudaSuccess)
    return fail(ctx, MOE_ERR_CUDA, "cudaMallocHost failed");
  ctx->P_host.assign(E, 0);
  ctx->cnt_host.assign((size_t)G * E, 0);
  // A-operand tensor maps over the context-owned activation buffers
  if (!make_tmap_2d(ctx->tmA1, ctx->recv, ctx->cap_rows, c.hidden, 128) ||
      !make_tmap_2d(ctx->tmA2, ctx->hbuf, ctx->cap_rows, ctx->Fl, 128))
    return fail(ctx, MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed for the activation buffers");
  if (!make_tmap_store_2d(ctx->tmDh, ctx->hbuf, ctx->cap_rows, ctx->Fl, ctx->Fl) ||
      !make_tmap_store_2d(ctx->tmDy, ctx->ybuf, ctx->cap_rows, c.hidden, c.hidden))
    return fail(ctx, MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed for the epilogue store maps");
  if (ctx->virt && tp > 1)
    for (int q = 0; q < tp; ++q) {
      if (!make_tmap_store_2d(ctx->tmDys[q], ctx->ybuf + (size_t)q * ctx->cap_rows * c.hidden, ctx->cap_rows,
                              c.hidden, c.hidden))
        return fail(ctx, MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed for a partial-output store map");
      if (!make_tmap_2d_ld(ctx->tmA2s[q], ctx->hbuf + (size_t)q * (c.ffn / tp), ctx->cap_rows, c.ffn / tp, c.ffn,
                           128))
        return fail(ctx, MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed for an h slice");
    }
  return MOE_OK;
}

// P2P mode: the side stream of the peers' row copies and its fork / join events,
// and the gather dispatch's token buffer and row map.
static moe_status p2p_streams(moe_ctx_t ctx) {
  ctx->p2p = true;
  if (const char* rc = getenv("MOE_SCATTER_CTAS")) ctx->remote_ctas = atoi(rc);
  CU(cudaSetDevice(ctx->cfg.device));
  const size_t tok_bytes = (size_t)ctx->G * std::max(ctx->cfg.max_tokens, 1) * ctx->H * 2;
  CU(cudaMalloc((void**)&ctx->tokbuf, tok_bytes));
  CU(cudaMalloc((void**)&ctx->xmap, sizeof(int32_t) * (size_t)ctx->cap_rows));
  CU(cudaMalloc((void**)&ctx->xmap_table, sizeof(void*) * (size_t)ctx->G));
  CU(cudaMalloc((void**)&ctx->tok_table, sizeof(void*) * (size_t)ctx->G));
  CU(cudaMalloc((void**)&ctx->exp_counter, sizeof(unsigned) * (size_t)ctx->G));
  CU(cudaMemset(ctx->exp_counter, 0, sizeof(unsigned) * (size_t)ctx->G));
  ctx->tok_peer.assign(ctx->G, nullptr);
  CU(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  CU(cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&ctx->ev_join, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&ctx->ev_fork_cap, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&ctx->ev_join_cap, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&ctx->ev_cnt, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&ctx->ev_staged, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&ctx->ev_k6, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&ctx->ev_side2, cudaEventDisableTiming));
  CU(cudaStreamCreateWithFlags(&ctx->side2, cudaStreamNonBlocking));
  return MOE_OK;
}

// Upload the slot -> buffer tables.  NCCL / virtual: slot 0 = this process's receive /
// expert-output buffers, slot 1 = the compact send / return buffers.  P2P: slot g =
// rank g's receive / expert-output buffer, signal block and return buffer (region tpi).
static moe_status upload_tables(moe_ctx_t ctx, std::vector<void*>& dst, std::vector<void*>& src,
                                std::vector<void*>& sig, std::vector<void*>& ret) {
  CU(cudaSetDevice(ctx->cfg.device));
  CU(cudaMemcpy(ctx->dst_table, dst.data(), sizeof(void*) * dst.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->src_table, src.data(), sizeof(void*) * src.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->peer_sig, sig.data(), sizeof(void*) * ctx->G, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->ret_table, ret.data(), sizeof(void*) * ctx->G, cudaMemcpyHostToDevice));
  CU(cudaDeviceSynchronize());
  ctx->recv_h.assign(dst.begin(), dst.begin() + std::min<size_t>(dst.size(), ctx->G));
  ctx->sig_h.assign(sig.begin(), sig.begin() + ctx->G);
  ctx->ret_h.assign(ret.begin(), ret.begin() + ctx->G);
  return MOE_OK;
}

moe_status moe_ctx_create(const moe_config* cfg, const uint8_t* uid, moe_ctx_t* out) {
  DeviceGuard device_guard;
  moe_ctx_t ctx = nullptr;
  if (!cfg || !out) return fail(ctx, MOE_ERR_INVALID_ARG, "cfg/out is NULL");
  const moe_config& c = *cfg;
  moe_status st = check_cfg(c);
  if (st != MOE_OK) return st;
  if (c.world > 1 && !uid) return fail(ctx, MOE_ERR_INVALID_ARG, "uid required when world > 1");
  auto bail = [&](moe_status s) {
    std::string m = ctx ? ctx->err : g_err;
    moe_ctx_destroy(ctx);
    fail(nullptr, s, "%s", m.c_str());
    return s;
  };
  st = ctx_alloc(c, 1, &ctx);
  if (st != MOE_OK) return bail(st);
  const int G = ctx->G;
  if (!ctx->virt && G > 1) {
    ncclUniqueId id;
    memcpy(&id, uid, 128);
    ncclResult_t r = ncclCommInitRank(&ctx->comm, G, id, c.rank);
    if (r != ncclSuccess) {
      fail(ctx, MOE_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
      return bail(MOE_ERR_NCCL);
    }
  }
  std::vector<void*> dst(std::max(G, 2)), src(std::max(G, 2)), sig(G, nullptr), ret(G, nullptr), xm;
  std::vector<void*> dsc(1, ctx->desc);   // NCCL / virtual / one rank: slot 0 = own
  ret[0] = ctx->retbuf;
  dst[0] = ctx->recv;
  dst[1] = ctx->sendbuf;
  src[0] = ctx->ybuf;
  src[1] = ctx->retbuf;
  sig[0] = ctx->sig;
  if (!ctx->virt && G > 1 && c.a2a_mode == MOE_A2A_P2P) {
    // the peers' buffers are mapped through CUDA IPC (NVLink peer memory); the
    // handles are exchanged once here over NCCL
    st = p2p_streams(ctx);
    if (st != MOE_OK) return bail(st);
    cudaIpcMemHandle_t h[7];
    if (cudaIpcGetMemHandle(&h[0], ctx->recv) != cudaSuccess || cudaIpcGetMemHandle(&h[1], ctx->ybuf) != cudaSuccess ||
        cudaIpcGetMemHandle(&h[2], ctx->sig) != cudaSuccess || cudaIpcGetMemHandle(&h[3], ctx->retbuf) != cudaSuccess ||
        cudaIpcGetMemHandle(&h[4], ctx->tokbuf) != cudaSuccess || cudaIpcGetMemHandle(&h[5], ctx->xmap) != cudaSuccess ||
        cudaIpcGetMemHandle(&h[6], ctx->desc) != cudaSuccess) {
      fail(ctx, MOE_ERR_CUDA, "cudaIpcGetMemHandle failed");
      return bail(MOE_ERR_CUDA);
    }
    const size_t hb = sizeof(h);
    uint8_t* dh = nullptr;
    std::vector<uint8_t> all(hb * G);
    if (cudaMalloc(&dh, hb * (G + 1)) != cudaSuccess ||
        cudaMemcpy(dh + hb * G, h, hb, cudaMemcpyHostToDevice) != cudaSuccess ||
        ncclAllGather(dh + hb * G, dh, hb, ncclUint8, ctx->comm, 0) != ncclSuccess ||
        cudaStreamSynchronize(0) != cudaSuccess || cudaMemcpy(all.data(), dh, hb * G, cudaMemcpyDeviceToHost) != cudaSuccess) {
      if (dh) cudaFree(dh);
      fail(ctx, MOE_ERR_NCCL, "IPC handle exchange failed");
      return bail(MOE_ERR_NCCL);
    }
    cudaFree(dh);
    xm.assign(G, nullptr);
    dsc.assign(G, nullptr);
    for (int g = 0; g < G; ++g) {
      if (g == c.rank) {
        dst[g] = ctx->recv;
        src[g] = ctx->ybuf;
        sig[g] = ctx->sig;
        ret[g] = ctx->retbuf + (size_t)ctx->tpi * ctx->send_rows * c.hidden;
        ctx->tok_peer[g] = ctx->tokbuf;
        xm[g] = ctx->xmap;
        dsc[g] = ctx->desc;
        continue;
      }
      const cudaIpcMemHandle_t* hg = reinterpret_cast<const cudaIpcMemHandle_t*>(all.data() + hb * g);
      void* p[7] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
      for (int i = 0; i < 7; ++i) {
        cudaError_t e = cudaIpcOpenMemHandle(&p[i], hg[i], cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          fail(ctx, MOE_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", g, cudaGetErrorString(e));
          return bail(MOE_ERR_CUDA);
        }
        ctx->ipc_opened.push_back(p[i]);
      }
      dst[g] = p[0];
      src[g] = p[1];
      sig[g] = p[2];
      // fused combine of TP slice tpi lands in partial region tpi of the source's buffer
      ret[g] = static_cast<uint16_t*>(p[3]) + (size_t)ctx->tpi * ctx->send_rows * c.hidden;
      ctx->tok_peer[g] = p[4];
      xm[g] = p[5];
      dsc[g] = p[6];
    }
  }
  if (cudaMemcpy(ctx->desc_table, dsc.data(), sizeof(void*) * dsc.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    fail(ctx, MOE_ERR_CUDA, "descriptor table upload failed");
    return bail(MOE_ERR_CUDA);
  }
  if (ctx->p2p && (cudaMemcpy(ctx->xmap_table, xm.data(), sizeof(void*) * G, cudaMemcpyHostToDevice) != cudaSuccess ||
                   cudaMemcpy(ctx->tok_table, ctx->tok_peer.data(), sizeof(void*) * G, cudaMemcpyHostToDevice) !=
                       cudaSuccess)) {
    fail(ctx, MOE_ERR_CUDA, "xmap table upload failed");
    return bail(MOE_ERR_CUDA);
  }
  st = upload_tables(ctx, dst, src, sig, ret);
  if (st != MOE_OK) return bail(st);
  *out = ctx;
  return MOE_OK;
}

moe_status moe_ctx_create_group(const moe_config* cfg, int32_t n, const int32_t* devices, moe_ctx_t* out) {
  DeviceGuard device_guard;
  moe_ctx_t ctx = nullptr;
  if (!cfg || !out) return fail(ctx, MOE_ERR_INVALID_ARG, "cfg/out is NULL");
  if (n < 2 || n > kMaxWorld) return fail(ctx, MOE_ERR_INVALID_ARG, "n=%d outside [2, %d]", n, kMaxWorld);
  if (cfg->a2a_mode != MOE_A2A_P2P) return fail(ctx, MOE_ERR_UNSUPPORTED, "a single-process group needs MOE_A2A_P2P");
  if (cfg->virtual_ranks > 1) return fail(ctx, MOE_ERR_INVALID_ARG, "a single-process group has no virtual ranks");
  std::vector<moe_config> cf(n, *cfg);
  for (int r = 0; r < n; ++r) {
    cf[r].world = n;
    cf[r].rank = r;
    if (devices) cf[r].device = devices[r];
    moe_status st = check_cfg(cf[r]);
    if (st != MOE_OK) return st;
  }
  std::vector<moe_ctx_t> cs(n, nullptr);
  auto bail = [&](moe_status s, moe_ctx_t culprit) {
    std::string m = culprit ? culprit->err : g_err;
    for (auto& c : cs) {
      if (c) c->local_group = false;  // plain teardown (no peer devices to drain)
      moe_ctx_destroy(c);
    }
    fail(nullptr, s, "%s", m.c_str());
    return s;
  };
  auto devs = std::make_shared<std::vector<int>>();
  for (int r = 0; r < n; ++r)
    if (std::find(devs->begin(), devs->end(), cf[r].device) == devs->end()) devs->push_back(cf[r].device);
  // Ranks sharing a device spin on each other's flags from different streams.  Each
  // rank drives two streams (its caller's and its side stream); when the device has
  // fewer hardware work queues than that, streams alias onto one queue and a spinning
  // kernel can sit in front of the peer kernel it waits for (a flag timeout).
  int conns = 8;   // CUDA's default
  if (const char* cm = getenv("CUDA_DEVICE_MAX_CONNECTIONS")) conns = atoi(cm);
  for (int d : *devs) {
    int share = 0;
    for (int r = 0; r < n; ++r) share += cf[r].device == d;
    if (share > 1 && 2 * share > conns)
      return fail(nullptr, MOE_ERR_UNSUPPORTED,
                  "%d ranks share device %d: needs CUDA_DEVICE_MAX_CONNECTIONS >= %d (set before CUDA "
                  "initialises; it is %d)", share, d, 2 * share, conns);
  }
  for (int r = 0; r < n; ++r) {
    int share = 0;
    for (int q = 0; q < n; ++q) share += cf[q].device == cf[r].device;
    moe_status st = ctx_alloc(cf[r], share, &cs[r]);
    if (st != MOE_OK) return bail(st, cs[r]);
    cs[r]->local_group = true;
    cs[r]->group_devices = devs;
    st = p2p_streams(cs[r]);
    if (st != MOE_OK) return bail(st, cs[r]);
  }
  // ranks on different devices of this process reach each other's memory as peers
  for (int a : *devs)
    for (int b : *devs) {
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (!can) {
        fail(cs[0], MOE_ERR_UNSUPPORTED, "device %d cannot access device %d as a peer", a, b);
        return bail(MOE_ERR_UNSUPPORTED, cs[0]);
      }
      cudaSetDevice(a);
      cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
        fail(cs[0], MOE_ERR_CUDA, "cudaDeviceEnablePeerAccess(%d -> %d): %s", a, b, cudaGetErrorString(e));
        return bail(MOE_ERR_CUDA, cs[0]);
      }
      cudaGetLastError();
    }
  for (int r = 0; r < n; ++r) {
    moe_ctx_t c = cs[r];
    std::vector<void*> dst(n), src(n), sig(n), ret(n), xm(n), dsc(n);
    for (int g = 0; g < n; ++g) {
      dst[g] = cs[g]->recv;
      src[g] = cs[g]->ybuf;
      sig[g] = cs[g]->sig;
      ret[g] = cs[g]->retbuf + (size_t)c->tpi * cs[g]->send_rows * c->H;
      c->tok_peer[g] = cs[g]->tokbuf;
      xm[g] = cs[g]->xmap;
      dsc[g] = cs[g]->desc;
    }
    cudaSetDevice(c->cfg.device);
    if (cudaMemcpy(c->xmap_table, xm.data(), sizeof(void*) * n, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->tok_table, c->tok_peer.data(), sizeof(void*) * n, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(c->desc_table, dsc.data(), sizeof(void*) * n, cudaMemcpyHostToDevice) != cudaSuccess) {
      fail(c, MOE_ERR_CUDA, "xmap table upload failed");
      return bail(MOE_ERR_CUDA, c);
    }
    moe_status st = upload_tables(c, dst, src, sig, ret);
    if (st != MOE_OK) return bail(st, c);
  }
  for (int r = 0; r < n; ++r) out[r] = cs[r];
  return MOE_OK;
}

moe_status moe_ctx_destroy(moe_ctx_t ctx) {
  DeviceGuard device_guard;
  if (!ctx) return MOE_OK;
  if (ctx->comm && ctx->cfg.world > 1) {
    // collective: no peer may still read this rank's mapped buffers (a slower peer's
    // combine pulling rows from ybuf) when they are freed -- barrier first
    cudaSetDevice(ctx->cfg.device);
    int* one = nullptr;
    if (cudaMalloc(&one, sizeof(int)) == cudaSuccess) {
      if (ncclAllReduce(one, one, 1, ncclInt32, ncclSum, ctx->comm, 0) == ncclSuccess) cudaStreamSynchronize(0);
      cudaFree(one);
    }
  }
  if (ctx->local_group && ctx->group_devices) {
    // single-process group: the peers' kernels run on this process's devices
    for (int d : *ctx->group_devices) {
      cudaSetDevice(d);
      cudaDeviceSynchronize();
    }
  }
  cudaSetDevice(ctx->cfg.device);
  cudaDeviceSynchronize();
  if (ctx->comm) {
    ncclCommFinalize(ctx->comm);
    ncclCommDestroy(ctx->comm);
  }
  for (void* p : ctx->ipc_opened) cudaIpcCloseMemHandle(p);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->ev_fork) cudaEventDestroy(ctx->ev_fork);
  if (ctx->ev_join) cudaEventDestroy(ctx->ev_join);
  if (ctx->ev_fork_cap) cudaEventDestroy(ctx->ev_fork_cap);
  if (ctx->ev_join_cap) cudaEventDestroy(ctx->ev_join_cap);
  void* dev[] = {ctx->P_dev, ctx->P_all, ctx->tile_hist, ctx->tile_base, ctx->cnt_local, ctx->cnt_all,
                 ctx->base_row, ctx->seg_meta, ctx->row_of_item, ctx->err_dev, ctx->recv, ctx->hbuf, ctx->ybuf,
                 ctx->sendbuf, ctx->retbuf, ctx->slot_of_item, ctx->dst_table, ctx->src_table, ctx->peer_sig,
                 ctx->sig, ctx->done_counter, ctx->seg_src, ctx->cslot_base, ctx->cslot_of_item, ctx->ret_table,
                 ctx->epoch_dev, ctx->splitk_ws, ctx->tokbuf, ctx->xmap, ctx->xmap_table, ctx->exp_counter,
                 ctx->desc, ctx->desc_table, ctx->tok_table, ctx->seg_e};
  for (void* p : dev)
    if (p) cudaFree(p);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : ctx->tl)
    if (e) cudaEventDestroy(e);
  if (ctx->P_all_pinned) cudaFreeHost(ctx->P_all_pinned);
  if (ctx->cnt_pinned) cudaFreeHost(ctx->cnt_pinned);
  if (ctx->ce_pinned) cudaFreeHost(ctx->ce_pinned);
  if (ctx->segdone) cudaFree(ctx->segdone);
  if (ctx->ev_cnt) cudaEventDestroy(ctx->ev_cnt);
  if (ctx->ev_staged) cudaEventDestroy(ctx->ev_staged);
  if (ctx->ev_k6) cudaEventDestroy(ctx->ev_k6);
  if (ctx->ev_side2) cudaEventDestroy(ctx->ev_side2);
  if (ctx->side2) cudaStreamDestroy(ctx->side2);
  delete ctx;
  return MOE_OK;
}

// Report a latched device error word e (and clear the word): the message names every
// set bit and every timed-out wait site.
static moe_status report_device_error(moe_ctx_t ctx, int e) {
  if (e) {
    cudaMemset(ctx->err_dev, 0, sizeof(int));
    std::string sites;
    static const char* kSite[] = {"count exchange (k_layout)", "peers' rows (K5)", "expert outputs (combine)",
                                  "flags (k_wait)", "gathered rows (k_expand)", "previous layer's outputs (direct)",
                                  "descriptors (direct)"};
    for (int i = 0; i < 7; ++i)
      if (e & (1 << (8 + i))) sites += std::string(sites.empty() ? " waiting for: " : ", ") + kSite[i];
    return fail(ctx, (e & kErrTimeout) ? MOE_ERR_TIMEOUT : MOE_ERR_DEVICE, "device error latched:%s%s%s%s%s%s%s%s",
                (e & kErrBadExpert) ? " expert id out of range" : "",
                (e & kErrCapacity) ? " receive capacity exceeded" : "",
                (e & kErrTimeout) ? " P2P peer flag timeout (a rank skipped a collective call?)" : "",
                (e & kErrPlacement) ? " ranks dispatched with different expert_to_rank maps" : "",
                (e & kErrNaN) ? " NaN router logit" : "",
                (e & kErrBadRank) ? " expert_to_rank value outside [0, G/tp)" : "",
                (e & kErrWeights) ? " moe_expert_ffn n_w differs from the experts the placement hosts here" : "",
                sites.c_str());
  }
  return MOE_OK;
}

static moe_status check_device_error(moe_ctx_t ctx) {
  int e = 0;
  CU(cudaMemcpy(&e, ctx->err_dev, sizeof(int), cudaMemcpyDeviceToHost));
  return report_device_error(ctx, e);
}

moe_status moe_ctx_sync(moe_ctx_t ctx) {
  DeviceGuard device_guard;
  if (!ctx) return fail(ctx, MOE_ERR_INVALID_ARG, "ctx is NULL");
  CU(cudaSetDevice(ctx->cfg.device));
  CU(cudaStreamSynchronize(ctx->last_stream));
  return check_device_error(ctx);
}

moe_status moe_route(moe_ctx_t ctx, const float* logits, int32_t T, int32_t E, int32_t k, int32_t* idx, float* w,
                     moe_stream_t stream) {
  if (!ctx) return fail(ctx, MOE_ERR_INVALID_ARG, "ctx is NULL");
  if (T < 0 || T > ctx->cfg.max_tokens) return fail(ctx, MOE_ERR_CAPACITY, "T=%d outside [0, max_tokens]", T);
  DeviceGuard device_guard;
  CU(cudaSetDevice(ctx->cfg.device));
  if (E != ctx->E) return fail(ctx, MOE_ERR_INVALID_ARG, "E=%d != context E=%d", E, ctx->E);
  if (k < 1 || k > E || k > ctx->cfg.max_k) return fail(ctx, MOE_ERR_INVALID_ARG, "k=%d outside [1, min(E, max_k)]", k);
  if (T > 0 && (!logits || !idx || !w)) return fail(ctx, MOE_ERR_INVALID_ARG, "NULL tensor");
  cudaStream_t s = (cudaStream_t)stream;
  ctx->last_stream = s;
  if (T == 0) return MOE_OK;
  launch_route(logits, T, E, k, idx, w, ctx->err_dev, s);
  LAUNCHED(ctx, 1);
  return MOE_OK;
}

moe_status moe_route_stats(moe_ctx_t ctx, const int32_t* idx_l, const int32_t* idx_l1, int32_t T, int32_t E,
                           int32_t k, int64_t* load, int64_t* coact, moe_stream_t stream) {
  if (!ctx) return fail(ctx, MOE_ERR_INVALID_ARG, "ctx is NULL");
  DeviceGuard device_guard;
  CU(cudaSetDevice(ctx->cfg.device));
  if (T < 0 || T > ctx->cfg.max_tokens) return fail(ctx, MOE_ERR_CAPACITY, "T=%d outside [0, max_tokens]", T);
  if (E != ctx->E) return fail(ctx, MOE_ERR_INVALID_ARG, "E=%d != context E=%d", E, ctx->E);
  if (k < 1 || k > E || k > ctx->cfg.max_k) return fail(ctx, MOE_ERR_INVALID_ARG, "k=%d outside [1, min(E, max_k)]", k);
  if (T > 0 && (!idx_l || !load)) return fail(ctx, MOE_ERR_INVALID_ARG, "NULL tensor");
  if (idx_l1 && !coact) return fail(ctx, MOE_ERR_INVALID_ARG, "coact is NULL but idx_l1 is given");
  cudaStream_t s = (cudaStream_t)stream;
  ctx->last_stream = s;
  if (T == 0) return MOE_OK;
  launch_route_stats(idx_l, idx_l1, T, E, k, load, coact, ctx->err_dev, ctx->num_sms, s);
  LAUNCHED(ctx, 1);
  return MOE_OK;
}

moe_status moe_stats_allreduce(moe_ctx_t ctx, int64_t* load, int64_t* coact, int32_t E, moe_stream_t stream) {
  if (!ctx) return fail(ctx, MOE_ERR_INVALID_ARG, "ctx is NULL");
  DeviceGuard device_guard;
  CU(cudaSetDevice(ctx->cfg.device));
  if (E != ctx->E || !load) return fail(ctx, MOE_ERR_INVALID_ARG, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  ctx->last_stream = s;
  if (ctx->local_group) return fail(ctx, MOE_ERR_UNSUPPORTED, "statistics all-reduce in a single-process group");
  if (!ctx->comm) return MOE_OK;
  NC(ncclGroupStart());
  NC(ncclAllReduce(load, load, E, ncclInt64, ncclSum, ctx->comm, s));
  if (coact) NC(ncclAllReduce(coact, coact, (size_t)E * E, ncclInt64, ncclSum, ctx->comm, s));
  NC(ncclGroupEnd());
  return MOE_OK;
}

moe_status moe_stats_allreduce_layers(moe_ctx_t ctx, int64_t* load, int64_t* coact, int32_t E, int32_t L,
                                      moe_stream_t stream) {
  if (!ctx) return fail(ctx, MOE_ERR_INVALID_ARG, "ctx is NULL");
  DeviceGuard device_guard;
  CU(cudaSetDevice(ctx->cfg.device));
  if (E != ctx->E || !load || L < 1) return fail(ctx, MOE_ERR_INVALID_ARG, "bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  ctx->last_stream = s;
  if (ctx->local_group) return fail(ctx, MOE_ERR_UNSUPPORTED, "statistics all-reduce in a single-process group");
  if (!ctx->comm) return MOE_OK;
  NC(ncclGroupStart());
  NC(ncclAllReduce(load, load, (size_t)L * E, ncclInt64, ncclSum, ctx->comm, s));
  if (coact && L > 1) NC(ncclAllReduce(coact, coact, (size_t)(L - 1) * E * E, ncclInt64, ncclSum, ctx->comm, s));
  NC(ncclGroupEnd());
  return MOE_OK;
}

moe_status moe_pack_w13(const moe_bf16* w1, const moe_bf16* w3, int32_t n, int32_t F, int32_t H, moe_bf16* w13,
                        moe_stream_t stream) {
  moe_ctx_t ctx = nullptr;
  if (!w1 || !w3 || !w13 || n < 0 || F <= 0 || H <= 0 || F % 64 || H % 64)
    return fail(ctx, MOE_ERR_INVALID_ARG, "bad arguments (F, H multiples of 64)");
  if (n == 0) return MOE_OK;
  launch_pack_w13(w1, w3, n, F, H, w13, (cudaStream_t)stream);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, MOE_ERR_CUDA, "pack launch: %s", cudaGetErrorString(e));
  return MOE_OK;
}

// moe_dispatch (prev == NULL) and moe_dispatch_from (prev = layer l's context: the
// rows are combined from layer l's expert outputs on the hosting ranks, NEXT-4).
static moe_status ce_dispatch_copies(moe_ctx_t ctx);

static moe_status dispatch_impl(moe_ctx_t ctx, const moe_bf16* x, const int32_t* idx, int32_t T, int32_t k,
                                const int32_t* expert_to_rank, moe_dispatch_info* info, cudaStream_t s,
                                moe_ctx_t prev, const float* w_prev) {
  DeviceGuard device_guard;
  const int E = ctx->E, G = ctx->G, H = ctx->H;
  const bool direct = prev != nullptr;
  const int n_grp = G / ctx->tp;  // EP ranks (groups of tp ranks when tp > 1)
  ctx->last_stream = s;
  CU(cudaSetDevice(ctx->cfg.device));

  ctx->tl_cur = ctx->tl_used < (int)ctx->tl_mask.size() ? ctx->tl_used : -1;
  if (ctx->tl_cur >= 0) ctx->tl_mask[ctx->tl_cur] = 0;
  tl_rec(ctx, 0, s);
  cudaEvent_t ev_fork = ctx->ev_fork, ev_join = ctx->ev_join;
  if (ctx->p2p) {
    // the previous layer's side-stream scatter reads plan arrays this call rewrites.
    // Inside a CUDA-graph capture the previous layer of the graph already joined the
    // side stream in its moe_combine (and graph launches are serialised), and an
    // event recorded outside the capture may not be waited on -- skip the wait and
    // fork/join through the capture-only events.
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CU(cudaStreamIsCapturing(s, &cs));
    if (cs == cudaStreamCaptureStatusNone) {
      CU(cudaStreamWaitEvent(s, ctx->ev_join, 0));
    } else {
      ev_fork = ctx->ev_fork_cap;
      ev_join = ctx->ev_join_cap;
    }
    ctx->cur_join = ev_join;
  }
  // gather dispatch (see moe_ctx::tokbuf): top-k >= G/tp, or MOE_DISPATCH
  bool gather = false;  // measured slower than scatter at E64 top-8 4EP: opt-in
  if (const char* dm = getenv("MOE_DISPATCH")) gather = ctx->p2p && !strcmp(dm, "gather");
  if (direct) gather = false;
  ctx->last_gather = gather;
  ctx->last_direct = direct;
  // copy-engine data plane (opt-in, MOE_A2A_CE=1): plain EP (tp 1) with 256-row GEMM
  // tiles, outside CUDA-graph capture (moe_expert_ffn reads the counts on the host)
  bool ce = false;
  if (ctx->p2p && !gather && !direct && ctx->tp == 1 && ctx->gemm_cg == 2) {
    if (const char* env = getenv("MOE_A2A_CE")) ce = atoi(env) != 0;
    // ranks sharing a device: three streams each (caller, side, side2) must not alias
    // onto one hardware queue -- a copy stream's value wait would block the GEMM behind it
    int conns = 8;
    if (const char* cm = getenv("CUDA_DEVICE_MAX_CONNECTIONS")) conns = atoi(cm);
    if (ctx->share > 1 && 3 * ctx->share > conns) ce = false;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CU(cudaStreamIsCapturing(s, &cs));
    if (cs != cudaStreamCaptureStatusNone) ce = false;
  }
  ctx->last_ce = ce;
  PlanArgs a = plan_args(ctx, T, k);
  a.gather = gather ? 1 : 0;
  a.direct = direct ? 1 : 0;
  PlanBuffers b = plan_buffers(ctx);
  b.P_in = expert_to_rank;
  if (direct) {
    b.prev_row = prev->row_of_item;
    b.prev_slot = prev->slot_of_item;
    b.prev_w = w_prev;
    b.prev_k = prev->last_k;
    b.prev_src = prev->src_table;
    b.prev_flag_y = prev->sig->flag_y;
    b.prev_epoch = prev->epoch_dev;
  }
  launch_count(a, idx, b, s);
  launch_scan(a, b, s);
  LAUNCHED(ctx, (a.n_tiles > 0) + 1);
  const bool nccl = ctx->comm != nullptr && !ctx->p2p;
  if (nccl) {
    // the counts and every rank's placement: one all-gather, one host read (the
    // send/recv segments are posted from the host); all ranks must dispatch with
    // the same map (the call discipline of moe_dispatch)
    NC(ncclGroupStart());
    NC(ncclAllGather(ctx->cnt_local, ctx->cnt_all, E, ncclInt32, ctx->comm, s));
    NC(ncclAllGather(expert_to_rank, ctx->P_all, E, ncclInt32, ctx->comm, s));
    NC(ncclGroupEnd());
    CU(cudaMemcpyAsync(ctx->cnt_pinned, ctx->cnt_all, sizeof(int32_t) * G * E, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(ctx->P_all_pinned, ctx->P_all, sizeof(int32_t) * G * E, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    memcpy(ctx->cnt_host.data(), ctx->cnt_pinned, sizeof(int32_t) * G * E);
    memcpy(ctx->P_host.data(), ctx->P_all_pinned + (size_t)ctx->me * E, sizeof(int32_t) * E);
    for (int e = 0; e < E; ++e)
      if (ctx->P_host[e] < 0 || ctx->P_host[e] >= n_grp) {
        ctx->have_plan = false;
        return fail(ctx, MOE_ERR_INVALID_ARG, "expert_to_rank[%d]=%d outside [0, %d)", e, ctx->P_host[e], n_grp);
      }
    for (int g = 0; g < G; ++g)
      if (memcmp(ctx->P_all_pinned + (size_t)g * E, ctx->P_host.data(), sizeof(int32_t) * E) != 0) {
        ctx->have_plan = false;
        return fail(ctx, MOE_ERR_DEVICE, "ranks dispatched with different expert_to_rank maps (rank %d differs)", g);
      }
  }
  launch_layout(a, b, ctx->cap_rows, s);  // validates P; P2P: also the in-kernel count all-gather
  tl_rec(ctx, 1, s);
  if (ce) {  // the count matrix, placement and flag epoch of this dispatch, for the host
    CU(cudaMemcpyAsync(ctx->ce_pinned, ctx->sig->cnt, sizeof(int32_t) * G * E, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(ctx->ce_pinned + (size_t)G * E, ctx->P_dev, sizeof(int32_t) * E, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(ctx->ce_pinned + (size_t)G * E + E, ctx->epoch_dev, sizeof(unsigned), cudaMemcpyDeviceToHost,
                       s));
    CU(cudaMemcpyAsync(ctx->ce_pinned + (size_t)G * E + E + 1, ctx->err_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
    CU(cudaEventRecord(ctx->ev_cnt, s));
  }
  if (direct && !ctx->p2p) {
    // virtual ranks / one rank: descriptors, then every receive row combined in place
    launch_scatter(a, x, idx, b, 6, s);
    launch_expand_direct(a, b, 2 * ctx->num_sms, s);
    tl_rec(ctx, 2, s);
    tl_rec(ctx, 3, s);
    LAUNCHED(ctx, 2);
  } else if (direct) {
    // side stream: every row's combine descriptors to its hosting rank (flag_data),
    // then this rank's rows combined from the layer-l outputs once every source's
    // descriptors and every rank's layer-l outputs are there (flag_exp for K5)
    CU(cudaEventRecord(ev_fork, s));
    CU(cudaStreamWaitEvent(ctx->side, ev_fork, 0));
    launch_scatter(a, x, idx, b, 6, ctx->side, ctx->remote_ctas);
    launch_expand_direct(a, b, 2 * ctx->num_sms, ctx->side);
    tl_rec(ctx, 3, ctx->side);
    CU(cudaEventRecord(ev_join, ctx->side));
    // every receive row -- this rank's own tokens' too -- comes out of the expansion,
    // so K5 has nothing to start on before it: join, and the expansion gets the
    // whole GPU.  (Letting K5 start and wait per tile for the sources' rows, as the
    // scatter dispatch does, measured as a stall: the expansion made no progress
    // next to the waiting K5 until K5's flag waits timed out -- gpurun_out r2l-r2n.)
    CU(cudaStreamWaitEvent(s, ev_join, 0));
    tl_rec(ctx, 2, s);
    LAUNCHED(ctx, 2);
  } else if (ce) {
    // copy-engine mode: this rank's own rows into its receive rows, the peers' rows
    // into the send buffer in send order; moe_expert_ffn queues the copies
    launch_scatter(a, x, idx, b, 7, s);
    CU(cudaEventRecord(ctx->ev_staged, s));
    tl_rec(ctx, 2, s);
    tl_rec(ctx, 3, s);
    LAUNCHED(ctx, 1);
    ctx->ce_dispatched = false;
    if (!ctx->local_group) {
      moe_status st = ce_dispatch_copies(ctx);
      if (st != MOE_OK) return st;
    }
  } else if (ctx->p2p) {
    // rows for peers: NVLink stores on the side stream (arrival flags raised by its
    // last CTA); rows hosted here: on `stream`, so K5 can start on them right away
    if (!gather) {
      // the plan arrays first (the TMA push reads them), then the fork
      launch_scatter(a, x, idx, b, 3, s);
      a.plan_done = 1;
      LAUNCHED(ctx, 1);
    }
    CU(cudaEventRecord(ev_fork, s));
    CU(cudaStreamWaitEvent(ctx->side, ev_fork, 0));
    if (!gather) {
      // the peers' rows on the TMA engines: one 1-warp CTA per SM (two 4 KB pieces in
      // flight each; ~12 KB of shared memory, so it fits next to the GEMM's CTA)
      launch_push_tma(a, x, b, ctx->num_sms, ctx->side);
    } else {
      // side stream: each token row once to every rank hosting one of its experts,
      // plus the row -> token-row map entries (flag_data), then this rank's expansion
      // of the rows its peers sent, source by source as they arrive.  (Reusing the
      // peers' token buffers is safe: every peer expanded the previous layer's rows
      // before raising the flag_y this rank's last combine waited for.)
      launch_scatter(a, x, idx, b, 5, ctx->side, ctx->remote_ctas);
      launch_expand(a, b, ctx->remote_ctas, ctx->side);
      LAUNCHED(ctx, 1);
    }
    tl_rec(ctx, 3, ctx->side);
    CU(cudaEventRecord(ev_join, ctx->side));
    launch_scatter(a, x, idx, b, 1, s);
    tl_rec(ctx, 2, s);
    LAUNCHED(ctx, 3);
  } else {
    launch_scatter(a, x, idx, b, 0, s);
    tl_rec(ctx, 2, s);
    tl_rec(ctx, 3, s);  // no separate peers' scatter: same as event 2
    LAUNCHED(ctx, 2);
  }
  if (nccl) {
    const int32_t* P = ctx->P_host.data();
    const int32_t* cnt = ctx->cnt_host.data();
    std::vector<int32_t> recv_base((size_t)G * E);
    layout_host_impl(E, G, P, cnt, ctx->seg_align, nullptr, recv_base.data(), nullptr, nullptr);
    NC(ncclGroupStart());
    // sends: remote experts in key (P[e], e) order; compact send buffer
    int64_t off = 0;
    for (int g = 0; g < G; ++g) {
      if (g == ctx->me) continue;
      for (int e = 0; e < E; ++e) {
        if (P[e] != g) continue;
        const int64_t n = cnt[ctx->me * E + e];
        if (n) NC(ncclSend(ctx->sendbuf + off * H, (size_t)n * H, ncclBfloat16, g, ctx->comm, s));
        off += n;
      }
    }
    for (int src = 0; src < G; ++src) {
      if (src == ctx->me) continue;
      for (int e = 0; e < E; ++e) {
        if (P[e] != ctx->me) continue;
        const int64_t n = cnt[src * E + e];
        if (n)
          NC(ncclRecv(ctx->recv + (int64_t)recv_base[src * E + e] * H, (size_t)n * H, ncclBfloat16, src, ctx->comm, s));
      }
    }
    NC(ncclGroupEnd());
  }
  ctx->have_plan = true;
  ctx->ffn_done = false;
  ctx->last_T = T;
  ctx->last_k = k;
  ctx->last_tiles = a.n_tiles;
  if (info) {
    memset(info, 0, sizeof *info);
    CU(cudaStreamSynchronize(s));
    std::vector<int32_t> cnt((size_t)G * E), P(E);
    CU(cudaMemcpy(cnt.data(), b.cnt_all, sizeof(int32_t) * G * E, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(P.data(), ctx->P_dev, sizeof(int32_t) * E, cudaMemcpyDeviceToHost));
    info->world = G;
    int n_hosted = 0;
    for (int e = 0; e < E; ++e) n_hosted += (ctx->virt || P[e] == ctx->grp);
    info->num_local_experts = n_hosted;
    int64_t rr = 0;
    for (int g = 0; g < n_grp && g < 64; ++g) {
      int64_t r = 0;
      for (int src = 0; src < G; ++src)
        for (int e = 0; e < E; ++e)
          if (P[e] == g) r += cnt[src * E + e];
      info->recv_counts[g] = (int32_t)r;
      if (ctx->virt || g == ctx->grp) rr += r;
    }
    if (!ctx->virt)
      for (int g = 0; g < n_grp && g < 64; ++g) {
        int64_t sc = 0;
        for (int e = 0; e < E; ++e)
          if (P[e] == g) sc += cnt[ctx->me * E + e];
        info->send_counts[g] = (int32_t)sc;
      }
    info->recv_rows = rr;
  }
  return MOE_OK;
}

moe_status moe_dispatch(moe_ctx_t ctx, const moe_bf16* x, const int32_t* idx, int32_t T, int32_t k,
                        const int32_t* expert_to_rank, moe_dispatch_info* info, moe_stream_t stream) {
  if (!ctx) return fail(ctx, MOE_ERR_INVALID_ARG, "ctx is NULL");
  if (T < 0 || T > ctx->cfg.max_tokens) return fail(ctx, MOE_ERR_CAPACITY, "T=%d outside [0, max_tokens]", T);
  if (k < 1 || k > ctx->E || k > ctx->cfg.max_k) return fail(ctx, MOE_ERR_INVALID_ARG, "k=%d outside [1, min(E, max_k)]", k);
  if (!expert_to_rank) return fail(ctx, MOE_ERR_INVALID_ARG, "expert_to_rank is NULL");
  if (T > 0 && (!x || !idx)) return fail(ctx, MOE_ERR_INVALID_ARG, "NULL tensor");
  return dispatch_impl(ctx, x, idx, T, k, expert_to_rank, info, (cudaStream_t)stream, nullptr, nullptr);
}

moe_status moe_dispatch_from(moe_ctx_t ctx, moe_ctx_t prev, const float* w_prev, const int32_t* idx, int32_t T,
                             int32_t k, const int32_t* expert_to_rank, moe_stream_t stream) {
  if (!ctx || !prev) return fail(ctx, MOE_ERR_INVALID_ARG, "ctx / prev is NULL");
  if (ctx == prev) return fail(ctx, MOE_ERR_INVALID_ARG, "prev must be another context (layer l's outputs stay in it)");
  if (T < 0 || T > ctx->cfg.max_tokens) return fail(ctx, MOE_ERR_CAPACITY, "T=%d outside [0, max_tokens]", T);
  if (k < 1 || k > ctx->E || k > ctx->cfg.max_k) return fail(ctx, MOE_ERR_INVALID_ARG, "k=%d outside [1, min(E, max_k)]", k);
  if (!expert_to_rank) return fail(ctx, MOE_ERR_INVALID_ARG, "expert_to_rank is NULL");
  if (T > 0 && (!idx || !w_prev)) return fail(ctx, MOE_ERR_INVALID_ARG, "NULL tensor");
  if (!prev->have_plan || !prev->out_stay || !prev->ffn_done)
    return fail(ctx, MOE_ERR_INVALID_ARG, "prev needs moe_set_output_mode(prev, MOE_OUT_STAY) and its moe_expert_ffn");
  if (prev->last_T != T) return fail(ctx, MOE_ERR_INVALID_ARG, "prev dispatched %d tokens, not %d", prev->last_T, T);
  if (prev->last_k > ctx->cfg.max_k) return fail(ctx, MOE_ERR_INVALID_ARG, "prev's k exceeds this context's max_k");
  if (prev->H != ctx->H || prev->G != ctx->G || prev->virt != ctx->virt || prev->p2p != ctx->p2p ||
      prev->me != ctx->me || prev->cfg.device != ctx->cfg.device)
    return fail(ctx, MOE_ERR_INVALID_ARG, "prev must be the same rank of the same EP group (H, G, mode, device)");
  if (ctx->tp > 1 || prev->tp > 1) return fail(ctx, MOE_ERR_UNSUPPORTED, "direct dispatch with tp > 1");
  if (ctx->comm && !ctx->p2p) return fail(ctx, MOE_ERR_UNSUPPORTED, "direct dispatch needs MOE_A2A_P2P");
  cudaStream_t s = (cudaStream_t)stream;
  if (prev->p2p) CU(cudaStreamWaitEvent(s, prev->cur_join, 0));  // layer l's side stream is done with its plan
  return dispatch_impl(ctx, nullptr, idx, T, k, expert_to_rank, nullptr, s, prev, w_prev);
}

moe_status moe_set_output_mode(moe_ctx_t ctx, int32_t mode) {
  if (!ctx || (mode != MOE_OUT_HOME && mode != MOE_OUT_STAY)) return fail(ctx, MOE_ERR_INVALID_ARG, "bad arguments");
  if (mode == MOE_OUT_STAY && ctx->tp > 1) return fail(ctx, MOE_ERR_UNSUPPORTED, "MOE_OUT_STAY with tp > 1");
  ctx->out_stay = mode == MOE_OUT_STAY;
  return MOE_OK;
}

// Stream memory operations (driver API, through the runtime's entry-point query):
// a copy-engine stream raises a peer's arrival flag after its copies
// (cuStreamWriteValue32, with its default memory barrier) and waits for K6's segment
// counters (cuStreamWaitValue32, GEQ).
typedef int (*PfnStreamValue32)(cudaStream_t, unsigned long long, unsigned, unsigned);
static PfnStreamValue32 stream_op(const char* name);
// the address of a SigBlock field in rank r's signal block (peer mapping)
static unsigned long long ce_flag(moe_ctx_t ctx, int r, const unsigned* field) {
  const size_t off = reinterpret_cast<const char*>(field) - reinterpret_cast<const char*>(ctx->sig);
  return (unsigned long long)(reinterpret_cast<char*>(ctx->sig_h[r]) + off);
}
static PfnStreamValue32 stream_op(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<PfnStreamValue32>(p);
}

// Copy-engine data plane, host half (MOE_A2A_CE; see moe_ctx::last_ce).
// ce_dispatch_copies: blocks until this dispatch's count matrix is on the host, then
// queues on the side stream, per destination rank (rotated from me + 1), one peer copy
// per hosted expert run of the staged send buffer into the destination's receive rows,
// then flag_data[me] = epoch on the destination (K5 there waits per tile for it).
// Called at the end of moe_dispatch (the scatter staging the rows is already queued,
// so the GPU works while the host waits), or -- single-process groups, whose ranks'
// calls come from one thread in rank order -- by the rank's moe_expert_ffn.
static moe_status ce_dispatch_copies(moe_ctx_t ctx) {
  static PfnStreamValue32 write32 = stream_op("cuStreamWriteValue32");
  if (!write32) return fail(ctx, MOE_ERR_UNSUPPORTED, "stream memory operations unavailable");
  const int E = ctx->E, G = ctx->G, H = ctx->H, me = ctx->me;
  CU(cudaEventSynchronize(ctx->ev_cnt));
  const int32_t* cnt = ctx->ce_pinned;
  const int32_t* P = cnt + (size_t)G * E;
  ctx->ce_epoch = (unsigned)cnt[(size_t)G * E + E];
  // a failed count exchange (timeout, placement mismatch, capacity) leaves the counts
  // unusable: queue no copy (the error word stays latched for moe_ctx_sync)
  if (cnt[(size_t)G * E + E + 1] != 0) return report_device_error(ctx, cnt[(size_t)G * E + E + 1]);
  for (int e = 0; e < E; ++e)
    if (P[e] < 0 || P[e] >= G) return fail(ctx, MOE_ERR_DEVICE, "expert_to_rank[%d]=%d outside [0, %d)", e, P[e], G);
  ctx->cnt_host.assign(cnt, cnt + (size_t)G * E);
  ctx->P_host.assign(P, P + E);
  ctx->ce_recv_base.resize((size_t)G * E);
  ctx->ce_send_base.resize((size_t)G * E);
  layout_host_impl(E, G, P, cnt, ctx->seg_align, nullptr, ctx->ce_recv_base.data(), nullptr,
                   ctx->ce_send_base.data());
  cudaStream_t cs = ctx->side;
  const size_t rowb = (size_t)H * 2;
  CU(cudaStreamWaitEvent(cs, ctx->ev_staged, 0));
  // the destinations' expert runs interleaved (round j: the j-th hosted expert of every
  // destination, rotated from me + 1), each followed by its (me, e) flag: every
  // receiver gets its segments in K5's order, at the same pace
  std::vector<std::vector<int>> runs(G);
  for (int e = 0; e < E; ++e)
    if (P[e] != me && cnt[me * E + e] > 0) runs[P[e]].push_back(e);
  size_t rounds = 0;
  for (auto& r : runs) rounds = std::max(rounds, r.size());
  for (size_t j = 0; j < rounds; ++j)
    for (int q = 1; q < G; ++q) {
      const int g = (me + q) % G;
      if (j >= runs[g].size()) continue;
      const int e = runs[g][j];
      const int n = cnt[me * E + e];
      if ((int64_t)ctx->ce_recv_base[me * E + e] + n > ctx->cap_rows ||
          (int64_t)ctx->ce_send_base[me * E + e] + n > ctx->send_rows)
        return fail(ctx, MOE_ERR_CAPACITY, "copy-engine dispatch run outside the buffers");
      CU(cudaMemcpyAsync(static_cast<char*>(ctx->recv_h[g]) + (size_t)ctx->ce_recv_base[me * E + e] * rowb,
                         reinterpret_cast<char*>(ctx->sendbuf) + (size_t)ctx->ce_send_base[me * E + e] * rowb,
                         n * rowb, cudaMemcpyDeviceToDevice, cs));
      if (write32(cs, ce_flag(ctx, g, ctx->sig->flag_se + me * E + e), ctx->ce_epoch, 0) != 0)
        return fail(ctx, MOE_ERR_CUDA, "cuStreamWriteValue32 failed");
    }
  for (int g = 0; g < G; ++g)  // every row of this dispatch sent (identity FFN, debug reads)
    if (write32(cs, ce_flag(ctx, g, ctx->sig->flag_data + me), ctx->ce_epoch, 0) != 0)
      return fail(ctx, MOE_ERR_CUDA, "cuStreamWriteValue32 failed");
  CU(cudaEventRecord(ctx->cur_join, cs));
  ctx->ce_dispatched = true;
  return MOE_OK;
}

// ce_combine_copies: called by moe_expert_ffn after K6 is queued (outputs: 0 = this
// rank hosts nothing; 1 = K6 was launched after ev_k6 and counts its tiles per
// segment; 2 = the outputs are complete once the caller's stream reaches this point --
// the identity FFN).  Queues on the side stream, per hosted segment (K6's tile order),
// a wait on the segment's counter (every epilogue warp of every tile) and one copy per
// source run of the expert-output rows into the source's return buffer at its
// send-order slot; then flag_y[me] = epoch on every rank (K8 there reads the return
// buffer, and this rank's own rows from its expert-output buffer).
static moe_status ce_combine_copies(moe_ctx_t ctx, int outputs) {
  static PfnStreamValue32 write32 = stream_op("cuStreamWriteValue32");
  static PfnStreamValue32 wait32 = stream_op("cuStreamWaitValue32");
  if (!write32 || !wait32) return fail(ctx, MOE_ERR_UNSUPPORTED, "stream memory operations unavailable");
  if (!ctx->ce_dispatched) {
    moe_status st = ce_dispatch_copies(ctx);
    if (st != MOE_OK) return st;
  }
  ctx->ce_dispatched = false;
  const int E = ctx->E, G = ctx->G, H = ctx->H, me = ctx->me;
  const int32_t* cnt = ctx->cnt_host.data();
  const int32_t* P = ctx->P_host.data();
  cudaStream_t cs = ctx->side;
  const size_t rowb = (size_t)H * 2;
  if (outputs == 2) CU(cudaEventRecord(ctx->ev_k6, ctx->last_stream));
  if (outputs > 0) {
    // two copy streams, the segments alternating between them, so one segment's copies
    // run while the other stream waits for the next segment
    CU(cudaStreamWaitEvent(cs, ctx->ev_k6, 0));
    CU(cudaStreamWaitEvent(ctx->side2, ctx->ev_k6, 0));
    const int bn = gemm_block_n(H, false), tile_m = 128 * ctx->gemm_cg;
    int i = 0, used2 = 0;
    for (int e = 0; e < E; ++e) {
      if (P[e] != me) continue;
      int64_t rows = 0;
      for (int src = 0; src < G; ++src) rows += cnt[src * E + e];
      const unsigned target = (unsigned)(((rows + tile_m - 1) / tile_m) * (H / bn) * 4 * ctx->gemm_cg);
      if (target > 0 && !ctx->out_stay) {
        cudaStream_t st = (i & 1) ? ctx->side2 : cs;
        used2 |= i & 1;
        if (outputs == 1 && wait32(st, (unsigned long long)(ctx->segdone + i), target, 0) != 0)
          return fail(ctx, MOE_ERR_CUDA, "cuStreamWaitValue32 failed");
        for (int src = 0; src < G; ++src) {
          const int n = cnt[src * E + e];
          if (src == me || n == 0) continue;
          CU(cudaMemcpyAsync(static_cast<char*>(ctx->ret_h[src]) + (size_t)ctx->ce_send_base[src * E + e] * rowb,
                             reinterpret_cast<char*>(ctx->ybuf) + (size_t)ctx->ce_recv_base[src * E + e] * rowb,
                             n * rowb, cudaMemcpyDeviceToDevice, st));
        }
      }
      ++i;
    }
    CU(cudaEventRecord(ctx->ev_side2, ctx->side2));
    CU(cudaStreamWaitEvent(cs, ctx->ev_side2, 0));
    (void)used2;
    if (ctx->out_stay && i > 0 && outputs == 1) {  // outputs stay here: flag_y once the whole K6 is done
      CU(cudaEventRecord(ctx->ev_k6, ctx->last_stream));
      CU(cudaStreamWaitEvent(cs, ctx->ev_k6, 0));
    }
  }
  for (int r = 0; r < G; ++r)
    if (write32(cs, ce_flag(ctx, r, ctx->sig->flag_y + me), ctx->ce_epoch, 0) != 0)
      return fail(ctx, MOE_ERR_CUDA, "cuStreamWriteValue32 failed");
  CU(cudaEventRecord(ctx->cur_join, cs));
  return MOE_OK;
}

moe_status moe_expert_ffn(moe_ctx_t ctx, const moe_bf16* w13, const moe_bf16* w2, int32_t n_w, moe_stream_t stream) {
  if (!ctx) return fail(ctx, MOE_ERR_INVALID_ARG, "ctx is NULL");
  DeviceGuard device_guard;
  CU(cudaSetDevice(ctx->cfg.device));
  if (!ctx->have_plan) return fail(ctx, MOE_ERR_INVALID_ARG, "moe_expert_ffn before moe_dispatch");
  if (n_w < 0 || n_w > ctx->E) return fail(ctx, MOE_ERR_INVALID_ARG, "n_w=%d outside [0, E]", n_w);
  if (ctx->virt && n_w != ctx->E)
    return fail(ctx, MOE_ERR_INVALID_ARG, "virtual ranks host every expert: n_w=%d != E=%d", n_w, ctx->E);
  if (n_w > 0 && (!w13 || !w2)) return fail(ctx, MOE_ERR_INVALID_ARG, "NULL weights");
  cudaStream_t s = (cudaStream_t)stream;
  ctx->last_stream = s;
  PlanArgs a = plan_args(ctx, ctx->last_T, ctx->last_k);
  PlanBuffers b = plan_buffers(ctx);
  // Fused combine (K6 returns rows over NVLink, staged in smem, one bulk copy per
  // row piece): pays off when the combine's NVLink time is a sizeable fraction of
  // K6's tensor time, t_nvl/t_gemm ~ 1.8e3 / F -- measured -7% per layer at F = 2048
  // (E64, 4EP; profiles/r1_v8_*) and no difference at F = 14336 (Mixtral 2/4EP,
  // gpurun call 47).  Default: on for F/tp <= 8192; MOE_FUSED_COMBINE=0/1 overrides.
  {
    bool fused = ctx->Fl <= 8192;
    if (const char* env = getenv("MOE_FUSED_COMBINE")) fused = atoi(env) != 0;
    ctx->ffn_fused = ctx->p2p && fused && !ctx->out_stay;  // MOE_OUT_STAY: the outputs stay here
  }
  ctx->ffn_done = true;
  // MOE_OUT_STAY: no moe_combine follows to join the side stream -- join at the end
  // of this call (keeps a captured chain's streams joined)
  const bool join_here = ctx->out_stay && ctx->p2p;
  if (n_w == 0) {
    // no expert here: the placement must host none on this rank (checked on the
    // device), and in P2P mode every rank still hears "my outputs are ready"
    launch_expect_nseg(ctx->seg_meta, 0, ctx->err_dev, s);
    LAUNCHED(ctx, 1);
    if (ctx->last_ce) {
      moe_status st = ce_combine_copies(ctx, 0);
      if (st != MOE_OK) return st;
    } else if (ctx->p2p) {
      launch_signal(a, b, 2, s);
      LAUNCHED(ctx, 1);
    }
    if (join_here) CU(cudaStreamWaitEvent(s, ctx->cur_join, 0));
    return MOE_OK;
  }
  const int H = ctx->H, F = ctx->Fl, tp = ctx->tp;
  const bool vslices = ctx->virt && tp > 1;  // virtual TP: K6 once per FFN slice
  if (w13 != ctx->tmB1_ptr || w2 != ctx->tmB2_ptr || ctx->tmB_nw != n_w) {
    const int bn1 = gemm_b_box_rows(2 * F, true, ctx->gemm_cg), bn2 = gemm_b_box_rows(H, false, ctx->gemm_cg);
    if (!make_tmap_2d(ctx->tmB1, w13, (uint64_t)n_w * 2 * F, H, bn1) ||
        !make_tmap_2d(ctx->tmB2, w2, (uint64_t)n_w * H, F, bn2))
      return fail(ctx, MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed for the weights");
    if (vslices)
      for (int q = 0; q < tp; ++q)
        if (!make_tmap_2d_ld(ctx->tmB2s[q], w2 + (size_t)q * (F / tp), (uint64_t)n_w * H, F / tp, F, bn2))
          return fail(ctx, MOE_ERR_CUDA, "cuTensorMapEncodeTiled failed for a W2 slice");
    ctx->tmB1_ptr = w13;
    ctx->tmB2_ptr = w2;
    ctx->tmB_nw = n_w;
  }
  tl_rec(ctx, 4, s);
  const bool rec = ctx->timing_used < (int)ctx->ev.size() / 3;
  cudaEvent_t* ev = rec ? &ctx->ev[3 * ctx->timing_used] : nullptr;
  if (rec) CU(cudaEventRecord(ev[0], s));
  // P2P: K5's producer waits per tile for the source ranks whose rows the tile reads;
  // the tiles of this rank's own rows go first (overlapping the peers' NVLink pushes)
  const unsigned* arrived = (ctx->last_gather || ctx->last_direct) ? ctx->sig->flag_exp : ctx->sig->flag_data;
  // (direct dispatch: this rank's own rows are combined by k_expand_direct too -- wait for all)
  // copy-engine dispatch: per (source, segment) flags, raised after each run's copy,
  // so K5's phase-B tiles of the first segments start while the later runs still cross
  const SrcWait wait1{ctx->p2p ? arrived : nullptr, ctx->last_ce ? ctx->sig->flag_se : nullptr, ctx->seg_e, ctx->E,
                      ctx->seg_src, ctx->G, ctx->last_direct ? -1 : ctx->me, ctx->epoch_dev, ctx->flag_timeout_ns};
  const SrcWait nowait{nullptr, nullptr, nullptr, 0, nullptr, 0, 0, nullptr, 0};
  const FusedRet plain{nullptr, nullptr, 0, 0};
  // fused combine (P2P): K6's epilogue stores every output row over NVLink into its
  // source rank's return buffer at the item's send-order slot -- the combine
  // all-to-all overlaps the expert GEMM tile by tile
  const FusedRet fused{ctx->ret_table, ctx->seg_src, ctx->G, ctx->ffn_fused ? 1 : 0,
                      (ctx->last_ce && !ctx->ffn_fused) ? ctx->segdone : nullptr};
  // Split-K of the down projection in decode-sized contexts (about one 128-row M tile
  // per hosted expert): when K6's output tiles cannot cover the SMs, split K into S
  // slices (fp32 partials in a workspace, ordered reduction -- deterministic).
  // Measured (graph replays, Mixtral layer, profiles/r1_v15_small_t_splitk_*): K6 at
  // 4 GPUs (32 tiles) 64 tokens 0.273 -> 0.252 ms, 256 tokens 0.293 -> 0.283 ms; no
  // gain at 2 GPUs (64 tiles) and a loss at 1 GPU (128 tiles: the partials' extra
  // traffic), so only grids below a quarter of the SMs are split.  (Splitting K5 the
  // same way measured slower -- round 1 -- and was removed.)
  int ksplit = 1;
  if (ctx->gemm_cg == 1 && !vslices && !ctx->ffn_fused) {
    const long long tiles = (long long)n_w * (H / gemm_block_n(H, false));
    const int nkb = F / 64;
    if (tiles * 4 < ctx->num_sms)
      while (tiles * ksplit < ctx->num_sms && ksplit < 8 && nkb / (2 * ksplit) >= 4) ksplit *= 2;
    if (const char* env = getenv("MOE_DECODE_SPLITK")) ksplit = std::max(1, atoi(env));
  }
  if (ksplit > 1) {
    const size_t need = (size_t)ksplit * ctx->cap_rows * H * sizeof(float);
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    CU(cudaStreamIsCapturing(s, &cs));
    if (need > ctx->splitk_bytes && (cs != cudaStreamCaptureStatusNone || ctx->shared_dev)) {
      // no allocation inside a CUDA-graph capture (an eager call before the capture
      // sizes the workspace), nor next to a peer rank's kernels on this device (a
      // cudaFree would wait for them): run this launch unsplit
      ksplit = 1;
    } else if (need > ctx->splitk_bytes) {
      if (ctx->splitk_ws) CU(cudaFree(ctx->splitk_ws));
      ctx->splitk_ws = nullptr;
      ctx->splitk_bytes = 0;
      CU(cudaMalloc((void**)&ctx->splitk_ws, need));
      ctx->splitk_bytes = need;
    }
  }
  cudaError_t e = launch_grouped_gemm(ctx->tmA1, ctx->tmB1, ctx->hbuf, F, ctx->seg_meta, ctx->E, n_w, 2 * F, H, true,
                                      ctx->gemm_cg, ctx->num_sms, wait1, ctx->err_dev, ctx->done_counter + 2, plain,
                                      s, 1, nullptr, 0, ctx->tmDh);
  if (e != cudaSuccess) return fail(ctx, MOE_ERR_CUDA, "gemm1 launch: %s", cudaGetErrorString(e));
  if (ctx->last_ce && !ctx->ce_dispatched) {  // single-process group: the dispatch copies now
    moe_status st = ce_dispatch_copies(ctx);
    if (st != MOE_OK) return st;
  }
  // copy-engine dispatch: the rows return through the copy engines, or -- fused
  // combine (F/tp <= 8192) -- K6's epilogue stores them as in the SM path
  const bool ce_return = ctx->last_ce && !ctx->ffn_fused;
  if (rec) CU(cudaEventRecord(ev[1], s));
  tl_rec(ctx, 5, s);
  if (!vslices) {
    const long long pstride = (long long)ctx->cap_rows * H;
    if (ce_return) {  // K6's per-segment counters start from zero (the copy stream waits on them)
      CU(cudaMemsetAsync(ctx->segdone, 0, sizeof(unsigned) * ctx->E, s));
      CU(cudaEventRecord(ctx->ev_k6, s));
    }
    e = launch_grouped_gemm(ctx->tmA2, ctx->tmB2, ctx->ybuf, H, ctx->seg_meta, ctx->E, n_w, H, F, false,
                            ctx->gemm_cg, ctx->num_sms, nowait, ctx->err_dev, ctx->done_counter + 2, fused, s, ksplit,
                            ctx->splitk_ws, pstride, ctx->tmDy);
    if (e != cudaSuccess) return fail(ctx, MOE_ERR_CUDA, "gemm2 launch: %s", cudaGetErrorString(e));
    if (ksplit > 1) {
      e = launch_splitk_reduce(ctx->splitk_ws, pstride, ksplit, ctx->seg_meta, ctx->E, H, ctx->gemm_cg, ctx->ybuf, H,
                               ctx->num_sms, s);
      if (e != cudaSuccess) return fail(ctx, MOE_ERR_CUDA, "split-K reduce launch: %s", cudaGetErrorString(e));
      ctx->launches += 1;
    }
  } else {
    // partial output of FFN slice q (h columns and W2 columns [q F/tp, (q+1) F/tp))
    // into expert-output buffer q; the combine sums the slices
    for (int q = 0; q < tp; ++q) {
      e = launch_grouped_gemm(ctx->tmA2s[q], ctx->tmB2s[q], ctx->ybuf + (size_t)q * ctx->cap_rows * H, H,
                              ctx->seg_meta, ctx->E, n_w, H, F / tp, false, ctx->gemm_cg, ctx->num_sms, nowait,
                              ctx->err_dev, ctx->done_counter + 2, plain, s, 1, nullptr, 0, ctx->tmDys[q]);
      if (e != cudaSuccess) return fail(ctx, MOE_ERR_CUDA, "gemm2 slice launch: %s", cudaGetErrorString(e));
    }
    ctx->launches += tp - 1;
  }
  if (rec) {
    CU(cudaEventRecord(ev[2], s));
    ++ctx->timing_used;
  }
  tl_rec(ctx, 6, s);
  ctx->launches += 2;
  if (ce_return) {  // the copy engines return the rows and raise flag_y
    moe_status st = ce_combine_copies(ctx, 1);
    if (st != MOE_OK) return st;
  } else if (ctx->p2p) {  // expert outputs of this rank are ready for the peers' combine
    launch_signal(a, b, 2, s);
    LAUNCHED(ctx, 1);
  }
  if (join_here) {
    CU(cudaStreamWaitEvent(s, ctx->cur_join, 0));
    tl_rec(ctx, 7, s);              // no combine follows: close this layer's timeline record
    if (ctx->tl_cur >= 0) {
      ++ctx->tl_used;
      ctx->tl_cur = -1;
    }
  }
  return MOE_OK;
}

moe_status moe_ffn_timing_enable(moe_ctx_t ctx, int32_t max_records) {
  DeviceGuard device_guard;
  if (!ctx || max_records < 0) return fail(ctx, MOE_ERR_INVALID_ARG, "bad arguments");
  CU(cudaSetDevice(ctx->cfg.device));
  CU(cudaDeviceSynchronize());
  for (auto& e : ctx->ev) cudaEventDestroy(e);
  ctx->ev.assign((size_t)3 * max_records, nullptr);
  for (auto& e : ctx->ev) CU(cudaEventCreate(&e));
  ctx->timing_used = 0;
  return MOE_OK;
}

moe_status moe_ffn_timing_read(moe_ctx_t ctx, float* ms, int32_t max_records, int32_t* n_out) {
  if (!ctx || !ms || !n_out || max_records < 0) return fail(ctx, MOE_ERR_INVALID_ARG, "bad arguments");
  const int n = std::min(ctx->timing_used, max_records);
  for (int i = 0; i < n; ++i) {
    CU(cudaEventSynchronize(ctx->ev[3 * i + 2]));
    CU(cudaEventElapsedTime(&ms[2 * i], ctx->ev[3 * i], ctx->ev[3 * i + 1]));
    CU(cudaEventElapsedTime(&ms[2 * i + 1], ctx->ev[3 * i + 1], ctx->ev[3 * i + 2]));
  }
  *n_out = n;
  ctx->timing_used = 0;
  return MOE_OK;
}

moe_status moe_timeline_enable(moe_ctx_t ctx, int32_t max_records) {
  DeviceGuard device_guard;
  if (!ctx || max_records < 0) return fail(ctx, MOE_ERR_INVALID_ARG, "bad arguments");
  CU(cudaSetDevice(ctx->cfg.device));
  CU(cudaDeviceSynchronize());
  for (auto& e : ctx->tl) cudaEventDestroy(e);
  ctx->tl.assign((size_t)kTimeline * max_records, nullptr);
  for (auto& e : ctx->tl) CU(cudaEventCreate(&e));
  ctx->tl_mask.assign(max_records, 0);
  ctx->tl_used = 0;
  ctx->tl_cur = -1;
  return MOE_OK;
}

moe_status moe_timeline_read(moe_ctx_t ctx, float* ms, int32_t max_records, int32_t* n_out) {
  DeviceGuard device_guard;
  if (!ctx || !ms || !n_out || max_records < 0) return fail(ctx, MOE_ERR_INVALID_ARG, "bad arguments");
  CU(cudaSetDevice(ctx->cfg.device));
  CU(cudaDeviceSynchronize());
  const int n = std::min(ctx->tl_used, max_records);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < kTimeline; ++j) {
      float v = -1.f;
      if ((ctx->tl_mask[i] & 1u) && (ctx->tl_mask[i] >> j & 1u))
        CU(cudaEventElapsedTime(&v, ctx->tl[(size_t)i * kTimeline], ctx->tl[(size_t)i * kTimeline + j]));
      ms[(size_t)i * kTimeline + j] = v;
    }
  *n_out = n;
  ctx->tl_used = 0;
  return MOE_OK;
}

moe_status moe_debug_identity_ffn(moe_ctx_t ctx, moe_stream_t stream) {
  if (!ctx || !ctx->have_plan) return fail(ctx, MOE_ERR_INVALID_ARG, "no plan");
  DeviceGuard device_guard;
  CU(cudaSetDevice(ctx->cfg.device));
  cudaStream_t s = (cudaStream_t)stream;
  ctx->last_stream = s;
  ctx->ffn_fused = false;  // identity rows stay in the expert-output buffer; combine pulls them
  PlanArgs a = plan_args(ctx, ctx->last_T, ctx->last_k);
  PlanBuffers b = plan_buffers(ctx);
  if (ctx->p2p) {
    // join the side-stream scatter first (never spin on a flag another kernel of
    // this GPU raises), then wait for the peers' rows
    CU(cudaStreamWaitEvent(s, ctx->cur_join, 0));
    launch_wait((ctx->last_gather || ctx->last_direct) ? ctx->sig->flag_exp : ctx->sig->flag_data, ctx->G,
                ctx->epoch_dev, ctx->err_dev, ctx->flag_timeout_ns, s);
    LAUNCHED(ctx, 1);
  }
  const size_t ybytes = (size_t)ctx->cap_rows * ctx->H * 2;
  if (ctx->tpi == 0) CU(cudaMemcpyAsync(ctx->ybuf, ctx->recv, ybytes, cudaMemcpyDeviceToDevice, s));
  else CU(cudaMemsetAsync(ctx->ybuf, 0, ybytes, s));  // TP slices > 0 return zeros
  if (ctx->virt && ctx->tp > 1) CU(cudaMemsetAsync(ctx->ybuf + ybytes / 2, 0, ybytes * (ctx->tp - 1), s));
  if (ctx->last_ce) return ce_combine_copies(ctx, 2);
  if (ctx->p2p) {
    launch_signal(a, b, 2, s);
    LAUNCHED(ctx, 1);
  }
  return MOE_OK;
}

moe_status moe_combine(moe_ctx_t ctx, const float* w, moe_bf16* out, moe_stream_t stream) {
  if (!ctx) return fail(ctx, MOE_ERR_INVALID_ARG, "ctx is NULL");
  DeviceGuard device_guard;
  CU(cudaSetDevice(ctx->cfg.device));
  if (!ctx->have_plan) return fail(ctx, MOE_ERR_INVALID_ARG, "moe_combine before moe_dispatch");
  if (ctx->last_T > 0 && (!w || !out)) return fail(ctx, MOE_ERR_INVALID_ARG, "NULL tensor");
  if (ctx->out_stay) return fail(ctx, MOE_ERR_INVALID_ARG, "MOE_OUT_STAY: the outputs go to moe_dispatch_from");
  cudaStream_t s = (cudaStream_t)stream;
  ctx->last_stream = s;
  const int E = ctx->E, G = ctx->G, H = ctx->H;
  if (ctx->comm && !ctx->p2p) {  // NCCL mode; P2P mode pulls rows inside K8
    const int32_t* P = ctx->P_host.data();
    const int32_t* cnt = ctx->cnt_host.data();
    std::vector<int32_t> recv_base((size_t)G * E);
    layout_host_impl(E, G, P, cnt, ctx->seg_align, nullptr, recv_base.data(), nullptr, nullptr);
    NC(ncclGroupStart());
    for (int src = 0; src < G; ++src) {
      if (src == ctx->me) continue;
      for (int e = 0; e < E; ++e) {
        if (P[e] != ctx->me) continue;
        const int64_t n = cnt[src * E + e];
        if (n)
          NC(ncclSend(ctx->ybuf + (int64_t)recv_base[src * E + e] * H, (size_t)n * H, ncclBfloat16, src, ctx->comm, s));
      }
    }
    int64_t off = 0;
    for (int g = 0; g < G; ++g) {
      if (g == ctx->me) continue;
      for (int e = 0; e < E; ++e) {
        if (P[e] != g) continue;
        const int64_t n = cnt[ctx->me * E + e];
        if (n) NC(ncclRecv(ctx->retbuf + off * H, (size_t)n * H, ncclBfloat16, g, ctx->comm, s));
        off += n;
      }
    }
    NC(ncclGroupEnd());
  }
  PlanArgs a = plan_args(ctx, ctx->last_T, ctx->last_k);
  PlanBuffers b = plan_buffers(ctx);
  if (ctx->p2p && ctx->last_direct) CU(cudaStreamWaitEvent(s, ctx->cur_join, 0));  // plan arrays (side stream)
  if (ctx->p2p && (a.n_tiles == 0 || ctx->shared_dev)) {
    // every rank's expert outputs of this layer are ready (flag_y).  A rank without
    // tokens must wait too: its next dispatch writes count rows into the peers'
    // signal blocks, which they read until their own layout kernel of this layer is
    // done -- and every peer raises flag_y only after that.  Ranks sharing a device
    // wait with one CTA here instead of with every CTA of the combine (those would
    // hold the SMs a peer's expert GEMM needs to raise the flag).
    launch_wait(ctx->sig->flag_y, ctx->G, ctx->epoch_dev, ctx->err_dev, ctx->flag_timeout_ns, s);
    LAUNCHED(ctx, 1);
  }
  launch_combine(a, w, b, out, s);
  LAUNCHED(ctx, a.n_tiles > 0);
  tl_rec(ctx, 7, s);
  if (ctx->tl_cur >= 0) {
    ++ctx->tl_used;
    ctx->tl_cur = -1;
  }
  if (ctx->p2p) CU(cudaStreamWaitEvent(s, ctx->cur_join, 0));  // join the side stream
  return MOE_OK;
}

// Decode the device plan into the oracle's C3 terms (unpadded receive position
// on the destination rank, source send-order slot).
moe_status moe_debug_plan(moe_ctx_t ctx, int32_t* dest_rank, int32_t* recv_pos, int32_t* send_slot, int32_t* cnt_out) {
  DeviceGuard device_guard;
  if (!ctx || !ctx->have_plan) return fail(ctx, MOE_ERR_INVALID_ARG, "no plan");
  CU(cudaSetDevice(ctx->cfg.device));
  CU(cudaStreamSynchronize(ctx->last_stream));
  moe_status st = check_device_error(ctx);
  if (st != MOE_OK) return st;
  const int E = ctx->E, G = ctx->G, T = ctx->last_T, k = ctx->last_k;
  std::vector<int32_t> cnt((size_t)G * E), rows((size_t)std::max(1, T * k)), Pv(E);
  CU(cudaMemcpy(Pv.data(), ctx->P_dev, sizeof(int32_t) * E, cudaMemcpyDeviceToHost));
  std::vector<uint8_t> slots((size_t)std::max(1, T * k));
  std::vector<int32_t> cslots((size_t)std::max(1, T * k));
  const int32_t* cnt_dev = plan_buffers(ctx).cnt_all;
  CU(cudaMemcpy(cnt.data(), cnt_dev, sizeof(int32_t) * G * E, cudaMemcpyDeviceToHost));
  if (T * k) {
    CU(cudaMemcpy(rows.data(), ctx->row_of_item, sizeof(int32_t) * T * k, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(slots.data(), ctx->slot_of_item, (size_t)T * k, cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(cslots.data(), ctx->cslot_of_item, sizeof(int32_t) * T * k, cudaMemcpyDeviceToHost));
  }
  // P2P: per-rank padded layout of the destination rank
  std::vector<int32_t> peer_base((size_t)G * E);
  layout_host_impl(E, G, Pv.data(), cnt.data(), ctx->seg_align, nullptr, peer_base.data(), nullptr, nullptr);
  if (cnt_out) memcpy(cnt_out, cnt.data(), sizeof(int32_t) * G * E);
  const int32_t* P = Pv.data();
  // unpadded receive start of (e, s) on rank P[e]
  std::vector<int64_t> ustart((size_t)G * E);
  for (int g = 0; g < G; ++g) {
    int64_t acc = 0;
    for (int e = 0; e < E; ++e) {
      if (P[e] != g) continue;
      for (int s = 0; s < G; ++s) {
        ustart[(size_t)s * E + e] = acc;
        acc += cnt[(size_t)s * E + e];
      }
    }
  }
  // padded device receive base of (s, e): virtual mode concatenates every rank's
  // segments in key (P[e], e) order; real mode uses this rank's own buffer.
  std::vector<int64_t> pstart((size_t)G * E, 0);
  {
    std::vector<int> order(E);
    for (int e = 0; e < E; ++e) order[e] = e;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return P[x] < P[y]; });
    int64_t acc = 0;
    for (int e : order) {
      if (!(ctx->virt || P[e] == ctx->grp)) continue;
      int64_t r = 0;
      for (int s = 0; s < G; ++s) {
        pstart[(size_t)s * E + e] = acc + r;
        r += cnt[(size_t)s * E + e];
      }
      acc += (r + ctx->seg_align - 1) / ctx->seg_align * ctx->seg_align;
    }
  }
  // compact send base (remote experts only) of this rank
  std::vector<int64_t> rbase(E, 0);
  {
    int64_t acc = 0;
    for (int g = 0; g < G; ++g)
      for (int e = 0; e < E; ++e)
        if (P[e] == g && !(ctx->virt || g == ctx->grp)) {
          rbase[e] = acc;
          acc += cnt[(size_t)ctx->me * E + e];
        }
  }
  // expert of each item is needed to decode; reconstruct from the row ranges
  for (int t = 0; t < T; ++t) {
    int s = ctx->virt ? 0 : ctx->me;
    if (ctx->virt) {
      const int base = T / G, rem = T % G;
      int acc = 0;
      for (s = 0; s < G; ++s) {
        const int n = base + (s < rem ? 1 : 0);
        if (t < acc + n) break;
        acc += n;
      }
    }
    for (int j = 0; j < k; ++j) {
      const int64_t row = rows[(size_t)t * k + j];
      const int slot = slots[(size_t)t * k + j];
      int32_t dr = -1, rp = -1, ss = -1;
      if (row >= 0) {
        // find the expert whose range (in the buffer the slot names) contains the row
        for (int e = 0; e < E; ++e) {
          const int64_t n = cnt[(size_t)s * E + e];
          if (n == 0) continue;
          bool match;
          int64_t b0;
          if (ctx->virt) {
            match = slot == 0;
            b0 = pstart[(size_t)s * E + e];
          } else if (ctx->p2p) {
            match = P[e] == slot;
            b0 = peer_base[(size_t)s * E + e];
          } else {
            const bool remote = P[e] != ctx->grp;
            match = slot == (remote ? 1 : 0);
            b0 = remote ? rbase[e] : pstart[(size_t)s * E + e];
          }
          if (match && row >= b0 && row < b0 + n) {
            const int64_t rank_within = row - b0;
            dr = P[e];
            rp = (int32_t)(ustart[(size_t)s * E + e] + rank_within);
            ss = cslots[(size_t)t * k + j];  // the device's own C3 send-order slot
            break;
          }
        }
      }
      if (dest_rank) dest_rank[(size_t)t * k + j] = dr;
      if (recv_pos) recv_pos[(size_t)t * k + j] = rp;
      if (send_slot) send_slot[(size_t)t * k + j] = ss;
    }
  }
  return MOE_OK;
}

moe_status moe_debug_send(moe_ctx_t ctx, moe_bf16* rows_host, int64_t max_rows, int64_t* rows_out) {
  DeviceGuard device_guard;
  if (!ctx || !ctx->have_plan) return fail(ctx, MOE_ERR_INVALID_ARG, "no plan");
  const bool ce = ctx->p2p && ctx->last_ce;
  if (!(ctx->comm && !ctx->p2p) && !ce)
    return fail(ctx, MOE_ERR_UNSUPPORTED, "a send buffer exists in MOE_A2A_NCCL and copy-engine modes only");
  if (ce && ctx->local_group && ctx->cnt_host.size() != (size_t)ctx->G * ctx->E)
    return fail(ctx, MOE_ERR_INVALID_ARG, "single-process group: call after the rank's moe_expert_ffn");
  CU(cudaSetDevice(ctx->cfg.device));
  CU(cudaStreamSynchronize(ctx->last_stream));
  const int E = ctx->E, H = ctx->H;
  int64_t n = 0;
  for (int e = 0; e < E; ++e)
    if (ce || ctx->P_host[e] != ctx->grp) n += ctx->cnt_host[(size_t)ctx->me * E + e];
  if (rows_out) *rows_out = n;
  if (!rows_host) return MOE_OK;
  if (n > max_rows) return fail(ctx, MOE_ERR_CAPACITY, "max_rows too small (%lld)", (long long)n);
  if (n) CU(cudaMemcpy(rows_host, ctx->sendbuf, (size_t)n * H * 2, cudaMemcpyDeviceToHost));
  return MOE_OK;
}

moe_status moe_debug_recv(moe_ctx_t ctx, moe_bf16* rows_host, int64_t max_rows, int64_t* rows_out) {
  DeviceGuard device_guard;
  if (!ctx || !ctx->have_plan) return fail(ctx, MOE_ERR_INVALID_ARG, "no plan");
  CU(cudaSetDevice(ctx->cfg.device));
  if (ctx->p2p) {  // the peers' rows of the last dispatch have landed here
    CU(cudaStreamWaitEvent(ctx->last_stream, ctx->cur_join, 0));
    launch_wait((ctx->last_gather || ctx->last_direct) ? ctx->sig->flag_exp : ctx->sig->flag_data, ctx->G,
                ctx->epoch_dev, ctx->err_dev, ctx->flag_timeout_ns, ctx->last_stream);
  }
  CU(cudaStreamSynchronize(ctx->last_stream));
  {  // a flag wait that timed out (e.g. the rows were never sent) surfaces here
    moe_status st = check_device_error(ctx);
    if (st != MOE_OK) return st;
  }
  const int E = ctx->E, H = ctx->H;
  std::vector<int32_t> meta(1 + 3 * E + 4);
  CU(cudaMemcpy(meta.data(), ctx->seg_meta, sizeof(int32_t) * meta.size(), cudaMemcpyDeviceToHost));
  const int nseg = meta[0];
  int64_t out = 0;
  for (int i = 0; i < nseg; ++i) {
    const int64_t r0 = meta[1 + i], n = meta[1 + E + i];
    if (rows_host && out + n <= max_rows && n > 0)
      CU(cudaMemcpy(rows_host + out * H, ctx->recv + r0 * H, (size_t)n * H * 2, cudaMemcpyDeviceToHost));
    out += n;
  }
  if (rows_out) *rows_out = out;
  if (rows_host && out > max_rows) return fail(ctx, MOE_ERR_CAPACITY, "max_rows too small (%lld)", (long long)out);
  return MOE_OK;
}

}  // extern "C"
