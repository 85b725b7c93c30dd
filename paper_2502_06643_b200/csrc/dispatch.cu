// dispatch.cu -- K2 (placement-aware histogram + stable scan), K3 (16-byte
// vectorised gather/permute into the receive / send buffers, or straight into
// the peer's receive buffer over NVLink), K8 (fused weighted unpermute /
// combine, pulling peer rows over NVLink in P2P mode), and the P2P flags.
//
// Paper: tokens are "routed to remote GPUs using all-to-all communication based
// on their assigned experts", with the all-to-all before and after
// the expert FFN and an arbitrary expert->GPU map.
// Readings: G7 token blocks, G8 ascending expert order per GPU,
// G9 send order (P[e], e, t) / receive order (e, s, t), G13 empty ranks.
//
// Positions are never taken from atomics: every item's row is
//   base_row[s][e] + tile_base[tile][e] + (stable rank inside the tile),
// so the permutation is deterministic and bit-exact with the oracle (C3).
#include "common.cuh"
#include "kernels.h"

namespace moe {

__host__ __device__ __forceinline__ void source_block(int T, int V, int s, int& t0, int& t1) {
  const int base = T / V, rem = T % V;
  t0 = s * base + (s < rem ? s : rem);
  t1 = t0 + base + (s < rem ? 1 : 0);
}

int plan_tiles(int T, int V) {
  int n = 0;
  for (int s = 0; s < V; ++s) {
    int t0, t1;
    source_block(T, V, s, t0, t1);
    n += (t1 - t0 + kTileTokens - 1) / kTileTokens;
  }
  return n;
}

// tile -> (source, first token, end token, first tile of the source)
__device__ __forceinline__ void tile_info(const PlanArgs& a, int tile, int& s, int& t0, int& t1, int& tile0) {
  int first = 0;
  for (s = 0; s < a.V; ++s) {
    int b0, b1;
    source_block(a.T, a.V, s, b0, b1);
    const int nt = (b1 - b0 + kTileTokens - 1) / kTileTokens;
    if (tile < first + nt) {
      tile0 = first;
      t0 = b0 + (tile - first) * kTileTokens;
      t1 = min(t0 + kTileTokens, b1);
      return;
    }
    first += nt;
  }
  s = -1;
  t0 = t1 = 0;
  tile0 = first;
}

// ----------------------------------------------------------------- system-scope flags (P2P)
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Spin (system-scope acquire) until flags[0..n) >= epoch.  A peer that never
// arrives (a rank that skipped a collective call, a dead process) latches
// kErrTimeout after kFlagTimeoutNs instead of hanging the GPU.
__device__ __forceinline__ unsigned cur_epoch(const unsigned* p) { return *(volatile const unsigned*)p; }
__device__ __forceinline__ void wait_flags_geq(const unsigned* flags, int n, unsigned epoch, int* err,
                                               unsigned long long timeout_ns, int site) {
  for (int g = threadIdx.x; g < n; g += blockDim.x) {
    const uint64_t t0 = globaltimer_ns();
    while ((int)(ld_acquire_sys(flags + g) - epoch) < 0) {
      __nanosleep(64);
      if (globaltimer_ns() - t0 > timeout_ns) {
        atomicOr(err, timeout_bits(site));
        break;
      }
    }
  }
  __syncthreads();
}
__device__ __forceinline__ unsigned* sig_flag(SigBlock* s, int which, int idx) {
  return which == 0 ? &s->flag_cnt[idx] : which == 1 ? &s->flag_data[idx] : &s->flag_y[idx];
}
// raise flag `which`[me] = epoch on every rank (after making this thread's and,
// via the caller's barrier, the CTA's prior writes visible system-wide)
__device__ __forceinline__ void signal_all(const PlanArgs& a, const PlanBuffers& b, int which) {
  __threadfence_system();
  const unsigned epoch = cur_epoch(a.epoch_ptr);
  for (int g = 0; g < a.G; ++g) st_release_sys(sig_flag(b.peer_sig[g], which, a.me), epoch);
}

// ----------------------------------------------------------------- K2a: per-tile histogram
__global__ void __launch_bounds__(128) k_count(PlanArgs a, const int32_t* __restrict__ idx, PlanBuffers b) {
  __shared__ int hist[kMaxExperts];
  for (int e = threadIdx.x; e < a.E; e += blockDim.x) hist[e] = 0;
  __syncthreads();
  int s, t0, t1, tile0;
  tile_info(a, blockIdx.x, s, t0, t1, tile0);
  const int lane = threadIdx.x & 31;
  const int n = (t1 - t0) * a.k;
  for (int base = 0; base < n; base += blockDim.x) {
    const int i = base + threadIdx.x;
    int e = -1;
    if (i < n) {
      e = idx[(long long)t0 * a.k + i];
      if (e < 0 || e >= a.E) {
        atomicOr(b.err, kErrBadExpert);
        e = -1;
      }
    }
    unsigned m = __match_any_sync(0xffffffffu, e);
    if (e >= 0 && lane == __ffs(m) - 1) atomicAdd(&hist[e], __popc(m));
  }
  __syncthreads();
  for (int e = threadIdx.x; e < a.E; e += blockDim.x) b.tile_hist[(long long)blockIdx.x * a.E + e] = hist[e];
}

// ----------------------------------------------------------------- K2b: scan over tiles
// One CTA per local source.  Thread (e, c) sums chunk c of the source's tiles
// for expert e; chunk partials are scanned per expert; then each thread writes
// the exclusive prefix of its tiles.  Also emits cnt_local[s][e].
__global__ void __launch_bounds__(1024) k_scan(PlanArgs a, PlanBuffers b) {
  __shared__ int part[1024];
  const int s = blockIdx.x;
  int tile0 = 0;
  for (int q = 0; q < s; ++q) {
    int b0, b1;
    source_block(a.T, a.V, q, b0, b1);
    tile0 += (b1 - b0 + kTileTokens - 1) / kTileTokens;
  }
  int b0, b1;
  source_block(a.T, a.V, s, b0, b1);
  const int nt = (b1 - b0 + kTileTokens - 1) / kTileTokens;
  const int C = blockDim.x / a.E;  // chunks per expert
  const int e = threadIdx.x % a.E, c = threadIdx.x / a.E;
  const bool active = c < C;
  const int per = (nt + C - 1) / C;
  const int c0 = min(nt, c * per), c1 = min(nt, c0 + per);
  int sum = 0;
  if (active)
    for (int t = c0; t < c1; ++t) sum += b.tile_hist[(long long)(tile0 + t) * a.E + e];
  if (active) part[c * a.E + e] = sum;
  __syncthreads();
  if (threadIdx.x < a.E) {
    int run = 0;
    for (int q = 0; q < C; ++q) {
      int v = part[q * a.E + threadIdx.x];
      part[q * a.E + threadIdx.x] = run;
      run += v;
    }
    b.cnt_local[s * a.E + threadIdx.x] = run;
  }
  __syncthreads();
  if (active) {
    int run = part[c * a.E + e];
    for (int t = c0; t < c1; ++t) {
      const long long o = (long long)(tile0 + t) * a.E + e;
      const int v = b.tile_hist[o];
      b.tile_base[o] = run;
      run += v;
    }
  }
}

// ----------------------------------------------------------------- K2c: layout (1 CTA)
// In P2P mode the CTA first pushes this rank's count row into every rank's
// signal block and waits for every source's row (the count all-gather).
// Per expert e on rank p = P[e]: padded segment start rstart[e] inside rank p's
// receive buffer (experts ascending), vstart[e] = the same in the concatenated
// buffer of all ranks (virtual mode).  base_row[s][e] = destination row of the
// first item of (source s, expert e); NCCL mode sends remote items through a
// compact send buffer in key (P[e], e) order instead.
__global__ void __launch_bounds__(kMaxExperts) k_layout(PlanArgs a, PlanBuffers b, long long cap_rows) {
  __shared__ int rows_s[kMaxExperts], pad_s[kMaxExperts], p_s[kMaxExperts], key_e[kMaxExperts];
  const int e = threadIdx.x;
  const int E = a.E;
  const int* cnt = b.cnt_all;
  // the placement of this dispatch (device input): validated, copied to the context
  // for the later kernels; an out-of-range value latches kErrBadRank and is replaced
  // by 0 so every buffer index stays in bounds
  if (e < E) {
    int p = b.P_in[e];
    if (p < 0 || p >= a.G / a.tp) {
      atomicOr(b.err, kErrBadRank);
      p = 0;
    }
    p_s[e] = p;
    b.P[e] = p;
  }
  __syncthreads();
  if (a.p2p) {
    // this dispatch's flag value: the device-side epoch advances here, once per
    // dispatch, so a captured CUDA graph of the layer replays with fresh flags
    if (threadIdx.x == 0) {
      unsigned* ep = const_cast<unsigned*>(a.epoch_ptr);
      *(volatile unsigned*)ep = cur_epoch(ep) + 1u;
      __threadfence();
    }
    __syncthreads();
    if (e < E) {
      for (int g = 0; g < a.G; ++g) b.peer_sig[g]->cnt[a.me * E + e] = b.cnt_local[e];
      __threadfence_system();
    }
    // the placement this rank dispatches with travels with its counts: every rank
    // checks that all ranks agree (the call discipline of moe_dispatch)
    __shared__ unsigned my_hash;
    if (threadIdx.x == 0) {
      unsigned h = 2166136261u;  // FNV-1a over the placement
      for (int q = 0; q < E; ++q) h = (h ^ (unsigned)p_s[q]) * 16777619u;
      my_hash = h;
      for (int g = 0; g < a.G; ++g) b.peer_sig[g]->phash[a.me] = h;
      __threadfence_system();
    }
    __syncthreads();
    if (threadIdx.x == 0) signal_all(a, b, 0);
    wait_flags_geq(b.my_sig->flag_cnt, a.G, cur_epoch(a.epoch_ptr), b.err, a.timeout_ns, kWaitCounts);
    for (int g = threadIdx.x; g < a.G; g += blockDim.x)
      if (((volatile unsigned*)b.my_sig->phash)[g] != my_hash) atomicOr(b.err, kErrPlacement);
    cnt = b.my_sig->cnt;
  }
  if (e < E) {
    int r = 0;
    for (int s = 0; s < a.G; ++s) r += ((volatile const int*)cnt)[s * E + e];
    rows_s[e] = r;
    pad_s[e] = (r + a.seg_align - 1) / a.seg_align * a.seg_align;
  }
  __syncthreads();
  int* nseg = b.seg_meta;
  int* seg_row0 = b.seg_meta + 1;
  int* seg_rows = b.seg_meta + 1 + E;
  int* seg_w = b.seg_meta + 1 + 2 * E;
  int* totals = b.seg_meta + 1 + 3 * E;  // [0] padded rows, [1] unpadded rows
  if (e < E) {
    const int p = p_s[e];
    const int key = p * E + e;
    long long rstart = 0, vstart = 0;
    int pos_v = 0, pos_r = 0, send_base = 0;
    for (int q = 0; q < E; ++q) {
      const int kq = p_s[q] * E + q;
      if (kq < key) {
        vstart += pad_s[q];
        ++pos_v;
        if (p_s[q] == p) {
          rstart += pad_s[q];
          ++pos_r;
        }
        if (!a.virt && !a.p2p && p_s[q] != a.grp) send_base += ((volatile const int*)cnt)[a.me * E + q];
      }
    }
    const bool hosted = a.virt || p == a.grp;
    if (hosted) {
      const int pos = a.virt ? pos_v : pos_r;
      const long long start = a.virt ? vstart : rstart;
      seg_row0[pos] = (int)start;
      seg_rows[pos] = rows_s[e];
      seg_w[pos] = a.virt ? e : pos_r;
      b.seg_e[pos] = e;
      if (start + pad_s[e] > cap_rows) atomicOr(b.err, kErrCapacity);
    }
    for (int s = 0; s < a.V; ++s) {
      const int gs = a.virt ? s : a.me;  // global source id of local source s
      int base;
      if (a.virt || a.p2p || hosted) {
        long long acc = a.virt ? vstart : rstart;
        for (int q = 0; q < gs; ++q) acc += ((volatile const int*)cnt)[q * E + e];
        base = (int)acc;
      } else {
        base = send_base;
      }
      b.base_row[s * E + e] = base;
    }
    key_e[pos_v] = e;  // experts in send-order key (P[e], e) order (for cslot_base below)
    if (a.p2p) {
      // fused combine: for each hosted segment and source s, the rows of s inside the
      // segment and the C3 send-order slot of their first item in s's send order
      if (hosted) {
        long long row = rstart;
        for (int s = 0; s < a.G; ++s) {
          int slot0 = 0;
          for (int q = 0; q < E; ++q)
            if (p_s[q] * E + q < key) slot0 += ((volatile const int*)cnt)[s * E + q];
          const int n = ((volatile const int*)cnt)[s * E + e];
          int32_t* d = b.seg_src + ((long long)pos_r * a.G + s) * 3;
          d[0] = (int)row;
          d[1] = n;
          d[2] = slot0;
          row += n;
        }
      }
    }
  }
  // C3 send order of every local source s (G9: key (P[e], e), then token): the slot of
  // the first item of (s, e) is the count of s's items with a smaller key.  Thread s
  // walks the experts in key order.  (P2P: the fused combine's return slots; every
  // mode: moe_debug_plan reports these device-computed slots.)
  __syncthreads();
  for (int sl = threadIdx.x; sl < a.V; sl += blockDim.x) {
    const int gs = a.virt ? sl : a.me;
    int acc = 0;
    for (int pos = 0; pos < E; ++pos) {
      const int q = key_e[pos];
      b.cslot_base[sl * E + q] = acc;
      acc += ((volatile const int*)cnt)[gs * E + q];
    }
  }
  if (e == 0) {
    int n = 0, tp = 0, tu = 0;
    for (int q = 0; q < E; ++q)
      if (a.virt || p_s[q] == a.grp) {
        ++n;
        tp += pad_s[q];
        tu += rows_s[q];
      }
    *nseg = n;
    totals[0] = tp;
    totals[1] = tu;
  }
}

// ----------------------------------------------------------------- K2d + K3: ranks + row copies
// Per tile: stable in-tile rank of every item among items with the same expert
// (warp __match_any_sync + per-warp counts), row = base_row + tile_base + rank;
// then every token row of x is read once (16-byte vectors) and stored k times
// into the destination chosen by the item's slot: this rank's receive buffer,
// the compact NCCL send buffer, or (P2P) the receive buffer of rank P[e].
constexpr int kScatterThreads = 512;
constexpr int kMaxTileItems = kTileTokens * kMaxK;

struct TileItems {
  int row[kMaxTileItems];
  uint8_t slot[kMaxTileItems];
};

__device__ __forceinline__ int item_slot(const PlanArgs& a, int p) {
  if (a.virt) return 0;
  if (a.p2p) return p;
  return p == a.grp ? 0 : 1;
}

__device__ __forceinline__ void tile_ranks(const PlanArgs& a, const int32_t* __restrict__ idx, const PlanBuffers& b,
                                           int tile, int s, int t0, int t1, TileItems& it, int* run, int* wcnt,
                                           bool write_plan, bool ce_stage = false) {
  const int E = a.E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  for (int e = threadIdx.x; e < E; e += blockDim.x) run[e] = 0;
  const int n = (t1 - t0) * a.k;
  for (int base = 0; base < n; base += blockDim.x) {
    for (int q = threadIdx.x; q < nwarps * E; q += blockDim.x) wcnt[q] = 0;
    __syncthreads();
    const int i = base + threadIdx.x;
    int e = -1;
    if (i < n) {
      e = idx[(long long)t0 * a.k + i];
      if (e < 0 || e >= E) e = -1;  // latched by k_count
    }
    const unsigned m = __match_any_sync(0xffffffffu, e);
    const int wrank = __popc(m & ((1u << lane) - 1));
    if (e >= 0 && wrank == 0) wcnt[warp * E + e] = __popc(m);
    __syncthreads();
    if (i < n) {
      int row = -1, slot = 0, cslot = -1;
      if (e >= 0) {
        int r = run[e] + wrank;
        for (int w = 0; w < warp; ++w) r += wcnt[w * E + e];
        const int within = b.tile_base[(long long)tile * E + e] + r;  // stable rank among (s, e) items
        row = b.base_row[s * E + e] + within;
        slot = item_slot(a, b.P[e]);
        cslot = b.cslot_base[s * E + e] + within;
      }
      // copy-engine staging (mode 7): a peer's row goes to the send buffer at its
      // send-order slot (slot marker 255), this rank's own rows to its receive rows
      const bool to_send = ce_stage && row >= 0 && slot != a.me;
      it.row[i] = to_send ? cslot : row;
      it.slot[i] = to_send ? (uint8_t)255 : (uint8_t)slot;
      if (write_plan) {
        b.row_of_item[(long long)t0 * a.k + i] = row;
        b.slot_of_item[(long long)t0 * a.k + i] = (uint8_t)slot;
        b.cslot_of_item[(long long)t0 * a.k + i] = cslot;
      }
    }
    __syncthreads();
    for (int e2 = threadIdx.x; e2 < E; e2 += blockDim.x) {
      int add = 0;
      for (int w = 0; w < nwarps; ++w) add += wcnt[w * E + e2];
      run[e2] += add;
    }
    __syncthreads();
  }
}

// mode: 0 every row; (P2P overlap) 1 = rows this rank hosts, plus the plan
// arrays; 2 = rows for peers only (runs on a side stream next to K5, whose
// producer waits per tile for the sources it needs), last CTA raises flag_data.
__global__ void __launch_bounds__(kScatterThreads, 2) k_scatter(PlanArgs a, const uint4* __restrict__ x,
                                                             const int32_t* __restrict__ idx, PlanBuffers b,
                                                             int mode) {
  __shared__ TileItems it;
  __shared__ int run[kMaxExperts];
  extern __shared__ int wcnt[];  // [warps][E] (dynamic: small, so mode 2 co-resides with K5)
  __shared__ uint4* dst_s[kMaxWorld];
  __shared__ unsigned last;
  // col_split CTAs share a token tile; each recomputes the (cheap) in-tile
  // ranks and copies one slice of the hidden dimension.  The grid may be smaller
  // than tiles x col_split (persistent: each CTA loops over work units).
  const int split = a.col_split;
  const int nslots = a.p2p ? a.G : 2;
  for (int q = threadIdx.x; q < nslots; q += blockDim.x) dst_s[q] = b.dst_table[q];
  for (int unit = blockIdx.x; unit < a.n_tiles * split; unit += gridDim.x) {
  const int part = unit % split;
  const int tile = unit / split;
  int s, t0, t1, tile0;
  tile_info(a, tile, s, t0, t1, tile0);
  // the plan arrays (row / slot / send slot of every item) come from the launch that
  // covers this rank's items on the caller's stream: modes 0 and 1, or -- direct
  // dispatch, which copies no rows -- mode 6
  tile_ranks(a, idx, b, tile, s, t0, t1, it, run, wcnt,
             part == 0 && (mode == 0 || (mode == 1 && !a.plan_done) || mode == 3 || mode == 6 || mode == 7),
             mode == 7);
  if (mode == 3) {  // plan arrays only
    __syncthreads();
    continue;
  }
  if (mode == 6) {
    // direct dispatch: instead of x rows, every destination row gets the locations and
    // gate weights of the k layer-l expert outputs it combines
    const int n = (t1 - t0) * a.k;
    const int pk = b.prev_k;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int row = it.row[i];
      if (row < 0) continue;
      const long long gt = t0 + i / a.k;
      int32_t* d = b.desc_table[a.virt || !a.p2p ? 0 : it.slot[i]] + (long long)row * b.desc_k * 3;
      for (int j = 0; j < pk; ++j) {
        const long long gi = gt * pk + j;
        const int pr = b.prev_row[gi];
        d[3 * j] = b.prev_slot[gi];
        d[3 * j + 1] = pr;
        d[3 * j + 2] = __float_as_int(pr < 0 ? 0.f : b.prev_w[gi]);
      }
    }
    __syncthreads();
    continue;
  }
  if (mode == 5) {
    // gather dispatch: each token row goes ONCE to every peer hosting at least one of
    // its experts (tp > 1: every rank of those groups), into the peer's token buffer
    // at (this source, token); the peer's row map learns which token-buffer row each
    // of its receive rows is, and k_expand fills the receive layout locally
    __shared__ unsigned long long tmask[kTileTokens];
    const int n = (t1 - t0) * a.k;
    const int tr = a.me * (int)b.tok_rows;
    for (int q = threadIdx.x; q < t1 - t0; q += blockDim.x) tmask[q] = 0ull;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int row = it.row[i];
      if (row < 0) continue;
      const int trow = tr + t0 + i / a.k;
      for (int q = 0; q < a.tp; ++q) {
        const int r = it.slot[i] * a.tp + q;
        if (r == a.me) continue;
        if (part == 0) b.xmap_table[r][row] = trow;
        atomicOr(&tmask[i / a.k], 1ull << r);
      }
    }
    __syncthreads();
    const int cpr = a.H / 8;
    const int cw = (cpr + a.col_split - 1) / a.col_split;
    const int c_lo = part * cw;
    const int width = max(0, min(cpr, c_lo + cw) - c_lo);
    const long long total = (long long)(t1 - t0) * width;
    constexpr int U = 4;
    for (long long p0 = threadIdx.x; p0 < total; p0 += (long long)blockDim.x * U) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long p = p0 + (long long)u * blockDim.x;
        if (p < total) v[u] = __ldg(x + (long long)(t0 + p / width) * cpr + c_lo + p % width);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long p = p0 + (long long)u * blockDim.x;
        if (p >= total) continue;
        const int tok = (int)(p / width), c = c_lo + (int)(p % width);
        const long long dst = (long long)(tr + t0 + tok) * cpr + c;
        for (unsigned long long m = tmask[tok]; m; m &= m - 1) b.tok_table[__ffsll((long long)m) - 1][dst] = v[u];
      }
    }
    __syncthreads();
    continue;
  }
  // P2P, tp > 1: slot p (an EP group) fans out to ranks p*tp .. p*tp+tp-1 (the TP
  // all-gather inside the dispatch); otherwise a slot is one destination buffer
  const bool fan = a.p2p && a.tp > 1;
  const bool local_only = mode == 1;
  if (mode != 0 && mode != 7) {  // drop the rows the other kernel copies
    const int n = (t1 - t0) * a.k;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (it.row[i] < 0) continue;
      const bool drop = fan ? (local_only && it.slot[i] != a.grp) : ((it.slot[i] == a.me) != local_only);
      if (drop) it.row[i] = -1;
    }
    __syncthreads();
  }
  // copy: (token, 16-byte chunk) pairs, consecutive threads -> consecutive chunks
  const int cpr = a.H / 8;
  const int cw = (cpr + a.col_split - 1) / a.col_split;
  const int c_lo = part * cw;
  const int width = max(0, min(cpr, c_lo + cw) - c_lo);
  const int k = a.k;
  const long long total = (long long)(t1 - t0) * width;
  constexpr int U = 8;
  for (long long p0 = threadIdx.x; p0 < total; p0 += (long long)blockDim.x * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long p = p0 + (long long)u * blockDim.x;
      if (p < total) {
        const int tok = (int)(p / width), c = c_lo + (int)(p % width);
        v[u] = __ldg(x + (long long)(t0 + tok) * cpr + c);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long p = p0 + (long long)u * blockDim.x;
      if (p < total) {
        const int tok = (int)(p / width), c = c_lo + (int)(p % width);
        for (int j = 0; j < k; ++j) {
          const int i = tok * k + j;
          const int row = it.row[i];
          if (row < 0) continue;
          if (!fan) {
            uint4* d = it.slot[i] == 255 ? b.sendbuf : dst_s[it.slot[i]];
            d[(long long)row * cpr + c] = v[u];
          } else {
            const int r0 = it.slot[i] * a.tp;
            for (int q = 0; q < a.tp; ++q) {
              const int r = r0 + q;
              if (mode == 0 || ((r == a.me) == local_only)) dst_s[r][(long long)row * cpr + c] = v[u];
            }
          }
        }
      }
    }
  }
  __syncthreads();  // it / run are reused by the next work unit
  }
  if (a.p2p && (mode == 0 || mode == 5 || mode == 6)) {
    // the last CTA to finish raises flag_data[me] on every rank
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(b.done_counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (last && threadIdx.x == 0) {
      *b.done_counter = 0;
      signal_all(a, b, 1);
    }
  }
}

__global__ void k_signal(PlanArgs a, PlanBuffers b, int which);

// ----------------------------------------------------------------- TMA push of the peers' rows
// The dispatch of the rows this rank sends to its peers (P2P; K3's remote half).
// One warp per CTA, tokens in batches of 32 (one per lane): each lane collects its
// token's remote destinations (receive rows on peers; tp > 1: every rank of the
// item's group but this one) into shared memory; then lane 0 drives the bulk-copy
// (TMA) engine over the batch's (token, 4 KB piece) units -- one global -> shared
// copy of the piece, one shared -> global copy into every remote receive row, with
// an L2 evict-first hint (the destination reads it only when its GEMM gets there)
// -- with two pieces in flight.  Almost no SM instructions, so the grid (one CTA
// per SM, ~12 KB of shared memory) interferes little with the expert GEMM it runs
// next to: measured against 32 CTAs of 16-byte SM stores (the round-1 design),
// −4% per layer at Mixtral 4EP balanced, −1-2% at E64 top-8 4EP
// (profiles/r2_timeline_push_*).
constexpr int kPushStages = 2;
constexpr int kPushPiece = 4096;
constexpr int kPushDest = kMaxK * kMaxTP;  // destinations per token (k items x tp ranks)
__global__ void __launch_bounds__(32) k_push_tma(PlanArgs a, const uint8_t* __restrict__ x, PlanBuffers b) {
  __shared__ alignas(128) uint8_t stage_s[kPushStages][kPushPiece];
  __shared__ alignas(8) uint64_t full[kPushStages];
  __shared__ int2 dst_s[32][kMaxK];   // (destination slot, receive row) per (token of the batch, item)
  __shared__ int ndst_s[32];
  const int lane = threadIdx.x;
  const int rowb = a.H * 2;
  const int piece = rowb % kPushPiece == 0 ? kPushPiece : rowb;  // rows <= 4 KB go whole
  const int npieces = rowb / piece;
  if (lane == 0) {
    for (int q = 0; q < kPushStages; ++q) mbar_init(&full[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint32_t phase_bits = 0;  // bit q = phase of stage q
  const uint64_t pol = l2_evict_first_policy();
  // tokens per batch: up to 32, fewer when T is small, so every CTA gets a batch
  const int bsz = max(1, min(32, (a.T + (int)gridDim.x - 1) / (int)gridDim.x));
  const int nbatch = (a.T + bsz - 1) / bsz;
  for (int bt = blockIdx.x; bt < nbatch; bt += gridDim.x) {
    const int t = bt * bsz + lane;
    int nd = 0;
    if (lane < bsz && t < a.T) {
      for (int j = 0; j < a.k; ++j) {
        const long long gi = (long long)t * a.k + j;
        const int row = b.row_of_item[gi], slot = b.slot_of_item[gi];
        // tp > 1: the slot is an EP group whose every rank but this one gets the row
        if (row >= 0 && (a.tp > 1 || slot != a.me)) dst_s[lane][nd++] = make_int2(slot, row);
      }
    }
    ndst_s[lane] = nd;
    __syncwarp();
    if (lane == 0) {
      // the batch's units (token l, piece pc) with ndst > 0, in order, through a ring of
      // kPushStages shared-memory slots: up to kPushStages pieces loading at once
      int l = 0, pc = 0;
      while (l < 32 && ndst_s[l] == 0) ++l;
      int lq[kPushStages], pq[kPushStages];
      int issued = 0, done = 0;
      while (true) {
        while (issued - done < kPushStages && l < 32) {
          const int q = issued % kPushStages;
          lq[q] = l;
          pq[q] = pc;
          const uint32_t bar = smem_u32(&full[q]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(piece) : "memory");
          bulk_g2s(smem_u32(stage_s[q]), x + (long long)(bt * bsz + l) * rowb + (long long)pc * piece, piece, bar);
          ++issued;
          if (++pc == npieces) {
            pc = 0;
            do ++l; while (l < 32 && ndst_s[l] == 0);
          }
        }
        if (done == issued) break;
        const int q = done % kPushStages;
        mbar_wait(&full[q], (phase_bits >> q) & 1u);
        phase_bits ^= 1u << q;
        const int lt = lq[q];
        const long long off = (long long)pq[q] * piece;
        for (int d = 0; d < ndst_s[lt]; ++d) {
          const int2 sr = dst_s[lt][d];
          for (int tq = 0; tq < a.tp; ++tq) {
            const int r = a.tp == 1 ? sr.x : sr.x * a.tp + tq;
            if (r == a.me) continue;
            bulk_s2g_hint(reinterpret_cast<uint8_t*>(b.dst_table[r]) + (long long)sr.y * rowb + off,
                          smem_u32(stage_s[q]), piece, pol);
          }
        }
        bulk_commit();
        ++done;
        // the slot is refilled next: its stores must have read it
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    }
    __syncwarp();
  }
  // every store complete and visible before the arrival flag
  __shared__ unsigned last;
  if (lane == 0) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
    __threadfence_system();
    last = atomicAdd(b.done_counter, 1u) == gridDim.x - 1;
    if (last) {
      *b.done_counter = 0;
      signal_all(a, b, 1);
    }
  }
}

void launch_push_tma(const PlanArgs& a, const uint16_t* x, const PlanBuffers& b, int ctas, cudaStream_t s) {
  if (a.T <= 0) {
    k_signal<<<1, 32, 0, s>>>(a, b, 1);
    return;
  }
  k_push_tma<<<ctas, 32, 0, s>>>(a, reinterpret_cast<const uint8_t*>(x), b);
}

// ----------------------------------------------------------------- gather dispatch: expand
// The receiving side of the gather dispatch.  Source by source (rotated from
// me + 1), once flag_data[s] says s's token block and row map have landed: every
// row of every hosted segment that came from s is copied from the token buffer
// (row xmap[row]) into the receive layout, one warp per row, 16-byte vectors.
// The last CTA done with a source raises flag_exp[s] (K5's per-tile wait).
__global__ void __launch_bounds__(kScatterThreads) k_expand(PlanArgs a, PlanBuffers b) {
  __shared__ unsigned last;
  const unsigned epoch = cur_epoch(a.epoch_ptr);
  const int nseg = b.seg_meta_c[0];
  const int cpr = a.H / 8;
  const int lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + (threadIdx.x >> 5), stride = gridDim.x * nw;
  for (int q = 1; q < a.G; ++q) {
    const int s = (a.me + q) % a.G;
    if (threadIdx.x == 0) {
      const uint64_t t0 = globaltimer_ns();
      while ((int)(ld_acquire_sys(&b.my_sig->flag_data[s]) - epoch) < 0) {
        __nanosleep(128);
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          atomicOr(b.err, timeout_bits(kWaitGatherRows));
          break;
        }
      }
    }
    __syncthreads();
    for (int pos = 0; pos < nseg; ++pos) {
      const int32_t* d = b.seg_src + ((long long)pos * a.G + s) * 3;
      const int row0 = d[0], n = d[1];
      for (int r = gw; r < n; r += stride) {
        const long long row = row0 + r;
        const uint4* src = b.tok_local + (long long)b.xmap_local[row] * cpr;
        uint4* dst = b.recv_local + row * cpr;
        for (int c = lane; c < cpr; c += 32) dst[c] = src[c];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(&b.exp_counter[s], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      b.exp_counter[s] = 0;
      __threadfence();
      st_release_sys(&b.my_sig->flag_exp[s], epoch);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) st_release_sys(&b.my_sig->flag_exp[a.me], epoch);
}

// ----------------------------------------------------------------- direct dispatch: combine here
// NEXT-4 (the inter-layer traffic Eq. 8 models): the rows of layer l+1
// are formed on the rank hosting their layer-(l+1) expert, straight from layer l's
// expert outputs where they were computed (a local read when ILP 2 put the two
// experts on one GPU, an NVLink load otherwise) -- no return to the home rank.
// Same arithmetic as K8 (fp32 FMA, j ascending, one bf16 rounding), so the layer
// input is bit-identical to the home-rank chain's.  P2P: once every rank's layer-l
// outputs are ready (layer-l flag_y), source by source in ascending order (the
// segments' row order, so K5's first tiles come free first) as each source's
// descriptors arrive (flag_data); flag_exp[s] is raised per source for K5's
// per-tile waits.  Virtual / one rank: every hosted row in one pass.
__device__ __forceinline__ void direct_rows(const PlanArgs& a, const PlanBuffers& b, const uint4* const* src_s,
                                            long long row0, int n, int gw, int stride, int lane) {
  const int cpr = a.H / 8, pk = b.prev_k, dk = b.desc_k;
  constexpr int U = 4;  // 16-byte chunks per lane in flight (k loads each)
  for (int r = gw; r < n; r += stride) {
    const long long row = row0 + r;
    const int32_t* d = b.desc_local + row * dk * 3;
    for (int c0 = lane; c0 < cpr; c0 += 32 * U) {
      float acc[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < 8; ++q) acc[u][q] = 0.f;
      for (int j = 0; j < pk; ++j) {
        const int prow = d[3 * j + 1];
        if (prow < 0) continue;
        const float wj = __int_as_float(d[3 * j + 2]);
        const uint4* src = src_s[d[3 * j]] + (long long)prow * cpr;
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int c = c0 + 32 * u;
          v[u] = c < cpr ? src[c] : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          acc[u][0] = fmaf(wj, bf16_lo(v[u].x), acc[u][0]);
          acc[u][1] = fmaf(wj, bf16_hi(v[u].x), acc[u][1]);
          acc[u][2] = fmaf(wj, bf16_lo(v[u].y), acc[u][2]);
          acc[u][3] = fmaf(wj, bf16_hi(v[u].y), acc[u][3]);
          acc[u][4] = fmaf(wj, bf16_lo(v[u].z), acc[u][4]);
          acc[u][5] = fmaf(wj, bf16_hi(v[u].z), acc[u][5]);
          acc[u][6] = fmaf(wj, bf16_lo(v[u].w), acc[u][6]);
          acc[u][7] = fmaf(wj, bf16_hi(v[u].w), acc[u][7]);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = c0 + 32 * u;
        if (c >= cpr) continue;
        uint4 o;
        o.x = pack_bf16x2(acc[u][0], acc[u][1]);
        o.y = pack_bf16x2(acc[u][2], acc[u][3]);
        o.z = pack_bf16x2(acc[u][4], acc[u][5]);
        o.w = pack_bf16x2(acc[u][6], acc[u][7]);
        b.recv_local[row * cpr + c] = o;
      }
    }
  }
}

__global__ void __launch_bounds__(kScatterThreads, 2) k_expand_direct(PlanArgs a, PlanBuffers b) {
  __shared__ const uint4* src_s[kMaxWorld];
  __shared__ unsigned last;
  const int nslots = a.p2p ? a.G : 1;
  for (int q = threadIdx.x; q < nslots; q += blockDim.x) src_s[q] = b.prev_src[q];
  const int E = a.E;
  const int nseg = b.seg_meta_c[0];
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int gw = blockIdx.x * nw + (threadIdx.x >> 5), stride = gridDim.x * nw;
  if (!a.p2p) {
    __syncthreads();
    for (int pos = 0; pos < nseg; ++pos)
      direct_rows(a, b, src_s, b.seg_meta_c[1 + pos], b.seg_meta_c[1 + E + pos], gw, stride, lane);
    return;
  }
  const unsigned ep = cur_epoch(a.epoch_ptr);
  if (threadIdx.x == 0) {          // every rank's layer-l outputs (any of them may be read)
    const unsigned pep = cur_epoch(b.prev_epoch);
    const uint64_t t0 = globaltimer_ns();
    for (int g = 0; g < a.G; ++g)
      while ((int)(ld_acquire_sys(b.prev_flag_y + g) - pep) < 0) {
        __nanosleep(128);
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          atomicOr(b.err, timeout_bits(kWaitPrevOutputs));
          break;
        }
      }
  }
  __syncthreads();
  for (int s = 0; s < a.G; ++s) {
    if (threadIdx.x == 0) {        // source s's descriptors have landed
      const uint64_t t0 = globaltimer_ns();
      while ((int)(ld_acquire_sys(&b.my_sig->flag_data[s]) - ep) < 0) {
        __nanosleep(128);
        if (globaltimer_ns() - t0 > a.timeout_ns) {
          atomicOr(b.err, timeout_bits(kWaitDescriptors));
          break;
        }
      }
    }
    __syncthreads();
    for (int pos = 0; pos < nseg; ++pos) {
      const int32_t* d = b.seg_src + ((long long)pos * a.G + s) * 3;
      direct_rows(a, b, src_s, d[0], d[1], gw, stride, lane);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(&b.exp_counter[s], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
      b.exp_counter[s] = 0;
      __threadfence();
      st_release_sys(&b.my_sig->flag_exp[s], ep);
    }
  }
}

__global__ void k_signal(PlanArgs a, PlanBuffers b, int which) {
  if (threadIdx.x == 0) signal_all(a, b, which);
}

// ----------------------------------------------------------------- K8: weighted unpermute
// out[t] = bf16( sum_{j ascending} w[t][j] * Y[item (t,j)] ), fp32 FMA (reading G4).
// KT = compile-time k (0: runtime k).  Every (token, 16-byte chunk) pair loads
// all k source rows before accumulating, so U*k 16-byte loads are in flight per
// thread; the accumulation order is still j ascending.  In P2P mode the rows
// are read from the hosting rank's expert-output buffer over NVLink.
template <int KT>
__global__ void __launch_bounds__(kScatterThreads, 2) k_combine(PlanArgs a, const float* __restrict__ w, PlanBuffers b,
                                                             uint4* __restrict__ out) {
  __shared__ int row_s[kMaxTileItems];
  __shared__ float w_s[kMaxTileItems];
  __shared__ uint8_t slot_s[kMaxTileItems];
  __shared__ const uint4* src_s[kMaxWorld];
  const int part = blockIdx.x % a.col_split;
  int s, t0, t1, tile0;
  tile_info(a, blockIdx.x / a.col_split, s, t0, t1, tile0);
  const int k = KT > 0 ? KT : a.k;
  const int n = (t1 - t0) * k;
  // source of partial q of an item with slot sl: src_s[sl * tp + q].  P2P pull: the
  // expert-output buffer of rank sl*tp+q; fused: the return buffer of slice q
  // (slot 0); virtual: the expert-output buffer of slice q (slot 0); NCCL: slot.
  const int nslots = a.ce ? 2 : (a.p2p && !a.fused) ? a.G : (a.tp > 1 ? a.tp : 2);
  for (int q = threadIdx.x; q < nslots; q += blockDim.x)
    src_s[q] = a.ce ? (q == 0 ? b.ret_local : b.src_table[a.me])
               : a.fused ? b.ret_local + q * b.part_stride
                         : ((a.virt && a.tp > 1) ? b.src_table[0] + q * b.part_stride : b.src_table[q]);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const long long gi = (long long)t0 * k + i;
    // fused combine: K6 already stored the row into this rank's return buffer at the C3
    // slot; copy-engine combine: the peers' rows were copied there, this rank's own rows
    // stay in its expert-output buffer
    const bool own = a.ce && b.slot_of_item[gi] == a.me;
    const int v = own ? b.row_of_item[gi] : (a.fused || a.ce) ? b.cslot_of_item[gi] : b.row_of_item[gi];
    row_s[i] = v;
    w_s[i] = v < 0 ? 0.f : w[gi];
    slot_s[i] = a.ce ? (own ? 1 : 0) : a.fused ? 0 : b.slot_of_item[gi];
  }
  if (a.p2p) wait_flags_geq(b.my_sig->flag_y, a.G, cur_epoch(a.epoch_ptr), b.err, a.timeout_ns, kWaitOutputs);
  __syncthreads();
  const int cpr = a.H / 8;
  const int cw = (cpr + a.col_split - 1) / a.col_split;
  const int c_lo = part * cw;
  const int width = max(0, min(cpr, c_lo + cw) - c_lo);
  const long long total = (long long)(t1 - t0) * width;
  if (a.tp > 1) {
    // Y[item] = sum_{q ascending} partial_q (fp32), then the j-ascending FMA of G4
    for (long long p = threadIdx.x; p < total; p += blockDim.x) {
      const int tok = (int)(p / width), c = c_lo + (int)(p % width);
      float acc[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[e] = 0.f;
      for (int j = 0; j < k; ++j) {
        const int i = tok * k + j;
        const int row = row_s[i];
        if (row < 0) continue;
        const uint4* const* srcs = src_s + slot_s[i] * a.tp;
        uint4 v[kMaxTP];
#pragma unroll
        for (int q = 0; q < kMaxTP; ++q)
          if (q < a.tp) v[q] = __ldg(srcs[q] + (long long)row * cpr + c);
        float y[8];
        bf16x8_to_f32(v[0], y);
#pragma unroll
        for (int q = 1; q < kMaxTP; ++q)
          if (q < a.tp) {
            float z[8];
            bf16x8_to_f32(v[q], z);
#pragma unroll
            for (int e = 0; e < 8; ++e) y[e] += z[e];
          }
        const float wj = w_s[i];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = fmaf(wj, y[e], acc[e]);
      }
      uint4 o;
      o.x = pack_bf16x2(acc[0], acc[1]);
      o.y = pack_bf16x2(acc[2], acc[3]);
      o.z = pack_bf16x2(acc[4], acc[5]);
      o.w = pack_bf16x2(acc[6], acc[7]);
      out[(long long)(t0 + tok) * cpr + c] = o;
    }
    return;
  }
  constexpr int U = KT == 0 ? 1 : (KT <= 2 ? 4 : (KT <= 4 ? 2 : 1));
  constexpr int KL = KT == 0 ? 1 : KT;  // rows loaded per batch
  for (long long p0 = threadIdx.x; p0 < total; p0 += (long long)blockDim.x * U) {
    float acc[U][8];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[u][q] = 0.f;
    for (int j0 = 0; j0 < k; j0 += KL) {
      uint4 v[U][KL];
      float wv[U][KL];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long p = p0 + (long long)u * blockDim.x;
        const int tok = (int)(p / width), c = c_lo + (int)(p % width);
#pragma unroll
        for (int jj = 0; jj < KL; ++jj) {
          v[u][jj] = make_uint4(0, 0, 0, 0);
          wv[u][jj] = 0.f;
          if (p < total) {
            const int i = tok * k + j0 + jj;
            const int row = row_s[i];
            if (row >= 0) {
              v[u][jj] = __ldg(src_s[slot_s[i]] + (long long)row * cpr + c);
              wv[u][jj] = w_s[i];
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int jj = 0; jj < KL; ++jj) {
          const float wj = wv[u][jj];
          acc[u][0] = fmaf(wj, bf16_lo(v[u][jj].x), acc[u][0]);
          acc[u][1] = fmaf(wj, bf16_hi(v[u][jj].x), acc[u][1]);
          acc[u][2] = fmaf(wj, bf16_lo(v[u][jj].y), acc[u][2]);
          acc[u][3] = fmaf(wj, bf16_hi(v[u][jj].y), acc[u][3]);
          acc[u][4] = fmaf(wj, bf16_lo(v[u][jj].z), acc[u][4]);
          acc[u][5] = fmaf(wj, bf16_hi(v[u][jj].z), acc[u][5]);
          acc[u][6] = fmaf(wj, bf16_lo(v[u][jj].w), acc[u][6]);
          acc[u][7] = fmaf(wj, bf16_hi(v[u][jj].w), acc[u][7]);
        }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long p = p0 + (long long)u * blockDim.x;
      if (p < total) {
        const int tok = (int)(p / width), c = c_lo + (int)(p % width);
        uint4 o;
        o.x = pack_bf16x2(acc[u][0], acc[u][1]);
        o.y = pack_bf16x2(acc[u][2], acc[u][3]);
        o.z = pack_bf16x2(acc[u][4], acc[u][5]);
        o.w = pack_bf16x2(acc[u][6], acc[u][7]);
        out[(long long)(t0 + tok) * cpr + c] = o;
      }
    }
  }
}

// ----------------------------------------------------------------- weight packing
int pack_block(int F) { return (F % 128 == 0) ? 128 : 64; }

__global__ void k_pack_w13(const uint4* __restrict__ w1, const uint4* __restrict__ w3, int n, int F, int H, int B,
                           uint4* __restrict__ w13) {
  const int cpr = H / 8;
  const long long total = (long long)n * 2 * F * cpr;
  for (long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x; p < total;
       p += (long long)gridDim.x * blockDim.x) {
    const int c = (int)(p % cpr);
    const long long r2 = p / cpr;  // row in [n*2F]
    const int ex = (int)(r2 / (2 * F));
    const int r = (int)(r2 % (2 * F));
    const int blk = r / (2 * B), within = r % (2 * B);
    const uint4* src = within < B ? w1 : w3;
    const int srow = blk * B + (within < B ? within : within - B);
    w13[p] = src[((long long)ex * F + srow) * cpr + c];
  }
}

// ----------------------------------------------------------------- launchers
void launch_count(const PlanArgs& a, const int32_t* idx, const PlanBuffers& b, cudaStream_t s) {
  if (a.n_tiles > 0) k_count<<<a.n_tiles, 128, 0, s>>>(a, idx, b);
}
void launch_scan(const PlanArgs& a, const PlanBuffers& b, cudaStream_t s) { k_scan<<<a.V, 1024, 0, s>>>(a, b); }
void launch_layout(const PlanArgs& a, const PlanBuffers& b, int64_t cap_rows, cudaStream_t s) {
  k_layout<<<1, kMaxExperts, 0, s>>>(a, b, (long long)cap_rows);
}
void launch_scatter(const PlanArgs& a, const uint16_t* x, const int32_t* idx, const PlanBuffers& b, int mode,
                    cudaStream_t s, int max_ctas) {
  const size_t smem = sizeof(int) * (kScatterThreads / 32) * a.E;
  int grid = a.n_tiles * ((mode == 6 || mode == 3) ? 1 : a.col_split);
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  if (a.n_tiles > 0) {
    if (mode == 6 || mode == 3) {  // one CTA per token tile (no column slices: no rows are copied)
      PlanArgs a1 = a;
      a1.col_split = 1;
      k_scatter<<<grid, kScatterThreads, smem, s>>>(a1, (const uint4*)x, idx, b, mode);
    } else {
      k_scatter<<<grid, kScatterThreads, smem, s>>>(a, (const uint4*)x, idx, b, mode);
    }
  } else if (a.p2p && (mode == 0 || mode == 5 || mode == 6)) {
    k_signal<<<1, 32, 0, s>>>(a, b, 1);
  }
}
void launch_signal(const PlanArgs& a, const PlanBuffers& b, int which, cudaStream_t s) {
  k_signal<<<1, 32, 0, s>>>(a, b, which);
}
__global__ void k_wait(const unsigned* flags, int n, const unsigned* epoch_ptr, int* err, unsigned long long tmo) {
  wait_flags_geq(flags, n, cur_epoch(epoch_ptr), err, tmo, kWaitFlags);
}
void launch_wait(const unsigned* flags, int n, const unsigned* epoch_ptr, int* err, unsigned long long timeout_ns,
                 cudaStream_t s) {
  k_wait<<<1, 64, 0, s>>>(flags, n, epoch_ptr, err, timeout_ns);
}
void launch_expand_direct(const PlanArgs& a, const PlanBuffers& b, int max_ctas, cudaStream_t s) {
  k_expand_direct<<<max_ctas > 0 ? max_ctas : 32, kScatterThreads, 0, s>>>(a, b);
}
void launch_expand(const PlanArgs& a, const PlanBuffers& b, int max_ctas, cudaStream_t s) {
  k_expand<<<max_ctas > 0 ? max_ctas : 32, kScatterThreads, 0, s>>>(a, b);
}

__global__ void k_expect_nseg(const int32_t* seg_meta, int n, int* err) {
  if (seg_meta[0] != n) atomicOr(err, kErrWeights);
}
void launch_expect_nseg(const int32_t* seg_meta, int n, int* err, cudaStream_t s) {
  k_expect_nseg<<<1, 1, 0, s>>>(seg_meta, n, err);
}
void launch_combine(const PlanArgs& a, const float* w, const PlanBuffers& b, uint16_t* out, cudaStream_t s) {
  if (a.n_tiles <= 0) return;
  auto go = [&](auto kern) { kern<<<a.n_tiles * a.col_split, kScatterThreads, 0, s>>>(a, w, b, (uint4*)out); };
  switch (a.k) {
    case 1: go(k_combine<1>); break;
    case 2: go(k_combine<2>); break;
    case 4: go(k_combine<4>); break;
    case 8: go(k_combine<8>); break;
    default: go(k_combine<0>); break;
  }
}
void launch_pack_w13(const uint16_t* w1, const uint16_t* w3, int n, int F, int H, uint16_t* w13, cudaStream_t s) {
  const long long total = (long long)n * 2 * F * (H / 8);
  int blocks = (int)((total + 255) / 256);
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_pack_w13<<<blocks, 256, 0, s>>>((const uint4*)w1, (const uint4*)w3, n, F, H, pack_block(F), (uint4*)w13);
}

void preload_dispatch_kernels() {
  cudaFuncAttributes fa;
  const void* fs[] = {(const void*)k_count, (const void*)k_scan, (const void*)k_layout, (const void*)k_scatter,
                      (const void*)k_signal, (const void*)k_wait, (const void*)k_expect_nseg,
                      (const void*)k_combine<0>, (const void*)k_combine<1>, (const void*)k_combine<2>,
                      (const void*)k_combine<4>, (const void*)k_combine<8>, (const void*)k_pack_w13,
                      (const void*)k_expand, (const void*)k_expand_direct, (const void*)k_push_tma};
  for (const void* f : fs) {
    cudaFuncGetAttributes(&fa, f);
    // these kernels run next to the persistent GEMM (which holds ~210 KB of shared
    // memory per SM): ask for the max-shared carveout so an SM never has to drain
    // the GEMM to switch its L1/shared split for them
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  }
}

}  // namespace moe
